"""bench.py launcher plumbing on CPU: ``--gpus 2`` outside torchrun re-launches itself as
two ranks (gloo in ``--dry`` mode, the same shard plan / barrier / max-over-ranks / gather
code as the NCCL run) and rank 0 prints one JSON line; the reference arm runs the
unmodified reference (baseline/_ref) or the oracle port on the host cores."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=240):
    env = dict(os.environ)
    for var in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(var, None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("gpus", [1, 2])
def test_bench_self_launches_ranks(gpus):
    d = _run("--dry", "--gpus", str(gpus), "--steps", "2", "--warmup", "1")
    assert d["n_gpus"] == gpus and d["dry"] and d["gather_ok"]
    assert d["steps"] == 2 and d["warmup"] == 3  # W >= 3 enforced


def test_bench_reference_arm_line():
    d = _run("--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "1")
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "TFLOPS"
    assert d["config"]["workload"] == "c1" and d["steps"] == 2
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
