import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    return np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))


def record_parity(case, pv, rel, mx, erel=None, emx=None, **extra):
    """Append one measured parity row (vs the oracle / vs the oracle + PV emulation) to
    gpurun_out/parity_<pid>.jsonl when DMA_PARITY_LOG is set (profiles/r02_parity.jsonl is
    the committed collection of these rows)."""
    if not os.environ.get("DMA_PARITY_LOG"):
        return
    import json

    d = os.path.join(ROOT, "gpurun_out")
    os.makedirs(d, exist_ok=True)
    row = {"case": case, "pv": pv, "rel_l2_vs_oracle": rel, "max_abs_vs_oracle": mx,
           "rel_l2_vs_emulation": erel, "max_abs_vs_emulation": emx, **extra}
    with open(os.path.join(d, f"parity_{os.getpid()}.jsonl"), "a") as f:
        f.write(json.dumps(row) + "\n")


def kv_split_of(cfg, lq, lk, d, dv, B=1, H=1, KVH=1):
    """The KV split count the forward uses for this problem (1 = unsplit): small problems
    cut each query tile's plan into ranges merged in the kernel, and the oracle's PV
    emulation must restart its lazy max / P quantization at the same range boundaries
    (mx_oracle.mixed_precision_attention(..., kv_split=n))."""
    import paper_2604_03950_b200 as m

    return m.attention.kv_split_count((B, H, lq, d), (B, KVH, lk, d), (B, KVH, lk, dv), cfg)
