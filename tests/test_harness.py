"""CPU: the experiment harness's host side -- MXT1 tensor files,
the seeded generator, sweep configuration and report formatting.  The sweeps
themselves run on the GPU (tests/test_gpu_harness.py)."""

import hashlib
import json
import struct

import numpy as np
import pytest

from paper_2604_03950_b200 import harness as H

# seed=42, L=8, D=4 (one head): SHA-256 of the Q, K, V float32 bytes, frozen at first
# generation ("golden checksum recorded at first generation")
GOLDEN_SEED42 = "5f1661b8f010a29bdfca401221b179e25362deaf7d01e7be0a04f51e850dd621"


def test_generator_golden_and_determinism():
    q, k, v = H.generate_tensors(8, 8, 4, 1, 42)
    assert q.shape == k.shape == v.shape == (1, 8, 4) and q.dtype == np.float32
    assert hashlib.sha256(q.tobytes() + k.tobytes() + v.tobytes()).hexdigest() == GOLDEN_SEED42
    again = H.generate_tensors(8, 8, 4, 1, 42)
    assert all(np.array_equal(a, b) for a, b in zip((q, k, v), again))
    other = H.generate_tensors(8, 8, 4, 1, 43)
    assert not np.array_equal(q, other[0])
    assert not np.array_equal(q, k) and not np.array_equal(k, v)


def test_generator_moments_and_stddev():
    q, k, _ = H.generate_tensors(2048, 1024, 64, 2, 0, stddev=0.5)
    assert q.shape == (2, 2048, 64) and k.shape == (2, 1024, 64)
    assert abs(float(q.mean())) < 0.01 and abs(float(q.std()) - 0.5) < 0.01
    with pytest.raises(ValueError, match="positive"):
        H.generate_tensors(0, 8, 4, 1, 0)


def test_mxt1_round_trip(tmp_path):
    for shape in [(5,), (3, 7), (2, 9, 32)]:
        x = np.random.default_rng(0).standard_normal(shape)
        p = str(tmp_path / f"t{len(shape)}.mxt")
        H.write_tensor(p, x)
        raw = open(p, "rb").read()
        assert raw[:4] == b"MXT1" and struct.unpack_from("<II", raw, 4) == (0, len(shape))
        assert struct.unpack_from(f"<{len(shape)}I", raw, 12) == shape
        assert len(raw) == 12 + 4 * len(shape) + 4 * x.size
        y = H.read_tensor(p)
        assert y.dtype == np.float32 and np.array_equal(y, x.astype(np.float32))


def test_mxt1_errors_name_path_and_field(tmp_path):
    good = tmp_path / "g.mxt"
    H.write_tensor(str(good), np.ones((2, 3)))
    raw = good.read_bytes()
    cases = {
        "magic": b"MXT2" + raw[4:],
        "dtype": raw[:4] + struct.pack("<I", 3) + raw[8:],
        "payload": raw[:-4],
        "header": raw[:6],
    }
    for field, data in cases.items():
        p = tmp_path / f"bad_{field}.mxt"
        p.write_bytes(data)
        with pytest.raises(H.TensorFileError, match=field) as e:
            H.read_tensor(str(p))
        assert str(p) in str(e.value)
    with pytest.raises(FileNotFoundError, match="missing.mxt"):
        H.read_tensor(str(tmp_path / "missing.mxt"))


def test_file_inputs_shape_checks(tmp_path):
    paths = {n: str(tmp_path / f"{n}.mxt") for n in "qkv"}
    H.write_tensor(paths["q"], np.zeros((2, 16, 32)))
    H.write_tensor(paths["k"], np.zeros((2, 16, 32)))
    H.write_tensor(paths["v"], np.zeros((2, 12, 32)))
    cfg = H.RunConfig(q_path=paths["q"], k_path=paths["k"], v_path=paths["v"])
    with pytest.raises(H.TensorFileError, match="v.mxt"):
        H.load_inputs(cfg)
    H.write_tensor(paths["v"], np.zeros((16, 32)))
    with pytest.raises(H.TensorFileError, match="heads"):
        H.load_inputs(cfg)
    H.write_tensor(paths["v"], np.ones((2, 16, 32)))
    q, k, v = H.load_inputs(cfg)
    assert q.shape == (2, 16, 32) and float(v.sum()) == 2 * 16 * 32


def test_run_config_and_cli_parsing():
    cfg = H.parse_args(["--seq-len", "256", "--head-dim", "64", "--heads", "3", "--format", "mxfp8", "nvfp4",
                        "--diag", "0", "128", "--sink", "0", "--granularity", "token", "block", "--non-causal",
                        "--report", "csv", "--target", "scores"])
    assert (cfg.seq_len, cfg.head_dim, cfg.heads, cfg.causal, cfg.report) == (256, 64, 3, False, "csv")
    pts = cfg.points()
    assert len(pts) == 2 * 2 * 1 * 2 and pts[0] == ("mxfp8", 0, 0, "token") and pts[-1] == ("nvfp4", 128, 0, "block")
    with pytest.raises(ValueError, match="--q, --k and --v"):
        H.RunConfig(q_path="a").validate()
    with pytest.raises(ValueError, match="format"):
        H.RunConfig(formats=["fp16"]).validate()
    with pytest.raises(SystemExit):
        H.parse_args(["--granularity", "row"])
    a = H.attention_config(cfg, "identity", 128, 0, "tensor")
    assert a.low_format is None and a.high_format is None and a.diag_window == 128 and not a.causal


def test_report_formats_are_deterministic():
    rows = [{"cos_sim": 0.1 + 0.2, "rel_l1": 1e-17, "psnr": float("inf"), "format": "nvfp4", "head": h}
            for h in range(3)]
    j = H.format_report(rows, "json")
    assert j == H.format_report([dict(r) for r in rows], "json")
    back = json.loads(j)
    assert isinstance(back, list) and len(back) == 3 and back[0]["cos_sim"] == 0.1 + 0.2
    c = H.format_report(rows, "csv").splitlines()
    assert c[0] == "cos_sim,rel_l1,psnr,format,head" and len(c) == 4
