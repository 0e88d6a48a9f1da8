"""GPU: harness sweeps (SPEC.md:364-373 and acceptance criteria 5, 6, 9) through the
fused forward and the GPU score helpers.  The trend checks use attention scores
(Table 2 measures scores) on the seeded Gaussian inputs; the orderings were
checked against the oracle restatement on the same inputs (cos_sim per seed:
MXFP8 0.9993 > NVFP4 0.9967 > MXFP4 0.9952 at T = S = 0; NVFP4 0.9967 -> 0.9985
-> 0.9993 for T = S = 0, 128, 2048).  The SPEC's absolute bands (MXFP4 < 0.95)
came from model tensors and do not hold for Gaussian inputs; the per-granularity
ordering (criterion 7) does not hold on them either (token 0.9967, block 0.9966,
tensor 0.9968 on seed 1), so neither is asserted."""

import json

import numpy as np
import pytest

from paper_2604_03950_b200 import harness as H

pytestmark = pytest.mark.gpu


def _cos(rows, **sel):
    return [r["cos_sim"] for r in rows if all(r[k] == v for k, v in sel.items())]


def test_report_completeness_and_determinism(tmp_path):
    cfg = H.RunConfig(seq_len=384, head_dim=64, heads=2, seed=0, formats=["nvfp4", "mxfp8"], diag=[0, 128],
                      sink=[128], granularity=["token", "tensor"])
    rows = H.run_experiment(cfg)
    assert len(rows) == len(cfg.points()) * cfg.heads == 16
    assert [(r["format"], r["diag_window"], r["granularity"], r["head"]) for r in rows[:3]] == \
        [("nvfp4", 0, "token", 0), ("nvfp4", 0, "token", 1), ("nvfp4", 0, "tensor", 0)]
    for r in rows:
        assert 0.98 < r["cos_sim"] <= 1.0 and r["rel_l1"] > 0 and np.isfinite(r["psnr"])
    out1, out2 = tmp_path / "a.json", tmp_path / "b.json"
    assert H.main(["--seq-len", "384", "--head-dim", "64", "--heads", "2", "--format", "nvfp4", "mxfp8",
                   "--diag", "0", "128", "--out", str(out1)]) == 0
    assert H.main(["--seq-len", "384", "--head-dim", "64", "--heads", "2", "--format", "nvfp4", "mxfp8",
                   "--diag", "0", "128", "--out", str(out2)]) == 0
    assert out1.read_bytes() == out2.read_bytes()  # criterion 9: byte-identical reports
    assert len(json.loads(out1.read_text())) == 2 * 2 * 2


def test_identity_passthrough_is_exact_up_to_bf16():
    rows = H.run_experiment(H.RunConfig(seq_len=256, head_dim=64, heads=1, seed=0, formats=["identity"],
                                        diag=[0], sink=[0], pv_mode="bf16"))
    assert rows[0]["cos_sim"] > 0.99999  # bf16 operands / bf16 PV on the tensor cores


def test_format_ordering_on_scores():
    for seed in range(3):
        rows = H.run_experiment(H.RunConfig(seq_len=1024, head_dim=64, heads=1, seed=seed, target="scores",
                                            formats=["mxfp8", "nvfp4", "mxfp4"], diag=[0], sink=[0]))
        c8, c4n, c4m = (_cos(rows, format=f)[0] for f in ("mxfp8", "nvfp4", "mxfp4"))
        assert c8 > c4n > c4m, (seed, c8, c4n, c4m)
        assert c8 > 0.97


def test_diagonal_window_benefit():
    for seed in range(3):
        cfg = H.RunConfig(seq_len=1024, head_dim=64, heads=1, seed=seed, target="scores", formats=["nvfp4"],
                          diag=[0, 128, 2048], sink=[0, 128, 2048])
        rows = H.run_experiment(cfg)
        pick = {(r["diag_window"], r["sink_window"]): r for r in rows}
        a, b, c = pick[(0, 0)], pick[(128, 128)], pick[(2048, 2048)]
        assert b["cos_sim"] > a["cos_sim"] and b["rel_l1"] < a["rel_l1"]
        assert c["cos_sim"] >= b["cos_sim"]
        assert a["high_precision_pct"] < b["high_precision_pct"] < c["high_precision_pct"] == 100.0


def test_scores_target_matches_oracle_values():
    """One sweep point on scores equals the oracle restatement (same bit-exact quantizer,
    float64 GEMMs on both sides)."""
    import os
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import mx_oracle as O

    cfg = H.RunConfig(seq_len=256, head_dim=64, heads=1, seed=5, target="scores", formats=["mxfp4"], diag=[128],
                      sink=[0])
    got = H.run_experiment(cfg)[0]
    q, k, _ = H.generate_tensors(256, 256, 64, 1, 5)
    q, k = q[0].astype(np.float64), k[0].astype(np.float64)
    ocfg = O.Cfg(tile_m=128, tile_n=128, diag_window=128, sink_window=0, causal=True, low_format=O.MXFP4,
                 high_format=O.MXFP8_E4M3, granularity=O.TOKEN)
    want = O.similarity(O.reference_scores(q, k, causal=True), O.mixed_precision_scores(q, k, ocfg))
    assert abs(got["cos_sim"] - want["cos_sim"]) < 1e-12
    assert abs(got["rel_l1"] - want["rel_l1"]) < 1e-9 * want["rel_l1"]


def test_tensor_file_input_equals_generated(tmp_path):
    q, k, v = H.generate_tensors(256, 256, 64, 2, 3)
    paths = []
    for n, x in zip("qkv", (q, k, v)):
        p = str(tmp_path / f"{n}.mxt")
        H.write_tensor(p, x)
        paths.append(p)
    base = dict(formats=["nvfp4"], diag=[128], sink=[128])
    from_files = H.run_experiment(H.RunConfig(q_path=paths[0], k_path=paths[1], v_path=paths[2], **base))
    generated = H.run_experiment(H.RunConfig(seq_len=256, head_dim=64, heads=2, seed=3, **base))
    for a, b in zip(from_files, generated):
        assert a["cos_sim"] == b["cos_sim"] and a["seed"] is None and b["seed"] == 3
