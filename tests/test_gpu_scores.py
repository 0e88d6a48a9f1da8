"""GPU: dense score helpers (attention.py:120-147, 313-335) vs golden vectors frozen from
the live reference.  Operands come from the bit-exact GPU quantizer / dequantizer; the
dense float64 GEMMs run on the GPU, so agreement is to float64 rounding of the sums."""

import numpy as np
import pytest

from cases import SCORE_CASES
from inputs import randn_bf16

pytestmark = pytest.mark.gpu

FMT = {None: None}


def D():
    import paper_2604_03950_b200 as m

    return m


def pkg_cfg(kw):
    d = D()
    fm = {None: None, "nvfp4": d.NVFP4, "mxfp4": d.MXFP4, "mxfp8_e4m3": d.MXFP8_E4M3, "mxfp8_e5m2": d.MXFP8_E5M2}
    gm = {"token": d.Granularity.TOKEN, "block": d.Granularity.BLOCK, "tensor": d.Granularity.TENSOR}
    kw = dict(kw)
    for key in ("low_format", "high_format"):
        if key in kw:
            kw[key] = fm[kw[key]]
    if "granularity" in kw:
        kw["granularity"] = gm[kw["granularity"]]
    return d.AttentionConfig(**kw)


@pytest.mark.parametrize("case", SCORE_CASES, ids=[c[0] for c in SCORE_CASES])
def test_mixed_precision_scores(golden, case):
    name, lq, d, seed, kw = case
    q, k = randn_bf16(seed, lq, d), randn_bf16(seed + 1, lq, d)
    got = D().mixed_precision_scores(q, k, pkg_cfg(kw))
    assert isinstance(got, np.ndarray) and got.dtype == np.float64
    np.testing.assert_allclose(got, golden[f"scores/{name}"], rtol=1e-10, atol=1e-13)


def test_reference_scores_and_attention(golden):
    import torch

    q, k, v = randn_bf16(31, 96, 64), randn_bf16(32, 96, 64), randn_bf16(33, 96, 64)
    np.testing.assert_allclose(D().reference_scores(q, k, causal=True), golden["refscores_causal"], rtol=1e-10,
                               atol=1e-13)
    np.testing.assert_allclose(D().reference_attention(q, k, v, causal=True), golden["refattn_causal"], rtol=1e-10,
                               atol=1e-13)
    t = D().reference_attention(torch.from_numpy(q), torch.from_numpy(k), torch.from_numpy(v), causal=False)
    assert t.is_cuda
    np.testing.assert_allclose(t.cpu().numpy(), golden["refattn_full"], rtol=1e-10, atol=1e-13)


@pytest.mark.parametrize("case", [0, 1, 2])
def test_score_similarity_tiled_matches_dense(case):
    """score_similarity (row-blocked, no N x N buffers) == similarity of the dense matrices."""
    name, lq, d, seed, kw = SCORE_CASES[case]
    q, k = randn_bf16(seed, lq, d), randn_bf16(seed + 1, lq, d)
    cfg = pkg_cfg(kw)
    dense = D().similarity(D().reference_scores(q, k, causal=cfg.causal), D().mixed_precision_scores(q, k, cfg))
    for rows in (cfg.tile_m, 3 * cfg.tile_m, None):
        tiled = D().score_similarity(q, k, cfg, block_rows=rows)
        for f in ("cos_sim", "rel_l1", "abs_l1", "rmse", "psnr"):
            np.testing.assert_allclose(getattr(tiled, f), getattr(dense, f), rtol=1e-10, err_msg=f)


def test_score_similarity_32k_without_dense_matrices():
    """A c3-length head (N = 32768): the dense path would allocate 2 x 8.6 GB of float64
    scores; the tiled metric stays under 1.5 GB of device memory."""
    import torch

    N, d = 32768, 128
    q, k = randn_bf16(7, N, d), randn_bf16(8, N, d)
    cfg = D().AttentionConfig(tile_m=128, tile_n=128, diag_window=128, sink_window=128)
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    m = D().score_similarity(q, k, cfg)
    peak = torch.cuda.max_memory_allocated() - base
    assert peak < 1.5 * 2**30, peak
    assert 0.9 < m.cos_sim <= 1.0 and 0 < m.rel_l1 < 1 and m.rmse > 0
