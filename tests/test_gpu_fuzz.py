"""GPU: seeded random configurations (shapes, formats, tiles, windows, GQA, causality) for the
prefill forward and the decode path, each against the oracle.  Complements the hand-picked
cases in test_gpu_attention.py / test_gpu_decode.py with combinations nobody picked."""

import numpy as np
import pytest
import torch

from conftest import kv_split_of
from inputs import randn_bf16
from oracle import mx_oracle as O

pytestmark = pytest.mark.gpu

TOL_EMU = {"bf16": (5e-4, 5e-3), "mxfp8": (5e-4, 5e-3)}  # test_gpu_attention.py
TOL_TILE64 = {"bf16": (2e-3, 5e-3), "mxfp8": (4e-2, 0.15)}  # 64-tiles: order-dependent emulation
TOL_DECODE = (2e-5, 2e-4)  # test_gpu_decode.py


def D():
    import paper_2604_03950_b200 as m

    return m


def fmts(m, low, high):
    lo = {"nvfp4": (m.NVFP4, O.NVFP4), "mxfp4": (m.MXFP4, O.MXFP4), "mxfp8": (m.MXFP8_E4M3, O.MXFP8_E4M3)}[low]
    hi = {"e4m3": (m.MXFP8_E4M3, O.MXFP8_E4M3), "e5m2": (m.MXFP8_E5M2, O.MXFP8_E5M2)}[high]
    return lo, hi


def prefill_case(seed):
    r = np.random.default_rng(seed)
    tile = int(r.choice([64, 128]))
    causal = bool(r.random() < 0.7)
    lq = int(r.integers(1, 700))
    lk = lq if causal else int(r.integers(1, 700))
    d = int(r.choice([64, 128]))
    dv = int(r.choice([64, 128]))
    T = tile * int(r.integers(0, 4))
    S = tile * int(r.integers(0, 3))
    low = str(r.choice(["nvfp4", "mxfp4", "mxfp8"]))
    high = str(r.choice(["e4m3", "e5m2"]))
    gran = str(r.choice(["token", "tensor"]))
    pv = str(r.choice(["bf16", "mxfp8"]))
    return tile, causal, lq, lk, d, dv, T, S, low, high, gran, pv


@pytest.mark.parametrize("seed", range(40))
def test_prefill_fuzz(seed):
    m = D()
    tile, causal, lq, lk, d, dv, T, S, low, high, gran, pv = prefill_case(seed)
    (lo_m, lo_o), (hi_m, hi_o) = fmts(m, low, high)
    g = {"token": m.Granularity.TOKEN, "tensor": m.Granularity.TENSOR}[gran]
    cfg = m.AttentionConfig(tile_m=tile, tile_n=tile, diag_window=T, sink_window=S, causal=causal, low_format=lo_m,
                            high_format=hi_m, granularity=g, pv_mode=pv)
    ocfg = O.Cfg(tile_m=tile, tile_n=tile, diag_window=T, sink_window=S, causal=causal, low_format=lo_o,
                 high_format=hi_o, granularity=gran)
    q, k, v = randn_bf16(seed, lq, d), randn_bf16(seed + 100, lk, d), randn_bf16(seed + 200, lk, dv)
    got = m.mixed_precision_attention(q, k, v, cfg)
    want = O.mixed_precision_attention(q, k, v, ocfg, pv=pv, kv_split=kv_split_of(cfg, lq, lk, d, dv))
    tol = TOL_EMU[pv] if tile == 128 else TOL_TILE64[pv]
    err = np.abs(got - want)
    rel = float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30))
    assert rel <= tol[0] and float(err.max()) <= tol[1], (prefill_case(seed), rel, float(err.max()))


@pytest.mark.parametrize("seed", range(24))
def test_decode_fuzz(seed):
    m = D()
    r = np.random.default_rng(1000 + seed)
    tile_m = int(r.choice([32, 64, 128]))
    tile_n = int(r.choice([32, 64, 128]))
    L = int(r.integers(40, 900))
    nq = int(r.integers(1, 5))
    kvh = int(r.choice([1, 2]))
    G = int(r.choice([1, 2, 4, 8]))
    d = int(r.choice([64, 128]))
    dv = int(r.choice([64, 128]))
    T, S = tile_n * int(r.integers(0, 3)), tile_n * int(r.integers(0, 2))
    low, high = str(r.choice(["nvfp4", "mxfp4", "mxfp8"])), str(r.choice(["e4m3", "e5m2"]))
    (lo_m, lo_o), (hi_m, hi_o) = fmts(m, low, high)
    H = kvh * G
    q, k, v = randn_bf16(seed, H, L, d), randn_bf16(seed + 1, kvh, L, d), randn_bf16(seed + 2, kvh, L, dv)
    cfg = m.AttentionConfig(tile_m=tile_m, tile_n=tile_n, diag_window=T, sink_window=S, low_format=lo_m,
                            high_format=hi_m)
    cache = m.DmaKVCache(cfg, batch=1, kv_heads=kvh, capacity=L, head_dim=d, v_dim=dv)
    kt, vt = torch.from_numpy(k).cuda()[None], torch.from_numpy(v).cuda()[None]
    cache.append(kt[:, :, :L - nq], vt[:, :, :L - nq])
    got = cache.step(torch.from_numpy(q[:, L - nq:]).cuda()[None], kt[:, :, L - nq:], vt[:, :, L - nq:])
    got = got[0].double().cpu().numpy()
    ocfg = O.Cfg(tile_m=tile_m, tile_n=tile_n, diag_window=T, sink_window=S, causal=True, low_format=lo_o,
                 high_format=hi_o, granularity=O.TOKEN)
    for h in range(H):
        want = O.mixed_precision_attention(q[h], k[h // G], v[h // G], ocfg)[L - nq:]
        rel = np.linalg.norm(got[h] - want) / np.linalg.norm(want)
        assert rel <= TOL_DECODE[0] and np.abs(got[h] - want).max() <= TOL_DECODE[1], (seed, h, rel)


TOL_DEQ_EMU = {"bf16": (1e-2, 5e-2), "mxfp8": (3e-2, 0.15)}  # test_gpu_attention.py (bf16 operand route)


@pytest.mark.parametrize("seed", range(16))
def test_bf16_operand_route_fuzz(seed):
    """BLOCK granularity and None (identity) formats: phase 1 dequantizes the bit-exact
    quantize_dual operands to bf16 and QK runs with kind::f16 (extra error: bf16 rounding)."""
    m = D()
    r = np.random.default_rng(5000 + seed)
    tile = int(r.choice([64, 128]))
    causal = bool(r.random() < 0.7)
    lq = int(r.integers(1, 600))
    lk = lq if causal else int(r.integers(1, 600))
    d = int(r.choice([64, 128]))
    T, S = tile * int(r.integers(0, 3)), tile * int(r.integers(0, 2))
    pv = str(r.choice(["bf16", "mxfp8"]))
    mode = str(r.choice(["block", "identity"]))
    if mode == "block":
        low = str(r.choice(["nvfp4", "mxfp4"]))
        (lo_m, lo_o), (hi_m, hi_o) = fmts(m, low, "e4m3")
        g_m, g_o = m.Granularity.BLOCK, "block"
    else:
        lo_m = lo_o = hi_m = hi_o = None
        g_m, g_o = m.Granularity.TOKEN, "token"
    cfg = m.AttentionConfig(tile_m=tile, tile_n=tile, diag_window=T, sink_window=S, causal=causal, low_format=lo_m,
                            high_format=hi_m, granularity=g_m, pv_mode=pv)
    ocfg = O.Cfg(tile_m=tile, tile_n=tile, diag_window=T, sink_window=S, causal=causal, low_format=lo_o,
                 high_format=hi_o, granularity=g_o)
    q, k, v = randn_bf16(seed, lq, d), randn_bf16(seed + 100, lk, d), randn_bf16(seed + 200, lk, d)
    got = m.mixed_precision_attention(q, k, v, cfg)
    want = O.mixed_precision_attention(q, k, v, ocfg, pv=pv)
    rel = float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30))
    mx = float(np.abs(got - want).max())
    # 64-tile plans: the kernel walks 128 x 128 tiles (per-quadrant masks), so its lazy MXFP8-PV
    # rescale points differ from the emulation's 64-tile walk (see TOL_TILE64)
    tol = TOL_DEQ_EMU[pv] if tile == 128 or pv == "bf16" else tuple(max(a, b) for a, b in
                                                                     zip(TOL_DEQ_EMU[pv], TOL_TILE64[pv]))
    assert rel <= tol[0] and mx <= tol[1], (seed, mode, tile, causal, lq, lk, d, pv, rel, mx)
