"""GPU: parity at every BASELINE.json configuration's real shape (attention.py:282-310,
quantize.py:122-212), on sampled query tiles against the CPU oracle run over the SAME
full-length K / V (plans, masks, quantization and indexing at full size):

* c2  B1 H32 KVH8 N8192 d128, MXFP8 diag/sink 128 + MXFP4 (GQA: heads of 4 KV groups);
* c3  B1 H32 N32768 (tests/test_gpu_attention.py::test_full_length_c3_sampled_tiles);
* c4  N16384 d128 NVFP4, window T = S in {0, 128, 2048} x granularity {TOKEN, TENSOR, BLOCK};
* c5  N131072 d128 NVFP4 (the metric's top length), 2 heads; and the full B8 H64 c5 shape
      once (8.6e9 elements per tensor: 64-bit offsets everywhere), checked on heads at the
      far end of the flattened (b, h) range.

Every case asserts against the oracle with the kernel's stated PV quantization
(TOL_EMU, what the kernel itself adds) and against the reference algorithm itself
(TOL, the drop-in error); the measured values are logged (conftest.record_parity)."""

import numpy as np
import pytest

from conftest import kv_split_of, record_parity
from inputs import randn_bf16
from oracle import mx_oracle as O
from test_gpu_attention import TOL, TOL_DEQ, TOL_DEQ_EMU, TOL_EMU, errs

pytestmark = pytest.mark.gpu


def _D():
    import paper_2604_03950_b200 as m

    return m


def _cfgs(low, gran, T, S, pv):
    m = _D()
    lo = {"nvfp4": (m.NVFP4, O.NVFP4), "mxfp4": (m.MXFP4, O.MXFP4)}[low]
    g = {"token": m.Granularity.TOKEN, "tensor": m.Granularity.TENSOR, "block": m.Granularity.BLOCK}[gran]
    c = m.AttentionConfig(tile_m=128, tile_n=128, diag_window=T, sink_window=S, causal=True, low_format=lo[0],
                          high_format=m.MXFP8_E4M3, granularity=g, pv_mode=pv)
    oc = O.Cfg(tile_m=128, tile_n=128, diag_window=T, sink_window=S, causal=True, low_format=lo[1],
               high_format=O.MXFP8_E4M3, granularity=gran)
    return c, oc


def _check_tiles(name, pv, got_head, q, k, v, oc, tiles, tol, tol_emu, kv_split=1):
    """got_head [N, DV] (f64) vs the oracle (pv f64 = the reference) and its PV emulation
    (with the forward's KV split count: small problems split each tile plan)."""
    want = O.mixed_precision_attention(q, k, v, oc, q_tiles=tiles)
    emu = O.mixed_precision_attention(q, k, v, oc, pv=pv, q_tiles=tiles, kv_split=kv_split)
    rows = np.concatenate([np.arange(128 * t, min(128 * t + 128, q.shape[0])) for t in tiles])
    rel, mx = errs(got_head[rows], want[rows])
    erel, emx = errs(got_head[rows], emu[rows])
    record_parity(name, pv, rel, mx, erel, emx, tiles=list(tiles))
    assert np.isfinite(got_head[rows]).all()
    assert erel <= tol_emu[0] and emx <= tol_emu[1], (name, erel, emx)
    assert rel <= tol[0] and mx <= tol[1], (name, rel, mx)


@pytest.mark.parametrize("pv", ["mxfp8", "bf16"])
def test_c2_full_shape(pv):
    import torch

    B, H, KVH, N, d = 1, 32, 8, 8192, 128
    c, oc = _cfgs("mxfp4", "token", 128, 128, pv)
    g = torch.Generator().manual_seed(2)
    q = torch.randn(B, H, N, d, generator=g).to(torch.bfloat16)
    k = torch.randn(B, KVH, N, d, generator=g).to(torch.bfloat16)
    v = torch.randn(B, KVH, N, d, generator=g).to(torch.bfloat16)
    out = _D().DmaAttention(c)(q.cuda(), k.cuda(), v.cuda(), out_dtype=torch.float32)[0].double().cpu().numpy()
    tiles = [0, 1, 33, 63]
    for h in (0, 5, 14, 31):  # KV groups 0, 1, 3, 7
        kh = h // (H // KVH)
        _check_tiles(f"c2_h{h}", pv, out[h], q[0, h].double().numpy(), k[0, kh].double().numpy(),
                     v[0, kh].double().numpy(), oc, tiles, TOL[pv], TOL_EMU[pv])


C4 = [(T, gran) for T in (0, 128, 2048) for gran in ("token", "tensor", "block")]


@pytest.mark.parametrize("T,gran", C4, ids=[f"T{T}_{g}" for T, g in C4])
def test_c4_window_granularity_sweep(T, gran):
    """c4: N = 16384, d = 128, NVFP4 off-diagonal, T = S; BLOCK runs on the bf16-operand route."""
    import torch

    pv = "mxfp8"
    N, d, H = 16384, 128, 2
    c, oc = _cfgs("nvfp4", gran, T, T, pv)
    q, k, v = (randn_bf16(70 + i, H, N, d) for i in range(3))
    got = _D().DmaAttention(c)(*(torch.from_numpy(x)[None].cuda() for x in (q, k, v)),
                               out_dtype=torch.float32)[0].double().cpu().numpy()
    tol, tol_emu = (TOL_DEQ[pv], TOL_DEQ_EMU[pv]) if gran == "block" else (TOL[pv], TOL_EMU[pv])
    ks = kv_split_of(c, N, N, d, d, H=H, KVH=H)
    for h in range(H):
        _check_tiles(f"c4_T{T}_{gran}_h{h}", pv, got[h], q[h], k[h], v[h], oc, [0, 1, 17, 64, 127], tol, tol_emu,
                     kv_split=ks)


@pytest.mark.parametrize("pv", ["mxfp8", "bf16"])
def test_c5_length_two_heads(pv):
    """N = 131072 (BASELINE c5 / the metric's top length), 2 heads."""
    import torch

    N, d, H = 131072, 128, 2
    c, oc = _cfgs("nvfp4", "token", 128, 128, pv)
    q, k, v = (randn_bf16(90 + i, H, N, d) for i in range(3))
    got = _D().DmaAttention(c)(*(torch.from_numpy(x)[None].cuda() for x in (q, k, v)),
                               out_dtype=torch.float32)[0].double().cpu().numpy()
    for h in range(H):
        _check_tiles(f"c5_N131072_h{h}", pv, got[h], q[h], k[h], v[h], oc, [0, 1, 500, 1023], TOL[pv], TOL_EMU[pv])


def test_c5_full_batch_shape():
    """The whole c5 problem on one B200: B8 H64 N131072 d128 (3 x 17.2 GB of bf16 inputs,
    34 GB f32 O, ~35 GB of operands), both PV modes on the same inputs.  Element offsets pass
    2^32; the first (b, h) head and the last two are checked on sampled tiles against the
    oracle (every head's result is computed before any is checked)."""
    import torch

    B, H, N, d = 8, 64, 131072, 128
    free, _ = torch.cuda.mem_get_info()
    if free < 130 * 2**30:
        pytest.skip(f"needs ~125 GB free device memory, {free / 2**30:.0f} GB free")
    g = torch.Generator(device="cuda").manual_seed(5)
    q, k, v = (torch.randn(B, H, N, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    heads = ((0, 0), (7, 62), (7, 63))
    got = {}
    for pv in ("mxfp8", "bf16"):
        c, _ = _cfgs("nvfp4", "token", 128, 128, pv)
        out = _D().DmaAttention(c)(q, k, v, out_dtype=torch.float32)  # f32 O: no bf16 rounding in the check
        torch.cuda.synchronize()
        for b, h in heads:
            got[(pv, b, h)] = out[b, h].double().cpu().numpy()
        del out
        torch.cuda.empty_cache()
    xs = {(b, h): [t[b, h].double().cpu().numpy() for t in (q, k, v)] for b, h in heads}
    del q, k, v
    torch.cuda.empty_cache()
    for pv in ("mxfp8", "bf16"):
        _, oc = _cfgs("nvfp4", "token", 128, 128, pv)
        for b, h in heads:
            _check_tiles(f"c5_full_b{b}_h{h}", pv, got[(pv, b, h)], *xs[(b, h)], oc, [0, 3, 1023], TOL[pv],
                         TOL_EMU[pv])
