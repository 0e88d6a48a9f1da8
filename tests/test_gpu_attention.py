"""GPU: DMA forward parity with the CPU oracle (same AttentionConfig, same inputs).

Two references, two tolerances per PV mode:

* the oracle exactly (``mixed_precision_attention`` of the reference, restated
  in oracle/; P and V stay float64 there, attention.py:174,250):
    pv_mode="bf16"  (P, V in bf16; scores fp32)       rel-L2 <= 4.5e-3, max-abs <= 1e-2
    pv_mode="mxfp8" (P -> E4M3 x2^4, V -> MXFP8/keys) rel-L2 <= 6e-2, max-abs <= 0.4
  (max-abs under MXFP8 PV is dominated by the first causal rows, where one or
  two quantized V rows carry the whole output: |v| ~ 4 x 2^-4 relative step);
* the oracle with the kernel's stated PV quantization applied
  (``pv="bf16"|"mxfp8"``), which isolates what the kernel itself adds
  (fp32 TMEM accumulation, ex2.approx, E4M3 rounding flips of P):
    both PV modes    rel-L2 <= 5e-4, max-abs <= 5e-3
  (first B200 run: rel-L2 1e-7 .. 6e-5, max-abs <= 6.3e-4 over these cases)
"""

import zlib

import numpy as np
import pytest

from conftest import kv_split_of, record_parity
from inputs import randn_bf16
from oracle import mx_oracle as O

pytestmark = pytest.mark.gpu

# vs the oracle = the reference algorithm, from the values measured over the parity suite
# (profiles/r02_parity.jsonl): bf16 PV 2.05e-3 / 7.6e-3 (full-mantissa f64 inputs through the
# INTEGRATION binding; 1.49e-3 / 3.14e-3 for bf16-representable inputs) -> 1.5x, max-abs at the
# survey's 1e-2 cap; MXFP8 PV 3.99e-2 rel-L2 -> 6e-2, max-abs 0.359 (Dv = 128, first causal
# row: one key, so the output IS the MXFP8 V row and its error is E4M3's 2^-4 relative step at
# |v| ~ 5.7) -> 0.4, above the survey's 0.35, which the V quantization alone exceeds
TOL = {"bf16": (4.5e-3, 1e-2), "mxfp8": (6e-2, 0.4)}
TOL_EMU = {"bf16": (5e-4, 5e-3), "mxfp8": (5e-4, 5e-3)}


def D():
    import paper_2604_03950_b200 as m

    return m


def cfgs(low, high, gran, T, S, causal, pv):
    d = D()
    lo = {"nvfp4": (d.NVFP4, O.NVFP4), "mxfp4": (d.MXFP4, O.MXFP4), "mxfp8": (d.MXFP8_E4M3, O.MXFP8_E4M3)}[low]
    hi = {"e4m3": (d.MXFP8_E4M3, O.MXFP8_E4M3), "e5m2": (d.MXFP8_E5M2, O.MXFP8_E5M2)}[high]
    g = {"token": (d.Granularity.TOKEN, "token"), "tensor": (d.Granularity.TENSOR, "tensor")}[gran]
    c = d.AttentionConfig(tile_m=128, tile_n=128, diag_window=T, sink_window=S, causal=causal,
                          low_format=lo[0], high_format=hi[0], granularity=g[0], pv_mode=pv)
    o = O.Cfg(tile_m=128, tile_n=128, diag_window=T, sink_window=S, causal=causal, low_format=lo[1],
              high_format=hi[1], granularity=g[1])
    return c, o


def errs(got, want):
    diff = got - want
    return float(np.linalg.norm(diff) / np.linalg.norm(want)), float(np.abs(diff).max())


CASES = [
    # name, Lq, Lk, d, low, high, gran, T, S, causal
    ("c1_n1024_d64_mxfp4", 1024, 1024, 64, "mxfp4", "e4m3", "token", 128, 128, True),
    ("n1024_d128_nvfp4", 1024, 1024, 128, "nvfp4", "e4m3", "token", 128, 128, True),
    ("n640_d128_mxfp4_T0", 640, 640, 128, "mxfp4", "e4m3", "token", 0, 0, True),
    ("ragged_1000_d128_nvfp4", 1000, 1000, 128, "nvfp4", "e4m3", "token", 256, 128, True),
    ("ragged_200_d64", 200, 200, 64, "nvfp4", "e4m3", "token", 128, 0, True),
    ("noncausal_384x700_d128", 384, 700, 128, "nvfp4", "e4m3", "token", 256, 128, False),
    ("noncausal_256x1024_d64_mx4", 256, 1024, 64, "mxfp4", "e4m3", "token", 128, 128, False),
    ("low8_512_d128", 512, 512, 128, "mxfp8", "e4m3", "token", 0, 0, True),
    ("e5m2_512_d128", 512, 512, 128, "nvfp4", "e5m2", "token", 128, 128, True),
    ("tensor_768_d128", 768, 768, 128, "nvfp4", "e4m3", "tensor", 128, 128, True),
    ("tensor_512_d64_mx4", 512, 512, 64, "mxfp4", "e4m3", "tensor", 0, 128, True),
]


@pytest.mark.parametrize("pv", ["bf16", "mxfp8"])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_attention_vs_oracle(case, pv):
    name, lq, lk, d, low, high, gran, T, S, causal = case
    c, oc = cfgs(low, high, gran, T, S, causal, pv)
    seed = zlib.crc32(name.encode()) % 1000
    q, k, v = randn_bf16(seed, lq, d), randn_bf16(seed + 1, lk, d), randn_bf16(seed + 2, lk, d)
    got = D().mixed_precision_attention(q, k, v, c)
    want = O.mixed_precision_attention(q, k, v, oc)
    assert got.shape == want.shape and got.dtype == np.float64
    emu = O.mixed_precision_attention(q, k, v, oc, pv=pv, kv_split=kv_split_of(c, lq, lk, d, d))
    rel, mx = errs(got, want)
    erel, emx = errs(got, emu)
    print(f"{name} pv={pv}: vs oracle rel_l2={rel:.3e} max_abs={mx:.3e}; "
          f"vs oracle+PV emulation rel_l2={erel:.3e} max_abs={emx:.3e}")
    record_parity(name, pv, rel, mx, erel, emx)
    assert np.isfinite(got).all()
    assert erel <= TOL_EMU[pv][0] and emx <= TOL_EMU[pv][1], (erel, emx)
    assert rel <= TOL[pv][0] and mx <= TOL[pv][1], (rel, mx)


@pytest.mark.parametrize("pv", ["bf16", "mxfp8"])
def test_gqa_batched_torch(pv):
    """c2-shaped GQA (H=8, KVH=2) batched 4-D bf16 path vs per-head oracle."""
    import torch

    B, H, KVH, N, d = 2, 8, 2, 512, 128
    c, oc = cfgs("mxfp4", "e4m3", "token", 128, 128, True, pv)
    g = torch.Generator().manual_seed(3)
    q = torch.randn(B, H, N, d, generator=g).to(torch.bfloat16)
    k = torch.randn(B, KVH, N, d, generator=g).to(torch.bfloat16)
    v = torch.randn(B, KVH, N, d, generator=g).to(torch.bfloat16)
    out = D().dma_attention(q.cuda(), k.cuda(), v.cuda(), c, out_dtype=torch.float32)
    assert out.shape == (B, H, N, d)
    out = out.cpu().double().numpy()
    for b in range(B):
        for h in (0, 3, 5, 7):
            kh = h // (H // KVH)
            want = O.mixed_precision_attention(q[b, h].double().numpy(), k[b, kh].double().numpy(),
                                               v[b, kh].double().numpy(), oc)
            rel, mx = errs(out[b, h], want)
            assert rel <= TOL[pv][0] and mx <= TOL[pv][1], (b, h, rel, mx)


def test_deterministic_and_bf16_out():
    import torch

    c, _ = cfgs("nvfp4", "e4m3", "token", 128, 128, True, "mxfp8")
    g = torch.Generator().manual_seed(5)
    q, k, v = (torch.randn(1, 4, 1024, 128, generator=g).to(torch.bfloat16).cuda() for _ in range(3))
    a = D().dma_attention(q, k, v, c)
    b = D().dma_attention(q, k, v, c)
    assert a.dtype == torch.bfloat16
    assert torch.equal(a, b)


def test_unsupported_configs_raise():
    d = D()
    q = randn_bf16(1, 256, 64)
    with pytest.raises(d._lib.DmaUnsupported):
        d.mixed_precision_attention(q, q, q, d.AttentionConfig(tile_m=32, tile_n=32))  # 32-tiles
    with pytest.raises(ValueError, match="causal"):
        d.mixed_precision_attention(q, q[:128], q[:128], d.AttentionConfig(tile_m=128, tile_n=128))


@pytest.mark.parametrize("chunk", [1, 3])
def test_forward_host_pipeline_matches_device(chunk):
    """DmaAttention on pinned host tensors (chunked H2D / forward / D2H pipeline) gives
    exactly the device-path result, including a ragged last chunk (KVH % chunk != 0)."""
    import torch

    B, H, KVH, N, d = 2, 8, 4, 768, 128
    c, _ = cfgs("nvfp4", "e4m3", "token", 128, 128, True, "mxfp8")
    g = torch.Generator().manual_seed(11)
    q = torch.randn(B, H, N, d, generator=g).to(torch.bfloat16).pin_memory()
    k = torch.randn(B, KVH, N, d, generator=g).to(torch.bfloat16).pin_memory()
    v = torch.randn(B, KVH, N, d, generator=g).to(torch.bfloat16).pin_memory()
    fwd = D().DmaAttention(c)
    out = torch.empty(B, H, N, d, dtype=torch.bfloat16).pin_memory()
    host = fwd.forward_host(q, k, v, out=out, chunk_kv_heads=chunk)  # eager run + CUDA-graph capture
    torch.cuda.synchronize()
    dev = D().DmaAttention(c)(q.cuda(), k.cuda(), v.cuda())
    assert not host.is_cuda and host.shape == (B, H, N, d)
    assert torch.equal(host, dev.cpu())
    out.zero_()
    fwd.forward_host(q, k, v, out=out, chunk_kv_heads=chunk)  # graph replay
    torch.cuda.synchronize()
    assert torch.equal(out, dev.cpu())


# bf16-operand route (BLOCK granularity, None formats): QK on bf16 copies of the
# reference's dequantized operands.  The bf16 rounding (2^-9 relative per operand
# element) is the only addition to the emulation: ~2.5e-3 rel-L2 with bf16 PV; with
# MXFP8 PV it also flips some E4M3 roundings of P (~1-1.4e-2 rel-L2 vs the emulation,
# first B200 run), while the distance to the reference itself stays at the MXFP8-PV level.
DEQ_CASES = [
    # name, Lq, Lk, d, low, high, gran, T, S, causal
    ("block_nvfp4_512_d128", 512, 512, 128, "nvfp4", "e4m3", "block", 128, 128, True),
    ("block_mxfp4_384_d64", 384, 384, 64, "mxfp4", "e4m3", "block", 128, 0, True),
    ("block_noncausal_256x512", 256, 512, 128, "nvfp4", "e4m3", "block", 256, 128, False),
    ("block_low8_256", 256, 256, 128, "mxfp8", "e5m2", "block", 0, 0, True),
    ("ident_low_512_d128", 512, 512, 128, None, "e4m3", "token", 128, 128, True),
    ("ident_high_256_d64", 256, 256, 64, "nvfp4", None, "tensor", 128, 0, True),
    ("ident_both_384", 384, 384, 128, None, None, "token", 0, 0, True),
]
TOL_DEQ = {"bf16": (5e-3, 1e-2), "mxfp8": (6e-2, 0.4)}  # measured 2.92e-3 / 7.0e-3, 3.95e-2 / 0.227
TOL_DEQ_EMU = {"bf16": (1e-2, 5e-2), "mxfp8": (3e-2, 0.15)}


@pytest.mark.parametrize("pv", ["bf16", "mxfp8"])
@pytest.mark.parametrize("case", DEQ_CASES, ids=[c[0] for c in DEQ_CASES])
def test_attention_bf16_operand_route(case, pv):
    name, lq, lk, d, low, high, gran, T, S, causal = case
    m = D()
    lo = {None: (None, None), "nvfp4": (m.NVFP4, O.NVFP4), "mxfp4": (m.MXFP4, O.MXFP4),
          "mxfp8": (m.MXFP8_E4M3, O.MXFP8_E4M3)}[low]
    hi = {None: (None, None), "e4m3": (m.MXFP8_E4M3, O.MXFP8_E4M3), "e5m2": (m.MXFP8_E5M2, O.MXFP8_E5M2)}[high]
    g = {"token": m.Granularity.TOKEN, "block": m.Granularity.BLOCK, "tensor": m.Granularity.TENSOR}[gran]
    c = m.AttentionConfig(tile_m=128, tile_n=128, diag_window=T, sink_window=S, causal=causal, low_format=lo[0],
                          high_format=hi[0], granularity=g, pv_mode=pv)
    oc = O.Cfg(tile_m=128, tile_n=128, diag_window=T, sink_window=S, causal=causal, low_format=lo[1],
               high_format=hi[1], granularity=gran)
    seed = zlib.crc32(name.encode()) % 1000
    q, k, v = randn_bf16(seed, lq, d), randn_bf16(seed + 1, lk, d), randn_bf16(seed + 2, lk, d)
    got = m.mixed_precision_attention(q, k, v, c)
    want = O.mixed_precision_attention(q, k, v, oc)
    emu = O.mixed_precision_attention(q, k, v, oc, pv=pv)
    rel, mx = errs(got, want)
    erel, emx = errs(got, emu)
    print(f"{name} pv={pv}: vs oracle rel_l2={rel:.3e} max_abs={mx:.3e}; vs emulation rel_l2={erel:.3e} "
          f"max_abs={emx:.3e}")
    record_parity(name, pv, rel, mx, erel, emx)
    assert np.isfinite(got).all()
    assert erel <= TOL_DEQ_EMU[pv][0] and emx <= TOL_DEQ_EMU[pv][1], (erel, emx)
    assert rel <= TOL_DEQ[pv][0] and mx <= TOL_DEQ[pv][1], (rel, mx)


# Plan tiles of 64 (the reference's default AttentionConfig): the single-stream kernel walks
# 128 x 128 tiles and masks per 64 x 64 quadrant (Plan2): a key tile whose quadrants mix
# precisions is visited once per precision.  Visit order is key order (not the plan's), so
# the lazy max decisions of the MXFP8-PV emulation can differ; bf16 PV stays tight.
TILE_CASES = [
    # name, Lq, Lk, d, low, tm, tn, T, S, causal
    ("default_cfg_512_d64", 512, 512, 64, "nvfp4", 64, 64, 0, 0, True),
    ("t64_w128_s64_640_d128", 640, 640, 128, "nvfp4", 64, 64, 128, 64, True),
    ("t64x128_w256_384_d128", 384, 384, 128, "mxfp4", 64, 128, 256, 128, True),
    ("t128x64_w64_320_d64", 320, 320, 64, "nvfp4", 128, 64, 64, 64, True),
    ("t64_noncausal_200x448", 200, 448, 128, "nvfp4", 64, 64, 128, 64, False),
]
TOL_TILE_EMU = {"bf16": (2e-3, 5e-3), "mxfp8": (4e-2, 0.15)}


@pytest.mark.parametrize("pv", ["bf16", "mxfp8"])
@pytest.mark.parametrize("case", TILE_CASES, ids=[c[0] for c in TILE_CASES])
def test_attention_plan_tiles_64(case, pv):
    name, lq, lk, d, low, tm, tn, T, S, causal = case
    m = D()
    lo = {"nvfp4": (m.NVFP4, O.NVFP4), "mxfp4": (m.MXFP4, O.MXFP4)}[low]
    c = m.AttentionConfig(tile_m=tm, tile_n=tn, diag_window=T, sink_window=S, causal=causal, low_format=lo[0],
                          pv_mode=pv)
    oc = O.Cfg(tile_m=tm, tile_n=tn, diag_window=T, sink_window=S, causal=causal, low_format=lo[1])
    seed = zlib.crc32(name.encode()) % 1000
    q, k, v = randn_bf16(seed, lq, d), randn_bf16(seed + 1, lk, d), randn_bf16(seed + 2, lk, d)
    got = m.mixed_precision_attention(q, k, v, c)
    want = O.mixed_precision_attention(q, k, v, oc)
    emu = O.mixed_precision_attention(q, k, v, oc, pv=pv)
    rel, mx = errs(got, want)
    erel, emx = errs(got, emu)
    print(f"{name} pv={pv}: vs oracle rel_l2={rel:.3e} max_abs={mx:.3e}; vs emulation rel_l2={erel:.3e} "
          f"max_abs={emx:.3e}")
    record_parity(name, pv, rel, mx, erel, emx)
    assert np.isfinite(got).all()
    assert erel <= TOL_TILE_EMU[pv][0] and emx <= TOL_TILE_EMU[pv][1], (erel, emx)
    assert rel <= TOL[pv][0] and mx <= TOL[pv][1], (rel, mx)


def test_default_config_runs():
    """AttentionConfig() (64 x 64 tiles, no windows: the reference default) is a drop-in call."""
    m = D()
    q, k, v = randn_bf16(5, 256, 64), randn_bf16(6, 256, 64), randn_bf16(7, 256, 64)
    got = m.mixed_precision_attention(q, k, v, m.AttentionConfig())
    want = O.mixed_precision_attention(q, k, v, O.Cfg(tile_m=64, tile_n=64))
    rel, mx = errs(got, want)
    assert rel <= TOL["mxfp8"][0] and mx <= TOL["mxfp8"][1], (rel, mx)


@pytest.mark.parametrize("pv", ["bf16", "mxfp8"])
@pytest.mark.parametrize("d,dv,low,causal", [(128, 64, "nvfp4", True), (64, 128, "mxfp4", True),
                                             (128, 64, "mxfp4", False)])
def test_attention_value_dim_differs(d, dv, low, causal, pv):
    """Dv != d (attention.py:109-119 allows it): V / O carry their own width."""
    c, oc = cfgs(low, "e4m3", "token", 128, 128, causal, pv)
    lq, lk = 384, 384 if causal else 512
    q, k, v = randn_bf16(21, lq, d), randn_bf16(22, lk, d), randn_bf16(23, lk, dv)
    got = D().mixed_precision_attention(q, k, v, c)
    assert got.shape == (lq, dv)
    want = O.mixed_precision_attention(q, k, v, oc)
    emu = O.mixed_precision_attention(q, k, v, oc, pv=pv, kv_split=kv_split_of(c, lq, lk, d, dv))
    rel, mx = errs(got, want)
    erel, emx = errs(got, emu)
    record_parity(f"dv_{d}_{dv}_{low}_{int(causal)}", pv, rel, mx, erel, emx)
    assert erel <= TOL_EMU[pv][0] and emx <= TOL_EMU[pv][1], (erel, emx)
    assert rel <= TOL[pv][0] and mx <= TOL[pv][1], (rel, mx)


def test_empty_inputs_match_reference():
    """attention.py:282-310 on zero-length inputs: no query rows -> an empty result; no keys
    (non-causal) -> every row normalises an l = 0 sum to 0 (checked against the reference)."""
    import torch

    import paper_2604_03950_b200 as m

    cfg = m.AttentionConfig(tile_m=128, tile_n=128, diag_window=128, sink_window=128)
    z = np.zeros((0, 64))
    out = m.mixed_precision_attention(z, z, z, cfg)
    assert out.shape == (0, 64) and out.dtype == np.float64
    nc = m.AttentionConfig(tile_m=128, tile_n=128, diag_window=128, sink_window=128, causal=False)
    out = m.mixed_precision_attention(np.ones((5, 64)), z, z, nc)
    assert out.shape == (5, 64) and not out.any()
    ref = O.mixed_precision_attention(np.ones((5, 64)), z, z, O.Cfg(tile_m=128, tile_n=128, diag_window=128,
                                                                     sink_window=128, causal=False))
    assert np.array_equal(out, ref)
    q = torch.zeros(2, 4, 0, 128, dtype=torch.bfloat16, device="cuda")
    o = m.DmaAttention(cfg)(q, q[:, :2], q[:, :2])
    assert o.shape == (2, 4, 0, 128)
    q = torch.randn(1, 2, 7, 128, device="cuda")
    o = m.DmaAttention(nc)(q, q[:, :, :0], q[:, :, :0])
    assert o.shape == (1, 2, 7, 128) and not o.any()


@pytest.mark.parametrize("pv", ["mxfp8", "bf16"])
def test_full_length_c3_sampled_tiles(pv):
    """BASELINE c3 sequence length (N = 32768, d = 128, NVFP4 + MXFP8, T = S = 128) on 2 heads:
    sampled query tiles (first, sink neighbourhood, middle, last) against the oracle run on the
    same full-length K / V -- the plan, masks and quantization at full size."""
    import torch

    N, d, H = 32768, 128, 2
    c, oc = cfgs("nvfp4", "e4m3", "token", 128, 128, True, pv)
    q, k, v = (randn_bf16(40 + i, H, N, d) for i in range(3))
    got = D().DmaAttention(c)(*(torch.from_numpy(x)[None].cuda() for x in (q, k, v)),
                              out_dtype=torch.float32)[0].double().cpu().numpy()
    tiles = [0, 1, 97, 255]
    for h in range(H):
        want = O.mixed_precision_attention(q[h], k[h], v[h], oc, pv=pv, q_tiles=tiles,
                                           kv_split=kv_split_of(c, N, N, d, d, H=H, KVH=H))
        for t in tiles:
            r = slice(128 * t, 128 * t + 128)
            rel, mx = errs(got[h, r], want[r])
            record_parity(f"c3_sampled_h{h}_t{t}", pv, None, None, rel, mx)
            assert rel <= TOL_EMU[pv][0] and mx <= TOL_EMU[pv][1], (pv, h, t, rel, mx)


@pytest.mark.parametrize("pv", ["mxfp8", "bf16"])
def test_float32_inputs_full_mantissa(pv):
    """f32 Q/K/V with full-width mantissas (phase 1 quantizes them bit-exactly from f32; V
    enters PV as MXFP8 or bf16 of the f32 values) against the oracle on the same values."""
    import torch

    rng = np.random.default_rng(21)
    H, N, d = 2, 640, 128
    q, k, v = (rng.standard_normal((H, N, d)).astype(np.float32) for _ in range(3))
    c, oc = cfgs("nvfp4", "e4m3", "token", 128, 128, True, pv)
    got = D().DmaAttention(c)(*(torch.from_numpy(x)[None].cuda() for x in (q, k, v)),
                              out_dtype=torch.float32)[0].double().cpu().numpy()
    for h in range(H):
        want = O.mixed_precision_attention(q[h].astype(np.float64), k[h].astype(np.float64),
                                           v[h].astype(np.float64), oc, pv=pv,
                                           kv_split=kv_split_of(c, N, N, d, d, H=H, KVH=H))
        rel, mx = errs(got[h], want)
        assert rel <= TOL_EMU[pv][0] and mx <= TOL_EMU[pv][1], (pv, h, rel, mx)
