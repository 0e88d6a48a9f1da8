"""GPU: decode over the MX key cache (decode.cuh, SURVEY §8 f rank 4) vs the oracle.

Query i at position p = pos + i must equal row p of the oracle's
``mixed_precision_attention`` (pv="f64", i.e. the reference, attention.py:282-310)
over the whole sequence.  Decode keeps P and V unquantized (f32 / bf16), so the only
differences are f32 sums of exact block-scaled products, the f32 S_q product and the
f32 softmax: TOL_DECODE = rel-L2 <= 2e-5, max-abs <= 2e-4 (outputs are O(1))."""

import numpy as np
import pytest
import torch

from inputs import randn_bf16
from oracle import mx_oracle as O

pytestmark = pytest.mark.gpu

TOL_DECODE = (2e-5, 2e-4)


def D():
    import paper_2604_03950_b200 as m

    return m


FMT = {"nvfp4": ("NVFP4", "NVFP4"), "mxfp4": ("MXFP4", "MXFP4"), "mxfp8": ("MXFP8_E4M3", "MXFP8_E4M3"),
       "e5m2": ("MXFP8_E5M2", "MXFP8_E5M2")}

# (name, L, n_q, H, KVH, d, dv, tile_m, tile_n, T, S, low, high)
CASES = [
    ("nv_d128_T128", 700, 1, 2, 2, 128, 128, 128, 128, 128, 128, "nvfp4", "mxfp8"),
    ("nv_gqa4_nq3", 515, 3, 8, 2, 128, 128, 128, 128, 256, 0, "nvfp4", "mxfp8"),
    ("mx4_d64_t64", 333, 2, 4, 1, 64, 64, 64, 64, 64, 64, "mxfp4", "mxfp8"),
    ("mx4_d128_gqa4_tc", 600, 1, 8, 2, 128, 128, 128, 128, 128, 128, "mxfp4", "mxfp8"),
    ("mx4_d128_single_row", 300, 1, 2, 2, 128, 128, 128, 128, 0, 0, "mxfp4", "mxfp8"),
    ("low8_e5m2", 260, 1, 2, 1, 128, 64, 128, 128, 0, 128, "mxfp8", "e5m2"),
    ("nv_T0_S0_tile_m32", 640, 4, 4, 4, 128, 128, 32, 64, 0, 0, "nvfp4", "mxfp8"),
    ("nv_gqa16_nq1", 1100, 1, 16, 1, 128, 128, 128, 128, 128, 128, "nvfp4", "mxfp8"),
    ("nv_rows_gt16", 400, 5, 8, 1, 128, 128, 128, 128, 128, 0, "nvfp4", "mxfp8"),
]


def _fmt(mod, key):
    return getattr(mod, FMT[key][0])


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_decode_matches_oracle_rows(case):
    name, L, nq, H, KVH, d, dv, tm, tn, T, S, low, high = case
    m = D()
    G = H // KVH
    seed = sum(map(ord, name))
    q = randn_bf16(seed, H, L, d)
    k = randn_bf16(seed + 1, KVH, L, d)
    v = randn_bf16(seed + 2, KVH, L, dv)
    cfg = m.AttentionConfig(tile_m=tm, tile_n=tn, diag_window=T, sink_window=S, causal=True,
                            low_format=_fmt(m, low), high_format=_fmt(m, high))
    cache = m.DmaKVCache(cfg, batch=1, kv_heads=KVH, capacity=L + 64, head_dim=d, v_dim=dv)
    kt = torch.from_numpy(k).cuda()[None]
    vt = torch.from_numpy(v).cuda()[None]
    cache.append(kt[:, :, :L - nq], vt[:, :, :L - nq])  # prompt, then one step of n_q tokens
    out = cache.step(torch.from_numpy(q[:, L - nq:]).cuda()[None], kt[:, :, L - nq:], vt[:, :, L - nq:])
    got = out[0].double().cpu().numpy()
    ocfg = O.Cfg(tile_m=tm, tile_n=tn, diag_window=T, sink_window=S, causal=True,
                 low_format=getattr(O, FMT[low][1]), high_format=getattr(O, FMT[high][1]), granularity=O.TOKEN)
    for h in range(H):
        want = O.mixed_precision_attention(q[h], k[h // G], v[h // G], ocfg)[L - nq:]
        rel = np.linalg.norm(got[h] - want) / np.linalg.norm(want)
        mx = np.abs(got[h] - want).max()
        assert rel <= TOL_DECODE[0] and mx <= TOL_DECODE[1], (name, h, rel, mx)


def test_decode_token_by_token_matches_prefill_rows():
    """Eight single-token steps after a prompt: every step is the corresponding row of the
    GPU prefill forward (bf16-PV parity mode, its own tolerance 5e-3 rel-L2)."""
    m = D()
    L, steps, H, KVH, d = 384, 8, 4, 2, 128
    g = torch.Generator(device="cuda").manual_seed(3)
    q, k, v = (torch.randn(1, h, L, d, device="cuda", generator=g).to(torch.bfloat16) for h in (H, KVH, KVH))
    cfg = m.AttentionConfig(tile_m=128, tile_n=128, diag_window=128, sink_window=128, pv_mode="bf16")
    ref = m.DmaAttention(cfg)(q, k, v, out_dtype=torch.float32)
    cache = m.DmaKVCache(cfg, batch=1, kv_heads=KVH, capacity=L, head_dim=d)
    cache.append(k[:, :, :L - steps], v[:, :, :L - steps])
    rows = []
    for i in range(L - steps, L):
        rows.append(cache.step(q[:, :, i:i + 1], k[:, :, i:i + 1], v[:, :, i:i + 1], validate=False))
    got = torch.cat(rows, dim=2)
    want = ref[:, :, L - steps:]
    rel = (torch.linalg.norm(got - want) / torch.linalg.norm(want)).item()
    assert rel < 5e-3, rel
    assert cache.length == L


def test_decode_batch_and_bf16_out():
    m = D()
    B, L, H, KVH, d = 3, 300, 4, 2, 64
    cfg = m.AttentionConfig(tile_m=64, tile_n=64, diag_window=64, sink_window=0)
    g = torch.Generator(device="cuda").manual_seed(5)
    q = torch.randn(B, H, 1, d, device="cuda", generator=g)
    k = torch.randn(B, KVH, L, d, device="cuda", generator=g)
    v = torch.randn(B, KVH, L, d, device="cuda", generator=g).to(torch.bfloat16)
    cache = m.DmaKVCache(cfg, batch=B, kv_heads=KVH, capacity=L, head_dim=d)
    cache.append(k, v)
    o32 = cache.attend(q)
    o16 = cache.attend(q, out_dtype=torch.bfloat16)
    assert o16.dtype == torch.bfloat16 and torch.allclose(o16.float(), o32, rtol=1e-2, atol=1e-2)
    ocfg = O.Cfg(tile_m=64, tile_n=64, diag_window=64, sink_window=0, causal=True, low_format=O.NVFP4,
                 high_format=O.MXFP8_E4M3, granularity=O.TOKEN)
    for b in range(B):
        for h in range(H):
            # the query row sits at position L - 1; give the oracle a full-length Q with it last
            qq = np.zeros((L, d))
            qq[-1] = q[b, h, 0].double().cpu().numpy()
            want = O.mixed_precision_attention(qq, k[b, h // 2].double().cpu().numpy(),
                                               v[b, h // 2].double().cpu().numpy(), ocfg)[-1]
            got = o32[b, h, 0].double().cpu().numpy()
            assert np.abs(got - want).max() <= TOL_DECODE[1]


def test_decode_errors():
    m = D()
    cfg = m.AttentionConfig(tile_m=128, tile_n=128)
    from paper_2604_03950_b200._lib import DmaUnsupported

    with pytest.raises(DmaUnsupported):
        m.DmaKVCache(m.AttentionConfig(granularity=m.Granularity.TENSOR), 1, 1, 64, 64)
    cache = m.DmaKVCache(cfg, batch=1, kv_heads=1, capacity=32, head_dim=64)
    k = torch.randn(1, 1, 40, 64, device="cuda")
    with pytest.raises(ValueError, match="overflow"):
        cache.append(k, k.to(torch.bfloat16))
    with pytest.raises(ValueError, match="non-finite"):
        cache.append(torch.full((1, 1, 4, 64), float("nan"), device="cuda"), k[:, :, :4])
    cache.append(k[:, :, :8], k[:, :, :8])
    with pytest.raises(ValueError, match="n_q"):
        cache.attend(torch.randn(1, 1, 9, 64, device="cuda"))


def test_decode_from_empty_cache():
    """First tokens of a sequence: no prompt, one step of 3 tokens (causal among themselves),
    then single tokens -- every row equals the oracle's row of the whole sequence."""
    m = D()
    L, H, KVH, d = 40, 2, 1, 64
    q, k, v = (randn_bf16(900 + i, h, L, d) for i, h in enumerate((H, KVH, KVH)))
    cfg = m.AttentionConfig(tile_m=64, tile_n=64, diag_window=64, sink_window=0)
    cache = m.DmaKVCache(cfg, batch=1, kv_heads=KVH, capacity=L, head_dim=d)
    qt, kt, vt = (torch.from_numpy(x).cuda()[None] for x in (q, k, v))
    outs = [cache.step(qt[:, :, :3], kt[:, :, :3], vt[:, :, :3])]
    for i in range(3, L):
        outs.append(cache.step(qt[:, :, i:i + 1], kt[:, :, i:i + 1], vt[:, :, i:i + 1]))
    got = torch.cat(outs, dim=2)[0].double().cpu().numpy()
    ocfg = O.Cfg(tile_m=64, tile_n=64, diag_window=64, sink_window=0, causal=True, low_format=O.NVFP4,
                 high_format=O.MXFP8_E4M3, granularity=O.TOKEN)
    for h in range(H):
        want = O.mixed_precision_attention(q[h], k[0], v[0], ocfg)
        assert np.abs(got[h] - want).max() <= TOL_DECODE[1]
