"""GPU: KV splits of the ping-pong forward (small problems: fewer head pairs x query tiles
than SMs).  Each query tile's plan (attention.py:191-233) is cut into contiguous ranges run
by different CTAs; kv_combine_kernel merges their online-softmax states (attention.py:
150-175).  Checked against the oracle (the reference, TOL) and against its PV emulation run
with the same ranges (``kv_split=n``, TOL_EMU), forced and automatic."""

import zlib

import numpy as np
import pytest

from conftest import kv_split_of, record_parity
from inputs import randn_bf16
from oracle import mx_oracle as O
from test_gpu_attention import TOL, TOL_EMU, cfgs, errs

pytestmark = pytest.mark.gpu

CASES = [
    # name, Lq, Lk, d, dv, low, T, S, causal
    ("c1_shape", 1024, 1024, 64, 64, "mxfp4", 128, 128, True),
    ("n1536_d128_nvfp4", 1536, 1536, 128, 128, "nvfp4", 128, 128, True),
    ("ragged_1000", 1000, 1000, 128, 128, "nvfp4", 256, 128, True),
    ("noncausal_384x1400", 384, 1400, 128, 64, "nvfp4", 256, 128, False),
    ("dv128_d64_T0", 900, 900, 64, 128, "mxfp4", 0, 0, True),
]


@pytest.fixture
def lib():
    from paper_2604_03950_b200 import _lib

    L = _lib.lib()
    prev = L.dma_attention_set_kv_split(-1)
    yield L
    L.dma_attention_set_kv_split(prev)


@pytest.mark.parametrize("n", [2, 3, 5])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_forced_splits_vs_oracle(case, n, lib):
    import paper_2604_03950_b200 as D

    name, lq, lk, d, dv, low, T, S, causal = case
    c, oc = cfgs(low, "e4m3", "token", T, S, causal, "mxfp8")
    seed = zlib.crc32(name.encode()) % 1000
    q, k, v = randn_bf16(seed, lq, d), randn_bf16(seed + 1, lk, d), randn_bf16(seed + 2, lk, dv)
    lib.dma_attention_set_kv_split(n)
    ks = kv_split_of(c, lq, lk, d, dv)
    assert 2 <= ks <= n
    got = D.mixed_precision_attention(q, k, v, c)
    want = O.mixed_precision_attention(q, k, v, oc)
    emu = O.mixed_precision_attention(q, k, v, oc, pv="mxfp8", kv_split=ks)
    rel, mx = errs(got, want)
    erel, emx = errs(got, emu)
    record_parity(f"kvsplit{n}_{name}", "mxfp8", rel, mx, erel, emx, kv_split=ks)
    assert np.isfinite(got).all()
    assert erel <= TOL_EMU["mxfp8"][0] and emx <= TOL_EMU["mxfp8"][1], (erel, emx)
    assert rel <= TOL["mxfp8"][0] and mx <= TOL["mxfp8"][1], (rel, mx)


def test_auto_policy_small_and_large(lib):
    """The default policy splits the c1 shape (8 pairs on 148 SMs) and leaves c3 alone."""
    import paper_2604_03950_b200 as D

    c = D.AttentionConfig(tile_m=128, tile_n=128, diag_window=128, sink_window=128, low_format=D.MXFP4)
    assert kv_split_of(c, 1024, 1024, 64, 64) > 1
    assert kv_split_of(c, 32768, 32768, 128, 128, H=32, KVH=32) == 1
    bf = D.AttentionConfig(tile_m=128, tile_n=128, diag_window=128, sink_window=128, pv_mode="bf16")
    assert kv_split_of(bf, 1024, 1024, 64, 64) == 1  # only the block-scaled ping-pong path splits


def test_batched_gqa_split_and_launches(lib):
    """B2 H8 KVH2 N640 (GQA, batched): split forward = per-head split emulation; the forward is
    phase 1 + the split attention kernel + the merge (3 launches), unsplit 2."""
    import torch

    import paper_2604_03950_b200 as D
    from paper_2604_03950_b200 import _lib

    B, H, KVH, N, d = 2, 8, 2, 640, 128
    c, oc = cfgs("nvfp4", "e4m3", "token", 128, 128, True, "mxfp8")
    g = torch.Generator().manual_seed(11)
    q = torch.randn(B, H, N, d, generator=g).to(torch.bfloat16)
    k = torch.randn(B, KVH, N, d, generator=g).to(torch.bfloat16)
    v = torch.randn(B, KVH, N, d, generator=g).to(torch.bfloat16)
    lib.dma_attention_set_kv_split(3)
    fwd = D.DmaAttention(c)
    a, out = fwd.prepare(q.cuda(), k.cuda(), v.cuda(), out_dtype=torch.float32)
    assert lib.dma_attention_kv_split(a) == 3
    _lib.check(lib.dma_attention_fwd(a, _lib.stream_ptr()), "fwd")
    assert lib.dma_last_launch_count() == 3
    got = out.cpu().double().numpy()
    for b in range(B):
        for h in (0, 5):
            kh = h // (H // KVH)
            emu = O.mixed_precision_attention(q[b, h].double().numpy(), k[b, kh].double().numpy(),
                                              v[b, kh].double().numpy(), oc, pv="mxfp8", kv_split=3)
            erel, emx = errs(got[b, h], emu)
            assert erel <= TOL_EMU["mxfp8"][0] and emx <= TOL_EMU["mxfp8"][1], (b, h, erel, emx)
    # per-call override: a.kv_split = 1 runs unsplit whatever the global mode
    a.kv_split = 1
    _lib.check(lib.dma_attention_fwd(a, _lib.stream_ptr()), "fwd")
    assert lib.dma_last_launch_count() == 2
    unsplit = out.cpu().double().numpy()
    emu = O.mixed_precision_attention(q[0, 0].double().numpy(), k[0, 0].double().numpy(),
                                      v[0, 0].double().numpy(), oc, pv="mxfp8")
    erel, emx = errs(unsplit[0, 0], emu)
    assert erel <= TOL_EMU["mxfp8"][0] and emx <= TOL_EMU["mxfp8"][1], (erel, emx)


def test_split_is_deterministic_and_bf16_out(lib):
    import torch

    import paper_2604_03950_b200 as D

    c, _ = cfgs("nvfp4", "e4m3", "token", 128, 128, True, "mxfp8")
    g = torch.Generator().manual_seed(5)
    q, k, v = (torch.randn(1, 2, 2048, 128, generator=g).to(torch.bfloat16).cuda() for _ in range(3))
    lib.dma_attention_set_kv_split(4)
    x = D.dma_attention(q, k, v, c)
    y = D.dma_attention(q, k, v, c)
    assert x.dtype == torch.bfloat16 and torch.equal(x, y)
    lib.dma_attention_set_kv_split(0)
    z = D.dma_attention(q, k, v, c)
    assert float((x.float() - z.float()).abs().max()) < 0.05  # split vs unsplit: P-rounding only


def test_pieces_with_whole_problem_count_are_bit_identical(lib):
    """A caller that runs a small problem in (b, kv-head) pieces (sharding.py, the host
    pipeline) passes the whole problem's split count: the pieces reproduce one call."""
    import torch

    import paper_2604_03950_b200 as D

    c, _ = cfgs("nvfp4", "e4m3", "token", 128, 128, True, "mxfp8")
    g = torch.Generator().manual_seed(17)
    B, H, KVH, N, d = 2, 4, 2, 1024, 128
    q = torch.randn(B, H, N, d, generator=g).to(torch.bfloat16).cuda()
    k = torch.randn(B, KVH, N, d, generator=g).to(torch.bfloat16).cuda()
    v = torch.randn(B, KVH, N, d, generator=g).to(torch.bfloat16).cuda()
    lib.dma_attention_set_kv_split(4)  # (the policy leaves this shape unsplit)
    n = D.attention.kv_split_count(q.shape, k.shape, v.shape, c)
    assert n == 4
    whole = D.dma_attention(q, k, v, c)
    lib.dma_attention_set_kv_split(-1)  # the pieces alone would pick their own count
    G = H // KVH
    for b in range(B):
        for kh in range(KVH):
            piece = D.dma_attention(q[b:b + 1, kh * G:(kh + 1) * G], k[b:b + 1, kh:kh + 1], v[b:b + 1, kh:kh + 1], c,
                                    kv_split=n)
            assert torch.equal(piece, whole[b:b + 1, kh * G:(kh + 1) * G]), (b, kh)
