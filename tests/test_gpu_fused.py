"""GPU: the fused forward (phase 1 inside the ping-pong kernel: quantizer warps + per-tile
ready flags, attn_pp.cuh FuseParams) against the two-phase path (phase-1 kernels, then the
attention kernel) on the same inputs.  Both quantize into the same operand layouts (the fused
kernel with q16_item_fast / qv4_block, the two-phase path with the same code for small
problems and quant32_bf16_kernel for large ones) and run the same attention code, so the
outputs must be bit-identical; the fused call launches exactly one kernel."""

import pytest

pytestmark = pytest.mark.gpu

CASES = [
    # B, H, KVH, Lq, Lk, d, dv, low, high, T, S, causal
    (1, 1, 1, 1024, 1024, 64, 64, "MXFP4", "MXFP8_E4M3", 128, 128, True),
    (1, 4, 4, 1000, 1000, 128, 128, "NVFP4", "MXFP8_E4M3", 256, 128, True),
    (2, 8, 2, 777, 777, 128, 128, "MXFP4", "MXFP8_E4M3", 128, 128, True),
    (1, 3, 1, 384, 700, 128, 128, "NVFP4", "MXFP8_E4M3", 256, 128, False),
    (1, 2, 2, 512, 512, 128, 128, "MXFP8_E4M3", "MXFP8_E4M3", 0, 0, True),
    (1, 2, 1, 640, 640, 128, 64, "NVFP4", "MXFP8_E5M2", 128, 128, True),
    (1, 2, 2, 4096, 4096, 128, 128, "NVFP4", "MXFP8_E4M3", 128, 128, True),
    # > 8 M phase-1 elements: the two-phase path runs quant32_bf16_kernel (32 columns per
    # thread, warp-compacted float64 redo) -- flattened heads (N % 128 == 0) and per-head (ragged)
    (1, 8, 2, 8192, 8192, 128, 128, "NVFP4", "MXFP8_E4M3", 128, 128, True),
    (1, 6, 3, 7000, 7000, 128, 128, "MXFP4", "MXFP8_E5M2", 256, 128, True),
    (2, 4, 4, 4096, 4608, 128, 128, "NVFP4", "MXFP8_E4M3", 128, 128, False),
]


@pytest.mark.parametrize("case", CASES)
def test_fused_forward_equals_two_phase(case):
    import torch

    import paper_2604_03950_b200 as D
    from paper_2604_03950_b200 import _lib

    B, H, KVH, lq, lk, d, dv, low, high, T, S, causal = case
    cfg = D.AttentionConfig(tile_m=128, tile_n=128, diag_window=T, sink_window=S, causal=causal,
                            low_format=getattr(D, low), high_format=getattr(D, high))
    g = torch.Generator(device="cuda").manual_seed(lq + H)
    q = torch.randn(B, H, lq, d, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(B, KVH, lk, d, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(B, KVH, lk, dv, device="cuda", generator=g).to(torch.bfloat16)
    fwd = D.DmaAttention(cfg)
    L = _lib.lib()
    sp = _lib.stream_ptr()
    a, out = fwd.prepare(q, k, v, out_dtype=torch.float32)
    prev = L.dma_attention_set_fused(1)
    try:
        for _ in range(2):  # twice: flags / counters are reset per call
            _lib.check(L.dma_attention_fwd(a, sp), "fused")
            assert L.dma_last_launch_count() == 1
    finally:
        L.dma_attention_set_fused(prev)
    fused = out.clone()
    # the fused forward never splits the KV range (one launch); compare with the unsplit
    # two-phase path (small cases would otherwise take the KV-split kernel + merge)
    prev_ks = L.dma_attention_set_kv_split(0)
    try:
        _lib.check(L.dma_attention_quantize(a, sp), "quantize")
        _lib.check(L.dma_attention_core(a, sp), "core")
        torch.cuda.synchronize()
    finally:
        L.dma_attention_set_kv_split(prev_ks)
    assert torch.isfinite(fused).all()
    assert torch.equal(fused, out), float((fused - out).abs().max())


def test_fused_nonfinite_raises():
    import torch

    import paper_2604_03950_b200 as D
    from paper_2604_03950_b200 import _lib

    cfg = D.AttentionConfig(tile_m=128, tile_n=128, diag_window=128, sink_window=128)
    q = torch.randn(1, 2, 256, 128, device="cuda").to(torch.bfloat16)
    k = q.clone()
    k[0, 1, 200, 7] = float("inf")
    prev = _lib.lib().dma_attention_set_fused(1)
    try:
        with pytest.raises(ValueError, match="non-finite"):
            D.dma_attention(q, k, q, cfg)
    finally:
        _lib.lib().dma_attention_set_fused(prev)
