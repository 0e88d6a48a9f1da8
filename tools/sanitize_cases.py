#!/usr/bin/env python
"""Small-shape runs of every libdma kernel family for compute-sanitizer (racecheck /
synccheck / memcheck): quantize_dual, the ping-pong attention (two-phase, KV-split and fused), the
single-stream attention (bf16 PV and the BLOCK bf16-operand route) and the decode kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_03950_b200 as D  # noqa: E402
from paper_2604_03950_b200 import _lib  # noqa: E402

torch.manual_seed(0)
q = torch.randn(1, 2, 384, 128, device="cuda").to(torch.bfloat16)
k = torch.randn(1, 2, 384, 128, device="cuda").to(torch.bfloat16)
v = torch.randn(1, 2, 384, 128, device="cuda").to(torch.bfloat16)
base = dict(tile_m=128, tile_n=128, diag_window=128, sink_window=128)
D.quantize_dual(q[0, 0], True, D.NVFP4, D.MXFP8_E4M3)
x = torch.randn(512, 128, device="cuda")
x[:, 3] = 168 / 32.0  # row maxima with a 21 * 2^k mantissa: many exact ties -> the warp-compacted redo
x = x.clamp(-168 / 32.0, 168 / 32.0).to(torch.bfloat16)
for low in (D.NVFP4, D.MXFP4):
    D.quantize_dual(x, False, low, D.MXFP8_E4M3)
print("quantize ok")
L = _lib.lib()
ks = L.dma_attention_set_kv_split(0)
D.dma_attention(q, k, v, D.AttentionConfig(**base))  # ping-pong kernel, two-phase
print("pp ok")
L.dma_attention_set_kv_split(3)
D.dma_attention(q, k, v, D.AttentionConfig(**base))  # KV-split ping-pong kernel + merge
L.dma_attention_set_kv_split(ks)
print("kv-split ok")
prev = L.dma_attention_set_fused(1)
D.dma_attention(q, k, v, D.AttentionConfig(**base))  # fused kernel
L.dma_attention_set_fused(prev)
print("fused ok")
D.dma_attention(q, k, v, D.AttentionConfig(pv_mode="bf16", **base))  # single-stream, bf16 PV
print("bf16-PV ok")
D.dma_attention(q, k, v, D.AttentionConfig(granularity=D.Granularity.BLOCK, **base))  # bf16-operand route
print("block ok")
cache = D.DmaKVCache(D.AttentionConfig(**base), batch=1, kv_heads=2, capacity=384, head_dim=128)
cache.append(k[:, :, :380], v[:, :, :380])
cache.step(q[:, :, 380:], k[:, :, 380:], v[:, :, 380:])
print("decode ok")
torch.cuda.synchronize()
print("all kernels ran")
