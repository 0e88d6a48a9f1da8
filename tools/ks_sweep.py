"""KV-split sweep: attention-core time (dma_attention_core, 50 back-to-back launches timed
with CUDA events) per split mode for small shapes.  python tools/ks_sweep.py"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_03950_b200 as D
from paper_2604_03950_b200 import _lib

L = _lib.lib()
shapes = [(1, 1, 1024, 64, 64, "mxfp4"), (1, 2, 4096, 128, 128, "nvfp4"), (1, 8, 2048, 128, 128, "nvfp4"),
          (1, 4, 8192, 128, 128, "nvfp4")]
for (B, H, N, d, dv, low) in shapes:
    cfg = D.AttentionConfig(tile_m=128, tile_n=128, diag_window=128, sink_window=128,
                            low_format={"nvfp4": D.NVFP4, "mxfp4": D.MXFP4}[low])
    g = torch.Generator(device="cuda").manual_seed(1)
    q = torch.randn(B, H, N, d, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(B, H, N, d, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(B, H, N, dv, device="cuda", generator=g).to(torch.bfloat16)
    row = []
    for mode in (0, -1, 2, 4, 8):
        L.dma_attention_set_kv_split(mode)
        fwd = D.DmaAttention(cfg)
        a, out = fwd.prepare(q, k, v)
        sp = _lib.stream_ptr(torch.cuda.current_stream())
        ns = L.dma_attention_kv_split(a)
        _lib.check(L.dma_attention_fwd(a, sp), "fwd")
        for _ in range(5):
            _lib.check(L.dma_attention_core(a, sp), "core")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(50):
            _lib.check(L.dma_attention_core(a, sp), "core")
        e1.record()
        torch.cuda.synchronize()
        row.append(f"mode {mode:2d} (ns {ns}): {e0.elapsed_time(e1) / 50 * 1000:7.1f} us")
    L.dma_attention_set_kv_split(-1)
    print(f"B{B} H{H} N{N} d{d}:", " | ".join(row), flush=True)
