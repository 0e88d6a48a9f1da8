#!/usr/bin/env python
"""Phase timers of the ws kernel (needs a -DDMA_PROFILE build in DMA_LIB_PATH, DMA_ATTN_KERNEL=ws)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_03950_b200 as D  # noqa: E402
from paper_2604_03950_b200 import _lib  # noqa: E402

cfgn = sys.argv[1] if len(sys.argv) > 1 else "c3"
B, H, KVH, N, d, low = {"c3": (1, 32, 32, 32768, 128, D.NVFP4), "c2": (1, 32, 8, 8192, 128, D.MXFP4)}[cfgn]
cfg = D.AttentionConfig(tile_m=128, tile_n=128, diag_window=128, sink_window=128, low_format=low)
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(B, h, N, d, device="cuda", generator=g).to(torch.bfloat16) for h in (H, KVH, KVH))
fwd = D.DmaAttention(cfg)
a, out = fwd.prepare(q, k, v)
L = _lib.lib()
L.dma_ws_prof_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
sp = _lib.stream_ptr()
_lib.check(L.dma_attention_quantize(a, sp), "q")
buf = (ctypes.c_ulonglong * 32)()
_lib.check(L.dma_attention_core(a, sp), "core")
torch.cuda.synchronize()
L.dma_ws_prof_read(buf, 32)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
_lib.check(L.dma_attention_core(a, sp), "core")
e1.record()
torch.cuda.synchronize()
L.dma_ws_prof_read(buf, 32)
print(f"{cfgn}: kernel {e0.elapsed_time(e1):.3f} ms")
for title, base, nm in (("MAX warps", 0, ["wait S", "max tile", "m publish + O rescale", "epilogue", "sched/loop"]),
                        ("EXP warps", 8, ["wait m", "wait S", "wait PV(g-2)", "exp tile", "tail (st wait, arrive)",
                                          "sched/loop/l publish"]),
                        ("QK issuer", 16, ["wait S free", "wait K", "SF copy + MMA issue"]),
                        ("PV issuer", 20, ["wait P", "wait O rescaled", "wait O free", "wait V", "SF copy + MMA"])):
    tot = sum(buf[base:base + len(nm)]) or 1
    print(f"{title} (total {tot / 1e9:.2f} G warp-cycles):")
    for i, n in enumerate(nm):
        print(f"  {n:24s} {buf[base + i] / tot * 100:6.1f}%")
