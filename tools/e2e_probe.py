"""Time DmaAttention.forward_host (host tensors) vs device-only forward for a config."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_03950_b200 as D  # noqa: E402

B, H, KVH, N, d = [int(v) for v in sys.argv[1:6]]
cfg = D.AttentionConfig(tile_m=128, tile_n=128, diag_window=128, sink_window=128, low_format=D.MXFP4)
g = torch.Generator().manual_seed(0)
q = torch.randn(B, H, N, d, generator=g).to(torch.bfloat16).pin_memory()
k = torch.randn(B, KVH, N, d, generator=g).to(torch.bfloat16).pin_memory()
v = torch.randn(B, KVH, N, d, generator=g).to(torch.bfloat16).pin_memory()
o = torch.empty(B, H, N, d, dtype=torch.bfloat16).pin_memory()
fwd = D.DmaAttention(cfg)
dq, dk, dv = q.cuda(), k.cuda(), v.cuda()
for name, fn in [("device fwd", lambda: fwd(dq, dk, dv)),
                 ("h2d only", lambda: (dq.copy_(q, non_blocking=True), dk.copy_(k, non_blocking=True), dv.copy_(v, non_blocking=True))),
                 ("d2h only", lambda: o.copy_(dq[:, :H], non_blocking=True))] + \
        [(f"forward_host chunk={c}", (lambda c=c: fwd.forward_host(q, k, v, out=o, chunk_kv_heads=c))) for c in (1, 2, 4, 8) if c <= KVH]:
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:28s} {e0.elapsed_time(e1) / 5:8.3f} ms (events)  {(time.perf_counter() - t0) / 5 * 1e3:8.3f} ms (wall)")
