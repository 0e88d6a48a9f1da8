"""End-to-end (pinned host in/out) per chunk size, graph vs eager (CUDA events per step).

  python tools/e2e_c2.py [H KVH N]   (default c2: 32 8 8192)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_03950_b200 as D  # noqa: E402
from bench import gpu_local_affinity  # noqa: E402

B, d = 1, 128
H, KVH, N = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (32, 8, 8192)
gpu_local_affinity(0)
cfg = D.AttentionConfig(tile_m=128, tile_n=128, diag_window=128, sink_window=128, low_format=D.MXFP4)
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(B, H, N, d, device="cuda", generator=g).to(torch.bfloat16)
k, v = (torch.randn(B, KVH, N, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(2))
hq, hk, hv = (x.cpu().pin_memory() for x in (q, k, v))
ho = torch.empty(B, H, N, d, dtype=torch.bfloat16).pin_memory()
fwd = D.DmaAttention(cfg)
s = torch.cuda.current_stream()


def timed(fn, n=9):
    fn()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for a0, a1 in evs:
        a0.record(s)
        fn()
        a1.record(s)
    torch.cuda.synchronize()
    return sorted(round(a0.elapsed_time(a1), 3) for a0, a1 in evs)[n // 2]


def h2d():
    q.copy_(hq, non_blocking=True)
    k.copy_(hk, non_blocking=True)
    v.copy_(hv, non_blocking=True)


print("h2d only", timed(h2d))
for chunk in [c for c in (1, 2, 4, 8) if c <= KVH]:
    for graph in (True, False):
        print("chunk", chunk, "graph", graph,
              timed(lambda: fwd.forward_host(hq, hk, hv, out=ho, chunk_kv_heads=chunk, graph=graph)), flush=True)
