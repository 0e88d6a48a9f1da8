"""Per-step variance of the c3 end-to-end path vs plain PCIe copies (CUDA events per step)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_03950_b200 as D  # noqa: E402
from bench import gpu_local_affinity  # noqa: E402

B, H, KVH, N, d = 1, 32, 32, 32768, 128
gpu_local_affinity(0)
cfg = D.AttentionConfig(tile_m=128, tile_n=128, diag_window=128, sink_window=128)
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(B, H, N, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
hq, hk, hv = (x.cpu().pin_memory() for x in (q, k, v))
ho = torch.empty(B, H, N, d, dtype=torch.bfloat16).pin_memory()
fwd = D.DmaAttention(cfg)
s = torch.cuda.current_stream()


def timed(fn, n):
    fn()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for a0, a1 in evs:
        a0.record(s)
        fn()
        a1.record(s)
    torch.cuda.synchronize()
    return [round(a0.elapsed_time(a1), 2) for a0, a1 in evs]


def h2d():
    q.copy_(hq, non_blocking=True)
    k.copy_(hk, non_blocking=True)
    v.copy_(hv, non_blocking=True)


def d2h():
    ho.copy_(q, non_blocking=True)


s2 = torch.cuda.Stream()


def both():
    s2.wait_stream(s)
    with torch.cuda.stream(s2):
        ho.copy_(q, non_blocking=True)
    h2d()
    s.wait_stream(s2)


for chunk in (1, 2, 4):
    print("forward_host chunk", chunk, timed(lambda: fwd.forward_host(hq, hk, hv, out=ho, chunk_kv_heads=chunk), 7),
          flush=True)
for name, fn in [("h2d 805MB + concurrent d2h 268MB", both), ("h2d 805MB", h2d), ("d2h 268MB", d2h), ("forward_host", lambda: fwd(hq, hk, hv, out=ho)),
                 ("h2d 805MB again", h2d), ("forward_host again", lambda: fwd(hq, hk, hv, out=ho))]:
    print(name, timed(fn, 15), flush=True)
