import os, sys, time, torch
sys.path.insert(0, os.getcwd())
import paper_2604_03950_b200 as D
B, H, KVH, N, d = 1, 32, 8, 8192, 128
cfg = D.AttentionConfig(tile_m=128, tile_n=128, diag_window=128, sink_window=128, causal=True, low_format=D.MXFP4,
                        high_format=D.MXFP8_E4M3, granularity=D.Granularity.TOKEN, pv_mode="mxfp8")
g = torch.Generator(device="cuda").manual_seed(1234)
q = torch.randn(B, H, N, d, device="cuda", generator=g).to(torch.bfloat16)
k = torch.randn(B, KVH, N, d, device="cuda", generator=g).to(torch.bfloat16)
v = torch.randn(B, KVH, N, d, device="cuda", generator=g).to(torch.bfloat16)
fwd = D.DmaAttention(cfg)
a, out = fwd.prepare(q, k, v, out_dtype=torch.bfloat16)
hq, hk, hv = (x.cpu().pin_memory() for x in (q, k, v))
ho = torch.empty(out.shape, dtype=out.dtype).pin_memory()
print("pinned:", hq.is_pinned(), ho.is_pinned(), hq.is_contiguous())
for trial in range(3):
    fwd(hq, hk, hv, out=ho); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    for _ in range(5): fwd(hq, hk, hv, out=ho)
    e1.record(); torch.cuda.synchronize()
    print("bench-like e2e", e0.elapsed_time(e1) / 5, "ms; wall", (time.perf_counter() - t0) / 5 * 1e3)
