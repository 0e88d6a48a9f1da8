#!/usr/bin/env python
"""Decode step timing over an MX key cache (decode.cuh): one new token per sequence.

Algorithmic bytes per step (what the kernel must read): for every (b, kv head) and cached
key, the K operand of the tile's precision (NVFP4 low: d/2 + d/16 bytes; MXFP8 high:
d + d/32) + S_q (8 B) + the bf16 V row (2 dv), plus the quantized queries and O.  Time:
CUDA events around attend() (query quantize + decode kernel + split combine), median.

  python tools/bench_decode.py [--batch 8] [--heads 32] [--kv-heads 8] [--ctx 32768]
"""

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_03950_b200 as D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--kv-heads", type=int, default=8)
    ap.add_argument("--ctx", type=int, default=32768)
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--nq", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--low", default="nvfp4", choices=["nvfp4", "mxfp4", "mxfp8"])
    args = ap.parse_args()
    B, H, KVH, L, d, nq = args.batch, args.heads, args.kv_heads, args.ctx, args.d, args.nq
    low = {"nvfp4": D.NVFP4, "mxfp4": D.MXFP4, "mxfp8": D.MXFP8_E4M3}[args.low]
    cfg = D.AttentionConfig(tile_m=128, tile_n=128, diag_window=128, sink_window=128, low_format=low)
    cache = D.DmaKVCache(cfg, batch=B, kv_heads=KVH, capacity=L, head_dim=d)
    g = torch.Generator(device="cuda").manual_seed(0)
    for b0 in range(0, L, 8192):  # fill in chunks (bounded temporaries)
        n = min(8192, L - b0)
        k = torch.randn(B, KVH, n, d, device="cuda", generator=g, dtype=torch.bfloat16)
        cache.append(k, k, validate=False)
    q = torch.randn(B, H, nq, d, device="cuda", generator=g, dtype=torch.bfloat16)
    out = torch.empty(B, H, nq, d, device="cuda")
    for _ in range(5):
        cache.attend(q, out=out, validate=False)
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cache.attend(q, out=out, validate=False)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    hfrac_keys = min(L, 128 + 256) / L  # sink tile + the window tiles (row's q tile and the one before)
    lo_bytes = {"nvfp4": d / 2 + d / 16, "mxfp4": d / 2 + d / 32, "mxfp8": d + d / 32}[args.low]
    per_key = hfrac_keys * (d + d / 32) + (1 - hfrac_keys) * lo_bytes + 8 + 2 * d
    nbytes = B * KVH * L * per_key + B * H * nq * (d + d / 2 + d / 16 + d / 32 + 8 + 4 * d)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    print(json.dumps({"metric": "decode_step_ms", "value": ms, "batch": B, "heads": H, "kv_heads": KVH, "ctx": L,
                      "d": d, "n_q": nq, "low": args.low, "bytes": nbytes, "achieved_GBps": nbytes / (ms * 1e-3) / 1e9,
                      "peaks": {k: v for k, v in peaks.items() if "hbm" in k.lower() or "copy" in k.lower()}}))


if __name__ == "__main__":
    main()
