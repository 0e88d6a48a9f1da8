#!/usr/bin/env python
"""c4: diagonal-window width x quantization-granularity ablation at N=16384, d=128
(BASELINE.json configs[3]; paper Table 2/6 style "precision vs TFLOPS").

For every (T = S, granularity) point: attention-kernel TFLOPS (device time, CUDA
events, median of --steps launches after warm-up; algorithmic causal FLOPs), the
Bit_high fraction of the plan, and the output error against full-precision attention
(cosine similarity and rel-L2 vs a float64 torch softmax(QK^T/sqrt(d))V on --heads
sampled heads).  One JSON line per point; writes gpurun_out/<tag>_c4_sweep.jsonl.

  python tools/ablation_c4.py [--steps 10] [--heads 2] [--tag r01]
"""

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_03950_b200 as D  # noqa: E402
from paper_2604_03950_b200 import _lib  # noqa: E402


def full_precision(q, k, v):
    """softmax(q k^T / sqrt(d)) v in float64 with the causal mask (attention.py:122-147)."""
    q, k, v = q.double(), k.double(), v.double()
    s = (q @ k.transpose(-1, -2)) / q.shape[-1] ** 0.5
    n = s.shape[-1]
    mask = torch.ones(n, n, dtype=torch.bool, device=s.device).triu(1)
    s.masked_fill_(mask, float("-inf"))
    return torch.softmax(s, dim=-1) @ v


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--heads", type=int, default=2)
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--n", type=int, default=16384)
    args = ap.parse_args()
    B, H, N, d = 1, 32, args.n, 128
    g = torch.Generator(device="cuda").manual_seed(7)
    q = torch.randn(B, H, N, d, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(B, H, N, d, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(B, H, N, d, device="cuda", generator=g).to(torch.bfloat16)
    refs = [full_precision(q[0, h], k[0, h], v[0, h]) for h in range(args.heads)]
    flops = 4.0 * d * N * (N + 1) / 2 * B * H
    L = _lib.lib()
    sp = _lib.stream_ptr()
    out_lines = []
    for gran in (D.Granularity.TOKEN, D.Granularity.TENSOR, D.Granularity.BLOCK):
        for T in (0, 128, 256, 512, 1024, 2048):
            cfg = D.AttentionConfig(tile_m=128, tile_n=128, diag_window=T, sink_window=T, causal=True,
                                    low_format=D.NVFP4, high_format=D.MXFP8_E4M3, granularity=gran)
            line = {"config": "c4", "N": N, "H": H, "d": d, "diag_window": T, "sink_window": T,
                    "granularity": gran.name.lower(), "low": "nvfp4", "high": "mxfp8_e4m3", "pv_mode": "mxfp8",
                    "bit_high": D.high_precision_fraction(N, N, 128, 128, T, T, True)}
            try:
                fwd = D.DmaAttention(cfg)
                a, out = fwd.prepare(q, k, v, out_dtype=torch.float32)
            except (_lib.DmaUnsupported, ValueError, RuntimeError) as e:
                line["unsupported"] = str(e).splitlines()[0][:160]
                print(json.dumps(line), flush=True)
                out_lines.append(line)
                continue
            _lib.check(L.dma_attention_quantize(a, sp), "quantize")
            for _ in range(3):
                _lib.check(L.dma_attention_core(a, sp), "core")
            torch.cuda.synchronize()
            ts = []
            for _ in range(args.steps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                _lib.check(L.dma_attention_core(a, sp), "core")
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = sorted(ts)[len(ts) // 2]
            cos, rel = [], []
            for h in range(args.heads):
                o = out[0, h].double()
                r = refs[h]
                cos.append(float(torch.nn.functional.cosine_similarity(o.flatten(), r.flatten(), dim=0)))
                rel.append(float(torch.linalg.norm(o - r) / torch.linalg.norm(r)))
            line.update({"attn_ms": ms, "tflops": flops / (ms * 1e-3) / 1e12,
                         "cos_vs_full_precision": sum(cos) / len(cos), "rel_l2_vs_full_precision": sum(rel) / len(rel),
                         "heads_checked": args.heads})
            print(json.dumps(line), flush=True)
            out_lines.append(line)
    # gpurun_out/ is what travels back from the GPU box; copy it under profiles/ to keep it
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"{args.tag}_c4_sweep.jsonl"), "w") as f:
        for ln in out_lines:
            f.write(json.dumps(ln) + "\n")


if __name__ == "__main__":
    main()
