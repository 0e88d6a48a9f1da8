#!/usr/bin/env python
"""Compare two phase-2 kernels (DMA_ATTN_KERNEL values) on the same inputs: per query tile
rel-L2 of kernel B against kernel A.  usage: kern_diff.py [H] [N] [low] (runs both in
subprocesses since the kernel choice is read once per process)."""
import os
import subprocess
import sys

import numpy as np

H, N = int(sys.argv[1]) if len(sys.argv) > 1 else 2, int(sys.argv[2]) if len(sys.argv) > 2 else 32768
LOW = sys.argv[3] if len(sys.argv) > 3 else "nvfp4"
A, B = os.environ.get("KA", "pp"), os.environ.get("KB", "ws")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, "{root}")
import paper_2604_03950_b200 as D
g = torch.Generator(device="cuda").manual_seed(7)
q, k, v = (torch.randn(1, {H}, {N}, 128, device="cuda", generator=g).to(torch.bfloat16).to(torch.{DT}) for _ in range(3))
c = D.AttentionConfig(tile_m=128, tile_n=128, diag_window=128, sink_window=128, low_format=D.{LOW})
o = D.DmaAttention(c)(q, k, v, out_dtype=torch.float32)
np.save("{out}", o[0].cpu().numpy())
'''
outs = {}
for kern in (A, B):
    path = f"/tmp/kd_{kern}.npy"
    env = dict(os.environ, DMA_ATTN_KERNEL=kern)
    r = subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT, H=H, N=N, LOW=LOW.upper(), out=path, DT=os.environ.get("DT", "bfloat16"))], env=env,
                       capture_output=True, text=True, timeout=300)
    if r.returncode:
        print(kern, "failed:", r.stderr[-1500:])
        sys.exit(1)
    outs[kern] = np.load(path)
a, b = outs[A], outs[B]
nt = N // 128
bad = []
for h in range(H):
    for t in range(nt):
        x, y = a[h, 128 * t:128 * t + 128], b[h, 128 * t:128 * t + 128]
        rel = float(np.linalg.norm(x - y) / max(np.linalg.norm(x), 1e-30))
        if rel > 1e-3:
            rows = np.where(np.abs(x - y).max(axis=1) > 1e-3 * np.abs(x).max())[0]
            bad.append((h, t, rel, len(rows), rows[:6].tolist()))
print(f"H={H} N={N} {LOW}: {len(bad)} of {H * nt} query tiles differ (rel > 1e-3) between {A} and {B}")
for x in bad[:25]:
    print("  head %d tile %d rel %.3e rows %d first %s" % x)
