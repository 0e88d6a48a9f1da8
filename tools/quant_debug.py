#!/usr/bin/env python
"""Which golden quantize_dual cases mismatch, and where (bit-exactness debugging)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import paper_2604_03950_b200 as D  # noqa: E402

G = np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))
GR = {"token": "TOKEN", "block": "BLOCK", "tensor": "TENSOR"}
nbad = 0
for key in [str(k) for k in G["quant_keys"]]:
    _, iname, lname, hname, gname, isq = key.split("/")
    low = {"nvfp4": D.NVFP4, "mxfp4": D.MXFP4}[lname]
    high = {"mxfp8_e4m3": D.MXFP8_E4M3, "mxfp8_e5m2": D.MXFP8_E5M2}[hname]
    x = G[f"qin/{iname}"]
    t = D.quantize_dual(x, bool(int(isq)), low, high, getattr(D.Granularity, GR[gname]))
    for f, got in (("packed_low", t.packed_low.bytes_), ("scales_low", t.scales_low), ("high_codes", t.high_codes),
                   ("scales_high", t.scales_high)):
        want = G[f"{key}/{f}"]
        if not np.array_equal(got, want):
            nbad += 1
            idx = np.argwhere(got != want)
            print(key, f, "mismatches", len(idx), "dtype", x.dtype, "first", idx[:3].tolist(),
                  "got", [int(got[tuple(i)]) for i in idx[:3]], "want", [int(want[tuple(i)]) for i in idx[:3]])
            if f == "high_codes" or f == "packed_low":
                r = idx[0][0]
                print("   row", r, "x[:8]", x[r][:8], "absmax", np.abs(x[r]).max())
print("bad fields:", nbad)
