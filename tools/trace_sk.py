#!/usr/bin/env python
"""Timeline of CTA 0 of the split-KV kernel (needs a -DDMA_TRACE build in DMA_LIB_PATH).

Roles: 0 / 1 = softmax WG0 / WG1 (warp quad 0), 2 = QK issuer, 3 = PV issuer."""
import bisect
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_03950_b200 as D  # noqa: E402
from paper_2604_03950_b200 import _lib  # noqa: E402

cfgn = sys.argv[1] if len(sys.argv) > 1 else "c3"
B, H, KVH, N, d, low = {"c3": (1, 32, 32, 32768, 128, D.NVFP4), "c2": (1, 32, 8, 8192, 128, D.MXFP4)}[cfgn]
cfg = D.AttentionConfig(tile_m=128, tile_n=128, diag_window=128, sink_window=128, low_format=low)
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(B, H, N, d, device="cuda", generator=g).to(torch.bfloat16)
k = torch.randn(B, KVH, N, d, device="cuda", generator=g).to(torch.bfloat16)
v = torch.randn(B, KVH, N, d, device="cuda", generator=g).to(torch.bfloat16)
a, out = D.DmaAttention(cfg).prepare(q, k, v)
L = _lib.lib()
sp = _lib.stream_ptr()
buf = (ctypes.c_ulonglong * (6 * 4096))()
cnt = (ctypes.c_uint * 6)()
_lib.check(L.dma_attention_quantize(a, sp), "q")
_lib.check(L.dma_attention_core(a, sp), "core")
torch.cuda.synchronize()
L.dma_trace_read(buf, cnt)
_lib.check(L.dma_attention_core(a, sp), "core")
torch.cuda.synchronize()
L.dma_trace_read(buf, cnt)
arr = np.frombuffer(buf, dtype=np.uint64).reshape(6, 4096)
t0 = min(int(arr[r][0] >> 8) for r in range(6) if cnt[r])
ev = {r: [(int(x >> 8) - t0, int(x & 255)) for x in arr[r][: min(cnt[r], 4096)]] for r in range(6)}
names = {1: "S ready", 2: "S loaded", 3: "m handed", 4: "exp start", 5: "exp end", 6: "P full", 7: "slow max", 8: "scaled", 9: "pre-pass start", 18: "K0 ready", 19: "K1 ready", 20: "SFK0 copied", 21: "SFK1 copied", 22: "V0 ready", 23: "V1 ready",
         30: "K issued", 31: "V issued",
         10: "QK0 go", 11: "QK1 go", 12: "QK0 issued", 13: "QK1 issued", 14: "PV0 go", 15: "PV1 go",
         16: "PV0 issued", 17: "PV1 issued"}
for r in range(6):
    e = ev[r]
    dd = {}
    for (t1, a1), (t2, a2) in zip(e, e[1:]):
        dd.setdefault((a1, a2), []).append(t2 - t1)
    print(f"role {['WG0', 'WG1', 'QK', 'PV', 'Kprod', 'Vprod'][r]}: {len(e)} events")
    for key, vals in sorted(dd.items()):
        if len(vals) > 10:
            print(f"  {names.get(key[0])} -> {names.get(key[1])}: median {np.median(vals):.0f} cyc  mean {np.mean(vals):.0f} (n={len(vals)})")
for w in (0, 1):
    n_slow = sum(1 for (t, a) in ev[w] if a == 7)
    n_t = sum(1 for (t, a) in ev[w] if a == 1)
    print(f"WG{w}: slow-path max on {n_slow} of {n_t} tiles")
# per-tile period of each WG (S ready -> next S ready)
for w in (0, 1):
    sr = [t for (t, a) in ev[w] if a == 1]
    if len(sr) > 20:
        dif = np.diff(sr[5:-5])
        print(f"WG{w}: S ready period median {np.median(dif):.0f} mean {np.mean(dif):.0f}")
# cross-role latencies
for w in (0, 1):
    pf = [t for (t, a) in ev[w] if a == 6]
    pv = [t for (t, a) in ev[3] if a == 14 + w]
    sl = [t for (t, a) in ev[w] if a == 2]
    qk = [t for (t, a) in ev[2] if a == 10 + w]
    d1 = [pv[i] - t for t in pf[5:-5] if (i := bisect.bisect_left(pv, t)) < len(pv)]
    d2 = [qk[i] - t for t in sl[5:-5] if (i := bisect.bisect_left(qk, t)) < len(qk)]
    if d1 and d2:
        print(f"WG{w}: P full -> PV go median {np.median(d1):.0f}; S loaded -> QK go median {np.median(d2):.0f}")
merged = sorted([(t, r, a) for r in range(6) for (t, a) in ev[r]])
mid = len(merged) // 2
print("timeline (cycles since start):")
for t, r, a in merged[mid:mid + 60]:
    print(f"  {t:10d} {['WG0', 'WG1', 'QK', 'PV', 'Kp', 'Vp'][r]:>4s} {names.get(a, a)}")
