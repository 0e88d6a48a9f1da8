#!/usr/bin/env python
"""Timeline of CTA 0 of the ping-pong kernel (needs a -DDMA_TRACE build in DMA_LIB_PATH)."""
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
ev = {}
t0 = min(int(arr[r][0] >> 8) for r in range(4) if cnt[r])
for r in range(4):
    n = min(cnt[r], 4096)
    ev[r] = [(int(x >> 8) - t0, int(x & 255)) for x in arr[r][:n]]
names = {1: "S ready", 2: "s_free", 3: "max done", 4: "exp start", 5: "exp end", 6: "P full",
         10: "QK_A go", 11: "QK_B go", 12: "QK_A issued", 13: "QK_B issued", 14: "PV_A go", 15: "PV_B go",
         16: "PV_A issued", 17: "PV_B issued", 18: "K_A ready", 19: "K_B ready", 20: "SF_K_A copied",
         21: "SF_K_B copied", 22: "V_A ready", 23: "V_B ready", 24: "PV_A committed", 25: "PV_B committed",
         26: "QK_A top", 27: "QK_B top", 28: "QK_A committed", 29: "QK_B committed"}
# per-stream phase durations (median over the middle of the trace)
for x in (0, 1):
    e = ev[x]
    d = {}
    for (t1, a1), (t2, a2) in zip(e, e[1:]):
        d.setdefault((a1, a2), []).append(t2 - t1)
    print(f"stream {'AB'[x]}: {len(e)} events")
    for key, vals in sorted(d.items()):
        if len(vals) > 10:
            print(f"  {names.get(key[0])} -> {names.get(key[1])}: median {np.median(vals):.0f} cyc  (n={len(vals)})")
for r in (2, 3):
    e = ev[r]
    dm = {}
    for (t1, a1), (t2, a2) in zip(e, e[1:]):
        dm.setdefault((a1, a2), []).append(t2 - t1)
    print(f"role {r} (MMA issuer / producer):")
    for key, vals in sorted(dm.items()):
        if len(vals) > 10:
            print(f"  {names.get(key[0])} -> {names.get(key[1])}: median {np.median(vals):.0f} cyc  (n={len(vals)})")

# cross-role: P full (stream x) -> next "PV_x go" / "PV_x issued" on the MMA issuer
mma = ev[2]
for x in (0, 1):
    pf = [t for (t, a) in ev[x] if a == 6]
    go = [t for (t, a) in mma if a == 14 + x]
    iss = [t for (t, a) in mma if a == 16 + x]
    import bisect
    d1, d2 = [], []
    for t in pf[5:-5]:
        i = bisect.bisect_left(go, t)
        if i < len(go):
            d1.append(go[i] - t)
        j = bisect.bisect_left(iss, t)
        if j < len(iss):
            d2.append(iss[j] - t)
    if d1:
        print(f"stream {'AB'[x]}: P full -> PV go median {np.median(d1):.0f}, -> PV issued median {np.median(d2):.0f}")
# window of the interleaved timeline
merged = sorted([(t, r, a) for r in range(4) for (t, a) in ev[r]])
mid = len(merged) // 2
print("timeline (cycles since start):")
for t, r, a in merged[mid:mid + 40]:
    print(f"  {t:10d} {['A', 'B', 'MMA', 'MMA2'][r]:>4s} {names.get(a, a)}")

# MUFU occupancy: union of the two streams' exp intervals ("exp start" -> "exp end") over the
# middle of the trace, and what each stream was doing when neither was in an exp phase
def intervals(x):
    e = ev[x]
    out, st = [], None
    for t, a in e:
        if a == 4:
            st = t
        elif a == 5 and st is not None:
            out.append((st, t))
            st = None
    return out


ia, ib = intervals(0), intervals(1)
if len(ia) > 20 and len(ib) > 20:
    lo = max(ia[5][0], ib[5][0])
    hi = min(ia[-5][1], ib[-5][1])
    span = hi - lo
    allv = sorted([(s, e_) for s, e_ in ia + ib if s >= lo and e_ <= hi])
    covered, cur_s, cur_e, gaps = 0, None, None, []
    for s_, e_ in allv:
        if cur_e is None or s_ > cur_e:
            if cur_e is not None:
                covered += cur_e - cur_s
                gaps.append((cur_e, s_))
            cur_s, cur_e = s_, e_
        else:
            cur_e = max(cur_e, e_)
    covered += cur_e - cur_s
    both = 0
    for s1, e1 in ia:
        for s2, e2 in ib:
            ov = min(e1, e2) - max(s1, s2)
            if ov > 0 and s1 >= lo and e1 <= hi:
                both += ov
    glen = [b - a for a, b in gaps]
    print(f"exp phases: A median {np.median([e_ - s for s, e_ in ia]):.0f} cyc, B median {np.median([e_ - s for s, e_ in ib]):.0f} cyc")
    print(f"window {span} cyc: some stream in exp {covered / span * 100:.1f} %, both {both / span * 100:.1f} %, "
          f"gaps {len(glen)} (median {np.median(glen) if glen else 0:.0f} cyc, total {sum(glen) / span * 100:.1f} %)")
    # what each stream was doing at gap midpoints: its last event before the midpoint
    from collections import Counter
    for x in (0, 1):
        c = Counter()
        ts = [t for t, a in ev[x]]
        for a, b in gaps:
            mid = (a + b) // 2
            i = bisect.bisect_right(ts, mid) - 1
            if i >= 0:
                c[names.get(ev[x][i][1], ev[x][i][1])] += 1
        print(f"  stream {'AB'[x]} during gaps (last event before): {dict(c.most_common(5))}")
