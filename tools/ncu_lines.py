#!/usr/bin/env python
"""Per-source-line warp-stall samples of an ncu report (top N lines), optionally
restricted to a line range of one file:  ncu_lines.py rep [N] [file:lo-hi]"""
import csv
import subprocess
import sys


def main(path, top=40, rng=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur, recs = None, []
    hdr = None
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) > 8 and r[0].isdigit() and r[2] == "-":
            ix = {h: i for i, h in enumerate(hdr)}
            st = {h: int(r[i] or 0) for h, i in ix.items() if h.startswith("stall_") and "Not" not in h
                  and (r[i] or "0").isdigit()}
            recs.append((int(r[4] or 0), cur, int(r[0]), r[1].strip()[:70],
                         int((r[7] or "0").replace(",", "")), st))
    tot = sum(x[0] for x in recs) or 1
    if rng:
        f, span = rng.split(":")
        lo, hi = map(int, span.split("-"))
        recs = [x for x in recs if x[1] == f and lo <= x[2] <= hi]
        print(f"range {rng}: {sum(x[0] for x in recs) / tot * 100:.1f}% of samples")
    for smp, f, ln, src, ex, st in sorted(recs, reverse=True)[:top]:
        top3 = sorted(st.items(), key=lambda kv: -kv[1])[:2]
        print(f"{smp / tot * 100:5.1f}% {f}:{ln:<4d} ex={ex / 1e6:7.1f}M {src:70s} "
              + " ".join(f"{k[6:]}={v / max(smp, 1) * 100:.0f}%" for k, v in top3))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40, sys.argv[3] if len(sys.argv) > 3 else None)
