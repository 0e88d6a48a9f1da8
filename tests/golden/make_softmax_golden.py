"""Golden vectors for the tile-level softmax helpers (attention.py:83-106, 150-184), frozen
from the live reference (``/root/reference``; build container only):

    python tests/golden/make_softmax_golden.py   ->  tests/golden/softmax_golden.npz

Cases: a chain of online_softmax_update calls over random / partly -inf / fully masked
tiles (base 2 and base e), apply_causal_mask at several offsets, and normalized()."""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from mxattn import attention as A  # noqa: E402


def cases():
    rng = np.random.default_rng(2604)
    out = {}
    for ci, (rows, cols, d, base2) in enumerate([(8, 16, 4, True), (5, 7, 3, False), (16, 32, 8, True)]):
        st = A.OnlineSoftmaxState.fresh(rows, d)
        for t in range(4):
            s = rng.standard_normal((rows, cols)) * 3
            if t == 0:
                s[: rows // 2] = -np.inf           # rows with nothing seen yet
            if t == 2:
                s[:, ::3] = -np.inf                # partly masked tile
            s = A.apply_causal_mask(s, query_start=t * 2, key_start=t * 3) if t == 3 else s
            v = rng.standard_normal((cols, d))
            out[f"c{ci}_t{t}_scores"], out[f"c{ci}_t{t}_v"] = s, v
            st = A.online_softmax_update(st, s, v, base2=base2)
            out[f"c{ci}_t{t}_m"], out[f"c{ci}_t{t}_l"], out[f"c{ci}_t{t}_o"] = st.m, st.l, st.o
        out[f"c{ci}_norm"] = st.normalized()
        out[f"c{ci}_meta"] = np.array([rows, cols, d, int(base2)])
    for mi, (qs, ks) in enumerate([(0, 0), (5, 3), (0, 12), (40, 0)]):
        s = rng.standard_normal((9, 11))
        out[f"mask{mi}_in"], out[f"mask{mi}_out"] = s, A.apply_causal_mask(s, qs, ks)
        out[f"mask{mi}_meta"] = np.array([qs, ks])
    return out


if __name__ == "__main__":
    path = os.path.join(HERE, "softmax_golden.npz")
    np.savez_compressed(path, **cases())
    print("wrote", path)
