"""Freeze golden vectors from the live reference (``/root/reference``).

Run in the build container (the reference is NOT present on GPU boxes):

    python tests/golden/make_golden.py

It imports the unmodified reference package ``mxattn`` from
``/root/reference/pkg/src`` and writes ``tests/golden/golden.npz``.  The
fixtures pin ``oracle/mx_oracle.py`` (tests/test_oracle_golden.py) and,
through the oracle, the CUDA path.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

from cases import ATTN_CASES, SCORE_CASES  # noqa: E402
from inputs import adversarial_rows, bf16_round, randn_bf16  # noqa: E402

from mxattn import attention as A  # noqa: E402
from mxattn import formats as F  # noqa: E402
from mxattn import metrics as M  # noqa: E402
from mxattn import quantize as Q  # noqa: E402

LOW = {"nvfp4": F.NVFP4, "mxfp4": F.MXFP4}
HIGH = {"mxfp8_e4m3": F.MXFP8_E4M3, "mxfp8_e5m2": F.MXFP8_E5M2}
GRAN = {"token": Q.Granularity.TOKEN, "block": Q.Granularity.BLOCK, "tensor": Q.Granularity.TENSOR}
FMT_ANY = {None: None, "nvfp4": F.NVFP4, "mxfp4": F.MXFP4, "mxfp8_e4m3": F.MXFP8_E4M3,
           "mxfp8_e5m2": F.MXFP8_E5M2}


def quant_inputs():
    rng = np.random.default_rng(123)
    return {
        "randn_64x128": randn_bf16(1, 64, 128),
        "adv_128": adversarial_rows(128),
        "adv_64": adversarial_rows(64, seed=9),
        "randn_16x256": randn_bf16(2, 16, 256),
        "f64_40x96": rng.standard_normal((40, 96)) * np.exp(rng.uniform(-4, 4, (40, 1))),
        "big_8x128": randn_bf16(3, 8, 128, scale=1000.0),
    }


FULL_SWEEP = {"randn_64x128", "adv_128", "adv_64"}



def make_cfg(kw):
    kw = dict(kw)
    for key in ("low_format", "high_format"):
        if key in kw:
            kw[key] = FMT_ANY[kw[key]]
    if "granularity" in kw:
        kw["granularity"] = GRAN[kw["granularity"]]
    return A.AttentionConfig(**kw)


def plan_cases(rng, n):
    out = []
    for _ in range(n):
        tm = int(rng.choice([16, 32, 64, 128, 256]))
        tn = int(rng.choice([16, 32, 64, 128, 256]))
        causal = bool(rng.integers(0, 2))
        lq = int(rng.integers(1, 1500))
        lk = lq if causal else int(rng.integers(1, 1500))
        T = tn * int(rng.integers(0, 12))
        S = tn * int(rng.integers(0, 6))
        qt = int(rng.integers(0, -(-lq // tm)))
        out.append((tm, tn, T, S, causal, lq, lk, qt))
    return out


def main():
    g = {}
    # --- codecs
    grid = np.linspace(-6, 6, 4801)
    mids = np.array([0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0])
    e2m1_x = np.concatenate([grid, mids, -mids, [0.0, -0.0, 6.0, -6.0, 1e-300, -1e-300]])
    g["e2m1_x"] = e2m1_x
    g["e2m1_codes"] = F.encode_e2m1(e2m1_x)
    for name, fmt in (("e4m3", F.E4M3), ("e5m2", F.E5M2)):
        dec = F.decode_fp8(np.arange(256, dtype=np.uint8), fmt)
        fin = np.sort(dec[np.isfinite(dec) & (dec >= 0)])
        midp = (fin[1:] + fin[:-1]) / 2
        rng = np.random.default_rng(5)
        xs = np.concatenate([fin, midp, np.nextafter(midp, 0), np.nextafter(midp, 1e9),
                             rng.uniform(0, fmt.upper, 3000), 2.0 ** rng.uniform(-30, 0, 2000)])
        xs = np.minimum(xs, fmt.upper)
        xs = np.concatenate([xs, -xs, [0.0, -0.0]])
        g[f"{name}_x"] = xs
        g[f"{name}_codes"] = F.encode_fp8(xs, fmt)
        g[f"{name}_table"] = dec

    # --- quantize_dual
    qnames = []
    for iname, x in quant_inputs().items():
        g[f"qin/{iname}"] = x
        for lname, low in LOW.items():
            for hname, high in HIGH.items():
                for gname, gran in GRAN.items():
                    for isq in (False, True):
                        if iname not in FULL_SWEEP and not (hname == "mxfp8_e4m3" and gname != "block"):
                            continue
                        key = f"q/{iname}/{lname}/{hname}/{gname}/{int(isq)}"
                        t = Q.quantize_dual(x, is_query=isq, low_format=low, high_format=high,
                                            granularity=gran)
                        g[key + "/packed_low"] = t.packed_low.bytes_
                        g[key + "/scales_low"] = t.scales_low
                        g[key + "/high_codes"] = t.high_codes
                        g[key + "/scales_high"] = t.scales_high
                        g[key + "/quant_scale"] = t.quant_scale
                        if iname in ("randn_64x128", "adv_64"):
                            g[key + "/deq_low"] = Q.dequantize_low(t)
                            g[key + "/deq_high"] = Q.dequantize_high(t)
                        qnames.append(key)
    g["quant_keys"] = np.array(qnames)

    # --- plans
    rng = np.random.default_rng(99)
    pcs = plan_cases(rng, 3000)
    flat, offs, hpf = [], [0], []
    for (tm, tn, T, S, causal, lq, lk, qt) in pcs:
        cfg = A.AttentionConfig(tile_m=tm, tile_n=tn, diag_window=T, sink_window=S, causal=causal)
        fn = A.causal_tile_plan if causal else A.noncausal_tile_plan
        plan = fn(qt, lq, lk, cfg)
        flat += [2 * t + int(h) for t, h in plan]
        offs.append(len(flat))
    g["plan_cases"] = np.array(pcs, dtype=np.int64)
    g["plan_flat"] = np.array(flat, dtype=np.int64)
    g["plan_offs"] = np.array(offs, dtype=np.int64)
    for (tm, tn, T, S, causal, lq, lk, qt) in pcs[:150]:
        hpf.append(M.high_precision_fraction(lq, lk, tm, tn, T, S, causal))
    g["hpf"] = np.array(hpf)
    big = [(1024, 1024, 128, 128, 128, 128, True), (8192, 8192, 128, 128, 128, 128, True),
           (32768, 32768, 128, 128, 128, 128, True), (16384, 16384, 128, 128, 0, 0, True),
           (16384, 16384, 128, 128, 2048, 2048, True), (4096, 4096, 64, 64, 128, 64, False)]
    g["hpf_big_cases"] = np.array(big, dtype=np.int64)
    g["hpf_big"] = np.array([M.high_precision_fraction(*c) for c in big])

    # --- attention
    for name, lq, lk, d, dv, seed, kw in ATTN_CASES:
        q = randn_bf16(seed, lq, d)
        k = randn_bf16(seed + 1000, lk, d)
        v = randn_bf16(seed + 2000, lk, dv)
        g[f"attn/{name}"] = A.mixed_precision_attention(q, k, v, make_cfg(kw))
    q = randn_bf16(31, 96, 64)
    k = randn_bf16(32, 96, 64)
    v = randn_bf16(33, 96, 64)
    g["refattn_causal"] = A.reference_attention(q, k, v, causal=True)
    g["refattn_full"] = A.reference_attention(q, k, v, causal=False)
    g["refscores_causal"] = A.reference_scores(q, k, causal=True)
    # --- mixed-precision score matrices (attention.py:313-335)
    for name, lq, d, seed, kw in SCORE_CASES:
        qq, kk = randn_bf16(seed, lq, d), randn_bf16(seed + 1, lq, d)
        g[f"scores/{name}"] = A.mixed_precision_scores(qq, kk, make_cfg(kw))
    rep = M.similarity(g["refattn_causal"], g["refattn_full"])
    g["similarity"] = np.array([rep.cos_sim, rep.rel_l1, rep.abs_l1, rep.rmse, rep.psnr])

    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **g)
    print(f"wrote {path}: {len(g)} arrays, {os.path.getsize(path) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
