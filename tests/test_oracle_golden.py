"""Pin the CPU oracle (oracle/mx_oracle.py) to golden vectors frozen from the
live reference (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from inputs import randn_bf16
from cases import ATTN_CASES, SCORE_CASES
from oracle import mx_oracle as O

LOW = {"nvfp4": O.NVFP4, "mxfp4": O.MXFP4}
HIGH = {"mxfp8_e4m3": O.MXFP8_E4M3, "mxfp8_e5m2": O.MXFP8_E5M2}
FMT_ANY = {None: None, "nvfp4": O.NVFP4, "mxfp4": O.MXFP4, "mxfp8_e4m3": O.MXFP8_E4M3,
           "mxfp8_e5m2": O.MXFP8_E5M2}


def oracle_cfg(kw):
    kw = dict(kw)
    for key in ("low_format", "high_format"):
        if key in kw:
            kw[key] = FMT_ANY[kw[key]]
    return O.Cfg(**kw)


def test_e2m1_codec(golden):
    np.testing.assert_array_equal(O.encode_e2m1(golden["e2m1_x"]), golden["e2m1_codes"])
    codes = np.arange(16)
    np.testing.assert_array_equal(O.encode_e2m1(O.decode_e2m1(codes)) & 7, codes & 7)


@pytest.mark.parametrize("name,elem", [("e4m3", O.E4M3), ("e5m2", O.E5M2)])
def test_fp8_codec(golden, name, elem):
    np.testing.assert_array_equal(O.encode_fp8(golden[f"{name}_x"], elem), golden[f"{name}_codes"])
    np.testing.assert_array_equal(O.decode_fp8(np.arange(256), elem), golden[f"{name}_table"])


def test_quantize_dual_bit_exact(golden):
    keys = [str(k) for k in golden["quant_keys"]]
    assert len(keys) >= 96
    for key in keys:
        _, iname, lname, hname, gname, isq = key.split("/")
        x = golden[f"qin/{iname}"]
        t = O.quantize_dual(x, bool(int(isq)), LOW[lname], HIGH[hname], gname)
        np.testing.assert_array_equal(t.packed_low, golden[key + "/packed_low"], err_msg=key)
        np.testing.assert_array_equal(t.scales_low, golden[key + "/scales_low"], err_msg=key)
        np.testing.assert_array_equal(t.high_codes, golden[key + "/high_codes"], err_msg=key)
        np.testing.assert_array_equal(t.scales_high, golden[key + "/scales_high"], err_msg=key)
        qs = golden[key + "/quant_scale"]
        assert t.quant_scale.shape == qs.shape, key
        np.testing.assert_array_equal(t.quant_scale.view(np.uint64), qs.view(np.uint64), err_msg=key)
        if key + "/deq_low" in golden.files:
            np.testing.assert_array_equal(O.dequantize_low(t), golden[key + "/deq_low"], err_msg=key)
            np.testing.assert_array_equal(O.dequantize_high(t), golden[key + "/deq_high"], err_msg=key)


def test_plans(golden):
    cases, flat, offs = golden["plan_cases"], golden["plan_flat"], golden["plan_offs"]
    for i, (tm, tn, T, S, causal, lq, lk, qt) in enumerate(cases):
        cfg = O.Cfg(tile_m=int(tm), tile_n=int(tn), diag_window=int(T), sink_window=int(S),
                    causal=bool(causal))
        plan = O.tile_plan(int(qt), int(lq), int(lk), cfg)
        want = flat[offs[i]:offs[i + 1]]
        assert [2 * t + int(h) for t, h in plan] == list(want), (i, cases[i])


def test_high_precision_fraction(golden):
    for c, want in zip(golden["plan_cases"][:150], golden["hpf"]):
        tm, tn, T, S, causal, lq, lk, _ = (int(v) for v in c)
        assert O.high_precision_fraction(lq, lk, tm, tn, T, S, bool(causal)) == want
    for c, want in zip(golden["hpf_big_cases"], golden["hpf_big"]):
        lq, lk, tm, tn, T, S, causal = (int(v) for v in c)
        assert O.high_precision_fraction(lq, lk, tm, tn, T, S, bool(causal)) == want


@pytest.mark.parametrize("case", ATTN_CASES, ids=[c[0] for c in ATTN_CASES])
def test_attention(golden, case):
    name, lq, lk, d, dv, seed, kw = case
    q = randn_bf16(seed, lq, d)
    k = randn_bf16(seed + 1000, lk, d)
    v = randn_bf16(seed + 2000, lk, dv)
    got = O.mixed_precision_attention(q, k, v, oracle_cfg(kw))
    want = golden[f"attn/{name}"]
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-13)


def test_reference_attention_and_similarity(golden):
    q, k, v = randn_bf16(31, 96, 64), randn_bf16(32, 96, 64), randn_bf16(33, 96, 64)
    a = O.reference_attention(q, k, v, causal=True)
    b = O.reference_attention(q, k, v, causal=False)
    np.testing.assert_allclose(a, golden["refattn_causal"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(b, golden["refattn_full"], rtol=1e-12, atol=1e-14)
    s = O.similarity(a, b)
    np.testing.assert_allclose([s["cos_sim"], s["rel_l1"], s["abs_l1"], s["rmse"], s["psnr"]],
                               golden["similarity"], rtol=1e-12)


def test_reference_scores(golden):
    q, k = randn_bf16(31, 96, 64), randn_bf16(32, 96, 64)
    np.testing.assert_allclose(O.reference_scores(q, k, causal=True), golden["refscores_causal"], rtol=1e-12,
                               atol=1e-15)


@pytest.mark.parametrize("case", SCORE_CASES, ids=[c[0] for c in SCORE_CASES])
def test_mixed_precision_scores(golden, case):
    name, lq, d, seed, kw = case
    q, k = randn_bf16(seed, lq, d), randn_bf16(seed + 1, lq, d)
    np.testing.assert_allclose(O.mixed_precision_scores(q, k, oracle_cfg(kw)), golden[f"scores/{name}"],
                               rtol=1e-12, atol=1e-15)
