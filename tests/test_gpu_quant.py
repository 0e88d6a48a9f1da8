"""GPU: bit-exact parity of phase 1 (quantize_dual) and the element codecs
with the oracle and with the golden vectors frozen from the reference."""

import numpy as np
import pytest

from inputs import adversarial_rows, randn_bf16
from oracle import mx_oracle as O

pytestmark = pytest.mark.gpu


def dma():
    import paper_2604_03950_b200 as D

    return D


def fmt_pair(lname, hname):
    D = dma()
    return ({"nvfp4": D.NVFP4, "mxfp4": D.MXFP4}[lname],
            {"mxfp8_e4m3": D.MXFP8_E4M3, "mxfp8_e5m2": D.MXFP8_E5M2}[hname])


GR = {"token": "TOKEN", "block": "BLOCK", "tensor": "TENSOR"}


def assert_same(t, want, key):
    np.testing.assert_array_equal(t.packed_low.bytes_, want["packed_low"], err_msg=key + " packed_low")
    np.testing.assert_array_equal(t.scales_low, want["scales_low"], err_msg=key + " scales_low")
    np.testing.assert_array_equal(t.high_codes, want["high_codes"], err_msg=key + " high_codes")
    np.testing.assert_array_equal(t.scales_high, want["scales_high"], err_msg=key + " scales_high")
    qs = np.asarray(want["quant_scale"])
    assert np.asarray(t.quant_scale).shape == qs.shape, key
    np.testing.assert_array_equal(np.asarray(t.quant_scale).view(np.uint64), qs.view(np.uint64),
                                  err_msg=key + " quant_scale")


def test_quantize_dual_golden(golden):
    D = dma()
    for key in [str(k) for k in golden["quant_keys"]]:
        _, iname, lname, hname, gname, isq = key.split("/")
        low, high = fmt_pair(lname, hname)
        t = D.quantize_dual(golden[f"qin/{iname}"], bool(int(isq)), low, high, getattr(D.Granularity, GR[gname]))
        want = {f: golden[f"{key}/{f}"] for f in ("packed_low", "scales_low", "high_codes", "scales_high",
                                                     "quant_scale")}
        assert_same(t, want, key)
        if key + "/deq_low" in golden.files:
            np.testing.assert_array_equal(D.dequantize_low(t), golden[key + "/deq_low"], err_msg=key)
            np.testing.assert_array_equal(D.dequantize_high(t), golden[key + "/deq_high"], err_msg=key)


@pytest.mark.parametrize("lname", ["nvfp4", "mxfp4"])
@pytest.mark.parametrize("hname", ["mxfp8_e4m3", "mxfp8_e5m2"])
@pytest.mark.parametrize("gname", ["token", "block", "tensor"])
@pytest.mark.parametrize("isq", [False, True])
def test_quantize_dual_vs_oracle_large(lname, hname, gname, isq):
    """c3-shaped slice (8192 x 128 bf16 rows + adversarial rows), bit-exact."""
    D = dma()
    low, high = fmt_pair(lname, hname)
    x = np.concatenate([randn_bf16(7, 8192, 128), adversarial_rows(128)])
    t = D.quantize_dual(x, isq, low, high, getattr(D.Granularity, GR[gname]))
    ol = {"nvfp4": O.NVFP4, "mxfp4": O.MXFP4}[lname]
    oh = {"mxfp8_e4m3": O.MXFP8_E4M3, "mxfp8_e5m2": O.MXFP8_E5M2}[hname]
    r = O.quantize_dual(x, isq, ol, oh, gname)
    want = dict(packed_low=r.packed_low, scales_low=r.scales_low, high_codes=r.high_codes,
                scales_high=r.scales_high, quant_scale=r.quant_scale)
    assert_same(t, want, f"{lname}/{hname}/{gname}/{isq}")


def test_quantize_dual_d64_and_wide():
    D = dma()
    for cols in (32, 64, 96, 256, 1024):
        x = randn_bf16(cols, 300, cols, scale=3.0)
        t = D.quantize_dual(x, True, D.NVFP4, D.MXFP8_E4M3, D.Granularity.TOKEN)
        r = O.quantize_dual(x, True, O.NVFP4, O.MXFP8_E4M3, "token")
        assert_same(t, dict(packed_low=r.packed_low, scales_low=r.scales_low, high_codes=r.high_codes,
                            scales_high=r.scales_high, quant_scale=r.quant_scale), f"cols={cols}")


def test_quantize_dual_torch_inputs():
    import torch

    D = dma()
    x = torch.from_numpy(randn_bf16(5, 1000, 128)).to(torch.bfloat16).cuda()
    t = D.quantize_dual(x, False, D.MXFP4, D.MXFP8_E4M3, D.Granularity.TOKEN)
    r = O.quantize_dual(x.double().cpu().numpy(), False, O.MXFP4, O.MXFP8_E4M3, "token")
    np.testing.assert_array_equal(t.high_codes.cpu().numpy(), r.high_codes)
    np.testing.assert_array_equal(t.packed_low.bytes_.cpu().numpy(), r.packed_low)
    bad = x.clone()
    bad[3, 5] = float("nan")
    with pytest.raises(ValueError, match="non-finite"):
        D.quantize_dual(bad)


def test_quantize_dual_errors():
    D = dma()
    with pytest.raises(ValueError, match="2-D"):
        D.quantize_dual(np.zeros(32))
    with pytest.raises(ValueError, match="divisible by 32"):
        D.quantize_dual(np.zeros((2, 48)))
    with pytest.raises(ValueError, match="non-finite"):
        D.quantize_dual(np.array([[np.inf] * 32]))
    with pytest.raises(ValueError, match="E2M1"):
        D.quantize_dual(np.zeros((2, 32)), low_format=D.MXFP8_E4M3)
    with pytest.raises(ValueError, match="FP8"):
        D.quantize_dual(np.zeros((2, 32)), high_format=D.NVFP4)
    t = D.quantize_dual(np.zeros((0, 64)))
    assert t.high_codes.shape == (0, 64)


def test_codecs_golden(golden):
    D = dma()
    np.testing.assert_array_equal(D.encode_e2m1(golden["e2m1_x"]), golden["e2m1_codes"])
    np.testing.assert_array_equal(D.encode_fp8(golden["e4m3_x"], D.E4M3), golden["e4m3_codes"])
    np.testing.assert_array_equal(D.encode_fp8(golden["e5m2_x"], D.E5M2), golden["e5m2_codes"])
    # SPEC KATs
    assert int(D.encode_e2m1(5.0)) == 0b0110
    assert int(D.encode_e2m1(-1.3)) == 0b1011
    assert int(D.encode_e2m1(0.25)) == 0
    assert int(D.encode_fp8(448.0, D.E4M3)) == 0x7E
    assert int(D.encode_fp8(57344.0, D.E5M2)) == 0x7B
    assert int(D.encode_fp8(1.0, D.E4M3)) == 0x38
    with pytest.raises(ValueError):
        D.encode_e2m1(6.5)
    with pytest.raises(ValueError):
        D.encode_fp8(np.nan, D.E4M3)


@pytest.mark.parametrize("dtype", ["float32", "float64"])
@pytest.mark.parametrize("gran", ["token", "tensor", "block"])
def test_quantize_dual_full_precision_inputs(dtype, gran):
    """f32 / f64 inputs with full-width mantissas (not bf16-representable): the quant16 f32
    path and the IEEE-division f64 path, bit-exact against the oracle, as query and as key."""
    import torch

    D = dma()
    rng = np.random.default_rng(11)
    x = rng.standard_normal((777, 128)) * np.exp(rng.uniform(-3, 3, size=(777, 1)))
    x[5] = 0.0
    x[6, :32] = 1e-30  # tiny block next to normal ones
    xt = torch.from_numpy(x.astype(dtype)).cuda()
    xd = xt.double().cpu().numpy()
    G = {"token": D.Granularity.TOKEN, "tensor": D.Granularity.TENSOR, "block": D.Granularity.BLOCK}[gran]
    for isq in (True, False):
        t = D.quantize_dual(xt, isq, D.NVFP4, D.MXFP8_E4M3, G)
        r = O.quantize_dual(xd, isq, O.NVFP4, O.MXFP8_E4M3, gran)
        np.testing.assert_array_equal(t.high_codes.cpu().numpy(), r.high_codes)
        np.testing.assert_array_equal(t.scales_high.cpu().numpy(), r.scales_high)
        np.testing.assert_array_equal(t.packed_low.bytes_.cpu().numpy(), r.packed_low)
        np.testing.assert_array_equal(t.scales_low.cpu().numpy(), r.scales_low)
        np.testing.assert_array_equal(t.quant_scale.cpu().numpy().ravel(), np.asarray(r.quant_scale).ravel())


def _np(a):
    return a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)


def _assert_same_t(t, r, key):
    np.testing.assert_array_equal(_np(t.packed_low.bytes_), r.packed_low, err_msg=key + " packed_low")
    np.testing.assert_array_equal(_np(t.scales_low), r.scales_low, err_msg=key + " scales_low")
    np.testing.assert_array_equal(_np(t.high_codes), r.high_codes, err_msg=key + " high_codes")
    np.testing.assert_array_equal(_np(t.scales_high), r.scales_high, err_msg=key + " scales_high")
    np.testing.assert_array_equal(_np(t.quant_scale).view(np.uint64), np.asarray(r.quant_scale).view(np.uint64),
                                  err_msg=key + " quant_scale")


@pytest.mark.parametrize("lname", ["nvfp4", "mxfp4"])
@pytest.mark.parametrize("hname", ["mxfp8_e4m3", "mxfp8_e5m2"])
@pytest.mark.parametrize("gname", ["token", "block", "tensor"])
@pytest.mark.parametrize("isq", [False, True])
def test_quantize_dual_bf16_device_inputs(lname, hname, gname, isq):
    """The forward's phase-1 kernel (bf16 device inputs: 32 columns per thread, float32 fast
    path + float64 redo of flagged pairs) bit-exact against the oracle, on random rows, the
    adversarial rows and rows whose maximum has a 21 * 2^k mantissa (many exact ties)."""
    import torch

    D = dma()
    low, high = fmt_pair(lname, hname)
    rng = np.random.default_rng(11)
    ties = randn_bf16(12, 512, 128)
    for i, m in enumerate((147, 168, 189, 210, 231, 252, 192, 224)):
        ties[64 * i:64 * i + 64, 7] = m * 2.0 ** -6
        ties[64 * i:64 * i + 64] = np.clip(ties[64 * i:64 * i + 64], -m * 2.0 ** -6, m * 2.0 ** -6)
    ties[:, 20:40] = np.round(ties[:, 20:40] * 16) / 16  # short mantissas: exact quotients
    x = np.concatenate([randn_bf16(7, 4096, 128), adversarial_rows(128), ties,
                        randn_bf16(8, 33, 128, scale=float(rng.uniform(1e-3, 1e3)))])
    xt = torch.from_numpy(x).to(torch.bfloat16)
    x = xt.double().numpy()  # the oracle sees the bf16 values
    t = D.quantize_dual(xt.cuda(), isq, low, high, getattr(D.Granularity, GR[gname]))
    ol = {"nvfp4": O.NVFP4, "mxfp4": O.MXFP4}[lname]
    oh = {"mxfp8_e4m3": O.MXFP8_E4M3, "mxfp8_e5m2": O.MXFP8_E5M2}[hname]
    _assert_same_t(t, O.quantize_dual(x, isq, ol, oh, gname), f"bf16/{lname}/{hname}/{gname}/{isq}")


@pytest.mark.parametrize("cols", [32, 64, 256, 512])
def test_quantize_dual_bf16_widths(cols):
    import torch

    D = dma()
    xt = torch.from_numpy(np.concatenate([randn_bf16(cols + 1, 301, cols, scale=2.0), adversarial_rows(cols)]))
    xt = xt.to(torch.bfloat16)
    x = xt.double().numpy()
    for isq, gname in ((True, "token"), (False, "block")):
        t = D.quantize_dual(xt.cuda(), isq, D.NVFP4, D.MXFP8_E4M3,
                            getattr(D.Granularity, GR[gname]))
        _assert_same_t(t, O.quantize_dual(x, isq, O.NVFP4, O.MXFP8_E4M3, gname), f"cols={cols}/{gname}")
