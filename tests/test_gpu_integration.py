"""GPU: the reference-side binding of INTEGRATION.md (integration/mxattn_dma_cuda.py, pure
ctypes over libdma) driven with the LIVE reference package ``mxattn`` (the unmodified
reference installed in baseline/_ref, shipped to the GPU box): its AttentionConfig in, its
own mixed_precision_attention as the comparison (attention.py:282-310)."""

import importlib.util
import os
import sys

import numpy as np
import pytest

from conftest import record_parity
from test_gpu_attention import TOL, TOL_DEQ, errs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mx():
    if not os.path.isdir(os.path.join(REF, "mxattn")):
        pytest.skip("baseline/_ref (the reference install) is absent")
    sys.path.insert(0, REF)
    from mxattn import attention as A, formats as F, quantize as Q

    os.environ["DMA_LIB"] = os.path.join(ROOT, "paper_2604_03950_b200", "libdma.so")
    spec = importlib.util.spec_from_file_location("mxattn_dma_cuda", os.path.join(ROOT, "integration",
                                                                                  "mxattn_dma_cuda.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return A, F, Q, mod


CASES = [  # Lq, d, low, granularity, T, S, causal, dtype
    (512, 128, "nvfp4", "token", 128, 128, True, np.float64),
    (640, 64, "mxfp4", "tensor", 128, 0, True, np.float64),
    (384, 128, "nvfp4", "block", 128, 128, True, np.float64),
    (256, 128, "nvfp4", "token", 128, 128, False, np.float32),
]


@pytest.mark.parametrize("pv_mode", [0, 1])
@pytest.mark.parametrize("case", CASES)
def test_binding_matches_live_reference(mx, case, pv_mode):
    A, F, Q, mod = mx
    lq, d, low, gran, T, S, causal, dt = case
    rng = np.random.default_rng(lq + d)
    q, k, v = (rng.standard_normal((lq, d)).astype(dt) for _ in range(3))  # full-mantissa f64 / f32
    cfg = A.AttentionConfig(tile_m=128, tile_n=128, diag_window=T, sink_window=S, causal=causal,
                            low_format={"nvfp4": F.NVFP4, "mxfp4": F.MXFP4}[low],
                            granularity={"token": Q.Granularity.TOKEN, "tensor": Q.Granularity.TENSOR,
                                         "block": Q.Granularity.BLOCK}[gran])
    got = mod.mixed_precision_attention_cuda(q, k, v, cfg, pv_mode=pv_mode)
    want = A.mixed_precision_attention(q, k, v, cfg)
    assert got.shape == want.shape and got.dtype == np.float64
    rel, mxa = errs(got, want)
    record_parity(f"binding_{lq}_{d}_{low}_{gran}_{int(causal)}_{np.dtype(dt).name}", "mxfp8" if pv_mode == 0 else "bf16",
                  rel, mxa)
    tol = (TOL_DEQ if gran == "block" else TOL)["mxfp8" if pv_mode == 0 else "bf16"]
    assert rel <= tol[0] and mxa <= tol[1], (rel, mxa)


def test_binding_codes_bit_exact_f64(mx):
    """f64 inputs pass through unrounded: the kernel's quantize_dual equals the live reference's
    on full-mantissa f64 values (checked via the attention-independent entry point)."""
    A, F, Q, mod = mx
    import paper_2604_03950_b200 as D

    rng = np.random.default_rng(4)
    x = rng.standard_normal((64, 128)) * np.exp(rng.uniform(-3, 3, (64, 1)))
    r = Q.quantize_dual(x, is_query=True, low_format=F.NVFP4, high_format=F.MXFP8_E4M3)
    t = D.quantize_dual(x, True, D.NVFP4, D.MXFP8_E4M3)
    assert np.array_equal(t.high_codes, r.high_codes)
    assert np.array_equal(t.packed_low.bytes_, r.packed_low.bytes_)


def test_binding_nonfinite_raises(mx):
    A, F, Q, mod = mx
    q = np.ones((128, 64))
    q[3, 5] = np.nan
    cfg = A.AttentionConfig(tile_m=128, tile_n=128)
    with pytest.raises(ValueError, match="non-finite"):
        A.mixed_precision_attention(q, q, q, cfg)
    with pytest.raises(ValueError, match="non-finite"):
        mod.mixed_precision_attention_cuda(q, q, q, cfg)
