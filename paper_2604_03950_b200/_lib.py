"""ctypes binding of ``libdma.so`` (include/dma.h).

The shared library is built in-tree by ``make`` (or ``__graft_entry__.build()``)
and lives next to this file.  There is no fallback: if the library is missing
or the GPU is absent, every compute entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DMA_LIB_PATH") or os.path.join(_HERE, "libdma.so")

DMA_EINVAL = -1
DMA_EUNSUPPORTED = -2

FMT_NONE, FMT_MXFP8_E4M3, FMT_MXFP8_E5M2, FMT_MXFP4, FMT_NVFP4 = 0, 1, 2, 3, 4
GRAN_TOKEN, GRAN_BLOCK, GRAN_TENSOR = 0, 1, 2
DT_F64, DT_F32, DT_BF16 = 0, 1, 2
PV_MXFP8, PV_BF16 = 0, 1


class DmaQuantArgs(C.Structure):
    _fields_ = [
        ("x", C.c_void_p),
        ("x_dtype", C.c_int32),
        ("is_query", C.c_int32),
        ("n_mat", C.c_int64),
        ("rows", C.c_int64),
        ("cols", C.c_int64),
        ("mat_stride", C.c_int64),
        ("row_stride", C.c_int64),
        ("prescale", C.c_double),
        ("low_format", C.c_int32),
        ("high_format", C.c_int32),
        ("granularity", C.c_int32),
        ("kv_split", C.c_int32),
        ("packed_low", C.c_void_p),
        ("scales_low", C.c_void_p),
        ("high_codes", C.c_void_p),
        ("scales_high", C.c_void_p),
        ("quant_scale", C.c_void_p),
        ("nonfinite", C.c_void_p),
        ("workspace", C.c_void_p),
        ("workspace_bytes", C.c_size_t),
    ]


class DmaAttnArgs(C.Structure):
    _fields_ = [
        ("q", C.c_void_p),
        ("k", C.c_void_p),
        ("v", C.c_void_p),
        ("o", C.c_void_p),
        ("in_dtype", C.c_int32),
        ("out_dtype", C.c_int32),
        ("batch", C.c_int64),
        ("heads", C.c_int64),
        ("kv_heads", C.c_int64),
        ("len_q", C.c_int64),
        ("len_k", C.c_int64),
        ("head_dim", C.c_int64),
        ("v_dim", C.c_int64),
        ("tile_m", C.c_int32),
        ("tile_n", C.c_int32),
        ("diag_window", C.c_int32),
        ("sink_window", C.c_int32),
        ("causal", C.c_int32),
        ("low_format", C.c_int32),
        ("high_format", C.c_int32),
        ("granularity", C.c_int32),
        ("pv_mode", C.c_int32),
        ("kv_split", C.c_int32),
        ("prescale", C.c_double),
        ("workspace", C.c_void_p),
        ("workspace_bytes", C.c_size_t),
        ("nonfinite", C.c_void_p),
    ]


ABI_VERSION = 2
_lib = None


class DmaError(RuntimeError):
    pass


class DmaUnsupported(DmaError):
    pass


def lib():
    """Load libdma.so once; raise loudly if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DmaError(f"{LIB_PATH} not found: build it with `make` (or __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, f64, sz = C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_size_t
        L.dma_last_error.restype = C.c_char_p
        L.dma_abi_version.restype = C.c_int
        L.dma_last_launch_count.restype = C.c_int
        L.dma_attention_set_fused.restype = C.c_int
        L.dma_attention_set_fused.argtypes = [C.c_int]
        L.dma_attention_set_kv_split.restype = C.c_int
        L.dma_attention_set_kv_split.argtypes = [C.c_int]
        L.dma_attention_kv_split.restype = C.c_int
        L.dma_attention_kv_split.argtypes = [C.POINTER(DmaAttnArgs)]
        L.dma_quantize_workspace_bytes.restype = sz
        L.dma_quantize_workspace_bytes.argtypes = [C.POINTER(DmaQuantArgs)]
        L.dma_quantize_dual.argtypes = [C.POINTER(DmaQuantArgs), vp]
        L.dma_dequantize.argtypes = [i32, i32, i32, i32, i64, i64, i64, vp, vp, vp, vp, vp, vp, vp]
        L.dma_encode_e2m1.argtypes = [vp, i64, vp, vp]
        L.dma_encode_fp8.argtypes = [vp, i64, i32, vp, vp]
        L.dma_attention_workspace_bytes.restype = sz
        L.dma_attention_workspace_bytes.argtypes = [C.POINTER(DmaAttnArgs)]
        L.dma_attention_supported.argtypes = [C.POINTER(DmaAttnArgs)]
        L.dma_attention_fwd.argtypes = [C.POINTER(DmaAttnArgs), vp]
        L.dma_attention_quantize.argtypes = [C.POINTER(DmaAttnArgs), vp]
        L.dma_attention_core.argtypes = [C.POINTER(DmaAttnArgs), vp]
        L.dma_tile_plan.restype = i64
        L.dma_tile_plan.argtypes = [i64, i64, i64, i32, i32, i32, i32, i32, C.POINTER(C.c_int64), i64]
        L.dma_high_precision_fraction.restype = f64
        L.dma_high_precision_fraction.argtypes = [i64, i64, i32, i32, i32, i32, i32]
        L.dma_selftest_mma.argtypes = [i32, i32, vp, vp, vp, vp, vp, vp]
        for name in ("dma_quantize_dual", "dma_dequantize", "dma_encode_e2m1", "dma_encode_fp8",
                     "dma_attention_supported", "dma_attention_fwd", "dma_attention_quantize",
                     "dma_attention_core", "dma_selftest_mma"):
            getattr(L, name).restype = C.c_int
        if L.dma_abi_version() != ABI_VERSION:
            raise DmaError(f"{LIB_PATH}: ABI {L.dma_abi_version()} != {ABI_VERSION} expected: rebuild with `make`")
        _lib = L
    return _lib


def check(rc: int, what: str) -> None:
    if rc == 0:
        return
    msg = lib().dma_last_error().decode(errors="replace")
    if rc == DMA_EUNSUPPORTED:
        raise DmaUnsupported(f"{what}: unsupported configuration: {msg}")
    if rc < 0:
        raise ValueError(f"{what}: {msg}")
    raise DmaError(f"{what}: CUDA error {rc}: {msg}")


EXPORTED_SYMBOLS = (
    "dma_quantize_workspace_bytes", "dma_quantize_dual", "dma_dequantize", "dma_encode_e2m1",
    "dma_encode_fp8", "dma_attention_workspace_bytes", "dma_attention_supported", "dma_attention_fwd",
    "dma_attention_quantize", "dma_attention_core", "dma_tile_plan", "dma_high_precision_fraction",
    "dma_selftest_mma", "dma_last_error", "dma_abi_version", "dma_last_launch_count",
    "dma_decode_workspace_bytes", "dma_decode_attention", "dma_attention_set_fused",
    "dma_attention_set_kv_split", "dma_attention_kv_split",
)


def stream_ptr(stream=None) -> int:
    """Raw cudaStream_t of a torch stream (current stream by default)."""
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
