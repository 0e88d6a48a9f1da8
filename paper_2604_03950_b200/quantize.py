"""Dual mixed-precision block quantization on the GPU (drop-in for ``mxattn.quantize``).

``quantize_dual`` runs phase 1 of the fused DMA kernel (csrc/quant.cuh) and
returns codes/scales that are bit-identical to the reference's
``quantize_dual`` (quantize.py:122-212).  numpy in -> numpy out (drop-in);
a CUDA torch tensor in -> CUDA torch tensors out (no host round trip).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _lib
from ._device import dtype_code, from_device, is_torch, to_device
from .formats import (
    MXFP8_E4M3,
    NVFP4,
    ElementKind,
    MxFormatSpec,
    PackedFp4Buffer,
    format_code,
)

QUANT_RANGE = 448.0 * 6.0  # quantize.py:54


class Granularity(Enum):
    """quantize.py:61-66."""

    TENSOR = "tensor"
    BLOCK = "block"
    TOKEN = "token"


_GRAN_CODE = {Granularity.TOKEN: _lib.GRAN_TOKEN, Granularity.BLOCK: _lib.GRAN_BLOCK,
              Granularity.TENSOR: _lib.GRAN_TENSOR}


def granularity_code(g: Granularity) -> int:
    if g not in _GRAN_CODE:
        raise ValueError(f"unknown granularity: {g!r}")
    return _GRAN_CODE[g]


@dataclass
class DualQuantizedTensor:
    """quantize.py:69-89 (arrays are numpy, or CUDA tensors for CUDA inputs)."""

    shape: tuple
    low_format: MxFormatSpec
    high_format: MxFormatSpec
    granularity: Granularity
    packed_low: PackedFp4Buffer
    scales_low: object
    high_codes: object
    scales_high: object
    quant_scale: object
    softmax_prescaled: bool


def prescale_constant(d: int) -> float:
    """log2(e)/sqrt(D) in float64, exactly as quantize.py:95 computes it."""
    return math.log2(math.e) / math.sqrt(d)


def softmax_prescale(x):
    """quantize.py:92-95 (host helper; the kernel folds the same constant)."""
    return x * prescale_constant(x.shape[-1])


def _validate(x_shape, low_format, high_format):
    if len(x_shape) != 2:
        raise ValueError(f"expected a 2-D tensor, got shape {tuple(x_shape)}")
    rows, cols = x_shape
    if cols % 32 != 0:
        raise ValueError(f"column count {cols} not divisible by 32")
    if low_format.element.kind is not ElementKind.E2M1:
        raise ValueError(f"low format must have E2M1 elements, got {low_format.name}")
    if high_format.element.bits != 8:
        raise ValueError(f"high format must have FP8 elements, got {high_format.name}")
    return rows, cols


def quantize_dual(x, is_query: bool = False, low_format: MxFormatSpec = NVFP4,
                  high_format: MxFormatSpec = MXFP8_E4M3,
                  granularity: Granularity = Granularity.TOKEN) -> DualQuantizedTensor:
    """Paper Alg. 2 on the GPU; bit-exact with quantize.py:122-212."""
    import torch

    torch_in = is_torch(x)
    if not torch_in:
        x = np.asarray(x, dtype=np.float64)
    rows, cols = _validate(tuple(x.shape), low_format, high_format)
    if not torch_in and not np.all(np.isfinite(x)):
        raise ValueError("quantize_dual: input contains non-finite values")
    gcode = granularity_code(granularity)
    dx = to_device(x)
    dev = dx.device
    nsf_low = cols // low_format.block_size
    u8 = dict(dtype=torch.uint8, device=dev)
    packed = torch.empty((rows, cols // 2), **u8)
    sl = torch.empty((rows, nsf_low), **u8)
    hc = torch.empty((rows, cols), **u8)
    sh = torch.empty((rows, cols // 32), **u8)
    qshape = {Granularity.TOKEN: (rows, 1), Granularity.BLOCK: (rows, cols // 32),
              Granularity.TENSOR: (1, 1)}[granularity]
    qs = torch.empty(qshape, dtype=torch.float64, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = torch.empty(8, dtype=torch.uint8, device=dev)
    a = _lib.DmaQuantArgs()
    a.x = dx.data_ptr()
    a.x_dtype = dtype_code(dx)
    a.is_query = int(bool(is_query))
    a.n_mat, a.rows, a.cols = 1, rows, cols
    a.mat_stride, a.row_stride = rows * cols, cols
    a.prescale = prescale_constant(cols)
    a.low_format, a.high_format, a.granularity = format_code(low_format), format_code(high_format), gcode
    a.packed_low, a.scales_low, a.high_codes = packed.data_ptr(), sl.data_ptr(), hc.data_ptr()
    a.scales_high, a.quant_scale, a.nonfinite = sh.data_ptr(), qs.data_ptr(), flag.data_ptr()
    a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
    if rows > 0:
        _lib.check(_lib.lib().dma_quantize_dual(a, _lib.stream_ptr()), "quantize_dual")
    if torch_in:
        if int(flag.item()):
            raise ValueError("quantize_dual: input contains non-finite values")
        conv = lambda t: t  # noqa: E731
    else:
        conv = from_device
    return DualQuantizedTensor(
        shape=(rows, cols), low_format=low_format, high_format=high_format, granularity=granularity,
        packed_low=PackedFp4Buffer(bytes_=conv(packed), logical_len=rows * cols),
        scales_low=conv(sl), high_codes=conv(hc), scales_high=conv(sh), quant_scale=conv(qs),
        softmax_prescaled=bool(is_query))


def _dequant(t: DualQuantizedTensor, which: int):
    import torch

    rows, cols = t.shape
    torch_in = is_torch(t.high_codes)
    dev = lambda a: (a if torch_in else torch.from_numpy(np.ascontiguousarray(a))).cuda()  # noqa: E731
    pl, sl, hc = dev(t.packed_low.bytes_), dev(t.scales_low), dev(t.high_codes)
    sh, qs = dev(t.scales_high), dev(np.asarray(t.quant_scale, dtype=np.float64) if not torch_in else t.quant_scale)
    out = torch.empty((rows, cols), dtype=torch.float64, device="cuda")
    if rows:
        _lib.check(_lib.lib().dma_dequantize(
            which, format_code(t.low_format), format_code(t.high_format), granularity_code(t.granularity),
            1, rows, cols, pl.data_ptr(), sl.data_ptr(), hc.data_ptr(), sh.data_ptr(), qs.data_ptr(),
            out.data_ptr(), _lib.stream_ptr()), "dequantize")
    return out if torch_in else from_device(out)


def dequantize_low(t: DualQuantizedTensor):
    """quantize.py:215-229: the tensor as the 4-bit path sees it."""
    return _dequant(t, 0)


def dequantize_high(t: DualQuantizedTensor):
    """quantize.py:232-237: the tensor as the 8-bit path sees it."""
    return _dequant(t, 1)
