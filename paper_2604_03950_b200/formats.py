"""MX number formats (drop-in for ``mxattn.formats``, formats.py:1-279).

Format constants mirror the reference registry (formats.py:57-112).  The
encoders run the device codec of libdma (the same code the fused kernel
uses: round-to-odd f64->f32 then ``cvt.rn.satfinite.{e2m1x2,e4m3x2,e5m2x2}``
plus the reference's signed-zero rules); decoders and nibble packing are
exact integer table lookups and stay on the host.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _lib
from ._device import from_device, to_device_f64


class ElementKind(Enum):
    E2M1 = "e2m1"
    E4M3 = "e4m3"
    E5M2 = "e5m2"


class ScaleKind(Enum):
    E8M0 = "e8m0"
    E4M3 = "e4m3"


@dataclass(frozen=True)
class ElementFormat:
    """formats.py:57-75."""

    kind: ElementKind
    bits: int
    exp_bits: int
    mant_bits: int
    bias: int
    e_max: int
    upper: float

    @property
    def lower(self) -> float:
        return -self.upper


E2M1 = ElementFormat(ElementKind.E2M1, bits=4, exp_bits=2, mant_bits=1, bias=1, e_max=2, upper=6.0)
E4M3 = ElementFormat(ElementKind.E4M3, bits=8, exp_bits=4, mant_bits=3, bias=7, e_max=8, upper=448.0)
E5M2 = ElementFormat(ElementKind.E5M2, bits=8, exp_bits=5, mant_bits=2, bias=15, e_max=15, upper=57344.0)


@dataclass(frozen=True)
class MxFormatSpec:
    """formats.py:86-98."""

    name: str
    element: ElementFormat
    scale_kind: ScaleKind
    block_size: int
    two_level: bool = True


MXFP8_E4M3 = MxFormatSpec("mxfp8_e4m3", E4M3, ScaleKind.E8M0, block_size=32)
MXFP8_E5M2 = MxFormatSpec("mxfp8_e5m2", E5M2, ScaleKind.E8M0, block_size=32)
MXFP4 = MxFormatSpec("mxfp4", E2M1, ScaleKind.E8M0, block_size=32, two_level=False)
NVFP4 = MxFormatSpec("nvfp4", E2M1, ScaleKind.E4M3, block_size=16)

FORMATS: dict[str, MxFormatSpec] = {f.name: f for f in (MXFP8_E4M3, MXFP8_E5M2, MXFP4, NVFP4)}
FORMATS["mxfp8"] = MXFP8_E4M3

E8M0_BIAS = 127
E8M0_MAX_RAW = 254

_FMT_CODE = {"mxfp8_e4m3": _lib.FMT_MXFP8_E4M3, "mxfp8_e5m2": _lib.FMT_MXFP8_E5M2,
             "mxfp4": _lib.FMT_MXFP4, "nvfp4": _lib.FMT_NVFP4}


def format_code(fmt: MxFormatSpec | None) -> int:
    return _lib.FMT_NONE if fmt is None else _FMT_CODE[fmt.name]


_E2M1_MAG = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0])


def _check_finite(x: np.ndarray, what: str) -> None:
    if not np.all(np.isfinite(x)):
        raise ValueError(f"{what}: input contains non-finite values")


def encode_e2m1(x) -> np.ndarray:
    """E2M1 codes, RNE ties-to-even (formats.py:124-145), on the GPU."""
    x = np.asarray(x, dtype=np.float64)
    _check_finite(x, "encode_e2m1")
    if np.any(np.abs(x) > 6.0):
        raise ValueError("encode_e2m1: input magnitude exceeds 6.0")
    dx = to_device_f64(x)
    import torch

    codes = torch.empty(dx.shape, dtype=torch.uint8, device=dx.device)
    _lib.check(_lib.lib().dma_encode_e2m1(dx.data_ptr(), dx.numel(), codes.data_ptr(), _lib.stream_ptr()),
               "encode_e2m1")
    return from_device(codes).reshape(x.shape)


def decode_e2m1(code) -> np.ndarray:
    """formats.py:148-151."""
    c = np.asarray(code).astype(np.int64) & 0xF
    mag = _E2M1_MAG[c & 7]
    return np.where(c & 8, -mag, mag)


@dataclass(frozen=True)
class PackedFp4Buffer:
    """formats.py:177-182."""

    bytes_: np.ndarray
    logical_len: int


def pack_fp4(codes) -> PackedFp4Buffer:
    """formats.py:154-165: byte = (odd << 4) | even, zero-padded odd tail."""
    c = np.asarray(codes, dtype=np.uint8).ravel() & 0xF
    n = c.size
    if n % 2:
        c = np.append(c, np.uint8(0))
    return PackedFp4Buffer(bytes_=((c[1::2] << 4) | c[0::2]).astype(np.uint8), logical_len=n)


def unpack_fp4(buf: PackedFp4Buffer) -> np.ndarray:
    """formats.py:168-174."""
    b = np.asarray(buf.bytes_, dtype=np.uint8).ravel()
    return np.stack([b & 0xF, b >> 4], axis=-1).ravel()[: buf.logical_len]


def e8m0_encode(e) -> np.ndarray:
    """formats.py:185-188."""
    return np.clip(np.asarray(e) + E8M0_BIAS, 0, E8M0_MAX_RAW).astype(np.uint8)


def e8m0_decode(raw) -> np.ndarray:
    """formats.py:191-194."""
    return np.exp2(np.asarray(raw).astype(np.float64) - E8M0_BIAS)


def _fp8(fmt):
    if isinstance(fmt, MxFormatSpec):
        fmt = fmt.element
    if fmt.kind not in (ElementKind.E4M3, ElementKind.E5M2):
        raise ValueError(f"not an 8-bit element format: {fmt.kind}")
    return fmt


def encode_fp8(x, fmt: ElementFormat) -> np.ndarray:
    """RNE-saturating FP8 encode, zero magnitudes -> +0 (formats.py:205-240), on the GPU."""
    fmt = _fp8(fmt)
    x = np.asarray(x, dtype=np.float64)
    _check_finite(x, "encode_fp8")
    dx = to_device_f64(x)
    import torch

    codes = torch.empty(dx.shape, dtype=torch.uint8, device=dx.device)
    _lib.check(_lib.lib().dma_encode_fp8(dx.data_ptr(), dx.numel(), int(fmt.kind is ElementKind.E5M2),
                                         codes.data_ptr(), _lib.stream_ptr()), "encode_fp8")
    return from_device(codes).reshape(x.shape)


_TABLES: dict[ElementKind, np.ndarray] = {}


def _fp8_table(fmt: ElementFormat) -> np.ndarray:
    t = _TABLES.get(fmt.kind)
    if t is None:
        c = np.arange(256)
        e = (c >> fmt.mant_bits) & ((1 << fmt.exp_bits) - 1)
        m = c & ((1 << fmt.mant_bits) - 1)
        frac = m / float(1 << fmt.mant_bits)
        mag = np.where(e > 0, np.ldexp(1.0 + frac, e - fmt.bias), np.ldexp(frac, 1 - fmt.bias))
        t = np.where(c >= 128, -mag, mag)
        if fmt.kind is ElementKind.E4M3:
            t = np.where((c & 0x7F) == 0x7F, np.nan, t)
        else:
            top = (1 << fmt.exp_bits) - 1
            t = np.where((e == top) & (m == 0), np.where(c >= 128, -np.inf, np.inf), t)
            t = np.where((e == top) & (m != 0), np.nan, t)
        _TABLES[fmt.kind] = t
    return t


def decode_fp8(code, fmt: ElementFormat) -> np.ndarray:
    """formats.py:243-279."""
    fmt = _fp8(fmt)
    return _fp8_table(fmt)[np.asarray(code, dtype=np.uint8)]
