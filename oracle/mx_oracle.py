"""CPU oracle for the DMA forward path -- TEST INFRASTRUCTURE ONLY.

This module is a float64 numpy restatement of the reference package
``mxattn`` (``/root/reference/pkg/src/mxattn``).  It is the *checker* the
CUDA path is compared against; nothing in ``paper_2604_03950_b200`` may
import it.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` use it.

Parity pinning: every function here is checked against golden vectors
produced by the live reference (``tests/golden/make_golden.py`` imports
``/root/reference`` and freezes outputs to ``tests/golden/*.npz``), see
``tests/test_oracle_golden.py``.

Each function cites the reference file:line it restates.  The arithmetic
order of every float64 operation that feeds a rounding decision follows
the reference exactly (that is what makes codes bit-exact); the
structure of the code is our own.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

# ---------------------------------------------------------------------------
# Formats (formats.py:57-112)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Elem:
    """Element format constants (formats.py:78-83)."""

    name: str
    bits: int
    mant: int
    bias: int
    e_max: int
    upper: float


E2M1 = Elem("e2m1", 4, 1, 1, 2, 6.0)
E4M3 = Elem("e4m3", 8, 3, 7, 8, 448.0)
E5M2 = Elem("e5m2", 8, 2, 15, 15, 57344.0)


@dataclass(frozen=True)
class Fmt:
    """MX format = element + scale kind + block size (formats.py:86-104)."""

    name: str
    elem: Elem
    scale: str  # "e8m0" | "e4m3"
    block: int
    two_level: bool = True


MXFP8_E4M3 = Fmt("mxfp8_e4m3", E4M3, "e8m0", 32)
MXFP8_E5M2 = Fmt("mxfp8_e5m2", E5M2, "e8m0", 32)
MXFP4 = Fmt("mxfp4", E2M1, "e8m0", 32, two_level=False)
NVFP4 = Fmt("nvfp4", E2M1, "e4m3", 16)
FORMATS = {f.name: f for f in (MXFP8_E4M3, MXFP8_E5M2, MXFP4, NVFP4)}
FORMATS["mxfp8"] = MXFP8_E4M3  # formats.py:109

QUANT_RANGE = 2688.0  # 448 * 6, quantize.py:54
E4M3_TINY = 2.0 ** -9  # quantize.py:58

# ---------------------------------------------------------------------------
# Codecs (formats.py:119-279)
# ---------------------------------------------------------------------------

_E2M1_GRID = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0])


def _finite_or_raise(x, who):
    if not np.isfinite(x).all():
        raise ValueError(f"{who}: input contains non-finite values")


def encode_e2m1(x) -> np.ndarray:
    """Nearest E2M1 code, ties to the even (M=0) code (formats.py:124-145).

    Restated as a nearest-grid search: the lower neighbour index ``lo`` and
    upper ``lo+1``; a strict ``>`` on the midpoint picks the upper one, an
    exact midpoint picks whichever index is even -- on this grid the even
    index is always the one with mantissa 0, as in formats.py:143.
    """
    x = np.asarray(x, dtype=np.float64)
    _finite_or_raise(x, "encode_e2m1")
    a = np.abs(x)
    if (a > 6.0).any():
        raise ValueError("encode_e2m1: input magnitude exceeds 6.0")
    lo = np.clip(np.searchsorted(_E2M1_GRID, a, side="right") - 1, 0, 6)
    hi = lo + 1
    mid = (_E2M1_GRID[lo] + _E2M1_GRID[hi]) * 0.5
    idx = np.where(a > mid, hi, np.where(a < mid, lo, np.where(lo % 2 == 0, lo, hi)))
    idx = np.where(a == 6.0, 7, idx)
    neg = np.signbit(x) & (a > 0)  # exact -0.0 -> +0 (formats.py:144)
    return (idx | (neg.astype(np.int64) << 3)).astype(np.uint8)


def decode_e2m1(code) -> np.ndarray:
    """formats.py:148-151."""
    c = np.asarray(code).astype(np.int64) & 0xF
    mag = _E2M1_GRID[c & 7]
    return np.where(c & 8, -mag, mag)


def pack_fp4(codes):
    """(odd << 4) | even, odd tail padded with 0 (formats.py:154-165).

    Returns ``(bytes, logical_len)``.
    """
    c = np.asarray(codes, dtype=np.uint8).ravel() & 0xF
    n = c.size
    if n % 2:
        c = np.concatenate([c, np.zeros(1, np.uint8)])
    return (c[1::2] << 4) | c[0::2], n


def unpack_fp4(buf, logical_len) -> np.ndarray:
    """formats.py:168-174."""
    b = np.asarray(buf, dtype=np.uint8).ravel()
    out = np.stack([b & 0xF, b >> 4], axis=-1).ravel()
    return out[:logical_len]


def e8m0_encode(e) -> np.ndarray:
    """formats.py:185-188."""
    return np.clip(np.asarray(e) + 127, 0, 254).astype(np.uint8)


def e8m0_decode(raw) -> np.ndarray:
    """formats.py:191-194."""
    return np.exp2(np.asarray(raw).astype(np.float64) - 127.0)


def _fp8_table(elem: Elem) -> np.ndarray:
    """Decoded value of all 256 codes (formats.py:254-279)."""
    c = np.arange(256)
    e = (c >> elem.mant) & ((1 << (7 - elem.mant)) - 1)
    m = c & ((1 << elem.mant) - 1)
    frac = m / float(1 << elem.mant)
    mag = np.where(e > 0, np.ldexp(1.0 + frac, e - elem.bias), np.ldexp(frac, 1 - elem.bias))
    val = np.where(c >= 128, -mag, mag)
    if elem is E4M3:
        val = np.where((c & 0x7F) == 0x7F, np.nan, val)
    else:
        top = (1 << (7 - elem.mant)) - 1
        val = np.where((e == top) & (m == 0), np.where(c >= 128, -np.inf, np.inf), val)
        val = np.where((e == top) & (m != 0), np.nan, val)
    return val


_TABLES = {"e4m3": _fp8_table(E4M3), "e5m2": _fp8_table(E5M2)}


def _elem_of(fmt):
    if isinstance(fmt, Fmt):
        fmt = fmt.elem
    if not isinstance(fmt, Elem) or fmt.bits != 8:
        raise ValueError(f"not an 8-bit element format: {getattr(fmt, 'name', fmt)}")
    return fmt


def encode_fp8(x, fmt) -> np.ndarray:
    """RNE, saturating FP8 encode; every zero magnitude -> +0 (formats.py:205-240).

    The rounding itself restates formats.py:220-224 (quantum 2^(e-mant)
    inside the clipped binade, np.round = half-to-even); the code is then
    recovered by exact lookup of the rounded magnitude in the decode table
    instead of re-deriving the bit fields.
    """
    elem = _elem_of(fmt)
    x = np.asarray(x, dtype=np.float64)
    _finite_or_raise(x, "encode_fp8")
    a = np.abs(x)
    _, ex = np.frexp(a)
    e = np.clip(ex - 1, 1 - elem.bias, elem.e_max)
    quantum = np.exp2(e.astype(np.float64) - elem.mant)
    mag = np.minimum(np.round(a / quantum) * quantum, elem.upper)
    pos = _TABLES[elem.name][:128]
    n_valid = 127 if elem is E4M3 else 124  # E4M3 0x7F is NaN; E5M2 0x7C.. are Inf/NaN
    code = np.searchsorted(pos[:n_valid], mag).astype(np.int64)
    code = code | (np.signbit(x).astype(np.int64) << 7)
    return np.where(mag == 0.0, 0, code).astype(np.uint8)


def decode_fp8(code, fmt) -> np.ndarray:
    """formats.py:243-248."""
    elem = _elem_of(fmt)
    return _TABLES[elem.name][np.asarray(code, dtype=np.uint8)]


# ---------------------------------------------------------------------------
# Dual quantizer (quantize.py:92-237)
# ---------------------------------------------------------------------------

TOKEN, BLOCK, TENSOR = "token", "block", "tensor"


def prescale_constant(d: int) -> float:
    """log2(e)/sqrt(D) in Python float64 (quantize.py:95)."""
    return math.log2(math.e) / math.sqrt(d)


def softmax_prescale(x: np.ndarray) -> np.ndarray:
    """quantize.py:92-95."""
    return x * prescale_constant(x.shape[-1])


def _floor_log2(v: np.ndarray) -> np.ndarray:
    """Exact floor(log2 v) for v > 0 via frexp (quantize.py:116-119)."""
    return np.frexp(v)[1] - 1


def _pow2_exponent(bmax: np.ndarray, e_max: int) -> np.ndarray:
    """Shared power-of-two exponent of a block (quantize.py:169-176,188-196)."""
    tiny = np.finfo(np.float64).tiny
    e = np.clip(_floor_log2(np.maximum(bmax, tiny)) - e_max, -127, 127)
    return np.where(bmax > 0, e, -127)


@dataclass
class DualQ:
    """Outputs of ``quantize_dual`` (quantize.py:69-89)."""

    shape: tuple
    low: Fmt
    high: Fmt
    granularity: str
    packed_low: np.ndarray  # [rows, cols//2] u8
    scales_low: np.ndarray  # [rows, cols//16 or cols//32] u8
    high_codes: np.ndarray  # [rows, cols] u8
    scales_high: np.ndarray  # [rows, cols//32] u8
    quant_scale: np.ndarray  # f64 [rows,1] | [1,1] | [rows, cols//32]
    prescaled: bool


def group_absmax(a: np.ndarray, granularity: str) -> np.ndarray:
    """quantize.py:98-106."""
    rows, cols = a.shape
    if granularity == TOKEN:
        return a.max(axis=1, keepdims=True)
    if granularity == TENSOR:
        return np.full((1, 1), a.max())
    if granularity == BLOCK:
        return a.reshape(rows, cols // 32, 32).max(axis=2)
    raise ValueError(f"unknown granularity: {granularity!r}")


def _expand_cols(s: np.ndarray, cols: int) -> np.ndarray:
    """quantize.py:109-113."""
    return s if s.shape[1] == 1 else np.repeat(s, cols // s.shape[1], axis=1)


def quantize_dual(x, is_query=False, low=NVFP4, high=MXFP8_E4M3, granularity=TOKEN) -> DualQ:
    """Paper Alg. 2, restating quantize.py:122-212."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim != 2:
        raise ValueError(f"expected a 2-D tensor, got shape {x.shape}")
    rows, cols = x.shape
    if cols % 32:
        raise ValueError(f"column count {cols} not divisible by 32")
    if not np.isfinite(x).all():
        raise ValueError("quantize_dual: input contains non-finite values")
    if low.elem is not E2M1:
        raise ValueError(f"low format must have E2M1 elements, got {low.name}")
    if high.elem.bits != 8:
        raise ValueError(f"high format must have FP8 elements, got {high.name}")

    xs = x * prescale_constant(cols) if is_query else x  # quantize.py:149
    gmax = group_absmax(np.abs(xs), granularity)
    sq = np.where(gmax > 0, gmax / QUANT_RANGE, 1.0)  # quantize.py:153
    xsc = xs / _expand_cols(sq, cols)  # quantize.py:154

    # ---- 4-bit path (quantize.py:156-184)
    src = xsc if low.two_level else xs
    blk = src.reshape(rows, cols // low.block, low.block)
    bmax = np.abs(blk).max(axis=2)
    if low.scale == "e4m3":
        sc = encode_fp8(np.where(bmax > 0, bmax / low.elem.upper, 1.0), E4M3)
        sv = decode_fp8(sc, E4M3)
        floor = (sv == 0) & (bmax > 0)  # quantize.py:164-167
        sc = np.where(floor, np.uint8(0x01), sc).astype(np.uint8)
        sv = np.where(floor, E4M3_TINY, sv)
    else:
        sc = (_pow2_exponent(bmax, low.elem.e_max) + 127).astype(np.uint8)
        sv = e8m0_decode(sc)
    lv = np.clip(blk / sv[:, :, None], -low.elem.upper, low.elem.upper)
    c4 = encode_e2m1(lv).reshape(rows, cols)
    packed = ((c4[:, 1::2] << 4) | c4[:, 0::2]).astype(np.uint8)

    # ---- 8-bit path (quantize.py:186-199)
    hblk = xsc.reshape(rows, cols // high.block, high.block)
    hexp = _pow2_exponent(np.abs(hblk).max(axis=2), high.elem.e_max)
    hv = np.clip(hblk / np.exp2(hexp)[:, :, None], -high.elem.upper, high.elem.upper)
    c8 = encode_fp8(hv, high.elem).reshape(rows, cols)

    return DualQ((rows, cols), low, high, granularity, packed, sc,
                 c8, (hexp + 127).astype(np.uint8), sq, is_query)


def dequantize_low(t: DualQ) -> np.ndarray:
    """quantize.py:215-229."""
    rows, cols = t.shape
    codes = np.stack([t.packed_low & 0xF, t.packed_low >> 4], axis=-1).reshape(rows, cols)
    s = decode_fp8(t.scales_low, E4M3) if t.low.scale == "e4m3" else e8m0_decode(t.scales_low)
    out = decode_e2m1(codes) * _expand_cols(s, cols)
    return out * _expand_cols(t.quant_scale, cols) if t.low.two_level else out


def dequantize_high(t: DualQ) -> np.ndarray:
    """quantize.py:232-237."""
    cols = t.shape[1]
    out = decode_fp8(t.high_codes, t.high.elem) * _expand_cols(e8m0_decode(t.scales_high), cols)
    return out * _expand_cols(t.quant_scale, cols)


# ---------------------------------------------------------------------------
# Attention (attention.py:51-335)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Cfg:
    """attention.py:51-80 (same defaults, same validation)."""

    tile_m: int = 64
    tile_n: int = 64
    diag_window: int = 0
    sink_window: int = 0
    causal: bool = True
    low_format: Fmt | None = NVFP4
    high_format: Fmt | None = MXFP8_E4M3
    granularity: str = TOKEN

    def __post_init__(self):
        if self.tile_m < 1 or self.tile_n < 1:
            raise ValueError("tile sizes must be >= 1")
        if self.diag_window < 0 or self.sink_window < 0:
            raise ValueError("window sizes must be >= 0")
        if self.diag_window % self.tile_n or self.sink_window % self.tile_n:
            raise ValueError(
                "diag_window and sink_window must be multiples of tile_n "
                f"(got {self.diag_window}/{self.sink_window} with tile_n={self.tile_n})")


def _cdiv(a: int, b: int) -> int:
    return -((-a) // b)


def causal_plan(q_tile, len_q, len_k, cfg):
    """attention.py:191-209 (sink-high, low span, diagonal-high)."""
    tm, tn = cfg.tile_m, cfg.tile_n
    q0 = q_tile * tm
    q_last = min(q0 + tm, len_q) - 1
    n_need = min(_cdiv(q_last + 1, tn), _cdiv(len_k, tn))
    n_sink = min(cfg.sink_window // tn, n_need)
    first_hi = min(max(_cdiv(q0 - cfg.diag_window, tn), n_sink), n_need)
    return ([(t, True) for t in range(n_sink)]
            + [(t, False) for t in range(n_sink, first_hi)]
            + [(t, True) for t in range(first_hi, n_need)])


def noncausal_plan(q_tile, len_q, len_k, cfg):
    """attention.py:212-233, integer form of the window bounds.

    ceil((q0 -/+ T/2)/tn) == cdiv(2*q0 -/+ T, 2*tn) exactly for integers.
    """
    tn = cfg.tile_n
    q0 = q_tile * cfg.tile_m
    n = _cdiv(len_k, tn)
    n_sink = min(cfg.sink_window // tn, n)
    w0 = min(max(_cdiv(2 * q0 - cfg.diag_window, 2 * tn), 0), n)
    w1 = min(max(_cdiv(2 * q0 + cfg.diag_window, 2 * tn), w0), n)
    if cfg.diag_window >= 2 * len_k:
        w0, w1 = 0, n
    outside = list(range(0, w0)) + list(range(w1, n))
    return [(t, t < n_sink) for t in outside] + [(t, True) for t in range(w0, w1)]


def tile_plan(q_tile, len_q, len_k, cfg):
    return (causal_plan if cfg.causal else noncausal_plan)(q_tile, len_q, len_k, cfg)


def _check_qkv(q, k, v, causal):
    """attention.py:109-119."""
    if q.ndim != 2 or k.ndim != 2 or v.ndim != 2:
        raise ValueError("Q, K, V must be 2-D matrices")
    if q.shape[1] != k.shape[1]:
        raise ValueError(f"head dim mismatch: Q {q.shape} vs K {k.shape}")
    if k.shape[0] != v.shape[0]:
        raise ValueError(f"K/V row mismatch: {k.shape} vs {v.shape}")
    if causal and q.shape[0] != k.shape[0]:
        raise ValueError(
            f"causal attention requires equal sequence lengths, got {q.shape[0]} and {k.shape[0]}")


def operands(q, k, v, cfg):
    """(q_low, q_high, k_low, k_high, v) as the engine sees them (attention.py:247-279)."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    _check_qkv(q, k, v, cfg.causal)
    if (cfg.low_format or cfg.high_format) and q.shape[1] % 32:
        raise ValueError(f"head dim {q.shape[1]} not divisible by 32")

    def pair(x, is_q):
        plain = x * prescale_constant(x.shape[1]) if is_q else x
        if cfg.low_format is None and cfg.high_format is None:
            return plain, plain
        lo_fmt = NVFP4 if (cfg.low_format is None or cfg.low_format.elem.bits == 8) else cfg.low_format
        t = quantize_dual(x, is_q, lo_fmt, cfg.high_format or MXFP8_E4M3, cfg.granularity)
        hi = dequantize_high(t) if cfg.high_format is not None else plain
        if cfg.low_format is None:
            lo = plain
        elif cfg.low_format.elem.bits == 8:
            lo = hi
        else:
            lo = dequantize_low(t)
        return lo, hi

    ql, qh = pair(q, True)
    kl, kh = pair(k, False)
    return ql, qh, kl, kh, v


def quantize_v_keys(v: np.ndarray) -> np.ndarray:
    """Dequantized MXFP8 (E4M3) V with one E8M0 scale per 32 keys per column.

    NOT part of the reference (which keeps V in float64, attention.py:250):
    this is the block-scaled PV operand the north star asks for, restated so
    tests can check the kernel against "reference algorithm + the kernel's
    stated PV quantization".  The exponent rule is the reference's MXFP8 rule
    (quantize.py:186-199, e = floor_log2(block max) - e_max, clip to +-448,
    RNE) applied along the key axis with no S_q level.
    """
    v = np.asarray(v, dtype=np.float64)
    n, dv = v.shape
    pad = -n % 32
    vp = np.concatenate([v, np.zeros((pad, dv))]) if pad else v
    blk = vp.reshape(-1, 32, dv)
    e = _pow2_exponent(np.abs(blk).max(axis=1), E4M3.e_max)[:, None, :]
    hv = np.clip(blk * np.exp2(-e.astype(np.float64)), -E4M3.upper, E4M3.upper)
    deq = decode_fp8(encode_fp8(hv, E4M3), E4M3) * np.exp2(e.astype(np.float64))
    return deq.reshape(-1, dv)[:n]


# The MXFP8-PV kernel (attn_pp.cuh) keeps a row's running max until a tile raises
# it by more than LAZY_RESCALE (log2 units) and stores P as E4M3(P * 2^(8 - LAZY)).
LAZY_RESCALE = {"mxfp8": 4.0}


def _quantize_p(p: np.ndarray, pv: str) -> np.ndarray:
    """P as the kernel feeds it to the PV contraction: E4M3(P * 2^s) * 2^-s, or bf16 (RNE)."""
    if pv == "mxfp8":
        sc = 2.0 ** (8.0 - LAZY_RESCALE["mxfp8"])
        return decode_fp8(encode_fp8(p * sc, E4M3), E4M3) / sc
    if pv == "bf16":
        b = p.astype(np.float32).view(np.uint32).astype(np.uint64)
        b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
        return b.astype(np.uint32).view(np.float32).astype(np.float64)
    return p


def mixed_precision_attention(q, k, v, cfg: Cfg, pv: str = "f64", q_tiles=None, kv_split: int = 1) -> np.ndarray:
    """Tile loop + base-2 online softmax (attention.py:150-175, 178-184, 282-310).

    ``pv="f64"`` is the reference exactly.  ``pv="mxfp8"`` / ``"bf16"`` add the
    sm_100a kernel's stated PV quantization (P -> E4M3 x 2^4 with V -> MXFP8
    along keys and lazy max rescaling, or P and V in bf16) on top of the same
    algorithm; the row sum l still uses the unquantized P, as the kernel does.
    ``q_tiles`` (optional): compute only these query tiles (rows of other tiles are NaN),
    for sampled checks at full sequence lengths.  ``kv_split`` > 1 emulates the kernel's KV
    splits for small problems: each query tile's plan is cut into ns = min(kv_split, n)
    contiguous entry ranges [s*n//ns, (s+1)*n//ns), each run from m = -inf, l = 0 (so the
    lazy max and the P quantization restart per range), then merged with weights
    2^(m_s - M).  With pv="f64" the split changes nothing but rounding.  Test
    infrastructure only.
    """
    lazy = LAZY_RESCALE.get(pv, 0.0)
    ql, qh, kl, kh, v = operands(q, k, v, cfg)
    if pv == "mxfp8":
        v = quantize_v_keys(v)
    elif pv == "bf16":
        v = _quantize_p(v, "bf16")
    lq, lk = ql.shape[0], kl.shape[0]
    tm, tn = cfg.tile_m, cfg.tile_n
    out = np.full((lq, v.shape[1]), np.nan)
    for qt in (range(_cdiv(lq, tm)) if q_tiles is None else q_tiles):
        q0, q1 = qt * tm, min(qt * tm + tm, lq)
        plan = tile_plan(qt, lq, lk, cfg)
        ns = max(1, min(kv_split, len(plan)))
        parts = []
        for s in range(ns):
            parts.append(_tile_range(ql, qh, kl, kh, v, cfg, pv, lazy, q0, q1, lk,
                                     plan[s * len(plan) // ns:(s + 1) * len(plan) // ns]))
        if ns == 1:
            m, l, acc = parts[0]
        else:
            mm = np.max(np.stack([p_[0] for p_ in parts]), axis=0)
            l = np.zeros(q1 - q0)
            acc = np.zeros((q1 - q0, v.shape[1]))
            for m_s, l_s, a_s in parts:
                ok = np.isfinite(m_s)
                w = np.where(ok, np.exp2(np.where(ok, m_s - np.where(np.isfinite(mm), mm, 0.0), 0.0)), 0.0)
                l = l + w * l_s
                acc = acc + w[:, None] * a_s
        out[q0:q1] = acc / np.where(l > 0, l, 1.0)[:, None]
    return out


def _tile_range(ql, qh, kl, kh, v, cfg, pv, lazy, q0, q1, lk, entries):
    """Online softmax (attention.py:150-175) of query rows [q0, q1) over plan entries."""
    tn = cfg.tile_n
    m = np.full(q1 - q0, -np.inf)
    l = np.zeros(q1 - q0)  # l0 = 0, attention.py:100
    acc = np.zeros((q1 - q0, v.shape[1]))
    for kt, hi in entries:
        k0, k1 = kt * tn, min(kt * tn + tn, lk)
        s = (qh if hi else ql)[q0:q1] @ (kh if hi else kl)[k0:k1].T
        if cfg.causal and k1 - 1 > q0:  # attention.py:306
            qi = np.arange(q0, q1)[:, None]
            kj = np.arange(k0, k1)[None, :]
            s = np.where(qi >= kj, s, -np.inf)
        m_new = np.maximum(m, s.max(axis=1))
        if lazy:
            m_new = np.where(m_new > m + lazy, m_new, m)
        alive = np.isfinite(m_new)
        alpha = np.where(alive, np.exp2(np.where(alive, m - m_new, 0.0)), 1.0)
        p = np.zeros_like(s)
        ok = np.isfinite(s)
        p[ok] = np.exp2((s - np.where(alive, m_new, 0.0)[:, None])[ok])
        l = l * alpha + p.sum(axis=1)
        acc = acc * alpha[:, None] + _quantize_p(p, pv) @ v[k0:k1]
        m = m_new
    return m, l, acc


def reference_attention(q, k, v, causal=False) -> np.ndarray:
    """Dense softmax(QK^T/sqrt(D))V, base e (attention.py:122-147)."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    _check_qkv(q, k, k, causal)
    z = q @ k.T / math.sqrt(q.shape[1])
    if causal:
        n = q.shape[0]
        z = np.where(np.arange(n)[:, None] >= np.arange(n)[None, :], z, -np.inf)
    mx = z.max(axis=1, keepdims=True)
    mx = np.where(np.isfinite(mx), mx, 0.0)
    p = np.exp(z - mx)
    p[~np.isfinite(z)] = 0.0
    den = p.sum(axis=1, keepdims=True)
    return (p / np.where(den > 0, den, 1.0)) @ v


def _softmax_rows(logits: np.ndarray, base2: bool) -> np.ndarray:
    """attention.py:138-147."""
    m = logits.max(axis=1, keepdims=True)
    m = np.where(np.isfinite(m), m, 0.0)
    z = logits - m
    p = np.exp2(z) if base2 else np.exp(z)
    p[~np.isfinite(logits)] = 0.0
    den = p.sum(axis=1, keepdims=True)
    return p / np.where(den > 0, den, 1.0)


def reference_scores(q, k, causal=False) -> np.ndarray:
    """Dense post-softmax probabilities, base e (attention.py:126-135)."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    _check_qkv(q, k, k, causal)
    z = q @ k.T / math.sqrt(q.shape[1])
    if causal:
        n = q.shape[0]
        z = np.where(np.arange(n)[:, None] >= np.arange(n)[None, :], z, -np.inf)
    return _softmax_rows(z, base2=False)


def mixed_precision_scores(q, k, cfg: Cfg) -> np.ndarray:
    """Dense base-2 probabilities under the per-tile precision plan (attention.py:313-335)."""
    ql, qh, kl, kh, _ = operands(q, k, np.asarray(k, dtype=np.float64), cfg)
    lq, lk = ql.shape[0], kl.shape[0]
    logits = np.full((lq, lk), -np.inf)
    for qt in range(-(-lq // cfg.tile_m)):
        q0, q1 = qt * cfg.tile_m, min((qt + 1) * cfg.tile_m, lq)
        for kt, high in tile_plan(qt, lq, lk, cfg):
            k0, k1 = kt * cfg.tile_n, min((kt + 1) * cfg.tile_n, lk)
            blk = (qh if high else ql)[q0:q1] @ (kh if high else kl)[k0:k1].T
            if cfg.causal:  # attention.py:178-184
                blk = np.where(np.arange(q0, q1)[:, None] >= np.arange(k0, k1)[None, :], blk, -np.inf)
            logits[q0:q1, k0:k1] = blk
    return _softmax_rows(logits, base2=True)


def high_precision_fraction(len_q, len_k, tile_m, tile_n, diag_window, sink_window, causal):
    """metrics.py:55-101 (Bit_high)."""
    cfg = Cfg(tile_m=tile_m, tile_n=tile_n, diag_window=diag_window,
              sink_window=sink_window, causal=causal)
    hi_cells = valid = 0
    for qt in range(_cdiv(len_q, tile_m)):
        q0, q1 = qt * tile_m, min(qt * tile_m + tile_m, len_q)
        mark = np.zeros(len_k, dtype=bool)
        for kt, hi in tile_plan(qt, len_q, len_k, cfg):
            if hi:
                mark[kt * tile_n:min(kt * tile_n + tile_n, len_k)] = True
        if causal:
            csum = np.cumsum(mark)
            kmax = np.minimum(np.arange(q0, q1), len_k - 1)
            hi_cells += int(csum[kmax].sum())
            valid += int((kmax + 1).sum())
        else:
            hi_cells += int(mark.sum()) * (q1 - q0)
            valid += len_k * (q1 - q0)
    return 0.0 if valid == 0 else hi_cells / valid


def similarity(ref, test) -> dict:
    """metrics.py:35-52."""
    r = np.asarray(ref, dtype=np.float64).ravel()
    t = np.asarray(test, dtype=np.float64).ravel()
    if r.shape != t.shape:
        raise ValueError(f"shape mismatch: {r.shape} vs {t.shape}")
    rn = np.linalg.norm(r)
    if rn == 0:
        raise ValueError("metrics are undefined for an all-zero reference")
    tn = np.linalg.norm(t)
    cos = float(r @ t / (rn * tn)) if tn > 0 else 0.0
    abs_l1 = float(np.abs(r - t).sum())
    rmse = float(np.sqrt(np.mean((r - t) ** 2)))
    peak = float(np.abs(r).max())
    return dict(cos_sim=cos, rel_l1=abs_l1 / float(np.abs(r).sum()), abs_l1=abs_l1, rmse=rmse,
                psnr=math.inf if rmse == 0 else 20.0 * math.log10(peak / rmse))
