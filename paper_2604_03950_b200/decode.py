"""Decode over an MX-quantized KV cache (SURVEY §8 f, rank 4; libdma ``dma_decode_attention``).

The reference is prefill-only (SPEC.md:287 lists decode as a non-goal); this is
the step after it, built on the same quantizer and precision plan.  Keys are
quantized once, with the bit-exact ``quantize_dual`` (TOKEN granularity: every
row has its own S_q, so a cached row never changes), into the canonical
layouts of include/dma.h; values are kept in bf16.  ``attend`` scores the new
query rows against the cache with the per-tile precision of
``mixed_precision_attention``: query i at absolute position p = pos + i gets
exactly row p of the prefill forward over the whole sequence (causal), up to
f32 arithmetic -- there is no PV quantization in decode.

    cache = DmaKVCache(cfg, batch=1, kv_heads=8, capacity=32768, head_dim=128)
    cache.append(k_prompt, v_prompt)          # [B, KVH, L, D] CUDA tensors
    o = cache.step(q_new, k_new, v_new)       # q [B, H, n_q, D] -> [B, H, n_q, Dv]
"""

from __future__ import annotations

from . import _lib
from ._device import _torch, dtype_code
from .attention import AttentionConfig
from .formats import MXFP8_E4M3, NVFP4, format_code
from .quantize import Granularity, prescale_constant


class DecodeArgs(_lib.C.Structure):
    """include/dma.h DmaDecodeArgs."""

    _fields_ = [(n, _lib.C.c_void_p) for n in (
        "q_packed_low", "q_scales_low", "q_high_codes", "q_scales_high", "q_quant_scale",
        "k_packed_low", "k_scales_low", "k_high_codes", "k_scales_high", "k_quant_scale", "v", "o")] + [
        ("v_dtype", _lib.C.c_int32), ("out_dtype", _lib.C.c_int32)] + [
        (n, _lib.C.c_int64) for n in ("batch", "heads", "kv_heads", "n_q", "capacity", "pos", "head_dim",
                                      "v_dim")] + [
        (n, _lib.C.c_int32) for n in ("tile_m", "tile_n", "diag_window", "sink_window", "low_format",
                                      "high_format", "granularity", "_pad")] + [
        ("workspace", _lib.C.c_void_p), ("workspace_bytes", _lib.C.c_size_t)]


def _bind():
    L = _lib.lib()
    if not getattr(L, "_dma_decode_bound", False):
        L.dma_decode_workspace_bytes.restype = _lib.C.c_size_t
        L.dma_decode_workspace_bytes.argtypes = [_lib.C.POINTER(DecodeArgs)]
        L.dma_decode_attention.restype = _lib.C.c_int
        L.dma_decode_attention.argtypes = [_lib.C.POINTER(DecodeArgs), _lib.C.c_void_p]
        L._dma_decode_bound = True
    return L


class _Rows:
    """Canonical quantize_dual outputs for [n_mat, rows, cols] (include/dma.h)."""

    def __init__(self, n_mat, rows, cols, low_block, device):
        torch = _torch()
        u8 = dict(dtype=torch.uint8, device=device)
        self.packed_low = torch.empty((n_mat, rows, cols // 2), **u8)
        self.scales_low = torch.empty((n_mat, rows, cols // low_block), **u8)
        self.high_codes = torch.empty((n_mat, rows, cols), **u8)
        self.scales_high = torch.empty((n_mat, rows, cols // 32), **u8)
        self.quant_scale = torch.empty((n_mat, rows), dtype=torch.float64, device=device)

    def parts(self):
        return (self.packed_low, self.scales_low, self.high_codes, self.scales_high, self.quant_scale)


class DmaKVCache:
    """A per-layer key / value cache for DMA decode (TOKEN granularity, MX high format)."""

    def __init__(self, cfg: AttentionConfig, batch: int, kv_heads: int, capacity: int, head_dim: int,
                 v_dim: int | None = None, device="cuda"):
        torch = _torch()
        if cfg.granularity is not Granularity.TOKEN:
            raise _lib.DmaUnsupported("decode: TOKEN granularity only (cache rows are quantized once)")
        if cfg.high_format is None or cfg.low_format is None:
            raise _lib.DmaUnsupported("decode: identity (None) formats are not supported")
        if not cfg.causal:
            raise ValueError("decode attention is causal")
        if head_dim % 32:
            raise ValueError(f"head dim {head_dim} not divisible by 32")
        self.cfg = cfg
        self.batch, self.kv_heads, self.capacity = batch, kv_heads, capacity
        self.head_dim, self.v_dim = head_dim, v_dim or head_dim
        self.length = 0
        # quantize_dual always runs with an E2M1 low format; an 8-bit low format means
        # "score with the high operands" (attention.py:269-276), the low copy is unused
        self._qlow = cfg.low_format if cfg.low_format.element.bits == 4 else NVFP4
        self._qhigh = cfg.high_format or MXFP8_E4M3
        # rows are allocated in whole 32-key groups (the kernel bulk-loads full groups)
        self._rows = -(-capacity // 32) * 32
        self.keys = _Rows(batch * kv_heads, self._rows, head_dim, self._qlow.block_size, device)
        self.values = torch.zeros((batch, kv_heads, self._rows, self.v_dim), dtype=torch.bfloat16, device=device)
        self._flag = torch.zeros(1, dtype=torch.int32, device=device)
        self._ws = torch.empty(256, dtype=torch.uint8, device=device)   # decode partials
        self._qws = torch.empty(256, dtype=torch.uint8, device=device)  # quantize (unused for TOKEN)
        self._qbuf = {}

    # ------------------------------------------------------------- quantize
    def _quantize(self, x, is_query, out: _Rows, validate):
        """dma_quantize_dual over x [n_mat, rows, cols] into ``out``."""
        n_mat, rows, cols = x.shape
        a = _lib.DmaQuantArgs()
        a.x, a.x_dtype, a.is_query = x.data_ptr(), dtype_code(x), int(is_query)
        a.n_mat, a.rows, a.cols = n_mat, rows, cols
        a.mat_stride, a.row_stride = rows * cols, cols
        a.prescale = prescale_constant(cols)
        a.low_format, a.high_format = format_code(self._qlow), format_code(self._qhigh)
        a.granularity = _lib.GRAN_TOKEN
        (a.packed_low, a.scales_low, a.high_codes, a.scales_high,
         a.quant_scale) = (t.data_ptr() for t in out.parts())
        if validate:
            self._flag.zero_()
        a.nonfinite = self._flag.data_ptr()
        a.workspace, a.workspace_bytes = self._qws.data_ptr(), self._qws.numel()
        _lib.check(_lib.lib().dma_quantize_dual(a, _lib.stream_ptr()), "quantize_dual")
        if validate and int(self._flag.item()):
            raise ValueError("quantize_dual: input contains non-finite values")

    @staticmethod
    def _operand(x, name, shape):
        torch = _torch()
        if not (isinstance(x, torch.Tensor) and x.is_cuda):
            raise TypeError(f"{name} must be a CUDA tensor")
        if tuple(x.shape) != tuple(shape):
            raise ValueError(f"{name} has shape {tuple(x.shape)}, expected {tuple(shape)}")
        if x.dtype not in (torch.float64, torch.float32, torch.bfloat16):
            x = x.to(torch.float32)
        return x.contiguous()

    def append(self, k, v, validate: bool = True):
        """Quantize k [B, KVH, n, D] into the cache and store v [B, KVH, n, Dv] (bf16)."""
        B, KVH = self.batch, self.kv_heads
        n = k.shape[2] if k.dim() == 4 else -1
        k = self._operand(k, "k", (B, KVH, n, self.head_dim))
        v = self._operand(v, "v", (B, KVH, n, self.v_dim))
        if self.length + n > self.capacity:
            raise ValueError(f"cache overflow: {self.length} + {n} > capacity {self.capacity}")
        if n == 0:
            return
        tmp = _Rows(B * KVH, n, self.head_dim, self._qlow.block_size, k.device)
        self._quantize(k.view(B * KVH, n, self.head_dim), False, tmp, validate)
        s = slice(self.length, self.length + n)
        for dst, src in zip(self.keys.parts(), tmp.parts()):
            dst[:, s].copy_(src)
        self.values[:, :, s].copy_(v)
        self.length += n

    def attend(self, q, out=None, out_dtype=None, validate: bool = True):
        """q [B, H, n_q, D] for the last n_q cached positions -> O [B, H, n_q, Dv]."""
        torch = _torch()
        B, KVH = self.batch, self.kv_heads
        if q.dim() != 4 or q.shape[0] != B or q.shape[3] != self.head_dim or q.shape[1] % KVH:
            raise ValueError(f"q must be [B={B}, H (multiple of {KVH}), n_q, D={self.head_dim}], "
                             f"got {tuple(q.shape)}")
        H, nq = q.shape[1], q.shape[2]
        if nq < 1 or nq > self.length:
            raise ValueError(f"n_q = {nq} must be in [1, cache length {self.length}]")
        q = self._operand(q, "q", (B, H, nq, self.head_dim))
        key = (H, nq)
        if key not in self._qbuf:
            self._qbuf = {key: _Rows(B * H, nq, self.head_dim, self._qlow.block_size, q.device)}
        qr = self._qbuf[key]
        self._quantize(q.view(B * H, nq, self.head_dim), True, qr, validate)
        odt = out_dtype or torch.float32
        if out is None:
            out = torch.empty((B, H, nq, self.v_dim), dtype=odt, device=q.device)
        cfg = self.cfg
        a = DecodeArgs()
        (a.q_packed_low, a.q_scales_low, a.q_high_codes, a.q_scales_high,
         a.q_quant_scale) = (t.data_ptr() for t in qr.parts())
        (a.k_packed_low, a.k_scales_low, a.k_high_codes, a.k_scales_high,
         a.k_quant_scale) = (t.data_ptr() for t in self.keys.parts())
        a.v, a.o = self.values.data_ptr(), out.data_ptr()
        a.v_dtype = _lib.DT_BF16
        a.out_dtype = _lib.DT_BF16 if out.dtype == torch.bfloat16 else _lib.DT_F32
        a.batch, a.heads, a.kv_heads, a.n_q = B, H, KVH, nq
        a.capacity, a.pos, a.head_dim, a.v_dim = self._rows, self.length - nq, self.head_dim, self.v_dim
        a.tile_m, a.tile_n, a.diag_window, a.sink_window = cfg.tile_m, cfg.tile_n, cfg.diag_window, cfg.sink_window
        a.low_format, a.high_format = format_code(cfg.low_format), format_code(cfg.high_format)
        a.granularity = _lib.GRAN_TOKEN
        L = _bind()
        need = L.dma_decode_workspace_bytes(a)
        if need == 0:  # invalid / unsupported: let the call report why
            _lib.check(L.dma_decode_attention(a, _lib.stream_ptr()), "decode_attention")
        if self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=q.device)
        a.workspace, a.workspace_bytes = self._ws.data_ptr(), self._ws.numel()
        _lib.check(L.dma_decode_attention(a, _lib.stream_ptr()), "decode_attention")
        return out

    def step(self, q, k, v, out=None, out_dtype=None, validate: bool = True):
        """Append the new tokens' k / v, then attend with their queries."""
        self.append(k, v, validate)
        return self.attend(q, out, out_dtype, validate)


__all__ = ["DmaKVCache"]
