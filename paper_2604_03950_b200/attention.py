"""DMA attention on the GPU (drop-in for ``mxattn.attention``).

``mixed_precision_attention`` (alias ``dma_attention``) runs the fused
sm_100a forward in libdma: phase 1 quantizes Q/K exactly like
``quantize_dual`` (and V to MXFP8 along keys), phase 2 runs the
diagonal-tiled attention with tcgen05 block-scaled MMAs following the same
tile plans as the reference (attention.py:191-233).

Differences from the float64 reference that are intrinsic to tensor cores
(and covered by the stated tolerances in DESIGN.md / tests):
  * scores accumulate in fp32 inside TMEM (the reference uses f64 dgemm);
  * P and V enter the PV contraction as E4M3 x E8M0 (``pv_mode="mxfp8"``,
    the default, block-scaled) or bf16 (``pv_mode="bf16"``, parity mode); the
    reference keeps both in float64 (attention.py:174, 250).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._device import dtype_code, from_device, is_torch, to_device
from .formats import MXFP8_E4M3, NVFP4, MxFormatSpec, format_code
from .quantize import Granularity, granularity_code, prescale_constant
from .softmax import OnlineSoftmaxState, apply_causal_mask, online_softmax_update  # noqa: F401  (attention.py:37-48)

_PV = {"mxfp8": _lib.PV_MXFP8, "bf16": _lib.PV_BF16}


@dataclass(frozen=True)
class AttentionConfig:
    """attention.py:51-80 (same fields, defaults and validation), plus ``pv_mode``.

    ``pv_mode`` is the one precision choice the reference does not have (its P and V stay
    float64, attention.py:174):

    * ``"mxfp8"`` (default, the north-star kernel): P -> E4M3 in registers, V -> MXFP8 per 32
      keys, block-scaled tcgen05 PV.  Measured 3.4-4.0e-2 relative L2 (max-abs <= 0.36) from
      the reference's own output on N(0,1) inputs (profiles/r02_parity.jsonl) -- the V / P
      quantization, not the kernel (<= 4.3e-4 from the oracle with the same PV quantization);
    * ``"bf16"`` (parity mode, ~1.7x slower): P and V in bf16, 1.1-1.5e-3 relative L2
      (max-abs <= 7.6e-3, full-mantissa f64 inputs) from the reference.
    """

    tile_m: int = 64
    tile_n: int = 64
    diag_window: int = 0
    sink_window: int = 0
    causal: bool = True
    low_format: MxFormatSpec | None = NVFP4
    high_format: MxFormatSpec | None = MXFP8_E4M3
    granularity: Granularity = Granularity.TOKEN
    pv_mode: str = "mxfp8"

    def __post_init__(self):
        if self.tile_m < 1 or self.tile_n < 1:
            raise ValueError("tile sizes must be >= 1")
        if self.diag_window < 0 or self.sink_window < 0:
            raise ValueError("window sizes must be >= 0")
        if self.diag_window % self.tile_n or self.sink_window % self.tile_n:
            raise ValueError(
                "diag_window and sink_window must be multiples of tile_n "
                f"(got {self.diag_window}/{self.sink_window} with tile_n={self.tile_n})")
        if self.pv_mode not in _PV:
            raise ValueError(f"pv_mode must be one of {sorted(_PV)}")


# ---------------------------------------------------------------- tile plans
def _plan(q_tile, len_q, len_k, cfg, causal):
    buf = (ctypes.c_int64 * (2 + -(-max(len_k, 1) // cfg.tile_n)))()
    n = _lib.lib().dma_tile_plan(q_tile, len_q, len_k, cfg.tile_m, cfg.tile_n, cfg.diag_window,
                                 cfg.sink_window, int(causal), buf, len(buf))
    return [(int(v) >> 1, bool(v & 1)) for v in buf[:n]]


def causal_tile_plan(q_tile: int, len_q: int, len_k: int, cfg: AttentionConfig) -> list[tuple[int, bool]]:
    """attention.py:191-209 (integer-exact; same code as the kernel's scheduler)."""
    return _plan(q_tile, len_q, len_k, cfg, True)


def noncausal_tile_plan(q_tile: int, len_q: int, len_k: int, cfg: AttentionConfig) -> list[tuple[int, bool]]:
    """attention.py:212-233 (integer-exact; same code as the kernel's scheduler)."""
    return _plan(q_tile, len_q, len_k, cfg, False)


# ---------------------------------------------------------------- validation
def _check_qkv(qs, ks, vs, causal):
    """attention.py:109-119 on shapes [..., L, D]."""
    if qs[-1] != ks[-1]:
        raise ValueError(f"head dim mismatch: Q {tuple(qs)} vs K {tuple(ks)}")
    if ks[-2] != vs[-2]:
        raise ValueError(f"K/V row mismatch: {tuple(ks)} vs {tuple(vs)}")
    if causal and qs[-2] != ks[-2]:
        raise ValueError(f"causal attention requires equal sequence lengths, got {qs[-2]} and {ks[-2]}")


def _args(cfg, q, k, v, o, B, H, KVH, Lq, Lk, D, DV, out_dtype):
    a = _lib.DmaAttnArgs()
    a.q, a.k, a.v, a.o = q.data_ptr(), k.data_ptr(), v.data_ptr(), (o.data_ptr() if o is not None else None)
    a.in_dtype = dtype_code(q)
    a.out_dtype = out_dtype
    a.batch, a.heads, a.kv_heads, a.len_q, a.len_k, a.head_dim, a.v_dim = B, H, KVH, Lq, Lk, D, DV
    a.tile_m, a.tile_n, a.diag_window, a.sink_window = cfg.tile_m, cfg.tile_n, cfg.diag_window, cfg.sink_window
    a.causal = int(cfg.causal)
    a.low_format = format_code(cfg.low_format)
    a.high_format = format_code(cfg.high_format)
    a.granularity = granularity_code(cfg.granularity)
    a.pv_mode = _PV[cfg.pv_mode]
    a.prescale = prescale_constant(D)
    return a


_NONFINITE_MSG = "quantize_dual: input contains non-finite values"


class DmaAttention:
    """Reusable forward for fixed shapes: owns the phase-1 workspace.

    q [B, H, Lq, D], k/v [B, KVH, Lk, D|DV] CUDA tensors (bf16/f32/f64), contiguous,
    one dtype, one device.  ``validate=True`` adds the reference's non-finite check
    (quantize.py:142-143: ValueError if Q or K holds NaN / Inf): phase 1 raises a
    device flag and the call reads it back (one 4-byte D2H + stream sync per call);
    the default leaves the forward asynchronous.
    """

    def __init__(self, cfg: AttentionConfig, validate: bool = False):
        self.cfg = cfg
        self.validate = validate
        self._ws = None
        self._flag = None

    def workspace_for(self, a):
        import torch

        need = int(_lib.lib().dma_attention_workspace_bytes(a))
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(max(need, 256), dtype=torch.uint8, device="cuda")
        return self._ws

    def prepare(self, q, k, v, out=None, out_dtype=None, kv_split=0):
        """Validate the operands and build the C-ABI arguments.  The library takes raw
        pointers without strides, so layout mismatches are errors here, not silent."""
        import torch

        if q.dim() != 4 or k.dim() != 4 or v.dim() != 4:
            raise ValueError("Q, K, V must be 4-D [B, H, L, D] (use dma_attention for 2-D / 3-D inputs)")
        B, H, Lq, D = q.shape
        _, KVH, Lk, _ = k.shape
        DV = v.shape[-1]
        _check_qkv(q.shape, k.shape, v.shape, self.cfg.causal)
        if k.shape[0] != B or v.shape[0] != B or v.shape[1] != KVH:
            raise ValueError(f"batch / kv-head mismatch: Q {tuple(q.shape)}, K {tuple(k.shape)}, V {tuple(v.shape)}")
        if (self.cfg.low_format or self.cfg.high_format) and D % 32:
            raise ValueError(f"head dim {D} not divisible by 32")
        if H % KVH:
            raise ValueError(f"heads {H} not divisible by kv_heads {KVH}")
        for name, t in (("Q", q), ("K", k), ("V", v)):
            if not t.is_cuda or t.device != q.device:
                raise ValueError(f"{name} must be a CUDA tensor on {q.device}, got {t.device}")
            if not t.is_contiguous():
                raise ValueError(f"{name} must be contiguous [B, H, L, D] (e.g. .transpose(1, 2).contiguous())")
        if not (q.dtype == k.dtype == v.dtype):
            raise ValueError(f"Q, K, V dtypes differ: {q.dtype}, {k.dtype}, {v.dtype}")
        odt = out_dtype or (torch.bfloat16 if q.dtype == torch.bfloat16 else torch.float32)
        if out is None:
            out = torch.empty((B, H, Lq, DV), dtype=odt, device=q.device)
        if out.dtype not in (torch.bfloat16, torch.float32):
            raise ValueError(f"out dtype must be bfloat16 or float32, got {out.dtype}")
        if tuple(out.shape) != (B, H, Lq, DV) or not out.is_contiguous() or out.device != q.device:
            raise ValueError(f"out must be a contiguous {q.device} tensor of shape {(B, H, Lq, DV)}")
        code = _lib.DT_BF16 if out.dtype == torch.bfloat16 else _lib.DT_F32
        a = _args(self.cfg, q, k, v, out, B, H, KVH, Lq, Lk, D, DV, code)
        a.kv_split = kv_split  # 0: the library's policy (set before the workspace query)
        rc = _lib.lib().dma_attention_supported(a)
        _lib.check(rc, "dma_attention")
        ws = self.workspace_for(a)
        a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
        if self.validate:
            if self._flag is None or self._flag.device != q.device:
                self._flag = torch.zeros(1, dtype=torch.int32, device=q.device)
            a.nonfinite = self._flag.data_ptr()
        return a, out

    def _check_finite(self, q, k, stream=None):
        """After a validate=True launch: raise like quantize_dual on NaN / Inf in Q or K."""
        import torch

        if q.shape[-2] == 0 or k.shape[-2] == 0:  # no phase 1 ran: check on the device directly
            bad = not (bool(torch.isfinite(q).all()) and bool(torch.isfinite(k).all()))
        else:
            s = stream if stream is not None else torch.cuda.current_stream()
            with torch.cuda.stream(s):
                bad = int(self._flag.item()) != 0
        if bad:
            raise ValueError(_NONFINITE_MSG)

    def __call__(self, q, k, v, out=None, out_dtype=None, stream=None, kv_split=0):
        if not q.is_cuda:
            return self.forward_host(q, k, v, out=out, out_dtype=out_dtype)
        a, out = self.prepare(q, k, v, out, out_dtype, kv_split=kv_split)
        _lib.check(_lib.lib().dma_attention_fwd(a, _lib.stream_ptr(stream)), "dma_attention")
        if self.validate:
            self._check_finite(q, k, stream)
        return out

    def forward_host(self, q, k, v, out=None, out_dtype=None, chunk_kv_heads=None, graph=True):
        """Forward on HOST tensors [B, H, Lq, D] / [B, KVH, Lk, D] (pinned for full speed).

        The problem is cut into chunks of whole KV-head groups (GQA groups never
        split); chunk i's host->device copy, chunk i-1's forward and chunk i-2's
        device->host copy run concurrently on three CUDA streams (two device
        buffer sets), so the PCIe transfers -- not the sum of transfers and
        compute -- bound the end-to-end time.  The pipeline (copies, phase-1 and
        phase-2 launches, cross-stream events) is captured once per (tensors,
        shapes) into a CUDA graph and replayed: one launch instead of ~15 host
        calls per chunk (graph=False runs it eagerly).  Returns ``out`` (host).
        """
        import torch

        B, H, Lq, D = q.shape
        _, KVH, Lk, _ = k.shape
        _check_qkv(q.shape, k.shape, v.shape, self.cfg.causal)
        if H % KVH:
            raise ValueError(f"heads {H} not divisible by kv_heads {KVH}")
        odt = out_dtype or (torch.bfloat16 if q.dtype == torch.bfloat16 else torch.float32)
        if out is None:
            out = torch.empty((B, H, Lq, v.shape[-1]), dtype=odt, pin_memory=True)
        if chunk_kv_heads is None:
            # about one chunk per 50 MB of Q/K/V, 4..16 chunks per call, >= 2 query heads per
            # chunk (a head pair x every q tile fills the 148 SMs at N >= 8K).  Measured best
            # (tools/e2e_chunks.py, e2e_var.py): c2 2 KV heads (4 chunks, 2.70 ms vs 2.87 with 1),
            # c3 2 (16 chunks), c4 4 (8 chunks, 8.24 vs 8.71 ms with 2)
            total = sum(t.numel() * t.element_size() for t in (q, k, v))
            n_target = min(16, max(4, total // (50 * 2**20)))
            want = KVH / max(1, n_target // B)
            pow2 = 1 << max(0, round(math.log2(want))) if want >= 1 else 1  # even chunks
            chunk_kv_heads = max(1, min(KVH, max(-(-2 // (H // KVH)), pow2)))
        # the graph pays off where the host calls outnumber the GPU work (small chunks, e.g.
        # c2: 8.9 -> 2.8 ms); with large chunks its copy nodes overlap worse than eager
        # streams (c3: 16.7 eager vs 18.2 ms graph), so big chunks run eagerly
        chunk_bytes = chunk_kv_heads * Lk * D * q.element_size() * (H // KVH + 2)
        # copies from pageable memory cannot be captured: graphs only for pinned host tensors
        pinned = all(t.is_pinned() for t in (q, k, v, out))
        if not graph or not pinned or chunk_bytes > 24 * 2**20:
            self._host_pipeline(q, k, v, out, chunk_kv_heads)
            if self.validate:
                self._check_finite_host(q, k)
            return out
        # a captured graph points into the pipe entry's device buffers and workspaces, so
        # it lives IN that entry: evicting the entry drops its graphs with the buffers
        entry = self._pipe_entry(q, k, v, out, chunk_kv_heads)
        graphs = entry[4]
        key = tuple((t.data_ptr(), tuple(t.shape), t.dtype) for t in (q, k, v, out))
        g = graphs.get(key)
        if g is None:
            self._host_pipeline(q, k, v, out, chunk_kv_heads)  # eager run: allocations, checks
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._host_pipeline(q, k, v, out, chunk_kv_heads)
            if len(graphs) >= 4:
                graphs.pop(next(iter(graphs)))
            graphs[key] = g
            torch.cuda.synchronize()
        else:
            g.replay()
        if self.validate:
            self._check_finite_host(q, k)
        return out

    def _check_finite_host(self, q, k):
        import torch

        if not (bool(torch.isfinite(q).all()) and bool(torch.isfinite(k).all())):
            raise ValueError(_NONFINITE_MSG)

    def _pipe_entry(self, q, k, v, out, chunk_kv_heads):
        """Streams, device buffers, per-slot forwards and captured graphs of one shape."""
        import torch

        B, H, Lq, D = q.shape
        _, KVH, Lk, _ = k.shape
        DV = v.shape[-1]
        G = H // KVH
        c0 = chunk_kv_heads
        key = (B, H, KVH, Lq, Lk, D, DV, q.dtype, k.dtype, v.dtype, out.dtype, c0)
        pipes = self.__dict__.setdefault("_pipes", {})
        if key not in pipes:
            n_units = B * -(-KVH // c0)
            streams = (torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream())
            bufs, fwds = [], []
            for _ in range(min(2, n_units)):
                bufs.append((torch.empty((1, c0 * G, Lq, D), dtype=q.dtype, device="cuda"),
                             torch.empty((1, c0, Lk, D), dtype=k.dtype, device="cuda"),
                             torch.empty((1, c0, Lk, DV), dtype=v.dtype, device="cuda"),
                             torch.empty((1, c0 * G, Lq, DV), dtype=out.dtype, device="cuda")))
                fwds.append(DmaAttention(self.cfg))
            if len(pipes) >= 2:
                pipes.pop(next(iter(pipes)))  # its graphs (entry[4]) go with it
            pipes[key] = (streams, bufs, fwds, [False], {})
        return pipes[key]

    def _host_pipeline(self, q, k, v, out, chunk_kv_heads):
        import torch

        B, H, Lq, D = q.shape
        _, KVH, Lk, _ = k.shape
        DV = v.shape[-1]
        G = H // KVH
        units = [(b, h0, min(KVH, h0 + chunk_kv_heads)) for b in range(B) for h0 in range(0, KVH, chunk_kv_heads)]
        if len(units) >= 4 and units[-1][2] - units[-1][1] > 1:
            # the pipeline tail (last chunk's forward + D2H) is exposed: finish with single
            # KV heads so it is as short as possible
            b, h0, h1 = units.pop()
            units += [(b, h, h + 1) for h in range(h0, h1)]
        cur = torch.cuda.current_stream()
        # streams, device buffers and per-slot workspaces persist across calls with the same
        # shapes: per-call allocations freed through record_stream kept the caching allocator
        # growing and now and then stalled a call on cudaMalloc / cudaFree (17 ms -> 30-100 ms)
        (s_in, s_cmp, s_out), bufs, fwds, marked, _ = self._pipe_entry(q, k, v, out, chunk_kv_heads)
        # the chunks take the whole problem's KV split count: bit-identical to one device call
        n_split = kv_split_count(q.shape, k.shape, v.shape, self.cfg)
        # every stream starts after the caller's prior work and after all of the previous call
        for st in (s_in, s_cmp, s_out):
            st.wait_stream(cur)
        s_in.wait_stream(s_cmp)
        s_in.wait_stream(s_out)
        s_cmp.wait_stream(s_out)
        ev_cmp = [None, None]  # compute of the slot's previous chunk done (inputs free)
        ev_out = [None, None]  # D2H of the slot's previous chunk done (output free)
        for i, (b, h0, h1) in enumerate(units):
            j = i % 2
            dq, dk, dv, do = (t[:, : (h1 - h0) * G] if n in (0, 3) else t[:, : h1 - h0] for n, t in enumerate(bufs[j]))
            with torch.cuda.stream(s_in):
                if ev_cmp[j] is not None:
                    s_in.wait_event(ev_cmp[j])
                dq.copy_(q[b : b + 1, h0 * G : h1 * G], non_blocking=True)
                dk.copy_(k[b : b + 1, h0:h1], non_blocking=True)
                dv.copy_(v[b : b + 1, h0:h1], non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(s_in)
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(ev_in)
                if ev_out[j] is not None:
                    s_cmp.wait_event(ev_out[j])
                a, _ = fwds[j].prepare(dq, dk, dv, out=do, kv_split=n_split)
                _lib.check(_lib.lib().dma_attention_fwd(a, _lib.stream_ptr(s_cmp)), "dma_attention")
                ev_cmp[j] = torch.cuda.Event()
                ev_cmp[j].record(s_cmp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_cmp[j])
                out[b : b + 1, h0 * G : h1 * G].copy_(do, non_blocking=True)
                ev_out[j] = torch.cuda.Event()
                ev_out[j].record(s_out)
        if not marked[0]:  # once per buffer: freeing waits for these streams
            for t in [x for bs in bufs for x in bs] + [f._ws for f in fwds]:
                for st in (s_in, s_cmp, s_out):
                    t.record_stream(st)
            marked[0] = True
        for st in (s_in, s_cmp, s_out):
            cur.wait_stream(st)


def dma_attention(q, k, v, cfg: AttentionConfig, out=None, out_dtype=None, stream=None, validate=True, kv_split=0):
    """Batched forward on CUDA tensors [B, H, L, D] (also accepts [H, L, D] / [L, D]).

    Functional drop-in: any layout (made contiguous), K / V cast to Q's dtype, and by
    default the reference's ValueError on non-finite Q / K (``validate``).  ``kv_split``:
    0 = the library's small-problem policy, else this many KV splits (1 = unsplit; a caller
    running pieces of a larger problem passes that problem's ``kv_split_count``)."""
    nd = q.dim()
    if nd not in (2, 3, 4):
        raise ValueError("Q, K, V must be 2-D, 3-D or 4-D")
    if not (k.dim() == nd and v.dim() == nd):
        raise ValueError("Q, K, V must have the same number of dimensions")
    while q.dim() < 4:
        q, k, v = q.unsqueeze(0), k.unsqueeze(0), v.unsqueeze(0)
    q, k, v = (to_device(t) for t in (q, k, v))
    if not (q.dtype == k.dtype == v.dtype):
        k, v = k.to(q.dtype), v.to(q.dtype)
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    o = DmaAttention(cfg, validate=validate)(q, k, v, out=out, out_dtype=out_dtype, stream=stream, kv_split=kv_split)
    while o.dim() > nd:
        o = o.squeeze(0)
    return o


class _Shape:
    """Stand-in operand for _args: shape only (no device memory)."""

    def __init__(self, dtype):
        self.dtype = dtype

    def data_ptr(self):
        return 0


def kv_split_count(q_shape, k_shape, v_shape, cfg: AttentionConfig) -> int:
    """KV splits dma_attention_fwd uses for these [B, H, L, D] shapes under the current
    mode (``dma_attention_set_kv_split``; 1 = unsplit).  Small problems (fewer head pairs x
    query tiles than SMs) cut each tile plan into ranges merged in the kernel; the oracle's
    PV emulation takes the same count (``kv_split=``)."""
    import torch

    B, H, Lq, D = q_shape
    _, KVH, Lk, _ = k_shape
    x = _Shape(torch.bfloat16)
    a = _args(cfg, x, x, x, None, B, H, KVH, Lq, Lk, D, v_shape[-1], _lib.DT_F32)
    n = int(_lib.lib().dma_attention_kv_split(a))
    if n < 1:
        _lib.check(-1, "dma_attention_kv_split")
    return n


def mixed_precision_attention(q, k, v, cfg: AttentionConfig):
    """attention.py:282-310 on the GPU.  numpy in -> float64 numpy [Lq, Dv] out."""
    if is_torch(q):
        return dma_attention(q, k, v, cfg)
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    if q.ndim != 2 or k.ndim != 2 or v.ndim != 2:
        raise ValueError("Q, K, V must be 2-D matrices")
    _check_qkv(q.shape, k.shape, v.shape, cfg.causal)
    if (cfg.low_format or cfg.high_format) and q.shape[1] % 32 != 0:
        raise ValueError(f"head dim {q.shape[1]} not divisible by 32")
    for x in (q, k):
        if not np.all(np.isfinite(x)):
            raise ValueError(_NONFINITE_MSG)
    import torch

    o = dma_attention(*(torch.from_numpy(np.ascontiguousarray(x)) for x in (q, k, v)), cfg,
                      out_dtype=torch.float32, validate=False)
    return from_device(o).astype(np.float64)
