"""Dense score matrices for error metrics (drop-in for attention.py:120-147, 313-335).

``reference_attention`` / ``reference_scores`` (the full-precision oracle the
reference uses for "error vs full precision") and ``mixed_precision_scores``
(post-softmax probabilities under the DMA per-tile precision assignment) are
reporting helpers: their output is an N x N matrix, so they are dense float64
GEMMs on the GPU (torch, CUDA) over operands produced by libdma -- the
bit-exact ``quantize_dual`` and ``dma_dequantize`` -- not the fused kernel.
Inputs: 2-D numpy arrays or torch tensors (one head, like the reference);
outputs match the input kind (numpy in -> float64 numpy out).
"""

from __future__ import annotations

import math

import numpy as np

from ._device import from_device, is_torch, to_device_f64
from .attention import AttentionConfig, _check_qkv, causal_tile_plan, noncausal_tile_plan
from .formats import MXFP8_E4M3, NVFP4
from .quantize import dequantize_high, dequantize_low, quantize_dual, softmax_prescale


def _softmax_rows(logits, base2: bool):
    """attention.py:138-147 (row max of -inf rows -> 0; masked entries -> 0; empty rows -> 0)."""
    import torch

    m = logits.max(dim=1, keepdim=True).values
    m = torch.where(torch.isfinite(m), m, torch.zeros_like(m))
    z = logits - m
    p = torch.exp2(z) if base2 else torch.exp(z)
    p = torch.where(torch.isfinite(logits), p, torch.zeros_like(p))
    denom = p.sum(dim=1, keepdim=True)
    return p / torch.where(denom > 0, denom, torch.ones_like(denom))


def _out(x, like_torch):
    return x if like_torch else from_device(x)


def reference_scores(q, k, causal: bool = False):
    """attention.py:126-135: dense softmax(Q K^T / sqrt(D)) probabilities (base e), float64."""
    import torch

    torch_in = is_torch(q)
    q, k = to_device_f64(q), to_device_f64(k)
    _check_qkv(tuple(q.shape), tuple(k.shape), tuple(k.shape), causal)
    logits = (q @ k.T) / math.sqrt(q.shape[1])
    if causal:
        lq = q.shape[0]
        keep = torch.arange(lq, device=q.device)[:, None] >= torch.arange(lq, device=q.device)[None, :]
        logits = torch.where(keep, logits, torch.full_like(logits, -math.inf))
    return _out(_softmax_rows(logits, base2=False), torch_in)


def reference_attention(q, k, v, causal: bool = False):
    """attention.py:120-123: reference_scores(q, k) @ v in float64."""
    torch_in = is_torch(q)
    p = reference_scores(to_device_f64(q), to_device_f64(k), causal)
    return _out(p @ to_device_f64(v), torch_in)


def _operands(q, k, cfg: AttentionConfig):
    """attention.py:247-279 (`both`): dequantized low / high copies of Q and K, base-2 logit domain."""

    def both(x, is_query):
        if cfg.low_format is None and cfg.high_format is None:
            ident = softmax_prescale(x) if is_query else x
            return ident, ident
        high_fmt = cfg.high_format or MXFP8_E4M3
        low_fmt = NVFP4 if (cfg.low_format is None or cfg.low_format.element.bits == 8) else cfg.low_format
        t = quantize_dual(x, is_query=is_query, low_format=low_fmt, high_format=high_fmt,
                          granularity=cfg.granularity)
        high = dequantize_high(t) if cfg.high_format is not None else (softmax_prescale(x) if is_query else x)
        if cfg.low_format is None:
            low = softmax_prescale(x) if is_query else x
        elif cfg.low_format.element.bits == 8:
            low = high
        else:
            low = dequantize_low(t)
        return low, high

    return both(q, True) + both(k, False)


def mixed_precision_scores(q, k, cfg: AttentionConfig):
    """attention.py:313-335: dense base-2 post-softmax probabilities under the same per-tile
    precision assignment as ``mixed_precision_attention`` (unvisited blocks fully masked)."""
    import torch

    torch_in = is_torch(q)
    q, k = to_device_f64(q), to_device_f64(k)
    _check_qkv(tuple(q.shape), tuple(k.shape), tuple(k.shape), cfg.causal)
    if (cfg.low_format or cfg.high_format) and q.shape[1] % 32 != 0:
        raise ValueError(f"head dim {q.shape[1]} not divisible by 32")
    if not (torch.isfinite(q).all() and torch.isfinite(k).all()):
        raise ValueError("quantize_dual: input contains non-finite values")
    q_low, q_high, k_low, k_high = _operands(q, k, cfg)
    len_q, len_k = q.shape[0], k.shape[0]
    plan_fn = causal_tile_plan if cfg.causal else noncausal_tile_plan
    logits = torch.full((len_q, len_k), -math.inf, dtype=torch.float64, device=q.device)
    for q_tile in range(-(-len_q // cfg.tile_m)):
        q0, q1 = q_tile * cfg.tile_m, min((q_tile + 1) * cfg.tile_m, len_q)
        # one GEMM per precision over the visited key tiles (same cells as the reference's tile loop)
        for high in (False, True):
            tiles = [t for t, h in plan_fn(q_tile, len_q, len_k, cfg) if h == high]
            if not tiles:
                continue
            cols = torch.cat([torch.arange(t * cfg.tile_n, min((t + 1) * cfg.tile_n, len_k), device=q.device)
                              for t in tiles])
            block = (q_high if high else q_low)[q0:q1] @ (k_high if high else k_low)[cols].T
            if cfg.causal:  # attention.py:178-184
                qpos = torch.arange(q0, q1, device=q.device)[:, None]
                block = torch.where(qpos >= cols[None, :], block, torch.full_like(block, -math.inf))
            logits[q0:q1, cols] = block
    return _out(_softmax_rows(logits, base2=True), torch_in)


def score_similarity(q, k, cfg: AttentionConfig, block_rows: int | None = None):
    """``similarity(reference_scores(q, k, causal), mixed_precision_scores(q, k, cfg))``
    (metrics.py:35-52 over attention.py:126-135 / 313-335) without the N x N matrices: the
    two probability matrices are produced ``block_rows`` query rows at a time (softmax is
    row-wise, and the row blocks are whole plan query tiles), and the metric sums
    (dot, squared norms, L1 terms, squared error, peak) are accumulated per block in float64.
    Memory is O(block_rows x Lk) instead of O(Lq x Lk): a 32K x 32K head needs ~0.3 GB, not
    the 2 x 8.6 GB of the dense matrices.  Returns a ``MetricReport``."""
    import torch

    from .metrics import MetricReport

    q, k = to_device_f64(q), to_device_f64(k)
    _check_qkv(tuple(q.shape), tuple(k.shape), tuple(k.shape), cfg.causal)
    if (cfg.low_format or cfg.high_format) and q.shape[1] % 32 != 0:
        raise ValueError(f"head dim {q.shape[1]} not divisible by 32")
    if not (torch.isfinite(q).all() and torch.isfinite(k).all()):
        raise ValueError("quantize_dual: input contains non-finite values")
    len_q, len_k, d = q.shape[0], k.shape[0], q.shape[1]
    if block_rows is None:
        block_rows = max(cfg.tile_m, (1 << 23) // max(len_k, 1) // cfg.tile_m * cfg.tile_m)
    block_rows = max(cfg.tile_m, block_rows // cfg.tile_m * cfg.tile_m)
    q_low, q_high, k_low, k_high = _operands(q, k, cfg)
    plan_fn = causal_tile_plan if cfg.causal else noncausal_tile_plan
    scale = 1.0 / math.sqrt(d)
    kcols = torch.arange(len_k, device=q.device)
    acc = torch.zeros(6, dtype=torch.float64, device=q.device)  # r.t, |r|^2, |t|^2, sum|r-t|, sum (r-t)^2, sum|r|
    peak = torch.zeros((), dtype=torch.float64, device=q.device)
    for r0 in range(0, len_q, block_rows):
        r1 = min(r0 + block_rows, len_q)
        qpos = torch.arange(r0, r1, device=q.device)[:, None]
        # reference probabilities (base e, working precision) for rows r0:r1
        lr = (q[r0:r1] @ k.T) * scale
        if cfg.causal:
            lr = torch.where(qpos >= kcols[None, :], lr, torch.full_like(lr, -math.inf))
        ref = _softmax_rows(lr, base2=False)
        del lr
        # mixed-precision probabilities (base 2, per-tile precision) for the same rows
        lt = torch.full((r1 - r0, len_k), -math.inf, dtype=torch.float64, device=q.device)
        for q_tile in range(r0 // cfg.tile_m, -(-r1 // cfg.tile_m)):
            q0, q1 = q_tile * cfg.tile_m, min((q_tile + 1) * cfg.tile_m, len_q)
            for high in (False, True):
                tiles = [t for t, h in plan_fn(q_tile, len_q, len_k, cfg) if h == high]
                if not tiles:
                    continue
                cols = torch.cat([torch.arange(t * cfg.tile_n, min((t + 1) * cfg.tile_n, len_k), device=q.device)
                                  for t in tiles])
                block = (q_high if high else q_low)[q0:q1] @ (k_high if high else k_low)[cols].T
                if cfg.causal:  # attention.py:178-184
                    qp = torch.arange(q0, q1, device=q.device)[:, None]
                    block = torch.where(qp >= cols[None, :], block, torch.full_like(block, -math.inf))
                lt[q0 - r0:q1 - r0, cols] = block
        tst = _softmax_rows(lt, base2=True)
        del lt
        diff = ref - tst
        acc += torch.stack([(ref * tst).sum(), (ref * ref).sum(), (tst * tst).sum(), diff.abs().sum(),
                            (diff * diff).sum(), ref.abs().sum()])
        peak = torch.maximum(peak, ref.abs().max())
        del ref, tst, diff
    dot, rr, tt, abs_l1, sq, r_l1 = (float(x) for x in acc.tolist())
    if rr == 0:
        raise ValueError("metrics are undefined for an all-zero reference")
    rn, tn = math.sqrt(rr), math.sqrt(tt)
    rmse = math.sqrt(sq / (len_q * len_k))
    pk = float(peak)
    return MetricReport(cos_sim=dot / (rn * tn) if tn > 0 else 0.0, rel_l1=abs_l1 / r_l1, abs_l1=abs_l1, rmse=rmse,
                        psnr=math.inf if rmse == 0 else 20.0 * math.log10(pk / rmse))


__all__ = ["mixed_precision_scores", "reference_attention", "reference_scores", "score_similarity"]
_ = np  # numpy inputs are accepted through to_device_f64
