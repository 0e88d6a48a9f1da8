"""Error metrics and Bit_high accounting (drop-in for ``mxattn.metrics``).

These are reporting helpers, not part of the forward path: ``similarity`` is
a host-side reduction over two result arrays (metrics.py:35-52);
``high_precision_fraction`` (metrics.py:55-101) uses libdma's integer plan
code -- the same scheduler the kernel runs -- in closed form per row.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib


@dataclass
class MetricReport:
    """metrics.py:16-32."""

    cos_sim: float
    rel_l1: float
    abs_l1: float
    rmse: float
    psnr: float
    high_precision_pct: float | None = None
    seed: int | None = None
    config_echo: dict | None = None


def _np(x):
    if hasattr(x, "detach"):
        x = x.detach().double().cpu().numpy()
    return np.asarray(x, dtype=np.float64).ravel()


def similarity(ref, test) -> MetricReport:
    """Cosine similarity, relative/absolute L1, RMSE, PSNR (metrics.py:35-52)."""
    r, t = _np(ref), _np(test)
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
    return MetricReport(cos_sim=cos, rel_l1=abs_l1 / float(np.abs(r).sum()), abs_l1=abs_l1, rmse=rmse,
                        psnr=math.inf if rmse == 0 else 20.0 * math.log10(peak / rmse))


def high_precision_fraction(len_q: int, len_k: int, tile_m: int, tile_n: int, diag_window: int,
                            sink_window: int, causal: bool) -> float:
    """Fraction of score cells computed on the high-precision path (metrics.py:55-101)."""
    from .attention import AttentionConfig

    AttentionConfig(tile_m=tile_m, tile_n=tile_n, diag_window=diag_window, sink_window=sink_window,
                    causal=causal)  # same validation as the reference
    return float(_lib.lib().dma_high_precision_fraction(len_q, len_k, tile_m, tile_n, diag_window,
                                                         sink_window, int(causal)))
