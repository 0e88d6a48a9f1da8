"""Deterministic synthetic inputs shared by the golden generator and the tests.

numpy's PCG64 stream is stable across numpy versions, so fixtures only need
to store the seed and shape, not the input arrays.
"""

from __future__ import annotations

import numpy as np


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float64 values to the nearest bfloat16 (ties to even), returned as float64."""
    f = np.asarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def randn_bf16(seed: int, *shape, scale: float = 1.0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return bf16_round(rng.standard_normal(shape) * scale)


def adversarial_rows(cols: int, seed: int = 7) -> np.ndarray:
    """Rows that stress the quantizer's edge cases (zeros, -0.0, ties, tiny blocks, huge range)."""
    rng = np.random.default_rng(seed)
    rows = []
    rows.append(np.zeros(cols))
    rows.append(-np.zeros(cols))
    rows.append(np.full(cols, 3.0))
    rows.append(np.full(cols, -6.0 * 1024))
    alt = np.zeros(cols)
    alt[1::2] = -0.0
    alt[::7] = 1.0
    rows.append(alt)
    r = bf16_round(rng.standard_normal(cols))
    r[:16] = 1e-6
    rows.append(r)
    r = bf16_round(rng.standard_normal(cols))
    r[16:32] = 2.0 ** -120
    r[40:44] = -(2.0 ** -121)
    rows.append(r)
    rows.append(bf16_round(rng.standard_normal(cols)) * 1e30)
    rows.append(bf16_round(rng.standard_normal(cols)) * 1e-30)
    # Row maxima whose mantissa sits on a structural E4M3 midpoint (21*2^k family).
    for mant in (147, 168, 189, 210, 231, 252):
        r = bf16_round(rng.standard_normal(cols))
        r[3] = mant * 2.0 ** -5
        r[5] = -mant * 2.0 ** -6
        r[:] = np.clip(r, -mant * 2.0 ** -5, mant * 2.0 ** -5)
        rows.append(r)
    # Exact E2M1/E4M3 midpoints after scaling.
    r = np.tile(np.array([0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0, 6.0]), cols // 8)
    rows.append(r * np.where(np.arange(cols) % 3 == 0, -1.0, 1.0))
    rows.append(np.tile(np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 2688.0]), cols // 8))
    return np.stack(rows)
