"""Tile-level online-softmax helpers of the reference API (attention.py:83-106, 150-184).

``OnlineSoftmaxState``, ``online_softmax_update`` and ``apply_causal_mask`` are the
building blocks the reference composes its tiled forward from; users of
``mxattn.attention`` call them to write their own tile loops.  The fused kernel
(``dma_attn_pp_kernel``) does the same arithmetic in registers / TMEM and never
calls these.  Here they are float64 torch ops on the GPU (like ``scores.py``):
numpy in -> numpy out, torch in -> torch out, same semantics as the reference:

* ``OnlineSoftmaxState.fresh(rows, d)``: m = -inf, l = 0, o = 0 (attention.py:97-102);
  ``normalized()`` divides by l where l > 0, else by 1 (:104-106);
* ``online_softmax_update``: rows whose running max stays -inf pass through with
  alpha = 1; -inf scores contribute 0; base 2 or e (:150-175);
* ``apply_causal_mask``: -inf where query_start + a < key_start + b (:178-184).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from ._device import from_device, is_torch, to_device_f64


@dataclass
class OnlineSoftmaxState:
    """Streaming softmax accumulator for one query tile (attention.py:83-106).

    ``m`` running row maximum, ``l`` running normalizer, ``o`` unnormalized output;
    float64 tensors on the GPU (``numpy()`` returns host copies)."""

    m: object
    l: object
    o: object

    @classmethod
    def fresh(cls, rows: int, head_dim: int) -> "OnlineSoftmaxState":
        import torch

        from ._device import _torch

        _torch()
        dev = "cuda"
        return cls(m=torch.full((rows,), -math.inf, dtype=torch.float64, device=dev),
                   l=torch.zeros(rows, dtype=torch.float64, device=dev),
                   o=torch.zeros((rows, head_dim), dtype=torch.float64, device=dev))

    def normalized(self):
        import torch

        l = torch.where(self.l > 0, self.l, torch.ones_like(self.l))
        return self.o / l[:, None]

    def numpy(self):
        return from_device(self.m), from_device(self.l), from_device(self.o)


def _state_on_device(state: OnlineSoftmaxState) -> OnlineSoftmaxState:
    return OnlineSoftmaxState(to_device_f64(state.m), to_device_f64(state.l), to_device_f64(state.o))


def online_softmax_update(state: OnlineSoftmaxState, scores, v_tile, base2: bool = False) -> OnlineSoftmaxState:
    """Fold one tile of scores and values into the running state (attention.py:150-175)."""
    import torch

    st = _state_on_device(state)
    s = to_device_f64(scores)
    v = to_device_f64(v_tile)
    exp = torch.exp2 if base2 else torch.exp
    tile_max = s.max(dim=1).values if s.shape[1] else torch.full_like(st.m, -math.inf)
    m_new = torch.maximum(st.m, tile_max)
    live = torch.isfinite(m_new)
    zero = torch.zeros_like(m_new)
    alpha = torch.where(live, exp(torch.where(live, st.m - m_new, zero)), torch.ones_like(m_new))
    finite = torch.isfinite(s)
    shifted = s - torch.where(live, m_new, zero)[:, None]
    p = torch.where(finite, exp(torch.where(finite, shifted, torch.zeros_like(shifted))), torch.zeros_like(s))
    return OnlineSoftmaxState(m=m_new, l=st.l * alpha + p.sum(dim=1), o=st.o * alpha[:, None] + p @ v)


def apply_causal_mask(scores, query_start: int, key_start: int):
    """-inf wherever query_start + a precedes key_start + b (attention.py:178-184)."""
    import torch

    torch_in = is_torch(scores)
    s = to_device_f64(scores)
    rows, cols = s.shape
    qpos = query_start + torch.arange(rows, device=s.device)[:, None]
    kpos = key_start + torch.arange(cols, device=s.device)[None, :]
    out = torch.where(qpos >= kpos, s, torch.full_like(s, -math.inf))
    return out if torch_in else from_device(out)
