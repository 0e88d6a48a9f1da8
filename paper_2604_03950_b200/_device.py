"""Host <-> device plumbing (torch is used for device memory and streams only)."""

from __future__ import annotations

import numpy as np


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2604_03950_b200 needs a CUDA (sm_100a) device; there is no CPU fallback")
    return torch


def is_torch(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def to_device_f64(x):
    torch = _torch()
    if is_torch(x):
        return x.to(device="cuda", dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64))).cuda()


def to_device(x, allowed=("float64", "float32", "bfloat16")):
    """Device tensor in one of the kernel's input dtypes, contiguous, 16B aligned."""
    torch = _torch()
    if is_torch(x):
        t = x
        if str(t.dtype).replace("torch.", "") not in allowed:
            t = t.to(torch.float64)
        t = t.to("cuda").contiguous()
        if t.data_ptr() % 16:
            t = t.clone()
        return t
    a = np.asarray(x)
    if a.dtype not in (np.float64, np.float32):
        a = a.astype(np.float64)
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def dtype_code(t) -> int:
    from . import _lib

    name = str(t.dtype).replace("torch.", "")
    return {"float64": _lib.DT_F64, "float32": _lib.DT_F32, "bfloat16": _lib.DT_BF16}[name]


def from_device(t) -> np.ndarray:
    return t.detach().cpu().numpy()
