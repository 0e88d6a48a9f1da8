"""The binding a maintainer of the reference package ``mxattn`` would add as
``mxattn/_dma_cuda.py`` (INTEGRATION.md shows it verbatim): ctypes over the C-ABI of
libdma (include/dma.h), no import of this repository's Python package.

``mixed_precision_attention_cuda(q, k, v, cfg)`` takes the reference's own arguments
(2-D q/k/v array-likes, an ``mxattn.attention.AttentionConfig``, attention.py:282) and
returns a float64 numpy array like the reference.  Inputs go to the device as float64
(``in_dtype`` DMA_DT_F64) so ``quantize_dual`` sees exactly the values the reference
quantizes (attention.py:248-250 widens to float64).  Validation stays with the reference
(attention.py:109-119, 252-253); NaN / Inf in Q or K raise ValueError like
quantize.py:142-143 through the ABI's device flag.  ``pv_mode`` 0 = block-scaled MXFP8
PV (the north-star kernel), 1 = bf16 PV (parity mode).
"""

import ctypes
import math
import os

import numpy as np
import torch

_lib = ctypes.CDLL(os.environ.get("DMA_LIB", "libdma.so"))


class DmaAttnArgs(ctypes.Structure):  # include/dma.h: DmaAttnArgs (ABI 2)
    _fields_ = [("q", ctypes.c_void_p), ("k", ctypes.c_void_p), ("v", ctypes.c_void_p),
                ("o", ctypes.c_void_p), ("in_dtype", ctypes.c_int32), ("out_dtype", ctypes.c_int32),
                ("batch", ctypes.c_int64), ("heads", ctypes.c_int64), ("kv_heads", ctypes.c_int64),
                ("len_q", ctypes.c_int64), ("len_k", ctypes.c_int64), ("head_dim", ctypes.c_int64),
                ("v_dim", ctypes.c_int64), ("tile_m", ctypes.c_int32), ("tile_n", ctypes.c_int32),
                ("diag_window", ctypes.c_int32), ("sink_window", ctypes.c_int32), ("causal", ctypes.c_int32),
                ("low_format", ctypes.c_int32), ("high_format", ctypes.c_int32),
                ("granularity", ctypes.c_int32), ("pv_mode", ctypes.c_int32), ("kv_split", ctypes.c_int32),
                ("prescale", ctypes.c_double), ("workspace", ctypes.c_void_p),
                ("workspace_bytes", ctypes.c_size_t), ("nonfinite", ctypes.c_void_p)]


_lib.dma_attention_workspace_bytes.restype = ctypes.c_size_t
_lib.dma_attention_workspace_bytes.argtypes = [ctypes.POINTER(DmaAttnArgs)]
_lib.dma_attention_fwd.argtypes = [ctypes.POINTER(DmaAttnArgs), ctypes.c_void_p]
_lib.dma_last_error.restype = ctypes.c_char_p
_FMT = {None: 0, "mxfp8_e4m3": 1, "mxfp8_e5m2": 2, "mxfp4": 3, "nvfp4": 4}  # formats.py:101-109
_GRAN = {"token": 0, "block": 1, "tensor": 2}                              # quantize.py:61-66
DMA_DT_F64, DMA_DT_F32 = 0, 1


def mixed_precision_attention_cuda(q, k, v, cfg, pv_mode=0):
    q, k, v = (torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64))).cuda() for x in (q, k, v))
    o = torch.empty(q.shape[0], v.shape[1], dtype=torch.float32, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    a = DmaAttnArgs(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), DMA_DT_F64, DMA_DT_F32,
                    1, 1, 1, q.shape[0], k.shape[0], q.shape[1], v.shape[1],
                    cfg.tile_m, cfg.tile_n, cfg.diag_window, cfg.sink_window, int(cfg.causal),
                    _FMT[getattr(cfg.low_format, "name", None)], _FMT[getattr(cfg.high_format, "name", None)],
                    _GRAN[cfg.granularity.value], pv_mode, 0,
                    math.log2(math.e) / math.sqrt(q.shape[1]))  # quantize.py:92-95, float64
    ws = torch.empty(max(1, _lib.dma_attention_workspace_bytes(a)), dtype=torch.uint8, device="cuda")
    a.workspace, a.workspace_bytes, a.nonfinite = ws.data_ptr(), ws.numel(), flag.data_ptr()
    rc = _lib.dma_attention_fwd(a, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    if rc != 0:
        raise (ValueError if rc < 0 else RuntimeError)(_lib.dma_last_error().decode())
    if int(flag.item()):
        raise ValueError("quantize_dual: input contains non-finite values")  # quantize.py:143
    return o.cpu().numpy().astype(np.float64)
