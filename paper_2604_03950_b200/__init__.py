"""B200-native (sm_100a) DMA: Diagonal-Tiled Mixed-Precision Attention.

Drop-in for the reference package ``mxattn`` (formats / quantize / attention /
metrics); every compute entry point runs hand-written CUDA in ``libdma.so``.
"""

from .formats import (  # noqa: F401
    E2M1, E4M3, E5M2, FORMATS, MXFP4, MXFP8_E4M3, MXFP8_E5M2, NVFP4, E8M0_BIAS, E8M0_MAX_RAW,
    ElementFormat, ElementKind, MxFormatSpec, PackedFp4Buffer, ScaleKind, decode_e2m1, decode_fp8,
    e8m0_decode, e8m0_encode, encode_e2m1, encode_fp8, pack_fp4, unpack_fp4,
)
from .quantize import (  # noqa: F401
    QUANT_RANGE, DualQuantizedTensor, Granularity, dequantize_high, dequantize_low, quantize_dual,
    softmax_prescale,
)
from .attention import (  # noqa: F401
    AttentionConfig, DmaAttention, causal_tile_plan, dma_attention, mixed_precision_attention,
    noncausal_tile_plan,
)
from .softmax import OnlineSoftmaxState, apply_causal_mask, online_softmax_update  # noqa: F401
from .metrics import MetricReport, high_precision_fraction, similarity  # noqa: F401
from .decode import DmaKVCache  # noqa: F401
from .scores import mixed_precision_scores, reference_attention, reference_scores, score_similarity  # noqa: F401
