/*
 * dma.h -- C-ABI of libdma (the B200-native DMA forward path).
 *
 * DMA = Diagonal-Tiled Mixed-Precision Attention (arXiv 2604.03950).  The
 * reference (``mxattn``, /root/reference/pkg/src/mxattn) is a Python/numpy
 * package with no FFI of its own; each entry point below replaces one of its
 * Python functions and is bound by ctypes from
 * ``paper_2604_03950_b200/_lib.py`` (see INTEGRATION.md for the binding a
 * maintainer of the reference would add).
 *
 *   dma_quantize_dual   <- quantize.py:122  quantize_dual(x, is_query, low_format, high_format, granularity)
 *   dma_dequantize      <- quantize.py:215  dequantize_low(t) / quantize.py:232 dequantize_high(t)
 *   dma_encode_e2m1     <- formats.py:124   encode_e2m1(x)
 *   dma_encode_fp8      <- formats.py:205   encode_fp8(x, fmt)
 *   dma_attention_fwd   <- attention.py:282 mixed_precision_attention(q, k, v, cfg)
 *   dma_attention_workspace_bytes           (sizing helper for the above)
 *   dma_high_precision_fraction <- metrics.py:55 high_precision_fraction(...)
 *   dma_tile_plan       <- attention.py:191 causal_tile_plan / :212 noncausal_tile_plan
 *   dma_decode_attention    (SURVEY 8 f rank 4: decode over an MX key cache; rows of
 *                            mixed_precision_attention, attention.py:282, for new tokens)
 *
 * Conventions
 *   - every pointer to tensor data is a DEVICE pointer (cudaMalloc / torch);
 *     the library never allocates, frees or synchronises; all work is
 *     enqueued on ``stream`` (a cudaStream_t passed as void*; NULL = legacy).
 *   - return 0 on success, DMA_EINVAL / DMA_EUNSUPPORTED (< 0) on bad
 *     arguments, a positive cudaError_t on a CUDA failure.  dma_last_error()
 *     returns a thread-local message for the last failure.
 *   - argument validation that raises ValueError in the reference is done by
 *     the Python layer before the call, with the reference's messages.
 */
#ifndef DMA_H_
#define DMA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DMA_ABI_VERSION 2

enum { DMA_OK = 0, DMA_EINVAL = -1, DMA_EUNSUPPORTED = -2 };

/* element / MX formats -- formats.py:101-104 */
enum {
  DMA_FMT_NONE = 0,       /* identity (AttentionConfig low/high_format=None) */
  DMA_FMT_MXFP8_E4M3 = 1, /* E4M3 elements, E8M0 scale per 32 */
  DMA_FMT_MXFP8_E5M2 = 2, /* E5M2 elements, E8M0 scale per 32 */
  DMA_FMT_MXFP4 = 3,      /* E2M1 elements, E8M0 scale per 32, single level */
  DMA_FMT_NVFP4 = 4       /* E2M1 elements, E4M3 scale per 16, two level */
};

/* quantization-scale grouping -- quantize.py:61-66 */
enum { DMA_GRAN_TOKEN = 0, DMA_GRAN_BLOCK = 1, DMA_GRAN_TENSOR = 2 };

/* input / output dtypes */
enum { DMA_DT_F64 = 0, DMA_DT_F32 = 1, DMA_DT_BF16 = 2 };

/* PV contraction mode (the reference keeps P and V in float64, attention.py:174) */
enum {
  DMA_PV_MXFP8 = 0, /* P -> E4M3 (x2^8) in registers, V -> MXFP8 along keys: block-scaled tcgen05 */
  DMA_PV_BF16 = 1   /* P -> bf16, V bf16: kind::f16 tcgen05 ("parity" mode) */
};

/* ---------------------------------------------------------------------------
 * quantize_dual over ``n_mat`` row-major matrices [rows, cols] (cols % 32 == 0).
 * Outputs use the reference's canonical layouts (quantize.py:69-89):
 *   packed_low  u8  [n_mat, rows, cols/2]          (even col = low nibble)
 *   scales_low  u8  [n_mat, rows, cols/16 (NVFP4) | cols/32 (MXFP4)]
 *   high_codes  u8  [n_mat, rows, cols]
 *   scales_high u8  [n_mat, rows, cols/32]
 *   quant_scale f64 [n_mat, rows] (TOKEN) | [n_mat, rows, cols/32] (BLOCK) | [n_mat] (TENSOR)
 *   nonfinite   u32 [1] (optional): set to 1 if any input is NaN/Inf
 * Any output pointer may be NULL to skip it.  ``workspace`` needs
 * dma_quantize_workspace_bytes() bytes (TENSOR granularity only).
 * ------------------------------------------------------------------------- */
typedef struct {
  const void* x;
  int32_t x_dtype;
  int32_t is_query; /* multiply by ``prescale`` first (quantize.py:92-95) */
  int64_t n_mat, rows, cols;
  int64_t mat_stride, row_stride; /* in elements */
  double prescale;                /* log2(e)/sqrt(cols), computed by the caller in float64 */
  int32_t low_format, high_format, granularity;
  int32_t _pad;
  uint8_t* packed_low;
  uint8_t* scales_low;
  uint8_t* high_codes;
  uint8_t* scales_high;
  double* quant_scale;
  uint32_t* nonfinite;
  void* workspace;
  size_t workspace_bytes;
} DmaQuantArgs;

size_t dma_quantize_workspace_bytes(const DmaQuantArgs* a);
int dma_quantize_dual(const DmaQuantArgs* a, void* stream);

/* dequantize_low (which = 0) / dequantize_high (which = 1) -> f64 [n_mat, rows, cols] */
int dma_dequantize(int32_t which, int32_t low_format, int32_t high_format, int32_t granularity,
                   int64_t n_mat, int64_t rows, int64_t cols, const uint8_t* packed_low,
                   const uint8_t* scales_low, const uint8_t* high_codes, const uint8_t* scales_high,
                   const double* quant_scale, double* out, void* stream);

/* element codecs over n f64 values (callers pre-validate range/finiteness) */
int dma_encode_e2m1(const double* x, int64_t n, uint8_t* codes, void* stream);
int dma_encode_fp8(const double* x, int64_t n, int32_t e5m2, uint8_t* codes, void* stream);

/* ---------------------------------------------------------------------------
 * The fused DMA forward: Q [B, H, Lq, D], K [B, KVH, Lk, D], V [B, KVH, Lk, DV]
 * (contiguous, dtype in_dtype) -> O [B, H, Lq, DV] (out_dtype f32 or bf16).
 * Query head h attends with key/value head h / (H / KVH) (GQA).
 * Phase 1 quantizes Q/K (bit-exact quantize_dual) and V into ``workspace``;
 * phase 2 runs the diagonal-tiled attention with tcgen05 block-scaled MMAs.
 * Covered: tile_m = tile_n = 128, head_dim = v_dim in {64, 128}, TOKEN / TENSOR
 * granularity with MX formats on the block-scaled QK path; BLOCK granularity and
 * None (identity) formats on the bf16-operand path (QK on bf16 copies of the
 * reference's dequantized operands, attention.py:247-279).
 * ------------------------------------------------------------------------- */
typedef struct {
  const void* q;
  const void* k;
  const void* v;
  void* o;
  int32_t in_dtype, out_dtype;
  int64_t batch, heads, kv_heads, len_q, len_k, head_dim, v_dim;
  int32_t tile_m, tile_n, diag_window, sink_window, causal;
  int32_t low_format, high_format, granularity, pv_mode;
  /* KV splits for this call (dma_attention_set_kv_split): 0 = the library's policy (default),
   * 1 = unsplit, n >= 2 = n splits (capped by the plan length and 16).  A caller that cuts
   * one problem into pieces passes the whole problem's count (dma_attention_kv_split) so the
   * pieces reproduce its output bit for bit.  (Formerly padding: old callers pass 0.) */
  int32_t kv_split;
  double prescale; /* log2(e)/sqrt(head_dim), float64 */
  void* workspace;
  size_t workspace_bytes;
  /* optional (may be NULL): u32 device flag, zeroed by the call and set to 1 if Q or K holds
   * a NaN / Inf (the reference raises ValueError there, quantize.py:142-143); ABI 2 */
  uint32_t* nonfinite;
} DmaAttnArgs;

size_t dma_attention_workspace_bytes(const DmaAttnArgs* a);
/* returns DMA_EUNSUPPORTED for configurations the sm_100a kernel does not cover */
int dma_attention_supported(const DmaAttnArgs* a);
int dma_attention_fwd(const DmaAttnArgs* a, void* stream);
/* phase 2 only, on operands already quantized into ``workspace`` by a previous
 * dma_attention_fwd (or dma_attention_quantize) with the same shapes */
int dma_attention_quantize(const DmaAttnArgs* a, void* stream);
int dma_attention_core(const DmaAttnArgs* a, void* stream);

/* ---------------------------------------------------------------------------
 * Host-side plan helpers (integer-exact restatements of attention.py:191-233
 * and metrics.py:55-101; the same arithmetic runs inside the kernel).
 * dma_tile_plan writes up to ``cap`` entries (key_tile*2 + high) and returns
 * the plan length.
 * ------------------------------------------------------------------------- */
int64_t dma_tile_plan(int64_t q_tile, int64_t len_q, int64_t len_k, int32_t tile_m, int32_t tile_n,
                      int32_t diag_window, int32_t sink_window, int32_t causal, int64_t* out,
                      int64_t cap);
double dma_high_precision_fraction(int64_t len_q, int64_t len_k, int32_t tile_m, int32_t tile_n,
                                   int32_t diag_window, int32_t sink_window, int32_t causal);

/* ---------------------------------------------------------------------------
 * Decode over a quantized key cache.  n_q new query rows per sequence at
 * absolute positions pos .. pos + n_q - 1; query i sees keys [0, pos + i] and
 * its output equals row pos + i of dma_attention_fwd / mixed_precision_attention
 * over the whole sequence (causal, same tile_m / tile_n / windows / formats;
 * TOKEN granularity, so every cached row is quantized once and never changes).
 *   q_*  : dma_quantize_dual outputs of the new queries, is_query = 1,
 *          n_mat = batch * heads, rows = n_q (canonical layouts above)
 *   k_*  : dma_quantize_dual outputs of the cached keys, is_query = 0,
 *          [batch * kv_heads, capacity, ...] (rows >= pos + n_q are ignored)
 *   v    : value cache [batch, kv_heads, capacity, v_dim], bf16
 *   o    : [batch, heads, n_q, v_dim], out_dtype f32 or bf16
 * The low_format pointers are unused (may be NULL) when low_format is MXFP8
 * (the reference then scores every tile with the high operands).
 * QK uses the block-scaled elements exactly (f32 products / sums), P and V stay
 * f32 / bf16 (no PV quantization in decode).  head_dim, v_dim in {64, 128}.
 * ------------------------------------------------------------------------- */
typedef struct {
  const uint8_t* q_packed_low;
  const uint8_t* q_scales_low;
  const uint8_t* q_high_codes;
  const uint8_t* q_scales_high;
  const double* q_quant_scale;
  const uint8_t* k_packed_low;
  const uint8_t* k_scales_low;
  const uint8_t* k_high_codes;
  const uint8_t* k_scales_high;
  const double* k_quant_scale;
  const void* v;
  void* o;
  int32_t v_dtype, out_dtype;
  int64_t batch, heads, kv_heads, n_q, capacity, pos, head_dim, v_dim;
  int32_t tile_m, tile_n, diag_window, sink_window;
  int32_t low_format, high_format, granularity;
  int32_t _pad;
  void* workspace;
  size_t workspace_bytes;
} DmaDecodeArgs;

size_t dma_decode_workspace_bytes(const DmaDecodeArgs* a);
int dma_decode_attention(const DmaDecodeArgs* a, void* stream);

/* self-test of one tcgen05 block-scaled MMA tile (used by the GPU tests) */
int dma_selftest_mma(int32_t kind, int32_t K, const uint8_t* a, const uint8_t* b, const uint8_t* sfa,
                     const uint8_t* sfb, float* d, void* stream);

const char* dma_last_error(void);
int dma_abi_version(void);
/* number of kernels launched by the last dma_attention_fwd on this thread */
int dma_last_launch_count(void);
/* Selects the fused forward for dma_attention_fwd (phase 1 inside the attention kernel, one
 * kernel per call; bf16 inputs, TOKEN granularity, block-scaled PV): 1 on, 0 off (default,
 * the two-phase path is faster on B200).  Returns the previous setting. */
int dma_attention_set_fused(int on);

/* KV splits of the ping-pong forward for small problems (fewer head pairs x query tiles
 * than SMs): each pair's tile plan (attention.py:191-233) is cut into ranges of >= 2 key
 * tiles processed by different CTAs and merged in the kernel (same online-softmax algebra
 * as attention.py:150-175 across the ranges).  mode: -1 auto (default), 0 or 1 off, n >= 2
 * force n splits (capped by the plan length and 16).  Also DMA_KV_SPLIT.  Returns the
 * previous mode. */
int dma_attention_set_kv_split(int mode);

/* The KV split count dma_attention_fwd uses for `a` under the current mode (1 = unsplit),
 * -1 on invalid arguments. */
int dma_attention_kv_split(const DmaAttnArgs* a);

#ifdef __cplusplus
}
#endif
#endif /* DMA_H_ */
