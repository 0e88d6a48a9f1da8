// C-ABI: the DMA forward = phase 1 (quantize Q, K, V into the workspace in
// tcgen05 operand layout) + phase 2 (dma_attn_kernel).  attention.py:282-310.
#include <cuda.h>
#include <cuda_bf16.h>

#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "attn.cuh"
#include "attn_pp.cuh"
#include "attn_sk.cuh"
#include "attn_ws.cuh"
#include "launch.h"
#include "common.cuh"
#include "quant.cuh"

namespace dma {

int quantize_impl(const DmaQuantArgs* a, uint8_t* sf_low_op, uint8_t* sf_high_op, float* qs_f32, int64_t rows_pad,
                  cudaStream_t st, int key_perm);

static thread_local int g_launches = 0;

// ------------------------------------------------------------ tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(f);
  });
  return fn;
}

static CUtensorMapSwizzle swizzle_for(int row_bytes) {
  return row_bytes >= 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                          : (row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
}

// 3-D map over [mats][rows][inner] elements; box = [1][128][box_inner]
// Encoded tensor maps are cached (small direct-mapped table keyed by every encode argument
// and the device): repeated calls on the same buffers -- the serving / benchmark loop -- skip
// the driver encode (5 per forward).
struct MapKey {
  const void* base;
  int dev, dt, elem_bytes, box_inner;
  int64_t inner, rows, mats;
  bool operator==(const MapKey& o) const {
    return base == o.base && dev == o.dev && dt == o.dt && elem_bytes == o.elem_bytes && box_inner == o.box_inner &&
           inner == o.inner && rows == o.rows && mats == o.mats;
  }
};
struct MapSlot {
  MapKey key;
  CUtensorMap map;
  bool valid;
};
static MapSlot g_map_cache[64];
static std::mutex g_map_mutex;

static int make_map_uncached(CUtensorMap* m, const void* base, CUtensorMapDataType dt, int elem_bytes, int64_t inner,
                             int64_t rows, int64_t mats, int box_inner);

static int make_map(CUtensorMap* m, const void* base, CUtensorMapDataType dt, int elem_bytes, int64_t inner,
                    int64_t rows, int64_t mats, int box_inner) {
  int dev = 0;
  cudaGetDevice(&dev);
  const MapKey key{base, dev, static_cast<int>(dt), elem_bytes, box_inner, inner, rows, mats};
  const size_t h = (reinterpret_cast<uintptr_t>(base) >> 8) ^ (static_cast<size_t>(inner) * 31u) ^
                   (static_cast<size_t>(rows) * 131u) ^ (static_cast<size_t>(mats) * 1031u) ^ static_cast<size_t>(box_inner);
  MapSlot& slot = g_map_cache[h % 64];
  {
    std::lock_guard<std::mutex> lk(g_map_mutex);
    if (slot.valid && slot.key == key) {
      *m = slot.map;
      return 0;
    }
  }
  if (int rc = make_map_uncached(m, base, dt, elem_bytes, inner, rows, mats, box_inner)) return rc;
  std::lock_guard<std::mutex> lk(g_map_mutex);
  slot.key = key;
  slot.map = *m;
  slot.valid = true;
  return 0;
}

static int make_map_uncached(CUtensorMap* m, const void* base, CUtensorMapDataType dt, int elem_bytes, int64_t inner,
                             int64_t rows, int64_t mats, int box_inner) {
  EncodeTiledFn fn = encode_fn();
  DMA_CHECK_ARG(fn != nullptr, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(mats)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(inner * elem_bytes), static_cast<cuuint64_t>(inner * rows * elem_bytes)};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(box_inner), 128u, 1u};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, dt, 3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle_for(box_inner * elem_bytes), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): inner=%lld rows=%lld mats=%lld box=%d", (int)r, (long long)inner,
              (long long)rows, (long long)mats, box_inner);
    return DMA_EINVAL;
  }
  return 0;
}

// DMA_SINGLE_STREAM=1 selects the one-stream kernel for the MXFP8 PV path too (A/B comparisons)
static bool force_single_stream() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DMA_SINGLE_STREAM");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// ------------------------------------------------------------ workspace layout
struct Layout {
  int64_t mq, mk, lq_pad, lk_pad, ch_hi, ch_lo;
  bool low_fp4, pv_bf16, v_convert, tensor_gran, pp;  // pp: ping-pong kernel (permuted, padded K operand)
  bool deq;        // bf16-operand route (BLOCK granularity or a None format): QK on dequantized bf16 copies
  bool quant_any;  // deq route needs quantize_dual (not both formats None)
  // deq route: quantize_dual outputs in the reference layout, per Q (0) / K (1)
  size_t r_pl[2], r_sl[2], r_hc[2], r_sh[2], r_qs[2];
  // byte offsets
  size_t q_hi, q_lo, k_hi, k_lo, v_codes, v_bf16;  // large buffers
  size_t small_begin, sf_q_hi, sf_q_lo, sf_k_hi, sf_k_lo, sf_v, qs_q, qs_k, ticket, fuse_flags, small_end;
  int kv_split;    // KV splits per pair (ping-pong kernel, small problems; 1 = off)
  size_t kv_part;  // split partials (kv_split > 1)
  size_t absmax_q, absmax_k, total;
};

static size_t up256(size_t x) { return (x + 255) & ~size_t(255); }

int num_sms();

// KV splits (attn_pp.cuh PPParams): with fewer head pairs x query tiles than SMs the
// persistent kernel leaves SMs idle and the longest causal row walks its whole plan alone
// (c1: 8 work items, the last one 8 key tiles).  Splitting each pair's plan into ns
// ranges of >= 2 tiles fills the GPU; the splits are merged in the kernel.
// dma_attention_set_kv_split / DMA_KV_SPLIT: -1 auto (default), 0 or 1 off, n >= 2 force n.
static std::atomic<int> g_kvsplit{-2};
static int kv_split_mode() {
  int v = g_kvsplit.load(std::memory_order_relaxed);
  if (v == -2) {
    const char* e = getenv("DMA_KV_SPLIT");
    v = (e && e[0]) ? atoi(e) : -1;
    if (v < -1) v = -1;
    g_kvsplit.store(v, std::memory_order_relaxed);
  }
  return v;
}
static constexpr int kMaxKvSplit = 16;

static int kv_split_for(const DmaAttnArgs* a, int64_t mq, int64_t lq_pad) {
  const int mode = a->kv_split > 0 ? (a->kv_split == 1 ? 1 : a->kv_split) : kv_split_mode();
  if (mode == 0 || mode == 1 || a->len_q <= 0 || a->len_k <= 0) return 1;
  const int64_t n_qt = lq_pad / 128, ppq = (mq + 1) / 2, pairs = ppq * n_qt;
  const int sms = num_sms();
  if (mode < 0 && pairs > sms) return 1;  // the dynamic scheduler balances the work items
  int64_t maxn = 0, total = 0;  // longest plan, pair steps over all pairs
  for (int64_t qt = 0; qt < n_qt && qt < 4096; ++qt) {
    Plan pl;
    pl.init(qt, a->len_q, a->len_k, 128, 128, a->diag_window, a->sink_window, a->causal != 0);
    maxn = pl.n > maxn ? pl.n : maxn;
    total += pl.n;
  }
  total *= ppq;
  if (maxn < 2) return 1;
  if (mode >= 2) {
    const int64_t n = mode < maxn ? mode : maxn;
    return static_cast<int>(n < kMaxKvSplit ? n : kMaxKvSplit);
  }
  // cost in pair steps (~1.6 us each on B200): the longest item or the average load per SM,
  // plus, when split, the merge launch (~1.5 steps) and the partial rows written by the
  // attention kernel and read back by the merge (~2.5 MB per us, fitted).  Measured on B200
  // (tools/ks_sweep.py): c1 14.5 -> 11.2 us, B1 H2 N4096 56.6 -> 30.0 us, B1 H4 N8192 108 -> 81 us.
  const double step_us = 1.6, mb_per_us = 2.5;
  auto cost = [&](int64_t n) {
    const double longest = static_cast<double>((maxn + n - 1) / n);
    const double avg = static_cast<double>(total) / sms;
    double c = longest > avg ? longest : avg;
    if (n > 1) {
      const double part_mb = static_cast<double>(mq) * n_qt * n * 128.0 * (a->v_dim + 4) * 4.0 * 2.0 / 1e6;
      c += 1.5 + part_mb / mb_per_us / step_us;
    }
    return c;
  };
  int64_t best = 1;
  double best_c = cost(1);
  for (int64_t n = 2; n <= maxn && n <= kMaxKvSplit; ++n) {
    const double c = cost(n);
    if (c < 0.9 * best_c) {  // a split must win clearly
      best = n;
      best_c = c;
    }
  }
  return static_cast<int>(best);
}

static Layout plan_layout(const DmaAttnArgs* a) {
  Layout L{};
  L.mq = a->batch * a->heads;
  L.mk = a->batch * a->kv_heads;
  L.lq_pad = ceil_div(a->len_q, 128) * 128;
  L.lk_pad = ceil_div(a->len_k, 128) * 128;
  L.low_fp4 = (a->low_format == DMA_FMT_NVFP4 || a->low_format == DMA_FMT_MXFP4);
  L.pv_bf16 = a->pv_mode == DMA_PV_BF16;
  L.v_convert = L.pv_bf16 && a->in_dtype != DMA_DT_BF16;
  L.tensor_gran = a->granularity == DMA_GRAN_TENSOR;
  L.deq = a->granularity == DMA_GRAN_BLOCK || a->low_format == DMA_FMT_NONE || a->high_format == DMA_FMT_NONE;
  L.quant_any = !(a->low_format == DMA_FMT_NONE && a->high_format == DMA_FMT_NONE);
  if (L.deq) L.low_fp4 = true;  // both operand copies exist (bf16)
  L.pp = !L.pv_bf16 && !force_single_stream() && !L.deq && a->tile_m == 128 && a->tile_n == 128;
  const int64_t k_rows = L.pp ? L.lk_pad : a->len_k;
  const int64_t D = a->head_dim, DV = a->v_dim;
  L.ch_hi = (D / 32 + 3) / 4;
  L.ch_lo = a->low_format == DMA_FMT_NVFP4 ? (D / 16 + 3) / 4 : (D / 32 + 3) / 4;
  if (L.deq) L.ch_hi = L.ch_lo = 0;  // no scale-factor atoms on the bf16-operand route
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = up256(off + bytes);
    return o;
  };
  const int64_t obytes_hi = L.deq ? 2 * D : D, obytes_lo = L.deq ? 2 * D : D / 2;  // operand bytes per row
  L.q_hi = take(L.mq * a->len_q * obytes_hi);
  L.q_lo = L.low_fp4 ? take(L.mq * a->len_q * obytes_lo) : 0;
  L.k_hi = take(L.mk * k_rows * obytes_hi);
  L.k_lo = L.low_fp4 ? take(L.mk * k_rows * obytes_lo) : 0;
  for (int w = 0; w < 2; ++w) {
    const int64_t n = (w == 0 ? L.mq * a->len_q : L.mk * a->len_k);  // rows of Q / K
    const bool on = L.deq && L.quant_any;
    const int64_t nq = a->granularity == DMA_GRAN_BLOCK ? n * (D / 32) : (a->granularity == DMA_GRAN_TOKEN ? n : (w == 0 ? L.mq : L.mk));
    L.r_pl[w] = on ? take(n * D / 2) : 0;
    L.r_sl[w] = on ? take(n * (D / 16)) : 0;
    L.r_hc[w] = on ? take(n * D) : 0;
    L.r_sh[w] = on ? take(n * (D / 32)) : 0;
    L.r_qs[w] = on ? take(nq * 8) : 0;
  }
  L.v_codes = L.pv_bf16 ? 0 : take(L.mk * L.lk_pad * DV);
  L.v_bf16 = L.v_convert ? take(L.mk * a->len_k * DV * 2) : 0;
  L.small_begin = off;
  L.sf_q_hi = take(L.mq * (L.lq_pad / 128) * L.ch_hi * 512);
  L.sf_q_lo = L.low_fp4 ? take(L.mq * (L.lq_pad / 128) * L.ch_lo * 512) : 0;
  L.sf_k_hi = take(L.mk * (L.lk_pad / 128) * L.ch_hi * 512);
  L.sf_k_lo = L.low_fp4 ? take(L.mk * (L.lk_pad / 128) * L.ch_lo * 512) : 0;
  L.sf_v = L.pv_bf16 ? 0 : take(L.mk * (L.lk_pad / 128) * ((DV + 127) / 128) * 512);
  L.qs_q = take(L.mq * L.lq_pad * 4);
  L.qs_k = take(L.pp ? L.mk * (L.lk_pad / 128) * kSqkTile * 4 : L.mk * L.lk_pad * 4);
  L.ticket = take(64);  // dynamic pair scheduler ticket (zeroed with the small region; self-resetting)
  // fused forward: per 128-row tile ready flags (Q, K, V) + the quantizer work counters
  L.fuse_flags = L.pp ? take((L.mq * (L.lq_pad / 128) + 2 * L.mk * (L.lk_pad / 128)) * 4 + 64) : 0;
  L.kv_split = L.pp ? kv_split_for(a, L.mq, L.lq_pad) : 1;
  L.small_end = off;
  L.kv_part = L.kv_split > 1 ? take(L.mq * (L.lq_pad / 128) * L.kv_split * 128 * (DV + 4) * 4) : 0;
  L.absmax_q = L.tensor_gran ? take(L.mq * 8) : 0;
  L.absmax_k = L.tensor_gran ? take(L.mk * 8) : 0;
  L.total = off + 256;  // base alignment slack
  return L;
}

static int validate(const DmaAttnArgs* a) {
  DMA_CHECK_ARG(a != nullptr, "null args");
  DMA_CHECK_ARG(a->batch >= 1 && a->heads >= 1 && a->kv_heads >= 1 && a->heads % a->kv_heads == 0,
                "bad batch/heads/kv_heads (%lld/%lld/%lld)", (long long)a->batch, (long long)a->heads,
                (long long)a->kv_heads);
  DMA_CHECK_ARG(a->len_q >= 0 && a->len_k >= 0, "negative sequence length");
  DMA_CHECK_ARG(!a->causal || a->len_q == a->len_k,
                "causal attention requires equal sequence lengths, got %lld and %lld", (long long)a->len_q,
                (long long)a->len_k);
  DMA_CHECK_ARG(a->tile_m >= 1 && a->tile_n >= 1, "tile sizes must be >= 1");
  DMA_CHECK_ARG(a->diag_window >= 0 && a->sink_window >= 0, "window sizes must be >= 0");
  DMA_CHECK_ARG(a->diag_window % a->tile_n == 0 && a->sink_window % a->tile_n == 0,
                "diag_window and sink_window must be multiples of tile_n");
  DMA_CHECK_ARG(a->in_dtype >= DMA_DT_F64 && a->in_dtype <= DMA_DT_BF16, "bad in_dtype");
  DMA_CHECK_ARG(a->out_dtype == DMA_DT_F32 || a->out_dtype == DMA_DT_BF16, "out_dtype must be f32 or bf16");
  return 0;
}

int attention_supported(const DmaAttnArgs* a) {
  if (int rc = validate(a)) return rc;
  auto unsup = [](const char* why) {
    set_error("%s", why);
    return DMA_EUNSUPPORTED;
  };
  if ((a->tile_m != 64 && a->tile_m != 128) || (a->tile_n != 64 && a->tile_n != 128))
    return unsup("plan tiles must be 64 or 128 (tile_m, tile_n); the sm_100a kernels walk 128 x 128 tiles");
  if (a->head_dim != 64 && a->head_dim != 128) return unsup("head_dim must be 64 or 128");
  if (a->v_dim != 64 && a->v_dim != 128) return unsup("v_dim must be 64 or 128");
  if (a->high_format != DMA_FMT_MXFP8_E4M3 && a->high_format != DMA_FMT_MXFP8_E5M2 && a->high_format != DMA_FMT_NONE)
    return unsup("high_format must be an MXFP8 format or None");
  if (a->granularity < 0 || a->granularity > 2) return unsup("unknown granularity");
  if (a->pv_mode != DMA_PV_MXFP8 && a->pv_mode != DMA_PV_BF16) return unsup("bad pv_mode");
  if (a->len_q > (int64_t(1) << 30) || a->len_k > (int64_t(1) << 30)) return unsup("sequence too long");
  return 0;
}

__global__ void to_bf16_kernel(const void* src, int dt, int64_t n, __nv_bfloat16* dst) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float v = dt == DMA_DT_F64 ? static_cast<float>(static_cast<const double*>(src)[i])
                               : static_cast<const float*>(src)[i];
    dst[i] = __float2bfloat16_rn(v);
  }
}


// bf16-operand route, phase 1b: the operands the reference's _prepare_operands builds
// (attention.py:247-279), rounded to bf16: mode 0 = identity (x * c for Q, attention.py:
// 256-258), 1 = dequantize_high (quantize.py:232-237), 2 = dequantize_low (:215-229),
// 3 = the low path reuses the high one (8-bit low format, :270-271).
__global__ void deq_bf16_kernel(int lo_mode, int hi_mode, int nv, int e5, int gran, int64_t n_mat, int64_t rows,
                                int cols, const uint8_t* pl, const uint8_t* sl, const uint8_t* hc, const uint8_t* sh,
                                const double* qs, const void* x, int x_dt, int is_query, double c,
                                __nv_bfloat16* out_hi, __nv_bfloat16* out_lo) {
  const int64_t n = n_mat * rows * cols;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t rr = i / cols;  // mat * rows + row
    const int col = static_cast<int>(i % cols);
    double ident;
    if (x_dt == DMA_DT_BF16) ident = __bfloat162float(static_cast<const __nv_bfloat16*>(x)[i]);
    else if (x_dt == DMA_DT_F32) ident = static_cast<const float*>(x)[i];
    else ident = static_cast<const double*>(x)[i];
    if (is_query) ident = __dmul_rn(ident, c);
    double s_q = 1.0;
    if (hi_mode == 1 || lo_mode == 2 || lo_mode == 3) {
      if (gran == DMA_GRAN_TOKEN) s_q = qs[rr];
      else if (gran == DMA_GRAN_BLOCK) s_q = qs[rr * (cols / 32) + col / 32];
      else s_q = qs[rr / rows];
    }
    double hi = ident;
    if (hi_mode == 1) {
      const uint32_t cd = hc[i];
      double e;
      if (e5) {
        const uint32_t ex = (cd >> 2) & 0x1F, m = cd & 3;
        e = ex ? (4.0 + m) * pow2(static_cast<int>(ex) - 17) : m * pow2(-16);
        if (cd & 0x80) e = -e;
      } else {
        e = decode_e4m3(cd);
      }
      hi = e * pow2(static_cast<int>(sh[rr * (cols / 32) + col / 32]) - 127) * s_q;
    }
    double lo = ident;
    if (lo_mode == 3) {
      lo = hi;
    } else if (lo_mode == 2) {
      const uint32_t byte = pl[rr * (cols / 2) + col / 2];
      const uint32_t code = (col & 1) ? (byte >> 4) : (byte & 0xF);
      const double mags[8] = {0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0};
      double e = mags[code & 7];
      if (code & 8) e = -e;
      lo = nv ? e * decode_e4m3(sl[rr * (cols / 16) + col / 16]) * s_q
              : e * pow2(static_cast<int>(sl[rr * (cols / 32) + col / 32]) - 127);
    }
    out_hi[i] = __float2bfloat16_rn(static_cast<float>(hi));
    out_lo[i] = __float2bfloat16_rn(static_cast<float>(lo));
  }
}

static int quantize_deq(const DmaAttnArgs* a, const Layout& L, uint8_t* ws, cudaStream_t st) {
  const int64_t D = a->head_dim;
  const bool low_e2m1 = a->low_format == DMA_FMT_NVFP4 || a->low_format == DMA_FMT_MXFP4;
  const int qlow = low_e2m1 ? a->low_format : DMA_FMT_NVFP4;
  const int qhigh = a->high_format != DMA_FMT_NONE ? a->high_format : DMA_FMT_MXFP8_E4M3;
  const int hi_mode = (a->high_format == DMA_FMT_NONE || !L.quant_any) ? 0 : 1;
  const int lo_mode = (a->low_format == DMA_FMT_NONE || !L.quant_any) ? 0 : (low_e2m1 ? 2 : 3);
  for (int w = 0; w < 2; ++w) {
    const bool isq = w == 0;
    const int64_t rows = isq ? a->len_q : a->len_k, nmat = isq ? L.mq : L.mk;
    if (rows == 0) continue;
    if (L.quant_any) {
      DmaQuantArgs q{};
      q.x = isq ? a->q : a->k;
      q.x_dtype = a->in_dtype;
      q.is_query = isq;
      q.n_mat = nmat;
      q.rows = rows;
      q.cols = D;
      q.mat_stride = rows * D;
      q.row_stride = D;
      q.prescale = a->prescale;
      q.low_format = qlow;
      q.high_format = qhigh;
      q.granularity = a->granularity;
      q.packed_low = ws + L.r_pl[w];
      q.scales_low = ws + L.r_sl[w];
      q.high_codes = ws + L.r_hc[w];
      q.scales_high = ws + L.r_sh[w];
      q.quant_scale = reinterpret_cast<double*>(ws + L.r_qs[w]);
      q.workspace = L.tensor_gran ? ws + (isq ? L.absmax_q : L.absmax_k) : nullptr;
      q.workspace_bytes = L.tensor_gran ? nmat * 8 : 0;
      q.nonfinite = a->nonfinite;
      if (int rc = quantize_impl(&q, nullptr, nullptr, nullptr, 0, st, 0)) return rc;
      g_launches += L.tensor_gran ? 2 : 1;
    }
    const int64_t n = nmat * rows * D;
    int64_t g = (n + 255) / 256;
    g = g > 148 * 16 ? 148 * 16 : g;
    deq_bf16_kernel<<<static_cast<unsigned>(g), 256, 0, st>>>(
        lo_mode, hi_mode, qlow == DMA_FMT_NVFP4, qhigh == DMA_FMT_MXFP8_E5M2, a->granularity, nmat, rows,
        static_cast<int>(D), ws + L.r_pl[w], ws + L.r_sl[w], ws + L.r_hc[w], ws + L.r_sh[w],
        reinterpret_cast<const double*>(ws + L.r_qs[w]), isq ? a->q : a->k, a->in_dtype, isq, a->prescale,
        reinterpret_cast<__nv_bfloat16*>(ws + (isq ? L.q_hi : L.k_hi)),
        reinterpret_cast<__nv_bfloat16*>(ws + (isq ? L.q_lo : L.k_lo)));
    DMA_LAUNCH_CHECK();
    ++g_launches;
  }
  return 0;
}

// Phase-2 kernel of the block-scaled MXFP8-PV path: DMA_ATTN_KERNEL=pp (ping-pong,
// attn_pp.cuh), ws (max / exp warp specialisation, attn_ws.cuh), sk (split-KV experiment,
// attn_sk.cuh; measured slower).
enum { kKernPP = 0, kKernSK = 1, kKernWS = 2 };
static int attn_kernel_choice() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DMA_ATTN_KERNEL");
    v = kKernPP;
    if (e && e[0] == 's' && e[1] == 'k') v = kKernSK;
    if (e && e[0] == 'w' && e[1] == 's') v = kKernWS;
  }
  return v;
}
// K/V megabytes per head-major group of head pairs (DMA_GROUP_MB; 0 = one pair per group)
static double group_kv_mb() {
  static double v = -1.0;
  if (v < 0.0) {
    const char* e = getenv("DMA_GROUP_MB");
    v = (e && e[0]) ? atof(e) : 48.0;
  }
  return v;
}

static bool use_sk_kernel() { return attn_kernel_choice() == kKernSK; }
static bool use_ws_kernel() { return attn_kernel_choice() == kKernWS; }
// The fused forward (phase 1 inside the ping-pong kernel, attn_pp.cuh FUSE) covers the
// north-star path: bf16 inputs, TOKEN granularity, MX formats, block-scaled MXFP8 PV,
// 128-tiles.  Its output is bit-identical to the two-phase path, but it is slower (DESIGN.md
// §4.6: two quantizer warps per SM are latency-bound), so it is opt-in:
// dma_attention_set_fused(1) or DMA_FUSE=1.
static std::atomic<int> g_fuse{-1};
static bool fuse_enabled() {
  int v = g_fuse.load(std::memory_order_relaxed);
  if (v < 0) {
    const char* e = getenv("DMA_FUSE");
    v = (e && e[0] == '1') ? 1 : 0;
    g_fuse.store(v, std::memory_order_relaxed);
  }
  return v == 1;
}

static bool fused_eligible(const DmaAttnArgs* a, const Layout& L) {
  return fuse_enabled() && L.pp && !use_sk_kernel() && !use_ws_kernel() && a->in_dtype == DMA_DT_BF16 &&
         a->granularity == DMA_GRAN_TOKEN && a->len_q > 0 && a->len_k > 0;
}

int attention_quantize(const DmaAttnArgs* a, const Layout& L, uint8_t* ws, cudaStream_t st) {
  const int64_t D = a->head_dim, DV = a->v_dim;
  const bool nv = a->low_format == DMA_FMT_NVFP4;
  // padded SF atoms / S_q entries must be finite: zero the small region once per call
  DMA_CUDA_TRY(cudaMemsetAsync(ws + L.small_begin, 0, L.small_end - L.small_begin, st));  // (a memset, not a kernel)
  if (a->nonfinite) DMA_CUDA_TRY(cudaMemsetAsync(a->nonfinite, 0, sizeof(uint32_t), st));
  // small problems (launch-bound: c1 0.047 -> 0.034 ms): Q, K and V in one launch
  // (phase1_bf16_kernel, the same device code as the three kernels); large ones keep three
  // full-GPU launches (merged, c3's phase 1 measured 0.75 vs 0.61 ms)
  const double p1_elems = static_cast<double>(L.mq) * a->len_q * D + static_cast<double>(L.mk) * a->len_k * (D + DV);
  if (a->in_dtype == DMA_DT_BF16 && a->granularity == DMA_GRAN_TOKEN && L.pp && !L.deq && !use_sk_kernel() &&
      !use_ws_kernel() && !L.pv_bf16 && a->len_q > 0 && a->len_k > 0 && D % 32 == 0 && D / 16 <= 32 &&
      p1_elems <= 8.0 * 1024 * 1024) {
    P1Job jq{}, jk{};
    for (int w = 0; w < 2; ++w) {
      P1Job& j = w == 0 ? jq : jk;
      j.x = static_cast<const __nv_bfloat16*>(w == 0 ? a->q : a->k);
      j.n_mat = w == 0 ? L.mq : L.mk;
      j.rows = w == 0 ? a->len_q : a->len_k;
      j.is_query = w == 0;
      QuantOut& o = j.out;
      o.packed_low = L.low_fp4 ? ws + (w == 0 ? L.q_lo : L.k_lo) : nullptr;
      o.high_codes = ws + (w == 0 ? L.q_hi : L.k_hi);
      o.sf_low_op = L.low_fp4 ? ws + (w == 0 ? L.sf_q_lo : L.sf_k_lo) : nullptr;
      o.sf_high_op = ws + (w == 0 ? L.sf_q_hi : L.sf_k_hi);
      o.qs_f32 = reinterpret_cast<float*>(ws + (w == 0 ? L.qs_q : L.qs_k));
      o.nonfinite = a->nonfinite;
      o.rows_pad = w == 0 ? L.lq_pad : L.lk_pad;
      o.key_perm = w == 0 ? 0 : 1;
    }
    // CTAs in proportion to the work (V ~ 1/3 of a Q/K element), ~8 per SM in total, each part
    // at least one CTA and at most one per item
    const int64_t rpb = 256 / (D / 16);
    const int64_t iq = L.mq * ((a->len_q + rpb - 1) / rpb), ik = L.mk * ((a->len_k + rpb - 1) / rpb);
    const int64_t kbpc = 256 / (DV / 4), iv = L.mk * ((L.lk_pad / 32 + kbpc - 1) / kbpc);
    const double wq = static_cast<double>(L.mq) * a->len_q, wk = static_cast<double>(L.mk) * a->len_k,
                 wv = static_cast<double>(L.mk) * a->len_k * DV / D / 3.0, wt = wq + wk + wv;
    const int total = num_sms() * 8;
    auto share = [&](double w, int64_t cap) {
      int64_t n = static_cast<int64_t>(total * w / wt + 0.5);
      n = n < 1 ? 1 : n;
      return static_cast<int>(n > cap ? cap : n);
    };
    const int nq = share(wq, iq), nk = share(wk, ik), nv = share(wv, iv);
    const bool nvf = L.low_fp4 ? a->low_format == DMA_FMT_NVFP4 : true, e5 = a->high_format == DMA_FMT_MXFP8_E5M2;
    auto kern = nvf ? (e5 ? phase1_bf16_kernel<true, true> : phase1_bf16_kernel<true, false>)
                    : (e5 ? phase1_bf16_kernel<false, true> : phase1_bf16_kernel<false, false>);
    kern<<<static_cast<unsigned>(nq + nk + nv), 256, 0, st>>>(jq, jk, static_cast<int>(D), a->prescale, nq, nk,
                                                              static_cast<const __nv_bfloat16*>(a->v), a->len_k,
                                                              static_cast<int>(DV), L.lk_pad, L.mk, ws + L.v_codes,
                                                              ws + L.sf_v);
    DMA_LAUNCH_CHECK();
    ++g_launches;
    return 0;
  }
  for (int which = 0; which < 2 && !L.deq; ++which) {
    const bool isq = which == 0;
    DmaQuantArgs q{};
    q.x = isq ? a->q : a->k;
    q.x_dtype = a->in_dtype;
    q.is_query = isq;
    q.n_mat = isq ? L.mq : L.mk;
    q.rows = isq ? a->len_q : a->len_k;
    q.cols = D;
    q.mat_stride = q.rows * D;
    q.row_stride = D;
    q.prescale = a->prescale;
    q.low_format = L.low_fp4 ? a->low_format : DMA_FMT_NVFP4;
    q.high_format = a->high_format;
    q.granularity = a->granularity;
    q.packed_low = L.low_fp4 ? ws + (isq ? L.q_lo : L.k_lo) : nullptr;
    q.high_codes = ws + (isq ? L.q_hi : L.k_hi);
    q.workspace = L.tensor_gran ? ws + (isq ? L.absmax_q : L.absmax_k) : nullptr;
    q.workspace_bytes = L.tensor_gran ? q.n_mat * 8 : 0;
    q.nonfinite = a->nonfinite;
    uint8_t* sfl = L.low_fp4 ? ws + (isq ? L.sf_q_lo : L.sf_k_lo) : nullptr;
    uint8_t* sfh = ws + (isq ? L.sf_q_hi : L.sf_k_hi);
    float* qs = reinterpret_cast<float*>(ws + (isq ? L.qs_q : L.qs_k));
    if (q.rows == 0) continue;
    const int kmode = (!isq && L.pp) ? ((use_sk_kernel() || use_ws_kernel()) ? 2 : 1) : 0;  // K operand layout
    // PDL: K's quantizer may start while Q's drains (independent outputs; the kernels chain
    // their completion with pdl_wait, the attention kernel waits for the last)
    g_pdl_next = !isq && pdl_enabled() && !L.tensor_gran;  // TENSOR: K reads its absmax kernel's result
    const int qrc = quantize_impl(&q, sfl, sfh, qs, isq ? L.lq_pad : L.lk_pad, st, kmode);
    g_pdl_next = false;
    if (qrc) return qrc;
    g_launches += L.tensor_gran ? 2 : 1;
    if (kmode == 2 && use_sk_kernel()) {
      const int64_t nt = L.mk * (L.lk_pad / 128);
      sqk_tile_stats_kernel<<<static_cast<unsigned>((nt + 7) / 8), 256, 0, st>>>(qs, nt, L.lk_pad / 128, a->len_k);
      DMA_LAUNCH_CHECK();
      ++g_launches;
    }
  }
  (void)nv;
  if (L.deq)
    if (int rc = quantize_deq(a, L, ws, st)) return rc;
  if (a->len_k > 0) {
    if (!L.pv_bf16) {
      // dv in {64, 128} (attention_supported): 256 threads = 256 / (dv/2) key blocks of 32
      const int kb_per_cta = 256 / static_cast<int>(DV / 2);
      dim3 grid(static_cast<unsigned>((L.lk_pad / 32 + kb_per_cta - 1) / kb_per_cta), static_cast<unsigned>(L.mk));
      cudaStream_t s = st;
      if (a->in_dtype == DMA_DT_BF16) {
        const int kb4 = 256 / static_cast<int>(DV / 4);
        dim3 grid4(static_cast<unsigned>((L.lk_pad / 32 + kb4 - 1) / kb4), static_cast<unsigned>(L.mk));
        DMA_CUDA_TRY(launch_kernel(pdl_enabled(), quant_v4_bf16_kernel, grid4, dim3(256), 0, s,
                                   static_cast<const __nv_bfloat16*>(a->v), a->len_k, static_cast<int>(DV), L.lk_pad,
                                   ws + L.v_codes, ws + L.sf_v));
      }
      else if (a->in_dtype == DMA_DT_F32)
        quant_v2_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(a->v), a->len_k, static_cast<int>(DV),
                                                    L.lk_pad, ws + L.v_codes, ws + L.sf_v);
      else
        quant_v2_kernel<double><<<grid, 256, 0, s>>>(static_cast<const double*>(a->v), a->len_k,
                                                     static_cast<int>(DV), L.lk_pad, ws + L.v_codes, ws + L.sf_v);
      DMA_LAUNCH_CHECK();
      ++g_launches;
    } else if (L.v_convert) {
      const int64_t n = L.mk * a->len_k * DV;
      int64_t g = (n + 255) / 256;
      g = g > 4096 ? 4096 : g;
      to_bf16_kernel<<<static_cast<unsigned>(g), 256, 0, st>>>(a->v, a->in_dtype, n,
                                                               reinterpret_cast<__nv_bfloat16*>(ws + L.v_bf16));
      DMA_LAUNCH_CHECK();
      ++g_launches;
    }
  }
  return 0;
}

int num_sms() {
  // per device (SM counts are cached; the attribute query is a driver call)
  static std::atomic<int> cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (n <= 0) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

int attention_core(const DmaAttnArgs* a, const Layout& L, uint8_t* ws, cudaStream_t st, bool fuse = false) {
  const int64_t D = a->head_dim, DV = a->v_dim;
  AttnParams p;
  std::memset(&p, 0, sizeof(p));
  const int64_t lq_rows = a->len_q > 0 ? a->len_q : 1, lk_rows = a->len_k > 0 ? a->len_k : 1;
  const int64_t k_rows = L.pp ? L.lk_pad : lk_rows;
  if (L.deq) {
    // bf16 operand copies, 64-column (128-byte, 128B-swizzled) boxes
    const auto bf = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    if (int rc = make_map(&p.tm_q_hi, ws + L.q_hi, bf, 2, D, lq_rows, L.mq, 64)) return rc;
    if (int rc = make_map(&p.tm_q_lo, ws + L.q_lo, bf, 2, D, lq_rows, L.mq, 64)) return rc;
    if (int rc = make_map(&p.tm_k_hi, ws + L.k_hi, bf, 2, D, lk_rows, L.mk, 64)) return rc;
    if (int rc = make_map(&p.tm_k_lo, ws + L.k_lo, bf, 2, D, lk_rows, L.mk, 64)) return rc;
  } else {
  if (int rc = make_map(&p.tm_q_hi, ws + L.q_hi, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, D, lq_rows, L.mq, (int)D)) return rc;
  if (int rc = make_map(&p.tm_k_hi, ws + L.k_hi, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, D, k_rows, L.mk, (int)D)) return rc;
  if (L.low_fp4) {
    if (int rc = make_map(&p.tm_q_lo, ws + L.q_lo, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, D / 2, lq_rows, L.mq, (int)D / 2)) return rc;
    if (int rc = make_map(&p.tm_k_lo, ws + L.k_lo, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, D / 2, k_rows, L.mk, (int)D / 2)) return rc;
  }
  }
  if (L.pv_bf16) {
    const void* vsrc = L.v_convert ? static_cast<const void*>(ws + L.v_bf16) : a->v;
    DMA_CHECK_ARG((reinterpret_cast<uintptr_t>(vsrc) & 15) == 0, "V must be 16-byte aligned");
    if (int rc = make_map(&p.tm_v, vsrc, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, DV, lk_rows, L.mk, 64)) return rc;
  } else {
    if (int rc = make_map(&p.tm_v, ws + L.v_codes, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, DV, L.lk_pad, L.mk, (int)DV)) return rc;
  }
  p.sf_q_hi = ws + L.sf_q_hi;
  p.sf_q_lo = L.low_fp4 ? ws + L.sf_q_lo : nullptr;
  p.sf_k_hi = ws + L.sf_k_hi;
  p.sf_k_lo = L.low_fp4 ? ws + L.sf_k_lo : nullptr;
  p.sf_v = L.pv_bf16 ? nullptr : ws + L.sf_v;
  p.qs_q = reinterpret_cast<const float*>(ws + L.qs_q);
  p.qs_k = reinterpret_cast<const float*>(ws + L.qs_k);
  p.o = a->o;
  p.out_bf16 = a->out_dtype == DMA_DT_BF16;
  p.heads = static_cast<int>(a->heads);
  p.kv_heads = static_cast<int>(a->kv_heads);
  p.group = static_cast<int>(a->heads / a->kv_heads);
  p.lq = static_cast<int>(a->len_q);
  p.lk = static_cast<int>(a->len_k);
  p.lq_pad = static_cast<int>(L.lq_pad);
  p.lk_pad = static_cast<int>(L.lk_pad);
  p.n_qt = static_cast<int>(L.lq_pad / 128);
  p.diag_window = a->diag_window;
  p.sink_window = a->sink_window;
  p.causal = a->causal;
  p.ch_hi = static_cast<int>(L.ch_hi);
  p.ch_lo = static_cast<int>(L.ch_lo);
  p.hfmt = a->high_format == DMA_FMT_MXFP8_E5M2 ? 1 : 0;
  p.tile_m = a->tile_m;
  p.tile_n = a->tile_n;
  const int64_t items = L.mq * p.n_qt;
  if (items == 0) return 0;
  DMA_CHECK_ARG(items < (int64_t(1) << 31), "too many work items");
  p.n_bh = static_cast<int>(L.mq);
  p.n_items = static_cast<int>(items);
  const int low = L.deq ? kLowBF16
                        : (a->low_format == DMA_FMT_NVFP4 ? kLowNV : (a->low_format == DMA_FMT_MXFP4 ? kLowMX4 : kLowHigh));
  if (L.pp && use_ws_kernel()) {
    // max / exp warp-specialised kernel: one query tile per work item, S double-buffered
    SKParams q{};
    q.n_items = static_cast<int>(items);
    const double kv_bytes = static_cast<double>(L.mk) * static_cast<double>(L.lk_pad) * (2.6 * static_cast<double>(D));
    q.head_major = kv_bytes > 48.0 * 1024 * 1024;
    q.ticket = reinterpret_cast<unsigned int*>(ws + L.ticket);
    const int rc = run_ws(p, q, static_cast<int>(D), static_cast<int>(DV), low, st);
    if (rc == 0) ++g_launches;
    return rc;
  }
  if (L.pp && use_sk_kernel()) {
    // split-KV kernel (block-scaled MXFP8 PV): one query tile per work item, plan entries
    // alternate between the two softmax warpgroups
    SKParams q{};
    q.n_items = static_cast<int>(items);
    const double kv_bytes = static_cast<double>(L.mk) * static_cast<double>(L.lk_pad) * (2.6 * static_cast<double>(D));
    q.head_major = kv_bytes > 48.0 * 1024 * 1024;
    q.ticket = reinterpret_cast<unsigned int*>(ws + L.ticket);
    const int rc = run_sk(p, q, static_cast<int>(D), static_cast<int>(DV), low, st);
    if (rc == 0) ++g_launches;
    return rc;
  }
  if (L.pp) {
    // ping-pong kernel (block-scaled MXFP8 PV): pairs of heads share one query-tile plan
    PPParams q{};
    q.pairs_per_qt = static_cast<int>((L.mq + 1) / 2);
    q.n_pairs = q.pairs_per_qt * p.n_qt;
    q.n_split = L.kv_split;
    DMA_CHECK_ARG(static_cast<int64_t>(q.n_pairs) * q.n_split < (int64_t(1) << 31), "too many work items");
    q.n_items = q.n_pairs * q.n_split;
    q.part = L.kv_split > 1 ? reinterpret_cast<float*>(ws + L.kv_part) : nullptr;
    const double kv_bytes = static_cast<double>(L.mk) * static_cast<double>(L.lk_pad) * (2.6 * static_cast<double>(D));
    q.head_major = kv_bytes > 48.0 * 1024 * 1024;  // K/V exceed ~L2/2: keep all CTAs on the same heads
    {
      // head pairs per group: as many as keep the group's K/V under ~48 MB (c3: 2, c4: 4, c5: 1)
      const double per_pair = kv_bytes / static_cast<double>(q.pairs_per_qt);
      int gp = static_cast<int>(group_kv_mb() * 1024.0 * 1024.0 / per_pair);
      gp = gp < 1 ? 1 : (gp > q.pairs_per_qt ? q.pairs_per_qt : gp);
      q.group_pairs = gp;
    }
    q.ticket = reinterpret_cast<unsigned int*>(ws + L.ticket);
    int rc;
    if (fuse) {
      // phase 1 inside the kernel (attn_pp.cuh FuseParams): raw bf16 inputs, operand outputs as
      // attention_quantize writes them
      FuseParams fz{};
      fz.q = static_cast<const __nv_bfloat16*>(a->q);
      fz.k = static_cast<const __nv_bfloat16*>(a->k);
      fz.v = static_cast<const __nv_bfloat16*>(a->v);
      for (int w = 0; w < 2; ++w) {
        QuantOut& o = w == 0 ? fz.out_q : fz.out_k;
        o.packed_low = L.low_fp4 ? ws + (w == 0 ? L.q_lo : L.k_lo) : nullptr;
        o.high_codes = ws + (w == 0 ? L.q_hi : L.k_hi);
        o.sf_low_op = L.low_fp4 ? ws + (w == 0 ? L.sf_q_lo : L.sf_k_lo) : nullptr;
        o.sf_high_op = ws + (w == 0 ? L.sf_q_hi : L.sf_k_hi);
        o.qs_f32 = reinterpret_cast<float*>(ws + (w == 0 ? L.qs_q : L.qs_k));
        o.nonfinite = a->nonfinite;
        o.rows_pad = w == 0 ? L.lq_pad : L.lk_pad;
        o.key_perm = w == 0 ? 0 : 1;
      }
      fz.v_codes = ws + L.v_codes;
      fz.sf_v = ws + L.sf_v;
      fz.c = a->prescale;
      fz.flags = reinterpret_cast<unsigned int*>(ws + L.fuse_flags);
      fz.counters = fz.flags + (L.mq * (L.lq_pad / 128) + 2 * L.mk * (L.lk_pad / 128));
      fz.e5 = a->high_format == DMA_FMT_MXFP8_E5M2;
      rc = run_pp_fused(p, q, fz, static_cast<int>(D), static_cast<int>(DV), low, st);
    } else {
      rc = run_pp(p, q, static_cast<int>(D), static_cast<int>(DV), low, st);
    }
    if (rc == 0) ++g_launches;
    if (rc == 0 && q.n_split > 1) {
      // merge the KV splits' partial rows (kv_combine_kernel, PDL: its launch overlaps the tail)
      rc = run_kv_combine(p, q.part, q.n_split, static_cast<int>(DV), st);
      if (rc == 0) ++g_launches;
    }
    return rc;
  }
  const int rc = run_attn(p, static_cast<int>(D), static_cast<int>(DV), low, L.pv_bf16, items, st);
  if (rc == 0) ++g_launches;
  return rc;
}

static uint8_t* ws_base(const DmaAttnArgs* a) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(a->workspace) + 255) & ~uintptr_t(255));
}

}  // namespace dma

using namespace dma;

extern "C" {

// Empty problems (attention.py:282-310 on zero-length inputs): no query rows -> nothing
// to write; no keys (non-causal) -> every row has l = 0 and normalises to 0.
// Returns 1 when the call was handled here.
static int empty_problem(const DmaAttnArgs* a, cudaStream_t st, int* rc) {
  if (a->len_q > 0 && a->len_k > 0) return 0;
  *rc = DMA_OK;
  if (a->len_q > 0) {
    if (!a->o) {
      set_error("null output");
      *rc = DMA_EINVAL;
      return 1;
    }
    const size_t n = static_cast<size_t>(a->batch * a->heads * a->len_q * a->v_dim) *
                     (a->out_dtype == DMA_DT_BF16 ? 2 : 4);
    const cudaError_t e = cudaMemsetAsync(a->o, 0, n, st);
    if (e != cudaSuccess) {
      set_error("cudaMemsetAsync: %s", cudaGetErrorString(e));
      *rc = static_cast<int>(e);
    }
  }
  return 1;
}

size_t dma_attention_workspace_bytes(const DmaAttnArgs* a) {
  if (validate(a)) return 0;
  return plan_layout(a).total;
}

int dma_attention_supported(const DmaAttnArgs* a) { return attention_supported(a); }

int dma_attention_quantize(const DmaAttnArgs* a, void* stream) {
  g_launches = 0;
  if (int rc = attention_supported(a)) return rc;
  if (a->len_q == 0 || a->len_k == 0) return DMA_OK;  // nothing to quantize
  Layout L = plan_layout(a);
  DMA_CHECK_ARG(a->workspace && a->workspace_bytes >= L.total, "workspace too small (%zu < %zu)",
                a->workspace_bytes, L.total);
  return attention_quantize(a, L, ws_base(a), static_cast<cudaStream_t>(stream));
}

int dma_attention_core(const DmaAttnArgs* a, void* stream) {
  if (int rc = attention_supported(a)) return rc;
  if (int rc; empty_problem(a, static_cast<cudaStream_t>(stream), &rc)) return rc;
  Layout L = plan_layout(a);
  DMA_CHECK_ARG(a->workspace && a->workspace_bytes >= L.total, "workspace too small (%zu < %zu)",
                a->workspace_bytes, L.total);
  DMA_CHECK_ARG(a->o != nullptr, "null output");
  return attention_core(a, L, ws_base(a), static_cast<cudaStream_t>(stream));
}

int dma_attention_fwd(const DmaAttnArgs* a, void* stream) {
  g_launches = 0;
  if (int rc = attention_supported(a)) return rc;
  if (int rc; empty_problem(a, static_cast<cudaStream_t>(stream), &rc)) return rc;
  Layout L = plan_layout(a);
  DMA_CHECK_ARG(a->workspace && a->workspace_bytes >= L.total, "workspace too small (%zu < %zu)",
                a->workspace_bytes, L.total);
  DMA_CHECK_ARG(a->q && a->k && a->v && a->o, "null tensor pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (fused_eligible(a, L)) {
    L.kv_split = 1;  // one kernel per call: no KV splits (their merge is a second launch)
    // one kernel: the ping-pong attention with phase 1 in warps 10 / 11 (attn_pp.cuh FUSE)
    uint8_t* ws = ws_base(a);
    DMA_CUDA_TRY(cudaMemsetAsync(ws + L.small_begin, 0, L.small_end - L.small_begin, st));
    if (a->nonfinite) DMA_CUDA_TRY(cudaMemsetAsync(a->nonfinite, 0, sizeof(uint32_t), st));
    return attention_core(a, L, ws, st, true);
  }
  if (int rc = attention_quantize(a, L, ws_base(a), st)) return rc;
  return attention_core(a, L, ws_base(a), st);
}

int dma_last_launch_count(void) { return g_launches; }

int dma_attention_set_kv_split(int mode) {
  const int prev = kv_split_mode();
  g_kvsplit.store(mode < -1 ? -1 : mode, std::memory_order_relaxed);
  return prev;
}

int dma_attention_kv_split(const DmaAttnArgs* a) {
  if (validate(a)) return -1;
  const Layout L = plan_layout(a);
  return fused_eligible(a, L) ? 1 : L.kv_split;  // the fused forward never splits
}

int dma_attention_set_fused(int on) {
  const int prev = fuse_enabled() ? 1 : 0;
  g_fuse.store(on ? 1 : 0, std::memory_order_relaxed);
  return prev;
}

// (DMA_TRACE builds: dma_trace_read lives in kern_pp.cu, next to the kernel's trace buffer)
// (DMA_PROFILE builds: dma_prof_read lives in kern_pp.cu, next to the kernel's counters)

}  // extern "C"
