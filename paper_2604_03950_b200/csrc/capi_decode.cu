// C-ABI: decode attention over an MX-quantized key cache (decode.cuh).
#include <atomic>
#include "common.cuh"
#include "decode.cuh"

namespace dma {

static int fail(int rc, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  set_error("%s", buf);
  return rc;
}

struct DecodeShape {
  int64_t rows_total;  // batch * heads * n_q
  int32_t group, rows_per_kvh, R, n_rg, splits, keys_per_split;
  int low;
};

static int pow2_at_least(int x) {
  int r = 1;
  while (r < x) r <<= 1;
  return r;
}

static int decode_shape(const DmaDecodeArgs* a, DecodeShape& s) {
  if (a->batch < 1 || a->heads < 1 || a->kv_heads < 1 || a->n_q < 1 || a->pos < 0 || a->capacity < 1)
    return fail(DMA_EINVAL, "decode: batch, heads, kv_heads, n_q, capacity must be >= 1 and pos >= 0");
  if (a->heads % a->kv_heads) return fail(DMA_EINVAL, "decode: heads %% kv_heads != 0");
  if (a->capacity % 32)
    return fail(DMA_EINVAL, "decode: capacity (%lld) must be a multiple of 32", (long long)a->capacity);
  if (a->pos + a->n_q > a->capacity)
    return fail(DMA_EINVAL, "decode: pos + n_q (%lld) exceeds the cache capacity (%lld)",
                (long long)(a->pos + a->n_q), (long long)a->capacity);
  if ((a->head_dim != 64 && a->head_dim != 128) || (a->v_dim != 64 && a->v_dim != 128))
    return fail(DMA_EUNSUPPORTED, "decode: head_dim and v_dim must be 64 or 128");
  if (a->tile_m < 1 || a->tile_n < 32 || a->tile_n % 32 || a->diag_window < 0 || a->sink_window < 0)
    return fail(DMA_EUNSUPPORTED, "decode: tile_n must be a multiple of 32 (tile_m >= 1)");
  if (a->granularity != DMA_GRAN_TOKEN)
    return fail(DMA_EUNSUPPORTED, "decode: TOKEN granularity only (cache rows are quantized once)");
  if (a->high_format != DMA_FMT_MXFP8_E4M3 && a->high_format != DMA_FMT_MXFP8_E5M2)
    return fail(DMA_EUNSUPPORTED, "decode: high format must be MXFP8 (E4M3 or E5M2)");
  switch (a->low_format) {
    case DMA_FMT_NVFP4: s.low = kDecLowNV; break;
    case DMA_FMT_MXFP4: s.low = kDecLowMX4; break;
    case DMA_FMT_MXFP8_E4M3:
    case DMA_FMT_MXFP8_E5M2: s.low = kDecLow8; break;
    default: return fail(DMA_EUNSUPPORTED, "decode: low format must be NVFP4, MXFP4 or an MXFP8 format");
  }
  if (a->v_dtype != DMA_DT_BF16) return fail(DMA_EUNSUPPORTED, "decode: the value cache must be bf16");
  if (a->out_dtype != DMA_DT_F32 && a->out_dtype != DMA_DT_BF16)
    return fail(DMA_EUNSUPPORTED, "decode: out_dtype must be f32 or bf16");
  s.group = static_cast<int32_t>(a->heads / a->kv_heads);
  const int64_t rows = static_cast<int64_t>(s.group) * a->n_q;
  if (rows > (1 << 20)) return fail(DMA_EUNSUPPORTED, "decode: too many query rows per KV head");
  s.rows_per_kvh = static_cast<int32_t>(rows);
  // R <= 8 query rows per CTA: more rows per KV head become more row groups (each streams
  // the cache again) -- measured faster than R = 16 (register-bound, spills)
  s.R = pow2_at_least(static_cast<int>(rows < 8 ? rows : 8));
  s.n_rg = static_cast<int32_t>((rows + s.R - 1) / s.R);
  s.rows_total = a->batch * a->heads * a->n_q;
  const int64_t units = a->batch * a->kv_heads * s.n_rg;
  const int64_t len = a->pos + a->n_q;
  // about three waves of resident CTAs (shared-memory bound residency): measured faster
  // than one long wave -- short CTAs keep every SM's warps busy through the tail
  const int per_sm = dec_ctas_per_sm(s.R, static_cast<int>(a->head_dim), static_cast<int>(a->v_dim), s.low);
  int64_t splits = (static_cast<int64_t>(3 * per_sm) * 148 + units - 1) / units;
  const int64_t max_splits = (len + 127) / 128;
  splits = splits < 1 ? 1 : (splits > max_splits ? max_splits : splits);
  int64_t kps = (len + splits - 1) / splits;
  kps = (kps + 127) / 128 * 128;
  splits = (len + kps - 1) / kps;
  if (units * splits > 0x7FFFFFFF) return fail(DMA_EUNSUPPORTED, "decode: grid too large");
  s.splits = static_cast<int32_t>(splits);
  s.keys_per_split = static_cast<int32_t>(kps);
  return DMA_OK;
}

static size_t decode_ws(const DmaDecodeArgs* a, const DecodeShape& s) {
  const size_t slots = static_cast<size_t>(s.rows_total) * s.splits;
  return (slots * a->v_dim * 4 + 255) / 256 * 256 + slots * 8 + 256;
}

template <int R, int D, int DV, int LOW>
static cudaError_t launch_decode(const DecodeParams& p, int grid, cudaStream_t st) {
  constexpr int smem = DecSmem<R, D, DV, LOW>::kBytes;
  static_assert(smem <= 227 * 1024, "decode smem");
  // the attribute is per device context: remember it per device (bit d), thread-safely
  static std::atomic<unsigned long long> attr_set{0ull};
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev); e != cudaSuccess) return e;
  const unsigned long long bit = dev < 64 ? (1ull << dev) : 0ull;
  if (!bit || !(attr_set.load(std::memory_order_acquire) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(dma_decode_kernel<R, D, DV, LOW>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(bit, std::memory_order_release);
  }
  dma_decode_kernel<R, D, DV, LOW><<<grid, 128, smem, st>>>(p);
  return cudaGetLastError();
}

template <int D, int DV, int LOW>
static cudaError_t dispatch_r(int R, const DecodeParams& p, int grid, cudaStream_t st) {
  switch (R) {
    case 1: return launch_decode<1, D, DV, LOW>(p, grid, st);
    case 2: return launch_decode<2, D, DV, LOW>(p, grid, st);
    case 4: return launch_decode<4, D, DV, LOW>(p, grid, st);
    default: return launch_decode<8, D, DV, LOW>(p, grid, st);
  }
}

template <int D, int DV>
static cudaError_t dispatch_low(int low, int R, const DecodeParams& p, int grid, cudaStream_t st) {
  switch (low) {
    case kDecLowNV: return dispatch_r<D, DV, kDecLowNV>(R, p, grid, st);
    case kDecLowMX4: return dispatch_r<D, DV, kDecLowMX4>(R, p, grid, st);
    default: return dispatch_r<D, DV, kDecLow8>(R, p, grid, st);
  }
}

}  // namespace dma

using namespace dma;

extern "C" {

size_t dma_decode_workspace_bytes(const DmaDecodeArgs* a) {
  DecodeShape s;
  if (!a || decode_shape(a, s) != DMA_OK) return 0;
  return decode_ws(a, s);
}

int dma_decode_attention(const DmaDecodeArgs* a, void* stream) {
  if (!a) return fail(DMA_EINVAL, "decode: null args");
  DecodeShape s;
  int rc = decode_shape(a, s);
  if (rc != DMA_OK) return rc;
  if (!a->q_high_codes || !a->q_scales_high || !a->q_quant_scale || !a->k_high_codes || !a->k_scales_high ||
      !a->k_quant_scale || !a->v || !a->o || (s.low != kDecLow8 && (!a->q_packed_low || !a->q_scales_low ||
                                                                     !a->k_packed_low || !a->k_scales_low)))
    return fail(DMA_EINVAL, "decode: missing operand pointer");
  const size_t need = decode_ws(a, s);
  if (!a->workspace || a->workspace_bytes < need)
    return fail(DMA_EINVAL, "decode: workspace too small (%zu < %zu)", a->workspace_bytes, need);
  const size_t slots = static_cast<size_t>(s.rows_total) * s.splits;
  uint8_t* ws = static_cast<uint8_t*>(a->workspace);
  DecodeParams p{};
  p.q_lo = a->q_packed_low;
  p.q_lo_sf = a->q_scales_low;
  p.q_hi = a->q_high_codes;
  p.q_hi_sf = a->q_scales_high;
  p.q_sq = a->q_quant_scale;
  p.k_lo = a->k_packed_low;
  p.k_lo_sf = a->k_scales_low;
  p.k_hi = a->k_high_codes;
  p.k_hi_sf = a->k_scales_high;
  p.k_sq = a->k_quant_scale;
  p.v = static_cast<const __nv_bfloat16*>(a->v);
  p.part_o = reinterpret_cast<float*>(ws);
  p.part_ml = reinterpret_cast<float2*>(ws + (slots * a->v_dim * 4 + 255) / 256 * 256);
  p.batch = a->batch;
  p.heads = a->heads;
  p.kv_heads = a->kv_heads;
  p.n_q = a->n_q;
  p.cap = a->capacity;
  p.pos = a->pos;
  p.group = s.group;
  p.rows_per_kvh = s.rows_per_kvh;
  p.n_rg = s.n_rg;
  p.splits = s.splits;
  p.keys_per_split = s.keys_per_split;
  p.tile_m = a->tile_m;
  p.tile_n = a->tile_n;
  p.diag_window = a->diag_window;
  p.sink_window = a->sink_window;
  p.hi_e5m2 = a->high_format == DMA_FMT_MXFP8_E5M2;
  const int grid = static_cast<int>(a->batch * a->kv_heads * s.n_rg * s.splits);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (a->head_dim == 128)
    e = a->v_dim == 128 ? dispatch_low<128, 128>(s.low, s.R, p, grid, st)
                        : dispatch_low<128, 64>(s.low, s.R, p, grid, st);
  else
    e = a->v_dim == 128 ? dispatch_low<64, 128>(s.low, s.R, p, grid, st)
                        : dispatch_low<64, 64>(s.low, s.R, p, grid, st);
  if (e != cudaSuccess) return fail(static_cast<int>(e), "decode kernel: %s", cudaGetErrorString(e));
  const int64_t threads = s.rows_total * 32;
  const int cgrid = static_cast<int>((threads + 255) / 256);
  if (a->v_dim == 128)
    dma_decode_combine_kernel<128><<<cgrid, 256, 0, st>>>(p.part_o, p.part_ml, s.rows_total, s.splits, a->o,
                                                           a->out_dtype == DMA_DT_BF16);
  else
    dma_decode_combine_kernel<64><<<cgrid, 256, 0, st>>>(p.part_o, p.part_ml, s.rows_total, s.splits, a->o,
                                                          a->out_dtype == DMA_DT_BF16);
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(static_cast<int>(e), "decode combine: %s", cudaGetErrorString(e));
  return DMA_OK;
}

}  // extern "C"
