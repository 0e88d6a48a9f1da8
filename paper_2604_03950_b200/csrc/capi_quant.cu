// C-ABI: quantize_dual / dequantize / element codecs / plans / error plumbing.
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "quant.cuh"

namespace dma {

static thread_local char g_err[1024] = "";
thread_local bool g_pdl_next = false;

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("DMA_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
const char* get_error() { return g_err; }

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// DMA_QUANT32=0 selects the 16-column bf16 kernel (A/B and debugging)
static bool quant32_enabled() {
  static const bool on = [] {
    const char* e = getenv("DMA_QUANT32");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename T, bool NV, bool E5, int GRAN>
static void launch_rows(const DmaQuantArgs* a, const unsigned long long* tmax, const QuantOut& out,
                        cudaStream_t st) {
  const int64_t nrows = a->n_mat * a->rows;
  const int64_t tpr = a->cols / 16;
  if (tpr <= 32 && (tpr & (tpr - 1)) == 0 && a->row_stride % 8 == 0 && a->mat_stride % 8 == 0) {
    if constexpr (sizeof(T) == 2) {
      if (quant32_enabled()) {  // bf16: 32 columns per thread (q32_item_bf16)
        // contiguous matrices of whole 128-row tiles run as one matrix of n_mat * rows rows
        // (every output offset is then the global row's; TENSOR needs the matrix index)
        const bool flat = GRAN != DMA_GRAN_TENSOR && a->n_mat > 1 && a->mat_stride == a->rows * a->row_stride &&
                          a->rows % 128 == 0 && out.rows_pad == a->rows;
        const int64_t n_mat = flat ? 1 : a->n_mat, rows = flat ? a->n_mat * a->rows : a->rows;
        const int64_t tpr32 = a->cols / 32;
        const int64_t nbx = (rows * tpr32 + 255) / 256;
        const int64_t by = n_mat < 65535 ? n_mat : 65535;
        int64_t bx = (148 * 8 + by - 1) / by;
        bx = bx < 1 ? 1 : (bx > nbx ? nbx : bx);
        QuantOut o = out;
        if (flat) o.rows_pad = rows;
        const cudaError_t e = launch_kernel(
            g_pdl_next, quant32_bf16_kernel<NV, E5, GRAN>, dim3(static_cast<unsigned>(bx), static_cast<unsigned>(by)),
            dim3(256), 0, st, static_cast<const __nv_bfloat16*>(a->x), n_mat, rows, static_cast<int>(a->cols),
            flat ? 0 : a->mat_stride, a->row_stride, a->is_query, a->prescale, tmax, o);
        if (e != cudaSuccess) set_error("quant32 launch: %s", cudaGetErrorString(e));
        return;
      }
    }
    // fast path: 16 columns per thread (cols in {32, 64, 128, 256, 512})
    // grid-stride over (row block, matrix) items: y covers the matrices (<= 65535),
    // x about 8 CTAs per SM in total so every CTA walks several row blocks (prefetching)
    const int64_t nbx = (a->rows * tpr + 255) / 256;
    const int64_t by = a->n_mat < 65535 ? a->n_mat : 65535;
    int64_t bx = (148 * 8 + by - 1) / by;
    bx = bx < 1 ? 1 : (bx > nbx ? nbx : bx);
    quant16_kernel<T, NV, E5, GRAN><<<dim3(static_cast<unsigned>(bx), static_cast<unsigned>(by)), 256, 0, st>>>(
        static_cast<const T*>(a->x), a->n_mat, a->rows, static_cast<int>(a->cols), a->mat_stride, a->row_stride,
        a->is_query, a->prescale, tmax, out);
    return;
  }
  const int64_t blocks = (nrows + 7) / 8;
  quant_rows_kernel<T, NV, E5, GRAN><<<static_cast<unsigned>(blocks), 256, 0, st>>>(
      static_cast<const T*>(a->x), a->n_mat, a->rows, static_cast<int>(a->cols), a->mat_stride, a->row_stride,
      a->is_query, a->prescale, tmax, out);
}

template <typename T, bool NV, bool E5>
static void dispatch_gran(const DmaQuantArgs* a, const unsigned long long* tmax, const QuantOut& out,
                          cudaStream_t st) {
  switch (a->granularity) {
    case DMA_GRAN_TOKEN: launch_rows<T, NV, E5, DMA_GRAN_TOKEN>(a, tmax, out, st); break;
    case DMA_GRAN_BLOCK: launch_rows<T, NV, E5, DMA_GRAN_BLOCK>(a, tmax, out, st); break;
    default: launch_rows<T, NV, E5, DMA_GRAN_TENSOR>(a, tmax, out, st); break;
  }
}

template <typename T>
static void dispatch_fmt(const DmaQuantArgs* a, const unsigned long long* tmax, const QuantOut& out,
                         cudaStream_t st) {
  const bool nv = a->low_format == DMA_FMT_NVFP4;
  const bool e5 = a->high_format == DMA_FMT_MXFP8_E5M2;
  if (nv && e5) dispatch_gran<T, true, true>(a, tmax, out, st);
  else if (nv) dispatch_gran<T, true, false>(a, tmax, out, st);
  else if (e5) dispatch_gran<T, false, true>(a, tmax, out, st);
  else dispatch_gran<T, false, false>(a, tmax, out, st);
}

template <typename T>
static void launch_absmax(const DmaQuantArgs* a, unsigned long long* tmax, cudaStream_t st) {
  const int64_t n = a->rows * a->cols;
  int64_t gx = (n + 255) / 256;
  if (gx > 1024) gx = 1024;
  if (gx < 1) gx = 1;
  absmax_kernel<T><<<dim3(static_cast<unsigned>(gx), static_cast<unsigned>(a->n_mat)), 256, 0, st>>>(
      static_cast<const T*>(a->x), a->rows, static_cast<int>(a->cols), a->mat_stride, a->row_stride, tmax);
}

// Validates and runs quantize_dual with explicit operand-layout outputs (used by
// the attention path as well as the public entry point).
int quantize_impl(const DmaQuantArgs* a, uint8_t* sf_low_op, uint8_t* sf_high_op, float* qs_f32,
                  int64_t rows_pad, cudaStream_t st, int key_perm) {
  DMA_CHECK_ARG(a && a->x, "quantize_dual: null input");
  DMA_CHECK_ARG(a->cols > 0 && a->cols % 32 == 0 && a->cols <= 1024,
                "quantize_dual: cols must be a multiple of 32 in [32, 1024], got %lld", (long long)a->cols);
  DMA_CHECK_ARG(a->rows >= 0 && a->n_mat >= 0, "quantize_dual: negative shape");
  DMA_CHECK_ARG(a->low_format == DMA_FMT_NVFP4 || a->low_format == DMA_FMT_MXFP4,
                "quantize_dual: low format must have E2M1 elements");
  DMA_CHECK_ARG(a->high_format == DMA_FMT_MXFP8_E4M3 || a->high_format == DMA_FMT_MXFP8_E5M2,
                "quantize_dual: high format must have FP8 elements");
  DMA_CHECK_ARG(a->granularity >= 0 && a->granularity <= 2, "quantize_dual: unknown granularity");
  DMA_CHECK_ARG(a->x_dtype >= DMA_DT_F64 && a->x_dtype <= DMA_DT_BF16, "quantize_dual: bad dtype");
  DMA_CHECK_ARG(a->row_stride % 4 == 0 && aligned16(a->x), "quantize_dual: input must be 16B aligned, row stride %% 4 == 0");
  if (a->n_mat == 0 || a->rows == 0) return 0;
  unsigned long long* tmax = nullptr;
  if (a->granularity == DMA_GRAN_TENSOR) {
    DMA_CHECK_ARG(a->workspace && a->workspace_bytes >= static_cast<size_t>(a->n_mat) * 8,
                  "quantize_dual: TENSOR granularity needs a workspace of %lld bytes", (long long)(a->n_mat * 8));
    tmax = static_cast<unsigned long long*>(a->workspace);
    DMA_CUDA_TRY(cudaMemsetAsync(tmax, 0, static_cast<size_t>(a->n_mat) * 8, st));
    if (a->x_dtype == DMA_DT_F64) launch_absmax<double>(a, tmax, st);
    else if (a->x_dtype == DMA_DT_F32) launch_absmax<float>(a, tmax, st);
    else launch_absmax<__nv_bfloat16>(a, tmax, st);
    DMA_LAUNCH_CHECK();
  }
  QuantOut out{};
  out.packed_low = a->packed_low;
  out.scales_low = a->scales_low;
  out.high_codes = a->high_codes;
  out.scales_high = a->scales_high;
  out.quant_scale = a->quant_scale;
  out.nonfinite = a->nonfinite;
  out.sf_low_op = sf_low_op;
  out.sf_high_op = sf_high_op;
  out.qs_f32 = qs_f32;
  out.rows_pad = rows_pad > 0 ? rows_pad : ((a->rows + 127) / 128) * 128;
  out.key_perm = key_perm;
  if (key_perm) {
    const int64_t tpr = a->cols / 16;
    DMA_CHECK_ARG(tpr <= 32 && (tpr & (tpr - 1)) == 0 && a->row_stride % 8 == 0 && a->mat_stride % 8 == 0,
                  "quantize_dual: permuted operand layout needs cols in {32..512} (power of two) and aligned rows");
  }
  if (a->x_dtype == DMA_DT_F64) dispatch_fmt<double>(a, tmax, out, st);
  else if (a->x_dtype == DMA_DT_F32) dispatch_fmt<float>(a, tmax, out, st);
  else dispatch_fmt<__nv_bfloat16>(a, tmax, out, st);
  DMA_LAUNCH_CHECK();
  return 0;
}

// ------------------------------------------------------------ dequantizers
__global__ void dequant_kernel(int which, int nv, int e5, int gran, int64_t n_mat, int64_t rows, int cols,
                               const uint8_t* pl, const uint8_t* sl, const uint8_t* hc, const uint8_t* sh,
                               const double* qs, double* out) {
  const int64_t n = n_mat * rows * cols;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t rr = i / cols;  // mat*rows + row
    const int col = static_cast<int>(i % cols);
    const int64_t mat = rr / rows;
    double s_q;
    if (gran == DMA_GRAN_TOKEN) s_q = qs[rr];
    else if (gran == DMA_GRAN_BLOCK) s_q = qs[rr * (cols / 32) + col / 32];
    else s_q = qs[mat];
    double v;
    if (which == 0) {
      uint32_t byte = pl[rr * (cols / 2) + col / 2];
      uint32_t code = (col & 1) ? (byte >> 4) : (byte & 0xF);
      const double mags[8] = {0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0};
      double e = mags[code & 7];
      if (code & 8) e = -e;
      if (nv) {
        v = e * decode_e4m3(sl[rr * (cols / 16) + col / 16]) * s_q;  // quantize.py:224-228
      } else {
        v = e * pow2(static_cast<int>(sl[rr * (cols / 32) + col / 32]) - 127);  // single level
      }
    } else {
      uint32_t c = hc[i];
      double e;
      if (e5) {
        uint32_t ex = (c >> 2) & 0x1F, m = c & 3;
        if (ex == 31) e = m ? NAN : INFINITY;
        else e = ex ? (4.0 + m) * pow2(static_cast<int>(ex) - 17) : m * pow2(-16);
        if (c & 0x80) e = -e;
      } else {
        e = ((c & 0x7F) == 0x7F) ? NAN : decode_e4m3(c);
      }
      v = e * pow2(static_cast<int>(sh[rr * (cols / 32) + col / 32]) - 127) * s_q;  // quantize.py:235-237
    }
    out[i] = v;
  }
}

__global__ void encode_e2m1_kernel(const double* x, int64_t n, uint8_t* codes) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    codes[i] = static_cast<uint8_t>(e2m1_pair(x[i], 0.0) & 0xF);
  }
}

__global__ void encode_fp8_kernel(const double* x, int64_t n, int e5, uint8_t* codes) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double u = e5 ? 57344.0 : 448.0;
    // formats.py:220-224 rounds, then saturates at the format maximum
    const double v = fmin(fmax(x[i], -u), u);
    codes[i] = static_cast<uint8_t>((e5 ? fp8_pair<true>(v, 0.0) : fp8_pair<false>(v, 0.0)) & 0xFF);
  }
}

static unsigned grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 4096) g = 4096;
  return static_cast<unsigned>(g < 1 ? 1 : g);
}

}  // namespace dma

using namespace dma;

extern "C" {

const char* dma_last_error(void) { return get_error(); }
int dma_abi_version(void) { return DMA_ABI_VERSION; }

size_t dma_quantize_workspace_bytes(const DmaQuantArgs* a) {
  return a && a->granularity == DMA_GRAN_TENSOR ? static_cast<size_t>(a->n_mat) * 8 : 0;
}

int dma_quantize_dual(const DmaQuantArgs* a, void* stream) {
  return quantize_impl(a, nullptr, nullptr, nullptr, 0, static_cast<cudaStream_t>(stream), 0);
}

int dma_dequantize(int32_t which, int32_t low_format, int32_t high_format, int32_t granularity, int64_t n_mat,
                   int64_t rows, int64_t cols, const uint8_t* packed_low, const uint8_t* scales_low,
                   const uint8_t* high_codes, const uint8_t* scales_high, const double* quant_scale, double* out,
                   void* stream) {
  DMA_CHECK_ARG(which == 0 || which == 1, "dequantize: which must be 0 (low) or 1 (high)");
  DMA_CHECK_ARG(cols % 32 == 0, "dequantize: cols %% 32 != 0");
  DMA_CHECK_ARG(low_format == DMA_FMT_NVFP4 || low_format == DMA_FMT_MXFP4, "dequantize: bad low format");
  const int64_t n = n_mat * rows * cols;
  if (n == 0) return 0;
  dequant_kernel<<<grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      which, low_format == DMA_FMT_NVFP4, high_format == DMA_FMT_MXFP8_E5M2, granularity, n_mat, rows,
      static_cast<int>(cols), packed_low, scales_low, high_codes, scales_high, quant_scale, out);
  DMA_LAUNCH_CHECK();
  return 0;
}

int dma_encode_e2m1(const double* x, int64_t n, uint8_t* codes, void* stream) {
  if (n == 0) return 0;
  encode_e2m1_kernel<<<grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(x, n, codes);
  DMA_LAUNCH_CHECK();
  return 0;
}

int dma_encode_fp8(const double* x, int64_t n, int32_t e5m2, uint8_t* codes, void* stream) {
  if (n == 0) return 0;
  encode_fp8_kernel<<<grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(x, n, e5m2, codes);
  DMA_LAUNCH_CHECK();
  return 0;
}

int64_t dma_tile_plan(int64_t q_tile, int64_t len_q, int64_t len_k, int32_t tile_m, int32_t tile_n,
                      int32_t diag_window, int32_t sink_window, int32_t causal, int64_t* out, int64_t cap) {
  Plan p;
  p.init(q_tile, len_q, len_k, tile_m, tile_n, diag_window, sink_window, causal != 0);
  for (int32_t i = 0; i < p.n && i < cap; ++i) {
    int32_t t;
    bool h;
    p.entry(i, t, h);
    out[i] = 2 * static_cast<int64_t>(t) + (h ? 1 : 0);
  }
  return p.n;
}

double dma_high_precision_fraction(int64_t len_q, int64_t len_k, int32_t tile_m, int32_t tile_n,
                                   int32_t diag_window, int32_t sink_window, int32_t causal) {
  // metrics.py:55-101 with the per-row cumulative count done in closed form
  // over the tile plan (one pass per query tile, O(plan) each).
  int64_t hi_cells = 0, valid = 0;
  const int64_t nqt = ceil_div(len_q, tile_m);
  for (int64_t qt = 0; qt < nqt; ++qt) {
    const int64_t q0 = qt * tile_m, q1 = std::min<int64_t>(q0 + tile_m, len_q);
    Plan p;
    p.init(qt, len_q, len_k, tile_m, tile_n, diag_window, sink_window, causal != 0);
    if (causal) {
      // high keys are tiles [0, lo0) and [lo1, n); row r sees keys [0, min(r, len_k-1)]
      for (int64_t r = q0; r < q1; ++r) {
        const int64_t kmax = std::min<int64_t>(r, len_k - 1);
        const int64_t seen = kmax + 1;
        auto high_upto = [&](int64_t kend) {  // # high keys among [0, kend)
          int64_t c = 0;
          int64_t a_end = std::min<int64_t>(static_cast<int64_t>(p.lo0) * tile_n, len_k);
          c += std::max<int64_t>(0, std::min(kend, a_end));
          int64_t b0 = static_cast<int64_t>(p.lo1) * tile_n;
          int64_t b1 = std::min<int64_t>(static_cast<int64_t>(p.n) * tile_n, len_k);
          c += std::max<int64_t>(0, std::min(kend, b1) - b0);
          return c;
        };
        hi_cells += high_upto(seen);
        valid += seen;
      }
    } else {
      int64_t high = 0;
      for (int32_t i = 0; i < p.n; ++i) {
        int32_t t;
        bool h;
        p.entry(i, t, h);
        if (h) high += std::min<int64_t>(static_cast<int64_t>(t + 1) * tile_n, len_k) - static_cast<int64_t>(t) * tile_n;
      }
      hi_cells += high * (q1 - q0);
      valid += len_k * (q1 - q0);
    }
  }
  return valid == 0 ? 0.0 : static_cast<double>(hi_cells) / static_cast<double>(valid);
}

}  // extern "C"
