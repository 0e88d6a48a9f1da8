// Phase 1 of the DMA forward: bit-exact dual MX quantization (paper Alg. 2).
//
// Restates quantize.py:122-212 on the GPU.  Every float64 operation that
// feeds a rounding decision is performed in IEEE float64 in the reference's
// order (x*c, gmax/2688, x_sm/S_q, bmax/6, blk/scale); the final f64 -> 8/4-bit
// rounding goes through a round-to-odd f64 -> f32 step followed by the
// hardware RNE-satfinite cvt, which is exact (no double rounding).  Two sign
// fixups reproduce formats.py:144 (exact -0 -> +0 in E2M1) and
// formats.py:240 (every zero magnitude -> +0 in FP8).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "common.cuh"
#include "ptx.cuh"

namespace dma {

// ------------------------------------------------------------- scalar codecs
__device__ __forceinline__ float rto_f32(double d) {
  // round-to-odd float64 -> float32: truncate, then set the sticky LSB if inexact
  float t = __double2float_rz(d);
  if (static_cast<double>(t) != d) t = __uint_as_float(__float_as_uint(t) | 1u);
  return t;
}

__device__ __forceinline__ int floor_log2_pos(double v) {
  // exact floor(log2 v) for v > 0 (f64 subnormals give -1023, which every
  // caller clamps to -127 exactly like np.maximum(v, tiny) in quantize.py:171)
  return static_cast<int>((__double_as_longlong(v) >> 52) & 0x7FF) - 1023;
}

__device__ __forceinline__ double pow2(int e) {  // 2^e for e in [-1022, 1023]
  return __hiloint2double((e + 1023) << 20, 0);
}

__device__ __forceinline__ double decode_e4m3(uint32_t c) {
  uint32_t e = (c >> 3) & 0xF, m = c & 7;
  double mag = e ? (8.0 + m) * pow2(static_cast<int>(e) - 10) : m * 0.001953125;  // 2^-9
  return (c & 0x80) ? -mag : mag;
}

// E2M1 code of two values (each already clamped to [-6, 6]); returns (c1 << 4) | c0
__device__ __forceinline__ uint32_t e2m1_pair(double v0, double v1) {
  uint32_t mag = ptx::cvt_e2m1x2(fabsf(rto_f32(v0)), fabsf(rto_f32(v1)));
  uint32_t s0 = (v0 < 0.0) ? 0x08u : 0u;  // exact -0.0 compares equal to 0 -> +0
  uint32_t s1 = (v1 < 0.0) ? 0x80u : 0u;
  return (mag | s0 | s1) & 0xFFu;
}

// FP8 codes of two values (clamped to the format range); byte0 = v0
template <bool E5>
__device__ __forceinline__ uint32_t fp8_pair(double v0, double v1) {
  float a = fabsf(rto_f32(v0)), b = fabsf(rto_f32(v1));
  uint32_t mag = E5 ? ptx::cvt_e5m2x2(a, b) : ptx::cvt_e4m3x2(a, b);
  uint32_t c0 = mag & 0xFF, c1 = (mag >> 8) & 0xFF;
  if (c0 && v0 < 0.0) c0 |= 0x80;  // rounded-to-zero magnitudes stay +0
  if (c1 && v1 < 0.0) c1 |= 0x80;
  return c0 | (c1 << 8);
}

__device__ __forceinline__ uint32_t e4m3_pos(double v) {  // code of a value > 0
  uint32_t c = ptx::cvt_e4m3x2(rto_f32(v), 0.0f) & 0xFF;
  return (c & 0x7F) ? c : 0u;
}

template <typename T>
struct Load4;
template <>
struct Load4<double> {
  __device__ static void run(const double* p, double (&v)[4]) {
    double2 a = *reinterpret_cast<const double2*>(p);
    double2 b = *reinterpret_cast<const double2*>(p + 2);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
};
template <>
struct Load4<float> {
  __device__ static void run(const float* p, double (&v)[4]) {
    float4 a = *reinterpret_cast<const float4*>(p);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  }
};
template <>
struct Load4<__nv_bfloat16> {
  __device__ static void run(const __nv_bfloat16* p, double (&v)[4]) {
    uint2 a = *reinterpret_cast<const uint2*>(p);
    v[0] = __uint_as_float(a.x << 16);
    v[1] = __uint_as_float(a.x & 0xFFFF0000u);
    v[2] = __uint_as_float(a.y << 16);
    v[3] = __uint_as_float(a.y & 0xFFFF0000u);
  }
};

// Where phase 1 writes its results.  Canonical = the reference layout
// (quantize.py:69-89); operand = what the phase-2 kernel loads (the element
// arrays are shared: row-major K-major codes ARE the tcgen05 operand layout).
struct QuantOut {
  uint8_t* packed_low;   // [mat, rows, cols/2]
  uint8_t* scales_low;   // [mat, rows, cols/V1]      canonical
  uint8_t* high_codes;   // [mat, rows, cols]
  uint8_t* scales_high;  // [mat, rows, cols/32]      canonical
  double* quant_scale;   // [mat, rows] | [mat, rows, cols/32] | [mat]
  uint8_t* sf_low_op;    // [mat, rtiles, chunks_low, 512]   tcgen05 scale-factor atoms
  uint8_t* sf_high_op;   // [mat, rtiles, chunks_high, 512]
  float* qs_f32;         // [mat, rows_pad] per-row S_q as f32 (TOKEN / TENSOR)
  uint32_t* nonfinite;
  int64_t rows_pad;      // rows rounded up to 128
  int key_perm;          // 0: canonical rows; 1: operand rows permuted inside 128-row tiles (attn_pp.cuh);
                         // 2: natural rows (attn_sk.cuh); 1 and 2 pad codes to rows_pad and keep S_q^K
                         // in per-tile blocks of kSqkTile slots
};


// 32-row x 4-SF interleave of one 128-row scale-factor atom (cutlass
// Sm1xxBlockScaledBasicChunk: offset (r%32)*16 + (r/32)*4 + k)
__device__ __forceinline__ int64_t sf_atom_offset(int64_t mat, int64_t row, int kb, int64_t rtiles, int chunks) {
  int r = static_cast<int>(row & 127);
  int64_t tile = (mat * rtiles + (row >> 7)) * chunks + (kb >> 2);
  return tile * 512 + (r & 31) * 16 + (r >> 5) * 4 + (kb & 3);
}

__device__ __forceinline__ double warp_max_xor(double v, int width_mask) {
  for (int o = 1; o <= width_mask; o <<= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// One warp per row; lane l handles columns [128*ch + 4l, +4) for chunk ch.
template <typename T, bool NV, bool E5, int GRAN>
__global__ void __launch_bounds__(256) quant_rows_kernel(const T* __restrict__ x, int64_t n_mat, int64_t rows,
                                                         int cols, int64_t mat_stride, int64_t row_stride,
                                                         int is_query, double c,
                                                         const unsigned long long* __restrict__ tensor_absmax,
                                                         QuantOut out) {
  constexpr int kMaxCh = 8;  // cols <= 1024
  const int lane = threadIdx.x & 31;
  const int64_t wrow = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wrow >= n_mat * rows) return;
  const int64_t mat = wrow / rows, row = wrow % rows;
  const T* xr = x + mat * mat_stride + row * row_stride;
  const int nch = (cols + 127) >> 7;

  double xs[kMaxCh][4];
  double amax = 0.0;
  bool bad = false;
#pragma unroll
  for (int ch = 0; ch < kMaxCh; ++ch) {
    if (ch < nch) {
      const int col0 = ch * 128 + lane * 4;
      if (col0 < cols) {
        Load4<T>::run(xr + col0, xs[ch]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          bad |= !isfinite(xs[ch][i]);
          if (is_query) xs[ch][i] = __dmul_rn(xs[ch][i], c);  // quantize.py:149 (x * c)
          amax = fmax(amax, fabs(xs[ch][i]));
        }
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) xs[ch][i] = 0.0;
      }
    }
  }
  if (out.nonfinite && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(out.nonfinite, 1u);

  // ---- group max -> S_q (quantize.py:152-153)
  double sq_row = 1.0;
  if (GRAN == DMA_GRAN_TOKEN) {
    double g = warp_max_xor(amax, 16);
    sq_row = g > 0.0 ? __ddiv_rn(g, 2688.0) : 1.0;
  } else if (GRAN == DMA_GRAN_TENSOR) {
    double g = __longlong_as_double(static_cast<long long>(tensor_absmax[mat]));
    if (is_query) g = __dmul_rn(g, c);  // max|x*c| == fl(max|x| * c): rounding is monotone
    sq_row = g > 0.0 ? __ddiv_rn(g, 2688.0) : 1.0;
  }
  const int nsf_low = cols / (NV ? 16 : 32);
  const int chunks_low = (nsf_low + 3) >> 2;
  const int chunks_high = ((cols / 32) + 3) >> 2;
  const int64_t rtiles = out.rows_pad >> 7;

#pragma unroll
  for (int ch = 0; ch < kMaxCh; ++ch) {
    if (ch >= nch) break;
    const int col0 = ch * 128 + lane * 4;
    const bool valid = col0 < cols;  // warp-uniform per 8-lane group (cols % 32 == 0)
    double sq = sq_row;
    if (GRAN == DMA_GRAN_BLOCK) {
      double m = fmax(fmax(fabs(xs[ch][0]), fabs(xs[ch][1])), fmax(fabs(xs[ch][2]), fabs(xs[ch][3])));
      m = warp_max_xor(m, 4);
      sq = m > 0.0 ? __ddiv_rn(m, 2688.0) : 1.0;
    }
    double xsc[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) xsc[i] = __ddiv_rn(xs[ch][i], sq);  // quantize.py:154

    // ---- 4-bit path (quantize.py:156-184)
    double lv[4];
    uint32_t sc_low;
    if (NV) {
      double bm = fmax(fmax(fabs(xsc[0]), fabs(xsc[1])), fmax(fabs(xsc[2]), fabs(xsc[3])));
      bm = warp_max_xor(bm, 2);  // 16-column block = 4 lanes
      uint32_t code = bm > 0.0 ? e4m3_pos(__ddiv_rn(bm, 6.0)) : 0x38u;
      if (code == 0 && bm > 0.0) code = 0x01;  // floor at 2^-9 (quantize.py:164-167)
      const double sv = decode_e4m3(code);
#pragma unroll
      for (int i = 0; i < 4; ++i) lv[i] = fmin(fmax(__ddiv_rn(xsc[i], sv), -6.0), 6.0);
      sc_low = code;
    } else {
      double bm = fmax(fmax(fabs(xs[ch][0]), fabs(xs[ch][1])), fmax(fabs(xs[ch][2]), fabs(xs[ch][3])));
      bm = warp_max_xor(bm, 4);  // 32-column block = 8 lanes, single-level on x_sm
      int e = bm > 0.0 ? min(max(floor_log2_pos(bm) - 2, -127), 127) : -127;
      const double inv = pow2(-e);
#pragma unroll
      for (int i = 0; i < 4; ++i) lv[i] = fmin(fmax(xs[ch][i] * inv, -6.0), 6.0);
      sc_low = static_cast<uint32_t>(e + 127);
    }
    const uint32_t p01 = e2m1_pair(lv[0], lv[1]);
    const uint32_t p23 = e2m1_pair(lv[2], lv[3]);

    // ---- 8-bit path (quantize.py:186-199)
    double hm = fmax(fmax(fabs(xsc[0]), fabs(xsc[1])), fmax(fabs(xsc[2]), fabs(xsc[3])));
    hm = warp_max_xor(hm, 4);
    constexpr int kEmax = E5 ? 15 : 8;
    constexpr double kUpper = E5 ? 57344.0 : 448.0;
    const int he = hm > 0.0 ? min(max(floor_log2_pos(hm) - kEmax, -127), 127) : -127;
    const double hinv = pow2(-he);
    double hv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) hv[i] = fmin(fmax(xsc[i] * hinv, -kUpper), kUpper);
    const uint32_t c01 = fp8_pair<E5>(hv[0], hv[1]);
    const uint32_t c23 = fp8_pair<E5>(hv[2], hv[3]);
    const uint32_t sc_high = static_cast<uint32_t>(he + 127);

    if (!valid) continue;
    const int64_t rbase = mat * rows + row;
    if (out.packed_low)
      *reinterpret_cast<uint16_t*>(out.packed_low + rbase * (cols / 2) + col0 / 2) =
          static_cast<uint16_t>(p01 | (p23 << 8));
    if (out.high_codes)
      *reinterpret_cast<uint32_t*>(out.high_codes + rbase * cols + col0) = c01 | (c23 << 16);
    const bool low_leader = NV ? (lane & 3) == 0 : (lane & 7) == 0;
    const int kb_low = col0 / (NV ? 16 : 32);
    if (low_leader) {
      if (out.scales_low) out.scales_low[rbase * nsf_low + kb_low] = static_cast<uint8_t>(sc_low);
      if (out.sf_low_op)
        out.sf_low_op[sf_atom_offset(mat, row, kb_low, rtiles, chunks_low)] = static_cast<uint8_t>(sc_low);
    }
    if ((lane & 7) == 0) {
      const int kb = col0 / 32;
      if (out.scales_high) out.scales_high[rbase * (cols / 32) + kb] = static_cast<uint8_t>(sc_high);
      if (out.sf_high_op)
        out.sf_high_op[sf_atom_offset(mat, row, kb, rtiles, chunks_high)] = static_cast<uint8_t>(sc_high);
      if (GRAN == DMA_GRAN_BLOCK && out.quant_scale) out.quant_scale[rbase * (cols / 32) + kb] = sq;
    }
  }
  if (lane == 0) {
    if (GRAN == DMA_GRAN_TOKEN && out.quant_scale) out.quant_scale[mat * rows + row] = sq_row;
    if (GRAN == DMA_GRAN_TENSOR && out.quant_scale && row == 0) out.quant_scale[mat] = sq_row;
    if (GRAN != DMA_GRAN_BLOCK && out.qs_f32) out.qs_f32[mat * out.rows_pad + row] = static_cast<float>(sq_row);
  }
}

// ------------------------------------------------------------------------
// Throughput variant (the one the forward path uses): one thread owns 16
// consecutive columns of one row (exactly one NVFP4 block, half an MX
// block), so a row of ``cols`` is ``tpr = cols/16`` adjacent lanes and every
// group reduction is a short xor-shuffle.  Same decisions as
// quant_rows_kernel, cheaper arithmetic:
//   * a/b in float64 as q = a*y, r = fma(-q, b, a), q' = fma(r, y, q) with
//     y = RN(1/b) (Markstein's theorem: q' == RN(a/b) for these operand
//     ranges; 4e8 brute-force cases in DESIGN.md) -- one reciprocal per row /
//     block instead of a full division per element;
//   * round-to-odd f64 -> f32 on the bit pattern (integer pipe);
//   * no clamps: cvt.rn.satfinite already saturates to +-6 / +-448 / +-57344
//     exactly like the reference's clip-then-round (formats.py:133-134,220-224).
// f64 inputs keep IEEE __ddiv_rn (their range is not bounded like bf16/f32).
// ------------------------------------------------------------------------
__device__ __forceinline__ double mk_div(double a, double b, double y) {
  const double q = __dmul_rn(a, y);
  const double r = __fma_rn(-q, b, a);
  return __fma_rn(r, y, q);
}

// |v| rounded to odd as an f32 (0 for |v| < 2^-126: rounds to +-0 in every target format)
__device__ __forceinline__ float rto_abs(double v) {
  const uint32_t hi = static_cast<uint32_t>(__double2hiint(v)) & 0x7FFFFFFFu;
  const uint32_t lo = static_cast<uint32_t>(__double2loint(v));
  if (hi < 0x38100000u) return 0.0f;
  uint32_t f = __funnelshift_l(lo, hi - 0x38000000u, 3);
  f |= (lo & 0x1FFFFFFFu) != 0u ? 1u : 0u;
  return __uint_as_float(f);
}
__device__ __forceinline__ bool neg_nonzero(double v) { return v < 0.0; }

template <typename T>
struct Load16;
template <>
struct Load16<__nv_bfloat16> {
  __device__ static void run(const __nv_bfloat16* p, double (&v)[16]) {
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(p));
    const uint4 b = __ldg(reinterpret_cast<const uint4*>(p) + 1);
    const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  }
};
template <>
struct Load16<float> {
  __device__ static void run(const float* p, double (&v)[16]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(p) + i);
      v[4 * i] = a.x; v[4 * i + 1] = a.y; v[4 * i + 2] = a.z; v[4 * i + 3] = a.w;
    }
  }
};
template <>
struct Load16<double> {
  __device__ static void run(const double* p, double (&v)[16]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const double2 a = __ldg(reinterpret_cast<const double2*>(p) + i);
      v[2 * i] = a.x; v[2 * i + 1] = a.y;
    }
  }
};

template <typename T>
__device__ __forceinline__ double qdiv(double a, double b, double y) {
  if constexpr (sizeof(T) == 8) return __ddiv_rn(a, b);
  else return mk_div(a, b, y);
}

__device__ __forceinline__ double shfl_max(double v, int lanes) {
  for (int o = 1; o < lanes; o <<= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// One quantize_dual step of one thread: 16 consecutive columns (``part``) of one row of one
// matrix (quantize.py:122-212), with the row's other tpr - 1 parts on the adjacent lanes.
// bf16 inputs arrive as the 32 prefetched bytes cur0 / cur1, other types are loaded here.
// Shared by quant16_kernel (phase 1) and the fused attention kernel (attn_pp.cuh).
template <typename T, bool NV, bool E5, int GRAN>
__device__ __forceinline__ void q16_item(const T* __restrict__ x, int64_t mat_stride, int64_t row_stride, int64_t mat,
                                         int64_t rows, int cols, int64_t row, bool live, int part, int tpr, int lane,
                                         uint4 cur0, uint4 cur1, int is_query, double c,
                                         const unsigned long long* __restrict__ tensor_absmax, const QuantOut& out) {
  // Maxima use monotonicity instead of per-element f64 compares: fl(|x| c) and the
  // correctly rounded fl(|x| / S_q) are non-decreasing in |x|, so the max of the
  // rounded values is the rounded max (the argument quantize.py's TENSOR path
  // already relies on).  For bf16 inputs max |x| is an integer max on the bit
  // patterns, which also flags Inf / NaN (magnitude >= 0x7F80).
  double xs[16];
  double amax;  // max |x| of this thread's 16 values (input precision, exact)
  bool bad;
  if constexpr (sizeof(T) == 2) {
    const uint32_t w[8] = {cur0.x, cur0.y, cur0.z, cur0.w, cur1.x, cur1.y, cur1.z, cur1.w};
    uint32_t mm = w[0] & 0x7FFF7FFFu;
#pragma unroll
    for (int i = 1; i < 8; ++i) mm = __vmaxu2(mm, w[i] & 0x7FFF7FFFu);
    const uint32_t m16 = max(mm & 0xFFFFu, mm >> 16);
    bad = m16 >= 0x7F80u;
    amax = static_cast<double>(__uint_as_float(m16 << 16));
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      xs[2 * i] = __uint_as_float(w[i] << 16);
      xs[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  } else {
    if (live) {
      Load16<T>::run(x + mat * mat_stride + row * row_stride + part * 16, xs);
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) xs[i] = 0.0;
    }
    bad = false;
    amax = 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      bad |= (static_cast<uint32_t>(__double2hiint(xs[i])) & 0x7FF00000u) == 0x7FF00000u;  // Inf / NaN
      amax = fmax(amax, fabs(xs[i]));
    }
  }
  if (out.nonfinite && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(out.nonfinite, 1u);

  // ---- group max -> S_q (quantize.py:98-106, 152-153), taken on max |x| before the prescale
  double g;
  if (GRAN == DMA_GRAN_TOKEN) {
    g = shfl_max(amax, tpr);
  } else if (GRAN == DMA_GRAN_BLOCK) {
    g = shfl_max(amax, 2);
  } else {
    g = __longlong_as_double(static_cast<long long>(tensor_absmax[mat]));
  }
  if (is_query) {
#pragma unroll
    for (int i = 0; i < 16; ++i) xs[i] = __dmul_rn(xs[i], c);  // quantize.py:149 (x * c)
    amax = __dmul_rn(amax, c);  // = max |x * c| (monotone rounding)
    g = __dmul_rn(g, c);
  }
  const double sq = g > 0.0 ? __ddiv_rn(g, 2688.0) : 1.0;
  const double ysq = __drcp_rn(sq);
  double xsc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) xsc[i] = qdiv<T>(xs[i], sq, ysq);  // quantize.py:154
  const double amax_sc = qdiv<T>(amax, sq, ysq);  // = max |x_scaled| of the 16 values

  // ---- 4-bit path (quantize.py:156-184)
  uint32_t packed[2] = {0u, 0u};
  uint32_t sc_low;
  if (NV) {
    const double bm = amax_sc;
    uint32_t code = bm > 0.0 ? e4m3_pos(__ddiv_rn(bm, 6.0)) : 0x38u;
    if (code == 0 && bm > 0.0) code = 0x01;  // floor at 2^-9 (quantize.py:164-167)
    const double sv = decode_e4m3(code);
    const double ysv = __drcp_rn(sv);
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      const double l0 = qdiv<T>(xsc[i], sv, ysv), l1 = qdiv<T>(xsc[i + 1], sv, ysv);
      uint32_t b = ptx::cvt_e2m1x2(rto_abs(l0), rto_abs(l1));
      b |= (neg_nonzero(l0) ? 0x08u : 0u) | (neg_nonzero(l1) ? 0x80u : 0u);
      packed[i >> 3] |= b << (4 * (i & 7));
    }
    sc_low = code;
  } else {
    const double bm = shfl_max(amax, 2);  // 32-column block = 2 lanes, single level on x_sm
    const int e = bm > 0.0 ? min(max(floor_log2_pos(bm) - 2, -127), 127) : -127;
    const double inv = pow2(-e);
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      const double l0 = xs[i] * inv, l1 = xs[i + 1] * inv;
      uint32_t b = ptx::cvt_e2m1x2(rto_abs(l0), rto_abs(l1));
      b |= (neg_nonzero(l0) ? 0x08u : 0u) | (neg_nonzero(l1) ? 0x80u : 0u);
      packed[i >> 3] |= b << (4 * (i & 7));
    }
    sc_low = static_cast<uint32_t>(e + 127);
  }

  // ---- 8-bit path (quantize.py:186-199)
  const double hm = shfl_max(amax_sc, 2);
  constexpr int kEmax = E5 ? 15 : 8;
  const int he = hm > 0.0 ? min(max(floor_log2_pos(hm) - kEmax, -127), 127) : -127;
  const double hinv = pow2(-he);
  uint32_t codes[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t w = 0;
#pragma unroll
    for (int i = 0; i < 4; i += 2) {
      const double h0 = xsc[4 * j + i] * hinv, h1 = xsc[4 * j + i + 1] * hinv;
      const float a = rto_abs(h0), b = rto_abs(h1);
      const uint32_t mag = E5 ? ptx::cvt_e5m2x2(a, b) : ptx::cvt_e4m3x2(a, b);
      uint32_t c0 = mag & 0xFF, c1 = (mag >> 8) & 0xFF;
      if (c0 && neg_nonzero(h0)) c0 |= 0x80;  // rounded-to-zero magnitudes stay +0
      if (c1 && neg_nonzero(h1)) c1 |= 0x80;
      w |= (c0 | (c1 << 8)) << (8 * i);
    }
    codes[j] = w;
  }
  const uint32_t sc_high = static_cast<uint32_t>(he + 127);
  if (!live) return;  // dead rows still take part in the shuffles above

  const int64_t rbase = mat * rows + row;
  // operand row of the codes / scale-factor atoms (permuted inside 128-row tiles for attn_pp)
  const int64_t orow = out.key_perm == 1 ? ((row & ~int64_t(127)) | perm_row(static_cast<int>(row & 127))) : row;
  const int64_t cbase = out.key_perm ? mat * out.rows_pad + orow : rbase;
  const int col0 = part * 16;
  if (out.packed_low)
    *reinterpret_cast<uint2*>(out.packed_low + cbase * (cols / 2) + col0 / 2) = make_uint2(packed[0], packed[1]);
  if (out.high_codes)
    *reinterpret_cast<uint4*>(out.high_codes + cbase * cols + col0) = make_uint4(codes[0], codes[1], codes[2], codes[3]);
  const int nsf_low = cols / (NV ? 16 : 32);
  const int chunks_low = (nsf_low + 3) >> 2;
  const int chunks_high = ((cols / 32) + 3) >> 2;
  const int64_t rtiles = out.rows_pad >> 7;
  const bool even = (part & 1) == 0;
  if (NV || even) {
    const int kb_low = NV ? part : (part >> 1);
    if (out.scales_low) out.scales_low[rbase * nsf_low + kb_low] = static_cast<uint8_t>(sc_low);
    if (out.sf_low_op) out.sf_low_op[sf_atom_offset(mat, orow, kb_low, rtiles, chunks_low)] = static_cast<uint8_t>(sc_low);
  }
  if (even) {
    const int kb = part >> 1;
    if (out.scales_high) out.scales_high[rbase * (cols / 32) + kb] = static_cast<uint8_t>(sc_high);
    if (out.sf_high_op) out.sf_high_op[sf_atom_offset(mat, orow, kb, rtiles, chunks_high)] = static_cast<uint8_t>(sc_high);
    if (GRAN == DMA_GRAN_BLOCK && out.quant_scale) out.quant_scale[rbase * (cols / 32) + kb] = sq;
  }
  if (part == 0) {
    if (GRAN == DMA_GRAN_TOKEN && out.quant_scale) out.quant_scale[rbase] = sq;
    if (GRAN == DMA_GRAN_TENSOR && out.quant_scale && row == 0) out.quant_scale[mat] = sq;
    if (GRAN != DMA_GRAN_BLOCK && out.qs_f32) {
      if (out.key_perm)
        out.qs_f32[(mat * (out.rows_pad >> 7) + (row >> 7)) * kSqkTile +
                   (out.key_perm == 1 ? perm_slot(static_cast<int>(row & 127)) : static_cast<int>(row & 127))] =
            static_cast<float>(sq);
      else
        out.qs_f32[mat * out.rows_pad + row] = static_cast<float>(sq);
    }
  }
}

// ------------------------------------------------------------------------
// Fast variant of q16_item (the one phase 1 and the fused kernel use): the per-row /
// per-block scale decisions stay exact float64 exactly as in q16_item, the per-element
// work runs in float32:
//   v_f = x * c * (1/S_q) [* (1/sv) | * 2^-e | * 2^-he]  (relative error < 8 * 2^-24
//         against the float64 value v the reference rounds, for rows whose S_q and blocks
//         whose max lie well inside the float32 range -- checked, else the float64 path);
//   the code of v is the code of every point of [v_f (1 - 2^-20), v_f (1 + 2^-20)] when
//   the two ends round to the same code (cvt RN is monotone), so the float32 codes are
//   taken when cvt(lo) == cvt(hi) for all 16 values of the thread, and the thread redoes
//   its 16 values in float64 (q16_item's arithmetic) otherwise -- near a rounding
//   midpoint, ~2^-17 of the elements.  Bit-exact either way.
// ------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void load16_f64(const T* __restrict__ x, int64_t off, uint4 cur0, uint4 cur1,
                                           double (&xs)[16]) {
  if constexpr (sizeof(T) == 2) {
    const uint32_t w[8] = {cur0.x, cur0.y, cur0.z, cur0.w, cur1.x, cur1.y, cur1.z, cur1.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      xs[2 * i] = __uint_as_float(w[i] << 16);
      xs[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  } else {
    Load16<T>::run(x + off, xs);
  }
}

// float64 per-element codes of one thread's 16 values (q16_item's arithmetic), given the
// row / block scale decisions: the fallback of q16_item_fast (rare; kept out of line so the
// fast path's register allocation does not carry the float64 arrays)
template <typename T, bool NV, bool E5>
__device__ __noinline__ void q16_codes_f64(const T* __restrict__ x, int64_t off, uint4 cur0, uint4 cur1, bool live,
                                           int is_query, double c, double sq, double ysq, double sv, double ysv,
                                           double inv, double hinv, uint32_t (&packed)[2], uint32_t (&codes)[4]) {
  double xs[16];
  if (live) {
    load16_f64<T>(x, off, cur0, cur1, xs);
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) xs[i] = 0.0;
  }
  if (is_query) {
#pragma unroll
    for (int i = 0; i < 16; ++i) xs[i] = __dmul_rn(xs[i], c);  // quantize.py:149 (x * c)
  }
  double xsc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) xsc[i] = qdiv<T>(xs[i], sq, ysq);  // quantize.py:154
  packed[0] = packed[1] = 0u;
#pragma unroll
  for (int i = 0; i < 16; i += 2) {
    double l0, l1;
    if (NV) {
      l0 = qdiv<T>(xsc[i], sv, ysv);
      l1 = qdiv<T>(xsc[i + 1], sv, ysv);
    } else {
      l0 = xs[i] * inv;
      l1 = xs[i + 1] * inv;
    }
    uint32_t b = ptx::cvt_e2m1x2(rto_abs(l0), rto_abs(l1));
    b |= (neg_nonzero(l0) ? 0x08u : 0u) | (neg_nonzero(l1) ? 0x80u : 0u);
    packed[i >> 3] |= b << (4 * (i & 7));
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t w = 0;
#pragma unroll
    for (int i = 0; i < 4; i += 2) {
      const double h0 = xsc[4 * j + i] * hinv, h1 = xsc[4 * j + i + 1] * hinv;
      const float a = rto_abs(h0), b = rto_abs(h1);
      const uint32_t mag = E5 ? ptx::cvt_e5m2x2(a, b) : ptx::cvt_e4m3x2(a, b);
      uint32_t c0 = mag & 0xFF, c1 = (mag >> 8) & 0xFF;
      if (c0 && neg_nonzero(h0)) c0 |= 0x80;  // rounded-to-zero magnitudes stay +0
      if (c1 && neg_nonzero(h1)) c1 |= 0x80;
      w |= (c0 | (c1 << 8)) << (8 * i);
    }
    codes[j] = w;
  }
}

template <typename T, bool NV, bool E5, int GRAN>
__device__ __forceinline__ void q16_item_fast(const T* __restrict__ x, int64_t mat_stride, int64_t row_stride,
                                              int64_t mat, int64_t rows, int cols, int64_t row, bool live, int part,
                                              int tpr, int lane, uint4 cur0, uint4 cur1, int is_query, double c,
                                              const unsigned long long* __restrict__ tensor_absmax,
                                              const QuantOut& out) {
  const int64_t off = mat * mat_stride + row * row_stride + part * 16;
  // ---- this thread's 16 inputs as float32 (exact for bf16 / f32) and max |x| (exact)
  float xf[16];
  double amax;
  bool bad;
  bool in_f32 = true;  // every input exactly representable in float32
  if constexpr (sizeof(T) == 2) {
    const uint32_t w[8] = {cur0.x, cur0.y, cur0.z, cur0.w, cur1.x, cur1.y, cur1.z, cur1.w};
    uint32_t mm = w[0] & 0x7FFF7FFFu;
#pragma unroll
    for (int i = 1; i < 8; ++i) mm = __vmaxu2(mm, w[i] & 0x7FFF7FFFu);
    const uint32_t m16 = max(mm & 0xFFFFu, mm >> 16);
    bad = m16 >= 0x7F80u;
    amax = static_cast<double>(__uint_as_float(m16 << 16));
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      xf[2 * i] = __uint_as_float(w[i] << 16);
      xf[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  } else {
    double xs[16];
    if (live) {
      Load16<T>::run(x + off, xs);
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) xs[i] = 0.0;
    }
    bad = false;
    amax = 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      bad |= (static_cast<uint32_t>(__double2hiint(xs[i])) & 0x7FF00000u) == 0x7FF00000u;  // Inf / NaN
      amax = fmax(amax, fabs(xs[i]));
      xf[i] = static_cast<float>(xs[i]);
      if constexpr (sizeof(T) == 8) in_f32 &= static_cast<double>(xf[i]) == xs[i];
    }
  }
  if (out.nonfinite && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(out.nonfinite, 1u);

  // ---- scale decisions in float64, exactly as q16_item (quantize.py:98-106, 152-199).
  // The lane maxima are taken on the magnitudes' float32 bit patterns (exact and monotone
  // for non-negative floats; one SHFL per step instead of a double's two) and the block
  // maxima of x_scaled from the block maximum of |x| (x -> x c -> x / S_q are monotone
  // roundings), so no double is shuffled for bf16 / f32 inputs.
  double g, amax2;  // amax2: max |x| over the 32-column block (2 lanes)
  if constexpr (sizeof(T) <= 4) {
    const uint32_t mb = __float_as_uint(static_cast<float>(amax));
    const uint32_t b2 = max(mb, __shfl_xor_sync(0xffffffffu, mb, 1));
    uint32_t gb = b2;
    if (GRAN == DMA_GRAN_TOKEN)
      for (int o = 2; o < tpr; o <<= 1) gb = max(gb, __shfl_xor_sync(0xffffffffu, gb, o));
    amax2 = static_cast<double>(__uint_as_float(b2));
    g = GRAN == DMA_GRAN_TENSOR ? __longlong_as_double(static_cast<long long>(tensor_absmax[mat]))
                                : static_cast<double>(__uint_as_float(gb));
  } else {
    amax2 = shfl_max(amax, 2);
    if (GRAN == DMA_GRAN_TOKEN) {
      g = shfl_max(amax2, tpr);
    } else if (GRAN == DMA_GRAN_BLOCK) {
      g = amax2;
    } else {
      g = __longlong_as_double(static_cast<long long>(tensor_absmax[mat]));
    }
  }
  if (is_query) {
    amax = __dmul_rn(amax, c);
    amax2 = __dmul_rn(amax2, c);
    g = __dmul_rn(g, c);
  }
  const double sq = g > 0.0 ? qdiv<T>(g, 2688.0, 1.0 / 2688.0) : 1.0;
  const double ysq = __drcp_rn(sq);
  const double amax_sc = qdiv<T>(amax, sq, ysq);
  uint32_t sc_low;
  double sv = 1.0, ysv = 1.0, inv = 1.0;
  if (NV) {
    const double bm = amax_sc;
    uint32_t code = bm > 0.0 ? e4m3_pos(qdiv<T>(bm, 6.0, 1.0 / 6.0)) : 0x38u;
    if (code == 0 && bm > 0.0) code = 0x01;  // floor at 2^-9 (quantize.py:164-167)
    sv = decode_e4m3(code);
    ysv = __drcp_rn(sv);
    sc_low = code;
  } else {
    const double bm = amax2;  // 32-column block = 2 lanes, single level on x_sm
    const int e = bm > 0.0 ? min(max(floor_log2_pos(bm) - 2, -127), 127) : -127;
    inv = pow2(-e);
    sc_low = static_cast<uint32_t>(e + 127);
  }
  const double hm = qdiv<T>(amax2, sq, ysq);  // = the block max of |x_scaled|
  constexpr int kEmax = E5 ? 15 : 8;
  const int he = hm > 0.0 ? min(max(floor_log2_pos(hm) - kEmax, -127), 127) : -127;
  const double hinv = pow2(-he);
  const uint32_t sc_high = static_cast<uint32_t>(he + 127);

  // ---- float32 fast path (guards: every factor and this thread's |x| range well inside float32)
  const double lfac = NV ? ysv : inv;
  const bool guard = in_f32 && sq >= 0x1p-100 && sq <= 0x1p+100 && (amax == 0.0 || (amax >= 0x1p-100 && amax <= 0x1p+100)) &&
                     lfac >= 0x1p-120 && lfac <= 0x1p+120 && hinv >= 0x1p-120 && hinv <= 0x1p+120;
  uint32_t packed[2] = {0u, 0u}, codes[4] = {0u, 0u, 0u, 0u};
  bool ok = guard;
  uint32_t fl = 0u;  // elements whose float32 interval straddles a rounding boundary
  if (guard) {
    const float cf = is_query ? static_cast<float>(c) : 1.0f;
    const float rsq = static_cast<float>(ysq);
    const float lf = static_cast<float>(lfac), hf = static_cast<float>(hinv);
    constexpr float kD = 0x1p-20f;
    uint32_t d4acc[2] = {0u, 0u}, d8acc[4] = {0u, 0u, 0u, 0u};  // codes of the interval ends, XORed
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      // x_sm (Q: x * c), x_scaled = x_sm / S_q.  The +0 addend of the first step turns an
      // input -0 into +0 (the reference's v < 0 tests see -0.0 as non-negative); later steps
      // are plain products, so a negative value that underflows keeps its sign (-0), as the
      // reference's negative nonzero float64 value does
      const float2 xsm = __ffma2_rn(make_float2(xf[i], xf[i + 1]), make_float2(cf, cf), make_float2(0.f, 0.f));
      const float2 xsc = __fmul2_rn(xsm, make_float2(rsq, rsq));
      // 4-bit: NVFP4 x_scaled / sv, MXFP4 x_sm * 2^-e
      const float2 l = NV ? __fmul2_rn(xsc, make_float2(lf, lf)) : __fmul2_rn(xsm, make_float2(lf, lf));
      const float2 lhi = __ffma2_rn(l, make_float2(kD, kD), l), llo = __ffma2_rn(l, make_float2(-kD, -kD), l);
      // signed conversions: RN is symmetric, and cvt keeps the sign of a negative value that
      // rounds to zero (E2M1 -0 = 0x8: the reference's sign rule for the 4-bit codes)
      const uint32_t ma = ptx::cvt_e2m1x2(lhi.x, lhi.y), mb = ptx::cvt_e2m1x2(llo.x, llo.y);
      packed[i >> 3] |= ma << (4 * (i & 7));
      // 8-bit: x_scaled * 2^-he
      const float2 h = __fmul2_rn(xsc, make_float2(hf, hf));
      const float2 hhi = __ffma2_rn(h, make_float2(kD, kD), h), hlo = __ffma2_rn(h, make_float2(-kD, -kD), h);
      const uint32_t ha = E5 ? ptx::cvt_e5m2x2(hhi.x, hhi.y) : ptx::cvt_e4m3x2(hhi.x, hhi.y);
      const uint32_t hb = E5 ? ptx::cvt_e5m2x2(hlo.x, hlo.y) : ptx::cvt_e4m3x2(hlo.x, hlo.y);
      // rounded-to-zero magnitudes stay +0 (-0 = 0x80 -> 0x00): keep bit 7 of a byte only when
      // its magnitude is >= 1 (bit 7 of magnitude + 0x7F; magnitudes <= 0x7E: no carry)
      codes[i >> 2] |= (ha & (((ha & 0x7F7Fu) + 0x7F7Fu) | 0x7F7Fu)) << (8 * (i & 3));
      d4acc[i >> 3] |= (ma ^ mb) << (4 * (i & 7));
      d8acc[i >> 2] |= (ha ^ hb) << (8 * (i & 3));
    }
    if ((d4acc[0] | d4acc[1] | d8acc[0] | d8acc[1] | d8acc[2] | d8acc[3]) != 0u) {
      // element flags: nonzero nibbles of d4acc, nonzero bytes of d8acc, gathered to bits 0..15
#pragma unroll
      for (int w = 0; w < 2; ++w) {
        uint32_t n = d4acc[w];
        n |= n >> 1;
        n |= n >> 2;
        n &= 0x11111111u;
        n = (n | (n >> 3)) & 0x03030303u;
        n = (n | (n >> 6)) & 0x000F000Fu;
        n = (n | (n >> 12)) & 0xFFu;
        fl |= n << (8 * w);
      }
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const uint32_t b = __vcmpne4(d8acc[w], 0u) & 0x01010101u;
        fl |= (((b * 0x01020408u) >> 24) & 0xFu) << (4 * w);
      }
    }
  }
  {
    // the flagged elements (~1-2 per row: the row maximum lands exactly on an E4M3 midpoint
    // after x / S_q = 2688) in float64, one per lane per round
    while (__any_sync(0xffffffffu, fl != 0u)) {
      if (fl) {
        const int j = __ffs(fl) - 1;
        fl &= fl - 1u;
        double xj;
        if constexpr (sizeof(T) == 2) {
          const uint32_t w = (j >> 1) < 4 ? ((j >> 1) == 0 ? cur0.x : (j >> 1) == 1 ? cur0.y : (j >> 1) == 2 ? cur0.z : cur0.w)
                                         : ((j >> 1) == 4 ? cur1.x : (j >> 1) == 5 ? cur1.y : (j >> 1) == 6 ? cur1.z : cur1.w);
          xj = __uint_as_float((j & 1) ? (w & 0xFFFF0000u) : (w << 16));
        } else {
          xj = static_cast<double>(x[off + j]);
        }
        const double xs = is_query ? __dmul_rn(xj, c) : xj;  // quantize.py:149
        const double xsc = qdiv<T>(xs, sq, ysq);               // quantize.py:154
        const double lv = NV ? qdiv<T>(xsc, sv, ysv) : xs * inv;
        const uint32_t lc = (ptx::cvt_e2m1x2(rto_abs(lv), 0.f) & 0xFu) | (neg_nonzero(lv) ? 0x8u : 0u);
        const double hv = xsc * hinv;
        const float ha = rto_abs(hv);
        uint32_t hc = (E5 ? ptx::cvt_e5m2x2(ha, 0.f) : ptx::cvt_e4m3x2(ha, 0.f)) & 0xFFu;
        if (hc && neg_nonzero(hv)) hc |= 0x80u;
        const uint32_t s4 = 4u * (j & 7), s8 = 8u * (j & 3);
        if (j < 8) packed[0] = (packed[0] & ~(0xFu << s4)) | (lc << s4);
        else packed[1] = (packed[1] & ~(0xFu << s4)) | (lc << s4);
        const int cw = j >> 2;
        const uint32_t m8 = ~(0xFFu << s8), v8 = hc << s8;
        codes[0] = cw == 0 ? ((codes[0] & m8) | v8) : codes[0];
        codes[1] = cw == 1 ? ((codes[1] & m8) | v8) : codes[1];
        codes[2] = cw == 2 ? ((codes[2] & m8) | v8) : codes[2];
        codes[3] = cw == 3 ? ((codes[3] & m8) | v8) : codes[3];
      }
    }
  }
  if (!ok) q16_codes_f64<T, NV, E5>(x, off, cur0, cur1, live, is_query, c, sq, ysq, sv, ysv, inv, hinv, packed, codes);
  if (!live) return;

  // ---- stores (as q16_item)
  const int64_t rbase = mat * rows + row;
  const int64_t orow = out.key_perm == 1 ? ((row & ~int64_t(127)) | perm_row(static_cast<int>(row & 127))) : row;
  const int64_t cbase = out.key_perm ? mat * out.rows_pad + orow : rbase;
  const int col0 = part * 16;
  if (out.packed_low)
    *reinterpret_cast<uint2*>(out.packed_low + cbase * (cols / 2) + col0 / 2) = make_uint2(packed[0], packed[1]);
  if (out.high_codes)
    *reinterpret_cast<uint4*>(out.high_codes + cbase * cols + col0) = make_uint4(codes[0], codes[1], codes[2], codes[3]);
  const int nsf_low = cols / (NV ? 16 : 32);
  const int chunks_low = (nsf_low + 3) >> 2;
  const int chunks_high = ((cols / 32) + 3) >> 2;
  const int64_t rtiles = out.rows_pad >> 7;
  const bool even = (part & 1) == 0;
  if (NV || even) {
    const int kb_low = NV ? part : (part >> 1);
    if (out.scales_low) out.scales_low[rbase * nsf_low + kb_low] = static_cast<uint8_t>(sc_low);
    if (out.sf_low_op) out.sf_low_op[sf_atom_offset(mat, orow, kb_low, rtiles, chunks_low)] = static_cast<uint8_t>(sc_low);
  }
  if (even) {
    const int kb = part >> 1;
    if (out.scales_high) out.scales_high[rbase * (cols / 32) + kb] = static_cast<uint8_t>(sc_high);
    if (out.sf_high_op) out.sf_high_op[sf_atom_offset(mat, orow, kb, rtiles, chunks_high)] = static_cast<uint8_t>(sc_high);
    if (GRAN == DMA_GRAN_BLOCK && out.quant_scale) out.quant_scale[rbase * (cols / 32) + kb] = sq;
  }
  if (part == 0) {
    if (GRAN == DMA_GRAN_TOKEN && out.quant_scale) out.quant_scale[rbase] = sq;
    if (GRAN == DMA_GRAN_TENSOR && out.quant_scale && row == 0) out.quant_scale[mat] = sq;
    if (GRAN != DMA_GRAN_BLOCK && out.qs_f32) {
      if (out.key_perm)
        out.qs_f32[(mat * (out.rows_pad >> 7) + (row >> 7)) * kSqkTile +
                   (out.key_perm == 1 ? perm_slot(static_cast<int>(row & 127)) : static_cast<int>(row & 127))] =
            static_cast<float>(sq);
      else
        out.qs_f32[mat * out.rows_pad + row] = static_cast<float>(sq);
    }
  }
}

// ------------------------------------------------------------------------
// bf16 phase-1 variant with 32 columns per thread (one MX block = two NVFP4 blocks), so the
// per-thread float64 scale decisions -- the instruction-bound part of q16_item_fast -- cover
// twice the elements.  Same decisions and codes as q16_item_fast / q16_item:
//   * float32 fast path with the +-2^-20 interval on every converted value; a pair of columns
//     whose interval ends give different codes (an exact or near-exact rounding tie: x / S_q
//     is a short number whenever S_q's mantissa shares factors with 2688 = 21 * 2^7, ~2.5 per
//     128-column row) is flagged;
//   * flagged pairs (or all 16 when the float32 guard fails) are recomputed in float64 one
//     pair per lane per round and written over the fast codes with 1- / 2-byte stores after
//     the row's vector stores (same thread, same address: program order);
//   * sign rules: E2M1 keeps -0 for a negative value that rounds to zero, FP8 maps every zero
//     magnitude to +0 (the word-wise fix after packing).
// ------------------------------------------------------------------------
constexpr double kRcp2688 = 1.0 / 2688.0;  // RN(1/2688): Markstein division by the constant
constexpr double kRcp6 = 1.0 / 6.0;

__device__ __forceinline__ uint32_t fp8_posz(uint32_t w) {  // bytes 0x80 -> 0x00
  const uint32_t b = (w & 0x7F7F7F7Fu) + 0x7F7F7F7Fu;      // bit 7 set iff magnitude != 0
  return w & (b | 0x7F7F7F7Fu);
}

template <bool NV, bool E5, int GRAN>
__device__ __forceinline__ void q32_item_bf16(const __nv_bfloat16* __restrict__ x, int64_t mat_stride,
                                              int64_t row_stride, int64_t mat, int64_t rows, int cols, int64_t row,
                                              bool live, int part, int tpr, int lane, const uint32_t (&w)[16],
                                              int is_query, double c,
                                              const unsigned long long* __restrict__ tensor_absmax,
                                              const QuantOut& out, const double* rcp_tab) {
  // ---- maxima of |x| per 16-column half (the NVFP4 blocks) and per thread (the MX block)
  uint32_t mm0 = w[0] & 0x7FFF7FFFu, mm1 = w[8] & 0x7FFF7FFFu;
#pragma unroll
  for (int i = 1; i < 8; ++i) {
    mm0 = __vmaxu2(mm0, w[i] & 0x7FFF7FFFu);
    mm1 = __vmaxu2(mm1, w[8 + i] & 0x7FFF7FFFu);
  }
  const uint32_t h0 = max(mm0 & 0xFFFFu, mm0 >> 16), h1 = max(mm1 & 0xFFFFu, mm1 >> 16);
  const uint32_t hb = max(h0, h1);
  if (out.nonfinite && __any_sync(0xffffffffu, hb >= 0x7F80u) && lane == 0) atomicOr(out.nonfinite, 1u);
  double a0 = static_cast<double>(__uint_as_float(h0 << 16));
  double a1 = static_cast<double>(__uint_as_float(h1 << 16));
  double amax2 = static_cast<double>(__uint_as_float(hb << 16));
  double g;
  if (GRAN == DMA_GRAN_TOKEN) {
    uint32_t gb = hb;
    for (int o = 1; o < tpr; o <<= 1) gb = max(gb, __shfl_xor_sync(0xffffffffu, gb, o));
    g = static_cast<double>(__uint_as_float(gb << 16));
  } else if (GRAN == DMA_GRAN_BLOCK) {
    g = amax2;
  } else {
    g = __longlong_as_double(static_cast<long long>(tensor_absmax[mat]));
  }
  if (is_query) {  // quantize.py:149; monotone rounding, so the max of x c is (max |x|) c
    a0 = __dmul_rn(a0, c);
    a1 = __dmul_rn(a1, c);
    amax2 = __dmul_rn(amax2, c);
    g = __dmul_rn(g, c);
  }
  // ---- scale decisions in float64 (quantize.py:98-106, 152-199)
  const double sq = g > 0.0 ? mk_div(g, 2688.0, kRcp2688) : 1.0;
  const double ysq = __drcp_rn(sq);
  uint32_t sc_low;  // NV: the two E4M3 block scales (byte 0 = columns 0-15); MX: E8M0
  double sv0 = 1.0, ysv0 = 1.0, sv1 = 1.0, ysv1 = 1.0, inv = 1.0;
  if (NV) {
    auto nv_scale = [&](double am, double& sv, double& ysv) -> uint32_t {
      const double bm = mk_div(am, sq, ysq);  // block max of |x_scaled|
      uint32_t code = e4m3_pos(mk_div(bm, 6.0, kRcp6));
      code = bm > 0.0 ? max(code, 1u) : 0x38u;  // floor at 2^-9 (quantize.py:164-167)
      // positive E4M3 value and its reciprocal: (1 + m/8) 2^(e-7) / m 2^-9, with
      // 1/sv = RN(1/(1 + m/8)) 2^(7-e) / RN(1/m) 2^9 from the table (exact power-of-two scaling)
      const int e = static_cast<int>(code >> 3), m = static_cast<int>(code & 7u);
      sv = e ? __hiloint2double(((e + 1016) << 20) | (m << 17), 0) : m * 0x1p-9;
      ysv = rcp_tab[e ? m : 8 + m] * pow2(e ? 7 - e : 9);
      return code;
    };
    sc_low = nv_scale(a0, sv0, ysv0);
    sc_low |= nv_scale(a1, sv1, ysv1) << 8;
  } else {
    const int e = amax2 > 0.0 ? min(max(floor_log2_pos(amax2) - 2, -127), 127) : -127;
    inv = pow2(-e);
    sc_low = static_cast<uint32_t>(e + 127);
  }
  const double hm = mk_div(amax2, sq, ysq);  // block max of |x_scaled|
  constexpr int kEmax = E5 ? 15 : 8;
  const int he = hm > 0.0 ? min(max(floor_log2_pos(hm) - kEmax, -127), 127) : -127;
  const double hinv = pow2(-he);
  const uint32_t sc_high = static_cast<uint32_t>(he + 127);

  // ---- float32 fast path
  const double lfac0 = NV ? ysv0 : inv, lfac1 = NV ? ysv1 : inv;
  const bool guard = sq >= 0x1p-100 && sq <= 0x1p+100 && (amax2 == 0.0 || (amax2 >= 0x1p-100 && amax2 <= 0x1p+100)) &&
                     lfac0 >= 0x1p-120 && lfac0 <= 0x1p+120 && lfac1 >= 0x1p-120 && lfac1 <= 0x1p+120 &&
                     hinv >= 0x1p-120 && hinv <= 0x1p+120;
  uint32_t packed[4], codes[8];
  uint32_t fl = 0xFFFFu;  // pairs to redo in float64
  {
    const float cf = is_query ? static_cast<float>(c) : 1.0f;
    const float rsq = static_cast<float>(ysq);
    const float lf0 = static_cast<float>(lfac0), lf1 = static_cast<float>(lfac1), hf = static_cast<float>(hinv);
    constexpr float kD = 0x1p-20f;
    uint32_t lb[16], hh[16], diff = 0u;
#pragma unroll
    for (int p = 0; p < 16; ++p) {
      const float lf = p < 8 ? lf0 : lf1;
      const float2 xv = make_float2(__uint_as_float(w[p] << 16), __uint_as_float(w[p] & 0xFFFF0000u));
      // +0 addend: an input -0 becomes +0 (the reference's v < 0 tests see -0.0 as non-negative)
      const float2 xsm = __ffma2_rn(xv, make_float2(cf, cf), make_float2(0.f, 0.f));
      const float2 xsc = __fmul2_rn(xsm, make_float2(rsq, rsq));
      const float2 l = NV ? __fmul2_rn(xsc, make_float2(lf, lf)) : __fmul2_rn(xsm, make_float2(lf, lf));
      const float2 lhi = __ffma2_rn(l, make_float2(kD, kD), l), llo = __ffma2_rn(l, make_float2(-kD, -kD), l);
      const uint32_t ma = ptx::cvt_e2m1x2(lhi.x, lhi.y), mb = ptx::cvt_e2m1x2(llo.x, llo.y);
      const float2 h = __fmul2_rn(xsc, make_float2(hf, hf));
      const float2 hhi = __ffma2_rn(h, make_float2(kD, kD), h), hlo = __ffma2_rn(h, make_float2(-kD, -kD), h);
      const uint32_t ha = E5 ? ptx::cvt_e5m2x2(hhi.x, hhi.y) : ptx::cvt_e4m3x2(hhi.x, hhi.y);
      const uint32_t hb2 = E5 ? ptx::cvt_e5m2x2(hlo.x, hlo.y) : ptx::cvt_e4m3x2(hlo.x, hlo.y);
      lb[p] = ma;
      hh[p] = ha;
      diff |= ((ma ^ mb) | (ha ^ hb2)) != 0u ? (1u << p) : 0u;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      packed[k] = lb[4 * k] | (lb[4 * k + 1] << 8) | (lb[4 * k + 2] << 16) | (lb[4 * k + 3] << 24);
#pragma unroll
    for (int k = 0; k < 8; ++k) codes[k] = fp8_posz(hh[2 * k] | (hh[2 * k + 1] << 16));
    if (guard) fl = diff;
  }
  if (!live) fl = 0u;

  // ---- stores (as q16_item_fast)
  const int64_t rbase = mat * rows + row;
  const int64_t orow = out.key_perm == 1 ? ((row & ~int64_t(127)) | perm_row(static_cast<int>(row & 127))) : row;
  const int64_t cbase = out.key_perm ? mat * out.rows_pad + orow : rbase;
  const int col0 = part * 32;
  if (live) {
    if (out.packed_low)
      *reinterpret_cast<uint4*>(out.packed_low + cbase * (cols / 2) + col0 / 2) =
          make_uint4(packed[0], packed[1], packed[2], packed[3]);
    if (out.high_codes) {
      uint4* hp = reinterpret_cast<uint4*>(out.high_codes + cbase * cols + col0);
      hp[0] = make_uint4(codes[0], codes[1], codes[2], codes[3]);
      hp[1] = make_uint4(codes[4], codes[5], codes[6], codes[7]);
    }
    const int nsf_low = cols / (NV ? 16 : 32);
    const int chunks_low = (nsf_low + 3) >> 2;
    const int chunks_high = ((cols / 32) + 3) >> 2;
    const int64_t rtiles = out.rows_pad >> 7;
    if (NV) {  // two adjacent scale bytes (block 2 part even: same 4-block chunk)
      if (out.scales_low)
        *reinterpret_cast<uint16_t*>(out.scales_low + rbase * nsf_low + 2 * part) = static_cast<uint16_t>(sc_low);
      if (out.sf_low_op)
        *reinterpret_cast<uint16_t*>(out.sf_low_op + sf_atom_offset(mat, orow, 2 * part, rtiles, chunks_low)) =
            static_cast<uint16_t>(sc_low);
    } else {
      if (out.scales_low) out.scales_low[rbase * nsf_low + part] = static_cast<uint8_t>(sc_low);
      if (out.sf_low_op) out.sf_low_op[sf_atom_offset(mat, orow, part, rtiles, chunks_low)] = static_cast<uint8_t>(sc_low);
    }
    if (out.scales_high) out.scales_high[rbase * (cols / 32) + part] = static_cast<uint8_t>(sc_high);
    if (out.sf_high_op) out.sf_high_op[sf_atom_offset(mat, orow, part, rtiles, chunks_high)] = static_cast<uint8_t>(sc_high);
    if (GRAN == DMA_GRAN_BLOCK && out.quant_scale) out.quant_scale[rbase * (cols / 32) + part] = sq;
    if (part == 0) {
      if (GRAN == DMA_GRAN_TOKEN && out.quant_scale) out.quant_scale[rbase] = sq;
      if (GRAN == DMA_GRAN_TENSOR && out.quant_scale && row == 0) out.quant_scale[mat] = sq;
      if (GRAN != DMA_GRAN_BLOCK && out.qs_f32) {
        if (out.key_perm)
          out.qs_f32[(mat * (out.rows_pad >> 7) + (row >> 7)) * kSqkTile +
                     (out.key_perm == 1 ? perm_slot(static_cast<int>(row & 127)) : static_cast<int>(row & 127))] =
              static_cast<float>(sq);
        else
          out.qs_f32[mat * out.rows_pad + row] = static_cast<float>(sq);
      }
    }
  }

  // ---- flagged pairs in float64 (q16_item's arithmetic), compacted over the warp: every lane
  // redoes one flagged (lane, pair) item per round with its owner's scales (shuffled), writing
  // over the vector stores above (ordered after them by __syncwarp)
  const uint32_t cnt = __popc(fl);
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  if (total == 0) return;
  __syncwarp();  // the vector stores of every lane before any lane's corrections
  const int64_t xoff = mat * mat_stride + row * row_stride + col0;
  const uint32_t base = incl - cnt;
  for (uint32_t chunk = 0; chunk < total; chunk += 32) {
    // worker lane k takes item chunk + k: owner = the lane whose [base, incl) holds it (binary
    // search on the inclusive counts), pair = the (item - base)-th set bit of the owner's mask
    const uint32_t k = chunk + lane;
    int lo = 0;
#pragma unroll
    for (int step = 16; step; step >>= 1) {
      const uint32_t v = __shfl_sync(0xffffffffu, incl, lo + step - 1);
      if (v <= k) lo += step;
    }
    const bool work = k < total;
    const int src = work ? lo : lane;
    uint32_t m = __shfl_sync(0xffffffffu, fl, src);
    uint32_t r = k - __shfl_sync(0xffffffffu, base, src);  // rank of the pair in the owner's mask
    int p = 0;
#pragma unroll
    for (int w = 8; w; w >>= 1) {  // select the r-th set bit of the 16-bit mask
      const uint32_t c = __popc(m & ((1u << w) - 1u));
      if (r >= c) {
        r -= c;
        m >>= w;
        p += w;
      }
    }
    const double psq = __shfl_sync(0xffffffffu, sq, src), pysq = __shfl_sync(0xffffffffu, ysq, src);
    const double psv0 = __shfl_sync(0xffffffffu, sv0, src), pysv0 = __shfl_sync(0xffffffffu, ysv0, src);
    const double psv1 = __shfl_sync(0xffffffffu, sv1, src), pysv1 = __shfl_sync(0xffffffffu, ysv1, src);
    const double pinv = __shfl_sync(0xffffffffu, inv, src), phinv = __shfl_sync(0xffffffffu, hinv, src);
    const int64_t pxoff = __shfl_sync(0xffffffffu, xoff, src), pcbase = __shfl_sync(0xffffffffu, cbase, src);
    if (work) {
      const int pcol0 = (src & (tpr - 1)) * 32;
      const uint32_t wp = __ldg(reinterpret_cast<const uint32_t*>(x + pxoff) + p);
      const double svp = p < 8 ? psv0 : psv1, ysvp = p < 8 ? pysv0 : pysv1;
      uint32_t lc = 0u, hc = 0u;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double xv = __uint_as_float(e ? (wp & 0xFFFF0000u) : (wp << 16));
        const double xs = is_query ? __dmul_rn(xv, c) : xv;  // quantize.py:149
        const double xsc = mk_div(xs, psq, pysq);              // quantize.py:154
        const double lv = NV ? mk_div(xsc, svp, ysvp) : xs * pinv;
        const uint32_t l4 = (ptx::cvt_e2m1x2(rto_abs(lv), 0.f) & 0xFu) | (neg_nonzero(lv) ? 0x8u : 0u);
        const double hv = xsc * phinv;
        const float ha = rto_abs(hv);
        uint32_t h8 = (E5 ? ptx::cvt_e5m2x2(ha, 0.f) : ptx::cvt_e4m3x2(ha, 0.f)) & 0xFFu;
        if (h8 && neg_nonzero(hv)) h8 |= 0x80u;
        lc |= l4 << (4 * e);
        hc |= h8 << (8 * e);
      }
      if (out.packed_low) out.packed_low[pcbase * (cols / 2) + pcol0 / 2 + p] = static_cast<uint8_t>(lc);
      if (out.high_codes)
        *reinterpret_cast<uint16_t*>(out.high_codes + pcbase * cols + pcol0 + 2 * p) = static_cast<uint16_t>(hc);
    }
  }
}

#ifndef DMA_QUANT_F64
#define DMA_QUANT_F64 0  // 1: phase 1 runs q16_item (all float64) instead of q16_item_fast
#endif

// bf16 phase 1 with q32_item_bf16: work item = (matrix, block of 256 / tpr rows), tpr =
// cols / 32 threads per row; grid-stride like quant16_kernel, next item's 64 input bytes
// prefetched.
#ifndef DMA_Q32_MINB
#define DMA_Q32_MINB 3  // min resident CTAs per SM for quant32_bf16_kernel (register cap)
#endif
template <bool NV, bool E5, int GRAN>
__global__ void __launch_bounds__(256, DMA_Q32_MINB) quant32_bf16_kernel(const __nv_bfloat16* __restrict__ x, int64_t n_mat,
                                                           int64_t rows, int cols, int64_t mat_stride,
                                                           int64_t row_stride, int is_query, double c,
                                                           const unsigned long long* __restrict__ tensor_absmax,
                                                           QuantOut out) {
  const int lg_tpr = __ffs(cols >> 5) - 1;
  const int tpr = 1 << lg_tpr;
  const int lane = threadIdx.x & 31;
  const int part = threadIdx.x & (tpr - 1);
  const int rpb = 256 >> lg_tpr;
  const int64_t nbx = (rows + rpb - 1) / rpb;
  const int rsub = threadIdx.x >> lg_tpr;
  __shared__ double rcp_tab[16];  // RN(1/(1 + m/8)) for m < 8, RN(1/(m - 8)) for m > 8
  if (threadIdx.x < 16) rcp_tab[threadIdx.x] = threadIdx.x < 8 ? 8.0 / (8 + threadIdx.x) : 1.0 / (threadIdx.x - 8);
  __syncthreads();
  uint32_t pf[16];
  auto fetch = [&](int64_t m, int64_t b) {
    const int64_t r = b * rpb + rsub;
    if (m < n_mat && r < rows) {
      const uint4* src = reinterpret_cast<const uint4*>(x + m * mat_stride + r * row_stride + part * 32);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint4 v = __ldg(src + k);
        pf[4 * k] = v.x; pf[4 * k + 1] = v.y; pf[4 * k + 2] = v.z; pf[4 * k + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < 16; ++k) pf[k] = 0u;
    }
  };
  ptx::pdl_launch_dependents();
  fetch(blockIdx.y, blockIdx.x);
  for (int64_t mat = blockIdx.y; mat < n_mat; mat += gridDim.y) {
    for (int64_t bx = blockIdx.x; bx < nbx; bx += gridDim.x) {
      const int64_t row = bx * rpb + rsub;
      const bool live = row < rows;
      uint32_t cur[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) cur[k] = pf[k];
      {
        int64_t nb = bx + gridDim.x, nm = mat;
        if (nb >= nbx) {
          nb = blockIdx.x;
          nm = mat + gridDim.y;
        }
        fetch(nm, nb);
      }
      if (__all_sync(0xffffffffu, !live)) continue;
      q32_item_bf16<NV, E5, GRAN>(x, mat_stride, row_stride, mat, rows, cols, row, live, part, tpr, lane, cur,
                                  is_query, c, tensor_absmax, out, rcp_tab);
    }
  }
  // PDL chain (forward's phase 1: Q, K, V kernels overlap; the attention kernel waits for the
  // last one): this grid completes only after the previous kernel in the stream
  ptx::pdl_wait();
}

template <typename T, bool NV, bool E5, int GRAN>
__global__ void __launch_bounds__(256) quant16_kernel(const T* __restrict__ x, int64_t n_mat, int64_t rows,
                                                      int cols, int64_t mat_stride, int64_t row_stride,
                                                      int is_query, double c,
                                                      const unsigned long long* __restrict__ tensor_absmax,
                                                      QuantOut out) {
  // Work item = (matrix, block of 256 / tpr rows); a CTA walks items grid-stride
  // (x over row blocks, y over matrices) and prefetches the next item's 32 input bytes
  // while it quantizes the current one (the kernel is latency-bound otherwise).
  const int lg_tpr = __ffs(cols >> 4) - 1;  // tpr = cols / 16, a power of two in [2, 32]
  const int tpr = 1 << lg_tpr;
  const int lane = threadIdx.x & 31;
  const int part = threadIdx.x & (tpr - 1);
  const int rpb = 256 >> lg_tpr;  // rows per block
  const int64_t nbx = (rows + rpb - 1) / rpb;
  const int rsub = threadIdx.x >> lg_tpr;
  uint4 pf0 = make_uint4(0u, 0u, 0u, 0u), pf1 = pf0;  // prefetched words (bf16 inputs)
  auto fetch = [&](int64_t m, int64_t b) {
    const int64_t r = b * rpb + rsub;
    if constexpr (sizeof(T) == 2) {
      if (m < n_mat && r < rows) {
        const uint4* src = reinterpret_cast<const uint4*>(x + m * mat_stride + r * row_stride + part * 16);
        pf0 = __ldg(src);
        pf1 = __ldg(src + 1);
      } else {
        pf0 = pf1 = make_uint4(0u, 0u, 0u, 0u);
      }
    }
  };
  fetch(blockIdx.y, blockIdx.x);
  for (int64_t mat = blockIdx.y; mat < n_mat; mat += gridDim.y) {
  for (int64_t bx = blockIdx.x; bx < nbx; bx += gridDim.x) {
  const int64_t row = bx * rpb + rsub;
  const bool live = row < rows;  // whole rows live or die together (tpr | 32)
  const uint4 cur0 = pf0, cur1 = pf1;
  {
    int64_t nb = bx + gridDim.x, nm = mat;
    if (nb >= nbx) {
      nb = blockIdx.x;
      nm = mat + gridDim.y;
    }
    fetch(nm, nb);
  }
  if (__all_sync(0xffffffffu, !live)) continue;

  if (DMA_QUANT_F64)
    q16_item<T, NV, E5, GRAN>(x, mat_stride, row_stride, mat, rows, cols, row, live, part, tpr, lane, cur0, cur1,
                              is_query, c, tensor_absmax, out);
  else
    q16_item_fast<T, NV, E5, GRAN>(x, mat_stride, row_stride, mat, rows, cols, row, live, part, tpr, lane, cur0,
                                   cur1, is_query, c, tensor_absmax, out);
  }  // row-block loop
  }  // matrix loop
}

// max |x| per matrix as the bit pattern of a non-negative double (atomicMax on u64)
template <typename T>
__global__ void __launch_bounds__(256) absmax_kernel(const T* __restrict__ x, int64_t rows, int cols,
                                                     int64_t mat_stride, int64_t row_stride,
                                                     unsigned long long* __restrict__ out) {
  const int64_t mat = blockIdx.y;
  const int64_t n = rows * cols;
  double m = 0.0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, cc = i % cols;
    double v;
    if constexpr (sizeof(T) == 2) {
      v = __bfloat162float(x[mat * mat_stride + r * row_stride + cc]);
    } else {
      v = static_cast<double>(x[mat * mat_stride + r * row_stride + cc]);
    }
    m = fmax(m, fabs(v));  // NaN inputs are reported separately through ``nonfinite``
  }
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ double red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    atomicMax(out + mat, static_cast<unsigned long long>(__double_as_longlong(m)));
  }
}

// V -> MXFP8 (E4M3) along the key axis, for the block-scaled PV contraction.
// One thread per (value column n, 32-key block).  Codes keep V's row-major
// [keys, dv] layout (the MN-major B operand); the E8M0 scales go straight to
// the tcgen05 atom layout with "row" = n and k-block = key block in the tile.
// (No reference counterpart: the reference keeps V in float64, attention.py:250.)
template <typename T>
__global__ void __launch_bounds__(128) quant_v_kernel(const T* __restrict__ v, int64_t keys, int dv,
                                                      int64_t keys_pad, uint8_t* __restrict__ codes,
                                                      uint8_t* __restrict__ sf_op) {
  const int n = blockIdx.x * 32 + (threadIdx.x & 31);
  const int64_t kblk = static_cast<int64_t>(blockIdx.y) * 4 + (threadIdx.x >> 5);
  const int64_t mat = blockIdx.z;
  if (n >= dv || kblk * 32 >= keys_pad) return;
  const T* src = v + mat * keys * dv;
  float vals[32];
  float vmax = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int64_t key = kblk * 32 + i;
    float f = 0.f;
    if (key < keys) {
      if constexpr (sizeof(T) == 2) f = __bfloat162float(src[key * dv + n]);
      else f = static_cast<float>(src[key * dv + n]);
    }
    vals[i] = f;
    vmax = fmaxf(vmax, fabsf(f));
  }
  int e = -127;
  if (vmax > 0.f) {
    const int fl = static_cast<int>((__float_as_uint(vmax) >> 23) & 0xFF) - 127;  // f32 subnormals -> -127
    e = min(max(fl - 8, -127), 127);
  }
  const float inv = exp2f(static_cast<float>(-e));
  uint8_t* dst = codes + mat * keys_pad * dv;
#pragma unroll
  for (int i = 0; i < 32; i += 2) {
    const uint32_t pr = ptx::cvt_e4m3x2(vals[i] * inv, vals[i + 1] * inv);
    const int64_t key = kblk * 32 + i;
    dst[key * dv + n] = static_cast<uint8_t>(pr & 0xFF);
    dst[(key + 1) * dv + n] = static_cast<uint8_t>(pr >> 8);
  }
  // scale atom: tile = key tile of 128, "row" = n, k-block = kblk % 4
  const int64_t ktile = kblk >> 2;
  const int64_t ntiles = keys_pad >> 7;
  const int nchunk = (dv + 127) >> 7;  // dv <= 128 -> 1
  const int64_t off = ((mat * ntiles + ktile) * nchunk + (n >> 7)) * 512 + ((n & 127) & 31) * 16 +
                      ((n & 127) >> 5) * 4 + (kblk & 3);
  sf_op[off] = static_cast<uint8_t>(e + 127);
}

// V -> MXFP8 (E4M3) along keys, coalesced variant: a thread owns two adjacent
// value columns of one 32-key block (4-byte loads, 2-byte code stores, a warp
// covers 64 contiguous columns of a key row).  Same arithmetic as
// quant_v_kernel.  blockDim = 256; a CTA covers 256 / (dv/2) key blocks.
template <typename T>
__global__ void __launch_bounds__(256) quant_v2_kernel(const T* __restrict__ v, int64_t keys, int dv,
                                                       int64_t keys_pad, uint8_t* __restrict__ codes,
                                                       uint8_t* __restrict__ sf_op) {
  const int tpb = dv >> 1;                      // threads per key block
  const int n = (threadIdx.x % tpb) * 2;        // first of my two columns
  const int64_t kblk = static_cast<int64_t>(blockIdx.x) * (blockDim.x / tpb) + threadIdx.x / tpb;
  const int64_t mat = blockIdx.y;
  if (kblk * 32 >= keys_pad) return;
  const T* src = v + mat * keys * dv + n;
  float a[32], b[32];
  float ma = 0.f, mb = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int64_t key = kblk * 32 + i;
    float f0 = 0.f, f1 = 0.f;
    if (key < keys) {
      if constexpr (sizeof(T) == 2) {
        const uint32_t w = __ldg(reinterpret_cast<const unsigned int*>(src + key * dv));
        f0 = __uint_as_float(w << 16);
        f1 = __uint_as_float(w & 0xFFFF0000u);
      } else {
        f0 = static_cast<float>(src[key * dv]);
        f1 = static_cast<float>(src[key * dv + 1]);
      }
    }
    a[i] = f0;
    b[i] = f1;
    ma = fmaxf(ma, fabsf(f0));
    mb = fmaxf(mb, fabsf(f1));
  }
  auto expo = [](float m) {
    if (!(m > 0.f)) return -127;
    const int fl = static_cast<int>((__float_as_uint(m) >> 23) & 0xFF) - 127;  // f32 subnormals -> -127
    return min(max(fl - 8, -127), 127);
  };
  const int ea = expo(ma), eb = expo(mb);
  const float ia = exp2f(static_cast<float>(-ea)), ib = exp2f(static_cast<float>(-eb));
  uint8_t* dst = codes + mat * keys_pad * dv + n;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const uint32_t pr = ptx::cvt_e4m3x2(a[i] * ia, b[i] * ib);
    *reinterpret_cast<uint16_t*>(dst + (kblk * 32 + i) * dv) = static_cast<uint16_t>(pr);
  }
  const int64_t ktile = kblk >> 2;
  const int64_t ntiles = keys_pad >> 7;
  const int nchunk = (dv + 127) >> 7;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int c = n + j;
    const int64_t off = ((mat * ntiles + ktile) * nchunk + (c >> 7)) * 512 + ((c & 127) & 31) * 16 +
                        ((c & 127) >> 5) * 4 + (kblk & 3);
    sf_op[off] = static_cast<uint8_t>((j ? eb : ea) + 127);
  }
}

// bf16 V -> MXFP8 along keys, wide variant: a thread owns four adjacent value columns
// of one 32-key block (8-byte loads, 4-byte code stores; a warp covers 128 contiguous
// columns of a key row).  Same arithmetic as quant_v2_kernel: the column maxima come
// from the bf16 bit patterns (integer max), exact like the f32 max it replaces.
// bf16 V -> MXFP8 along keys for one 32-key block (kblk) and four value columns n..n+3 of one
// matrix (quant_v2_kernel arithmetic); shared by quant_v4_bf16_kernel and the fused kernel.
__device__ __forceinline__ void qv4_block(const __nv_bfloat16* __restrict__ v, int64_t keys, int dv, int64_t keys_pad,
                                          uint8_t* __restrict__ codes, uint8_t* __restrict__ sf_op, int64_t mat,
                                          int64_t kblk, int n) {
  const __nv_bfloat16* src = v + mat * keys * dv + n;
  uint2 w[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int64_t key = kblk * 32 + i;
    w[i] = key < keys ? __ldg(reinterpret_cast<const uint2*>(src + key * dv)) : make_uint2(0u, 0u);
  }
  uint32_t m01 = 0u, m23 = 0u;  // per-column max |bf16| bit patterns, two columns per word
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    m01 = __vmaxu2(m01, w[i].x & 0x7FFF7FFFu);
    m23 = __vmaxu2(m23, w[i].y & 0x7FFF7FFFu);
  }
  auto expo = [](uint32_t m16) {  // exponent of the column max, as quant_v2_kernel
    if (m16 == 0u) return -127;
    const int fl = static_cast<int>((m16 >> 7) & 0xFF) - 127;  // bf16 / f32 subnormals -> -127
    return min(max(fl - 8, -127), 127);
  };
  const int e[4] = {expo(m01 & 0xFFFFu), expo(m01 >> 16), expo(m23 & 0xFFFFu), expo(m23 >> 16)};
  float inv[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) inv[j] = exp2f(static_cast<float>(-e[j]));
  uint8_t* dst = codes + mat * keys_pad * dv + n;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const float f0 = __uint_as_float(w[i].x << 16), f1 = __uint_as_float(w[i].x & 0xFFFF0000u);
    const float f2 = __uint_as_float(w[i].y << 16), f3 = __uint_as_float(w[i].y & 0xFFFF0000u);
    const uint32_t lo = ptx::cvt_e4m3x2(f0 * inv[0], f1 * inv[1]);
    const uint32_t hi = ptx::cvt_e4m3x2(f2 * inv[2], f3 * inv[3]);
    *reinterpret_cast<uint32_t*>(dst + (kblk * 32 + i) * dv) = (lo & 0xFFFFu) | (hi << 16);
  }
  const int64_t ktile = kblk >> 2;
  const int64_t ntiles = keys_pad >> 7;
  const int nchunk = (dv + 127) >> 7;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int c = n + j;
    const int64_t off = ((mat * ntiles + ktile) * nchunk + (c >> 7)) * 512 + ((c & 127) & 31) * 16 +
                        ((c & 127) >> 5) * 4 + (kblk & 3);
    sf_op[off] = static_cast<uint8_t>(e[j] + 127);
  }
}

static __global__ void __launch_bounds__(256) quant_v4_bf16_kernel(const __nv_bfloat16* __restrict__ v, int64_t keys, int dv,
                                                            int64_t keys_pad, uint8_t* __restrict__ codes,
                                                            uint8_t* __restrict__ sf_op) {
  const int tpb = dv >> 2;                      // threads per key block
  const int n = (threadIdx.x % tpb) * 4;        // first of my four columns
  const int64_t kblk = static_cast<int64_t>(blockIdx.x) * (blockDim.x / tpb) + threadIdx.x / tpb;
  const int64_t mat = blockIdx.y;
  ptx::pdl_launch_dependents();
  if (kblk * 32 < keys_pad) qv4_block(v, keys, dv, keys_pad, codes, sf_op, mat, kblk, n);
  ptx::pdl_wait();  // PDL chain: this grid completes only after the previous phase-1 kernel
}

// Split-KV experiment (attn_sk.cuh, key_perm = 2): per 128-key tile of S_q^K (natural
// order, kSqkTile slots per tile) the max / min over the valid keys into slots kSqkMaxSlot /
// kSqkMinSlot, and S_q^K = 1 for the padded keys of the last tile.  One warp per tile.
static __global__ void __launch_bounds__(256) sqk_tile_stats_kernel(float* __restrict__ qs, int64_t n_tiles_total,
                                                             int64_t rtiles, int64_t rows) {
  const int lane = threadIdx.x & 31;
  const int64_t wt = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (wt >= n_tiles_total) return;
  const int64_t tile = wt % rtiles;
  float* blk = qs + wt * kSqkTile;
  float vmax = 0.f, vmin = INFINITY;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = 32 * i + lane;
    if (tile * 128 + k < rows) {
      const float v = blk[k];
      vmax = fmaxf(vmax, v);
      vmin = fminf(vmin, v);
    } else {
      blk[k] = 1.0f;
    }
  }
  for (int o = 16; o; o >>= 1) {
    vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
    vmin = fminf(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
  }
  if (lane == 0) {
    reinterpret_cast<unsigned int*>(blk)[kSqkMaxSlot] = __float_as_uint(vmax);
    reinterpret_cast<unsigned int*>(blk)[kSqkMinSlot] = ~__float_as_uint(vmin);
  }
}

// ------------------------------------------------------------------------
// Phase 1 of the attention path in ONE launch (bf16 inputs, TOKEN granularity): CTAs
// [0, nq) quantize Q, [nq, nq + nk) K -- each part a grid-stride walk over (matrix, row
// block) items with the next item's 32 input bytes per thread prefetched, as
// quant16_kernel -- and the remaining CTAs quantize V key blocks (qv4_block).  Saves two
// launches per forward (small problems are launch-bound).
// ------------------------------------------------------------------------
struct P1Job {
  const __nv_bfloat16* x;
  int64_t n_mat, rows;
  int is_query;
  QuantOut out;
};

template <bool NV, bool E5>
__device__ __forceinline__ void phase1_rows(const P1Job& j, int cols, double c, int cta, int ncta) {
  const int lg_tpr = __ffs(cols >> 4) - 1;
  const int tpr = 1 << lg_tpr;
  const int lane = threadIdx.x & 31;
  const int part = threadIdx.x & (tpr - 1);
  const int rpb = 256 >> lg_tpr;
  const int rsub = threadIdx.x >> lg_tpr;
  const int64_t nbx = (j.rows + rpb - 1) / rpb;
  const int64_t items = j.n_mat * nbx;
  const int64_t mstride = j.rows * cols;
  uint4 pf0 = make_uint4(0u, 0u, 0u, 0u), pf1 = pf0;
  auto fetch = [&](int64_t it) {
    const int64_t m = it / nbx, r = (it - m * nbx) * rpb + rsub;
    if (it < items && r < j.rows) {
      const uint4* src = reinterpret_cast<const uint4*>(j.x + m * mstride + r * cols + part * 16);
      pf0 = __ldg(src);
      pf1 = __ldg(src + 1);
    } else {
      pf0 = pf1 = make_uint4(0u, 0u, 0u, 0u);
    }
  };
  fetch(cta);
  for (int64_t it = cta; it < items; it += ncta) {
    const uint4 cur0 = pf0, cur1 = pf1;
    fetch(it + ncta);
    const int64_t mat = it / nbx, row = (it - mat * nbx) * rpb + rsub;
    const bool live = row < j.rows;
    if (__all_sync(0xffffffffu, !live)) continue;
    q16_item_fast<__nv_bfloat16, NV, E5, DMA_GRAN_TOKEN>(j.x, mstride, cols, mat, j.rows, cols, row, live, part, tpr,
                                                        lane, cur0, cur1, j.is_query, c, nullptr, j.out);
  }
}

template <bool NV, bool E5>
__global__ void __launch_bounds__(256) phase1_bf16_kernel(const __grid_constant__ P1Job jq, const __grid_constant__ P1Job jk,
                                                          int cols, double c, int nq, int nk,
                                                          const __nv_bfloat16* __restrict__ v, int64_t keys, int dv,
                                                          int64_t keys_pad, int64_t mk, uint8_t* __restrict__ v_codes,
                                                          uint8_t* __restrict__ sf_v) {
  const int b = blockIdx.x;
  ptx::pdl_launch_dependents();
  if (b < nq) {
    phase1_rows<NV, E5>(jq, cols, c, b, nq);
  } else if (b < nq + nk) {
    phase1_rows<NV, E5>(jk, cols, c, b - nq, nk);
  } else {
    const int tpb = dv >> 2;                  // threads per 32-key block
    const int kbpc = 256 / tpb;               // key blocks per CTA pass
    const int64_t groups = (keys_pad / 32 + kbpc - 1) / kbpc;
    const int nv = gridDim.x - nq - nk;
    for (int64_t it = b - nq - nk; it < mk * groups; it += nv) {
      const int64_t mat = it / groups;
      const int64_t kblk = (it - mat * groups) * kbpc + threadIdx.x / tpb;
      if (kblk * 32 < keys_pad) qv4_block(v, keys, dv, keys_pad, v_codes, sf_v, mat, kblk, (threadIdx.x % tpb) * 4);
    }
  }
}

}  // namespace dma
