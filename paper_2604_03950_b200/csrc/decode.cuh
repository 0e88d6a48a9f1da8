// Decode (KV-cache) variant of the DMA forward: n_q new query rows per sequence against
// a key cache held in the canonical quantize_dual layouts (SURVEY §8 f, rank 4).
//
// Semantics: query i of a sequence sits at absolute position p = pos + i and sees keys
// [0, p]; its output equals row p of mixed_precision_attention (attention.py:282-310)
// over the whole sequence: key tile t (tile_n keys) is scored in high precision iff
// t < sink_window / tile_n or t >= ceil((q0 - diag_window) / tile_n), q0 = (p / tile_m)
// * tile_m (attention.py:191-209 with every clip resolved for a visible key), in low
// precision otherwise.  TOKEN granularity only: every K / Q row is quantized on its own,
// so a cache row never changes once written.
//
// Memory-bound split-KV kernel on the CUDA cores (one query row per GQA head and new
// token is far below a tcgen05 M=128 tile): a CTA takes R query rows of one KV head and
// a key range; its 4 warps walk 32-key groups (lane = key for QK: one 16-byte load per
// 32 packed-FP4 elements, hardware F2FP unpack, f32 FMAs against the dequantized query
// rows in shared memory; lane = 4 value columns for PV); online softmax in base 2 per
// warp, warps merged in shared memory, splits merged by dma_decode_combine_kernel.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <type_traits>

#include "common.cuh"
#include "ptx.cuh"

namespace dma {

#ifndef DMA_DEC_STAGES
#define DMA_DEC_STAGES 1  // cache-row stages per warp ring (1: more resident CTAs, measured
                          // 11-13 % faster than 2 and far ahead of 3)
#endif

#ifndef DMA_DEC_MMA_MIN_R
#define DMA_DEC_MMA_MIN_R 2  // tensor-core QK from this many query rows per CTA
#endif
#ifndef DMA_DEC_MINB
#define DMA_DEC_MINB(R) ((R) <= 4 ? 4 : ((R) <= 8 ? 3 : 2))  // min resident CTAs (register cap)
#endif

enum { kDecLowNV = 0, kDecLowMX4 = 1, kDecLow8 = 2 };

struct DecodeParams {
  const uint8_t *q_lo, *q_lo_sf, *q_hi, *q_hi_sf;
  const double* q_sq;
  const uint8_t *k_lo, *k_lo_sf, *k_hi, *k_hi_sf;
  const double* k_sq;
  const __nv_bfloat16* v;
  float* part_o;   // [rows_total, splits, DV]
  float2* part_ml; // [rows_total, splits] (m, l)
  int64_t batch, heads, kv_heads, n_q, cap, pos;
  int32_t group, rows_per_kvh, n_rg, splits, keys_per_split;
  int32_t tile_m, tile_n, diag_window, sink_window;
  int32_t hi_e5m2;
};

__device__ __forceinline__ float2 e2m1x2_to_f2(uint32_t byte) {
  uint32_t h;
  asm("{\n\t.reg .b8 b;\n\tcvt.u8.u32 b, %1;\n\tcvt.rn.f16x2.e2m1x2 %0, b;\n\t}" : "=r"(h) : "r"(byte));
  return __half22float2(*reinterpret_cast<__half2*>(&h));
}
__device__ __forceinline__ float2 fp8x2_to_f2(uint32_t two, bool e5m2) {
  uint32_t h;
  if (e5m2)
    asm("{\n\t.reg .b16 b;\n\tcvt.u16.u32 b, %1;\n\tcvt.rn.f16x2.e5m2x2 %0, b;\n\t}" : "=r"(h) : "r"(two));
  else
    asm("{\n\t.reg .b16 b;\n\tcvt.u16.u32 b, %1;\n\tcvt.rn.f16x2.e4m3x2 %0, b;\n\t}" : "=r"(h) : "r"(two));
  return __half22float2(*reinterpret_cast<__half2*>(&h));
}
__device__ __forceinline__ float e8m0_to_f(uint32_t raw) {  // 2^(raw - 127), raw <= 254
  return raw ? __uint_as_float(raw << 23) : 5.877471754111438e-39f;  // 2^-127 (subnormal)
}
__device__ __forceinline__ float e4m3_to_f(uint32_t code) {
  return fp8x2_to_f2(code & 0xFFu, false).x;
}

// 32 dequantized (block-scaled, no S_q) elements of one operand row chunk c (32 columns)
template <int LOW>
__device__ __forceinline__ void load_lo32(const uint8_t* row, const uint8_t* sf, int c, float (&x)[32]) {
  const uint4 w = __ldg(reinterpret_cast<const uint4*>(row + 16 * c));
  float s0, s1;
  if (LOW == kDecLowNV) {
    s0 = e4m3_to_f(sf[2 * c]);
    s1 = e4m3_to_f(sf[2 * c + 1]);
  } else {
    s0 = s1 = e8m0_to_f(sf[c]);
  }
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const float2 f = e2m1x2_to_f2((ws[i] >> (8 * b)) & 0xFFu);
      const float s = i < 2 ? s0 : s1;
      x[8 * i + 2 * b] = f.x * s;
      x[8 * i + 2 * b + 1] = f.y * s;
    }
}
__device__ __forceinline__ void load_hi32(const uint8_t* row, const uint8_t* sf, int c, bool e5m2, float (&x)[32]) {
  const uint4 w0 = __ldg(reinterpret_cast<const uint4*>(row + 32 * c));
  const uint4 w1 = __ldg(reinterpret_cast<const uint4*>(row + 32 * c + 16));
  const float s = e8m0_to_f(sf[c]);
  const uint32_t ws[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float2 f = fp8x2_to_f2((ws[i] >> (16 * h)) & 0xFFFFu, e5m2);
      x[4 * i + 2 * h] = f.x * s;
      x[4 * i + 2 * h + 1] = f.y * s;
    }
}

// 32 element values (no block scale) of chunk c as 16 f32 pairs, plus the chunk's block
// scales (NVFP4: one per 16 elements; MX: one per 32, s1 == s0)
template <int LOW>
__device__ __forceinline__ void load_lo32_raw(const uint8_t* row, const uint8_t* sf, int c, float2 (&x)[16],
                                              float& s0, float& s1) {  // shared-memory rows
  const uint4 w = *reinterpret_cast<const uint4*>(row + 16 * c);
  if (LOW == kDecLowNV) {
    const uint32_t two = *reinterpret_cast<const uint16_t*>(sf + 2 * c);
    const float2 f = fp8x2_to_f2(two, false);
    s0 = f.x;
    s1 = f.y;
  } else {
    s0 = s1 = e8m0_to_f(sf[c]);
  }
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int b = 0; b < 4; ++b) x[4 * i + b] = e2m1x2_to_f2((ws[i] >> (8 * b)) & 0xFFu);
}
template <bool kGlobal>
__device__ __forceinline__ void load_hi32_raw(const uint8_t* row, const uint8_t* sf, int c, bool e5m2,
                                              float2 (&x)[16], float& s) {
  uint4 w0, w1;
  if (kGlobal) {
    w0 = __ldg(reinterpret_cast<const uint4*>(row + 32 * c));
    w1 = __ldg(reinterpret_cast<const uint4*>(row + 32 * c + 16));
    s = e8m0_to_f(__ldg(sf + c));
  } else {
    w0 = *reinterpret_cast<const uint4*>(row + 32 * c);
    w1 = *reinterpret_cast<const uint4*>(row + 32 * c + 16);
    s = e8m0_to_f(sf[c]);
  }
  const uint32_t ws[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int h = 0; h < 2; ++h) x[2 * i + h] = fp8x2_to_f2((ws[i] >> (16 * h)) & 0xFFFFu, e5m2);
}
// sum over pairs [i0, i0 + n) of q * x (packed f32x2 FMAs), q from shared memory
template <int N>
__device__ __forceinline__ float dot_pairs(const float* q, const float2 (&x)[16], int i0) {
  const float4* q4 = reinterpret_cast<const float4*>(q);
  float4 qv[N / 2];  // all loads first (independent), then two FFMA2 chains
#pragma unroll
  for (int e = 0; e < N / 2; ++e) qv[e] = q4[(i0 >> 1) + e];
  float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
#pragma unroll
  for (int e = 0; e < N / 2; ++e) {
    a0 = __ffma2_rn(make_float2(qv[e].x, qv[e].y), x[i0 + 2 * e], a0);
    a1 = __ffma2_rn(make_float2(qv[e].z, qv[e].w), x[i0 + 2 * e + 1], a1);
  }
  return (a0.x + a1.x) + (a0.y + a1.y);
}

// ---- NVFP4 QK on the tensor cores (mma.sync m16n8k16, f16 in, f32 accumulate).  An
// NVFP4 element times its E4M3 block scale has <= 6 significant bits and lies in
// [2^-10, 2688], so both dequantized operands are exact in f16 and every product is
// exact in the f32 accumulator -- the same arithmetic class as the FFMA path.  One
// k16 step is exactly one NVFP4 block.
__device__ __forceinline__ uint32_t e2m1x2_to_h2(uint32_t byte) {
  uint32_t h;
  asm("{\n\t.reg .b8 b;\n\tcvt.u8.u32 b, %1;\n\tcvt.rn.f16x2.e2m1x2 %0, b;\n\t}" : "=r"(h) : "r"(byte));
  return h;
}
__device__ __forceinline__ uint32_t e4m3x2_to_h2(uint32_t two) {
  uint32_t h;
  asm("{\n\t.reg .b16 b;\n\tcvt.u16.u32 b, %1;\n\tcvt.rn.f16x2.e4m3x2 %0, b;\n\t}" : "=r"(h) : "r"(two));
  return h;
}
__device__ __forceinline__ uint32_t hmul2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ void mma_16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// the two f16x2 fragment words of one NVFP4 row for k16 step ks: bytes 8 ks + j and
// 8 ks + 4 + j (j = lane % 4) of the packed row, times the block scale (f16x2 splat)
__device__ __forceinline__ void nv_frag(const uint32_t (&w)[16], int ks, int j, uint32_t s2, uint32_t& f0,
                                        uint32_t& f1) {
  f0 = hmul2(e2m1x2_to_h2((w[2 * ks] >> (8 * j)) & 0xFFu), s2);
  f1 = hmul2(e2m1x2_to_h2((w[2 * ks + 1] >> (8 * j)) & 0xFFu), s2);
}
__device__ __forceinline__ uint32_t splat_lo(uint32_t h2) { return (h2 & 0xFFFFu) | (h2 << 16); }
__device__ __forceinline__ uint32_t splat_hi(uint32_t h2) { return (h2 >> 16) | (h2 & 0xFFFF0000u); }

// shared memory: dequantized query rows (low, high) [R][D] f32, P [4 warps][R][32],
// warp partials (m, l) [4][R] and O [4][R][DV]
template <int R, int D, int DV, int LOW>
struct DecSmem {
  // per-warp ring of kStages stages; a stage holds one 32-key group of the cache:
  // the "A" key rows (packed FP4 low, or FP8 high codes when the low format is 8-bit),
  // their block scales, S_q and the bf16 value rows, all filled by cp.async.bulk
  static constexpr int kStages = DMA_DEC_STAGES;
  static constexpr int kA = LOW == kDecLow8 ? 32 * D : 32 * D / 2;
  static constexpr int kAsf = 32 * (D / (LOW == kDecLowNV ? 16 : 32));
  static constexpr int sA = 0, sAsf = kA, sSq = sAsf + kAsf, sV = sSq + 32 * 8;
  static constexpr int kStage = (sV + 32 * DV * 2 + 127) / 128 * 128;
  static constexpr bool kMma = (LOW == kDecLowNV || LOW == kDecLowMX4) && R >= DMA_DEC_MMA_MIN_R;
  static constexpr int oRing = 0;
  static constexpr int oQlo = oRing + 4 * kStages * kStage;
  // dequantized low query rows: only the FFMA low path reads them
  static constexpr int oQhi = oQlo + (kMma || LOW == kDecLow8 ? 0 : R * D * 4);
  static constexpr int oP = oQhi + R * D * 4;
  static constexpr int oML = oP + 4 * R * 32 * 4;
  static constexpr int oSmma = oML + 4 * R * 8;  // tensor-core QK: S tile [16][32] f32 per warp
  // rows' S_q^Q and positions [16] (f32, i32), per-warp row maxima [4][16] (tensor-core path)
  static constexpr int oRows = oSmma + (kMma ? 4 * 16 * 32 * 4 : 0);
  static constexpr int oBar = oRows + (kMma ? 16 * 4 * 2 + 4 * 16 * 4 : 0);
  static constexpr int oO = oRing;  // warp partials reuse the rings once every warp is done
  static_assert(4 * R * DV * 4 <= 4 * kStages * kStage, "partials fit in the rings");
  static constexpr int kBytes = oBar + 4 * kStages * 8;
};

// host: resident CTAs per SM of dma_decode_kernel<R, D, DV, LOW> (shared memory bound)
inline int dec_ctas_per_sm(int R, int D, int DV, int low) {
  int bytes = 0;
  auto get = [&](auto tag) { bytes = decltype(tag)::kBytes; };
  auto by_low = [&](auto r, auto d, auto dv) {
    constexpr int Rv = decltype(r)::value, Dv = decltype(d)::value, DVv = decltype(dv)::value;
    if (low == kDecLowNV) get(DecSmem<Rv, Dv, DVv, kDecLowNV>{});
    else if (low == kDecLowMX4) get(DecSmem<Rv, Dv, DVv, kDecLowMX4>{});
    else get(DecSmem<Rv, Dv, DVv, kDecLow8>{});
  };
  auto by_dims = [&](auto r) {
    using I64 = std::integral_constant<int, 64>;
    using I128 = std::integral_constant<int, 128>;
    if (D == 64 && DV == 64) by_low(r, I64{}, I64{});
    else if (D == 64) by_low(r, I64{}, I128{});
    else if (DV == 64) by_low(r, I128{}, I64{});
    else by_low(r, I128{}, I128{});
  };
  switch (R) {
    case 1: by_dims(std::integral_constant<int, 1>{}); break;
    case 2: by_dims(std::integral_constant<int, 2>{}); break;
    case 4: by_dims(std::integral_constant<int, 4>{}); break;
    default: by_dims(std::integral_constant<int, 8>{}); break;
  }
  const int n = (228 * 1024) / (bytes + 1024);  // 228 KB per SM, ~1 KB reserved per CTA
  return n < 1 ? 1 : (n > 4 ? 4 : n);
}

template <int R, int D, int DV, int LOW>
__global__ void __launch_bounds__(128, DMA_DEC_MINB(R)) dma_decode_kernel(const DecodeParams p) {
  using S = DecSmem<R, D, DV, LOW>;
  extern __shared__ __align__(16) uint8_t smem[];
  float* q_lo = reinterpret_cast<float*>(smem + S::oQlo);
  float* q_hi = reinterpret_cast<float*>(smem + S::oQhi);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // work item: (b * kv_heads + kvh, row group, split)
  int item = blockIdx.x;
  const int split = item % p.splits;
  item /= p.splits;
  const int rg = item % p.n_rg;
  const int mk = item / p.n_rg;  // key matrix b * kv_heads + kvh
  const int b = mk / static_cast<int>(p.kv_heads), kvh = mk % static_cast<int>(p.kv_heads);
  const bool e5 = p.hi_e5m2 != 0;

  // rows of this CTA: local row r -> (head in group, new token); invalid rows are padding
  auto row_of = [&](int r) -> int64_t {  // row in the [B*H, n_q] query arrays, -1 = padding
    const int lr = rg * R + r;
    if (lr >= p.rows_per_kvh) return -1;
    const int gq = lr / static_cast<int>(p.n_q), i = lr % static_cast<int>(p.n_q);
    return (static_cast<int64_t>(b) * p.heads + static_cast<int64_t>(kvh) * p.group + gq) * p.n_q + i;
  };
  int64_t qrow[R];  // row in the [B*H, n_q] query arrays, -1 = padding
  int qpos[R];      // absolute position of the row (-1: padding row; positions < 2^31)
  int hs[R];        // first high tile of the row's diagonal window
  float sqq[R];
  const int sink_t = p.sink_window / p.tile_n;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int lr = rg * R + r;
    if (lr < p.rows_per_kvh) {
      const int gq = lr / static_cast<int>(p.n_q), i = lr % static_cast<int>(p.n_q);
      const int64_t h = static_cast<int64_t>(kvh) * p.group + gq;
      qrow[r] = (static_cast<int64_t>(b) * p.heads + h) * p.n_q + i;
      qpos[r] = static_cast<int>(p.pos + i);
      const int64_t q0 = (static_cast<int64_t>(qpos[r]) / p.tile_m) * p.tile_m;
      hs[r] = static_cast<int>(ceil_div(q0 - p.diag_window, static_cast<int64_t>(p.tile_n)));
      sqq[r] = static_cast<float>(p.q_sq[qrow[r]]);
    } else {
      qrow[r] = -1;
      qpos[r] = -1;
      hs[r] = 0;
      sqq[r] = 0.f;
    }
  }
  if constexpr (S::kMma) {
    float* rs = reinterpret_cast<float*>(smem + S::oRows);
    int* rp = reinterpret_cast<int*>(smem + S::oRows + 64);
    if (threadIdx.x < 16) {
      float v = 0.f;
      int q = -1;
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (r == static_cast<int>(threadIdx.x)) {
          v = sqq[r];
          q = qpos[r];
        }
      rs[threadIdx.x] = v;
      rp[threadIdx.x] = q;
    }
  }
  // dequantize the query rows (block scales only; S_q folds in per logit)
  for (int idx = threadIdx.x; idx < R * (D / 32); idx += blockDim.x) {
    const int r = idx / (D / 32), c = idx % (D / 32);
    float x[32];
    const int64_t qr = row_of(r);
    if (qr >= 0) {
      if (LOW != kDecLow8 && !S::kMma) {
        load_lo32<LOW>(p.q_lo + qr * (D / 2), p.q_lo_sf + qr * (D / (LOW == kDecLowNV ? 16 : 32)), c, x);
#pragma unroll
        for (int j = 0; j < 32; ++j) q_lo[r * D + 32 * c + j] = x[j];
      }
      load_hi32(p.q_hi + qr * D, p.q_hi_sf + qr * (D / 32), c, e5, x);
#pragma unroll
      for (int j = 0; j < 32; ++j) q_hi[r * D + 32 * c + j] = x[j];
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (LOW != kDecLow8 && !S::kMma) q_lo[r * D + 32 * c + j] = 0.f;
        q_hi[r * D + 32 * c + j] = 0.f;
      }
    }
  }
  __syncthreads();

  // NVFP4: this warp's A fragments (16 query rows x D, f16) for the tensor-core QK;
  // rows beyond the CTA's valid rows are zero
  // (R = 1 wastes 15/16 of every MMA: measured faster on the FFMA path)
  constexpr bool kMma = S::kMma;
  uint32_t qa[kMma ? D / 16 : 1][4];
  float qsc[2][LOW == kDecLowMX4 ? D / 32 : 1];  // MXFP4: E8M0 block scales of rows n, n + 8
  if constexpr (kMma) {
    const int j = lane & 3;
#pragma unroll
    for (int h8 = 0; h8 < 2; ++h8) {
      const int r = (lane >> 2) + 8 * h8;
      const int64_t qr = r < R ? row_of(r) : -1;
      uint32_t w[16];
      uint32_t sc[D / 32];  // NVFP4: E4M3 scale pairs; MXFP4: E8M0 bytes
      if (qr >= 0) {
#pragma unroll
        for (int i = 0; i < D / 8; ++i) w[i] = __ldg(reinterpret_cast<const uint32_t*>(p.q_lo + qr * (D / 2)) + i);
#pragma unroll
        for (int i = 0; i < D / 32; ++i)
          sc[i] = LOW == kDecLowNV ? __ldg(reinterpret_cast<const uint16_t*>(p.q_lo_sf + qr * (D / 16)) + i)
                                   : __ldg(p.q_lo_sf + qr * (D / 32) + i);
      } else {
#pragma unroll
        for (int i = 0; i < D / 8; ++i) w[i] = 0u;
#pragma unroll
        for (int i = 0; i < D / 32; ++i) sc[i] = 0u;
      }
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
        // NVFP4: element x E4M3 block scale (exact in f16); MXFP4: the raw element, the
        // power-of-two block scale is applied to the block's f32 partial sums below
        uint32_t s2 = 0x3C003C00u;  // f16x2 (1, 1)
        if constexpr (LOW == kDecLowNV) {
          const uint32_t s2h = e4m3x2_to_h2(sc[ks >> 1]);
          s2 = (ks & 1) ? splat_hi(s2h) : splat_lo(s2h);
        }
        uint32_t f0, f1;
        nv_frag(*reinterpret_cast<const uint32_t(*)[16]>(&w[0]), ks, j, s2, f0, f1);
        qa[ks][h8] = f0;      // a0 / a1: k = 2j + {0, 1}
        qa[ks][2 + h8] = f1;  // a2 / a3: k = 2j + 8 + {0, 1}
      }
      if constexpr (LOW == kDecLowMX4) {
#pragma unroll
        for (int b = 0; b < D / 32; ++b) qsc[h8][b] = qr >= 0 ? e8m0_to_f(sc[b]) : 0.f;
      }
    }
  }
  float* smma = reinterpret_cast<float*>(smem + S::oSmma) + warp * 16 * 32;
  const float* rows_sq = reinterpret_cast<const float*>(smem + S::oRows);
  const int* rows_pos = reinterpret_cast<const int*>(smem + S::oRows + 64);
  float* rmax_w = reinterpret_cast<float*>(smem + S::oRows + 128) + warp * 16;

  int64_t last = -1;  // last visible key of any row
#pragma unroll
  for (int r = 0; r < R; ++r) last = qpos[r] > last ? qpos[r] : last;  // (int64 last)
  const int64_t k_begin = static_cast<int64_t>(split) * p.keys_per_split;
  int64_t k_end = k_begin + p.keys_per_split;
  k_end = k_end < last + 1 ? k_end : last + 1;

  constexpr int NP = DV / 64;  // value-column pairs per lane
  float m[R], l[R];
  float2 o[R][NP];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    m[r] = -INFINITY;
    l[r] = 0.f;
#pragma unroll
    for (int c = 0; c < NP; ++c) o[r][c] = make_float2(0.f, 0.f);
  }
  float* ps = reinterpret_cast<float*>(smem + S::oP) + warp * R * 32;
  const int64_t krow0 = static_cast<int64_t>(mk) * p.cap;

  // which operand copies a 32-key group needs (per row: the tile's precision for that row)
  auto needs = [&](int64_t g, bool& nlo, bool& nhi) {
    const int t = static_cast<int>(static_cast<uint32_t>(g) / static_cast<uint32_t>(p.tile_n));  // one key tile per group
    nlo = nhi = false;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const bool h = LOW == kDecLow8 || t < sink_t || t >= hs[r];
      if (static_cast<int>(g) <= qpos[r]) (h ? nhi : nlo) = true;  // padding rows: qpos = -1
    }
  };
  // producer side of this warp's ring (lane 0): bulk-load the 32 cache rows of group g
  // (capacity is a multiple of 32, so whole groups stay inside the cache)
  uint8_t* ring = smem + S::oRing + warp * S::kStages * S::kStage;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::oBar) + warp * S::kStages;
  auto issue = [&](int st, int64_t g) {
    if (g >= k_end) return;
    bool nlo, nhi;
    needs(g, nlo, nhi);
    const bool ldA = LOW == kDecLow8 || nlo;
    const int64_t r0 = krow0 + g;
    uint8_t* dst = ring + st * S::kStage;
    uint32_t bytes = 32 * 8 + 32 * DV * 2 + (ldA ? S::kA + S::kAsf : 0);
    ptx::mbar_arrive_expect_tx(full + st, bytes);
    if (ldA) {
      if (LOW == kDecLow8) {
        ptx::bulk_load(dst + S::sA, p.k_hi + r0 * D, S::kA, full + st);
        ptx::bulk_load(dst + S::sAsf, p.k_hi_sf + r0 * (D / 32), S::kAsf, full + st);
      } else {
        ptx::bulk_load(dst + S::sA, p.k_lo + r0 * (D / 2), S::kA, full + st);
        ptx::bulk_load(dst + S::sAsf, p.k_lo_sf + r0 * (S::kAsf / 32), S::kAsf, full + st);
      }
    }
    ptx::bulk_load(dst + S::sSq, p.k_sq + r0, 32 * 8, full + st);
    ptx::bulk_load(dst + S::sV, p.v + r0 * DV, 32 * DV * 2, full + st);
  };
  if (lane == 0) {
#pragma unroll
    for (int st = 0; st < S::kStages; ++st) ptx::mbar_init(full + st, 1);
    ptx::fence_barrier_init();
#pragma unroll
    for (int st = 0; st < S::kStages; ++st) issue(st, k_begin + 32 * warp + 128 * st);
  }
  __syncwarp();

  int it = 0;
  for (int64_t g0 = k_begin + 32 * warp; g0 < k_end; g0 += 128, ++it) {
    const int st = it % S::kStages;
    const uint8_t* stage = ring + st * S::kStage;
    const int64_t j = g0 + lane;
    const bool in = j < k_end;
    const int t = static_cast<int>(static_cast<uint32_t>(g0) / static_cast<uint32_t>(p.tile_n));
    bool hi[R];
#pragma unroll
    for (int r = 0; r < R; ++r) hi[r] = LOW == kDecLow8 || t < sink_t || t >= hs[r];
    bool need_lo, need_hi;
    needs(g0, need_lo, need_hi);
    const int64_t kr = krow0 + (in ? j : k_begin);
    ptx::mbar_wait(full + st, (it / S::kStages) & 1);
    float s[R];
#pragma unroll
    for (int r = 0; r < R; ++r) s[r] = 0.f;
    // tensor-core groups where no row needs the high copy finish their logits and row
    // maxima in the MMA epilogue (no per-row warp shuffles below)
    const bool lo_only = kMma && need_lo && !need_hi;
    if (need_lo && kMma) {
      // S[16 rows][32 keys] = A (q_lo) x B (this group's keys), four n8 tiles of keys
      const int j = lane & 3, n = lane >> 2;
      const float sq_n = rows_sq[n];
      const int qp_n = rows_pos[n];
      float lmax = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const uint8_t* krow = stage + S::sA + (nt * 8 + n) * (D / 2);
        uint32_t w[16];
#pragma unroll
        for (int i = 0; i < D / 32; ++i) {
          const uint4 v4 = reinterpret_cast<const uint4*>(krow)[i];
          w[4 * i] = v4.x;
          w[4 * i + 1] = v4.y;
          w[4 * i + 2] = v4.z;
          w[4 * i + 3] = v4.w;
        }
        float c[4] = {0.f, 0.f, 0.f, 0.f};
        if constexpr (LOW == kDecLowNV) {
          const uint8_t* ksf = stage + S::sAsf + (nt * 8 + n) * (D / 16);
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks) {
            const uint32_t scl = e4m3x2_to_h2(*reinterpret_cast<const uint16_t*>(ksf + (ks & ~1)));
            const uint32_t s2 = (ks & 1) ? splat_hi(scl) : splat_lo(scl);
            uint32_t b0, b1;
            nv_frag(*reinterpret_cast<const uint32_t(*)[16]>(&w[0]), ks, j, s2, b0, b1);
            mma_16816(c, qa[ks], b0, b1);
          }
        } else {
          // MXFP4: per 32-column block, raw-element MMAs (2 x k16) into a fresh accumulator,
          // then x 2^(e_q + e_k) for the accumulator's rows (n, n + 8) and keys (2j, 2j + 1)
          const uint8_t* ksf0 = stage + S::sAsf + (nt * 8 + 2 * j) * (D / 32);
#pragma unroll
          for (int b = 0; b < D / 32; ++b) {
            float cb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              uint32_t b0, b1;
              nv_frag(*reinterpret_cast<const uint32_t(*)[16]>(&w[0]), 2 * b + h, j, 0x3C003C00u, b0, b1);
              mma_16816(cb, qa[2 * b + h], b0, b1);
            }
            const float k0 = e8m0_to_f(ksf0[b]), k1 = e8m0_to_f(ksf0[D / 32 + b]);
            c[0] = fmaf(cb[0], qsc[0][b] * k0, c[0]);
            c[1] = fmaf(cb[1], qsc[0][b] * k1, c[1]);
            c[2] = fmaf(cb[2], qsc[1][b] * k0, c[2]);
            c[3] = fmaf(cb[3], qsc[1][b] * k1, c[3]);
          }
        }
        // C: rows n and n + 8 (padding: R <= 8), keys nt * 8 + 2 j + {0, 1}
        if (lo_only) {
          // final logits here: S_q^Q S_q^K (NVFP4), causal / ragged mask, running row max
          const int kk = nt * 8 + 2 * j;
          const double* sqd = reinterpret_cast<const double*>(stage + S::sSq);
          float x0 = c[0], x1 = c[1];
          if (LOW == kDecLowNV) {
            x0 *= sq_n * static_cast<float>(sqd[kk]);
            x1 *= sq_n * static_cast<float>(sqd[kk + 1]);
          }
          const int key0 = static_cast<int>(g0) + kk;
          x0 = (key0 < k_end && key0 <= qp_n) ? x0 : -INFINITY;
          x1 = (key0 + 1 < k_end && key0 + 1 <= qp_n) ? x1 : -INFINITY;
          *reinterpret_cast<float2*>(smma + n * 32 + kk) = make_float2(x0, x1);
          lmax = fmaxf(lmax, fmaxf(x0, x1));
        } else {
          *reinterpret_cast<float2*>(smma + n * 32 + nt * 8 + 2 * j) = make_float2(c[0], c[1]);
        }
      }
      if (lo_only) {
        lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, 1));
        lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, 2));
        if (j == 0 && n < 16) rmax_w[n] = lmax;
      }
      __syncwarp();
      if (!lo_only) {
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (!hi[r]) s[r] = smma[r * 32 + lane];
        __syncwarp();
      }
    } else if (need_lo) {
      if constexpr (LOW != kDecLow8) {
        const uint8_t* row = stage + S::sA + lane * (D / 2);
        const uint8_t* sf = stage + S::sAsf + lane * (S::kAsf / 32);
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          float2 x[16];
          float s0, s1;
          load_lo32_raw<LOW>(row, sf, c, x, s0, s1);
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (hi[r]) continue;
            const float* q = q_lo + r * D + 32 * c;
            s[r] = fmaf(dot_pairs<8>(q, x, 0), s0, s[r]);
            s[r] = fmaf(dot_pairs<8>(q, x, 8), s1, s[r]);
          }
        }
      }
    }
    if (need_hi) {
      // 8-bit low format: the staged rows are the high codes; otherwise the (rare) window /
      // sink groups read the high copy straight from global memory
      const bool staged = LOW == kDecLow8;
      const uint8_t* row = staged ? stage + S::sA + lane * D : p.k_hi + kr * D;
      const uint8_t* sf = staged ? stage + S::sAsf + lane * (D / 32) : p.k_hi_sf + kr * (D / 32);
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        float2 x[16];
        float sc;
        if (staged)
          load_hi32_raw<false>(row, sf, c, e5, x, sc);
        else
          load_hi32_raw<true>(row, sf, c, e5, x, sc);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (!hi[r]) continue;
          s[r] = fmaf(dot_pairs<16>(q_hi + r * D + 32 * c, x, 0), sc, s[r]);
        }
      }
    }
    // logits (base 2): S_q of both operands (MXFP4 low is single level: no S_q),
    // causal mask, online softmax per row
    const float sqk = static_cast<float>(reinterpret_cast<const double*>(stage + S::sSq)[lane]);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      bool vis;
      float x, gm;
      if (lo_only) {
        x = smma[r * 32 + lane];
        vis = x != -INFINITY;
        gm = rmax_w[r];
      } else {
        vis = in && static_cast<int>(j) <= qpos[r];
        const bool use_sq = hi[r] || LOW == kDecLowNV;
        x = use_sq ? s[r] * (sqq[r] * sqk) : s[r];
        x = vis ? x : -INFINITY;
        gm = x;
#pragma unroll
        for (int off = 16; off; off >>= 1) gm = fmaxf(gm, __shfl_xor_sync(0xffffffffu, gm, off));
      }
      const float mn = fmaxf(m[r], gm);
      float pv = 0.f;
      if (mn != -INFINITY) {
        const float alpha = exp2f(m[r] - mn);  // m = -inf -> 0
        pv = vis ? exp2f(x - mn) : 0.f;
        l[r] = l[r] * alpha + pv;              // lane-partial sum
#pragma unroll
        for (int c = 0; c < NP; ++c) o[r][c] = __fmul2_rn(o[r][c], make_float2(alpha, alpha));
        m[r] = mn;
      }
      ps[r * 32 + lane] = pv;
    }
    __syncwarp();
    // PV: lane owns value columns [DV/32 * lane, DV/32 * (lane + 1)), P of 4 keys per load
    const int nk = static_cast<int>((k_end - g0) < 32 ? (k_end - g0) : 32);
    const __nv_bfloat16* vst = reinterpret_cast<const __nv_bfloat16*>(stage + S::sV);
    auto pv_key = [&](int jj, const float* pr) {
      const __nv_bfloat16* vrow = vst + jj * DV + (DV / 32) * lane;
      float2 vv[NP];
      if constexpr (NP == 2) {
        const uint2 w = *reinterpret_cast<const uint2*>(vrow);
        vv[0] = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w.x));
        vv[1] = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w.y));
      } else {
        const uint32_t w = *reinterpret_cast<const uint32_t*>(vrow);
        vv[0] = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w));
      }
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int c = 0; c < NP; ++c) o[r][c] = __ffma2_rn(make_float2(pr[r], pr[r]), vv[c], o[r][c]);
    };
    int jj = 0;
#pragma unroll 2
    for (; jj + 4 <= nk; jj += 4) {
      float4 p4[R];
#pragma unroll
      for (int r = 0; r < R; ++r) p4[r] = *reinterpret_cast<const float4*>(ps + r * 32 + jj);
      float pr[R];
#pragma unroll
      for (int r = 0; r < R; ++r) pr[r] = p4[r].x;
      pv_key(jj, pr);
#pragma unroll
      for (int r = 0; r < R; ++r) pr[r] = p4[r].y;
      pv_key(jj + 1, pr);
#pragma unroll
      for (int r = 0; r < R; ++r) pr[r] = p4[r].z;
      pv_key(jj + 2, pr);
#pragma unroll
      for (int r = 0; r < R; ++r) pr[r] = p4[r].w;
      pv_key(jj + 3, pr);
    }
    for (; jj < nk; ++jj) {
      float pr[R];
#pragma unroll
      for (int r = 0; r < R; ++r) pr[r] = ps[r * 32 + jj];
      pv_key(jj, pr);
    }
    __syncwarp();
    // the stage is consumed: refill it with this warp's group kStages ahead
    if (lane == 0) {
      ptx::fence_proxy_async_smem();
      issue(st, g0 + 128 * S::kStages);
    }
  }

  // warp partials -> shared memory (over the rings: wait for every warp), merged per row
  __syncthreads();
  float2* ml = reinterpret_cast<float2*>(smem + S::oML);
  float* ow = reinterpret_cast<float*>(smem + S::oO);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    float ls = l[r];
#pragma unroll
    for (int off = 16; off; off >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, off);
    if (lane == 0) ml[warp * R + r] = make_float2(m[r], ls);
#pragma unroll
    for (int c = 0; c < NP; ++c)
      reinterpret_cast<float2*>(ow)[((warp * R + r) * DV + (DV / 32) * lane) / 2 + c] = o[r][c];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < R * DV; idx += blockDim.x) {
    const int r = idx / DV, c = idx % DV;
    const int64_t row = row_of(r);
    if (row < 0) continue;
    float mm = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) mm = fmaxf(mm, ml[w * R + r].x);
    float ls = 0.f, acc = 0.f;
    if (mm != -INFINITY) {
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const float2 x = ml[w * R + r];
        const float f = exp2f(x.x - mm);
        ls += x.y * f;
        acc += ow[(w * R + r) * DV + c] * f;
      }
    }
    const int64_t slot = row * p.splits + split;
    p.part_o[slot * DV + c] = acc;
    if (c == 0) p.part_ml[slot] = make_float2(mm, ls);
  }
}

// merge the splits of every query row: one warp per row
template <int DV>
__global__ void dma_decode_combine_kernel(const float* part_o, const float2* part_ml, int64_t rows, int splits,
                                          void* out, int out_bf16) {
  const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  float mm = -INFINITY;
  for (int s = 0; s < splits; ++s) mm = fmaxf(mm, part_ml[row * splits + s].x);
  float ls = 0.f, acc[DV / 32];
#pragma unroll
  for (int c = 0; c < DV / 32; ++c) acc[c] = 0.f;
  if (mm != -INFINITY) {
    for (int s = 0; s < splits; ++s) {
      const float2 x = part_ml[row * splits + s];
      const float f = exp2f(x.x - mm);
      ls += x.y * f;
#pragma unroll
      for (int c = 0; c < DV / 32; ++c) acc[c] += part_o[(row * splits + s) * DV + 32 * c + lane] * f;
    }
  }
  const float inv = ls > 0.f ? 1.f / ls : 1.f;  // attention.py:104-106 (l = 0 -> divide by 1)
#pragma unroll
  for (int c = 0; c < DV / 32; ++c) {
    const float v = acc[c] * inv;
    if (out_bf16)
      static_cast<__nv_bfloat16*>(out)[row * DV + 32 * c + lane] = __float2bfloat16_rn(v);
    else
      static_cast<float*>(out)[row * DV + 32 * c + lane] = v;
  }
}

}  // namespace dma
