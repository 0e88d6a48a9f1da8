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

#include "common.cuh"

namespace dma {

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

// shared memory: dequantized query rows (low, high) [R][D] f32, P [4 warps][R][32],
// warp partials (m, l) [4][R] and O [4][R][DV]
template <int R, int D, int DV>
struct DecSmem {
  static constexpr int oQlo = 0;
  static constexpr int oQhi = oQlo + R * D * 4;
  static constexpr int oP = oQhi + R * D * 4;
  static constexpr int oML = oP + 4 * R * 32 * 4;
  static constexpr int oO = oML + 4 * R * 8;
  static constexpr int kBytes = oO + 4 * R * DV * 4;
};

template <int R, int D, int DV, int LOW>
__global__ void __launch_bounds__(128) dma_decode_kernel(const DecodeParams p) {
  using S = DecSmem<R, D, DV>;
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
  int64_t qpos[R];  // absolute position of the row
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
      qpos[r] = p.pos + i;
      const int64_t q0 = (qpos[r] / p.tile_m) * p.tile_m;
      hs[r] = static_cast<int>(ceil_div(q0 - p.diag_window, static_cast<int64_t>(p.tile_n)));
      sqq[r] = static_cast<float>(p.q_sq[qrow[r]]);
    } else {
      qrow[r] = -1;
      qpos[r] = -1;
      hs[r] = 0;
      sqq[r] = 0.f;
    }
  }
  // dequantize the query rows (block scales only; S_q folds in per logit)
  for (int idx = threadIdx.x; idx < R * (D / 32); idx += blockDim.x) {
    const int r = idx / (D / 32), c = idx % (D / 32);
    float x[32];
    const int64_t qr = row_of(r);
    if (qr >= 0) {
      if (LOW != kDecLow8) {
        load_lo32<LOW>(p.q_lo + qr * (D / 2), p.q_lo_sf + qr * (D / (LOW == kDecLowNV ? 16 : 32)), c, x);
#pragma unroll
        for (int j = 0; j < 32; ++j) q_lo[r * D + 32 * c + j] = x[j];
      }
      load_hi32(p.q_hi + qr * D, p.q_hi_sf + qr * (D / 32), c, e5, x);
#pragma unroll
      for (int j = 0; j < 32; ++j) q_hi[r * D + 32 * c + j] = x[j];
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) q_lo[r * D + 32 * c + j] = q_hi[r * D + 32 * c + j] = 0.f;
    }
  }
  __syncthreads();

  int64_t last = -1;  // last visible key of any row
#pragma unroll
  for (int r = 0; r < R; ++r) last = qpos[r] > last ? qpos[r] : last;
  const int64_t k_begin = static_cast<int64_t>(split) * p.keys_per_split;
  int64_t k_end = k_begin + p.keys_per_split;
  k_end = k_end < last + 1 ? k_end : last + 1;

  float m[R], l[R], o[R][DV / 32];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    m[r] = -INFINITY;
    l[r] = 0.f;
#pragma unroll
    for (int c = 0; c < DV / 32; ++c) o[r][c] = 0.f;
  }
  float* ps = reinterpret_cast<float*>(smem + S::oP) + warp * R * 32;
  const int64_t krow0 = static_cast<int64_t>(mk) * p.cap;

  for (int64_t g0 = k_begin + 32 * warp; g0 < k_end; g0 += 128) {
    const int64_t j = g0 + lane;
    const bool in = j < k_end;
    const int t = static_cast<int>(g0 / p.tile_n);  // the 32-key group lies in one key tile
    bool hi[R];
    bool need_lo = false, need_hi = false;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      hi[r] = LOW == kDecLow8 || t < sink_t || t >= hs[r];
      if (qrow[r] >= 0 && g0 <= qpos[r]) (hi[r] ? need_hi : need_lo) = true;
    }
    const int64_t kr = krow0 + (in ? j : k_begin);
    float s[R];
#pragma unroll
    for (int r = 0; r < R; ++r) s[r] = 0.f;
    if (need_lo) {
      if constexpr (LOW != kDecLow8) {
        const uint8_t* row = p.k_lo + kr * (D / 2);
        const uint8_t* sf = p.k_lo_sf + kr * (D / (LOW == kDecLowNV ? 16 : 32));
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          float x[32];
          load_lo32<LOW>(row, sf, c, x);
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (hi[r]) continue;
            const float4* q4 = reinterpret_cast<const float4*>(q_lo + r * D + 32 * c);
            float acc = s[r];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float4 qv = q4[e];
              acc = fmaf(qv.x, x[4 * e], acc);
              acc = fmaf(qv.y, x[4 * e + 1], acc);
              acc = fmaf(qv.z, x[4 * e + 2], acc);
              acc = fmaf(qv.w, x[4 * e + 3], acc);
            }
            s[r] = acc;
          }
        }
      }
    }
    if (need_hi) {
      const uint8_t* row = p.k_hi + kr * D;
      const uint8_t* sf = p.k_hi_sf + kr * (D / 32);
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        float x[32];
        load_hi32(row, sf, c, e5, x);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (!hi[r]) continue;
          const float4* q4 = reinterpret_cast<const float4*>(q_hi + r * D + 32 * c);
          float acc = s[r];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float4 qv = q4[e];
            acc = fmaf(qv.x, x[4 * e], acc);
            acc = fmaf(qv.y, x[4 * e + 1], acc);
            acc = fmaf(qv.z, x[4 * e + 2], acc);
            acc = fmaf(qv.w, x[4 * e + 3], acc);
          }
          s[r] = acc;
        }
      }
    }
    // logits (base 2): S_q of both operands (MXFP4 low is single level: no S_q),
    // causal mask, online softmax per row
    const float sqk = static_cast<float>(p.k_sq[kr]);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const bool vis = in && qrow[r] >= 0 && j <= qpos[r];
      const bool use_sq = hi[r] || LOW == kDecLowNV;
      float x = use_sq ? s[r] * (sqq[r] * sqk) : s[r];
      x = vis ? x : -INFINITY;
      float gm = x;
#pragma unroll
      for (int off = 16; off; off >>= 1) gm = fmaxf(gm, __shfl_xor_sync(0xffffffffu, gm, off));
      const float mn = fmaxf(m[r], gm);
      float pv = 0.f;
      if (mn != -INFINITY) {
        const float alpha = exp2f(m[r] - mn);  // m = -inf -> 0
        pv = vis ? exp2f(x - mn) : 0.f;
        l[r] = l[r] * alpha + pv;              // lane-partial sum
#pragma unroll
        for (int c = 0; c < DV / 32; ++c) o[r][c] *= alpha;
        m[r] = mn;
      }
      ps[r * 32 + lane] = pv;
    }
    __syncwarp();
    // PV: lane owns value columns [DV/32 * lane, DV/32 * (lane + 1))
    const int nk = static_cast<int>((k_end - g0) < 32 ? (k_end - g0) : 32);
#pragma unroll 4
    for (int jj = 0; jj < nk; ++jj) {
      const __nv_bfloat16* vrow = p.v + (krow0 + g0 + jj) * DV + (DV / 32) * lane;
      float vv[DV / 32];
      if constexpr (DV == 128) {
        const uint2 w = __ldg(reinterpret_cast<const uint2*>(vrow));
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w.x));
        const float2 c = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w.y));
        vv[0] = a.x; vv[1] = a.y; vv[2] = c.x; vv[3] = c.y;
      } else {
        const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(vrow));
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w));
        vv[0] = a.x; vv[1] = a.y;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const float pr = ps[r * 32 + jj];
#pragma unroll
        for (int c = 0; c < DV / 32; ++c) o[r][c] = fmaf(pr, vv[c], o[r][c]);
      }
    }
    __syncwarp();
  }

  // warp partials -> shared memory, merged per row by all 128 threads
  float2* ml = reinterpret_cast<float2*>(smem + S::oML);
  float* ow = reinterpret_cast<float*>(smem + S::oO);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    float ls = l[r];
#pragma unroll
    for (int off = 16; off; off >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, off);
    if (lane == 0) ml[warp * R + r] = make_float2(m[r], ls);
#pragma unroll
    for (int c = 0; c < DV / 32; ++c) ow[(warp * R + r) * DV + (DV / 32) * lane + c] = o[r][c];
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
