// Phase 2 of the DMA forward: diagonal-tiled mixed-precision flash attention
// on sm_100a (tcgen05 block-scaled MMAs, TMEM accumulators, TMA loads).
//
// Restates attention.py:282-310 (tile loop) with the tile scheduler of
// attention.py:191-233 (Plan, common.cuh) and the base-2 online softmax of
// attention.py:150-175 (l0 = 0, dead rows keep alpha = 1, normalisation
// guard l > 0 from attention.py:104-106).
//
// Persistent kernel: one CTA per SM walks the work items (batch, head,
// 128-row query tile) in longest-first order (causal cost grows with the
// query tile), CTA c taking items c, c + grid, c + 2 grid, ...  Consecutive
// items share the query tile and differ in head, so co-resident CTAs of one
// GQA group read the same K/V tiles through L2.
//
// Warp roles (384 threads):
//   warp 0      TMA producer: Q (hi + lo codes, SF atoms) per item into a
//               2-deep ring, then per plan entry the K tile in the entry's
//               precision (+ SF + S_q^K) into a kNK ring and V (+ SF) into a
//               kNV ring
//   warp 1      MMA issuer (one thread): S = Q K^T (kind::mxf8f6f4 for high
//               tiles, kind::mxf4nvf4 4X / kind::mxf4 2X for low tiles) into
//               a double-buffered S in TMEM, one tile of look-ahead (also
//               across items); O += P V (kind::mxf8f6f4 with P read from TMEM,
//               or kind::f16 in the bf16 parity mode)
//   warps 4-7   softmax half 0: key columns [0, 64) of every S tile
//   warps 8-11  softmax half 1: key columns [64, 128)
//               Thread (half g, quadrant q, lane l) owns query row 32q + l.
//               Per tile: S_q^Q x S_q^K rescale, causal / ragged mask, row max
//               (exchanged with the partner half through shared memory), exp2,
//               P -> E4M3 (x 2^8) or bf16 written back into its own S columns
//               in TMEM, row sum, O rescale of its half of the O columns;
//               epilogue O / l of its O columns.
// TMEM (512 cols): S0 [0,128) S1 [128,256) O [256,256+DV) scale factors [384,436)
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>

#include "common.cuh"
#include "ptx.cuh"

namespace dma {

// kLowBF16: both score operands are bf16 copies of the reference's dequantized Q / K
// (S_q and the block scales folded in, or the identity path), QK by kind::f16 -- the
// route for BLOCK granularity (S_q varies along the contraction) and None formats.
enum LowKind { kLowNV = 0, kLowMX4 = 1, kLowHigh = 2, kLowBF16 = 3 };

struct __align__(64) AttnParams {
  CUtensorMap tm_q_hi, tm_q_lo, tm_k_hi, tm_k_lo, tm_v;
  const uint8_t* sf_q_hi;  // [mat_q][rt_q][ch_hi][512]
  const uint8_t* sf_q_lo;  // [mat_q][rt_q][ch_lo][512]
  const uint8_t* sf_k_hi;  // [mat_k][rt_k][ch_hi][512]
  const uint8_t* sf_k_lo;
  const uint8_t* sf_v;     // [mat_k][rt_k][512]
  const float* qs_q;       // [mat_q][lq_pad]
  const float* qs_k;       // [mat_k][lk_pad]
  void* o;                 // [B][H][Lq][DV]
  int out_bf16;
  int heads, kv_heads, group;  // group = heads / kv_heads
  int lq, lk, lq_pad, lk_pad;
  int n_qt, n_bh, n_items;
  int diag_window, sink_window, causal;
  int ch_hi, ch_lo;
  int hfmt;  // high-path element format: 0 = E4M3, 1 = E5M2
  int tile_m, tile_n;  // plan tile sizes (attention.py:51-80); the kernels' tiles are 128 x 128
};

template <int D, int DV, int LOW, bool PVBF16>
struct AttnCfg {
  static constexpr int kBM = 128, kBN = 128;
  static constexpr bool kBF = LOW == kLowBF16;
  static constexpr int kNQ = kBF ? 1 : 2, kNK = kBF ? 2 : 4, kNV = kBF ? 2 : 3;
  static constexpr int kQHiBytes = kBF ? kBM * D * 2 : kBM * D;
  static constexpr int kQLoBytes = kBF ? kBM * D * 2 : kBM * D / 2;
  static constexpr int kQStage = ((kQHiBytes + (LOW != kLowHigh ? kQLoBytes : 0) + 1023) / 1024) * 1024;
  static constexpr int kKBytes = kBF ? kBN * D * 2 : kBN * D;  // fp8 size; fp4 tiles use half
  static constexpr int kVBytes = PVBF16 ? kBN * DV * 2 : kBN * DV;
  static constexpr int kChHi = kBF ? 0 : (D / 32 + 3) / 4;
  static constexpr int kChLo = kBF ? 0 : (LOW == kLowNV ? (D / 16 + 3) / 4 : (D / 32 + 3) / 4);
  static constexpr int kChK = kChHi > kChLo ? kChHi : kChLo;
  // smem carve-up (offsets from a 1024-aligned base)
  static constexpr int oQ = 0;
  static constexpr int oK = oQ + kNQ * kQStage;
  static constexpr int oV = oK + kNK * kKBytes;
  static constexpr int oSmall = oV + kNV * kVBytes;
  static constexpr int oSfQ = oSmall;                        // [kNQ][kChHi + kChLo][512]
  static constexpr int kSfQStage = 512 * (kChHi + kChLo);
  static constexpr int oSfK = oSfQ + kNQ * kSfQStage;        // [kNK][kChK][512]
  static constexpr int oSqK = oSfK + kNK * 512 * kChK;       // [kNK][128] f32
  static constexpr int oSfV = oSqK + kNK * 512;              // [kNV][512]
  static constexpr int oSfP = oSfV + kNV * 512;              // 512
  static constexpr int oRed = oSfP + 512;                    // [2 buf][2 half][128] f32 row maxima
  static constexpr int oRedL = oRed + 2 * 2 * 128 * 4;       // [2 half][128] f32 row sums
  static constexpr int oBar = oRedL + 2 * 128 * 4;
  static constexpr int kSmemBytes = oBar + 256 + 1024;       // + alignment slack
  static_assert(kSmemBytes <= 227 * 1024, "smem budget");
  // TMEM columns
  static constexpr uint32_t tS0 = 0, tS1 = 128, tO = 256;
  static constexpr uint32_t tSfQ = 384;  // [kNQ][hi 4 | lo 8] = 24 cols
  static constexpr uint32_t tSfK = 408;  // [2][8]
  static constexpr uint32_t tSfV = 424;  // [2][4]
  static constexpr uint32_t tSfP = 432;  // 4
  static_assert(tSfP + 4 <= 512, "TMEM budget");
};

__device__ __forceinline__ uint32_t swz_mode(int row_bytes) {
  return row_bytes >= 128 ? ptx::kSw128 : (row_bytes == 64 ? ptx::kSw64 : ptx::kSw32);
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA pipe for a pair (x <= 0; masked -inf inputs never reach it):
// x = n + f with n = floor(x) (round-down add of 1.5*2^23), f in [0, 1);
// 2^f by a degree-4 polynomial (max rel. error 3e-6, below the E4M3 / bf16
// rounding of P), 2^n added to the exponent field.  Offloads MUFU.EX2
// (16/clk/SM), the softmax's throughput limit.
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  x.x = fmaxf(x.x, -127.f);
  x.y = fmaxf(x.y, -127.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);
  const float2 t = __fadd2_rd(x, magic);
  const float2 fl = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-fl.x, -fl.y));
  float2 p = __ffma2_rn(make_float2(0.013426235f, 0.013426235f), f, make_float2(0.052243195f, 0.052243195f));
  p = __ffma2_rn(p, f, make_float2(0.24127987f, 0.24127987f));
  p = __ffma2_rn(p, f, make_float2(0.6930449f, 0.6930449f));
  p = __ffma2_rn(p, f, make_float2(1.0f, 1.0f));
  return make_float2(__uint_as_float(__float_as_uint(p.x) + (__float_as_uint(t.x) << 23)),
                     __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(t.y) << 23)));
}

// work item w -> (bh, qt): longest causal query tiles first, heads innermost
__device__ __forceinline__ void item_coords(const AttnParams& p, int w, int& bh, int& qt) {
  const int r = w / p.n_bh;
  bh = w - r * p.n_bh;
  qt = p.causal ? p.n_qt - 1 - r : r;
}

#ifndef DMA_POLY_PAIRS
#define DMA_POLY_PAIRS 3  // 2 * DMA_POLY_PAIRS of every 16 exponentials go to the FMA pipe
#endif
constexpr int kPolyPairs = DMA_POLY_PAIRS;

template <int D, int DV, int LOW, bool PVBF16>
__global__ void __launch_bounds__(384, 1) dma_attn_kernel(const __grid_constant__ AttnParams p) {
  using C = AttnCfg<D, DV, LOW, PVBF16>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared address space
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::oBar);
  uint64_t* q_full = bars + 0;                // [kNQ]
  uint64_t* q_empty = q_full + C::kNQ;        // [kNQ]
  uint64_t* k_full = q_empty + C::kNQ;        // [kNK]
  uint64_t* k_empty = k_full + C::kNK;        // [kNK]
  uint64_t* v_full = k_empty + C::kNK;        // [kNV]
  uint64_t* v_empty = v_full + C::kNV;        // [kNV]
  uint64_t* s_full = v_empty + C::kNV;        // [2]
  uint64_t* p_full = s_full + 2;
  uint64_t* o_done = p_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rt_q = p.lq_pad >> 7, rt_k = p.lk_pad >> 7;

  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < C::kNQ; ++i) {
        ptx::mbar_init(q_full + i, 1);
        ptx::mbar_init(q_empty + i, 1);
      }
      for (int i = 0; i < C::kNK; ++i) {
        ptx::mbar_init(k_full + i, 1);
        ptx::mbar_init(k_empty + i, 1 + 8);  // MMA commit + the 8 softmax warps (S_q^K reads)
      }
      for (int i = 0; i < C::kNV; ++i) {
        ptx::mbar_init(v_full + i, 1);
        ptx::mbar_init(v_empty + i, 1);
      }
      ptx::mbar_init(s_full + 0, 1);
      ptx::mbar_init(s_full + 1, 1);
      ptx::mbar_init(p_full, 8);  // one arrive per softmax warp
      ptx::mbar_init(o_done, 1);
      ptx::fence_barrier_init();
      ptx::tma_prefetch_desc(&p.tm_q_hi);
      ptx::tma_prefetch_desc(&p.tm_k_hi);
      ptx::tma_prefetch_desc(&p.tm_v);
      if (LOW != kLowHigh) {
        ptx::tma_prefetch_desc(&p.tm_q_lo);
        ptx::tma_prefetch_desc(&p.tm_k_lo);
      }
    }
  } else if (warp == 1) {
    ptx::tmem_alloc<512>(tmem_slot);
  } else if (warp == 2 && !PVBF16) {
    // constant P scale-factor atom: E8M0 127 (= 1.0) for every row / k-block
    uint32_t* sfp = reinterpret_cast<uint32_t*>(smem + C::oSfP);
    for (int i = lane; i < 128; i += 32) sfp[i] = 0x7F7F7F7Fu;
    ptx::fence_proxy_async_smem();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // =========================== TMA producer ===========================
    {  // whole warp: issue ops elect one lane inside the asm (ptx::wu)
      uint32_t kc = 0, vc = 0, ic = 0;  // ring counters (continue across items)
      for (int w = blockIdx.x; w < p.n_items; w += gridDim.x) {
        int bh, qt;
        item_coords(p, w, bh, qt);
        const int b = bh / p.heads, h = bh % p.heads;
        const int mat_q = bh, mat_k = b * p.kv_heads + h / p.group;
        Plan2 plan;
        plan.init(qt, p.lq, p.lk, p.tile_m, p.tile_n, p.diag_window, p.sink_window, p.causal != 0);
        if (plan.n == 0) continue;  // nothing to load (the softmax side writes zeros)
        const int qs = ic % C::kNQ;
        ++ic;
        ptx::mbar_wait(q_empty + qs, (((ic - 1) / C::kNQ) & 1) ^ 1);
        uint32_t qbytes = C::kQHiBytes + 512 * C::kChHi;
        if (LOW != kLowHigh) qbytes += C::kQLoBytes + 512 * C::kChLo;
        uint8_t* qdst = smem + C::oQ + qs * C::kQStage;
        uint8_t* sfq = smem + C::oSfQ + qs * C::kSfQStage;
        ptx::wu::mbar_arrive_expect_tx(q_full + qs, qbytes);
        if constexpr (C::kBF) {
          // bf16 operands: 64-column (128-byte) swizzle boxes, hi then lo
#pragma unroll
          for (int hb = 0; hb < D / 64; ++hb) {
            ptx::wu::tma_load_3d(qdst + hb * (C::kBM * 128), &p.tm_q_hi, q_full + qs, hb * 64, qt * C::kBM, mat_q);
            ptx::wu::tma_load_3d(qdst + C::kQHiBytes + hb * (C::kBM * 128), &p.tm_q_lo, q_full + qs, hb * 64, qt * C::kBM,
                             mat_q);
          }
        } else {
        ptx::wu::tma_load_3d(qdst, &p.tm_q_hi, q_full + qs, 0, qt * C::kBM, mat_q);
        ptx::wu::bulk_load(sfq, p.sf_q_hi + (static_cast<int64_t>(mat_q) * rt_q + qt) * p.ch_hi * 512,
                       512 * C::kChHi, q_full + qs);
        if (LOW != kLowHigh) {
          ptx::wu::tma_load_3d(qdst + C::kQHiBytes, &p.tm_q_lo, q_full + qs, 0, qt * C::kBM, mat_q);
          ptx::wu::bulk_load(sfq + 512 * C::kChHi, p.sf_q_lo + (static_cast<int64_t>(mat_q) * rt_q + qt) * p.ch_lo * 512,
                         512 * C::kChLo, q_full + qs);
        }
        }
        for (int e = 0; e < plan.n; ++e, ++kc, ++vc) {
          int t;
          bool hi;
          uint32_t keep;
          plan.entry(e, qt, t, hi, keep);
          if (LOW == kLowHigh) hi = true;
          const int ks = kc % C::kNK;
          ptx::mbar_wait(k_empty + ks, ((kc / C::kNK) & 1) ^ 1);
          const int ch = hi ? C::kChHi : C::kChLo;
          const uint32_t kb = (hi || C::kBF) ? C::kKBytes : C::kKBytes / 2;
          ptx::wu::mbar_arrive_expect_tx(k_full + ks, kb + 512 * ch + 512);
          if constexpr (C::kBF) {
#pragma unroll
            for (int hb = 0; hb < D / 64; ++hb)
              ptx::wu::tma_load_3d(smem + C::oK + ks * C::kKBytes + hb * (C::kBN * 128), hi ? &p.tm_k_hi : &p.tm_k_lo,
                               k_full + ks, hb * 64, t * C::kBN, mat_k);
          } else {
          ptx::wu::tma_load_3d(smem + C::oK + ks * C::kKBytes, hi ? &p.tm_k_hi : &p.tm_k_lo, k_full + ks, 0,
                           t * C::kBN, mat_k);
          const uint8_t* sfsrc = (hi ? p.sf_k_hi : p.sf_k_lo) +
                                 (static_cast<int64_t>(mat_k) * rt_k + t) * (hi ? p.ch_hi : p.ch_lo) * 512;
          ptx::wu::bulk_load(smem + C::oSfK + ks * 512 * C::kChK, sfsrc, 512 * ch, k_full + ks);
          }
          ptx::wu::bulk_load(smem + C::oSqK + ks * 512, p.qs_k + static_cast<int64_t>(mat_k) * p.lk_pad + t * C::kBN,
                         512, k_full + ks);

          const int vs = vc % C::kNV;
          ptx::mbar_wait(v_empty + vs, ((vc / C::kNV) & 1) ^ 1);
          uint8_t* vdst = smem + C::oV + vs * C::kVBytes;
          if (PVBF16) {
            ptx::wu::mbar_arrive_expect_tx(v_full + vs, C::kVBytes);
#pragma unroll
            for (int half = 0; half < DV / 64; ++half)
              ptx::wu::tma_load_3d(vdst + half * (C::kBN * 128), &p.tm_v, v_full + vs, half * 64, t * C::kBN, mat_k);
          } else {
            ptx::wu::mbar_arrive_expect_tx(v_full + vs, C::kVBytes + 512);
            ptx::wu::tma_load_3d(vdst, &p.tm_v, v_full + vs, 0, t * C::kBN, mat_k);
            ptx::wu::bulk_load(smem + C::oSfV + vs * 512, p.sf_v + (static_cast<int64_t>(mat_k) * rt_k + t) * 512, 512,
                           v_full + vs);
          }
        }
      }
    }
  } else if (warp == 1) {
    // =========================== MMA issuer ===========================
    {  // whole warp: issue ops elect one lane inside the asm (ptx::wu)
      if (!PVBF16)
        ptx::wu::tc_cp_sf(tmem + C::tSfP, ptx::smem_desc(ptx::smem_u32(smem + C::oSfP), 0, 128, ptx::kSwNone));
      // The tile stream of this CTA, flattened across items.  QK of tile
      // (g + 1) is issued before the PV of tile g (S is double buffered).
      struct Cursor {
        int w = 0, e = 0, n = 0, qt = 0;
        uint32_t ic = 0;  // item ordinal in this CTA
        Plan2 plan;
      };
      auto load_item = [&](Cursor& c) {  // advance c to the first item with a non-empty plan
        while (c.w < p.n_items) {
          int bh, qt;
          item_coords(p, c.w, bh, qt);
          c.plan.init(qt, p.lq, p.lk, p.tile_m, p.tile_n, p.diag_window, p.sink_window, p.causal != 0);
          c.qt = qt;
          c.n = c.plan.n;
          c.e = 0;
          if (c.n > 0) return true;
          c.w += gridDim.x;  // empty plan: nothing to issue (the softmax side writes zeros)
        }
        return false;
      };
      uint32_t kc = 0, vc = 0, g = 0;  // ring counters, tile ordinal
      Cursor cq;  // next QK to issue
      cq.w = blockIdx.x;
      bool more = load_item(cq);

      auto issue_qk = [&](Cursor& c, uint32_t tile_ord) {
        const int qs = c.ic % C::kNQ;
        if (c.e == 0) {
          ptx::mbar_wait(q_full + qs, (c.ic / C::kNQ) & 1);
          ptx::tc_fence_after();
          const uint8_t* sfq = smem + C::oSfQ + qs * C::kSfQStage;
          for (int j = 0; j < C::kChHi; ++j)
            ptx::wu::tc_cp_sf(tmem + C::tSfQ + 12 * qs + 4 * j,
                          ptx::smem_desc(ptx::smem_u32(sfq + 512 * j), 0, 128, ptx::kSwNone));
          if (LOW != kLowHigh)
            for (int j = 0; j < C::kChLo; ++j)
              ptx::wu::tc_cp_sf(tmem + C::tSfQ + 12 * qs + 4 + 4 * j,
                            ptx::smem_desc(ptx::smem_u32(sfq + 512 * (C::kChHi + j)), 0, 128, ptx::kSwNone));
        }
        int t;
        bool hi;
        uint32_t keep;
        c.plan.entry(c.e, c.qt, t, hi, keep);
        if (LOW == kLowHigh) hi = true;
        const int ks = kc % C::kNK;
        ptx::mbar_wait(k_full + ks, (kc / C::kNK) & 1);
        ptx::tc_fence_after();
        const uint32_t tsfk = tmem + C::tSfK + 8 * (tile_ord & 1);
        const int ch = hi ? C::kChHi : C::kChLo;
        for (int j = 0; j < ch; ++j)
          ptx::wu::tc_cp_sf(tsfk + 4 * j, ptx::smem_desc(ptx::smem_u32(smem + C::oSfK + ks * 512 * C::kChK + 512 * j),
                                                     0, 128, ptx::kSwNone));
        const uint32_t tS = tmem + ((tile_ord & 1) ? C::tS1 : C::tS0);
        const uint32_t kaddr = ptx::smem_u32(smem + C::oK + ks * C::kKBytes);
        const uint32_t qaddr = ptx::smem_u32(smem + C::oQ + qs * C::kQStage);
        const uint32_t tsfq = tmem + C::tSfQ + 12 * qs;
        if constexpr (C::kBF) {
          // bf16 x bf16 -> f32, K = 16 per MMA; 128-byte swizzle atoms of 64 columns, 16 KB apart
          const uint32_t qb = qaddr + (hi ? 0u : static_cast<uint32_t>(C::kQHiBytes));
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = 32 * (kk & 3) + (C::kBM * 128) * (kk >> 2);
            const uint64_t ad = ptx::smem_desc(qb + off, 16, 1024, ptx::kSw128);
            const uint64_t bd = ptx::smem_desc(kaddr + off, 16, 1024, ptx::kSw128);
            ptx::wu::mma_f16_ss(tS, ad, bd, ptx::idesc_bf16(0, 0, 128, 128), kk > 0);
          }
        } else if (hi) {
          constexpr int rb = D;  // fp8 row bytes
          const uint32_t sw = swz_mode(rb);
#pragma unroll
          for (int kk = 0; kk < D / 32; ++kk) {
            const uint64_t ad = ptx::smem_desc(qaddr + 32 * kk, 16, 8 * rb, sw);
            const uint64_t bd = ptx::smem_desc(kaddr + 32 * kk, 16, 8 * rb, sw);
            const uint32_t f = static_cast<uint32_t>(p.hfmt);
            const uint32_t id = ptx::idesc_bs(f, f, 0, 0, 128, 128, 1, kk & 3, kk & 3);
            ptx::wu::mma_mxf8f6f4(tS, ad, bd, id, tsfq + 4 * (kk >> 2), tsfk + 4 * (kk >> 2), kk > 0);
          }
        } else {
          const uint32_t qlo = qaddr + C::kQHiBytes;
          constexpr int rb = D / 2;  // packed fp4 row bytes
          const uint32_t sw = swz_mode(rb);
#pragma unroll
          for (int kk = 0; kk < D / 64; ++kk) {
            const uint64_t ad = ptx::smem_desc(qlo + 32 * kk, 16, 8 * rb, sw);
            const uint64_t bd = ptx::smem_desc(kaddr + 32 * kk, 16, 8 * rb, sw);
            if (LOW == kLowNV) {
              const uint32_t id = ptx::idesc_bs(1, 1, 0, 0, 128, 128, 0, 0, 0);
              ptx::wu::mma_nvf4(tS, ad, bd, id, tsfq + 4 + 4 * kk, tsfk + 4 * kk, kk > 0);
            } else {
              const uint32_t sid = (kk & 1) * 2;
              const uint32_t id = ptx::idesc_bs(1, 1, 0, 0, 128, 128, 1, sid, sid);
              ptx::wu::mma_mxf4(tS, ad, bd, id, tsfq + 4 + 4 * (kk >> 1), tsfk + 4 * (kk >> 1), kk > 0);
            }
          }
        }
        ptx::wu::tc_commit(k_empty + ks);
        ptx::wu::tc_commit(s_full + (tile_ord & 1));
        ++kc;
        if (++c.e == c.n) {
          ptx::wu::tc_commit(q_empty + qs);  // Q smem free once these MMAs complete
          c.w += gridDim.x;
          ++c.ic;
          return load_item(c);
        }
        return true;
      };

      // PV cursor trails the QK cursor by one tile
      Cursor cp = cq;
      if (more) more = issue_qk(cq, 0);
      bool pv_more = cp.w < p.n_items && cp.n > 0;
      while (pv_more) {
        if (more) more = issue_qk(cq, g + 1);
        ptx::mbar_wait(p_full, g & 1);
        ptx::tc_fence_after();
        const int vs = vc % C::kNV;
        ptx::mbar_wait(v_full + vs, (vc / C::kNV) & 1);
        ptx::tc_fence_after();
        const uint32_t tP = tmem + ((g & 1) ? C::tS1 : C::tS0);
        const uint32_t vaddr = ptx::smem_u32(smem + C::oV + vs * C::kVBytes);
        const bool first = cp.e == 0;
        if (PVBF16) {
#pragma unroll
          for (int kk = 0; kk < C::kBN / 16; ++kk) {
            const uint64_t bd = ptx::smem_desc(vaddr + kk * 16 * 128, C::kBN * 128, 1024, ptx::kSw128);
            const uint32_t pa = tP + 64 * (kk >> 2) + 8 * (kk & 3);
            ptx::wu::mma_f16_ts(tmem + C::tO, pa, bd, ptx::idesc_bf16(0, 1, 128, DV), !(first && kk == 0));
          }
        } else {
          const uint32_t tsfv = tmem + C::tSfV + 4 * (g & 1);
          ptx::wu::tc_cp_sf(tsfv, ptx::smem_desc(ptx::smem_u32(smem + C::oSfV + vs * 512), 0, 128, ptx::kSwNone));
          constexpr int rb = DV;  // fp8 V row bytes (MN-major)
#pragma unroll
          for (int kk = 0; kk < C::kBN / 32; ++kk) {
            const uint64_t bd = ptx::smem_desc(vaddr + kk * 32 * rb, 16, 8 * rb, swz_mode(rb));
            const uint32_t id = ptx::idesc_bs(0, 0, 0, 1, 128, DV, 1, kk & 3, kk & 3);
            const uint32_t pa = tP + 64 * (kk >> 1) + 8 * (kk & 1);
            ptx::wu::mma_mxf8f6f4_ts(tmem + C::tO, pa, bd, id, tmem + C::tSfP, tsfv, !(first && kk == 0));
          }
        }
        ptx::wu::tc_commit(v_empty + vs);
        ptx::wu::tc_commit(o_done);
        ++vc;
        ++g;
        if (++cp.e == cp.n) {
          cp.w += gridDim.x;
          ++cp.ic;
          pv_more = load_item(cp);
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // =========================== softmax / correction / epilogue ===========================
    const int half = (warp - 4) >> 2;          // key columns [64 half, 64 half + 64)
    const int quad = warp & 3;                  // TMEM lane quadrant
    const int r = quad * 32 + lane;             // query row within the tile == TMEM lane
    const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t bar_id = 1 + quad;           // partner warps (4 + quad, 8 + quad)
    float* red = reinterpret_cast<float*>(smem + C::oRed);
    float* red_l = reinterpret_cast<float*>(smem + C::oRedL);
    // MXFP8 PV: lazy rescaling as in attn_pp.cuh (a row keeps its max until a tile raises
    // it by more than kLazy), P <= 2^kLazy stored as E4M3(P * 2^(8 - kLazy)); bf16 PV: exact max
    constexpr float kLazy = PVBF16 ? 0.f : 4.f;
    constexpr float kPShift = PVBF16 ? 0.f : 8.f - kLazy;
    constexpr int kOC = DV / 2;                     // O columns owned by this half
    uint32_t g = 0;                                 // tile ordinal (matches the MMA issuer)

    for (int w = blockIdx.x; w < p.n_items; w += gridDim.x) {
      int bh, qt;
      item_coords(p, w, bh, qt);
      const int q0 = qt * C::kBM;
      const int qrow = q0 + r;
      Plan2 plan;
      plan.init(qt, p.lq, p.lk, p.tile_m, p.tile_n, p.diag_window, p.sink_window, p.causal != 0);
      const float sq_q = (qrow < p.lq) ? p.qs_q[static_cast<int64_t>(bh) * p.lq_pad + qrow] : 1.0f;
      float m_run = -INFINITY;
      float2 l2 = make_float2(0.f, 0.f);

      for (int e = 0; e < plan.n; ++e, ++g) {
        int t;
        bool hi;
        uint32_t keep;
        plan.entry(e, qt, t, hi, keep);
        // quadrant kept by this entry (64-row half a of the tile, 64-column half of this warp)
        const bool kept = (keep >> (2 * (r >> 6) + half)) & 1u;
        if (LOW == kLowHigh) hi = true;
        const bool two_level = (LOW != kLowBF16) && (hi || (LOW == kLowNV));  // bf16 operands: S_q folded in
        const int k0 = t * C::kBN;
        ptx::mbar_wait(s_full + (g & 1), (g >> 1) & 1);
        ptx::tc_fence_after();
        const uint32_t tS = tmem + ((g & 1) ? C::tS1 : C::tS0) + lane_base + 64 * half;
        float s[64];
        {
          uint32_t r0[32], r1[32];
          ptx::tmem_ld32(tS, r0);
          ptx::tmem_ld32(tS + 32, r1);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            s[i] = __uint_as_float(r0[i]);
            s[32 + i] = __uint_as_float(r1[i]);
          }
        }
        // S_q^K column factors for two-level tiles (staged by the producer with the K tile)
        const float rowf = two_level ? sq_q : 1.0f;
        if (two_level) {
          const uint32_t sqk = ptx::smem_u32(smem + C::oSqK + ((g % C::kNK) * 512)) + 256 * half;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float4 f = ptx::lds_f4(sqk + 16 * j);
            float2 a = __fmul2_rn(make_float2(s[4 * j], s[4 * j + 1]), make_float2(f.x, f.y));
            float2 b = __fmul2_rn(make_float2(s[4 * j + 2], s[4 * j + 3]), make_float2(f.z, f.w));
            s[4 * j] = a.x; s[4 * j + 1] = a.y; s[4 * j + 2] = b.x; s[4 * j + 3] = b.y;
          }
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(k_empty + (g % C::kNK));  // done with this K slot's S_q^K
        // causal (attention.py:178-184, applied when k1-1 > q0, :306) and ragged-key masks
        const int kvalid = p.lk - k0;  // keys [k0, k0+kvalid) exist
        const bool need_causal = p.causal && (k0 + (kvalid < C::kBN ? kvalid : C::kBN) - 1 > q0);
        const bool masked = need_causal || kvalid < C::kBN || keep != 0xFu;
        if (masked) {
          const int lim = !kept ? 0 : (need_causal ? min(qrow - k0 + 1, kvalid) : kvalid) - 64 * half;  // keep j < lim
#pragma unroll
          for (int j = 0; j < 64; ++j)
            if (j >= lim) s[j] = -INFINITY;
        }
        float mx = fmaxf(s[0], s[1]);
#pragma unroll
        for (int j = 2; j < 64; j += 2) mx = ptx::fmax3(mx, s[j], s[j + 1]);
        // row max across the two halves
        float* rb = red + (g & 1) * 256;
        rb[half * 128 + r] = mx;
        ptx::named_bar_sync(bar_id, 64);
        mx = fmaxf(mx, rb[(half ^ 1) * 128 + r]);
        const float m_tile = mx * rowf;
        const float m_cand = fmaxf(m_run, m_tile);
        const bool upd = PVBF16 ? true : (m_cand > m_run + kLazy);  // always for the first live tile
        const float m_new = upd ? m_cand : m_run;
        const bool dead = (m_new == -INFINITY);
        const float alpha = (dead || !upd) ? 1.0f : fast_exp2(m_run - m_new);  // m_run = -inf -> 0
        const float bias = dead ? 0.f : (kPShift - m_new);
        const float2 rf2 = make_float2(rowf, rowf), b2 = make_float2(bias, bias);
        float2 ls = make_float2(0.f, 0.f);
        const uint32_t tP = tmem + ((g & 1) ? C::tS1 : C::tS0) + lane_base + 64 * half;
        if (PVBF16) {
          uint32_t pk[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            float2 x = __ffma2_rn(make_float2(s[2 * j], s[2 * j + 1]), rf2, b2);
            x.x = fast_exp2(x.x);
            x.y = fast_exp2(x.y);
            ls = __fadd2_rn(ls, x);
            __nv_bfloat162 v = __floats2bfloat162_rn(x.x, x.y);
            pk[j] = *reinterpret_cast<uint32_t*>(&v);
          }
          ptx::tmem_st32(tP, pk);
        } else {
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float2 x0 = __ffma2_rn(make_float2(s[4 * j], s[4 * j + 1]), rf2, b2);
            float2 x1 = __ffma2_rn(make_float2(s[4 * j + 2], s[4 * j + 3]), rf2, b2);
            if (!masked && (j % 4) < kPolyPairs) {  // FMA-pipe exp2 on a fixed share of the pairs
              x0 = exp2_poly2(x0);
            } else {
              x0.x = fast_exp2(x0.x);
              x0.y = fast_exp2(x0.y);
            }
            x1.x = fast_exp2(x1.x);
            x1.y = fast_exp2(x1.y);
            ls = __fadd2_rn(ls, __fadd2_rn(x0, x1));
            pk[j] = static_cast<uint32_t>(ptx::cvt_e4m3x2(x0.x, x0.y)) |
                    (static_cast<uint32_t>(ptx::cvt_e4m3x2(x1.x, x1.y)) << 16);
          }
          ptx::tmem_st16(tP, pk);
        }
        l2 = __ffma2_rn(l2, make_float2(alpha, alpha), ls);
        m_run = m_new;
        // O *= alpha once the previous PV has landed (rows whose max moved)
        if (e > 0) {
          ptx::mbar_wait(o_done, (g - 1) & 1);
          ptx::tc_fence_after();
          if (__any_sync(0xffffffffu, alpha != 1.0f)) {
            const uint32_t tO = tmem + C::tO + lane_base + kOC * half;
            const float2 a2 = make_float2(alpha, alpha);
#pragma unroll
            for (int c = 0; c < kOC / 32; ++c) {
              uint32_t rr[32];
              ptx::tmem_ld32(tO + 32 * c, rr);
              ptx::tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                float2 v = __fmul2_rn(make_float2(__uint_as_float(rr[2 * i]), __uint_as_float(rr[2 * i + 1])), a2);
                rr[2 * i] = __float_as_uint(v.x);
                rr[2 * i + 1] = __float_as_uint(v.y);
              }
              ptx::tmem_st32(tO + 32 * c, rr);
            }
          }
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(p_full);
      }

      // ---- epilogue: O / l (attention.py:104-106); l = sum of both halves
      float l_part = l2.x + l2.y;
      red_l[half * 128 + r] = l_part;
      ptx::named_bar_sync(bar_id, 64);
      const float l_run = l_part + red_l[(half ^ 1) * 128 + r];
      ptx::named_bar_sync(bar_id, 64);  // red_l reusable by the next item
      const float inv_l = 1.0f / (l_run > 0.f ? l_run : 1.0f);
      if (plan.n > 0) {
        ptx::mbar_wait(o_done, (g - 1) & 1);
        ptx::tc_fence_after();
      }
      const uint32_t tO = tmem + C::tO + lane_base + kOC * half;
      const int64_t orow = static_cast<int64_t>(bh) * p.lq + qrow;
#pragma unroll
      for (int c = 0; c < kOC / 32; ++c) {
        uint32_t rr[32];
        if (plan.n > 0) {
          ptx::tmem_ld32(tO + 32 * c, rr);
          ptx::tmem_ld_wait();
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) rr[i] = 0u;
        }
        if (qrow < p.lq) {
          const int col = kOC * half + 32 * c;
          if (p.out_bf16) {
            uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.o) + orow * DV + col);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              uint32_t wv[4];
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                __nv_bfloat162 v = __floats2bfloat162_rn(__uint_as_float(rr[8 * i + 2 * k]) * inv_l,
                                                         __uint_as_float(rr[8 * i + 2 * k + 1]) * inv_l);
                wv[k] = *reinterpret_cast<uint32_t*>(&v);
              }
              dst[i] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
            }
          } else {
            float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.o) + orow * DV + col);
#pragma unroll
            for (int i = 0; i < 8; ++i)
              dst[i] = make_float4(__uint_as_float(rr[4 * i]) * inv_l, __uint_as_float(rr[4 * i + 1]) * inv_l,
                                   __uint_as_float(rr[4 * i + 2]) * inv_l, __uint_as_float(rr[4 * i + 3]) * inv_l);
          }
        }
      }
      // the next item's first PV overwrites O: the p_full arrive of its first tile
      // (issued after these tcgen05.ld completed) orders it after this read
      ptx::tc_fence_before();
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc<512>(tmem);
}

}  // namespace dma
