// Phase 2 of the DMA forward, split-KV variant (block-scaled MXFP8 PV) -- an EXPERIMENT,
// selected with DMA_ATTN_KERNEL=sk; correct (the parity suite passes on it) but slower
// than attn_pp.cuh at c2 / c3: the per-warp critical path is longer,
// the two warpgroups' exp phases phase-lock, and 128 live scores + the pipelined next
// tile do not fit the 216-register budget without spills.
//
// Same algorithm as attn_pp.cuh (attention.py:282-310, plans of attention.py:
// 191-233, base-2 online softmax of :150-175 with lazy rescaling), organised so
// that the two softmax warpgroups never wait on each other's TMEM traffic:
//
//   * a work item is ONE 128-row query tile (b, h, qt); its plan entries are
//     split between the warpgroups by parity: WG0 takes entries 0, 2, 4, ...,
//     WG1 entries 1, 3, 5, ...;
//   * each warpgroup owns an S buffer and a P buffer in TMEM, so QK(e + 2) is
//     issued as soon as WG (e & 1) has copied S(e) into registers -- the next
//     tile's scores are ready long before the warpgroup finishes its exps;
//   * both warpgroups accumulate into ONE O (a thread of WG0 and one of WG1
//     own the same query row: warps w and w + 4 share a TMEM sub-partition).
//     They keep one common running max m: WG (e & 1) reads m(e - 1) from the
//     other warpgroup (shared memory + a named barrier per warp pair), updates
//     it with tile e and hands m(e) on.  The hand-over costs a few instructions
//     because the tile max is taken on the RAW scores against a per-tile bound
//     of S_q^K (slots kSqkMaxSlot / kSqkMinSlot of the tile's S_q^K block, written by
//     phase 1; K rows are in natural order in this kernel's operand, key_perm = 2):
//     when bound(tile) * S_q^Q <= m(e - 1) + tau the lazy rule keeps m (exactly
//     what the exact max would decide) and the scaling moves into the exp pass;
//     only otherwise is the exact scaled max computed;
//   * an update of m rescales O (after PV(e - 1), before PV(e)); each
//     warpgroup keeps its own row sum l relative to the last m it saw, and the
//     epilogue combines l0 2^(m0 - m) + l1 2^(m1 - m).
//
// TMEM (512 columns):
//   S0 [0,128)  S1 [128,256)  O [256,256+DV)  P0 [384,416)  P1 [416,448)
//   SF: Q 448 / 460 (per Q stage: hi 4*kChHi | lo 4*kChLo) | K0 472 | K1 480 | V0 488 | V1 492 | P 496
//
// Warps: 0-3 softmax WG0, 4-7 softmax WG1, 8 producer (TMA + scheduler),
//        9 QK issuer, 10 PV issuer, 11 V producer.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <type_traits>

#include "attn.cuh"
#include "attn_pp.cuh"
#include "common.cuh"
#include "ptx.cuh"

namespace dma {

#ifndef DMA_SK_POLY
#define DMA_SK_POLY 0
#endif
// exp2 pairs (out of every 8 per 16-pair group) computed on the FMA pipe (exp2_poly3)
constexpr int kPolySK = DMA_SK_POLY;

struct SKParams {
  int n_items;
  int head_major;
  unsigned int* ticket;  // [0] next item, [1] CTAs done (self-resetting)
};

template <int D, int DV, int LOW>
struct SKCfg {
  static constexpr int kBM = 128, kBN = 128;
  static constexpr int kNK = 4, kNV = 3, kNS = 4, kNSch = 4;
  static constexpr int kThreads = 384;
  static constexpr int kRegSoft = 216, kRegCtl = 72;
  static_assert(256 * kRegSoft + 128 * kRegCtl <= kThreads * 168, "register pool");
  static constexpr int kQHiBytes = kBM * D;
  static constexpr int kQLoBytes = kBM * D / 2;
  static constexpr int kQStage = ((kQHiBytes + (LOW != kLowHigh ? kQLoBytes : 0) + 1023) / 1024) * 1024;
  static constexpr int kKBytes = kBN * D;
  static constexpr int kVBytes = kBN * DV;
  static constexpr int kChHi = (D / 32 + 3) / 4;
  static constexpr int kChLo = LOW == kLowNV ? (D / 16 + 3) / 4 : (D / 32 + 3) / 4;
  static constexpr int kChK = kChHi > kChLo ? kChHi : kChLo;
  static constexpr int kSfQ = 512 * (kChHi + kChLo);
  static constexpr int kSqkBytes = 4 * kSqkTile;  // 576
  // smem (offsets from a 1024-aligned base)
  static constexpr int oQ = 0;                          // [2 slot][kQStage]
  static constexpr int oK = oQ + 2 * kQStage;           // [kNK][kKBytes]
  static constexpr int oV = oK + kNK * kKBytes;         // [kNV][kVBytes]
  static constexpr int oSfQ = oV + kNV * kVBytes;       // [2 slot][kSfQ]
  static constexpr int oSfK = oSfQ + 2 * kSfQ;          // [kNK][kChK][512]
  static constexpr int oSfV = oSfK + kNK * kChK * 512;  // [kNV][512]
  static constexpr int oSqK = oSfV + kNV * 512;         // [kNS][kSqkBytes]
  static constexpr int oSfP = oSqK + kNS * kSqkBytes;   // 512
  static constexpr int oSch = oSfP + 512;               // [kNSch] int
  static constexpr int oHand = oSch + 64;               // [2 wg][128] f32: m(e) handed to the other WG
  static constexpr int oEpi = oHand + 2 * 128 * 4;      // [2 parity][2 wg][128] float2 (m_l, l)
  static constexpr int oBar = oEpi + 2 * 2 * 128 * 8;
  static constexpr int kSmemBytes = oBar + 512 + 1024;
  static_assert(kSmemBytes <= 227 * 1024, "smem budget");
  // TMEM columns
  static constexpr uint32_t tO = 256, tSfP = 496;
  __device__ static constexpr uint32_t tSfQ(int slot) { return 448u + 12u * slot; }
  __device__ static constexpr uint32_t tS(int b) { return 128u * b; }
  __device__ static constexpr uint32_t tP(int b) { return 384u + 32u * b; }
  __device__ static constexpr uint32_t tSfK(int b) { return 472u + 8u * b; }
  __device__ static constexpr uint32_t tSfV(int b) { return 488u + 4u * b; }
  static_assert(4 * (kChHi + kChLo) <= 12 && 4 * kChK <= 8, "TMEM scale-factor slots");
};

__device__ __forceinline__ void sk_item_coords(const AttnParams& p, const SKParams& q, int k, int& bh, int& qt) {
  int r;
  if (q.head_major) {
    bh = k / p.n_qt;
    r = k - bh * p.n_qt;
  } else {
    r = k / p.n_bh;
    bh = k - r * p.n_bh;
  }
  qt = p.causal ? p.n_qt - 1 - r : r;
}

// 2^x for a pair on the FMA pipe, degree-3 minimax on [0, 1) (rel. error 8.8e-5, far
// below the E4M3 rounding of P); x >= -127 after the clamp (masked -inf -> 2^-127 ~ 0)
__device__ __forceinline__ float2 exp2_poly3(float2 x) {
  x.x = fmaxf(x.x, -127.f);
  x.y = fmaxf(x.y, -127.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);
  const float2 t = __fadd2_rd(x, magic);
  const float2 fl = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-fl.x, -fl.y));
  float2 p = __ffma2_rn(make_float2(0.07944023f, 0.07944023f), f, make_float2(0.22449434f, 0.22449434f));
  p = __ffma2_rn(p, f, make_float2(0.69606566f, 0.69606566f));
  p = __ffma2_rn(p, f, make_float2(1.0f, 1.0f));
  return make_float2(__uint_as_float(__float_as_uint(p.x) + (__float_as_uint(t.x) << 23)),
                     __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(t.y) << 23)));
}

// key group G of the exponent arguments: S * S_q^K (two-level tiles) * S_q^Q + bias
template <bool TL, int G>
__device__ __forceinline__ void sk_prep(float (&tv)[128], uint32_t sqk, float2 rf2, float2 b2) {
#pragma unroll
  for (int w4 = 8 * G; w4 < 8 * G + 8; ++w4) {
    float2 a = make_float2(tv[4 * w4], tv[4 * w4 + 1]);
    float2 c = make_float2(tv[4 * w4 + 2], tv[4 * w4 + 3]);
    if constexpr (TL) {
      const float4 f = ptx::lds_f4(sqk + 16 * w4);
      a = __fmul2_rn(a, make_float2(f.x, f.y));
      c = __fmul2_rn(c, make_float2(f.z, f.w));
    }
    a = __ffma2_rn(a, rf2, b2);
    c = __ffma2_rn(c, rf2, b2);
    tv[4 * w4] = a.x;
    tv[4 * w4 + 1] = a.y;
    tv[4 * w4 + 2] = c.x;
    tv[4 * w4 + 3] = c.y;
  }
}

// exps of key group Q4 interleaved with the E4M3 packs of group Q4 - 1 (software pipeline)
template <int Q4>
__device__ __forceinline__ void sk_exp_group(float (&tv)[128], uint32_t (&pk)[8], float2& ls) {
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    if (Q4 < 4) {
      const int kk = 32 * Q4 + 2 * j;
      if ((j & 7) < kPolySK) {
        const float2 e2 = exp2_poly3(make_float2(tv[kk], tv[kk + 1]));
        tv[kk] = e2.x;
        tv[kk + 1] = e2.y;
      } else {
        tv[kk] = exp2_ordered(tv[kk]);
        tv[kk + 1] = exp2_ordered(tv[kk + 1]);
      }
    }
    if (Q4 > 0) {
      const int kk = 32 * (Q4 - 1) + 2 * j;
      const uint32_t hv = cvt_e4m3x2_ordered(tv[kk], tv[kk + 1]);
      if (j & 1) {
        pk[j >> 1] |= hv << 16;
      } else {
        pk[j >> 1] = hv;
      }
      const float2 e2 = make_float2(tv[kk], tv[kk + 1]);
      ls = (Q4 == 1 && j == 0) ? e2 : __fadd2_rn(ls, e2);
    }
  }
}

// running max of 32 raw S columns (key group G); keys >= lim are masked
template <bool MASK, int G>
__device__ __forceinline__ float sk_group_max(const uint32_t (&r)[32], float m, int lim) {
  float m4[4] = {m, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
  for (int c = 0; c < 32; c += 8) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float a = __uint_as_float(r[c + 2 * q]), b = __uint_as_float(r[c + 2 * q + 1]);
      if (MASK) {
        a = 32 * G + c + 2 * q < lim ? a : -INFINITY;
        b = 32 * G + c + 2 * q + 1 < lim ? b : -INFINITY;
      }
      m4[q] = ptx::fmax3(m4[q], a, b);
    }
  }
  return fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
}

// One tile of the softmax after m is known: exp2 + E4M3 requantisation of P into TMEM
// (tP).  When the warpgroup has a next tile (e + 2), its raw row max is taken on the way
// (S columns loaded into the registers the finished key groups free), so the next
// tile's m hand-over does not wait for a full S load and max.
template <bool TL>
__device__ __forceinline__ void sk_exp_tile(float (&tv)[128], float2& ls, uint32_t sqk, float2 rf2, float2 b2,
                                            bool next, bool mask_next, int lim_next, float& mraw_next,
                                            uint32_t jown, int lane, uint32_t tS, uint32_t tP,
                                            uint64_t* sq_empty_slot, uint64_t* o_done_w, uint64_t* s_full_w) {
  uint32_t pk[8];
  sk_prep<TL, 0>(tv, sqk, rf2, b2);
  sk_exp_group<0>(tv, pk, ls);
  sk_prep<TL, 1>(tv, sqk, rf2, b2);
  sk_exp_group<1>(tv, pk, ls);
  sk_prep<TL, 2>(tv, sqk, rf2, b2);
  if (jown > 0) {  // P(w) was read by this warpgroup's previous PV
    ptx::mbar_wait(o_done_w, (jown - 1) & 1);
    ptx::tc_fence_after();
  }
  ptx::tmem_st8(tP + 0, pk);
  sk_exp_group<2>(tv, pk, ls);
  sk_prep<TL, 3>(tv, sqk, rf2, b2);
  __syncwarp();
  if (lane == 0) ptx::mbar_arrive(sq_empty_slot);  // S_q^K slot read (bound, scale)
  ptx::tmem_st8(tP + 8, pk);
  uint32_t r0[32], r1[32];
  float mx = -INFINITY;
  // temporaries are loaded as the key groups of this tile die (at most 96 live scores)
  if (next) {
    // QK(e + 2) ran while tile e was processed: its scores are in the warpgroup's S buffer
    ptx::mbar_wait(s_full_w, (jown + 1) & 1);
    ptx::tc_fence_after();
    ptx::tmem_ld32(tS + 0, r0);
  }
  sk_exp_group<3>(tv, pk, ls);
  ptx::tmem_st8(tP + 16, pk);
  if (next) {
    ptx::tmem_ld_wait();
    mx = mask_next ? sk_group_max<true, 0>(r0, mx, lim_next) : sk_group_max<false, 0>(r0, mx, lim_next);
    ptx::tmem_ld32(tS + 32, r0);
    ptx::tmem_ld32(tS + 64, r1);
  }
  sk_exp_group<4>(tv, pk, ls);
  ptx::tmem_st8(tP + 24, pk);
  if (next) {
    ptx::tmem_ld_wait();
    if (mask_next) {
      mx = sk_group_max<true, 1>(r0, mx, lim_next);
      mx = sk_group_max<true, 2>(r1, mx, lim_next);
    } else {
      mx = sk_group_max<false, 1>(r0, mx, lim_next);
      mx = sk_group_max<false, 2>(r1, mx, lim_next);
    }
    ptx::tmem_ld32(tS + 96, r0);
    ptx::tmem_ld_wait();
    mx = mask_next ? sk_group_max<true, 3>(r0, mx, lim_next) : sk_group_max<false, 3>(r0, mx, lim_next);
    mraw_next = mx;
  }
}

template <int D, int DV, int LOW>
__global__ void __launch_bounds__(384, 1) dma_attn_sk_kernel(const __grid_constant__ AttnParams p,
                                                             const __grid_constant__ SKParams sp) {
  using C = SKCfg<D, DV, LOW>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::oBar);
  uint64_t* q_full = bars;                  // [2]
  uint64_t* q_empty = q_full + 2;           // [2]
  uint64_t* k_full = q_empty + 2;           // [kNK]
  uint64_t* k_empty = k_full + C::kNK;      // [kNK]
  uint64_t* v_full = k_empty + C::kNK;      // [kNV]
  uint64_t* v_empty = v_full + C::kNV;      // [kNV]
  uint64_t* sq_empty = v_empty + C::kNV;    // [kNS]
  uint64_t* s_full = sq_empty + C::kNS;     // [2] QK(e) into S(e & 1) done
  uint64_t* s_free = s_full + 2;            // [2] WG b copied S(b) out
  uint64_t* p_full = s_free + 2;            // [2] WG b stored P(b) (and rescaled O)
  uint64_t* o_done = p_full + 2;            // [2] PV of a WG-b tile done
  uint64_t* o_free = o_done + 2;            // [1] epilogue read O
  uint64_t* sch_full = o_free + 1;          // [kNSch]
  uint64_t* sch_empty = sch_full + C::kNSch;  // [kNSch]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sch_empty + C::kNSch);
  int* sched = reinterpret_cast<int*>(smem + C::oSch);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rt_q = p.lq_pad >> 7, rt_k = p.lk_pad >> 7;
  constexpr int kProducer = 8, kMmaQK = 9, kMmaPV = 10, kProdV = 11;

  if (warp == kProducer) {
    if (lane == 0) {
      for (int i = 0; i < 2; ++i) {
        ptx::mbar_init(q_full + i, 1);
        ptx::mbar_init(q_empty + i, 1);
        ptx::mbar_init(s_full + i, 1);
        ptx::mbar_init(s_free + i, 4);
        ptx::mbar_init(p_full + i, 4);
        ptx::mbar_init(o_done + i, 1);
      }
      ptx::mbar_init(o_free, 8);
      for (int i = 0; i < C::kNK; ++i) {
        ptx::mbar_init(k_full + i, 1);
        ptx::mbar_init(k_empty + i, 1);
      }
      for (int i = 0; i < C::kNV; ++i) {
        ptx::mbar_init(v_full + i, 1);
        ptx::mbar_init(v_empty + i, 1);
      }
      for (int i = 0; i < C::kNS; ++i) ptx::mbar_init(sq_empty + i, 4);
      for (int i = 0; i < C::kNSch; ++i) {
        ptx::mbar_init(sch_full + i, 1);
        ptx::mbar_init(sch_empty + i, 3 + 8);
      }
      ptx::fence_barrier_init();
      ptx::tma_prefetch_desc(&p.tm_q_hi);
      ptx::tma_prefetch_desc(&p.tm_k_hi);
      ptx::tma_prefetch_desc(&p.tm_v);
      if (LOW != kLowHigh) {
        ptx::tma_prefetch_desc(&p.tm_q_lo);
        ptx::tma_prefetch_desc(&p.tm_k_lo);
      }
    }
  } else if (warp == kMmaQK) {
    ptx::tmem_alloc<512>(tmem_slot);
  } else if (warp == 0) {
    uint32_t* sfp = reinterpret_cast<uint32_t*>(smem + C::oSfP);  // P scale factors: E8M0 127 = 1.0
    for (int i = lane; i < 128; i += 32) sfp[i] = 0x7F7F7F7Fu;
    ptx::fence_proxy_async_smem();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= 8) {
    ptx::setmaxnreg_dec<C::kRegCtl>();
    const uint32_t sbase = ptx::smem_u32(smem);
    if (warp == kProducer) {
      // =========================== scheduler + TMA producer ===========================
      uint32_t ks = 0, kph = 0, po = 0, gq = 0;
      TRACE_DECL
      for (uint32_t i = 0;; ++i) {
        const int ss = i % C::kNSch;
        ptx::mbar_wait(sch_empty + ss, ((i / C::kNSch) & 1) ^ 1);
        unsigned int tk = 0;
        if (lane == 0) tk = atomicAdd(sp.ticket, 1u);
        tk = __shfl_sync(0xffffffffu, tk, 0);
        const int k = tk < static_cast<unsigned int>(sp.n_items) ? static_cast<int>(tk) : -1;
        if (lane == 0) {
          sched[ss] = k;
          ptx::mbar_arrive(sch_full + ss);
        }
        __syncwarp();
        if (k < 0) break;
        int bh, qt;
        sk_item_coords(p, sp, k, bh, qt);
        Plan plan;
        plan.init(qt, p.lq, p.lk, C::kBM, C::kBN, p.diag_window, p.sink_window, p.causal != 0);
        if (plan.n == 0) continue;
        const int mk = mat_k_of(p, bh);
        const int qs = po & 1;
        ptx::mbar_wait(q_empty + qs, ((po >> 1) & 1) ^ 1);
        ++po;
        uint32_t qbytes = C::kQHiBytes + 512 * C::kChHi;
        if (LOW != kLowHigh) qbytes += C::kQLoBytes + 512 * C::kChLo;
        ptx::wu::mbar_arrive_expect_tx(q_full + qs, qbytes);
        uint8_t* qdst = smem + C::oQ + qs * C::kQStage;
        uint8_t* sfq = smem + C::oSfQ + qs * C::kSfQ;
        ptx::wu::tma_load_3d(qdst, &p.tm_q_hi, q_full + qs, 0, qt * C::kBM, bh);
        ptx::wu::bulk_load(sfq, p.sf_q_hi + (static_cast<int64_t>(bh) * rt_q + qt) * p.ch_hi * 512, 512 * C::kChHi,
                           q_full + qs);
        if (LOW != kLowHigh) {
          ptx::wu::tma_load_3d(qdst + C::kQHiBytes, &p.tm_q_lo, q_full + qs, 0, qt * C::kBM, bh);
          ptx::wu::bulk_load(sfq + 512 * C::kChHi, p.sf_q_lo + (static_cast<int64_t>(bh) * rt_q + qt) * p.ch_lo * 512,
                             512 * C::kChLo, q_full + qs);
        }
        for (int e = 0; e < plan.n; ++e, ++gq) {
          int t;
          bool hi;
          plan.entry(e, t, hi);
          if (LOW == kLowHigh) hi = true;
          const int ch = hi ? C::kChHi : C::kChLo;
          const uint32_t kbytes = hi ? C::kKBytes : C::kKBytes / 2;
          ptx::mbar_wait(k_empty + ks, kph ^ 1);
          const uint32_t sqs = gq % C::kNS;
          ptx::mbar_wait(sq_empty + sqs, ((gq / C::kNS) & 1) ^ 1);
          ptx::wu::mbar_arrive_expect_tx(k_full + ks, kbytes + 512 * ch + C::kSqkBytes);
          ptx::wu::tma_load_3d(smem + C::oK + ks * C::kKBytes, hi ? &p.tm_k_hi : &p.tm_k_lo, k_full + ks, 0,
                               t * C::kBN, mk);
          const uint8_t* sfsrc =
              (hi ? p.sf_k_hi : p.sf_k_lo) + (static_cast<int64_t>(mk) * rt_k + t) * (hi ? p.ch_hi : p.ch_lo) * 512;
          ptx::wu::bulk_load(smem + C::oSfK + ks * 512 * C::kChK, sfsrc, 512 * ch, k_full + ks);
          ptx::wu::bulk_load(smem + C::oSqK + sqs * C::kSqkBytes,
                             p.qs_k + (static_cast<int64_t>(mk) * rt_k + t) * kSqkTile, C::kSqkBytes, k_full + ks);
          TRACE(true, 4, 30);
          if (++ks == C::kNK) { ks = 0; kph ^= 1; }
        }
      }
      // last CTA out resets the ticket for the next launch (stream-ordered)
      if (lane == 0) {
        __threadfence();
        const unsigned int done = atomicAdd(sp.ticket + 1, 1u);
        if (done == gridDim.x - 1) {
          sp.ticket[0] = 0u;
          sp.ticket[1] = 0u;
          __threadfence();
        }
      }
    } else if (warp == kProdV) {
      // =========================== V producer (own ring, never blocks the K loads) ===========================
      uint32_t vs = 0, vph = 0;
      TRACE_DECL
      for (uint32_t i = 0;; ++i) {
        const int ss = i % C::kNSch;
        ptx::mbar_wait(sch_full + ss, (i / C::kNSch) & 1);
        const int k = sched[ss];
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(sch_empty + ss);
        if (k < 0) break;
        int bh, qt;
        sk_item_coords(p, sp, k, bh, qt);
        Plan plan;
        plan.init(qt, p.lq, p.lk, C::kBM, C::kBN, p.diag_window, p.sink_window, p.causal != 0);
        const int mk = mat_k_of(p, bh);
        for (int e = 0; e < plan.n; ++e) {
          int t;
          bool hi;
          plan.entry(e, t, hi);
          ptx::mbar_wait(v_empty + vs, vph ^ 1);
          ptx::wu::mbar_arrive_expect_tx(v_full + vs, C::kVBytes + 512);
          ptx::wu::tma_load_3d(smem + C::oV + vs * C::kVBytes, &p.tm_v, v_full + vs, 0, t * C::kBN, mk);
          ptx::wu::bulk_load(smem + C::oSfV + vs * 512, p.sf_v + (static_cast<int64_t>(mk) * rt_k + t) * 512, 512,
                             v_full + vs);
          TRACE(true, 5, 31);
          if (++vs == C::kNV) { vs = 0; vph ^= 1; }
        }
      }
    } else if (warp == kMmaQK || warp == kMmaPV) {
      // ============ MMA issuers: warp 9 issues every QK, warp 10 every PV ============
      // (separate warps, so QK(e + 2) never queues behind PV(e), which waits for the
      // softmax of tile e to finish)
      const uint64_t sf_desc_hi = static_cast<uint64_t>(ptx::desc_hi(128, ptx::kSwNone)) << 32;
      auto sf_desc = [&](uint32_t off) { return sf_desc_hi | ptx::desc_lo(sbase + off, 0); };
      const bool is_qk = warp == kMmaQK;
      if (!is_qk) ptx::wu::tc_cp_sf(tmem + C::tSfP, sf_desc(C::oSfP));
      uint32_t ks = 0, kph = 0, vs = 0, vph = 0, po = 0, n_items_done = 0;
      uint32_t s_use0 = 0, s_use1 = 0, pvc0 = 0, pvc1 = 0;  // scalars: no local-memory arrays
      TRACE_DECL
      const uint32_t hf = static_cast<uint32_t>(p.hfmt);
      for (uint32_t i = 0;; ++i) {
        const int ss = i % C::kNSch;
        ptx::mbar_wait(sch_full + ss, (i / C::kNSch) & 1);
        const int k = sched[ss];
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(sch_empty + ss);
        if (k < 0) break;
        int bh, qt;
        sk_item_coords(p, sp, k, bh, qt);
        Plan plan;
        plan.init(qt, p.lq, p.lk, C::kBM, C::kBN, p.diag_window, p.sink_window, p.causal != 0);
        if (plan.n == 0) continue;
        if (is_qk) {
          const int qs = po & 1;
          ptx::mbar_wait(q_full + qs, (po >> 1) & 1);
          ++po;
          ptx::tc_fence_after();
          const uint32_t oq = C::oQ + qs * C::kQStage;
          const uint32_t osfq = C::oSfQ + qs * C::kSfQ;
          // Q scale factors into the slot of this Q stage (the other slot may still feed
          // the previous item's last QK)
          const uint32_t tsfq = tmem + C::tSfQ(qs), tsfql = tsfq + 4 * C::kChHi;
          for (int j = 0; j < C::kChHi; ++j) ptx::wu::tc_cp_sf(tsfq + 4 * j, sf_desc(osfq + 512 * j));
          if (LOW != kLowHigh)
            for (int j = 0; j < C::kChLo; ++j) ptx::wu::tc_cp_sf(tsfql + 4 * j, sf_desc(osfq + 512 * (C::kChHi + j)));
          for (int e = 0; e < plan.n; ++e) {
            int t;
            bool hi;
            plan.entry(e, t, hi);
            if (LOW == kLowHigh) hi = true;
            const int b = e & 1;
            const uint32_t su = b ? s_use1++ : s_use0++;
            ptx::mbar_wait(s_free + b, (su & 1) ^ 1);  // WG b copied out its previous S
            TRACE(true, 2, 10 + b);
            ptx::mbar_wait(k_full + ks, kph);
            ptx::tc_fence_after();
            TRACE(true, 2, 18 + b);
            const uint32_t kslt = ks;
            if (++ks == C::kNK) { ks = 0; kph ^= 1; }
            const int ch = hi ? C::kChHi : C::kChLo;
            for (int j = 0; j < ch; ++j)
              ptx::wu::tc_cp_sf(tmem + C::tSfK(b) + 4 * j, sf_desc(C::oSfK + kslt * 512 * C::kChK + 512 * j));
            TRACE(true, 2, 20 + b);
            const uint32_t tSd = tmem + C::tS(b), tsfk = tmem + C::tSfK(b);
            if (hi) {
              constexpr int rb = D;
              const uint32_t kaddr = sbase + C::oK + kslt * C::kKBytes;
              const uint64_t dh = static_cast<uint64_t>(ptx::desc_hi(8 * rb, swz_mode(rb))) << 32;
#pragma unroll
              for (int kk = 0; kk < D / 32; ++kk) {
                const uint64_t ad = dh | ptx::desc_lo(sbase + oq + 32 * kk, 16);
                const uint64_t bd = dh | ptx::desc_lo(kaddr + 32 * kk, 16);
                const uint32_t id = ptx::idesc_bs(hf, hf, 0, 0, 128, 128, 1, kk & 3, kk & 3);
                ptx::wu::mma_mxf8f6f4(tSd, ad, bd, id, tsfq + 4 * (kk >> 2), tsfk + 4 * (kk >> 2), kk > 0);
              }
            } else {
              constexpr int rb = D / 2;
              const uint32_t kaddr = sbase + C::oK + kslt * C::kKBytes;
              const uint64_t dh = static_cast<uint64_t>(ptx::desc_hi(8 * rb, swz_mode(rb))) << 32;
#pragma unroll
              for (int kk = 0; kk < D / 64; ++kk) {
                const uint64_t ad = dh | ptx::desc_lo(sbase + oq + C::kQHiBytes + 32 * kk, 16);
                const uint64_t bd = dh | ptx::desc_lo(kaddr + 32 * kk, 16);
                if (LOW == kLowNV) {
                  const uint32_t id = ptx::idesc_bs(1, 1, 0, 0, 128, 128, 0, 0, 0);
                  ptx::wu::mma_nvf4(tSd, ad, bd, id, tsfql + 4 * kk, tsfk + 4 * kk, kk > 0);
                } else {
                  const uint32_t sid = (kk & 1) * 2;
                  const uint32_t id = ptx::idesc_bs(1, 1, 0, 0, 128, 128, 1, sid, sid);
                  ptx::wu::mma_mxf4(tSd, ad, bd, id, tsfql + 4 * (kk >> 1), tsfk + 4 * (kk >> 1), kk > 0);
                }
              }
            }
            ptx::wu::tc_commit(k_empty + kslt);
            ptx::wu::tc_commit(s_full + b);
            TRACE(true, 2, 12 + b);
            if (e == plan.n - 1) ptx::wu::tc_commit(q_empty + qs);  // Q slot free after the last QK
          }
        } else {
          for (int e = 0; e < plan.n; ++e) {
            const int b = e & 1;
            const uint32_t pc = b ? pvc1++ : pvc0++;
            ptx::mbar_wait(p_full + b, pc & 1);
            TRACE(true, 3, 14 + b);
            if (e == 0 && n_items_done > 0) ptx::mbar_wait(o_free, (n_items_done - 1) & 1);  // epilogue read O
            ptx::mbar_wait(v_full + vs, vph);
            ptx::tc_fence_after();
            TRACE(true, 3, 22 + b);
            const uint32_t vslt = vs;
            if (++vs == C::kNV) { vs = 0; vph ^= 1; }
            ptx::wu::tc_cp_sf(tmem + C::tSfV(b), sf_desc(C::oSfV + vslt * 512));
            const uint32_t vaddr = sbase + C::oV + vslt * C::kVBytes;
            constexpr int rb = DV;  // fp8 V row bytes (MN-major)
            const uint64_t dh = static_cast<uint64_t>(ptx::desc_hi(8 * rb, swz_mode(rb))) << 32;
#pragma unroll
            for (int kk = 0; kk < C::kBN / 32; ++kk) {
              const uint64_t bd = dh | ptx::desc_lo(vaddr + kk * 32 * rb, 16);
              const uint32_t id = ptx::idesc_bs(0, 0, 0, 1, 128, DV, 1, kk & 3, kk & 3);
              ptx::wu::mma_mxf8f6f4_ts(tmem + C::tO, tmem + C::tP(b) + 8 * kk, bd, id, tmem + C::tSfP,
                                       tmem + C::tSfV(b), !(e == 0 && kk == 0));
            }
            ptx::wu::tc_commit(v_empty + vslt);
            ptx::wu::tc_commit(o_done + b);
            TRACE(true, 3, 16 + b);
          }
        }
        ++n_items_done;
      }
    }
  } else {
    ptx::setmaxnreg_inc<C::kRegSoft>();
    // =========================== softmax: WG w takes plan entries e = w (mod 2) ===========================
    const int w = warp >> 2;      // warpgroup
    const int quad = warp & 3;    // TMEM sub-partition
    const int row = quad * 32 + lane;
    const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t bar_give = 1 + 4 * w + quad;        // this WG -> the other: m(e) ready
    const uint32_t bar_take = 1 + 4 * (1 - w) + quad;  // the other WG -> this one
    const uint32_t bar_epi = 9 + quad;
    float* hand = reinterpret_cast<float*>(smem + C::oHand);
    float2* epi = reinterpret_cast<float2*>(smem + C::oEpi);
    constexpr float kLazy = 4.f;  // lazy rescale threshold (log2 units), P <= 2^kLazy
    constexpr float kPShift = 8.f - kLazy;
    uint32_t cb0 = 0, cb1 = 0;  // PV tiles of WG 0 / 1 in earlier items (o_done phase counts)
    uint32_t gq = 0;             // tiles of earlier items (S_q^K ring position)
    uint32_t n_items_done = 0;
    const bool tw = quad == 0;  // traced warp of this WG (DMA_TRACE)
    (void)tw;
    TRACE_DECL

    for (uint32_t it = 0;; ++it) {
      const int ss = it % C::kNSch;
      ptx::mbar_wait(sch_full + ss, (it / C::kNSch) & 1);
      const int k = sched[ss];
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(sch_empty + ss);
      if (k < 0) break;
      int bh, qt;
      sk_item_coords(p, sp, k, bh, qt);
      Plan plan;
      plan.init(qt, p.lq, p.lk, C::kBM, C::kBN, p.diag_window, p.sink_window, p.causal != 0);
      const int q0 = qt * C::kBM;
      const int qrow = q0 + row;
      const int64_t orow = static_cast<int64_t>(bh) * p.lq + qrow;
      constexpr int OC = DV / 2;  // O columns this warpgroup writes in the epilogue
      if (plan.n == 0) {
        if (qrow < p.lq) {
          uint32_t z[32];
#pragma unroll
          for (int i2 = 0; i2 < 32; ++i2) z[i2] = 0u;
#pragma unroll
          for (int c = 0; c < OC / 32; ++c) store_orow<DV>(p, orow, (OC / 32) * w + c, z, 1.0f);
        }
        continue;
      }
      const float sq_q = (qrow < p.lq) ? p.qs_q[static_cast<int64_t>(bh) * p.lq_pad + qrow] : 1.0f;
      float m_l = -INFINITY;  // the m this warpgroup's l is relative to
      float2 l2 = make_float2(0.f, 0.f);

      // Per tile: the raw row max mraw is known before the tile starts (taken during the
      // previous tile's exps, or right after the load for a warpgroup's first tile), so the
      // m hand-over and the bound check overlap the reload of S into registers.
      float mraw = -INFINITY;
      for (int e = w; e < plan.n; e += 2) {
        int t;
        bool hi;
        plan.entry(e, t, hi);
        if (LOW == kLowHigh) hi = true;
        const bool two_level = hi || (LOW == kLowNV);
        const int k0 = t * C::kBN;
        const uint32_t jown = (w ? cb1 : cb0) + e / 2;
        const int sl = (gq + e) % C::kNS;
        const uint32_t sqk = ptx::smem_u32(smem + C::oSqK + sl * C::kSqkBytes);
        const float rowf = two_level ? sq_q : 1.0f;
        // causal (attention.py:178-184, applied when k1-1 > q0, :306) and ragged-key masks
        const int kvalid = p.lk - k0;
        const bool need_causal = p.causal && (k0 + (kvalid < C::kBN ? kvalid : C::kBN) - 1 > q0);
        const bool masked = need_causal || kvalid < C::kBN;
        const int lim = need_causal ? min(qrow - k0 + 1, kvalid) : kvalid;
        ptx::mbar_wait(s_full + w, jown & 1);  // (already passed when the max was taken early)
        ptx::tc_fence_after();
        TRACE(tw, w, 1);
        uint32_t sr[128];
#pragma unroll
        for (int c = 0; c < 128; c += 32)
          ptx::tmem_ld32(tmem + C::tS(w) + lane_base + c, *reinterpret_cast<uint32_t(*)[32]>(&sr[c]));
        if (e == w) {  // first tile of this warpgroup in the item: raw max now
          ptx::tmem_ld_wait();
          float mx = -INFINITY;
          if (masked) {
            mx = sk_group_max<true, 0>(*reinterpret_cast<uint32_t(*)[32]>(&sr[0]), mx, lim);
            mx = sk_group_max<true, 1>(*reinterpret_cast<uint32_t(*)[32]>(&sr[32]), mx, lim);
            mx = sk_group_max<true, 2>(*reinterpret_cast<uint32_t(*)[32]>(&sr[64]), mx, lim);
            mx = sk_group_max<true, 3>(*reinterpret_cast<uint32_t(*)[32]>(&sr[96]), mx, lim);
          } else {
            mx = sk_group_max<false, 0>(*reinterpret_cast<uint32_t(*)[32]>(&sr[0]), mx, lim);
            mx = sk_group_max<false, 1>(*reinterpret_cast<uint32_t(*)[32]>(&sr[32]), mx, lim);
            mx = sk_group_max<false, 2>(*reinterpret_cast<uint32_t(*)[32]>(&sr[64]), mx, lim);
            mx = sk_group_max<false, 3>(*reinterpret_cast<uint32_t(*)[32]>(&sr[96]), mx, lim);
          }
          mraw = mx;
        }
        float bound = mraw;
        if (two_level) {
          const float2 mm = *reinterpret_cast<const float2*>(smem + C::oSqK + sl * C::kSqkBytes + 4 * kSqkMaxSlot);
          const float smax = mm.x, smin = __uint_as_float(~__float_as_uint(mm.y));
          bound = mraw >= 0.f ? mraw * smax : mraw * smin;
        }
        // running max hand-over: m(e - 1) from the other warpgroup
        float m_prev = -INFINITY;
        if (e > 0) {
          ptx::named_bar_sync(bar_take, 64);
          m_prev = hand[(1 - w) * 128 + row];
        }
        TRACE(tw, w, 3);
        const bool fast = m_prev != -INFINITY && bound * rowf <= m_prev + kLazy;
        float m_new = m_prev;
        if (__all_sync(0xffffffffu, fast) && e + 1 < plan.n) {
          hand[w * 128 + row] = m_new;  // publish before the S reload completes
          ptx::named_bar_arrive(bar_give, 64);
        }
        ptx::tmem_ld_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(s_free + w);  // S(w) may take QK(e + 2)
        TRACE(tw, w, 2);
        float tv[128];
#pragma unroll
        for (int i = 0; i < 128; ++i) tv[i] = __uint_as_float(sr[i]);
        if (masked) {
#pragma unroll
          for (int j = 0; j < 128; ++j)
            if (j >= lim) tv[j] = -INFINITY;
        }
        if (!__all_sync(0xffffffffu, fast)) {
          if (!fast) {
            // exact scaled max (the first tile of a row, or a tile whose bound exceeds the window)
            TRACE(tw && lane == 0, w, 7);
            float mx = -INFINITY;
            if (two_level) {
#pragma unroll
              for (int w4 = 0; w4 < 32; ++w4) {
                const float4 f = ptx::lds_f4(sqk + 16 * w4);
                const float2 a = __fmul2_rn(make_float2(tv[4 * w4], tv[4 * w4 + 1]), make_float2(f.x, f.y));
                const float2 b2 = __fmul2_rn(make_float2(tv[4 * w4 + 2], tv[4 * w4 + 3]), make_float2(f.z, f.w));
                mx = fmaxf(mx, ptx::fmax3(a.x, a.y, fmaxf(b2.x, b2.y)));
              }
            } else {
              mx = mraw;
            }
            const float m_cand = fmaxf(m_prev, mx * rowf);
            if (m_cand > m_prev + kLazy) m_new = m_cand;  // always for the first live tile (m_prev = -inf)
          }
          if (e + 1 < plan.n) {
            hand[w * 128 + row] = m_new;
            ptx::named_bar_arrive(bar_give, 64);
          }
        }
        const bool dead = (m_new == -INFINITY);
        // l is kept relative to m_l; O is relative to m(e - 1) until rescaled
        if (m_new != m_l) {
          const float f = (m_l == -INFINITY) ? 0.f : fast_exp2(m_l - m_new);
          l2 = make_float2(l2.x * f, l2.y * f);
          m_l = m_new;
        }
        const float alpha = (m_prev == -INFINITY || m_new == m_prev) ? 1.0f : fast_exp2(m_prev - m_new);
        if (e > 0 && __any_sync(0xffffffffu, alpha != 1.0f)) {
          // O *= alpha after PV(e - 1) (the other warpgroup's tile), before PV(e)
          const int v = 1 - w;
          const uint32_t idx = (v ? cb1 : cb0) + (e - 1) / 2;
          ptx::mbar_wait(o_done + v, idx & 1);
          ptx::tc_fence_after();
          const float2 a2 = make_float2(alpha, alpha);
#pragma unroll 1
          for (int cq = 0; cq < DV / 16; ++cq) {  // 16-column chunks: the scores stay live in registers
            const uint32_t ta = tmem + C::tO + lane_base + 16 * cq;
            uint32_t rr[16];
            ptx::tmem_ld16(ta, rr);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float2 x2 = __fmul2_rn(make_float2(__uint_as_float(rr[2 * i]), __uint_as_float(rr[2 * i + 1])), a2);
              rr[2 * i] = __float_as_uint(x2.x);
              rr[2 * i + 1] = __float_as_uint(x2.y);
            }
            ptx::tmem_st16(ta, rr);
          }
        }
        // exponent arguments S * S_q^K * S_q^Q + bias (attention.py:168-174 in base 2, with the
        // 2^(8 - tau) E4M3 headroom shift folded into the bias)
        const float bias = dead ? 0.f : (kPShift - m_new);
        const float2 rf2 = make_float2(rowf, rowf), b2 = make_float2(bias, bias);
        const bool next = e + 2 < plan.n;
        bool mask_next = false;
        int lim_next = 0;
        if (next) {
          int t2;
          bool hi2;
          plan.entry(e + 2, t2, hi2);
          const int k2 = t2 * C::kBN, kv2 = p.lk - k2;
          const bool nc2 = p.causal && (k2 + (kv2 < C::kBN ? kv2 : C::kBN) - 1 > q0);
          mask_next = nc2 || kv2 < C::kBN;
          lim_next = nc2 ? min(qrow - k2 + 1, kv2) : kv2;
        }
        float2 ls = make_float2(0.f, 0.f);
        TRACE(tw, w, 4);
        if (two_level) {
          sk_exp_tile<true>(tv, ls, sqk, rf2, b2, next, mask_next, lim_next, mraw, jown, lane,
                            tmem + C::tS(w) + lane_base, tmem + C::tP(w) + lane_base, sq_empty + sl, o_done + w,
                            s_full + w);
        } else {
          sk_exp_tile<LOW == kLowNV>(tv, ls, sqk, rf2, b2, next, mask_next, lim_next, mraw, jown, lane,
                                     tmem + C::tS(w) + lane_base, tmem + C::tP(w) + lane_base, sq_empty + sl,
                                     o_done + w, s_full + w);
        }
        TRACE(tw, w, 5);
        l2 = __fadd2_rn(l2, ls);
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(p_full + w);
        TRACE(tw, w, 6);
      }

      // ---- epilogue: O / l (attention.py:104-106); WG w writes O columns [w DV/2, (w+1) DV/2)
      const int par = n_items_done & 1;
      epi[(par * 2 + w) * 128 + row] = make_float2(m_l, l2.x + l2.y);
      ptx::named_bar_sync(bar_epi, 64);
      const float2 o2 = epi[(par * 2 + (1 - w)) * 128 + row];
      const float my_l = l2.x + l2.y;
      const float m_fin = fmaxf(m_l, o2.x);
      float l_tot = 0.f;
      if (my_l > 0.f) l_tot += my_l * (m_l == m_fin ? 1.f : fast_exp2(m_l - m_fin));
      if (o2.y > 0.f) l_tot += o2.y * (o2.x == m_fin ? 1.f : fast_exp2(o2.x - m_fin));
      const float inv_l = 1.0f / (l_tot > 0.f ? l_tot : 1.0f);
      {
        const int el = plan.n - 1, v = el & 1;
        const uint32_t idx = (v ? cb1 : cb0) + el / 2;
        ptx::mbar_wait(o_done + v, idx & 1);
        ptx::tc_fence_after();
      }
      const uint32_t tOw = tmem + C::tO + lane_base + OC * w;
#pragma unroll
      for (int c = 0; c < OC / 32; ++c) {
        uint32_t rr[32];
        ptx::tmem_ld32(tOw + 32 * c, rr);
        ptx::tmem_ld_wait();
        if (qrow < p.lq) store_orow<DV>(p, orow, (OC / 32) * w + c, rr, inv_l);
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(o_free);
      cb0 += (plan.n + 1) / 2;
      cb1 += plan.n / 2;
      gq += plan.n;
      ++n_items_done;
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == kMmaQK) ptx::tmem_dealloc<512>(tmem);
}

}  // namespace dma
