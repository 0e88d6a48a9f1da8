// Phase 2 of the DMA forward, max / exp split variant (block-scaled MXFP8 PV).
//
// Same algorithm as attn_pp.cuh (attention.py:282-310 with the plans of
// attention.py:191-233 and the base-2 online softmax of :150-175, lazy rescaling
// tau = 4, P -> E4M3(P * 2^4) in registers, PV with A = P from TMEM), organised so
// that the exp2 warps (the MUFU consumers) do nothing but exponentials:
//
//   * a work item is ONE 128-row query tile (b, h, qt); the tiles of all items form one
//     stream per CTA (global tile counter g), S double-buffered in TMEM (slot g & 1);
//   * the MAX warpgroup (warps 0-3, thread = query row) reads S(g) once, scales it by
//     S_q^K, masks, takes the row max, applies the lazy rule and hands m(g) to the exp
//     warps through shared memory; when m rises it rescales O (after PV(g - 1), before
//     PV(g)); it also runs the epilogue O / l of every item;
//   * the EXP warpgroups (kNE of them, tile g goes to warpgroup g % kNE) stream S(g)
//     from TMEM in 32-column chunks (two chunks in flight), exp2, E4M3-pack and store
//     P(g) into P slot g & 1, keeping their own row sums l (relative to the last m they
//     saw; the epilogue combines them);
//   * producer warps: Q + K (+ SF, S_q^K) TMA, V (+ SF) TMA; one QK issuer warp, one PV
//     issuer warp (they never wait on each other: QK(g + 2) is issued as soon as S(g) was
//     read by both softmax roles).
// K rows are in natural order in the operand (phase 1 key_perm = 2).
//
// TMEM (512 columns):
//   S0 [0,128)  S1 [128,256)  P0 [256,288)  P1 [288,320)  O [320,320+DV)
//   SF: Q 448 / 460 (per Q slot: hi 4*kChHi | lo 4*kChLo) | K 472 / 480 | V 488 / 492 | P 496
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>

#include "attn.cuh"
#include "attn_pp.cuh"
#include "attn_sk.cuh"
#include "common.cuh"
#include "ptx.cuh"

namespace dma {

#ifndef DMA_WS_NE
#define DMA_WS_NE 2
#endif
#ifndef DMA_WS_POLY
#define DMA_WS_POLY 0
#endif
// exp2 pairs (out of every 16 per 32-key chunk) on the FMA pipe (exp2_poly3)
constexpr int kPolyWS = DMA_WS_POLY;

template <int D, int DV, int LOW>
struct WSCfg {
  static constexpr int kBM = 128, kBN = 128;
  static constexpr int kNE = DMA_WS_NE;  // exp warpgroups
  static constexpr int kNK = 4, kNV = 4, kNS = 4, kNSch = 4;
  static constexpr int kWarps = 4 + 4 * kNE + 4;
  static constexpr int kThreads = 32 * kWarps;
  static constexpr int kLaunchRegs = kNE == 2 ? 128 : 168;
  static constexpr int kRegCtl = kNE == 2 ? 56 : 72;
  static constexpr int kRegSm = kNE == 2 ? 152 : 216;  // max and exp warpgroups
  static_assert(128 * (kNE + 1) * kRegSm + 128 * kRegCtl <= kThreads * kLaunchRegs, "register pool");
  static constexpr int kQHiBytes = kBM * D;
  static constexpr int kQLoBytes = kBM * D / 2;
  static constexpr int kQSlot = ((kQHiBytes + (LOW != kLowHigh ? kQLoBytes : 0) + 1023) / 1024) * 1024;
  static constexpr int kKBytes = kBN * D;
  static constexpr int kVBytes = kBN * DV;
  static constexpr int kChHi = (D / 32 + 3) / 4;
  static constexpr int kChLo = LOW == kLowNV ? (D / 16 + 3) / 4 : (D / 32 + 3) / 4;
  static constexpr int kChK = kChHi > kChLo ? kChHi : kChLo;
  static constexpr int kSfQ = 512 * (kChHi + kChLo);
  static constexpr int kSqkBytes = 4 * kSqkTile;  // 576
  // smem (offsets from a 1024-aligned base)
  static constexpr int oQ = 0;                          // [2 slot][kQSlot]
  static constexpr int oK = oQ + 2 * kQSlot;            // [kNK][kKBytes]
  static constexpr int oV = oK + kNK * kKBytes;         // [kNV][kVBytes]
  static constexpr int oSfQ = oV + kNV * kVBytes;       // [2 slot][kSfQ]
  static constexpr int oSfK = oSfQ + 2 * kSfQ;          // [kNK][kChK][512]
  static constexpr int oSfV = oSfK + kNK * kChK * 512;  // [kNV][512]
  static constexpr int oSqK = oSfV + kNV * 512;         // [kNS][kSqkBytes]
  static constexpr int oSfP = oSqK + kNS * kSqkBytes;   // 512
  static constexpr int oOnes = oSfP + 512;              // [128] f32 1.0: S_q^K of single-level tiles
  static constexpr int oSch = oOnes + 512;              // [kNSch] int
  static constexpr int oM = oSch + 64;                  // [2 slot][128] f32: m(g) for the exp warps
  static constexpr int oL = oM + 2 * 128 * 4;           // [2 item parity][kNE][128] float2 (l, m of l)
  static constexpr int oBar = oL + 2 * kNE * 128 * 8;
  static constexpr int kSmemBytes = oBar + 512 + 1024;
  static_assert(kSmemBytes <= 227 * 1024, "smem budget");
  // TMEM columns
  static constexpr uint32_t tO = 320, tSfP = 496;
  __device__ static constexpr uint32_t tS(int b) { return 128u * b; }
  __device__ static constexpr uint32_t tP(int b) { return 256u + 32u * b; }
  __device__ static constexpr uint32_t tSfQ(int slot) { return 448u + 12u * slot; }
  __device__ static constexpr uint32_t tSfK(int b) { return 472u + 8u * b; }
  __device__ static constexpr uint32_t tSfV(int b) { return 488u + 4u * b; }
  static_assert(tO + DV <= 448 && 4 * (kChHi + kChLo) <= 12 && 4 * kChK <= 8, "TMEM budget");
};

// registers written by an asynchronous tcgen05.ld must not be read before tcgen05.wait::ld;
// an empty asm that "modifies" them after the wait pins their uses behind it
__device__ __forceinline__ void reg_fence32(uint32_t (&r)[32]) {
#pragma unroll
  for (int i = 0; i < 32; ++i) asm volatile("" : "+r"(r[i]));
}

// causal (attention.py:178-184, applied when k1 - 1 > q0, :306) / ragged-key limit of a tile:
// keys >= lim of this row are masked; 128 = no mask
__device__ __forceinline__ int ws_key_limit(const AttnParams& p, int k0, int q0, int qrow) {
  const int kvalid = p.lk - k0;
  const bool need_causal = p.causal && (k0 + (kvalid < 128 ? kvalid : 128) - 1 > q0);
  if (!need_causal && kvalid >= 128) return 128;
  return need_causal ? min(qrow - k0 + 1, kvalid) : kvalid;
}

// max of one 32-key chunk (natural key order) of S * S_q^K; sqk = the chunk's 32 factors in
// shared memory (all ones on single-level tiles); MASK: keys >= lim (chunk-relative) -> -inf
template <bool MASK>
__device__ __forceinline__ float ws_chunk_max(const uint32_t (&r)[32], uint32_t sqk, int lim, float m) {
  float m4[4] = {m, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    const float4 f = ptx::lds_f4(sqk + 16 * w);
    float2 a = __fmul2_rn(make_float2(__uint_as_float(r[4 * w]), __uint_as_float(r[4 * w + 1])), make_float2(f.x, f.y));
    float2 b = __fmul2_rn(make_float2(__uint_as_float(r[4 * w + 2]), __uint_as_float(r[4 * w + 3])),
                          make_float2(f.z, f.w));
    if (MASK) {
      a.x = 4 * w < lim ? a.x : -INFINITY;
      a.y = 4 * w + 1 < lim ? a.y : -INFINITY;
      b.x = 4 * w + 2 < lim ? b.x : -INFINITY;
      b.y = 4 * w + 3 < lim ? b.y : -INFINITY;
    }
    m4[w & 3] = ptx::fmax3(m4[w & 3], ptx::fmax3(a.x, a.y, b.x), b.y);
  }
  return fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
}

// exp2 + E4M3 pack of one 32-key chunk: P word w holds keys 4w..4w+3 (x 2^kPShift via the bias)
template <bool MASK>
__device__ __forceinline__ void ws_chunk_exp(const uint32_t (&r)[32], uint32_t sqk, int lim, float2 rf2, float2 b2,
                                             uint32_t (&pk)[8], float2& ls) {
  float t[32];
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    const float4 f = ptx::lds_f4(sqk + 16 * w);
    float2 a = __fmul2_rn(make_float2(__uint_as_float(r[4 * w]), __uint_as_float(r[4 * w + 1])), make_float2(f.x, f.y));
    float2 b = __fmul2_rn(make_float2(__uint_as_float(r[4 * w + 2]), __uint_as_float(r[4 * w + 3])),
                          make_float2(f.z, f.w));
    a = __ffma2_rn(a, rf2, b2);
    b = __ffma2_rn(b, rf2, b2);
    if (MASK) {
      a.x = 4 * w < lim ? a.x : -INFINITY;
      a.y = 4 * w + 1 < lim ? a.y : -INFINITY;
      b.x = 4 * w + 2 < lim ? b.x : -INFINITY;
      b.y = 4 * w + 3 < lim ? b.y : -INFINITY;
    }
    t[4 * w] = a.x;
    t[4 * w + 1] = a.y;
    t[4 * w + 2] = b.x;
    t[4 * w + 3] = b.y;
  }
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    if (j < kPolyWS) {
      const float2 e2 = exp2_poly3(make_float2(t[2 * j], t[2 * j + 1]));
      t[2 * j] = e2.x;
      t[2 * j + 1] = e2.y;
    } else {
      t[2 * j] = exp2_ordered(t[2 * j]);
      t[2 * j + 1] = exp2_ordered(t[2 * j + 1]);
    }
  }
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    const uint32_t lo = cvt_e4m3x2_ordered(t[4 * w], t[4 * w + 1]);
    const uint32_t hi = cvt_e4m3x2_ordered(t[4 * w + 2], t[4 * w + 3]);
    pk[w] = lo | (hi << 16);
    ls = __fadd2_rn(ls, __fadd2_rn(make_float2(t[4 * w], t[4 * w + 1]), make_float2(t[4 * w + 2], t[4 * w + 3])));
  }
}

// Row max of one S tile (max warps): two 64-column halves, S released to the QK issuer as
// soon as the second half is in registers.  lim: key limit of the row (128 = no mask).
template <bool MASK>
__device__ __forceinline__ float ws_max_tile(uint32_t tS, uint32_t sqk, int lim, uint64_t* s_free_b, int lane) {
  uint32_t ra[32], rb[32];
  float mx = -INFINITY;
#pragma unroll 1
  for (int i = 0; i < 2; ++i) {
    ptx::tmem_ld32(tS + 64 * i, ra);
    ptx::tmem_ld32(tS + 64 * i + 32, rb);
    ptx::tmem_ld_wait();
    reg_fence32(ra);
    reg_fence32(rb);
    if (i == 1) {
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(s_free_b);
    }
    mx = ws_chunk_max<MASK>(ra, sqk + 256 * i, lim - 64 * i, mx);
    mx = ws_chunk_max<MASK>(rb, sqk + 256 * i + 128, lim - 64 * i - 32, mx);
  }
  return mx;
}

// exp2 / P of one S tile (exp warps): 32-column chunks, the next chunk's TMEM load in flight
// while the current one is computed.  The exponentials use the caller's guess m_use of the
// running max; once the last chunk has landed the true m(g) is read (the max warps are done
// with the tile by then): if it differs for any row of the warp, S is kept and the caller
// redoes the tile with m(g) (rare: the lazy max changes only when a row max rises by more
// than tau); otherwise S is released to the QK issuer.  Returns m(g).
template <bool MASK>
__device__ __forceinline__ float ws_exp_tile(uint32_t tS, uint32_t tP, uint32_t sqk, int lim, float2 rf2, float2 b2,
                                             float2& ls, uint64_t* s_free_b, int lane, uint64_t* m_full_b,
                                             uint32_t m_par, const float* m_row, float m_use, bool& redo) {
  uint32_t ra[32], rb[32], pk[8];
  float m_true = m_use;
  ptx::tmem_ld32(tS, ra);
  ptx::tmem_ld_wait();
  reg_fence32(ra);
#pragma unroll 1
  for (int i = 0; i < 2; ++i) {
    ptx::tmem_ld32(tS + 64 * i + 32, rb);
    ws_chunk_exp<MASK>(ra, sqk + 256 * i, lim - 64 * i, rf2, b2, pk, ls);
    ptx::tmem_st8(tP + 16 * i, pk);
    ptx::tmem_ld_wait();
    reg_fence32(rb);
    if (i == 0) {
      ptx::tmem_ld32(tS + 64, ra);
    } else {
      if (m_full_b) {
        ptx::mbar_wait(m_full_b, m_par);
        m_true = *m_row;
      }
      redo = __any_sync(0xffffffffu, m_true != m_use);
      if (!redo) {
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(s_free_b);  // S fully read: QK(g + 2) may overwrite it
      }
    }
    ws_chunk_exp<MASK>(rb, sqk + 256 * i + 128, lim - 64 * i - 32, rf2, b2, pk, ls);
    ptx::tmem_st8(tP + 16 * i + 8, pk);
    if (i == 0) {
      ptx::tmem_ld_wait();
      reg_fence32(ra);
    }
  }
  return m_true;
}

template <int D, int DV, int LOW>
__global__ void __launch_bounds__(WSCfg<D, DV, LOW>::kThreads, 1)
    dma_attn_ws_kernel(const __grid_constant__ AttnParams p, const __grid_constant__ SKParams sp) {
  using C = WSCfg<D, DV, LOW>;
  constexpr int kNE = C::kNE;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::oBar);
  uint64_t* q_full = bars;                    // [2]
  uint64_t* q_empty = q_full + 2;             // [2]
  uint64_t* k_full = q_empty + 2;             // [kNK]
  uint64_t* k_empty = k_full + C::kNK;        // [kNK]
  uint64_t* v_full = k_empty + C::kNK;        // [kNV]
  uint64_t* v_empty = v_full + C::kNV;        // [kNV]
  uint64_t* sq_empty = v_empty + C::kNV;      // [kNS]  max (4) + exp (4) warps
  uint64_t* s_full = sq_empty + C::kNS;       // [2]    QK commit
  uint64_t* s_free = s_full + 2;              // [2]    max (4) + exp (4) warps have read S
  uint64_t* m_full = s_free + 2;              // [2]    m(g) written (4 max warps)
  // [4] O rescaled for tile g (4 max warps).  Four slots: the max warps may run two tiles
  // ahead of the PV issuer (M(g + 2) needs only that S(g) was read), so a 2-slot barrier
  // would complete twice before PV(g) waits on it
  uint64_t* c_done = m_full + 2;
  uint64_t* p_full = c_done + 4;              // [2]    P(g) stored (4 exp warps)
  // [4] PV(g) complete (commit), slot g & 3.  A parity wait only tells the waited phase from
  // the one before it: the max warps wait for PV(g - 1) while PV(g - 3) may still be pending
  // (only PV(g - 4) is known complete), so two slots would alias
  uint64_t* pv_done = p_full + 2;
  uint64_t* o_free = pv_done + 4;             // [1]    epilogue read O (4 max warps)
  uint64_t* l_full = o_free + 1;              // [2 item parity][kNE] row sums published (4 exp warps)
  uint64_t* sch_full = l_full + 2 * kNE;      // [kNSch]
  uint64_t* sch_empty = sch_full + C::kNSch;  // [kNSch]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sch_empty + C::kNSch);
  int* sched = reinterpret_cast<int*>(smem + C::oSch);
  float* mbuf = reinterpret_cast<float*>(smem + C::oM);
  float2* lbuf = reinterpret_cast<float2*>(smem + C::oL);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rt_q = p.lq_pad >> 7, rt_k = p.lk_pad >> 7;
  constexpr int kProd = 4 + 4 * kNE, kQK = kProd + 1, kPV = kProd + 2, kVProd = kProd + 3;
  constexpr int kSchConsumers = 4 + 4 * kNE + 3;

  if (warp == kProd) {
    if (lane == 0) {
      for (int i = 0; i < 2; ++i) {
        ptx::mbar_init(q_full + i, 1);
        ptx::mbar_init(q_empty + i, 1);
        ptx::mbar_init(s_full + i, 1);
        ptx::mbar_init(s_free + i, 8);
        ptx::mbar_init(m_full + i, 4);
        ptx::mbar_init(c_done + i, 4);
        ptx::mbar_init(c_done + 2 + i, 4);
        ptx::mbar_init(p_full + i, 4);
        ptx::mbar_init(pv_done + i, 1);
        ptx::mbar_init(pv_done + 2 + i, 1);
      }
      ptx::mbar_init(o_free, 4);
      for (int i = 0; i < 2 * kNE; ++i) ptx::mbar_init(l_full + i, 4);
      for (int i = 0; i < C::kNK; ++i) {
        ptx::mbar_init(k_full + i, 1);
        ptx::mbar_init(k_empty + i, 1);
      }
      for (int i = 0; i < C::kNV; ++i) {
        ptx::mbar_init(v_full + i, 1);
        ptx::mbar_init(v_empty + i, 1);
      }
      for (int i = 0; i < C::kNS; ++i) ptx::mbar_init(sq_empty + i, 8);
      for (int i = 0; i < C::kNSch; ++i) {
        ptx::mbar_init(sch_full + i, 1);
        ptx::mbar_init(sch_empty + i, kSchConsumers);
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
  } else if (warp == kQK) {
    ptx::tmem_alloc<512>(tmem_slot);
  } else if (warp == 0) {
    // constant P scale-factor atom: E8M0 127 (= 1.0) for every row / k-block
    uint32_t* sfp = reinterpret_cast<uint32_t*>(smem + C::oSfP);
    for (int i = lane; i < 128; i += 32) sfp[i] = 0x7F7F7F7Fu;
    float* ones = reinterpret_cast<float*>(smem + C::oOnes);
    for (int i = lane; i < 128; i += 32) ones[i] = 1.0f;
    ptx::fence_proxy_async_smem();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sones = ptx::smem_u32(smem + C::oOnes);

  // every role walks the same item sequence from the scheduler ring
  auto next_item = [&](uint32_t i) -> int {
    const int ss = i % C::kNSch;
    ptx::mbar_wait(sch_full + ss, (i / C::kNSch) & 1);
    const int k = sched[ss];
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(sch_empty + ss);
    return k;
  };

  if (warp >= kProd) {
    // kNE = 2: 512 threads x 128 registers is the whole file, nothing to move; kNE = 1:
    // the control warpgroup gives registers to the softmax warpgroups (ptxas allocates the
    // kernel at the launch bound, so this only matters for the register pool)
    if (kNE == 1) ptx::setmaxnreg_dec<C::kRegCtl>();
    const uint32_t sbase = ptx::smem_u32(smem);
    const uint64_t sf_desc_hi = static_cast<uint64_t>(ptx::desc_hi(128, ptx::kSwNone)) << 32;
    auto sf_desc = [&](uint32_t off) { return sf_desc_hi | ptx::desc_lo(sbase + off, 0); };
    if (warp == kProd) {
      // =========================== scheduler + Q / K producer ===========================
      uint32_t ks = 0, kph = 0, po = 0, sqs = 0, sqph = 0;
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
        uint8_t* qdst = smem + C::oQ + qs * C::kQSlot;
        uint8_t* sfq = smem + C::oSfQ + qs * C::kSfQ;
        ptx::wu::tma_load_3d(qdst, &p.tm_q_hi, q_full + qs, 0, qt * C::kBM, bh);
        ptx::wu::bulk_load(sfq, p.sf_q_hi + (static_cast<int64_t>(bh) * rt_q + qt) * p.ch_hi * 512, 512 * C::kChHi,
                           q_full + qs);
        if (LOW != kLowHigh) {
          ptx::wu::tma_load_3d(qdst + C::kQHiBytes, &p.tm_q_lo, q_full + qs, 0, qt * C::kBM, bh);
          ptx::wu::bulk_load(sfq + 512 * C::kChHi, p.sf_q_lo + (static_cast<int64_t>(bh) * rt_q + qt) * p.ch_lo * 512,
                             512 * C::kChLo, q_full + qs);
        }
        for (int e = 0; e < plan.n; ++e) {
          int t;
          bool hi;
          plan.entry(e, t, hi);
          if (LOW == kLowHigh) hi = true;
          const int ch = hi ? C::kChHi : C::kChLo;
          const uint32_t kbytes = hi ? C::kKBytes : C::kKBytes / 2;
          ptx::mbar_wait(k_empty + ks, kph ^ 1);
          ptx::mbar_wait(sq_empty + sqs, sqph ^ 1);
          ptx::wu::mbar_arrive_expect_tx(k_full + ks, kbytes + 512 * ch + C::kSqkBytes);
          ptx::wu::tma_load_3d(smem + C::oK + ks * C::kKBytes, hi ? &p.tm_k_hi : &p.tm_k_lo, k_full + ks, 0,
                               t * C::kBN, mk);
          const uint8_t* sfsrc =
              (hi ? p.sf_k_hi : p.sf_k_lo) + (static_cast<int64_t>(mk) * rt_k + t) * (hi ? p.ch_hi : p.ch_lo) * 512;
          ptx::wu::bulk_load(smem + C::oSfK + ks * 512 * C::kChK, sfsrc, 512 * ch, k_full + ks);
          ptx::wu::bulk_load(smem + C::oSqK + sqs * C::kSqkBytes,
                             p.qs_k + (static_cast<int64_t>(mk) * rt_k + t) * kSqkTile, C::kSqkBytes, k_full + ks);
          if (++sqs == C::kNS) { sqs = 0; sqph ^= 1; }
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
    } else if (warp == kVProd) {
      // =========================== V producer ===========================
      uint32_t vs = 0, vph = 0;
      for (uint32_t i = 0;; ++i) {
        const int k = next_item(i);
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
          if (++vs == C::kNV) { vs = 0; vph ^= 1; }
        }
      }
    } else if (warp == kQK) {
      // =========================== QK issuer ===========================
      PROF_DECL
      const uint32_t hf = static_cast<uint32_t>(p.hfmt);
      uint32_t ks = 0, kph = 0, po = 0, g = 0;
      for (uint32_t i = 0;; ++i) {
        const int k = next_item(i);
        if (k < 0) break;
        int bh, qt;
        sk_item_coords(p, sp, k, bh, qt);
        Plan plan;
        plan.init(qt, p.lq, p.lk, C::kBM, C::kBN, p.diag_window, p.sink_window, p.causal != 0);
        if (plan.n == 0) continue;
        const int qs = po & 1;
        ptx::mbar_wait(q_full + qs, (po >> 1) & 1);
        ++po;
        ptx::tc_fence_after();
        const uint32_t oq = C::oQ + qs * C::kQSlot;
        const uint32_t osfq = C::oSfQ + qs * C::kSfQ;
        const uint32_t tsfq = tmem + C::tSfQ(qs);
        for (int j = 0; j < C::kChHi; ++j) ptx::wu::tc_cp_sf(tsfq + 4 * j, sf_desc(osfq + 512 * j));
        if (LOW != kLowHigh)
          for (int j = 0; j < C::kChLo; ++j) ptx::wu::tc_cp_sf(tsfq + 4 + 4 * j, sf_desc(osfq + 512 * (C::kChHi + j)));
        for (int e = 0; e < plan.n; ++e, ++g) {
          int t;
          bool hi;
          plan.entry(e, t, hi);
          if (LOW == kLowHigh) hi = true;
          const int b = g & 1;
          ptx::mbar_wait(s_free + b, ((g >> 1) & 1) ^ 1);  // S(g - 2) read by both softmax roles
          PROF_MARK(0); /*qk*/
          ptx::mbar_wait(k_full + ks, kph);
          PROF_MARK(1); /*qk*/
          ptx::tc_fence_after();
          const uint32_t kslt = ks;
          if (++ks == C::kNK) { ks = 0; kph ^= 1; }
          const int ch = hi ? C::kChHi : C::kChLo;
          const uint32_t tsfk = tmem + C::tSfK(b);
          for (int j = 0; j < ch; ++j)
            ptx::wu::tc_cp_sf(tsfk + 4 * j, sf_desc(C::oSfK + kslt * 512 * C::kChK + 512 * j));
          const uint32_t tSd = tmem + C::tS(b);
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
                ptx::wu::mma_nvf4(tSd, ad, bd, id, tsfq + 4 + 4 * kk, tsfk + 4 * kk, kk > 0);
              } else {
                const uint32_t sid = (kk & 1) * 2;
                const uint32_t id = ptx::idesc_bs(1, 1, 0, 0, 128, 128, 1, sid, sid);
                ptx::wu::mma_mxf4(tSd, ad, bd, id, tsfq + 4 + 4 * (kk >> 1), tsfk + 4 * (kk >> 1), kk > 0);
              }
            }
          }
          ptx::wu::tc_commit(k_empty + kslt);
          ptx::wu::tc_commit(s_full + b);
          PROF_MARK(2); /*qk*/
          if (e == plan.n - 1) ptx::wu::tc_commit(q_empty + qs);
        }
      }
      PROF_FLUSH(16, 3);
    } else {
      // =========================== PV issuer (warp kPV) ===========================
      ptx::wu::tc_cp_sf(tmem + C::tSfP, sf_desc(C::oSfP));
      PROF_DECL
      uint32_t vs = 0, vph = 0, g = 0, ui = 0;
      constexpr int rb = DV;  // fp8 V row bytes (MN-major)
      const uint64_t dh = static_cast<uint64_t>(ptx::desc_hi(8 * rb, swz_mode(rb))) << 32;
      for (uint32_t i = 0;; ++i) {
        const int k = next_item(i);
        if (k < 0) break;
        int bh, qt;
        sk_item_coords(p, sp, k, bh, qt);
        Plan plan;
        plan.init(qt, p.lq, p.lk, C::kBM, C::kBN, p.diag_window, p.sink_window, p.causal != 0);
        if (plan.n == 0) continue;
        for (int e = 0; e < plan.n; ++e, ++g) {
          const int b = g & 1;
          ptx::mbar_wait(p_full + b, (g >> 1) & 1);
          PROF_MARK(0); /*pv*/
          ptx::mbar_wait(c_done + (g & 3), (g >> 2) & 1);
          PROF_MARK(1); /*pv*/
          if (e == 0 && ui > 0) ptx::mbar_wait(o_free, (ui - 1) & 1);  // previous item's O read out
          PROF_MARK(2); /*pv*/
          ptx::mbar_wait(v_full + vs, vph);
          PROF_MARK(3); /*pv*/
          ptx::tc_fence_after();
          const uint32_t vslt = vs;
          if (++vs == C::kNV) { vs = 0; vph ^= 1; }
          ptx::wu::tc_cp_sf(tmem + C::tSfV(b), sf_desc(C::oSfV + vslt * 512));
          const uint32_t vaddr = sbase + C::oV + vslt * C::kVBytes;
#pragma unroll
          for (int kk = 0; kk < C::kBN / 32; ++kk) {
            const uint64_t bd = dh | ptx::desc_lo(vaddr + kk * 32 * rb, 16);
            const uint32_t id = ptx::idesc_bs(0, 0, 0, 1, 128, DV, 1, kk & 3, kk & 3);
            ptx::wu::mma_mxf8f6f4_ts(tmem + C::tO, tmem + C::tP(b) + 8 * kk, bd, id, tmem + C::tSfP,
                                     tmem + C::tSfV(b), !(e == 0 && kk == 0));
          }
          ptx::wu::tc_commit(v_empty + vslt);
          ptx::wu::tc_commit(pv_done + (g & 3));
          PROF_MARK(4); /*pv*/
        }
        ++ui;
      }
      PROF_FLUSH(20, 5);
    }
  } else {
    if (kNE == 1) ptx::setmaxnreg_inc<C::kRegSm>();
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
    constexpr float kLazy = 4.f;           // lazy rescaling threshold (log2 units)
    constexpr float kPShift = 8.f - kLazy;  // P <= 2^kLazy stored as E4M3(P * 2^kPShift) <= 256
    if (warp < 4) {
      // =========================== MAX warpgroup: row max, lazy m, O rescale, epilogue ===========================
      PROF_DECL
      uint32_t g = 0, ui = 0;
      // pending epilogue (the previous item): run after the next item's first max so the exp
      // warps never wait on it
      bool pend = false;
      int pend_bh = 0, pend_qrow = 0, pend_ui = 0;
      uint32_t pend_glast = 0;
      float pend_m = -INFINITY;
      auto epilogue = [&]() {
        const int pp2 = pend_ui & 1;
        float l = 0.f;
#pragma unroll
        for (int x = 0; x < kNE; ++x) {
          ptx::mbar_wait(l_full + 2 * x + pp2, (pend_ui >> 1) & 1);
          const float2 lm = lbuf[(pp2 * kNE + x) * 128 + row];
          if (lm.y != -INFINITY) l += lm.x * (lm.y == pend_m ? 1.f : fast_exp2(lm.y - pend_m));
        }
        const float inv_l = 1.0f / (l > 0.f ? l : 1.0f);
        ptx::mbar_wait(pv_done + (pend_glast & 3), (pend_glast >> 2) & 1);
        ptx::tc_fence_after();
        const int64_t orow = static_cast<int64_t>(pend_bh) * p.lq + pend_qrow;
#pragma unroll
        for (int c = 0; c < DV / 32; ++c) {
          uint32_t rr[32];
          ptx::tmem_ld32(tmem + C::tO + lane_base + 32 * c, rr);
          ptx::tmem_ld_wait();
          reg_fence32(rr);
          if (pend_qrow < p.lq) store_orow<DV>(p, orow, c, rr, inv_l);
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(o_free);
        pend = false;
      };
      for (uint32_t i = 0;; ++i) {
        const int k = next_item(i);
        PROF_MARK(4);
        if (k < 0) break;
        int bh, qt;
        sk_item_coords(p, sp, k, bh, qt);
        Plan plan;
        plan.init(qt, p.lq, p.lk, C::kBM, C::kBN, p.diag_window, p.sink_window, p.causal != 0);
        const int q0 = qt * C::kBM;
        const int qrow = q0 + row;
        if (plan.n == 0) {  // no keys: l = 0 -> the row normalises to 0 (attention.py:104-106)
          if (qrow < p.lq) {
            uint32_t rr[32];
#pragma unroll
            for (int i2 = 0; i2 < 32; ++i2) rr[i2] = 0u;
            const int64_t orow = static_cast<int64_t>(bh) * p.lq + qrow;
#pragma unroll
            for (int c = 0; c < DV / 32; ++c) store_orow<DV>(p, orow, c, rr, 1.f);
          }
          continue;
        }
        const float sq_q = (qrow < p.lq) ? p.qs_q[static_cast<int64_t>(bh) * p.lq_pad + qrow] : 1.0f;
        float m_run = -INFINITY;
        for (int e = 0; e < plan.n; ++e, ++g) {
          int t;
          bool hi;
          plan.entry(e, t, hi);
          if (LOW == kLowHigh) hi = true;
          const bool tl = hi || (LOW == kLowNV);
          const int b = g & 1;
          const int lim = ws_key_limit(p, t * C::kBN, q0, qrow);
          const uint32_t sqk = ptx::smem_u32(smem + C::oSqK + (g % C::kNS) * C::kSqkBytes);
          ptx::mbar_wait(s_full + b, (g >> 1) & 1);
          PROF_MARK(0);
          ptx::tc_fence_after();
          const uint32_t tS = tmem + C::tS(b) + lane_base;
          const uint32_t sqk_t = tl ? sqk : sones;
          const float mx = __any_sync(0xffffffffu, lim < 128) ? ws_max_tile<true>(tS, sqk_t, lim, s_free + b, lane)
                                                              : ws_max_tile<false>(tS, sqk_t, lim, s_free + b, lane);
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(sq_empty + g % C::kNS);
          const float rowf = tl ? sq_q : 1.0f;
          const float m_cand = fmaxf(m_run, mx * rowf);
          const bool upd = m_cand > m_run + kLazy;  // always for the first live tile (m_run = -inf)
          const float m_new = upd ? m_cand : m_run;
          PROF_MARK(1);
          mbuf[b * 128 + row] = m_new;
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(m_full + b);
          // O *= 2^(m_run - m_new) after PV(g - 1), before PV(g)
          const float alpha = (upd && m_run != -INFINITY) ? fast_exp2(m_run - m_new) : 1.0f;
          if (e > 0 && __any_sync(0xffffffffu, alpha != 1.0f)) {
            ptx::mbar_wait(pv_done + ((g - 1) & 3), ((g - 1) >> 2) & 1);
            ptx::tc_fence_after();
            const float2 a2 = make_float2(alpha, alpha);
#pragma unroll
            for (int cq = 0; cq < DV / 32; ++cq) {
              const uint32_t ta = tmem + C::tO + lane_base + 32 * cq;
              uint32_t rr[32];
              ptx::tmem_ld32(ta, rr);
              ptx::tmem_ld_wait();
              reg_fence32(rr);
#pragma unroll
              for (int i2 = 0; i2 < 16; ++i2) {
                const float2 v =
                    __fmul2_rn(make_float2(__uint_as_float(rr[2 * i2]), __uint_as_float(rr[2 * i2 + 1])), a2);
                rr[2 * i2] = __float_as_uint(v.x);
                rr[2 * i2 + 1] = __float_as_uint(v.y);
              }
              ptx::tmem_st32(ta, rr);
            }
            ptx::tmem_st_wait();
          }
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(c_done + (g & 3));
          PROF_MARK(2);
          m_run = m_new;
          if (e == 0 && pend) epilogue();
          PROF_MARK(3);
        }
        if (pend) epilogue();  // (only when this item had no first-tile slot for it)
        pend = true;
        pend_bh = bh;
        pend_qrow = qrow;
        pend_ui = static_cast<int>(ui);
        pend_glast = g - 1;
        pend_m = m_run;
        ++ui;
      }
      if (pend) epilogue();
      PROF_FLUSH(0, 5);
    } else {
      // =========================== EXP warpgroup x: exp2, P -> E4M3, row sums ===========================
      const int x = (warp - 4) >> 2;
      PROF_DECL
      uint32_t g = 0, ui = 0;
      for (uint32_t i = 0;; ++i) {
        const int k = next_item(i);
        PROF_MARK(13);
        if (k < 0) break;
        int bh, qt;
        sk_item_coords(p, sp, k, bh, qt);
        Plan plan;
        plan.init(qt, p.lq, p.lk, C::kBM, C::kBN, p.diag_window, p.sink_window, p.causal != 0);
        if (plan.n == 0) continue;
        const int q0 = qt * C::kBM;
        const int qrow = q0 + row;
        const float sq_q = (qrow < p.lq) ? p.qs_q[static_cast<int64_t>(bh) * p.lq_pad + qrow] : 1.0f;
        float l = 0.f, m_prev = -INFINITY;
        for (int e = 0; e < plan.n; ++e, ++g) {
          if (kNE > 1 && static_cast<int>(g % kNE) != x) continue;
          int t;
          bool hi;
          plan.entry(e, t, hi);
          if (LOW == kLowHigh) hi = true;
          const bool tl = hi || (LOW == kLowNV);
          const int b = g & 1;
          const int lim = ws_key_limit(p, t * C::kBN, q0, qrow);
          const uint32_t sqk = ptx::smem_u32(smem + C::oSqK + (g % C::kNS) * C::kSqkBytes);
          // running max: m(g) from the max warps for the item's first tile; afterwards the
          // last m this warpgroup saw, checked against m(g) at the end of the tile
          float m_use = m_prev;
          if (e == 0) {
            ptx::mbar_wait(m_full + b, (g >> 1) & 1);
            m_use = mbuf[b * 128 + row];
          }
          PROF_MARK(8);
          ptx::mbar_wait(s_full + b, (g >> 1) & 1);
          ptx::tc_fence_after();
          PROF_MARK(9);
          const float rowf = tl ? sq_q : 1.0f;
          const float2 rf2 = make_float2(rowf, rowf);
          // P slot b was read by PV(g - 2)
          if (g >= 2) {
            ptx::mbar_wait(pv_done + ((g - 2) & 3), ((g - 2) >> 2) & 1);
            ptx::tc_fence_after();
          }
          PROF_MARK(10);
          const uint32_t tS = tmem + C::tS(b) + lane_base;
          const uint32_t tP = tmem + C::tP(b) + lane_base;
          const uint32_t sqk_t = tl ? sqk : sones;
          const bool msk = __any_sync(0xffffffffu, lim < 128);
          float2 ls = make_float2(0.f, 0.f);
          float m_new = m_use;
          bool redo = false;
          {
            const float bias = m_use == -INFINITY ? 0.f : (kPShift - m_use);
            const float2 b2 = make_float2(bias, bias);
            uint64_t* mf = e == 0 ? nullptr : m_full + b;
            m_new = msk ? ws_exp_tile<true>(tS, tP, sqk_t, lim, rf2, b2, ls, s_free + b, lane, mf, (g >> 1) & 1,
                                            mbuf + b * 128 + row, m_use, redo)
                        : ws_exp_tile<false>(tS, tP, sqk_t, lim, rf2, b2, ls, s_free + b, lane, mf, (g >> 1) & 1,
                                             mbuf + b * 128 + row, m_use, redo);
          }
          if (redo) {  // the running max moved: redo the tile with m(g) (S was kept)
            const float bias = m_new == -INFINITY ? 0.f : (kPShift - m_new);
            const float2 b2 = make_float2(bias, bias);
            bool again = false;
            ls = make_float2(0.f, 0.f);
            if (msk)
              ws_exp_tile<true>(tS, tP, sqk_t, lim, rf2, b2, ls, s_free + b, lane, nullptr, 0, nullptr, m_new, again);
            else
              ws_exp_tile<false>(tS, tP, sqk_t, lim, rf2, b2, ls, s_free + b, lane, nullptr, 0, nullptr, m_new, again);
          }
          if (m_new != m_prev && m_prev != -INFINITY) l *= fast_exp2(m_prev - m_new);
          m_prev = m_new;
          PROF_MARK(11);
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(sq_empty + g % C::kNS);
          l += ls.x + ls.y;
          ptx::tmem_st_wait();
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(p_full + b);
          PROF_MARK(12);
        }
        // row sum of this warpgroup's tiles (relative to m_prev) for the epilogue
        PROF_MARK(13);
        lbuf[((ui & 1) * kNE + x) * 128 + row] = make_float2(l, m_prev);
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(l_full + 2 * x + (ui & 1));
        ++ui;
      }
      PROF_FLUSH(0, 14);
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == kQK) ptx::tmem_dealloc<512>(tmem);
}

}  // namespace dma
