// Phase 2 of the DMA forward, ping-pong variant (block-scaled MXFP8 PV).
//
// Same algorithm as attn.cuh (attention.py:282-310 with the plans of
// attention.py:191-233 and the base-2 online softmax of :150-175), organised
// for overlap: every CTA runs TWO independent query-tile streams A and B,
// each with its own softmax warpgroup, so that one stream's exp2 phase
// (MUFU-bound) overlaps the other's TMEM loads / max / bookkeeping.
//
// Work unit = a *pair*: the same 128-row query tile of two heads (bh, bh+1).
// Both heads have the same tile plan, so the two streams walk identical
// (key tile, precision) sequences; with GQA they usually share the KV head,
// and then every K / V tile is loaded once and used by both.  Pairs are
// handed out dynamically (global atomic ticket), head-major when the K/V
// footprint exceeds L2 (the 148 CTAs then stream the same K/V), otherwise
// longest-causal-tile first.
//
// TMEM (512 columns), one S buffer shared by the streams:
//   S [0,128)  P_A [128,160)  P_B [160,192)  O_A [192,+DV)  O_B [320,+DV)
//   SF: Q_A 448 | Q_B 460 | K_A 472 | K_B 480 | V_A 488 | V_B 492 | P 496
// The MMA issuer runs QK_A(0) QK_B(0) { QK_A(j+1) PV_A(j) QK_B(j+1) PV_B(j) }:
// a QK waits until the previous S consumer has copied S into registers.
//
// Warps: 0-3 softmax stream A, 4-7 softmax stream B, 8 producer (TMA +
//        scheduler), 9 MMA issuer, 10-11 idle.  setmaxnreg moves registers from
//        warpgroup 2 (72 each) to the softmax warpgroups (216 each), whose
//        128-value S fragment stays in registers.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>

#include "attn.cuh"
#include "common.cuh"
#include "ptx.cuh"

namespace dma {

// Optional phase timers (-DDMA_PROFILE): per-role cycle counters summed over
// all warps into g_prof (read back with dma_prof_read).  Off in normal builds.
#ifdef DMA_PROFILE
__device__ unsigned long long g_prof[32];
#define PROF_DECL unsigned long long prof_acc[16] = {0}; long long prof_t = clock64();
#define PROF_MARK(i)                       \
  do {                                     \
    const long long _t = clock64();        \
    prof_acc[i] += (unsigned long long)(_t - prof_t); \
    prof_t = _t;                           \
  } while (0)
#define PROF_FLUSH(base, n)                                          \
  do {                                                               \
    if ((threadIdx.x & 31) == 0)                                     \
      for (int _i = 0; _i < (n); ++_i) atomicAdd(&g_prof[(base) + _i], prof_acc[_i]); \
  } while (0)
#else
#define PROF_DECL
#define PROF_MARK(i) do {} while (0)
#define PROF_FLUSH(base, n) do {} while (0)
#endif

#ifndef DMA_PP_TURNS
#define DMA_PP_TURNS 0
#endif
// 1: the two softmax warpgroups take strict turns for their exp2 phases
constexpr bool kTurns = DMA_PP_TURNS != 0;
#ifndef DMA_PP_FRAG16
#define DMA_PP_FRAG16 0
#endif
// 1: softmax threads hold 4 rows x 32 columns (16x256b TMEM shape); 0: one row each (32x32b)
constexpr bool kFrag16 = DMA_PP_FRAG16 != 0;

struct PPParams {
  int n_pairs;
  int pairs_per_qt;
  int head_major;
  unsigned int* ticket;  // [0] next pair, [1] CTAs done (self-resetting)
};

template <int D, int DV, int LOW>
struct PPCfg {
  static constexpr int kBM = 128, kBN = 128;
  static constexpr int kNK = 4, kNV = 3, kNS = 4, kNSch = 4;
  static constexpr int kQHiBytes = kBM * D;
  static constexpr int kQLoBytes = kBM * D / 2;
  static constexpr int kQStream = ((kQHiBytes + (LOW != kLowHigh ? kQLoBytes : 0) + 1023) / 1024) * 1024;
  static constexpr int kKBytes = kBN * D;
  static constexpr int kVBytes = kBN * DV;
  static constexpr int kChHi = (D / 32 + 3) / 4;
  static constexpr int kChLo = LOW == kLowNV ? (D / 16 + 3) / 4 : (D / 32 + 3) / 4;
  static constexpr int kChK = kChHi > kChLo ? kChHi : kChLo;
  static constexpr int kSfQ = 512 * (kChHi + kChLo);
  // smem (offsets from a 1024-aligned base)
  static constexpr int oQ = 0;                                // [2 slot][2 stream][kQStream]
  static constexpr int oK = oQ + 4 * kQStream;                // [kNK][kKBytes]
  static constexpr int oV = oK + kNK * kKBytes;               // [kNV][kVBytes]
  static constexpr int oSfQ = oV + kNV * kVBytes;             // [2 slot][2 stream][kSfQ]
  static constexpr int oSfK = oSfQ + 4 * kSfQ;                // [kNK][kChK][512]
  static constexpr int oSfV = oSfK + kNK * kChK * 512;        // [kNV][512]
  static constexpr int kSqkBytes = 4 * kSqkTile;              // 576: S_q^K of one tile, bank-padded
  static constexpr int oSqK = oSfV + kNV * 512;               // [2 stream][kNS][kSqkBytes]
  static constexpr int oSfP = oSqK + 2 * kNS * kSqkBytes;     // 512
  static constexpr int oSch = oSfP + 512;                     // [kNSch] int
  static constexpr int oBar = oSch + 64;
  static constexpr int kSmemBytes = oBar + 512 + 1024;
  // TMEM columns
  static constexpr uint32_t tS = 0, tSfP = 496;
  __device__ static constexpr uint32_t tP(int x) { return 128u + 32u * x; }
  __device__ static constexpr uint32_t tO(int x) { return 192u + 128u * x; }
  __device__ static constexpr uint32_t tSfQ(int x) { return 448u + 12u * x; }
  __device__ static constexpr uint32_t tSfK(int x) { return 472u + 8u * x; }
  __device__ static constexpr uint32_t tSfV(int x) { return 488u + 4u * x; }
};

__device__ __forceinline__ void pair_coords(const AttnParams& p, const PPParams& q, int k, int& bh0, int& bh1,
                                            int& qt) {
  int r, hp;
  if (q.head_major) {
    hp = k / p.n_qt;
    r = k - hp * p.n_qt;
  } else {
    r = k / q.pairs_per_qt;
    hp = k - r * q.pairs_per_qt;
  }
  qt = p.causal ? p.n_qt - 1 - r : r;
  bh0 = 2 * hp;
  bh1 = 2 * hp + 1 < p.n_bh ? 2 * hp + 1 : -1;
}

__device__ __forceinline__ int mat_k_of(const AttnParams& p, int bh) {
  const int b = bh / p.heads, h = bh - b * p.heads;
  return b * p.kv_heads + h / p.group;
}


// one 32-column chunk c of an output row: O[row, 32c + i] = acc[i] * inv_l (bf16 or f32)
template <int DV>
__device__ __forceinline__ void store_orow(const AttnParams& p, int64_t orow, int c, const uint32_t (&rr)[32],
                                           float inv_l) {
  if (p.out_bf16) {
    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.o) + orow * DV + 32 * c);
#pragma unroll
    for (int i2 = 0; i2 < 4; ++i2) {
      uint32_t wv[4];
#pragma unroll
      for (int k2 = 0; k2 < 4; ++k2) {
        __nv_bfloat162 v = __floats2bfloat162_rn(__uint_as_float(rr[8 * i2 + 2 * k2]) * inv_l,
                                                 __uint_as_float(rr[8 * i2 + 2 * k2 + 1]) * inv_l);
        wv[k2] = *reinterpret_cast<uint32_t*>(&v);
      }
      dst[i2] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
    }
  } else {
    float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.o) + orow * DV + 32 * c);
#pragma unroll
    for (int i2 = 0; i2 < 8; ++i2)
      dst[i2] = make_float4(__uint_as_float(rr[4 * i2]) * inv_l, __uint_as_float(rr[4 * i2 + 1]) * inv_l,
                            __uint_as_float(rr[4 * i2 + 2]) * inv_l, __uint_as_float(rr[4 * i2 + 3]) * inv_l);
  }
}

template <int D, int DV, int LOW>
__global__ void __launch_bounds__(384, 1) dma_attn_pp_kernel(const __grid_constant__ AttnParams p,
                                                             const __grid_constant__ PPParams pp) {
  using C = PPCfg<D, DV, LOW>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared address space
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::oBar);
  uint64_t* q_full = bars;                        // [2]
  uint64_t* q_empty = q_full + 2;                 // [2]
  uint64_t* k_full = q_empty + 2;                 // [kNK]
  uint64_t* k_empty = k_full + C::kNK;            // [kNK]
  uint64_t* v_full = k_empty + C::kNK;            // [kNV]
  uint64_t* v_empty = v_full + C::kNV;            // [kNV]
  uint64_t* sq_empty = v_empty + C::kNV;          // [2][kNS]
  uint64_t* s_free = sq_empty + 2 * C::kNS;       // 1
  uint64_t* s_full = s_free + 1;                  // [2]
  uint64_t* p_full = s_full + 2;                  // [2]
  uint64_t* o_done = p_full + 2;                  // [2]
  uint64_t* sch_full = o_done + 2;                // [kNSch]
  uint64_t* sch_empty = sch_full + C::kNSch;      // [kNSch]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sch_empty + C::kNSch);
  int* sched = reinterpret_cast<int*>(smem + C::oSch);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rt_q = p.lq_pad >> 7, rt_k = p.lk_pad >> 7;

  constexpr int kProducer = 8, kMma = 9;  // warps 0-7: softmax (stream = warp / 4)
  if (warp == kProducer) {
    if (lane == 0) {
      for (int i = 0; i < 2; ++i) {
        ptx::mbar_init(q_full + i, 1);
        ptx::mbar_init(q_empty + i, 1);
        ptx::mbar_init(s_full + i, 1);
        ptx::mbar_init(p_full + i, 4);
        ptx::mbar_init(o_done + i, 1);
      }
      for (int i = 0; i < C::kNK; ++i) {
        ptx::mbar_init(k_full + i, 1);
        ptx::mbar_init(k_empty + i, 1);
      }
      for (int i = 0; i < C::kNV; ++i) {
        ptx::mbar_init(v_full + i, 1);
        ptx::mbar_init(v_empty + i, 1);
      }
      for (int i = 0; i < 2 * C::kNS; ++i) ptx::mbar_init(sq_empty + i, 4);
      ptx::mbar_init(s_free, 4);
      for (int i = 0; i < C::kNSch; ++i) {
        ptx::mbar_init(sch_full + i, 1);
        ptx::mbar_init(sch_empty + i, 1 + 8);
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
  } else if (warp == kMma) {
    ptx::tmem_alloc<512>(tmem_slot);
  } else if (warp == 0) {
    // constant P scale-factor atom: E8M0 127 (= 1.0) for every row / k-block
    uint32_t* sfp = reinterpret_cast<uint32_t*>(smem + C::oSfP);
    for (int i = lane; i < 128; i += 32) sfp[i] = 0x7F7F7F7Fu;
    ptx::fence_proxy_async_smem();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= 8) {
  // register budget: warpgroup 2 gives registers to the softmax warpgroups
  ptx::setmaxnreg_dec<72>();
  // Producer and MMA issuer run as whole warps in lock-step (warp-uniform control
  // flow) and issue their async ops through ptx::wu: one elected lane, operands in
  // uniform registers, one SASS instruction per TMA / tcgen05 op.
  const uint32_t sbase = ptx::smem_u32(smem);
  if (warp == kProducer) {
    // =========================== scheduler + TMA producer ===========================
    PROF_DECL
    uint32_t ks = 0, kph = 0, vs = 0, vph = 0, po = 0;
    uint32_t sqs[2] = {0, 0}, sqph[2] = {0, 0};
    for (uint32_t i = 0;; ++i) {
      const int ss = i % C::kNSch;
      PROF_MARK(0);
      ptx::mbar_wait(sch_empty + ss, ((i / C::kNSch) & 1) ^ 1);
      PROF_MARK(1);
      unsigned int tk = 0;
      if (lane == 0) tk = atomicAdd(pp.ticket, 1u);
      tk = __shfl_sync(0xffffffffu, tk, 0);
      const int k = tk < static_cast<unsigned int>(pp.n_pairs) ? static_cast<int>(tk) : -1;
      if (lane == 0) {
        sched[ss] = k;
        ptx::mbar_arrive(sch_full + ss);  // release: the slot write is visible to waiters
      }
      __syncwarp();
      if (k < 0) break;
      int bh[2], qt;
      pair_coords(p, pp, k, bh[0], bh[1], qt);
      Plan plan;
      plan.init(qt, p.lq, p.lk, C::kBM, C::kBN, p.diag_window, p.sink_window, p.causal != 0);
      if (plan.n == 0) continue;
      const int ns = bh[1] >= 0 ? 2 : 1;
      const int mk[2] = {mat_k_of(p, bh[0]), ns == 2 ? mat_k_of(p, bh[1]) : -1};
      const bool shared_kv = ns == 2 && mk[0] == mk[1];
      // ---- Q (both streams) into the pair's slot
      const int qs = po & 1;
      PROF_MARK(0);
      ptx::mbar_wait(q_empty + qs, ((po >> 1) & 1) ^ 1);
      PROF_MARK(2);
      ++po;
      uint32_t qbytes = C::kQHiBytes + 512 * C::kChHi;
      if (LOW != kLowHigh) qbytes += C::kQLoBytes + 512 * C::kChLo;
      ptx::wu::mbar_arrive_expect_tx(q_full + qs, qbytes * ns);
      for (int x = 0; x < ns; ++x) {
        uint8_t* qdst = smem + C::oQ + (qs * 2 + x) * C::kQStream;
        uint8_t* sfq = smem + C::oSfQ + (qs * 2 + x) * C::kSfQ;
        ptx::wu::tma_load_3d(qdst, &p.tm_q_hi, q_full + qs, 0, qt * C::kBM, bh[x]);
        ptx::wu::bulk_load(sfq, p.sf_q_hi + (static_cast<int64_t>(bh[x]) * rt_q + qt) * p.ch_hi * 512,
                           512 * C::kChHi, q_full + qs);
        if (LOW != kLowHigh) {
          ptx::wu::tma_load_3d(qdst + C::kQHiBytes, &p.tm_q_lo, q_full + qs, 0, qt * C::kBM, bh[x]);
          ptx::wu::bulk_load(sfq + 512 * C::kChHi,
                             p.sf_q_lo + (static_cast<int64_t>(bh[x]) * rt_q + qt) * p.ch_lo * 512, 512 * C::kChLo,
                             q_full + qs);
        }
      }
      // ---- per tile: K (+SF +S_q^K) per distinct KV head, then V (+SF)
      const int nk = shared_kv ? 1 : ns;
      for (int e = 0; e < plan.n; ++e) {
        int t;
        bool hi;
        plan.entry(e, t, hi);
        if (LOW == kLowHigh) hi = true;
        const int ch = hi ? C::kChHi : C::kChLo;
        const uint32_t kbytes = hi ? C::kKBytes : C::kKBytes / 2;
        for (int x = 0; x < nk; ++x) {
          PROF_MARK(0);
          ptx::mbar_wait(k_empty + ks, kph ^ 1);
          PROF_MARK(3);
          // S_q^K for the stream(s) reading this K tile
          const int s0 = x, s1 = shared_kv ? ns : x + 1;
          for (int y = s0; y < s1; ++y) ptx::mbar_wait(sq_empty + y * C::kNS + sqs[y], sqph[y] ^ 1);
          PROF_MARK(4);
          ptx::wu::mbar_arrive_expect_tx(k_full + ks, kbytes + 512 * ch + C::kSqkBytes * (s1 - s0));
          ptx::wu::tma_load_3d(smem + C::oK + ks * C::kKBytes, hi ? &p.tm_k_hi : &p.tm_k_lo, k_full + ks, 0,
                               t * C::kBN, mk[x]);
          const uint8_t* sfsrc = (hi ? p.sf_k_hi : p.sf_k_lo) +
                                 (static_cast<int64_t>(mk[x]) * rt_k + t) * (hi ? p.ch_hi : p.ch_lo) * 512;
          ptx::wu::bulk_load(smem + C::oSfK + ks * 512 * C::kChK, sfsrc, 512 * ch, k_full + ks);
          for (int y = s0; y < s1; ++y) {
            ptx::wu::bulk_load(smem + C::oSqK + (y * C::kNS + sqs[y]) * C::kSqkBytes,
                               p.qs_k + (static_cast<int64_t>(mk[x]) * rt_k + t) * kSqkTile, C::kSqkBytes,
                               k_full + ks);
            if (++sqs[y] == C::kNS) { sqs[y] = 0; sqph[y] ^= 1; }
          }
          if (++ks == C::kNK) { ks = 0; kph ^= 1; }
        }
        for (int x = 0; x < nk; ++x) {
          PROF_MARK(0);
          ptx::mbar_wait(v_empty + vs, vph ^ 1);
          PROF_MARK(5);
          ptx::wu::mbar_arrive_expect_tx(v_full + vs, C::kVBytes + 512);
          ptx::wu::tma_load_3d(smem + C::oV + vs * C::kVBytes, &p.tm_v, v_full + vs, 0, t * C::kBN, mk[x]);
          ptx::wu::bulk_load(smem + C::oSfV + vs * 512, p.sf_v + (static_cast<int64_t>(mk[x]) * rt_k + t) * 512, 512,
                             v_full + vs);
          if (++vs == C::kNV) { vs = 0; vph ^= 1; }
        }
      }
    }
    PROF_MARK(0);
    PROF_FLUSH(22, 6);
    // last CTA out resets the ticket for the next launch (stream-ordered)
    if (lane == 0) {
      __threadfence();
      const unsigned int done = atomicAdd(pp.ticket + 1, 1u);
      if (done == gridDim.x - 1) {
        pp.ticket[0] = 0u;
        pp.ticket[1] = 0u;
        __threadfence();
      }
    }
  } else if (warp == kMma) {
    // =========================== MMA issuer ===========================
    const uint64_t sf_desc_hi = static_cast<uint64_t>(ptx::desc_hi(128, ptx::kSwNone)) << 32;
    auto sf_desc = [&](uint32_t off) { return sf_desc_hi | ptx::desc_lo(sbase + off, 0); };
    ptx::wu::tc_cp_sf(tmem + C::tSfP, sf_desc(C::oSfP));
    PROF_DECL
    uint32_t ks = 0, kph = 0, vs = 0, vph = 0, su = 0, po = 0, pvc[2] = {0, 0};
    // instruction descriptors (loop-invariant)
    const uint32_t hf = static_cast<uint32_t>(p.hfmt);
    for (uint32_t i = 0;; ++i) {
      const int ss = i % C::kNSch;
      PROF_MARK(0);
      ptx::mbar_wait(sch_full + ss, (i / C::kNSch) & 1);
      PROF_MARK(1);
      const int k = sched[ss];
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(sch_empty + ss);
      if (k < 0) break;
      int bh[2], qt;
      pair_coords(p, pp, k, bh[0], bh[1], qt);
      Plan plan;
      plan.init(qt, p.lq, p.lk, C::kBM, C::kBN, p.diag_window, p.sink_window, p.causal != 0);
      if (plan.n == 0) continue;
      const int ns = bh[1] >= 0 ? 2 : 1;
      const bool shared_kv = ns == 2 && mat_k_of(p, bh[0]) == mat_k_of(p, bh[1]);
      const int qs = po & 1;
      PROF_MARK(0);
      ptx::mbar_wait(q_full + qs, (po >> 1) & 1);
      PROF_MARK(2);
      ++po;
      ptx::tc_fence_after();
      uint32_t kslot[2] = {0, 0}, vslot[2] = {0, 0};

      auto issue_qk = [&](int x, int e) {
        int t;
        bool hi;
        plan.entry(e, t, hi);
        if (LOW == kLowHigh) hi = true;
        // the single S buffer: wait until its previous user copied it out
        PROF_MARK(0);
        ptx::mbar_wait(s_free, (su & 1) ^ 1);
        PROF_MARK(3);
        ++su;
        ptx::tc_fence_after();
        const uint32_t oq = C::oQ + (qs * 2 + x) * C::kQStream;
        if (e == 0) {
          const uint32_t osfq = C::oSfQ + (qs * 2 + x) * C::kSfQ;
          for (int j = 0; j < C::kChHi; ++j) ptx::wu::tc_cp_sf(tmem + C::tSfQ(x) + 4 * j, sf_desc(osfq + 512 * j));
          if (LOW != kLowHigh)
            for (int j = 0; j < C::kChLo; ++j)
              ptx::wu::tc_cp_sf(tmem + C::tSfQ(x) + 4 + 4 * j, sf_desc(osfq + 512 * (C::kChHi + j)));
        }
        if (x == 0 || !shared_kv) {
          kslot[x] = ks;
          PROF_MARK(0);
          ptx::mbar_wait(k_full + ks, kph);
          PROF_MARK(4);
          if (++ks == C::kNK) { ks = 0; kph ^= 1; }
          ptx::tc_fence_after();
        } else {
          kslot[1] = kslot[0];
        }
        const uint32_t kslt = kslot[x];
        const int ch = hi ? C::kChHi : C::kChLo;
        PROF_MARK(0);
        for (int j = 0; j < ch; ++j)
          ptx::wu::tc_cp_sf(tmem + C::tSfK(x) + 4 * j, sf_desc(C::oSfK + kslt * 512 * C::kChK + 512 * j));
        PROF_MARK(7);
        const uint32_t kaddr = sbase + C::oK + kslt * C::kKBytes;
        const uint32_t tsfq = tmem + C::tSfQ(x), tsfk = tmem + C::tSfK(x), tSd = tmem + C::tS;
        if (hi) {
          constexpr int rb = D;
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
        PROF_MARK(8);
        if (x == ns - 1 || !shared_kv) ptx::wu::tc_commit(k_empty + kslt);  // last reader of this K slot
        ptx::wu::tc_commit(s_full + x);
        if (e == plan.n - 1 && x == ns - 1) ptx::wu::tc_commit(q_empty + qs);  // Q slot free after these
        PROF_MARK(9);
      };

      auto issue_pv = [&](int x, int e) {
        PROF_MARK(0);
        ptx::mbar_wait(p_full + x, pvc[x] & 1);
        PROF_MARK(5);
        ++pvc[x];
        ptx::tc_fence_after();
        if (x == 0 || !shared_kv) {
          vslot[x] = vs;
          PROF_MARK(0);
          ptx::mbar_wait(v_full + vs, vph);
          PROF_MARK(6);
          if (++vs == C::kNV) { vs = 0; vph ^= 1; }
          ptx::tc_fence_after();
        } else {
          vslot[1] = vslot[0];
        }
        const uint32_t vslt = vslot[x];
        PROF_MARK(0);
        ptx::wu::tc_cp_sf(tmem + C::tSfV(x), sf_desc(C::oSfV + vslt * 512));
        PROF_MARK(7);
        const uint32_t vaddr = sbase + C::oV + vslt * C::kVBytes;
        constexpr int rb = DV;  // fp8 V row bytes (MN-major)
        const uint64_t dh = static_cast<uint64_t>(ptx::desc_hi(8 * rb, swz_mode(rb))) << 32;
#pragma unroll
        for (int kk = 0; kk < C::kBN / 32; ++kk) {
          const uint64_t bd = dh | ptx::desc_lo(vaddr + kk * 32 * rb, 16);
          const uint32_t id = ptx::idesc_bs(0, 0, 0, 1, 128, DV, 1, kk & 3, kk & 3);
          ptx::wu::mma_mxf8f6f4_ts(tmem + C::tO(x), tmem + C::tP(x) + 8 * kk, bd, id, tmem + C::tSfP,
                                   tmem + C::tSfV(x), !(e == 0 && kk == 0));
        }
        PROF_MARK(8);
        if (x == ns - 1 || !shared_kv) ptx::wu::tc_commit(v_empty + vslt);
        ptx::wu::tc_commit(o_done + x);
        PROF_MARK(9);
      };

      issue_qk(0, 0);
      if (ns == 2) issue_qk(1, 0);
      for (int e = 0; e < plan.n; ++e) {
        if (e + 1 < plan.n) issue_qk(0, e + 1);
        issue_pv(0, e);
        if (ns == 2) {
          if (e + 1 < plan.n) issue_qk(1, e + 1);
          issue_pv(1, e);
        }
      }
    }
    PROF_MARK(0);
    PROF_FLUSH(10, 10);
  }
  } else if (!kFrag16) {
    ptx::setmaxnreg_inc<216>();  // the 128-value S row stays in registers
    // =========================== softmax (one warpgroup per stream) ===========================
    // TMEM is read in the 32x32b shape: thread = one query row (lane of its warp's
    // 32-lane sub-partition), all 128 S columns.  Row max / sum need no shuffles and
    // the per-row bookkeeping (max, alpha, bias) is done once per thread.  K rows are
    // permuted inside every 128-key tile (perm_row, for the 16x256b variant); since
    // a thread owns the whole row, undoing it is register renaming at compile time:
    // key k sits in S column perm_row(k), its S_q^K in slot perm_slot(k).
    const int x = warp >> 2;  // stream
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
    // lazy rescaling (see the 16x256b variant below): P <= 2^kLazy, stored as E4M3(P * 2^(8 - kLazy))
    constexpr float kLazy = 4.f;
    constexpr float kPShift = 8.f - kLazy;
    uint32_t g = 0, sc = 0;
    if (kTurns && x == 1) ptx::named_bar_arrive(1, 256);  // A takes the first exp phase
    PROF_DECL

    for (uint32_t it = 0;; ++it) {
      const int ss = it % C::kNSch;
      ptx::mbar_wait(sch_full + ss, (it / C::kNSch) & 1);
      const int k = sched[ss];
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(sch_empty + ss);
      if (k < 0) break;
      int bh[2], qt;
      pair_coords(p, pp, k, bh[0], bh[1], qt);
      const int my_bh = bh[x];
      Plan plan;
      plan.init(qt, p.lq, p.lk, C::kBM, C::kBN, p.diag_window, p.sink_window, p.causal != 0);
      if (my_bh < 0) continue;  // odd head count: stream B idles on this pair
      const bool pair2 = bh[1] >= 0;
      const int q0 = qt * C::kBM;
      const int qrow = q0 + row;
      const float sq_q = (qrow < p.lq) ? p.qs_q[static_cast<int64_t>(my_bh) * p.lq_pad + qrow] : 1.0f;
      float m_run = -INFINITY;
      float2 l2 = make_float2(0.f, 0.f);

      for (int e = 0; e < plan.n; ++e, ++g) {
        int t;
        bool hi;
        plan.entry(e, t, hi);
        if (LOW == kLowHigh) hi = true;
        const bool two_level = hi || (LOW == kLowNV);
        const int k0 = t * C::kBN;
        PROF_MARK(9);
        ptx::mbar_wait(s_full + x, g & 1);
        ptx::tc_fence_after();
        PROF_MARK(0);
        // S columns [0, 64) hold keys [0, 64) (permuted), [64, 128) keys [64, 128):
        // load the first half, start the second, scale the first while it lands
        uint32_t sr[128];
        ptx::tmem_ld32(tmem + C::tS + lane_base, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
        ptx::tmem_ld32(tmem + C::tS + lane_base + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
        ptx::tmem_ld_wait();
        ptx::tmem_ld32(tmem + C::tS + lane_base + 64, *reinterpret_cast<uint32_t(*)[32]>(&sr[64]));
        ptx::tmem_ld32(tmem + C::tS + lane_base + 96, *reinterpret_cast<uint32_t(*)[32]>(&sr[96]));
        PROF_MARK(1);
        // t[k] = S[key k] * S_q^K[k] in natural key order (FMUL2 over key pairs 4w + {0,1}, {2,3},
        // which are adjacent S columns perm_row(4w) + {0, 1})
        const int sl = sc % C::kNS;
        ++sc;
        const uint32_t sqk = ptx::smem_u32(smem + C::oSqK + (x * C::kNS + sl) * C::kSqkBytes);
        float tv[128];
        auto scale_words = [&](int w0) {
#pragma unroll
          for (int w = w0; w < w0 + 16; ++w) {
            const int c0 = perm_row(4 * w), c1 = perm_row(4 * w + 2);
            float2 a = make_float2(__uint_as_float(sr[c0]), __uint_as_float(sr[c0 + 1]));
            float2 b = make_float2(__uint_as_float(sr[c1]), __uint_as_float(sr[c1 + 1]));
            if (two_level) {
              const float4 f = ptx::lds_f4(sqk + 4 * perm_slot(4 * w));
              a = __fmul2_rn(a, make_float2(f.x, f.y));
              b = __fmul2_rn(b, make_float2(f.z, f.w));
            }
            tv[4 * w] = a.x;
            tv[4 * w + 1] = a.y;
            tv[4 * w + 2] = b.x;
            tv[4 * w + 3] = b.y;
          }
        };
        scale_words(0);
        ptx::tmem_ld_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(s_free);  // S buffer may be overwritten by the next QK
        scale_words(16);
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(sq_empty + x * C::kNS + sl);
        PROF_MARK(2);
        // causal (attention.py:178-184, applied when k1-1 > q0, :306) and ragged-key masks
        const int kvalid = p.lk - k0;
        const bool need_causal = p.causal && (k0 + (kvalid < C::kBN ? kvalid : C::kBN) - 1 > q0);
        if (need_causal || kvalid < C::kBN) {
          const int lim = need_causal ? min(qrow - k0 + 1, kvalid) : kvalid;
#pragma unroll
          for (int j = 0; j < 128; ++j)
            if (j >= lim) tv[j] = -INFINITY;
        }
        float mx = ptx::fmax3(tv[0], tv[1], tv[2]);
        float mx2 = ptx::fmax3(tv[3], tv[4], tv[5]);
#pragma unroll
        for (int j = 6; j < 126; j += 4) {
          mx = ptx::fmax3(mx, tv[j], tv[j + 1]);
          mx2 = ptx::fmax3(mx2, tv[j + 2], tv[j + 3]);
        }
        mx = ptx::fmax3(mx, mx2, fmaxf(tv[126], tv[127]));
        const float rowf = two_level ? sq_q : 1.0f;
        const float m_cand = fmaxf(m_run, mx * rowf);
        const bool upd = m_cand > m_run + kLazy;  // always for the first live tile (m_run = -inf)
        const float m_new = upd ? m_cand : m_run;
        const bool dead = (m_new == -INFINITY);
        const float alpha = (dead || !upd) ? 1.0f : fast_exp2(m_run - m_new);  // m_run = -inf -> 0
        const float bias = dead ? 0.f : (kPShift - m_new);
        m_run = m_new;
        PROF_MARK(3);
        // P_x (and O_x) are read by PV(e-1): wait for it before overwriting
        if (e > 0) {
          ptx::mbar_wait(o_done + x, (g - 1) & 1);
          ptx::tc_fence_after();
        }
        PROF_MARK(4);
        // exp phases of the two streams alternate (A, B, A, B, ...): MUFU.EX2 is the
        // shared bottleneck; each stream's S load / scale / max / O rescale runs during
        // the other's exp phase (named barriers 1 = "A may exp", 2 = "B may exp")
        if (kTurns && pair2) ptx::named_bar_sync(1 + x, 256);
        PROF_MARK(5);
        const float2 rf2 = make_float2(rowf, rowf), b2 = make_float2(bias, bias);
        float2 ls = make_float2(0.f, 0.f);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {  // 32 keys = 8 P words per tcgen05.st
          uint32_t pk[8];
#pragma unroll
          for (int w = 0; w < 8; ++w) {
            const int k4 = 32 * q4 + 4 * w;
            float2 x0 = __ffma2_rn(make_float2(tv[k4], tv[k4 + 1]), rf2, b2);
            float2 x1 = __ffma2_rn(make_float2(tv[k4 + 2], tv[k4 + 3]), rf2, b2);
            x0.x = fast_exp2(x0.x);
            x0.y = fast_exp2(x0.y);
            x1.x = fast_exp2(x1.x);
            x1.y = fast_exp2(x1.y);
            const float2 s01 = __fadd2_rn(x0, x1);
            ls = (q4 == 0 && w == 0) ? s01 : __fadd2_rn(ls, s01);
            pk[w] = static_cast<uint32_t>(ptx::cvt_e4m3x2(x0.x, x0.y)) |
                    (static_cast<uint32_t>(ptx::cvt_e4m3x2(x1.x, x1.y)) << 16);
          }
          ptx::tmem_st8(tmem + C::tP(x) + lane_base + 8 * q4, pk);
        }
        if (kTurns && pair2) ptx::named_bar_arrive(2 - x, 256);
        l2 = __ffma2_rn(l2, make_float2(alpha, alpha), ls);
        PROF_MARK(6);
        if (e > 0 && __any_sync(0xffffffffu, alpha != 1.0f)) {
          // O row *= alpha
          const float2 a2 = make_float2(alpha, alpha);
#pragma unroll
          for (int cq = 0; cq < DV / 32; ++cq) {
            const uint32_t ta = tmem + C::tO(x) + lane_base + 32 * cq;
            uint32_t rr[32];
            ptx::tmem_ld32(ta, rr);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float2 v = __fmul2_rn(make_float2(__uint_as_float(rr[2 * i]), __uint_as_float(rr[2 * i + 1])), a2);
              rr[2 * i] = __float_as_uint(v.x);
              rr[2 * i + 1] = __float_as_uint(v.y);
            }
            ptx::tmem_st32(ta, rr);
          }
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(p_full + x);
        PROF_MARK(7);
      }

      // ---- epilogue: O / l (attention.py:104-106), one row per thread (32x32b)
      const float my_l = l2.x + l2.y;
      const float inv_l = 1.0f / (my_l > 0.f ? my_l : 1.0f);
      if (plan.n > 0) {
        ptx::mbar_wait(o_done + x, (g - 1) & 1);
        ptx::tc_fence_after();
      }
      const uint32_t tO = tmem + C::tO(x) + lane_base;
      const int64_t orow = static_cast<int64_t>(my_bh) * p.lq + qrow;
#pragma unroll
      for (int c = 0; c < DV / 32; ++c) {
        uint32_t rr[32];
        if (plan.n > 0) {
          ptx::tmem_ld32(tO + 32 * c, rr);
          ptx::tmem_ld_wait();
        } else {
#pragma unroll
          for (int i2 = 0; i2 < 32; ++i2) rr[i2] = 0u;
        }
        if (qrow < p.lq) store_orow<DV>(p, orow, c, rr, inv_l);
      }
      ptx::tc_fence_before();
      PROF_MARK(8);
    }
    if (kTurns && x == 0) ptx::named_bar_sync(1, 256);  // consume B's last hand-over
    PROF_FLUSH(0, 10);
  } else {
    ptx::setmaxnreg_inc<216>();  // the 128-value S fragment stays in registers
    // =========================== softmax (one warpgroup per stream) ===========================
    // TMEM is read in the 16x256b shape: thread (r0 = lane/4, m = lane%4) of a warp
    // holds rows quad*32 + r0 + 8i (i = 0..3) and the 32 S columns 8g + 2m + b.
    // K rows are permuted inside every 128-key tile (quant.cuh, kPermKeys) so that
    // these 32 columns are exactly the keys 32g' + 8m + (0..7) whose E4M3 P bytes
    // form the P words this thread owns in the same shape: no shuffles for P,
    // and only 32 (not 128) S_q^K factors per thread per tile.
    const int x = warp >> 2;  // stream
    const int quad = warp & 3;
    const int m4 = lane & 3, r0 = lane >> 2;
    const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
    constexpr uint32_t kHalf = 16u << 16;  // lane offset of the second 16-lane block
    // Lazy rescaling (the FA4 trick): a row keeps its running max until a tile
    // raises it by more than kLazy (log2 units), so O is rarely rescaled.  P can
    // then reach 2^kLazy and is stored as E4M3(P * 2^(8 - kLazy)) <= 256 < 448.
    constexpr float kLazy = 4.f;
    constexpr float kPShift = 8.f - kLazy;
    uint32_t g = 0, sc = 0;                // this stream's tile ordinal / S_q^K ring counter
    if (kTurns && x == 1) ptx::named_bar_arrive(1, 256);  // A takes the first exp phase
    PROF_DECL

    for (uint32_t it = 0;; ++it) {
      const int ss = it % C::kNSch;
      ptx::mbar_wait(sch_full + ss, (it / C::kNSch) & 1);
      const int k = sched[ss];
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(sch_empty + ss);
      if (k < 0) break;
      int bh[2], qt;
      pair_coords(p, pp, k, bh[0], bh[1], qt);
      const int my_bh = bh[x];
      Plan plan;
      plan.init(qt, p.lq, p.lk, C::kBM, C::kBN, p.diag_window, p.sink_window, p.causal != 0);
      if (my_bh < 0) continue;  // odd head count: stream B idles on this pair
      const bool pair2 = bh[1] >= 0;
      const int q0 = qt * C::kBM;
      int qrow[4];
      float sq_q[4], m_run[4], l_run[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        qrow[i] = q0 + quad * 32 + r0 + 8 * i;
        sq_q[i] = (qrow[i] < p.lq) ? p.qs_q[static_cast<int64_t>(my_bh) * p.lq_pad + qrow[i]] : 1.0f;
        m_run[i] = -INFINITY;
        l_run[i] = 0.f;
      }

      for (int e = 0; e < plan.n; ++e, ++g) {
        int t;
        bool hi;
        plan.entry(e, t, hi);
        if (LOW == kLowHigh) hi = true;
        const bool two_level = hi || (LOW == kLowNV);
        const int k0 = t * C::kBN;
        PROF_MARK(9);
        ptx::mbar_wait(s_full + x, g & 1);
        ptx::tc_fence_after();
        PROF_MARK(0);
        // S fragment, loaded in place: s[64 (i / 2) + 4 g + 2 (i % 2) + b] = S[row i][col 8g + 2m + b]
        float s[128];
        ptx::tmem_ld_16x256b_x16(tmem + C::tS + lane_base, *reinterpret_cast<uint32_t(*)[64]>(&s[0]));
        ptx::tmem_ld_16x256b_x16(tmem + C::tS + lane_base + kHalf, *reinterpret_cast<uint32_t(*)[64]>(&s[64]));
        ptx::tmem_ld_wait();
#define SIDX(i, gg, b) (64 * ((i) >> 1) + 4 * (gg) + 2 * ((i) & 1) + (b))
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(s_free);  // S buffer may be overwritten by the next QK
        PROF_MARK(1);
        {
          const int sl = sc % C::kNS;
          ++sc;
          if (two_level) {
            // this thread's 32 factors are contiguous: [36 m + 2 g + b]
            const uint32_t sqk = ptx::smem_u32(smem + C::oSqK + (x * C::kNS + sl) * C::kSqkBytes) + 144 * m4;
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // factors for columns g = 2j, 2j + 1
              const float4 f = ptx::lds_f4(sqk + 16 * j);
              const float2 f0 = make_float2(f.x, f.y), f1 = make_float2(f.z, f.w);
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float2 a = __fmul2_rn(make_float2(s[SIDX(i, 2 * j, 0)], s[SIDX(i, 2 * j, 1)]), f0);
                const float2 b = __fmul2_rn(make_float2(s[SIDX(i, 2 * j + 1, 0)], s[SIDX(i, 2 * j + 1, 1)]), f1);
                s[SIDX(i, 2 * j, 0)] = a.x;
                s[SIDX(i, 2 * j, 1)] = a.y;
                s[SIDX(i, 2 * j + 1, 0)] = b.x;
                s[SIDX(i, 2 * j + 1, 1)] = b.y;
              }
            }
          }
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(sq_empty + x * C::kNS + sl);
        }
        PROF_MARK(2);
        // causal (attention.py:178-184, applied when k1-1 > q0, :306) and ragged-key masks;
        // column 8g + 2m + b holds key k0 + 32(g/4) + 8m + 2(g%4) + b
        const int kvalid = p.lk - k0;
        const bool need_causal = p.causal && (k0 + (kvalid < C::kBN ? kvalid : C::kBN) - 1 > q0);
        if (need_causal || kvalid < C::kBN) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int lim = need_causal ? min(qrow[i] - k0 + 1, kvalid) : kvalid;
#pragma unroll
            for (int gg = 0; gg < 16; ++gg)
#pragma unroll
              for (int b = 0; b < 2; ++b)
                if (32 * (gg >> 2) + 8 * m4 + 2 * (gg & 3) + b >= lim) s[SIDX(i, gg, b)] = -INFINITY;
          }
        }
        float rowf[4], bias[4], alpha[4];
        bool any_alpha = false;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float mx = fmaxf(s[SIDX(i, 0, 0)], s[SIDX(i, 0, 1)]);
#pragma unroll
          for (int gg = 1; gg < 16; ++gg) mx = ptx::fmax3(mx, s[SIDX(i, gg, 0)], s[SIDX(i, gg, 1)]);
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
          rowf[i] = two_level ? sq_q[i] : 1.0f;
          const float m_cand = fmaxf(m_run[i], mx * rowf[i]);
          const bool upd = m_cand > m_run[i] + kLazy;  // always for the first live tile (m_run = -inf)
          const float m_new = upd ? m_cand : m_run[i];
          const bool dead = (m_new == -INFINITY);
          alpha[i] = (dead || !upd) ? 1.0f : fast_exp2(m_run[i] - m_new);  // m_run = -inf -> 0
          bias[i] = dead ? 0.f : (kPShift - m_new);
          m_run[i] = m_new;
          any_alpha |= alpha[i] != 1.0f;
        }
        PROF_MARK(3);
        // P_x (and O_x) are read by PV(e-1): wait for it before overwriting
        if (e > 0) {
          ptx::mbar_wait(o_done + x, (g - 1) & 1);
          ptx::tc_fence_after();
        }
        PROF_MARK(4);
        // exp phases of the two streams alternate (A, B, A, B, ...): MUFU.EX2 is the
        // shared bottleneck; each stream's loads / max / O rescale run during the
        // other's exp phase (named barriers 1 = "A may exp", 2 = "B may exp")
        if (kTurns && pair2) ptx::named_bar_sync(1 + x, 256);
        PROF_MARK(5);
#pragma unroll
        for (int blk = 0; blk < 2; ++blk) {  // rows 2 blk, 2 blk + 1 (one 16-lane TMEM block)
          uint32_t pk[16];  // st.16x256b.x4: rep G -> {row 2blk: word 8G+2m, 8G+2m+1; row 2blk+1: same}
#pragma unroll
          for (int ii = 0; ii < 2; ++ii) {
            const int i = 2 * blk + ii;
            const float2 rf2 = make_float2(rowf[i], rowf[i]), b2 = make_float2(bias[i], bias[i]);
            float2 ls = make_float2(0.f, 0.f);
#pragma unroll
            for (int G = 0; G < 4; ++G) {
#pragma unroll
              for (int h = 0; h < 2; ++h) {  // word h of rep G = keys of columns g = 4G + 2h, 4G + 2h + 1
                const int gg = 4 * G + 2 * h;
                float2 x0 = __ffma2_rn(make_float2(s[SIDX(i, gg, 0)], s[SIDX(i, gg, 1)]), rf2, b2);
                float2 x1 = __ffma2_rn(make_float2(s[SIDX(i, gg + 1, 0)], s[SIDX(i, gg + 1, 1)]), rf2, b2);
                x0.x = fast_exp2(x0.x);
                x0.y = fast_exp2(x0.y);
                x1.x = fast_exp2(x1.x);
                x1.y = fast_exp2(x1.y);
                ls = __fadd2_rn(ls, __fadd2_rn(x0, x1));
                pk[4 * G + 2 * ii + h] = static_cast<uint32_t>(ptx::cvt_e4m3x2(x0.x, x0.y)) |
                                         (static_cast<uint32_t>(ptx::cvt_e4m3x2(x1.x, x1.y)) << 16);
              }
            }
            l_run[i] = fmaf(l_run[i], alpha[i], ls.x + ls.y);
          }
          ptx::tmem_st_16x256b_x4(tmem + C::tP(x) + lane_base + (blk ? kHalf : 0u), pk);
        }
#undef SIDX
        if (kTurns && pair2) ptx::named_bar_arrive(2 - x, 256);
        PROF_MARK(6);
        if (e > 0 && __any_sync(0xffffffffu, any_alpha)) {
          // O rows (same 16x256b ownership as S / P) *= alpha
#pragma unroll
          for (int blk = 0; blk < 2; ++blk) {
            const float2 a0 = make_float2(alpha[2 * blk], alpha[2 * blk]);
            const float2 a1 = make_float2(alpha[2 * blk + 1], alpha[2 * blk + 1]);
#pragma unroll
            for (int cq = 0; cq < DV / 32; ++cq) {
              const uint32_t ta = tmem + C::tO(x) + lane_base + (blk ? kHalf : 0u) + 32 * cq;
              uint32_t rr[16];
              ptx::tmem_ld_16x256b_x4(ta, rr);
              ptx::tmem_ld_wait();
#pragma unroll
              for (int G = 0; G < 4; ++G) {
                const float2 u = __fmul2_rn(make_float2(__uint_as_float(rr[4 * G]), __uint_as_float(rr[4 * G + 1])), a0);
                const float2 v = __fmul2_rn(make_float2(__uint_as_float(rr[4 * G + 2]), __uint_as_float(rr[4 * G + 3])), a1);
                rr[4 * G] = __float_as_uint(u.x);
                rr[4 * G + 1] = __float_as_uint(u.y);
                rr[4 * G + 2] = __float_as_uint(v.x);
                rr[4 * G + 3] = __float_as_uint(v.y);
              }
              ptx::tmem_st_16x256b_x4(ta, rr);
            }
          }
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(p_full + x);
        PROF_MARK(7);
      }

      // ---- epilogue: O / l (attention.py:104-106), one row per thread (32x32b)
      float my_l = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float l = l_run[i];
        l += __shfl_xor_sync(0xffffffffu, l, 1);
        l += __shfl_xor_sync(0xffffffffu, l, 2);
        const float v = __shfl_sync(0xffffffffu, l, 4 * (lane & 7));  // row (lane & 7) + 8 i
        if ((lane >> 3) == i) my_l = v;
      }
      const float inv_l = 1.0f / (my_l > 0.f ? my_l : 1.0f);
      if (plan.n > 0) {
        ptx::mbar_wait(o_done + x, (g - 1) & 1);
        ptx::tc_fence_after();
      }
      const int orow_q = q0 + quad * 32 + lane;
      const uint32_t tO = tmem + C::tO(x) + lane_base;
      const int64_t orow = static_cast<int64_t>(my_bh) * p.lq + orow_q;
#pragma unroll
      for (int c = 0; c < DV / 32; ++c) {
        uint32_t rr[32];
        if (plan.n > 0) {
          ptx::tmem_ld32(tO + 32 * c, rr);
          ptx::tmem_ld_wait();
        } else {
#pragma unroll
          for (int i2 = 0; i2 < 32; ++i2) rr[i2] = 0u;
        }
        if (orow_q < p.lq) store_orow<DV>(p, orow, c, rr, inv_l);
      }
      ptx::tc_fence_before();
      PROF_MARK(8);
    }
    if (kTurns && x == 0) ptx::named_bar_sync(1, 256);  // consume B's last hand-over
    PROF_FLUSH(0, 10);
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == kMma) ptx::tmem_dealloc<512>(tmem);
}

}  // namespace dma
