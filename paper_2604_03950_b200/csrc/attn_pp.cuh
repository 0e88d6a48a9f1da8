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
#include "quant.cuh"

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

// Optional event trace of CTA 0 (-DDMA_TRACE): clock64 << 8 | event per role
// (0/1 softmax stream A/B, 2 MMA issuer, 3 producer; attn_sk.cuh: 0/1 WG0/WG1, 2 QK, 3 PV,
// 4 K producer, 5 V producer), read back with dma_trace_read.
#ifdef DMA_TRACE
__device__ unsigned long long g_trace[6][4096];
__device__ unsigned int g_trace_n[6];
// the event index lives in a register (trace_i, declared by TRACE_DECL in each role);
// stores are fire-and-forget, so a trace point costs a few issue slots
#define TRACE_DECL unsigned int trace_i = 0;
#define TRACE(cond, role, ev)                                                                 \
  do {                                                                                        \
    if ((cond) && blockIdx.x == 0 && (threadIdx.x & 31) == 0 && trace_i < 4096) {             \
      g_trace[role][trace_i] = (static_cast<unsigned long long>(clock64()) << 8) | (ev);      \
      g_trace_n[role] = ++trace_i;                                                            \
    }                                                                                         \
  } while (0)
#else
#define TRACE_DECL
#define TRACE(cond, role, ev) do {} while (0)
#endif

#ifndef DMA_PP_POLY
#define DMA_PP_POLY 0
#endif
// pairs (out of every 4) of the softmax exponentials computed by the degree-4 FMA-pipe
// polynomial (exp2_poly2) instead of MUFU.EX2
constexpr int kPolyPP = DMA_PP_POLY;

#ifndef DMA_PP_MAXCH8
#define DMA_PP_MAXCH8 0
#endif
#ifndef DMA_PP_LATE_PV_WAIT
#define DMA_PP_LATE_PV_WAIT 0
#endif
#ifndef DMA_PP_SPLIT_PV
#define DMA_PP_SPLIT_PV 0
#endif
// 1: PVs are issued by one warp per stream (kMma + 1 + x); the kMma warp issues only QKs
constexpr bool kSplitPV = DMA_PP_SPLIT_PV != 0;

#ifndef DMA_PP_HALF_FREE
#define DMA_PP_HALF_FREE 0
#endif
// 1: the S buffer is handed over per 64-column half (s_free[0] / s_free[1]); the next
// QK is issued as two N = 64 halves, the first overlapping the consumer's second-half load
constexpr bool kHalfFree = DMA_PP_HALF_FREE != 0;

#ifndef DMA_PP_PV_LATE
#define DMA_PP_PV_LATE 0
#endif
// 1: MMA issue order QK_A(e+1) PV_B(e-1) PV_A(e) QK_B(e+1) instead of QK_A(e+1) PV_A(e) QK_B(e+1) PV_B(e)
constexpr bool kPvLate = DMA_PP_PV_LATE != 0;

#ifndef DMA_FUSE_Q_PROLOGUE
#define DMA_FUSE_Q_PROLOGUE 5
#endif
// eighths of the Q tiles quantized by all warps before the attention starts (fused kernel)
constexpr int kFuseQPrologue = DMA_FUSE_Q_PROLOGUE;

#ifndef DMA_PP_EARLY_SF
#define DMA_PP_EARLY_SF 0
#endif
// 1: the QK's scale-factor copies (and the K-tile wait) are issued before the S hand-over wait
constexpr bool kEarlySF = DMA_PP_EARLY_SF != 0;

#ifndef DMA_PP_EARLY_FREE
#define DMA_PP_EARLY_FREE 0
#endif

#ifndef DMA_PP_TURNS
#define DMA_PP_TURNS 0
#endif
// 1: the two softmax warpgroups take strict turns for their exp2 phases
constexpr bool kTurns = DMA_PP_TURNS != 0;
#ifndef DMA_PP_SPLIT
#define DMA_PP_SPLIT 1
#endif
// softmax warpgroups per stream: 1 = a thread owns a whole S row (128 columns);
// 2 = two warps share each row, one key half each (4 softmax warps per SM sub-partition)
constexpr int kSplit = DMA_PP_SPLIT;

#ifndef DMA_PP_PSMEM
#define DMA_PP_PSMEM 0
#endif
// 1: P goes through shared memory (E4M3, 128B-swizzled K-major, the PV MMA's A operand from
// smem), double-buffered per stream, so a stream writes P(j) while PV(j-1) still reads P(j-1)
// (no PV wait on the softmax chain).  Pays for the 64 KB with one Q slot per stream and a
// 3-stage K ring.
constexpr bool kPSmem = DMA_PP_PSMEM != 0 && kSplit == 1 && !kSplitPV;


struct PPParams {
  int n_pairs;
  int pairs_per_qt;
  int head_major;
  int group_pairs;       // head_major: head pairs per group (their K/V share L2), walked longest-first
  unsigned int* ticket;  // [0] next work item, [1] CTAs done (self-resetting)
  // KV splits (small problems: fewer pairs than SMs).  Work item k = pair k / n_split, split
  // k % n_split: a contiguous range of the pair's plan entries (item_range).  A split writes
  // its unnormalised O rows with (m, l) to `part`; kv_combine_kernel merges the splits
  // (flash-decoding style) and stores O.  n_split = 1: one item per pair.
  int n_split;
  int n_items;               // n_pairs * n_split (ticket bound)
  float* part;               // [n_bh][n_qt][n_split][128 rows][DV + 4] f32: O row, (m, l), padding
};

// Plan entries [e0, e1) of split s of a pair whose plan has n entries: ns = min(n_split, n)
// splits (at least 1) of near-equal length; s >= ns is an empty item (skipped by every role).
// ns = 1 is the unsplit path (a pair with an empty plan still writes its zero rows).
struct ItemRange {
  int e0, e1, ns;
  bool skip;
};
template <bool SPLIT>
__device__ __forceinline__ ItemRange item_range(const PPParams& q, const Plan& plan, int s) {
  ItemRange r;
  if (!SPLIT) {  // one item per pair: compile-time constants, the unsplit kernel is unchanged
    r.e0 = 0;
    r.e1 = plan.n;
    r.ns = 1;
    r.skip = false;
    return r;
  }
  r.ns = q.n_split < plan.n ? q.n_split : plan.n;
  if (r.ns < 1) r.ns = 1;
  r.skip = s >= r.ns;
  r.e0 = r.skip ? 0 : static_cast<int>(static_cast<int64_t>(s) * plan.n / r.ns);
  r.e1 = r.skip ? 0 : static_cast<int>(static_cast<int64_t>(s + 1) * plan.n / r.ns);
  return r;
}

// Fused phase 1 (FUSE instantiations, bf16 inputs, TOKEN granularity): warps 10 / 11 of
// every CTA quantize K + V tiles / Q tiles of the raw inputs into the operand layouts
// (the same q16_item / qv4_block code as quant16_kernel / quant_v4_bf16_kernel, so the codes
// are bit-identical), in the order the attention consumes them, and publish each 128-row
// tile with a ready flag (generic stores -> fence.proxy.async.global -> release store); the
// TMA producer acquires the flag before it loads the tile.  Flags and counters live in the
// workspace's small region, zeroed by the per-call memset.
struct FuseParams {
  const __nv_bfloat16* q;
  const __nv_bfloat16* k;
  const __nv_bfloat16* v;
  QuantOut out_q, out_k;     // as phase 1 (K: permuted operand rows, key_perm = 1)
  uint8_t* v_codes;          // [mk][lk_pad][DV] E4M3
  uint8_t* sf_v;             // V scale-factor atoms
  double c;                  // softmax prescale log2(e) / sqrt(D) (quantize.py:92-95)
  unsigned int* flags;       // [mq * rt_q] Q | [mk * rt_k] K | [mk * rt_k] V tile ready (0 / 1)
  unsigned int* counters;    // [0] next K/V item, [1] next Q item
  int e5;                    // high format E5M2
};

__device__ __forceinline__ void fuse_publish(unsigned int* flag, int lane) {
  ptx::fence_proxy_async_global();  // this lane's generic stores -> visible to the async proxy (TMA)
  __syncwarp();
  if (lane == 0) {
    __threadfence();
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(1u) : "memory");
  }
}

// One 128-row tile of bf16 Q or K quantized by one warp (fused kernel): tpr = D / 16 lanes per
// row (q16_item_fast), 32 / tpr rows per pass, input bytes prefetched four passes ahead.  Out
// of line: one copy of the quantizer code next to the attention code (instruction cache).
template <int D, bool NV, bool E5>
__device__ __forceinline__ void fuse_quant_tile(const __nv_bfloat16* __restrict__ x, int64_t rows, int64_t mat, int t,
                                             int is_query, double c, const QuantOut& out, int lane) {
  constexpr int tpr = D / 16, rpp = 32 / tpr;
  const int part = lane & (tpr - 1), rsub = lane / tpr;
  const int64_t mstride = rows * D;
  constexpr int kPasses = 128 / rpp, kPf = 4;
  uint4 pf[kPf][2];
  auto fetch = [&](int ps, uint4 (&dst)[2]) {
    const int64_t r = static_cast<int64_t>(t) * 128 + ps * rpp + rsub;
    if (ps < kPasses && r < rows) {
      const uint4* src = reinterpret_cast<const uint4*>(x + mat * mstride + r * D + part * 16);
      dst[0] = __ldg(src);
      dst[1] = __ldg(src + 1);
    } else {
      dst[0] = dst[1] = make_uint4(0u, 0u, 0u, 0u);
    }
  };
#pragma unroll
  for (int i = 0; i < kPf; ++i) fetch(i, pf[i]);
  for (int p0 = 0; p0 < kPasses; p0 += kPf) {
#pragma unroll
    for (int i = 0; i < kPf; ++i) {
      const int ps = p0 + i;
      const uint4 cur0 = pf[i][0], cur1 = pf[i][1];
      fetch(ps + kPf, pf[i]);
      const int64_t row = static_cast<int64_t>(t) * 128 + ps * rpp + rsub;
      const bool live = row < rows;
      if (!__all_sync(0xffffffffu, !live))
        q16_item_fast<__nv_bfloat16, NV, E5, DMA_GRAN_TOKEN>(x, mstride, D, mat, rows, D, row, live, part, tpr, lane,
                                                              cur0, cur1, is_query, c, nullptr, out);
    }
  }
}

__device__ __forceinline__ float ld_acquire_f32(const float* ptr) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ptr) : "memory");
  return __uint_as_float(v);
}

__device__ __forceinline__ void fuse_acquire(const unsigned int* flag) {
  uint32_t v;
  for (;;) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (v) break;
    __nanosleep(64);
  }
  ptx::fence_proxy_async_global();
}

template <int D, int DV, int LOW>
struct PPCfg {
  static constexpr int kBM = 128, kBN = 128;
  static constexpr int kNK = (kSplit == 2 || kPSmem) ? 3 : 4, kNV = 3, kNS = 4, kNSch = 4;
  static constexpr int kNQ = kPSmem ? 1 : 2;  // Q slots (pairs in flight)
  static constexpr int kPBytes = 128 * 128;   // one P tile: 128 rows x 128 keys, E4M3
  static constexpr int kSoftWarps = 8 * kSplit;        // softmax warps (2 streams x kSplit warpgroups)
  static constexpr int kThreads = 32 * (kSoftWarps + 4);  // + producer, MMA issuer, 2 idle
  // setmaxnreg budgets: softmax warpgroups grow, the producer/MMA warpgroup shrinks.  The
  // CTA's register pool is what the launch allocated (kThreads x the launch-bound count,
  // 168 / 96), so 2 x 128 x 216 + 128 x 72 <= 384 x 168 and 4 x 128 x 104 + 128 x 64 <= 640 x 96.
  static constexpr int kRegSoft = kSplit == 1 ? 216 : 104;
  static constexpr int kRegCtl = kSplit == 1 ? 72 : 64;
  static_assert(kSoftWarps * 32 * kRegSoft + 128 * kRegCtl <= kThreads * (kSplit == 1 ? 168 : 96), "register pool");
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
  static constexpr int oQ = 0;                                // [kNQ slot][2 stream][kQStream]
  static constexpr int oK = oQ + 2 * kNQ * kQStream;          // [kNK][kKBytes]
  static constexpr int oV = oK + kNK * kKBytes;               // [kNV][kVBytes]
  static constexpr int oP = oV + kNV * kVBytes;               // kPSmem: [2 stream][2 buf][kPBytes]
  static constexpr int oSfQ = oP + (kPSmem ? 4 * kPBytes : 0);  // [kNQ slot][2 stream][kSfQ]
  static constexpr int oSfK = oSfQ + 2 * kNQ * kSfQ;          // [kNK][kChK][512]
  static constexpr int oSfV = oSfK + kNK * kChK * 512;        // [kNV][512]
  static constexpr int kSqkBytes = 4 * kSqkTile;              // 576: S_q^K of one tile, bank-padded
  static constexpr int oSqK = oSfV + kNV * 512;               // [2 stream][kNS][kSqkBytes]
  static constexpr int oSfP = oSqK + 2 * kNS * kSqkBytes;     // 512
  static constexpr int oSch = oSfP + 512;                     // [kNSch] int
  static constexpr int oRed = oSch + 128;                     // [2 parity][2 stream][2 half][128] f32 row maxima, then l
  static constexpr int kItmSlot = 16;                         // sched[16 + warp]: a softmax warp's current item
  static constexpr int oBar = oRed + (kSplit == 2 ? 2 * 4096 : 0);
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
    // groups of group_pairs head pairs (K/V of a group fit in L2 with the others' traffic);
    // inside a group, query-tile rank major: the longest tiles of all its pairs go first, so
    // a group's long items never start at the very end of the launch (tail)
    const int gsz = q.group_pairs * p.n_qt;
    const int grp = k / gsz;
    const int kin = k - grp * gsz;
    const int g0 = grp * q.group_pairs;
    const int gn = q.pairs_per_qt - g0 < q.group_pairs ? q.pairs_per_qt - g0 : q.group_pairs;
    r = kin / gn;
    hp = g0 + (kin - r * gn);
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


// exp2 / E4M3 pack as volatile asm: the softmax orders them explicitly (software pipelining)
// (pipe experiments, WRONG results: -DDMA_EXP_NOMUFU replaces ex2 by an FMA-pipe multiply,
// -DDMA_EXP_NOCVT the E4M3 pack by an ALU shift/or -- to see which pipe bounds the softmax)
__device__ __forceinline__ float exp2_ordered(float x) {
  float y;
#ifdef DMA_EXP_NOMUFU
  asm volatile("mul.rn.f32 %0, %1, 0f3F000000;" : "=f"(y) : "f"(x));
#else
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
#endif
  return y;
}
#ifndef DMA_PP_EXP_INTERLEAVE
#define DMA_PP_EXP_INTERLEAVE 0
#endif
// 1: the exp arguments' FFMA2 is issued inside the software-pipelined MUFU loop
constexpr bool kExpInterleave = DMA_PP_EXP_INTERLEAVE != 0;
__device__ __forceinline__ float2 ffma2_ordered(float2 a, float2 b, float2 c) {
  float2 d;
  asm volatile(
      "{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ uint32_t cvt_e4m3x2_ordered(float lo, float hi) {
#ifdef DMA_EXP_NOCVT
  uint32_t r;
  asm volatile("{\n\t.reg .b32 t;\n\tshr.b32 t, %1, 24;\n\tshf.l.wrap.b32 %0, %2, t, 8;\n\t}" : "=r"(r) : "r"(__float_as_uint(lo)), "r"(__float_as_uint(hi)));
  return r & 0xFFFFu;
#else
  uint16_t r;
  asm volatile("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
#endif
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

template <int D, int DV, int LOW, bool FUSE, bool SPLIT>
__global__ void __launch_bounds__(PPCfg<D, DV, LOW>::kThreads, 1) dma_attn_pp_kernel(const __grid_constant__ AttnParams p,
                                                             const __grid_constant__ PPParams pp,
                                                             const __grid_constant__ FuseParams fz) {
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
  uint64_t* s_free = sq_empty + 2 * C::kNS;       // [2] S columns [0,64) / [64,128) copied out
  uint64_t* s_full = s_free + 2;                  // [2]
  uint64_t* p_full = s_full + 2;                  // [2 stream][2 buf] (kPSmem: per P buffer)
  uint64_t* o_done = p_full + 4;                  // [2 stream][2 buf]
  uint64_t* sch_full = o_done + 4;                // [kNSch]
  uint64_t* sch_empty = sch_full + C::kNSch;      // [kNSch]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sch_empty + C::kNSch);
  int* sched = reinterpret_cast<int*>(smem + C::oSch);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rt_q = p.lq_pad >> 7, rt_k = p.lk_pad >> 7;

  constexpr int kProducer = C::kSoftWarps, kMma = C::kSoftWarps + 1;  // warps below: softmax
  if (warp == kProducer) {
    if (lane == 0) {
      for (int i = 0; i < 2; ++i) {
        ptx::mbar_init(q_full + i, 1);
        ptx::mbar_init(q_empty + i, 1);
        ptx::mbar_init(s_full + i, 1);
        ptx::mbar_init(p_full + i, 4 * kSplit);
        ptx::mbar_init(o_done + i, 1);
        ptx::mbar_init(p_full + 2 + i, 4 * kSplit);
        ptx::mbar_init(o_done + 2 + i, 1);
      }
      for (int i = 0; i < C::kNK; ++i) {
        ptx::mbar_init(k_full + i, 1);
        ptx::mbar_init(k_empty + i, 1);
      }
      for (int i = 0; i < C::kNV; ++i) {
        ptx::mbar_init(v_full + i, 1);
        ptx::mbar_init(v_empty + i, kSplitPV ? 2 : 1);
      }
      for (int i = 0; i < 2 * C::kNS; ++i) ptx::mbar_init(sq_empty + i, 4 * kSplit);
      ptx::mbar_init(s_free, kHalfFree ? 4 : 4 * kSplit);
      ptx::mbar_init(s_free + 1, kHalfFree ? 4 : 4 * kSplit);
      for (int i = 0; i < C::kNSch; ++i) {
        ptx::mbar_init(sch_full + i, 1);
        ptx::mbar_init(sch_empty + i, (kSplitPV ? 3 : 1) + C::kSoftWarps);
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
  ptx::pdl_wait();  // phase-1 outputs visible (PDL launch: the prologue above overlapped phase 1)
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // Fused phase 1 (FUSE): one quantizer work queue -- K and V tiles (kv_role; kv-head major
  // for head-major pair order, tile major otherwise) or Q tiles in the pair order.  One warp
  // per 128-row tile (fuse_quant_tile / qv4_block), each tile published by its ready flag.
  // items [first, last) of the queue, handed out by counters[ctr] (0: K/V, 1: the Q items the
  // Q warps take, 2: the Q items of the prologue); a taken item is always processed
  auto fuse_quant_loop = [&](bool kv_role, int ctr, int64_t first, int64_t last) {
      const int mq = p.n_bh, mkn = p.n_bh / p.group;
      const int64_t n_all = kv_role ? 2ll * mkn * rt_k : 2ll * pp.n_pairs;
      const int64_t n_items = last < n_all ? last : n_all;
      auto quant_tile = [&](const __nv_bfloat16* x, int64_t rows, int64_t mat, int t, int is_query, const QuantOut& out) {
        if (fz.e5)
          fuse_quant_tile<D, LOW != kLowMX4, true>(x, rows, mat, t, is_query, fz.c, out, lane);
        else
          fuse_quant_tile<D, LOW != kLowMX4, false>(x, rows, mat, t, is_query, fz.c, out, lane);
      };
      for (;;) {
        unsigned int it = 0;
        if (lane == 0) it = static_cast<unsigned int>(first) + atomicAdd(fz.counters + ctr, 1u);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (static_cast<int64_t>(it) >= n_items) break;
        if (kv_role) {
          const int kind = static_cast<int>(it & 1);  // 0 = K, 1 = V of the same tile
          const int u = static_cast<int>(it >> 1);
          int m, t;
          if (pp.head_major) {
            m = u / rt_k;
            t = u - m * rt_k;
          } else {
            t = u / mkn;
            m = u - t * mkn;
          }
          if (kind == 0) {
            quant_tile(fz.k, p.lk, m, t, 0, fz.out_k);
            fuse_publish(fz.flags + static_cast<int64_t>(mq) * rt_q + static_cast<int64_t>(m) * rt_k + t, lane);
          } else {
            // V: 4 key blocks of 32, DV / 4 lanes per block (qv4_block: 4 value columns per lane)
            constexpr int tpb = DV / 4, bpp = 32 / tpb;
            for (int kb = lane / tpb; kb < 4; kb += bpp)
              qv4_block(fz.v, p.lk, DV, p.lk_pad, fz.v_codes, fz.sf_v, m, static_cast<int64_t>(t) * 4 + kb,
                        (lane % tpb) * 4);
            fuse_publish(fz.flags + static_cast<int64_t>(mq) * rt_q + static_cast<int64_t>(mkn + m) * rt_k + t, lane);
          }
        } else {
          int bh[2], qt;
          pair_coords(p, pp, static_cast<int>(it >> 1), bh[0], bh[1], qt);
          const int b = bh[it & 1];
          if (b < 0) continue;
          quant_tile(fz.q, p.lq, b, qt, 1, fz.out_q);
          fuse_publish(fz.flags + static_cast<int64_t>(b) * rt_q + qt, lane);
        }
      }
  };
  // prologue: every warp but the two quantizer warps drains the K / V queue first (the
  // attention needs all K / V tiles of its first heads at once); warps 10 / 11 quantize Q in
  // the pair order, overlapped with the attention
  const int64_t fuse_q_pro = 2ll * pp.n_pairs * kFuseQPrologue / 8;  // Q items of the prologue
  if (FUSE && warp != kMma + 1 && warp != kMma + 2) {
    fuse_quant_loop(true, 0, 0, INT64_MAX);
    // then the first kFuseQPrologue / 8 of the Q queue (the two Q warps alone cannot keep up
    // with the attention on short pairs); the Q warps take the rest
    fuse_quant_loop(false, 2, 0, fuse_q_pro);
  }

  if (warp >= C::kSoftWarps) {
  // register budget: the last warpgroup gives registers to the softmax warpgroups (not when
  // warps 10 / 11 quantize: the quantizer needs its registers; ptxas compiles every role at
  // the launch bound anyway)
  if (!FUSE) ptx::setmaxnreg_dec<C::kRegCtl>();
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
      const int k = tk < static_cast<unsigned int>(pp.n_items) ? static_cast<int>(tk) : -1;
      if (lane == 0) {
        sched[ss] = k;
        ptx::mbar_arrive(sch_full + ss);  // release: the slot write is visible to waiters
      }
      __syncwarp();
      if (k < 0) break;
      int bh[2], qt;
      pair_coords(p, pp, SPLIT ? k / pp.n_split : k, bh[0], bh[1], qt);
      Plan plan;
      plan.init(qt, p.lq, p.lk, C::kBM, C::kBN, p.diag_window, p.sink_window, p.causal != 0);
      const ItemRange ir = item_range<SPLIT>(pp, plan, SPLIT ? k % pp.n_split : 0);
      if (ir.e0 >= ir.e1) continue;
      const int ns = bh[1] >= 0 ? 2 : 1;
      const int mk[2] = {mat_k_of(p, bh[0]), ns == 2 ? mat_k_of(p, bh[1]) : -1};
      const bool shared_kv = ns == 2 && mk[0] == mk[1];
      // ---- Q (both streams) into the pair's slot
      const int qs = static_cast<int>(po % C::kNQ);
      PROF_MARK(0);
      ptx::mbar_wait(q_empty + qs, ((po / C::kNQ) & 1) ^ 1);
      PROF_MARK(2);
      ++po;
      uint32_t qbytes = C::kQHiBytes + 512 * C::kChHi;
      if (LOW != kLowHigh) qbytes += C::kQLoBytes + 512 * C::kChLo;
      if (FUSE)
        for (int x = 0; x < ns; ++x) fuse_acquire(fz.flags + static_cast<int64_t>(bh[x]) * rt_q + qt);
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
      for (int e = ir.e0; e < ir.e1; ++e) {
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
          if (FUSE) fuse_acquire(fz.flags + static_cast<int64_t>(p.n_bh) * rt_q + static_cast<int64_t>(mk[x]) * rt_k + t);
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
          if (FUSE)
            fuse_acquire(fz.flags + static_cast<int64_t>(p.n_bh) * rt_q +
                         static_cast<int64_t>(p.n_bh / p.group + mk[x]) * rt_k + t);
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
    TRACE_DECL
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
      pair_coords(p, pp, SPLIT ? k / pp.n_split : k, bh[0], bh[1], qt);
      Plan plan;
      plan.init(qt, p.lq, p.lk, C::kBM, C::kBN, p.diag_window, p.sink_window, p.causal != 0);
      const ItemRange ir = item_range<SPLIT>(pp, plan, SPLIT ? k % pp.n_split : 0);
      if (ir.e0 >= ir.e1) continue;
      const int ns = bh[1] >= 0 ? 2 : 1;
      const bool shared_kv = ns == 2 && mat_k_of(p, bh[0]) == mat_k_of(p, bh[1]);
      const int qs = static_cast<int>(po % C::kNQ);
      PROF_MARK(0);
      ptx::mbar_wait(q_full + qs, (po / C::kNQ) & 1);
      PROF_MARK(2);
      ++po;
      ptx::tc_fence_after();
      uint32_t kslot[2] = {0, 0}, vslot[2] = {0, 0};

      auto issue_qk = [&](int x, int e) {
        int t;
        bool hi;
        plan.entry(e, t, hi);
        if (LOW == kLowHigh) hi = true;
        // the single S buffer: wait until its previous user copied it out.  With
        // DMA_PP_EARLY_SF the scale-factor copies of this QK go first (off the S hand-over
        // path): their TMEM slots were last read by this stream's previous QK, which had
        // completed before the MMA warp passed the other stream's last s_free wait
        const uint32_t sfp = (su & 1) ^ 1;
        auto wait_s_free = [&]() {
          TRACE(true, 2, 26 + x);
          PROF_MARK(0);
          ptx::mbar_wait(s_free, sfp);
          PROF_MARK(3);
          TRACE(true, 2, 10 + x);
          ++su;
          ptx::tc_fence_after();
        };
        if (!kEarlySF) wait_s_free();
        const uint32_t oq = C::oQ + (qs * 2 + x) * C::kQStream;
        if (e == ir.e0) {
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
          TRACE(true, 2, 18 + x);
          if (++ks == C::kNK) { ks = 0; kph ^= 1; }
          ptx::tc_fence_after();
        } else {
          kslot[1] = kslot[0];
        }
        const uint32_t kslt = kslot[x];
        const int ch = hi ? C::kChHi : C::kChLo;
        PROF_MARK(0);
#ifndef DMA_EXP_NOSFK
        for (int j = 0; j < ch; ++j)
          ptx::wu::tc_cp_sf(tmem + C::tSfK(x) + 4 * j, sf_desc(C::oSfK + kslt * 512 * C::kChK + 512 * j));
#endif
        PROF_MARK(7);
        if (kEarlySF) wait_s_free();
        TRACE(true, 2, 20 + x);
        const uint32_t tsfq = tmem + C::tSfQ(x), tsfk0 = tmem + C::tSfK(x);
        // one N = 128 QK, or two N = 64 halves (kHalfFree: the second waits for s_free[1]);
        // the K scale factors of key rows 64h.. are the atom's words 2h, 2h + 1
        constexpr int kNH = kHalfFree ? 2 : 1, kN = 128 / kNH;
#pragma unroll
        for (int hh = 0; hh < kNH; ++hh) {
          if (hh == 1) {
            ptx::mbar_wait(s_free + 1, sfp);
            ptx::tc_fence_after();
          }
          const uint32_t tSd = tmem + C::tS + kN * hh, tsfk = tsfk0 + 2 * hh;
          if (hi) {
            constexpr int rb = D;
            const uint32_t kaddr = sbase + C::oK + kslt * C::kKBytes + hh * (kN * rb);
            const uint64_t dh = static_cast<uint64_t>(ptx::desc_hi(8 * rb, swz_mode(rb))) << 32;
#pragma unroll
            for (int kk = 0; kk < D / 32; ++kk) {
              const uint64_t ad = dh | ptx::desc_lo(sbase + oq + 32 * kk, 16);
              const uint64_t bd = dh | ptx::desc_lo(kaddr + 32 * kk, 16);
              const uint32_t id = ptx::idesc_bs(hf, hf, 0, 0, 128, kN, 1, kk & 3, kk & 3);
              ptx::wu::mma_mxf8f6f4(tSd, ad, bd, id, tsfq + 4 * (kk >> 2), tsfk + 4 * (kk >> 2), kk > 0);
            }
          } else {
            constexpr int rb = D / 2;
            const uint32_t kaddr = sbase + C::oK + kslt * C::kKBytes + hh * (kN * rb);
            const uint64_t dh = static_cast<uint64_t>(ptx::desc_hi(8 * rb, swz_mode(rb))) << 32;
#pragma unroll
            for (int kk = 0; kk < D / 64; ++kk) {
              const uint64_t ad = dh | ptx::desc_lo(sbase + oq + C::kQHiBytes + 32 * kk, 16);
              const uint64_t bd = dh | ptx::desc_lo(kaddr + 32 * kk, 16);
              if (LOW == kLowNV) {
                const uint32_t id = ptx::idesc_bs(1, 1, 0, 0, 128, kN, 0, 0, 0);
                ptx::wu::mma_nvf4(tSd, ad, bd, id, tsfq + 4 + 4 * kk, tsfk + 4 * kk, kk > 0);
              } else {
                const uint32_t sid = (kk & 1) * 2;
                const uint32_t id = ptx::idesc_bs(1, 1, 0, 0, 128, kN, 1, sid, sid);
                ptx::wu::mma_mxf4(tSd, ad, bd, id, tsfq + 4 + 4 * (kk >> 1), tsfk + 4 * (kk >> 1), kk > 0);
              }
            }
          }
        }
        PROF_MARK(8);
        TRACE(true, 2, 12 + x);
        if (x == ns - 1 || !shared_kv) ptx::wu::tc_commit(k_empty + kslt);  // last reader of this K slot
        ptx::wu::tc_commit(s_full + x);
        if (e == ir.e1 - 1 && x == ns - 1) ptx::wu::tc_commit(q_empty + qs);  // Q slot free after these
        TRACE(true, 2, 28 + x);
        PROF_MARK(9);
      };

      auto issue_pv = [&](int x, int e) {
        PROF_MARK(0);
        // kPSmem: P buffer pb of stream x (its PV count parity), barrier slot per buffer
        const uint32_t pb = kPSmem ? (pvc[x] & 1) : 0u;
        if (kPSmem)
          ptx::mbar_wait(p_full + 2 * x + pb, (pvc[x] >> 1) & 1);
        else
          ptx::mbar_wait(p_full + x, pvc[x] & 1);
        PROF_MARK(5);
        TRACE(true, 2, 14 + x);
        ++pvc[x];
        ptx::tc_fence_after();
        if (x == 0 || !shared_kv) {
          vslot[x] = vs;
          PROF_MARK(0);
          ptx::mbar_wait(v_full + vs, vph);
          PROF_MARK(6);
          TRACE(true, 2, 22 + x);
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
        if (kPSmem) {
          // A = P from shared memory: 128 rows x 128 B, K-major, 128B swizzle (as the Q operand)
          const uint32_t paddr = sbase + C::oP + (2 * x + pb) * C::kPBytes;
          const uint64_t dhp = static_cast<uint64_t>(ptx::desc_hi(8 * 128, swz_mode(128))) << 32;
#pragma unroll
          for (int kk = 0; kk < C::kBN / 32; ++kk) {
            const uint64_t ad = dhp | ptx::desc_lo(paddr + 32 * kk, 16);
            const uint64_t bd = dh | ptx::desc_lo(vaddr + kk * 32 * rb, 16);
            const uint32_t id = ptx::idesc_bs(0, 0, 0, 1, 128, DV, 1, kk & 3, kk & 3);
            ptx::wu::mma_mxf8f6f4(tmem + C::tO(x), ad, bd, id, tmem + C::tSfP, tmem + C::tSfV(x), !(e == ir.e0 && kk == 0));
          }
        } else {
#pragma unroll
        for (int kk = 0; kk < C::kBN / 32; ++kk) {
          const uint64_t bd = dh | ptx::desc_lo(vaddr + kk * 32 * rb, 16);
          const uint32_t id = ptx::idesc_bs(0, 0, 0, 1, 128, DV, 1, kk & 3, kk & 3);
          ptx::wu::mma_mxf8f6f4_ts(tmem + C::tO(x), tmem + C::tP(x) + 8 * kk, bd, id, tmem + C::tSfP,
                                   tmem + C::tSfV(x), !(e == ir.e0 && kk == 0));
        }
        }
        PROF_MARK(8);
        TRACE(true, 2, 16 + x);
        if (x == ns - 1 || !shared_kv) ptx::wu::tc_commit(v_empty + vslt);
        ptx::wu::tc_commit(o_done + (kPSmem ? 2 * x + pb : x));
        TRACE(true, 2, 24 + x);
        PROF_MARK(9);
      };

      if (kSplitPV) {
        for (int e = ir.e0; e < ir.e1; ++e) {
          issue_qk(0, e);
          if (ns == 2) issue_qk(1, e);
        }
      } else {
      issue_qk(0, ir.e0);
      if (ns == 2) issue_qk(1, ir.e0);
      if (kPvLate) {
        // stream B's PV(e - 1) after QK_A(e + 1): the QK that gates the S hand-over is not
        // queued behind four PV MMAs (measured slower with one P buffer per stream; with
        // kPSmem the PV is off the softmax chain)
        for (int e = ir.e0; e < ir.e1; ++e) {
          if (e + 1 < ir.e1) issue_qk(0, e + 1);
          if (ns == 2 && e > ir.e0) issue_pv(1, e - 1);
          issue_pv(0, e);
          if (ns == 2 && e + 1 < ir.e1) issue_qk(1, e + 1);
        }
        if (ns == 2) issue_pv(1, ir.e1 - 1);
      } else {
      for (int e = ir.e0; e < ir.e1; ++e) {
        if (e + 1 < ir.e1) issue_qk(0, e + 1);
        issue_pv(0, e);
        if (ns == 2) {
          if (e + 1 < ir.e1) issue_qk(1, e + 1);
          issue_pv(1, e);
        }
      }
      }
      }
    }
    PROF_MARK(0);
    PROF_FLUSH(10, 10);
  } else if (FUSE && (warp == kMma + 1 || warp == kMma + 2)) {
    // =========================== fused phase 1: Q quantizer warps ===========================
    fuse_quant_loop(false, 1, fuse_q_pro, INT64_MAX);
  } else if (kSplitPV && (warp == kMma + 1 || warp == kMma + 2)) {
    // =========================== PV issuers (kSplitPV): warp kMma + 1 + x issues stream x's PVs ===========================
    // PV_x(e) depends only on P_x(e) and V, so it must not queue behind QK_x(e + 1), which
    // waits for the other stream to release the shared S buffer.  V slots follow the
    // producer's ring order; a slot is released by 2 arrivals (one commit per reading
    // stream, or two from the only reader).
    const int x = warp - (kMma + 1);
    const uint64_t sf_desc_hi = static_cast<uint64_t>(ptx::desc_hi(128, ptx::kSwNone)) << 32;
    auto sf_desc = [&](uint32_t off) { return sf_desc_hi | ptx::desc_lo(sbase + off, 0); };
    const uint32_t tsfp = tmem + C::tSfP + 4u * x, tsfv = tmem + C::tSfV(x), tO = tmem + C::tO(x);
    ptx::wu::tc_cp_sf(tsfp, sf_desc(C::oSfP));
    uint32_t vc = 0, pvc = 0;
    for (uint32_t i = 0;; ++i) {
      const int ss = i % C::kNSch;
      ptx::mbar_wait(sch_full + ss, (i / C::kNSch) & 1);
      const int k = sched[ss];
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(sch_empty + ss);
      if (k < 0) break;
      int bh0, bh1, qt;
      pair_coords(p, pp, SPLIT ? k / pp.n_split : k, bh0, bh1, qt);
      Plan plan;
      plan.init(qt, p.lq, p.lk, C::kBM, C::kBN, p.diag_window, p.sink_window, p.causal != 0);
      const ItemRange ir = item_range<SPLIT>(pp, plan, SPLIT ? k % pp.n_split : 0);
      if (ir.e0 >= ir.e1) continue;
      const int ns = bh1 >= 0 ? 2 : 1;
      const bool shared_kv = ns == 2 && mat_k_of(p, bh0) == mat_k_of(p, bh1);
      const int nk = shared_kv ? 1 : ns;
      const uint32_t vc0 = vc;
      vc += nk * (ir.e1 - ir.e0);
      if (x >= ns) continue;  // odd head count: stream B idles on this pair
      constexpr int rb = DV;  // fp8 V row bytes (MN-major)
      const uint64_t dh = static_cast<uint64_t>(ptx::desc_hi(8 * rb, swz_mode(rb))) << 32;
      for (int e = ir.e0; e < ir.e1; ++e) {
        ptx::mbar_wait(p_full + x, pvc & 1);
        ++pvc;
        ptx::tc_fence_after();
        const uint32_t vpos = vc0 + nk * (e - ir.e0) + (shared_kv ? 0 : x);
        const uint32_t vslt = vpos % C::kNV;
        ptx::mbar_wait(v_full + vslt, (vpos / C::kNV) & 1);
        ptx::tc_fence_after();
        ptx::wu::tc_cp_sf(tsfv, sf_desc(C::oSfV + vslt * 512));
        const uint32_t vaddr = sbase + C::oV + vslt * C::kVBytes;
#pragma unroll
        for (int kk = 0; kk < C::kBN / 32; ++kk) {
          const uint64_t bd = dh | ptx::desc_lo(vaddr + kk * 32 * rb, 16);
          const uint32_t id = ptx::idesc_bs(0, 0, 0, 1, 128, DV, 1, kk & 3, kk & 3);
          ptx::wu::mma_mxf8f6f4_ts(tO, tmem + C::tP(x) + 8 * kk, bd, id, tsfp, tsfv, !(e == ir.e0 && kk == 0));
        }
        ptx::wu::tc_commit(v_empty + vslt);
        if (!shared_kv) ptx::wu::tc_commit(v_empty + vslt);
        ptx::wu::tc_commit(o_done + x);
      }
    }
  }
  } else {
    if (!FUSE) ptx::setmaxnreg_inc<C::kRegSoft>();
    // =========================== softmax (kSplit warpgroups per stream) ===========================
    // TMEM is read in the 32x32b shape: thread = one query row (lane of its warp's
    // 32-lane sub-partition) and NK = 128 / kSplit S columns.  With kSplit = 2 the two
    // warps sharing a row each take one half of the key tile (4 softmax warps per SM
    // sub-partition, for latency hiding) and exchange their partial row maxima through
    // shared memory.  K rows are permuted inside every 128-key tile (perm_row); the
    // permutation maps 32-key group G onto S columns [32G, 32G + 32), so a thread's key
    // half is its column half and undoing the order is compile-time register renaming:
    // key k sits in S column perm_row(k), its S_q^K in slot perm_slot(k).
    constexpr int NK = 128 / kSplit;  // keys (S columns) per thread
    constexpr int NW = NK / 4;        // E4M3 P words per thread
    constexpr int NG = NK / 32;       // 32-key groups per thread
    constexpr int OC = DV / kSplit;   // O columns per thread
    const int x = warp / (4 * kSplit);  // stream
    const int hh = kSplit == 1 ? 0 : (warp >> 2) & 1;
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    const int kb = NK * hh;  // first key / S column of this thread's half
    const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t xbar = 3 + x * 4 + quad;
    const bool tw = quad == 0 && hh == 0;  // the traced warp of this stream (DMA_TRACE)
    (void)tw;
    TRACE_DECL  // named barrier of the kSplit warps sharing these rows
    float* red = reinterpret_cast<float*>(smem + C::oRed);  // [2 parity][2 stream][2 half][128]
    // lazy rescaling (the FA4 trick): a row keeps its running max until a tile raises it
    // by more than kLazy (log2 units), so O is rarely rescaled; P <= 2^kLazy is stored as
    // E4M3(P * 2^(8 - kLazy)) <= 256 < 448.
    constexpr float kLazy = 4.f;
    constexpr float kPShift = 8.f - kLazy;
    uint32_t g = 0, sc = 0;
    if (kTurns && x == 1) ptx::named_bar_arrive(1, 256 * kSplit);  // A takes the first exp phase
    PROF_DECL

    for (uint32_t it = 0;; ++it) {
      const int ss = it % C::kNSch;
      ptx::mbar_wait(sch_full + ss, (it / C::kNSch) & 1);
      const int k = sched[ss];
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(sch_empty + ss);
      if (k < 0) break;
      int bh[2], qt;
      pair_coords(p, pp, SPLIT ? k / pp.n_split : k, bh[0], bh[1], qt);
      const int my_bh = bh[x];
      Plan plan;
      plan.init(qt, p.lq, p.lk, C::kBM, C::kBN, p.diag_window, p.sink_window, p.causal != 0);
      const ItemRange ir = item_range<SPLIT>(pp, plan, SPLIT ? k % pp.n_split : 0);
      if (my_bh < 0 || ir.skip) continue;  // odd head count: stream B idles on this pair
      // the item index is parked in shared memory for the epilogue (the softmax runs at its
      // register limit: nothing extra may stay live across the tile loop)
      if (SPLIT && lane == 0) sched[C::kItmSlot + warp] = k;
      const bool pair2 = bh[1] >= 0;
      const int q0 = qt * C::kBM;
      const int qrow = q0 + row;
      // S_q^Q of this row; in the fused kernel it is written by the quantizer warps, so it is
      // read after the pair's first S is ready (which follows the producer's acquire of the Q flag)
      float sq_q = (!FUSE && qrow < p.lq) ? p.qs_q[static_cast<int64_t>(my_bh) * p.lq_pad + qrow] : 1.0f;
      float m_run = -INFINITY;
      float2 l2 = make_float2(0.f, 0.f);

      bool first_split_tile = true;
      for (int e = ir.e0; e < ir.e1; ++e, ++g, first_split_tile = false) {
        const bool first_tile = SPLIT ? first_split_tile : e == 0;
        int t;
        bool hi;
        plan.entry(e, t, hi);
        if (LOW == kLowHigh) hi = true;
        const bool two_level = hi || (LOW == kLowNV);
        const int k0 = t * C::kBN;
        PROF_MARK(9);
        ptx::mbar_wait(s_full + x, g & 1);
        ptx::tc_fence_after();
        if (FUSE && first_tile && qrow < p.lq) sq_q = ld_acquire_f32(p.qs_q + static_cast<int64_t>(my_bh) * p.lq_pad + qrow);
        TRACE(tw, x, 1);
        PROF_MARK(0);
        // load the first half of this thread's columns, start the second, scale the first while it lands
        uint32_t sr[NK];
#pragma unroll
        for (int c = 0; c < NK / 2; c += 32)
          ptx::tmem_ld32(tmem + C::tS + lane_base + kb + c, *reinterpret_cast<uint32_t(*)[32]>(&sr[c]));
        ptx::tmem_ld_wait();
#pragma unroll
        for (int c = NK / 2; c < NK; c += 32)
          ptx::tmem_ld32(tmem + C::tS + lane_base + kb + c, *reinterpret_cast<uint32_t(*)[32]>(&sr[c]));
        PROF_MARK(1);
        // tv[i] = S[key kb + i] * S_q^K[kb + i], natural key order (FMUL2 over key pairs
        // 4w + {0,1}, {2,3}, which are adjacent S columns perm_row(4w) + {0, 1})
        const int sl = sc % C::kNS;
        ++sc;
        const uint32_t sqk = ptx::smem_u32(smem + C::oSqK + (x * C::kNS + sl) * C::kSqkBytes) + kb;
        float tv[NK];
        auto scale_words = [&](int w0) {
#pragma unroll
          for (int w = w0; w < w0 + NW / 2; ++w) {
            // perm_row(kb + i) = kb + perm_row(i) for kb in {0, 64}: compile-time register indices
            const int c0 = perm_row(4 * w), c1 = perm_row(4 * w + 2);
            float2 a = make_float2(__uint_as_float(sr[c0]), __uint_as_float(sr[c0 + 1]));
            float2 b = make_float2(__uint_as_float(sr[c1]), __uint_as_float(sr[c1 + 1]));
            if (two_level) {
              const float4 f = ptx::lds_f4(sqk + 4 * perm_slot(4 * w));  // perm_slot(kb + i) = perm_slot(i) + kb / 4
              a = __fmul2_rn(a, make_float2(f.x, f.y));
              b = __fmul2_rn(b, make_float2(f.z, f.w));
            }
            tv[4 * w] = a.x;
            tv[4 * w + 1] = a.y;
            tv[4 * w + 2] = b.x;
            tv[4 * w + 3] = b.y;
          }
        };
#if DMA_PP_HALF_FREE
        if (kSplit == 1) {
          // first half already landed (waited above): hand S columns [0, 64) back now
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(s_free);
          scale_words(0);
          ptx::tmem_ld_wait();
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(s_free + 1);
        } else {
          scale_words(0);
          ptx::tmem_ld_wait();
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(s_free + hh);  // this warp's column half
        }
        TRACE(tw, x, 2);
#elif DMA_PP_EARLY_FREE
        ptx::tmem_ld_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(s_free);  // S buffer may be overwritten by the next QK
        TRACE(tw, x, 2);
        scale_words(0);
#else
        scale_words(0);
        ptx::tmem_ld_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(s_free);  // S buffer may be overwritten by the next QK
        TRACE(tw, x, 2);
#endif
        scale_words(NW / 2);
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(sq_empty + x * C::kNS + sl);
        PROF_MARK(2);
        // causal (attention.py:178-184, applied when k1-1 > q0, :306) and ragged-key masks
        const int kvalid = p.lk - k0;
        const bool need_causal = p.causal && (k0 + (kvalid < C::kBN ? kvalid : C::kBN) - 1 > q0);
        if (need_causal || kvalid < C::kBN) {
          const int lim = (need_causal ? min(qrow - k0 + 1, kvalid) : kvalid) - kb;
#pragma unroll
          for (int j = 0; j < NK; ++j)
            if (j >= lim) tv[j] = -INFINITY;
        }
#if DMA_PP_MAXCH8
        // row max: 8 independent FMNMX3 chains
        float m8[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) m8[c] = fmaxf(tv[2 * c], tv[2 * c + 1]);
#pragma unroll
        for (int j = 16; j < NK; j += 16)
#pragma unroll
          for (int c = 0; c < 8; ++c) m8[c] = ptx::fmax3(m8[c], tv[j + 2 * c], tv[j + 2 * c + 1]);
        float mx = fmaxf(ptx::fmax3(ptx::fmax3(m8[0], m8[1], m8[2]), ptx::fmax3(m8[3], m8[4], m8[5]), m8[6]), m8[7]);
#else
        // row max: 4 independent FMNMX3 chains
        float m4[4] = {fmaxf(tv[0], tv[1]), fmaxf(tv[2], tv[3]), fmaxf(tv[4], tv[5]), fmaxf(tv[6], tv[7])};
#pragma unroll
        for (int j = 8; j < NK; j += 8) {
          m4[0] = ptx::fmax3(m4[0], tv[j], tv[j + 1]);
          m4[1] = ptx::fmax3(m4[1], tv[j + 2], tv[j + 3]);
          m4[2] = ptx::fmax3(m4[2], tv[j + 4], tv[j + 5]);
          m4[3] = ptx::fmax3(m4[3], tv[j + 6], tv[j + 7]);
        }
        float mx = fmaxf(ptx::fmax3(m4[0], m4[1], m4[2]), m4[3]);
#endif
        if (kSplit == 2) {
          float* rb = red + ((g & 1) * 2 + x) * 256;
          rb[hh * 128 + row] = mx;
          ptx::named_bar_sync(xbar, 64);
          mx = fmaxf(mx, rb[(hh ^ 1) * 128 + row]);
        }
        const float rowf = two_level ? sq_q : 1.0f;
        const float m_cand = fmaxf(m_run, mx * rowf);
        const bool upd = m_cand > m_run + kLazy;  // always for the first live tile (m_run = -inf)
        const float m_new = upd ? m_cand : m_run;
        const bool dead = (m_new == -INFINITY);
        const float alpha = (dead || !upd) ? 1.0f : fast_exp2(m_run - m_new);  // m_run = -inf -> 0
        const float bias = dead ? 0.f : (kPShift - m_new);
        m_run = m_new;
        TRACE(tw, x, 3);
        PROF_MARK(3);
        // P_x (and O_x) are read by PV(e-1): wait for it before overwriting.  Late wait:
        // just before the first P store, so the exps of key group 0 hide the wait
#if !DMA_PP_LATE_PV_WAIT
        if (kPSmem) {
          // P buffer g & 1 was read by PV(g - 2) (this stream's tile count g)
          if (g >= 2) ptx::mbar_wait(o_done + 2 * x + (g & 1), ((g - 2) >> 1) & 1);
        } else if (!first_tile) {
          ptx::mbar_wait(o_done + x, (g - 1) & 1);
          ptx::tc_fence_after();
        }
#endif
        PROF_MARK(4);
        // exp phases of the two streams alternate when kTurns (named barriers 1 = "A may
        // exp", 2 = "B may exp"): MUFU.EX2 is the shared bottleneck
        if (kTurns && pair2) ptx::named_bar_sync(1 + x, 256 * kSplit);
        TRACE(tw, x, 4);
        PROF_MARK(5);
        // exp2 + E4M3 requantisation of P, software-pipelined: the 32 MUFU.EX2 of key
        // group q are interleaved with the F2FP packs of group q - 1
        const float2 rf2 = make_float2(rowf, rowf), b2 = make_float2(bias, bias);
        float2 ls = make_float2(0.f, 0.f);
        if (!kExpInterleave) {
#pragma unroll
          for (int k2 = 0; k2 < NK; k2 += 2) {
            const float2 v = __ffma2_rn(make_float2(tv[k2], tv[k2 + 1]), rf2, b2);
            tv[k2] = v.x;
            tv[k2 + 1] = v.y;
          }
        }
        uint32_t pk[8];
#pragma unroll
        for (int q4 = 0; q4 <= NG; ++q4) {  // key group q4 = keys kb + [32 q4, 32 q4 + 32)
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (q4 < NG) {
              const int kk = 32 * q4 + 2 * j;
              if ((j & 3) < kPolyPP) {  // FMA-pipe exp2 for a fixed share of the pairs (offloads MUFU)
                const float2 e2 = exp2_poly2(make_float2(tv[kk], tv[kk + 1]));
                tv[kk] = e2.x;
                tv[kk + 1] = e2.y;
              } else if (kExpInterleave) {
                // the argument FFMA2 issued in program order right before its MUFU pair (no
                // 64-instruction prologue ahead of the first exp)
                const float2 v = ffma2_ordered(make_float2(tv[kk], tv[kk + 1]), rf2, b2);
                tv[kk] = exp2_ordered(v.x);
                tv[kk + 1] = exp2_ordered(v.y);
              } else {
                tv[kk] = exp2_ordered(tv[kk]);
                tv[kk + 1] = exp2_ordered(tv[kk + 1]);
              }
            }
            if (q4 > 0) {
              const int kk = 32 * (q4 - 1) + 2 * j;  // pack P of group q4 - 1
              const uint32_t hv = cvt_e4m3x2_ordered(tv[kk], tv[kk + 1]);
              if (j & 1) {
                pk[j >> 1] |= hv << 16;
              } else {
                pk[j >> 1] = hv;
              }
              const float2 e2 = make_float2(tv[kk], tv[kk + 1]);
              ls = (q4 == 1 && j == 0) ? e2 : __fadd2_rn(ls, e2);
            }
          }
#if DMA_PP_LATE_PV_WAIT
          if (q4 == 1 && !first_tile) {
            ptx::mbar_wait(o_done + x, (g - 1) & 1);
            ptx::tc_fence_after();
          }
#endif
          if (q4 > 0) {
            if (kPSmem) {
              // row `row` of the 128B-swizzled K-major tile: 16-byte chunk c at c ^ (row & 7)
              const uint32_t rbase = ptx::smem_u32(smem + C::oP + (2 * x + (g & 1)) * C::kPBytes) + row * 128;
              const uint32_t c0 = 2 * (q4 - 1), c1 = c0 + 1;
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rbase + ((c0 ^ (row & 7)) << 4)),
                           "r"(pk[0]), "r"(pk[1]), "r"(pk[2]), "r"(pk[3]) : "memory");
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rbase + ((c1 ^ (row & 7)) << 4)),
                           "r"(pk[4]), "r"(pk[5]), "r"(pk[6]), "r"(pk[7]) : "memory");
            } else {
              ptx::tmem_st8(tmem + C::tP(x) + lane_base + NW * hh + 8 * (q4 - 1), pk);
            }
          }
        }
        if (kTurns && pair2) ptx::named_bar_arrive(2 - x, 256 * kSplit);
        TRACE(tw, x, 5);
        l2 = __ffma2_rn(l2, make_float2(alpha, alpha), ls);
        PROF_MARK(6);
        if (!first_tile && __any_sync(0xffffffffu, alpha != 1.0f)) {
          // this thread's O columns *= alpha
          if (kPSmem) {  // O holds PV(g - 1) once it completes
            ptx::mbar_wait(o_done + 2 * x + ((g - 1) & 1), ((g - 1) >> 1) & 1);
            ptx::tc_fence_after();
          }
          const float2 a2 = make_float2(alpha, alpha);
#pragma unroll
          for (int cq = 0; cq < OC / 32; ++cq) {
            const uint32_t ta = tmem + C::tO(x) + lane_base + OC * hh + 32 * cq;
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
        if (kPSmem) ptx::fence_proxy_async_smem();  // P stores -> visible to the PV MMA (async proxy)
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(kPSmem ? p_full + 2 * x + (g & 1) : p_full + x);
        TRACE(tw, x, 6);
        PROF_MARK(7);
      }

      // ---- epilogue: O / l (attention.py:104-106), one row per thread (32x32b)
      float my_l = l2.x + l2.y;
      if (kSplit == 2) {
        float* rl = red + 1024 + ((it & 1) * 2 + x) * 256;
        rl[hh * 128 + row] = my_l;
        ptx::named_bar_sync(xbar, 64);
        my_l += rl[(hh ^ 1) * 128 + row];
      }
      const float inv_l = 1.0f / (my_l > 0.f ? my_l : 1.0f);
      if (SPLIT) __syncwarp();
      const int k_me = SPLIT ? sched[C::kItmSlot + warp] : k;
      int qt_me;
      {
        int b0, b1;
        pair_coords(p, pp, SPLIT ? k_me / pp.n_split : k_me, b0, b1, qt_me);
      }
      const int s_me = SPLIT ? k_me % pp.n_split : 0;
      const ItemRange ir_me = item_range<SPLIT>(pp, plan, s_me);
      const bool any = ir_me.e1 > ir_me.e0;
      if (any) {
        if (kPSmem)
          ptx::mbar_wait(o_done + 2 * x + ((g - 1) & 1), ((g - 1) >> 1) & 1);
        else
          ptx::mbar_wait(o_done + x, (g - 1) & 1);
        ptx::tc_fence_after();
      }
      const uint32_t tO = tmem + C::tO(x) + lane_base + OC * hh;
      const int64_t orow = static_cast<int64_t>(my_bh) * p.lq + qrow;
      constexpr int kPartW = DV + 4;  // floats per partial row: O, (m, l), 2 of padding (16-byte rows)
      const bool split = SPLIT && ir_me.ns > 1;
      const int64_t pslot = SPLIT ? (static_cast<int64_t>(my_bh) * p.n_qt + qt_me) * pp.n_split : 0;
#pragma unroll
      for (int c = 0; c < OC / 32; ++c) {
        uint32_t rr[32];
        if (any) {
          ptx::tmem_ld32(tO + 32 * c, rr);
          ptx::tmem_ld_wait();
        } else {
#pragma unroll
          for (int i2 = 0; i2 < 32; ++i2) rr[i2] = 0u;
        }
        if (split) {
          // unnormalised O of this split (relative to 2^(kPShift - m_run), as l)
          float4* dst = reinterpret_cast<float4*>(pp.part + ((pslot + s_me) * 128 + row) * kPartW + OC * hh + 32 * c);
#pragma unroll
          for (int i2 = 0; i2 < 8; ++i2)
            dst[i2] = make_float4(__uint_as_float(rr[4 * i2]), __uint_as_float(rr[4 * i2 + 1]),
                                  __uint_as_float(rr[4 * i2 + 2]), __uint_as_float(rr[4 * i2 + 3]));
        } else if (qrow < p.lq) {
          store_orow<DV>(p, orow, (OC / 32) * hh + c, rr, inv_l);
        }
      }
      ptx::tc_fence_before();
      if (split && hh == 0) {
        // (m, l) of the split next to its O row (the row's, shared by both column halves);
        // kv_combine_kernel merges the splits
        float* me = pp.part + ((pslot + s_me) * 128 + row) * kPartW + DV;
        me[0] = m_run;
        me[1] = my_l;
      }
      PROF_MARK(8);
    }
    if (kTurns && x == 0) ptx::named_bar_sync(1, 256 * kSplit);  // consume B's last hand-over
    PROF_FLUSH(0, 10);
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == kMma) ptx::tmem_dealloc<512>(tmem);
}

// Merge of the KV splits (PPParams n_split > 1): one warp per query row, lane = 4 output
// columns.  O = sum_s 2^(m_s - M) O_s / sum_s 2^(m_s - M) l_s with M = max_s m_s: the online
// softmax state merge of attention.py:150-175 across plan ranges.  Row blocks whose plan
// has a single range were written by the attention kernel directly.
template <int DV>
__global__ void __launch_bounds__(256) kv_combine_kernel(const __grid_constant__ AttnParams p, const float* __restrict__ part,
                                                         int n_split) {
  constexpr int kPartW = DV + 4, kLanes = DV / 4;
  ptx::pdl_wait();  // the attention kernel's partials
  const int rows_per_cta = 256 / kLanes;
  const int64_t blk = blockIdx.x;  // (bh, qt, row group)
  const int groups = 128 / rows_per_cta;
  const int64_t bq = blk / groups;
  const int qt = static_cast<int>(bq % p.n_qt);
  const int64_t bh = bq / p.n_qt;
  const int row = static_cast<int>(blk % groups) * rows_per_cta + threadIdx.x / kLanes;
  const int c4 = (threadIdx.x % kLanes) * 4;
  const int qrow = qt * 128 + row;
  if (qrow >= p.lq) return;
  const float* base = part + ((bq * n_split) * 128 + row) * kPartW;
  const int64_t sstride = 128 * kPartW;
  // (m, l) of every slot in one round of loads (issued before the plan arithmetic); slots
  // past this tile's range count ns were not written by this launch and are masked once ns
  // is known.  ns = 1: the attention kernel wrote O itself
  float ms[16], ls[16];
#pragma unroll
  for (int s = 0; s < 16; ++s) {
    if (s < n_split) {
      const float4 h = __ldcg(reinterpret_cast<const float4*>(base + s * sstride + DV));
      ms[s] = h.x;
      ls[s] = h.y;
    } else {
      ms[s] = -INFINITY;
      ls[s] = 0.f;
    }
  }
  Plan plan;
  plan.init(qt, p.lq, p.lk, 128, 128, p.diag_window, p.sink_window, p.causal != 0);
  const int ns = n_split < plan.n ? n_split : plan.n;
  if (ns <= 1) return;
  float mm = -INFINITY;
#pragma unroll
  for (int s = 0; s < 16; ++s) {
    if (s >= ns) {
      ms[s] = -INFINITY;
      ls[s] = 0.f;
    }
    mm = fmaxf(mm, ms[s]);
  }
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  float ll = 0.f;
#pragma unroll
  for (int s = 0; s < 16; ++s) {
    if (s < ns) {
      const float w = ms[s] == -INFINITY ? 0.f : exp2f(ms[s] - mm);
      const float4 v = __ldcg(reinterpret_cast<const float4*>(base + s * sstride + c4));
      ll += w * ls[s];
      acc.x += w * v.x;
      acc.y += w * v.y;
      acc.z += w * v.z;
      acc.w += w * v.w;
    }
  }
  const float inv = 1.0f / (ll > 0.f ? ll : 1.0f);
  const int64_t o = (bh * p.lq + qrow) * DV + c4;
  if (p.out_bf16) {
    __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(reinterpret_cast<__nv_bfloat16*>(p.o) + o);
    dst[0] = __floats2bfloat162_rn(acc.x * inv, acc.y * inv);
    dst[1] = __floats2bfloat162_rn(acc.z * inv, acc.w * inv);
  } else {
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(p.o) + o) =
        make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
  }
}

}  // namespace dma
