// Phase 2 of the DMA forward: diagonal-tiled mixed-precision flash attention
// on sm_100a (tcgen05 block-scaled MMAs, TMEM accumulators, TMA loads).
//
// Restates attention.py:282-310 (tile loop) with the tile scheduler of
// attention.py:191-233 (Plan, common.cuh) and the base-2 online softmax of
// attention.py:150-175 (l0 = 0, dead rows keep alpha = 1, normalisation
// guard l > 0 from attention.py:104-106).
//
// One CTA = one (batch, head, 128-row query tile).  Warp roles:
//   warp 0      TMA producer: Q (hi+lo codes, SF atoms) once, then per plan
//               entry the K tile in the entry's precision (+SF, +S_q^K) into
//               a 3-stage ring and the V tile into a 2-stage ring
//   warp 1      MMA issuer (one thread): S = Q K^T (kind::mxf8f6f4 for high
//               tiles, kind::mxf4nvf4 4X / kind::mxf4 2X for low tiles) into a
//               double-buffered S in TMEM; O += P V (kind::mxf8f6f4 with P
//               read from TMEM, or kind::f16 in the bf16 parity mode)
//   warps 4-7   softmax: one query row per thread; S_q^Q x S_q^K rescale,
//               causal / ragged mask, online max/sum, exp2, P -> E4M3 (x2^8)
//               or bf16 written back into the S columns in TMEM, O rescale,
//               final O / l epilogue
// TMEM (512 cols): S0 [0,128) S1 [128,256) O [256,256+DV) scale factors [384,424)
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>

#include "common.cuh"
#include "ptx.cuh"

namespace dma {

enum LowKind { kLowNV = 0, kLowMX4 = 1, kLowHigh = 2 };

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
  int n_qt;
  int diag_window, sink_window, causal;
  int ch_hi, ch_lo;
  int hfmt;  // high-path element format: 0 = E4M3, 1 = E5M2
};

template <int D, int DV, int LOW, bool PVBF16>
struct AttnCfg {
  static constexpr int kBM = 128, kBN = 128;
  static constexpr int kNK = 3, kNV = 2;
  static constexpr int kQHiBytes = kBM * D;
  static constexpr int kQLoBytes = kBM * D / 2;
  static constexpr int kKBytes = kBN * D;  // fp8 size; fp4 tiles use half
  static constexpr int kVBytes = PVBF16 ? kBN * DV * 2 : kBN * DV;
  static constexpr int kChHi = (D / 32 + 3) / 4;
  static constexpr int kChLo = LOW == kLowNV ? (D / 16 + 3) / 4 : (D / 32 + 3) / 4;
  static constexpr int kChK = kChHi > kChLo ? kChHi : kChLo;
  // smem carve-up (offsets from a 1024-aligned base)
  static constexpr int oQHi = 0;
  static constexpr int oQLo = oQHi + kQHiBytes;
  static constexpr int oK = ((oQLo + kQLoBytes + 1023) / 1024) * 1024;
  static constexpr int kKStage = kKBytes;
  static constexpr int oV = oK + kNK * kKStage;
  static constexpr int oSmall = oV + kNV * kVBytes;
  static constexpr int oSfQHi = oSmall;
  static constexpr int oSfQLo = oSfQHi + 512 * kChHi;
  static constexpr int oSfK = oSfQLo + 512 * kChLo;
  static constexpr int oSqK = oSfK + kNK * 512 * kChK;
  static constexpr int oSfV = oSqK + kNK * 512;
  static constexpr int oSfP = oSfV + kNV * 512;
  static constexpr int oBar = oSfP + 512;
  static constexpr int kSmemBytes = oBar + 256 + 1024;  // + alignment slack
  // TMEM columns
  static constexpr uint32_t tS0 = 0, tS1 = 128, tO = 256;
  static constexpr uint32_t tSfQHi = 384, tSfQLo = 388, tSfK0 = 396, tSfK1 = 404, tSfV0 = 412, tSfV1 = 416,
                            tSfP = 420;
};

__device__ __forceinline__ uint32_t swz_mode(int row_bytes) {
  return row_bytes >= 128 ? ptx::kSw128 : (row_bytes == 64 ? ptx::kSw64 : ptx::kSw32);
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int D, int DV, int LOW, bool PVBF16>
__global__ void __launch_bounds__(256, 1) dma_attn_kernel(const __grid_constant__ AttnParams p) {
  using C = AttnCfg<D, DV, LOW, PVBF16>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::oBar);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;            // [kNK]
  uint64_t* k_empty = bars + 1 + C::kNK;  // [kNK]
  uint64_t* v_full = bars + 1 + 2 * C::kNK;
  uint64_t* v_empty = v_full + C::kNV;
  uint64_t* s_full = v_empty + C::kNV;  // [2]
  uint64_t* p_full = s_full + 2;
  uint64_t* o_done = p_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- work item: heaviest causal query tile of each head first (LPT within a head)
  const int item = blockIdx.x;
  const int bh = item / p.n_qt;
  const int qt = p.n_qt - 1 - (item % p.n_qt);
  const int b = bh / p.heads, h = bh % p.heads;
  const int mat_q = bh;
  const int mat_k = b * p.kv_heads + h / p.group;
  const int q0 = qt * C::kBM;
  Plan plan;
  plan.init(qt, p.lq, p.lk, C::kBM, C::kBN, p.diag_window, p.sink_window, p.causal != 0);
  const int n_ent = plan.n;
  const int rt_q = p.lq_pad >> 7, rt_k = p.lk_pad >> 7;

  if (warp == 0) {
    if (lane == 0) {
      ptx::mbar_init(q_full, 1);
      for (int i = 0; i < C::kNK; ++i) {
        ptx::mbar_init(k_full + i, 1);
        ptx::mbar_init(k_empty + i, 1);
      }
      for (int i = 0; i < C::kNV; ++i) {
        ptx::mbar_init(v_full + i, 1);
        ptx::mbar_init(v_empty + i, 1);
      }
      ptx::mbar_init(s_full + 0, 1);
      ptx::mbar_init(s_full + 1, 1);
      ptx::mbar_init(p_full, 4);
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
    reinterpret_cast<uint32_t*>(smem + C::oSfP)[lane] = 0x7F7F7F7Fu;
    reinterpret_cast<uint32_t*>(smem + C::oSfP)[lane + 32] = 0x7F7F7F7Fu;
    reinterpret_cast<uint32_t*>(smem + C::oSfP)[lane + 64] = 0x7F7F7F7Fu;
    reinterpret_cast<uint32_t*>(smem + C::oSfP)[lane + 96] = 0x7F7F7F7Fu;
    ptx::fence_proxy_async_smem();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // =========================== TMA producer ===========================
    if (lane == 0 && n_ent > 0) {
      uint32_t qbytes = C::kQHiBytes + 512 * C::kChHi;
      if (LOW != kLowHigh) qbytes += C::kQLoBytes + 512 * C::kChLo;
      ptx::mbar_arrive_expect_tx(q_full, qbytes);
      ptx::tma_load_3d(smem + C::oQHi, &p.tm_q_hi, q_full, 0, q0, mat_q);
      ptx::bulk_load(smem + C::oSfQHi, p.sf_q_hi + (static_cast<int64_t>(mat_q) * rt_q + qt) * p.ch_hi * 512,
                     512 * C::kChHi, q_full);
      if (LOW != kLowHigh) {
        ptx::tma_load_3d(smem + C::oQLo, &p.tm_q_lo, q_full, 0, q0, mat_q);
        ptx::bulk_load(smem + C::oSfQLo, p.sf_q_lo + (static_cast<int64_t>(mat_q) * rt_q + qt) * p.ch_lo * 512,
                       512 * C::kChLo, q_full);
      }
      for (int e = 0; e < n_ent; ++e) {
        int t;
        bool hi;
        plan.entry(e, t, hi);
        if (LOW == kLowHigh) hi = true;
        const int ks = e % C::kNK;
        ptx::mbar_wait(k_empty + ks, ((e / C::kNK) & 1) ^ 1);
        const int ch = hi ? C::kChHi : C::kChLo;
        const uint32_t kb = hi ? C::kKBytes : C::kKBytes / 2;
        ptx::mbar_arrive_expect_tx(k_full + ks, kb + 512 * ch + 512);
        ptx::tma_load_3d(smem + C::oK + ks * C::kKStage, hi ? &p.tm_k_hi : &p.tm_k_lo, k_full + ks, 0,
                         t * C::kBN, mat_k);
        const uint8_t* sfsrc = (hi ? p.sf_k_hi : p.sf_k_lo) +
                               (static_cast<int64_t>(mat_k) * rt_k + t) * (hi ? p.ch_hi : p.ch_lo) * 512;
        ptx::bulk_load(smem + C::oSfK + ks * 512 * C::kChK, sfsrc, 512 * ch, k_full + ks);
        ptx::bulk_load(smem + C::oSqK + ks * 512, p.qs_k + static_cast<int64_t>(mat_k) * p.lk_pad + t * C::kBN,
                       512, k_full + ks);

        const int vs = e % C::kNV;
        ptx::mbar_wait(v_empty + vs, ((e / C::kNV) & 1) ^ 1);
        uint8_t* vdst = smem + C::oV + vs * C::kVBytes;
        if (PVBF16) {
          ptx::mbar_arrive_expect_tx(v_full + vs, C::kVBytes);
#pragma unroll
          for (int half = 0; half < DV / 64; ++half)
            ptx::tma_load_3d(vdst + half * (C::kBN * 128), &p.tm_v, v_full + vs, half * 64, t * C::kBN, mat_k);
        } else {
          ptx::mbar_arrive_expect_tx(v_full + vs, C::kVBytes + 512);
          ptx::tma_load_3d(vdst, &p.tm_v, v_full + vs, 0, t * C::kBN, mat_k);
          ptx::bulk_load(smem + C::oSfV + vs * 512, p.sf_v + (static_cast<int64_t>(mat_k) * rt_k + t) * 512, 512,
                         v_full + vs);
        }
      }
    }
  } else if (warp == 1) {
    // =========================== MMA issuer ===========================
    if (lane == 0 && n_ent > 0) {
      ptx::mbar_wait(q_full, 0);
      ptx::tc_fence_after();
      for (int j = 0; j < C::kChHi; ++j)
        ptx::tc_cp_sf(tmem + C::tSfQHi + 4 * j,
                      ptx::smem_desc(ptx::smem_u32(smem + C::oSfQHi + 512 * j), 0, 128, ptx::kSwNone));
      if (LOW != kLowHigh)
        for (int j = 0; j < C::kChLo; ++j)
          ptx::tc_cp_sf(tmem + C::tSfQLo + 4 * j,
                        ptx::smem_desc(ptx::smem_u32(smem + C::oSfQLo + 512 * j), 0, 128, ptx::kSwNone));
      if (!PVBF16)
        ptx::tc_cp_sf(tmem + C::tSfP, ptx::smem_desc(ptx::smem_u32(smem + C::oSfP), 0, 128, ptx::kSwNone));

      auto issue_qk = [&](int e) {
        int t;
        bool hi;
        plan.entry(e, t, hi);
        if (LOW == kLowHigh) hi = true;
        const int ks = e % C::kNK;
        ptx::mbar_wait(k_full + ks, (e / C::kNK) & 1);
        ptx::tc_fence_after();
        const uint32_t tsfk = tmem + ((e & 1) ? C::tSfK1 : C::tSfK0);
        const int ch = hi ? C::kChHi : C::kChLo;
        for (int j = 0; j < ch; ++j)
          ptx::tc_cp_sf(tsfk + 4 * j, ptx::smem_desc(ptx::smem_u32(smem + C::oSfK + ks * 512 * C::kChK + 512 * j),
                                                     0, 128, ptx::kSwNone));
        const uint32_t tS = tmem + ((e & 1) ? C::tS1 : C::tS0);
        const uint32_t kaddr = ptx::smem_u32(smem + C::oK + ks * C::kKStage);
        if (hi) {
          const uint32_t qaddr = ptx::smem_u32(smem + C::oQHi);
          constexpr int rb = D;  // fp8 row bytes
          const uint32_t sw = swz_mode(rb);
#pragma unroll
          for (int kk = 0; kk < D / 32; ++kk) {
            const uint64_t ad = ptx::smem_desc(qaddr + 32 * kk, 16, 8 * rb, sw);
            const uint64_t bd = ptx::smem_desc(kaddr + 32 * kk, 16, 8 * rb, sw);
            const uint32_t f = static_cast<uint32_t>(p.hfmt);
            const uint32_t id = ptx::idesc_bs(f, f, 0, 0, 128, 128, 1, kk & 3, kk & 3);
            ptx::mma_mxf8f6f4(tS, ad, bd, id, tmem + C::tSfQHi + 4 * (kk >> 2), tsfk + 4 * (kk >> 2), kk > 0);
          }
        } else {
          const uint32_t qaddr = ptx::smem_u32(smem + C::oQLo);
          constexpr int rb = D / 2;  // packed fp4 row bytes
          const uint32_t sw = swz_mode(rb);
#pragma unroll
          for (int kk = 0; kk < D / 64; ++kk) {
            const uint64_t ad = ptx::smem_desc(qaddr + 32 * kk, 16, 8 * rb, sw);
            const uint64_t bd = ptx::smem_desc(kaddr + 32 * kk, 16, 8 * rb, sw);
            if (LOW == kLowNV) {
              const uint32_t id = ptx::idesc_bs(1, 1, 0, 0, 128, 128, 0, 0, 0);
              ptx::mma_nvf4(tS, ad, bd, id, tmem + C::tSfQLo + 4 * kk, tsfk + 4 * kk, kk > 0);
            } else {
              const uint32_t sid = (kk & 1) * 2;
              const uint32_t id = ptx::idesc_bs(1, 1, 0, 0, 128, 128, 1, sid, sid);
              ptx::mma_mxf4(tS, ad, bd, id, tmem + C::tSfQLo + 4 * (kk >> 1), tsfk + 4 * (kk >> 1), kk > 0);
            }
          }
        }
        ptx::tc_commit(k_empty + ks);
        ptx::tc_commit(s_full + (e & 1));
      };

      issue_qk(0);
      for (int e = 0; e < n_ent; ++e) {
        if (e + 1 < n_ent) issue_qk(e + 1);
        ptx::mbar_wait(p_full, e & 1);
        ptx::tc_fence_after();
        const int vs = e % C::kNV;
        ptx::mbar_wait(v_full + vs, (e / C::kNV) & 1);
        ptx::tc_fence_after();
        const uint32_t tP = tmem + ((e & 1) ? C::tS1 : C::tS0);
        const uint32_t vaddr = ptx::smem_u32(smem + C::oV + vs * C::kVBytes);
        if (PVBF16) {
#pragma unroll
          for (int kk = 0; kk < C::kBN / 16; ++kk) {
            const uint64_t bd = ptx::smem_desc(vaddr + kk * 16 * 128, C::kBN * 128, 1024, ptx::kSw128);
            ptx::mma_f16_ts(tmem + C::tO, tP + 8 * kk, bd, ptx::idesc_bf16(0, 1, 128, DV), (e > 0 || kk > 0));
          }
        } else {
          const uint32_t tsfv = tmem + ((e & 1) ? C::tSfV1 : C::tSfV0);
          ptx::tc_cp_sf(tsfv, ptx::smem_desc(ptx::smem_u32(smem + C::oSfV + vs * 512), 0, 128, ptx::kSwNone));
          constexpr int rb = DV;  // fp8 V row bytes (MN-major)
#pragma unroll
          for (int kk = 0; kk < C::kBN / 32; ++kk) {
            const uint64_t bd = ptx::smem_desc(vaddr + kk * 32 * rb, 16, 8 * rb, swz_mode(rb));
            const uint32_t id = ptx::idesc_bs(0, 0, 0, 1, 128, DV, 1, kk & 3, kk & 3);
            ptx::mma_mxf8f6f4_ts(tmem + C::tO, tP + 8 * kk, bd, id, tmem + C::tSfP, tsfv, (e > 0 || kk > 0));
          }
        }
        ptx::tc_commit(v_empty + vs);
        ptx::tc_commit(o_done);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // =========================== softmax / correction / epilogue ===========================
    const int r = threadIdx.x - 128;  // query row within the tile == TMEM lane
    const uint32_t lane_base = static_cast<uint32_t>((warp - 4) * 32) << 16;
    const int qrow = q0 + r;
    const float sq_q = (qrow < p.lq) ? p.qs_q[static_cast<int64_t>(mat_q) * p.lq_pad + qrow] : 1.0f;
    float m_run = -INFINITY, l_run = 0.f;
    constexpr float kPShift = PVBF16 ? 0.f : 8.f;  // P stored as E4M3(P * 2^8)

    for (int e = 0; e < n_ent; ++e) {
      int t;
      bool hi;
      plan.entry(e, t, hi);
      if (LOW == kLowHigh) hi = true;
      const bool two_level = hi || (LOW == kLowNV);
      const int k0 = t * C::kBN;
      ptx::mbar_wait(s_full + (e & 1), (e >> 1) & 1);
      ptx::tc_fence_after();
      const uint32_t tS = tmem + ((e & 1) ? C::tS1 : C::tS0) + lane_base;
      float s[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t rr[32];
        ptx::tmem_ld32(tS + 32 * c, rr);
#pragma unroll
        for (int i = 0; i < 32; ++i) s[32 * c + i] = __uint_as_float(rr[i]);
      }
      ptx::tmem_ld_wait();

      // S_q^K column factors for two-level tiles (staged by the producer with the K tile)
      const float rowf = two_level ? sq_q : 1.0f;
      if (two_level) {
        const float4* sqk = reinterpret_cast<const float4*>(smem + C::oSqK + (e % C::kNK) * 512);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float4 f = sqk[j];
          s[4 * j + 0] *= f.x;
          s[4 * j + 1] *= f.y;
          s[4 * j + 2] *= f.z;
          s[4 * j + 3] *= f.w;
        }
      }
      // causal (attention.py:178-184, applied when k1-1 > q0, :306) and ragged-key masks
      const int kvalid = p.lk - k0;  // keys [k0, k0+kvalid) exist
      const bool need_causal = p.causal && (k0 + (kvalid < C::kBN ? kvalid : C::kBN) - 1 > q0);
      if (need_causal || kvalid < C::kBN) {
        const int lim = need_causal ? min(qrow - k0 + 1, kvalid) : kvalid;  // keep j < lim
#pragma unroll
        for (int j = 0; j < 128; ++j)
          if (j >= lim) s[j] = -INFINITY;
      }
      float mx = -INFINITY;
#pragma unroll
      for (int j = 0; j < 128; ++j) mx = fmaxf(mx, s[j]);
      const float m_tile = mx * rowf;
      const float m_new = fmaxf(m_run, m_tile);
      const bool dead = (m_new == -INFINITY);
      const float alpha = dead ? 1.0f : fast_exp2(m_run - m_new);  // m_run = -inf -> 0
      const float bias = dead ? 0.f : (kPShift - m_new);
      float lsum = 0.f;
      if (PVBF16) {
        uint32_t pk[64];
#pragma unroll
        for (int j = 0; j < 64; ++j) {
          const float p0 = fast_exp2(fmaf(s[2 * j], rowf, bias));
          const float p1 = fast_exp2(fmaf(s[2 * j + 1], rowf, bias));
          lsum += p0 + p1;
          __nv_bfloat162 v = __floats2bfloat162_rn(p0, p1);
          pk[j] = *reinterpret_cast<uint32_t*>(&v);
        }
        const uint32_t tP = tmem + ((e & 1) ? C::tS1 : C::tS0) + lane_base;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t w[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) w[i] = pk[16 * c + i];
          ptx::tmem_st16(tP + 16 * c, w);
        }
      } else {
        uint32_t pk[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float p0 = fast_exp2(fmaf(s[4 * j + 0], rowf, bias));
          const float p1 = fast_exp2(fmaf(s[4 * j + 1], rowf, bias));
          const float p2 = fast_exp2(fmaf(s[4 * j + 2], rowf, bias));
          const float p3 = fast_exp2(fmaf(s[4 * j + 3], rowf, bias));
          lsum += (p0 + p1) + (p2 + p3);
          pk[j] = static_cast<uint32_t>(ptx::cvt_e4m3x2(p0, p1)) | (static_cast<uint32_t>(ptx::cvt_e4m3x2(p2, p3)) << 16);
        }
        const uint32_t tP = tmem + ((e & 1) ? C::tS1 : C::tS0) + lane_base;
        uint32_t w0[16], w1[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          w0[i] = pk[i];
          w1[i] = pk[16 + i];
        }
        ptx::tmem_st16(tP, w0);
        ptx::tmem_st16(tP + 16, w1);
      }
      l_run = l_run * alpha + lsum;
      m_run = m_new;
      // O *= alpha once the previous PV has landed (rows whose max moved)
      if (e > 0) {
        ptx::mbar_wait(o_done, (e - 1) & 1);
        ptx::tc_fence_after();
        if (__any_sync(0xffffffffu, alpha != 1.0f)) {
          const uint32_t tO = tmem + C::tO + lane_base;
#pragma unroll
          for (int c = 0; c < DV / 32; ++c) {
            uint32_t rr[32];
            ptx::tmem_ld32(tO + 32 * c, rr);
            ptx::tmem_ld_wait();
            uint32_t w0[16], w1[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              w0[i] = __float_as_uint(__uint_as_float(rr[i]) * alpha);
              w1[i] = __float_as_uint(__uint_as_float(rr[16 + i]) * alpha);
            }
            ptx::tmem_st16(tO + 32 * c, w0);
            ptx::tmem_st16(tO + 32 * c + 16, w1);
          }
        }
      }
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(p_full);
    }

    // ---- epilogue: O / l (attention.py:104-106)
    float inv_l = 1.0f / (l_run > 0.f ? l_run : 1.0f);
    if (n_ent > 0) {
      ptx::mbar_wait(o_done, (n_ent - 1) & 1);
      ptx::tc_fence_after();
    }
    const uint32_t tO = tmem + C::tO + lane_base;
    const int64_t orow = static_cast<int64_t>(mat_q) * p.lq + qrow;
#pragma unroll
    for (int c = 0; c < DV / 32; ++c) {
      uint32_t rr[32];
      if (n_ent > 0) {
        ptx::tmem_ld32(tO + 32 * c, rr);
        ptx::tmem_ld_wait();
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) rr[i] = 0u;
      }
      if (qrow < p.lq) {
        if (p.out_bf16) {
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.o) + orow * DV + 32 * c);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            uint32_t w[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              __nv_bfloat162 v = __floats2bfloat162_rn(__uint_as_float(rr[8 * i + 2 * k]) * inv_l,
                                                       __uint_as_float(rr[8 * i + 2 * k + 1]) * inv_l);
              w[k] = *reinterpret_cast<uint32_t*>(&v);
            }
            dst[i] = make_uint4(w[0], w[1], w[2], w[3]);
          }
        } else {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.o) + orow * DV + 32 * c);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            dst[i] = make_float4(__uint_as_float(rr[4 * i]) * inv_l, __uint_as_float(rr[4 * i + 1]) * inv_l,
                                 __uint_as_float(rr[4 * i + 2]) * inv_l, __uint_as_float(rr[4 * i + 3]) * inv_l);
        }
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc<512>(tmem);
}

}  // namespace dma
