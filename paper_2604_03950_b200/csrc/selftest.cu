// One-tile self-test of the tcgen05 block-scaled MMA conventions the DMA
// kernel relies on (UMMA descriptors, swizzles, scale-factor atoms in TMEM,
// A-from-TMEM).  D[128x128] = A[128xK] * B[128xK]^T with scales, or the PV
// form D = P[128xK] * V[Kx128].  Inputs are device pointers in the canonical
// row-major layouts; the GPU test compares D with a numpy decode.
#include "common.cuh"
#include "ptx.cuh"

namespace dma {

enum SelftestKind {
  kSTMxf8E4M3 = 0,  // A,B E4M3 K-major, E8M0 per 32
  kSTNvf4 = 1,      // A,B packed E2M1 K-major, E4M3 per 16
  kSTMxf4 = 2,      // A,B packed E2M1 K-major, E8M0 per 32
  kSTPvFp8 = 3,     // A = P E4M3 from TMEM, B = V E4M3 MN-major, E8M0 per 32 keys
  kSTPvBf16 = 4,    // A = P bf16 from TMEM, B = V bf16 MN-major
  kSTMxf8E5M2 = 5,
};

// byte offset of logical (row, byte) in a swizzled K-major tile with row_bytes per row
__device__ __forceinline__ uint32_t swz_offset(uint32_t row, uint32_t byte, uint32_t row_bytes) {
  uint32_t lin = row * row_bytes + byte;
  uint32_t mask = row_bytes == 128 ? 7u : (row_bytes == 64 ? 3u : 1u);
  return lin ^ (((lin >> 7) & mask) << 4);
}

__global__ void __launch_bounds__(128, 1) selftest_kernel(int kind, int K, const uint8_t* __restrict__ a,
                                                          const uint8_t* __restrict__ b,
                                                          const uint8_t* __restrict__ sfa,
                                                          const uint8_t* __restrict__ sfb, float* __restrict__ d) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                 // 32 KB
  uint8_t* sB = smem + 32768;         // 32 KB
  uint8_t* sSFA = smem + 65536;       // 2 KB
  uint8_t* sSFB = smem + 65536 + 2048;
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base_s;

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const bool fp4 = (kind == kSTNvf4 || kind == kSTMxf4);
  const bool pv = (kind == kSTPvFp8 || kind == kSTPvBf16);
  const int a_row_bytes = fp4 ? K / 2 : K;  // K-major operand row bytes (not used for pv A)

  if (warp == 0) ptx::tmem_alloc<512>(&tmem_base_s);
  if (tid == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_barrier_init();
  }

  // ---- operands -> smem
  if (!pv) {
    for (int i = tid; i < 128 * a_row_bytes; i += 128) {
      int r = i / a_row_bytes, c = i % a_row_bytes;
      sA[swz_offset(r, c, a_row_bytes)] = a[i];
      sB[swz_offset(r, c, a_row_bytes)] = b[i];
    }
  } else if (kind == kSTPvFp8) {
    // V [K keys][128] row-major E4M3: MN-major, 128 B per key row, SW128
    for (int i = tid; i < K * 128; i += 128) {
      int r = i / 128, c = i % 128;
      sB[swz_offset(r, c, 128)] = b[i];
    }
  } else {
    // V [K keys][128] bf16: two 64-column halves, each [K][128 B] SW128, LBO = K*128
    for (int i = tid; i < K * 256; i += 128) {
      int r = i / 256, c = i % 256;
      int half = c / 128;
      sB[half * K * 128 + swz_offset(r, c % 128, 128)] = b[i];
    }
  }
  // scale factors -> 512-byte atoms (r%32)*16 + (r/32)*4 + kb%4, chunk kb/4
  const int nsf = (kind == kSTNvf4) ? K / 16 : K / 32;
  const int chunks = (nsf + 3) / 4;
  if (kind != kSTPvBf16) {
    for (int i = tid; i < 128 * chunks * 4; i += 128) {
      int r = i / (chunks * 4), kb = i % (chunks * 4);
      int off = (kb / 4) * 512 + (r % 32) * 16 + (r / 32) * 4 + (kb % 4);
      sSFA[off] = kb < nsf ? sfa[r * nsf + kb] : 0;
      sSFB[off] = kb < nsf ? sfb[r * nsf + kb] : 0;
    }
  }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_s;
  const uint32_t tD = tmem, tSFA = tmem + 256, tSFB = tmem + 272, tP = tmem + 384;

  // ---- P -> TMEM (row = lane)
  if (pv) {
    const int row = tid;
    const uint32_t lane_addr = tP + ((warp * 32u) << 16);
    const int words = (kind == kSTPvFp8) ? K / 4 : K / 2;
    const uint32_t* src = reinterpret_cast<const uint32_t*>(a) + row * words;
    for (int j = 0; j < words; j += 8) {
      uint32_t r[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) r[i] = src[j + i];
      ptx::tmem_st8(lane_addr + j, r);
    }
    ptx::tmem_st_wait();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();

  if (tid == 0) {
    if (kind != kSTPvBf16) {
      for (int j = 0; j < chunks; ++j) {
        ptx::tc_cp_sf(tSFA + 4 * j, ptx::smem_desc(ptx::smem_u32(sSFA + 512 * j), 0, 128, ptx::kSwNone));
        ptx::tc_cp_sf(tSFB + 4 * j, ptx::smem_desc(ptx::smem_u32(sSFB + 512 * j), 0, 128, ptx::kSwNone));
      }
    }
    const uint32_t sw = a_row_bytes == 128 ? ptx::kSw128 : (a_row_bytes == 64 ? ptx::kSw64 : ptx::kSw32);
    const uint32_t sbo = 8 * a_row_bytes;
    if (kind == kSTMxf8E4M3 || kind == kSTMxf8E5M2) {
      const uint32_t f = kind == kSTMxf8E5M2 ? 1 : 0;
      for (int kk = 0; kk < K / 32; ++kk) {
        uint64_t ad = ptx::smem_desc(ptx::smem_u32(sA) + 32 * kk, 16, sbo, sw);
        uint64_t bd = ptx::smem_desc(ptx::smem_u32(sB) + 32 * kk, 16, sbo, sw);
        uint32_t id = ptx::idesc_bs(f, f, 0, 0, 128, 128, 1, kk & 3, kk & 3);
        ptx::mma_mxf8f6f4(tD, ad, bd, id, tSFA + 4 * (kk >> 2), tSFB + 4 * (kk >> 2), kk > 0);
      }
    } else if (kind == kSTNvf4) {
      for (int kk = 0; kk < K / 64; ++kk) {
        uint64_t ad = ptx::smem_desc(ptx::smem_u32(sA) + 32 * kk, 16, sbo, sw);
        uint64_t bd = ptx::smem_desc(ptx::smem_u32(sB) + 32 * kk, 16, sbo, sw);
        uint32_t id = ptx::idesc_bs(1, 1, 0, 0, 128, 128, 0, 0, 0);
        ptx::mma_nvf4(tD, ad, bd, id, tSFA + 4 * kk, tSFB + 4 * kk, kk > 0);
      }
    } else if (kind == kSTMxf4) {
      for (int kk = 0; kk < K / 64; ++kk) {
        uint64_t ad = ptx::smem_desc(ptx::smem_u32(sA) + 32 * kk, 16, sbo, sw);
        uint64_t bd = ptx::smem_desc(ptx::smem_u32(sB) + 32 * kk, 16, sbo, sw);
        uint32_t sid = (kk & 1) * 2;
        uint32_t id = ptx::idesc_bs(1, 1, 0, 0, 128, 128, 1, sid, sid);
        ptx::mma_mxf4(tD, ad, bd, id, tSFA + 4 * (kk >> 1), tSFB + 4 * (kk >> 1), kk > 0);
      }
    } else if (kind == kSTPvFp8) {
      for (int kk = 0; kk < K / 32; ++kk) {
        uint64_t bd = ptx::smem_desc(ptx::smem_u32(sB) + kk * 32 * 128, 16, 1024, ptx::kSw128);
        uint32_t id = ptx::idesc_bs(0, 0, 0, 1, 128, 128, 1, kk & 3, kk & 3);
        ptx::mma_mxf8f6f4_ts(tD, tP + 8 * kk, bd, id, tSFA + 4 * (kk >> 2), tSFB + 4 * (kk >> 2), kk > 0);
      }
    } else {
      for (int kk = 0; kk < K / 16; ++kk) {
        uint64_t bd = ptx::smem_desc(ptx::smem_u32(sB) + kk * 16 * 128, K * 128, 1024, ptx::kSw128);
        uint32_t id = ptx::idesc_bf16(0, 1, 128, 128);
        ptx::mma_f16_ts(tD, tP + 8 * kk, bd, id, kk > 0);
      }
    }
    ptx::tc_commit(&bar);
  }
  __syncwarp();
  ptx::mbar_wait(&bar, 0);
  ptx::tc_fence_after();

  // ---- D (TMEM) -> global; thread = row
  const uint32_t lane_addr = tD + ((warp * 32u) << 16);
  for (int c = 0; c < 128; c += 32) {
    uint32_t r[32];
    ptx::tmem_ld32(lane_addr + c, r);
    ptx::tmem_ld_wait();
    for (int i = 0; i < 32; ++i) d[tid * 128 + c + i] = __uint_as_float(r[i]);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc<512>(tmem);
}

}  // namespace dma

extern "C" int dma_selftest_mma(int32_t kind, int32_t K, const uint8_t* a, const uint8_t* b, const uint8_t* sfa,
                                const uint8_t* sfb, float* d, void* stream) {
  DMA_CHECK_ARG(kind >= 0 && kind <= 5, "selftest: bad kind %d", kind);
  DMA_CHECK_ARG(K == 64 || K == 128, "selftest: K must be 64 or 128");
  const int smem = 65536 + 4096 + 1024;
  DMA_CUDA_TRY(cudaFuncSetAttribute(dma::selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  dma::selftest_kernel<<<1, 128, smem, static_cast<cudaStream_t>(stream)>>>(kind, K, a, b, sfa, sfb, d);
  DMA_LAUNCH_CHECK();
  return 0;
}
