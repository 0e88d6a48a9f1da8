// Issue cost of tcgen05 ops from one warp (warp-uniform, elect inside asm), as used by the
// ping-pong kernel's MMA issuer: cycles per iteration of
//   mode 0: 2 x mma mxf4nvf4 (M=N=128, K=64)        [QK low]
//   mode 1: 2 x tcgen05.cp SF + 2 x mma               [QK low with K scale factors]
//   mode 2: mode 1 + commit + mbarrier wait           [one QK round trip]
//   mode 3: 4 x mma mxf8f6f4 (N=128, K=32), A from TMEM [PV]
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Ipaper_2604_03950_b200/csrc -o tools/umma_ubench tools/umma_ubench.cu
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"
using namespace dma;

template <int MODE>
__global__ void __launch_bounds__(128, 1) k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) ptx::tmem_alloc<512>(&tslot);
  if (threadIdx.x == 32) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_barrier_init();
  }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c3c3c3cu;
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0) {
    const uint32_t sb = ptx::smem_u32(sm);
    const uint64_t dh = static_cast<uint64_t>(ptx::desc_hi(8 * 64, ptx::kSw64)) << 32;
    const uint64_t sfh = static_cast<uint64_t>(ptx::desc_hi(128, ptx::kSwNone)) << 32;
    long long t0 = clock64();
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      if (MODE == 1 || MODE == 2) {
        ptx::wu::tc_cp_sf(tmem + 472, sfh | ptx::desc_lo(sb + 32768, 0));
        ptx::wu::tc_cp_sf(tmem + 476, sfh | ptx::desc_lo(sb + 33280, 0));
      }
      if (MODE <= 2) {
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const uint64_t ad = dh | ptx::desc_lo(sb + 32 * kk, 16);
          const uint64_t bd = dh | ptx::desc_lo(sb + 16384 + 32 * kk, 16);
          ptx::wu::mma_nvf4(tmem, ad, bd, ptx::idesc_bs(1, 1, 0, 0, 128, 128, 0, 0, 0), tmem + 452 + 4 * kk,
                            tmem + 472 + 4 * kk, kk > 0);
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t bd = (static_cast<uint64_t>(ptx::desc_hi(8 * 128, ptx::kSw128)) << 32) |
                              ptx::desc_lo(sb + kk * 32 * 128, 16);
          ptx::wu::mma_mxf8f6f4_ts(tmem + 192, tmem + 128 + 8 * kk, bd, ptx::idesc_bs(0, 0, 0, 1, 128, 128, 1, kk, kk),
                                   tmem + 496, tmem + 488, 1);
        }
      }
      if (MODE == 2) {
        ptx::wu::tc_commit(&bar);
        ptx::mbar_wait(&bar, ph);
        ph ^= 1;
      }
    }
    ptx::wu::tc_commit(&bar);
    ptx::mbar_wait(&bar, ph);
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc<512>(tmem);
}

template <int MODE>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 8);
  auto kern = k<MODE>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int iters : {1, 1000}) {
    kern<<<1, 128, 64 * 1024>>>(d, iters);
    long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    printf("%-40s iters %5d: %8.1f cycles/iter %s\n", name, iters, double(h) / iters,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  cudaFree(d);
}

int main() {
  run<0>("2x mma nvf4 128x128x64");
  run<1>("2x cp SF + 2x mma nvf4");
  run<2>("2x cp + 2x mma + commit + wait");
  run<3>("4x mma mxf8f6f4 A=TMEM 128x128x32");
  return 0;
}
