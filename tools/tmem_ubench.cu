// TMEM read throughput on sm_100a: W warps (W/4 per sub-partition) each load 128
// columns (32x32b.x32 x 4) of their lane quadrant repeatedly; bytes / cycle per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Ipaper_2604_03950_b200/csrc -o tools/tmem_ubench tools/tmem_ubench.cu
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"
using namespace dma;

__global__ void __launch_bounds__(512, 1) k(long long* out, int iters, float* sink) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) ptx::tmem_alloc<512>(&tslot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot + (static_cast<uint32_t>((warp & 3) * 32) << 16);
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[4][32];
#pragma unroll
    for (int c = 0; c < 4; ++c) ptx::tmem_ld32(tmem + 32 * c + 128 * ((warp >> 2) & 3), r[c]);
    ptx::tmem_ld_wait();
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int i = 0; i < 32; i += 8) acc += __uint_as_float(r[c][i]);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  if (acc == 1234.5f) sink[0] = acc;
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc<512>(tslot);
}

int main() {
  long long* d;
  float* s;
  cudaMalloc(&d, 8);
  cudaMalloc(&s, 4);
  for (int warps : {4, 8, 16}) {
    const int iters = 2000;
    k<<<148, warps * 32>>>(d, iters, s);
    long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double bytes = double(warps) * 32 * 128 * 4 * iters;  // per CTA (= per SM)
    printf("warps %2d: %.1f cycles per 16 KB warp-load round, %.1f bytes/clk/SM  %s\n", warps,
           double(h) / iters, bytes / double(h), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
