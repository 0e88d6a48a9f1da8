// Is F2FP (cvt e4m3x2) on the same pipe as MUFU.EX2?  Times MUFU-only, F2FP-only and the
// 2:1 mix of the softmax inner loop; additive times => shared pipe.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipes_mix tools/pipes_mix.cu
#include <cstdio>
#include <cstdint>
constexpr int kIters = 2048;
template <int MODE>
__global__ void k(float* out, float seed) {
  float r[16];
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = seed * (threadIdx.x + i) * 1e-3f;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      if (MODE & 1) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(r[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(r[i + 1]));
      }
      if (MODE & 2) {
        uint16_t h;
        asm volatile("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(h) : "f"(r[i]), "f"(r[i + 1]));
        acc += h;
      }
      if (MODE & 4) {  // FFMA2 pair
        asm volatile("{.reg .b64 t; mov.b64 t, {%0, %1}; fma.rn.f32x2 t, t, t, t; mov.b64 {%0, %1}, t;}"
                     : "+f"(r[i]), "+f"(r[i + 1]));
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += r[i];
  if (s == 1234.5f || acc == 77) out[0] = s + acc;
}
template <int MODE>
float run(int warps_per_smsp) {
  float* d;
  cudaMalloc(&d, 4);
  const int threads = 128 * warps_per_smsp, blocks = 148;
  k<MODE><<<blocks, threads>>>(d, 1.f);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<MODE><<<blocks, threads>>>(d, 1.f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(d);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  // cycles per (warp, 16-element group iteration) per SMSP
  const double cyc = ms * 1e-3 * clk * 1e3;
  return cyc / (double(kIters) * warps_per_smsp);
}
int main() {
  for (int w : {1, 2, 4}) {
    printf("warps/SMSP=%d  cycles per 16 elements/warp: MUFU %.1f  F2FP %.1f  MUFU+F2FP %.1f  FFMA2 %.1f  MUFU+FFMA2 %.1f  all %.1f\n",
           w, run<1>(w), run<2>(w), run<3>(w), run<4>(w), run<5>(w), run<7>(w));
  }
  return 0;
}
