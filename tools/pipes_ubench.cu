// Micro-benchmark of the softmax instruction mix on sm_100a: throughput (ops per
// SM per clock) of ex2.approx.f32, ex2.approx.f16x2, cvt e4m3x2 from f32 / f16x2,
// fma.rn.f32x2, add.f32x2, max3 and the cvt f32->f16x2 pack.  Each thread runs a
// long chain of independent ops over 8 registers; 148 x 4 CTAs of 256 threads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipes tools/pipes_ubench.cu && /tmp/pipes
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

constexpr int kIters = 4096;

template <int OP>
__global__ void bench(float* out, float seed) {
  float r[8];
  uint32_t u[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    r[i] = seed * (threadIdx.x + i) * 1e-3f;
    u[i] = __float_as_uint(r[i]);
  }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) {  // ex2.approx.ftz.f32
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(r[i]));
      } else if (OP == 1) {  // ex2.approx.f16x2 (2 results)
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(u[i]));
      } else if (OP == 2) {  // cvt e4m3x2 <- f32 pair
        uint16_t h;
        asm volatile("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(h) : "f"(r[i]), "f"(r[(i + 1) & 7]));
        r[i] = __uint_as_float(__float_as_uint(r[i]) ^ h);
      } else if (OP == 3) {  // cvt e4m3x2 <- f16x2
        uint16_t h;
        asm volatile("cvt.rn.satfinite.e4m3x2.f16x2 %0, %1;" : "=h"(h) : "r"(u[i]));
        u[i] = (u[i] >> 1) + h;
      } else if (OP == 4) {  // fma.rn.f32x2
        uint64_t a = (uint64_t(u[i]) << 32) | u[(i + 1) & 7];
        asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(a));
        u[i] = uint32_t(a) ^ uint32_t(a >> 32);
      } else if (OP == 5) {  // plain ffma
        r[i] = fmaf(r[i], 1.0001f, 0.5f * r[(i + 3) & 7]);
      } else if (OP == 6) {  // cvt.rn.f16x2.f32 pack
        uint32_t h;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(r[i]), "f"(r[(i + 1) & 7]));
        r[i] = __uint_as_float(h ^ u[i]);
      } else if (OP == 7) {  // 3-input max
        asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(r[i]) : "f"(r[(i + 1) & 7]), "f"(r[(i + 2) & 7]));
      } else if (OP == 8) {  // ex2.approx.ftz.bf16x2
        asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(u[i]));
      }
    }
  }
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc += r[i] + __uint_as_float(u[i]);
  if (acc == 1234.5f) out[0] = acc;
}

template <int OP>
void run(const char* name, float elems_per_op) {
  float* d;
  cudaMalloc(&d, 4);
  const int blocks = 148 * 4, threads = 256;
  bench<OP><<<blocks, threads>>>(d, 1.f);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  bench<OP><<<blocks, threads>>>(d, 1.f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  int clk_khz;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double ops = double(blocks) * threads * kIters * 8;
  const double cyc = ms * 1e-3 * clk_khz * 1e3;  // at the nominal max clock
  printf("%-28s %8.3f ms  %7.1f lane-ops/clk/SM  %7.1f results/clk/SM\n", name, ms, ops / cyc / 148,
         ops * elems_per_op / cyc / 148);
  cudaFree(d);
}

int main() {
  run<0>("ex2.approx.ftz.f32", 1);
  run<1>("ex2.approx.f16x2", 2);
  run<8>("ex2.approx.ftz.bf16x2", 2);
  run<2>("cvt.e4m3x2.f32", 2);
  run<3>("cvt.e4m3x2.f16x2", 2);
  run<4>("fma.rn.f32x2", 2);
  run<5>("ffma", 1);
  run<6>("cvt.rn.f16x2.f32", 2);
  run<7>("max.f32 (3-input)", 1);
  return 0;
}
