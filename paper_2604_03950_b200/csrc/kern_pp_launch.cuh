// Launch templates of the ping-pong kernel (attn_pp.cuh), instantiated by kern_pp.cu
// (phase 2 only) and kern_ppf.cu (phase 1 fused in) -- two translation units so the
// instantiations compile in parallel.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "attn_pp.cuh"
#include "common.cuh"
#include "launch.h"

namespace dma {

template <int D, int DV, int LOW, bool FUSE, bool SPLIT>
static int launch_pp(const AttnParams& p, const PPParams& q, const FuseParams& fz, cudaStream_t st) {
  using C = PPCfg<D, DV, LOW>;
  auto kern = dma_attn_pp_kernel<D, DV, LOW, FUSE, SPLIT>;
  static_assert(C::kSmemBytes <= 227 * 1024, "smem budget");
  DMA_SET_SMEM_ONCE(kern, C::kSmemBytes);
  const int grid = q.n_items < num_sms() ? q.n_items : num_sms();
  // PDL: the prologue (barriers, TMEM, descriptor prefetch) overlaps phase 1's tail; the
  // kernel pdl_waits before its first read of phase-1 data (the fused kernel has no
  // producer kernel before it: the attribute is then a no-op)
  DMA_CUDA_TRY(launch_kernel(pdl_enabled() && !FUSE, kern, dim3(static_cast<unsigned>(grid)), dim3(C::kThreads),
                             C::kSmemBytes, st, p, q, fz));
  return 0;
}

template <int D, int DV, bool FUSE, bool SPLIT>
static int dispatch_pp(const AttnParams& p, const PPParams& q, const FuseParams& fz, int low, cudaStream_t st) {
  if (low == kLowNV) return launch_pp<D, DV, kLowNV, FUSE, SPLIT>(p, q, fz, st);
  if (low == kLowMX4) return launch_pp<D, DV, kLowMX4, FUSE, SPLIT>(p, q, fz, st);
  return launch_pp<D, DV, kLowHigh, FUSE, SPLIT>(p, q, fz, st);
}

// SPLIT: the KV-split instantiation (PPParams n_split > 1, small problems); the unsplit
// kernels carry none of its state (the softmax runs at its register limit)
template <bool FUSE, bool SPLIT>
static int run_pp_t(const AttnParams& p, const PPParams& q, const FuseParams& fz, int D, int DV, int low,
                    cudaStream_t st) {
  if (D == 64)
    return DV == 64 ? dispatch_pp<64, 64, FUSE, SPLIT>(p, q, fz, low, st) : dispatch_pp<64, 128, FUSE, SPLIT>(p, q, fz, low, st);
  return DV == 64 ? dispatch_pp<128, 64, FUSE, SPLIT>(p, q, fz, low, st) : dispatch_pp<128, 128, FUSE, SPLIT>(p, q, fz, low, st);
}

}  // namespace dma
