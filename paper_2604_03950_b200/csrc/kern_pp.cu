// Phase-2 launcher: attn_pp.cuh (see launch.h).
#include <cuda.h>
#include <cuda_bf16.h>

#include "attn_pp.cuh"
#include "common.cuh"
#include "launch.h"

namespace dma {

template <int D, int DV, int LOW>
static int launch_pp(const AttnParams& p, const PPParams& q, cudaStream_t st) {
  using C = PPCfg<D, DV, LOW>;
  auto kern = dma_attn_pp_kernel<D, DV, LOW>;
  static_assert(C::kSmemBytes <= 227 * 1024, "smem budget");
  DMA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes));
  const int grid = q.n_pairs < num_sms() ? q.n_pairs : num_sms();
  kern<<<static_cast<unsigned>(grid), C::kThreads, C::kSmemBytes, st>>>(p, q);
  DMA_LAUNCH_CHECK();
  return 0;
}

template <int D, int DV>
static int dispatch_pp(const AttnParams& p, const PPParams& q, int low, cudaStream_t st) {
  if (low == kLowNV) return launch_pp<D, DV, kLowNV>(p, q, st);
  if (low == kLowMX4) return launch_pp<D, DV, kLowMX4>(p, q, st);
  return launch_pp<D, DV, kLowHigh>(p, q, st);
}

int run_pp(const AttnParams& p, const PPParams& q, int D, int DV, int low, cudaStream_t st) {
  if (D == 64) return DV == 64 ? dispatch_pp<64, 64>(p, q, low, st) : dispatch_pp<64, 128>(p, q, low, st);
  return DV == 64 ? dispatch_pp<128, 64>(p, q, low, st) : dispatch_pp<128, 128>(p, q, low, st);
}

}  // namespace dma
