// Phase-2 launcher: attn_sk.cuh (see launch.h).
#include <cuda.h>
#include <cuda_bf16.h>

#include "attn_sk.cuh"
#include "common.cuh"
#include "launch.h"

namespace dma {

template <int D, int DV, int LOW>
static int launch_sk(const AttnParams& p, const SKParams& q, cudaStream_t st) {
  using C = SKCfg<D, DV, LOW>;
  auto kern = dma_attn_sk_kernel<D, DV, LOW>;
  DMA_SET_SMEM_ONCE(kern, C::kSmemBytes);
  const int grid = q.n_items < num_sms() ? q.n_items : num_sms();
  kern<<<static_cast<unsigned>(grid), C::kThreads, C::kSmemBytes, st>>>(p, q);
  DMA_LAUNCH_CHECK();
  return 0;
}

template <int D, int DV>
static int dispatch_sk(const AttnParams& p, const SKParams& q, int low, cudaStream_t st) {
  if (low == kLowNV) return launch_sk<D, DV, kLowNV>(p, q, st);
  if (low == kLowMX4) return launch_sk<D, DV, kLowMX4>(p, q, st);
  return launch_sk<D, DV, kLowHigh>(p, q, st);
}

int run_sk(const AttnParams& p, const SKParams& q, int D, int DV, int low, cudaStream_t st) {
  if (D == 64) return DV == 64 ? dispatch_sk<64, 64>(p, q, low, st) : dispatch_sk<64, 128>(p, q, low, st);
  return DV == 64 ? dispatch_sk<128, 64>(p, q, low, st) : dispatch_sk<128, 128>(p, q, low, st);
}

}  // namespace dma
