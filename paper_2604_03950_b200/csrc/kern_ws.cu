// Phase-2 launcher: attn_ws.cuh (see launch.h).
#include <cuda.h>
#include <cuda_bf16.h>

#include "attn_ws.cuh"
#include "common.cuh"
#include "launch.h"

namespace dma {

template <int D, int DV, int LOW>
static int launch_ws(const AttnParams& p, const SKParams& q, cudaStream_t st) {
  using C = WSCfg<D, DV, LOW>;
  auto kern = dma_attn_ws_kernel<D, DV, LOW>;
  DMA_SET_SMEM_ONCE(kern, C::kSmemBytes);
  const int grid = q.n_items < num_sms() ? q.n_items : num_sms();
  kern<<<static_cast<unsigned>(grid), C::kThreads, C::kSmemBytes, st>>>(p, q);
  DMA_LAUNCH_CHECK();
  return 0;
}

template <int D, int DV>
static int dispatch_ws(const AttnParams& p, const SKParams& q, int low, cudaStream_t st) {
  if (low == kLowNV) return launch_ws<D, DV, kLowNV>(p, q, st);
  if (low == kLowMX4) return launch_ws<D, DV, kLowMX4>(p, q, st);
  return launch_ws<D, DV, kLowHigh>(p, q, st);
}

int run_ws(const AttnParams& p, const SKParams& q, int D, int DV, int low, cudaStream_t st) {
  if (D == 64) return DV == 64 ? dispatch_ws<64, 64>(p, q, low, st) : dispatch_ws<64, 128>(p, q, low, st);
  return DV == 64 ? dispatch_ws<128, 64>(p, q, low, st) : dispatch_ws<128, 128>(p, q, low, st);
}

}  // namespace dma

#ifdef DMA_PROFILE
// phase cycle counters of the ws kernel (-DDMA_PROFILE builds; tools/prof_ws.py)
extern "C" int dma_ws_prof_read(unsigned long long* out, int n) {
  using namespace dma;
  DMA_CUDA_TRY(cudaMemcpyFromSymbol(out, g_prof, sizeof(unsigned long long) * (n < 32 ? n : 32)));
  static const unsigned long long z[32] = {0};
  DMA_CUDA_TRY(cudaMemcpyToSymbol(g_prof, z, sizeof(z)));
  return 0;
}
#endif
