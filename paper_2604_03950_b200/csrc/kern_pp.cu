// Phase-2 launcher: attn_pp.cuh without the fused quantizer (see launch.h).
#include "kern_pp_launch.cuh"

namespace dma {

int run_pp(const AttnParams& p, const PPParams& q, int D, int DV, int low, cudaStream_t st) {
  const FuseParams none{};
  if (q.n_split > 1) return run_pp_split(p, q, D, DV, low, st);
  return run_pp_t<false, false>(p, q, none, D, DV, low, st);
}

}  // namespace dma

#ifdef DMA_PROFILE
// profiling builds only: copy out and clear the ping-pong kernel's phase timers
extern "C" int dma_prof_read(unsigned long long* out, int n) {
  using namespace dma;
  DMA_CUDA_TRY(cudaMemcpyFromSymbol(out, g_prof, sizeof(unsigned long long) * (n < 32 ? n : 32)));
  static const unsigned long long z[32] = {0};
  DMA_CUDA_TRY(cudaMemcpyToSymbol(g_prof, z, sizeof(z)));
  return 0;
}
#endif

#ifdef DMA_TRACE
// tracing builds only: copy out and clear the CTA-0 event trace ([6][4096] + counts)
extern "C" int dma_trace_read(unsigned long long* out, unsigned int* counts) {
  using namespace dma;
  DMA_CUDA_TRY(cudaMemcpyFromSymbol(out, g_trace, sizeof(unsigned long long) * 6 * 4096));
  DMA_CUDA_TRY(cudaMemcpyFromSymbol(counts, g_trace_n, sizeof(unsigned int) * 6));
  static const unsigned int z[6] = {0, 0, 0, 0, 0, 0};
  DMA_CUDA_TRY(cudaMemcpyToSymbol(g_trace_n, z, sizeof(z)));
  return 0;
}
#endif
