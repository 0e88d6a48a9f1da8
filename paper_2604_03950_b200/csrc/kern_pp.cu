// Phase-2 launcher: attn_pp.cuh without the fused quantizer (see launch.h).
#include "kern_pp_launch.cuh"

namespace dma {

int run_pp(const AttnParams& p, const PPParams& q, int D, int DV, int low, cudaStream_t st) {
  const FuseParams none{};
  return run_pp_t<false>(p, q, none, D, DV, low, st);
}

}  // namespace dma
