// Launcher of the fused forward: attn_pp.cuh with phase 1 (quantize_dual of bf16 Q / K,
// MXFP8 V) inside the same kernel (see launch.h).
#include "kern_pp_launch.cuh"

namespace dma {

int run_pp_fused(const AttnParams& p, const PPParams& q, const FuseParams& fz, int D, int DV, int low, cudaStream_t st) {
  // the fused forward is one launch: never split (dma_attention_fwd forces n_split = 1)
  return run_pp_t<true, false>(p, q, fz, D, DV, low, st);
}

}  // namespace dma
