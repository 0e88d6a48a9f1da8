// KV-split instantiations of the ping-pong kernel (attn_pp.cuh SPLIT; small problems, two-phase
// path only: the fused forward stays one launch) and the split merge kernel, in a translation
// unit of their own so they compile in parallel (see launch.h).
#include "kern_pp_launch.cuh"

namespace dma {

int run_pp_split(const AttnParams& p, const PPParams& q, int D, int DV, int low, cudaStream_t st) {
  const FuseParams none{};
  return run_pp_t<false, true>(p, q, none, D, DV, low, st);
}

int run_kv_combine(const AttnParams& p, const float* part, int n_split, int DV, cudaStream_t st) {
  const int lanes = DV / 4, rows_per_cta = 256 / lanes;
  const int64_t blocks = static_cast<int64_t>(p.n_bh) * p.n_qt * (128 / rows_per_cta);
  DMA_CHECK_ARG(blocks < (int64_t(1) << 31), "too many row blocks");
  auto kern = DV == 64 ? kv_combine_kernel<64> : kv_combine_kernel<128>;
  DMA_CUDA_TRY(launch_kernel(pdl_enabled(), kern, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, st, p, part,
                             n_split));
  return 0;
}

}  // namespace dma
