// Phase-2 launcher: attn.cuh (see launch.h).
#include <cuda.h>
#include <cuda_bf16.h>

#include "attn.cuh"
#include "common.cuh"
#include "launch.h"

namespace dma {

template <int D, int DV, int LOW, bool PVBF16>
static int launch_attn(const AttnParams& p, int64_t items, cudaStream_t st) {
  using C = AttnCfg<D, DV, LOW, PVBF16>;
  auto kern = dma_attn_kernel<D, DV, LOW, PVBF16>;
  const int smem = C::kSmemBytes > 120 * 1024 ? C::kSmemBytes : 120 * 1024;  // one CTA per SM (TMEM 512 cols)
  DMA_SET_SMEM_ONCE(kern, smem);
  // persistent: one CTA per SM, items strided across CTAs (longest first)
  const int64_t grid = items < num_sms() ? items : num_sms();
  kern<<<static_cast<unsigned>(grid), 384, smem, st>>>(p);
  DMA_LAUNCH_CHECK();
  return 0;
}

template <int D, int DV>
static int dispatch_attn(const AttnParams& p, int low, bool pv_bf16, int64_t items, cudaStream_t st) {
  if (low == kLowBF16) return pv_bf16 ? launch_attn<D, DV, kLowBF16, true>(p, items, st) : launch_attn<D, DV, kLowBF16, false>(p, items, st);
  if (low == kLowNV) return pv_bf16 ? launch_attn<D, DV, kLowNV, true>(p, items, st) : launch_attn<D, DV, kLowNV, false>(p, items, st);
  if (low == kLowMX4) return pv_bf16 ? launch_attn<D, DV, kLowMX4, true>(p, items, st) : launch_attn<D, DV, kLowMX4, false>(p, items, st);
  return pv_bf16 ? launch_attn<D, DV, kLowHigh, true>(p, items, st) : launch_attn<D, DV, kLowHigh, false>(p, items, st);
}

int run_attn(const AttnParams& p, int D, int DV, int low, bool pv_bf16, int64_t items, cudaStream_t st) {
  if (D == 64) return DV == 64 ? dispatch_attn<64, 64>(p, low, pv_bf16, items, st) : dispatch_attn<64, 128>(p, low, pv_bf16, items, st);
  return DV == 64 ? dispatch_attn<128, 64>(p, low, pv_bf16, items, st) : dispatch_attn<128, 128>(p, low, pv_bf16, items, st);
}

}  // namespace dma
