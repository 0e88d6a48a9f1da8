// Kernel launchers of phase 2, one translation unit per kernel family (kern_*.cu) so the
// template instantiations compile in parallel.  Each returns 0 or an error code (message
// via set_error) and launches exactly one kernel on success.
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

#include "attn.cuh"

namespace dma {

// cudaFuncSetAttribute(max dynamic smem) once per kernel instantiation and device: the
// attribute is per device context; a per-instantiation bitmask of devices it was set on
// (devices >= 64 always set it).  Saves a driver call per launch on small problems.
#define DMA_SET_SMEM_ONCE(kern, bytes)                                                        \
  do {                                                                                        \
    static std::atomic<unsigned long long> _dma_attr_mask{0};                                 \
    int _dev = 0;                                                                             \
    cudaGetDevice(&_dev);                                                                     \
    if (_dev >= 64 || !((_dma_attr_mask.load(std::memory_order_relaxed) >> _dev) & 1ull)) {   \
      DMA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (bytes))); \
      if (_dev < 64) _dma_attr_mask.fetch_or(1ull << _dev, std::memory_order_relaxed);        \
    }                                                                                         \
  } while (0)

struct PPParams;
struct FuseParams;
struct SKParams;
int num_sms();
int run_attn(const AttnParams& p, int D, int DV, int low, bool pv_bf16, int64_t items, cudaStream_t st);
int run_pp(const AttnParams& p, const PPParams& q, int D, int DV, int low, cudaStream_t st);
int run_pp_fused(const AttnParams& p, const PPParams& q, const FuseParams& fz, int D, int DV, int low, cudaStream_t st);
int run_pp_split(const AttnParams& p, const PPParams& q, int D, int DV, int low, cudaStream_t st);
int run_kv_combine(const AttnParams& p, const float* part, int n_split, int DV, cudaStream_t st);
int run_sk(const AttnParams& p, const SKParams& q, int D, int DV, int low, cudaStream_t st);
int run_ws(const AttnParams& p, const SKParams& q, int D, int DV, int low, cudaStream_t st);
}  // namespace dma
