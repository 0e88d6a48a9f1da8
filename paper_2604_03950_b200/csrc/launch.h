// Kernel launchers of phase 2, one translation unit per kernel family (kern_*.cu) so the
// template instantiations compile in parallel.  Each returns 0 or an error code (message
// via set_error) and launches exactly one kernel on success.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "attn.cuh"

namespace dma {
struct PPParams;
struct FuseParams;
struct SKParams;
int num_sms();
int run_attn(const AttnParams& p, int D, int DV, int low, bool pv_bf16, int64_t items, cudaStream_t st);
int run_pp(const AttnParams& p, const PPParams& q, int D, int DV, int low, cudaStream_t st);
int run_pp_fused(const AttnParams& p, const PPParams& q, const FuseParams& fz, int D, int DV, int low, cudaStream_t st);
int run_sk(const AttnParams& p, const SKParams& q, int D, int DV, int low, cudaStream_t st);
int run_ws(const AttnParams& p, const SKParams& q, int D, int DV, int low, cudaStream_t st);
}  // namespace dma
