// Shared host/device helpers for libdma.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cstdarg>
#include <cuda_runtime.h>

#include "../../include/dma.h"

namespace dma {

// ---- thread-local error message (dma_last_error)
void set_error(const char* fmt, ...);
const char* get_error();

#define DMA_CHECK_ARG(cond, ...)       \
  do {                                 \
    if (!(cond)) {                     \
      ::dma::set_error(__VA_ARGS__);   \
      return DMA_EINVAL;               \
    }                                  \
  } while (0)

#define DMA_CUDA_TRY(expr)                                                              \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess) {                                                            \
      ::dma::set_error("%s:%d: %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
      return static_cast<int>(_e);                                                      \
    }                                                                                   \
  } while (0)

#define DMA_LAUNCH_CHECK() DMA_CUDA_TRY(cudaGetLastError())

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) {
  // ceil(a / b) for b > 0 and any sign of a
  return (a >= 0) ? (a + b - 1) / b : -((-a) / b);
}

// Integer-exact tile plan (attention.py:191-233).
struct Plan {
  int32_t n;        // number of entries
  int32_t n_sink;   // key tiles [0, n_sink) are sink tiles (high)
  int32_t lo0, lo1; // causal: low span [lo0, lo1); high elsewhere in [0, n)
  int32_t w0, w1;   // non-causal: window [w0, w1) visited last
  int32_t n_tiles;  // non-causal: total key tiles
  bool causal;
  __host__ __device__ void init(int64_t q_tile, int64_t len_q, int64_t len_k, int32_t tm, int32_t tn,
                                int32_t T, int32_t S, bool is_causal) {
    causal = is_causal;
    const int64_t q0 = q_tile * tm;
    if (causal) {
      int64_t q_last = (q0 + tm < len_q ? q0 + tm : len_q) - 1;
      int64_t a = ceil_div(q_last + 1, tn), b = ceil_div(len_k, tn);
      int64_t need = a < b ? a : b;
      int64_t sink = S / tn < need ? S / tn : need;
      int64_t hi = ceil_div(q0 - T, tn);
      hi = hi > sink ? hi : sink;
      hi = hi < need ? hi : need;
      n = static_cast<int32_t>(need);
      n_sink = static_cast<int32_t>(sink);
      lo0 = n_sink;
      lo1 = static_cast<int32_t>(hi);
      w0 = w1 = 0;
      n_tiles = n;
    } else {
      int64_t nt = ceil_div(len_k, tn);
      int64_t sink = S / tn < nt ? S / tn : nt;
      int64_t d0 = ceil_div(2 * q0 - T, 2 * (int64_t)tn);
      d0 = d0 < 0 ? 0 : (d0 > nt ? nt : d0);
      int64_t d1 = ceil_div(2 * q0 + T, 2 * (int64_t)tn);
      d1 = d1 < d0 ? d0 : (d1 > nt ? nt : d1);
      if ((int64_t)T >= 2 * len_k) {
        d0 = 0;
        d1 = nt;
      }
      n = static_cast<int32_t>(nt);
      n_tiles = n;
      n_sink = static_cast<int32_t>(sink);
      w0 = static_cast<int32_t>(d0);
      w1 = static_cast<int32_t>(d1);
      lo0 = lo1 = 0;
    }
  }
  // entry i -> key tile and precision, in the reference's visit order
  __host__ __device__ void entry(int32_t i, int32_t& tile, bool& high) const {
    if (causal) {
      tile = i;
      high = (i < lo0) || (i >= lo1);
    } else {
      int32_t before = w0, after = n_tiles - w1;
      if (i < before) {
        tile = i;
        high = tile < n_sink;
      } else if (i < before + after) {
        tile = w1 + (i - before);
        high = tile < n_sink;
      } else {
        tile = w0 + (i - before - after);
        high = true;
      }
    }
  }
};

// Key permutation of the ping-pong kernel (attn_pp.cuh): inside a 128-key tile,
// key k = 32 G + 8 m + r sits in operand row 8 (4 G + r / 2) + 2 m + r % 2, and its
// S_q^K in slot 36 m + 8 G + r of the tile's 144 (kSqkTile) slots.  (With this order the 16x256b TMEM fragment a
// softmax thread holds covers exactly the keys whose P bytes it stores.)
__host__ __device__ __forceinline__ int perm_row(int k) {
  return 8 * (4 * (k >> 5) + ((k & 7) >> 1)) + 2 * ((k >> 3) & 3) + (k & 1);
}
// S_q^K slots per 128-key tile: 4 groups of 32 (one per m), padded to 36 so the
// four groups start in different shared-memory banks
constexpr int kSqkTile = 144;
__host__ __device__ __forceinline__ int perm_slot(int k) { return 36 * ((k >> 3) & 3) + 8 * (k >> 5) + (k & 7); }

}  // namespace dma
