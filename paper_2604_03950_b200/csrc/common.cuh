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

// Kernel launch with the programmatic-stream-serialization attribute when `pdl` (the kernel
// may start while the previous kernel in the stream drains; it must ptx::pdl_wait() before
// touching that kernel's results).  pdl_enabled(): env DMA_PDL=0 turns it off (A/B, debug).
bool pdl_enabled();
extern thread_local bool g_pdl_next;  // set around quantize_impl: launch its kernel with PDL
template <typename... KArgs, typename... Args>
inline cudaError_t launch_kernel(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                 cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

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

// Precision / visit status of key tile kj in this plan (the inverse of entry()).
__host__ __device__ inline void plan_status(const Plan& pl, int32_t kj, bool& visited, bool& high) {
  if (pl.causal) {
    visited = kj < pl.n;
    high = (kj < pl.lo0) || (kj >= pl.lo1);
  } else {
    visited = kj < pl.n_tiles;
    high = (kj < pl.n_sink) || (kj >= pl.w0 && kj < pl.w1);
  }
}

// Entries of a 128 x 128 kernel tile walk for a plan with tile_m, tile_n in {64, 128}
// (attention.py:191-233 at the plan's own tile size): for query tile q128 and key tile
// kt the 2 x 2 (or 2 x 1, 1 x 2) plan sub-tiles ("quadrants") are classified
// high / low / unvisited; a key tile gives one entry per precision present, with a
// 4-bit mask (bit 2a + b) of the quadrants the entry keeps -- the softmax sets the
// other quadrants to -inf.  tile_m = tile_n = 128 gives exactly Plan's tiles (in key
// order).  Used by the single-stream kernel; sequential (next()), like every consumer.
struct Plan2 {
  Plan pa[2];
  int32_t ra, rb, nq, n_kt, n;
  int32_t kt, sub;  // generator state
  __host__ __device__ void init(int64_t q128, int64_t len_q, int64_t len_k, int32_t tm, int32_t tn, int32_t T,
                                int32_t S, bool causal) {
    ra = tm == 64 ? 2 : 1;
    rb = tn == 64 ? 2 : 1;
    nq = static_cast<int32_t>(ceil_div(len_q, tm));
    // constant indices only (pa[] must stay in registers, not local memory)
#pragma unroll
    for (int a = 0; a < 2; ++a)
      if (a < ra) pa[a].init(q128 * ra + a, len_q, len_k, tm, tn, T, S, causal);
    n_kt = static_cast<int32_t>(ceil_div(len_k, 128));
    kt = 0;
    sub = 0;
    if (ra == 1 && rb == 1) {  // 128 x 128 plan tiles: the plan itself (no quadrant walk)
      n = pa[0].n;
      return;
    }
    n = 0;
    for (int32_t t = 0; t < n_kt; ++t) {
      uint32_t hm, lm;
      masks(q128, t, hm, lm);
      n += (hm ? 1 : 0) + (lm ? 1 : 0);
    }
    kt = 0;
    sub = 0;
  }
  __host__ __device__ void masks(int64_t q128, int32_t t, uint32_t& hm, uint32_t& lm) const {
    hm = lm = 0u;
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      if (a >= ra || q128 * ra + a >= nq) continue;  // ragged end: no such query sub-tile
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        if (b >= rb) continue;
        bool vis, hi;
        plan_status(pa[a], t * rb + b, vis, hi);
        if (!vis) continue;
        // a 128-row / 128-column plan tile covers both quadrants of its dimension
        uint32_t bits = 0u;
#pragma unroll
        for (int aa = 0; aa < 2; ++aa)
#pragma unroll
          for (int bb = 0; bb < 2; ++bb)
            if ((ra == 2 ? aa == a : true) && (rb == 2 ? bb == b : true)) bits |= 1u << (2 * aa + bb);
        (hi ? hm : lm) |= bits;
      }
    }
  }
  // entry e (callers walk e = 0, 1, 2, ... in order): tile_m = tile_n = 128 keeps the
  // reference's visit order exactly (Plan::entry); otherwise key order.
  __host__ __device__ void entry(int32_t e, int64_t q128, int32_t& t, bool& high, uint32_t& keep) {
    if (ra == 1 && rb == 1) {
      pa[0].entry(e, t, high);
      keep = 0xFu;
      return;
    }
    next(q128, t, high, keep);
  }
  // next entry: key tile t, precision, quadrant keep mask; false when done
  __host__ __device__ bool next(int64_t q128, int32_t& t, bool& high, uint32_t& keep) {
    while (kt < n_kt) {
      uint32_t hm, lm;
      masks(q128, kt, hm, lm);
      if (sub == 0) {
        sub = 1;
        if (hm) {
          t = kt;
          high = true;
          keep = hm;
          return true;
        }
      }
      ++kt;
      sub = 0;
      if (lm) {
        t = kt - 1;
        high = false;
        keep = lm;
        return true;
      }
    }
    return false;
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
// padding slots of the S_q^K block (in the permuted and in the natural layout): 140 = max
// S_q^K of the tile (f32 bits), 141 = ~bits of the min (both written by phase 1 with
// atomicMax on zeroed words; read by attn_sk.cuh)
constexpr int kSqkMaxSlot = 140, kSqkMinSlot = 141;
__host__ __device__ __forceinline__ int perm_slot(int k) { return 36 * ((k >> 3) & 3) + 8 * (k >> 5) + (k & 7); }

}  // namespace dma
