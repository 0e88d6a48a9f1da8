// Hand-written sm_100a PTX wrappers: mbarrier, TMA, tcgen05 (alloc / mma /
// cp / ld / st / commit), UMMA shared-memory and instruction descriptors.
// No CUTLASS/CuTe: the descriptor bit layouts follow the PTX ISA (and match
// cute/arch/mma_sm100_desc.hpp, which we only read as documentation).
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace dma {
namespace ptx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t warp_id() { return threadIdx.x >> 5; }

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// Programmatic dependent launch (PDL).  launch_dependents: this CTA no longer blocks the
// launch of the next kernel in the stream (launched with the programmatic-serialization
// attribute); wait: block until the preceding kernel has completed and its writes are
// visible (returns at once when the kernel was launched without the attribute).
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;"
               ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
#ifndef DMA_WAIT_HINT
#define DMA_WAIT_HINT 0  // > 0: try_wait suspend-time hint in ns (the thread sleeps until the phase completes)
#endif
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
#if DMA_WAIT_HINT > 0
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "n"(DMA_WAIT_HINT)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
#endif
  return ok != 0;
}
#ifdef DMA_DEBUG_WAITS
// per-CTA progress words of the roles (MMA, producer, softmax A, softmax B), printed on a wait timeout
__device__ volatile unsigned int dbg_progress[4 * 1024];
#define DMA_PROGRESS(role, v) do { if ((threadIdx.x & 31) == 0) ::dma::ptx::dbg_progress[blockIdx.x * 4 + (role)] = (v); } while (0)
#else
#define DMA_PROGRESS(role, v) do {} while (0)
#endif
// clock read (deadlock guard) every DMA_SPIN_CHECK spins.  1 measured fastest: the clock
// read slows the spin down, so waiting warps take fewer issue slots from the working ones
// (c3 attention 5.74 ms with 1, 5.80-5.95 ms with 256)
#ifndef DMA_SPIN_CHECK
#define DMA_SPIN_CHECK 1u
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  const long long t0 = clock64();
  uint32_t spins = 0;
  while (!mbar_try_wait(bar, parity)) {
    if ((++spins & (DMA_SPIN_CHECK - 1u)) != 0u) continue;  // deadlock guard: clock read every DMA_SPIN_CHECK spins
#ifdef DMA_DEBUG_WAITS
    if (clock64() - t0 > (1ll << 36)) {  // deadlock guard (~35 s): say which barrier, then fail loudly
      if ((threadIdx.x & 31) == 0)
        printf("dma: mbarrier wait timeout: block %d warp %d smem 0x%x parity %u  progress %08x %08x %08x %08x\n",
               blockIdx.x, threadIdx.x >> 5, smem_u32(bar), parity, dbg_progress[blockIdx.x * 4],
               dbg_progress[blockIdx.x * 4 + 1], dbg_progress[blockIdx.x * 4 + 2], dbg_progress[blockIdx.x * 4 + 3]);
      __trap();
    }
#else
    if (clock64() - t0 > (1ll << 36)) __trap();  // deadlock guard (~35 s): fail loudly, never hang
#endif
  }
}

// ---------------------------------------------------------------- fences
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// per-warpgroup register budget (all 4 warps of the warpgroup execute it)
template <uint32_t N>
__device__ __forceinline__ void setmaxnreg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}
template <uint32_t N>
__device__ __forceinline__ void setmaxnreg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}

// ---------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch_desc(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}
// 3-D tiled load: coords (c0 = innermost, bytes/elements; c1 = row; c2 = matrix)
__device__ __forceinline__ void tma_load_3d(void* smem_dst, const void* tmap, uint64_t* bar,
                                            int32_t c0, int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(smem_u32(smem_dst)), "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)),
        "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// 1-D bulk copy global -> shared (size multiple of 16, 16B aligned)
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(smem_dst)), "l"(reinterpret_cast<uint64_t>(gsrc)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------- TMEM
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_result) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
               ::"r"(smem_u32(smem_result)), "n"(kCols) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}

// tcgen05.commit: arrive on an mbarrier once all prior tcgen05 ops of this thread complete.
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               ::"r"(smem_u32(bar)) : "memory");
}

// L2 prefetch of a contiguous global range (16-byte aligned address, size a multiple of 16)
__device__ __forceinline__ void bulk_prefetch_l2(const void* gsrc, uint32_t bytes) {
  // [gsrc, gsrc + bytes) shrunk to 16-byte boundaries (never touches bytes outside the range)
  const uint64_t a = (reinterpret_cast<uint64_t>(gsrc) + 15) & ~15ull;
  const uint64_t e = (reinterpret_cast<uint64_t>(gsrc) + bytes) & ~15ull;
  if (e > a)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(static_cast<uint32_t>(e - a)) : "memory");
}
// smem -> TMEM copy of one 512-byte scale-factor atom (32 rows x 16 B, broadcast to 4 lane quadrants)
__device__ __forceinline__ void tc_cp_sf(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}

// ----- MMAs (single CTA).  acc != 0 accumulates into D.
__device__ __forceinline__ void mma_mxf8f6f4(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t sfa, uint32_t sfb, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t setp.ne.b32 p, %6, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale.scale_vec::1X [%0], %1, %2, %3, [%4], [%5], p;\n\t}"
      ::"r"(d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(sfa), "r"(sfb), "r"(acc)
      : "memory");
}
// A operand from TMEM
__device__ __forceinline__ void mma_mxf8f6f4_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                                uint32_t sfa, uint32_t sfb, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t setp.ne.b32 p, %6, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale.scale_vec::1X [%0], [%1], %2, %3, [%4], [%5], p;\n\t}"
      ::"r"(d), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(sfa), "r"(sfb), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_nvf4(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t sfa, uint32_t sfb, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t setp.ne.b32 p, %6, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4nvf4.block_scale.scale_vec::4X [%0], %1, %2, %3, [%4], [%5], p;\n\t}"
      ::"r"(d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(sfa), "r"(sfb), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_mxf4(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t sfa, uint32_t sfb, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t setp.ne.b32 p, %6, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%4], [%5], p;\n\t}"
      ::"r"(d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(sfa), "r"(sfb), "r"(acc)
      : "memory");
}
// bf16 x bf16 -> f32, A from TMEM
__device__ __forceinline__ void mma_f16_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                           uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
      ::"r"(d), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_f16_ss(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

// ----- TMEM <-> registers.  32x32b shape: thread t of warp w (w%4 = quadrant q)
// accesses TMEM lane 32q+t; .xN = N consecutive 32-bit columns.
#define DMA_TMEM_LD_32x32b_X16(taddr, r)                                                            \
  asm volatile(                                                                                     \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}," \
      " [%16];"                                                                                     \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),          \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),      \
        "=r"(r[14]), "=r"(r[15])                                                                    \
      : "r"(taddr))

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  DMA_TMEM_LD_32x32b_X16(taddr, r);
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
// 32 columns as four .x8 loads: each needs only 8 consecutive destination registers
// (an .x32 load pins a 32-register aligned block, which a loop-carried fragment
// could not be coalesced with -- the split-KV softmax spilled hundreds of bytes)
__device__ __forceinline__ void tmem_ld32_x8(uint32_t taddr, uint32_t (&r)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[8 * q]), "=r"(r[8 * q + 1]), "=r"(r[8 * q + 2]), "=r"(r[8 * q + 3]), "=r"(r[8 * q + 4]),
                   "=r"(r[8 * q + 5]), "=r"(r[8 * q + 6]), "=r"(r[8 * q + 7])
                 : "r"(taddr + 8 * q));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]),
                 "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
      ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
        "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
      ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
        "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
        "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
// 16x256b shape: thread t of the warp reads lanes (t/4) and (t/4 + 8) of the
// 16-lane block at taddr, columns 2(t mod 4) and 2(t mod 4)+1 of every 8-column
// repetition; per repetition the registers are {lane t/4: col 2m, 2m+1,
// lane t/4+8: col 2m, 2m+1}.  .x16 = 16 repetitions = 128 columns.
__device__ __forceinline__ void tmem_ld_16x256b_x16(uint32_t taddr, uint32_t (&r)[64]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_16x256b_x4(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_st_16x256b_x4(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile("tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
               ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
               : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------- descriptors
// UMMA shared-memory matrix descriptor (sm_100 "version 1").
enum : uint32_t { kSwNone = 0, kSw128 = 2, kSw64 = 4, kSw32 = 6 };

__host__ __device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes,
                                                       uint32_t layout) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // version
  d |= static_cast<uint64_t>(layout & 7) << 61;
  return d;
}

// Instruction descriptor, block-scaled kinds (mxf8f6f4 / mxf4 / mxf4nvf4).
// fmt: mxf8f6f4 -> 0 = E4M3, 1 = E5M2, 5 = E2M1; mxf4/mxf4nvf4 -> 1 = E2M1.
// sf_e8m0: scale format 1 = UE8M0, 0 = UE4M3.
__host__ __device__ __forceinline__ uint32_t idesc_bs(uint32_t afmt, uint32_t bfmt, uint32_t a_mn_major,
                                                      uint32_t b_mn_major, uint32_t M, uint32_t N,
                                                      uint32_t sf_e8m0, uint32_t a_sf_id, uint32_t b_sf_id) {
  uint32_t d = 0;
  d |= (b_sf_id & 3) << 4;
  d |= (afmt & 7) << 7;
  d |= (bfmt & 7) << 10;
  d |= (a_mn_major & 1) << 15;
  d |= (b_mn_major & 1) << 16;
  d |= ((N >> 3) & 0x3F) << 17;
  d |= (sf_e8m0 & 1) << 23;
  d |= ((M >> 4) & 0x1F) << 24;
  d |= (a_sf_id & 3) << 29;
  return d;
}

// Instruction descriptor, kind::f16 (bf16 inputs, f32 accumulator).
__host__ __device__ __forceinline__ uint32_t idesc_bf16(uint32_t a_mn_major, uint32_t b_mn_major, uint32_t M,
                                                        uint32_t N) {
  uint32_t d = 0;
  d |= 1u << 4;   // C = F32
  d |= 1u << 7;   // A = BF16
  d |= 1u << 10;  // B = BF16
  d |= (a_mn_major & 1) << 15;
  d |= (b_mn_major & 1) << 16;
  d |= ((N >> 3) & 0x3F) << 17;
  d |= ((M >> 4) & 0x1F) << 24;
  return d;
}

// explicit shared-memory vector load (generic LD.E would take the long-latency path)
__device__ __forceinline__ float4 lds_f4(uint32_t saddr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(saddr));
  return v;
}

// 3-input max (FMNMX3 on sm_100)
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// ---------------------------------------------------------------- conversions
// f32x2 -> packed e4m3x2 / e5m2x2 / e2m1x2 (RNE, saturate-to-finite).
__device__ __forceinline__ uint16_t cvt_e4m3x2(float lo, float hi) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ uint16_t cvt_e5m2x2(float lo, float hi) {
  uint16_t r;
  asm("cvt.rn.satfinite.e5m2x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ uint8_t cvt_e2m1x2(float lo, float hi) {
  uint32_t r;
  asm("{\n\t.reg .b8 t;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 t, %1, %2;\n\t"
      "cvt.u32.u8 %0, t;\n\t}"
      : "=r"(r)
      : "f"(hi), "f"(lo));
  return static_cast<uint8_t>(r);
}


// ---------------------------------------------------------------- warp-uniform issue
// Versions of the single-thread async ops for code that a whole warp executes in
// lock-step (warp-uniform control flow): elect.sync picks one lane inside the asm,
// so ptxas emits ONE warp-level UTC*/UTMA*/SYNCS instruction with its operands in
// uniform registers -- no per-thread ELECT/BRA.U.ANY loop and no R2UR moves, which
// made a lane-0-only issuer latency-bound (~15 instructions per tcgen05 op).
namespace wu {
#define DMA_WU_ELECT "elect.sync _|e, 0xffffffff;\n\t"
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .pred e;\n\t" DMA_WU_ELECT "@e mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n\t}"
               ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .pred e;\n\t" DMA_WU_ELECT
               "@e mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n\t}"
               ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* smem_dst, const void* tmap, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile("{\n\t.reg .pred e;\n\t" DMA_WU_ELECT
               "@e cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
               " [%0], [%1, {%3, %4, %5}], [%2];\n\t}"
               ::"r"(smem_u32(smem_dst)), "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("{\n\t.reg .pred e;\n\t" DMA_WU_ELECT
               "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n\t}"
               ::"r"(smem_u32(smem_dst)), "l"(reinterpret_cast<uint64_t>(gsrc)), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("{\n\t.reg .pred e;\n\t" DMA_WU_ELECT
               "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
               ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tc_cp_sf(uint32_t taddr, uint64_t sdesc) {
  asm volatile("{\n\t.reg .pred e;\n\t" DMA_WU_ELECT "@e tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;\n\t}"
               ::"r"(taddr), "l"(sdesc) : "memory");
}
#define DMA_WU_MMA(name, kind_str, a_operand, a_constraint, a_type)                                          \
  __device__ __forceinline__ void name(uint32_t d, a_type a, uint64_t bdesc, uint32_t idesc, uint32_t sfa,    \
                                       uint32_t sfb, uint32_t acc) {                                         \
    asm volatile("{\n\t.reg .pred p, e;\n\t setp.ne.b32 p, %6, 0;\n\t" DMA_WU_ELECT                           \
                 "@e tcgen05.mma.cta_group::1." kind_str " [%0], " a_operand ", %2, %3, [%4], [%5], p;\n\t}"    \
                 ::"r"(d), a_constraint(a), "l"(bdesc), "r"(idesc), "r"(sfa), "r"(sfb), "r"(acc)               \
                 : "memory");                                                                                \
  }
DMA_WU_MMA(mma_mxf8f6f4, "kind::mxf8f6f4.block_scale.scale_vec::1X", "%1", "l", uint64_t)
DMA_WU_MMA(mma_mxf8f6f4_ts, "kind::mxf8f6f4.block_scale.scale_vec::1X", "[%1]", "r", uint32_t)
DMA_WU_MMA(mma_nvf4, "kind::mxf4nvf4.block_scale.scale_vec::4X", "%1", "l", uint64_t)
DMA_WU_MMA(mma_mxf4, "kind::mxf4.block_scale.scale_vec::2X", "%1", "l", uint64_t)
#undef DMA_WU_MMA
// bf16 x bf16 -> f32 (kind::f16, no scale factors); A from shared memory or TMEM
__device__ __forceinline__ void mma_f16_ss(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\t setp.ne.b32 p, %4, 0;\n\t" DMA_WU_ELECT
               "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_f16_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\t setp.ne.b32 p, %4, 0;\n\t" DMA_WU_ELECT
               "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               ::"r"(d), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}

// Two chained block-scaled MMAs (K chunks 0 and 1 of one tile) + a commit, from one
// elected lane in one asm block: the second MMA's smem descriptors are the first's +
// dstep (16-byte units), its A/B scale-factor columns + sfstep; idesc1 may differ
// (scale-factor id).  acc0 = accumulate flag of the first MMA (the second accumulates).
#define DMA_WU_MMA2(name, kind_str, a_operand, a_constraint, a_type, a_add)                                  \
  __device__ __forceinline__ void name(uint32_t d, a_type a, uint64_t bdesc, uint32_t idesc0, uint32_t idesc1, \
                                       uint32_t sfa, uint32_t sfb, uint32_t sfstep, uint32_t acc0, uint64_t bstep,\
                                       uint64_t* bar) {                                                        \
    asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b64 b1;\n\t.reg .b32 sa1, sb1;\n\t"                          \
                 a_add                                                                                         \
                 "add.s64 b1, %2, %10;\n\tadd.u32 sa1, %5, %7;\n\tadd.u32 sb1, %6, %7;\n\t"                   \
                 "setp.ne.b32 p, %8, 0;\n\t" DMA_WU_ELECT                                                      \
                 "@e tcgen05.mma.cta_group::1." kind_str " [%0], " a_operand ", %2, %3, [%5], [%6], p;\n\t"    \
                 "@e tcgen05.mma.cta_group::1." kind_str " [%0], a1, b1, %4, [sa1], [sb1], 1;\n\t"              \
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%9];\n\t}"         \
                 ::"r"(d), a_constraint(a), "l"(bdesc), "r"(idesc0), "r"(idesc1), "r"(sfa), "r"(sfb),          \
                   "r"(sfstep), "r"(acc0), "r"(smem_u32(bar)), "l"(bstep)                                      \
                 : "memory");                                                                                  \
  }
// A from shared memory: the second A descriptor is the first + bstep as well
DMA_WU_MMA2(mma2_nvf4_commit, "kind::mxf4nvf4.block_scale.scale_vec::4X", "%1", "l", uint64_t,
            ".reg .b64 a1;\n\tadd.s64 a1, %1, %10;\n\t")
DMA_WU_MMA2(mma2_mxf4_commit, "kind::mxf4.block_scale.scale_vec::2X", "%1", "l", uint64_t,
            ".reg .b64 a1;\n\tadd.s64 a1, %1, %10;\n\t")
#undef DMA_WU_MMA2

// PV: two MXFP8 MMAs with A = P from TMEM (second A block 8 columns on), B = V (MN-major,
// second block bstep further), V scale factors with sf ids in idesc0 / idesc1, then a
// commit when bar != nullptr
template <bool kCommit>
__device__ __forceinline__ void mma2_f8ts_impl(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc0,
                                               uint32_t idesc1, uint32_t sfa, uint32_t sfb, uint32_t acc0,
                                               uint64_t bstep, uint64_t* bar) {
  asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b64 b1;\n\t.reg .b32 a1;\n\t"
               "add.u32 a1, %1, 8;\n\tadd.s64 b1, %2, %9;\n\t"
               "setp.ne.b32 p, %7, 0;\n\t" DMA_WU_ELECT
               "@e tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale.scale_vec::1X [%0], [%1], %2, %3, [%5], [%6], p;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale.scale_vec::1X [%0], [a1], b1, %4, [%5], [%6], 1;\n\t"
               "}"
               ::"r"(d), "r"(a_tmem), "l"(bdesc), "r"(idesc0), "r"(idesc1), "r"(sfa), "r"(sfb), "r"(acc0),
                 "r"(0), "l"(bstep)
               : "memory");
  if (kCommit) tc_commit(bar);
}
__device__ __forceinline__ void mma2_f8ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc0,
                                          uint32_t idesc1, uint32_t sfa, uint32_t sfb, uint32_t acc0,
                                          uint64_t bstep) {
  mma2_f8ts_impl<false>(d, a_tmem, bdesc, idesc0, idesc1, sfa, sfb, acc0, bstep, nullptr);
}
__device__ __forceinline__ void mma2_f8ts_commit(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc0,
                                                 uint32_t idesc1, uint32_t sfa, uint32_t sfb, uint32_t acc0,
                                                 uint64_t bstep, uint64_t* bar) {
  mma2_f8ts_impl<true>(d, a_tmem, bdesc, idesc0, idesc1, sfa, sfb, acc0, bstep, bar);
}
}  // namespace wu

// Low word of a UMMA smem descriptor for a 16-B aligned shared address below 256 KB:
// the start-address field is addr >> 4 (14 bits, never overflows) and the LBO field
// sits above it, so the masks of smem_desc reduce to an add.
__host__ __device__ __forceinline__ uint32_t desc_lo(uint32_t saddr, uint32_t lbo_bytes) {
  return (saddr >> 4) + ((lbo_bytes >> 4) << 16);
}
__host__ __device__ __forceinline__ uint32_t desc_hi(uint32_t sbo_bytes, uint32_t layout) {
  return (sbo_bytes >> 4) | (1u << 14) | ((layout & 7) << 29);
}
__host__ __device__ __forceinline__ uint64_t desc_of(uint32_t lo, uint32_t hi) {
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

}  // namespace ptx
}  // namespace dma
