// ptx.cuh — sm_100a primitives: mbarrier pipelines, TMA, tcgen05 MMA / TMEM, UMMA descriptors.
//
// Layout conventions used by every kernel in this library
// -------------------------------------------------------
// Shared-memory operand tiles are stored the way a TMA load with CU_TENSOR_MAP_SWIZZLE_128B
// and a 64-element (128-byte) inner box writes them: a matrix stored row-major as
// [R rows][C bf16 columns] becomes C/64 "column chunks", each [R rows x 128 B] and
// 1024-byte aligned; inside a chunk the 16-byte unit u of row r lives at unit (u ^ (r & 7)).
// The same bytes serve both operand orientations:
//   * K-major operand (rows = M or N, columns = K): SBO = 1024 (8-row group stride); a
//     16-wide K step inside a chunk is +32 bytes on the start address; chunk = +R*128.
//   * MN-major operand (rows = K, columns = M or N): LBO = R*128 (stride between 64-element
//     MN chunks), SBO = 1024 (8-row K group stride); a 16-deep K step is +2048 bytes.
// TMEM accumulators with M = 128 map row m -> lane m; with M = 64 rows [16q, 16q+16) map to
// lanes [32q, 32q+16) (CUTLASS tmem_frg "half subpartition" atom).  TMEM addresses are
// (lane << 16) | column; a warp may only touch lanes [32*(warp%4), 32*(warp%4)+32).
#pragma once

#include <cuda.h>
#include <stdint.h>

// K loops of tcgen05.mma issued as one asm block per loop (one elect for 4-8 MMAs): -2.5 % on the
// dQ kernel.  -DSPA2_NO_MMA_BATCH restores one asm statement per MMA (A/B builds).
#ifndef SPA2_NO_MMA_BATCH
#define SPA2_MMA_BATCH 1
#endif
#ifndef SPA2_WATCHDOG_NS
#define SPA2_WATCHDOG_NS 4000000000ull  // trap instead of hanging if a barrier never flips
#endif

namespace spa2 {
namespace ptx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// ---- mbarrier ----------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ uint32_t mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
#if defined(SPA2_WAIT_TEST)  // diagnostic: non-suspending test_wait polls
  asm volatile(
      "{\n\t.reg .pred P;\n\tmbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
#elif defined(SPA2_WAIT_HINT_NS)
  asm volatile(
      "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity), "n"(SPA2_WAIT_HINT_NS)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
#endif
  return ok;
}
// Non-blocking probe: has the phase with parity `parity` of `bar` completed?
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\tmbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Wait until the phase with parity `parity` of `bar` has completed.  Traps (instead of
// hanging the GPU) if it does not happen within SPA2_WATCHDOG_NS.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  if (mbar_try_wait(addr, parity)) return;
#ifdef SPA2_DEBUG_WAIT
  // diagnostic build: name the stuck barrier after SPA2_WATCHDOG_NS of wall time
  const uint64_t t0 = globaltimer();
  uint32_t spins = 0;
  while (!mbar_try_wait(addr, parity)) {
    if ((++spins & 1023u) == 0 && globaltimer() - t0 > SPA2_WATCHDOG_NS) {
      printf("spa2 watchdog: block %d/%d (%d threads) thread %d stuck on mbarrier smem+%u parity %u\n",
             blockIdx.x, gridDim.x, blockDim.x, threadIdx.x, addr, parity);
      __trap();
    }
  }
#else
  // production: a bare spin with a wall-clock backstop read only every 2^16 failed polls,
  // on the 32-bit nanosecond timer (wrap-safe difference; one register): trap after ~2 s
  // instead of hanging the GPU.  The every-poll timer + printf variant above costs 2-4 % in
  // the hot loops (register pressure, stack).
  uint32_t spins = 0, t0 = 0;
  while (!mbar_try_wait(addr, parity)) {
#ifdef SPA2_WAIT_SLEEP_NS
    if (spins >= 8) __nanosleep(SPA2_WAIT_SLEEP_NS);
#endif
    if ((++spins & 0xFFFFu) == 0) {
      uint32_t now;
      asm volatile("mov.u32 %0, %%globaltimer_lo;" : "=r"(now));
      if (spins == 0x10000u) t0 = now;
      else if (now - t0 > 2000000000u) __trap();
    }
  }
#endif
}

// ---- fences --------------------------------------------------------------------------
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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

// ---- TMA -----------------------------------------------------------------------------
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* src, int c0, int c1,
                                             int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
__device__ __forceinline__ void tma_store_5d(const CUtensorMap* map, const void* src, int c0, int c1, int c2,
                                             int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
__device__ __forceinline__ void tma_store_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void tma_store_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// ---- TMEM allocation -------------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// ---- UMMA descriptors -----------------------------------------------------------------
// Shared-memory matrix descriptor, SWIZZLE_128B, sm100 version bits.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}
// Instruction descriptor: kind::f16 with bf16 A/B, fp32 accumulate.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// D[tmem] (+)= A[smem] · B[smem]ᵀ, issued by one thread.
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[tmem] (+)= A[tmem] · B[smem]ᵀ (A is M lanes x K/2 packed-bf16 columns), one thread.
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive once on `bar` when every MMA previously issued by this thread has completed.
// smem -> TMEM copy of a 128-row x 32-byte slab described by a UMMA smem descriptor: row r
// lands in TMEM lane r, 8 consecutive 32-bit columns (the TMEM A-operand layout of one
// K=16 bf16 step).  Asynchronous; ordered with tcgen05.mma issued by the same thread.
__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// ---- warp-collective issue forms -------------------------------------------------------
// Executed by ALL 32 lanes of a converged warp; one lane is elected inside the asm.  Keeping
// the issuing code warp-uniform lets the compiler hold descriptors in uniform registers and
// drops the per-instruction divergence wrapper: single-thread issue costs ~100 cycles per
// N=64 MMA, more than the tensor pipe needs to execute it (tools/mma_mix.py).
__device__ __forceinline__ void mma_bf16_w(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_bf16_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// A whole K loop of TS-MMAs in ONE asm block with a single elect: D (+)= A[tmem a0 + ks*8 cols]
// · B[b0 + off(ks)], ks = 0..7 (or 0..3), off(ks) = (ks/4)*OFF4 + (ks%4)*OFF1 in 16-byte units.
// Cuts the per-MMA issue sequence (elect, votes, predicate moves) that the one-MMA-per-asm
// form repeats; `acc0` is the accumulate flag of the first step, later steps accumulate.
template <uint32_t A_STEP, uint64_t OFF1, uint64_t OFF4>
__device__ __forceinline__ void mma_bf16_ts_k8_w(uint32_t d_tmem, uint32_t a0, uint64_t b0, uint32_t idesc,
                                                 uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred p, q, e;\n\t.reg .b32 a;\n\t.reg .b64 b;\n\t"
      "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 q, %4, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t"
      "add.u32 a, %1, %5;\n\tadd.s64 b, %2, %6;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, q;\n\t"
      "add.u32 a, %1, %7;\n\tadd.s64 b, %2, %8;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, q;\n\t"
      "add.u32 a, %1, %9;\n\tadd.s64 b, %2, %10;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, q;\n\t"
      "add.u32 a, %1, %11;\n\tadd.s64 b, %2, %12;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, q;\n\t"
      "add.u32 a, %1, %13;\n\tadd.s64 b, %2, %14;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, q;\n\t"
      "add.u32 a, %1, %15;\n\tadd.s64 b, %2, %16;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, q;\n\t"
      "add.u32 a, %1, %17;\n\tadd.s64 b, %2, %18;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, q;\n\t"
      "}" ::"r"(d_tmem),
      "r"(a0), "l"(b0), "r"(idesc), "r"(acc0), "n"(A_STEP), "n"(OFF1), "n"(2 * A_STEP), "n"(2 * OFF1),
      "n"(3 * A_STEP), "n"(3 * OFF1), "n"(4 * A_STEP), "n"(OFF4), "n"(5 * A_STEP), "n"(OFF4 + OFF1),
      "n"(6 * A_STEP), "n"(OFF4 + 2 * OFF1), "n"(7 * A_STEP), "n"(OFF4 + 3 * OFF1)
      : "memory");
}
// TS form, A columns a0 + (ks/2)*A2 + (ks%2)*A1 (operands packed per 32-column group).
template <uint32_t A1, uint32_t A2, uint64_t OFF1, uint64_t OFF4>
__device__ __forceinline__ void mma_bf16_ts_k8p_w(uint32_t d_tmem, uint32_t a0, uint64_t b0, uint32_t idesc,
                                                  uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred p, q, e;\n\t.reg .b32 a;\n\t.reg .b64 b;\n\t"
      "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 q, %4, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t"
      "add.u32 a, %1, %5;\n\tadd.s64 b, %2, %6;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, q;\n\t"
      "add.u32 a, %1, %7;\n\tadd.s64 b, %2, %8;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, q;\n\t"
      "add.u32 a, %1, %9;\n\tadd.s64 b, %2, %10;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, q;\n\t"
      "add.u32 a, %1, %11;\n\tadd.s64 b, %2, %12;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, q;\n\t"
      "add.u32 a, %1, %13;\n\tadd.s64 b, %2, %14;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, q;\n\t"
      "add.u32 a, %1, %15;\n\tadd.s64 b, %2, %16;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, q;\n\t"
      "add.u32 a, %1, %17;\n\tadd.s64 b, %2, %18;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, q;\n\t"
      "}" ::"r"(d_tmem),
      "r"(a0), "l"(b0), "r"(idesc), "r"(acc0), "n"(A1), "n"(OFF1), "n"(A2), "n"(2 * OFF1), "n"(A2 + A1),
      "n"(3 * OFF1), "n"(2 * A2), "n"(OFF4), "n"(2 * A2 + A1), "n"(OFF4 + OFF1), "n"(3 * A2), "n"(OFF4 + 2 * OFF1),
      "n"(3 * A2 + A1), "n"(OFF4 + 3 * OFF1)
      : "memory");
}
// SS form: D (+)= A[a0 + offA(ks)] · B[b0 + offB(ks)], ks = 0..7, off(ks) = (ks/4)*O4 + (ks%4)*O1.
template <uint64_t A1, uint64_t A4, uint64_t B1, uint64_t B4>
__device__ __forceinline__ void mma_bf16_ss_k8_w(uint32_t d_tmem, uint64_t a0, uint64_t b0, uint32_t idesc,
                                                 uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred p, q, e;\n\t.reg .b64 a, b;\n\t"
      "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 q, %4, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "add.s64 a, %1, %5;\n\tadd.s64 b, %2, %6;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, q;\n\t"
      "add.s64 a, %1, %7;\n\tadd.s64 b, %2, %8;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, q;\n\t"
      "add.s64 a, %1, %9;\n\tadd.s64 b, %2, %10;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, q;\n\t"
      "add.s64 a, %1, %11;\n\tadd.s64 b, %2, %12;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, q;\n\t"
      "add.s64 a, %1, %13;\n\tadd.s64 b, %2, %14;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, q;\n\t"
      "add.s64 a, %1, %15;\n\tadd.s64 b, %2, %16;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, q;\n\t"
      "add.s64 a, %1, %17;\n\tadd.s64 b, %2, %18;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, q;\n\t"
      "}" ::"r"(d_tmem),
      "l"(a0), "l"(b0), "r"(idesc), "r"(acc0), "n"(A1), "n"(B1), "n"(2 * A1), "n"(2 * B1), "n"(3 * A1), "n"(3 * B1),
      "n"(A4), "n"(B4), "n"(A4 + A1), "n"(B4 + B1), "n"(A4 + 2 * A1), "n"(B4 + 2 * B1), "n"(A4 + 3 * A1),
      "n"(B4 + 3 * B1)
      : "memory");
}
// TS form with four steps: a = a0 + ks*A_STEP columns, b = b0 + ks*B1.
template <uint32_t A_STEP, uint64_t B1>
__device__ __forceinline__ void mma_bf16_ts_k4_w(uint32_t d_tmem, uint32_t a0, uint64_t b0, uint32_t idesc,
                                                 uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred p, q, e;\n\t.reg .b32 a;\n\t.reg .b64 b;\n\t"
      "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 q, %4, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t"
      "add.u32 a, %1, %5;\n\tadd.s64 b, %2, %6;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, q;\n\t"
      "add.u32 a, %1, %7;\n\tadd.s64 b, %2, %8;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, q;\n\t"
      "add.u32 a, %1, %9;\n\tadd.s64 b, %2, %10;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, q;\n\t"
      "}" ::"r"(d_tmem),
      "r"(a0), "l"(b0), "r"(idesc), "r"(acc0), "n"(A_STEP), "n"(B1), "n"(2 * A_STEP), "n"(2 * B1), "n"(3 * A_STEP),
      "n"(3 * B1)
      : "memory");
}
__device__ __forceinline__ void mma_commit_w(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tmem_cp_128x256b_w(uint32_t taddr, uint64_t sdesc) {
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.cp.cta_group::1.128x256b [%0], %1;\n\t}" ::"r"(
                   taddr),
               "l"(sdesc)
               : "memory");
}
// Warp-uniform mbarrier probe: every lane tests, the vote makes the result provably uniform.
__device__ __forceinline__ bool mbar_test_w(uint64_t* bar, uint32_t parity) {
  return __all_sync(0xffffffffu, mbar_test(bar, parity));
}

// ---- TMEM <-> registers (32 lanes x 32-bit, one row per thread) -----------------------
// Loads include tcgen05.wait::ld so the destination registers are valid on return.
#define SPA2_R8(i) "=r"(r[i]), "=r"(r[i + 1]), "=r"(r[i + 2]), "=r"(r[i + 3]), "=r"(r[i + 4]), \
                   "=r"(r[i + 5]), "=r"(r[i + 6]), "=r"(r[i + 7])
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15},"
      " [%16];\n\ttcgen05.wait::ld.sync.aligned;"
      : SPA2_R8(0), SPA2_R8(8)
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : SPA2_R8(0), SPA2_R8(8), SPA2_R8(16), SPA2_R8(24)
      : "r"(taddr)
      : "memory");
}
// Two 32-column loads in flight, one wait.
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, uint32_t (&r)[64]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%64];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,"
      "%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%65];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : SPA2_R8(0), SPA2_R8(8), SPA2_R8(16), SPA2_R8(24), SPA2_R8(32), SPA2_R8(40), SPA2_R8(48),
        SPA2_R8(56)
      : "r"(taddr), "r"(taddr + 32u)
      : "memory");
}
#undef SPA2_R8
#define SPA2_W8(i) "r"(r[i]), "r"(r[i + 1]), "r"(r[i + 2]), "r"(r[i + 3]), "r"(r[i + 4]), "r"(r[i + 5]), \
                   "r"(r[i + 6]), "r"(r[i + 7])
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      SPA2_W8(0), SPA2_W8(8), SPA2_W8(16), SPA2_W8(24)
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16};" ::"r"(taddr),
      SPA2_W8(0), SPA2_W8(8)
      : "memory");
}
#undef SPA2_W8
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void st_shared_b16(uint32_t addr, uint16_t v) {
  asm volatile("st.shared.b16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ---- math helpers --------------------------------------------------------------------
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x for a pair on the FMA pipe (no MUFU): round-to-nearest split x = n + f, f in
// [-1/2, 1/2], degree-4 minimax polynomial for 2^f (max relative error 2.9e-6, far below
// the bf16 rounding the results go through), exponent added as an integer.  Used for a
// fraction of each row so the MUFU pipe (16 ex2/clk/SM) stops being the softmax limit.
// x below -126 is clamped (result ~1e-38 instead of 0: harmless where it is used).
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 t = __fadd2_rn(x, make_float2(12582912.f, 12582912.f));  // 1.5 * 2^23: rint(x) in the low bits
  const float2 n = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __ffma2_rn(n, make_float2(-1.f, -1.f), x);
  float2 q = __ffma2_rn(make_float2(0.00958312675356865f, 0.00958312675356865f), f,
                        make_float2(0.05590587109327316f, 0.05590587109327316f));
  q = __ffma2_rn(q, f, make_float2(0.24024085700511932f, 0.24024085700511932f));
  q = __ffma2_rn(q, f, make_float2(0.6931242346763611f, 0.6931242346763611f));
  q = __ffma2_rn(q, f, make_float2(1.f, 1.f));
  return make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(q.y) + (__float_as_int(t.y) << 23)));
}
// Two exponentials per MUFU op: ex2.approx.f16x2 on an fp16-rounded argument pair.
__device__ __forceinline__ float2 ex2_f16x2(float2 x) {
  const __half2 h = __float22half2_rn(x);
  uint32_t r;
  asm("ex2.approx.f16x2 %0, %1;" : "=r"(r) : "r"(*reinterpret_cast<const uint32_t*>(&h)));
  return __half22float2(*reinterpret_cast<const __half2*>(&r));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// Byte offset of 16-byte unit `u` of row `r` inside a SWIZZLE_128B chunk.
__device__ __forceinline__ uint32_t sw128_offset(uint32_t r, uint32_t u) {
  return r * 128u + ((u ^ (r & 7u)) << 4);
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
__device__ __forceinline__ uint4 ld_shared_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}

// Dynamic shared memory base, rounded up to 1 KB (SWIZZLE_128B tiles and UMMA descriptors
// need it).  The runtime only guarantees a small alignment for the dynamic window: a CTA that
// shares its SM with CTAs of another kernel (programmatic dependent launch overlap, two CTAs
// per SM) can start at any 128-byte boundary, so every kernel reserves kSmemAlignSlack extra.
constexpr int kSmemAlignSlack = 1024;
__device__ __forceinline__ uint8_t* smem_align_1k(uint8_t* p) {
  const uint32_t a = smem_u32(p);
  return p + (((a + 1023u) & ~1023u) - a);
}

}  // namespace ptx
}  // namespace spa2
