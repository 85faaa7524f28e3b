// common.cuh — error plumbing and small helpers shared by every libspa2 translation unit.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/spa2.h"

namespace spa2 {

void set_error(const char* fmt, ...);

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace spa2

#define SPA2_REQUIRE(cond, status, ...)      \
  do {                                       \
    if (!(cond)) {                           \
      ::spa2::set_error(__VA_ARGS__);        \
      return (status);                       \
    }                                        \
  } while (0)

#define SPA2_CUDA_TRY(call)                                                              \
  do {                                                                                   \
    cudaError_t err_ = (call);                                                           \
    if (err_ != cudaSuccess) {                                                           \
      ::spa2::set_error("%s failed: %s (%s:%d)", #call, cudaGetErrorString(err_), __FILE__, \
                        __LINE__);                                                       \
      return SPA2_ERR_CUDA;                                                              \
    }                                                                                    \
  } while (0)

#define SPA2_LAUNCH_CHECK() SPA2_CUDA_TRY(cudaPeekAtLastError())

// ---- element loads as double / float ------------------------------------------------
template <typename T>
__device__ __forceinline__ double to_f64(T x);
template <>
__device__ __forceinline__ double to_f64<double>(double x) { return x; }
template <>
__device__ __forceinline__ double to_f64<float>(float x) { return (double)x; }
template <>
__device__ __forceinline__ double to_f64<__nv_bfloat16>(__nv_bfloat16 x) {
  return (double)__bfloat162float(x);
}
template <>
__device__ __forceinline__ double to_f64<__half>(__half x) { return (double)__half2float(x); }

// ---- diagnostic pipeline trace (compiled only with -DSPA2_TRACE, see tools/trace_bwd.py) ----
// SPA2_TR(kind, idx): clock64 of event `kind` for tile / item `idx` of CTA 0, lane 0 of the
// calling warp, into a per-translation-unit device array fetched by spa2_trace_fetch().
#ifdef SPA2_TRACE
#define SPA2_TRACE_SLOTS 2048
#define SPA2_TR(kind, idx)                                                                             \
  do {                                                                                                 \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && (idx) < SPA2_TRACE_SLOTS)                        \
      g_spa2_trace[(kind) * SPA2_TRACE_SLOTS + (idx)] = clock64();                                     \
  } while (0)
#else
#define SPA2_TR(kind, idx) \
  do {                     \
  } while (0)
#endif
// ---- diagnostic per-CTA timing (compiled only with -DSPA2_CTA_TIMES, tools/cta_times.py) ----
// SPA2_CT(kind, slot): thread 0 of the CTA stores globaltimer (slot 0 start of work, 1 end, 3
// kernel entry, 4.. kernel-specific) or its SM id (slot 2) into a per-translation-unit device array fetched by spa2_cta_fetch_{fwd,bwd}().
#ifdef SPA2_CTA_TIMES
#define SPA2_CTA_MAX 4096
#define SPA2_CTA_SLOTS 8
#ifdef SPA2_CTA_CLOCK  // SM cycle counter instead of the global nanosecond timer
#define SPA2_CTA_READ_TIMER(v) asm volatile("mov.u64 %0, %%clock64;" : "=l"(v))
#else
#define SPA2_CTA_READ_TIMER(v) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v))
#endif
#define SPA2_CT_IF(cond, kind, slot)                                                                  \
  do {                                                                                                \
    if ((cond) && blockIdx.x < SPA2_CTA_MAX) {                                                        \
      unsigned long long v_;                                                                          \
      if ((slot) == 2) {                                                                              \
        unsigned s_;                                                                                  \
        asm volatile("mov.u32 %0, %%smid;" : "=r"(s_));                                               \
        v_ = s_;                                                                                      \
      } else {                                                                                        \
        SPA2_CTA_READ_TIMER(v_);                                                                      \
      }                                                                                               \
      g_spa2_cta[((kind) * SPA2_CTA_MAX + blockIdx.x) * SPA2_CTA_SLOTS + (slot)] = v_;                \
    }                                                                                                 \
  } while (0)
#else
#define SPA2_CT_IF(cond, kind, slot) \
  do {                               \
  } while (0)
#endif
// thread 0 of the CTA / lane 0 of the calling warp; SPA2_CTC: the SM cycle counter instead
#ifdef SPA2_CTA_TIMES
#define SPA2_CTC(kind, slot)                                                                          \
  do {                                                                                                \
    if (threadIdx.x == 0 && blockIdx.x < SPA2_CTA_MAX) {                                              \
      unsigned long long v_;                                                                          \
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(v_));                                             \
      g_spa2_cta[((kind) * SPA2_CTA_MAX + blockIdx.x) * SPA2_CTA_SLOTS + (slot)] = v_;                \
    }                                                                                                 \
  } while (0)
#else
#define SPA2_CTC(kind, slot) \
  do {                       \
  } while (0)
#endif
#define SPA2_CT(kind, slot) SPA2_CT_IF(threadIdx.x == 0, kind, slot)
#define SPA2_CTL(kind, slot) SPA2_CT_IF((threadIdx.x & 31) == 0, kind, slot)
// ---- block-list entries -----------------------------------------------------------------
// bits 0-29: block index; bits 30-31: which 64-row half of the 128-row query block keeps the
// tile (masks with b_q = 64): 0 both, 1 the top half (rows 0-63) only, 2 the bottom half only.
__device__ __forceinline__ int list_blk(int32_t e) { return e & 0x3FFFFFFF; }
// true if query row `row` (0..127 within its query block) is NOT part of tile entry e
__device__ __forceinline__ bool list_row_dropped(int32_t e, int row) {
  const uint32_t code = (uint32_t)e >> 30;
  return (code == 1u && row >= 64) || (code == 2u && row < 64);
}
// ---- programmatic dependent launch (PDL) ---------------------------------------------
// Hot-path kernels are launched with programmatic stream serialization: the next kernel's
// CTAs may be scheduled (and run their prologue: barrier init, TMEM alloc, descriptor
// prefetch) while this one drains; pdl_wait() blocks until the previous grid has completed
// and its writes are visible, so it must precede every global-memory access.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

namespace spa2 {
bool pdl_enabled();
// kernel<<<grid, block, smem, stream>>>(args...) with the PDL launch attribute when enabled.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
}  // namespace spa2

