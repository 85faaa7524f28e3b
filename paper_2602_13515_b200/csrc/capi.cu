#include <stdlib.h>
// capi.cu — library-wide C-ABI entry points: version, thread-local error, device check,
// and the host-side TMA descriptor encoder shared by the attention launchers.
#include <cudaTypedefs.h>
#include <stdarg.h>
#include <string.h>

#include <mutex>

#include "common.cuh"
#include "tma_host.h"


namespace spa2 {

static thread_local char g_last_error[1024] = "";
bool pdl_enabled() {
  static const bool v = [] {
    const char* e = getenv("SPA2_PDL");
    return !(e != nullptr && e[0] == '0');
  }();
  return v;
}


void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int make_tma_bf16_4d(CUtensorMap* map, const void* base, const uint64_t dims[4], const uint64_t strides_elems[3],
                     const uint32_t box[4]) {
  auto fn = encode_fn();
  SPA2_REQUIRE(fn != nullptr, SPA2_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  SPA2_REQUIRE((reinterpret_cast<uintptr_t>(base) & 15) == 0, SPA2_ERR_UNSUPPORTED,
               "TMA operand base pointer must be 16-byte aligned");
  cuuint64_t gdim[4] = {dims[0], dims[1], dims[2], dims[3]};
  cuuint64_t gstride[3];
  for (int i = 0; i < 3; ++i) {
    gstride[i] = strides_elems[i] * 2;
    SPA2_REQUIRE(gstride[i] % 16 == 0 || dims[i + 1] == 1, SPA2_ERR_UNSUPPORTED,
                 "TMA operand strides must be multiples of 8 elements (got %llu)",
                 (unsigned long long)strides_elems[i]);
    if (gstride[i] % 16 != 0) gstride[i] = (gstride[i] + 15) / 16 * 16;  // size-1 axis: unused
  }
  cuuint32_t bx[4] = {box[0], box[1], box[2], box[3]};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), gdim, gstride, bx, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SPA2_REQUIRE(r == CUDA_SUCCESS, SPA2_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return SPA2_OK;
}

int make_tma_bf16_5d(CUtensorMap* map, const void* base, const uint64_t dims[5], const uint64_t strides_bytes[4],
                     const uint32_t box[5]) {
  auto fn = encode_fn();
  SPA2_REQUIRE(fn != nullptr, SPA2_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  SPA2_REQUIRE((reinterpret_cast<uintptr_t>(base) & 15) == 0, SPA2_ERR_UNSUPPORTED,
               "TMA operand base pointer must be 16-byte aligned");
  cuuint64_t gdim[5], gstride[4];
  cuuint32_t bx[5], es[5] = {1, 1, 1, 1, 1};
  for (int i = 0; i < 5; ++i) {
    gdim[i] = dims[i];
    bx[i] = box[i];
  }
  for (int i = 0; i < 4; ++i) {
    gstride[i] = strides_bytes[i];
    if (gstride[i] % 16 != 0) {
      SPA2_REQUIRE(dims[i + 1] == 1, SPA2_ERR_UNSUPPORTED,
                   "TMA operand strides must be multiples of 8 elements (got %llu bytes)",
                   (unsigned long long)strides_bytes[i]);
      gstride[i] = (gstride[i] + 15) / 16 * 16;  // size-1 axis: unused
    }
  }
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), gdim, gstride, bx, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SPA2_REQUIRE(r == CUDA_SUCCESS, SPA2_ERR_CUDA, "cuTensorMapEncodeTiled (5-D) failed (%d)", (int)r);
  return SPA2_OK;
}

int make_tma_bf16_2d(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint64_t row_stride_elems,
                     uint32_t box_cols, uint32_t box_rows) {
  auto fn = encode_fn();
  SPA2_REQUIRE(fn != nullptr, SPA2_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  cuuint64_t gdim[2] = {cols, rows};
  cuuint64_t gstride[1] = {row_stride_elems * 2};
  cuuint32_t bx[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), gdim, gstride, bx, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SPA2_REQUIRE(r == CUDA_SUCCESS, SPA2_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return SPA2_OK;
}

// 2-D map over a row-major [rows][cols] fp32 matrix, no swizzle (row statistics tiles).
int make_tma_f32_2d(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint64_t row_stride_elems,
                    uint32_t box_cols, uint32_t box_rows) {
  auto fn = encode_fn();
  SPA2_REQUIRE(fn != nullptr, SPA2_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  cuuint64_t gdim[2] = {cols, rows};
  cuuint64_t gstride[1] = {row_stride_elems * 4};
  cuuint32_t bx[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), gdim, gstride, bx, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SPA2_REQUIRE(r == CUDA_SUCCESS, SPA2_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return SPA2_OK;
}

}  // namespace spa2

extern "C" const char* spa2_version(void) { return "spa2 0.1.0 sm_100a"; }

extern "C" const char* spa2_last_error(void) { return spa2::g_last_error; }

extern "C" int spa2_device_supported(int device) {
  cudaDeviceProp prop;
  SPA2_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  SPA2_REQUIRE(prop.major == 10 && prop.minor == 0, SPA2_ERR_UNSUPPORTED,
               "device %d is sm_%d%d; libspa2 is built for sm_100a only", device, prop.major, prop.minor);
  return SPA2_OK;
}
