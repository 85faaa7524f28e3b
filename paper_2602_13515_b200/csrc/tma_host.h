// tma_host.h — host-side TMA descriptor encoding (bf16, SWIZZLE_128B, zero OOB fill).
#pragma once
#include <cuda.h>
#include <stdint.h>

namespace spa2 {
// 4-D map over a [dims[3]][dims[2]][dims[1]][dims[0]] bf16 tensor with element strides
// strides_elems = {axis1, axis2, axis3} (axis 0 is contiguous).
int make_tma_bf16_4d(CUtensorMap* map, const void* base, const uint64_t dims[4], const uint64_t strides_elems[3],
                     const uint32_t box[4]);
// 5-D map, strides in BYTES for axes 1..4 (axis 0 contiguous).
int make_tma_bf16_5d(CUtensorMap* map, const void* base, const uint64_t dims[5], const uint64_t strides_bytes[4],
                     const uint32_t box[5]);
// 2-D map over a row-major [rows][cols] bf16 matrix.
int make_tma_bf16_2d(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint64_t row_stride_elems,
                     uint32_t box_cols, uint32_t box_rows);
// 2-D map over a row-major [rows][cols] fp32 matrix, no swizzle.
int make_tma_f32_2d(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint64_t row_stride_elems,
                    uint32_t box_cols, uint32_t box_rows);
}  // namespace spa2

#include "../../include/spa2.h"
namespace spa2 {
// Map over a [B,H,N,d] bf16 view as 5-D (64 columns, N rows, d/64 column chunks, H, B) with a
// (64, rows, d/64, 1, 1) box: ONE request fetches a whole operand tile, landing chunk-major
// ([chunk][row][128 B], SWIZZLE_128B) — the layout the UMMA descriptors expect (defined in fwd.cu).
int make_qkv_map(CUtensorMap* m, const spa2_view& v, int64_t B, int64_t H, int64_t N, int64_t d, int rows);
}  // namespace spa2
