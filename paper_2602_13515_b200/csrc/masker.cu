// masker.cu — K1 pooled map, K2 select, K3 block lists (CUDA cores, HBM/L2-bound).
//
// Reference stages replaced (paths under /root/reference/pkg/src/sparseattn_lab):
//   K1  numerics.block_mean_pool (numerics.py:55-65), masker.pooled_map (masker.py:100-110),
//       numerics.softmax_rows (numerics.py:46-52)
//   K2  masker._descending_order .. hybrid_mask (masker.py:113-146)
//   K3  the row-major kept-block iteration of attention.py:97/151-157 and its KV-major
//       transpose for the backward.
//
// Everything after the bf16 load is IEEE float64, so the pooled map agrees with the
// reference to ~1e-16 relative and the block selection is bit-exact for a given map.
#include <math.h>
#include <stdlib.h>

#include <algorithm>
#include <type_traits>

#include "common.cuh"

namespace spa2 {
namespace {

// ---------------------------------------------------------------------------------------
// K1a: block-mean pooling of Q (by b_q) and K (by b_kv) in float64.
// One thread per (b, h, block, group of CPT columns): it walks the block's rows in order
// and accumulates in float64 starting from the first row — the same left-to-right order
// numpy's add.reduceat uses along axis 0 — then divides by the true row count
// (numerics.py:62-65).  Rows are read 16 bytes at a time with 8 loads in flight.
// ---------------------------------------------------------------------------------------
template <typename T, int CPT>
__global__ void __launch_bounds__(256) k_pool(spa2_view q, spa2_view k, int H, int N, int d, int b_q, int b_kv,
                                              int T_m, int T_n, int64_t BH, double* __restrict__ qbar,
                                              double* __restrict__ kbar, int32_t* __restrict__ nonfinite) {
  const int cpr = d / CPT;  // threads per block row
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nq = BH * T_m * cpr, nk = BH * T_n * cpr;
  bool bad = false;
  if (gid < nq + nk) {
    const bool is_q = gid < nq;
    const int64_t gl = is_q ? gid : gid - nq;
    const int cg = (int)(gl % cpr);
    const int64_t blk_g = gl / cpr;
    const int nblk = is_q ? T_m : T_n;
    const int64_t bh = blk_g / nblk;
    const int blk = (int)(blk_g % nblk);
    const int bsz = is_q ? b_q : b_kv;
    const spa2_view vw = is_q ? q : k;
    const int row0 = blk * bsz;
    const int rows = min(bsz, N - row0);
    const T* base = reinterpret_cast<const T*>(vw.ptr) + (bh / H) * vw.sb + (bh % H) * vw.sh +
                    (int64_t)row0 * vw.sn + cg * CPT;
    double acc[CPT];
#pragma unroll
    for (int e = 0; e < CPT; ++e) acc[e] = 0.0;
    constexpr int U = 8;
    for (int r0 = 0; r0 < rows; r0 += U) {
      T buf[U][CPT];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (r0 + u < rows) {
          const T* p = base + (int64_t)(r0 + u) * vw.sn;
          if constexpr (CPT * sizeof(T) == 16) {
            *reinterpret_cast<uint4*>(buf[u]) = __ldg(reinterpret_cast<const uint4*>(p));
          } else {
#pragma unroll
            for (int e = 0; e < CPT; ++e) buf[u][e] = p[e];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (r0 + u < rows) {
#pragma unroll
          for (int e = 0; e < CPT; ++e) {
            double x;
            if constexpr (std::is_same<T, __nv_bfloat16>::value) {
              // non-finite test on the bf16 bits (exponent all ones) instead of on the double
              bad |= (__bfloat16_as_ushort(buf[u][e]) & 0x7F80u) == 0x7F80u;
              x = (double)__bfloat162float(buf[u][e]);
            } else {
              x = to_f64<T>(buf[u][e]);
              bad |= !isfinite(x);
            }
            acc[e] += x;
          }
        }
      }
    }
    double* out = (is_q ? qbar : kbar) + blk_g * (int64_t)d + cg * CPT;
#pragma unroll
    for (int e = 0; e < CPT; ++e) out[e] = acc[e] / (double)rows;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0 && nonfinite != nullptr) *nonfinite = 1;
}

// ---------------------------------------------------------------------------------------
// K1a (bf16, default): the k_pool mapping (one thread per (block, 8 columns), rows added in
// order into 8 float64 chains) with the row loads software-pipelined: the next 8 rows are in
// flight while the current 8 are added, so twice the bytes are outstanding per thread.
// ---------------------------------------------------------------------------------------
// Streaming loads for the pooling pass (each byte of Q and K is read exactly once): not
// allocating in L1 took K1 (pooling + scores) from 69.0 to 63.4 us at the bench shape
// (tools/masker_time.py; the L2 prefetch-size hint made no difference).
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
#define POOL_LD(p) ld_stream(p)
__global__ void __launch_bounds__(256) k_pool_bf16_pipe(spa2_view q, spa2_view k, int H, int N, int d, int b_q,
                                                        int b_kv, int T_m, int T_n, int64_t BH,
                                                        double* __restrict__ qbar, double* __restrict__ kbar,
                                                        int32_t* __restrict__ nonfinite) {
  pdl_wait();
  pdl_trigger();
  constexpr int U = 8;
  const int cpr = d / 8;
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nq = BH * T_m * cpr, nk = BH * T_n * cpr;
  uint32_t badbits = 0;
  if (gid < nq + nk) {
    const bool is_q = gid < nq;
    const int64_t gl = is_q ? gid : gid - nq;
    const int cg = (int)(gl % cpr);
    const int64_t blk_g = gl / cpr;
    const int nblk = is_q ? T_m : T_n;
    const int64_t bh = blk_g / nblk;
    const int blk = (int)(blk_g % nblk);
    const int bsz = is_q ? b_q : b_kv;
    const spa2_view vw = is_q ? q : k;
    const int row0 = blk * bsz;
    const int rows = min(bsz, N - row0);
    const uint4* base = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(vw.ptr) +
                                                       (bh / H) * vw.sb + (bh % H) * vw.sh + (int64_t)row0 * vw.sn +
                                                       cg * 8);
    const int64_t rs = vw.sn / 8;  // row stride in uint4
    double acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.0;
    uint4 cur[U], nxt[U];
#pragma unroll
    for (int u = 0; u < U; ++u) cur[u] = u < rows ? POOL_LD(base + u * rs) : make_uint4(0, 0, 0, 0);
    for (int r0 = 0; r0 < rows; r0 += U) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        nxt[u] = (r0 + U + u < rows) ? POOL_LD(base + (int64_t)(r0 + U + u) * rs) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (r0 + u < rows) {
          const uint32_t w[4] = {cur[u].x, cur[u].y, cur[u].z, cur[u].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            badbits |= ((w[e] & 0x7F80u) == 0x7F80u) | ((w[e] & 0x7F800000u) == 0x7F800000u);
            acc[2 * e] += (double)__uint_as_float(w[e] << 16);
            acc[2 * e + 1] += (double)__uint_as_float(w[e] & 0xFFFF0000u);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) cur[u] = nxt[u];
    }
    double* out = (is_q ? qbar : kbar) + blk_g * (int64_t)d + cg * 8;
#pragma unroll
    for (int e = 0; e < 8; ++e) out[e] = acc[e] / (double)rows;
  }
  if (__any_sync(0xffffffffu, badbits != 0) && (threadIdx.x & 31) == 0 && nonfinite != nullptr) *nonfinite = 1;
}

// ---------------------------------------------------------------------------------------
// K0: finiteness scan of one [B, H, N, d] bf16 operand (the reference's ensure_finite,
// numerics.py:29-32, for the tensors K1 does not read: v, dO).  Grid-stride over groups of
// kK0Unroll 16-byte chunks per thread, all loads issued before any is tested (HBM-bound:
// one pass over the operand); a NaN/Inf (exponent bits all ones) sets *nonfinite = 1 with
// a plain store, so the flag may live in mapped pinned host memory (no atomics over PCIe).
// ---------------------------------------------------------------------------------------
constexpr int kK0Unroll = 8;
#define K0_LD(p) __ldg(p)  // (the streaming form of the pooling loads measured 3 % slower here)
__global__ void __launch_bounds__(256) k_nonfinite_bf16(spa2_view x, int H, int N, int cpr_log2,
                                                        int32_t* __restrict__ nonfinite) {
  pdl_wait();
  pdl_trigger();
  // blockIdx.y = (b, h); chunk c of the head -> row c >> cpr_log2, column chunk c & (cpr - 1):
  // 32-bit index math only (64-bit divisions per chunk made this kernel ALU-bound)
  const int bh = blockIdx.y;
  const __nv_bfloat16* base = reinterpret_cast<const __nv_bfloat16*>(x.ptr) + (int64_t)(bh / H) * x.sb +
                              (int64_t)(bh % H) * x.sh;
  const int chunks = N << cpr_log2;
  const int cmask = (1 << cpr_log2) - 1;
  const int stride = gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (int c0 = blockIdx.x * blockDim.x + threadIdx.x; c0 < chunks; c0 += stride * kK0Unroll) {
    uint4 v[kK0Unroll];
#pragma unroll
    for (int u = 0; u < kK0Unroll; ++u) {
      const int c = c0 + u * stride;
      v[u] = c < chunks ? K0_LD(reinterpret_cast<const uint4*>(base + (int64_t)(c >> cpr_log2) * x.sn + (c & cmask) * 8))
                        : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < kK0Unroll; ++u) {
      const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
        acc |= (((w[i] & 0x7F80u) == 0x7F80u) | ((w[i] & 0x7F800000u) == 0x7F800000u)) ? 1u : 0u;
    }
  }
  if (__any_sync(0xffffffffu, acc != 0) && (threadIdx.x & 31) == 0) *nonfinite = 1;
}

// ---------------------------------------------------------------------------------------
// K1b: scores S = Q̄ K̄ᵀ / √d in float64 (written into `probs`).  64x64 output tiles, 256
// threads, each owning the 4x4 outputs (ty + 16x, tx + 16y): a warp reads 2 Q̄ rows
// (broadcast) and 16 consecutive K̄ rows per k step, so with a 33-double row pitch the
// shared-memory reads are conflict-free and the fp64 pipe, not the LSU, is the limit.
// ---------------------------------------------------------------------------------------
constexpr int kSTI = 64, kSTJ = 64, kSTK = 32, kSTP = kSTK + 1;

__device__ __forceinline__ void cp_async_f64(double* dst, const double* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(valid ? 8 : 0)
               : "memory");
}

__global__ void __launch_bounds__(256, 3) k_scores(const double* __restrict__ qbar,
                                                   const double* __restrict__ kbar, int T_m, int T_n,
                                                   int d, double sqrt_d, double* __restrict__ s_out) {
  pdl_wait();
  pdl_trigger();
  // two k-chunk buffers: chunk c+1 streams in (cp.async) while chunk c is multiplied
  extern __shared__ double sc_smem[];  // [2][sq 64 x 33 | sk 64 x 33]
  const int64_t bh = blockIdx.z;
  const int i0 = blockIdx.y * kSTI, j0 = blockIdx.x * kSTJ;
  const double* qb = qbar + bh * (int64_t)T_m * d;
  const double* kb = kbar + bh * (int64_t)T_n * d;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  auto load = [&](int c0, int buf) {
    double* sq = sc_smem + buf * 2 * kSTI * kSTP;
    double* sk = sq + kSTI * kSTP;
#pragma unroll
    for (int e = threadIdx.x; e < kSTI * kSTK; e += 256) {
      const int rr = e / kSTK, cc = e % kSTK;
      const int i = i0 + rr, j = j0 + rr, c = c0 + cc;
      const bool vq = i < T_m && c < d, vk = j < T_n && c < d;
      cp_async_f64(&sq[rr * kSTP + cc], vq ? qb + (int64_t)i * d + c : qb, vq);
      cp_async_f64(&sk[rr * kSTP + cc], vk ? kb + (int64_t)j * d + c : kb, vk);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc[4][4] = {};
  const int nch = (d + kSTK - 1) / kSTK;
  load(0, 0);
  for (int ch = 0; ch < nch; ++ch) {
    if (ch + 1 < nch) {
      load((ch + 1) * kSTK, (ch + 1) & 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const double* sq = sc_smem + (ch & 1) * 2 * kSTI * kSTP;
    const double* sk = sq + kSTI * kSTP;
#pragma unroll 8
    for (int cc = 0; cc < kSTK; ++cc) {
      double a[4], b[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) a[x] = sq[(ty + 16 * x) * kSTP + cc];
#pragma unroll
      for (int y = 0; y < 4; ++y) b[y] = sk[(tx + 16 * y) * kSTP + cc];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = fma(a[x], b[y], acc[x][y]);
    }
    __syncthreads();  // buffer (ch & 1) is refilled by the load issued in iteration ch + 1
  }
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int i = i0 + ty + 16 * x;
    if (i >= T_m) continue;
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int j = j0 + tx + 16 * y;
      if (j < T_n) s_out[(bh * T_m + i) * (int64_t)T_n + j] = acc[x][y] / sqrt_d;
    }
  }
}
constexpr int kScoresSmem = 2 * 2 * kSTI * kSTP * 8;

// K1b on the fp64 tensor cores (default): DMMA m8n8k4 (mma.sync .f64).  CTA = 64 x 64 outputs,
// 4 warps each owning 32 x 32 (4 x 4 DMMA tiles, 32 fp64 accumulators per thread); k chunks of
// 32 staged by 16-byte cp.async into a 36-double pitch, so the fragment loads (8 rows x 4
// consecutive k per DMMA operand) are conflict-free.  The fp64 FMA rate is the same as the
// DFMA pipe's, but a DMMA needs 1 shared-memory wavefront per 256 FMAs instead of ~4, so the
// kernel is no longer bound by the LSU (k_scores, 70 % L1 throughput).  Results differ from
// k_scores only in fp64 summation order (<= 1e-16 relative; the map's tolerance is 1e-13).
constexpr int kDmK = 32, kDmP = 36;
constexpr int kDmSmem = 2 * 2 * 64 * kDmP * 8;

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}

__global__ void __launch_bounds__(128, 3) k_scores_dmma(const double* __restrict__ qbar,
                                                        const double* __restrict__ kbar, int T_m, int T_n, int d,
                                                        double inv_sqrt_d, double* __restrict__ s_out) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ double dm_smem[];  // [2 bufs][sq 64 x 36 | sk 64 x 36]
  const int64_t bh = blockIdx.z;
  const int i0 = blockIdx.y * 64, j0 = blockIdx.x * 64;
  const double* qb = qbar + bh * (int64_t)T_m * d;
  const double* kb = kbar + bh * (int64_t)T_n * d;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int wi = (warp >> 1) * 32, wj = (warp & 1) * 32;  // warp tile origin inside the CTA tile
  const int fr = lane >> 2, fk = lane & 3;                // fragment row / k of this lane
  auto load = [&](int c0, int buf) {
    double* sq = dm_smem + buf * 2 * 64 * kDmP;
    double* sk = sq + 64 * kDmP;
    // 64 rows x 32 doubles per operand = 512 chunks of 16 B each; 128 threads x 4
#pragma unroll
    for (int e = threadIdx.x; e < 64 * (kDmK / 2); e += 128) {
      const int rr = e / (kDmK / 2), cc = (e % (kDmK / 2)) * 2;
      const int i = i0 + rr, j = j0 + rr, c = c0 + cc;
      const bool vq = i < T_m && c < d, vk = j < T_n && c < d;
      cp_async16(&sq[rr * kDmP + cc], vq ? qb + (int64_t)i * d + c : qb, vq);
      cp_async16(&sk[rr * kDmP + cc], vk ? kb + (int64_t)j * d + c : kb, vk);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc[4][4][2];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  const int nch = (d + kDmK - 1) / kDmK;
  load(0, 0);
  for (int ch = 0; ch < nch; ++ch) {
    if (ch + 1 < nch) {
      load((ch + 1) * kDmK, (ch + 1) & 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const double* sq = dm_smem + (ch & 1) * 2 * 64 * kDmP;
    const double* sk = sq + 64 * kDmP;
#pragma unroll
    for (int k0 = 0; k0 < kDmK; k0 += 4) {
      double a[4], b[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) a[x] = sq[(wi + 8 * x + fr) * kDmP + k0 + fk];
#pragma unroll
      for (int y = 0; y < 4; ++y) b[y] = sk[(wj + 8 * y + fr) * kDmP + k0 + fk];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(acc[x][y][0]), "+d"(acc[x][y][1])
                       : "d"(a[x]), "d"(b[y]));
    }
    __syncthreads();  // buffer (ch & 1) is refilled by the load issued in iteration ch + 1
  }
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int i = i0 + wi + 8 * x + fr;
    if (i >= T_m) continue;
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int j = j0 + wj + 8 * y + fk * 2;
      double* dst = s_out + (bh * T_m + i) * (int64_t)T_n + j;
      if (j + 1 < T_n && ((T_n & 1) == 0)) {
        *reinterpret_cast<double2*>(dst) = make_double2(acc[x][y][0] * inv_sqrt_d, acc[x][y][1] * inv_sqrt_d);
      } else {
        if (j < T_n) dst[0] = acc[x][y][0] * inv_sqrt_d;
        if (j + 1 < T_n) dst[1] = acc[x][y][1] * inv_sqrt_d;
      }
    }
  }
}

// K1c: in-place row softmax with max subtraction (numerics.py:46-52). One warp per row.
__global__ void k_softmax_rows(double* __restrict__ p, int64_t rows, int T_n) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= rows) return;
  double* x = p + row * (int64_t)T_n;
  double m = -INFINITY;
  for (int j = lane; j < T_n; j += 32) m = fmax(m, x[j]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  double s = 0.0;
  for (int j = lane; j < T_n; j += 32) {
    double e = exp(x[j] - m);
    x[j] = e;
    s += e;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  for (int j = lane; j < T_n; j += 32) x[j] = x[j] / s;
}

// ---------------------------------------------------------------------------------------
// K2: per-row selection.  One CTA per row: block-wide bitonic sort of (value, column)
// pairs in shared memory into the reference's stable descending order (masker.py:113-115:
// larger value first, equal values by ascending column), then the hybrid count
//   kept = min(max(K, cnt_p), T_n),  cnt_p = searchsorted_left(cumsum(sorted), thr) + 1
// with the cumsum evaluated strictly sequentially in float64 exactly like np.cumsum.
// For non-negative rows the running sum is monotone, so a linear scan that stops at the
// first prefix >= thr equals numpy's binary search; if a row has a negative entry the
// full cumsum is built and numpy's left binary search is replayed step for step.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ bool goes_before(double va, int ca, double vb, int cb) {
  return va > vb || (va == vb && ca < cb);
}

constexpr int kSelThreads = 128;
constexpr int kBuckets = 256;  // 4 buckets per octave from 1 down to 2^-63; bucket 255 also holds 0

// Order-preserving bucket of a non-negative double: bucket 0 holds the largest values.
__device__ __forceinline__ int value_bucket(double v) {
  const long long bits = __double_as_longlong(v);
  const int key = (int)((bits >> 50) & 0x1FFF);  // exponent (11 bits) and top 2 mantissa bits
  return min(kBuckets - 1, max(0, ((1023 << 2) | 3) - key));
}
// Smallest value a bucket can hold (a lower bound used for the candidate mass).
__device__ __forceinline__ double bucket_floor(int b) {
  if (b >= kBuckets - 1) return 0.0;
  const int key = ((1023 << 2) | 3) - b;
  return ldexp(1.0 + 0.25 * (key & 3), (key >> 2) - 1023);
}

// One CTA per row.  (1) histogram of the row over order-preserving value buckets (4 per
// octave); (2) walking buckets from the largest, the shortest bucket prefix holding at least
// K entries whose mass LOWER BOUND (count x bucket floor) reaches p + 1e-9 is a candidate set
// guaranteed to contain the answer: entries outside it are strictly smaller than every
// candidate, and the candidates' exact mass exceeds the threshold by >= 1e-9, far above the
// rounding of a <=16384-term float64 running sum, so the sequential cumsum reaches `thr`
// inside it; (3) only the candidates are sorted (bitonic, shared memory) and scanned.  Rows with negative entries
// (non-monotone cumsum) take every entry as a candidate.  Output is identical to sorting the
// whole row.
// FROM_SCORES: the input rows are pre-softmax scores; the row softmax is applied first, into
// shared memory, with exactly k_softmax_rows' arithmetic (warp 0: lane-strided max and
// exp-sums, xor-butterfly combine; p = exp(x - m) / s), so the selection is identical to
// spa2_pooled_map + spa2_select while the float64 map never goes through HBM.
template <bool FROM_SCORES>
__global__ void __launch_bounds__(kSelThreads) k_select(const double* __restrict__ probs, int T_n, int k_count,
                                                        double thr, int use_p, uint8_t* __restrict__ keep,
                                                        int32_t* __restrict__ counts) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char smem_raw[];  // [p row (FROM_SCORES)] cand_v[T_pad], cand_c[T_pad]
  __shared__ int h_cnt[kBuckets];
  __shared__ int s_neg, s_bstar, s_npos, s_kept;
  __shared__ double s_s;
  const int64_t row = blockIdx.x;
  const double* x = probs + row * (int64_t)T_n;
  if constexpr (FROM_SCORES) {
    // max: any reduction order is exact; exponentials by all threads; the sum in
    // k_softmax_rows' order (lane l adds j = l, l+32, ... sequentially, xor-butterfly).
    double* pr = reinterpret_cast<double*>(smem_raw);
    __shared__ double s_red[kSelThreads / 32];
    double m = -INFINITY;
    for (int j = threadIdx.x; j < T_n; j += blockDim.x) m = fmax(m, x[j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = m;
    __syncthreads();
    m = s_red[0];
#pragma unroll
    for (int w = 1; w < kSelThreads / 32; ++w) m = fmax(m, s_red[w]);
    for (int j = threadIdx.x; j < T_n; j += blockDim.x) pr[j] = exp(x[j] - m);
    __syncthreads();
    if (threadIdx.x < 32) {
      double sum = 0.0;
      for (int j = threadIdx.x; j < T_n; j += 32) sum += pr[j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (threadIdx.x == 0) s_s = sum;
    }
    __syncthreads();
    const double sum = s_s;
    for (int j = threadIdx.x; j < T_n; j += blockDim.x) pr[j] = pr[j] / sum;
    __syncthreads();
    x = pr;
  }
  for (int b = threadIdx.x; b < kBuckets; b += blockDim.x) h_cnt[b] = 0;
  if (threadIdx.x == 0) {
    s_neg = 0;
    s_npos = 0;
  }
  __syncthreads();
  bool neg = false;
  for (int t = threadIdx.x; t < T_n; t += blockDim.x) {
    const double v = x[t];
    // negative entries take the exact all-candidates path (numpy semantics); so do NaN/Inf
    // (non-finite q/k, reported by the finiteness flag): garbage mask, but no fault
    if (!(v >= 0.0) || v == INFINITY) {
      neg = true;
    } else {
      atomicAdd(&h_cnt[value_bucket(v)], 1);
    }
  }
  if (neg) s_neg = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    int bstar = kBuckets;  // kBuckets = "every entry"
    if (!s_neg) {
      int cnt = 0;
      double mass = 0.0;
      const double need = thr + 1e-9;
      for (int b = 0; b < kBuckets; ++b) {
        cnt += h_cnt[b];
        mass += h_cnt[b] * bucket_floor(b);
        if (cnt >= k_count && (!use_p || mass >= need)) {
          bstar = b;
          break;
        }
      }
    }
    s_bstar = bstar;
  }
  __syncthreads();
  const int bstar = s_bstar;
  double* cv = reinterpret_cast<double*>(smem_raw) + (FROM_SCORES ? T_n : 0);
  int T_pad = 1;
  while (T_pad < T_n) T_pad <<= 1;
  int* cc = reinterpret_cast<int*>(cv + T_pad);
  for (int t = threadIdx.x; t < T_n; t += blockDim.x) {
    const double v = x[t];
    if (bstar == kBuckets || (v >= 0.0 && value_bucket(v) <= bstar)) {
      const int pos = atomicAdd(&s_npos, 1);
      cv[pos] = v;
      cc[pos] = t;
    }
  }
  __syncthreads();
  const int C = s_npos;
  int C_pad = 1;
  while (C_pad < C) C_pad <<= 1;
  for (int t = C + threadIdx.x; t < C_pad; t += blockDim.x) {
    cv[t] = -INFINITY;
    cc[t] = 0x7fffffff;
  }
  __syncthreads();
  for (int size = 2; size <= C_pad; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < (C_pad >> 1); t += blockDim.x) {
        const int i = 2 * t - (t & (stride - 1));
        const int j = i + stride;
        const bool up = (i & size) == 0;
        const double vi = cv[i], vj = cv[j];
        const int ci = cc[i], cj = cc[j];
        if (goes_before(vj, cj, vi, ci) == up) {
          cv[i] = vj;
          cv[j] = vi;
          cc[i] = cj;
          cc[j] = ci;
        }
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    int cnt_p = 1;
    if (use_p) {
      if (!s_neg) {
        double run = 0.0;
        int t = 0;
        for (; t < C; ++t) {
          run = (t == 0) ? cv[0] : run + cv[t];
          if (run >= thr) break;
        }
        cnt_p = (t < C) ? t + 1 : T_n + 1;  // t == C only when every entry is a candidate
      } else {
        double run = 0.0;
        for (int t = 0; t < T_n; ++t) {
          run = (t == 0) ? cv[0] : run + cv[t];
          cv[t] = run;  // sorted values are no longer needed
        }
        int lo = 0, hi = T_n;  // numpy npy_binsearch (side='left'), single key
        while (lo < hi) {
          const int mid = lo + ((hi - lo) >> 1);
          if (cv[mid] < thr) lo = mid + 1;
          else hi = mid;
        }
        cnt_p = lo + 1;
      }
    }
    s_kept = min(max(k_count, cnt_p), T_n);
    if (counts != nullptr) counts[row] = s_kept;
  }
  uint8_t* out = keep + row * (int64_t)T_n;
  for (int t = threadIdx.x; t < T_n; t += blockDim.x) out[t] = 0;
  __syncthreads();
  const int kept = min(s_kept, C);  // == s_kept for finite rows (the candidates hold the answer)
  for (int t = threadIdx.x; t < kept; t += blockDim.x) {
    const int c = cc[t];
    if ((unsigned)c < (unsigned)T_n) out[c] = 1;  // NaN rows may sort padding forward
  }
}

// ---------------------------------------------------------------------------------------
// K3: block lists.
// ---------------------------------------------------------------------------------------
// Column counts and column lists: one CTA per (head, 32-column chunk); lane = column, the
// 8 warps split the T_m rows into contiguous ranges (coalesced 32-byte row segments).
constexpr int kColWarps = 16;

__device__ __forceinline__ void col_range(int T_m, int w, int& r0, int& r1) {
  const int per = (T_m + kColWarps - 1) / kColWarps;
  r0 = min(w * per, T_m);
  r1 = min(r0 + per, T_m);
}

constexpr int kScanThreads = 1024;

// Inclusive scan across the 1024 threads of a CTA (warp-shuffle scan).
__device__ int32_t cta_inclusive_scan_1024(int32_t v, int32_t* sh_warp) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  if (lane == 31) sh_warp[w] = v;
  __syncthreads();
  if (w == 0) {
    int32_t t = sh_warp[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t u = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += u;
    }
    sh_warp[lane] = t;
  }
  __syncthreads();
  const int32_t r = v + (w > 0 ? sh_warp[w - 1] : 0);
  __syncthreads();
  return r;
}

// Longest-first order: counting sort of ids base..base+n-1 by descending count (counts in
// [0, maxc]); ids are written to order[base ...].
__device__ void cta_order_desc(const int32_t* cnt, int64_t n, int maxc, int32_t* order, int32_t* bins, int32_t* sh,
                               int64_t base) {
  cnt += base;
  order += base;
  for (int c = threadIdx.x; c <= maxc; c += kScanThreads) bins[c] = 0;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < n; i += kScanThreads) atomicAdd(&bins[maxc - cnt[i]], 1);
  __syncthreads();
  // bins (indexed by maxc - count, i.e. descending count) -> exclusive starts, in place
  const int nb = maxc + 1;
  const int per = (nb + kScanThreads - 1) / kScanThreads;
  const int beg = min((int)threadIdx.x * per, nb), end = min(beg + per, nb);
  int32_t local = 0;
  for (int b = beg; b < end; ++b) local += bins[b];
  int32_t run = cta_inclusive_scan_1024(local, sh) - local;
  for (int b = beg; b < end; ++b) {
    int32_t c = bins[b];
    bins[b] = run;
    run += c;
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < n; i += kScanThreads) {
    int pos = atomicAdd(&bins[maxc - cnt[i]], 1);
    order[pos] = (int32_t)(base + i);
  }
  __syncthreads();
}

// Launch orders (k_scan_orders): head-major (so one or two heads' K/V or Q/dO stay resident
// in the 126 MB L2 while their blocks are processed) and longest-first within each head.
// ---------------------------------------------------------------------------------------
// K3 (3 launches): counts -> per-head scan + launch orders -> fill.
// ---------------------------------------------------------------------------------------
// (a) blockIdx.x < col_chunks: column counts of 32 columns of head blockIdx.y (as k_col_counts);
//     otherwise row counts, one warp per row (as k_row_counts).
__global__ void __launch_bounds__(kColWarps * 32) k_counts(const uint8_t* __restrict__ keep, int T_m, int T_n,
                                                           int col_chunks, int32_t* __restrict__ row_cnt,
                                                           int32_t* __restrict__ col_cnt) {
  pdl_wait();
  pdl_trigger();
  const int64_t bh = blockIdx.y;
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  if ((int)blockIdx.x < col_chunks) {
    __shared__ int part[kColWarps][32];
    const int j = blockIdx.x * 32 + lane;
    int r0, r1;
    col_range(T_m, w, r0, r1);
    const uint8_t* base = keep + bh * (int64_t)T_m * T_n + j;
    int c = 0;
    if (j < T_n) {
#pragma unroll 8
      for (int i = r0; i < r1; ++i) c += base[(int64_t)i * T_n] != 0;
    }
    part[w][lane] = c;
    __syncthreads();
    if (w == 0 && j < T_n) {
      int sum = 0;
#pragma unroll
      for (int x = 0; x < kColWarps; ++x) sum += part[x][lane];
      col_cnt[bh * T_n + j] = sum;
    }
  } else {
    const int i = ((int)blockIdx.x - col_chunks) * kColWarps + w;
    if (i >= T_m) return;
    const uint8_t* rowp = keep + (bh * (int64_t)T_m + i) * T_n;
    int c = 0;
    for (int j = lane; j < T_n; j += 32) c += rowp[j] != 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) row_cnt[bh * T_m + i] = c;
  }
}

// (b) one CTA per (head, rows|columns): CSR offsets of that head's rows (or columns) — base =
//     kept blocks of all earlier heads, summed here so no second global pass is needed — and
//     its longest-first launch order.
__global__ void __launch_bounds__(kScanThreads) k_scan_orders(const int32_t* __restrict__ row_cnt,
                                                              const int32_t* __restrict__ col_cnt, int T_m, int T_n,
                                                              int64_t bh_total, int32_t* row_ptr, int32_t* col_ptr,
                                                              int32_t* row_order, int32_t* col_order) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ int32_t sh_ord[];  // [kScanThreads] + bins[max(T_m,T_n)+1]
  int32_t* bins = sh_ord + kScanThreads;
  __shared__ int32_t s_base;
  const int64_t bh = blockIdx.x;
  const bool rows = blockIdx.y == 0;
  const int n = rows ? T_m : T_n;
  const int32_t* cnt_all = rows ? row_cnt : col_cnt;
  // kept blocks of the earlier heads
  int32_t pre = 0;
  for (int64_t e = threadIdx.x; e < bh * n; e += kScanThreads) pre += cnt_all[e];
  pre = cta_inclusive_scan_1024(pre, sh_ord);
  if (threadIdx.x == kScanThreads - 1) s_base = pre;
  __syncthreads();
  const int32_t base = s_base;
  const int32_t* cnt = cnt_all + bh * n;
  int32_t* ptr = (rows ? row_ptr : col_ptr) + bh * n;
  const int per = (n + kScanThreads - 1) / kScanThreads;
  const int beg = min((int)threadIdx.x * per, n), end = min(beg + per, n);
  int32_t local = 0;
  for (int i = beg; i < end; ++i) local += cnt[i];
  const int32_t incl = cta_inclusive_scan_1024(local, sh_ord);
  int32_t run = base + incl - local;
  for (int i = beg; i < end; ++i) {
    const int32_t c = cnt[i];
    ptr[i] = run;
    run += c;
  }
  if (bh == bh_total - 1 && threadIdx.x == kScanThreads - 1) ptr[n] = base + incl;  // the CSR end entry
  __syncthreads();
  if (rows)
    cta_order_desc(row_cnt, T_m, T_n, row_order, bins, sh_ord, bh * T_m);
  else
    cta_order_desc(col_cnt, T_n, T_m, col_order, bins, sh_ord, bh * T_n);
}

// (c) blockIdx.x < col_chunks: column lists (as k_fill_cols); otherwise row lists, one warp
//     per row (as k_fill_rows).
__global__ void __launch_bounds__(kColWarps * 32) k_fill(const uint8_t* __restrict__ keep, int T_m, int T_n,
                                                         int col_chunks, const int32_t* __restrict__ row_ptr,
                                                         int32_t* __restrict__ row_idx,
                                                         const int32_t* __restrict__ col_ptr,
                                                         int32_t* __restrict__ col_idx) {
  pdl_wait();
  pdl_trigger();
  const int64_t bh = blockIdx.y;
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  if ((int)blockIdx.x < col_chunks) {
    __shared__ int part[kColWarps][32];
    const int j = blockIdx.x * 32 + lane;
    int r0, r1;
    col_range(T_m, w, r0, r1);
    const uint8_t* base = keep + bh * (int64_t)T_m * T_n + j;
    int c = 0;
    if (j < T_n) {
#pragma unroll 8
      for (int i = r0; i < r1; ++i) c += base[(int64_t)i * T_n] != 0;
    }
    part[w][lane] = c;
    __syncthreads();
    if (j >= T_n) return;
    int off = col_ptr[bh * T_n + j];
    for (int x = 0; x < w; ++x) off += part[x][lane];
#pragma unroll 8
    for (int i = r0; i < r1; ++i) {
      const int v = base[(int64_t)i * T_n];  // 1 = both query-block halves keep it, 2 top only, 3 bottom only
      if (v != 0) col_idx[off++] = i | ((v - 1) << 30);
    }
  } else {
    const int i = ((int)blockIdx.x - col_chunks) * kColWarps + w;
    if (i >= T_m) return;
    const int64_t row = bh * T_m + i;
    int b = row_ptr[row];
    for (int j0 = 0; j0 < T_n; j0 += 32) {
      const int j = j0 + lane;
      const int v = j < T_n ? keep[row * T_n + j] : 0;
      const bool f = v != 0;
      const unsigned m = __ballot_sync(0xffffffffu, f);
      if (f) row_idx[b + __popc(m & ((1u << lane) - 1u))] = j | ((v - 1) << 30);
      b += __popc(m);
    }
  }
}

template <typename T>
int launch_pool(spa2_view q, spa2_view k, int64_t B, int64_t H, int64_t N, int64_t d, int64_t b_q, int64_t b_kv,
                int64_t T_m, int64_t T_n, double* qbar, double* kbar, int32_t* nonfinite, cudaStream_t st) {
  const int64_t BH = B * H;
  constexpr int CV = 16 / (int)sizeof(T) < 8 ? 16 / (int)sizeof(T) : 8;
  auto aligned = [&](const spa2_view& v) {
    return ((uintptr_t)v.ptr % 16 == 0) && (v.sb % CV == 0) && (v.sh % CV == 0) && (v.sn % CV == 0);
  };
  const bool vec = (d % CV == 0) && aligned(q) && aligned(k);
  const int cpt = vec ? CV : 1;
  const int64_t threads = BH * (T_m + T_n) * (d / cpt);
  SPA2_REQUIRE(threads < (1ll << 40), SPA2_ERR_UNSUPPORTED, "pooled_map: problem too large");
  const unsigned grid = (unsigned)ceil_div(threads, 256);
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    if (vec && d % 8 == 0) {
      SPA2_CUDA_TRY(launch_pdl(k_pool_bf16_pipe, dim3(grid), dim3(256), 0, st, q, k, (int)H, (int)N, (int)d, (int)b_q,
                               (int)b_kv, (int)T_m, (int)T_n, BH, qbar, kbar, nonfinite));
      SPA2_LAUNCH_CHECK();
      return SPA2_OK;
    }
  }
  if (vec)
    k_pool<T, CV><<<grid, 256, 0, st>>>(q, k, (int)H, (int)N, (int)d, (int)b_q, (int)b_kv, (int)T_m, (int)T_n, BH,
                                        qbar, kbar, nonfinite);
  else
    k_pool<T, 1><<<grid, 256, 0, st>>>(q, k, (int)H, (int)N, (int)d, (int)b_q, (int)b_kv, (int)T_m, (int)T_n, BH,
                                       qbar, kbar, nonfinite);
  SPA2_LAUNCH_CHECK();
  return SPA2_OK;
}

}  // namespace
}  // namespace spa2

using namespace spa2;

static int pooled_map_impl(spa2_view q, spa2_view k, int dtype, int64_t B, int64_t H, int64_t N, int64_t d,
                           int64_t b_q, int64_t b_kv, double* probs, double* workspace, int32_t* nonfinite,
                           void* stream, bool softmax) {
  SPA2_REQUIRE(B >= 1 && H >= 1 && N >= 1 && d >= 1, SPA2_ERR_VALUE,
               "pooled_map: bad shape B=%lld H=%lld N=%lld d=%lld", (long long)B, (long long)H,
               (long long)N, (long long)d);
  SPA2_REQUIRE(b_q >= 1 && b_kv >= 1, SPA2_ERR_VALUE, "block sizes must be >= 1: b_q=%lld, b_kv=%lld",
               (long long)b_q, (long long)b_kv);
  SPA2_REQUIRE(q.ptr && k.ptr && probs && workspace, SPA2_ERR_VALUE, "pooled_map: null pointer");
  SPA2_REQUIRE(N < (1ll << 31), SPA2_ERR_UNSUPPORTED, "pooled_map: N too large");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t T_m = ceil_div(N, b_q), T_n = ceil_div(N, b_kv), BH = B * H;
  double* qbar = workspace;
  double* kbar = workspace + BH * T_m * d;
  int rc;
  switch (dtype) {
    case SPA2_BF16: rc = launch_pool<__nv_bfloat16>(q, k, B, H, N, d, b_q, b_kv, T_m, T_n, qbar, kbar, nonfinite, st); break;
    case SPA2_F16: rc = launch_pool<__half>(q, k, B, H, N, d, b_q, b_kv, T_m, T_n, qbar, kbar, nonfinite, st); break;
    case SPA2_F32: rc = launch_pool<float>(q, k, B, H, N, d, b_q, b_kv, T_m, T_n, qbar, kbar, nonfinite, st); break;
    case SPA2_F64: rc = launch_pool<double>(q, k, B, H, N, d, b_q, b_kv, T_m, T_n, qbar, kbar, nonfinite, st); break;
    default: SPA2_REQUIRE(false, SPA2_ERR_UNSUPPORTED, "pooled_map: unsupported dtype %d", dtype);
  }
  if (rc != SPA2_OK) return rc;
  if (d % 2 == 0) {  // 16-byte row chunks for cp.async (d is even for every supported head dim)
    dim3 grid((unsigned)ceil_div(T_n, 64), (unsigned)ceil_div(T_m, 64), (unsigned)BH);
    SPA2_CUDA_TRY(cudaFuncSetAttribute(k_scores_dmma, cudaFuncAttributeMaxDynamicSharedMemorySize, kDmSmem));
    SPA2_CUDA_TRY(launch_pdl(k_scores_dmma, grid, dim3(128), kDmSmem, st, qbar, kbar, (int)T_m, (int)T_n, (int)d,
                             1.0 / sqrt((double)d), probs));
  } else {
    dim3 grid((unsigned)ceil_div(T_n, kSTJ), (unsigned)ceil_div(T_m, kSTI), (unsigned)BH);
    SPA2_CUDA_TRY(cudaFuncSetAttribute(k_scores, cudaFuncAttributeMaxDynamicSharedMemorySize, kScoresSmem));
    SPA2_CUDA_TRY(launch_pdl(k_scores, grid, dim3(256), kScoresSmem, st, qbar, kbar, (int)T_m, (int)T_n, (int)d,
                             sqrt((double)d), probs));
  }
  SPA2_LAUNCH_CHECK();
  if (!softmax) return SPA2_OK;
  const int64_t rows = BH * T_m;
  k_softmax_rows<<<(unsigned)ceil_div(rows, 8), 256, 0, st>>>(probs, rows, (int)T_n);
  SPA2_LAUNCH_CHECK();
  return SPA2_OK;
}

extern "C" int spa2_pooled_map(spa2_view q, spa2_view k, int dtype, int64_t B, int64_t H, int64_t N,
                               int64_t d, int64_t b_q, int64_t b_kv, double* probs,
                               double* workspace, int32_t* nonfinite, void* stream) {
  return pooled_map_impl(q, k, dtype, B, H, N, d, b_q, b_kv, probs, workspace, nonfinite, stream, true);
}

extern "C" int spa2_select(const double* probs, int64_t rows, int64_t t_n, int64_t k_count,
                           double p_threshold, uint8_t* keep, int32_t* counts, void* stream) {
  SPA2_REQUIRE(rows >= 1 && t_n >= 1, SPA2_ERR_VALUE, "select: empty map (%lld x %lld)",
               (long long)rows, (long long)t_n);
  SPA2_REQUIRE(k_count >= 1, SPA2_ERR_VALUE, "select: k_count must be >= 1");
  SPA2_REQUIRE(probs && keep, SPA2_ERR_VALUE, "select: null pointer");
  SPA2_REQUIRE(!isnan(p_threshold), SPA2_ERR_VALUE, "select: p_threshold is NaN");
  SPA2_REQUIRE(rows < (1ll << 31), SPA2_ERR_UNSUPPORTED, "select: too many rows");
  int t_pad = 1;
  while (t_pad < t_n) t_pad <<= 1;
  const size_t smem = (size_t)t_pad * (sizeof(double) + sizeof(int));
  SPA2_REQUIRE(smem <= 200 * 1024, SPA2_ERR_UNSUPPORTED, "select: T_n=%lld exceeds 16384", (long long)t_n);
  cudaStream_t st = (cudaStream_t)stream;
  if (smem > 48 * 1024)
    SPA2_CUDA_TRY(cudaFuncSetAttribute(k_select<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int use_p = isinf(p_threshold) && p_threshold < 0 ? 0 : 1;
  const int kk = (int)std::min<int64_t>(k_count, t_n);
  k_select<false><<<(unsigned)rows, kSelThreads, smem, st>>>(probs, (int)t_n, kk, p_threshold, use_p, keep, counts);
  SPA2_LAUNCH_CHECK();
  return SPA2_OK;
}

extern "C" int spa2_block_mean_pool(spa2_view q, spa2_view k, int dtype, int64_t B, int64_t H, int64_t N, int64_t d,
                                    int64_t b_q, int64_t b_kv, double* qbar, double* kbar, int32_t* nonfinite,
                                    void* stream) {
  SPA2_REQUIRE(B >= 1 && H >= 1 && N >= 1 && d >= 1, SPA2_ERR_VALUE,
               "block_mean_pool: bad shape B=%lld H=%lld N=%lld d=%lld", (long long)B, (long long)H,
               (long long)N, (long long)d);
  SPA2_REQUIRE(b_q >= 1 && b_kv >= 1, SPA2_ERR_VALUE, "block sizes must be >= 1: b_q=%lld, b_kv=%lld",
               (long long)b_q, (long long)b_kv);
  SPA2_REQUIRE(q.ptr && k.ptr && qbar && kbar, SPA2_ERR_VALUE, "block_mean_pool: null pointer");
  SPA2_REQUIRE(N < (1ll << 31), SPA2_ERR_UNSUPPORTED, "block_mean_pool: N too large");
  SPA2_REQUIRE(kbar == qbar + B * H * ceil_div(N, b_q) * d, SPA2_ERR_VALUE,
               "block_mean_pool: kbar must directly follow qbar (one workspace)");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t T_m = ceil_div(N, b_q), T_n = ceil_div(N, b_kv);
  switch (dtype) {
    case SPA2_BF16: return launch_pool<__nv_bfloat16>(q, k, B, H, N, d, b_q, b_kv, T_m, T_n, qbar, kbar, nonfinite, st);
    case SPA2_F16: return launch_pool<__half>(q, k, B, H, N, d, b_q, b_kv, T_m, T_n, qbar, kbar, nonfinite, st);
    case SPA2_F32: return launch_pool<float>(q, k, B, H, N, d, b_q, b_kv, T_m, T_n, qbar, kbar, nonfinite, st);
    case SPA2_F64: return launch_pool<double>(q, k, B, H, N, d, b_q, b_kv, T_m, T_n, qbar, kbar, nonfinite, st);
    default: SPA2_REQUIRE(false, SPA2_ERR_UNSUPPORTED, "block_mean_pool: unsupported dtype %d", dtype);
  }
}

extern "C" int spa2_pooled_scores(spa2_view q, spa2_view k, int dtype, int64_t B, int64_t H, int64_t N, int64_t d,
                                  int64_t b_q, int64_t b_kv, double* scores, double* workspace, int32_t* nonfinite,
                                  void* stream) {
  return pooled_map_impl(q, k, dtype, B, H, N, d, b_q, b_kv, scores, workspace, nonfinite, stream, false);
}

extern "C" int spa2_select_scores(const double* scores, int64_t rows, int64_t t_n, int64_t k_count,
                                  double p_threshold, uint8_t* keep, int32_t* counts, void* stream) {
  SPA2_REQUIRE(rows >= 1 && t_n >= 1, SPA2_ERR_VALUE, "select_scores: empty map (%lld x %lld)", (long long)rows,
               (long long)t_n);
  SPA2_REQUIRE(k_count >= 1, SPA2_ERR_VALUE, "select_scores: k_count must be >= 1");
  SPA2_REQUIRE(scores && keep, SPA2_ERR_VALUE, "select_scores: null pointer");
  SPA2_REQUIRE(!isnan(p_threshold), SPA2_ERR_VALUE, "select_scores: p_threshold is NaN");
  SPA2_REQUIRE(rows < (1ll << 31), SPA2_ERR_UNSUPPORTED, "select_scores: too many rows");
  SPA2_REQUIRE(t_n <= 4096, SPA2_ERR_UNSUPPORTED, "select_scores: T_n=%lld > 4096 (use pooled_map + select)",
               (long long)t_n);
  int t_pad = 1;
  while (t_pad < t_n) t_pad <<= 1;
  const size_t smem = (size_t)t_n * sizeof(double) + (size_t)t_pad * (sizeof(double) + sizeof(int));
  cudaStream_t st = (cudaStream_t)stream;
  if (smem > 48 * 1024)
    SPA2_CUDA_TRY(cudaFuncSetAttribute(k_select<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int use_p = isinf(p_threshold) && p_threshold < 0 ? 0 : 1;
  const int kk = (int)std::min<int64_t>(k_count, t_n);
  SPA2_CUDA_TRY(launch_pdl(k_select<true>, dim3((unsigned)rows), dim3(kSelThreads), smem, st, scores, (int)t_n, kk,
                           p_threshold, use_p, keep, counts));
  SPA2_LAUNCH_CHECK();
  return SPA2_OK;
}

extern "C" int spa2_build_lists(const uint8_t* keep, int64_t bh, int64_t t_m, int64_t t_n,
                                int32_t* row_ptr, int32_t* row_idx, int32_t* col_ptr,
                                int32_t* col_idx, int32_t* row_order, int32_t* col_order,
                                int32_t* scratch, void* stream) {
  SPA2_REQUIRE(bh >= 1 && t_m >= 1 && t_n >= 1, SPA2_ERR_VALUE, "build_lists: empty grid");
  SPA2_REQUIRE(keep && row_ptr && row_idx && col_ptr && col_idx && row_order && col_order && scratch,
               SPA2_ERR_VALUE, "build_lists: null pointer");
  SPA2_REQUIRE(bh * t_m * t_n < (1ll << 31), SPA2_ERR_UNSUPPORTED, "build_lists: grid too large");
  SPA2_REQUIRE(std::max(t_m, t_n) <= 32768 && bh < 65536, SPA2_ERR_UNSUPPORTED,
               "build_lists: T_m/T_n > 32768 or B*H >= 65536");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t ncols = bh * t_n;
  int32_t* col_cnt = scratch;          // [ncols]
  int32_t* row_cnt = scratch + ncols;  // [nrows]
  const int col_chunks = (int)ceil_div(t_n, 32);
  const dim3 grid((unsigned)(col_chunks + ceil_div(t_m, kColWarps)), (unsigned)bh);
  SPA2_CUDA_TRY(launch_pdl(k_counts, grid, dim3(kColWarps * 32), 0, st, keep, (int)t_m, (int)t_n, col_chunks, row_cnt,
                           col_cnt));
  SPA2_LAUNCH_CHECK();
  const size_t smem = (kScanThreads + std::max(t_m, t_n) + 1) * sizeof(int32_t);
  if (smem > 48 * 1024)
    SPA2_CUDA_TRY(cudaFuncSetAttribute(k_scan_orders, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  SPA2_CUDA_TRY(launch_pdl(k_scan_orders, dim3((unsigned)bh, 2), dim3(kScanThreads), smem, st, row_cnt, col_cnt,
                           (int)t_m, (int)t_n, bh, row_ptr, col_ptr, row_order, col_order));
  SPA2_LAUNCH_CHECK();
  SPA2_CUDA_TRY(launch_pdl(k_fill, grid, dim3(kColWarps * 32), 0, st, keep, (int)t_m, (int)t_n, col_chunks, row_ptr,
                           row_idx, col_ptr, col_idx));
  SPA2_LAUNCH_CHECK();
  return SPA2_OK;
}

extern "C" int spa2_check_finite(spa2_view x, int dtype, int64_t B, int64_t H, int64_t N, int64_t d,
                                 int32_t* nonfinite, void* stream) {
  SPA2_REQUIRE(dtype == SPA2_BF16, SPA2_ERR_UNSUPPORTED, "check_finite: only bf16 operands are supported");
  SPA2_REQUIRE(B >= 1 && H >= 1 && N >= 1 && d >= 8 && d % 8 == 0, SPA2_ERR_VALUE,
               "check_finite: bad shape B=%lld H=%lld N=%lld d=%lld", (long long)B, (long long)H, (long long)N,
               (long long)d);
  SPA2_REQUIRE(x.ptr && nonfinite, SPA2_ERR_VALUE, "check_finite: null pointer");
  SPA2_REQUIRE((uintptr_t)x.ptr % 16 == 0 && x.sb % 8 == 0 && x.sh % 8 == 0 && x.sn % 8 == 0, SPA2_ERR_UNSUPPORTED,
               "check_finite: operand must be 16-byte aligned with strides %% 8 == 0");
  SPA2_REQUIRE(N * (d / 8) < (1ll << 31), SPA2_ERR_UNSUPPORTED, "check_finite: N too large");
  SPA2_REQUIRE((d & (d - 1)) == 0 && B * H < 65536, SPA2_ERR_UNSUPPORTED,
               "check_finite: d must be a power of two and B*H < 65536");
  int cpr_log2 = 0;
  while ((8 << cpr_log2) < d) ++cpr_log2;
  const int64_t per_head = N * (d / 8);
  // ~8 resident 256-thread blocks per SM over all heads, each thread kK0Unroll chunks per pass
  const int64_t want = std::max<int64_t>(1, (148 * 8 + B * H - 1) / (B * H));
  const unsigned gx = (unsigned)std::min<int64_t>(want, ceil_div(per_head, 256 * kK0Unroll));
  SPA2_CUDA_TRY(launch_pdl(k_nonfinite_bf16, dim3(gx, (unsigned)(B * H)), dim3(256), 0, (cudaStream_t)stream, x,
                           (int)H, (int)N, cpr_log2, nonfinite));
  SPA2_LAUNCH_CHECK();
  return SPA2_OK;
}
