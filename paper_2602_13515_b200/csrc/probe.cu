// probe.cu — a one-CTA tcgen05 GEMM that exercises exactly the operand layouts, UMMA
// descriptors, TMA swizzle and TMEM read-back the attention kernels rely on.  It is a
// diagnostic entry point (spa2_probe_gemm) used by the GPU tests to validate those
// building blocks in isolation before they are trusted inside the fused kernels.
#include "common.cuh"
#include "ptx.cuh"
#include "tma_host.h"

namespace spa2 {
namespace {

using namespace ptx;

// Stage a row-major [R][C] bf16 matrix into SWIZZLE_128B column chunks with generic stores.
__device__ void stage_generic(uint8_t* dst, const __nv_bfloat16* src, int R, int C) {
  const int units_per_row = C / 8;
  for (int e = threadIdx.x; e < R * units_per_row; e += blockDim.x) {
    const int r = e / units_per_row, u = e % units_per_row;
    const uint4 v = *reinterpret_cast<const uint4*>(src + (int64_t)r * C + u * 8);
    const uint32_t addr = smem_u32(dst) + (uint32_t)((u / 8) * R * 128) + sw128_offset(r, u % 8);
    st_shared_v4(addr, v.x, v.y, v.z, v.w);
  }
}

// Descriptor for the k-step `ks` (16 deep) of an operand stored as described in ptx.cuh.
__device__ uint64_t operand_desc(uint32_t base, bool mn_major, int R, int ks) {
  if (!mn_major) {
    const int k0 = ks * 16;
    return sw128_desc(base + (uint32_t)((k0 / 64) * R * 128 + (k0 % 64) * 2), 16, 1024);
  }
  return sw128_desc(base + (uint32_t)(ks * 16 * 128), (uint32_t)(R * 128), 1024);
}

__global__ void __launch_bounds__(128) k_probe(const __nv_bfloat16* a, const __nv_bfloat16* b, float* d, int M,
                                               int N, int K, int a_mn, int b_mn, int use_tma,
                                               const __grid_constant__ CUtensorMap ta,
                                               const __grid_constant__ CUtensorMap tb) {
  extern __shared__ uint8_t smem_dyn[];
  __shared__ uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_base;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = base;
  uint8_t* sb = base + 32768;
  const int Ra = a_mn ? K : M, Ca = a_mn ? M : K;
  const int Rb = b_mn ? K : N, Cb = b_mn ? N : K;
  if (warp_id() == 0) tmem_alloc(&tmem_base, 256);
  if (threadIdx.x == 32) {
    mbar_init(&bar_load, 1);
    mbar_init(&bar_mma, 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (use_tma == 1) {
    if (threadIdx.x == 0) {
      mbar_expect_tx(&bar_load, (uint32_t)((Ra * Ca + Rb * Cb) * 2));
      for (int c = 0; c < Ca / 64; ++c) tma_load_2d(sa + c * Ra * 128, &ta, &bar_load, c * 64, 0);
      for (int c = 0; c < Cb / 64; ++c) tma_load_2d(sb + c * Rb * 128, &tb, &bar_load, c * 64, 0);
    }
    mbar_wait(&bar_load, 0);
  } else {
    if (use_tma == 2) {
      // A -> TMEM columns [128, 128 + K/2): thread row m packs its K bf16 values in pairs
      const int m = 32 * (int)warp_id() + (int)lane_id();
      for (int c0 = 0; c0 < K / 2; c0 += 32) {
        uint32_t r[32];
        const uint32_t* src = reinterpret_cast<const uint32_t*>(a + (int64_t)m * K) + c0;
        for (int e = 0; e < 32; ++e) r[e] = src[e];
        tmem_st32(tbase + ((uint32_t)(32 * warp_id()) << 16) + 128u + (uint32_t)c0, r);
      }
      tmem_st_wait();
    } else {
      stage_generic(sa, a, Ra, Ca);
    }
    stage_generic(sb, b, Rb, Cb);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    tc_fence_after();
    const uint32_t idesc = idesc_bf16(M, N, a_mn != 0, b_mn != 0);
    if (use_tma == 3)  // A: smem (K-major SW128) -> TMEM columns [128, 128 + K/2) by tcgen05.cp
      for (int ks = 0; ks < K / 16; ++ks)
        tmem_cp_128x256b(tbase + 128u + (uint32_t)(ks * 8), operand_desc(smem_u32(sa), false, Ra, ks));
    for (int ks = 0; ks < K / 16; ++ks) {
      if (use_tma >= 2)
        mma_bf16_ts(tbase, tbase + 128u + (uint32_t)(ks * 8), operand_desc(smem_u32(sb), b_mn, Rb, ks), idesc,
                    ks > 0 ? 1u : 0u);
      else
        mma_bf16(tbase, operand_desc(smem_u32(sa), a_mn, Ra, ks), operand_desc(smem_u32(sb), b_mn, Rb, ks), idesc,
                 ks > 0 ? 1u : 0u);
    }
    mma_commit(&bar_mma);
  }
  __syncwarp();
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  const int w = warp_id(), l = lane_id();
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t r[16];
    tmem_ld16(tbase + ((uint32_t)(32 * w) << 16) + (uint32_t)c0, r);
    int m = -1;
    if (M == 128) m = 32 * w + l;
    else if (l < 16) m = 16 * w + l;
    if (m >= 0)
      for (int e = 0; e < 16; ++e) d[(int64_t)m * N + c0 + e] = __uint_as_float(r[e]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc(tbase, 256);
}


// Variant: `issuers` warps each run their own ring of `stages` requests; a request is either
// one tensor-map box of (64 cols x box_rows x chunks) over a [rows][128] bf16 matrix (mode 0)
// or one 1-D cp.async.bulk of the same byte count from a contiguous random offset (mode 1).
__global__ void __launch_bounds__(512) k_tma_rate2(const __grid_constant__ CUtensorMap map, const uint8_t* gbuf,
                                                  int rows_total, int iters, int stages, int box_rows, int chunks,
                                                  int mode, unsigned long long* cycles) {
  extern __shared__ uint8_t smem_dyn[];
  __shared__ uint64_t full[4][8];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  const uint32_t bytes = (uint32_t)box_rows * 128u * (uint32_t)chunks;
  const int stride = max(1, mode >> 8);
  mode &= 0xff;
  const int w = (int)warp_id() / stride;
  const bool issuer = lane_id() == 0 && (int)warp_id() % stride == 0;
  if (issuer) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[w][s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (issuer) {
    uint8_t* mine = base + (size_t)w * stages * bytes;
    const int tiles = rows_total / box_rows;
    uint32_t r = ((uint32_t)blockIdx.x * 4u + (uint32_t)w) * 2654435761u;
    const uint64_t t0 = clock64();
    for (int i = 0; i < iters + stages; ++i) {
      const int s = i % stages;
      if (i >= stages) mbar_wait(&full[w][s], (uint32_t)((i - stages) / stages) & 1u);
      if (i < iters) {
        r = r * 1664525u + 1013904223u;
        const int tile = (int)((r >> 8) % (uint32_t)tiles);
        mbar_expect_tx(&full[w][s], bytes);
        if (mode == 0) {
          tma_load_5d(mine + s * bytes, &map, &full[w][s], 0, tile * box_rows, 0, 0, 0);
        } else {
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(mine + s * bytes)),
              "l"(gbuf + (size_t)tile * box_rows * 256), "r"(bytes), "r"(smem_u32(&full[w][s]))
              : "memory");
        }
      }
    }
    cycles[blockIdx.x * 4 + w] = clock64() - t0;
  }
}
}  // namespace
}  // namespace spa2

using namespace spa2;

extern "C" int spa2_probe_gemm(const void* a, const void* b, float* d, int m, int n, int k, int a_mn, int b_mn,
                               int use_tma, void* stream) {
  SPA2_REQUIRE(m == 64 || m == 128, SPA2_ERR_UNSUPPORTED, "probe: m must be 64 or 128");
  SPA2_REQUIRE(n == 64 || n == 128, SPA2_ERR_UNSUPPORTED, "probe: n must be 64 or 128");
  SPA2_REQUIRE(k == 64 || k == 128, SPA2_ERR_UNSUPPORTED, "probe: k must be 64 or 128");
  SPA2_REQUIRE(use_tma >= 0 && use_tma <= 3, SPA2_ERR_VALUE, "probe: mode must be 0..3");
  SPA2_REQUIRE(use_tma < 2 || (m == 128 && a_mn == 0), SPA2_ERR_UNSUPPORTED, "probe: TMEM A needs m=128, K-major");
  CUtensorMap ta, tb;
  memset(&ta, 0, sizeof(ta));
  memset(&tb, 0, sizeof(tb));
  if (use_tma == 1) {
    const int Ra = a_mn ? k : m, Ca = a_mn ? m : k;
    const int Rb = b_mn ? k : n, Cb = b_mn ? n : k;
    int rc = make_tma_bf16_2d(&ta, a, Ca, Ra, Ca, 64, Ra);
    if (rc) return rc;
    rc = make_tma_bf16_2d(&tb, b, Cb, Rb, Cb, 64, Rb);
    if (rc) return rc;
  }
  const size_t smem = 65536 + 1024;
  SPA2_CUDA_TRY(cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_probe<<<1, 128, smem, (cudaStream_t)stream>>>((const __nv_bfloat16*)a, (const __nv_bfloat16*)b, d, m, n, k,
                                                  a_mn, b_mn, use_tma, ta, tb);
  SPA2_LAUNCH_CHECK();
  return SPA2_OK;
}

// ---- tensor-pipe rate probe (diagnostic): cycles per tcgen05.mma for an operand layout ----
namespace spa2 {
namespace {
__global__ void __launch_bounds__(128) k_mma_rate(int M, int N, int K, int a_mn, int b_mn, int a_tmem, int reps,
                                                  unsigned long long* cycles) {
  extern __shared__ uint8_t smem_dyn[];
  __shared__ uint64_t bar_mma;
  __shared__ uint32_t tmem_base;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = base;
  uint8_t* sb = base + 65536;
  for (int i = threadIdx.x; i < 131072 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(base)[i] = make_uint4(0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u);
  const int Ra = a_mn ? K : M, Rb = b_mn ? K : N;
  if (warp_id() == 0) tmem_alloc(&tmem_base, 512);
  if (threadIdx.x == 32) {
    mbar_init(&bar_mma, 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16(M, N, a_mn != 0, b_mn != 0);
    uint64_t da[8], db[8];
    uint32_t ta[8];
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int kk = ks % (K / 16);
      da[ks] = operand_desc(smem_u32(sa), a_mn, Ra, kk);
      db[ks] = operand_desc(smem_u32(sb), b_mn, Rb, kk);
      ta[ks] = tbase + 256u + (uint32_t)(kk * 8);
    }
    const uint64_t t0 = clock64();
    if (a_tmem & 2) {  // weight-stationary form (tcgen05.mma.ws), A from TMEM (bit 0) or smem
      const bool at = (a_tmem & 1) != 0;
      for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          if (at)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.ws.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tbase),
                         "r"(ta[ks]), "l"(db[ks]), "r"(idesc), "r"(1u)
                         : "memory");
          else
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.ws.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tbase),
                         "l"(da[ks]), "l"(db[ks]), "r"(idesc), "r"(1u)
                         : "memory");
        }
      }
    } else if (a_tmem) {
      for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) mma_bf16_ts(tbase, ta[ks], db[ks], idesc, 1u);
      }
    } else {
      for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) mma_bf16(tbase, da[ks], db[ks], idesc, 1u);
      }
    }
    mma_commit(&bar_mma);
    mbar_wait(&bar_mma, 0);
    const uint64_t t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc(tbase, 512);
}
}  // namespace
}  // namespace spa2

extern "C" int spa2_probe_mma_rate(int m, int n, int k, int a_mn, int b_mn, int a_tmem, int reps, int ctas,
                                   unsigned long long* cycles, void* stream) {
  SPA2_REQUIRE((m == 64 || m == 128) && (n == 64 || n == 128 || n == 256) && (k == 64 || k == 128), SPA2_ERR_UNSUPPORTED,
               "mma_rate: unsupported shape");
  const size_t smem = 131072 + 1024;
  SPA2_CUDA_TRY(cudaFuncSetAttribute(k_mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_mma_rate<<<ctas, 128, smem, (cudaStream_t)stream>>>(m, n, k, a_mn, b_mn, a_tmem, reps, cycles);
  SPA2_LAUNCH_CHECK();
  return SPA2_OK;
}

// ---- MMA mix probe (diagnostic): the dQ kernel's per-tile MMA sequence in isolation ----
// S (8 TS steps, N=64) + dP (8 TS steps) + dQ (4 TS steps, N=128) per rep, buffers
// alternating like the kernel.  flags: 1 = random operand data, 2 = 256 noise threads doing
// tcgen05.ld/st on other TMEM columns, 4 = SS form (A from smem) for S/dP,
// 8 = wait for each rep's completion before the next (serialised), 16 = S only (8 steps),
// 32 = accumulate into D from the first step too, 64 = one S/dP buffer (no alternation),
// 128 = S B operand from the same K=16 slab every step (no k offset),
// 256 = warp-collective issue with precomputed descriptors (TS, the kernels' new form),
// 512 = (with 256) commit to mbarriers after each group like the kernel,
// 1024 = (with 256) wait for the S group's commit before issuing dP (a dependent consumer),
// 2048 = two extra warps stream 16 KB bulk copies from `gsrc` into unused smem meanwhile.
namespace spa2 {
namespace {
__global__ void __launch_bounds__(448) k_mma_mix(int reps, int flags, const uint8_t* gsrc, unsigned long long* cycles) {
  extern __shared__ uint8_t smem_dyn[];
  __shared__ uint64_t bar_mma, bars[8];
  __shared__ uint32_t tmem_base;
  __shared__ volatile int stop;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 131072 / 16; i += blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u + 12345u;
    const uint32_t v = (flags & 1) ? ((x >> 9) & 0x007f007fu) | 0x3c003c00u : 0x3f803f80u;
    reinterpret_cast<uint4*>(base)[i] = make_uint4(v, v ^ 0x00010001u, v, v ^ 0x00020002u);
  }
  if (warp_id() == 0) tmem_alloc(&tmem_base, 512);
  if (threadIdx.x == 32) {
    mbar_init(&bar_mma, 1);
    for (int i = 0; i < 8; ++i) mbar_init(&bars[i], 1);
    stop = 0;
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  const uint32_t sK = smem_u32(base), sV = sK + 16384, sQ = sK + 32768, sDO = sK + 65536;
  if ((flags & 4096) && warp_id() < 3) {
    // three warps issue the S, dP and dQ streams concurrently (no cross-stream waits)
    constexpr uint32_t idS = idesc_bf16(128, 64, false, false);
    constexpr uint32_t idQ = idesc_bf16(128, 128, false, true);
    const uint64_t dK = sw128_desc(sK, 16, 1024), dV = sw128_desc(sV, 16, 1024);
    const uint64_t dKm = sw128_desc(sK, 64 * 128, 1024);
    const int w = (int)warp_id();
    const uint64_t t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t sb = tbase + 128u + (uint32_t)((r & 1) * 128);
      if (w == 0) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          mma_bf16_ts_w(sb, tbase + (uint32_t)(ks * 8), dK + (uint64_t)((((ks / 4) * 64 * 128 + (ks % 4) * 32)) >> 4), idS,
                        ks > 0 ? 1u : 0u);
      } else if (w == 1) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          mma_bf16_ts_w(sb + 64, tbase + 64u + (uint32_t)(ks * 8),
                        dV + (uint64_t)((((ks / 4) * 64 * 128 + (ks % 4) * 32)) >> 4), idS, ks > 0 ? 1u : 0u);
      } else {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          mma_bf16_ts_w(tbase + 384u, sb + (uint32_t)(32 * (ks >> 1) + 8 * (ks & 1)), dKm + (uint64_t)((ks * 2048) >> 4),
                        idQ, 1u);
      }
      if (flags & 512) mma_commit_w(&bars[w]);
    }
    mma_commit_w(&bars[4 + w]);
    mbar_wait(&bars[4 + w], 0);
    if (lane_id() == 0) atomicMax(reinterpret_cast<unsigned long long*>(&cycles[blockIdx.x]), clock64() - t0);
    if (w == 0) {
      __syncwarp();
    }
    stop = 1;
  } else if ((flags & 256) && warp_id() == 0) {
    constexpr uint32_t idS = idesc_bf16(128, 64, false, false);
    constexpr uint32_t idQ = idesc_bf16(128, 128, false, true);
    const uint64_t dK = sw128_desc(sK, 16, 1024), dV = sw128_desc(sV, 16, 1024);
    const uint64_t dKm = sw128_desc(sK, 64 * 128, 1024);
    const uint64_t t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t sb = tbase + 128u + (uint32_t)((r & 1) * 128);
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)
        mma_bf16_ts_w(sb, tbase + (uint32_t)(ks * 8), dK + (uint64_t)((((ks / 4) * 64 * 128 + (ks % 4) * 32)) >> 4), idS,
                      ks > 0 ? 1u : 0u);
      if (flags & 1536) mma_commit_w(&bars[0]);
      if (flags & 1024) mbar_wait(&bars[0], (uint32_t)r & 1u);
      if (!(flags & 16)) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          mma_bf16_ts_w(sb + 64, tbase + 64u + (uint32_t)(ks * 8),
                        dV + (uint64_t)((((ks / 4) * 64 * 128 + (ks % 4) * 32)) >> 4), idS, ks > 0 ? 1u : 0u);
        if (flags & 512) {
          mma_commit_w(&bars[1]);
          mma_commit_w(&bars[2]);
        }
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          mma_bf16_ts_w(tbase + 384u, sb + (uint32_t)(32 * (ks >> 1) + 8 * (ks & 1)), dKm + (uint64_t)((ks * 2048) >> 4),
                        idQ, 1u);
        if (flags & 512) {
          mma_commit_w(&bars[3]);
          mma_commit_w(&bars[4]);
        }
      }
    }
    mma_commit_w(&bar_mma);
    mbar_wait(&bar_mma, 0);
    if (lane_id() == 0) cycles[blockIdx.x] = clock64() - t0;
    stop = 1;
  } else if (threadIdx.x == 0 && !(flags & 256)) {
    constexpr uint32_t idS = idesc_bf16(128, 64, false, false);
    constexpr uint32_t idQ = idesc_bf16(128, 128, false, true);
    const uint64_t t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t sb = tbase + 128u + (uint32_t)((flags & 64) ? 0 : (r & 1) * 128);
      const uint32_t acc0 = (flags & 32) ? 1u : 0u;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const uint32_t ko = (flags & 128) ? 0u : (uint32_t)((ks / 4) * 64 * 128 + (ks % 4) * 32);
        const uint32_t qo = (uint32_t)((ks / 4) * 128 * 128 + (ks % 4) * 32);
        if (flags & 4) mma_bf16(sb, sw128_desc(sQ + qo, 16, 1024), sw128_desc(sK + ko, 16, 1024), idS, ks > 0 ? 1u : acc0);
        else mma_bf16_ts(sb, tbase + (uint32_t)(ks * 8), sw128_desc(sK + ko, 16, 1024), idS, ks > 0 ? 1u : acc0);
      }
      if (!(flags & 16)) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const uint32_t ko = (uint32_t)((ks / 4) * 64 * 128 + (ks % 4) * 32);
          const uint32_t qo = (uint32_t)((ks / 4) * 128 * 128 + (ks % 4) * 32);
          if (flags & 4) mma_bf16(sb + 64, sw128_desc(sDO + qo, 16, 1024), sw128_desc(sV + ko, 16, 1024), idS, ks > 0);
          else mma_bf16_ts(sb + 64, tbase + 64u + (uint32_t)(ks * 8), sw128_desc(sV + ko, 16, 1024), idS, ks > 0);
        }
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          mma_bf16_ts(tbase + 384u, sb + (uint32_t)(32 * (ks >> 1) + 8 * (ks & 1)),
                      sw128_desc(sK + (uint32_t)(ks * 2048), 64 * 128, 1024), idQ, 1u);
      }
      if (flags & 8) {
        mma_commit(&bar_mma);
        mbar_wait(&bar_mma, (uint32_t)r & 1u);
      }
    }
    mma_commit(&bar_mma);
    if (!(flags & 8)) mbar_wait(&bar_mma, 0);
    else mbar_wait(&bar_mma, (uint32_t)reps & 1u);
    cycles[blockIdx.x] = clock64() - t0;
    stop = 1;
  } else if (threadIdx.x >= 384 && (flags & 2048)) {
    // TMA noise: two warps, each with a 2-deep ring of 16 KB bulk copies into [96 KB, 128 KB)
    if (lane_id() == 0) {
      const int w = (int)warp_id() - 12;
      uint64_t* fb = &bars[5 + w];
      uint8_t* dst = base + 98304 + w * 16384;
      uint32_t ph = 0;
      uint32_t x = 12345u + (uint32_t)w;
      while (!stop) {
        x = x * 1664525u + 1013904223u;
        mbar_expect_tx(fb, 16384);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(dst)),
                     "l"(gsrc + (size_t)((x >> 8) % 1024) * 16384), "r"(16384), "r"(smem_u32(fb))
                     : "memory");
        mbar_wait(fb, ph);
        ph ^= 1u;
      }
    }
  } else if (threadIdx.x >= 128 && threadIdx.x < 384 && (flags & 2)) {
    // noise: tcgen05.ld/st on columns [256, 384) of this warp's lane quarter
    const int w = (int)warp_id();
    const uint32_t lane_off = (uint32_t)((w & 3) * 32) << 16;
    uint32_t acc = 0;
    while (!stop) {
      uint32_t r32[32];
      tmem_ld32(tbase + lane_off + 256u + (uint32_t)(32 * ((w >> 2) & 1)), r32);
      uint32_t pk[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) pk[c] = r32[2 * c] ^ r32[2 * c + 1];
      tmem_st16(tbase + lane_off + 256u + (uint32_t)(32 * ((w >> 2) & 1)), pk);
      tmem_st_wait();
      acc += pk[0];
    }
    if (acc == 0xdeadbeefu) cycles[gridDim.x] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc(tbase, 512);
}
}  // namespace
}  // namespace spa2

extern "C" int spa2_probe_mma_mix(int reps, int flags, int ctas, const void* gsrc, unsigned long long* cycles,
                                  void* stream) {
  const size_t smem = 131072 + 1024;
  SPA2_CUDA_TRY(cudaFuncSetAttribute(k_mma_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_mma_mix<<<ctas, (flags & 2048) ? 448 : (flags & 2) ? 384 : 128, smem, (cudaStream_t)stream>>>(
      reps, flags, (const uint8_t*)gsrc, cycles);
  SPA2_LAUNCH_CHECK();
  return SPA2_OK;
}

// ---- TMA streaming-rate probe (diagnostic): L2/HBM -> SMEM bandwidth with no compute ----
namespace spa2 {
namespace {
__global__ void __launch_bounds__(32) k_tma_rate(const __grid_constant__ CUtensorMap map, int rows_total, int iters,
                                                 int stages, int box_rows, unsigned long long* cycles) {
  extern __shared__ uint8_t smem_dyn[];
  __shared__ uint64_t full[8];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  const uint32_t bytes = (uint32_t)box_rows * 128u;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (threadIdx.x == 0) {
    const int tiles = rows_total / box_rows;
    uint32_t r = (uint32_t)blockIdx.x * 2654435761u;
    const uint64_t t0 = clock64();
    for (int i = 0; i < iters + stages; ++i) {
      const int s = i % stages;
      if (i >= stages) mbar_wait(&full[s], (uint32_t)((i - stages) / stages) & 1u);
      if (i < iters) {
        r = r * 1664525u + 1013904223u;
        mbar_expect_tx(&full[s], bytes);
        tma_load_2d(base + s * bytes, &map, &full[s], 0, (int)((r >> 8) % (uint32_t)tiles) * box_rows);
      }
    }
    cycles[blockIdx.x] = clock64() - t0;
  }
}
}  // namespace
}  // namespace spa2

extern "C" int spa2_probe_tma_rate(const void* buf, long long rows, int box_rows, int stages, int iters, int ctas,
                                   unsigned long long* cycles, void* stream) {
  SPA2_REQUIRE(stages >= 1 && stages <= 8 && box_rows >= 8 && box_rows <= 256, SPA2_ERR_VALUE, "tma_rate: bad args");
  CUtensorMap map;
  int rc = make_tma_bf16_2d(&map, buf, 64, (uint64_t)rows, 64, 64, (uint32_t)box_rows);
  if (rc) return rc;
  const size_t smem = (size_t)stages * box_rows * 128 + 1024;
  SPA2_CUDA_TRY(cudaFuncSetAttribute(k_tma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_tma_rate<<<ctas, 32, smem, (cudaStream_t)stream>>>(map, (int)rows, iters, stages, box_rows, cycles);
  SPA2_LAUNCH_CHECK();
  return SPA2_OK;
}

extern "C" int spa2_probe_tma_rate2(const void* buf, long long rows, int box_rows, int chunks, int stages, int issuers,
                                    int mode, int iters, int ctas, unsigned long long* cycles, void* stream) {
  SPA2_REQUIRE(stages >= 1 && stages <= 8 && issuers >= 1 && issuers <= 4 && box_rows >= 8 && box_rows <= 256 &&
                   (chunks == 1 || chunks == 2),
               SPA2_ERR_VALUE, "tma_rate2: bad args");
  CUtensorMap map;
  const uint64_t dims[5] = {64, (uint64_t)rows, 2, 1, 1};
  const uint64_t strides[4] = {256, 128, (uint64_t)rows * 256, (uint64_t)rows * 256};
  const uint32_t box[5] = {64, (uint32_t)box_rows, (uint32_t)chunks, 1, 1};
  int rc = make_tma_bf16_5d(&map, buf, dims, strides, box);
  if (rc) return rc;
  const size_t smem = (size_t)issuers * stages * box_rows * 128 * chunks + 1024;
  SPA2_REQUIRE(smem <= 232448, SPA2_ERR_VALUE, "tma_rate2: %zu bytes of smem", smem);
  SPA2_CUDA_TRY(cudaFuncSetAttribute(k_tma_rate2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_tma_rate2<<<ctas, 32 * issuers * max(1, mode >> 8), smem, (cudaStream_t)stream>>>(map, (const uint8_t*)buf, (int)rows, iters, stages,
                                                                  box_rows, chunks, mode, cycles);
  SPA2_LAUNCH_CHECK();
  return SPA2_OK;
}

// ---- TMEM load/store rate probe (diagnostic): tcgen05.ld / tcgen05.st bytes per cycle per SM ----
namespace spa2 {
namespace {
__global__ void __launch_bounds__(512, 1) k_tmem_rate(int reps, int mode, unsigned long long* cycles) {
  __shared__ uint32_t holder;
  const int warp = (int)warp_id();
  if (warp == 0) tmem_alloc(&holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = holder;
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const uint32_t col = (uint32_t)((warp >> 2) * 32) & 511u;
  uint32_t acc = 0;
  __syncthreads();
  if (mode >= 4) {
    // modes 4/5: warp 0 keeps the tensor core busy with N=128 SS MMAs into columns [384, 512)
    // (mode 5: N=64 into [448, 512)) while the other warps time 32-column loads of [0, 256)
    extern __shared__ __align__(1024) uint8_t ops[];
    __shared__ volatile int stop;
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
      stop = 0;
      mbar_init(&bar, 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (warp == 0) {
      const uint64_t da = sw128_desc(smem_u32(ops), 16, 1024), db = sw128_desc(smem_u32(ops) + 16384, 16, 1024);
      const uint32_t id = mode == 4 ? idesc_bf16(128, 128, false, false) : idesc_bf16(128, 64, false, false);
      const uint32_t dcol = mode == 4 ? 384u : 448u;
      int n = 0;
      while (!stop) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) mma_bf16_w(tbase + dcol, da + (uint64_t)(ks * 2), db + (uint64_t)(ks * 2), id, ks > 0);
        ++n;
      }
      mma_commit_w(&bar);
      mbar_wait(&bar, 0);
      if (lane_id() == 0) cycles[blockIdx.x * 16] = (unsigned long long)n;
    } else {
      const uint64_t t0 = clock64();
      for (int i = 0; i < reps; ++i) {
        uint32_t r[32];
        tmem_ld32(tbase + lane_off + ((col + (uint32_t)i * 64u) & 255u), r);
#pragma unroll
        for (int c = 0; c < 32; ++c) acc ^= r[c];
      }
      const uint64_t t1 = clock64();
      if ((threadIdx.x & 31) == 0) cycles[blockIdx.x * 16 + warp] = t1 - t0;
      asm volatile("bar.sync 1, %0;" ::"r"((int)blockDim.x - 32));
      if (threadIdx.x == 32) stop = 1;
    }
    if (acc == 0xdeadbeefu) cycles[0] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tbase, 512);
    return;
  }
  const uint64_t t0 = clock64();
  if (mode == 0) {
    for (int i = 0; i < reps; ++i) {
      uint32_t r[32];
      tmem_ld32(tbase + lane_off + ((col + (uint32_t)i * 64u) & 511u), r);
#pragma unroll
      for (int c = 0; c < 32; ++c) acc ^= r[c];
    }
  } else if (mode == 1) {
    for (int i = 0; i < reps; i += 2) {
      uint32_t r[64];
      tmem_ld64(tbase + lane_off + ((col + (uint32_t)i * 64u) & 447u), r);
#pragma unroll
      for (int c = 0; c < 64; ++c) acc ^= r[c];
    }
  } else if (mode == 2) {
    for (int i = 0; i < reps; ++i) {
      uint32_t r[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) r[c] = acc + (uint32_t)c;
      tmem_ld16(tbase + lane_off + ((col + (uint32_t)i * 64u) & 511u), r);
#pragma unroll
      for (int c = 0; c < 16; ++c) acc ^= r[c];
    }
  } else {
    for (int i = 0; i < reps; ++i) {
      uint32_t r[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) r[c] = acc + (uint32_t)c;
      tmem_st16(tbase + lane_off + ((col + (uint32_t)i * 64u) & 511u), r);
      tmem_st_wait();
      acc += 1;
    }
  }
  const uint64_t t1 = clock64();
  __syncthreads();
  if ((threadIdx.x & 31) == 0) cycles[blockIdx.x * 16 + warp] = t1 - t0;
  if (acc == 0xdeadbeefu) cycles[0] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 512);
}
}  // namespace
}  // namespace spa2

// mode 0: 32-column loads (4 KB per warp instruction), 1: two 32-column loads per wait,
// 2: 16-column loads, 3: 16-column stores, 4/5: 32-column loads by warps 1.. while warp 0
// streams N=128 / N=64 MMAs (cycles[cta*16] = MMA groups issued).  cycles[ctas * 16] per warp.
extern "C" int spa2_probe_tmem_rate(int reps, int mode, int warps, int ctas, unsigned long long* cycles, void* stream) {
  const int smem = mode >= 4 ? 32768 + 1024 : 0;
  if (mode >= 4) SPA2_CUDA_TRY(cudaFuncSetAttribute(k_tmem_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_tmem_rate<<<ctas, 32 * warps, smem, (cudaStream_t)stream>>>(reps, mode, cycles);
  SPA2_LAUNCH_CHECK();
  return SPA2_OK;
}

// ---- mbarrier wait latency probe (diagnostic): cycles per try_wait / test_wait on a phase
// that has ALREADY completed (the cost a consumer pays even when it never has to wait) ----
namespace spa2 {
namespace {
__global__ void k_mbar_lat(int reps, int mode, unsigned long long* cycles) {
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) mbar_arrive(&bar);  // phase 0 completes
  __syncthreads();
  uint32_t ok = 0;
  const uint64_t t0 = clock64();
  for (int i = 0; i < reps; ++i) {
    if (mode == 0) ok += mbar_try_wait(smem_u32(&bar), 0u);
    else if (mode == 1) ok += mbar_test(&bar, 0u) ? 1u : 0u;
    else {
      mbar_wait(&bar, 0u);
      ok += 1;
    }
  }
  const uint64_t t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  if (ok == 0xdeadbeefu) cycles[1] = ok;
}
}  // namespace
}  // namespace spa2

// mode 0: mbarrier.try_wait, 1: mbarrier.test_wait, 2: mbar_wait() — each on a completed phase.
extern "C" int spa2_probe_mbar_latency(int reps, int mode, int threads, unsigned long long* cycles, void* stream) {
  k_mbar_lat<<<1, threads, 0, (cudaStream_t)stream>>>(reps, mode, cycles);
  SPA2_LAUNCH_CHECK();
  return SPA2_OK;
}

namespace spa2 {
namespace {
// fp32 reduction throughput into L2: each CTA adds `tiles` 128 x 128 fp32 tiles (one row of 128
// floats = 512 B per thread, red.global.add.v4.f32) into a rotating set of `nslots` tiles of `dst`
// (the access pattern of a dQ partial per kept tile in a fused backward).  mode 1: plain
// st.global.v4 instead (store bandwidth reference).
__global__ void __launch_bounds__(128) k_red_rate(float* __restrict__ dst, int tiles, int nslots, int mode) {
  // mode 0/1: thread = row (the TMEM lane layout of a partial); mode 2: coalesced — each warp
  // covers 512 contiguous bytes per instruction (a transposed / staged partial)
  const int row = mode == 2 ? (threadIdx.x / 32) * 32 + 0 : threadIdx.x;
  float v = 1.0f + 1e-3f * (float)threadIdx.x;
  for (int t = 0; t < tiles; ++t) {
    const int slot = (blockIdx.x * 7 + t * 13) % nslots;
    if (mode == 2) {
      float* base = dst + (int64_t)slot * 128 * 128;
#pragma unroll 8
      for (int i = 0; i < 32; ++i) {  // 128 threads x 16 B x 32 = 64 KB
        float* p = base + (int64_t)(i * 128 + threadIdx.x) * 4;
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v), "f"(v), "f"(v), "f"(v)
                     : "memory");
      }
      continue;
    }
    float* p = dst + ((int64_t)slot * 128 + row) * 128;
#pragma unroll 8
    for (int c = 0; c < 128; c += 4) {
      if (mode == 0)
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p + c), "f"(v), "f"(v), "f"(v), "f"(v)
                     : "memory");
      else
        asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p + c), "f"(v), "f"(v), "f"(v), "f"(v)
                     : "memory");
    }
  }
}
}  // namespace
}  // namespace spa2

// mode 3: the TMA bulk-reduce path a fused backward would use — each CTA holds one 64 KB fp32
// partial in shared memory and adds it into a global tile with cp.reduce.async.bulk .add.f32 (four
// 16 KB requests per tile from one elected thread, up to 4 tiles in flight).
namespace spa2 {
namespace {
__global__ void __launch_bounds__(128) k_red_bulk(float* __restrict__ dst, int tiles, int nslots) {
  extern __shared__ __align__(128) uint8_t smem_red[];
  float* part = reinterpret_cast<float*>(smem_red);
  for (int i = threadIdx.x; i < 128 * 128; i += blockDim.x) part[i] = 1.0f + 1e-3f * (float)(i & 127);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int t = 0; t < tiles; ++t) {
      const int slot = (blockIdx.x * 7 + t * 13) % nslots;
      float* base = dst + (int64_t)slot * 128 * 128;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(base + c * 4096),
                     "r"(smem_u32(part + c * 4096)), "r"(16384)
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  __syncthreads();
}
}  // namespace
}  // namespace spa2

extern "C" int spa2_probe_red_rate(float* dst, int tiles, int nslots, int ctas, int mode, void* stream) {
  if (mode == 3) {
    const int smem = 128 * 128 * 4;
    SPA2_CUDA_TRY(cudaFuncSetAttribute(spa2::k_red_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    spa2::k_red_bulk<<<ctas, 128, smem, (cudaStream_t)stream>>>(dst, tiles, nslots);
  } else {
    spa2::k_red_rate<<<ctas, 128, 0, (cudaStream_t)stream>>>(dst, tiles, nslots, mode);
  }
  SPA2_LAUNCH_CHECK();
  return SPA2_OK;
}

// ---- SM clock probe (diagnostic): the clock the SMs run at right now ----
// Each CTA spins `spin_ns` of %globaltimer and records (Δclock64, Δglobaltimer); launched right
// after a hot kernel on the same stream it reports the clock the power manager had settled on
// for that kernel (the regulator reacts on a millisecond scale; NVML's samples are coarser).
namespace spa2 {
namespace {
__global__ void k_probe_clock(int spin_ns, unsigned long long* out) {
  if (threadIdx.x != 0) return;
  unsigned long long g0, g1, c0, c1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  } while (g1 - g0 < (unsigned long long)spin_ns);
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c1));
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  out[2 * blockIdx.x] = c1 - c0;
  out[2 * blockIdx.x + 1] = g1 - g0;
}
}  // namespace
}  // namespace spa2

extern "C" int spa2_probe_clock(int spin_ns, int ctas, unsigned long long* out, void* stream) {
  SPA2_REQUIRE(spin_ns > 0 && ctas > 0 && out, SPA2_ERR_VALUE, "probe_clock: bad arguments");
  spa2::k_probe_clock<<<ctas, 32, 0, (cudaStream_t)stream>>>(spin_ns, out);
  SPA2_LAUNCH_CHECK();
  return SPA2_OK;
}

// ---- shared-memory contention probe (diagnostic) ----
// Does other traffic slow the tensor core's SS operand reads?  Warp 0 issues reps x 8 SS MMAs
// M=128 N=64 K=16 (A 128x128 and B 64x128 bf16, K-major SW128, 6 KB of operands per MMA) and
// times them; meanwhile, by `mode` bits, warps 1-2 stream 16 KB bulk copies global->smem (1),
// warps 4-7 store STS.128 (2), warps 8-11 load LDS.128 (4), warps 4-7 instead load TMEM with
// tcgen05.ld.32x32b.x32 from other columns (8, replaces 2), and (16) each rep's A operand rotates
// over three 32 KB tiles.  out[cta*4 + {0,1,2,3}] = MMA cycles, bulk bytes, STS or TMEM bytes,
// LDS bytes moved while the MMAs ran.
namespace spa2 {
namespace {
__global__ void __launch_bounds__(384) k_smem_contend(int reps, int mode, const uint8_t* gsrc,
                                                     unsigned long long* out) {
  extern __shared__ uint8_t smem_dyn[];
  __shared__ uint64_t bar_mma, bars[2];
  __shared__ uint32_t tmem_base;
  __shared__ volatile int stop;
  __shared__ unsigned long long moved[3];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  // [0, 96K) three A tiles | [96K, 112K) B | [112K, 144K) bulk | [144K, 160K) STS | [160K, 176K) LDS
  for (int i = threadIdx.x; i < 114688 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(base)[i] = make_uint4(0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u);
  if (warp_id() == 0) tmem_alloc(&tmem_base, 512);
  if (threadIdx.x == 32) {
    mbar_init(&bar_mma, 1);
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    stop = 0;
    moved[0] = moved[1] = moved[2] = 0;
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  const int warp = (int)warp_id();
  if (warp == 0) {
    // warp-collective batched issue exactly as in the kernels (one elect per 8-step group)
    constexpr uint32_t idS = idesc_bf16(128, 64, false, false);
    const uint64_t dA = sw128_desc(smem_u32(base), 16, 1024);
    const uint64_t dB = sw128_desc(smem_u32(base + 98304), 16, 1024);
    const bool rot = (mode & 16) != 0;
    const bool ts = (mode & 32) != 0;  // A from TMEM columns [384, 448) (TS form, 32-cycle steps)
    const uint64_t t0 = clock64();
    if (ts) {
      for (int r = 0; r < reps; ++r)
        mma_bf16_ts_k8_w<8u, 2ull, (uint64_t)(64 * 128 / 16)>(tbase + (uint32_t)((r & 3) * 64), tbase + 384u, dB, idS, 0u);
    } else {
      for (int r = 0; r < reps; ++r) {
        const uint64_t aoff = rot ? (uint64_t)(((r % 3) * 32768) >> 4) : 0ull;
        mma_bf16_ss_k8_w<2ull, (uint64_t)(128 * 128 / 16), 2ull, (uint64_t)(64 * 128 / 16)>(
            tbase + (uint32_t)((r & 3) * 64), dA + aoff, dB, idS, 0u);
      }
    }
    mma_commit_w(&bar_mma);
    mbar_wait(&bar_mma, 0);
    if (lane_id() == 0) out[blockIdx.x * 4] = clock64() - t0;
    __syncwarp();
    if (lane_id() == 0) stop = 1;
  } else if ((warp == 1 || warp == 2) && (mode & 1)) {
    if (lane_id() == 0) {
      const int w = warp - 1;
      uint8_t* dst = base + 114688 + w * 16384;
      uint32_t ph = 0, x = 777u + (uint32_t)w;
      unsigned long long n = 0;
      while (!stop) {
        x = x * 1664525u + 1013904223u;
        mbar_expect_tx(&bars[w], 16384);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(dst)),
                     "l"(gsrc + (size_t)((x >> 8) % 1024) * 16384), "r"(16384), "r"(smem_u32(&bars[w]))
                     : "memory");
        mbar_wait(&bars[w], ph);
        ph ^= 1u;
        n += 16384;
      }
      atomicAdd(&moved[0], n);
    }
  } else if (warp >= 4 && warp < 8 && (mode & 8)) {
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    unsigned long long n = 0;
    uint32_t acc = 0;
    while (!stop) {
      uint32_t r[32];
      tmem_ld32(tbase + lane_off + 256u + (uint32_t)((n >> 7) & 3) * 32u, r);
#pragma unroll
      for (int i = 0; i < 32; ++i) acc ^= r[i];
      n += 128;
    }
    if (acc == 0x12345678u) n += 1;
    atomicAdd(&moved[1], n);
  } else if (warp >= 4 && warp < 8 && (mode & 2)) {
    const uint32_t dst = smem_u32(base + 147456) + (uint32_t)((warp - 4) * 4096);
    unsigned long long n = 0;
    uint32_t v = threadIdx.x;
    while (!stop) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        st_shared_v4(dst + (uint32_t)(((u * 32 + (int)lane_id()) * 16) & 4095), v, v + 1, v + 2, v + 3);
        ++v;
      }
      n += 8 * 16;
    }
    atomicAdd(&moved[1], n);
  } else if (warp >= 8 && (mode & 4)) {
    const uint4* src = reinterpret_cast<const uint4*>(base + 163840 + (warp - 8) * 4096);
    unsigned long long n = 0;
    uint32_t acc = 0;
    while (!stop) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        uint32_t x0, x1, x2, x3;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3)
                     : "r"(smem_u32(src + ((u * 32 + (int)lane_id()) & 255))));
        acc ^= x0 ^ x1 ^ x2 ^ x3;
      }
      n += 8 * 16;
    }
    if (acc == 0x12345678u) n += 1;  // keep the loads
    atomicAdd(&moved[2], n);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    out[blockIdx.x * 4 + 1] = moved[0];
    out[blockIdx.x * 4 + 2] = moved[1];
    out[blockIdx.x * 4 + 3] = moved[2];
  }
  if (warp == 0) tmem_dealloc(tbase, 512);
}
}  // namespace
}  // namespace spa2

extern "C" int spa2_probe_smem_contend(int reps, int mode, int ctas, const void* gsrc, unsigned long long* out,
                                       void* stream) {
  const size_t smem = 180224 + 1024;
  SPA2_CUDA_TRY(cudaFuncSetAttribute(spa2::k_smem_contend, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  spa2::k_smem_contend<<<ctas, 384, smem, (cudaStream_t)stream>>>(reps, mode, (const uint8_t*)gsrc, out);
  SPA2_LAUNCH_CHECK();
  return SPA2_OK;
}

// ---- dK/dV MMA mix probe (diagnostic): the K6 kernel's four MMA groups per tile in isolation ----
// S = Q Kᵀ, dP = dO Vᵀ (M=128 N=64, K-major SW128 A and B), dVᵀ += dOᵀ P, dKᵀ += Qᵀ dS (M=128 N=64,
// MN-major A and B), each 8 K=16 steps, with exactly the kernel's descriptors and its
// warp-collective batched issue (mma_bf16_ss_k8_w), back to back without dependencies.
// which: bits 0-1: 0 = all four per tile, 1 = S and dP only, 2 = dVᵀ and dKᵀ only; 32 = S only;
// 64 = issue from a single thread (one MMA per asm block) instead of the warp batch.
// cycles[cta] = clock64 span of reps tiles.
namespace spa2 {
namespace {
__global__ void __launch_bounds__(128) k_dkdv_mix(int reps, int which, unsigned long long* cycles) {
  extern __shared__ uint8_t smem_dyn[];
  __shared__ uint64_t bar_mma;
  __shared__ uint32_t tmem_base;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 196608 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(base)[i] = make_uint4(0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u);
  if (warp_id() == 0) tmem_alloc(&tmem_base, 512);
  if (threadIdx.x == 32) {
    mbar_init(&bar_mma, 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  const bool single = (which & 64) != 0;
  const bool ts = (which & 128) != 0;
  __shared__ volatile int stop_flag;
  __shared__ unsigned long long staged[4];
  if (threadIdx.x == 0) stop_flag = 0;
  __syncthreads();
  if (warp_id() != 0 && (which & 256)) {
    // Q / dO staging traffic as a TS-MMA K6 would add: each warp reads its 32 rows of a
    // K-major SW128 128 x 128 tile (LDS.128, conflict-free) and stores them into TMEM columns
    // [384, 448) of its lane quarter (tcgen05.st), until warp 0's MMA chain is done.
    // region (bits 8192 / 16384): the Q tile S reads (default), the P tile dVᵀ reads, or
    // [160K, 192K) which no MMA reads
    const uint32_t row = (warp_id() & 3) * 32 + lane_id();
    // (bit 32768: region at ((which >> 16) & 15) x 16 KB instead)
    const uint32_t src = smem_u32(base) + ((which & 32768) ? (uint32_t)(((which >> 16) & 15) * 16384)
                                           : (which & 8192) ? 98304u : (which & 16384) ? 163840u : 0u);
    const uint32_t tq = tbase + ((uint32_t)((warp_id() & 3) * 32) << 16) + 384u;
    unsigned long long n = 0;
    while (!stop_flag) {
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        uint32_t r[32];
        if (which & 2048) {  // mbarrier polls (try_wait on a phase that never completes) at the region
          if (lane_id() == 0 && warp_id() == 1 && h == 0 && n == 0) mbar_init(reinterpret_cast<uint64_t*>(base + (src - smem_u32(base))), 1);
          __syncwarp();
          uint32_t spins = 0;
#pragma unroll 1
          for (int i = 0; i < 64; ++i) spins += mbar_try_wait(src, 1u);
          n += 64 + (spins & 0);  // counts polls, not bytes
          continue;
        }
        if (which & 4096) {  // shared-memory stores only (STS.128 of swizzled rows, like P / dS)
#pragma unroll
          for (int u = 0; u < 8; ++u)
            st_shared_v4(src + (uint32_t)(h * 16384) + sw128_offset(row, (uint32_t)u), (uint32_t)n, u, h, 1u);
          n += 32 * 128;
          continue;
        }
        if (which & 512) {  // TMEM stores only (register data, no shared-memory reads)
#pragma unroll
          for (int u = 0; u < 32; ++u) r[u] = (uint32_t)(n + u);
        } else if (which & 1024) {  // shared-memory reads only (no TMEM stores)
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const uint4 v = ld_shared_v4(src + (uint32_t)(h * 16384) + sw128_offset(row, (uint32_t)u));
            r[4 * u] = v.x; r[4 * u + 1] = v.y; r[4 * u + 2] = v.z; r[4 * u + 3] = v.w;
          }
          uint32_t x = 0;
#pragma unroll
          for (int u = 0; u < 32; ++u) x ^= r[u];
          if (x == 0x12345678u) staged[0] = x;  // keep the loads
          n += 32 * 128;
          continue;
        } else {
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const uint4 v = ld_shared_v4(src + (uint32_t)(h * 16384) + sw128_offset(row, (uint32_t)u));
            r[4 * u] = v.x; r[4 * u + 1] = v.y; r[4 * u + 2] = v.z; r[4 * u + 3] = v.w;
          }
        }
        tmem_st32(tq + (uint32_t)(h * 32), r);
        tmem_st_wait();
        n += 32 * 128;
      }
    }
    if (lane_id() == 0) staged[warp_id()] = n;
  }
  if (warp_id() == 0 && (!single || lane_id() == 0)) {
    // [0,32K) Q | [32K,64K) dO | [64K,80K) K | [80K,96K) V | [96K,112K) P | [112K,128K) dS
    constexpr uint32_t idS = idesc_bf16(128, 64, false, false);
    constexpr uint32_t idT = idesc_bf16(128, 64, true, true);
    const uint64_t dQk = sw128_desc(smem_u32(base), 16, 1024), dDOk = sw128_desc(smem_u32(base + 32768), 16, 1024);
    const uint64_t dK = sw128_desc(smem_u32(base + 65536), 16, 1024), dV = sw128_desc(smem_u32(base + 81920), 16, 1024);
    const uint64_t dQm = sw128_desc(smem_u32(base), 128 * 128, 1024), dDOm = sw128_desc(smem_u32(base + 32768), 128 * 128, 1024);
    const uint64_t dPm = sw128_desc(smem_u32(base + 98304), 128 * 128, 1024), dDSm = sw128_desc(smem_u32(base + 114688), 128 * 128, 1024);
    const int w2 = which & 3;
    const uint64_t t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t b = (uint32_t)(r & 1) * 64u;
      if (w2 != 2 && ts) {
        // S and dP as TS MMAs: A (Q / dO, K-major bf16 pairs) from TMEM columns 384 / 448
        mma_bf16_ts_k8_w<8u, 2ull, (uint64_t)(64 * 128 / 16)>(tbase + b, tbase + 384u, dK, idS, 0u);
        if (!(which & 32))
          mma_bf16_ts_k8_w<8u, 2ull, (uint64_t)(64 * 128 / 16)>(tbase + 128u + b, tbase + 448u, dV, idS, 0u);
      } else if (w2 != 2) {
        if (single) {
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const uint64_t qo = (uint64_t)((((ks * 16) / 64) * 128 * 128 + ((ks * 16) % 64) * 2) >> 4);
            const uint64_t ko = (uint64_t)((((ks * 16) / 64) * 64 * 128 + ((ks * 16) % 64) * 2) >> 4);
            mma_bf16(tbase + b, dQk + qo, dK + ko, idS, ks > 0 ? 1u : 0u);
          }
        } else {
          mma_bf16_ss_k8_w<2ull, (uint64_t)(128 * 128 / 16), 2ull, (uint64_t)(64 * 128 / 16)>(tbase + b, dQk, dK, idS, 0u);
        }
        if (!(which & 32)) {
          if (single) {
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
              const uint64_t qo = (uint64_t)((((ks * 16) / 64) * 128 * 128 + ((ks * 16) % 64) * 2) >> 4);
              const uint64_t ko = (uint64_t)((((ks * 16) / 64) * 64 * 128 + ((ks * 16) % 64) * 2) >> 4);
              mma_bf16(tbase + 128u + b, dDOk + qo, dV + ko, idS, ks > 0 ? 1u : 0u);
            }
          } else {
            mma_bf16_ss_k8_w<2ull, (uint64_t)(128 * 128 / 16), 2ull, (uint64_t)(64 * 128 / 16)>(tbase + 128u + b, dDOk, dV,
                                                                                              idS, 0u);
          }
        }
      }
      if (w2 != 1 && !(which & 32)) {
        if (single) {
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) mma_bf16(tbase + 256u, dDOm + (uint64_t)(ks * 128), dPm + (uint64_t)(ks * 128), idT, 1u);
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) mma_bf16(tbase + 320u, dQm + (uint64_t)(ks * 128), dDSm + (uint64_t)(ks * 128), idT, 1u);
        } else {
          mma_bf16_ss_k8_w<128ull, 512ull, 128ull, 512ull>(tbase + 256u, dDOm, dPm, idT, 1u);
          mma_bf16_ss_k8_w<128ull, 512ull, 128ull, 512ull>(tbase + 320u, dQm, dDSm, idT, 1u);
        }
      }
    }
    if (!single) {
      mma_commit_w(&bar_mma);
    } else {
      mma_commit(&bar_mma);
    }
    mbar_wait(&bar_mma, 0);
    if (lane_id() == 0) cycles[blockIdx.x] = clock64() - t0;
    if (lane_id() == 0) stop_flag = 1;
  }
  tc_fence_before();
  __syncthreads();
  if ((which & 256) && threadIdx.x == 0)
    cycles[gridDim.x + blockIdx.x] = staged[1] + staged[2] + staged[3];  // bytes staged by warps 1-3
  if (warp_id() == 0) tmem_dealloc(tbase, 512);
}
}  // namespace
}  // namespace spa2

extern "C" int spa2_probe_dkdv_mix(int reps, int which, int ctas, unsigned long long* cycles, void* stream) {
  const size_t smem = 196608 + 1024;
  SPA2_CUDA_TRY(cudaFuncSetAttribute(spa2::k_dkdv_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  spa2::k_dkdv_mix<<<ctas, 128, smem, (cudaStream_t)stream>>>(reps, which, cycles);
  SPA2_LAUNCH_CHECK();
  return SPA2_OK;
}

// ---- tcgen05.cp rate probe (diagnostic): smem -> TMEM copies alone, SS MMAs alone, both ----
// One warp issues, per rep, 8 tcgen05.cp.128x256b (a 32 KB K-major SW128 tile into TMEM
// columns [256, 320)) and/or one 8-step SS MMA group (M=128, N=64, from other smem) into
// columns [0, 64).  mode: 1 = copies only, 2 = MMAs only, 3 = both.  cycles[cta] = span.
namespace spa2 {
namespace {
__global__ void __launch_bounds__(128) k_cp_rate(int reps, int mode, unsigned long long* cycles) {
  extern __shared__ uint8_t smem_dyn[];
  __shared__ uint64_t bar_mma;
  __shared__ uint32_t tmem_base;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 98304 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(base)[i] = make_uint4(0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u);
  if (warp_id() == 0) tmem_alloc(&tmem_base, 512);
  if (threadIdx.x == 32) {
    mbar_init(&bar_mma, 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (warp_id() == 0) {
    // [0, 32K) copy source (K-major SW128 128 x 128) | [32K, 64K) MMA A | [64K, 80K) MMA B
    const uint64_t dC = sw128_desc(smem_u32(base), 16, 1024);
    const uint64_t dA = sw128_desc(smem_u32(base + 32768), 16, 1024);
    const uint64_t dB = sw128_desc(smem_u32(base + 65536), 16, 1024);
    constexpr uint32_t idS = idesc_bf16(128, 64, false, false);
    const uint64_t t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (mode & 1) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const uint64_t qo = (uint64_t)((((ks * 16) / 64) * 128 * 128 + ((ks * 16) % 64) * 2) >> 4);
          tmem_cp_128x256b_w(tbase + 256u + (uint32_t)(ks * 8), dC + qo);
        }
      }
      if (mode & 2)
        mma_bf16_ss_k8_w<2ull, (uint64_t)(128 * 128 / 16), 2ull, (uint64_t)(64 * 128 / 16)>(
            tbase + (uint32_t)((r & 1) * 64), dA, dB, idS, 0u);
    }
    mma_commit_w(&bar_mma);
    mbar_wait(&bar_mma, 0);
    if (lane_id() == 0) cycles[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc(tbase, 512);
}
}  // namespace
}  // namespace spa2

extern "C" int spa2_probe_cp_rate(int reps, int mode, int ctas, unsigned long long* cycles, void* stream) {
  const size_t smem = 98304 + 1024;
  SPA2_CUDA_TRY(cudaFuncSetAttribute(spa2::k_cp_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  spa2::k_cp_rate<<<ctas, 128, smem, (cudaStream_t)stream>>>(reps, mode, cycles);
  SPA2_LAUNCH_CHECK();
  return SPA2_OK;
}
