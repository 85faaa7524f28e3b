// bwd.cu — K5 δ, K7 dQ (query-major) and K6 dK/dV (key-major) on tcgen05 (sm_100a).
//
// Replaces attention.attention_backward (attention.py:128-166).  The reference walks kept
// (i, j) pairs row-major and accumulates into dq/dk/dv; here every accumulator lives in
// TMEM of exactly one CTA, so the result is deterministic and needs no atomics:
//   K5  δ_i = rowsum(dO ∘ O)                                          (attention.py:149)
//   K7  work item = query block i, tiles = its row list j:
//         S = Q_i K_jᵀ, dP = dO_i V_jᵀ  ->  dS = P ∘ (dP − δ), P = exp2(S·c − LSE·log2e)
//         dQ_i += dS K_j                   (dS packed bf16 into TMEM = TS-MMA A operand)
//   K6  work item = key block j, tiles = its column list i:
//         same S, dP, P, dS (written bf16 into swizzled smem), then with the accumulators
//         kept TRANSPOSED so every MMA has M = 128:
//         dVᵀ += dO_iᵀ P    (M = d, N = 64, K = 128; both operands MN-major in smem)
//         dKᵀ += Q_iᵀ dS
// Both kernels are persistent (one CTA per SM walking a head-major, longest-first work
// list) and warp-specialised with 10 warps:
//   warp 0 TMA producer (runs ahead across work items), warp 1 tcgen05.mma issuer (issues
//   S/dP of tile g before the accumulate MMAs of tile g-1, also across items), warps 2-5
//   elementwise (one TMEM lane = one row per thread), warps 6-9 epilogue (TMEM -> smem ->
//   TMA store) overlapping the next item.  TMEM: S[2] | dP[2] | accumulator[2] = 512 cols.
// The query-block-major and key-block-major passes both recompute S and dP (7 MMAs per
// kept tile instead of 5) in exchange for zero global reductions.
// Key blocks no query keeps get exact zeros (attention.py:152-157: dropped blocks
// contribute nothing); so do query blocks with empty lists.
#include <math.h>

#include <algorithm>
#include <stdlib.h>

#include "common.cuh"
#include "ptx.cuh"
#include "tma_host.h"

namespace spa2 {
namespace {

// Share of the elementwise exponentials computed by exp2_poly2 on the FMA pipe instead of
// MUFU: CPT*NUM/64 of each thread's CPT/2 pairs (NUM = 8: a quarter).  Measured in the
// power-capped 400-step regime (tools/ab400.sh): dQ is fastest with none (MUFU exponentials
// cost less energy), dK/dV with a quarter.
#ifndef SPA2_DQ_POLY_NUM
#define SPA2_DQ_POLY_NUM 0
#endif
#ifndef SPA2_DKDV_POLY_NUM
#define SPA2_DKDV_POLY_NUM 8
#endif
#ifndef SPA2_DQ_NK
#define SPA2_DQ_NK 4
#endif
#ifndef SPA2_DQ_NV
#define SPA2_DQ_NV 4
#endif
using namespace ptx;

constexpr int BQ = 128;
constexpr int BKV = 64;
constexpr int kThreads = 320;  // 10 warps
constexpr int kEpiTid0 = 192;  // first epilogue thread (warp 6)
constexpr float kLog2e = 1.4426950408889634f;

struct BwdParams {
  int H, N, T_m, T_n;
  int num_items;
  const int32_t* ptr;    // row_ptr (dq) / col_ptr (dkdv)
  const int32_t* idx;    // row_idx / col_idx
  const int32_t* order;  // head-major, longest-first work order
  const float* lse;      // natural log, [B*H, N]
  const float* delta;    // [B*H, N]
  float scale;           // 1/sqrt(d)
  float sl2;             // scale * log2(e)
  __nv_bfloat16* out0;   // dq (K7) / dk (K6), for empty lists
  int64_t o0_sb, o0_sh, o0_sn;
  __nv_bfloat16* out1;   // dv (K6)
  int64_t o1_sb, o1_sh, o1_sn;
  unsigned long long* trace;  // diagnostic (spa2_debug_trace), normally null
  int trace_cap;
  // fused δ (k_dq3 with delta_out != null): δ = rowsum(dO ∘ O) computed in the kernel
  const __nv_bfloat16* o_in;
  int64_t oi_sb, oi_sh, oi_sn;
  const __nv_bfloat16* do_in;
  int64_t di_sb, di_sh, di_sn;
  float* delta_out;
};

struct Item {
  int bh, blk, beg, n;
};

__device__ __forceinline__ Item get_item(const BwdParams& p, int wi, int nblk) {
  const int w = p.order ? p.order[wi] : wi;
  Item m;
  m.bh = w / nblk;
  m.blk = w % nblk;
  m.beg = p.ptr[w];
  m.n = p.ptr[w + 1] - m.beg;
  return m;
}

// Work-list cursor shared by the roles of the persistent kernels: walks this CTA's items
// (blockIdx.x, +gridDim.x, ...) skipping empty ones, one tile at a time.
struct Cursor {
  int wi, it, t, n, beg, bh, blk, g;
  bool valid;
};
__device__ __forceinline__ void cursor_item(Cursor& c, const BwdParams& p, int nblk) {
  for (;;) {
    c.wi += gridDim.x;
    if (c.wi >= p.num_items) {
      c.valid = false;
      return;
    }
    const Item m = get_item(p, c.wi, nblk);
    if (m.n > 0) {
      c.n = m.n;
      c.beg = m.beg;
      c.bh = m.bh;
      c.blk = m.blk;
      c.t = 0;
      ++c.it;
      c.valid = true;
      return;
    }
  }
}
__device__ __forceinline__ void cursor_init(Cursor& c, const BwdParams& p, int nblk) {
  c.wi = (int)blockIdx.x - (int)gridDim.x;
  c.it = -1;
  c.g = 0;
  c.valid = false;
  cursor_item(c, p, nblk);
}
__device__ __forceinline__ void cursor_next(Cursor& c, const BwdParams& p, int nblk) {
  ++c.g;
  if (++c.t >= c.n) cursor_item(c, p, nblk);
}

// δ of one row computed by a single thread with exactly k_delta's arithmetic (HD/8 parts
// of 8 fused multiply-adds, then the xor-butterfly combination), so fused and separate δ
// are bit-identical.
template <int HD>
__device__ __forceinline__ float row_delta(const __nv_bfloat16* op, const __nv_bfloat16* dp) {
  constexpr int TPR = HD / 8;
  float part[TPR];
#pragma unroll
  for (int q = 0; q < TPR; q += 4) {
    uint4 a[4], c[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[u] = __ldg(reinterpret_cast<const uint4*>(op + (q + u) * 8));
      c[u] = __ldg(reinterpret_cast<const uint4*>(dp + (q + u) * 8));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a[u]);
      const __nv_bfloat162* c2 = reinterpret_cast<const __nv_bfloat162*>(&c[u]);
      float acc = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 x = __bfloat1622float2(a2[e]);
        const float2 y = __bfloat1622float2(c2[e]);
        acc = fmaf(x.x, y.x, acc);
        acc = fmaf(x.y, y.y, acc);
      }
      part[q + u] = acc;
    }
  }
#pragma unroll
  for (int off = TPR / 2; off > 0; off >>= 1)
#pragma unroll
    for (int i = 0; i < TPR; ++i)
      if ((i & off) == 0) part[i] = part[i] + part[i | off];
  return part[0];
}

// ---------------------------------------------------------------------------------------
// K5: δ = rowsum(dO ∘ O) in fp32.  HD/8 threads per row, 16-byte loads.
// ---------------------------------------------------------------------------------------
template <int HD>
__global__ void __launch_bounds__(256) k_delta(spa2_view o, spa2_view dout, float* __restrict__ delta, int H, int N,
                                               int64_t rows_total) {
  constexpr int TPR = HD / 8;
  constexpr int RPC = 256 / TPR;
  const int64_t row = (int64_t)blockIdx.x * RPC + threadIdx.x / TPR;
  const int part = threadIdx.x % TPR;
  float acc = 0.f;
  if (row < rows_total) {
    const int64_t bh = row / N, tok = row % N;
    const int64_t b = bh / H, h = bh % H;
    const __nv_bfloat16* op = reinterpret_cast<const __nv_bfloat16*>(o.ptr) + b * o.sb + h * o.sh + tok * o.sn + part * 8;
    const __nv_bfloat16* dp =
        reinterpret_cast<const __nv_bfloat16*>(dout.ptr) + b * dout.sb + h * dout.sh + tok * dout.sn + part * 8;
    const uint4 a = *reinterpret_cast<const uint4*>(op);
    const uint4 c = *reinterpret_cast<const uint4*>(dp);
    const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* c2 = reinterpret_cast<const __nv_bfloat162*>(&c);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 x = __bfloat1622float2(a2[e]);
      const float2 y = __bfloat1622float2(c2[e]);
      acc = fmaf(x.x, y.x, acc);
      acc = fmaf(x.y, y.y, acc);
    }
  }
#pragma unroll
  for (int off = TPR / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (part == 0 && row < rows_total) delta[row] = acc;
}

// ---------------------------------------------------------------------------------------
// K7: dQ.  Work item = query block; tiles = kept key blocks.
// ---------------------------------------------------------------------------------------
template <int HD>
struct DqCfg {
  static constexpr int NSK = 3, NSV = 2;
  static constexpr int Q_BYTES = BQ * HD * 2;
  static constexpr int KV_BYTES = BKV * HD * 2;
  static constexpr int OFF_QDO = 0;  // [2 item stages][Q | dO]
  static constexpr int OFF_K = 4 * Q_BYTES;
  static constexpr int OFF_V = OFF_K + NSK * KV_BYTES;
  static constexpr int OFF_BAR = OFF_V + NSV * KV_BYTES;
  static constexpr int NUM_BARS = 4 + 2 * NSK + 2 * NSV + 2 + 2 + 1 + 4;
  static constexpr int SMEM = OFF_BAR + NUM_BARS * 8 + 16 + kSmemAlignSlack;
  static constexpr uint32_t S_COL = 0, DP_COL = 128, ACC_COL = 256;
};

template <int HD>
__global__ void __launch_bounds__(kThreads, 1)
    k_dq(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
         const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
         const __grid_constant__ CUtensorMap tmDQ, const BwdParams p) {
  using C = DqCfg<HD>;
  constexpr int NSK = C::NSK, NSV = C::NSV;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* const smem = smem_align_1k(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* qdo_full = bars;            // [2]
  uint64_t* qdo_empty = qdo_full + 2;   // [2]
  uint64_t* k_full = qdo_empty + 2;     // [NSK]
  uint64_t* k_empty = k_full + NSK;     // [NSK]
  uint64_t* v_full = k_empty + NSK;     // [NSV]
  uint64_t* v_empty = v_full + NSV;     // [NSV]
  uint64_t* s_full = v_empty + NSV;     // [2] S and dP of tile g landed
  uint64_t* ds_full = s_full + 2;       // [2] dS of tile g packed into TMEM
  uint64_t* dq_done = ds_full + 2;      // one completion per dQ MMA group
  uint64_t* acc_full = dq_done + 1;     // [2]
  uint64_t* acc_empty = acc_full + 2;   // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = (int)warp_id(), lane = (int)lane_id();
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&qdo_full[s], 1);
      mbar_init(&qdo_empty[s], 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&ds_full[s], 128);
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], 128);
    }
    for (int s = 0; s < NSK; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < NSV; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    mbar_init(dq_done, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_holder;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (elect_one()) {
      tma_prefetch(&tmQ);
      tma_prefetch(&tmDO);
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
      int it = 0, g = 0;
      for (int wi = blockIdx.x; wi < p.num_items; wi += gridDim.x) {
        const Item m = get_item(p, wi, p.T_m);
        if (m.n == 0) continue;
        const int hh = m.bh % p.H, bb = m.bh / p.H;
        const int st = it & 1;
        if (it >= 2) mbar_wait(&qdo_empty[st], ((uint32_t)(it >> 1) + 1u) & 1u);
        mbar_expect_tx(&qdo_full[st], 2 * C::Q_BYTES);
        uint8_t* sq = smem + C::OFF_QDO + st * 2 * C::Q_BYTES;
        {
          tma_load_5d(sq, &tmQ, &qdo_full[st], 0, m.blk * BQ, 0, hh, bb);
          tma_load_5d(sq + C::Q_BYTES, &tmDO, &qdo_full[st], 0, m.blk * BQ, 0, hh, bb);
        }
        for (int t = 0; t < m.n; ++t, ++g) {
          const int j = p.idx[m.beg + t];
          const int sk = g % NSK, sv = g % NSV;
          trace_ev(p.trace, p.trace_cap, 0, 1, g);
          if (g >= NSK) mbar_wait(&k_empty[sk], ((uint32_t)(g / NSK) + 1u) & 1u);
          trace_ev(p.trace, p.trace_cap, 0, 2, g);
          mbar_expect_tx(&k_full[sk], C::KV_BYTES);
          tma_load_5d(smem + C::OFF_K + sk * C::KV_BYTES, &tmK, &k_full[sk], 0, j * BKV, 0, hh, bb);
          if (g >= NSV) mbar_wait(&v_empty[sv], ((uint32_t)(g / NSV) + 1u) & 1u);
          mbar_expect_tx(&v_full[sv], C::KV_BYTES);
          tma_load_5d(smem + C::OFF_V + sv * C::KV_BYTES, &tmV, &v_full[sv], 0, j * BKV, 0, hh, bb);
        }
        ++it;
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (elect_one()) {
      constexpr uint32_t idS = idesc_bf16(BQ, BKV, false, false);
      constexpr uint32_t idQ = idesc_bf16(BQ, HD, false, true);
      struct Pend {
        int g, it, sk;
        bool first, last, valid;
      } pd{0, 0, 0, false, false, false};
      auto issue_dq = [&](const Pend& q) {
        const uint32_t acc = tbase + C::ACC_COL + (uint32_t)((q.it & 1) * 128);
        if (q.first && q.it >= 2) mbar_wait(&acc_empty[q.it & 1], ((uint32_t)(q.it >> 1) + 1u) & 1u);
        trace_ev(p.trace, p.trace_cap, 1, 3, q.g);
        mbar_wait(&ds_full[q.g & 1], (uint32_t)(q.g >> 1) & 1u);
        trace_ev(p.trace, p.trace_cap, 1, 4, q.g);
        tc_fence_after();
        const uint32_t sK = smem_u32(smem + C::OFF_K + q.sk * C::KV_BYTES);
#pragma unroll
        for (int ks = 0; ks < BKV / 16; ++ks)
          mma_bf16_ts(acc, tbase + C::S_COL + (uint32_t)((q.g & 1) * 64 + ks * 8),
                      sw128_desc(sK + (uint32_t)(ks * 2048), BKV * 128, 1024), idQ, (!q.first || ks > 0) ? 1u : 0u);
        mma_commit(dq_done);
        mma_commit(&k_empty[q.sk]);
        if (q.last) mma_commit(&acc_full[q.it & 1]);
      };
      int it = 0, g = 0;
      for (int wi = blockIdx.x; wi < p.num_items; wi += gridDim.x) {
        const Item m = get_item(p, wi, p.T_m);
        if (m.n == 0) continue;
        const int st = it & 1;
        mbar_wait(&qdo_full[st], (uint32_t)(it >> 1) & 1u);
        tc_fence_after();
        const uint32_t sQ = smem_u32(smem + C::OFF_QDO + st * 2 * C::Q_BYTES);
        const uint32_t sDO = sQ + C::Q_BYTES;
        for (int t = 0; t < m.n; ++t, ++g) {
          const uint32_t b = (uint32_t)(g & 1);
          const int sk = g % NSK, sv = g % NSV;
          trace_ev(p.trace, p.trace_cap, 1, 1, g);
          if (g >= 2) mbar_wait(dq_done, (uint32_t)(g - 2) & 1u);  // dS_{g-2} lives in S[b]
          trace_ev(p.trace, p.trace_cap, 1, 5, g);
          mbar_wait(&k_full[sk], (uint32_t)(g / NSK) & 1u);
          trace_ev(p.trace, p.trace_cap, 1, 2, g);
          tc_fence_after();
          const uint32_t sK = smem_u32(smem + C::OFF_K + sk * C::KV_BYTES);
#pragma unroll
          for (int ks = 0; ks < HD / 16; ++ks) {
            const uint32_t qo = (uint32_t)((ks * 16 / 64) * BQ * 128 + (ks * 16 % 64) * 2);
            const uint32_t ko = (uint32_t)((ks * 16 / 64) * BKV * 128 + (ks * 16 % 64) * 2);
            mma_bf16(tbase + C::S_COL + b * 64, sw128_desc(sQ + qo, 16, 1024), sw128_desc(sK + ko, 16, 1024), idS,
                     ks > 0 ? 1u : 0u);
          }
          mbar_wait(&v_full[sv], (uint32_t)(g / NSV) & 1u);
          tc_fence_after();
          const uint32_t sV = smem_u32(smem + C::OFF_V + sv * C::KV_BYTES);
#pragma unroll
          for (int ks = 0; ks < HD / 16; ++ks) {
            const uint32_t qo = (uint32_t)((ks * 16 / 64) * BQ * 128 + (ks * 16 % 64) * 2);
            const uint32_t vo = (uint32_t)((ks * 16 / 64) * BKV * 128 + (ks * 16 % 64) * 2);
            mma_bf16(tbase + C::DP_COL + b * 64, sw128_desc(sDO + qo, 16, 1024), sw128_desc(sV + vo, 16, 1024), idS,
                     ks > 0 ? 1u : 0u);
          }
          mma_commit(&s_full[b]);
          mma_commit(&v_empty[sv]);
          if (pd.valid) issue_dq(pd);
          pd = Pend{g, it, sk, t == 0, t == m.n - 1, true};
        }
        ++it;
      }
      if (pd.valid) issue_dq(pd);
    }
    __syncwarp();
  } else if (warp < 6) {
    // ---------------- dS warps (2..5) ----------------
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const int kv_tail = p.N - (p.T_n - 1) * BKV;
    const float sl2 = p.sl2;
    int g = 0;
    for (int wi = blockIdx.x; wi < p.num_items; wi += gridDim.x) {
      const Item m = get_item(p, wi, p.T_m);
      if (m.n == 0) continue;
      const int tok = m.blk * BQ + row;
      const bool valid = tok < p.N;
      const float lse2 = valid ? p.lse[(int64_t)m.bh * p.N + tok] * kLog2e : INFINITY;
      const float dlt = valid ? p.delta[(int64_t)m.bh * p.N + tok] : 0.f;
      for (int t = 0; t < m.n; ++t, ++g) {
        const uint32_t b = (uint32_t)(g & 1);
        const bool tail = p.idx[m.beg + t] == p.T_n - 1 && kv_tail < BKV;
        const bool tr = threadIdx.x == 64;
        if (tr) trace_ev(p.trace, p.trace_cap, 2, 1, g);
        mbar_wait(&s_full[b], (uint32_t)(g >> 1) & 1u);
        if (tr) trace_ev(p.trace, p.trace_cap, 2, 2, g);
        tc_fence_after();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t sr[32], dr[32];
          tmem_ld32(tbase + lane_off + C::S_COL + b * 64 + (uint32_t)(32 * h), sr);
          tmem_ld32(tbase + lane_off + C::DP_COL + b * 64 + (uint32_t)(32 * h), dr);
          uint32_t pk[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            float p0 = ex2(fmaf(__uint_as_float(sr[2 * c]), sl2, -lse2));
            float p1 = ex2(fmaf(__uint_as_float(sr[2 * c + 1]), sl2, -lse2));
            if (tail) {
              if (32 * h + 2 * c >= kv_tail) p0 = 0.f;
              if (32 * h + 2 * c + 1 >= kv_tail) p1 = 0.f;
            }
            pk[c] = pack_bf16(p0 * (__uint_as_float(dr[2 * c]) - dlt), p1 * (__uint_as_float(dr[2 * c + 1]) - dlt));
          }
          tmem_st16(tbase + lane_off + C::S_COL + b * 64 + (uint32_t)(16 * h), pk);
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&ds_full[b]);
        if (tr) trace_ev(p.trace, p.trace_cap, 2, 4, g);
      }
    }
  } else {
    // ---------------- epilogue warps (6..9) ----------------
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    int it = 0;
    for (int wi = blockIdx.x; wi < p.num_items; wi += gridDim.x) {
      const Item m = get_item(p, wi, p.T_m);
      const int hh = m.bh % p.H, bb = m.bh / p.H;
      if (m.n == 0) {
        const int tok = m.blk * BQ + row;
        if (tok < p.N) {
          __nv_bfloat16* o = p.out0 + bb * p.o0_sb + hh * p.o0_sh + (int64_t)tok * p.o0_sn;
          for (int c = 0; c < HD; ++c) o[c] = __float2bfloat16(0.f);
        }
        continue;
      }
      const int st = it & 1;
      mbar_wait(&acc_full[st], (uint32_t)(it >> 1) & 1u);
      tc_fence_after();
      uint8_t* sOut = smem + C::OFF_QDO + st * 2 * C::Q_BYTES;  // Q of this item is dead
      fence_proxy_async_smem();
#pragma unroll 1
      for (int c0 = 0; c0 < HD; c0 += 32) {
        uint32_t o[32];
        tmem_ld32(tbase + lane_off + C::ACC_COL + (uint32_t)(st * 128 + c0), o);
        uint32_t pk[16];
#pragma unroll
        for (int c = 0; c < 16; ++c)
          pk[c] = pack_bf16(__uint_as_float(o[2 * c]) * p.scale, __uint_as_float(o[2 * c + 1]) * p.scale);
        const uint32_t base = smem_u32(sOut + (c0 / 64) * BQ * 128);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          st_shared_v4(base + sw128_offset((uint32_t)row, (uint32_t)((c0 % 64) / 8 + u)), pk[4 * u], pk[4 * u + 1],
                       pk[4 * u + 2], pk[4 * u + 3]);
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[st]);
      fence_proxy_async_smem();
      named_bar_sync(1, 128);
      if (threadIdx.x == kEpiTid0) {
        tma_store_5d(&tmDQ, sOut, 0, m.blk * BQ, 0, hh, bb);
        tma_store_commit();
        tma_store_wait_read();
        mbar_arrive(&qdo_empty[st]);
      }
      ++it;
    }
    if (threadIdx.x == kEpiTid0) tma_store_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tbase, 512);
}

// ---------------------------------------------------------------------------------------
// K6: dK and dV.  Work item = key block; tiles = query blocks keeping it.  Accumulators
// transposed (TMEM lanes = head dim).
// ---------------------------------------------------------------------------------------
// ---------------------------------------------------------------------------------------
// K7 variant: dQ with one query block per CTA and TWO CTAs per SM (TMEM 256 columns and
// <= 112 KB smem each).  The per-CTA pipeline is simple (S/dP single-buffered, the tensor
// pipe idles while this CTA's warps compute dS) and the second CTA on the SM fills those
// gaps — the same structure as the forward kernel.
// ---------------------------------------------------------------------------------------
constexpr int kDq2Threads = 224;  // warp 6: second TMA producer (dO, V)

template <int HD>
struct Dq2Cfg {
  static constexpr int NSK = 2;
  static constexpr int Q_BYTES = BQ * HD * 2;
  static constexpr int KV_BYTES = BKV * HD * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_DO = Q_BYTES;
  static constexpr int OFF_K = 2 * Q_BYTES;
  static constexpr int OFF_V = OFF_K + NSK * KV_BYTES;
  static constexpr int OFF_BAR = OFF_V + KV_BYTES;
  static constexpr int NUM_BARS = 1 + 2 * NSK + 2 + 4;
  static constexpr int SMEM_USED = OFF_BAR + NUM_BARS * 8 + 16;
  static constexpr int SMEM = SMEM_USED + kSmemAlignSlack < 80 * 1024 ? 80 * 1024 : SMEM_USED + kSmemAlignSlack;  // never 3 CTAs/SM (TMEM)
  static constexpr uint32_t S_COL = 0, DP_COL = 64, ACC_COL = 128;
};

template <int HD>
__global__ void __launch_bounds__(kDq2Threads, 2)
    k_dq2(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
          const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
          const __grid_constant__ CUtensorMap tmDQ, const BwdParams p) {
  using C = Dq2Cfg<HD>;
  constexpr int NSK = C::NSK;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* const smem = smem_align_1k(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* qdo_full = bars;
  uint64_t* k_full = qdo_full + 1;   // [NSK]
  uint64_t* k_empty = k_full + NSK;  // [NSK]
  uint64_t* v_full = k_empty + NSK;
  uint64_t* v_empty = v_full + 1;
  uint64_t* s_full = v_empty + 1;    // S and dP of tile t landed
  uint64_t* ds_full = s_full + 1;    // dS of tile t packed into TMEM
  uint64_t* dq_done = ds_full + 1;   // dQ MMA of tile t done
  uint64_t* acc_full = dq_done + 1;  // last dQ MMA done
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(acc_full + 1);

  const int warp = (int)warp_id(), lane = (int)lane_id();
  const int w = p.order ? p.order[blockIdx.x] : (int)blockIdx.x;
  const int bh = w / p.T_m, qi = w % p.T_m;
  const int hh = bh % p.H, bb = bh / p.H;
  const int beg = p.ptr[w];
  const int n = p.ptr[w + 1] - beg;
  const int32_t* list = p.idx + beg;

  if (threadIdx.x == 0) {
    mbar_init(qdo_full, 2);  // Q from warp 0, dO from warp 6
    for (int s = 0; s < NSK; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    mbar_init(v_full, 1);
    mbar_init(v_empty, 1);
    mbar_init(s_full, 1);
    mbar_init(ds_full, 128);
    mbar_init(dq_done, 1);
    mbar_init(acc_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_holder, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_holder;

  if (n == 0) {
    if (warp >= 2 && warp < 6) {
      const int tok = qi * BQ + (warp & 3) * 32 + lane;
      if (tok < p.N) {
        __nv_bfloat16* o = p.out0 + bb * p.o0_sb + hh * p.o0_sh + (int64_t)tok * p.o0_sn;
        for (int c = 0; c < HD; ++c) o[c] = __float2bfloat16(0.f);
      }
    }
  } else if (warp == 0) {
    if (elect_one()) {
      tma_prefetch(&tmQ);
      tma_prefetch(&tmDO);
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
      mbar_expect_tx(qdo_full, C::Q_BYTES);
      tma_load_5d(smem + C::OFF_Q, &tmQ, qdo_full, 0, qi * BQ, 0, hh, bb);
      for (int t = 0; t < n; ++t) {
        const int j = list[t];
        const int sk = t % NSK;
        if (t >= NSK) mbar_wait(&k_empty[sk], ((uint32_t)(t / NSK) + 1u) & 1u);
        mbar_expect_tx(&k_full[sk], C::KV_BYTES);
        tma_load_5d(smem + C::OFF_K + sk * C::KV_BYTES, &tmK, &k_full[sk], 0, j * BKV, 0, hh, bb);
      }
    }
  } else if (warp == 6) {
    // second producer: dO, then V (TMA requests issued by one warp are served one at a
    // time; two issuing warps double the fill rate, tools/tma_rate.py)
    if (elect_one()) {
      mbar_expect_tx(qdo_full, C::Q_BYTES);
      tma_load_5d(smem + C::OFF_DO, &tmDO, qdo_full, 0, qi * BQ, 0, hh, bb);
      for (int t = 0; t < n; ++t) {
        if (t >= 1) mbar_wait(v_empty, (uint32_t)(t - 1) & 1u);
        mbar_expect_tx(v_full, C::KV_BYTES);
        tma_load_5d(smem + C::OFF_V, &tmV, v_full, 0, list[t] * BKV, 0, hh, bb);
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idS = idesc_bf16(BQ, BKV, false, false);
      constexpr uint32_t idQ = idesc_bf16(BQ, HD, false, true);
      const uint32_t sQ = smem_u32(smem + C::OFF_Q), sDO = smem_u32(smem + C::OFF_DO);
      const uint32_t sV = smem_u32(smem + C::OFF_V);
      mbar_wait(qdo_full, 0);
      for (int t = 0; t < n; ++t) {
        const int sk = t % NSK;
        if (t >= 1) mbar_wait(dq_done, (uint32_t)(t - 1) & 1u);  // dS_{t-1} (in S) consumed
        mbar_wait(&k_full[sk], (uint32_t)(t / NSK) & 1u);
        tc_fence_after();
        const uint32_t sK = smem_u32(smem + C::OFF_K + sk * C::KV_BYTES);
#pragma unroll
        for (int ks = 0; ks < HD / 16; ++ks) {
          const uint32_t qo = (uint32_t)((ks * 16 / 64) * BQ * 128 + (ks * 16 % 64) * 2);
          const uint32_t ko = (uint32_t)((ks * 16 / 64) * BKV * 128 + (ks * 16 % 64) * 2);
          mma_bf16(tbase + C::S_COL, sw128_desc(sQ + qo, 16, 1024), sw128_desc(sK + ko, 16, 1024), idS,
                   ks > 0 ? 1u : 0u);
        }
        mbar_wait(v_full, (uint32_t)t & 1u);
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < HD / 16; ++ks) {
          const uint32_t qo = (uint32_t)((ks * 16 / 64) * BQ * 128 + (ks * 16 % 64) * 2);
          const uint32_t vo = (uint32_t)((ks * 16 / 64) * BKV * 128 + (ks * 16 % 64) * 2);
          mma_bf16(tbase + C::DP_COL, sw128_desc(sDO + qo, 16, 1024), sw128_desc(sV + vo, 16, 1024), idS,
                   ks > 0 ? 1u : 0u);
        }
        mma_commit(s_full);
        mma_commit(v_empty);
        mbar_wait(ds_full, (uint32_t)t & 1u);
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < BKV / 16; ++ks)
          mma_bf16_ts(tbase + C::ACC_COL, tbase + C::S_COL + (uint32_t)(ks * 8),
                      sw128_desc(sK + (uint32_t)(ks * 2048), BKV * 128, 1024), idQ, (t > 0 || ks > 0) ? 1u : 0u);
        mma_commit(dq_done);
        mma_commit(&k_empty[sk]);
      }
      mma_commit(acc_full);
    }
    __syncwarp();
  } else if (warp < 6) {
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const int tok = qi * BQ + row;
    const bool valid = tok < p.N;
    const float lse2 = valid ? p.lse[(int64_t)bh * p.N + tok] * kLog2e : INFINITY;
    const float dlt = valid ? p.delta[(int64_t)bh * p.N + tok] : 0.f;
    const int kv_tail = p.N - (p.T_n - 1) * BKV;
    const float sl2 = p.sl2;
    for (int t = 0; t < n; ++t) {
      const bool tail = list[t] == p.T_n - 1 && kv_tail < BKV;
      mbar_wait(s_full, (uint32_t)t & 1u);
      tc_fence_after();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t sr[32], dr[32];
        tmem_ld32(tbase + lane_off + C::S_COL + (uint32_t)(32 * h), sr);
        tmem_ld32(tbase + lane_off + C::DP_COL + (uint32_t)(32 * h), dr);
        uint32_t pk[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          float p0 = ex2(fmaf(__uint_as_float(sr[2 * c]), sl2, -lse2));
          float p1 = ex2(fmaf(__uint_as_float(sr[2 * c + 1]), sl2, -lse2));
          if (tail) {
            if (32 * h + 2 * c >= kv_tail) p0 = 0.f;
            if (32 * h + 2 * c + 1 >= kv_tail) p1 = 0.f;
          }
          pk[c] = pack_bf16(p0 * (__uint_as_float(dr[2 * c]) - dlt), p1 * (__uint_as_float(dr[2 * c + 1]) - dlt));
        }
        tmem_st16(tbase + lane_off + C::S_COL + (uint32_t)(16 * h), pk);
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(ds_full);
    }
    mbar_wait(acc_full, 0);
    tc_fence_after();
    uint8_t* sOut = smem + C::OFF_Q;  // every MMA has completed: Q is dead
#pragma unroll 1
    for (int c0 = 0; c0 < HD; c0 += 32) {
      uint32_t o[32];
      tmem_ld32(tbase + lane_off + C::ACC_COL + (uint32_t)c0, o);
      uint32_t pk[16];
#pragma unroll
      for (int c = 0; c < 16; ++c)
        pk[c] = pack_bf16(__uint_as_float(o[2 * c]) * p.scale, __uint_as_float(o[2 * c + 1]) * p.scale);
      const uint32_t base = smem_u32(sOut + (c0 / 64) * BQ * 128);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        st_shared_v4(base + sw128_offset((uint32_t)row, (uint32_t)((c0 % 64) / 8 + u)), pk[4 * u], pk[4 * u + 1],
                     pk[4 * u + 2], pk[4 * u + 3]);
    }
    fence_proxy_async_smem();
    named_bar_sync(1, 128);
    if (threadIdx.x == 64) {
      tma_store_5d(&tmDQ, sOut, 0, qi * BQ, 0, hh, bb);
      tma_store_commit();
      tma_store_wait_all();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tbase, 256);
}

// ---------------------------------------------------------------------------------------
// K7 (default): dQ, persistent (one CTA per SM), with Q_i and dO_i RESIDENT IN TMEM.
// Work item = query block i; tiles = its kept key blocks j.  Q_i and dO_i are staged once
// per item by TMA and copied into TMEM with tcgen05.cp, so S = Q K_jᵀ and dP = dO V_jᵀ are
// TS-MMAs that read only K_j / V_j from shared memory (2 KB per K=16 step instead of 6 KB:
// the SS form is smem-bandwidth bound at 48 cycles per step, profiles/mma_rate_r01.md).
// TMEM (512 columns): Q [0,64) | dO [64,128) | S/dP double buffer [128,384) | dQ acc [384,512).
// dS (bf16) overwrites the S columns its thread group read and feeds dQ += dS K_j (TS).
// Warps: 0 TMA (Q, K ring), 1 MMA, 2-9 elementwise (2 per TMEM lane quarter, 32 columns
// each), 10-13 epilogue (acc -> bf16 -> global), 14 TMA (dO, V ring).
// ---------------------------------------------------------------------------------------
// Warp roles of k_dq3 for EWW elementwise warps (EWW/4 per TMEM lane quarter).
template <int EWW>
struct Dq3Roles {
  static constexpr int EPI0 = 2 + EWW, PROD2 = EPI0 + 4, ISSUE_DP = PROD2 + 1, ISSUE_DQ = PROD2 + 2;
  static constexpr int THREADS = 32 * (ISSUE_DQ + 1);
  static constexpr int CPT = 256 / EWW;  // S/dP columns per elementwise thread
};

template <int HD>
struct Dq3Cfg {
  static constexpr int NK = SPA2_DQ_NK, NV = SPA2_DQ_NV;  // K / V ring depths
  static constexpr int Q_BYTES = BQ * HD * 2;
  static constexpr int KV_BYTES = BKV * HD * 2;
  static constexpr int OFF_QS = 0;  // staging [Q | dO] of the next item
  static constexpr int OFF_K = 2 * Q_BYTES;
  static constexpr int OFF_V = OFF_K + NK * KV_BYTES;
  static constexpr int OFF_DLT = OFF_V + NV * KV_BYTES;  // fused δ: float [2 items][128 rows]
  static constexpr int OFF_BAR = OFF_DLT + 2 * BQ * 4;
  static constexpr int NUM_BARS = 4 + 2 * NK + 2 * NV + 2 * 5 + 2 + 2;
  static constexpr int SMEM = OFF_BAR + NUM_BARS * 8 + 16 + kSmemAlignSlack;
  static constexpr uint32_t Q_COL = 0, DO_COL = 64, SDP_COL = 128, ACC_COL = 384;  // S at +b*128, dP at +64
};

// TMEM column of the packed bf16 dS for K step ks: thread group g read S columns
// [CPT·g, CPT·(g+1)) and packs its dS into the first CPT/2 of them.
template <int CPT>
__device__ __forceinline__ uint32_t ds_col(int ks) {
  return (uint32_t)((16 * ks / CPT) * CPT + (16 * ks % CPT) / 2);
}

template <int HD, int EWW>
__global__ void __launch_bounds__(Dq3Roles<EWW>::THREADS, 1)
    k_dq3(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
          const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO, const BwdParams p) {
  using C = Dq3Cfg<HD>;
  using R = Dq3Roles<EWW>;
  constexpr int NK = C::NK, NV = C::NV;
  constexpr int CPT = R::CPT;
  constexpr int kPolyPairs = CPT * SPA2_DQ_POLY_NUM / 64;  // of CPT/2 pairs
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* const smem = smem_align_1k(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* qs_full = bars;         // staging holds Q_i and dO_i of item `it`
  uint64_t* qs_free = bars + 1;     // tcgen05.cp of item `it` done: staging reusable
  uint64_t* qd_free = bars + 2;     // last S/dP MMA of item `it` done: TMEM Q/dO reusable
  uint64_t* qd_ready = bars + 3;    // Q/dO of item `it` copied into TMEM
  uint64_t* k_full = bars + 4;      // [NK]
  uint64_t* k_empty = k_full + NK;  // [NK]
  uint64_t* v_full = k_empty + NK;  // [NV]
  uint64_t* v_empty = v_full + NV;  // [NV]
  uint64_t* s_full = v_empty + NV;  // [2]
  uint64_t* dp_full = s_full + 2;   // [2]
  uint64_t* ds_full = dp_full + 2;  // [2] dS of tile g packed into TMEM buffer g&1
  uint64_t* dq_done = ds_full + 2;  // [2] dQ MMA of tile g done (buffer and K slot free)
  uint64_t* acc_full = dq_done + 2;
  uint64_t* acc_empty = acc_full + 1;
  uint64_t* dlt_full = acc_empty + 1;  // [2] fused δ of item `it` in sdelta[it & 1]
  uint64_t* s_free = dlt_full + 2;     // [2] S of tile g read out of TMEM buffer g&1
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(s_free + 2);
  float* sdelta = reinterpret_cast<float*>(smem + C::OFF_DLT);
  const bool fused_delta = p.delta_out != nullptr;

  const int warp = (int)warp_id(), lane = (int)lane_id();
  if (threadIdx.x == 0) {
    mbar_init(qs_full, 2);  // Q from warp 0, dO from warp 14
    mbar_init(qs_free, 1);
    mbar_init(qd_free, 2);  // last S (warp 1) and last dP (warp 15) of the item
    mbar_init(qd_ready, 1);
    for (int s = 0; s < NK; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < NV; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&dp_full[b], 1);
      mbar_init(&ds_full[b], 32 * EWW);
      mbar_init(&s_free[b], 32 * EWW);
      mbar_init(&dq_done[b], 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 128);
    mbar_init(&dlt_full[0], 128);
    mbar_init(&dlt_full[1], 128);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_holder;
  pdl_wait();  // everything above touched only this CTA's smem/TMEM
  pdl_trigger();

  if (warp == 0 || warp == R::PROD2) {
    // ---------------- TMA producers: warp 0 Q + K ring, warp 14 dO + V ring ----------------
    if (elect_one()) {
      const bool second = warp == R::PROD2;
      const CUtensorMap* tmR = second ? &tmDO : &tmQ;
      const CUtensorMap* tmKV = second ? &tmV : &tmK;
      tma_prefetch(tmR);
      tma_prefetch(tmKV);
      uint64_t* full = second ? v_full : k_full;
      uint64_t* empty = second ? v_empty : k_empty;
      const int ns = second ? NV : NK;
      uint8_t* const ring = smem + (second ? C::OFF_V : C::OFF_K);
      int it = 0, g = 0;
      for (int wi = blockIdx.x; wi < p.num_items; wi += gridDim.x) {
        const Item m = get_item(p, wi, p.T_m);
        if (m.n == 0) continue;
        const int hh = m.bh % p.H, bb = m.bh / p.H;
        if (it >= 1) mbar_wait(qs_free, (uint32_t)(it - 1) & 1u);
        mbar_expect_tx(qs_full, C::Q_BYTES);
        tma_load_5d(smem + C::OFF_QS + (second ? C::Q_BYTES : 0), tmR, qs_full, 0, m.blk * BQ, 0, hh, bb);
        for (int t = 0; t < m.n; ++t, ++g) {
          const int s = g % ns;
          if (!second) trace_ev(p.trace, p.trace_cap, 0, 1, g);
          if (g >= ns) mbar_wait(&empty[s], ((uint32_t)(g / ns) + 1u) & 1u);
          if (!second) trace_ev(p.trace, p.trace_cap, 0, 2, g);
          mbar_expect_tx(&full[s], C::KV_BYTES);
          tma_load_5d(ring + s * C::KV_BYTES, tmKV, &full[s], 0, p.idx[m.beg + t] * BKV, 0, hh, bb);
        }
        ++it;
      }
    }
  } else if (warp == 1 || warp == R::ISSUE_DP || warp == R::ISSUE_DQ) {
    // ---------------- MMA issue: three warps, one per independent stream ----------------
    // warp 1: (Q/dO copy into TMEM per item) + S = Q K_jᵀ;  warp 15: dP = dO V_jᵀ;
    // warp 16: dQ += dS K_j.  One issuing warp cannot feed N=64 MMAs (32 cycles each) fast
    // enough; the streams only meet through mbarriers.  Each warp issues warp-collectively.
    constexpr uint32_t idS = idesc_bf16(BQ, BKV, false, false);
    constexpr uint32_t idQ = idesc_bf16(BQ, HD, false, true);
    const uint64_t dQS = sw128_desc(smem_u32(smem + C::OFF_QS), 16, 1024);
    const uint64_t dK0 = sw128_desc(smem_u32(smem + C::OFF_K), 16, 1024);
    const uint64_t dV0 = sw128_desc(smem_u32(smem + C::OFF_V), 16, 1024);
    const uint64_t dKm0 = sw128_desc(smem_u32(smem + C::OFF_K), BKV * 128, 1024);
    constexpr uint64_t KV16 = (uint64_t)(C::KV_BYTES >> 4);
    Cursor c;
    cursor_init(c, p, p.T_m);
    if (warp == 1) {
      for (; c.valid; cursor_next(c, p, p.T_m)) {
        if (c.t == 0) {
          mbar_wait(qs_full, (uint32_t)c.it & 1u);
          if (c.it >= 1) mbar_wait(qd_free, (uint32_t)(c.it - 1) & 1u);
          tc_fence_after();
#pragma unroll
          for (int ks = 0; ks < HD / 16; ++ks) {
            const uint64_t qo = (uint64_t)(((ks * 16 / 64) * BQ * 128 + (ks * 16 % 64) * 2) >> 4);
            tmem_cp_128x256b_w(tbase + C::Q_COL + (uint32_t)(ks * 8), dQS + qo);
            tmem_cp_128x256b_w(tbase + C::DO_COL + (uint32_t)(ks * 8), dQS + (uint64_t)(C::Q_BYTES >> 4) + qo);
          }
          mma_commit_w(qs_free);
          mma_commit_w(qd_ready);
        }
        const int b = c.g & 1, sk = c.g % NK;
        // S columns of buffer b are free once the elementwise warps have read S of tile g-2
        // (dS goes into the dP columns, so S never waits for the dQ MMA)
        if (c.g >= 2) mbar_wait(&s_free[b], (uint32_t)((c.g - 2) >> 1) & 1u);
        mbar_wait(&k_full[sk], (uint32_t)(c.g / NK) & 1u);
        tc_fence_after();
        trace_ev(p.trace, p.trace_cap, 1, 2, c.g);
        const uint64_t dK = dK0 + (uint64_t)sk * KV16;
        const uint32_t sb = tbase + C::SDP_COL + (uint32_t)(b * 128);
#ifdef SPA2_MMA_BATCH
        if constexpr (HD == 128) {
          mma_bf16_ts_k8_w<8u, 2ull, (uint64_t)(BKV * 128 / 16)>(sb, tbase + C::Q_COL, dK, idS, 0u);
        } else
#endif
        {
#pragma unroll
          for (int ks = 0; ks < HD / 16; ++ks)
            mma_bf16_ts_w(sb, tbase + C::Q_COL + (uint32_t)(ks * 8),
                          dK + (uint64_t)((((ks * 16 / 64) * BKV * 128 + (ks * 16 % 64) * 2)) >> 4), idS, ks > 0 ? 1u : 0u);
        }
        mma_commit_w(&s_full[b]);
        if (c.t == c.n - 1) mma_commit_w(qd_free);
        trace_ev(p.trace, p.trace_cap, 1, 3, c.g);
      }
    } else {
      // dP = dO V_jᵀ (TS) and dQ += dS K_j (TS), by two warps (dP(g) waits for dQ(g-2) to
      // COMPLETE: it overwrites the TMEM columns dQ(g-2) reads dS from).  With
      // -DSPA2_DQ_MERGED one warp issues both as dQ(g-2), dP(g), ...: tcgen05 MMAs issued by
      // one thread execute in issue order, so the completion wait disappears.
      auto issue_dp = [&](const Cursor& cc) {
        if (cc.t == 0) mbar_wait(qd_ready, (uint32_t)cc.it & 1u);
        const int b = cc.g & 1, sv = cc.g % NV;
#ifndef SPA2_DQ_MERGED
        if (cc.g >= 2) mbar_wait(&dq_done[b], (uint32_t)((cc.g - 2) >> 1) & 1u);
#endif
        mbar_wait(&v_full[sv], (uint32_t)(cc.g / NV) & 1u);
        tc_fence_after();
        const uint64_t dV = dV0 + (uint64_t)sv * KV16;
        const uint32_t sb = tbase + C::SDP_COL + (uint32_t)(b * 128) + 64u;
#ifdef SPA2_MMA_BATCH
        if constexpr (HD == 128) {
          mma_bf16_ts_k8_w<8u, 2ull, (uint64_t)(BKV * 128 / 16)>(sb, tbase + C::DO_COL, dV, idS, 0u);
        } else
#endif
        {
#pragma unroll
          for (int ks = 0; ks < HD / 16; ++ks)
            mma_bf16_ts_w(sb, tbase + C::DO_COL + (uint32_t)(ks * 8),
                          dV + (uint64_t)((((ks * 16 / 64) * BKV * 128 + (ks * 16 % 64) * 2)) >> 4), idS, ks > 0 ? 1u : 0u);
        }
        mma_commit_w(&dp_full[b]);
        mma_commit_w(&v_empty[sv]);
        if (cc.t == cc.n - 1) mma_commit_w(qd_free);
      };
      auto issue_dq = [&](const Cursor& cc) {
        const int b = cc.g & 1, sk = cc.g % NK;
        if (cc.t == 0 && cc.it >= 1) mbar_wait(acc_empty, (uint32_t)(cc.it - 1) & 1u);
        mbar_wait(&ds_full[b], (uint32_t)(cc.g >> 1) & 1u);
        tc_fence_after();
        trace_ev(p.trace, p.trace_cap, 1, 4, cc.g);
        const uint64_t dKm = dKm0 + (uint64_t)sk * KV16;
        const uint32_t sb = tbase + C::SDP_COL + (uint32_t)(b * 128);
#ifdef SPA2_MMA_BATCH
        if constexpr (CPT == 16) {
          mma_bf16_ts_k4_w<16u, 128ull>(tbase + C::ACC_COL, sb + 64u, dKm, idQ, cc.t > 0 ? 1u : 0u);
        } else
#endif
        {
#pragma unroll
          for (int ks = 0; ks < BKV / 16; ++ks)
            mma_bf16_ts_w(tbase + C::ACC_COL, sb + 64u + ds_col<CPT>(ks), dKm + (uint64_t)((ks * 2048) >> 4), idQ,
                          (cc.t > 0 || ks > 0) ? 1u : 0u);
        }
#ifndef SPA2_DQ_MERGED
        mma_commit_w(&dq_done[b]);
#endif
        mma_commit_w(&k_empty[sk]);
        if (cc.t == cc.n - 1) mma_commit_w(acc_full);
        trace_ev(p.trace, p.trace_cap, 1, 5, cc.g);
      };
#ifdef SPA2_DQ_MERGED
      if (warp == R::ISSUE_DP) {
        // order dQ(g-2), dP(g): dP(g) reuses the TMEM buffer of tile g-2, and dQ(g-2) (its dS
        // reader) is issued just before it by this thread
        Cursor q0 = c, q1 = c;  // pending dQ tiles g-2, g-1
        int pending = 0;
        for (; c.valid; cursor_next(c, p, p.T_m)) {
          if (pending == 2) {
            issue_dq(q0);
            q0 = q1;
            pending = 1;
          }
          issue_dp(c);
          if (pending == 0) q0 = c;
          else q1 = c;
          ++pending;
        }
        if (pending >= 1) issue_dq(q0);
        if (pending == 2) issue_dq(q1);
      }
#else
      if (warp == R::ISSUE_DP) {
        for (; c.valid; cursor_next(c, p, p.T_m)) issue_dp(c);
      } else {
        for (; c.valid; cursor_next(c, p, p.T_m)) issue_dq(c);
      }
#endif
    }
  } else if (warp < R::EPI0) {
    // ---------------- elementwise: dS = P ∘ (dP − δ), P = exp2(S·c − LSE·log2e) ----------------
    const int q4 = warp & 3;
    const int grp = (warp - 2) >> 2;
    const int row = q4 * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const int col0 = CPT * grp;
    const int kv_tail = p.N - (p.T_n - 1) * BKV;
    const float sl2 = p.sl2;
    int g = 0, it = 0;
    for (int wi = blockIdx.x; wi < p.num_items; wi += gridDim.x) {
      const Item m = get_item(p, wi, p.T_m);
      if (m.n == 0) continue;
      const int tok = m.blk * BQ + row;
      const bool valid = tok < p.N;
      const float lse2 = valid ? __ldg(p.lse + (int64_t)m.bh * p.N + tok) * kLog2e : INFINITY;
      float dlt;
      if (fused_delta) {  // computed one item ahead by the epilogue warps
        mbar_wait(&dlt_full[it & 1], (uint32_t)(it >> 1) & 1u);
        dlt = valid ? sdelta[(it & 1) * BQ + row] : 0.f;
      } else {
        dlt = valid ? __ldg(p.delta + (int64_t)m.bh * p.N + tok) : 0.f;
      }
      ++it;
      // key-block index of the next tile is loaded one tile ahead (off the critical path)
      int j_next = __ldg(p.idx + m.beg);
      for (int t = 0; t < m.n; ++t, ++g) {
        const int b = g & 1;
        const bool tail = kv_tail < BKV && j_next == p.T_n - 1;
        if (t + 1 < m.n) j_next = __ldg(p.idx + m.beg + t + 1);
        const uint32_t sb = tbase + lane_off + C::SDP_COL + (uint32_t)(b * 128);
        if (threadIdx.x == 64) trace_ev(p.trace, p.trace_cap, 2, 1, g);
        mbar_wait(&s_full[b], (uint32_t)(g >> 1) & 1u);
        if (threadIdx.x == 64) trace_ev(p.trace, p.trace_cap, 2, 2, g);
        tc_fence_after();
        uint32_t sr[CPT];
        if constexpr (CPT == 32) tmem_ld32(sb + (uint32_t)col0, sr);
        else tmem_ld16(sb + (uint32_t)col0, sr);
        tc_fence_before();
        mbar_arrive(&s_free[b]);  // S(g) is in registers: the S issuer may overwrite it
        // packed fp32x2 math (FFMA2/FADD2/FMUL2): the issue slots of this SM sub-partition are
        // shared with an MMA-issuing warp, so fewer instructions per element = faster MMAs
        float pv[CPT];
#pragma unroll
        for (int c = 0; c < CPT / 2; ++c) {
          const float2 x = __ffma2_rn(make_float2(__uint_as_float(sr[2 * c]), __uint_as_float(sr[2 * c + 1])),
                                      make_float2(sl2, sl2), make_float2(-lse2, -lse2));
          if (c < kPolyPairs) {  // a quarter of the exponentials on the FMA pipe
            const float2 e = exp2_poly2(x);
            pv[2 * c] = e.x;
            pv[2 * c + 1] = e.y;
          } else {
            pv[2 * c] = ex2(x.x);
            pv[2 * c + 1] = ex2(x.y);
          }
        }
        if (tail) {
#pragma unroll
          for (int c = 0; c < CPT; ++c)
            if (col0 + c >= kv_tail) pv[c] = 0.f;
        }
        mbar_wait(&dp_full[b], (uint32_t)(g >> 1) & 1u);
        if (threadIdx.x == 64) trace_ev(p.trace, p.trace_cap, 2, 3, g);
        tc_fence_after();
        uint32_t dr[CPT];
        if constexpr (CPT == 32) tmem_ld32(sb + 64u + (uint32_t)col0, dr);
        else tmem_ld16(sb + 64u + (uint32_t)col0, dr);
        uint32_t pk[CPT / 2];
#pragma unroll
        for (int c = 0; c < CPT / 2; ++c) {
          const float2 ds = __fmul2_rn(make_float2(pv[2 * c], pv[2 * c + 1]),
                                       __fadd2_rn(make_float2(__uint_as_float(dr[2 * c]), __uint_as_float(dr[2 * c + 1])),
                                                  make_float2(-dlt, -dlt)));
          pk[c] = pack_bf16(ds.x, ds.y);
        }
        if constexpr (CPT == 32) tmem_st16(sb + 64u + (uint32_t)col0, pk);  // dS over the dP columns read
        else tmem_st8(sb + 64u + (uint32_t)col0, pk);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&ds_full[b]);
        if (threadIdx.x == 64) trace_ev(p.trace, p.trace_cap, 2, 4, g);
      }
    }
  } else if (warp < R::PROD2) {
    // ---------------- epilogue: dQ = scale · acc -> bf16, direct 16-byte row stores ----------------
    // With fused δ these warps also compute δ = rowsum(dO ∘ O) of each item BEFORE draining
    // the previous item's accumulator, so the elementwise warps find it ready.
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    auto drain = [&](const Item& m, int it) {
      const int hh = m.bh % p.H, bb = m.bh / p.H;
      const int tok = m.blk * BQ + row;
      __nv_bfloat16* dst = p.out0 + bb * p.o0_sb + hh * p.o0_sh + (int64_t)tok * p.o0_sn;
      mbar_wait(acc_full, (uint32_t)it & 1u);
      tc_fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < HD; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tbase + lane_off + C::ACC_COL + (uint32_t)c0, r);
        if (c0 + 32 == HD) {
          tc_fence_before();
          mbar_arrive(acc_empty);
        }
        uint32_t pk[16];
#pragma unroll
        for (int c = 0; c < 16; ++c)
          pk[c] = pack_bf16(__uint_as_float(r[2 * c]) * p.scale, __uint_as_float(r[2 * c + 1]) * p.scale);
        if (tok < p.N) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            *reinterpret_cast<uint4*>(dst + c0 + 8 * u) = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        }
      }
    };
    int it = 0;
    bool pend = false;
    Item pm{};
    for (int wi = blockIdx.x; wi < p.num_items; wi += gridDim.x) {
      const Item m = get_item(p, wi, p.T_m);
      const int hh = m.bh % p.H, bb = m.bh / p.H;
      const int tok = m.blk * BQ + row;
      if (fused_delta) {
        float dl = 0.f;
        if (tok < p.N) {
          dl = row_delta<HD>(p.o_in + bb * p.oi_sb + hh * p.oi_sh + (int64_t)tok * p.oi_sn,
                             p.do_in + bb * p.di_sb + hh * p.di_sh + (int64_t)tok * p.di_sn);
          p.delta_out[(int64_t)m.bh * p.N + tok] = dl;
        }
        if (m.n > 0) {
          sdelta[(it & 1) * BQ + row] = dl;  // slot last read at the start of item it-2 (drained)
          mbar_arrive(&dlt_full[it & 1]);
        }
      }
      if (m.n == 0) {
        if (tok < p.N) {
          __nv_bfloat16* dst = p.out0 + bb * p.o0_sb + hh * p.o0_sh + (int64_t)tok * p.o0_sn;
          for (int c = 0; c < HD; c += 8) *reinterpret_cast<uint4*>(dst + c) = make_uint4(0, 0, 0, 0);
        }
        continue;
      }
      if (pend) drain(pm, it - 1);
      pm = m;
      pend = true;
      ++it;
    }
    if (pend) drain(pm, it - 1);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tbase, 512);
}

// ---------------------------------------------------------------------------------------
// K7 variant 4 (SPA2_DQ_VARIANT=4): k_dq3 with a 3-deep dP/dS ring.  The dQ pipeline is paced
// by barrier hops around its 2-deep S/dP TMEM ring (a build without elementwise work still
// takes 0.39 ms), so S moves to an SS-MMA reading Q from shared memory (Q double-buffered per
// item) and the freed TMEM holds a third dP/dS buffer: TMEM dO 64 | S 2x64 | dP/dS 3x64 |
// dQ 128.  The dO copy into TMEM is issued by the dP warp between the items' dP MMAs (in-order
// tcgen05 pipeline), so S of the next item never waits for it.
// ---------------------------------------------------------------------------------------
#ifndef SPA2_DQ4_NK
#define SPA2_DQ4_NK 3
#endif
#ifndef SPA2_DQ4_NV
#define SPA2_DQ4_NV 3
#endif
template <int HD>
struct Dq4Cfg {
  static constexpr int NK = SPA2_DQ4_NK, NV = SPA2_DQ4_NV;
  static constexpr int Q_BYTES = BQ * HD * 2;
  static constexpr int KV_BYTES = BKV * HD * 2;
  static constexpr int OFF_Q = 0;                        // [2 items] Q
  static constexpr int OFF_DOS = 2 * Q_BYTES;            // dO staging of the next item
  static constexpr int OFF_K = 3 * Q_BYTES;
  static constexpr int OFF_V = OFF_K + NK * KV_BYTES;
  static constexpr int OFF_DLT = OFF_V + NV * KV_BYTES;  // fused δ: float [2 items][128 rows]
  static constexpr int OFF_BAR = OFF_DLT + 2 * BQ * 4;
  static constexpr int NUM_BARS = 2 + 2 + 2 + 2 * NK + 2 * NV + 2 + 2 + 9 + 2 + 2;
  static constexpr int SMEM = OFF_BAR + NUM_BARS * 8 + 16 + kSmemAlignSlack;
  static constexpr uint32_t DO_COL = 0, S_COL = 64, DP_COL = 192, ACC_COL = 384;
};

template <int HD, int EWW>
__global__ void __launch_bounds__(Dq3Roles<EWW>::THREADS, 1)
    k_dq4(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
          const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO, const BwdParams p) {
  using C = Dq4Cfg<HD>;
  using R = Dq3Roles<EWW>;
  constexpr int NK = C::NK, NV = C::NV;
  constexpr int CPT = R::CPT;
  constexpr int kPolyPairs = CPT * SPA2_DQ_POLY_NUM / 64;  // of CPT/2 pairs
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* const smem = smem_align_1k(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars;             // [2] Q of item `it` in smem buffer it&1
  uint64_t* q_free = q_full + 2;       // [2] last S MMA of the item using buffer it&1 done
  uint64_t* do_full = q_free + 2;      // dO staging holds dO of item `it`
  uint64_t* do_free = do_full + 1;     // tcgen05.cp of dO(it) done: staging reusable
  uint64_t* k_full = do_free + 1;      // [NK]
  uint64_t* k_empty = k_full + NK;     // [NK]
  uint64_t* v_full = k_empty + NK;     // [NV]
  uint64_t* v_empty = v_full + NV;     // [NV]
  uint64_t* s_full = v_empty + NV;     // [2] S of tile g in S buffer g&1
  uint64_t* s_free = s_full + 2;       // [2] S of tile g read out
  uint64_t* dp_full = s_free + 2;      // [3] dP of tile g in dP buffer g%3
  uint64_t* ds_full = dp_full + 3;     // [3] dS of tile g packed over its dP columns
  uint64_t* dq_done = ds_full + 3;     // [3] dQ MMA of tile g done (dP buffer reusable)
  uint64_t* acc_full = dq_done + 3;
  uint64_t* acc_empty = acc_full + 1;
  uint64_t* dlt_full = acc_empty + 1;  // [2] fused δ of item `it` in sdelta[it & 1]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(dlt_full + 2);
  float* sdelta = reinterpret_cast<float*>(smem + C::OFF_DLT);
  const bool fused_delta = p.delta_out != nullptr;

  const int warp = (int)warp_id(), lane = (int)lane_id();
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_free[s], 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&s_free[s], 32 * EWW);
    }
    mbar_init(do_full, 1);
    mbar_init(do_free, 1);
    for (int s = 0; s < NK; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < NV; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int r = 0; r < 3; ++r) {
      mbar_init(&dp_full[r], 1);
      mbar_init(&ds_full[r], 32 * EWW);
      mbar_init(&dq_done[r], 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 128);
    mbar_init(&dlt_full[0], 128);
    mbar_init(&dlt_full[1], 128);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_holder;
  pdl_wait();  // everything above touched only this CTA's smem/TMEM
  pdl_trigger();

  if (warp == 0 || warp == R::PROD2) {
    // ---------------- TMA producers: warp 0 Q + K ring, warp 14 dO + V ring ----------------
    if (elect_one()) {
      const bool second = warp == R::PROD2;
      const CUtensorMap* tmR = second ? &tmDO : &tmQ;
      const CUtensorMap* tmKV = second ? &tmV : &tmK;
      tma_prefetch(tmR);
      tma_prefetch(tmKV);
      uint64_t* full = second ? v_full : k_full;
      uint64_t* empty = second ? v_empty : k_empty;
      const int ns = second ? NV : NK;
      uint8_t* const ring = smem + (second ? C::OFF_V : C::OFF_K);
      int it = 0, g = 0;
      for (int wi = blockIdx.x; wi < p.num_items; wi += gridDim.x) {
        const Item m = get_item(p, wi, p.T_m);
        if (m.n == 0) continue;
        const int hh = m.bh % p.H, bb = m.bh / p.H;
        if (!second) {  // Q(it) into its own buffer: read by the S MMAs for the whole item
          if (it >= 2) mbar_wait(&q_free[it & 1], ((uint32_t)(it >> 1) + 1u) & 1u);
          mbar_expect_tx(&q_full[it & 1], C::Q_BYTES);
          tma_load_5d(smem + C::OFF_Q + (it & 1) * C::Q_BYTES, tmR, &q_full[it & 1], 0, m.blk * BQ, 0, hh, bb);
        } else {  // dO(it) into the staging buffer, copied into TMEM by the dP issuer
          if (it >= 1) mbar_wait(do_free, (uint32_t)(it - 1) & 1u);
          mbar_expect_tx(do_full, C::Q_BYTES);
          tma_load_5d(smem + C::OFF_DOS, tmR, do_full, 0, m.blk * BQ, 0, hh, bb);
        }
        for (int t = 0; t < m.n; ++t, ++g) {
          const int s = g % ns;
          if (!second) trace_ev(p.trace, p.trace_cap, 0, 1, g);
          if (g >= ns) mbar_wait(&empty[s], ((uint32_t)(g / ns) + 1u) & 1u);
          if (!second) trace_ev(p.trace, p.trace_cap, 0, 2, g);
          mbar_expect_tx(&full[s], C::KV_BYTES);
          tma_load_5d(ring + s * C::KV_BYTES, tmKV, &full[s], 0, p.idx[m.beg + t] * BKV, 0, hh, bb);
        }
        ++it;
      }
    }
  } else if (warp == 1 || warp == R::ISSUE_DP || warp == R::ISSUE_DQ) {
    // ---------------- MMA issue: three warps, one per independent stream ----------------
    // warp 1: S = Q K_jᵀ (SS, Q from smem);  ISSUE_DP: dO copy into TMEM per item (issued after
    // the previous item's last dP and before this item's first: tcgen05.cp and tcgen05.mma of
    // one thread execute in order) + dP = dO V_jᵀ (TS);  ISSUE_DQ: dQ += dS K_j (TS).
    constexpr uint32_t idS = idesc_bf16(BQ, BKV, false, false);
    constexpr uint32_t idQ = idesc_bf16(BQ, HD, false, true);
    const uint64_t dQ0 = sw128_desc(smem_u32(smem + C::OFF_Q), 16, 1024);
    const uint64_t dDOS = sw128_desc(smem_u32(smem + C::OFF_DOS), 16, 1024);
    const uint64_t dK0 = sw128_desc(smem_u32(smem + C::OFF_K), 16, 1024);
    const uint64_t dV0 = sw128_desc(smem_u32(smem + C::OFF_V), 16, 1024);
    const uint64_t dKm0 = sw128_desc(smem_u32(smem + C::OFF_K), BKV * 128, 1024);
    constexpr uint64_t KV16 = (uint64_t)(C::KV_BYTES >> 4);
    Cursor c;
    cursor_init(c, p, p.T_m);
    if (warp == 1) {
      for (; c.valid; cursor_next(c, p, p.T_m)) {
        if (c.t == 0) mbar_wait(&q_full[c.it & 1], (uint32_t)(c.it >> 1) & 1u);
        const int b = c.g & 1, sk = c.g % NK;
        if (c.g >= 2) mbar_wait(&s_free[b], (uint32_t)((c.g - 2) >> 1) & 1u);  // S(g-2) read out
        mbar_wait(&k_full[sk], (uint32_t)(c.g / NK) & 1u);
        tc_fence_after();
        trace_ev(p.trace, p.trace_cap, 1, 2, c.g);
        const uint64_t dK = dK0 + (uint64_t)sk * KV16;
        const uint64_t dQ = dQ0 + (uint64_t)((c.it & 1) * (C::Q_BYTES >> 4));
        const uint32_t sb = tbase + C::S_COL + (uint32_t)(b * 64);
#ifdef SPA2_MMA_BATCH
        if constexpr (HD == 128) {
          mma_bf16_ss_k8_w<2ull, (uint64_t)(BQ * 128 / 16), 2ull, (uint64_t)(BKV * 128 / 16)>(sb, dQ, dK, idS, 0u);
        } else
#endif
        {
#pragma unroll
          for (int ks = 0; ks < HD / 16; ++ks) {
            const uint64_t qo = (uint64_t)(((ks * 16 / 64) * BQ * 128 + (ks * 16 % 64) * 2) >> 4);
            const uint64_t ko = (uint64_t)(((ks * 16 / 64) * BKV * 128 + (ks * 16 % 64) * 2) >> 4);
            mma_bf16_w(sb, dQ + qo, dK + ko, idS, ks > 0 ? 1u : 0u);
          }
        }
        mma_commit_w(&s_full[b]);
        if (c.t == c.n - 1) mma_commit_w(&q_free[c.it & 1]);
        trace_ev(p.trace, p.trace_cap, 1, 3, c.g);
      }
    } else {
      // dP = dO V_jᵀ (TS) and dQ += dS K_j (TS), by two warps (dP(g) waits for dQ(g-2) to
      // COMPLETE: it overwrites the TMEM columns dQ(g-2) reads dS from).  With
      // -DSPA2_DQ_MERGED one warp issues both as dQ(g-2), dP(g), ...: tcgen05 MMAs issued by
      // one thread execute in issue order, so the completion wait disappears.
      auto issue_dp = [&](const Cursor& cc) {
        if (cc.t == 0) {  // dO(it) into TMEM, in issue order after dP of the previous item
          mbar_wait(do_full, (uint32_t)cc.it & 1u);
          tc_fence_after();
#pragma unroll
          for (int ks = 0; ks < HD / 16; ++ks) {
            const uint64_t qo = (uint64_t)(((ks * 16 / 64) * BQ * 128 + (ks * 16 % 64) * 2) >> 4);
            tmem_cp_128x256b_w(tbase + C::DO_COL + (uint32_t)(ks * 8), dDOS + qo);
          }
          mma_commit_w(do_free);
        }
        const int r = cc.g % 3, sv = cc.g % NV;
        if (cc.g >= 3) mbar_wait(&dq_done[r], (uint32_t)((cc.g - 3) / 3) & 1u);  // dS(g-3) consumed
        mbar_wait(&v_full[sv], (uint32_t)(cc.g / NV) & 1u);
        tc_fence_after();
        const uint64_t dV = dV0 + (uint64_t)sv * KV16;
        const uint32_t pb = tbase + C::DP_COL + (uint32_t)(r * 64);
#ifdef SPA2_MMA_BATCH
        if constexpr (HD == 128) {
          mma_bf16_ts_k8_w<8u, 2ull, (uint64_t)(BKV * 128 / 16)>(pb, tbase + C::DO_COL, dV, idS, 0u);
        } else
#endif
        {
#pragma unroll
          for (int ks = 0; ks < HD / 16; ++ks)
            mma_bf16_ts_w(pb, tbase + C::DO_COL + (uint32_t)(ks * 8),
                          dV + (uint64_t)((((ks * 16 / 64) * BKV * 128 + (ks * 16 % 64) * 2)) >> 4), idS, ks > 0 ? 1u : 0u);
        }
        mma_commit_w(&dp_full[r]);
        mma_commit_w(&v_empty[sv]);
      };
      auto issue_dq = [&](const Cursor& cc) {
        const int r = cc.g % 3, sk = cc.g % NK;
        if (cc.t == 0 && cc.it >= 1) mbar_wait(acc_empty, (uint32_t)(cc.it - 1) & 1u);
        mbar_wait(&ds_full[r], (uint32_t)(cc.g / 3) & 1u);
        tc_fence_after();
        trace_ev(p.trace, p.trace_cap, 1, 4, cc.g);
        const uint64_t dKm = dKm0 + (uint64_t)sk * KV16;
        const uint32_t pb = tbase + C::DP_COL + (uint32_t)(r * 64);
#ifdef SPA2_MMA_BATCH
        if constexpr (CPT == 16) {
          mma_bf16_ts_k4_w<16u, 128ull>(tbase + C::ACC_COL, pb, dKm, idQ, cc.t > 0 ? 1u : 0u);
        } else
#endif
        {
#pragma unroll
          for (int ks = 0; ks < BKV / 16; ++ks)
            mma_bf16_ts_w(tbase + C::ACC_COL, pb + ds_col<CPT>(ks), dKm + (uint64_t)((ks * 2048) >> 4), idQ,
                          (cc.t > 0 || ks > 0) ? 1u : 0u);
        }
        mma_commit_w(&dq_done[r]);
        mma_commit_w(&k_empty[sk]);
        if (cc.t == cc.n - 1) mma_commit_w(acc_full);
        trace_ev(p.trace, p.trace_cap, 1, 5, cc.g);
      };
      if (warp == R::ISSUE_DP) {
        for (; c.valid; cursor_next(c, p, p.T_m)) issue_dp(c);
      } else {
        for (; c.valid; cursor_next(c, p, p.T_m)) issue_dq(c);
      }
    }
  } else if (warp < R::EPI0) {
    // ---------------- elementwise: dS = P ∘ (dP − δ), P = exp2(S·c − LSE·log2e) ----------------
    const int q4 = warp & 3;
    const int grp = (warp - 2) >> 2;
    const int row = q4 * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const int col0 = CPT * grp;
    const int kv_tail = p.N - (p.T_n - 1) * BKV;
    const float sl2 = p.sl2;
    int g = 0, it = 0;
    for (int wi = blockIdx.x; wi < p.num_items; wi += gridDim.x) {
      const Item m = get_item(p, wi, p.T_m);
      if (m.n == 0) continue;
      const int tok = m.blk * BQ + row;
      const bool valid = tok < p.N;
      const float lse2 = valid ? __ldg(p.lse + (int64_t)m.bh * p.N + tok) * kLog2e : INFINITY;
      float dlt;
      if (fused_delta) {  // computed one item ahead by the epilogue warps
        mbar_wait(&dlt_full[it & 1], (uint32_t)(it >> 1) & 1u);
        dlt = valid ? sdelta[(it & 1) * BQ + row] : 0.f;
      } else {
        dlt = valid ? __ldg(p.delta + (int64_t)m.bh * p.N + tok) : 0.f;
      }
      ++it;
      // key-block index of the next tile is loaded one tile ahead (off the critical path)
      int j_next = __ldg(p.idx + m.beg);
      for (int t = 0; t < m.n; ++t, ++g) {
        const int b = g & 1;
        const bool tail = kv_tail < BKV && j_next == p.T_n - 1;
        if (t + 1 < m.n) j_next = __ldg(p.idx + m.beg + t + 1);
        const int r = g % 3;
        const uint32_t sb = tbase + lane_off + C::S_COL + (uint32_t)(b * 64);
        const uint32_t pb = tbase + lane_off + C::DP_COL + (uint32_t)(r * 64);
        if (threadIdx.x == 64) trace_ev(p.trace, p.trace_cap, 2, 1, g);
        mbar_wait(&s_full[b], (uint32_t)(g >> 1) & 1u);
        if (threadIdx.x == 64) trace_ev(p.trace, p.trace_cap, 2, 2, g);
        tc_fence_after();
        uint32_t sr[CPT];
        if constexpr (CPT == 32) tmem_ld32(sb + (uint32_t)col0, sr);
        else tmem_ld16(sb + (uint32_t)col0, sr);
        tc_fence_before();
        mbar_arrive(&s_free[b]);  // S(g) is in registers: the S issuer may overwrite it
        // packed fp32x2 math (FFMA2/FADD2/FMUL2): the issue slots of this SM sub-partition are
        // shared with an MMA-issuing warp, so fewer instructions per element = faster MMAs
        float pv[CPT];
#pragma unroll
        for (int c = 0; c < CPT / 2; ++c) {
          const float2 x = __ffma2_rn(make_float2(__uint_as_float(sr[2 * c]), __uint_as_float(sr[2 * c + 1])),
                                      make_float2(sl2, sl2), make_float2(-lse2, -lse2));
          if (c < kPolyPairs) {  // a quarter of the exponentials on the FMA pipe
            const float2 e = exp2_poly2(x);
            pv[2 * c] = e.x;
            pv[2 * c + 1] = e.y;
          } else {
            pv[2 * c] = ex2(x.x);
            pv[2 * c + 1] = ex2(x.y);
          }
        }
        if (tail) {
#pragma unroll
          for (int c = 0; c < CPT; ++c)
            if (col0 + c >= kv_tail) pv[c] = 0.f;
        }
        mbar_wait(&dp_full[r], (uint32_t)(g / 3) & 1u);
        if (threadIdx.x == 64) trace_ev(p.trace, p.trace_cap, 2, 3, g);
        tc_fence_after();
        uint32_t dr[CPT];
        if constexpr (CPT == 32) tmem_ld32(pb + (uint32_t)col0, dr);
        else tmem_ld16(pb + (uint32_t)col0, dr);
        uint32_t pk[CPT / 2];
#pragma unroll
        for (int c = 0; c < CPT / 2; ++c) {
          const float2 ds = __fmul2_rn(make_float2(pv[2 * c], pv[2 * c + 1]),
                                       __fadd2_rn(make_float2(__uint_as_float(dr[2 * c]), __uint_as_float(dr[2 * c + 1])),
                                                  make_float2(-dlt, -dlt)));
          pk[c] = pack_bf16(ds.x, ds.y);
        }
        if constexpr (CPT == 32) tmem_st16(pb + (uint32_t)col0, pk);  // dS over the dP columns read
        else tmem_st8(pb + (uint32_t)col0, pk);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&ds_full[r]);
        if (threadIdx.x == 64) trace_ev(p.trace, p.trace_cap, 2, 4, g);
      }
    }
  } else if (warp < R::PROD2) {
    // ---------------- epilogue: dQ = scale · acc -> bf16, direct 16-byte row stores ----------------
    // With fused δ these warps also compute δ = rowsum(dO ∘ O) of each item BEFORE draining
    // the previous item's accumulator, so the elementwise warps find it ready.
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    auto drain = [&](const Item& m, int it) {
      const int hh = m.bh % p.H, bb = m.bh / p.H;
      const int tok = m.blk * BQ + row;
      __nv_bfloat16* dst = p.out0 + bb * p.o0_sb + hh * p.o0_sh + (int64_t)tok * p.o0_sn;
      mbar_wait(acc_full, (uint32_t)it & 1u);
      tc_fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < HD; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tbase + lane_off + C::ACC_COL + (uint32_t)c0, r);
        if (c0 + 32 == HD) {
          tc_fence_before();
          mbar_arrive(acc_empty);
        }
        uint32_t pk[16];
#pragma unroll
        for (int c = 0; c < 16; ++c)
          pk[c] = pack_bf16(__uint_as_float(r[2 * c]) * p.scale, __uint_as_float(r[2 * c + 1]) * p.scale);
        if (tok < p.N) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            *reinterpret_cast<uint4*>(dst + c0 + 8 * u) = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        }
      }
    };
    int it = 0;
    bool pend = false;
    Item pm{};
    for (int wi = blockIdx.x; wi < p.num_items; wi += gridDim.x) {
      const Item m = get_item(p, wi, p.T_m);
      const int hh = m.bh % p.H, bb = m.bh / p.H;
      const int tok = m.blk * BQ + row;
      if (fused_delta) {
        float dl = 0.f;
        if (tok < p.N) {
          dl = row_delta<HD>(p.o_in + bb * p.oi_sb + hh * p.oi_sh + (int64_t)tok * p.oi_sn,
                             p.do_in + bb * p.di_sb + hh * p.di_sh + (int64_t)tok * p.di_sn);
          p.delta_out[(int64_t)m.bh * p.N + tok] = dl;
        }
        if (m.n > 0) {
          sdelta[(it & 1) * BQ + row] = dl;  // slot last read at the start of item it-2 (drained)
          mbar_arrive(&dlt_full[it & 1]);
        }
      }
      if (m.n == 0) {
        if (tok < p.N) {
          __nv_bfloat16* dst = p.out0 + bb * p.o0_sb + hh * p.o0_sh + (int64_t)tok * p.o0_sn;
          for (int c = 0; c < HD; c += 8) *reinterpret_cast<uint4*>(dst + c) = make_uint4(0, 0, 0, 0);
        }
        continue;
      }
      if (pend) drain(pm, it - 1);
      pm = m;
      pend = true;
      ++it;
    }
    if (pend) drain(pm, it - 1);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tbase, 512);
}

int dq_ew_warps() {
  static const int v = [] {
    const char* e = getenv("SPA2_DQ_EW");
    return (e != nullptr && atoi(e) == 8) ? 8 : 16;
  }();
  return v;
}

int dq_variant() {
  static const int v = [] {
    const char* e = getenv("SPA2_DQ_VARIANT");
    return e != nullptr ? atoi(e) : 3;
  }();
  return v;
}

bool dq_variant2() {
  static const bool v = [] {
    const char* e = getenv("SPA2_DQ_PERSISTENT");
    return !(e != nullptr && e[0] == '1');
  }();
  return v;
}


// Warp roles: 0 TMA (K, Q), 1 MMA, 2 .. 2+EWW-1 elementwise (EWW/4 warps per TMEM lane
// quarter, 256/EWW columns each), then 4 epilogue warps, then TMA (V, dO).
template <int EWW>
struct DkvRoles {
  static constexpr int EPI0 = 2 + EWW;           // first epilogue warp
  static constexpr int PROD2 = EPI0 + 4;         // second producer warp
  static constexpr int ISSUE2 = PROD2 + 1;       // dV/dK issuing warp
  static constexpr int THREADS = 32 * (ISSUE2 + 1);
  static constexpr int CPT = 256 / EWW;          // S/dP columns per elementwise thread
};

template <int HD>
struct DkvCfg {
  static constexpr int NS = 2;
  static constexpr int KV_BYTES = BKV * HD * 2;
  static constexpr int Q_BYTES = BQ * HD * 2;
  static constexpr int PB = BQ * BKV * 2;
  static constexpr int OFF_KV = 0;                            // [K | V] of the current item
  static constexpr int OFF_QDO = 2 * KV_BYTES;                // [NS stages][Q | dO]
  static constexpr int OFF_PDS = OFF_QDO + NS * 2 * Q_BYTES;  // [2 buffers][P | dS]
  static constexpr int OFF_BAR = OFF_PDS + 2 * 2 * PB;
  static constexpr int NUM_BARS = 2 + 2 * NS + 2 * 7;
  static constexpr int SMEM = OFF_BAR + NUM_BARS * 8 + 16 + kSmemAlignSlack;
  static constexpr uint32_t S_COL = 0, DP_COL = 128, ACC_COL = 256;  // acc a: dV at +a*128, dK at +a*128+64
};

template <int HD, int EWW>
__global__ void __launch_bounds__(DkvRoles<EWW>::THREADS, 1)
    k_dkdv(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
           const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO, const BwdParams p) {
  using C = DkvCfg<HD>;
  using R = DkvRoles<EWW>;
  constexpr int NS = C::NS;
  constexpr int EWT = 32 * EWW;  // elementwise threads
  constexpr int kDkvPolyPairs = R::CPT * SPA2_DKDV_POLY_NUM / 64;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* const smem = smem_align_1k(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* kv_full = bars;             // K/V of item `it` landed
  uint64_t* kv_empty = kv_full + 1;     // last S/dP MMA of item `it` done: K/V slot reusable
  uint64_t* qdo_full = kv_empty + 1;    // [NS]
  uint64_t* qdo_empty = qdo_full + NS;  // [NS]
  uint64_t* s_full = qdo_empty + NS;    // [2] S of tile g in TMEM buffer g&1
  uint64_t* dp_full = s_full + 2;       // [2] dP of tile g
  uint64_t* p_full = dp_full + 2;       // [2] P of tile g in smem buffer g&1
  uint64_t* ds_full = p_full + 2;       // [2] dS of tile g in smem (S/dP TMEM buffer read)
  uint64_t* pds_free = ds_full + 2;     // [2] dV/dK MMAs reading buffer b done
  uint64_t* acc_full = pds_free + 2;    // [2]
  uint64_t* acc_empty = acc_full + 2;   // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = (int)warp_id(), lane = (int)lane_id();
  if (threadIdx.x == 0) {
    mbar_init(kv_full, 2);  // two producers: warp 0 (K, Q) and warp PROD2 (V, dO)
    mbar_init(kv_empty, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&dp_full[s], 1);
      mbar_init(&p_full[s], EWT);
      mbar_init(&ds_full[s], EWT);
      mbar_init(&pds_free[s], 1);
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], 128);
    }
    for (int s = 0; s < NS; ++s) {
      mbar_init(&qdo_full[s], 2);
      mbar_init(&qdo_empty[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_holder;

  if (warp == 0 || warp == R::PROD2) {
    // ---------------- TMA producers: warp 0 loads K and Q, warp PROD2 loads V and dO ----------------
    // (requests issued by one warp are served one at a time; two issuing warps double the
    // per-SM fill rate, tools/tma_rate.py)
    if (elect_one()) {
      const bool second = warp == R::PROD2;
      const CUtensorMap* tmKV = second ? &tmV : &tmK;
      const CUtensorMap* tmR = second ? &tmDO : &tmQ;
      tma_prefetch(tmKV);
      tma_prefetch(tmR);
      uint8_t* const kv_dst = smem + C::OFF_KV + (second ? C::KV_BYTES : 0);
      const int r_off = second ? C::Q_BYTES : 0;
      int it = 0, g = 0;
      for (int wi = blockIdx.x; wi < p.num_items; wi += gridDim.x) {
        const Item m = get_item(p, wi, p.T_n);
        if (m.n == 0) continue;
        const int hh = m.bh % p.H, bb = m.bh / p.H;
        if (it >= 1) mbar_wait(kv_empty, (uint32_t)(it - 1) & 1u);
        mbar_expect_tx(kv_full, C::KV_BYTES);
        tma_load_5d(kv_dst, tmKV, kv_full, 0, m.blk * BKV, 0, hh, bb);
        for (int t = 0; t < m.n; ++t, ++g) {
          const int i = p.idx[m.beg + t];
          const int s = g % NS;
          if (!second) trace_ev(p.trace, p.trace_cap, 0, 1, g);
          if (g >= NS) mbar_wait(&qdo_empty[s], ((uint32_t)(g / NS) + 1u) & 1u);
          if (!second) trace_ev(p.trace, p.trace_cap, 0, 2, g);
          mbar_expect_tx(&qdo_full[s], C::Q_BYTES);
          tma_load_5d(smem + C::OFF_QDO + s * 2 * C::Q_BYTES + r_off, tmR, &qdo_full[s], 0, i * BQ, 0, hh, bb);
        }
        ++it;
      }
    }
  } else if (warp == 1 || warp == R::ISSUE2) {
    // ---------------- MMA issue: two warps, one per stream ----------------
    // warp 1: S = Q_i K_jᵀ and dP = dO_i V_jᵀ of tile g into TMEM buffer g&1 (free once the
    // elementwise warps have consumed tile g-2);  warp ISSUE2: dVᵀ += dO_iᵀ P (after P is in
    // smem) then dKᵀ += Q_iᵀ dS (after dS).  Warp-collective issue, warp-uniform descriptors.
    constexpr uint32_t idS = idesc_bf16(BQ, BKV, false, false);
    constexpr uint32_t idT = idesc_bf16(HD, BKV, true, true);
    const uint64_t dK = sw128_desc(smem_u32(smem + C::OFF_KV), 16, 1024);
    const uint64_t dV = dK + (uint64_t)(C::KV_BYTES >> 4);
    const uint64_t dQk0 = sw128_desc(smem_u32(smem + C::OFF_QDO), 16, 1024);        // K-major Q / dO
    const uint64_t dQm0 = sw128_desc(smem_u32(smem + C::OFF_QDO), BQ * 128, 1024);  // MN-major Q / dO
    const uint64_t dPm0 = sw128_desc(smem_u32(smem + C::OFF_PDS), BQ * 128, 1024);  // MN-major P / dS
    constexpr uint64_t STAGE16 = (uint64_t)((2 * C::Q_BYTES) >> 4), Q16 = (uint64_t)(C::Q_BYTES >> 4);
    constexpr uint64_t PBUF16 = (uint64_t)((2 * C::PB) >> 4), PB16 = (uint64_t)(C::PB >> 4);
    Cursor c;
    cursor_init(c, p, p.T_n);
    if (warp == 1) {
      for (; c.valid; cursor_next(c, p, p.T_n)) {
        if (c.t == 0) mbar_wait(kv_full, (uint32_t)c.it & 1u);
        const int s = c.g % NS;
        const uint32_t b = (uint32_t)(c.g & 1);
        if (c.g >= 2) mbar_wait(&ds_full[b], (uint32_t)((c.g - 2) >> 1) & 1u);  // S/dP buffer b read
        mbar_wait(&qdo_full[s], (uint32_t)(c.g / NS) & 1u);
        tc_fence_after();
        trace_ev(p.trace, p.trace_cap, 1, 2, c.g);
        const uint64_t dQ = dQk0 + (uint64_t)s * STAGE16, dDO = dQ + Q16;
#pragma unroll
        for (int ks = 0; ks < HD / 16; ++ks) {
          const uint64_t qo = (uint64_t)(((ks * 16 / 64) * BQ * 128 + (ks * 16 % 64) * 2) >> 4);
          const uint64_t ko = (uint64_t)(((ks * 16 / 64) * BKV * 128 + (ks * 16 % 64) * 2) >> 4);
          mma_bf16_w(tbase + C::S_COL + b * 64, dQ + qo, dK + ko, idS, ks > 0 ? 1u : 0u);
        }
        mma_commit_w(&s_full[b]);
#pragma unroll
        for (int ks = 0; ks < HD / 16; ++ks) {
          const uint64_t qo = (uint64_t)(((ks * 16 / 64) * BQ * 128 + (ks * 16 % 64) * 2) >> 4);
          const uint64_t ko = (uint64_t)(((ks * 16 / 64) * BKV * 128 + (ks * 16 % 64) * 2) >> 4);
          mma_bf16_w(tbase + C::DP_COL + b * 64, dDO + qo, dV + ko, idS, ks > 0 ? 1u : 0u);
        }
        mma_commit_w(&dp_full[b]);
        if (c.t == c.n - 1) mma_commit_w(kv_empty);  // K_j / V_j are only read by S and dP
      }
    } else {
      for (; c.valid; cursor_next(c, p, p.T_n)) {
        const int pb = c.g & 1;
        const int s = c.g % NS;
        const uint32_t acc = tbase + C::ACC_COL + (uint32_t)((c.it & 1) * 128);
        const uint64_t dQm = dQm0 + (uint64_t)s * STAGE16, dDOm = dQm + Q16;
        const uint64_t dP = dPm0 + (uint64_t)pb * PBUF16, dDS = dP + PB16;
        const bool first = c.t == 0;
        if (first && c.it >= 2) mbar_wait(&acc_empty[c.it & 1], ((uint32_t)(c.it >> 1) + 1u) & 1u);
        mbar_wait(&p_full[pb], (uint32_t)(c.g >> 1) & 1u);
        tc_fence_after();
        trace_ev(p.trace, p.trace_cap, 1, 4, c.g);
#pragma unroll
        for (int ks = 0; ks < BQ / 16; ++ks)
          mma_bf16_w(acc, dDOm + (uint64_t)(ks * 128), dP + (uint64_t)(ks * 128), idT, (!first || ks > 0) ? 1u : 0u);
        mbar_wait(&ds_full[pb], (uint32_t)(c.g >> 1) & 1u);
        tc_fence_after();
        trace_ev(p.trace, p.trace_cap, 1, 5, c.g);
#pragma unroll
        for (int ks = 0; ks < BQ / 16; ++ks)
          mma_bf16_w(acc + 64, dQm + (uint64_t)(ks * 128), dDS + (uint64_t)(ks * 128), idT, (!first || ks > 0) ? 1u : 0u);
        mma_commit_w(&pds_free[pb]);
        mma_commit_w(&qdo_empty[s]);
        if (c.t == c.n - 1) mma_commit_w(&acc_full[c.it & 1]);
      }
    }
  } else if (warp < R::EPI0) {
    // ---------------- P / dS warps: EWW/4 warps per TMEM lane quarter, CPT columns each ----
    constexpr int CPT = R::CPT;
    const int q4 = warp & 3;
    const int grp = (warp - 2) >> 2;
    const int row = q4 * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const uint32_t col0 = (uint32_t)(CPT * grp);
    const float sl2 = p.sl2;
    const bool tr = threadIdx.x == 64;
    int g = 0;
    for (int wi = blockIdx.x; wi < p.num_items; wi += gridDim.x) {
      const Item m = get_item(p, wi, p.T_n);
      if (m.n == 0) continue;
      const int64_t rowbase = (int64_t)m.bh * p.N;
      auto load_stats = [&](int t, float& lse2, float& dlt) {
        const int tok = p.idx[m.beg + t] * BQ + row;
        const bool valid = tok < p.N;
        lse2 = valid ? __ldg(p.lse + rowbase + tok) * kLog2e : INFINITY;
        dlt = valid ? __ldg(p.delta + rowbase + tok) : 0.f;
      };
      float lse2, dlt;
      load_stats(0, lse2, dlt);
      for (int t = 0; t < m.n; ++t, ++g) {
        const uint32_t b = (uint32_t)(g & 1);
        float lse2_n = 0.f, dlt_n = 0.f;
        if (t + 1 < m.n) load_stats(t + 1, lse2_n, dlt_n);  // prefetch the next tile's row statistics
        if (tr) trace_ev(p.trace, p.trace_cap, 2, 1, g);
        mbar_wait(&s_full[b], (uint32_t)(g >> 1) & 1u);
        if (tr) trace_ev(p.trace, p.trace_cap, 2, 2, g);
        tc_fence_after();
        uint32_t sr[CPT];
        if constexpr (CPT == 32) tmem_ld32(tbase + lane_off + C::S_COL + b * 64 + col0, sr);
        else tmem_ld16(tbase + lane_off + C::S_COL + b * 64 + col0, sr);
        float pv[CPT];
        uint32_t pk[CPT / 2];
#pragma unroll
        for (int c = 0; c < CPT / 2; ++c) {
          const float2 x = __ffma2_rn(make_float2(__uint_as_float(sr[2 * c]), __uint_as_float(sr[2 * c + 1])),
                                      make_float2(sl2, sl2), make_float2(-lse2, -lse2));
          if (c < kDkvPolyPairs) {  // part of the exponentials on the FMA pipe (exp2_poly2)
            const float2 e = exp2_poly2(x);
            pv[2 * c] = e.x;
            pv[2 * c + 1] = e.y;
          } else {
            pv[2 * c] = ex2(x.x);
            pv[2 * c + 1] = ex2(x.y);
          }
          pk[c] = pack_bf16(pv[2 * c], pv[2 * c + 1]);
        }
        if (g >= 2) mbar_wait(&pds_free[b], ((uint32_t)(g >> 1) + 1u) & 1u);  // buffer b free (tile g-2 done)
        if (tr) trace_ev(p.trace, p.trace_cap, 2, 3, g);
        const uint32_t sP = smem_u32(smem + C::OFF_PDS + (int)b * 2 * C::PB), sDS = sP + C::PB;
#pragma unroll
        for (int u = 0; u < CPT / 8; ++u) {
          const uint32_t off = sw128_offset((uint32_t)row, col0 / 8 + (uint32_t)u);
          st_shared_v4(sP + off, pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        }
        fence_proxy_async_smem();
        mbar_arrive(&p_full[b]);
        if (tr) trace_ev(p.trace, p.trace_cap, 2, 5, g);
        mbar_wait(&dp_full[b], (uint32_t)(g >> 1) & 1u);
        tc_fence_after();
        uint32_t dr[CPT];
        if constexpr (CPT == 32) tmem_ld32(tbase + lane_off + C::DP_COL + b * 64 + col0, dr);
        else tmem_ld16(tbase + lane_off + C::DP_COL + b * 64 + col0, dr);
#pragma unroll
        for (int c = 0; c < CPT / 2; ++c) {
          const float2 ds = __fmul2_rn(make_float2(pv[2 * c], pv[2 * c + 1]),
                                       __fadd2_rn(make_float2(__uint_as_float(dr[2 * c]), __uint_as_float(dr[2 * c + 1])),
                                                  make_float2(-dlt, -dlt)));
          pk[c] = pack_bf16(ds.x, ds.y);
        }
#pragma unroll
        for (int u = 0; u < CPT / 8; ++u) {
          const uint32_t off = sw128_offset((uint32_t)row, col0 / 8 + (uint32_t)u);
          st_shared_v4(sDS + off, pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        }
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(&ds_full[b]);
        if (tr) trace_ev(p.trace, p.trace_cap, 2, 4, g);
        lse2 = lse2_n;
        dlt = dlt_n;
      }
    }
  } else if (warp < R::PROD2) {
    // ---------------- epilogue warps: TMEM -> registers -> coalesced global stores ----
    const int q4 = warp & 3;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const int dim = (HD == 128) ? q4 * 32 + lane : 16 * q4 + lane;  // M=64 accumulators: lanes 0-15 per quarter
    const bool own = (HD == 128) || lane < 16;
    const bool tr = threadIdx.x == 32 * R::EPI0;
    int it = 0;
    for (int wi = blockIdx.x; wi < p.num_items; wi += gridDim.x) {
      const Item m = get_item(p, wi, p.T_n);
      const int hh = m.bh % p.H, bb = m.bh / p.H;
      __nv_bfloat16* dk = p.out0 + bb * p.o0_sb + hh * p.o0_sh + (int64_t)m.blk * BKV * p.o0_sn + dim;
      __nv_bfloat16* dv = p.out1 + bb * p.o1_sb + hh * p.o1_sh + (int64_t)m.blk * BKV * p.o1_sn + dim;
      const int rows = min(BKV, p.N - m.blk * BKV);
      if (m.n == 0) {
        // no query block keeps this key block: its dK and dV rows are exactly zero
        if (own)
          for (int r = 0; r < rows; ++r) {
            dk[(int64_t)r * p.o0_sn] = __float2bfloat16(0.f);
            dv[(int64_t)r * p.o1_sn] = __float2bfloat16(0.f);
          }
        continue;
      }
      const int st = it & 1;
      if (tr) trace_ev(p.trace, p.trace_cap, 3, 1, it);
      mbar_wait(&acc_full[st], (uint32_t)(it >> 1) & 1u);
      if (tr) trace_ev(p.trace, p.trace_cap, 3, 2, it);
      tc_fence_after();
#pragma unroll 1
      for (int part = 0; part < 4; ++part) {  // dV rows 0-31, 32-63, then dK rows 0-31, 32-63
        uint32_t r32[32];
        tmem_ld32(tbase + lane_off + C::ACC_COL + (uint32_t)(st * 128 + part * 32), r32);
        if (part == 3) {
          tc_fence_before();
          mbar_arrive(&acc_empty[st]);  // both accumulators read: TMEM set reusable
        }
        const bool is_k = part >= 2;
        __nv_bfloat16* dst = (is_k ? dk : dv) + (int64_t)((part & 1) * 32) * (is_k ? p.o0_sn : p.o1_sn);
        const int64_t sn = is_k ? p.o0_sn : p.o1_sn;
        const float mul = is_k ? p.scale : 1.f;
        const int rr = rows - (part & 1) * 32;
        if (own) {
#pragma unroll
          for (int r = 0; r < 32; ++r)
            if (r < rr) dst[(int64_t)r * sn] = __float2bfloat16(__uint_as_float(r32[r]) * mul);
        }
      }
      if (tr) trace_ev(p.trace, p.trace_cap, 3, 3, it);
      ++it;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tbase, 512);
}

template <int HD, int NSL_ = 5, int NPB_ = 1>
struct Dkv5Cfg {
  static constexpr int NSL = NSL_;  // 32 KB operand slots: Q(g) -> slot 2g mod NSL, dO(g) -> slot 2g+1 mod NSL
  static constexpr int NPB = NPB_;  // [P | dS] buffers
  static constexpr int KV_BYTES = BKV * HD * 2;
  static constexpr int Q_BYTES = BQ * HD * 2;
  static constexpr int PB = BQ * BKV * 2;
  static constexpr int OFF_KV = 0;                         // [K | V] of the current item
  static constexpr int OFF_SL = 2 * KV_BYTES;              // [NSL] Q / dO operand slots
  static constexpr int OFF_PDS = OFF_SL + NSL * Q_BYTES;   // [NPB][P | dS]
  static constexpr int OFF_BAR = OFF_PDS + NPB * 2 * PB;
  static constexpr int NUM_BARS = 2 + 2 * NSL + 6 + 4 * NPB + 4;
  static constexpr int SMEM = OFF_BAR + NUM_BARS * 8 + 16 + kSmemAlignSlack;
  static constexpr uint32_t S_COL = 0, DP_COL = 128, ACC_COL = 256;
};

// K6 variant 5: the Q and dO tiles of a kept tile live in a 5-slot ring of 32 KB operand slots
// (2.5 tiles in flight instead of 2 stages of [Q|dO]).  Each operand has two readers issued by
// different warps (Q: S and dKᵀ, dO: dP and dVᵀ), so its slot is released by two commits, one
// per issuer; the dVᵀ issuer also waits for dO(g) to land (P(g) existing only proves S(g)
// finished).  P and dS share one smem buffer.
template <int HD, int EWW, int NSL_ = 5, int NPB_ = 1>
__global__ void __launch_bounds__(DkvRoles<EWW>::THREADS, 1)
    k_dkdv5(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
           const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO, const BwdParams p) {
  using C = Dkv5Cfg<HD, NSL_, NPB_>;
  using R = DkvRoles<EWW>;
  constexpr int NSL = C::NSL;
  constexpr int NPB = C::NPB;
  constexpr int EWT = 32 * EWW;  // elementwise threads
  constexpr int kDkvPolyPairs = R::CPT * SPA2_DKDV_POLY_NUM / 64;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* const smem = smem_align_1k(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* kv_full = bars;             // K/V of item `it` landed
  uint64_t* kv_empty = kv_full + 1;     // last S/dP MMA of item `it` done: K/V slot reusable
  uint64_t* sl_full = kv_empty + 1;     // [NSL] operand slot holds operand u (Q(g): u=2g, dO(g): u=2g+1)
  uint64_t* sl_empty = sl_full + NSL;   // [NSL] both MMAs reading operand u are done
  uint64_t* s_full = sl_empty + NSL;    // [2] S of tile g in TMEM buffer g&1
  uint64_t* dp_full = s_full + 2;       // [2] dP of tile g
  uint64_t* sdp_read = dp_full + 2;     // [2] S and dP of tile g read out of TMEM
  uint64_t* p_full = sdp_read + 2;      // [NPB] P of tile g in smem buffer g % NPB
  uint64_t* ds_full = p_full + NPB;     // [NPB] dS of tile g in smem
  uint64_t* p_free = ds_full + NPB;     // [NPB] dV MMA of tile g done
  uint64_t* ds_free = p_free + NPB;     // [NPB] dK MMA of tile g done
  uint64_t* acc_full = ds_free + NPB;   // [2]
  uint64_t* acc_empty = acc_full + 2;   // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = (int)warp_id(), lane = (int)lane_id();
  if (threadIdx.x == 0) {
    mbar_init(kv_full, 2);  // two producers: warp 0 (K, Q) and warp PROD2 (V, dO)
    mbar_init(kv_empty, 1);
    for (int s = 0; s < NSL; ++s) {
      mbar_init(&sl_full[s], 1);
      mbar_init(&sl_empty[s], 2);  // released by the S/dP issuer AND the dVᵀ/dKᵀ issuer
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&dp_full[s], 1);
      mbar_init(&sdp_read[s], EWT);
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], 128);
    }
    for (int s = 0; s < NPB; ++s) {
      mbar_init(&p_full[s], EWT);
      mbar_init(&ds_full[s], EWT);
      mbar_init(&p_free[s], 1);
      mbar_init(&ds_free[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_holder;
  pdl_wait();  // everything above touched only this CTA's smem/TMEM
  pdl_trigger();

  if (warp == 0 || warp == R::PROD2) {
    // ---------------- TMA producers: warp 0 loads K and Q, warp PROD2 loads V and dO ----------------
    // (requests issued by one warp are served one at a time; two issuing warps double the
    // per-SM fill rate, tools/tma_rate.py)
    if (elect_one()) {
      const bool second = warp == R::PROD2;
      const CUtensorMap* tmKV = second ? &tmV : &tmK;
      const CUtensorMap* tmR = second ? &tmDO : &tmQ;
      tma_prefetch(tmKV);
      tma_prefetch(tmR);
      uint8_t* const kv_dst = smem + C::OFF_KV + (second ? C::KV_BYTES : 0);
      int it = 0, g = 0;
      for (int wi = blockIdx.x; wi < p.num_items; wi += gridDim.x) {
        const Item m = get_item(p, wi, p.T_n);
        if (m.n == 0) continue;
        const int hh = m.bh % p.H, bb = m.bh / p.H;
        if (it >= 1) mbar_wait(kv_empty, (uint32_t)(it - 1) & 1u);
        mbar_expect_tx(kv_full, C::KV_BYTES);
        tma_load_5d(kv_dst, tmKV, kv_full, 0, m.blk * BKV, 0, hh, bb);
        for (int t = 0; t < m.n; ++t, ++g) {
          const int i = p.idx[m.beg + t];
          const int u = 2 * g + (second ? 1 : 0);  // operand index: Q(g) even, dO(g) odd
          const int s = u % NSL;
          if (!second) trace_ev(p.trace, p.trace_cap, 0, 1, g);
          if (u >= NSL) mbar_wait(&sl_empty[s], ((uint32_t)(u / NSL) + 1u) & 1u);
          if (!second) trace_ev(p.trace, p.trace_cap, 0, 2, g);
          mbar_expect_tx(&sl_full[s], C::Q_BYTES);
          tma_load_5d(smem + C::OFF_SL + s * C::Q_BYTES, tmR, &sl_full[s], 0, i * BQ, 0, hh, bb);
        }
        ++it;
      }
    }
  } else if (warp == 1 || warp == R::ISSUE2) {
    // ---------------- MMA issue: two warps, one per stream ----------------
    // warp 1: S = Q_i K_jᵀ and dP = dO_i V_jᵀ of tile g into TMEM buffer g&1 (free once the
    // elementwise warps have consumed tile g-2);  warp ISSUE2: dVᵀ += dO_iᵀ P (after P is in
    // smem) then dKᵀ += Q_iᵀ dS (after dS).  Warp-collective issue, warp-uniform descriptors.
    constexpr uint32_t idS = idesc_bf16(BQ, BKV, false, false);
    constexpr uint32_t idT = idesc_bf16(HD, BKV, true, true);
    const uint64_t dK = sw128_desc(smem_u32(smem + C::OFF_KV), 16, 1024);
    const uint64_t dV = dK + (uint64_t)(C::KV_BYTES >> 4);
    const uint64_t dSLk0 = sw128_desc(smem_u32(smem + C::OFF_SL), 16, 1024);        // K-major Q / dO slots
    const uint64_t dSLm0 = sw128_desc(smem_u32(smem + C::OFF_SL), BQ * 128, 1024);  // MN-major Q / dO slots
    const uint64_t dPm = sw128_desc(smem_u32(smem + C::OFF_PDS), BQ * 128, 1024);   // MN-major P
    constexpr uint64_t SLOT16 = (uint64_t)(C::Q_BYTES >> 4), PB16 = (uint64_t)(C::PB >> 4);
    const uint64_t dDSm = dPm + PB16;                                                // MN-major dS
    Cursor c;
    cursor_init(c, p, p.T_n);
    if (warp == 1) {
      // S (needs Q) and dP (needs dO) of tile g into TMEM buffer g&1, each as soon as its
      // operand has landed (Q and dO live in separate ring slots)
      for (; c.valid; cursor_next(c, p, p.T_n)) {
        if (c.t == 0) mbar_wait(kv_full, (uint32_t)c.it & 1u);
        const uint32_t b = (uint32_t)(c.g & 1);
        if (c.g >= 2) mbar_wait(&sdp_read[b], (uint32_t)((c.g - 2) >> 1) & 1u);  // buffer b read out
        const int uq = 2 * c.g, ud = uq + 1;
        mbar_wait(&sl_full[uq % NSL], (uint32_t)(uq / NSL) & 1u);
        tc_fence_after();
        trace_ev(p.trace, p.trace_cap, 1, 2, c.g);
        const uint64_t dQ = dSLk0 + (uint64_t)(uq % NSL) * SLOT16, dDO = dSLk0 + (uint64_t)(ud % NSL) * SLOT16;
#ifdef SPA2_MMA_BATCH
        if constexpr (HD == 128) {
          mma_bf16_ss_k8_w<2ull, (uint64_t)(BQ * 128 / 16), 2ull, (uint64_t)(BKV * 128 / 16)>(tbase + C::S_COL + b * 64, dQ, dK,
                                                                                            idS, 0u);
        } else
#endif
        {
#pragma unroll
          for (int ks = 0; ks < HD / 16; ++ks) {
            const uint64_t qo = (uint64_t)(((ks * 16 / 64) * BQ * 128 + (ks * 16 % 64) * 2) >> 4);
            const uint64_t ko = (uint64_t)(((ks * 16 / 64) * BKV * 128 + (ks * 16 % 64) * 2) >> 4);
            mma_bf16_w(tbase + C::S_COL + b * 64, dQ + qo, dK + ko, idS, ks > 0 ? 1u : 0u);
          }
        }
        mma_commit_w(&s_full[b]);
        mma_commit_w(&sl_empty[uq % NSL]);  // S(g) no longer reads Q(g) once complete
        mbar_wait(&sl_full[ud % NSL], (uint32_t)(ud / NSL) & 1u);
        tc_fence_after();
#ifdef SPA2_MMA_BATCH
        if constexpr (HD == 128) {
          mma_bf16_ss_k8_w<2ull, (uint64_t)(BQ * 128 / 16), 2ull, (uint64_t)(BKV * 128 / 16)>(tbase + C::DP_COL + b * 64, dDO,
                                                                                            dV, idS, 0u);
        } else
#endif
        {
#pragma unroll
          for (int ks = 0; ks < HD / 16; ++ks) {
            const uint64_t qo = (uint64_t)(((ks * 16 / 64) * BQ * 128 + (ks * 16 % 64) * 2) >> 4);
            const uint64_t ko = (uint64_t)(((ks * 16 / 64) * BKV * 128 + (ks * 16 % 64) * 2) >> 4);
            mma_bf16_w(tbase + C::DP_COL + b * 64, dDO + qo, dV + ko, idS, ks > 0 ? 1u : 0u);
          }
        }
        mma_commit_w(&dp_full[b]);
        mma_commit_w(&sl_empty[ud % NSL]);  // dP(g) no longer reads dO(g) once complete
        if (c.t == c.n - 1) mma_commit_w(kv_empty);  // K_j / V_j are only read by S and dP
      }
    } else {
      for (; c.valid; cursor_next(c, p, p.T_n)) {
        const int uq = 2 * c.g, ud = uq + 1;
        const uint32_t acc = tbase + C::ACC_COL + (uint32_t)((c.it & 1) * 128);
        const uint64_t dQm = dSLm0 + (uint64_t)(uq % NSL) * SLOT16, dDOm = dSLm0 + (uint64_t)(ud % NSL) * SLOT16;
        const bool first = c.t == 0;
        if (first && c.it >= 2) mbar_wait(&acc_empty[c.it & 1], ((uint32_t)(c.it >> 1) + 1u) & 1u);
        const int pb = c.g % NPB;
        const uint64_t pbo = (uint64_t)pb * 2 * PB16;
        mbar_wait(&p_full[pb], (uint32_t)(c.g / NPB) & 1u);
        // dVᵀ reads dO(g): P(g) only proves S(g) finished, not that dO(g) has landed
        mbar_wait(&sl_full[ud % NSL], (uint32_t)(ud / NSL) & 1u);
        tc_fence_after();
        trace_ev(p.trace, p.trace_cap, 1, 4, c.g);
#ifdef SPA2_MMA_BATCH
        mma_bf16_ss_k8_w<128ull, 512ull, 128ull, 512ull>(acc, dDOm, dPm + pbo, idT, first ? 0u : 1u);
#else
#pragma unroll
        for (int ks = 0; ks < BQ / 16; ++ks)
          mma_bf16_w(acc, dDOm + (uint64_t)(ks * 128), dPm + pbo + (uint64_t)(ks * 128), idT, (!first || ks > 0) ? 1u : 0u);
#endif
        mma_commit_w(&p_free[pb]);
        mma_commit_w(&sl_empty[ud % NSL]);  // dVᵀ(g) was the other reader of dO(g)
        mbar_wait(&ds_full[pb], (uint32_t)(c.g / NPB) & 1u);
        tc_fence_after();
        trace_ev(p.trace, p.trace_cap, 1, 5, c.g);
#ifdef SPA2_MMA_BATCH
        mma_bf16_ss_k8_w<128ull, 512ull, 128ull, 512ull>(acc + 64, dQm, dDSm + pbo, idT, first ? 0u : 1u);
#else
#pragma unroll
        for (int ks = 0; ks < BQ / 16; ++ks)
          mma_bf16_w(acc + 64, dQm + (uint64_t)(ks * 128), dDSm + pbo + (uint64_t)(ks * 128), idT, (!first || ks > 0) ? 1u : 0u);
#endif
        mma_commit_w(&ds_free[pb]);
        mma_commit_w(&sl_empty[uq % NSL]);  // dKᵀ(g) was the other reader of Q(g)
        if (c.t == c.n - 1) mma_commit_w(&acc_full[c.it & 1]);
      }
    }
  } else if (warp < R::EPI0) {
    // ---------------- P / dS warps: EWW/4 warps per TMEM lane quarter, CPT columns each ----
    constexpr int CPT = R::CPT;
    const int q4 = warp & 3;
    const int grp = (warp - 2) >> 2;
    const int row = q4 * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const uint32_t col0 = (uint32_t)(CPT * grp);
    const float sl2 = p.sl2;
    const bool tr = threadIdx.x == 64;
    int g = 0;
    for (int wi = blockIdx.x; wi < p.num_items; wi += gridDim.x) {
      const Item m = get_item(p, wi, p.T_n);
      if (m.n == 0) continue;
      const int64_t rowbase = (int64_t)m.bh * p.N;
      auto load_stats = [&](int t, float& lse2, float& dlt) {
        const int tok = p.idx[m.beg + t] * BQ + row;
        const bool valid = tok < p.N;
        lse2 = valid ? __ldg(p.lse + rowbase + tok) * kLog2e : INFINITY;
        dlt = valid ? __ldg(p.delta + rowbase + tok) : 0.f;
      };
      float lse2, dlt;
      load_stats(0, lse2, dlt);
      for (int t = 0; t < m.n; ++t, ++g) {
        const uint32_t b = (uint32_t)(g & 1);
        float lse2_n = 0.f, dlt_n = 0.f;
        if (t + 1 < m.n) load_stats(t + 1, lse2_n, dlt_n);  // prefetch the next tile's row statistics
        if (tr) trace_ev(p.trace, p.trace_cap, 2, 1, g);
        mbar_wait(&s_full[b], (uint32_t)(g >> 1) & 1u);
        if (tr) trace_ev(p.trace, p.trace_cap, 2, 2, g);
        tc_fence_after();
        uint32_t sr[CPT];
        if constexpr (CPT == 32) tmem_ld32(tbase + lane_off + C::S_COL + b * 64 + col0, sr);
        else tmem_ld16(tbase + lane_off + C::S_COL + b * 64 + col0, sr);
        float pv[CPT];
        uint32_t pk[CPT / 2];
#pragma unroll
        for (int c = 0; c < CPT / 2; ++c) {
          const float2 x = __ffma2_rn(make_float2(__uint_as_float(sr[2 * c]), __uint_as_float(sr[2 * c + 1])),
                                      make_float2(sl2, sl2), make_float2(-lse2, -lse2));
          if (c < kDkvPolyPairs) {  // part of the exponentials on the FMA pipe (exp2_poly2)
            const float2 e = exp2_poly2(x);
            pv[2 * c] = e.x;
            pv[2 * c + 1] = e.y;
          } else {
            pv[2 * c] = ex2(x.x);
            pv[2 * c + 1] = ex2(x.y);
          }
          pk[c] = pack_bf16(pv[2 * c], pv[2 * c + 1]);
        }
        const int pb = g % NPB;
        if (g >= NPB) mbar_wait(&p_free[pb], (uint32_t)((g - NPB) / NPB) & 1u);  // dV of tile g-NPB has read P
        if (tr) trace_ev(p.trace, p.trace_cap, 2, 3, g);
        const uint32_t sP = smem_u32(smem + C::OFF_PDS) + (uint32_t)(pb * 2 * C::PB), sDS = sP + C::PB;
#pragma unroll
        for (int u = 0; u < CPT / 8; ++u) {
          const uint32_t off = sw128_offset((uint32_t)row, col0 / 8 + (uint32_t)u);
          st_shared_v4(sP + off, pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        }
        fence_proxy_async_smem();
        mbar_arrive(&p_full[pb]);
        if (tr) trace_ev(p.trace, p.trace_cap, 2, 5, g);
        mbar_wait(&dp_full[b], (uint32_t)(g >> 1) & 1u);
        tc_fence_after();
        uint32_t dr[CPT];
        if constexpr (CPT == 32) tmem_ld32(tbase + lane_off + C::DP_COL + b * 64 + col0, dr);
        else tmem_ld16(tbase + lane_off + C::DP_COL + b * 64 + col0, dr);
        tc_fence_before();
        mbar_arrive(&sdp_read[b]);  // S(g) and dP(g) are in registers: TMEM buffer b is free
#pragma unroll
        for (int c = 0; c < CPT / 2; ++c) {
          const float2 ds = __fmul2_rn(make_float2(pv[2 * c], pv[2 * c + 1]),
                                       __fadd2_rn(make_float2(__uint_as_float(dr[2 * c]), __uint_as_float(dr[2 * c + 1])),
                                                  make_float2(-dlt, -dlt)));
          pk[c] = pack_bf16(ds.x, ds.y);
        }
        if (g >= NPB) mbar_wait(&ds_free[pb], (uint32_t)((g - NPB) / NPB) & 1u);  // dK of tile g-NPB has read dS
#pragma unroll
        for (int u = 0; u < CPT / 8; ++u) {
          const uint32_t off = sw128_offset((uint32_t)row, col0 / 8 + (uint32_t)u);
          st_shared_v4(sDS + off, pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        }
        fence_proxy_async_smem();
        mbar_arrive(&ds_full[pb]);
        if (tr) trace_ev(p.trace, p.trace_cap, 2, 4, g);
        lse2 = lse2_n;
        dlt = dlt_n;
      }
    }
  } else if (warp < R::PROD2) {
    // ---------------- epilogue warps: TMEM -> registers -> coalesced global stores ----
    const int q4 = warp & 3;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const int dim = (HD == 128) ? q4 * 32 + lane : 16 * q4 + lane;  // M=64 accumulators: lanes 0-15 per quarter
    const bool own = (HD == 128) || lane < 16;
    const bool tr = threadIdx.x == 32 * R::EPI0;
    int it = 0;
    for (int wi = blockIdx.x; wi < p.num_items; wi += gridDim.x) {
      const Item m = get_item(p, wi, p.T_n);
      const int hh = m.bh % p.H, bb = m.bh / p.H;
      __nv_bfloat16* dk = p.out0 + bb * p.o0_sb + hh * p.o0_sh + (int64_t)m.blk * BKV * p.o0_sn + dim;
      __nv_bfloat16* dv = p.out1 + bb * p.o1_sb + hh * p.o1_sh + (int64_t)m.blk * BKV * p.o1_sn + dim;
      const int rows = min(BKV, p.N - m.blk * BKV);
      if (m.n == 0) {
        // no query block keeps this key block: its dK and dV rows are exactly zero
        if (own)
          for (int r = 0; r < rows; ++r) {
            dk[(int64_t)r * p.o0_sn] = __float2bfloat16(0.f);
            dv[(int64_t)r * p.o1_sn] = __float2bfloat16(0.f);
          }
        continue;
      }
      const int st = it & 1;
      if (tr) trace_ev(p.trace, p.trace_cap, 3, 1, it);
      mbar_wait(&acc_full[st], (uint32_t)(it >> 1) & 1u);
      if (tr) trace_ev(p.trace, p.trace_cap, 3, 2, it);
      tc_fence_after();
#pragma unroll 1
      for (int part = 0; part < 4; ++part) {  // dV rows 0-31, 32-63, then dK rows 0-31, 32-63
        uint32_t r32[32];
        tmem_ld32(tbase + lane_off + C::ACC_COL + (uint32_t)(st * 128 + part * 32), r32);
        if (part == 3) {
          tc_fence_before();
          mbar_arrive(&acc_empty[st]);  // both accumulators read: TMEM set reusable
        }
        const bool is_k = part >= 2;
        __nv_bfloat16* dst = (is_k ? dk : dv) + (int64_t)((part & 1) * 32) * (is_k ? p.o0_sn : p.o1_sn);
        const int64_t sn = is_k ? p.o0_sn : p.o1_sn;
        const float mul = is_k ? p.scale : 1.f;
        const int rr = rows - (part & 1) * 32;
        if (own) {
#pragma unroll
          for (int r = 0; r < 32; ++r)
            if (r < rr) dst[(int64_t)r * sn] = __float2bfloat16(__uint_as_float(r32[r]) * mul);
        }
      }
      if (tr) trace_ev(p.trace, p.trace_cap, 3, 3, it);
      ++it;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tbase, 512);
}

// ---------------------------------------------------------------------------------------
// K6 variant 7 (SPA2_DKDV_VARIANT=7, d = 128): KEY-PAIR items.  An item is two adjacent key
// blocks (128 keys) over the UNION of their column lists; a union tile keeps one or both
// halves.  With keys on the TMEM lanes every MMA is M = 128, N = 128:
//   Sᵀ = [K_j; K_j+1] Qᵢᵀ, dPᵀ = [V_j; V_j+1] dOᵢᵀ   (SS, 8 KB of operands per 64 cycles —
//        the N = 64 MMAs of the other variants move 6 KB per 48)
//   dV += Pᵀ dOᵢ, dK += dSᵀ Qᵢ                       (TS: Pᵀ / dSᵀ packed bf16 in TMEM)
// TMEM: Sᵀ→Pᵀ 0 | dPᵀ→dSᵀ 128 | dV 256 | dK 384 (full, single-buffered).  ONE warp issues
// all four MMA streams in the order Sᵀ(g), dPᵀ(g), dV(g), dK(g): tcgen05 MMAs of one thread
// execute in issue order, so Sᵀ(g+1) overwriting Pᵀ(g) and dPᵀ(g+1) overwriting dSᵀ(g) need
// no completion waits.  A half whose key block does not keep the query block gets exact-zero
// P and dS rows (its exponentials are skipped), so results equal the per-block kernels'.
// Warps: 0 TMA (K pair, Q ring), 1 MMA issue, 2-17 elementwise (4 per lane quarter, 32
// query columns each), 18-21 epilogue, 22 TMA (V pair, dO ring).
// ---------------------------------------------------------------------------------------
#ifndef SPA2_DKDV7_NSL
#define SPA2_DKDV7_NSL 4
#endif
#ifndef SPA2_DKDV7_NST
#define SPA2_DKDV7_NST 2
#endif
struct Dkv7Cfg {
  static constexpr int NSL = SPA2_DKDV7_NSL;          // 32 KB Q / dO operand slots
  static constexpr int PAIR = 2 * BKV;                // 128 keys
  static constexpr int KVP_BYTES = PAIR * 128 * 2;    // 32 KB
  static constexpr int Q_BYTES = BQ * 128 * 2;        // 32 KB
  static constexpr int OFF_K = 0, OFF_V = KVP_BYTES, OFF_SL = 2 * KVP_BYTES;
  static constexpr int NST = SPA2_DKDV7_NST;               // LSE/δ slots (tiles in flight)
  static constexpr int OFF_ST = OFF_SL + NSL * Q_BYTES;  // [NST tiles][LSE 128 | δ 128] fp32
  static constexpr int OFF_BAR = OFF_ST + NST * 2 * BQ * 4;
  static constexpr int NUM_BARS = 2 + 2 * NSL + 6 + 4;
  static constexpr int SMEM = OFF_BAR + NUM_BARS * 8 + 16 + kSmemAlignSlack;
  static constexpr uint32_t S_COL = 0, DP_COL = 128, DV_COL = 256, DK_COL = 384;
  static constexpr int EPI0 = 18, PROD2 = 22, THREADS = 32 * 23;
};

// Merge cursor over the column lists of key blocks 2jp and 2jp+1 (both ascending).  The head
// of each list is held in a register and the next entry is loaded as soon as a head is
// consumed, so the global-load latency is paid one union tile ahead, not on the issue path.
struct PairCursor {
  int a, ae, b, be, va, vb;
};
__device__ __forceinline__ void pair_init(PairCursor& pc, const BwdParams& p, int bh, int jp) {
  const int j0 = 2 * jp, j1 = j0 + 1;
  const int64_t base = (int64_t)bh * p.T_n;
  pc.a = p.ptr[base + j0];
  pc.ae = p.ptr[base + j0 + 1];
  if (j1 < p.T_n) {
    pc.b = p.ptr[base + j1];
    pc.be = p.ptr[base + j1 + 1];
  } else {
    pc.b = pc.be = 0;
  }
  pc.va = pc.a < pc.ae ? __ldg(p.idx + pc.a) : 0x7fffffff;
  pc.vb = pc.b < pc.be ? __ldg(p.idx + pc.b) : 0x7fffffff;
}
__device__ __forceinline__ bool pair_done(const PairCursor& pc) { return pc.a >= pc.ae && pc.b >= pc.be; }
// Next query block of the union; flags bit h = key block 2jp+h keeps it.
__device__ __forceinline__ int pair_next(PairCursor& pc, const int32_t* idx, int& flags) {
  const int i = min(pc.va, pc.vb);
  flags = (pc.va == i ? 1 : 0) | (pc.vb == i ? 2 : 0);
  if (pc.va == i) {
    ++pc.a;
    pc.va = pc.a < pc.ae ? __ldg(idx + pc.a) : 0x7fffffff;
  }
  if (pc.vb == i) {
    ++pc.b;
    pc.vb = pc.b < pc.be ? __ldg(idx + pc.b) : 0x7fffffff;
  }
  return i;
}

__global__ void __launch_bounds__(Dkv7Cfg::THREADS, 1)
    k_dkdv7(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKP,
            const __grid_constant__ CUtensorMap tmVP, const __grid_constant__ CUtensorMap tmDO,
            const __grid_constant__ CUtensorMap tmL, const __grid_constant__ CUtensorMap tmD, const BwdParams p) {
  using C = Dkv7Cfg;
  constexpr int NSL = C::NSL;
  constexpr int EWT = 32 * 16;
  constexpr int kPolyPairs = 16 * SPA2_DKDV_POLY_NUM / 64;  // of 16 exponential pairs per thread
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* const smem = smem_align_1k(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* kv_full = bars;            // K/V pair of item `it` landed (two producers)
  uint64_t* kv_empty = kv_full + 1;    // last Sᵀ/dPᵀ of item `it` done
  uint64_t* sl_full = kv_empty + 1;    // [NSL] operand u landed (Q(g): u = 2g, dO(g): u = 2g+1)
  uint64_t* sl_empty = sl_full + NSL;  // [NSL] both MMAs reading operand u done
  uint64_t* s_full = sl_empty + NSL;   // Sᵀ(g) in TMEM
  uint64_t* dp_full = s_full + 1;      // dPᵀ(g) in TMEM
  uint64_t* p_full = dp_full + 1;      // Pᵀ(g) packed over the Sᵀ columns
  uint64_t* ds_full = p_full + 1;      // dSᵀ(g) packed over the dPᵀ columns
  uint64_t* acc_full = ds_full + 1;    // last dV/dK of item `it` done
  uint64_t* acc_empty = acc_full + 1;  // accumulators read out
  constexpr int NST = C::NST;
  uint64_t* st_full = acc_empty + 1;   // [NST] LSE/δ of the query block of tile g in slot g % NST
  uint64_t* st_empty = st_full + 2;    // [NST] elementwise warps done with them
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(st_empty + 2);
  const float* stats = reinterpret_cast<const float*>(smem + C::OFF_ST);

  const int warp = (int)warp_id(), lane = (int)lane_id();
  const int TP = (p.T_n + 1) / 2;
  if (threadIdx.x == 0) {
    mbar_init(kv_full, 2);
    mbar_init(kv_empty, 1);
    for (int s = 0; s < NSL; ++s) {
      mbar_init(&sl_full[s], 1);
      mbar_init(&sl_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(dp_full, 1);
    mbar_init(p_full, EWT);
    mbar_init(ds_full, EWT);
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 128);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&st_full[s], 1);
      mbar_init(&st_empty[s], EWT);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_holder;
  pdl_wait();
  pdl_trigger();

  if (warp == 0 || warp == C::PROD2) {
    // ---------------- TMA producers ----------------
    if (elect_one()) {
      const bool second = warp == C::PROD2;
      const CUtensorMap* tmKV = second ? &tmVP : &tmKP;
      const CUtensorMap* tmR = second ? &tmDO : &tmQ;
      tma_prefetch(tmKV);
      tma_prefetch(tmR);
      if (!second) {
        tma_prefetch(&tmL);
        tma_prefetch(&tmD);
      }
      uint8_t* const kv_dst = smem + (second ? C::OFF_V : C::OFF_K);
      int it = 0, g = 0;
      for (int wi = blockIdx.x; wi < p.num_items; wi += gridDim.x) {
        const int bh = wi / TP, jp = wi % TP, hh = bh % p.H, bb = bh / p.H;
        PairCursor pc;
        pair_init(pc, p, bh, jp);
        if (pair_done(pc)) continue;
        if (it >= 1) mbar_wait(kv_empty, (uint32_t)(it - 1) & 1u);
        mbar_expect_tx(kv_full, C::KVP_BYTES);
        tma_load_5d(kv_dst, tmKV, kv_full, 0, jp * C::PAIR, 0, hh, bb);
        while (!pair_done(pc)) {
          int fl;
          const int i = pair_next(pc, p.idx, fl);
          if (!second) {  // the query block's LSE and δ (128 each; TMA zero-fills past N)
            const int ss = g % NST;
            if (g >= NST) mbar_wait(&st_empty[ss], ((uint32_t)(g / NST) + 1u) & 1u);
            mbar_expect_tx(&st_full[ss], 2 * BQ * 4);
            uint8_t* sdst = smem + C::OFF_ST + ss * 2 * BQ * 4;
            tma_load_2d(sdst, &tmL, &st_full[ss], i * BQ, bh);
            tma_load_2d(sdst + BQ * 4, &tmD, &st_full[ss], i * BQ, bh);
          }
          const int u = 2 * g + (second ? 1 : 0);
          const int s = u % NSL;
          if (!second) trace_ev(p.trace, p.trace_cap, 0, 1, g);
          if (u >= NSL) mbar_wait(&sl_empty[s], ((uint32_t)(u / NSL) + 1u) & 1u);
          if (!second) trace_ev(p.trace, p.trace_cap, 0, 2, g);
          mbar_expect_tx(&sl_full[s], C::Q_BYTES);
          tma_load_5d(smem + C::OFF_SL + s * C::Q_BYTES, tmR, &sl_full[s], 0, i * BQ, 0, hh, bb);
          ++g;
        }
        ++it;
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issue: all four streams, in order ----------------
    constexpr uint32_t idS = idesc_bf16(C::PAIR, BQ, false, false);  // Sᵀ, dPᵀ: M keys, N queries
    constexpr uint32_t idT = idesc_bf16(C::PAIR, 128, false, true);  // dV, dK: B = dO / Q, N (dims) major
    const uint64_t dKP = sw128_desc(smem_u32(smem + C::OFF_K), 16, 1024);
    const uint64_t dVP = sw128_desc(smem_u32(smem + C::OFF_V), 16, 1024);
    const uint64_t dSLk0 = sw128_desc(smem_u32(smem + C::OFF_SL), 16, 1024);        // K-major Q / dO
    const uint64_t dSLm0 = sw128_desc(smem_u32(smem + C::OFF_SL), BQ * 128, 1024);  // N-major Q / dO
    constexpr uint64_t SLOT16 = (uint64_t)(C::Q_BYTES >> 4);
    // Issue order  Sᵀ(0) dPᵀ(0) | dV(0) Sᵀ(1) | dK(0) dPᵀ(1) | dV(1) Sᵀ(2) | dK(1) dPᵀ(2) ...:
    // Sᵀ(g+1) may follow dV(g) (which reads Pᵀ(g) from the Sᵀ columns) and dPᵀ(g+1) may follow
    // dK(g) (dSᵀ(g) lives in the dPᵀ columns) without waits, so the tensor pipe works on tile
    // g+1 while the elementwise warps turn Sᵀ(g)/dPᵀ(g) into Pᵀ/dSᵀ.  Across items the S/dP
    // of the next item's first tile come after the last dK of the previous item.
    int it = 0, g = 0;
    auto issue_s = [&](int gg) {
      const int uq = 2 * gg;
      mbar_wait(&sl_full[uq % NSL], (uint32_t)(uq / NSL) & 1u);
      tc_fence_after();
      trace_ev(p.trace, p.trace_cap, 1, 1, gg);
      mma_bf16_ss_k8_w<2ull, 1024ull, 2ull, 1024ull>(tbase + C::S_COL, dKP, dSLk0 + (uint64_t)(uq % NSL) * SLOT16, idS, 0u);
      mma_commit_w(s_full);
    };
    auto issue_dp = [&](int gg, bool last) {
      const int ud = 2 * gg + 1;
      mbar_wait(&sl_full[ud % NSL], (uint32_t)(ud / NSL) & 1u);
      tc_fence_after();
      mma_bf16_ss_k8_w<2ull, 1024ull, 2ull, 1024ull>(tbase + C::DP_COL, dVP, dSLk0 + (uint64_t)(ud % NSL) * SLOT16, idS, 0u);
      mma_commit_w(dp_full);
      trace_ev(p.trace, p.trace_cap, 1, 2, gg);
      if (last) mma_commit_w(kv_empty);  // the K/V pair is only read by Sᵀ and dPᵀ
    };
    for (int wi = blockIdx.x; wi < p.num_items; wi += gridDim.x) {
      const int bh = wi / TP, jp = wi % TP;
      PairCursor pc;
      pair_init(pc, p, bh, jp);
      if (pair_done(pc)) continue;
      mbar_wait(kv_full, (uint32_t)it & 1u);
      int fl;
      pair_next(pc, p.idx, fl);
      bool last = pair_done(pc);
      issue_s(g);
      issue_dp(g, last);
      if (it >= 1) mbar_wait(acc_empty, (uint32_t)(it - 1) & 1u);
      bool first = true;
      for (;;) {
        const int uq = 2 * g, ud = uq + 1;
        const uint64_t sq = (uint64_t)(uq % NSL) * SLOT16, sd = (uint64_t)(ud % NSL) * SLOT16;
        mbar_wait(p_full, (uint32_t)g & 1u);
        tc_fence_after();
        trace_ev(p.trace, p.trace_cap, 1, 3, g);
        mma_bf16_ts_k8p_w<8u, 32u, 128ull, 512ull>(tbase + C::DV_COL, tbase + C::S_COL, dSLm0 + sd, idT, first ? 0u : 1u);
        mma_commit_w(&sl_empty[ud % NSL]);  // dO(g): dPᵀ(g) and dV(g) both issued by this thread
        const bool more = !last;
        bool next_last = false;
        if (more) {
          pair_next(pc, p.idx, fl);
          next_last = pair_done(pc);
          issue_s(g + 1);
        }
        mbar_wait(ds_full, (uint32_t)g & 1u);
        tc_fence_after();
        trace_ev(p.trace, p.trace_cap, 1, 4, g);
        mma_bf16_ts_k8p_w<8u, 32u, 128ull, 512ull>(tbase + C::DK_COL, tbase + C::DP_COL, dSLm0 + sq, idT, first ? 0u : 1u);
        mma_commit_w(&sl_empty[uq % NSL]);  // Q(g): Sᵀ(g) and dK(g)
        if (!more) {
          mma_commit_w(acc_full);
          ++g;
          break;
        }
        issue_dp(g + 1, next_last);
        first = false;
        last = next_last;
        ++g;
      }
      ++it;
    }
  } else if (warp < C::EPI0) {
    // ---------------- elementwise: Pᵀ = exp2(Sᵀ·c − lse2[q]), dSᵀ = Pᵀ ∘ (dPᵀ − δ[q]) ----------------
    const int q4 = warp & 3;
    const int grp = (warp - 2) >> 2;  // query columns [32·grp, 32·grp + 32)
    const int half = q4 >> 1;         // lanes 0-63: key block 2jp, 64-127: 2jp+1
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const uint32_t col0 = (uint32_t)(32 * grp);
    const float sl2 = p.sl2;
    int g = 0;
    for (int wi = blockIdx.x; wi < p.num_items; wi += gridDim.x) {
      const int bh = wi / TP, jp = wi % TP;
      PairCursor pc;
      pair_init(pc, p, bh, jp);
      if (pair_done(pc)) continue;
      const bool key_ok = jp * C::PAIR + q4 * 32 + lane < p.N;
      while (!pair_done(pc)) {
        int fl;
        const int i = pair_next(pc, p.idx, fl);
        const bool kept = (fl >> half) & 1;  // warp- and lane-quarter-uniform
        const int q0 = i * BQ + (int)col0;
        const float* st = stats + (g % NST) * 2 * BQ + col0;  // this thread's 32 columns: LSE, then δ at +BQ
        if (threadIdx.x == 64) trace_ev(p.trace, p.trace_cap, 2, 1, g);
        mbar_wait(&st_full[g % NST], (uint32_t)(g / NST) & 1u);
        mbar_wait(s_full, (uint32_t)g & 1u);
        if (threadIdx.x == 64) trace_ev(p.trace, p.trace_cap, 2, 2, g);
        tc_fence_after();
        float pv[32];  // fp32 P of this thread's 32 query columns, kept for dS
        uint32_t pk[16];
        if (kept) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {  // two passes of 16 columns keep register pressure down
            float lse2[16];
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {
              const float4 l4 = *reinterpret_cast<const float4*>(st + 16 * h + 4 * c4);
              const float lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
              for (int e = 0; e < 4; ++e)
                lse2[4 * c4 + e] = q0 + 16 * h + 4 * c4 + e < p.N ? lv[e] * kLog2e : INFINITY;
            }
            uint32_t sr[16];
            tmem_ld16(tbase + lane_off + C::S_COL + col0 + 16u * h, sr);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const float2 x = __ffma2_rn(make_float2(__uint_as_float(sr[2 * c]), __uint_as_float(sr[2 * c + 1])),
                                          make_float2(sl2, sl2), make_float2(-lse2[2 * c], -lse2[2 * c + 1]));
              float2 e;
              if (c < kPolyPairs / 2) {
                e = exp2_poly2(x);
              } else {
                e.x = ex2(x.x);
                e.y = ex2(x.y);
              }
              pv[16 * h + 2 * c] = key_ok ? e.x : 0.f;
              pv[16 * h + 2 * c + 1] = key_ok ? e.y : 0.f;
              pk[8 * h + c] = pack_bf16(pv[16 * h + 2 * c], pv[16 * h + 2 * c + 1]);
            }
          }
        } else {
#pragma unroll
          for (int c = 0; c < 16; ++c) pk[c] = 0u;
        }
        // packed Pᵀ goes into the first 16 of this thread's own 32 columns (the MMA reads the
        // K steps at column offsets 0, 8, 32, 40, ...): no other thread's S is overwritten
        tmem_st16(tbase + lane_off + C::S_COL + col0, pk);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(p_full);
        if (threadIdx.x == 64) trace_ev(p.trace, p.trace_cap, 2, 3, g);
        mbar_wait(dp_full, (uint32_t)g & 1u);
        if (threadIdx.x == 64) trace_ev(p.trace, p.trace_cap, 2, 4, g);
        tc_fence_after();
        if (kept) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint32_t dr[16];
            tmem_ld16(tbase + lane_off + C::DP_COL + col0 + 16u * h, dr);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const float2 dl = *reinterpret_cast<const float2*>(st + BQ + 16 * h + 2 * c);
              const float2 ds = __fmul2_rn(make_float2(pv[16 * h + 2 * c], pv[16 * h + 2 * c + 1]),
                                           __fadd2_rn(make_float2(__uint_as_float(dr[2 * c]), __uint_as_float(dr[2 * c + 1])),
                                                      make_float2(-dl.x, -dl.y)));
              pk[8 * h + c] = pack_bf16(ds.x, ds.y);
            }
          }
        }
        mbar_arrive(&st_empty[g % NST]);
        tmem_st16(tbase + lane_off + C::DP_COL + col0, pk);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(ds_full);
        if (threadIdx.x == 64) trace_ev(p.trace, p.trace_cap, 2, 5, g);
        ++g;
      }
    }
  } else if (warp < C::PROD2) {
    // ---------------- epilogue: dV, dK rows (one key per thread) ----------------
    const int q4 = warp & 3;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    int it = 0;
    for (int wi = blockIdx.x; wi < p.num_items; wi += gridDim.x) {
      const int bh = wi / TP, jp = wi % TP, hh = bh % p.H, bb = bh / p.H;
      const int key = jp * C::PAIR + q4 * 32 + lane;
      __nv_bfloat16* dk = p.out0 + bb * p.o0_sb + hh * p.o0_sh + (int64_t)key * p.o0_sn;
      __nv_bfloat16* dv = p.out1 + bb * p.o1_sb + hh * p.o1_sh + (int64_t)key * p.o1_sn;
      PairCursor pc;
      pair_init(pc, p, bh, jp);
      if (pair_done(pc)) {  // no query block keeps either key block: exact zero rows
        if (key < p.N)
          for (int c = 0; c < 128; c += 8) {
            *reinterpret_cast<uint4*>(dk + c) = make_uint4(0, 0, 0, 0);
            *reinterpret_cast<uint4*>(dv + c) = make_uint4(0, 0, 0, 0);
          }
        continue;
      }
      mbar_wait(acc_full, (uint32_t)it & 1u);
      tc_fence_after();
#pragma unroll 1
      for (int part = 0; part < 8; ++part) {  // dV cols 0-127 in 32s, then dK
        const bool is_k = part >= 4;
        const uint32_t c0 = (uint32_t)((part & 3) * 32);
        uint32_t r[32];
        tmem_ld32(tbase + lane_off + (is_k ? C::DK_COL : C::DV_COL) + c0, r);
        if (part == 7) {
          tc_fence_before();
          mbar_arrive(acc_empty);
        }
        const float mul = is_k ? p.scale : 1.f;
        uint32_t pk[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) pk[c] = pack_bf16(__uint_as_float(r[2 * c]) * mul, __uint_as_float(r[2 * c + 1]) * mul);
        if (key < p.N) {
          __nv_bfloat16* dst = (is_k ? dk : dv) + c0;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            *reinterpret_cast<uint4*>(dst + 8 * u) = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        }
      }
      ++it;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tbase, 512);
}

int dkdv_variant() {
  static const int v = [] {
    const char* e = getenv("SPA2_DKDV_VARIANT");
    return e != nullptr ? atoi(e) : 5;
  }();
  return v;
}

int dkdv_ew_warps() {
  static const int v = [] {
    const char* e = getenv("SPA2_DKDV_EW");
    return (e != nullptr && atoi(e) == 8) ? 8 : 16;
  }();
  return v;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

struct FusedDelta {
  const __nv_bfloat16* o;
  int64_t o_sb, o_sh, o_sn;
  const __nv_bfloat16* dout;
  int64_t d_sb, d_sh, d_sn;
  float* delta;
};

struct BwdMaps {
  CUtensorMap q, k, v, dout, out0, out1;
};

// which: 0 = dq kernel (out0 = dq), 1 = dk/dv kernel (out0 = dk, out1 = dv)
template <int HD>
int launch_attn_bwd(int which, const spa2_view& q, const spa2_view& k, const spa2_view& v, const spa2_view& dout,
                    const float* lse, const float* delta, const spa2_view& out0, const spa2_view* out1, int64_t B,
                    int64_t H, int64_t N, const int32_t* ptr, const int32_t* idx, const int32_t* order, float scale,
                    cudaStream_t st, const FusedDelta* fd = nullptr) {
  const int64_t T_m = ceil_div(N, BQ), T_n = ceil_div(N, BKV);
  BwdMaps m;
  int rc;
  if ((rc = make_qkv_map(&m.q, q, B, H, N, HD, BQ))) return rc;
  if ((rc = make_qkv_map(&m.dout, dout, B, H, N, HD, BQ))) return rc;
  if ((rc = make_qkv_map(&m.k, k, B, H, N, HD, BKV))) return rc;
  if ((rc = make_qkv_map(&m.v, v, B, H, N, HD, BKV))) return rc;
  if (which == 0 && (rc = make_qkv_map(&m.out0, out0, B, H, N, HD, BQ))) return rc;

  BwdParams prm{};
  prm.H = (int)H;
  prm.N = (int)N;
  prm.T_m = (int)T_m;
  prm.T_n = (int)T_n;
  prm.lse = lse;
  prm.delta = delta;
  prm.scale = scale;
  prm.sl2 = scale * kLog2e;
  prm.ptr = ptr;
  prm.idx = idx;
  prm.order = order;
  prm.out0 = (__nv_bfloat16*)out0.ptr;
  prm.o0_sb = out0.sb, prm.o0_sh = out0.sh, prm.o0_sn = out0.sn;
  prm.num_items = (int)(B * H * (which == 0 ? T_m : T_n));
  prm.trace = g_trace_buf;
  prm.trace_cap = g_trace_cap;
  if (fd != nullptr) {
    prm.o_in = fd->o;
    prm.oi_sb = fd->o_sb, prm.oi_sh = fd->o_sh, prm.oi_sn = fd->o_sn;
    prm.do_in = fd->dout;
    prm.di_sb = fd->d_sb, prm.di_sh = fd->d_sh, prm.di_sn = fd->d_sn;
    prm.delta_out = fd->delta;
  }
  const unsigned grid = (unsigned)std::min<int64_t>(prm.num_items, num_sms());
  if (which == 0 && dq_variant() == 4) {
    if (dq_ew_warps() == 16) {
      auto kern = k_dq4<HD, 16>;
      SPA2_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Dq4Cfg<HD>::SMEM));
      SPA2_CUDA_TRY(launch_pdl(kern, dim3(grid), dim3(Dq3Roles<16>::THREADS), Dq4Cfg<HD>::SMEM, st, m.q, m.k, m.v, m.dout,
                               prm));
    } else {
      auto kern = k_dq4<HD, 8>;
      SPA2_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Dq4Cfg<HD>::SMEM));
      SPA2_CUDA_TRY(launch_pdl(kern, dim3(grid), dim3(Dq3Roles<8>::THREADS), Dq4Cfg<HD>::SMEM, st, m.q, m.k, m.v, m.dout,
                               prm));
    }
  } else if (which == 0 && dq_variant() == 3) {
    if (dq_ew_warps() == 16) {
      auto kern = k_dq3<HD, 16>;
      SPA2_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Dq3Cfg<HD>::SMEM));
      SPA2_CUDA_TRY(launch_pdl(kern, dim3(grid), dim3(Dq3Roles<16>::THREADS), Dq3Cfg<HD>::SMEM, st, m.q, m.k, m.v, m.dout,
                               prm));
    } else {
      auto kern = k_dq3<HD, 8>;
      SPA2_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Dq3Cfg<HD>::SMEM));
      SPA2_CUDA_TRY(launch_pdl(kern, dim3(grid), dim3(Dq3Roles<8>::THREADS), Dq3Cfg<HD>::SMEM, st, m.q, m.k, m.v, m.dout,
                               prm));
    }
  } else if (which == 0 && dq_variant2()) {
    auto kern = k_dq2<HD>;
    SPA2_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Dq2Cfg<HD>::SMEM));
    kern<<<(unsigned)prm.num_items, kDq2Threads, Dq2Cfg<HD>::SMEM, st>>>(m.q, m.k, m.v, m.dout, m.out0, prm);
  } else if (which == 0) {
    auto kern = k_dq<HD>;
    SPA2_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, DqCfg<HD>::SMEM));
    kern<<<grid, kThreads, DqCfg<HD>::SMEM, st>>>(m.q, m.k, m.v, m.dout, m.out0, prm);
  } else {
    prm.out1 = (__nv_bfloat16*)out1->ptr;
    prm.o1_sb = out1->sb, prm.o1_sh = out1->sh, prm.o1_sn = out1->sn;
    if (HD == 128 && dkdv_variant() == 7 && N % 4 == 0) {  // LSE/δ rows must be 16-byte aligned for TMA
      CUtensorMap kp, vp, tl, td;  // 128-row boxes: one key PAIR per load; LSE/δ tiles
      if ((rc = make_qkv_map(&kp, k, B, H, N, HD, 2 * BKV))) return rc;
      if ((rc = make_qkv_map(&vp, v, B, H, N, HD, 2 * BKV))) return rc;
      if ((rc = make_tma_f32_2d(&tl, lse, (uint64_t)N, (uint64_t)(B * H), (uint64_t)N, BQ, 1))) return rc;
      if ((rc = make_tma_f32_2d(&td, delta, (uint64_t)N, (uint64_t)(B * H), (uint64_t)N, BQ, 1))) return rc;
      prm.num_items = (int)(B * H * ((T_n + 1) / 2));
      const unsigned pgrid = (unsigned)std::min<int64_t>(prm.num_items, num_sms());
      SPA2_CUDA_TRY(cudaFuncSetAttribute(k_dkdv7, cudaFuncAttributeMaxDynamicSharedMemorySize, Dkv7Cfg::SMEM));
      SPA2_CUDA_TRY(launch_pdl(k_dkdv7, dim3(pgrid), dim3(Dkv7Cfg::THREADS), Dkv7Cfg::SMEM, st, m.q, kp, vp, m.dout, tl, td,
                               prm));
    } else if (dkdv_variant() == 6 && dkdv_ew_warps() == 16) {
      using C6 = Dkv5Cfg<HD, 4, 2>;
      auto kern = k_dkdv5<HD, 16, 4, 2>;
      SPA2_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C6::SMEM));
      SPA2_CUDA_TRY(launch_pdl(kern, dim3(grid), dim3(DkvRoles<16>::THREADS), C6::SMEM, st, m.q, m.k, m.v, m.dout,
                               prm));
    } else if (dkdv_variant() >= 5 && dkdv_ew_warps() == 16) {
      auto kern = k_dkdv5<HD, 16>;
      SPA2_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Dkv5Cfg<HD>::SMEM));
      SPA2_CUDA_TRY(launch_pdl(kern, dim3(grid), dim3(DkvRoles<16>::THREADS), Dkv5Cfg<HD>::SMEM, st, m.q, m.k, m.v, m.dout,
                               prm));
    } else if (dkdv_variant() >= 5) {
      auto kern = k_dkdv5<HD, 8>;
      SPA2_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Dkv5Cfg<HD>::SMEM));
      SPA2_CUDA_TRY(launch_pdl(kern, dim3(grid), dim3(DkvRoles<8>::THREADS), Dkv5Cfg<HD>::SMEM, st, m.q, m.k, m.v, m.dout,
                               prm));
    } else if (dkdv_ew_warps() == 16) {
      auto kern = k_dkdv<HD, 16>;
      SPA2_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, DkvCfg<HD>::SMEM));
      kern<<<grid, DkvRoles<16>::THREADS, DkvCfg<HD>::SMEM, st>>>(m.q, m.k, m.v, m.dout, prm);
    } else {
      auto kern = k_dkdv<HD, 8>;
      SPA2_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, DkvCfg<HD>::SMEM));
      kern<<<grid, DkvRoles<8>::THREADS, DkvCfg<HD>::SMEM, st>>>(m.q, m.k, m.v, m.dout, prm);
    }
  }
  SPA2_LAUNCH_CHECK();
  return SPA2_OK;
}

int check_bwd_args(int dtype, int64_t B, int64_t H, int64_t N, int64_t d, int64_t b_q, int64_t b_kv) {
  SPA2_REQUIRE(dtype == SPA2_BF16, SPA2_ERR_UNSUPPORTED, "bwd: only bf16 operands are supported");
  SPA2_REQUIRE(d == 64 || d == 128, SPA2_ERR_UNSUPPORTED, "bwd: head dim %lld not in {64, 128}", (long long)d);
  SPA2_REQUIRE(b_q == BQ && b_kv == BKV, SPA2_ERR_UNSUPPORTED, "bwd: block sizes (%lld, %lld) != (128, 64)",
               (long long)b_q, (long long)b_kv);
  SPA2_REQUIRE(B >= 1 && H >= 1 && N >= 1, SPA2_ERR_VALUE, "bwd: empty problem");
  SPA2_REQUIRE(N < (1ll << 31) && B * H * ceil_div(N, BKV) < (1ll << 31), SPA2_ERR_UNSUPPORTED, "bwd: too large");
  return SPA2_OK;
}

bool al16(const spa2_view& x) {
  return ((uintptr_t)x.ptr % 16 == 0) && x.sb % 8 == 0 && x.sh % 8 == 0 && x.sn % 8 == 0;
}

}  // namespace
}  // namespace spa2

using namespace spa2;
extern "C" int spa2_bwd_delta(spa2_view o, spa2_view dout, float* delta, int dtype, int64_t B, int64_t H,
                              int64_t N, int64_t d, void* stream) {
  int rc;
  if ((rc = check_bwd_args(dtype, B, H, N, d, BQ, BKV))) return rc;
  SPA2_REQUIRE(o.ptr && dout.ptr && delta, SPA2_ERR_VALUE, "bwd_delta: null pointer");
  SPA2_REQUIRE(al16(o) && al16(dout), SPA2_ERR_UNSUPPORTED, "bwd_delta: o/dout must be 16-byte aligned, strides % 8");
  const int64_t rows = B * H * N;
  cudaStream_t st = (cudaStream_t)stream;
  if (d == 128)
    k_delta<128><<<(unsigned)ceil_div(rows, 16), 256, 0, st>>>(o, dout, delta, (int)H, (int)N, rows);
  else
    k_delta<64><<<(unsigned)ceil_div(rows, 32), 256, 0, st>>>(o, dout, delta, (int)H, (int)N, rows);
  SPA2_LAUNCH_CHECK();
  return SPA2_OK;
}

extern "C" int spa2_bwd_dq(spa2_view q, spa2_view k, spa2_view v, spa2_view dout, const float* lse, const float* delta,
                           spa2_view dq, int dtype, int64_t B, int64_t H, int64_t N, int64_t d, int64_t b_q,
                           int64_t b_kv, const int32_t* row_ptr, const int32_t* row_idx, const int32_t* row_order,
                           float scale, void* stream) {
  int rc;
  if ((rc = check_bwd_args(dtype, B, H, N, d, b_q, b_kv))) return rc;
  SPA2_REQUIRE(q.ptr && k.ptr && v.ptr && dout.ptr && lse && delta && dq.ptr && row_ptr && row_idx, SPA2_ERR_VALUE,
               "bwd_dq: null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  if (d == 128)
    return launch_attn_bwd<128>(0, q, k, v, dout, lse, delta, dq, nullptr, B, H, N, row_ptr, row_idx, row_order,
                                scale, st);
  return launch_attn_bwd<64>(0, q, k, v, dout, lse, delta, dq, nullptr, B, H, N, row_ptr, row_idx, row_order, scale,
                             st);
}

extern "C" int spa2_bwd_dq_delta(spa2_view q, spa2_view k, spa2_view v, spa2_view o, spa2_view dout,
                                 const float* lse, float* delta, spa2_view dq, int dtype, int64_t B, int64_t H, int64_t N,
                                 int64_t d, int64_t b_q, int64_t b_kv, const int32_t* row_ptr, const int32_t* row_idx,
                                 const int32_t* row_order, float scale, void* stream) {
  int rc;
  if ((rc = check_bwd_args(dtype, B, H, N, d, b_q, b_kv))) return rc;
  SPA2_REQUIRE(q.ptr && k.ptr && v.ptr && o.ptr && dout.ptr && lse && delta && dq.ptr && row_ptr && row_idx,
               SPA2_ERR_VALUE, "bwd_dq_delta: null pointer");
  SPA2_REQUIRE(((uintptr_t)o.ptr % 16 == 0) && ((uintptr_t)dout.ptr % 16 == 0) && o.sn % 8 == 0 && o.sh % 8 == 0 &&
                   o.sb % 8 == 0 && dout.sn % 8 == 0 && dout.sh % 8 == 0 && dout.sb % 8 == 0,
               SPA2_ERR_VALUE, "bwd_dq_delta: o / dout rows must be 16-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  static const bool no_fuse = [] {
    const char* e = getenv("SPA2_NO_FUSED_DELTA");
    return e != nullptr && e[0] == '1';
  }();
  if ((dq_variant() != 3 && dq_variant() != 4) || no_fuse) {  // other dQ kernels take δ from a separate pass
    if ((rc = spa2_bwd_delta(o, dout, delta, dtype, B, H, N, d, stream))) return rc;
    return spa2_bwd_dq(q, k, v, dout, lse, delta, dq, dtype, B, H, N, d, b_q, b_kv, row_ptr, row_idx, row_order,
                       scale, stream);
  }
  FusedDelta fd{(const __nv_bfloat16*)o.ptr, o.sb, o.sh, o.sn, (const __nv_bfloat16*)dout.ptr, dout.sb, dout.sh,
                dout.sn, delta};
  if (d == 128)
    return launch_attn_bwd<128>(0, q, k, v, dout, lse, delta, dq, nullptr, B, H, N, row_ptr, row_idx, row_order,
                                scale, st, &fd);
  return launch_attn_bwd<64>(0, q, k, v, dout, lse, delta, dq, nullptr, B, H, N, row_ptr, row_idx, row_order, scale,
                             st, &fd);
}

extern "C" int spa2_bwd_dkdv(spa2_view q, spa2_view k, spa2_view v, spa2_view dout, const float* lse,
                             const float* delta, spa2_view dk, spa2_view dv, int dtype, int64_t B, int64_t H,
                             int64_t N, int64_t d, int64_t b_q, int64_t b_kv, const int32_t* col_ptr,
                             const int32_t* col_idx, const int32_t* col_order, float scale, void* stream) {
  int rc;
  if ((rc = check_bwd_args(dtype, B, H, N, d, b_q, b_kv))) return rc;
  SPA2_REQUIRE(q.ptr && k.ptr && v.ptr && dout.ptr && lse && delta && dk.ptr && dv.ptr && col_ptr && col_idx,
               SPA2_ERR_VALUE, "bwd_dkdv: null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  if (d == 128)
    return launch_attn_bwd<128>(1, q, k, v, dout, lse, delta, dk, &dv, B, H, N, col_ptr, col_idx, col_order, scale,
                                st);
  return launch_attn_bwd<64>(1, q, k, v, dout, lse, delta, dk, &dv, B, H, N, col_ptr, col_idx, col_order, scale, st);
}

extern "C" int spa2_bwd(spa2_view q, spa2_view k, spa2_view v, spa2_view o, spa2_view dout, const float* lse,
                        float* delta, spa2_view dq, spa2_view dk, spa2_view dv, int dtype, int64_t B, int64_t H,
                        int64_t N, int64_t d, int64_t b_q, int64_t b_kv, const int32_t* row_ptr,
                        const int32_t* row_idx, const int32_t* row_order, const int32_t* col_ptr,
                        const int32_t* col_idx, const int32_t* col_order, float scale, void* stream) {
  int rc;
  if ((rc = spa2_bwd_dq_delta(q, k, v, o, dout, lse, delta, dq, dtype, B, H, N, d, b_q, b_kv, row_ptr, row_idx,
                              row_order, scale, stream)))
    return rc;
  return spa2_bwd_dkdv(q, k, v, dout, lse, delta, dk, dv, dtype, B, H, N, d, b_q, b_kv, col_ptr, col_idx, col_order,
                       scale, stream);
}
