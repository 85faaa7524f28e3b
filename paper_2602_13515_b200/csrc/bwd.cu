// bwd.cu — K5 δ, K7 dQ (query-major) and K6 dK/dV (key-major) on tcgen05 (sm_100a).
//
// Replaces attention.attention_backward (attention.py:128-166).  The reference walks kept
// (i, j) pairs row-major and accumulates into dq/dk/dv; here every accumulator lives in
// TMEM of exactly one CTA, so the result is deterministic and needs no atomics:
//   K5  δ_i = rowsum(dO ∘ O)                                          (attention.py:149)
//       computed inside K7 one query block ahead (k_delta remains for spa2_bwd_delta)
//   K7  k_dq3, work item = query block i, tiles = its row list j:
//         S = Q_i K_jᵀ, dP = dO_i V_jᵀ (TS: Q_i, dO_i copied into TMEM once per item)
//         dS = P ∘ (dP − δ), P = exp2(S·c − LSE·log2e), packed bf16 into TMEM
//         dQ_i += dS K_j (TS)
//   K6  k_dkdv5, work item = key block j, tiles = its column list i:
//         same S, dP (SS), P and dS written bf16 into swizzled smem, then with the
//         accumulators kept TRANSPOSED so every MMA has M = 128:
//         dVᵀ += dO_iᵀ P    (M = d, N = 64, K = 128; both operands MN-major in smem)
//         dKᵀ += Q_iᵀ dS
// Both kernels are persistent (one CTA per SM walking a head-major, longest-first work
// list) and warp-specialised: two TMA producer warps, separate MMA-issuing warps per
// tcgen05 stream, 16 elementwise warps (4 per TMEM lane quarter) and 4 epilogue warps that
// drain one item's accumulators while the next item runs (kernel comments below).
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

#ifdef SPA2_TRACE
__device__ unsigned long long g_spa2_trace[32 * SPA2_TRACE_SLOTS];  // kinds 0-15 dQ, 16-31 dK/dV
#endif

namespace spa2 {
#ifdef SPA2_CTA_TIMES
static __device__ unsigned long long g_spa2_cta[3 * SPA2_CTA_MAX * SPA2_CTA_SLOTS];  // [kind 0 fwd, 1 dQ, 2 dK/dV][cta][slot]
#endif
namespace {

// Share of the elementwise exponentials computed by exp2_poly2 on the FMA pipe instead of
// MUFU: CPT*NUM/64 of each thread's CPT/2 pairs (NUM = 8: a quarter).  Measured in the
// power-capped 400-step regime (tools/ab400.sh): dQ is fastest with none (MUFU exponentials
// cost less energy), dK/dV with a quarter.
#ifndef SPA2_DQ_POLY_NUM
#define SPA2_DQ_POLY_NUM 0
#endif
#ifndef SPA2_DKDV_POLY_NUM
#define SPA2_DKDV_POLY_NUM 4
#endif
#ifndef SPA2_DQ_NK
#define SPA2_DQ_NK 5
#endif
#ifndef SPA2_DQ_NV
#define SPA2_DQ_NV 5
#endif
using namespace ptx;

constexpr int BQ = 128;
constexpr int BKV = 64;
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

// δ of the 32 rows [row0, row0 + 32) of one query block, computed by one warp with k_delta's
// thread layout and arithmetic (HD/8 lanes per row, one 16-byte chunk of O and dO each, the same
// FMA chain and xor-butterfly), so the result is bit-identical to k_delta and row_delta, but every
// load instruction reads whole rows (coalesced) instead of one row per thread, which made the fused
// δ depend on L1 capacity.  Rows past N get δ = 0 in `sd` (if given) and are not stored to `gd`.
template <int HD>
__device__ __forceinline__ void warp_delta_rows(const __nv_bfloat16* o_blk, int64_t o_sn, const __nv_bfloat16* d_blk,
                                                int64_t d_sn, int row0, int rows_valid, float* sd, float* gd) {
  constexpr int TPR = HD / 8;        // lanes per row
  constexpr int RPI = 32 / TPR;      // rows per warp instruction
  const int lane = (int)(threadIdx.x & 31);
  const int part = lane % TPR, sub = lane / TPR;
#pragma unroll 1
  for (int r = 0; r < 32; r += 4 * RPI) {
    uint4 a[4], c[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int row = row0 + r + u * RPI + sub;
      if (row < rows_valid) {
        a[u] = __ldg(reinterpret_cast<const uint4*>(o_blk + (int64_t)row * o_sn + part * 8));
        c[u] = __ldg(reinterpret_cast<const uint4*>(d_blk + (int64_t)row * d_sn + part * 8));
      } else {
        a[u] = make_uint4(0, 0, 0, 0);
        c[u] = make_uint4(0, 0, 0, 0);
      }
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
#pragma unroll
      for (int off = TPR / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      const int row = row0 + r + u * RPI + sub;
      if (part == 0) {
        const bool valid = row < rows_valid;
        if (sd != nullptr) sd[row] = valid ? acc : 0.f;
        if (valid) gd[row] = acc;
      }
    }
  }
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
#ifndef SPA2_DQ_BAR_PAD
#define SPA2_DQ_BAR_PAD 0
#endif
  static constexpr int OFF_BAR = OFF_DLT + 2 * BQ * 4 + SPA2_DQ_BAR_PAD;
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

template <int HD, int EWW, bool HALF = false>
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
  SPA2_CT(1, 0); SPA2_CT(1, 2); SPA2_CTC(1, 4);
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
          if (g >= ns) mbar_wait(&empty[s], ((uint32_t)(g / ns) + 1u) & 1u);
          mbar_expect_tx(&full[s], C::KV_BYTES);
          tma_load_5d(ring + s * C::KV_BYTES, tmKV, &full[s], 0, list_blk(p.idx[m.beg + t]) * BKV, 0, hh, bb);
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
        SPA2_TR(9, c.g);
        if (c.t == 0) {
          SPA2_TR(6, c.g);
          mbar_wait(qs_full, (uint32_t)c.it & 1u);
          if (c.it >= 1) mbar_wait(qd_free, (uint32_t)(c.it - 1) & 1u);
          SPA2_TR(10, c.g);
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
        SPA2_TR(0, c.g);
        if (c.t == c.n - 1) mma_commit_w(qd_free);
      }
    } else {
      // dP = dO V_jᵀ (TS) and dQ += dS K_j (TS), by two warps (dP(g) waits for dQ(g-2) to
      // COMPLETE: it overwrites the TMEM columns dQ(g-2) reads dS from).  One warp issuing
      // both in the order dQ(g-2), dP(g) avoids that wait but measured 12 % slower.
      auto issue_dp = [&](const Cursor& cc) {
        SPA2_TR(7, cc.g);
        const int b = cc.g & 1, sv = cc.g % NV;
        if (cc.g >= 2) mbar_wait(&dq_done[b], (uint32_t)((cc.g - 2) >> 1) & 1u);
        SPA2_TR(13, cc.g);
        mbar_wait(&v_full[sv], (uint32_t)(cc.g / NV) & 1u);
        const uint64_t dV = dV0 + (uint64_t)sv * KV16;
        const uint32_t sb = tbase + C::SDP_COL + (uint32_t)(b * 128) + 64u;
        if (cc.t == 0) mbar_wait(qd_ready, (uint32_t)cc.it & 1u);
        tc_fence_after();
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
        SPA2_TR(1, cc.g);
        mma_commit_w(&v_empty[sv]);
        if (cc.t == cc.n - 1) mma_commit_w(qd_free);
      };
      auto issue_dq = [&](const Cursor& cc) {
        SPA2_TR(8, cc.g);
        const int b = cc.g & 1, sk = cc.g % NK;
        if (cc.t == 0 && cc.it >= 1) mbar_wait(acc_empty, (uint32_t)(cc.it - 1) & 1u);
        mbar_wait(&ds_full[b], (uint32_t)(cc.g >> 1) & 1u);
        SPA2_TR(12, cc.g);
        tc_fence_after();
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
        mma_commit_w(&dq_done[b]);
        SPA2_TR(2, cc.g);
        mma_commit_w(&k_empty[sk]);
        if (cc.t == cc.n - 1) mma_commit_w(acc_full);
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
      int32_t e_next = __ldg(p.idx + m.beg);
      for (int t = 0; t < m.n; ++t, ++g) {
        const int b = g & 1;
        const bool tail = kv_tail < BKV && list_blk(e_next) == p.T_n - 1;
        const bool dropped = HALF && list_row_dropped(e_next, row);  // b_q = 64 masks (warp-uniform)
        if (t + 1 < m.n) e_next = __ldg(p.idx + m.beg + t + 1);
        const uint32_t sb = tbase + lane_off + C::SDP_COL + (uint32_t)(b * 128);
        mbar_wait(&s_full[b], (uint32_t)(g >> 1) & 1u);
        if (warp == 2) SPA2_TR(3, g);
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
        if constexpr (HALF) {
          if (dropped) {
#pragma unroll
            for (int c = 0; c < CPT; ++c) pv[c] = 0.f;
          }
        }
        mbar_wait(&dp_full[b], (uint32_t)(g >> 1) & 1u);
        if (warp == 2) SPA2_TR(4, g);
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
        if (warp == 2) SPA2_TR(5, g);
#ifdef SPA2_TRACE
        {  // trace builds: stamp the LAST elementwise warp to finish dS(g) (kind 11)
          __shared__ uint32_t tr_cnt[2];
          uint32_t old = 0;
          if (lane == 0) old = atomicAdd(&tr_cnt[b], 1u);
          old = __shfl_sync(0xffffffffu, old, 0);
          if ((old % EWW) == EWW - 1) SPA2_TR(11, g);
          tc_fence_before();
          mbar_arrive(&ds_full[b]);
          if ((old % EWW) == EWW - 1) SPA2_TR(14, g);
        }
#else
        tc_fence_before();
        mbar_arrive(&ds_full[b]);
#endif
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
#ifdef SPA2_DQ_ROW_DELTA  // one row per thread (L1-dependent loads)
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
#else
        // this warp's 32 rows of the block, cooperatively (the smem slot was last read at the start
        // of item it-2, which has been drained); rows of an empty list still get their global δ
        const int64_t tok0 = (int64_t)m.blk * BQ;
        warp_delta_rows<HD>(p.o_in + bb * p.oi_sb + hh * p.oi_sh + tok0 * p.oi_sn, p.oi_sn,
                            p.do_in + bb * p.di_sb + hh * p.di_sh + tok0 * p.di_sn, p.di_sn, q4 * 32,
                            (int)(p.N - tok0 < BQ ? p.N - tok0 : BQ), m.n > 0 ? sdelta + (it & 1) * BQ : nullptr,
                            p.delta_out + (int64_t)m.bh * p.N + tok0);
        if (m.n > 0) {
          __syncwarp();
          mbar_arrive(&dlt_full[it & 1]);
        }
#endif
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
  SPA2_CT(1, 1); SPA2_CTC(1, 5);
  if (warp == 1) tmem_dealloc(tbase, 512);
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

#ifndef SPA2_DKDV_NSL
#define SPA2_DKDV_NSL 5  // 32 KB Q / dO operand slots
#endif
#ifndef SPA2_DKDV_NKV
#define SPA2_DKDV_NKV 1  // [K | V] item buffers (2: the next item's K/V load overlaps this item)
#endif
// Operand slots: Q and dO in separate pools, Q(g) in slot g mod NQ and dO(g) in slot
// NQ + g mod (NSL-NQ).  Q is held from S(g) to dKᵀ(g), the tile's last MMA, dO only until dVᵀ(g),
// so Q gets the larger pool; with one interleaved ring (NQ = 0: operand u = 2g + [dO] in slot
// u mod NSL) dO(g+2) reused Q(g)'s slot and waited for dKᵀ(g).  Per-CTA cycles per kept tile
// (tools/ab_cycles.sh): NQ 3 2139-2147, interleaved 2180, NQ 4 2445, NQ 2 slower.
#ifndef SPA2_DKDV_NQ
#define SPA2_DKDV_NQ 3
#endif
#ifndef SPA2_DKDV_NPB
#define SPA2_DKDV_NPB 1  // [P | dS] smem buffers (2 with NSL = 4: 2362 cycles per tile vs 2180)
#endif
template <int HD, int NSL_ = SPA2_DKDV_NSL, int NPB_ = SPA2_DKDV_NPB, int NKV_ = SPA2_DKDV_NKV>
struct Dkv5Cfg {
  static constexpr int NSL = NSL_;  // 32 KB operand slots
  static constexpr int NQ = SPA2_DKDV_NQ, ND = NSL - SPA2_DKDV_NQ;
  static_assert(NQ == 0 || (NQ >= 1 && ND >= 1), "slot pools");
  // slot and use count of operand `which` (0 = Q, 1 = dO) of tile g
  __device__ static __forceinline__ int slot(int g, int which) {
    if constexpr (NQ == 0) return (2 * g + which) % NSL;
    else return which ? NQ + g % (ND > 0 ? ND : 1) : g % (NQ > 0 ? NQ : 1);
  }
  __device__ static __forceinline__ uint32_t use(int g, int which) {
    if constexpr (NQ == 0) return (uint32_t)((2 * g + which) / NSL);
    else return (uint32_t)(which ? g / (ND > 0 ? ND : 1) : g / (NQ > 0 ? NQ : 1));
  }
  static constexpr int NPB = NPB_;  // [P | dS] buffers
  static constexpr int NKV = NKV_;  // [K | V] buffers: item it uses buffer it % NKV
  static constexpr int KV_BYTES = BKV * HD * 2;
  static constexpr int Q_BYTES = BQ * HD * 2;
  static constexpr int PB = BQ * BKV * 2;
  static constexpr int OFF_KV = 0;                         // [NKV][K | V]
  static constexpr int OFF_SL = NKV * 2 * KV_BYTES;        // [NSL] Q / dO operand slots
  static constexpr int OFF_PDS = OFF_SL + NSL * Q_BYTES;   // [NPB][P | dS]
  static constexpr int OFF_BAR = OFF_PDS + NPB * 2 * PB;
  static constexpr int NUM_BARS = 2 * NKV + 2 * NSL + 6 + 4 * NPB + 4;
  static constexpr int SMEM = OFF_BAR + NUM_BARS * 8 + 16 + kSmemAlignSlack;
  static constexpr uint32_t S_COL = 0, DP_COL = 128, ACC_COL = 256;
};

// K6: the Q and dO tiles of a kept tile live in a 5-slot ring of 32 KB operand slots
// (2.5 tiles in flight instead of 2 stages of [Q|dO]).  Each operand has two readers issued by
// different warps (Q: S and dKᵀ, dO: dP and dVᵀ), so its slot is released by two commits, one
// per issuer; the dVᵀ issuer also waits for dO(g) to land (P(g) existing only proves S(g)
// finished).  P and dS share one smem buffer.
template <int HD, int EWW, bool HALF = false, int NSL_ = SPA2_DKDV_NSL, int NPB_ = SPA2_DKDV_NPB>
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
  constexpr int NKV = C::NKV;
  uint64_t* kv_full = bars;             // [NKV] K/V of item `it` landed in buffer it % NKV
  uint64_t* kv_empty = kv_full + NKV;   // [NKV] last S/dP MMA of item `it` done: K/V buffer reusable
  uint64_t* sl_full = kv_empty + NKV;   // [NSL] operand slot holds operand u (Q(g): u=2g, dO(g): u=2g+1)
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
    for (int s = 0; s < NKV; ++s) {
      mbar_init(&kv_full[s], 2);  // two producers: warp 0 (K, Q) and warp PROD2 (V, dO)
      mbar_init(&kv_empty[s], 1);
    }
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
  SPA2_CT(2, 0); SPA2_CT(2, 2); SPA2_CTC(2, 4);
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
        const int kb = it % NKV;
        if (it >= NKV) mbar_wait(&kv_empty[kb], (uint32_t)((it - NKV) / NKV) & 1u);
        mbar_expect_tx(&kv_full[kb], C::KV_BYTES);
        tma_load_5d(kv_dst + kb * 2 * C::KV_BYTES, tmKV, &kv_full[kb], 0, m.blk * BKV, 0, hh, bb);
        for (int t = 0; t < m.n; ++t, ++g) {
          const int i = list_blk(p.idx[m.beg + t]);
          const int s = C::slot(g, second ? 1 : 0);
          const uint32_t use = C::use(g, second ? 1 : 0);
          if (use >= 1) mbar_wait(&sl_empty[s], (use + 1u) & 1u);
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
    const uint64_t dK0 = sw128_desc(smem_u32(smem + C::OFF_KV), 16, 1024);
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
        SPA2_TR(25, c.g);
        if (c.t == 0) {
          SPA2_TR(22, c.g);
          mbar_wait(&kv_full[c.it % NKV], (uint32_t)(c.it / NKV) & 1u);
          SPA2_TR(26, c.g);
        }
        const uint64_t dK = dK0 + (uint64_t)((c.it % NKV) * 2 * C::KV_BYTES >> 4);
        const uint64_t dV = dK + (uint64_t)(C::KV_BYTES >> 4);
        const uint32_t b = (uint32_t)(c.g & 1);
        if (c.g >= 2) mbar_wait(&sdp_read[b], (uint32_t)((c.g - 2) >> 1) & 1u);  // buffer b read out
        const int sq = C::slot(c.g, 0), sd = C::slot(c.g, 1);
        mbar_wait(&sl_full[sq], C::use(c.g, 0) & 1u);
        SPA2_TR(29, c.g);
        tc_fence_after();
        const uint64_t dQ = dSLk0 + (uint64_t)sq * SLOT16, dDO = dSLk0 + (uint64_t)sd * SLOT16;
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
        mma_commit_w(&sl_empty[sq]);  // S(g) no longer reads Q(g) once complete
        mbar_wait(&sl_full[sd], C::use(c.g, 1) & 1u);
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
        SPA2_TR(16, c.g);
        mma_commit_w(&sl_empty[sd]);  // dP(g) no longer reads dO(g) once complete
        if (c.t == c.n - 1) mma_commit_w(&kv_empty[c.it % NKV]);  // K_j / V_j are only read by S and dP
      }
    } else {
      // dVᵀ(g) += dO_iᵀ P (after P is in smem), then dKᵀ(g) += Q_iᵀ dS (after dS).  Issuing
      // dVᵀ(g+1) before dKᵀ(g) measured 3 250 vs 2 152 cycles per tile (P(g+1) waits for dVᵀ(g),
      // dS(g+1) for dKᵀ(g)).
      auto issue_dv = [&](const Cursor& cc) {
        const int sd = C::slot(cc.g, 1);
        const uint32_t acc = tbase + C::ACC_COL + (uint32_t)((cc.it & 1) * 128);
        const uint64_t dDOm = dSLm0 + (uint64_t)sd * SLOT16;
        const bool first = cc.t == 0;
        if (first && cc.it >= 2) mbar_wait(&acc_empty[cc.it & 1], ((uint32_t)(cc.it >> 1) + 1u) & 1u);
        const int pb = cc.g % NPB;
        const uint64_t pbo = (uint64_t)pb * 2 * PB16;
        SPA2_TR(27, cc.g);
        mbar_wait(&p_full[pb], (uint32_t)(cc.g / NPB) & 1u);
        // dVᵀ reads dO(g): P(g) only proves S(g) finished, not that dO(g) has landed
        mbar_wait(&sl_full[sd], C::use(cc.g, 1) & 1u);
        SPA2_TR(17, cc.g);
        tc_fence_after();
#ifdef SPA2_MMA_BATCH
        mma_bf16_ss_k8_w<128ull, 512ull, 128ull, 512ull>(acc, dDOm, dPm + pbo, idT, first ? 0u : 1u);
#else
#pragma unroll
        for (int ks = 0; ks < BQ / 16; ++ks)
          mma_bf16_w(acc, dDOm + (uint64_t)(ks * 128), dPm + pbo + (uint64_t)(ks * 128), idT, (!first || ks > 0) ? 1u : 0u);
#endif
        mma_commit_w(&p_free[pb]);
        mma_commit_w(&sl_empty[sd]);  // dVᵀ(g) was the other reader of dO(g)
      };
      auto issue_dk = [&](const Cursor& cc) {
        const int sq = C::slot(cc.g, 0);
        const uint32_t acc = tbase + C::ACC_COL + (uint32_t)((cc.it & 1) * 128);
        const uint64_t dQm = dSLm0 + (uint64_t)sq * SLOT16;
        const bool first = cc.t == 0;
        const int pb = cc.g % NPB;
        const uint64_t pbo = (uint64_t)pb * 2 * PB16;
        mbar_wait(&ds_full[pb], (uint32_t)(cc.g / NPB) & 1u);
        SPA2_TR(28, cc.g);
        tc_fence_after();
#ifdef SPA2_MMA_BATCH
        mma_bf16_ss_k8_w<128ull, 512ull, 128ull, 512ull>(acc + 64, dQm, dDSm + pbo, idT, first ? 0u : 1u);
#else
#pragma unroll
        for (int ks = 0; ks < BQ / 16; ++ks)
          mma_bf16_w(acc + 64, dQm + (uint64_t)(ks * 128), dDSm + pbo + (uint64_t)(ks * 128), idT, (!first || ks > 0) ? 1u : 0u);
#endif
        mma_commit_w(&ds_free[pb]);
        SPA2_TR(18, cc.g);
        mma_commit_w(&sl_empty[sq]);  // dKᵀ(g) was the other reader of Q(g)
        if (cc.t == cc.n - 1) mma_commit_w(&acc_full[cc.it & 1]);
      };
      for (; c.valid; cursor_next(c, p, p.T_n)) {
        issue_dv(c);
        issue_dk(c);
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
    int g = 0;
    for (int wi = blockIdx.x; wi < p.num_items; wi += gridDim.x) {
      const Item m = get_item(p, wi, p.T_n);
      if (m.n == 0) continue;
      const int64_t rowbase = (int64_t)m.bh * p.N;
      // row statistics of tile t+1 are loaded during tile t from the list entry loaded during tile
      // t-1, and only consumed (scaled, selected) in tile t+1: no load result is waited for in
      // the tile it is issued in (the dependent idx -> LSE load pair stalled these warps)
      auto stats_raw = [&](int32_t e, float& lse_raw, float& dlt_raw, bool& valid) {
        const int tok = list_blk(e) * BQ + row;
        // rows outside the query block's range, or of a half that does not keep the tile (b_q = 64
        // masks), get LSE = +inf: P = 0 and dS = 0
        valid = tok < p.N && !(HALF && list_row_dropped(e, row));
        const int64_t off = rowbase + (valid ? tok : 0);
        lse_raw = __ldg(p.lse + off);
        dlt_raw = __ldg(p.delta + off);
      };
      float lse_r, dlt_r;
      bool vld;
      stats_raw(__ldg(p.idx + m.beg), lse_r, dlt_r, vld);
      int32_t e_nxt = m.n > 1 ? __ldg(p.idx + m.beg + 1) : 0;
      for (int t = 0; t < m.n; ++t, ++g) {
        const uint32_t b = (uint32_t)(g & 1);
        const int32_t e_nn = t + 2 < m.n ? __ldg(p.idx + m.beg + t + 2) : 0;
        float lse_rn = 0.f, dlt_rn = 0.f;
        bool vld_n = false;
        if (t + 1 < m.n) stats_raw(e_nxt, lse_rn, dlt_rn, vld_n);  // prefetch the next tile's row statistics
        const float lse2 = vld ? lse_r * kLog2e : INFINITY;
        const float dlt = vld ? dlt_r : 0.f;
        mbar_wait(&s_full[b], (uint32_t)(g >> 1) & 1u);
        if (warp == 2) SPA2_TR(19, g);
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
#ifdef SPA2_TRACE
        if (warp == 2 && pk[CPT / 2 - 1] != 0xFFFFFFFFu) SPA2_TR(31, g);  // P computed (stamp after the math)
#endif
        if (g >= NPB) mbar_wait(&p_free[pb], (uint32_t)((g - NPB) / NPB) & 1u);  // dV of tile g-NPB has read P
        if (warp == 2) SPA2_TR(23, g);
        const uint32_t sP = smem_u32(smem + C::OFF_PDS) + (uint32_t)(pb * 2 * C::PB), sDS = sP + C::PB;
#pragma unroll
        for (int u = 0; u < CPT / 8; ++u) {
          const uint32_t off = sw128_offset((uint32_t)row, col0 / 8 + (uint32_t)u);
          st_shared_v4(sP + off, pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        }
        fence_proxy_async_smem();
        mbar_arrive(&p_full[pb]);
        mbar_wait(&dp_full[b], (uint32_t)(g >> 1) & 1u);
        if (warp == 2) SPA2_TR(20, g);
#ifdef SPA2_TRACE
        if (warp == 2) SPA2_TR(30, g);  // (dP wait passed; kind 30 = same point, kept for the tool)
#endif
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
        if (warp == 2) SPA2_TR(24, g);
#pragma unroll
        for (int u = 0; u < CPT / 8; ++u) {
          const uint32_t off = sw128_offset((uint32_t)row, col0 / 8 + (uint32_t)u);
          st_shared_v4(sDS + off, pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        }
        fence_proxy_async_smem();
        if (warp == 2) SPA2_TR(21, g);
        mbar_arrive(&ds_full[pb]);
        lse_r = lse_rn;
        dlt_r = dlt_rn;
        vld = vld_n;
        e_nxt = e_nn;
      }
    }
  } else if (warp < R::PROD2) {
    // ---------------- epilogue warps: TMEM -> registers -> coalesced global stores ----
    const int q4 = warp & 3;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const int dim = (HD == 128) ? q4 * 32 + lane : 16 * q4 + lane;  // M=64 accumulators: lanes 0-15 per quarter
    const bool own = (HD == 128) || lane < 16;
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
      mbar_wait(&acc_full[st], (uint32_t)(it >> 1) & 1u);
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
          // (these warps share their SM sub-partitions with the elementwise warps: keep the store
          // loop lean — a running pointer, the full-block case without per-row predicates)
          __nv_bfloat16* q = dst;
          if (rr >= 32) {
#pragma unroll
            for (int r = 0; r < 32; ++r, q += sn) *q = __float2bfloat16(__uint_as_float(r32[r]) * mul);
          } else {
#pragma unroll
            for (int r = 0; r < 32; ++r, q += sn)
              if (r < rr) *q = __float2bfloat16(__uint_as_float(r32[r]) * mul);
          }
        }
      }
      ++it;
    }
  }
  tc_fence_before();
  __syncthreads();
  SPA2_CT(2, 1); SPA2_CTC(2, 5);
  if (warp == 1) tmem_dealloc(tbase, 512);
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
                    cudaStream_t st, const FusedDelta* fd = nullptr, bool half = false) {
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
  if (fd != nullptr) {
    prm.o_in = fd->o;
    prm.oi_sb = fd->o_sb, prm.oi_sh = fd->o_sh, prm.oi_sn = fd->o_sn;
    prm.do_in = fd->dout;
    prm.di_sb = fd->d_sb, prm.di_sh = fd->d_sh, prm.di_sn = fd->d_sn;
    prm.delta_out = fd->delta;
  }
  const unsigned grid = (unsigned)std::min<int64_t>(prm.num_items, num_sms());
  constexpr int EWW = 16;  // elementwise warps (4 per TMEM lane quarter); 8 measured slower
  if (which == 0) {
    auto kern = half ? k_dq3<HD, EWW, true> : k_dq3<HD, EWW, false>;
    SPA2_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Dq3Cfg<HD>::SMEM));
    SPA2_CUDA_TRY(launch_pdl(kern, dim3(grid), dim3(Dq3Roles<EWW>::THREADS), Dq3Cfg<HD>::SMEM, st, m.q, m.k, m.v, m.dout,
                             prm));
  } else {
    prm.out1 = (__nv_bfloat16*)out1->ptr;
    prm.o1_sb = out1->sb, prm.o1_sh = out1->sh, prm.o1_sn = out1->sn;
    auto kern = half ? k_dkdv5<HD, EWW, true> : k_dkdv5<HD, EWW, false>;
    SPA2_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Dkv5Cfg<HD>::SMEM));
    SPA2_CUDA_TRY(launch_pdl(kern, dim3(grid), dim3(DkvRoles<EWW>::THREADS), Dkv5Cfg<HD>::SMEM, st, m.q, m.k, m.v,
                             m.dout, prm));
  }
  SPA2_LAUNCH_CHECK();
  return SPA2_OK;
}

int check_bwd_args(int dtype, int64_t B, int64_t H, int64_t N, int64_t d, int64_t b_q, int64_t b_kv) {
  SPA2_REQUIRE(dtype == SPA2_BF16, SPA2_ERR_UNSUPPORTED, "bwd: only bf16 operands are supported");
  SPA2_REQUIRE(d == 64 || d == 128, SPA2_ERR_UNSUPPORTED, "bwd: head dim %lld not in {64, 128}", (long long)d);
  SPA2_REQUIRE((b_q == BQ || b_q == BQ / 2) && b_kv == BKV, SPA2_ERR_UNSUPPORTED,
               "bwd: block sizes (%lld, %lld) not in {(128, 64), (64, 64)}",
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
                                scale, st, nullptr, b_q != BQ);
  return launch_attn_bwd<64>(0, q, k, v, dout, lse, delta, dq, nullptr, B, H, N, row_ptr, row_idx, row_order, scale,
                             st, nullptr, b_q != BQ);
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
  static const bool no_fuse = [] {  // A/B switch: δ by the separate k_delta pass
    const char* e = getenv("SPA2_NO_FUSED_DELTA");
    return e != nullptr && e[0] == '1';
  }();
  if (no_fuse) {
    if ((rc = spa2_bwd_delta(o, dout, delta, dtype, B, H, N, d, stream))) return rc;
    return spa2_bwd_dq(q, k, v, dout, lse, delta, dq, dtype, B, H, N, d, b_q, b_kv, row_ptr, row_idx, row_order,
                       scale, stream);
  }
  FusedDelta fd{(const __nv_bfloat16*)o.ptr, o.sb, o.sh, o.sn, (const __nv_bfloat16*)dout.ptr, dout.sb, dout.sh,
                dout.sn, delta};
  if (d == 128)
    return launch_attn_bwd<128>(0, q, k, v, dout, lse, delta, dq, nullptr, B, H, N, row_ptr, row_idx, row_order,
                                scale, st, &fd, b_q != BQ);
  return launch_attn_bwd<64>(0, q, k, v, dout, lse, delta, dq, nullptr, B, H, N, row_ptr, row_idx, row_order, scale,
                             st, &fd, b_q != BQ);
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
                                st, nullptr, b_q != BQ);
  return launch_attn_bwd<64>(1, q, k, v, dout, lse, delta, dk, &dv, B, H, N, col_ptr, col_idx, col_order, scale, st,
                             nullptr, b_q != BQ);
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

#ifdef SPA2_TRACE
// diagnostic (trace builds only): copy and clear the pipeline trace of CTA 0
extern "C" int spa2_trace_fetch(unsigned long long* host_dst) {
  SPA2_CUDA_TRY(cudaDeviceSynchronize());
  SPA2_CUDA_TRY(cudaMemcpyFromSymbol(host_dst, g_spa2_trace, sizeof(g_spa2_trace)));
  static unsigned long long zeros[32 * SPA2_TRACE_SLOTS];
  SPA2_CUDA_TRY(cudaMemcpyToSymbol(g_spa2_trace, zeros, sizeof(g_spa2_trace)));
  return SPA2_OK;
}
#endif

#ifdef SPA2_CTA_TIMES
// diagnostic (-DSPA2_CTA_TIMES builds only): copy and clear this unit's per-CTA timings
extern "C" int spa2_cta_fetch_bwd(unsigned long long* host_dst) {
  SPA2_CUDA_TRY(cudaDeviceSynchronize());
  SPA2_CUDA_TRY(cudaMemcpyFromSymbol(host_dst, spa2::g_spa2_cta, sizeof(spa2::g_spa2_cta)));
  static unsigned long long zeros[3 * SPA2_CTA_MAX * SPA2_CTA_SLOTS];
  SPA2_CUDA_TRY(cudaMemcpyToSymbol(spa2::g_spa2_cta, zeros, sizeof(spa2::g_spa2_cta)));
  return SPA2_OK;
}
#endif
