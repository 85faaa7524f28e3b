// fwd.cu — K4: block-sparse FlashAttention forward on tcgen05 / TMEM / TMA (sm_100a).
//
// Replaces attention.sparse_attention_with_mask (attention.py:73-114): for each query
// block i (128 rows) visit only its kept key blocks j (64 rows) from the row list, with
// an online softmax (running max m, normaliser l, rescaled accumulator) and emit
// O = acc / l (bf16) and LSE = m + ln l (fp32, natural log, attention.py:112-113).
//
// One CTA = one query block; 192 threads, warp-specialised:
//   warp 0      TMA producer: Q once, then K_j into an NS-deep ring
//   warp 6      TMA producer: V_j into an NS-deep ring (TMA requests issued by one warp are
//               served one at a time: two issuing warps double the per-CTA fill rate,
//               tools/tma_rate.py)
//   warp 1      TMEM owner + single-thread tcgen05.mma issuer
//   warps 2..5  softmax: one TMEM lane (= query row) per thread; rescale O in TMEM only
//               when the running max grows by > 8 (log2 units); epilogue via TMA store
// TMEM (256 columns): S double buffer [0,64) [64,128); O accumulator [128, 128+HD).
// P (bf16) either overwrites the first 32 columns of its S buffer and feeds the PV MMA
// as the TMEM A operand (P_TMEM, default) or goes through a swizzled smem tile.
// Two CTAs fit per SM (smem <= 113 KB, TMEM 256 cols) so one CTA's softmax overlaps
// the other's MMAs.  Per kept block: S = Q·Kᵀ (M128 N64 K=HD), O += P·V (M128 N=HD K64).
#include <math.h>
#include <algorithm>
#include <stdlib.h>

#include "common.cuh"
#include "ptx.cuh"
#include "tma_host.h"

namespace spa2 {
namespace {

using namespace ptx;

constexpr int BQ = 128;
constexpr int BKV = 64;
constexpr int kFwdThreads = 224;  // + warp 6: second TMA producer (V)
constexpr float kRescaleThreshold = 8.0f;  // log2 units: P entries stay <= 2^8
#ifndef SPA2_FWD1_POLY_PAIRS
#define SPA2_FWD1_POLY_PAIRS 8  // variant 1: exponential pairs (of 32) by polynomial
#endif
#ifndef SPA2_FWD_EXP_MODE
#define SPA2_FWD_EXP_MODE 0
#endif
constexpr int kExpMode = SPA2_FWD_EXP_MODE;  // 1: f16x2 MUFU exponentials, 0: fp32 MUFU + FMA polynomial

template <int HD, bool P_TMEM>
struct FwdCfg {
  static constexpr int NS = (HD == 128) ? 2 : 4;
  static constexpr int Q_BYTES = BQ * HD * 2;
  static constexpr int KV_BYTES = BKV * HD * 2;
  static constexpr int P_BYTES = P_TMEM ? 0 : BQ * BKV * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_V = OFF_K + NS * KV_BYTES;
  static constexpr int OFF_P = OFF_V + NS * KV_BYTES;
  static constexpr int OFF_BAR = OFF_P + P_BYTES;
  static constexpr int NUM_BARS = 1 + 4 * NS + 2 + 2 + 1 + 1;
  static constexpr int SMEM_USED = OFF_BAR + NUM_BARS * 8 + 16;
  // never let a third CTA share the SM's 512 TMEM columns
  static constexpr int SMEM = SMEM_USED + kSmemAlignSlack < 80 * 1024 ? 80 * 1024 : SMEM_USED + kSmemAlignSlack;
  static constexpr uint32_t O_COL = 128;
};

struct FwdParams {
  int H, N, T_m, T_n;
  const int32_t* row_ptr;
  const int32_t* row_idx;
  const int32_t* row_order;
  float* lse;
  float scale_log2;
  unsigned long long* counter;
  __nv_bfloat16* o_ptr;  // for rows of empty lists only
  int64_t o_sb, o_sh, o_sn;
  unsigned long long* trace;  // diagnostic (spa2_debug_trace), normally null
  int trace_cap;
};

template <int HD, bool P_TMEM>
__global__ void __launch_bounds__(kFwdThreads, 2)
    k_fwd(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
          const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO, const FwdParams p) {
  using C = FwdCfg<HD, P_TMEM>;
  constexpr int NS = C::NS;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* const smem = smem_align_1k(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = k_full + NS;
  uint64_t* v_full = k_empty + NS;
  uint64_t* v_empty = v_full + NS;
  uint64_t* s_full = v_empty + NS;  // [2]
  uint64_t* p_full = s_full + 2;  // [2]: softmax warps may drift by one block, so one per parity
  uint64_t* o_done = p_full + 2;   // one completion per PV MMA group
  uint64_t* o_final = o_done + 1;  // the last PV group (unambiguous single phase)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(o_final + 1);

  const int warp = (int)warp_id(), lane = (int)lane_id();
  const int w = p.row_order ? p.row_order[blockIdx.x] : (int)blockIdx.x;
  const int bh = w / p.T_m, qi = w % p.T_m;
  const int hh = bh % p.H, bb = bh / p.H;
  const int beg = p.row_ptr[w];
  const int n = p.row_ptr[w + 1] - beg;
  const int32_t* list = p.row_idx + beg;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    mbar_init(&s_full[0], 1);
    mbar_init(&s_full[1], 1);
    mbar_init(&p_full[0], 128);
    mbar_init(&p_full[1], 128);
    mbar_init(o_done, 1);
    mbar_init(o_final, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_holder, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_holder;

  if (n == 0) {
    // A query block with no kept key block (rejected by BlockMask; reachable only through
    // the raw C ABI): define O = 0 and LSE = -inf rather than reading garbage.
    if (warp >= 2 && warp < 6) {
      const int row = (warp & 3) * 32 + lane;
      const int tok = qi * BQ + row;
      if (tok < p.N) {
        __nv_bfloat16* o = p.o_ptr + bb * p.o_sb + hh * p.o_sh + (int64_t)tok * p.o_sn;
        for (int c = 0; c < HD; ++c) o[c] = __float2bfloat16(0.f);
        p.lse[(int64_t)bh * p.N + tok] = -INFINITY;
      }
    }
  } else if (warp == 0) {
    // ---------------- TMA producer: Q, K ----------------
    if (elect_one()) {
      tma_prefetch(&tmQ);
      tma_prefetch(&tmK);
      mbar_expect_tx(q_full, C::Q_BYTES);
      tma_load_5d(smem + C::OFF_Q, &tmQ, q_full, 0, qi * BQ, 0, hh, bb);
      for (int t = 0; t < n; ++t) {
        const int s = t % NS;
        const uint32_t ph = (uint32_t)(t / NS) & 1u;
        trace_ev(p.trace, p.trace_cap, 0, 1, t);
        if (t >= NS) mbar_wait(&k_empty[s], ph ^ 1u);
        trace_ev(p.trace, p.trace_cap, 0, 2, t);
        mbar_expect_tx(&k_full[s], C::KV_BYTES);
        tma_load_5d(smem + C::OFF_K + s * C::KV_BYTES, &tmK, &k_full[s], 0, list[t] * BKV, 0, hh, bb);
      }
    }
  } else if (warp == 6) {
    // ---------------- TMA producer: V ----------------
    if (elect_one()) {
      tma_prefetch(&tmV);
      for (int t = 0; t < n; ++t) {
        const int s = t % NS;
        const uint32_t ph = (uint32_t)(t / NS) & 1u;
        if (t >= NS) mbar_wait(&v_empty[s], ph ^ 1u);
        mbar_expect_tx(&v_full[s], C::KV_BYTES);
        tma_load_5d(smem + C::OFF_V + s * C::KV_BYTES, &tmV, &v_full[s], 0, list[t] * BKV, 0, hh, bb);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (whole warp: warp-collective issue) ----------------
    constexpr uint32_t idS = idesc_bf16(BQ, BKV, false, false);
    constexpr uint32_t idO = idesc_bf16(BQ, HD, false, true);
    const uint64_t dQ = sw128_desc(smem_u32(smem + C::OFF_Q), 16, 1024);
    const uint64_t dK0 = sw128_desc(smem_u32(smem + C::OFF_K), 16, 1024);
    const uint64_t dV0 = sw128_desc(smem_u32(smem + C::OFF_V), BKV * 128, 1024);
    const uint64_t dP = sw128_desc(smem_u32(smem + C::OFF_P), 16, 1024);
    constexpr uint64_t KV16 = (uint64_t)(C::KV_BYTES >> 4);
    mbar_wait(q_full, 0);
    for (int t = 0; t <= n; ++t) {
      if (t < n) {
        const uint32_t s_col = tbase + (uint32_t)((t & 1) * 64);
        if (P_TMEM && t >= 2) mbar_wait(o_done, (uint32_t)(t - 2) & 1u);  // P_{t-2} lives in this buffer
        const int s = t % NS;
        mbar_wait(&k_full[s], (uint32_t)(t / NS) & 1u);
        tc_fence_after();
        trace_ev(p.trace, p.trace_cap, 1, 2, t);
        const uint64_t dK = dK0 + (uint64_t)s * KV16;
#pragma unroll
        for (int ks = 0; ks < HD / 16; ++ks) {
          const int k0 = ks * 16;
          mma_bf16_w(s_col, dQ + (uint64_t)(((k0 / 64) * BQ * 128 + (k0 % 64) * 2) >> 4),
                     dK + (uint64_t)(((k0 / 64) * BKV * 128 + (k0 % 64) * 2) >> 4), idS, ks > 0 ? 1u : 0u);
        }
        mma_commit_w(&s_full[t & 1]);
        mma_commit_w(&k_empty[s]);
      }
      if (t >= 1) {
        const int u = t - 1;
        const int s = u % NS;
        mbar_wait(&p_full[u & 1], (uint32_t)(u >> 1) & 1u);
        mbar_wait(&v_full[s], (uint32_t)(u / NS) & 1u);
        tc_fence_after();
        trace_ev(p.trace, p.trace_cap, 1, 4, u);
        const uint64_t dV = dV0 + (uint64_t)s * KV16;
#pragma unroll
        for (int ks = 0; ks < BKV / 16; ++ks) {
          const uint32_t acc = (u > 0 || ks > 0) ? 1u : 0u;
          if constexpr (P_TMEM) {
            mma_bf16_ts_w(tbase + C::O_COL, tbase + (uint32_t)((u & 1) * 64 + ks * 8), dV + (uint64_t)(ks * 128), idO,
                          acc);
          } else {
            mma_bf16_w(tbase + C::O_COL, dP + (uint64_t)(ks * 2), dV + (uint64_t)(ks * 128), idO, acc);
          }
        }
        mma_commit_w(o_done);
        mma_commit_w(&v_empty[s]);
        if (u == n - 1) mma_commit_w(o_final);
      }
    }
  } else if (warp < 6) {
    // ---------------- softmax warps (2..5) ----------------
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const int kv_tail = p.N - (p.T_n - 1) * BKV;  // valid columns of the last key block
    const float sl2 = p.scale_log2;
    float m = -INFINITY, l = 0.f;
    int j_next = list[0];  // key-block index of the next tile, loaded one tile ahead
    for (int t = 0; t < n; ++t) {
      const bool tail = j_next == p.T_n - 1 && kv_tail < BKV;
      if (t + 1 < n) j_next = list[t + 1];
      const uint32_t s_col = tbase + lane_off + (uint32_t)((t & 1) * 64);
      if (threadIdx.x == 64) trace_ev(p.trace, p.trace_cap, 2, 1, t);
      mbar_wait(&s_full[t & 1], (uint32_t)(t >> 1) & 1u);
      if (threadIdx.x == 64) trace_ev(p.trace, p.trace_cap, 2, 2, t);
      tc_fence_after();
      uint32_t r[64];
      tmem_ld64(s_col, r);
      float sv[64];
#pragma unroll
      for (int c = 0; c < 64; ++c) sv[c] = __uint_as_float(r[c]);
      if (tail) {
#pragma unroll
        for (int c = 0; c < 64; ++c)
          if (c >= kv_tail) sv[c] = -INFINITY;
      }
      float mx8[8];  // tree max: short dependency chains
#pragma unroll
      for (int u = 0; u < 8; ++u)
        mx8[u] = fmaxf(fmaxf(fmaxf(sv[8 * u], sv[8 * u + 1]), fmaxf(sv[8 * u + 2], sv[8 * u + 3])),
                       fmaxf(fmaxf(sv[8 * u + 4], sv[8 * u + 5]), fmaxf(sv[8 * u + 6], sv[8 * u + 7])));
      const float smax = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                               fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      const float mx = smax * sl2;
      if (threadIdx.x == 64) trace_ev(p.trace, p.trace_cap, 2, 5, t);
      bool waited = false;
      if (t == 0) {
        m = mx;
      } else if (__any_sync(0xffffffffu, mx > m + kRescaleThreshold)) {
        // warp-uniform: tcgen05.ld/st are warp-collective (.sync.aligned)
        const float m_new = fmaxf(m, mx);
        const float alpha = ex2(m - m_new);
        mbar_wait(o_done, (uint32_t)(t - 1) & 1u);  // PV_{t-1} has landed in O
        waited = true;
        tc_fence_after();
#pragma unroll 1
        for (int c0 = 0; c0 < HD; c0 += 32) {
          uint32_t o[32];
          tmem_ld32(tbase + lane_off + C::O_COL + (uint32_t)c0, o);
#pragma unroll
          for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * alpha);
          tmem_st32(tbase + lane_off + C::O_COL + (uint32_t)c0, o);
        }
        tmem_st_wait();
        l *= alpha;
        m = m_new;
        if (threadIdx.x == 64) trace_ev(p.trace, p.trace_cap, 2, 6, t);
      }
      // P = 2^(S·c − m): packed fp32x2 math, a quarter of the exponentials on the FMA pipe
      // (exp2_poly2) so the MUFU pipe (16/clk/SM) is not the limit of the two softmax CTAs
      uint32_t pk[32];
      float2 lsum = make_float2(0.f, 0.f);
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const float2 x = __ffma2_rn(make_float2(sv[2 * c], sv[2 * c + 1]), make_float2(sl2, sl2), make_float2(-m, -m));
        float2 e;
        if (kExpMode == 1) {  // two exponentials per MUFU op (ex2.approx.f16x2); error below P's bf16 rounding
          e = ex2_f16x2(x);
        } else if (c < SPA2_FWD1_POLY_PAIRS) {  // part of the exponentials on the FMA pipe
          e = exp2_poly2(x);
        } else {
          e.x = ex2(x.x);
          e.y = ex2(x.y);
        }
        lsum = __fadd2_rn(lsum, e);
        pk[c] = pack_bf16(e.x, e.y);
      }
      l += lsum.x + lsum.y;
      if (threadIdx.x == 64) trace_ev(p.trace, p.trace_cap, 2, 7, t);
      if constexpr (P_TMEM) {
        tmem_st32(s_col, pk);
        tmem_st_wait();
      } else {
        if (t >= 1 && !waited) mbar_wait(o_done, (uint32_t)(t - 1) & 1u);  // PV_{t-1} done with sP
        const uint32_t sP = smem_u32(smem + C::OFF_P);
#pragma unroll
        for (int u = 0; u < 8; ++u)
          st_shared_v4(sP + sw128_offset((uint32_t)row, (uint32_t)u), pk[4 * u], pk[4 * u + 1], pk[4 * u + 2],
                       pk[4 * u + 3]);
        fence_proxy_async_smem();
      }
      tc_fence_before();
      mbar_arrive(&p_full[t & 1]);
      if (threadIdx.x == 64) trace_ev(p.trace, p.trace_cap, 2, 4, t);
    }
    // ---------------- epilogue ----------------
    mbar_wait(o_final, 0);
    tc_fence_after();
    const float inv_l = 1.f / l;
    uint8_t* sO = smem + C::OFF_Q;  // Q is dead: every MMA has completed
#pragma unroll 1
    for (int c0 = 0; c0 < HD; c0 += 32) {
      uint32_t o[32];
      tmem_ld32(tbase + lane_off + C::O_COL + (uint32_t)c0, o);
      uint32_t pk[16];
#pragma unroll
      for (int c = 0; c < 16; ++c)
        pk[c] = pack_bf16(__uint_as_float(o[2 * c]) * inv_l, __uint_as_float(o[2 * c + 1]) * inv_l);
      const uint32_t base = smem_u32(sO + (c0 / 64) * BQ * 128);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        st_shared_v4(base + sw128_offset((uint32_t)row, (uint32_t)((c0 % 64) / 8 + u)), pk[4 * u], pk[4 * u + 1],
                     pk[4 * u + 2], pk[4 * u + 3]);
    }
    fence_proxy_async_smem();
    const int tok = qi * BQ + row;
    if (tok < p.N) p.lse[(int64_t)bh * p.N + tok] = (m + log2f(l)) * 0.69314718055994530942f;
    named_bar_sync(1, 128);
    if (threadIdx.x == 64) {
      tma_store_5d(&tmO, sO, 0, qi * BQ, 0, hh, bb);
      tma_store_commit();
      if (p.counter) atomicAdd(p.counter, (unsigned long long)n);
      tma_store_wait_all();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tbase, 256);
}

// ---------------------------------------------------------------------------------------
// K4 (default): the k_fwd pipeline made PERSISTENT — two CTAs per SM, each walking query
// blocks head-major / longest-first (blockIdx.x, +gridDim.x, ...).  Barrier phases run on a
// CTA-global tile counter g, so the producers prefetch the next query block's Q and first
// K/V tiles while the current one finishes, and the softmax warps drain O (direct row
// stores) while the next block's first S is already in flight.  TMEM (256 columns):
// S[g&1] at 0 / 64 (P overwrites its first 32 columns), O at 128.
// Warps: 0 TMA (Q, K ring), 1 MMA (S, PV), 2-5 softmax + epilogue, 6 TMA (V ring).
// ---------------------------------------------------------------------------------------
#ifndef SPA2_FWD3_POLY_PAIRS
// Exponential pairs (of 32 per row and tile) evaluated by exp2_poly2 on the FMA pipe instead of
// MUFU.  0 since the board runs at its power cap in sustained use: 10 was 2 % faster at full
// clocks, 0 is 3 % faster at the cap (MUFU exponentials cost less energy than 6-instruction
// polynomials; tools/ab400.sh).
#define SPA2_FWD3_POLY_PAIRS 0
#endif
template <int HD>
struct Fwd3Cfg {
  static constexpr int NS = (HD == 128) ? 2 : 4;
  static constexpr int Q_BYTES = BQ * HD * 2;
  static constexpr int KV_BYTES = BKV * HD * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_V = OFF_K + NS * KV_BYTES;
  static constexpr int OFF_BAR = OFF_V + NS * KV_BYTES;
  static constexpr int NUM_BARS = 2 + 4 * NS + 2 * 3 + 2;
  static constexpr int SMEM_USED = OFF_BAR + NUM_BARS * 8 + 16;
  static constexpr int SMEM = SMEM_USED + kSmemAlignSlack < 80 * 1024 ? 80 * 1024 : SMEM_USED + kSmemAlignSlack;
  static constexpr uint32_t O_COL = 128;
};

__device__ __forceinline__ void fwd_item(const FwdParams& p, int wi, int& bh, int& qi, int& beg, int& n) {
  const int w = p.row_order ? p.row_order[wi] : wi;
  bh = w / p.T_m;
  qi = w % p.T_m;
  beg = p.row_ptr[w];
  n = p.row_ptr[w + 1] - beg;
}

template <int HD>
__global__ void __launch_bounds__(kFwdThreads, 2)
    k_fwd3(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
           const __grid_constant__ CUtensorMap tmV, const FwdParams p, int num_items) {
  using C = Fwd3Cfg<HD>;
  constexpr int NS = C::NS;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* const smem = smem_align_1k(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars;            // Q of item `it` landed
  uint64_t* q_empty = bars + 1;       // last S MMA of item `it` done
  uint64_t* k_full = bars + 2;        // [NS]
  uint64_t* k_empty = k_full + NS;
  uint64_t* v_full = k_empty + NS;
  uint64_t* v_empty = v_full + NS;
  uint64_t* s_full = v_empty + NS;    // [2] S of tile g in buffer g&1
  uint64_t* p_full = s_full + 2;      // [2] P of tile g written
  uint64_t* o_done = p_full + 2;      // [2] PV of tile g done
  uint64_t* acc_full = o_done + 2;    // last PV of item `it` done
  uint64_t* acc_empty = acc_full + 1;  // O of item `it` read out
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(acc_empty + 1);

  const int warp = (int)warp_id(), lane = (int)lane_id();
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], 128);
      mbar_init(&o_done[b], 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 128);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_holder, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_holder;
  pdl_wait();  // everything above touched only this CTA's smem/TMEM
  pdl_trigger();

  if (warp == 0 || warp == 6) {
    // ---------------- TMA producers: warp 0 Q + K ring, warp 6 V ring ----------------
    if (elect_one()) {
      const bool second = warp == 6;
      if (second) {
        tma_prefetch(&tmV);
      } else {
        tma_prefetch(&tmQ);
        tma_prefetch(&tmK);
      }
      int it = 0, g = 0;
      for (int wi = blockIdx.x; wi < num_items; wi += gridDim.x) {
        int bh, qi, beg, n;
        fwd_item(p, wi, bh, qi, beg, n);
        if (n == 0) continue;
        const int hh = bh % p.H, bb = bh / p.H;
        if (!second) {
          if (it >= 1) mbar_wait(q_empty, (uint32_t)(it - 1) & 1u);
          mbar_expect_tx(q_full, C::Q_BYTES);
          tma_load_5d(smem + C::OFF_Q, &tmQ, q_full, 0, qi * BQ, 0, hh, bb);
        }
        for (int t = 0; t < n; ++t, ++g) {
          const int s = g % NS;
          const uint32_t ph = (uint32_t)(g / NS) & 1u;
          const int j = p.row_idx[beg + t];
          if (!second) {
            trace_ev(p.trace, p.trace_cap, 0, 1, g);
            if (g >= NS) mbar_wait(&k_empty[s], ph ^ 1u);
            trace_ev(p.trace, p.trace_cap, 0, 2, g);
            mbar_expect_tx(&k_full[s], C::KV_BYTES);
            tma_load_5d(smem + C::OFF_K + s * C::KV_BYTES, &tmK, &k_full[s], 0, j * BKV, 0, hh, bb);
          } else {
            if (g >= NS) mbar_wait(&v_empty[s], ph ^ 1u);
            mbar_expect_tx(&v_full[s], C::KV_BYTES);
            tma_load_5d(smem + C::OFF_V + s * C::KV_BYTES, &tmV, &v_full[s], 0, j * BKV, 0, hh, bb);
          }
        }
        ++it;
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (whole warp): S(g), then PV(g-1) ----------------
    constexpr uint32_t idS = idesc_bf16(BQ, BKV, false, false);
    constexpr uint32_t idO = idesc_bf16(BQ, HD, false, true);
    const uint64_t dQ = sw128_desc(smem_u32(smem + C::OFF_Q), 16, 1024);
    const uint64_t dK0 = sw128_desc(smem_u32(smem + C::OFF_K), 16, 1024);
    const uint64_t dV0 = sw128_desc(smem_u32(smem + C::OFF_V), BKV * 128, 1024);
    constexpr uint64_t KV16 = (uint64_t)(C::KV_BYTES >> 4);
    // the pending PV: tile g-1 (its item index, position and whether it ends the item)
    int pv_g = -1, pv_it = 0;
    bool pv_first = false, pv_last = false;
    auto issue_pv = [&]() {
      const int b = pv_g & 1, s = pv_g % NS;
      if (pv_first && pv_it >= 1) mbar_wait(acc_empty, (uint32_t)(pv_it - 1) & 1u);  // O drained
      mbar_wait(&p_full[b], (uint32_t)(pv_g >> 1) & 1u);
      mbar_wait(&v_full[s], (uint32_t)(pv_g / NS) & 1u);
      tc_fence_after();
      trace_ev(p.trace, p.trace_cap, 1, 4, pv_g);
      const uint64_t dV = dV0 + (uint64_t)s * KV16;
#ifdef SPA2_MMA_BATCH
      mma_bf16_ts_k4_w<8u, 128ull>(tbase + C::O_COL, tbase + (uint32_t)(b * 64), dV, idO, pv_first ? 0u : 1u);
#else
#pragma unroll
      for (int ks = 0; ks < BKV / 16; ++ks)
        mma_bf16_ts_w(tbase + C::O_COL, tbase + (uint32_t)(b * 64 + ks * 8), dV + (uint64_t)(ks * 128), idO,
                      (!pv_first || ks > 0) ? 1u : 0u);
#endif
      mma_commit_w(&o_done[b]);
      mma_commit_w(&v_empty[s]);
      if (pv_last) mma_commit_w(acc_full);
    };
    int it = 0, g = 0;
    for (int wi = blockIdx.x; wi < num_items; wi += gridDim.x) {
      int bh, qi, beg, n;
      fwd_item(p, wi, bh, qi, beg, n);
      if (n == 0) continue;
      for (int t = 0; t < n; ++t, ++g) {
        const int b = g & 1, s = g % NS;
        if (t == 0) mbar_wait(q_full, (uint32_t)it & 1u);
        if (g >= 2) mbar_wait(&o_done[b], (uint32_t)((g - 2) >> 1) & 1u);  // P of tile g-2 consumed
        mbar_wait(&k_full[s], (uint32_t)(g / NS) & 1u);
        tc_fence_after();
        trace_ev(p.trace, p.trace_cap, 1, 2, g);
        const uint64_t dK = dK0 + (uint64_t)s * KV16;
#ifdef SPA2_MMA_BATCH
        if constexpr (HD == 128) {
          mma_bf16_ss_k8_w<2ull, (uint64_t)(BQ * 128 / 16), 2ull, (uint64_t)(BKV * 128 / 16)>(tbase + (uint32_t)(b * 64), dQ,
                                                                                            dK, idS, 0u);
        } else
#endif
        {
#pragma unroll
          for (int ks = 0; ks < HD / 16; ++ks) {
            const int k0 = ks * 16;
            mma_bf16_w(tbase + (uint32_t)(b * 64), dQ + (uint64_t)(((k0 / 64) * BQ * 128 + (k0 % 64) * 2) >> 4),
                       dK + (uint64_t)(((k0 / 64) * BKV * 128 + (k0 % 64) * 2) >> 4), idS, ks > 0 ? 1u : 0u);
          }
        }
        mma_commit_w(&s_full[b]);
        mma_commit_w(&k_empty[s]);
        if (t == n - 1) mma_commit_w(q_empty);
        trace_ev(p.trace, p.trace_cap, 1, 3, g);
        if (pv_g >= 0) issue_pv();
        pv_g = g;
        pv_it = it;
        pv_first = t == 0;
        pv_last = t == n - 1;
      }
      ++it;
    }
    if (pv_g >= 0) issue_pv();
  } else {
    // ---------------- softmax warps (2..5) + epilogue ----------------
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const int kv_tail = p.N - (p.T_n - 1) * BKV;
    const float sl2 = p.scale_log2;
    int it = 0, g = 0;
    for (int wi = blockIdx.x; wi < num_items; wi += gridDim.x) {
      int bh, qi, beg, n;
      fwd_item(p, wi, bh, qi, beg, n);
      const int hh = bh % p.H, bb = bh / p.H;
      const int tok = qi * BQ + row;
      __nv_bfloat16* orow = p.o_ptr + bb * p.o_sb + hh * p.o_sh + (int64_t)tok * p.o_sn;
      if (n == 0) {  // reachable only through the raw C ABI: O = 0, LSE = -inf
        if (tok < p.N) {
          for (int c = 0; c < HD; c += 8) *reinterpret_cast<uint4*>(orow + c) = make_uint4(0, 0, 0, 0);
          p.lse[(int64_t)bh * p.N + tok] = -INFINITY;
        }
        continue;
      }
      const int32_t* list = p.row_idx + beg;
      float m = -INFINITY, l = 0.f;
      int j_next = list[0];
      for (int t = 0; t < n; ++t, ++g) {
        const int b = g & 1;
        const bool tail = j_next == p.T_n - 1 && kv_tail < BKV;
        if (t + 1 < n) j_next = list[t + 1];
        const uint32_t s_col = tbase + lane_off + (uint32_t)(b * 64);
        if (threadIdx.x == 64) trace_ev(p.trace, p.trace_cap, 2, 1, g);
        mbar_wait(&s_full[b], (uint32_t)(g >> 1) & 1u);
        if (threadIdx.x == 64) trace_ev(p.trace, p.trace_cap, 2, 2, g);
        tc_fence_after();
        uint32_t r[64];
        tmem_ld64(s_col, r);
        float sv[64];
#pragma unroll
        for (int c = 0; c < 64; ++c) sv[c] = __uint_as_float(r[c]);
        if (tail) {
#pragma unroll
          for (int c = 0; c < 64; ++c)
            if (c >= kv_tail) sv[c] = -INFINITY;
        }
        float mx8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          mx8[u] = fmaxf(fmaxf(fmaxf(sv[8 * u], sv[8 * u + 1]), fmaxf(sv[8 * u + 2], sv[8 * u + 3])),
                         fmaxf(fmaxf(sv[8 * u + 4], sv[8 * u + 5]), fmaxf(sv[8 * u + 6], sv[8 * u + 7])));
        const float mx = sl2 * fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                     fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
        if (t == 0) {
          m = mx;
        } else if (__any_sync(0xffffffffu, mx > m + kRescaleThreshold)) {
          const float m_new = fmaxf(m, mx);
          const float alpha = ex2(m - m_new);
          mbar_wait(&o_done[(g - 1) & 1], (uint32_t)((g - 1) >> 1) & 1u);  // PV(g-1) has landed in O
          tc_fence_after();
#pragma unroll 1
          for (int c0 = 0; c0 < HD; c0 += 32) {
            uint32_t o[32];
            tmem_ld32(tbase + lane_off + C::O_COL + (uint32_t)c0, o);
#pragma unroll
            for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * alpha);
            tmem_st32(tbase + lane_off + C::O_COL + (uint32_t)c0, o);
          }
          tmem_st_wait();
          l *= alpha;
          m = m_new;
        }
        if (threadIdx.x == 64) trace_ev(p.trace, p.trace_cap, 2, 5, g);
        uint32_t pk[32];
        float2 lsum = make_float2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float2 x = __ffma2_rn(make_float2(sv[2 * c], sv[2 * c + 1]), make_float2(sl2, sl2), make_float2(-m, -m));
          float2 e;
          if (c < SPA2_FWD3_POLY_PAIRS) {  // part of the exponentials on the FMA pipe
            e = exp2_poly2(x);
          } else {
            e.x = ex2(x.x);
            e.y = ex2(x.y);
          }
          lsum = __fadd2_rn(lsum, e);
          pk[c] = pack_bf16(e.x, e.y);
        }
        l += lsum.x + lsum.y;
        tmem_st32(s_col, pk);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&p_full[b]);
        if (threadIdx.x == 64) trace_ev(p.trace, p.trace_cap, 2, 4, g);
      }
      // ---------------- epilogue: O / l -> bf16 rows, LSE ----------------
      mbar_wait(acc_full, (uint32_t)it & 1u);
      tc_fence_after();
      const float inv_l = 1.f / l;
#pragma unroll 1
      for (int c0 = 0; c0 < HD; c0 += 32) {
        uint32_t o[32];
        tmem_ld32(tbase + lane_off + C::O_COL + (uint32_t)c0, o);
        if (c0 + 32 == HD) {
          tc_fence_before();
          mbar_arrive(acc_empty);
        }
        uint32_t pk[16];
#pragma unroll
        for (int c = 0; c < 16; ++c)
          pk[c] = pack_bf16(__uint_as_float(o[2 * c]) * inv_l, __uint_as_float(o[2 * c + 1]) * inv_l);
        if (tok < p.N) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            *reinterpret_cast<uint4*>(orow + c0 + 8 * u) = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        }
      }
      if (tok < p.N) p.lse[(int64_t)bh * p.N + tok] = (m + log2f(l)) * 0.69314718055994530942f;
      if (row == 0 && p.counter) atomicAdd(p.counter, (unsigned long long)n);
      ++it;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tbase, 256);
}

// ---------------------------------------------------------------------------------------
// K4 variant 2 (SPA2_FWD_VARIANT=2, experimental; slower than variant 1 at the bench shape
// because each softmax group has a single S buffer): persistent forward, one CTA per SM walking query blocks head-major,
// longest first.  Q_i is staged by TMA and copied into TMEM (tcgen05.cp), so S = Q K_jᵀ is
// a TS-MMA reading only K_j from shared memory.  The kept key blocks of a query block are
// split between TWO softmax groups by tile parity; each group keeps its own running max m,
// normaliser l and accumulator O (TMEM), so the two groups' softmax work overlaps (one
// group exponentiates while the other's S or PV runs) with no cross-group dependency; the
// two partial results are merged once per query block:
//   m = max(m_A, m_B),  O = (2^(m_A−m) O_A + 2^(m_B−m) O_B) / (2^(m_A−m) l_A + 2^(m_B−m) l_B).
// TMEM: Q [0,64) | S_A [64,128) | S_B [128,192) | O_A [256,384) | O_B [384,512).
// Warps: 0 TMA (Q, K ring), 1 / 12 S issue for group A / B, 2-5 softmax group A, 6-9
// group B, 10 TMA (V ring), 11 / 13 PV issue for A / B.  Each group has its own issuing
// warps so the two pipelines never wait on each other; the K/V rings are shared (tiles in
// list order, each slot released by whichever group consumed it).
// ---------------------------------------------------------------------------------------
constexpr int kFwd2Threads = 448;
constexpr int kFwd2Prod2 = 10, kFwd2PV_A = 11, kFwd2S_B = 12, kFwd2PV_B = 13;

template <int HD>
struct Fwd2Cfg {
  static constexpr int NK = 5, NV = 5;
  static constexpr int Q_BYTES = BQ * HD * 2;
  static constexpr int KV_BYTES = BKV * HD * 2;
  static constexpr int OFF_QS = 0;
  static constexpr int OFF_K = Q_BYTES;
  static constexpr int OFF_V = OFF_K + NK * KV_BYTES;
  static constexpr int OFF_RED = OFF_V + NV * KV_BYTES;  // float [2 groups][2 (m, l)][128 rows]
  static constexpr int OFF_BAR = OFF_RED + 4 * BQ * 4;
  static constexpr int NUM_BARS = 4 + 2 * NK + 2 * NV + 2 * 3 + 2;
  static constexpr int SMEM = OFF_BAR + NUM_BARS * 8 + 16 + kSmemAlignSlack;
  static constexpr uint32_t Q_COL = 0, S_COL = 64, O_COL = 256;  // group x: S at S_COL + 64x, O at O_COL + 128x
};

struct Fwd2Item {
  int bh, qi, beg, n;
};
__device__ __forceinline__ Fwd2Item fwd2_item(const FwdParams& p, int wi) {
  const int w = p.row_order ? p.row_order[wi] : wi;
  Fwd2Item m;
  m.bh = w / p.T_m;
  m.qi = w % p.T_m;
  m.beg = p.row_ptr[w];
  m.n = p.row_ptr[w + 1] - m.beg;
  return m;
}

template <int HD>
__global__ void __launch_bounds__(kFwd2Threads, 1)
    k_fwd2(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
           const __grid_constant__ CUtensorMap tmV, const FwdParams p, int num_items) {
  using C = Fwd2Cfg<HD>;
  constexpr int NK = C::NK, NV = C::NV;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* const smem = smem_align_1k(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* qs_full = bars;            // Q of item `it` staged
  uint64_t* qs_free = bars + 1;        // its tcgen05.cp done
  uint64_t* qd_free = bars + 2;        // last S MMA of item `it` done (TMEM Q reusable)
  uint64_t* q_ready = bars + 3;        // Q of item `it` copied into TMEM (by the group-A S warp)
  uint64_t* k_full = bars + 4;         // [NK]
  uint64_t* k_empty = k_full + NK;     // [NK]
  uint64_t* v_full = k_empty + NK;     // [NV]
  uint64_t* v_empty = v_full + NV;     // [NV]
  uint64_t* s_full = v_empty + NV;     // [2 groups] S of the group's current tile landed
  uint64_t* p_full = s_full + 2;       // [2] its P written
  uint64_t* o_done = p_full + 2;       // [2] its PV done (S/P buffer and O consistent)
  uint64_t* acc_full = o_done + 2;     // every PV of item `it` done
  uint64_t* acc_empty = acc_full + 1;  // O_A, O_B of item `it` read
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(acc_empty + 1);
  float* red = reinterpret_cast<float*>(smem + C::OFF_RED);

  const int warp = (int)warp_id(), lane = (int)lane_id();
  if (threadIdx.x == 0) {
    mbar_init(qs_full, 1);
    mbar_init(qs_free, 1);
    mbar_init(qd_free, 2);  // both S warps done with the item
    mbar_init(q_ready, 1);
    for (int i = 0; i < NK; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < NV; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(&s_full[x], 1);
      mbar_init(&p_full[x], 128);
      mbar_init(&o_done[x], 1);
    }
    mbar_init(acc_full, 2);  // both PV warps done with the item
    mbar_init(acc_empty, 256);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_holder;

  if (warp == 0 || warp == kFwd2Prod2) {
    // ---------------- TMA producers: warp 0 Q + K ring, warp 10 V ring ----------------
    if (elect_one()) {
      const bool second = warp == kFwd2Prod2;
      if (!second) {
        tma_prefetch(&tmQ);
        tma_prefetch(&tmK);
      } else {
        tma_prefetch(&tmV);
      }
      int it = 0, g = 0;
      for (int wi = blockIdx.x; wi < num_items; wi += gridDim.x) {
        const Fwd2Item m = fwd2_item(p, wi);
        if (m.n == 0) continue;
        const int hh = m.bh % p.H, bb = m.bh / p.H;
        if (!second) {
          if (it >= 1) mbar_wait(qs_free, (uint32_t)(it - 1) & 1u);
          mbar_expect_tx(qs_full, C::Q_BYTES);
          tma_load_5d(smem + C::OFF_QS, &tmQ, qs_full, 0, m.qi * BQ, 0, hh, bb);
        }
        for (int t = 0; t < m.n; ++t, ++g) {
          const int j = p.row_idx[m.beg + t];
          if (!second) {
            const int s = g % NK;
            if (g >= NK) mbar_wait(&k_empty[s], ((uint32_t)(g / NK) + 1u) & 1u);
            mbar_expect_tx(&k_full[s], C::KV_BYTES);
            tma_load_5d(smem + C::OFF_K + s * C::KV_BYTES, &tmK, &k_full[s], 0, j * BKV, 0, hh, bb);
          } else {
            const int s = g % NV;
            if (g >= NV) mbar_wait(&v_empty[s], ((uint32_t)(g / NV) + 1u) & 1u);
            mbar_expect_tx(&v_full[s], C::KV_BYTES);
            tma_load_5d(smem + C::OFF_V + s * C::KV_BYTES, &tmV, &v_full[s], 0, j * BKV, 0, hh, bb);
          }
        }
        ++it;
      }
    }
  } else if (warp == 1 || warp >= kFwd2PV_A) {
    // ---------------- MMA issue (warp-collective), one S and one PV warp per group ----------------
    constexpr uint32_t idS = idesc_bf16(BQ, BKV, false, false);
    constexpr uint32_t idO = idesc_bf16(BQ, HD, false, true);
    const uint64_t dQS = sw128_desc(smem_u32(smem + C::OFF_QS), 16, 1024);
    const uint64_t dK0 = sw128_desc(smem_u32(smem + C::OFF_K), 16, 1024);
    const uint64_t dV0 = sw128_desc(smem_u32(smem + C::OFF_V), BKV * 128, 1024);
    constexpr uint64_t KV16 = (uint64_t)(C::KV_BYTES >> 4);
    const bool is_s = warp == 1 || warp == kFwd2S_B;
    const int x = (warp == kFwd2S_B || warp == kFwd2PV_B) ? 1 : 0;  // group
    const uint32_t sb = tbase + C::S_COL + (uint32_t)(64 * x);
    int it = 0, g0 = 0;
    for (int wi = blockIdx.x; wi < num_items; wi += gridDim.x) {
      const Fwd2Item m = fwd2_item(p, wi);
      if (m.n == 0) continue;
      if (is_s) {
        if (x == 0) {
          mbar_wait(qs_full, (uint32_t)it & 1u);
          if (it >= 1) mbar_wait(qd_free, (uint32_t)(it - 1) & 1u);
          tc_fence_after();
#pragma unroll
          for (int ks = 0; ks < HD / 16; ++ks)
            tmem_cp_128x256b_w(tbase + C::Q_COL + (uint32_t)(ks * 8),
                               dQS + (uint64_t)((((ks * 16 / 64) * BQ * 128 + (ks * 16 % 64) * 2)) >> 4));
          mma_commit_w(qs_free);
          mma_commit_w(q_ready);
        } else {
          mbar_wait(q_ready, (uint32_t)it & 1u);
        }
      } else if (it >= 1) {
        mbar_wait(acc_empty, (uint32_t)(it - 1) & 1u);
      }
      const int t_first = ((g0 & 1) == x) ? 0 : 1;
      for (int t = t_first; t < m.n; t += 2) {
        const int g = g0 + t;
        if (is_s) {
          if (g >= 2) mbar_wait(&o_done[x], (uint32_t)((g - 2) >> 1) & 1u);  // group's previous P consumed
          const int sk = g % NK;
          mbar_wait(&k_full[sk], (uint32_t)(g / NK) & 1u);
          tc_fence_after();
          trace_ev(p.trace, p.trace_cap, 1, 2, g);
          const uint64_t dK = dK0 + (uint64_t)sk * KV16;
#pragma unroll
          for (int ks = 0; ks < HD / 16; ++ks)
            mma_bf16_ts_w(sb, tbase + C::Q_COL + (uint32_t)(ks * 8),
                          dK + (uint64_t)((((ks * 16 / 64) * BKV * 128 + (ks * 16 % 64) * 2)) >> 4), idS,
                          ks > 0 ? 1u : 0u);
          mma_commit_w(&k_empty[sk]);
          mma_commit_w(&s_full[x]);
        } else {
          mbar_wait(&p_full[x], (uint32_t)(g >> 1) & 1u);
          const int sv = g % NV;
          mbar_wait(&v_full[sv], (uint32_t)(g / NV) & 1u);
          tc_fence_after();
          trace_ev(p.trace, p.trace_cap, 1, 4, g);
          const uint64_t dV = dV0 + (uint64_t)sv * KV16;
#pragma unroll
          for (int ks = 0; ks < BKV / 16; ++ks)
            mma_bf16_ts_w(tbase + C::O_COL + (uint32_t)(128 * x), sb + (uint32_t)(ks * 8), dV + (uint64_t)(ks * 128),
                          idO, (t >= 2 || ks > 0) ? 1u : 0u);  // the group's first tile of the item overwrites O
          mma_commit_w(&v_empty[sv]);
          mma_commit_w(&o_done[x]);
        }
      }
      // item done for this warp's stream (a group with no tile still arrives)
      mma_commit_w(is_s ? qd_free : acc_full);
      g0 += m.n;
      ++it;
    }
  } else {
    // ---------------- softmax groups: warps 2..5 (A), 6..9 (B); one thread per row ----------------
    const int q4 = warp & 3;
    const int x = (warp - 2) >> 2;  // group
    const int row = q4 * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const uint32_t s_col = tbase + lane_off + C::S_COL + (uint32_t)(64 * x);
    const int kv_tail = p.N - (p.T_n - 1) * BKV;
    const float sl2 = p.scale_log2;
    constexpr int OC = HD / 2;  // O columns this thread writes in the epilogue
    int it = 0, g0 = 0;         // g0: global index of the item's first tile
    for (int wi = blockIdx.x; wi < num_items; wi += gridDim.x) {
      const Fwd2Item m = fwd2_item(p, wi);
      const int hh = m.bh % p.H, bb = m.bh / p.H;
      const int tok = m.qi * BQ + row;
      __nv_bfloat16* orow = p.o_ptr + bb * p.o_sb + hh * p.o_sh + (int64_t)tok * p.o_sn + x * OC;
      if (m.n == 0) {
        // a query block with no kept key block (reachable only through the raw C ABI)
        if (tok < p.N) {
          for (int c = 0; c < OC; c += 8) *reinterpret_cast<uint4*>(orow + c) = make_uint4(0, 0, 0, 0);
          if (x == 0) p.lse[(int64_t)m.bh * p.N + tok] = -INFINITY;
        }
        continue;
      }
      float mrow = -INFINITY, l = 0.f;
      // this group's tiles: global index g ≡ x (mod 2)
      const int t_first = ((g0 & 1) == x) ? 0 : 1;
      for (int t = t_first; t < m.n; t += 2) {
        const int g = g0 + t;
        const int j = __ldg(p.row_idx + m.beg + t);
        if (threadIdx.x == 64 || threadIdx.x == 192) trace_ev(p.trace, p.trace_cap, 2, 1, g);
        mbar_wait(&s_full[x], (uint32_t)(g >> 1) & 1u);
        if (threadIdx.x == 64 || threadIdx.x == 192) trace_ev(p.trace, p.trace_cap, 2, 2, g);
        tc_fence_after();
        uint32_t r[64];
        tmem_ld64(s_col, r);
        float sv[64];
#pragma unroll
        for (int c = 0; c < 64; ++c) sv[c] = __uint_as_float(r[c]);
        if (j == p.T_n - 1 && kv_tail < BKV) {
#pragma unroll
          for (int c = 0; c < 64; ++c)
            if (c >= kv_tail) sv[c] = -INFINITY;
        }
        float mx8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          mx8[u] = fmaxf(fmaxf(fmaxf(sv[8 * u], sv[8 * u + 1]), fmaxf(sv[8 * u + 2], sv[8 * u + 3])),
                         fmaxf(fmaxf(sv[8 * u + 4], sv[8 * u + 5]), fmaxf(sv[8 * u + 6], sv[8 * u + 7])));
        const float mx = sl2 * fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                     fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
        if (t < 2) {
          mrow = mx;
        } else if (__any_sync(0xffffffffu, mx > mrow + kRescaleThreshold)) {
          const float m_new = fmaxf(mrow, mx);
          const float alpha = ex2(mrow - m_new);
          mbar_wait(&o_done[x], (uint32_t)((g - 2) >> 1) & 1u);  // the group's previous PV has landed
          tc_fence_after();
#pragma unroll 1
          for (int c0 = 0; c0 < HD; c0 += 32) {
            uint32_t o[32];
            const uint32_t oa = tbase + lane_off + C::O_COL + (uint32_t)(128 * x + c0);
            tmem_ld32(oa, o);
#pragma unroll
            for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * alpha);
            tmem_st32(oa, o);
          }
          tmem_st_wait();
          l *= alpha;
          mrow = m_new;
        }
        uint32_t pk[32];
        float2 lsum = make_float2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float2 xx =
              __ffma2_rn(make_float2(sv[2 * c], sv[2 * c + 1]), make_float2(sl2, sl2), make_float2(-mrow, -mrow));
          float2 e;
          if (c < 8) {  // a quarter of the exponentials on the FMA pipe
            e = exp2_poly2(xx);
          } else {
            e.x = ex2(xx.x);
            e.y = ex2(xx.y);
          }
          lsum = __fadd2_rn(lsum, e);
          pk[c] = pack_bf16(e.x, e.y);
        }
        l += lsum.x + lsum.y;
        tmem_st32(s_col, pk);  // P (bf16) over the first 32 S columns
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&p_full[x]);
        if (threadIdx.x == 64 || threadIdx.x == 192) trace_ev(p.trace, p.trace_cap, 2, 4, g);
      }
      // ---------------- merge the two groups and write O / LSE ----------------
      red[(x * 2 + 0) * BQ + row] = mrow;
      red[(x * 2 + 1) * BQ + row] = l;
      named_bar_sync(1 + q4, 64);
      const float mo = red[((1 - x) * 2 + 0) * BQ + row], lo = red[((1 - x) * 2 + 1) * BQ + row];
      const float ma = x == 0 ? mrow : mo, mb = x == 0 ? mo : mrow;  // group A / B maxima
      const float la = x == 0 ? l : lo, lb = x == 0 ? lo : l;
      const float mm = fmaxf(ma, mb);
      const float fa = ma == -INFINITY ? 0.f : ex2(ma - mm), fb = mb == -INFINITY ? 0.f : ex2(mb - mm);
      const float inv_l = 1.f / (fa * la + fb * lb);
      mbar_wait(acc_full, (uint32_t)it & 1u);
      tc_fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < OC; c0 += 32) {
        const uint32_t oc = tbase + lane_off + C::O_COL + (uint32_t)(x * OC + c0);
        uint32_t oA[32], oB[32];
        tmem_ld32(oc, oA);
        tmem_ld32(oc + 128u, oB);
        if (c0 + 32 == OC) {
          tc_fence_before();
          mbar_arrive(acc_empty);
        }
        uint32_t pk[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const float a0 = fa == 0.f ? 0.f : fa * __uint_as_float(oA[2 * c]);
          const float a1 = fa == 0.f ? 0.f : fa * __uint_as_float(oA[2 * c + 1]);
          const float b0 = fb == 0.f ? 0.f : fb * __uint_as_float(oB[2 * c]);
          const float b1 = fb == 0.f ? 0.f : fb * __uint_as_float(oB[2 * c + 1]);
          pk[c] = pack_bf16((a0 + b0) * inv_l, (a1 + b1) * inv_l);
        }
        if (tok < p.N) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            *reinterpret_cast<uint4*>(orow + c0 + 8 * u) = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        }
      }
      if (x == 0 && tok < p.N) p.lse[(int64_t)m.bh * p.N + tok] = (mm + log2f(fa * la + fb * lb)) * 0.69314718055994530942f;
      if (x == 0 && row == 0 && p.counter) atomicAdd(p.counter, (unsigned long long)m.n);
      named_bar_sync(1 + q4, 64);  // `red` reads done before the next item overwrites it
      g0 += m.n;
      ++it;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tbase, 512);
}

int fwd_variant() {
  static const int v = [] {
    // default 1 (one CTA per query block, 2 per SM, the hardware block scheduler balancing
    // the uneven list lengths): 5 % faster than the persistent variant 3 at full clocks and 2 %
    // at the power cap once both run without trace code (tools/ab.sh, tools/ab400.sh)
    const char* e = getenv("SPA2_FWD_VARIANT");
    return e != nullptr ? atoi(e) : 1;
  }();
  return v;
}

template <int HD, bool P_TMEM>
int launch_fwd(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const CUtensorMap& to,
               const FwdParams& prm, unsigned grid, cudaStream_t st) {
  using C = FwdCfg<HD, P_TMEM>;
  auto kern = k_fwd<HD, P_TMEM>;
  SPA2_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  kern<<<grid, kFwdThreads, C::SMEM, st>>>(tq, tk, tv, to, prm);
  SPA2_LAUNCH_CHECK();
  return SPA2_OK;
}

bool fwd_p_in_smem() {
  static const bool v = [] {
    const char* e = getenv("SPA2_FWD_P_SMEM");
    return e != nullptr && e[0] == '1';
  }();
  return v;
}

}  // namespace

int make_qkv_map(CUtensorMap* m, const spa2_view& v, int64_t B, int64_t H, int64_t N, int64_t d, int rows) {
  const uint64_t dims[5] = {64, (uint64_t)N, (uint64_t)(d / 64), (uint64_t)H, (uint64_t)B};
  const uint64_t strides[4] = {(uint64_t)v.sn * 2, 128, (uint64_t)v.sh * 2, (uint64_t)v.sb * 2};
  const uint32_t box[5] = {64, (uint32_t)rows, (uint32_t)(d / 64), 1, 1};
  return make_tma_bf16_5d(m, v.ptr, dims, strides, box);
}

}  // namespace spa2

using namespace spa2;

extern "C" int spa2_fwd(spa2_view q, spa2_view k, spa2_view v, spa2_view o, float* lse, int dtype, int64_t B,
                        int64_t H, int64_t N, int64_t d, int64_t b_q, int64_t b_kv, const int32_t* row_ptr,
                        const int32_t* row_idx, const int32_t* row_order, float scale,
                        unsigned long long* block_counter, void* stream) {
  SPA2_REQUIRE(dtype == SPA2_BF16, SPA2_ERR_UNSUPPORTED, "fwd: only bf16 operands are supported");
  SPA2_REQUIRE(d == 64 || d == 128, SPA2_ERR_UNSUPPORTED, "fwd: head dim %lld not in {64, 128}", (long long)d);
  SPA2_REQUIRE(b_q == BQ && b_kv == BKV, SPA2_ERR_UNSUPPORTED, "fwd: block sizes (%lld, %lld) != (128, 64)",
               (long long)b_q, (long long)b_kv);
  SPA2_REQUIRE(B >= 1 && H >= 1 && N >= 1, SPA2_ERR_VALUE, "fwd: empty problem");
  SPA2_REQUIRE(N < (1ll << 31) && B * H < (1ll << 31), SPA2_ERR_UNSUPPORTED, "fwd: problem too large");
  SPA2_REQUIRE(q.ptr && k.ptr && v.ptr && o.ptr && lse && row_ptr && row_idx, SPA2_ERR_VALUE, "fwd: null pointer");
  const int64_t T_m = ceil_div(N, BQ), T_n = ceil_div(N, BKV);
  SPA2_REQUIRE(B * H * T_m < (1ll << 31), SPA2_ERR_UNSUPPORTED, "fwd: grid too large");
  CUtensorMap tq, tk, tv, to;
  int rc;
  if ((rc = make_qkv_map(&tq, q, B, H, N, d, BQ))) return rc;
  if ((rc = make_qkv_map(&tk, k, B, H, N, d, BKV))) return rc;
  if ((rc = make_qkv_map(&tv, v, B, H, N, d, BKV))) return rc;
  if ((rc = make_qkv_map(&to, o, B, H, N, d, BQ))) return rc;
  FwdParams prm;
  prm.H = (int)H;
  prm.N = (int)N;
  prm.T_m = (int)T_m;
  prm.T_n = (int)T_n;
  prm.row_ptr = row_ptr;
  prm.row_idx = row_idx;
  prm.row_order = row_order;
  prm.lse = lse;
  prm.scale_log2 = scale * 1.4426950408889634f;
  prm.counter = block_counter;
  prm.o_ptr = (__nv_bfloat16*)o.ptr;
  prm.o_sb = o.sb;
  prm.o_sh = o.sh;
  prm.o_sn = o.sn;
  prm.trace = g_trace_buf;
  prm.trace_cap = g_trace_cap;
  const unsigned grid = (unsigned)(B * H * T_m);
  cudaStream_t st = (cudaStream_t)stream;
  if (fwd_variant() == 3) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned pgrid = (unsigned)std::min<int64_t>(B * H * T_m, 2 * (int64_t)sms);
    if (d == 128) {
      SPA2_CUDA_TRY(cudaFuncSetAttribute(k_fwd3<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, Fwd3Cfg<128>::SMEM));
      SPA2_CUDA_TRY(launch_pdl(k_fwd3<128>, dim3(pgrid), dim3(kFwdThreads), Fwd3Cfg<128>::SMEM, st, tq, tk, tv, prm,
                               (int)(B * H * T_m)));
    } else {
      SPA2_CUDA_TRY(cudaFuncSetAttribute(k_fwd3<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, Fwd3Cfg<64>::SMEM));
      SPA2_CUDA_TRY(launch_pdl(k_fwd3<64>, dim3(pgrid), dim3(kFwdThreads), Fwd3Cfg<64>::SMEM, st, tq, tk, tv, prm,
                               (int)(B * H * T_m)));
    }
    SPA2_LAUNCH_CHECK();
    return SPA2_OK;
  }
  if (fwd_variant() == 2) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned pgrid = (unsigned)std::min<int64_t>(B * H * T_m, sms);
    if (d == 128) {
      SPA2_CUDA_TRY(cudaFuncSetAttribute(k_fwd2<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, Fwd2Cfg<128>::SMEM));
      k_fwd2<128><<<pgrid, kFwd2Threads, Fwd2Cfg<128>::SMEM, st>>>(tq, tk, tv, prm, (int)(B * H * T_m));
    } else {
      SPA2_CUDA_TRY(cudaFuncSetAttribute(k_fwd2<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, Fwd2Cfg<64>::SMEM));
      k_fwd2<64><<<pgrid, kFwd2Threads, Fwd2Cfg<64>::SMEM, st>>>(tq, tk, tv, prm, (int)(B * H * T_m));
    }
    SPA2_LAUNCH_CHECK();
    return SPA2_OK;
  }
  const bool psmem = fwd_p_in_smem();
  if (d == 128) return psmem ? launch_fwd<128, false>(tq, tk, tv, to, prm, grid, st)
                             : launch_fwd<128, true>(tq, tk, tv, to, prm, grid, st);
  return psmem ? launch_fwd<64, false>(tq, tk, tv, to, prm, grid, st) : launch_fwd<64, true>(tq, tk, tv, to, prm, grid, st);
}
