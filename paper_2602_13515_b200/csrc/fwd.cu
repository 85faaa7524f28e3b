// fwd.cu — K4: block-sparse FlashAttention forward on tcgen05 / TMEM / TMA (sm_100a).
//
// Replaces attention.sparse_attention_with_mask (attention.py:73-114): for each query
// block i (128 rows) visit only its kept key blocks j (64 rows) from the row list, with
// an online softmax (running max m, normaliser l, rescaled accumulator) and emit
// O = acc / l (bf16) and LSE = m + ln l (fp32, natural log, attention.py:112-113).
//
// One CTA = one query block, launched longest-list-first so the hardware block scheduler
// balances the uneven list lengths; 224 threads, warp-specialised:
//   warp 0      TMA producer: Q once, then K_j into an NS-deep ring
//   warp 6      TMA producer: V_j into an NS-deep ring (TMA requests issued by one warp are
//               served one at a time: two issuing warps double the per-CTA fill rate)
//   warp 1      TMEM owner + tcgen05.mma issuer (warp-collective issue, one elect per K loop)
//   warps 2..5  softmax: one TMEM lane (= query row) per thread; rescale O in TMEM only
//               when the running max grows by > 8 (log2 units); epilogue via TMA store
// TMEM (256 columns): S double buffer [0,64) [64,128); O accumulator [128, 128+HD).
// P (bf16) overwrites the first 32 columns of its S buffer and feeds the PV MMA as the TMEM
// A operand.  Two CTAs fit per SM (smem <= 113 KB, TMEM 256 cols) so one CTA's softmax
// overlaps the other's MMAs.  Per kept block: S = Q·Kᵀ (M128 N64 K=HD, SS),
// O += P·V (M128 N=HD K64, TS).
#include <math.h>
#include <algorithm>
#include <stdlib.h>

#include "common.cuh"
#include "ptx.cuh"
#include "tma_host.h"

namespace spa2 {
#ifdef SPA2_CTA_TIMES
static __device__ unsigned long long g_spa2_cta[3 * SPA2_CTA_MAX * SPA2_CTA_SLOTS];  // [kind 0 fwd, 1 dQ, 2 dK/dV][cta][slot]
#endif
namespace {

using namespace ptx;

constexpr int BQ = 128;
constexpr int BKV = 64;
constexpr int kFwdThreads = 224;  // + warp 6: second TMA producer (V)
#ifndef SPA2_FWD_RESCALE
#define SPA2_FWD_RESCALE 8.0f
#endif
constexpr float kRescaleThreshold = SPA2_FWD_RESCALE;  // log2 units: P entries stay <= 2^8
#ifndef SPA2_FWD1_POLY_PAIRS
#define SPA2_FWD1_POLY_PAIRS 4  // exponential pairs (of 32 per row and tile) by FMA polynomial (forward span: 0: 295.8, 4: 291.9, 8: 296.4, 12: 295.7 us)
#endif

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
};

template <int HD, bool P_TMEM, bool HALF>
__global__ void __launch_bounds__(kFwdThreads, 2)
    k_fwd(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
          const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO, const FwdParams p) {
  using C = FwdCfg<HD, P_TMEM>;
  constexpr int NS = C::NS;
  SPA2_CT(0, 3);
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
  SPA2_CT(0, 0); SPA2_CT(0, 2);
  tc_fence_after();
  const uint32_t tbase = *tmem_holder;
  // programmatic dependent launch: the setup above overlapped the list kernel's tail; the block
  // lists (and q/k/v) are read only after it completes
  pdl_wait();
  pdl_trigger();
  const int w = p.row_order ? p.row_order[blockIdx.x] : (int)blockIdx.x;
  const int bh = w / p.T_m, qi = w % p.T_m;
  const int hh = bh % p.H, bb = bh / p.H;
  const int beg = p.row_ptr[w];
  const int n = p.row_ptr[w + 1] - beg;
  const int32_t* list = p.row_idx + beg;

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
        if (t >= NS) mbar_wait(&k_empty[s], ph ^ 1u);
        mbar_expect_tx(&k_full[s], C::KV_BYTES);
        tma_load_5d(smem + C::OFF_K + s * C::KV_BYTES, &tmK, &k_full[s], 0, list_blk(list[t]) * BKV, 0, hh, bb);
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
        tma_load_5d(smem + C::OFF_V + s * C::KV_BYTES, &tmV, &v_full[s], 0, list_blk(list[t]) * BKV, 0, hh, bb);
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
        if (u == n - 1) {
          mma_commit_w(o_final);
          SPA2_CTL(0, 7);
        }
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
    int32_t e_next = list[0];  // list entry of the next tile, loaded one tile ahead
    for (int t = 0; t < n; ++t) {
      const bool tail = list_blk(e_next) == p.T_n - 1 && kv_tail < BKV;
      // b_q = 64 masks (HALF instantiation only): this row's half of the query block does not
      // keep the tile (warp-uniform)
      const bool dropped = HALF && list_row_dropped(e_next, row);
      if (t + 1 < n) e_next = list[t + 1];
      const uint32_t s_col = tbase + lane_off + (uint32_t)((t & 1) * 64);
      mbar_wait(&s_full[t & 1], (uint32_t)(t >> 1) & 1u);
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
      if constexpr (HALF) {
        if (dropped) {
#pragma unroll
          for (int c = 0; c < 64; ++c) sv[c] = -INFINITY;
        }
      }
      float mx8[8];  // tree max: short dependency chains
#pragma unroll
      for (int u = 0; u < 8; ++u)
        mx8[u] = fmaxf(fmaxf(fmaxf(sv[8 * u], sv[8 * u + 1]), fmaxf(sv[8 * u + 2], sv[8 * u + 3])),
                       fmaxf(fmaxf(sv[8 * u + 4], sv[8 * u + 5]), fmaxf(sv[8 * u + 6], sv[8 * u + 7])));
      const float smax = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                               fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      const float mx = smax * sl2;
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
      }
      // P = 2^(S·c − m): packed fp32x2 math, a quarter of the exponentials on the FMA pipe
      // (exp2_poly2) so the MUFU pipe (16/clk/SM) is not the limit of the two softmax CTAs
      uint32_t pk[32];
      float2 lsum = make_float2(0.f, 0.f);
      if (dropped) {
        // the tile contributes P = 0 to this row (its -inf scores minus a still -inf running
        // max would give NaN if the row has not seen a kept tile yet)
#pragma unroll
        for (int c = 0; c < 32; ++c) pk[c] = 0u;
      } else {
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const float2 x = __ffma2_rn(make_float2(sv[2 * c], sv[2 * c + 1]), make_float2(sl2, sl2), make_float2(-m, -m));
        float2 e;
        if (c < SPA2_FWD1_POLY_PAIRS) {  // part of the exponentials on the FMA pipe
          e = exp2_poly2(x);
        } else {
          e.x = ex2(x.x);
          e.y = ex2(x.y);
        }
        lsum = __fadd2_rn(lsum, e);
        pk[c] = pack_bf16(e.x, e.y);
      }
      }
      l += lsum.x + lsum.y;
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
    }
    // ---------------- epilogue ----------------
    mbar_wait(o_final, 0);
    if (warp == 2) SPA2_CTL(0, 4);
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
      SPA2_CT_IF(true, 0, 5);
    }
  }
  tc_fence_before();
  __syncthreads();
  SPA2_CT(0, 1);
  if (warp == 1) {
    tmem_dealloc(tbase, 256);
    SPA2_CTL(0, 6);
  }
}

template <int HD, bool P_TMEM, bool HALF>
int launch_fwd(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const CUtensorMap& to,
               const FwdParams& prm, unsigned grid, cudaStream_t st) {
  using C = FwdCfg<HD, P_TMEM>;
  auto kern = k_fwd<HD, P_TMEM, HALF>;
  SPA2_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  SPA2_CUDA_TRY(launch_pdl(kern, dim3(grid), dim3(kFwdThreads), C::SMEM, st, tq, tk, tv, to, prm));
  SPA2_LAUNCH_CHECK();
  return SPA2_OK;
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
  // b_q = 64: the row lists carry half-block codes (bits 30-31) from a b_q = 64 mask
  SPA2_REQUIRE((b_q == BQ || b_q == BQ / 2) && b_kv == BKV, SPA2_ERR_UNSUPPORTED,
               "fwd: block sizes (%lld, %lld) not in {(128, 64), (64, 64)}",
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
  const unsigned grid = (unsigned)(B * H * T_m);
  cudaStream_t st = (cudaStream_t)stream;
  if (b_q == BQ) {
    if (d == 128) return launch_fwd<128, true, false>(tq, tk, tv, to, prm, grid, st);
    return launch_fwd<64, true, false>(tq, tk, tv, to, prm, grid, st);
  }
  if (d == 128) return launch_fwd<128, true, true>(tq, tk, tv, to, prm, grid, st);
  return launch_fwd<64, true, true>(tq, tk, tv, to, prm, grid, st);
}

#ifdef SPA2_CTA_TIMES
// diagnostic (-DSPA2_CTA_TIMES builds only): copy and clear this unit's per-CTA timings
extern "C" int spa2_cta_fetch_fwd(unsigned long long* host_dst) {
  SPA2_CUDA_TRY(cudaDeviceSynchronize());
  SPA2_CUDA_TRY(cudaMemcpyFromSymbol(host_dst, spa2::g_spa2_cta, sizeof(spa2::g_spa2_cta)));
  static unsigned long long zeros[3 * SPA2_CTA_MAX * SPA2_CTA_SLOTS];
  SPA2_CUDA_TRY(cudaMemcpyToSymbol(spa2::g_spa2_cta, zeros, sizeof(spa2::g_spa2_cta)));
  return SPA2_OK;
}
#endif
