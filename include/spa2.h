/*
 * spa2.h — C ABI of libspa2.so, the B200 (sm_100a) SpargeAttention2 hot path.
 *
 * Drop-in boundary for the reference package `sparseattn_lab` (arxiv 2602.13515 lab
 * release, /root/reference/pkg/src).  Each entry point replaces one stage of the
 * reference's Python/numpy path; the reference function it replaces is cited.
 *
 * Conventions (all entry points)
 *   - Every pointer is a DEVICE pointer allocated by the caller; the library holds no
 *     global state and allocates nothing.  Inputs are never written.
 *   - Work is enqueued on `stream` (a cudaStream_t passed as void*); calls return
 *     after enqueueing.  Calls on different streams are independent (re-entrant).
 *   - Return SPA2_OK (0) or a negative status; spa2_last_error() then holds a
 *     thread-local message.  The Python shim maps SPA2_ERR_VALUE/SPA2_ERR_UNSUPPORTED
 *     -> ValueError, SPA2_ERR_NONFINITE -> FloatingPointError, SPA2_ERR_CUDA ->
 *     RuntimeError (the reference raises ValueError / ShapeError / FloatingPointError,
 *     numerics.py:17-32, attention.py:50-59, masker.py:72-86).
 *   - Tensors are logical [B, H, N, d] (the reference contract is one head [N, d],
 *     attention.py:50-59; B = H = 1 reproduces it).  A spa2_view gives the base
 *     pointer and element strides of the B, H and N axes; the d axis is contiguous.
 *   - Block geometry: T_m = ceil(N / b_q) query blocks, T_n = ceil(N / b_kv) key
 *     blocks (numerics.py:68-69).  Block index lists are CSR over the flattened
 *     (b, h, block) rows/columns, int32, ascending within a row/column.
 */
#ifndef SPA2_H
#define SPA2_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPA2_OK 0
#define SPA2_ERR_VALUE (-1)       /* bad argument / geometry            -> ValueError         */
#define SPA2_ERR_NONFINITE (-2)   /* NaN or Inf where finite required   -> FloatingPointError */
#define SPA2_ERR_UNSUPPORTED (-3) /* shape/dtype outside the GPU path   -> ValueError         */
#define SPA2_ERR_CUDA (-4)        /* CUDA runtime / driver failure      -> RuntimeError       */

typedef enum spa2_dtype { SPA2_BF16 = 0, SPA2_F16 = 1, SPA2_F32 = 2, SPA2_F64 = 3 } spa2_dtype;

typedef struct spa2_view {
  const void* ptr;   /* device base pointer of element [0, 0, 0, 0]   */
  int64_t sb;        /* element stride of the batch axis               */
  int64_t sh;        /* element stride of the head axis                */
  int64_t sn;        /* element stride of the token axis (d stride 1)  */
} spa2_view;

/* Library identification and last error of the calling thread. */
const char* spa2_version(void);
const char* spa2_last_error(void);

/* 0 if `device` is an sm_100 (B200-class) GPU this library's cubin runs on. */
int spa2_device_supported(int device);

/* ---- K1: pooled map ----------------------------------------------------------------
 * Replaces masker.pooled_map (masker.py:100-110) = numerics.block_mean_pool x2
 * (numerics.py:55-65) + Q̄K̄ᵀ/√d + numerics.softmax_rows (numerics.py:46-52).
 * q, k: [B,H,N,d] of `dtype` (any of spa2_dtype).  All arithmetic after the load is
 * IEEE float64; the ragged tail block divides by its true row count.
 * probs: float64 [B*H, T_m, T_n] (row-stochastic).
 * workspace: float64, >= B*H*(T_m + T_n)*d elements (pooled Q̄ then K̄).
 * nonfinite: optional int32 device flag (may be NULL); set to 1 if any q/k element is
 * NaN/Inf (the reference's ensure_finite, numerics.py:29-32).  Not cleared first. */
int spa2_pooled_map(spa2_view q, spa2_view k, int dtype, int64_t B, int64_t H, int64_t N,
                    int64_t d, int64_t b_q, int64_t b_kv, double* probs, double* workspace,
                    int32_t* nonfinite, void* stream);

/* K1a alone: numerics.block_mean_pool (numerics.py:55-65) of q (b_q-row groups) and k (b_kv-row
 * groups) into qbar float64 [B*H, T_m, d] and kbar float64 [B*H, T_n, d], with exactly
 * spa2_pooled_map's pooling arithmetic (rows added in order in float64, ragged tail divided by
 * its true count) and its non-finite flag.  The HBM-bound part of the masker. */
int spa2_block_mean_pool(spa2_view q, spa2_view k, int dtype, int64_t B, int64_t H, int64_t N, int64_t d,
                         int64_t b_q, int64_t b_kv, double* qbar, double* kbar, int32_t* nonfinite,
                         void* stream);

/* ---- K2: select --------------------------------------------------------------------
 * Replaces masker._descending_order/top_k_mask/top_p_row_count/top_p_mask/hybrid_mask
 * (masker.py:113-146).  Per row of `probs` (float64 [rows, t_n]): stable descending
 * order (ties -> lower column); kept = min(max(k_count, cnt_p), t_n) where cnt_p =
 * searchsorted_left(sequential float64 cumsum of the sorted row, p_threshold) + 1.
 * Pass p_threshold = p_frac - 1e-12 (masker.py:27,133-134) or -INFINITY to disable
 * top-p; k_count = max(1, ceil(k_frac*t_n)) computed by the caller in IEEE double
 * (masker.py:118-119), or 1 to disable top-k.  Bit-exact with the reference for any
 * float64 input map.
 * keep: uint8 [rows, t_n] (0/1); counts: int32 [rows] (may be NULL). */
int spa2_select(const double* probs, int64_t rows, int64_t t_n, int64_t k_count,
                double p_threshold, uint8_t* keep, int32_t* counts, void* stream);

/* Fused K1+K2 for sparse_attention (the map itself is not returned): spa2_pooled_scores is
 * spa2_pooled_map without its softmax stage (scores = Q̄K̄ᵀ/√d, float64), and
 * spa2_select_scores applies the row softmax to those scores in shared memory with
 * spa2_pooled_map's exact arithmetic before selecting — the keep/counts outputs are
 * bit-identical to spa2_pooled_map + spa2_select.  t_n <= 4096. */
int spa2_pooled_scores(spa2_view q, spa2_view k, int dtype, int64_t B, int64_t H, int64_t N,
                       int64_t d, int64_t b_q, int64_t b_kv, double* scores, double* workspace,
                       int32_t* nonfinite, void* stream);
int spa2_select_scores(const double* scores, int64_t rows, int64_t t_n, int64_t k_count,
                       double p_threshold, uint8_t* keep, int32_t* counts, void* stream);

/* ---- K3: block lists ---------------------------------------------------------------
 * From keep uint8 [bh, t_m, t_n] build
 *   row CSR: row_ptr int32 [bh*t_m + 1], row_idx int32 [>= nnz]  (kept key blocks of
 *            each query block, ascending — the reference's visit order, attention.py:97)
 *   col CSR: col_ptr int32 [bh*t_n + 1], col_idx int32 [>= nnz]  (query blocks that keep
 *            each key block, ascending — the KV-major transpose the backward needs)
 *   row_order int32 [bh*t_m], col_order int32 [bh*t_n]: rows/columns sorted by
 *            descending list length (longest-first launch order for load balance).
 * nnz <= bh*t_m*t_n; pass buffers of that size when nnz is unknown.
 * keep values: 0 dropped, 1 kept; for masks on a 64-row query grid (b_q = 64) paired into
 * 128-row query blocks: 2 = only the top half (rows 0-63) keeps the tile, 3 = only the
 * bottom half; entries then carry (value - 1) in bits 30-31 (block index in bits 0-29).
 * scratch: int32 >= bh*(t_m + t_n) elements. */
int spa2_build_lists(const uint8_t* keep, int64_t bh, int64_t t_m, int64_t t_n, int32_t* row_ptr,
                     int32_t* row_idx, int32_t* col_ptr, int32_t* col_idx, int32_t* row_order,
                     int32_t* col_order, int32_t* scratch, void* stream);

/* ---- K4: block-sparse forward ------------------------------------------------------
 * Replaces attention.sparse_attention_with_mask (attention.py:73-114).
 * q, k, v, o: bf16 [B,H,N,d], d in {64, 128}; b_kv = 64; b_q = 128 (lists from a 0/1 keep)
 * or b_q = 64 (lists carrying half-block codes, see spa2_build_lists: rows of the half that
 * does not keep a tile get P = 0 for it).  The same applies to the backward entry points.
 * lse: float32 [B*H, N], natural log (attention.py:113).  o/lse rows are written for
 * every query block (each row keeps >= 1 block, masker.py:78-79).
 * row_ptr/row_idx/row_order from spa2_build_lists; scale = 1/sqrt(d) (attention.py:86).
 * block_counter: optional int64 device counter (may be NULL); the kernel adds the number
 * of (query block, key block) tiles it computed — the BlockCounter hook, attention.py:36-43. */
int spa2_fwd(spa2_view q, spa2_view k, spa2_view v, spa2_view o, float* lse, int dtype, int64_t B,
             int64_t H, int64_t N, int64_t d, int64_t b_q, int64_t b_kv, const int32_t* row_ptr,
             const int32_t* row_idx, const int32_t* row_order, float scale,
             unsigned long long* block_counter, void* stream);

/* ---- K5-K7: backward ---------------------------------------------------------------
 * Replaces attention.attention_backward (attention.py:128-166) without its forward
 * recompute (o and lse come from spa2_fwd).  delta: float32 [B*H, N] workspace
 * (δ = rowsum(dO ∘ O), attention.py:149).  dq, dk, dv: bf16 [B,H,N,d]; every row of
 * dk/dv is written (key blocks no query keeps get exact zeros, attention.py:152-157). */
int spa2_bwd(spa2_view q, spa2_view k, spa2_view v, spa2_view o, spa2_view dout, const float* lse,
             float* delta, spa2_view dq, spa2_view dk, spa2_view dv, int dtype, int64_t B,
             int64_t H, int64_t N, int64_t d, int64_t b_q, int64_t b_kv, const int32_t* row_ptr,
             const int32_t* row_idx, const int32_t* row_order, const int32_t* col_ptr,
             const int32_t* col_idx, const int32_t* col_order, float scale, void* stream);

/* The three launches spa2_bwd makes, individually (same arguments; used to time each).
 * K5: delta = rowsum(dout ∘ o) (attention.py:149).
 * K7: dq over the row lists (the dq term of attention.py:164).
 * K6: dk, dv over the column lists (attention.py:162, 165). */
int spa2_bwd_delta(spa2_view o, spa2_view dout, float* delta, int dtype, int64_t B, int64_t H,
                   int64_t N, int64_t d, void* stream);
int spa2_bwd_dq(spa2_view q, spa2_view k, spa2_view v, spa2_view dout, const float* lse,
                const float* delta, spa2_view dq, int dtype, int64_t B, int64_t H, int64_t N,
                int64_t d, int64_t b_q, int64_t b_kv, const int32_t* row_ptr, const int32_t* row_idx,
                const int32_t* row_order, float scale, void* stream);
/* K5 fused into K7: dq AND delta (written to `delta` for spa2_bwd_dkdv) in one launch; the
 * dQ kernel's idle epilogue warps compute δ = rowsum(dout ∘ o) one query block ahead with
 * spa2_bwd_delta's exact arithmetic (bit-identical δ).  o/dout rows must be 16-byte aligned. */
int spa2_bwd_dq_delta(spa2_view q, spa2_view k, spa2_view v, spa2_view o, spa2_view dout, const float* lse,
                      float* delta, spa2_view dq, int dtype, int64_t B, int64_t H, int64_t N, int64_t d,
                      int64_t b_q, int64_t b_kv, const int32_t* row_ptr, const int32_t* row_idx,
                      const int32_t* row_order, float scale, void* stream);
int spa2_bwd_dkdv(spa2_view q, spa2_view k, spa2_view v, spa2_view dout, const float* lse,
                  const float* delta, spa2_view dk, spa2_view dv, int dtype, int64_t B, int64_t H,
                  int64_t N, int64_t d, int64_t b_q, int64_t b_kv, const int32_t* col_ptr,
                  const int32_t* col_idx, const int32_t* col_order, float scale, void* stream);

/* Finiteness scan (numerics.ensure_finite, numerics.py:29-32) of one bf16 [B, H, N, d]
 * operand: sets *nonfinite = 1 if any element is NaN or +-Inf (never clears it, so several
 * scans can share one flag with spa2_pooled_map's).  16-byte aligned base, strides % 8. */
int spa2_check_finite(spa2_view x, int dtype, int64_t B, int64_t H, int64_t N, int64_t d, int32_t* nonfinite,
                      void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SPA2_H */
