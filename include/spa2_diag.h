/*
 * spa2_diag.h — C ABI of libspa2_diag.so: micro-benchmarks and building-block probes for
 * the sm_100a kernels in libspa2.so (tcgen05 operand layouts, MMA issue rates, TMA and
 * TMEM throughput, mbarrier latency).  NOT part of the drop-in boundary (include/spa2.h):
 * only tests/ and tools/ load this library.  Same conventions as spa2.h (device
 * pointers, stream as void*, SPA2_OK or a negative status + spa2_last_error()).
 */
#ifndef SPA2_DIAG_H
#define SPA2_DIAG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* spa2_last_error(void);

/* tcgen05 probe (test-only): D = A·Bᵀ with logical A [m,k], B [n,k] (bf16), D fp32
 * row-major [m,n], computed by ONE tcgen05 MMA chain through exactly the shared-memory
 * layouts and descriptors the attention kernels use.  A is stored row-major as [m,k]
 * (a_mn = 0, staged K-major) or as [k,m] (a_mn = 1, staged MN-major); likewise B as
 * [n,k] or [k,n].  use_tma (staging mode): 0 = generic swizzled stores, 1 = TMA
 * (SWIZZLE_128B), 2 = A packed into TMEM by tcgen05.st and consumed by the TS form of
 * tcgen05.mma (m = 128, K-major A only).  m in {64,128}; n, k in {64,128}. */
int spa2_probe_gemm(const void* a, const void* b, float* d, int m, int n, int k, int a_mn, int b_mn,
                    int use_tma, void* stream);

/* tcgen05 issue-rate probe (diagnostic): `ctas` CTAs each issue reps*(k/16) dependent-free
 * MMAs of shape m x n x 16 with the given operand layout (a_tmem = A from TMEM) and record
 * the clock64 cycles of the whole chain in cycles[cta]. */
int spa2_probe_mma_rate(int m, int n, int k, int a_mn, int b_mn, int a_tmem, int reps, int ctas,
                        unsigned long long* cycles, void* stream);

/* TMA streaming-rate probe (diagnostic): `ctas` CTAs each load `iters` random (box_rows x 64)
 * bf16 tiles of a [rows, 64] buffer through a `stages`-deep ring; cycles[cta] = clock64 span. */
int spa2_probe_tma_rate(const void* buf, long long rows, int box_rows, int stages, int iters, int ctas,
                        unsigned long long* cycles, void* stream);
/* Variant (diagnostic): `issuers` warps per CTA with their own rings; requests are tensor boxes
 * of box_rows x 64 x chunks (mode 0) or 1-D bulk copies of the same size (mode 1) over a
 * [rows][128] bf16 matrix.  cycles[ctas*4] receives per-(CTA, issuer) cycle counts. */
/* MMA mix probe (diagnostic): the dQ kernel's per-tile tcgen05 sequence in isolation; see probe.cu. */
int spa2_probe_mma_mix(int reps, int flags, int ctas, const void* gsrc, unsigned long long* cycles, void* stream);
/* Diagnostic: tcgen05.ld / tcgen05.st throughput (mode 0 32-col loads, 1 two loads per wait,
 * 2 16-col loads, 3 16-col stores), `warps` warps per CTA (<= 16); cycles[ctas * 16] per warp. */
/* Diagnostic: cycles per mbarrier try_wait (mode 0) / test_wait (1) / mbar_wait (2) on an
 * already-completed phase, one CTA of `threads` threads; cycles[0] = total for `reps` polls. */
int spa2_probe_mbar_latency(int reps, int mode, int threads, unsigned long long* cycles, void* stream);
int spa2_probe_tmem_rate(int reps, int mode, int warps, int ctas, unsigned long long* cycles, void* stream);
int spa2_probe_tma_rate2(const void* buf, long long rows, int box_rows, int chunks, int stages, int issuers,
                         int mode, int iters, int ctas, unsigned long long* cycles, void* stream);

/* Diagnostic: fp32 reduction (mode 0, red.global.add.v4.f32 one row per thread; 2, coalesced),
 * store (mode 1) or TMA bulk reduction (mode 3, cp.reduce.async.bulk .add.f32 of a 64 KB shared-
 * memory tile) throughput of `ctas` CTAs each adding `tiles` 128x128 fp32 tiles into a rotating
 * set of `nslots` tiles of dst. */
int spa2_probe_red_rate(float* dst, int tiles, int nslots, int ctas, int mode, void* stream);

/* SM clock probe (diagnostic): `ctas` CTAs each spin spin_ns nanoseconds of %globaltimer and
 * store (clock64 cycles, nanoseconds) elapsed into out[2*cta], out[2*cta+1]; their ratio is
 * the SM clock in GHz at that moment (e.g. right after a hot kernel on the same stream). */
int spa2_probe_clock(int spin_ns, int ctas, unsigned long long* out, void* stream);

/* Shared-memory contention probe (diagnostic): warp 0 times reps x 8 SS MMAs (M=128, N=64,
 * K=16) while, by mode bits, 16 KB bulk copies from gsrc (>= 16 MB) (1), STS.128 stores (2),
 * LDS.128 loads (4) or TMEM loads (8) run in other warps, (16) rotating the A operand over three
 * tiles; out[4*cta] = MMA cycles, then bytes moved by each. */
int spa2_probe_smem_contend(int reps, int mode, int ctas, const void* gsrc, unsigned long long* out, void* stream);

/* dK/dV MMA mix probe (diagnostic): the four MMA groups of one K6 tile (S, dP K-major; dVᵀ, dKᵀ
 * MN-major; M=128 N=64, 8 K=16 steps each) issued back to back by one thread, reps tiles;
 * which = 0 all four, 1 S+dP only, 2 dVᵀ+dKᵀ only; +32 S only, +64 single-thread issue, +128 S/dP
 * as TS MMAs (A from TMEM); +256 three other warps add traffic while the chain runs: LDS.128 +
 * tcgen05.st (default), +512 tcgen05.st only, +1024 LDS.128 only, +4096 STS.128 only, of the
 * region at 0 (the Q tile), +8192 96 KB (the P tile), +16384 160 KB (no operand), or +32768 at
 * ((which >> 16) & 15) x 16 KB.  cycles[cta] = clock64 span; cycles[ctas + cta] = bytes moved. */
int spa2_probe_dkdv_mix(int reps, int which, int ctas, unsigned long long* cycles, void* stream);

/* tcgen05.cp rate probe (diagnostic): per rep, 8 tcgen05.cp.128x256b (one 32 KB K-major tile
 * into TMEM) and/or one 8-step SS MMA group (M=128, N=64), by mode bits 1 / 2; cycles[cta]. */
int spa2_probe_cp_rate(int reps, int mode, int ctas, unsigned long long* cycles, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SPA2_DIAG_H */
