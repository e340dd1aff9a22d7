/*
 * tsm2x.h — C ABI of libtsm2x.so, the B200 (sm_100a) TSM2R / TSM2L tall-and-skinny GEMM.
 *
 * Semantics (all entry points):  C_out = C + A * B   (or C_out = A * B with TSM2X_FLAG_C_IS_ZERO)
 *   A is m x k, B is k x n, C is m x n, all column-major with leading dimensions lda/ldb/ldc
 *   (element (i, j) at ptr[i + j * ld]) — the storage convention of the reference `Matrix`
 *   (reference pkg/src/tsgemm/core.py:84-91, flat index i + j*rows).
 *   Naming follows the reference (m, k, n) with the skinny dimension n.
 *
 * Which reference interface each entry point replaces:
 *   tsm2x_validate   <- tsgemm.kernels._check_dims            (pkg/src/tsgemm/kernels.py:36-44)
 *                       tsgemm.core.KernelParams.__post_init__ (pkg/src/tsgemm/core.py:176-181)
 *                       tsgemm.core.KernelParams.validate_for  (pkg/src/tsgemm/core.py:183-190)
 *   tsm2x_run_host   <- tsgemm.kernels.run_native             (pkg/src/tsgemm/kernels.py:391-416)
 *                       host buffers in, host buffer out (the reference's Matrix boundary);
 *                       L_OPT2 zero-C rule of kernels.py:366-368 checked on the host copy.
 *   tsm2x_run        <- the same operation on device-resident buffers, stream-ordered
 *                       (the GPU-native form of run_native; no reference equivalent exists
 *                       because the reference has no device — SURVEY.md §8b).
 *   tsm2x_last_error <- the ValueError / RuntimeError message text.
 *
 * Return codes: 0 = OK; TSM2X_EINVAL maps to Python ValueError (same conditions as the
 * reference, plus a device C that overlaps A or B in memory), every other negative code maps to
 * RuntimeError. Messages are thread-local.
 * All entry points are re-entrant and thread-safe; device work is stream-ordered.
 */
#ifndef TSM2X_H_
#define TSM2X_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSM2X_OK 0
#define TSM2X_EINVAL (-1)      /* argument/shape/param/zero-C violation -> ValueError   */
#define TSM2X_ECUDA (-2)       /* CUDA runtime failure                  -> RuntimeError */
#define TSM2X_ENOMEM (-3)      /* device or pinned allocation failure   -> RuntimeError */
#define TSM2X_EUNSUPPORTED (-4)/* no sm_100a device / unsupported case  -> RuntimeError */

/* reference core.py:57-81 (Variant), same ordinal order as the enum definition */
enum tsm2x_variant {
  TSM2X_V0 = 0,      /* inner product, Alg 1                 */
  TSM2X_V1 = 1,      /* outer product, Alg 2                 */
  TSM2X_V2 = 2,      /* + shared-memory B tile, Alg 3        */
  TSM2X_V3 = 3,      /* + prefetch (the TSM2R kernel), Alg 4 */
  TSM2X_L_OPT1 = 4,  /* TSM2L row-tile loop, Alg 6           */
  TSM2X_L_OPT2 = 5   /* TSM2L interleaved, zero C, Alg 7     */
};

/* reference core.py:23-46 (Precision) */
enum tsm2x_precision { TSM2X_SINGLE = 0, TSM2X_DOUBLE = 1 };

/* reference core.py:160-190 (KernelParams): t1 threads/block, t2 C columns per pass,
 * t3 A elements per prefetch, tcf row tiles per thread (TSM2L); variant = the params' own
 * variant field (validate_for rejects tcf > 1 unless it is a TSM2L variant). */
typedef struct tsm2x_params {
  int32_t t1, t2, t3, tcf;
  int32_t variant;
} tsm2x_params;

/* flags */
#define TSM2X_FLAG_C_IS_ZERO 0x1u   /* caller guarantees C == 0: C is written, never read  */
#define TSM2X_FLAG_CHECK_ZERO_C 0x2u/* tsm2x_run + L_OPT2: verify C == 0 on the device
                                       (synchronises the stream); EINVAL if not          */
#define TSM2X_FLAG_DETERMINISTIC 0x4u/* bitwise run-to-run reproducible: split row blocks are
                                       combined in column order (per-row-block tickets)
                                       instead of with fp64 atomics (the default)          */

/* Kernel implementation override (tsm2x_run_ex); AUTO uses the B200 tuning table. */
enum tsm2x_impl {
  TSM2X_IMPL_AUTO = 0,
  TSM2X_IMPL_STREAM_LDG = 1,  /* TSM2R: register-prefetched LDG.128 stream, stream-K split  */
  TSM2X_IMPL_STREAM_TMA = 2,  /* TSM2R: bulk-copy (TMA engine) smem ring, warp-specialised  */
  TSM2X_IMPL_TSM2L = 3,       /* TSM2L: whole B in smem, grid-stride row stream              */
  TSM2X_IMPL_ABLATION = 4,    /* the paper's V0/V1/V2 algorithms as written (ablation only)  */
  TSM2X_IMPL_TSM2L_SPLITN = 5 /* TSM2L split-n: 4 lanes per row group, warp-shuffle combine
                                 (A/B candidate, k <= 64; profiles/splitn_r02.json)           */
};

/* Validation only (no device work): mirrors the reference's ValueError conditions. */
int tsm2x_validate(int variant, int64_t m, int64_t k, int64_t n, const tsm2x_params* params);

/* Device-resident run. A, B, C are device pointers; stream is a cudaStream_t (NULL = legacy
 * default stream). Returns after enqueueing (asynchronous) unless CHECK_ZERO_C is set.
 * CUDA graphs: calls may be captured once an eager call of the same (or a larger) shape has run
 * on the stream (its workspace is then large enough; growth during a capture is refused with
 * TSM2X_EUNSUPPORTED). Captured calls reuse the capturing stream's workspace, so graphs
 * captured on one stream must not replay concurrently with each other or with eager calls on
 * that stream. */
int tsm2x_run(int variant, int precision, int64_t m, int64_t k, int64_t n,
              const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
              const tsm2x_params* params, uint32_t flags, void* stream);

/* As tsm2x_run with an explicit implementation choice (benchmarks / ablations). */
int tsm2x_run_ex(int variant, int precision, int64_t m, int64_t k, int64_t n,
                 const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                 const tsm2x_params* params, uint32_t flags, int impl, void* stream);

/* Host-buffer run (the drop-in for reference run_native): A (m x k, lda), B, C_in are host
 * pointers (pinned or pageable); the result C_in + A*B is written to C_out (host, ldc; may
 * alias C_in). H2D of A is pipelined with the kernels in column slabs (TSM2R) or row slabs
 * (TSM2L). Synchronous. device = CUDA ordinal. */
int tsm2x_run_host(int variant, int precision, int64_t m, int64_t k, int64_t n,
                   const void* A, int64_t lda, const void* B, int64_t ldb,
                   const void* C_in, void* C_out, int64_t ldc,
                   const tsm2x_params* params, uint32_t flags, int device);

/* tsm2x_run_host over several GPUs of one process: rows of A / C are split into contiguous
 * 32-row-aligned shards, one per entry of devices[] (a device may repeat), each shard runs the
 * host pipeline on its own thread, so the PCIe links (the end-to-end bound) add up. B is copied to
 * every device; rows are independent (reference SPEC.md:262), so no reduction. Synchronous. */
int tsm2x_run_host_multi(int variant, int precision, int64_t m, int64_t k, int64_t n,
                         const void* A, int64_t lda, const void* B, int64_t ldb,
                         const void* C_in, void* C_out, int64_t ldc,
                         const tsm2x_params* params, uint32_t flags, int ndev, const int* devices);

/* Device-resident run over several GPUs of one process (the
 * single-process form of the row sharding in multi.py). A and C are row-sharded: shard g holds
 * rows [r0, r1) = tsm2x_row_range(m, ndev, g) as its own column-major block A[g] (lda[g]) and C[g]
 * (ldc[g]) on devices[g] (a device may repeat). B (k x n, ldb) lives on devices[0]; each shard's
 * stream waits for B on streams[0], every other device receives a copy over NVLink
 * (cudaMemcpy3DPeerAsync into a per-(device, stream) buffer; peer access enabled once), and the
 * shard runs as tsm2x_run on streams[g] (streams = NULL: every device's legacy default stream).
 * No reduction: rows are independent (reference SPEC.md:262); each shard's rows are exactly what
 * tsm2x_run on that shard alone returns (the column-chunk split of a row block follows the
 * shard's size, so in general not the bits of the whole-matrix call, which is within the same
 * tolerance). Asynchronous (stream-ordered per shard); restores the current device. */
int tsm2x_run_multi(int variant, int precision, int64_t m, int64_t k, int64_t n, int ndev, const int* devices,
                    const void* const* A, const int64_t* lda, const void* B, int64_t ldb, void* const* C,
                    const int64_t* ldc, const tsm2x_params* params, uint32_t flags, void* const* streams);

/* Row range [*r0, *r1) of shard g of an m-row problem over ndev shards: contiguous, balanced in
 * 32-row units, the last shard takes the ragged tail (paper_2002_03258_b200.multi.row_partition). */
void tsm2x_row_range(int64_t m, int ndev, int g, int64_t* r0, int64_t* r1);

/* Frees the library's cached device memory on `device` (-1 = every device): the per-(device,
 * stream) workspaces (Bt, fp64 accumulators, queue counters; kept across calls and grown on
 * demand) and the host path's staging buffers, pinned buffers, events and streams. Synchronises
 * the device first. Call it when a long-lived process is done with a set of streams (workspaces
 * are keyed by stream, so a process that keeps creating streams would otherwise keep their
 * workspaces); later calls re-allocate what they need. Not a reference interface. */
int tsm2x_release_cached(int device);

/* Synthetic-input utility (not a reference interface): fills the rows x cols column-major
 * block at ptr (leading dimension ld) with the counter-based uniform [0, 1) generator
 *   x = splitmix64(seed * 0x9E3779B97F4A7C15 + ((col_offset + j) << 32 | (row_offset + i)))
 *   u = (x >> 11) * 2^-53   (float64; cast to float32 for single, like Matrix.random)
 * where (row_offset + i, col_offset + j) is the element's position in the full matrix, so
 * any row slab or shard regenerates bit-identically on the host (oracle/rng.py). */
int tsm2x_fill_uniform(int precision, int64_t rows, int64_t cols, void* ptr, int64_t ld, int64_t row_offset,
                       int64_t col_offset, uint64_t seed, void* stream);

/* Parameter selection — the B200 re-derivation of the paper's (t1, t2, t3, tcf) choice
 * (reference tuner.py:218-363). Process-wide knobs; 0 = the shipped B200 default. */
typedef struct tsm2x_tuning {
  int32_t consumer;   /* 0 auto, 1 FMA, 2 DMMA (fp64, 8/16 columns), 3 FFMA2 (fp32),
                         4 TC (fp32 16-column passes: split-precision tf32 on tcgen05),
                         5 DMMA with the k-step software-pipelined loop (experimental)       */
  int32_t small_kb;   /* KB of A per "small" work item (end of the queue)                     */
  int32_t big_kb;     /* KB of A per "big" work item                                          */
  int32_t tail_pct;   /* % of each row block's columns handed out as small items              */
  int32_t batch_kb;   /* single-chunk row blocks (TSM2L): KB of A per queue grab (tcf analogue) */
  int32_t combine;    /* split row blocks: 0 auto (atomics; ordered if DETERMINISTIC), 1 chunk-ordered,
                         2 fp64 atomics, 3 static stream-K split (reproducible)                 */
} tsm2x_tuning;
int tsm2x_set_tuning(const tsm2x_tuning* t); /* NULL restores the defaults */
int tsm2x_get_tuning(tsm2x_tuning* out);

/* What a tsm2x_run_ex call with these arguments would launch (first 16-column pass). */
typedef struct tsm2x_plan {
  int32_t impl;            /* enum tsm2x_impl actually used (AUTO resolved)                    */
  int32_t consumer;        /* 1 FMA, 2 DMMA, 3 FFMA2, 5 TC (tensor-core fp32), 6 DMMA pipelined
                              (TMA kernels), 0 otherwise                                       */
  int32_t rows_per_block;  /* R: rows per row block            (the paper's t1 analogue)      */
  int32_t cols_per_pass;   /* NT: skinny columns per pass       (t2)                           */
  int32_t cols_per_stage;  /* KC: columns per pipeline stage                                   */
  int32_t stages;          /* ring depth; STAGES*KC columns of A in flight per SM (t3)         */
  int32_t passes;          /* ceil(n / 16)                                                     */
  int32_t deterministic;   /* 1 when the static fixed-order combine is used                    */
  int64_t grid;            /* CTAs                                                             */
  int64_t items, nbig, kbig, nsmall, ksmall, batch; /* dynamic work items (TMA dynamic path)   */
} tsm2x_plan;
int tsm2x_plan_for(int precision, int64_t m, int64_t k, int64_t n, int64_t lda, int a_aligned16, uint32_t flags,
                   int impl, tsm2x_plan* out);

/* Profiling hook (bench evidence): the NEXT device-resident call made by this thread
 * (tsm2x_run / tsm2x_run_ex) is bracketed by cudaEventRecord of these two cudaEvent_t on its
 * stream — before its first launch (prep_dyn, when the call has one) and after its last (the
 * stream kernel, or tsm2_finalize for fp32 split passes), so the events never sit inside the
 * programmatic-dependent-launch chain between those kernels; the hook then clears. Pass NULLs to
 * clear explicitly. */
int tsm2x_set_kernel_events(void* start_event, void* stop_event);

/* Thread-local message describing the last non-OK return on this thread. */
const char* tsm2x_last_error(void);

/* Library version (major*10000 + minor*100 + patch) and build target ("sm_100a"). */
int tsm2x_version(void);
const char* tsm2x_build_target(void);

/* Number of kernels this process has launched through the library since load (bench evidence). */
int64_t tsm2x_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* TSM2X_H_ */
