/*
 * gemm_f64.h -- C ABI of the B200-native double-precision GEMM library
 * (libgemm_f64.so, built from paper_1706_10086_b200/csrc/).
 *
 * The one hot path of arXiv 1706.10086 (Matthes et al., "Tuning and
 * optimization for a variety of many-core architectures without changing a
 * single line of implementation code using the Alpaka library"):
 *
 *     C = alpha * A * B + beta * C                 PAPER.md Eq. (1)
 *
 * computed as a tiled GEMM (Fig. 2; §2.1) whose tile size
 * and elements-per-thread are compile-time parameters (Listing 1).
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 * - Storage is ROW-MAJOR (the paper's inner loop `lineC[j] += a * lineB[j]`,
 *   Listing 2, walks rows): element (i, j) of an R x S matrix X with
 *   leading dimension ldX lives at X[i * ldX + j].  A is M x K, B is K x N,
 *   C is M x N.  Square N x N is the special case M = N = K.
 * - Matrix pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors) on
 *   the current device, except in gemm_f64_host().  The caller owns every
 *   matrix buffer and stream; the library never frees caller memory.
 * - Calls are asynchronous (enqueue and return, like cuBLAS): launch errors are
 *   reported through the return code, faults inside a kernel surface at the
 *   caller's next synchronisation.
 * - On any argument error NOTHING is enqueued; gemm_last_error() returns a
 *   thread-local message naming the offending argument.
 * - Arithmetic: IEEE binary64, round-to-nearest-even, no fast-math.  The sum
 *   over k is accumulated by the FP64 tensor pipe (mma.sync m8n8k4 f64 ->
 *   SASS DMMA.8x8x4) in an order different from the oracle's; alpha is applied
 *   once to the finished sum (reading R5).  Results satisfy,
 *   elementwise, with u = 2^-53 and mag = |A| |B|:
 *       |C - C_exact| <= 4 K u |alpha| mag + 4 u |beta| |C0| + 1e-300
 *   (BASELINE.json north_star).
 * - BLAS special cases (reading R6):
 *     M == 0 or N == 0                  -> no-op
 *     (alpha == 0 or K == 0), beta == 1 -> no-op
 *     alpha == 0 or K == 0              -> C = beta * C without reading A or B
 *     beta == 0                         -> C is not read (NaN in C is harmless)
 * - Argument rules: M, N, K >= 0; lda >= max(1, K); ldb >= max(1, N);
 *   ldc >= max(1, N); A, B non-NULL when alpha != 0 and K > 0 and M*N > 0;
 *   C non-NULL when M*N > 0; all pointers 8-byte aligned; C must not overlap
 *   A or B.  M, N, K < 2^31 - 4096 (32-bit tile arithmetic / TMA coordinates).
 *   Pointers 16-byte aligned with even lda/ldb take the TMA path; anything
 *   else takes a slower GPU path (cp.async staging).  There is no CPU path.
 */
#ifndef GEMM_F64_H
#define GEMM_F64_H

#include <stdint.h>

#if defined(__GNUC__)
#define GEMM_API __attribute__((visibility("default")))
#else
#define GEMM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GEMM_OK = 0,
    GEMM_ERR_ARG = 1,          /* invalid argument (message names it)        */
    GEMM_ERR_CUDA = 2,         /* CUDA runtime / launch error                */
    GEMM_ERR_NCCL = 3,         /* NCCL error in a sharded / comm call        */
    GEMM_ERR_UNSUPPORTED = 4,  /* valid but unsupported (e.g. ldb != N sharded) */
    GEMM_ERR_ALLOC = 5         /* device or host allocation failed           */
} gemm_status;

/* ------------------------------------------------------------------ single GPU */

/* Launch behaviour (all entry points that enqueue GEMM kernels).  Kernels are launched with
 * programmatic stream serialization (CUDA programmatic dependent launch): a GEMM kernel may
 * become resident while the previous kernel in the stream is still finishing, but it executes
 * griddepcontrol.wait -- which returns once that kernel has completed and its memory is
 * visible -- before its first global-memory access, so stream order is preserved for every
 * caller.  Setting the environment variable GEMM_PDL=0 (read once per process) launches them
 * without the attribute.
 *
 * Workspace and CUDA graphs.  Split-K / stream-K partials, tile counters and repack buffers
 * are library workspace cached per (device, stream) and created on first use.  Calls are
 * capturable into CUDA graphs after one eager warm-up call of the largest shape on the
 * capture stream (an allocation during capture fails with GEMM_ERR_ALLOC).  Workspace that a
 * call used is never freed while the process runs unless gemm_workspace_release() is called:
 * when a later call needs more, the old buffer is retired (kept) and a larger one allocated,
 * so a captured graph stays valid.  A graph replays on its capture stream's workspace: do
 * not replay it concurrently with eager calls on that stream, or with itself. */

/* C[MxN] = alpha*A[MxK]*B[KxN] + beta*C, row-major, device pointers.
 * Enqueued on the legacy default stream (stream 0, torch's default stream).
 * Returns a gemm_status. */
GEMM_API int gemm_f64(int64_t M, int64_t N, int64_t K, double alpha,
             const double *A, int64_t lda, const double *B, int64_t ldb,
             double beta, double *C, int64_t ldc);

/* Same, enqueued on `cuda_stream` (a cudaStream_t; NULL = legacy default). */
GEMM_API int gemm_f64_stream(int64_t M, int64_t N, int64_t K, double alpha,
                    const double *A, int64_t lda, const double *B, int64_t ldb,
                    double beta, double *C, int64_t ldc, void *cuda_stream);

/* Same, forcing kernel configuration `cfg_id` (0 <= cfg_id < gemm_num_cfgs())
 * instead of the built-in heuristic; cfg_id = -1 means "heuristic".  Used by
 * the tuning sweep (the paper's "multidimensional parameter tuning").
 * A TMA configuration given arguments that fail the TMA alignment rules
 * returns GEMM_ERR_UNSUPPORTED. */
GEMM_API int gemm_f64_cfg(int64_t M, int64_t N, int64_t K, double alpha,
                 const double *A, int64_t lda, const double *B, int64_t ldb,
                 double beta, double *C, int64_t ldc, int cfg_id, void *cuda_stream);

/* Same as gemm_f64_cfg, additionally forcing the number of deterministic split-K
 * slices for a *_splitk configuration (splits = 0: the model's choice; 1: no
 * split).  Forcing splits > 1 on a configuration without split-K returns
 * GEMM_ERR_UNSUPPORTED.  With cfg_id = -1: splits = 0 is gemm_f64_cfg(-1); splits = 1
 * restricts the heuristic to one k-pass per tile (no split-K / stream-K); splits > 1
 * restricts it to the *_splitk configurations and launches exactly `splits` slices. */
GEMM_API int gemm_f64_ex(int64_t M, int64_t N, int64_t K, double alpha,
                const double *A, int64_t lda, const double *B, int64_t ldb,
                double beta, double *C, int64_t ldc, int cfg_id, int splits, void *cuda_stream);

/* Single precision (the paper's second precision): C = alpha*A*B + beta*C on
 * row-major FP32 device buffers, computed on the tensor cores with the 3xTF32 split
 * (x = hi + lo, A_lo*B_hi + A_hi*B_lo + A_hi*B_hi accumulated in FP32 in TMEM by
 * tcgen05.mma kind::tf32).  Accuracy is FP32-class; the acceptance bound used by the
 * tests is DESIGN.md reading R16.  Any alignment (4-byte) and leading dimension: A and B
 * are split into library workspace first (per stream).  Same argument rules and BLAS
 * special cases as gemm_f64. */
GEMM_API int gemm_f32(int64_t M, int64_t N, int64_t K, float alpha,
             const float *A, int64_t lda, const float *B, int64_t ldb,
             float beta, float *C, int64_t ldc);
GEMM_API int gemm_f32_stream(int64_t M, int64_t N, int64_t K, float alpha,
                    const float *A, int64_t lda, const float *B, int64_t ldb,
                    float beta, float *C, int64_t ldc, void *cuda_stream);
/* Same, forcing single-precision tile configuration cfg_id (-1 = default);
 * gemm_f32_num_cfgs / gemm_f32_cfg_name enumerate them ("tf32x3_128x<BN>x<BK>_s<stages>"). */
GEMM_API int gemm_f32_cfg(int64_t M, int64_t N, int64_t K, float alpha,
                 const float *A, int64_t lda, const float *B, int64_t ldb,
                 float beta, float *C, int64_t ldc, int cfg_id, void *cuda_stream);
GEMM_API int gemm_f32_num_cfgs(void);
GEMM_API int gemm_f32_cfg_name(int cfg_id, char *buf, int len);

/* Host-buffer entry point ("the call a user makes" with host data): A, B, C are
 * HOST pointers (pinned for full copy/compute overlap; pageable works but
 * serialises).  The library allocates device buffers from a cached pool, copies
 * B and row panels of A (and of C when beta != 0) host->device, computes each
 * row panel as it lands, and copies result panels device->host while the next
 * panel computes.  Synchronous: C holds the result when it returns. */
GEMM_API int gemm_f64_host(int64_t M, int64_t N, int64_t K, double alpha,
                  const double *A, int64_t lda, const double *B, int64_t ldb,
                  double beta, double *C, int64_t ldc);

/* The block schedule gemm_f64_host uses for this shape (introspection, tests, tools): writes
 * geometry[7] = {R0 first row panel, Ra its first block's rows, cb0 first column block, cb
 * later column blocks, Rp later row panels, Rlast thin last panel (0: none), nlast its column
 * blocks} (caller-owned) and, if sim_seconds != NULL, the copy/compute simulation's predicted
 * seconds for it (tools/e2e_sim.py --r02 is the same model).  num_sms <= 0: the current
 * device's SM count.  Host-only arithmetic, no device work.  Negative sizes or NULL geometry
 * -> GEMM_ERR_ARG. */
GEMM_API int gemm_host_plan(int64_t M, int64_t N, int64_t K, int beta_nonzero, int num_sms,
                   int64_t geometry[7], double *sim_seconds);

/* Release the device buffers cached by gemm_f64_host on the current device. */
GEMM_API int gemm_host_pool_release(void);

/* Synchronizes the current device, then frees every workspace buffer the device entry points
 * cached on it (FP64 split-K / stream-K partials and counters, repack buffers, FP32 split
 * workspace), retired ones included.  CUDA graphs captured from earlier calls must not be
 * replayed afterwards. */
GEMM_API int gemm_workspace_release(void);

/* ------------------------------------------------------------ configurations */

typedef struct {
    int bm, bn, bk;     /* CTA tile of C (BM x BN) and k-depth per pipeline stage */
    int wm, wn;         /* warp tile; elements (accumulators) per thread = wm*wn/32 */
    int stages;         /* shared-memory pipeline depth                            */
    int threads;        /* threads per CTA (TMA refills are issued by lane 0 of warps 0..3 in turn) */
    int smem_bytes;     /* dynamic shared memory per CTA                           */
    int tma;            /* 1: TMA + mbarrier pipeline; 0: cp.async staging          */
    int split_k;        /* 1: no split-K; 0: deterministic split-K, slices chosen per call;
                           -1: stream-K (persistent grid, even k-step share per CTA);
                           -2: hybrid (full data-parallel waves + stream-K tail + fix-up) */
    int regs;           /* registers per thread (from cudaFuncGetAttributes; 0 before first use) */
} gemm_cfg_desc;

GEMM_API int gemm_num_cfgs(void);
/* Writes a NUL-terminated name such as "tma_128x128x16_w64x32_s4" into buf. */
GEMM_API int gemm_cfg_name(int cfg_id, char *buf, int len);
GEMM_API int gemm_cfg_info(int cfg_id, gemm_cfg_desc *out);
/* The configuration the heuristic picks for this shape / alignment (for large operands that
 * miss the TMA rules -- 2MNK >= 4e9, M, N >= 64, K >= 16 -- the TMA plan the call launches on
 * its repacked copies; gemm_plan / gemm_plan_ex likewise). */
GEMM_API int gemm_cfg_select(int64_t M, int64_t N, int64_t K, const double *A, int64_t lda,
                    const double *B, int64_t ldb);

/* The full launch plan of the heuristic: configuration id and number of
 * deterministic split-K slices (1 = no split; >1 only for *_splitk / *_csplit configurations:
 * each slice multiplies a contiguous k-range; slices 0..S-2 publish a workspace partial and the
 * last slice adds them and its own in slice order (*_csplit: through distributed shared memory
 * of the slices' cluster), row a5). */
GEMM_API int gemm_plan(int64_t M, int64_t N, int64_t K, const double *A, int64_t lda,
              const double *B, int64_t ldb, int *cfg_id, int *splits);

/* gemm_plan, optionally restricted (one_pass != 0) to plans that run each tile's k-range in
 * one pass (no split-K / stream-K / hybrid) -- the plan gemm_f64_ex(cfg_id = -1, splits = 1),
 * gemm_f64_host's blocks and gemm_f64_sharded launch (*splits is then 1). */
GEMM_API int gemm_plan_ex(int64_t M, int64_t N, int64_t K, const double *A, int64_t lda,
                 const double *B, int64_t ldb, int one_pass, int *cfg_id, int *splits);

/* Auto-tuner hooks (the paper's per-architecture tuning, §2.3, as a
 * persisted per-shape table).  gemm_plan_set pins the plan the heuristic entry
 * points use for (M, N, K, TMA-eligible) on every device; gemm_plan_clear
 * forgets all pinned and cached plans; gemm_tune_load reads a text table with
 * lines "M N K tma cfg_name splits" ('#' comments), pinning each, and writes the
 * number of entries loaded to *n_loaded (may be NULL). */
GEMM_API int gemm_plan_set(int64_t M, int64_t N, int64_t K, int tma, int cfg_id, int splits);
GEMM_API int gemm_plan_clear(void);
GEMM_API int gemm_tune_load(const char *path, int *n_loaded);
/* Writes every pinned plan (gemm_plan_set, gemm_tune_load, gemm_plan_autotune) to `path` in
 * gemm_tune_load's format, replacing the file; *n_saved (may be NULL) = lines written.
 * NULL path / unwritable file -> GEMM_ERR_ARG. */
GEMM_API int gemm_tune_save(const char *path, int *n_saved);

/* Run-time tuning of one shape (§2.3 P:315-320 done at first use instead of offline): times
 * the plan currently in force for (M, N, K) -- pinned or the heuristic's -- and the heuristic's
 * next best-scored plans, `top` in all (0 = 8, at most 64), on the caller's device A (M x K,
 * lda) and B (K x N, ldb) writing a library scratch C (cudaMalloc'd and freed inside; alpha = 1,
 * beta = 0), each as batches of back-to-back launches (>= ~2 ms, best of 3) timed with CUDA
 * events on `cuda_stream`.  The fastest (ties within 0.3 % go to the plan in force, then to
 * the better model score) is pinned as by gemm_plan_set and written to *cfg_id / *splits, its
 * device seconds per call to *seconds (may be NULL).  Synchronous; A and B are only read.
 * Candidates: the plan in force, each of the `top` best-scored configurations at its
 * best-scored slice count, and slice counts 1, S - 1, S + 1, 2S of the three best-scored ones;
 * each costs about 5 calls of the shape.  Operands that miss the TMA rules (alignment, odd
 * leading dimension) are timed on packed copies when the problem is large enough for the
 * heuristic call to repack them (2MNK >= 4e9, M, N >= 64, K >= 16), which then launches the
 * pinned plan; smaller ones run their size class's cp.async configuration and are not timed
 * (the heuristic's plan is returned, *seconds = 0).  Results of the pinned plan are within the
 * documented bound like every plan; different plans may round differently.
 * Errors: M, N or K <= 0, NULL pointers, lda < K, ldb < N, top out of range -> GEMM_ERR_ARG; called while
 * `cuda_stream` is capturing -> GEMM_ERR_UNSUPPORTED; scratch allocation -> GEMM_ERR_ALLOC;
 * launch failures -> GEMM_ERR_CUDA (nothing pinned).
 * With the environment variable GEMM_AUTOTUNE=1 (read once per process) the heuristic entry
 * points (gemm_f64, gemm_f64_stream, gemm_f64_cfg / _ex with cfg_id = -1 and splits = 0) call
 * this themselves, on the caller's stream, the first time they see a TMA shape that no table
 * pins (that first call is then synchronous; skipped while capturing; attempted once per
 * shape); gemm_tune_save persists the result for gemm_tune_load in later processes. */
GEMM_API int gemm_plan_autotune(int64_t M, int64_t N, int64_t K, const double *A, int64_t lda,
                       const double *B, int64_t ldb, int top, int *cfg_id, int *splits,
                       double *seconds, void *cuda_stream);

/* Thread-local message for the last non-OK return on this thread. */
GEMM_API const char *gemm_last_error(void);

/* -------------------------------------------------------- synthetic inputs */

/* Fills rows [row0, row0+nrows) of a logical rows x cols matrix into
 * X (device, row-major, leading dimension ldx; X points at logical row row0)
 * with the counter-based generator documented in synth/__init__.py:
 * mode 0 uniform[-1,1), 1 dyadic m/256, 2 integers [-8,8], 3 ones,
 * 4 identity, 5 zeros; mat = matrix id (A=0, B=1, C0=2).  Bitwise identical
 * to synth.matrix() (tested).  Input synthesis only -- no GEMM arithmetic. */
GEMM_API int gemm_fill_f64(int mode, uint64_t seed, int mat, int64_t rows, int64_t cols,
                  int64_t row0, int64_t nrows, double *X, int64_t ldx, void *cuda_stream);

/* ------------------------------------------------- FP64 peak microbenchmarks */

/* Launches `blocks` x (32*warps) threads; each warp issues `iters` rounds of
 * 8 independent mma.m8n8k4.f64 (DMMA.8x8x4, 512 FLOP each) or, with
 * kind = 1, each thread issues `iters` rounds of 8 independent DFMA.
 * Writes one double per block to out[blocks] (to defeat dead-code removal) and
 * the SM cycle count of block 0 to cycles_out[0] (device int64).
 * FLOPs issued = blocks*warps*iters*8*512 (DMMA) or blocks*warps*32*iters*8*2 (DFMA). */
GEMM_API int gemm_peak_probe(int kind, int blocks, int warps, int64_t iters,
                    double *out, int64_t *cycles_out, void *cuda_stream);

/* --------------------------------------------------- multi-GPU (one process per GPU) */

/* The paper computes on one device and has no communication ("Alpaka does not abstract the
 * inter-node communication", §1.2); the multi-GPU split below is the north star's
 * (BASELINE.json: "C is partitioned by row blocks: A is row-sharded, B is broadcast over
 * NVLink with NCCL"), SURVEY.md §8(b)/(e).  Errors follow SPEC's "dimension/tile mismatch ->
 * error" and "error naming n, t, e": a non-OK code plus gemm_last_error().
 *
 * Rank 0 creates the 128-byte NCCL unique id (id_out: caller-owned 128 bytes; NCCL failure ->
 * GEMM_ERR_NCCL); distribute it to all ranks (e.g. with torch.distributed.broadcast) before
 * gemm_comm_init. */
GEMM_API int gemm_comm_unique_id(unsigned char id_out[128]);
/* Creates the library-owned communicator for `rank` of `nranks` on the current device
 * (collective over the nranks processes).  *comm_out receives an opaque handle owned by the
 * library (a private NCCL communicator, a communication stream, events and the column-panel
 * workspace), released by gemm_comm_destroy.  The environment variable GEMM_NCCL_MAX_CTAS (> 0)
 * sets the communicator's maxCTAs, i.e. caps the SMs a panel broadcast running beside the
 * GEMM (bcast_chunks > 1) can take; unset, NCCL chooses.  Bad rank / nranks / NULL -> GEMM_ERR_ARG;
 * NCCL failure -> GEMM_ERR_NCCL (nothing is left allocated). */
GEMM_API int gemm_comm_init(void **comm_out, int nranks, const unsigned char id[128], int rank);
/* Destroys a communicator (NULL is a no-op).  Collective like ncclCommDestroy; the caller
 * must have synchronized the streams its calls used. */
GEMM_API int gemm_comm_destroy(void *comm);
/* The communicator's size and this process's rank as NCCL reports them (ncclCommCount,
 * ncclCommUserRank): *nranks, *rank (caller-owned ints).  NULL -> GEMM_ERR_ARG; NCCL failure
 * -> GEMM_ERR_NCCL.  bench.py logs it per rank. */
GEMM_API int gemm_comm_info(void *comm, int *nranks, int *rank);

/* Row-block-sharded GEMM (collective: every rank calls it with the same N, K,
 * alpha, beta, root).  Rank r owns rows [floor(r*M/P), floor((r+1)*M/P)) of A
 * and C (M_local of them; may differ between ranks).  B (K x N, contiguous,
 * ldb == N required else GEMM_ERR_UNSUPPORTED) is the source on `root` and a
 * receive buffer (overwritten) elsewhere; it is broadcast over NVLink with
 * NCCL, in `bcast_chunks` column panels (>= 1) so that panel j+1 travels while
 * panel j is multiplied -- per-entry arithmetic is unchanged, so the result is
 * bitwise equal to the single-GPU call with the same configuration.
 * Then each rank computes C_local = alpha*A_local*B + beta*C_local (Eq. (1) P:77-79 on its
 * rows).  `bcast_chunks` extends SURVEY §8(b)'s signature with §8(e)'s overlap option
 * ("N-panel chunking"): 1 = one broadcast of B, then the local GEMM; c > 1 = c column panels
 * (widths multiples of 16, at most N/64 panels).  The library's column-panel workspace is
 * reused by the next call only after this call's GEMMs finished (stream-ordered), whatever
 * stream either call uses.  Asynchronous on `cuda_stream`; argument errors as gemm_f64 ->
 * nothing enqueued; NCCL errors -> GEMM_ERR_NCCL. */
GEMM_API int gemm_f64_sharded(int64_t M_local, int64_t N, int64_t K, double alpha,
                     const double *A_local, int64_t lda, double *B, int64_t ldb,
                     double beta, double *C_local, int64_t ldc,
                     void *comm, int root, int bcast_chunks, void *cuda_stream);

/* Plain broadcast of a device buffer of `count` doubles from `root` (in place, ncclBroadcast;
 * the one exchange step of SURVEY §8(e), exposed for tests and for timing it alone).
 * count < 0, bad root or NULL -> GEMM_ERR_ARG; NCCL failure -> GEMM_ERR_NCCL. */
GEMM_API int gemm_bcast_f64(double *buf, int64_t count, int root, void *comm, void *cuda_stream);

/* Library version string. */
GEMM_API const char *gemm_version(void);

#ifdef __cplusplus
}
#endif

#endif /* GEMM_F64_H */
