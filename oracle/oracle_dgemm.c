/*
 * oracle_dgemm.c -- TEST INFRASTRUCTURE ONLY.
 *
 * The plain, slow, obviously-correct CPU oracle for the one hot path of
 * arXiv 1706.10086: the general matrix multiply
 *
 *     C = alpha * A * B + beta * C                  (Eq. (1))
 *
 * on row-major matrices (the paper's inner loop `lineC[j] += a * lineB[j]`,
 * Listing 2, walks rows of B and C contiguously).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load this library.  The product path
 * (paper_1706_10086_b200/) never links, imports or calls it, and shares no
 * code with it.
 *
 * Written as the plain definition: for every entry (i, j)
 *
 *     acc  = sum_{k = 0 .. K-1, ascending} fl(A[i][k] * B[k][j])   (rounded product, rounded sum)
 *     C_ij = alpha * acc + beta * C0_ij         (alpha applied once on the sum: DESIGN.md reading R5)
 *
 * evaluated in the paper's i-k-j loop order (Listing 2): for each row i, for
 * each k, the row of B scaled by a = A[i][k] is added into an accumulator row.
 * No FMA contraction (built with -ffp-contract=off), no reassociation across k
 * (no -ffast-math): every entry sees exactly the ascending-k sum above, so the
 * result is bitwise identical to the i-j-k dot-product order and independent of
 * the number of threads (rows are split across threads, never k).
 *
 * BLAS conventions (reading R6): beta == 0 -> C is not read;
 * alpha == 0 or K == 0 -> A and B are not read and C = beta * C0.
 *
 * Optionally also returns mag_ij = sum_k |A[i][k]| * |B[k][j]| (same ascending
 * order), the magnitude term of the elementwise acceptance bound
 *     |C_gpu - C_ref| <= 4 K 2^-53 |alpha| mag + 4 2^-53 |beta| |C0| + 1e-300
 * (BASELINE.json north_star).
 *
 * Parity pins: tests/test_oracle.py (worked examples of SPEC.md, brute force in
 * exact rational arithmetic, closed forms, exact dyadic regime, transposition).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int64_t M, N, K;
    double alpha, beta;
    const double *A; int64_t lda;
    const double *B; int64_t ldb;
    double *C; int64_t ldc;
    double *mag; int64_t ldmag;
    int64_t row_begin, row_end;
    int status;
} oracle_job;

static void oracle_rows(oracle_job *job)
{
    const int64_t N = job->N, K = job->K;
    double *acc = (double *)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
    double *m = job->mag ? (double *)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1)) : NULL;
    if (!acc || (job->mag && !m)) { free(acc); free(m); job->status = 1; return; }

    for (int64_t i = job->row_begin; i < job->row_end; ++i) {
        for (int64_t j = 0; j < N; ++j) acc[j] = 0.0;
        if (m) for (int64_t j = 0; j < N; ++j) m[j] = 0.0;

        if (job->alpha != 0.0) {
            /* i-k-j: lineC[j] += a * lineB[j]  (Listing 2) */
            for (int64_t k = 0; k < K; ++k) {
                const double a = job->A[i * job->lda + k];
                const double *lineB = job->B + k * job->ldb;
                for (int64_t j = 0; j < N; ++j) {
                    const double p = a * lineB[j];   /* rounded product */
                    acc[j] = acc[j] + p;             /* rounded sum     */
                }
                if (m) {
                    const double aa = fabs(a);
                    for (int64_t j = 0; j < N; ++j) m[j] = m[j] + aa * fabs(lineB[j]);
                }
            }
        }

        double *lineC = job->C + i * job->ldc;
        for (int64_t j = 0; j < N; ++j) {
            const double t = (job->alpha != 0.0) ? job->alpha * acc[j] : 0.0;
            lineC[j] = (job->beta == 0.0) ? t : t + job->beta * lineC[j];
        }
        if (m) {
            double *lineM = job->mag + i * job->ldmag;
            for (int64_t j = 0; j < N; ++j) lineM[j] = m[j];
        }
    }
    free(acc);
    free(m);
    job->status = 0;
}

static void *oracle_thread(void *p) { oracle_rows((oracle_job *)p); return NULL; }

/*
 * C (in/out, holds C0 on entry) = alpha*A*B + beta*C0, row-major.
 * mag (optional, may be NULL): M x N output with leading dimension ldmag.
 * nthreads <= 0 -> 1 thread.  Returns 0 on success, nonzero on bad arguments
 * or allocation failure.
 */
int oracle_dgemm(int64_t M, int64_t N, int64_t K, double alpha,
                 const double *A, int64_t lda, const double *B, int64_t ldb,
                 double beta, double *C, int64_t ldc,
                 double *mag, int64_t ldmag, int nthreads)
{
    if (M < 0 || N < 0 || K < 0) return 2;
    if (M == 0 || N == 0) return 0;
    if (lda < (K > 1 ? K : 1) || ldb < N || ldc < N) return 2;
    if (mag && ldmag < N) return 2;
    if (nthreads <= 0) nthreads = 1;
    if (nthreads > M) nthreads = (int)M;
    if (K == 0) alpha = 0.0;   /* empty sum: C = beta*C0 without reading A, B */

    oracle_job *jobs = (oracle_job *)calloc((size_t)nthreads, sizeof(oracle_job));
    pthread_t *tids = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    if (!jobs || !tids) { free(jobs); free(tids); return 1; }
    for (int t = 0; t < nthreads; ++t) {
        oracle_job j = { M, N, K, alpha, beta, A, lda, B, ldb, C, ldc, mag, ldmag,
                         (M * t) / nthreads, (M * (t + 1)) / nthreads, 0 };
        jobs[t] = j;
    }
    char *started = (char *)calloc((size_t)nthreads, 1);
    if (!started) { free(jobs); free(tids); return 1; }
    int rc = 0;
    for (int t = 1; t < nthreads; ++t)
        started[t] = (pthread_create(&tids[t], NULL, oracle_thread, &jobs[t]) == 0);
    oracle_rows(&jobs[0]);
    for (int t = 1; t < nthreads; ++t) {
        if (started[t]) pthread_join(tids[t], NULL);
        else oracle_rows(&jobs[t]);          /* could not spawn: do it here */
    }
    for (int t = 0; t < nthreads; ++t) if (jobs[t].status != 0) rc = 1;
    free(started);
    free(jobs);
    free(tids);
    return rc;
}
