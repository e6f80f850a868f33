/*
 * bsa_oracle.c -- CPU restatement of the reference block-scoring stage.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the package
 * paper_2509_07120_b200 and its CUDA library) may link or call this file;
 * it is used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg as the checker and the timed CPU baseline.
 *
 * It restates, in plain C with an explicit operation order, what the
 * reference computes through numpy / OpenBLAS:
 *
 *   block_pool     /root/reference/pkg/src/bsattn/maskpred.py:104-120
 *                  np.add.reduceat -> out = x0 + pairwise_sum(x1..x_{n-1}),
 *                  then an IEEE fp32 divide by the true block length.
 *   pooled_scores  /root/reference/pkg/src/bsattn/maskpred.py:123-139
 *                  qp @ kp.T (OpenBLAS sgemm: one sequential fmaf chain per
 *                  output, k = 0..d-1), then row_softmax
 *                  (/root/reference/pkg/src/bsattn/tensorio.py:73-87):
 *                  z = acc * f32(scale); z -= rowmax; z = np.exp(z);
 *                  z /= pairwise_sum(row).
 *   np.exp         numpy's float32 SIMD exp (Cody-Waite range reduction +
 *                  rational minimax polynomial + scalef), restated in
 *                  oracle_np_expf below.
 *   select_blocks  /root/reference/pkg/src/bsattn/maskpred.py:142-174
 *                  stable rank by (p desc, index asc), float64 sequential
 *                  cumsum, cdf_len = min(#(cum < tau) + 1, nk),
 *                  take = max(cdf_len, k_floor), mask = rank < take.
 *
 * The third-party arithmetic (numpy 2.3.5 ufunc loops, scipy-openblas 0.3.30
 * SkylakeX sgemm) is not vendored under /root/reference; this restatement is
 * pinned against the reference's own outputs by tests/golden/make_golden.py
 * (fixtures committed under tests/golden/) and by tests/test_cpu_oracle_host.py.
 *
 * Build: see oracle/Makefile (gcc -O2 -ffp-contract=off -pthread).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <pthread.h>
#include <unistd.h>

/* ---------------------------------------------------------------------- */
/* Minimal static parallel-for over [0, n) on POSIX threads (no OpenMP in  */
/* this toolchain).  Thread count: $BSA_ORACLE_THREADS or online CPUs.     */
/* ---------------------------------------------------------------------- */
typedef void (*range_fn)(int64_t lo, int64_t hi, void *ctx);
typedef struct { range_fn fn; void *ctx; int64_t lo, hi; } range_job;

static void *range_trampoline(void *arg)
{
    range_job *j = (range_job *)arg;
    if (j->lo < j->hi) j->fn(j->lo, j->hi, j->ctx);
    return NULL;
}

int oracle_num_threads(void)
{
    const char *env = getenv("BSA_ORACLE_THREADS");
    long t = env ? atol(env) : sysconf(_SC_NPROCESSORS_ONLN);
    if (t < 1) t = 1;
    if (t > 256) t = 256;
    return (int)t;
}

static void parallel_for(int64_t n, range_fn fn, void *ctx)
{
    int nt = oracle_num_threads();
    if (nt > n) nt = (int)(n > 0 ? n : 1);
    if (nt <= 1) { fn(0, n, ctx); return; }
    pthread_t tid[256];
    range_job jobs[256];
    int64_t chunk = (n + nt - 1) / nt;
    for (int t = 0; t < nt; ++t) {
        jobs[t].fn = fn; jobs[t].ctx = ctx;
        jobs[t].lo = t * chunk; jobs[t].hi = (t + 1) * chunk < n ? (t + 1) * chunk : n;
        if (pthread_create(&tid[t], NULL, range_trampoline, &jobs[t]) != 0) {
            range_trampoline(&jobs[t]);
            tid[t] = 0;
        }
    }
    for (int t = 0; t < nt; ++t) if (tid[t]) pthread_join(tid[t], NULL);
}

/* ---------------------------------------------------------------------- */
/* numpy pairwise summation (loops_utils.h.src pairwise_sum), fp32,        */
/* over `n` values spaced `stride` floats apart.                           */
/* ---------------------------------------------------------------------- */
static float pw_sum(const float *a, int64_t n, int64_t stride)
{
    if (n < 8) {
        float res = 0.0f;
        for (int64_t i = 0; i < n; ++i) res += a[i * stride];
        return res;
    }
    if (n <= 128) {
        float r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j * stride];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[(i + j) * stride];
        float res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i * stride];
        return res;
    }
    int64_t half = n / 2;
    half -= half % 8;
    return pw_sum(a, half, stride) + pw_sum(a + half * stride, n - half, stride);
}

float oracle_pairwise_sum(const float *a, int64_t n) { return pw_sum(a, n, 1); }

/* ---------------------------------------------------------------------- */
/* numpy float32 exp (AVX512F / AVX2 simd_exp_f32 algorithm).              */
/* ---------------------------------------------------------------------- */
float oracle_np_expf(float x)
{
    const float LOG2E = 1.442695040888963407359924681001892137f;
    const float MAGIC = 12582912.0f; /* 0x1.8p+23 */
    const float C1 = -6.93145752e-1f, C2 = -1.42860677e-6f;
    const float P0 = 9.999999999980870924916e-01f, P1 = 7.257664613233124478488e-01f,
                P2 = 2.473615434895520810817e-01f, P3 = 5.114512081637298353406e-02f,
                P4 = 6.757896990527504603057e-03f, P5 = 5.082762527590693718096e-04f;
    const float Q0 = 1.0f, Q1 = -2.742335390411667452936e-01f, Q2 = 2.159509375685829852307e-02f;
    if (x >= 88.72283935546875f) return INFINITY;
    if (x <= -103.97208404541015625f) return 0.0f;
    volatile float t = x * LOG2E;      /* separate rounding, no contraction */
    volatile float u = t + MAGIC;
    float quad = u - MAGIC;
    float r = fmaf(quad, C1, x);
    r = fmaf(quad, C2, r);
    float num = fmaf(P5, r, P4);
    num = fmaf(num, r, P3);
    num = fmaf(num, r, P2);
    num = fmaf(num, r, P1);
    num = fmaf(num, r, P0);
    float den = fmaf(Q2, r, Q1);
    den = fmaf(den, r, Q0);
    float poly = num / den;
    return ldexpf(poly, (int)quad); /* single rounding, denormals kept */
}

/* ---------------------------------------------------------------------- */
/* block_pool: x (H, n, d) row-major fp32 -> out (H, ceil(n/block), d).    */
/* ---------------------------------------------------------------------- */
typedef struct { const float *x; int64_t n, d, block, nb; float *out; } pool_ctx;

static void pool_range(int64_t lo, int64_t hi, void *vctx)
{
    const pool_ctx *c = (const pool_ctx *)vctx;
    for (int64_t hb = lo; hb < hi; ++hb) {
        int64_t h = hb / c->nb, b = hb % c->nb;
        int64_t r0 = b * c->block, r1 = r0 + c->block < c->n ? r0 + c->block : c->n;
        int64_t len = r1 - r0;
        const float *src = c->x + (h * c->n + r0) * c->d;
        float *dst = c->out + hb * c->d;
        for (int64_t col = 0; col < c->d; ++col) {
            float s = src[col];
            if (len > 1) s = s + pw_sum(src + c->d + col, len - 1, c->d);
            dst[col] = s / (float)len;
        }
    }
}

int oracle_block_pool(const float *x, int64_t H, int64_t n, int64_t d, int64_t block,
                      float *out)
{
    if (block < 1 || H < 1 || n < 1 || d < 1) return 1;
    pool_ctx c = { x, n, d, block, (n + block - 1) / block, out };
    parallel_for(H * c.nb, pool_range, &c);
    return 0;
}

/* ---------------------------------------------------------------------- */
/* pooled_scores: per head softmax(qp @ kp.T * scale) -> (H, nq, nk).      */
/* ---------------------------------------------------------------------- */
typedef struct { const float *qp, *kp; int64_t nq, nk, d; float scale; float *out; } score_ctx;

static void score_range(int64_t lo, int64_t hi, void *vctx)
{
    const score_ctx *c = (const score_ctx *)vctx;
    for (int64_t hi_row = lo; hi_row < hi; ++hi_row) {
        int64_t h = hi_row / c->nq;
        const float *q = c->qp + hi_row * c->d;
        float *row = c->out + hi_row * c->nk;
        float mx = -INFINITY;
        for (int64_t j = 0; j < c->nk; ++j) {
            const float *k = c->kp + (h * c->nk + j) * c->d;
            float acc = 0.0f;
            for (int64_t t = 0; t < c->d; ++t) acc = fmaf(q[t], k[t], acc);
            volatile float z = acc * c->scale;
            row[j] = z;
            if (z > mx) mx = z;
        }
        for (int64_t j = 0; j < c->nk; ++j) row[j] = oracle_np_expf(row[j] - mx);
        float total = 0.0f + pw_sum(row, c->nk, 1);
        for (int64_t j = 0; j < c->nk; ++j) row[j] = row[j] / total;
    }
}

int oracle_pooled_scores(const float *qp, const float *kp, int64_t H, int64_t nq,
                         int64_t nk, int64_t d, float scale, float *out)
{
    if (H < 1 || nq < 1 || nk < 1 || d < 1) return 1;
    score_ctx c = { qp, kp, nq, nk, d, scale, out };
    parallel_for(H * nq, score_range, &c);
    return 0;
}

/* ---------------------------------------------------------------------- */
/* select_blocks                                                          */
/* ---------------------------------------------------------------------- */
typedef struct { float p; int32_t idx; } rank_item;

static int rank_cmp(const void *a, const void *b)
{
    const rank_item *x = (const rank_item *)a, *y = (const rank_item *)b;
    /* the reference sorts -p ascending with a stable sort: descending
       probability, ties by ascending block index */
    float nx = -x->p, ny = -y->p;
    if (nx < ny) return -1;
    if (nx > ny) return 1;
    return (x->idx > y->idx) - (x->idx < y->idx);
}

typedef struct {
    const float *probs; int64_t nk; double tau; int64_t k_floor;
    uint8_t *mask; int32_t *counts; int failed;
} select_ctx;

static void select_range(int64_t lo, int64_t hi, void *vctx)
{
    select_ctx *c = (select_ctx *)vctx;
    int64_t nk = c->nk;
    rank_item *buf = (rank_item *)malloc(sizeof(rank_item) * (size_t)nk);
    if (!buf) { c->failed = 1; return; }
    for (int64_t row = lo; row < hi; ++row) {
        const float *p = c->probs + row * nk;
        for (int64_t j = 0; j < nk; ++j) { buf[j].p = p[j]; buf[j].idx = (int32_t)j; }
        qsort(buf, (size_t)nk, sizeof(rank_item), rank_cmp);
        double cum = 0.0;
        int64_t below = 0;
        for (int64_t j = 0; j < nk; ++j) {
            cum += (double)buf[j].p;
            if (cum < c->tau) ++below;
        }
        int64_t cdf_len = below + 1 < nk ? below + 1 : nk;
        int64_t take = cdf_len > c->k_floor ? cdf_len : c->k_floor;
        if (take > nk) take = nk;
        uint8_t *m = c->mask + row * nk;
        memset(m, 0, (size_t)nk);
        for (int64_t j = 0; j < take; ++j) m[buf[j].idx] = 1;
        if (c->counts) c->counts[row] = (int32_t)take;
    }
    free(buf);
}

/* mask: H*nq*nk bytes (0/1, the reference's bool layout); counts nullable. */
int oracle_select_blocks(const float *probs, int64_t H, int64_t nq, int64_t nk, double tau,
                         int64_t k_floor, uint8_t *mask, int32_t *counts)
{
    if (H < 1 || nq < 1 || nk < 1) return 1;
    select_ctx c = { probs, nk, tau, k_floor, mask, counts, 0 };
    parallel_for(H * nq, select_range, &c);
    return c.failed ? 3 : 0;
}

/* predict_mask on patch-only inputs (maskpred.py:177-194). probs_out nullable. */
int oracle_predict_mask(const float *q, const float *k, int64_t H, int64_t tp, int64_t d,
                        int64_t block_q, int64_t block_k, float scale, double tau,
                        int64_t k_floor, uint8_t *mask, int32_t *counts, float *probs_out)
{
    int64_t nq = (tp + block_q - 1) / block_q, nk = (tp + block_k - 1) / block_k;
    float *qp = (float *)malloc(sizeof(float) * (size_t)(H * nq * d));
    float *kp = (float *)malloc(sizeof(float) * (size_t)(H * nk * d));
    float *pr = probs_out ? probs_out : (float *)malloc(sizeof(float) * (size_t)(H * nq * nk));
    int rc = 3;
    if (qp && kp && pr) {
        rc = oracle_block_pool(q, H, tp, d, block_q, qp);
        if (!rc) rc = oracle_block_pool(k, H, tp, d, block_k, kp);
        if (!rc) rc = oracle_pooled_scores(qp, kp, H, nq, nk, d, scale, pr);
        if (!rc) rc = oracle_select_blocks(pr, H, nq, nk, tau, k_floor, mask, counts);
    }
    free(qp);
    free(kp);
    if (!probs_out) free(pr);
    return rc;
}
