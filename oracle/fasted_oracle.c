/*
 * fasted_oracle.c -- CPU restatement of the reference mpjoin arithmetic.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load it.  The product path (paper_2508_21230_b200) never does.
 *
 * Parity pin: tests/golden/ holds vectors produced by the reference package
 * itself (tests/golden/make_golden.py imports /root/reference/pkg/src), and
 * tests/test_oracle.py checks this file against every one of them, plus the
 * C1 known answer (16384x128, |R| = 1,199,444, result sha256 a48ef1db...).
 *
 * What is restated (reference file:line under /root/reference/pkg/src/mpjoin):
 *   - to_half cast: FP32 -> FP16 round-to-nearest-even, overflow (result is
 *     inf) reported with the first row-major offending index
 *     (dataset.py:164-187, numpy astype(float16)).
 *   - squared norms: per row, sequential ascending-k round-toward-zero FP32
 *     sum of exact squares of the widened FP16 values (dataset.py:152-156,
 *     _kernel.py:79-93).
 *   - join: per ordered pair (i, j), a = RZ-sum over k ascending of exact
 *     FP32 products (_kernel.py:57-76, mma.py:1-21), then
 *     d2 = max(((-2 a) + s_i) + s_j, 0) in round-to-nearest (mma.py:143-157),
 *     kept iff d2 <= eps_sq (tiling.py:273-274), rows/cols >= n_logical
 *     dropped by index (tiling.py:275-279), 1-based uint32 indices
 *     (tiling.py:280-285), canonical (i, j) order (tiling.py:116-122).
 *
 * The reference emulates RZ with an FP64 2Sum (_kernel.py:39-54); here the
 * same IEEE operation is the hardware FP32 add under FE_TOWARDZERO (MXCSR is
 * per thread, so every worker thread sets it).  Products of two FP16 values
 * have at most 22 significant bits and are exact in FP32 under any mode.
 */
#include <fenv.h>
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#pragma STDC FENV_ACCESS ON

/* ---------------------------------------------------------------- FP16 */

/* FP32 -> FP16 bits, round to nearest even; overflow gives +-inf. Same rule
 * as numpy's float32 -> float16 cast used at dataset.py:176. */
uint16_t oracle_f32_to_f16(float f) {
    uint32_t x;
    memcpy(&x, &f, 4);
    uint32_t sign = (x >> 16) & 0x8000u;
    uint32_t exp = (x >> 23) & 0xffu;
    uint32_t man = x & 0x7fffffu;
    if (exp == 0xffu) return (uint16_t)(sign | 0x7c00u | (man ? 0x200u : 0u));
    int e = (int)exp - 127 + 15;
    if (e >= 31) return (uint16_t)(sign | 0x7c00u);
    if (e <= 0) {
        if (e < -10) return (uint16_t)sign;
        uint32_t full = man | 0x800000u;
        int shift = 14 - e;               /* 14 .. 24 */
        uint32_t hm = full >> shift;
        uint32_t rem = full & ((1u << shift) - 1u);
        uint32_t half = 1u << (shift - 1);
        if (rem > half || (rem == half && (hm & 1u))) hm++;
        return (uint16_t)(sign | hm);     /* a carry into the exponent is correct */
    }
    uint32_t h = sign | ((uint32_t)e << 10) | (man >> 13);
    uint32_t rem = man & 0x1fffu;
    if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) h++;  /* may carry to inf: correct */
    return (uint16_t)h;
}

/* FP16 bits -> FP32, exact (the widening at tiling.py:193-195). */
float oracle_f16_to_f32(uint16_t h) {
    uint32_t sign = ((uint32_t)h & 0x8000u) << 16;
    uint32_t exp = ((uint32_t)h >> 10) & 0x1fu;
    uint32_t man = (uint32_t)h & 0x3ffu;
    uint32_t x;
    if (exp == 0) {
        if (man == 0) {
            x = sign;
        } else {               /* subnormal: normalise */
            int e = -1;
            do { man <<= 1; e++; } while (!(man & 0x400u));
            man &= 0x3ffu;
            x = sign | ((uint32_t)(127 - 15 - e) << 23) | (man << 13);
        }
    } else if (exp == 31) {
        x = sign | 0x7f800000u | (man << 13);
    } else {
        x = sign | ((exp + 112u) << 23) | (man << 13);
    }
    float f;
    memcpy(&f, &x, 4);
    return f;
}

/* ---------------------------------------------------------------- to_half */

/* Restates to_half (dataset.py:164-193): cast, overflow scan, zero-pad to
 * [n_pad, d_pad], RZ norms.  Returns 0, or 3 (RangeError) with
 * *first_overflow = row-major index of the first value that became inf. */
int oracle_to_half(const float* x, int64_t n, int64_t d, uint16_t* out,
                   int64_t n_pad, int64_t d_pad, float* norms,
                   int64_t* first_overflow) {
    *first_overflow = -1;
    for (int64_t i = 0; i < n; i++)
        for (int64_t k = 0; k < d; k++) {
            uint16_t h = oracle_f32_to_f16(x[i * d + k]);
            if ((h & 0x7fffu) == 0x7c00u) {
                *first_overflow = i * d + k;
                return 3;
            }
        }
    memset(out, 0, (size_t)(n_pad * d_pad) * sizeof(uint16_t));
    for (int64_t i = 0; i < n; i++)
        for (int64_t k = 0; k < d; k++)
            out[i * d_pad + k] = oracle_f32_to_f16(x[i * d + k]);
    int old = fegetround();
    fesetround(FE_TOWARDZERO);
    for (int64_t i = 0; i < n_pad; i++) {
        volatile float acc = 0.0f;   /* keep every add a separate RZ op */
        for (int64_t k = 0; k < d_pad; k++) {
            float v = oracle_f16_to_f32(out[i * d_pad + k]);
            float p = v * v;             /* exact */
            acc = acc + p;               /* RZ (_kernel.py:91) */
        }
        norms[i] = acc;
    }
    fesetround(old);
    return 0;
}

/* RZ squared norms of an already-quantised matrix (compute_squared_norms,
 * dataset.py:159-161). */
void oracle_norms(const uint16_t* X, int64_t n_pad, int64_t d_pad, float* norms) {
    int old = fegetround();
    fesetround(FE_TOWARDZERO);
    for (int64_t i = 0; i < n_pad; i++) {
        volatile float acc = 0.0f;
        for (int64_t k = 0; k < d_pad; k++) {
            float v = oracle_f16_to_f32(X[i * d_pad + k]);
            float p = v * v;
            acc = acc + p;
        }
        norms[i] = acc;
    }
    fesetround(old);
}

/* ---------------------------------------------------------------- join */

#define RB 16    /* rows per register block   */
#define CB 256   /* columns per column chunk  */

typedef struct {
    uint32_t* i;
    uint32_t* j;
    float* d;
    int64_t n, cap;
} pairbuf;

static int pb_push(pairbuf* b, uint32_t i, uint32_t j, float d) {
    if (b->n == b->cap) {
        int64_t nc = b->cap ? b->cap * 2 : 4096;
        uint32_t* ni = realloc(b->i, (size_t)nc * 4);
        uint32_t* nj = realloc(b->j, (size_t)nc * 4);
        float* nd = realloc(b->d, (size_t)nc * 4);
        if (!ni || !nj || !nd) return -1;
        b->i = ni; b->j = nj; b->d = nd; b->cap = nc;
    }
    b->i[b->n] = i; b->j[b->n] = j; b->d[b->n] = d; b->n++;
    return 0;
}

typedef struct {
    const uint16_t* X;
    const float* norms;
    int64_t n_logical, d_pad, r0, r1, c0, c1;
    float eps_sq;
    int count_only;
    pairbuf out;
    int64_t count;
    int err;
} job_t;

/* The RZ accumulation kernel: acc[r][c] over k ascending.  Kept in its own
 * function so the vectoriser sees a plain (i, k, j) nest like
 * accumulate_panel (_kernel.py:66-70).  MXCSR is RZ while it runs. */
__attribute__((target_clones("avx2", "default")))
static void rz_block(const float* P, const float* QT, float* acc,
                     int rows, int cols, int64_t d_pad) {
    for (int r = 0; r < rows; r++) {
        float* a = acc + (size_t)r * CB;
        for (int c = 0; c < cols; c++) a[c] = 0.0f;
        const float* p = P + (size_t)r * d_pad;
        for (int64_t k = 0; k < d_pad; k++) {
            const float pk = p[k];
            const float* q = QT + (size_t)k * CB;
            for (int c = 0; c < cols; c++) a[c] = a[c] + pk * q[c];
        }
    }
}

static void* join_worker(void* arg) {
    job_t* jb = (job_t*)arg;
    fesetround(FE_TOWARDZERO);
    const int64_t d_pad = jb->d_pad;
    float* P = malloc((size_t)RB * d_pad * sizeof(float));
    float* QT = malloc((size_t)d_pad * CB * sizeof(float));
    float* acc = malloc((size_t)RB * CB * sizeof(float));
    /* per-row staging so pairs leave in canonical (i, j) order */
    pairbuf rowbuf[RB];
    memset(rowbuf, 0, sizeof(rowbuf));
    if (!P || !QT || !acc) { jb->err = 1; goto done; }
    for (int64_t r0 = jb->r0; r0 < jb->r1; r0 += RB) {
        int rows = (int)((jb->r1 - r0) < RB ? (jb->r1 - r0) : RB);
        for (int r = 0; r < rows; r++)
            for (int64_t k = 0; k < d_pad; k++)
                P[(size_t)r * d_pad + k] = oracle_f16_to_f32(jb->X[(r0 + r) * d_pad + k]);
        for (int r = 0; r < RB; r++) rowbuf[r].n = 0;
        for (int64_t c0 = jb->c0; c0 < jb->c1; c0 += CB) {
            int cols = (int)((jb->c1 - c0) < CB ? (jb->c1 - c0) : CB);
            for (int64_t k = 0; k < d_pad; k++)
                for (int c = 0; c < cols; c++)
                    QT[(size_t)k * CB + c] = oracle_f16_to_f32(jb->X[(c0 + c) * d_pad + k]);
            rz_block(P, QT, acc, rows, cols, d_pad);
            /* epilogue in round-to-nearest (mma.py:143-157) */
            fesetround(FE_TONEAREST);
            for (int r = 0; r < rows; r++) {
                int64_t i = r0 + r;
                if (i >= jb->n_logical) continue;           /* tiling.py:276-278 */
                const float si = jb->norms[i];
                for (int c = 0; c < cols; c++) {
                    int64_t j = c0 + c;
                    if (j >= jb->n_logical) break;          /* tiling.py:277-279 */
                    volatile float t = -2.0f * acc[(size_t)r * CB + c];
                    t = t + si;
                    volatile float d2 = t + jb->norms[j];
                    float dc = d2 > 0.0f ? d2 : 0.0f;       /* np.maximum(d2, 0) */
                    if (dc <= jb->eps_sq) {                 /* tiling.py:274, on the clamped d2 */
                        jb->count++;
                        if (!jb->count_only &&
                            pb_push(&rowbuf[r], (uint32_t)(i + 1), (uint32_t)(j + 1), dc)) {
                            jb->err = 1; goto done;
                        }
                    }
                }
            }
            fesetround(FE_TOWARDZERO);
        }
        if (!jb->count_only)
            for (int r = 0; r < rows; r++)
                for (int64_t q = 0; q < rowbuf[r].n; q++)
                    if (pb_push(&jb->out, rowbuf[r].i[q], rowbuf[r].j[q], rowbuf[r].d[q])) {
                        jb->err = 1; goto done;
                    }
    }
done:
    for (int r = 0; r < RB; r++) { free(rowbuf[r].i); free(rowbuf[r].j); free(rowbuf[r].d); }
    free(P); free(QT); free(acc);
    fesetround(FE_TONEAREST);
    return NULL;
}

/* The whole self-join restricted to rows [row_begin, row_end) x columns
 * [col_begin, col_end) (full range = self_join, tiling.py:288-359; one
 * 128x128 range = compute_block_tile, tiling.py:199-285).  Returns the
 * total number of qualifying pairs; records are written in canonical order
 * up to `capacity` (pass capacity 0 / NULL arrays to count only).  Returns
 * -1 on allocation failure. */
int64_t oracle_join(const uint16_t* X, const float* norms, int64_t n_logical,
                    int64_t n_pad, int64_t d_pad, int64_t row_begin, int64_t row_end,
                    int64_t col_begin, int64_t col_end, float eps_sq, int nthreads,
                    uint32_t* out_i, uint32_t* out_j, float* out_d, int64_t capacity) {
    (void)n_pad;
    if (nthreads < 1) nthreads = 1;
    int64_t rows = row_end - row_begin;
    if (rows <= 0 || col_end <= col_begin) return 0;
    int64_t nblk = (rows + RB - 1) / RB;
    if (nthreads > nblk) nthreads = (int)nblk;
    job_t* jobs = calloc((size_t)nthreads, sizeof(job_t));
    pthread_t* th = calloc((size_t)nthreads, sizeof(pthread_t));
    if (!jobs || !th) { free(jobs); free(th); return -1; }
    int count_only = (capacity <= 0 || !out_i);
    for (int t = 0; t < nthreads; t++) {
        int64_t b0 = nblk * t / nthreads, b1 = nblk * (t + 1) / nthreads;
        jobs[t].X = X; jobs[t].norms = norms; jobs[t].n_logical = n_logical;
        jobs[t].d_pad = d_pad;
        jobs[t].r0 = row_begin + b0 * RB;
        jobs[t].r1 = row_begin + b1 * RB < row_end ? row_begin + b1 * RB : row_end;
        jobs[t].c0 = col_begin; jobs[t].c1 = col_end;
        jobs[t].eps_sq = eps_sq; jobs[t].count_only = count_only;
    }
    for (int t = 1; t < nthreads; t++) pthread_create(&th[t], NULL, join_worker, &jobs[t]);
    join_worker(&jobs[0]);
    for (int t = 1; t < nthreads; t++) pthread_join(th[t], NULL);
    int64_t total = 0, w = 0;
    int err = 0;
    for (int t = 0; t < nthreads; t++) {
        err |= jobs[t].err;
        total += jobs[t].count;
        for (int64_t q = 0; q < jobs[t].out.n && w < capacity; q++, w++) {
            out_i[w] = jobs[t].out.i[q];
            out_j[w] = jobs[t].out.j[q];
            out_d[w] = jobs[t].out.d[q];
        }
        free(jobs[t].out.i); free(jobs[t].out.j); free(jobs[t].out.d);
    }
    free(jobs); free(th);
    return err ? -1 : total;
}

/* Reference dist_sq for an explicit list of pairs (1-based indices), same
 * arithmetic as the join; used to classify GPU pairs against the eps band
 * without re-running a full join. */
void oracle_pair_d2(const uint16_t* X, const float* norms, int64_t d_pad, int64_t npairs,
                    const uint32_t* pi, const uint32_t* pj, float* out) {
    int old = fegetround();
    for (int64_t q = 0; q < npairs; q++) {
        const uint16_t* a = X + (int64_t)(pi[q] - 1) * d_pad;
        const uint16_t* b = X + (int64_t)(pj[q] - 1) * d_pad;
        fesetround(FE_TOWARDZERO);
        volatile float acc = 0.0f;
        for (int64_t k = 0; k < d_pad; k++) {
            float p = oracle_f16_to_f32(a[k]) * oracle_f16_to_f32(b[k]);
            acc = acc + p;
        }
        fesetround(FE_TONEAREST);
        volatile float t = -2.0f * acc;
        t = t + norms[pi[q] - 1];
        volatile float d2 = t + norms[pj[q] - 1];
        out[q] = d2 > 0.0f ? d2 : 0.0f;
    }
    fesetround(old);
}
