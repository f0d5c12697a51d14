/*
 * hk_oracle.c -- ORACLE for the exact multiprecision Hankel / Toeplitz / circulant matvec.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load or call this file.  It shares no code, header, table or
 * constant with the CUDA path (paper_1402_5287_b200/, include/) and includes none of it.
 *
 * What it computes: the plain definition, written out with schoolbook big-integer arithmetic.
 *   Numbers ("a = B0 sum_k B^k a_k", B = 2^64): signed mantissas
 *   A_k = a_sign[k] * sum_u a_mag[k][u] 2^(64u), likewise X_j; value = mantissa * 2^-P.
 *   Hankel   (P:50-60 matrix A_H; P:87-90 schoolbook, index typo read as sum over j, DESIGN R1):
 *       Y_i = sum_{j=1..n} A_{i+j-1} X_j,              i = 1..m   (m = n for the square case)
 *   Toeplitz (P:63-72 matrix A_T[i][j] = a_{n-i+j}):
 *       Y_i = sum_{j=1..n} A_{n-i+j} X_j
 *   Circulant (P:74-83 matrix A_C[i][j] = a_{((i-j) mod n)+1}):
 *       Y_i = sum_{j=1..n} A_{((i-j) mod n)+1} X_j
 *   Output y_i = Y_i * 2^-2P, exact (no rounding), Ly = 2L+1 limbs, sign-magnitude, canonical
 *   zero (sign 0, all limbs 0).
 * The three kinds are coded from their own index formulas, not through each other.
 *
 * Arithmetic: per output row, two column accumulators (positive and negative sign products).
 * Column t = u+v receives the 128-bit limb product |A|_u |X|_v; its low and high 64-bit halves
 * are summed into separate unsigned 128-bit sums (<= n*L < 2^64 terms each, so no overflow),
 * then both accumulators are normalised into 64-bit limbs and subtracted.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

enum { ORC_HANKEL = 0, ORC_TOEPLITZ = 1, ORC_CIRCULANT = 2 };

typedef struct {
    int kind;
    int64_t m, n;
    int32_t L, Ly;
    const uint64_t *a_mag;
    const int8_t *a_sign;
    const uint64_t *x_mag;
    const int8_t *x_sign;
    const int64_t *rows;
    int64_t nrows;
    uint64_t *y_mag;
    int8_t *y_sign;
    int64_t begin, end; /* slice of rows[] handled by this thread */
    int status;
} job_t;

/* 0-based index into the defining vector for 0-based (i, j). */
static int64_t a_index(int kind, int64_t n, int64_t i, int64_t j) {
    switch (kind) {
    case ORC_HANKEL:    return i + j;                   /* a_{i+j-1}, 1-based            */
    case ORC_TOEPLITZ:  return (n - 1) - i + j;         /* a_{n-i+j}, 1-based            */
    default:            return ((i - j) % n + n) % n;   /* a_{((i-j) mod n)+1}, 1-based  */
    }
}

/* acc (2L columns of lo/hi sums) -> Ly limbs */
static void normalise(const u128 *lo, const u128 *hi, int32_t L, int32_t Ly, uint64_t *out) {
    u128 carry = 0;
    for (int32_t t = 0; t < Ly; ++t) {
        u128 v = carry;
        if (t < 2 * L) v += lo[t];
        if (t >= 1 && t - 1 < 2 * L) v += hi[t - 1];
        out[t] = (uint64_t)v;
        carry = v >> 64;
    }
}

/* returns -1, 0, +1 for a <=> b over Ly limbs */
static int cmp_limbs(const uint64_t *a, const uint64_t *b, int32_t Ly) {
    for (int32_t t = Ly - 1; t >= 0; --t) {
        if (a[t] != b[t]) return a[t] > b[t] ? 1 : -1;
    }
    return 0;
}

/* out = a - b, requires a >= b */
static void sub_limbs(const uint64_t *a, const uint64_t *b, int32_t Ly, uint64_t *out) {
    unsigned borrow = 0;
    for (int32_t t = 0; t < Ly; ++t) {
        uint64_t d = a[t] - b[t];
        unsigned b1 = a[t] < b[t];
        uint64_t d2 = d - borrow;
        unsigned b2 = d < (uint64_t)borrow;
        out[t] = d2;
        borrow = b1 | b2;
    }
}

static void *worker(void *arg) {
    job_t *jb = (job_t *)arg;
    const int32_t L = jb->L, Ly = jb->Ly;
    u128 *acc = (u128 *)calloc((size_t)8 * L, sizeof(u128));
    uint64_t *pos = (uint64_t *)malloc((size_t)Ly * sizeof(uint64_t));
    uint64_t *neg = (uint64_t *)malloc((size_t)Ly * sizeof(uint64_t));
    if (!acc || !pos || !neg) { jb->status = -3; free(acc); free(pos); free(neg); return NULL; }
    u128 *plo = acc, *phi = acc + 2 * L, *nlo = acc + 4 * L, *nhi = acc + 6 * L;
    for (int64_t r = jb->begin; r < jb->end; ++r) {
        const int64_t i = jb->rows[r];
        memset(acc, 0, (size_t)8 * L * sizeof(u128));
        for (int64_t j = 0; j < jb->n; ++j) {
            const int64_t k = a_index(jb->kind, jb->n, i, j);
            const int s = (int)jb->a_sign[k] * (int)jb->x_sign[j];
            if (s == 0) continue; /* a zero factor contributes nothing */
            u128 *lo = s > 0 ? plo : nlo;
            u128 *hi = s > 0 ? phi : nhi;
            const uint64_t *A = jb->a_mag + (size_t)k * L;
            const uint64_t *X = jb->x_mag + (size_t)j * L;
            for (int32_t u = 0; u < L; ++u) {
                const uint64_t au = A[u];
                if (!au) continue;
                for (int32_t v = 0; v < L; ++v) {
                    const u128 p = (u128)au * X[v];
                    lo[u + v] += (uint64_t)p;
                    hi[u + v] += (uint64_t)(p >> 64);
                }
            }
        }
        normalise(plo, phi, L, Ly, pos);
        normalise(nlo, nhi, L, Ly, neg);
        uint64_t *y = jb->y_mag + (size_t)r * Ly;
        const int c = cmp_limbs(pos, neg, Ly);
        if (c >= 0) sub_limbs(pos, neg, Ly, y); else sub_limbs(neg, pos, Ly, y);
        jb->y_sign[r] = (int8_t)c;
    }
    free(acc); free(pos); free(neg);
    return NULL;
}

/*
 * Computes the requested output rows (0-based indices rows[0..nrows)) of the m x n product.
 *   kind  0 Hankel: a has m+n-1 entries;  1 Toeplitz: m == n, a has 2n-1;  2 circulant: m == n,
 *         a has n entries.
 *   y_mag[r][0..Ly), y_sign[r] receive row rows[r].  Returns 0, or a negative code on bad args.
 */
int hk_oracle_matvec(int kind, int64_t m, int64_t n, int32_t P,
                     const uint64_t *a_mag, const int8_t *a_sign,
                     const uint64_t *x_mag, const int8_t *x_sign,
                     const int64_t *rows, int64_t nrows,
                     uint64_t *y_mag, int8_t *y_sign, int nthreads) {
    if (kind < 0 || kind > 2 || m < 1 || n < 1 || P < 1 || nrows < 0) return -1;
    if (kind != ORC_HANKEL && m != n) return -1;
    for (int64_t r = 0; r < nrows; ++r)
        if (rows[r] < 0 || rows[r] >= m) return -1;
    const int32_t L = (P + 63) / 64, Ly = 2 * L + 1;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > nrows) nthreads = nrows > 0 ? (int)nrows : 1;
    job_t *jobs = (job_t *)calloc((size_t)nthreads, sizeof(job_t));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    if (!jobs || !th) { free(jobs); free(th); return -3; }
    for (int t = 0; t < nthreads; ++t) {
        job_t *jb = &jobs[t];
        jb->kind = kind; jb->m = m; jb->n = n; jb->L = L; jb->Ly = Ly;
        jb->a_mag = a_mag; jb->a_sign = a_sign; jb->x_mag = x_mag; jb->x_sign = x_sign;
        jb->rows = rows; jb->nrows = nrows; jb->y_mag = y_mag; jb->y_sign = y_sign;
        jb->begin = nrows * t / nthreads; jb->end = nrows * (t + 1) / nthreads;
    }
    int rc = 0;
    for (int t = 1; t < nthreads; ++t)
        if (pthread_create(&th[t], NULL, worker, &jobs[t]) != 0) { jobs[t].status = -4; }
    worker(&jobs[0]);
    for (int t = 1; t < nthreads; ++t)
        if (jobs[t].status != -4) pthread_join(th[t], NULL);
    for (int t = 0; t < nthreads; ++t)
        if (jobs[t].status) rc = jobs[t].status;
    if (rc == -4) { /* thread creation failed: finish serially */
        for (int t = 1; t < nthreads; ++t) if (jobs[t].status == -4) { jobs[t].status = 0; worker(&jobs[t]); }
        rc = 0;
        for (int t = 0; t < nthreads; ++t) if (jobs[t].status) rc = jobs[t].status;
    }
    free(jobs); free(th);
    return rc;
}
