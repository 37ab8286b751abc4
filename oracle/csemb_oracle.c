/*
 * csemb_oracle.c -- CPU ORACLE for the fused SpMM-Legendre recurrence.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker (or the timed CPU baseline), never as the product path.
 *
 * This is a plain-C restatement of the reference's algorithm for the hot path
 * (reference = the `csemb` Python package, /root/reference/pkg/src/csemb):
 *
 *   oracle_spmm            <- sparse.spmv_multi (sparse.py:171-188), which calls
 *                             scipy `_sparsetools.csr_matvecs` (third-party C++,
 *                             scipy 1.18.1, not vendored): per row, for each
 *                             stored entry in stored order, y[i,:] += a*x[j,:],
 *                             starting from zero, multiply and add rounded
 *                             separately (no FMA; compile with -ffp-contract=off).
 *   oracle_run_stage       <- engine._run_stage (engine.py:205-228), exact
 *                             numpy rounding sequence: q = alpha*y;
 *                             q = q - (beta*q2); acc = acc + (theta*q).
 *   oracle_apply_expansion <- engine._apply_expansion (engine.py:231-258); the
 *                             32-column chunking only affects the per-chunk
 *                             max|Q(r)| log / divergence report, not values.
 *   oracle_sample_projection <- engine.sample_projection / _mix64
 *                             (engine.py:44-50, 79-99).
 *
 * Parity is pinned: tests/test_oracle.py checks every function here against
 * the golden vectors in tests/golden/ generated from the reference itself
 * (tests/golden/make_golden.py).
 *
 * Threading: OpenMP over rows.  Each output element's arithmetic is the same
 * for any thread count (rows are independent), so results are bit-identical
 * for any OMP_NUM_THREADS -- the analogue of the reference's worker-count
 * invariance (tests/test_engine.py:162-171).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define GOLDEN 0x9E3779B97F4A7C15ULL
#define MIX_A 0xBF58476D1CE4E5B9ULL
#define MIX_B 0x94D049BB133111EBULL

static inline uint64_t mix64(uint64_t z) {
    z += GOLDEN;
    z = (z ^ (z >> 30)) * MIX_A;
    z = (z ^ (z >> 27)) * MIX_B;
    return z ^ (z >> 31);
}

uint64_t oracle_mix64(uint64_t z) { return mix64(z); }

/* engine.fold_seed (engine.py:53-56): mix64(seed + index), wrapping. */
uint64_t oracle_fold_seed(uint64_t seed, uint64_t index) { return mix64(seed + index); }

/* engine.sample_projection (engine.py:79-99) restricted to columns
 * [col0, col0+w) of an n x d_global block; out is n x w row-major. */
int oracle_sample_projection(int64_t n, int64_t d_global, uint64_t seed, int64_t col0,
                             int64_t w, double *out) {
    if (n < 1 || d_global < 1 || col0 < 0 || w < 0 || col0 + w > d_global) return 1;
    const uint64_t key = mix64(seed);
    const double scale = 1.0 / sqrt((double)d_global);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t c = 0; c < w; ++c) {
            uint64_t h = mix64(((uint64_t)i * (uint64_t)d_global + (uint64_t)(col0 + c)) ^ key);
            out[i * w + c] = (h >> 63) ? scale : -scale;
        }
    }
    return 0;
}

/* Y = S X, X is n_cols x w, Y is n_rows x w (row-major).  csr_matvecs order. */
int oracle_spmm(int64_t n_rows, const int64_t *row_offsets, const int64_t *col_indices,
                const double *values, const double *X, int64_t w, double *Y) {
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < n_rows; ++i) {
        double *y = Y + i * w;
        for (int64_t k = 0; k < w; ++k) y[k] = 0.0;
        for (int64_t jj = row_offsets[i]; jj < row_offsets[i + 1]; ++jj) {
            const double a = values[jj];
            const double *x = X + col_indices[jj] * w;
            for (int64_t k = 0; k < w; ++k) y[k] += a * x[k];
        }
    }
    return 0;
}

static inline uint64_t abs_bits(double v) {
    uint64_t b;
    memcpy(&b, &v, sizeof b);
    return b & 0x7FFFFFFFFFFFFFFFULL;
}

/*
 * One stage of the expansion over an n x w block (engine.py:205-228).
 *   coeffs[0..order]; block (n x w) in; out (n x w) = sum_r coeffs[r] Q(r).
 *   max_abs (optional): order x n_chunks array, n_chunks = ceil(w/32), the
 *   reference's per-chunk max|Q(r)| (NaN propagates as in np.max).
 *   first_bad_r (optional): the r the reference raises DivergenceError at, i.e.
 *   the first non-finite r of the FIRST chunk (in column order) that has one
 *   (serial chunk loop, engine.py:250-252); 0 if none.
 * Work buffers are allocated here.  Returns 0 on success, 2 on allocation failure.
 */
int oracle_run_stage(int64_t n, const int64_t *row_offsets, const int64_t *col_indices,
                     const double *values, const double *coeffs, int order,
                     const double *block, int64_t w, double *out, double *max_abs,
                     int *first_bad_r) {
    const int64_t nw = n * w;
    const int64_t n_chunks = (w + 31) / 32;
    double *q_prev = (double *)malloc(sizeof(double) * (size_t)(nw ? nw : 1));
    double *q_prev2 = (double *)malloc(sizeof(double) * (size_t)(nw ? nw : 1));
    double *q = (double *)malloc(sizeof(double) * (size_t)(nw ? nw : 1));
    uint64_t *peaks = (uint64_t *)calloc((size_t)(n_chunks ? n_chunks : 1), sizeof(uint64_t));
    if (!q_prev || !q_prev2 || !q || !peaks) {
        free(q_prev); free(q_prev2); free(q); free(peaks);
        return 2;
    }
    int *bad = (int *)calloc((size_t)(n_chunks ? n_chunks : 1), sizeof(int));
    const double c0 = coeffs[0];
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < nw; ++t) {
        q_prev[t] = block[t];
        out[t] = c0 * block[t];
    }
    for (int r = 1; r <= order; ++r) {
        const double alpha = 2.0 - 1.0 / (double)r;
        const double beta = 1.0 - 1.0 / (double)r;
        const double theta = coeffs[r];
        oracle_spmm(n, row_offsets, col_indices, values, q_prev, w, q);
        memset(peaks, 0, sizeof(uint64_t) * (size_t)n_chunks);
#pragma omp parallel
        {
            uint64_t *local = (uint64_t *)calloc((size_t)n_chunks, sizeof(uint64_t));
#pragma omp for schedule(static)
            for (int64_t i = 0; i < n; ++i) {
                for (int64_t k = 0; k < w; ++k) {
                    const int64_t t = i * w + k;
                    double v = alpha * q[t];
                    if (r > 1) {
                        const double sub = beta * q_prev2[t];
                        v = v - sub;
                    }
                    q[t] = v;
                    const uint64_t b = abs_bits(v);
                    if (b > local[k >> 5]) local[k >> 5] = b;
                    const double add = theta * v;
                    out[t] = out[t] + add;
                }
            }
#pragma omp critical
            for (int64_t c = 0; c < n_chunks; ++c)
                if (local[c] > peaks[c]) peaks[c] = local[c];
            free(local);
        }
        for (int64_t c = 0; c < n_chunks; ++c) {
            double pk;
            memcpy(&pk, &peaks[c], sizeof pk);
            if (max_abs) max_abs[(int64_t)(r - 1) * n_chunks + c] = pk;
            if (!bad[c] && peaks[c] >= 0x7FF0000000000000ULL) bad[c] = r;
        }
        double *tmp = q_prev2;
        q_prev2 = q_prev;
        q_prev = q;
        q = tmp;
    }
    if (first_bad_r) {
        *first_bad_r = 0;
        for (int64_t c = 0; c < n_chunks; ++c)
            if (bad[c]) { *first_bad_r = bad[c]; break; }
    }
    free(q_prev); free(q_prev2); free(q); free(peaks); free(bad);
    return 0;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
