// downstream.cuh -- sm_100a kernels for the consumers of an embedding
// (reference cluster.py:34-128, oracle.py:88-119), SURVEY 8(f) rank 4.
//
// K5  k_pair_cos       cosine of sampled row pairs          _pair_correlations (oracle.py:88-96)
// K6  k_sqnorm_rows    squared row norms, numpy's order     np.sum(X*X, axis=1) (cluster.py:36-37)
// K7  k_km_dist1       distance to one new centroid and     _plus_plus_init (cluster.py:43-56)
//                      the running minimum
// K8  k_km_assign      fused distance GEMM + argmin         kmeans Lloyd step (cluster.py:74-77)
// K9  k_km_seg_*       stable counting sort of rows by      np.add.at(sums, labels, rows)
//     k_km_sums        label, then per-cluster sums in       (cluster.py:98-100)
//                      row order (bit-identical to np.add.at)
// K10 k_modularity     intra-cluster edge and degree        modularity (cluster.py:110-128)
//                      counts over the CSR pattern
// plus fixed-order reductions (sum, first-argmax, weighted pick) so every
// result is deterministic run to run.
//
// Rounding notes.  Row squared norms follow numpy's pairwise summation exactly
// (8 interleaved accumulators for blocks <= 128, recursive halving above; see
// pw_dot8), so xx / ||x|| are bit-identical to the reference.  Dot products use
// the same order with separately rounded products, so x.x == np.sum(x*x) and a
// point's distance to an identical centroid is exactly 0 (the reference's
// ++ seeding and empty-cluster logic branch on such zeros).  The reference
// takes its dot products from BLAS (X @ C.T, einsum), whose order is not
// specified, so general distances and cosines agree to a few ulps.  Centroid
// sums are sequential in row order from +0.0 with separately rounded adds:
// bit-identical to np.add.at given the same labels.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

namespace csemb {

// ---------------------------------------------------------------------------
// numpy pairwise sum of the products a[i]*b[i] (b == a: np.sum(x*x)), computed
// by the 8 lanes of an aligned group.  numpy (loops_utils.h pairwise_sum):
// n < 8 -> sequential from -0.0; n <= 128 -> r[j] = p[j], r[j] += p[i + j]
// for i = 8, 16, .. < n - n % 8, ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 +
// r7)), then the n % 8 tail in order; n > 128 -> n2 = n / 2 - (n / 2) % 8,
// sum(p[:n2]) + sum(p[n2:]).  Products are rounded before the adds (numpy
// forms x*c first).  Every lane of the group returns the same value.
// ---------------------------------------------------------------------------
template <typename TA, typename TB>
__device__ __forceinline__ double prod_of(const TA *a, const TB *b, int64_t i) {
    return __dmul_rn((double)a[i], (double)b[i]);
}

__device__ __forceinline__ double tree8(double r) {
    // the shuffles pair lanes (j, j^1), (j, j^2), (j, j^4); IEEE addition is
    // commutative, so every lane ends with numpy's ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
    return __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
}

template <typename TA, typename TB>
__device__ __forceinline__ double pw_leaf8(const TA *a, const TB *b, int n, int j) {
    if (n < 8) {
        double res = -0.0;
        for (int i = 0; i < n; ++i) res = __dadd_rn(res, prod_of(a, b, i));
        return res;
    }
    const int body = n - (n % 8);
    double r = prod_of(a, b, j);
    for (int i = 8; i < body; i += 8) r = __dadd_rn(r, prod_of(a, b, i + j));
    r = tree8(r);
    for (int i = body; i < n; ++i) r = __dadd_rn(r, prod_of(a, b, i));
    return r;
}

template <typename TA, typename TB>
__device__ __noinline__ double pw_split8(const TA *a, const TB *b, int n, int j) {  // n > 128
    int n2 = n / 2;
    n2 -= n2 % 8;
    const double lo = n2 <= 128 ? pw_leaf8(a, b, n2, j) : pw_split8(a, b, n2, j);
    const double hi = n - n2 <= 128 ? pw_leaf8(a + n2, b + n2, n - n2, j) : pw_split8(a + n2, b + n2, n - n2, j);
    return __dadd_rn(lo, hi);
}

template <typename TA, typename TB>
__device__ __forceinline__ double pw_dot8(const TA *a, const TB *b, int n, int j) {
    return n <= 128 ? pw_leaf8(a, b, n, j) : pw_split8(a, b, n, j);
}

template <typename T>
__device__ __forceinline__ double sumsq_group8(const T *a, int n, int j) {
    return pw_dot8(a, a, n, j);
}

// np.maximum(d2, 0.0) / np.minimum(a, b) semantics: (a >= b || isnan(a)) ? a : b
__device__ __forceinline__ double np_max0(double v) { return (v >= 0.0 || isnan(v)) ? v : 0.0; }
__device__ __forceinline__ double np_min(double a, double b) { return (a <= b || isnan(a)) ? a : b; }

// ---------------------------------------------------------------------------
// K5: cosines of row pairs (oracle.py:88-96).  norms = sqrt(np.sum(x*x)) in
// numpy's order; denom = |a| |b|; zero denominators give 0 and set zero[p].
// One 8-lane group per pair, 4 pairs per warp, grid-stride.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) k_pair_cos(const T *__restrict__ E, int d, int64_t ld,
                                                  const int64_t *__restrict__ pairs, int64_t n_pairs,
                                                  double *__restrict__ out, uint8_t *__restrict__ zero) {
    const int j = threadIdx.x & 7;
    const int64_t groups = (int64_t)gridDim.x * (blockDim.x / 8);
    for (int64_t base = (int64_t)blockIdx.x * (blockDim.x / 8); base < n_pairs; base += groups) {
        // the whole warp iterates together (shuffles need full participation)
        const int64_t p = base + (threadIdx.x >> 3);
        const bool live = p < n_pairs;
        const int64_t pa = live ? pairs[2 * p] : 0, pb = live ? pairs[2 * p + 1] : 0;
        const T *a = E + pa * ld, *b = E + pb * ld;
        const double na = sqrt(sumsq_group8(a, d, j));
        const double nb = sqrt(sumsq_group8(b, d, j));
        const double dot = pw_dot8(a, b, d, j);
        const double den = na * nb;
        if (live && j == 0) {
            const bool z = den == 0.0;
            out[p] = z ? 0.0 : dot / den;
            if (zero) zero[p] = z ? 1 : 0;
        }
    }
}

// K6: out[i] = np.sum(X[i]*X[i]) in numpy's order (one 8-lane group per row)
template <typename T>
__global__ void __launch_bounds__(256) k_sqnorm_rows(const T *__restrict__ X, int64_t n, int d, int64_t ld,
                                                     double *__restrict__ out) {
    const int j = threadIdx.x & 7;
    const int64_t groups = (int64_t)gridDim.x * (blockDim.x / 8);
    for (int64_t base = (int64_t)blockIdx.x * (blockDim.x / 8); base < n; base += groups) {
        const int64_t i = base + (threadIdx.x >> 3);
        const bool live = i < n;
        const double s = sumsq_group8(X + (live ? i : 0) * ld, d, j);
        if (live && j == 0) out[i] = s;
    }
}

// K7: d2 = max((xx + cc) - 2 x.c, 0) to the centroid `c`; closest = d2 (first)
// or np.minimum(closest, d2) (cluster.py:47, 55)
__global__ void __launch_bounds__(256) k_km_dist1(const double *__restrict__ X, int64_t n, int d, int64_t ld,
                                                  const double *__restrict__ xx, const double *__restrict__ c,
                                                  const double *__restrict__ cc, double *__restrict__ closest,
                                                  int first) {
    const int j = threadIdx.x & 7;
    const double ccv = *cc;
    const int64_t groups = (int64_t)gridDim.x * (blockDim.x / 8);
    for (int64_t base = (int64_t)blockIdx.x * (blockDim.x / 8); base < n; base += groups) {
        const int64_t i = base + (threadIdx.x >> 3);
        const bool live = i < n;
        const double dot = pw_dot8(X + (live ? i : 0) * ld, c, d, j);
        if (live && j == 0) {
            const double d2 = np_max0(__dsub_rn(__dadd_rn(xx[i], ccv), 2.0 * dot));
            closest[i] = first ? d2 : np_min(closest[i], d2);
        }
    }
}

// ---------------------------------------------------------------------------
// Fixed-order reductions (deterministic for a given n; the grid size is a
// function of n only).
// ---------------------------------------------------------------------------
constexpr int RED_THREADS = 256;

__device__ __forceinline__ double block_sum(double v, double *sh) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x < 32) {
        t = threadIdx.x < blockDim.x / 32 ? sh[threadIdx.x] : 0.0;
        for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    }
    __syncthreads();
    return t;  // valid in thread 0
}

// part[b] = sum over the elements b*chunk .. (b+1)*chunk of v[i] * scale
// (scale = 1 / total for the ++ pick: p_i = closest_i / total, cluster.py:53)
__global__ void __launch_bounds__(RED_THREADS) k_chunk_sums(const double *__restrict__ v, int64_t n, int64_t chunk,
                                                            const double *__restrict__ divisor,
                                                            double *__restrict__ part) {
    __shared__ double sh[32];
    const int64_t lo = (int64_t)blockIdx.x * chunk, hi = min(n, lo + chunk);
    const double dv = divisor ? *divisor : 1.0;
    double s = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) s += divisor ? v[i] / dv : v[i];
    s = block_sum(s, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void k_sum_final(const double *__restrict__ part, int64_t m, double *__restrict__ out) {
    __shared__ double sh[32];
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) s += part[i];
    s = block_sum(s, sh);
    if (threadIdx.x == 0) *out = s;
}

// ++ pick (cluster.py:53): rng.choice(n, p=closest/total) == first i with
// cumsum(p)[i] / cumsum(p)[-1] > u (verified against numpy's Generator.choice).
// Chunk sums locate the chunk; the element scan is sequential from there.
__global__ void k_km_pick(const double *__restrict__ closest, int64_t n, int64_t chunk,
                          const double *__restrict__ part, int64_t m, const double *__restrict__ total, double u,
                          int64_t *__restrict__ out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double T = 0.0;
    for (int64_t c = 0; c < m; ++c) T += part[c];
    const double tot = *total;
    double s = 0.0;
    int64_t c = 0;
    for (; c < m; ++c) {
        if ((s + part[c]) / T > u) break;
        s += part[c];
    }
    if (c == m) c = m - 1, s -= part[m - 1];
    int64_t pick = -1, last_pos = -1;
    for (int64_t i = c * chunk; i < n; ++i) {
        const double p = closest[i] / tot;
        if (p > 0.0) last_pos = i;
        s += p;
        if (s / T > u && p > 0.0) {
            pick = i;
            break;
        }
    }
    if (pick < 0) {  // rounding left u above the scanned total: last positive entry
        if (last_pos < 0)
            for (int64_t i = c * chunk - 1; i >= 0; --i)
                if (closest[i] > 0.0) {
                    last_pos = i;
                    break;
                }
        pick = last_pos < 0 ? 0 : last_pos;
    }
    *out = pick;
}

// first index of the maximum (np.argmax) -- two stages: per block, then final
__device__ __forceinline__ void argmax_merge(double &v, int64_t &i, double ov, int64_t oi) {
    if (ov > v || (ov == v && oi < i)) v = ov, i = oi;
}

__global__ void __launch_bounds__(RED_THREADS) k_argmax_part(const double *__restrict__ v, int64_t n, int64_t chunk,
                                                             double *__restrict__ pv, int64_t *__restrict__ pi) {
    __shared__ double sv[32];
    __shared__ int64_t si[32];
    const int64_t lo = (int64_t)blockIdx.x * chunk, hi = min(n, lo + chunk);
    double bv = -CUDART_INF;
    int64_t bi = INT64_MAX;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) argmax_merge(bv, bi, v[i], i);
    for (int o = 16; o; o >>= 1)
        argmax_merge(bv, bi, __shfl_xor_sync(0xffffffffu, bv, o), __shfl_xor_sync(0xffffffffu, bi, o));
    if ((threadIdx.x & 31) == 0) sv[threadIdx.x >> 5] = bv, si[threadIdx.x >> 5] = bi;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x / 32); ++w) argmax_merge(bv, bi, sv[w], si[w]);
        pv[blockIdx.x] = bv, pi[blockIdx.x] = bi;
    }
}

// empty-cluster re-seed (cluster.py:85-90): far = argmax(avail);
// centroid c = X[far]; new_labels[far] = c; avail[far] = -1
__global__ void k_km_reseed(const double *__restrict__ pv, const int64_t *__restrict__ pi, int64_t m,
                            const double *__restrict__ X, int d, int64_t ld, double *__restrict__ C, int64_t ldc,
                            int c, int *__restrict__ lab_new, double *__restrict__ avail,
                            int64_t *__restrict__ out_far) {
    __shared__ int64_t s_far;
    if (threadIdx.x == 0) {
        double bv = -CUDART_INF;
        int64_t bi = INT64_MAX;
        for (int64_t b = 0; b < m; ++b) argmax_merge(bv, bi, pv[b], pi[b]);
        if (bi == INT64_MAX) bi = 0;  // all -inf/NaN: numpy would return 0 as well
        s_far = bi;
    }
    __syncthreads();
    const int64_t far = s_far;
    for (int k = threadIdx.x; k < d; k += blockDim.x) C[(int64_t)c * ldc + k] = X[far * ld + k];
    if (threadIdx.x == 0) {
        lab_new[far] = c;
        avail[far] = -1.0;
        *out_far = far;
    }
}

// ---------------------------------------------------------------------------
// K8: Lloyd assignment (cluster.py:74-77): labels = argmin_k d2, mindist,
// with d2 = max((xx + cc) - 2 x.c, 0) (cluster.py:34-40).
//
// k_km_assign (d <= 128, one pairwise leaf): CTA tile of 32 rows x 32
// centroids; the rows of the tile and the centroids (all of them when they
// fit, CFULL, else one 32-centroid tile at a time) are staged in shared memory
// with an odd row stride.  8-lane group g of the CTA owns a 4-row x 8-centroid
// micro-tile; lane j of the group is residue class j of numpy's 8-accumulator
// sum, so after the body three xor-shuffles (tree8) and the in-order d % 8
// tail give x.c with exactly np.sum(x*c)'s rounding.  The 4 groups of a warp
// share the row quad and cover the tile's 32 centroids; the running
// lexicographic (d2, k) minimum is np.argmin's first-minimum rule.  Epilogue:
// label / min-distance store, #changed vs the previous labels, per-cluster
// counts (shared histogram, one atomic per cluster per block).
// ---------------------------------------------------------------------------
constexpr int KA_TM = 32, KA_TK = 32, KA_THREADS = 256, KA_MAXD = 128;

__device__ __forceinline__ void lexmin(double &bd, int &bk, double od, int ok) {
    if (od < bd || (od == bd && ok < bk)) bd = od, bk = ok;
}

template <bool CFULL>
__global__ void __launch_bounds__(KA_THREADS) k_km_assign(
    const double *__restrict__ X, int64_t n, int d, int64_t ld, const double *__restrict__ xx,
    const double *__restrict__ C, int K, int64_t ldc, const double *__restrict__ cc,
    const int *__restrict__ lab_old, int *__restrict__ lab_new, double *__restrict__ mind,
    unsigned long long *__restrict__ counts, unsigned long long *__restrict__ changed) {
    extern __shared__ __align__(16) double sm[];
    const int dp = d | 1;                      // odd stride: 4 centroid rows hit 2 bank halves
    const int Kp = (K + KA_TK - 1) / KA_TK * KA_TK;
    double *Xs = sm;                           // [KA_TM][dp]
    double *Cs = Xs + KA_TM * dp;              // [CFULL ? Kp : KA_TK][dp]
    unsigned *s_cnt = reinterpret_cast<unsigned *>(Cs + (CFULL ? Kp : KA_TK) * dp);
    const int tid = threadIdx.x, j = tid & 7, g = tid >> 3;
    const int rq = (g >> 2) * 4;               // this group's 4 rows within the tile
    const int co = (g & 3) * 8;                // this group's 8 centroids within the tile
    const int body = d < 8 ? 0 : d - (d % 8);

    for (int k = tid; k < K; k += KA_THREADS) s_cnt[k] = 0;
    if (CFULL) {
        for (int64_t t = tid; t < (int64_t)Kp * d; t += KA_THREADS) {
            const int k = (int)(t / d), c = (int)(t % d);
            Cs[k * dp + c] = k < K ? C[(int64_t)k * ldc + c] : 0.0;
        }
    }
    unsigned long long n_changed = 0;

    for (int64_t row0 = (int64_t)blockIdx.x * KA_TM; row0 < n; row0 += (int64_t)gridDim.x * KA_TM) {
        __syncthreads();  // previous tile consumed (and CFULL staging / counters visible)
        for (int t = tid; t < KA_TM * d; t += KA_THREADS) {
            const int r = t / d, c = t % d;
            const int64_t gr = row0 + r;
            Xs[r * dp + c] = gr < n ? X[gr * ld + c] : 0.0;
        }
        double bd[4];
        int bk[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) bd[i] = CUDART_INF, bk[i] = INT32_MAX;

        for (int k0 = 0; k0 < K; k0 += KA_TK) {
            const double *Ct = Cs;
            if (!CFULL) {
                __syncthreads();
                for (int t = tid; t < KA_TK * d; t += KA_THREADS) {
                    const int k = t / d, c = t % d;
                    Cs[k * dp + c] = k0 + k < K ? C[(int64_t)(k0 + k) * ldc + c] : 0.0;
                }
            } else {
                Ct = Cs + (int64_t)k0 * dp;
            }
            __syncthreads();
            const double *xr = Xs + rq * dp;
            const double *cr = Ct + co * dp;
            double acc[4][8];
            if (d >= 8) {
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int q = 0; q < 8; ++q) acc[i][q] = __dmul_rn(xr[i * dp + j], cr[q * dp + j]);
                for (int c = 8 + j; c < body; c += 8) {
                    double xv[4], cv[8];
#pragma unroll
                    for (int i = 0; i < 4; ++i) xv[i] = xr[i * dp + c];
#pragma unroll
                    for (int q = 0; q < 8; ++q) cv[q] = cr[q * dp + c];
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int q = 0; q < 8; ++q) acc[i][q] = __dadd_rn(acc[i][q], __dmul_rn(xv[i], cv[q]));
                }
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int q = 0; q < 8; ++q) acc[i][q] = tree8(acc[i][q]);
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int q = 0; q < 8; ++q) acc[i][q] = -0.0;
            }
            for (int c = body; c < d; ++c) {  // tail, in order (all lanes alike)
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        acc[i][q] = __dadd_rn(acc[i][q], __dmul_rn(xr[i * dp + c], cr[q * dp + c]));
            }
            // epilogue of this centroid tile: every lane of the group holds all 32 dots
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int64_t row = row0 + rq + i;
                const double xi = row < n ? xx[row] : 0.0;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int k = k0 + co + q;
                    if (k < K) lexmin(bd[i], bk[i], np_max0(__dsub_rn(__dadd_rn(xi, cc[k]), 2.0 * acc[i][q])), k);
                }
                // merge the 4 groups of the warp (lane offsets 8 and 16)
                lexmin(bd[i], bk[i], __shfl_xor_sync(0xffffffffu, bd[i], 8), __shfl_xor_sync(0xffffffffu, bk[i], 8));
                lexmin(bd[i], bk[i], __shfl_xor_sync(0xffffffffu, bd[i], 16), __shfl_xor_sync(0xffffffffu, bk[i], 16));
            }
        }
        if ((g & 3) == 0 && j < 4) {  // lane j of the warp's first group writes row rq + j
            double v = bd[0];
            int k = bk[0];
#pragma unroll
            for (int i = 1; i < 4; ++i)
                if (j == i) v = bd[i], k = bk[i];
            const int64_t row = row0 + rq + j;
            if (row < n) {
                if (k == INT32_MAX) k = 0;  // all distances NaN: np.argmin returns 0
                n_changed += lab_old[row] != k;
                lab_new[row] = k;
                mind[row] = v;
                atomicAdd(&s_cnt[k], 1u);
            }
        }
    }
    for (int o = 16; o; o >>= 1) n_changed += __shfl_xor_sync(0xffffffffu, n_changed, o);
    if ((tid & 31) == 0 && n_changed) atomicAdd(changed, n_changed);
    __syncthreads();
    for (int k = tid; k < K; k += KA_THREADS)
        if (s_cnt[k]) atomicAdd(&counts[k], (unsigned long long)s_cnt[k]);
}

// d > 128 (several pairwise leaves): one 8-lane group per row, centroids in
// order, pw_dot8 per centroid -- the same arithmetic as the tiled kernel.
__global__ void __launch_bounds__(256) k_km_assign_wide(
    const double *__restrict__ X, int64_t n, int d, int64_t ld, const double *__restrict__ xx,
    const double *__restrict__ C, int K, int64_t ldc, const double *__restrict__ cc,
    const int *__restrict__ lab_old, int *__restrict__ lab_new, double *__restrict__ mind,
    unsigned long long *__restrict__ counts, unsigned long long *__restrict__ changed) {
    const int j = threadIdx.x & 7;
    const int64_t groups = (int64_t)gridDim.x * (blockDim.x / 8);
    for (int64_t base = (int64_t)blockIdx.x * (blockDim.x / 8); base < n; base += groups) {
        const int64_t i = base + (threadIdx.x >> 3);
        const bool live = i < n;
        const double *x = X + (live ? i : 0) * ld;
        const double xi = xx[live ? i : 0];
        double bd = CUDART_INF;
        int bk = INT32_MAX;
        for (int k = 0; k < K; ++k) {
            const double dot = pw_dot8(x, C + (int64_t)k * ldc, d, j);
            lexmin(bd, bk, np_max0(__dsub_rn(__dadd_rn(xi, cc[k]), 2.0 * dot)), k);
        }
        if (live && j == 0) {
            if (bk == INT32_MAX) bk = 0;
            if (lab_old[i] != bk) atomicAdd(changed, 1ull);
            lab_new[i] = bk;
            mind[i] = bd;
            atomicAdd(&counts[bk], 1ull);
        }
    }
}

// ---------------------------------------------------------------------------
// K9: stable counting sort of rows by label, then per-cluster sums in row
// order.  Segments of `seg` consecutive rows: histogram per segment, an
// exclusive scan over (label, segment), a one-warp-per-segment stable scatter
// (match_any ranks lanes with equal labels), and one warp per (cluster,
// 32-column slice) summing its rows sequentially.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_km_seg_hist(const int *__restrict__ lab, int64_t n, int K, int64_t seg,
                                                     int64_t *__restrict__ seg_off) {
    extern __shared__ unsigned s_h[];
    for (int k = threadIdx.x; k < K; k += blockDim.x) s_h[k] = 0;
    __syncthreads();
    const int64_t lo = (int64_t)blockIdx.x * seg, hi = min(n, lo + seg);
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) atomicAdd(&s_h[lab[i]], 1u);
    __syncthreads();
    for (int k = threadIdx.x; k < K; k += blockDim.x) seg_off[(int64_t)blockIdx.x * K + k] = s_h[k];
}

// seg_off[s][k] <- start[k] + sum_{s' < s} count[s'][k];  start = exclusive scan of totals
__global__ void k_km_seg_scan(int64_t *__restrict__ seg_off, int64_t nseg, int K, int64_t *__restrict__ start) {
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
        int64_t t = 0;
        for (int64_t s = 0; s < nseg; ++s) {
            const int64_t c = seg_off[s * K + k];
            seg_off[s * K + k] = t;
            t += c;
        }
        start[k + 1] = t;  // totals, scanned below
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        start[0] = 0;
        for (int k = 0; k < K; ++k) start[k + 1] += start[k];
    }
    __syncthreads();
    for (int k = threadIdx.x; k < K; k += blockDim.x)
        for (int64_t s = 0; s < nseg; ++s) seg_off[s * K + k] += start[k];
}

__global__ void k_km_seg_scatter(const int *__restrict__ lab, int64_t n, int K, int64_t seg,
                                 int64_t *__restrict__ seg_off, int64_t *__restrict__ order) {
    const int lane = threadIdx.x & 31;
    const int64_t s = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int64_t lo = s * seg, hi = min(n, lo + seg);
    if (lo >= n) return;
    int64_t *off = seg_off + s * K;
    const unsigned lt = (1u << lane) - 1u;
    for (int64_t b = lo; b < hi; b += 32) {
        const int64_t i = b + lane;
        const bool live = i < hi;
        const int l = live ? lab[i] : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, l);
        const int rank = __popc(peers & lt);
        if (live) order[off[l] + rank] = i;
        __syncwarp();
        if (live && rank == 0) off[l] += __popc(peers);
        __syncwarp();
    }
}

// C[k][col] = (sum over the cluster's rows in row order) / count   (cluster.py:98-100)
__global__ void __launch_bounds__(256) k_km_sums(const double *__restrict__ X, int d, int64_t ld,
                                                 const int64_t *__restrict__ order, const int64_t *__restrict__ start,
                                                 int K, double *__restrict__ C, int64_t ldc) {
    const int lane = threadIdx.x & 31;
    const int slices = (d + 31) / 32;
    const int64_t w = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (w >= (int64_t)K * slices) return;
    const int k = (int)(w / slices);
    const int col = (int)(w % slices) * 32 + lane;
    const bool live = col < d;
    const int64_t b = start[k], e = start[k + 1];
    double acc = 0.0;
    for (int64_t j = b; j < e; j += 32) {
        const int cnt = (int)min((int64_t)32, e - j);
        const int64_t my = lane < cnt ? order[j + lane] : 0;
        double v[32];
#pragma unroll
        for (int t = 0; t < 32; ++t) {
            const int64_t r = __shfl_sync(0xffffffffu, my, t);
            v[t] = (live && t < cnt) ? X[r * ld + col] : 0.0;
        }
#pragma unroll
        for (int t = 0; t < 32; ++t)
            if (t < cnt) acc = __dadd_rn(acc, v[t]);
    }
    if (live) C[(int64_t)k * ldc + col] = __ddiv_rn(acc, (double)(e - b));
}

// ---------------------------------------------------------------------------
// K10: modularity counts (cluster.py:110-128) over the symmetric CSR pattern
// of the simple graph (every undirected edge stored twice, no diagonal):
// intra2[c] = stored entries (i, j) with label i == label j == c (2x the
// reference's intra count), degsum[c] = sum of row lengths over c's vertices.
// Integer counts: exact and order-independent.  SMEM_HIST: per-block 64-bit
// shared histograms flushed with one global atomic per label (K <= smem).
// ---------------------------------------------------------------------------
template <bool SMEM_HIST>
__global__ void __launch_bounds__(256) k_modularity(const int64_t *__restrict__ rowptr, const int *__restrict__ cols,
                                                    int64_t n, const int *__restrict__ lab, int K,
                                                    unsigned long long *__restrict__ intra2,
                                                    unsigned long long *__restrict__ degsum) {
    extern __shared__ unsigned long long s_m[];  // [K] intra2, [K] degsum
    if (SMEM_HIST) {
        for (int k = threadIdx.x; k < 2 * K; k += blockDim.x) s_m[k] = 0;
        __syncthreads();
    }
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int l = lab[i];
        const int64_t b = rowptr[i], e = rowptr[i + 1];
        unsigned long long same = 0;
        for (int64_t q = b; q < e; ++q) same += lab[cols[q]] == l;
        unsigned long long *ti = SMEM_HIST ? s_m : intra2, *tg = SMEM_HIST ? s_m + K : degsum;
        if (same) atomicAdd(&ti[l], same);
        if (e > b) atomicAdd(&tg[l], (unsigned long long)(e - b));
    }
    if (SMEM_HIST) {
        __syncthreads();
        for (int k = threadIdx.x; k < K; k += blockDim.x) {
            if (s_m[k]) atomicAdd(&intra2[k], s_m[k]);
            if (s_m[K + k]) atomicAdd(&degsum[k], s_m[K + k]);
        }
    }
}

}  // namespace csemb
