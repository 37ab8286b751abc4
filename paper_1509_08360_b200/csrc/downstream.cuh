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

#include <climits>

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
__device__ __forceinline__ double np_max0(double v) { return v < 0.0 ? 0.0 : v; }  // keeps NaN and -0.0
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

// block-wide exclusive scan of one value per thread; *total = the block sum
__device__ __forceinline__ double block_excl_scan(double v, double *sh, double &total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double inc = v;
    for (int o = 1; o < 32; o <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) sh[w] = inc;
    __syncthreads();
    if (w == 0) {
        double x = lane < nw ? sh[lane] : 0.0;
        for (int o = 1; o < 32; o <<= 1) {
            const double t = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += t;
        }
        sh[lane] = x;
    }
    __syncthreads();
    const double base = w ? sh[w - 1] : 0.0;
    total = sh[nw - 1];
    __syncthreads();
    return base + inc - v;
}

// ++ pick (cluster.py:53): rng.choice(n, p=closest/total) == first i with
// cumsum(p)[i] / cumsum(p)[-1] > u (verified against numpy's Generator.choice).
// One block: a block scan over the chunk sums finds the chunk, a block scan
// over that chunk's p_i = closest_i / total finds the element (fixed order,
// deterministic; the prefix rounding is not numpy's sequential cumsum).
__global__ void __launch_bounds__(1024) k_km_pick(const double *__restrict__ closest, int64_t n, int64_t chunk,
                                                  const double *__restrict__ part, int64_t m,
                                                  const double *__restrict__ total, double u,
                                                  int64_t *__restrict__ out) {
    __shared__ double sh[32];
    __shared__ long long s_c, s_pick;
    __shared__ double s_base;
    const int t = threadIdx.x, nt = blockDim.x;
    const double tot = *total;
    // chunk level
    const int64_t per = (m + nt - 1) / nt, lo = min(m, (int64_t)t * per), hi = min(m, lo + per);
    double loc = 0.0;
    for (int64_t c = lo; c < hi; ++c) loc += part[c];
    double T;
    const double ex = block_excl_scan(loc, sh, T);
    if (t == 0) s_c = m, s_pick = LLONG_MAX;
    __syncthreads();
    double run = ex;
    for (int64_t c = lo; c < hi; ++c) {
        if ((run + part[c]) / T > u) {
            atomicMin(&s_c, (long long)c);
            break;
        }
        run += part[c];
    }
    __syncthreads();
    int64_t c0 = s_c < m ? s_c : m - 1;
    if (c0 >= lo && c0 < hi) {  // the owner of chunk c0 knows the prefix before it
        double b = ex;
        for (int64_t c = lo; c < c0; ++c) b += part[c];
        s_base = b;
    }
    __syncthreads();
    double base = s_base;
    // element level, from chunk c0 on (later chunks only if rounding moved the crossing)
    for (int64_t c = c0; c < m; ++c) {
        const int64_t elo = c * chunk, ehi = min(n, elo + chunk);
        const int64_t eper = (ehi - elo + nt - 1) / nt;
        const int64_t a = min(ehi, elo + (int64_t)t * eper), z = min(ehi, a + eper);
        double ls = 0.0;
        for (int64_t i = a; i < z; ++i) ls += closest[i] / tot;
        double ct;
        double r = base + block_excl_scan(ls, sh, ct);
        for (int64_t i = a; i < z; ++i) {
            const double p = closest[i] / tot;
            r += p;
            if (p > 0.0 && r / T > u) {
                atomicMin(&s_pick, (long long)i);
                break;
            }
        }
        __syncthreads();
        if (s_pick != LLONG_MAX) break;
        base += ct;
    }
    if (t == 0) {
        int64_t pick = s_pick;
        if (pick == LLONG_MAX) {  // u above the rounded total: the last positive entry
            pick = 0;
            for (int64_t i = n - 1; i >= 0; --i)
                if (closest[i] > 0.0) {
                    pick = i;
                    break;
                }
        }
        *out = pick;
    }
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
// k_km_assign (d <= 128, one pairwise leaf).  One 512-thread CTA per SM; a
// CTA step covers 64 rows x 16 centroids.  Warp w owns 16 rows (4 row quads,
// one per 8-lane group) x one centroid quartet; lane j of a group is residue
// class j of numpy's 8-accumulator pairwise sum, so after the body three
// xor-shuffles (tree8) and the in-order d % 8 tail give x.c with exactly
// np.sum(x*c)'s rounding.  Shared memory holds rows and centroids
// residue-major -- element c at [c % 8][c / 8], residue length padded to
// 2 mod 4 (conflict-free 16-byte reads, two body steps per load) -- with the
// row tiles double-buffered through cp.async and the centroids staged once
// per CTA when they fit (CFULL).  Quartets past K are skipped (warp-uniform).
// Each thread keeps its rows' running minimum over its quartets in ascending k
// (strict <: np.argmin's first minimum); the four quartet warps of a row merge
// once per row tile through shared memory.  The 8 residue lanes reduce by a
// transpose-reduce in numpy's tree order, leaving each lane 2 finished dot
// products, so the tail, the d2 epilogue and the argmin run once per (row,
// centroid) pair rather than once per lane.  Epilogue: label / min-distance
// store, #changed vs the previous labels, per-cluster counts.
// ---------------------------------------------------------------------------
constexpr int KA_TM = 64, KA_TK = 16, KA_THREADS = 512, KA_MAXD = 128;
constexpr int KM_SMEM_K = 16384;  // above this many clusters, counts use global atomics

// 8-byte async copy global -> shared (src_bytes 0 zero-fills), commit / wait
__device__ __forceinline__ void ca8(double *dst, const double *src, int src_bytes) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void ca_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void ca_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// np.argmin order: NaN is smallest (the first NaN wins), then value, then index
__device__ __forceinline__ bool np_before(double v, int k, double bv, int bk) {
    const bool vn = isnan(v), bn = isnan(bv);
    if (vn | bn) return vn && (!bn || k < bk);
    return v < bv || (v == bv && k < bk);
}
__device__ __forceinline__ void lexmin(double &bd, int &bk, double od, int ok) {
    if (np_before(od, ok, bd, bk)) bd = od, bk = ok;
}

// residue-major geometry of one row: body elements c < body at [c % 8][c / 8]
// (residue length tp), tail elements at 8 * tp + (c - body); row stride rs
struct KaGeom {
    int body, tp, rs;
    __host__ __device__ KaGeom(int d) {
        body = d < 8 ? 0 : d - d % 8;
        const int t = body / 8;
        tp = t == 0 ? 0 : (t % 4 == 2 ? t : t + ((2 - t % 4) + 4) % 4);
        rs = 8 * tp + 8;
    }
    __device__ __forceinline__ int pos(int c) const { return c < body ? (c & 7) * tp + (c >> 3) : 8 * tp + (c - body); }
};

template <bool CFULL>
__global__ void __launch_bounds__(KA_THREADS, 1) k_km_assign(
    const double *__restrict__ X, int64_t n, int d, int64_t ld, const double *__restrict__ xx,
    const double *__restrict__ C, int K, int64_t ldc, const double *__restrict__ cc,
    const int *__restrict__ lab_old, int *__restrict__ lab_new, double *__restrict__ mind,
    unsigned long long *__restrict__ counts, unsigned long long *__restrict__ changed) {
    extern __shared__ __align__(16) double sm[];
    const KaGeom G(d);
    const int T = G.body / 8;
    const int Kp = (K + KA_TK - 1) / KA_TK * KA_TK;
    double *Xb = sm;                                 // [2][KA_TM][rs] row tiles
    double *Cs = Xb + 2 * KA_TM * G.rs;              // [CFULL ? Kp : KA_TK][rs]
    double *cand_d = Cs + (CFULL ? Kp : KA_TK) * G.rs;  // [4 quartets][KA_TM]
    int *cand_k = reinterpret_cast<int *>(cand_d + 4 * KA_TM);
    unsigned *s_cnt = reinterpret_cast<unsigned *>(cand_k + 4 * KA_TM);
    const int tid = threadIdx.x, j = tid & 7, w = tid >> 5;
    const int oct = w & 3;                           // centroid quartet within a 16-tile
    const int rq = (w >> 2) * 16 + ((tid >> 3) & 3) * 4;  // this group's 4 rows within the tile
    const int co = oct * 4;

    const bool scnt = K <= KM_SMEM_K;  // per-block shared histogram, else direct global counts
    if (scnt)
        for (int k = tid; k < K; k += KA_THREADS) s_cnt[k] = 0;
    auto stage_c = [&](int k_first, int k_count) {
        for (int t = tid; t < k_count * d; t += KA_THREADS) {
            const int k = t / d, c = t % d;
            Cs[k * G.rs + G.pos(c)] = k_first + k < K ? C[(int64_t)(k_first + k) * ldc + c] : 0.0;
        }
    };
    if (CFULL) stage_c(0, Kp);
    auto stage_x = [&](double *dst, int64_t r0) {
        for (int t = tid; t < KA_TM * d; t += KA_THREADS) {
            const int r = t / d, c = t % d;
            const int64_t gr = r0 + r;
            ca8(dst + r * G.rs + G.pos(c), X + (gr < n ? gr : 0) * ld + c, gr < n ? 8 : 0);
        }
        ca_commit();
    };
    unsigned long long n_changed = 0;
    const int64_t stride = (int64_t)gridDim.x * KA_TM;
    int buf = 0;
    if ((int64_t)blockIdx.x * KA_TM < n) stage_x(Xb, (int64_t)blockIdx.x * KA_TM);

    for (int64_t row0 = (int64_t)blockIdx.x * KA_TM; row0 < n; row0 += stride, buf ^= 1) {
        __syncthreads();  // previous tile consumed (CFULL staging, counters and candidates visible)
        if (row0 + stride < n)
            stage_x(Xb + (buf ^ 1) * KA_TM * G.rs, row0 + stride);
        else
            ca_commit();  // empty group keeps the wait count uniform
        ca_wait<1>();
        __syncthreads();
        const double *xr = Xb + buf * KA_TM * G.rs + rq * G.rs;
        // after the transpose-reduce below, lane j holds row mi = 2 b0 + b1 of
        // its quad and centroids 2 b2 + {0, 1} of its quartet
        const int b0 = j & 1, b1 = (j >> 1) & 1, b2 = (j >> 2) & 1;
        const int mi = 2 * b0 + b1;
        const double xim = row0 + rq + mi < n ? xx[row0 + rq + mi] : 0.0;
        double bd = CUDART_INF;
        int bk = INT32_MAX;

        for (int k0 = 0; k0 < K; k0 += KA_TK) {
            const double *Ct = Cs;
            if (!CFULL) {
                __syncthreads();
                stage_c(k0, KA_TK);
                __syncthreads();
            } else {
                Ct = Cs + (int64_t)k0 * G.rs;
            }
            if (k0 + co >= K) continue;  // whole quartet past K (warp-uniform)
            const double *cr = Ct + co * G.rs;
            double dot[2];
            if (T > 0) {
                // lane-permuted slots: row slot i holds row i ^ mi, centroid slot q holds
                // q ^ 2 b2, so the transpose-reduce below keeps fixed registers (no
                // lane-dependent selects) and partners' halves line up slot for slot
                double acc[4][4];
                const double *xs[4], *cs[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) xs[i] = xr + (i ^ mi) * G.rs + j * G.tp;
#pragma unroll
                for (int q = 0; q < 4; ++q) cs[q] = cr + (q ^ (2 * b2)) * G.rs + j * G.tp;
                {
                    double2 xv[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) xv[i] = *reinterpret_cast<const double2 *>(xs[i]);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const double2 cv = *reinterpret_cast<const double2 *>(cs[q]);
#pragma unroll
                        for (int i = 0; i < 4; ++i) acc[i][q] = __dmul_rn(xv[i].x, cv.x);
                    }
                    if (T > 1) {
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const double cy = cs[q][1];
#pragma unroll
                            for (int i = 0; i < 4; ++i) acc[i][q] = __dadd_rn(acc[i][q], __dmul_rn(xv[i].y, cy));
                        }
                    }
                }
                int t = 2;
                for (; t + 1 < T; t += 2) {
                    double2 xv[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) xv[i] = *reinterpret_cast<const double2 *>(xs[i] + t);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const double2 cv = *reinterpret_cast<const double2 *>(cs[q] + t);
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            acc[i][q] = __dadd_rn(acc[i][q], __dmul_rn(xv[i].x, cv.x));
                            acc[i][q] = __dadd_rn(acc[i][q], __dmul_rn(xv[i].y, cv.y));
                        }
                    }
                }
                if (t < T) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const double cx = cs[q][t];
#pragma unroll
                        for (int i = 0; i < 4; ++i) acc[i][q] = __dadd_rn(acc[i][q], __dmul_rn(xs[i][t], cx));
                    }
                }
                // transpose-reduce over the 8 residue lanes in numpy's tree order
                // (xor 1, 2, 4 = (r0+r1), (r01+r23), (r0123+r4567)): keep slots 0..half-1,
                // send the rest; the partner holds the same pairs in those slots
                double r1[8], r2[4];
#pragma unroll
                for (int e = 0; e < 8; ++e)  // slots (i, q) = (e >> 2, e & 3) kept, (2 + (e >> 2), e & 3) sent
                    r1[e] = __dadd_rn(acc[e >> 2][e & 3], __shfl_xor_sync(0xffffffffu, acc[2 + (e >> 2)][e & 3], 1));
#pragma unroll
                for (int e = 0; e < 4; ++e)  // row slot 0 kept, 1 sent
                    r2[e] = __dadd_rn(r1[e], __shfl_xor_sync(0xffffffffu, r1[4 + e], 2));
#pragma unroll
                for (int e = 0; e < 2; ++e)  // centroid slots 0, 1 kept, 2, 3 sent
                    dot[e] = __dadd_rn(r2[e], __shfl_xor_sync(0xffffffffu, r2[2 + e], 4));
            } else {
                dot[0] = dot[1] = -0.0;  // numpy: rows shorter than 8 sum from -0.0
            }
            const double *xm = xr + mi * G.rs;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int q = 2 * b2 + e;
                for (int c = G.body; c < d; ++c) {  // tail, in order
                    const int pc = 8 * G.tp + (c - G.body);
                    dot[e] = __dadd_rn(dot[e], __dmul_rn(xm[pc], cr[q * G.rs + pc]));
                }
                const int k = k0 + co + q;
                if (k < K) {
                    double v = __dsub_rn(__dadd_rn(xim, cc[k]), __dadd_rn(dot[e], dot[e]));
                    v = v < 0.0 ? 0.0 : v;  // np.maximum(v, 0.0): keeps NaN and -0.0
                    if (v < bd || (isnan(v) && !isnan(bd))) bd = v, bk = k;  // ascending k: np.argmin
                }
            }
        }
        // lanes j and j^4 share a row (different centroid pairs)
        lexmin(bd, bk, __shfl_xor_sync(0xffffffffu, bd, 4), __shfl_xor_sync(0xffffffffu, bk, 4));
        if (b2 == 0) cand_d[oct * KA_TM + rq + mi] = bd, cand_k[oct * KA_TM + rq + mi] = bk;

        // merge the four quartet warps of each row (lexicographic (d2, k): first minimum)
        __syncthreads();
        if (tid < KA_TM) {
            const int64_t row = row0 + tid;
            double v = cand_d[tid];
            int k = cand_k[tid];
#pragma unroll
            for (int o = 1; o < 4; ++o) lexmin(v, k, cand_d[o * KA_TM + tid], cand_k[o * KA_TM + tid]);
            if (row < n) {
                if (k == INT32_MAX) k = 0;  // all distances NaN: np.argmin returns 0
                n_changed += lab_old[row] != k;
                lab_new[row] = k;
                mind[row] = v;
                if (scnt)
                    atomicAdd(&s_cnt[k], 1u);
                else
                    atomicAdd(&counts[k], 1ull);
            }
        }
    }
    for (int o = 16; o; o >>= 1) n_changed += __shfl_xor_sync(0xffffffffu, n_changed, o);
    if ((tid & 31) == 0 && n_changed) atomicAdd(changed, n_changed);
    __syncthreads();
    if (scnt)
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
    const int64_t lo = (int64_t)blockIdx.x * seg, hi = min(n, lo + seg);
    int64_t *row = seg_off + (int64_t)blockIdx.x * K;
    if (K > KM_SMEM_K) {  // large K: count straight into this segment's row
        for (int k = threadIdx.x; k < K; k += blockDim.x) row[k] = 0;
        __syncthreads();
        for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x)
            atomicAdd(reinterpret_cast<unsigned long long *>(row + lab[i]), 1ull);
        return;
    }
    for (int k = threadIdx.x; k < K; k += blockDim.x) s_h[k] = 0;
    __syncthreads();
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) atomicAdd(&s_h[lab[i]], 1u);
    __syncthreads();
    for (int k = threadIdx.x; k < K; k += blockDim.x) row[k] = s_h[k];
}

// seg_off[s][k] <- sum_{s' < s} count[s'][k] (one warp per label, shuffle scan
// over 32 segments at a time); tot[k] = the label's row count
__global__ void __launch_bounds__(256) k_km_seg_scan(int64_t *__restrict__ seg_off, int64_t nseg, int K,
                                                     int64_t *__restrict__ tot) {
    const int lane = threadIdx.x & 31;
    const int k = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (k >= K) return;
    int64_t run = 0;
    for (int64_t s0 = 0; s0 < nseg; s0 += 32) {
        const int64_t s = s0 + lane;
        const int64_t c = s < nseg ? seg_off[s * K + k] : 0;
        int64_t inc = c;
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
        }
        if (s < nseg) seg_off[s * K + k] = run + inc - c;
        run += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) tot[k] = run;
}

// start[0] = 0, start[k + 1] = start[k] + tot[k] (one block; thread t owns a
// contiguous run of labels)
__global__ void __launch_bounds__(1024) k_km_start_scan(const int64_t *__restrict__ tot, int K,
                                                        int64_t *__restrict__ start) {
    __shared__ int64_t part[1024];
    const int per = (K + blockDim.x - 1) / blockDim.x;
    const int lo = min(K, (int)threadIdx.x * per), hi = min(K, lo + per);
    int64_t s = 0;
    for (int k = lo; k < hi; ++k) s += tot[k];
    part[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t run = 0;
        for (int t = 0; t < (int)blockDim.x; ++t) {
            const int64_t v = part[t];
            part[t] = run;
            run += v;
        }
        start[K] = run;
    }
    __syncthreads();
    int64_t run = part[threadIdx.x];
    for (int k = lo; k < hi; ++k) {
        start[k] = run;
        run += tot[k];
    }
}

__global__ void k_km_seg_scatter(const int *__restrict__ lab, int64_t n, int K, int64_t seg,
                                 int64_t *__restrict__ seg_off, const int64_t *__restrict__ start,
                                 int64_t *__restrict__ order) {
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
        if (live) order[start[l] + off[l] + rank] = i;
        __syncwarp();
        if (live && rank == 0) off[l] += __popc(peers);
        __syncwarp();
    }
}

// C[k][col] = (sum over the cluster's rows in row order) / count   (cluster.py:98-100).
// One warp (block) per (cluster, 32-column slice), lane = column.  The adds are
// a sequential chain in row order, so the rows are streamed ahead through a
// per-warp ring of KS_D 32-row batches in shared memory (8-byte cp.async per
// lane and row, zero-filled past the cluster / the row width); row indices
// are loaded one batch ahead of their copies.
constexpr int KS_D = 8;

__global__ void __launch_bounds__(32) k_km_sums(const double *__restrict__ X, int d, int64_t ld,
                                                const int64_t *__restrict__ order, const int64_t *__restrict__ start,
                                                int K, double *__restrict__ C, int64_t ldc) {
    extern __shared__ double ring[];  // [KS_D][32 rows][32 lanes]
    const int lane = threadIdx.x;
    const int slices = (d + 31) / 32;
    const int k = blockIdx.x / slices;
    const int col = (blockIdx.x % slices) * 32 + lane;
    const bool live = col < d;
    const int64_t b = start[k], e = start[k + 1];
    const int64_t nb = (e - b + 31) / 32;
    auto index_of = [&](int64_t bi) -> int64_t {
        const int64_t j = b + bi * 32 + lane;
        return (bi < nb && j < e) ? order[j] : 0;
    };
    auto issue = [&](int64_t bi, int64_t my) {
        if (bi < nb) {
            const int cnt = (int)min((int64_t)32, e - (b + bi * 32));
            double *slot = ring + (bi % KS_D) * 1024;
#pragma unroll 8
            for (int t = 0; t < 32; ++t) {
                const int64_t r = __shfl_sync(0xffffffffu, my, t);
                ca8(slot + t * 32 + lane, X + r * ld + (live ? col : 0), (live && t < cnt) ? 8 : 0);
            }
        }
        ca_commit();  // possibly empty: one group per batch slot keeps the wait count uniform
    };
    for (int bi = 0; bi < KS_D - 1; ++bi) issue(bi, index_of(bi));
    int64_t my_next = index_of(KS_D - 1);
    double acc = 0.0;
    for (int64_t bi = 0; bi < nb; ++bi) {
        const int64_t my = my_next;
        my_next = index_of(bi + KS_D);
        issue(bi + KS_D - 1, my);
        ca_wait<KS_D - 1>();
        __syncwarp();
        const int cnt = (int)min((int64_t)32, e - (b + bi * 32));
        const double *slot = ring + (bi % KS_D) * 1024;
        for (int t = 0; t < cnt; ++t) acc = __dadd_rn(acc, slot[t * 32 + lane]);
        __syncwarp();  // slot free for batch bi + KS_D
    }
    ca_wait<0>();
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
                                                    unsigned long long *__restrict__ degsum,
                                                    unsigned long long *__restrict__ bad) {
    extern __shared__ unsigned long long s_m[];  // [K] intra2, [K] degsum
    if (SMEM_HIST) {
        for (int k = threadIdx.x; k < 2 * K; k += blockDim.x) s_m[k] = 0;
        __syncthreads();
    }
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int l = lab[i];
        if (l < 0 || l >= K) {  // caller-supplied device labels: flag, never index out of range
            atomicAdd(bad, 1ull);
            continue;
        }
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
