// downstream.cu -- C ABI of the embedding consumers (include/csemb_cuda.h,
// "downstream" section): sampled-pair cosines, k-means primitives and
// modularity counts over the kernels in downstream.cuh.
//
// The reference drives k-means from Python with numpy's Generator
// (cluster.py:59-107); the random draws stay with the caller, so this ABI
// exposes the loop's device steps and the host mirror
// (paper_1509_08360_b200/cluster.py) replays the reference's control flow and
// draw sequence exactly.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "downstream.cuh"
#include "runtime.h"

using namespace csemb;

namespace {

constexpr int64_t RED_CHUNK = 4096;  // elements per partial of the fixed-order reductions

int64_t n_chunks(int64_t n) { return std::max<int64_t>(1, (n + RED_CHUNK - 1) / RED_CHUNK); }

int group8_grid(int64_t rows, int sm) {  // 32 rows (8-lane groups) per 256-thread block
    return grid_for(rows * 8, 256, sm, 16);
}

}  // namespace

struct csemb_kmeans {
    csemb_ctx *ctx = nullptr;
    int64_t n = 0, ld = 0;
    int d = 0, K = 0;
    int64_t ldc = 0;
    double *X = nullptr;        // n x ld owned copy (f64)
    double *xx = nullptr;       // n squared row norms (numpy order)
    double *C = nullptr;        // K x ldc centroids
    double *cc = nullptr;       // K squared centroid norms
    double *closest = nullptr;  // ++ seeding distances
    double *mind = nullptr;     // min distance of the last assignment (then `avail`)
    int *lab = nullptr;         // current labels (-1 before the first commit)
    int *lab_new = nullptr;     // labels of the last assignment
    unsigned long long *counts = nullptr;  // K (+1: changed counter at counts[K])
    double *part = nullptr;     // n_chunks partial sums
    int64_t *part_i = nullptr;  // n_chunks argmax indices; K label totals in commit
    double *scal = nullptr;     // [0] closest total, [1] inertia
    int64_t *pick = nullptr;    // [0] picked / reseeded row
    int64_t *seg_off = nullptr, *order = nullptr, *start = nullptr;
    int64_t seg = 0, nseg = 0;
};

static void km_free(csemb_kmeans *k) {
    if (!k) return;
    for (void *p : {(void *)k->X, (void *)k->xx, (void *)k->C, (void *)k->cc, (void *)k->closest, (void *)k->mind,
                    (void *)k->lab, (void *)k->lab_new, (void *)k->counts, (void *)k->part, (void *)k->part_i,
                    (void *)k->scal, (void *)k->pick, (void *)k->seg_off, (void *)k->order, (void *)k->start})
        dfree(k->ctx, p);
    delete k;
}

// ---------------------------------------------------------------------------
// pair cosines
// ---------------------------------------------------------------------------
extern "C" int csemb_pair_cosines(csemb_ctx *c, const void *E, int dtype, int on_device, int64_t n, int64_t d,
                                  int64_t ld, const int64_t *pairs_host, int64_t n_pairs, double *cos_out,
                                  uint8_t *zero_out) {
    if (!c || (!E && n > 0) || (n_pairs > 0 && (!pairs_host || !cos_out)))
        return fail(CSEMB_ERR_INVALID, "null argument");
    if (n < 0 || d < 1 || ld < d || n_pairs < 0 || d > INT32_MAX) return fail(CSEMB_ERR_INVALID, "bad shape");
    if (dtype != CSEMB_F64 && dtype != CSEMB_F32) return fail(CSEMB_ERR_INVALID, "bad dtype");
    for (int64_t p = 0; p < 2 * n_pairs; ++p)
        if (pairs_host[p] < 0 || pairs_host[p] >= n)
            return fail(CSEMB_ERR_INVALID, "pair index %lld outside [0, %lld)", (long long)pairs_host[p],
                        (long long)n);
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    if (n_pairs == 0) return CSEMB_OK;
    const size_t es = dsize(dtype);
    void *scr = nullptr;
    void *dE = nullptr;
    cudaStream_t s = c->stream;
    cudaError_t e = ctx_scratch(c, 25 * (size_t)n_pairs + 64, &scr);  // pairs, cosines, flags
    int64_t *dp = (int64_t *)scr;
    double *dout = (double *)(dp + 2 * n_pairs);
    uint8_t *dz = (uint8_t *)(dout + n_pairs);
    if (e == cudaSuccess && !on_device) {  // host block: one upload, row stride d
        e = dmalloc(c, &dE, es * n * d);
        if (e == cudaSuccess) e = cudaMemcpy2DAsync(dE, es * d, E, es * ld, es * d, n, cudaMemcpyHostToDevice, s);
    }
    const void *src = on_device ? E : dE;
    const int64_t lds = on_device ? ld : d;
    if (e == cudaSuccess) e = cudaMemcpyAsync(dp, pairs_host, 16 * n_pairs, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) {
        const int g = group8_grid(n_pairs, c->sm_count);
        if (dtype == CSEMB_F64)
            k_pair_cos<double><<<g, 256, 0, s>>>((const double *)src, (int)d, lds, dp, n_pairs, dout, dz);
        else
            k_pair_cos<float><<<g, 256, 0, s>>>((const float *)src, (int)d, lds, dp, n_pairs, dout, dz);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(cos_out, dout, 8 * n_pairs, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && zero_out) e = cudaMemcpyAsync(zero_out, dz, n_pairs, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    dfree(c, dE);
    CK(e);
    return CSEMB_OK;
}

// ---------------------------------------------------------------------------
// k-means
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_to_f64(const T *__restrict__ src, int64_t n, int d, int64_t lds, double *__restrict__ dst,
                         int64_t ldd) {
    const int64_t total = n * (int64_t)d;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / d, k = t % d;
        dst[i * ldd + k] = (double)src[i * lds + k];
    }
}

extern "C" int csemb_kmeans_create(csemb_ctx *c, const void *X, int dtype, int on_device, int64_t n, int64_t d,
                                   int64_t ld, int K, csemb_kmeans **out) {
    if (!c || !out || (!X && n > 0)) return fail(CSEMB_ERR_INVALID, "null argument");
    *out = nullptr;
    if (n < 1 || d < 1 || ld < d || d > INT32_MAX) return fail(CSEMB_ERR_INVALID, "bad block shape");
    if (K < 1 || K > n) return fail(CSEMB_ERR_INVALID, "K=%d must lie in [1, n_rows=%lld]", K, (long long)n);
    if (dtype != CSEMB_F64 && dtype != CSEMB_F32) return fail(CSEMB_ERR_INVALID, "bad dtype");
    if (dtype == CSEMB_F32 && !on_device) return fail(CSEMB_ERR_INVALID, "host blocks must be float64");
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    csemb_kmeans *k = new csemb_kmeans;
    k->ctx = c;
    k->n = n, k->d = (int)d, k->K = K;
    k->ld = (d + 1) / 2 * 2;
    k->ldc = k->ld;
    const int64_t m = n_chunks(n);
    // segments for the counting sort: >= 1024 rows, and nseg * K bounded
    k->seg = std::max<int64_t>(1024, ((n * (int64_t)K) / (1 << 24) + 1) * 32);
    k->nseg = (n + k->seg - 1) / k->seg;
    cudaError_t e = cudaSuccess;
    auto A = [&](void **p, size_t bytes) {
        if (e == cudaSuccess) e = dmalloc(c, p, std::max<size_t>(bytes, 8));
    };
    A((void **)&k->X, 8 * n * k->ld);
    A((void **)&k->xx, 8 * n);
    A((void **)&k->C, 8 * (size_t)K * k->ldc);
    A((void **)&k->cc, 8 * (size_t)K);
    A((void **)&k->closest, 8 * n);
    A((void **)&k->mind, 8 * n);
    A((void **)&k->lab, 4 * n);
    A((void **)&k->lab_new, 4 * n);
    A((void **)&k->counts, 8 * ((size_t)K + 1));
    A((void **)&k->part, 8 * m);
    A((void **)&k->part_i, 8 * std::max<int64_t>(m, K));  // argmax indices / label totals
    A((void **)&k->scal, 16);
    A((void **)&k->pick, 8);
    A((void **)&k->seg_off, 8 * (size_t)k->nseg * K);
    A((void **)&k->order, 8 * n);
    A((void **)&k->start, 8 * ((size_t)K + 1));
    cudaStream_t s = c->stream;
    if (e == cudaSuccess) {
        if (dtype == CSEMB_F64)
            e = cudaMemcpy2DAsync(k->X, 8 * k->ld, X, 8 * ld, 8 * d, n,
                                  on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s);
        else
            k_to_f64<float><<<grid_for(n * d, 256, c->sm_count), 256, 0, s>>>((const float *)X, n, (int)d, ld, k->X,
                                                                               k->ld);
    }
    if (e == cudaSuccess) e = cudaMemsetAsync(k->C, 0, 8 * (size_t)K * k->ldc, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(k->lab, 0xff, 4 * n, s);  // -1: no labels yet
    if (e == cudaSuccess) {
        k_sqnorm_rows<double><<<group8_grid(n, c->sm_count), 256, 0, s>>>(k->X, n, k->d, k->ld, k->xx);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        km_free(k);
        cudaGetLastError();
        return fail(e == cudaErrorMemoryAllocation ? CSEMB_ERR_NOMEM : CSEMB_ERR_CUDA, "kmeans_create: %s",
                    cudaGetErrorString(e));
    }
    *out = k;
    return CSEMB_OK;
}

extern "C" int csemb_kmeans_destroy(csemb_kmeans *k) {
    if (!k) return CSEMB_OK;
    std::lock_guard<std::mutex> lk(k->ctx->mu);
    cudaSetDevice(k->ctx->device);
    // other streams (caller code reading an output buffer) may still use this
    // memory: wait for the device, as cudaFree would, before the blocks return
    // to the stream-ordered pool
    cudaDeviceSynchronize();
    km_free(k);
    return CSEMB_OK;
}

// deterministic sum of v[0..n) into *dst (device)
static cudaError_t fixed_sum(csemb_kmeans *k, const double *v, const double *divisor, double *dst) {
    const int64_t m = n_chunks(k->n);
    cudaStream_t s = k->ctx->stream;
    k_chunk_sums<<<(unsigned)m, RED_THREADS, 0, s>>>(v, k->n, RED_CHUNK, divisor, k->part);
    k_sum_final<<<1, 256, 0, s>>>(k->part, m, dst);
    return cudaGetLastError();
}

extern "C" int csemb_kmeans_seed(csemb_kmeans *k, int idx, int64_t row, double *total) {
    if (!k) return fail(CSEMB_ERR_INVALID, "null argument");
    if (idx < 0 || idx >= k->K) return fail(CSEMB_ERR_INVALID, "centroid index %d outside [0, %d)", idx, k->K);
    if (row < 0 || row >= k->n) return fail(CSEMB_ERR_INVALID, "row %lld outside [0, %lld)", (long long)row,
                                            (long long)k->n);
    csemb_ctx *c = k->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    double *cen = k->C + (int64_t)idx * k->ldc;
    CK(cudaMemcpyAsync(cen, k->X + row * k->ld, 8 * (size_t)k->d, cudaMemcpyDeviceToDevice, s));
    k_sqnorm_rows<double><<<1, 256, 0, s>>>(cen, 1, k->d, k->ldc, k->cc + idx);
    k_km_dist1<<<group8_grid(k->n, c->sm_count), 256, 0, s>>>(k->X, k->n, k->d, k->ld, k->xx, cen, k->cc + idx,
                                                              k->closest, idx == 0);
    CK(cudaGetLastError());
    CK(fixed_sum(k, k->closest, nullptr, k->scal));
    double t = 0;
    CK(cudaMemcpyAsync(&t, k->scal, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (total) *total = t;
    return CSEMB_OK;
}

extern "C" int csemb_kmeans_pick(csemb_kmeans *k, double u, int64_t *row) {
    if (!k || !row) return fail(CSEMB_ERR_INVALID, "null argument");
    if (!(u >= 0.0 && u < 1.0)) return fail(CSEMB_ERR_INVALID, "u=%g outside [0, 1)", u);
    csemb_ctx *c = k->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    const int64_t m = n_chunks(k->n);
    k_chunk_sums<<<(unsigned)m, RED_THREADS, 0, s>>>(k->closest, k->n, RED_CHUNK, k->scal, k->part);
    k_km_pick<<<1, 1024, 0, s>>>(k->closest, k->n, RED_CHUNK, k->part, m, k->scal, u, k->pick);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(row, k->pick, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return CSEMB_OK;
}

extern "C" int csemb_kmeans_assign(csemb_kmeans *k, double *inertia, int64_t *changed, int64_t *counts) {
    if (!k) return fail(CSEMB_ERR_INVALID, "null argument");
    csemb_ctx *c = k->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    const int K = k->K;
    k_sqnorm_rows<double><<<group8_grid(K, c->sm_count), 256, 0, s>>>(k->C, K, k->d, k->ldc, k->cc);
    CK(cudaMemsetAsync(k->counts, 0, 8 * ((size_t)K + 1), s));
    const int64_t tiles = (k->n + KA_TM - 1) / KA_TM;
    if (k->d <= KA_MAXD) {
        const KaGeom geo(k->d);
        const int Kp = (K + KA_TK - 1) / KA_TK * KA_TK;
        const size_t base = 16 * (size_t)KA_TM * geo.rs + 12 * 4 * (size_t)KA_TM +
                            (K <= KM_SMEM_K ? 4 * (size_t)K : 0);  // count histogram
        const size_t full = base + 8 * (size_t)Kp * geo.rs, tiled = base + 8 * (size_t)KA_TK * geo.rs;
        const bool cfull = full <= 220 * 1024;  // one 512-thread CTA per SM
        const size_t smem = cfull ? full : tiled;
        if (smem > 220 * 1024) return fail(CSEMB_ERR_UNSUPPORTED, "assignment tile does not fit shared memory");
        const void *fn = cfull ? (const void *)k_km_assign<true> : (const void *)k_km_assign<false>;
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const int g = (int)std::min<int64_t>(tiles, (int64_t)c->sm_count);
        if (cfull)
            k_km_assign<true><<<g, KA_THREADS, smem, s>>>(k->X, k->n, k->d, k->ld, k->xx, k->C, K, k->ldc, k->cc,
                                                          k->lab, k->lab_new, k->mind, k->counts, k->counts + K);
        else
            k_km_assign<false><<<g, KA_THREADS, smem, s>>>(k->X, k->n, k->d, k->ld, k->xx, k->C, K, k->ldc, k->cc,
                                                           k->lab, k->lab_new, k->mind, k->counts, k->counts + K);
    } else {
        k_km_assign_wide<<<group8_grid(k->n, c->sm_count), 256, 0, s>>>(k->X, k->n, k->d, k->ld, k->xx, k->C, K,
                                                                        k->ldc, k->cc, k->lab, k->lab_new, k->mind,
                                                                        k->counts, k->counts + K);
    }
    CK(cudaGetLastError());
    CK(fixed_sum(k, k->mind, nullptr, k->scal + 1));
    std::vector<unsigned long long> h(K + 1);
    double in = 0;
    CK(cudaMemcpyAsync(h.data(), k->counts, 8 * ((size_t)K + 1), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&in, k->scal + 1, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (inertia) *inertia = in;
    if (changed) *changed = (int64_t)h[K];
    if (counts)
        for (int q = 0; q < K; ++q) counts[q] = (int64_t)h[q];
    return CSEMB_OK;
}

extern "C" int csemb_kmeans_reseed(csemb_kmeans *k, int idx, int64_t *row) {
    if (!k) return fail(CSEMB_ERR_INVALID, "null argument");
    if (idx < 0 || idx >= k->K) return fail(CSEMB_ERR_INVALID, "centroid index %d outside [0, %d)", idx, k->K);
    csemb_ctx *c = k->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    const int64_t m = n_chunks(k->n);
    k_argmax_part<<<(unsigned)m, RED_THREADS, 0, s>>>(k->mind, k->n, RED_CHUNK, k->part, k->part_i);
    k_km_reseed<<<1, 128, 0, s>>>(k->part, k->part_i, m, k->X, k->d, k->ld, k->C, k->ldc, idx, k->lab_new, k->mind,
                                  k->pick);
    CK(cudaGetLastError());
    int64_t far = 0;
    CK(cudaMemcpyAsync(&far, k->pick, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (row) *row = far;
    return CSEMB_OK;
}

extern "C" int csemb_kmeans_commit(csemb_kmeans *k, int update_centroids) {
    if (!k) return fail(CSEMB_ERR_INVALID, "null argument");
    csemb_ctx *c = k->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    std::swap(k->lab, k->lab_new);  // labels = new_labels
    if (update_centroids) {
        const int K = k->K;
        const size_t hsmem = K <= KM_SMEM_K ? 4 * (size_t)K : 0;
        if (hsmem > 48 * 1024)
            CK(cudaFuncSetAttribute(k_km_seg_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsmem));
        k_km_seg_hist<<<(unsigned)k->nseg, 256, hsmem, s>>>(k->lab, k->n, K, k->seg, k->seg_off);
        k_km_seg_scan<<<(unsigned)((K + 7) / 8), 256, 0, s>>>(k->seg_off, k->nseg, K, k->part_i);
        k_km_start_scan<<<1, 1024, 0, s>>>(k->part_i, K, k->start);
        k_km_seg_scatter<<<(unsigned)((k->nseg + 3) / 4), 128, 0, s>>>(k->lab, k->n, K, k->seg, k->seg_off,
                                                                        k->start, k->order);
        const int64_t warps = (int64_t)K * ((k->d + 31) / 32);
        const int ring = KS_D * 32 * 32 * 8;
        CK(cudaFuncSetAttribute(k_km_sums, cudaFuncAttributeMaxDynamicSharedMemorySize, ring));
        k_km_sums<<<(unsigned)warps, 32, ring, s>>>(k->X, k->d, k->ld, k->order, k->start, K, k->C, k->ldc);
        CK(cudaGetLastError());
    }
    return CSEMB_OK;
}

extern "C" int csemb_kmeans_download(csemb_kmeans *k, int64_t *labels, double *centroids) {
    if (!k) return fail(CSEMB_ERR_INVALID, "null argument");
    csemb_ctx *c = k->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    std::vector<int> h;
    if (labels) {
        h.resize(k->n);
        CK(cudaMemcpyAsync(h.data(), k->lab, 4 * k->n, cudaMemcpyDeviceToHost, s));
    }
    if (centroids)
        CK(cudaMemcpy2DAsync(centroids, 8 * (size_t)k->d, k->C, 8 * k->ldc, 8 * (size_t)k->d, k->K,
                             cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (labels)
        for (int64_t i = 0; i < k->n; ++i) labels[i] = h[i];
    return CSEMB_OK;
}

extern "C" int csemb_kmeans_set_centroids(csemb_kmeans *k, const double *centroids) {
    if (!k || !centroids) return fail(CSEMB_ERR_INVALID, "null argument");
    csemb_ctx *c = k->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    CK(cudaMemcpy2DAsync(k->C, 8 * k->ldc, centroids, 8 * (size_t)k->d, 8 * (size_t)k->d, k->K,
                         cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return CSEMB_OK;
}

extern "C" int csemb_kmeans_reset(csemb_kmeans *k) {
    if (!k) return fail(CSEMB_ERR_INVALID, "null argument");
    csemb_ctx *c = k->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    CK(cudaMemsetAsync(k->lab, 0xff, 4 * k->n, c->stream));
    CK(cudaMemsetAsync(k->C, 0, 8 * (size_t)k->K * k->ldc, c->stream));
    return CSEMB_OK;
}

extern "C" const int32_t *csemb_kmeans_labels(csemb_kmeans *k) { return k ? k->lab : nullptr; }

// ---------------------------------------------------------------------------
// modularity counts
// ---------------------------------------------------------------------------
extern "C" int csemb_modularity_counts(csemb_mat *m, const int32_t *labels, int on_device, int64_t k,
                                       int64_t *intra, int64_t *degsum) {
    if (!m || !labels || !intra || !degsum) return fail(CSEMB_ERR_INVALID, "null argument");
    if (m->n_rows != m->n_cols) return fail(CSEMB_ERR_INVALID, "modularity needs a square (adjacency) matrix");
    if (k < 1 || k > INT32_MAX) return fail(CSEMB_ERR_INVALID, "bad label count %lld", (long long)k);
    const int64_t n = m->n_rows;
    if (!on_device)
        for (int64_t i = 0; i < n; ++i)
            if (labels[i] < 0 || labels[i] >= k)
                return fail(CSEMB_ERR_INVALID, "label %d of vertex %lld outside [0, %lld)", labels[i], (long long)i,
                            (long long)k);
    csemb_ctx *c = m->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    int *dl = nullptr;
    unsigned long long *cnt = nullptr;
    cudaError_t e = dmalloc(c, &cnt, 16 * (size_t)k + 8);  // [k] intra2, [k] degsum, bad-label count
    if (e == cudaSuccess && !on_device) e = dmalloc(c, &dl, 4 * std::max<int64_t>(n, 1));
    if (e == cudaSuccess && !on_device && n) e = cudaMemcpyAsync(dl, labels, 4 * n, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(cnt, 0, 16 * (size_t)k + 8, s);
    if (e == cudaSuccess && n) {
        const int *lab = on_device ? labels : dl;
        const size_t smem = 16 * (size_t)k;
        const int g = grid_for(n, 256, c->sm_count, 4);
        if (smem <= 96 * 1024) {
            if (smem > 48 * 1024)
                e = cudaFuncSetAttribute(k_modularity<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e == cudaSuccess)
                k_modularity<true><<<g, 256, smem, s>>>(m->rowptr, m->cols, n, lab, (int)k, cnt, cnt + k, cnt + 2 * k);
        } else {
            k_modularity<false><<<g, 256, 0, s>>>(m->rowptr, m->cols, n, lab, (int)k, cnt, cnt + k, cnt + 2 * k);
        }
        if (e == cudaSuccess) e = cudaGetLastError();
    }
    std::vector<unsigned long long> h(2 * (size_t)k + 1);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h.data(), cnt, 16 * (size_t)k + 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    dfree(c, dl);
    dfree(c, cnt);
    CK(e);
    if (h[2 * k]) return fail(CSEMB_ERR_INVALID, "%llu labels outside [0, %lld)", h[2 * k], (long long)k);
    for (int64_t q = 0; q < k; ++q) {
        intra[q] = (int64_t)(h[q] / 2);  // each intra edge is stored as (u, v) and (v, u)
        degsum[q] = (int64_t)h[k + q];
    }
    return CSEMB_OK;
}
