// build.cu -- device-side input construction.
//
// The reference builds its operators on the host with numpy (sparse.py:191-237):
//   normalized_adjacency (sparse.py:202-226): drop self-loops, dedupe the
//     undirected edges, degrees by bincount, value 1/sqrt(deg u * deg v),
//     isolated vertices keep empty rows;
//   dilate (sparse.py:191-199): [0 A^T; A 0], the first n indices are A's
//     columns, the last m its rows.
// At config 2-5 scale that host work (20.5 s at n = 1e6) dominates the
// end-to-end embed time, so here it is a handful of kernels on the context
// stream: edge keys -> radix sort -> unique -> degree counts -> scan -> the
// symmetric keys -> radix sort -> one fused pass writing column ids and values.
// The keys are the reference's own (min*n + max, row*n + col), sorted into the
// same canonical order, and every value is the same IEEE expression
// (__dmul_rn, __dsqrt_rn, __ddiv_rn: numpy's multiply, sqrt and true divide),
// so the CSR is bit-identical to the host builders.  Radix sort, select and
// scan are CUB's device primitives (plumbing, like cuBLAS for a GEMM); the
// key construction, counting, expansion and fill are the kernels below.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cub/cub.cuh>
#include <mutex>

#include "runtime.h"

namespace {

constexpr uint64_t NO_EDGE = ~0ull;  // self-loop / invalid marker: sorts after every real key

// bits needed to hold keys in [0, n*n)
int key_bits(int64_t n) {
    const unsigned long long top = (unsigned long long)n * (unsigned long long)n - 1ull;
    int b = 1;
    while (b < 64 && (top >> b)) ++b;
    return b;
}

// key of edge t: min(u,v)*n + max(u,v) (sparse.py:216 `np.minimum(u, v) * n +
// np.maximum(u, v)`), NO_EDGE for self-loops; out-of-range ends raise *bad
__global__ void k_edge_keys(const int64_t *__restrict__ edges, int64_t n_edges, int64_t n, uint64_t *keys, int *bad) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_edges;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = edges[2 * t], v = edges[2 * t + 1];
        uint64_t k = NO_EDGE;
        if (u < 0 || v < 0 || u >= n || v >= n) {
            atomicExch(bad, 1);
        } else if (u != v) {
            const int64_t lo = u < v ? u : v, hi = u < v ? v : u;
            k = (uint64_t)lo * (uint64_t)n + (uint64_t)hi;
        }
        keys[t] = k;
    }
}

// deg[lo] += 1, deg[hi] += 1 per unique edge (np.bincount(lo) + np.bincount(hi));
// integer atomics, so the counts do not depend on the order
__global__ void k_degree(const uint64_t *__restrict__ uniq, int64_t m, int64_t n, unsigned long long *deg) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = uniq[t];
        atomicAdd(deg + k / (uint64_t)n, 1ull);
        atomicAdd(deg + k % (uint64_t)n, 1ull);
    }
}

// both orientations of every unique edge: lo*n+hi and hi*n+lo
__global__ void k_symmetric_keys(const uint64_t *__restrict__ uniq, int64_t m, int64_t n, uint64_t *sym) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = uniq[t];
        const uint64_t lo = k / (uint64_t)n, hi = k % (uint64_t)n;
        sym[2 * t] = k;
        sym[2 * t + 1] = hi * (uint64_t)n + lo;
    }
}

// entry j of the canonical CSR: column id and 1/sqrt(deg r * deg c)
// (sparse.py:224 `1.0 / np.sqrt(degf[r] * degf[c])`, the same three IEEE ops)
template <typename T>
__global__ void k_fill_normalized(const uint64_t *__restrict__ sym, int64_t cnt, int64_t n,
                                  const unsigned long long *__restrict__ deg, int *cols, T *vals) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = sym[t];
        const uint64_t r = k / (uint64_t)n, c = k % (uint64_t)n;
        const double p = __dmul_rn((double)deg[r], (double)deg[c]);
        cols[t] = (int)c;
        vals[t] = (T)__ddiv_rn(1.0, __dsqrt_rn(p));
    }
}

// row of every stored entry (binary search in the offsets)
__global__ void k_entry_rows(const int64_t *__restrict__ rowptr, int64_t n_rows, int64_t nnz, int64_t *rows) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nnz; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = n_rows;  // last row r with rowptr[r] <= t
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (rowptr[mid] <= t) lo = mid;
            else hi = mid;
        }
        rows[t] = lo;
    }
}

// transposed keys of A's entries: col * m + row, payload = entry index
__global__ void k_transpose_keys(const int *__restrict__ cols, const int64_t *__restrict__ rows, int64_t nnz,
                                 int64_t m, uint64_t *keys, int64_t *idx, unsigned long long *colcount) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nnz; t += (int64_t)gridDim.x * blockDim.x) {
        const int c = cols[t];
        keys[t] = (uint64_t)c * (uint64_t)m + (uint64_t)rows[t];
        idx[t] = t;
        atomicAdd(colcount + c, 1ull);
    }
}

// [0 A^T; A 0]: top block (rows 0..n-1) from the transposed order, bottom
// block (rows n..n+m-1) is A's own entries; S row offsets of the bottom block
template <typename T>
__global__ void k_fill_dilation(const uint64_t *__restrict__ tkeys, const int64_t *__restrict__ tidx, int64_t nnz,
                                int64_t m, int64_t n, const int *__restrict__ acols, const T *__restrict__ avals,
                                int *scols, T *svals) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nnz; t += (int64_t)gridDim.x * blockDim.x) {
        scols[t] = (int)(n + (int64_t)(tkeys[t] % (uint64_t)m));
        svals[t] = avals[tidx[t]];
        scols[nnz + t] = acols[t];
        svals[nnz + t] = avals[t];
    }
}

__global__ void k_bottom_offsets(const int64_t *__restrict__ arow, int64_t m, int64_t nnz, int64_t n, int64_t *srow) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t <= m; t += (int64_t)gridDim.x * blockDim.x)
        srow[n + t] = nnz + arow[t];
}

// scratch allocations of one build, released together (stream-ordered)
struct Scratch {
    csemb_ctx *c;
    void *p[16] = {};
    int k = 0;
    explicit Scratch(csemb_ctx *ctx) : c(ctx) {}
    template <typename T>
    cudaError_t get(T **out, size_t bytes) {
        void *q = nullptr;
        cudaError_t e = dmalloc(c, &q, std::max<size_t>(bytes, 16));
        if (e == cudaSuccess) p[k++] = q;
        *out = (T *)q;
        return e;
    }
    ~Scratch() {
        for (int i = 0; i < k; ++i) dfree(c, p[i]);
    }
};

int finish_matrix(csemb_mat *m) {
    m->rowptr_host.resize((size_t)m->n_rows + 1);
    CK(cudaMemcpyAsync(m->rowptr_host.data(), m->rowptr, 8 * ((size_t)m->n_rows + 1), cudaMemcpyDeviceToHost,
                       m->ctx->stream));
    CK(cudaStreamSynchronize(m->ctx->stream));
    return CSEMB_OK;
}

// CK that also releases the half-built matrix `mat`
#define CKB(x)                                \
    do {                                      \
        const cudaError_t eb_ = (x);          \
        if (eb_ != cudaSuccess) {             \
            mat_free(mat);                    \
            CK(eb_);                          \
        }                                     \
    } while (0)

// Row partition with overlap (csemb_plan_partition_split): per row, the
// entries whose column lies in the rank's own row range [lo, hi) and the rest.
// One warp per row; each part keeps the row's stored order.
__global__ void k_split_count(const int64_t *__restrict__ rowptr, const int *__restrict__ cols, int64_t n_rows,
                              int64_t lo, int64_t hi, int64_t *cnt_loc, int64_t *cnt_rem) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n_rows; r += nw) {
        const int64_t b = rowptr[r], e = rowptr[r + 1];
        unsigned n_loc = 0;
        for (int64_t q = b + lane; q < e; q += 32) n_loc += (cols[q] >= lo && cols[q] < hi) ? 1u : 0u;
        n_loc = __reduce_add_sync(0xFFFFFFFFu, n_loc);
        if (lane == 0) {
            cnt_loc[r] = n_loc;
            cnt_rem[r] = (e - b) - (int64_t)n_loc;
        }
    }
}

template <typename T>
__global__ void k_split_fill(const int64_t *__restrict__ rowptr, const int *__restrict__ cols,
                             const T *__restrict__ vals, int64_t n_rows, int64_t lo, int64_t hi,
                             const int64_t *__restrict__ off_loc, const int64_t *__restrict__ off_rem,
                             int *cols_loc, T *vals_loc, int *cols_rem, T *vals_rem) {
    const int lane = threadIdx.x & 31;
    const unsigned below = (1u << lane) - 1u;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n_rows; r += nw) {
        const int64_t b = rowptr[r], e = rowptr[r + 1];
        int64_t pl = off_loc[r], pr = off_rem[r];
        for (int64_t q0 = b; q0 < e; q0 += 32) {
            const int64_t q = q0 + lane;
            const bool ok = q < e;
            const int c = ok ? cols[q] : 0;
            const bool loc = ok && c >= lo && c < hi;
            const unsigned ml = __ballot_sync(0xFFFFFFFFu, loc), mr = __ballot_sync(0xFFFFFFFFu, ok && !loc);
            if (loc) {
                cols_loc[pl + __popc(ml & below)] = (int)(c - lo);
                vals_loc[pl + __popc(ml & below)] = vals[q];
            } else if (ok) {
                cols_rem[pr + __popc(mr & below)] = c;
                vals_rem[pr + __popc(mr & below)] = vals[q];
            }
            pl += __popc(ml);
            pr += __popc(mr);
        }
    }
}

// schedule keys: (window index, min(exact ? len : ceil(len / G), cap)), ids = row
__global__ void k_sched_keys(const int64_t *__restrict__ rowptr, int64_t n, int G, int exact, int64_t window,
                             uint64_t *keys, int *ids) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t len = rowptr[i + 1] - rowptr[i];
        const int64_t k = exact ? len : (len + G - 1) / G;
        const uint64_t key = (uint64_t)(k < (1 << 16) ? k : (1 << 16));
        const uint64_t w = window > 0 ? (uint64_t)(i / window) : 0ull;
        keys[i] = (w << 17) | key;
        ids[i] = (int)i;
    }
}

}  // namespace

int sched_order_device(csemb_mat *m, int G, bool exact, int64_t window, int **perm_out) {
    csemb_ctx *c = m->ctx;
    cudaStream_t s = c->stream;
    const int64_t n = m->n_rows;
    *perm_out = nullptr;
    Scratch tmp(c);
    uint64_t *keys = nullptr, *keys2 = nullptr;
    int *ids = nullptr, *perm = nullptr;
    CK(tmp.get(&keys, 8 * (size_t)n));
    CK(tmp.get(&keys2, 8 * (size_t)n));
    CK(tmp.get(&ids, 4 * (size_t)n));
    CK(dmalloc(c, &perm, 4 * (size_t)n));
    const int64_t nwin = window > 0 ? (n + window - 1) / window : 1;
    int bits = 17;
    while (bits < 64 && (nwin - 1) >> (bits - 17)) ++bits;
    auto run = [&]() -> cudaError_t {
        k_sched_keys<<<c->sm_count * 8, 256, 0, s>>>(m->rowptr, n, G, exact ? 1 : 0, window, keys, ids);
        cudaError_t e = cudaGetLastError();
        size_t tb = 0;
        void *ts = nullptr;
        if (e == cudaSuccess) e = cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys2, ids, perm, n, 0, bits, s);
        if (e == cudaSuccess) e = tmp.get(&ts, tb);
        // LSD radix sort: stable, so rows of equal (window, key) keep their order
        if (e == cudaSuccess) e = cub::DeviceRadixSort::SortPairs(ts, tb, keys, keys2, ids, perm, n, 0, bits, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // the scratch is released on return
        return e;
    };
    const cudaError_t e = run();
    if (e != cudaSuccess) {
        dfree(c, perm);
        CK(e);
    }
    *perm_out = perm;
    return CSEMB_OK;
}

int mat_split_columns(csemb_mat *m, int64_t lo, int64_t hi, csemb_mat **loc_out, csemb_mat **rem_out) {
    csemb_ctx *c = m->ctx;
    cudaStream_t s = c->stream;
    const int64_t n = m->n_rows;
    const int g = c->sm_count * 8;
    *loc_out = *rem_out = nullptr;
    Scratch tmp(c);
    int64_t *cnt = nullptr;  // [0, n): local counts, [n, 2n): remote counts
    CK(tmp.get(&cnt, 16 * (size_t)std::max<int64_t>(n, 1)));
    if (n > 0) {
        k_split_count<<<g, 256, 0, s>>>(m->rowptr, m->cols, n, lo, hi, cnt, cnt + n);
        CK(cudaGetLastError());
    }
    csemb_mat *loc = nullptr, *rem = nullptr;
    // the two parts' sizes (one small read back)
    int64_t tot[2] = {0, 0};
    {
        int64_t *sums = nullptr;
        CK(tmp.get(&sums, 16));
        size_t tb = 0;
        void *ts = nullptr;
        CK(cub::DeviceReduce::Sum(nullptr, tb, cnt, sums, std::max<int64_t>(n, 1), s));
        CK(tmp.get(&ts, tb));
        if (n > 0) {
            CK(cub::DeviceReduce::Sum(ts, tb, cnt, sums, n, s));
            CK(cub::DeviceReduce::Sum(ts, tb, cnt + n, sums + 1, n, s));
            CK(cudaMemcpyAsync(tot, sums, 16, cudaMemcpyDeviceToHost, s));
        }
        CK(cudaStreamSynchronize(s));
    }
    int rc = mat_alloc(c, n, hi - lo, tot[0], m->dtype, &loc);
    if (rc) return rc;
    rc = mat_alloc(c, n, m->n_cols, tot[1], m->dtype, &rem);
    if (rc) {
        mat_free(loc);
        return rc;
    }
    auto bail = [&](cudaError_t e) {
        mat_free(loc);
        mat_free(rem);
        cudaGetLastError();
        return fail(e == cudaErrorMemoryAllocation ? CSEMB_ERR_NOMEM : CSEMB_ERR_CUDA, "row split: %s",
                    cudaGetErrorString(e));
    };
    cudaError_t e = cudaMemsetAsync(loc->rowptr, 0, 8, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(rem->rowptr, 0, 8, s);
    if (e == cudaSuccess && n > 0) {
        size_t tb = 0;
        void *ts = nullptr;
        e = cub::DeviceScan::InclusiveSum(nullptr, tb, cnt, loc->rowptr + 1, n, s);
        if (e == cudaSuccess) e = tmp.get(&ts, tb);
        if (e == cudaSuccess) e = cub::DeviceScan::InclusiveSum(ts, tb, cnt, loc->rowptr + 1, n, s);
        if (e == cudaSuccess) e = cub::DeviceScan::InclusiveSum(ts, tb, cnt + n, rem->rowptr + 1, n, s);
        if (e == cudaSuccess) {
            if (m->dtype == CSEMB_F64)
                k_split_fill<double><<<g, 256, 0, s>>>(m->rowptr, m->cols, (const double *)m->vals, n, lo, hi,
                                                       loc->rowptr, rem->rowptr, loc->cols, (double *)loc->vals,
                                                       rem->cols, (double *)rem->vals);
            else
                k_split_fill<float><<<g, 256, 0, s>>>(m->rowptr, m->cols, (const float *)m->vals, n, lo, hi,
                                                      loc->rowptr, rem->rowptr, loc->cols, (float *)loc->vals,
                                                      rem->cols, (float *)rem->vals);
            e = cudaGetLastError();
        }
    } else if (e == cudaSuccess) {
        e = cudaMemsetAsync(loc->rowptr, 0, 8 * ((size_t)n + 1), s);
        if (e == cudaSuccess) e = cudaMemsetAsync(rem->rowptr, 0, 8 * ((size_t)n + 1), s);
    }
    if (e != cudaSuccess) return bail(e);
    rc = finish_matrix(loc);
    if (!rc) rc = finish_matrix(rem);
    if (rc) {
        mat_free(loc);
        mat_free(rem);
        return rc;
    }
    *loc_out = loc;
    *rem_out = rem;
    return CSEMB_OK;
}

extern "C" int csemb_build_normalized_adjacency(csemb_ctx *c, int64_t n, int64_t n_edges, const int64_t *edges,
                                                int edges_on_device, int dtype, csemb_mat **out) {
    if (!c || !out || (n_edges > 0 && !edges)) return fail(CSEMB_ERR_INVALID, "null argument");
    if (n < 1) return fail(CSEMB_ERR_INVALID, "vertex count must be positive");
    if (n_edges < 0) return fail(CSEMB_ERR_INVALID, "negative edge count");
    if (n > 0x7FFFFFFFLL) return fail(CSEMB_ERR_UNSUPPORTED, "vertex count above 2^31-1 (int32 column indices)");
    std::lock_guard<std::mutex> lk(c->mu);
    *out = nullptr;
    CK(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    const int g = c->sm_count * 8;
    Scratch tmp(c);
    int64_t *dedges = nullptr;
    uint64_t *keys = nullptr, *keys2 = nullptr;
    int *bad = nullptr;
    int64_t *nsel = nullptr;
    CK(tmp.get(&bad, sizeof(int)));
    CK(tmp.get(&nsel, sizeof(int64_t)));
    CK(cudaMemsetAsync(bad, 0, sizeof(int), s));
    int64_t m_edges = 0;
    const int bits = key_bits(n);
    if (n_edges > 0) {
        const int64_t *src = edges;
        if (!edges_on_device) {
            CK(tmp.get(&dedges, 16 * (size_t)n_edges));
            CK(cudaMemcpyAsync(dedges, edges, 16 * (size_t)n_edges, cudaMemcpyHostToDevice, s));
            src = dedges;
        }
        CK(tmp.get(&keys, 8 * (size_t)n_edges));
        CK(tmp.get(&keys2, 8 * (size_t)n_edges));
        k_edge_keys<<<g, 256, 0, s>>>(src, n_edges, n, keys, bad);
        CK(cudaGetLastError());
        size_t tb = 0, tb2 = 0;
        CK(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, keys2, n_edges, 0, bits, s));
        CK(cub::DeviceSelect::Unique(nullptr, tb2, keys2, keys, nsel, n_edges, s));
        void *ts = nullptr;
        CK(tmp.get(&ts, std::max(tb, tb2)));
        tb = std::max(tb, tb2);
        CK(cub::DeviceRadixSort::SortKeys(ts, tb, keys, keys2, n_edges, 0, bits, s));
        CK(cub::DeviceSelect::Unique(ts, tb, keys2, keys, nsel, n_edges, s));
        int64_t hsel = 0;
        uint64_t last = 0;
        int hbad = 0;
        CK(cudaMemcpyAsync(&hsel, nsel, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (hbad) return fail(CSEMB_ERR_INVALID, "edge endpoint out of range [0, n)");
        if (hsel > 0) {
            CK(cudaMemcpyAsync(&last, keys + hsel - 1, 8, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
        }
        m_edges = hsel - ((hsel > 0 && last == NO_EDGE) ? 1 : 0);  // the self-loop marker sorts last
    }
    const int64_t nnz = 2 * m_edges;
    csemb_mat *mat = nullptr;
    int rc = mat_alloc(c, n, n, nnz, dtype, &mat);
    if (rc) return rc;
    unsigned long long *deg = nullptr;
    CKB(tmp.get(&deg, 8 * (size_t)n));
    CKB(cudaMemsetAsync(deg, 0, 8 * (size_t)n, s));
    CKB(cudaMemsetAsync(mat->rowptr, 0, 8, s));
    if (m_edges > 0) {
        k_degree<<<g, 256, 0, s>>>(keys, m_edges, n, deg);
        CKB(cudaGetLastError());
        uint64_t *sym = nullptr, *sym2 = nullptr;
        CKB(tmp.get(&sym, 8 * (size_t)nnz));
        CKB(tmp.get(&sym2, 8 * (size_t)nnz));
        k_symmetric_keys<<<g, 256, 0, s>>>(keys, m_edges, n, sym);
        CKB(cudaGetLastError());
        size_t tb = 0, tb2 = 0;
        CKB(cub::DeviceRadixSort::SortKeys(nullptr, tb, sym, sym2, nnz, 0, bits, s));
        CKB(cub::DeviceScan::InclusiveSum(nullptr, tb2, (const int64_t *)deg, mat->rowptr + 1, n, s));
        void *ts = nullptr;
        CKB(tmp.get(&ts, std::max(tb, tb2)));
        tb = std::max(tb, tb2);
        CKB(cub::DeviceRadixSort::SortKeys(ts, tb, sym, sym2, nnz, 0, bits, s));
        CKB(cub::DeviceScan::InclusiveSum(ts, tb, (const int64_t *)deg, mat->rowptr + 1, n, s));
        if (dtype == CSEMB_F64)
            k_fill_normalized<double><<<g, 256, 0, s>>>(sym2, nnz, n, deg, mat->cols, (double *)mat->vals);
        else
            k_fill_normalized<float><<<g, 256, 0, s>>>(sym2, nnz, n, deg, mat->cols, (float *)mat->vals);
        CKB(cudaGetLastError());
    } else {
        CKB(cudaMemsetAsync(mat->rowptr, 0, 8 * ((size_t)n + 1), s));
    }
    rc = finish_matrix(mat);
    if (rc) {
        mat_free(mat);
        return rc;
    }
    *out = mat;
    return CSEMB_OK;
}

extern "C" int csemb_build_dilation(csemb_mat *A, csemb_mat **out) {
    if (!A || !out) return fail(CSEMB_ERR_INVALID, "null argument");
    csemb_ctx *c = A->ctx;
    const int64_t m = A->n_rows, n = A->n_cols, nnz = A->nnz;
    if (m < 1 || n < 1) return fail(CSEMB_ERR_INVALID, "cannot dilate an empty matrix");
    if (m + n > 0x7FFFFFFFLL) return fail(CSEMB_ERR_UNSUPPORTED, "dilated dimension above 2^31-1");
    std::lock_guard<std::mutex> lk(c->mu);
    *out = nullptr;
    CK(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    const int g = c->sm_count * 8;
    csemb_mat *mat = nullptr;
    int rc = mat_alloc(c, m + n, m + n, 2 * nnz, A->dtype, &mat);
    if (rc) return rc;
    Scratch tmp(c);
    unsigned long long *colcount = nullptr;
    CKB(tmp.get(&colcount, 8 * (size_t)n));
    CKB(cudaMemsetAsync(colcount, 0, 8 * (size_t)n, s));
    CKB(cudaMemsetAsync(mat->rowptr, 0, 8, s));
    if (nnz > 0) {
        int64_t *rows = nullptr, *idx = nullptr, *idx2 = nullptr;
        uint64_t *keys = nullptr, *keys2 = nullptr;
        CKB(tmp.get(&rows, 8 * (size_t)nnz));
        CKB(tmp.get(&idx, 8 * (size_t)nnz));
        CKB(tmp.get(&idx2, 8 * (size_t)nnz));
        CKB(tmp.get(&keys, 8 * (size_t)nnz));
        CKB(tmp.get(&keys2, 8 * (size_t)nnz));
        k_entry_rows<<<g, 256, 0, s>>>(A->rowptr, m, nnz, rows);
        CKB(cudaGetLastError());
        k_transpose_keys<<<g, 256, 0, s>>>(A->cols, rows, nnz, m, keys, idx, colcount);
        CKB(cudaGetLastError());
        const int bits = key_bits(std::max(m, n));
        size_t tb = 0, tb2 = 0;
        CKB(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys2, idx, idx2, nnz, 0, bits, s));
        CKB(cub::DeviceScan::InclusiveSum(nullptr, tb2, (const int64_t *)colcount, mat->rowptr + 1, n, s));
        void *ts = nullptr;
        CKB(tmp.get(&ts, std::max(tb, tb2)));
        tb = std::max(tb, tb2);
        // (col, row) keys are unique, so the sort order is the canonical one
        CKB(cub::DeviceRadixSort::SortPairs(ts, tb, keys, keys2, idx, idx2, nnz, 0, bits, s));
        CKB(cub::DeviceScan::InclusiveSum(ts, tb, (const int64_t *)colcount, mat->rowptr + 1, n, s));
        if (A->dtype == CSEMB_F64)
            k_fill_dilation<double><<<g, 256, 0, s>>>(keys2, idx2, nnz, m, n, A->cols, (const double *)A->vals,
                                                      mat->cols, (double *)mat->vals);
        else
            k_fill_dilation<float><<<g, 256, 0, s>>>(keys2, idx2, nnz, m, n, A->cols, (const float *)A->vals,
                                                     mat->cols, (float *)mat->vals);
        CKB(cudaGetLastError());
    } else {
        CKB(cudaMemsetAsync(mat->rowptr, 0, 8 * ((size_t)n + 1), s));
    }
    k_bottom_offsets<<<g, 256, 0, s>>>(A->rowptr, m, nnz, n, mat->rowptr);
    CKB(cudaGetLastError());
    rc = finish_matrix(mat);
    if (rc) {
        mat_free(mat);
        return rc;
    }
    *out = mat;
    return CSEMB_OK;
}

// copy of a device matrix in another dtype (values converted; f32 -> f64 is exact)
template <typename S, typename D>
__global__ void k_convert_vals(const S *__restrict__ src, D *dst, int64_t cnt) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += (int64_t)gridDim.x * blockDim.x)
        dst[t] = (D)src[t];
}

extern "C" int csemb_matrix_convert(csemb_mat *A, int dtype, csemb_mat **out) {
    if (!A || !out) return fail(CSEMB_ERR_INVALID, "null argument");
    csemb_ctx *c = A->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    *out = nullptr;
    CK(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    csemb_mat *mat = nullptr;
    int rc = mat_alloc(c, A->n_rows, A->n_cols, A->nnz, dtype, &mat);
    if (rc) return rc;
    const int g = grid_for(std::max<int64_t>(A->nnz, 1), 256, c->sm_count);
    CKB(cudaMemcpyAsync(mat->rowptr, A->rowptr, 8 * ((size_t)A->n_rows + 1), cudaMemcpyDeviceToDevice, s));
    if (A->nnz > 0) {
        CKB(cudaMemcpyAsync(mat->cols, A->cols, 4 * (size_t)A->nnz, cudaMemcpyDeviceToDevice, s));
        if (A->dtype == dtype)
            CKB(cudaMemcpyAsync(mat->vals, A->vals, dsize(dtype) * (size_t)A->nnz, cudaMemcpyDeviceToDevice, s));
        else if (dtype == CSEMB_F32)
            k_convert_vals<double, float><<<g, 256, 0, s>>>((const double *)A->vals, (float *)mat->vals, A->nnz);
        else
            k_convert_vals<float, double><<<g, 256, 0, s>>>((const float *)A->vals, (double *)mat->vals, A->nnz);
        CKB(cudaGetLastError());
    }
    mat->rowptr_host = A->rowptr_host;
    CKB(cudaStreamSynchronize(s));
    *out = mat;
    return CSEMB_OK;
}

extern "C" int csemb_matrix_device_arrays(csemb_mat *A, void **row_offsets, void **col_indices, void **values) {
    if (!A) return fail(CSEMB_ERR_INVALID, "null matrix");
    if (row_offsets) *row_offsets = A->rowptr;
    if (col_indices) *col_indices = A->cols;
    if (values) *values = A->vals;
    return CSEMB_OK;
}
