// gatherbench.cu -- K1's gather+accumulate shape under three load paths on sm_100a.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -o tools/gatherbench tools/gatherbench.cu
//   tools/gatherbench [n_rows] [row_len]
//
// Y[i,:] = sum_k a_ik * X[col_ik, :] in stored order (separately rounded DMUL/DADD),
// X fp64 n x 80 (640-byte rows), rows of fixed length with the config-2 SBM
// pattern (blocks of 10^4 rows, 75% of entries inside the row's block, 25%
// uniform).  Variants:
//   ldg : 16 lanes per row, 3 double2 per lane, 4 entries of 16-byte gathers in
//         flight per lane in registers (round-1 K1's load path)
//   blk : 2 rows per warp (16 lanes x 5 doubles), gathered rows staged in a
//         per-warp shared-memory ring by cp.async.bulk (one 640-byte copy per
//         entry), one mbarrier per stage of 4 entries per row
//   g4  : same ring, filled by TMA tile::gather4 (one instruction per 4 rows)
// All variants must produce bit-identical Y.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e = (x);                                                    \
        if (e != cudaSuccess) {                                                 \
            printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
            exit(1);                                                            \
        }                                                                       \
    } while (0)

constexpr int LD = 80;  // doubles per row

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
            smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_row(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tma_gather4(void *dst, const CUtensorMap *map, int c0, int r0, int r1, int r2, int r3,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
        "%4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ double madd(double acc, double a, double x) { return __dadd_rn(acc, __dmul_rn(a, x)); }

// ---------------- ldg: register pipeline ----------------
template <int D>
__global__ void __launch_bounds__(256, 2) k_ldg(const double2 *__restrict__ X, const int *__restrict__ cols,
                                                 const double *__restrict__ vals, double2 *Y, int n, int len) {
    const int lane = threadIdx.x & 31, gl = lane & 15, grp = lane >> 4;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    constexpr int NV = LD / 2;  // 40 vectors
    for (int rs = warp; rs * 2 < n; rs += nw) {
        const int row = rs * 2 + grp;
        const int64_t base = (int64_t)row * len;
        double2 acc[3], buf[D][3];
#pragma unroll
        for (int k = 0; k < 3; ++k) acc[k] = make_double2(0.0, 0.0);
        auto issue = [&](int slot, int e) {
            const int j = e < len ? __ldg(cols + base + e) : 0;
            const double2 *x = X + (int64_t)j * NV + gl;
#pragma unroll
            for (int k = 0; k < 3; ++k)
                buf[slot][k] = (e < len && gl + 16 * k < NV) ? __ldg(x + 16 * k) : make_double2(0.0, 0.0);
        };
#pragma unroll
        for (int e = 0; e < D - 1; ++e) issue(e, e);
        for (int t = 0; t < len; t += D) {
#pragma unroll
            for (int u = 0; u < D; ++u) {
                issue((u + D - 1) % D, t + u + D - 1);
                const double a = t + u < len ? __ldg(vals + base + t + u) : 0.0;
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    acc[k].x = madd(acc[k].x, a, buf[u][k].x);
                    acc[k].y = madd(acc[k].y, a, buf[u][k].y);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < 3; ++k)
            if (gl + 16 * k < NV) Y[(int64_t)row * NV + gl + 16 * k] = acc[k];
    }
}

// ---------------- staged: smem ring filled by bulk copies or gather4 ----------------
// warp = 2 rows (16 lanes x 5 doubles); stage = K=4 entries of both rows (8 x 640 B)
template <int S, int G4>
__global__ void __launch_bounds__(512, 1) k_staged(const double *__restrict__ X, const __grid_constant__ CUtensorMap map,
                                                    const int *__restrict__ cols, const double *__restrict__ vals,
                                                    double *Y, int n, int len) {
    extern __shared__ __align__(1024) unsigned char smem[];
    constexpr int K = 4;
    constexpr int ROWB = LD * 8;          // 640
    constexpr int STB = 2 * K * ROWB;     // 5120 bytes per stage
    const int lane = threadIdx.x & 31, gl = lane & 15, grp = lane >> 4;
    const int wib = threadIdx.x >> 5;
    unsigned char *wsm = smem + (size_t)wib * (S * STB + 128);
    uint64_t *bars = reinterpret_cast<uint64_t *>(wsm + S * STB);
    if (lane < S) mbar_init(bars + lane, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const int warp = blockIdx.x * (blockDim.x >> 5) + wib;
    const int nw = gridDim.x * (blockDim.x >> 5);
    const int spr = (len + K - 1) / K;  // stages per row set
    const int nrs = (n + 1) / 2;
    const int my_sets = warp < nrs ? (nrs - 1 - warp) / nw + 1 : 0;
    const int total = my_sets * spr;
    // stage s -> row set warp + (s / spr) * nw, entries (s % spr) * K ...
    // lane 0 holds the column ids of the next stage to issue (loaded one stage ahead)
    int cn[2 * K];
    auto load_cols = [&](int s) {
#pragma unroll
        for (int i = 0; i < 2 * K; ++i) cn[i] = n;
        if (lane != 0 || s >= total) return;
        const int rs = warp + (s / spr) * nw, t0 = (s % spr) * K;
#pragma unroll
        for (int g = 0; g < 2; ++g) {
            const int row = rs * 2 + g;
#pragma unroll
            for (int k = 0; k < K; ++k)
                if (row < n && t0 + k < len) cn[g * K + k] = __ldg(cols + (int64_t)row * len + t0 + k);
        }
    };
    auto issue = [&](int s) {
        if (lane == 0 && s < total) {
            uint64_t *bar = bars + (s % S);
            unsigned char *dst = wsm + (size_t)(s % S) * STB;
            mbar_expect(bar, STB);
#pragma unroll
            for (int g = 0; g < 2; ++g) {
                if (G4) {
                    tma_gather4(dst + g * K * ROWB, &map, 0, cn[g * K], cn[g * K + 1], cn[g * K + 2], cn[g * K + 3], bar);
                } else {
#pragma unroll
                    for (int k = 0; k < K; ++k)  // row n is the zero row (keeps the byte count)
                        bulk_row(dst + (g * K + k) * ROWB, X + (int64_t)cn[g * K + k] * LD, ROWB, bar);
                }
            }
        }
        load_cols(s + 1);
    };
    load_cols(0);
    for (int s = 0; s < S - 1; ++s) issue(s);
    double acc[5];
    for (int s = 0; s < total; ++s) {
        issue(s + S - 1);
        const int rs = warp + (s / spr) * nw, t0 = (s % spr) * K;
        const int row = rs * 2 + grp;
        if (t0 == 0) {
#pragma unroll
            for (int k = 0; k < 5; ++k) acc[k] = 0.0;
        }
        double a[K];
#pragma unroll
        for (int k = 0; k < K; ++k) a[k] = (row < n && t0 + k < len) ? __ldg(vals + (int64_t)row * len + t0 + k) : 0.0;
        mbar_wait(bars + (s % S), (s / S) & 1);
        const double *st = reinterpret_cast<const double *>(wsm + (size_t)(s % S) * STB) + grp * K * LD + gl;
#pragma unroll
        for (int k = 0; k < K; ++k)
#pragma unroll
            for (int v = 0; v < 5; ++v) acc[v] = madd(acc[v], a[k], st[k * LD + 16 * v]);
        __syncwarp();
        if (t0 + K >= len && row < n) {
#pragma unroll
            for (int v = 0; v < 5; ++v) Y[(int64_t)row * LD + gl + 16 * v] = acc[v];
        }
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char **argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 1000000;
    const int len = argc > 2 ? atoi(argv[2]) : 20;
    const int blk = 10000;
    printf("gatherbench: n=%d len=%d (entries %lld, gathered %.2f GB/pass)\n", n, len, (long long)n * len,
           (double)n * len * LD * 8 / 1e9);
    std::vector<int> cols((size_t)n * len);
    std::vector<double> vals((size_t)n * len);
    uint64_t h = 88172645463325252ull;
    auto rnd = [&]() {
        h ^= h << 13;
        h ^= h >> 7;
        h ^= h << 17;
        return h;
    };
    for (int i = 0; i < n; ++i) {
        int *c = &cols[(size_t)i * len];
        const int b0 = (i / blk) * blk, bn = (b0 + blk <= n) ? blk : n - b0;
        for (int k = 0; k < len; ++k) {
            if ((int)(rnd() % 4) != 0) c[k] = b0 + (int)(rnd() % bn);
            else c[k] = (int)(rnd() % n);
            vals[(size_t)i * len + k] = 1.0 / (1.0 + (double)(rnd() % 1000));
        }
        std::sort(c, c + len);
    }
    std::vector<double> X((size_t)(n + 1) * LD);
    for (size_t t = 0; t < (size_t)n * LD; ++t) X[t] = (double)(rnd() % 100000) * 1e-5 - 0.5;
    for (int c = 0; c < LD; ++c) X[(size_t)n * LD + c] = 0.0;
    double *dX, *dV, *dY[3];
    int *dC;
    CK(cudaMalloc(&dX, X.size() * 8));
    CK(cudaMalloc(&dV, vals.size() * 8));
    CK(cudaMalloc(&dC, cols.size() * 4));
    for (int v = 0; v < 3; ++v) CK(cudaMalloc(&dY[v], (size_t)n * LD * 8));
    CK(cudaMemcpy(dX, X.data(), X.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dV, vals.data(), vals.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dC, cols.data(), cols.size() * 4, cudaMemcpyHostToDevice));

    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q));
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)LD, (cuuint64_t)n};  // row n is out of bounds (zero fill)
    cuuint64_t strides[1] = {(cuuint64_t)LD * 8};
    cuuint32_t box[2] = {(cuuint32_t)LD, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, dX, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("tensor map encode: %d\n", (int)cr);
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const double gbytes = (double)n * len * LD * 8 / 1e9;
    auto timeit = [&](const char *name, auto launch) {
        launch();
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        float best = 1e30f;
        for (int r = 0; r < 7; ++r) {
            CK(cudaEventRecord(e0));
            launch();
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            best = ms < best ? ms : best;
        }
        printf("%-28s %8.3f ms  %8.0f GB/s gathered\n", name, best, gbytes / best * 1e3);
        fflush(stdout);
    };
    timeit("ldg D=4 (2 CTA x 256)", [&] { k_ldg<4><<<sms * 2, 256>>>((const double2 *)dX, dC, dV, (double2 *)dY[0], n, len); });
    timeit("ldg D=2 (2 CTA x 256)", [&] { k_ldg<2><<<sms * 2, 256>>>((const double2 *)dX, dC, dV, (double2 *)dY[0], n, len); });
    auto staged = [&](auto kern, int S, int warps, int which, const char *name) {
        const size_t sm = (size_t)warps * (S * 5120 + 128);
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        timeit(name, [&] { kern<<<sms, warps * 32, sm>>>(dX, map, dC, dV, dY[which], n, len); });
    };
    staged(k_staged<4, 0>, 4, 10, 1, "blk S=4 10 warps");
    staged(k_staged<8, 0>, 8, 5, 1, "blk S=8 5 warps");
    staged(k_staged<3, 0>, 3, 14, 1, "blk S=3 14 warps");
    staged(k_staged<4, 1>, 4, 10, 2, "g4 S=4 10 warps");
    staged(k_staged<8, 1>, 8, 5, 2, "g4 S=8 5 warps");
    staged(k_staged<3, 1>, 3, 14, 2, "g4 S=3 14 warps");
    staged(k_staged<6, 1>, 6, 7, 2, "g4 S=6 7 warps");
    std::vector<double> y0((size_t)n * LD), y1((size_t)n * LD), y2((size_t)n * LD);
    CK(cudaMemcpy(y0.data(), dY[0], y0.size() * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(y1.data(), dY[1], y1.size() * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(y2.data(), dY[2], y2.size() * 8, cudaMemcpyDeviceToHost));
    printf("blk == ldg: %s   g4 == ldg: %s\n", memcmp(y0.data(), y1.data(), y0.size() * 8) ? "NO" : "yes",
           memcmp(y0.data(), y2.data(), y0.size() * 8) ? "NO" : "yes");
    // spot check against the host
    int bad = 0;
    for (int i = 0; i < n; i += 9973) {
        for (int c = 0; c < LD; ++c) {
            double acc = 0.0;
            for (int k = 0; k < len; ++k) {
                volatile double p = vals[(size_t)i * len + k] * X[(size_t)cols[(size_t)i * len + k] * LD + c];
                acc = acc + p;
            }
            if (acc != y0[(size_t)i * LD + c]) ++bad;
        }
    }
    printf("host spot check mismatches: %d\n", bad);
    return 0;
}
