// membench.cu -- B200 memory-hierarchy ceilings that bound K1 (gather-heavy SpMM).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/membench tools/membench.cu
//   tools/membench
//
// Measures (CUDA events, best of 5):
//   stream-DRAM  : coalesced float4 reads of a 2 GiB buffer
//   stream-L2    : coalesced float4 re-reads of an L2-resident buffer (ld.global.cg)
//   gather-L2/DRAM: 128-byte rows at random row ids (8 lanes x 16 B per row) within
//                  an L2-resident / 2 GiB window; with L1 caching (ld.global.nc) and without (.cg)
//   copy-DRAM    : read + write 1 GiB (the MEASURED_PEAKS definition)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ float4 ld_cg(const float4 *p) {
    float4 v;
    asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}

template <int CG>
__global__ void k_stream(const float4 *__restrict__ a, size_t n, int reps, float *sink) {
    float acc = 0.f;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
            float4 v = CG ? ld_cg(a + i) : __ldg(a + i);
            acc += v.x + v.y + v.z + v.w;
        }
    if (acc == 1234.5f) *sink = acc;
}

// each group of 8 lanes reads one 128-byte row chosen by a hash; rows in [0, nrows)
__device__ __forceinline__ float4 ld_na(const float4 *p) {
    float4 v;
    asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}

// 8 lanes per row; each row is LINES x 128 B (lane l reads vectors l, l+8, ...)
template <int MODE, int LINES>
__global__ void k_gather_rows(const float4 *__restrict__ a, uint32_t nrows, uint32_t iters, float *sink) {
    const uint32_t lane = threadIdx.x & 7;
    uint32_t g = (blockIdx.x * blockDim.x + threadIdx.x) >> 3;
    uint32_t h = g * 2654435761u + 12345u;
    float acc = 0.f;
    for (uint32_t it = 0; it < iters; it += 2) {
        float4 v[2][LINES];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            h = h * 1664525u + 1013904223u;
            const uint32_t row = (uint32_t)(((uint64_t)(h >> 3) * nrows) >> 29);
            const float4 *p = a + (size_t)row * 8 * LINES + lane;
#pragma unroll
            for (int k = 0; k < LINES; ++k) v[u][k] = MODE == 0 ? __ldg(p + 8 * k) : MODE == 1 ? ld_na(p + 8 * k) : ld_cg(p + 8 * k);
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int k = 0; k < LINES; ++k) acc += v[u][k].x + v[u][k].w;
    }
    if (acc == 1234.5f) *sink = acc;
}

// 8 lanes per 320-byte row (f32 d=80): lane l reads vectors l, l+8 and (l < 4) l+16
__global__ void k_gather_rows320(const float4 *__restrict__ a, uint32_t nrows, uint32_t iters, float *sink) {
    const uint32_t lane = threadIdx.x & 7;
    uint32_t g = (blockIdx.x * blockDim.x + threadIdx.x) >> 3;
    uint32_t h = g * 2654435761u + 12345u;
    float acc = 0.f;
    for (uint32_t it = 0; it < iters; it += 2) {
        float4 v[2][3];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            h = h * 1664525u + 1013904223u;
            const uint32_t row = (uint32_t)(((uint64_t)(h >> 3) * nrows) >> 29);
            const float4 *p = a + (size_t)row * 20 + lane;
            v[u][0] = __ldg(p);
            v[u][1] = __ldg(p + 8);
            v[u][2] = lane < 4 ? __ldg(p + 16) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int k = 0; k < 3; ++k) acc += v[u][k].x + v[u][k].w;
    }
    if (acc == 1234.5f) *sink = acc;
}

// 256-bit loads (sm_100a LDG.E.256): 8 lanes per row of NV 32-byte vectors,
// lane l reads vectors l, l+8, l+16 (< NV); 640-byte rows: NV = 20, 320-byte: NV = 10
struct alignas(32) v8f { float v[8]; };
__device__ __forceinline__ v8f ld256(const v8f *p) {
    v8f r;
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]), "=f"(r.v[6]),
                   "=f"(r.v[7]) : "l"(p));
    return r;
}
template <int NV>
__global__ void k_gather_rows256(const v8f *__restrict__ a, uint32_t nrows, uint32_t iters, float *sink) {
    constexpr int K = (NV + 7) / 8;
    const uint32_t lane = threadIdx.x & 7;
    uint32_t g = (blockIdx.x * blockDim.x + threadIdx.x) >> 3;
    uint32_t h = g * 2654435761u + 12345u;
    float acc = 0.f;
    for (uint32_t it = 0; it < iters; it += 2) {
        v8f v[2][K];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            h = h * 1664525u + 1013904223u;
            const uint32_t row = (uint32_t)(((uint64_t)(h >> 3) * nrows) >> 29);
            const v8f *p = a + (size_t)row * NV + lane;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (lane + 8 * k < NV) v[u][k] = ld256(p + 8 * k);
                else v[u][k].v[0] = v[u][k].v[7] = 0.f;
            }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int k = 0; k < K; ++k) acc += v[u][k].v[0] + v[u][k].v[7];
    }
    if (acc == 1234.5f) *sink = acc;
}

template <int CG, int UNROLL>
__global__ void k_gather(const float4 *__restrict__ a, uint32_t nrows, uint32_t iters, float *sink) {
    const uint32_t lane = threadIdx.x & 7;
    uint32_t g = (blockIdx.x * blockDim.x + threadIdx.x) >> 3;
    uint32_t h = g * 2654435761u + 12345u;
    float acc = 0.f;
    for (uint32_t it = 0; it < iters; it += UNROLL) {
        float4 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            h = h * 1664525u + 1013904223u;
            const uint32_t row = (uint32_t)(((uint64_t)(h >> 3) * nrows) >> 29);
            v[u] = CG ? ld_cg(a + (size_t)row * 8 + lane) : __ldg(a + (size_t)row * 8 + lane);
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) acc += v[u].x + v[u].w;
    }
    if (acc == 1234.5f) *sink = acc;
}

__global__ void k_copy(const float4 *__restrict__ a, float4 *b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

template <typename F>
static float best_ms(F f) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    f();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int i = 0; i < 5; ++i) {
        cudaEventRecord(e0);
        f();
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int l2;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
    printf("SMs %d, L2 %d MB\n", sms, l2 >> 20);
    const size_t big = (size_t)2 << 30;
    float4 *a, *b;
    float *sink;
    CK(cudaMalloc(&a, big));
    CK(cudaMalloc(&b, big / 2));
    CK(cudaMalloc(&sink, 4));
    CK(cudaMemset(a, 0, big));
    const int grid = sms * 8, block = 256;
    {
        size_t n = big / 16;
        float ms = best_ms([&] { k_stream<0><<<grid, block>>>(a, n, 1, sink); });
        printf("stream-DRAM   read %.0f GB/s\n", big / ms / 1e6);
    }
    {
        size_t n = (big / 2) / 16;
        float ms = best_ms([&] { k_copy<<<grid, block>>>(a, b, n); });
        printf("copy-DRAM     r+w  %.0f GB/s\n", 2.0 * (big / 2) / ms / 1e6);
    }
    for (size_t mb : {16, 48, 96}) {
        size_t bytes = mb << 20, n = bytes / 16;
        int reps = 50;
        float ms = best_ms([&] { k_stream<1><<<grid, block>>>(a, n, reps, sink); });
        printf("stream-L2 %3zu MB (cg)  %.0f GB/s\n", mb, (double)bytes * reps / ms / 1e6);
        ms = best_ms([&] { k_stream<0><<<grid, block>>>(a, n, reps, sink); });
        printf("stream-L2 %3zu MB (nc)  %.0f GB/s\n", mb, (double)bytes * reps / ms / 1e6);
    }
    const uint32_t iters = 256;
    const size_t lanes_total = (size_t)grid * block;
    const double gbytes = (double)lanes_total * iters * 16;
    for (size_t mb : {4, 48, 96, 2048}) {
        uint32_t nrows = (uint32_t)((mb << 20) / 128);
        float ms = best_ms([&] { k_gather<1, 8><<<grid, block>>>(a, nrows, iters, sink); });
        printf("gather %4zu MB window (cg) %.0f GB/s\n", mb, gbytes / ms / 1e6);
        ms = best_ms([&] { k_gather<0, 8><<<grid, block>>>(a, nrows, iters, sink); });
        printf("gather %4zu MB window (nc) %.0f GB/s\n", mb, gbytes / ms / 1e6);
    }
    // K1-shaped gathers: 640-byte rows (f64 d=80), 8 lanes x 5 vectors
    for (size_t mb : {48, 640, 2048}) {
        uint32_t nrows = (uint32_t)((mb << 20) / 640);
        const uint32_t it2 = 64;
        const double gb2 = (double)lanes_total * it2 * 16 * 5;
        const char *names[3] = {"nc", "nc.L1::no_allocate", "cg"};
        float ms0 = best_ms([&] { k_gather_rows<0, 5><<<grid, block>>>(a, nrows, it2, sink); });
        float ms1 = best_ms([&] { k_gather_rows<1, 5><<<grid, block>>>(a, nrows, it2, sink); });
        float ms2 = best_ms([&] { k_gather_rows<2, 5><<<grid, block>>>(a, nrows, it2, sink); });
        printf("gather640 %4zu MB: %s %.0f  %s %.0f  %s %.0f GB/s\n", mb, names[0], gb2 / ms0 / 1e6, names[1],
               gb2 / ms1 / 1e6, names[2], gb2 / ms2 / 1e6);
    }
    // the same rows through 256-bit loads (8 lanes x 32 B)
    for (size_t mb : {48, 640, 2048}) {
        uint32_t nrows = (uint32_t)((mb << 20) / 640);
        const uint32_t it2 = 64;
        const double gb2 = (double)lanes_total / 8 * it2 * 640;
        float ms0 = best_ms([&] { k_gather_rows256<20><<<grid, block>>>((const v8f *)a, nrows, it2, sink); });
        printf("gather640x256 %4zu MB: nc %.0f GB/s\n", mb, gb2 / ms0 / 1e6);
    }
    for (size_t mb : {48, 320, 2048}) {
        uint32_t nrows = (uint32_t)((mb << 20) / 320);
        const uint32_t it2 = 64;
        const double gb2 = (double)lanes_total / 8 * it2 * 320;
        float ms0 = best_ms([&] { k_gather_rows256<10><<<grid, block>>>((const v8f *)a, nrows, it2, sink); });
        printf("gather320x256 %4zu MB: nc %.0f GB/s\n", mb, gb2 / ms0 / 1e6);
    }
    // 320-byte rows (f32 d=80, K1's fp32 gather), ld.global.nc
    for (size_t mb : {48, 320, 2048}) {
        uint32_t nrows = (uint32_t)((mb << 20) / 320);
        const uint32_t it2 = 64;
        const double gb2 = (double)lanes_total / 8 * it2 * 320;
        float ms0 = best_ms([&] { k_gather_rows320<<<grid, block>>>(a, nrows, it2, sink); });
        printf("gather320 %4zu MB: nc %.0f GB/s\n", mb, gb2 / ms0 / 1e6);
    }
    return 0;
}
