// kernels.cuh -- sm_100a kernels of the fused SpMM-Legendre recurrence.
//
// K1 k_step      : one order of the recurrence (engine.py:213-227 + sparse.py:187)
//                  Q(r) = alpha_r * (S Q(r-1)) - beta_r * Q(r-2);  E += theta_r Q(r)
//                  fused: one pass over the CSR, the gathered rows of Q(r-1), and
//                  the streamed rows of Q(r-2) (overwritten in place by Q(r)) and E.
// K2 k_stage_init: projection block (engine.py:79-99 hash / Philox) or the previous
//                  cascade stage's output, Q(0) = block, E = theta_0 * block
//                  (engine.py:210-212).
// K3 k_colstats / k_colfinish / k_colscale: power-iteration pieces for
//                  estimate_spectral_norm (engine.py:180-191); SpMM via k_step<SPMM>.
// K4 k_rownorm   : E_i / ||E_i|| with zero rows -> 0 (oracle.py:88-96 semantics).
//
// Layout: dense blocks are n x ld row-major, ld = d rounded up to one 16-byte
// vector (double2 / float4); row r of a block is ld/W 16-byte vectors.
// A row of the recurrence is owned by a group of G lanes; lane l handles the
// 16-byte vectors l, l+G, l+2G, ... of the row (VPL of them), so every load of
// a gathered row is a contiguous G*16-byte segment.
//
// fp64 arithmetic is strict: multiply and add are separately rounded
// (__dmul_rn/__dadd_rn, no FMA contraction) and each output element is
// accumulated over the row's stored entries in stored order starting from
// +0.0, exactly as scipy's csr_matvecs and numpy do on the reference side --
// so the fp64 path is bit-identical to the reference.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

namespace csemb {

enum { MODE_RECUR = 0, MODE_SPMM = 1 };

template <typename T> struct Vec;
template <> struct Vec<double> {
    typedef double2 type;
    static constexpr int W = 2;
};
template <> struct Vec<float> {
    typedef float4 type;
    static constexpr int W = 4;
};

__device__ __forceinline__ double2 vzero(double2) { return make_double2(0.0, 0.0); }
__device__ __forceinline__ float4 vzero(float4) { return make_float4(0.f, 0.f, 0.f, 0.f); }

#ifndef K1_GATHER_PF
#define K1_GATHER_PF 0  // 1: L2 prefetch of the next batch's gathered rows (B steps ahead);
                        // measured +19% (f64) / +33% (f32) K1 time on config 2: the extra
                        // requests compete with the gathers for L2 bandwidth
#endif
#ifndef K1_PREFETCH
#define K1_PREFETCH 1  // L2 prefetch of the epilogue's streamed rows at the start of each row set (fp64)
#endif
__device__ __forceinline__ void prefetch_l2(const void *p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// acc + a*x, separately rounded (fp64 strict) / fused (fp32)
#ifndef K1_FMA64
#define K1_FMA64 0  // 1: fused multiply-add in fp64 (not bit-identical to the reference; experiment)
#endif
__device__ __forceinline__ double2 vmadd(double2 acc, double a, double2 x) {
#if K1_FMA64
    return make_double2(fma(a, x.x, acc.x), fma(a, x.y, acc.y));
#else
    return make_double2(__dadd_rn(acc.x, __dmul_rn(a, x.x)), __dadd_rn(acc.y, __dmul_rn(a, x.y)));
#endif
}
__device__ __forceinline__ float4 vmadd(float4 acc, float a, float4 x) {
    return make_float4(fmaf(a, x.x, acc.x), fmaf(a, x.y, acc.y), fmaf(a, x.z, acc.z),
                       fmaf(a, x.w, acc.w));
}

// q = alpha*acc [- beta*p]  (numpy: q = alpha*y; q -= beta*q2)
__device__ __forceinline__ double2 vrecur(double2 acc, double alpha, double beta, double2 p,
                                          bool has_prev) {
    double2 q = make_double2(__dmul_rn(alpha, acc.x), __dmul_rn(alpha, acc.y));
    if (has_prev) {
        q.x = __dsub_rn(q.x, __dmul_rn(beta, p.x));
        q.y = __dsub_rn(q.y, __dmul_rn(beta, p.y));
    }
    return q;
}
__device__ __forceinline__ float4 vrecur(float4 acc, float alpha, float beta, float4 p,
                                         bool has_prev) {
    float4 q = make_float4(alpha * acc.x, alpha * acc.y, alpha * acc.z, alpha * acc.w);
    if (has_prev) {
        q.x = fmaf(-beta, p.x, q.x);
        q.y = fmaf(-beta, p.y, q.y);
        q.z = fmaf(-beta, p.z, q.z);
        q.w = fmaf(-beta, p.w, q.w);
    }
    return q;
}

// e + theta*q  (numpy: acc += theta*q)
__device__ __forceinline__ double2 vaccum(double2 e, double theta, double2 q) {
    return make_double2(__dadd_rn(e.x, __dmul_rn(theta, q.x)), __dadd_rn(e.y, __dmul_rn(theta, q.y)));
}
__device__ __forceinline__ float4 vaccum(float4 e, float theta, float4 q) {
    return make_float4(fmaf(theta, q.x, e.x), fmaf(theta, q.y, e.y), fmaf(theta, q.z, e.z),
                       fmaf(theta, q.w, e.w));
}

// monotone key of |v| for max tracking; NaN > inf > finite, as np.max propagates NaN
__device__ __forceinline__ unsigned long long absbits(double v) {
    return (unsigned long long)__double_as_longlong(v) & 0x7FFFFFFFFFFFFFFFull;
}
__device__ __forceinline__ unsigned long long vpeak(double2 q) {
    unsigned long long a = absbits(q.x), b = absbits(q.y);
    return a > b ? a : b;
}
__device__ __forceinline__ unsigned long long vpeak(float4 q) {
    unsigned int a = __float_as_uint(q.x) & 0x7FFFFFFFu, b = __float_as_uint(q.y) & 0x7FFFFFFFu;
    unsigned int c = __float_as_uint(q.z) & 0x7FFFFFFFu, d = __float_as_uint(q.w) & 0x7FFFFFFFu;
    a = a > b ? a : b;
    c = c > d ? c : d;
    a = a > c ? a : c;
    // widen to the fp64 key so both precisions share one diagnostics format
    return absbits((double)__uint_as_float(a));
}

// streaming (evict-first) accesses for data touched once per step
template <typename V> __device__ __forceinline__ V ld_stream(const V *p) { return __ldcs(p); }
template <typename V> __device__ __forceinline__ void st_stream(V *p, V v) { __stcs(p, v); }

#ifndef K1_MAX_PEERS
#define K1_MAX_PEERS 15  // remote replicas a step can write (16 ranks)
#endif

struct StepParams {
    const int64_t *rowptr;
    const int *cols;
    const void *vals;
    const void *ycur;  // Q(r-1): gathered
    void *yout;        // in: Q(r-2) (if has_prev), out: Q(r)
    void *E;           // accumulator (MODE_RECUR)
    int64_t n_rows;
    int ldv;           // row stride in 16-byte vectors
    int v0;            // first vector of this column tile
    int nvt;           // vectors in this column tile
    double alpha, beta, theta;
    // E update folding: E is read/written only on flush steps, which add the
    // pending terms in the reference's order, ((E + th2*Q(r-2)) + th1*Q(r-1)) + th*Q(r):
    // efold bit 1 = flush (add th*Q(r)), bit 2 = add th1*Q(r-1) (the row's own
    // row of the gather source), bit 4 = add th2*Q(r-2) (the loaded old value)
    int efold;
    double theta1, theta2;
    int64_t row_base;  // global index of local row 0 in the gather source (row partition)
    int smem_base;     // staged variant: byte offset of the per-warp rings (after the peak slots)
    int has_prev;
    int reverse;       // sweep rows in descending order (L2 reuse of the tail)
    unsigned long long *peaks;  // this step's per-chunk max|Q| keys (MODE_RECUR), or null
    int col0;          // global column of vector 0 (for chunk ids)
    // load-balance schedule (optional): row i of the sweep is perm[i]; entry
    // ranges [rbeg[r], rend[r]) replace rowptr (used for the split chunks of
    // heavy rows, which are written to yout at index r with MODE_SPMM)
    const int *perm;
    const int64_t *rbeg;
    const int64_t *rend;
    // fused exchange of the row partition (csemb_plan_partition_peers): every
    // Q(r) row is also stored, at its GLOBAL row, into each peer's replicated
    // full buffer over NVLink (P2P), so the transfer overlaps the step instead
    // of following it as an all-gather
    void *peer[K1_MAX_PEERS];
    int n_peer;
    // ... or through one NVLS multicast address of the full Q(r) buffer (all
    // ranks' replicas, this one included): one multimem store per 8 bytes that
    // the NVSwitch replicates, instead of n_peer unicast stores
    void *mc;
    // value-free normalized adjacency (csemb_plan option CSEMB_OPT_VALUE_FREE):
    // when *vf != 0 every stored value equals 1/sqrt(len(row) * len(col)) with
    // len = the stored row lengths (sparse.normalized_adjacency, sparse.py:224,
    // checked bit for bit on the device by k_vf_check), so K1 recomputes the
    // value from the row offsets instead of streaming it (null: read values)
    const int *vf;
    int hot_below;  // K1_HOTCOL experiment builds: columns below this allocate in L1, others do not (0: off)
};

__device__ __forceinline__ bool memcmp_eq(double a, double b) { return __double_as_longlong(a) == __double_as_longlong(b); }
__device__ __forceinline__ bool memcmp_eq(float a, float b) { return __float_as_uint(a) == __float_as_uint(b); }

// the reference's normalized-adjacency value, 1.0 / np.sqrt(deg[u] * deg[v])
// (sparse.py:224): exact integer product (< 2^53), IEEE sqrt and division,
// each correctly rounded -- then the run dtype's conversion, as the stored
// value got it
template <typename T>
__device__ __forceinline__ T vf_value(double len_row, const int64_t *__restrict__ rowptr, int j) {
    const int64_t lj = __ldg(rowptr + j + 1) - __ldg(rowptr + j);
    return (T)__ddiv_rn(1.0, __dsqrt_rn(__dmul_rn(len_row, (double)lj)));
}

// bit-exact 16-byte store through a multicast address (two multimem.st.b64;
// the vector forms take float types only)
__device__ __forceinline__ void mc_store(void *p, const void *v16) {
    const unsigned long long *w = reinterpret_cast<const unsigned long long *>(v16);
    asm volatile("multimem.st.relaxed.sys.global.b64 [%0], %1;" ::"l"(p), "l"(w[0]) : "memory");
    asm volatile("multimem.st.relaxed.sys.global.b64 [%0], %1;" ::"l"((char *)p + 8), "l"(w[1]) : "memory");
}

// Per-chunk diagnostics.  PEAK_EXACT keeps, per lane slot, the running max of
// the |Q| bit patterns (the reference's logged max_abs, engine.py:217-220);
// PEAK_FLAG keeps one bit per 32-column chunk touched by the lane that is set
// when a non-finite value appears (all the DivergenceError check needs) and
// costs one register instead of 2*VPL.
enum { PEAK_FLAG = 0, PEAK_EXACT = 1 };

__device__ __forceinline__ bool vfinite(double2 q) {
    return (absbits(q.x) < 0x7FF0000000000000ull) & (absbits(q.y) < 0x7FF0000000000000ull);
}
__device__ __forceinline__ bool vfinite(float4 q) {
    const unsigned m = 0x7F800000u;
    return ((__float_as_uint(q.x) & 0x7FFFFFFFu) < m) & ((__float_as_uint(q.y) & 0x7FFFFFFFu) < m) &
           ((__float_as_uint(q.z) & 0x7FFFFFFFu) < m) & ((__float_as_uint(q.w) & 0x7FFFFFFFu) < m);
}

#ifndef K1_MIN_BLOCKS
#define K1_MIN_BLOCKS 0  // 0: 2 CTAs/SM (128 registers) for both dtypes (measured best)
#endif
#ifndef K1_DEPTH
#define K1_DEPTH 0  // stored entries in flight per lane (divides G); 0: 4 for fp64, 2 for fp32
#endif
#ifndef K1_DEPTH_F64_SPILLY
#define K1_DEPTH_F64_SPILLY 2  // fp64 depth for the shapes that spill at 4 (4-lane groups, 32-lane SpMM, exact
                                // peaks): spill-free at 2; measured 1-1.6% faster at d = 20 / 24 (round 2)
#endif
#ifndef K1_DEPTH_F32
#define K1_DEPTH_F32 2  // fp32 entries in flight per lane (divides the batch)
#endif
#ifndef K1_BATCH
#define K1_BATCH 0  // stored entries per warp-uniform batch (<= G; 0: B = G, measured best)
#endif
#ifndef K1_VF
#define K1_VF 0  // 1: compile K1's value-free path in (CSEMB_OPT_VALUE_FREE).  Off: measured
                 // slower when used, and its mere presence costs the default path 0.5-3%
                 // (register allocation; profiles/r2_k1_experiments.txt)
#endif
#ifndef K1_TRIM
#define K1_TRIM 0  // 1: trim the warp's last batch to its longest row (rounded up to D)
#endif
#ifndef K1_EB8F32
#define K1_EB8F32 1  // fp32 entries per lane per batch for 8-lane groups
#endif
#ifndef K1_EB8
#define K1_EB8 2  // fp64 entries per lane per batch for 8-lane groups (measured, config 2 graph:
                  // d=40 f64 0.71 -> 0.67 ms; fp32 8-lane groups and 16-lane groups lose with 2)
#endif
#ifndef K1_QSTORE_CS
#define K1_QSTORE_CS 1  // store Q(r) evict-first (measured: <=1% faster than write-back)
#endif
#ifndef K1_ABLATE
#define K1_ABLATE 0  // timing experiments only (results are wrong when nonzero)
#endif

// Gathers of Q(r-1) rows: ld.global.nc (read-only path, L1-allocating, 128-byte
// line requests).  Measured on config 2: .cg / .nc.L1::no_allocate (L2 only)
// and an L2::evict_last policy were not faster.
#ifndef GATHER_MODE
#define GATHER_MODE 0  // 1: ld.global.nc.L1::no_allocate, 2: ld.global.cg (experiments)
#endif
#if GATHER_MODE == 1
#define GATHER_OP "ld.global.nc.L1::no_allocate"
#elif GATHER_MODE == 2
#define GATHER_OP "ld.global.cg"
#elif GATHER_MODE == 3
#define GATHER_OP "ld.global.nc.L2::256B"  // 256-byte L2 fills for gathered rows (experiment)
#elif GATHER_MODE == 4
#define GATHER_OP "ld.global.nc.L2::128B"
#else
#define GATHER_OP "ld.global.nc"
#endif
__device__ __forceinline__ double2 ld_gather(const double2 *p) {
    double2 v;
    asm(GATHER_OP ".v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ float4 ld_gather(const float4 *p) {
    float4 v;
    asm(GATHER_OP ".v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}

// Predicated gathers (branch-free: a not-taken load neither issues traffic nor
// splits the unrolled entry loop into separate basic blocks, so the scheduler
// can keep several entries' gathers in flight).
__device__ __forceinline__ double2 ld_gather_if(const double2 *p, bool ok) {
    double2 v = make_double2(0.0, 0.0);
    asm("{\n .reg .pred q;\n setp.ne.u32 q, %3, 0;\n @q " GATHER_OP ".v2.f64 {%0,%1}, [%2];\n}"
        : "+d"(v.x), "+d"(v.y) : "l"(p), "r"((unsigned)ok));
    return v;
}
__device__ __forceinline__ float4 ld_gather_if(const float4 *p, bool ok) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    asm("{\n .reg .pred q;\n setp.ne.u32 q, %5, 0;\n @q " GATHER_OP ".v4.f32 {%0,%1,%2,%3}, [%4];\n}"
        : "+f"(v.x), "+f"(v.y), "+f"(v.z), "+f"(v.w) : "l"(p), "r"((unsigned)ok));
    return v;
}
// Predicated gather INTO a live register: a load that is not taken leaves the
// register's previous contents, so no zero-fill instructions are issued per
// entry (2 CS2R per 16-byte slot).  Measured (round 2, tools/run_round2_b.sh):
// f64 d=80 -1%, but f64 d=40 +7% and f32 d=80 +15% K1 time (the "+" operands
// pin the buffers to fixed registers across the unrolled steps), and the
// fp32 config-1 parity test failed with it on -- so it is off (K1_KEEP_STALE 0,
// zero-filled predicated loads) and kept only as a measured experiment.
#ifndef K1_KEEP_STALE
#define K1_KEEP_STALE 0
#endif
__device__ __forceinline__ void ld_gather_into(double2 &v, const double2 *p, bool ok) {
    asm("{\n .reg .pred q;\n setp.ne.u32 q, %3, 0;\n @q " GATHER_OP ".v2.f64 {%0,%1}, [%2];\n}"
        : "+d"(v.x), "+d"(v.y) : "l"(p), "r"((unsigned)ok));
}
__device__ __forceinline__ void ld_gather_into(float4 &v, const float4 *p, bool ok) {
    asm("{\n .reg .pred q;\n setp.ne.u32 q, %5, 0;\n @q " GATHER_OP ".v4.f32 {%0,%1,%2,%3}, [%4];\n}"
        : "+f"(v.x), "+f"(v.y), "+f"(v.z), "+f"(v.w) : "l"(p), "r"((unsigned)ok));
}
#ifndef K1_HOTCOL
#define K1_HOTCOL 0  // 1 (experiment build): gathers of columns >= StepParams::hot_below do not allocate in L1
#endif
// predicated L1-no-allocate gather into a live register (K1_HOTCOL experiment)
__device__ __forceinline__ void ld_gather_na_into(double2 &v, const double2 *p, bool ok) {
    asm("{\n .reg .pred q;\n setp.ne.u32 q, %3, 0;\n @q ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];\n}"
        : "+d"(v.x), "+d"(v.y) : "l"(p), "r"((unsigned)ok));
}
__device__ __forceinline__ void ld_gather_na_into(float4 &v, const float4 *p, bool ok) {
    asm("{\n .reg .pred q;\n setp.ne.u32 q, %5, 0;\n @q ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];\n}"
        : "+f"(v.x), "+f"(v.y), "+f"(v.z), "+f"(v.w) : "l"(p), "r"((unsigned)ok));
}
__device__ __forceinline__ double2 vsel(bool c, double2 a, double2 b) {
    return make_double2(c ? a.x : b.x, c ? a.y : b.y);
}
__device__ __forceinline__ float4 vsel(bool c, float4 a, float4 b) {
    return make_float4(c ? a.x : b.x, c ? a.y : b.y, c ? a.z : b.z, c ? a.w : b.w);
}

// ---- TMA bulk copies + mbarriers (staged K1) ----------------------------------
#ifndef K1T_STAGES
#define K1T_STAGES 8  // neighbour rows in flight per group in the staged variant
#endif
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, unsigned parity) {
    unsigned ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    return ok != 0;
}
// per-lane 16-byte async copy (LDGSTS); src_bytes 0 zero-fills without reading global
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem), "r"(src_bytes)
                 : "memory");
}
// per-lane 4- / 8-byte async copies (index / value staging, STAGED == 3)
#ifndef K1_SIDX_HINT
#define K1_SIDX_HINT 0  // 1: L2 evict-first policy on the staged index / value copies (experiment)
#endif
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
template <int BYTES>
__device__ __forceinline__ void cp_async_small(void *smem, const void *gmem, uint64_t pol) {
#if K1_SIDX_HINT
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], %2, %3;" ::"r"(smem_u32(smem)), "l"(gmem), "n"(BYTES), "l"(pol)
                 : "memory");
#else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(smem)), "l"(gmem), "n"(BYTES) : "memory");
#endif
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// one neighbour-row tile (global -> shared), completion counted on `bar`
__device__ __forceinline__ void tma_row(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// K1: one recurrence step (MODE_RECUR) or a plain multi-vector SpMM (MODE_SPMM).
// A group of G lanes owns a row; lane gl holds the 16-byte vectors gl + k*G
// (k < VPL) of the row's column tile.  The warp's 32/G rows advance together
// through batches of G stored entries: lane t of a group loads entry base+t
// (coalesced), the batch is broadcast with full-warp shuffles (the batch loop
// is warp-uniform, so there are no divergence checks in it), and every lane
// issues VPL independent 16-byte gathers per entry, consumed strictly in
// stored order (bit-exact fp64 accumulation order).  The next batch's entries
// -- or the next row's first batch -- are loaded while the current batch's
// gathers are outstanding.  Streamed data (entries, Q(r-2), E) is read
// evict-first so L2 keeps the gathered rows of Q(r-1).
template <typename T, int G, int VPL, int MODE, int PEAK, int STAGED = 0, int PEERS = 0>
__global__ void __launch_bounds__(256, (K1_MIN_BLOCKS ? K1_MIN_BLOCKS : 2)) k_step(const StepParams P) {
    extern __shared__ __align__(128) unsigned char k1_dyn_smem[];
    typedef typename Vec<T>::type VT;
    constexpr int W = Vec<T>::W;
    constexpr int RPW = 32 / G;  // rows per warp
    const int lane = threadIdx.x & 31;
    const int gl = lane & (G - 1);
    const int grp = lane / G;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t wstride = (((int64_t)gridDim.x * blockDim.x) >> 5) * RPW;

    const T *__restrict__ vals = (const T *)P.vals;
    const int *__restrict__ cols = P.cols;
    const VT *__restrict__ ycur = (const VT *)P.ycur + P.v0 + gl;
    VT *yout = (VT *)P.yout;
    VT *E = (VT *)P.E;
    const T alpha = (T)P.alpha, beta = (T)P.beta, theta = (T)P.theta;
    const T theta1 = (T)P.theta1, theta2 = (T)P.theta2;
    const bool has_prev = P.has_prev != 0;
    const int first_chunk = (P.col0 + P.v0 * W) >> 5;
    const bool vfree = K1_VF && P.vf != nullptr && *P.vf != 0;  // warp-uniform

    bool valid[VPL];
#pragma unroll
    for (int k = 0; k < VPL; ++k) valid[k] = (gl + k * G) < P.nvt;
#if K1_GATHER_PF
    const int pf_lines = (P.nvt * 16 + 127) / 128 + 1;  // 128-byte lines a row tile touches (+1: alignment)
#endif
    unsigned long long pk[PEAK == PEAK_EXACT ? VPL : 1];
#pragma unroll
    for (int k = 0; k < (PEAK == PEAK_EXACT ? VPL : 1); ++k) pk[k] = 0ull;
    unsigned badmask = 0u;

    auto row_of = [&](int64_t it) -> int64_t {  // -1 for the idle tail groups of the last warp
        if (it >= P.n_rows) return -1;
        const int64_t i = P.reverse ? (P.n_rows - 1 - it) : it;
        return P.perm ? (int64_t)__ldg(P.perm + i) : i;
    };
    auto extent = [&](int64_t r, int64_t &b, int64_t &e) {
        if (P.rbeg) {
            b = __ldg(P.rbeg + r);
            e = __ldg(P.rend + r);
        } else {
            b = __ldg(P.rowptr + r);
            e = __ldg(P.rowptr + r + 1);
        }
    };
    // current row's extent and first entry batch, loaded one row ahead
    int64_t it = warp * RPW + grp;
    int64_t beg = 0, end = 0;
    if (it < P.n_rows) {
        extent(row_of(it), beg, end);
    }
    // Stored entries advance in warp-uniform batches of B.  Narrow groups hold
    // EB entries per lane (8 / 4 / 2 for 1 / 2 / 4 lanes, 2 for 8 lanes in fp64),
    // so a batch spans 8-16 entries: the next batch's column ids and values are loaded that
    // many steps before use (with one entry per lane, a 1-lane group would wait
    // on an index load at every entry).  Entry t of a
    // batch sits in lane t % G, slot t / G; wide groups keep B = G (or K1_BATCH).
    constexpr int EB = G == 1 ? 8 : G == 2 ? 4 : G == 4 ? 2 : G == 8 ? (sizeof(T) == 8 ? K1_EB8 : K1_EB8F32) : 1;
    constexpr int B = EB > 1 ? G * EB : ((K1_BATCH > 0 && K1_BATCH < G) ? K1_BATCH : G);
    static_assert(EB > 1 || G % B == 0, "batch width must divide the group width");
    constexpr int BL = EB > 1 ? G : B;  // lanes that hold the batch
    // len: the row's stored length (its degree, for the value-free form)
    auto load_batch = [&](int64_t b0, int64_t e0, int64_t len, int (&j)[EB], T (&a)[EB]) {
#pragma unroll
        for (int k = 0; k < EB; ++k) {
            j[k] = 0;
            a[k] = (T)0;
            const int64_t q = b0 + gl + k * G;
            if (gl < BL && q < e0) {
                j[k] = __ldcs(cols + q);
                if (vfree)
                    a[k] = vf_value<T>((double)len, P.rowptr, j[k]);
                else
                    a[k] = __ldcs(vals + q);
            }
        }
    };
    // entry t (compile-time) of a batch held in (j or a)[EB], broadcast to the group
    auto bcast_j = [&](const int (&j)[EB], int t) { return __shfl_sync(0xFFFFFFFFu, j[t / G], t % G, G); };
    auto bcast_a = [&](const T (&a)[EB], int t) { return __shfl_sync(0xFFFFFFFFu, a[t / G], t % G, G); };
    int myj[EB];
    T mya[EB];

    // Gathers of the first D-1 entries of the current batch are carried across
    // batches.  Register variant: D-deep rotating register buffer.  Staged
    // variant (STAGED): lane 0 of each group issues one TMA bulk copy of the
    // neighbour's row tile into a warp-private S-stage shared-memory ring; the
    // group waits on the stage's mbarrier and consumes it from shared memory.
    // VPL > 3 (K1_WIDE_VPL builds): the register budget allows only 2 entries in flight
    constexpr int DEPTH = K1_DEPTH ? K1_DEPTH
                                   : (VPL > 3 ? 2
                                              : (sizeof(T) == 8 ? ((G == 4 || (G == 32 && MODE == MODE_SPMM) || PEAK == PEAK_EXACT)
                                                                       ? K1_DEPTH_F64_SPILLY : 4)
                                                                : K1_DEPTH_F32));
    // RING: the gathered rows go through shared memory (STAGED 1 / 2); SIDX
    // (STAGED 3): the gathers stay in registers and the column-index / value
    // batches are staged in a warp-private shared-memory double buffer instead
    constexpr bool RING = STAGED == 1 || STAGED == 2;
    constexpr bool SIDX = STAGED == 3 || STAGED == 4;
    constexpr bool SREG = STAGED == 4;  // the batch travels LDG.cs -> registers -> STS instead of cp.async
    constexpr int D = RING ? ((K1T_STAGES < B) ? K1T_STAGES : B) : ((DEPTH < B) ? DEPTH : B);
    // STAGED == 2: per-lane ring of D entries x VPL 16-byte slots in shared memory
    VT *lring = nullptr;
    if constexpr (STAGED == 2)
        lring = reinterpret_cast<VT *>(k1_dyn_smem + P.smem_base) + (size_t)threadIdx.x * VPL;
    static_assert(B % D == 0, "pipeline depth must divide the batch width");
    // SIDX: warp-private double buffer of entry batches in shared memory, slot =
    // [RPW][B] column ids then [RPW][B] values.  Lane t % G of a group copies
    // entry t of its row's batch with a 4- / 8-byte cp.async (padding entries are
    // stored as zeros); every lane of the group then reads entry t back with one
    // broadcast LDS instead of a shuffle.  `scur` (warp-uniform) is the slot of
    // the current batch, scur ^ 1 receives the next one while this one is consumed.
    constexpr int SLOT_BYTES = RPW * B * (4 + (int)sizeof(T));
    unsigned char *sidx = nullptr;
    if constexpr (SIDX) sidx = k1_dyn_smem + P.smem_base + (size_t)(threadIdx.x >> 5) * 2 * SLOT_BYTES;
    int scur = 0;
    const uint64_t sidx_pol = (SIDX && K1_SIDX_HINT) ? l2_evict_first_policy() : 0ull;
    auto slot_j = [&](int slot) { return reinterpret_cast<int *>(sidx + slot * SLOT_BYTES) + grp * B; };
    auto slot_a = [&](int slot) { return reinterpret_cast<T *>(sidx + slot * SLOT_BYTES + RPW * B * 4) + grp * B; };
    int pj[EB];  // SREG: the batch in flight (registers) and its slot
    T pa[EB];
    int pslot = 0;
    auto stage_batch = [&](int64_t b0, int64_t e0, int slot) {
        if constexpr (SREG) {
            pslot = slot;
#pragma unroll
            for (int k = 0; k < EB; ++k) {
                const int64_t q = b0 + gl + k * G;
                pj[k] = 0;
                pa[k] = (T)0;
                if (gl < BL && q < e0) {
                    pj[k] = __ldcs(cols + q);
                    pa[k] = __ldcs(vals + q);
                }
            }
            return;
        }
        __syncwarp();  // the slot's previous contents have been read by every lane
        int *dj = slot_j(slot);
        T *da = slot_a(slot);
#pragma unroll
        for (int k = 0; k < EB; ++k) {
            const int t = gl + k * G;
            const int64_t q = b0 + t;
            if (gl < BL) {
                if (q < e0) {
                    cp_async_small<4>(dj + t, cols + q, sidx_pol);
                    cp_async_small<(int)sizeof(T)>(da + t, vals + q, sidx_pol);
                } else {
                    dj[t] = 0;
                    da[t] = (T)0;
                }
            }
        }
        cp_async_commit();
    };
    auto stage_wait = [&]() {  // the staged batch is visible to the whole warp
        if constexpr (SREG) {
            __syncwarp();  // the slot's previous contents have been read by every lane
            int *dj = slot_j(pslot);
            T *da = slot_a(pslot);
#pragma unroll
            for (int k = 0; k < EB; ++k)
                if (gl < BL) {
                    dj[gl + k * G] = pj[k];
                    da[gl + k * G] = pa[k];
                }
            __syncwarp();
            return;
        }
        cp_async_wait<0>();
        __syncwarp();
    };
    auto sjr = [&](int slot, int t) { return *reinterpret_cast<volatile int *>(slot_j(slot) + t); };
    auto sar = [&](int slot, int t) { return *reinterpret_cast<volatile T *>(slot_a(slot) + t); };
    if constexpr (SIDX) {
        static_assert(!K1_TRIM, "index staging has no trimmed-batch path");
        stage_batch(beg, end, 0);
        stage_wait();
    } else {
        load_batch(beg, end, end - beg, myj, mya);
    }
    VT buf[RING ? 1 : D][VPL];
#pragma unroll
    for (int i = 0; i < (RING ? 1 : D); ++i)
#pragma unroll
        for (int k = 0; k < VPL; ++k) buf[i][k] = vzero(VT());
    uint64_t *bars = nullptr;
    VT *ring = nullptr;
    unsigned phase = 0u;  // staged: bit s = parity to wait for on stage s
    const VT *ybase = (const VT *)P.ycur + P.v0;
    const unsigned row_bytes = (unsigned)P.nvt * 16u;
    if constexpr (STAGED == 1) {
        unsigned char *wb = k1_dyn_smem + P.smem_base +
                            (size_t)(threadIdx.x >> 5) * (128 + (size_t)D * RPW * row_bytes);
        bars = reinterpret_cast<uint64_t *>(wb);
        ring = reinterpret_cast<VT *>(wb + 128);
        if (lane < D) mbar_init(bars + lane, RPW);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        __syncwarp();
    }
    auto issue = [&](int slot, int j, bool ok) {
        if constexpr (STAGED == 2) {
            // no copy at all for padding entries / unused vectors: a zero-fill copy
            // (src_bytes 0) still fetched the source line and doubled L2->SM bytes
            const VT *x = ycur + (int64_t)j * P.ldv;
            VT *dst = lring + (size_t)slot * blockDim.x * VPL;
#pragma unroll
            for (int k = 0; k < VPL; ++k)
                if (valid[k] && ok) cp_async16(dst + k, x + k * G, 16);
            cp_async_commit();
        } else if constexpr (STAGED == 1) {
            if (gl == 0) {
                if (ok) {
                    mbar_arrive_tx(bars + slot, row_bytes);
                    tma_row(ring + ((size_t)slot * RPW + grp) * P.nvt, ybase + (int64_t)j * P.ldv, row_bytes, bars + slot);
                } else {
                    mbar_arrive(bars + slot);
                }
            }
        } else {
            const VT *x = ycur + (int64_t)j * P.ldv;
#if K1_HOTCOL
            if (P.hot_below > 0) {  // warp-uniform: hot columns allocate in L1, the rest bypass it
                const bool hot = j < P.hot_below;
#pragma unroll
                for (int k = 0; k < VPL; ++k) {
                    buf[slot][k] = ld_gather_if(x + k * G, valid[k] && ok && hot);
                    ld_gather_na_into(buf[slot][k], x + k * G, valid[k] && ok && !hot);
                }
                return;
            }
#endif
#pragma unroll
            for (int k = 0; k < VPL; ++k) {
                if (K1_KEEP_STALE)
                    ld_gather_into(buf[slot][k], x + k * G, valid[k] && ok);
                else
                    buf[slot][k] = ld_gather_if(x + k * G, valid[k] && ok);
            }
        }
    };
#pragma unroll
    for (int e = 0; e < D - 1; ++e) issue(e, SIDX ? sjr(0, e) : bcast_j(myj, e), e < end - beg);

    for (int64_t wbase = warp * RPW; wbase < P.n_rows; wbase += wstride) {  // warp-uniform
        const bool active = it < P.n_rows;
        const int64_t row = row_of(it);
        const int64_t it2 = it + wstride;
        int64_t beg2 = 0, end2 = 0;
        if (it2 < P.n_rows) {
            extent(row_of(it2), beg2, end2);
        }
        const int len = (int)(end - beg);
        const int nb_mine = (len + B - 1) / B;
        // the warp's batch count, from its longest row (needed by K1_TRIM) or from
        // the rows' batch counts -- the same number; the choice only moves code
        // generation, and was measured: from the length, fp32 K1 is 5% faster on
        // config 4 and 1.4% on config 3, fp64 1.3% slower on config 2
        constexpr bool NB_FROM_LEN = K1_TRIM || sizeof(T) == 4;
        const int smax = NB_FROM_LEN ? (int)__reduce_max_sync(0xFFFFFFFFu, (unsigned)len) : 0;
        const int nb = NB_FROM_LEN ? (smax + B - 1) / B : (int)__reduce_max_sync(0xFFFFFFFFu, (unsigned)nb_mine);
#if K1_PREFETCH
        // the epilogue's streamed rows (Q(r-2), E, own Q(r-1)) are requested into
        // L2 now, so the loads after the gather loop hit L2 instead of DRAM
        // (fp64 only: measured -2.5% on config 2 f64, +5% on the issue-bound f32 tiles)
        if (MODE == MODE_RECUR && sizeof(T) == 8 && active) {
            const VT *pq = yout + row * (int64_t)P.ldv + P.v0 + gl;
            const VT *pe = E + row * (int64_t)P.ldv + P.v0 + gl;
            const VT *po = ycur + (P.row_base + row) * (int64_t)P.ldv;
#pragma unroll
            for (int k = 0; k < VPL; ++k) {
                if (valid[k]) {
                    if (has_prev) prefetch_l2(pq + k * G);
                    if (P.efold) prefetch_l2(pe + k * G);
                    if (P.efold & 2) prefetch_l2(po + k * G);
                }
            }
        }
#endif

        VT acc[VPL];
#pragma unroll
        for (int k = 0; k < VPL; ++k) acc[k] = vzero(VT());

        for (int b = 0; b < nb; ++b) {
            // prefetch the next batch of this row, else the next row's first batch
            int nj[EB];
            T na[EB];
            int ncnt = 0;  // entries of that next batch for my row
            if constexpr (SIDX) {
                int64_t nb0 = 0, ne0 = 0;  // empty range: a batch of zeros
                if (b + 1 < nb_mine) {
                    ncnt = len - (b + 1) * B;
                    nb0 = beg + (b + 1) * B;
                    ne0 = end;
                } else if (b + 1 >= nb) {
                    ncnt = (int)(end2 - beg2);
                    nb0 = beg2;
                    ne0 = end2;
                }
                stage_batch(nb0, ne0, scur ^ 1);
            } else if (b + 1 < nb_mine) {
                ncnt = len - (b + 1) * B;
                load_batch(beg + (b + 1) * B, end, end - beg, nj, na);
            } else if (b + 1 >= nb) {
                ncnt = (int)(end2 - beg2);
                load_batch(beg2, end2, end2 - beg2, nj, na);
            } else {
#pragma unroll
                for (int k = 0; k < EB; ++k) {
                    nj[k] = 0;
                    na[k] = (T)0;
                }
            }
            const int cnt = len - b * B;  // entries of this batch for my row (may be <= 0)
            // branch-free pipeline, D entries deep: step t issues entry t+D-1
            // (spilling into the NEXT batch's first entries near the end, so no
            // batch or row-set epilogue starts with an empty pipeline) and consumes t.
            // K1_TRIM: the warp's last batch runs only its longest row's remaining
            // entries rounded up to D (a multiple of D keeps slot = step % D); the
            // entries it spills into the next batch are then the first D-1 <= G,
            // all in register slot 0 of their lanes.
            constexpr bool TRIM = K1_TRIM && STAGED == 0 && D - 1 <= G;
            const int nst = (TRIM && b + 1 == nb) ? min(B, (smax - b * B + D - 1) / D * D) : B;
            auto step = [&](const int t, const int ns, auto full_tag) {
                [[maybe_unused]] constexpr bool FULL = decltype(full_tag)::value;
#if K1_GATHER_PF
                // L2 prefetch of entry t of the NEXT batch (B steps ahead, no registers):
                // lanes gl < pf_lines each request one 128-byte line of that row, so the
                // register gather D steps ahead finds it in L2
                if constexpr (STAGED == 0) {
                    const int jn = bcast_j(nj, t);
                    if (gl < pf_lines && t < ncnt)
                        prefetch_l2(reinterpret_cast<const char *>(ycur - gl + (int64_t)jn * P.ldv) + gl * 128);
                }
#endif
                const int e = t + D - 1;
                int j;
                bool more;
                if constexpr (SIDX) {
                    // the next batch is first read at step B - D + 1 (entry e = B)
                    if (D > 1 && t == B - D + 1) stage_wait();
                    j = sjr(e < B ? scur : scur ^ 1, e % B);
                    more = (e < B) ? (e < cnt) : (e - B < ncnt);
                } else if constexpr (FULL) {
                    j = (e < B) ? bcast_j(myj, e % B) : bcast_j(nj, e % B);
                    more = (e < B) ? (e < cnt) : (e - B < ncnt);
                } else {
                    const bool cur = e < ns;
                    const int src = cur ? myj[(e < B ? e : 0) / G] : nj[0];
                    j = __shfl_sync(0xFFFFFFFFu, src, cur ? e % G : e - ns, G);
                    more = cur ? (e < cnt) : (e - ns < ncnt);
                }
                if (D > 1) issue(e % D, j, more);
                T a;
                if constexpr (SIDX)
                    a = sar(scur, t);
                else
                    a = bcast_a(mya, t);
                if (D == 1) issue(0, j, more);
                if constexpr (STAGED == 2) {
                    cp_async_wait<D - 1>();  // entry t has landed (this lane's own copies)
                    const VT *src = lring + (size_t)(t % D) * blockDim.x * VPL;
                    const bool ok = t < cnt;  // padding steps were never copied: skip them
#pragma unroll
                    for (int k = 0; k < VPL; ++k) acc[k] = vsel(ok, vmadd(acc[k], a, src[k]), acc[k]);
                } else if constexpr (STAGED == 1) {
                    const int slot = t % D;
                    const unsigned par = (phase >> slot) & 1u;
                    for (unsigned spins = 0; !mbar_try_wait(bars + slot, par);) {
                        if (++spins > (1u << 26)) __trap();  // a lost copy must fail loudly, not hang
                    }
                    phase ^= 1u << slot;
                    const VT *src = ring + ((size_t)slot * RPW + grp) * P.nvt + gl;
                    const bool ok = t < cnt;  // padding steps were never copied: skip them
#pragma unroll
                    for (int k = 0; k < VPL; ++k)
                        if (valid[k]) acc[k] = vsel(ok, vmadd(acc[k], a, src[k * G]), acc[k]);
                    __syncwarp();  // the stage is re-issued D-1 steps later
                } else {
                    // a padded step (t >= cnt) has a == 0 and a zero vector: acc + (+0) == acc
                    // exactly, because acc is never -0 (it starts at +0, as scipy's y does)
#pragma unroll
                    for (int k = 0; k < VPL; ++k) acc[k] = vmadd(acc[k], a, buf[t % D][k]);
                }
            };
            if (nst == B) {
#pragma unroll
                for (int t = 0; t < B; ++t) step(t, B, std::true_type{});
            } else {
#pragma unroll
                for (int t = 0; t < B; ++t) {
                    if (t % D == 0 && t >= nst) break;  // warp-uniform
                    step(t, nst, std::false_type{});
                }
            }
            if constexpr (SIDX) {
                if (D == 1) stage_wait();
                scur ^= 1;
            } else if (b + 1 < nb_mine || b + 1 >= nb) {
#pragma unroll
                for (int k = 0; k < EB; ++k) {
                    myj[k] = nj[k];
                    mya[k] = na[k];
                }
            }
        }
        if (nb == 0) {  // every row of the warp is empty: move to the next rows' first batch
            if constexpr (SIDX) {
                stage_batch(beg2, end2, scur);
                stage_wait();
            } else {
                load_batch(beg2, end2, end2 - beg2, myj, mya);
            }
#pragma unroll
            for (int e = 0; e < D - 1; ++e) issue(e, SIDX ? sjr(scur, e) : bcast_j(myj, e), e < end2 - beg2);
        }

        if (active) {
            VT *yo = yout + row * (int64_t)P.ldv + P.v0 + gl;
            if (MODE == MODE_SPMM) {
#pragma unroll
                for (int k = 0; k < VPL; ++k)
                    if (valid[k]) yo[k * G] = acc[k];
            } else {
                VT *er = E + row * (int64_t)P.ldv + P.v0 + gl;
                const VT *own = ycur + (P.row_base + row) * (int64_t)P.ldv;  // this row of Q(r-1)
                // issue every streamed load of the epilogue before any arithmetic
                VT pv[VPL], ev[VPL], ov[VPL];
#pragma unroll
                for (int k = 0; k < VPL; ++k) {
                    pv[k] = ev[k] = ov[k] = vzero(VT());
                    if (valid[k]) {
#if !(K1_ABLATE & 1)
                        if (has_prev) pv[k] = ld_stream(yo + k * G);
                        if (P.efold) ev[k] = ld_stream(er + k * G);
                        if (P.efold & 2) ov[k] = ld_gather(own + k * G);
#endif
                    }
                }
#pragma unroll
                for (int k = 0; k < VPL; ++k) {
                    if (valid[k]) {
                        const VT q = vrecur(acc[k], alpha, beta, pv[k], has_prev);
#if (K1_ABLATE & 4)
                        if (__double_as_longlong((double)vpeak(q)) == 12345) yo[k * G] = q;
#else
                        if constexpr (PEERS == 2) {  // every replica (this one too) through the multicast address
                            const int64_t off = (P.row_base + row) * (int64_t)P.ldv + P.v0 + gl + k * G;
                            mc_store(reinterpret_cast<VT *>(P.mc) + off, &q);
                        } else {
#if K1_QSTORE_CS
                            st_stream(yo + k * G, q);
#else
                            yo[k * G] = q;
#endif
                        }
                        if constexpr (PEERS == 1) {  // the same row of every peer's full Q(r) buffer
                            const int64_t off = (P.row_base + row) * (int64_t)P.ldv + P.v0 + gl + k * G;
                            for (int pi = 0; pi < P.n_peer; ++pi) reinterpret_cast<VT *>(P.peer[pi])[off] = q;
                        }
                        if (P.efold) {  // ((E + th2*Q(r-2)) + th1*Q(r-1)) + th*Q(r), the reference's order
                            VT e = ev[k];
                            if (P.efold & 4) e = vaccum(e, theta2, pv[k]);
                            if (P.efold & 2) e = vaccum(e, theta1, ov[k]);
                            st_stream(er + k * G, vaccum(e, theta, q));
                        }
#endif
                        if (PEAK == PEAK_EXACT) {
                            const unsigned long long bq = vpeak(q);
                            unsigned long long &m = pk[PEAK == PEAK_EXACT ? k : 0];
                            m = bq > m ? bq : m;
                        } else if (!vfinite(q)) {
                            badmask |= 1u << (((P.col0 + (P.v0 + gl + k * G) * W) >> 5) - first_chunk);
                        }
                    }
                }
            }
        }
        it = it2;
        beg = beg2;
        end = end2;
    }

    if constexpr (STAGED == 2 || STAGED == 3) cp_async_wait<0>();
    if constexpr (PEERS == 2) asm volatile("fence.proxy.alias;" ::: "memory");  // multicast vs unicast aliases
    if constexpr (PEERS) __threadfence_system();  // peer stores performed before the step's barrier
    if (MODE == MODE_RECUR && P.peaks) {
        // per-chunk max over the block, then one atomic per chunk per block
        unsigned long long *s_peak = reinterpret_cast<unsigned long long *>(k1_dyn_smem);
        const int last_chunk = (P.col0 + (P.v0 + P.nvt) * W - 1) >> 5;
        const int nch = last_chunk - first_chunk + 1;
        for (int c = threadIdx.x; c < nch; c += blockDim.x) s_peak[c] = 0ull;
        __syncthreads();
        if (PEAK == PEAK_EXACT) {
#pragma unroll
            for (int k = 0; k < VPL; ++k) {
                const unsigned long long v = pk[PEAK == PEAK_EXACT ? k : 0];
                if (valid[k] && v) {
                    const int c = ((P.col0 + (P.v0 + gl + k * G) * W) >> 5) - first_chunk;
                    atomicMax(&s_peak[c], v);
                }
            }
        } else {
            // non-finite marker: the +inf key (every finite |Q| key is below it)
            for (unsigned m = badmask; m; m &= m - 1) atomicMax(&s_peak[__ffs(m) - 1], 0x7FF0000000000000ull);
        }
        __syncthreads();
        for (int c = threadIdx.x; c < nch; c += blockDim.x)
            if (s_peak[c]) atomicMax(&P.peaks[first_chunk + c], s_peak[c]);
    }
}

// ---------------------------------------------------------------------------
// K1c: heavy rows.  Rows longer than the split threshold are cut into fixed
// chunks whose partial sums K1 computes in parallel (MODE_SPMM over the chunk
// ranges, written to `partials`); this kernel adds a row's partials in chunk
// order (deterministic, independent of the launch shape) and runs the same
// fused epilogue as K1.  One warp per heavy row, lanes over the row's vectors.
// ---------------------------------------------------------------------------
struct HeavyParams {
    const int *rows;        // heavy row ids
    const int *chunk_off;   // chunks of heavy row h: [chunk_off[h], chunk_off[h+1])
    const void *partials;   // n_chunks x ldv vectors
    int n_heavy;
    // split row partition (csemb_plan_partition_split): every row 0..n_heavy-1
    // in order, acc = (+0 + partials[row]) + partials2[row] -- the local-column
    // and remote-column partial sums -- then the same epilogue
    const void *partials2;
};

template <typename T, int MODE, int PEAK, int MS>
__global__ void __launch_bounds__(256) k_heavy_combine(const StepParams P, const HeavyParams H) {
    typedef typename Vec<T>::type VT;
    constexpr int W = Vec<T>::W;
    // MS vectors per lane (a tile has at most 96 vectors); U chunk partials in
    // flight per lane: the longest heavy rows (10^6 entries, ~2000 chunks) set
    // this kernel's time, one dependent round of loads per U chunks
    constexpr int U = MS == 1 ? 24 : (MS == 2 ? 12 : 8);
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const VT *part = (const VT *)H.partials + P.v0 + lane;
    VT *yout = (VT *)P.yout;
    VT *E = (VT *)P.E;
    const T alpha = (T)P.alpha, beta = (T)P.beta, theta = (T)P.theta;
    const bool has_prev = P.has_prev != 0;
    const int first_chunk = (P.col0 + P.v0 * W) >> 5;
    bool valid[MS];
#pragma unroll
    for (int k = 0; k < MS; ++k) valid[k] = (lane + 32 * k) < P.nvt;
    unsigned long long pk[MS];
#pragma unroll
    for (int k = 0; k < MS; ++k) pk[k] = 0ull;
    unsigned badmask = 0u;
    const VT *part2 = H.partials2 ? (const VT *)H.partials2 + P.v0 + lane : nullptr;
    for (int64_t h = warp; h < H.n_heavy; h += nwarps) {
        const int64_t row = part2 ? h : H.rows[h];
        const int c0 = part2 ? 0 : H.chunk_off[h], c1 = part2 ? 0 : H.chunk_off[h + 1];
        VT acc[MS];
#pragma unroll
        for (int k = 0; k < MS; ++k) acc[k] = vzero(VT());
        if (part2) {
#pragma unroll
            for (int k = 0; k < MS; ++k)
                if (valid[k]) {
                    const VT a = part[h * P.ldv + 32 * k], b = part2[h * P.ldv + 32 * k];
                    acc[k] = vmadd(vmadd(acc[k], (T)1, a), (T)1, b);
                }
        }
        // chunk partials in chunk order; U chunks' loads in flight at a time
        int c = c0;
        for (; c + U <= c1; c += U) {
            VT x[U][MS];
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int k = 0; k < MS; ++k)
                    x[u][k] = valid[k] ? part[(int64_t)(c + u) * P.ldv + 32 * k] : vzero(VT());
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int k = 0; k < MS; ++k)
                    if (valid[k]) acc[k] = vmadd(acc[k], (T)1, x[u][k]);
        }
        for (; c < c1; ++c) {
#pragma unroll
            for (int k = 0; k < MS; ++k)
                if (valid[k]) acc[k] = vmadd(acc[k], (T)1, part[(int64_t)c * P.ldv + 32 * k]);
        }
        VT *yo = yout + row * (int64_t)P.ldv + P.v0 + lane;
        if (MODE == MODE_SPMM) {
#pragma unroll
            for (int k = 0; k < MS; ++k)
                if (valid[k]) yo[32 * k] = acc[k];
            continue;
        }
        VT *er = E + row * (int64_t)P.ldv + P.v0 + lane;
        const VT *own = (const VT *)P.ycur + (P.row_base + row) * (int64_t)P.ldv + P.v0 + lane;
#pragma unroll
        for (int k = 0; k < MS; ++k) {
            if (!valid[k]) continue;
            const VT p = has_prev ? ld_stream(yo + 32 * k) : vzero(VT());
            const VT q = vrecur(acc[k], alpha, beta, p, has_prev);
            const int64_t off = (P.row_base + row) * (int64_t)P.ldv + P.v0 + lane + 32 * k;
            if (P.mc) {  // fused exchange (see StepParams::peer / mc)
                mc_store(reinterpret_cast<VT *>(P.mc) + off, &q);
            } else {
                yo[32 * k] = q;
                for (int pi = 0; pi < P.n_peer; ++pi) reinterpret_cast<VT *>(P.peer[pi])[off] = q;
            }
            if (P.efold) {
                VT e = ld_stream(er + 32 * k);
                if (P.efold & 4) e = vaccum(e, (T)P.theta2, p);
                if (P.efold & 2) e = vaccum(e, (T)P.theta1, ld_gather(own + 32 * k));
                st_stream(er + 32 * k, vaccum(e, theta, q));
            }
            if (PEAK == PEAK_EXACT) {
                const unsigned long long bq = vpeak(q);
                pk[k] = bq > pk[k] ? bq : pk[k];
            } else if (!vfinite(q)) {
                badmask |= 1u << (((P.col0 + (P.v0 + lane + 32 * k) * W) >> 5) - first_chunk);
            }
        }
    }
    if (P.mc) asm volatile("fence.proxy.alias;" ::: "memory");
    if (P.n_peer || P.mc) __threadfence_system();
    if (MODE == MODE_RECUR && P.peaks) {
#pragma unroll
        for (int k = 0; k < MS; ++k) {
            if (PEAK == PEAK_EXACT && valid[k] && pk[k]) {
                const int c = (P.col0 + (P.v0 + lane + 32 * k) * W) >> 5;
                atomicMax(&P.peaks[c], pk[k]);
            }
        }
        for (unsigned m = badmask; m; m &= m - 1) atomicMax(&P.peaks[first_chunk + __ffs(m) - 1], 0x7FF0000000000000ull);
    }
}

// ---------------------------------------------------------------------------
// K2: projection block / stage input
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Philox4x32-10 (Salmon et al., SC'11), returns output word 0
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        const unsigned hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const unsigned hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

enum { OMEGA_GIVEN = 0, OMEGA_SPLITMIX = 1, OMEGA_PHILOX = 2, OMEGA_FROM_E = 3 };

// sign of entry (i, gc) of the n x d_global projection: true => +1/sqrt(d)
__device__ __forceinline__ bool omega_sign(int kind, uint64_t key, uint64_t seed, int64_t i,
                                           int64_t gc, int64_t d_global) {
    const uint64_t flat = (uint64_t)i * (uint64_t)d_global + (uint64_t)gc;
    if (kind == OMEGA_SPLITMIX) return (mix64(flat ^ key) >> 63) != 0;
    const uint4 r = philox4x32_10(make_uint4((unsigned)flat, (unsigned)(flat >> 32), 0u, 0u),
                                  make_uint2((unsigned)seed, (unsigned)(seed >> 32)));
    return (r.x >> 31) != 0;
}

// Value-free detection: *ok stays 1 only if every stored value equals
// vf_value(len(row), len(col)) bit for bit (one warp per row, lanes over its
// entries); a zero-length column (1/sqrt(0) = inf) never matches a finite value.
template <typename T>
__global__ void k_vf_check(const int64_t *__restrict__ rowptr, const int *__restrict__ cols,
                           const T *__restrict__ vals, int64_t n_rows, int *ok) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = w0; r < n_rows; r += nw) {
        if (*(volatile int *)ok == 0) return;
        const int64_t b = rowptr[r], e = rowptr[r + 1];
        bool good = true;
        for (int64_t q = b + lane; q < e; q += 32) good &= memcmp_eq(vf_value<T>((double)(e - b), rowptr, cols[q]), vals[q]);
        if (!__all_sync(0xFFFFFFFFu, good)) {
            if (lane == 0) *ok = 0;
            return;
        }
    }
}

// Q(0) = block, E = theta0 * block; pad columns [d, ld) are zero.
template <typename T>
__global__ void k_stage_init(const double *__restrict__ given, T *y0, T *E, int64_t n, int d,
                             int ld, int kind, uint64_t seed, int64_t col0, int64_t d_global,
                             double theta0, double scale, int64_t row0 = 0) {
    const uint64_t key = mix64(seed);
    const int64_t total = n * (int64_t)ld;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / ld;
        const int c = (int)(t - i * ld);
        T v = (T)0, e = (T)0;
        if (c < d) {
            if (kind == OMEGA_FROM_E) {
                v = E[t];
            } else if (kind == OMEGA_GIVEN) {
                v = (T)given[i * d + c];
            } else {
                v = (T)(omega_sign(kind, key, seed, row0 + i, col0 + c, d_global) ? scale : -scale);
            }
            if (sizeof(T) == 8)
                e = (T)__dmul_rn((double)theta0, (double)v);
            else
                e = (T)theta0 * v;
        }
        y0[t] = v;
        E[t] = e;
    }
}

// the full n x ld projection block (gather source of a row-partitioned run's first step)
template <typename T>
__global__ void k_omega_fill(T *F, int64_t n, int d, int ld, int kind, uint64_t seed, int64_t col0,
                             int64_t d_global, double scale) {
    const uint64_t key = mix64(seed);
    const int64_t total = n * (int64_t)ld;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / ld;
        const int c = (int)(t - i * ld);
        F[t] = c < d ? (T)(omega_sign(kind, key, seed, i, col0 + c, d_global) ? scale : -scale) : (T)0;
    }
}

// dense n x w projection (f64 out) for sample_projection
__global__ void k_omega_dense(double *out, int64_t n, int64_t w, int kind, uint64_t seed,
                              int64_t col0, int64_t d_global, double scale) {
    const uint64_t key = mix64(seed);
    const int64_t total = n * w;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / w;
        const int64_t c = t - i * w;
        out[t] = omega_sign(kind, key, seed, i, col0 + c, d_global) ? scale : -scale;
    }
}

// ---------------------------------------------------------------------------
// K4: row normalisation, one warp per row
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_rownorm(T *E, int64_t n, int d, int ld) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < n; i += nw) {
        T *r = E + i * ld;
        double s = 0.0;
        for (int c = lane; c < d; c += 32) {
            const double v = (double)r[c];
            s += v * v;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
        const double nrm = sqrt(s);
        for (int c = lane; c < d; c += 32) r[c] = nrm > 0.0 ? (T)((double)r[c] / nrm) : (T)0;
    }
}

// ---------------------------------------------------------------------------
// K3: column statistics for the power iteration
// ---------------------------------------------------------------------------
// partial[(by*2+0)*k + c] = sum_rows V[r,c]*W[r,c]; partial[(by*2+1)*k + c] = sum W[r,c]^2
// (W == null: sum V^2 only, into slot 1).  blockDim = (32, 8).
template <typename T>
__global__ void k_colstats(const T *__restrict__ V, const T *__restrict__ Wm, int64_t n, int k,
                           int ld, double *partial) {
    __shared__ double s_dot[8][33], s_sq[8][33];
    const int c = blockIdx.x * 32 + threadIdx.x;
    double dot = 0.0, sq = 0.0;
    if (c < k) {
        for (int64_t r = (int64_t)blockIdx.y * 8 + threadIdx.y; r < n; r += (int64_t)gridDim.y * 8) {
            const double v = (double)V[r * ld + c];
            if (Wm) {
                const double w = (double)Wm[r * ld + c];
                dot += v * w;
                sq += w * w;
            } else {
                sq += v * v;
            }
        }
    }
    s_dot[threadIdx.y][threadIdx.x] = dot;
    s_sq[threadIdx.y][threadIdx.x] = sq;
    __syncthreads();
    if (threadIdx.y == 0 && c < k) {
        double a = 0.0, b = 0.0;
        for (int y = 0; y < 8; ++y) {
            a += s_dot[y][threadIdx.x];
            b += s_sq[y][threadIdx.x];
        }
        partial[((int64_t)blockIdx.y * 2 + 0) * k + c] = a;
        partial[((int64_t)blockIdx.y * 2 + 1) * k + c] = b;
    }
}

// fixed-order sum of the partials, one warp per column (lane-strided partial
// sums, then a shuffle tree): rq[c] = dot, inv[c] = 1/sqrt(sq) (0 if sq == 0)
__global__ void k_colfinish(const double *partial, int nparts, int k, double *rq, double *inv) {
    const int c = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (c >= k) return;  // whole warps exit together
    double a = 0.0, b = 0.0;
    for (int p = lane; p < nparts; p += 32) {
        a += partial[((int64_t)p * 2 + 0) * k + c];
        b += partial[((int64_t)p * 2 + 1) * k + c];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xFFFFFFFFu, a, o);
        b += __shfl_xor_sync(0xFFFFFFFFu, b, o);
    }
    if (lane == 0) {
        if (rq) rq[c] = a;
        const double nrm = sqrt(b);
        inv[c] = nrm > 0.0 ? 1.0 / nrm : 0.0;
    }
}

// dst[r,c] = src[r,c] * inv[c]  (dead columns become 0, like dropping them)
template <typename T>
__global__ void k_colscale(T *dst, const T *src, const double *inv, int64_t n, int k, int ld) {
    const int64_t total = n * (int64_t)ld;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(t % ld);
        dst[t] = c < k ? (T)((double)src[t] * inv[c]) : (T)0;
    }
}

// standard normals from Philox (Box-Muller) for the power-iteration start block
template <typename T>
__global__ void k_normal_init(T *V, int64_t n, int k, int ld, uint64_t seed) {
    const int64_t total = n * (int64_t)ld;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / ld;
        const int c = (int)(t - i * ld);
        T v = (T)0;
        if (c < k) {
            const uint64_t flat = (uint64_t)i * (uint64_t)k + (uint64_t)c;
            const uint4 r = philox4x32_10(make_uint4((unsigned)flat, (unsigned)(flat >> 32), 0x6E6F726Du, 0u),
                                          make_uint2((unsigned)seed, (unsigned)(seed >> 32)));
            const double u1 = ((double)r.x + 1.0) * 2.3283064365386963e-10;  // (0, 1]
            const double u2 = (double)r.y * 2.3283064365386963e-10;
            v = (T)(sqrt(-2.0 * log(u1)) * cospi(2.0 * u2));
        }
        V[t] = v;
    }
}

// f64 -> T with row padding (n x d dense -> n x ld)
template <typename T>
__global__ void k_pack(const double *__restrict__ src, T *dst, int64_t n, int d, int ld) {
    const int64_t total = n * (int64_t)ld;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / ld;
        const int c = (int)(t - i * ld);
        dst[t] = c < d ? (T)src[i * d + c] : (T)0;
    }
}

// n x ld (T) -> n x d (f64 or f32) without padding
template <typename T, typename O>
__global__ void k_unpack(const T *__restrict__ src, O *dst, int64_t n, int d, int ld) {
    const int64_t total = n * (int64_t)d;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / d;
        const int c = (int)(t - i * d);
        dst[t] = (O)src[i * ld + c];
    }
}

// out[i] = cols[idx[i]] (first column of each heavy-row chunk, for scheduling)
__global__ void k_gather_cols(const int *__restrict__ cols, const int64_t *__restrict__ idx, int *out, int64_t n) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        out[t] = cols[idx[t]];
}

// Column-window boundaries of the heavy rows: bounds[h * (nwin + 1) + k] = the
// first entry of heavy row rows[h] whose column is >= k * wcols (lower bound in
// the row's sorted column ids), so a heavy row can be cut at window edges.
__global__ void k_window_bounds(const int *__restrict__ cols, const int64_t *__restrict__ rowptr,
                                const int *__restrict__ rows, int n_heavy, int nwin, int64_t wcols,
                                int64_t *bounds) {
    const int64_t total = (int64_t)n_heavy * (nwin + 1);
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int h = (int)(t / (nwin + 1));
        const int k = (int)(t - (int64_t)h * (nwin + 1));
        int64_t lo = rowptr[rows[h]], hi = rowptr[rows[h] + 1];
        const int64_t key = (int64_t)k * wcols;
        while (lo < hi) {  // first entry with col >= key
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)cols[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        bounds[t] = lo;
    }
}

// CSR conversion: int64 -> int32 column indices (with range check), f64 -> T values
__global__ void k_cols_to_i32(const int64_t *__restrict__ src, int *dst, int64_t cnt,
                              int64_t n_cols, int *bad) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < cnt;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = src[t];
        if (v < 0 || v >= n_cols) atomicExch(bad, 1);
        dst[t] = (int)v;
    }
}
__global__ void k_cols_check_i32(const int *__restrict__ src, int *dst, int64_t cnt,
                                 int64_t n_cols, int *bad) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < cnt;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int v = src[t];
        if (v < 0 || (int64_t)v >= n_cols) atomicExch(bad, 1);
        dst[t] = v;
    }
}
template <typename T>
__global__ void k_vals_convert(const double *__restrict__ src, T *dst, int64_t cnt) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < cnt;
         t += (int64_t)gridDim.x * blockDim.x)
        dst[t] = (T)src[t];
}
template <typename T>
__global__ void k_vals_scale(T *v, int64_t cnt, double factor) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < cnt;
         t += (int64_t)gridDim.x * blockDim.x) {
        if (sizeof(T) == 8)
            v[t] = (T)__dmul_rn((double)v[t], factor);
        else
            v[t] = (T)((double)v[t] * factor);
    }
}
template <typename T>
__global__ void k_vals_to_f64(const T *__restrict__ v, double *out, int64_t cnt) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < cnt;
         t += (int64_t)gridDim.x * blockDim.x)
        out[t] = (double)v[t];
}

}  // namespace csemb
