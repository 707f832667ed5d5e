// common.cuh — error handling, launch helpers and deterministic reductions.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace mpm2p {

// errors.hpp:9-24 — mapped to C-ABI status codes at the boundary.
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct NumericError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CapacityError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess)
        throw CudaError(std::string(what) + ": " + cudaGetErrorString(e) + " at " + file + ":" + std::to_string(line));
}
#define CK(x) ::mpm2p::cuda_check((x), #x, __FILE__, __LINE__)
#define CK_LAUNCH() ::mpm2p::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

// Device error word bits (checked once per step on the host).
enum : unsigned {
    ERR_CFL = 1u << 0,          // upwind_step: saturation left [0,1] (transport.cpp:115-116)
    ERR_KAPPA = 1u << 1,        // conductivity not positive/finite (elliptic.cpp:73-75)
    ERR_PIVOT = 1u << 2,        // local LDL^T breakdown (elliptic.cpp:185-188)
    ERR_SINGULAR = 1u << 3,     // interface matrix numerically singular (mrcm.cpp:227-238)
    ERR_EPS_ZERO = 1u << 4,     // epsilon: zero reference norm (mpm.cpp:23)
    ERR_ROBIN_BETA = 1u << 5,   // Robin face requires beta > 0 (elliptic.cpp:134-135)
    ERR_REPAIR_SINGULAR = 1u << 6,
    ERR_FINE_NOCONV = 1u << 7,  // fine-reference PCG did not reach its tolerance (fine.cu)
    ERR_TRACK_ZERO = 1u << 8,   // relative_flux/sat_error: zero reference norm (simulation.cpp:37-41,53-57)
    ERR_STRUCT = 1u << 9        // solve with a boundary structure other than the factorization's (elliptic.cpp:155-160)
};

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

// ---- double-double helpers for order-robust sums (H4) --------------------
struct DD {
    double hi, lo;
};
__device__ __forceinline__ DD dd_add(DD a, DD b) {
    const double s = __dadd_rn(a.hi, b.hi);
    const double bb = __dsub_rn(s, a.hi);
    const double err = __dadd_rn(__dsub_rn(a.hi, __dsub_rn(s, bb)), __dsub_rn(b.hi, bb));
    const double lo = __dadd_rn(err, __dadd_rn(a.lo, b.lo));
    const double hi = __dadd_rn(s, lo);
    return DD{hi, __dsub_rn(lo, __dsub_rn(hi, s))};
}
__device__ __forceinline__ DD dd_shfl_down(DD v, int off) {
    return DD{__shfl_down_sync(0xffffffffu, v.hi, off), __shfl_down_sync(0xffffffffu, v.lo, off)};
}
__device__ __forceinline__ DD warp_sum_dd(DD v) {
    for (int o = 16; o > 0; o >>= 1) v = dd_add(v, dd_shfl_down(v, o));
    return v;
}
__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_min(double v) {
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_down_sync(0xffffffffu, v, o));
    return v;
}

// ---- Programmatic dependent launch (griddepcontrol, sm_90+) ----------------
// Every kernel starts with pdl_begin(): it waits until the previous kernel in
// the stream has completed and its writes are visible (a no-op when the
// launch carried no programmatic dependency), then lets the next kernel be
// scheduled. Kernels are launched with programmatic stream serialisation
// (launch_k), so the next kernel's launch and block scheduling overlap this
// kernel's execution instead of following its completion.
__device__ __forceinline__ void pdl_begin() {
#ifdef MPM2P_PDL_EARLY_TRIGGER
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#else
    asm volatile("griddepcontrol.wait;" ::: "memory");  // dependents are released as this grid's blocks exit
#endif
}

// ---- TMA bulk copies (cp.async.bulk, SASS UBLKCP) completing on an mbarrier
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // init visible to the async (TMA) proxy
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// global -> shared, `bytes` a multiple of 16, both addresses 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(sdst)),
                 "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra "
        "WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Predicated global store without a divergent branch (the compiler otherwise
// wraps lane-conditional stores in BSSY/WARPSYNC regions, which stall the
// latency-bound pivot loop). No memory clobber: callers order it with later
// reads through __syncwarp.
__device__ __forceinline__ void st_global_if(double* p, double v, bool pred) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.f64 [%0], %1;\n\t}" ::"l"(p), "d"(v),
        "r"((int)pred));
}

// 1/d without the IEEE-division slow path: MUFU reciprocal approximation and
// two Newton steps (relative error ~1 ulp; d is a positive pivot).
__device__ __forceinline__ double fast_rcp(double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0);
    r = fma(r, e, r);
    e = fma(-d, r, 1.0);
    return fma(r, e, r);
}

// Block-wide reduction (result valid in thread 0). sh: >= 32 doubles of smem.
template <typename F>
__device__ __forceinline__ double block_reduce_op(double v, F op, double ident, double* sh) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_down_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    if (w == 0) {
        v = lane < (int)(blockDim.x >> 5) ? sh[lane] : ident;
        for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_down_sync(0xffffffffu, v, o));
    }
    __syncthreads();
    return v;
}

// The last block of a grid combines the per-block partials part[b*stride+off]
// (b < nparts) in parallel, in a fixed tree order (deterministic).
template <typename F>
__device__ __forceinline__ double reduce_partials(const double* part, int nparts, int stride, int off, F op,
                                                  double ident, double* sh) {
    double v = ident;
    for (int b = threadIdx.x; b < nparts; b += blockDim.x) v = op(v, __ldcg(part + (size_t)b * stride + off));
    return block_reduce_op(v, op, ident, sh);
}

// N values reduced at once (bit `i` of sum_mask: slot i is a sum, else a
// max), one barrier: warp shuffles per slot, then thread i < N combines the
// warps of slot i. Results land in out[0..N-1] (shared), valid after the
// trailing barrier. sh must hold 32 * N doubles.
template <int N>
__device__ __forceinline__ void block_reduce_multi(double (&v)[N], unsigned sum_mask, double* sh, double* out) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const bool sm = (sum_mask >> i) & 1u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double t = __shfl_down_sync(0xffffffffu, v[i], o);
            v[i] = sm ? v[i] + t : fmax(v[i], t);
        }
    }
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < N; ++i) sh[w * N + i] = v[i];
    }
    __syncthreads();
    if (threadIdx.x < N) {
        const int i = threadIdx.x;
        const bool sm = (sum_mask >> i) & 1u;
        double a = sh[i];
        for (int ww = 1; ww < nw; ++ww) a = sm ? a + sh[ww * N + i] : fmax(a, sh[ww * N + i]);
        out[i] = a;
    }
    __syncthreads();
}

}  // namespace mpm2p
