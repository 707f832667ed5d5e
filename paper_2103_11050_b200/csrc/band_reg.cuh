// band_reg.cuh — register-resident banded LDL^T, one warp per subdomain,
// bandwidth B known at compile time (B <= 32). Replaces Eigen
// SimplicialLDLT (proj/src/elliptic.cpp:68-199) for the 5-point subdomain
// systems; same mathematics as band.cuh, restructured for latency:
//
//  * lane l owns the window row r == l (mod B); its B lower-band entries
//    (columns r-B+1 .. r) live in registers indexed by column mod B. The
//    row leaving the window at pivot k (row k, lane k mod B) is replaced in
//    the same lane by the row entering it (row k+B), whose coupling to
//    column k is carried separately, so B lanes suffice for half-bandwidth B.
//  * the k-loop is unrolled in chunks of B pivots, so every register index
//    and every shuffle source lane is a compile-time constant;
//  * lane l prefetches the data of the row that will enter its slot one
//    chunk (B pivots) ahead, so the pivot chain never waits on memory;
//  * entries right of the diagonal receive harmless garbage (the entering
//    row resets its registers), so the rank-1 update needs no predicates.
// Per pivot the critical path is one shuffle, one reciprocal and two FMAs.
// Outputs match band.cuh: D[n], Lcol[n][B] (L[k+1+j][k]), Lrow[n][B]
// (L[k][k-B+o]); right-hand sides are transformed in place b -> y -> x.
#pragma once

#include "band.cuh"

namespace mpm2p {

constexpr unsigned FULL = 0xffffffffu;

// Depth of the L prefetch ring in the sweeps: a divisor of B (ring slots stay
// aligned with the chunk-unrolled step index).
template <int B>
__host__ __device__ constexpr int band_lq() {
    return B <= 20 ? B : (B % 16 == 0 ? 16 : (B % 8 == 0 ? 8 : 4));
}

template <int B>
__device__ __forceinline__ int band_j_of(int lane, int u) {  // window position of lane's row at pivot k0+u
    return (lane - u - 1 + 2 * B) % B;
}

// Factorization with the forward sweep of NR right-hand sides fused in.
// stage: B*B doubles of shared memory (per warp) used to transpose L rows.
template <int B, int NR>
__device__ bool factor_fwd_reg(int n, const BandRows A, double* __restrict__ D, double* __restrict__ Lcol,
                               double* __restrict__ Lrow, double* __restrict__ Y, int nr, int ldy,
                               double* __restrict__ stage) {
    const int lane = threadIdx.x & 31;
    const bool act = lane < B;
    double reg[B];
    double yv[NR];
    // rows 0..B-1: lane l holds row l (diag in reg[l], west coupling in reg[l-1])
#pragma unroll
    for (int t = 0; t < B; ++t) {
        double v = 0.0;
        if (act && lane < n) {
            if (t == lane % B) v = A.diag[lane];
            else if (lane >= 1 && t == (lane + B - 1) % B) v = -A.offw[lane];
        }
        reg[t] = v;
    }
#pragma unroll
    for (int m = 0; m < NR; ++m) yv[m] = (act && lane < n && m < nr) ? Y[(size_t)m * ldy + lane] : 0.0;
    for (int x = lane; x < B * B; x += 32) stage[x] = 0.0;
    // entering-row data for the first chunk: row B + lane
    auto fetch = [&](int row, double& fd, double& fw, double& fs, double* fb) {
        const bool ok = act && row < n;
        fd = ok ? A.diag[row] : 0.0;
        fw = ok ? A.offw[row] : 0.0;
        fs = ok ? A.offs[row] : 0.0;
#pragma unroll
        for (int m = 0; m < NR; ++m) fb[m] = (ok && m < nr) ? Y[(size_t)m * ldy + row] : 0.0;
    };
    double cd, cw, cs, cb[NR];
    fetch(B + lane, cd, cw, cs, cb);
    bool ok = true;
    __syncwarp();
    for (int k0 = 0; k0 < n; k0 += B) {
        double nd, nw, ns, nbv[NR];
        fetch(k0 + 2 * B + lane, nd, nw, ns, nbv);
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int k = k0 + u;
            const bool piv = lane == u;
            const double d = __shfl_sync(FULL, reg[u], u);
            double yk[NR];
#pragma unroll
            for (int m = 0; m < NR; ++m) yk[m] = __shfl_sync(FULL, yv[m], u);
            if (piv) {
                D[k] = d;
#pragma unroll
                for (int m = 0; m < NR; ++m)
                    if (m < nr) Y[(size_t)m * ldy + k] = yk[m];
            }
            if (act) Lrow[(size_t)k * B + lane] = stage[u * B + lane];
            __syncwarp();
            if (!(d > 0.0)) ok = false;
            const bool ent = k + B < n;
            const double c = piv ? (ent ? -cs : 0.0) : reg[u];
            if (piv) {
#pragma unroll
                for (int t = 0; t < B; ++t) reg[t] = 0.0;
                if (ent) {
                    reg[(u + B - 1) % B] = -cw;
                    reg[u] = cd;
                }
#pragma unroll
                for (int m = 0; m < NR; ++m) yv[m] = ent ? cb[m] : 0.0;
            }
            const double l = c * (1.0 / d);
            const int j = band_j_of<B>(lane, u);
            if (act) {
                if (Lcol) Lcol[(size_t)k * B + j] = l;
                stage[lane * B + (B - 1 - j)] = l;
            }
#pragma unroll
            for (int i = 0; i < B; ++i) {
                const int ci = (u + 1 + i) % B;
                const double a = __shfl_sync(FULL, c, ci);
                reg[ci] -= l * a;
            }
#pragma unroll
            for (int m = 0; m < NR; ++m) yv[m] -= l * yk[m];
            __syncwarp();
        }
        cd = nd;
        cw = nw;
        cs = ns;
#pragma unroll
        for (int m = 0; m < NR; ++m) cb[m] = nbv[m];
    }
    return __all_sync(FULL, ok);
}

// Forward sweep L y = b with a stored factor (Lcol), NR RHS in place.
template <int B, int NR>
__device__ void forward_reg(int n, const double* __restrict__ Lcol, double* __restrict__ Y, int nr, int ldy) {
    const int lane = threadIdx.x & 31;
    const bool act = lane < B;
    double yv[NR];
#pragma unroll
    for (int m = 0; m < NR; ++m) yv[m] = (act && lane < n && m < nr) ? Y[(size_t)m * ldy + lane] : 0.0;
    // L entries flow through an LQ-deep register ring (step k+LQ is loaded at step k)
    constexpr int LQ = band_lq<B>();
    auto lcol_at = [&](int k, int u) {  // lane's entry of Lcol[k], u = k mod B
        return (act && k < n) ? Lcol[(size_t)k * B + band_j_of<B>(lane, u)] : 0.0;
    };
    double lq[LQ];
#pragma unroll
    for (int t = 0; t < LQ; ++t) lq[t] = lcol_at(t, t % B);
    double cb[NR], nbv[NR];
#pragma unroll
    for (int m = 0; m < NR; ++m) cb[m] = (act && B + lane < n && m < nr) ? Y[(size_t)m * ldy + B + lane] : 0.0;
    for (int k0 = 0; k0 < n; k0 += B) {
        const int er = k0 + 2 * B + lane;
#pragma unroll
        for (int m = 0; m < NR; ++m) nbv[m] = (act && er < n && m < nr) ? Y[(size_t)m * ldy + er] : 0.0;
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int k = k0 + u;
            const bool piv = lane == u;
            const double l = lq[u % LQ];
            lq[u % LQ] = lcol_at(k + LQ, (u + LQ) % B);
            double yk[NR];
#pragma unroll
            for (int m = 0; m < NR; ++m) yk[m] = __shfl_sync(FULL, yv[m], u);
            if (piv) {
#pragma unroll
                for (int m = 0; m < NR; ++m) {
                    if (m < nr) Y[(size_t)m * ldy + k] = yk[m];
                    yv[m] = cb[m];
                }
            }
#pragma unroll
            for (int m = 0; m < NR; ++m) yv[m] -= l * yk[m];
        }
#pragma unroll
        for (int m = 0; m < NR; ++m) cb[m] = nbv[m];
    }
}

// Backward sweep L^T x = D^-1 y with a stored factor (Lrow, D), NR RHS in place.
template <int B, int NR>
__device__ void backward_reg(int n, const double* __restrict__ D, const double* __restrict__ Lrow,
                             double* __restrict__ Y, int nr, int ldy) {
    const int lane = threadIdx.x & 31;
    const bool act = lane < B;
    double z[NR];
    {
        const int c = n - B + lane;  // c == lane (mod B)
        const double dc = (act && c >= 0) ? D[c] : 1.0;
#pragma unroll
        for (int m = 0; m < NR; ++m) z[m] = (act && c >= 0 && m < nr) ? Y[(size_t)m * ldy + c] / dc : 0.0;
    }
    constexpr int LQ = band_lq<B>();
    auto lrow_at = [&](int k, int u) {  // lane's entry of Lrow[k]: o = (lane - u) mod B, u = k mod B
        return (act && k >= 0) ? Lrow[(size_t)k * B + (lane - u + B) % B] : 0.0;
    };
    double lq[LQ], eb[NR], nbv[NR], ed, nd;
    const int k0_last = n - B;
    // ring slot of step k is (k mod LQ); prefill steps n-1 .. n-LQ
#pragma unroll
    for (int t = 0; t < LQ; ++t) {
        const int u = B - 1 - t;  // k = k0_last + u
        lq[u % LQ] = lrow_at(k0_last + u, u);
    }
    {
        const int er = k0_last - B + lane;
        const bool okr = act && er >= 0;
        ed = okr ? D[er] : 1.0;
#pragma unroll
        for (int m = 0; m < NR; ++m) eb[m] = (okr && m < nr) ? Y[(size_t)m * ldy + er] : 0.0;
    }
    for (int k0 = k0_last; k0 >= 0; k0 -= B) {
        {
            const int er = k0 - 2 * B + lane;
            const bool okr = act && er >= 0;
            nd = okr ? D[er] : 1.0;
#pragma unroll
            for (int m = 0; m < NR; ++m) nbv[m] = (okr && m < nr) ? Y[(size_t)m * ldy + er] : 0.0;
        }
#pragma unroll
        for (int uu = B - 1; uu >= 0; --uu) {
            const int k = k0 + uu;
            const bool piv = lane == uu;
            const double l = lq[uu % LQ];
            lq[uu % LQ] = lrow_at(k - LQ, (uu + B - LQ % B) % B);
            double xk[NR];
#pragma unroll
            for (int m = 0; m < NR; ++m) xk[m] = __shfl_sync(FULL, z[m], uu);
            if (piv) {
#pragma unroll
                for (int m = 0; m < NR; ++m) {
                    if (m < nr) Y[(size_t)m * ldy + k] = xk[m];
                    z[m] = (k - B >= 0) ? eb[m] / ed : 0.0;
                }
            }
#pragma unroll
            for (int m = 0; m < NR; ++m) z[m] -= l * xk[m];
        }
        ed = nd;
#pragma unroll
        for (int m = 0; m < NR; ++m) eb[m] = nbv[m];
    }
}

}  // namespace mpm2p
