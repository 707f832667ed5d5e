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
//  * no pointer here is __restrict__: every buffer is written by one lane and
//    read by others (a restrict pointer licenses the compiler to hoist a
//    lane's load above another lane's store across __syncwarp);
//  * the pivot column is broadcast through a per-warp shared-memory exchange
//    buffer (one STS per lane, then LDS.128 broadcasts), not warp shuffles:
//    a 64-bit shuffle issues once per ~10 cycles per warp on B200
//    (tools/lat_probe.cu), so B of them per pivot made the step MIO-bound.
// Per pivot the critical path is one smem round trip (~43 cycles), one
// reciprocal and two FMAs.
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

// Per-warp exchange buffer (doubles, 16-byte aligned): two parity slots of
// the pivot column (B), of the pivot (2, padded) and of the pivot's RHS values.
template <int NR>
__host__ __device__ constexpr int xchg_ys() {
    return (NR + 1) & ~1;
}
template <int B, int NR>
__host__ __device__ constexpr int xchg_doubles() {
    return 2 * B + 4 + 2 * xchg_ys<NR>();
}

template <int B>
__device__ __forceinline__ int band_j_of(int lane, int u) {  // window position of lane's row at pivot k0+u
    return (lane - u - 1 + 2 * B) % B;
}

// Factorization with the forward sweep of NR right-hand sides fused in.
// stage: B*B doubles of shared memory (per warp) used to transpose L rows.
template <int B, int NR>
__device__ bool factor_fwd_reg(int n, const BandRows A, double* D, double* Lcol,
                               double* Lrow, double* Y, int nr, int ldy,
                               double* stage, double* xb) {
    static_assert(B % 2 == 0 || B == 1, "pairs of the pivot column are read as double2");
    constexpr int YS = xchg_ys<NR>();
    const int lane = threadIdx.x & 31;
    const bool act = lane < B;
    const int lane_c = act ? lane : 0;  // in-bounds smem index for idle lanes
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
    // entering-row data for the first chunk: row B + lane. Loads use clamped
    // (always valid) indices and no select: a value is only consumed under
    // `ent` (the row exists), so the prefetch never stalls the issuing step.
    // Slots m >= nr carry a copy of RHS nr-1 (finite, never stored).
    auto fetch = [&](int row, double& fd, double& fw, double& fs, double* fb) {
        const int rr = row < n ? row : n - 1;
        fd = A.diag[rr];
        fw = A.offw[rr];
        fs = A.offs[rr];
#pragma unroll
        for (int m = 0; m < NR; ++m) fb[m] = Y[(size_t)(m < nr ? m : nr - 1) * ldy + rr];
    };
    double cd, cw, cs, cb[NR];
    fetch(B + lane, cd, cw, cs, cb);
    bool ok = true;
    const bool has_lcol = Lcol != nullptr;
    double st_l = 0.0;  // deferred stage write (position st_pos of this lane's row)
    int st_pos = 0;
    __syncwarp();
    for (int k0 = 0; k0 < n; k0 += B) {
        double nd, nw, ns, nbv[NR];
        fetch(k0 + 2 * B + lane, nd, nw, ns, nbv);
        const bool ent_chunk = k0 + 2 * B <= n;  // every row k+B of this chunk exists
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int k = k0 + u;
            const bool piv = lane == u;
            // pivot lane: row k leaves, row k+B enters (its coupling to column k is c)
            const bool ent = ent_chunk;
            const double c = piv ? (ent ? -cs : 0.0) : reg[u];
            double* cbuf = xb + (u & 1) * B;            // column k of the window
            double* dbuf = xb + 2 * B + (u & 1) * 2;    // pivot d_k
            double* ybuf = xb + 2 * B + 4 + (u & 1) * YS;  // y_k of the NR right-hand sides
            // previous step's L entry into the transposition tile (ordered after
            // every read of step k-1 by the end-of-step barrier)
            if (act) stage[lane * B + st_pos] = st_l;
            if (act) cbuf[lane] = c;
            if (piv) {
                dbuf[0] = reg[u];
#pragma unroll
                for (int m = 0; m < NR; ++m) ybuf[m] = yv[m];
            }
            __syncwarp();
            const double d = dbuf[0];
            double yk[NR];
#pragma unroll
            for (int m = 0; m < NR; ++m) yk[m] = ybuf[m];
            st_global_if(D + k, d, piv);
#pragma unroll
            for (int m = 0; m < NR; ++m) st_global_if(Y + (size_t)m * ldy + k, yk[m], piv && m < nr);
            st_global_if(Lrow + (size_t)k * B + lane, stage[u * B + lane_c], act);
            ok = ok && (d > 0.0);
            const double keep = piv ? 0.0 : 1.0;
            const double fd_ = (piv && ent) ? cd : 0.0, fw_ = (piv && ent) ? -cw : 0.0;
            const double l = c * fast_rcp(d);
            const int j = band_j_of<B>(lane, u);
            if (has_lcol) st_global_if(Lcol + (size_t)k * B + j, l, act);
            st_l = l;
            st_pos = B - 1 - j;
            const double2* cb2 = reinterpret_cast<const double2*>(cbuf);
#pragma unroll
            for (int q = 0; q < B / 2; ++q) {
                const double2 a2 = cb2[q];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int ci = 2 * q + h;
                    if (ci == u) continue;  // column k itself: reset below
                    const double a = h ? a2.y : a2.x;
                    const double fresh = (ci == (u + B - 1) % B) ? fw_ : 0.0;
                    reg[ci] = fma(-l, a, fma(reg[ci], keep, fresh));
                }
            }
            // register u (column k leaves, column k+B enters): a = c of the pivot lane
            reg[u] = fma(-l, u % 2 ? cb2[u / 2].y : cb2[u / 2].x, fma(reg[u], keep, fd_));
#pragma unroll
            for (int m = 0; m < NR; ++m) yv[m] = fma(-l, yk[m], fma(yv[m], keep, (piv && ent) ? cb[m] : 0.0));
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

// Prefetches in both sweeps load raw values from clamped (always valid)
// addresses and select nothing: a value is consumed only for an existing row
// on an active lane, so the loads never stall the step that issues them
// (a select right after a load would). Idle lanes and missing rows carry
// finite junk that is never stored.

// Deep prefetch of the stored factor for the sweeps: whole B x B chunks of
// Lcol / Lrow (rows k0..k0+B-1, contiguous) are copied by cp.async into a
// per-warp shared-memory ring SWEEP_RING<B> chunks ahead (the register ring
// alone looks only B steps ahead, shorter than an HBM round trip once L2 is
// cold). Widths above 16 keep the register ring (0: no smem ring).
template <int B>
__host__ __device__ constexpr int sweep_ring() {
    return B <= 16 ? 4 : 0;
}

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Copy chunk `c` (clamped to the last chunk; rows past n are never consumed)
// of a B-wide band factor into ring slot `slot`.
template <int B>
__device__ __forceinline__ void sweep_fetch(const double* Lb, int nchunks, int c, double* ring, int slot) {
    const int cc = c < 0 ? 0 : (c < nchunks ? c : nchunks - 1);
    const double* g = Lb + (size_t)cc * B * B;
    double* d = ring + (size_t)slot * B * B;
    for (int p = threadIdx.x & 31; p < B * B / 2; p += 32) cp_async16(d + 2 * p, g + 2 * p);
    cp_async_commit();
}

// Forward sweep L y = b with a stored factor (Lcol), NR RHS in place.
template <int B, int NR>
__device__ void forward_reg(int n, const double* Lcol, double* Y, int nr, int ldy, double* xb,
                            double* ring = nullptr) {
    constexpr int YS = xchg_ys<NR>();
    constexpr int RG = sweep_ring<B>();
    const int lane = threadIdx.x & 31;
    const int nchunks = n / B;
    auto yat = [&](int m, int row) {
        return Y[(size_t)(m < nr ? m : nr - 1) * ldy + (row < n ? row : n - 1)];
    };
    double yv[NR];
#pragma unroll
    for (int m = 0; m < NR; ++m) yv[m] = yat(m, lane);
    // L entries flow through an LQ-deep register ring (step k+LQ is loaded at step k)
    constexpr int LQ = band_lq<B>();
    auto lcol_at = [&](int k, int u) {  // lane's entry of Lcol[k], u = k mod B
        return Lcol[(size_t)(k < n ? k : n - 1) * B + band_j_of<B>(lane, u)];
    };
    double lq[LQ];
    if constexpr (RG > 0) {
#pragma unroll
        for (int c = 0; c < RG; ++c) sweep_fetch<B>(Lcol, nchunks, c, ring, c);
    } else {
#pragma unroll
        for (int t = 0; t < LQ; ++t) lq[t] = lcol_at(t, t % B);
    }
    double cb[NR], nbv[NR];
#pragma unroll
    for (int m = 0; m < NR; ++m) cb[m] = yat(m, B + lane);
    for (int k0 = 0; k0 < n; k0 += B) {
#pragma unroll
        for (int m = 0; m < NR; ++m) nbv[m] = yat(m, k0 + 2 * B + lane);
        if constexpr (RG > 0) {  // chunk k0/B has landed: its B entries of this lane into registers
            const int c = k0 / B, slot = c % RG;
            cp_async_wait<RG - 1>();
            __syncwarp();
            const double* rs = ring + (size_t)slot * B * B;
#pragma unroll
            for (int u = 0; u < B; ++u) lq[u] = rs[u * B + band_j_of<B>(lane, u)];
            __syncwarp();
            sweep_fetch<B>(Lcol, nchunks, c + RG, ring, slot);
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int k = k0 + u;
            const bool piv = lane == u;
            const double keep = piv ? 0.0 : 1.0;
            const double l = lq[u % LQ];
            if constexpr (RG == 0) lq[u % LQ] = lcol_at(k + LQ, (u + LQ) % B);
            double yk[NR];
            if constexpr (NR == 1) {
                yk[0] = __shfl_sync(FULL, yv[0], u);
            } else {  // smem broadcast (NR 64-bit shuffles would be issue-bound)
                double* ybuf = xb + (u & 1) * YS;
                if (piv) {
#pragma unroll
                    for (int m = 0; m < NR; ++m) ybuf[m] = yv[m];
                }
                __syncwarp();
#pragma unroll
                for (int m = 0; m < NR; ++m) yk[m] = ybuf[m];
            }
#pragma unroll
            for (int m = 0; m < NR; ++m) {
                st_global_if(Y + (size_t)m * ldy + k, yk[m], piv && m < nr);
                yv[m] = fma(-l, yk[m], fma(yv[m], keep, piv ? cb[m] : 0.0));
            }
        }
#pragma unroll
        for (int m = 0; m < NR; ++m) cb[m] = nbv[m];
    }
    if constexpr (RG > 0) {  // drain the trailing prefetches: the next sweep refills the same ring slots
        cp_async_wait<0>();
        __syncwarp();
    }
}

// Backward sweep L^T x = D^-1 y with a stored factor (Lrow, D), NR RHS in place.
template <int B, int NR>
__device__ void backward_reg(int n, const double* D, const double* Lrow, double* Y, int nr, int ldy, double* xb,
                             double* ring = nullptr) {
    constexpr int YS = xchg_ys<NR>();
    constexpr int RG = sweep_ring<B>();
    const int lane = threadIdx.x & 31;
    const int nchunks = n / B;
    // raw (d, y) of row `row`; z = y * (1/d) is formed one chunk later, at use
    auto raw = [&](int row, double& d, double* y) {
        const int rr = row < 0 ? 0 : (row < n ? row : n - 1);
        d = D[rr];
#pragma unroll
        for (int m = 0; m < NR; ++m) y[m] = Y[(size_t)(m < nr ? m : nr - 1) * ldy + rr];
    };
    auto scale = [&](double d, const double* y, double* z) {
        const double dinv = 1.0 / d;
#pragma unroll
        for (int m = 0; m < NR; ++m) z[m] = y[m] * dinv;
    };
    double z[NR], ez[NR], rd, ry[NR];
    raw(n - B + lane, rd, ry);  // row n-B+lane == lane (mod B)
    scale(rd, ry, z);
    constexpr int LQ = band_lq<B>();
    auto lrow_at = [&](int k, int u) {  // lane's entry of Lrow[k]: o = (lane - u) mod B, u = k mod B
        return Lrow[(size_t)(k >= 0 ? k : 0) * B + (lane - u + B) % B];
    };
    double lq[LQ];
    const int k0_last = n - B;
    if constexpr (RG > 0) {  // chunks are consumed last to first: ring position i holds chunk nchunks-1-i
#pragma unroll
        for (int i = 0; i < RG; ++i) sweep_fetch<B>(Lrow, nchunks, nchunks - 1 - i, ring, i);
    } else {
        // ring slot of step k is (k mod LQ); prefill steps n-1 .. n-LQ
#pragma unroll
        for (int t = 0; t < LQ; ++t) {
            const int u = B - 1 - t;  // k = k0_last + u
            lq[u % LQ] = lrow_at(k0_last + u, u);
        }
    }
    raw(k0_last - B + lane, rd, ry);
    for (int k0 = k0_last; k0 >= 0; k0 -= B) {
        scale(rd, ry, ez);                 // entering rows of this chunk (loaded one chunk ago)
        raw(k0 - 2 * B + lane, rd, ry);    // ... and of the next
        if constexpr (RG > 0) {
            const int i = nchunks - 1 - k0 / B, slot = i % RG;
            cp_async_wait<RG - 1>();
            __syncwarp();
            const double* rs = ring + (size_t)slot * B * B;
#pragma unroll
            for (int u = 0; u < B; ++u) lq[u] = rs[u * B + (lane - u + B) % B];
            __syncwarp();
            sweep_fetch<B>(Lrow, nchunks, nchunks - 1 - (i + RG), ring, slot);
        }
#pragma unroll
        for (int uu = B - 1; uu >= 0; --uu) {
            const int k = k0 + uu;
            const bool piv = lane == uu;
            const double keep = piv ? 0.0 : 1.0;
            const double l = lq[uu % LQ];
            if constexpr (RG == 0) lq[uu % LQ] = lrow_at(k - LQ, (uu + B - LQ % B) % B);
            double xk[NR];
            if constexpr (NR == 1) {
                xk[0] = __shfl_sync(FULL, z[0], uu);
            } else {
                double* zbuf = xb + (uu & 1) * YS;
                if (piv) {
#pragma unroll
                    for (int m = 0; m < NR; ++m) zbuf[m] = z[m];
                }
                __syncwarp();
#pragma unroll
                for (int m = 0; m < NR; ++m) xk[m] = zbuf[m];
            }
#pragma unroll
            for (int m = 0; m < NR; ++m) {
                st_global_if(Y + (size_t)m * ldy + k, xk[m], piv && m < nr);
                z[m] = fma(-l, xk[m], fma(z[m], keep, piv ? ez[m] : 0.0));
            }
        }
    }
    if constexpr (RG > 0) {  // no copy may still be landing in the ring when the caller reuses it
        cp_async_wait<0>();
        __syncwarp();
    }
}

}  // namespace mpm2p
