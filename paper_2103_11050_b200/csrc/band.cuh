// band.cuh — one-warp-per-subdomain banded LDL^T for the 5-point TPFA
// subdomain systems (replaces Eigen SimplicialLDLT in
// proj/src/elliptic.cpp:68-150 (factorize) and :152-199 (solve)).
//
// A subdomain of snx x sny cells, eliminated in natural row-major order, is
// an SPD band matrix of half-bandwidth B = snx with three nonzero diagonals
// per row: diag[r], the "west" coupling -offw[r] to r-1 and the "south"
// coupling -offs[r] to r-B. One warp owns one subdomain; lane j owns window
// row k+1+j while pivot k is eliminated. The active window (B+1 rows x B+1
// lower-band entries) and the right-hand-side rings live in shared memory as
// circular buffers indexed by row mod (B+1), so no data moves between steps.
// Rows entering the window are prefetched PD steps ahead into registers so
// the sequential pivot chain never waits on global memory.
//
// Outputs of a factorization: D[n], Lcol[n][B] (column k of L below the
// diagonal: L[k+1+j][k]) for forward sweeps and Lrow[n][B] (row k of L:
// L[k][k-B+o]) for backward sweeps; both are written coalesced (one 8*B-byte
// row per step). Right-hand sides are transformed in place: b -> y (forward,
// L y = b) -> x (backward, L^T x = D^-1 y).
#pragma once

#include "common.cuh"

namespace mpm2p {

constexpr int BAND_MAX = 32;  // lanes map 1:1 to window rows
constexpr int RING_NR = 29;   // RHS carried through one ring (lanes 3..31 prefetch them)
constexpr int PD = 4;         // prefetch distance (steps)

// Shared-memory doubles one warp needs for bandwidth B and nr ring RHS.
__host__ __device__ inline int band_smem_doubles(int B, int nr) {
    const int S = B + 1, P = B + 2;
    return S * P + S + S * (nr > 0 ? nr : 1);
}

struct BandRows {
    const double* diag;
    const double* offw;
    const double* offs;
};

__device__ __forceinline__ double band_entry(int r, int n, int B, const BandRows& A, const double* Y, int nr,
                                             int ldy, int lane) {
    if (r >= n) return 0.0;
    if (lane == 0) return A.diag[r];
    if (lane == 1) return A.offw[r];
    if (lane == 2) return r >= B ? A.offs[r] : 0.0;
    const int m = lane - 3;
    return m < nr ? Y[(size_t)m * ldy + r] : 0.0;
}

// Writes row r (entries held as lane-distributed `e`) into ring slot `slot`.
__device__ __forceinline__ void band_store_row(double e, int B, int P, int slot, double* sW, double* sy, int nr,
                                               int lane) {
    const double dg = __shfl_sync(0xffffffffu, e, 0);
    const double ow = __shfl_sync(0xffffffffu, e, 1);
    const double os = __shfl_sync(0xffffffffu, e, 2);
    const double ym = __shfl_sync(0xffffffffu, e, (lane + 3) & 31);
    double* w = sW + slot * P;
    for (int o = lane; o <= B; o += 32) {
        double v = 0.0;
        if (o == B) v = dg;
        if (o == B - 1) v -= ow;
        if (o == 0) v -= os;
        w[o] = v;
    }
    if (lane < nr) sy[slot * nr + lane] = ym;
}

// Factorization with the forward sweep of nr (<= RING_NR) right-hand sides
// fused in. Y: nr vectors of length n at stride ldy (in: b, out: y).
// Lcol may be null. Returns false (on all lanes) if a pivot was not positive.
static __device__ bool band_factor_fwd(int n, int B, const BandRows A, double* __restrict__ D, double* __restrict__ Lcol,
                                double* __restrict__ Lrow, double* __restrict__ Y, int nr, int ldy, double* smem) {
    const int lane = threadIdx.x & 31;
    const int S = B + 1, P = B + 2;
    double* sW = smem;
    double* sdinv = sW + S * P;
    double* sy = sdinv + S;
    bool ok = true;
    for (int r = 0; r < S && r < n; ++r)
        band_store_row(band_entry(r, n, B, A, Y, nr, ldy, lane), B, P, r, sW, sy, nr, lane);
    double q[PD];
#pragma unroll
    for (int t = 0; t < PD; ++t) q[t] = band_entry(S + t, n, B, A, Y, nr, ldy, lane);
    __syncwarp();
    int slot = 0;
    for (int k = 0; k < n; ++k) {
        const double d = sW[slot * P + B];
        if (!(d > 0.0)) ok = false;
        const double dinv = 1.0 / d;
        if (lane < B) {
            const int c = k - B + lane;
            Lrow[(size_t)k * B + lane] = c >= 0 ? sW[slot * P + lane] * sdinv[(slot + S - B + lane) % S] : 0.0;
        }
        if (lane == 0) D[k] = d;
        if (lane < nr) Y[(size_t)lane * ldy + k] = sy[slot * nr + lane];  // y_k is final
        const int r = k + 1 + lane;
        const bool valid = lane < B && r < n;
        const int rs = (slot + 1 + lane) % S;
        const double cj = valid ? sW[rs * P + B - 1 - lane] : 0.0;
        const double lj = cj * dinv;
        if (Lcol && lane < B) Lcol[(size_t)k * B + lane] = valid ? lj : 0.0;
        // next entering row (k+1+B) is q[0]; refill the queue
        const double e = q[0];
#pragma unroll
        for (int t = 0; t + 1 < PD; ++t) q[t] = q[t + 1];
        q[PD - 1] = band_entry(k + 1 + B + PD, n, B, A, Y, nr, ldy, lane);
        __syncwarp();
        if (lane == 0) sdinv[slot] = dinv;
        double* wr = sW + rs * P + B - lane;
        for (int i = 0; i < B; ++i) {
            const double ai = __shfl_sync(0xffffffffu, cj, i);
            if (valid && i <= lane) wr[i] -= lj * ai;
        }
        if (valid)
            for (int m = 0; m < nr; ++m) sy[rs * nr + m] -= lj * sy[slot * nr + m];
        __syncwarp();
        if (k + 1 + B < n) band_store_row(e, B, P, slot, sW, sy, nr, lane);
        __syncwarp();
        slot = slot + 1 == S ? 0 : slot + 1;
    }
    return __all_sync(0xffffffffu, ok);
}

// Forward sweep L y = b with a stored factor (Lcol), nr (<= 32) RHS in place.
static __device__ void band_forward(int n, int B, const double* __restrict__ Lcol, double* __restrict__ Y, int nr, int ldy,
                             double* smem) {
    const int lane = threadIdx.x & 31;
    const int S = B + 1;
    double* sy = smem;
    for (int i = lane; i < S * nr; i += 32) {
        const int r = i / nr, m = i % nr;
        if (r < n) sy[(r % S) * nr + m] = Y[(size_t)m * ldy + r];
    }
    double ql[PD], qy[PD];
#pragma unroll
    for (int t = 0; t < PD; ++t) {
        ql[t] = (t < n && lane < B) ? Lcol[(size_t)t * B + lane] : 0.0;
        qy[t] = (S + t < n && lane < nr) ? Y[(size_t)lane * ldy + S + t] : 0.0;
    }
    __syncwarp();
    int slot = 0;
    for (int k = 0; k < n; ++k) {
        const double l = ql[0], ye = qy[0];
#pragma unroll
        for (int t = 0; t + 1 < PD; ++t) { ql[t] = ql[t + 1]; qy[t] = qy[t + 1]; }
        ql[PD - 1] = (k + PD < n && lane < B) ? Lcol[(size_t)(k + PD) * B + lane] : 0.0;
        qy[PD - 1] = (k + S + PD < n && lane < nr) ? Y[(size_t)lane * ldy + k + S + PD] : 0.0;
        if (lane < nr) Y[(size_t)lane * ldy + k] = sy[slot * nr + lane];
        const int r = k + 1 + lane;
        const int rs = (slot + 1 + lane) % S;
        if (lane < B && r < n)
            for (int m = 0; m < nr; ++m) sy[rs * nr + m] -= l * sy[slot * nr + m];
        __syncwarp();
        if (k + S < n && lane < nr) sy[slot * nr + lane] = ye;
        __syncwarp();
        slot = slot + 1 == S ? 0 : slot + 1;
    }
}

// Backward sweep L^T x = D^-1 y with a stored factor (Lrow, D), nr (<= 32) RHS in place.
static __device__ void band_backward(int n, int B, const double* __restrict__ D, const double* __restrict__ Lrow,
                              double* __restrict__ Y, int nr, int ldy, double* smem) {
    const int lane = threadIdx.x & 31;
    const int S = B + 1;
    double* sx = smem;
    for (int i = lane; i < S * nr; i += 32) {
        const int c = n - 1 - i / nr, m = i % nr;
        if (c >= 0) sx[(c % S) * nr + m] = Y[(size_t)m * ldy + c] / D[c];
    }
    double ql[PD], qy[PD], qd[PD];
#pragma unroll
    for (int t = 0; t < PD; ++t) {
        const int k = n - 1 - t, c = n - 1 - S - t;
        ql[t] = (k >= 0 && lane < B) ? Lrow[(size_t)k * B + lane] : 0.0;
        qy[t] = (c >= 0 && lane < nr) ? Y[(size_t)lane * ldy + c] : 0.0;
        qd[t] = c >= 0 ? D[c] : 1.0;
    }
    __syncwarp();
    int slot = (n - 1) % S;
    for (int k = n - 1; k >= 0; --k) {
        const double l = ql[0], ye = qy[0], de = qd[0];
#pragma unroll
        for (int t = 0; t + 1 < PD; ++t) { ql[t] = ql[t + 1]; qy[t] = qy[t + 1]; qd[t] = qd[t + 1]; }
        {
            const int kk = k - PD, c = k - 1 - B - PD;
            ql[PD - 1] = (kk >= 0 && lane < B) ? Lrow[(size_t)kk * B + lane] : 0.0;
            qy[PD - 1] = (c >= 0 && lane < nr) ? Y[(size_t)lane * ldy + c] : 0.0;
            qd[PD - 1] = c >= 0 ? D[c] : 1.0;
        }
        if (lane < nr) Y[(size_t)lane * ldy + k] = sx[slot * nr + lane];
        const int c = k - B + lane;
        if (lane < B && c >= 0) {
            const int cs = (slot + S - B + lane) % S;
            for (int m = 0; m < nr; ++m) sx[cs * nr + m] -= l * sx[slot * nr + m];
        }
        __syncwarp();
        if (k - 1 - B >= 0 && lane < nr) sx[slot * nr + lane] = ye / de;
        __syncwarp();
        slot = slot == 0 ? S - 1 : slot - 1;
    }
}

}  // namespace mpm2p
