// band_twist.cuh — two-sided ("twisted") banded LDL^T of one subdomain
// system, for even half-bandwidth B <= 32: on one warp (two half-warps of 16
// lanes) for B <= 16, on a team of two warps (one per block) for B > 16.
//
// The register-window factorisation (band_reg.cuh) is a sequential chain of
// n pivots. Here two halves (half-warps, or warps of a two-warp team) run the
// same register-window step at once on two halves of the matrix:
//   * the top half (lanes 0..15) eliminates rows 0 .. m-1 in natural order;
//   * the bottom half (lanes 16..31) eliminates rows n-1 .. m+B in reverse
//     order, i.e. the natural elimination of the reversed matrix
//     A'[i][j] = A[n-1-i][n-1-j] (band structure preserved; "virtual" rows);
// and the middle rows m .. m+B-1 (m = B * floor((rows-1)/2)) stay. Each
// elimination only updates the middle block besides its own rows, so the
// middle Schur complement is S = W_top + W_bot^T - A_mid (both register
// windows end holding the middle rows, each reduced by its own side). S
// (B x B, SPD) is solved or inverted densely in registers; both halves then
// back-substitute outwards from the middle after folding the middle solution
// into their window with the multipliers L[mid][*] of their side.
// The sequential chain drops from 2n steps to about n + B.
//
// Storage of a factor (twisted layout): top rows at [0, m) of D / Lcol /
// Lrow, the top's middle multipliers as Lrow rows [m, m+B); bottom rows in
// virtual order at [m+B, n); the bottom's middle multipliers and S^-1 in two
// per-subdomain B x B arrays. A right-hand side is kept in natural order
// throughout: a half stores the eliminated value of a pivot row at that row's
// original position (its input was consumed when the row entered the window).
#pragma once

#include "band_reg.cuh"

namespace mpm2p {

template <int B>
__host__ __device__ constexpr bool twist_warps() {  // halves are whole warps (team of two per block)
    return B > 16;
}
template <int B>
__host__ __device__ constexpr int twist_ring() {  // chunks of stored factor in flight per half
    return B > 16 ? 2 : 4;
}
template <int B>
__host__ __device__ constexpr int twist_threads() {
    return twist_warps<B>() ? 64 : 32;
}
// shared memory per warp of the twisted kernels
template <int B>
__host__ __device__ constexpr int twist_smem_doubles() {
    return 2 * B * B                       // stage tiles (one per half)
           + 2 * xchg_doubles<B, 1>()      // exchange buffers (one per half)
           + 2 * twist_ring<B>() * B * B   // cp.async rings for the sweeps (one per half)
           + 2 * B * B + 4 * B + 2 * B;    // middle block: both windows, RHS, solution
}

// Per-lane geometry of the two-sided scheme.
template <int B>
struct Twist {
    static constexpr bool W = twist_warps<B>();
    static constexpr int NL = W ? 32 : 16;  // lanes per half
    int n, rows, Ct, Cb, m, Ch, obase, h, ll, llc;
    bool act;
    __device__ Twist(int n_) : n(n_) {
        const int lane = threadIdx.x & 31;
        h = W ? ((threadIdx.x >> 5) & 1) : (lane >> 4);
        ll = W ? lane : (lane & 15);
        act = ll < B;
        llc = act ? ll : 0;
        rows = n / B;
        Ct = (rows - 1) / 2;
        Cb = rows - 1 - Ct;
        m = Ct * B;
        Ch = h ? Cb : Ct;
        obase = h ? m + B : 0;
    }
    __device__ int orig(int v) const { return h ? n - 1 - v : v; }  // virtual row -> natural row
    __device__ int src(int u) const { return W ? u : (h << 4) + u; }  // shuffle source lane of row slot u
    __device__ bool leader() const { return !W || h == 0; }           // the half that solves the middle block
    __device__ void team_sync() const {
        if (W) __syncthreads();  // one team per block
        else __syncwarp();
    }
    __device__ bool team_all(bool v) const { return W ? (__syncthreads_and(v) != 0) : (__all_sync(FULL, v) != 0); }
};

// ---- phase 1: elimination ---------------------------------------------------
// Both halves eliminate their rows (top idles for chunk >= Ct), carrying one
// right-hand side Y (natural order, eliminated values written in place).
// Stores D, Lrow and (LCOL) Lcol in the twisted layout. On return the window
// registers hold the middle rows and `stage` (per half) their multipliers.
template <int B, bool LCOL>
__device__ bool twist_eliminate(const Twist<B>& T, const BandRows A, double* D, double* Lcol, double* Lrow, double* Y,
                                double* stage, double* xb, double (&reg)[B], double& yv) {
    const int n = T.n, h = T.h, ll = T.ll, llc = T.llc;
    const bool act = T.act;
    auto vdiag = [&](int i) { return A.diag[h ? n - 1 - i : i]; };
    auto vofw = [&](int i) { return A.offw[h ? n - i : i]; };          // i >= 1
    auto vofs = [&](int i) { return A.offs[h ? n - 1 - i + B : i]; };  // i >= B
#pragma unroll
    for (int t = 0; t < B; ++t) {
        double v = 0.0;
        if (act) {
            if (t == ll) v = vdiag(ll);
            else if (ll >= 1 && t == ll - 1) v = -vofw(ll);
        }
        reg[t] = v;
    }
    yv = Y[T.orig(llc)];
    for (int x = ll; x < B * B; x += T.NL) stage[x] = 0.0;
    auto fetch = [&](int row, double& fd, double& fw, double& fs, double& fb) {
        const int rr = row < n ? row : n - 1;
        fd = vdiag(rr);
        fw = vofw(rr < 1 ? 1 : rr);
        fs = vofs(rr < B ? B : rr);
        fb = Y[T.orig(rr)];
    };
    // entering-row data two chunks ahead
    double cd, cw, cs, cb, md, mw, ms, mb;
    fetch(B + llc, cd, cw, cs, cb);
    fetch(2 * B + llc, md, mw, ms, mb);
    bool ok = true;
    double st_l = 0.0;
    int st_pos = 0;
    bool st_act = false;
    __syncwarp();
    for (int c = 0; c < T.Cb; ++c) {
        const int k0 = c * B;
        const bool active = c < T.Ch;
        double nd, nw, ns, nb;
        fetch(k0 + 3 * B + llc, nd, nw, ns, nb);
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int k = k0 + u;
            const bool piv = ll == u;
            const double cval = piv ? (active ? -cs : 0.0) : reg[u];
            double* cbuf = xb + (u & 1) * B;
            double* dbuf = xb + 2 * B + (u & 1) * 2;
            double* ybuf = xb + 2 * B + 4 + (u & 1) * 2;
            if (act && st_act) stage[ll * B + st_pos] = st_l;
            if (act) cbuf[ll] = cval;
            if (piv) {
                dbuf[0] = reg[u];
                ybuf[0] = yv;
            }
            __syncwarp();
            const double d = dbuf[0];
            const double yk = ybuf[0];
            st_global_if(D + T.obase + k, d, piv && active);
            st_global_if(Y + T.orig(k), yk, piv && active);
            st_global_if(Lrow + (size_t)(T.obase + k) * B + llc, stage[u * B + llc], act && active);
            ok = ok && (!active || d > 0.0);
            const bool reset = piv && active;
            const double keep = reset ? 0.0 : 1.0;
            const double fd_ = reset ? cd : 0.0, fw_ = reset ? -cw : 0.0;
            const double l = active ? cval * fast_rcp(d) : 0.0;
            const int j = band_j_of<B>(ll, u);
            if (LCOL) st_global_if(Lcol + (size_t)(T.obase + k) * B + j, l, act && active);
            st_l = l;
            st_pos = B - 1 - j;
            st_act = active;
            const double2* cb2 = reinterpret_cast<const double2*>(cbuf);
#pragma unroll
            for (int q = 0; q < B / 2; ++q) {
                const double2 a2 = cb2[q];
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const int ci = 2 * q + hh;
                    if (ci == u) continue;
                    const double a = hh ? a2.y : a2.x;
                    const double fresh = (ci == (u + B - 1) % B) ? fw_ : 0.0;
                    reg[ci] = fma(-l, a, fma(reg[ci], keep, fresh));
                }
            }
            reg[u] = fma(-l, u % 2 ? cb2[u / 2].y : cb2[u / 2].x, fma(reg[u], keep, fd_));
            yv = fma(-l, yk, fma(yv, keep, reset ? cb : 0.0));
            __syncwarp();
        }
        cd = md;
        cw = mw;
        cs = ms;
        cb = mb;
        md = nd;
        mw = nw;
        ms = ns;
        mb = nb;
    }
    if (act && st_act) stage[ll * B + st_pos] = st_l;
    __syncwarp();
    return ok;
}

// ---- phase 2: the middle block ----------------------------------------------
// Writes both windows and RHS to `mid`, assembles S in lanes 0..B-1 (row i of
// S in srow) and the middle RHS r_i = y_top[i] + y_bot[B-1-i] - b[m+i].
// The middle rows' operator entries and RHS (untouched by the elimination),
// fetched by the leader lanes before it, so the assembly waits on no load.
struct MidPre {
    double d, wi, wi1, y;  // diag[m+i], offw[m+i], offw[m+i+1], Y[m+i] of leader lane i
};
template <int B>
__device__ __forceinline__ MidPre mid_prefetch(const Twist<B>& T, const BandRows A, const double* Y) {
    MidPre p{0.0, 0.0, 0.0, 0.0};
    const int i = threadIdx.x & 31;
    if (T.leader() && i < B) {
        p.d = A.diag[T.m + i];
        p.wi = A.offw[T.m + i];
        p.wi1 = A.offw[T.m + (i + 1 < B ? i + 1 : i)];
        p.y = Y[T.m + i];
    }
    return p;
}
template <int B>
__device__ void twist_middle_assemble(const Twist<B>& T, const BandRows A, const double* Y, const double (&reg)[B],
                                      double yv, double* mid, double (&srow)[B], double& sr, const MidPre& pre) {
    const int lane = threadIdx.x & 31, m = T.m;
    double* W = mid + T.h * B * B;
    double* rhs = mid + 2 * B * B;  // [2][B]
    if (T.act) {
#pragma unroll
        for (int t = 0; t < B; ++t) W[T.ll * B + t] = reg[t];
        rhs[T.h * B + T.ll] = yv;
    }
    T.team_sync();
    sr = 0.0;
    if (T.leader() && lane < B) {
        const int i = lane;
#pragma unroll
        for (int jj = 0; jj < B; ++jj) {
            const int lo = jj <= i ? i : jj, hi2 = jj <= i ? jj : i;  // (row lo, col hi2), hi2 <= lo
            double a0 = 0.0;  // A.diag[m + lo] on the diagonal, -A.offw[m + lo] one below
            if (lo == hi2) a0 = pre.d;
            else if (lo == hi2 + 1) a0 = -(lo == i ? pre.wi : pre.wi1);
            srow[jj] = mid[lo * B + hi2] + mid[B * B + (B - 1 - hi2) * B + (B - 1 - lo)] - a0;
        }
        sr = rhs[i] + rhs[B + B - 1 - i] - pre.y;
        (void)Y;
        (void)m;
    } else {
#pragma unroll
        for (int jj = 0; jj < B; ++jj) srow[jj] = (jj == 0 ? 1.0 : 0.0);
    }
    __syncwarp();
}

// Dense Gauss-Jordan (SPD, no pivoting) on rows [S | I | r] held by lanes
// 0..B-1; on return srow is row i of S^-1 (if INV) and sr is x_i. pr: 2(2B+2)
// doubles of shared scratch (may alias the window area of `mid`).
template <int B, bool INV>
__device__ bool twist_middle_gj(double (&srow)[B], double& sr, double* pr) {
    const int lane = threadIdx.x & 31;
    double iv[B];
#pragma unroll
    for (int jj = 0; jj < B; ++jj) iv[jj] = (INV && lane == jj) ? 1.0 : 0.0;
    bool ok = true;
    constexpr int W = 2 * B + 2;
#pragma unroll
    for (int k = 0; k < B; ++k) {
        double* prk = pr + (k & 1) * W;
        if (lane == k) {
#pragma unroll
            for (int jj = 0; jj < B; ++jj) prk[jj] = srow[jj];
            if (INV) {
#pragma unroll
                for (int jj = 0; jj < B; ++jj) prk[B + jj] = iv[jj];
            }
            prk[2 * B] = sr;
        }
        __syncwarp();
        const double p = 1.0 / prk[k];
        ok = ok && (prk[k] > 0.0);
        const bool on = lane == k;
        const double f = on ? 0.0 : srow[k] * p;
        const double sc = on ? p : 1.0;
#pragma unroll
        for (int jj = 0; jj < B; ++jj) srow[jj] = fma(-f, prk[jj], srow[jj]) * sc;
        if (INV) {
#pragma unroll
            for (int jj = 0; jj < B; ++jj) iv[jj] = fma(-f, prk[B + jj], iv[jj]) * sc;
        }
        sr = fma(-f, prk[2 * B], sr) * sc;
        __syncwarp();
    }
    if (INV) {
#pragma unroll
        for (int jj = 0; jj < B; ++jj) srow[jj] = iv[jj];
    }
    return ok;
}

// ---- phase 3: back substitution, both halves outwards from the middle -------
// midL(i, o): multiplier of this half's middle row i (its virtual order) at
// Lrow position o; xm: the middle solution (natural order, shared memory).
// dfirst: D of this lane's first back-substitution row when the caller
// prefetched it (negative: load it here).
template <int B, typename MidL>
__device__ void twist_backward(const Twist<B>& T, const double* D, const double* Lrow, double* Y, const double* xm,
                               double* ring, MidL midL, double dfirst = -1.0) {
    constexpr int RG = twist_ring<B>();
    const int h = T.h, ll = T.ll, llc = T.llc, nch = T.Cb;
    auto xmid = [&](int i) { return xm[h ? B - 1 - i : i]; };
    double z;
    {
        const int row = (T.Ch - 1) * B + llc;
        z = Y[T.orig(row)] * (1.0 / (dfirst > 0.0 ? dfirst : D[T.obase + row]));
        double corr = 0.0;
        for (int i = 0; i <= llc; ++i) corr = fma(midL(i, llc - i), xmid(i), corr);
        z -= corr;
    }
    auto rfetch = [&](int c, int slot) {
        const int cc = c < 0 ? 0 : c;
        const double* g = Lrow + (size_t)(T.obase + cc * B) * B;
        double* dst = ring + (size_t)slot * B * B;
        for (int p = ll; p < B * B / 2; p += T.NL) cp_async16(dst + 2 * p, g + 2 * p);
        cp_async_commit();
    };
#pragma unroll
    for (int i = 0; i < RG; ++i) rfetch(nch - 1 - i, i);
    auto raw = [&](int row, double& d, double& y) {
        const int rr = row < 0 ? 0 : row;
        d = D[T.obase + rr];
        y = Y[T.orig(rr)];
    };
    double rd, ry, rd2, ry2;  // (d, y) of the entering rows one and two chunks ahead
    raw((nch - 2) * B + llc, rd, ry);
    raw((nch - 3) * B + llc, rd2, ry2);
    double lq[B];
    for (int t = 0; t < nch; ++t) {
        const int c = nch - 1 - t, k0 = c * B;
        const bool active = c < T.Ch;
        const double ez = ry * (1.0 / rd);
        rd = rd2;
        ry = ry2;
        raw(k0 - 3 * B + llc, rd2, ry2);
        {
            const int slot = t % RG;
            cp_async_wait<RG - 1>();
            __syncwarp();
            const double* rs = ring + (size_t)slot * B * B;
#pragma unroll
            for (int u = 0; u < B; ++u) lq[u] = rs[u * B + (llc - u + B) % B];
            __syncwarp();
            rfetch(nch - 1 - (t + RG), slot);
        }
#pragma unroll
        for (int uu = B - 1; uu >= 0; --uu) {
            const int k = k0 + uu;
            const bool piv = ll == uu;
            const double xk = __shfl_sync(FULL, z, T.src(uu));
            st_global_if(Y + T.orig(k), xk, piv && active);
            const bool reset = piv && active;
            const double keep = reset ? 0.0 : 1.0;
            const double l = active ? lq[uu] : 0.0;
            z = fma(-l, xk, fma(z, keep, reset ? ez : 0.0));
        }
    }
    cp_async_wait<0>();  // drain the trailing ring prefetches before the caller reuses shared memory
    __syncwarp();
}

// ---- phase 1': forward sweep with a stored factor ---------------------------
// On return yv (window lanes) holds this half's reduced middle RHS.
template <int B>
__device__ void twist_forward(const Twist<B>& T, const double* Lcol, double* Y, double* ring, double& yv) {
    constexpr int RG = twist_ring<B>();
    const int n = T.n, h = T.h, ll = T.ll, llc = T.llc, nch = T.Cb;
    yv = Y[T.orig(llc)];
    auto yat = [&](int row) { return Y[T.orig(row < n ? row : n - 1)]; };
    auto rfetch = [&](int c, int slot) {
        const int cc = c < nch ? c : nch - 1;
        const double* g = Lcol + (size_t)(T.obase + cc * B) * B;
        double* dst = ring + (size_t)slot * B * B;
        for (int p = ll; p < B * B / 2; p += T.NL) cp_async16(dst + 2 * p, g + 2 * p);
        cp_async_commit();
    };
#pragma unroll
    for (int i = 0; i < RG; ++i) rfetch(i, i);
    double cb = yat(B + llc), mb = yat(2 * B + llc);
    double lq[B];
    for (int c = 0; c < nch; ++c) {
        const int k0 = c * B;
        const bool active = c < T.Ch;
        const double nb = yat(k0 + 3 * B + llc);
        {
            const int slot = c % RG;
            cp_async_wait<RG - 1>();
            __syncwarp();
            const double* rs = ring + (size_t)slot * B * B;
#pragma unroll
            for (int u = 0; u < B; ++u) lq[u] = rs[u * B + band_j_of<B>(llc, u)];
            __syncwarp();
            rfetch(c + RG, slot);
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int k = k0 + u;
            const bool piv = ll == u;
            const double yk = __shfl_sync(FULL, yv, T.src(u));
            st_global_if(Y + T.orig(k), yk, piv && active);
            const bool reset = piv && active;
            const double keep = reset ? 0.0 : 1.0;
            const double l = active ? lq[u] : 0.0;
            yv = fma(-l, yk, fma(yv, keep, reset ? cb : 0.0));
        }
        cb = mb;
        mb = nb;
    }
    cp_async_wait<0>();
    __syncwarp();
}

// ---- solvers built from the phases -------------------------------------------
// Shared-memory carve-up of one team (twist_smem_doubles<B>() doubles).
template <int B>
struct TwistSmem {
    double *stage, *xb, *ring, *mid;
    __device__ TwistSmem(const Twist<B>& T, double* sm) {
        constexpr int XB = xchg_doubles<B, 1>();
        constexpr int RG = twist_ring<B>();
        stage = sm + T.h * B * B;
        xb = sm + 2 * B * B + T.h * XB;
        ring = sm + 2 * B * B + 2 * XB + T.h * RG * B * B;
        mid = sm + 2 * B * B + 2 * XB + 2 * RG * B * B;
    }
};

// Fresh operator, one RHS (the downscale): x in Y; D / Lrow used as scratch.
template <int B>
__device__ bool twisted_solve(int n, const BandRows A, double* D, double* Lrow, double* Y, double* sm) {
    static_assert(B <= 32 && B % 2 == 0, "two halves of B lanes");
    const Twist<B> T(n);
    const TwistSmem<B> S(T, sm);
    const MidPre pre = mid_prefetch<B>(T, A, Y);
    double reg[B], yv;
    bool ok = twist_eliminate<B, false>(T, A, D, nullptr, Lrow, Y, S.stage, S.xb, reg, yv);
    double srow[B], sr;
    twist_middle_assemble<B>(T, A, Y, reg, yv, S.mid, srow, sr, pre);
    double* xm = S.mid + 2 * B * B + 2 * B;
    const int lane = threadIdx.x & 31;
    if (T.leader()) {
        ok = twist_middle_gj<B, false>(srow, sr, S.mid) && ok;
        if (lane < B) {
            xm[lane] = sr;
            Y[T.m + lane] = sr;
        }
    }
    T.team_sync();
    const double* st = S.stage;  // this half's middle multipliers, Lrow layout
    twist_backward<B>(T, D, Lrow, Y, xm, S.ring, [&](int i, int o) { return st[i * B + o]; });
    return T.team_all(ok);
}

// Rebuild factor: stores the twisted factor (D, Lcol, Lrow, the bottom's
// middle multipliers MidB and S^-1 Sinv, B x B each) and solves one RHS.
template <int B>
__device__ bool twisted_factor(int n, const BandRows A, double* D, double* Lcol, double* Lrow, double* MidB,
                               double* Sinv, double* Y, double* sm) {
    static_assert(B <= 32 && B % 2 == 0, "two halves of B lanes");
    const Twist<B> T(n);
    const TwistSmem<B> S(T, sm);
    const MidPre pre = mid_prefetch<B>(T, A, Y);
    double reg[B], yv;
    bool ok = twist_eliminate<B, true>(T, A, D, Lcol, Lrow, Y, S.stage, S.xb, reg, yv);
    {  // middle multipliers of each side: top as Lrow rows [m, m+B), bottom in MidB
        double* dst = T.h ? MidB : Lrow + (size_t)T.m * B;
        for (int x = T.ll; x < B * B; x += T.NL) dst[x] = S.stage[x];
    }
    double srow[B], sr;
    twist_middle_assemble<B>(T, A, Y, reg, yv, S.mid, srow, sr, pre);
    double* xm = S.mid + 2 * B * B + 2 * B;
    const int lane = threadIdx.x & 31;
    if (T.leader()) {
        ok = twist_middle_gj<B, true>(srow, sr, S.mid) && ok;
        if (lane < B) {
#pragma unroll
            for (int jj = 0; jj < B; ++jj) Sinv[lane * B + jj] = srow[jj];
            xm[lane] = sr;
            Y[T.m + lane] = sr;
        }
    }
    T.team_sync();
    const double* st = S.stage;
    twist_backward<B>(T, D, Lrow, Y, xm, S.ring, [&](int i, int o) { return st[i * B + o]; });
    return T.team_all(ok);
}

// Solve with a stored twisted factor (rebuild's homogeneous RHS, MPM-2P's
// particular RHS): forward sweeps, x_mid = S^-1 r_mid, back substitution.
template <int B>
__device__ void twisted_sweep(int n, const double* D, const double* Lcol, const double* Lrow, const double* MidB,
                              const double* Sinv, double* Y, double* sm) {
    const Twist<B> T(n);
    const TwistSmem<B> S(T, sm);
    // Static operands of the middle solve and of the back substitution's first
    // step (this half's middle multipliers, S^-1, the middle rows' RHS, which
    // the forward phase does not touch, and the first pivot) are fetched now,
    // asynchronously, instead of on the chain after the forward phase.
    double* mids_s = S.stage;           // B x B, this half (stage is idle in a sweep)
    double* sinv_s = S.mid;             // B x B (leader half)
    double* ymid_s = S.mid + B * B;     // B
    {
        const double* mids_g = T.h ? MidB : Lrow + (size_t)T.m * B;
        for (int p = T.ll; p < B * B / 2; p += T.NL) cp_async16(mids_s + 2 * p, mids_g + 2 * p);
        if (T.leader()) {
            for (int p = T.ll; p < B * B / 2; p += T.NL) cp_async16(sinv_s + 2 * p, Sinv + 2 * p);
            for (int p = T.ll; p < B / 2; p += T.NL) cp_async16(ymid_s + 2 * p, Y + T.m + 2 * p);
        }
        cp_async_commit();
    }
    const double dfirst = D[T.obase + (T.Ch - 1) * B + T.llc];
    double yv;
    twist_forward<B>(T, Lcol, Y, S.ring, yv);  // drains every cp.async group (ours included)
    double* rhs = S.mid + 2 * B * B;  // [2][B]
    double* xm = rhs + 2 * B;
    if (T.act) rhs[T.h * B + T.ll] = yv;
    T.team_sync();
    const int lane = threadIdx.x & 31;
    if (T.leader() && lane < B) {
        double x = 0.0;
#pragma unroll
        for (int jj = 0; jj < B; ++jj) x = fma(sinv_s[lane * B + jj], rhs[jj] + rhs[B + B - 1 - jj] - ymid_s[jj], x);
        xm[lane] = x;
    }
    T.team_sync();
    if (T.leader() && lane < B) Y[T.m + lane] = xm[lane];
    twist_backward<B>(T, D, Lrow, Y, xm, S.ring, [&](int i, int o) { return mids_s[i * B + o]; }, dfirst);
    T.team_sync();
}

}  // namespace mpm2p
