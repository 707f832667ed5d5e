// band_twist.cuh — two-sided ("twisted") banded LDL^T solve of one subdomain
// system on one warp, for half-bandwidth B <= 16.
//
// The register-window factorisation (band_reg.cuh) is a sequential chain of
// n pivots and, for B <= 16, leaves lanes 16..31 idle. Here the two half-warps
// run the same register-window step at once on two halves of the matrix:
//   * the top half (lanes 0..15) eliminates rows 0 .. m-1 in natural order;
//   * the bottom half (lanes 16..31) eliminates rows n-1 .. m+B in reverse
//     order, i.e. the natural elimination of the reversed matrix
//     A'[i][j] = A[n-1-i][n-1-j] (band structure preserved);
// where the middle rows m .. m+B-1 (m = B * floor((rows-1)/2)) stay. Each
// elimination only updates the middle block besides its own rows, so its
// Schur complement is S = W_top + W_bot^T - A_mid (both windows end holding
// the middle rows, each reduced by its own side). S (B x B, SPD) is solved
// densely in registers, then both halves back-substitute outwards from the
// middle, first folding the middle solution into their window with the
// multipliers L[mid][*] left in their stage tiles.
// The sequential chain drops from 2n steps to about n + B + small.
//
// Outputs: x in Y (natural order). Factor storage (used inside the kernel
// only): top rows in D/Lrow[0, m), bottom rows (reversed order) in
// D/Lrow[m+B, n); the bottom's forward-eliminated RHS goes to Yv[0, n-m-B)
// (a separate buffer: Y's entries there are still unread inputs).
#pragma once

#include "band_reg.cuh"

namespace mpm2p {

template <int B>
__host__ __device__ constexpr int twist_ring() {
    return 2;
}
template <int B>
__host__ __device__ constexpr int twist_smem_doubles() {  // per warp
    return 2 * B * B                 // stage tiles (one per half)
           + 2 * xchg_doubles<B, 1>()  // exchange buffers (one per half)
           + 2 * twist_ring<B>() * B * B  // cp.async rings for the back substitution (one per half)
           + 2 * B * B + 4 * B + 2 * B;   // middle block: both windows, RHS, solution
}

template <int B>
__device__ bool twisted_solve(int n, const BandRows A, double* D, double* Lrow, double* Y, double* Yv, double* sm) {
    static_assert(B <= 16 && B % 2 == 0, "two half-warps of B lanes");
    constexpr int XB = xchg_doubles<B, 1>();
    constexpr int RG = twist_ring<B>();
    const int lane = threadIdx.x & 31;
    const int h = lane >> 4, ll = lane & 15;
    const bool act = ll < B;
    const int llc = act ? ll : 0;
    const int rows = n / B;
    const int Ct = (rows - 1) / 2, Cb = rows - 1 - Ct;  // chunks eliminated by each half (Cb >= Ct)
    const int m = Ct * B;                              // first middle row
    const int Ch = h ? Cb : Ct;
    const int obase = h ? m + B : 0;                   // storage offset of this half's factor rows
    double* stage = sm + h * B * B;
    double* xb = sm + 2 * B * B + h * XB;
    double* ring = sm + 2 * B * B + 2 * XB + h * RG * B * B;
    double* mid = sm + 2 * B * B + 2 * XB + 2 * RG * B * B;  // [2][B][B] windows, then RHS and x
    double* Yel = h ? Yv : Y;                           // forward-eliminated RHS, virtual order
    // virtual row -> matrix entries of this half
    auto vdiag = [&](int i) { return A.diag[h ? n - 1 - i : i]; };
    auto vofw = [&](int i) { return A.offw[h ? n - i : i]; };          // i >= 1
    auto vofs = [&](int i) { return A.offs[h ? n - 1 - i + B : i]; };  // i >= B
    auto vrhs = [&](int i) { return Y[h ? n - 1 - i : i]; };
    double reg[B];
    double yv;
#pragma unroll
    for (int t = 0; t < B; ++t) {
        double v = 0.0;
        if (act) {
            if (t == ll) v = vdiag(ll);
            else if (ll >= 1 && t == ll - 1) v = -vofw(ll);
        }
        reg[t] = v;
    }
    yv = vrhs(llc);
    for (int x = ll; x < B * B; x += 16) stage[x] = 0.0;
    auto fetch = [&](int row, double& fd, double& fw, double& fs, double& fb) {
        const int rr = row < n ? row : n - 1;
        fd = vdiag(rr);
        fw = vofw(rr < 1 ? 1 : rr);
        fs = vofs(rr < B ? B : rr);
        fb = vrhs(rr);
    };
    // entering-row data two chunks ahead (one chunk of steps is shorter than a
    // cold HBM round trip)
    double cd, cw, cs, cb, md, mw, ms, mb;
    fetch(B + llc, cd, cw, cs, cb);
    fetch(2 * B + llc, md, mw, ms, mb);
    bool ok = true;
    double st_l = 0.0;
    int st_pos = 0;
    bool st_act = false;
    __syncwarp();
    // ---- elimination: chunk c, both halves; the top idles for c >= Ct ------
    for (int c = 0; c < Cb; ++c) {
        const int k0 = c * B;
        const bool active = c < Ch;
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
            st_global_if(D + obase + k, d, piv && active);
            st_global_if(Yel + k, yk, piv && active);
            st_global_if(Lrow + (size_t)(obase + k) * B + llc, stage[u * B + llc], act && active);
            ok = ok && (!active || d > 0.0);
            const bool reset = piv && active;
            const double keep = reset ? 0.0 : 1.0;
            const double fd_ = reset ? cd : 0.0, fw_ = reset ? -cw : 0.0;
            const double l = active ? cval * fast_rcp(d) : 0.0;
            const int j = band_j_of<B>(ll, u);
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
    // ---- middle block ------------------------------------------------------
    // window lane i of each half holds middle row (top) m+i / (bottom) m+B-1-i;
    // register j holds its entry in middle column (top) m+j / (bottom) m+B-1-j
    double* W = mid + h * B * B;
    double* rhs = mid + 2 * B * B;  // [2][B]
    double* xm = rhs + 2 * B;       // [B] middle solution (+ B spare)
    if (act) {
#pragma unroll
        for (int t = 0; t < B; ++t) W[ll * B + t] = reg[t];
        rhs[h * B + ll] = yv;
    }
    __syncwarp();
    // lanes 0..B-1: row i of S = W_top[i][j] + W_bot[B-1-j][B-1-i] - A_mid[i][j] (j <= i, mirrored)
    double srow[B];
    double sr = 0.0;
    if (lane < B) {
        const int i = lane;
#pragma unroll
        for (int jj = 0; jj < B; ++jj) {
            const int lo = jj <= i ? i : jj, hi2 = jj <= i ? jj : i;  // (row lo, col hi2), hi2 <= lo
            double a0 = 0.0;
            if (lo == hi2) a0 = A.diag[m + lo];
            else if (lo == hi2 + 1) a0 = -A.offw[m + lo];
            srow[jj] = mid[lo * B + hi2] + mid[B * B + (B - 1 - hi2) * B + (B - 1 - lo)] - a0;
        }
        sr = rhs[i] + rhs[B + B - 1 - i] - Y[m + i];
    } else {
#pragma unroll
        for (int jj = 0; jj < B; ++jj) srow[jj] = (jj == 0 ? 1.0 : 0.0);
    }
    __syncwarp();
    // dense Gauss-Jordan on [S | r] (SPD: no pivoting), row i in lane i
    double* pr = mid;  // reuse the window area: pivot row broadcast (B + 1 doubles, two parities)
#pragma unroll
    for (int k = 0; k < B; ++k) {
        double* prk = pr + (k & 1) * (B + 2);
        if (lane == k) {
#pragma unroll
            for (int jj = 0; jj < B; ++jj) prk[jj] = srow[jj];
            prk[B] = sr;
        }
        __syncwarp();
        const double p = 1.0 / prk[k];
        ok = ok && (prk[k] > 0.0);
        const bool on = lane == k;
        const double f = on ? 0.0 : srow[k] * p;
        const double sc = on ? p : 1.0;
#pragma unroll
        for (int jj = 0; jj < B; ++jj) srow[jj] = fma(-f, prk[jj], srow[jj]) * sc;
        sr = fma(-f, prk[B], sr) * sc;
        __syncwarp();
    }
    if (lane < B) {
        xm[lane] = sr;
        Y[m + lane] = sr;
    }
    __syncwarp();
    // ---- back substitution, both halves outwards from the middle ------------
    // this half's middle solution in its own (virtual) order
    auto xmid = [&](int i) { return xm[h ? B - 1 - i : i]; };
    const int nch = Cb;
    // window: rows of this half's last chunk Ch-1 (virtual), z = y/d - sum_mid L[mid][row] x_mid
    double z;
    {
        const int row = (Ch - 1) * B + llc;
        z = Yel[row] * (1.0 / D[obase + row]);
        double corr = 0.0;
        for (int i = 0; i <= llc; ++i) corr = fma(stage[i * B + (llc - i)], xmid(i), corr);
        z -= corr;
    }
    // stored factor rows of this half: chunk c of Lrow starts at row obase + c*B
    auto rfetch = [&](int c, int slot) {
        const int cc = c < 0 ? 0 : c;
        const double* g = Lrow + (size_t)(obase + cc * B) * B;
        double* dst = ring + (size_t)slot * B * B;
        for (int p = ll; p < B * B / 2; p += 16) cp_async16(dst + 2 * p, g + 2 * p);
        cp_async_commit();
    };
#pragma unroll
    for (int i = 0; i < RG; ++i) rfetch(nch - 1 - i, i);
    auto raw = [&](int row, double& d, double& y) {
        const int rr = row < 0 ? 0 : row;
        d = D[obase + rr];
        y = Yel[rr];
    };
    double rd, ry, rd2, ry2;  // (d, y) of the entering rows one and two chunks ahead
    raw((nch - 2) * B + llc, rd, ry);
    raw((nch - 3) * B + llc, rd2, ry2);
    double lq[B];
    for (int t = 0; t < nch; ++t) {
        const int c = nch - 1 - t, k0 = c * B;
        const bool active = c < Ch;
        const double ez = ry * (1.0 / rd);  // entering rows of this chunk (chunk c-1), loaded two chunks ago
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
            const double xk = __shfl_sync(FULL, z, (h << 4) + uu);
            st_global_if(Y + (h ? n - 1 - k : k), xk, piv && active);
            const bool reset = piv && active;
            const double keep = reset ? 0.0 : 1.0;
            const double l = active ? lq[uu] : 0.0;
            z = fma(-l, xk, fma(z, keep, reset ? ez : 0.0));
        }
    }
    cp_async_wait<0>();  // drain the trailing ring prefetches before the caller reuses shared memory
    __syncwarp();
    return __all_sync(FULL, ok);
}

}  // namespace mpm2p
