// fine.cu — the fine-reference pressure solve on the device (SURVEY.md §8(f)
// item 1). The reference builds a fresh CellCenteredSolver on the whole grid
// (proj/src/simulation.cpp:143-150 -> elliptic.cpp:68-243: 5-point assembly,
// Eigen SimplicialLDLT, velocity recovery) every step of the FineReference
// method and, with track_errors, for the reference saturation s_ref.
//
// B200 design: the global system is never factored. It is solved by
// preconditioned CG in ONE cooperative persistent kernel (k_fine_pcg):
//  * preconditioner: two-level Schwarz in the A-DEF2 (deflation) form —
//    block-Jacobi over the MRCM subdomains, each block the principal
//    submatrix of A factored once per solve by the register-window banded
//    LDL^T of band_reg.cuh (one warp per subdomain), plus the piecewise-
//    constant coarse space A0 = R A R^T (n_sub x n_sub, inverted densely):
//        y = B^-1 r,   z = y + R^T A0^-1 R (r - A y),
//    started from the deflated guess x0 = x_prev + R^T A0^-1 R (b - A x_prev)
//    (x_prev: the previous fine solution of the run, else 0). On C2 this
//    needs ~120 iterations to ||r|| <= 1e-13 ||b|| against ~190 for the
//    additive form (tools/fine_pcg_proto.py);
//  * every reduction is formed per subdomain (warp sums) and the n_sub
//    partials are combined by every block in the same order, so all blocks
//    hold bit-identical CG scalars and a solve is deterministic;
//  * stop at ||r||_2 <= tol ||b||_2 (tol 1e-13, MPM2P_FINE_TOL; the
//    reference's own CG fallback stops at 1e-12, elliptic.cpp:185-197);
//    no convergence within maxit sets ERR_FINE_NOCONV (NumericError).
// Vectors live in the subdomain-blocked order (s * ncs + local row-major),
// the order the band kernels use; p and u come back in the global layouts.
#include <cooperative_groups.h>

#include <cmath>
#include <cstdlib>
#include <cstring>

#include "band_reg.cuh"
#include "context.cuh"
#include "cr.cuh"

namespace cg = cooperative_groups;

namespace mpm2p {

namespace {

constexpr int TPB = 256;
constexpr int FWPB = 4;  // warps (subdomains) per block in the fine kernels

__device__ __forceinline__ int sub_of(const Layout& L, int i, int j) { return (j / L.sny) * L.nsx + i / L.snx; }
__device__ __forceinline__ int bidx(const Layout& L, int i, int j) {
    return sub_of(L, i, j) * L.ncs + (j % L.sny) * L.snx + i % L.snx;
}

// Boundary face data in BoundarySpec order W(ny) E(ny) S(nx) N(nx).
__device__ __forceinline__ int gbc_w(const Layout& L, int j) { return j; }
__device__ __forceinline__ int gbc_e(const Layout& L, int j) { return L.ny + j; }
__device__ __forceinline__ int gbc_s(const Layout& L, int i) { return 2 * L.ny + i; }
__device__ __forceinline__ int gbc_n(const Layout& L, int i) { return 2 * L.ny + L.nx + i; }

// ---------------------------------------------------------------- assembly ----
// elliptic.cpp:44-61 (transmissibility, boundary faces carry kappa*area/(h/2))
// and :80-141 (5-point rows: interior couplings in the order W, E, S, N, then
// the boundary faces W, E, S, N: Pressure adds t_half; the anchor row becomes
// identity with its couplings zeroed) and the rhs of :161-180 (q vol +
// t_half g - z area; anchor rhs 0). Written straight into the blocked band
// rows of the block-Jacobi factorisation (BW/BS: coupling magnitudes inside
// a subdomain only) plus the global face transmissibilities T for the SpMV.
__global__ void k_fine_assemble(Layout L, int anchor, const double* __restrict__ kappa,
                                const double* __restrict__ q, const int* __restrict__ bc_kind,
                                const double* __restrict__ bc_value, double* __restrict__ T,
                                double* __restrict__ BD, double* __restrict__ BW, double* __restrict__ BS,
                                double* __restrict__ b, Scalars* sc) {
    pdl_begin();
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < L.cells(); c += gridDim.x * blockDim.x) {
        const int i = c % L.nx, j = c / L.nx;
        const double k = kappa[c];
        if (!(k > 0.0) || !isfinite(k)) atomicOr(&sc->err, ERR_KAPPA);
        const double tw = i > 0 ? harm_trans_v(L, kappa[c - 1], k) : half_trans(L, SIDE_W, k);
        const double te = i < L.nx - 1 ? harm_trans_v(L, k, kappa[c + 1]) : half_trans(L, SIDE_E, k);
        const double ts = j > 0 ? harm_trans_h(L, kappa[c - L.nx], k) : half_trans(L, SIDE_S, k);
        const double tn = j < L.ny - 1 ? harm_trans_h(L, k, kappa[c + L.nx]) : half_trans(L, SIDE_N, k);
        T[L.vface(i, j)] = tw;
        T[L.hface(i, j)] = ts;
        if (i == L.nx - 1) T[L.vface(L.nx, j)] = te;
        if (j == L.ny - 1) T[L.hface(i, L.ny)] = tn;
        double diag = 0.0;
        if (i > 0) diag += tw;
        if (i < L.nx - 1) diag += te;
        if (j > 0) diag += ts;
        if (j < L.ny - 1) diag += tn;
        const double vol = L.vol();
        double rhs = q ? q[c] * vol : 0.0;
        auto bnd = [&](int gbc, double th, double area) {
            const int kind = bc_kind[gbc];
            if (kind == BC_PRESSURE) {
                diag += th;
                rhs += th * bc_value[gbc];
            } else if (kind == BC_FLUX) {
                rhs -= bc_value[gbc] * area;
            } else {  // Robin (elliptic.cpp:133-136,176-177)
                if (!(L.rb_beta[gbc] > 0.0)) atomicOr(&sc->err, ERR_ROBIN_BETA);
                const double er = eff_robin(th, L.rb_beta[gbc], area);
                diag += er;
                rhs += er * L.rb_rhs[gbc];
            }
        };
        if (i == 0) bnd(gbc_w(L, j), tw, L.hy);
        if (i == L.nx - 1) bnd(gbc_e(L, j), te, L.hy);
        if (j == 0) bnd(gbc_s(L, i), ts, L.hx);
        if (j == L.ny - 1) bnd(gbc_n(L, i), tn, L.hx);
        const int kb = bidx(L, i, j);
        const bool anc = c == anchor;
        BD[kb] = anc ? 1.0 : diag;
        // band rows carry the coupling magnitude (A[r][r-1] = -BW[r], A[r][r-B] = -BS[r]; k_band_entries)
        BW[kb] = (i % L.snx > 0 && !anc && c - 1 != anchor) ? tw : 0.0;
        BS[kb] = (j % L.sny > 0 && !anc && c - L.nx != anchor) ? ts : 0.0;
        b[kb] = anc ? 0.0 : rhs;
    }
}

// The global operator applied to a blocked vector v at blocked row k (cell
// (i, j)); with e != nullptr it is applied to v + R^T e (v may then be null).
// v and e are written by other blocks between grid barriers of k_fine_pcg
// (y is even rewritten in place, y := z, between two phases that read the
// neighbours' y), so they are read through L2 (ld.cg): a plain load could
// hit a line this SM cached before the barrier.
__device__ __forceinline__ double fine_apply(const Layout& L, int anchor, const double* __restrict__ T,
                                             const double* __restrict__ BD, const double* v, const double* e,
                                             int k, int i, int j) {
    auto val = [&](int ii, int jj) {
        double t = v ? __ldcg(v + bidx(L, ii, jj)) : 0.0;
        if (e) t += __ldcg(e + sub_of(L, ii, jj));
        return t;
    };
    const int c = L.cell(i, j);
    double y = BD[k] * val(i, j);
    if (c == anchor) return y;
    if (i > 0 && c - 1 != anchor) y -= T[L.vface(i, j)] * val(i - 1, j);
    if (i < L.nx - 1 && c + 1 != anchor) y -= T[L.vface(i + 1, j)] * val(i + 1, j);
    if (j > 0 && c - L.nx != anchor) y -= T[L.hface(i, j)] * val(i, j - 1);
    if (j < L.ny - 1 && c + L.nx != anchor) y -= T[L.hface(i, j + 1)] * val(i, j + 1);
    return y;
}

// Block-Jacobi factorisation: one warp per subdomain (the band rows of its
// principal submatrix), Y is scratch for the fused forward sweep.
template <int B>
__global__ void __launch_bounds__(FWPB * 32) k_fine_factor(Layout L, const double* __restrict__ BD,
                                                           const double* __restrict__ BW,
                                                           const double* __restrict__ BS, double* D, double* Lc,
                                                           double* Lr, double* Y, Scalars* sc) {
    pdl_begin();
    __shared__ double stage[FWPB][B * B];
    __shared__ __align__(16) double xbuf[FWPB][xchg_doubles<B, 1>()];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = blockIdx.x * FWPB + w;
    if (s >= L.n_sub) return;
    const int n = L.ncs;
    const size_t so = (size_t)s * n;
    const BandRows A{BD + so, BW + so, BS + so};
    for (int r = lane; r < n; r += 32) Y[so + r] = 0.0;
    __syncwarp();
    const bool ok = factor_fwd_reg<B, 1>(n, A, D + so, Lc + so * B, Lr + so * B, Y + so, 1, n, stage[w], xbuf[w]);
    if (!ok && lane == 0) atomicOr(&sc->err, ERR_PIVOT);
}

// Coarse operator A0 = R A R^T (R: subdomain indicator rows), one warp per
// subdomain row; the cross-subdomain entries sum -T over the shared edge in
// edge order, so A0 is bitwise symmetric. A0 must be zeroed beforehand.
__global__ void k_fine_coarse(Layout L, int anchor, const double* __restrict__ T, const double* __restrict__ BD,
                              const double* __restrict__ BW, const double* __restrict__ BS,
                              double* __restrict__ A0) {
    pdl_begin();
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int s = w;
    if (s >= L.n_sub) return;
    const int n = L.ncs, ns = L.n_sub;
    const size_t so = (size_t)s * n;
    double d = 0.0;
    for (int r = lane; r < n; r += 32) d += BD[so + r] - 2.0 * (BW[so + r] + BS[so + r]);
    d = warp_sum(d);
    const int sx = s % L.nsx, sy = s / L.nsx, i0 = L.sub_i0(s), j0 = L.sub_j0(s);
    auto edge = [&](int cnt, bool vert, int fi, int fj) {  // sum of -T over the shared edge
        double t = 0.0;
        for (int m = lane; m < cnt; m += 32) {
            const int ii = vert ? fi : fi + m, jj = vert ? fj + m : fj;
            int ca, cb;  // the two cells of the face
            double tf;
            if (vert) {
                ca = L.cell(ii - 1, jj);
                cb = L.cell(ii, jj);
                tf = T[L.vface(ii, jj)];
            } else {
                ca = L.cell(ii, jj - 1);
                cb = L.cell(ii, jj);
                tf = T[L.hface(ii, jj)];
            }
            if (ca != anchor && cb != anchor) t -= tf;
        }
        return warp_sum(t);
    };
    const double ew = sx > 0 ? edge(L.sny, true, i0, j0) : 0.0;
    const double ee = sx < L.nsx - 1 ? edge(L.sny, true, i0 + L.snx, j0) : 0.0;
    const double es = sy > 0 ? edge(L.snx, false, i0, j0) : 0.0;
    const double en = sy < L.nsy - 1 ? edge(L.snx, false, i0, j0 + L.sny) : 0.0;
    if (lane == 0) {
        double* row = A0 + (size_t)s * ns;
        row[s] = d;
        if (sx > 0) row[s - 1] = ew;
        if (sx < L.nsx - 1) row[s + 1] = ee;
        if (sy > 0) row[s - L.nsx] = es;
        if (sy < L.nsy - 1) row[s + L.nsx] = en;
    }
}

// The same coarse operator into block-tridiagonal form for the cyclic
// reduction: block sy = the subdomains of row sy (S >= nsx, identity pad),
// D[sy][sx][sx'] and the upper coupling Up[sy][sx][sx] to row sy + 1. Same
// per-edge sums and order as k_fine_coarse.
__global__ void k_fine_coarse_cr(Layout L, int anchor, const double* __restrict__ T, const double* __restrict__ BD,
                                 const double* __restrict__ BW, const double* __restrict__ BS, int S,
                                 double* __restrict__ D, double* __restrict__ Up) {
    pdl_begin();
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nblk_rows = L.nsy * S;
    if (w >= nblk_rows) return;
    const int sy = w / S, sx = w % S;
    double* drow = D + ((size_t)sy * S + sx) * S;
    if (sx >= L.nsx) {  // pad row: identity
        if (lane == 0) drow[sx] = 1.0;
        return;
    }
    const int s = sy * L.nsx + sx;
    const int n = L.ncs;
    const size_t so = (size_t)s * n;
    double d = 0.0;
    for (int r = lane; r < n; r += 32) d += BD[so + r] - 2.0 * (BW[so + r] + BS[so + r]);
    d = warp_sum(d);
    const int i0 = L.sub_i0(s), j0 = L.sub_j0(s);
    auto edge = [&](int cnt, bool vert, int fi, int fj) {
        double t = 0.0;
        for (int m = lane; m < cnt; m += 32) {
            const int ii = vert ? fi : fi + m, jj = vert ? fj + m : fj;
            int ca, cb;
            double tf;
            if (vert) {
                ca = L.cell(ii - 1, jj);
                cb = L.cell(ii, jj);
                tf = T[L.vface(ii, jj)];
            } else {
                ca = L.cell(ii, jj - 1);
                cb = L.cell(ii, jj);
                tf = T[L.hface(ii, jj)];
            }
            if (ca != anchor && cb != anchor) t -= tf;
        }
        return warp_sum(t);
    };
    const double ew = sx > 0 ? edge(L.sny, true, i0, j0) : 0.0;
    const double ee = sx < L.nsx - 1 ? edge(L.sny, true, i0 + L.snx, j0) : 0.0;
    const double en = sy < L.nsy - 1 ? edge(L.snx, false, i0, j0 + L.sny) : 0.0;
    if (lane == 0) {
        drow[sx] = d;
        if (sx > 0) drow[sx - 1] = ew;
        if (sx < L.nsx - 1) drow[sx + 1] = ee;
        if (sy < L.nsy - 1) Up[((size_t)sy * S + sx) * S + sx] = en;
    }
}

struct FineArgs {
    Layout L;
    int anchor;
    const double* T;
    const double* BD;
    const double* D;
    const double* Lc;
    const double* Lr;
    const double* A0i;  // n_sub x n_sub
    const double* b;
    double *x, *r, *p, *q, *y;
    double *c0, *e;
    double* part;  // 4 * n_sub partials
    double tol;
    int maxit;
    Scalars* sc;
    // cyclic-reduction coarse solve (cr_nphase > 0): jobs read cy, write cx
    const GemvJob* cr_jobs;
    const int2* cr_phases;
    int cr_nphase, cr_S;
    double *cy, *cx;
};

// Sum of n per-subdomain partials; every block forms it in the same order.
__device__ __forceinline__ double fine_all_sum(const double* part, int n, double* sh) {
    double v = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) v += __ldcg(part + i);
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += sh[k];
    return s;
}

// e = A0^-1 c0: one warp per coarse row of the dense inverse, or the
// cyclic-reduction phases (c0 into the padded block vector, the solve, e out)
__device__ __forceinline__ void fine_coarse_solve(const FineArgs& a, int gw, int nw, int lane,
                                                  cg::grid_group& grid) {
    const int ns = a.L.n_sub;
    if (a.cr_nphase > 0) {
        const int nsx = a.L.nsx;
        for (int s = gw * 32 + lane; s < ns; s += nw * 32) a.cy[(size_t)(s / nsx) * a.cr_S + s % nsx] = __ldcg(a.c0 + s);
        grid.sync();
        cr_solve_in_kernel(a.cr_jobs, a.cr_phases, a.cr_nphase, a.cr_S, grid);
        for (int s = gw * 32 + lane; s < ns; s += nw * 32) a.e[s] = __ldcg(a.cx + (size_t)(s / nsx) * a.cr_S + s % nsx);
        return;
    }
    for (int row = gw; row < ns; row += nw) {
        const double* ar = a.A0i + (size_t)row * ns;
        double t = 0.0;
        for (int k = lane; k < ns; k += 32) t += ar[k] * __ldcg(a.c0 + k);
        t = warp_sum(t);
        if (lane == 0) a.e[row] = t;
    }
}

template <int B>
__global__ void __launch_bounds__(FWPB * 32) k_fine_pcg(FineArgs a) {
    pdl_begin();
    cg::grid_group grid = cg::this_grid();
    __shared__ __align__(16) double ring[FWPB][sweep_ring<B>() * B * B + 2];
    __shared__ double sh[32];
    const Layout& L = a.L;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gw = blockIdx.x * FWPB + w, nw = gridDim.x * FWPB;
    const int n = L.ncs, ns = L.n_sub;
    double* pb = a.part;       // ||b||^2 per subdomain
    double* p1 = a.part + ns;  // rho / pq / rr partials
    double* p2 = a.part + 2 * ns;
    double* p3 = a.part + 3 * ns;
    auto cell_ij = [&](int s, int rr, int& i, int& j) {
        i = L.sub_i0(s) + rr % L.snx;
        j = L.sub_j0(s) + rr / L.snx;
    };
    // start: r = b - A x_prev; c0 = R r
    for (int s = gw; s < ns; s += nw) {
        double sb = 0.0, sr = 0.0;
        for (int rr = lane; rr < n; rr += 32) {
            const int k = s * n + rr;
            int i, j;
            cell_ij(s, rr, i, j);
            const double bk = a.b[k];
            const double res = bk - fine_apply(L, a.anchor, a.T, a.BD, a.x, nullptr, k, i, j);
            a.r[k] = res;
            sb += bk * bk;
            sr += res;
        }
        sb = warp_sum(sb);
        sr = warp_sum(sr);
        if (lane == 0) {
            pb[s] = sb;
            a.c0[s] = sr;
        }
    }
    grid.sync();
    fine_coarse_solve(a, gw, nw, lane, grid);
    grid.sync();
    // deflated start: x += R^T e, r -= A R^T e
    for (int s = gw; s < ns; s += nw) {
        double sr = 0.0;
        const double es = __ldcg(a.e + s);
        for (int rr = lane; rr < n; rr += 32) {
            const int k = s * n + rr;
            int i, j;
            cell_ij(s, rr, i, j);
            a.x[k] += es;
            const double res = a.r[k] - fine_apply(L, a.anchor, a.T, a.BD, nullptr, a.e, k, i, j);
            a.r[k] = res;
            sr += res * res;
        }
        sr = warp_sum(sr);
        if (lane == 0) p3[s] = sr;
    }
    grid.sync();
    const double bb = fine_all_sum(pb, ns, sh);
    double rr2 = fine_all_sum(p3, ns, sh);
    const double stop2 = a.tol * a.tol * bb;
    int it = 0;
    bool conv = !(rr2 > stop2);
    double rho_old = 1.0;
    while (!conv && it < a.maxit) {
        ++it;
        // y = B^-1 r (block-Jacobi, in place on y)
        for (int s = gw; s < ns; s += nw) {
            const size_t so = (size_t)s * n;
            for (int rr = lane; rr < n; rr += 32) a.y[so + rr] = a.r[so + rr];
            __syncwarp();
            forward_reg<B, 1>(n, a.Lc + so * B, a.y + so, 1, n, nullptr, ring[w]);
            __syncwarp();
            backward_reg<B, 1>(n, a.D + so, a.Lr + so * B, a.y + so, 1, n, nullptr, ring[w]);
            __syncwarp();
        }
        grid.sync();
        // c0 = R (r - A y)
        for (int s = gw; s < ns; s += nw) {
            double sr = 0.0;
            for (int rr = lane; rr < n; rr += 32) {
                const int k = s * n + rr;
                int i, j;
                cell_ij(s, rr, i, j);
                sr += a.r[k] - fine_apply(L, a.anchor, a.T, a.BD, a.y, nullptr, k, i, j);
            }
            sr = warp_sum(sr);
            if (lane == 0) a.c0[s] = sr;
        }
        grid.sync();
        fine_coarse_solve(a, gw, nw, lane, grid);
        grid.sync();
        // z = y + R^T e (in place on y); rho = r . z
        for (int s = gw; s < ns; s += nw) {
            double sr = 0.0;
            const double es = __ldcg(a.e + s);
            for (int rr = lane; rr < n; rr += 32) {
                const int k = s * n + rr;
                const double z = a.y[k] + es;
                a.y[k] = z;
                sr += a.r[k] * z;
            }
            sr = warp_sum(sr);
            if (lane == 0) p1[s] = sr;
        }
        grid.sync();
        const double rho = fine_all_sum(p1, ns, sh);
        const double beta = it == 1 ? 0.0 : rho / rho_old;
        // p = z + beta p; q = A z + beta q (A p without another barrier)
        for (int s = gw; s < ns; s += nw) {
            double sr = 0.0;
            for (int rr = lane; rr < n; rr += 32) {
                const int k = s * n + rr;
                int i, j;
                cell_ij(s, rr, i, j);
                const double az = fine_apply(L, a.anchor, a.T, a.BD, a.y, nullptr, k, i, j);
                const double pk = it == 1 ? a.y[k] : a.y[k] + beta * a.p[k];
                const double qk = it == 1 ? az : az + beta * a.q[k];
                a.p[k] = pk;
                a.q[k] = qk;
                sr += pk * qk;
            }
            sr = warp_sum(sr);
            if (lane == 0) p2[s] = sr;
        }
        grid.sync();
        const double alpha = rho / fine_all_sum(p2, ns, sh);
        for (int s = gw; s < ns; s += nw) {
            double sr = 0.0;
            for (int rr = lane; rr < n; rr += 32) {
                const int k = s * n + rr;
                a.x[k] += alpha * a.p[k];
                const double res = a.r[k] - alpha * a.q[k];
                a.r[k] = res;
                sr += res * res;
            }
            sr = warp_sum(sr);
            if (lane == 0) p3[s] = sr;
        }
        grid.sync();
        rr2 = fine_all_sum(p3, ns, sh);
        rho_old = rho;
        conv = !(rr2 > stop2);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.sc->fine_iters = it;
        a.sc->fine_relres = bb > 0.0 ? sqrt(rr2 / bb) : 0.0;
        a.sc->fine_iters_total += it;
        if (!conv) atomicOr(&a.sc->err, ERR_FINE_NOCONV);
    }
}

// Pressure to the global layout and the face velocities of elliptic.cpp:
// 199-240 (interior t (p_L - p_R)/area; Pressure faces t_half (p_c - g)/area,
// Flux faces z, in global orientation), plus conservation_residual /
// residual_scale (elliptic.cpp:252-267) of the result.
__global__ void k_fine_velocity(Layout L, const double* __restrict__ T, const int* __restrict__ bc_kind,
                                const double* __restrict__ bc_value, const double* __restrict__ q,
                                const double* __restrict__ x, double* __restrict__ p, double* __restrict__ u,
                                Scalars* sc, double* part, unsigned* counter) {
    pdl_begin();
    double res = 0.0, scale = 0.0;
    const double vol = L.vol();
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < L.cells(); c += gridDim.x * blockDim.x) {
        const int i = c % L.nx, j = c / L.nx;
        const double xc = x[bidx(L, i, j)];
        p[c] = xc;
        auto bnd = [&](int gbc, int f, double area, double sgn) {
            const int kind = bc_kind[gbc];
            const double un = kind == BC_PRESSURE ? T[f] * (xc - bc_value[gbc]) / area
                              : kind == BC_ROBIN  ? eff_robin(T[f], L.rb_beta[gbc], area) * (xc - L.rb_rhs[gbc]) / area
                                                  : bc_value[gbc];
            return sgn * un;
        };
        const int fw = L.vface(i, j), fe = L.vface(i + 1, j), fs = L.hface(i, j), fn = L.hface(i, j + 1);
        const double uW = i > 0 ? T[fw] * (x[bidx(L, i - 1, j)] - xc) / L.hy : bnd(gbc_w(L, j), fw, L.hy, -1.0);
        const double uE = i < L.nx - 1 ? T[fe] * (xc - x[bidx(L, i + 1, j)]) / L.hy : bnd(gbc_e(L, j), fe, L.hy, 1.0);
        const double uS = j > 0 ? T[fs] * (x[bidx(L, i, j - 1)] - xc) / L.hx : bnd(gbc_s(L, i), fs, L.hx, -1.0);
        const double uN = j < L.ny - 1 ? T[fn] * (xc - x[bidx(L, i, j + 1)]) / L.hx : bnd(gbc_n(L, i), fn, L.hx, 1.0);
        u[fw] = uW;
        u[fs] = uS;
        scale = fmax(scale, fabs(uW) * L.hy / vol);
        scale = fmax(scale, fabs(uS) * L.hx / vol);
        if (i == L.nx - 1) {
            u[fe] = uE;
            scale = fmax(scale, fabs(uE) * L.hy / vol);
        }
        if (j == L.ny - 1) {
            u[fn] = uN;
            scale = fmax(scale, fabs(uN) * L.hx / vol);
        }
        const double qc = q ? q[c] : 0.0;
        const double fx = (uE - uW) * L.hy;
        const double fy = (uN - uS) * L.hx;
        res = fmax(res, fabs((fx + fy) / vol - qc));
        scale = fmax(scale, fabs(qc));
    }
    __shared__ double shm[32 * 2];
    __shared__ double red[2];
    double v[2] = {res, scale};
    block_reduce_multi<2>(v, 0u, shm, red);
    if (threadIdx.x < 2) part[2 * blockIdx.x + threadIdx.x] = red[threadIdx.x];
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    double t[2] = {0.0, 0.0};
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
        t[0] = fmax(t[0], __ldcg(part + 2 * b));
        t[1] = fmax(t[1], __ldcg(part + 2 * b + 1));
    }
    block_reduce_multi<2>(t, 0u, shm, red);
    if (threadIdx.x == 0) {
        sc->div_residual = red[0];
        sc->div_scale = red[1] > 0.0 ? red[1] : 1.0;
        *counter = 0;
    }
}

#define MPM2P_FINE_WIDTHS(X) X(4) X(8) X(10) X(12) X(16) X(20) X(24) X(32)

template <int B>
void fine_launch(Ctx& c, const FineArgs& fa) {
    const Layout& L = c.L;
    {
        PROF(c, "k_fine_factor");
        launch_k(c, k_fine_factor<B>, cdiv(L.n_sub, FWPB), FWPB * 32, 0, L, c.f_BD.p, c.f_BW.p, c.f_BS.p, c.f_D.p,
                 c.f_Lc.p, c.f_Lr.p, c.f_y.p, c.sc.p);
        CK_LAUNCH();
    }
    if (c.f_cr) {  // block-tridiagonal coarse operator, cyclic reduction
        const CrView v = cr_view(c.f_cr_plan);
        cr_zero(c, c.f_cr_plan);
        {
            PROF(c, "k_fine_coarse");
            launch_k(c, k_fine_coarse_cr, cdiv((long long)L.nsy * v.S * 32, TPB), TPB, 0, L, c.f_anchor, c.f_T.p,
                     c.f_BD.p, c.f_BW.p, c.f_BS.p, v.S, v.D, v.Up0);
            CK_LAUNCH();
        }
        cr_factor(c, c.f_cr_plan, ERR_FINE_NOCONV);  // a zero coarse pivot: the solve cannot proceed
    } else {
        {
            PROF(c, "k_fine_coarse");
            CK(cudaMemsetAsync(c.f_A0.p, 0, (size_t)L.n_sub * L.n_sub * sizeof(double), c.st));
            launch_k(c, k_fine_coarse, cdiv((long long)L.n_sub * 32, TPB), TPB, 0, L, c.f_anchor, c.f_T.p, c.f_BD.p,
                     c.f_BW.p, c.f_BS.p, c.f_A0.p);
            CK_LAUNCH();
        }
        CK(cudaMemcpyAsync(c.f_A0i.p, c.f_A0.p, (size_t)L.n_sub * L.n_sub * sizeof(double), cudaMemcpyDeviceToDevice,
                           c.st));
        block_gj_inplace_pub(c, c.f_A0i.p, L.n_sub);  // SPD: pivot-free blocked Gauss-Jordan
    }
    static DeviceCache per_sm;  // one per instantiation B, per device
    int occ = per_sm.at().load();
    if (occ < 0) {
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fine_pcg<B>, FWPB * 32, 0));
        per_sm.at().store(occ);
    }
    if (occ < 1) throw CudaError("fine solve: the PCG kernel does not fit on an SM");
    const int blocks = std::max(1, std::min(occ * c.num_sms, cdiv(L.n_sub, FWPB)));
    FineArgs a = fa;
    void* args[] = {&a};
    {
        PROF(c, "k_fine_pcg");
        CK(cudaLaunchCooperativeKernel((void*)k_fine_pcg<B>, blocks, FWPB * 32, args, 0, c.st));
        CK_LAUNCH();
    }
}

}  // namespace

void fine_setup(Ctx& c) {
    const Layout& L = c.L;
    if (c.f_ready) return;
    // the dense coarse inverse up to 4,096 subdomains, cyclic reduction above
    c.f_cr = L.n_sub > 4096;
    if (const char* e = std::getenv("MPM2P_FINE_COARSE")) {
        if (std::strcmp(e, "cr") == 0) c.f_cr = true;
        else if (std::strcmp(e, "dense") == 0) c.f_cr = false;
    }
    switch (L.snx) {
#define X(BW_) \
    case BW_:  \
        break;
        MPM2P_FINE_WIDTHS(X)
#undef X
        default:
            throw CapacityError("fine solve: subdomain width " + std::to_string(L.snx) + " has no PCG kernel instantiation (supported: 4, 8, 10, 12, 16, 20, 24, 32)");
    }
    const size_t nc = L.cells(), nb = (size_t)L.n_sub * L.ncs, ns = L.n_sub;
    c.f_T.alloc(L.faces());
    c.f_BD.alloc(nb);
    c.f_BW.alloc(nb);
    c.f_BS.alloc(nb);
    c.f_D.alloc(nb);
    c.f_Lc.alloc(nb * L.snx);
    c.f_Lr.alloc(nb * L.snx);
    c.f_b.alloc(nb);
    c.f_x.alloc(nb);
    c.f_r.alloc(nb);
    c.f_p.alloc(nb);
    c.f_q.alloc(nb);
    c.f_y.alloc(nb);
    if (c.f_cr) {
        const int S = (L.nsx + 63) / 64 * 64;
        c.f_cy.alloc((size_t)L.nsy * S);
        c.f_cx.alloc((size_t)L.nsy * S);
        c.f_cy.zero(c.st);
        c.f_cx.zero(c.st);
        c.f_cr_plan = cr_create(c, L.nsy, S, c.f_cy.p, c.f_cx.p);
    } else {
        c.f_A0.alloc(ns * ns);
        c.f_A0i.alloc(ns * ns);
    }
    c.f_c0.alloc(ns);
    c.f_e.alloc(ns);
    c.f_part.alloc(4 * ns);
    (void)nc;
    // pure Neumann (every physical face Flux) -> anchor cell 0 (simulation.cpp:130-131)
    bool neumann = true;
    for (int k : c.bc_kind_h)
        if (k != BC_FLUX) neumann = false;
    c.f_anchor = neumann ? 0 : -1;
    if (const char* e = std::getenv("MPM2P_FINE_TOL")) c.f_tol = std::atof(e);
    c.f_warm = false;
    c.f_ready = true;
}

// One fine-reference solve with conductivity kappa (device, cells): p (cells)
// and u (faces) in the global layouts; the previous solution of this context
// is the warm start unless cold.
void fine_solve(Ctx& c, const double* kappa, double* p, double* u, bool cold) {
    fine_setup(c);
    const Layout& L = c.L;
    if (cold || !c.f_warm) CK(cudaMemsetAsync(c.f_x.p, 0, c.f_x.n * sizeof(double), c.st));
    {
        PROF(c, "k_fine_assemble");
        launch_k(c, k_fine_assemble, std::max(1, cdiv(L.cells(), TPB)), TPB, 0, L, c.f_anchor, kappa, c.q.p, c.bc_kind.p,
                 c.bc_value.p, c.f_T.p, c.f_BD.p, c.f_BW.p, c.f_BS.p, c.f_b.p, c.sc.p);
        CK_LAUNCH();
    }
    FineArgs fa{L, c.f_anchor, c.f_T.p, c.f_BD.p, c.f_D.p, c.f_Lc.p, c.f_Lr.p, c.f_A0i.p, c.f_b.p, c.f_x.p,
                c.f_r.p, c.f_p.p, c.f_q.p, c.f_y.p, c.f_c0.p, c.f_e.p, c.f_part.p, c.f_tol,
                std::max(1000, std::min(4 * L.n_sub, 20000)), c.sc.p, nullptr, nullptr, 0, 0, nullptr, nullptr};
    if (c.f_cr) {
        const CrView v = cr_view(c.f_cr_plan);
        fa.cr_jobs = static_cast<const GemvJob*>(v.jobs);
        fa.cr_phases = v.phases;
        fa.cr_nphase = v.nphase;
        fa.cr_S = v.S;
        fa.cy = c.f_cy.p;
        fa.cx = c.f_cx.p;
    }
    switch (L.snx) {
#define X(BW_)                  \
    case BW_:                   \
        fine_launch<BW_>(c, fa); \
        break;
        MPM2P_FINE_WIDTHS(X)
#undef X
        default:
            throw CapacityError("fine solve: subdomain width has no PCG kernel instantiation");
    }
    {
        PROF(c, "k_fine_velocity");
        launch_k(c, k_fine_velocity, red_blocks(c, k_fine_velocity, L.cells()), TPB, 0, L, c.f_T.p, c.bc_kind.p,
                 c.bc_value.p, c.q.p, c.f_x.p, p, u, c.sc.p, c.red.p, c.red_count.p);
        CK_LAUNCH();
    }
    c.f_warm = true;
    c.c_fine += 1;
}

}  // namespace mpm2p
