// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see mrcm_oracle.hpp).
// Restatement of the reference path; each block cites the reference lines it
// follows (paths relative to /root/reference/proj). Floating-point expressions
// keep the reference's operation order where it fixes bits (transport,
// transmissibility); build with -ffp-contract=off like the reference's
// default (no -march) Release build.
#include "mrcm_oracle.hpp"

#include <algorithm>
#include <atomic>
#include <exception>
#include <mutex>
#include <optional>
#include <thread>
#include <chrono>
#include <cstdio>
#include <fstream>
#include <random>

namespace orc {

// ----------------------------------------------------------------- grid ----
Grid build_grid(int nx, int ny, Real lx, Real ly) {  // grid.cpp:9-15
    if (nx < 1 || ny < 1)
        throw ConfigError("build_grid: cell counts must be >= 1, got " + std::to_string(nx) + "x" +
                          std::to_string(ny));
    if (!(lx > 0.0) || !(ly > 0.0)) throw ConfigError("build_grid: domain lengths must be positive");
    return Grid(nx, ny, lx, ly);
}

Vec divergence(const Grid& g, const Vec& u) {  // grid.cpp:19-31
    Vec d(g.cells());
    const Real vol = g.vol();
    for (int j = 0; j < g.ny; ++j)
        for (int i = 0; i < g.nx; ++i) {
            const Real fx = (u[g.vface(i + 1, j)] - u[g.vface(i, j)]) * g.hy;
            const Real fy = (u[g.hface(i, j + 1)] - u[g.hface(i, j)]) * g.hx;
            d[g.cell(i, j)] = (fx + fy) / vol;
        }
    return d;
}

// -------------------------------------------------------- decomposition ----
int Decomp::skeleton_edges() const {  // decomposition.cpp:9-13
    int n = 0;
    for (const auto& f : ifaces) n += (int)f.faces.size();
    return n;
}
Real Decomp::coarse_h() const {  // decomposition.cpp:15-19
    const Real hxs = grid.lx / nsx, hys = grid.ly / nsy;
    return hxs > hys ? hxs : hys;
}
Vec Decomp::restrict_cells(const Vec& global, int s) const {  // decomposition.cpp:21-28
    const Rect& r = subs[s];
    Vec out((size_t)r.nx * r.ny);
    for (int jj = 0; jj < r.ny; ++jj)
        for (int ii = 0; ii < r.nx; ++ii) out[jj * r.nx + ii] = global[grid.cell(r.i0 + ii, r.j0 + jj)];
    return out;
}

Decomp build_decomposition(const Grid& g, int nsx, int nsy) {  // decomposition.cpp:35-132
    if (nsx < 1 || nsy < 1) throw ConfigError("build_decomposition: subdomain counts must be >= 1");
    if (g.nx % nsx != 0 || g.ny % nsy != 0)
        throw ConfigError("build_decomposition: subdomains do not divide the grid");
    Decomp dd;
    dd.grid = g;
    dd.nsx = nsx;
    dd.nsy = nsy;
    const int snx = g.nx / nsx, sny = g.ny / nsy;
    for (int sy = 0; sy < nsy; ++sy)
        for (int sx = 0; sx < nsx; ++sx) {
            dd.subs.push_back({sx * snx, sy * sny, snx, sny});
            dd.subgrids.emplace_back(snx, sny, snx * g.hx, sny * g.hy);
        }
    auto sid = [&](int sx, int sy) { return sy * nsx + sx; };
    for (int sy = 0; sy < nsy; ++sy)  // vertical interfaces, edges by j (:62-74)
        for (int sx = 0; sx + 1 < nsx; ++sx) {
            Interface f;
            f.minus = sid(sx, sy);
            f.plus = sid(sx + 1, sy);
            f.vertical = true;
            const int iface = (sx + 1) * snx;
            for (int j = sy * sny; j < (sy + 1) * sny; ++j) f.faces.push_back(g.vface(iface, j));
            dd.ifaces.push_back(std::move(f));
        }
    for (int sy = 0; sy + 1 < nsy; ++sy)  // horizontal interfaces, edges by i (:75-87)
        for (int sx = 0; sx < nsx; ++sx) {
            Interface f;
            f.minus = sid(sx, sy);
            f.plus = sid(sx, sy + 1);
            f.vertical = false;
            const int jface = (sy + 1) * sny;
            for (int i = sx * snx; i < (sx + 1) * snx; ++i) f.faces.push_back(g.hface(i, jface));
            dd.ifaces.push_back(std::move(f));
        }
    std::vector<int> fi(g.faces(), -1), fp(g.faces(), -1);  // :91-99
    for (int k = 0; k < dd.n_iface(); ++k)
        for (int e = 0; e < (int)dd.ifaces[k].faces.size(); ++e) {
            fi[dd.ifaces[k].faces[e]] = k;
            fp[dd.ifaces[k].faces[e]] = e;
        }
    dd.sub_boundary.resize(dd.subs.size());
    for (size_t s = 0; s < dd.subs.size(); ++s) {  // :101-129
        const Rect& r = dd.subs[s];
        const Grid& lg = dd.subgrids[s];
        auto& edges = dd.sub_boundary[s];
        auto add = [&](int side, int gf, int lf, int lc) {
            BoundaryEdge e;
            e.global_face = gf;
            e.local_face = lf;
            e.local_cell = lc;
            e.side = side;
            e.sign = side_sign(side);
            e.iface = fi[gf];
            e.pos = fp[gf];
            e.on_skeleton = e.iface >= 0;
            edges.push_back(e);
        };
        for (int jj = 0; jj < r.ny; ++jj) add(West, g.vface(r.i0, r.j0 + jj), lg.vface(0, jj), lg.cell(0, jj));
        for (int jj = 0; jj < r.ny; ++jj)
            add(East, g.vface(r.i0 + r.nx, r.j0 + jj), lg.vface(r.nx, jj), lg.cell(r.nx - 1, jj));
        for (int ii = 0; ii < r.nx; ++ii) add(South, g.hface(r.i0 + ii, r.j0), lg.hface(ii, 0), lg.cell(ii, 0));
        for (int ii = 0; ii < r.nx; ++ii)
            add(North, g.hface(r.i0 + ii, r.j0 + r.ny), lg.hface(ii, r.ny), lg.cell(ii, r.ny - 1));
    }
    return dd;
}

// ------------------------------------------------------------- elliptic ----
namespace {
// elliptic.cpp:13-22 — boundary faces in BoundarySpec order.
template <typename F>
void for_each_boundary_face(const Grid& g, F&& fn) {
    for (int j = 0; j < g.ny; ++j) fn(j, -1.0, g.cell(0, j), g.vface(0, j));
    for (int j = 0; j < g.ny; ++j) fn(g.ny + j, +1.0, g.cell(g.nx - 1, j), g.vface(g.nx, j));
    for (int i = 0; i < g.nx; ++i) fn(2 * g.ny + i, -1.0, g.cell(i, 0), g.hface(i, 0));
    for (int i = 0; i < g.nx; ++i) fn(2 * g.ny + g.nx + i, +1.0, g.cell(i, g.ny - 1), g.hface(i, g.ny));
}
Real eff_robin(Real t_half, Real beta, Real area) {  // elliptic.cpp:24-26
    return 1.0 / (1.0 / t_half + beta / area);
}
}  // namespace

Vec transmissibility(const Grid& g, const Vec& k) {  // elliptic.cpp:44-61
    Vec t(g.faces());
    auto harm = [](Real a, Real b) { return 2.0 * a * b / (a + b); };
    auto K = [&](int i, int j) { return k[g.cell(i, j)]; };
    for (int j = 0; j < g.ny; ++j) {
        t[g.vface(0, j)] = K(0, j) * g.hy / (g.hx / 2.0);
        t[g.vface(g.nx, j)] = K(g.nx - 1, j) * g.hy / (g.hx / 2.0);
        for (int i = 1; i < g.nx; ++i) t[g.vface(i, j)] = harm(K(i - 1, j), K(i, j)) * g.hy / g.hx;
    }
    for (int i = 0; i < g.nx; ++i) {
        t[g.hface(i, 0)] = K(i, 0) * g.hx / (g.hy / 2.0);
        t[g.hface(i, g.ny)] = K(i, g.ny - 1) * g.hx / (g.hy / 2.0);
        for (int j = 1; j < g.ny; ++j) t[g.hface(i, j)] = harm(K(i, j - 1), K(i, j)) * g.hx / g.hy;
    }
    return t;
}

// Elimination order of every banded solve: 0 natural, 1 reversed. Reversing
// is an equally exact direct method with different rounding; tests use it to
// measure the solver-roundoff floor the reference's own answer carries.
static int g_elim_order = 0;
void set_elimination_order(int order) { g_elim_order = order; }

void BandLDLT::factor(const Vec& band_in) {
    rev = g_elim_order == 1;
    Vec rb;
    if (rev) {  // A'[r'][c'] = A[n-1-r'][n-1-c'] = A[n-1-c'][n-1-r'] (symmetric)
        rb.assign(band_in.size(), 0.0);
        for (int r2 = 0; r2 < n; ++r2)
            for (int c2 = std::max(0, r2 - w); c2 <= r2; ++c2) {
                const int R = n - 1 - c2, Cc = n - 1 - r2;
                rb[(size_t)r2 * (w + 1) + (c2 - r2 + w)] = band_in[(size_t)R * (w + 1) + (Cc - R + w)];
            }
    }
    const Vec& band = rev ? rb : band_in;
    // Left-looking banded LDL^T: L[r][c] = (A[r][c] - sum_m L[r][m] D[m] L[c][m]) / D[c].
    L.assign((size_t)n * std::max(w, 1), 0.0);
    D.assign(n, 0.0);
    auto Lr = [&](int r, int c) -> Real& { return L[(size_t)r * w + (c - r + w)]; };
    for (int r = 0; r < n; ++r) {
        const int c0 = std::max(0, r - w);
        for (int c = c0; c < r; ++c) {
            Real s = band[(size_t)r * (w + 1) + (c - r + w)];
            const int m0 = std::max(c0, c - w);
            for (int m = m0; m < c; ++m) s -= Lr(r, m) * D[m] * L[(size_t)c * w + (m - c + w)];
            Lr(r, c) = s / D[c];
        }
        Real d = band[(size_t)r * (w + 1) + w];
        for (int m = c0; m < r; ++m) d -= Lr(r, m) * Lr(r, m) * D[m];
        if (!(d > 0.0) || !std::isfinite(d)) throw NumericError("CellCenteredSolver: direct solve failed");
        D[r] = d;
    }
}

void BandLDLT::solve(Vec& x) const {
    if (rev) std::reverse(x.begin(), x.end());
    solve_natural(x);
    if (rev) std::reverse(x.begin(), x.end());
}

void BandLDLT::solve_natural(Vec& x) const {
    for (int r = 0; r < n; ++r) {
        Real s = x[r];
        for (int c = std::max(0, r - w); c < r; ++c) s -= L[(size_t)r * w + (c - r + w)] * x[c];
        x[r] = s;
    }
    for (int r = 0; r < n; ++r) x[r] /= D[r];
    for (int r = n - 1; r >= 0; --r) {
        const Real xr = x[r];
        for (int c = std::max(0, r - w); c < r; ++c) x[c] -= L[(size_t)r * w + (c - r + w)] * xr;
    }
}

void LocalSolver::factorize(const Vec& kappa, const BoundarySpec& bc, int anchor) {  // elliptic.cpp:68-150
    const Grid& g = g_;
    if (bc.nx != g.nx || bc.ny != g.ny) throw ConfigError("CellCenteredSolver: boundary spec does not match grid");
    for (Real k : kappa)
        if (!(k > 0.0) || !std::isfinite(k))
            throw NumericError("CellCenteredSolver: conductivity must be positive and finite");
    if (bc.pure_neumann() && anchor < 0)
        throw NumericError("CellCenteredSolver: pure-Neumann problem requires an anchor cell");
    trans_ = transmissibility(g, kappa);
    bc_struct_ = bc;
    anchor_ = anchor;
    const int n = g.cells(), w = g.nx;
    Vec band((size_t)n * (w + 1), 0.0);
    auto add = [&](int r, int c, Real v) {  // lower triangle only (symmetric)
        if (c > r) return;
        if (r == anchor || c == anchor) v = 0.0;
        band[(size_t)r * (w + 1) + (c - r + w)] += v;
    };
    for (int j = 0; j < g.ny; ++j)
        for (int i = 0; i < g.nx; ++i) {
            const int c = g.cell(i, j);
            Real diag = 0.0;
            if (i > 0) { const Real t = trans_[g.vface(i, j)]; diag += t; add(c, g.cell(i - 1, j), -t); }
            if (i < g.nx - 1) { const Real t = trans_[g.vface(i + 1, j)]; diag += t; }
            if (j > 0) { const Real t = trans_[g.hface(i, j)]; diag += t; add(c, g.cell(i, j - 1), -t); }
            if (j < g.ny - 1) { const Real t = trans_[g.hface(i, j + 1)]; diag += t; }
            add(c, c, diag);
        }
    for_each_boundary_face(g, [&](int b, Real, int c, int f) {  // :123-139
        const FaceBc& fb = bc.faces[b];
        const Real area = g.area(f), th = trans_[f];
        if (fb.kind == Pressure) add(c, c, th);
        else if (fb.kind == Robin) {
            if (!(fb.beta > 0.0)) throw ConfigError("CellCenteredSolver: Robin face requires beta > 0");
            add(c, c, eff_robin(th, fb.beta, area));
        }
    });
    if (anchor >= 0) band[(size_t)anchor * (w + 1) + w] = 1.0;  // :141
    ldlt_.n = n;
    ldlt_.w = w;
    ldlt_.factor(band);
}

LocalSolution LocalSolver::solve(const Vec& q, const BoundarySpec& bc) const {  // elliptic.cpp:152-243
    const Grid& g = g_;
    if (bc.count() != bc_struct_.count())
        throw NumericError("CellCenteredSolver: boundary spec does not match the factorization");
    for (int i = 0; i < bc.count(); ++i)
        if (bc.faces[i].kind != bc_struct_.faces[i].kind || bc.faces[i].beta != bc_struct_.faces[i].beta)
            throw NumericError("CellCenteredSolver: boundary structure changed since factorization");
    const Real vol = g.vol();
    Vec x(g.cells());
    for (int c = 0; c < g.cells(); ++c) x[c] = q[c] * vol;
    for_each_boundary_face(g, [&](int b, Real, int c, int f) {
        const FaceBc& fb = bc.faces[b];
        const Real area = g.area(f), th = trans_[f];
        if (fb.kind == Pressure) x[c] += th * fb.value;
        else if (fb.kind == Flux) x[c] -= fb.value * area;
        else x[c] += eff_robin(th, fb.beta, area) * fb.robin_rhs;
    });
    if (anchor_ >= 0) x[anchor_] = 0.0;
    ldlt_.solve(x);
    LocalSolution sol;
    sol.p = x;
    sol.u.assign(g.faces(), 0.0);
    sol.boundary_p.assign(bc.count(), 0.0);
    for (int j = 0; j < g.ny; ++j)
        for (int i = 1; i < g.nx; ++i) {
            const int f = g.vface(i, j);
            sol.u[f] = trans_[f] * (x[g.cell(i - 1, j)] - x[g.cell(i, j)]) / g.area(f);
        }
    for (int i = 0; i < g.nx; ++i)
        for (int j = 1; j < g.ny; ++j) {
            const int f = g.hface(i, j);
            sol.u[f] = trans_[f] * (x[g.cell(i, j - 1)] - x[g.cell(i, j)]) / g.area(f);
        }
    for_each_boundary_face(g, [&](int b, Real sgn, int c, int f) {
        const FaceBc& fb = bc.faces[b];
        const Real area = g.area(f), th = trans_[f];
        Real un = 0.0, pf = 0.0;
        if (fb.kind == Pressure) {
            un = th * (x[c] - fb.value) / area;
            pf = fb.value;
        } else if (fb.kind == Flux) {
            un = fb.value;
            pf = x[c] - fb.value * area / th;
        } else {
            const Real te = eff_robin(th, fb.beta, area);
            un = te * (x[c] - fb.robin_rhs) / area;
            pf = fb.robin_rhs + fb.beta * un;
        }
        sol.u[f] = sgn * un;
        sol.boundary_p[b] = pf;
    });
    return sol;
}

LocalSolution solve_cell_centered(const Grid& g, const Vec& kappa, const Vec& q, const BoundarySpec& bc,
                                  int anchor) {  // elliptic.cpp:245-250
    LocalSolver s(g);
    s.factorize(kappa, bc, anchor);
    return s.solve(q, bc);
}

Real conservation_residual(const Grid& g, const LocalSolution& sol, const Vec& q) {  // :252-257
    const Vec d = divergence(g, sol.u);
    Real r = 0.0;
    for (int c = 0; c < g.cells(); ++c) r = std::max(r, std::abs(d[c] - q[c]));
    return r;
}

Real residual_scale(const Grid& g, const LocalSolution& sol, const Vec& q) {  // :259-267
    Real s = 0.0;
    for (Real v : q) s = std::max(s, std::abs(v));
    const Real vol = g.vol();
    for (int f = 0; f < g.faces(); ++f) s = std::max(s, std::abs(sol.u[f]) * g.area(f) / vol);
    return s > 0.0 ? s : 1.0;
}

// ------------------------------------------------------ interface space ----
Space build_interface_space(const Decomp& dd, int kind, HbarSpec hbar) {  // interface_space.cpp:9-52
    Space sp;
    sp.kind = kind;
    const int ni = dd.n_iface();
    sp.flux_by_iface.resize(ni);
    sp.pres_by_iface.resize(ni);
    auto push = [&](int k, Vec vals) {
        sp.flux_by_iface[k].push_back(sp.dim_flux());
        sp.flux.push_back({k, vals});
        sp.pres_by_iface[k].push_back(sp.dim_pres());
        sp.pres.push_back({k, std::move(vals)});
    };
    for (int k = 0; k < ni; ++k) {
        const int n = (int)dd.ifaces[k].faces.size();
        if (kind == 1) {
            push(k, Vec(n, 1.0));
            Vec lin(n);
            for (int e = 0; e < n; ++e) lin[e] = 2.0 * (e + 0.5) / n - 1.0;
            push(k, std::move(lin));
            continue;
        }
        int seg = n;
        if (hbar.mode == 1) seg = n / 2;
        else if (hbar.mode == 2) seg = 1;
        else if (hbar.mode == 3) seg = hbar.edges;
        if (seg < 1 || n % seg != 0)
            throw ConfigError("build_interface_space: segment length " + std::to_string(seg) +
                              " does not divide interface " + std::to_string(k));
        for (int st = 0; st < n; st += seg) {
            Vec v(n, 0.0);
            for (int e = st; e < st + seg; ++e) v[e] = 1.0;
            push(k, std::move(v));
        }
    }
    return sp;
}

// ---------------------------------------------------------------- robin ----
namespace {
std::pair<int, int> adjacent_cells(const Grid& g, const Interface& f, int pos) {  // robin.cpp:13-24
    const int fc = f.faces[pos];
    if (f.vertical) {
        const int i = fc % (g.nx + 1), j = fc / (g.nx + 1);
        return {g.cell(i - 1, j), g.cell(i, j)};
    }
    const int fh = fc - g.vcount();
    const int i = fh % g.nx, j = fh / g.nx;
    return {g.cell(i, j - 1), g.cell(i, j)};
}
Real quantile(const Vec& v, Real pct) {  // robin.cpp:26-35
    const size_t m = v.size();
    if (m == 0) return 0.0;
    Real idx = pct / 100.0 * (Real)(m - 1);
    idx = std::clamp<Real>(idx, 0.0, (Real)(m - 1));
    const size_t lo = (size_t)idx;
    const size_t hi = std::min(lo + 1, m - 1);
    const Real w = idx - (Real)lo;
    return (1.0 - w) * v[lo] + w * v[hi];
}
}  // namespace

RobinParameter compute_beta(const Vec& kappa, const Decomp& dd, const AlphaSpec& spec) {  // robin.cpp:39-92
    for (Real k : kappa) if (!(k > 0.0)) throw NumericError("compute_beta: conductivity must be positive");
    const Real H = dd.coarse_h();
    const int ni = dd.n_iface();
    RobinParameter rp;
    rp.beta_minus.resize(ni);
    rp.beta_plus.resize(ni);
    rp.alpha.resize(ni);
    std::vector<Vec> fk(ni);
    Vec all;
    for (int k = 0; k < ni; ++k) {
        const Interface& f = dd.ifaces[k];
        fk[k].resize(f.faces.size());
        for (int e = 0; e < (int)f.faces.size(); ++e) {
            auto [cm, cp] = adjacent_cells(dd.grid, f, e);
            const Real hm = 2.0 * kappa[cm] * kappa[cp] / (kappa[cm] + kappa[cp]);
            fk[k][e] = hm;
            all.push_back(hm);
        }
    }
    Real qlo = 0.0, qhi = 0.0;
    if (spec.mode == 1 && !all.empty()) {
        std::sort(all.begin(), all.end());
        qlo = quantile(all, spec.pct_lo);
        qhi = quantile(all, spec.pct_hi);
    }
    for (int k = 0; k < ni; ++k) {
        const Interface& f = dd.ifaces[k];
        const int n = (int)f.faces.size();
        rp.beta_minus[k].resize(n);
        rp.beta_plus[k].resize(n);
        rp.alpha[k].resize(n);
        for (int e = 0; e < n; ++e) {
            Real a = spec.alpha;
            if (spec.mode == 1) {
                const Real v = fk[k][e];
                a = v > qhi ? spec.alpha_min : (v < qlo ? spec.alpha_max : 1.0);
            }
            auto [cm, cp] = adjacent_cells(dd.grid, f, e);
            rp.alpha[k][e] = a;
            rp.beta_minus[k][e] = a * H / kappa[cm];
            rp.beta_plus[k][e] = a * H / kappa[cp];
        }
    }
    return rp;
}

// ------------------------------------------------------------- dense LU ----
void DenseLU::compute(const Vec& M, int n_) {
    n = n_;
    A = M;
    perm.resize(n);
    for (int i = 0; i < n; ++i) perm[i] = i;
    for (int k = 0; k < n; ++k) {
        int piv = k;
        Real best = std::abs(A[(size_t)k * n + k]);
        for (int i = k + 1; i < n; ++i) {
            const Real v = std::abs(A[(size_t)i * n + k]);
            if (v > best) { best = v; piv = i; }
        }
        if (piv != k) {
            for (int j = 0; j < n; ++j) std::swap(A[(size_t)k * n + j], A[(size_t)piv * n + j]);
            std::swap(perm[k], perm[piv]);
        }
        const Real d = A[(size_t)k * n + k];
        if (d == 0.0) continue;  // singular: rcond() reports it
        for (int i = k + 1; i < n; ++i) {
            Real* ri = &A[(size_t)i * n];
            const Real l = ri[k] / d;
            ri[k] = l;
            if (l == 0.0) continue;
            const Real* rk = &A[(size_t)k * n];
            for (int j = k + 1; j < n; ++j) ri[j] -= l * rk[j];
        }
    }
}

Vec DenseLU::solve(const Vec& b) const {
    Vec x(n);
    for (int i = 0; i < n; ++i) x[i] = b[perm[i]];
    for (int i = 0; i < n; ++i) {
        Real s = x[i];
        const Real* ri = &A[(size_t)i * n];
        for (int j = 0; j < i; ++j) s -= ri[j] * x[j];
        x[i] = s;
    }
    for (int i = n - 1; i >= 0; --i) {
        Real s = x[i];
        const Real* ri = &A[(size_t)i * n];
        for (int j = i + 1; j < n; ++j) s -= ri[j] * x[j];
        x[i] = s / ri[i];
    }
    return x;
}

Vec DenseLU::solve_transposed(const Vec& b) const {  // A^T x = b with PA = LU
    Vec y = b;
    for (int i = 0; i < n; ++i) {  // U^T y = b
        Real s = y[i];
        for (int j = 0; j < i; ++j) s -= A[(size_t)j * n + i] * y[j];
        y[i] = s / A[(size_t)i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {  // L^T z = y
        Real s = y[i];
        for (int j = i + 1; j < n; ++j) s -= A[(size_t)j * n + i] * y[j];
        y[i] = s;
    }
    Vec x(n);
    for (int i = 0; i < n; ++i) x[perm[i]] = y[i];
    return x;
}

namespace {
// 1-norm reciprocal condition estimate (Hager 1984 / Higham 1988), the
// quantity Eigen's PartialPivLU::rcond() estimates.
template <class S, class ST>
Real hager_rcond(int n, Real anorm, S&& solve, ST&& solve_t) {
    Vec x(n, 1.0 / n);
    Real est = 0.0;
    for (int it = 0; it < 5; ++it) {
        Vec y = solve(x);
        Real ny = 0.0;
        for (Real v : y) ny += std::abs(v);
        if (!std::isfinite(ny)) return 0.0;
        if (it > 0 && ny <= est) break;
        est = ny;
        Vec xi(n);
        for (int i = 0; i < n; ++i) xi[i] = y[i] >= 0 ? 1.0 : -1.0;
        Vec z = solve_t(xi);
        int jm = 0;
        Real zm = -1.0, ztx = 0.0;
        for (int i = 0; i < n; ++i) {
            ztx += z[i] * x[i];
            if (std::abs(z[i]) > zm) { zm = std::abs(z[i]); jm = i; }
        }
        if (zm <= ztx) break;
        std::fill(x.begin(), x.end(), 0.0);
        x[jm] = 1.0;
    }
    if (!(est > 0.0) || !(anorm > 0.0)) return 0.0;
    return 1.0 / anorm / est;
}
}  // namespace

Real DenseLU::rcond(const Vec& M) const {
    if (n == 0) return 1.0;
    for (int i = 0; i < n; ++i) {
        const Real d = A[(size_t)i * n + i];
        if (d == 0.0 || !std::isfinite(d)) return 0.0;
    }
    Real anorm = 0.0;
    for (int j = 0; j < n; ++j) {
        Real s = 0.0;
        for (int i = 0; i < n; ++i) s += std::abs(M[(size_t)i * n + j]);
        anorm = std::max(anorm, s);
    }
    return hager_rcond(n, anorm, [&](const Vec& b) { return solve(b); },
                       [&](const Vec& b) { return solve_transposed(b); });
}

// ------------------------------------------------------------- banded LU ----
void BandLU::init(int n_, std::vector<int> prow_, std::vector<int> pcol_, int kl_, int ku_) {
    n = n_;
    kl = kl_;
    ku = ku_;
    ld = 2 * kl + ku + 1;
    prow = std::move(prow_);
    pcol = std::move(pcol_);
    AB.assign((size_t)n * ld, 0.0);
    ipiv.assign(n, 0);
    singular = false;
}

void BandLU::factor() {  // dgbtf2: partial pivoting, fill into kl extra super-diagonals
    int ju = 0;
    for (int j = 0; j < n; ++j) {
        const int km = std::min(kl, n - 1 - j);
        int jp = 0;
        Real best = std::abs(get(j, j));
        for (int i = 1; i <= km; ++i) {
            const Real v = std::abs(get(j + i, j));
            if (v > best) { best = v; jp = i; }
        }
        ipiv[j] = j + jp;
        if (get(j + jp, j) == 0.0) { singular = true; continue; }
        ju = std::max(ju, std::min(j + ku + jp, n - 1));
        if (jp != 0)
            for (int c = j; c <= ju; ++c) std::swap(at(j, c), at(j + jp, c));
        const Real d = get(j, j);
        Real* colj = &AB[(size_t)j * ld + kl + ku];  // colj[i] = A'(j + i, j)
        for (int i = 1; i <= km; ++i) colj[i] /= d;
        for (int c = j + 1; c <= ju; ++c) {
            Real* colc = &AB[(size_t)c * ld + kl + ku + j - c];  // colc[i] = A'(j + i, c)
            const Real a = colc[0];
            if (a == 0.0) continue;
            for (int i = 1; i <= km; ++i) colc[i] -= colj[i] * a;
        }
    }
}

Vec BandLU::solve(const Vec& b) const {
    Vec y(n);
    for (int i = 0; i < n; ++i) y[i] = b[prow[i]];
    for (int j = 0; j < n; ++j) {  // L: row swaps and unit lower columns
        const int km = std::min(kl, n - 1 - j);
        if (ipiv[j] != j) std::swap(y[j], y[ipiv[j]]);
        const Real yj = y[j];
        if (yj == 0.0) continue;
        const Real* colj = &AB[(size_t)j * ld + kl + ku];
        for (int i = 1; i <= km; ++i) y[j + i] -= colj[i] * yj;
    }
    const int w = kl + ku;
    for (int j = n - 1; j >= 0; --j) {  // U: upper band of width kl + ku
        y[j] /= get(j, j);
        const Real yj = y[j];
        if (yj == 0.0) continue;
        for (int i = std::max(0, j - w); i < j; ++i) y[i] -= get(i, j) * yj;
    }
    Vec x(n);
    for (int j = 0; j < n; ++j) x[pcol[j]] = y[j];
    return x;
}

Vec BandLU::solve_transposed(const Vec& b) const {  // A'^T y = b', x = P_row^T y
    Vec y(n);
    for (int j = 0; j < n; ++j) y[j] = b[pcol[j]];
    const int w = kl + ku;
    for (int j = 0; j < n; ++j) {  // U^T
        Real s = y[j];
        for (int i = std::max(0, j - w); i < j; ++i) s -= get(i, j) * y[i];
        y[j] = s / get(j, j);
    }
    for (int j = n - 1; j >= 0; --j) {  // L^T, then the row swaps in reverse
        const int km = std::min(kl, n - 1 - j);
        const Real* colj = &AB[(size_t)j * ld + kl + ku];
        Real s = y[j];
        for (int i = 1; i <= km; ++i) s -= colj[i] * y[j + i];
        y[j] = s;
        if (ipiv[j] != j) std::swap(y[j], y[ipiv[j]]);
    }
    Vec x(n);
    for (int i = 0; i < n; ++i) x[prow[i]] = y[i];
    return x;
}

Real BandLU::rcond(Real anorm) const {
    if (n == 0) return 1.0;
    if (singular) return 0.0;
    for (int j = 0; j < n; ++j)
        if (!std::isfinite(get(j, j))) return 0.0;
    return hager_rcond(n, anorm, [&](const Vec& b) { return solve(b); },
                       [&](const Vec& b) { return solve_transposed(b); });
}

static int g_iface_mode = 0;
void set_interface_solver(int mode) { g_iface_mode = mode; }
int interface_solver_mode() { return g_iface_mode; }
static int g_threads = 1;
void set_threads(int n) { g_threads = std::max(1, n); }

// ----------------------------------------------------------------- mrcm ----
namespace {
// Per-subdomain loops (independent local solves). One thread by default, in
// the reference's order; with set_threads(n > 1) the subdomains run in
// parallel (fixture generation for the large configs; results are identical
// because every subdomain's arithmetic is unchanged).
template <class F>
void for_subdomains(int n, F&& fn) {
    if (g_threads <= 1) {
        for (int s = 0; s < n; ++s) fn(s);
        return;
    }
    std::exception_ptr err;
    std::mutex mu;
    std::atomic<int> next{0};
    auto worker = [&] {
        for (int s; (s = next.fetch_add(1)) < n;) {
            try {
                fn(s);
            } catch (...) {
                std::lock_guard<std::mutex> lk(mu);
                if (!err) err = std::current_exception();
            }
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < g_threads; ++t) pool.emplace_back(worker);
    worker();
    for (auto& t : pool) t.join();
    if (err) std::rethrow_exception(err);
}
}  // namespace
namespace {
int global_bc_index(const Grid& g, int f) {  // mrcm.cpp:14-28
    if (g.is_vface(f)) {
        const int i = f % (g.nx + 1), j = f / (g.nx + 1);
        if (i == 0) return j;
        if (i == g.nx) return g.ny + j;
        return -1;
    }
    const int fh = f - g.vcount();
    const int i = fh % g.nx, j = fh / g.nx;
    if (j == 0) return 2 * g.ny + i;
    if (j == g.ny) return 2 * g.ny + g.nx + i;
    return -1;
}
int local_to_global_face(const Decomp& dd, int s, int lf) {  // mrcm.cpp:30-42
    const Grid& lg = dd.subgrids[s];
    const Rect& r = dd.subs[s];
    if (lf < lg.vcount()) {
        const int i = lf % (lg.nx + 1), j = lf / (lg.nx + 1);
        return dd.grid.vface(r.i0 + i, r.j0 + j);
    }
    const int fh = lf - lg.vcount();
    const int i = fh % lg.nx, j = fh / lg.nx;
    return dd.grid.hface(r.i0 + i, r.j0 + j);
}
struct FaceMap { std::vector<std::vector<int>> minus, plus; };
FaceMap build_face_map(const Decomp& dd) {  // mrcm.cpp:49-67
    FaceMap m;
    m.minus.resize(dd.n_iface());
    m.plus.resize(dd.n_iface());
    for (int k = 0; k < dd.n_iface(); ++k) {
        m.minus[k].assign(dd.ifaces[k].faces.size(), -1);
        m.plus[k].assign(dd.ifaces[k].faces.size(), -1);
    }
    for (int s = 0; s < dd.n_sub(); ++s)
        for (const auto& e : dd.sub_boundary[s]) {
            if (!e.on_skeleton) continue;
            (e.sign > 0 ? m.minus : m.plus)[e.iface][e.pos] = e.local_face;
        }
    return m;
}
Vec assemble_interface_rhs(const BasisSet& b, const std::vector<LocalSolution>& bar) {  // mrcm.cpp:80-100
    const Decomp& dd = *b.dd;
    const Space& sp = *b.space;
    Vec rhs(b.dim(), 0.0);
    for (int s = 0; s < dd.n_sub(); ++s)
        for (const auto& e : dd.sub_boundary[s]) {
            if (!e.on_skeleton) continue;
            const int k = e.iface;
            const Real len = dd.grid.area(e.global_face);
            const Real beta = b.beta.beta(k, e.pos, e.sign > 0);
            const Real un = e.sign * bar[s].u[e.local_face];
            for (int r : sp.pres_by_iface[k]) rhs[r] -= un * sp.pres[r].values[e.pos] * len;
            for (int r : sp.flux_by_iface[k])
                rhs[b.n_pres + r] -= beta * un * sp.flux[r].values[e.pos] * e.sign * len;
        }
    return rhs;
}
}  // namespace

std::vector<LocalData> restrict_physical_data(const Decomp& dd, const RobinParameter& beta, const Vec& q,
                                              const BoundarySpec& bc) {  // mrcm.cpp:104-130
    if (bc.nx != dd.grid.nx || bc.ny != dd.grid.ny)
        throw ConfigError("restrict_physical_data: boundary spec does not match grid");
    std::vector<LocalData> data;
    for (int s = 0; s < dd.n_sub(); ++s) {
        LocalData d{dd.restrict_cells(q, s), BoundarySpec(dd.subs[s].nx, dd.subs[s].ny)};
        const auto& edges = dd.sub_boundary[s];
        for (size_t i = 0; i < edges.size(); ++i) {
            const auto& e = edges[i];
            if (e.on_skeleton) {
                FaceBc fb;
                fb.kind = Robin;
                fb.beta = beta.beta(e.iface, e.pos, e.sign > 0);
                d.bc.faces[i] = fb;
            } else {
                const int gi = global_bc_index(dd.grid, e.global_face);
                if (gi < 0) throw NumericError("restrict_physical_data: inconsistent decomposition");
                d.bc.faces[i] = bc.faces[gi];
            }
        }
        data.push_back(std::move(d));
    }
    return data;
}

namespace {
// The interface matrix entries in the reference's accumulation order
// (mrcm.cpp:196-224): rows [psi-rows | phi-rows], columns [U | P]. `add` is
// called once per contribution; every (r, c) receives its terms in the same
// sequence whichever storage is used.
template <class F>
void assemble_interface_matrix(const BasisSet& b, F&& add) {
    const Decomp& dd = *b.dd;
    const Space& sp = *b.space;
    for (int s = 0; s < dd.n_sub(); ++s)
        for (const auto& e : dd.sub_boundary[s]) {
            if (!e.on_skeleton) continue;
            const int k = e.iface;
            const Real len = dd.grid.area(e.global_face);
            const Real bse = b.beta.beta(k, e.pos, e.sign > 0);
            for (const auto& h : b.subs[s].hom) {
                const Real un = e.sign * h.sol.u[e.local_face];
                for (int r : sp.pres_by_iface[k]) add(r, h.col, un * sp.pres[r].values[e.pos] * len);
                for (int r : sp.flux_by_iface[k])
                    add(b.n_pres + r, h.col, bse * un * sp.flux[r].values[e.pos] * e.sign * len);
            }
            for (int bb : sp.flux_by_iface[k]) {
                const Real ub = sp.flux[bb].values[e.pos];
                for (int r : sp.flux_by_iface[k])
                    add(b.n_pres + r, bb, -(bse * ub * e.sign * sp.flux[r].values[e.pos] * e.sign * len));
            }
        }
}

// Unknowns ordered by interface position in the subdomain grid: the vertical
// interfaces of subdomain row j (west to east), then the horizontal ones
// between rows j and j+1. An interface couples only to interfaces sharing a
// subdomain, so the permuted M is banded with half-bandwidth about one
// subdomain row of interfaces.
void interface_band_order(const BasisSet& b, std::vector<int>& prow, std::vector<int>& pcol) {
    const Decomp& dd = *b.dd;
    const Space& sp = *b.space;
    std::vector<int> ord(dd.n_iface());
    for (int k = 0; k < dd.n_iface(); ++k) ord[k] = k;
    auto key = [&](int k) {
        const Interface& f = dd.ifaces[k];
        const int sx = f.minus % dd.nsx, sy = f.minus / dd.nsx;
        return std::make_pair(2 * sy + (f.vertical ? 0 : 1), sx);
    };
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int c) { return key(a) < key(c); });
    prow.clear();
    pcol.clear();
    for (int k : ord) {
        for (int r : sp.pres_by_iface[k]) prow.push_back(r);
        for (int r : sp.flux_by_iface[k]) prow.push_back(b.n_pres + r);
        for (int c : sp.flux_by_iface[k]) pcol.push_back(c);
        for (int c : sp.pres_by_iface[k]) pcol.push_back(b.n_flux + c);
    }
}
}  // namespace

std::shared_ptr<BasisSet> compute_basis_set(const Vec& kappa, std::shared_ptr<const Decomp> ddp,
                                            std::shared_ptr<const Space> spp, const RobinParameter& beta,
                                            const Vec& q, const BoundarySpec& bc, SolveCounters& cnt) {
    // mrcm.cpp:132-240
    const Decomp& dd = *ddp;
    const Space& sp = *spp;
    auto b = std::make_shared<BasisSet>();
    b->dd = ddp;
    b->space = spp;
    b->beta = beta;
    b->kappa_m = kappa;
    b->n_flux = sp.dim_flux();
    b->n_pres = sp.dim_pres();
    const auto data = restrict_physical_data(dd, beta, q, bc);
    b->particular.resize(dd.n_sub());
    std::vector<std::optional<BasisSet::Sub>> built(dd.n_sub());
    for_subdomains(dd.n_sub(), [&](int s) {
        built[s].emplace(BasisSet::Sub{LocalSolver(dd.subgrids[s]), data[s].bc, {}});
        BasisSet::Sub& mach = *built[s];
        const Vec ks = dd.restrict_cells(kappa, s);
        const int anchor = mach.bc_struct.pure_neumann() ? 0 : -1;
        mach.solver.factorize(ks, mach.bc_struct, anchor);
        std::vector<int> inc;  // :157-162
        for (const auto& e : dd.sub_boundary[s])
            if (e.on_skeleton && std::find(inc.begin(), inc.end(), e.iface) == inc.end()) inc.push_back(e.iface);
        std::sort(inc.begin(), inc.end());
        const Vec zq(dd.subgrids[s].cells(), 0.0);
        BoundarySpec hb = mach.bc_struct;  // :164-167
        for (auto& f : hb.faces) if (f.kind != Robin) f.value = 0.0;
        auto solve_hom = [&](int col, bool fluxb, const InterfaceBasis& ib) {  // :169-183
            for (size_t i = 0; i < dd.sub_boundary[s].size(); ++i) {
                const auto& e = dd.sub_boundary[s][i];
                if (!e.on_skeleton) continue;
                Real r = 0.0;
                if (e.iface == ib.iface) {
                    const Real v = ib.values[e.pos];
                    r = fluxb ? -hb.faces[i].beta * v * e.sign : v;
                }
                hb.faces[i].robin_rhs = r;
            }
            mach.hom.push_back({col, mach.solver.solve(zq, hb)});
        };
        for (int k : inc) for (int bb : sp.flux_by_iface[k]) solve_hom(bb, true, sp.flux[bb]);
        for (int k : inc) for (int bb : sp.pres_by_iface[k]) solve_hom(b->n_flux + bb, false, sp.pres[bb]);
        b->particular[s] = mach.solver.solve(data[s].q, data[s].bc);  // :191-192
    });
    for (int s = 0; s < dd.n_sub(); ++s) {
        cnt.homogeneous += (long)built[s]->hom.size();
        ++cnt.particular;
        b->subs.push_back(std::move(*built[s]));
    }
    const int dim = b->dim();
    Real anorm = 0.0;
    const int mode = interface_solver_mode();
    b->banded = dim > 0 && (mode == 2 || (mode == 0 && dim > kDenseInterfaceMax));
    if (!b->banded) {
        Vec M((size_t)dim * dim, 0.0);
        assemble_interface_matrix(*b, [&](int r, int c, Real v) { M[(size_t)r * dim + c] += v; });
        b->M = M;
        b->lu.compute(M, dim);  // :225-238
        if (dim > 0) {
            const Real rc = b->lu.rcond(M);
            if (!(rc > 1e-14))
                throw NumericError("compute_basis_set: interface matrix is numerically singular (rcond=" +
                                   std::to_string(rc) + ")");
        }
        return b;
    }
    // banded path: the same entries, accumulated in the same order, stored in
    // the permuted band (see BandLU)
    std::vector<int> prow, pcol;
    interface_band_order(*b, prow, pcol);
    std::vector<int> rpos(dim), cpos(dim);
    for (int i = 0; i < dim; ++i) { rpos[prow[i]] = i; cpos[pcol[i]] = i; }
    int kl = 0, ku = 0;
    assemble_interface_matrix(*b, [&](int r, int c, Real) {
        kl = std::max(kl, rpos[r] - cpos[c]);
        ku = std::max(ku, cpos[c] - rpos[r]);
    });
    b->blu.init(dim, prow, pcol, kl, ku);
    assemble_interface_matrix(*b, [&](int r, int c, Real v) { b->blu.at(rpos[r], cpos[c]) += v; });
    {  // 1-norm of M (column sums of the assembled entries)
        for (int j = 0; j < dim; ++j) {
            Real s = 0.0;
            for (int i = std::max(0, j - ku); i <= std::min(dim - 1, j + kl); ++i) s += std::abs(b->blu.get(i, j));
            anorm = std::max(anorm, s);
        }
    }
    b->blu.factor();
    const Real rc = b->blu.rcond(anorm);
    if (!(rc > 1e-14))
        throw NumericError("compute_basis_set: interface matrix is numerically singular (rcond=" +
                           std::to_string(rc) + ")");
    return b;
}

Vec BasisSet::dense_matrix() const {
    if (!banded) return M;
    const int d = dim();
    Vec out((size_t)d * d, 0.0);
    assemble_interface_matrix(*this, [&](int r, int c, Real v) { out[(size_t)r * d + c] += v; });
    return out;
}

std::vector<LocalSolution> solve_particular(const BasisSet& b, const std::vector<LocalData>& data,
                                            SolveCounters& c) {  // mrcm.cpp:242-252
    std::vector<LocalSolution> part(b.dd->n_sub());
    for_subdomains(b.dd->n_sub(), [&](int s) { part[s] = b.subs[s].solver.solve(data[s].q, data[s].bc); });
    c.particular += b.dd->n_sub();
    return part;
}

SkeletonCoeffs solve_interface(const BasisSet& b, const std::vector<LocalSolution>& part,
                               SolveCounters& c) {  // mrcm.cpp:254-268
    SkeletonCoeffs co;
    ++c.interface_solves;
    if (b.dim() == 0) return co;
    const Vec rhs = assemble_interface_rhs(b, part);
    const Vec x = b.banded ? b.blu.solve(rhs) : b.lu.solve(rhs);
    co.flux.assign(x.begin(), x.begin() + b.n_flux);
    co.pres.assign(x.begin() + b.n_flux, x.end());
    return co;
}

std::vector<LocalSolution> reconstruct(const BasisSet& b, const SkeletonCoeffs& co,
                                       const std::vector<LocalSolution>& part) {  // mrcm.cpp:270-288
    std::vector<LocalSolution> recon = part;
    for_subdomains(b.dd->n_sub(), [&](int s) {
        LocalSolution& sol = recon[s];
        for (const auto& h : b.subs[s].hom) {
            const Real c = h.col < b.n_flux ? co.flux[h.col] : co.pres[h.col - b.n_flux];
            if (c == 0.0) continue;
            for (size_t i = 0; i < sol.p.size(); ++i) sol.p[i] += c * h.sol.p[i];
            for (size_t i = 0; i < sol.u.size(); ++i) sol.u[i] += c * h.sol.u[i];
            for (size_t i = 0; i < sol.boundary_p.size(); ++i) sol.boundary_p[i] += c * h.sol.boundary_p[i];
        }
    });
    return recon;
}

std::vector<Vec> averaged_skeleton_flux(const Decomp& dd, const std::vector<LocalSolution>& recon) {
    // mrcm.cpp:290-304
    const FaceMap m = build_face_map(dd);
    std::vector<Vec> flux(dd.n_iface());
    for (int k = 0; k < dd.n_iface(); ++k) {
        const Interface& f = dd.ifaces[k];
        flux[k].resize(f.faces.size());
        for (int e = 0; e < (int)f.faces.size(); ++e) {
            const Real um = recon[f.minus].u[m.minus[k][e]];
            const Real up = recon[f.plus].u[m.plus[k][e]];
            flux[k][e] = 0.5 * (um + up);
        }
    }
    return flux;
}

DownscaleResult downscale(const Decomp& dd, const Vec& kappa, const Vec& q, const BoundarySpec& bc,
                          const std::vector<LocalSolution>& recon, const std::vector<Vec>& skel,
                          SolveCounters& cnt) {  // mrcm.cpp:306-439
    const int ns = dd.n_sub();
    const Real vol = dd.grid.vol();
    DownscaleResult out;
    for (const auto& f : skel) for (Real v : f) out.flux_scale = std::max(out.flux_scale, std::abs(v));
    Vec resid(ns, 0.0), ground(ns, 0.0);
    for (int s = 0; s < ns; ++s) {  // :315-340
        Real qsum = 0.0;
        const Rect& r = dd.subs[s];
        for (int jj = 0; jj < r.ny; ++jj)
            for (int ii = 0; ii < r.nx; ++ii) qsum += q[dd.grid.cell(r.i0 + ii, r.j0 + jj)] * vol;
        Real outflow = 0.0;
        for (const auto& e : dd.sub_boundary[s]) {
            const Real len = dd.grid.area(e.global_face);
            const Real un = e.on_skeleton ? e.sign * skel[e.iface][e.pos] : e.sign * recon[s].u[e.local_face];
            outflow += un * len;
            if (!e.on_skeleton && bc.faces[global_bc_index(dd.grid, e.global_face)].kind == Pressure)
                ground[s] += len;
        }
        resid[s] = qsum - outflow;
    }
    std::vector<Real> corr(dd.n_iface(), 0.0);  // :347-383
    Vec delta(ns, 0.0);
    Real gsum = 0.0;
    for (Real v : ground) gsum += v;
    const bool grounded = gsum > 0.0;
    if (ns > 1 || grounded) {
        // L is the area-weighted subdomain-adjacency Laplacian; banded in s
        // (half-bandwidth nsx) — same operator as the reference's dense L.
        const int w = dd.nsx;
        Vec band((size_t)ns * (w + 1), 0.0);
        auto B = [&](int r, int c) -> Real& { return band[(size_t)r * (w + 1) + (c - r + w)]; };
        for (int k = 0; k < dd.n_iface(); ++k) {
            const Interface& f = dd.ifaces[k];
            const Real area = f.faces.size() * dd.grid.area(f.faces[0]);
            B(f.minus, f.minus) += area;
            B(f.plus, f.plus) += area;
            B(f.plus, f.minus) -= area;  // plus > minus: lower triangle
        }
        Vec rhs = resid;
        if (grounded) {
            for (int s = 0; s < ns; ++s) B(s, s) += ground[s];
        } else {
            for (int c = 0; c <= std::min(w, ns - 1); ++c) B(c, 0) = 0.0;  // row/col 0 pinned
            B(0, 0) = 1.0;
            rhs[0] = 0.0;
        }
        BandLDLT ld;
        ld.n = ns;
        ld.w = w;
        ld.factor(band);
        ld.solve(rhs);
        delta = rhs;
        for (int k = 0; k < dd.n_iface(); ++k) {
            corr[k] = delta[dd.ifaces[k].minus] - delta[dd.ifaces[k].plus];
            out.repair_max = std::max(out.repair_max, std::abs(corr[k]));
        }
        if (grounded)
            for (int s = 0; s < ns; ++s)
                if (ground[s] > 0.0) out.repair_max = std::max(out.repair_max, std::abs(delta[s]));
    }
    out.repair_warning = out.repair_max > 0.1 * (out.flux_scale > 0 ? out.flux_scale : 1.0);
    out.p.assign(dd.grid.cells(), 0.0);
    out.u.assign(dd.grid.faces(), 0.0);
    for_subdomains(ns, [&](int s) {  // :388-427
        const Grid& lg = dd.subgrids[s];
        const Rect& r = dd.subs[s];
        BoundarySpec lb(lg.nx, lg.ny);
        const auto& edges = dd.sub_boundary[s];
        for (size_t i = 0; i < edges.size(); ++i) {
            const auto& e = edges[i];
            Real un;
            if (e.on_skeleton) {
                un = e.sign * (skel[e.iface][e.pos] + corr[e.iface]);
            } else {
                un = e.sign * recon[s].u[e.local_face];
                if (grounded && bc.faces[global_bc_index(dd.grid, e.global_face)].kind == Pressure) un += delta[s];
            }
            lb.faces[i].kind = Flux;
            lb.faces[i].value = un;
        }
        const Vec qs = dd.restrict_cells(q, s);
        LocalSolver solver(lg);
        solver.factorize(dd.restrict_cells(kappa, s), lb, 0);
        const LocalSolution sol = solver.solve(qs, lb);
        Real mref = 0.0, msol = 0.0;
        for (int c = 0; c < lg.cells(); ++c) {
            mref += recon[s].p[c];
            msol += sol.p[c];
        }
        const Real shift = (mref - msol) / lg.cells();
        for (int jj = 0; jj < r.ny; ++jj)
            for (int ii = 0; ii < r.nx; ++ii) out.p[dd.grid.cell(r.i0 + ii, r.j0 + jj)] = sol.p[lg.cell(ii, jj)] + shift;
        for (int lf = 0; lf < lg.faces(); ++lf) out.u[local_to_global_face(dd, s, lf)] = sol.u[lf];
    });
    cnt.downscale += ns;
    const Vec d = divergence(dd.grid, out.u);  // :429-437
    for (int c = 0; c < dd.grid.cells(); ++c) out.div_residual = std::max(out.div_residual, std::abs(d[c] - q[c]));
    Real sc = 0.0;
    for (Real v : q) sc = std::max(sc, std::abs(v));
    for (int f = 0; f < dd.grid.faces(); ++f) sc = std::max(sc, std::abs(out.u[f]) * dd.grid.area(f) / vol);
    out.div_scale = sc > 0.0 ? sc : 1.0;
    return out;
}

GlobalSolution mrcm_solve(const Vec& kappa, std::shared_ptr<const Decomp> dd, std::shared_ptr<const Space> sp,
                          const RobinParameter& beta, const Vec& q, const BoundarySpec& bc,
                          SolveCounters& c) {  // mrcm.cpp:441-457
    GlobalSolution g;
    g.basis = compute_basis_set(kappa, dd, sp, beta, q, bc, c);
    g.coeffs = solve_interface(*g.basis, g.basis->particular, c);
    g.recon = reconstruct(*g.basis, g.coeffs, g.basis->particular);
    const auto skel = averaged_skeleton_flux(*dd, g.recon);
    g.ds = downscale(*dd, kappa, q, bc, g.recon, skel, c);
    return g;
}

WeakResiduals weak_continuity_residuals(const BasisSet& b, const std::vector<LocalSolution>& recon) {
    // mrcm.cpp:459-483
    const Decomp& dd = *b.dd;
    const Space& sp = *b.space;
    Vec fj(std::max(1, b.n_pres), 0.0), pj(std::max(1, b.n_flux), 0.0);
    for (int s = 0; s < dd.n_sub(); ++s) {
        const auto& edges = dd.sub_boundary[s];
        for (size_t i = 0; i < edges.size(); ++i) {
            const auto& e = edges[i];
            if (!e.on_skeleton) continue;
            const int k = e.iface;
            const Real len = dd.grid.area(e.global_face);
            const Real un = e.sign * recon[s].u[e.local_face];
            const Real tp = recon[s].boundary_p[i];
            for (int r : sp.pres_by_iface[k]) fj[r] += un * sp.pres[r].values[e.pos] * len;
            for (int r : sp.flux_by_iface[k]) pj[r] -= e.sign * tp * sp.flux[r].values[e.pos] * len;
        }
    }
    WeakResiduals w;
    for (int r = 0; r < b.n_pres; ++r) w.flux_jump = std::max(w.flux_jump, std::abs(fj[r]));
    for (int r = 0; r < b.n_flux; ++r) w.pressure_jump = std::max(w.pressure_jump, std::abs(pj[r]));
    return w;
}

// ------------------------------------------------------------------ mpm ----
Real epsilon(const Grid& g, const Vec& kn, const Vec& km, int mode) {  // mpm.cpp:9-25
    if (mode == EpsMobility) throw ConfigError("epsilon: mobility mode needs saturation fields, not conductivities");
    if (kn.size() != km.size()) throw ConfigError("epsilon: fields live on different grids");
    const Real vol = g.vol();
    Real num = 0.0, den = 0.0;
    for (size_t c = 0; c < km.size(); ++c) {
        const Real d = kn[c] - km[c];
        num += d * d * vol;
        den += km[c] * km[c] * vol;
    }
    const Real a = std::sqrt(num);
    if (mode == EpsAbsolute) return a;
    if (!(den > 0.0)) throw NumericError("epsilon: zero reference norm in relative mode");
    return a / std::sqrt(den);
}

MpmResult mpm_pressure_update(const PerturbationState& st, const Vec& kappa_n, const Vec& q,
                              const BoundarySpec& bc, SolveCounters& cnt) {  // mpm.cpp:31-114
    const BasisSet& b = *st.basis;
    const Decomp& dd = *b.dd;
    if ((int)kappa_n.size() != dd.grid.cells())
        throw ConfigError("mpm_pressure_update: kappa_n does not match the decomposition grid");
    if ((int)st.recon_m.size() != dd.n_sub())
        throw ConfigError("mpm_pressure_update: stored solution does not match the basis set");
    std::vector<LocalData> data = restrict_physical_data(dd, b.beta, q, bc);
    std::vector<Vec> w(dd.n_sub());
    for_subdomains(dd.n_sub(), [&](int s) {  // :48-86
        const Grid& lg = dd.subgrids[s];
        const LocalSolution& m = st.recon_m[s];
        const Vec tn = transmissibility(lg, dd.restrict_cells(kappa_n, s));
        Vec& ws = w[s];
        ws.assign(lg.faces(), 0.0);
        for (int j = 0; j < lg.ny; ++j)
            for (int i = 1; i < lg.nx; ++i) {
                const int f = lg.vface(i, j);
                ws[f] = tn[f] * (m.p[lg.cell(i - 1, j)] - m.p[lg.cell(i, j)]) / lg.area(f);
            }
        for (int i = 0; i < lg.nx; ++i)
            for (int j = 1; j < lg.ny; ++j) {
                const int f = lg.hface(i, j);
                ws[f] = tn[f] * (m.p[lg.cell(i, j - 1)] - m.p[lg.cell(i, j)]) / lg.area(f);
            }
        const auto& edges = dd.sub_boundary[s];
        for (size_t i = 0; i < edges.size(); ++i) {
            const auto& e = edges[i];
            const int f = e.local_face;
            const Real un = tn[f] * (m.p[e.local_cell] - m.boundary_p[i]) / lg.area(f);
            ws[f] = e.sign * un;
            FaceBc& fb = data[s].bc.faces[i];
            if (fb.kind == Pressure) fb.value -= m.boundary_p[i];
            else if (fb.kind == Flux) fb.value -= un;
        }
        const Vec dw = divergence(lg, ws);
        for (int c = 0; c < lg.cells(); ++c) data[s].q[c] -= dw[c];
    });
    const std::vector<LocalSolution> dbar = solve_particular(b, data, cnt);
    MpmResult out;
    out.delta = solve_interface(b, dbar, cnt);
    const std::vector<LocalSolution> delta = reconstruct(b, out.delta, dbar);
    out.recon_n.resize(dd.n_sub());
    for (int s = 0; s < dd.n_sub(); ++s) {  // :93-103
        LocalSolution sol = delta[s];
        const LocalSolution& m = st.recon_m[s];
        for (size_t i = 0; i < sol.p.size(); ++i) sol.p[i] += m.p[i];
        for (size_t i = 0; i < sol.u.size(); ++i) sol.u[i] += w[s][i];
        for (size_t i = 0; i < sol.boundary_p.size(); ++i) sol.boundary_p[i] += m.boundary_p[i];
        out.recon_n[s] = std::move(sol);
    }
    const auto skel = averaged_skeleton_flux(dd, out.recon_n);
    out.ds = downscale(dd, kappa_n, q, bc, out.recon_n, skel, cnt);
    return out;
}

// ------------------------------------------------------------ transport ----
namespace {
std::atomic<int64_t> g_clamp{0};
Real clamp_s(Real s) {  // transport.cpp:13-21
    if (s < 0.0 || s > 1.0) {
        ++g_clamp;
        return std::clamp<Real>(s, 0.0, 1.0);
    }
    return s;
}
Real fprime(Real s, Real M) {  // transport.cpp:23-27
    const Real d = M * s * s + (1.0 - s) * (1.0 - s);
    const Real dd = 2.0 * M * s - 2.0 * (1.0 - s);
    return (2.0 * M * s * d - M * s * s * dd) / (d * d);
}
}  // namespace
int64_t clamp_count() { return g_clamp.load(); }
void reset_clamp_count() { g_clamp.store(0); }

Real total_mobility(Real s, Real M) {  // transport.cpp:34-37
    s = clamp_s(s);
    return M * s * s + (1.0 - s) * (1.0 - s);
}
Real fractional_flow(Real s, Real M) {  // transport.cpp:39-43
    s = clamp_s(s);
    const Real w = M * s * s;
    return w / (w + (1.0 - s) * (1.0 - s));
}
Real max_fractional_flow_slope(Real M) {  // transport.cpp:45-49
    Real m = 0.0;
    for (int k = 0; k <= 1000; ++k) m = std::max(m, fprime(k * 1e-3, M));
    return m;
}
Real cfl_timestep(const Grid& g, const Vec& u, Real M, Real safety, Real dt_cap) {  // transport.cpp:51-71
    const Real vol = g.vol();
    const Real slope = max_fractional_flow_slope(M);
    Real dt = dt_cap / safety;
    bool any = false;
    for (int j = 0; j < g.ny; ++j)
        for (int i = 0; i < g.nx; ++i) {
            Real out = 0.0;
            out += std::max<Real>(0.0, u[g.vface(i + 1, j)]) * g.hy;
            out += std::max<Real>(0.0, -u[g.vface(i, j)]) * g.hy;
            out += std::max<Real>(0.0, u[g.hface(i, j + 1)]) * g.hx;
            out += std::max<Real>(0.0, -u[g.hface(i, j)]) * g.hx;
            if (out > 0.0) {
                any = true;
                dt = std::min(dt, vol / (out * slope));
            }
        }
    if (!any) return dt_cap;
    return std::min(safety * dt, dt_cap);
}
Vec upwind_step(const Grid& g, const Vec& s, Real inflow, const Vec& u, Real dt, Real M) {  // transport.cpp:73-120
    if ((int)s.size() != g.cells()) throw ConfigError("upwind_step: grid mismatch");
    Vec wf(g.faces());
    const Real fin = fractional_flow(inflow, M);
    for (int j = 0; j < g.ny; ++j)
        for (int i = 0; i <= g.nx; ++i) {
            const int f = g.vface(i, j);
            const Real un = u[f];
            Real fs;
            if (un >= 0.0) fs = (i == 0) ? fin : fractional_flow(s[g.cell(i - 1, j)], M);
            else fs = (i == g.nx) ? fin : fractional_flow(s[g.cell(i, j)], M);
            wf[f] = fs * un * g.hy;
        }
    for (int i = 0; i < g.nx; ++i)
        for (int j = 0; j <= g.ny; ++j) {
            const int f = g.hface(i, j);
            const Real un = u[f];
            Real fs;
            if (un >= 0.0) fs = (j == 0) ? fin : fractional_flow(s[g.cell(i, j - 1)], M);
            else fs = (j == g.ny) ? fin : fractional_flow(s[g.cell(i, j)], M);
            wf[f] = fs * un * g.hx;
        }
    Vec out = s;
    const Real vol = g.vol();
    for (int j = 0; j < g.ny; ++j)
        for (int i = 0; i < g.nx; ++i) {
            const int c = g.cell(i, j);
            const Real net = wf[g.vface(i + 1, j)] - wf[g.vface(i, j)] + wf[g.hface(i, j + 1)] - wf[g.hface(i, j)];
            const Real sn = s[c] - dt / vol * net;
            if (sn < -1e-12 || sn > 1.0 + 1e-12)
                throw NumericError("upwind_step: saturation left [0,1]; CFL condition violated");
            out[c] = std::clamp<Real>(sn, 0.0, 1.0);
        }
    return out;
}
Vec conductivity(const Vec& K, const Vec& s, Real M) {  // transport.cpp:122-126
    Vec k(K.size());
    for (size_t c = 0; c < K.size(); ++c) k[c] = total_mobility(s[c], M) * K[c];
    return k;
}

// ----------------------------------------------------------- simulation ----
Real rcr(long nhat, long n, long te, long tm) {  // simulation.cpp:11-19
    if (te <= 0) throw ConfigError("rcr: te must be positive");
    if (nhat < 0 || n < 0 || tm < 0) throw ConfigError("rcr: negative counter");
    if (tm > te) throw ConfigError("rcr: tm exceeds te");
    const Real frac = (Real)(te - tm) / (Real)te;
    const Real bf = 1.0 - 2.0 * (Real)n / (Real)(nhat + 2 * n);
    return frac * bf * 100.0;
}
Real relative_flux_error(const Grid& g, const Vec& u, const Vec& ur) {  // simulation.cpp:30-45
    Real num = 0.0, den = 0.0;
    for (int f = 0; f < g.faces(); ++f) {
        const Real w = g.area(f), d = u[f] - ur[f];
        num += w * d * d;
        den += w * ur[f] * ur[f];
    }
    if (!(den > 0.0)) {
        if (num == 0.0) return 0.0;
        throw NumericError("relative_flux_error: zero reference norm");
    }
    return std::sqrt(num / den);
}
Real relative_sat_error(const Vec& s, const Vec& sr) {  // simulation.cpp:47-59
    Real num = 0.0, den = 0.0;
    for (size_t c = 0; c < s.size(); ++c) {
        num += std::abs(s[c] - sr[c]);
        den += std::abs(sr[c]);
    }
    if (!(den > 0.0)) {
        if (num == 0.0) return 0.0;
        throw NumericError("relative_sat_error: zero reference norm");
    }
    return num / den;
}
Real max_outlet_saturation(const Grid& g, const Vec& s, const Vec& u) {  // simulation.cpp:61-83
    Real m = 0.0;
    auto side = [&](auto&& face_of, auto&& cell_of, int count, Real area) {
        Real net = 0.0;
        for (int k = 0; k < count; ++k) net += face_of(k) * area;
        if (!(net > 1e-14)) return;
        for (int k = 0; k < count; ++k)
            if (face_of(k) > 1e-14) m = std::max(m, s[cell_of(k)]);
    };
    side([&](int j) { return -u[g.vface(0, j)]; }, [&](int j) { return g.cell(0, j); }, g.ny, g.hy);
    side([&](int j) { return u[g.vface(g.nx, j)]; }, [&](int j) { return g.cell(g.nx - 1, j); }, g.ny, g.hy);
    side([&](int i) { return -u[g.hface(i, 0)]; }, [&](int i) { return g.cell(i, 0); }, g.nx, g.hx);
    side([&](int i) { return u[g.hface(i, g.ny)]; }, [&](int i) { return g.cell(i, g.ny - 1); }, g.nx, g.hx);
    return m;
}
Real injection_rate(const Grid& g, const Vec& u, Real inflow, Real M) {  // simulation.cpp:85-101
    const Real fin = fractional_flow(inflow, M);
    Real rate = 0.0;
    auto consider = [&](Real un, Real area) { if (un < 0.0) rate += -un * area * fin; };
    for (int j = 0; j < g.ny; ++j) {
        consider(-u[g.vface(0, j)], g.hy);
        consider(u[g.vface(g.nx, j)], g.hy);
    }
    for (int i = 0; i < g.nx; ++i) {
        consider(-u[g.hface(i, 0)], g.hx);
        consider(u[g.hface(i, g.ny)], g.hx);
    }
    return rate;
}

// Runner: simulation.cpp:118-340 split at the loop boundary.
Runner::Runner(const RunInputs& in) : in_(in) {
    const Grid& g = in_.dd->grid;
    if ((int)in_.K.size() != g.cells()) throw ConfigError("run: permeability grid mismatch");
    if ((int)in_.s0.size() != g.cells()) throw ConfigError("run: initial saturation grid mismatch");
    const Split& sc = in_.split;
    if (sc.cn < 1) throw ConfigError("run: cn must be >= 1");
    if (sc.te <= 0 && sc.pvi_max <= 0.0 && !sc.stop_on_breakthrough) throw ConfigError("run: no stop condition configured");
    if (sc.method == Mpm2p && sc.eta < 0.0) throw ConfigError("run: negative eta");
    q_ = in_.q.size() > 0 ? in_.q : Vec(g.cells(), 0.0);
    multiscale_ = sc.method != FineReference;
    track_ = sc.track_errors && multiscale_;
    rec_.n_sub = in_.dd->n_sub();
    s_main_ = in_.s0;
    s_ref_ = s_main_;
    fine_ = std::make_unique<LocalSolver>(g);
    fine_anchor_ = in_.bc.pure_neumann() ? 0 : -1;
    state_.eta = sc.eta;
    state_.mode = sc.eta_mode;
}

LocalSolution Runner::fine_solve(const Vec& kappa) {  // simulation.cpp:143-150
    fine_->factorize(kappa, in_.bc, fine_anchor_);
    ++rec_.counters.fine;
    return fine_->solve(q_, in_.bc);
}

Real Runner::drift(const Vec& kappa_n) {  // simulation.cpp:162-174
    const Grid& g = in_.dd->grid;
    if (in_.split.eta_mode == EpsMobility) {
        Vec lam(g.cells());
        for (int c = 0; c < g.cells(); ++c) lam[c] = total_mobility(s_main_[c], in_.M);
        return epsilon(g, lam, lambda_rebuild_, EpsAbsolute) / in_.M;
    }
    return epsilon(g, kappa_n, state_.basis->kappa_m, in_.split.eta_mode);
}

void Runner::note(Real dres, Real dscale, bool warn) {  // simulation.cpp:176-181
    step_div_ = dres;
    rec_.max_div_residual = std::max(rec_.max_div_residual, dres);
    rec_.max_div_ratio = std::max(rec_.max_div_ratio, dres / dscale);
    if (warn) ++rec_.repair_warnings;
}

void Runner::rebuild(const Vec& kappa) {  // simulation.cpp:183-193
    const RobinParameter beta = compute_beta(kappa, *in_.dd, in_.alpha);
    // the old basis is not needed by the new one: release it first, so the
    // peak footprint is one basis (C5 in long double: ~35 GB) instead of two
    state_.basis.reset();
    state_.recon_m.clear();
    GlobalSolution sol = mrcm_solve(kappa, in_.dd, in_.space, beta, q_, in_.bc, rec_.counters);
    state_.basis = sol.basis;
    state_.recon_m = std::move(sol.recon);
    rec_.nhat = state_.basis->nhat();
    p_main_ = std::move(sol.ds.p);
    u_main_ = std::move(sol.ds.u);
    const Grid& g = in_.dd->grid;
    lambda_rebuild_.resize(g.cells());
    for (int c = 0; c < g.cells(); ++c) lambda_rebuild_[c] = total_mobility(s_main_[c], in_.M);
    note(sol.ds.div_residual, sol.ds.div_scale, sol.ds.repair_warning);
}

void Runner::reuse(const Vec& kappa) {  // simulation.cpp:195-200
    MpmResult r = mpm_pressure_update(state_, kappa, q_, in_.bc, rec_.counters);
    p_main_ = std::move(r.ds.p);
    u_main_ = std::move(r.ds.u);
    note(r.ds.div_residual, r.ds.div_scale, r.ds.repair_warning);
}

void Runner::record_step(int rebuilt, Real eps, Real dt, Real wall) {  // simulation.cpp:207-227
    StepRecord sr;
    sr.step = n_;
    sr.pvi = pvi_;
    sr.epsilon = eps;
    sr.rebuilt = rebuilt;
    if (track_) {
        sr.flux_err = relative_flux_error(in_.dd->grid, u_main_, u_ref_);
        Real num = 0.0;
        for (size_t c = 0; c < s_main_.size(); ++c) num += std::abs(s_main_[c] - s_ref_[c]);
        sr.sat_err = num == 0.0 ? 0.0 : relative_sat_error(s_main_, s_ref_);
    }
    sr.bf_homog_cum = rec_.counters.homogeneous;
    sr.bf_part_cum = rec_.counters.particular;
    sr.dt = dt;
    sr.wall_s = wall;
    sr.div_residual = step_div_;
    rec_.steps.push_back(sr);
    if (rebuilt) rec_.update_steps.push_back(n_);
}

void Runner::breakthrough_check() {  // simulation.cpp:253-259
    if (rec_.breakthrough_step >= 0) return;
    if (max_outlet_saturation(in_.dd->grid, s_main_, u_main_) > in_.split.breakthrough_threshold) {
        rec_.breakthrough_step = n_ - 1;
        rec_.breakthrough_pvi = pvi_;
    }
}

void Runner::begin() {  // simulation.cpp:232-260
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    pvi_ = 0.0;
    n_ = 0;
    ell_ = 0;
    eps_ = in_.split.eta;
    const Vec k0 = conductivity(in_.K, s_main_, in_.M);
    if (track_ || !multiscale_) {
        LocalSolution ref = fine_solve(k0);
        u_ref_ = ref.u;
        p_ref_ = ref.p;
        if (!multiscale_) {
            p_main_ = p_ref_;
            u_main_ = u_ref_;
            note(conservation_residual(in_.dd->grid, ref, q_), residual_scale(in_.dd->grid, ref, q_), false);
        }
    }
    if (multiscale_) rebuild(k0);
    record_step(1, 0.0, 0.0, std::chrono::duration<double>(clk::now() - t0).count());
    n_ = 1;
    breakthrough_check();
}

bool Runner::step() {  // simulation.cpp:262-329
    const Split& sc = in_.split;
    if (sc.te > 0 && n_ >= sc.te) return false;
    if (sc.pvi_max > 0.0 && pvi_ >= sc.pvi_max) return false;
    if (sc.stop_on_breakthrough && rec_.breakthrough_step >= 0) return false;
    if (n_ >= sc.max_steps_hard) return false;
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    const Grid& g = in_.dd->grid;
    const Vec& usched = track_ ? u_ref_ : u_main_;
    const Real dt = cfl_timestep(g, usched, in_.M, sc.cfl_safety, sc.dt_cap);
    int sub = 1;
    if (track_) {
        const Real dtm = cfl_timestep(g, u_main_, in_.M, sc.cfl_safety, sc.dt_cap);
        if (dt > dtm * (1.0 + 1e-12)) sub = (int)std::ceil(dt / dtm - 1e-12);
    }
    const Real inj = injection_rate(g, usched, in_.inflow_sat, in_.M);
    const Real pore = g.lx * g.ly;
    for (int k = 0; k < sc.cn; ++k) {
        for (int j = 0; j < sub; ++j) s_main_ = upwind_step(g, s_main_, in_.inflow_sat, u_main_, dt / sub, in_.M);
        if (track_) s_ref_ = upwind_step(g, s_ref_, in_.inflow_sat, u_ref_, dt, in_.M);
        pvi_ += inj * dt / pore;
    }
    const Vec kn = conductivity(in_.K, s_main_, in_.M);
    if (track_) {
        LocalSolution ref = fine_solve(conductivity(in_.K, s_ref_, in_.M));
        u_ref_ = ref.u;
        p_ref_ = ref.p;
    }
    int rebuilt = 0;
    if (!multiscale_) {
        LocalSolution sol = fine_solve(kn);
        p_main_ = sol.p;
        u_main_ = sol.u;
        note(conservation_residual(g, sol, q_), residual_scale(g, sol, q_), false);
        rebuilt = 1;
    } else {
        bool do_rebuild = false;
        if (sc.method == MrcmEveryStep) do_rebuild = true;
        else if (sc.method == Mpm2p) {
            do_rebuild = (sc.eta <= 0.0) || (eps_ > sc.eta);
            if (sc.eta > 0.0 && n_ > 1)  // step 1 compares eps0 = eta by construction
                rec_.min_eps_margin = std::min(rec_.min_eps_margin, std::abs(eps_ - sc.eta) / sc.eta);
        }
        if (do_rebuild) {
            ++ell_;
            rebuild(kn);
            rebuilt = 1;
        } else {
            reuse(kn);
        }
        eps_ = drift(kn);
    }
    record_step(rebuilt, multiscale_ ? eps_ : 0.0, dt, std::chrono::duration<double>(clk::now() - t0).count());
    ++n_;
    breakthrough_check();
    return true;
}

RunResult Runner::finish() {  // simulation.cpp:331-340
    rec_.te = n_;
    rec_.tm_updates = ell_;
    rec_.tm_total = (long)rec_.update_steps.size();
    rec_.final_pvi = pvi_;
    RunResult r;
    r.rec = rec_;
    r.s_final = s_main_;
    r.p_final = p_main_;
    r.u_final = u_main_;
    return r;
}

RunResult run(const RunInputs& in) {
    Runner r(in);
    r.begin();
    while (r.step()) {}
    return r.finish();
}

// -------------------------------------------------------------- fields ----
Vec gaussian_field(const Grid& g, Real delta, Real mean_coeff, uint64_t seed, bool range_norm,
                   Real range_target) {  // fields_io.cpp:25-85
    const int n = g.cells();
    if (n > (1 << 16)) throw CapacityError("generate_gaussian: grid exceeds the dense-covariance guard (2^16 cells)");
    if (!(delta > 0.0) || !(mean_coeff > 0.0)) throw ConfigError("generate_gaussian: delta and mean_coeff must be positive");
    Vec C((size_t)n * n);
    const Real hmin = g.hx < g.hy ? g.hx : g.hy;
    const Real diag = 1.0 / std::sqrt(hmin / 2.0);
    Real trace = 0.0;
    for (int j1 = 0; j1 < g.ny; ++j1)
        for (int i1 = 0; i1 < g.nx; ++i1) {
            const int a = g.cell(i1, j1);
            for (int j2 = 0; j2 < g.ny; ++j2)
                for (int i2 = 0; i2 < g.nx; ++i2) {
                    const int b = g.cell(i2, j2);
                    if (a == b) C[(size_t)a * n + b] = diag;
                    else {
                        const Real dx = g.cx(i1) - g.cx(i2), dy = g.cy(j1) - g.cy(j2);
                        C[(size_t)a * n + b] = 1.0 / std::sqrt(std::sqrt(dx * dx + dy * dy));
                    }
                }
        }
    for (int i = 0; i < n; ++i) trace += C[(size_t)i * n + i];
    const Real jitter = 1e-8 * trace / n;
    for (int i = 0; i < n; ++i) C[(size_t)i * n + i] += jitter;
    // Blocked right-looking Cholesky, lower factor stored in place (row-major).
    const int nb = 64;
    for (int k0 = 0; k0 < n; k0 += nb) {
        const int k1 = std::min(n, k0 + nb);
        for (int k = k0; k < k1; ++k) {  // panel factorization
            Real d = C[(size_t)k * n + k];
            for (int m = k0; m < k; ++m) d -= C[(size_t)k * n + m] * C[(size_t)k * n + m];
            if (!(d > 0.0)) throw NumericError("generate_gaussian: covariance matrix is not positive definite");
            d = std::sqrt(d);
            C[(size_t)k * n + k] = d;
            for (int i = k + 1; i < n; ++i) {
                Real s = C[(size_t)i * n + k];
                const Real* ri = &C[(size_t)i * n];
                const Real* rk = &C[(size_t)k * n];
                for (int m = k0; m < k; ++m) s -= ri[m] * rk[m];
                C[(size_t)i * n + k] = s / d;
            }
        }
        for (int i = k1; i < n; ++i) {  // trailing update, lower triangle
            Real* ri = &C[(size_t)i * n];
            for (int j = k1; j <= i; ++j) {
                const Real* rj = &C[(size_t)j * n];
                Real s = 0.0;
                for (int m = k0; m < k1; ++m) s += ri[m] * rj[m];
                ri[j] -= s;
            }
        }
    }
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> normal(0.0, 1.0);
    Vec z(n);
    for (int i = 0; i < n; ++i) z[i] = normal(rng);
    Vec xi(n, 0.0);
    for (int i = 0; i < n; ++i) {
        Real s = 0.0;
        for (int m = 0; m <= i; ++m) s += C[(size_t)i * n + m] * z[m];
        xi[i] = s;
    }
    if (range_norm) {
        Real lo = xi[0], hi = xi[0];
        for (Real v : xi) { lo = std::min(lo, v); hi = std::max(hi, v); }
        const Real mid = 0.5 * (lo + hi), span = hi - lo;
        if (span > 0.0) for (Real& v : xi) v = (v - mid) * (range_target / span);
    }
    Vec K(n);
    for (int c = 0; c < n; ++c) K[c] = mean_coeff * std::exp(delta * xi[c]);
    return K;
}

Vec load_cell_field(const std::string& path, const Grid& g) {  // fields_io.cpp:97-116
    std::ifstream in(path);
    if (!in) throw ConfigError("load_field: cannot open " + path);
    int nx = -1, ny = -1;
    if (!(in >> nx >> ny)) throw ConfigError("load_field: bad header in " + path);
    if (nx != g.nx || ny != g.ny) throw ConfigError("load_field: " + path + " has the wrong shape");
    Vec f(g.cells());
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            Real v;
            if (!(in >> v)) throw ConfigError("load_field: parse failure in " + path);
            f[g.cell(i, j)] = v;
        }
    return f;
}

void save_cell_field(const std::string& path, const Grid& g, const Vec& f) {  // fields_io.cpp:118-136
    FILE* fp = std::fopen(path.c_str(), "w");
    if (!fp) throw ConfigError("save_cell_field: cannot write " + path);
    std::fprintf(fp, "%d %d\n", g.nx, g.ny);
    for (int j = 0; j < g.ny; ++j) {
        for (int i = 0; i < g.nx; ++i) std::fprintf(fp, i ? " %.17g" : "%.17g", (double)f[g.cell(i, j)]);
        std::fprintf(fp, "\n");
    }
    std::fclose(fp);
}

BoundarySpec preset_bc(const Grid& g, int preset) {  // config.cpp:525-538
    BoundarySpec bc(g.nx, g.ny);
    auto set = [&](FaceBc w, FaceBc e, FaceBc s, FaceBc n) {
        for (int j = 0; j < g.ny; ++j) { bc.faces[j] = w; bc.faces[g.ny + j] = e; }
        for (int i = 0; i < g.nx; ++i) { bc.faces[2 * g.ny + i] = s; bc.faces[2 * g.ny + g.nx + i] = n; }
    };
    auto P = [](Real v) { FaceBc f; f.kind = Pressure; f.value = v; return f; };
    auto F = [](Real v) { FaceBc f; f.kind = Flux; f.value = v; return f; };
    if (preset == 0) set(P(1.0), P(0.0), F(0.0), F(0.0));
    else if (preset == 1) set(F(-1.0), P(0.0), F(0.0), F(0.0));
    else if (preset == 2) set(P(0.0), P(-1e4), F(0.0), F(0.0));
    else throw ConfigError("preset_bc: unknown preset");
    return bc;
}

}  // namespace orc
