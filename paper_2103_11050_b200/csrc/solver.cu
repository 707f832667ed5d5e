// solver.cu — the velocity-update path on the device:
//   K2  MPM data prep (w, q', g', z')                 proj/src/mpm.cpp:48-86
//   K3  local Robin solves, cached factor             proj/src/mrcm.cpp:242-252, elliptic.cpp:152-243
//   K4  rebuild: factor + homogeneous/particular       proj/src/mrcm.cpp:132-194
//   K5  interface-matrix assembly (CSR, deterministic) proj/src/mrcm.cpp:196-224
//   K6  interface rhs                                  proj/src/mrcm.cpp:80-100
//   K8  trace recombination (reconstruct)              proj/src/mrcm.cpp:270-288
//   K9  averaged skeleton flux + compatibility resid   proj/src/mrcm.cpp:290-304,315-340
//   K10 static repair solve (graph Laplacian inverse)  proj/src/mrcm.cpp:347-383
//   K11 downscale: fresh Neumann solve with kappa_n,   proj/src/mrcm.cpp:388-437
//       mean shift, scatter, divergence residual
//   K12 Robin parameter beta (adaptive quantiles)      proj/src/robin.cpp:39-92
// One warp owns one subdomain in the banded kernels (band.cuh); everything
// else is one thread per cell / face / edge / matrix entry. No floating-point
// atomics: every sum has a fixed order, so runs are bitwise reproducible.
#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>

#include "band.cuh"
#include "band_reg.cuh"
#include "band_blk.cuh"
#include "band_twist.cuh"
#include "context.cuh"

namespace mpm2p {

namespace {

constexpr int TPB = 256;
constexpr int WPB = 4;  // warps (subdomains) per block in banded kernels
constexpr int HOM_GROUP = 8;  // homogeneous right-hand sides per warp in k_hom_solve_rm

__device__ __forceinline__ bool last_block_done(unsigned* counter) {
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x * gridDim.y * gridDim.z - 1;
    __syncthreads();
    return last;
}

__device__ __forceinline__ double block_max(double v, double* sh) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = warp_max(v);
    if (lane == 0) sh[w] = v;
    __syncthreads();
    if (w == 0) {
        v = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
        v = warp_max(v);
    }
    __syncthreads();
    return v;
}

__device__ __forceinline__ size_t xoff(const Layout& L, int max_rhs, int s, int m) {
    return ((size_t)s * max_rhs + m) * L.ncs;
}

// beta of a skeleton edge seen from subdomain side (RobinParameter::beta, robin.hpp:24-26)
__device__ __forceinline__ double edge_beta(const Layout& L, const EdgeInfo& e, const double* bm, const double* bp) {
    const int i = L.skel_index(e.iface, e.pos);
    return e.sign > 0 ? bm[i] : bp[i];
}

// ---------------------------------------------------------------- K12 ----
__global__ void k_face_kappa(Layout L, const double* __restrict__ kappa, double* __restrict__ fk) {
    pdl_begin();
    const int E = L.skeleton_edges();
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < E; x += gridDim.x * blockDim.x) {
        const int k = x < L.NV * L.sny ? x / L.sny : L.NV + (x - L.NV * L.sny) / L.snx;
        const int pos = x < L.NV * L.sny ? x % L.sny : (x - L.NV * L.sny) % L.snx;
        int cm, cp;
        L.iface_cells(k, pos, cm, cp);
        fk[x] = 2.0 * kappa[cm] * kappa[cp] / (kappa[cm] + kappa[cp]);
    }
}

__device__ double quantile_sorted(const double* v, int m, double pct) {  // robin.cpp:26-35
    if (m == 0) return 0.0;
    double idx = pct / 100.0 * (double)(m - 1);
    idx = fmin(fmax(idx, 0.0), (double)(m - 1));
    const int lo = (int)idx;
    const int hi = lo + 1 < m - 1 ? lo + 1 : m - 1;
    const double w = idx - (double)lo;
    return (1.0 - w) * v[lo] + w * v[hi];
}

__global__ void k_beta(Layout L, const double* __restrict__ kappa, const double* __restrict__ fk,
                       const double* __restrict__ sorted, int adaptive, double alpha, double amin, double amax,
                       double plo, double phi, double* bm, double* bp, double* al, Scalars* sc) {
    pdl_begin();
    const int E = L.skeleton_edges();
    double qlo = 0.0, qhi = 0.0;
    if (adaptive && E > 0) {
        qlo = quantile_sorted(sorted, E, plo);
        qhi = quantile_sorted(sorted, E, phi);
    }
    const double Lx = L.lx / L.nsx, Ly = L.ly / L.nsy;
    const double H = Lx > Ly ? Lx : Ly;  // coarse_h (decomposition.cpp:15-19)
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < E; x += gridDim.x * blockDim.x) {
        const int k = x < L.NV * L.sny ? x / L.sny : L.NV + (x - L.NV * L.sny) / L.snx;
        const int pos = x < L.NV * L.sny ? x % L.sny : (x - L.NV * L.sny) % L.snx;
        int cm, cp;
        L.iface_cells(k, pos, cm, cp);
        if (!(kappa[cm] > 0.0) || !(kappa[cp] > 0.0)) atomicOr(&sc->err, ERR_KAPPA);
        double a = alpha;
        if (adaptive) {
            const double v = fk[x];
            a = v > qhi ? amin : (v < qlo ? amax : 1.0);
        }
        al[x] = a;
        bm[x] = a * H / kappa[cm];
        bp[x] = a * H / kappa[cp];
    }
}

// ---------------------------------------------------------- transmissibility
__global__ void k_trans(Layout L, const double* __restrict__ kappa, double* __restrict__ T) {
    pdl_begin();  // elliptic.cpp:44-61
    const int F = L.faces();
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < F; f += gridDim.x * blockDim.x) {
        double t = 0.0;
        if (f < L.vcount()) {
            const int i = f % (L.nx + 1), j = f / (L.nx + 1);
            if (i > 0 && i < L.nx) t = harm_trans_v(L, kappa[L.cell(i - 1, j)], kappa[L.cell(i, j)]);
        } else {
            const int fh = f - L.vcount(), i = fh % L.nx, j = fh / L.nx;
            if (j > 0 && j < L.ny) t = harm_trans_h(L, kappa[L.cell(i, j - 1)], kappa[L.cell(i, j)]);
        }
        T[f] = t;
    }
}

// boundary-edge indices of a cell in W,E,S,N order (the for_each_boundary_face order)
__device__ __forceinline__ int cell_edges(const Layout& L, int ii, int jj, int* idx) {
    int n = 0;
    if (ii == 0) idx[n++] = jj;
    if (ii == L.snx - 1) idx[n++] = L.sny + jj;
    if (jj == 0) idx[n++] = 2 * L.sny + ii;
    if (jj == L.sny - 1) idx[n++] = 2 * L.sny + L.snx + ii;
    return n;
}

// Band entries of the subdomain operator (elliptic.cpp:80-141).
// mode 0: rebuild operator (Robin beta on the skeleton, physical kinds), anchor if anchor!=0
// mode 1: downscale operator (all Flux, anchor cell 0)
__global__ void k_band_entries(Layout L, const double* __restrict__ kappa, const double* __restrict__ T, int mode,
                               int anchor, const double* __restrict__ bm, const double* __restrict__ bp,
                               const int* __restrict__ bc_kind, double* __restrict__ BD, double* __restrict__ BW,
                               double* __restrict__ BS, Scalars* sc) {
    pdl_begin();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= L.cells()) return;
    const int i = c % L.nx, j = c / L.nx;
    const int s = (j / L.sny) * L.nsx + i / L.snx;
    const int ii = i % L.snx, jj = j % L.sny, r = jj * L.snx + ii;
    const double kc = kappa[c];
    if (!(kc > 0.0) || !isfinite(kc)) atomicOr(&sc->err, ERR_KAPPA);
    double diag = 0.0;
    if (ii > 0) diag += T[L.vface(i, j)];
    if (ii < L.snx - 1) diag += T[L.vface(i + 1, j)];
    if (jj > 0) diag += T[L.hface(i, j)];
    if (jj < L.sny - 1) diag += T[L.hface(i, j + 1)];
    double ow = ii > 0 ? T[L.vface(i, j)] : 0.0;
    double os = jj > 0 ? T[L.hface(i, j)] : 0.0;
    if (mode == 0) {
        int idx[4];
        const int ne = cell_edges(L, ii, jj, idx);
        for (int t = 0; t < ne; ++t) {
            const EdgeInfo e = L.edge(s, idx[t]);
            const double th = half_trans(L, e.side, kc);
            if (e.iface >= 0) {
                const double beta = edge_beta(L, e, bm, bp);
                if (!(beta > 0.0)) atomicOr(&sc->err, ERR_ROBIN_BETA);
                diag += eff_robin(th, beta, e.area);
            } else if (bc_kind[e.gbc] == BC_PRESSURE) {
                diag += th;
            } else if (bc_kind[e.gbc] == BC_ROBIN) {  // elliptic.cpp:133-136
                const double beta = L.rb_beta[e.gbc];
                if (!(beta > 0.0)) atomicOr(&sc->err, ERR_ROBIN_BETA);
                diag += eff_robin(th, beta, e.area);
            }
        }
    }
    if (anchor) {
        if (r == 0) diag = 1.0;
        if (r == 1) ow = 0.0;
        if (r == L.snx) os = 0.0;
    }
    const size_t o = (size_t)s * L.ncs + r;
    BD[o] = diag;
    BW[o] = ow;
    BS[o] = os;
}

// ---------------------------------------------------------------- K4 ----
// Particular (m = 0) and homogeneous (m = 1 + h) right-hand sides
// (elliptic.cpp:161-180 with the data of mrcm.cpp:164-191).
__global__ void k_rebuild_rhs(Layout L, int max_rhs, const double* __restrict__ kappa, const double* __restrict__ q,
                              const int* __restrict__ bc_kind, const double* __restrict__ bc_value,
                              const double* __restrict__ bm, const double* __restrict__ bp, int anchor,
                              double* __restrict__ X) {
    pdl_begin();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= L.cells()) return;
    const int i = c % L.nx, j = c / L.nx;
    const int s = (j / L.sny) * L.nsx + i / L.snx;
    const int ii = i % L.snx, jj = j % L.sny, r = jj * L.snx + ii;
    const double vol = L.vol();
    int idx[4];
    const int ne = cell_edges(L, ii, jj, idx);
    EdgeInfo e[4];
    double th[4], beta[4], er[4];
    for (int t = 0; t < ne; ++t) {
        e[t] = L.edge(s, idx[t]);
        th[t] = half_trans(L, e[t].side, kappa[c]);
        const bool prob = e[t].iface < 0 && bc_kind[e[t].gbc] == BC_ROBIN;  // physical Robin face
        beta[t] = e[t].iface >= 0 ? edge_beta(L, e[t], bm, bp) : prob ? L.rb_beta[e[t].gbc] : 0.0;
        er[t] = (e[t].iface >= 0 || prob) ? eff_robin(th[t], beta[t], e[t].area) : 0.0;
    }
    // m = 0 (particular): interface edges contribute er * 0
    {
        double b = q[c] * vol;
        for (int t = 0; t < ne; ++t) {
            if (e[t].iface >= 0) {
                b += er[t] * 0.0;
            } else {
                const double val = bc_value[e[t].gbc];
                const int kind = bc_kind[e[t].gbc];
                if (kind == BC_PRESSURE) b += th[t] * val;
                else if (kind == BC_ROBIN) b += er[t] * L.rb_rhs[e[t].gbc];  // elliptic.cpp:176-177
                else b -= val * e[t].area;
            }
        }
        if (anchor && r == 0) b = 0.0;
        X[xoff(L, max_rhs, s, 0) + r] = b;
    }
    // m > 0 (homogeneous): only edges on the function's interface are nonzero
    // (the skipped terms are +-0 additions; the sums are bit-identical)
    const int nh = L.n_hom(s);
    for (int m = 1; m <= nh; ++m) {
        int hk, ht, hcol;
        bool hflux;
        L.hom(s, m - 1, hk, ht, hflux, hcol);
        double b = 0.0;
        for (int t = 0; t < ne; ++t) {
            if (e[t].iface == hk) {
                const double v = L.basis_val(hk, ht, e[t].pos);
                const double rr = hflux ? -beta[t] * v * e[t].sign : v;
                b += er[t] * rr;
            } else if (e[t].iface < 0 && bc_kind[e[t].gbc] == BC_ROBIN) {
                // the homogeneous problems keep a physical Robin face's data
                // (only non-Robin values are zeroed, mrcm.cpp:166-167)
                b += er[t] * L.rb_rhs[e[t].gbc];
            }
        }
        if (anchor && r == 0) b = 0.0;
        X[xoff(L, max_rhs, s, m) + r] = b;
    }
}

// Factor the rebuild operator (stored) and solve all its right-hand sides.
__global__ void k_factor_solve(Layout L, int max_rhs, const double* __restrict__ BD, const double* __restrict__ BW,
                               const double* __restrict__ BS, double* __restrict__ D, double* __restrict__ Lc,
                               double* __restrict__ Lr, double* __restrict__ X, Scalars* sc) {
    pdl_begin();
    extern __shared__ double smem[];
    const int w = threadIdx.x >> 5;
    const int s = blockIdx.x * WPB + w;
    if (s >= L.n_sub) return;
    const int n = L.ncs, B = L.snx;
    double* sm = smem + (size_t)w * band_smem_doubles(B, RING_NR);
    const size_t so = (size_t)s * n;
    const BandRows A{BD + so, BW + so, BS + so};
    const int nr = 1 + L.n_hom(s);
    double* Xs = X + xoff(L, max_rhs, s, 0);
    const int n0 = nr < RING_NR ? nr : RING_NR;
    const bool ok = band_factor_fwd(n, B, A, D + so, Lc + so * B, Lr + so * B, Xs, n0, n, sm);
    if (!ok && (threadIdx.x & 31) == 0) atomicOr(&sc->err, ERR_PIVOT);
    for (int m0 = n0; m0 < nr; m0 += RING_NR) {
        const int cnt = nr - m0 < RING_NR ? nr - m0 : RING_NR;
        band_forward(n, B, Lc + so * B, Xs + (size_t)m0 * n, cnt, n, sm);
    }
    for (int m0 = 0; m0 < nr; m0 += RING_NR) {
        const int cnt = nr - m0 < RING_NR ? nr - m0 : RING_NR;
        band_backward(n, B, D + so, Lr + so * B, Xs + (size_t)m0 * n, cnt, n, sm);
    }
}

// Traces of every rebuild solution: outward normal velocity and face
// pressure per boundary edge (elliptic.cpp:222-240).
__global__ void k_rebuild_traces(Layout L, int max_rhs, const double* __restrict__ kappa,
                                 const int* __restrict__ bc_kind, const double* __restrict__ bc_value,
                                 const double* __restrict__ bm, const double* __restrict__ bp,
                                 const double* __restrict__ X, double* __restrict__ PU, double* __restrict__ PB,
                                 double* __restrict__ HU, double* __restrict__ HB) {
    pdl_begin();
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= L.n_sub * L.nbe) return;
    const int s = x / L.nbe, idx = x % L.nbe;
    const EdgeInfo e = L.edge(s, idx);
    const double th = half_trans(L, e.side, kappa[e.global_cell]);
    const int nh = L.n_hom(s);
    double beta = 0.0, te = 0.0;
    if (e.iface >= 0) {
        beta = edge_beta(L, e, bm, bp);
        te = eff_robin(th, beta, e.area);
    }
    for (int m = 0; m <= nh; ++m) {
        const double pc = X[xoff(L, max_rhs, s, m) + e.local_cell];
        double un, pf;
        if (e.iface >= 0) {
            double rr = 0.0;
            if (m > 0) {
                int hk, ht, hcol;
                bool hflux;
                L.hom(s, m - 1, hk, ht, hflux, hcol);
                if (e.iface == hk) {
                    const double v = L.basis_val(hk, ht, e.pos);
                    rr = hflux ? -beta * v * e.sign : v;
                }
            }
            un = te * (pc - rr) / e.area;
            pf = rr + beta * un;
        } else if (bc_kind[e.gbc] == BC_ROBIN) {  // elliptic.cpp:231-235, every m (mrcm.cpp:166-167)
            const double rb = L.rb_beta[e.gbc], rr = L.rb_rhs[e.gbc];
            un = eff_robin(th, rb, e.area) * (pc - rr) / e.area;
            pf = rr + rb * un;
        } else {
            const double val = m == 0 ? bc_value[e.gbc] : 0.0;
            if (bc_kind[e.gbc] == BC_PRESSURE) {
                un = th * (pc - val) / e.area;
                pf = val;
            } else {
                un = val;
                pf = pc - val * e.area / th;
            }
        }
        if (m == 0) {
            PU[x] = un;
            PB[x] = pf;
        } else {
            const size_t o = ((size_t)s * L.max_hom + (m - 1)) * L.nbe + idx;
            HU[o] = un;
            HB[o] = pf;
        }
    }
}

// Per-(subdomain, solution) pressure sums, one warp each.
__global__ void k_psums(Layout L, int max_rhs, const double* __restrict__ X, double* __restrict__ PS,
                        double* __restrict__ HP) {
    pdl_begin();
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (gw >= L.n_sub * max_rhs) return;
    const int s = gw / max_rhs, m = gw % max_rhs;
    if (m > L.n_hom(s)) return;
    const double* x = X + xoff(L, max_rhs, s, m);
    double v = 0.0;
    for (int r = lane; r < L.ncs; r += 32) v += x[r];
    v = warp_sum(v);
    if (lane == 0) {
        if (m == 0) PS[s] = v;
        else HP[(size_t)s * L.max_hom + m - 1] = v;
    }
}

// ---------------------------------------------------------------- K5 ----
// Interface matrix in CSR (rows: psi-rows then phi-rows; cols: U then P).
// Each entry sums the contributions of the (at most two) subdomains it
// couples through, edge by edge in the reference's order (mrcm.cpp:199-224).
__device__ __forceinline__ int hom_index(const Layout& L, int s, int col) {
    const bool flux = col < L.dim_flux;
    const int b = flux ? col : col - L.dim_flux;
    const int k = L.basis_iface(b);
    const int t = b - L.iface_first_basis(k);
    int inc[4];
    const int ni = L.incident(s, inc);
    int half = 0, before = -1, acc = 0;
    for (int a = 0; a < ni; ++a) {
        if (inc[a] == k) before = acc;
        acc += L.iface_nb(inc[a]);
        half += L.iface_nb(inc[a]);
    }
    if (before < 0) return -1;
    return (flux ? 0 : half) + before + t;
}

__global__ void k_assemble(Layout L, const int* __restrict__ rowv, const int* __restrict__ colv, int nnz,
                           const double* __restrict__ HU, const double* __restrict__ bm,
                           const double* __restrict__ bp, double* __restrict__ val) {
    pdl_begin();
    const int z = blockIdx.x * blockDim.x + threadIdx.x;  // one thread per nonzero
    if (z >= nnz) return;
    const int row = rowv[z];
    const int np = L.dim_flux;
    const bool phi = row >= np;
    const int rb = phi ? row - np : row;
    const int k = L.basis_iface(rb);
    const int rt = rb - L.iface_first_basis(k);
    const int ne = L.iface_edges(k);
    const int subs[2] = {L.iface_minus(k), L.iface_plus(k)};
    {
        const int col = colv[z];
        const bool ucol = col < L.dim_flux;
        const int cb = ucol ? col : col - L.dim_flux;
        const bool same = phi && ucol && L.basis_iface(cb) == k;
        const int ct = same ? cb - L.iface_first_basis(k) : 0;
        double acc = 0.0;
        for (int a = 0; a < 2; ++a) {
            const int s = subs[a];
            const int h = hom_index(L, s, col);
            const double sign = a == 0 ? 1.0 : -1.0;
            for (int pos = 0; pos < ne; ++pos) {
                const int idx = L.edge_index_on_iface(s, k, pos);
                const double len = k < L.NV ? L.hy : L.hx;
                const double bse = a == 0 ? bm[L.skel_index(k, pos)] : bp[L.skel_index(k, pos)];
                const double vr = L.basis_val(k, rt, pos);
                if (h >= 0) {
                    const double un = HU[((size_t)s * L.max_hom + h) * L.nbe + idx];
                    if (phi) acc += bse * un * vr * sign * len;
                    else acc += un * vr * len;
                }
                if (same) {
                    const double ub = L.basis_val(k, ct, pos);
                    acc -= bse * ub * sign * vr * sign * len;
                }
            }
        }
        val[z] = acc;
    }
}

__global__ void k_csr_to_dense(const int* __restrict__ ptr, const int* __restrict__ colv,
                               const double* __restrict__ val, int n, double* __restrict__ A) {
    pdl_begin();
    const int row = blockIdx.x;
    for (int j = threadIdx.x; j < n; j += blockDim.x) A[(size_t)row * n + j] = 0.0;
    __syncthreads();
    for (int z = ptr[row] + threadIdx.x; z < ptr[row + 1]; z += blockDim.x) A[(size_t)row * n + colv[z]] = val[z];
}

// ---------------------------------------------------------------- K6 ----
// Interface rhs from the particular traces (mrcm.cpp:80-100).
__global__ void k_iface_rhs(Layout L, const double* __restrict__ PU, const double* __restrict__ bm,
                            const double* __restrict__ bp, double* __restrict__ rhs) {
    pdl_begin();
    // one warp per row; lanes stride the (side, position) terms
    const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int np = L.dim_flux;
    if (row >= 2 * np) return;
    const bool phi = row >= np;
    const int rb = phi ? row - np : row;
    const int k = L.basis_iface(rb);
    const int rt = rb - L.iface_first_basis(k);
    const int ne = L.iface_edges(k);
    const double len = k < L.NV ? L.hy : L.hx;
    double acc = 0.0;
    for (int t = lane; t < 2 * ne; t += 32) {
        const int a = t / ne, pos = t % ne;
        {
            const int s = a == 0 ? L.iface_minus(k) : L.iface_plus(k);
            const double sign = a == 0 ? 1.0 : -1.0;
            const int idx = L.edge_index_on_iface(s, k, pos);
            const double un = PU[(size_t)s * L.nbe + idx];
            const double v = L.basis_val(k, rt, pos);
            if (phi) {
                const double beta = a == 0 ? bm[L.skel_index(k, pos)] : bp[L.skel_index(k, pos)];
                acc -= beta * un * v * sign * len;
            } else {
                acc -= un * v * len;
            }
        }
    }
    acc = warp_sum(acc);
    if (lane == 0) rhs[row] = acc;
}

// ---------------------------------------------------------------- K8 ----
// Recombined traces: recon = particular + sum_h c_h hom_h (+ w for MPM),
// in hom order, skipping zero coefficients (mrcm.cpp:270-288, mpm.cpp:93-103).
__global__ void k_recon_traces(Layout L, const double* __restrict__ coef, const double* __restrict__ PU,
                               const double* __restrict__ PB, const double* __restrict__ HU,
                               const double* __restrict__ HB, const double* __restrict__ WU,
                               double* __restrict__ RU, double* __restrict__ RB) {
    pdl_begin();
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= L.n_sub * L.nbe) return;
    const int s = x / L.nbe, idx = x % L.nbe;
    double u = PU[x], b = RB ? PB[x] : 0.0;
    const int nh = L.n_hom(s);
    for (int h = 0; h < nh; ++h) {
        int k, t, col;
        bool fl;
        L.hom(s, h, k, t, fl, col);
        const double c = coef[col];
        if (c == 0.0) continue;
        const size_t o = ((size_t)s * L.max_hom + h) * L.nbe + idx;
        u += c * HU[o];
        if (RB) b += c * HB[o];
    }
    if (WU) u += WU[x];
    RU[x] = u;
    if (RB) RB[x] = b;
}

// MPM-2P recombination, one warp per subdomain: boundary traces
// RU = PU + sum_h c_h HU_h + WU (k_recon_traces) and the pressure sum
// RS = PS + sum_h c_h HP_h + pmsum (k_recon_psum), same operation order. Lane
// h looks up the coefficient of homogeneous function h (one round trip for
// all of them) and the warp shares them by shuffle; each lane then issues
// every HU load of its edges before the sums (terms with c_h = 0 are skipped,
// as in k_recon_traces).
__global__ void __launch_bounds__(128) k_recon_mpm(Layout L, const double* __restrict__ coef,
                                                   const double* __restrict__ PU, const double* __restrict__ HU,
                                                   const double* __restrict__ WU, double* __restrict__ RU,
                                                   const double* __restrict__ PS, const double* __restrict__ HP,
                                                   const double* __restrict__ pmsum, double* __restrict__ RS) {
    pdl_begin();
    constexpr int MAXH = 16;
    const int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (s >= L.n_sub) return;
    const int nh = L.n_hom(s);
    double cl = 0.0, hp = 0.0;
    if (lane < nh) {
        int k, t, col;
        bool fl;
        L.hom(s, lane, k, t, fl, col);
        cl = coef[col];
        hp = HP[(size_t)s * L.max_hom + lane];
    }
    double ch[MAXH];
#pragma unroll
    for (int h = 0; h < MAXH; ++h) ch[h] = __shfl_sync(0xffffffffu, cl, h);
    const double* hu = HU + (size_t)s * L.max_hom * L.nbe;
    for (int i0 = 0; i0 < L.nbe; i0 += 64) {  // two edges per lane and pass
        const int ia = i0 + lane, ib = i0 + 32 + lane;
        const bool va = ia < L.nbe, vb = ib < L.nbe;
        const int ja = va ? ia : 0, jb = vb ? ib : 0;
        const size_t xa = (size_t)s * L.nbe + ja, xb = (size_t)s * L.nbe + jb;
        double ha[MAXH], hb[MAXH];
#pragma unroll
        for (int h = 0; h < MAXH; ++h) {
            ha[h] = h < nh ? hu[(size_t)h * L.nbe + ja] : 0.0;  // nh is warp-uniform
            hb[h] = h < nh ? hu[(size_t)h * L.nbe + jb] : 0.0;
        }
        double ua = PU[xa], ub = PU[xb];
        const double wa = WU ? WU[xa] : 0.0, wb = WU ? WU[xb] : 0.0;
#pragma unroll
        for (int h = 0; h < MAXH; ++h) {
            const bool on = h < nh && ch[h] != 0.0;
            ua = on ? ua + ch[h] * ha[h] : ua;
            ub = on ? ub + ch[h] * hb[h] : ub;
        }
        if (WU) {
            ua += wa;
            ub += wb;
        }
        if (va) RU[xa] = ua;
        if (vb) RU[xb] = ub;
    }
    // pressure sum: lane 0 adds the terms in order
    double v = PS[s];
#pragma unroll
    for (int h = 0; h < MAXH; ++h) {
        const double hv = __shfl_sync(0xffffffffu, hp, h);
        if (h < nh && ch[h] != 0.0) v += ch[h] * hv;
    }
    if (lane == 0) {
        if (pmsum) v += pmsum[s];
        RS[s] = v;
    }
}

__global__ void k_recon_psum(Layout L, const double* __restrict__ coef, const double* __restrict__ PS,
                             const double* __restrict__ HP, const double* __restrict__ pmsum,
                             double* __restrict__ RS) {
    pdl_begin();
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= L.n_sub) return;
    double v = PS[s];
    const int nh = L.n_hom(s);
    for (int h = 0; h < nh; ++h) {
        int k, t, col;
        bool fl;
        L.hom(s, h, k, t, fl, col);
        const double c = coef[col];
        if (c != 0.0) v += c * HP[(size_t)s * L.max_hom + h];
    }
    if (pmsum) v += pmsum[s];
    RS[s] = v;
}

// Full reconstructed pressure at a rebuild (recon_m.p, kept for MPM steps).
__global__ void k_recon_p(Layout L, int max_rhs, const double* __restrict__ coef, const double* __restrict__ X,
                          double* __restrict__ pm) {
    pdl_begin();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= L.cells()) return;
    const int i = c % L.nx, j = c / L.nx;
    const int s = (j / L.sny) * L.nsx + i / L.snx;
    const int r = (j % L.sny) * L.snx + i % L.snx;
    double v = X[xoff(L, max_rhs, s, 0) + r];
    const int nh = L.n_hom(s);
    for (int h = 0; h < nh; ++h) {
        int k, t, col;
        bool fl;
        L.hom(s, h, k, t, fl, col);
        const double cc = coef[col];
        if (cc != 0.0) v += cc * X[xoff(L, max_rhs, s, 1 + h) + r];
    }
    pm[c] = v;
}

__global__ void k_sub_sum(Layout L, const double* __restrict__ field, double* __restrict__ out) {
    pdl_begin();
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (gw >= L.n_sub) return;
    double v = 0.0;
    for (int r = lane; r < L.ncs; r += 32) v += field[L.gcell_of(gw, r)];
    v = warp_sum(v);
    if (lane == 0) out[gw] = v;
}

// ---------------------------------------------------------------- K9 ----
// Compatibility residual per subdomain, in the reference's edge order
// (mrcm.cpp:315-340), plus flux_scale = max |skeleton flux|.
__global__ void k_resid(Layout L, const double* skel, const double* __restrict__ RU,
                        const double* __restrict__ qsum, double* __restrict__ resid, Scalars* sc, double* part,
                        unsigned* counter, int fuse_skel = 0) {
    pdl_begin();
    // one warp per subdomain; lanes stride the boundary edges (W,E,S,N order)
    __shared__ double sh[32];
    const int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    double fmaxv = 0.0;
    if (s < L.n_sub) {
        double outflow = 0.0;
        for (int idx = lane; idx < L.nbe; idx += 32) {
            const EdgeInfo e = L.edge(s, idx);
            double un;
            if (e.iface >= 0) {
                double v;
                if (fuse_skel) {  // k_skel's arithmetic, written once (by the minus side) for k_ds_prep
                    const int k = e.iface, sm = L.iface_minus(k), sp = L.iface_plus(k);
                    const double um = RU[(size_t)sm * L.nbe + L.edge_index_on_iface(sm, k, e.pos)];
                    const double up = -RU[(size_t)sp * L.nbe + L.edge_index_on_iface(sp, k, e.pos)];
                    v = 0.5 * (um + up);
                    if (s == sm) const_cast<double*>(skel)[L.skel_index(k, e.pos)] = v;
                } else {
                    v = skel[L.skel_index(e.iface, e.pos)];
                }
                un = e.sign * v;
                fmaxv = fmax(fmaxv, fabs(v));
            } else {
                un = RU[(size_t)s * L.nbe + idx];
            }
            outflow += un * e.area;
        }
        outflow = warp_sum(outflow);
        if (lane == 0) resid[s] = qsum[s] - outflow;
    }
    fmaxv = block_max(fmaxv, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = fmaxv;
    if (last_block_done(counter)) {
        const double m = reduce_partials(part, gridDim.x, 1, 0, [](double a, double b) { return fmax(a, b); }, 0.0, sh);
        if (threadIdx.x == 0) {
            sc->flux_scale = m;
            *counter = 0;
        }
    }
}

// ---------------------------------------------------------------- K10 ----
// delta = Linv * resid, one warp per subdomain row; then interface corrections.
__device__ void repair_corr_last(const Layout& L, int grounded, const double* delta, const double* ground,
                                 double* corr, Scalars* sc, double* sh);

// With the last block also forming the interface corrections and the repair
// diagnostics (k_repair_corr's work, active repair only).
__global__ void k_repair_delta(int n, const double* __restrict__ Linv, const double* __restrict__ resid,
                               double* delta, Layout L, int grounded, const double* __restrict__ ground,
                               double* __restrict__ corr, Scalars* sc, unsigned* counter) {
    pdl_begin();
    __shared__ double sh[32];
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (gw < n) {
        const double* row = Linv + (size_t)gw * n;
        double v = 0.0;
        // pure-flux physical data: the pinned row's right-hand side is 0
        // (rhs[0] = 0.0, mrcm.cpp:364-367), so resid[0] does not enter
        for (int t = lane; t < n; t += 32) v += row[t] * ((grounded || t != 0) ? resid[t] : 0.0);
        v = warp_sum(v);
        if (lane == 0) delta[gw] = v;
    }
    if (last_block_done(counter)) {
        repair_corr_last(L, grounded, delta, ground, corr, sc, sh);
        if (threadIdx.x == 0) *counter = 0;
    }
}

// corr = delta_minus - delta_plus per interface; repair_max and the warning
// flag, by one block (the last of k_repair_delta), deterministic order.
__device__ void repair_corr_last(const Layout& L, int grounded, const double* delta, const double* ground,
                                 double* corr, Scalars* sc, double* sh) {
    double m = 0.0;
    for (int x = threadIdx.x; x < L.n_iface; x += blockDim.x) {
        const double cv = __ldcg(delta + L.iface_minus(x)) - __ldcg(delta + L.iface_plus(x));
        corr[x] = cv;
        m = fmax(m, fabs(cv));
    }
    if (grounded)
        for (int x = threadIdx.x; x < L.n_sub; x += blockDim.x)
            if (ground[x] > 0.0) m = fmax(m, fabs(__ldcg(delta + x)));
    m = block_max(m, sh);
    if (threadIdx.x == 0) {
        sc->repair_max = m;
        const double fs = sc->flux_scale;
        sc->repair_warning = m > 0.1 * (fs > 0 ? fs : 1.0);
    }
}

__global__ void k_repair_corr(Layout L, int active, int grounded, const double* __restrict__ delta,
                              const double* __restrict__ ground, double* __restrict__ corr, Scalars* sc, double* part,
                              unsigned* counter) {
    pdl_begin();
    __shared__ double sh[32];
    double m = 0.0;
    const int nthreads = L.n_iface > L.n_sub ? L.n_iface : L.n_sub;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < nthreads; x += gridDim.x * blockDim.x) {
        if (x < L.n_iface) {
            const double cv = active ? delta[L.iface_minus(x)] - delta[L.iface_plus(x)] : 0.0;
            corr[x] = cv;
            m = fmax(m, fabs(cv));
        }
        if (active && grounded && x < L.n_sub && ground[x] > 0.0) m = fmax(m, fabs(delta[x]));
    }
    m = block_max(m, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = m;
    if (last_block_done(counter)) {
        const double r = reduce_partials(part, gridDim.x, 1, 0, [](double a, double b) { return fmax(a, b); }, 0.0, sh);
        if (threadIdx.x == 0) {
            sc->repair_max = r;
            const double fs = sc->flux_scale;
            sc->repair_warning = r > 0.1 * (fs > 0 ? fs : 1.0);
            *counter = 0;
        }
    }
}

// ---------------------------------------------------------------- K11 ----
// Downscale operator entries (kappa_n, all Flux, anchor 0) and rhs
// (mrcm.cpp:391-411; elliptic.cpp:161-181), one thread per cell; the edge's
// imposed outward velocity is kept in EU for the velocity scatter.
__global__ void k_ds_prep(Layout L, const double* __restrict__ kappa, const double* __restrict__ T,
                          const double* __restrict__ q, const int* __restrict__ bc_kind,
                          const double* __restrict__ skel, const double* __restrict__ corr,
                          const double* __restrict__ RU, const double* __restrict__ delta, int grounded,
                          double* __restrict__ BD, double* __restrict__ BW, double* __restrict__ BS,
                          double* __restrict__ Xd, double* __restrict__ EU, Scalars* sc, int mode = 0) {
    // mode 0: operator and rhs; 1: operator only (split downscale, side
    // stream); 2: rhs only (the operator was factored on the side stream)
    pdl_begin();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= L.cells()) return;
    const int i = c % L.nx, j = c / L.nx;
    const int s = (j / L.sny) * L.nsx + i / L.snx;
    const int ii = i % L.snx, jj = j % L.sny, r = jj * L.snx + ii;
    if (mode == 1) {
        double diag = 0.0;
        if (ii > 0) diag += T[L.vface(i, j)];
        if (ii < L.snx - 1) diag += T[L.vface(i + 1, j)];
        if (jj > 0) diag += T[L.hface(i, j)];
        if (jj < L.sny - 1) diag += T[L.hface(i, j + 1)];
        const size_t o = (size_t)s * L.ncs + r;
        BD[o] = r == 0 ? 1.0 : diag;
        BW[o] = (ii > 0 && r != 1) ? T[L.vface(i, j)] : 0.0;
        BS[o] = (jj > 0 && r != L.snx) ? T[L.hface(i, j)] : 0.0;
        return;
    }
    const double kc = kappa[c];
    if (!(kc > 0.0) || !isfinite(kc)) atomicOr(&sc->err, ERR_KAPPA);
    double diag = 0.0;
    if (ii > 0) diag += T[L.vface(i, j)];
    if (ii < L.snx - 1) diag += T[L.vface(i + 1, j)];
    if (jj > 0) diag += T[L.hface(i, j)];
    if (jj < L.sny - 1) diag += T[L.hface(i, j + 1)];
    double ow = ii > 0 ? T[L.vface(i, j)] : 0.0;
    double os = jj > 0 ? T[L.hface(i, j)] : 0.0;
    double b = q[c] * L.vol();
    int idx[4];
    const int ne = cell_edges(L, ii, jj, idx);
    for (int t = 0; t < ne; ++t) {
        const EdgeInfo e = L.edge(s, idx[t]);
        double un;
        if (e.iface >= 0) {
            un = e.sign * (skel[L.skel_index(e.iface, e.pos)] + corr[e.iface]);
        } else {
            un = RU[(size_t)s * L.nbe + idx[t]];
            if (grounded && bc_kind[e.gbc] == BC_PRESSURE) un += delta[s];
        }
        EU[(size_t)s * L.nbe + idx[t]] = un;
        b -= un * e.area;
    }
    if (r == 0) {
        diag = 1.0;
        b = 0.0;
    }
    if (r == 1) ow = 0.0;
    if (r == L.snx) os = 0.0;
    const size_t o = (size_t)s * L.ncs + r;
    if (mode == 0) {
        BD[o] = diag;
        BW[o] = ow;
        BS[o] = os;
    }
    Xd[o] = b;
}

// The downscale right-hand side alone (k_ds_prep mode 2's output, for the
// paths whose operator is formed elsewhere: the split factor, the blocked
// factor from T), in two kernels. k_ds_edges: per subdomain-boundary edge,
// the imposed outward flux (skeleton average + interface correction, or the
// recon trace + the grounded delta) into EU (kept for the scatter) and ET.
// k_ds_rhs: per cell q vol minus its edges' un * area in W, E, S, N order,
// anchor row 0 (the same arithmetic as k_ds_prep).
__global__ void __launch_bounds__(256) k_ds_edges(Layout L, const int* __restrict__ bc_kind,
                                                  const double* __restrict__ skel, const double* __restrict__ corr,
                                                  const double* __restrict__ RU, const double* __restrict__ delta,
                                                  int grounded, double* __restrict__ EU, double* __restrict__ ET) {
    pdl_begin();
    const int ne = L.n_sub * L.nbe;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < ne; x += gridDim.x * blockDim.x) {
        const int s = x / L.nbe, idx = x % L.nbe;
        const EdgeInfo e = L.edge(s, idx);
        double un;
        if (e.iface >= 0) {
            un = e.sign * (skel[L.skel_index(e.iface, e.pos)] + corr[e.iface]);
        } else {
            un = RU[x];
            if (grounded && bc_kind[e.gbc] == BC_PRESSURE) un += delta[s];
        }
        EU[x] = un;
        ET[x] = un;
    }
}

// kappa (nullable) is checked as k_ds_prep does when it did not come from
// the driver's k_kappa
__global__ void __launch_bounds__(256) k_ds_rhs(Layout L, const double* __restrict__ kappa,
                                                const double* __restrict__ q, const double* __restrict__ ET,
                                                double* __restrict__ Xd, Scalars* sc) {
    pdl_begin();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;  // 2-D grid as k_ds_u_div
    if (i >= L.nx) return;
    const int sx = i / L.snx, ii = i - sx * L.snx;
    for (int j = blockIdx.y; j < L.ny; j += gridDim.y) {
        const int sy = j / L.sny, jj = j - sy * L.sny;
        const int c = j * L.nx + i;
        const int s = sy * L.nsx + sx, r = jj * L.snx + ii;
        const size_t eo = (size_t)s * L.nbe;
        const bool bw = ii == 0, be = ii == L.snx - 1, bs = jj == 0, bn = jj == L.sny - 1;
        const double qc = q[c];
        const double tw = bw ? ET[eo + jj] : 0.0, te = be ? ET[eo + L.sny + jj] : 0.0;
        const double ts = bs ? ET[eo + 2 * L.sny + ii] : 0.0, tn = bn ? ET[eo + 2 * L.sny + L.snx + ii] : 0.0;
        if (kappa) {
            const double kc = kappa[c];
            if (!(kc > 0.0) || !isfinite(kc)) atomicOr(&sc->err, ERR_KAPPA);
        }
        double b = qc * L.vol();  // b -= un * area, contracted as in k_ds_prep
        if (bw) b = fma(-tw, L.hy, b);
        if (be) b = fma(-te, L.hy, b);
        if (bs) b = fma(-ts, L.hx, b);
        if (bn) b = fma(-tn, L.hx, b);
        if (r == 0) b = 0.0;
        Xd[(size_t)s * L.ncs + r] = b;
    }
}

// Fresh factorization + solve per subdomain; mean shift to the recon mean
// (mrcm.cpp:409-424). x (unshifted) stays in Xd for the velocity scatter.
__global__ void k_ds_solve(Layout L, const double* __restrict__ BD, const double* __restrict__ BW,
                           const double* __restrict__ BS, double* __restrict__ D, double* __restrict__ Lr,
                           double* __restrict__ Xd, const double* __restrict__ RS, double* __restrict__ p,
                           Scalars* sc) {
    pdl_begin();
    extern __shared__ double smem[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = blockIdx.x * WPB + w;
    if (s >= L.n_sub) return;
    const int n = L.ncs, B = L.snx;
    double* sm = smem + (size_t)w * band_smem_doubles(B, 1);
    const size_t so = (size_t)s * n;
    const BandRows A{BD + so, BW + so, BS + so};
    double* x = Xd + so;
    const bool ok = band_factor_fwd(n, B, A, D + so, nullptr, Lr + so * B, x, 1, n, sm);
    if (!ok && lane == 0) atomicOr(&sc->err, ERR_PIVOT);
    band_backward(n, B, D + so, Lr + so * B, x, 1, n, sm);
    __syncwarp();
    double v = 0.0;
    for (int r = lane; r < n; r += 32) v += x[r];
    v = warp_sum(v);
    const double shift = (__shfl_sync(0xffffffffu, RS[s], 0) - __shfl_sync(0xffffffffu, v, 0)) / n;
    for (int r = lane; r < n; r += 32) p[L.gcell_of(s, r)] = x[r] + shift;
}

// Register-window variants (band_reg.cuh) for the common subdomain widths.
template <int B>
__global__ void __launch_bounds__(WPB * 32, 4) k_ds_solve_r(Layout L, const double* __restrict__ BD,
                                                         const double* __restrict__ BW, const double* __restrict__ BS,
                                                         double* D, double* Lr,
                                                         double* Xd, const double* __restrict__ RS,
                                                         double* p, Scalars* sc) {
    pdl_begin();
    __shared__ double stage[WPB][B * B];
    __shared__ __align__(16) double xbuf[WPB][xchg_doubles<B, 1>()];
    __shared__ __align__(16) double ring[WPB][sweep_ring<B>() * B * B + 2];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = blockIdx.x * WPB + w;
    if (s >= L.n_sub) return;
    const int n = L.ncs;
    const size_t so = (size_t)s * n;
    const BandRows A{BD + so, BW + so, BS + so};
    double* x = Xd + so;
    const bool ok = factor_fwd_reg<B, 1>(n, A, D + so, nullptr, Lr + so * B, x, 1, n, stage[w], xbuf[w]);
    if (!ok && lane == 0) atomicOr(&sc->err, ERR_PIVOT);
    __syncwarp();
    backward_reg<B, 1>(n, D + so, Lr + so * B, x, 1, n, xbuf[w], ring[w]);
    __syncwarp();
    double v = 0.0;
    for (int r = lane; r < n; r += 32) v += x[r];
    v = warp_sum(v);
    const double shift = (__shfl_sync(0xffffffffu, RS[s], 0) - __shfl_sync(0xffffffffu, v, 0)) / n;
    for (int r = lane; r < n; r += 32) p[L.gcell_of(s, r)] = x[r] + shift;
}

// Downscale on the fp64 tensor cores (band_blk.cuh), two kernels: the
// blocked LDL^T with DMMA Schur updates and the forward sweep (X panels in
// Lr, t1 in D; register-heavy, latency-bound), then the backward sweep from
// the stored panels with the mean shift (few registers, full occupancy,
// bandwidth-bound on the panel stream). Four blocks per SM below B = 32
// (tools/blk_bench at 16,384 subdomains: B = 16 298 against 337 us, B = 24 759
// against 818 us; B = 32 1,873 against 1,799 us, so three there).
template <int B>
__global__ void __launch_bounds__(WPB * 32, B < 32 ? 4 : 3) k_ds_blk_factor(Layout L, const double* __restrict__ T,
                                                            double* T1, double* Xs, const double* Xd, Scalars* sc) {
    pdl_begin();
    __shared__ __align__(16) double sm[WPB][blk_smem_doubles<B>()];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = blockIdx.x * WPB + w;
    if (s >= L.n_sub) return;
    const int n = L.ncs;
    const size_t so = (size_t)s * n;
    // the operator straight from T(kappa_n): k_ds_prep writes only the rhs
    const BlkTransSrc<B> src{T, Xd + so, n, L.sny, L.nx, L.vcount(), L.sub_i0(s), L.sub_j0(s)};
    const bool ok = blk_factor_fwd<B>(n, src, Xs + so * B, T1 + so, sm[w]);
    if (!ok && lane == 0) atomicOr(&sc->err, ERR_PIVOT);
}

// The blocked factor alone (no right-hand side), with the pivot inverses
// stored: with few subdomains per SM it runs on the side stream concurrently
// with the particular / interface chain (ds_factor_fork), and the sweeps
// follow the join (k_ds_blk_sweeps).
template <int B>
__global__ void __launch_bounds__(WPB * 32, B < 32 ? 4 : 3) k_ds_blk_factor_only(Layout L, const double* __restrict__ T,
                                                                              double* Xs, double* Gs, Scalars* sc) {
    pdl_begin();
    __shared__ __align__(16) double sm[WPB][blk_smem_doubles<B>()];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = blockIdx.x * WPB + w;
    if (s >= L.n_sub) return;
    const int n = L.ncs;
    const size_t so = (size_t)s * n;
    const BlkTransSrc<B> src{T, nullptr, n, L.sny, L.nx, L.vcount(), L.sub_i0(s), L.sub_j0(s)};
    const bool ok = blk_factor_fwd<B, BlkTransSrc<B>, false, false>(n, src, Xs + so * B, nullptr, sm[w], Gs + so * 8);
    if (!ok && lane == 0) atomicOr(&sc->err, ERR_PIVOT);
}

// Forward and backward sweeps from the stored panels and pivot inverses, then
// the mean shift (k_ds_blk_solve's epilogue).
template <int B>
__global__ void __launch_bounds__(WPB * 32) k_ds_blk_sweeps(Layout L, double* T1, const double* __restrict__ Xs,
                                                            const double* __restrict__ Gs, double* Xd,
                                                            const double* __restrict__ RS, double* p) {
    pdl_begin();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = blockIdx.x * WPB + w;
    if (s >= L.n_sub) return;
    const int n = L.ncs;
    const size_t so = (size_t)s * n;
    double* x = Xd + so;
    blk_forward<B>(n, Xs + so * B, Gs + so * 8, x, T1 + so);
    __syncwarp();  // t1 written by the row lanes, read by the column lanes
    const double part = blk_backward<B>(n, Xs + so * B, T1 + so, x);
    __syncwarp();
    const double v = warp_sum(part);
    const double shift = (__shfl_sync(0xffffffffu, RS[s], 0) - __shfl_sync(0xffffffffu, v, 0)) / n;
    for (int r = lane; r < n; r += 32) p[L.gcell_of(s, r)] = x[r] + shift;
}

template <int B>
__global__ void __launch_bounds__(WPB * 32) k_ds_blk_solve(Layout L, const double* __restrict__ T1,
                                                           const double* __restrict__ Xs, double* Xd,
                                                           const double* __restrict__ RS, double* p) {
    pdl_begin();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = blockIdx.x * WPB + w;
    if (s >= L.n_sub) return;
    const int n = L.ncs;
    const size_t so = (size_t)s * n;
    double* x = Xd + so;
    const double part = blk_backward<B>(n, Xs + so * B, T1 + so, x);
    __syncwarp();
    const double v = warp_sum(part);
    const double shift = (__shfl_sync(0xffffffffu, RS[s], 0) - __shfl_sync(0xffffffffu, v, 0)) / n;
    for (int r = lane; r < n; r += 32) p[L.gcell_of(s, r)] = x[r] + shift;
}

// Outward normal velocity of the particular solution on boundary edge idx of
// subdomain s (the k_part_traces formula, mpm.cpp:86-96).
__device__ __forceinline__ double part_trace(const Layout& L, int s, int idx, double pc, const double* km,
                                             const int* bc_kind, const double* bm, const double* bp,
                                             const double* GZ) {
    const EdgeInfo e = L.edge(s, idx);
    const double th = half_trans(L, e.side, km[e.global_cell]);
    const size_t x = (size_t)s * L.nbe + idx;
    if (e.iface >= 0) {
        const double te = eff_robin(th, edge_beta(L, e, bm, bp), e.area);
        return te * (pc - 0.0) / e.area;
    }
    if (bc_kind[e.gbc] == BC_PRESSURE) return th * (pc - GZ[x]) / e.area;
    if (bc_kind[e.gbc] == BC_ROBIN) return eff_robin(th, L.rb_beta[e.gbc], e.area) * (pc - GZ[x]) / e.area;
    return GZ[x];
}

// MPM-2P particular solve with the cached factor, then (same warp, same
// subdomain) its boundary traces PU and pressure sum PS — the work of
// k_part_traces / k_part_psum without two more launches.
template <int B>
__global__ void __launch_bounds__(WPB * 32) k_part_solve_r(Layout L, int max_rhs, const double* __restrict__ D,
                                                           const double* __restrict__ Lc,
                                                           const double* __restrict__ Lr, double* X,
                                                           const double* __restrict__ km,
                                                           const int* __restrict__ bc_kind,
                                                           const double* __restrict__ bm,
                                                           const double* __restrict__ bp,
                                                           const double* __restrict__ GZ, double* __restrict__ PU,
                                                           double* __restrict__ PS) {
    pdl_begin();
    __shared__ __align__(16) double ring[WPB][sweep_ring<B>() * B * B + 2];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = blockIdx.x * WPB + w;
    if (s >= L.n_sub) return;
    const int n = L.ncs;
    const size_t so = (size_t)s * n;
    double* x = X + xoff(L, max_rhs, s, 0);
    forward_reg<B, 1>(n, Lc + so * B, x, 1, n, nullptr, ring[w]);
    __syncwarp();
    backward_reg<B, 1>(n, D + so, Lr + so * B, x, 1, n, nullptr, ring[w]);
    __syncwarp();  // x written by the pivot lanes is read by all lanes below
    for (int idx = lane; idx < L.nbe; idx += 32) {
        const EdgeInfo e = L.edge(s, idx);
        PU[(size_t)s * L.nbe + idx] = part_trace(L, s, idx, x[e.local_cell], km, bc_kind, bm, bp, GZ);
    }
    double v = 0.0;
    for (int r = lane; r < n; r += 32) v += x[r];
    v = warp_sum(v);
    if (lane == 0) PS[s] = v;
}

// Rebuild, split for parallelism: k_factor1_r factors each subdomain operator
// with only the particular right-hand side carried through the (sequential)
// elimination, then k_hom_solve_r solves the homogeneous right-hand sides with
// the stored factor, one warp per (subdomain, function) — 8x more warps than
// carrying all of them through the factorisation, same arithmetic per RHS.
template <int B>
__global__ void __launch_bounds__(WPB * 32) k_factor1_r(Layout L, int max_rhs, const double* __restrict__ BD,
                                                        const double* __restrict__ BW, const double* __restrict__ BS,
                                                        double* D, double* Lc, double* Lr, double* X, Scalars* sc) {
    pdl_begin();
    __shared__ double stage[WPB][B * B];
    __shared__ __align__(16) double xbuf[WPB][xchg_doubles<B, 1>()];
    __shared__ __align__(16) double ring[WPB][sweep_ring<B>() * B * B + 2];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = blockIdx.x * WPB + w;
    if (s >= L.n_sub) return;
    const int n = L.ncs;
    const size_t so = (size_t)s * n;
    const BandRows A{BD + so, BW + so, BS + so};
    double* x = X + xoff(L, max_rhs, s, 0);
    const bool ok = factor_fwd_reg<B, 1>(n, A, D + so, Lc + so * B, Lr + so * B, x, 1, n, stage[w], xbuf[w]);
    if (!ok && lane == 0) atomicOr(&sc->err, ERR_PIVOT);
    __syncwarp();
    backward_reg<B, 1>(n, D + so, Lr + so * B, x, 1, n, nullptr, ring[w]);
}

template <int B>
__global__ void __launch_bounds__(WPB * 32) k_hom_solve_r(Layout L, int max_rhs, const double* __restrict__ D,
                                                          const double* __restrict__ Lc,
                                                          const double* __restrict__ Lr, double* X) {
    pdl_begin();
    __shared__ __align__(16) double ring[WPB][sweep_ring<B>() * B * B + 2];
    const int w = threadIdx.x >> 5;
    const int gw = blockIdx.x * WPB + w;
    const int s = gw / L.max_hom, h = gw % L.max_hom;
    if (s >= L.n_sub || h >= L.n_hom(s)) return;
    const int n = L.ncs;
    const size_t so = (size_t)s * n;
    double* x = X + xoff(L, max_rhs, s, 1 + h);
    forward_reg<B, 1>(n, Lc + so * B, x, 1, n, nullptr, ring[w]);
    __syncwarp();
    backward_reg<B, 1>(n, D + so, Lr + so * B, x, 1, n, nullptr, ring[w]);
}

// Homogeneous solves, HR right-hand sides per warp: one warp per (subdomain,
// group of HR functions) streams the subdomain's stored factor once for the
// whole group (the single-RHS kernel above streams it once per function).
// Per function the arithmetic and its order are those of k_hom_solve_r, so
// the solutions are bit-identical.
template <int B, int HR>
__global__ void __launch_bounds__(WPB * 32) k_hom_solve_rm(Layout L, int max_rhs, int groups,
                                                           const double* __restrict__ D,
                                                           const double* __restrict__ Lc,
                                                           const double* __restrict__ Lr, double* X) {
    pdl_begin();
    __shared__ __align__(16) double ring[WPB][sweep_ring<B>() * B * B + 2];
    __shared__ __align__(16) double xb[WPB][2 * xchg_ys<HR>()];
    const int w = threadIdx.x >> 5;
    const int gw = blockIdx.x * WPB + w;
    const int s = gw / groups, h0 = (gw % groups) * HR;
    if (s >= L.n_sub) return;
    const int nh = L.n_hom(s) - h0;
    if (nh <= 0) return;
    const int nr = nh < HR ? nh : HR;
    const int n = L.ncs;
    const size_t so = (size_t)s * n;
    double* x = X + xoff(L, max_rhs, s, 1 + h0);
    forward_reg<B, HR>(n, Lc + so * B, x, nr, n, xb[w], ring[w]);
    __syncwarp();
    backward_reg<B, HR>(n, D + so, Lr + so * B, x, nr, n, xb[w], ring[w]);
}

// Two-sided band kernels (band_twist.cuh): one team per block — one warp
// (two half-warps) for B <= 16, two warps for B > 16 — dynamic shared memory
// twist_smem_doubles<B>() doubles.
template <int B>
constexpr size_t twist_smem_bytes() {  // dynamic part (two-warp teams only)
    return twist_warps<B>() ? (size_t)twist_smem_doubles<B>() * sizeof(double) : 0;
}

// Downscale solve with the two-sided elimination: the two halves factor from
// both ends, so the dependent chain is ~half as long.
template <int B>
__global__ void __launch_bounds__(twist_threads<B>()) k_ds_solve_t(Layout L, const double* __restrict__ BD,
                                                                   const double* __restrict__ BW,
                                                                   const double* __restrict__ BS, double* D, double* Lr,
                                                                   double* Xd, const double* __restrict__ RS,
                                                                   double* p, Scalars* sc) {
    pdl_begin();
    double* tsm;  // static shared memory for one-warp teams (faster code), dynamic for two-warp teams
    if constexpr (twist_warps<B>()) {
        extern __shared__ __align__(16) double tsm_dyn[];
        tsm = tsm_dyn;
    } else {
        __shared__ __align__(16) double tsm_st[twist_smem_doubles<B>()];
        tsm = tsm_st;
    }
    const int lane = threadIdx.x & 31;
    const int s = blockIdx.x;
    if (s >= L.n_sub) return;
    const int n = L.ncs;
    const size_t so = (size_t)s * n;
    const BandRows A{BD + so, BW + so, BS + so};
    double* x = Xd + so;
    const bool ok = twisted_solve<B>(n, A, D + so, Lr + so * B, x, tsm);
    if (threadIdx.x >= 32) return;  // epilogue on warp 0
    if (!ok && lane == 0) atomicOr(&sc->err, ERR_PIVOT);
    // mean shift (mrcm.cpp:430-437): all loads of x first, then the scatter
    constexpr int PER = 8;
    double v = 0.0;
    const double rs = RS[s];
    for (int r0 = 0; r0 < n; r0 += 32 * PER) {
        double xv[PER];
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int r = r0 + lane + 32 * q;
            xv[q] = r < n ? __ldcg(x + r) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < PER; ++q) v += xv[q];
    }
    v = warp_sum(v);
    const double shift = (rs - __shfl_sync(0xffffffffu, v, 0)) / n;
    for (int r0 = 0; r0 < n; r0 += 32 * PER) {
        double xv[PER];
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int r = r0 + lane + 32 * q;
            xv[q] = r < n ? __ldcg(x + r) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int r = r0 + lane + 32 * q;
            if (r < n) p[L.gcell_of(s, r)] = xv[q] + shift;
        }
    }
}
#define MPM2P_TWIST_WIDTHS(X) X(4) X(8) X(10) X(12) X(16) X(20) X(24) X(32)

// Split downscale, critical-path half: the two sweeps with the kappa_n factor
// stored by k_factor1_t on the side stream, then k_ds_solve_t's mean shift
// (mrcm.cpp:414-424) and scatter.
template <int B>
__global__ void __launch_bounds__(twist_threads<B>()) k_ds_sweep_t(Layout L, const double* __restrict__ D,
                                                                   const double* __restrict__ Lc,
                                                                   const double* __restrict__ Lr,
                                                                   const double* __restrict__ MidB,
                                                                   const double* __restrict__ Sinv, double* Xd,
                                                                   const double* __restrict__ RS, double* p) {
    pdl_begin();
    double* tsm;
    if constexpr (twist_warps<B>()) {
        extern __shared__ __align__(16) double tsm_dyn[];
        tsm = tsm_dyn;
    } else {
        __shared__ __align__(16) double tsm_st[twist_smem_doubles<B>()];
        tsm = tsm_st;
    }
    const int lane = threadIdx.x & 31;
    const int s = blockIdx.x;
    if (s >= L.n_sub) return;
    const int n = L.ncs;
    const size_t so = (size_t)s * n;
    double* x = Xd + so;
    const double rs = RS[s];  // before the sweep: off the chain
    twisted_sweep<B>(n, D + so, Lc + so * B, Lr + so * B, MidB + (size_t)s * B * B, Sinv + (size_t)s * B * B, x, tsm);
    if (threadIdx.x >= 32) return;
    constexpr int PER = 8;
    double v = 0.0;
    for (int r0 = 0; r0 < n; r0 += 32 * PER) {
        double xv[PER];
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int r = r0 + lane + 32 * q;
            xv[q] = r < n ? __ldcg(x + r) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < PER; ++q) v += xv[q];
    }
    v = warp_sum(v);
    const double shift = (rs - __shfl_sync(0xffffffffu, v, 0)) / n;
    for (int r0 = 0; r0 < n; r0 += 32 * PER) {
        double xv[PER];
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int r = r0 + lane + 32 * q;
            xv[q] = r < n ? __ldcg(x + r) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int r = r0 + lane + 32 * q;
            if (r < n) p[L.gcell_of(s, r)] = xv[q] + shift;
        }
    }
}

// Rebuild with the two-sided scheme: the factor (twisted layout + the middle
// block's S^-1 and bottom multipliers) and the particular solve...
template <int B>
__global__ void __launch_bounds__(twist_threads<B>()) k_factor1_t(Layout L, int max_rhs, const double* __restrict__ BD,
                                                                  const double* __restrict__ BW,
                                                                  const double* __restrict__ BS, double* D, double* Lc,
                                                                  double* Lr, double* MidB, double* Sinv, double* X,
                                                                  Scalars* sc) {
    pdl_begin();
    double* tsm;  // static shared memory for one-warp teams (faster code), dynamic for two-warp teams
    if constexpr (twist_warps<B>()) {
        extern __shared__ __align__(16) double tsm_dyn[];
        tsm = tsm_dyn;
    } else {
        __shared__ __align__(16) double tsm_st[twist_smem_doubles<B>()];
        tsm = tsm_st;
    }
    const int s = blockIdx.x;
    if (s >= L.n_sub) return;
    const int n = L.ncs;
    const size_t so = (size_t)s * n;
    const BandRows A{BD + so, BW + so, BS + so};
    const bool ok = twisted_factor<B>(n, A, D + so, Lc + so * B, Lr + so * B, MidB + (size_t)s * B * B,
                                      Sinv + (size_t)s * B * B, X + xoff(L, max_rhs, s, 0), tsm);
    if (!ok && threadIdx.x == 0) atomicOr(&sc->err, ERR_PIVOT);
}

// ... then one team per (subdomain, homogeneous function) with the stored factor.
template <int B>
__global__ void __launch_bounds__(twist_threads<B>()) k_hom_solve_t(Layout L, int max_rhs, const double* __restrict__ D,
                                                                    const double* __restrict__ Lc,
                                                                    const double* __restrict__ Lr,
                                                                    const double* __restrict__ MidB,
                                                                    const double* __restrict__ Sinv, double* X) {
    pdl_begin();
    double* tsm;  // static shared memory for one-warp teams (faster code), dynamic for two-warp teams
    if constexpr (twist_warps<B>()) {
        extern __shared__ __align__(16) double tsm_dyn[];
        tsm = tsm_dyn;
    } else {
        __shared__ __align__(16) double tsm_st[twist_smem_doubles<B>()];
        tsm = tsm_st;
    }
    const int gw = blockIdx.x;
    const int s = gw / L.max_hom, h = gw % L.max_hom;
    if (s >= L.n_sub || h >= L.n_hom(s)) return;
    const int n = L.ncs;
    const size_t so = (size_t)s * n;
    twisted_sweep<B>(n, D + so, Lc + so * B, Lr + so * B, MidB + (size_t)s * B * B, Sinv + (size_t)s * B * B,
                     X + xoff(L, max_rhs, s, 1 + h), tsm);
}

// MPM-2P particular solve with the stored two-sided factor + traces + psum.
template <int B>
__global__ void __launch_bounds__(twist_threads<B>()) k_part_solve_t(Layout L, int max_rhs, const double* __restrict__ D,
                                                                     const double* __restrict__ Lc,
                                                                     const double* __restrict__ Lr,
                                                                     const double* __restrict__ MidB,
                                                                     const double* __restrict__ Sinv, double* X,
                                                                     const double* __restrict__ km,
                                                                     const int* __restrict__ bc_kind,
                                                                     const double* __restrict__ bm,
                                                                     const double* __restrict__ bp,
                                                                     const double* __restrict__ GZ,
                                                                     double* __restrict__ PU, double* __restrict__ PS) {
    pdl_begin();
    double* tsm;  // static shared memory for one-warp teams (faster code), dynamic for two-warp teams
    if constexpr (twist_warps<B>()) {
        extern __shared__ __align__(16) double tsm_dyn[];
        tsm = tsm_dyn;
    } else {
        __shared__ __align__(16) double tsm_st[twist_smem_doubles<B>()];
        tsm = tsm_st;
    }
    const int lane = threadIdx.x & 31;
    const int s = blockIdx.x;
    if (s >= L.n_sub) return;
    const int n = L.ncs;
    const size_t so = (size_t)s * n;
    double* x = X + xoff(L, max_rhs, s, 0);
    twisted_sweep<B>(n, D + so, Lc + so * B, Lr + so * B, MidB + (size_t)s * B * B, Sinv + (size_t)s * B * B, x, tsm);
    if (threadIdx.x >= 32) return;  // epilogue on warp 0
    for (int idx = lane; idx < L.nbe; idx += 32) {
        const EdgeInfo e = L.edge(s, idx);
        PU[(size_t)s * L.nbe + idx] = part_trace(L, s, idx, x[e.local_cell], km, bc_kind, bm, bp, GZ);
    }
    double v = 0.0;
    for (int r = lane; r < n; r += 32) v += x[r];
    v = warp_sum(v);
    if (lane == 0) PS[s] = v;
}

// Dynamic shared memory opt-in for each instantiation (once, outside capture).
template <int B>
void twist_configure() {
    static DeviceCache done;  // per device
    if (done.at().load() > 0 || !twist_warps<B>()) return;
    const int bytes = (int)twist_smem_bytes<B>();
    CK(cudaFuncSetAttribute(k_ds_solve_t<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    CK(cudaFuncSetAttribute(k_factor1_t<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    CK(cudaFuncSetAttribute(k_hom_solve_t<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    CK(cudaFuncSetAttribute(k_part_solve_t<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    CK(cudaFuncSetAttribute(k_ds_sweep_t<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done.at().store(1);
}

// Subdomain widths with a register-window instantiation; others use band.cuh.
#define MPM2P_BAND_WIDTHS(X) X(4) X(8) X(10) X(12) X(16) X(20) X(24) X(32)


// max_c |div u - q| and max(|q|, |u_f| area / vol) (mrcm.cpp:429-437).
// Velocity scatter + divergence residual (+ outlet probe) in one pass: each
// cell evaluates its four face velocities with k_ds_u's formulas (interior
// faces from the unshifted local pressure Xd, subdomain-edge faces from the
// imposed outward velocity EU), writes the faces it owns (west, south, and
// the east / north domain boundary), and feeds k_divres's reductions with the
// same face values.
//
// With cfl.on it also takes the NEXT step's cfl_timestep + injection_rate
// (transport.cpp:51-71, simulation.cpp:85-101) from the same face values, so
// the step needs no separate k_cfl pass: dt_next / any_next / inj_next are
// promoted by the first upwind sub-step (k_upwind take_next). The CFL terms
// use explicitly rounded operations (no FMA contraction) in k_cfl's order,
// so dt is bit-identical to the separate reduction.
struct CflNext {
    int on = 0;
    double safety = 0.0, dt_cap = 0.0, inflow = 0.0, M = 1.0;
};
// Block and grid reduction of k_ds_u_div's six maxima and the scalars formed
// from them (div_residual, div_scale, the next step's dt).
__device__ __forceinline__ void udiv_finish(const Layout& L, double res, double vmax, double hmax, double qmax,
                                            double dmax, double anyf, Scalars* sc, double* part, unsigned* counter,
                                            const CflNext& cfl) {
    constexpr int NP = 6;
    const double vol = L.vol(), hx = L.hx, hy = L.hy;
    __shared__ double shm[32 * NP];
    __shared__ double red[NP];
    double v[NP] = {res, vmax, hmax, qmax, dmax, anyf};
    block_reduce_multi<NP>(v, 0u, shm, red);
    if (threadIdx.x < NP) part[NP * (blockIdx.y * gridDim.x + blockIdx.x) + threadIdx.x] = red[threadIdx.x];
    if (last_block_done(counter)) {
        double a[NP];
#pragma unroll
        for (int k = 0; k < NP; ++k) a[k] = 0.0;
        for (int b = threadIdx.x; b < (int)(gridDim.x * gridDim.y); b += blockDim.x) {
#pragma unroll
            for (int k = 0; k < NP; ++k) a[k] = fmax(a[k], __ldcg(part + (size_t)NP * b + k));
        }
        block_reduce_multi<NP>(a, 0u, shm, red);
        if (threadIdx.x == 0) {
            sc->div_residual = red[0];
            // max(|q|, |u_f| area_f / vol) (mrcm.cpp:432-437)
            const double scale = fmax(fmax(red[3], __ddiv_rn(__dmul_rn(red[1], hy), vol)),
                                      __ddiv_rn(__dmul_rn(red[2], hx), vol));
            sc->div_scale = scale > 0.0 ? scale : 1.0;
            if (cfl.on) {  // cfl_timestep's epilogue (transport.cpp:55-70), for the next step
                const bool af = red[5] > 0.0;
                const double dt = af ? fmin(cfl.dt_cap / cfl.safety, __ddiv_rn(vol, red[4])) : 0.0;
                sc->any_next = af;
                sc->dt_next = af ? fmin(cfl.safety * dt, cfl.dt_cap) : cfl.dt_cap;
            }
            *counter = 0;
        }
    }
}

// Velocity scatter of the downscaled solution (mrcm.cpp:409-431) with the
// divergence residual and scale (mrcm.cpp:429-437) and the next step's CFL
// reduction (cfl_timestep, transport.cpp:51-71) in the same pass. One thread
// per cell, warps over 32 consecutive cells of a row, every load of a cell
// issued before its arithmetic (one memory round trip per iteration). Each
// face velocity is one division: the east face of a cell is the west face
// of the next lane's cell (shuffle; computed directly only by lane 31 and on
// the east boundary). The divisions of the maxima are pulled out of them
// (correctly rounded multiplication and division are monotone):
// max_f fl(fl(|u_f| h) / vol) = fl(fl(max_f |u_f| h) / vol) per face
// orientation, and cfl_timestep's min_c fl(vol / d_c) = fl(vol / max_c d_c)
// for d_c = fl(outflux_c slope) > 0 — bit-identical to the per-face form.
// The boundary-face work (injection rate, outlet probe) is k_bnd_probe's.
// Slots: res, vmax, hmax, qmax, dmax, any.
__global__ void __launch_bounds__(256, 4) k_ds_u_div(Layout L, const double* __restrict__ T,
                                                  const double* __restrict__ Xd, const double* __restrict__ EU,
                                                  double* __restrict__ u, const double* __restrict__ q, Scalars* sc,
                                                  double* part, unsigned* counter, CflNext cfl) {
    pdl_begin();
    const int lane = threadIdx.x & 31;
    double res = 0.0, vmax = 0.0, hmax = 0.0, qmax = 0.0, dmax = 0.0, anyf = 0.0;
    const double vol = L.vol(), hx = L.hx, hy = L.hy;
    const double slope = cfl.on ? sc->slope : 1.0;
    // 2-D grid: blockIdx.x over 256-column strips (warps = 32 consecutive
    // cells of a row), rows strided by blockIdx.y: the column's subdomain
    // index math once per thread, the row's once per row (block-uniform)
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = i < L.nx;
    const int ic = valid ? i : L.nx - 1;
    const int sx = ic / L.snx, ii = ic - sx * L.snx;
    for (int j = blockIdx.y; j < L.ny; j += gridDim.y) {
        const int sy = j / L.sny, jj = j - sy * L.sny;
        const int cc = j * L.nx + ic;
        const int s = sy * L.nsx + sx;
        const size_t xo = (size_t)s * L.ncs;
        const int r = jj * L.snx + ii;
        const size_t eo = (size_t)s * L.nbe;
        const bool de = lane == 31 || i + 1 >= L.nx;  // east face not held by lane + 1
        const bool hw = ii > 0, he = ii + 1 < L.snx, hs = jj > 0, hn = jj + 1 < L.sny;
        const double xc = Xd[xo + r];
        const double xw = hw ? Xd[xo + r - 1] : 0.0;
        const double tw = hw ? T[L.vface(ic, j)] : 0.0;
        const double ew = hw ? 0.0 : EU[eo + jj];
        const double xe = (de && he) ? Xd[xo + r + 1] : 0.0;
        const double te = (de && he) ? T[L.vface(ic + 1, j)] : 0.0;
        // east face on a subdomain edge: the west edge of the subdomain to the east, or the domain boundary
        const double ee = (de && !he) ? (ic + 1 < L.nx ? -EU[eo + L.nbe + jj] : EU[eo + L.sny + jj]) : 0.0;
        const double xs = hs ? Xd[xo + r - L.snx] : 0.0;
        const double ts = hs ? T[L.hface(ic, j)] : 0.0;
        const double es = hs ? 0.0 : EU[eo + 2 * L.sny + ii];
        const double xn = hn ? Xd[xo + r + L.snx] : 0.0;
        const double tn = hn ? T[L.hface(ic, j + 1)] : 0.0;
        // north face on a subdomain edge: the south edge of the one above, or the domain boundary
        const double en = hn ? 0.0 : (j + 1 < L.ny ? -EU[(size_t)(s + L.nsx) * L.nbe + 2 * L.sny + ii]
                                                   : EU[eo + 2 * L.sny + L.snx + ii]);
        const double qc = q[cc];
        const double uW = hw ? L.div_hy(tw * (xw - xc)) : -ew;
        double uE = __shfl_down_sync(0xffffffffu, uW, 1);
        if (de) uE = he ? L.div_hy(te * (xc - xe)) : ee;
        if (!valid) continue;
        const double uS = hs ? L.div_hx(ts * (xs - xc)) : -es;
        const double uN = hn ? L.div_hx(tn * (xc - xn)) : en;
        u[L.vface(i, j)] = uW;
        u[L.hface(i, j)] = uS;
        vmax = fmax(vmax, fabs(uW));
        hmax = fmax(hmax, fabs(uS));
        if (i == L.nx - 1) {
            u[L.vface(i + 1, j)] = uE;
            vmax = fmax(vmax, fabs(uE));
        }
        if (j == L.ny - 1) {
            u[L.hface(i, j + 1)] = uN;
            hmax = fmax(hmax, fabs(uN));
        }
        // divergence(u) - q (grid.cpp:19-31), unfused as in the reference build
        const double fx = __dmul_rn(__dsub_rn(uE, uW), hy);
        const double fy = __dmul_rn(__dsub_rn(uN, uS), hx);
        res = fmax(res, fabs(__dsub_rn(L.div_vol(__dadd_rn(fx, fy)), qc)));
        qmax = fmax(qmax, fabs(qc));
        if (cfl.on) {  // cfl_timestep's per-cell outflux (transport.cpp:59-67), same order and rounding
            double o = __dmul_rn(0.0 < uE ? uE : 0.0, hy);
            o = __dadd_rn(o, __dmul_rn(0.0 < -uW ? -uW : 0.0, hy));
            o = __dadd_rn(o, __dmul_rn(0.0 < uN ? uN : 0.0, hx));
            o = __dadd_rn(o, __dmul_rn(0.0 < -uS ? -uS : 0.0, hx));
            if (o > 0.0) {
                anyf = 1.0;
                dmax = fmax(dmax, __dmul_rn(o, slope));
            }
        }
    }
    udiv_finish(L, res, vmax, hmax, qmax, dmax, anyf, sc, part, counter, cfl);
}

// The boundary-face half of the downscale epilogue, over the 2(nx + ny)
// exterior faces in BoundarySpec order: the next step's injection rate
// (injection_rate, simulation.cpp:85-101; inflow faces, outward velocity < 0)
// and the outlet probe (max_outlet_saturation, simulation.cpp:61-83: the
// largest saturation behind an outflow face of a side whose net outflow is
// positive). Slots: net W/E/S/N (sums), smax W/E/S/N, rate (sum).
__global__ void __launch_bounds__(256) k_bnd_probe(Layout L, const double* __restrict__ u,
                                                   const double* __restrict__ s_out, Scalars* sc, double* part,
                                                   unsigned* counter, CflNext cfl) {
    pdl_begin();
    constexpr int NP = 9;
    double net[4] = {0.0, 0.0, 0.0, 0.0}, smax[4] = {0.0, 0.0, 0.0, 0.0}, rate = 0.0;
    const double hx = L.hx, hy = L.hy;
    double fin = 0.0;  // frac_flow(inflow) (transport.cpp:39-43), clamped, unrounded-FMA-free
    if (cfl.on) {
        const double si = cfl.inflow < 0.0 ? 0.0 : (cfl.inflow > 1.0 ? 1.0 : cfl.inflow);
        const double w = __dmul_rn(__dmul_rn(cfl.M, si), si), t = 1.0 - si;
        fin = __ddiv_rn(w, __dadd_rn(w, __dmul_rn(t, t)));
    }
    const int nb = L.bfaces();
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x) {
        int side, c;
        double ug, area;  // face velocity in global orientation
        if (b < L.ny) {
            side = 0, c = L.cell(0, b), ug = u[L.vface(0, b)], area = hy;
        } else if (b < 2 * L.ny) {
            side = 1, c = L.cell(L.nx - 1, b - L.ny), ug = u[L.vface(L.nx, b - L.ny)], area = hy;
        } else if (b < 2 * L.ny + L.nx) {
            side = 2, c = L.cell(b - 2 * L.ny, 0), ug = u[L.hface(b - 2 * L.ny, 0)], area = hx;
        } else {
            side = 3, c = L.cell(b - 2 * L.ny - L.nx, L.ny - 1), ug = u[L.hface(b - 2 * L.ny - L.nx, L.ny)], area = hx;
        }
        const bool lo = side == 0 || side == 2;  // W / S: outward normal is -x / -y
        const double fo = lo ? -ug : ug;         // outward normal velocity
        if (cfl.on && fo < 0.0) rate = __dadd_rn(rate, __dmul_rn(__dmul_rn(lo ? ug : -ug, area), fin));
        if (s_out) {
            net[side] += fo * area;
            if (fo > 1e-14) smax[side] = fmax(smax[side], s_out[c]);
        }
    }
    __shared__ double shm[32 * NP];
    __shared__ double red[NP];
    constexpr unsigned SUMS = 0x10Fu;  // slots 0..3 (side nets) and 8 (rate) are sums, 4..7 maxima
    double v[NP] = {net[0], net[1], net[2], net[3], smax[0], smax[1], smax[2], smax[3], rate};
    block_reduce_multi<NP>(v, SUMS, shm, red);
    if (threadIdx.x < NP) part[NP * blockIdx.x + threadIdx.x] = red[threadIdx.x];
    if (last_block_done(counter)) {
        double a[NP];
#pragma unroll
        for (int k = 0; k < NP; ++k) a[k] = 0.0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
#pragma unroll
            for (int k = 0; k < NP; ++k) {
                const double t = __ldcg(part + (size_t)NP * b + k);
                a[k] = ((SUMS >> k) & 1u) ? a[k] + t : fmax(a[k], t);
            }
        }
        block_reduce_multi<NP>(a, SUMS, shm, red);
        if (threadIdx.x == 0) {
            if (s_out) {
                double om = 0.0;
                for (int sd = 0; sd < 4; ++sd)
                    if (red[sd] > 1e-14) om = fmax(om, red[4 + sd]);
                sc->outlet_max = om;
            }
            if (cfl.on) sc->inj_next = red[8];
            *counter = 0;
        }
    }
}


// ---------------------------------------------------------------- K2 ----
// MPM-2P data: w from p^m under kappa_n; q' = q - div w; g' = g - p^m_face;
// z' = z - w.n_out; particular rhs under the cached (kappa_m, beta) operator
// (mpm.cpp:48-86; elliptic.cpp:161-181).
__global__ void k_mpm_rhs(Layout L, int max_rhs, int anchor, const double* __restrict__ kn,
                          const double* __restrict__ km, const double* __restrict__ Tn,
                          const double* __restrict__ q, const int* __restrict__ bc_kind,
                          const double* __restrict__ bc_value, const double* __restrict__ bm,
                          const double* __restrict__ bp, const double* __restrict__ pm,
                          const double* __restrict__ bpm, double* __restrict__ X, double* __restrict__ GZ,
                          double* __restrict__ WU) {
    pdl_begin();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= L.cells()) return;
    const int i = c % L.nx, j = c / L.nx;
    const int s = (j / L.sny) * L.nsx + i / L.snx;
    const int ii = i % L.snx, jj = j % L.sny, r = jj * L.snx + ii;
    const double pc = pm[c];
    int idx[4];
    const int ne = cell_edges(L, ii, jj, idx);
    double wun[4];
    for (int t = 0; t < ne; ++t) {
        const EdgeInfo e = L.edge(s, idx[t]);
        const double tn = half_trans(L, e.side, kn[c]);
        wun[t] = tn * (pc - bpm[(size_t)s * L.nbe + idx[t]]) / e.area;
    }
    auto bw = [&](int side) -> double {  // boundary w (global orientation) for a side of this cell
        for (int t = 0; t < ne; ++t) {
            const int id = idx[t];
            const int sd = id < L.sny ? SIDE_W : id < 2 * L.sny ? SIDE_E : id < 2 * L.sny + L.snx ? SIDE_S : SIDE_N;
            if (sd == side) return (side == SIDE_E || side == SIDE_N) ? wun[t] : -wun[t];
        }
        return 0.0;
    };
    const double wW = ii > 0 ? Tn[L.vface(i, j)] * (pm[L.cell(i - 1, j)] - pc) / L.hy : bw(SIDE_W);
    const double wE = ii < L.snx - 1 ? Tn[L.vface(i + 1, j)] * (pc - pm[L.cell(i + 1, j)]) / L.hy : bw(SIDE_E);
    const double wS = jj > 0 ? Tn[L.hface(i, j)] * (pm[L.cell(i, j - 1)] - pc) / L.hx : bw(SIDE_S);
    const double wN = jj < L.sny - 1 ? Tn[L.hface(i, j + 1)] * (pc - pm[L.cell(i, j + 1)]) / L.hx : bw(SIDE_N);
    const double fx = (wE - wW) * L.hy;
    const double fy = (wN - wS) * L.hx;
    const double divw = (fx + fy) / L.vol();
    double b = (q[c] - divw) * L.vol();
    for (int t = 0; t < ne; ++t) {
        const EdgeInfo e = L.edge(s, idx[t]);
        const double th = half_trans(L, e.side, km[c]);
        const size_t eo = (size_t)s * L.nbe + idx[t];
        WU[eo] = wun[t];
        if (e.iface >= 0) {
            b += eff_robin(th, edge_beta(L, e, bm, bp), e.area) * 0.0;
            GZ[eo] = 0.0;
        } else if (bc_kind[e.gbc] == BC_PRESSURE) {
            const double g = bc_value[e.gbc] - bpm[eo];
            GZ[eo] = g;
            b += th * g;
        } else if (bc_kind[e.gbc] == BC_ROBIN) {  // kept as restricted (mpm.cpp:80-81)
            const double rr = L.rb_rhs[e.gbc];
            GZ[eo] = rr;
            b += eff_robin(th, L.rb_beta[e.gbc], e.area) * rr;
        } else {
            const double z = bc_value[e.gbc] - wun[t];
            GZ[eo] = z;
            b -= z * e.area;
        }
    }
    if (anchor && r == 0) b = 0.0;
    X[xoff(L, max_rhs, s, 0) + r] = b;
}

// k_mpm_rhs split in two for many subdomains. k_mpm_edges: one thread per
// subdomain boundary edge — the edge's w (outward, this subdomain's own:
// tn (p^m - p^m_face) / area, mpm.cpp:73-75), its modified data g' / z' and
// its term in the particular right-hand side (mpm.cpp:76-85,
// elliptic.cpp:161-181) into WU, GZ and ET.
__global__ void __launch_bounds__(256) k_mpm_edges(Layout L, const double* __restrict__ kn,
                                                   const double* __restrict__ km, const int* __restrict__ bc_kind,
                                                   const double* __restrict__ bc_value, const double* __restrict__ bm,
                                                   const double* __restrict__ bp, const double* __restrict__ pm,
                                                   const double* __restrict__ bpm, double* __restrict__ GZ,
                                                   double* __restrict__ WU, double* __restrict__ ET,
                                                   double* __restrict__ PD) {
    pdl_begin();
    const int ne = L.n_sub * L.nbe;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < ne; x += gridDim.x * blockDim.x) {
        const int s = x / L.nbe, idx = x % L.nbe;
        const EdgeInfo e = L.edge(s, idx);
        const double kc = kn[e.global_cell], kmc = km[e.global_cell], pc = pm[e.global_cell], bpv = bpm[x];
        const double pd = __dsub_rn(pc, bpv);
        if (PD) PD[x] = pd;
        const double wun = half_trans(L, e.side, kc) * pd / e.area;
        const double th = half_trans(L, e.side, kmc);
        WU[x] = wun;
        double term;
        if (e.iface >= 0) {
            term = __dmul_rn(eff_robin(th, edge_beta(L, e, bm, bp), e.area), 0.0);
            GZ[x] = 0.0;
        } else if (bc_kind[e.gbc] == BC_PRESSURE) {
            const double g = __dsub_rn(bc_value[e.gbc], bpv);
            GZ[x] = g;
            term = __dmul_rn(th, g);
        } else if (bc_kind[e.gbc] == BC_ROBIN) {  // kept as restricted (mpm.cpp:80-81)
            const double rr = L.rb_rhs[e.gbc];
            GZ[x] = rr;
            term = __dmul_rn(eff_robin(th, L.rb_beta[e.gbc], e.area), rr);
        } else {
            const double z = __dsub_rn(bc_value[e.gbc], wun);
            GZ[x] = z;
            term = -__dmul_rn(z, e.area);
        }
        ET[x] = term;
    }
}

// Between rebuilds only kappa_n changes: p^m, the face pressures and the
// cached operator are those of the last rebuild, so an edge's pressure drop
// PD = p^m - p^m_face and the g' / right-hand-side terms of interface,
// pressure and Robin edges are static (written by k_mpm_edges at the rebuild
// into arrays the MPM-2P path owns). Per step: w from kappa_n and PD (the
// same product and quotient as k_mpm_edges), and the z' / term of flux faces.
__global__ void __launch_bounds__(256) k_mpm_edges_kn(Layout L, const double* __restrict__ kn,
                                                      const int* __restrict__ bc_kind,
                                                      const double* __restrict__ bc_value,
                                                      const double* __restrict__ PD, double* __restrict__ GZ,
                                                      double* __restrict__ WU, double* __restrict__ ET) {
    pdl_begin();
    const int ne = L.n_sub * L.nbe;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < ne; x += gridDim.x * blockDim.x) {
        const int s = x / L.nbe, idx = x % L.nbe;
        const EdgeInfo e = L.edge(s, idx);
        const double wun = half_trans(L, e.side, kn[e.global_cell]) * PD[x] / e.area;
        WU[x] = wun;
        if (e.iface < 0) {
            const int kind = bc_kind[e.gbc];
            if (kind != BC_PRESSURE && kind != BC_ROBIN) {
                const double z = __dsub_rn(bc_value[e.gbc], wun);
                GZ[x] = z;
                ET[x] = -__dmul_rn(z, e.area);
            }
        }
    }
}

// ... and k_mpm_rhs_w: one thread per cell, warps over 32 consecutive cells
// of a row, every load of the cell issued before its arithmetic. An interior
// east face's w is the next lane's west face (shuffle); a subdomain-edge face
// takes the edge's own w from k_mpm_edges (w is per subdomain). The
// divergence and the right-hand side are unfused, as in the reference build;
// the edge terms are added in W, E, S, N order (k_mpm_rhs's).
__global__ void __launch_bounds__(256, 4) k_mpm_rhs_w(Layout L, int max_rhs, int anchor,
                                                   const double* __restrict__ Tn, const double* __restrict__ q,
                                                   const double* __restrict__ pm, const double* __restrict__ WU,
                                                   const double* __restrict__ ET, double* __restrict__ X) {
    pdl_begin();
    const int lane = threadIdx.x & 31;
    const double vol = L.vol(), hx = L.hx, hy = L.hy;
    // 2-D grid as k_ds_u_div: column strips x rows
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = i < L.nx;
    const int ic = valid ? i : L.nx - 1;
    const int sx = ic / L.snx, ii = ic - sx * L.snx;
    for (int j = blockIdx.y; j < L.ny; j += gridDim.y) {
        const int sy = j / L.sny, jj = j - sy * L.sny;
        const int cc = j * L.nx + ic;
        const int s = sy * L.nsx + sx;
        const int r = jj * L.snx + ii;
        const size_t eo = (size_t)s * L.nbe;
        const bool de = lane == 31 || i + 1 >= L.nx;
        const bool hw = ii > 0, he = ii + 1 < L.snx, hs = jj > 0, hn = jj + 1 < L.sny;
        const int eW = jj, eE = L.sny + jj, eS = 2 * L.sny + ii, eN = 2 * L.sny + L.snx + ii;
        const double pc = pm[cc];
        const double pw = hw ? pm[cc - 1] : 0.0;
        const double tw = hw ? Tn[L.vface(ic, j)] : 0.0;
        const double pe = (de && he) ? pm[cc + 1] : 0.0;
        const double te = (de && he) ? Tn[L.vface(ic + 1, j)] : 0.0;
        const double ps = hs ? pm[cc - L.nx] : 0.0;
        const double ts = hs ? Tn[L.hface(ic, j)] : 0.0;
        const double pn = hn ? pm[cc + L.nx] : 0.0;
        const double tn = hn ? Tn[L.hface(ic, j + 1)] : 0.0;
        const double qc = q[cc];
        const double uw = hw ? 0.0 : WU[eo + eW], ue = he ? 0.0 : WU[eo + eE];
        const double us = hs ? 0.0 : WU[eo + eS], un = hn ? 0.0 : WU[eo + eN];
        const double xw = hw ? 0.0 : ET[eo + eW], xe = he ? 0.0 : ET[eo + eE];
        const double xs = hs ? 0.0 : ET[eo + eS], xn = hn ? 0.0 : ET[eo + eN];
        const double wW = hw ? L.div_hy(tw * (pw - pc)) : -uw;
        double wE = __shfl_down_sync(0xffffffffu, wW, 1);
        if (!he) wE = ue;
        else if (de) wE = L.div_hy(te * (pc - pe));
        if (!valid) continue;
        const double wS = hs ? L.div_hx(ts * (ps - pc)) : -us;
        const double wN = hn ? L.div_hx(tn * (pc - pn)) : un;
        const double fx = __dmul_rn(__dsub_rn(wE, wW), hy);
        const double fy = __dmul_rn(__dsub_rn(wN, wS), hx);
        const double divw = L.div_vol(__dadd_rn(fx, fy));
        double b = __dmul_rn(__dsub_rn(qc, divw), vol);
        if (!hw) b = __dadd_rn(b, xw);
        if (!he) b = __dadd_rn(b, xe);
        if (!hs) b = __dadd_rn(b, xs);
        if (!hn) b = __dadd_rn(b, xn);
        if (anchor && r == 0) b = 0.0;
        X[xoff(L, max_rhs, s, 0) + r] = b;
    }
}

// Particular solve with the cached rebuild factor (mrcm.cpp:248).
// k_mpm_rhs restructured per subdomain: one 256-thread CTA per subdomain.
// Every operand (the cells' face transmissibilities, q, neighbour pressures
// and the boundary edges' data) is loaded in one round, the boundary-edge
// terms are formed once per edge by dedicated threads (no divergent edge
// loop in the cell threads), and each cell applies its edges' terms to b in
// k_mpm_rhs's W, E, S, N order, so X, GZ and WU are bit-identical.
constexpr int RHS_TPB = 256, RHS_CPT = 4;  // cells per thread (subdomains up to 1,024 cells)
__global__ void __launch_bounds__(RHS_TPB) k_mpm_rhs_sub(Layout L, int max_rhs, int anchor,
                                                         const double* __restrict__ kn, const double* __restrict__ km,
                                                         const double* __restrict__ Tn, const double* __restrict__ q,
                                                         const int* __restrict__ bc_kind,
                                                         const double* __restrict__ bc_value,
                                                         const double* __restrict__ bm, const double* __restrict__ bp,
                                                         const double* __restrict__ pm, const double* __restrict__ bpm,
                                                         double* __restrict__ X, double* __restrict__ GZ,
                                                         double* __restrict__ WU) {
    pdl_begin();
    extern __shared__ double rsm[];
    double* pmS = rsm;                 // ncs
    double* wunS = rsm + L.ncs;        // nbe: outward w of each boundary edge
    double* termS = wunS + L.nbe;      // nbe: the edge's term in b
    const int s = blockIdx.x;
    const int i0 = L.sub_i0(s), j0 = L.sub_j0(s);
    // cell operands (registers), issued together with the pm / edge loads
    double pc[RHS_CPT], tW[RHS_CPT], tE[RHS_CPT], tS[RHS_CPT], tN[RHS_CPT], qv[RHS_CPT];
#pragma unroll
    for (int k = 0; k < RHS_CPT; ++k) {
        const int r = threadIdx.x + RHS_TPB * k;
        pc[k] = tW[k] = tE[k] = tS[k] = tN[k] = qv[k] = 0.0;
        if (r < L.ncs) {
            const int ii = r % L.snx, jj = r / L.snx, i = i0 + ii, j = j0 + jj;
            pc[k] = pm[L.cell(i, j)];
            tW[k] = Tn[L.vface(i, j)];
            tE[k] = Tn[L.vface(i + 1, j)];
            tS[k] = Tn[L.hface(i, j)];
            tN[k] = Tn[L.hface(i, j + 1)];
            qv[k] = q[L.cell(i, j)];
        }
    }
    // boundary edges (k_mpm_rhs's per-edge arithmetic, mpm.cpp:64-85)
    for (int idx = threadIdx.x; idx < L.nbe; idx += RHS_TPB) {
        const EdgeInfo e = L.edge(s, idx);
        const size_t eo = (size_t)s * L.nbe + idx;
        const double pce = pm[e.global_cell];
        const double tn = half_trans(L, e.side, kn[e.global_cell]);
        const double wun = tn * (pce - bpm[eo]) / e.area;
        const double th = half_trans(L, e.side, km[e.global_cell]);
        WU[eo] = wun;
        double term;
        if (e.iface >= 0) {
            term = eff_robin(th, edge_beta(L, e, bm, bp), e.area) * 0.0;
            GZ[eo] = 0.0;
        } else if (bc_kind[e.gbc] == BC_PRESSURE) {
            const double g = bc_value[e.gbc] - bpm[eo];
            GZ[eo] = g;
            term = th * g;
        } else if (bc_kind[e.gbc] == BC_ROBIN) {  // kept as restricted (mpm.cpp:80-81)
            const double rr = L.rb_rhs[e.gbc];
            GZ[eo] = rr;
            term = eff_robin(th, L.rb_beta[e.gbc], e.area) * rr;
        } else {
            const double z = bc_value[e.gbc] - wun;
            GZ[eo] = z;
            term = -(z * e.area);
        }
        wunS[idx] = (e.side == SIDE_E || e.side == SIDE_N) ? wun : -wun;  // global orientation
        termS[idx] = term;
    }
#pragma unroll
    for (int k = 0; k < RHS_CPT; ++k) {
        const int r = threadIdx.x + RHS_TPB * k;
        if (r < L.ncs) pmS[r] = pc[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < RHS_CPT; ++k) {
        const int r = threadIdx.x + RHS_TPB * k;
        if (r >= L.ncs) continue;
        const int ii = r % L.snx, jj = r / L.snx;
        const double p0 = pc[k];
        const int eW = jj, eE = L.sny + jj, eS = 2 * L.sny + ii, eN = 2 * L.sny + L.snx + ii;
        const double wW = ii > 0 ? tW[k] * (pmS[r - 1] - p0) / L.hy : wunS[eW];
        const double wE = ii < L.snx - 1 ? tE[k] * (p0 - pmS[r + 1]) / L.hy : wunS[eE];
        const double wS = jj > 0 ? tS[k] * (pmS[r - L.snx] - p0) / L.hx : wunS[eS];
        const double wN = jj < L.sny - 1 ? tN[k] * (p0 - pmS[r + L.snx]) / L.hx : wunS[eN];
        const double fx = (wE - wW) * L.hy;
        const double fy = (wN - wS) * L.hx;
        const double divw = (fx + fy) / L.vol();
        double b = (qv[k] - divw) * L.vol();
        if (ii == 0) b += termS[eW];
        if (ii == L.snx - 1) b += termS[eE];
        if (jj == 0) b += termS[eS];
        if (jj == L.sny - 1) b += termS[eN];
        if (anchor && r == 0) b = 0.0;
        X[xoff(L, max_rhs, s, 0) + r] = b;
    }
}

__global__ void k_part_solve(Layout L, int max_rhs, const double* __restrict__ D, const double* __restrict__ Lc,
                             const double* __restrict__ Lr, double* __restrict__ X) {
    pdl_begin();
    extern __shared__ double smem[];
    const int w = threadIdx.x >> 5;
    const int s = blockIdx.x * WPB + w;
    if (s >= L.n_sub) return;
    const int n = L.ncs, B = L.snx;
    double* sm = smem + (size_t)w * band_smem_doubles(B, 1);
    const size_t so = (size_t)s * n;
    double* x = X + xoff(L, max_rhs, s, 0);
    band_forward(n, B, Lc + so * B, x, 1, n, sm);
    band_backward(n, B, D + so, Lr + so * B, x, 1, n, sm);
}

// Particular traces under the cached operator with the modified data.
__global__ void k_part_traces(Layout L, int max_rhs, const double* __restrict__ km,
                              const int* __restrict__ bc_kind, const double* __restrict__ bm,
                              const double* __restrict__ bp, const double* __restrict__ GZ,
                              const double* __restrict__ X, double* __restrict__ PU) {
    pdl_begin();
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= L.n_sub * L.nbe) return;
    const int s = x / L.nbe, idx = x % L.nbe;
    const EdgeInfo e = L.edge(s, idx);
    const double th = half_trans(L, e.side, km[e.global_cell]);
    const double pc = X[xoff(L, max_rhs, s, 0) + e.local_cell];
    double un;
    if (e.iface >= 0) {
        const double te = eff_robin(th, edge_beta(L, e, bm, bp), e.area);
        un = te * (pc - 0.0) / e.area;
    } else if (bc_kind[e.gbc] == BC_PRESSURE) {
        un = th * (pc - GZ[x]) / e.area;
    } else if (bc_kind[e.gbc] == BC_ROBIN) {
        un = eff_robin(th, L.rb_beta[e.gbc], e.area) * (pc - GZ[x]) / e.area;
    } else {
        un = GZ[x];
    }
    PU[x] = un;
}

__global__ void k_part_psum(Layout L, int max_rhs, const double* __restrict__ X, double* __restrict__ PS) {
    pdl_begin();
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (gw >= L.n_sub) return;
    const double* x = X + xoff(L, max_rhs, gw, 0);
    double v = 0.0;
    for (int r = lane; r < L.ncs; r += 32) v += x[r];
    v = warp_sum(v);
    if (lane == 0) PS[gw] = v;
}

// ---------------------------------------------------------------- static --
// Separable repair solve (uniform subdomains, ground split by subdomain
// column + row): L = I (x) Ax + Ay (x) I, so with Ax = Qx Lx Qx^T and
// Ay = Qy Ly Qy^T, delta = Qy [(Qy^T R Qx) ./ (ly_i + lx_j)] Qx^T, where
// R[sy][sx] = resid[sy nsx + sx]. One small GEMM per launch, one thread per
// output: C[m x n] = op(A) op(B), op(X) = X or X^T (row-major, square
// factors), optionally divided by (ly_i + lx_j).
// 32 x 32 output tile per 256-thread block, k in slabs of 32 staged in
// shared memory (all of a slab's loads issued together), 4 outputs per thread
__device__ __forceinline__ void sep_gemm_tile(int m, int n, int kk, const double* A, int ta, const double* Bm, int tb,
                                              double* C, const double* lx, const double* ly, int i0, int j0,
                                              double (*As)[33], double (*Bs)[33]) {
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // output column tx, rows ty + 8 q
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k0 = 0; k0 < kk; k0 += 32) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int r = ty + 8 * q;  // As[r][c] = op(A)[i0 + r][k0 + c]; Bs[r][c] = op(B)[k0 + r][j0 + c]
            const int ia = i0 + r, ka = k0 + tx;
            As[r][tx] = (ia < m && ka < kk) ? (ta ? A[(size_t)ka * m + ia] : A[(size_t)ia * kk + ka]) : 0.0;
            const int kb = k0 + r, jb = j0 + tx;
            Bs[r][tx] = (kb < kk && jb < n) ? (tb ? Bm[(size_t)jb * kk + kb] : Bm[(size_t)kb * n + jb]) : 0.0;
        }
        __syncthreads();
#pragma unroll 8
        for (int t = 0; t < 32; ++t) {
            const double b = Bs[t][tx];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] = fma(As[ty + 8 * q][t], b, acc[q]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int i = i0 + ty + 8 * q, j = j0 + tx;
        if (i < m && j < n) C[(size_t)i * n + j] = lx ? acc[q] / (ly[i] + lx[j]) : acc[q];
    }
}
__global__ void __launch_bounds__(256) k_sep_gemm(int m, int n, int kk, const double* __restrict__ A, int ta,
                                                  const double* __restrict__ Bm, int tb, double* __restrict__ C,
                                                  const double* __restrict__ lx, const double* __restrict__ ly) {
    pdl_begin();
    __shared__ double As[32][33], Bs[32][33];
    sep_gemm_tile(m, n, kk, A, ta, Bm, tb, C, lx, ly, blockIdx.y * 32, blockIdx.x * 32, As, Bs);
}
// The four products of the separable solve in one cooperative launch (every
// product has the ny x nx output, so a block keeps its tile; grid barriers
// between the products): delta = Qy [(Qy^T (R Qx)) ./ (ly + lx)] Qx^T. The
// intermediates are read with plain loads (written by other blocks of this
// launch), the arithmetic and its order are k_sep_gemm's.
__global__ void __launch_bounds__(256) k_sep_solve(int nx, int ny, const double* R, const double* Qx, const double* Qy,
                                                   const double* lx, const double* ly, double* z1, double* z2,
                                                   double* delta) {
    __shared__ double As[32][33], Bs[32][33];
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
    const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
    sep_gemm_tile(ny, nx, nx, R, 0, Qx, 0, z1, nullptr, nullptr, i0, j0, As, Bs);
    grid.sync();
    sep_gemm_tile(ny, nx, ny, Qy, 1, z1, 0, z2, lx, ly, i0, j0, As, Bs);
    grid.sync();
    sep_gemm_tile(ny, nx, ny, Qy, 0, z2, 0, z1, nullptr, nullptr, i0, j0, As, Bs);
    grid.sync();
    sep_gemm_tile(ny, nx, nx, z1, 0, Qx, 1, delta, nullptr, nullptr, i0, j0, As, Bs);
}

__global__ void k_static(Layout L, const double* __restrict__ q, const int* __restrict__ bc_kind,
                         double* __restrict__ qsum, double* __restrict__ ground) {
    pdl_begin();
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= L.n_sub) return;
    const double vol = L.vol();
    double qs = 0.0;  // mrcm.cpp:323-325, row-major order
    for (int jj = 0; jj < L.sny; ++jj)
        for (int ii = 0; ii < L.snx; ++ii) qs += q[L.cell(L.sub_i0(s) + ii, L.sub_j0(s) + jj)] * vol;
    qsum[s] = qs;
    double g = 0.0;  // mrcm.cpp:333-336
    for (int idx = 0; idx < L.nbe; ++idx) {
        const EdgeInfo e = L.edge(s, idx);
        if (e.iface < 0 && bc_kind[e.gbc] == BC_PRESSURE) g += e.area;
    }
    ground[s] = g;
}

// Dense repair operator (mrcm.cpp:351-371): one thread per row.
__global__ void k_repair_matrix(Layout L, int grounded, const double* __restrict__ ground, double* __restrict__ A) {
    pdl_begin();
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    const int n = L.n_sub;
    if (s >= n) return;
    double* row = A + (size_t)s * n;
    for (int t = 0; t < n; ++t) row[t] = 0.0;
    int inc[4];
    const int ni = L.incident(s, inc);
    for (int a = 0; a < ni; ++a) {
        const int k = inc[a];
        const double area = L.iface_edges(k) * (k < L.NV ? L.hy : L.hx);
        row[s] += area;
        const int other = L.iface_minus(k) == s ? L.iface_plus(k) : L.iface_minus(k);
        row[other] -= area;
    }
    if (grounded) {
        row[s] += ground[s];
    } else {
        if (s == 0)
            for (int t = 0; t < n; ++t) row[t] = 0.0;
        row[0] = 0.0;
        if (s == 0) row[0] = 1.0;
    }
}

int grid_for(long long n) { return std::max(1, cdiv(n, TPB)); }
// 2-D grid of the row kernels: 256-column strips x rows, about `cap` blocks
dim3 grid2d(const Ctx& c, const Layout& L, int cap = 0) {
    if (cap <= 0) cap = 8 * c.num_sms;
    const int gx = cdiv(L.nx, TPB);
    const int gy = std::max(1, std::min(L.ny, cap / gx));
    return dim3(gx, gy);
}
int band_blocks(const Layout& L) { return cdiv(L.n_sub, WPB); }

}  // namespace

void launch_trans(Ctx& c, const double* kappa) {
    if (c.trans_fresh) {  // the driver's k_kappa already wrote T for this kappa
        c.trans_fresh = false;
        return;
    }
    {
        PROF(c, "k_trans");
        launch_k(c, k_trans, std::min(grid_for(c.L.faces()), 8 * c.num_sms), TPB, 0, c.L, kappa, c.T);
        CK_LAUNCH();
    }
}

void launch_beta(Ctx& c, const double* kappa) {
    const Layout& L = c.L;
    const int E = L.skeleton_edges();
    if (E == 0) return;
    {
        PROF(c, "k_face_kappa");
        launch_k(c, k_face_kappa, grid_for(E), TPB, 0, L, kappa, c.face_kappa);
        CK_LAUNCH();
    }
    if (c.alpha_mode == 1) {
        size_t bytes = c.sort_tmp_bytes;
        CK(cub::DeviceRadixSort::SortKeys(c.sort_tmp.p, bytes, c.face_kappa.p, c.sort_keys.p, E, 0, 64, c.st));
    }
    {
        PROF(c, "k_beta");
        launch_k(c, k_beta, grid_for(E), TPB, 0, L, kappa, c.face_kappa, c.sort_keys, c.alpha_mode, c.alpha, c.alpha_min,
                                              c.alpha_max, c.pct_lo, c.pct_hi, c.beta_m, c.beta_p, c.alpha_e, c.sc);
        CK_LAUNCH();
    }
}

namespace {
// Eigen-decomposition of a symmetric tridiagonal matrix (diagonal d,
// sub-diagonal e[i] = A[i][i-1], e[0] unused) by the implicit QL algorithm
// with Wilkinson-type shifts: A = V diag(d) V^T, V row-major with the
// eigenvectors in its columns. O(n^2) rotations, O(n^3) for V (C5: two
// 128 x 128 chains in ~2 ms, against ~150 ms for cyclic Jacobi).
bool tridiag_eigen(std::vector<double>& d, std::vector<double> e, int n, std::vector<double>& V) {
    std::vector<double> Vt((size_t)n * n, 0.0);  // eigenvector i contiguous: Vt[i n + k] = V[k][i]
    for (int i = 0; i < n; ++i) Vt[(size_t)i * n + i] = 1.0;
    for (int i = 1; i < n; ++i) e[i - 1] = e[i];
    e[n - 1] = 0.0;
    for (int l = 0; l < n; ++l) {
        int iter = 0, m;
        do {
            for (m = l; m < n - 1; ++m) {
                const double dd = std::fabs(d[m]) + std::fabs(d[m + 1]);
                if (std::fabs(e[m]) <= 1e-17 * dd) break;
            }
            if (m == l) break;
            if (++iter > 60) return false;
            double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
            double r = std::hypot(g, 1.0);
            g = d[m] - d[l] + e[l] / (g + (g >= 0.0 ? r : -r));
            double sn = 1.0, cs = 1.0, p = 0.0;
            bool deflated = false;
            for (int i = m - 1; i >= l; --i) {
                const double f = sn * e[i], b = cs * e[i];
                r = std::hypot(f, g);
                e[i + 1] = r;
                if (r == 0.0) {  // underflow: split here and restart
                    d[i + 1] -= p;
                    e[m] = 0.0;
                    deflated = true;
                    break;
                }
                sn = f / r;
                cs = g / r;
                g = d[i + 1] - p;
                r = (d[i] - g) * sn + 2.0 * cs * b;
                p = sn * r;
                d[i + 1] = g + p;
                g = cs * r - b;
                double* vi = &Vt[(size_t)i * n];
                double* vj = vi + n;
                for (int k = 0; k < n; ++k) {
                    const double fz = vj[k];
                    vj[k] = sn * vi[k] + cs * fz;
                    vi[k] = cs * vi[k] - sn * fz;
                }
            }
            if (deflated) continue;
            d[l] -= p;
            e[l] = g;
            e[m] = 0.0;
        } while (m != l);
    }
    V.resize((size_t)n * n);
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < n; ++k) V[(size_t)k * n + i] = Vt[(size_t)i * n + k];
    return true;
}
}  // namespace

// The repair Laplacian (mrcm.cpp:347-371) is a Kronecker sum when every
// vertical interface has the same area, every horizontal one too, and the
// ground splits as g[s] = gx[sx] + gy[sy] (e.g. pressure faces on whole
// west / east sides): L = I (x) Ax + Ay (x) I. Then the static n_sub x n_sub
// inverse (C5: 16,384^2 = 2.1 GB, inverted at creation and read every step)
// is replaced by two small eigen-decompositions and four small GEMMs per
// step. Used above 4,096 subdomains (below, the dense GEMV is one launch);
// MPM2P_REPAIR=sep / dense overrides.
bool sep_repair_setup(Ctx& c) {
    const Layout& L = c.L;
    const char* env = std::getenv("MPM2P_REPAIR");
    const bool force = env && std::strcmp(env, "sep") == 0;
    if (env && std::strcmp(env, "dense") == 0) return false;
    if (!c.grounded || L.n_sub < 2 || (!force && L.n_sub <= 4096)) return false;
    const int nx = L.nsx, ny = L.nsy;
    std::vector<double> g(L.n_sub, 0.0);  // k_static's ground, mrcm.cpp:333-336
    for (int sd = 0; sd < L.n_sub; ++sd)
        for (int idx = 0; idx < L.nbe; ++idx) {
            const EdgeInfo e = L.edge(sd, idx);
            if (e.iface < 0 && c.bc_kind_h[e.gbc] == BC_PRESSURE) g[sd] += e.area;
        }
    std::vector<double> gx(nx), gy(ny);
    for (int i = 0; i < nx; ++i) gx[i] = g[i];
    for (int j = 0; j < ny; ++j) gy[j] = g[(size_t)j * nx] - g[0];
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            const double d = g[(size_t)j * nx + i] - (gx[i] + gy[j]);
            if (std::fabs(d) > 1e-13 * (std::fabs(g[(size_t)j * nx + i]) + 1e-300)) return false;
        }
    const double av = L.sny * L.hy, ah = L.snx * L.hx;  // interface areas (uniform subdomains)
    std::vector<double> Ax((size_t)nx * nx, 0.0), Ay((size_t)ny * ny, 0.0);
    for (int i = 0; i + 1 < nx; ++i) {
        Ax[(size_t)i * nx + i] += av;
        Ax[(size_t)(i + 1) * nx + i + 1] += av;
        Ax[(size_t)i * nx + i + 1] -= av;
        Ax[(size_t)(i + 1) * nx + i] -= av;
    }
    for (int j = 0; j + 1 < ny; ++j) {
        Ay[(size_t)j * ny + j] += ah;
        Ay[(size_t)(j + 1) * ny + j + 1] += ah;
        Ay[(size_t)j * ny + j + 1] -= ah;
        Ay[(size_t)(j + 1) * ny + j] -= ah;
    }
    for (int i = 0; i < nx; ++i) Ax[(size_t)i * nx + i] += gx[i];
    for (int j = 0; j < ny; ++j) Ay[(size_t)j * ny + j] += gy[j];
    // both are tridiagonal (a chain of subdomains plus the ground)
    std::vector<double> Qx, Qy, lx(nx), ly(ny), ex(nx, 0.0), ey(ny, 0.0);
    for (int i = 0; i < nx; ++i) {
        lx[i] = Ax[(size_t)i * nx + i];
        if (i > 0) ex[i] = Ax[(size_t)i * nx + i - 1];
    }
    for (int j = 0; j < ny; ++j) {
        ly[j] = Ay[(size_t)j * ny + j];
        if (j > 0) ey[j] = Ay[(size_t)j * ny + j - 1];
    }
    if (!tridiag_eigen(lx, ex, nx, Qx) || !tridiag_eigen(ly, ey, ny, Qy)) return false;
    double mn = INFINITY, mx = 0.0;
    for (double a : lx)
        for (double b : ly) {
            mn = std::min(mn, a + b);
            mx = std::max(mx, std::fabs(a + b));
        }
    if (!(mn > 1e-12 * mx)) return false;  // singular: keep the dense path and its guard
    c.sep_qx.alloc(Qx.size());
    c.sep_qy.alloc(Qy.size());
    c.sep_lam.alloc(nx + ny);
    c.sep_z1.alloc((size_t)nx * ny);
    c.sep_z2.alloc((size_t)nx * ny);
    std::vector<double> lam(lx);
    lam.insert(lam.end(), ly.begin(), ly.end());
    CK(cudaMemcpyAsync(c.sep_qx.p, Qx.data(), Qx.size() * sizeof(double), cudaMemcpyHostToDevice, c.st));
    CK(cudaMemcpyAsync(c.sep_qy.p, Qy.data(), Qy.size() * sizeof(double), cudaMemcpyHostToDevice, c.st));
    CK(cudaMemcpyAsync(c.sep_lam.p, lam.data(), lam.size() * sizeof(double), cudaMemcpyHostToDevice, c.st));
    CK(cudaStreamSynchronize(c.st));
    return true;
}

void launch_setup_static(Ctx& c) {
    const Layout& L = c.L;
    {
        PROF(c, "k_static");
        launch_k(c, k_static, grid_for(L.n_sub), TPB, 0, L, c.q, c.bc_kind, c.qsum_sub, c.ground);
        CK_LAUNCH();
    }
    if (c.repair_active && !c.sep_repair) {
        DevBuf<double> A;
        A.alloc((size_t)L.n_sub * L.n_sub);
        {
            PROF(c, "k_repair_matrix");
            launch_k(c, k_repair_matrix, grid_for(L.n_sub), TPB, 0, L, c.grounded ? 1 : 0, c.ground, A);
            CK_LAUNCH();
        }
        const double rc = spd_inverse(c, A, c.Linv, L.n_sub);
        if (!(rc > 0.0)) throw NumericError("downscale: compatibility-repair operator is singular");
    }
}

// split downscale, downscale, interface solve (declared in context.cuh)

// Split downscale, side-stream half: the downscale operator depends only on
// T = transmissibility(kappa_n) (pure Neumann, all-Flux, anchor 0;
// mrcm.cpp:391-411), so it is assembled and factored (two-sided layout) on
// st2 as soon as T is formed, concurrently with the particular solve,
// interface solve and recombination on the main stream. downscale() joins
// before its sweeps. Works both captured into a graph (fork/join edges) and
// eagerly.
void ds_factor_fork(Ctx& c) {
    if ((!c.ds_split && !c.blk_split) || c.ds_pending) return;
    const Layout& L = c.L;
    CK(cudaEventRecord(c.ev_fork, c.st));
    CK(cudaStreamWaitEvent(c.st2, c.ev_fork, 0));
    const cudaStream_t main_st = c.st;
    c.st = c.st2;
    if (c.blk_split) {  // the blocked DMMA factor of T(kappa_n), pivot inverses stored
        PROF(c, "k_ds_factor");
        switch (L.snx) {
#define X(BW_)                                                                                                  \
    case BW_:                                                                                                   \
        launch_k(c, k_ds_blk_factor_only<BW_>, band_blocks(L), WPB * 32, 0, L, (const double*)c.T, c.Lrd.p,      \
                 c.Gd.p, c.sc.p);                                                                               \
        break;
            X(16) X(24) X(32)
#undef X
            default:
                c.st = main_st;
                throw ConfigError("blocked split downscale: unsupported subdomain width");
        }
        CK_LAUNCH();
        CK(cudaEventRecord(c.ev_join, c.st2));
        c.st = main_st;
        c.ds_pending = true;
        return;
    }
    {
        PROF(c, "k_ds_band");
        launch_k(c, k_ds_prep, grid_for(L.cells()), TPB, 0, L, nullptr, c.T, nullptr, nullptr, nullptr, nullptr,
                 nullptr, nullptr, 0, c.BDd, c.BWd, c.BSd, nullptr, nullptr, c.sc.p, 1);
        CK_LAUNCH();
    }
    {
        PROF(c, "k_ds_factor");
        switch (L.snx) {
#define X(BW_)                                                                                                  \
    case BW_:                                                                                                   \
        twist_configure<BW_>();                                                                                 \
        launch_k(c, k_factor1_t<BW_>, L.n_sub, twist_threads<BW_>(), twist_smem_bytes<BW_>(), L, 1, c.BDd, c.BWd, \
                 c.BSd, c.Dd, c.Lcd, c.Lrd, c.ds_midb, c.ds_sinv, c.ds_yscr, c.sc);                             \
        break;
            MPM2P_TWIST_WIDTHS(X)
#undef X
            default:
                c.st = main_st;
                throw ConfigError("split downscale: unsupported subdomain width");
        }
        CK_LAUNCH();
    }
    CK(cudaEventRecord(c.ev_join, c.st2));
    c.st = main_st;
    c.ds_pending = true;
}

// Downscale shared by the rebuild and the MPM step (mrcm.cpp:306-439); needs
// c.T = transmissibility(kappa), RU/RS = recon traces and pressure sums.
void downscale(Ctx& c, const double* kappa, bool skel_given) {
    const Layout& L = c.L;
    {  // skeleton fluxes (k_skel) are formed inside k_resid unless given
        PROF(c, "k_resid");
        launch_k(c, k_resid, grid_for(32LL * L.n_sub), TPB, 0, L, c.skel, c.RU, c.qsum_sub, c.resid, c.sc, c.red,
                                                             c.red_count, skel_given ? 0 : 1);
        CK_LAUNCH();
    }
    if (c.repair_active && c.sep_repair) {  // delta = Qy [(Qy^T R Qx) ./ (ly + lx)] Qx^T
        const int nx = L.nsx, ny = L.nsy;
        const dim3 g(cdiv(nx, 32), cdiv(ny, 32));
        const double* lx = c.sep_lam.p;
        const double* ly = c.sep_lam.p + nx;
        if ((int)(g.x * g.y) <= red_blocks(c, k_sep_solve, 1LL << 30)) {  // co-resident: one cooperative launch
            PROF(c, "k_sep_solve");
            int nxa = nx, nya = ny;
            const double *R = c.resid.p, *qx = c.sep_qx.p, *qy = c.sep_qy.p;
            double *z1 = c.sep_z1.p, *z2 = c.sep_z2.p, *dl = c.delta.p;
            void* args[] = {&nxa, &nya, &R, &qx, &qy, &lx, &ly, &z1, &z2, &dl};
            CK(cudaLaunchCooperativeKernel((void*)k_sep_solve, g, dim3(TPB), args, 0, c.st));
        } else {
            {
                PROF(c, "k_sep_gemm");
                launch_k(c, k_sep_gemm, g, TPB, 0, ny, nx, nx, c.resid.p, 0, c.sep_qx.p, 0, c.sep_z1.p, nullptr, nullptr);
                CK_LAUNCH();
            }
            {
                PROF(c, "k_sep_gemm");
                launch_k(c, k_sep_gemm, g, TPB, 0, ny, nx, ny, c.sep_qy.p, 1, c.sep_z1.p, 0, c.sep_z2.p, lx, ly);
                CK_LAUNCH();
            }
            {
                PROF(c, "k_sep_gemm");
                launch_k(c, k_sep_gemm, g, TPB, 0, ny, nx, ny, c.sep_qy.p, 0, c.sep_z2.p, 0, c.sep_z1.p, nullptr, nullptr);
                CK_LAUNCH();
            }
            {
                PROF(c, "k_sep_gemm");
                launch_k(c, k_sep_gemm, g, TPB, 0, ny, nx, nx, c.sep_z1.p, 0, c.sep_qx.p, 1, c.delta.p, nullptr, nullptr);
                CK_LAUNCH();
            }
        }
        PROF(c, "k_repair_corr");
        launch_k(c, k_repair_corr, std::min(grid_for(std::max(L.n_iface, L.n_sub)), 2 * c.num_sms), TPB, 0, L, 1,
                 1, c.delta, c.ground, c.corr, c.sc, c.red, c.red_count);
        CK_LAUNCH();
    } else if (c.repair_active) {
        PROF(c, "k_repair_delta");
        launch_k(c, k_repair_delta, cdiv((long long)L.n_sub * 32, TPB), TPB, 0, 
            L.n_sub, c.Linv, c.resid, c.delta, L, c.grounded ? 1 : 0, c.ground, c.corr, c.sc, c.red_count);
        CK_LAUNCH();
    } else {
        PROF(c, "k_repair_corr");
        launch_k(c, k_repair_corr, std::min(grid_for(std::max(L.n_iface, L.n_sub)), 2 * c.num_sms), TPB, 0, 
            L, 0, c.grounded ? 1 : 0, c.delta, c.ground, c.corr, c.sc, c.red, c.red_count);
        CK_LAUNCH();
    }
    const bool split = c.ds_split;
    if (split) ds_factor_fork(c);  // no-op when the caller already forked it
    // the blocked DMMA downscale forms its operator from T itself
    const bool blk = c.ds_blk == 1 || c.blk_split || (c.ds_blk < 0 && (L.snx == 24 || L.snx == 32));
    // With few subdomains per SM (twist_ok) the two-sided scalar solve wins up to B = 24; at B = 32 the
    // blocked DMMA factor is faster even one-sided (C4, 256 subdomains: 163 against 191 us)
    const bool blk_path = !split && (!c.twist_ok || L.snx == 32 || c.blk_split) && blk && L.snx % 8 == 0 && L.snx >= 16 && L.snx <= 32;
    if (c.blk_split && blk_path) ds_factor_fork(c);  // no-op when the caller already forked it
    const bool kappa_checked = c.kappa_checked;  // the driver's k_kappa checked this kappa
    c.kappa_checked = false;
    if (split || blk_path) {  // the operator is formed by the factor: the rhs alone
        PROF(c, "k_ds_rhs");
        launch_k(c, k_ds_edges, std::min(grid_for((long long)L.n_sub * L.nbe), 8 * c.num_sms), TPB, 0, L,
                 (const int*)c.bc_kind.p, (const double*)c.skel.p, (const double*)c.corr.p, (const double*)c.RU.p,
                 (const double*)c.delta.p, c.grounded ? 1 : 0, c.GZ.p, c.ET.p);
        CK_LAUNCH();
        launch_k(c, k_ds_rhs, grid2d(c, L, red_blocks(c, k_ds_rhs, L.cells())), TPB, 0, L,
                 kappa_checked ? nullptr : kappa, (const double*)c.q.p, (const double*)c.ET.p, c.Xd.p, c.sc.p);
        CK_LAUNCH();
    } else {
        PROF(c, "k_ds_prep");
        launch_k(c, k_ds_prep, grid_for(L.cells()), TPB, 0, L, kappa, c.T, c.q, c.bc_kind, c.skel, c.corr, c.RU, c.delta,
                                                         c.grounded ? 1 : 0, c.BDd, c.BWd, c.BSd, c.Xd, c.GZ, c.sc, 0);
        CK_LAUNCH();
    }
    const size_t sm1 = (size_t)WPB * band_smem_doubles(L.snx, 1) * sizeof(double);
    const bool twist = c.twist_ok && !blk_path;
    bool done = false;
    if (split) {
        CK(cudaStreamWaitEvent(c.st, c.ev_join, 0));
        c.ds_pending = false;
        PROF(c, "k_ds_sweep");
        switch (L.snx) {
#define X(BW_)                                                                                                  \
    case BW_:                                                                                                   \
        launch_k(c, k_ds_sweep_t<BW_>, L.n_sub, twist_threads<BW_>(), twist_smem_bytes<BW_>(), L, c.Dd, c.Lcd,  \
                 c.Lrd, c.ds_midb, c.ds_sinv, c.Xd, c.RS, c.p);                                                 \
        done = true;                                                                                            \
        break;
            MPM2P_TWIST_WIDTHS(X)
#undef X
            default:
                break;
        }
        if (done) CK_LAUNCH();
    }
    if (!done && twist) {
        PROF(c, "k_ds_solve");
        switch (L.snx) {
#define X(BW_)                                                                                                  \
    case BW_:                                                                                                   \
        twist_configure<BW_>();                                                                                 \
        launch_k(c, k_ds_solve_t<BW_>, L.n_sub, twist_threads<BW_>(), twist_smem_bytes<BW_>(), L, c.BDd, c.BWd, c.BSd, c.Dd, c.Lrd, c.Xd, \
                                                                       c.RS, c.p, c.sc);                        \
        done = true;                                                                                            \
        break;
            MPM2P_TWIST_WIDTHS(X)
#undef X
            default:
                break;
        }
        if (done) CK_LAUNCH();
    }
    if (!done && blk_path && c.blk_split) {  // the factor ran on the side stream: join, then both sweeps
        CK(cudaStreamWaitEvent(c.st, c.ev_join, 0));
        c.ds_pending = false;
        PROF(c, "k_ds_blk_solve");
        switch (L.snx) {
#define X(BW_)                                                                                                  \
    case BW_:                                                                                                   \
        launch_k(c, k_ds_blk_sweeps<BW_>, band_blocks(L), WPB * 32, 0, L, c.Dd.p, (const double*)c.Lrd,          \
                 (const double*)c.Gd, c.Xd.p, (const double*)c.RS, c.p.p);                                      \
        break;
            X(16) X(24) X(32)
#undef X
            default:
                throw ConfigError("blocked split downscale: unsupported subdomain width");
        }
        CK_LAUNCH();
        done = true;
    }
    if (!done && blk_path) {
        switch (L.snx) {
#define X(BW_)                                                                                                     \
    case BW_:                                                                                                      \
        {                                                                                                          \
            PROF(c, "k_ds_blk_factor");                                                                            \
            launch_k(c, k_ds_blk_factor<BW_>, band_blocks(L), WPB * 32, 0, L, (const double*)c.T, c.Dd.p, c.Lrd.p, \
                     (const double*)c.Xd, c.sc.p);                                                               \
        }                                                                                                          \
        CK_LAUNCH();                                                                                               \
        {                                                                                                          \
            PROF(c, "k_ds_blk_solve");                                                                             \
            launch_k(c, k_ds_blk_solve<BW_>, band_blocks(L), WPB * 32, 0, L, (const double*)c.Dd,                 \
                     (const double*)c.Lrd, c.Xd, c.RS, c.p);                                                      \
        }                                                                                                          \
        done = true;                                                                                               \
        break;
            X(16) X(24) X(32)
#undef X
            default:
                break;
        }
        if (done) CK_LAUNCH();
    }
    if (!done) {
        PROF(c, "k_ds_solve");
        switch (c.no_regband ? -1 : L.snx) {
#define X(BW_)                                                                                                     \
    case BW_:                                                                                                      \
        launch_k(c, k_ds_solve_r<BW_>, band_blocks(L), WPB * 32, 0, L, c.BDd, c.BWd, c.BSd, c.Dd, c.Lrd, c.Xd, c.RS, \
                                                                  c.p, c.sc);                                     \
        break;
            MPM2P_BAND_WIDTHS(X)
#undef X
            default:
                launch_k(c, k_ds_solve, band_blocks(L), WPB * 32, sm1, L, c.BDd, c.BWd, c.BSd, c.Dd, c.Lrd, c.Xd, c.RS,
                                                                    c.p, c.sc);
        }
        CK_LAUNCH();
    }
    {  // velocity scatter + divergence residual (+ outlet probe) in one pass
        PROF(c, "k_ds_u_div");
        CflNext cfl;
        if (c.cfl_fused) cfl = CflNext{1, c.cfl_safety, c.cfl_dt_cap, c.cfl_inflow, c.M};
        launch_k(c, k_ds_u_div, grid2d(c, L, red_blocks(c, k_ds_u_div, L.cells())), TPB, 0, L, c.T, c.Xd, c.GZ, c.u, c.q,
                 c.sc.p, c.red.p, c.red_count.p, cfl);
        CK_LAUNCH();
    }
    if (c.cfl_fused || c.outlet_s) {
        PROF(c, "k_bnd_probe");
        CflNext cfl;
        if (c.cfl_fused) cfl = CflNext{1, c.cfl_safety, c.cfl_dt_cap, c.cfl_inflow, c.M};
        launch_k(c, k_bnd_probe, std::min(cdiv(L.bfaces(), TPB), 4 * c.num_sms), TPB, 0, L, c.u, c.outlet_s,
                 c.sc.p, c.red.p, c.red_count.p, cfl);
        CK_LAUNCH();
    }
    c.c_down += L.n_sub;
}

void interface_solve(Ctx& c, bool refine) {
    const Layout& L = c.L;
    c.c_iface += 1;
    if (c.dim == 0) return;
    {
        PROF(c, "k_iface_rhs");
        launch_k(c, k_iface_rhs, grid_for(32LL * c.dim), TPB, 0, L, c.PU, c.beta_m, c.beta_p, c.irhs);
        CK_LAUNCH();
    }
    if (c.use_krylov) {
        krylov_solve(c, c.irhs, c.icoef);
        return;
    }
    if (c.use_blocktri) {
        bt_solve(c, c.irhs, c.icoef);
        return;
    }
    launch_gemv(c, c.Minv, c.irhs, c.icoef, c.dim);
    if (!refine) return;
    // one step of iterative refinement against the sparse operator
    for (int it = 0; it < 1; ++it) {
        launch_csr_residual(c, c.csr_ptr, c.csr_col, c.csr_val, c.icoef, c.irhs, c.ires, c.dim);
        launch_gemv_acc(c, c.Minv, c.ires, c.icoef, c.dim);  // x += M^-1 (b - M x)
    }
}



void configure_kernels() {
    CK(cudaFuncSetAttribute(k_factor_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_ds_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_part_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
}

void launch_rebuild(Ctx& c, const double* kappa, bool compute_beta) {  // compute_beta + mrcm_solve (simulation.cpp:183-193)
    const Layout& L = c.L;
    if (compute_beta) launch_beta(c, kappa);
    launch_trans(c, kappa);
    ds_factor_fork(c);  // downscale operator of kappa, concurrent with the basis rebuild
    launch_basis_core(c, kappa);
    interface_solve(c, true);  // the new inverse's rcond is not known yet
    // recon_m (kept for MPM steps) and its traces
    if (c.dim == 0) CK(cudaMemsetAsync(c.icoef, 0, sizeof(double), c.st));
    {
        PROF(c, "k_recon_traces");
        launch_k(c, k_recon_traces, grid_for((long long)L.n_sub * L.nbe), TPB, 0, L, c.icoef, c.PU, c.PB, c.HU, c.HB, nullptr,
                                                                               c.RU, c.bpm);
        CK_LAUNCH();
    }
    {
        PROF(c, "k_recon_p");
        launch_k(c, k_recon_p, grid_for(L.cells()), TPB, 0, L, c.max_rhs, c.icoef, c.X, c.pm);
        CK_LAUNCH();
    }
    {
        PROF(c, "k_sub_sum");
        launch_k(c, k_sub_sum, cdiv((long long)L.n_sub * 32, TPB), TPB, 0, L, c.pm, c.pmsum);
        CK_LAUNCH();
    }
    CK(cudaMemcpyAsync(c.RS, c.pmsum, L.n_sub * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
    if (c.rhs_w) {  // the MPM-2P edge data that stay fixed until the next rebuild (k_mpm_edges_kn)
        PROF(c, "k_mpm_rhs");
        launch_k(c, k_mpm_edges, std::min(grid_for((long long)L.n_sub * L.nbe), 8 * c.num_sms), TPB, 0, L, kappa,
                 c.kappa_m, c.bc_kind, c.bc_value, c.beta_m, c.beta_p, c.pm, c.bpm, c.MGZ, c.WU, c.MET, c.PD.p);
        CK_LAUNCH();
        c.mpm_static_ok = true;
    }
    downscale(c, kappa);
    c.has_basis = true;
}

// compute_basis_set (mrcm.cpp:132-240): with beta_m / beta_p and T =
// transmissibility(kappa) in place, factor every subdomain operator, solve
// the particular (q, bc) and homogeneous problems, their traces and pressure
// sums, assemble the interface matrix and factor it (with the rcond guard).
// Leaves the particular solution in X[s][0] and the homogeneous ones in
// X[s][1..]; kappa_m = kappa.
void launch_basis_core(Ctx& c, const double* kappa) {
    const Layout& L = c.L;
    c.mpm_static_ok = false;  // kappa_m changes: launch_rebuild re-forms the static MPM-2P edge data
    {
        PROF(c, "k_band_entries");
        launch_k(c, k_band_entries, grid_for(L.cells()), TPB, 0, L, kappa, c.T, 0, c.anchor_m ? 1 : 0, c.beta_m, c.beta_p,
                                                              c.bc_kind, c.BDm, c.BWm, c.BSm, c.sc);
        CK_LAUNCH();
    }
    {
        PROF(c, "k_rebuild_rhs");
        launch_k(c, k_rebuild_rhs, grid_for(L.cells()), TPB, 0, L, c.max_rhs, kappa, c.q, c.bc_kind, c.bc_value, c.beta_m,
                                                             c.beta_p, c.anchor_m ? 1 : 0, c.X);
        CK_LAUNCH();
    }
    const size_t smr = (size_t)WPB * band_smem_doubles(L.snx, RING_NR) * sizeof(double);
    if (c.twist_store) {  // two-sided factor (band_twist.cuh)
        {
            PROF(c, "k_factor_solve");
            switch (L.snx) {
#define X(BW_)                                                                                                  \
    case BW_:                                                                                                   \
        twist_configure<BW_>();                                                                                 \
        launch_k(c, k_factor1_t<BW_>, L.n_sub, twist_threads<BW_>(), twist_smem_bytes<BW_>(), L, c.max_rhs, c.BDm, c.BWm, c.BSm, c.Dm,   \
                                                                      c.Lcm, c.Lrm, c.tw_midb, c.tw_sinv, c.X, \
                                                                      c.sc);                                   \
        break;
                MPM2P_TWIST_WIDTHS(X)
#undef X
                default:
                    throw ConfigError("two-sided factor: unsupported subdomain width");
            }
            CK_LAUNCH();
        }
        if (L.max_hom > 0) {
            PROF(c, "k_hom_solve");
            switch (L.snx) {
#define X(BW_)                                                                                                  \
    case BW_:                                                                                                   \
        launch_k(c, k_hom_solve_t<BW_>, L.n_sub * L.max_hom, twist_threads<BW_>(), twist_smem_bytes<BW_>(),    \
            L, c.max_rhs, c.Dm, c.Lcm, c.Lrm, c.tw_midb, c.tw_sinv, c.X);                                       \
        break;
                MPM2P_TWIST_WIDTHS(X)
#undef X
                default:
                    break;
            }
            CK_LAUNCH();
        }
    } else {
        PROF(c, "k_factor_solve");
        switch (c.no_regband ? -1 : L.snx) {
#define X(BW_)                                                                                                      \
    case BW_:                                                                                                       \
        launch_k(c, k_factor1_r<BW_>, band_blocks(L), WPB * 32, 0, L, c.max_rhs, c.BDm, c.BWm, c.BSm, c.Dm, c.Lcm,   \
                                                                c.Lrm, c.X, c.sc);                                  \
        if (L.max_hom > 0) {                                                                                        \
            CK_LAUNCH();                                                                                            \
            PROF(c, "k_hom_solve");                                                                                 \
            if (c.hom_group > 1) {                                                                                  \
                const int groups = cdiv(L.max_hom, HOM_GROUP);                                                      \
                launch_k(c, k_hom_solve_rm<BW_, HOM_GROUP>, cdiv((long long)L.n_sub * groups, WPB), WPB * 32, 0,    \
                    L, c.max_rhs, groups, c.Dm, c.Lcm, c.Lrm, c.X);                                                 \
            } else {                                                                                                \
                launch_k(c, k_hom_solve_r<BW_>, cdiv((long long)L.n_sub * L.max_hom, WPB), WPB * 32, 0,             \
                    L, c.max_rhs, c.Dm, c.Lcm, c.Lrm, c.X);                                                         \
            }                                                                                                       \
        }                                                                                                           \
        break;
            MPM2P_BAND_WIDTHS(X)
#undef X
            default:
                launch_k(c, k_factor_solve, band_blocks(L), WPB * 32, smr, L, c.max_rhs, c.BDm, c.BWm, c.BSm, c.Dm,
                                                                        c.Lcm, c.Lrm, c.X, c.sc);
        }
        CK_LAUNCH();
    }
    {
        PROF(c, "k_rebuild_traces");
        launch_k(c, k_rebuild_traces, grid_for((long long)L.n_sub * L.nbe), TPB, 0, 
            L, c.max_rhs, kappa, c.bc_kind, c.bc_value, c.beta_m, c.beta_p, c.X, c.PU, c.PB, c.HU, c.HB);
        CK_LAUNCH();
    }
    {
        PROF(c, "k_psums");
        launch_k(c, k_psums, cdiv((long long)L.n_sub * c.max_rhs * 32, TPB), TPB, 0, L, c.max_rhs, c.X, c.PS, c.HP);
        CK_LAUNCH();
    }
    c.c_hom += c.nhat;
    c.c_part += L.n_sub;
    // interface matrix: assemble, invert, guard (mrcm.cpp:196-238)
    if (c.dim > 0) {
        {
            PROF(c, "k_assemble");
            launch_k(c, k_assemble, grid_for(c.nnz), TPB, 0, L, c.csr_row, c.csr_col, c.nnz, c.HU, c.beta_m, c.beta_p,
                                                          c.csr_val);
            CK_LAUNCH();
        }
        if (c.use_krylov) {
            // no dense factorisation: the rcond guard becomes MINRES
            // non-convergence (ERR_SINGULAR raised by k_minres)
            krylov_prepare(c);
        } else if (c.use_blocktri) {
            // block LDL^T; a zero / non-finite pivot in any block raises
            // ERR_SINGULAR, and so does the reference's rcond guard
            // (mrcm.cpp:227-238), estimated with the block solves
            krylov_prepare(c);
            bt_factor(c);
            bt_rcond(c, 1e-14, ERR_SINGULAR);
        } else if (!interface_inverse_csr(c, &c.sc.p->rcond, ERR_SINGULAR, 1e-14)) {
            // non-symmetric fallback through a dense copy of M
            c.Mdense.alloc((size_t)c.dim * c.dim);
            {
                PROF(c, "k_csr_to_dense");
                launch_k(c, k_csr_to_dense, c.dim, TPB, 0, c.csr_ptr, c.csr_col, c.csr_val, c.dim, c.Mdense);
                CK_LAUNCH();
            }
            // rcond guard (mrcm.cpp:227-238) is evaluated on the device; a trip
            // surfaces as ERR_SINGULAR at the step's scalar readback.
            interface_inverse_async(c, c.Mdense, c.Minv, c.dim, &c.sc.p->rcond, ERR_SINGULAR, 1e-14);
        }
    }
    if (kappa != c.kappa_m.p)
        CK(cudaMemcpyAsync(c.kappa_m, kappa, L.cells() * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
}

// The particular solve with the cached basis factor, in place on X[s][0]
// (mrcm.cpp:242-252). The register-window kernels also write the traces PU
// and pressure sums PS of the MPM-2P data (GZ); returns whether they did.
bool particular_solve_x(Ctx& c) {
    const Layout& L = c.L;
    const size_t sm1 = (size_t)WPB * band_smem_doubles(L.snx, 1) * sizeof(double);
    bool fused_traces = false;  // the register-window kernel also writes PU / PS
    if (c.twist_store) {
        PROF(c, "k_part_solve");
        switch (L.snx) {
#define X(BW_)                                                                                                  \
    case BW_:                                                                                                   \
        launch_k(c, k_part_solve_t<BW_>, L.n_sub, twist_threads<BW_>(), twist_smem_bytes<BW_>(),                  \
            L, c.max_rhs, c.Dm, c.Lcm, c.Lrm, c.tw_midb, c.tw_sinv, c.X, c.kappa_m, c.bc_kind, c.beta_m,        \
            c.beta_p, c.MGZ, c.PU, c.PS);                                                                        \
        break;
            MPM2P_TWIST_WIDTHS(X)
#undef X
            default:
                throw ConfigError("two-sided factor: unsupported subdomain width");
        }
        fused_traces = true;
        CK_LAUNCH();
    } else {
        PROF(c, "k_part_solve");
        switch (c.no_regband ? -1 : L.snx) {
#define X(BW_)                                                                                                  \
    case BW_:                                                                                                   \
        launch_k(c, k_part_solve_r<BW_>, band_blocks(L), WPB * 32, 0, L, c.max_rhs, c.Dm, c.Lcm, c.Lrm, c.X,     \
                                                                   c.kappa_m, c.bc_kind, c.beta_m, c.beta_p,   \
                                                                   c.MGZ, c.PU, c.PS);                          \
        fused_traces = true;                                                                                    \
        break;
            MPM2P_BAND_WIDTHS(X)
#undef X
            default:
                launch_k(c, k_part_solve, band_blocks(L), WPB * 32, sm1, L, c.max_rhs, c.Dm, c.Lcm, c.Lrm, c.X);
        }
        CK_LAUNCH();
    }
    return fused_traces;
}

void launch_mpm(Ctx& c, const double* kn) {  // mpm_pressure_update (mpm.cpp:31-114)
    const Layout& L = c.L;
    if (!c.has_basis) throw ConfigError("mpm_pressure_update: no basis set (rebuild first)");
    launch_trans(c, kn);
    ds_factor_fork(c);  // downscale operator of kappa_n, concurrent with the particular / interface chain
    {
        PROF(c, "k_mpm_rhs");
        if (c.rhs_w) {
            if (c.mpm_static_ok)  // the rebuild left PD and the static g' / terms in MGZ / MET
                launch_k(c, k_mpm_edges_kn, std::min(grid_for((long long)L.n_sub * L.nbe), 8 * c.num_sms), TPB, 0, L, kn,
                         c.bc_kind, c.bc_value, c.PD, c.MGZ, c.WU, c.MET);
            else
                launch_k(c, k_mpm_edges, std::min(grid_for((long long)L.n_sub * L.nbe), 8 * c.num_sms), TPB, 0, L, kn,
                         c.kappa_m, c.bc_kind, c.bc_value, c.beta_m, c.beta_p, c.pm, c.bpm, c.MGZ, c.WU, c.MET,
                         (double*)nullptr);
            CK_LAUNCH();
            launch_k(c, k_mpm_rhs_w, grid2d(c, L, red_blocks(c, k_mpm_rhs_w, L.cells())), TPB, 0, L, c.max_rhs,
                     c.anchor_m ? 1 : 0, c.T, c.q, c.pm, c.WU, c.MET, c.X);
        }
        else if (c.rhs_sub && L.ncs <= RHS_TPB * RHS_CPT)
            launch_k(c, k_mpm_rhs_sub, L.n_sub, RHS_TPB, (size_t)(L.ncs + 2 * L.nbe) * sizeof(double), L, c.max_rhs,
                     c.anchor_m ? 1 : 0, kn, c.kappa_m, c.T, c.q, c.bc_kind, c.bc_value, c.beta_m, c.beta_p, c.pm,
                     c.bpm, c.X, c.MGZ, c.WU);
        else
            launch_k(c, k_mpm_rhs, grid_for(L.cells()), TPB, 0, L, c.max_rhs, c.anchor_m ? 1 : 0, kn, c.kappa_m, c.T,
                     c.q, c.bc_kind, c.bc_value, c.beta_m, c.beta_p, c.pm, c.bpm, c.X, c.MGZ, c.WU);
        CK_LAUNCH();
    }
    const bool fused_traces = particular_solve_x(c);
    if (!fused_traces) {
        {
            PROF(c, "k_part_traces");
            launch_k(c, k_part_traces, grid_for((long long)L.n_sub * L.nbe), TPB, 0, 
                L, c.max_rhs, c.kappa_m, c.bc_kind, c.beta_m, c.beta_p, c.MGZ, c.X, c.PU);
            CK_LAUNCH();
        }
        {
            PROF(c, "k_part_psum");
            launch_k(c, k_part_psum, cdiv((long long)L.n_sub * 32, TPB), TPB, 0, L, c.max_rhs, c.X, c.PS);
            CK_LAUNCH();
        }
    }
    c.c_part += L.n_sub;
    interface_solve(c, c.refine);
    if (c.dim == 0) CK(cudaMemsetAsync(c.icoef, 0, sizeof(double), c.st));
    if (L.max_hom <= 16) {
        PROF(c, "k_recon_mpm");
        launch_k(c, k_recon_mpm, cdiv((long long)L.n_sub * 32, 128), 128, 0, L, c.icoef, c.PU, c.HU, c.WU, c.RU, c.PS,
                                                                          c.HP, c.pmsum, c.RS);
        CK_LAUNCH();
    } else {  // per-edge interface spaces: more homogeneous functions than k_recon_mpm keeps in registers
        {
            PROF(c, "k_recon_traces");
            launch_k(c, k_recon_traces, grid_for((long long)L.n_sub * L.nbe), TPB, 0, L, c.icoef, c.PU, nullptr, c.HU,
                                                                                   nullptr, c.WU, c.RU, nullptr);
            CK_LAUNCH();
        }
        {
            PROF(c, "k_recon_psum");
            launch_k(c, k_recon_psum, grid_for(L.n_sub), TPB, 0, L, c.icoef, c.PS, c.HP, c.pmsum, c.RS);
            CK_LAUNCH();
        }
    }
    downscale(c, kn);
}

}  // namespace mpm2p
