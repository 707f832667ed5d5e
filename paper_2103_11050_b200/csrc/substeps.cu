// substeps.cu — the MRCM sub-step entry points (proj/include/mrcmflow/mrcm.hpp:
// 77-136, 157-161) on the device: restrict_physical_data, solve_particular,
// solve_interface, reconstruct, averaged_skeleton_flux, downscale and
// weak_continuity_residuals, each over the per-subdomain LocalData /
// LocalSolution layouts of the C ABI (include/mpm2p_b200.h):
//   q_local / p_local   [s][r]    r = jj * snx + ii (local cells row-major)
//   u_local             [s][lf]   local faces: vertical (snx+1)*sny, then
//                                 horizontal snx*(sny+1); global orientation
//   bc_* / bp_local     [s][idx]  boundary edges W(sny) E(sny) S(snx) N(snx)
// The hot path (launch_rebuild / launch_mpm) keeps these fused; here each
// reference function is one call, for parity tests and for callers that
// drive the sub-steps themselves. Arithmetic follows the reference's
// unfused order (__dadd_rn / __dmul_rn) where it forms a sum of products.
#include "context.cuh"

namespace mpm2p {

namespace {

constexpr int TPB = 256;

__device__ __forceinline__ size_t xoff(const Layout& L, int max_rhs, int s, int m) {
    return ((size_t)s * max_rhs + m) * L.ncs;
}

__device__ __forceinline__ double edge_beta(const Layout& L, const EdgeInfo& e, const double* bm, const double* bp) {
    const int i = L.skel_index(e.iface, e.pos);
    return e.sign > 0 ? bm[i] : bp[i];
}

// restrict_physical_data (mrcm.cpp:104-130): sources per subdomain, skeleton
// edges Robin(beta, 0), physical edges copied from the global BoundarySpec
__global__ void k_sub_restrict(Layout L, const double* __restrict__ q, const int* __restrict__ bc_kind,
                               const double* __restrict__ bc_value, const double* __restrict__ bm,
                               const double* __restrict__ bp, double* __restrict__ qL, int* __restrict__ kindL,
                               double* __restrict__ valL, double* __restrict__ betaL, double* __restrict__ rhsL) {
    const long long ncell = (long long)L.n_sub * L.ncs, nedge = (long long)L.n_sub * L.nbe;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < ncell + nedge;
         x += (long long)gridDim.x * blockDim.x) {
        if (x < ncell) {
            const int s = (int)(x / L.ncs), r = (int)(x % L.ncs);
            qL[x] = q[L.gcell_of(s, r)];
            continue;
        }
        const long long y = x - ncell;
        const int s = (int)(y / L.nbe), idx = (int)(y % L.nbe);
        const EdgeInfo e = L.edge(s, idx);
        if (e.iface >= 0) {
            kindL[y] = BC_ROBIN;
            valL[y] = 0.0;
            betaL[y] = edge_beta(L, e, bm, bp);
            rhsL[y] = 0.0;
        } else {
            const int k = bc_kind[e.gbc];
            kindL[y] = k;
            valL[y] = k == BC_ROBIN ? 0.0 : bc_value[e.gbc];
            betaL[y] = k == BC_ROBIN ? L.rb_beta[e.gbc] : 0.0;
            rhsL[y] = k == BC_ROBIN ? L.rb_rhs[e.gbc] : 0.0;
        }
    }
}

// CellCenteredSolver::solve's right-hand side (elliptic.cpp:152-181) with the
// cached (kappa_m, beta) operator: q vol, then the cell's boundary faces in
// W, E, S, N order; the structure check of elliptic.cpp:155-160
__global__ void k_sub_rhs(Layout L, int max_rhs, int anchor, const double* __restrict__ km,
                          const double* __restrict__ qL, const int* __restrict__ kindL,
                          const double* __restrict__ valL, const double* __restrict__ betaL,
                          const double* __restrict__ rhsL, const int* __restrict__ bc_kind,
                          const double* __restrict__ bm, const double* __restrict__ bp, double* __restrict__ X,
                          Scalars* sc) {
    const long long ncell = (long long)L.n_sub * L.ncs;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < ncell;
         x += (long long)gridDim.x * blockDim.x) {
        const int s = (int)(x / L.ncs), r = (int)(x % L.ncs);
        const int ii = r % L.snx, jj = r / L.snx;
        const int gc = L.gcell_of(s, r);
        double b = __dmul_rn(qL[x], L.vol());
        const int ids[4] = {ii == 0 ? jj : -1, ii == L.snx - 1 ? L.sny + jj : -1, jj == 0 ? 2 * L.sny + ii : -1,
                            jj == L.sny - 1 ? 2 * L.sny + L.snx + ii : -1};
        for (int t = 0; t < 4; ++t) {
            const int idx = ids[t];
            if (idx < 0) continue;
            const EdgeInfo e = L.edge(s, idx);
            const size_t o = (size_t)s * L.nbe + idx;
            const int kind = kindL[o];
            // the factorization's structure: skeleton Robin(beta), physical kinds
            const int k0 = e.iface >= 0 ? BC_ROBIN : bc_kind[e.gbc];
            const double b0 = e.iface >= 0 ? edge_beta(L, e, bm, bp) : (k0 == BC_ROBIN ? L.rb_beta[e.gbc] : 0.0);
            if (kind != k0 || (kind == BC_ROBIN && betaL[o] != b0)) atomicOr(&sc->err, ERR_STRUCT);
            const double th = half_trans(L, e.side, km[gc]);
            if (kind == BC_PRESSURE) b = __dadd_rn(b, __dmul_rn(th, valL[o]));
            else if (kind == BC_FLUX) b = __dsub_rn(b, __dmul_rn(valL[o], e.area));
            else b = __dadd_rn(b, __dmul_rn(eff_robin(th, betaL[o], e.area), rhsL[o]));
        }
        if (anchor && r == 0) b = 0.0;
        X[xoff(L, max_rhs, s, 0) + r] = b;
    }
}

__device__ __forceinline__ int lfaces(const Layout& L) { return L.lvcount() + L.snx * (L.sny + 1); }

// The local solution (elliptic.cpp:214-241) of one right-hand side m of X:
// p, u on every local face (interior: harmonic transmissibility of kappa_m;
// boundary: the edge's condition) and the boundary-face pressures.
__global__ void k_sub_local_solution(Layout L, int max_rhs, const double* __restrict__ km,
                                     const double* __restrict__ X, const int* __restrict__ kindL,
                                     const double* __restrict__ valL, const double* __restrict__ betaL,
                                     const double* __restrict__ rhsL, double* __restrict__ pL,
                                     double* __restrict__ uL, double* __restrict__ bpL) {
    const int nf = lfaces(L);
    const long long ncell = (long long)L.n_sub * L.ncs, nface = (long long)L.n_sub * nf;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < ncell + nface;
         x += (long long)gridDim.x * blockDim.x) {
        if (x < ncell) {
            const int s = (int)(x / L.ncs), r = (int)(x % L.ncs);
            pL[x] = X[xoff(L, max_rhs, s, 0) + r];
            continue;
        }
        const long long y = x - ncell;
        const int s = (int)(y / nf), lf = (int)(y % nf);
        const double* xs = X + xoff(L, max_rhs, s, 0);
        int idx = -1;  // boundary edge of this face, if any
        double u = 0.0;
        if (lf < L.lvcount()) {
            const int i = lf % (L.snx + 1), j = lf / (L.snx + 1);
            if (i == 0) idx = j;
            else if (i == L.snx) idx = L.sny + j;
            else {
                const double t = harm_trans_v(L, km[L.gcell_of(s, j * L.snx + i - 1)], km[L.gcell_of(s, j * L.snx + i)]);
                u = __ddiv_rn(__dmul_rn(t, __dsub_rn(xs[j * L.snx + i - 1], xs[j * L.snx + i])), L.hy);
            }
        } else {
            const int h = lf - L.lvcount(), i = h % L.snx, j = h / L.snx;
            if (j == 0) idx = 2 * L.sny + i;
            else if (j == L.sny) idx = 2 * L.sny + L.snx + i;
            else {
                const double t =
                    harm_trans_h(L, km[L.gcell_of(s, (j - 1) * L.snx + i)], km[L.gcell_of(s, j * L.snx + i)]);
                u = __ddiv_rn(__dmul_rn(t, __dsub_rn(xs[(j - 1) * L.snx + i], xs[j * L.snx + i])), L.hx);
            }
        }
        if (idx >= 0) {
            const EdgeInfo e = L.edge(s, idx);
            const size_t o = (size_t)s * L.nbe + idx;
            const double th = half_trans(L, e.side, km[e.global_cell]);
            const double pc = xs[e.local_cell];
            const int kind = kindL[o];
            double un, pf;
            if (kind == BC_PRESSURE) {
                un = __ddiv_rn(__dmul_rn(th, __dsub_rn(pc, valL[o])), e.area);
                pf = valL[o];
            } else if (kind == BC_FLUX) {
                un = valL[o];
                pf = __dsub_rn(pc, __ddiv_rn(__dmul_rn(valL[o], e.area), th));
            } else {
                const double te = eff_robin(th, betaL[o], e.area);
                un = __ddiv_rn(__dmul_rn(te, __dsub_rn(pc, rhsL[o])), e.area);
                pf = __dadd_rn(rhsL[o], __dmul_rn(betaL[o], un));
            }
            u = e.sign * un;
            bpL[o] = pf;
        }
        uL[y] = u;
    }
}

// outward normal velocity per boundary edge from a local solution's u
__global__ void k_sub_traces(Layout L, const double* __restrict__ uL, double* __restrict__ U) {
    const int nf = lfaces(L);
    const long long ne = (long long)L.n_sub * L.nbe;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < ne; x += (long long)gridDim.x * blockDim.x) {
        const int s = (int)(x / L.nbe), idx = (int)(x % L.nbe);
        const EdgeInfo e = L.edge(s, idx);
        U[x] = e.sign * uL[(size_t)s * nf + e.local_face];
    }
}

// reconstruct (mrcm.cpp:270-288): particular + sum_h c_h hom_h in hom order,
// zero coefficients skipped; the homogeneous solutions' p are X[s][1 + h],
// their interior face velocities re-formed with the basis operator, their
// boundary traces HU (outward) and pressures HB
__global__ void k_sub_reconstruct(Layout L, int max_rhs, const double* __restrict__ km,
                                  const double* __restrict__ coef, const double* __restrict__ X,
                                  const double* __restrict__ HU, const double* __restrict__ HB,
                                  const double* __restrict__ pL, const double* __restrict__ uL,
                                  const double* __restrict__ bpL, double* __restrict__ pO, double* __restrict__ uO,
                                  double* __restrict__ bpO) {
    const int nf = lfaces(L);
    const long long ncell = (long long)L.n_sub * L.ncs, nface = (long long)L.n_sub * nf,
                    nedge = (long long)L.n_sub * L.nbe;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < ncell + nface + nedge;
         x += (long long)gridDim.x * blockDim.x) {
        if (x < ncell) {
            const int s = (int)(x / L.ncs), r = (int)(x % L.ncs);
            double v = pL[x];
            for (int h = 0; h < L.n_hom(s); ++h) {
                int k, t, col;
                bool fl;
                L.hom(s, h, k, t, fl, col);
                const double cv = coef[col];
                if (cv == 0.0) continue;
                v = __dadd_rn(v, __dmul_rn(cv, X[xoff(L, max_rhs, s, 1 + h) + r]));
            }
            pO[x] = v;
        } else if (x < ncell + nface) {
            const long long y = x - ncell;
            const int s = (int)(y / nf), lf = (int)(y % nf);
            double v = uL[y];
            int idx = -1, ca = -1, cb = -1;
            bool vert = lf < L.lvcount();
            double t = 0.0;
            if (vert) {
                const int i = lf % (L.snx + 1), j = lf / (L.snx + 1);
                if (i == 0) idx = j;
                else if (i == L.snx) idx = L.sny + j;
                else {
                    ca = j * L.snx + i - 1, cb = j * L.snx + i;
                    t = harm_trans_v(L, km[L.gcell_of(s, ca)], km[L.gcell_of(s, cb)]);
                }
            } else {
                const int h = lf - L.lvcount(), i = h % L.snx, j = h / L.snx;
                if (j == 0) idx = 2 * L.sny + i;
                else if (j == L.sny) idx = 2 * L.sny + L.snx + i;
                else {
                    ca = (j - 1) * L.snx + i, cb = j * L.snx + i;
                    t = harm_trans_h(L, km[L.gcell_of(s, ca)], km[L.gcell_of(s, cb)]);
                }
            }
            const double sgn = idx >= 0 ? L.edge(s, idx).sign : 1.0;
            for (int h = 0; h < L.n_hom(s); ++h) {
                int k, tt, col;
                bool fl;
                L.hom(s, h, k, tt, fl, col);
                const double cv = coef[col];
                if (cv == 0.0) continue;
                double uh;
                if (idx >= 0) {
                    uh = sgn * HU[((size_t)s * L.max_hom + h) * L.nbe + idx];
                } else {
                    const double* xh = X + xoff(L, max_rhs, s, 1 + h);
                    uh = __ddiv_rn(__dmul_rn(t, __dsub_rn(xh[ca], xh[cb])), vert ? L.hy : L.hx);
                }
                v = __dadd_rn(v, __dmul_rn(cv, uh));
            }
            uO[y] = v;
        } else {
            const long long y = x - ncell - nface;
            const int s = (int)(y / L.nbe), idx = (int)(y % L.nbe);
            double v = bpL[y];
            for (int h = 0; h < L.n_hom(s); ++h) {
                int k, tt, col;
                bool fl;
                L.hom(s, h, k, tt, fl, col);
                const double cv = coef[col];
                if (cv == 0.0) continue;
                v = __dadd_rn(v, __dmul_rn(cv, HB[((size_t)s * L.max_hom + h) * L.nbe + idx]));
            }
            bpO[y] = v;
        }
    }
}

// averaged_skeleton_flux (mrcm.cpp:290-304): per skeleton edge, interface-major
__global__ void k_sub_skel(Layout L, const double* __restrict__ uL, double* __restrict__ flux) {
    const int nf = lfaces(L);
    const int E = L.skeleton_edges();
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < E; x += gridDim.x * blockDim.x) {
        const int k = x < L.NV * L.sny ? x / L.sny : L.NV + (x - L.NV * L.sny) / L.snx;
        const int pos = x < L.NV * L.sny ? x % L.sny : (x - L.NV * L.sny) % L.snx;
        const int sm = L.iface_minus(k), sp = L.iface_plus(k);
        const double um = uL[(size_t)sm * nf + L.edge(sm, L.edge_index_on_iface(sm, k, pos)).local_face];
        const double up = uL[(size_t)sp * nf + L.edge(sp, L.edge_index_on_iface(sp, k, pos)).local_face];
        flux[L.skel_index(k, pos)] = 0.5 * __dadd_rn(um, up);
    }
}

// per-subdomain sums of a local cell field, in local order
__global__ void k_sub_psum(Layout L, const double* __restrict__ pL, double* __restrict__ out) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= L.n_sub) return;
    double v = 0.0;
    for (int r = 0; r < L.ncs; ++r) v = __dadd_rn(v, pL[(size_t)s * L.ncs + r]);
    out[s] = v;
}

// weak_continuity_residuals (mrcm.cpp:459-483): one warp per interface-system
// row — pressure-basis rows sum u.n psi over both sides, flux-basis rows the
// pressure jump -sign p_face phi — then the max of |row| per family
__global__ void k_sub_weak(Layout L, const double* __restrict__ U, const double* __restrict__ BP,
                           double* __restrict__ rowabs) {
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
        const int s = a == 0 ? L.iface_minus(k) : L.iface_plus(k);
        const double sign = a == 0 ? 1.0 : -1.0;
        const int idx = L.edge_index_on_iface(s, k, pos);
        const double v = L.basis_val(k, rt, pos);
        if (phi) acc -= sign * BP[(size_t)s * L.nbe + idx] * v * len;
        else acc += U[(size_t)s * L.nbe + idx] * v * len;
    }
    acc = warp_sum(acc);
    if (lane == 0) rowabs[row] = fabs(acc);
}

__global__ void k_sub_weak_max(int np, const double* __restrict__ rowabs, double* __restrict__ out) {
    __shared__ double sh[2][32];
    double a = 0.0, b = 0.0;
    for (int r = threadIdx.x; r < np; r += blockDim.x) {
        a = fmax(a, rowabs[r]);
        b = fmax(b, rowabs[np + r]);
    }
    a = warp_max(a);
    b = warp_max(b);
    if ((threadIdx.x & 31) == 0) {
        sh[0][threadIdx.x >> 5] = a;
        sh[1][threadIdx.x >> 5] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            sh[0][0] = fmax(sh[0][0], sh[0][w]);
            sh[1][0] = fmax(sh[1][0], sh[1][w]);
        }
        out[0] = sh[0][0];  // flux_jump (pressure-basis rows)
        out[1] = sh[1][0];  // pressure_jump (flux-basis rows)
    }
}

int grid_of(long long n) { return (int)std::max(1LL, std::min((n + TPB - 1) / TPB, 65535LL)); }

}  // namespace

int sub_local_faces(const Layout& L) { return L.lvcount() + L.snx * (L.sny + 1); }

void sub_restrict(Ctx& c, double* qL, int* kindL, double* valL, double* betaL, double* rhsL) {
    const Layout& L = c.L;
    launch_k(c, k_sub_restrict, grid_of((long long)L.n_sub * (L.ncs + L.nbe)), TPB, 0, L, c.q.p, c.bc_kind.p,
             c.bc_value.p, c.beta_m.p, c.beta_p.p, qL, kindL, valL, betaL, rhsL);
    CK_LAUNCH();
}

void sub_solve_particular(Ctx& c, const double* qL, const int* kindL, const double* valL, const double* betaL,
                          const double* rhsL, double* pL, double* uL, double* bpL) {
    const Layout& L = c.L;
    launch_k(c, k_sub_rhs, grid_of((long long)L.n_sub * L.ncs), TPB, 0, L, c.max_rhs, c.anchor_m ? 1 : 0,
             c.kappa_m.p, qL, kindL, valL, betaL, rhsL, c.bc_kind.p, c.beta_m.p, c.beta_p.p, c.X.p, c.sc.p);
    CK_LAUNCH();
    particular_solve_x(c);
    launch_k(c, k_sub_local_solution, grid_of((long long)L.n_sub * (L.ncs + sub_local_faces(L))), TPB, 0, L,
             c.max_rhs, c.kappa_m.p, c.X.p, kindL, valL, betaL, rhsL, pL, uL, bpL);
    CK_LAUNCH();
    c.c_part += L.n_sub;
}

void sub_solve_interface(Ctx& c, const double* uL) {
    const Layout& L = c.L;
    launch_k(c, k_sub_traces, grid_of((long long)L.n_sub * L.nbe), TPB, 0, L, uL, c.PU.p);
    CK_LAUNCH();
    interface_solve(c, c.refine);
    if (c.dim == 0) CK(cudaMemsetAsync(c.icoef, 0, sizeof(double), c.st));
}

void sub_reconstruct(Ctx& c, const double* coef, const double* pL, const double* uL, const double* bpL,
                     double* pO, double* uO, double* bpO) {
    const Layout& L = c.L;
    launch_k(c, k_sub_reconstruct, grid_of((long long)L.n_sub * (L.ncs + sub_local_faces(L) + L.nbe)), TPB, 0, L,
             c.max_rhs, c.kappa_m.p, coef, c.X.p, c.HU.p, c.HB.p, pL, uL, bpL, pO, uO, bpO);
    CK_LAUNCH();
}

void sub_skeleton_flux(Ctx& c, const double* uL, double* flux) {
    const Layout& L = c.L;
    if (L.skeleton_edges() == 0) return;
    launch_k(c, k_sub_skel, grid_of(L.skeleton_edges()), TPB, 0, L, uL, flux);
    CK_LAUNCH();
}

// downscale with a given reconstruction and skeleton flux: RU, RS and skel
// from the caller's arrays, then the hot path's repair / Neumann solves /
// scatter (solver.cu downscale) with T = transmissibility(kappa)
void sub_downscale(Ctx& c, const double* kappa, const double* pL, const double* uL, const double* flux) {
    const Layout& L = c.L;
    launch_k(c, k_sub_traces, grid_of((long long)L.n_sub * L.nbe), TPB, 0, L, uL, c.RU.p);
    CK_LAUNCH();
    launch_k(c, k_sub_psum, grid_of(L.n_sub), TPB, 0, L, pL, c.RS.p);
    CK_LAUNCH();
    if (L.skeleton_edges() > 0)
        CK(cudaMemcpyAsync(c.skel.p, flux, L.skeleton_edges() * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
    c.trans_fresh = false;
    launch_trans(c, kappa);
    downscale(c, kappa, true);
}

void sub_weak_residuals(Ctx& c, const double* uL, const double* bpL, double* out2) {
    const Layout& L = c.L;
    const int np = L.dim_flux;
    if (np == 0) {
        CK(cudaMemsetAsync(out2, 0, 2 * sizeof(double), c.st));
        return;
    }
    launch_k(c, k_sub_traces, grid_of((long long)L.n_sub * L.nbe), TPB, 0, L, uL, c.RU.p);
    CK_LAUNCH();
    launch_k(c, k_sub_weak, grid_of(64LL * np), TPB, 0, L, (const double*)c.RU.p, bpL, c.ires.p);
    CK_LAUNCH();
    launch_k(c, k_sub_weak_max, 1, 1024, 0, np, (const double*)c.ires.p, out2);
    CK_LAUNCH();
}

}  // namespace mpm2p
