// layout.cuh — host+device index arithmetic for the grid, the decomposition
// and the interface space. Closed-form versions of the tables the reference
// builds with loops (bit-exact integer indexing is part of the parity
// contract):
//   grid faces            proj/include/mrcmflow/grid.hpp:9-13
//   subdomains/interfaces proj/src/decomposition.cpp:35-132
//   boundary-edge order   W(ny) E(ny) S(nx) N(nx), decomposition.cpp:101-129
//   global BC index       proj/src/mrcm.cpp:14-28
//   interface bases       proj/src/interface_space.cpp:9-52
//   hom column order      proj/src/mrcm.cpp:157-189 (incident interfaces
//                         ascending; all flux bases, then all pressure bases)
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define HD __host__ __device__ __forceinline__
#else
#define HD inline
#endif

namespace mpm2p {

enum { BC_PRESSURE = 0, BC_FLUX = 1, BC_ROBIN = 2 };
enum { SIDE_W = 0, SIDE_E = 1, SIDE_S = 2, SIDE_N = 3 };

struct EdgeInfo {
    int side;         // W,E,S,N
    int along;        // jj (W/E) or ii (S/N)
    int local_cell;   // row-major in the subdomain
    int local_face;   // subdomain-local face index
    int global_cell;
    int global_face;
    int iface;        // -1 for a physical boundary edge
    int pos;          // position on the interface
    int gbc;          // index into the global BoundarySpec (physical edges), else -1
    double sign;      // side_sign: -1 W/S, +1 E/N (decomposition.hpp:14-16)
    double area;
};

struct Layout {
    // grid (grid.hpp:14-43)
    int nx, ny;
    double lx, ly, hx, hy;
    // decomposition
    int nsx, nsy, snx, sny;
    int n_sub, NV, NH, n_iface;
    int nbe;    // boundary edges per subdomain = 2(snx+sny)
    int ncs;    // cells per subdomain
    // interface space: bases per vertical / horizontal interface
    int space_kind;  // 0 constant, 1 linear
    int segv, segh;  // constant: segment length in edges
    int nbv, nbh;
    int dim_flux;    // == dim_pressure
    int max_hom;     // max homogeneous solves per subdomain
    const int4* homtab = nullptr;  // device table of hom(s, h) (set once the context exists)
    // physical Robin faces (FaceBc::beta / robin_rhs by global BoundarySpec
    // index; elliptic.hpp:16-28), device pointers, read only where
    // bc_kind == BC_ROBIN
    const double* rb_beta = nullptr;
    const double* rb_rhs = nullptr;
    // hx, hy (hence vol) exact powers of two: a division by them is then the
    // multiplication by the exact reciprocal, bit for bit (both round the same
    // real number), and the hot kernels take that path
    bool pow2 = false;
    double inv_hx = 0.0, inv_hy = 0.0, inv_vol = 0.0;

    HD int cells() const { return nx * ny; }
    HD int vcount() const { return (nx + 1) * ny; }
    HD int faces() const { return vcount() + nx * (ny + 1); }
    HD int bfaces() const { return 2 * (nx + ny); }
    HD int cell(int i, int j) const { return j * nx + i; }
    HD int vface(int i, int j) const { return j * (nx + 1) + i; }
    HD int hface(int i, int j) const { return vcount() + j * nx + i; }
    HD double vol() const { return hx * hy; }
    HD double area(int f) const { return f < vcount() ? hy : hx; }
    // x / hx, x / hy, x / vol with the reference's rounding
#ifdef __CUDA_ARCH__
    __device__ double div_hx(double x) const { return pow2 ? __dmul_rn(x, inv_hx) : __ddiv_rn(x, hx); }
    __device__ double div_hy(double x) const { return pow2 ? __dmul_rn(x, inv_hy) : __ddiv_rn(x, hy); }
    __device__ double div_vol(double x) const { return pow2 ? __dmul_rn(x, inv_vol) : __ddiv_rn(x, hx * hy); }
#else
    double div_hx(double x) const { return x / hx; }
    double div_hy(double x) const { return x / hy; }
    double div_vol(double x) const { return x / vol(); }
#endif

    // subdomain-local grid (snx x sny, same spacing)
    HD int lvcount() const { return (snx + 1) * sny; }
    HD int lfaces() const { return lvcount() + snx * (sny + 1); }
    HD int lvface(int i, int j) const { return j * (snx + 1) + i; }
    HD int lhface(int i, int j) const { return lvcount() + j * snx + i; }

    HD int sub_i0(int s) const { return (s % nsx) * snx; }
    HD int sub_j0(int s) const { return (s / nsx) * sny; }
    HD int gcell_of(int s, int lc) const {
        return cell(sub_i0(s) + lc % snx, sub_j0(s) + lc / snx);
    }

    // interfaces (decomposition.cpp:62-87)
    HD bool iface_vertical(int k) const { return k < NV; }
    HD int iface_edges(int k) const { return k < NV ? sny : snx; }
    HD int iface_minus(int k) const {
        if (k < NV) { const int sy = k / (nsx - 1), sx = k % (nsx - 1); return sy * nsx + sx; }
        const int kk = k - NV;
        return kk;  // (sy*nsx + sx) with sy = kk / nsx
    }
    HD int iface_plus(int k) const {
        return k < NV ? iface_minus(k) + 1 : iface_minus(k) + nsx;
    }
    HD int iface_face(int k, int pos) const {
        if (k < NV) {
            const int sy = k / (nsx - 1), sx = k % (nsx - 1);
            return vface((sx + 1) * snx, sy * sny + pos);
        }
        const int kk = k - NV, sy = kk / nsx, sx = kk % nsx;
        return hface(sx * snx + pos, (sy + 1) * sny);
    }
    // cells on either side of an interface edge (robin.cpp:13-24)
    HD void iface_cells(int k, int pos, int& cm, int& cp) const {
        if (k < NV) {
            const int sy = k / (nsx - 1), sx = k % (nsx - 1);
            const int i = (sx + 1) * snx, j = sy * sny + pos;
            cm = cell(i - 1, j);
            cp = cell(i, j);
        } else {
            const int kk = k - NV, sy = kk / nsx, sx = kk % nsx;
            const int i = sx * snx + pos, j = (sy + 1) * sny;
            cm = cell(i, j - 1);
            cp = cell(i, j);
        }
    }
    // flattened skeleton-edge index of (k, pos): interface-major
    HD int skel_index(int k, int pos) const {
        return k < NV ? k * sny + pos : NV * sny + (k - NV) * snx + pos;
    }
    HD int skeleton_edges() const { return NV * sny + NH * snx; }

    // interface space (interface_space.cpp:9-52)
    HD int iface_nb(int k) const { return k < NV ? nbv : nbh; }
    HD int iface_first_basis(int k) const { return k < NV ? k * nbv : NV * nbv + (k - NV) * nbh; }
    HD int basis_iface(int b) const {
        const int nvb = NV * nbv;
        return b < nvb ? b / nbv : NV + (b - nvb) / nbh;
    }
    // value of basis t (0-based on interface k) at edge e
    HD double basis_val(int k, int t, int e) const {
        const int n = iface_edges(k);
        if (space_kind == 1) return t == 0 ? 1.0 : 2.0 * (e + 0.5) / n - 1.0;
        const int seg = k < NV ? segv : segh;
        return (e >= t * seg && e < (t + 1) * seg) ? 1.0 : 0.0;
    }

    // incident interfaces of s in ascending id order (mrcm.cpp:157-162): W,E,S,N
    HD int incident(int s, int* out) const {
        const int sx = s % nsx, sy = s / nsx;
        int n = 0;
        if (sx > 0) out[n++] = sy * (nsx - 1) + sx - 1;
        if (sx < nsx - 1) out[n++] = sy * (nsx - 1) + sx;
        if (sy > 0) out[n++] = NV + (sy - 1) * nsx + sx;
        if (sy < nsy - 1) out[n++] = NV + sy * nsx + sx;
        return n;
    }
    HD int n_hom(int s) const {
        int inc[4];
        const int n = incident(s, inc);
        int c = 0;
        for (int i = 0; i < n; ++i) c += iface_nb(inc[i]);
        return 2 * c;
    }
    // homogeneous solve h of subdomain s: interface, basis t on it, flux?, column
    HD void hom(int s, int h, int& k, int& t, bool& flux, int& col) const {
#ifdef __CUDA_ARCH__
        if (homtab) {  // precomputed (interface, basis, flux?, column) per (subdomain, function)
            const int4 v = homtab[(size_t)s * max_hom + h];
            k = v.x;
            t = v.y;
            flux = v.z != 0;
            col = v.w;
            return;
        }
#endif
        int inc[4];
        const int n = incident(s, inc);
        int half = 0;
        for (int i = 0; i < n; ++i) half += iface_nb(inc[i]);
        flux = h < half;
        int r = flux ? h : h - half;
        k = inc[0];
        t = 0;
        for (int i = 0; i < n; ++i) {
            const int nb = iface_nb(inc[i]);
            if (r < nb) {
                k = inc[i];
                t = r;
                break;
            }
            r -= nb;
        }
        const int b = iface_first_basis(k) + t;
        col = flux ? b : dim_flux + b;
    }

    // boundary edge idx of subdomain s (decomposition.cpp:101-129, mrcm.cpp:14-28)
    HD EdgeInfo edge(int s, int idx) const {
        EdgeInfo e;
        const int sx = s % nsx, sy = s / nsx;
        const int i0 = sx * snx, j0 = sy * sny;
        e.iface = -1;
        e.pos = -1;
        e.gbc = -1;
        if (idx < sny) {
            const int jj = idx;
            e.side = SIDE_W; e.along = jj; e.sign = -1.0; e.area = hy;
            e.local_cell = jj * snx;
            e.local_face = lvface(0, jj);
            e.global_face = vface(i0, j0 + jj);
            if (sx > 0) { e.iface = sy * (nsx - 1) + sx - 1; e.pos = jj; }
            else e.gbc = j0 + jj;
        } else if (idx < 2 * sny) {
            const int jj = idx - sny;
            e.side = SIDE_E; e.along = jj; e.sign = 1.0; e.area = hy;
            e.local_cell = jj * snx + snx - 1;
            e.local_face = lvface(snx, jj);
            e.global_face = vface(i0 + snx, j0 + jj);
            if (sx < nsx - 1) { e.iface = sy * (nsx - 1) + sx; e.pos = jj; }
            else e.gbc = ny + j0 + jj;
        } else if (idx < 2 * sny + snx) {
            const int ii = idx - 2 * sny;
            e.side = SIDE_S; e.along = ii; e.sign = -1.0; e.area = hx;
            e.local_cell = ii;
            e.local_face = lhface(ii, 0);
            e.global_face = hface(i0 + ii, j0);
            if (sy > 0) { e.iface = NV + (sy - 1) * nsx + sx; e.pos = ii; }
            else e.gbc = 2 * ny + i0 + ii;
        } else {
            const int ii = idx - 2 * sny - snx;
            e.side = SIDE_N; e.along = ii; e.sign = 1.0; e.area = hx;
            e.local_cell = (sny - 1) * snx + ii;
            e.local_face = lhface(ii, sny);
            e.global_face = hface(i0 + ii, j0 + sny);
            if (sy < nsy - 1) { e.iface = NV + sy * nsx + sx; e.pos = ii; }
            else e.gbc = 2 * ny + nx + i0 + ii;
        }
        e.global_cell = cell(i0 + e.local_cell % snx, j0 + e.local_cell / snx);
        return e;
    }
    // boundary-edge index of subdomain s that lies on interface k at pos
    HD int edge_index_on_iface(int s, int k, int pos) const {
        const bool minus = iface_minus(k) == s;
        if (k < NV) return minus ? sny + pos : pos;          // minus: its East side; plus: West
        return minus ? 2 * sny + snx + pos : 2 * sny + pos;  // minus: North; plus: South
    }
};

// Local subdomain half transmissibility of a boundary face: kappa*area/(h/2)
// (elliptic.cpp:48-49,54-55).
HD double half_trans(const Layout& L, int side, double kappa) {
    return (side == SIDE_W || side == SIDE_E) ? kappa * L.hy / (L.hx / 2.0) : kappa * L.hx / (L.hy / 2.0);
}
// effective Robin transmissibility (elliptic.cpp:24-26)
HD double eff_robin(double t_half, double beta, double area) {
    return 1.0 / (1.0 / t_half + beta / area);
}
// harmonic-mean interior transmissibility (elliptic.cpp:46,50,56)
HD double harm_trans_v(const Layout& L, double a, double b) { return L.div_hx(2.0 * a * b / (a + b) * L.hy); }
HD double harm_trans_h(const Layout& L, double a, double b) { return L.div_hy(2.0 * a * b / (a + b) * L.hx); }

}  // namespace mpm2p
