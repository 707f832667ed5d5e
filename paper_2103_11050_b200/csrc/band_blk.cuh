// band_blk.cuh — blocked banded LDL^T of the 5-point subdomain operator on the
// fp64 tensor cores (DMMA, mma.sync.m8n8k4.f64), one warp per subdomain.
//
// Replaces Eigen SimplicialLDLT (proj/src/elliptic.cpp:68-199) for the fresh
// per-step downscale solves (proj/src/mrcm.cpp:388-427) at bandwidths that are
// multiples of 8 (C4/C5: 32). Same mathematics as band_reg.cuh, reorganised
// into 8-pivot panels so the rank-8 Schur updates run as 8x8x4 DMMA tiles:
//
//  * A is symmetric positive definite with half-bandwidth B (cells row-major
//    in a snx = B wide subdomain): diagonal, west (offset 1) and south (offset
//    B) couplings. Panel p eliminates rows k0 = 8p .. k0+7 against a sliding
//    window of rows k0 .. k0+B+7, held as the lower (NT+1) x (NT+1) triangle
//    of 8x8 tiles, NT = B/8, in DMMA accumulator layout (lane l: tile row l/4,
//    columns 2(l%4), 2(l%4)+1). Everything left of the window is final.
//  * Block LDL^T with 8x8 pivot blocks: G = S11^-1 (Gauss-Jordan, in shared
//    memory, 2x2 pivot blocks, no pivoting: S11 is SPD), X = S21 G, S22 -= X S21^T. Row tile NT
//    of S21 holds only the original south couplings of the rows that just
//    entered (a diagonal tile), so its products are row scalings: X_NT =
//    diag(s) G, S22[NT][J] -= diag(s) X_J^T, S22[NT][NT] -= diag(s) G diag(s).
//    DMMA count per panel: 2(NT-1) for X plus NT(NT-1) for the update
//    (C5: 18 DMMA per 8 pivots).
//  * Solve: forward y2 -= X y1 and t1 = G y1 fused into the factorisation
//    (DMMA with y1 as column 0 of the B operand);
//    backward x1 = t1 - X^T x2. Only X (B x 8 per panel, the accumulator
//    fragments as they are) and t1 are stored: n*B + n doubles per subdomain,
//    the same footprint as the scalar factor's L.
#pragma once

#include "band.cuh"

namespace mpm2p {

// D += A B, m8n8k4 fp64: A 8x4 row-major (lane l: A[l/4][l%4]), B 4x8
// (lane l: B[l%4][l/4]), C/D 8x8 (lane l: D[l/4][2(l%4) + {0,1}]).
__device__ __forceinline__ void blk_dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int B>
__host__ __device__ constexpr int blk_nt() {
    return B / 8;
}
// per-warp shared memory (doubles): two Gauss-Jordan buffers, NT tiles of
// S21, NT tiles of X, 8 right-hand-side values
template <int B>
__host__ __device__ constexpr int blk_smem_doubles() {
    return 2 * 64 + 2 * blk_nt<B>() * 64 + 8;
}

struct BlkTile {
    double v[2];
};

// Entries of row tile `t` (rows 8t..8t+7) as they enter the window: its
// diagonal tile (tridiagonal: diag, west, and the mirrored west coupling of
// the next row), the west coupling of row 8t into tile t-1 (entry (0,7)) and
// the south couplings into tile t-NT (diagonal). Rows >= n are identity rows.
// A source's fetch() issues raw loads only (clamped, always-valid addresses):
// a loaded value is first touched one panel later, when the row enters the
// window, so the load never stalls the panel that issues it; decode() forms
// the row's diag / west / next row's west / south / rhs from them then.
struct BlkRowData {
    double a0, a1, a2, a3, b;
};
// the stored band rows BD / BW / BS of k_ds_prep / k_band_entries
struct BlkBandSrc {
    BandRows A;
    const double* y;
    int n;
    __device__ __forceinline__ BlkRowData fetch(int row) const {
        const int rr = row < n ? row : n - 1;
        const int r1 = row + 1 < n ? row + 1 : n - 1;
        return BlkRowData{A.diag[rr], A.offw[rr], A.offw[r1], A.offs[rr], y[rr]};
    }
    __device__ __forceinline__ void decode(int, const BlkRowData& e, double& d, double& w, double& w1,
                                           double& s) const {
        d = e.a0, w = e.a1, w1 = e.a2, s = e.a3;
    }
};
// the downscale operator straight from the global transmissibilities T of
// kappa_n (pure Neumann, anchor cell 0; k_ds_prep's rules and summation
// order, mrcm.cpp:391-411): no band rows are written or read back
struct BlkTransSrc {
    const double* T;
    const double* y;
    int n, snx, sny, nx, vcount, i0, j0;
    __device__ __forceinline__ BlkRowData fetch(int row) const {
        const int rr = row < n ? row : n - 1;
        const int ii = rr % snx, jj = rr / snx, i = i0 + ii, j = j0 + jj;
        const int vf = j * (nx + 1) + i, hf = vcount + j * nx + i;
        return BlkRowData{T[vf], T[vf + 1], T[hf], T[hf + nx], y[rr]};  // W, E, S, N faces
    }
    __device__ __forceinline__ void decode(int row, const BlkRowData& e, double& d, double& w, double& w1,
                                           double& s) const {
        const int rr = row < n ? row : n - 1;
        const int ii = rr % snx, jj = rr / snx;
        double diag = 0.0;
        if (ii > 0) diag += e.a0;
        if (ii < snx - 1) diag += e.a1;
        if (jj > 0) diag += e.a2;
        if (jj < sny - 1) diag += e.a3;
        d = rr == 0 ? 1.0 : diag;
        w = (ii > 0 && rr != 1) ? e.a0 : 0.0;
        w1 = (ii + 1 < snx && rr != 0) ? e.a1 : 0.0;  // the next row's west coupling is this cell's east face
        s = (jj > 0 && rr != snx) ? e.a2 : 0.0;
    }
};

// Factorisation with the forward substitution of one right-hand side fused
// in. y (length n): rhs in, untouched. Xs: n*B doubles, Ts: n doubles
// (per-panel X fragments and t1 = G y1). sm: blk_smem_doubles<B>() doubles of
// this warp's shared memory. Returns false if a pivot block is not SPD.
template <int B, class Src>
__device__ bool blk_factor_fwd(int n, const Src& src, double* Xs, double* Ts, double* sm) {
    constexpr int NT = blk_nt<B>();
    static_assert(B % 8 == 0 && NT >= 2, "blocked band solver: B must be a multiple of 8, >= 16");
    const int lane = threadIdx.x & 31;
    const int r = lane >> 2, q = lane & 3, c0 = 2 * q, c1 = c0 + 1;
    double* sg0 = sm;             // Gauss-Jordan ping-pong buffers (8 x 8, row-major)
    double* sg1 = sm + 64;
    double* sS = sm + 128;        // S21 tiles 1..NT (index I-1)
    double* sX = sS + NT * 64;    // X tiles 1..NT-1 (index I-1)
    double* sy = sX + NT * 64;    // y1
    BlkTile w[NT + 1][NT + 1];    // lower triangle used (J <= I)
    double yw[NT + 1];            // y of window rows 8I + r (column 0 of a DMMA accumulator: lanes q == 0)
#pragma unroll
    for (int I = 0; I <= NT; ++I)
#pragma unroll
        for (int J = 0; J <= NT; ++J) w[I][J].v[0] = w[I][J].v[1] = 0.0;
    // row tile I of the window receives the entries of rows `row0 + r`:
    // tridiagonal diagonal tile, west coupling (0,7) into tile I-1, south
    // couplings into tile I-NT (rows >= n are identity rows)
    auto place = [&](int I, int row0, const BlkRowData& e) {
        const int row = row0 + r;
        const bool in = row < n;
        double ed, ew, ew1, es;
        src.decode(row, e, ed, ew, ew1, es);
        const double d = in ? ed : 1.0, wv = in ? -ew : 0.0, sv = in ? -es : 0.0;
        const double w1 = (row + 1 < n && r < 7) ? -ew1 : 0.0;
        w[I][I].v[0] = c0 == r ? d : (c0 == r - 1 ? wv : (c0 == r + 1 ? w1 : 0.0));
        w[I][I].v[1] = c1 == r ? d : (c1 == r - 1 ? wv : (c1 == r + 1 ? w1 : 0.0));
        yw[I] = in ? e.b : 0.0;
        if (I >= 1) w[I][I - 1].v[1] = (r == 0 && q == 3) ? wv : 0.0;
        if (I == NT) {
            w[I][0].v[0] = c0 == r ? sv : 0.0;
            w[I][0].v[1] = c1 == r ? sv : 0.0;
        }
    };
    // initial window: row tiles 0..NT
#pragma unroll
    for (int I = 0; I <= NT; ++I) place(I, 8 * I, src.fetch(8 * I + r));
    const int np = n / 8;
    // rows entering at the end of panels 0 and 1; each panel refetches its slot
    // for two panels ahead. The loop is unrolled by two so the in-flight loads
    // are never moved between registers (a move waits for the load)
    BlkRowData e0 = src.fetch(8 * (NT + 1) + r);
    BlkRowData e1 = src.fetch(8 * (NT + 2) + r);
    bool ok = true;
    auto panel = [&](const int p, BlkRowData& ent) {
        const int k0 = 8 * p;
        // ---- G = S11^-1 by Gauss-Jordan (SPD: no pivoting); each lane owns
        // entries (r, c0), (r, c1) and publishes them every step
        double g0 = w[0][0].v[0], g1 = w[0][0].v[1];
        *reinterpret_cast<double2*>(sg0 + r * 8 + c0) = make_double2(g0, g1);
        // the S21 tiles go to shared memory at the same time (read back in
        // the DMMA operand layout below)
#pragma unroll
        for (int I = 1; I <= NT; ++I)
            *reinterpret_cast<double2*>(sS + (I - 1) * 64 + r * 8 + c0) = make_double2(w[I][0].v[0], w[I][0].v[1]);
        if (q == 0) sy[r] = yw[0];
        __syncwarp();
        // four steps with 2 x 2 pivot blocks K = {2m, 2m+1} (half the
        // dependent chain of scalar pivots); a lane's column pair is a block
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const double* src = (m & 1) ? sg1 : sg0;
            double* dst = (m & 1) ? sg0 : sg1;
            const double2 k0r = *reinterpret_cast<const double2*>(src + (2 * m) * 8 + 2 * m);      // a, b
            const double2 k1r = *reinterpret_cast<const double2*>(src + (2 * m + 1) * 8 + 2 * m);  // b', d
            const double2 arK = *reinterpret_cast<const double2*>(src + r * 8 + 2 * m);            // A[r][K]
            const double2 aK0 = *reinterpret_cast<const double2*>(src + (2 * m) * 8 + c0);         // A[2m][c]
            const double2 aK1 = *reinterpret_cast<const double2*>(src + (2 * m + 1) * 8 + c0);     // A[2m+1][c]
            const double det = fma(k0r.x, k1r.y, -(k0r.y * k1r.x));
            ok = ok && (k0r.x > 0.0) && (det > 0.0);
            const double id = fast_rcp(det);
            const double p00 = k1r.y * id, p01 = -k0r.y * id, p10 = -k1r.x * id, p11 = k0r.x * id;  // P^-1
            const double u0 = fma(arK.x, p00, arK.y * p10), u1 = fma(arK.x, p01, arK.y * p11);  // A[r][K] P^-1
            double n0 = fma(-u0, aK0.x, fma(-u1, aK1.x, g0));
            double n1 = fma(-u0, aK0.y, fma(-u1, aK1.y, g1));
            if ((r >> 1) == m) {  // pivot rows: P^-1 A[K][c]
                const double pr0 = (r & 1) ? p10 : p00, pr1 = (r & 1) ? p11 : p01;
                n0 = fma(pr0, aK0.x, pr1 * aK1.x);
                n1 = fma(pr0, aK0.y, pr1 * aK1.y);
                if (q == m) {
                    n0 = pr0;
                    n1 = pr1;
                }
            } else if (q == m) {  // pivot columns: -A[r][K] P^-1
                n0 = -u0;
                n1 = -u1;
            }
            g0 = n0;
            g1 = n1;
            *reinterpret_cast<double2*>(dst + r * 8 + c0) = make_double2(g0, g1);
            __syncwarp();
        }
        const double* sg = sg0;  // 4 steps: the inverse is in buffer 0
        // ---- operands in DMMA layout
        const double gb0 = sg[q * 8 + r], gb1 = sg[(q + 4) * 8 + r];  // B = G: lane holds G[q][r], G[q+4][r]
        double sa[NT][2];                                                // A layout of S21 tiles 1..NT-1
#pragma unroll
        for (int I = 1; I < NT; ++I) {
            sa[I - 1][0] = sS[(I - 1) * 64 + r * 8 + q];
            sa[I - 1][1] = sS[(I - 1) * 64 + r * 8 + q + 4];
        }
        const double* sN = sS + (NT - 1) * 64;  // S21 tile NT (diagonal: south couplings)
        const double s_r = sN[r * 8 + r], s_c0 = sN[c0 * 8 + c0], s_c1 = sN[c1 * 8 + c1];
        // ---- X = S21 G
        BlkTile x[NT + 1];
#pragma unroll
        for (int I = 1; I < NT; ++I) {
            x[I].v[0] = x[I].v[1] = 0.0;
            blk_dmma(x[I].v[0], x[I].v[1], sa[I - 1][0], gb0);
            blk_dmma(x[I].v[0], x[I].v[1], sa[I - 1][1], gb1);
        }
        x[NT].v[0] = s_r * g0;
        x[NT].v[1] = s_r * g1;
        // stored for the backward sweep: tiles 1..NT, fragment order (coalesced)
        double* xs = Xs + (size_t)p * NT * 64;
#pragma unroll
        for (int I = 1; I <= NT; ++I)
            *reinterpret_cast<double2*>(xs + (I - 1) * 64 + 2 * lane) = make_double2(x[I].v[0], x[I].v[1]);
        // ---- trailing update S22 -= X S21^T
#pragma unroll
        for (int I = 1; I < NT; ++I)
            *reinterpret_cast<double2*>(sX + (I - 1) * 64 + r * 8 + c0) = make_double2(x[I].v[0], x[I].v[1]);
        __syncwarp();
        // forward substitution on the tensor cores too: y1 is the B operand
        // column 0 (lane (0, q) holds y1[q], y1[q+4]), so X_I Y1 and t1 = G y1
        // land in column 0 of the accumulators, lanes q == 0 (no shuffles)
        const double yb0 = r == 0 ? sy[q] : 0.0, yb1 = r == 0 ? sy[q + 4] : 0.0;
        {
            double t1 = 0.0, z1 = 0.0;
            blk_dmma(t1, z1, sg[r * 8 + q], yb0);
            blk_dmma(t1, z1, sg[r * 8 + q + 4], yb1);
            st_global_if(Ts + k0 + r, t1, q == 0);
            yw[NT] -= s_r * t1;  // X_NT y1 = diag(s) G y1
        }
#pragma unroll
        for (int I = 1; I < NT; ++I) {
            const double xa0 = -sX[(I - 1) * 64 + r * 8 + q], xa1 = -sX[(I - 1) * 64 + r * 8 + q + 4];
            double z1 = 0.0;
            blk_dmma(yw[I], z1, xa0, yb0);
            blk_dmma(yw[I], z1, xa1, yb1);
#pragma unroll
            for (int J = 1; J <= I; ++J) {
                blk_dmma(w[I][J].v[0], w[I][J].v[1], xa0, sa[J - 1][0]);
                blk_dmma(w[I][J].v[0], w[I][J].v[1], xa1, sa[J - 1][1]);
            }
        }
        // row tile NT: S21_NT = diag(s), so X_NT = diag(s) G
#pragma unroll
        for (int J = 1; J < NT; ++J) {  // -= diag(s) X_J^T
            w[NT][J].v[0] -= s_r * sX[(J - 1) * 64 + c0 * 8 + r];
            w[NT][J].v[1] -= s_r * sX[(J - 1) * 64 + c1 * 8 + r];
        }
        w[NT][NT].v[0] -= s_r * g0 * s_c0;
        w[NT][NT].v[1] -= s_r * g1 * s_c1;
        // ---- shift the window by one row tile; row tile NT enters
#pragma unroll
        for (int I = 0; I < NT; ++I)
#pragma unroll
            for (int J = 0; J <= I; ++J) w[I][J] = w[I + 1][J + 1];
#pragma unroll
        for (int I = 0; I < NT; ++I) yw[I] = yw[I + 1];
#pragma unroll
        for (int J = 0; J < NT; ++J) w[NT][J].v[0] = w[NT][J].v[1] = 0.0;
        place(NT, k0 + 8 * (NT + 1), ent);
        ent = src.fetch(k0 + 8 * (NT + 3) + r);
        __syncwarp();  // shared buffers are rewritten by the next panel
    };
    for (int p = 0; p < np; p += 2) {  // np = B^2/8 is even
        panel(p, e0);
        panel(p + 1, e1);
    }
    return __all_sync(0xffffffffu, ok);
}

// Backward sweep x1 = t1 - X^T x2 from the stored panels; x (length n) out.
// Returns this lane's partial sum of x (lanes 0..3 hold all of it).
template <int B>
__device__ double blk_backward(int n, const double* Xs, const double* Ts, double* x) {
    constexpr int NT = blk_nt<B>();
    const int lane = threadIdx.x & 31;
    const int r = lane >> 2, q = lane & 3, c0 = 2 * q;
    const int np = n / 8;
    double xw[NT];  // x of rows k0+8+8i+r (i = 0..NT-1): the rows after the panel
#pragma unroll
    for (int i = 0; i < NT; ++i) xw[i] = 0.0;
    double sum = 0.0;
    auto fetch = [&](int p, double2* xt, double2& tt) {
        const int pp = p < 0 ? 0 : p;
        const double* xs = Xs + (size_t)pp * NT * 64;
#pragma unroll
        for (int I = 0; I < NT; ++I) xt[I] = *reinterpret_cast<const double2*>(xs + I * 64 + 2 * lane);
        tt = *reinterpret_cast<const double2*>(Ts + 8 * pp + c0);
    };
    // four-panel-deep register ring of the stored panels (an HBM round trip
    // is several panels long); unrolled by four so slots are never moved
    constexpr int DEPTH = 4;
    double2 ring[DEPTH][NT], tr[DEPTH];
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) fetch(np - 1 - d, ring[d], tr[d]);
    auto step = [&](const int p, double2* xt, double2& tt) {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int I = 0; I < NT; ++I) {
            a0 = fma(xt[I].x, xw[I], a0);
            a1 = fma(xt[I].y, xw[I], a1);
        }
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
            a0 += __shfl_xor_sync(0xffffffffu, a0, o);
            a1 += __shfl_xor_sync(0xffffffffu, a1, o);
        }
        const double x0 = tt.x - a0, x1 = tt.y - a1;
        if (r == 0) {
            *reinterpret_cast<double2*>(x + 8 * p + c0) = make_double2(x0, x1);
            sum += x0 + x1;
        }
        const double v0 = __shfl_sync(0xffffffffu, x0, r >> 1), v1 = __shfl_sync(0xffffffffu, x1, r >> 1);
#pragma unroll
        for (int i = NT - 1; i > 0; --i) xw[i] = xw[i - 1];
        xw[0] = (r & 1) ? v1 : v0;
        fetch(p - DEPTH, xt, tt);
    };
    for (int p = np - 1; p >= 0; p -= DEPTH) {  // np = B^2/8 is a multiple of 8
#pragma unroll
        for (int d = 0; d < DEPTH; ++d) step(p - d, ring[d], tr[d]);
    }
    return sum;
}

}  // namespace mpm2p
