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
//    (quad dot products); backward x1 = t1 - X^T x2. Only X (B x 8 per panel,
//    the accumulator fragments as they are) and t1 are stored: n*B + n doubles
//    per subdomain, the same footprint as the scalar factor's L.
//  * No operand ever changes layout: the k index of an m8n8k4 product is a
//    dummy, so labelling slab s of lane (r, q) as k = 2q + s makes an
//    accumulator fragment (lane: [r][2q], [r][2q+1]) usable as it is both as
//    the A operand (rows r) and, for a product with the tile's transpose, as
//    the B operand (B[k][n = r] = tile[r][k]). X = S21 G takes S21's fragment
//    as A and G's as B (G is symmetric), S22 -= X S21^T takes X's and S21's.
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
// per-warp shared memory (doubles): two Gauss-Jordan buffers, 8 right-hand-
// side values, 8 south couplings, NT-1 tiles of X^T
template <int B>
__host__ __device__ constexpr int blk_smem_doubles() {
    return 2 * 64 + 16 + (blk_nt<B>() - 1) * 64;
}
// an 8x8 tile in shared memory, row-major, columns XORed with 6 on rows 2, 3,
// 6, 7 (the accumulator pairs (r, 2q..2q+1) stay contiguous)
__device__ __forceinline__ int blk_sw(int row, int col) {
    return row * 8 + (col ^ (((row >> 1) & 1) * 6));
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
// order, mrcm.cpp:391-411): no band rows are written or read back. SNX (the
// subdomain width, = the bandwidth) is a compile-time constant: the row's
// local cell coordinates cost a shift or a multiply, not a division.
template <int SNX>
struct BlkTransSrc {
    const double* T;
    const double* y;
    int n, sny, nx, vcount, i0, j0;
    __device__ __forceinline__ BlkRowData fetch(int row) const {
        const int rr = row < n ? row : n - 1;
        const int jj = rr / SNX, ii = rr - jj * SNX, i = i0 + ii, j = j0 + jj;
        const int vf = j * (nx + 1) + i, hf = vcount + j * nx + i;
        return BlkRowData{T[vf], T[vf + 1], T[hf], T[hf + nx], y ? y[rr] : 0.0};  // W, E, S, N faces
    }
    __device__ __forceinline__ void decode(int row, const BlkRowData& e, double& d, double& w, double& w1,
                                           double& s) const {
        const int rr = row < n ? row : n - 1;
        const int jj = rr / SNX, ii = rr - jj * SNX;
        double diag = 0.0;
        if (ii > 0) diag += e.a0;
        if (ii < SNX - 1) diag += e.a1;
        if (jj > 0) diag += e.a2;
        if (jj < sny - 1) diag += e.a3;
        d = rr == 0 ? 1.0 : diag;
        w = (ii > 0 && rr != 1) ? e.a0 : 0.0;
        w1 = (ii + 1 < SNX && rr != 0) ? e.a1 : 0.0;  // the next row's west coupling is this cell's east face
        s = (jj > 0 && rr != SNX) ? e.a2 : 0.0;
    }
};

// Factorisation with the forward substitution of one right-hand side fused
// in. y (length n): rhs in, untouched. Xs: n*B doubles, Ts: n doubles
// (per-panel X tiles and t1 = G y1). sm: blk_smem_doubles<B>() doubles of
// this warp's shared memory. Returns false if a pivot block is not SPD.
//
// The kernel is bound by the shared-memory data pipe and by issue slots, not
// by the DMMA pipe (profiles/blk_factor_r02_analysis.txt), so everything but
// the pivot block's Gauss-Jordan stays in registers:
//  * X_I = S21_I G and S22[I][J] -= X_I S21_J^T take their operands straight
//    from the accumulator fragments (see the header);
//  * row tile NT (S21_NT = diag(s), so X_NT = diag(s) G is a row scaling of
//    G's fragment) is updated by row scalings of X^T, read back transposed
//    from shared memory (NTD = false), or by the same DMMA products with X_NT
//    as A (NTD = true: 2(NT-1) more DMMA per panel, no shared memory; measured
//    2 % slower at B = 32, 1810 against 1774 us for 16,384 subdomains);
//  * the right-hand-side products (t1 = G y1, X_I y1) are quad dot products
//    (two FMAs and a two-step butterfly).
//
// RHS = false factors alone (no right-hand side: src's y may be null) and
// also stores every panel's G (64 doubles, fragment order) in Gs, for a
// forward sweep run later by blk_forward — the factor can then run
// concurrently with the chain that produces the right-hand side.
template <int B, class Src, bool NTD = false, bool RHS = true>
__device__ bool blk_factor_fwd(int n, const Src& src, double* Xs, double* Ts, double* sm, double* Gs = nullptr) {
    constexpr int NT = blk_nt<B>();
    static_assert(B % 8 == 0 && NT >= 2, "blocked band solver: B must be a multiple of 8, >= 16");
    const int lane = threadIdx.x & 31;
    const int r = lane >> 2, q = lane & 3, c0 = 2 * q, c1 = c0 + 1;
    double* sg0 = sm;        // Gauss-Jordan ping-pong buffers (swizzled 8 x 8)
    double* sg1 = sm + 64;
    double* sy = sm + 128;   // y1
    double* ss = sy + 8;     // s of row tile NT
    double* sT = ss + 8;     // (NTD = false) X^T tiles 1..NT-1
    BlkTile w[NT + 1][NT + 1];               // lower triangle used (J <= I), w[NT][0] unused
    double yw[NT + 1];   // y of window rows 8I + r (every lane of the row)
    double s_row = 0.0;  // south coupling of row tile NT's row r into pivot row r
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
        const double d = in ? ed : 1.0, wv = in ? -ew : 0.0;
        const double w1 = (row + 1 < n && r < 7) ? -ew1 : 0.0;
        w[I][I].v[0] = c0 == r ? d : (c0 == r - 1 ? wv : (c0 == r + 1 ? w1 : 0.0));
        w[I][I].v[1] = c1 == r ? d : (c1 == r - 1 ? wv : (c1 == r + 1 ? w1 : 0.0));
        yw[I] = in ? e.b : 0.0;
        if (I >= 1) w[I][I - 1].v[1] = (r == 0 && q == 3) ? wv : 0.0;
        if (I == NT) s_row = in ? -es : 0.0;
    };
    // positive and finite, on the high word's bits (keeps the check off the
    // fp64 pipe; a value whose high word is 0 — zero or a denormal below
    // 2^-1042 — counts as not positive)
    auto spd = [](double v) { return (unsigned)(__double2hiint(v) - 1) < 0x7fefffffu; };
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
        // entries (r, c0), (r, c0+1) and publishes them every step but the last
        double g0 = w[0][0].v[0], g1 = w[0][0].v[1];
        *reinterpret_cast<double2*>(sg0 + blk_sw(r, c0)) = make_double2(g0, g1);
        if (q == 0) {
            if (RHS) sy[r] = yw[0];
            ss[r] = s_row;
        }
        __syncwarp();
        // four steps with 2 x 2 pivot blocks K = {2m, 2m+1} (half the
        // dependent chain of scalar pivots); a lane's column pair is a block.
        // Branch-free: pivot rows take P^-1 A[K][c], pivot columns the
        // multipliers, the rest A[r][c] - A[r][K] P^-1 A[K][c]
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const double* src = (m & 1) ? sg1 : sg0;
            double* dst = (m & 1) ? sg0 : sg1;
            const double2 k0r = *reinterpret_cast<const double2*>(src + blk_sw(2 * m, 2 * m));      // a, b
            const double2 k1r = *reinterpret_cast<const double2*>(src + blk_sw(2 * m + 1, 2 * m));  // b', d
            const double2 arK = *reinterpret_cast<const double2*>(src + blk_sw(r, 2 * m));          // A[r][K]
            const double2 aK0 = *reinterpret_cast<const double2*>(src + blk_sw(2 * m, c0));         // A[2m][c]
            const double2 aK1 = *reinterpret_cast<const double2*>(src + blk_sw(2 * m + 1, c0));     // A[2m+1][c]
            const double det = fma(k0r.x, k1r.y, -(k0r.y * k1r.x));
            ok = ok & spd(k0r.x) & spd(det);
            const double id = fast_rcp(det);
            const double p00 = k1r.y * id, p01 = -k0r.y * id, p10 = -k1r.x * id, p11 = k0r.x * id;  // P^-1
            const double u0 = fma(arK.x, p00, arK.y * p10), u1 = fma(arK.x, p01, arK.y * p11);  // A[r][K] P^-1
            const bool prow = (r >> 1) == m;
            const double al0 = prow ? ((r & 1) ? p10 : p00) : -u0;
            const double al1 = prow ? ((r & 1) ? p11 : p01) : -u1;
            const double h0 = prow ? 0.0 : g0, h1 = prow ? 0.0 : g1;
            g0 = fma(al0, aK0.x, fma(al1, aK1.x, h0));
            g1 = fma(al0, aK0.y, fma(al1, aK1.y, h1));
            if (q == m) {
                g0 = al0;
                g1 = al1;
            }
            if (m < 3) {
                *reinterpret_cast<double2*>(dst + blk_sw(r, c0)) = make_double2(g0, g1);
                __syncwarp();
            }
        }
        // G[r][c0], G[r][c1] are in g0, g1: G's accumulator fragment
        const double2 yq = RHS ? *reinterpret_cast<const double2*>(sy + c0) : make_double2(0.0, 0.0);  // y1 of rows c0, c0+1
        if (!RHS) *reinterpret_cast<double2*>(Gs + (size_t)p * 64 + 2 * lane) = make_double2(g0, g1);
        const double2 sc = *reinterpret_cast<const double2*>(ss + c0);  // s of rows c0, c0+1
        // ---- X = S21 G (lane: X[r][c0], X[r][c1]); X_NT = diag(s) G
        BlkTile x[NT + 1];
#pragma unroll
        for (int I = 1; I < NT; ++I) {
            x[I].v[0] = x[I].v[1] = 0.0;
            blk_dmma(x[I].v[0], x[I].v[1], w[I][0].v[0], g0);
            blk_dmma(x[I].v[0], x[I].v[1], w[I][0].v[1], g1);
        }
        x[NT].v[0] = s_row * g0;
        x[NT].v[1] = s_row * g1;
        // stored for the backward sweep: tiles 1..NT, row-major (coalesced)
        double* xs = Xs + (size_t)p * NT * 64;
#pragma unroll
        for (int I = 1; I <= NT; ++I)
            *reinterpret_cast<double2*>(xs + (I - 1) * 64 + 2 * lane) = make_double2(x[I].v[0], x[I].v[1]);
        // ---- forward substitution: t1 = G y1 and y_I -= X_I y1 as quad dot
        // products (lane: columns c0 and c1)
        if (RHS) {
            double t1 = fma(g0, yq.x, g1 * yq.y);
            double py[NT];
#pragma unroll
            for (int I = 1; I < NT; ++I) py[I] = fma(x[I].v[0], yq.x, x[I].v[1] * yq.y);
#pragma unroll
            for (int o = 1; o < 4; o <<= 1) {
                t1 += __shfl_xor_sync(0xffffffffu, t1, o);
#pragma unroll
                for (int I = 1; I < NT; ++I) py[I] += __shfl_xor_sync(0xffffffffu, py[I], o);
            }
            st_global_if(Ts + k0 + r, t1, q == 0);
            yw[NT] -= s_row * t1;  // X_NT y1 = diag(s) G y1
#pragma unroll
            for (int I = 1; I < NT; ++I) yw[I] -= py[I];
        }
        // ---- trailing update S22[I][J] -= X_I S21_J^T on DMMA (row tiles
        // 1..NT, column tiles 1..min(I, NT-1): S21_NT only meets itself)
#pragma unroll
        for (int I = 1; I <= NT; ++I) {
            const double xa0 = -x[I].v[0], xa1 = -x[I].v[1];
#pragma unroll
            for (int J = 1; J <= I && J < NT; ++J) {
                if (!NTD && I == NT) continue;
                blk_dmma(w[I][J].v[0], w[I][J].v[1], xa0, w[J][0].v[0]);
                blk_dmma(w[I][J].v[0], w[I][J].v[1], xa1, w[J][0].v[1]);
            }
        }
        if (!NTD) {
#pragma unroll
            for (int J = 1; J < NT; ++J) {
                sT[(J - 1) * 64 + blk_sw(c0, r)] = x[J].v[0];
                sT[(J - 1) * 64 + blk_sw(c1, r)] = x[J].v[1];
            }
            __syncwarp();
#pragma unroll
            for (int J = 1; J < NT; ++J) {
                const double2 xt = *reinterpret_cast<const double2*>(sT + (J - 1) * 64 + blk_sw(r, c0));
                w[NT][J].v[0] = fma(-s_row, xt.x, w[NT][J].v[0]);
                w[NT][J].v[1] = fma(-s_row, xt.y, w[NT][J].v[1]);
            }
        }
        // S22[NT][NT] -= diag(s) G diag(s)
        w[NT][NT].v[0] = fma(-x[NT].v[0], sc.x, w[NT][NT].v[0]);
        w[NT][NT].v[1] = fma(-x[NT].v[1], sc.y, w[NT][NT].v[1]);
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

// Forward sweep from the stored panels and pivot inverses (blk_factor_fwd with
// RHS = false): t1 = G y1 into Ts, y_I -= X_I y1 on the window of the next B
// rows, the products as in the fused sweep (quad dot products; row tile NT
// uses its stored X_NT = diag(s) G). y (length n): rhs in, untouched.
template <int B>
__device__ void blk_forward(int n, const double* Xs, const double* Gs, const double* y, double* Ts) {
    constexpr int NT = blk_nt<B>();
    const int lane = threadIdx.x & 31;
    const int r = lane >> 2, q = lane & 3, c0 = 2 * q;
    const int np = n / 8;
    double yw[NT + 1];  // y of window rows 8I + r (every lane of the row)
#pragma unroll
    for (int I = 0; I <= NT; ++I) yw[I] = 8 * I + r < n ? y[8 * I + r] : 0.0;
    auto fetch = [&](int p, double2* xt, double2& g, double& yn) {
        const int pp = p < np ? p : np - 1;
        const double* xs = Xs + (size_t)pp * NT * 64;
#pragma unroll
        for (int I = 0; I < NT; ++I) xt[I] = *reinterpret_cast<const double2*>(xs + I * 64 + 2 * lane);
        g = *reinterpret_cast<const double2*>(Gs + (size_t)pp * 64 + 2 * lane);
        const int row = 8 * (pp + NT + 1) + r;  // the row entering the window after panel pp
        yn = row < n ? y[row] : 0.0;
    };
    constexpr int DEPTH = 4;  // panels in flight (an HBM round trip is several panels long)
    double2 ring[DEPTH][NT], gr[DEPTH];
    double yr[DEPTH];
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) fetch(d, ring[d], gr[d], yr[d]);
    auto step = [&](const int p, double2* xt, double2& g, double& yn) {
        // y1 of rows c0, c0+1: row j of the pivot block is held by the lanes with r = j
        const double y0 = __shfl_sync(0xffffffffu, yw[0], 4 * c0), y1 = __shfl_sync(0xffffffffu, yw[0], 4 * c0 + 4);
        double t1 = fma(g.x, y0, g.y * y1);
        double py[NT];
#pragma unroll
        for (int I = 0; I < NT; ++I) py[I] = fma(xt[I].x, y0, xt[I].y * y1);
#pragma unroll
        for (int o = 1; o < 4; o <<= 1) {
            t1 += __shfl_xor_sync(0xffffffffu, t1, o);
#pragma unroll
            for (int I = 0; I < NT; ++I) py[I] += __shfl_xor_sync(0xffffffffu, py[I], o);
        }
        st_global_if(Ts + 8 * p + r, t1, q == 0);
#pragma unroll
        for (int I = 0; I < NT; ++I) yw[I] = yw[I + 1] - py[I];  // stored tile I is row tile I + 1; then the window shifts
        yw[NT] = yn;
        fetch(p + DEPTH, xt, g, yn);
    };
    for (int p = 0; p < np; p += DEPTH) {  // np = B^2/8 is a multiple of 8
#pragma unroll
        for (int d = 0; d < DEPTH; ++d) step(p + d, ring[d], gr[d], yr[d]);
    }
}

// Backward sweep x1 = t1 - X^T x2 from the stored panels; x (length n) out.
// Lane (r, q) holds X[r][2q], X[r][2q+1] of each stored tile, so the column
// sums over r give x1[2q] and x1[2q+1]. Returns this lane's partial sum of x
// (lanes 0..3 hold all of it).
template <int B>
__device__ double blk_backward(int n, const double* Xs, const double* Ts, double* x) {
    constexpr int NT = blk_nt<B>();
    const int lane = threadIdx.x & 31;
    const int r = lane >> 2, q = lane & 3;
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
        tt = *reinterpret_cast<const double2*>(Ts + 8 * pp + 2 * q);
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
        const double x0 = tt.x - a0, x1 = tt.y - a1;  // x1[2q], x1[2q+1]
        if (r == 0) {
            *reinterpret_cast<double2*>(x + 8 * p + 2 * q) = make_double2(x0, x1);
            sum += x0 + x1;
        }
        // row r of the pivot block is column r: lanes with q = r/2 hold it
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
