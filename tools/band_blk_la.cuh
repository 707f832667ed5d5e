// band_blk_la.cuh — the blocked banded LDL^T of band_blk.cuh with the pivot
// block's inversion taken off the panel's critical path ("lookahead").
//
// Per 8-pivot panel the dependent chain of blk_factor_fwd is
//   G = S11^-1 (four 2x2 Gauss-Jordan steps through shared memory)
//   -> X = S21 G -> S22 -= X S21^T -> window shift -> next panel's G,
// and one warp issues it in order, so the trailing update, the stores, the
// forward substitution and the window shift all sit between two inversions.
// Only X_1 and the update of tile (1,1) feed the next pivot block. Here a
// panel forms X_1 and S22[1][1] first, publishes it, and runs the next
// panel's Gauss-Jordan steps interleaved with the rest of its own work
// (the other X tiles, the stores, the remaining DMMA updates, the forward
// substitution, row tile NT), which has no dependence on them: the chain per
// panel is LDS -> 4 DMMA -> STS -> Gauss-Jordan, everything else fills its
// latency. Every entry sees the same operations in the same order as in
// blk_factor_fwd (mrcm.cpp:388-427's Neumann solves), so factors, panels and
// solutions are bit-identical.
#pragma once

#include "../paper_2103_11050_b200/csrc/band_blk.cuh"

namespace mpm2p {

template <int B, class Src>
__device__ bool blk_factor_fwd_la(int n, const Src& src, double* Xs, double* Ts, double* sm) {
    constexpr int NT = blk_nt<B>();
    static_assert(B % 8 == 0 && NT >= 2, "blocked band solver: B must be a multiple of 8, >= 16");
    const int lane = threadIdx.x & 31;
    const int r = lane >> 2, q = lane & 3, c0 = 2 * q, c1 = c0 + 1;
    const int pr = (r >> 1) + 4 * (r & 1);  // pi(r)
    double* sg0 = sm;                        // Gauss-Jordan ping-pong buffers (swizzled 8 x 8)
    double* sg1 = sm + 64;
    double* sS = sm + 128;                   // S21 tiles 1..NT-1 (index I-1)
    double* sT = sS + (NT - 1) * 64;         // X^T tiles 1..NT-1
    double* sy = sT + (NT - 1) * 64;         // y1
    double* ss = sy + 8;                     // s of row tile NT
    BlkTile w[NT + 1][NT + 1];               // lower triangle used (J <= I)
    double yw[NT + 1];
    double s_row = 0.0;
#pragma unroll
    for (int I = 0; I <= NT; ++I)
#pragma unroll
        for (int J = 0; J <= NT; ++J) w[I][J].v[0] = w[I][J].v[1] = 0.0;
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
    auto spd = [](double v) {
        return (unsigned long long)(__double_as_longlong(v) - 1) < 0x7fefffffffffffffull;
    };
    bool ok = true;
    // one 2 x 2-pivot Gauss-Jordan step (band_blk.cuh), buffer m&1 -> the other
    auto gj_step = [&](const int m, double& g0, double& g1) {
        const double* from = (m & 1) ? sg1 : sg0;
        double* to = (m & 1) ? sg0 : sg1;
        const double2 k0r = *reinterpret_cast<const double2*>(from + blk_sw(2 * m, 2 * m));
        const double2 k1r = *reinterpret_cast<const double2*>(from + blk_sw(2 * m + 1, 2 * m));
        const double2 arK = *reinterpret_cast<const double2*>(from + blk_sw(r, 2 * m));
        const double2 aK0 = *reinterpret_cast<const double2*>(from + blk_sw(2 * m, c0));
        const double2 aK1 = *reinterpret_cast<const double2*>(from + blk_sw(2 * m + 1, c0));
        const double det = fma(k0r.x, k1r.y, -(k0r.y * k1r.x));
        ok = ok & spd(k0r.x) & spd(det);
        const double id = fast_rcp(det);
        const double p00 = k1r.y * id, p01 = -k0r.y * id, p10 = -k1r.x * id, p11 = k0r.x * id;
        const double u0 = fma(arK.x, p00, arK.y * p10), u1 = fma(arK.x, p01, arK.y * p11);
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
        *reinterpret_cast<double2*>(to + blk_sw(r, c0)) = make_double2(g0, g1);
        __syncwarp();
    };
    // the window's first block column goes to shared memory in the layouts
    // the next panel reads: S11 for the Gauss-Jordan, S21 tiles, y1, s
    auto publish_col = [&]() {
#pragma unroll
        for (int I = 1; I < NT; ++I)
            *reinterpret_cast<double2*>(sS + (I - 1) * 64 + blk_sw(r, c0)) = make_double2(w[I][0].v[0], w[I][0].v[1]);
        if (q == 0) {
            sy[r] = yw[0];
            ss[r] = s_row;
        }
    };
#pragma unroll
    for (int I = 0; I <= NT; ++I) place(I, 8 * I, src.fetch(8 * I + r));
    const int np = n / 8;
    BlkRowData e0 = src.fetch(8 * (NT + 1) + r);
    BlkRowData e1 = src.fetch(8 * (NT + 2) + r);
    // prologue: G of panel 0 (not overlapped)
    double g0 = w[0][0].v[0], g1 = w[0][0].v[1];
    *reinterpret_cast<double2*>(sg0 + blk_sw(r, c0)) = make_double2(g0, g1);
    publish_col();
    __syncwarp();
#pragma unroll
    for (int m = 0; m < 4; ++m) gj_step(m, g0, g1);

    auto panel = [&](const int p, BlkRowData& ent) {
        const int k0 = 8 * p;
        // ---- this panel's operands: G (in buffer 0) as A and, permuted, as
        // B; the S21 tiles as A; y1; s
        const double ga0 = sg0[blk_sw(r, q)], ga1 = sg0[blk_sw(r, q + 4)];
        const double gb0 = sg0[blk_sw(q, pr)], gb1 = sg0[blk_sw(q + 4, pr)];
        double sa[NT - 1][2];
#pragma unroll
        for (int I = 1; I < NT; ++I) {
            sa[I - 1][0] = sS[(I - 1) * 64 + blk_sw(r, q)];
            sa[I - 1][1] = sS[(I - 1) * 64 + blk_sw(r, q + 4)];
        }
        const double yq0 = sy[q], yq1 = sy[q + 4];
        const double2 sc = *reinterpret_cast<const double2*>(ss + c0);
        const double gc0 = g0, gc1 = g1;  // this lane's G entries (r, c0), (r, c1)
        __syncwarp();                     // all reads of buffer 0 done before it is refilled
        // ---- critical path: X_1, S22[1][1], the next pivot block
        BlkTile x[NT + 1];
        x[1].v[0] = x[1].v[1] = 0.0;
        blk_dmma(x[1].v[0], x[1].v[1], sa[0][0], gb0);
        blk_dmma(x[1].v[0], x[1].v[1], sa[0][1], gb1);
        blk_dmma(w[1][1].v[0], w[1][1].v[1], -x[1].v[0], sa[0][0]);
        blk_dmma(w[1][1].v[0], w[1][1].v[1], -x[1].v[1], sa[0][1]);
        g0 = w[1][1].v[0], g1 = w[1][1].v[1];
        *reinterpret_cast<double2*>(sg0 + blk_sw(r, c0)) = make_double2(g0, g1);
        __syncwarp();
        // ---- A: the other X tiles; the stored panel
#pragma unroll
        for (int I = 2; I < NT; ++I) {
            x[I].v[0] = x[I].v[1] = 0.0;
            blk_dmma(x[I].v[0], x[I].v[1], sa[I - 1][0], gb0);
            blk_dmma(x[I].v[0], x[I].v[1], sa[I - 1][1], gb1);
        }
        x[NT].v[0] = s_row * ga0;
        x[NT].v[1] = s_row * ga1;
        double* xs = Xs + (size_t)p * NT * 64;
#pragma unroll
        for (int I = 1; I <= NT; ++I)
            *reinterpret_cast<double2*>(xs + (I - 1) * 64 + 2 * lane) = make_double2(x[I].v[0], x[I].v[1]);
#pragma unroll
        for (int J = 1; J < NT; ++J) {
            sT[(J - 1) * 64 + blk_sw(q, r)] = x[J].v[0];
            sT[(J - 1) * 64 + blk_sw(q + 4, r)] = x[J].v[1];
        }
        gj_step(0, g0, g1);  // its barrier also publishes X^T
        // ---- B: trailing update of row tile 2; row tile NT from X^T
        if constexpr (NT > 2) {
            const double xa0 = -x[2].v[0], xa1 = -x[2].v[1];
#pragma unroll
            for (int J = 1; J <= 2; ++J) {
                blk_dmma(w[2][J].v[0], w[2][J].v[1], xa0, sa[J - 1][0]);
                blk_dmma(w[2][J].v[0], w[2][J].v[1], xa1, sa[J - 1][1]);
            }
        }
#pragma unroll
        for (int J = 1; J < NT; ++J) {
            const double2 xt = *reinterpret_cast<const double2*>(sT + (J - 1) * 64 + blk_sw(r, c0));
            w[NT][J].v[0] = fma(-s_row, xt.x, w[NT][J].v[0]);
            w[NT][J].v[1] = fma(-s_row, xt.y, w[NT][J].v[1]);
        }
        w[NT][NT].v[0] = fma(-(s_row * gc0), sc.x, w[NT][NT].v[0]);
        w[NT][NT].v[1] = fma(-(s_row * gc1), sc.y, w[NT][NT].v[1]);
        gj_step(1, g0, g1);
        // ---- C: trailing update of row tiles 3..NT-1
#pragma unroll
        for (int I = 3; I < NT; ++I) {
            const double xa0 = -x[I].v[0], xa1 = -x[I].v[1];
#pragma unroll
            for (int J = 1; J <= I; ++J) {
                blk_dmma(w[I][J].v[0], w[I][J].v[1], xa0, sa[J - 1][0]);
                blk_dmma(w[I][J].v[0], w[I][J].v[1], xa1, sa[J - 1][1]);
            }
        }
        gj_step(2, g0, g1);
        // ---- D: forward substitution: t1 = G y1, y_I -= X_I y1
        double t1 = fma(ga0, yq0, ga1 * yq1);
        double py[NT];
#pragma unroll
        for (int I = 1; I < NT; ++I) py[I] = fma(x[I].v[0], yq0, x[I].v[1] * yq1);
#pragma unroll
        for (int o = 1; o < 4; o <<= 1) {
            t1 += __shfl_xor_sync(0xffffffffu, t1, o);
#pragma unroll
            for (int I = 1; I < NT; ++I) py[I] += __shfl_xor_sync(0xffffffffu, py[I], o);
        }
        st_global_if(Ts + k0 + r, t1, q == 0);
        yw[NT] -= s_row * t1;
#pragma unroll
        for (int I = 1; I < NT; ++I) yw[I] -= py[I];
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
        publish_col();       // S21 tiles, y1, s of the next panel
        gj_step(3, g0, g1);  // the next panel's G is in buffer 0; its barrier publishes the column
    };
    for (int p = 0; p < np; p += 2) {  // np = B^2/8 is even
        panel(p, e0);
        panel(p + 1, e1);
    }
    return __all_sync(0xffffffffu, ok);
}

}  // namespace mpm2p
