// transport.cu — K1: explicit upwind saturation update, CFL reduction,
// conductivity, drift (epsilon) partial sums, injection rate / PVI clock and
// the outlet-saturation breakthrough probe (proj/src/transport.cpp:13-126,
// proj/src/mpm.cpp:9-29, proj/src/simulation.cpp:61-101,162-174,274-289).
//
// Compiled with --fmad=false: every per-cell expression keeps the
// reference's operation order and IEEE rounding, so saturation is
// bit-identical to the CPU path given the same velocity field (Appendix B
// items 6-7 of SURVEY.md). HBM-bound: one cell-update reads s (8 B) and two
// faces' u (16 B amortised) and writes s (8 B).
#include "context.cuh"

namespace mpm2p {

namespace {

constexpr int TPB = 256;

__device__ __forceinline__ double clamp_s(double s, long long* cnt) {  // transport.cpp:13-21
    if (s < 0.0 || s > 1.0) {
        if (cnt) atomicAdd((unsigned long long*)cnt, 1ull);
        return s < 0.0 ? 0.0 : 1.0;
    }
    return s;
}
__device__ __forceinline__ double frac_flow(double s, double M, long long* cnt) {  // transport.cpp:39-43
    s = clamp_s(s, cnt);
    const double w = M * s * s;
    // w == +0 (s == 0 ahead of the flood front, the bulk of C5's cells) gives
    // +0 / 1 == +0 exactly; returning it directly keeps every bit and skips the
    // IEEE division, whose zero-dividend operand takes its slow-path subroutine
    return w == 0.0 ? 0.0 : w / (w + (1.0 - s) * (1.0 - s));
}
__device__ __forceinline__ double total_mob(double s, double M, long long* cnt) {  // transport.cpp:34-37
    s = clamp_s(s, cnt);
    return M * s * s + (1.0 - s) * (1.0 - s);
}
__device__ __forceinline__ double fprime(double s, double M) {  // transport.cpp:23-27
    const double d = M * s * s + (1.0 - s) * (1.0 - s);
    const double dd = 2.0 * M * s - 2.0 * (1.0 - s);
    return (2.0 * M * s * d - M * s * s * dd) / (d * d);
}

// Block reduction helpers; the final combination over blocks is done by the
// last block to finish, in block order, so results are deterministic.
__device__ __forceinline__ bool last_block_done(unsigned* counter) {
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned t = atomicAdd(counter, 1u);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    return last;
}

template <typename F>
__device__ __forceinline__ double block_reduce(double v, F op, double* sh, double ident) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_down_sync(0xffffffffu, v, o));
    if (lane == 0) sh[w] = v;
    __syncthreads();
    if (w == 0) {
        v = lane < (int)(blockDim.x >> 5) ? sh[lane] : ident;
        for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_down_sync(0xffffffffu, v, o));
    }
    __syncthreads();
    return v;
}

__device__ __forceinline__ DD block_reduce_dd(DD v, DD* sh) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = warp_sum_dd(v);
    if (lane == 0) sh[w] = v;
    __syncthreads();
    if (w == 0) {
        v = lane < (int)(blockDim.x >> 5) ? sh[lane] : DD{0.0, 0.0};
        v = warp_sum_dd(v);
    }
    __syncthreads();
    return v;
}

// Two double-double sums reduced together (one barrier pair instead of two).
__device__ __forceinline__ void block_reduce_dd2(DD& a, DD& b, DD* sh /* 64 */) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    a = warp_sum_dd(a);
    b = warp_sum_dd(b);
    if (lane == 0) {
        sh[w] = a;
        sh[32 + w] = b;
    }
    __syncthreads();
    if (w == 0) {
        const bool in = lane < (int)(blockDim.x >> 5);
        a = warp_sum_dd(in ? sh[lane] : DD{0.0, 0.0});
        b = warp_sum_dd(in ? sh[32 + lane] : DD{0.0, 0.0});
    }
    __syncthreads();
}

// Parallel double-double combination of per-block partials (hi at off, lo at off+1).
__device__ __forceinline__ DD reduce_dd_partials(const double* part, int nparts, int off, DD* sh) {
    DD v{0.0, 0.0};
    for (int b = threadIdx.x; b < nparts; b += blockDim.x)
        v = dd_add(v, DD{__ldcg(part + 4 * b + off), __ldcg(part + 4 * b + off + 1)});
    __syncthreads();
    return block_reduce_dd(v, sh);
}

// max over the reference's 1001 sample points (transport.cpp:45-49); max is
// order-independent, so one thread per point gives the same value.
__global__ void k_max_slope(Scalars* sc, double M) {
    pdl_begin();
    __shared__ double sh[32];
    double m = 0.0;
    for (int k = threadIdx.x; k <= 1000; k += blockDim.x) m = fmax(m, fprime(k * 1e-3, M));
    m = block_reduce_op(m, [](double a, double b) { return fmax(a, b); }, 0.0, sh);
    if (threadIdx.x == 0) sc->slope = m;
}

// cfl_timestep (transport.cpp:51-71): min over cells of vol/(outflux*slope).
__device__ double inj_rate_block(const Layout& L, const double* __restrict__ u, double fin, double* sh);

// With inj_cn > 0 the last block also evaluates injection_rate and advances
// the PVI clock inj_cn times (the driver's k_cfl + k_inj_pvi in one launch).
__global__ void k_cfl(Layout L, const double* __restrict__ u, Scalars* sc, double safety, double dt_cap,
                      double* part, unsigned* counter, int inj_cn = 0, double inflow = 0.0, double M = 1.0) {
    pdl_begin();
    const double vol = L.vol(), slope = sc->slope;
    double best = INFINITY;
    double any = 0.0;
    double rate = 0.0;  // injection_rate terms (simulation.cpp:85-101) when inj_cn > 0
    const int nterms = inj_cn > 0 ? 2 * (L.nx + L.ny) : 0;
    const double fin = inj_cn > 0 ? frac_flow(inflow, M, nullptr) : 0.0;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < nterms; x += gridDim.x * blockDim.x) {
        double un, area;
        if (x < 2 * L.ny) {
            const int j = x >> 1;
            un = (x & 1) == 0 ? -u[L.vface(0, j)] : u[L.vface(L.nx, j)];
            area = L.hy;
        } else {
            const int k = x - 2 * L.ny, i = k >> 1;
            un = (k & 1) == 0 ? -u[L.hface(i, 0)] : u[L.hface(i, L.ny)];
            area = L.hx;
        }
        if (un < 0.0) rate += -un * area * fin;
    }
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < L.cells(); c += gridDim.x * blockDim.x) {
        const int i = c % L.nx, j = c / L.nx;
        double out = 0.0;
        const double uE = u[L.vface(i + 1, j)], uW = u[L.vface(i, j)];
        const double uN = u[L.hface(i, j + 1)], uS = u[L.hface(i, j)];
        out += (0.0 < uE ? uE : 0.0) * L.hy;
        out += (0.0 < -uW ? -uW : 0.0) * L.hy;
        out += (0.0 < uN ? uN : 0.0) * L.hx;
        out += (0.0 < -uS ? -uS : 0.0) * L.hx;
        if (out > 0.0) {
            any = 1.0;
            best = fmin(best, vol / (out * slope));
        }
    }
    // one multi-value reduction: -best (max), any (max), rate (sum)
    __shared__ double shm[32 * 3];
    __shared__ double red[3];
    double v[3] = {-best, any, rate};
    block_reduce_multi<3>(v, 0x4u, shm, red);
    if (threadIdx.x < 3) part[3 * blockIdx.x + threadIdx.x] = red[threadIdx.x];
    if (last_block_done(counter)) {
        double a[3] = {-INFINITY, 0.0, 0.0};
        for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
            a[0] = fmax(a[0], __ldcg(part + 3 * b));
            a[1] = fmax(a[1], __ldcg(part + 3 * b + 1));
            a[2] += __ldcg(part + 3 * b + 2);
        }
        block_reduce_multi<3>(a, 0x4u, shm, red);
        if (threadIdx.x == 0) {
            const double best_all = -red[0];
            const double dt = fmin(dt_cap / safety, best_all);  // min is order-independent
            const bool anyf = red[1] > 0.0;
            sc->any_flow = anyf;
            sc->dt = anyf ? fmin(safety * dt, dt_cap) : dt_cap;
            *counter = 0;
            if (inj_cn > 0) {
                const double rt = red[2];
                sc->inj = rt;
                const double pore = L.lx * L.ly;
                for (int k = 0; k < inj_cn; ++k) sc->pvi += rt * sc->dt / pore;
            }
        }
    }
}

// injection_rate (simulation.cpp:85-101) as a one-block tree sum (the terms
// are the reference's; only the summation order differs — the PVI clock is a
// reported quantity, not a parity one), then the PVI clock advanced cn times
// (simulation.cpp:288).
__device__ double inj_rate_block(const Layout& L, const double* __restrict__ u, double fin, double* sh) {
    const int nterms = 2 * (L.nx + L.ny);
    double rate = 0.0;
    for (int idx = threadIdx.x; idx < nterms; idx += blockDim.x) {
        double un, area;
        if (idx < 2 * L.ny) {
            const int j = idx >> 1;
            un = (idx & 1) == 0 ? -u[L.vface(0, j)] : u[L.vface(L.nx, j)];
            area = L.hy;
        } else {
            const int k = idx - 2 * L.ny, i = k >> 1;
            un = (k & 1) == 0 ? -u[L.hface(i, 0)] : u[L.hface(i, L.ny)];
            area = L.hx;
        }
        if (un < 0.0) rate += -un * area * fin;
    }
    return block_reduce_op(rate, [](double a, double b) { return a + b; }, 0.0, sh);
}

__global__ void k_inj_pvi(Layout L, const double* __restrict__ u, Scalars* sc, double inflow, double M, int cn,
                          int add_pvi) {
    pdl_begin();
    __shared__ double sh[32];
    const double rate = inj_rate_block(L, u, frac_flow(inflow, M, nullptr), sh);
    if (threadIdx.x == 0) {
        sc->inj = rate;
        if (add_pvi) {
            const double pore = L.lx * L.ly;
            for (int k = 0; k < cn; ++k) sc->pvi += rate * sc->dt / pore;
        }
    }
}

// upwind_step (transport.cpp:73-120), one thread per cell; both cells of a
// face compute its water flux with identical IEEE operations.
// take_next: the step's cfl_timestep / injection_rate were formed by the
// previous pressure update's k_ds_u_div (CflNext); this first sub-step reads
// dt_next and thread 0 promotes it (dt, any_flow, inj) and advances the PVI
// clock inj_cn times exactly as k_cfl's epilogue does.
// sub > 1: the track_errors sub-cycling of s_main, dt / sub per sub-step
// (simulation.cpp:270-276).
__global__ void k_upwind(Layout L, const double* __restrict__ s, double* __restrict__ s_out,
                         const double* __restrict__ u, Scalars* sc, double inflow, double M, int take_next = 0,
                         int inj_cn = 0, int sub = 1) {
    pdl_begin();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const double dt = take_next ? sc->dt_next : (sub > 1 ? sc->dt / sub : sc->dt);
    if (c == 0) {
        (void)frac_flow(inflow, M, &sc->clamp);  // f_in is evaluated once per call
        if (take_next) {
            sc->dt = dt;
            sc->any_flow = sc->any_next;
            const double rt = sc->inj_next;
            sc->inj = rt;
            const double pore = L.lx * L.ly;
            for (int k = 0; k < inj_cn; ++k) sc->pvi += rt * dt / pore;
        }
    }
    if (c >= L.cells()) return;
    const int i = c % L.nx, j = c / L.nx;
    const double fin = frac_flow(inflow, M, nullptr);
    long long* cnt = &sc->clamp;
    // every operand loaded up front, unconditionally (one memory round trip;
    // the upwind choice below only selects among registers)
    const double uW = u[L.vface(i, j)], uE = u[L.vface(i + 1, j)];
    const double uS = u[L.hface(i, j)], uN = u[L.hface(i, j + 1)];
    const double sC = s[c];
    const double sW = i > 0 ? s[c - 1] : 0.0, sE = i + 1 < L.nx ? s[c + 1] : 0.0;
    const double sS = j > 0 ? s[c - L.nx] : 0.0, sN = j + 1 < L.ny ? s[c + L.nx] : 0.0;
    // face water flux from the upwind side; vertical faces: owner counts clamps
    // (face i is owned by cell i, face nx by cell nx-1)
    auto flux = [&](double un, bool lo_bnd, double s_lo, bool hi_bnd, double s_hi, bool own, double area) {
        double fs;
        if (un >= 0.0) fs = lo_bnd ? fin : frac_flow(s_lo, M, own ? cnt : nullptr);
        else fs = hi_bnd ? fin : frac_flow(s_hi, M, own ? cnt : nullptr);
        return fs * un * area;
    };
    const double wE = flux(uE, false, sC, i + 1 == L.nx, sE, i + 1 == L.nx, L.hy);
    const double wW = flux(uW, i == 0, sW, false, sC, true, L.hy);
    const double wN = flux(uN, false, sC, j + 1 == L.ny, sN, j + 1 == L.ny, L.hx);
    const double wS = flux(uS, j == 0, sS, false, sC, true, L.hx);
    const double net = wE - wW + wN - wS;
    const double sn = sC - dt / L.vol() * net;
    if (sn < -1e-12 || sn > 1.0 + 1e-12) atomicOr(&sc->err, ERR_CFL);
    s_out[c] = sn < 0.0 ? 0.0 : (sn > 1.0 ? 1.0 : sn);
}

// Tiled upwind_step: a CTA owns a 32 x 8 tile of cells. Every cell's
// fractional flow f(s) is evaluated ONCE into shared memory (tile + one-cell
// halo: 340 evaluations for 256 cells, against 4 per cell when each cell
// evaluates both sides of its faces); a face then only selects the upwind
// cell's value. f is a pure function of s, so every face flux, and hence s,
// is bit-identical to k_upwind. Clamp counting follows k_upwind: a face's
// owner (west / south face of each cell, plus the east / north domain
// boundary) counts an out-of-range upwind saturation.
constexpr int UT_X = 32, UT_Y = 8;
__global__ void __launch_bounds__(UT_X * UT_Y) k_upwind_tile(Layout L, const double* __restrict__ s,
                                                             double* __restrict__ s_out, const double* __restrict__ u,
                                                             Scalars* sc, double inflow, double M, int take_next = 0,
                                                             int inj_cn = 0, int sub = 1) {
    pdl_begin();
    __shared__ double F[UT_Y + 2][UT_X + 2];
    __shared__ unsigned char OOR[UT_Y + 2][UT_X + 2];
    const int i0 = blockIdx.x * UT_X, j0 = blockIdx.y * UT_Y;
    const int ti = threadIdx.x % UT_X, tj = threadIdx.x / UT_X;
    const int i = i0 + ti, j = j0 + tj;
    const double dt = take_next ? sc->dt_next : (sub > 1 ? sc->dt / sub : sc->dt);
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
        (void)frac_flow(inflow, M, &sc->clamp);  // f_in is evaluated once per call
        if (take_next) {
            sc->dt = dt;
            sc->any_flow = sc->any_next;
            const double rt = sc->inj_next;
            sc->inj = rt;
            const double pore = L.lx * L.ly;
            for (int k = 0; k < inj_cn; ++k) sc->pvi += rt * dt / pore;
        }
    }
    const bool in = i < L.nx && j < L.ny;
    // the thread's own operands first (one round trip with the halo loads)
    double uW = 0.0, uE = 0.0, uS = 0.0, uN = 0.0, sC = 0.0;
    if (in) {
        uW = u[L.vface(i, j)];
        uE = u[L.vface(i + 1, j)];
        uS = u[L.hface(i, j)];
        uN = u[L.hface(i, j + 1)];
        sC = s[L.cell(i, j)];
    }
    constexpr int HN = (UT_X + 2) * (UT_Y + 2);
    for (int h = threadIdx.x; h < HN; h += UT_X * UT_Y) {
        const int hx = h % (UT_X + 2), hy = h / (UT_X + 2);
        const int gi = i0 + hx - 1, gj = j0 + hy - 1;
        double f = 0.0;
        unsigned char o = 0;
        if (gi >= 0 && gi < L.nx && gj >= 0 && gj < L.ny) {
            const double sv = s[L.cell(gi, gj)];
            o = (sv < 0.0 || sv > 1.0) ? 1 : 0;
            f = frac_flow(sv, M, nullptr);
        }
        F[hy][hx] = f;
        OOR[hy][hx] = o;
    }
    __shared__ double cst[2];  // f(inflow) and dt / vol: evaluated once per CTA (same IEEE operations)
    if (threadIdx.x == 0) {
        cst[0] = frac_flow(inflow, M, nullptr);
        cst[1] = dt / L.vol();
    }
    __syncthreads();
    if (!in) return;
    const double fin = cst[0];
    const double fC = F[tj + 1][ti + 1];
    const bool lastx = i + 1 == L.nx, lasty = j + 1 == L.ny;
    // face fluxes with k_upwind's operations: (f * u) * area
    const double fE = uE >= 0.0 ? fC : (lastx ? fin : F[tj + 1][ti + 2]);
    const double fWv = uW >= 0.0 ? (i == 0 ? fin : F[tj + 1][ti]) : fC;
    const double fN = uN >= 0.0 ? fC : (lasty ? fin : F[tj + 2][ti + 1]);
    const double fSv = uS >= 0.0 ? (j == 0 ? fin : F[tj][ti + 1]) : fC;
    const double wE = fE * uE * L.hy, wW = fWv * uW * L.hy;
    const double wN = fN * uN * L.hx, wS = fSv * uS * L.hx;
    {  // clamp counts of the owned faces' evaluations
        int cnt = 0;
        cnt += uW >= 0.0 ? (i > 0 && OOR[tj + 1][ti]) : OOR[tj + 1][ti + 1];
        cnt += uS >= 0.0 ? (j > 0 && OOR[tj][ti + 1]) : OOR[tj + 1][ti + 1];
        if (lastx && uE >= 0.0) cnt += OOR[tj + 1][ti + 1];
        if (lasty && uN >= 0.0) cnt += OOR[tj + 1][ti + 1];
        if (cnt) atomicAdd((unsigned long long*)&sc->clamp, (unsigned long long)cnt);
    }
    const double net = wE - wW + wN - wS;
    const double sn = sC - cst[1] * net;
    if (sn < -1e-12 || sn > 1.0 + 1e-12) atomicOr(&sc->err, ERR_CFL);
    s_out[L.cell(i, j)] = sn < 0.0 ? 0.0 : (sn > 1.0 ? 1.0 : sn);
}

// Column-marching upwind_step. A warp owns 30 columns (lanes 1..30; lanes 0
// and 31 are the west / east halo columns and only evaluate f) and marches
// `rows` rows northwards. The f of the rows below / at / above stays in
// registers and the west / east neighbours' f come by shuffle, so a cell costs
// one f evaluation (plus 1/rows for the segment's two halo rows and 2/30 for
// the halo lanes) and no shared-memory round trip or CTA barrier. k_upwind_tile
// spent ~370 issued instructions per cell (C2 ncu: issue-bound at C5). Each
// chunk of RB rows issues its loads one chunk ahead of its arithmetic. Face fluxes
// use k_upwind's operations in the same order, so s is bit-identical; clamp
// counts follow k_upwind_tile (the owner of a face counts an out-of-range
// upwind saturation).
constexpr int UC_COLS = 30;
__device__ __forceinline__ bool out_of_range(double v) { return v < 0.0 || v > 1.0; }
template <int RB, int MINB>
__global__ void __launch_bounds__(256, MINB) k_upwind_col(Layout L, const double* __restrict__ s, double* __restrict__ s_out,
                                                    const double* __restrict__ u, Scalars* sc, double inflow, double M,
                                                    int take_next, int inj_cn, int sub, int rows) {
    pdl_begin();
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int ncw = (L.nx + UC_COLS - 1) / UC_COLS;
    const int wc = gw % ncw, wr = gw / ncw;
    const int j0 = wr * rows;
    const double dt = take_next ? sc->dt_next : (sub > 1 ? sc->dt / sub : sc->dt);
    if (gw == 0 && lane == 0) {
        (void)frac_flow(inflow, M, &sc->clamp);  // f_in is evaluated once per call
        if (take_next) {
            sc->dt = dt;
            sc->any_flow = sc->any_next;
            const double rt = sc->inj_next;
            sc->inj = rt;
            const double pore = L.lx * L.ly;
            for (int k = 0; k < inj_cn; ++k) sc->pvi += rt * dt / pore;
        }
    }
    if (j0 >= L.ny) return;  // warp-uniform
    const int j1 = min(j0 + rows, L.ny);
    const int i = wc * UC_COLS + lane - 1;
    const bool col = i >= 0 && i < L.nx;
    const bool own = col && lane >= 1 && lane <= UC_COLS;
    const bool firstx = i == 0, lastx = i + 1 == L.nx;
    const double fin = frac_flow(inflow, M, nullptr);
    const double dtv = dt / L.vol();
    const double hx = L.hx, hy = L.hy;
    // the row below the segment and the segment's first row
    double fS = 0.0, fC = 0.0, uS = 0.0;
    bool oS = false, oC = false;
    const double sc0 = col ? s[L.cell(i, j0)] : 0.0;
    {
        const double sb = (col && j0 > 0) ? s[L.cell(i, j0 - 1)] : 0.0;
        if (own) uS = u[L.hface(i, j0)];
        if (col && j0 > 0) {
            oS = out_of_range(sb);
            fS = frac_flow(sb, M, nullptr);
        }
        if (col) {
            oC = out_of_range(sc0);
            fC = frac_flow(sc0, M, nullptr);
        }
    }
    double sCv = sc0;
    unsigned long long cnt = 0;
    bool err = false;
    unsigned obS = __ballot_sync(0xffffffffu, oS);
    // running row pointers (clamped column for the lanes that load nothing)
    const int ic = col ? i : 0;
    const double* ps = s + L.cell(ic, j0) + L.nx;   // s of row j + 1
    const double* pv = u + L.vface(ic, j0);          // vertical faces of row j
    const double* ph = u + L.hface(ic, j0) + L.nx;   // horizontal face north of row j
    double* po = s_out + L.cell(ic, j0);
    // software pipeline: chunk n + 1's loads are in flight while chunk n computes
    double sN[RB], uW[RB], uE[RB], uN[RB];
    auto load_chunk = [&](int jb, double* a, double* w, double* e, double* n) {
#pragma unroll
        for (int k = 0; k < RB; ++k) {
            const int j = jb + k;
            a[k] = (col && j < j1 && j + 1 < L.ny) ? ps[k * L.nx] : 0.0;
            const bool ld = own && j < j1;
            w[k] = ld ? pv[k * (L.nx + 1)] : 0.0;
            e[k] = ld ? pv[k * (L.nx + 1) + 1] : 0.0;
            n[k] = ld ? ph[k * L.nx] : 0.0;
        }
        ps += RB * L.nx;
        pv += RB * (L.nx + 1);
        ph += RB * L.nx;
    };
    load_chunk(j0, sN, uW, uE, uN);
    for (int jb = j0; jb < j1; jb += RB) {
        double sN2[RB], uW2[RB], uE2[RB], uN2[RB];
        load_chunk(jb + RB, sN2, uW2, uE2, uN2);
#pragma unroll
        for (int k = 0; k < RB; ++k) {
            // the tail rows of a segment (j >= j1) run predicated, so the
            // shuffles below stay outside any divergent region
            const int j = jb + k;
            const bool row = j < j1;
            // rows / lanes without a north cell loaded s = 0 (in range, f = 0),
            // and their f is never selected: no branch around the division
            const bool oN = out_of_range(sN[k]);
            const double fN = frac_flow(sN[k], M, nullptr);
            const double fWc = __shfl_up_sync(0xffffffffu, fC, 1);
            const double fEc = __shfl_down_sync(0xffffffffu, fC, 1);
            const unsigned ob = __ballot_sync(0xffffffffu, oC);
            if (own && row) {
                const bool lasty = j + 1 == L.ny;
                const double fE = uE[k] >= 0.0 ? fC : (lastx ? fin : fEc);
                const double fWv = uW[k] >= 0.0 ? (firstx ? fin : fWc) : fC;
                const double fNv = uN[k] >= 0.0 ? fC : (lasty ? fin : fN);
                const double fSv = uS >= 0.0 ? (j == 0 ? fin : fS) : fC;
                const double wE = fE * uE[k] * hy, wW = fWv * uW[k] * hy;
                const double wN = fNv * uN[k] * hx, wS = fSv * uS * hx;
                if (ob | obS) {  // warp-uniform: some saturation of this row or the one below is out of range
                    const bool oW = (ob >> (lane - 1)) & 1u;
                    cnt += uW[k] >= 0.0 ? (!firstx && oW) : oC;
                    cnt += uS >= 0.0 ? (j > 0 && oS) : oC;
                    cnt += (lastx && uE[k] >= 0.0) ? oC : 0;
                    cnt += (lasty && uN[k] >= 0.0) ? oC : 0;
                }
                const double net = wE - wW + wN - wS;
                const double sn = sCv - dtv * net;
                err |= sn < -1e-12 || sn > 1.0 + 1e-12;
                po[k * L.nx] = sn < 0.0 ? 0.0 : (sn > 1.0 ? 1.0 : sn);
            }
            fS = fC;
            oS = oC;
            obS = ob;
            fC = fN;
            oC = oN;
            sCv = sN[k];
            uS = uN[k];
        }
        po += RB * L.nx;
#pragma unroll
        for (int k = 0; k < RB; ++k) {
            sN[k] = sN2[k];
            uW[k] = uW2[k];
            uE[k] = uE2[k];
            uN[k] = uN2[k];
        }
    }
    if (cnt) atomicAdd((unsigned long long*)&sc->clamp, cnt);
    if (err) atomicOr(&sc->err, ERR_CFL);
}


int upwind_col_rows(const Layout& L, int nsm) {
    const long ncw = (L.nx + UC_COLS - 1) / UC_COLS;
    int rows = 32;
    while (rows > 4 && ncw * ((L.ny + rows - 1) / rows) < 48L * nsm) rows >>= 1;
    return rows;
}

// conductivity (transport.cpp:122-126) + the drift partial sums
// (mpm.cpp:14-20 / simulation.cpp:169-172) in double-double.
// eps_mode: -1 none, 0 relative, 1 absolute, 2 mobility (vs lam_reb)
__device__ __forceinline__ void decide(Scalars* sc, int rebuilt, int method, double eta, int step);

// Block partials of the drift sums, then (last block) the combination in
// block order, eps and the next-step decision.
__device__ __forceinline__ void kappa_eps_tail(DD num, DD den, Scalars* sc, double M, int eps_mode, double* part,
                                               unsigned* counter, int decide_method, int rebuilt, double eta) {
    __shared__ DD shd2[64];
    block_reduce_dd2(num, den, shd2);
    if (threadIdx.x == 0) {
        part[4 * blockIdx.x + 0] = num.hi;
        part[4 * blockIdx.x + 1] = num.lo;
        part[4 * blockIdx.x + 2] = den.hi;
        part[4 * blockIdx.x + 3] = den.lo;
    }
    if (last_block_done(counter)) {
        DD n{0.0, 0.0}, d{0.0, 0.0};
        for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
            n = dd_add(n, DD{__ldcg(part + 4 * b), __ldcg(part + 4 * b + 1)});
            d = dd_add(d, DD{__ldcg(part + 4 * b + 2), __ldcg(part + 4 * b + 3)});
        }
        block_reduce_dd2(n, d, shd2);
        if (threadIdx.x == 0) {
            const double a = sqrt(n.hi);
            double e;
            if (eps_mode == 1) e = a;
            else if (eps_mode == 2) e = a / M;
            else {
                if (!(d.hi > 0.0)) atomicOr(&sc->err, ERR_EPS_ZERO);
                e = a / sqrt(d.hi);
            }
            sc->eps_pending = e;
            sc->eps_num_hi = n.hi;
            sc->eps_num_lo = n.lo;
            sc->eps_den_hi = d.hi;
            sc->eps_den_lo = d.lo;
            *counter = 0;
            if (decide_method >= 0) decide(sc, rebuilt, decide_method, eta, 1);
        }
    }
}

// With decide_method >= 0 the last block also takes the next-step decision
// (k_decide) from the drift it just formed.
// With T != nullptr it also writes the face transmissibilities of k_trans for
// the faces each cell owns (west/south, plus the east/north domain boundary),
// recomputing the neighbour's conductivity with the same operations.
__global__ void k_kappa(Layout L, const double* __restrict__ K, const double* __restrict__ s,
                        double* __restrict__ kappa, const double* __restrict__ kappa_m,
                        const double* __restrict__ lam_reb, Scalars* sc, double M, int eps_mode, double* part,
                        unsigned* counter, int decide_method = -1, int rebuilt = 0, double eta = 0.0,
                        double* __restrict__ T = nullptr) {
    pdl_begin();
    const double vol = L.vol();
    DD num{0.0, 0.0}, den{0.0, 0.0};
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < L.cells(); c += gridDim.x * blockDim.x) {
        const double lam = total_mob(s[c], M, &sc->clamp);
        const double k = lam * K[c];
        kappa[c] = k;
        if (T) {  // elliptic.cpp:44-61 for this cell's faces (boundary faces carry 0)
            const int i = c % L.nx, j = c / L.nx;
            const int cw = L.cell(i - 1, j), cs = L.cell(i, j - 1);
            T[L.vface(i, j)] = i > 0 ? harm_trans_v(L, total_mob(s[cw], M, nullptr) * K[cw], k) : 0.0;
            T[L.hface(i, j)] = j > 0 ? harm_trans_h(L, total_mob(s[cs], M, nullptr) * K[cs], k) : 0.0;
            if (i == L.nx - 1) T[L.vface(L.nx, j)] = 0.0;
            if (j == L.ny - 1) T[L.hface(i, L.ny)] = 0.0;
        }
        if (!(k > 0.0) || !isfinite(k)) atomicOr(&sc->err, ERR_KAPPA);
        if (eps_mode == 0 || eps_mode == 1) {
            const double d = k - kappa_m[c];
            num = dd_add(num, DD{d * d * vol, 0.0});
            den = dd_add(den, DD{kappa_m[c] * kappa_m[c] * vol, 0.0});
        } else if (eps_mode == 2) {
            const double d = lam - lam_reb[c];
            num = dd_add(num, DD{d * d * vol, 0.0});
        }
    }
    if (eps_mode < 0) return;
    kappa_eps_tail(num, den, sc, M, eps_mode, part, counter, decide_method, rebuilt, eta);
}

// Row-marching k_kappa (same outputs): a warp owns 31 columns (lane 0 is the
// west halo column) and `rows` rows. The west neighbour's conductivity comes
// by shuffle and the south one stays in a register, so each cell's total
// mobility is evaluated once (k_kappa evaluates it three times per cell with
// T and recovers (i, j) by a division). Transmissibilities use the same
// harm_trans_v / harm_trans_h operations on the same conductivity values, so
// kappa and T are bit-identical; the drift sums are double-double as in
// k_kappa (only the partition into partials differs). Warp tasks are
// grid-strided over one resident wave, so c.red holds the block partials.
constexpr int KC_COLS = 31;
__global__ void __launch_bounds__(256) k_kappa_col(Layout L, const double* __restrict__ K, const double* __restrict__ s,
                                                   double* __restrict__ kappa, const double* __restrict__ kappa_m,
                                                   const double* __restrict__ lam_reb, Scalars* sc, double M,
                                                   int eps_mode, double* part, unsigned* counter, int decide_method,
                                                   int rebuilt, double eta, double* __restrict__ T, int rows) {
    pdl_begin();
    const double vol = L.vol();
    const int lane = threadIdx.x & 31;
    const int ncw = (L.nx + KC_COLS - 1) / KC_COLS, tasks = ncw * ((L.ny + rows - 1) / rows);
    DD num{0.0, 0.0}, den{0.0, 0.0};
    unsigned long long clampc = 0;
    bool bad = false;
    for (int task = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); task < tasks;
         task += gridDim.x * (blockDim.x >> 5)) {  // warp-uniform
        const int wc = task % ncw, j0 = (task / ncw) * rows, j1 = min(j0 + rows, L.ny);
        const int i = wc * KC_COLS + lane - 1;
        const bool col = i >= 0 && i < L.nx, own = col && lane >= 1;
        const int ic = col ? i : 0;
        double kS = 0.0;
        if (col && j0 > 0) kS = total_mob(s[L.cell(ic, j0 - 1)], M, nullptr) * K[L.cell(ic, j0 - 1)];
#pragma unroll 2
        for (int j = j0; j < j1; ++j) {
            const int c = L.cell(ic, j);
            const double sv = col ? s[c] : 0.0, Kv = col ? K[c] : 1.0;
            const double km = (own && (eps_mode == 0 || eps_mode == 1)) ? kappa_m[c] : 0.0;
            const double lr = (own && eps_mode == 2) ? lam_reb[c] : 0.0;
            const double lam = total_mob(sv, M, nullptr);
            const double k = lam * Kv;
            const double kW = __shfl_up_sync(0xffffffffu, k, 1);
            if (own) {
                clampc += (sv < 0.0 || sv > 1.0) ? 1 : 0;  // the cell's own evaluation counts (transport.cpp:13-21)
                kappa[c] = k;
                if (T) {  // elliptic.cpp:44-61 for this cell's faces (boundary faces carry 0)
                    T[L.vface(i, j)] = i > 0 ? harm_trans_v(L, kW, k) : 0.0;
                    T[L.hface(i, j)] = j > 0 ? harm_trans_h(L, kS, k) : 0.0;
                    if (i == L.nx - 1) T[L.vface(L.nx, j)] = 0.0;
                    if (j == L.ny - 1) T[L.hface(i, L.ny)] = 0.0;
                }
                bad |= !(k > 0.0) || !isfinite(k);
                if (eps_mode == 0 || eps_mode == 1) {
                    const double d = k - km;
                    num = dd_add(num, DD{d * d * vol, 0.0});
                    den = dd_add(den, DD{km * km * vol, 0.0});
                } else if (eps_mode == 2) {
                    const double d = lam - lr;
                    num = dd_add(num, DD{d * d * vol, 0.0});
                }
            }
            kS = k;
        }
    }
    if (clampc) atomicAdd((unsigned long long*)&sc->clamp, clampc);
    if (bad) atomicOr(&sc->err, ERR_KAPPA);
    if (eps_mode < 0) return;
    kappa_eps_tail(num, den, sc, M, eps_mode, part, counter, decide_method, rebuilt, eta);
}

// The MPM-2P vs MRCM decision for the NEXT step, on the device
// (simulation.cpp:307-323): eps is exactly 0 after a rebuild.
__device__ __forceinline__ void decide(Scalars* sc, int rebuilt, int method, double eta, int step) {
    const double eps = rebuilt ? 0.0 : sc->eps_pending;
    sc->eps = eps;
    int rb = 0;
    if (method == 1) rb = 1;                                // MrcmEveryStep
    else if (method == 2) rb = (eta <= 0.0) || (eps > eta);  // Mpm2p, strict >
    sc->rebuild_next = rb;
    if (method == 2 && eta > 0.0 && step >= 1) {
        const double m = fabs(eps - eta) / eta;
        if (m < sc->min_margin) sc->min_margin = m;
    }
}
__global__ void k_decide(Scalars* sc, int rebuilt, int method, double eta, int step) {
    pdl_begin();
    decide(sc, rebuilt, method, eta, step);
}

// max_outlet_saturation (simulation.cpp:61-83): one block, four sides.
__global__ void k_outlet(Layout L, const double* __restrict__ s, const double* __restrict__ u, Scalars* sc) {
    pdl_begin();
    __shared__ double sh[32];
    double m = 0.0;
    for (int side = 0; side < 4; ++side) {
        const int count = side < 2 ? L.ny : L.nx;
        const double area = side < 2 ? L.hy : L.hx;
        auto face_of = [&](int k) {
            switch (side) {
                case 0: return -u[L.vface(0, k)];
                case 1: return u[L.vface(L.nx, k)];
                case 2: return -u[L.hface(k, 0)];
                default: return u[L.hface(k, L.ny)];
            }
        };
        auto cell_of = [&](int k) {
            switch (side) {
                case 0: return L.cell(0, k);
                case 1: return L.cell(L.nx - 1, k);
                case 2: return L.cell(k, 0);
                default: return L.cell(k, L.ny - 1);
            }
        };
        double net = 0.0;
        for (int k = threadIdx.x; k < count; k += blockDim.x) net += face_of(k) * area;
        net = block_reduce(net, [](double a, double b) { return a + b; }, sh, 0.0);
        __shared__ double net_s;
        if (threadIdx.x == 0) net_s = net;
        __syncthreads();
        if (net_s > 1e-14) {
            double mm = 0.0;
            for (int k = threadIdx.x; k < count; k += blockDim.x)
                if (face_of(k) > 1e-14) mm = fmax(mm, s[cell_of(k)]);
            mm = block_reduce(mm, [](double a, double b) { return fmax(a, b); }, sh, 0.0);
            m = fmax(m, mm);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) sc->outlet_max = m;
}

__global__ void k_divergence(Layout L, const double* __restrict__ u, double* __restrict__ div) {
    pdl_begin();  // grid.cpp:19-31
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= L.cells()) return;
    const int i = c % L.nx, j = c / L.nx;
    const double fx = (u[L.vface(i + 1, j)] - u[L.vface(i, j)]) * L.hy;
    const double fy = (u[L.hface(i, j + 1)] - u[L.hface(i, j)]) * L.hx;
    div[c] = (fx + fy) / L.vol();
}

// epsilon(kappa_n, kappa_m, mode) on two arbitrary fields (mpm.cpp:9-25).
__global__ void k_eps_fields(Layout L, const double* __restrict__ kn, const double* __restrict__ km, Scalars* sc,
                             int mode, double* part, unsigned* counter) {
    pdl_begin();
    __shared__ DD shd[32];
    const double vol = L.vol();
    DD num{0.0, 0.0}, den{0.0, 0.0};
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < L.cells(); c += gridDim.x * blockDim.x) {
        const double d = kn[c] - km[c];
        num = dd_add(num, DD{d * d * vol, 0.0});
        den = dd_add(den, DD{km[c] * km[c] * vol, 0.0});
    }
    num = block_reduce_dd(num, shd);
    den = block_reduce_dd(den, shd);
    if (threadIdx.x == 0) {
        part[4 * blockIdx.x + 0] = num.hi;
        part[4 * blockIdx.x + 1] = num.lo;
        part[4 * blockIdx.x + 2] = den.hi;
        part[4 * blockIdx.x + 3] = den.lo;
    }
    if (last_block_done(counter)) {
        const DD n = reduce_dd_partials(part, gridDim.x, 0, shd);
        const DD d = reduce_dd_partials(part, gridDim.x, 2, shd);
        if (threadIdx.x == 0) {
            const double a = sqrt(n.hi);
            if (mode == 1) sc->eps_pending = a;
            else {
                if (!(d.hi > 0.0)) atomicOr(&sc->err, ERR_EPS_ZERO);
                sc->eps_pending = a / sqrt(d.hi);
            }
            *counter = 0;
        }
    }
}

__global__ void k_lambda(Layout L, const double* __restrict__ s, double* __restrict__ lam, Scalars* sc, double M) {
    pdl_begin();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;  // mobility_field (simulation.cpp:156-160)
    if (c < L.cells()) lam[c] = total_mob(s[c], M, &sc->clamp);
}



// relative_flux_error / relative_sat_error (simulation.cpp:30-59) in
// double-double: area-weighted L2 of u - u_ref over all faces, L1 of
// s - s_ref over cells, each relative to the reference's norm.
__global__ void k_track_errors(Layout L, const double* __restrict__ u, const double* __restrict__ ur,
                               const double* __restrict__ s, const double* __restrict__ sr, Scalars* sc,
                               double* part, unsigned* counter) {
    pdl_begin();
    DD fn{0.0, 0.0}, fd{0.0, 0.0}, sn{0.0, 0.0}, sd{0.0, 0.0};
    const int nf = L.faces(), nc = L.cells();
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nf; f += gridDim.x * blockDim.x) {
        const double w = L.area(f), d = u[f] - ur[f];
        fn = dd_add(fn, DD{w * d * d, 0.0});
        fd = dd_add(fd, DD{w * ur[f] * ur[f], 0.0});
        if (f < nc) {
            sn = dd_add(sn, DD{fabs(s[f] - sr[f]), 0.0});
            sd = dd_add(sd, DD{fabs(sr[f]), 0.0});
        }
    }
    __shared__ DD shd[64];
    block_reduce_dd2(fn, fd, shd);
    block_reduce_dd2(sn, sd, shd);
    if (threadIdx.x == 0) {
        double* pp = part + 8 * blockIdx.x;
        pp[0] = fn.hi; pp[1] = fn.lo; pp[2] = fd.hi; pp[3] = fd.lo;
        pp[4] = sn.hi; pp[5] = sn.lo; pp[6] = sd.hi; pp[7] = sd.lo;
    }
    if (!last_block_done(counter)) return;
    DD a{0.0, 0.0}, b{0.0, 0.0}, e{0.0, 0.0}, g{0.0, 0.0};
    for (int k = threadIdx.x; k < (int)gridDim.x; k += blockDim.x) {
        const double* pp = part + 8 * k;
        a = dd_add(a, DD{__ldcg(pp + 0), __ldcg(pp + 1)});
        b = dd_add(b, DD{__ldcg(pp + 2), __ldcg(pp + 3)});
        e = dd_add(e, DD{__ldcg(pp + 4), __ldcg(pp + 5)});
        g = dd_add(g, DD{__ldcg(pp + 6), __ldcg(pp + 7)});
    }
    block_reduce_dd2(a, b, shd);
    block_reduce_dd2(e, g, shd);
    if (threadIdx.x == 0) {
        const double num = a.hi + a.lo, den = b.hi + b.lo, sn2 = e.hi + e.lo, sd2 = g.hi + g.lo;
        if (!(den > 0.0)) {
            sc->flux_err = 0.0;
            if (num != 0.0) atomicOr(&sc->err, ERR_TRACK_ZERO);
        } else {
            sc->flux_err = sqrt(num / den);
        }
        if (sn2 == 0.0) sc->sat_err = 0.0;  // simulation.cpp:219-221: exact agreement reports 0
        else if (!(sd2 > 0.0)) atomicOr(&sc->err, ERR_TRACK_ZERO);
        else sc->sat_err = sn2 / sd2;
        *counter = 0;
    }
}

__global__ void k_save_dt_main(Scalars* sc) {
    pdl_begin();
    sc->dt_main = sc->dt;
}

}  // namespace

void launch_max_slope(Ctx& c) {
    {
        PROF(c, "k_max_slope");
        launch_k(c, k_max_slope, 1, 1024, 0, c.sc, c.M);
        CK_LAUNCH();
    }
}
void launch_cfl(Ctx& c, const double* u, double safety, double dt_cap) {
    {
        PROF(c, "k_cfl");
        launch_k(c, k_cfl, red_blocks(c, k_cfl, c.L.cells()), TPB, 0, c.L, u, c.sc, safety, dt_cap, c.red, c.red_count, 0, 0.0, 1.0);
        CK_LAUNCH();
    }
}
void launch_inj_pvi(Ctx& c, const double* u, double inflow, int cn, bool add_pvi) {
    {
        PROF(c, "k_inj_pvi");
        launch_k(c, k_inj_pvi, 1, TPB, 0, c.L, u, c.sc, inflow, c.M, cn, add_pvi ? 1 : 0);
        CK_LAUNCH();
    }
}
void launch_upwind(Ctx& c, const double* s_in, double* s_out, const double* u, double inflow, bool take_next,
                   int inj_cn, int sub) {
    {
        PROF(c, "k_upwind");
        const int rows = upwind_col_rows(c.L, c.num_sms);
        // auto (-1): column marching where each warp gets a long segment
        // (C5: 191 vs 254 us); short segments (C2, C4) keep the tiled step
        if (c.upwind_col > 0 || (c.upwind_col < 0 && rows >= 16)) {
            const long ncw = (c.L.nx + UC_COLS - 1) / UC_COLS, warps = ncw * ((c.L.ny + rows - 1) / rows);
            launch_k(c, k_upwind_col<1, 4>, (int)((warps + 7) / 8), 256, 0, c.L, s_in, s_out, u, c.sc, inflow, c.M,
                     take_next ? 1 : 0, inj_cn, sub, rows);
        } else if (c.upwind_tiled)
            launch_k(c, k_upwind_tile, dim3(cdiv(c.L.nx, UT_X), cdiv(c.L.ny, UT_Y)), UT_X * UT_Y, 0, c.L, s_in, s_out, u,
                     c.sc, inflow, c.M, take_next ? 1 : 0, inj_cn, sub);
        else
            launch_k(c, k_upwind, cdiv(c.L.cells(), TPB), TPB, 0, c.L, s_in, s_out, u, c.sc, inflow, c.M,
                     take_next ? 1 : 0, inj_cn, sub);
        CK_LAUNCH();
    }
}
void launch_cfl_inj(Ctx& c, const double* u, double safety, double dt_cap, double inflow, int cn) {
    PROF(c, "k_cfl");
    launch_k(c, k_cfl, red_blocks(c, k_cfl, c.L.cells()), TPB, 0, c.L, u, c.sc, safety, dt_cap, c.red, c.red_count, cn, inflow, c.M);
    CK_LAUNCH();
}
// auto (kappa_col < 0): the row-marching kernel where warps get long row
// segments (C5); otherwise the one-thread-per-cell k_kappa
static void launch_kappa(Ctx& c, const double* s, double* kappa, int eps_mode, int method, int rebuilt, double eta,
                         double* T) {
    const long ncw = (c.L.nx + KC_COLS - 1) / KC_COLS;
    int rows = 32;
    while (rows > 4 && ncw * ((c.L.ny + rows - 1) / rows) < 48L * c.num_sms) rows >>= 1;
    if (c.kappa_col > 0 || (c.kappa_col < 0 && rows >= 16)) {
        const long tasks = ncw * ((c.L.ny + rows - 1) / rows);
        launch_k(c, k_kappa_col, red_blocks(c, k_kappa_col, 32 * tasks), TPB, 0, c.L, c.K, s, kappa, c.kappa_m,
                 c.lam_reb, c.sc, c.M, eps_mode, c.red, c.red_count, method, rebuilt, eta, T, rows);
    } else {
        launch_k(c, k_kappa, red_blocks(c, k_kappa, c.L.cells()), TPB, 0, c.L, c.K, s, kappa, c.kappa_m, c.lam_reb,
                 c.sc, c.M, eps_mode, c.red, c.red_count, method, rebuilt, eta, T);
    }
}
void launch_conductivity_decide(Ctx& c, const double* s, double* kappa, int eps_mode, int rebuilt, int method,
                                double eta) {
    PROF(c, "k_kappa");
    launch_kappa(c, s, kappa, eps_mode, method, rebuilt, eta, c.T.p);
    c.trans_fresh = true;
    c.kappa_checked = true;  // k_kappa flags a non-positive / non-finite kappa itself  // T = transmissibility(kappa) is current: the next rebuild / MPM step skips k_trans
    CK_LAUNCH();
}
void launch_conductivity(Ctx& c, const double* s, double* kappa, int eps_mode, bool want_eps) {
    {
        PROF(c, "k_kappa");
        launch_kappa(c, s, kappa, want_eps ? eps_mode : -1, -1, 0, 0.0, nullptr);
        CK_LAUNCH();
    }
}
void launch_lambda(Ctx& c, const double* s, double* lam) {
    {
        PROF(c, "k_lambda");
        launch_k(c, k_lambda, cdiv(c.L.cells(), TPB), TPB, 0, c.L, s, lam, c.sc, c.M);
        CK_LAUNCH();
    }
}
void launch_outlet(Ctx& c, const double* s, const double* u) {
    {
        PROF(c, "k_outlet");
        launch_k(c, k_outlet, 1, TPB, 0, c.L, s, u, c.sc);
        CK_LAUNCH();
    }
}
void launch_divergence(Ctx& c, const double* u, double* div) {
    {
        PROF(c, "k_divergence");
        launch_k(c, k_divergence, cdiv(c.L.cells(), TPB), TPB, 0, c.L, u, div);
        CK_LAUNCH();
    }
}
void launch_decide(Ctx& c, int rebuilt, int method, double eta, int step) {
    {
        PROF(c, "k_decide");
        launch_k(c, k_decide, 1, 1, 0, c.sc, rebuilt, method, eta, step);
        CK_LAUNCH();
    }
}
void launch_epsilon_fields(Ctx& c, const double* kn, const double* km, int mode) {
    {
        PROF(c, "k_eps_fields");
        launch_k(c, k_eps_fields, red_blocks(c, k_eps_fields, c.L.cells()), TPB, 0, c.L, kn, km, c.sc, mode, c.red, c.red_count);
        CK_LAUNCH();
    }
}

}  // namespace mpm2p

namespace mpm2p {
void launch_track_errors(Ctx& c, const double* u, const double* ur, const double* s, const double* sr) {
    PROF(c, "k_track_errors");
    launch_k(c, k_track_errors, red_blocks(c, k_track_errors, c.L.faces()), TPB, 0, c.L, u, ur, s, sr, c.sc, c.red,
             c.red_count);
    CK_LAUNCH();
}
void launch_save_dt_main(Ctx& c) {
    PROF(c, "k_save_dt_main");
    launch_k(c, k_save_dt_main, 1, 1, 0, c.sc.p);
    CK_LAUNCH();
}
}  // namespace mpm2p
