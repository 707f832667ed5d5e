// dense.cu — dense interface-system machinery (stand-in for Eigen
// PartialPivLU + rcond, proj/src/mrcm.cpp:225-238,264, and the dense LDLT of
// the repair Laplacian, mrcm.cpp:372).
//
// The interface matrix is fixed between rebuilds, so it is inverted once per
// rebuild and every later interface solve is a dense GEMV plus one step of
// iterative refinement against the sparse CSR operator — as accurate as the
// reference's LU solve, and bandwidth-bound rather than latency-bound.
//
// Inversion is blocked Gauss-Jordan with partial pivoting on [A | I], one
// cooperative kernel, per panel of b columns:
//   1. CTA 0 factors the n x b panel in shared memory (pivot search, row
//      swaps, elimination), keeping the elimination vectors v_c in place of
//      the eliminated columns; the product T = prod_c (I - v_c e_c^T) of the
//      panel's b steps is I - G E_R^T with G = V * alpha (alpha: a b x b
//      triangular recurrence on the pivot rows).
//   2. all CTAs apply the panel's row swaps and snapshot the b pivot rows;
//   3. all CTAs apply the rank-b update W -= G * W[R, :] (GEMM-shaped).
// Three grid barriers per panel instead of three per pivot.
// rcond = 1 / (||A||_1 ||A^-1||_1) is computed on the device (the quantity
// Eigen's rcond() estimates) and compared to the reference's 1e-14 guard
// there, so a rebuild needs no host synchronisation.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

#include "context.cuh"

namespace cg = cooperative_groups;

namespace mpm2p {

namespace {

constexpr int TPB = 256;
constexpr int GJ_THREADS = 1024;

struct GJArgs {
    double* W;      // n x 2n, row-major
    int n, b;
    double* G;      // n x b
    int* swp;       // n: pivot row chosen for each column
    double* Rb;     // b x 2n pivot-row snapshot
    int* singular;
};

__global__ void __launch_bounds__(GJ_THREADS) k_gauss_jordan(GJArgs a) {
    pdl_begin();
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double sp[];  // panel n x b, row-major
    __shared__ double prow[16];
    __shared__ double alpha[16 * 16];
    __shared__ double wv[32];
    __shared__ int wi[32];
    const int n = a.n, b = a.b, n2 = 2 * n;
    const int tid = threadIdx.x, nt = blockDim.x;
    const long long gtid = (long long)blockIdx.x * blockDim.x + tid;
    const long long gnt = (long long)gridDim.x * blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
    for (int k0 = 0; k0 < n; k0 += b) {
        const int bb = (n - k0) < b ? (n - k0) : b;
        // ---- phase 1: panel factorization on CTA 0 --------------------------
        if (blockIdx.x == 0) {
            for (int x = tid; x < n * bb; x += nt) {
                const int i = x / bb, j = x % bb;
                sp[i * b + j] = a.W[(size_t)i * n2 + k0 + j];
            }
            __syncthreads();
            for (int c = 0; c < bb; ++c) {
                const int kc = k0 + c;
                double best = -1.0;
                int bi = kc;
                for (int i = kc + tid; i < n; i += nt) {
                    const double v = fabs(sp[i * b + c]);
                    if (v > best) { best = v; bi = i; }
                }
                for (int o = 16; o > 0; o >>= 1) {
                    const double ov = __shfl_down_sync(0xffffffffu, best, o);
                    const int oi = __shfl_down_sync(0xffffffffu, bi, o);
                    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
                }
                if (lane == 0) { wv[warp] = best; wi[warp] = bi; }
                __syncthreads();
                if (tid == 0) {
                    double bv = wv[0];
                    int bx = wi[0];
                    for (int w = 1; w < nwarps; ++w)
                        if (wv[w] > bv || (wv[w] == bv && wi[w] < bx)) { bv = wv[w]; bx = wi[w]; }
                    wi[0] = bx;
                    a.swp[kc] = bx;
                    if (!(bv > 0.0)) *a.singular = 1;
                }
                __syncthreads();
                const int q = wi[0];
                if (q != kc && tid < bb) {
                    const double t = sp[kc * b + tid];
                    sp[kc * b + tid] = sp[q * b + tid];
                    sp[q * b + tid] = t;
                }
                __syncthreads();
                if (tid < bb) prow[tid] = sp[kc * b + tid];
                __syncthreads();
                const double piv = prow[c];
                const double pinv = 1.0 / piv;
                for (int i = tid; i < n; i += nt) {
                    double* r = sp + i * b;
                    if (i == kc) {
                        for (int j = c + 1; j < bb; ++j) r[j] = prow[j] * pinv;
                        r[c] = (piv - 1.0) * pinv;  // v_c at the pivot row
                    } else {
                        const double m = r[c] * pinv;
                        for (int j = c + 1; j < bb; ++j) r[j] -= m * prow[j];
                        r[c] = m;                   // v_c elsewhere
                    }
                }
                __syncthreads();
            }
            // alpha: g_j = sum_{c>=j} v_c alpha[c][j] (thread j owns column j)
            if (tid < bb) {
                const int j = tid;
                double y[16];
                for (int r = 0; r < bb; ++r) y[r] = (r == j ? 1.0 : 0.0) - sp[(k0 + r) * b + j];
                for (int c = 0; c < bb; ++c) alpha[c * 16 + j] = 0.0;
                alpha[j * 16 + j] = 1.0;
                for (int c = j + 1; c < bb; ++c) {
                    const double yc = y[c];
                    alpha[c * 16 + j] = yc;
                    for (int r = 0; r < bb; ++r) y[r] -= sp[(k0 + r) * b + c] * yc;
                }
            }
            __syncthreads();
            for (int i = tid; i < n; i += nt) {
                double g[16];
                for (int j = 0; j < bb; ++j) g[j] = 0.0;
                for (int c = 0; c < bb; ++c) {
                    const double v = sp[i * b + c];
                    for (int j = 0; j <= c; ++j) g[j] += v * alpha[c * 16 + j];
                }
                for (int j = 0; j < bb; ++j) a.G[(size_t)i * b + j] = g[j];
            }
        }
        grid.sync();
        // ---- phase 2: row swaps on the active columns, pivot-row snapshot ----
        for (long long j = k0 + gtid; j < n2; j += gnt) {
            for (int c = 0; c < bb; ++c) {
                const int kc = k0 + c, q = a.swp[kc];
                if (q != kc) {
                    const double t = a.W[(size_t)kc * n2 + j];
                    a.W[(size_t)kc * n2 + j] = a.W[(size_t)q * n2 + j];
                    a.W[(size_t)q * n2 + j] = t;
                }
            }
            for (int c = 0; c < bb; ++c) a.Rb[(size_t)c * n2 + j] = a.W[(size_t)(k0 + c) * n2 + j];
        }
        grid.sync();
        // ---- phase 3: W[:, k0:] -= G * Rb, tiles of 64 rows x 128 columns -----
        {
            double* sg = sp;               // 64 x 16 tile of G
            double* sr = sp + 64 * 16;     // 16 x 128 tile of Rb
            const int ncol = n2 - k0;
            const int tr = (n + 63) / 64, tc = (ncol + 127) / 128;
            const int ty = tid >> 5, tx = tid & 31;  // 32 x 32 threads: 2 rows x 4 cols each
            for (int tile = blockIdx.x; tile < tr * tc; tile += gridDim.x) {
                const int i0 = (tile / tc) * 64, j0 = k0 + (tile % tc) * 128;
                __syncthreads();
                for (int x = tid; x < 64 * 16; x += nt) {
                    const int i = i0 + x / 16, c = x % 16;
                    sg[x] = (i < n && c < bb) ? a.G[(size_t)i * b + c] : 0.0;
                }
                for (int x = tid; x < 16 * 128; x += nt) {
                    const int c = x / 128, j = j0 + x % 128;
                    sr[x] = (c < bb && j < n2) ? a.Rb[(size_t)c * n2 + j] : 0.0;
                }
                __syncthreads();
                double acc[2][4];
#pragma unroll
                for (int r = 0; r < 2; ++r)
#pragma unroll
                    for (int q = 0; q < 4; ++q) acc[r][q] = 0.0;
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                    double gv[2], rv[4];
#pragma unroll
                    for (int r = 0; r < 2; ++r) gv[r] = sg[(ty + 32 * r) * 16 + c];
#pragma unroll
                    for (int q = 0; q < 4; ++q) rv[q] = sr[c * 128 + tx + 32 * q];
#pragma unroll
                    for (int r = 0; r < 2; ++r)
#pragma unroll
                        for (int q = 0; q < 4; ++q) acc[r][q] += gv[r] * rv[q];
                }
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const int i = i0 + ty + 32 * r;
                    if (i >= n) continue;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int j = j0 + tx + 32 * q;
                        if (j < n2) a.W[(size_t)i * n2 + j] -= acc[r][q];
                    }
                }
            }
        }
        grid.sync();
    }
}


// ---- ping-pong blocked Gauss-Jordan with lookahead -------------------------
// Pivot-free Gauss-Jordan over 32 x 32 blocks of a padded npad x npad matrix
// (stable without pivoting for the quasi-definite K = J M, SURVEY.md H1, and
// the SPD repair Laplacian), structured so each block step costs ONE grid
// barrier: step k reads W_src and writes W_dst (no read/write conflicts inside
// a step), and a dedicated lookahead CTA updates the next diagonal block and
// inverts it during step k, so P_{k+1} = W_{k+1,k+1}^-1 is ready when step k+1
// starts. Work items are (block row i, chunk of cpb block columns). Per step:
//   i != k : T = W_ik P_k ;  W'_ij = W_ij - T W_kj (j != k) ;  W'_ik = -T
//   i == k : W'_kj = P_k W_kj (j != k) ;  W'_kk = P_k
constexpr int PPB = 32;
struct PPArgs {
    double* W0;
    double* W1;
    double* P;  // two 32 x 32 slots (P_k in slot k % 2)
    int ld;     // = npad = nb * 32
    int nb, nch, cpb;
    int* singular;
    int* aux;  // [0] the lookahead CTA's SM id, [1] the worker CTA sharing that SM (-1: none)
    unsigned long long* trace;  // optional (MPM2P_GJ_TRACE=1): per-step %globaltimer marks
};
typedef double PPTile[PPB][PPB + 1];

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// All loads issued before any store (one L2 round trip, not four); 256 threads.
__device__ __forceinline__ void pp_load(PPTile S, const double* g, int ld) {
    double v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int x = threadIdx.x + 256 * q;
        v[q] = __ldcg(g + (size_t)(x >> 5) * ld + (x & 31));
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int x = threadIdx.x + 256 * q;
        S[x >> 5][x & 31] = v[q];
    }
}
// D += A B on the fp64 tensor cores (mma.sync m8n8k4, DMMA): A 8 x 4 row-major,
// lane l holds A[l / 4][l % 4]; B 4 x 8, lane l holds B[l % 4][l / 4]; C/D
// 8 x 8, lane l holds D[l / 4][2 (l % 4) + {0, 1}].
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}
// Split load: every thread's four loads of a 32 x 32 tile into registers
// (pp_fetch), later stored to shared memory (pp_put), so several tiles'
// loads are in flight together (one L2 round trip for all of them).
__device__ __forceinline__ void pp_fetch(double (&v)[4], const double* g, int ld) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int x = threadIdx.x + 256 * q;
        v[q] = __ldcg(g + (size_t)(x >> 5) * ld + (x & 31));
    }
}
__device__ __forceinline__ void pp_put(PPTile S, const double (&v)[4]) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int x = threadIdx.x + 256 * q;
        S[x >> 5][x & 31] = v[q];
    }
}
// thread t owns row t >> 3 and columns (t & 7) + 8 m of a 32 x 32 result
__device__ __forceinline__ void pp_mul(const PPTile X, const PPTile Y, double out[4]) {
    const int r = threadIdx.x >> 3, c0 = threadIdx.x & 7;
#pragma unroll
    for (int m = 0; m < 4; ++m) out[m] = 0.0;
#pragma unroll 8
    for (int t = 0; t < PPB; ++t) {
        const double x = X[r][t];
#pragma unroll
        for (int m = 0; m < 4; ++m) out[m] = fma(x, Y[t][c0 + 8 * m], out[m]);
    }
}
// In-place inverse of S (pivot-free GJ) on 4 warps (one per SM sub-
// partition): warp w keeps columns 8w..8w+7 of row `lane` in registers. Per
// pivot k the 8-column slice of row k is exchanged inside each warp and
// column k (with the pivot) across the 4 warps, double-buffered by pivot
// parity: one 128-thread named barrier per pivot. Row update
// v = fma(-f, r_k, v) * s with (f, s) = (A_rk p, 1) off the pivot row and
// (0, p) on it, so the new pivot row is r_k * p exactly. Flags a zero /
// non-finite pivot. Uses xb[2 * 32 + 4 * 2 * 8] doubles (16-byte aligned).
__device__ void pp_invert(PPTile S, double* xb, int* singular) {
    if (threadIdx.x < 128) {
        const int w = threadIdx.x >> 5, r = threadIdx.x & 31;
        double v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = S[r][8 * w + j];
#pragma unroll
        for (int k = 0; k < PPB; ++k) {
            const int kw = k >> 3, kj = k & 7;
            double* cb = xb + (k & 1) * PPB;
            double2* rb = reinterpret_cast<double2*>(xb + 2 * PPB + (w * 2 + (k & 1)) * 8);
            if (r == k) {
#pragma unroll
                for (int q = 0; q < 4; ++q) rb[q] = make_double2(v[2 * q], v[2 * q + 1]);
            }
            if (w == kw) cb[r] = v[kj];
            asm volatile("bar.sync 1, 128;" ::: "memory");
            double rk[8];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double2 t = rb[q];
                rk[2 * q] = t.x;
                rk[2 * q + 1] = t.y;
            }
            const double piv = cb[k];
            const double colk = cb[r];
            const double p = fast_rcp(piv);  // Newton-refined (<= 1 ulp), off the division slow path
            if (threadIdx.x == 0 && (!(piv != 0.0) || !isfinite(piv))) *singular = 1;
            const bool on = r == k;
            const double f = on ? 0.0 : colk * p;
            const double sc = on ? p : 1.0;
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = fma(-f, rk[j], v[j]) * sc;
            if (w == kw) v[kj] = on ? p : -f;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) S[r][8 * w + j] = v[j];
    }
    __syncthreads();
}

// Dynamic shared memory of k_gj_pp: four 32 x 33 tiles, a 32 x 128 slice of
// the pivot block row, and the pivot row/column exchange buffers.
constexpr int PPW = 128;  // columns per work item (4 blocks)
constexpr int PWS = PPW + 8;  // padded row stride of the pivot block-row slice (conflict-free DMMA B loads)
constexpr size_t PP_SMEM = (4 * PPB * (PPB + 1) + PPB * PWS + 2 * PPB + 4 * 2 * 8) * sizeof(double);

__global__ void __launch_bounds__(256, 2) k_gj_pp(PPArgs a) {
    pdl_begin();
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double pp_sm[];
    PPTile& Ps = *reinterpret_cast<PPTile*>(pp_sm);
    PPTile& Cs = *reinterpret_cast<PPTile*>(pp_sm + PPB * (PPB + 1));
    PPTile& Ts = *reinterpret_cast<PPTile*>(pp_sm + 2 * PPB * (PPB + 1));
    PPTile& Bs = *reinterpret_cast<PPTile*>(pp_sm + 3 * PPB * (PPB + 1));
    double* Ws = pp_sm + 4 * PPB * (PPB + 1);  // 32 x 128, row-major, row stride PWS
    double* xrow = Ws + PPB * PWS;  // pivot-row exchange (2 x 32, 16-byte aligned)
    const int ld = a.ld, nb = a.nb, np = nb * PPB;
    const int r = threadIdx.x >> 3, c0 = threadIdx.x & 7;
    // DMMA (mma.m8n8k4.f64) fragments: warp w owns rows 8 (w & 3).. of the item and
    // columns 64 (w >> 2).. (eight 8 x 8 tiles); lane (lr, lc) = (lane / 4, lane % 4)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int lr = lane >> 2, lc = lane & 3, rg = warp & 3, ch = warp >> 2;
    const bool look = blockIdx.x == gridDim.x - 1;
    const int nch = (np + PPW - 1) / PPW;
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (look && threadIdx.x == 0) a.aux[0] = (int)smid;
    auto blk = [&](double* W, int I, int J) { return W + (size_t)I * PPB * ld + (size_t)J * PPB; };
    auto pslot = [&](int k) { return a.P + (size_t)(k & 1) * PPB * PPB; };
    if (look) {  // P_0
        pp_load(Cs, a.W0, ld);
        __syncthreads();
        pp_invert(Cs, xrow, a.singular);
        for (int x = threadIdx.x; x < PPB * PPB; x += blockDim.x) pslot(0)[x] = Cs[x >> 5][x & 31];
    }
    grid.sync();
    // The lookahead chain (load, two 32^3 products, a 32-pivot inverse) is the
    // critical path of every step; a worker CTA on the same SM competes for
    // its shared-memory and FP64 issue slots (measured: prep 3.2 -> 6.0 us).
    // That worker sits the steps out; the others take its items.
    if (!look && gridDim.x > 2 && threadIdx.x == 0 && __ldcg(a.aux) == (int)smid) a.aux[1] = (int)blockIdx.x;
    grid.sync();
    const int idle = __ldcg(a.aux + 1);
    const int nwork = gridDim.x - 1 - (idle >= 0 ? 1 : 0);
    const int widx = (idle >= 0 && (int)blockIdx.x > idle) ? (int)blockIdx.x - 1 : (int)blockIdx.x;
    const bool works = !look && (int)blockIdx.x != idle;
    for (int k = 0; k < nb; ++k) {
        double* src = (k & 1) ? a.W1 : a.W0;
        double* dst = (k & 1) ? a.W0 : a.W1;
        auto mark = [&](int slot) {
            if (a.trace && threadIdx.x == 0) a.trace[(size_t)k * 8 + slot] = gtimer();
        };
        double pv[4];
        pp_fetch(pv, pslot(k), PPB);  // P_k: put into Ps together with each branch's first loads
        if (look) mark(0);
        if (!look && blockIdx.x == 0) mark(5);
        if (look) {
            if (k + 1 < nb) {  // next pivot block: W_{k+1,k+1} - (W_{k+1,k} P_k) W_{k,k+1}, inverted
                // all inputs (P_k, W_{k+1,k+1}, W_{k+1,k}, W_{k,k+1}) in one round of loads
                const double* g = blk(src, k + 1, k + 1);
                double gv[4], cv[4], bv[4];
#pragma unroll
                for (int m = 0; m < 4; ++m) gv[m] = __ldcg(g + (size_t)r * ld + c0 + 8 * m);
                pp_fetch(cv, blk(src, k + 1, k), ld);
                pp_fetch(bv, blk(src, k, k + 1), ld);
                pp_put(Ps, pv);
                pp_put(Cs, cv);
                pp_put(Bs, bv);
                __syncthreads();
                double t[4];
                pp_mul(Cs, Ps, t);
#pragma unroll
                for (int m = 0; m < 4; ++m) Ts[r][c0 + 8 * m] = t[m];
                __syncthreads();
                pp_mul(Ts, Bs, t);
                __syncthreads();
#pragma unroll
                for (int m = 0; m < 4; ++m) Cs[r][c0 + 8 * m] = gv[m] - t[m];
                __syncthreads();
                mark(1);
                const long long cy0 = clock64();
                pp_invert(Cs, xrow, a.singular);
                if (a.trace && threadIdx.x == 0) a.trace[(size_t)k * 8 + 4] = (unsigned long long)(clock64() - cy0);
                mark(2);
                for (int x = threadIdx.x; x < PPB * PPB; x += blockDim.x) pslot(k + 1)[x] = Cs[x >> 5][x & 31];
                mark(3);
            }
        } else if (works) {
            for (int item = widx; item < nb * nch; item += nwork) {
                const int i = item / nch, q = item % nch;
                const int col0 = q * PPW;
                const int row = rg * 8 + lr;  // this lane's output row in the block row
                // this lane's source values (the C fragments' positions), issued first, used last
                double2 gsrc[8];
#pragma unroll
                for (int cg = 0; cg < 8; ++cg) {
                    const int col = col0 + ch * 64 + cg * 8 + lc * 2;
                    gsrc[cg] = col < np ? __ldcg(reinterpret_cast<const double2*>(src + (size_t)(i * PPB + row) * ld + col))
                                        : make_double2(0.0, 0.0);
                }
                {  // W_ik and the pivot block-row slice W_k,[col0, col0+128) (columns past np
                   // read as 0): issued with gsrc's loads, one L2 round trip per item
                    double cv[4];
                    if (i != k) pp_fetch(cv, blk(src, i, k), ld);
                    double v[PPB * PPW / 256];
#pragma unroll
                    for (int qq = 0; qq < PPB * PPW / 256; ++qq) {
                        const int x = threadIdx.x + 256 * qq, rr = x / PPW, cc = col0 + x % PPW;
                        v[qq] = cc < np ? __ldcg(src + (size_t)(k * PPB + rr) * ld + cc) : 0.0;
                    }
                    __syncthreads();  // previous item's readers of Ps / Cs / Ts / Ws are done
                    if (item == widx) pp_put(Ps, pv);
                    if (i != k) pp_put(Cs, cv);
#pragma unroll
                    for (int qq = 0; qq < PPB * PPW / 256; ++qq) {
                        const int x = threadIdx.x + 256 * qq;
                        Ws[(x / PPW) * PWS + x % PPW] = v[qq];
                    }
                }
                __syncthreads();
                if (i != k) {  // T = W_ik P_k: warp w computes tiles (rg, 2 ch), (rg, 2 ch + 1)
                    double t[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
                    for (int kk = 0; kk < PPB / 4; ++kk) {
                        const double av = Cs[row][4 * kk + lc];
#pragma unroll
                        for (int f = 0; f < 2; ++f) dmma_8x8x4(t[f][0], t[f][1], av, Ps[4 * kk + lc][(2 * ch + f) * 8 + lr]);
                    }
#pragma unroll
                    for (int f = 0; f < 2; ++f) {
                        Ts[row][(2 * ch + f) * 8 + 2 * lc] = t[f][0];
                        Ts[row][(2 * ch + f) * 8 + 2 * lc + 1] = t[f][1];
                    }
                    __syncthreads();
                }
                const PPTile& Lf = (i == k) ? Ps : Ts;
                double af[PPB / 4];
#pragma unroll
                for (int kk = 0; kk < PPB / 4; ++kk) af[kk] = Lf[row][4 * kk + lc];
                double acc[8][2];
#pragma unroll
                for (int cg = 0; cg < 8; ++cg) acc[cg][0] = acc[cg][1] = 0.0;
#pragma unroll
                for (int kk = 0; kk < PPB / 4; ++kk) {
                    const double* wrow = Ws + (4 * kk + lc) * PWS + ch * 64 + lr;
#pragma unroll
                    for (int cg = 0; cg < 8; ++cg) dmma_8x8x4(acc[cg][0], acc[cg][1], af[kk], wrow[cg * 8]);
                }
                double* orow = dst + (size_t)(i * PPB + row) * ld;
#pragma unroll
                for (int cg = 0; cg < 8; ++cg) {
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int col = col0 + ch * 64 + cg * 8 + lc * 2 + e;
                        if (col >= np) continue;
                        const int jb = col / PPB, cl = col % PPB;
                        double o;
                        if (jb == k) o = (i == k) ? Ps[row][cl] : -Ts[row][cl];
                        else if (i == k) o = acc[cg][e];
                        else if (i == k + 1 && jb == k + 1) continue;  // the lookahead's block
                        else o = (e ? gsrc[cg].y : gsrc[cg].x) - acc[cg][e];
                        orow[col] = o;
                    }
                }
            }
            if (blockIdx.x == 0) mark(6);
        }
        grid.sync();
        if (blockIdx.x == 0) mark(7);
    }
}

// Rebuild path straight from the sparse operator (no dense M, no extra
// n^2 passes): padded K = J M is written row by row from the CSR rows of M
// (one warp per row: zero the row, then scatter), and the Gauss-Jordan
// result is turned into M^-1 = K^-1 J together with its column 1-norm
// partials in one pass (k_kinv_out); ||M||_1 comes from the CSR through the
// transposed-position table (the pattern is structurally symmetric).
__global__ void k_build_k(const int* __restrict__ ptr, const int* __restrict__ col, const double* __restrict__ val,
                          int n, double* __restrict__ W, int ld) {
    pdl_begin();
    const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (r >= ld) return;
    double* row = W + (size_t)r * ld;
    for (int j = lane; j < ld; j += 32) row[j] = (r >= n && j == r) ? 1.0 : 0.0;
    __syncwarp();
    if (r < n) {
        const int h = n / 2;
        const int srow = r < h ? h + r : r - h;
        const double sg = r < h ? 1.0 : -1.0;
        for (int z = ptr[srow] + lane; z < ptr[srow + 1]; z += 32) row[col[z]] = sg * val[z];
    }
}

// Minv[i][j] = (j < h ? -Kinv[i][h+j] : Kinv[i][j-h]); part[slab][n + j] =
// sum over the slab's 64 rows of |Minv[i][j]| (fixed order), part[slab][j] = 0
// (the A half is filled by k_mnorm). Block: 32 columns x 8 row groups.
__global__ void k_kinv_out(const double* __restrict__ Kinv, int ld, int n, double* __restrict__ Minv, double* part) {
    pdl_begin();
    __shared__ double red[8][33];
    const int c = threadIdx.x & 31, rg = threadIdx.x >> 5;
    const int j = blockIdx.x * 32 + c, slab = blockIdx.y;
    const int h = n / 2;
    double acc = 0.0;
    if (j < n) {
        const int pj = j < h ? h + j : j - h;
        const double sg = j < h ? -1.0 : 1.0;
        for (int t = 0; t < 8; ++t) {
            const int i = slab * 64 + rg + 8 * t;
            if (i >= n) break;
            const double v = sg * Kinv[(size_t)i * ld + pj];
            Minv[(size_t)i * n + j] = v;
            acc += fabs(v);
        }
    }
    red[rg][c] = acc;
    __syncthreads();
    if (rg == 0 && j < n) {
        double sacc = red[0][c];
        for (int g = 1; g < 8; ++g) sacc += red[g][c];
        part[(size_t)slab * 2 * n + n + j] = sacc;
        part[(size_t)slab * 2 * n + j] = 0.0;
    }
}

// ||M||_1 column sums from the CSR: column j's entries are M[i][j] for the
// pattern of row j (symmetric pattern), found at tpos[z] (z in row j).
__global__ void k_mnorm(const int* __restrict__ ptr, const int* __restrict__ tpos, const double* __restrict__ val,
                        int n, double* part) {
    pdl_begin();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    double s = 0.0;
    for (int z = ptr[j]; z < ptr[j + 1]; ++z) s += fabs(val[tpos[z]]);
    part[j] = s;  // slab 0, A half
}

// npad x npad copy with identity padding (and back).
__global__ void k_pad_in(const double* __restrict__ A, int n, double* __restrict__ W, int ld) {
    pdl_begin();
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < (long long)ld * ld;
         x += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(x / ld), j = (int)(x % ld);
        W[x] = (i < n && j < n) ? A[(size_t)i * n + j] : (i == j ? 1.0 : 0.0);
    }
}
__global__ void k_pad_out(const double* __restrict__ W, int ld, double* __restrict__ A, int n) {
    pdl_begin();
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < (long long)n * n;
         x += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(x / n), j = (int)(x % n);
        A[x] = W[(size_t)i * ld + j];
    }
}


// K = J M: phi-rows first, then the negated psi-rows.
__global__ void k_j_times(const double* __restrict__ M, double* __restrict__ K, int n) {
    pdl_begin();
    const int h = n / 2;
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < (long long)n * n;
         x += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(x / n), j = (int)(x % n);
        K[x] = i < h ? M[(size_t)(h + i) * n + j] : -M[(size_t)(i - h) * n + j];
    }
}

// M^-1 = K^-1 J: columns permuted and the psi half negated.
__global__ void k_times_j(const double* __restrict__ Kinv, double* __restrict__ Minv, int n) {
    pdl_begin();
    const int h = n / 2;
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < (long long)n * n;
         x += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(x / n), j = (int)(x % n);
        Minv[x] = j < h ? -Kinv[(size_t)i * n + h + j] : Kinv[(size_t)i * n + (j - h)];
    }
}

// max |A_ij - A_ji| and max |A_ij| (symmetry check of J M, once per context).
__global__ void k_asym(const double* __restrict__ A, int n, double* out) {
    pdl_begin();
    __shared__ double sh[32];
    double d = 0.0, m = 0.0;
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < (long long)n * n;
         x += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(x / n), j = (int)(x % n);
        d = fmax(d, fabs(A[x] - A[(size_t)j * n + i]));
        m = fmax(m, fabs(A[x]));
    }
    auto mx = [](double a, double b) { return fmax(a, b); };
    d = block_reduce_op(d, mx, 0.0, sh);
    m = block_reduce_op(m, mx, 0.0, sh);
    if (threadIdx.x == 0) {
        out[2 * blockIdx.x] = d;
        out[2 * blockIdx.x + 1] = m;
    }
}

__global__ void k_augment(const double* __restrict__ A, double* __restrict__ W, int n) {
    pdl_begin();
    const long long tot = 2LL * n * n;
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < tot; x += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(x / (2 * n)), j = (int)(x % (2 * n));
        W[x] = j < n ? A[(size_t)i * n + j] : (j - n == i ? 1.0 : 0.0);
    }
}

__global__ void k_extract(const double* __restrict__ W, double* __restrict__ Ainv, int n) {
    pdl_begin();
    const long long tot = (long long)n * n;
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < tot; x += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(x / n), j = (int)(x % n);
        Ainv[x] = W[(size_t)i * 2 * n + n + j];
    }
}

// Column 1-norms of A and B: partial column sums over row blocks of 64
// (grid y), coalesced along rows...
__global__ void k_colsum(const double* __restrict__ A, const double* __restrict__ B, int n, double* part) {
    pdl_begin();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const int i0 = blockIdx.y * 64, i1 = min(n, i0 + 64);
    double s1 = 0.0, s2 = 0.0;
    for (int i = i0; i < i1; ++i) {
        s1 += fabs(A[(size_t)i * n + j]);
        s2 += fabs(B[(size_t)i * n + j]);
    }
    part[(size_t)blockIdx.y * 2 * n + j] = s1;
    part[(size_t)blockIdx.y * 2 * n + n + j] = s2;
}

// ...then one block forms rcond = 1/(||A||_1 ||B||_1) and applies the guard.
__global__ void k_rcond(const double* __restrict__ part, int n, int nrb, const int* singular, double* rcond_out,
                        unsigned* err, unsigned err_bit, double threshold) {
    pdl_begin();
    __shared__ double sa[32], sb[32];
    double ma = 0.0, mb = 0.0;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        double s1 = 0.0, s2 = 0.0;
        for (int r = 0; r < nrb; ++r) {
            s1 += part[(size_t)r * 2 * n + j];
            s2 += part[(size_t)r * 2 * n + n + j];
        }
        ma = fmax(ma, s1);
        mb = fmax(mb, s2);
    }
    ma = warp_max(ma);
    mb = warp_max(mb);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) { sa[w] = ma; sb[w] = mb; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double na = sa[0], nb = sb[0];
        for (int t = 1; t < (int)(blockDim.x >> 5); ++t) { na = fmax(na, sa[t]); nb = fmax(nb, sb[t]); }
        double rc = 0.0;
        if (!*singular && isfinite(nb) && na > 0.0 && nb > 0.0) rc = 1.0 / (na * nb);
        *rcond_out = rc;
        if (!(rc > threshold)) atomicOr(err, err_bit);
    }
}

// y = A x: a 256-thread block covers 2 rows, 4 warps per row, each warp a
// quarter of the row with 4 independent loads in flight per lane (the GEMV is
// load-latency bound at these sizes, so more bytes in flight is the lever).
// y = A x (ACC: y += A x), one warp per row. HBM-bound: every lane issues
// its 16-byte loads of the row (and of x, L1/L2-resident) for 1024 columns
// before any FMA, so ~8 KB per warp is in flight. Rows must be 16-byte
// aligned (n even); odd n takes the scalar loop.
template <bool ACC>
__global__ void __launch_bounds__(256) k_gemv_w(const double* __restrict__ A, const double* __restrict__ x,
                                                double* __restrict__ y, int n) {
    pdl_begin();
    const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (row >= n) return;
    const double* a = A + (size_t)row * n;
    double acc0 = 0.0, acc1 = 0.0;
    if ((n & 1) == 0) {
        const double2* a2 = reinterpret_cast<const double2*>(a);
        const double2* x2 = reinterpret_cast<const double2*>(x);
        const int n2 = n >> 1;
        for (int base = 0; base < n2; base += 512) {  // n <= 1024: the whole row in one round trip
            double2 av[16], xv[16];
#pragma unroll
            for (int t = 0; t < 16; ++t) {
                const int q = base + lane + 32 * t;
                av[t] = q < n2 ? __ldg(a2 + q) : make_double2(0.0, 0.0);
                xv[t] = q < n2 ? __ldg(x2 + q) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int t = 0; t < 16; ++t) {
                acc0 = fma(av[t].x, xv[t].x, acc0);
                acc1 = fma(av[t].y, xv[t].y, acc1);
            }
        }
    } else {
        for (int j = lane; j < n; j += 32) acc0 = fma(__ldg(a + j), __ldg(x + j), acc0);
    }
    const double v = warp_sum(acc0 + acc1);
    if (lane == 0) y[row] = ACC ? y[row] + v : v;
}

// Same product for n <= GEMV_TMA_MAX (even): one elected thread moves x and
// the block's 8 rows into shared memory with TMA bulk copies on one mbarrier
// (all bytes in flight at once, no per-load issue slots), then each warp
// reduces its row from shared memory.
constexpr int GEMV_TMA_MAX = 2816;  // 9 n doubles of dynamic shared memory <= 198 KB
template <bool ACC>
__global__ void __launch_bounds__(256) k_gemv_tma(const double* __restrict__ A, const double* __restrict__ x,
                                                  double* __restrict__ y, int n) {
    pdl_begin();
    extern __shared__ __align__(128) double gsm[];
    __shared__ __align__(8) unsigned long long bar;
    const int r0 = blockIdx.x * 8, nr = min(8, n - r0);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* xs = gsm;
    double* rows = gsm + n;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        const unsigned rb = (unsigned)n * 8u;
        mbar_expect_tx(&bar, rb * (unsigned)(1 + nr));
        bulk_g2s(xs, x, rb, &bar);
        for (int k = 0; k < nr; ++k) bulk_g2s(rows + (size_t)k * n, A + (size_t)(r0 + k) * n, rb, &bar);
    }
    __syncthreads();  // barrier initialised before anyone waits on it
    mbar_wait(&bar, 0);
    if (w >= nr) return;
    const double2* a2 = reinterpret_cast<const double2*>(rows + (size_t)w * n);
    const double2* x2 = reinterpret_cast<const double2*>(xs);
    double acc0 = 0.0, acc1 = 0.0;
    for (int q = lane; q < (n >> 1); q += 32) {
        const double2 a = a2[q], b = x2[q];
        acc0 = fma(a.x, b.x, acc0);
        acc1 = fma(a.y, b.y, acc1);
    }
    const double v = warp_sum(acc0 + acc1);
    if (lane == 0) y[r0 + w] = ACC ? y[r0 + w] + v : v;
}

// r = b - M x with M in CSR, one thread per row.
__global__ void k_csr_residual(const int* __restrict__ ptr, const int* __restrict__ col, const double* __restrict__ val,
                               const double* __restrict__ x, const double* __restrict__ b, double* __restrict__ r, int n) {
    pdl_begin();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double acc = 0.0;
    for (int z = ptr[i]; z < ptr[i + 1]; ++z) acc += val[z] * x[col[z]];
    r[i] = b[i] - acc;
}

__global__ void k_axpy(double* __restrict__ y, const double* __restrict__ x, int n) {
    pdl_begin();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] += x[i];
}

}  // namespace

namespace {

void gj_pp_run(Ctx& c, double* W0, double* W1, int nb, int ld, int n);

// In-place inverse of W (n x n) by the ping-pong blocked GJ (k_gj_pp).
void block_gj_inplace(Ctx& c, double* W, int n) {
    const int nb = cdiv(n, PPB), ld = nb * PPB;
    c.gj_pp.alloc(std::max(c.gj_pp.n, 2 * (size_t)ld * ld + 2 * PPB * PPB));
    c.gj_piv.alloc(std::max(c.gj_piv.n, (size_t)n + 1));
    CK(cudaMemsetAsync(c.gj_piv.p + n, 0, sizeof(int), c.st));
    double* W0 = c.gj_pp.p;
    double* W1 = W0 + (size_t)ld * ld;
    const int g = std::min(cdiv((long long)ld * ld, TPB), 8 * c.num_sms);
    {
        PROF(c, "k_pad_in");
        launch_k(c, k_pad_in, g, TPB, 0, W, n, W0, ld);
        CK_LAUNCH();
    }
    gj_pp_run(c, W0, W1, nb, ld, n);
    {
        PROF(c, "k_pad_out");
        launch_k(c, k_pad_out, g, TPB, 0, (nb & 1) ? W1 : W0, ld, W, n);
        CK_LAUNCH();
    }
}

// k_gj_pp on the padded pair (W0 holds the matrix; the inverse ends in
// W[nb % 2]).
void gj_pp_run(Ctx& c, double* W0, double* W1, int nb, int ld, int n) {
    static DeviceCache occ;
    int per_sm = occ.at().load();
    if (per_sm < 0) {  // once per device, outside any graph capture
        CK(cudaFuncSetAttribute(k_gj_pp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PP_SMEM));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gj_pp, 256, PP_SMEM));
        occ.at().store(per_sm);
    }
    const int cap = per_sm * c.num_sms;
    if (cap < 2) throw CudaError("dense_inverse: ping-pong Gauss-Jordan does not fit");
    const int nch = cdiv(ld, PPW), cpb = PPW / PPB;  // work item: one block row x PPW columns
    // one worker per item, plus one spare: the worker that shares the lookahead
    // CTA's SM sits out (k_gj_pp), so nb * nch workers stay active
    const int blocks = std::min(nb * nch + 1, cap - 1) + 1;
    static const bool trace = [] {
        const char* e = std::getenv("MPM2P_GJ_TRACE");
        return e && e[0] == '1';
    }();
    DevBuf<unsigned long long> tr;
    if (trace) {
        tr.alloc((size_t)nb * 8);
        tr.zero(c.st);
    }
    c.gj_aux.alloc(2);
    CK(cudaMemsetAsync(c.gj_aux.p, 0xFF, 2 * sizeof(int), c.st));  // aux[1] = -1: no idle worker yet
    PPArgs pa{W0, W1, W1 + (size_t)ld * ld, ld, nb, nch, cpb, c.gj_piv.p + n, c.gj_aux.p, trace ? tr.p : nullptr};
    void* args[] = {&pa};
    {
        PROF(c, "k_gj_pp");
        CK(cudaLaunchCooperativeKernel((void*)k_gj_pp, blocks, 256, args, PP_SMEM, c.st));
        CK_LAUNCH();
    }
    if (trace) {  // developer trace: lookahead load+mul / invert / publish, worker, barrier (us)
        std::vector<unsigned long long> h((size_t)nb * 8);
        CK(cudaMemcpyAsync(h.data(), tr.p, h.size() * 8, cudaMemcpyDeviceToHost, c.st));
        CK(cudaStreamSynchronize(c.st));
        std::fprintf(stderr, "k_gj_pp n=%d nb=%d nch=%d cpb=%d blocks=%d\n", n, nb, nch, cpb, blocks);
        for (int k = 0; k < nb && k < 6; ++k) {
            const unsigned long long* t = h.data() + (size_t)k * 8;
            std::fprintf(stderr,
                         "  step %d: look prep %.2f inv %.2f (%llu cycles) pub %.2f | worker %.2f | step %.2f\n", k,
                         (t[1] - t[0]) * 1e-3, (t[2] - t[1]) * 1e-3, t[4], (t[3] - t[2]) * 1e-3, (t[6] - t[5]) * 1e-3,
                         (t[7] - t[5]) * 1e-3);
        }
    }
}


void launch_rcond(Ctx& c, const double* A, const double* Ainv, int n, double* rcond_dev, unsigned err_bit,
                  double threshold) {
    const int nrb = cdiv(n, 64);
    {
        PROF(c, "k_colsum");
        launch_k(c, k_colsum, dim3(cdiv(n, TPB), nrb), TPB, 0, A, Ainv, n, c.gj_work.p);
        CK_LAUNCH();
    }
    {
        PROF(c, "k_rcond");
        launch_k(c, k_rcond, 1, 1024, 0, c.gj_work.p, n, nrb, c.gj_piv.p + n, rcond_dev, &c.sc.p->err, err_bit,
                                      threshold);
        CK_LAUNCH();
    }
}

}  // namespace

// Public entry for the block-tridiagonal solver (blocktri.cu).
void block_gj_inplace_pub(Ctx& c, double* W, int n) { block_gj_inplace(c, W, n); }

// Interface inverse from the CSR operator (dense path): K = J M built padded
// into the ping-pong buffer, k_gj_pp, then M^-1 and the rcond guard. The
// symmetry of K is checked once per context on the CSR values (host).
bool interface_inverse_csr(Ctx& c, double* rcond_dev, unsigned err_bit, double threshold) {
    const int n = c.dim;
    if (n == 0) return true;
    if (c.iface_sym < 0) {
        std::vector<int> ptr(n + 1), col(c.nnz), tpos(c.nnz);
        std::vector<double> val(c.nnz);
        CK(cudaMemcpyAsync(ptr.data(), c.csr_ptr.p, ptr.size() * sizeof(int), cudaMemcpyDeviceToHost, c.st));
        CK(cudaMemcpyAsync(col.data(), c.csr_col.p, col.size() * sizeof(int), cudaMemcpyDeviceToHost, c.st));
        CK(cudaMemcpyAsync(tpos.data(), c.csr_tpos.p, tpos.size() * sizeof(int), cudaMemcpyDeviceToHost, c.st));
        CK(cudaMemcpyAsync(val.data(), c.csr_val.p, val.size() * sizeof(double), cudaMemcpyDeviceToHost, c.st));
        CK(cudaStreamSynchronize(c.st));
        const int h = n / 2;
        auto kval = [&](int r, int z) { return (r < h ? 1.0 : -1.0) * val[z]; };  // K row r = J-permuted M row
        auto src = [&](int r) { return r < h ? h + r : r - h; };
        // K[i][j] with i = K row: its CSR row is M row src(i); K[j][i] likewise.
        double d = 0.0, m = 0.0;
        std::vector<int> inv(n);
        for (int r = 0; r < n; ++r) inv[src(r)] = r;  // M row -> K row
        for (int mr = 0; mr < n; ++mr) {
            const int kr = inv[mr];
            for (int z = ptr[mr]; z < ptr[mr + 1]; ++z) {
                const int kc = col[z];  // K[kr][kc] = kval(kr, z); K[kc][kr] lives in M row src(kc)
                const int mr2 = src(kc);
                double other = 0.0;
                for (int z2 = ptr[mr2]; z2 < ptr[mr2 + 1]; ++z2)
                    if (col[z2] == kr) other = kval(kc, z2);
                d = std::max(d, std::fabs(kval(kr, z) - other));
                m = std::max(m, std::fabs(kval(kr, z)));
            }
        }
        c.iface_sym = (m > 0.0 && d <= 1e-12 * m) ? 1 : 0;
    }
    if (c.iface_sym != 1) return false;  // caller takes the pivoted dense path
    const int nb = cdiv(n, PPB), ld = nb * PPB;
    c.gj_pp.alloc(std::max(c.gj_pp.n, 2 * (size_t)ld * ld + 2 * PPB * PPB));
    c.gj_piv.alloc(std::max(c.gj_piv.n, (size_t)n + 1));
    CK(cudaMemsetAsync(c.gj_piv.p + n, 0, sizeof(int), c.st));
    double* W0 = c.gj_pp.p;
    double* W1 = W0 + (size_t)ld * ld;
    {
        PROF(c, "k_build_k");
        launch_k(c, k_build_k, cdiv((long long)ld * 32, TPB), TPB, 0, c.csr_ptr, c.csr_col, c.csr_val, n, W0, ld);
        CK_LAUNCH();
    }
    gj_pp_run(c, W0, W1, nb, ld, n);
    const int nrb = cdiv(n, 64);
    c.gj_work.alloc(std::max(c.gj_work.n, (size_t)2 * n * nrb));
    {
        PROF(c, "k_kinv_out");
        launch_k(c, k_kinv_out, dim3(cdiv(n, 32), nrb), 256, 0, (nb & 1) ? W1 : W0, ld, n, c.Minv, c.gj_work.p);
        CK_LAUNCH();
    }
    {
        PROF(c, "k_mnorm");
        launch_k(c, k_mnorm, cdiv(n, TPB), TPB, 0, c.csr_ptr, c.csr_tpos, c.csr_val, n, c.gj_work.p);
        CK_LAUNCH();
    }
    {
        PROF(c, "k_rcond");
        launch_k(c, k_rcond, 1, 1024, 0, c.gj_work.p, n, nrb, c.gj_piv.p + n, rcond_dev, &c.sc.p->err, err_bit,
                                      threshold);
        CK_LAUNCH();
    }
    return true;
}

// Interface matrix inverse: pivot-free blocked GJ on K = J M when K is
// symmetric (checked once per context; the formulation makes it so), else the
// pivoted panel GJ on M.
void interface_inverse_async(Ctx& c, const double* M, double* Minv, int n, double* rcond_dev, unsigned err_bit,
                             double threshold) {
    if (n == 0) return;
    c.gj_work.alloc(std::max(c.gj_work.n, (size_t)2 * n * n));
    c.gj_piv.alloc(std::max(c.gj_piv.n, (size_t)n + 1));
    {
        PROF(c, "k_j_times");
        launch_k(c, k_j_times, std::min(cdiv((long long)n * n, TPB), 8 * c.num_sms), TPB, 0, M, c.gj_work, n);
        CK_LAUNCH();
    }
    if (c.iface_sym < 0) {
        const int g = std::min(cdiv((long long)n * n, TPB), 2 * c.num_sms);
        DevBuf<double> part;
        part.alloc(2 * g);
        launch_k(c, k_asym, g, TPB, 0, c.gj_work, n, part);
        CK_LAUNCH();
        std::vector<double> h(2 * g);
        CK(cudaMemcpyAsync(h.data(), part.p, h.size() * sizeof(double), cudaMemcpyDeviceToHost, c.st));
        CK(cudaStreamSynchronize(c.st));
        double d = 0.0, m = 0.0;
        for (int b = 0; b < g; ++b) {
            d = std::max(d, h[2 * b]);
            m = std::max(m, h[2 * b + 1]);
        }
        c.iface_sym = (m > 0.0 && d <= 1e-12 * m) ? 1 : 0;
    }
    if (c.iface_sym == 1) {
        block_gj_inplace(c, c.gj_work, n);
        {
            PROF(c, "k_times_j");
            launch_k(c, k_times_j, std::min(cdiv((long long)n * n, TPB), 8 * c.num_sms), TPB, 0, c.gj_work, Minv, n);
            CK_LAUNCH();
        }
        launch_rcond(c, M, Minv, n, rcond_dev, err_bit, threshold);
    } else {
        dense_inverse_async(c, M, Minv, n, rcond_dev, err_bit, threshold);
    }
}

// SPD inverse (the static repair Laplacian): pivot-free blocked GJ.
double spd_inverse(Ctx& c, const double* A, double* Ainv, int n) {
    if (n == 0) return 1.0;
    c.gj_work.alloc(std::max(c.gj_work.n, (size_t)2 * n * n));
    c.gj_piv.alloc(std::max(c.gj_piv.n, (size_t)n + 1));
    CK(cudaMemcpyAsync(Ainv, A, (size_t)n * n * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
    block_gj_inplace(c, Ainv, n);
    launch_rcond(c, A, Ainv, n, &c.sc.p->rcond, 0u, 0.0);
    double rc = 0.0;
    CK(cudaMemcpyAsync(&rc, &c.sc.p->rcond, sizeof(double), cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
    return rc;
}

void dense_inverse_async(Ctx& c, const double* A, double* Ainv, int n, double* rcond_dev, unsigned err_bit,
                         double threshold) {
    if (n == 0) return;
    int b = 16;
    const size_t smem_cap = 180 * 1024;
    while (b > 2 && (size_t)n * b * sizeof(double) > smem_cap) b /= 2;
    if ((size_t)n * b * sizeof(double) > smem_cap)
        throw CapacityError("dense_inverse: interface system of dimension " + std::to_string(n) +
                            " is too large for the dense path");
    // panel (CTA 0, phase 1) or the 64x16 + 16x128 GEMM tiles (phase 3)
    const size_t smem = std::max<size_t>((size_t)n * b, 64 * 16 + 16 * 128) * sizeof(double);
    CK(cudaFuncSetAttribute(k_gauss_jordan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cap));
    c.gj_work.alloc(std::max(c.gj_work.n, (size_t)2 * n * n));
    c.gj_col.alloc(std::max(c.gj_col.n, (size_t)n * b));   // G
    c.gj_row.alloc(std::max(c.gj_row.n, (size_t)b * 2 * n));  // Rb
    c.gj_piv.alloc(std::max(c.gj_piv.n, (size_t)n + 1));    // swaps + singular flag
    {
        PROF(c, "k_augment");
        launch_k(c, k_augment, std::min(cdiv(2LL * n * n, TPB), 8 * c.num_sms), TPB, 0, A, c.gj_work, n);
        CK_LAUNCH();
    }
    CK(cudaMemsetAsync(c.gj_piv.p + n, 0, sizeof(int), c.st));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gauss_jordan, GJ_THREADS, smem));
    if (per_sm < 1) throw CudaError("dense_inverse: cooperative kernel does not fit on an SM");
    const int blocks = c.num_sms;  // one CTA per SM
    GJArgs ga{c.gj_work.p, n, b, c.gj_col.p, c.gj_piv.p, c.gj_row.p, c.gj_piv.p + n};
    void* args[] = {&ga};
    {
        PROF(c, "k_gauss_jordan");
        CK(cudaLaunchCooperativeKernel((void*)k_gauss_jordan, blocks, GJ_THREADS, args, smem, c.st));
        CK_LAUNCH();
    }
    {
        PROF(c, "k_extract");
        launch_k(c, k_extract, std::min(cdiv((long long)n * n, TPB), 8 * c.num_sms), TPB, 0, c.gj_work, Ainv, n);
        CK_LAUNCH();
    }
    const int nrb = cdiv(n, 64);
    {
        PROF(c, "k_colsum");
        launch_k(c, k_colsum, dim3(cdiv(n, TPB), nrb), TPB, 0, A, Ainv, n, c.gj_work.p);  // W is free now
        CK_LAUNCH();
    }
    {
        PROF(c, "k_rcond");
        launch_k(c, k_rcond, 1, 1024, 0, c.gj_work.p, n, nrb, c.gj_piv.p + n, rcond_dev, &c.sc.p->err, err_bit,
                                      threshold);
        CK_LAUNCH();
    }
}

double dense_inverse(Ctx& c, const double* A, double* Ainv, int n) {
    if (n == 0) return 1.0;
    dense_inverse_async(c, A, Ainv, n, &c.sc.p->rcond, 0u, 0.0);
    double rc = 0.0;
    CK(cudaMemcpyAsync(&rc, &c.sc.p->rcond, sizeof(double), cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
    return rc;
}

template <bool ACC>
void gemv_dispatch(Ctx& c, const double* A, const double* x, double* y, int n) {
    PROF(c, "k_gemv");
    if ((n & 1) == 0 && n <= GEMV_TMA_MAX) {
        static DeviceCache attr;  // once per device, outside any graph capture (first use is eager)
        if (attr.at().load() < 0) {
            CK(cudaFuncSetAttribute(k_gemv_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    9 * GEMV_TMA_MAX * (int)sizeof(double)));
            CK(cudaFuncSetAttribute(k_gemv_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    9 * GEMV_TMA_MAX * (int)sizeof(double)));
            attr.at().store(1);
        }
        launch_k(c, k_gemv_tma<ACC>, cdiv(n, 8), 256, (size_t)9 * n * sizeof(double), A, x, y, n);
    } else {
        launch_k(c, k_gemv_w<ACC>, cdiv(n, 8), 256, 0, A, x, y, n);
    }
    CK_LAUNCH();
}

void launch_gemv(Ctx& c, const double* A, const double* x, double* y, int n) { gemv_dispatch<false>(c, A, x, y, n); }
void launch_gemv_acc(Ctx& c, const double* A, const double* x, double* y, int n) {
    gemv_dispatch<true>(c, A, x, y, n);
}

void launch_csr_residual(Ctx& c, const int* ptr, const int* col, const double* val, const double* x, const double* b,
                         double* r, int n) {
    PROF(c, "k_csr_residual");
    launch_k(c, k_csr_residual, cdiv(n, TPB), TPB, 0, ptr, col, val, x, b, r, n);
    CK_LAUNCH();
}

void launch_axpy(Ctx& c, double* y, const double* x, int n) {
    PROF(c, "k_axpy");
    launch_k(c, k_axpy, cdiv(n, TPB), TPB, 0, y, x, n);
    CK_LAUNCH();
}

}  // namespace mpm2p
