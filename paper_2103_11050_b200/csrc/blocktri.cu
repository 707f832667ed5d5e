// blocktri.cu — K7b: direct block-tridiagonal interface solve for systems
// above the dense limit (C5: dim 65,024; the reference's dense PartialPivLU
// there would be 34 GB, proj/src/mrcm.cpp:198,226,264).
//
// Ordered by subdomain row (the vertical interfaces of row j and the
// horizontal interfaces between rows j and j+1 form block j), K = J M is
// block tridiagonal: an interface only couples to interfaces that share a
// subdomain with it. K is symmetric quasi-definite: every
// principal submatrix and Schur complement is factorable without pivoting.
//
// Block cyclic reduction (odd-even), all blocks padded to one size S (a
// multiple of 64; the pad is an identity block):
//   level l works on the blocks j = 0 (mod 2^l); at every level the odd
//   members o are eliminated and the even members e keep a block-tridiagonal
//   system of half the size:
//     Dinv_o = D_o^-1, P_o = Dinv_o Lo_o, Q_o = Dinv_o Up_o
//     D_e <- D_e - Lo_e Q_{o-} - Up_e P_{o+}
//     Lo_e <- -Lo_e P_{o-},  Up_e <- -Up_e Q_{o+}
//   until one block is left (Dinv_0). A solve is then
//     forward,  per level: c_o = Dinv_o y_o;  y_e -= Lo_e c_{o-} + Up_e c_{o+}
//     top:      x_0 = Dinv_0 y_0
//     backward, per level: x_o = c_o - P_o x_{o-} - Q_o x_{o+}
// i.e. 2 log2(nb) + 1 dependent batched GEMV launches (C5: 15) instead of the
// 2 nb - 1 block steps of a sequential block LDL^T (255), each launch
// streaming a whole level's matrices. The factorization is per level one
// batched Gauss-Jordan inversion (one launch pair per 32-column panel for all
// of the level's blocks) and batched GEMMs on the fp64 tensor cores
// (mma.sync.m8n8k4, DMMA).

#include "context.cuh"
#include "cr.cuh"


namespace mpm2p {

namespace {

constexpr int TPB = 256;

__device__ __forceinline__ void cr_dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// One batched GEMM job: C = C0 + a1 A1 B1 (+ a2 A2 B2), all S x S row-major
// (C may alias C0).
struct GemmJob {
    double* C;
    const double* C0;
    const double* A1;
    const double* B1;
    const double* A2;
    const double* B2;
    double a1, a2;
};

// 64 x 64 output tile per CTA (4 warps, 32 x 32 each = 4 x 4 DMMA tiles),
// k-slabs of 16 staged in shared memory (padded rows: conflict-free fragment
// loads), the next slab loaded into registers while the current one is used.
constexpr int GT = 64, GK = 16, LDA = GK + 4, LDB = GT + 4;
__global__ void __launch_bounds__(128) k_cr_gemm(const GemmJob* __restrict__ jobs, int S) {
    __shared__ double As[GT * LDA], Bs[GK * LDB];
    const GemmJob jb = jobs[blockIdx.z];
    const int tiles = S / GT;
    const int i0 = (blockIdx.x / tiles) * GT, j0 = (blockIdx.x % tiles) * GT;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wr = (w >> 1) * 32, wc = (w & 1) * 32;
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    for (int term = 0; term < 2; ++term) {
        const double* A = term ? jb.A2 : jb.A1;
        const double* B = term ? jb.B2 : jb.B1;
        if (!A) continue;
        const double alpha = term ? jb.a2 : jb.a1;
        double ra[8], rb[8];
        auto fetch = [&](int k0) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int x = threadIdx.x + 128 * q;           // 0..1023
                ra[q] = A[(size_t)(i0 + (x >> 4)) * S + k0 + (x & 15)];  // 64 x 16
                rb[q] = B[(size_t)(k0 + (x >> 6)) * S + j0 + (x & 63)];  // 16 x 64
            }
        };
        fetch(0);
        for (int k0 = 0; k0 < S; k0 += GK) {
            __syncthreads();
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int x = threadIdx.x + 128 * q;
                As[(x >> 4) * LDA + (x & 15)] = alpha * ra[q];
                Bs[(x >> 6) * LDB + (x & 63)] = rb[q];
            }
            __syncthreads();
            if (k0 + GK < S) fetch(k0 + GK);
#pragma unroll
            for (int kk = 0; kk < GK; kk += 4) {
                double af[4], bf[4];
#pragma unroll
                for (int a = 0; a < 4; ++a) af[a] = As[(wr + a * 8 + (lane >> 2)) * LDA + kk + (lane & 3)];
#pragma unroll
                for (int b = 0; b < 4; ++b) bf[b] = Bs[(kk + (lane & 3)) * LDB + wc + b * 8 + (lane >> 2)];
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) cr_dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
            }
        }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int r = i0 + wr + a * 8 + (lane >> 2), col = j0 + wc + b * 8 + 2 * (lane & 3);
            const size_t o = (size_t)r * S + col;
            double v0 = acc[a][b][0], v1 = acc[a][b][1];
            if (jb.C0) {
                v0 += jb.C0[o];
                v1 += jb.C0[o + 1];
            }
            jb.C[o] = v0;
            jb.C[o + 1] = v1;
        }
}

// ---- batched Gauss-Jordan inversion without pivoting (in place), one
// launch pair per 32-column panel k for all matrices of the batch:
//   k_gj_pivot: per matrix, save the panel column W[:, k] (S x 32), invert
//               the pivot block (one warp per row, pivot by pivot) and form
//               R = P W[k, :] (the new row panel)
//   k_gj_update: W[i, j] -= C_i R_j (i outside the panel), W[k, :] = R,
//               W[i, k] = -C_i P
constexpr int GP = 32;
// grid (S / 32 column tiles, batch): every CTA inverts the 32 x 32 pivot block
// in shared memory (redundantly, it is small), forms its 32 x 32 tile of R and
// saves its 32 rows of the panel column
__global__ void __launch_bounds__(256) k_gj_pivot(double* const* __restrict__ mats, int S, int k0,
                                                  double* __restrict__ colbuf, double* __restrict__ rowbuf,
                                                  int* __restrict__ flag) {
    pdl_begin();
    __shared__ double Pv[GP][GP + 1];
    __shared__ double Wk[GP][GP + 1];
    double* W = mats[blockIdx.y];
    double* Cb = colbuf + (size_t)blockIdx.y * S * GP;
    double* Rb = rowbuf + (size_t)blockIdx.y * S * GP;
    const int j0 = blockIdx.x * GP;
    for (int x = threadIdx.x; x < GP * GP; x += blockDim.x) {
        const int r = x / GP, q = x % GP;
        Pv[r][q] = W[(size_t)(k0 + r) * S + k0 + q];
        Wk[r][q] = W[(size_t)(k0 + r) * S + j0 + q];  // this CTA's tile of the pivot rows
        Cb[(size_t)(j0 + r) * GP + q] = W[(size_t)(j0 + r) * S + k0 + q];  // rows j0.. of the panel column
    }
    __syncthreads();
    // Gauss-Jordan of the pivot block in place (no pivoting): thread (r, q-group)
    const int r = threadIdx.x >> 3, qg = (threadIdx.x & 7) * 4;
    for (int p = 0; p < GP; ++p) {
        const double d = Pv[p][p];
        const double inv = 1.0 / d;
        const double f = Pv[r][p];
        double rp[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) rp[t] = Pv[p][qg + t];
        __syncthreads();
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int q = qg + t;
            if (r == p) Pv[r][q] = q == p ? inv : rp[t] * inv;
            else Pv[r][q] = q == p ? -f * inv : Pv[r][q] - f * rp[t] * inv;
        }
        __syncthreads();
        if (threadIdx.x == 0 && blockIdx.x == 0 && (!(d != 0.0) || !isfinite(d))) atomicOr(flag, 1);
    }
    // R tile = P W[k, j0..j0+31]; the panel's own tile is P itself
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const int q = qg + t;
        double v;
        if (j0 == k0) {
            v = Pv[r][q];
        } else {
            v = 0.0;
#pragma unroll 8
            for (int u = 0; u < GP; ++u) v = fma(Pv[r][u], Wk[u][q], v);
        }
        Rb[(size_t)r * S + j0 + q] = v;
    }
}

// tiles of 32 rows x 64 columns; C_i = saved panel rows, R = new row panel
__global__ void __launch_bounds__(256) k_gj_update(double* const* __restrict__ mats, int S, int k0,
                                                   const double* __restrict__ colbuf, const double* __restrict__ rowbuf) {
    __shared__ double Cs[GP][GP + 1];
    __shared__ double Rs[GP][64 + 1];
    double* W = mats[blockIdx.z];
    const double* Cb = colbuf + (size_t)blockIdx.z * S * GP;
    const double* Rb = rowbuf + (size_t)blockIdx.z * S * GP;
    const int i0 = blockIdx.y * GP, j0 = blockIdx.x * 64;
    for (int x = threadIdx.x; x < GP * GP; x += blockDim.x) Cs[x / GP][x % GP] = Cb[(size_t)(i0 + x / GP) * GP + x % GP];
    for (int x = threadIdx.x; x < GP * 64; x += blockDim.x) Rs[x / 64][x % 64] = Rb[(size_t)(x / 64) * S + j0 + x % 64];
    __syncthreads();
    const bool pivot_rows = i0 == k0;
    for (int x = threadIdx.x; x < GP * 64; x += blockDim.x) {
        const int r = x / 64, cc = x % 64, col = j0 + cc;
        const size_t o = (size_t)(i0 + r) * S + col;
        if (pivot_rows) {
            W[o] = Rs[r][cc];
        } else if (col >= k0 && col < k0 + GP) {
            // -C_i P: R's panel columns hold P
            double v = 0.0;
            for (int q = 0; q < GP; ++q) v += Cs[r][q] * Rs[q][cc];
            W[o] = -v;
        } else {
            double v = W[o];
            for (int q = 0; q < GP; ++q) v -= Cs[r][q] * Rs[q][cc];
            W[o] = v;
        }
    }
}

// ---- batched GEMV jobs: out = base + s1 M1 v1 (+ s2 M2 v2), S x S matrices
// RPW rows per warp, 8 warps per CTA (the rows' loads interleaved); the
// launcher picks RPW = 4 for wide levels and RPW = 1 for the last levels of
// the reduction, where few blocks remain and more warps per row set hide
// the load latency
template <int RPW>
__global__ void __launch_bounds__(256) k_cr_gemv(const GemvJob* __restrict__ jobs, int S) {
    pdl_begin();
    extern __shared__ double vs[];  // 2 S
    const GemvJob jb = jobs[blockIdx.y];
    for (int x = threadIdx.x; x < S; x += blockDim.x) {
        vs[x] = jb.v1 ? jb.v1[x] : 0.0;
        vs[S + x] = jb.v2 ? jb.v2[x] : 0.0;
    }
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r0 = (blockIdx.x * 8 + w) * RPW;
    double a[RPW];
#pragma unroll
    for (int q = 0; q < RPW; ++q) a[q] = 0.0;
    for (int term = 0; term < 2; ++term) {
        const double* M = term ? jb.M2 : jb.M1;
        if (!M) continue;
        const double s = term ? jb.s2 : jb.s1;
        const double* v = vs + term * S;
        double t[RPW];
#pragma unroll
        for (int q = 0; q < RPW; ++q) t[q] = 0.0;
        // S is a multiple of 64; several column slabs in flight per round
        // trip (the narrow levels are a handful of dependent round trips)
#pragma unroll(RPW == 1 ? 8 : 2)
        for (int c = lane; c < S; c += 64) {
            double m[RPW][2];
#pragma unroll
            for (int q = 0; q < RPW; ++q) {
                m[q][0] = __ldg(M + (size_t)(r0 + q) * S + c);
                m[q][1] = __ldg(M + (size_t)(r0 + q) * S + c + 32);
            }
            const double v0 = v[c], v1 = v[c + 32];
#pragma unroll
            for (int q = 0; q < RPW; ++q) t[q] = fma(m[q][1], v1, fma(m[q][0], v0, t[q]));
        }
#pragma unroll
        for (int q = 0; q < RPW; ++q) a[q] += s * warp_sum(t[q]);
    }
    if (lane == 0)  // warp_sum leaves the total in lane 0
#pragma unroll
        for (int q = 0; q < RPW; ++q) jb.out[r0 + q] = (jb.base ? jb.base[r0 + q] : 0.0) + a[q];
}

// D_j (padded, identity on the pad) and Up_j = K[block j, block j+1] from the CSR of K
__global__ void k_cr_scatter(const int* __restrict__ kptr, const int* __restrict__ kcol, const double* __restrict__ kval,
                             int n, const int* __restrict__ blk, const int* __restrict__ loc, int S,
                             double* __restrict__ D, double* __restrict__ Up) {
    pdl_begin();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int j = blk[r], lr = loc[r];
    for (int z = kptr[r]; z < kptr[r + 1]; ++z) {
        const int c = kcol[z], jc = blk[c], lc = loc[c];
        if (jc == j) D[((size_t)j * S + lr) * S + lc] = kval[z];
        else if (jc == j + 1) Up[((size_t)j * S + lr) * S + lc] = kval[z];
    }
}
__global__ void k_cr_pad(const int* __restrict__ bsz, int nb, int S, double* __restrict__ D) {
    const long long n = (long long)nb * S;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < n; x += (long long)gridDim.x * blockDim.x) {
        const int j = (int)(x / S), r = (int)(x % S);
        if (r >= bsz[j]) D[((size_t)j * S + r) * S + r] = 1.0;
    }
}
// Lo_{j+1} = Up_j^T (batched 32 x 32 tile transposes)
__global__ void k_cr_transpose(double* const* __restrict__ dst, const double* const* __restrict__ src, int S) {
    __shared__ double t[32][33];
    const double* in = src[blockIdx.z];
    double* out = dst[blockIdx.z];
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    for (int y = threadIdx.y; y < 32; y += blockDim.y) t[y][threadIdx.x] = in[(size_t)(by + y) * S + bx + threadIdx.x];
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += blockDim.y) out[(size_t)(bx + y) * S + by + threadIdx.x] = t[threadIdx.x][y];
}

__global__ void k_flag_err(const int* flag, Scalars* sc, unsigned bit) {
    if (*flag) atomicOr(&sc->err, bit);
}

// y (padded block order) <- J rhs (transposed = 0) or rhs (1)
__global__ void k_bt_gather(const double* __restrict__ rhs, int n, const int* __restrict__ blk,
                            const int* __restrict__ loc, int S, double* __restrict__ y, int transposed) {
    pdl_begin();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int h = n / 2;
    const double v = transposed ? rhs[r] : (r < h ? rhs[h + r] : -rhs[r - h]);
    y[(size_t)blk[r] * S + loc[r]] = v;
}

// (transposed = 0) x = xb, (1) x = J^T xb, from padded block order
__global__ void k_bt_unpermute(const double* __restrict__ xb, int n, const int* __restrict__ blk,
                               const int* __restrict__ loc, int S, double* __restrict__ x, int transposed) {
    pdl_begin();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int h = n / 2;
    if (!transposed) {
        x[r] = xb[(size_t)blk[r] * S + loc[r]];
    } else {  // (J^T w)_i = -w_{i+h} (i < h), w_{i-h} (i >= h)
        const int q = r < h ? r + h : r - h;
        const double w = xb[(size_t)blk[q] * S + loc[q]];
        x[r] = r < h ? -w : w;
    }
}

// ---- 1-norm condition estimate of the interface matrix M (the reference's
// rcond() guard, mrcm.cpp:227-238; Hager 1984 / Higham 1988 as the oracle's
// hager_rcond): at most five rounds of y = M^-1 x, xi = sign(y),
// z = M^-T xi, x = e_argmax|z|. Every round's kernels are always launched
// (graph-capturable); a device flag freezes the state once the estimate has
// converged. M^-T v = J^T K^-1 v (K = J M symmetric).
struct HagerState {
    double est, anorm;
    int done;
};

// ||M||_1 = max column sum of |M|: column j's entries are row j's transposed
// positions (the CSR pattern is structurally symmetric)
__global__ void __launch_bounds__(1024) k_hager_init(const int* __restrict__ ptr, const int* __restrict__ tpos,
                                                     const double* __restrict__ val, int n, double* __restrict__ x,
                                                     HagerState* st) {
    __shared__ double sh[32];
    double m = 0.0;
    for (int jc = threadIdx.x; jc < n; jc += blockDim.x) {
        double s = 0.0;
        for (int z = ptr[jc]; z < ptr[jc + 1]; ++z) s += fabs(val[tpos[z]]);
        m = fmax(m, s);
        x[jc] = 1.0 / n;
    }
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
        m = warp_max(m);
        if (threadIdx.x == 0) {
            st->anorm = m;
            st->est = 0.0;
            st->done = 0;
        }
    }
}

// round `it`, after y = M^-1 x: ny = ||y||_1; stop if it does not grow; else xi = sign(y)
__global__ void __launch_bounds__(1024) k_hager_a(const double* __restrict__ y, int n, int it,
                                                  double* __restrict__ xi, HagerState* st) {
    __shared__ double sh[32];
    __shared__ int stop;
    if (st->done) return;
    double a = 0.0;
    for (int r = threadIdx.x; r < n; r += blockDim.x) a += fabs(y[r]);
    a = warp_sum(a);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
        double ny = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) ny += sh[w];
        int sp = 0;
        if (!isfinite(ny)) {
            st->est = 0.0;
            sp = 1;
        } else if (it > 0 && ny <= st->est) {
            sp = 1;
        } else {
            st->est = ny;
        }
        st->done = sp;
        stop = sp;
    }
    __syncthreads();
    if (stop) return;
    for (int r = threadIdx.x; r < n; r += blockDim.x) xi[r] = y[r] >= 0.0 ? 1.0 : -1.0;
}

// after z = M^-T xi: j = first argmax |z|; stop if |z_j| <= z.x; else x = e_j
__global__ void __launch_bounds__(1024) k_hager_b(const double* __restrict__ z, int n, double* __restrict__ x,
                                                  HagerState* st) {
    __shared__ double shv[32], shz[32];
    __shared__ int shi[32];
    __shared__ int stop, jbest;
    if (st->done) return;
    double zm = -1.0, ztx = 0.0;
    int jm = 0x7fffffff;
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
        const double a = fabs(z[r]);
        ztx += z[r] * x[r];
        if (a > zm) {
            zm = a;
            jm = r;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_down_sync(0xffffffffu, zm, o);
        const int j2 = __shfl_down_sync(0xffffffffu, jm, o);
        if (v2 > zm || (v2 == zm && j2 < jm)) {
            zm = v2;
            jm = j2;
        }
        ztx += __shfl_down_sync(0xffffffffu, ztx, o);
    }
    if ((threadIdx.x & 31) == 0) {
        shv[threadIdx.x >> 5] = zm;
        shi[threadIdx.x >> 5] = jm;
        shz[threadIdx.x >> 5] = ztx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double bv = -1.0, t = 0.0;
        int bj = 0x7fffffff;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            if (shv[w] > bv || (shv[w] == bv && shi[w] < bj)) {
                bv = shv[w];
                bj = shi[w];
            }
            t += shz[w];
        }
        const int sp = bv <= t;
        st->done = sp;
        stop = sp;
        jbest = bj;
    }
    __syncthreads();
    if (stop) return;
    for (int r = threadIdx.x; r < n; r += blockDim.x) x[r] = r == jbest ? 1.0 : 0.0;
}

// rcond = 1 / (||M||_1 est); the reference's guard rcond > 1e-14
__global__ void k_hager_fin(HagerState* st, Scalars* sc, double threshold, unsigned bit) {
    const double est = st->est, an = st->anorm;
    const double rc = (est > 0.0 && an > 0.0) ? 1.0 / an / est : 0.0;
    sc->rcond = rc;
    if (!(rc > threshold)) atomicOr(&sc->err, bit);
}

// The factorization / solve plan, built once from the block layout: device
// job arrays and the host launch sequence.
struct CrLaunch {
    int kind;  // 0 gemm, 1 gj (pivot+update pair over all panels), 2 gemv
    int first, count;  // job range (gemm / gemv jobs) or matrix-pointer range (gj)
};
struct CrPlan {
    int S = 0, nb = 0, max_batch = 1;
    DevBuf<GemmJob> gemm;
    DevBuf<GemvJob> gemv;
    DevBuf<int2> phases;  // the solve's launches as (first job, count), for in-kernel solves
    DevBuf<double*> gjmats;
    DevBuf<double*> tr_dst;
    DevBuf<const double*> tr_src;
    std::vector<CrLaunch> factor, solve;
    DevBuf<double> D, LU, P, Q, cvec, colbuf, rowbuf;
    DevBuf<int> flag;
    std::vector<long long> lu_first;  // first LU slot of each level: Lo slots p, then Up slots m_l + p
};

CrPlan& plan_of(Ctx& c) { return *static_cast<CrPlan*>(c.cr_plan.get()); }

void run_gj(Ctx& c, CrPlan& pl, int first, int count) {
    for (int k0 = 0; k0 < pl.S; k0 += GP) {
        {
            PROF(c, "k_gj_pivot");
            launch_k(c, k_gj_pivot, dim3(pl.S / GP, count), 256, 0, (double* const*)(pl.gjmats.p + first), pl.S, k0,
                     pl.colbuf.p, pl.rowbuf.p, pl.flag.p);
            CK_LAUNCH();
        }
        {
            PROF(c, "k_gj_update");
            launch_k(c, k_gj_update, dim3(pl.S / 64, pl.S / GP, count), 256, 0, (double* const*)(pl.gjmats.p + first),
                     pl.S, k0, (const double*)pl.colbuf.p, (const double*)pl.rowbuf.p);
            CK_LAUNCH();
        }
    }
}

}  // namespace

// A cyclic-reduction system of nb blocks of S x S (S a multiple of 64): its
// level buffers, the factor's launch plan and the solve's job lists, which
// read y and write x (nb * S each, caller-owned; y is overwritten).
std::shared_ptr<void> cr_create(Ctx& c, int nblk, int S, double* yvec, double* xvec) {
    auto plp = std::make_shared<CrPlan>();
    CrPlan& pl = *plp;
    pl.S = S;
    pl.nb = nblk;
    const size_t SS = (size_t)S * S;
    // active block lists per level
    std::vector<std::vector<int>> act(1);
    for (int j = 0; j < nblk; ++j) act[0].push_back(j);
    while (act.back().size() > 1) {
        std::vector<int> nx;
        for (size_t p = 0; p < act.back().size(); p += 2) nx.push_back(act.back()[p]);
        act.push_back(nx);
    }
    const int levels = (int)act.size() - 1;  // levels with an elimination
    long long slots = 0;
    for (int l = 0; l <= levels; ++l) {
        pl.lu_first.push_back(slots);
        slots += 2 * (long long)act[l].size();
    }
    pl.D.alloc(nblk * SS);
    pl.LU.alloc(std::max<long long>(slots, 1) * SS);
    pl.P.alloc(nblk * SS);
    pl.Q.alloc(nblk * SS);
    pl.cvec.alloc((size_t)nblk * S);
    auto Dp = [&](int j) { return pl.D.p + j * SS; };
    auto Lo = [&](int l, int p) { return pl.LU.p + (pl.lu_first[l] + p) * SS; };
    auto Up = [&](int l, int p) { return pl.LU.p + (pl.lu_first[l] + (long long)act[l].size() + p) * SS; };
    auto Pp = [&](int j) { return pl.P.p + j * SS; };
    auto Qp = [&](int j) { return pl.Q.p + j * SS; };
    auto yv = [&](int j) { return yvec + (size_t)j * S; };
    auto xv = [&](int j) { return xvec + (size_t)j * S; };
    auto cv = [&](int j) { return pl.cvec.p + (size_t)j * S; };
    std::vector<GemmJob> gemm;
    std::vector<GemvJob> gemv;
    std::vector<double*> gjm;
    auto gj = [&](const std::vector<double*>& mats) {
        pl.factor.push_back({1, (int)gjm.size(), (int)mats.size()});
        gjm.insert(gjm.end(), mats.begin(), mats.end());
        pl.max_batch = std::max(pl.max_batch, (int)mats.size());
    };
    auto gemm_launch = [&](const std::vector<GemmJob>& jobs) {
        if (jobs.empty()) return;
        pl.factor.push_back({0, (int)gemm.size(), (int)jobs.size()});
        gemm.insert(gemm.end(), jobs.begin(), jobs.end());
    };
    auto gemv_launch = [&](const std::vector<GemvJob>& jobs) {
        if (jobs.empty()) return;
        pl.solve.push_back({2, (int)gemv.size(), (int)jobs.size()});
        gemv.insert(gemv.end(), jobs.begin(), jobs.end());
    };
    // factorization (levels), then the solve's launches in order
    for (int l = 0; l < levels; ++l) {
        const std::vector<int>& A = act[l];
        const int m = (int)A.size();
        std::vector<double*> odd;
        for (int p = 1; p < m; p += 2) odd.push_back(Dp(A[p]));
        gj(odd);  // Dinv_o in place of D_o
        std::vector<GemmJob> pq, ev;
        for (int p = 1; p < m; p += 2) {
            const int o = A[p];
            pq.push_back({Pp(o), nullptr, Dp(o), Lo(l, p), nullptr, nullptr, 1.0, 0.0});
            if (p + 1 < m) pq.push_back({Qp(o), nullptr, Dp(o), Up(l, p), nullptr, nullptr, 1.0, 0.0});
        }
        gemm_launch(pq);
        for (int p = 0; p < m; p += 2) {
            const int e = A[p];
            const bool lo = p >= 1, hi = p + 1 < m;
            GemmJob d{Dp(e), Dp(e), nullptr, nullptr, nullptr, nullptr, -1.0, -1.0};
            if (lo) d.A1 = Lo(l, p), d.B1 = Qp(A[p - 1]);
            if (hi) {
                if (!d.A1) d.A1 = Up(l, p), d.B1 = Pp(A[p + 1]);
                else d.A2 = Up(l, p), d.B2 = Pp(A[p + 1]);
            }
            if (d.A1) ev.push_back(d);
            if (p >= 2) ev.push_back({Lo(l + 1, p / 2), nullptr, Lo(l, p), Pp(A[p - 1]), nullptr, nullptr, -1.0, 0.0});
            if (p + 2 < m) ev.push_back({Up(l + 1, p / 2), nullptr, Up(l, p), Qp(A[p + 1]), nullptr, nullptr, -1.0, 0.0});
        }
        gemm_launch(ev);
        // solve, forward half of level l: c_o = Dinv_o y_o, then the evens
        std::vector<GemvJob> fo, fe;
        for (int p = 1; p < m; p += 2) fo.push_back({cv(A[p]), nullptr, Dp(A[p]), yv(A[p]), nullptr, nullptr, 1.0, 0.0});
        for (int p = 0; p < m; p += 2) {
            GemvJob j{yv(A[p]), yv(A[p]), nullptr, nullptr, nullptr, nullptr, -1.0, -1.0};
            if (p >= 1) j.M1 = Lo(l, p), j.v1 = cv(A[p - 1]);
            if (p + 1 < m) {
                if (!j.M1) j.M1 = Up(l, p), j.v1 = cv(A[p + 1]);
                else j.M2 = Up(l, p), j.v2 = cv(A[p + 1]);
            }
            fe.push_back(j);
        }
        gemv_launch(fo);
        gemv_launch(fe);
    }
    gj({Dp(act[levels][0])});
    gemv_launch({{xv(act[levels][0]), nullptr, Dp(act[levels][0]), yv(act[levels][0]), nullptr, nullptr, 1.0, 0.0}});
    for (int l = levels - 1; l >= 0; --l) {  // backward: x_o = c_o - P_o x_{o-} - Q_o x_{o+}
        const std::vector<int>& A = act[l];
        const int m = (int)A.size();
        std::vector<GemvJob> bo;
        for (int p = 1; p < m; p += 2) {
            GemvJob j{xv(A[p]), cv(A[p]), Pp(A[p]), xv(A[p - 1]), nullptr, nullptr, -1.0, -1.0};
            if (p + 1 < m) j.M2 = Qp(A[p]), j.v2 = xv(A[p + 1]);
            bo.push_back(j);
        }
        gemv_launch(bo);
    }
    pl.gemm.alloc(std::max<size_t>(gemm.size(), 1));
    pl.gemv.alloc(std::max<size_t>(gemv.size(), 1));
    pl.gjmats.alloc(std::max<size_t>(gjm.size(), 1));
    if (!gemm.empty()) CK(cudaMemcpyAsync(pl.gemm.p, gemm.data(), gemm.size() * sizeof(GemmJob), cudaMemcpyHostToDevice, c.st));
    if (!gemv.empty()) CK(cudaMemcpyAsync(pl.gemv.p, gemv.data(), gemv.size() * sizeof(GemvJob), cudaMemcpyHostToDevice, c.st));
    CK(cudaMemcpyAsync(pl.gjmats.p, gjm.data(), gjm.size() * sizeof(double*), cudaMemcpyHostToDevice, c.st));
    // level-0 Lo_j = Up_{j-1}^T
    std::vector<double*> td;
    std::vector<const double*> ts;
    for (int p = 1; p < nblk; ++p) {
        td.push_back(Lo(0, p));
        ts.push_back(Up(0, p - 1));
    }
    pl.tr_dst.alloc(std::max<size_t>(td.size(), 1));
    pl.tr_src.alloc(std::max<size_t>(ts.size(), 1));
    if (!td.empty()) {
        CK(cudaMemcpyAsync(pl.tr_dst.p, td.data(), td.size() * sizeof(double*), cudaMemcpyHostToDevice, c.st));
        CK(cudaMemcpyAsync(pl.tr_src.p, ts.data(), ts.size() * sizeof(const double*), cudaMemcpyHostToDevice, c.st));
    }
    pl.colbuf.alloc((size_t)pl.max_batch * S * GP);
    pl.rowbuf.alloc((size_t)pl.max_batch * S * GP);
    pl.flag.alloc(1);
    std::vector<int2> ph;
    for (const CrLaunch& st : pl.solve) ph.push_back(make_int2(st.first, st.count));
    pl.phases.alloc(std::max<size_t>(ph.size(), 1));
    if (!ph.empty()) CK(cudaMemcpyAsync(pl.phases.p, ph.data(), ph.size() * sizeof(int2), cudaMemcpyHostToDevice, c.st));
    CK(cudaStreamSynchronize(c.st));
    return plp;
}


CrView cr_view(const std::shared_ptr<void>& plan) {
    CrPlan& pl = *static_cast<CrPlan*>(plan.get());
    const size_t SS = (size_t)pl.S * pl.S;
    return CrView{pl.D.p, pl.LU.p + (size_t)pl.nb * SS, pl.nb, pl.S, pl.gemv.p, pl.phases.p, (int)pl.solve.size()};
}

// zero D and the level-0 Lo / Up slots before the caller fills them
void cr_zero(Ctx& c, const std::shared_ptr<void>& plan) {
    CrPlan& pl = *static_cast<CrPlan*>(plan.get());
    const size_t SS = (size_t)pl.S * pl.S;
    CK(cudaMemsetAsync(pl.D.p, 0, pl.nb * SS * sizeof(double), c.st));
    CK(cudaMemsetAsync(pl.LU.p, 0, 2 * (size_t)pl.nb * SS * sizeof(double), c.st));
    CK(cudaMemsetAsync(pl.flag.p, 0, sizeof(int), c.st));
}

// factor after D and Up_0 hold the system: Lo_0 = Up^T, the level plan,
// ERR_SINGULAR on a zero / non-finite pivot
void cr_factor(Ctx& c, const std::shared_ptr<void>& plan, unsigned err_bit) {
    CrPlan& pl = *static_cast<CrPlan*>(plan.get());
    const int S = pl.S, nb = pl.nb;
    if (nb > 1) {
        PROF(c, "k_transpose");
        launch_k(c, k_cr_transpose, dim3(S / 32, S / 32, nb - 1), dim3(32, 8), 0, (double* const*)pl.tr_dst.p,
                 (const double* const*)pl.tr_src.p, S);
        CK_LAUNCH();
    }
    for (const CrLaunch& st : pl.factor) {
        if (st.kind == 1) {
            run_gj(c, pl, st.first, st.count);
        } else {
            PROF(c, "k_cr_gemm");
            launch_k(c, k_cr_gemm, dim3((S / GT) * (S / GT), 1, st.count), 128, 0,
                     (const GemmJob*)(pl.gemm.p + st.first), S);
            CK_LAUNCH();
        }
    }
    {
        PROF(c, "k_flag_err");
        launch_k(c, k_flag_err, 1, 1, 0, (const int*)pl.flag.p, c.sc.p, err_bit);
        CK_LAUNCH();
    }
}

namespace {

// the solve's batched GEMV launches (y -> x)
void cr_solve_launches(Ctx& c, CrPlan& pl) {
    const int S = pl.S;
    for (const CrLaunch& st : pl.solve) {
        PROF(c, "k_cr_gemv");
        if ((long long)st.count * (S / 32) >= 4LL * c.num_sms)
            launch_k(c, k_cr_gemv<4>, dim3(S / 32, st.count), 256, 2 * S * sizeof(double),
                     (const GemvJob*)(pl.gemv.p + st.first), S);
        else
            launch_k(c, k_cr_gemv<1>, dim3(S / 8, st.count), 256, 2 * S * sizeof(double),
                     (const GemvJob*)(pl.gemv.p + st.first), S);
        CK_LAUNCH();
    }
}

}  // namespace

void bt_setup(Ctx& c) {
    const Layout& L = c.L;
    const int n = c.dim, np = L.dim_flux;
    auto block_of_iface = [&](int k) { return k < L.NV ? k / (L.nsx - 1) : (k - L.NV) / L.nsx; };
    std::vector<int> blk(n), loc(n);
    int nblk = 0;
    for (int r = 0; r < n; ++r) {
        blk[r] = block_of_iface(L.basis_iface(r % np));
        nblk = std::max(nblk, blk[r] + 1);
    }
    std::vector<int> sz(nblk, 0);
    for (int r = 0; r < n; ++r) loc[r] = sz[blk[r]]++;
    int smax = 0;
    for (int j = 0; j < nblk; ++j) {
        if (sz[j] == 0) throw ConfigError("block-tridiagonal interface solve: empty block");
        smax = std::max(smax, sz[j]);
    }
    const int S = (smax + 63) / 64 * 64;
    c.bt_nblk = nblk;
    c.bt_sz = sz;
    auto up_i = [&](DevBuf<int>& d, const std::vector<int>& h) {
        d.alloc(std::max<size_t>(h.size(), 1));
        CK(cudaMemcpyAsync(d.p, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice, c.st));
    };
    up_i(c.bt_blk, blk);
    up_i(c.bt_loc, loc);
    up_i(c.bt_bsz, sz);
    c.bt_y.alloc((size_t)nblk * S);
    c.bt_x.alloc((size_t)nblk * S);
    c.cr_plan = cr_create(c, nblk, S, c.bt_y.p, c.bt_x.p);
    c.hg_x.alloc(n);
    c.hg_y.alloc(n);
    c.hg_z.alloc(n);
    c.hg_xi.alloc(n);
    c.hg_state.alloc(sizeof(HagerState) / sizeof(double) + 1);
    CK(cudaStreamSynchronize(c.st));
}

// Factorisation at every rebuild (after the CSR of K holds the new values).
void bt_factor(Ctx& c) {
    CrPlan& pl = plan_of(c);
    const int n = c.dim, S = pl.S, nb = pl.nb;
    const size_t SS = (size_t)S * S;
    cr_zero(c, c.cr_plan);
    {
        PROF(c, "k_bt_scatter");
        launch_k(c, k_cr_scatter, cdiv(n, TPB), TPB, 0, (const int*)c.k_ptr.p, (const int*)c.k_col.p,
                 (const double*)c.k_val.p, n, (const int*)c.bt_blk.p, (const int*)c.bt_loc.p, S, pl.D.p,
                 pl.LU.p + (size_t)nb * SS);
        CK_LAUNCH();
    }
    {
        PROF(c, "k_bt_scatter");
        launch_k(c, k_cr_pad, cdiv((long long)nb * S, TPB), TPB, 0, (const int*)c.bt_bsz.p, nb, S, pl.D.p);
        CK_LAUNCH();
    }
    cr_factor(c, c.cr_plan, ERR_SINGULAR);
}

// x = M^-1 rhs through K x = J rhs (transposed: x = M^-T rhs = J^T K^-1 rhs).
void bt_solve_t(Ctx& c, const double* rhs, double* x, int transposed) {
    CrPlan& pl = plan_of(c);
    const int n = c.dim, S = pl.S;
    CK(cudaMemsetAsync(c.bt_y.p, 0, (size_t)pl.nb * S * sizeof(double), c.st));
    {
        PROF(c, "k_bt_gather");
        launch_k(c, k_bt_gather, cdiv(n, TPB), TPB, 0, rhs, n, (const int*)c.bt_blk.p, (const int*)c.bt_loc.p, S,
                 c.bt_y.p, transposed);
        CK_LAUNCH();
    }
    cr_solve_launches(c, pl);
    {
        PROF(c, "k_bt_unpermute");
        launch_k(c, k_bt_unpermute, cdiv(n, TPB), TPB, 0, (const double*)c.bt_x.p, n, (const int*)c.bt_blk.p,
                 (const int*)c.bt_loc.p, S, x, transposed);
        CK_LAUNCH();
    }
}

void bt_solve(Ctx& c, const double* rhs, double* x) { bt_solve_t(c, rhs, x, 0); }

// The rcond guard of the block-tridiagonal path (each rebuild, after bt_factor):
// the oracle's Hager/Higham estimate with device solves; sets sc->rcond and
// ERR_SINGULAR when !(rcond > threshold).
void bt_rcond(Ctx& c, double threshold, unsigned err_bit) {
    const int n = c.dim;
    HagerState* st = reinterpret_cast<HagerState*>(c.hg_state.p);
    {
        PROF(c, "k_hager");
        launch_k(c, k_hager_init, 1, 1024, 0, c.csr_ptr.p, c.csr_tpos.p, c.csr_val.p, n, c.hg_x.p, st);
        CK_LAUNCH();
    }
    for (int it = 0; it < 5; ++it) {
        bt_solve_t(c, c.hg_x, c.hg_y, 0);
        {
            PROF(c, "k_hager");
            launch_k(c, k_hager_a, 1, 1024, 0, (const double*)c.hg_y.p, n, it, c.hg_xi.p, st);
            CK_LAUNCH();
        }
        bt_solve_t(c, c.hg_xi, c.hg_z, 1);
        {
            PROF(c, "k_hager");
            launch_k(c, k_hager_b, 1, 1024, 0, (const double*)c.hg_z.p, n, c.hg_x.p, st);
            CK_LAUNCH();
        }
    }
    {
        PROF(c, "k_hager");
        launch_k(c, k_hager_fin, 1, 1, 0, st, c.sc.p, threshold, err_bit);
        CK_LAUNCH();
    }
}

}  // namespace mpm2p
