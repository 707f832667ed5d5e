// blocktri.cu — K7b: direct block-tridiagonal interface solve for systems
// above the dense limit (C5: dim 65,024; the reference's dense PartialPivLU
// there would be 34 GB, proj/src/mrcm.cpp:198,226,264).
//
// Ordered by subdomain row (the vertical interfaces of row j and the
// horizontal interfaces between rows j and j+1 form block j), K = J M is
// block tridiagonal: an interface only couples to interfaces that share a
// subdomain with it. K is symmetric quasi-definite, so block
// LDL^T needs no pivoting:
//   S_0 = D_0,  T_{j-1} = S_{j-1}^-1 E_{j-1},  S_j = D_j - E_{j-1}^T T_{j-1};
//   solve: y_j = b_j - T_{j-1}^T y_{j-1} (forward),
//          x_j = S_j^-1 y_j - T_j x_{j+1} (backward).
// Per rebuild: nblk dense inversions (ping-pong Gauss-Jordan, dense.cu) and
// two GEMMs per block; per solve: 2 nblk - 1 dependent block products, each
// HBM-bound. At C5: 128 blocks of 510 unknowns, S^-1 / T / T^T / D / E about
// 0.27 GB each.

#include "context.cuh"


namespace mpm2p {

namespace {

constexpr int TPB = 256;

// C[m x n] = op(A)[m x k] * B[k x n] (+ beta C0), row-major. TA: A is stored
// k x m (use A^T). 64 x 64 tiles, k-slabs of 16, 4 x 4 outputs per thread.
template <bool TA>
__global__ void __launch_bounds__(256) k_dgemm(int m, int n, int kk, const double* __restrict__ A, int lda,
                                               const double* __restrict__ Bm, int ldb, double* __restrict__ C,
                                               int ldc, double alpha, const double* __restrict__ C0, int ldc0) {
    pdl_begin();
    __shared__ double As[16][64 + 1], Bs[16][64 + 1];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int i0 = blockIdx.y * 64, j0 = blockIdx.x * 64;
    double acc[4][4] = {};
    for (int k0 = 0; k0 < kk; k0 += 16) {
        for (int x = threadIdx.x; x < 16 * 64; x += 256) {
            const int kq = x / 64, ii = x % 64;  // As[kq][ii] = op(A)[i0+ii][k0+kq]
            const int gi = i0 + ii, gk = k0 + kq;
            double v = 0.0;
            if (gi < m && gk < kk) v = TA ? A[(size_t)gk * lda + gi] : A[(size_t)gi * lda + gk];
            As[kq][ii] = v;
            const int gj = j0 + ii;  // Bs[kq][jj] = B[k0+kq][j0+jj]
            Bs[kq][ii] = (gj < n && gk < kk) ? Bm[(size_t)gk * ldb + gj] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kq = 0; kq < 16; ++kq) {
            double a[4], b[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                a[q] = As[kq][ty + 16 * q];
                b[q] = Bs[kq][tx + 16 * q];
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int r = 0; r < 4; ++r) acc[q][r] = fma(a[q], b[r], acc[q][r]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int gi = i0 + ty + 16 * q, gj = j0 + tx + 16 * r;
            if (gi < m && gj < n) {
                double v = alpha * acc[q][r];
                if (C0) v += C0[(size_t)gi * ldc0 + gj];
                C[(size_t)gi * ldc + gj] = v;
            }
        }
}

// D_j and E_j (= K[block j, block j+1]) from the CSR of K.
__global__ void k_bt_scatter(const int* __restrict__ kptr, const int* __restrict__ kcol, const double* __restrict__ kval,
                             int n, const int* __restrict__ blk, const int* __restrict__ loc,
                             const long long* __restrict__ doff, const long long* __restrict__ eoff,
                             const int* __restrict__ bsz, double* __restrict__ D, double* __restrict__ E) {
    pdl_begin();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int j = blk[r], lr = loc[r];
    for (int z = kptr[r]; z < kptr[r + 1]; ++z) {
        const int c = kcol[z], jc = blk[c], lc = loc[c];
        if (jc == j) D[doff[j] + (long long)lr * bsz[j] + lc] = kval[z];
        else if (jc == j + 1) E[eoff[j] + (long long)lr * bsz[j + 1] + lc] = kval[z];
    }
}

// out[cols x rows] = in[rows x cols]^T
__global__ void k_transpose(const double* __restrict__ in, int rows, int cols, double* __restrict__ out) {
    pdl_begin();
    __shared__ double t[32][33];
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int r = by + y, cc = bx + threadIdx.x;
        t[y][threadIdx.x] = (r < rows && cc < cols) ? in[(size_t)r * cols + cc] : 0.0;
    }
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int cc = bx + y, r = by + threadIdx.x;
        if (cc < cols && r < rows) out[(size_t)cc * rows + r] = t[threadIdx.x][y];
    }
}

__global__ void k_flag_err(const int* flag, Scalars* sc, unsigned bit) {
    pdl_begin();
    if (*flag) atomicOr(&sc->err, bit);
}

// y (block order) <- J rhs gathered: y[off[blk[r]] + loc[r]] = (J rhs)_r
// (transposed = 0) y = J rhs, (1) y = rhs, in block order
__global__ void k_bt_gather(const double* __restrict__ rhs, int n, const int* __restrict__ blk,
                            const int* __restrict__ loc, const int* __restrict__ voff, double* __restrict__ y,
                            int transposed) {
    pdl_begin();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int h = n / 2;
    const double v = transposed ? rhs[r] : (r < h ? rhs[h + r] : -rhs[r - h]);
    y[voff[blk[r]] + loc[r]] = v;
}

// (transposed = 0) x = xb, (1) x = J^T xb, from block order
__global__ void k_bt_unpermute(const double* __restrict__ xb, int n, const int* __restrict__ blk,
                               const int* __restrict__ loc, const int* __restrict__ voff, double* __restrict__ x,
                               int transposed) {
    pdl_begin();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int h = n / 2;
    if (!transposed) {
        x[r] = xb[voff[blk[r]] + loc[r]];
    } else {  // (J^T w)_i = -w_{i+h} (i < h), w_{i-h} (i >= h)
        const int q = r < h ? r + h : r - h;
        const double w = xb[voff[blk[q]] + loc[q]];
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

// The block steps of a solve are a dependent chain of small products, each
// latency-bound (one L2/HBM round trip for the block plus the launch). The
// matrices are constant between rebuilds, so each kernel loads its rows into
// registers BEFORE griddepcontrol.wait and triggers its dependents at entry:
// launched with programmatic dependent launch (bt_solve), step j+1's block
// streams in while step j finishes, and only the vector part is serialised.
constexpr int BT_Q = 8;     // warps per row: a row's columns are split in BT_Q quarters
constexpr int BT_NPL = 6;   // prefetched doubles per lane: quarters of up to 32 * 6 columns
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Lane's share of a row quarter [c0, c1): columns c0 + lane + 32 q.
__device__ __forceinline__ void bt_prefetch(double (&v)[BT_NPL], const double* row, int c0, int c1, bool on, int lane) {
#pragma unroll
    for (int q = 0; q < BT_NPL; ++q) {
        const int c = c0 + lane + 32 * q;
        v[q] = (on && c < c1) ? __ldg(row + c) : 0.0;
    }
}
__device__ __forceinline__ double bt_dot(const double (&v)[BT_NPL], const double* row, int c0, int c1,
                                         const double* x, double acc, int lane) {
#pragma unroll
    for (int q = 0; q < BT_NPL; ++q) {
        const int c = c0 + lane + 32 * q;
        if (c < c1) acc = fma(v[q], __ldcg(x + c), acc);
    }
    for (int c = c0 + lane + 32 * BT_NPL; c < c1; c += 32) acc = fma(row[c], __ldcg(x + c), acc);  // wider blocks
    return acc;
}
// Quarter partials of the block's rows, combined in quarter order (deterministic).
__device__ __forceinline__ bool bt_combine(double& acc, int lane) {
    __shared__ double part[256 / 32];
    const int w = threadIdx.x >> 5;
    acc = warp_sum(acc);
    if (lane == 0) part[w] = acc;
    __syncthreads();
    if ((w % BT_Q) != 0 || lane != 0) return false;
    acc = part[w];
#pragma unroll
    for (int q = 1; q < BT_Q; ++q) acc += part[w + q];
    return true;
}

// y_j -= G y_{j-1} (G = T_{j-1}^T, rows x cols): BT_Q warps per row (two rows
// per 256-thread block, so a step spreads over ~4x more SMs than one warp per
// row would), the row's quarter loaded before griddepcontrol.wait.
__global__ void __launch_bounds__(256) k_bt_fwd(const double* __restrict__ G, int rows, int cols,
                                                const double* yprev, double* y) {
    pdl_trigger();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = blockIdx.x * (256 / 32 / BT_Q) + w / BT_Q, qw = w % BT_Q;
    const bool on = row < rows;
    const int qlen = (cols + BT_Q - 1) / BT_Q, c0 = qw * qlen, c1 = min(cols, c0 + qlen);
    const double* g = G + (size_t)(on ? row : 0) * cols;
    double gv[BT_NPL];
    bt_prefetch(gv, g, c0, c1, on, lane);
    pdl_begin();  // y_{j-1} is complete and visible
    double acc = on ? bt_dot(gv, g, c0, c1, yprev, 0.0, lane) : 0.0;
    if (bt_combine(acc, lane) && on) y[row] -= acc;
}

// x_j = Sinv_j y_j - T_j x_{j+1} (T_j: rows x cols_next), BT_Q warps per row
__global__ void __launch_bounds__(256) k_bt_bwd(const double* __restrict__ Sinv, const double* __restrict__ T,
                                                int rows, int cols_next, const double* y, const double* xnext,
                                                double* x) {
    pdl_trigger();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = blockIdx.x * (256 / 32 / BT_Q) + w / BT_Q, qw = w % BT_Q;
    const bool on = row < rows;
    const int qs = (rows + BT_Q - 1) / BT_Q, s0 = qw * qs, s1 = min(rows, s0 + qs);
    const int qt = (cols_next + BT_Q - 1) / BT_Q, t0 = qw * qt, t1 = min(cols_next, t0 + qt);
    const double* sr = Sinv + (size_t)(on ? row : 0) * rows;
    const double* tr = T ? T + (size_t)(on ? row : 0) * cols_next : nullptr;
    double sv[BT_NPL], tv[BT_NPL];
    bt_prefetch(sv, sr, s0, s1, on, lane);
    bt_prefetch(tv, tr, t0, T ? t1 : t0, on && T, lane);
    pdl_begin();  // x_{j+1} is complete and visible (y_j was finished by the forward sweep)
    double acc = 0.0;
    if (on) {
        acc = bt_dot(sv, sr, s0, s1, y, 0.0, lane);
        if (T) {
            double a2 = bt_dot(tv, tr, t0, t1, xnext, 0.0, lane);
            acc -= a2;
        }
    }
    if (bt_combine(acc, lane) && on) x[row] = acc;
}

}  // namespace

// In-place inverse of an n x n row-major matrix (dense.cu).
void block_gj_inplace_pub(Ctx& c, double* W, int n);

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
    std::vector<long long> doff(nblk + 1, 0), eoff(nblk + 1, 0);
    std::vector<int> voff(nblk + 1, 0);
    for (int j = 0; j < nblk; ++j) {
        if (sz[j] == 0) throw ConfigError("block-tridiagonal interface solve: empty block");
        doff[j + 1] = doff[j] + (long long)sz[j] * sz[j];
        eoff[j + 1] = eoff[j] + (j + 1 < nblk ? (long long)sz[j] * sz[j + 1] : 0);
        voff[j + 1] = voff[j] + sz[j];
    }
    c.bt_nblk = nblk;
    c.bt_sz = sz;
    c.bt_doff = doff;
    c.bt_eoff = eoff;
    c.bt_voff = voff;
    auto up_i = [&](DevBuf<int>& d, const std::vector<int>& h) {
        d.alloc(std::max<size_t>(h.size(), 1));
        CK(cudaMemcpyAsync(d.p, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice, c.st));
    };
    up_i(c.bt_blk, blk);
    up_i(c.bt_loc, loc);
    up_i(c.bt_bsz, sz);
    up_i(c.bt_voffd, voff);
    c.bt_doffd.alloc(doff.size());
    c.bt_eoffd.alloc(eoff.size());
    CK(cudaMemcpyAsync(c.bt_doffd.p, doff.data(), doff.size() * sizeof(long long), cudaMemcpyHostToDevice, c.st));
    CK(cudaMemcpyAsync(c.bt_eoffd.p, eoff.data(), eoff.size() * sizeof(long long), cudaMemcpyHostToDevice, c.st));
    c.bt_D.alloc(doff[nblk]);
    c.bt_Sinv.alloc(doff[nblk]);
    c.bt_E.alloc(std::max<long long>(eoff[nblk], 1));
    c.bt_T.alloc(std::max<long long>(eoff[nblk], 1));
    c.bt_G.alloc(std::max<long long>(eoff[nblk], 1));
    c.bt_y.alloc(n);
    c.bt_x.alloc(n);
    c.bt_sy.alloc(n);
    c.hg_x.alloc(n);
    c.hg_y.alloc(n);
    c.hg_z.alloc(n);
    c.hg_xi.alloc(n);
    c.hg_state.alloc(sizeof(HagerState) / sizeof(double) + 1);
    CK(cudaStreamSynchronize(c.st));
}

// Factorisation at every rebuild (after the CSR of K holds the new values).
void bt_factor(Ctx& c) {
    const int n = c.dim, nb = c.bt_nblk;
    c.bt_D.zero(c.st);
    c.bt_E.zero(c.st);
    {
        PROF(c, "k_bt_scatter");
        launch_k(c, k_bt_scatter, cdiv(n, TPB), TPB, 0, c.k_ptr, c.k_col, c.k_val, n, c.bt_blk, c.bt_loc, c.bt_doffd,
                 c.bt_eoffd, c.bt_bsz, c.bt_D, c.bt_E);
        CK_LAUNCH();
    }
    auto gemm = [&](bool ta, int m, int nn, int kk, const double* A, int lda, const double* Bm, int ldb, double* C,
                    int ldc, double alpha, const double* C0, int ldc0) {
        PROF(c, "k_dgemm");
        const dim3 g(cdiv(nn, 64), cdiv(m, 64));
        if (ta) launch_k(c, k_dgemm<true>, g, 256, 0, m, nn, kk, A, lda, Bm, ldb, C, ldc, alpha, C0, ldc0);
        else launch_k(c, k_dgemm<false>, g, 256, 0, m, nn, kk, A, lda, Bm, ldb, C, ldc, alpha, C0, ldc0);
        CK_LAUNCH();
    };
    for (int j = 0; j < nb; ++j) {
        const int s = c.bt_sz[j];
        double* Sj = c.bt_Sinv.p + c.bt_doff[j];
        const double* Dj = c.bt_D.p + c.bt_doff[j];
        if (j == 0) {
            CK(cudaMemcpyAsync(Sj, Dj, (size_t)s * s * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
        } else {
            const int sp = c.bt_sz[j - 1];
            const double* Sp = c.bt_Sinv.p + c.bt_doff[j - 1];
            const double* Ep = c.bt_E.p + c.bt_eoff[j - 1];  // sp x s
            double* Tp = c.bt_T.p + c.bt_eoff[j - 1];         // sp x s
            gemm(false, sp, s, sp, Sp, sp, Ep, s, Tp, s, 1.0, nullptr, 0);  // T = Sinv_{j-1} E_{j-1}
            gemm(true, s, s, sp, Ep, s, Tp, s, Sj, s, -1.0, Dj, s);         // S_j = D_j - E^T T
            {
                PROF(c, "k_transpose");
                launch_k(c, k_transpose, dim3(cdiv(s, 32), cdiv(sp, 32)), dim3(32, 8), 0, Tp, sp, s,
                         c.bt_G.p + c.bt_eoff[j - 1]);  // G = T^T (s x sp)
                CK_LAUNCH();
            }
        }
        block_gj_inplace_pub(c, Sj, s);
        {
            PROF(c, "k_flag_err");
            launch_k(c, k_flag_err, 1, 1, 0, c.gj_piv.p + s, c.sc.p, ERR_SINGULAR);
            CK_LAUNCH();
        }
    }
}

// x = M^-1 rhs through K x = J rhs (transposed: x = M^-T rhs = J^T K^-1 rhs).
void bt_solve_t(Ctx& c, const double* rhs, double* x, int transposed) {
    const int n = c.dim, nb = c.bt_nblk;
    double* y = c.bt_y.p;
    double* xb = c.bt_x.p;
    {
        PROF(c, "k_bt_gather");
        launch_k(c, k_bt_gather, cdiv(n, TPB), TPB, 0, rhs, n, c.bt_blk, c.bt_loc, c.bt_voffd, y, transposed);
        CK_LAUNCH();
    }
    // block steps with programmatic dependent launch (see k_bt_fwd)
    auto launch_pdl = [&](auto kern, int grid, auto... args) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(TPB);
        cfg.dynamicSmemBytes = 0;
        cfg.stream = c.st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = c.bt_pdl ? 1 : 0;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, kern, args...));
    };
    for (int j = 1; j < nb; ++j) {
        const int s = c.bt_sz[j], sp = c.bt_sz[j - 1];
        PROF(c, "k_bt_fwd");
        launch_pdl(k_bt_fwd, cdiv((long long)s * 32 * BT_Q, TPB), (const double*)(c.bt_G.p + c.bt_eoff[j - 1]), s, sp,
                   (const double*)(y + c.bt_voff[j - 1]), y + c.bt_voff[j]);
        CK_LAUNCH();
    }
    for (int j = nb - 1; j >= 0; --j) {
        const int s = c.bt_sz[j];
        const bool last = j == nb - 1;
        const int sn = last ? 0 : c.bt_sz[j + 1];
        PROF(c, "k_bt_bwd");
        launch_pdl(k_bt_bwd, cdiv((long long)s * 32 * BT_Q, TPB), (const double*)(c.bt_Sinv.p + c.bt_doff[j]),
                   (const double*)(last ? nullptr : c.bt_T.p + c.bt_eoff[j]), s, sn, (const double*)(y + c.bt_voff[j]),
                   (const double*)(last ? nullptr : xb + c.bt_voff[j + 1]), xb + c.bt_voff[j]);
        CK_LAUNCH();
    }
    {
        PROF(c, "k_bt_unpermute");
        launch_k(c, k_bt_unpermute, cdiv(n, TPB), TPB, 0, xb, n, c.bt_blk, c.bt_loc, c.bt_voffd, x, transposed);
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
