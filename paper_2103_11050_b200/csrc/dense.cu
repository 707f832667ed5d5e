// dense.cu — dense interface-system machinery (stand-in for Eigen
// PartialPivLU + rcond, proj/src/mrcm.cpp:225-238,264, and the dense LDLT of
// the repair Laplacian, mrcm.cpp:372).
//
// The interface matrix is fixed between rebuilds, so it is inverted once per
// rebuild by Gauss-Jordan elimination with partial pivoting (one cooperative
// kernel, three grid barriers per pivot) and every later interface solve is a
// dense GEMV plus one step of iterative refinement against the sparse CSR
// operator — as accurate as the reference's LU solve, and bandwidth-bound
// rather than latency-bound. rcond is computed exactly as
// 1 / (||M||_1 ||M^-1||_1) (the quantity Eigen's rcond() estimates).
#include <cooperative_groups.h>

#include "context.cuh"

namespace cg = cooperative_groups;

namespace mpm2p {

namespace {

constexpr int TPB = 256;

// W: n x 2n augmented [A | I], row-major. piv/colbuf/rowbuf/krow: scratch.
__global__ void k_gauss_jordan(double* __restrict__ W, int n, int* __restrict__ piv, double* __restrict__ colbuf,
                               double* __restrict__ rowbuf, double* __restrict__ krow, int* __restrict__ singular) {
    cg::grid_group grid = cg::this_grid();
    const int n2 = 2 * n;
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nth = (long long)gridDim.x * blockDim.x;
    __shared__ double sv[32];
    __shared__ int si[32];
    for (int k = 0; k < n; ++k) {
        // phase A: pivot search in column k (block 0)
        if (blockIdx.x == 0) {
            double best = -1.0;
            int bi = k;
            for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
                const double v = fabs(W[(size_t)i * n2 + k]);
                if (v > best || (v == best && i < bi)) { best = v; bi = i; }
            }
            const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_down_sync(0xffffffffu, best, o);
                const int oi = __shfl_down_sync(0xffffffffu, bi, o);
                if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
            }
            if (lane == 0) { sv[w] = best; si[w] = bi; }
            __syncthreads();
            if (threadIdx.x == 0) {
                for (int t = 1; t < (int)(blockDim.x >> 5); ++t)
                    if (sv[t] > sv[0] || (sv[t] == sv[0] && si[t] < si[0])) { sv[0] = sv[t]; si[0] = si[t]; }
                piv[0] = si[0];
                if (!(sv[0] > 0.0)) *singular = 1;
            }
        }
        grid.sync();
        const int p = piv[0];
        // phase B: snapshot the pivot row (after the swap), column k and old row k
        for (long long x = tid; x < n2; x += nth) {
            rowbuf[x] = W[(size_t)p * n2 + x];
            krow[x] = W[(size_t)k * n2 + x];
        }
        for (long long i = tid; i < n; i += nth) {
            const int src = i == k ? p : (i == p ? k : (int)i);
            colbuf[i] = W[(size_t)src * n2 + k];
        }
        grid.sync();
        // phase C: eliminate column k from every other row, scale the pivot row
        const double pv = rowbuf[k];
        const double pinv = 1.0 / pv;
        for (long long x = tid; x < (long long)n * n2; x += nth) {
            const int i = (int)(x / n2), j = (int)(x % n2);
            if (i == k) {
                W[x] = rowbuf[j] * pinv;
            } else {
                const double base = (i == p) ? krow[j] : W[x];
                W[x] = base - (colbuf[i] * pinv) * rowbuf[j];
            }
        }
        grid.sync();
    }
}

__global__ void k_augment(const double* __restrict__ A, double* __restrict__ W, int n) {
    const long long tot = 2LL * n * n;
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < tot; x += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(x / (2 * n)), j = (int)(x % (2 * n));
        W[x] = j < n ? A[(size_t)i * n + j] : (j - n == i ? 1.0 : 0.0);
    }
}

__global__ void k_extract(const double* __restrict__ W, double* __restrict__ Ainv, int n) {
    const long long tot = (long long)n * n;
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < tot; x += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(x / n), j = (int)(x % n);
        Ainv[x] = W[(size_t)i * 2 * n + n + j];
    }
}

// 1-norms: out[0] = max_j sum_i |A_ij|, out[1] = same for B.
__global__ void k_norm1(const double* __restrict__ A, const double* __restrict__ B, int n, double* out) {
    __shared__ double sa[32], sb[32];
    double ma = 0.0, mb = 0.0;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        double a = 0.0, b = 0.0;
        for (int i = 0; i < n; ++i) {
            a += fabs(A[(size_t)i * n + j]);
            b += fabs(B[(size_t)i * n + j]);
        }
        ma = fmax(ma, a);
        mb = fmax(mb, b);
    }
    ma = warp_max(ma);
    mb = warp_max(mb);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) { sa[w] = ma; sb[w] = mb; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int t = 1; t < (int)(blockDim.x >> 5); ++t) { sa[0] = fmax(sa[0], sa[t]); sb[0] = fmax(sb[0], sb[t]); }
        out[0] = sa[0];
        out[1] = sb[0];
    }
}

// y = A x, one warp per row (coalesced row reads).
__global__ void k_gemv(const double* __restrict__ A, const double* __restrict__ x, double* __restrict__ y, int n) {
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (gw >= n) return;
    const double* row = A + (size_t)gw * n;
    double v = 0.0;
    for (int j = lane; j < n; j += 32) v += row[j] * x[j];
    v = warp_sum(v);
    if (lane == 0) y[gw] = v;
}

// r = b - M x with M in CSR, one thread per row.
__global__ void k_csr_residual(const int* __restrict__ ptr, const int* __restrict__ col, const double* __restrict__ val,
                               const double* __restrict__ x, const double* __restrict__ b, double* __restrict__ r, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double acc = 0.0;
    for (int z = ptr[i]; z < ptr[i + 1]; ++z) acc += val[z] * x[col[z]];
    r[i] = b[i] - acc;
}

__global__ void k_axpy(double* __restrict__ y, const double* __restrict__ x, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] += x[i];
}

}  // namespace

double dense_inverse(Ctx& c, const double* A, double* Ainv, int n) {
    if (n == 0) return 1.0;
    c.gj_work.alloc(std::max(c.gj_work.n, (size_t)2 * n * n));
    c.gj_col.alloc(std::max(c.gj_col.n, (size_t)n));
    c.gj_row.alloc(std::max(c.gj_row.n, (size_t)2 * n));
    c.gj_krow.alloc(std::max(c.gj_krow.n, (size_t)2 * n));
    c.gj_piv.alloc(std::max(c.gj_piv.n, (size_t)2));
    {
        PROF(c, "k_augment");
        k_augment<<<std::min(cdiv(2LL * n * n, TPB), 8 * c.num_sms), TPB, 0, c.st>>>(A, c.gj_work, n);
        CK_LAUNCH();
    }
    CK(cudaMemsetAsync(c.gj_piv.p + 1, 0, sizeof(int), c.st));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gauss_jordan, TPB, 0));
    const long long work = 2LL * n * n;
    int blocks = std::max(1, std::min(per_sm * c.num_sms, cdiv(work, TPB)));
    double* W = c.gj_work.p;
    int* piv = c.gj_piv.p;
    double* colb = c.gj_col.p;
    double* rowb = c.gj_row.p;
    double* krow = c.gj_krow.p;
    int* sing = c.gj_piv.p + 1;
    void* args[] = {&W, &n, &piv, &colb, &rowb, &krow, &sing};
    {
        PROF(c, "k_gauss_jordan");
        CK(cudaLaunchCooperativeKernel((void*)k_gauss_jordan, blocks, TPB, args, 0, c.st));
        CK_LAUNCH();
    }
    {
        PROF(c, "k_extract");
        k_extract<<<std::min(cdiv((long long)n * n, TPB), 8 * c.num_sms), TPB, 0, c.st>>>(c.gj_work, Ainv, n);
        CK_LAUNCH();
    }
    DevBuf<double> norms;
    norms.alloc(2);
    {
        PROF(c, "k_norm1");
        k_norm1<<<1, 1024, 0, c.st>>>(A, Ainv, n, norms);
        CK_LAUNCH();
    }
    double h[2];
    int singular = 0;
    CK(cudaMemcpyAsync(h, norms.p, sizeof(h), cudaMemcpyDeviceToHost, c.st));
    CK(cudaMemcpyAsync(&singular, sing, sizeof(int), cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
    if (singular || !std::isfinite(h[1]) || !(h[0] > 0.0) || !(h[1] > 0.0)) return 0.0;
    return 1.0 / (h[0] * h[1]);
}

void launch_gemv(Ctx& c, const double* A, const double* x, double* y, int n) {
    {
        PROF(c, "k_gemv");
        k_gemv<<<cdiv((long long)n * 32, TPB), TPB, 0, c.st>>>(A, x, y, n);
        CK_LAUNCH();
    }
}

void launch_csr_residual(Ctx& c, const int* ptr, const int* col, const double* val, const double* x, const double* b,
                         double* r, int n) {
    {
        PROF(c, "k_csr_residual");
        k_csr_residual<<<cdiv(n, TPB), TPB, 0, c.st>>>(ptr, col, val, x, b, r, n);
        CK_LAUNCH();
    }
}

void launch_axpy(Ctx& c, double* y, const double* x, int n) {
    {
        PROF(c, "k_axpy");
        k_axpy<<<cdiv(n, TPB), TPB, 0, c.st>>>(y, x, n);
        CK_LAUNCH();
    }
}

}  // namespace mpm2p
