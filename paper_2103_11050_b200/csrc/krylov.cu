// krylov.cu — K7: the interface solve as preconditioned MINRES over a
// custom CSR SpMV, for systems too large for the dense inverse (C5: dim
// 65,024; the reference's dense PartialPivLU there would be 34 GB,
// proj/src/mrcm.cpp:198,226,264).
//
// SURVEY.md H1 (verified numerically): K = J M — phi-rows
// first, then the negated psi-rows — is symmetric quasi-definite, so MINRES
// applies to K x = J b with the SPD Jacobi preconditioner P = |diag K|.
// One cooperative persistent kernel runs the whole iteration: each thread
// owns a fixed set of rows; per iteration one SpMV + preconditioner + AXPYs
// and two dot products, i.e. two grid barriers (block partials are combined
// redundantly and in a fixed order by every block, so all blocks see
// bit-identical scalars and the run is deterministic).
#include <cooperative_groups.h>

#include "context.cuh"

namespace cg = cooperative_groups;

namespace mpm2p {

namespace {

constexpr int KTPB = 256;

struct MinresArgs {
    const int* ptr;
    const int* col;
    const double* val;   // K in CSR
    const double* pinv;  // 1 / |diag K|
    const double* b;     // J * rhs
    double* x;           // solution (M x = rhs)
    double *y, *v, *r1, *r2, *w, *w1, *w2, *t;
    double* part;        // 2 * gridDim doubles
    int n;
    double tol;
    int maxit;
    Scalars* sc;
};

__device__ __forceinline__ double block_sum(double v, double* sh) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[wi] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
        s = warp_sum(s);
    }
    return s;  // valid in thread 0
}

// Every block combines the partials in the same order -> identical scalars.
__device__ __forceinline__ double all_sum(const double* part, int nb, double* sh) {
    double v = 0.0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) v += __ldcg(part + i);
    v = block_sum(v, sh);
    __shared__ double bc;
    if (threadIdx.x == 0) bc = v;
    __syncthreads();
    return bc;
}

__global__ void __launch_bounds__(KTPB) k_minres(MinresArgs a) {
    pdl_begin();
    cg::grid_group grid = cg::this_grid();
    __shared__ double sh[32];
    const int n = a.n;
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gnt = gridDim.x * blockDim.x;
    const int nb = gridDim.x;
    // r1 = b, y = P^-1 r1, beta1^2 = r1 . y ; x = 0, w = w2 = 0
    double loc = 0.0;
    for (int i = gtid; i < n; i += gnt) {
        const double r = a.b[i];
        const double yy = r * a.pinv[i];
        a.r1[i] = r;
        a.r2[i] = r;
        a.y[i] = yy;
        a.x[i] = 0.0;
        a.w[i] = 0.0;
        a.w2[i] = 0.0;
        loc += r * yy;
    }
    loc = block_sum(loc, sh);
    if (threadIdx.x == 0) a.part[blockIdx.x] = loc;
    grid.sync();
    const double beta1 = sqrt(all_sum(a.part, nb, sh));
    if (!(beta1 > 0.0)) {
        return;
    }
    double oldb = 0.0, beta = beta1, dbar = 0.0, epsln = 0.0, phibar = beta1;
    double cs = -1.0, sn = 0.0;
    int it = 0;
    for (it = 1; it <= a.maxit; ++it) {
        const double s = 1.0 / beta;
        // phase A: v = s y ; t = K v - (beta/oldb) r1 ; alfa = v . t
        loc = 0.0;
        for (int i = gtid; i < n; i += gnt) {
            double acc = 0.0;
            for (int z = a.ptr[i]; z < a.ptr[i + 1]; ++z) acc += a.val[z] * __ldcg(a.y + a.col[z]);
            const double vi = s * __ldcg(a.y + i);
            double ti = s * acc;
            if (it >= 2) ti -= (beta / oldb) * a.r1[i];
            a.v[i] = vi;
            a.t[i] = ti;
            loc += vi * ti;
        }
        loc = block_sum(loc, sh);
        if (threadIdx.x == 0) a.part[blockIdx.x] = loc;
        grid.sync();
        const double alfa = all_sum(a.part, nb, sh);
        // phase B: y = t - (alfa/beta) r2 ; r1 = r2 ; r2 = y ; y = P^-1 r2 ; beta^2 = r2 . y
        loc = 0.0;
        for (int i = gtid; i < n; i += gnt) {
            const double yi = a.t[i] - (alfa / beta) * a.r2[i];
            a.r1[i] = a.r2[i];
            a.r2[i] = yi;
            const double zi = yi * a.pinv[i];
            a.y[i] = zi;
            loc += yi * zi;
        }
        loc = block_sum(loc, sh);
        if (threadIdx.x == 0) a.part[nb + blockIdx.x] = loc;
        grid.sync();
        oldb = beta;
        beta = sqrt(all_sum(a.part + nb, nb, sh));
        // Givens rotation (scalars identical in every thread)
        const double oldeps = epsln;
        const double delta = cs * dbar + sn * alfa;
        const double gbar = sn * dbar - cs * alfa;
        epsln = sn * beta;
        dbar = -cs * beta;
        const double gamma = fmax(hypot(gbar, beta), 1e-300);
        cs = gbar / gamma;
        sn = beta / gamma;
        const double phi = cs * phibar;
        phibar = sn * phibar;
        const double denom = 1.0 / gamma;
        // w1 = w2 ; w2 = w ; w = (v - oldeps w1 - delta w2) / gamma ; x += phi w  (own rows only)
        for (int i = gtid; i < n; i += gnt) {
            const double w1 = a.w2[i], w2 = a.w[i];
            const double wn = (a.v[i] - oldeps * w1 - delta * w2) * denom;
            a.w2[i] = w2;
            a.w[i] = wn;
            a.x[i] += phi * wn;
        }
        if (phibar <= a.tol * beta1 || !(beta > 0.0)) break;
    }
    if (gtid == 0) {
        const int used = it > a.maxit ? a.maxit : it;
        a.sc->kr_iters_total += used;
        a.sc->kr_iters_max = max(a.sc->kr_iters_max, used);
        a.sc->kr_solves += 1;
        if (it > a.maxit) atomicOr(&a.sc->err, ERR_SINGULAR);  // no convergence: treated as a singular system
    }
}

// K = J M in CSR: K row r is M row (r < h ? h + r : r - h), negated for r >= h.
__global__ void k_fill_k(const int* __restrict__ mptr, const double* __restrict__ mval,
                         const int* __restrict__ kptr, double* __restrict__ kval, int n) {
    pdl_begin();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int h = n / 2;
    const int src = r < h ? h + r : r - h;
    const double sg = r < h ? 1.0 : -1.0;
    const int d0 = kptr[r], s0 = mptr[src], cnt = mptr[src + 1] - s0;
    for (int z = 0; z < cnt; ++z) kval[d0 + z] = sg * mval[s0 + z];
}

// Jacobi preconditioner 1/|K_rr| (K_rr = M_(src) diagonal entry of column r).
__global__ void k_kdiag(const int* __restrict__ kptr, const int* __restrict__ kcol, const double* __restrict__ kval,
                        double* __restrict__ pinv, int n) {
    pdl_begin();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    double d = 0.0;
    for (int z = kptr[r]; z < kptr[r + 1]; ++z)
        if (kcol[z] == r) d = kval[z];
    pinv[r] = d != 0.0 ? 1.0 / fabs(d) : 1.0;
}

// b_K = J b: phi-rows first, then the negated psi-rows.
__global__ void k_jvec(const double* __restrict__ b, double* __restrict__ bk, int n) {
    pdl_begin();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int h = n / 2;
    bk[r] = r < h ? b[h + r] : -b[r - h];
}

}  // namespace

// Host-side K pattern: rows of M permuted (same column indices).
void krylov_setup(Ctx& c, const std::vector<int>& mptr, const std::vector<int>& mcol) {
    const int n = (int)mptr.size() - 1, h = n / 2;
    std::vector<int> kptr(1, 0), kcol;
    for (int r = 0; r < n; ++r) {
        const int src = r < h ? h + r : r - h;
        for (int z = mptr[src]; z < mptr[src + 1]; ++z) kcol.push_back(mcol[z]);
        kptr.push_back((int)kcol.size());
    }
    c.k_ptr.alloc(kptr.size());
    c.k_col.alloc(std::max<size_t>(kcol.size(), 1));
    c.k_val.alloc(std::max<size_t>(kcol.size(), 1));
    CK(cudaMemcpyAsync(c.k_ptr.p, kptr.data(), kptr.size() * sizeof(int), cudaMemcpyHostToDevice, c.st));
    if (!kcol.empty())
        CK(cudaMemcpyAsync(c.k_col.p, kcol.data(), kcol.size() * sizeof(int), cudaMemcpyHostToDevice, c.st));
    const size_t v = (size_t)n;
    c.kr_pinv.alloc(v);
    c.kr_work.alloc(10 * v + 4 * (size_t)c.num_sms * 8);
    CK(cudaStreamSynchronize(c.st));
}

// After assembly (rebuild): K values and the Jacobi preconditioner.
void krylov_prepare(Ctx& c) {
    const int n = c.dim;
    {
        PROF(c, "k_fill_k");
        launch_k(c, k_fill_k, cdiv(n, KTPB), KTPB, 0, c.csr_ptr, c.csr_val, c.k_ptr, c.k_val, n);
        CK_LAUNCH();
    }
    {
        PROF(c, "k_kdiag");
        launch_k(c, k_kdiag, cdiv(n, KTPB), KTPB, 0, c.k_ptr, c.k_col, c.k_val, c.kr_pinv, n);
        CK_LAUNCH();
    }
}

// x = M^-1 rhs by MINRES on K x = J rhs.
void krylov_solve(Ctx& c, const double* rhs, double* x) {
    const int n = c.dim;
    static DeviceCache occ;
    int per_sm = occ.at().load();
    if (per_sm < 0) {
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_minres, KTPB, 0));
        occ.at().store(per_sm);
    }
    if (per_sm < 1) throw CudaError("krylov_solve: cooperative kernel does not fit on an SM");
    const int blocks = std::max(1, std::min(per_sm * c.num_sms, cdiv(n, KTPB)));
    double* wk = c.kr_work.p;
    const size_t v = (size_t)n;
    double* bk = wk + 9 * v;
    {
        PROF(c, "k_jvec");
        launch_k(c, k_jvec, cdiv(n, KTPB), KTPB, 0, rhs, bk, n);
        CK_LAUNCH();
    }
    MinresArgs a{c.k_ptr, c.k_col, c.k_val, c.kr_pinv, bk, x, wk, wk + v, wk + 2 * v, wk + 3 * v, wk + 4 * v,
                 wk + 5 * v, wk + 6 * v, wk + 7 * v, wk + 10 * v, n, c.krylov_tol, c.krylov_maxit, c.sc.p};
    void* args[] = {&a};
    PROF(c, "k_minres");
    CK(cudaLaunchCooperativeKernel((void*)k_minres, blocks, KTPB, args, 0, c.st));
    CK_LAUNCH();
}

}  // namespace mpm2p
