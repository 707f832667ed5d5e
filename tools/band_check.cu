// Register-window banded LDL^T unit check (developer tool): factor_fwd_reg +
// forward_reg/backward_reg of band_reg.cuh against a dense CPU LDL^T on
// random 5-point SPD systems. Prints max |D - D_ref| / |D_ref| and the
// solution error per (B, NR).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/band_check tools/band_check.cu
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "../paper_2103_11050_b200/csrc/band_reg.cuh"
#include "../paper_2103_11050_b200/csrc/band_twist.cuh"

using namespace mpm2p;

template <int B, int NR>
__global__ void k_check(int n, const double* BD, const double* BW, const double* BS, double* D, double* Lc,
                        double* Lr, double* Y, int nr, int two_pass) {
    __shared__ double stage[B * B];
    __shared__ __align__(16) double xb[xchg_doubles<B, NR>()];
    __shared__ __align__(16) double ring[sweep_ring<B>() * B * B + 2];
    const BandRows A{BD, BW, BS};
    const int n0 = two_pass ? (nr < NR ? nr : NR) : nr;
    factor_fwd_reg<B, NR>(n, A, D, Lc, Lr, Y, n0, n, stage, xb);
    __syncwarp();
    if (two_pass && nr > n0) forward_reg<B, NR>(n, Lc, Y + (size_t)n0 * n, nr - n0, n, xb, ring);
    __syncwarp();
    backward_reg<B, NR>(n, D, Lr, Y, nr, n, xb, ring);
}

// Same as k_check with 4 warps per block, one independent system per warp
// (as in the solver's banded kernels); systems are copies of the same data.
template <int B, int NR>
__global__ void k_check4(int n, const double* BD, const double* BW, const double* BS, double* D, double* Lc,
                         double* Lr, double* Y, int nr) {
    __shared__ double stage[4][B * B];
    __shared__ __align__(16) double xb[4][xchg_doubles<B, NR>()];
    __shared__ __align__(16) double ring[4][sweep_ring<B>() * B * B + 2];
    const int w = threadIdx.x >> 5;
    const BandRows A{BD, BW, BS};
    double* Yw = Y + (size_t)w * nr * n;
    factor_fwd_reg<B, NR>(n, A, D + w * n, Lc + (size_t)w * n * B, Lr + (size_t)w * n * B, Yw, nr, n, stage[w], xb[w]);
    __syncwarp();
    backward_reg<B, NR>(n, D + w * n, Lr + (size_t)w * n * B, Yw, nr, n, xb[w], ring[w]);
}

// Twisted (two-sided) solve, WARPS independent copies per block.
// one team per block (blockIdx = copy index), dynamic shared memory
template <int B, int WARPS>
__global__ void k_twist(int n, const double* BD, const double* BW, const double* BS, double* D, double* Lr,
                        double* Y, double* Yv, int* okf) {
    extern __shared__ __align__(16) double sm[];
    const int w = blockIdx.x;
    const BandRows A{BD, BW, BS};
    const bool ok = twisted_solve<B>(n, A, D + w * n, Lr + (size_t)w * n * B, Y + (size_t)w * n, sm);
    if (threadIdx.x == 0) okf[w] = ok;
}

// Stored two-sided factor: factor with RHS Y (solved in place), then solve Y2 with the stored factor.
template <int B>
__global__ void k_twist_fs(int n, const double* BD, const double* BW, const double* BS, double* D, double* Lc,
                           double* Lr, double* MidB, double* Sinv, double* Y, double* Y2, int* okf) {
    extern __shared__ __align__(16) double sm[];
    const BandRows A{BD, BW, BS};
    const bool ok = twisted_factor<B>(n, A, D, Lc, Lr, MidB, Sinv, Y, sm);
    __syncthreads();
    twisted_sweep<B>(n, D, Lc, Lr, MidB, Sinv, Y2, sm);
    if (threadIdx.x == 0) okf[0] = ok;
}

template <int B, int WARPS>
void run_twist(int m) {
    const int n = B * m;
    std::mt19937_64 g(B * 7000 + m);
    std::uniform_real_distribution<double> U(0.1, 2.0);
    std::vector<double> bd(n), bw(n), bs(n), y(n);
    for (int r = 0; r < n; ++r) {
        bw[r] = (r % B) ? U(g) : 0.0;
        bs[r] = (r >= B) ? U(g) : 0.0;
    }
    for (int r = 0; r < n; ++r) {
        double s = bw[r] + bs[r] + 0.05;
        if (r % B != B - 1 && r + 1 < n) s += bw[r + 1];
        if (r + B < n) s += bs[r + B];
        bd[r] = s;
    }
    for (auto& v : y) v = U(g) - 1.0;
    // dense CPU LDL^T solve
    std::vector<double> A((size_t)n * n, 0.0);
    for (int r = 0; r < n; ++r) {
        A[(size_t)r * n + r] = bd[r];
        if (r % B) A[(size_t)r * n + r - 1] = A[(size_t)(r - 1) * n + r] = -bw[r];
        if (r >= B) A[(size_t)r * n + r - B] = A[(size_t)(r - B) * n + r] = -bs[r];
    }
    std::vector<double> x = y;
    for (int k = 0; k < n; ++k) {
        const double d = A[(size_t)k * n + k];
        const int hi = std::min(n, k + B + 1);
        for (int i = k + 1; i < hi; ++i) {
            const double l = A[(size_t)i * n + k] / d;
            for (int j = k + 1; j <= i; ++j) A[(size_t)i * n + j] -= l * A[(size_t)j * n + k];
            x[i] -= l * x[k];
        }
        for (int i = k + 1; i < hi; ++i) A[(size_t)i * n + k] /= d;
    }
    for (int i = 0; i < n; ++i) x[i] /= A[(size_t)i * n + i];
    for (int i = n - 1; i >= 0; --i)
        for (int k = i + 1; k < std::min(n, i + B + 1); ++k) x[i] -= A[(size_t)k * n + i] * x[k];
    double *dBD, *dBW, *dBS, *dD, *dLr, *dY, *dYv;
    int* dok;
    cudaMalloc(&dBD, n * 8);
    cudaMalloc(&dBW, n * 8);
    cudaMalloc(&dBS, n * 8);
    cudaMalloc(&dD, WARPS * n * 8);
    cudaMalloc(&dLr, (size_t)WARPS * n * B * 8);
    cudaMalloc(&dY, (size_t)WARPS * n * 8);
    cudaMalloc(&dYv, (size_t)WARPS * n * 8);
    cudaMalloc(&dok, WARPS * 4);
    cudaMemcpy(dBD, bd.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dBW, bw.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dBS, bs.data(), n * 8, cudaMemcpyHostToDevice);
    for (int w = 0; w < WARPS; ++w) cudaMemcpy(dY + (size_t)w * n, y.data(), n * 8, cudaMemcpyHostToDevice);
    const int smb = twist_smem_doubles<B>() * 8;
    cudaFuncSetAttribute(k_twist<B, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smb);
    cudaFuncSetAttribute(k_twist_fs<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, smb);
    k_twist<B, WARPS><<<WARPS, twist_threads<B>(), smb>>>(n, dBD, dBW, dBS, dD, dLr, dY, dYv, dok);
    cudaError_t e = cudaDeviceSynchronize();
    {  // factor + stored sweep (RHS 2 = reversed RHS 1), single warp
        double *dLc, *dMid, *dS, *dY2;
        cudaMalloc(&dLc, (size_t)n * B * 8);
        cudaMalloc(&dMid, B * B * 8);
        cudaMalloc(&dS, B * B * 8);
        cudaMalloc(&dY2, n * 8);
        std::vector<double> y2(y.rbegin(), y.rend());
        cudaMemcpy(dY, y.data(), n * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(dY2, y2.data(), n * 8, cudaMemcpyHostToDevice);
        k_twist_fs<B><<<1, twist_threads<B>(), smb>>>(n, dBD, dBW, dBS, dD, dLc, dLr, dMid, dS, dY, dY2, dok);
        cudaError_t e2 = cudaDeviceSynchronize();
        std::vector<double> x1(n), x2g(n);
        cudaMemcpy(x1.data(), dY, n * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(x2g.data(), dY2, n * 8, cudaMemcpyDeviceToHost);
        // CPU x2 from the same dense factor
        std::vector<double> x2 = y2;
        for (int i = 0; i < n; ++i)
            for (int k = std::max(0, i - B); k < i; ++k) x2[i] -= A[(size_t)i * n + k] * x2[k];
        for (int i = 0; i < n; ++i) x2[i] /= A[(size_t)i * n + i];
        for (int i = n - 1; i >= 0; --i)
            for (int k = i + 1; k < std::min(n, i + B + 1); ++k) x2[i] -= A[(size_t)k * n + i] * x2[k];
        double e1 = 0, e2m = 0, n1 = 0, n2 = 0;
        for (int i = 0; i < n; ++i) {
            e1 = std::max(e1, std::fabs(x1[i] - x[i]));
            n1 = std::max(n1, std::fabs(x[i]));
            e2m = std::max(e2m, std::fabs(x2g[i] - x2[i]));
            n2 = std::max(n2, std::fabs(x2[i]));
        }
        printf("twisted factor+sweep B=%2d rows=%3d: factor-solve rel %.2e  stored-sweep rel %.2e %s\n", B, m,
               e1 / n1, e2m / n2, cudaGetErrorString(e2));
        cudaFree(dLc); cudaFree(dMid); cudaFree(dS); cudaFree(dY2);
    }
    std::vector<double> xg((size_t)WARPS * n);
    int okh[WARPS];
    cudaMemcpy(xg.data(), dY, xg.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(okh, dok, WARPS * 4, cudaMemcpyDeviceToHost);
    double ex = 0.0, nx = 0.0;
    bool nan = false;
    for (int w = 0; w < WARPS; ++w)
        for (int i = 0; i < n; ++i) {
            const double v = xg[(size_t)w * n + i];
            if (!(v == v)) nan = true;
            ex = std::max(ex, std::fabs(v - x[i]));
            nx = std::max(nx, std::fabs(x[i]));
        }
    printf("twisted B=%2d rows=%3d warps=%d: x rel err %.2e ok=%d nan=%d %s\n", B, m, WARPS, ex / nx, okh[0], nan,
           cudaGetErrorString(e));
    cudaFree(dBD); cudaFree(dBW); cudaFree(dBS); cudaFree(dD); cudaFree(dLr); cudaFree(dY); cudaFree(dYv);
    cudaFree(dok);
}

template <int B, int NR>
void run(int m, int nr, int two_pass) {
    const int n = B * m;
    std::mt19937_64 g(B * 1000 + NR);
    std::uniform_real_distribution<double> U(0.1, 2.0);
    std::vector<double> bd(n), bw(n), bs(n), y((size_t)nr * n);
    for (int r = 0; r < n; ++r) {
        bw[r] = (r % B) ? U(g) : 0.0;
        bs[r] = (r >= B) ? U(g) : 0.0;
    }
    for (int r = 0; r < n; ++r) {
        double s = bw[r] + bs[r] + 0.05;
        if (r % B != B - 1 && r + 1 < n) s += bw[r + 1];
        if (r + B < n) s += bs[r + B];
        bd[r] = s;
    }
    for (auto& v : y) v = U(g) - 1.0;
    // dense CPU LDL^T
    std::vector<double> A((size_t)n * n, 0.0);
    for (int r = 0; r < n; ++r) {
        A[(size_t)r * n + r] = bd[r];
        if (r % B) A[(size_t)r * n + r - 1] = A[(size_t)(r - 1) * n + r] = -bw[r];
        if (r >= B) A[(size_t)r * n + r - B] = A[(size_t)(r - B) * n + r] = -bs[r];
    }
    std::vector<double> Dref(n);
    for (int k = 0; k < n; ++k) {
        const double d = A[(size_t)k * n + k];
        Dref[k] = d;
        const int hi = std::min(n, k + B + 1);
        for (int i = k + 1; i < hi; ++i) {  // rank-1 update with the unscaled column k
            const double l = A[(size_t)i * n + k] / d;
            for (int j = k + 1; j <= i; ++j) A[(size_t)i * n + j] -= l * A[(size_t)j * n + k];
        }
        for (int i = k + 1; i < hi; ++i) A[(size_t)i * n + k] /= d;
    }
    std::vector<double> xref = y;
    for (int m2 = 0; m2 < nr; ++m2) {
        double* x = xref.data() + (size_t)m2 * n;
        for (int i = 0; i < n; ++i)
            for (int k = std::max(0, i - B); k < i; ++k) x[i] -= A[(size_t)i * n + k] * x[k];
        for (int i = 0; i < n; ++i) x[i] /= Dref[i];
        for (int i = n - 1; i >= 0; --i)
            for (int k = i + 1; k < std::min(n, i + B + 1); ++k) x[i] -= A[(size_t)k * n + i] * x[k];
    }
    if (two_pass == 2) {  // 4-warp variant
        double *dBD, *dBW, *dBS, *dD, *dLc, *dLr, *dY;
        cudaMalloc(&dBD, n * 8);
        cudaMalloc(&dBW, n * 8);
        cudaMalloc(&dBS, n * 8);
        cudaMalloc(&dD, 4 * n * 8);
        cudaMalloc(&dLc, 4 * (size_t)n * B * 8);
        cudaMalloc(&dLr, 4 * (size_t)n * B * 8);
        cudaMalloc(&dY, 4 * (size_t)nr * n * 8);
        cudaMemcpy(dBD, bd.data(), n * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(dBW, bw.data(), n * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(dBS, bs.data(), n * 8, cudaMemcpyHostToDevice);
        for (int w = 0; w < 4; ++w)
            cudaMemcpy(dY + (size_t)w * nr * n, y.data(), (size_t)nr * n * 8, cudaMemcpyHostToDevice);
        k_check4<B, NR><<<1, 128>>>(n, dBD, dBW, dBS, dD, dLc, dLr, dY, nr);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<double> D(4 * n), x(4 * (size_t)nr * n);
        cudaMemcpy(D.data(), dD, 4 * n * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(x.data(), dY, 4 * (size_t)nr * n * 8, cudaMemcpyDeviceToHost);
        double ed = 0, ex = 0, nx = 0;
        for (int w = 0; w < 4; ++w) {
            for (int i = 0; i < n; ++i) ed = std::max(ed, std::fabs(D[w * n + i] - Dref[i]) / std::fabs(Dref[i]));
            for (size_t i = 0; i < (size_t)nr * n; ++i) {
                ex = std::max(ex, std::fabs(x[(size_t)w * nr * n + i] - xref[i]));
                nx = std::max(nx, std::fabs(xref[i]));
            }
        }
        printf("4-warp B=%2d NR=%2d nr=%2d n=%4d: D rel err %.2e  x rel err %.2e  %s\n", B, NR, nr, n, ed, ex / nx,
               cudaGetErrorString(e));
        return;
    }
    double *dBD, *dBW, *dBS, *dD, *dLc, *dLr, *dY;
    cudaMalloc(&dBD, n * 8);
    cudaMalloc(&dBW, n * 8);
    cudaMalloc(&dBS, n * 8);
    cudaMalloc(&dD, n * 8);
    cudaMalloc(&dLc, (size_t)n * B * 8);
    cudaMalloc(&dLr, (size_t)n * B * 8);
    cudaMalloc(&dY, (size_t)nr * n * 8);
    cudaMemcpy(dBD, bd.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dBW, bw.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dBS, bs.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dY, y.data(), (size_t)nr * n * 8, cudaMemcpyHostToDevice);
    k_check<B, NR><<<1, 32>>>(n, dBD, dBW, dBS, dD, dLc, dLr, dY, nr, two_pass);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> D(n), x((size_t)nr * n);
    cudaMemcpy(D.data(), dD, n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(x.data(), dY, (size_t)nr * n * 8, cudaMemcpyDeviceToHost);
    double ed = 0, ex = 0, nx = 0;
    int first = -1;
    for (int i = 0; i < n; ++i) {
        const double r = std::fabs(D[i] - Dref[i]) / std::fabs(Dref[i]);
        if (r > 1e-12 && first < 0) first = i;
        ed = std::max(ed, r);
    }
    for (size_t i = 0; i < x.size(); ++i) {
        ex = std::max(ex, std::fabs(x[i] - xref[i]));
        nx = std::max(nx, std::fabs(xref[i]));
    }
    printf("   D[0..2] gpu %.17g %.17g %.17g cpu %.17g %.17g %.17g | x[n-1] gpu %.17g cpu %.17g\n", D[0], D[1], D[2],
           Dref[0], Dref[1], Dref[2], x[n - 1], xref[n - 1]);
    printf("B=%2d NR=%2d nr=%2d two_pass=%d n=%4d: D rel err %.2e (first bad %d)  x rel err %.2e  %s\n", B, NR, nr,
           two_pass, n, ed, first, ex / nx, cudaGetErrorString(e));
    cudaFree(dBD);
    cudaFree(dBW);
    cudaFree(dBS);
    cudaFree(dD);
    cudaFree(dLc);
    cudaFree(dLr);
    cudaFree(dY);
}

int main() {
    run<4, 1>(8, 1, 0);
    run<16, 1>(16, 1, 0);
    run<32, 1>(32, 1, 0);
    run<16, 9>(16, 9, 0);
    run<16, 9>(16, 5, 0);
    run<32, 9>(32, 9, 0);
    run<8, 17>(8, 17, 0);
    run<8, 9>(8, 5, 0);
    run<8, 9>(8, 5, 2);
    run<16, 1>(16, 1, 2);
    run<32, 1>(32, 1, 2);
    run<32, 9>(32, 9, 2);
    run_twist<16, 1>(16);
    run_twist<16, 1>(15);
    run_twist<12, 2>(12);
    run_twist<32, 1>(32);
    run_twist<32, 1>(9);
    run_twist<20, 1>(20);
    run_twist<24, 1>(7);
    run_twist<16, 1>(3);
    run_twist<16, 1>(4);
    run_twist<8, 1>(8);
    run_twist<8, 2>(9);
    run_twist<4, 1>(8);
    run_twist<12, 1>(12);
    return 0;
}
