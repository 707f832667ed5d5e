// Blocked banded LDL^T micro-benchmark (developer tool): band_blk.cuh's
// blk_factor_fwd (3 and 4 blocks per SM; the product's variant and the one with
// the entering row tile on DMMA) and blk_backward on random
// 5-point SPD systems, one warp per system, the product kernel's launch shape
// (4 warps per block). Checks the solution's residual on the host, that the
// two builds' panels are bit-identical, and times the factor kernels.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -o tools/blk_bench tools/blk_bench.cu
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "../paper_2103_11050_b200/csrc/band_blk.cuh"

using namespace mpm2p;
constexpr int WPBK = 4;

template <int B, int V, int MINB>
__global__ void __launch_bounds__(WPBK * 32, MINB) k_factor(int nsub, int n, const double* BD, const double* BW,
                                                           const double* BS, const double* Y, double* Xs, double* Ts,
                                                           int* bad) {
    __shared__ __align__(16) double sm[WPBK][blk_smem_doubles<B>()];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = blockIdx.x * WPBK + w;
    if (s >= nsub) return;
    const size_t so = (size_t)s * n;
    const BlkBandSrc src{BandRows{BD + so, BW + so, BS + so}, Y + so, n};
    bool ok;
    ok = blk_factor_fwd<B, BlkBandSrc, V == 0>(n, src, Xs + so * B, Ts + so, sm[w]);
    if (!ok && lane == 0) atomicAdd(bad, 1);
}

template <int B>
__global__ void __launch_bounds__(WPBK * 32) k_back(int nsub, int n, const double* Xs, const double* Ts, double* X) {
    const int w = threadIdx.x >> 5;
    const int s = blockIdx.x * WPBK + w;
    if (s >= nsub) return;
    const size_t so = (size_t)s * n;
    blk_backward<B>(n, Xs + so * B, Ts + so, X + so);
}

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e_ = (x);                                                       \
        if (e_ != cudaSuccess) {                                                    \
            printf("CUDA error %s at line %d\n", cudaGetErrorString(e_), __LINE__); \
            return 1;                                                               \
        }                                                                           \
    } while (0)

template <int B>
int run(int nsub) {
    const int n = B * B;
    const size_t N = (size_t)nsub * n;
    std::vector<double> bd(N), bw(N), bs(N), y(N);
    std::mt19937_64 rng(12345);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    // 5-point operator with log-uniform couplings over three decades; diag =
    // sum of the four couplings (+1 on row 0: the anchor)
    const int nu = nsub < 8 ? nsub : 8;  // distinct systems, tiled
    for (int s = 0; s < nu; ++s) {
        double* d = &bd[(size_t)s * n];
        double* w = &bw[(size_t)s * n];
        double* so = &bs[(size_t)s * n];
        for (int r = 0; r < n; ++r) {
            w[r] = (r % B) ? std::pow(10.0, 3.0 * U(rng) - 1.5) : 0.0;
            so[r] = (r >= B) ? std::pow(10.0, 3.0 * U(rng) - 1.5) : 0.0;
            y[(size_t)s * n + r] = U(rng) - 0.5;
        }
        for (int r = 0; r < n; ++r) {
            double dd = w[r] + so[r];
            if (r + 1 < n) dd += w[r + 1];
            if (r + B < n) dd += so[r + B];
            d[r] = dd + (r == 0 ? 1.0 : 0.0);
        }
    }
    for (int s = nu; s < nsub; ++s) {
        std::memcpy(&bd[(size_t)s * n], &bd[(size_t)(s % nu) * n], n * 8);
        std::memcpy(&bw[(size_t)s * n], &bw[(size_t)(s % nu) * n], n * 8);
        std::memcpy(&bs[(size_t)s * n], &bs[(size_t)(s % nu) * n], n * 8);
        std::memcpy(&y[(size_t)s * n], &y[(size_t)(s % nu) * n], n * 8);
    }
    double *dBD, *dBW, *dBS, *dY, *dXs[2], *dTs[2], *dX;
    int* dbad;
    CK(cudaMalloc(&dBD, N * 8));
    CK(cudaMalloc(&dBW, N * 8));
    CK(cudaMalloc(&dBS, N * 8));
    CK(cudaMalloc(&dY, N * 8));
    CK(cudaMalloc(&dX, N * 8));
    for (int v = 0; v < 2; ++v) {
        CK(cudaMalloc(&dXs[v], N * B * 8));
        CK(cudaMalloc(&dTs[v], N * 8));
    }
    CK(cudaMalloc(&dbad, 4));
    CK(cudaMemset(dbad, 0, 4));
    CK(cudaMemcpy(dBD, bd.data(), N * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dBW, bw.data(), N * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dBS, bs.data(), N * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dY, y.data(), N * 8, cudaMemcpyHostToDevice));
    const int blocks = (nsub + WPBK - 1) / WPBK;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](auto launch, const char* name) {
        for (int i = 0; i < 2; ++i) launch();
        cudaEventRecord(e0);
        const int reps = 5;
        for (int i = 0; i < reps; ++i) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("B=%d nsub=%d %-28s %9.1f us\n", B, nsub, name, 1e3 * ms / reps);
        return 0;
    };
    timeit([&] { k_factor<B, 1, 3><<<blocks, WPBK * 32>>>(nsub, n, dBD, dBW, dBS, dY, dXs[0], dTs[0], dbad); },
           "blk_factor_fwd (3 blk/SM)");
    timeit([&] { k_factor<B, 1, 4><<<blocks, WPBK * 32>>>(nsub, n, dBD, dBW, dBS, dY, dXs[1], dTs[1], dbad); },
           "blk_factor_fwd (4 blk/SM)");
    timeit([&] { k_factor<B, 0, 3><<<blocks, WPBK * 32>>>(nsub, n, dBD, dBW, dBS, dY, dXs[1], dTs[1], dbad); },
           "NTD variant (3 blk/SM)");
    timeit([&] { k_factor<B, 0, 4><<<blocks, WPBK * 32>>>(nsub, n, dBD, dBW, dBS, dY, dXs[1], dTs[1], dbad); },
           "NTD variant (4 blk/SM)");
    k_factor<B, 1, 4><<<blocks, WPBK * 32>>>(nsub, n, dBD, dBW, dBS, dY, dXs[1], dTs[1], dbad);
    timeit([&] { k_back<B><<<blocks, WPBK * 32>>>(nsub, n, dXs[1], dTs[1], dX); }, "blk_backward");
    CK(cudaDeviceSynchronize());
    int bad;
    CK(cudaMemcpy(&bad, dbad, 4, cudaMemcpyDeviceToHost));
    // bit-identity of the panels of the first nu systems
    const size_t cmp = (size_t)nu * n;
    std::vector<double> a(cmp * B), b(cmp * B), ta(cmp), tb(cmp);
    CK(cudaMemcpy(a.data(), dXs[0], cmp * B * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b.data(), dXs[1], cmp * B * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ta.data(), dTs[0], cmp * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(tb.data(), dTs[1], cmp * 8, cudaMemcpyDeviceToHost));
    const bool same = !std::memcmp(a.data(), b.data(), cmp * B * 8) && !std::memcmp(ta.data(), tb.data(), cmp * 8);
    // residual of the lookahead variant's solution
    k_back<B><<<blocks, WPBK * 32>>>(nsub, n, dXs[1], dTs[1], dX);
    CK(cudaDeviceSynchronize());
    std::vector<double> x(cmp);
    CK(cudaMemcpy(x.data(), dX, cmp * 8, cudaMemcpyDeviceToHost));
    double rmax = 0.0, ymax = 0.0;
    for (int s = 0; s < nu; ++s) {
        const double* d = &bd[(size_t)s * n];
        const double* w = &bw[(size_t)s * n];
        const double* so = &bs[(size_t)s * n];
        const double* xx = &x[(size_t)s * n];
        for (int r = 0; r < n; ++r) {
            double ax = d[r] * xx[r];
            if (r % B) ax -= w[r] * xx[r - 1];
            if ((r + 1) % B && r + 1 < n) ax -= w[r + 1] * xx[r + 1];
            if (r >= B) ax -= so[r] * xx[r - B];
            if (r + B < n) ax -= so[r + B] * xx[r + B];
            rmax = std::fmax(rmax, std::fabs(ax - y[(size_t)s * n + r]));
            ymax = std::fmax(ymax, std::fabs(y[(size_t)s * n + r]));
        }
    }
    printf("B=%d: not-SPD flags %d, panels bit-identical: %s, max residual %.3e (|y| max %.3e)\n", B, bad,
           same ? "yes" : "NO", rmax, ymax);
    cudaFree(dBD), cudaFree(dBW), cudaFree(dBS), cudaFree(dY), cudaFree(dX), cudaFree(dbad);
    for (int v = 0; v < 2; ++v) cudaFree(dXs[v]), cudaFree(dTs[v]);
    return 0;
}

int main(int argc, char** argv) {
    const int nsub = argc > 1 ? atoi(argv[1]) : 16384;
    if (run<32>(nsub)) return 1;
    if (run<16>(nsub)) return 1;
    if (run<24>(nsub)) return 1;
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
