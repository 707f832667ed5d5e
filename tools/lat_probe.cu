// Dependent-chain latency probe (developer tool): cycles per op for the
// instructions on the banded-LDL^T pivot critical path.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_probe tools/lat_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 1024;

__global__ void probe(double seed, long long* out, double* sink) {
    __shared__ double sm[64];
    const int lane = threadIdx.x;
    double x = seed + lane * 1e-9;
    sm[lane] = x;
    sm[lane + 32] = x;
    __syncwarp();
    long long t0, t1;
    // 1. DFMA chain
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = fma(x, 0.999999, 1e-7);
    t1 = clock64();
    out[0] = t1 - t0;
    // 2. 64-bit SHFL chain (broadcast from a varying lane)
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (lane + i + 1) & 31);
    t1 = clock64();
    out[1] = t1 - t0;
    // 3. rcp.approx + 2 Newton steps chain
    t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N; ++i) {
        double r;
        asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
        double e = fma(-x, r, 1.0);
        r = fma(r, e, r);
        e = fma(-x, r, 1.0);
        r = fma(r, e, r);
        x = r + 1.0;
    }
    t1 = clock64();
    out[2] = t1 - t0;
    // 4. IEEE division chain
    t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N; ++i) x = 1.0 / x + 1.0;
    t1 = clock64();
    out[3] = t1 - t0;
    // 5. STS + syncwarp + LDS (broadcast) chain
    t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N; ++i) {
        sm[lane] = x;
        __syncwarp();
        x = sm[(lane + i) & 31] + 1e-9;
        __syncwarp();
    }
    t1 = clock64();
    out[4] = t1 - t0;
    // 6. 32-bit SHFL chain
    float f = (float)x;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) f = __shfl_sync(0xffffffffu, f, (lane + i + 1) & 31);
    t1 = clock64();
    out[5] = t1 - t0;
    // 7. DMUL chain
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = x * 0.9999999;
    t1 = clock64();
    out[6] = t1 - t0;
    // 8. throughput: 16 independent DFMA chains
    double y[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) y[j] = x + j;
    t0 = clock64();
    for (int i = 0; i < N / 16; ++i) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int j = 0; j < 16; ++j) y[j] = fma(y[j], 0.999999, 1e-7);
    }
    t1 = clock64();
    out[7] = t1 - t0;
    // 9. throughput: 16 independent 64-bit shuffles per iteration
    t0 = clock64();
    for (int i = 0; i < N / 16; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) y[j] = __shfl_sync(0xffffffffu, y[j], (lane + j + i) & 31);
    }
    t1 = clock64();
    out[8] = t1 - t0;
    // 10. DMMA (mma.sync m8n8k4 f64) dependent chain through the accumulator
    double d0 = x, d1 = x;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                     : "+d"(d0), "+d"(d1)
                     : "d"(0.5), "d"(0.25));
    t1 = clock64();
    out[9] = t1 - t0;
    // 11. DMMA throughput: 8 independent accumulators
    double acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = x;
    t0 = clock64();
    for (int i = 0; i < N / 8; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(acc[2 * j]), "+d"(acc[2 * j + 1])
                         : "d"(0.5), "d"(0.25));
    }
    t1 = clock64();
    out[10] = t1 - t0;
    double s = x + f + d0 + d1;
#pragma unroll
    for (int j = 0; j < 16; ++j) s += acc[j];
#pragma unroll
    for (int j = 0; j < 16; ++j) s += y[j];
    sink[lane] = s;
}

int main() {
    long long* d_out;
    double* d_sink;
    cudaMalloc(&d_out, 16 * sizeof(long long));
    cudaMalloc(&d_sink, 64 * sizeof(double));
    for (int rep = 0; rep < 2; ++rep) probe<<<1, 32>>>(1.5, d_out, d_sink);
    long long h[16];
    cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
    const char* names[] = {"DFMA dep", "SHFL64 dep", "RCP64+2Newton+DADD dep", "IEEE div dep", "STS+LDS bcast dep",
                           "SHFL32 dep", "DMUL dep", "DFMA thrpt (per warp-instr)", "SHFL64 thrpt (per shfl64)",
                           "DMMA.884 dep", "DMMA.884 thrpt (1 warp)"};
    const double per[] = {N, N, N, N, N, N, N, 16.0 * N, N, N, N};
    for (int i = 0; i < 11; ++i) printf("%-32s %8.2f cycles\n", names[i], h[i] / per[i]);
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
