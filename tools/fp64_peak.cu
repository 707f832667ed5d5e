// Measures fp64 DFMA and DMMA (mma.sync m8n8k4 f64) peak throughput on the box.
// These are the fp64 roofline denominators (MEASURED_PEAKS.json has none).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void dmma_kernel(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 - a;
    double c[4][2];
    for (int t = 0; t < 4; ++t) { c[t][0] = 0; c[t][1] = 0; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
#pragma unroll
            for (int t = 0; t < 4; ++t)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
        }
    }
    double s = 0;
    for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}

int main() {
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    printf("device %s SMs %d cc %d.%d clock %d kHz\n", p.name, p.multiProcessorCount, p.major, p.minor, p.clockRate);
    double* out; cudaMalloc(&out, 148 * 64 * 1024 * sizeof(double));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4096;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
        printf("DFMA: %.3f ms  %.2f TFLOP/s\n", ms, flops / ms / 1e9);
    }
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        dmma_kernel<<<blocks, threads>>>(out, iters / 4);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8 * 8 * 4 * 16 * 4 * (double)(iters / 4) * blocks * (threads / 32);
        printf("DMMA m8n8k4: %.3f ms  %.2f TFLOP/s\n", ms, flops / ms / 1e9);
    }
    size_t n = (size_t)1 << 28;  // 4 GiB per buffer of double2? 2^28 * 16 B = 4 GiB
    double2 *a, *b; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16);
    cudaMemset(a, 0, n * 16);
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        copy_kernel<<<p.multiProcessorCount * 16, 512>>>(a, b, n);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("copy: %.3f ms  %.1f GB/s\n", ms, 2.0 * n * 16 / ms / 1e6);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
