// Grid-barrier cost probe (developer tool): one CTA per SM, co-resident via a
// cooperative launch, `steps` barriers of the k_bt_persist kind, optionally
// with a dependent vector read from L2 after each one.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bar_probe tools/bar_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void bar_fence(unsigned* ctr, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1u);
        unsigned v;
        do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while (v < target);
    }
    __syncthreads();
}
__device__ __forceinline__ void bar_release(unsigned* ctr, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        unsigned v;
        do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while (v < target);
    }
    __syncthreads();
}

template <int MODE>
__global__ void probe(unsigned* ctr, int steps, double* vec, double* out) {
    const unsigned G = gridDim.x;
    double acc = 0.0;
    for (int t = 0; t < steps; ++t) {
        if (MODE >= 2) {  // dependent L2 vector read + a write, like a block step
            acc += __ldcg(vec + ((t * 37 + threadIdx.x) & 1023));
            if (threadIdx.x == 0) vec[1024 + blockIdx.x] = acc;
        }
        if (MODE == 0 || MODE == 2) bar_fence(ctr, (unsigned)(t + 1) * G);
        else bar_release(ctr, (unsigned)(t + 1) * G);
    }
    if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned* ctr;
    double *vec, *out;
    cudaMalloc(&ctr, 4);
    cudaMalloc(&vec, 8 * 4096);
    cudaMalloc(&out, 8 * 4096);
    cudaMemset(vec, 0, 8 * 4096);
    int steps = 2000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](auto kern, const char* name, int grid) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemset(ctr, 0, 4);
            void* args[] = {&ctr, &steps, &vec, &out};
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)kern, grid, 256, args, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep == 2) printf("%-28s grid %4d: %.3f us per barrier\n", name, grid, 1e3 * ms / steps);
        }
    };
    for (int g : {sms, 64, 16}) {
        run(probe<0>, "fence+atomicAdd", g);
        run(probe<1>, "red.release", g);
        run(probe<2>, "fence+atomicAdd + L2 read", g);
        run(probe<3>, "red.release + L2 read", g);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
