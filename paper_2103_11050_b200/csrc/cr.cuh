// cr.cuh — the cyclic-reduction block-tridiagonal solver (blocktri.cu) seen
// from other files: one batched-GEMV job, and the solve run inside a
// persistent cooperative kernel (phases separated by grid barriers).
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace mpm2p {

// out = base + s1 M1 v1 (+ s2 M2 v2), M S x S row-major (any pointer may be null)
struct GemvJob {
    double* out;
    const double* base;
    const double* M1;
    const double* v1;
    const double* M2;
    const double* v2;
    double s1, s2;
};

// The solve's phases (forward levels, top block, backward levels) inside a
// persistent kernel: every warp of the grid takes rows of the phase's jobs;
// vectors written by other blocks in earlier phases are read through L2.
__device__ __forceinline__ void cr_solve_in_kernel(const GemvJob* jobs, const int2* phases, int nphase, int S,
                                                   cooperative_groups::grid_group& grid) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (int ph = 0; ph < nphase; ++ph) {
        const int2 pf = phases[ph];
        const long long rows = (long long)pf.y * S;
        for (long long x = gw; x < rows; x += nw) {
            const GemvJob jb = jobs[pf.x + (int)(x / S)];
            const int r = (int)(x % S);
            double a1 = 0.0, a2 = 0.0;
            if (jb.M1)
                for (int c = lane; c < S; c += 32) a1 = fma(jb.M1[(size_t)r * S + c], __ldcg(jb.v1 + c), a1);
            if (jb.M2)
                for (int c = lane; c < S; c += 32) a2 = fma(jb.M2[(size_t)r * S + c], __ldcg(jb.v2 + c), a2);
            a1 = warp_sum(a1);
            a2 = warp_sum(a2);
            if (lane == 0) jb.out[r] = (jb.base ? __ldcg(jb.base + r) : 0.0) + jb.s1 * a1 + jb.s2 * a2;
        }
        grid.sync();
    }
}

}  // namespace mpm2p
