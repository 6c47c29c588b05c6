// Microbenchmark of the wavefront stage functions in isolation (no band
// synchronization): times one call of each interior fast path per warp.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a --fmad=false
//        -o scripts/micro_wf scripts/micro_wf.cu
#include <cstdio>
#include <vector>

#include "../paper_1502_03917_b200/csrc/ocmg_wavefront.cuh"

using namespace ocmg;

template <int which>
__global__ void __launch_bounds__(wf::NTHREADS, 1)
k_micro(WfParams P, int reps, int nhelp, unsigned long long *out) {
    using namespace wf;
    extern __shared__ double sm[];
    __shared__ WfCtx ctx;
    double *sAW = sm, *sWF = sAW + SM_AW;
    double *g1 = sWF + SM_WF + 2 * SM_WIN + 2 * SM_EXT;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        ctx.P = P;
        ctx.b = blockIdx.x + 1;
        ctx.iy0 = ctx.b * REAL;
        ctx.nreal = REAL;
        ctx.N = (int64_t)P.n1 * P.n1;
        ctx.ps1 = (int64_t)ROWS * RW;
        ctx.psu = 2 * (int64_t)ROWS * RW;
        ctx.sAW = sAW;
        ctx.sWF = sWF;
    }
    for (int t = threadIdx.x; t < SM_AW + SM_WF; t += blockDim.x) sm[t] = 0.001;
    __syncthreads();
    const int hw = warp - 2;
    const int rloG = hw >= 0 ? (hw % NW_G) * HR_G : 0;
    const int rloA = hw >= 0 ? (hw % NW_A) * HR_A : 0;
    unsigned long long t0, t1;
    __syncthreads();
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    for (int r = 0; r < reps; ++r) {
        const int j = 4 + (r % 100);
        if (which < 3 && hw >= 0 && hw < nhelp) {
            if (which == 0)
                wf_stage_G<false, HR_G>(&ctx, j, 0, g1, 0, rloG, ROWS);
            else if (which == 1)
                wf_stage_apply<false, HR_A>(&ctx, j, 0, 0, ROWS, 0, 0, rloA, ROWS_U);
            else if (which == 2)
                wf_stage_G<false, HR_G>(&ctx, j, 1, g1, 1, rloG, ROWS_G2);
        }
        if (which == 3 && warp == 0)
            wf_chain<false>(&ctx, j, 0, 36, ROWS, sm + SM_AW + SM_WF,
                            sm + SM_AW + SM_WF + 2 * SM_WIN, g1, P.ring1);
        if (which == 4) {  // the real kernel's warp mix, no band sync
            if (warp == 0)
                wf_chain<false>(&ctx, j, 0, 36, ROWS, sm + SM_AW + SM_WF,
                                sm + SM_AW + SM_WF + 2 * SM_WIN, g1, P.ring1);
            else if (warp == 1)
                wf_chain<false>(&ctx, j, 9, 37, ROWS_C2, sm + SM_AW + SM_WF + SM_WIN,
                                sm + SM_AW + SM_WF + 2 * SM_WIN + SM_EXT, g1 + SM_G, P.ring2);
            else if (hw < 2)
                wf_stage_G<false, HR_G>(&ctx, j, 0, g1, 0, hw * 16, ROWS);
            else if (hw < 4)
                wf_stage_apply<false, HR_A>(&ctx, j, 0, 0, ROWS, 0, 0, (hw - 2) * 16, ROWS_U);
            else if (hw < 6)
                wf_stage_G<false, HR_G>(&ctx, j, 1, g1 + SM_G, 1, (hw - 4) * 16, ROWS_G2);
            else
                wf_stage_apply<false, HR_A>(&ctx, j, 1, 1, ROWS_C2, 1, 1, (hw - 6) * 16, REAL);
        }
        __syncthreads();
    }
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
    using namespace wf;
    const int k = 12, n1 = (1 << k) + 1;
    const int64_t N = (int64_t)n1 * n1;
    const int nb = (n1 + REAL - 1) / REAL;
    double *x, *r, *ring1, *ring2, *ringu;
    cudaMalloc(&x, 2 * N * 8);
    cudaMalloc(&r, 2 * N * 8);
    cudaMemset(x, 0, 2 * N * 8);
    cudaMemset(r, 0, 2 * N * 8);
    const size_t plane = (size_t)nb * ROWS * RW;
    cudaMalloc(&ring1, plane * 8);
    cudaMalloc(&ring2, plane * 8);
    cudaMalloc(&ringu, 2 * plane * 8);
    cudaMemset(ring1, 0, plane * 8);
    cudaMemset(ring2, 0, plane * 8);
    cudaMemset(ringu, 0, 2 * plane * 8);
    unsigned long long *out;
    cudaMalloc(&out, 1024 * 8);
    WfParams P{};
    P.n1 = n1;
    P.nb = nb;
    P.x = x;
    P.r = r;
    P.ring1 = ring1;
    P.ring2 = ring2;
    P.ringu = ringu;
    cudaFuncSetAttribute(k_micro<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)SM_BYTES);
    cudaFuncSetAttribute(k_micro<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)SM_BYTES);
    cudaFuncSetAttribute(k_micro<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)SM_BYTES);
    cudaFuncSetAttribute(k_micro<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)SM_BYTES);
    cudaFuncSetAttribute(k_micro<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)SM_BYTES);
    const char *names[] = {"G1 stage (r source)", "u stage (apply)",
                           "G2 stage (ring source)", "chain (32 steps)",
                           "all stages together"};
    for (int grid : {1, 140}) {
      for (int nhelp : {1, 2}) {
        for (int which = 0; which < 5; ++which) {
            if (which >= 3 && nhelp != 1) continue;
            const int reps = 200;
            if (which == 0) k_micro<0><<<grid, NTHREADS, SM_BYTES>>>(P, reps, nhelp, out);
            if (which == 1) k_micro<1><<<grid, NTHREADS, SM_BYTES>>>(P, reps, nhelp, out);
            if (which == 2) k_micro<2><<<grid, NTHREADS, SM_BYTES>>>(P, reps, nhelp, out);
            if (which == 3) k_micro<3><<<grid, NTHREADS, SM_BYTES>>>(P, reps, nhelp, out);
            if (which == 4) k_micro<4><<<grid, NTHREADS, SM_BYTES>>>(P, reps, nhelp, out);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("error %s\n", cudaGetErrorString(e));
                return 1;
            }
            std::vector<unsigned long long> h(grid);
            cudaMemcpy(h.data(), out, grid * 8, cudaMemcpyDeviceToHost);
            double mx = 0;
            for (auto v : h) mx = v > mx ? v : mx;
            printf("grid %3d helpers %2d %-24s %8.3f us per call\n", grid, nhelp,
                   names[which], mx / 1e3 / reps);
        }
      }
    }
    return 0;
}
