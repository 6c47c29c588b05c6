// The exact-order sweep's chain stage (wf_chain, FAST path) alone on one
// warp, cycles per step, and variants of its step (dev tool).
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a --fmad=false -o scripts/micro_wfchain scripts/micro_wfchain.cu
#include <cstdio>
#include "../paper_1502_03917_b200/csrc/ocmg_wavefront.cuh"
using namespace ocmg;

// V bits: 1 plain smem stores (no asm), 2 no inv select, 4 no v2 shuffle,
// 8 stores inside the step loop
template <int V>
__device__ __forceinline__ void chain_var(WfChain &S, const double (&K)[10], int tau0, int n1,
                                          const double *gw, double *pw) {
    using namespace wf;
    const int i = threadIdx.x & 31;
    double g[CW], e1[CW], e2[CW];
#pragma unroll
    for (int s = 0; s < CW; ++s) {
        const int sl = (tau0 + s) & (WS - 1);
        g[s] = gw[i * SS + ((tau0 + s + 6) & (WS - 1))];
        e1[s] = pw[1 * SS + sl];
        e2[s] = pw[0 * SS + sl];
    }
    double pout[CW];
#pragma unroll
    for (int s = 0; s < CW; ++s) {
        const int tau = tau0 + s;
        const int x = tau - 2 * i;
        const double inv = (V & 2) ? K[9] : wf_sel((unsigned)x < (unsigned)n1, K[9], 0.0);
        double a = fma(K[8], S.pprev, S.acc[0]);
        a = fma(K[6], S.v1prev, a);
        const double p = a * inv;
        pout[s] = p;
        if (V & 8) pw[(i + 2) * SS + (tau & (WS - 1))] = p;
        const double u1 = __shfl_up_sync(0xffffffffu, p, 1);
        const double u2 = (V & 4) ? S.v1prev : __shfl_up_sync(0xffffffffu, p, 2);
        const double v1 = wf_sel(i == 0, e1[s], u1);
        const double v2 = wf_sel(i == 0, e2[s], wf_sel(i == 1, e1[s], u2));
        double a2 = fma(K[7], p, S.acc[2]);
        a2 = fma(K[5], v1, a2);
        const double a3 = fma(K[4], v1, S.acc[3]);
        double a4 = fma(K[3], v1, S.acc[4]);
        a4 = fma(K[2], v2, a4);
        const double a5 = fma(K[1], v2, S.acc[5]);
        const double a6 = fma(K[0], v2, g[s]);
        S.acc[0] = S.acc[1];
        S.acc[1] = a2;
        S.acc[2] = a3;
        S.acc[3] = a4;
        S.acc[4] = a5;
        S.acc[5] = a6;
        S.pprev = p;
        S.v1prev = v1;
    }
    if (!(V & 8)) {
#pragma unroll
        for (int s = 0; s < CW; ++s) {
            double *q = pw + (i + 2) * SS + ((tau0 + s) & (WS - 1));
            if (V & 1)
                *q = pout[s];
            else
                wf_sts(q, pout[s], true);
        }
    }
}

template <int MODE, int V>
__global__ void k(long long *out, double *sink, int iters, int n1) {
    __shared__ double g1[wf::SM_G1], p1[wf::SM_P1];
    for (int t = threadIdx.x; t < wf::SM_G1; t += blockDim.x) g1[t] = 1e-3 * (t % 7);
    for (int t = threadIdx.x; t < wf::SM_P1; t += blockDim.x) p1[t] = 1e-3 * (t % 5);
    __syncthreads();
    WfBand B{};
    B.n1 = n1;
    B.iy0 = 100;
    B.nreal = 29;
    B.hsink = sink + (1 << 19);
    WfChain S;
    for (int m = 0; m < 7; ++m) S.acc[m] = 0.0;
    S.pprev = S.v1prev = 0.0;
    double K[10];
    for (int m = 0; m < 10; ++m) K[m] = -0.01 * (m + 1);
    K[9] = 0.5;
    long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int t0 = 8 * (it + 20);
        if (MODE < 2)
            wf_chain<false, true>(B, S, K, t0, 0, 36, 32, g1, p1, MODE ? sink : nullptr, 0);
        else
            chain_var<V>(S, K, t0, n1, g1, p1);
    }
    long long c1 = clock64();
    if (threadIdx.x == 0) out[MODE * 16 + V] = c1 - c0;
    sink[threadIdx.x] += S.pprev + S.acc[1];
}

int main() {
    long long *out;
    double *sink;
    cudaMallocManaged(&out, 64 * sizeof(long long));
    cudaMalloc(&sink, (1 << 20) * sizeof(double));
    const int iters = 200;
    for (int rep = 0; rep < 2; ++rep) {
        k<0, 0><<<1, 32>>>(out, sink, iters, 4097);
        k<1, 0><<<1, 32>>>(out, sink, iters, 4097);
        k<2, 0><<<1, 32>>>(out, sink, iters, 4097);
        k<2, 1><<<1, 32>>>(out, sink, iters, 4097);
        k<2, 3><<<1, 32>>>(out, sink, iters, 4097);
        k<2, 7><<<1, 32>>>(out, sink, iters, 4097);
        k<2, 9><<<1, 32>>>(out, sink, iters, 4097);
        cudaDeviceSynchronize();
    }
    const double st = 8.0 * iters;
    printf("wf_chain FAST, no hand-off stores: %.1f cycles/step\n", out[0] / st);
    printf("wf_chain FAST, hand-off stores:    %.1f cycles/step\n", out[16] / st);
    printf("variant 0 (asm stores):            %.1f\n", out[32] / st);
    printf("variant 1 (plain stores):          %.1f\n", out[33] / st);
    printf("variant 3 (+ no inv select):       %.1f\n", out[35] / st);
    printf("variant 7 (+ no v2 shuffle):       %.1f\n", out[39] / st);
    printf("variant 9 (plain, stores in loop): %.1f\n", out[41] / st);
    return 0;
}
