// The exact-order sweep's G and apply stages alone on one warp (FAST path),
// cycles per step (dev tool).
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a --fmad=false -o scripts/micro_wfstage scripts/micro_wfstage.cu
#include <cstdio>
#include "../paper_1502_03917_b200/csrc/ocmg_wavefront.cuh"
using namespace ocmg;


// variants of the G stage (same loads; H outputs per pass; split = two
// partial sums per output, one per field)
template <int H, bool SPLIT>
__device__ __forceinline__ void gvar(const WfBand &B, int F, int tau0, int nrows, double *gw) {
    using namespace wf;
    const int i = threadIdx.x & 31;
    const int ii = min(i, nrows - 1);
    const double *Wi = B.sW + 24 * 28 + F * 14;
    double w[2][7];
#pragma unroll
    for (int f = 0; f < 2; ++f)
#pragma unroll
        for (int e = 0; e < 7; ++e) w[f][e] = Wi[f * 7 + e];
#pragma unroll
    for (int h = 0; h < CW / H; ++h) {
        const int t0 = tau0 + h * H;
        double up[2][H + 1], md[2][H + 2], dn[2][H + 1];
#pragma unroll
        for (int f = 0; f < 2; ++f) {
#pragma unroll
            for (int k = 0; k <= H; ++k) {
                up[f][k] = wf_re(B, f, ii - 1, t0 - 3 + k);
                dn[f][k] = wf_re(B, f, ii + 1, t0 + 2 + k);
            }
#pragma unroll
            for (int k = 0; k < H + 2; ++k) md[f][k] = wf_re(B, f, ii, t0 - 1 + k);
        }
        double out[H];
#pragma unroll
        for (int s = 0; s < H; ++s) {
            double g[2] = {0.0, 0.0};
#pragma unroll
            for (int f = 0; f < 2; ++f) {
                double &a = g[SPLIT ? f : 0];
                a = fma(w[f][0], up[f][s], a);
                a = fma(w[f][1], up[f][s + 1], a);
                a = fma(w[f][2], md[f][s], a);
                a = fma(w[f][3], md[f][s + 1], a);
                a = fma(w[f][4], md[f][s + 2], a);
                a = fma(w[f][5], dn[f][s], a);
                a = fma(w[f][6], dn[f][s + 1], a);
            }
            out[s] = SPLIT ? g[0] + g[1] : g[0];
        }
#pragma unroll
        for (int s = 0; s < H; ++s) gw[ii * SS + ((t0 + s) & (WS - 1))] = out[s];
    }
}

template <int MODE>
__global__ void k(long long *out, int iters, int n1) {
    extern __shared__ __align__(16) double sm[];
    using namespace wf;
    for (int t = threadIdx.x; t < SM_TOTAL; t += blockDim.x) sm[t] = 1e-3 * (t % 11);
    __syncthreads();
    WfBand B{};
    B.n1 = n1;
    B.iy0 = 100;
    B.nreal = 29;
    B.N = (int64_t)n1 * n1;
    B.sA = sm;
    B.sW = sm + kP1Classes * 28;
    B.sN = sm + SM_AW;
    B.re = sm + SM_AW + SM_N;
    B.xw = B.re + SM_RE;
    B.g1 = B.xw + SM_X;
    B.p1 = B.g1 + SM_G1;
    B.g2 = B.p1 + SM_P1;
    B.p2 = B.g2 + SM_G2;
    long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int t0 = 8 * (it + 20);
        if (MODE == 0) wf_gstage<false, true>(B, 0, t0, 32, B.g1, nullptr);
        if (MODE == 1) wf_astage<false, true>(B, 0, t0, 31, B.p1, 32, nullptr, 2);
        if (MODE == 2) gvar<4, false>(B, 0, t0, 32, B.g1);
        if (MODE == 3) gvar<4, true>(B, 0, t0, 32, B.g1);
        if (MODE == 4) gvar<8, false>(B, 0, t0, 32, B.g1);
        if (MODE == 5) gvar<8, true>(B, 0, t0, 32, B.g1);
    }
    long long c1 = clock64();
    if (threadIdx.x == 0) out[MODE] = c1 - c0;
}

int main() {
    long long *out;
    cudaMallocManaged(&out, 16 * sizeof(long long));
    const int iters = 200;
    cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wf::SM_BYTES);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wf::SM_BYTES);
    cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wf::SM_BYTES);
    cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wf::SM_BYTES);
    cudaFuncSetAttribute(k<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wf::SM_BYTES);
    cudaFuncSetAttribute(k<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wf::SM_BYTES);
    for (int rep = 0; rep < 2; ++rep) {
        k<0><<<1, 32, wf::SM_BYTES>>>(out, iters, 4097);
        k<1><<<1, 32, wf::SM_BYTES>>>(out, iters, 4097);
        k<2><<<1, 32, wf::SM_BYTES>>>(out, iters, 4097);
        k<3><<<1, 32, wf::SM_BYTES>>>(out, iters, 4097);
        k<4><<<1, 32, wf::SM_BYTES>>>(out, iters, 4097);
        k<5><<<1, 32, wf::SM_BYTES>>>(out, iters, 4097);
        cudaDeviceSynchronize();
    }
    printf("G stage:     %.1f cycles/step\n", out[0] / (8.0 * iters));
    printf("apply stage: %.1f cycles/step\n", out[1] / (8.0 * iters));
    printf("G H=4 plain stores:   %.1f\n", out[2] / (8.0 * iters));
    printf("G H=4 split sums:     %.1f\n", out[3] / (8.0 * iters));
    printf("G H=8:                %.1f\n", out[4] / (8.0 * iters));
    printf("G H=8 split sums:     %.1f\n", out[5] / (8.0 * iters));
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
