// Cycles per step of the multicolour vertex update (both unknowns,
// node_update_u arithmetic, coefficients as kernel parameters) on W warps of
// an SM, in the variants that separate the hardware's cost from the sweep
// kernels' (dev tool):
//   KV vertices per lane (independent chains), NL/NS 16-byte shared-memory
//   loads / stores per vertex with the lanes LS bytes apart, a CTA barrier
//   per step, G CTAs (1 or one per SM), DS bytes of dynamic shared memory.
// nvcc -O3 --fmad=false -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/micro_node scripts/micro_node.cu
#include <cstdio>
struct Cf { double c[20]; };
__device__ __forceinline__ double upd(double2 (&v)[7], const double *c, int o) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int d = 0; d < 7; ++d) {
        s0 = __fma_rn(c[(o + d) % 19], v[d].x, s0);
        s1 = __fma_rn(c[(o + 3 + d) % 19], v[d].y, s1);
    }
    const double p = __dmul_rn(__dadd_rn(s0, s1), c[19]);
#pragma unroll
    for (int d = 0; d < 7; ++d)
        v[d] = make_double2(__fma_rn(-c[(o + 5 + d) % 19], p, v[d].x), __fma_rn(-c[(o + 9 + d) % 19], p, v[d].y));
    return p;
}
template <int KV, int NL, int LS, bool BAR>
__global__ void k(long long *out, const __grid_constant__ Cf C, int n, double *sink) {
    extern __shared__ __align__(16) double2 sh[];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) sh[i] = make_double2(1e-3 * i, 1.0);
    __syncthreads();
    double2 v[KV][7];
    for (int j = 0; j < KV; ++j)
        for (int d = 0; d < 7; ++d) v[j][d] = make_double2(threadIdx.x + d + j, 1.0 / (1 + d));
    double acc = 0;
    // lane's base: warps 4 KB apart (wrapped), lanes LS bytes apart
    char *base = reinterpret_cast<char *>(sh) + ((threadIdx.x / 32) * 4096) % 16384 + (threadIdx.x % 32) * LS;
    long long c0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int j = 0; j < KV; ++j)
#pragma unroll
            for (int d = 0; d < NL; ++d)
                v[j][d] = *reinterpret_cast<double2 *>(base + 16 * d + 8192 * j + (i & 1) * 16384);
#pragma unroll
        for (int j = 0; j < KV; ++j) acc += upd(v[j], C.c, 0);
#pragma unroll
        for (int j = 0; j < KV; ++j) acc += upd(v[j], C.c, 7);
#pragma unroll
        for (int j = 0; j < KV; ++j)
#pragma unroll
            for (int d = 0; d < NL; ++d)
                *reinterpret_cast<double2 *>(base + 16 * d + 8192 * j + (i & 1) * 16384) = v[j][d];
        if (BAR) __syncthreads();
    }
    long long c1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = c1 - c0;
    sink[(blockIdx.x * blockDim.x + threadIdx.x) % 4096] = acc + v[0][0].x + v[KV - 1][3].y;
}
template <int KV, int NL, int LS, bool BAR>
double run(long long *out, double *sink, int w, int grid, int ds) {
    Cf C; for (int i = 0; i < 20; ++i) C.c[i] = 1e-3 * (i + 1);
    const int n = 2000;
    auto f = k<KV, NL, LS, BAR>;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    f<<<grid, 32 * w, ds>>>(out, C, n, sink); cudaDeviceSynchronize();
    f<<<grid, 32 * w, ds>>>(out, C, n, sink); cudaDeviceSynchronize();
    return (double)out[0] / n;
}
int main() {
    long long *out; double *sink;
    cudaMallocManaged(&out, 64 * sizeof(long long));
    cudaMalloc(&sink, 4096 * sizeof(double));
    const int small = 40 * 1024, big = 215 * 1024;
    printf("cycles per step (7 warps unless stated)\n");
    printf("1 vertex, 3+3 smem, 16 B lanes, barrier, 1 CTA, small smem: %.0f\n", run<1, 3, 16, true>(out, sink, 7, 1, small));
    printf("1 vertex, 3+3 smem, 112 B lanes: %.0f\n", run<1, 3, 112, true>(out, sink, 7, 1, small));
    printf("1 vertex, 7+7 smem, 112 B lanes: %.0f\n", run<1, 7, 112, true>(out, sink, 7, 1, small));
    printf("2 vertices, 7+7 smem, 112 B lanes: %.0f\n", run<2, 7, 112, true>(out, sink, 7, 1, small));
    printf("2 vertices, 7+7, 112 B, no barrier: %.0f\n", run<2, 7, 112, false>(out, sink, 7, 1, small));
    printf("2 vertices, 7+7, 112 B, barrier, 215 KB smem: %.0f\n", run<2, 7, 112, true>(out, sink, 7, 1, big));
    printf("2 vertices, 7+7, 112 B, barrier, 215 KB smem, 148 CTAs: %.0f\n", run<2, 7, 112, true>(out, sink, 7, 148, big));
    printf("2 vertices, 7+7, 112 B, barrier, 215 KB, 148 CTAs, 8 warps: %.0f\n", run<2, 7, 112, true>(out, sink, 8, 148, big));
    printf("1 vertex, 3+3, 112 B, barrier, 215 KB, 148 CTAs, 7 warps: %.0f\n", run<1, 3, 112, true>(out, sink, 7, 148, big));
    printf("1 vertex, 3+3, 112 B, barrier, 215 KB, 148 CTAs, 22 warps (all compute): %.0f\n", run<1, 3, 112, true>(out, sink, 22, 148, big));
    return 0;
}
