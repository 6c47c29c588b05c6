// FP64 FMA throughput per warp / SM (dev tool): W warps, each with 8
// independent DFMA chains.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/micro_fp64 scripts/micro_fp64.cu
#include <cstdio>
__global__ void k(long long *out, double a, double b, int n, double *sink) {
    double x[8];
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
    __syncthreads();
    long long c0 = clock64();
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
    long long c1 = clock64();
    if (threadIdx.x == 0) out[blockDim.x / 32] = c1 - c0;
    double s = 0;
    for (int j = 0; j < 8; ++j) s += x[j];
    sink[threadIdx.x] = s;
}
int main() {
    long long *out; double *sink;
    cudaMallocManaged(&out, 64 * sizeof(long long));
    cudaMalloc(&sink, 4096 * sizeof(double));
    const int n = 4096;
    for (int w : {1, 2, 4, 8, 16, 32}) {
        k<<<1, 32 * w>>>(out, 0.999, 1e-3, n, sink);
        cudaDeviceSynchronize();
        k<<<1, 32 * w>>>(out, 0.999, 1e-3, n, sink);
        cudaDeviceSynchronize();
        const double per = (double)out[w] / (8.0 * n);
        printf("%2d warps: %.2f cycles per warp-DFMA per warp -> %.1f FMA/clk/SM\n", w, per, 32.0 * w / per);
    }
    return 0;
}
