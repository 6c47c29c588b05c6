// Dependent DFMA / DADD / DMUL latency and LDS.128 latency on one warp (dev tool).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/micro_dfma_lat scripts/micro_dfma_lat.cu
#include <cstdio>
__global__ void k(long long *out, double a, double b, int n, double *sink) {
    __shared__ double2 sh[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sh[i] = make_double2(i * 1e-3, 1.0);
    __syncthreads();
    double x = threadIdx.x;
    long long c0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, a, b);
    long long c1 = clock64();
    double y = threadIdx.x;
    for (int i = 0; i < n; ++i) y = y * a;
    long long c2 = clock64();
    double z = threadIdx.x;
    for (int i = 0; i < n; ++i) z = z + a;
    long long c3 = clock64();
    // pointer chase through shared memory, 16-byte loads, lanes 112 B apart
    unsigned idx = (threadIdx.x & 31) * 7;
    double acc = 0;
    for (int i = 0; i < n; ++i) {
        double2 t = sh[idx & 1023];
        acc += t.x;
        idx = idx + (unsigned)t.y;
    }
    long long c4 = clock64();
    if (threadIdx.x % 32 == 0) {
        out[0] = c1 - c0; out[1] = c2 - c1; out[2] = c3 - c2; out[3] = c4 - c3;
    }
    sink[threadIdx.x] = x + y + z + acc;
}
int main() {
    long long *out; double *sink;
    cudaMallocManaged(&out, 64 * sizeof(long long));
    cudaMalloc(&sink, 4096 * sizeof(double));
    const int n = 4096;
    for (int w : {1, 8}) {
        k<<<1, 32 * w>>>(out, 0.999, 1e-3, n, sink);
        cudaDeviceSynchronize();
        k<<<1, 32 * w>>>(out, 0.999, 1e-3, n, sink);
        cudaDeviceSynchronize();
        printf("%d warps: DFMA %.1f  DMUL %.1f  DADD %.1f  LDS.128+DADD+IADD chase %.1f cycles per dependent op\n", w,
               (double)out[0] / n, (double)out[1] / n, (double)out[2] / n, (double)out[3] / n);
    }
    return 0;
}
