// Cycles per vertex update (both unknowns, node_update_u arithmetic) on W warps
// of one SM, with coefficients as kernel parameters (dev tool).
// nvcc -O3 --fmad=false -gencode arch=compute_100a,code=sm_100a -o /tmp/micro_node scripts/micro_node.cu
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
template <int MODE>
__global__ void k(long long *out, const __grid_constant__ Cf C, int n, double *sink) {
    __shared__ double2 sh[7 * 256];
    for (int i = threadIdx.x; i < 7 * 256; i += blockDim.x) sh[i] = make_double2(1e-3 * i, 1.0);
    __syncthreads();
    double2 v[7];
    for (int d = 0; d < 7; ++d) v[d] = make_double2(threadIdx.x + d, 1.0 / (1 + d));
    double acc = 0;
    long long c0 = clock64();
    for (int i = 0; i < n; ++i) {
        if (MODE >= 1) {  // 3 entries in from shared memory
            v[1] = sh[threadIdx.x]; v[4] = sh[256 + threadIdx.x]; v[6] = sh[512 + threadIdx.x];
        }
        acc += upd(v, C.c, 0);
        acc += upd(v, C.c, 7);
        if (MODE >= 1) {  // 3 entries out
            sh[768 + threadIdx.x] = v[0]; sh[1024 + threadIdx.x] = v[2]; sh[1280 + threadIdx.x] = v[5];
        }
        if (MODE >= 2) __syncthreads();
    }
    long long c1 = clock64();
    if (threadIdx.x % 32 == 0) out[threadIdx.x / 32] = c1 - c0;
    sink[threadIdx.x] = acc + v[0].x + v[3].y;
}
int main() {
    long long *out; double *sink;
    cudaMallocManaged(&out, 64 * sizeof(long long));
    cudaMalloc(&sink, 4096 * sizeof(double));
    Cf C; for (int i = 0; i < 20; ++i) C.c[i] = 1e-3 * (i + 1);
    const int n = 2000;
    for (int w : {1, 4, 7, 8, 14}) {
        k<0><<<1, 32 * w>>>(out, C, n, sink); cudaDeviceSynchronize();
        double a = (double)out[0] / n;
        k<1><<<1, 32 * w>>>(out, C, n, sink); cudaDeviceSynchronize();
        double b = (double)out[0] / n;
        k<2><<<1, 32 * w>>>(out, C, n, sink); cudaDeviceSynchronize();
        double c = (double)out[0] / n;
        printf("%2d warps: registers only %.0f, + 3 LDS.128 / 3 STS.128 %.0f, + __syncthreads %.0f cycles per vertex\n", w, a, b, c);
    }
    return 0;
}
