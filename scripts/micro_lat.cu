// Dependent-chain latencies on one warp (dev tool): DFMA, DADD, DMUL,
// IEEE DDIV (__ddiv_rn), DRCP+DMUL, LDS.64 pointer chase, BAR.SYNC with
// 1..8 warps.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/micro_lat scripts/micro_lat.cu
#include <cstdio>

__global__ void k_lat(long long *out, double a, double b, int n) {
    __shared__ long long sm_idx[1024];
    __shared__ double sm_d[1024];
    const int t = threadIdx.x;
    for (int i = t; i < 1024; i += blockDim.x) {
        sm_idx[i] = (i * 17 + 1) & 1023;
        sm_d[i] = 1.0 + 1e-9 * i;
    }
    __syncthreads();
    double x = a + t;
    long long c0, c1;
    // DFMA
    c0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, b, a);
    c1 = clock64();
    if (t == 0) out[0] = c1 - c0;
    // DADD
    c0 = clock64();
    for (int i = 0; i < n; ++i) x = x + b;
    c1 = clock64();
    if (t == 0) out[1] = c1 - c0;
    // DMUL
    c0 = clock64();
    for (int i = 0; i < n; ++i) x = x * b;
    c1 = clock64();
    if (t == 0) out[2] = c1 - c0;
    // DDIV
    c0 = clock64();
    for (int i = 0; i < n; ++i) x = __ddiv_rn(x, b);
    c1 = clock64();
    if (t == 0) out[3] = c1 - c0;
    // rcp + mul
    c0 = clock64();
    for (int i = 0; i < n; ++i) x = x * __drcp_rn(b + x * 1e-300);
    c1 = clock64();
    if (t == 0) out[4] = c1 - c0;
    // LDS chase
    long long p = t & 1023;
    c0 = clock64();
    for (int i = 0; i < n; ++i) p = sm_idx[p];
    c1 = clock64();
    if (t == 0) out[5] = c1 - c0;
    // LDS.64 double dependent (address from value)
    double y = sm_d[t & 1023];
    c0 = clock64();
    for (int i = 0; i < n; ++i) y = sm_d[((long long)(y * 1e9)) & 1023];
    c1 = clock64();
    if (t == 0) out[6] = c1 - c0;
    // barrier
    __syncthreads();
    c0 = clock64();
    for (int i = 0; i < n; ++i) __syncthreads();
    c1 = clock64();
    if (t == 0) out[7] = c1 - c0;
    if (x == 12345.0 || p == 99999 || y == 1.5) out[8] = 1;
}

int main() {
    long long *d, h[9];
    cudaMalloc(&d, 9 * sizeof(long long));
    const int n = 1000;
    const char *names[8] = {"DFMA", "DADD", "DMUL", "DDIV (__ddiv_rn)", "DRCP+DMUL",
                            "LDS.64 chase (int)", "LDS.64 chase (double)", "BAR.SYNC"};
    for (int w : {1, 2, 4, 8}) {
        for (int rep = 0; rep < 2; ++rep) k_lat<<<1, 32 * w>>>(d, 1.0000001, 0.9999999, n);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d, 9 * sizeof(long long), cudaMemcpyDeviceToHost);
        printf("warps=%d:", w);
        for (int i = 0; i < 8; ++i) printf("  %s %.1f", names[i], (double)h[i] / n);
        printf("\n");
    }
    return 0;
}
