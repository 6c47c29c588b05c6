// Latency microbenchmarks (single warp, dependent chains), cycles per op.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/micro_lat scripts/micro_lat.cu
#include <cstdio>

__global__ void k_lat(double *out, const double *g, long long *cyc, int n) {
    __shared__ double sh[64];
    const int lane = threadIdx.x;
    sh[lane] = 1.0 + lane * 1e-3;
    sh[lane + 32] = 1.0;
    __syncwarp();
    double a = out[lane], b = out[lane + 32], c = 1.0000001;
    long long t0, t1;
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) a = fma(a, c, b);
    t1 = clock64();
    cyc[0] = t1 - t0;
    // DADD chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) a = a + b;
    t1 = clock64();
    cyc[1] = t1 - t0;
    // SHFL (double) chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) a = __shfl_down_sync(0xffffffffu, a, 1) + 0.0;
    t1 = clock64();
    cyc[2] = t1 - t0;
    // LDS chain (address depends on loaded value)
    int idx = lane;
    t0 = clock64();
    for (int i = 0; i < n; ++i) idx = (int)sh[idx & 63] & 31;
    t1 = clock64();
    cyc[3] = t1 - t0;
    // L2 (ld.cg) pointer chase over a 16 MB region
    long long j = lane;
    t0 = clock64();
    for (int i = 0; i < n / 16; ++i) j = (long long)__ldcg(g + j);
    t1 = clock64();
    cyc[4] = (t1 - t0) * 16;
    // __syncwarp cost
    t0 = clock64();
    for (int i = 0; i < n; ++i) __syncwarp();
    t1 = clock64();
    cyc[5] = t1 - t0;
    out[lane] = a + (double)idx + (double)j;
}

int main() {
    const int n = 4096;
    double *out, *g;
    long long *cyc;
    cudaMalloc(&out, 64 * 8);
    cudaMemset(out, 0, 64 * 8);
    const size_t ng = 2 * 1024 * 1024;  // 16 MB
    cudaMalloc(&g, ng * 8);
    double *h = new double[ng];
    for (size_t i = 0; i < ng; ++i) h[i] = (double)((i * 7919 + 4099) % ng);
    cudaMemcpy(g, h, ng * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&cyc, 8 * 8);
    k_lat<<<1, 32>>>(out, g, cyc, n);
    k_lat<<<1, 32>>>(out, g, cyc, n);
    cudaDeviceSynchronize();
    long long c[8];
    cudaMemcpy(c, cyc, 6 * 8, cudaMemcpyDeviceToHost);
    const char *nm[] = {"DFMA", "DADD", "SHFL.f64+DADD", "LDS", "LDG.cg (L2)", "SYNCWARP"};
    for (int i = 0; i < 6; ++i) printf("%-16s %6.1f cycles/op\n", nm[i], (double)c[i] / n);
    return 0;
}
