// Does ld.global.cg (LDG.E.64.STRONG.GPU) pipeline?  One warp, 32
// independent loads per round, cycles per round for several load flavours.
#include <cstdio>
template <int MODE>
__global__ void k(const double *g, double *out, long long *cyc, int rounds) {
    const int lane = threadIdx.x;
    double acc = 0.0;
    long long t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
        double v[32];
        const double *p = g + (size_t)r * 4096 * 32 + lane;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const double *q = p + k * 4096;
            if (MODE == 0) v[k] = *q;
            if (MODE == 1) v[k] = __ldcg(q);
            if (MODE == 2) v[k] = __ldg(q);
            if (MODE == 3) asm volatile("ld.global.relaxed.gpu.f64 %0, [%1];" : "=d"(v[k]) : "l"(q));
            if (MODE == 4) asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v[k]) : "l"(q));
            if (MODE == 5) asm volatile("ld.global.cg.L2::128B.f64 %0, [%1];" : "=d"(v[k]) : "l"(q));
        }
#pragma unroll
        for (int k = 0; k < 32; ++k) acc += v[k];
    }
    long long t1 = clock64();
    if (lane == 0) cyc[MODE] = (t1 - t0) / rounds;
    out[lane] = acc;
}
int main() {
    const size_t n = (size_t)64 * 4096 * 32;
    double *g, *out;
    long long *cyc;
    cudaMalloc(&g, n * 8);
    cudaMemset(g, 0, n * 8);
    cudaMalloc(&out, 256);
    cudaMalloc(&cyc, 64);
    for (int rep = 0; rep < 2; ++rep) {
        k<0><<<1, 32>>>(g, out, cyc, 64);
        k<1><<<1, 32>>>(g, out, cyc, 64);
        k<2><<<1, 32>>>(g, out, cyc, 64);
        k<3><<<1, 32>>>(g, out, cyc, 64);
        k<4><<<1, 32>>>(g, out, cyc, 64);
        k<5><<<1, 32>>>(g, out, cyc, 64);
    }
    cudaDeviceSynchronize();
    long long h[6];
    cudaMemcpy(h, cyc, 48, cudaMemcpyDeviceToHost);
    const char *nm[] = {"plain ld", "__ldcg", "__ldg", "ld.relaxed.gpu", "ld.cg (asm volatile)", "ld.cg.L2::128B"};
    for (int i = 0; i < 6; ++i) printf("%-22s %6lld cycles per round of 32 loads\n", nm[i], h[i]);
    return 0;
}
