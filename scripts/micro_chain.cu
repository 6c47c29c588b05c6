// Cycles per step of the exact-order sweep's chain recurrence on one warp
// (dev tool), in variants that remove one ingredient at a time:
//   0  as k_wavefront: shuffles of p (2 x double), lane-0/1 selects, p
//      guarded by a select, 7 off-path FMAs, G loads, p stores
//   1  p = a * inv_eff (no select on the critical path)
//   2  1 + v1 / v2 selects through precomputed masks (no ternary chain)
//   3  2 + only the v1 shuffle on the path (v2 from the last step's v1)
//   4  critical path only: a = fma(n8, p, acc); a = fma(n6, shfl(p), a); p = a*inv
//   5  4 without the shuffle (own p): the FP64 latency floor
//   6  2 with branch-free bit selects (LOP3 on the bit patterns)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/micro_chain scripts/micro_chain.cu
#include <cstdio>

__device__ __forceinline__ double bsel(bool c, double a, double b) {
    // c ? a : b without a branch (the compiler turns ternaries on loaded
    // values into divergent branches)
    const long long m = -(long long)c;
    return __longlong_as_double((__double_as_longlong(a) & m) | (__double_as_longlong(b) & ~m));
}

template <int V>
__global__ void k_chain(long long *out, const double *K, int nsteps, double *sink) {
    __shared__ double gw[32 * 33], pw[34 * 33];
    const int i = threadIdx.x & 31;
    for (int t = threadIdx.x; t < 32 * 33; t += blockDim.x) gw[t] = 1e-3 * (t % 7);
    for (int t = threadIdx.x; t < 34 * 33; t += blockDim.x) pw[t] = 1e-3 * (t % 5);
    __syncthreads();
    double k[10];
    for (int m = 0; m < 10; ++m) k[m] = K[m];
    double acc[7] = {0, 0, 0, 0, 0, 0, 0}, pprev = 0.0, v1prev = 0.0, v2prev = 0.0;
    const bool l0 = i == 0, l1 = i == 1;
    long long c0 = clock64();
    for (int tau0 = 0; tau0 < nsteps; tau0 += 8) {
        double g[8], e1[8], e2[8];
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            g[s] = gw[i * 33 + ((tau0 + s + 6) & 31)];
            e1[s] = pw[33 + ((tau0 + s) & 31)];
            e2[s] = pw[((tau0 + s) & 31)];
        }
        double pout[8];
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            const int x = tau0 + s - 2 * i;
            const bool ok = (unsigned)x < 4000u;
            double p, v1, v2;
            if (V >= 4) {
                double a = fma(k[8], pprev, acc[0]);
                const double u = V == 5 ? pprev : __shfl_up_sync(0xffffffffu, pprev, 1);
                a = fma(k[6], u, a);
                p = a * k[9];
                pout[s] = p;
                pprev = p;
                continue;
            }
            double a = fma(k[8], pprev, acc[0]);
            a = fma(k[6], v1prev, a);
            if (V == 0)
                p = ok ? a * k[9] : 0.0;
            else
                p = a * (ok ? k[9] : 0.0);
            pout[s] = p;
            const double u1 = __shfl_up_sync(0xffffffffu, p, 1);
            if (V == 3) {
                v1 = l0 ? e1[s] : u1;
                v2 = l0 ? e2[s] : (l1 ? e1[s] : v2prev);  // stand-in, off path
            } else {
                const double u2 = __shfl_up_sync(0xffffffffu, p, 2);
                if (V == 0) {
                    v1 = i == 0 ? e1[s] : u1;
                    v2 = i == 0 ? e2[s] : i == 1 ? e1[s] : u2;
                } else if (V == 6) {
                    v1 = bsel(l0, e1[s], u1);
                    v2 = bsel(l0, e2[s], bsel(l1, e1[s], u2));
                } else {
                    v1 = l0 ? e1[s] : u1;
                    const double t2 = l1 ? e1[s] : u2;
                    v2 = l0 ? e2[s] : t2;
                }
            }
            double a2 = fma(k[7], p, acc[2]);
            a2 = fma(k[5], v1, a2);
            const double a3 = fma(k[4], v1, acc[3]);
            double a4 = fma(k[3], v1, acc[4]);
            a4 = fma(k[2], v2, a4);
            const double a5 = fma(k[1], v2, acc[5]);
            const double a6 = fma(k[0], v2, g[s]);
            acc[0] = acc[1];
            acc[1] = a2;
            acc[2] = a3;
            acc[3] = a4;
            acc[4] = a5;
            acc[5] = a6;
            pprev = p;
            v2prev = v1prev;
            v1prev = v1;
        }
#pragma unroll
        for (int s = 0; s < 8; ++s) pw[(i + 2) * 33 + ((tau0 + s) & 31)] = pout[s];
    }
    long long c1 = clock64();
    if (threadIdx.x == 0) out[V] = c1 - c0;
    sink[threadIdx.x] = pprev + acc[1];
}

int main() {
    long long *out;
    double *K, *sink;
    cudaMallocManaged(&out, 16 * sizeof(long long));
    cudaMallocManaged(&K, 16 * sizeof(double));
    cudaMallocManaged(&sink, 1024 * sizeof(double));
    for (int m = 0; m < 10; ++m) K[m] = -0.01 * (m + 1);
    K[9] = 0.5;
    const int n = 4096;
    for (int rep = 0; rep < 2; ++rep) {
        k_chain<0><<<1, 32>>>(out, K, n, sink);
        k_chain<1><<<1, 32>>>(out, K, n, sink);
        k_chain<2><<<1, 32>>>(out, K, n, sink);
        k_chain<3><<<1, 32>>>(out, K, n, sink);
        k_chain<4><<<1, 32>>>(out, K, n, sink);
        k_chain<5><<<1, 32>>>(out, K, n, sink);
        k_chain<6><<<1, 32>>>(out, K, n, sink);
        cudaDeviceSynchronize();
    }
    const char *names[] = {"as kernel", "no p select", "mask selects", "one shuffle",
                           "critical path only", "no shuffle (FP64 floor)", "bit selects"};
    for (int v = 0; v < 7; ++v)
        printf("variant %d %-24s %.1f cycles/step\n", v, names[v], (double)out[v] / n);
    return 0;
}
