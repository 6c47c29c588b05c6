// Step-cost probe for the multicolour sweep's core (dev tool): 7 warps per
// CTA, each step every lane loads a 7-point (state, adjoint) neighbourhood
// from a shared-memory ring, runs the two NE-GS unknown updates (58 DFMA)
// and stores it back.  Variants of the synchronisation between warps:
//   0: __syncthreads per step (the current kernel's scheme)
//   1: mbarrier chain (warp q waits for warp q-1's previous step only)
//   2: __syncthreads per step, two independent vertices per lane
// Prints cycles per step (per CTA), with 2 CTAs per SM on every SM.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/micro_mc scripts/micro_mc.cu
#include <cstdio>

constexpr int NT = 224, RING = 26, STRIDE = 206;

__device__ __forceinline__ double upd(double2 (&v)[7], const double *c) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int d = 0; d < 7; ++d) {
        s0 = fma(c[d], v[d].x, s0);
        s1 = fma(c[7 + d], v[d].y, s1);
    }
    const double p = (s0 + s1) * c[28];
#pragma unroll
    for (int d = 0; d < 7; ++d)
        v[d] = make_double2(fma(-c[14 + d], p, v[d].x), fma(-c[21 + d], p, v[d].y));
    return p;
}

struct Co {
    double c[2][29];
};

template <int MODE>
__global__ void __launch_bounds__(NT, 2) k_probe(const __grid_constant__ Co co, int steps,
                                                  long long *cyc, double *sink) {
    extern __shared__ __align__(16) double2 ring[];
    __shared__ int done[8];
    const int tid = threadIdx.x, lane = tid & 31, q = tid >> 5;
    for (int i = tid; i < RING * STRIDE; i += NT) ring[i] = make_double2(1e-3 * i, 1.0);
    if (tid < 8) done[tid] = 0;
    __syncthreads();
    double acc = 0.0;
    int o = q % 7;
    unsigned sy = (unsigned)((RING - 3 * q) % RING);
    const long long t0 = clock64();
    for (int s = 0; s < steps; ++s) {
        if (MODE == 1 && q > 0) {
            // wait for warp q-1's step s-1 (done[q-1] >= s)
            if (lane == 0) {
                const unsigned a = (unsigned)__cvta_generic_to_shared(&done[q - 1]);
                int v;
                do {
                    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
                } while (v < s);
            }
            __syncwarp();
        }
        const int c0 = o + 7 * lane + 1;
        const unsigned sb = sy == 0 ? RING - 1 : sy - 1, su = sy == RING - 1 ? 0 : sy + 1;
        double2 *rb = ring + sb * STRIDE + c0, *rc = ring + sy * STRIDE + c0,
                *ru = ring + su * STRIDE + c0;
        if (MODE == 2) {
            const int c1 = (o + 3) % 7 + 7 * lane + 1;
            const unsigned s2 = su, s3 = su == RING - 1 ? 0 : su + 1;
            double2 *rb2 = ring + sy * STRIDE + c1, *rc2 = ring + s2 * STRIDE + c1,
                    *ru2 = ring + s3 * STRIDE + c1;
            double2 v[7] = {rb[-1], rb[0], rc[-1], rc[0], rc[1], ru[0], ru[1]};
            double2 w[7] = {rb2[-1], rb2[0], rc2[-1], rc2[0], rc2[1], ru2[0], ru2[1]};
            acc += upd(v, co.c[0]);
            acc += upd(w, co.c[0]);
            acc += upd(v, co.c[1]);
            acc += upd(w, co.c[1]);
            rb[-1] = v[0]; rb[0] = v[1]; rc[-1] = v[2]; rc[0] = v[3]; rc[1] = v[4];
            ru[0] = v[5]; ru[1] = v[6];
            rb2[-1] = w[0]; rb2[0] = w[1]; rc2[-1] = w[2]; rc2[0] = w[3]; rc2[1] = w[4];
            ru2[0] = w[5]; ru2[1] = w[6];
        } else {
            double2 v[7] = {rb[-1], rb[0], rc[-1], rc[0], rc[1], ru[0], ru[1]};
            acc += upd(v, co.c[0]);
            acc += upd(v, co.c[1]);
            rb[-1] = v[0]; rb[0] = v[1]; rc[-1] = v[2]; rc[0] = v[3]; rc[1] = v[4];
            ru[0] = v[5]; ru[1] = v[6];
        }
        sy = sy + (MODE == 2 ? 2 : 1);
        sy = sy >= RING ? sy - RING : sy;
        o = o >= 2 ? o - 2 : o + 5;
        if (MODE == 1) {
            __syncwarp();
            if (lane == 0) {
                const unsigned a = (unsigned)__cvta_generic_to_shared(&done[q]);
                asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"(a), "r"(s + 1) : "memory");
            }
            __syncwarp();
        } else {
            __syncthreads();
        }
    }
    const long long t1 = clock64();
    if (tid == 0 && blockIdx.x == 0) cyc[MODE] = t1 - t0;
    if (acc == 12345.0) sink[tid] = acc;
}

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e_ = (x);                                                   \
        if (e_ != cudaSuccess) {                                                \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));   \
            return 1;                                                           \
        }                                                                       \
    } while (0)

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    printf("start\n");
    Co co;
    for (int f = 0; f < 2; ++f)
        for (int i = 0; i < 29; ++i) co.c[f][i] = 1e-3 * (i + 1) * (f ? -1 : 1);
    long long *cyc;
    double *sink;
    CK(cudaMalloc(&cyc, 8 * 8));
    CK(cudaMalloc(&sink, 1024 * 8));
    printf("alloc ok\n");
    const int smem = (RING * STRIDE + 64) * 16;  // lanes read up to 20 entries past a row
    CK(cudaFuncSetAttribute(k_probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(k_probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(k_probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    printf("attr ok\n");
    const int steps = 400;
    for (int rep = 0; rep < 2; ++rep) {
        k_probe<0><<<296, NT, smem>>>(co, steps, cyc, sink);
        k_probe<1><<<296, NT, smem>>>(co, steps, cyc, sink);
        k_probe<2><<<296, NT, smem>>>(co, steps / 2, cyc, sink);
        CK(cudaGetLastError());
    }
    cudaError_t e = cudaDeviceSynchronize();
    long long c[3];
    cudaMemcpy(c, cyc, 3 * 8, cudaMemcpyDeviceToHost);
    printf("err=%s\n", cudaGetErrorString(e));
    printf("syncthreads      %8.1f cycles/step\n", (double)c[0] / steps);
    printf("flag chain       %8.1f cycles/step\n", (double)c[1] / steps);
    printf("2 rows/step      %8.1f cycles/row-step\n", (double)c[2] / steps);
    // timing of a whole grid too
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int m = 0; m < 3; ++m) {
        cudaEventRecord(a);
        if (m == 0) k_probe<0><<<296, NT, smem>>>(co, steps, cyc, sink);
        if (m == 1) k_probe<1><<<296, NT, smem>>>(co, steps, cyc, sink);
        if (m == 2) k_probe<2><<<296, NT, smem>>>(co, steps / 2, cyc, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("mode %d grid %.3f ms (%.1f ns per row-step)\n", m, ms, 1e6 * ms / steps);
    }
    return 0;
}
