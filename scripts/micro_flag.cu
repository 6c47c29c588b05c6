// Flag hand-off latency between CTAs on different SMs (dev tool): a token
// passes down a chain of CTAs (CTA b waits for CTA b-1's counter, then bumps
// its own), as the exact-order sweep's bands do.  Variants:
//   0  st.release.gpu / ld.relaxed.gpu poll + fence.acq_rel.gpu (k_wavefront)
//   1  st.relaxed.gpu after fence.acq_rel / ld.acquire.gpu poll
//   2  as 0 plus a 64-double payload written before the release and read
//      (__ldcg) after the acquire
//   3  as 2 with the payload carrying its own sequence tag (no flag): the
//      consumer polls the payload's last 16 B
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o scripts/micro_flag scripts/micro_flag.cu
#include <cstdio>

__device__ __forceinline__ int ld_relaxed(const int *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int *p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed(int *p, int v) {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

template <int V>
__global__ void k_chain(int *flags, double *pay, int rounds, long long *out, double *sink) {
    const int b = blockIdx.x, lane = threadIdx.x;
    int *mine = flags + b * 64, *prev = flags + (b - 1) * 64;
    double acc = 0.0;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 1; i <= rounds; ++i) {
        if (b > 0) {
            if (V == 3) {
                // payload slot i: 64 doubles, tag = double(i) in the last one
                volatile double *q = pay + ((size_t)(b - 1) * rounds + (i - 1)) * 64;
                if (lane == 0)
                    while (q[63] != (double)i) {
                    }
                __syncwarp();
                acc += __ldcg(pay + ((size_t)(b - 1) * rounds + (i - 1)) * 64 + lane);
            } else {
                if (lane == 0) {
                    if (V == 1)
                        while (ld_acquire(prev) < i) {
                        }
                    else {
                        while (ld_relaxed(prev) < i) {
                        }
                        fence();
                    }
                }
                __syncwarp();
                if (V == 2) acc += __ldcg(pay + (size_t)(b - 1) * 64 + lane);
            }
        }
        if (V >= 2) {
            double *q = V == 3 ? pay + ((size_t)b * rounds + (i - 1)) * 64 : pay + (size_t)b * 64;
            q[lane] = acc + i;
            q[lane + 32] = V == 3 && lane == 31 ? (double)i : acc;
        }
        __syncwarp();
        if (V == 3) {
            if (lane == 0) __threadfence();
            __syncwarp();
            if (lane == 31) {
                volatile double *q = pay + ((size_t)b * rounds + (i - 1)) * 64;
                q[63] = (double)i;
            }
        } else if (lane == 0) {
            if (V == 1) {
                fence();
                st_relaxed(mine, i);
            } else
                st_release(mine, i);
        }
    }
    long long t1 = clock64();
    if (lane == 0) out[b] = t1 - t0;
    sink[b * 32 + lane] = acc;
}

int main() {
    const int nb = 142, rmax = 200;
    int *flags;
    double *pay, *sink;
    long long *out;
    cudaMalloc(&flags, nb * 64 * sizeof(int));
    cudaMalloc(&pay, (size_t)nb * rmax * 64 * sizeof(double));
    cudaMalloc(&sink, nb * 32 * sizeof(double));
    cudaMallocManaged(&out, nb * sizeof(long long));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char *names[] = {"release/relaxed+fence", "fence+relaxed/acquire", "release + payload",
                           "tagged payload (no flag)"};
    for (int rounds : {1, 8, rmax})
    for (int v = 0; v < 4; ++v)
        for (int rep = 0; rep < 2; ++rep) {
            cudaMemset(flags, 0, nb * 64 * sizeof(int));
            cudaMemset(pay, 0, (size_t)nb * rounds * 64 * sizeof(double));
            cudaEventRecord(e0);
            if (v == 0) k_chain<0><<<nb, 32>>>(flags, pay, rounds, out, sink);
            if (v == 1) k_chain<1><<<nb, 32>>>(flags, pay, rounds, out, sink);
            if (v == 2) k_chain<2><<<nb, 32>>>(flags, pay, rounds, out, sink);
            if (v == 3) k_chain<3><<<nb, 32>>>(flags, pay, rounds, out, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            // the last CTA finishes after (nb - 1) hops of latency + rounds x period
            if (rep)
                printf("rounds %3d %-26s total %.1f us; per hop %.2f us; last CTA %lld cycles\n",
                       rounds, names[v], ms * 1e3, ms * 1e3 / nb, out[nb - 1]);
        }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
