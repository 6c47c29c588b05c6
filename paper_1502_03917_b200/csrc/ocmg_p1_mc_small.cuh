// Multicolour NE-GS sweep for the small and middle levels of a cycle, where
// the pipelined strip kernel (ocmg_p1_mc.cuh) would spend most of its steps
// filling and draining.  Same order and arithmetic (p1_mc_vertex /
// mcs::node_update), so all three forms are bit-identical.
//
//   k <= 6  (n1 <= 65):  k_p1_mc_small -- one CTA, the whole residual, x and
//                        the class table in shared memory, 7 colour phases
//                        separated by __syncthreads.
//   k_p1_mc_grid -- one cooperative launch, 7 colour phases separated by a
//                        grid barrier, in place; kept, but the one-launch
//                        strip kernel (ocmg_p1_mc.cuh) now runs from k = 7.
#pragma once

#include "ocmg_p1_mc.cuh"

namespace ocmg {

constexpr int kMcSmallMaxN1 = 65;
// the cooperative tier is kept but unused: the one-launch strip kernel is
// faster from L7 up in the cycle (W-cycle L12 37.3 -> 35.4 ms)
constexpr int kMcGridMaxN1 = 65;

__host__ __device__ constexpr int mc_small_smem(int n1) {
    // residual with a zero guard ring, x pairs, the class table [49][2][29]
    return (n1 + 2) * (n1 + 2) * 16 + n1 * n1 * 16 + 49 * 58 * 8;
}

// x, r and the class table all in shared memory: the 7 colour phases touch
// global memory not at all
__global__ void __launch_bounds__(1024)
    k_p1_mc_small(int n1, int forward, const double *__restrict__ C,
                  double *__restrict__ x, double *__restrict__ r) {
    pdl_trigger();  // launched with PDL (short dependent launches of a cycle)
    pdl_wait();
    extern __shared__ double2 g[];  // [(n1+2)^2] (state, adjoint), zero guards
    const int P = n1 + 2;
    const int N = n1 * n1;
    double2 *const xs = g + P * P;  // [n1^2] (state, adjoint)
    double *const Cs = reinterpret_cast<double *>(xs + N);  // [49][2][29]
    // staging: every global read is an asynchronous copy, one wait for all
    for (int i = threadIdx.x; i < P * P; i += blockDim.x) {
        const int gy = i / P, gx = i - gy * P;
        const int ix = gx - 1, iy = gy - 1;
        if (ix >= 0 && ix < n1 && iy >= 0 && iy < n1) {
            const int k = iy * n1 + ix;
            mcs_cp8((unsigned)__cvta_generic_to_shared(&g[i].x), r + k, true);
            mcs_cp8((unsigned)__cvta_generic_to_shared(&g[i].y), r + N + k, true);
        } else {
            g[i] = make_double2(0.0, 0.0);
        }
    }
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        mcs_cp8((unsigned)__cvta_generic_to_shared(&xs[i].x), x + i, true);
        mcs_cp8((unsigned)__cvta_generic_to_shared(&xs[i].y), x + N + i, true);
    }
    for (int i = threadIdx.x; i < 49 * 58; i += blockDim.x)
        mcs_cp8((unsigned)__cvta_generic_to_shared(Cs + i), C + i, true);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    const int per_row = (n1 + 6) / 7;
    const int count = per_row * n1;
    const int f0 = forward ? 0 : 1;
    for (int b = 0; b < kMcColours; ++b) {
        const int cm = forward ? b : kMcColours - 1 - b;
        for (int k = threadIdx.x; k < count; k += blockDim.x) {
            const int iy = k / per_row, jj = k - iy * per_row;
            const int ix = ((cm - 2 * iy) % 7 + 7) % 7 + 7 * jj;
            if (ix >= n1) continue;
            const int c = (iy + 1) * P + ix + 1;
            double2 *const adr[7] = {g + c - P - 1, g + c - P, g + c - 1, g + c,
                                     g + c + 1,     g + c + P, g + c + P + 1};
            double2 v[7];
#pragma unroll
            for (int d = 0; d < 7; ++d) v[d] = *adr[d];
            const int cls = 7 * p1_axis_class(iy, n1) + p1_axis_class(ix, n1);
            double p[2];
            p[f0] = mcs::node_update(v, Cs + (cls * 2 + f0) * 29);
            p[1 - f0] = mcs::node_update(v, Cs + (cls * 2 + 1 - f0) * 29);
#pragma unroll
            for (int d = 0; d < 7; ++d) *adr[d] = v[d];
            const int xi = iy * n1 + ix;
            const double2 xo = xs[xi];
            xs[xi] = make_double2(__dadd_rn(xo.x, p[0]), __dadd_rn(xo.y, p[1]));
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < P * P; i += blockDim.x) {
        const int gy = i / P, gx = i - gy * P;
        const int ix = gx - 1, iy = gy - 1;
        if (ix >= 0 && ix < n1 && iy >= 0 && iy < n1) {
            const int k = iy * n1 + ix;
            r[k] = g[i].x;
            r[N + k] = g[i].y;
        }
    }
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        x[i] = xs[i].x;
        x[N + i] = xs[i].y;
    }
}

// sense-counting grid barrier for a cooperative launch (all CTAs resident)
__device__ __forceinline__ void mc_grid_barrier(unsigned *count, unsigned *gen,
                                                unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g0 = *(volatile unsigned *)gen;
        __threadfence();
        if (atomicAdd(count, 1u) == nblocks - 1) {
            *(volatile unsigned *)count = 0u;
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (*(volatile unsigned *)gen == g0) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void __launch_bounds__(256)
    k_p1_mc_grid(int n1, int forward, const double *__restrict__ T,
                 double *__restrict__ x, double *__restrict__ r, unsigned *bar) {
    const int per_row = (n1 + 6) / 7;
    const int64_t count = (int64_t)per_row * n1;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int b = 0; b < kMcColours; ++b) {
        const int cm = forward ? b : kMcColours - 1 - b;
        for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count;
             k += stride) {
            const int iy = (int)(k / per_row), jj = (int)(k - (int64_t)iy * per_row);
            const int ix = ((cm - 2 * iy) % 7 + 7) % 7 + 7 * jj;
            if (ix < n1) p1_mc_vertex(ix, iy, n1, forward != 0, T, x, r);
        }
        if (b < kMcColours - 1) mc_grid_barrier(bar, bar + 1, gridDim.x);
    }
}

}  // namespace ocmg
