// Shared plumbing for the ocmg_b200 CUDA library: error handling, device
// buffers, launch helpers, deterministic reductions.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ocmg_b200.h"

namespace ocmg {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

#define OCMG_CUDA(expr)                                                      \
    do {                                                                     \
        cudaError_t e_ = (expr);                                             \
        if (e_ != cudaSuccess)                                               \
            throw ::ocmg::Error(OCMG_E_CUDA, std::string(#expr) + ": " +     \
                                                 cudaGetErrorString(e_));    \
    } while (0)

#define OCMG_REQUIRE(cond, msg)                                              \
    do {                                                                     \
        if (!(cond)) throw ::ocmg::Error(OCMG_E_ARG, (msg));                 \
    } while (0)

#define OCMG_LAUNCH_CHECK() OCMG_CUDA(cudaGetLastError())

// Every kernel launch of the library goes through OCMG_LAUNCH so that the
// number of device kernels a call issued can be reported (bench.py's
// gpu_launches comes from ocmg_launch_count, not from an estimate).
inline std::atomic<long long> &launch_counter() {
    static std::atomic<long long> c{0};
    return c;
}
#define OCMG_LAUNCH(kernel, grid, block, smem, stream, ...)                  \
    do {                                                                     \
        ::ocmg::launch_counter().fetch_add(1, std::memory_order_relaxed);    \
        kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);          \
    } while (0)

// The same with programmatic dependent launch: the grid may be scheduled
// while the previous kernel on the stream is still running; the kernel must
// execute griddepcontrol.wait (pdl_wait) before touching what that kernel
// writes.  Used for chains of short dependent launches (one per dependency
// level), where it hides the launch latency behind the previous level.
#define OCMG_LAUNCH_PDL(kernel, grid, block, smem, strm_, ...)                \
    do {                                                                     \
        ::ocmg::launch_counter().fetch_add(1, std::memory_order_relaxed);    \
        cudaLaunchConfig_t cfg_{};                                           \
        cfg_.gridDim = dim3(grid);                                           \
        cfg_.blockDim = dim3(block);                                         \
        cfg_.dynamicSmemBytes = (smem);                                      \
        cfg_.stream = (strm_);                                               \
        cudaLaunchAttribute at_[1];                                          \
        at_[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;      \
        at_[0].val.programmaticStreamSerializationAllowed = 1;               \
        cfg_.attrs = at_;                                                    \
        cfg_.numAttrs = 1;                                                   \
        OCMG_CUDA(cudaLaunchKernelEx(&cfg_, kernel, __VA_ARGS__));           \
    } while (0)

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Owning device allocation (cudaMalloc/cudaFree).
template <class T>
struct DevBuf {
    T *p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    DevBuf(DevBuf &&o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DevBuf &operator=(DevBuf &&o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t count) {
        release();
        n = count;
        if (count) OCMG_CUDA(cudaMalloc(&p, count * sizeof(T)));
    }
    void upload(const T *host, size_t count) {
        alloc(count);
        if (count)
            OCMG_CUDA(cudaMemcpy(p, host, count * sizeof(T),
                                 cudaMemcpyHostToDevice));
    }
    void upload(const std::vector<T> &v) { upload(v.data(), v.size()); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

inline unsigned grid_for(int64_t work, int block) {
    int64_t g = (work + block - 1) / block;
    if (g < 1) g = 1;
    if (g > 2147483647LL) g = 2147483647LL;
    return static_cast<unsigned>(g);
}

// ---------------------------------------------------------------------------
// deterministic two-pass reductions (fixed grid, fixed tree) so that repeated
// solves give bit-identical norms and means.
// ---------------------------------------------------------------------------
constexpr int kRedBlock = 256;
constexpr int kRedGrid = 592;  // 4 x 148 SMs

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double block_sum(double v, double *sh) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v = warp_sum(v);
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    const int nw = blockDim.x >> 5;
    v = (threadIdx.x < nw) ? sh[threadIdx.x] : 0.0;
    if (wid == 0) v = warp_sum(v);
    __syncthreads();
    return v;
}

// partial[b] = sum over a grid-strided slice of w_i * x_i^2 (w may be null)
__global__ void k_sumsq_partial(int64_t n, const double *__restrict__ x,
                                const double *__restrict__ w,
                                double *__restrict__ partial) {
    __shared__ double sh[32];
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double v = x[i];
        acc += (w ? w[i] * v : v) * v;
    }
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

// partial[b] = sum of x_i over a grid-strided slice of [lo, hi)
__global__ void k_sum_partial(int64_t lo, int64_t hi,
                              const double *__restrict__ x,
                              double *__restrict__ partial) {
    __shared__ double sh[32];
    double acc = 0.0;
    for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
         i < hi; i += (int64_t)gridDim.x * blockDim.x)
        acc += x[i];
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

// out[0] = sum(partial[0..m)) / divisor   (divisor 1 for plain sums; the
// count for a mean, matching numpy's sum/n rather than sum*(1/n))
__global__ void k_finish_sum(int m, const double *__restrict__ partial,
                             double divisor, double *__restrict__ out) {
    __shared__ double sh[32];
    double acc = 0.0;
    for (int i = threadIdx.x; i < m; i += blockDim.x) acc += partial[i];
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) out[0] = acc / divisor;
}

// x[lo:hi) -= *mean
__global__ void k_sub_scalar(int64_t lo, int64_t hi, double *__restrict__ x,
                             const double *__restrict__ mean) {
    const int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < hi) x[i] -= mean[0];
}

}  // namespace ocmg
