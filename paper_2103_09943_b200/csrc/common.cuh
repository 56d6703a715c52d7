// common.cuh -- shared device/host infrastructure for the sm_100a blind-pansharpening path.
#pragma once

#include <cuda_runtime.h>
#include <cufft.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "fbmp_gpu.h"

namespace fbmp_gpu {

// ---------------------------------------------------------------------------------------
// Errors: the reference taxonomy (errors.hpp:8-33) as status codes at the C ABI.
// ---------------------------------------------------------------------------------------
struct Failure : std::runtime_error {
    int code;
    Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void param_error(const std::string& m) { throw Failure(FBMP_PARAM_ERROR, m); }
[[noreturn]] inline void dim_error(const std::string& m) { throw Failure(FBMP_DIMENSION_ERROR, m); }
[[noreturn]] inline void num_error(const std::string& m) { throw Failure(FBMP_NUMERICAL_ERROR, m); }

#define FBMP_NCCL(call)                                                                          \
    do {                                                                                         \
        const int rc_ = static_cast<int>(call);                                                  \
        if (rc_ != 0) throw ::fbmp_gpu::Failure(4, std::string("NCCL error ") + std::to_string(rc_) + " at " #call); \
    } while (0)

#define FBMP_CUDA(call)                                                                          \
    do {                                                                                         \
        cudaError_t e_ = (call);                                                                 \
        if (e_ != cudaSuccess)                                                                   \
            throw ::fbmp_gpu::Failure(FBMP_RUNTIME_ERROR, std::string("CUDA error: ") +          \
                                                              cudaGetErrorString(e_) + " at " +  \
                                                              __FILE__ + ":" + std::to_string(__LINE__)); \
    } while (0)

#define FBMP_CUFFT(call)                                                                         \
    do {                                                                                         \
        cufftResult r_ = (call);                                                                 \
        if (r_ != CUFFT_SUCCESS)                                                                 \
            throw ::fbmp_gpu::Failure(FBMP_RUNTIME_ERROR, "cuFFT error " + std::to_string(r_) +  \
                                                              " at " + __FILE__ + ":" +          \
                                                              std::to_string(__LINE__));         \
    } while (0)

// ---------------------------------------------------------------------------------------
// Device buffers
// ---------------------------------------------------------------------------------------
template <class T>
struct DevBuf {
    T* ptr = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) { resize(count); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : ptr(o.ptr), n(o.n) { o.ptr = nullptr; o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) { release(); ptr = o.ptr; n = o.n; o.ptr = nullptr; o.n = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        n = 0;
    }
    void resize(size_t count) {
        if (count <= n && ptr) return;
        release();
        if (count) FBMP_CUDA(cudaMalloc(&ptr, count * sizeof(T)));
        n = count;
    }
    T* get() const { return ptr; }
};

// ---------------------------------------------------------------------------------------
// Context: device, stream, cached workspaces and cuFFT plans.
// ---------------------------------------------------------------------------------------
// Host-side phase trace (env FBMP_TRACE=1): prints the wall time since the previous mark.
inline void trace(const char* what) {
    static const bool on = std::getenv("FBMP_TRACE") != nullptr;
    if (!on) return;
    using clk = std::chrono::steady_clock;
    static thread_local clk::time_point last = clk::now();
    const auto now = clk::now();
    std::fprintf(stderr, "[fbmp] %-28s %9.3f ms\n", what, std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
}

struct Context {
    int device = 0;
    cudaStream_t stream = nullptr;
    long long launches = 0;
    fbmp_gpu_stats stats{};
    std::vector<int> cg_iters_all;  // every channel of the last solve (stats.cg_iters keeps 64)
    std::map<std::string, std::unique_ptr<DevBuf<unsigned char>>> ws;
    std::map<std::tuple<int, int, int, int, int>, cufftHandle> plans;  // (kind, rows, cols, batch, 0)
    int sm_count = 148;
    // kernel profiling of the CG loop (bench.py roofline): total device ms and launches that
    // did work, per kernel class {K_Q, K_D, K_L (or the single K_A), K_U}
    bool profile = false;
    int precision = 64;  // 64: reference precision; 32: fp32 mode of the HRMS CG (north_star)
    double prof_ms[4] = {0, 0, 0, 0};  // K_Q, K_D, K_L (K_A), K_U
    long long prof_n[4] = {0, 0, 0, 0};

    explicit Context(int dev);
    ~Context();
    // named scratch buffer of at least `bytes` (contents undefined, reused across calls)
    template <class T>
    T* scratch(const std::string& name, size_t count) {
        auto& b = ws[name];
        if (!b) b = std::make_unique<DevBuf<unsigned char>>();
        b->resize(count * sizeof(T));
        return reinterpret_cast<T*>(b->get());
    }
    cufftHandle plan(int kind, int rows, int cols, int batch);
    void count(int k = 1) { launches += k; }
    // pinned host staging (grown, never shrunk): cudaMallocHost per call costs 1-300 ms
    void* pinned(size_t bytes);
    void* pinned_buf = nullptr;
    size_t pinned_bytes = 0;
    cudaEvent_t poll_ev[2] = {nullptr, nullptr};  // CG flag polling
    cudaStream_t aux_streams[3] = {nullptr, nullptr, nullptr};  // further CG chains inside the chunk graph
    // host-pointer solves: the HRMS planes are downloaded per channel on copy_stream as soon as
    // each is final (overlapping the remaining channels' last FFT and unscale); null = no sink
    double* host_out = nullptr;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t copy_ev[2] = {nullptr, nullptr};
    cudaEvent_t fork_ev = nullptr, join_evs[3] = {nullptr, nullptr, nullptr};
    // instantiated CG-chunk graphs keyed on their launch parameters (bytes of geometry + pointers)
    std::map<std::string, cudaGraphExec_t> graphs;
    // NCCL communicator of a row-strip (multi-GPU) solve (fbmp_gpu_ctx_set_comm), or null
    void* nccl = nullptr;
    int nranks = 1, rank = 0;
};

// RAII device selection for calls made from arbitrary host threads.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

inline void h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    FBMP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
}
inline void d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    FBMP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
}
inline void check_launch() { FBMP_CUDA(cudaGetLastError()); }

template <class... KArgs, class... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    FBMP_CUDA(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}

inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

// ---------------------------------------------------------------------------------------
// Device helpers
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ int floordiv(int a, int b) {  // b > 0
    return (a >= 0) ? a / b : -((-a + b - 1) / b);
}
__device__ __forceinline__ int wrapi(int a, int m) {
    int r = a % m;
    return r < 0 ? r + m : r;
}

// Programmatic dependent launch (PDL): a kernel launched with launch_pdl may start while its
// predecessor in the stream is still running. pdl_wait() blocks until the predecessor has
// completed and its writes are visible (a no-op for a normal launch); pdl_trigger() lets the
// successor start launching. Rule used by the CG kernels: before pdl_wait() read only data
// that the immediate predecessor does not write; trigger only after the wait.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Deterministic block reduction of one double (fixed shuffle tree + fixed warp order).
// Every thread must call it; the result is valid in all threads.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red /* >= NT/32 + 1 */) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    if (wid == 0) {
        double s = lane < NT / 32 ? red[lane] : 0.0;
        s = warp_sum(s);
        if (lane == 0) red[NT / 32] = s;
    }
    __syncthreads();
    return red[NT / 32];
}

// Two block sums in one pass (same trees as two block_sum calls: identical bits, 3 barriers
// instead of 6). red: >= 2 (NT/32 + 1) doubles.
template <int NT>
__device__ __forceinline__ double2 block_sum2(double a, double b, double* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    a = warp_sum(a);
    b = warp_sum(b);
    __syncthreads();
    if (lane == 0) {
        red[wid] = a;
        red[NT / 32 + 1 + wid] = b;
    }
    __syncthreads();
    if (wid == 0) {
        double x = lane < NT / 32 ? red[lane] : 0.0;
        double y = lane < NT / 32 ? red[NT / 32 + 1 + lane] : 0.0;
        x = warp_sum(x);
        y = warp_sum(y);
        if (lane == 0) {
            red[NT / 32] = x;
            red[2 * (NT / 32) + 1] = y;
        }
    }
    __syncthreads();
    return make_double2(red[NT / 32], red[2 * (NT / 32) + 1]);
}
// Two interleaved partial arrays (stride 2) summed in the fixed order of sum_partials.
template <int NT>
__device__ __forceinline__ double2 sum_partials2(const double* part, int n, double* red) {
    double s0 = 0.0, s1 = 0.0;
    for (int i = threadIdx.x; i < n; i += NT) {
        s0 += __ldcg(part + 2 * static_cast<size_t>(i));
        s1 += __ldcg(part + 2 * static_cast<size_t>(i) + 1);
    }
    return block_sum2<NT>(s0, s1, red);
}

// Sum of a partial array in a fixed order (identical bits in every block that calls it).
template <int NT>
__device__ __forceinline__ double sum_partials(const double* part, int n, int stride, double* red) {
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += NT) s += __ldcg(part + static_cast<size_t>(i) * stride);
    return block_sum<NT>(s, red);
}

// Last-block election (threadFenceReduction pattern). Call after the block's partial
// has been written by thread 0; returns true in every thread of the last block.
__device__ __forceinline__ bool elect_last_block(unsigned int* counter, unsigned int nblocks) {
    __shared__ bool am_last;
    __syncthreads();  // thread 0 wrote the block partial; all threads are past their reads
    if (threadIdx.x == 0) {
        __threadfence();  // publish the partial before the arrival is counted
        const unsigned int prev = atomicAdd(counter, 1u);
        am_last = (prev == nblocks - 1);
        if (am_last) __threadfence();
    }
    __syncthreads();
    return am_last;
}

}  // namespace fbmp_gpu
