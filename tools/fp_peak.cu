// Measured FP64 / FP32 FMA peak of the device (the compute roofline of the CG operator kernels).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/fp_peak.cu -o tools/fp_peak
// Each thread runs 8 independent FMA chains; grid = 148 SMs x 8 CTAs x 256 threads.
#include <cstdio>
#include <cuda_runtime.h>

template <class T>
__global__ void k_fma(T* out, int iters, T a, T b) {
    T x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = static_cast<T>(threadIdx.x + j);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = x[j] * a + b;
    }
    T s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    if (s == static_cast<T>(-1.2345)) out[0] = s;
}

template <class T>
double run(const char* name) {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    T* out;
    cudaMalloc(&out, sizeof(T));
    const int blocks = sms * 8, threads = 256, iters = 4096;
    k_fma<T><<<blocks, threads>>>(out, 16, T(0.999), T(1e-3));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_fma<T><<<blocks, threads>>>(out, iters, T(0.999), T(1e-3));
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double fma = double(blocks) * threads * iters * 16 * 8;
    const double tf = 2.0 * fma / (best * 1e-3) / 1e12;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    printf("{\"type\": \"%s\", \"tflops\": %.2f, \"fma_per_clk_per_sm_at_max_clock\": %.1f, \"sms\": %d, \"max_clock_mhz\": %d}\n",
           name, tf, fma / (best * 1e-3) / sms / (clk * 1e3), sms, clk / 1000);
    cudaFree(out);
    return tf;
}

// dependent-chain latency of one FMA (one thread, clock64 around 1024 chained FMAs)
template <class T>
__global__ void k_lat(T* out, long long* cyc, T a, T b) {
    T x = static_cast<T>(threadIdx.x);
    const long long t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < 1024; ++i) x = x * a + b;
    const long long t1 = clock64();
    out[0] = x;
    cyc[0] = t1 - t0;
}
template <class T>
void lat(const char* name) {
    T* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(T));
    cudaMalloc(&cyc, sizeof(long long));
    long long best = 1LL << 60;
    for (int r = 0; r < 3; ++r) {
        k_lat<T><<<1, 1>>>(out, cyc, T(0.999), T(1e-3));
        long long c;
        cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
        if (c < best) best = c;
    }
    printf("{\"type\": \"%s latency\", \"cycles_per_dependent_fma\": %.2f}\n", name, best / 1024.0);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    run<double>("fp64 DFMA");
    run<float>("fp32 FFMA");
    lat<double>("fp64 DFMA");
    lat<float>("fp32 FFMA");
    return 0;
}
