// FP64 pipe microbenchmark (SURVEY §7 step 0 / §8(d) ceilings): DFMA and DADD throughput of one
// B200, measured with CUDA events. Every thread runs 8 independent dependency chains (ILP 8) of
// `iters` instructions; grid = 148 SMs x 8 CTAs x 256 threads. Prints one JSON line:
//   {"dfma_tflops": ..., "dadd_gops": ..., "sm_count": ..., "clock_mhz": ...}
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/fp64_peak scripts/microbench/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <bool FMA>
__global__ void k_chain(double *out, double a, double b, int iters) {
    double x0 = threadIdx.x * 1e-9, x1 = x0 + 1e-9, x2 = x0 + 2e-9, x3 = x0 + 3e-9;
    double x4 = x0 + 4e-9, x5 = x0 + 5e-9, x6 = x0 + 6e-9, x7 = x0 + 7e-9;
#pragma unroll 4
    for (int i = 0; i < iters; i++) {
        if (FMA) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        } else {
            x0 = x0 + a; x1 = x1 + b; x2 = x2 + a; x3 = x3 + b;
            x4 = x4 + a; x5 = x5 + b; x6 = x6 + a; x7 = x7 + b;
        }
    }
    const double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 12345.678) out[0] = s;     // keeps the chains alive
}

template <bool FMA>
static double run(int sms, double *d) {
    const int blocks = sms * 8, threads = 256, iters = 1 << 14;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_chain<FMA><<<blocks, threads>>>(d, 0.999999, 1e-7, iters);   // warm-up
    float best = 1e30f;
    for (int r = 0; r < 5; r++) {
        cudaEventRecord(e0);
        k_chain<FMA><<<blocks, threads>>>(d, 0.999999, 1e-7, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double ops = (double)blocks * threads * iters * 8.0;          // instructions (one per lane)
    return ops / (best * 1e-3);
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    double *d;
    cudaMalloc(&d, 8);
    const double fma_ips = run<true>(p.multiProcessorCount, d);
    const double add_ips = run<false>(p.multiProcessorCount, d);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("{\"dfma_tflops\": %.3f, \"dadd_gops\": %.1f, \"fp64_lanes_per_sm_per_clk\": %.2f, \"sm_count\": %d, "
           "\"clock_mhz\": %.0f, \"how\": \"8 independent DFMA/DADD chains per thread, %d x 8 CTAs x 256 threads, "
           "best of 5, CUDA events\"}\n",
           2.0 * fma_ips / 1e12, add_ips / 1e9, fma_ips / (p.multiProcessorCount * (clk * 1e3)), p.multiProcessorCount,
           clk / 1e3, p.multiProcessorCount);
    return cudaGetLastError() != cudaSuccess;
}
