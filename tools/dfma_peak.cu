// dfma_peak.cu -- measured fp64 FMA (DFMA) throughput of the GPU, for bench.py's fp64-pipe
// figures ("measure it with a DFMA microbenchmark before quoting fp64-pipe
// utilisation").  Independent chains of fused multiply-adds per thread, a full grid of 148 x 8
// blocks; prints one JSON line {"dfma_tflops": ..., "ops_per_clock_per_sm": ...}.
// (A measurement tool: not part of libcem.)
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) k_dfma(double *out, int iters, double s) {
    double a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(a[i], s, 1e-7);
    double t = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += a[i];
    if (t == 12345.678) out[0] = t;  // keeps the chains alive
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);  // kHz
    double *out;
    cudaMalloc(&out, 8);
    const int blocks = sms * 8, iters = 4096;
    k_dfma<<<blocks, 256>>>(out, 64, 0.999999);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_dfma<<<blocks, 256>>>(out, iters, 0.999999);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double fmas = (double)blocks * 256.0 * iters * 8.0;
    const double tflops = 2.0 * fmas / (best * 1e-3) / 1e12;
    const double per_clk_sm = fmas / (best * 1e-3) / ((double)clk * 1e3) / sms;
    printf("{\"dfma_tflops\": %.3f, \"dfma_per_clock_per_sm\": %.2f, \"sms\": %d, \"max_clock_mhz\": %.0f, "
           "\"ms\": %.4f}\n", tflops, per_clk_sm, sms, clk / 1e3, best);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
