// FP32 FFMA throughput microbenchmark (SURVEY §8(d).2 asks for a measured FP32 peak): 8
// independent register-operand FFMA chains per thread, every SM filled, timed with CUDA events.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ffma_chains(float *out, int iters, float b, float c) {
    float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    float b1 = b + 1e-7f, c1 = c - 1e-7f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            a0 = fmaf(a0, b, c); a1 = fmaf(a1, b1, c1); a2 = fmaf(a2, b, c1); a3 = fmaf(a3, b1, c);
            a4 = fmaf(a4, b, c); a5 = fmaf(a5, b1, c1); a6 = fmaf(a6, b, c1); a7 = fmaf(a7, b1, c);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const int threads = 512, blocks = sms * 4, iters = 4096;
    float *out;
    cudaMalloc(&out, (size_t)threads * blocks * sizeof(float));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    ffma_chains<<<blocks, threads>>>(out, 64, 0.999f, 1e-3f);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        ffma_chains<<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double flops = 2.0 * 8 * 16 * (double)iters * threads * blocks;
    printf("{\"ffma_tflops\": %.2f, \"sms\": %d, \"clock_mhz_attr\": %d, \"ms\": %.3f}\n", flops / best / 1e9, sms,
           clk / 1000, best);
    return 0;
}
