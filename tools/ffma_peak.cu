// FP32 issue-rate microbenchmark behind the roofline denominator (SURVEY §8(d).2 "measure it";
// check whether 128 FFMA/clk/SM is reachable).  Every SM filled (4 CTAs x 512 threads),
// 8 independent chains per thread, timed with CUDA events, best of 5.  Forms:
//   ffma_reg   a = fma(a, b, c), all three operands registers (b, c shared by the chains: the
//              operand-reuse cache can serve them)
//   ffma_reg3  a = fma(a, b_i, c_i), distinct register b_i / c_i per chain (no reuse)
//   ffma_imm   a = fma(a, b, 1.0e-3f): c an immediate (the FFMA imm form)
//   fmul_imm   a = a * 0.999f
//   fadd_reg   a = a + c
//   hfma2      packed fp16 a = fma(a, b, c) on half2 (2 flops x 2 lanes)
// Prints one JSON line: TFLOP/s per form (FMA = 2 flops; hfma2 = 4 flops per lane-instruction) and
// the per-SM per-clock instruction rate at the attribute clock.
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

template <int FORM>
__global__ void chains(float *out, int iters, float b, float c) {
    float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    float b1 = b + 1e-7f, c1 = c - 1e-7f, b2 = b + 2e-7f, c2 = c - 2e-7f, b3 = b + 3e-7f, c3 = c - 3e-7f;
    float b4 = b + 4e-7f, c4 = c - 4e-7f, b5 = b + 5e-7f, c5 = c - 5e-7f, b6 = b + 6e-7f, c6 = c - 6e-7f;
    float b7 = b + 7e-7f, c7 = c - 7e-7f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            if (FORM == 0) {
                a0 = fmaf(a0, b, c); a1 = fmaf(a1, b1, c1); a2 = fmaf(a2, b, c1); a3 = fmaf(a3, b1, c);
                a4 = fmaf(a4, b, c); a5 = fmaf(a5, b1, c1); a6 = fmaf(a6, b, c1); a7 = fmaf(a7, b1, c);
            } else if (FORM == 1) {
                a0 = fmaf(a0, b, c); a1 = fmaf(a1, b1, c1); a2 = fmaf(a2, b2, c2); a3 = fmaf(a3, b3, c3);
                a4 = fmaf(a4, b4, c4); a5 = fmaf(a5, b5, c5); a6 = fmaf(a6, b6, c6); a7 = fmaf(a7, b7, c7);
            } else if (FORM == 2) {
                a0 = fmaf(a0, b, 1.0e-3f); a1 = fmaf(a1, b1, 1.0e-3f); a2 = fmaf(a2, b, 1.0e-3f); a3 = fmaf(a3, b1, 1.0e-3f);
                a4 = fmaf(a4, b, 1.0e-3f); a5 = fmaf(a5, b1, 1.0e-3f); a6 = fmaf(a6, b, 1.0e-3f); a7 = fmaf(a7, b1, 1.0e-3f);
            } else if (FORM == 3) {
                a0 *= 0.999f; a1 *= 0.999f; a2 *= 0.999f; a3 *= 0.999f; a4 *= 0.999f; a5 *= 0.999f; a6 *= 0.999f; a7 *= 0.999f;
            } else {
                a0 += c; a1 += c1; a2 += c; a3 += c1; a4 += c; a5 += c1; a6 += c; a7 += c1;
            }
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void hchains(float *out, int iters, float b, float c) {
    __half2 a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = __floats2half2_rn(threadIdx.x * 1e-3f + j, j);
    const __half2 hb = __floats2half2_rn(b, b), hc = __floats2half2_rn(c, c);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k)
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = __hfma2(a[j], hb, hc);
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += __low2float(a[j]) + __high2float(a[j]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
static float best_ms(K kern, float *out, int blocks, int threads, int iters) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    kern<<<blocks, threads>>>(out, 64, 0.999f, 1e-3f);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        kern<<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const int threads = 512, blocks = sms * 4, iters = 4096;
    float *out;
    cudaMalloc(&out, (size_t)threads * blocks * sizeof(float));
    const double inst = 8.0 * 16 * (double)iters * threads * blocks;   // lane-instructions per launch
    const char *names[] = {"ffma_reg", "ffma_reg3", "ffma_imm", "fmul_imm", "fadd_reg"};
    const double flops_per[] = {2, 2, 2, 1, 1};
    float ms[5];
    ms[0] = best_ms(chains<0>, out, blocks, threads, iters);
    ms[1] = best_ms(chains<1>, out, blocks, threads, iters);
    ms[2] = best_ms(chains<2>, out, blocks, threads, iters);
    ms[3] = best_ms(chains<3>, out, blocks, threads, iters);
    ms[4] = best_ms(chains<4>, out, blocks, threads, iters);
    const float msh = best_ms(hchains, out, blocks, threads, iters);
    printf("{\"sms\": %d, \"clock_mhz_attr\": %d", sms, clk / 1000);
    for (int f = 0; f < 5; ++f)
        printf(", \"%s\": {\"tflops\": %.2f, \"lane_inst_per_clk_per_sm\": %.1f}", names[f],
               inst * flops_per[f] / ms[f] / 1e9, inst / (ms[f] * 1e-3) / sms / (clk * 1e3));
    printf(", \"hfma2\": {\"tflops\": %.2f, \"lane_inst_per_clk_per_sm\": %.1f}}\n", inst * 4 / msh / 1e9,
           inst / (msh * 1e-3) / sms / (clk * 1e3));
    return 0;
}
