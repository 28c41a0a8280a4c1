// Legacy warp-level mma.sync m16n8k8 TF32 throughput on sm_100a (is it worth moving the cuboid
// screen's affine transform onto tensor cores?).  8 independent accumulator chains per warp,
// 8 warps per CTA, 2 CTAs per SM; also an FFMA-interleaved variant (the screen would mix both).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma_tf32(float (&d)[4], const unsigned (&a)[4], const unsigned (&b)[2]) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};\n"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

__device__ __forceinline__ void mma_tf32_k4(float (&d)[4], const unsigned (&a)[4], const unsigned (&b)[2]) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
                 "{%0,%1,%2,%3};\n"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(b[0]));
}
__device__ __forceinline__ void mma_f16_k16(float (&d)[4], const unsigned (&a)[4], const unsigned (&b)[2]) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};\n"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
template <int KIND>
__device__ __forceinline__ void mma_any(float (&d)[4], const unsigned (&a)[4], const unsigned (&b)[2]) {
    if (KIND == 0) mma_tf32(d, a, b); else if (KIND == 1) mma_tf32_k4(d, a, b); else mma_f16_k16(d, a, b);
}
template <int FFMA_PER_MMA, int KIND = 0>
__global__ void __launch_bounds__(256, 2) mma_chains(float *out, int iters) {
    unsigned a[4], b[2];
    for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(1e-3f * (threadIdx.x + i));
    for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(1e-3f * (threadIdx.x - i));
    float acc[8][4];
    for (int c = 0; c < 8; ++c)
        for (int i = 0; i < 4; ++i) acc[c][i] = 0.f;
    float f0 = threadIdx.x, f1 = f0 + 1, f2 = f0 + 2, f3 = f0 + 3;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            mma_any<KIND>(acc[c], a, b);
#pragma unroll
            for (int k = 0; k < FFMA_PER_MMA / 4; ++k) {
                f0 = fmaf(f0, 0.999f, 1e-3f); f1 = fmaf(f1, 0.999f, 1e-3f);
                f2 = fmaf(f2, 0.999f, 1e-3f); f3 = fmaf(f3, 0.999f, 1e-3f);
            }
        }
    }
    float s = f0 + f1 + f2 + f3;
    for (int c = 0; c < 8; ++c)
        for (int i = 0; i < 4; ++i) s += acc[c][i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int F, int KIND = 0>
void run(int sms, float *out) {
    const int threads = 256, blocks = sms * 2, iters = 2048;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    mma_chains<F, KIND><<<blocks, threads>>>(out, 16);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        mma_chains<F, KIND><<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double mmas = (double)blocks * (threads / 32) * iters * 8;
    const int kk = KIND == 0 ? 8 : KIND == 1 ? 4 : 16;
    const double tf = mmas * 16 * 8 * kk * 2 / (best * 1e-3) / 1e12;
    const double ffma = (double)blocks * threads * iters * 8 * F;
    printf("{\"kind\": \"%s\", \"ffma_per_mma\": %d, \"ms\": %.3f, \"mma_per_sm_per_us\": %.1f, \"tf32_tflops\": %.1f, "
           "\"ffma_tflops\": %.1f}\n", KIND == 0 ? "tf32_m16n8k8" : KIND == 1 ? "tf32_m16n8k4" : "f16_m16n8k16", F, best, mmas / sms / (best * 1e3), tf, ffma * 2 / (best * 1e-3) / 1e12);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out;
    cudaMalloc(&out, (size_t)sms * 2 * 256 * sizeof(float));
    run<0>(sms, out);
    run<4>(sms, out);
    run<8>(sms, out);
    run<16>(sms, out);
    run<0, 1>(sms, out);
    run<8, 1>(sms, out);
    run<16, 1>(sms, out);
    run<0, 2>(sms, out);
    run<16, 2>(sms, out);
    return 0;
}
