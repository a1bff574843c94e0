// pipe_microbench.cu -- measures per-SM issue rates of MUFU.EX2, FFMA and FFMA2 on this B200
// (the roofline denominators of DESIGN.md §8).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_ex2(float *out, int iters) {
    float a[8];
    for (int i = 0; i < 8; ++i) a[i] = -1e-3f * (threadIdx.x + i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float y;
            asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a[i]));
            a[i] = y * -0.5f;   // FMUL keeps the chain; 1 MUFU + 1 FMUL per element
        }
    }
    float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 1234.5f) out[0] = s;
}

__global__ void k_ffma(float *out, int iters) {
    float a[8], b = 1.0001f, c = 1e-7f;
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = __fmaf_rn(a[i], b, c);
    }
    float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 1234.5f) out[0] = s;
}

__global__ void k_ffma2(float *out, int iters) {
    float2 a[8], b = make_float2(1.0001f, 0.9999f), c = make_float2(1e-7f, 2e-7f);
    for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x + i, i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], b, c);
    }
    float s = 0; for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
    if (s == 1234.5f) out[0] = s;
}

// 3 distinct register operands per FMA (no immediates, no repeated registers)
__global__ void k_ffma_3reg(float *out, int iters) {
    float a[8], b[8], c[8];
    for (int i = 0; i < 8; ++i) {  // runtime values: no immediate forms
        a[i] = threadIdx.x + i;
        b[i] = 1.0f + out[1 + i] * (i + 1);
        c[i] = out[9 + i] * (i + threadIdx.x);
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = __fmaf_rn(a[i], b[i], c[i]);
    }
    float s = 0; for (int i = 0; i < 8; ++i) s += a[i] + b[i] + c[i];
    if (s == 1234.5f) out[0] = s;
}

// FFMA2 with three distinct register pairs
__global__ void k_ffma2_3pair(float *out, int iters) {
    float2 a[8], b[8], c[8];
    for (int i = 0; i < 8; ++i) {
        a[i] = make_float2(threadIdx.x + i, i);
        b[i] = make_float2(1.0f + out[1 + i], 1.0f - out[1 + i]);
        c[i] = make_float2(out[9 + i] * (i + threadIdx.x), out[9 + i] * i);
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], b[i], c[i]);
    }
    float s = 0; for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y + b[i].x + c[i].y;
    if (s == 1234.5f) out[0] = s;
}

// FFMA2 with a broadcast scalar (per-i) and two register pairs
__global__ void k_ffma2_bcast(float *out, int iters) {
    float2 a[8], c[8];
    float b[8];
    for (int i = 0; i < 8; ++i) {
        a[i] = make_float2(threadIdx.x + i, i);
        b[i] = 1.0f + out[1 + i] * (i + threadIdx.x);
        c[i] = make_float2(out[9 + i] * (i + threadIdx.x), out[9 + i] * i);
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], make_float2(b[i], b[i]), c[i]);
    }
    float s = 0; for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y + b[i] + c[i].y;
    if (s == 1234.5f) out[0] = s;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    float *out;
    cudaMalloc(&out, 64 * sizeof(float));
    cudaMemset(out, 0, 64 * sizeof(float));
    const int iters = 20000, threads = 512, blocks = sms * 4;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    struct { const char *name; void (*k)(float *, int); double ops_per_elem; } ks[] = {
        {"ex2 (+1 FMUL)", k_ex2, 1.0}, {"ffma", k_ffma, 1.0}, {"ffma2 (2 FMA each)", k_ffma2, 2.0},
        {"ffma 3 distinct regs", k_ffma_3reg, 1.0}, {"ffma2 3 distinct pairs", k_ffma2_3pair, 2.0},
        {"ffma2 broadcast scalar", k_ffma2_bcast, 2.0}};
    for (auto &kk : ks) {
        kk.k<<<blocks, threads>>>(out, 100);
        cudaEventRecord(a);
        kk.k<<<blocks, threads>>>(out, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double ops = (double)blocks * threads * iters * 8 * kk.ops_per_elem;
        printf("{\"op\": \"%s\", \"per_s\": %.4e, \"per_sm_per_clk_at_max\": %.2f, \"ms\": %.3f, \"sms\": %d, \"max_clock_mhz\": %d}\n",
               kk.name, ops / (ms * 1e-3), ops / (ms * 1e-3) / sms / (clk * 1e3), ms, sms, clk / 1000);
    }
    return 0;
}
