// Pipe-throughput microbenchmarks on the B200: FP32 FFMA,
// packed FFMA2 (fma.rn.f32x2), MUFU.EX2 and an FFMA2+EX2 mix.  Prints one JSON
// line with the measured per-SM per-clock rates and the FP32 FLOP/s peak that
// DESIGN.md §8.3 uses as the measured roofline denominator.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096

__device__ __forceinline__ unsigned long long pk(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float2 upk(unsigned long long v) {
    float a, b;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
    return make_float2(a, b);
}
__device__ __forceinline__ void fma2(unsigned long long &d, unsigned long long a, unsigned long long b) {
    asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}
__device__ __forceinline__ float ex2(float x) {
    float r;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__global__ void k_ffma(float *out, float a, float b) {
    float x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3f + j;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fmaf(x[j], a, b);
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2(float *out, float a, float b) {
    unsigned long long x[8];
    const unsigned long long A = pk(a, a), B = pk(b, b);
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = pk(threadIdx.x * 1e-3f + j, j * 0.5f);
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            unsigned long long d = B;
            fma2(d, x[j], A);
            x[j] = d;
        }
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) { float2 v = upk(x[j]); s += v.x + v.y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ex2(float *out, float a) {
    float x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = -(threadIdx.x & 7) * 0.01f - j * 0.1f;
    for (int i = 0; i < ITERS / 4; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = ex2(x[j]) * a;  // 1 MUFU + 1 FMUL
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_mix(float *out, float a, float b) {  // 1 EX2 : 4 FFMA2 : 1 FMUL
    unsigned long long x[8];
    float y[4];
    const unsigned long long A = pk(a, a), B = pk(b, b);
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = pk(threadIdx.x * 1e-3f + j, j * 0.5f);
#pragma unroll
    for (int j = 0; j < 4; ++j) y[j] = -(threadIdx.x & 7) * 0.01f - j * 0.1f;
    for (int i = 0; i < ITERS / 4; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            unsigned long long d = B;
            fma2(d, x[j], A);
            x[j] = d;
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) y[j] = ex2(y[j]) * a;
    }
    float s = y[0] + y[1] + y[2] + y[3];
#pragma unroll
    for (int j = 0; j < 8; ++j) { float2 v = upk(x[j]); s += v.x + v.y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class F>
float time_ms(F f) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    f();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 5;
}

int main() {
    int dev = 0, sms = 0, clk_khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    const int threads = 256, blocks = sms * 8;
    float *out;
    cudaMalloc(&out, sizeof(float) * threads * blocks);
    const double nthr = (double)threads * blocks;
    const double ghz = clk_khz / 1e6;
    float t1 = time_ms([&] { k_ffma<<<blocks, threads>>>(out, 0.999f, 1e-3f); });
    float t2 = time_ms([&] { k_ffma2<<<blocks, threads>>>(out, 0.999f, 1e-3f); });
    float t3 = time_ms([&] { k_ex2<<<blocks, threads>>>(out, 0.5f); });
    float t4 = time_ms([&] { k_mix<<<blocks, threads>>>(out, 0.999f, 1e-3f); });
    cudaError_t e = cudaGetLastError();
    const double ffma_s = nthr * ITERS * 8 / (t1 * 1e-3);          // FMA / s
    const double ffma2_s = nthr * ITERS * 8 * 2 / (t2 * 1e-3);     // FMA / s
    const double ex2_s = nthr * (ITERS / 4) * 8 / (t3 * 1e-3);     // EX2 / s
    const double mix_fma_s = nthr * (ITERS / 4) * 16 / (t4 * 1e-3);
    const double mix_ex2_s = nthr * (ITERS / 4) * 2 / (t4 * 1e-3);
    printf("{\"sms\": %d, \"attr_clock_ghz\": %.3f, \"err\": \"%s\", "
           "\"ffma_tflops\": %.2f, \"ffma2_tflops\": %.2f, \"ex2_per_s\": %.4e, "
           "\"ffma_per_sm_clk\": %.1f, \"ffma2_fma_per_sm_clk\": %.1f, \"ex2_per_sm_clk\": %.2f, "
           "\"mix_fma_per_sm_clk\": %.1f, \"mix_ex2_per_sm_clk\": %.2f, \"ms\": [%.3f, %.3f, %.3f, %.3f]}\n",
           sms, ghz, cudaGetErrorString(e), 2 * ffma_s / 1e12, 2 * ffma2_s / 1e12, ex2_s,
           ffma_s / sms / (ghz * 1e9), ffma2_s / sms / (ghz * 1e9), ex2_s / sms / (ghz * 1e9),
           mix_fma_s / sms / (ghz * 1e9), mix_ex2_s / sms / (ghz * 1e9), t1, t2, t3, t4);
    return 0;
}
