// Co-issue microbenchmark: can MUFU.EX2 and FFMA2 run at their
// full rates concurrently on one SM?  Each thread runs NF independent FFMA2
// chains and NM independent EX2 chains per iteration; rates are reported per SM
// per clock (FMA lane-ops and EX2 lane-ops).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipe_mix tools/pipe_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float lo(u64 a) { float x, y; asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(a)); return x; }

template <int NF, int NM>
__global__ void mix(float *out, float a, float b, int iters) {
    u64 f[NF > 0 ? NF : 1];
    float m[NM > 0 ? NM : 1];
    const u64 A = pk(a, a), B = pk(b, b);
#pragma unroll
    for (int j = 0; j < NF; ++j) f[j] = pk(threadIdx.x * 1e-3f + j, j);
#pragma unroll
    for (int j = 0; j < NM; ++j) m[j] = -(threadIdx.x & 7) * 0.01f - j * 0.03f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < (NF > NM ? NF : NM); ++j) {
            if (j < NF) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(f[j]) : "l"(A), "l"(B));
            if (j < NM) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(m[j]));
        }
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < NF; ++j) s += lo(f[j]);
#pragma unroll
    for (int j = 0; j < NM; ++j) s += m[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NF, int NM>
void run(int threads, float *d, int sms, double ghz) {
    const int iters = 2048, blocks = sms * (2048 / threads);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    mix<NF, NM><<<blocks, threads>>>(d, 0.999f, 1e-3f, 16);
    cudaEventRecord(e0);
    mix<NF, NM><<<blocks, threads>>>(d, 0.999f, 1e-3f, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double thr = (double)blocks * threads * iters;
    const double clk = ms * 1e-3 * ghz * 1e9 * sms;
    printf("{\"NF_ffma2\": %d, \"NM_ex2\": %d, \"threads\": %d, \"fma_lanes_per_sm_clk\": %.1f, \"ex2_per_sm_clk\": %.2f, \"ms\": %.3f}\n",
           NF, NM, threads, thr * NF * 2 / clk, thr * NM / clk, ms);
}

int main() {
    int dev = 0, sms = 0, khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev);
    const double ghz = khz / 1e6;
    float *d;
    cudaMalloc(&d, sizeof(float) * sms * 2048);
    run<16, 0>(256, d, sms, ghz);
    run<0, 8>(256, d, sms, ghz);
    run<16, 8>(256, d, sms, ghz);
    run<16, 4>(256, d, sms, ghz);
    run<16, 2>(256, d, sms, ghz);
    run<8, 8>(256, d, sms, ghz);
    run<12, 6>(256, d, sms, ghz);
    run<16, 8>(128, d, sms, ghz);
    run<16, 8>(512, d, sms, ghz);
    printf("{\"err\": \"%s\", \"ghz_attr\": %.3f}\n", cudaGetErrorString(cudaGetLastError()), ghz);
    return 0;
}
