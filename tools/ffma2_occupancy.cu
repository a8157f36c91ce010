// FFMA2 throughput vs warps per SMSP and independent chains per thread:
// the stage kernel runs 2 conv warps per SMSP with 10 accumulator pairs each.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ffma2_occupancy tools/ffma2_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float lo(u64 a) { float x, y; asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(a)); return x + y * 0.f; }

template <int NC>
__global__ void chains(float *out, float k, int iters) {
    u64 acc[NC];
    const u64 x = pk(threadIdx.x * 1e-3f, 1.0f);
#pragma unroll
    for (int j = 0; j < NC; ++j) acc[j] = pk(j, -j);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < NC; ++j)
            asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[j]) : "l"(x), "l"(pk(k, k)));
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < NC; ++j) s += lo(acc[j]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NC>
void run(int warps_per_sm, int sms, double ghz, float *d) {
    const int iters = 20000 / NC * 10;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    chains<NC><<<sms, 32 * warps_per_sm>>>(d, 0.9999f, 10);
    cudaEventRecord(e0);
    chains<NC><<<sms, 32 * warps_per_sm>>>(d, 0.9999f, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double fma = (double)sms * 32 * warps_per_sm * iters * NC * 2;
    printf("{\"warps_per_smsp\": %d, \"chains\": %d, \"fma_lanes_per_sm_clk\": %.1f}\n", warps_per_sm / 4, NC,
           fma / (ms * 1e-3 * ghz * 1e9 * sms));
}

int main() {
    int sms, khz;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    float *d;
    cudaMalloc(&d, sizeof(float) * sms * 1024);
    for (int w : {4, 8, 16}) { run<4>(w, sms, khz / 1e6, d); run<10>(w, sms, khz / 1e6, d); run<20>(w, sms, khz / 1e6, d); }
    return 0;
}
