// Throughput of the stage kernel's phi core in isolation:
// horner-unit evaluation of NP pairs per thread, no shared memory traffic
// beyond the uniform coefficient loads, no barriers.  Reports SM-cycles per
// warp-unit (one unit of 8 centres for 32 lanes x NP pairs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1510_02930_b200/csrc -o tools/phi_core tools/phi_core.cu
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long f2;
__device__ __forceinline__ f2 pk(float a, float b) { f2 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ f2 bc(float s) { return pk(s, s); }
__device__ __forceinline__ float lo(f2 a) { float x, y; asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(a)); return x; }
__device__ __forceinline__ float hi(f2 a) { float x, y; asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(a)); return y; }
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) { f2 d; asm("fma.rn.f32x2 %0,%1,%2,%3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ f2 mul2(f2 a, f2 b) { f2 d; asm("mul.rn.f32x2 %0,%1,%2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ float ex2(float x) { float r; asm("ex2.approx.ftz.f32 %0,%1;" : "=f"(r) : "f"(x)); return r; }

template <int NP, int VARIANT>
__global__ void core(const float4 *__restrict__ coef, float *out, int nunits, int reps) {
    __shared__ float4 sc[3 * 64];
    for (int j = threadIdx.x; j < 3 * 64; j += blockDim.x) sc[j] = coef[j];
    __syncthreads();
    f2 v[NP], w[NP];
#pragma unroll
    for (int e = 0; e < NP; ++e) { v[e] = pk(0.01f * (threadIdx.x & 31) + e, 0.02f * e); w[e] = 0; }
    const float a_s = 0.03f, two_sg = 1.7f;
    for (int r = 0; r < reps; ++r) {
        for (int u = 0; u < nunits; ++u) {
            const float4 q0 = sc[3 * u], q1 = sc[3 * u + 1], q2 = sc[3 * u + 2];
#pragma unroll
            for (int e = 0; e < NP; ++e) {
                const f2 ys = fma2(v[e], bc(a_s), bc(q0.x));
                const f2 sq = mul2(ys, ys);
                const f2 G = pk(ex2(-lo(sq)), ex2(-hi(sq)));
                const f2 yr = mul2(ys, bc(two_sg));
                const f2 R = pk(ex2(lo(yr)), ex2(hi(yr)));
                if (VARIANT == 0) {
                    const f2 Ri = pk(ex2(-lo(yr)), ex2(-hi(yr)));
                    const f2 pp = fma2(fma2(fma2(R, bc(q2.x), bc(q1.w)), R, bc(q1.z)), R, bc(q1.y));
                    const f2 pm = fma2(fma2(fma2(Ri, bc(q0.y), bc(q0.z)), Ri, bc(q0.w)), Ri, bc(q1.x));
                    w[e] = fma2(G, fma2(pm, Ri, pp), w[e]);
                } else {  // 2 MUFU per element: one-sided degree-7 Horner in R
                    f2 p = fma2(R, bc(q2.x), bc(q1.w));
                    p = fma2(p, R, bc(q1.z)); p = fma2(p, R, bc(q1.y)); p = fma2(p, R, bc(q1.x));
                    p = fma2(p, R, bc(q0.w)); p = fma2(p, R, bc(q0.z)); p = fma2(p, R, bc(q0.y));
                    w[e] = fma2(G, p, w[e]);
                }
            }
        }
        // keep v changing so nothing is hoisted
#pragma unroll
        for (int e = 0; e < NP; ++e) v[e] = fma2(w[e], bc(1e-30f), v[e]);
    }
    float s = 0;
#pragma unroll
    for (int e = 0; e < NP; ++e) s += lo(w[e]) + hi(w[e]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NP, int VARIANT>
void run(int threads, int nunits, float4 *c, float *o, int sms, double ghz) {
    const int reps = 64, blocks = sms;  // one CTA per SM
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    core<NP, VARIANT><<<blocks, threads>>>(c, o, nunits, 2);
    cudaEventRecord(e0);
    core<NP, VARIANT><<<blocks, threads>>>(c, o, nunits, reps);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double warp_units = (double)(threads / 32) * nunits * reps;  // per SM
    const double cyc = ms * 1e-3 * ghz * 1e9;
    printf("{\"NP\": %d, \"variant\": %d, \"warps_per_sm\": %d, \"sm_cycles_per_warp_unit\": %.1f, "
           "\"ex2_per_sm_clk\": %.2f}\n", NP, VARIANT, threads / 32, cyc / warp_units,
           warp_units * 32 * NP * 2 * (VARIANT == 0 ? 3 : 2) / cyc);
}

int main() {
    int sms = 0, khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    float4 *c; float *o;
    cudaMalloc(&c, sizeof(float4) * 3 * 64);
    cudaMemset(c, 0, sizeof(float4) * 3 * 64);
    cudaMalloc(&o, sizeof(float) * sms * 1024);
    const double ghz = khz / 1e6;
    run<10, 0>(256, 8, c, o, sms, ghz);
    run<10, 0>(512, 8, c, o, sms, ghz);
    run<5, 0>(512, 8, c, o, sms, ghz);
    run<5, 0>(1024, 8, c, o, sms, ghz);
    run<10, 1>(256, 8, c, o, sms, ghz);
    run<10, 1>(512, 8, c, o, sms, ghz);
    printf("{\"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
