// Device helpers shared by the sm_100a stage kernels (tnrd_kernels.cu: FP32
// engine; tnrd_tc.cu: tensor-core engine).  Internal, header-only.
#pragma once

#include <cuda_runtime.h>

namespace tnrd {
namespace {

typedef unsigned long long f2;  // packed fp32x2: low word = tile A, high word = tile B

__device__ __forceinline__ f2 pk(float a, float b) {
    f2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ f2 bc(float s) { return pk(s, s); }
__device__ __forceinline__ float lo(f2 a) {
    float x, y;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a));
    return x;
}
__device__ __forceinline__ float hi(f2 a) {
    float x, y;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a));
    return y;
}
// d = a * b + c, elementwise, round-to-nearest (FFMA2)
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
    f2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
    f2 d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
    f2 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

__device__ __forceinline__ float ex2_ftz(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// Warp-wide min / max (CREDUX on sm_100a).  All 32 lanes must be converged.
__device__ __forceinline__ float warp_min(float x) {
    float r;
    asm volatile("redux.sync.min.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float warp_max(float x) {
    float r;
    asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(x));
    return r;
}

// Named CTA barriers for the producer/consumer hand-off of the w slots.
// bar.arrive does not wait; both order the participants' shared-memory accesses.
__device__ __forceinline__ void named_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Warpgroup register rebalancing (sm_90a+): the X warpgroups hand registers
// to the Y warpgroups, whose phi keeps all RUNW Horner chains in flight.
template <int N>
__device__ __forceinline__ void regs_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N)); }
template <int N>
__device__ __forceinline__ void regs_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N)); }

// Half-sample symmetric index (S l.73), single reflection, clamped for safety.
__device__ __forceinline__ int reflect(int x, int n) {
    x = x < 0 ? -1 - x : x;
    x = x >= n ? 2 * n - 1 - x : x;
    return min(max(x, 0), n - 1);
}

// Poisson proximal map, P Eq.12 with tau = 1; stable branch for ut < lambda
// (S l.215); f = 0 gives max(ut - lambda, 0) exactly.
__device__ __forceinline__ float prox_poisson(float ut, float lam, float f) {
    const float delta = ut - lam;
    const float sigma = __fsqrt_rn(fmaf(delta, delta, 4.0f * lam * f));
    if (delta >= 0.0f) return 0.5f * (delta + sigma);
    if (f == 0.0f) return 0.0f;
    return __fdiv_rn(2.0f * lam * f, sigma - delta);
}

// Reaction of the stage (tnrd_reaction), pointwise, after the diffusion
// ut = u - d: the Poisson prox of Eq.13 (P l.326-333), or P Eq.3 with
// psi = lambda (u - f) (Gaussian, l.150-158) or psi = lambda (1 - f/u) (the
// direct Poisson gradient, l.247-252; f/u taken as 0 where f = 0).
__device__ __forceinline__ float reaction_step(int kind, float u, float ut, float lam, float f) {
    if (kind == 1) return fmaf(-lam, u - f, ut);
    if (kind == 2) return fmaf(-lam, 1.0f - (f == 0.0f ? 0.0f : __fdiv_rn(f, u)), ut);
    return prox_poisson(ut, lam, f);
}



}  // namespace
}  // namespace tnrd
