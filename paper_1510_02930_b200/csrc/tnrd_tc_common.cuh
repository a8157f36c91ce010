// tcgen05 / TMEM / mbarrier / TMA helpers and the packed-pair phi shared by the
// tensor-core kernels (tnrd_tc.cu: the persistent stage kernel and the gradient's
// banks).  Internal, header-only.
#pragma once

#include "tnrd_internal.h"
#include "tnrd_device.cuh"

#include <cuda.h>

#include <climits>
#include <stdint.h>

namespace tnrd {
namespace {
#ifndef TNRD_TC_PG
#define TNRD_TC_PG 4
#endif
constexpr int kPG = TNRD_TC_PG;    // phi warp groups (4 warps each, one per TMEM lane quarter)
constexpr int kNT = (4 * kPG + 5) * 32;  // phi warps, 4 build / gather warps, 1 MMA warp
constexpr int kSlots = 3;          // M-blocks in flight (TMEM slots)
constexpr int kZP = 132;           // Z row pitch in smem: a warp spanning two gather rows stays conflict-free
constexpr int kTmemCols = 512;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// high part of the 3xTF32 split of a data operand: x truncated to its high 19 bits
// (TF32); x - hi is exact in fp32 and |x - hi| < 2^-10 |x|
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }
// the same split with the high part rounded to nearest (ties away): |x - hi| <= 2^-11 |x|
// and the rounding errors are unbiased — the training gradient's operands (its tape and
// banks), whose sums over whole images would accumulate truncation's one-sided bias
// (DESIGN.md §5.9); one more integer add than truncation
__device__ __forceinline__ float tf32_hi_rn(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
template <bool RN>
__device__ __forceinline__ float tf32_hi_t(float x) { return RN ? tf32_hi_rn(x) : tf32_hi(x); }

// UMMA shared-memory descriptor, K-major, no swizzle (sm_100 version 1): 8-row x
// 16-byte core matrices, K-adjacent core matrices 128 B apart (LBO), 8-row groups
// `sbo` bytes apart.
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
           (1ull << 46);
}
// instruction descriptor: kind::tf32, fp32 accumulate, A and B K-major, M = 128
__host__ __device__ constexpr uint32_t idesc_tf32(int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
#ifdef TNRD_EXP_NOMMA
    return;
#endif
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                 "r"(a), "l"(b), "r"(idesc), "r"(acc));
}
// Warp-collective forms: the whole (converged) warp runs the issue code, so the
// operands stay in uniform registers, and one elected lane issues: the tensor pipe
// then runs at its rate (24 cycles per N = 48 MMA against ~55 for a lone thread,
// tools/tc_rate.cu, profiles/r01_tc_rate.json).
__device__ __forceinline__ void mma_tf32_warp(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                 "r"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit_warp(uint64_t *bar) {
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    // try_wait with a suspend-time hint: the thread sleeps until the phase completes
    // (or the hint expires) instead of spinning on issue slots
    uint32_t done = 0;
    while (!done) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done)
                     : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
                     : "memory");
    }
}
// non-blocking test of an mbarrier phase; warp-uniform (lane 0's result) when `warp`
__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t parity, bool warp) {
    uint32_t done;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done)
                 : "r"(smem_u32(bar)), "r"(parity)
                 : "memory");
    if (warp) done = __shfl_sync(0xffffffffu, done, 0);
    return done != 0;
}
// floor / ceil of |x| < 2^22 as an int without the XU pipe (F2I): a directed-
// rounding add of 1.5 * 2^23 leaves the integer in the low mantissa bits
__device__ __forceinline__ int floor_i(float x) { return __float_as_int(__fadd_rd(x, 12582912.0f)) - 0x4B400000; }
__device__ __forceinline__ int ceil_i(float x) { return __float_as_int(__fadd_ru(x, 12582912.0f)) - 0x4B400000; }

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// TMEM <-> registers, 32 lanes x N consecutive 32-bit columns (this warp's lanes);
// the load waits for completion inside the same asm statement.
__device__ __forceinline__ void tmem_st8(uint32_t addr, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(addr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
__device__ __forceinline__ void tmem_st4(uint32_t addr, const uint32_t *r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(r[0]), "r"(r[1]),
                 "r"(r[2]), "r"(r[3])
                 : "memory");
}
__device__ __forceinline__ void tmem_st2(uint32_t addr, const uint32_t *r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(addr), "r"(r[0]), "r"(r[1])
                 : "memory");
}
// N columns (N even) as chunks of 8 / 4 / 2, without waiting; tmem_wait_ld(r)
// waits for all outstanding loads and orders every later use of r after it.
template <int N>
__device__ __forceinline__ void tmem_ld_nowait(uint32_t addr, uint32_t (&r)[N]) {
    static_assert(N % 2 == 0, "even column count");
    int c = 0;
#pragma unroll
    for (; c + 8 <= N; c += 8)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[c]), "=r"(r[c + 1]), "=r"(r[c + 2]), "=r"(r[c + 3]), "=r"(r[c + 4]), "=r"(r[c + 5]),
                       "=r"(r[c + 6]), "=r"(r[c + 7])
                     : "r"(addr + c));
    if constexpr (N % 8 >= 4) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r[c]), "=r"(r[c + 1]), "=r"(r[c + 2]), "=r"(r[c + 3])
                     : "r"(addr + c));
        c += 4;
    }
    if constexpr (N % 4 >= 2)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(r[c]), "=r"(r[c + 1]) : "r"(addr + c));
}
template <int N>
__device__ __forceinline__ void tmem_wait_ld(uint32_t (&r)[N]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < N; ++i) asm volatile("" : "+r"(r[i]));
}
template <int N>
__device__ __forceinline__ void tmem_st(uint32_t addr, const uint32_t (&r)[N]) {
    static_assert(N % 2 == 0, "even column count");
    int c = 0;
#pragma unroll
    for (; c + 8 <= N; c += 8) {
        const uint32_t q[8] = {r[c], r[c + 1], r[c + 2], r[c + 3], r[c + 4], r[c + 5], r[c + 6], r[c + 7]};
        tmem_st8(addr + c, q);
    }
    if constexpr (N % 8 >= 4) { tmem_st4(addr + c, r + c); c += 4; }
    if constexpr (N % 4 >= 2) tmem_st2(addr + c, r + c);
}

// phi of NP filter pairs (2p, 2p+1) on this thread's pixel: v[2p], v[2p+1] are
// the two responses, evaluated together in packed fp32x2 with the interleaved pair
// constants (tnrd_internal.h), so every constant is an aligned 64-bit operand.  Per
// filter: the FP32 engine's blocked-Horner units in ascending
// order.  A pair runs the union of its two filters' warp-uniform unit ranges (min /
// max over the warp's 32 pixels) and pairs run in lockstep groups of GP: a pair
// runs units u0 + j for j < nmax, past its own range into real units outside it or
// into the zero units NB..2NB-1.  A unit outside a filter's own range is exactly 0
// for every lane (the FP32 engine skips it for that reason), so each w is bitwise
// the FP32 engine's phi of the same v.  Warp-collective.
template <int NP>
__device__ __forceinline__ void phi_fpairs(const float *__restrict__ s_pp, int pps, const uint32_t (&vr)[2 * NP],
                                           f2 (&w)[NP]) {
#ifndef TNRD_TC_GP
#define TNRD_TC_GP 2
#endif
    constexpr int GP = NP % TNRD_TC_GP == 0 ? TNRD_TC_GP : (NP % 2 == 0 ? 2 : 1);
#pragma unroll
    for (int g = 0; g < NP; g += GP) {
        f2 vv[GP], as2[GP], tsg2[GP];
        float yra[GP], yrb[GP];
        const char *up[GP];
        int nmax = 0;
#pragma unroll
        for (int p = 0; p < GP; ++p) {
            const float *hp = s_pp + (g + p) * pps;
            const float4 h0 = *reinterpret_cast<const float4 *>(hp);       // a_s, two_sg
            const ulonglong2 h1 = *reinterpret_cast<const ulonglong2 *>(hp + 4);  // {A}, {B0}
            const float4 h2 = *reinterpret_cast<const float4 *>(hp + 8);   // B1, yrmax
            const int nb = __float_as_int(hp[12]);
            const float va = __uint_as_float(vr[2 * (g + p)]), vb = __uint_as_float(vr[2 * (g + p) + 1]);
            vv[p] = pk(va, vb);
            as2[p] = pk(h0.x, h0.y);
            tsg2[p] = pk(h0.z, h0.w);
            yra[p] = h2.z;
            yrb[p] = h2.w;
#ifdef TNRD_TC_OLDRANGE
            const f2 lo2 = fma2(pk(warp_min(va), warp_min(vb)), h1.x, h1.y);
            const f2 hi2 = fma2(pk(warp_max(va), warp_max(vb)), h1.x, pk(h2.x, h2.y));
            // ceil / floor are monotone: min / max first, one conversion each
            const int u0 = max(0, ceil_i(fminf(lo(lo2), hi(lo2))));
            const int u1 = min(nb - 1, floor_i(fmaxf(lo(hi2), hi(hi2))));
#else
            // A > 0 and fma rounding is monotone, so min_lanes fma(v, A, B0) ==
            // fma(min_lanes v, A, B0) bit for bit: combine the pair per lane first and
            // reduce once per bound (2 warp reductions per pair instead of 4)
            const f2 lo2 = fma2(vv[p], h1.x, h1.y);
            const f2 hi2 = fma2(vv[p], h1.x, pk(h2.x, h2.y));
            const int u0 = max(0, ceil_i(warp_min(fminf(lo(lo2), hi(lo2)))));
            const int u1 = min(nb - 1, floor_i(warp_max(fmaxf(lo(hi2), hi(hi2)))));
#endif
            up[p] = reinterpret_cast<const char *>(hp + kTcPairHdr) + u0 * (4 * kTcPairUnit);
            nmax = max(nmax, u1 - u0 + 1);
            w[g + p] = 0ull;
        }
        // one unit of pair p: t, the cut, G and R (two ex2 each), the degree-7 Horner sum
        const auto unit = [&](int p) {
            const ulonglong2 *qp = reinterpret_cast<const ulonglong2 *>(up[p]);
            up[p] += 4 * kTcPairUnit;
            const ulonglong2 q0 = qp[0], q1 = qp[1], q2 = qp[2], q3 = qp[3];
            const unsigned long long c7 = reinterpret_cast<const unsigned long long *>(qp + 4)[0];
            // q0 = {ct, c0}, q1 = {c1, c2}, q2 = {c3, c4}, q3 = {c5, c6}  (pairs)
            const f2 t = fma2(vv[p], as2[p], q0.x);
            const f2 q = fma2(t, bc(-kCutBig), bc(-kCutBig * kCutT));
            const f2 sq = fma2(t, t, pk(fmaxf(lo(q), 0.0f), fmaxf(hi(q), 0.0f)));
            const f2 G = pk(ex2_ftz(-lo(sq)), ex2_ftz(-hi(sq)));
            const f2 yr = mul2(t, tsg2[p]);
            const f2 Rr = pk(ex2_ftz(fminf(lo(yr), yra[p])), ex2_ftz(fminf(hi(yr), yrb[p])));
            f2 h = fma2(Rr, c7, q3.y);
            h = fma2(h, Rr, q3.x);
            h = fma2(h, Rr, q2.y);
            h = fma2(h, Rr, q2.x);
            h = fma2(h, Rr, q1.y);
            h = fma2(h, Rr, q1.x);
            h = fma2(h, Rr, q0.y);
            w[g + p] = fma2(G, h, w[g + p]);
        };
        for (int j = 0; j < nmax; ++j) {
#pragma unroll
            for (int p = 0; p < GP; ++p) unit(p);
        }
    }
}

// The same phi with the warp's filters split between its half-warps: lanes L and
// L + 16 (two pixels 16 columns apart in one row) swap half of their responses, so
// lane L < 16 holds filters [0, NF/2) and lane L + 16 filters [NF/2, NF) of BOTH
// pixels.  A thread then runs each of its NF/4 filter pairs on two pixels with one
// set of constants: half the broadcast constant loads (a 128-bit shared-memory load
// costs two wavefronts whether its lanes read one address or one per half-warp) and
// half the range set-ups per warp; the influences of the partner's pixel go back by
// a second swap.  Per value the arithmetic is phi_fpairs': the same units in the
// same order; a half-warp's unit range is the union over its 32 values' pixels (the
// same 32 pixels as before), and units outside a value's own range are exactly 0, so
// w is bitwise unchanged.  Warp-collective (shuffles, warp reductions, votes).
template <int NF>
__device__ __forceinline__ void phi_halfwarp(const float *__restrict__ s_pp, int pps, const uint32_t (&vr)[NF],
                                             f2 (&w)[NF / 2], int lane) {
    static_assert(NF % 4 == 0, "two filter pairs per half-warp at least");
    constexpr int HF = NF / 2, NP = NF / 4;   // filters, filter pairs per half-warp
    const bool upper = lane >= 16;
    uint32_t mine[HF], oth[HF];
#pragma unroll
    for (int k = 0; k < HF; ++k) {
        mine[k] = upper ? vr[HF + k] : vr[k];
        oth[k] = __shfl_xor_sync(0xffffffffu, upper ? vr[k] : vr[HF + k], 16);
    }
    const float *hp0 = s_pp + (upper ? NP * pps : 0);
    const float inf = __int_as_float(0x7f800000);
    f2 wm[NP], wo[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const float *hp = hp0 + p * pps;
        const float4 h0 = *reinterpret_cast<const float4 *>(hp);       // a_s, two_sg
        const ulonglong2 h1 = *reinterpret_cast<const ulonglong2 *>(hp + 4);  // {A}, {B0}
        const float4 h2 = *reinterpret_cast<const float4 *>(hp + 8);   // B1, yrmax
        const int nb = __float_as_int(hp[12]);
        const f2 va = pk(__uint_as_float(mine[2 * p]), __uint_as_float(mine[2 * p + 1]));
        const f2 vb = pk(__uint_as_float(oth[2 * p]), __uint_as_float(oth[2 * p + 1]));
        const f2 as2 = pk(h0.x, h0.y), tsg2 = pk(h0.z, h0.w);
        const float yra = h2.z, yrb = h2.w;
        // unit range of this half-warp's 32 values per filter: A > 0 and fma rounding
        // is monotone, so the min / max commute with the fma (phi_fpairs)
        const f2 la = fma2(va, h1.x, h1.y), lb = fma2(vb, h1.x, h1.y);
        const f2 ha = fma2(va, h1.x, pk(h2.x, h2.y)), hb = fma2(vb, h1.x, pk(h2.x, h2.y));
        const float l = fminf(fminf(lo(la), hi(la)), fminf(lo(lb), hi(lb)));
        const float g = fmaxf(fmaxf(lo(ha), hi(ha)), fmaxf(lo(hb), hi(hb)));
        const float lL = warp_min(upper ? inf : l), lU = warp_min(upper ? l : inf);
        const float gL = warp_max(upper ? -inf : g), gU = warp_max(upper ? g : -inf);
        const int u0r = max(0, ceil_i(upper ? lU : lL));
        const int u1 = min(nb - 1, floor_i(upper ? gU : gL));
        const int u0 = min(u0r, max(2 * nb - 2, 0));   // two units from u0 stay inside the 2 NB stored
        const int n = u1 - u0r + 1;                    // own units; <= 0: none (u0 = u0r whenever n > 0)
        const char *up = reinterpret_cast<const char *>(hp + kTcPairHdr) + u0 * (4 * kTcPairUnit);
        f2 acca = 0ull, accb = 0ull;
        const auto unit = [&]() {
            const ulonglong2 *qp = reinterpret_cast<const ulonglong2 *>(up);
            up += 4 * kTcPairUnit;
            const ulonglong2 q0 = qp[0], q1 = qp[1], q2 = qp[2], q3 = qp[3];
            const unsigned long long c7 = reinterpret_cast<const unsigned long long *>(qp + 4)[0];
            const f2 ta = fma2(va, as2, q0.x), tb = fma2(vb, as2, q0.x);
            const f2 qa = fma2(ta, bc(-kCutBig), bc(-kCutBig * kCutT)), qb = fma2(tb, bc(-kCutBig), bc(-kCutBig * kCutT));
            const f2 sa = fma2(ta, ta, pk(fmaxf(lo(qa), 0.0f), fmaxf(hi(qa), 0.0f)));
            const f2 sb = fma2(tb, tb, pk(fmaxf(lo(qb), 0.0f), fmaxf(hi(qb), 0.0f)));
            const f2 Ga = pk(ex2_ftz(-lo(sa)), ex2_ftz(-hi(sa))), Gb = pk(ex2_ftz(-lo(sb)), ex2_ftz(-hi(sb)));
            const f2 ya = mul2(ta, tsg2), yb = mul2(tb, tsg2);
            const f2 Ra = pk(ex2_ftz(fminf(lo(ya), yra)), ex2_ftz(fminf(hi(ya), yrb)));
            const f2 Rb = pk(ex2_ftz(fminf(lo(yb), yra)), ex2_ftz(fminf(hi(yb), yrb)));
            f2 xa = fma2(Ra, c7, q3.y), xb = fma2(Rb, c7, q3.y);
            xa = fma2(xa, Ra, q3.x); xb = fma2(xb, Rb, q3.x);
            xa = fma2(xa, Ra, q2.y); xb = fma2(xb, Rb, q2.y);
            xa = fma2(xa, Ra, q2.x); xb = fma2(xb, Rb, q2.x);
            xa = fma2(xa, Ra, q1.y); xb = fma2(xb, Rb, q1.y);
            xa = fma2(xa, Ra, q1.x); xb = fma2(xb, Rb, q1.x);
            xa = fma2(xa, Ra, q0.y); xb = fma2(xb, Rb, q0.y);
            acca = fma2(Ga, xa, acca);
            accb = fma2(Gb, xb, accb);
        };
        unit();
        unit();
        // further units (the evaluation window of 32 adjacent pixels rarely spans
        // more than two): only the lanes that own them, the others' pointers stay put
#pragma unroll 1
        for (int j = 2; __any_sync(0xffffffffu, j < n); ++j)
            if (j < n) unit();
        wm[p] = acca;
        wo[p] = accb;
    }
    // the partner's influences go back; own pixel: filters [0, HF) from the lower
    // lane of the pair, [HF, NF) from the upper one
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const f2 r = __shfl_xor_sync(0xffffffffu, wo[p], 16);
        w[p] = upper ? r : wm[p];
        w[NP + p] = upper ? wm[p] : r;
    }
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// ---- TMA (cp.async.bulk.tensor): tensor maps are encoded on the host through the
// driver entry point (no -lcuda link), passed as __grid_constant__ kernel parameters.
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// box at (x, y, z) of a 3-D tensor map -> shared memory, completion on `bar`;
// out-of-range elements are zero filled (they still count toward the bytes)
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *tm, int x, int y, int z, uint64_t *bar) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
                 "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
                 "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
                 : "memory");
}

typedef CUresult (*EncodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiled encoder() {
    static EncodeTiled fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiled>(f);
        cudaGetLastError();
    }
    return fn;
}

inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace
}  // namespace tnrd
