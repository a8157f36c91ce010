// Tensor-core TNRD stage for sm_100a (B200): both filter banks of P Eq.13 as
// 3xTF32 tcgen05 GEMMs, phi in fp32 on the CUDA cores.
//
// One launch = one stage over a batch or a row slab, like
// the FP32 engine (tnrd_kernels.cu), with the same arithmetic except the two
// contractions:
//
//   forward bank  V[p][i] = sum_t A[p][t] k_i[t],  A[p][t] = E(u)(p - tap(t))  (P l.137)
//                 an implicit GEMM: M = 128 pixels, N = N_k, K = k*k taps (padded to 8)
//   influence     w_i(p) = phi_i(V[p][i])          (P l.145; S l.104-107)
//   adjoint bank  Z[q][t] = sum_i w_i(q) k_i[t]    GEMM M = 128, N = k*k (padded), K = N_k
//                 d(p)    = sum_t Z[p + tap(t)][t]  (col2im gather = kbar_i * w_i, P l.309-311)
//   reaction      u+ = prox(u - d)                 (P Eq.12, l.318-322)
//
// 3xTF32: every fp32 operand x is split as x = hi + lo with hi = tf32(x) (round to
// nearest) and the GEMM accumulates A_lo B_hi + A_hi B_lo + A_hi B_hi in fp32 TMEM,
// dropping only A_lo B_lo (< 2^-22 relative).  Measured on B200 (tools/tc_probe.cu):
// 3e-7 of sum |products| against 3e-4 for plain TF32, which fails the 1e-4 peak
// tolerance by 30x.
//
// Data flow per tile (output OW x OH, v region 64 x (OH + 2r), u region + 2r):
// the v region is cut into M-blocks of two 64-pixel rows.  TMEM lane m = pixel m
// of the block.  For each block: (1) every thread writes its pixel's im2col row
// (hi, lo) into TMEM with tcgen05.st (A from TMEM; for out-of-image pixels the row
// of the mirrored pixel, so w is the half-sample mirror of the in-image w, R1);
// (2) one thread issues the forward MMAs (B = taps in shared memory); (3) each
// thread reads its pixel's responses back (tcgen05.ld), evaluates phi with the
// FP32 engine's blocked-Horner units (bitwise the same phi), and writes w (hi, lo)
// over the dead im2col columns; (4) one thread issues the adjoint MMAs into Z;
// (5) Z goes to shared memory and every output pixel adds its K tap rows of this
// block to d in a fixed order (a ascending, b ascending), so d is deterministic and
// independent of tiling and batching.
#include "tnrd_internal.h"
#include "tnrd_device.cuh"

#include <climits>
#include <stdint.h>

namespace tnrd {
namespace {

constexpr int kNWG = 4;            // warpgroups per CTA; all share the 128 TMEM lanes
constexpr int kNT = 128 * kNWG;    // 512 threads
constexpr int kColStride = 128, kColV = 256, kColZ = 384, kTmemCols = 512;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// tf32 round-to-nearest of x (the high 19 bits), as fp32
__device__ __forceinline__ float tf32_rn(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

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
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                 "r"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done)
                     : "r"(smem_u32(bar)), "r"(parity)
                     : "memory");
    }
}
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

// phi_i on the pixel pair (block X, block Y) of this thread for NF consecutive
// filters, in lockstep groups of GF filters.  Per filter: the FP32 engine's
// blocked-Horner units (tnrd_internal.h) in ascending order over
// the warp-uniform range (min / max over the warp's 64 pixels); a filter whose
// range is shorter than its group's runs the extra iterations on its zero unit
// (index NB, all coefficients 0), which adds exactly 0.  Every w is therefore
// bitwise the FP32 engine's phi of the same v.  Warp-collective.
template <int NF>
__device__ __forceinline__ void phi_pairs(const float *__restrict__ s_phi, int pst, const f2 (&v)[NF],
                                          f2 (&w)[NF]) {
    constexpr int GF = (NF % 4 == 0) ? 4 : 2;
#pragma unroll
    for (int g = 0; g < NF; g += GF) {
        int u0[GF], nu[GF], zu[GF];
        float as[GF], tsg[GF], yrm[GF];
        const float *units[GF];
        int nmax = 0;
#pragma unroll
        for (int f = 0; f < GF; ++f) {
            const float *fp = s_phi + (g + f) * pst;
            const float4 fc = *reinterpret_cast<const float4 *>(fp);
            const float4 fd = *reinterpret_cast<const float4 *>(fp + 4);
            const int nb = __float2int_rn(fc.w);
            as[f] = fc.x;
            tsg[f] = fc.y;
            yrm[f] = fd.x;
            units[f] = fp + kFc;
            const float cs0 = fp[kFc];
            const float vmin = fminf(lo(v[g + f]), hi(v[g + f])), vmax = fmaxf(lo(v[g + f]), hi(v[g + f]));
            const float ylo = warp_min(fmaf(fc.x, vmin, cs0)), yhi = warp_max(fmaf(fc.x, vmax, cs0));
            u0[f] = max(0, __float2int_ru((ylo - kWindow) * fc.z));
            const int u1 = min(nb - 1, __float2int_rd((yhi + kCutT + 0.01f) * fc.z));
            nu[f] = u1 - u0[f] + 1;
            zu[f] = nb;
            nmax = max(nmax, nu[f]);
            w[g + f] = 0ull;
        }
        for (int j = 0; j < nmax; ++j) {
#pragma unroll
            for (int f = 0; f < GF; ++f) {
                const int u = j < nu[f] ? u0[f] + j : zu[f];
                const float4 *up = reinterpret_cast<const float4 *>(units[f] + u * kHornerUnit);
                const float4 q0 = up[0], q1 = up[1], q2 = up[2];
                // q0 = {ct, c0, c1, c2}, q1 = {c3, c4, c5, c6}, q2 = {c7, ...}
                const f2 t = fma2(v[g + f], bc(as[f]), bc(q0.x));
                const f2 q = fma2(t, bc(-kCutBig), bc(-kCutBig * kCutT));
                const f2 sq = fma2(t, t, pk(fmaxf(lo(q), 0.0f), fmaxf(hi(q), 0.0f)));
                const f2 G = pk(ex2_ftz(-lo(sq)), ex2_ftz(-hi(sq)));
                const f2 yr = mul2(t, bc(tsg[f]));
                const f2 Rr = pk(ex2_ftz(fminf(lo(yr), yrm[f])), ex2_ftz(fminf(hi(yr), yrm[f])));
                f2 h = fma2(Rr, bc(q2.x), bc(q1.w));
                h = fma2(h, Rr, bc(q1.z));
                h = fma2(h, Rr, bc(q1.y));
                h = fma2(h, Rr, bc(q1.x));
                h = fma2(h, Rr, bc(q0.w));
                h = fma2(h, Rr, bc(q0.z));
                h = fma2(h, Rr, bc(q0.y));
                w[g + f] = fma2(G, h, w[g + f]);
            }
        }
    }
}

template <int K, int NK>
struct TcGeo {
    static constexpr int R = K / 2, KT = K * K;
    static constexpr int KTP = tc_ktp(K), NZ = tc_nz(K);
    static constexpr int OW = kTcVW - 2 * R;   // output columns per tile
    static constexpr int UW = kTcVW + 2 * R;   // u tile columns
    static constexpr int NFW = NK / kNWG;      // filters per warpgroup in phi
    static constexpr int NCH = KTP / 8;        // 8-column chunks of an im2col row
    static_assert(NK % 8 == 0 && NK <= 64 && NFW % 2 == 0, "N_k: multiple of 8, at most 64");
    static_assert(2 * KTP <= kColStride && 2 * NK <= kColStride && NK <= 64 && NZ <= 64, "TMEM column plan");
};

__host__ __device__ constexpr int round4(int x) { return (x + 3) / 4 * 4; }

// Shared memory: operand block, u tile, Z of a super-block [KT][256], d [OH][OW],
// mbarrier + TMEM address.
template <int K, int NK>
__host__ __device__ constexpr int tc_smem_floats(int oh, int par_floats) {
    using G = TcGeo<K, NK>;
    return par_floats + round4((oh + 4 * G::R) * G::UW) + G::KT * 256 + round4(oh * G::OW) + 4;
}

// One CTA = one output tile of OW x OH.  The v region (64 x (OH + 2r)) is walked in
// super-blocks of four rows = two M-blocks, X (rows j0, j0+1) and Y (j0+2, j0+3);
// TMEM lane m is pixel (j0 + 2b + m/64, m%64) of block b.  Each thread owns lane m
// of both blocks, so phi runs on pixel pairs {X_m, Y_m} in packed fp32x2 with the
// coefficients as broadcast scalars (as in the FP32 engine).
//   TMEM columns (512):  block b: A / W at 128 b (hi, then lo at +KTP or +NK),
//                        V at 256 + 64 b, Z at 384 + 64 b.
template <int K, int NK>
__global__ void __launch_bounds__(kNT, 1) tc_stage_kernel(const __grid_constant__ StageArgs a) {
    using G = TcGeo<K, NK>;
    constexpr int R = G::R, KT = G::KT, KTP = G::KTP, NZ = G::NZ, OW = G::OW, UW = G::UW, NFW = G::NFW;
    constexpr int NCH = G::NCH;
    extern __shared__ __align__(1024) float4 smem4[];
    float *s_par = reinterpret_cast<float *>(smem4);
    const float *s_bf = s_par;                       // hi [NK x KTP], lo after it
    const float *s_ba = s_par + 2 * NK * KTP;        // hi [NZ x NK], lo after it
    const float *s_phi = s_ba + 2 * NZ * NK;         // [NK][pst]
    const int OH = a.tc_oh, VH = OH + 2 * R, UH = OH + 4 * R;
    float *s_u = s_par + a.tc_par_floats;
    float *s_z = s_u + round4(UH * UW);              // [KT][256]
    float *s_d = s_z + KT * 256;                     // [OH][OW]
    uint64_t *mbar = reinterpret_cast<uint64_t *>(s_d + round4(OH * OW));
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(mbar + 1);

    const int tid = threadIdx.x, warp = tid >> 5, wg = tid >> 7, m = tid & 127;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const int H = a.H, W = a.W;

    // ---- tile
    const int per_img = a.tiles_x * a.tiles_y;
    const int b = blockIdx.x / per_img;
    const int rem = blockIdx.x - b * per_img;
    const int ty = rem / a.tiles_x;
    const int x0 = (rem - ty * a.tiles_x) * OW;
    const int y0 = a.y_begin + ty * OH;

    // ---- stage operands -> smem, u tile (+2r, mirrored), d = 0
    {
        const float4 *src = reinterpret_cast<const float4 *>(a.params);
        for (int j = tid; j < a.tc_par_floats / 4; j += kNT) smem4[j] = __ldg(src + j);
        const float *ub = a.u_in.ptr + (long long)b * a.u_in.img_stride;
        for (int j = tid; j < UH * UW; j += kNT) {
            const int r = j / UW, c = j - r * UW;
            int gy = reflect(y0 - 2 * R + r, H);
            gy = min(max(gy, a.avail_lo), a.avail_hi - 1);
            const int gx = reflect(x0 - 2 * R + c, W);
            s_u[j] = __ldg(ub + (long long)(gy - a.u_in.row_base) * a.u_in.ld + gx);
        }
        for (int j = tid; j < OH * OW; j += kNT) s_d[j] = 0.0f;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                     "n"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // operands visible to the MMA (async proxy)
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *s_tmem;
    const uint32_t bf_hi = smem_u32(s_bf), bf_lo = bf_hi + 4 * NK * KTP;
    const uint32_t ba_hi = smem_u32(s_ba), ba_lo = ba_hi + 4 * NZ * NK;
    constexpr uint32_t SBO_F = (KTP / 4) * 128, SBO_A = (NK / 4) * 128;
    const int pst = a.pstride;
    const uint32_t tl = tmem + lane_off;  // this warp's lanes

    // MMA issue (thread 0) and completion: thread 0 waits on the mbarrier, the CTA
    // on a hardware barrier (no spinning warps).
    uint32_t phase = 0;
    const auto mma_wait_all = [&]() {
        if (tid == 0) mbar_wait(mbar, phase);
        phase ^= 1;
        __syncthreads();
        tc_fence_after();
    };

    const int nsb = (VH + 3) / 4;
    for (int sb = 0; sb < nsb; ++sb) {
        const int j0 = 4 * sb;
        // (1) im2col rows (hi, lo) of pixel m of blocks X and Y.  v-region pixel
        // (j, c) uses its mirror in the image (R1), clamped into the tile for pixels
        // no output needs.  Chunk task k = (block, 8-tap chunk) goes to warpgroup k % 4.
        {
            const float *up[2];
#pragma unroll
            for (int blk = 0; blk < 2; ++blk) {
                const int j = j0 + 2 * blk + (m >> 6), c = m & 63;
                const int gy = reflect(y0 - R + j, H), gx = reflect(x0 - R + c, W);
                const int pj = min(max(gy - y0 + R, 0), VH - 1);
                const int pc = min(max(gx - x0 + R, 0), kTcVW - 1);
                up[blk] = s_u + (pj + 2 * R) * UW + pc + 2 * R;  // tap (ta, tb) reads up[-ta*UW - tb]
            }
#pragma unroll
            for (int k = 0; k < 2 * NCH; ++k) {
                if (k % kNWG != wg) continue;
                const int blk = k / NCH, ch = k % NCH;
                uint32_t h[8], l[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const int t = ch * 8 + e;
                    float x = 0.0f;
                    if (t < KT) x = up[blk][-(t / K) * UW - (t % K)];
                    const float xh = tf32_rn(x);
                    h[e] = __float_as_uint(xh);
                    l[e] = __float_as_uint(x - xh);
                }
                tmem_st8(tl + kColStride * blk + ch * 8, h);
                tmem_st8(tl + kColStride * blk + KTP + ch * 8, l);
            }
        }
        tc_wait_st();
        tc_fence_before();
        __syncthreads();
        // (2) forward bank, both blocks: V = A_lo B_hi + A_hi B_lo + A_hi B_hi
        if (tid == 0) {
            tc_fence_after();
            constexpr uint32_t id = idesc_tf32(NK);
#pragma unroll
            for (int blk = 0; blk < 2; ++blk) {
                const uint32_t tA = tmem + kColStride * blk, tV = tmem + kColV + 64 * blk;
#pragma unroll
                for (int s = 0; s < KTP / 8; ++s) {
                    mma_tf32(tV, tA + KTP + 8 * s, umma_desc(bf_hi + 256 * s, SBO_F), id, s > 0);
                    mma_tf32(tV, tA + 8 * s, umma_desc(bf_lo + 256 * s, SBO_F), id, 1);
                    mma_tf32(tV, tA + 8 * s, umma_desc(bf_hi + 256 * s, SBO_F), id, 1);
                }
            }
            mma_commit(mbar);
        }
        mma_wait_all();
        // (3) phi of this warpgroup's filters on the pixel pairs; w (hi, lo) of each
        // block over its dead im2col columns
        {
            uint32_t vx[NFW], vy[NFW];
            tmem_ld_nowait<NFW>(tl + kColV + wg * NFW, vx);
            tmem_ld_nowait<NFW>(tl + kColV + 64 + wg * NFW, vy);
            tmem_wait_ld(vx);
            tmem_wait_ld(vy);
            f2 v[NFW], w[NFW];
#pragma unroll
            for (int e = 0; e < NFW; ++e) v[e] = pk(__uint_as_float(vx[e]), __uint_as_float(vy[e]));
#ifdef TNRD_EXP_NOPHI
#pragma unroll
            for (int e = 0; e < NFW; ++e) w[e] = v[e];
#else
            phi_pairs<NFW>(s_phi + wg * NFW * pst, pst, v, w);
#endif
#pragma unroll
            for (int blk = 0; blk < 2; ++blk) {
                uint32_t wh[NFW], wl[NFW];
#pragma unroll
                for (int e = 0; e < NFW; ++e) {
                    const float x = blk ? hi(w[e]) : lo(w[e]);
                    const float xh = tf32_rn(x);
                    wh[e] = __float_as_uint(xh);
                    wl[e] = __float_as_uint(x - xh);
                }
                tmem_st<NFW>(tl + kColStride * blk + wg * NFW, wh);
                tmem_st<NFW>(tl + kColStride * blk + NK + wg * NFW, wl);
            }
        }
        tc_wait_st();
        tc_fence_before();
        __syncthreads();
        // (4) adjoint bank, both blocks: Z = W_lo B_hi + W_hi B_lo + W_hi B_hi
        if (tid == 0) {
            tc_fence_after();
            constexpr uint32_t id = idesc_tf32(NZ);
#pragma unroll
            for (int blk = 0; blk < 2; ++blk) {
                const uint32_t tW = tmem + kColStride * blk, tZ = tmem + kColZ + 64 * blk;
#pragma unroll
                for (int s = 0; s < NK / 8; ++s) {
                    mma_tf32(tZ, tW + NK + 8 * s, umma_desc(ba_hi + 256 * s, SBO_A), id, s > 0);
                    mma_tf32(tZ, tW + 8 * s, umma_desc(ba_lo + 256 * s, SBO_A), id, 1);
                    mma_tf32(tZ, tW + 8 * s, umma_desc(ba_hi + 256 * s, SBO_A), id, 1);
                }
            }
            mma_commit(mbar);
        }
        mma_wait_all();
        // (5) Z -> smem [tap][pixel of the super-block], then for every output pixel
        // d(y, x) += sum_b Z[(y + a, x + b)][a K + b] for the super-block's rows, a
        // ascending (rows in order), b ascending
#pragma unroll
        for (int k = 0; k < 2 * (NZ / 8); ++k) {
            if (k % kNWG != wg) continue;
            const int blk = k / (NZ / 8), ch = k % (NZ / 8);
            if (ch * 8 >= KT) continue;
            uint32_t z[8];
            tmem_ld_nowait<8>(tl + kColZ + 64 * blk + ch * 8, z);
            tmem_wait_ld(z);
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (ch * 8 + e < KT) s_z[(ch * 8 + e) * 256 + 128 * blk + m] = __uint_as_float(z[e]);
        }
        __syncthreads();
        for (int it = tid; it < (K + 3) * OW; it += kNT) {
            const int y = j0 - (K - 1) + it / OW, x = it % OW;
            if (y < 0 || y >= OH) continue;
            float d = s_d[y * OW + x];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                const int ta = j0 + jj - y;
                if (ta < 0 || ta >= K) continue;
                const float *zp = s_z + (ta * K) * 256 + jj * 64 + x;
                float S = 0.0f;
#pragma unroll
                for (int tb = 0; tb < K; ++tb) S += zp[tb * 256 + tb];
                d += S;
            }
            s_d[y * OW + x] = d;
        }
        // the next super-block writes s_z / s_d only after two more CTA barriers
    }
    __syncthreads();

    // ---- epilogue: ut = u - d, u+ = reaction(ut)
    {
        const float *fb = a.f.ptr + (long long)b * a.f.img_stride;
        float *ob = a.u_out + (long long)b * a.out_img_stride;
        for (int it = tid; it < OH * OW; it += kNT) {
            const int y = it / OW, x = it - y * OW;
            const int oy = y0 + y, ox = x0 + x;
            if (oy >= a.y_end || ox >= W) continue;
            const float u = s_u[(y + 2 * R) * UW + x + 2 * R];
            const float ut = u - s_d[it];
            const float fv = __ldg(fb + (long long)(oy - a.f.row_base) * a.f.ld + ox);
            const long long oi = (long long)(oy - a.out_row_base) * a.out_ld + ox;
            ob[oi] = reaction_step(a.reaction, u, ut, a.lambda, fv);
            if (a.ut_out) a.ut_out[(long long)b * a.out_img_stride + oi] = ut;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols));
}

template <int K, int NK>
cudaError_t launch_tc(StageArgs &a, int B, cudaStream_t s) {
    using G = TcGeo<K, NK>;
    auto kern = tc_stage_kernel<K, NK>;
    if (a.tc_oh <= 0 || a.tc_oh % 2 != 0) return cudaErrorInvalidValue;
    const size_t smem = sizeof(float) * (size_t)tc_smem_floats<K, NK>(a.tc_oh, a.tc_par_floats);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    a.tiles_x = (a.W + G::OW - 1) / G::OW;
    a.tiles_y = (a.y_end - a.y_begin + a.tc_oh - 1) / a.tc_oh;
    const long long n = (long long)B * a.tiles_x * a.tiles_y;
    if (n > INT_MAX) return cudaErrorInvalidValue;
    a.n_tiles = (int)n;
    if (n > 0) kern<<<(unsigned)n, kNT, smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace

bool tc_supported(int ksize, int Nk) {
    return (ksize == 3 && Nk == 8) || (ksize == 5 && Nk == 24) || (ksize == 7 && Nk == 48);
}

// Output rows per tile: 128 (v region 64 x 134 at k = 7: 1.155 pixel-stages of
// work per output pixel) when the launch has at least one tile per SM, else halved
// until it has (or 16 rows).
int tc_choose_rows(int ksize, int B, int H, int W, int num_sms) {
    const int ow = kTcVW - 2 * (ksize / 2);
    int oh = 128;
    while (oh > 16 && (long long)B * ((W + ow - 1) / ow) * ((H + oh - 1) / oh) < num_sms) oh /= 2;
    return oh;
}

cudaError_t launch_stage_tc(int ksize, StageArgs &a, int B, cudaStream_t s) {
    if (ksize == 3 && a.Nk == 8) return launch_tc<3, 8>(a, B, s);
    if (ksize == 5 && a.Nk == 24) return launch_tc<5, 24>(a, B, s);
    if (ksize == 7 && a.Nk == 48) return launch_tc<7, 48>(a, B, s);
    return cudaErrorInvalidValue;
}

}  // namespace tnrd
