// Persistent streaming tensor-core stage kernel for sm_100a (B200): one launch = one
// stage of P Eq.13 (l.326-333) over a batch or a row slab, with the arithmetic of the
// per-tile tensor engine (tnrd_tc.cu: 3xTF32 tcgen05 filter banks, the FP32 engine's
// blocked-Horner phi, fixed-order col2im gather, fused reaction) organised for the
// machine instead of per tile:
//
//  * persistent: one CTA per SM; the stage operands (taps, phi constants) are loaded
//    into shared memory once per CTA, TMEM is allocated once, and the CTA streams
//    through a contiguous range of work units (image, 58-column strip, output row
//    pair) -- every CTA gets the same number of row pairs, so there is no tail wave;
//  * a unit range is cut into segments (one strip each); a segment's v rows (the
//    output rows +- r) are processed in M-blocks of two 64-pixel rows, so the y halo
//    is paid once per segment instead of once per 128-row tile;
//  * u and f rows arrive by TMA (cp.async.bulk.tensor, one row box per row) into
//    shared-memory rings, several blocks ahead of use, tracked by mbarriers;
//  * im2col without per-tap thread work: each new u row is expanded once into an
//    "E row" (per pixel the 8 u values of one tap row, split hi / lo, in the UMMA
//    K-major core-matrix layout), and the MMA thread copies each tap row's 128 x 8
//    block from two adjacent E rows into TMEM with tcgen05.cp (tensor-pipe order:
//    the MMAs that follow see the copy);
//  * R1 mirrored rows are not computed: the gather adds each in-image Z row also at
//    its mirror position (the half-sample extension of w, P l.302-311); mirrored
//    columns take the im2col row of their mirror pixel (R1) as before;
//  * the epilogue (u - d, reaction, store) streams behind the gather: after each
//    block the output rows whose taps are complete are written, so it overlaps the
//    rest of the pipeline.
//
// Per output pixel the operations are the same sequence wherever the pixel lies in
// a segment, so results do not depend on the unit split (batch / slab / CTA count).
#include "tnrd_tc_common.cuh"

#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

namespace tnrd {

struct alignas(64) StreamArgs {
    CUtensorMap tm_u;      // u_in rows [avail_lo, avail_hi): dims (W, rows, B), box (kUBW, 1, 1)
    CUtensorMap tm_f;      // f rows [y_begin, y_end): dims (W, rows, B), box (kFBW, 1, 1)
    StageArgs a;
    long long units;       // B * nstrips * nrp
    int nstrips, nrp;      // strips per image, output row pairs per strip
    unsigned long long *prof;   // TNRD_SX_PROF builds: per-CTA role timers [grid][16], else null
};

namespace {

constexpr int kNUR = 64;    // raw u / f ring rows
constexpr int kUBW = 80;    // u row box: columns [xr, xr + 80), xr = floor4(x0 - 8)
constexpr int kUP = 96;     // u ring pitch (floats): 384 B, 128-byte aligned rows
constexpr int kFBW = 64;    // f row box: columns [xf, xf + 64), xf = floor4(x0)
constexpr int kSD = 32;     // d ring rows (rows of the gather window and of the lagging epilogue)
constexpr int kNTB = 8;     // TMA group barriers: a group's barrier is re-armed well after its last wait
constexpr int kTmaAhead = 2;
#ifndef TNRD_SX_PG
#define TNRD_SX_PG 4
#endif
#ifndef TNRD_SX_BG
#define TNRD_SX_BG 4
#endif
constexpr int kSPG = TNRD_SX_PG;                  // phi warp groups (4 warps each, one per lane quarter)
constexpr int kSBG = TNRD_SX_BG;                  // BG warps (4 or 8: one or two per lane quarter)
constexpr int kSNT = (4 * kSPG + kSBG + 1) * 32;  // + the MMA warp
constexpr int kNBG = 32 * kSBG;                   // BG threads
constexpr int kNEF = 4;     // E_full barriers (E rows of block g, built by the BG warps)
constexpr int kNG = 8;      // G_done / epi_done barriers (gather -> epilogue -> d-ring reuse)

__device__ __forceinline__ int floor4(int x) { return x >= 0 ? (x & ~3) : -((-x + 3) & ~3); }
__device__ __forceinline__ int clampi(int x, int lo, int hi) { return min(max(x, lo), hi); }

template <int K, int NK>
struct SGeo {
    static constexpr int R = K / 2, KT = K * K;
    static constexpr int OW = kTcVW - 2 * R;     // output columns per strip
    static constexpr int KTS = 8 * K;            // forward GEMM K: one 8-column chunk per tap row
    static constexpr int NZ = tc_nz(K);
    static constexpr int SLOT = 2 * (KTS > NK ? KTS : NK);
    static constexpr int VZW = NK > NZ ? NK : NZ;
    static constexpr int PG = (NK % (2 * kSPG) == 0) ? kSPG : 2;
    static constexpr int NFW = NK / PG;
    static constexpr int NZC = NZ / 8;
    static constexpr int NR = 2 * (2 * R + 2);   // E ring rows (two blocks' tap rows) + 1 shadow row
    static constexpr int EROW = 512;             // floats of an E row (64 pixels x 8)
    static_assert(NK % 8 == 0 && NK <= 64 && NFW % 2 == 0, "N_k: multiple of 8, at most 64");
    static_assert(kSlots * (SLOT + VZW) <= kTmemCols, "TMEM column plan");
    static_assert(K <= 7 && 4 * (2 * R + 2) <= kSD, "tap rows fit one 8-column chunk; d ring");
    static_assert(OW + 2 <= kFBW, "f box covers the strip for even x0");
};

template <int K, int NK>
__host__ __device__ constexpr int stream_smem_floats(int par_floats) {
    using G = SGeo<K, NK>;
    return par_floats + 2 * (G::NR + 1) * G::EROW + kNUR * kUP + kNUR * kFBW + G::KT * kZP + kSD * 64 +
           2 * (3 * kSlots + kSlots + kNEF + kNTB + 2 * kNG) + 4;
}

// The CTA's work as a sequence of M-blocks.  Units are (image, strip, output row
// pair) in that order; CTA c owns units [U c / G, U (c+1) / G).  A segment is the
// run of the CTA's units inside one strip; its v rows [vr0, vr1) are cut into
// blocks of two rows (the second row of the last block may be past vr1: a dummy).
// E / raw-row counters: the segment's rows u = vr0 - R ... get consecutive counter
// values from `eb`; block j's tap rows are counters [eb + 2j, eb + 2j + 2R + 2).
template <int K>
struct BlockIter {
    static constexpr int R = K / 2, OW = kTcVW - 2 * R;
    long long u, uend;
    int b, x0, oy0, oy1, vr0, vr1, nb, eb, j, g;
    __device__ __forceinline__ void load(const StreamArgs &p) {
        const long long si = u / p.nrp;
        const int rp0 = (int)(u - si * p.nrp);
        const int rp1 = (int)min((long long)p.nrp, (long long)rp0 + (uend - u));
        u += rp1 - rp0;
        b = (int)(si / p.nstrips);
        x0 = (int)(si - (long long)b * p.nstrips) * OW;
        oy0 = p.a.y_begin + 2 * rp0;
        oy1 = min(p.a.y_begin + 2 * rp1, p.a.y_end);
        vr0 = max(oy0 - R, 0);
        vr1 = min(oy1 + R, p.a.H);
        nb = (vr1 - vr0 + 1) / 2;
        j = 0;
    }
    __device__ __forceinline__ void init(const StreamArgs &p) {
        const long long G = gridDim.x;
        u = p.units * (long long)blockIdx.x / G;
        uend = p.units * ((long long)blockIdx.x + 1) / G;
        g = 0;
        eb = 0;
        nb = 0;
        j = 0;
        if (u < uend) load(p);
    }
    __device__ __forceinline__ bool valid() const { return j < nb; }
    __device__ __forceinline__ void next(const StreamArgs &p) {
        ++g;
        if (++j == nb) {
            eb += 2 * nb + 2 * R;
            nb = 0;
            j = 0;
            if (u < uend) load(p);
        }
    }
    __device__ __forceinline__ int m0() const { return vr0 + 2 * j; }
    __device__ __forceinline__ int e0() const { return eb + 2 * j; }
    // counters of the rows this block adds: all 2R + 2 for the first block, else 2
    __device__ __forceinline__ int new_lo() const { return j == 0 ? eb : eb + 2 * j + 2 * R; }
    __device__ __forceinline__ int new_hi() const { return eb + 2 * j + 2 * R + 2; }
    __device__ __forceinline__ int urow(int c) const { return vr0 - R + (c - eb); }   // u row of counter c
};

// mbarrier wait with a deadline: a lost hand-off (a bug) ends the kernel with a trap
// after ~10 s instead of hanging the GPU
__device__ __forceinline__ void mbar_wait_dl(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    uint64_t t0 = 0;
    for (int it = 0; !done; ++it) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done)
                     : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
                     : "memory");
        if (!done && (it & 255) == 255) {
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t0 == 0) t0 = t;
            else if (t - t0 > 10000000000ull) __trap();
        }
    }
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_row(void *dst, const CUtensorMap *tm, int x, int y, int z, uint64_t *bar) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
                 "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
                 "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
                 : "memory");
}
// 128 x 8-word block of a K-major no-swizzle smem operand -> TMEM (lanes 0..127)
__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t desc) {
    asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(desc));
}
__device__ __forceinline__ void tmem_cp_128x256b_warp(uint32_t taddr, uint64_t desc) {
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.cp.cta_group::1.128x256b [%0], %1;\n\t}" ::"r"(taddr), "l"(desc));
}

// Warp roles (672 threads, one CTA per SM; no CTA-wide barrier in the main loop):
//   warps 0..15   phi: as in tc_stage_kernel (warp w: lane quarter w % 4, NFW filters)
//   warps 16..19  BG (build / gather, lane quarter w % 4): TMA issue (one thread),
//                 E rows, Z -> smem, gather, streaming epilogue
//   warp 20       MMA: tcgen05.cp of the A blocks + the forward and adjoint GEMMs
// Hand-offs per block g (slot s = g % 3): E_full (BG -> MMA), V_full (MMA -> phi),
// W_full (phi -> MMA), Z_full (MMA -> BG), Z_free (BG -> MMA: Z read, slot reusable);
// TMA groups (TMA -> BG) per block g % kNTB.
#ifdef TNRD_SX_PROF
#define SXP_T0(v) const long long v = clock64()
#define SXP_ADD(k, v) sxp[k] += clock64() - v
#define SXP_DECL() unsigned long long sxp[16] = {0}; const long long sxp_start = clock64()
#define SXP_OUT(pred) if ((pred) && p.prof) { sxp[15] = clock64() - sxp_start; \
        for (int k_ = 0; k_ < 16; ++k_) if (sxp[k_]) p.prof[blockIdx.x * 16 + k_] = sxp[k_]; }
#else
#define SXP_T0(v)
#define SXP_ADD(k, v)
#define SXP_DECL()
#define SXP_OUT(pred)
#endif

template <int K, int NK, bool TABLE, bool R2, bool RN>
__global__ void __launch_bounds__(kSNT, 1) tc_stream_kernel(const __grid_constant__ StreamArgs p) {
    using G = SGeo<K, NK>;
    constexpr int R = G::R, KT = G::KT, KTS = G::KTS, NZ = G::NZ, OW = G::OW, NFW = G::NFW;
    constexpr int NZC = G::NZC, SLOT = G::SLOT, PG = G::PG, NR = G::NR, EROW = G::EROW;
    constexpr int WBG = 4 * kSPG, WMMA = WBG + kSBG;
    static_assert(kSBG == 4 || kSBG == 8, "BG warps");
    constexpr int VZ0 = kSlots * SLOT, VZW = G::VZW;
    constexpr int BAR_BG = 1;
    const StageArgs &a = p.a;
    extern __shared__ __align__(1024) float4 smem4[];
    float *s_par = reinterpret_cast<float *>(smem4);
    const float *s_bf = s_par;                         // hi [NK x KTS], lo after it
    const float *s_ba = s_par + 2 * NK * KTS;          // hi [NZ x NK], lo after it
    const float *s_pp = s_ba + 2 * NZ * NK;            // [NK/2][pps] filter-pair phi
    float *s_eh = s_par + a.tc_par_floats;             // E rows, hi [NR + 1][512]
    float *s_el = s_eh + (NR + 1) * EROW;              // E rows, lo
    float *s_ur = s_el + (NR + 1) * EROW;              // raw u rows [kNUR][kUP]
    float *s_fr = s_ur + kNUR * kUP;                   // raw f rows [kNUR][kFBW]
    float *s_z = s_fr + kNUR * kFBW;                   // [KT][kZP]
    float *s_d = s_z + KT * kZP;                       // [kSD][64]
    uint64_t *bar_v = reinterpret_cast<uint64_t *>(s_d + kSD * 64);
    uint64_t *bar_w = bar_v + kSlots, *bar_z = bar_w + kSlots, *bar_zf = bar_z + kSlots;
    uint64_t *bar_e = bar_zf + kSlots, *bar_t = bar_e + kNEF, *bar_g = bar_t + kNTB, *bar_ep = bar_g + kNG;
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(bar_ep + kNG);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int quarter = warp & 3, m = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const int H = a.H, W = a.W;

    {
        const float4 *src = reinterpret_cast<const float4 *>(a.params);
        for (int jj = tid; jj < a.tc_par_floats / 4; jj += kSNT) smem4[jj] = __ldg(src + jj);
        for (int jj = tid; jj < kSD * 64; jj += kSNT) s_d[jj] = 0.0f;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                     "n"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int s = 0; s < kSlots; ++s) {
            mbar_init(bar_v + s, 1);
            mbar_init(bar_w + s, 128 * PG);
            mbar_init(bar_z + s, 1);
            mbar_init(bar_zf + s, kNBG);
        }
        for (int s = 0; s < kNEF; ++s) mbar_init(bar_e + s, kNBG);
        for (int s = 0; s < kNG; ++s) {
            mbar_init(bar_g + s, kNBG);
            mbar_init(bar_ep + s, 1);
        }
        for (int s = 0; s < kNTB; ++s) mbar_init(bar_t + s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *s_tmem;
    const uint32_t tl = tmem + lane_off;

    // E rows of block `it` (its new rows), by threads t = 0..nt-1: per pixel c of the
    // 64-column v region and word jw, E[c][jw] = u_ext(row, xs(c) + R - 7 + jw) (tap
    // column 7 - jw; word 0 is padding for K = 7), xs(c) the v column's mirror pixel
    // (R1), split hi / lo.  The caller guarantees the forward bank of block g - 2 (and
    // its copies) completed: the E ring holds two blocks' tap rows.
    const auto build_e = [&](const BlockIter<K> &it, int t, int nt) {
        mbar_wait_dl(bar_t + it.g % kNTB, (it.g / kNTB) & 1);
        const int xr = floor4(it.x0 - 8);
        // every column x0 - 7 .. x0 + 63 in the image: no mirror needed
        const bool interior = it.x0 - 7 >= 0 && it.x0 + 63 <= W - 1;
        const int n = (it.new_hi() - it.new_lo()) * 64;
        for (int item = t; item < n; item += nt) {
            const int c = it.new_lo() + (item >> 6), px = item & 63;
            const float *ur = s_ur + (c % kNUR) * kUP;
            float v[8];
            if (interior) {
                const float *q = ur + (it.x0 + px - 7) - xr;
#pragma unroll
                for (int jw = 0; jw < 8; ++jw) v[jw] = q[jw];
            } else {
                const int xs = reflect(it.x0 - R + px, W);
#pragma unroll
                for (int jw = 0; jw < 8; ++jw) v[jw] = ur[clampi(reflect(xs + R - 7 + jw, W) - xr, 0, kUBW - 1)];
            }
            float vh[8], vl[8];
#pragma unroll
            for (int jw = 0; jw < 8; ++jw) {
                vh[jw] = tf32_hi_t<RN>(v[jw]);
                vl[jw] = v[jw] - vh[jw];
            }
            const int slot = c % NR;
            const int off = ((px >> 3) * 2) * 32 + (px & 7) * 4;   // core matrices (px / 8, words 0-3 | 4-7)
#pragma unroll
            for (int rep = 0; rep < 2; ++rep) {
                if (rep == 1 && slot != 0) break;   // slot 0 is also kept in the shadow row NR
                float *eh = s_eh + (rep ? NR : slot) * EROW + off, *el = s_el + (rep ? NR : slot) * EROW + off;
                *reinterpret_cast<float4 *>(eh) = make_float4(vh[0], vh[1], vh[2], vh[3]);
                *reinterpret_cast<float4 *>(eh + 32) = make_float4(vh[4], vh[5], vh[6], vh[7]);
                *reinterpret_cast<float4 *>(el) = make_float4(vl[0], vl[1], vl[2], vl[3]);
                *reinterpret_cast<float4 *>(el + 32) = make_float4(vl[4], vl[5], vl[6], vl[7]);
            }
        }
#ifndef TNRD_SX_NOFENCE
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // E rows visible to tcgen05.cp
#endif
        mbar_arrive(bar_e + it.g % kNEF);
    };

    if (warp < 4 * PG) {
        // ======================= phi warps (tc_stage_kernel's, block by block)
        const int h = warp >> 2;
        const int pps = a.pstride;
        BlockIter<K> it;
        SXP_DECL();
        for (it.init(p); it.valid(); it.next(p)) {
            const int s = it.g % kSlots;
            {
                SXP_T0(sxt1);
                mbar_wait_dl(bar_v + s, (it.g / kSlots) & 1);
                SXP_ADD(0, sxt1);
            }
            SXP_T0(sxt2);
            tc_fence_after();
            uint32_t vr[NFW];
            tmem_ld_nowait<NFW>(tl + VZ0 + VZW * s + h * NFW, vr);
            tmem_wait_ld(vr);
            f2 w[NFW / 2];
            if constexpr (TABLE) {
#pragma unroll
                for (int e = 0; e < NFW; ++e) {
                    const int fi = h * NFW + e;
                    const float4 fc = *reinterpret_cast<const float4 *>(s_pp + 4 * fi);
                    const float vv = __uint_as_float(vr[e]);
                    const float kf = floorf(fmaf(vv, fc.x, fc.y));
                    const float fr = fmaf(vv, fc.x, fc.y - kf) + fc.w;
                    const unsigned nint = (unsigned)__float2int_rn(fc.z);
                    const int k = __float2int_rz(kf);
                    const float4 c = __ldg(a.table + (size_t)fi * a.table_stride + ((unsigned)k < nint ? (unsigned)k : nint));
                    const float r = fmaf(fmaf(fmaf(c.w, fr, c.z), fr, c.y), fr, c.x);
                    if (e & 1) w[e / 2] = pk(lo(w[e / 2]), r);
                    else w[e / 2] = pk(r, 0.0f);
                }
            } else {
#ifdef TNRD_SX_NOPHI
#pragma unroll
                for (int e = 0; e < NFW / 2; ++e) w[e] = pk(__uint_as_float(vr[2 * e]), __uint_as_float(vr[2 * e + 1]));
#else
                phi_fpairs<NFW / 2>(s_pp + h * (NFW / 2) * pps, pps, vr, w);
#endif
            }
            // R2: w = 0 at v pixels outside the image (only columns: v rows are in-image)
            const int gxp = it.x0 - R + (m & 63);
            const bool zero_w = R2 && (unsigned)gxp >= (unsigned)W;
            uint32_t wh[NFW], wl[NFW];
#pragma unroll
            for (int e = 0; e < NFW; ++e) {
                const float x = zero_w ? 0.0f : ((e & 1) ? hi(w[e / 2]) : lo(w[e / 2]));
                const float xh = tf32_hi_t<RN>(x);
                wh[e] = __float_as_uint(xh);
                wl[e] = __float_as_uint(x - xh);
            }
            tmem_st<NFW>(tl + SLOT * s + h * NFW, wh);
            tmem_st<NFW>(tl + SLOT * s + NK + h * NFW, wl);
            tc_wait_st();
            tc_fence_before();
            mbar_arrive(bar_w + s);
            SXP_ADD(1, sxt2);
        }
        SXP_OUT(tid == 0);
    } else if (warp < WBG) {
        // phi warps of an unused group: idle
    } else if (warp < WMMA) {
        // ======================= BG warps: TMA, E rows, Z -> smem, gather, epilogue
        const int gt = tid - 32 * WBG;   // 0 .. kNBG - 1
        const int zhalf = kSBG == 8 ? (warp - WBG) >> 2 : 0;   // two BG warps per lane quarter split Z
        SXP_DECL();
        const CUtensorMap *tmu = &p.tm_u, *tmf = &p.tm_f;
        // TMA group of block `it`: its new u rows (and the f rows among them that are
        // output rows of the segment) into ring slots counter % kNUR (one elected lane)
        const auto tma_group = [&](const BlockIter<K> &it) {
            if (gt == 0) {
                const int xr = floor4(it.x0 - 8), xf = floor4(it.x0);
                uint32_t bytes = 0;
                for (int c = it.new_lo(); c < it.new_hi(); ++c) {
                    const int y = it.urow(c);
                    bytes += kUBW * 4 + ((y >= it.oy0 && y < it.oy1) ? kFBW * 4 : 0);
                }
                uint64_t *bar = bar_t + it.g % kNTB;
                mbar_expect_tx(bar, bytes);
                for (int c = it.new_lo(); c < it.new_hi(); ++c) {
                    const int y = it.urow(c);
                    const int ys = clampi(reflect(y, H), a.avail_lo, a.avail_hi - 1);
                    tma_row(s_ur + (c % kNUR) * kUP, tmu, xr, ys - a.avail_lo, it.b, bar);
                    if (y >= it.oy0 && y < it.oy1) tma_row(s_fr + (c % kNUR) * kFBW, tmf, xf, y - a.y_begin, it.b, bar);
                }
            }
        };
        BlockIter<K> gi, ei, ti;
        gi.init(p);
        ei = gi;
        ti = gi;
        for (int k = 0; k < 3 + kTmaAhead && ti.valid(); ++k, ti.next(p)) tma_group(ti);
        // The E ring holds two blocks' tap rows: block k's rows are written once the
        // forward bank of block k - 2 (and its copies) completed (V_full(k - 2)).
        const auto build_e_after = [&](const BlockIter<K> &it) {
            if (it.g >= 2) mbar_wait_dl(bar_v + (it.g - 2) % kSlots, ((it.g - 2) / kSlots) & 1);
            build_e(it, gt, kNBG);
        };
        for (int k = 0; k < 3 && ei.valid(); ++k, ei.next(p)) build_e_after(ei);
        int bg_next = 0;
        for (; gi.valid(); gi.next(p)) {
            const int s = gi.g % kSlots;
            if (ti.valid()) {   // TMA groups run kTmaAhead blocks ahead of the E rows
                tma_group(ti);
                ti.next(p);
            }
            // E rows of block g + 3 (the forward bank of g + 1 completed before Z_full(g - 1))
            // while the phi / adjoint bank of block g run
            if (ei.valid()) {
                SXP_T0(sxt5);
                build_e_after(ei);
                ei.next(p);
                SXP_ADD(3, sxt5);
            }
            {
                SXP_T0(sxt4);
                mbar_wait_dl(bar_z + s, (gi.g / kSlots) & 1);
                SXP_ADD(2, sxt4);
            }
            tc_fence_after();
            SXP_T0(sxt6);
            named_sync(BAR_BG, kNBG);   // every BG thread is done with gather(g - 1) / epilogue(g - 1)
#pragma unroll
            for (int ch = 0; ch < NZC; ++ch) {
                if (ch * 8 >= KT || (kSBG == 8 && (ch & 1) != zhalf)) continue;
                uint32_t z[8];
                tmem_ld_nowait<8>(tl + VZ0 + VZW * s + ch * 8, z);
                tmem_wait_ld(z);
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    if (ch * 8 + e < KT) s_z[(ch * 8 + e) * kZP + m] = __uint_as_float(z[e]);
            }
            tc_fence_before();
            mbar_arrive(bar_zf + s);   // slot s may take block g + 3
            SXP_ADD(5, sxt6);
            SXP_T0(sxt7);
#ifdef TNRD_SX_MMAEPI
            if (gi.g >= 2) mbar_wait_dl(bar_ep + (gi.g - 2) % kNG, ((gi.g - 2) / kNG) & 1);
#endif
            named_sync(BAR_BG, kNBG);
            // ---- gather: d(oy, x) += sum_b Z[(m, x + b)][ta K + b] for the block's rows m,
            // ta = m - oy + R; R1 adds row m again at its mirror row; R2 adds the terms of
            // the output pixel's mirror images (S l.57-65)
            const int m0 = gi.m0(), x0 = gi.x0;
            const auto S_cols = [&](int jj, int ta, int xc) {
                const float *zp = s_z + (ta * K) * kZP + jj * 64;
                float S = 0.0f;
#pragma unroll
                for (int tb = 0; tb < K; ++tb) {
                    const int c = xc + tb;
                    if (!R2 || (unsigned)c < 64u) S += zp[tb * kZP + c];
                }
                return S;
            };
#ifdef TNRD_SX_NOGATHER
            for (int item = gt; item < 0; item += kNBG) {
#else
            for (int item = gt; item < (2 * R + 2) * 64; item += kNBG) {
#endif
                const int oy = m0 - R + (item >> 6), x = item & 63;
                if (x >= OW || oy < gi.oy0 || oy >= gi.oy1 || x0 + x >= W) continue;
                float *dp = s_d + (oy & (kSD - 1)) * 64 + x;
                float d = *dp;
                const int gx = x0 + x;
                const int gxm = R2 ? (gx < R ? -1 - gx : (gx >= W - R ? 2 * W - 1 - gx : INT_MIN)) : INT_MIN;
                const int xm = gxm == INT_MIN ? 0 : gxm - x0;
                const int oym = R2 ? (oy < R ? -1 - oy : (oy >= H - R ? 2 * H - 1 - oy : INT_MIN)) : INT_MIN;
#pragma unroll
                for (int jj = 0; jj < 2; ++jj) {
                    const int mm = m0 + jj;
                    if (mm >= gi.vr1) break;
                    const int ta = mm - oy + R;
                    if (ta >= 0 && ta < K) {
                        d += S_cols(jj, ta, x);
                        if (R2 && gxm != INT_MIN) d += S_cols(jj, ta, xm);
                    }
                    if constexpr (R2) {
                        if (oym != INT_MIN) {
                            const int ta2 = mm - oym + R;
                            if (ta2 >= 0 && ta2 < K) {
                                d += S_cols(jj, ta2, x);
                                if (gxm != INT_MIN) d += S_cols(jj, ta2, xm);
                            }
                        }
                    } else {
                        // R1: w at mirror row mm' is w at mm (half-sample extension)
                        if (mm < R) {
                            const int ta1 = (-1 - mm) - oy + R;
                            if (ta1 >= 0 && ta1 < K) d += S_cols(jj, ta1, x);
                        }
                        if (mm >= H - R) {
                            const int ta1 = (2 * H - 1 - mm) - oy + R;
                            if (ta1 >= 0 && ta1 < K) d += S_cols(jj, ta1, x);
                        }
                    }
                }
                *dp = d;
            }
            SXP_ADD(6, sxt7);
#ifndef TNRD_SX_MMAEPI
            {
                const int mlast = min(m0 + 1, gi.vr1 - 1);
                if (gi.j == 0) bg_next = gi.oy0;
                const int done = gi.j == gi.nb - 1 ? gi.oy1 : min(gi.oy1, mlast - R + 1);
                mbar_wait_dl(bar_t + gi.g % kNTB, (gi.g / kNTB) & 1);
                if (done > bg_next) {
                    named_sync(BAR_BG, kNBG);
                    const int xr = floor4(x0 - 8), xf = floor4(x0);
                    float *ob = a.u_out + (long long)gi.b * a.out_img_stride;
                    for (int item = gt; item < (done - bg_next) * 64; item += kNBG) {
                        const int oy = bg_next + (item >> 6), x = item & 63;
                        if (x < OW && x0 + x < W) {
                            const int c = gi.eb + (oy - (gi.vr0 - R));
                            const float u = s_ur[(c % kNUR) * kUP + x0 + x - xr];
                            const float fv = s_fr[(c % kNUR) * kFBW + x0 + x - xf];
                            float *dp = s_d + (oy & (kSD - 1)) * 64 + x;
                            const float ut = u - *dp;
                            *dp = 0.0f;
                            const long long oi = (long long)(oy - a.out_row_base) * a.out_ld + x0 + x;
                            ob[oi] = reaction_step(a.reaction, u, ut, a.lambda, fv);
                            if (a.ut_out) a.ut_out[(long long)gi.b * a.out_img_stride + oi] = ut;
                        }
                    }
                    bg_next = done;
                }
            }
#endif
            mbar_arrive(bar_g + gi.g % kNG);   // d rows of block g summed (epilogue in the MMA warp)
        }
        SXP_OUT(gt == 0);
    } else {
        // ======================= MMA warp: TMA issue, E rows, copies of the A blocks, both GEMMs
        SXP_DECL();
        const uint32_t bf_hi = smem_u32(s_bf), bf_lo = bf_hi + 4 * NK * KTS;
        const uint32_t ba_hi = smem_u32(s_ba), ba_lo = ba_hi + 4 * NZ * NK;
        const uint32_t eh = smem_u32(s_eh), el = smem_u32(s_el);
        constexpr uint32_t SBO_F = (KTS / 4) * 128, SBO_A = (NK / 4) * 128;
        constexpr uint32_t id_f = idesc_tf32(NK), id_a = idesc_tf32(NZ);
        const uint64_t df_hi = umma_desc(bf_hi, SBO_F), df_lo = umma_desc(bf_lo, SBO_F);
        const uint64_t da_hi = umma_desc(ba_hi, SBO_A), da_lo = umma_desc(ba_lo, SBO_A);
        const auto fwd = [&](const BlockIter<K> &it) {
            const int g = it.g, s = g % kSlots;
            mbar_wait_dl(bar_e + g % kNEF, (g / kNEF) & 1);
            {
                SXP_T0(sxt10);
                if (g >= kSlots) mbar_wait_dl(bar_zf + s, ((g - kSlots) / kSlots) & 1);
                SXP_ADD(9, sxt10);
            }
            SXP_T0(sxt11);
            tc_fence_after();
            const uint32_t tA = tmem + SLOT * s, tV = tmem + VZ0 + VZW * s;
            const int e0 = it.e0();
            // warp-collective issue (operands in uniform registers, one elected lane):
            // the tensor pipe then runs at its own rate
            // tap row ta of the block: E rows of u rows (m0 + R - ta, m0 + 1 + R - ta),
            // counters e0 + 2R - ta and the next (adjacent in the ring, shadow row NR)
#pragma unroll
            for (int ta = 0; ta < K; ++ta) {
#ifndef TNRD_SX_NOCP
                const uint32_t rowoff = (uint32_t)((e0 + 2 * R - ta) % NR) * (EROW * 4);
                tmem_cp_128x256b_warp(tA + 8 * ta, umma_desc(eh + rowoff, 256));
                tmem_cp_128x256b_warp(tA + KTS + 8 * ta, umma_desc(el + rowoff, 256));
#endif
            }
#pragma unroll
            for (int k = 0; k < K; ++k) {   // V = A_lo B_hi + A_hi B_lo + A_hi B_hi
                mma_tf32_warp(tV, tA + KTS + 8 * k, df_hi + 16 * k, id_f, k > 0);
                mma_tf32_warp(tV, tA + 8 * k, df_lo + 16 * k, id_f, 1);
                mma_tf32_warp(tV, tA + 8 * k, df_hi + 16 * k, id_f, 1);
            }
            mma_commit_warp(bar_v + s);
            __syncwarp();
            SXP_ADD(11, sxt11);
        };
        const auto adj = [&](const BlockIter<K> &it) {
            const int g = it.g, s = g % kSlots;
            {
                SXP_T0(sxt12);
                mbar_wait_dl(bar_w + s, (g / kSlots) & 1);
                SXP_ADD(10, sxt12);
            }
            SXP_T0(sxt13);
            tc_fence_after();
            const uint32_t tW = tmem + SLOT * s, tZ = tmem + VZ0 + VZW * s;
#pragma unroll
            for (int k = 0; k < NK / 8; ++k) {   // Z = W_lo B_hi + W_hi B_lo + W_hi B_hi
                mma_tf32_warp(tZ, tW + NK + 8 * k, da_hi + 16 * k, id_a, k > 0);
                mma_tf32_warp(tZ, tW + 8 * k, da_lo + 16 * k, id_a, 1);
                mma_tf32_warp(tZ, tW + 8 * k, da_hi + 16 * k, id_a, 1);
            }
            mma_commit_warp(bar_z + s);
            __syncwarp();
            SXP_ADD(12, sxt13);
        };
        // epilogue of block `it` (32 lanes): the output rows whose taps are complete after
        // its gather -- u - d, the reaction, the store -- then the d rows are cleared
        int next_out = 0;
        const auto epilogue = [&](const BlockIter<K> &it) {
            SXP_T0(sxt14);
            if (it.j == 0) next_out = it.oy0;
            mbar_wait_dl(bar_g + it.g % kNG, (it.g / kNG) & 1);
            mbar_wait_dl(bar_t + it.g % kNTB, (it.g / kNTB) & 1);   // u / f rows of blocks <= g
            const int x0 = it.x0, m0 = it.m0();
            const int mlast = min(m0 + 1, it.vr1 - 1);
            const int done = it.j == it.nb - 1 ? it.oy1 : min(it.oy1, mlast - R + 1);
            const int xr = floor4(x0 - 8), xf = floor4(x0);
            const float lam = a.lambda;
            float *ob = a.u_out + (long long)it.b * a.out_img_stride;
            for (int item = lane; item < (done - next_out) * 64; item += 32) {
                const int oy = next_out + (item >> 6), x = item & 63;
                if (x < OW && x0 + x < W) {
                    const int c = it.eb + (oy - (it.vr0 - R));
                    const float u = s_ur[(c % kNUR) * kUP + x0 + x - xr];
                    const float fv = s_fr[(c % kNUR) * kFBW + x0 + x - xf];
                    float *dp = s_d + (oy & (kSD - 1)) * 64 + x;
                    const float ut = u - *dp;
                    *dp = 0.0f;
                    const long long oi = (long long)(oy - a.out_row_base) * a.out_ld + x0 + x;
#ifdef TNRD_SX_NOEPI
                    if (ut == 12345.0f)
#endif
                    ob[oi] = reaction_step(a.reaction, u, ut, lam, fv);
                    if (a.ut_out) a.ut_out[(long long)it.b * a.out_img_stride + oi] = ut;
                }
            }
            next_out = max(next_out, done);
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_ep + it.g % kNG);   // d rows of block g cleared
            __syncwarp();
            SXP_ADD(7, sxt14);
        };
        BlockIter<K> fi, ai, pi;
        fi.init(p);
        ai = fi;
        pi = fi;
        for (int k = 0; k < kSlots && fi.valid(); ++k, fi.next(p)) fwd(fi);
        for (; ai.valid(); ai.next(p)) {
            adj(ai);
            if (fi.valid()) {
                fwd(fi);
                fi.next(p);
            }
#ifndef TNRD_SX_MMAEPI
            if (ai.g < 0) {
#else
            if (ai.g >= 1) {   // block g - 1 (its gather ran during phi(g))
#endif
                epilogue(pi);
                pi.next(p);
            }
        }
#ifdef TNRD_SX_MMAEPI
        for (; pi.valid(); pi.next(p)) epilogue(pi);
#endif
        SXP_OUT(lane == 0);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols));
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encoder() {
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

// rows [r0, r1) of an Image as a (W, rows, B) fp32 tensor map with a one-row box
bool encode_rows(CUtensorMap *tm, const float *base, long long ld, long long img_stride, int W, int rows, int B,
                 int box) {
    EncodeTiled enc = encoder();
    if (!enc || rows < 1) return false;
    cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)rows, (cuuint64_t)B};
    const long long s2 = B > 1 ? img_stride : (long long)rows * ld;
    cuuint64_t strides[2] = {(cuuint64_t)ld * 4, (cuuint64_t)s2 * 4};
    cuuint32_t boxd[3] = {(cuuint32_t)box, 1, 1}, es[3] = {1, 1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(base), dims, strides, boxd, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <int K, int NK>
cudaError_t launch_stream(const StageArgs &a, int B, int num_sms, cudaStream_t s) {
    using G = SGeo<K, NK>;
    auto kern = a.tc_rn ? (a.boundary == 1 ? tc_stream_kernel<K, NK, false, true, true>
                                           : tc_stream_kernel<K, NK, false, false, true>)
              : a.boundary == 1 ? (a.mode == MODE_TABLE ? tc_stream_kernel<K, NK, true, true, false>
                                                        : tc_stream_kernel<K, NK, false, true, false>)
                                : (a.mode == MODE_TABLE ? tc_stream_kernel<K, NK, true, false, false>
                                                        : tc_stream_kernel<K, NK, false, false, false>);
    if (a.tc_rn && a.mode == MODE_TABLE) return cudaErrorInvalidValue;
    StreamArgs p;   // kernel parameter (copied at launch)
    std::memset(&p, 0, sizeof p);
    p.a = a;
    const long long u_off = (long long)(a.avail_lo - a.u_in.row_base) * a.u_in.ld;
    const long long f_off = (long long)(a.y_begin - a.f.row_base) * a.f.ld;
    if (!encode_rows(&p.tm_u, a.u_in.ptr + u_off, a.u_in.ld, a.u_in.img_stride, a.W, a.avail_hi - a.avail_lo, B, kUBW) ||
        !encode_rows(&p.tm_f, a.f.ptr + f_off, a.f.ld, a.f.img_stride, a.W, a.y_end - a.y_begin, B, kFBW))
        return cudaErrorInvalidValue;
    p.nstrips = (a.W + G::OW - 1) / G::OW;
    p.nrp = (a.y_end - a.y_begin + 1) / 2;
    p.units = (long long)B * p.nstrips * p.nrp;
    if (p.units < 1) return cudaSuccess;
    const size_t smem = sizeof(float) * (size_t)stream_smem_floats<K, NK>(a.tc_par_floats);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int grid = (int)std::min<long long>(num_sms, p.units);
#ifdef TNRD_SX_PROF
    // role timers: phi (wait V, compute), BG (wait Z, build E, wait TMA, Z move, gather,
    // epilogue), MMA (wait E, wait Z_free, wait W, fwd issue, adj issue); slot 15 = total
    static unsigned long long *prof = nullptr;
    if (!prof) cudaMalloc(&prof, sizeof(unsigned long long) * 16 * 1024);
    cudaMemsetAsync(prof, 0, sizeof(unsigned long long) * 16 * 1024, s);
    p.prof = prof;
    kern<<<grid, kSNT, smem, s>>>(p);
    std::vector<unsigned long long> hp(16 * (size_t)grid);
    cudaMemcpyAsync(hp.data(), prof, sizeof(unsigned long long) * hp.size(), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    double acc[16] = {0};
    for (int c = 0; c < grid; ++c)
        for (int k = 0; k < 16; ++k) acc[k] += (double)hp[c * 16 + k] / grid;
    fprintf(stderr, "SXPROF");
    for (int k = 0; k < 16; ++k) fprintf(stderr, " %.0f", acc[k]);
    fprintf(stderr, "\n");
    return cudaGetLastError();
#else
    kern<<<grid, kSNT, smem, s>>>(p);
    return cudaGetLastError();
#endif
}

}  // namespace

// The streaming engine applies to (ksize, N_k) = (7, 48) with 16-byte aligned rows
// (TMA): ld, image strides and the row bases of u_in, f multiples of 4 floats.
bool stream_supported(int ksize, int Nk) { return ksize == 7 && Nk == 48; }

bool stream_args_ok(const StageArgs &a) {
    const long long u_off = (long long)(a.avail_lo - a.u_in.row_base) * a.u_in.ld;
    const long long f_off = (long long)(a.y_begin - a.f.row_base) * a.f.ld;
    return a.u_in.ld % 4 == 0 && a.f.ld % 4 == 0 && a.u_in.img_stride % 4 == 0 && a.f.img_stride % 4 == 0 &&
           aligned16(a.u_in.ptr + u_off) && aligned16(a.f.ptr + f_off) && encoder() != nullptr;
}

size_t stream_smem_bytes(int ksize, int Nk, int par_floats) {
    if (ksize == 7 && Nk == 48) return sizeof(float) * (size_t)stream_smem_floats<7, 48>(par_floats);
    return 0;
}

cudaError_t launch_stage_stream(int ksize, const StageArgs &a, int B, int num_sms, cudaStream_t s) {
    if (ksize == 7 && a.Nk == 48) return launch_stream<7, 48>(a, B, num_sms, s);
    return cudaErrorInvalidValue;
}

}  // namespace tnrd
