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
// 3xTF32: every fp32 operand x is split as x = hi + lo (hi: TF32, x - hi exact in
// fp32) and the GEMM accumulates A_lo B_hi + A_hi B_lo + A_hi B_hi in fp32 TMEM,
// dropping A_lo B_lo.  Taps (B) are split on the host with round-to-nearest (|lo| <=
// 2^-11 |x|), data (A: u, w) here by truncation (one LOP3; |lo| < 2^-10 |x|), so
// each product is exact to < 2^-20 relative.  Measured on B200 (tools/tc_probe.cu):
// 3e-7 of sum |products| against 3e-4 for plain TF32, which fails the 1e-4 peak
// tolerance by 30x; an fp32 emulation of the whole pass with this split stays at
// 0.04-0.06 of the tolerance on C4/C5 windows, as fp32 does.
//
// Data flow per tile (output OW x OH, v region 64 x (OH + 2r), u region + 2r):
// the v region is cut into M-blocks of two 64-pixel rows; TMEM lane m = pixel m of
// the block; up to three blocks are in flight in three TMEM slots.  Per block:
// (1) build warps write each pixel's im2col row (hi, lo) into TMEM (tcgen05.st, A
// from TMEM; out-of-image pixels take the row of their mirror pixel, so w there is
// the half-sample mirror of the in-image w, R1); (2) the MMA thread issues the
// forward bank (B = taps in shared memory); (3) phi warps read the responses back
// (tcgen05.ld), evaluate phi with the FP32 engine's blocked-Horner units (bitwise
// the same phi) and write w (hi, lo) over the dead im2col columns; (4) the MMA
// thread issues the adjoint bank into Z; (5) gather warps move Z to shared memory
// and add each output pixel's K tap rows of the block to d in a fixed order (a
// ascending, b ascending), so d is deterministic and independent of tiling and
// batching (R2: mirror-image terms at image edges, w = 0 outside the image).
// (6) the same warps finish the two output rows the block completed (u - d, the
// reaction, the store).  The kernel is persistent: one CTA per SM walks its tiles
// with one M-block pipeline across tile boundaries, u tiles arrive by TMA, and the
// forward / adjoint MMAs are issued by two warps.  Hand-offs are
// mbarriers; see tc_stage_kernel.  Macros TNRD_EXP_*, TNRD_TC_PROF and TNRD_TC_{BG,
// GP, PG, MMAW, 2MMA, RELAY, PHI_HW, NAP_*} are timing experiments / tuning knobs
// whose defaults are the product.
#include "tnrd_tc_common.cuh"

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

namespace tnrd {
namespace {

#ifndef TNRD_TC_BG
#define TNRD_TC_BG 8
#endif
constexpr int kBG = TNRD_TC_BG;                 // build / gather warps (4 or 8: one or two per lane quarter)
constexpr int kNBG = 32 * kBG;                  // build / gather threads
#ifndef TNRD_TC_PHI_HW
#define TNRD_TC_PHI_HW 1
#endif
#ifndef TNRD_TC_MMAW
#define TNRD_TC_MMAW 0
#endif
#ifndef TNRD_TC_2MMA
#define TNRD_TC_2MMA 1
#endif
constexpr bool kMmaWarp = TNRD_TC_MMAW;         // MMAs issued by the converged warp (elected lane)
constexpr int kNMMA = TNRD_TC_2MMA ? 2 : 1;     // MMA issuer warps (2: forward and adjoint banks apart)
#ifndef TNRD_TC_RELAY
#define TNRD_TC_RELAY 3
#endif
constexpr int kRelay = TNRD_TC_RELAY;           // a relay warp turns V_full into hardware barriers for the phi warps (3: one per filter group; 2: one per lane quarter; 1: one; 0: the phi warps poll)
#ifdef TNRD_TC_TRACE
constexpr int kObs = 1;                         // trace builds: an observer warp stamps Z_full(g)
#else
constexpr int kObs = 0;
#endif
constexpr int kTNT = (4 * kPG + kBG + kNMMA + (kRelay ? 1 : 0) + kObs) * 32;  // phi warps, build / gather warps, MMA warp(s), relay
static_assert(kBG == 4 || kBG == 8, "build / gather warps");

template <int K, int NK>
struct TcGeo {
    static constexpr int R = K / 2, KT = K * K;
    static constexpr int KTP = tc_ktp(K), NZ = tc_nz(K);
    static constexpr int OW = kTcVW - 2 * R;   // output columns per tile
    static constexpr int UW = kTcVW + 2 * R;   // u tile columns
    static constexpr int UP = (UW + 3 + 3) / 4 * 4;   // u tile pitch = TMA box width (16-byte start, <= 3 lead)
    static constexpr int PG = (NK % (2 * kPG) == 0) ? kPG : 2;  // phi groups used
    static constexpr int NFW = NK / PG;        // filters per phi warp
    static constexpr int NCH = KTP / 8;        // 8-column chunks of an im2col row
    static constexpr int NZC = NZ / 8;         // 8-column chunks of a Z row
    static constexpr int SLOT = 2 * (KTP > NK ? KTP : NK);   // A / W columns of a slot
    static constexpr int DR = 8;               // d ring rows (>= K + 1 rows live per block)
    static_assert(NK % 8 == 0 && NK <= 64 && NFW % 2 == 0, "N_k: multiple of 8, at most 64");
    static_assert(kSlots * (SLOT + (NK > NZ ? NK : NZ)) <= kTmemCols, "TMEM column plan");
    static_assert(K + 1 <= DR, "d ring");
};

__host__ __device__ constexpr int round4(int x) { return (x + 3) / 4 * 4; }
__host__ __device__ constexpr int round32(int x) { return (x + 31) / 32 * 32; }

// Kernel parameter: the stage arguments plus the TMA map of u_in's rows
// [avail_lo, avail_hi) as a (W, rows, B) tensor with a (UP, UH, 1) box.
struct alignas(64) TcArgs {
    CUtensorMap tm_u;
    StageArgs a;
    int use_tma;   // 0: u tiles by per-element loads (rows not 16-byte aligned / no driver entry point)
    unsigned long long *prof;   // TNRD_TC_PROF builds: per CTA and warp {wait cycles, total cycles}
};
// phi (V) and build/gather (Z) waits: test_wait + __nanosleep(NAP ns) polls (0: try_wait
// with a suspend hint)
#ifndef TNRD_TC_NAP_PHI
#define TNRD_TC_NAP_PHI 256
#endif
#ifndef TNRD_TC_NAP_BG
#define TNRD_TC_NAP_BG 0
#endif
template <int NAP>
__device__ __forceinline__ void mbar_wait_nap(uint64_t *bar, uint32_t parity) {
    if constexpr (NAP == 0) {
        mbar_wait(bar, parity);
    } else {
        while (!mbar_test(bar, parity, false)) __nanosleep(NAP);
    }
}
// TNRD_TC_TRACE builds (with TNRD_TC_PROF): CTA 0 stamps clock64 per block g and event e
// into prof[16384 + 64 (g - 1000) + e], 1000 <= g < 1256 (e >= 8: build / gather warp (e - 8) / 6,
// step (e - 8) % 6: has Z, Z moved, A built, second sync passed, gathered, epilogue done; e: 0 phi warp 0 has V, 1 its W arrived, 2 build/gather has
// Z, 3 A(g + 3) arrived, 4 epilogue done, 5 relay saw V_full, 6 Adj issuer saw W_full,
// 7 F issuer saw A_full); launch_tc writes them to gpurun_out/tc_trace.bin
#ifdef TNRD_TC_TRACE
// TNRD_TC_TRACE=1: only events 0, 1, 2 and 56 (light: the stamps themselves cost issue slots)
#define TCT(g, e, cond) if ((TNRD_TC_TRACE > 1 || (e) <= 2 || (e) == 56) && blockIdx.x == 0 && (cond) && (g) >= 1000 && (g) < 1256) p.prof[16384 + 64 * ((g) - 1000) + (e)] = (unsigned long long)clock64()
#else
#define TCT(g, e, cond)
#endif
#ifdef TNRD_TC_PROF
#define TCP_WAIT(NAP, bar, par) { const long long t0_ = clock64(); mbar_wait_nap<NAP>(bar, par); tcp_wait += clock64() - t0_; }
#define TCP_SYNC(id, n) { const long long t0_ = clock64(); named_sync(id, n); tcp_wait += clock64() - t0_; }
#else
#define TCP_WAIT(NAP, bar, par) mbar_wait_nap<NAP>(bar, par)
#define TCP_SYNC(id, n) named_sync(id, n)
#endif

// Shared memory (floats): operand block | u tiles [2][UH][UP] (128-byte aligned, TMA
// destinations) | d ring [DR][OW] | Z of two M-blocks [2][KT][kZP] (one with the
// tabulated phi, whose table lives in L1: the unified L1 / shared memory is 256 KB) | mbarriers
// (4 x kSlots + 2) | TMEM address.
template <int K, int NK>
__host__ __device__ constexpr int tc_u_floats(int oh) {
    using G = TcGeo<K, NK>;
    return round32((oh + 4 * G::R) * G::UP);
}
template <int K, int NK>
__host__ __device__ constexpr int tc_smem_floats(int oh, int par_floats, int zb = 2) {
    using G = TcGeo<K, NK>;
    return round32(par_floats) + 2 * tc_u_floats<K, NK>(oh) + round4(G::DR * G::OW) + zb * G::KT * kZP +
           2 * (4 * kSlots + 2) + 4;
}


// Persistent: one CTA per SM walks the tiles blockIdx.x, + gridDim.x, ... (58 x OH
// outputs each; v region 64 x (OH + 2r)).  The stage operands are loaded and TMEM
// is allocated once per CTA, and the M-blocks of consecutive tiles form one
// pipeline (global block g = tile n * nmb + i, TMEM slot g % 3), so the next
// tile's first blocks are built and multiplied while the current tile's last ones
// are in phi and the gather: there is no fill / drain per tile.  TMEM lane m =
// pixel (2i + m/64, m%64) of block i.  Warp roles, handing blocks over through
// mbarriers (no CTA-wide barrier until the end):
//   4 PG phi warps: warp w serves lane quarter w % 4, filters [NFW (w/4), +NFW):
//               wait V(g), tcgen05.ld, phi, W (hi, lo) -> TMEM, arrive W_full(g)
//   4 build / gather warps (lane quarter w % 4): im2col A(g) -> TMEM, arrive
//               A_full(g); wait Z(g), Z -> smem, A(g+3) into the freed slot, then
//               d += the block's taps (blocks in order: d summed in v-row order),
//               then the epilogue of the two output rows the block completed
//               (u - d, reaction, store).  u tiles are double buffered: tile n+1's
//               is requested by TMA when tile n starts and waited for (plus the
//               mirror fix-up of edge tiles) before its first im2col row.
//   2 MMA warps (lane 0 issues the 3xTF32 MMAs; the converged warp with an elected lane
//               for the tabulated phi): one issues F(g) on A_full(g) -> V_full(g), the
//               other Adj(g) on W_full(g) -> Z_full(g)
//   relay warp  waits for V_full(g) (the mbarrier the MMA commit arrives on) and
//               arrives on the hardware barriers (one per slot and filter group: the 4 phi warps
//               of a scheduler belong to 4 different barriers, so they are not forced into
//               the same phase) the phi warps sleep in:
//               16 polling phi warps cost 1.06 G spin instructions per C4 launch
//               (13 % of all issued, ncu) - a bar.sync wait costs none
// phi: the two half-warps of a phi warp swap half of their responses, so a thread
// evaluates NFW/2 filters on two pixels with one set of constants (phi_halfwarp:
// half the broadcast constant loads and range set-ups, bitwise the same w).
template <int K, int NK, bool TABLE, bool R2, bool RN>
__global__ void __launch_bounds__(kTNT, 1) tc_stage_kernel(const __grid_constant__ TcArgs p) {
    using G = TcGeo<K, NK>;
    constexpr int R = G::R, KT = G::KT, KTP = G::KTP, NZ = G::NZ, OW = G::OW, UW = G::UW, UP = G::UP;
    constexpr int NFW = G::NFW, NCH = G::NCH, NZC = G::NZC, SLOT = G::SLOT, PG = G::PG, DR = G::DR;
    constexpr int WBG = 4 * kPG, WMMA = WBG + kBG;   // first build / gather warp, MMA warp
    constexpr int VZ0 = kSlots * SLOT, VZW = NK > NZ ? NK : NZ;  // V / Z columns of slot s at VZ0 + VZW s
    constexpr int BAR_BG = 1, BAR_V = 2;             // named barriers: build / gather group, V of slot s at BAR_V + s
    const StageArgs &a = p.a;
    extern __shared__ __align__(1024) float4 smem4[];
    float *s_par = reinterpret_cast<float *>(smem4);
    const float *s_bf = s_par;                       // hi [NK x KTP], lo after it
    const float *s_ba = s_par + 2 * NK * KTP;        // hi [NZ x NK], lo after it
    const float *s_pp = s_ba + 2 * NZ * NK;          // [NK/2][pps] filter-pair phi
    const int OH = a.tc_oh, VH = OH + 2 * R, UH = OH + 4 * R;
    const int UF = tc_u_floats<K, NK>(OH);
    float *s_u0 = s_par + round32(a.tc_par_floats);  // u tile of local tile n: s_u0 + (n & 1) UF
    float *s_d = s_u0 + 2 * UF;                      // ring: output row y at (y % DR) OW
    constexpr int ZB = TABLE ? 1 : 2;                // Z buffers (tabulated phi: one, the table wants the L1)
    float *s_z0 = s_d + round4(DR * OW);             // [ZB][KT][kZP]: Z of block g at (g % ZB) KT kZP
    uint64_t *bar_a = reinterpret_cast<uint64_t *>(s_z0 + ZB * KT * kZP);   // A_full[kSlots]
    uint64_t *bar_v = bar_a + kSlots, *bar_w = bar_v + kSlots, *bar_z = bar_w + kSlots;
    uint64_t *bar_u = bar_z + kSlots;                // u tile landed [2]
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(bar_u + 2);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int quarter = warp & 3, m = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const int H = a.H, W = a.W;
    const int nmb = VH / 2;
    const int ntl = (a.n_tiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;  // tiles of this CTA
    const int nblk = ntl * nmb;                      // M-blocks of this CTA
    const int per_img = a.tiles_x * a.tiles_y;
    struct Tile { int b, x0, y0; };
    const auto tile_of = [&](int n) {                // local tile n
        const int t = (int)blockIdx.x + n * (int)gridDim.x;
        Tile T;
        T.b = t / per_img;
        const int rem = t - T.b * per_img;
        const int ty = rem / a.tiles_x;
        T.x0 = (rem - ty * a.tiles_x) * OW;
        T.y0 = a.y_begin + ty * OH;
        return T;
    };
    // tile column x0 - 2r + c lives at s_u[r UP + c + lead]: TMA boxes start 16-byte aligned
    const auto lead_of = [](int x0) { const int gx = x0 - 2 * R; return gx - (gx >= 0 ? (gx & ~3) : -((-gx + 3) & ~3)); };

    // ---- stage operands -> smem, d ring = 0, TMEM, barriers
    {
        const float4 *src = reinterpret_cast<const float4 *>(a.params);
        for (int j = tid; j < a.tc_par_floats / 4; j += kTNT) smem4[j] = __ldg(src + j);
        for (int j = tid; j < DR * OW; j += kTNT) s_d[j] = 0.0f;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                     "n"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int s = 0; s < kSlots; ++s) {
            mbar_init(bar_a + s, kBG);          // one arrival per warp (lane 0 after __syncwarp)
            mbar_init(bar_v + s, 1);
            mbar_init(bar_w + s, 4 * PG);
            mbar_init(bar_z + s, 1);
        }
        mbar_init(bar_u, 1);
        mbar_init(bar_u + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // operands visible to the MMA (async proxy)
    // programmatic dependent launch: the set-up above overlaps the previous stage's
    // tail; images (u_in, f, u_out) are touched only after that grid has completed
    asm volatile("griddepcontrol.wait;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *s_tmem;
    const uint32_t tl = tmem + lane_off;
#ifdef TNRD_TC_PROF
    long long tcp_wait = 0;
    const long long tcp_t0 = clock64();
#endif

    if (warp < 4 * PG) {
        // ======================= phi warps
        const int h = warp >> 2;
        const int pps = a.pstride;
        int tn = 0, ti = 0;            // tile / block of g (R2's out-of-image test)
        Tile tT = tile_of(0);
        for (int g = 0; g < nblk; ++g) {
            const int s = g % kSlots;
            if constexpr (kRelay) {
#ifdef TNRD_TC_PROF
                const long long t0_ = clock64();
#endif
                if constexpr (kRelay == 3)   // one barrier per slot and filter group: its 4 warps sit on 4 schedulers
                    asm volatile("bar.sync %0, %1;" ::"r"(BAR_V + PG * s + h), "n"(5 * 32) : "memory");
                else if constexpr (kRelay == 2)   // one barrier per slot and lane quarter (the PG warps of one scheduler)
                    asm volatile("bar.sync %0, %1;" ::"r"(BAR_V + 4 * s + quarter), "n"((PG + 1) * 32) : "memory");
                else
                    asm volatile("bar.sync %0, %1;" ::"r"(BAR_V + s), "n"((4 * PG + 1) * 32) : "memory");
#ifdef TNRD_TC_PROF
                tcp_wait += clock64() - t0_;
#endif
            } else {
                TCP_WAIT(TNRD_TC_NAP_PHI, bar_v + s, (g / kSlots) & 1);
            }
            tc_fence_after();
            TCT(g, 0, tid == 0);
            uint32_t vr[NFW];
            tmem_ld_nowait<NFW>(tl + VZ0 + VZW * s + h * NFW, vr);
            tmem_wait_ld(vr);
            f2 w[NFW / 2];
#ifdef TNRD_EXP_NOPHI
#pragma unroll
            for (int e = 0; e < NFW / 2; ++e) w[e] = pk(__uint_as_float(vr[2 * e]), __uint_as_float(vr[2 * e + 1]));
#else
            if constexpr (TABLE) {
                // tabulated phi (TNRD_PHI_TABLE): per filter {a_t, b_t,
                // n_int, b_lo} in the operand block, the cubic intervals in global
                // memory; the FP32 engine's arithmetic (phi_table_x2), value by value
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
#if TNRD_TC_PHI_HW
                if constexpr (NFW % 4 == 0) phi_halfwarp<NFW>(s_pp + h * (NFW / 2) * pps, pps, vr, w, lane);
                else phi_fpairs<NFW / 2>(s_pp + h * (NFW / 2) * pps, pps, vr, w);
#else
                phi_fpairs<NFW / 2>(s_pp + h * (NFW / 2) * pps, pps, vr, w);
#endif
            }
#endif
            // R2 (exact K^T): w is zero outside the image (the gather adds the mirror
            // images instead); R1 keeps the mirrored w of out-of-image pixels
            bool zero_w = false;
            if constexpr (R2) {
                const int gyp = tT.y0 - R + 2 * ti + (m >> 6), gxp = tT.x0 - R + (m & 63);
                zero_w = (unsigned)gyp >= (unsigned)H || (unsigned)gxp >= (unsigned)W;
                if (++ti == nmb) { ti = 0; if (++tn < ntl) tT = tile_of(tn); }
            }
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
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_w + s);
            TCT(g, 1, tid == 0);
        }
    } else if (warp < WBG) {
        // phi warps of an unused group (N_k not divisible): idle until the end
    } else if (warp < WMMA) {
        // ======================= build / gather warps
        const int gt = tid - 32 * WBG;  // 0 .. kNBG - 1
        const int half = kBG == 8 ? gt >> 7 : 0;   // which of a lane quarter's BG warps
        // u tile of local tile n -> s_u0 + (n & 1) UF: rows y0 - 2r .., columns x0 - 2r ..
        // at [r][c + lead]; element (r, c) = u(clamp(mirror(y0 - 2r + r)), mirror(x0 - 2r + c))
        const auto request_u = [&](int n) {       // TMA of the box (one thread)
            if (!p.use_tma || gt != 0) return;
            const Tile T = tile_of(n);
            const int gx = T.x0 - 2 * R;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic reads of the buffer
            mbar_expect_tx(bar_u + (n & 1), (uint32_t)(UH * UP * 4));
            tma_load_3d(s_u0 + (n & 1) * UF, &p.tm_u, gx - lead_of(T.x0), T.y0 - 2 * R - a.avail_lo, T.b,
                        bar_u + (n & 1));
        };
        const auto ensure_u = [&](int n) {        // all BG threads: tile n's u is complete in smem
            const Tile T = tile_of(n);
            float *su = s_u0 + (n & 1) * UF + lead_of(T.x0);
            const float *ub = a.u_in.ptr + (long long)T.b * a.u_in.img_stride;
            const int gy0 = T.y0 - 2 * R, gx0 = T.x0 - 2 * R;
            const auto load = [&](int r, int c) {
                int gy = reflect(gy0 + r, H);
                gy = min(max(gy, a.avail_lo), a.avail_hi - 1);
                const int gx = reflect(gx0 + c, W);
                su[r * UP + c] = __ldg(ub + (long long)(gy - a.u_in.row_base) * a.u_in.ld + gx);
            };
            if (p.use_tma) {
                mbar_wait(bar_u + (n & 1), (n >> 1) & 1);
                // mirror fix-up (TMA zero-filled what lies outside rows [avail_lo, avail_hi)
                // or columns [0, W)): rows [0, rA) and [rB, UH) whole, the others' columns
                // [0, cA) and [cB, UW)
                const int rA = min(max(a.avail_lo - gy0, 0), UH), rB = max(min(a.avail_hi - gy0, UH), rA);
                const int cA = min(max(-gx0, 0), UW), cB = max(min(W - gx0, UW), cA);
                const int nrow = rA + UH - rB, ncol = cA + UW - cB;
                for (int j = gt; j < nrow * UW; j += kNBG) {
                    const int q = j / UW, c = j - q * UW;
                    load(q < rA ? q : rB + (q - rA), c);
                }
                for (int j = gt; j < (rB - rA) * ncol; j += kNBG) {
                    const int q = j / ncol, c = j - q * ncol;
                    load(rA + q, c < cA ? c : cB + (c - cA));
                }
            } else {
                for (int j = gt; j < UH * UW; j += kNBG) {
                    const int r = j / UW;
                    load(r, j - r * UW);
                }
            }
            named_sync(BAR_BG, kNBG);
        };
        int bn = 0, bi = 0;            // tile / block of the next build (builds run in g order)
        Tile bT = tile_of(0);
        int bcol = 0;                  // per tile: float offset of this thread's im2col column in the u tiles
        const auto build = [&](int s) {
            // im2col row (hi, lo) of pixel m of the next block (TMEM slot s): v-region (j, c)
            // uses its mirror in the image (R1), clamped into the tile for pixels no
            // output needs.  The column part of the address is per tile, the row part
            // per block
            const int n = bn, i = bi;
            if (i == 0) {
                ensure_u(n);
                const int c = m & 63;
                const int gx = reflect(bT.x0 - R + c, W);
                const int pc = min(max(gx - bT.x0 + R, 0), kTcVW - 1);
                bcol = (n & 1) * UF + lead_of(bT.x0) + 2 * R * UP + pc + 2 * R;
            }
            const int yv = bT.y0 - R;  // first v row of the tile
            const int pj = min(max(reflect(yv + 2 * i + (m >> 6), H) - yv, 0), VH - 1);
            const float *up = s_u0 + bcol + pj * UP;   // tap (ta, tb) reads up[-ta*UP - tb]
            if (++bi == nmb) { bi = 0; if (++bn < ntl) bT = tile_of(bn); }
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) {
                if (kBG == 8 && (ch < (NCH + 1) / 2) != (half == 0)) continue;   // chunks split by half
                uint32_t hv[8], lv[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const int t = ch * 8 + e;
                    float x = 0.0f;
                    if (t < KT) x = up[-(t / K) * UP - (t % K)];
                    const float xh = tf32_hi_t<RN>(x);
                    hv[e] = __float_as_uint(xh);
                    lv[e] = __float_as_uint(x - xh);
                }
                tmem_st8(tl + SLOT * s + ch * 8, hv);
                tmem_st8(tl + SLOT * s + KTP + ch * 8, lv);
            }
            tc_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_a + s);
        };
        if (nblk > 0) request_u(0);
        for (int g = 0; g < kSlots && g < nblk; ++g) build(g);   // slot g
        const int x = gt & 63;
        // gather row group of this thread (rows rg, rg + kNBG/64, ... of the block's K + 1;
        // groups 0 and 1 also run the epilogue).  With two warps per lane quarter the
        // second half - whose share of the im2col / Z chunks is the smaller one (the
        // last chunk is mostly padding) - takes groups 0 and 1, so the epilogue lands
        // on the less loaded warps
        const int rg = kBG == 8 ? ((gt >> 6) + 2) & 3 : gt >> 6;
        int n = 0, i = 0;              // tile / block of g
        Tile T = tile_of(0);
        // per tile: element index of this thread's column in tile row 0 of f and of the output
        long long fi_t = 0, oi_t = 0;
        const auto tile_bases = [&]() {
            fi_t = (long long)T.b * a.f.img_stride + (long long)(T.y0 - a.f.row_base) * a.f.ld + (T.x0 + x);
            oi_t = (long long)T.b * a.out_img_stride + (long long)(T.y0 - a.out_row_base) * a.out_ld + (T.x0 + x);
        };
        tile_bases();
        for (int g = 0; g < nblk; ++g) {
            const int s = g % kSlots;
            // the epilogue pixel of this block (row groups 0 and 1: output row 2i - (K-1) +
            // rg, column x): its f is fetched now, used after the gather
            const int ye = rg < 2 ? 2 * i - (K - 1) + rg : -1, oye = T.y0 + ye, oxe = T.x0 + x;
            const bool epi = ye >= 0 && x < OW && oye < a.y_end && oxe < W;
            float fv = 0.0f;
            if (epi) fv = __ldg(a.f.ptr + (fi_t + ye * a.f.ld));
            TCP_WAIT(TNRD_TC_NAP_BG, bar_z + s, (g / kSlots) & 1);
            tc_fence_after();
            TCT(g, 57 + (gt >> 5), lane == 0 && gt < 224);
            TCT(g, 2, gt == 0);
            TCT(g, 8 + 6 * (gt >> 5) + 0, lane == 0);
            // Z(g) -> s_z[g & 1] (two buffers: the gather of block g - 1 may still be reading
            // the other one; buffer g & 1 was last read by gather(g - 2), which every thread
            // finished before the barrier of iteration g - 1)
            float *s_z = s_z0 + (ZB == 2 ? (g & 1) * (KT * kZP) : 0);
            if constexpr (ZB == 1) TCP_SYNC(BAR_BG, kNBG);   // one buffer: gather(g - 1) must be over
#pragma unroll
            for (int ch = 0; ch < NZC; ++ch) {
                if (ch * 8 >= KT) continue;
                if (kBG == 8 && (ch < ((KT + 7) / 8 + 1) / 2) != (half == 0)) continue;
                uint32_t z[8];
                tmem_ld_nowait<8>(tl + VZ0 + VZW * s + ch * 8, z);
                tmem_wait_ld(z);
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    if (ch * 8 + e < KT) s_z[(ch * 8 + e) * kZP + m] = __uint_as_float(z[e]);
            }
            tc_fence_before();
            TCT(g, 8 + 6 * (gt >> 5) + 1, lane == 0);
            if (g + kSlots < nblk) build(s);           // block g + 3 into slot s, free: W(g) consumed, Z(g) read
            TCT(g, 3, gt == 0);
            TCT(g, 8 + 6 * (gt >> 5) + 2, lane == 0);
            TCP_SYNC(BAR_BG, kNBG);    // Z(g) is in shared memory; every thread is done with iteration g - 1
            TCT(g, 8 + 6 * (gt >> 5) + 3, lane == 0);
            if (i == 0 && n + 1 < ntl) request_u(n + 1);   // its buffer's last reader was tile n - 1
            // d(y, x) += sum_b Z[(y + a, x + b)][a K + b] over rows 2i, 2i + 1 (v row y + a):
            // thread gt takes column x and the rows r = rg (mod kNBG/64) of the block's
            // K + 1; the epilogue rows (r = 0, 1) are last written by their epilogue thread
            const int j0 = 2 * i;
            const bool r2_edge = R2 && (T.y0 - R < 0 || T.y0 + OH + R > H || T.x0 - R < 0 || T.x0 + OW + R > W);
            if (!R2 || !r2_edge) {
                constexpr int NRG = kNBG / 64;
#pragma unroll
                for (int k = 0; k < (K + NRG) / NRG; ++k) {    // output rows j0 - (K-1) .. j0 + 1
                    const int r = rg + NRG * k;
                    const int y = j0 - (K - 1) + r;
                    if (r > K || x >= OW || y < 0 || y >= OH) continue;
                    float *dp = s_d + (y % DR) * OW + x;
                    float d = *dp;
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj) {
                        const int ta = j0 + jj - y;
                        if (ta < 0 || ta >= K) continue;
                        const float *zp = s_z + (ta * K) * kZP + jj * 64 + x;
                        float S = 0.0f;
#pragma unroll
                        for (int tb = 0; tb < K; ++tb) S += zp[tb * kZP + tb];
                        d += S;
                    }
                    *dp = d;
                }
            } else if constexpr (R2) {
                // R2 tile at an image edge: d(q) = sum_t sum_{x in M(q)} Z[x + a_t][t] over
                // the mirror images M(q) of q (itself, across the nearest vertical and
                // horizontal edges, both; Z = 0 outside the image).  Per source row, in order:
                // row term of q then of its row mirror, each over q's and the column mirror's
                // columns (S l.57-65, the exact transpose)
                const auto S_cols = [&](int jj, int ta, int xc) {  // sum_b Z[(row jj, col xc + b)][ta K + b]
                    const float *zp = s_z + (ta * K) * kZP + jj * 64;
                    float S = 0.0f;
#pragma unroll
                    for (int tb = 0; tb < K; ++tb) {
                        const int c = xc + tb;
                        if ((unsigned)c < 64u) S += zp[tb * kZP + c];
                    }
                    return S;
                };
                for (int r = rg; r < K + 1; r += kNBG / 64) {
                    const int y = j0 - (K - 1) + r;
                    if (x >= OW || y < 0 || y >= OH) continue;
                    const int gy = T.y0 + y, gx = T.x0 + x;
                    const int gym = gy < R ? -1 - gy : (gy >= H - R ? 2 * H - 1 - gy : INT_MIN);
                    const int gxm = gx < R ? -1 - gx : (gx >= W - R ? 2 * W - 1 - gx : INT_MIN);
                    const int xm = gxm == INT_MIN ? 0 : gxm - T.x0;  // source col of tap b: xm + b
                    float *dp = s_d + (y % DR) * OW + x;
                    float d = *dp;
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj) {
                        const int ta = j0 + jj - y;
                        if (ta >= 0 && ta < K) {
                            d += S_cols(jj, ta, x);
                            if (gxm != INT_MIN) d += S_cols(jj, ta, xm);
                        }
                        if (gym != INT_MIN) {
                            const int ta2 = (T.y0 - R + j0 + jj) - gym + R;
                            if (ta2 >= 0 && ta2 < K) {
                                d += S_cols(jj, ta2, x);
                                if (gxm != INT_MIN) d += S_cols(jj, ta2, xm);
                            }
                        }
                    }
                    *dp = d;
                }
            }
            TCT(g, 8 + 6 * (gt >> 5) + 4, lane == 0);
            // epilogue: output row ye is complete (its last v row, ye + K - 1, is in this
            // block): ut = u - d, u+ = reaction(ut); the ring row is cleared for reuse
            if (ye >= 0 && x < OW) {
                float *dp = s_d + (ye % DR) * OW + x;
#ifdef TNRD_EXP_NOEPI
                if (epi && fv == -1.0f) {
#else
                if (epi) {
#endif
                    const float u = s_u0[(n & 1) * UF + lead_of(T.x0) + (ye + 2 * R) * UP + x + 2 * R];
                    const float ut = u - *dp;
                    const long long oi = oi_t + ye * a.out_ld;
                    a.u_out[oi] = reaction_step(a.reaction, u, ut, a.lambda, fv);
                    if (a.ut_out) a.ut_out[oi] = ut;
                }
                *dp = 0.0f;
            }
            TCT(g, 4, gt == 0);
            TCT(g, 8 + 6 * (gt >> 5) + 5, lane == 0);
            if (++i == nmb) { i = 0; if (++n < ntl) { T = tile_of(n); tile_bases(); } }
        }
    } else if (kRelay && warp == WMMA + kNMMA) {
        // ======================= relay: V_full(g) (an mbarrier the MMA commit arrives on)
        // becomes an arrival on the hardware barrier BAR_V + s the phi warps sleep in, so
        // 16 warps do not poll.  A slot's barrier is reused only after every phi warp has
        // left it: V(g + 3) needs A(g + 3), built after Z(g), i.e. after W_full(g).
        for (int g = 0; g < nblk; ++g) {
            const int s = g % kSlots;
            mbar_wait(bar_v + s, (g / kSlots) & 1);
            TCT(g, 5, lane == 0);
            tc_fence_after();
            tc_fence_before();
            if constexpr (kRelay == 3) {
#pragma unroll
                for (int q = 0; q < PG; ++q)
                    asm volatile("bar.arrive %0, %1;" ::"r"(BAR_V + PG * s + q), "n"(5 * 32) : "memory");
            } else if constexpr (kRelay == 2) {
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    asm volatile("bar.arrive %0, %1;" ::"r"(BAR_V + 4 * s + q), "n"((PG + 1) * 32) : "memory");
            } else {
                asm volatile("bar.arrive %0, %1;" ::"r"(BAR_V + s), "n"((4 * PG + 1) * 32) : "memory");
            }
        }
    } else if (kObs && warp == WMMA + kNMMA + (kRelay ? 1 : 0)) {
        for (int g = 0; g < nblk; ++g) {
            mbar_wait(bar_z + g % kSlots, (g / kSlots) & 1);
            TCT(g, 56, lane == 0);
        }
    } else if (TABLE || kMmaWarp || lane == 0) {
        // ======================= MMA issuer: one thread with the exact phi; the
        // converged warp with an elected lane for the tabulated phi, whose shorter phi
        // puts the MMA chain on the critical path
        const uint32_t bf_hi = smem_u32(s_bf), bf_lo = bf_hi + 4 * NK * KTP;
        const uint32_t ba_hi = smem_u32(s_ba), ba_lo = ba_hi + 4 * NZ * NK;
        constexpr uint32_t SBO_F = (KTP / 4) * 128, SBO_A = (NK / 4) * 128;
        constexpr uint32_t id_f = idesc_tf32(NK), id_a = idesc_tf32(NZ);
        const uint64_t df_hi = umma_desc(bf_hi, SBO_F), df_lo = umma_desc(bf_lo, SBO_F);
        const uint64_t da_hi = umma_desc(ba_hi, SBO_A), da_lo = umma_desc(ba_lo, SBO_A);
        const auto fwd = [&](int g) {  // V = A_lo B_hi + A_hi B_lo + A_hi B_hi (A_full(g) seen)
            const int s = g % kSlots;
            tc_fence_after();
            const uint32_t tA = tmem + SLOT * s, tV = tmem + VZ0 + VZW * s;
            if constexpr (TABLE || kMmaWarp) {
#pragma unroll
                for (int k = 0; k < KTP / 8; ++k) {   // K-chunk k: descriptor + 16 k (256 B)
                    mma_tf32_warp(tV, tA + KTP + 8 * k, df_hi + 16 * k, id_f, k > 0);
                    mma_tf32_warp(tV, tA + 8 * k, df_lo + 16 * k, id_f, 1);
                    mma_tf32_warp(tV, tA + 8 * k, df_hi + 16 * k, id_f, 1);
                }
                mma_commit_warp(bar_v + s);
            } else {
#pragma unroll
                for (int k = 0; k < KTP / 8; ++k) {
                    mma_tf32(tV, tA + KTP + 8 * k, umma_desc(bf_hi + 256 * k, SBO_F), id_f, k > 0);
                    mma_tf32(tV, tA + 8 * k, umma_desc(bf_lo + 256 * k, SBO_F), id_f, 1);
                    mma_tf32(tV, tA + 8 * k, umma_desc(bf_hi + 256 * k, SBO_F), id_f, 1);
                }
                mma_commit(bar_v + s);
            }
        };
        const auto adj = [&](int g) {  // Z = W_lo B_hi + W_hi B_lo + W_hi B_hi (W_full(g) seen)
            const int s = g % kSlots;
            tc_fence_after();
            const uint32_t tW = tmem + SLOT * s, tZ = tmem + VZ0 + VZW * s;
            if constexpr (TABLE || kMmaWarp) {
#pragma unroll
                for (int k = 0; k < NK / 8; ++k) {
                    mma_tf32_warp(tZ, tW + NK + 8 * k, da_hi + 16 * k, id_a, k > 0);
                    mma_tf32_warp(tZ, tW + 8 * k, da_lo + 16 * k, id_a, 1);
                    mma_tf32_warp(tZ, tW + 8 * k, da_hi + 16 * k, id_a, 1);
                }
                mma_commit_warp(bar_z + s);
            } else {
#pragma unroll
                for (int k = 0; k < NK / 8; ++k) {
                    mma_tf32(tZ, tW + NK + 8 * k, umma_desc(ba_hi + 256 * k, SBO_A), id_a, k > 0);
                    mma_tf32(tZ, tW + 8 * k, umma_desc(ba_lo + 256 * k, SBO_A), id_a, 1);
                    mma_tf32(tZ, tW + 8 * k, umma_desc(ba_hi + 256 * k, SBO_A), id_a, 1);
                }
                mma_commit(bar_z + s);
            }
        };
        // Issue F(g) once A_full(g) and Adj(g) once W_full(g) complete, whichever comes
        // first (F(g) also needs slot g % 3 free: A(g) is built only after Z(g - 3) was
        // read, which needed Adj(g - 3)).  Polling both keeps a late im2col block from
        // holding up the adjoint of a block whose w is ready, and vice versa.
        if constexpr (kNMMA == 2) {
            // two issuers (warps on different SM sub-partitions): F(g) after A_full(g),
            // Adj(g) after W_full(g); each commit tracks its own thread's MMAs
            if (warp == WMMA) {
                for (int g = 0; g < nblk; ++g) { mbar_wait(bar_a + g % kSlots, (g / kSlots) & 1); TCT(g, 7, lane == 0); fwd(g); }
            } else {
                for (int g = 0; g < nblk; ++g) { mbar_wait(bar_w + g % kSlots, (g / kSlots) & 1); TCT(g, 6, lane == 0); adj(g); }
            }
        } else {
            int gf = 0, ga = 0;
            while (ga < nblk) {
                bool did = false;
                if (gf < nblk && gf < ga + kSlots && mbar_test(bar_a + gf % kSlots, (gf / kSlots) & 1, TABLE || kMmaWarp)) {
                    fwd(gf++);
                    did = true;
                }
                if (ga < gf && mbar_test(bar_w + ga % kSlots, (ga / kSlots) & 1, TABLE || kMmaWarp)) {
                    adj(ga++);
                    did = true;
                }
                if (!did) __nanosleep(32);
            }
        }
    }
#ifdef TNRD_TC_PROF
    if (lane == 0 && p.prof) {
        p.prof[(blockIdx.x * 32 + warp) * 2] = tcp_wait;
        p.prof[(blockIdx.x * 32 + warp) * 2 + 1] = clock64() - tcp_t0;
    }
#endif
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols));
}

// u_in rows [avail_lo, avail_hi) as a (W, rows, B) tensor map with a (UP, UH, 1) box
template <int K, int NK>
bool encode_u_tiles(CUtensorMap *tm, const StageArgs &a, int B) {
    using G = TcGeo<K, NK>;
    EncodeTiled enc = encoder();
    const int rows = a.avail_hi - a.avail_lo, UH = a.tc_oh + 4 * G::R;
    if (!enc || rows < 1 || UH > 256) return false;
    const float *base = a.u_in.ptr + (long long)(a.avail_lo - a.u_in.row_base) * a.u_in.ld;
    const long long s2 = B > 1 ? a.u_in.img_stride : (long long)rows * a.u_in.ld;
    if (!aligned16(base) || a.u_in.ld % 4 != 0 || s2 % 4 != 0) return false;
    cuuint64_t dims[3] = {(cuuint64_t)a.W, (cuuint64_t)rows, (cuuint64_t)B};
    cuuint64_t strides[2] = {(cuuint64_t)a.u_in.ld * 4, (cuuint64_t)s2 * 4};
    cuuint32_t boxd[3] = {(cuuint32_t)G::UP, (cuuint32_t)UH, 1}, es[3] = {1, 1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(base), dims, strides, boxd, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct DevInfo { int optin = 0, sms = 0; };
DevInfo dev_info() {
    int dev = 0;
    cudaGetDevice(&dev);
    static DevInfo cache[64];  // per device, filled on first use
    DevInfo d = dev < 64 ? cache[dev] : DevInfo{};
    if (d.sms == 0) {
        cudaDeviceGetAttribute(&d.optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
        if (dev < 64) cache[dev] = d;
    }
    return d;
}

template <int K, int NK>
cudaError_t launch_tc(StageArgs &a, int B, cudaStream_t s) {
    using G = TcGeo<K, NK>;
    // exact phi with the round-to-nearest split only for the training gradient's tape
    if (a.tc_rn && a.mode == MODE_TABLE) return cudaErrorInvalidValue;
    auto kern = a.tc_rn ? (a.boundary == 1 ? tc_stage_kernel<K, NK, false, true, true>
                                           : tc_stage_kernel<K, NK, false, false, true>)
              : a.boundary == 1 ? (a.mode == MODE_TABLE ? tc_stage_kernel<K, NK, true, true, false>
                                                        : tc_stage_kernel<K, NK, false, true, false>)
                                : (a.mode == MODE_TABLE ? tc_stage_kernel<K, NK, true, false, false>
                                                        : tc_stage_kernel<K, NK, false, false, false>);
    if (a.tc_oh <= 0 || a.tc_oh % 2 != 0) return cudaErrorInvalidValue;
    // the u tile of tile n + 1 is requested when tile n starts: a tile needs >= 4 M-blocks
    a.tc_oh = std::max(a.tc_oh, 8 - 2 * G::R);
    const DevInfo di = dev_info();
    const int zb = a.mode == MODE_TABLE ? 1 : 2;      // Z buffers (ZB of the kernel)
    size_t smem = sizeof(float) * (size_t)tc_smem_floats<K, NK>(a.tc_oh, a.tc_par_floats, zb);
    while (smem > (size_t)di.optin && a.tc_oh > 8) {  // fewer rows per tile until it fits
        a.tc_oh -= 8;
        smem = sizeof(float) * (size_t)tc_smem_floats<K, NK>(a.tc_oh, a.tc_par_floats, zb);
    }
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    a.tiles_x = (a.W + G::OW - 1) / G::OW;
    a.tiles_y = (a.y_end - a.y_begin + a.tc_oh - 1) / a.tc_oh;
    const long long n = (long long)B * a.tiles_x * a.tiles_y;
    if (n > INT_MAX / 128) return cudaErrorInvalidValue;
    a.n_tiles = (int)n;
    if (n == 0) return cudaSuccess;
    TcArgs p;   // kernel parameter (copied at launch)
    std::memset(&p, 0, sizeof p);
    p.a = a;
    p.use_tma = encode_u_tiles<K, NK>(&p.tm_u, a, B) ? 1 : 0;
    const int grid = (int)std::min<long long>(n, di.sms > 0 ? di.sms : 148);
#ifdef TNRD_TC_PROF
    // per warp: mean wait fraction over the CTAs (stderr), one line per launch
    static unsigned long long *prof = nullptr;
    if (!prof) cudaMalloc(&prof, sizeof(unsigned long long) * 64 * 1024);
    cudaMemsetAsync(prof, 0, sizeof(unsigned long long) * 64 * 1024, s);
    p.prof = prof;
    kern<<<grid, kTNT, smem, s>>>(p);
    std::vector<unsigned long long> hp(64 * (size_t)grid);
    cudaMemcpyAsync(hp.data(), prof, sizeof(unsigned long long) * hp.size(), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    fprintf(stderr, "TCPROF wait%% per warp:");
    for (int w = 0; w < kTNT / 32; ++w) {
        double wt = 0, tt = 0;
        for (int c = 0; c < grid; ++c) { wt += (double)hp[(c * 32 + w) * 2]; tt += (double)hp[(c * 32 + w) * 2 + 1]; }
        fprintf(stderr, " %.1f", tt > 0 ? 100.0 * wt / tt : 0.0);
    }
    fprintf(stderr, "\n");
#ifdef TNRD_TC_TRACE
    {
        std::vector<unsigned long long> tr(64 * 256);
        cudaMemcpy(tr.data(), prof + 16384, sizeof(unsigned long long) * tr.size(), cudaMemcpyDeviceToHost);
        if (FILE *fh = fopen("gpurun_out/tc_trace.bin", "wb")) { fwrite(tr.data(), sizeof(unsigned long long), tr.size(), fh); fclose(fh); }
    }
#endif
    return cudaGetLastError();
#else
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kTNT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
#endif
}


// ---------------------------------------------------------------------------
// Tensor-core adjoint bank for the training gradient (tnrd_grad.cu, P Eq.15):
// gn -= sum_f K_f^T b_f, K_f the symmetric-boundary convolution of the forward
// bank, as one GEMM per M-block (Z[q][t] = sum_f b_f(q) k_f[t], 3xTF32) and the
// exact-transpose gather of the stage kernel's R2 path (b = 0 outside the image,
// mirror-image terms at image edges).  512 threads (lane m of each warpgroup loads
// and splits NK/4 of the maps, one block ahead); two TMEM slots, so block i's MMA
// overlaps the gather of block i - 1.
struct TcAdjArgs {
    const float *b;    // [NK][B*H*W]
    const float *ba;   // ba_hi [NZ x NK], then ba_lo
    float *gn;         // [B][H][W], updated in place
    int B, H, W, oh, tiles_x, tiles_y;
};

template <int K, int NK>
__global__ void __launch_bounds__(512, 1) tc_adjoint_kernel(const __grid_constant__ TcAdjArgs a) {
    constexpr int R = K / 2, KT = K * K, NZ = tc_nz(K), OW = kTcVW - 2 * R, NFQ = NK / 4;
    extern __shared__ __align__(1024) float4 smem4[];
    float *s_ba = reinterpret_cast<float *>(smem4);          // [2][NZ x NK]
    const int OH = a.oh, VH = OH + 2 * R;
    float *s_z = s_ba + 2 * NZ * NK;                          // [KT][kZP]
    float *s_d = s_z + KT * kZP;                              // [OH][OW]
    uint64_t *mbar = reinterpret_cast<uint64_t *>(s_d + round4(OH * OW));   // [2]
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(mbar + 2);
    const int tid = threadIdx.x, warp = tid >> 5, wg = tid >> 7, m = tid & 127;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const int H = a.H, W = a.W;
    const long long n = (long long)a.B * H * W;
    const int per_img = a.tiles_x * a.tiles_y;
    const int bi = blockIdx.x / per_img, rem = blockIdx.x - bi * per_img;
    const int ty = rem / a.tiles_x, x0 = (rem - ty * a.tiles_x) * OW, y0 = ty * OH;
    for (int j = tid; j < (2 * NZ * NK) / 4; j += 512) smem4[j] = __ldg(reinterpret_cast<const float4 *>(a.ba) + j);
    for (int j = tid; j < OH * OW; j += 512) s_d[j] = 0.0f;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mbar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mbar + 1)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // two slots: W (hi, lo) at slot * 2 NK, Z at 256 + slot * NZ; block i's MMA runs
    // while block i - 1 is gathered, and block i + 1's maps are already in flight
    const uint32_t tmem = *s_tmem, tl = tmem + lane_off;
    const uint32_t ba_hi = smem_u32(s_ba), ba_lo = ba_hi + 4 * NZ * NK;
    constexpr uint32_t SBO_A = (NK / 4) * 128;
    constexpr uint32_t id_a = idesc_tf32(NZ);
    static_assert(256 + 2 * NZ <= 512 && 4 * NK <= 256, "TMEM plan");
    const float *bb = a.b + (long long)bi * H * W;
    const int nmb = VH / 2;
    float wv[NFQ];
    const auto load_w = [&](int i) {   // the b maps of pixel m of block i, 0 outside the image
        const int gy = y0 - R + 2 * i + (m >> 6), gx = x0 - R + (m & 63);
        const bool in = (unsigned)gy < (unsigned)H && (unsigned)gx < (unsigned)W;
        const long long off = (long long)gy * W + gx;
#pragma unroll
        for (int e = 0; e < NFQ; ++e) wv[e] = in ? __ldg(bb + (long long)(wg * NFQ + e) * n + off) : 0.0f;
    };
    load_w(0);
    for (int i = 0; i <= nmb; ++i) {
        const int sl = i & 1;
        if (i < nmb) {
            uint32_t wh[NFQ], wl[NFQ];
#pragma unroll
            for (int e = 0; e < NFQ; ++e) {
                const float xh = tf32_hi_rn(wv[e]);
                wh[e] = __float_as_uint(xh);
                wl[e] = __float_as_uint(wv[e] - xh);
            }
            tmem_st<NFQ>(tl + sl * 2 * NK + wg * NFQ, wh);
            tmem_st<NFQ>(tl + sl * 2 * NK + NK + wg * NFQ, wl);
            tc_wait_st();
            if (i + 1 < nmb) load_w(i + 1);
        }
        tc_fence_before();
        __syncthreads();   // W(i) written; the gather of block i - 2 is done with s_z
        if (i < nmb && warp == 0) {
            tc_fence_after();
            const uint32_t tW = tmem + sl * 2 * NK, tZ = tmem + 256 + sl * NZ;
#pragma unroll
            for (int k = 0; k < NK / 8; ++k) {
                mma_tf32_warp(tZ, tW + NK + 8 * k, umma_desc(ba_hi + 256 * k, SBO_A), id_a, k > 0);
                mma_tf32_warp(tZ, tW + 8 * k, umma_desc(ba_lo + 256 * k, SBO_A), id_a, 1);
                mma_tf32_warp(tZ, tW + 8 * k, umma_desc(ba_hi + 256 * k, SBO_A), id_a, 1);
            }
            mma_commit_warp(mbar + sl);
        }
        if (i == 0) continue;
        const int ib = i - 1, sp = ib & 1;
        mbar_wait(mbar + sp, (ib >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int ch = 0; ch < NZ / 8; ++ch) {
            if (ch % 4 != wg || ch * 8 >= KT) continue;
            uint32_t z[8];
            tmem_ld_nowait<8>(tl + 256 + sp * NZ + ch * 8, z);
            tmem_wait_ld(z);
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (ch * 8 + e < KT) s_z[(ch * 8 + e) * kZP + m] = __uint_as_float(z[e]);
        }
        tc_fence_before();
        __syncthreads();
        // d(q) += sum_t sum_{x in M(q)} Z[x + a_t][t] over block ib's rows (mirror
        // images M(q): q, across the nearest vertical / horizontal edge, both)
        const int j0 = 2 * ib;
        const auto S_cols = [&](int jj, int ta, int xc) {
            const float *zp = s_z + (ta * K) * kZP + jj * 64;
            float S = 0.0f;
#pragma unroll
            for (int tb = 0; tb < K; ++tb) {
                const int c = xc + tb;
                if ((unsigned)c < 64u) S += zp[tb * kZP + c];
            }
            return S;
        };
        for (int it = tid; it < (K + 1) * 64; it += 512) {
            const int y = j0 - (K - 1) + it / 64, x = it & 63;
            if (x >= OW || y < 0 || y >= OH) continue;
            const int gy = y0 + y, gx = x0 + x;
            const int gym = gy < R ? -1 - gy : (gy >= H - R ? 2 * H - 1 - gy : INT_MIN);
            const int gxm = gx < R ? -1 - gx : (gx >= W - R ? 2 * W - 1 - gx : INT_MIN);
            const int xm = gxm == INT_MIN ? 0 : gxm - x0;
            float d = s_d[y * OW + x];
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
                const int ta = j0 + jj - y;
                if (ta >= 0 && ta < K) {
                    d += S_cols(jj, ta, x);
                    if (gxm != INT_MIN) d += S_cols(jj, ta, xm);
                }
                if (gym != INT_MIN) {
                    const int ta2 = (y0 - R + j0 + jj) - gym + R;
                    if (ta2 >= 0 && ta2 < K) {
                        d += S_cols(jj, ta2, x);
                        if (gxm != INT_MIN) d += S_cols(jj, ta2, xm);
                    }
                }
            }
            s_d[y * OW + x] = d;
        }
    }
    __syncthreads();
    float *gb = a.gn + (long long)bi * H * W;
    for (int it = tid; it < OH * OW; it += 512) {
        const int y = it / OW, x = it - y * OW;
        if (y0 + y < H && x0 + x < W) gb[(long long)(y0 + y) * W + x0 + x] -= s_d[it];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int K, int NK>
cudaError_t launch_tc_adj(const float *b, const float *ba, float *gn, int B, int H, int W, int oh, cudaStream_t s) {
    constexpr int R = K / 2, OW = kTcVW - 2 * R;
#ifdef TNRD_ADJ_OH
    oh = TNRD_ADJ_OH;
#endif
    TcAdjArgs a{b, ba, gn, B, H, W, oh, (W + OW - 1) / OW, (H + oh - 1) / oh};
    const size_t smem = sizeof(float) * (2 * (size_t)tc_nz(K) * NK + (size_t)K * K * kZP + round4(oh * OW) + 8);
    cudaError_t e = cudaFuncSetAttribute(tc_adjoint_kernel<K, NK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const long long nt = (long long)B * a.tiles_x * a.tiles_y;
    if (nt > INT_MAX) return cudaErrorInvalidValue;
    if (nt > 0) tc_adjoint_kernel<K, NK><<<(unsigned)nt, 512, smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_tc_adjoint(int ksize, int Nk, const float *b, const float *ba, float *gn, int B, int H, int W,
                              int oh, cudaStream_t s) {
    if (oh <= 0 || oh % 2) return cudaErrorInvalidValue;
    if (ksize == 3 && Nk == 8) return launch_tc_adj<3, 8>(b, ba, gn, B, H, W, oh, s);
    if (ksize == 5 && Nk == 24) return launch_tc_adj<5, 24>(b, ba, gn, B, H, W, oh, s);
    if (ksize == 7 && Nk == 48) return launch_tc_adj<7, 48>(b, ba, gn, B, H, W, oh, s);
    return cudaErrorInvalidValue;
}

namespace {

// ---------------------------------------------------------------------------
// Tensor-core forward bank for the training gradient (tnrd_grad.cu): out[f][p] =
// (k_f * E(in))(p) for all filters, the stage kernel's 3xTF32 implicit GEMM on
// output pixels (M-block = two 64-pixel output rows; no halo), written to HBM in
// filter-major maps.  512 threads, two TMEM slots: block i's MMA overlaps the
// build of block i + 1 and the read-back of block i - 1.
struct TcFwdArgs {
    const float *in;   // [B][H][W]
    const float *bf;   // bf_hi [NK x KTP], then bf_lo
    float *out;        // [NK][B*H*W]
    int B, H, W, tiles_x, tiles_y;
};

#ifndef TNRD_FWD_OH
#define TNRD_FWD_OH 32
#endif
constexpr int kFwdOH = TNRD_FWD_OH;   // output rows per tile of the gradient's forward bank

template <int K, int NK>
__global__ void __launch_bounds__(512, 1) tc_fwdbank_kernel(const __grid_constant__ TcFwdArgs a) {
    constexpr int R = K / 2, KT = K * K, KTP = tc_ktp(K), UW = kTcVW + 2 * R, UH = kFwdOH + 2 * R, NFQ = NK / 4;
    extern __shared__ __align__(1024) float4 smem4[];
    float *s_bf = reinterpret_cast<float *>(smem4);           // [2][NK x KTP]
    float *s_u = s_bf + 2 * NK * KTP;                         // [UH][UW]
    uint64_t *mbar = reinterpret_cast<uint64_t *>(s_u + round4(UH * UW));   // [2]
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(mbar + 2);
    const int tid = threadIdx.x, warp = tid >> 5, wg = tid >> 7, m = tid & 127;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const int H = a.H, W = a.W;
    const long long n = (long long)a.B * H * W;
    const int per_img = a.tiles_x * a.tiles_y;
    const int bi = blockIdx.x / per_img, rem = blockIdx.x - bi * per_img;
    const int ty = rem / a.tiles_x, x0 = (rem - ty * a.tiles_x) * kTcVW, y0 = ty * kFwdOH;
    for (int j = tid; j < (2 * NK * KTP) / 4; j += 512) smem4[j] = __ldg(reinterpret_cast<const float4 *>(a.bf) + j);
    const float *ib = a.in + (long long)bi * H * W;
    for (int j = tid; j < UH * UW; j += 512) {
        const int r = j / UW, c = j - r * UW;
        s_u[j] = __ldg(ib + (long long)reflect(y0 - R + r, H) * W + reflect(x0 - R + c, W));
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mbar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mbar + 1)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // two slots: A (hi, lo) at slot * 2 KTP, V at 4 KTP + slot * NK; block i's MMA
    // runs while block i + 1 is built and block i - 1 is read back
    const uint32_t tmem = *s_tmem, tl = tmem + lane_off;
    const uint32_t bf_hi = smem_u32(s_bf), bf_lo = bf_hi + 4 * NK * KTP;
    constexpr uint32_t SBO_F = (KTP / 4) * 128;
    constexpr uint32_t id_f = idesc_tf32(NK);
    constexpr int NB = kFwdOH / 2;
    for (int i = 0; i <= NB; ++i) {
        const int sl = i & 1;
        if (i < NB) {   // im2col row (hi, lo) of block i: tap (ta, tb) reads u(y + R - ta, x + R - tb), tile offset R
            const int y = 2 * i + (m >> 6), x = m & 63;
            const float *up = s_u + (y + 2 * R) * UW + x + 2 * R;
#pragma unroll
            for (int ch = 0; ch < KTP / 8; ++ch) {
                if (ch % 4 != wg) continue;
                uint32_t hv[8], lv[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const int t = ch * 8 + e;
                    float v = 0.0f;
                    if (t < KT) v = up[-(t / K) * UW - (t % K)];
                    const float vh = tf32_hi_rn(v);
                    hv[e] = __float_as_uint(vh);
                    lv[e] = __float_as_uint(v - vh);
                }
                tmem_st8(tl + sl * 2 * KTP + ch * 8, hv);
                tmem_st8(tl + sl * 2 * KTP + KTP + ch * 8, lv);
            }
            tc_wait_st();
        }
        tc_fence_before();
        __syncthreads();   // A(i) written; every thread has read V(i - 2)
        if (i < NB && warp == 0) {
            tc_fence_after();
            const uint32_t tA = tmem + sl * 2 * KTP, tV = tmem + 4 * KTP + sl * NK;
#pragma unroll
            for (int k = 0; k < KTP / 8; ++k) {
                mma_tf32_warp(tV, tA + KTP + 8 * k, umma_desc(bf_hi + 256 * k, SBO_F), id_f, k > 0);
                mma_tf32_warp(tV, tA + 8 * k, umma_desc(bf_lo + 256 * k, SBO_F), id_f, 1);
                mma_tf32_warp(tV, tA + 8 * k, umma_desc(bf_hi + 256 * k, SBO_F), id_f, 1);
            }
            mma_commit_warp(mbar + sl);
        }
        if (i >= 1) {   // V(i - 1) -> out maps (this warpgroup's filters), lanes = consecutive pixels
            const int ip = i - 1, sp = ip & 1;
            mbar_wait(mbar + sp, (ip >> 1) & 1);
            tc_fence_after();
            uint32_t vr[NFQ];
            tmem_ld_nowait<NFQ>(tl + 4 * KTP + sp * NK + wg * NFQ, vr);
            tmem_wait_ld(vr);
            const int gy = y0 + 2 * ip + (m >> 6), gx = x0 + (m & 63);
            if (gy < H && gx < W) {
                float *op = a.out + (long long)bi * H * W + (long long)gy * W + gx;
#pragma unroll
                for (int e = 0; e < NFQ; ++e) op[(long long)(wg * NFQ + e) * n] = __uint_as_float(vr[e]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int K, int NK>
cudaError_t launch_tc_fwd(const float *in, const float *bf, float *out, int B, int H, int W, cudaStream_t s) {
    constexpr int R = K / 2;
    TcFwdArgs a{in, bf, out, B, H, W, (W + kTcVW - 1) / kTcVW, (H + kFwdOH - 1) / kFwdOH};
    const size_t smem = sizeof(float) * (2 * (size_t)NK * tc_ktp(K) + round4((kFwdOH + 2 * R) * (kTcVW + 2 * R)) + 8);
    cudaError_t e = cudaFuncSetAttribute(tc_fwdbank_kernel<K, NK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const long long nt = (long long)B * a.tiles_x * a.tiles_y;
    if (nt > INT_MAX) return cudaErrorInvalidValue;
    if (nt > 0) tc_fwdbank_kernel<K, NK><<<(unsigned)nt, 512, smem, s>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Tensor-core filter gradient (P Eq.18-20, the k-part of dL/dθ): for every tap t =
// (ta, tb) of the k x k support, displacement d_t = (ta - r, tb - r), and filter f
//   inner[f][t] = sum_p b_f(p) E(u)(p - d_t)
//   outer[f][t] = sum_p e(p) w_f(mirror(p - d_t))                                    (R1)
//               = sum_q w_f(q) Ẽ_t(q),  Ẽ_t(q) = sum_{p in Ω: mirror(p - d_t) = q} e(p)
//   outer[f][t] = sum_p w_f(p) E(e)(p - d_t)                                         (R2)
// — the sums kgrad_pair_kernel (tnrd_grad.cu) forms pixel by pixel — as one GEMM
// over pixels: D[t][f] = sum_p A[t][p] Bm[f][p], M = 128 rows = taps (rows >= k^2
// zero), N = N_k filters, K = pixels.  A (the tap-shifted images, one per tap) is
// written into TMEM by the thread owning lane t; Bm (the b and w maps) is staged in
// shared memory in the K-major core-matrix layout; 3xTF32 as in the stage kernel.
// Two accumulators (inner, outer) stay in TMEM for the CTA's whole pixel range;
// each CTA writes its D once to `partial` in the layout reduce_f_kernel sums.
// Work: 32-pixel chunks (half a tile row of a 64 x kKgTH tile), kKgBuf chunks in
// flight in TMEM and shared memory between 16 builder warps and one MMA warp
// (mbarriers full / empty); b and w arrive through a cp.async ring kKgS - 1 chunks
// ahead; one CTA per SM, tiles grid-strided over the CTAs.  TNRD_KG_EXP_* are
// timing experiments (wrong results), never set in the product build.
struct TcKgArgs {
    const float *u, *e;       // [B][H][W]
    const float *b, *w;       // [NK][B*H*W]
    float *partial;           // [NK][nblk][2 k^2]
    int boundary, B, H, W, tiles_x, tiles_y;
};

#ifndef TNRD_KG_TH
#define TNRD_KG_TH 4
#endif
constexpr int kKgTH = TNRD_KG_TH;     // tile rows
#ifndef TNRD_KG_S
#define TNRD_KG_S 4
#endif
constexpr int kKgS = TNRD_KG_S;      // Bm prefetch depth (chunks in flight, cp.async)
constexpr int kKgBuf = 3;    // chunks in TMEM / shared memory between the builders and the MMA warp
constexpr int kKgBuilders = 512;              // 16 builder warps
constexpr int kKgThreads = kKgBuilders + 32;  // + the MMA warp

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, int bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void *src, int bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int K, int NK>
__global__ void __launch_bounds__(kKgThreads, 1) tc_kgrad_kernel(const __grid_constant__ TcKgArgs a) {
    constexpr int R = K / 2, KT = K * K, UW = kTcVW + 2 * R + 1, UH = kKgTH + 2 * R, UT = round4(UH * UW);
    constexpr int QA = (KT + 31) / 32;          // TMEM lane quarters holding taps
    constexpr int BMF = NK * 32;                // floats of one (map, hi|lo) Bm block
    constexpr uint32_t SBO = (32 / 4) * 128;    // 8-filter groups, 32 pixels of K
    constexpr uint32_t id = idesc_tf32(NK);
    constexpr uint32_t kDin = kKgBuf * 128, kDout = kDin + 64;   // TMEM columns of the accumulators
    static_assert(NK % 8 == 0 && NK <= 64 && kDout + NK <= 512, "N_k");
    extern __shared__ __align__(1024) float4 smem4[];
    float *s_bm = reinterpret_cast<float *>(smem4);   // [kKgBuf][b_hi, b_lo, w_hi, w_lo][BMF]
    float *s_u = s_bm + kKgBuf * 4 * BMF;             // [2 tiles][UH][UW], E(u)
    float *s_e = s_u + 2 * UT;                        // [2 tiles][UH][UW], E(e) (R1: raw e where used)
    float *s_st = s_e + 2 * UT;                       // [kKgS][2 maps][NK][32] raw b, w (prefetch ring)
    uint64_t *full = reinterpret_cast<uint64_t *>(s_st + kKgS * 2 * BMF);   // [kKgBuf] builders -> MMA
    uint64_t *empty = full + kKgBuf;                                        // [kKgBuf] MMA -> builders
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(empty + kKgBuf);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, q = warp & 3;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const int H = a.H, W = a.W;
    const long long n = (long long)a.B * H * W;
    const int per_img = a.tiles_x * a.tiles_y, ntiles = a.B * per_img;
    const int nch = 2 * kKgTH * ((ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1);   // this CTA's chunks
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < kKgBuf; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(full + i)), "r"(kKgBuilders / 32));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(empty + i)));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *s_tmem, tl = tmem + lane_off;
    if (warp == kKgBuilders / 32) {
        // MMA warp: chunk c in buffer c % kKgBuf once its 16 builder warps arrived
        for (int c = 0; c < nch; ++c) {
            const int bb = c % kKgBuf;
            mbar_wait(full + bb, (c / kKgBuf) & 1);
            tc_fence_after();
            const uint32_t ab = tmem + bb * 128, sb = smem_u32(s_bm + bb * 4 * BMF);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
#ifdef TNRD_KG_EXP_NOMMA
                if (c >= 0) break;
#endif
                const uint32_t ko = 256 * k;
                mma_tf32_warp(tmem + kDin, ab + 32 + 8 * k, umma_desc(sb + ko, SBO), id, c > 0 || k > 0);
                mma_tf32_warp(tmem + kDin, ab + 8 * k, umma_desc(sb + 4 * BMF + ko, SBO), id, 1);
                mma_tf32_warp(tmem + kDin, ab + 8 * k, umma_desc(sb + ko, SBO), id, 1);
                mma_tf32_warp(tmem + kDout, ab + 96 + 8 * k, umma_desc(sb + 8 * BMF + ko, SBO), id, c > 0 || k > 0);
                mma_tf32_warp(tmem + kDout, ab + 64 + 8 * k, umma_desc(sb + 12 * BMF + ko, SBO), id, 1);
                mma_tf32_warp(tmem + kDout, ab + 64 + 8 * k, umma_desc(sb + 8 * BMF + ko, SBO), id, 1);
            }
            mma_commit_warp(empty + bb);
        }
    } else {
        // A rows >= QA*32 (lane quarters without taps) stay zero: write them once
        if (q >= QA) {
            const uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (int c = (warp >> 2) * 8; c < kKgBuf * 128; c += 32) tmem_st8(tl + c, z);
            tc_wait_st();
        }
        const int t = q * 32 + lane;                     // this thread's tap (A builders)
        const int ta = t / K, tb = t - (t / K) * K;
        const int sub = warp >> 2;                       // A builders: pixels 8 sub .. 8 sub + 7 of a chunk
        // Bm builders (lane quarters >= QA): float4 slots j = bt, bt + nbt, ... of a
        // chunk's 2 x NK x 32 values, prefetched kKgS - 1 chunks ahead into their own
        // ring slots with cp.async (zero-filled outside the image)
        const int nbt = kKgBuilders - QA * 128;
        const int bt = ((warp >> 2) * (4 - QA) + (q - QA)) * 32 + lane;
        // this thread's float4 slots j = bt + r nbt (r < NJ): per slot the map /
        // filter offset in global memory, the pixel offset 4 kq within the chunk and
        // the element offset in the canonical Bm block (all chunk-invariant)
        constexpr int NJ = (2 * NK * 8 + (kKgBuilders - QA * 128) - 1) / (kKgBuilders - QA * 128);
        long long goff[NJ];
        int kq4[NJ], soff[NJ];
#pragma unroll
        for (int r = 0; r < NJ; ++r) {
            const int j = bt + r * nbt;
            const int fl = j & 7, kq = (j >> 3) & 7, fg = (j >> 6) % (NK / 8), map = j / (8 * NK);
            goff[r] = (long long)(fg * 8 + fl) * n + (map ? (a.w - a.b) : 0);
            kq4[r] = 4 * kq;
            soff[r] = 2 * map * BMF + (fg * 8 + kq) * 32 + fl * 4;
        }
        // 16-byte copies need every chunk row segment 16-byte aligned
        const bool al16 = (W % 4) == 0 && (n % 4) == 0 && ((reinterpret_cast<uintptr_t>(a.b) | reinterpret_cast<uintptr_t>(a.w)) & 15) == 0 &&
                          ((a.w - a.b) % 4) == 0;
        auto prefetch = [&](int cc) {
            if (cc < nch) {
                const int tile = blockIdx.x + (cc / (2 * kKgTH)) * gridDim.x, chh = cc % (2 * kKgTH);
                const int bi = tile / per_img, rem = tile - bi * per_img;
                const int ty = rem / a.tiles_x, x0 = (rem - ty * a.tiles_x) * kTcVW;
                const int gy = ty * kKgTH + (chh >> 1), xb = x0 + (chh & 1) * 32;
                const float *pb = a.b + (long long)bi * H * W + (long long)gy * W + xb;
                const int wrem = gy < H ? W - xb : 0;          // valid pixels from xb on
                const uint32_t st = smem_u32(s_st + (cc % kKgS) * 2 * BMF);
#pragma unroll
                for (int r = 0; r < NJ; ++r) {
                    if (r < NJ - 1 || bt + r * nbt < 2 * NK * 8) {
                        const int valid = min(max(wrem - kq4[r], 0), 4);
                        const float *src = valid > 0 ? pb + goff[r] + kq4[r] : a.b;
                        const uint32_t dst = st + 16 * (bt + r * nbt);
                        if (al16) {
                            cp_async16(dst, src, 4 * valid);
                        } else {
#pragma unroll
                            for (int e4 = 0; e4 < 4; ++e4)
                                cp_async4(dst + 4 * e4, e4 < valid ? src + e4 : a.b, e4 < valid ? 4 : 0);
                        }
                    }
                }
            }
            cp_async_commit();
        };
        if (q >= QA)
            for (int cc = 0; cc < kKgS - 1; ++cc) prefetch(cc);
        int chunk = 0, it = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const int bi = tile / per_img, rem = tile - bi * per_img;
            const int ty = rem / a.tiles_x, x0 = (rem - ty * a.tiles_x) * kTcVW, y0 = ty * kKgTH;
            const float *ub = a.u + (long long)bi * H * W, *eb = a.e + (long long)bi * H * W;
            // tiles alternate between two u / e buffers: the one written here was last
            // read in tile it - 2, which every builder finished before the barrier of it - 1
            float *tu = s_u + (it & 1) * UT, *te = s_e + (it & 1) * UT;
            for (int j = tid; j < UH * (UW - 1); j += kKgBuilders) {
                const int r = j / (UW - 1), c = j - r * (UW - 1);
                const long long o = (long long)reflect(y0 - R + r, H) * W + reflect(x0 - R + c, W);
                tu[r * UW + c] = __ldg(ub + o);
                te[r * UW + c] = __ldg(eb + o);
            }
            named_sync(1, kKgBuilders);
            for (int ch = 0; ch < 2 * kKgTH; ++ch, ++chunk) {
                const int bb = chunk % kKgBuf, yr = ch >> 1, xc0 = (ch & 1) * 32;
                if (chunk >= kKgBuf) mbar_wait(empty + bb, (chunk / kKgBuf - 1) & 1);   // MMAs of chunk - kKgBuf done
                tc_fence_after();
                const int gy = y0 + yr;
#ifdef TNRD_KG_EXP_NOA
                if (q < QA) {
                } else
#endif
                if (q < QA) {   // A: lane t = tap t, 8 pixels per thread
                    uint32_t ih[8], il[8], oh[8], ol[8];
                    const int xc = xc0 + 8 * sub;
                    const float *pu = tu + (yr + 2 * R - ta) * UW + xc + 2 * R - tb;
#ifdef TNRD_KG_EXP_NOEDGE
                    const bool r1edge = false;
#else
                    const bool r1edge = a.boundary == 0 &&
                                        (gy < R || gy >= H - R || x0 + xc < R || x0 + xc + 7 >= W - R);
#endif
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        float vi = 0.0f, vo = 0.0f;
                        if (t < KT) {
                            vi = pu[i];
                            if (a.boundary == 1) {
                                vo = te[(yr + 2 * R - ta) * UW + xc + i + 2 * R - tb];
                            } else {   // interior value; the edge pixels are redone below
                                vo = te[(yr + ta) * UW + xc + i + tb];
                            }
                        }
                        const float hi_i = tf32_hi_rn(vi), hi_o = tf32_hi_rn(vo);
                        ih[i] = __float_as_uint(hi_i); il[i] = __float_as_uint(vi - hi_i);
                        oh[i] = __float_as_uint(hi_o); ol[i] = __float_as_uint(vo - hi_o);
                    }
                    if (r1edge && t < KT) {   // Ẽ_t(q): every in-image preimage p of q (warp-uniform branch)
                        // the mirror is separable: p ranges over (rows py with
                        // reflect(py - dy) = qy) x (columns px with reflect(px - dx) = qx),
                        // at most 2 x 2 pixels, all inside this tile's halo (raw e there)
                        const int dy = ta - R, dx = tb - R, qy = gy;
                        int ro[3];
#pragma unroll
                        for (int iy = 0; iy < 3; ++iy) {
                            const int py = iy == 0 ? qy + dy : (iy == 1 ? dy - 1 - qy : 2 * H - 1 - qy + dy);
                            const bool ok = qy < H && py >= 0 && py < H && reflect(py - dy, H) == qy &&
                                            (iy == 0 || py != qy + dy);
                            ro[iy] = ok ? (py - y0 + R) * UW : -1;
                        }
                        const bool rowedge = gy < R || gy >= H - R;
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const int qx = x0 + xc + i;
                            if (!rowedge && qx >= R && qx < W - R) continue;   // interior pixel (uniform)
                            float sum = 0.0f;
#pragma unroll
                            for (int ix = 0; ix < 3; ++ix) {
                                const int px = ix == 0 ? qx + dx : (ix == 1 ? dx - 1 - qx : 2 * W - 1 - qx + dx);
                                const bool ok = qx < W && px >= 0 && px < W && reflect(px - dx, W) == qx &&
                                                (ix == 0 || px != qx + dx);
                                if (ok) {
                                    const int co = px - x0 + R;
#pragma unroll
                                    for (int iy = 0; iy < 3; ++iy)
                                        if (ro[iy] >= 0) sum += te[ro[iy] + co];
                                }
                            }
                            const float hs = tf32_hi_rn(sum);
                            oh[i] = __float_as_uint(hs); ol[i] = __float_as_uint(sum - hs);
                        }
                    }
                    const uint32_t base = tl + bb * 128 + 8 * sub;
                    tmem_st8(base, ih);
                    tmem_st8(base + 32, il);
                    tmem_st8(base + 64, oh);
                    tmem_st8(base + 96, ol);
                    tc_wait_st();
                    tc_fence_before();
                } else {        // Bm: b and w of this chunk's 32 pixels, float4 per (map, filter, 4 pixels)
#ifdef TNRD_KG_EXP_NOB
                    if (chunk >= 0) { __syncwarp(); if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(full + bb)) : "memory"); continue; }
#endif
                    prefetch(chunk + kKgS - 1);
                    cp_async_wait<kKgS - 1>();   // this thread's copies of this chunk have landed
                    float *sbm = s_bm + bb * 4 * BMF;
                    const float *st = s_st + (chunk % kKgS) * 2 * BMF;
#pragma unroll
                    for (int r = 0; r < NJ; ++r) {
                        if (r < NJ - 1 || bt + r * nbt < 2 * NK * 8) {
                            const float4 v = *reinterpret_cast<const float4 *>(st + 4 * (bt + r * nbt));
                            const float4 h = make_float4(tf32_hi_rn(v.x), tf32_hi_rn(v.y), tf32_hi_rn(v.z), tf32_hi_rn(v.w));
                            const float4 l = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
                            *reinterpret_cast<float4 *>(sbm + soff[r]) = h;
                            *reinterpret_cast<float4 *>(sbm + soff[r] + BMF) = l;
                        }
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                }
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(full + bb)) : "memory");
            }
        }
        cp_async_wait<0>();
    }
    // the last chunk's commit covers every MMA of this CTA
    if (nch > 0) mbar_wait(empty + (nch - 1) % kKgBuf, ((nch - 1) / kKgBuf) & 1);
    tc_fence_after();
    if (warp < QA) {   // D lanes = taps: write inner / outer for this CTA
        const int t = q * 32 + lane;
        uint32_t di[NK], dout[NK];
        tmem_ld_nowait<NK>(tl + kDin, di);
        tmem_ld_nowait<NK>(tl + kDout, dout);
        tmem_wait_ld(di);
        tmem_wait_ld(dout);
        if (t < KT) {
#pragma unroll
            for (int f = 0; f < NK; ++f) {
                float *pp = a.partial + ((long long)f * gridDim.x + blockIdx.x) * 2 * KT;
                pp[t] = nch > 0 ? __uint_as_float(di[f]) : 0.0f;
                pp[KT + t] = nch > 0 ? __uint_as_float(dout[f]) : 0.0f;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int K, int NK>
cudaError_t launch_tc_kg(const float *u, const float *e, const float *b, const float *w, int boundary, int B, int H,
                         int W, float *partial, int nblk, cudaStream_t s) {
    constexpr int R = K / 2, UW = kTcVW + 2 * R + 1, UH = kKgTH + 2 * R;
    TcKgArgs a{u, e, b, w, partial, boundary, B, H, W, (W + kTcVW - 1) / kTcVW, (H + kKgTH - 1) / kKgTH};
    const size_t smem = sizeof(float) * ((4 * kKgBuf + 2 * kKgS) * (size_t)NK * 32 + 4 * (size_t)round4(UH * UW) + 16);
    cudaError_t err = cudaFuncSetAttribute(tc_kgrad_kernel<K, NK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    if (nblk > 0) tc_kgrad_kernel<K, NK><<<(unsigned)nblk, kKgThreads, smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace

int tc_kgrad_blocks(int B, int H, int W, int num_sms) {
    const long long nt = (long long)B * ((W + kTcVW - 1) / kTcVW) * ((H + kKgTH - 1) / kKgTH);
    return (int)std::max<long long>(1, std::min<long long>(nt, num_sms));
}

cudaError_t launch_tc_kgrad(int ksize, int Nk, const float *u, const float *e, const float *b, const float *w,
                            int boundary, int B, int H, int W, float *partial, int nblk, cudaStream_t s) {
    if (ksize == 3 && Nk == 8) return launch_tc_kg<3, 8>(u, e, b, w, boundary, B, H, W, partial, nblk, s);
    if (ksize == 5 && Nk == 24) return launch_tc_kg<5, 24>(u, e, b, w, boundary, B, H, W, partial, nblk, s);
    if (ksize == 7 && Nk == 48) return launch_tc_kg<7, 48>(u, e, b, w, boundary, B, H, W, partial, nblk, s);
    return cudaErrorInvalidValue;
}

namespace {

}  // namespace

cudaError_t launch_tc_fwdbank(int ksize, int Nk, const float *in, const float *bf, float *out, int B, int H, int W,
                              cudaStream_t s) {
    if (ksize == 3 && Nk == 8) return launch_tc_fwd<3, 8>(in, bf, out, B, H, W, s);
    if (ksize == 5 && Nk == 24) return launch_tc_fwd<5, 24>(in, bf, out, B, H, W, s);
    if (ksize == 7 && Nk == 48) return launch_tc_fwd<7, 48>(in, bf, out, B, H, W, s);
    return cudaErrorInvalidValue;
}

namespace {
}  // namespace

bool tc_supported(int ksize, int Nk) {
    return (ksize == 3 && Nk == 8) || (ksize == 5 && Nk == 24) || (ksize == 7 && Nk == 48);
}

// Shared memory the tensor engine needs with its smallest tile (16 rows) for a model
// whose stage operand block has `par_floats` floats (0 if (ksize, N_k) is not built).
size_t tc_min_smem_bytes(int ksize, int Nk, int par_floats) {
    if (ksize == 3 && Nk == 8) return sizeof(float) * (size_t)tc_smem_floats<3, 8>(16, par_floats);
    if (ksize == 5 && Nk == 24) return sizeof(float) * (size_t)tc_smem_floats<5, 24>(16, par_floats);
    if (ksize == 7 && Nk == 48) return sizeof(float) * (size_t)tc_smem_floats<7, 48>(16, par_floats);
    return 0;
}

// Output rows per tile: the OH in {128, 96, 64, 48, 32, 24, 16} that minimises
// waves x (M-blocks per tile + ~6 blocks of per-tile set-up and pipeline fill):
// C4 / C5 take 128 (1.155 pixel-stages per output pixel), one 512^2 image 32
// (144 tiles: one wave of 58 x 32 tiles).
int tc_choose_rows(int ksize, int B, int H, int W, int num_sms) {
    const int R = ksize / 2, ow = kTcVW - 2 * R;
    const int cand[] = {128, 96, 64, 48, 32, 24, 16};
    int best = 128;
    double best_cost = 1e300;
    for (int oh : cand) {
        const long long tiles = (long long)B * ((W + ow - 1) / ow) * ((H + oh - 1) / oh);
        const long long waves = (tiles + num_sms - 1) / num_sms;
        const double cost = (double)waves * ((oh + 2 * R) / 2 + 6);
        if (cost < best_cost) { best_cost = cost; best = oh; }
    }
    return best;
}

cudaError_t launch_stage_tc(int ksize, StageArgs &a, int B, cudaStream_t s) {
    if (ksize == 3 && a.Nk == 8) return launch_tc<3, 8>(a, B, s);
    if (ksize == 5 && a.Nk == 24) return launch_tc<5, 24>(a, B, s);
    if (ksize == 7 && a.Nk == 48) return launch_tc<7, 48>(a, B, s);
    return cudaErrorInvalidValue;
}

}  // namespace tnrd
