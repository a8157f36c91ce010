// Fused TNRD/TRDPD diffusion stage for sm_100a (B200).
//
// One launch = one stage of P Eq.13 over a batch of
// images or a row slab:
//
//   v_i = k_i * u          forward filter bank          (P l.137, l.309)
//   w_i = phi_i(v_i)       Gaussian-RBF influence       (P l.145; S l.104-107)
//   d  += kbar_i * w_i     rotated-filter convolution   (P l.309-311)
//   ut  = u - d            explicit diffusion, tau = 1  (P l.331-333)
//   u+  = prox_lambda(ut)  Poisson proximal map         (P Eq.12, l.318-322)
//
// Tile pairs and packed fp32x2.  One CTA owns TWO TWxTH output
// tiles, A and B (consecutive in x-fastest / y / image order).  Shared memory
// holds u (tile + 2r halo) and, per filter, w_i (tile + r halo) of both tiles
// interleaved as float2 {A, B}, so every multiply-add of both convolutions and
// of the phi evaluation is one sm_100a FFMA2 on a register pair, with the
// filter tap or phi coefficient as a broadcast scalar operand.  FFMA2 does the
// two lanes' FMAs with the same per-element IEEE rounding as FFMA; it halves
// the issue slots per FMA, which is what bounded the one-pixel-per-lane kernel
// (ncu: 73% issue active at 12.3k instructions/pixel/stage).
//
// Per filter i the CTA computes w_i on the tile + r halo (phase A: runs of
// RUNW pixel pairs per thread), then every thread accumulates its BR x 2 block
// of kbar_i * w_i in registers (phase B).  The N_k response maps never leave
// the SM; HBM sees u, f and u+ once per stage (12 B/pixel).  Every pixel's
// arithmetic is a fixed sequence of IEEE fp32 operations, independent of its
// tile, its partner tile, batching or slabbing.
//
// Boundary R1 (P l.302-311): w is extended by the half-sample mirror.  Out-of-
// image w positions are written by the thread that computes their mirror
// partner, so no extra barrier is needed.  Boundary R2 (exact K^T, S l.57-65):
// taps whose source lies outside the image use the mirrored tap.
#include "tnrd_internal.h"
#include "tnrd_device.cuh"

#include <climits>

namespace tnrd {
namespace {

// Horner units [u0, u1] on NP pairs (see tnrd_internal.h).  Each unit is
// expanded from its first centre: t = sg (x - 8b), G = 2^(-t^2), R = 2^(two_sg t),
// block sum = G * sum_{e<8} c_e R^e  (2 MUFU per element).  R is clamped above at
// two_sg*tclamp so R^7 stays finite for lanes right of the block; the clamp only
// binds where every term of the block is below 2^-20 of its weight (host check).
template <int NP>
__device__ __forceinline__ void horner_units(const float *__restrict__ units, float a_s, float two_sg,
                                             float yrmax, int u0, int u1, const f2 (&v)[NP],
                                             f2 (&w)[NP]) {
    for (int u = u0; u <= u1; ++u) {
        const float4 *up = reinterpret_cast<const float4 *>(units + u * kHornerUnit);
        const float4 q0 = up[0], q1 = up[1], q2 = up[2];
        // q0 = {ct, c0, c1, c2}, q1 = {c3, c4, c5, c6}, q2 = {c7, ...}
#pragma unroll
        for (int e = 0; e < NP; ++e) {
            const f2 t = fma2(v[e], bc(a_s), bc(q0.x));
            const f2 q = fma2(t, bc(-kCutBig), bc(-kCutBig * kCutT));  // kCutBig * relu(-t - kCutT)
            const f2 sq = fma2(t, t, pk(fmaxf(lo(q), 0.0f), fmaxf(hi(q), 0.0f)));
            const f2 G = pk(ex2_ftz(-lo(sq)), ex2_ftz(-hi(sq)));
            const f2 yr = mul2(t, bc(two_sg));
            const f2 R = pk(ex2_ftz(fminf(lo(yr), yrmax)), ex2_ftz(fminf(hi(yr), yrmax)));
            f2 p = fma2(R, bc(q2.x), bc(q1.w));
            p = fma2(p, R, bc(q1.z));
            p = fma2(p, R, bc(q1.y));
            p = fma2(p, R, bc(q1.x));
            p = fma2(p, R, bc(q0.w));
            p = fma2(p, R, bc(q0.z));
            p = fma2(p, R, bc(q0.y));
            w[e] = fma2(G, p, w[e]);
        }
    }
}

// phi_i on NP value pairs of one lane.  Warp-collective: all lanes must call it
// with the same `fp` and `mode`.
// Tabulated phi (MODE_TABLE): one 16-byte table read and a cubic per value.
template <int NP>
__device__ __forceinline__ void phi_table_x2(const float4 fc, const float4 *__restrict__ tab, const f2 (&v)[NP],
                                             f2 (&w)[NP]) {
    const float a_t = fc.x, b_t = fc.y, b_lo = fc.w;  // b = b_t + b_lo (hi/lo split)
    const unsigned nint = (unsigned)__float2int_rn(fc.z);
#pragma unroll
    for (int e = 0; e < NP; ++e) {
        float r[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float vv = h ? hi(v[e]) : lo(v[e]);
            const float kf = floorf(fmaf(vv, a_t, b_t));
            // b_t - kf is exact, so f carries the full fp32 precision of the fraction
            const float f = fmaf(vv, a_t, b_t - kf) + b_lo;
            const int k = __float2int_rz(kf);
            const float4 c = __ldg(tab + ((unsigned)k < nint ? (unsigned)k : nint));
            r[h] = fmaf(fmaf(fmaf(c.w, f, c.z), f, c.y), f, c.x);
        }
        w[e] = pk(r[0], r[1]);
    }
}

template <int NP>
__device__ __forceinline__ void phi_x2(const float *__restrict__ fp, int mode, const float4 *__restrict__ tab,
                                       const f2 (&v)[NP], f2 (&w)[NP]) {
    const float4 fc = *reinterpret_cast<const float4 *>(fp);
    if (mode == MODE_TABLE) {
        phi_table_x2<NP>(fc, tab, v, w);
        return;
    }
    const float a_s = fc.x, two_sg = fc.y, inv_ustep = fc.z;
    const int nunits = __float2int_rn(fc.w);
    const float yclamp = fp[4];  // Horner: upper bound of the R exponent
    const float *units = fp + kFc;
    float vmin = INFINITY, vmax = -INFINITY;
#pragma unroll
    for (int e = 0; e < NP; ++e) {
        vmin = fminf(vmin, fminf(lo(v[e]), hi(v[e])));
        vmax = fmaxf(vmax, fmaxf(lo(v[e]), hi(v[e])));
        w[e] = 0ull;
    }
    // a_s > 0 and fmaf rounding is monotone, so these are the min / max of ys_0
    const float cs0 = units[0];
    const float ylo = warp_min(fmaf(a_s, vmin, cs0));
    const float yhi = warp_max(fmaf(a_s, vmax, cs0));
    // unit u has ys_u = ys_0 - u*ustep; it can be nonzero only if |ys_u| <= kWindow
    const int u0 = max(0, __float2int_ru((ylo - kWindow) * inv_ustep));
    // Horner units are also exactly zero for a lane with t < -(kCutT + 0.01) (left cut)
    const int u1 = min(nunits - 1, __float2int_rd((yhi + (mode == MODE_HORNER ? kCutT + 0.01f : kWindow)) * inv_ustep));
    if (mode == MODE_HORNER) {
        horner_units<NP>(units, a_s, two_sg, yclamp, u0, u1, v, w);
    } else {
        for (int u = u0; u <= u1; ++u) {
            const float2 q = *reinterpret_cast<const float2 *>(units + u * kDirectUnit);
#pragma unroll
            for (int e = 0; e < NP; ++e) {
                const f2 ys = fma2(v[e], bc(a_s), bc(q.x));
                const f2 sq = mul2(ys, ys);
                const f2 E = pk(ex2_ftz(-lo(sq)), ex2_ftz(-hi(sq)));
                w[e] = fma2(E, bc(q.y), w[e]);
            }
        }
    }
}

// pitch p >= need (in float2) with p == r (mod 16)
constexpr int pitch_mod16(int need, int r) { return need + (((r - need) % 16) + 16) % 16; }

// Kernel geometry for filter size K and tile configuration C (see Cfg0 / Cfg1).
template <int K_, class C>
struct Geo {
    static constexpr int K = K_;
    static constexpr int TW = C::TW, TH = C::TH, BR = C::BR;
    static constexpr int NX = 32 * C::XW;                          // X threads: convolutions
    static constexpr int NY = 32 * C::YW;                          // Y threads: phi
    static constexpr int NT = NX + NY;
    static constexpr int NSLOT = C::NSLOT;                         // v/w slots in flight
    static constexpr bool ACC_SMEM = C::ACC_SMEM;                  // park d between filters in smem
    static constexpr int RUNWX = 10, RUNWY = C::RUNWY;             // pairs per conv run / phi run
    static constexpr int R = K / 2;
    static constexpr int K8 = tap_pitch(K);
    static constexpr int KT = tap_floats(K);
    static constexpr int BC = 2;                                   // adjoint block width (pairs)
    static constexpr int WWc = (TW + 2 * R + RUNWX - 1) / RUNWX * RUNWX;  // w region width
    static constexpr int RPRX = WWc / RUNWX, RPRY = WWc / RUNWY;   // runs per w row
    static constexpr int WH = TH + 2 * R;                          // w region rows
    static constexpr int NRUNX = WH * RPRX, NRUNY = WH * RPRY;
    static constexpr int SEG = RUNWX + 2 * R;                      // u window of a conv run
    static constexpr int SEGB = BC + 2 * R;                        // w window of an adjoint row
    static constexpr int UH = TH + 4 * R;
    static constexpr int UWc = WWc + 2 * R;
    // Bank-conflict-free shared loads: conv lanes sit 2*RUNWX = 20
    // words apart; with a pitch == 10*RPRX (mod 16) float2, any 8 consecutive runs
    // hit 8 distinct 4-bank groups (LDS.128), and for RUNWY = 5 any 16 consecutive
    // phi runs hit 16 distinct 2-bank groups (LDS.64).
    static constexpr int PU = pitch_mod16(UWc, (10 * RPRX) % 16);
    static constexpr int PW = pitch_mod16(WWc, (10 * RPRX) % 16);
    static constexpr int NBX = TW / BC;
    static constexpr int NBY = TH / BR;
    static constexpr int ACC_F2 = ACC_SMEM ? NX * BR * BC : 0;
    static_assert(WWc % RUNWY == 0 && (RUNWY == 10 || RUNWY == 5), "phi runs tile the w row");
    static_assert(SEG % 2 == 0 && SEGB % 2 == 0, "whole 16-byte segments");
    static_assert(NBX * NBY == NX, "exactly one adjoint block per X thread");
    static_assert(NBX % 8 == 0, "a quarter warp stays in one adjoint row");
    static_assert(NSLOT == 2 || NSLOT == 3, "slot ring");
    static constexpr int smem_f2 = UH * PU + NSLOT * WH * PW + ACC_F2;
};

template <int N>
__device__ __forceinline__ void load_f2(const f2 *p, f2 (&s)[N]) {
#pragma unroll
    for (int j = 0; j < N; j += 2) {
        const ulonglong2 q = *reinterpret_cast<const ulonglong2 *>(p + j);
        s[j] = q.x;
        s[j + 1] = q.y;
    }
}

// N consecutive pairs from shared memory: 16-byte loads when N is even and the
// start is 16-byte aligned (ALIGNED), else 8-byte loads.
template <int N, bool ALIGNED>
__device__ __forceinline__ void load_pairs(const f2 *p, f2 (&s)[N]) {
    if constexpr (ALIGNED && N % 2 == 0) {
        load_f2<N>(p, s);
    } else {
#pragma unroll
        for (int j = 0; j < N; ++j) s[j] = p[j];
    }
}
template <int N, bool ALIGNED>
__device__ __forceinline__ void store_pairs(f2 *p, const f2 (&s)[N]) {
    if constexpr (ALIGNED && N % 2 == 0) {
#pragma unroll
        for (int j = 0; j < N; j += 2) *reinterpret_cast<ulonglong2 *>(p + j) = make_ulonglong2(s[j], s[j + 1]);
    } else {
#pragma unroll
        for (int j = 0; j < N; ++j) p[j] = s[j];
    }
}

template <int K>
__device__ __forceinline__ void load_taps_row(const float *p, float (&t)[tap_pitch(K)]) {
#pragma unroll
    for (int j = 0; j < tap_pitch(K); j += 4) {
        const float4 q = *reinterpret_cast<const float4 *>(p + j);
        t[j] = q.x; t[j + 1] = q.y; t[j + 2] = q.z; t[j + 3] = q.w;
    }
}

struct TileGeo {
    int b, x0, y0;
    bool border;
};

__device__ __forceinline__ TileGeo tile_geo(const StageArgs &a, int t, int TW, int TH, int R) {
    const int per_img = a.tiles_x * a.tiles_y;
    TileGeo g;
    g.b = t / per_img;
    const int rem = t - g.b * per_img;
    const int ty = rem / a.tiles_x;
    g.x0 = (rem - ty * a.tiles_x) * TW;
    g.y0 = a.y_begin + ty * TH;
    g.border = (g.x0 - R < 0) || (g.x0 + TW + R > a.W) || (g.y0 - R < 0) || (g.y0 + TH + R > a.H);
    return g;
}

// Mirror partners of an in-image w position (py, px) within r of an edge (R1).
// `h` selects the half (0 = tile A, 1 = tile B) of the float2 w slot.
template <int R, int WH, int WWc, int PW>
__device__ __forceinline__ void mirror_store(float *Wf, int h, int H, int W, int y0, int x0, int wr, int wcol,
                                             int py, int px, float val) {
    const int my = py < R ? -1 - py : (py >= H - R ? 2 * H - 1 - py : INT_MIN);
    const int mx = px < R ? -1 - px : (px >= W - R ? 2 * W - 1 - px : INT_MIN);
    const int ty = my - (y0 - R), tx = mx - (x0 - R);
    const bool ym = my != INT_MIN && ty >= 0 && ty < WH;
    const bool xm = mx != INT_MIN && tx >= 0 && tx < WWc;
    if (xm) Wf[2 * (wr * PW + tx) + h] = val;
    if (ym) Wf[2 * (ty * PW + wcol) + h] = val;
    if (xm && ym) Wf[2 * (ty * PW + tx) + h] = val;
}

// Forward filter bank of filter i (X threads xt in [0, NX)): v_i = k_i * u on
// the tile + r halo of both tiles, every region position, into the slot Vb.
template <class G>
__device__ __forceinline__ void phase_conv(const float *__restrict__ fpar, const f2 *s_u, f2 *Vb, int xt) {
    constexpr int K = G::K, R = G::R, K8 = G::K8, RUNW = G::RUNWX;
    constexpr int RPR = G::RPRX, NRUN = G::NRUNX, PU = G::PU, PW = G::PW, SEG = G::SEG;
    for (int run = xt; run < NRUN; run += G::NX) {
        const int wr = run / RPR;
        const int wc = (run - wr * RPR) * RUNW;
        f2 v[RUNW];
#pragma unroll
        for (int e = 0; e < RUNW; ++e) v[e] = 0ull;
#pragma unroll
        for (int ta = 0; ta < K; ++ta) {  // tap row a = ta - R reads u row (py - a)
            float tk[K8];
            load_taps_row<K>(fpar + ta * K8, tk);
            const f2 *urow = s_u + (wr + 2 * R - ta) * PU + wc;
            // stream the SEG-pair u window two pairs at a time: pair j feeds
            // v[e] with tap col tb = e + 2R - j (tap col b = tb - R reads u col px - b)
#pragma unroll
            for (int j0 = 0; j0 < SEG; j0 += 2) {
                const ulonglong2 q = *reinterpret_cast<const ulonglong2 *>(urow + j0);
                const f2 uj[2] = {q.x, q.y};
#pragma unroll
                for (int jj = 0; jj < 2; ++jj) {
                    const int j = j0 + jj;
#pragma unroll
                    for (int e = 0; e < RUNW; ++e) {
                        const int tb = e + 2 * R - j;
                        if (tb >= 0 && tb < K) v[e] = fma2(uj[jj], bc(tk[tb]), v[e]);
                    }
                }
            }
        }
        f2 *vrow = Vb + wr * PW + wc;
#pragma unroll
        for (int e = 0; e < RUNW; e += 2)
            *reinterpret_cast<ulonglong2 *>(vrow + e) = make_ulonglong2(v[e], v[e + 1]);
    }
}

// Influence of filter i (Y threads yt in [0, NY)), in place on the slot:
// w_i = phi_i(v_i) at in-image positions, plus the R1 mirror partners of
// in-image positions within r of an edge (out-of-image slots, which no run
// reads as an in-image v).  Warp-collective per run.
template <class G>
__device__ __forceinline__ void phase_phi(const StageArgs &a, const TileGeo &gA, const TileGeo &gB,
                                          const float *__restrict__ fpar, const float4 *__restrict__ tab, f2 *Wb,
                                          int yt) {
    constexpr int R = G::R, KT = G::KT, RUNW = G::RUNWY;
    constexpr int WWc = G::WWc, RPR = G::RPRY, WH = G::WH, NRUN = G::NRUNY, PW = G::PW;
    constexpr bool AL = RUNW % 2 == 0;  // runs start 16-byte aligned
    const int lane = yt & 31, ywarp = yt >> 5;
    const int H = a.H, W = a.W;
    for (int base = ywarp * 32; base < NRUN; base += G::NY) {
        const bool valid = base + lane < NRUN;
        const int run = valid ? base + lane : NRUN - 1;
        const int wr = run / RPR;
        const int wc = (run - wr * RPR) * RUNW;
        f2 *wrow = Wb + wr * PW + wc;
        f2 v[RUNW];
        load_pairs<RUNW, AL>(wrow, v);
        f2 w[RUNW];
#ifdef TNRD_EXP_NOPHI
#pragma unroll
        for (int e = 0; e < RUNW; ++e) w[e] = v[e];
#else
        phi_x2<RUNW>(fpar + KT, a.mode, tab, v, w);
#endif
        if (valid) {
            const int pyA = gA.y0 - R + wr, pyB = gB.y0 - R + wr;
            const int pxA = gA.x0 - R + wc, pxB = gB.x0 - R + wc;
            const bool rowA = (unsigned)pyA < (unsigned)H, rowB = (unsigned)pyB < (unsigned)H;
            if (rowA && rowB && pxA >= 0 && pxA + RUNW <= W && pxB >= 0 && pxB + RUNW <= W) {
                store_pairs<RUNW, AL>(wrow, w);
            } else {
                float *wf = reinterpret_cast<float *>(wrow);
#pragma unroll
                for (int e = 0; e < RUNW; ++e) {
                    if (rowA && (unsigned)(pxA + e) < (unsigned)W) wf[2 * e] = lo(w[e]);
                    if (rowB && (unsigned)(pxB + e) < (unsigned)W) wf[2 * e + 1] = hi(w[e]);
                }
            }
            // mirror partners exist only for runs that reach within r of an edge
            const auto near_edge = [&](int py, int px) {
                return py < R || py >= H - R || px < R || px + RUNW > W - R;
            };
            float *Wf = reinterpret_cast<float *>(Wb);
            if (gA.border && rowA && near_edge(pyA, pxA)) {
                for (int e = 0; e < RUNW; ++e)
                    if ((unsigned)(pxA + e) < (unsigned)W)
                        mirror_store<R, WH, WWc, PW>(Wf, 0, H, W, gA.y0, gA.x0, wr, wc + e, pyA, pxA + e, lo(w[e]));
            }
            if (gB.border && rowB && near_edge(pyB, pxB)) {
                for (int e = 0; e < RUNW; ++e)
                    if ((unsigned)(pxB + e) < (unsigned)W)
                        mirror_store<R, WH, WWc, PW>(Wf, 1, H, W, gB.y0, gB.x0, wr, wc + e, pyB, pxB + e, hi(w[e]));
            }
        }
    }
}

// Phase B for filter i (consumer threads): acc += kbar_i * w_i on the thread's
// BR x BC pair block at (oyl, oxl) -- a correlation of the w slot with k_i.
template <class G>
__device__ __forceinline__ void phase_b(const StageArgs &a, const TileGeo &gA, const TileGeo &gB, bool r2A,
                                        bool r2B, const float *__restrict__ fpar, const f2 *Wb, int oyl, int oxl,
                                        f2 (&acc)[G::BR][G::BC]) {
    constexpr int K = G::K, R = G::R, K8 = G::K8, BR = G::BR, BC = G::BC, PW = G::PW, SEGB = G::SEGB;
    if (!(r2A || r2B)) {
        if constexpr (!G::ACC_SMEM) {
            float tk[K][K8];  // all taps of filter i, loaded once
#pragma unroll
            for (int ta = 0; ta < K; ++ta) load_taps_row<K>(fpar + ta * K8, tk[ta]);
#pragma unroll
            for (int wrow = 0; wrow < BR + 2 * R; ++wrow) {
                f2 seg[SEGB];
                load_f2<SEGB>(Wb + (oyl + wrow) * PW + oxl, seg);
#pragma unroll
                for (int ry = 0; ry < BR; ++ry) {
                    const int ta = wrow - ry;  // tap row index a + R
                    if (ta < 0 || ta >= K) continue;
#pragma unroll
                    for (int tb = 0; tb < K; ++tb)
#pragma unroll
                        for (int e = 0; e < BC; ++e) acc[ry][e] = fma2(seg[e + tb], bc(tk[ta][tb]), acc[ry][e]);
                }
            }
        } else {
            // register-lean variant: one tap row at a time (same operation order)
#pragma unroll
            for (int wrow = 0; wrow < BR + 2 * R; ++wrow) {
                f2 seg[SEGB];
                load_f2<SEGB>(Wb + (oyl + wrow) * PW + oxl, seg);
#pragma unroll
                for (int ry = 0; ry < BR; ++ry) {
                    const int ta = wrow - ry;
                    if (ta < 0 || ta >= K) continue;
                    float tk[K8];
                    load_taps_row<K>(fpar + ta * K8, tk);
#pragma unroll
                    for (int tb = 0; tb < K; ++tb)
#pragma unroll
                        for (int e = 0; e < BC; ++e) acc[ry][e] = fma2(seg[e + tb], bc(tk[tb]), acc[ry][e]);
                }
            }
        }
        return;
    }
    // R2 (exact K^T) near an image edge: a tap whose source lies outside the
    // image uses the tap mirrored in that direction.  Scalar,
    // per tile half, same operation order as the fast path.
    const int H = a.H, W = a.W;
    const float *Wf = reinterpret_cast<const float *>(Wb);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const TileGeo &g = h ? gB : gA;
        const bool r2 = h ? r2B : r2A;
        float accs[BR][BC];
#pragma unroll
        for (int ry = 0; ry < BR; ++ry)
#pragma unroll
            for (int e = 0; e < BC; ++e) accs[ry][e] = h ? hi(acc[ry][e]) : lo(acc[ry][e]);
        for (int wrow = 0; wrow < BR + 2 * R; ++wrow) {
            const int sy = g.y0 + oyl + wrow - R;  // source row
            const bool yout = r2 && (unsigned)sy >= (unsigned)H;
#pragma unroll
            for (int ry = 0; ry < BR; ++ry) {
                const int ta = wrow - ry;
                if (ta < 0 || ta >= K) continue;
                const int tay = yout ? (K - 1 - ta) : ta;
#pragma unroll
                for (int tb = 0; tb < K; ++tb) {
#pragma unroll
                    for (int e = 0; e < BC; ++e) {
                        const int sx = g.x0 + oxl + e + tb - R;
                        const int tbx = (r2 && (unsigned)sx >= (unsigned)W) ? (K - 1 - tb) : tb;
                        const float wv = Wf[2 * ((oyl + wrow) * PW + oxl + e + tb) + h];
                        accs[ry][e] = fmaf(fpar[tay * K8 + tbx], wv, accs[ry][e]);
                    }
                }
            }
        }
#pragma unroll
        for (int ry = 0; ry < BR; ++ry)
#pragma unroll
            for (int e = 0; e < BC; ++e)
                acc[ry][e] = h ? pk(lo(acc[ry][e]), accs[ry][e]) : pk(accs[ry][e], hi(acc[ry][e]));
    }
}

// Warp-specialised stage kernel.  Warps [0, XW) are "X": the
// FMA-only work -- forward filter bank of filter i+1 into slot (i+1)%NSLOT, then
// the adjoint of filter i from slot i%NSLOT, then the epilogue.  The remaining
// YW warps are "Y": the MUFU-heavy phi of filter i, in place on slot i%NSLOT.
// Named barriers: VFULL_s (X arrive, Y wait) and WFULL_s (Y arrive, X wait).
// With three slots no "empty" barrier is needed: X rewrites slot (i+1)%3 only
// after its own WFULL wait of iteration i-1, i.e. after every X thread finished
// the adjoint of filter i-2 that read it.  With two slots an X-only barrier
// before conv(i+1) ensures every X thread finished the adjoint of filter i-1.
// Either way phi(i) runs concurrently with conv(i+1) and the adjoint of i-1.
template <int K_, class C>
__global__ void __launch_bounds__(32 * (C::XW + C::YW), C::MINB) stage_kernel(const __grid_constant__ StageArgs a) {
    using G = Geo<K_, C>;
    constexpr int NT = G::NT, NSLOT = G::NSLOT;
    constexpr int R = G::R, BR = G::BR, BC = G::BC, TW = G::TW, TH = G::TH;
    constexpr int UH = G::UH, UWc = G::UWc, PU = G::PU, SLOT = G::WH * G::PW;
    constexpr int BAR_VFULL = 1, BAR_WFULL = 4, BAR_X = 7;  // ids 1-3, 4-6, 7 (0 = __syncthreads)

    extern __shared__ float4 smem4[];
    float *s_par = reinterpret_cast<float *>(smem4);
    f2 *s_u = reinterpret_cast<f2 *>(s_par + a.Nk * a.pstride);
    f2 *s_w = s_u + UH * PU;              // NSLOT slots
    f2 *s_acc = s_w + NSLOT * SLOT;       // G::ACC_F2 pairs (ACC_SMEM)

    const int tid = threadIdx.x;
    const int H = a.H, W = a.W;
    const int Nk = a.Nk;

    const int tA = 2 * blockIdx.x;
    const bool hasB = tA + 1 < a.n_tiles;
    const TileGeo gA = tile_geo(a, tA, TW, TH, R);
    const TileGeo gB = hasB ? tile_geo(a, tA + 1, TW, TH, R) : gA;

    // ---- stage parameters -> smem (float4 copy)
    {
        const float4 *src = reinterpret_cast<const float4 *>(a.params);
        const int n4 = Nk * a.pstride / 4;
        for (int j = tid; j < n4; j += NT) smem4[j] = __ldg(src + j);
    }
    // ---- u of both tiles (tile + 2r halo), half-sample mirror at the image edges
    {
        const float *ubA = a.u_in.ptr + (long long)gA.b * a.u_in.img_stride;
        const float *ubB = a.u_in.ptr + (long long)gB.b * a.u_in.img_stride;
        for (int j = tid; j < UH * UWc; j += NT) {
            const int r = j / UWc, c = j - r * UWc;
            int gyA = reflect(gA.y0 - 2 * R + r, H), gyB = reflect(gB.y0 - 2 * R + r, H);
            gyA = min(max(gyA, a.avail_lo), a.avail_hi - 1);
            gyB = min(max(gyB, a.avail_lo), a.avail_hi - 1);
            const int gxA = reflect(gA.x0 - 2 * R + c, W), gxB = reflect(gB.x0 - 2 * R + c, W);
            const float uA = __ldg(ubA + (long long)(gyA - a.u_in.row_base) * a.u_in.ld + gxA);
            const float uB = __ldg(ubB + (long long)(gyB - a.u_in.row_base) * a.u_in.ld + gxB);
            s_u[r * PU + c] = pk(uA, uB);
        }
    }
    __syncthreads();

    if (tid >= G::NX) {
        // ======================= Y: phi in place, filter by filter
        const int yt = tid - G::NX;
        for (int i = 0; i < Nk; ++i) {
            const int slot = i % NSLOT;
            named_sync(BAR_VFULL + slot, NT);
            phase_phi<G>(a, gA, gB, s_par + i * a.pstride, a.table + (size_t)i * a.table_stride,
                         s_w + slot * SLOT, yt);
            named_arrive(BAR_WFULL + slot, NT);
        }
        return;
    }

    // ======================= X: forward conv (i+1), adjoint (i), epilogue
    const int xt = tid;
    const int oyl = (xt / G::NBX) * BR, oxl = (xt % G::NBX) * BC;
    const auto r2_edge = [&](const TileGeo &g) {
        return (a.boundary == 1) && ((g.x0 + oxl - R < 0) || (g.x0 + oxl + BC + R > W) ||
                                     (g.y0 + oyl - R < 0) || (g.y0 + oyl + BR + R > H));
    };
    const bool r2A = r2_edge(gA), r2B = r2_edge(gB);
    // accumulator block of this thread in smem: 16-byte chunk j of thread xt at
    // [j][xt] (lane-consecutive, conflict-free)
    ulonglong2 *accp = reinterpret_cast<ulonglong2 *>(s_acc) + xt;
    constexpr int ACC_CHUNKS = BR * BC / 2;

    // d of this thread's block: in registers across filters (S), or parked in smem
    // between filters so it is not live during the forward conv (L, 80 registers)
    f2 acc_reg[BR][BC];
#pragma unroll
    for (int ry = 0; ry < BR; ++ry)
#pragma unroll
        for (int e = 0; e < BC; ++e) acc_reg[ry][e] = 0ull;

    phase_conv<G>(s_par, s_u, s_w, xt);
    named_arrive(BAR_VFULL + 0, NT);
    for (int i = 0; i < Nk; ++i) {
        if (i + 1 < Nk) {
            const int nslot = (i + 1) % NSLOT;
            if (NSLOT == 2 && i >= 1) named_sync(BAR_X, G::NX);  // adjoint(i-1) done with this slot
#ifndef TNRD_EXP_NOCONV
            phase_conv<G>(s_par + (i + 1) * a.pstride, s_u, s_w + nslot * SLOT, xt);
#endif
            named_arrive(BAR_VFULL + nslot, NT);
        }
        const int slot = i % NSLOT;
        named_sync(BAR_WFULL + slot, NT);  // phi of filter i done
        if constexpr (G::ACC_SMEM) {
            f2 acc[BR][BC];
#pragma unroll
            for (int j = 0; j < ACC_CHUNKS; ++j) {
                const ulonglong2 q = i > 0 ? accp[j * G::NX] : make_ulonglong2(0ull, 0ull);
                acc[(2 * j) / BC][(2 * j) % BC] = q.x;
                acc[(2 * j + 1) / BC][(2 * j + 1) % BC] = q.y;
            }
#ifndef TNRD_EXP_NOADJ
            phase_b<G>(a, gA, gB, r2A, r2B, s_par + i * a.pstride, s_w + slot * SLOT, oyl, oxl, acc);
#endif
#pragma unroll
            for (int j = 0; j < ACC_CHUNKS; ++j)
                accp[j * G::NX] = make_ulonglong2(acc[(2 * j) / BC][(2 * j) % BC],
                                                  acc[(2 * j + 1) / BC][(2 * j + 1) % BC]);
        } else {
#ifndef TNRD_EXP_NOADJ
            phase_b<G>(a, gA, gB, r2A, r2B, s_par + i * a.pstride, s_w + slot * SLOT, oyl, oxl, acc_reg);
#endif
        }
    }
    if constexpr (G::ACC_SMEM) {
#pragma unroll
        for (int j = 0; j < ACC_CHUNKS; ++j) {
            const ulonglong2 q = accp[j * G::NX];
            acc_reg[(2 * j) / BC][(2 * j) % BC] = q.x;
            acc_reg[(2 * j + 1) / BC][(2 * j + 1) % BC] = q.y;
        }
    }
    f2 (&acc)[BR][BC] = acc_reg;

    // ---------------- epilogue: ut = u - d, u+ = prox(ut), store (per tile half)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        if (h == 1 && !hasB) break;
        const TileGeo &g = h ? gB : gA;
        const float *fb = a.f.ptr + (long long)g.b * a.f.img_stride;
        float *ob = a.u_out + (long long)g.b * a.out_img_stride;
#pragma unroll
        for (int ry = 0; ry < BR; ++ry) {
            const int oy = g.y0 + oyl + ry;
            if (oy >= a.y_end) continue;
#pragma unroll
            for (int e = 0; e < BC; ++e) {
                const int ox = g.x0 + oxl + e;
                if (ox >= W) continue;
                const f2 u2 = s_u[(oyl + ry + 2 * R) * PU + oxl + e + 2 * R];
                const float u = h ? hi(u2) : lo(u2);
                const float d = h ? hi(acc[ry][e]) : lo(acc[ry][e]);
                const float fv = __ldg(fb + (long long)(oy - a.f.row_base) * a.f.ld + ox);
                const long long oi = (long long)(oy - a.out_row_base) * a.out_ld + ox;
                ob[oi] = reaction_step(a.reaction, u, u - d, a.lambda, fv);
                if (a.ut_out) a.ut_out[(long long)g.b * a.out_img_stride + oi] = u - d;
            }
        }
    }
}

// Tile configurations.
//  0 = "L": two 64x64 output tiles, 8 X warps + 8 Y warps (512 threads, 128
//      registers), 3 slots, d in registers; 1 CTA per SM (~200 KB shared memory).
//      (8 + 16 warps at 80 registers, d parked in smem, 2 slots: 27.1 vs 23.8 ms.)
//  1 = "S": two 32x32 output tiles, 8 + 8 warps (one conv / phi pass each per
//      filter), 3 slots, d in registers, for images too small to fill the GPU with
//      "L" tiles (C3, one 512^2 image: 1.66 ms; 2.34 ms with 2 + 2 warps).
struct Cfg0 { static constexpr int TW = 64, TH = 64, XW = 8, YW = 8, RUNWY = 10, BR = 8, NSLOT = 3, MINB = 1;
              static constexpr bool ACC_SMEM = false; };
struct Cfg1 { static constexpr int TW = 32, TH = 32, XW = 8, YW = 8, RUNWY = 10, BR = 2, NSLOT = 3, MINB = 1;
              static constexpr bool ACC_SMEM = false; };

template <int K, class C>
size_t smem_bytes(int Nk, int pstride) {
    return sizeof(float) * (size_t)Nk * pstride + sizeof(f2) * (size_t)Geo<K, C>::smem_f2;
}

template <int K, class C>
cudaError_t launch(StageArgs &a, int B, cudaStream_t s) {
    auto kern = stage_kernel<K, C>;
    const size_t smem = smem_bytes<K, C>(a.Nk, a.pstride);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    a.tiles_x = (a.W + C::TW - 1) / C::TW;
    a.tiles_y = (a.y_end - a.y_begin + C::TH - 1) / C::TH;
    const long long n = (long long)B * a.tiles_x * a.tiles_y;
    if (n > INT_MAX - 1) return cudaErrorInvalidValue;
    a.n_tiles = (int)n;
    kern<<<(unsigned)((n + 1) / 2), Geo<K, C>::NT, smem, s>>>(a);
    return cudaGetLastError();
}

__global__ void debug_phi_kernel(const float *__restrict__ fp, int mode, const float4 *__restrict__ tab,
                                 const float *__restrict__ v, float *__restrict__ out, long long n) {
    // each thread evaluates a pair (elements 2t, 2t+1) through the stage kernel's phi_x2
    const long long i = 2 * ((long long)blockIdx.x * blockDim.x + threadIdx.x);
    f2 vv[1] = {pk(i < n ? v[i] : 0.0f, i + 1 < n ? v[i + 1] : 0.0f)};
    f2 ww[1];
    phi_x2<1>(fp, mode, tab, vv, ww);  // every lane participates (warp-collective)
    if (i < n) out[i] = lo(ww[0]);
    if (i + 1 < n) out[i + 1] = hi(ww[0]);
}

__global__ void debug_prox_kernel(const float *ut, const float *f, float lam, float *out, long long n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = prox_poisson(ut[i], lam, f[i]);
}

}  // namespace

size_t stage_smem_bytes(int ksize, int tile, int Nk, int pstride) {
    switch (ksize * 2 + tile) {
        case 6: return smem_bytes<3, Cfg0>(Nk, pstride);
        case 7: return smem_bytes<3, Cfg1>(Nk, pstride);
        case 10: return smem_bytes<5, Cfg0>(Nk, pstride);
        case 11: return smem_bytes<5, Cfg1>(Nk, pstride);
        case 14: return smem_bytes<7, Cfg0>(Nk, pstride);
        case 15: return smem_bytes<7, Cfg1>(Nk, pstride);
        case 18: return smem_bytes<9, Cfg0>(Nk, pstride);
        case 19: return smem_bytes<9, Cfg1>(Nk, pstride);
        case 22: return smem_bytes<11, Cfg0>(Nk, pstride);
        case 23: return smem_bytes<11, Cfg1>(Nk, pstride);
    }
    return 0;
}

int choose_tile(int ksize, int B, int H, int W, int num_sms) {
    (void)ksize;
    // "L" once its tile pairs fill at least half a wave: measured on 512^2 images
    // (profiles/r01_tile_crossover.json) L takes 2.94 ms for 1..4 images (<= one
    // wave) while S takes 1.61 / 2.80 / 3.94 ms for 1 / 2 / 3 images.
    const long long pairs = ((long long)B * ((H + 63) / 64) * ((W + 63) / 64) + 1) / 2;
    return 2 * pairs >= num_sms ? 0 : 1;
}

cudaError_t launch_stage(int ksize, int tile, StageArgs &a, int B, cudaStream_t s) {
    switch (ksize * 2 + tile) {
        case 6: return launch<3, Cfg0>(a, B, s);
        case 7: return launch<3, Cfg1>(a, B, s);
        case 10: return launch<5, Cfg0>(a, B, s);
        case 11: return launch<5, Cfg1>(a, B, s);
        case 14: return launch<7, Cfg0>(a, B, s);
        case 15: return launch<7, Cfg1>(a, B, s);
        case 18: return launch<9, Cfg0>(a, B, s);
        case 19: return launch<9, Cfg1>(a, B, s);
        case 22: return launch<11, Cfg0>(a, B, s);
        case 23: return launch<11, Cfg1>(a, B, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_debug_phi(const float *params, int pstride, int mode, const float4 *table, int ksize, int i,
                             const float *v, float *out, long long n, cudaStream_t s) {
    const float *fp = params + (long long)i * pstride + tap_floats(ksize);
    const int threads = 256;
    const long long blocks = ((n + 1) / 2 + threads - 1) / threads;
    if (blocks > 0) debug_phi_kernel<<<(unsigned)blocks, threads, 0, s>>>(fp, mode, table, v, out, n);
    return cudaGetLastError();
}

cudaError_t launch_debug_prox(const float *ut, const float *f, float lambda, float *out, long long n,
                              cudaStream_t s) {
    const int threads = 256;
    const long long blocks = (n + threads - 1) / threads;
    if (blocks > 0) debug_prox_kernel<<<(unsigned)blocks, threads, 0, s>>>(ut, f, lambda, out, n);
    return cudaGetLastError();
}

cudaError_t launch_copy_rows(const float *src, long long src_ld, float *dst, long long dst_ld, int rows,
                             int W, cudaStream_t s) {
    return cudaMemcpy2DAsync(dst, dst_ld * sizeof(float), src, src_ld * sizeof(float), W * sizeof(float),
                             rows, cudaMemcpyDeviceToDevice, s);
}

}  // namespace tnrd
