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
// One CTA owns a TWxTH output tile.  u (tile + 2r halo) and the stage
// parameters live in shared memory; for each filter the CTA computes w_i on
// the tile + r halo into a double-buffered shared array (phase A), then every
// thread accumulates its output block's kbar_i * w_i in registers (phase B).
// The N_k response maps never leave the SM; HBM sees u, f and u+ once per
// stage (12 B/pixel).  All arithmetic is fp32 with explicit fmaf in a fixed
// per-pixel order, so results do not depend on tiling, batching or slabbing.
//
// Boundary R1 (P l.302-311): w is extended by the half-sample mirror.  Out-of-
// image w positions are written by the thread that computes their mirror
// partner, so no extra barrier is needed.  Boundary R2 (exact K^T, S l.57-65):
// taps whose source lies outside the image use the mirrored tap.
#include "tnrd_internal.h"

#include <climits>

namespace tnrd {
namespace {

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

// phi_i on NP values of one lane.  Warp-collective: all lanes must call it
// with the same `fp` and `mode` (see tnrd_internal.h for the scheme).
template <int NP>
__device__ __forceinline__ void phi_eval(const float *__restrict__ fp, int mode,
                                         const float (&v)[NP], float (&w)[NP]) {
    const float4 fc = *reinterpret_cast<const float4 *>(fp);
    const float a_s = fc.x, two_sg = fc.y, inv_ustep = fc.z;
    const int nunits = __float2int_rn(fc.w);
    const float *units = fp + 4;
    const float cs0 = units[0];
    float lo = INFINITY, hi = -INFINITY;
#pragma unroll
    for (int e = 0; e < NP; ++e) {
        const float ys0 = fmaf(a_s, v[e], cs0);
        lo = fminf(lo, ys0);
        hi = fmaxf(hi, ys0);
        w[e] = 0.0f;
    }
    lo = warp_min(lo);
    hi = warp_max(hi);
    // unit u has ys_u = ys_0 - u*ustep; it can be nonzero only if |ys_u| <= kWindow
    const int u0 = max(0, __float2int_ru((lo - kWindow) * inv_ustep));
    const int u1 = min(nunits - 1, __float2int_rd((hi + kWindow) * inv_ustep));
    if (mode == MODE_HORNER) {
        for (int u = u0; u <= u1; ++u) {
            const float4 *up = reinterpret_cast<const float4 *>(units + u * kHornerUnit);
            const float4 q0 = up[0], q1 = up[1], q2 = up[2];
            // q0 = {cs, c-4, c-3, c-2}, q1 = {c-1, c0, c1, c2}, q2 = {c3, ...}
#pragma unroll
            for (int e = 0; e < NP; ++e) {
                const float ys = fmaf(a_s, v[e], q0.x);
                const float G = ex2_ftz(ys * -ys);
                const float yr = fminf(fmaxf(ys, -kClamp), kClamp) * two_sg;
                const float R = ex2_ftz(yr);
                const float Ri = ex2_ftz(-yr);
                const float pp = fmaf(fmaf(fmaf(q2.x, R, q1.w), R, q1.z), R, q1.y);
                const float pm = fmaf(fmaf(fmaf(q0.y, Ri, q0.z), Ri, q0.w), Ri, q1.x) * Ri;
                w[e] = fmaf(G, pp + pm, w[e]);
            }
        }
    } else {
        for (int u = u0; u <= u1; ++u) {
            const float2 q = *reinterpret_cast<const float2 *>(units + u * kDirectUnit);
#pragma unroll
            for (int e = 0; e < NP; ++e) {
                const float ys = fmaf(a_s, v[e], q.x);
                w[e] = fmaf(q.y, ex2_ftz(ys * -ys), w[e]);
            }
        }
    }
}

template <int K, int TW, int TH, int NT, int BR>
struct Tile {
    static constexpr int R = K / 2;
    static constexpr int KK = K * K;
    static constexpr int KK4 = (KK + 3) / 4 * 4;
    static constexpr int WW = (TW + 2 * R + 3) / 4 * 4;  // phi-region buffer width
    static constexpr int WH = TH + 2 * R;                 // phi-region rows
    static constexpr int RUNS_ROW = WW / 4;
    static constexpr int NRUN = RUNS_ROW * WH;
    static constexpr int SEG = 4 + 2 * R;                 // row window of a 4-wide run
    static constexpr int UW = (WW + 2 * R + 3) / 4 * 4;   // u tile width
    static constexpr int UH = TH + 4 * R;
    static constexpr int NBX = TW / 4;
    static constexpr int NBY = TH / BR;
    static_assert(NBX * NBY == NT, "exactly one phase-B block per thread");
    static_assert(NT % 32 == 0, "whole warps");
    static constexpr int smem_floats_fixed = UH * UW + 2 * WH * WW;
};

// Load SEG consecutive floats starting at a 16-byte aligned shared address.
template <int SEG>
__device__ __forceinline__ void load_seg(const float *p, float (&s)[SEG]) {
#pragma unroll
    for (int j = 0; j + 4 <= SEG; j += 4) {
        const float4 q = *reinterpret_cast<const float4 *>(p + j);
        s[j] = q.x; s[j + 1] = q.y; s[j + 2] = q.z; s[j + 3] = q.w;
    }
    if constexpr (SEG % 4 == 2) {
        const float2 q = *reinterpret_cast<const float2 *>(p + SEG - 2);
        s[SEG - 2] = q.x; s[SEG - 1] = q.y;
    }
}

template <int K, int TW, int TH, int NT, int BR, int MINB>
__global__ void __launch_bounds__(NT, MINB) stage_kernel(const __grid_constant__ StageArgs a) {
    using Tl = Tile<K, TW, TH, NT, BR>;
    constexpr int R = Tl::R, KK4 = Tl::KK4, WW = Tl::WW, WH = Tl::WH, UW = Tl::UW, UH = Tl::UH;
    constexpr int SEG = Tl::SEG;

    extern __shared__ float4 smem4[];
    float *s_par = reinterpret_cast<float *>(smem4);
    float *s_u = s_par + a.Nk * a.pstride;
    float *s_w = s_u + UH * UW;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int b = blockIdx.z;
    const int x0 = blockIdx.x * TW;
    const int y0 = a.y_begin + blockIdx.y * TH;
    const int H = a.H, W = a.W;

    // ---- stage parameters -> smem (float4 copy)
    {
        const float4 *src = reinterpret_cast<const float4 *>(a.params);
        const int n4 = a.Nk * a.pstride / 4;
        for (int j = tid; j < n4; j += NT) smem4[j] = __ldg(src + j);
    }
    // ---- u tile (tile + 2r halo), half-sample mirror at the image edges
    {
        const float *ub = a.u_in.ptr + (long long)b * a.u_in.img_stride;
        for (int j = tid; j < UH * UW; j += NT) {
            const int r = j / UW, c = j - r * UW;
            int gy = reflect(y0 - 2 * R + r, H);
            gy = min(max(gy, a.avail_lo), a.avail_hi - 1);
            const int gx = reflect(x0 - 2 * R + c, W);
            s_u[j] = __ldg(ub + (long long)(gy - a.u_in.row_base) * a.u_in.ld + gx);
        }
    }
    __syncthreads();

    const bool border = (x0 - R < 0) || (x0 + TW + R > W) || (y0 - R < 0) || (y0 + TH + R > H);
    // phase-B block of this thread: BR rows x 4 cols at (oyl, oxl) in the tile
    const int oyl = (tid / Tl::NBX) * BR, oxl = (tid % Tl::NBX) * 4;
    const bool r2_edge = (a.boundary == 1) &&
                         ((x0 + oxl - R < 0) || (x0 + oxl + 4 + R > W) ||
                          (y0 + oyl - R < 0) || (y0 + oyl + BR + R > H));

    float acc[BR][4];
#pragma unroll
    for (int ry = 0; ry < BR; ++ry)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[ry][e] = 0.0f;

    for (int i = 0; i < a.Nk; ++i) {
        const float *fpar = s_par + i * a.pstride;
        float *Wb = s_w + (i & 1) * (WH * WW);
        float tk[KK4];
#pragma unroll
        for (int j = 0; j < KK4; j += 4) {
            const float4 q = *reinterpret_cast<const float4 *>(fpar + j);
            tk[j] = q.x; tk[j + 1] = q.y; tk[j + 2] = q.z; tk[j + 3] = q.w;
        }

        // ---------------- phase A: w_i = phi_i(k_i * u) on the tile + r halo
        for (int base = warp * 32; base < Tl::NRUN; base += NT) {
            const bool valid = base + lane < Tl::NRUN;
            const int run = valid ? base + lane : Tl::NRUN - 1;
            const int wr = run / Tl::RUNS_ROW;
            const int wc = (run - wr * Tl::RUNS_ROW) * 4;
            float v[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
            for (int ta = 0; ta < K; ++ta) {  // tap row a = ta - R reads u row (py - a)
                float seg[SEG];
                load_seg<SEG>(s_u + (wr + 2 * R - ta) * UW + wc, seg);
#pragma unroll
                for (int tb = 0; tb < K; ++tb) {  // tap col b = tb - R reads u col (px - b)
                    const float kv = tk[ta * K + tb];
#pragma unroll
                    for (int e = 0; e < 4; ++e) v[e] = fmaf(kv, seg[e + 2 * R - tb], v[e]);
                }
            }
            float w[4];
            phi_eval<4>(fpar + KK4, a.mode, v, w);
            if (valid) {
                const int py = y0 - R + wr, px0 = x0 - R + wc;
                float *wrow = Wb + wr * WW + wc;
                const bool row_in = (unsigned)py < (unsigned)H;
                if (row_in && px0 >= 0 && px0 + 3 < W) {
                    *reinterpret_cast<float4 *>(wrow) = make_float4(w[0], w[1], w[2], w[3]);
                } else if (row_in) {
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if ((unsigned)(px0 + e) < (unsigned)W) wrow[e] = w[e];
                }
                if (border && row_in) {
                    // mirror partners of in-image positions within r of an edge
                    const int my = py < R ? -1 - py : (py >= H - R ? 2 * H - 1 - py : INT_MIN);
                    const int ty = my - (y0 - R);
                    const bool ym = my != INT_MIN && ty >= 0 && ty < WH;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int px = px0 + e;
                        if ((unsigned)px >= (unsigned)W) continue;
                        const int mx = px < R ? -1 - px : (px >= W - R ? 2 * W - 1 - px : INT_MIN);
                        const int tx = mx - (x0 - R);
                        const bool xm = mx != INT_MIN && tx >= 0 && tx < WW;
                        if (xm) Wb[wr * WW + tx] = w[e];
                        if (ym) Wb[ty * WW + wc + e] = w[e];
                        if (xm && ym) Wb[ty * WW + tx] = w[e];
                    }
                }
            }
        }
        __syncthreads();

        // ---------------- phase B: acc += kbar_i * w_i (correlation with k_i)
        if (!r2_edge) {
#pragma unroll
            for (int wrow = 0; wrow < BR + 2 * R; ++wrow) {
                float seg[SEG];
                load_seg<SEG>(Wb + (oyl + wrow) * WW + oxl, seg);
#pragma unroll
                for (int ry = 0; ry < BR; ++ry) {
                    const int ta = wrow - ry;  // tap row index a + R
                    if (ta < 0 || ta >= K) continue;
#pragma unroll
                    for (int tb = 0; tb < K; ++tb) {
                        const float kv = tk[ta * K + tb];
#pragma unroll
                        for (int e = 0; e < 4; ++e) acc[ry][e] = fmaf(kv, seg[e + tb], acc[ry][e]);
                    }
                }
            }
        } else {
            // R2 (exact K^T) near an image edge: a tap whose source lies outside the
            // image uses the tap mirrored in that direction.
            for (int wrow = 0; wrow < BR + 2 * R; ++wrow) {
                float seg[SEG];
                load_seg<SEG>(Wb + (oyl + wrow) * WW + oxl, seg);
                const int sy = y0 + oyl + wrow - R;  // source row
                const bool yout = (unsigned)sy >= (unsigned)H;
#pragma unroll
                for (int ry = 0; ry < BR; ++ry) {
                    const int ta = wrow - ry;
                    if (ta < 0 || ta >= K) continue;
                    const int tay = yout ? (K - 1 - ta) : ta;
#pragma unroll
                    for (int tb = 0; tb < K; ++tb) {
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int sx = x0 + oxl + e + tb - R;
                            const int tbx = ((unsigned)sx >= (unsigned)W) ? (K - 1 - tb) : tb;
                            acc[ry][e] = fmaf(fpar[tay * K + tbx], seg[e + tb], acc[ry][e]);
                        }
                    }
                }
            }
        }
    }

    // ---------------- epilogue: ut = u - d, u+ = prox(ut), store
    const float *fb = a.f.ptr + (long long)b * a.f.img_stride;
    float *ob = a.u_out + (long long)b * a.out_img_stride;
#pragma unroll
    for (int ry = 0; ry < BR; ++ry) {
        const int oy = y0 + oyl + ry;
        if (oy >= a.y_end) continue;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int ox = x0 + oxl + e;
            if (ox >= W) continue;
            const float u = s_u[(oyl + ry + 2 * R) * UW + oxl + e + 2 * R];
            const float fv = __ldg(fb + (long long)(oy - a.f.row_base) * a.f.ld + ox);
            ob[(long long)(oy - a.out_row_base) * a.out_ld + ox] =
                prox_poisson(u - acc[ry][e], a.lambda, fv);
        }
    }
}

// Tile configurations: 0 = "L" 64x64 output tile, 256 threads, 2 CTAs/SM;
//                      1 = "S" 32x32 output tile, 128 threads (small images).
template <int K>
struct Cfg0 { static constexpr int TW = 64, TH = 64, NT = 256, BR = 4, MINB = 2; };
template <int K>
struct Cfg1 { static constexpr int TW = 32, TH = 32, NT = 128, BR = 2, MINB = 4; };

template <int K, class C>
size_t smem_bytes(int Nk, int pstride) {
    using Tl = Tile<K, C::TW, C::TH, C::NT, C::BR>;
    return sizeof(float) * ((size_t)Nk * pstride + Tl::smem_floats_fixed);
}

template <int K, class C>
cudaError_t launch(const StageArgs &a, int B, cudaStream_t s) {
    auto kern = stage_kernel<K, C::TW, C::TH, C::NT, C::BR, C::MINB>;
    const size_t smem = smem_bytes<K, C>(a.Nk, a.pstride);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((a.W + C::TW - 1) / C::TW, (a.y_end - a.y_begin + C::TH - 1) / C::TH, B);
    kern<<<grid, C::NT, smem, s>>>(a);
    return cudaGetLastError();
}

__global__ void debug_phi_kernel(const float *__restrict__ fp, int mode, const float *__restrict__ v,
                                 float *__restrict__ out, long long n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    float vv[1] = {i < n ? v[i] : 0.0f};
    float ww[1];
    phi_eval<1>(fp, mode, vv, ww);  // every lane participates (warp-collective)
    if (i < n) out[i] = ww[0];
}

__global__ void debug_prox_kernel(const float *ut, const float *f, float lam, float *out, long long n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = prox_poisson(ut[i], lam, f[i]);
}

}  // namespace

size_t stage_smem_bytes(int ksize, int tile, int Nk, int pstride) {
    switch (ksize * 2 + tile) {
        case 6: return smem_bytes<3, Cfg0<3>>(Nk, pstride);
        case 7: return smem_bytes<3, Cfg1<3>>(Nk, pstride);
        case 10: return smem_bytes<5, Cfg0<5>>(Nk, pstride);
        case 11: return smem_bytes<5, Cfg1<5>>(Nk, pstride);
        case 14: return smem_bytes<7, Cfg0<7>>(Nk, pstride);
        case 15: return smem_bytes<7, Cfg1<7>>(Nk, pstride);
    }
    return 0;
}

int choose_tile(int ksize, int B, int H, int W, int num_sms) {
    (void)ksize;
    const long long big = (long long)B * ((H + 63) / 64) * ((W + 63) / 64);
    return big >= 2LL * num_sms ? 0 : 1;
}

cudaError_t launch_stage(int ksize, int tile, const StageArgs &a, int B, cudaStream_t s) {
    switch (ksize * 2 + tile) {
        case 6: return launch<3, Cfg0<3>>(a, B, s);
        case 7: return launch<3, Cfg1<3>>(a, B, s);
        case 10: return launch<5, Cfg0<5>>(a, B, s);
        case 11: return launch<5, Cfg1<5>>(a, B, s);
        case 14: return launch<7, Cfg0<7>>(a, B, s);
        case 15: return launch<7, Cfg1<7>>(a, B, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_debug_phi(const float *params, int pstride, int mode, int ksize, int i,
                             const float *v, float *out, long long n, cudaStream_t s) {
    const int KK4 = (ksize * ksize + 3) / 4 * 4;
    const float *fp = params + (long long)i * pstride + KK4;
    const int threads = 256;
    const long long blocks = (n + threads - 1) / threads;
    if (blocks > 0) debug_phi_kernel<<<(unsigned)blocks, threads, 0, s>>>(fp, mode, v, out, n);
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
