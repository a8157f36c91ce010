// Training-loss gradient of the TNRD inference pass on sm_100a.
//
// loss = 1/2 sum_b ||u_T - u_gt||^2 (P Eq.6, l.199-222), gradient w.r.t.
// Theta_t = {lambda_t, RBF weights of phi_i^t, k_i^t} by the chain rule of
// P l.343-420 (Eq.14-20), reaction 0 (Eq.13).  The host (tnrd_api.cpp) runs the
// forward pass with a tape (u_t and ut_t from the fused stage kernel), then for
// t = T-1 .. 0 these batch-wide kernels:
//
//   bw_prox        e = y (.) g (Eq.16), gn = e, partial sums of z (.) g (Eq.19)
//   conv_sym       x_i = k_i * u_t                         (symmetric extension)
//   conv_adjoint   a_i = outer_i^T e  (R1: Kbar_i^T, R2: K_i)  and  gn -= K_i^T b_i
//   phi_point      w_i = phi(x_i), b_i = phi'(x_i) a_i (Lambda_i, P l.369-371),
//                  partial sums of -a_i G_j(x_i)           (d l / d w_ij)
//   kernel_grad    partial sums of e(p) E(x)(p - tap)       (d l / d k_i)
//   reduce         deterministic fixed-order sums of the per-block partials
//
// Every partial sum is a fixed-order warp-shuffle tree plus a fixed-order sum over
// warps and blocks, so gradients are bitwise reproducible.  These kernels are the
// correct, simple form of the backward (one HBM pass per operation); the fused
// forward stage kernel (tnrd_kernels.cu) is the optimised hot path.
#include "tnrd_internal.h"
#include "tnrd_device.cuh"

#include <algorithm>

namespace tnrd {
namespace {

constexpr int kGradThreads = 256;

__device__ __forceinline__ int mirror(int x, int n) {
    x = x < 0 ? -1 - x : x;
    x = x >= n ? 2 * n - 1 - x : x;
    return min(max(x, 0), n - 1);
}

// Sum vals[0..NV) over the block (fixed order) into out[0..NV) (thread j writes j).
template <int NV>
__device__ __forceinline__ void block_sum(float (&vals)[NV], float *out) {
    __shared__ float red[kGradThreads / 32][NV];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        float x = vals[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) red[warp][j] = x;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < NV; j += blockDim.x) {
        float s = 0.0f;
        for (int w = 0; w < kGradThreads / 32; ++w) s += red[w][j];
        out[j] = s;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kGradThreads) loss_kernel(const float *__restrict__ uT, const float *__restrict__ gt,
                                                            long long gt_ld, int B, int H, int W, float *__restrict__ g,
                                                            float *__restrict__ partial) {
    const long long n = (long long)B * H * W;
    float v[1] = {0.0f};
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
        const long long b = p / ((long long)H * W), r = p - b * H * W;
        const int y = (int)(r / W), x = (int)(r - (long long)y * W);
        const float d = uT[p] - gt[b * H * gt_ld + (long long)y * gt_ld + x];  // dl/du_T = u_T - u_gt (l.348-353)
        g[p] = d;
        v[0] = fmaf(0.5f * d, d, v[0]);
    }
    block_sum<1>(v, partial + blockIdx.x);
}

// e = y (.) g with the prox Jacobian y (Eq.16); z (Eq.19) weights g into d l / d lambda.
__global__ void __launch_bounds__(kGradThreads) bw_prox_kernel(const float *__restrict__ ut, const float *__restrict__ f,
                                                               long long f_ld, int B, int H, int W, float lam,
                                                               const float *__restrict__ g, float *__restrict__ e,
                                                               float *__restrict__ gn, float *__restrict__ partial) {
    const long long n = (long long)B * H * W;
    float v[1] = {0.0f};
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
        const long long b = p / ((long long)H * W), r = p - b * H * W;
        const int y = (int)(r / W), x = (int)(r - (long long)y * W);
        const float fv = f[b * H * f_ld + (long long)y * f_ld + x];
        const float delta = ut[p] - lam;
        const float sigma = sqrtf(fmaf(delta, delta, 4.0f * lam * fv));
        float yv = 0.5f, zv = -0.5f;
        if (sigma > 0.0f) {
            // stable forms: 1 + delta/sigma = 4 lam f / (sigma (sigma - delta)) for delta < 0
            yv = delta >= 0.0f ? 0.5f * (1.0f + delta / sigma) : 2.0f * lam * fv / (sigma * (sigma - delta));
            zv = 0.5f * (-1.0f + (2.0f * fv - delta) / sigma);
        }
        const float gv = g[p];
        const float ev = yv * gv;
        e[p] = ev;
        gn[p] = ev;  // identity part of Eq.15
        v[0] = fmaf(zv, gv, v[0]);
    }
    block_sum<1>(v, partial + blockIdx.x);
}

// ---- filter-batched backward kernels: blockIdx.y = filter f of the chunk [i0, i0 + F)
// of stage t; per-filter parameters at raw + (t*Nk + i0 + f) * stride.

struct GradFilterArgs {
    const float *k, *kbar, *rw, *grid3;  // [T*Nk][m*m], [T*Nk][m*m], [T*Nk][M], [T*Nk][3] (mu0, step, gamma)
    int fi0;                             // t*Nk + i0
    int m, M, B, H, W;
    long long n;                         // B*H*W
};

// conv2d_sym at pixel (y, x) of image xb (dense H x W): sum_{a,c} k[a][c] E(x)(y-(a-r), x-(c-r)).
template <int m>
__device__ __forceinline__ float conv_at(const float *__restrict__ xb, const float *__restrict__ k, int y, int x,
                                         int H, int W, bool interior) {
    constexpr int r = m / 2;
    float s = 0.0f;
    if (interior) {
#pragma unroll
        for (int a = 0; a < m; ++a) {
            const float *row = xb + (long long)(y - (a - r)) * W + x + r;
#pragma unroll
            for (int c = 0; c < m; ++c) s = fmaf(k[a * m + c], row[-c], s);
        }
    } else {
#pragma unroll
        for (int a = 0; a < m; ++a) {
            const float *row = xb + (long long)mirror(y - (a - r), H) * W;
#pragma unroll
            for (int c = 0; c < m; ++c) s = fmaf(k[a * m + c], row[mirror(x - (c - r), W)], s);
        }
    }
    return s;
}

// (K^T y)(q): the exact transpose of conv2d_sym; interior outputs see only the
// direct sources q + d (a correlation), edge outputs also the mirror preimages.
template <int m>
__device__ __forceinline__ float adj_at(const float *__restrict__ yb, const float *__restrict__ k, int qy, int qx,
                                        int H, int W, bool interior) {
    constexpr int r = m / 2;
    float s = 0.0f;
    if (interior) {
#pragma unroll
        for (int a = 0; a < m; ++a) {
            const float *row = yb + (long long)(qy + a - r) * W + qx - r;
#pragma unroll
            for (int c = 0; c < m; ++c) s = fmaf(k[a * m + c], row[c], s);
        }
        return s;
    }
    for (int a = 0; a < m; ++a) {
        const int dy = a - r;
        const int cy[3] = {qy + dy, dy - 1 - qy, 2 * H - 1 - qy + dy};
        for (int iy = 0; iy < 3; ++iy) {
            const int py = cy[iy];
            if (py < 0 || py >= H || mirror(py - dy, H) != qy) continue;
            for (int c = 0; c < m; ++c) {
                const int dx = c - r;
                const int cx[3] = {qx + dx, dx - 1 - qx, 2 * W - 1 - qx + dx};
                for (int ix = 0; ix < 3; ++ix) {
                    const int px = cx[ix];
                    if (px < 0 || px >= W || mirror(px - dx, W) != qx) continue;
                    s = fmaf(k[a * m + c], yb[(long long)py * W + px], s);
                }
            }
        }
    }
    return s;
}

// x_f = k_f * u  and  a_f = outer_f^T e  (R1: Kbar_f^T e, R2: K_f e).
template <int m>
__global__ void __launch_bounds__(kGradThreads) fwd_pair_kernel(GradFilterArgs g, const float *__restrict__ u,
                                                                const float *__restrict__ e, int boundary,
                                                                float *__restrict__ xo, float *__restrict__ ao) {
    constexpr int r = m / 2;
    __shared__ float sk[2][m * m];
    const int f = blockIdx.y;
    for (int j = threadIdx.x; j < m * m; j += blockDim.x) {
        sk[0][j] = g.k[(long long)(g.fi0 + f) * m * m + j];
        sk[1][j] = g.kbar[(long long)(g.fi0 + f) * m * m + j];
    }
    __syncthreads();
    const int H = g.H, W = g.W;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < g.n; p += (long long)gridDim.x * blockDim.x) {
        const long long b = p / ((long long)H * W), rr = p - b * H * W;
        const int y = (int)(rr / W), x = (int)(rr - (long long)y * W);
        const bool in = y >= r && y < H - r && x >= r && x < W - r;
        xo[(long long)f * g.n + p] = conv_at<m>(u + b * H * W, sk[0], y, x, H, W, in);
        ao[(long long)f * g.n + p] = boundary == 1 ? conv_at<m>(e + b * H * W, sk[0], y, x, H, W, in)
                                                   : adj_at<m>(e + b * H * W, sk[1], y, x, H, W, in);
    }
}

// a_f = Kbar_f^T e on the pixels within r of an image edge (R1), where the exact
// transpose differs from the mirrored convolution the tensor forward bank computed.
// A block takes kBorderPix border pixels: first E~_t(q) for every (pixel q, tap t),
// the sum of e over the preimages p of q (the mirror is separable: rows py with
// mirror(py - dy) = qy times columns px with mirror(px - dx) = qx, at most 2 x 2),
// into shared memory; then a_f(q) = sum_t kbar_f[t] E~_t(q) in tap order for every
// (pixel, filter).
constexpr int kBorderThreads = 128;
constexpr int kBorderMaxF = 64;
#ifndef TNRD_BORDER_PIX
#define TNRD_BORDER_PIX 8
#endif
constexpr int kBorderPix = TNRD_BORDER_PIX;

__device__ __forceinline__ bool border_pixel(long long idx, int r, int H, int W, long long nb, long long &b, int &y,
                                             int &x) {
    const long long top = (long long)r * W;
    b = idx / nb;
    const long long k = idx - b * nb;
    if (k < top) { y = (int)(k / W); x = (int)(k - (long long)y * W); }
    else if (k < 2 * top) { const long long q = k - top; y = H - r + (int)(q / W); x = (int)(q % W); }
    else { const long long q = k - 2 * top; y = r + (int)(q / (2 * r)); const int c = (int)(q % (2 * r)); x = c < r ? c : W - 2 * r + c; }
    return y >= 0 && y < H;
}

template <int m>
__global__ void __launch_bounds__(kBorderThreads) adj_border_kernel(GradFilterArgs g, int F, const float *__restrict__ e,
                                                                    float *__restrict__ ao) {
    constexpr int r = m / 2, mm = m * m;
    __shared__ float sk[kBorderMaxF * mm];
    __shared__ float set[kBorderPix][mm + 1];
    for (int j = threadIdx.x; j < F * mm; j += blockDim.x) sk[j] = g.kbar[(long long)g.fi0 * mm + j];
    const int H = g.H, W = g.W;
    const long long nb = 2LL * r * W + 2LL * r * (H - 2 * r > 0 ? H - 2 * r : 0);  // border pixels per image
    const long long total = (long long)g.B * nb;
    for (long long i0 = (long long)blockIdx.x * kBorderPix; i0 < total; i0 += (long long)gridDim.x * kBorderPix) {
        __syncthreads();   // sk loaded / the previous pixels' set consumed
        for (int w = threadIdx.x; w < kBorderPix * mm; w += blockDim.x) {
            const int pi = w / mm, t = w - pi * mm;
            long long b;
            int y, x;
            float v = 0.0f;
            if (i0 + pi < total && border_pixel(i0 + pi, r, H, W, nb, b, y, x)) {
                const int dy = t / m - r, dx = t % m - r;
                const float *eb = e + b * H * W;
#pragma unroll
                for (int iy = 0; iy < 3; ++iy) {
                    const int py = iy == 0 ? y + dy : (iy == 1 ? dy - 1 - y : 2 * H - 1 - y + dy);
                    if (py < 0 || py >= H || mirror(py - dy, H) != y) continue;
#pragma unroll
                    for (int ix = 0; ix < 3; ++ix) {
                        const int px = ix == 0 ? x + dx : (ix == 1 ? dx - 1 - x : 2 * W - 1 - x + dx);
                        if (px < 0 || px >= W || mirror(px - dx, W) != x) continue;
                        v += __ldg(eb + (long long)py * W + px);
                    }
                }
            }
            set[pi][t] = v;
        }
        __syncthreads();
        for (int w = threadIdx.x; w < kBorderPix * F; w += blockDim.x) {
            const int pi = w % kBorderPix, f = w / kBorderPix;
            long long b;
            int y, x;
            if (i0 + pi >= total || !border_pixel(i0 + pi, r, H, W, nb, b, y, x)) continue;
            float v = 0.0f;
#pragma unroll
            for (int t = 0; t < mm; ++t) v = fmaf(sk[f * mm + t], set[pi][t], v);
            ao[(long long)f * g.n + b * H * W + (long long)y * W + x] = v;
        }
    }
}

// w_f = phi(x_f), b_f = phi'(x_f) a_f (Lambda, P l.369-371), partial sums of
// -a_f G_j(x_f) (d l / d w_j) for j < M <= 64: every Gaussian evaluated once.
// Two threads per pixel (lanes l and l ^ 16 of a warp: 16 pixels per warp), half h
// owning the centres j = 2i + h, i < 32, as 16 pairs (i, i + 1) in packed fp32x2
// (weights and accumulators in registers).  With sc = sqrt(log2 e / 2) / gamma and
// d'_j = (x - mu_j) sc, G_j = 2^(-d'_j^2); phi' uses sum_j w_j d'_j G_j / sc.
// phi and phi' are the two halves' sums, each half's pair lanes added low + high,
// then half 0 + half 1 (fixed order).  Pairs run in groups of TNRD_PHI_GP behind
// warp-uniform branches: a group is skipped when all its centres lie outside
// [jlo, jhi], the centres within dmax of some value of the warp; beyond dmax every
// G_j is exactly 0 (ex2.approx.ftz of < -126 flushes, kPhiCut = 126), so skipping
// changes no sum.  (A cut at 2^-40 instead measured no faster: DESIGN.md §5.9.)
#ifndef TNRD_PHI_THREADS
#define TNRD_PHI_THREADS 512
#endif
constexpr int kPhiThreads = TNRD_PHI_THREADS;
#ifndef TNRD_PHI_CUT
#define TNRD_PHI_CUT 126.0f
#endif
#ifndef TNRD_PHI_GP
#define TNRD_PHI_GP 4
#endif
constexpr float kPhiCut = TNRD_PHI_CUT;   // 2^(-t) for t > kPhiCut is not evaluated (exactly 0 at 126)

#ifndef TNRD_PHI_MINB
#define TNRD_PHI_MINB 1
#endif
__global__ void __launch_bounds__(kPhiThreads, TNRD_PHI_MINB) phi_all_kernel(GradFilterArgs g, const float *__restrict__ xv,
                                                                 const float *__restrict__ av, float *__restrict__ wo,
                                                                 float *__restrict__ bo, float *__restrict__ partial) {
    __shared__ float red[kPhiThreads / 32][64];
    const int f = blockIdx.y, M = g.M, lane = threadIdx.x & 31, warp = threadIdx.x >> 5, h = lane >> 4;
    const float mu0 = g.grid3[(g.fi0 + f) * 3], step = g.grid3[(g.fi0 + f) * 3 + 1], gam = g.grid3[(g.fi0 + f) * 3 + 2];
    const float sc = sqrtf(0.72134752044448170f) / gam;             // sqrt(log2(e) / 2) / gamma
    const float s2 = 2.0f * step * sc, base = fmaf((float)h, step, mu0), invg2 = 1.0f / (gam * gam);
    // 2^(-t) = 0 (flushed) for t = d^2 log2(e) / (2 gamma^2) > kPhiCut = 126: |d| > dmax
    const float dmax = sqrtf(kPhiCut / 0.72134752044448170f) * gam * 1.0001f + 1e-6f * (fabsf(mu0) + 64.0f * step);
    const float rstep = 1.0f / step, bscale = invg2 / sc;
    const f2 s2v = bc(s2), m2s2 = bc(-2.0f * s2);
    f2 w2[16], acc2[16];
#pragma unroll
    for (int ip = 0; ip < 16; ++ip) {
        const int j0 = 4 * ip + h, j1 = 4 * ip + 2 + h;    // centres of local i = 2ip, 2ip + 1
        const float *rw = g.rw + (long long)(g.fi0 + f) * M;
        w2[ip] = pk(j0 < M ? rw[j0] : 0.0f, j1 < M ? rw[j1] : 0.0f);
        acc2[ip] = 0ull;
    }
    const long long n = g.n;
    const float *xf = xv + (long long)f * n, *af = av + (long long)f * n;
    const long long pstep = (long long)gridDim.x * (kPhiThreads / 32) * 16;
    long long p = ((long long)blockIdx.x * (kPhiThreads / 32) + warp) * 16 + (lane & 15);
    // loads run TNRD_PHI_PF iterations ahead (a register ring)
#ifndef TNRD_PHI_PF
#define TNRD_PHI_PF 2
#endif
    constexpr int PF = TNRD_PHI_PF;
    float xr[PF], ar[PF];
#pragma unroll
    for (int k = 0; k < PF; ++k) {
        const long long q = p + k * pstep;
        xr[k] = q < n ? xf[q] : 0.0f;
        ar[k] = q < n ? af[q] : 0.0f;
    }
    for (; p - (lane & 15) < n; p += pstep) {
        const bool valid = p < n;
        const float x = xr[0], na = valid ? -ar[0] : 0.0f;
#pragma unroll
        for (int k = 0; k + 1 < PF; ++k) { xr[k] = xr[k + 1]; ar[k] = ar[k + 1]; }
        {
            const long long q = p + PF * pstep;
            if (q < n) { xr[PF - 1] = xf[q]; ar[PF - 1] = af[q]; }
        }
        const float wmin = warp_min(valid ? x : 3.0e38f), wmax = warp_max(valid ? x : -3.0e38f);
        // the warp's centre range (its 16 pixels), as local indices i = j >> 1 of
        // both halves: warp-uniform
        // floor / ceil by directed-rounding adds of 1.5 * 2^23 (no F2I on the XU pipe the
        // exponentials use), after clamping into [-4, 68]
        const float flo = fminf(fmaxf((wmin - dmax - mu0) * rstep, -4.0f), 68.0f);
        const float fhi = fminf(fmaxf((wmax + dmax - mu0) * rstep, -4.0f), 68.0f);
        const int ilo = max(__float_as_int(__fadd_rd(flo, 12582912.0f)) - 0x4B400000, -2) >> 1;
        const int ihi = min(__float_as_int(__fadd_ru(fhi, 12582912.0f)) - 0x4B400000, 64) >> 1;
        const float xs = (x - base) * sc;
        const f2 na2 = bc(na);
        f2 phi2 = 0ull, dphi2 = 0ull;
        const f2 xs2 = bc(xs);
#pragma unroll
        for (int gg = 0; gg < 16 / TNRD_PHI_GP; ++gg) {
            if (2 * TNRD_PHI_GP * gg + 2 * TNRD_PHI_GP - 1 >= ilo && 2 * TNRD_PHI_GP * gg <= ihi) {
                // d' of the group's first pair from its constants, later pairs by
                // steps of -2 s2 (one FADD2 each)
                f2 d2 = fma2(pk(-(float)(2 * TNRD_PHI_GP * gg), -(float)(2 * TNRD_PHI_GP * gg + 1)), s2v, xs2);
#pragma unroll
                for (int ip = TNRD_PHI_GP * gg; ip < TNRD_PHI_GP * gg + TNRD_PHI_GP; ++ip) {
                    if (ip > TNRD_PHI_GP * gg) d2 = add2(d2, m2s2);
                    const f2 t2 = mul2(d2, d2);
                    const f2 G2 = pk(ex2_ftz(-lo(t2)), ex2_ftz(-hi(t2)));
                    phi2 = fma2(w2[ip], G2, phi2);
                    dphi2 = fma2(mul2(w2[ip], d2), G2, dphi2);
                    acc2[ip] = fma2(na2, G2, acc2[ip]);
                }
            }
        }
        const float phi = lo(phi2) + hi(phi2), dphi = lo(dphi2) + hi(dphi2);
        // phi = half 0 + half 1 on both lanes of the pair, in that order
        const float phi_o = __shfl_xor_sync(0xffffffffu, phi, 16), dphi_o = __shfl_xor_sync(0xffffffffu, dphi, 16);
        const float phi_t = h ? phi_o + phi : phi + phi_o, dphi_t = h ? dphi_o + dphi : dphi + dphi_o;
        if (valid && h == 0) {
            wo[(long long)f * n + p] = phi_t;
            bo[(long long)f * n + p] = dphi_t * bscale * na;   // -(sum w d G / gamma^2) a
        }
    }
    // block sum of acc: lanes of a half, then warps, in fixed orders
#pragma unroll
    for (int ip = 0; ip < 16; ++ip) {
        float v0 = lo(acc2[ip]), v1 = hi(acc2[ip]);
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
            v0 += __shfl_xor_sync(0xffffffffu, v0, o);
            v1 += __shfl_xor_sync(0xffffffffu, v1, o);
        }
        if ((lane & 15) == 0) {
            red[warp][4 * ip + h] = v0;
            red[warp][4 * ip + 2 + h] = v1;
        }
    }
    __syncthreads();
    if (threadIdx.x < 64) {
        float s = 0.0f;
        for (int w = 0; w < kPhiThreads / 32; ++w) s += red[w][threadIdx.x];
        partial[((long long)f * gridDim.x + blockIdx.x) * 64 + threadIdx.x] = s;
    }
}

// t_f = K_f^T b_f.
template <int m>
__global__ void __launch_bounds__(kGradThreads) adj_b_kernel(GradFilterArgs g, const float *__restrict__ bv,
                                                             float *__restrict__ to) {
    constexpr int r = m / 2;
    __shared__ float sk[m * m];
    const int f = blockIdx.y;
    for (int j = threadIdx.x; j < m * m; j += blockDim.x) sk[j] = g.k[(long long)(g.fi0 + f) * m * m + j];
    __syncthreads();
    const int H = g.H, W = g.W;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < g.n; p += (long long)gridDim.x * blockDim.x) {
        const long long b = p / ((long long)H * W), rr = p - b * H * W;
        const int y = (int)(rr / W), x = (int)(rr - (long long)y * W);
        const bool in = y >= r && y < H - r && x >= r && x < W - r;
        to[(long long)f * g.n + p] = adj_at<m>(bv + (long long)f * g.n + b * H * W, sk, y, x, H, W, in);
    }
}

// gn -= sum_{f < F} t_f, filters in ascending order.
__global__ void __launch_bounds__(kGradThreads) sub_sum_kernel(const float *__restrict__ t, int F, long long n,
                                                               float *__restrict__ gn) {
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
        float v = gn[p];
        for (int f = 0; f < F; ++f) v -= t[(long long)f * n + p];
        gn[p] = v;
    }
}

// partial sums of the filter derivatives: inner b_f(p) E(u)(p - tap), outer
// R1: e(p) E(w_f)(p - tap) (kbar's taps), R2: w_f(p) E(e)(p - tap).
template <int m>
__global__ void __launch_bounds__(kGradThreads) kgrad_pair_kernel(GradFilterArgs g, const float *__restrict__ u,
                                                                  const float *__restrict__ e, int boundary,
                                                                  const float *__restrict__ bv,
                                                                  const float *__restrict__ wv,
                                                                  float *__restrict__ partial) {
    constexpr int r = m / 2, mm = m * m;
    const int f = blockIdx.y, H = g.H, W = g.W;
    float acc[2 * mm];
#pragma unroll
    for (int j = 0; j < 2 * mm; ++j) acc[j] = 0.0f;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < g.n; p += (long long)gridDim.x * blockDim.x) {
        const long long b = p / ((long long)H * W), rr = p - b * H * W;
        const int y = (int)(rr / W), x = (int)(rr - (long long)y * W);
        const bool in = y >= r && y < H - r && x >= r && x < W - r;
        const float bp = bv[(long long)f * g.n + p];
        const float *ub = u + b * H * W;
        const float *wb = wv + (long long)f * g.n + b * H * W;
        const float *eb = e + b * H * W;
        const float op = boundary == 1 ? wb[rr] : eb[rr];     // the weight of the outer sum
        const float *ob = boundary == 1 ? eb : wb;            // the image it correlates with
#pragma unroll
        for (int a = 0; a < m; ++a) {
            const int yy = in ? y - (a - r) : mirror(y - (a - r), H);
#pragma unroll
            for (int c = 0; c < m; ++c) {
                const int xx = in ? x - (c - r) : mirror(x - (c - r), W);
                const long long o = (long long)yy * W + xx;
                acc[a * m + c] = fmaf(bp, ub[o], acc[a * m + c]);
                acc[mm + a * m + c] = fmaf(op, ob[o], acc[mm + a * m + c]);
            }
        }
    }
    block_sum<2 * mm>(acc, partial + ((long long)f * gridDim.x + blockIdx.x) * 2 * mm);
}

// out[f*np + j] = sum_b partial[(f*nblk + b)*np + j] (fixed order, double).
__global__ void __launch_bounds__(kGradThreads) reduce_f_kernel(const float *__restrict__ partial, int nblk, int np,
                                                                double *__restrict__ out, int out_stride,
                                                                int out_off) {
    __shared__ double red[kGradThreads];
    const int f = blockIdx.y, j = blockIdx.x;
    double s = 0.0;
    for (int b = threadIdx.x; b < nblk; b += kGradThreads) s += (double)partial[((long long)f * nblk + b) * np + j];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = kGradThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[(long long)f * out_stride + out_off + j] = red[0];
}

// The same sums with one warp per (j, f): lane l takes blocks l, l + 32, ... in order,
// then a fixed shuffle tree (for the short partial lists of the phi and tensor-core
// filter-gradient kernels: <= a few hundred blocks).
__global__ void __launch_bounds__(32) reduce_f_warp_kernel(const float *__restrict__ partial, int nblk, int np,
                                                          double *__restrict__ out, int out_stride, int out_off) {
    const int f = blockIdx.y, j = blockIdx.x, lane = threadIdx.x;
    double s = 0.0;
    for (int b = lane; b < nblk; b += 32) s += (double)partial[((long long)f * nblk + b) * np + j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[(long long)f * out_stride + out_off + j] = s;
}

// out[j] = sum over blocks of partial[blk * stride + j], j < np, in double: block j
// sums parameter j; thread t takes blocks t, t + 256, ... in order, then a fixed
// shared-memory tree (bitwise reproducible).
__global__ void __launch_bounds__(kGradThreads) reduce_kernel(const float *__restrict__ partial, int nblk, int stride,
                                                              double *__restrict__ out) {
    __shared__ double red[kGradThreads];
    const int j = blockIdx.x;
    double s = 0.0;
    for (int b = threadIdx.x; b < nblk; b += kGradThreads) s += (double)partial[(long long)b * stride + j];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = kGradThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[j] = red[0];
}

int grid_for(long long n, int num_sms) {
    const long long want = (n + kGradThreads - 1) / kGradThreads;
    return (int)std::min<long long>(std::max<long long>(want, 1), (long long)num_sms * 4);
}

}  // namespace

int grad_grid(long long n, int num_sms) { return grid_for(n, num_sms); }

cudaError_t grad_loss(const float *uT, const float *gt, long long gt_ld, int B, int H, int W, float *g,
                      float *partial, int grid, cudaStream_t s) {
    loss_kernel<<<grid, kGradThreads, 0, s>>>(uT, gt, gt_ld, B, H, W, g, partial);
    return cudaGetLastError();
}

cudaError_t grad_bw_prox(const float *ut, const float *f, long long f_ld, int B, int H, int W, float lam, const float *g,
                         float *e, float *gn, float *partial, int grid, cudaStream_t s) {
    bw_prox_kernel<<<grid, kGradThreads, 0, s>>>(ut, f, f_ld, B, H, W, lam, g, e, gn, partial);
    return cudaGetLastError();
}

int grad_chunk_grid(long long n, int F, int num_sms) {
    const long long want = (n + kGradThreads - 1) / kGradThreads;
    const long long cap = std::max<long long>(1, ((long long)num_sms * 4 + F - 1) / F);
    return (int)std::min<long long>(std::max<long long>(want, 1), cap);
}

cudaError_t grad_chunk(const GradChunk &c, cudaStream_t s) {
    GradFilterArgs g{c.k, c.kbar, c.rw, c.grid3, c.fi0, c.m, c.M, c.B, c.H, c.W, (long long)c.B * c.H * c.W};
    const dim3 grid(c.gx, c.F);
    const int mm = c.m * c.m;
#define TNRD_M(NAME, ...)                                                         \
    switch (c.m) {                                                                \
        case 3: NAME<3><<<grid, kGradThreads, 0, s>>>(__VA_ARGS__); break;        \
        case 5: NAME<5><<<grid, kGradThreads, 0, s>>>(__VA_ARGS__); break;        \
        case 7: NAME<7><<<grid, kGradThreads, 0, s>>>(__VA_ARGS__); break;        \
        default: return cudaErrorInvalidValue;                                    \
    }
    if (c.M > 64) return cudaErrorInvalidValue;
    if (c.tc_bf) {  // both forward banks on the tensor cores (all N_k filters in this chunk)
        cudaError_t e = launch_tc_fwdbank(c.m, c.F, c.u, c.tc_bf, c.x, c.B, c.H, c.W, s);
        if (e == cudaSuccess) e = launch_tc_fwdbank(c.m, c.F, c.e, c.tc_bf, c.a, c.B, c.H, c.W, s);
        if (e != cudaSuccess) return e;
        if (c.boundary == 0) {  // R1: Kbar^T e differs from k * E(e) only within r of an edge
            const int r = c.m / 2;
            const long long nb = (long long)c.B * (2LL * r * c.W + 2LL * r * std::max(c.H - 2 * r, 0));
            if (c.F > kBorderMaxF) return cudaErrorInvalidValue;
            const unsigned bgrid = (unsigned)std::max<long long>(1, std::min<long long>((nb + kBorderPix - 1) / kBorderPix, 8192));
            switch (c.m) {
                case 3: adj_border_kernel<3><<<bgrid, kBorderThreads, 0, s>>>(g, c.F, c.e, c.a); break;
                case 5: adj_border_kernel<5><<<bgrid, kBorderThreads, 0, s>>>(g, c.F, c.e, c.a); break;
                case 7: adj_border_kernel<7><<<bgrid, kBorderThreads, 0, s>>>(g, c.F, c.e, c.a); break;
                default: return cudaErrorInvalidValue;
            }
        }
    } else {
        TNRD_M(fwd_pair_kernel, g, c.u, c.e, c.boundary, c.x, c.a)
    }
    {   // phi_all: one full wave of resident blocks (its grid-stride loop then balances)
        // resident blocks per SM, cached per device (it sets the grid and with it the
        // summation order, so it must not depend on which device ran first)
        static int occ_cache[64] = {0};
        int dev = 0;
        cudaGetDevice(&dev);
        int occ = dev < 64 ? occ_cache[dev] : 0;
        if (occ == 0) {
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, phi_all_kernel, kPhiThreads, 0) != cudaSuccess)
                occ = 1;
            if (dev < 64) occ_cache[dev] = occ;
        }
        const int gphi = std::max(1, std::min(c.gx, std::max(1, c.num_sms * std::max(occ, 1) / c.F)));
        phi_all_kernel<<<dim3(gphi, c.F), kPhiThreads, 0, s>>>(g, c.x, c.a, c.w, c.b, c.partial);
        reduce_f_warp_kernel<<<dim3(c.M, c.F), 32, 0, s>>>(c.partial, gphi, 64, c.red, c.red_stride, 2 * mm);
    }
    if (c.tc_ba) {  // gn -= sum_f K_f^T b_f on the tensor cores (all N_k filters in this chunk)
        const cudaError_t e = launch_tc_adjoint(c.m, c.F, c.b, c.tc_ba, c.gn, c.B, c.H, c.W, c.tc_oh, s);
        if (e != cudaSuccess) return e;
    } else {
        TNRD_M(adj_b_kernel, g, c.b, c.t)
        sub_sum_kernel<<<c.gx * c.F, kGradThreads, 0, s>>>(c.t, c.F, g.n, c.gn);
    }
    if (c.tc_kg_nblk > 0) {  // filter gradient as one GEMM over pixels on the tensor cores
        const cudaError_t e = launch_tc_kgrad(c.m, c.F, c.u, c.e, c.b, c.w, c.boundary, c.B, c.H, c.W, c.partial,
                                              c.tc_kg_nblk, s);
        if (e != cudaSuccess) return e;
        reduce_f_warp_kernel<<<dim3(2 * mm, c.F), 32, 0, s>>>(c.partial, c.tc_kg_nblk, 2 * mm, c.red,
                                                                     c.red_stride, 0);
    } else {
        TNRD_M(kgrad_pair_kernel, g, c.u, c.e, c.boundary, c.b, c.w, c.partial)
        reduce_f_kernel<<<dim3(2 * mm, c.F), kGradThreads, 0, s>>>(c.partial, c.gx, 2 * mm, c.red, c.red_stride, 0);
    }
#undef TNRD_M
    return cudaGetLastError();
}

cudaError_t grad_reduce(const float *partial, int nblk, int stride, int np, double *out, cudaStream_t s) {
    if (np > 0) reduce_kernel<<<np, kGradThreads, 0, s>>>(partial, nblk, stride, out);
    return cudaGetLastError();
}

}  // namespace tnrd
