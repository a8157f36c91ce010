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

// out = conv2d_sym(x, k): out(p) = sum_{a,b} k[a][b] x(mirror(p - (a - r, b - r))).
__global__ void __launch_bounds__(kGradThreads) conv_sym_kernel(const float *__restrict__ x, const float *__restrict__ k,
                                                                int m, int B, int H, int W, float *__restrict__ out) {
    const long long n = (long long)B * H * W;
    const int r = m / 2;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
        const long long b = p / ((long long)H * W), rr = p - b * H * W;
        const int y = (int)(rr / W), xq = (int)(rr - (long long)y * W);
        const float *xb = x + b * H * W;
        float s = 0.0f;
        for (int a = 0; a < m; ++a) {
            const float *row = xb + (long long)mirror(y - (a - r), H) * W;
            for (int c = 0; c < m; ++c) s = fmaf(k[a * m + c], row[mirror(xq - (c - r), W)], s);
        }
        out[p] = s;
    }
}

// Exact transpose of conv2d_sym: out(q) = sum_p y(p) sum_{taps} k[tap] [mirror(p - tap) == q],
// gathered per output: along each axis the sources are q + d, d - 1 - q and 2n - 1 - q + d.
// mode 0: out = K^T y;  mode 1: out -= K^T y.
__global__ void __launch_bounds__(kGradThreads) conv_adjoint_kernel(const float *__restrict__ yv,
                                                                    const float *__restrict__ k, int m, int B, int H,
                                                                    int W, float *__restrict__ out, int mode) {
    const long long n = (long long)B * H * W;
    const int r = m / 2;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
        const long long b = p / ((long long)H * W), rr = p - b * H * W;
        const int qy = (int)(rr / W), qx = (int)(rr - (long long)qy * W);
        const float *yb = yv + b * H * W;
        float s = 0.0f;
        for (int a = 0; a < m; ++a) {
            const int dy = a - r;
            const int cy[3] = {qy + dy, dy - 1 - qy, 2 * H - 1 - qy + dy};
            for (int iy = 0; iy < 3; ++iy) {
                const int py = cy[iy];
                if (py < 0 || py >= H || mirror(py - dy, H) != qy) continue;
                if (iy > 0 && py == cy[0]) continue;
                if (iy > 1 && py == cy[1]) continue;
                for (int c = 0; c < m; ++c) {
                    const int dx = c - r;
                    const int cx[3] = {qx + dx, dx - 1 - qx, 2 * W - 1 - qx + dx};
                    for (int ix = 0; ix < 3; ++ix) {
                        const int px = cx[ix];
                        if (px < 0 || px >= W || mirror(px - dx, W) != qx) continue;
                        if (ix > 0 && px == cx[0]) continue;
                        if (ix > 1 && px == cx[1]) continue;
                        s = fmaf(k[a * m + c], yb[(long long)py * W + px], s);
                    }
                }
            }
        }
        out[p] = mode ? out[p] - s : s;
    }
}

// w = phi(x), b = phi'(x) a; partial sums of -a G_j(x), j in [j0, j0 + 32).
__global__ void __launch_bounds__(kGradThreads) phi_point_kernel(const float *__restrict__ xv, const float *__restrict__ av,
                                                                 long long n, const float *__restrict__ rw, int M,
                                                                 float mu0, float step, float gamma, int j0,
                                                                 float *__restrict__ wout, float *__restrict__ bout,
                                                                 float *__restrict__ partial /* [grid][32] */) {
    float acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = 0.0f;
    const float inv2g2 = 1.0f / (2.0f * gamma * gamma), invg2 = 1.0f / (gamma * gamma);
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
        const float x = xv[p], a = av[p];
        if (j0 == 0) {
            float phi = 0.0f, dphi = 0.0f;
            for (int j = 0; j < M; ++j) {
                const float d = x - fmaf((float)j, step, mu0);
                const float G = __expf(-d * d * inv2g2);
                phi = fmaf(rw[j], G, phi);
                dphi = fmaf(-rw[j] * d * invg2, G, dphi);
            }
            wout[p] = phi;
            bout[p] = dphi * a;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            if (j0 + j < M) {
                const float d = x - fmaf((float)(j0 + j), step, mu0);
                acc[j] = fmaf(-a, __expf(-d * d * inv2g2), acc[j]);
            }
        }
    }
    block_sum<32>(acc, partial + (long long)blockIdx.x * 32);
}

// partial sums of e(p) E(x)(p - (a - r, c - r)) for every tap (a, c).
template <int MM>
__global__ void __launch_bounds__(kGradThreads) kernel_grad_kernel(const float *__restrict__ x, const float *__restrict__ e,
                                                                   int B, int H, int W, float *__restrict__ partial) {
    constexpr int m = MM, r = MM / 2;
    float acc[m * m];
#pragma unroll
    for (int j = 0; j < m * m; ++j) acc[j] = 0.0f;
    const long long n = (long long)B * H * W;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
        const long long b = p / ((long long)H * W), rr = p - b * H * W;
        const int y = (int)(rr / W), xq = (int)(rr - (long long)y * W);
        const float ev = e[p];
        const float *xb = x + b * H * W;
#pragma unroll
        for (int a = 0; a < m; ++a) {
            const float *row = xb + (long long)mirror(y - (a - r), H) * W;
#pragma unroll
            for (int c = 0; c < m; ++c) acc[a * m + c] = fmaf(ev, row[mirror(xq - (c - r), W)], acc[a * m + c]);
        }
    }
    block_sum<m * m>(acc, partial + (long long)blockIdx.x * m * m);
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

cudaError_t grad_conv_sym(const float *x, const float *k, int m, int B, int H, int W, float *out, int grid,
                          cudaStream_t s) {
    conv_sym_kernel<<<grid, kGradThreads, 0, s>>>(x, k, m, B, H, W, out);
    return cudaGetLastError();
}

cudaError_t grad_conv_adjoint(const float *y, const float *k, int m, int B, int H, int W, float *out, int mode,
                              int grid, cudaStream_t s) {
    conv_adjoint_kernel<<<grid, kGradThreads, 0, s>>>(y, k, m, B, H, W, out, mode);
    return cudaGetLastError();
}

cudaError_t grad_phi_point(const float *x, const float *a, long long n, const float *rw, int M, float mu0, float step,
                           float gamma, int j0, float *wout, float *bout, float *partial, int grid, cudaStream_t s) {
    phi_point_kernel<<<grid, kGradThreads, 0, s>>>(x, a, n, rw, M, mu0, step, gamma, j0, wout, bout, partial);
    return cudaGetLastError();
}

cudaError_t grad_kernel(const float *x, const float *e, int m, int B, int H, int W, float *partial, int grid,
                        cudaStream_t s) {
    switch (m) {
        case 3: kernel_grad_kernel<3><<<grid, kGradThreads, 0, s>>>(x, e, B, H, W, partial); break;
        case 5: kernel_grad_kernel<5><<<grid, kGradThreads, 0, s>>>(x, e, B, H, W, partial); break;
        case 7: kernel_grad_kernel<7><<<grid, kGradThreads, 0, s>>>(x, e, B, H, W, partial); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t grad_reduce(const float *partial, int nblk, int stride, int np, double *out, cudaStream_t s) {
    if (np > 0) reduce_kernel<<<np, kGradThreads, 0, s>>>(partial, nblk, stride, out);
    return cudaGetLastError();
}

}  // namespace tnrd
