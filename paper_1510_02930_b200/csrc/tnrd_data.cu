// Steps either side of the inference path on sm_100a:
//
//   sample_poisson  f ~ Poisson(u) per pixel (P Eq.1, l.103-111; u = 0 gives 0),
//                   counter-based: Philox4x32-10 (Salmon et al., SC'11) keyed by the
//                   seed, counter = flat pixel index; U in [0,1) from 53 bits; exact
//                   inversion by sequential search of the CDF in double with a fixed
//                   fma-only exp, so the integer decision is taken in the same
//                   precision and operations as the oracle's (oracle_poisson_draw).
//   psnr            10 log10(peak^2 / MSE(u, clean)) per image (reading C15), the
//                   squared errors summed in double in a fixed order.
#include "tnrd_internal.h"

#include <algorithm>
#include <cmath>
#include <stdint.h>

namespace tnrd {
namespace {

__device__ __forceinline__ void philox4x32_10(uint64_t counter, uint64_t seed, uint32_t (&c)[4]) {
    c[0] = (uint32_t)counter; c[1] = (uint32_t)(counter >> 32); c[2] = 0u; c[3] = 0u;
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
        const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

// exp(x), x in [-745, 0]: Cody-Waite reduction with hi/lo ln2, degree-13 Taylor
// Horner in fma, times 2^n -- only IEEE fma / mul / add (bitwise as oracle_exp_fixed).
__device__ __forceinline__ double exp_fixed(double x) {
    if (x < -745.0) return 0.0;
    const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
    const double n = nearbyint(__dmul_rn(x, 1.44269504088896338700e+00));
    const double r = __fma_rn(-n, ln2_lo, __fma_rn(-n, ln2_hi, x));
    const double inv[13] = {1.0 / 479001600.0, 1.0 / 39916800.0, 1.0 / 3628800.0, 1.0 / 362880.0, 1.0 / 40320.0,
                            1.0 / 5040.0, 1.0 / 720.0, 1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0, 0.5, 1.0, 1.0};
    double p = 1.0 / 6227020800.0;
#pragma unroll
    for (int i = 0; i < 13; ++i) p = __fma_rn(p, r, inv[i]);
    return ldexp(p, (int)n);
}

__global__ void sample_poisson_kernel(const float *__restrict__ u, float *__restrict__ f, int B, int H, int W,
                                      long long ld, uint64_t seed, int *__restrict__ bad) {
    const long long n = (long long)B * H * W;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long b = i / ((long long)H * W), r = i - b * H * W;
        const int y = (int)(r / W), x = (int)(r - (long long)y * W);
        const long long o = b * H * ld + (long long)y * ld + x;
        const double m = (double)u[o];
        double k = 0.0;
        if (!(m >= 0.0)) {
            atomicExch(bad, 1);  // negative or NaN mean
        } else if (m > 0.0) {
            uint32_t w[4];
            philox4x32_10((uint64_t)i, seed, w);
            const double U = __dmul_rn(__fma_rn((double)w[0], 2097152.0, (double)(w[1] >> 11)),
                                       1.0 / 9007199254740992.0);
            double p = exp_fixed(-m), F = p;
            // same rounding sequence as the oracle: (m + 40 sqrt(m)) + 40
            const double kmax = floor(__dadd_rn(__dadd_rn(m, __dmul_rn(40.0, sqrt(m))), 40.0));
            while (U >= F && k < kmax) {
                k += 1.0;
                p = __dmul_rn(p, __ddiv_rn(m, k));
                F = __dadd_rn(F, p);
            }
        }
        f[o] = (float)k;
    }
}

__global__ void sq_err_kernel(const float *__restrict__ u, const float *__restrict__ c, int H, int W, long long ld,
                              double *__restrict__ partial /* [B][gridDim.x] */) {
    __shared__ double red[256];
    const int b = blockIdx.y;
    const long long n = (long long)H * W;
    double s = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int y = (int)(i / W), x = (int)(i - (long long)y * W);
        const long long o = (long long)b * H * ld + (long long)y * ld + x;
        const double d = (double)u[o] - (double)c[o];
        s = __fma_rn(d, d, s);
    }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[(long long)b * gridDim.x + blockIdx.x] = red[0];
}

// Peak scaling (S l.351-358): per-image max as the largest fp32 bit pattern (the
// inputs are non-negative, so the integer order is the float order; atomicMax
// makes it exact and order-independent), a negative or NaN input flags `bad`.
__global__ void image_max_kernel(const float *__restrict__ x, int H, int W, long long ld,
                                 unsigned *__restrict__ mx /* [B] */, int *bad) {
    const int b = blockIdx.y;
    const long long n = (long long)H * W;
    unsigned m = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int y = (int)(i / W), xx = (int)(i - (long long)y * W);
        const float v = x[(long long)b * H * ld + (long long)y * ld + xx];
        if (!(v >= 0.0f)) *bad = 1;
        m = max(m, __float_as_uint(v));
    }
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(mx + b, m);
}
// out = x * (peak / max), exactly peak where x == max (the oracle's operations in fp32)
__global__ void scale_kernel(const float *__restrict__ x, float *__restrict__ out, int H, int W, long long ld,
                             const unsigned *__restrict__ mx, const float *__restrict__ peak /* device [B] */) {
    const int b = blockIdx.y;
    const long long n = (long long)H * W;
    const float m = __uint_as_float(mx[b]), pk = peak[b], r = __fdiv_rn(pk, m);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int y = (int)(i / W), xx = (int)(i - (long long)y * W);
        const long long o = (long long)b * H * ld + (long long)y * ld + xx;
        const float v = x[o];
        out[o] = v == m ? pk : __fmul_rn(v, r);
    }
}

// SSIM (S l.381-389; reading M2): one thread per valid 11 x 11 window (top-left
// corner (i, j)), the window's Gaussian-weighted moments of the 255/peak-rescaled
// images in double (weights g[a] g[b], g the normalised 1-D Gaussian, sigma 1.5),
// the local SSIM, then a fixed-order block sum per (block, image).
constexpr int kSsimWin = 11;
__constant__ double c_ssim_g[kSsimWin];
__global__ void ssim_kernel(const float *__restrict__ x, const float *__restrict__ y, int H, int W, long long ld,
                            const double *__restrict__ scale /* [B]: 255 / peak */, double *__restrict__ partial) {
    __shared__ double red[256];
    const int b = blockIdx.y;
    const int VW = W - kSsimWin + 1;
    const long long nv = (long long)(H - kSsimWin + 1) * VW;
    const double sc = scale[b], C1 = (0.01 * 255.0) * (0.01 * 255.0), C2 = (0.03 * 255.0) * (0.03 * 255.0);
    const float *xb = x + (long long)b * H * ld, *yb = y + (long long)b * H * ld;
    double acc = 0.0;
    for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(v / VW), j = (int)(v - (long long)i * VW);
        double mx = 0, my = 0, xx = 0, yy = 0, xy = 0;
        for (int a = 0; a < kSsimWin; ++a) {
            const float *xr = xb + (long long)(i + a) * ld + j, *yr = yb + (long long)(i + a) * ld + j;
#pragma unroll
            for (int c = 0; c < kSsimWin; ++c) {
                const double w = c_ssim_g[a] * c_ssim_g[c];
                const double xv = sc * (double)__ldg(xr + c), yv = sc * (double)__ldg(yr + c);
                mx = fma(w, xv, mx);
                my = fma(w, yv, my);
                xx = fma(w * xv, xv, xx);
                yy = fma(w * yv, yv, yy);
                xy = fma(w * xv, yv, xy);
            }
        }
        const double vx = xx - mx * mx, vy = yy - my * my, cxy = xy - mx * my;
        acc += ((2 * mx * my + C1) * (2 * cxy + C2)) / ((mx * mx + my * my + C1) * (vx + vy + C2));
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[(long long)b * gridDim.x + blockIdx.x] = red[0];
}

}  // namespace

cudaError_t data_scale_to_peak(const float *x, float *out, int B, int H, int W, long long ld, const float *peak_dev,
                               unsigned *mx, int *bad, int num_sms, cudaStream_t s) {
    const int blocks = data_sq_err_blocks((long long)H * W, num_sms);
    cudaError_t e = cudaMemsetAsync(mx, 0, sizeof(unsigned) * (size_t)B, s);
    if (e != cudaSuccess) return e;
    image_max_kernel<<<dim3(blocks, B), 256, 0, s>>>(x, H, W, ld, mx, bad);
    scale_kernel<<<dim3(blocks, B), 256, 0, s>>>(x, out, H, W, ld, mx, peak_dev);
    return cudaGetLastError();
}

int data_ssim_blocks(long long windows, int num_sms) {
    return (int)std::max<long long>(1, std::min<long long>((windows + 255) / 256, (long long)num_sms * 4));
}

cudaError_t data_ssim(const float *x, const float *y, int B, int H, int W, long long ld, const double *scale_dev,
                      double *partial, int blocks, cudaStream_t s) {
    static bool init[64] = {false};   // per device: the normalised 1-D Gaussian (host, double)
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 64) return cudaErrorInvalidDevice;
    if (!init[dev]) {
        double g[kSsimWin], sum = 0.0;
        for (int a = 0; a < kSsimWin; ++a) {
            const double d = a - kSsimWin / 2;
            g[a] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
            sum += g[a];
        }
        for (int a = 0; a < kSsimWin; ++a) g[a] /= sum;
        cudaError_t e = cudaMemcpyToSymbol(c_ssim_g, g, sizeof g);
        if (e != cudaSuccess) return e;
        init[dev] = true;
    }
    ssim_kernel<<<dim3(blocks, B), 256, 0, s>>>(x, y, H, W, ld, scale_dev, partial);
    return cudaGetLastError();
}

cudaError_t data_sample_poisson(const float *u, float *f, int B, int H, int W, long long ld, uint64_t seed, int *bad,
                                int num_sms, cudaStream_t s) {
    const long long n = (long long)B * H * W;
    const int grid = (int)std::min<long long>((n + 255) / 256, (long long)num_sms * 16);
    if (n > 0) sample_poisson_kernel<<<grid, 256, 0, s>>>(u, f, B, H, W, ld, seed, bad);
    return cudaGetLastError();
}

int data_sq_err_blocks(long long per_image, int num_sms) {
    return (int)std::max<long long>(1, std::min<long long>((per_image + 255) / 256, (long long)num_sms * 2));
}

cudaError_t data_sq_err(const float *u, const float *c, int B, int H, int W, long long ld, double *partial,
                        int blocks, cudaStream_t s) {
    sq_err_kernel<<<dim3(blocks, B), 256, 0, s>>>(u, c, H, W, ld, partial);
    return cudaGetLastError();
}

}  // namespace tnrd
