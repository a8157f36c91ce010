// Internal declarations shared by the host ABI (tnrd_api.cpp) and the sm_100a
// kernels (tnrd_kernels.cu).  Not part of the public ABI (include/tnrd.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace tnrd {

// ---------------------------------------------------------------------------
// Per-stage parameter block (device global memory, copied to shared memory by
// every CTA).  Per filter i, `pstride` floats (multiple of 4):
//
//   taps  [K][K8]   k_i row-major, each row zero padded to K8 = roundup(K, 4)
//                   floats so that a tap row is whole float4s
//   fc    [8]       { a_s, two_sg, inv_ustep, n_units, yclamp, 0, 0, 0 }
//   units [n_units][UNIT]
//
// phi evaluation.  With x = (v - mu0)/step the response in
// centre units, rho = step/gamma and sg = rho*sqrt(log2(e)/2):
//
//  MODE_HORNER: unit b covers centres j = 8b..8b+7, expanded from its first
//    centre.  t = sg*(x - 8b) = a_s*v + ct_b,
//      G = 2^(-t^2) = exp(-rho^2 (x-8b)^2 / 2),   R = 2^(two_sg*t) = exp(rho^2 (x - 8b)),
//      sum_{e=0..7} w_{8b+e} exp(-rho^2 (x-8b-e)^2/2) = G * sum_{e=0..7} c_e R^e,
//      c_e = w_{8b+e} exp(-rho^2 e^2 / 2)                (exact identity)
//    unit layout (12 floats): { ct_b, c_0, ..., c_7, 0, 0, 0 }
//    fc[4] = yrmax: R's exponent is clamped at yrmax = two_sg * tclamp with
//    sum|c| * 2^(7 yrmax) <= 2^126 (no overflow of R^7).  Where the clamp binds
//    (t > tclamp) every term of the block is below 2^-20 of its weight: the host
//    requires tclamp >= 7 sg + 4.5 or uses MODE_DIRECT.
//  MODE_DIRECT (any rho): unit j is centre j: ys = a_s*v + cs_j, term w_j 2^(-ys^2)
//    unit layout (4 floats): { cs_j, w_j, 0, 0 }
//
//  G (or the direct term) is exactly 0 in fp32 (ex2.approx.ftz flushes results
//  below 2^-126) once |ys| > 11.2249; the kernel evaluates, per warp, the units
//  whose |ys| <= kWindow for some lane, so every unit it skips contributes
//  exactly 0 as well: the result does not depend on which pixels share a warp.
// ---------------------------------------------------------------------------
//  MODE_TABLE (TNRD_PHI_TABLE, reported separately): per filter a cubic Hermite
//    table on nodes x_k = x_lo + k/kTabPerCentre, x_lo = -kTabPad, built on the
//    host in double from the exact phi and phi'; interval k holds {c0, c1, c2, c3}
//    with phi(x_k + f/S) ~= c0 + f (c1 + f (c2 + f c3)), f in [0, 1).  Interval
//    n_int (one past the last) is all zeros and serves every out-of-range x.
//    fc = { a_t = S/step, b_t, n_int, b_lo, ... } with b_t + b_lo = -(mu0/step + x_lo) * S
//    split into fp32 hi/lo words: xs = a_t v + b_t, k = floor(xs),
//    f = fma(v, a_t, b_t - k) + b_lo (b_t - k is exact).
enum { MODE_HORNER = 0, MODE_DIRECT = 1, MODE_TABLE = 2 };
constexpr int kTabPerCentre = 16;     // table intervals per RBF centre spacing
constexpr int kTabPad = 14;           // centres of zero-free margin on each side
constexpr int kHornerUnit = 12;
constexpr int kDirectUnit = 4;
constexpr int kFc = 8;                // floats of per-filter constants
constexpr float kWindow = 11.25f;     // > sqrt(126): all nonzero G lie inside
// Per-lane left cut of the Horner units: a lane with t < -kCutT
// sees only block terms below 2^-30.25 of their weight, so G's exponent is pushed
// below -126 there (an exact zero, decided per lane, so skipping stays warp-
// independent); bitwise unchanged where the cut does not bind.
constexpr float kCutT = 5.5f, kCutBig = 1048576.0f;


__host__ __device__ constexpr int tap_pitch(int K) { return (K + 3) / 4 * 4; }
__host__ __device__ constexpr int tap_floats(int K) { return K * tap_pitch(K); }

struct Image {
    const float *ptr;      // element (b, y, x) at ptr + b*img_stride + (y - row_base)*ld + x
    long long ld;
    long long img_stride;
    int row_base;
};

struct StageArgs {
    const float *params;   // this stage's parameter block (Nk * pstride floats)
    Image u_in;            // u_t  (rows [avail_lo, avail_hi) addressable)
    Image f;               // f    (rows [y_begin, y_end) addressable)
    float *u_out;          // u_{t+1}, addressed like out_* below
    float *ut_out;         // optional (training tape): ut = u - d, addressed like u_out
    long long out_ld;
    long long out_img_stride;
    int out_row_base;
    int H, W;              // global image size (mirror at rows 0/H, cols 0/W)
    int y_begin, y_end;    // output rows of this launch
    int avail_lo, avail_hi;// rows of u_in that may be read
    int Nk, pstride, mode;
    int boundary;          // 0 = R1, 1 = R2
    int reaction;          // tnrd_reaction
    float lambda;
    const float4 *table;   // MODE_TABLE: this stage's tables, filter i at table + i*table_stride
    int table_stride;      // float4s per filter (n_int + 1)
    // tiling (filled by launch_stage): tiles in x-fastest, then y, then image order
    int tiles_x, tiles_y, n_tiles;
    // tensor-core engine (tnrd_tc.cu): output rows per tile and floats of the
    // stage's operand block at `params` (pstride = phi floats per filter there)
    int tc_oh, tc_par_floats;
    int tc_rn;                 // tensor engine: round-to-nearest operand split (gradient tape)
};

// Kernel launchers (tnrd_kernels.cu).  Return cudaSuccess or the launch error.
size_t stage_smem_bytes(int ksize, int tile, int Nk, int pstride);
int choose_tile(int ksize, int B, int H, int W, int num_sms);
cudaError_t launch_stage(int ksize, int tile, StageArgs &a, int B, cudaStream_t s);
cudaError_t launch_debug_phi(const float *params, int pstride, int mode, const float4 *table, int ksize, int i,
                             const float *v, float *out, long long n, cudaStream_t s);
cudaError_t launch_debug_prox(const float *ut, const float *f, float lambda, float *out,
                              long long n, cudaStream_t s);
cudaError_t launch_copy_rows(const float *src, long long src_ld, float *dst, long long dst_ld,
                             int rows, int W, cudaStream_t s);

// Tensor-core engine (tnrd_tc.cu): 3xTF32 tcgen05 GEMMs for both filter banks.
// Stage operand block (floats), built by the host (tnrd_api.cpp, pack_tc_stage):
//   bf_hi, bf_lo [Nk x KTP]  k_i taps, UMMA K-major no-swizzle layout (tc_b_index)
//   ba_hi, ba_lo [NZ x Nk]   the same taps transposed (tap-major rows)
//   phi  [Nk/2][tc_pair_stride(M)]  Horner phi of filter pairs (2p, 2p+1), each
//        value interleaved {filter 2p, filter 2p+1} so that every constant pair is
//        one aligned 64-bit operand of fma.rn.f32x2:
//          header {a_s, a_s', two_sg, two_sg'} {A, A', B0, B0'} {B1, B1', yrmax, yrmax'} {NB, 0, 0, 0}
//            (unit range of a warp: u0 = ceil(A vmin + B0), u1 = floor(A vmax + B1))
//          unit b {ct, ct', c0, c0'} {c1, c1', c2, c2'} {c3, c3', c4, c4'} {c5, c5', c6, c6'} {c7, c7', 0, 0}
//        for b = 0..NB-1, then NB all-zero units (so u0 + j needs no bound check).
// KTP = roundup(k*k, 8) (GEMM K of the forward bank), NZ = max(16, KTP).
constexpr int kTcVW = 64;       // v-region columns per tile (an M = 128 block is two rows)
constexpr int kTcPairHdr = 16, kTcPairUnit = 20;
__host__ __device__ constexpr int tc_ktp(int K) { return (K * K + 7) / 8 * 8; }
__host__ __device__ constexpr int tc_nz(int K) { return tc_ktp(K) < 16 ? 16 : tc_ktp(K); }
__host__ __device__ constexpr int tc_pair_stride(int M) { return kTcPairHdr + 2 * ((M + 7) / 8) * kTcPairUnit; }
__host__ __device__ constexpr int tc_par_floats(int K, int Nk, int M) {
    return 2 * Nk * tc_ktp(K) + 2 * tc_nz(K) * Nk + (Nk / 2) * tc_pair_stride(M);
}
// element (row n, column k) of a rows x kdim K-major operand (8-row x 4-float core matrices)
__host__ __device__ constexpr int tc_b_index(int n, int k, int kdim) {
    return ((n >> 3) * (kdim >> 2) + (k >> 2)) * 32 + (n & 7) * 4 + (k & 3);
}
bool tc_supported(int ksize, int Nk);
size_t tc_min_smem_bytes(int ksize, int Nk, int par_floats);
int tc_choose_rows(int ksize, int B, int H, int W, int num_sms);
cudaError_t launch_stage_tc(int ksize, StageArgs &a, int B, cudaStream_t s);

// Training-gradient kernels (tnrd_grad.cu); all images dense [B][H][W] unless an ld is given.
int grad_grid(long long n, int num_sms);
cudaError_t grad_loss(const float *uT, const float *gt, long long gt_ld, int B, int H, int W, float *g,
                      float *partial, int grid, cudaStream_t s);
cudaError_t grad_bw_prox(const float *ut, const float *f, long long f_ld, int B, int H, int W, float lam,
                         const float *g, float *e, float *gn, float *partial, int grid, cudaStream_t s);
// One chunk of F filters of stage t (filters t*Nk + fi0 .. + F): every per-filter
// step of the backward in 7 launches (tnrd_grad.cu).  Per-filter images x, a, b, w, t
// are [F][B*H*W]; red[f*red_stride + ...] receives {inner taps, outer taps, -a G_j}.
struct GradChunk {
    const float *k, *kbar, *rw, *grid3;
    int fi0, F, m, M, B, H, W, boundary, gx;
    const float *u, *e;
    float *gn, *x, *a, *b, *w, *t, *partial;
    double *red;
    int red_stride;
    const float *tc_ba;   // stage's tensor-engine adjoint operands (ba_hi, ba_lo) or null
    const float *tc_bf;   // stage's tensor-engine forward operands (bf_hi, bf_lo) or null
    int tc_oh;            // tile rows for the tensor adjoint bank
    int tc_kg_nblk;       // > 0: the filter gradient on the tensor cores with this many CTAs
    int num_sms;          // of the device (grid sizing)
};
// gn -= sum_f K_f^T b_f over all N_k filters of a stage on the tensor cores (tnrd_tc.cu):
// b [N_k][B*H*W] dense, ba = the stage's adjoint operand block (tc_par layout).
cudaError_t launch_tc_adjoint(int ksize, int Nk, const float *b, const float *ba, float *gn, int B, int H, int W,
                              int oh, cudaStream_t s);
// out[f][p] = (k_f * E(in))(p), the forward bank with the symmetric extension, for all
// N_k filters on the tensor cores (tnrd_tc.cu): in [B][H][W] dense, out [N_k][B*H*W],
// bf = the stage's forward operand block (bf_hi, bf_lo).
cudaError_t launch_tc_fwdbank(int ksize, int Nk, const float *in, const float *bf, float *out, int B, int H, int W,
                              cudaStream_t s);
// The filter-gradient sums (kgrad_pair_kernel's inner / outer) for all N_k filters
// as a 3xTF32 GEMM over pixels (tnrd_tc.cu): partial[(f*nblk + blk)*2k^2 + j],
// nblk = tc_kgrad_blocks(...) CTAs, summed by reduce_f_kernel.
int tc_kgrad_blocks(int B, int H, int W, int num_sms);
cudaError_t launch_tc_kgrad(int ksize, int Nk, const float *u, const float *e, const float *b, const float *w,
                            int boundary, int B, int H, int W, float *partial, int nblk, cudaStream_t s);
int grad_chunk_grid(long long n, int F, int num_sms);
cudaError_t grad_chunk(const GradChunk &c, cudaStream_t s);
cudaError_t grad_reduce(const float *partial, int nblk, int stride, int np, double *out, cudaStream_t s);

// Data generation and evaluation (tnrd_data.cu).
cudaError_t data_sample_poisson(const float *u, float *f, int B, int H, int W, long long ld, uint64_t seed,
                                int *bad, int num_sms, cudaStream_t s);
int data_sq_err_blocks(long long per_image, int num_sms);
cudaError_t data_sq_err(const float *u, const float *c, int B, int H, int W, long long ld, double *partial,
                        int blocks, cudaStream_t s);
// x -> x * (peak_b / max_b(x)) per image (exactly peak_b at the max); mx [B] scratch,
// *bad set if an input is negative or NaN.
cudaError_t data_scale_to_peak(const float *x, float *out, int B, int H, int W, long long ld, const float *peak_dev,
                               unsigned *mx, int *bad, int num_sms, cudaStream_t s);
// SSIM partial sums over the valid 11 x 11 windows: partial[b * blocks + k]
int data_ssim_blocks(long long windows, int num_sms);
cudaError_t data_ssim(const float *x, const float *y, int B, int H, int W, long long ld, const double *scale_dev,
                      double *partial, int blocks, cudaStream_t s);

}  // namespace tnrd
