/*
 * tnrd.h -- C ABI of libtnrd.so: B200-native (sm_100a) inference pass of the
 * trained nonlinear reaction-diffusion Poisson denoiser TRDPD (Feng & Chen,
 * arXiv 1510.02930).  "P l.N" cites PAPER.md, "S l.N" SPEC.md.
 *
 * The operation (P Eq.13, l.326-333; Eq.3 l.134-149):
 *
 *     u_0 = f                                         (P l.136, l.148)
 *     for t = 0..T-1:
 *        ut      = u_t - sum_{i<N_k} kbar_i^t * phi_i^t(k_i^t * u_t)   (tau = 1, l.333)
 *        u_{t+1} = (ut - lam_t + sqrt((ut - lam_t)^2 + 4 lam_t f)) / 2 (Eq.12, l.318-322)
 *
 *   "*" is true 2-D convolution with the symmetric (half-sample mirror)
 *   boundary (P l.302; S l.73), kbar_i the 180-degree rotation of k_i
 *   (P l.143-144), and phi_i^t(z) = sum_{j<M} w_ij exp(-(z - mu_ij)^2 / (2 gamma_i^2)),
 *   mu_ij = mu0_i + j*step_i: a Gaussian-RBF mixture on uniform centres
 *   (P l.145-146 leaves phi free; S l.104-107; BASELINE.json north_star).
 *
 * Arithmetic is IEEE fp32 on the device (DESIGN.md §5 states the error budget
 * against the double-precision oracle: max|du| <= 1e-4 * peak).
 *
 * Conventions for every entry point:
 *   - images are row-major fp32, element (b, y, x) at ptr[b*H*ld + y*ld + x];
 *     ld (in floats) >= W;
 *   - pointers named *_dev are device pointers on the handle's device; *_host
 *     are host pointers (pinned or pageable);
 *   - calls are stream-ordered on `cuda_stream` (a cudaStream_t, NULL = legacy
 *     default stream) and return after enqueueing, except where stated;
 *   - errors are reported by return code only; nothing aborts or throws across
 *     the ABI; tnrd_last_error(h) returns a message for the last failure on h.
 *   - a handle is not thread-safe: one host thread at a time per handle.
 */
#ifndef TNRD_H_
#define TNRD_H_

#ifdef __cplusplus
extern "C" {
#endif

#define TNRD_ABI_VERSION 1

#if defined(__GNUC__)
#define TNRD_API __attribute__((visibility("default")))
#else
#define TNRD_API
#endif

typedef struct tnrd_handle tnrd_handle;

typedef enum {
    TNRD_OK = 0,
    TNRD_EINVAL = 1,       /* invalid argument (value, size, alignment, aliasing)       */
    TNRD_ESTATE = 2,       /* handle state: stage params unset, comm not initialised    */
    TNRD_ENOMEM = 3,       /* device or host allocation failed                          */
    TNRD_ECUDA = 4,        /* CUDA runtime error (message in tnrd_last_error)           */
    TNRD_ENCCL = 5,        /* NCCL error or NCCL library not loadable                   */
    TNRD_EUNSUPPORTED = 6  /* valid request this build does not implement               */
} tnrd_status;

typedef enum {
    /* R1 (default): explicit rotated-kernel convolution of the symmetrically
     * extended phi response, P l.302-311 ("revise the above formulation as
     * explicit convolutions", nabla F = sum kbar_i * phi_i(k_i * u)). */
    TNRD_BC_SYMMETRIC_EXPLICIT = 0,
    /* R2: exact transpose K_i^T of the symmetric-boundary convolution
     * (P l.295-301; S l.57-65).  Differs from R1 only in the outer r = k/2 pixels. */
    TNRD_BC_SYMMETRIC_ADJOINT = 1
} tnrd_boundary;

typedef enum {
    TNRD_PHI_EXACT = 0,    /* exact RBF sum (blocked Horner)            */
    TNRD_PHI_TABLE = 1     /* tabulated phi: per-filter cubic Hermite table, 16 intervals
                              per centre, built on the host in double from the exact phi
                              (DESIGN.md §5.6); an optional variant, reported separately */
} tnrd_phi_mode;

typedef enum {
    /* Poisson denoising (the method): proximal step of P Eq.12-13 (l.313-333). */
    TNRD_REACTION_POISSON_PROX = 0,
    /* Gaussian denoising: P Eq.3 (l.134-141) with psi(u_t, f) = lambda (u_t - f),
     * i.e. lambda A^T (A u - f) with A = I (l.150-158). */
    TNRD_REACTION_GAUSSIAN = 1,
    /* Ablation: the direct Poisson gradient psi = lambda (1 - f / u_t) that the
     * paper rejects (l.247-252); f / u_t is taken as 0 where f = 0.  Not
     * positivity preserving; undefined (IEEE inf/NaN) where u_t = 0 < f. */
    TNRD_REACTION_POISSON_GRADIENT = 2
} tnrd_reaction;

/* Execution engine of the stage kernel (tnrd_set_engine).  Both compute P Eq.13
 * in fp32 storage with the same phi and reaction; they differ in the two filter-bank
 * contractions (P l.137, l.309-311):
 *   FP32:   fp32 FMAs on the CUDA cores (tnrd_kernels.cu);
 *   TENSOR: tcgen05 tensor-core GEMMs in 3xTF32 (each operand split hi + lo, three
 *           TF32 products, fp32 accumulation; tnrd_tc.cu), for
 *           (ksize, N_k) in {(3, 8), (5, 24), (7, 48)}, boundary R1 or R2, exact
 *           or tabulated phi (the exact path's direct-sum fallback runs on FP32);
 *   AUTO:   TENSOR where it applies, else FP32 (the default). */
typedef enum {
    TNRD_ENGINE_AUTO = 0,
    TNRD_ENGINE_FP32 = 1,
    TNRD_ENGINE_TENSOR = 2
} tnrd_engine;

/* Model shape.  T >= 1 stages, n_filters = N_k >= 1 (P l.423: N_k = m^2 - 1 if
 * not specified, not enforced), ksize = m odd >= 3 (P l.458-469, Fig.3, studies
 * m = 3..9; this build runs m in {3, 5, 7, 9, 11}: the tensor engine for
 * (m, N_k) in {(3, 8), (5, 24), (7, 48)}, the FP32 engine for every m),
 * n_rbf = M in [1, 256], device = CUDA ordinal, reaction = tnrd_reaction
 * (0 = the paper's Eq.13). */
typedef struct {
    int T;
    int n_filters;
    int ksize;
    int n_rbf;
    int boundary;   /* tnrd_boundary */
    int phi_mode;   /* tnrd_phi_mode */
    int device;
    int reaction;   /* tnrd_reaction (was a reserved 0 field: 0 keeps Eq.13) */
} tnrd_desc;

/* ABI version this library implements (TNRD_ABI_VERSION). */
TNRD_API int tnrd_abi_version(void);

/* Human-readable name of a status code (static string). */
TNRD_API const char *tnrd_status_string(tnrd_status s);

/* Create a handle for model shape *d on d->device.  *out receives the handle
 * (owned by the caller, released with tnrd_destroy).  Allocates the device
 * parameter store.  EINVAL: bad shape (T, N_k or M out of range; ksize even or
 * < 3; bad enum); EUNSUPPORTED: odd ksize > 11, or a model whose stage operands
 * exceed the shared memory of one CTA; ECUDA/ENOMEM: device errors.  Synchronous. */
TNRD_API tnrd_status tnrd_create(const tnrd_desc *d, tnrd_handle **out);

/* Select the engine (tnrd_engine) for later tnrd_denoise* and tnrd_loss_grad calls
 * on h (tnrd_loss_grad: its forward tape and backward banks; on the tensor engine the
 * tape splits operands with round-to-nearest).  EINVAL: bad value.
 * Host-only. */
TNRD_API tnrd_status tnrd_set_engine(tnrd_handle *h, int engine);

/* The engine (TNRD_ENGINE_FP32 or TNRD_ENGINE_TENSOR) tnrd_denoise would use for
 * a B x H x W batch now; -1 if h is null or a stage is unset.  Host-only. */
TNRD_API int tnrd_engine_for(tnrd_handle *h, int B, int H, int W);

/* Set Theta^t = {lambda^t, phi_i^t, k_i^t} of stage t in [0, T) (P l.206-207).
 * All pointers are HOST arrays, copied before return (the caller may free them):
 *   filters   [N_k][m][m]  k_i^t row-major, the true-convolution kernel (kbar derived)
 *   rbf_w     [N_k][M]     RBF weights w_ij
 *   rbf_mu0   [N_k]        first centre mu_i0
 *   rbf_step  [N_k]        centre spacing, > 0
 *   rbf_gamma [N_k]        Gaussian width, > 0
 *   lambda                 lambda^t > 0 (P Eq.13; not beta = log lambda, P l.415)
 * EINVAL on non-finite values, step/gamma <= 0, lambda <= 0, t out of range.
 * Derived fp32 evaluation constants are computed on the host in double.
 * Synchronous (uploads with a blocking copy). */
TNRD_API tnrd_status tnrd_set_stage_params(tnrd_handle *h, int t, const float *filters, const float *rbf_w,
                                  const float *rbf_mu0, const float *rbf_step,
                                  const float *rbf_gamma, float lambda);

/* Denoise B images: u_dev <- u_T(f_dev) (P Eq.13 iterated, u_0 = f).
 *   f_dev  device [B][H][ld]  Poisson counts (non-negative; not validated)
 *   u_dev  device [B][H][ld]  output; must not alias f_dev (f is read every stage)
 *   H, W >= ksize, B >= 1, ld >= W
 *   peak   host [B] or NULL: per-image peak (P l.113-116), metadata only -- Eq.13
 *          does not use it; it is validated (> 0, finite) when given.
 * Scratch (one ping-pong image batch) is owned by the handle and grown on demand
 * (synchronously, before enqueueing).  ESTATE if any stage is unset.
 * Stream-ordered and asynchronous: the T stage launches are captured once per
 * argument set (pointers, sizes, ld) as a CUDA graph on a handle-owned stream and
 * replayed on cuda_stream (16 most recent kept; dropped by tnrd_set_stage_params /
 * tnrd_set_engine; TNRD_GRAPH=0 in the environment launches eagerly).  Each stage
 * kernel is a programmatic dependent launch: its set-up overlaps the previous
 * stage's tail, its image accesses wait for that stage to complete
 * (DESIGN.md §5.13). */
TNRD_API tnrd_status tnrd_denoise(tnrd_handle *h, const float *f_dev, float *u_dev, int B, int H, int W,
                         long long ld, const float *peak, void *cuda_stream);

/* End-to-end variant: f_host -> device -> denoise -> u_host, dense rows (ld = W).
 * Large batches are pipelined in up to 8 chunks: the host-to-device copy of chunk
 * c+1 and the device-to-host copy of chunk c-1 run on handle-owned copy streams
 * while chunk c is denoised on cuda_stream (results identical to one call).
 * The copy streams start after the work already enqueued on cuda_stream, and
 * cuda_stream is ordered after the last copy; the call synchronises before
 * returning (u_host is valid on return).  Pinned host memory is needed for the
 * copies to overlap (and gives full PCIe bandwidth). */
TNRD_API tnrd_status tnrd_denoise_host(tnrd_handle *h, const float *f_host, float *u_host, int B, int H,
                              int W, const float *peak, void *cuda_stream);

/* Release the handle and everything it owns (device buffers, events, NCCL
 * communicator).  NULL is a no-op.  Synchronises the device first. */
TNRD_API tnrd_status tnrd_destroy(tnrd_handle *h);

/* Message for the last failing call on h (or on the thread, if h is NULL).
 * Valid until the next call on h. */
TNRD_API const char *tnrd_last_error(const tnrd_handle *h);

/* Number of kernels this handle has launched so far (evidence for the bench's
 * gpu_launches count). */
TNRD_API unsigned long long tnrd_launch_count(const tnrd_handle *h);

/* ---------------- training gradient (P Eq.6-7, 14-20) ----------------
 * loss = 1/2 sum_b ||u_T^b - u_gt^b||^2 over the batch (P Eq.6, l.199-222) and its
 * gradient w.r.t. Theta_t = {lambda_t, phi_i^t, k_i^t} by the chain rule of
 * P l.343-420: dl/du_T = u_T - u_gt (l.348-353), the prox Jacobian y (Eq.16),
 * Eq.15's K_i^T Lambda_i Kbar_i^T with the exact transposes of the symmetric-
 * boundary convolutions (R1 and R2), the RBF-weight and filter derivatives, and
 * z = du/dlambda (Eq.19).  For lambda = e^beta (Eq.20) dl/dbeta = lambda dl/dlambda.
 *   f_dev, u_gt_dev  device [B][H][ld]
 *   grad_filters     host [T][N_k][m][m]   dl/dk_i^t
 *   grad_rbf_w       host [T][N_k][M]      dl/dw_ij^t
 *   grad_lambda      host [T]              dl/dlambda_t
 *   loss             host                  the loss (double)
 * Reaction 0 and TNRD_PHI_EXACT only (else EUNSUPPORTED).  Runs the forward pass
 * with a tape (2T+1 images of scratch, owned by the handle), then the backward
 * stages: where (k, N_k) has tensor instantiations and the engine is not FP32, the
 * tape, both filter banks and the filter-gradient sums run as 3xTF32 tcgen05 GEMMs
 * (round-to-nearest operand split) when all N_k filters fit one backward chunk.
 * The backward's per-filter scratch (5 images per filter) is chunked by filters:
 * F = min(N_k, tnrd_set_grad_chunk's cap, filters whose scratch fits half the
 * device's TOTAL memory) -- a function of the shape and the device, never of the
 * memory that happens to be free, so every call with the same arguments uses the
 * same chunks and summation order (bitwise reproducible).  ENOMEM if that scratch
 * cannot be allocated (nothing is retried smaller).  Synchronous: returns after the
 * host outputs are written. */
TNRD_API tnrd_status tnrd_loss_grad(tnrd_handle *h, const float *f_dev, const float *u_gt_dev, int B, int H,
                                    int W, long long ld, float *grad_filters, float *grad_rbf_w,
                                    float *grad_lambda, double *loss, void *cuda_stream);

/* Cap the filters per backward chunk of tnrd_loss_grad (0 = automatic, the
 * default).  F < N_k keeps the filter-bank steps on the CUDA cores (the tensor
 * banks need every filter of a stage in one chunk).  EINVAL if max_filters < 0.
 * Host-only. */
TNRD_API tnrd_status tnrd_set_grad_chunk(tnrd_handle *h, int max_filters);

/* ---------------- steps either side of the path ----------------
 * Poisson noise (P Eq.1, l.103-111): f_dev[b][y][x] ~ Poisson(u_dev[b][y][x]) as
 * exact integer-valued fp32 counts; u = 0 gives 0.  Counter-based and reproducible:
 * Philox4x32-10 keyed by `seed`, counter = (b*H + y)*W + x, one 53-bit uniform per
 * pixel, exact inversion of the Poisson CDF in double with a fixed fma-only exp --
 * the same draw as the oracle's oracle_sample_poisson, bit for bit.
 *   u_dev, f_dev  device [B][H][ld] (may alias)
 * EINVAL if any mean is negative or NaN (checked on the device; synchronous). */
TNRD_API tnrd_status tnrd_sample_poisson(const float *u_dev, float *f_dev, int B, int H, int W, long long ld,
                                         unsigned long long seed, void *cuda_stream);

/* PSNR per image (reading C15: 10 log10(peak_b^2 / MSE(u_b, clean_b)), unclamped;
 * +inf for equal images): u_dev, clean_dev device [B][H][ld]; peak host [B];
 * psnr_out host [B].  Squared errors summed in double in a fixed order.
 * EINVAL: B outside [1, 65535], H or W < 1, ld < W.  Synchronous. */
TNRD_API tnrd_status tnrd_psnr(const float *u_dev, const float *clean_dev, int B, int H, int W, long long ld,
                               const float *peak, double *psnr_out, void *cuda_stream);

/* Peak scaling (S l.351-358; P l.113-116, "the noise level ... is generally defined
 * as the peak value (the maximal value)"): out_b = x_b * (peak_b / max(x_b)) in fp32,
 * and exactly peak_b where x_b == max(x_b), so max(out_b) == peak_b.
 *   x_dev, out_dev  device [B][H][ld] (may alias); peak host [B], > 0
 * EINVAL: bad sizes, B > 65535, a peak <= 0, a negative / NaN input or an all-zero
 * image (S l.355; out is then undefined).  Synchronous. */
TNRD_API tnrd_status tnrd_scale_to_peak(const float *x_dev, float *out_dev, int B, int H, int W, long long ld,
                                        const float *peak, void *cuda_stream);

/* SSIM per image (S l.381-389; P l.444-445; reading M2 in DESIGN.md): both images
 * rescaled by 255/peak_b, the mean over every 11 x 11 window inside the image of
 * ((2 mu_u mu_c + C1)(2 s_uc + C2)) / ((mu_u^2 + mu_c^2 + C1)(s_u^2 + s_c^2 + C2)),
 * Gaussian-weighted window moments (sigma = 1.5, weights summing to 1), C1 = (0.01 *
 * 255)^2, C2 = (0.03 * 255)^2.  Moments in double; window sums in a fixed order.
 *   u_dev, clean_dev device [B][H][ld]; peak host [B]; ssim_out host [B]
 * EINVAL: H or W < 11, ld < W, B outside [1, 65535], a peak <= 0.  Synchronous. */
TNRD_API tnrd_status tnrd_ssim(const float *u_dev, const float *clean_dev, int B, int H, int W, long long ld,
                               const float *peak, double *ssim_out, void *cuda_stream);

/* ---------------- multi-GPU: row slabs of one large image ----------------
 * Rank rho of N owns rows [row0, row0 + rows) of an H_global x W image.
 * Before every stage each rank exchanges 2r = ksize-1 rows of u_t with each
 * neighbour (ncclSend/ncclRecv on cuda_stream; DESIGN.md §6 reading C18: a
 * fused stage depends on u within 2r rows).  f needs no exchange (the prox is
 * pointwise).  Global top/bottom rows use the mirror; seams use neighbour data,
 * so the result is bitwise equal to the single-GPU tnrd_denoise. */

/* Fill id128 (128 bytes, host) with a fresh ncclUniqueId.  The caller
 * broadcasts it to all ranks (e.g. with torch.distributed).  ENCCL if NCCL
 * cannot be loaded (libnccl.so.2 is opened at run time; set TNRD_NCCL_LIB to
 * its path to override the search). */
TNRD_API tnrd_status tnrd_nccl_unique_id(void *id128);

/* Create the handle's communicator (ncclCommInitRank) for rank of nranks.
 * Collective across ranks; synchronous. */
TNRD_API tnrd_status tnrd_comm_init(tnrd_handle *h, const void *id128, int rank, int nranks);

/* Denoise this rank's slab.  f_slab_dev / u_slab_dev: device [rows][ld], the
 * rank's own rows only.  rows >= ksize - 1 on every rank.  Enqueued on
 * cuda_stream (NCCL calls included). */
TNRD_API tnrd_status tnrd_denoise_slab(tnrd_handle *h, const float *f_slab_dev, float *u_slab_dev,
                              int H_global, int W, int row0, int rows, long long ld, float peak,
                              void *cuda_stream);

/* Wait for the work enqueued on cuda_stream (e.g. tnrd_denoise_slab) while polling
 * the communicator's asynchronous error every 200 us (ncclCommGetAsyncError).  A
 * NCCL error, or no completion within timeout_ms (< 0: no limit), aborts the
 * communicator (ncclCommAbort: pending NCCL kernels return) and returns ENCCL; the
 * handle then needs tnrd_comm_init again.  ECUDA for a failed stream.  OK when the
 * stream has drained without error.  Failure detection for the slab path (SURVEY
 * §5); every tnrd_denoise_slab also polls once per exchange without blocking. */
TNRD_API tnrd_status tnrd_comm_wait(tnrd_handle *h, void *cuda_stream, int timeout_ms);

/* Single-device emulation of the slab path: the image f_dev [H][ld] is split
 * into nslabs row slabs processed with the same slab kernels and halo buffers,
 * the halo exchange done with device-to-device copies instead of NCCL.  Used
 * to test the partition on one GPU; result equals tnrd_denoise bitwise. */
TNRD_API tnrd_status tnrd_denoise_slabs_loopback(tnrd_handle *h, const float *f_dev, float *u_dev, int H,
                                        int W, long long ld, int nslabs, void *cuda_stream);

/* The same single-device slab partition with every halo transfer done by NCCL:
 * per stage one grouped exchange of ncclSend / ncclRecv pairs whose peer is the
 * caller's own rank, on the handle's communicator, which must have been created
 * with tnrd_comm_init(h, id, 0, 1) (else ESTATE).  Moves exactly the rows and
 * bytes the multi-rank path moves (2r rows per seam and direction), so it runs the
 * NCCL transport of the slab path on one GPU; result equals tnrd_denoise bitwise.
 * ENCCL on an NCCL failure. */
TNRD_API tnrd_status tnrd_denoise_slabs_nccl_self(tnrd_handle *h, const float *f_dev, float *u_dev, int H,
                                         int W, long long ld, int nslabs, void *cuda_stream);

/* ---------------- instrumentation and micro-parity ---------------- */

/* Enable (1) / disable (0) per-launch CUDA-event timing of the stage kernels. */
TNRD_API tnrd_status tnrd_set_profiling(tnrd_handle *h, int enable);

/* After a profiled, completed tnrd_denoise: writes min(n, launches) per-launch
 * durations in milliseconds to ms_out (host) and the count to *n_out.
 * Synchronises on the recorded events. */
TNRD_API tnrd_status tnrd_get_launch_times(tnrd_handle *h, float *ms_out, int n, int *n_out);

/* Evaluate the device phi_i^t on n device values v_dev -> out_dev (same code
 * as the stage kernel).  Stage t must be set. */
TNRD_API tnrd_status tnrd_debug_phi(tnrd_handle *h, int t, int i, const float *v_dev, float *out_dev,
                           long long n, void *cuda_stream);

/* Evaluate the device Poisson prox (Eq.12, tau = 1) elementwise on n device
 * values: out = prox_lambda(ut; f). */
TNRD_API tnrd_status tnrd_debug_prox(const float *ut_dev, const float *f_dev, float lambda, float *out_dev,
                            long long n, void *cuda_stream);

#ifdef __cplusplus
}
#endif

#endif /* TNRD_H_ */
