/*
 * TNRD / TRDPD Poisson-denoising ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, double-precision CPU implementation of the inference pass of
 * Feng & Chen, "Fast and Accurate Poisson Denoising with Optimized Nonlinear
 * Diffusion" (arXiv 1510.02930).  Citations "P l.N" are lines of PAPER.md,
 * "S l.N" lines of SPEC.md.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header or
 * constant with the CUDA path (paper_1510_02930_b200/csrc) and never calls it.
 *
 * Conventions (DESIGN.md §2 lists every reading):
 *   - images are row-major [H][W] (S l.22-27), u in R^N (P l.101-102);
 *   - "*" is true 2-D convolution (P l.137, l.142-144; S l.50);
 *   - symmetric boundary = half-sample mirror, edge pixel duplicated
 *     (P l.302 "symmetric boundary condition"; S l.73);
 *   - stage s = 0..T-1 uses params[s] for k, phi and lambda (P Eq.13 l.328-332).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define EXPORT __attribute__((visibility("default")))

/* Half-sample symmetric extension index: x -> [0, n).  Folds repeatedly so
 * that it is defined for any x (S l.73: pad value at -1 equals value at 0). */
static long mirror_index(long x, long n) {
    long period = 2 * n;
    long m = x % period;
    if (m < 0) m += period;
    return m < n ? m : period - 1 - m;
}

/* rot180: kbar[i][j] = k[m-1-i][m-1-j]  (P l.143-144 "rotating the kernel k_i
 * 180 degrees"; S l.40). */
EXPORT void oracle_rot180(int m, const double *k, double *kbar) {
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j)
            kbar[i * m + j] = k[(m - 1 - i) * m + (m - 1 - j)];
}

/* conv2d_sym: out(p,q) = sum_{a,b=-r..r} k[a+r][b+r] * E(x)(p-a, q-b), E the
 * symmetric extension (P l.137 "k_i * u", l.302 symmetric boundary; S l.47-55). */
EXPORT void oracle_conv2d_sym(int H, int W, const double *x, int m, const double *k, double *out) {
    int r = m / 2;
#pragma omp parallel for schedule(static)
    for (int p = 0; p < H; ++p) {
        for (int q = 0; q < W; ++q) {
            double s = 0.0;
            for (int a = -r; a <= r; ++a) {
                long pp = mirror_index((long)p - a, H);
                for (int b = -r; b <= r; ++b) {
                    long qq = mirror_index((long)q - b, W);
                    s += k[(a + r) * m + (b + r)] * x[pp * W + qq];
                }
            }
            out[(long)p * W + q] = s;
        }
    }
}

/* conv2d_adjoint: the exact transpose K^T of conv2d_sym (P l.295-301 "K_i^T";
 * S l.57-65: scatter-add of reflected contributions).  Boundary reading R2. */
EXPORT void oracle_conv2d_adjoint(int H, int W, const double *y, int m, const double *k, double *out) {
    int r = m / 2;
    memset(out, 0, sizeof(double) * (size_t)H * W);
    for (int p = 0; p < H; ++p)
        for (int q = 0; q < W; ++q)
            for (int a = -r; a <= r; ++a) {
                long pp = mirror_index((long)p - a, H);
                for (int b = -r; b <= r; ++b) {
                    long qq = mirror_index((long)q - b, W);
                    out[pp * W + qq] += k[(a + r) * m + (b + r)] * y[(long)p * W + q];
                }
            }
}

/* Influence function phi(z) = sum_{j<M} w_j exp(-(z - mu_j)^2 / (2 gamma^2)),
 * mu_j = mu0 + j*step: Gaussian-RBF mixture on uniform centres
 * (P l.145-146 phi "not restricted to be of a certain kind"; S l.104-107, l.140;
 * BASELINE.json north_star).  Direct sum over all M terms. */
EXPORT double oracle_phi(int M, const double *w, double mu0, double step, double gamma, double z) {
    double s = 0.0;
    for (int j = 0; j < M; ++j) {
        double d = z - (mu0 + j * step);
        s += w[j] * exp(-(d * d) / (2.0 * gamma * gamma));
    }
    return s;
}

/* Poisson proximal map, P Eq.12 (l.318-322) with tau = 1 (l.333):
 *   u = (ut - lam + sqrt((ut - lam)^2 + 4 lam f)) / 2.
 * For ut - lam < 0 the algebraically equal form 2 lam f / (sqrt(.) - (ut - lam))
 * avoids cancellation (S l.215); f = 0 then gives exactly max(ut - lam, 0) (S l.183). */
EXPORT double oracle_prox(double ut, double lam, double f) {
    double delta = ut - lam;
    double sigma = sqrt(delta * delta + 4.0 * lam * f);
    if (delta >= 0.0) return 0.5 * (delta + sigma);
    if (f == 0.0) return 0.0;
    return 2.0 * lam * f / (sigma - delta);
}

/* Reaction of one stage (pointwise), given u_t, the diffusion result
 * ut = u_t - sum_i kbar_i * phi_i(k_i * u_t) and f:
 *   reaction 0: Poisson proximal step, P Eq.13 (l.326-333): prox_lambda(ut).
 *   reaction 1: Gaussian denoising, P Eq.3 (l.134-141) with the reaction
 *               psi(u_t, f) = lambda A^T (A u_t - f), A = I (l.150-158):
 *               ut - lambda (u_t - f).
 *   reaction 2: the direct Poisson gradient the paper rejects (l.247-252):
 *               P Eq.3 with psi = grad of D = lambda <u - f log u, 1> (Eq.4,
 *               l.163-167), i.e. ut - lambda (1 - f / u_t); where f = 0 the data
 *               term is lambda u, so f / u_t is taken as 0 there. */
EXPORT double oracle_reaction(double u, double ut, double f, double lam, int reaction) {
    if (reaction == 1) return ut - lam * (u - f);
    if (reaction == 2) return ut - lam * (1.0 - (f == 0.0 ? 0.0 : f / u));
    return oracle_prox(ut, lam, f);
}

/* One diffusion stage, P Eq.13 (l.326-333):
 *   ut = u - sum_i kbar_i * phi_i(k_i * u),   u_next = prox_lambda(ut).
 * boundary 0 (R1, default): the second convolution is the explicit rotated-kernel
 *   convolution with the symmetric boundary (P l.302-311 "revise the above
 *   formulation as explicit convolutions").
 * boundary 1 (R2): the exact transpose K_i^T (P l.298-301; S l.57-65).
 * phi_mode 0: RBF phi;  phi_mode 1: linear phi_i(z) = w[i][0] * z (oracle-only
 *   switch used to pin linear diffusion, BASELINE.json north_star).
 * Filters are taken in ascending i (S l.219). */
EXPORT void oracle_stage(int H, int W, const double *u, const double *f,
                         int Nk, int m, int M,
                         const double *filters, /* [Nk][m][m] */
                         const double *rbf_w,   /* [Nk][M] */
                         const double *mu0, const double *step, const double *gamma, /* [Nk] */
                         double lam, int boundary, int phi_mode, int reaction,
                         double *u_next, double *u_tilde_out /* may be NULL */) {
    size_t N = (size_t)H * W;
    double *v = (double *)malloc(sizeof(double) * N);
    double *d = (double *)calloc(N, sizeof(double));
    double *t = (double *)malloc(sizeof(double) * N);
    double *kbar = (double *)malloc(sizeof(double) * m * m);
    for (int i = 0; i < Nk; ++i) {
        const double *k = filters + (size_t)i * m * m;
        oracle_conv2d_sym(H, W, u, m, k, v);                      /* v = k_i * u     */
#pragma omp parallel for schedule(static)
        for (long p = 0; p < (long)N; ++p)                        /* w = phi_i(v)    */
            v[p] = phi_mode == 1 ? rbf_w[(size_t)i * M] * v[p]
                                 : oracle_phi(M, rbf_w + (size_t)i * M, mu0[i], step[i], gamma[i], v[p]);
        if (boundary == 1) {
            oracle_conv2d_adjoint(H, W, v, m, k, t);              /* t = K_i^T w     */
        } else {
            oracle_rot180(m, k, kbar);
            oracle_conv2d_sym(H, W, v, m, kbar, t);               /* t = kbar_i * w  */
        }
        for (size_t p = 0; p < N; ++p) d[p] += t[p];
    }
    for (size_t p = 0; p < N; ++p) {
        double ut = u[p] - d[p];                                  /* tau = 1, l.333  */
        if (u_tilde_out) u_tilde_out[p] = ut;
        u_next[p] = oracle_reaction(u[p], ut, f[p], lam, reaction);
    }
    free(v); free(d); free(t); free(kbar);
}

/* Inference pass: u_0 = f (P l.136 "u_0 = I_0", l.148 "I_0 ... can be set as f"),
 * then T stages of Eq.13.  No floor or clamp (P never clamps; S l.228). */
EXPORT void oracle_denoise(int H, int W, const double *f, int T, int Nk, int m, int M,
                           const double *filters, const double *rbf_w, const double *mu0,
                           const double *step, const double *gamma, const double *lam,
                           int boundary, int phi_mode, int reaction, double *u_out) {
    size_t N = (size_t)H * W;
    double *a = (double *)malloc(sizeof(double) * N);
    double *b = (double *)malloc(sizeof(double) * N);
    memcpy(a, f, sizeof(double) * N);
    for (int s = 0; s < T; ++s) {
        oracle_stage(H, W, a, f, Nk, m, M,
                     filters + (size_t)s * Nk * m * m, rbf_w + (size_t)s * Nk * M,
                     mu0 + (size_t)s * Nk, step + (size_t)s * Nk, gamma + (size_t)s * Nk,
                     lam[s], boundary, phi_mode, reaction, b, NULL);
        double *tmp = a; a = b; b = tmp;
    }
    memcpy(u_out, a, sizeof(double) * N);
    free(a); free(b);
}

/* ------------------------------------------------------------------ training gradient
 * Loss l = 1/2 ||u_T - u_gt||^2 (P Eq.6, l.199-222) and its gradient w.r.t.
 * Theta_t = {lambda_t, phi_i^t (RBF weights), k_i^t} by the chain rule of
 * P l.343-420 (Eq.14-20), reaction 0 (Eq.13), in double.  Pinned against
 * central finite differences of oracle_denoise (tests/test_oracle_pins.py). */

/* out[a][b] = d/dk[a][b] <e, conv2d_sym(x, k)> = sum_p e(p) E(x)(p - (a-r, b-r)). */
EXPORT void oracle_kernel_grad(int H, int W, const double *x, const double *e, int m, double *out) {
    int r = m / 2;
    for (int a = 0; a < m; ++a)
        for (int b = 0; b < m; ++b) {
            double s = 0.0;
#pragma omp parallel for reduction(+ : s) schedule(static)
            for (int p = 0; p < H; ++p) {
                long pp = mirror_index((long)p - (a - r), H);
                for (int q = 0; q < W; ++q)
                    s += e[(long)p * W + q] * x[pp * W + mirror_index((long)q - (b - r), W)];
            }
            out[a * m + b] = s;
        }
}

/* phi'(z) = sum_j w_j (-(z - mu_j) / gamma^2) exp(-(z - mu_j)^2 / (2 gamma^2))
 * (the diagonal of Lambda_i, P l.369-371); G_out[j] = exp(-(z - mu_j)^2/(2 gamma^2)),
 * the derivative of phi w.r.t. w_j. */
EXPORT double oracle_phi_prime(int M, const double *w, double mu0, double step, double gamma, double z,
                               double *G_out /* [M] or NULL */) {
    double s = 0.0;
    for (int j = 0; j < M; ++j) {
        double d = z - (mu0 + j * step);
        double g = exp(-d * d / (2.0 * gamma * gamma));
        if (G_out) G_out[j] = g;
        s += w[j] * (-d / (gamma * gamma)) * g;
    }
    return s;
}

EXPORT double oracle_loss_grad(int H, int W, const double *f, const double *u_gt, int T, int Nk, int m, int M,
                               const double *filters, const double *rbf_w, const double *mu0,
                               const double *step, const double *gamma, const double *lam, int boundary,
                               double *g_filters /* [T][Nk][m][m] */, double *g_w /* [T][Nk][M] */,
                               double *g_lam /* [T] */) {
    size_t N = (size_t)H * W, mm = (size_t)m * m;
    double *u = (double *)malloc(sizeof(double) * N * (T + 1));   /* tape u_0..u_T  */
    double *ut = (double *)malloc(sizeof(double) * N * T);         /* tape ut_0..    */
    memcpy(u, f, sizeof(double) * N);
    for (int s = 0; s < T; ++s)
        oracle_stage(H, W, u + s * N, f, Nk, m, M, filters + s * Nk * mm, rbf_w + (size_t)s * Nk * M,
                     mu0 + (size_t)s * Nk, step + (size_t)s * Nk, gamma + (size_t)s * Nk, lam[s], boundary, 0, 0,
                     u + (s + 1) * N, ut + s * N);
    double loss = 0.0;
    double *g = (double *)malloc(sizeof(double) * N);
    for (size_t p = 0; p < N; ++p) {                               /* dl/du_T = u_T - u_gt (l.348-353) */
        g[p] = u[T * N + p] - u_gt[p];
        loss += 0.5 * g[p] * g[p];
    }
    double *e = (double *)malloc(sizeof(double) * N), *gn = (double *)malloc(sizeof(double) * N);
    double *v = (double *)malloc(sizeof(double) * N), *wv = (double *)malloc(sizeof(double) * N);
    double *av = (double *)malloc(sizeof(double) * N), *bv = (double *)malloc(sizeof(double) * N);
    double *tmp = (double *)malloc(sizeof(double) * N), *kbar = (double *)malloc(sizeof(double) * mm);
    double *kg = (double *)malloc(sizeof(double) * mm), *G = (double *)malloc(sizeof(double) * M);
    for (int s = T - 1; s >= 0; --s) {
        const double L = lam[s];
        const double *us = u + s * N, *uts = ut + s * N;
        g_lam[s] = 0.0;
        for (size_t p = 0; p < N; ++p) {
            double delta = uts[p] - L, sigma = sqrt(delta * delta + 4.0 * L * f[p]);
            double y = sigma > 0.0 ? 0.5 * (1.0 + delta / sigma) : 0.5;          /* Eq.16 */
            double z = sigma > 0.0 ? 0.5 * (-1.0 + (-delta + 2.0 * f[p]) / sigma) : -0.5; /* Eq.19 */
            e[p] = y * g[p];                                       /* dl/d ut                */
            g_lam[s] += z * g[p];
            gn[p] = e[p];                                          /* identity part of Eq.15 */
        }
        for (int i = 0; i < Nk; ++i) {
            const double *k = filters + (s * Nk + i) * mm;
            const double *wi = rbf_w + ((size_t)s * Nk + i) * M;
            const double m0 = mu0[(size_t)s * Nk + i], st = step[(size_t)s * Nk + i], ga = gamma[(size_t)s * Nk + i];
            double *gwi = g_w + ((size_t)s * Nk + i) * M, *gki = g_filters + (s * Nk + i) * mm;
            for (int j = 0; j < M; ++j) gwi[j] = 0.0;
            for (size_t q = 0; q < mm; ++q) gki[q] = 0.0;
            oracle_conv2d_sym(H, W, us, m, k, v);                  /* x = k_i * u_t          */
            oracle_rot180(m, k, kbar);
            /* a = (outer operator)^T e: R1 outer = conv with kbar (symmetric ext.), R2 outer = K^T */
            if (boundary == 1) oracle_conv2d_sym(H, W, e, m, k, av);
            else oracle_conv2d_adjoint(H, W, e, m, kbar, av);
            for (size_t p = 0; p < N; ++p) {
                double dphi = oracle_phi_prime(M, wi, m0, st, ga, v[p], G);
                wv[p] = oracle_phi(M, wi, m0, st, ga, v[p]);
                for (int j = 0; j < M; ++j) gwi[j] -= av[p] * G[j];   /* d ut / d w_ij = -outer(G_j) */
                bv[p] = dphi * av[p];                              /* Lambda_i outer^T e     */
            }
            oracle_conv2d_adjoint(H, W, bv, m, k, tmp);           /* K_i^T Lambda_i outer^T e (Eq.15) */
            for (size_t p = 0; p < N; ++p) gn[p] -= tmp[p];
            oracle_kernel_grad(H, W, us, bv, m, kg);              /* inner: x = k_i * u_t   */
            for (size_t q = 0; q < mm; ++q) gki[q] -= kg[q];
            if (boundary == 1) {                                  /* outer K^T w: <e, K^T w> = <K e, w> */
                oracle_kernel_grad(H, W, e, wv, m, kg);
                for (size_t q = 0; q < mm; ++q) gki[q] -= kg[q];
            } else {                                              /* outer conv(w, kbar)    */
                oracle_kernel_grad(H, W, wv, e, m, kg);
                for (int a = 0; a < m; ++a)
                    for (int b = 0; b < m; ++b) gki[(m - 1 - a) * m + (m - 1 - b)] -= kg[a * m + b];
            }
        }
        memcpy(g, gn, sizeof(double) * N);                         /* dl/du_s                */
    }
    free(u); free(ut); free(g); free(e); free(gn); free(v); free(wv); free(av); free(bv);
    free(tmp); free(kbar); free(kg); free(G);
    return loss;
}

/* ------------------------------------------------------------------ data generation
 * Poisson sampling (P Eq.1, l.103-111: f_i ~ Poisson(u_i), u_i = 0 gives f_i = 0)
 * with a counter-based generator both sides implement: Philox4x32-10 (Salmon et al.,
 * SC'11) keyed by the 64-bit seed, counter = (pixel index, 0, 0, 0); the uniform
 * U = (w0 * 2^21 + (w1 >> 11)) * 2^-53 in [0,1); inversion by sequential search of
 * the Poisson CDF in double: k = 0, p = exp(-u), F = p; while U >= F: k += 1,
 * p *= u / k, F += p (capped at u + 40 sqrt(u) + 40).  exp is a fixed fma-only
 * routine (2^k * Horner polynomial), so the integer decision is taken in the same
 * precision with the same operations on both sides. */
#include <stdint.h>

static void philox_round(uint32_t c[4], const uint32_t k[2]) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c[0], p1 = (uint64_t)0xCD9E8D57u * c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0, hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k[0], n1 = lo1, n2 = hi0 ^ c[3] ^ k[1], n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
}

EXPORT void oracle_philox4x32(uint64_t counter, uint64_t seed, uint32_t out[4]) {
    uint32_t c[4] = {(uint32_t)counter, (uint32_t)(counter >> 32), 0u, 0u};
    uint32_t k[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    for (int r = 0; r < 10; ++r) {
        philox_round(c, k);
        k[0] += 0x9E3779B9u;
        k[1] += 0xBB67AE85u;
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

/* exp(x) for x in [-745, 0]: x = n ln2 + r (Cody-Waite, hi/lo ln2), exp(r) by a
 * degree-13 Taylor Horner in fma, times 2^n.  Only IEEE fma / mul / add. */
EXPORT double oracle_exp_fixed(double x) {
    if (x < -745.0) return 0.0;
    const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
    const double n = nearbyint(x * 1.44269504088896338700e+00);
    const double r = fma(-n, ln2_lo, fma(-n, ln2_hi, x));
    double p = 1.0 / 6227020800.0;  /* 1/13! */
    const double inv[13] = {1.0 / 479001600.0, 1.0 / 39916800.0, 1.0 / 3628800.0, 1.0 / 362880.0, 1.0 / 40320.0,
                            1.0 / 5040.0, 1.0 / 720.0, 1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0, 0.5, 1.0, 1.0};
    for (int i = 0; i < 13; ++i) p = fma(p, r, inv[i]);
    return ldexp(p, (int)n);
}

EXPORT double oracle_poisson_draw(double u, uint64_t counter, uint64_t seed) {
    if (!(u > 0.0)) return 0.0;
    uint32_t w[4];
    oracle_philox4x32(counter, seed, w);
    const double U = ((double)w[0] * 2097152.0 + (double)(w[1] >> 11)) * (1.0 / 9007199254740992.0);
    double p = oracle_exp_fixed(-u), F = p, k = 0.0;
    const double kmax = floor(u + 40.0 * sqrt(u) + 40.0);
    while (U >= F && k < kmax) {
        k += 1.0;
        p *= u / k;
        F += p;
    }
    return k;
}

/* f[b][y][x] = Poisson(u[b][y][x]), counter = (b*H + y)*W + x. */
EXPORT void oracle_sample_poisson(int B, int H, int W, const double *u, uint64_t seed, double *f) {
#pragma omp parallel for schedule(static)
    for (long i = 0; i < (long)B * H * W; ++i) f[i] = oracle_poisson_draw(u[i], (uint64_t)i, seed);
}

/* ---------------------------------------------------------------------------
 * Steps either side of the path: peak scaling and SSIM.
 * ------------------------------------------------------------------------- */

/* Peak scaling (S l.351-358, "scale_to_peak"; P l.113-116: the noise level "is
 * generally defined as the peak value (the maximal value)" of the clean image):
 * out = x * (peak / max(x)), and exactly peak where x == max(x) (S l.354's post-
 * condition max(u) == peak, which the rounded product need not meet).  Returns -1
 * (out untouched) if max(x) <= 0 (S l.355: all-zero image is an error) or any
 * x < 0, else 0. */
EXPORT int oracle_scale_to_peak(long n, const double *x, double peak, double *out) {
    double m = 0.0;
    for (long i = 0; i < n; ++i) {
        if (x[i] < 0.0) return -1;
        if (x[i] > m) m = x[i];
    }
    if (m <= 0.0) return -1;
    const double r = peak / m;
    for (long i = 0; i < n; ++i) out[i] = x[i] == m ? peak : x[i] * r;
    return 0;
}

/* SSIM (S l.381-389; P l.444-445 cites the structural similarity index): both
 * images rescaled by 255/peak (S l.374), then the mean over every 11 x 11 window
 * that lies inside the image ("valid" windows, reading M2 in DESIGN.md §2) of
 *   ((2 mu_x mu_y + C1)(2 s_xy + C2)) / ((mu_x^2 + mu_y^2 + C1)(s_x^2 + s_y^2 + C2)),
 * mu, s^2, s_xy the window's Gaussian-weighted (sigma = 1.5, weights normalised to
 * sum 1) means, variances and covariance, C1 = (0.01 L)^2, C2 = (0.03 L)^2, L = 255.
 * Returns -1 if H or W < 11. */
EXPORT double oracle_ssim(int H, int W, const double *x, const double *y, double peak) {
    enum { WIN = 11, HALF = 5 };
    if (H < WIN || W < WIN) return -1.0;
    double wgt[WIN][WIN], wsum = 0.0;
    for (int a = 0; a < WIN; ++a)
        for (int b = 0; b < WIN; ++b) {
            const double da = a - HALF, db = b - HALF;
            wgt[a][b] = exp(-(da * da + db * db) / (2.0 * 1.5 * 1.5));
            wsum += wgt[a][b];
        }
    const double s = 255.0 / peak, C1 = (0.01 * 255.0) * (0.01 * 255.0), C2 = (0.03 * 255.0) * (0.03 * 255.0);
    double total = 0.0;
    for (int i = 0; i + WIN <= H; ++i)
        for (int j = 0; j + WIN <= W; ++j) {
            double mx = 0, my = 0, xx = 0, yy = 0, xy = 0;
            for (int a = 0; a < WIN; ++a)
                for (int b = 0; b < WIN; ++b) {
                    const double w = wgt[a][b] / wsum;
                    const double xv = s * x[(long)(i + a) * W + j + b], yv = s * y[(long)(i + a) * W + j + b];
                    mx += w * xv;
                    my += w * yv;
                    xx += w * xv * xv;
                    yy += w * yv * yv;
                    xy += w * xv * yv;
                }
            const double vx = xx - mx * mx, vy = yy - my * my, cxy = xy - mx * my;
            total += ((2 * mx * my + C1) * (2 * cxy + C2)) / ((mx * mx + my * my + C1) * (vx + vy + C2));
        }
    return total / ((double)(H - WIN + 1) * (W - WIN + 1));
}
