"""Seeded synthetic workloads for TNRD/TRDPD Poisson denoising (arXiv 1510.02930).

Stand-ins for the paper's data, which is not in this container:
  * the 68-image test set and the 256^2 / 512^2 timing images at peak 4
     -> piecewise-constant images plus a ramp,
    scaled to a peak ("the noise level ... is generally
    defined as the peak value") and Poisson-sampled (Eq. 1);
  * the trained TRDPD parameters (Theta^t = {lambda^t,
    phi_i^t, k_i^t}) -> random zero-mean unit-norm DCT-combination filters,
    Gaussian-RBF influence functions with uniform centres, and random lambda_t.

Recipe (BASELINE.json configs[0..4]; SURVEY.md §8(c) C7-C10 and §8(d);
DESIGN.md §3 restates it).  Nothing here evaluates the method: no
convolution, no influence function, no proximal step.
"""
from __future__ import annotations

import dataclasses
import functools
from typing import Optional, Sequence

import numpy as np

MASTER_SEED = 151002930  # + config id (1-based), SURVEY.md §8(d)

# BASELINE.json configs[0..4] -> C1..C5.
CONFIGS = {
    1: dict(name="C1", B=1, H=64, W=64, peaks=[4.0], T=2, Nk=8, k=3, M=63, lam="one"),
    2: dict(name="C2", B=1, H=256, W=256, peaks=[4.0], T=5, Nk=24, k=5, M=63, lam="uniform"),
    3: dict(name="C3", B=1, H=512, W=512, peaks=[1.0], T=8, Nk=48, k=7, M=63, lam="uniform"),
    4: dict(name="C4", B=256, H=512, W=512, peaks=[0.1, 0.2, 1.0, 2.0, 4.0], T=8, Nk=48, k=7,
            M=63, lam="uniform"),
    5: dict(name="C5", B=1, H=8192, W=8192, peaks=[0.1], T=8, Nk=48, k=7, M=63, lam="uniform"),
}


@dataclasses.dataclass
class Model:
    """Stage parameters Theta^t for t = 0..T-1, all float32.

    filters  [T][Nk][k][k]  k_i^t, true-convolution kernels (rotated twin derived)
    rbf_w    [T][Nk][M]     weights of phi_i^t = sum_j w_j exp(-(z-mu_j)^2/(2 gamma^2))
    rbf_mu0  [T][Nk]        first centre mu_{i,0}
    rbf_step [T][Nk]        centre spacing Delta_i (mu_j = mu0 + j*Delta)
    rbf_gamma[T][Nk]        Gaussian width gamma_i
    lam      [T]            lambda^t > 0 (Eq. 13, l.328-333)
    """

    filters: np.ndarray
    rbf_w: np.ndarray
    rbf_mu0: np.ndarray
    rbf_step: np.ndarray
    rbf_gamma: np.ndarray
    lam: np.ndarray

    @property
    def T(self) -> int:
        return int(self.filters.shape[0])

    @property
    def Nk(self) -> int:
        return int(self.filters.shape[1])

    @property
    def k(self) -> int:
        return int(self.filters.shape[2])

    @property
    def M(self) -> int:
        return int(self.rbf_w.shape[2])

    def stage(self, t: int) -> "Model":
        s = slice(t, t + 1)
        return Model(self.filters[s], self.rbf_w[s], self.rbf_mu0[s], self.rbf_step[s],
                     self.rbf_gamma[s], self.lam[s])


@dataclasses.dataclass
class Problem:
    cfg: dict
    f: np.ndarray       # [B][H][W] float32 Poisson counts (exact integers)
    clean: np.ndarray   # [B][H][W] float32 clean image, max == peak_b
    peaks: np.ndarray   # [B] float32
    model: Model
    f_max: float        # max f over all images sharing the model (>= 1), SURVEY C8


def dct_atoms(m: int) -> np.ndarray:
    """Orthonormal 2-D DCT-II atoms, shape [m*m][m][m], atom 0 = the constant one."""
    n = np.arange(m)
    C = np.cos(np.pi * (2 * n[None, :] + 1) * n[:, None] / (2 * m))
    C[0] *= np.sqrt(1.0 / m)
    C[1:] *= np.sqrt(2.0 / m)
    atoms = np.einsum("pi,qj->pqij", C, C).reshape(m * m, m, m)
    return atoms


def _filters(rng: np.random.Generator, T: int, Nk: int, m: int) -> np.ndarray:
    """Zero-mean unit-L2 filters: N(0,1) coefficients on the m^2-1 non-constant
    DCT-II atoms, normalised, rounded to fp32."""
    atoms = dct_atoms(m)[1:]  # drop the constant atom -> zero mean
    coef = rng.standard_normal((T, Nk, m * m - 1))
    k = np.einsum("tia,axy->tixy", coef, atoms)
    k /= np.sqrt((k ** 2).sum(axis=(2, 3), keepdims=True))
    return k.astype(np.float32)


def _paint(rng: np.random.Generator, H: int, W: int) -> np.ndarray:
    """Clean image before peak scaling: ramp + overpainted disks/rectangles."""
    a0 = rng.uniform(0.1, 0.3)
    a1, a2 = rng.uniform(-0.2, 0.2, size=2)
    yy = np.arange(H, dtype=np.float64)[:, None]
    xx = np.arange(W, dtype=np.float64)[None, :]
    img = a0 + a1 * xx / W + a2 * yy / H + np.zeros((H, W))
    n = max(8, (H * W) // 8192)
    s = min(H, W, 512)  # shape sizes as for a <=512^2 image
    for _ in range(n):
        inten = rng.uniform(0.0, 1.0)
        if rng.uniform() < 0.5:
            rad = rng.uniform(4.0, s / 4.0)
            cy, cx = rng.uniform(0, H), rng.uniform(0, W)
            y0, y1 = max(0, int(cy - rad)), min(H, int(cy + rad) + 1)
            x0, x1 = max(0, int(cx - rad)), min(W, int(cx + rad) + 1)
            if y0 >= y1 or x0 >= x1:
                continue
            sub = img[y0:y1, x0:x1]
            m = (yy[y0:y1] - cy) ** 2 + (xx[:, x0:x1] - cx) ** 2 <= rad * rad
            sub[m] = inten
        else:
            h, w = rng.uniform(8.0, s / 2.0, size=2)
            cy, cx = rng.uniform(0, H), rng.uniform(0, W)
            y0, y1 = max(0, int(cy - h / 2)), min(H, int(cy + h / 2))
            x0, x1 = max(0, int(cx - w / 2)), min(W, int(cx + w / 2))
            img[y0:y1, x0:x1] = inten
    return np.clip(img, 0.0, None)


def clean_image(rng: np.random.Generator, H: int, W: int, peak: float) -> np.ndarray:
    """Piecewise-constant + ramp image scaled so that max == peak."""
    img = _paint(rng, H, W)
    return (img * (peak / img.max())).astype(np.float32)


def make_model(rng: np.random.Generator, T: int, Nk: int, k: int, M: int, f_max: float,
               lam_mode: str = "uniform", grid_scale: float = 3.0, w_std: float = 0.1) -> Model:
    """Random Theta^t.  RBF grid per (t,i): R = grid_scale * F_max * ||k||_1 / 2,
    mu0 = -R, Delta = 2R/(M-1), gamma = Delta; w ~ N(0, w_std^2) (C9);
    lambda = 1 (C1) or U[0.5, 2]."""
    filt = _filters(rng, T, Nk, k)
    w = (w_std * rng.standard_normal((T, Nk, M))).astype(np.float32)
    if lam_mode == "one":
        lam = np.ones(T, np.float32)
    else:
        lam = rng.uniform(0.5, 2.0, size=T).astype(np.float32)
    l1 = np.abs(filt.astype(np.float64)).sum(axis=(2, 3))
    R = grid_scale * max(f_max, 1.0) * l1 / 2.0
    mu0 = (-R).astype(np.float32)
    step = (2.0 * R / (M - 1)).astype(np.float32)
    gamma = step.copy()
    return Model(filt, w, mu0, step, gamma, lam)


@functools.lru_cache(maxsize=8)
def _problem_cached(c: int, batch: Optional[int]) -> Problem:
    cfg = dict(CONFIGS[c])
    B = cfg["B"] if batch is None else batch
    H, W = cfg["H"], cfg["W"]
    ss_clean, ss_pois, ss_par = np.random.SeedSequence(MASTER_SEED + c).spawn(3)
    kids_c = ss_clean.spawn(B)
    kids_p = ss_pois.spawn(B)
    peaks = np.array([cfg["peaks"][b % len(cfg["peaks"])] for b in range(B)], np.float32)
    clean = np.empty((B, H, W), np.float32)
    f = np.empty((B, H, W), np.float32)
    for b in range(B):
        clean[b] = clean_image(np.random.default_rng(kids_c[b]), H, W, float(peaks[b]))
        f[b] = np.random.default_rng(kids_p[b]).poisson(clean[b].astype(np.float64)).astype(np.float32)
    f_max = max(1.0, float(f.max()))
    model = make_model(np.random.default_rng(ss_par), cfg["T"], cfg["Nk"], cfg["k"], cfg["M"],
                       f_max, cfg["lam"])
    cfg["B"] = B
    return Problem(cfg, f, clean, peaks, model, f_max)


def make_problem(c: int, batch: Optional[int] = None) -> Problem:
    """Config c in 1..5 (BASELINE.json configs[c-1]).  `batch` overrides B (C4 only:
    the model's F_max then comes from the first `batch` images, and the problem is
    no longer C4's exact workload -- tests that need exact C4 pass batch=None)."""
    return _problem_cached(c, batch)


def stress_model(rng: np.random.Generator, T: int, Nk: int, k: int, M: int, f_max: float) -> Model:
    """phi-stress parameters: a grid 6x narrower than the standard one and
    weights 5x larger, so responses reach the outer centres and phi is strongly nonlinear."""
    return make_model(rng, T, Nk, k, M, f_max, "uniform", grid_scale=0.5, w_std=0.5)


def zero_model(T: int, Nk: int, k: int, M: int, zero: str, lam: Sequence[float],
               rng: Optional[np.random.Generator] = None, f_max: float = 4.0) -> Model:
    """P7/P8 parameters: zero filters ('filters') or zero RBF weights ('weights')."""
    rng = rng or np.random.default_rng(7)
    m = make_model(rng, T, Nk, k, M, f_max)
    if zero == "filters":
        m.filters[...] = 0.0
        m.rbf_mu0[...] = -1.0
        m.rbf_step[...] = np.float32(2.0 / (M - 1))
        m.rbf_gamma[...] = m.rbf_step
    elif zero == "weights":
        m.rbf_w[...] = 0.0
    else:
        raise ValueError(zero)
    m.lam[...] = np.asarray(lam, np.float32)
    return m
