"""Double-precision CPU oracle for TNRD/TRDPD inference -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product path
(paper_1510_02930_b200) never imports it and shares no code with it.

The arithmetic lives in tnrd_oracle.c (plain C, double, OpenMP over rows);
this module compiles it with gcc and exposes it through ctypes.  Every C
function cites the PAPER.md / SPEC.md passage it follows.

Parity pins (tests/test_oracle_pins.py) tie each function to something other
than itself: brute-force dense matrices, scipy.ndimage.convolve, closed forms,
scalar minimisation of Eq.10, invariants.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tnrd_oracle.c")
_LIB = os.path.join(_HERE, "libtnrd_oracle.so")
_lock = threading.Lock()
_lib = None

BOUNDARY_EXPLICIT = 0  # R1: symmetric-extension rotated-kernel convolution (P l.302-311)
BOUNDARY_ADJOINT = 1   # R2: exact transpose K^T (P l.298-301; S l.57-65)
PHI_RBF = 0
PHI_LINEAR = 1
REACTION_PROX = 0      # Poisson proximal step, P Eq.13 (the method)
REACTION_GAUSSIAN = 1  # psi = lambda (u_t - f), P Eq.3 with A = I (l.150-158)
REACTION_POISSON_GRADIENT = 2  # psi = lambda (1 - f/u_t), the rejected direct step (l.247-252)


def build(force: bool = False) -> str:
    """Compile the oracle shared library with gcc (-O2, OpenMP, IEEE math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c99", "-Wall",
               "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


def lib() -> ctypes.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            dp = ctypes.POINTER(ctypes.c_double)
            i = ctypes.c_int
            L.oracle_rot180.argtypes = [i, dp, dp]
            L.oracle_conv2d_sym.argtypes = [i, i, dp, i, dp, dp]
            L.oracle_conv2d_adjoint.argtypes = [i, i, dp, i, dp, dp]
            L.oracle_phi.argtypes = [i, dp, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double]
            L.oracle_phi.restype = ctypes.c_double
            L.oracle_prox.argtypes = [ctypes.c_double] * 3
            L.oracle_prox.restype = ctypes.c_double
            L.oracle_stage.argtypes = [i, i, dp, dp, i, i, i, dp, dp, dp, dp, dp, ctypes.c_double,
                                       i, i, i, dp, dp]
            L.oracle_denoise.argtypes = [i, i, dp, i, i, i, i, dp, dp, dp, dp, dp, dp, i, i, i, dp]
            L.oracle_loss_grad.argtypes = [i, i, dp, dp, i, i, i, i, dp, dp, dp, dp, dp, dp, i, dp, dp, dp]
            L.oracle_loss_grad.restype = ctypes.c_double
            L.oracle_kernel_grad.argtypes = [i, i, dp, dp, i, dp]
            L.oracle_sample_poisson.argtypes = [i, i, i, dp, ctypes.c_uint64, dp]
            L.oracle_philox4x32.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint32)]
            L.oracle_exp_fixed.argtypes = [ctypes.c_double]
            L.oracle_exp_fixed.restype = ctypes.c_double
            L.oracle_reaction.argtypes = [ctypes.c_double] * 4 + [i]
            L.oracle_reaction.restype = ctypes.c_double
            L.oracle_scale_to_peak.argtypes = [ctypes.c_long, dp, ctypes.c_double, dp]
            L.oracle_scale_to_peak.restype = i
            L.oracle_ssim.argtypes = [i, i, dp, dp, ctypes.c_double]
            L.oracle_ssim.restype = ctypes.c_double
            _lib = L
    return _lib


def _d(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def rot180(k) -> np.ndarray:
    k = _d(k)
    out = np.empty_like(k)
    lib().oracle_rot180(k.shape[0], _p(k), _p(out))
    return out


def conv2d_sym(x, k) -> np.ndarray:
    x, k = _d(x), _d(k)
    out = np.empty_like(x)
    lib().oracle_conv2d_sym(x.shape[0], x.shape[1], _p(x), k.shape[0], _p(k), _p(out))
    return out


def conv2d_adjoint(y, k) -> np.ndarray:
    y, k = _d(y), _d(k)
    out = np.empty_like(y)
    lib().oracle_conv2d_adjoint(y.shape[0], y.shape[1], _p(y), k.shape[0], _p(k), _p(out))
    return out


def phi(w, mu0: float, step: float, gamma: float, z) -> np.ndarray:
    w = _d(w)
    L = lib()
    zz = np.asarray(z, dtype=np.float64)
    out = np.array([L.oracle_phi(w.shape[0], _p(w), float(mu0), float(step), float(gamma), float(v))
                    for v in zz.ravel()])
    return out.reshape(zz.shape)


def reaction(u, ut, f, lam, kind: int) -> np.ndarray:
    """The stage's pointwise reaction (oracle_reaction) on arrays."""
    u, ut, f = np.broadcast_arrays(*(np.asarray(x, np.float64) for x in (u, ut, f)))
    L = lib()
    out = np.array([L.oracle_reaction(float(a), float(b), float(c), float(lam), int(kind))
                    for a, b, c in zip(u.ravel(), ut.ravel(), f.ravel())])
    return out.reshape(u.shape)


def prox(ut, lam, f) -> np.ndarray:
    ut, lam, f = np.broadcast_arrays(np.asarray(ut, np.float64), np.asarray(lam, np.float64),
                                     np.asarray(f, np.float64))
    L = lib()
    out = np.array([L.oracle_prox(float(a), float(b), float(c))
                    for a, b, c in zip(ut.ravel(), lam.ravel(), f.ravel())])
    return out.reshape(ut.shape)


def _model_arrays(model):
    return (_d(model.filters), _d(model.rbf_w), _d(model.rbf_mu0), _d(model.rbf_step),
            _d(model.rbf_gamma), _d(model.lam))


def stage(u, f, model, t: int = 0, boundary: int = BOUNDARY_EXPLICIT, phi_mode: int = PHI_RBF,
          return_u_tilde: bool = False, reaction: int = REACTION_PROX):
    """One stage of Eq.13 (or Eq.3 with another reaction) with params[t]."""
    u, f = _d(u), _d(f)
    H, W = u.shape
    filt, w, mu0, step, gam, lam = _model_arrays(model)
    Nk, m, M = filt.shape[1], filt.shape[2], w.shape[2]
    out = np.empty_like(u)
    ut = np.empty_like(u)
    lib().oracle_stage(H, W, _p(u), _p(f), Nk, m, M, _p(_d(filt[t])), _p(_d(w[t])),
                       _p(_d(mu0[t])), _p(_d(step[t])), _p(_d(gam[t])), float(lam[t]),
                       boundary, phi_mode, reaction, _p(out), _p(ut))
    return (out, ut) if return_u_tilde else out


def denoise(f, model, boundary: int = BOUNDARY_EXPLICIT, phi_mode: int = PHI_RBF,
            reaction: int = REACTION_PROX) -> np.ndarray:
    """u_T for one image f [H][W] (or a batch [B][H][W], looped)."""
    f = _d(f)
    if f.ndim == 3:
        return np.stack([denoise(fi, model, boundary, phi_mode, reaction) for fi in f])
    H, W = f.shape
    filt, w, mu0, step, gam, lam = _model_arrays(model)
    T, Nk, m, M = filt.shape[0], filt.shape[1], filt.shape[2], w.shape[2]
    out = np.empty_like(f)
    lib().oracle_denoise(H, W, _p(f), T, Nk, m, M, _p(filt), _p(w), _p(mu0), _p(step), _p(gam),
                         _p(lam), boundary, phi_mode, reaction, _p(out))
    return out


def loss_grad(f, u_gt, model, boundary: int = BOUNDARY_EXPLICIT):
    """Loss 1/2 ||u_T - u_gt||^2 (P Eq.6) and its gradient (P Eq.14-20) for one image.
    Returns (loss, d_filters [T][Nk][k][k], d_rbf_w [T][Nk][M], d_lambda [T]).  Summed
    over a batch [B][H][W] when given."""
    f, g = _d(f), _d(u_gt)
    if f.ndim == 3:
        parts = [loss_grad(fi, gi, model, boundary) for fi, gi in zip(f, g)]
        return (sum(p[0] for p in parts), sum(p[1] for p in parts), sum(p[2] for p in parts),
                sum(p[3] for p in parts))
    H, W = f.shape
    filt, w, mu0, step, gam, lam = _model_arrays(model)
    T, Nk, m, M = filt.shape[0], filt.shape[1], filt.shape[2], w.shape[2]
    gf, gw, gl = np.zeros_like(filt), np.zeros_like(w), np.zeros_like(lam)
    loss = lib().oracle_loss_grad(H, W, _p(f), _p(g), T, Nk, m, M, _p(filt), _p(w), _p(mu0), _p(step),
                                  _p(gam), _p(lam), boundary, _p(gf), _p(gw), _p(gl))
    return float(loss), gf, gw, gl


def denoise_window(f, model, y0: int, y1: int, x0: int, x1: int,
                   boundary: int = BOUNDARY_EXPLICIT, reaction: int = REACTION_PROX) -> np.ndarray:
    """u_T on the window [y0,y1) x [x0,x1) of a large image, computed exactly on a
    crop with a 2rT dependency margin (pin P12: the output depends on the input
    only within radius 2rT; crop edges on true image edges need no margin)."""
    f = np.asarray(f)
    H, W = f.shape
    R = 2 * (model.k // 2) * model.T
    cy0, cy1 = max(0, y0 - R), min(H, y1 + R)
    cx0, cx1 = max(0, x0 - R), min(W, x1 + R)
    u = denoise(f[cy0:cy1, cx0:cx1], model, boundary, reaction=reaction)
    return u[y0 - cy0:y1 - cy0, x0 - cx0:x1 - cx0]


def sample_poisson(u, seed: int) -> np.ndarray:
    """f ~ Poisson(u) per pixel (P Eq.1) with the shared counter-based generator
    (Philox4x32-10, counter = flat pixel index of the [B][H][W] array)."""
    u = _d(u)
    shp = u.shape
    u3 = u.reshape((-1,) + shp[-2:]) if u.ndim >= 2 else u.reshape(1, 1, -1)
    out = np.empty_like(u3)
    lib().oracle_sample_poisson(u3.shape[0], u3.shape[1], u3.shape[2], _p(np.ascontiguousarray(u3)),
                                ctypes.c_uint64(seed), _p(out))
    return out.reshape(shp)


def philox4x32(counter: int, seed: int) -> np.ndarray:
    out = (ctypes.c_uint32 * 4)()
    lib().oracle_philox4x32(ctypes.c_uint64(counter), ctypes.c_uint64(seed), out)
    return np.array(list(out), dtype=np.uint32)


def exp_fixed(x: float) -> float:
    return lib().oracle_exp_fixed(float(x))


def psnr(u, clean, peak: float) -> float:
    """10 log10(peak^2 / MSE), unclamped (S l.374 after the 255/peak rescale)."""
    mse = float(np.mean((np.asarray(u, np.float64) - np.asarray(clean, np.float64)) ** 2))
    return float("inf") if mse == 0 else 10.0 * np.log10(peak * peak / mse)


def scale_to_peak(x, peak: float) -> np.ndarray:
    """x * peak / max(x) (S l.351-358); ValueError for an all-zero or negative image."""
    x = _d(x)
    out = np.empty_like(x)
    if lib().oracle_scale_to_peak(x.size, _p(x), float(peak), _p(out)) != 0:
        raise ValueError("scale_to_peak: all-zero or negative image")
    return out


def ssim(u, clean, peak: float) -> float:
    """Mean SSIM over the valid 11x11 Gaussian (sigma 1.5) windows after the 255/peak
    rescale (S l.381-389; reading M2)."""
    u, c = _d(u), _d(clean)
    if u.shape != c.shape or u.ndim != 2:
        raise ValueError("ssim: two images of the same [H][W] shape")
    r = lib().oracle_ssim(u.shape[0], u.shape[1], _p(u), _p(c), float(peak))
    if r == -1.0:
        raise ValueError("ssim: image smaller than the 11x11 window")
    return float(r)


def num_threads() -> int:
    v = os.environ.get("OMP_NUM_THREADS")
    return int(v) if v else (os.cpu_count() or 1)
