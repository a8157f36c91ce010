"""Faithful fp32 CPU emulation of the inference pass -- TEST INFRASTRUCTURE ONLY.

Used by pin P16 (the fp32 noise-floor gate): every arithmetic
step of P Eq.13 (l.326-333) is done in IEEE float32 with sequential tap sums,
float32 exp and float32 sqrt.  If this emulation drifts from the double oracle
by more than a tenth of the parity tolerance (1e-4 * peak), the config's
parameters are ill-conditioned for fp32, not the CUDA kernel wrong.

Independent of tnrd_oracle.c: the boundary comes from numpy.pad(mode="symmetric")
(half-sample mirror, S l.73), the RBF sum from numpy float32 exp.
"""
from __future__ import annotations

import numpy as np

f32 = np.float32


def _conv_sym_f32(x: np.ndarray, k: np.ndarray) -> np.ndarray:
    """True convolution with symmetric extension, taps summed sequentially in fp32."""
    m = k.shape[0]
    r = m // 2
    H, W = x.shape
    xe = np.pad(x, r, mode="symmetric")
    out = np.zeros((H, W), f32)
    for a in range(-r, r + 1):
        for b in range(-r, r + 1):
            # out(p,q) += k[a+r][b+r] * xe(p - a + r, q - b + r)
            out += k[a + r, b + r] * xe[r - a:r - a + H, r - b:r - b + W]
    return out


def _phi_f32(v: np.ndarray, w: np.ndarray, mu0, step, gamma) -> np.ndarray:
    out = np.zeros_like(v)
    inv = f32(1.0) / (f32(2.0) * f32(gamma) * f32(gamma))
    for j in range(w.shape[0]):
        d = v - (f32(mu0) + f32(j) * f32(step))
        out += w[j] * np.exp(-(d * d) * inv)
    return out


def _prox_f32(ut, lam, f):
    lam = f32(lam)
    delta = ut - lam
    sigma = np.sqrt(delta * delta + f32(4.0) * lam * f)
    with np.errstate(divide="ignore", invalid="ignore"):
        neg = np.where(f == 0, f32(0.0), f32(2.0) * lam * f / (sigma - delta))
    return np.where(delta >= 0, f32(0.5) * (delta + sigma), neg).astype(f32)


def denoise_f32(f: np.ndarray, model) -> np.ndarray:
    """u_T in float32, boundary R1 (explicit rotated-kernel convolution, P l.302-311)."""
    f = np.asarray(f, f32)
    u = f.copy()
    for s in range(model.T):
        d = np.zeros_like(u)
        for i in range(model.Nk):
            k = model.filters[s, i].astype(f32)
            v = _conv_sym_f32(u, k)
            w = _phi_f32(v, model.rbf_w[s, i].astype(f32), model.rbf_mu0[s, i],
                         model.rbf_step[s, i], model.rbf_gamma[s, i])
            d += _conv_sym_f32(w, k[::-1, ::-1].copy())
        u = _prox_f32(u - d, model.lam[s], f)
    return u
