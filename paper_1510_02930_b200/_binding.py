"""ctypes binding of libtnrd.so (include/tnrd.h).  Argument marshalling only:
every step of the computation runs in the library's sm_100a kernels.

Functions keep the ABI names (tnrd_create, tnrd_set_stage_params, tnrd_denoise,
tnrd_destroy, ...).  Tensors are torch CUDA tensors (device memory and streams
come from PyTorch); host arrays are numpy.  The `TNRD` class bundles a handle
with a model for convenience.

There is no fallback: if libtnrd.so is missing or fails to load, importing
this module raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TNRD_LIB_OVERRIDE") or os.path.join(_HERE, "libtnrd.so")  # override: dev experiments only

TNRD_OK = 0
STATUS = {0: "TNRD_OK", 1: "TNRD_EINVAL", 2: "TNRD_ESTATE", 3: "TNRD_ENOMEM", 4: "TNRD_ECUDA",
          5: "TNRD_ENCCL", 6: "TNRD_EUNSUPPORTED"}
BC_SYMMETRIC_EXPLICIT = 0
BC_SYMMETRIC_ADJOINT = 1
PHI_EXACT = 0
PHI_TABLE = 1
REACTION_POISSON_PROX = 0
REACTION_GAUSSIAN = 1
REACTION_POISSON_GRADIENT = 2
ENGINE_AUTO = 0      # tnrd_engine: tensor cores where they apply, else FP32
ENGINE_FP32 = 1
ENGINE_TENSOR = 2


class TNRDError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class tnrd_desc(ctypes.Structure):
    _fields_ = [("T", ctypes.c_int), ("n_filters", ctypes.c_int), ("ksize", ctypes.c_int),
                ("n_rbf", ctypes.c_int), ("boundary", ctypes.c_int), ("phi_mode", ctypes.c_int),
                ("device", ctypes.c_int), ("reaction", ctypes.c_int)]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() "
                          "(python -m paper_1510_02930_b200._build)")
    if not os.environ.get("TNRD_NCCL_LIB"):
        try:
            from ._build import nccl_library
            p = nccl_library()
            if os.path.exists(p):
                os.environ["TNRD_NCCL_LIB"] = p
        except Exception:
            pass
    L = ctypes.CDLL(LIB_PATH)
    vp, i, ll, f = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_float
    fp = ctypes.POINTER(ctypes.c_float)
    sigs = {
        "tnrd_abi_version": ([], i),
        "tnrd_status_string": ([i], ctypes.c_char_p),
        "tnrd_create": ([ctypes.POINTER(tnrd_desc), ctypes.POINTER(vp)], i),
        "tnrd_set_stage_params": ([vp, i, fp, fp, fp, fp, fp, f], i),
        "tnrd_denoise": ([vp, vp, vp, i, i, i, ll, fp, vp], i),
        "tnrd_denoise_host": ([vp, fp, fp, i, i, i, fp, vp], i),
        "tnrd_destroy": ([vp], i),
        "tnrd_last_error": ([vp], ctypes.c_char_p),
        "tnrd_launch_count": ([vp], ctypes.c_ulonglong),
        "tnrd_nccl_unique_id": ([vp], i),
        "tnrd_comm_init": ([vp, vp, i, i], i),
        "tnrd_denoise_slab": ([vp, vp, vp, i, i, i, i, ll, f, vp], i),
        "tnrd_denoise_slabs_loopback": ([vp, vp, vp, i, i, ll, i, vp], i),
        "tnrd_denoise_slabs_nccl_self": ([vp, vp, vp, i, i, ll, i, vp], i),
        "tnrd_set_profiling": ([vp, i], i),
        "tnrd_get_launch_times": ([vp, fp, i, ctypes.POINTER(i)], i),
        "tnrd_debug_phi": ([vp, i, i, vp, vp, ll, vp], i),
        "tnrd_debug_prox": ([vp, vp, f, vp, ll, vp], i),
        "tnrd_loss_grad": ([vp, vp, vp, i, i, i, ll, fp, fp, fp, ctypes.POINTER(ctypes.c_double), vp], i),
        "tnrd_sample_poisson": ([vp, vp, i, i, i, ll, ctypes.c_ulonglong, vp], i),
        "tnrd_psnr": ([vp, vp, i, i, i, ll, fp, ctypes.POINTER(ctypes.c_double), vp], i),
        "tnrd_scale_to_peak": ([vp, vp, i, i, i, ll, fp, vp], i),
        "tnrd_comm_wait": ([vp, vp, i], i),
        "tnrd_ssim": ([vp, vp, i, i, i, ll, fp, ctypes.POINTER(ctypes.c_double), vp], i),
        "tnrd_set_engine": ([vp, i], i),
        "tnrd_engine_for": ([vp, i, i, i], i),
        "tnrd_set_grad_chunk": ([vp, i], i),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    return L


_lib = _load()
EXPORTED = (
    "tnrd_abi_version", "tnrd_status_string", "tnrd_create", "tnrd_set_stage_params",
    "tnrd_denoise", "tnrd_denoise_host", "tnrd_destroy", "tnrd_last_error", "tnrd_launch_count",
    "tnrd_nccl_unique_id", "tnrd_comm_init", "tnrd_denoise_slab", "tnrd_denoise_slabs_loopback",
    "tnrd_denoise_slabs_nccl_self",
    "tnrd_set_profiling", "tnrd_get_launch_times", "tnrd_debug_phi", "tnrd_debug_prox", "tnrd_loss_grad",
    "tnrd_sample_poisson", "tnrd_psnr", "tnrd_scale_to_peak", "tnrd_ssim", "tnrd_comm_wait", "tnrd_set_engine", "tnrd_engine_for", "tnrd_set_grad_chunk",
)


def lib() -> ctypes.CDLL:
    return _lib


def _check(status: int, handle=None):
    if status != TNRD_OK:
        msg = _lib.tnrd_last_error(handle)
        raise TNRDError(status, msg.decode() if msg else "")


def _f32p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def _host_f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def _stream_ptr(stream) -> Optional[int]:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def _dev_ptr(t) -> int:
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32):
        raise TypeError("expected a float32 CUDA tensor")
    return t.data_ptr()


# ------------------------------------------------------------------ ABI-named functions
def tnrd_abi_version() -> int:
    return _lib.tnrd_abi_version()


def tnrd_status_string(status: int) -> str:
    return _lib.tnrd_status_string(int(status)).decode()


def tnrd_create(T: int, n_filters: int, ksize: int, n_rbf: int, boundary: int = 0,
                phi_mode: int = 0, device: int = 0, reaction: int = 0) -> int:
    d = tnrd_desc(T, n_filters, ksize, n_rbf, boundary, phi_mode, device, reaction)
    h = ctypes.c_void_p()
    _check(_lib.tnrd_create(ctypes.byref(d), ctypes.byref(h)))
    return h.value


def tnrd_set_stage_params(h: int, t: int, filters, rbf_w, rbf_mu0, rbf_step, rbf_gamma, lam) -> None:
    arrs = [_host_f32(x) for x in (filters, rbf_w, rbf_mu0, rbf_step, rbf_gamma)]
    _check(_lib.tnrd_set_stage_params(h, t, *[_f32p(a) for a in arrs], float(lam)), h)


def tnrd_denoise(h: int, f, u, peak: Optional[Sequence[float]] = None, stream=None) -> None:
    """f, u: float32 CUDA tensors [B][H][W] or [H][W] (row stride = stride(-2))."""
    if f.dim() == 2:
        f, u = f.unsqueeze(0), u.unsqueeze(0)
    B, H, W = f.shape
    ld = f.stride(1)
    if f.stride(2) != 1 or u.stride(2) != 1 or u.stride(1) != ld or u.shape != f.shape or \
            (B > 1 and (f.stride(0) != H * ld or u.stride(0) != H * ld)):
        raise ValueError("f and u must be [B][H][W] with unit column stride and equal row strides")
    pk = None if peak is None else _host_f32(peak)
    _check(_lib.tnrd_denoise(h, _dev_ptr(f), _dev_ptr(u), B, H, W, ld,
                             None if pk is None else _f32p(pk), _stream_ptr(stream)), h)


def tnrd_denoise_host(h: int, f_host: np.ndarray, u_host: np.ndarray,
                      peak: Optional[Sequence[float]] = None, stream=None) -> None:
    """Host arrays [B][H][W] float32 C-contiguous (pinned memory if possible)."""
    f3 = f_host if f_host.ndim == 3 else f_host[None]
    u3 = u_host if u_host.ndim == 3 else u_host[None]
    assert f3.dtype == np.float32 and u3.dtype == np.float32
    assert f3.flags.c_contiguous and u3.flags.c_contiguous and f3.shape == u3.shape
    B, H, W = f3.shape
    pk = None if peak is None else _host_f32(peak)
    _check(_lib.tnrd_denoise_host(h, _f32p(f3), _f32p(u3), B, H, W,
                                  None if pk is None else _f32p(pk), _stream_ptr(stream)), h)


def tnrd_denoise_host_ptr(h: int, f_ptr: int, u_ptr: int, B: int, H: int, W: int,
                          peak: Optional[np.ndarray] = None, stream=None) -> None:
    """Same as tnrd_denoise_host on raw host addresses (e.g. pinned torch CPU tensors)."""
    fp = ctypes.cast(f_ptr, ctypes.POINTER(ctypes.c_float))
    up = ctypes.cast(u_ptr, ctypes.POINTER(ctypes.c_float))
    _check(_lib.tnrd_denoise_host(h, fp, up, B, H, W, None if peak is None else _f32p(peak),
                                  _stream_ptr(stream)), h)


def tnrd_destroy(h: int) -> None:
    if h:
        _check(_lib.tnrd_destroy(h))


def tnrd_last_error(h: Optional[int] = None) -> str:
    m = _lib.tnrd_last_error(h)
    return m.decode() if m else ""


def tnrd_launch_count(h: int) -> int:
    return int(_lib.tnrd_launch_count(h))


def tnrd_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.tnrd_nccl_unique_id(buf))
    return buf.raw


def tnrd_comm_init(h: int, uid: bytes, rank: int, nranks: int) -> None:
    buf = ctypes.create_string_buffer(bytes(uid), 128)
    _check(_lib.tnrd_comm_init(h, buf, rank, nranks), h)


def tnrd_denoise_slab(h: int, f_slab, u_slab, H_global: int, row0: int, peak: float,
                      stream=None) -> None:
    rows, W = f_slab.shape
    _check(_lib.tnrd_denoise_slab(h, _dev_ptr(f_slab), _dev_ptr(u_slab), H_global, W, row0, rows,
                                  f_slab.stride(0), float(peak), _stream_ptr(stream)), h)


def tnrd_denoise_slabs_loopback(h: int, f, u, nslabs: int, stream=None) -> None:
    H, W = f.shape
    _check(_lib.tnrd_denoise_slabs_loopback(h, _dev_ptr(f), _dev_ptr(u), H, W, f.stride(0),
                                            nslabs, _stream_ptr(stream)), h)


def tnrd_denoise_slabs_nccl_self(h: int, f, u, nslabs: int, stream=None) -> None:
    H, W = f.shape
    _check(_lib.tnrd_denoise_slabs_nccl_self(h, _dev_ptr(f), _dev_ptr(u), H, W, f.stride(0),
                                             nslabs, _stream_ptr(stream)), h)


def tnrd_set_engine(h: int, engine: int) -> None:
    _check(_lib.tnrd_set_engine(h, engine), h)


def tnrd_set_grad_chunk(h: int, max_filters: int) -> None:
    _check(_lib.tnrd_set_grad_chunk(h, int(max_filters)), h)


def tnrd_engine_for(h: int, B: int, H: int, W: int) -> int:
    return int(_lib.tnrd_engine_for(h, B, H, W))


def tnrd_set_profiling(h: int, enable: bool) -> None:
    _check(_lib.tnrd_set_profiling(h, 1 if enable else 0), h)


def tnrd_get_launch_times(h: int, max_n: int = 4096) -> np.ndarray:
    buf = np.zeros(max_n, np.float32)
    n = ctypes.c_int(0)
    _check(_lib.tnrd_get_launch_times(h, _f32p(buf), max_n, ctypes.byref(n)), h)
    return buf[:min(n.value, max_n)].copy()


def tnrd_debug_phi(h: int, t: int, i: int, v, out, stream=None) -> None:
    _check(_lib.tnrd_debug_phi(h, t, i, _dev_ptr(v), _dev_ptr(out), v.numel(), _stream_ptr(stream)), h)


def tnrd_debug_prox(ut, f, lam: float, out, stream=None) -> None:
    _check(_lib.tnrd_debug_prox(_dev_ptr(ut), _dev_ptr(f), float(lam), _dev_ptr(out), ut.numel(),
                                _stream_ptr(stream)))


def tnrd_loss_grad(h: int, f, u_gt, T: int, Nk: int, k: int, M: int, stream=None):
    """loss = 1/2 ||u_T - u_gt||^2 and its gradient (P Eq.14-20) for f, u_gt float32
    CUDA tensors [B][H][W] or [H][W].  Returns (loss, d_filters [T][Nk][k][k],
    d_rbf_w [T][Nk][M], d_lambda [T]) as numpy arrays."""
    if f.dim() == 2:
        f, u_gt = f.unsqueeze(0), u_gt.unsqueeze(0)
    B, H, W = f.shape
    if f.stride(2) != 1 or u_gt.stride() != f.stride() or u_gt.shape != f.shape:
        raise ValueError("f and u_gt must be [B][H][W] with equal strides")
    gf = np.zeros((T, Nk, k, k), np.float32)
    gw = np.zeros((T, Nk, M), np.float32)
    gl = np.zeros(T, np.float32)
    loss = ctypes.c_double(0.0)
    _check(_lib.tnrd_loss_grad(h, _dev_ptr(f), _dev_ptr(u_gt), B, H, W, f.stride(1), _f32p(gf), _f32p(gw),
                               _f32p(gl), ctypes.byref(loss), _stream_ptr(stream)), h)
    return loss.value, gf, gw, gl


def tnrd_sample_poisson(u, f=None, seed: int = 0, stream=None):
    """f ~ Poisson(u) (P Eq.1), float32 CUDA tensors [B][H][W] or [H][W]; returns f."""
    import torch
    if f is None:
        f = torch.empty_like(u)
    u3, f3 = (u, f) if u.dim() == 3 else (u.unsqueeze(0), f.unsqueeze(0))
    B, H, W = u3.shape
    if u3.stride(2) != 1 or f3.stride() != u3.stride():
        raise ValueError("u and f must have unit column stride and equal strides")
    _check(_lib.tnrd_sample_poisson(_dev_ptr(u3), _dev_ptr(f3), B, H, W, u3.stride(1), int(seed),
                                    _stream_ptr(stream)))
    return f


def tnrd_psnr(u, clean, peak, stream=None) -> np.ndarray:
    """PSNR per image, 10 log10(peak^2 / MSE) (reading C15)."""
    u3, c3 = (u, clean) if u.dim() == 3 else (u.unsqueeze(0), clean.unsqueeze(0))
    B, H, W = u3.shape
    pk = _host_f32(np.broadcast_to(np.asarray(peak, np.float32), (B,)))
    out = np.zeros(B, np.float64)
    _check(_lib.tnrd_psnr(_dev_ptr(u3), _dev_ptr(c3), B, H, W, u3.stride(1), _f32p(pk),
                          out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _stream_ptr(stream)))
    return out


def tnrd_scale_to_peak(x, peak, out=None, stream=None):
    """out = x * (peak / max(x)) per image, exactly peak at the max (S l.351-358)."""
    x3 = x if x.dim() == 3 else x.unsqueeze(0)
    if out is None:
        out = torch_empty_like(x3)
    o3 = out if out.dim() == 3 else out.unsqueeze(0)
    B, H, W = x3.shape
    if o3.shape != x3.shape or o3.stride(1) != x3.stride(1):
        raise ValueError("out must match x")
    pk = _host_f32(np.broadcast_to(np.asarray(peak, np.float32), (B,)))
    _check(_lib.tnrd_scale_to_peak(_dev_ptr(x3), _dev_ptr(o3), B, H, W, x3.stride(1), _f32p(pk), _stream_ptr(stream)))
    return out


def tnrd_ssim(u, clean, peak, stream=None) -> np.ndarray:
    """Mean SSIM per image over the valid 11x11 Gaussian windows (S l.381-389, reading M2)."""
    u3, c3 = (u, clean) if u.dim() == 3 else (u.unsqueeze(0), clean.unsqueeze(0))
    B, H, W = u3.shape
    pk = _host_f32(np.broadcast_to(np.asarray(peak, np.float32), (B,)))
    out = np.zeros(B, np.float64)
    _check(_lib.tnrd_ssim(_dev_ptr(u3), _dev_ptr(c3), B, H, W, u3.stride(1), _f32p(pk),
                          out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _stream_ptr(stream)))
    return out


def tnrd_comm_wait(h: int, stream=None, timeout_ms: int = -1) -> None:
    """Drain `stream` while polling the communicator's asynchronous error (ENCCL on error
    or timeout; the communicator is then aborted)."""
    _check(_lib.tnrd_comm_wait(h, _stream_ptr(stream), int(timeout_ms)), h)


def torch_empty_like(x):
    import torch
    return torch.empty_like(x)


# ------------------------------------------------------------------ convenience wrapper
class TNRD:
    """A handle plus its model: TNRD(model).denoise(f) -> u (torch CUDA tensors).

    `model` is any object with fields filters [T][Nk][k][k], rbf_w [T][Nk][M],
    rbf_mu0 / rbf_step / rbf_gamma [T][Nk], lam [T] (e.g. synth.Model).
    """

    def __init__(self, model, boundary: int = BC_SYMMETRIC_EXPLICIT, device: int = 0, phi_mode: int = PHI_EXACT,
                 reaction: int = REACTION_POISSON_PROX, engine: int = 0):
        T, Nk, k, _ = np.shape(model.filters)
        M = np.shape(model.rbf_w)[2]
        self.T, self.Nk, self.k, self.M = int(T), int(Nk), int(k), int(M)
        self.device = device
        self.h = tnrd_create(self.T, self.Nk, self.k, self.M, boundary, phi_mode, device, reaction)
        for t in range(self.T):
            tnrd_set_stage_params(self.h, t, model.filters[t], model.rbf_w[t], model.rbf_mu0[t],
                                  model.rbf_step[t], model.rbf_gamma[t], model.lam[t])
        tnrd_set_engine(self.h, engine)

    def engine_for(self, B: int, H: int, W: int) -> int:
        """ENGINE_FP32 or ENGINE_TENSOR: the engine a B x H x W denoise runs on."""
        return tnrd_engine_for(self.h, B, H, W)

    def denoise(self, f, u=None, peak=None, stream=None):
        import torch
        if u is None:
            u = torch.empty_like(f)
        tnrd_denoise(self.h, f, u, peak, stream)
        return u

    def denoise_host(self, f_host: np.ndarray, peak=None) -> np.ndarray:
        u = np.empty_like(f_host)
        tnrd_denoise_host(self.h, f_host, u, peak)
        return u

    def loss_grad(self, f, u_gt, stream=None):
        """(loss, d_filters, d_rbf_w, d_lambda) of 1/2 ||u_T - u_gt||^2 (P Eq.6, 14-20)."""
        return tnrd_loss_grad(self.h, f, u_gt, self.T, self.Nk, self.k, self.M, stream)

    @property
    def launches(self) -> int:
        return tnrd_launch_count(self.h)

    def close(self):
        if self.h:
            tnrd_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
