"""GPU training gradient (tnrd_loss_grad) against the oracle's analytic
gradient of P Eq.14-20, which is itself pinned by central finite differences
(tests/test_oracle_pins.py::test_loss_grad_matches_central_finite_differences).

Tolerance: the fp32 forward differs from the double oracle by
~1e-6 relative, and each gradient entry is a sum over B*H*W pixels accumulated in
fp32 per block and in double across blocks.  Measured: <= 2.1e-6 of max|g| per
array (up to the full 48x7x7, T=8 model); required, per parameter array and
stage: max|g_gpu - g_ref| <= 2e-5 * max|g_ref|, and the loss to 1e-5 relative.
"""
import numpy as np
import pytest

import oracle
from synth import make_model

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _case(seed, B, H, W, T, Nk, k, M, w_scale=1.0):
    rng = np.random.default_rng(seed)
    f = rng.poisson(3.0, size=(B, H, W)).astype(np.float32)
    gt = (f + rng.normal(0, 0.5, size=f.shape)).astype(np.float32)
    m = make_model(rng, T, Nk, k, M, float(f.max()))
    m.rbf_w *= np.float32(w_scale)
    return f, gt, m


def _check(got, ref, what):
    scale = float(np.max(np.abs(ref)))
    err = float(np.max(np.abs(np.asarray(got, np.float64) - ref)))
    assert err <= 2e-5 * scale + 1e-12, f"{what}: max err {err:.3e} vs scale {scale:.3e}"


@pytest.mark.parametrize("boundary", [0, 1])
@pytest.mark.parametrize("B,H,W,T,Nk,k,M", [(2, 24, 20, 2, 4, 3, 15), (1, 33, 40, 3, 6, 5, 31),
                                           (1, 40, 36, 2, 8, 7, 63), (1, 96, 80, 8, 48, 7, 63),
                                           # tensor-core banks: (k, N_k) = (3, 8), (5, 24), (7, 48)
                                           (2, 37, 70, 2, 8, 3, 63), (1, 45, 131, 2, 24, 5, 63),
                                           (2, 70, 67, 3, 48, 7, 63)])
def test_loss_grad_parity(torch_cuda, B, H, W, T, Nk, k, M, boundary):
    import paper_1510_02930_b200 as P
    torch = torch_cuda
    f, gt, m = _case(5 + k + T, B, H, W, T, Nk, k, M, w_scale=3.0)
    eng = P.TNRD(m, boundary=boundary)
    loss, gf, gw, gl = eng.loss_grad(torch.from_numpy(f).cuda(), torch.from_numpy(gt).cuda())
    eng.close()
    rl, rf, rw, rlam = oracle.loss_grad(f, gt, m, boundary)
    assert abs(loss - rl) <= 1e-5 * abs(rl), (loss, rl)
    for t in range(T):
        _check(gf[t], rf[t], f"d filters t={t}")
        _check(gw[t], rw[t], f"d rbf_w t={t}")
    _check(gl, rlam, "d lambda")


@pytest.mark.parametrize("boundary", [0, 1])
def test_loss_grad_fp32_engine_on_tensor_shapes(torch_cuda, boundary):
    """ENGINE_FP32 keeps the tape and the backward banks on the CUDA cores for a
    (k, N_k) that has tensor instantiations (AUTO uses them); same bound."""
    import paper_1510_02930_b200 as P
    torch = torch_cuda
    B, H, W, T, Nk, k, M = 1, 45, 131, 2, 24, 5, 63
    f, gt, m = _case(5 + k + T, B, H, W, T, Nk, k, M, w_scale=3.0)
    eng = P.TNRD(m, boundary=boundary, engine=P.ENGINE_FP32)
    assert eng.engine_for(B, H, W) == P.ENGINE_FP32
    loss, gf, gw, gl = eng.loss_grad(torch.from_numpy(f).cuda(), torch.from_numpy(gt).cuda())
    eng.close()
    rl, rf, rw, rlam = oracle.loss_grad(f, gt, m, boundary)
    assert abs(loss - rl) <= 1e-5 * abs(rl), (loss, rl)
    for t in range(T):
        _check(gf[t], rf[t], f"d filters t={t}")
        _check(gw[t], rw[t], f"d rbf_w t={t}")
    _check(gl, rlam, "d lambda")


@pytest.mark.parametrize("Nk,k", [(4, 3), (48, 7)])
def test_loss_grad_is_deterministic_and_batch_additive(torch_cuda, Nk, k):
    """Bitwise reproducible, and the batch gradient is the sum over images (CUDA-core
    and tensor-core banks)."""
    import paper_1510_02930_b200 as P
    torch = torch_cuda
    f, gt, m = _case(9, 3, 20, 24, 2, Nk, k, 15)
    eng = P.TNRD(m)
    a = eng.loss_grad(torch.from_numpy(f).cuda(), torch.from_numpy(gt).cuda())
    b = eng.loss_grad(torch.from_numpy(f).cuda(), torch.from_numpy(gt).cuda())
    assert a[0] == b[0] and all(np.array_equal(x, y) for x, y in zip(a[1:], b[1:]))
    parts = [eng.loss_grad(torch.from_numpy(f[i:i + 1]).cuda(), torch.from_numpy(gt[i:i + 1]).cuda())
             for i in range(3)]
    eng.close()
    for j in (1, 2, 3):
        s = sum(np.asarray(p[j], np.float64) for p in parts)
        assert np.max(np.abs(a[j] - s)) <= 1e-5 * np.max(np.abs(s)) + 1e-9
    assert abs(a[0] - sum(p[0] for p in parts)) <= 1e-6 * abs(a[0])


_KG_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, "tests")
import paper_1510_02930_b200 as P
from test_gpu_grad import _case
B, H, W, T, Nk, k, M, bnd = map(int, sys.argv[1:9])
f, gt, m = _case(11, B, H, W, T, Nk, k, M, w_scale=3.0)
eng = P.TNRD(m, boundary=bnd)
loss, gf, gw, gl = eng.loss_grad(torch.from_numpy(f).cuda(), torch.from_numpy(gt).cuda())
eng.close()
np.save(sys.argv[9], np.stack([np.asarray(g, np.float64) for g in gf]))
"""


@pytest.mark.parametrize("boundary", [0, 1])
def test_filter_gradient_tensor_gemm_vs_cuda_cores(torch_cuda, tmp_path, boundary):
    """The tensor-core filter-gradient GEMM against the CUDA-core tap sums
    (TNRD_GRAD_KG=fp32) on the same tape: same filter gradient to the test bound,
    on a ragged (k, N_k) = (7, 48) batch."""
    import os
    import subprocess
    import sys
    args = ["2", "37", "70", "2", "48", "7", "63", str(boundary)]
    out = {}
    for name, extra in (("tc", {}), ("fp32", {"TNRD_GRAD_KG": "fp32"})):
        env = dict(os.environ, **extra)
        path = str(tmp_path / f"{name}.npy")
        subprocess.run([sys.executable, "-c", _KG_SCRIPT, *args, path], check=True, env=env,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        out[name] = np.load(path)
    a, b = out["tc"], out["fp32"]
    for t in range(a.shape[0]):
        scale = float(np.max(np.abs(b[t])))
        err = float(np.max(np.abs(a[t] - b[t])))
        assert err <= 2e-5 * scale, (t, err, scale)


@pytest.mark.parametrize("F", [1, 5, 16])
def test_loss_grad_multi_chunk(torch_cuda, F):
    """The backward split into chunks of F < N_k filters (tnrd_set_grad_chunk; the
    CUDA-core banks, since the tensor banks need all filters in one chunk): same
    oracle bound, and two calls with the same cap are bitwise equal."""
    import paper_1510_02930_b200 as P
    torch = torch_cuda
    f, gt, m = _case(41 + F, 2, 40, 52, 2, 48, 7, 63, w_scale=3.0)
    eng = P.TNRD(m)
    P.tnrd_set_grad_chunk(eng.h, F)
    ft, gtt = torch.from_numpy(f).cuda(), torch.from_numpy(gt).cuda()
    loss, gf, gw, gl = eng.loss_grad(ft, gtt)
    loss2, gf2, gw2, gl2 = eng.loss_grad(ft, gtt)
    eng.close()
    assert loss == loss2 and np.array_equal(gf, gf2) and np.array_equal(gw, gw2) and np.array_equal(gl, gl2)
    rl, rf, rw, rlam = oracle.loss_grad(f, gt, m, 0)
    assert abs(loss - rl) <= 1e-5 * abs(rl), (loss, rl)
    for t in range(m.T):
        _check(gf[t], rf[t], f"F={F} d filters t={t}")
        _check(gw[t], rw[t], f"F={F} d rbf_w t={t}")
    _check(gl, rlam, f"F={F} d lambda")
