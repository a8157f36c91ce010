"""GPU Poisson sampler and PSNR against the oracle.

The sampler's integer counts are compared bit-exactly: both sides implement the same
counter-based draw (Philox4x32-10 keyed by the seed, counter = flat pixel index,
inversion in double with the same fixed exp), so the decision is taken in the same
precision with the same operations.
"""
import numpy as np
import pytest

import oracle
from synth import make_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def test_sample_poisson_bit_exact_vs_oracle(torch_cuda):
    import paper_1510_02930_b200 as P
    torch = torch_cuda
    rng = np.random.default_rng(5)
    u = np.concatenate([make_problem(2).clean,                       # peak-4 image, many small means
                        rng.uniform(0, 45, size=(1, 256, 256)).astype(np.float32)])
    u[1, :3, :3] = 0.0
    for seed in (0, 151002930, 2**63 + 12345):
        f = P.tnrd_sample_poisson(torch.from_numpy(u).cuda(), seed=seed).cpu().numpy()
        ref = oracle.sample_poisson(u.astype(np.float64), seed)
        assert np.array_equal(f.astype(np.float64), ref), (seed, int(np.sum(f != ref)))
    assert np.all(f[1, :3, :3] == 0)


def test_sample_poisson_strided_and_rejects_negative(torch_cuda):
    import paper_1510_02930_b200 as P
    torch = torch_cuda
    u = torch.full((2, 40, 64), 3.0, device="cuda")[:, :, :50]  # row stride 64
    f = torch.zeros((2, 40, 64), device="cuda")[:, :, :50]
    P.tnrd_sample_poisson(u, f, seed=7)
    ref = oracle.sample_poisson(np.full((2, 40, 50), 3.0), 7)
    assert np.array_equal(f.cpu().numpy().astype(np.float64), ref)
    bad = torch.full((1, 8, 8), 1.0, device="cuda")
    bad[0, 3, 3] = -0.5
    with pytest.raises(P.TNRDError):
        P.tnrd_sample_poisson(bad, seed=1)


def test_psnr_matches_oracle(torch_cuda):
    import paper_1510_02930_b200 as P
    torch = torch_cuda
    p = make_problem(4, batch=5)
    rng = np.random.default_rng(6)
    u = (p.clean + rng.normal(0, 0.05, size=p.clean.shape)).astype(np.float32)
    got = P.tnrd_psnr(torch.from_numpy(u).cuda(), torch.from_numpy(p.clean).cuda(), p.peaks)
    for b in range(5):
        assert abs(got[b] - oracle.psnr(u[b], p.clean[b], float(p.peaks[b]))) < 1e-9
    same = P.tnrd_psnr(torch.from_numpy(p.clean).cuda(), torch.from_numpy(p.clean).cuda(), p.peaks)
    assert np.all(np.isinf(same))


def test_scale_to_peak_matches_oracle(torch_cuda):
    """GPU peak scaling (S l.351-358) against the oracle: max(out) == peak exactly, every
    pixel within 1 fp32 rounding of x * (peak / max) (a product of two correctly rounded
    fp32 operations: relative error < 2^-22), strided rows, in place, SPEC examples."""
    import paper_1510_02930_b200 as P
    torch = torch_cuda
    rng = np.random.default_rng(11)
    x = rng.gamma(2.0, 40.0, size=(4, 70, 90)).astype(np.float32)
    x[2] = 255.0                                       # constant image -> constant peak
    peaks = np.array([0.1, 1.0, 4.0, 40.0], np.float32)
    out = P.tnrd_scale_to_peak(torch.from_numpy(x).cuda(), peaks).cpu().numpy()
    for b in range(4):
        ref = oracle.scale_to_peak(x[b].astype(np.float64), float(peaks[b]))
        assert out[b].max() == peaks[b]
        assert np.all(np.abs(out[b] - ref) <= 2.0 ** -22 * np.abs(ref) + 1e-30), b
    assert np.all(out[2] == peaks[2])
    # strided rows, in place; peak == max is the identity
    big = torch.from_numpy(rng.uniform(0, 9, size=(2, 33, 64)).astype(np.float32)).cuda()
    view = big[:, :, :41]
    mx = view.amax(dim=(1, 2)).cpu().numpy()
    before = view.clone()
    P.tnrd_scale_to_peak(view, mx, out=view)
    assert torch.equal(view, before)
    two = torch.tensor([[[0.0, 255.0], [255.0, 0.0]]], device="cuda")
    assert torch.equal(P.tnrd_scale_to_peak(two, 1.0), two / 255.0)
    with pytest.raises(P.TNRDError):
        P.tnrd_scale_to_peak(torch.zeros((1, 8, 8), device="cuda"), 1.0)
    neg = torch.ones((1, 8, 8), device="cuda")
    neg[0, 2, 2] = -1.0
    with pytest.raises(P.TNRDError):
        P.tnrd_scale_to_peak(neg, 1.0)


def test_ssim_matches_oracle(torch_cuda):
    """GPU SSIM (S l.381-389, reading M2) against the oracle on denoised-like images:
    both sum the same window terms in double, so they agree to 1e-12; identity gives 1;
    strided rows; images smaller than the window are rejected."""
    import paper_1510_02930_b200 as P
    torch = torch_cuda
    p = make_problem(4, batch=5)
    rng = np.random.default_rng(12)
    u = np.clip(p.clean + rng.normal(0, 0.1, size=p.clean.shape) * p.peaks[:, None, None], 0, None).astype(np.float32)
    got = P.tnrd_ssim(torch.from_numpy(u).cuda(), torch.from_numpy(p.clean).cuda(), p.peaks)
    for b in range(5):
        ref = oracle.ssim(u[b], p.clean[b], float(p.peaks[b]))
        assert abs(got[b] - ref) < 1e-12, (b, got[b], ref)
    same = P.tnrd_ssim(torch.from_numpy(u[:2]).cuda(), torch.from_numpy(u[:2]).cuda(), p.peaks[:2])
    assert np.all(np.abs(same - 1.0) < 1e-12)
    a = torch.from_numpy(rng.uniform(0, 4, size=(1, 30, 48)).astype(np.float32)).cuda()
    c = torch.from_numpy(rng.uniform(0, 4, size=(1, 30, 48)).astype(np.float32)).cuda()
    got = P.tnrd_ssim(a[:, :, :37], c[:, :, :37], 4.0)
    ref = oracle.ssim(a[0, :, :37].cpu().numpy(), c[0, :, :37].cpu().numpy(), 4.0)
    assert abs(got[0] - ref) < 1e-12
    with pytest.raises(P.TNRDError):
        P.tnrd_ssim(a[:, :10, :], c[:, :10, :], 4.0)
