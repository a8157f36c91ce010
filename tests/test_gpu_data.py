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
