"""GPU parity: the sm_100a path (through the C ABI) against the double-precision
oracle on seeded synthetic inputs.

Bar (BASELINE.json north_star): max |u_gpu - u_oracle| <= 1e-4 * peak per pixel
and |PSNR_gpu - PSNR_oracle| < 0.01 dB, for every image.  Configs C1-C3 are
compared on every pixel; C4 and C5 run at full size in the bench's launch
configuration and are compared on dependency-cone windows (pin P12: the
oracle on a crop with a 2rT margin is exact on the window).
"""
import json
import os

import numpy as np
import pytest

import oracle
from synth import make_model, make_problem, stress_model, zero_model

pytestmark = pytest.mark.gpu

TOL = 1e-4  # x peak
MARGINS = {}  # what -> max|du| / tol, written to $TNRD_PARITY_REPORT (json) if set


@pytest.fixture(scope="module", autouse=True)
def _report():
    yield
    path = os.environ.get("TNRD_PARITY_REPORT")
    if path and MARGINS:
        with open(path, "w") as fh:
            json.dump(MARGINS, fh, indent=1, sort_keys=True)


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(scope="module")
def P():
    import paper_1510_02930_b200 as P
    return P


def _gpu_denoise(P, torch, model, f, boundary=0, peak=None, phi_mode=0, reaction=0, engine=0):
    eng = P.TNRD(model, boundary=boundary, phi_mode=phi_mode, reaction=reaction, engine=engine)
    ft = torch.from_numpy(np.ascontiguousarray(f, np.float32)).cuda()
    u = eng.denoise(ft, peak=peak)
    torch.cuda.synchronize()
    out = u.cpu().numpy()
    eng.close()
    return out


def _assert_parity(u_gpu, u_ref, peak, clean=None, what=""):
    err = float(np.max(np.abs(u_gpu.astype(np.float64) - u_ref)))
    assert np.all(np.isfinite(u_gpu)), what
    MARGINS[what] = max(MARGINS.get(what, 0.0), err / (TOL * peak))
    assert err <= TOL * peak, f"{what}: max|du| = {err:.3e} > {TOL * peak:.1e} ({err / (TOL * peak):.3f} x tol)"
    if clean is not None:
        d = abs(oracle.psnr(u_gpu, clean, peak) - oracle.psnr(u_ref, clean, peak))
        MARGINS[what + " |dPSNR| dB"] = max(MARGINS.get(what + " |dPSNR| dB", 0.0), d)
        assert d < 0.01, f"{what}: dPSNR {d}"
    MARGINS[what] = max(MARGINS.get(what, 0.0), err / (TOL * peak))
    return err / (TOL * peak)


# ------------------------------------------------------------------ full-image configs
@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_full_config_parity(torch_cuda, P, cfg):
    p = make_problem(cfg)
    u_ref = oracle.denoise(p.f[0], p.model)
    u = _gpu_denoise(P, torch_cuda, p.model, p.f, peak=p.peaks)[0]
    _assert_parity(u, u_ref, float(p.peaks[0]), p.clean[0], f"C{cfg}")


@pytest.mark.parametrize("engine", ["fp32", "tensor"])
@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_engine_parity(torch_cuda, P, cfg, engine):
    """Both engines (tnrd_engine) against the oracle on C1-C3, every pixel, and the
    tensor-core engine is the one AUTO picks for these (ksize, N_k) under R1."""
    p = make_problem(cfg)
    e = P.ENGINE_FP32 if engine == "fp32" else P.ENGINE_TENSOR
    eng = P.TNRD(p.model, engine=e)
    assert eng.engine_for(1, *p.f.shape[1:]) == e
    eng.close()
    auto = P.TNRD(p.model)
    assert auto.engine_for(1, *p.f.shape[1:]) == P.ENGINE_TENSOR
    auto.close()
    u_ref = oracle.denoise(p.f[0], p.model)
    u = _gpu_denoise(P, torch_cuda, p.model, p.f, peak=p.peaks, engine=e)[0]
    _assert_parity(u, u_ref, float(p.peaks[0]), p.clean[0], f"C{cfg} engine={engine}")


@pytest.mark.parametrize("M", [9, 31, 100])
def test_tensor_engine_other_rbf_counts(torch_cuda, P, M):
    """The tensor engine with M != 63 Gaussians (unit count and constant layout scale
    with M) against the oracle, 48 x 7 x 7, T = 2."""
    rng = np.random.default_rng(300 + M)
    f = rng.poisson(rng.uniform(0, 4, (1, 90, 75))).astype(np.float32)
    model = make_model(rng, 2, 48, 7, M, float(max(f.max(), 1.0)))
    eng = P.TNRD(model)
    assert eng.engine_for(1, 90, 75) == P.ENGINE_TENSOR
    eng.close()
    u = _gpu_denoise(P, torch_cuda, model, f)[0]
    _assert_parity(u, oracle.denoise(f[0], model), 4.0, what=f"tensor M={M}")


@pytest.mark.parametrize("engine", ["fp32", "tensor"])
@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_r2_boundary_parity(torch_cuda, P, cfg, engine):
    """R2 (exact K^T) on both engines against the oracle, every pixel."""
    p = make_problem(cfg)
    e = P.ENGINE_FP32 if engine == "fp32" else P.ENGINE_TENSOR
    eng = P.TNRD(p.model, boundary=1, engine=e)
    assert eng.engine_for(1, *p.f.shape[1:]) == e
    eng.close()
    u_ref = oracle.denoise(p.f[0], p.model, boundary=oracle.BOUNDARY_ADJOINT)
    u = _gpu_denoise(P, torch_cuda, p.model, p.f, boundary=1, engine=e)[0]
    _assert_parity(u, u_ref, float(p.peaks[0]), p.clean[0], f"C{cfg}/R2 engine={engine}")


def _windows(H, W, n_rand, rng, size=64):
    wins = [(0, size, 0, size), (0, size, W - size, W), (H - size, H, 0, size), (H - size, H, W - size, W),
            (0, size, W // 2, W // 2 + size), (H // 2, H // 2 + size, 0, size)]
    for _ in range(n_rand):
        y, x = rng.integers(0, H - size), rng.integers(0, W - size)
        wins.append((y, y + size, x, x + size))
    return wins


def _seam_windows(H, W, rng, n_seam=2, n_int=1, size=48, oh=128, ow=58):
    """Windows centred on tile seams of the tensor engine's launch geometry (output
    tiles of ow columns; row seams every oh rows, and the persistent kernel's row
    segments start anywhere, so row seams are drawn at random too) plus interior
    windows away from every image edge."""
    wins = []
    for _ in range(n_seam):
        ky = int(rng.integers(1, max(2, H // oh)))
        kx = int(rng.integers(1, max(2, W // ow)))
        yc = min(max(ky * oh + int(rng.integers(-6, 7)), size // 2), H - size // 2)
        xc = min(max(kx * ow + int(rng.integers(-6, 7)), size // 2), W - size // 2)
        wins.append((yc - size // 2, yc + size // 2, xc - size // 2, xc + size // 2))
    for _ in range(n_int):
        y, x = int(rng.integers(64, H - 64 - size)), int(rng.integers(64, W - 64 - size))
        wins.append((y, y + size, x, x + size))
    return wins


def test_c4_full_batch_windows(torch_cuda, P):
    """C4: all 256 images at 512^2 in one call (the bench's launch); windows of one
    image per peak plus random images are checked against the oracle: the four
    corners and an edge (image boundaries), tile-seam windows and an interior one,
    each also on |dPSNR| < 0.01 dB against its clean window."""
    p = make_problem(4)
    u = _gpu_denoise(P, torch_cuda, p.model, p.f, peak=p.peaks)
    rng = np.random.default_rng(4)
    for b in [0, 1, 2, 3, 4, 137, 255]:
        for (y0, y1, x0, x1) in _windows(512, 512, 0, rng)[:5] + _seam_windows(512, 512, rng):
            ref = oracle.denoise_window(p.f[b], p.model, y0, y1, x0, x1)
            _assert_parity(u[b, y0:y1, x0:x1], ref, float(p.peaks[b]), p.clean[b, y0:y1, x0:x1],
                           what=f"C4 b={b} win=({y0},{x0})")


def test_c4_c5_fp32_engine_windows_and_engine_agreement(torch_cuda, P):
    """The FP32 engine at C4 / C5 scale (the default engine is the tensor one): oracle
    windows, and the two engines agree to within the bar everywhere."""
    p4 = make_problem(4)
    sub = slice(0, 16)
    u_fp = _gpu_denoise(P, torch_cuda, p4.model, p4.f[sub], engine=P.ENGINE_FP32)
    u_tc = _gpu_denoise(P, torch_cuda, p4.model, p4.f[sub], engine=P.ENGINE_TENSOR)
    for b in range(16):
        assert np.max(np.abs(u_fp[b] - u_tc[b])) <= 2 * TOL * float(p4.peaks[b]), b
    rng = np.random.default_rng(44)
    for b in (0, 3):
        for (y0, y1, x0, x1) in _windows(512, 512, 1, rng)[:3]:
            ref = oracle.denoise_window(p4.f[b], p4.model, y0, y1, x0, x1)
            _assert_parity(u_fp[b, y0:y1, x0:x1], ref, float(p4.peaks[b]), what=f"C4/fp32 b={b} win=({y0},{x0})")
    p5 = make_problem(5)
    u5 = _gpu_denoise(P, torch_cuda, p5.model, p5.f, engine=P.ENGINE_FP32)[0]
    for (y0, y1, x0, x1) in [(0, 48, 0, 48), (4000, 4048, 5000, 5048), (8144, 8192, 8144, 8192)]:
        ref = oracle.denoise_window(p5.f[0], p5.model, y0, y1, x0, x1)
        _assert_parity(u5[y0:y1, x0:x1], ref, 0.1, what=f"C5/fp32 win=({y0},{x0})")


def test_c5_full_image_windows(torch_cuda, P):
    """C5 (one 8192^2 image, peak 0.1) in the bench's one-GPU launch: corner, edge,
    random, tile-seam and 8-way slab-seam windows against the oracle, each with
    |dPSNR| < 0.01 dB against its clean window."""
    p = make_problem(5)
    u = _gpu_denoise(P, torch_cuda, p.model, p.f)[0]
    rng = np.random.default_rng(5)
    clean = p.clean[0]
    for (y0, y1, x0, x1) in _windows(8192, 8192, 6, rng, size=48) + _seam_windows(8192, 8192, rng, 3, 0):
        ref = oracle.denoise_window(p.f[0], p.model, y0, y1, x0, x1)
        _assert_parity(u[y0:y1, x0:x1], ref, 0.1, clean[y0:y1, x0:x1], what=f"C5 win=({y0},{x0})")
    # also the seams of an 8-way slab partition (rows 1024*k)
    for k in (1, 4, 7):
        y = 1024 * k - 24
        ref = oracle.denoise_window(p.f[0], p.model, y, y + 48, 4000, 4048)
        _assert_parity(u[y:y + 48, 4000:4048], ref, 0.1, clean[y:y + 48, 4000:4048], what=f"C5 seam {k}")


# ------------------------------------------------------------------ edge cases
@pytest.mark.parametrize("k,H,W", [(3, 3, 3), (5, 5, 9), (7, 7, 7), (7, 7, 70), (7, 67, 131), (7, 130, 65),
                                   (5, 33, 257), (3, 1, 1)])
def test_ragged_and_minimum_sizes(torch_cuda, P, k, H, W):
    rng = np.random.default_rng(H * 1000 + W + k)
    model = make_model(rng, 3, k * k - 1, k, 63, 6.0)
    f = rng.poisson(rng.uniform(0, 4, (2, H, W))).astype(np.float32)
    if H < k or W < k:
        eng = P.TNRD(model)
        with pytest.raises(P.TNRDError) as ei:
            eng.denoise(torch_cuda.from_numpy(f).cuda())
        assert ei.value.status == 1
        return
    u = _gpu_denoise(P, torch_cuda, model, f)
    for b in range(2):
        _assert_parity(u[b], oracle.denoise(f[b], model), 4.0, what=f"k{k} {H}x{W} b{b}")


@pytest.mark.parametrize("k,H,W,bc", [(9, 9, 9, 0), (9, 41, 70, 0), (9, 38, 45, 1), (11, 47, 33, 0)])
def test_large_ksize_fp32_engine(torch_cuda, P, k, H, W, bc):
    """P l.458-469 (Fig.3) studies filters up to 9x9 (N_k = m^2 - 1 = 80): the FP32
    engine against the oracle, R1 and R2, at minimum and ragged sizes; and 11x11."""
    rng = np.random.default_rng(900 + k + H)
    nk = k * k - 1 if k <= 9 else 48   # 11x11: fewer filters so the operands fit shared memory
    model = make_model(rng, 2, nk, k, 63, 6.0)
    f = rng.poisson(rng.uniform(0, 4, (1, H, W))).astype(np.float32)
    eng = P.TNRD(model, boundary=bc)
    assert eng.engine_for(1, H, W) == P.ENGINE_FP32
    eng.close()
    u = _gpu_denoise(P, torch_cuda, model, f, boundary=bc)
    _assert_parity(u[0], oracle.denoise(f[0], model, boundary=bc), 4.0, what=f"k{k} {H}x{W} bc{bc}")


def test_stress_stage_phi_nonlinear(torch_cuda, P):
    """P17: narrow grid and large weights -- responses reach every RBF index."""
    rng = np.random.default_rng(17)
    p = make_problem(2)
    f = p.f[0][:160, :192]
    for k in (3, 5, 7):
        model = stress_model(rng, 1, k * k - 1, k, 63, p.f_max)
        u_ref = oracle.denoise(f, model)
        u = _gpu_denoise(P, torch_cuda, model, f[None])[0]
        _assert_parity(u, u_ref, 4.0, what=f"stress k={k}")


def test_direct_phi_mode_for_narrow_gaussians(torch_cuda, P):
    """gamma < step/1.5 selects the per-centre (direct) phi evaluation."""
    rng = np.random.default_rng(18)
    p = make_problem(2)
    f = p.f[0][:96, :96]
    model = make_model(rng, 2, 24, 5, 63, p.f_max)
    model.rbf_gamma[...] = model.rbf_step / np.float32(2.5)
    u = _gpu_denoise(P, torch_cuda, model, f[None])[0]
    _assert_parity(u, oracle.denoise(f, model), 4.0, what="direct phi")


@pytest.mark.parametrize("zero", ["filters", "weights"])
def test_zero_diffusion_fixed_point_exact(torch_cuda, P, zero):
    """P7/P8 on the GPU: from u_0 = f the output is exactly f."""
    p = make_problem(2)
    model = zero_model(3, 24, 5, 63, zero, lam=[1.0, 0.6, 1.7])
    u = _gpu_denoise(P, torch_cuda, model, p.f)[0]
    assert np.array_equal(u, p.f[0])


def test_flat_image_stays_flat(torch_cuda, P):
    p = make_problem(3)
    f = np.full((1, 100, 120), 3.0, np.float32)
    u = _gpu_denoise(P, torch_cuda, p.model, f)[0]
    assert np.max(np.abs(u - 3.0)) < 1e-4


def test_all_zero_counts(torch_cuda, P):
    p = make_problem(3)
    f = np.zeros((1, 64, 64), np.float32)
    u = _gpu_denoise(P, torch_cuda, p.model, f)[0]
    _assert_parity(u, oracle.denoise(f[0], p.model), 0.1, what="f=0")


def test_flip_equivariance_on_gpu(torch_cuda, P):
    """P11 on the GPU (within tolerance): catches side-asymmetric border handling."""
    from synth import Model
    p = make_problem(3)
    f = p.f[0][:90, :77]
    m = p.model
    rot = Model(np.ascontiguousarray(m.filters[:, :, ::-1, ::-1]), m.rbf_w, m.rbf_mu0, m.rbf_step,
                m.rbf_gamma, m.lam)
    a = _gpu_denoise(P, torch_cuda, m, f[None])[0]
    b = _gpu_denoise(P, torch_cuda, rot, np.ascontiguousarray(np.rot90(f, 2))[None])[0]
    assert np.max(np.abs(np.rot90(b, 2) - a)) <= TOL * 1.0


# ------------------------------------------------------------------ determinism / partition independence
def test_bitwise_determinism_batch_and_tile_independence(torch_cuda, P):
    """P13/P14: runs are bitwise repeatable; an image's output does not depend on its
    batch position or on the tile configuration (a lone image uses the small tile,
    the 32-image batch the large one)."""
    torch = torch_cuda
    p = make_problem(4)
    eng = P.TNRD(p.model)
    fb = torch.from_numpy(p.f[:32]).cuda()
    u1 = eng.denoise(fb)
    u2 = eng.denoise(fb)
    alone = eng.denoise(fb[7:8].contiguous())
    torch.cuda.synchronize()
    assert torch.equal(u1, u2)
    assert torch.equal(u1[7], alone[0])
    eng.close()


@pytest.mark.parametrize("boundary", [0, 1])
@pytest.mark.parametrize("engine", ["auto", "fp32"])
@pytest.mark.parametrize("nslabs", [2, 3, 8])
def test_loopback_slabs_bitwise_equal_full(torch_cuda, P, nslabs, engine, boundary):
    """The row-slab path (halo exchange emulated by device copies) reproduces the
    single-image result bitwise (P15), on the default (tensor) and the FP32 engine,
    R1 and R2 (the slab seams are interior rows, the global edges mirror)."""
    torch = torch_cuda
    p = make_problem(3)
    eng = P.TNRD(p.model, boundary=boundary, engine=P.ENGINE_FP32 if engine == "fp32" else P.ENGINE_AUTO)
    f = torch.from_numpy(p.f[0]).cuda()
    full = eng.denoise(f)
    u = torch.empty_like(f)
    P.tnrd_denoise_slabs_loopback(eng.h, f, u, nslabs)
    torch.cuda.synchronize()
    assert torch.equal(full, u)
    eng.close()


@pytest.mark.parametrize("nslabs", [2, 3, 8])
def test_nccl_self_exchange_slabs_bitwise_equal_full(torch_cuda, P, nslabs):
    """The slab halos moved by real NCCL point-to-point (ncclSend / ncclRecv to the
    own rank of a 1-rank communicator, grouped per stage): bitwise equal to the
    single-image result, like the copy loopback (P15)."""
    torch = torch_cuda
    p = make_problem(3)
    eng = P.TNRD(p.model)
    P.tnrd_comm_init(eng.h, P.tnrd_nccl_unique_id(), 0, 1)
    f = torch.from_numpy(p.f[0]).cuda()
    full = eng.denoise(f)
    u = torch.empty_like(f)
    P.tnrd_denoise_slabs_nccl_self(eng.h, f, u, nslabs)
    P.tnrd_comm_wait(eng.h, timeout_ms=60000)   # drains the stream, polls the async error
    assert torch.equal(full, u)
    eng.close()


def test_c5_eight_slabs_full_size_every_seam(torch_cuda, P):
    """C5 at full size (8192^2, peak 0.1) as the 8-way slab partition (halos by NCCL
    to self, the multi-GPU bench's row split): bitwise equal to the one-call result,
    and oracle windows (with dPSNR) straddling each of the 7 seams."""
    torch = torch_cuda
    p = make_problem(5)
    eng = P.TNRD(p.model)
    P.tnrd_comm_init(eng.h, P.tnrd_nccl_unique_id(), 0, 1)
    f = torch.from_numpy(p.f[0]).cuda()
    full = eng.denoise(f)
    u = torch.empty_like(f)
    P.tnrd_denoise_slabs_nccl_self(eng.h, f, u, 8)
    torch.cuda.synchronize()
    assert torch.equal(full, u)
    un = u.cpu().numpy()
    eng.close()
    rng = np.random.default_rng(55)
    for k in range(1, 8):
        y = 1024 * k - 24
        x = int(rng.integers(0, 8192 - 48))
        ref = oracle.denoise_window(p.f[0], p.model, y, y + 48, x, x + 48)
        _assert_parity(un[y:y + 48, x:x + 48], ref, 0.1, p.clean[0, y:y + 48, x:x + 48], what=f"C5 8-slab seam {k}")


def test_host_entry_point_matches_device_path(torch_cuda, P):
    p = make_problem(2)
    eng = P.TNRD(p.model)
    u_host = eng.denoise_host(p.f.copy())
    u_dev = eng.denoise(torch_cuda.from_numpy(p.f).cuda()).cpu().numpy()
    assert np.array_equal(u_host, u_dev)
    eng.close()


@pytest.mark.parametrize("engine", ["tensor", "fp32"])
def test_strided_rows(torch_cuda, P, engine):
    torch = torch_cuda
    p = make_problem(2)
    eng = P.TNRD(p.model, engine=P.ENGINE_TENSOR if engine == "tensor" else P.ENGINE_FP32)
    big = torch.zeros((1, 256, 300), device="cuda")
    big[:, :, :256] = torch.from_numpy(p.f).cuda()
    ub = torch.full_like(big, -7.0)
    P.tnrd_denoise(eng.h, big[:, :, :256], ub[:, :, :256])
    dense = eng.denoise(torch.from_numpy(p.f).cuda())
    torch.cuda.synchronize()
    assert torch.equal(ub[:, :, :256], dense)
    assert torch.all(ub[:, :, 256:] == -7.0)  # padding untouched
    eng.close()


@pytest.mark.parametrize("shape", [(1, 7, 300), (3, 200, 7), (2, 129, 59), (1, 58, 58), (1, 59, 117)])
def test_tensor_engine_tile_edges(torch_cuda, P, shape):
    """Tensor engine on shapes around its 58-column / 2-row-block tiling (one column,
    one row, exact and ragged tile multiples) against the oracle, both boundaries."""
    B, H, W = shape
    rng = np.random.default_rng(H * 7 + W)
    f = rng.poisson(rng.uniform(0, 4, shape)).astype(np.float32)
    model = make_model(rng, 2, 48, 7, 63, float(max(f.max(), 1.0)))
    for bc in (0, 1):
        u = _gpu_denoise(P, torch_cuda, model, f, boundary=bc, engine=P.ENGINE_TENSOR)
        for b in range(B):
            _assert_parity(u[b], oracle.denoise(f[b], model, boundary=bc), 4.0, what=f"tc edges {shape} bc{bc} b{b}")


# ------------------------------------------------------------------ phi / prox micro-parity
def test_phi_micro_parity(torch_cuda, P):
    """The device phi against the oracle's direct double sum over x = (v-mu0)/step in
    [-15, 77].  fp32 error model: each 8-centre unit is G * P(R) with
    P of degree 7 in R = 2^(2 sg t), so a term carries ~7x the relative error of R
    (ex2.approx plus the rounding of its exponent) plus the rounding of t^2 in G:
    about 5e-6 of the term for the highest power.  Bound: 8e-6 * max|w| in the
    centre band (|x - 31| <= 8, where the workloads' responses lie), growing with
    the distance from the grid centre (the rounded unit constants)."""
    torch = torch_cuda
    p = make_problem(3)
    eng = P.TNRD(p.model)
    for (t, i) in [(0, 0), (3, 17), (7, 47)]:
        mu0, step = float(p.model.rbf_mu0[t, i]), float(p.model.rbf_step[t, i])
        xs = np.linspace(-15, 77, 20000)
        v = (mu0 + step * xs).astype(np.float32)
        vt = torch.from_numpy(v).cuda()
        out = torch.empty_like(vt)
        P.tnrd_debug_phi(eng.h, t, i, vt, out)
        ref = oracle.phi(p.model.rbf_w[t, i], mu0, step, float(p.model.rbf_gamma[t, i]), v.astype(np.float64))
        err = np.abs(out.cpu().numpy() - ref)
        scale = float(np.abs(p.model.rbf_w[t, i]).max())
        centre = np.abs(xs - 31) <= 8
        MARGINS[f"phi t{t} i{i} centre"] = float(err[centre].max() / scale)
        MARGINS[f"phi t{t} i{i} all"] = float(err.max() / scale)
        assert err[centre].max() < 8e-6 * scale, (t, i, err[centre].max())
        assert np.all(err < 8e-6 * scale * (1 + np.abs(xs - 31) / 16)), (t, i, err.max())
    eng.close()


def test_prox_micro_parity(torch_cuda, P):
    torch = torch_cuda
    rng = np.random.default_rng(9)
    ut = rng.uniform(-6, 12, 100000).astype(np.float32)
    f = rng.integers(0, 20, 100000).astype(np.float32)
    for lam in (0.5, 1.0, 1.93):
        out = torch.empty(ut.shape, device="cuda")
        P.tnrd_debug_prox(torch.from_numpy(ut).cuda(), torch.from_numpy(f).cuda(), lam, out)
        ref = oracle.prox(ut.astype(np.float64), np.float32(lam), f)
        got = out.cpu().numpy()
        assert np.all(got >= 0) and np.all(got[f > 0] > 0)
        assert np.max(np.abs(got - ref) / np.maximum(1.0, np.abs(ref))) < 4e-7
        assert np.array_equal(got[f == 0], np.maximum(ut[f == 0] - np.float32(lam), 0))


def test_invalid_arguments_on_device(torch_cuda, P):
    torch = torch_cuda
    p = make_problem(1)
    eng = P.TNRD(p.model)
    f = torch.from_numpy(p.f).cuda()
    with pytest.raises(P.TNRDError) as ei:
        P.tnrd_denoise(eng.h, f, f)  # aliasing
    assert ei.value.status == 1
    with pytest.raises(P.TNRDError):
        eng.denoise(f, peak=[-1.0])
    h = P.tnrd_create(2, 8, 3, 63)
    with pytest.raises(P.TNRDError) as ei:
        P.tnrd_denoise(h, f, torch.empty_like(f))  # stages unset
    assert ei.value.status == 2
    with pytest.raises(P.TNRDError):
        P.tnrd_set_stage_params(h, 0, p.model.filters[0], p.model.rbf_w[0], p.model.rbf_mu0[0],
                                p.model.rbf_step[0], p.model.rbf_gamma[0], -1.0)
    P.tnrd_destroy(h)
    eng.close()


# ------------------------------------------------------------------ tabulated phi (TNRD_PHI_TABLE)
# The optional variant of BASELINE.json north_star item 2, held to the same
# tolerance as the exact path.
@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_table_phi_full_config_parity(torch_cuda, P, cfg):
    p = make_problem(cfg)
    u_ref = oracle.denoise(p.f[0], p.model)
    u = _gpu_denoise(P, torch_cuda, p.model, p.f, peak=p.peaks, phi_mode=P.PHI_TABLE)[0]
    _assert_parity(u, u_ref, float(p.peaks[0]), p.clean[0], f"table C{cfg}")


def test_table_phi_c4_windows(torch_cuda, P):
    p = make_problem(4)
    u = _gpu_denoise(P, torch_cuda, p.model, p.f, peak=p.peaks, phi_mode=P.PHI_TABLE)
    rng = np.random.default_rng(44)
    for b in [0, 1, 2, 3, 4, 200]:
        for (y0, y1, x0, x1) in _windows(512, 512, 0, rng)[:3] + _seam_windows(512, 512, rng):
            ref = oracle.denoise_window(p.f[b], p.model, y0, y1, x0, x1)
            _assert_parity(u[b, y0:y1, x0:x1], ref, float(p.peaks[b]), p.clean[b, y0:y1, x0:x1],
                           what=f"table C4 b={b} win=({y0},{x0})")


def test_table_phi_stress_and_micro(torch_cuda, P):
    """phi-stress stage (narrow grid, large weights) and the table against the
    oracle's direct sum over the whole grid, including out-of-range values."""
    torch = torch_cuda
    rng = np.random.default_rng(17)
    f = rng.poisson(3.0, size=(96, 96)).astype(np.float32)
    m = stress_model(rng, 1, 24, 5, 63, float(f.max()))
    u = _gpu_denoise(P, torch, m, f[None], phi_mode=P.PHI_TABLE)[0]
    _assert_parity(u, oracle.denoise(f, m), 4.0, what="table stress k=5")
    p = make_problem(3)
    eng = P.TNRD(p.model, phi_mode=P.PHI_TABLE)
    for (t, i) in [(0, 0), (5, 31)]:
        mu0, step = float(p.model.rbf_mu0[t, i]), float(p.model.rbf_step[t, i])
        xs = np.linspace(-20, 82, 30001)
        v = (mu0 + step * xs).astype(np.float32)
        out = torch.empty(v.shape, device="cuda")
        P.tnrd_debug_phi(eng.h, t, i, torch.from_numpy(v).cuda(), out)
        ref = oracle.phi(p.model.rbf_w[t, i], mu0, step, float(p.model.rbf_gamma[t, i]), v.astype(np.float64))
        got = out.cpu().numpy()
        err = np.abs(got - ref)
        scale = float(np.abs(p.model.rbf_w[t, i]).max())
        MARGINS[f"table phi t{t} i{i}"] = float(err.max() / scale)
        # cubic Hermite error h^4/384 * max|phi^(4)| with h = 1/16 centre is ~1e-8 of
        # scale; the fp32 cubic and fraction add a few ulp of phi
        assert err.max() < 1e-6 * scale, (t, i, err.max())
        assert np.all(got[np.abs(xs - 31) > 45.5] == 0.0)  # outside the table: exactly 0
    eng.close()


# ------------------------------------------------------------------ reaction variants
@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_gaussian_reaction_parity(torch_cuda, P, cfg):
    """P Eq.3 with psi = lambda (u_t - f) (Gaussian denoising, A = I, P l.150-158)."""
    p = make_problem(cfg)
    u_ref = oracle.denoise(p.f[0], p.model, reaction=oracle.REACTION_GAUSSIAN)
    u = _gpu_denoise(P, torch_cuda, p.model, p.f, reaction=P.REACTION_GAUSSIAN)[0]
    _assert_parity(u, u_ref, float(p.peaks[0]), what=f"gaussian C{cfg}")


@pytest.mark.parametrize("cfg", [1, 2])
def test_poisson_gradient_reaction_parity(torch_cuda, P, cfg):
    """The direct Poisson gradient step (P l.247-252), on counts shifted to be
    positive so that the step stays defined."""
    p = make_problem(cfg)
    f = p.f + 1.0
    u_ref = oracle.denoise(f[0], p.model, reaction=oracle.REACTION_POISSON_GRADIENT)
    assert np.all(np.isfinite(u_ref))
    u = _gpu_denoise(P, torch_cuda, p.model, f, reaction=P.REACTION_POISSON_GRADIENT)[0]
    _assert_parity(u, u_ref, float(p.peaks[0]) + 1.0, what=f"poisson-gradient C{cfg}")


def test_host_entry_point_pipelined_chunks_bitwise(torch_cuda, P):
    """tnrd_denoise_host pipelines large batches in chunks (copies on their own
    streams); 40 images of 512^2 give 2 chunks.  Results equal the device path bitwise."""
    torch = torch_cuda
    p = make_problem(4, batch=40)
    eng = P.TNRD(p.model)
    u_dev = eng.denoise(torch.from_numpy(p.f).cuda()).cpu().numpy()
    f_pin = torch.from_numpy(p.f).pin_memory()
    u_pin = torch.empty_like(f_pin).pin_memory()
    P.tnrd_denoise_host_ptr(eng.h, f_pin.data_ptr(), u_pin.data_ptr(), 40, 512, 512)
    eng.close()
    assert np.array_equal(u_pin.numpy(), u_dev)


    eng = P.TNRD(p.model)
    f = torch.from_numpy(p.f[0]).cuda()
    full = eng.denoise(f)
    us = torch.empty_like(f)
    P.tnrd_denoise_slabs_loopback(eng.h, f, us, 3)
    torch.cuda.synchronize()
    assert torch.equal(full, us)
    eng.close()


# ------------------------------------------------------------------ CUDA-graph replay
def test_graph_replay_bitwise_equal_to_eager_and_invalidated(torch_cuda, P):
    """tnrd_denoise replays a captured graph of its T launches: repeated calls (and the
    profiled variant with event nodes) equal eager launches (TNRD_GRAPH=0) bitwise, and
    new stage parameters (here a new lambda_0) take effect on the next call."""
    torch = torch_cuda
    p = make_problem(2)
    f = torch.from_numpy(np.ascontiguousarray(p.f)).cuda()
    os.environ["TNRD_GRAPH"] = "0"
    try:
        eager = P.TNRD(p.model)
        u_eager = eager.denoise(f)
        torch.cuda.synchronize()
    finally:
        del os.environ["TNRD_GRAPH"]
    eng = P.TNRD(p.model)
    outs = [eng.denoise(f).clone() for _ in range(3)]
    P.tnrd_set_profiling(eng.h, True)
    outs.append(eng.denoise(f).clone())
    outs.append(eng.denoise(f).clone())
    torch.cuda.synchronize()
    times = P.tnrd_get_launch_times(eng.h)
    P.tnrd_set_profiling(eng.h, False)
    assert len(times) == 2 * p.model.filters.shape[0] and all(t > 0 for t in times)
    for o in outs:
        assert torch.equal(o, u_eager)
    assert eng.launches == 5 * p.model.filters.shape[0]
    # new lambda_0: the cached graph must not replay the old launch arguments
    m = p.model
    P.tnrd_set_stage_params(eng.h, 0, m.filters[0], m.rbf_w[0], m.rbf_mu0[0], m.rbf_step[0], m.rbf_gamma[0],
                            2.0 * float(m.lam[0]))
    P.tnrd_set_stage_params(eager.h, 0, m.filters[0], m.rbf_w[0], m.rbf_mu0[0], m.rbf_step[0], m.rbf_gamma[0],
                            2.0 * float(m.lam[0]))
    u2 = eng.denoise(f)
    u2_eager = eager.denoise(f)
    torch.cuda.synchronize()
    assert not torch.equal(u2, u_eager)
    assert torch.equal(u2, u2_eager)
    eng.close()
    eager.close()


def test_unaligned_rows_take_the_per_element_u_path_bitwise(torch_cuda, P):
    """Rows whose pitch is not a multiple of 16 bytes cannot be TMA boxes: the
    persistent kernel then loads u tiles element by element (reflect + clamp), the
    operation the TMA box + mirror fix-up replaces.  Both give the same bits."""
    torch = torch_cuda
    p = make_problem(2)
    H, W = p.f.shape[1:]
    dense = torch.from_numpy(np.ascontiguousarray(p.f)).cuda()
    eng = P.TNRD(p.model)
    u_dense = eng.denoise(dense)
    for pitch in (W + 3, W + 5):       # 4 * pitch % 16 != 0
        buf = torch.zeros((1, H, pitch), device="cuda")
        buf[:, :, :W] = dense
        f_view = buf[:, :, :W]
        u_buf = torch.full((1, H, pitch), float("nan"), device="cuda")
        u_view = u_buf[:, :, :W]
        eng.denoise(f_view, u_view)
        torch.cuda.synchronize()
        assert torch.equal(u_view, u_dense), pitch
    eng.close()
