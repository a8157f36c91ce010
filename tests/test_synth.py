"""Host-side checks of the seeded generator."""
import numpy as np

from synth import CONFIGS, dct_atoms, make_problem


def test_dct_atoms_orthonormal():
    for m in (3, 5, 7):
        A = dct_atoms(m).reshape(m * m, -1)
        assert np.allclose(A @ A.T, np.eye(m * m), atol=1e-12)
        assert np.allclose(A[1:].sum(axis=1), 0, atol=1e-12)  # non-constant atoms are zero-mean


def test_problem_recipe_c1_c2_c3():
    for c in (1, 2, 3):
        p = make_problem(c)
        cfg = CONFIGS[c]
        assert p.f.shape == (1, cfg["H"], cfg["W"]) and p.f.dtype == np.float32
        assert np.all(p.f == np.round(p.f)) and np.all(p.f >= 0)
        assert abs(p.clean.max() - cfg["peaks"][0]) < 1e-6
        m = p.model
        assert m.filters.shape == (cfg["T"], cfg["Nk"], cfg["k"], cfg["k"])
        assert np.max(np.abs(m.filters.sum(axis=(2, 3)))) < 1e-6         # zero mean
        assert np.allclose((m.filters.astype(float) ** 2).sum(axis=(2, 3)), 1, atol=1e-6)
        assert np.all(m.rbf_step > 0) and np.all(m.rbf_gamma == m.rbf_step)
        assert np.allclose(m.rbf_mu0 + (cfg["M"] - 1) * m.rbf_step, -m.rbf_mu0, rtol=1e-5)
        assert np.all(m.lam > 0)
        if c == 1:
            assert np.all(m.lam == 1.0)
        else:
            assert np.all((m.lam >= 0.5) & (m.lam <= 2.0))
        assert p.f_max == max(1.0, float(p.f.max()))


def test_generator_is_deterministic():
    from synth.generator import _problem_cached
    a = make_problem(2)
    _problem_cached.cache_clear()
    b = make_problem(2)
    assert np.array_equal(a.f, b.f) and np.array_equal(a.model.rbf_w, b.model.rbf_w)


def test_c4_peaks_cycle():
    p = make_problem(4)
    assert p.f.shape == (256, 512, 512)
    assert list(p.peaks[:6]) == [np.float32(x) for x in (0.1, 0.2, 1.0, 2.0, 4.0, 0.1)]
    for b in range(5):
        assert abs(p.clean[b].max() - p.peaks[b]) < 1e-6
