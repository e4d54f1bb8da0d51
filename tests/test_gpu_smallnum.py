"""GPU smallnum API (smallnum.py:54-142) against numpy and the reference's unit tests
(tests/test_smallnum.py): SVD reconstruction/order, solves with the conditioning
flag, monic roots, pencil round trips including rank overshoot."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_svd(rng):
    from paper_2011_05749_b200.smallnum import svd

    assert np.allclose(svd([[0.0, 1.0], [1.0, 0.0]]).sigma, [1.0, 1.0])
    assert np.allclose(svd(np.zeros((3, 3))).sigma, 0.0)
    assert np.allclose(svd(np.diag([3.0, 2.0, 1.0])).sigma, [3.0, 2.0, 1.0])
    for rows, cols in ((4, 4), (6, 3), (3, 6), (16, 8), (2, 7)):
        a = rng.normal(size=(rows, cols)) + 1j * rng.normal(size=(rows, cols))
        r = svd(a)
        assert np.all(np.diff(r.sigma) <= 1e-12)
        assert np.allclose(r.sigma, np.linalg.svd(a, compute_uv=False), atol=1e-12)
        sig = np.zeros(a.shape, dtype=complex)
        k = min(a.shape)
        sig[:k, :k] = np.diag(r.sigma)
        assert np.linalg.norm(r.u @ sig @ r.v.conj().T - a) <= 1e-10 * np.linalg.norm(a)
        assert np.allclose(r.u.conj().T @ r.u, np.eye(rows), atol=1e-10)
        assert np.allclose(r.v.conj().T @ r.v, np.eye(cols), atol=1e-10)
    with pytest.raises(ValueError):
        svd(np.zeros((65, 2)))


def test_solves(rng):
    from paper_2011_05749_b200.smallnum import least_squares, solve_linear

    out = solve_linear(np.eye(3), [1.0, 2.0, 3.0])
    assert np.allclose(out.x, [1, 2, 3]) and out.well_conditioned
    out = solve_linear([[1.0, 1.0], [1.0, 1.0]], [2.0, 2.0])
    assert np.allclose(out.x, [1.0, 1.0]) and not out.well_conditioned  # least-norm
    for m, n in ((4, 4), (15, 8), (12, 3)):
        a = rng.normal(size=(m, n)) + 1j * rng.normal(size=(m, n))
        b = rng.normal(size=m) + 1j * rng.normal(size=m)
        got = least_squares(a, b) if m > n else solve_linear(a, b)
        ref, *_ = np.linalg.lstsq(a, b, rcond=None)
        assert np.allclose(got.x, ref, atol=1e-10)
        assert abs(got.residual - np.linalg.norm(a @ ref - b)) < 1e-9
    with pytest.raises(ValueError):
        least_squares(np.zeros((2, 3)), [0.0, 0.0])


def test_roots_and_pencil(rng):
    from paper_2011_05749_b200.smallnum import pencil_eigenvalues, poly_roots

    for a in (1, 2, 3, 4):
        z = np.exp(2j * np.pi * rng.random(a))
        coeffs = np.poly(z)[::-1][:-1]
        got = poly_roots(coeffs)
        assert max(min(abs(g - t) for t in z) for g in got) < 1e-8
    with pytest.raises(ValueError):
        poly_roots(np.ones(5))
    n = 64
    for tones in (1, 2, 3, 4):
        freqs = rng.choice(n, size=tones, replace=False)
        vals = np.exp(2j * np.pi * rng.random(tones))
        z = np.exp(-2j * np.pi * freqs / n)
        m = {t: np.sum(vals * z**t) for t in range(-tones, tones + 1)}
        full = np.array([[m[r - c] for c in range(tones + 1)] for r in range(tones + 1)])
        res = pencil_eigenvalues(full[:, :-1], full[:, 1:], tones)
        assert res.ok
        assert max(min(abs(v - t) for t in z) for v in res.values) < 1e-7
    # asking for more than the numerical rank flags ok=False and truncates
    z = np.exp(-2j * np.pi * 5 / n)
    m = {t: z**t for t in range(-3, 4)}
    full = np.array([[m[r - c] for c in range(4)] for r in range(4)])
    res = pencil_eigenvalues(full[:, :-1], full[:, 1:], 3)
    assert not res.ok and res.values.size == 1 and abs(res.values[0] - z) < 1e-8
