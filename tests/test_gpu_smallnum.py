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


# ---- shapes beyond the per-thread templates, up to the reference's 64 x 64 cap
# (smallnum.py:15,21-29): the CTA-cooperative solvers of csrc/smallnum_cta.cu


def _numpy_pencil(y1, y2, rank):
    """The reference's pencil_eigenvalues (smallnum.py:110-142) restated in numpy."""
    full = np.hstack([y1, y2[:, -1:]])
    sv = np.linalg.svd(full, compute_uv=False)
    nrank = int(np.sum(sv > sv[0] * 1e-10))
    r = min(rank, nrank)
    _, _, vh = np.linalg.svd(full)
    rb = vh[:r, :]
    return np.conj(np.linalg.eigvals(rb[:, 1:] @ np.linalg.pinv(rb[:, :-1]))), rank <= nrank


@pytest.mark.parametrize("shape", [(64, 64), (64, 9), (9, 64), (40, 33), (33, 40), (17, 17),
                                   (64, 1), (1, 64)])
def test_svd_large_shapes(rng, shape):
    from paper_2011_05749_b200.smallnum import svd

    rows, cols = shape
    a = rng.normal(size=shape) + 1j * rng.normal(size=shape)
    r = svd(a)
    assert np.all(np.diff(r.sigma) <= 1e-12)
    ref = np.linalg.svd(a, compute_uv=False)
    assert np.allclose(r.sigma, ref, rtol=1e-12, atol=1e-12 * ref[0])
    sig = np.zeros(shape, dtype=complex)
    k = min(shape)
    sig[:k, :k] = np.diag(r.sigma)
    assert np.linalg.norm(r.u @ sig @ r.v.conj().T - a) <= 1e-12 * np.linalg.norm(a)
    assert np.allclose(r.u.conj().T @ r.u, np.eye(rows), atol=1e-12)
    assert np.allclose(r.v.conj().T @ r.v, np.eye(cols), atol=1e-12)


def test_svd_large_rank_deficient_and_zero(rng):
    from paper_2011_05749_b200.smallnum import svd

    z = svd(np.zeros((16, 16)))
    assert np.allclose(z.sigma, 0.0) and np.allclose(z.u.conj().T @ z.u, np.eye(16))
    b = rng.normal(size=(48, 5)) + 1j * rng.normal(size=(48, 5))
    a = b @ (rng.normal(size=(5, 20)) + 1j * rng.normal(size=(5, 20)))  # rank 5
    r = svd(a)
    assert np.allclose(r.sigma, np.linalg.svd(a, compute_uv=False), atol=1e-10)
    assert np.all(r.sigma[5:] < 1e-10 * r.sigma[0])
    sig = np.zeros(a.shape, dtype=complex)
    sig[:20, :20] = np.diag(r.sigma)
    assert np.linalg.norm(r.u @ sig @ r.v.conj().T - a) <= 1e-11 * np.linalg.norm(a)
    assert np.allclose(r.u.conj().T @ r.u, np.eye(48), atol=1e-10)


def test_solves_large_shapes(rng):
    from paper_2011_05749_b200.smallnum import least_squares, solve_linear

    for m, n in ((64, 64), (64, 20), (33, 9), (12, 12)):
        a = rng.normal(size=(m, n)) + 1j * rng.normal(size=(m, n))
        x0 = rng.normal(size=n) + 1j * rng.normal(size=n)
        out = (solve_linear if m == n else least_squares)(a, a @ x0)
        assert np.allclose(out.x, x0, atol=1e-9) and out.residual < 1e-9 * np.linalg.norm(a @ x0)
        assert out.well_conditioned
        bn = rng.normal(size=m) + 1j * rng.normal(size=m)
        out = least_squares(a, bn)
        want = np.linalg.lstsq(a, bn, rcond=None)[0]
        assert np.allclose(out.x, want, atol=1e-9)
        assert abs(out.residual - np.linalg.norm(a @ want - bn)) <= 1e-9 * np.linalg.norm(bn)
    # singular square system: least-norm solution, flagged (reference test_smallnum.py:61-64)
    s = np.ones((16, 16))
    out = solve_linear(s, np.full(16, 16.0))
    assert not out.well_conditioned and np.isfinite(out.x).all()
    assert np.allclose(out.x, np.linalg.lstsq(s, np.full(16, 16.0), rcond=None)[0], atol=1e-9)
    with pytest.raises(ValueError):
        solve_linear(np.eye(65), np.ones(65))


@pytest.mark.parametrize("a_", [5, 9, 16, 24])
def test_pencil_large(a_):
    from paper_2011_05749_b200.smallnum import pencil_eigenvalues

    n = 128
    rng = np.random.default_rng(a_)
    freqs = rng.choice(n, size=a_, replace=False)
    z = np.exp(-2j * np.pi * freqs / n)
    p = rng.uniform(0.5, 2.0, a_) * np.exp(2j * np.pi * rng.uniform(size=a_))
    ks = np.arange(-a_, a_ + 1)
    mom = {int(k): complex(np.sum(p * z ** k)) for k in ks}
    full = np.array([[mom[r - c] for c in range(a_ + 1)] for r in range(a_ + 1)])
    y1, y2 = full[:, :-1], full[:, 1:]
    res = pencil_eigenvalues(y1, y2, a_)
    want, ok = _numpy_pencil(y1, y2, a_)
    assert res.ok == ok and res.values.size == want.size == a_
    dist = max(max(min(abs(v - t) for t in z) for v in res.values),
               max(min(abs(v - t) for v in res.values) for t in z))
    assert dist < 1e-7, dist
    # rank overshoot on the same size: a rank-3 signal in an a_-tone pencil
    mom3 = {int(k): complex(np.sum(p[:3] * z[:3] ** k)) for k in ks}
    f3 = np.array([[mom3[r - c] for c in range(a_ + 1)] for r in range(a_ + 1)])
    r3 = pencil_eigenvalues(f3[:, :-1], f3[:, 1:], a_)
    w3, ok3 = _numpy_pencil(f3[:, :-1], f3[:, 1:], a_)
    assert not r3.ok and not ok3 and r3.values.size == w3.size == 3
    assert max(min(abs(v - t) for t in z[:3]) for v in r3.values) < 1e-7
