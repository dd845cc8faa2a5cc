"""Host small-dense analysis used by the gram-analysis path:
fgs_rate (gram.cpp:148-174) and kappa_2(W) (solver.cpp:69-74) against the
reference library's LAPACK-backed versions (dgesvd / dgeev / dsyevd). The
product uses its own Jacobi / Hessenberg-QR solvers, so agreement is to
rounding (1e-10 relative), not bitwise. CPU only."""
import ctypes as C

import numpy as np
import pytest

import paper_2603_09790_b200 as cs


def _ref_rate(ref, w):
    f = ref.lib.ref_fgs_rate_normalized
    f.argtypes = [C.c_int, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    a, b = C.c_double(), C.c_double()
    wf = np.asfortranarray(w)
    ref._check(f(w.shape[0], wf.ctypes.data, C.byref(a), C.byref(b)))
    return a.value, b.value


def _ref_eig(ref, w):
    f = ref.lib.ref_sym_eigvals
    f.argtypes = [C.c_int, C.c_void_p, C.c_void_p]
    out = np.zeros(w.shape[0])
    wf = np.asfortranarray(w)
    ref._check(f(w.shape[0], wf.ctypes.data, out.ctypes.data))
    return out


def _grams(rng):
    out = []
    for s in (1, 2, 3, 4, 6, 8, 12, 16, 24):
        a = rng.standard_normal((s, s))
        w = a @ a.T + s * np.eye(s)
        out.append(w)
        # Chebyshev-basis-like: strongly coupled, ill conditioned
        x = np.linspace(-1, 1, 400)
        t = np.polynomial.chebyshev.chebvander(x, s - 1)
        v = t.T @ (t * (1.0 + 0.5 * x[:, None]))
        out.append(0.5 * (v + v.T))
    return out


def test_fgs_rate_matches_reference(ref):
    rng = np.random.default_rng(2)
    for w in _grams(rng):
        w = 0.5 * (w + w.T)
        g = cs.normalize_gram(cs.gram_from_matrix(w))
        r = cs.fgs_rate(g)
        n_ref, rad_ref = _ref_rate(ref, w)
        assert r.spectral_norm == pytest.approx(n_ref, rel=1e-10, abs=1e-13)
        assert r.spectral_radius == pytest.approx(rad_ref, rel=1e-9, abs=1e-12)


def test_nonsymmetric_eigen_moduli_known():
    # rotation-scaled block + real eigenvalues: radius known exactly
    w = np.eye(3)
    w[1, 0] = w[0, 1] = 0.9
    w[2, 1] = w[1, 2] = -0.3
    g = cs.normalize_gram(cs.gram_from_matrix(w))
    r = cs.fgs_rate(g)
    l = np.tril(w, -1)
    m = l.T @ np.linalg.inv(np.eye(3) + l)
    assert r.spectral_radius == pytest.approx(max(abs(np.linalg.eigvals(m))), rel=1e-12)
    assert r.spectral_norm == pytest.approx(np.linalg.norm(m, 2), rel=1e-12)


def test_kappa_matches_reference(ref):
    rng = np.random.default_rng(4)
    for w in _grams(rng):
        w = 0.5 * (w + w.T)
        e = _ref_eig(ref, w)
        want = e[-1] / e[0] if e[0] > 0 else np.inf
        assert cs.kappa_sym(w) == pytest.approx(want, rel=1e-8)
    assert cs.kappa_sym(np.array([[1.0, 2.0], [2.0, 1.0]])) == np.inf


def test_fgs_rate_requires_normalized():
    with pytest.raises(cs.InvalidArgumentError):
        cs.fgs_rate(cs.gram_from_matrix(np.eye(2)))
    with pytest.raises(cs.InvalidMatrixError):
        cs.gram_from_matrix(np.array([[1.0, 0.5], [0.4, 1.0]]))
