"""GPU parity of the kernel-level entries against the CPU oracle (bitwise where
the reference's arithmetic is order-pinned). Every call goes through the
C ABI of libchebstep_gpu.so."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _csr(cs, o):
    return cs.CsrMatrix(o.n, o.rowptr, o.col, o.val)


def _same(a, b):
    return np.asarray(a).tobytes() == np.asarray(b).tobytes()


@pytest.mark.parametrize("dims", [(1, 1, 1), (2, 1, 1), (4, 4, 4), (5, 7, 3), (16, 16, 16), (64, 64, 64)])
def test_poisson27_assembly_bitwise(cs, port, dims):
    """problems.cpp:13-53 assembled on the device == CPU assembly, bit for bit."""
    sysd = cs.poisson27(cs.PoissonSpec(*dims))
    o = port.poisson27(*dims)
    assert _same(sysd.a.row_offsets, o.rowptr)
    assert _same(sysd.a.col_indices, o.col)
    assert _same(sysd.a.values, o.val)
    assert np.all(sysd.rhs == 1.0)


def test_poisson27_spec_examples(cs):
    """SPEC.md:135-137 KATs."""
    a = cs.poisson27(cs.PoissonSpec(1, 1, 1)).a
    assert a.values.tolist() == [26.0]
    a = cs.poisson27(cs.PoissonSpec(2, 1, 1)).a
    assert a.values.tolist() == [26.0, -1.0, -1.0, 26.0]
    a = cs.poisson27(cs.PoissonSpec(4, 4, 4)).a
    assert a.nnz() == 1000
    assert a.row_offsets[1] - a.row_offsets[0] == 8
    assert a.values[a.row_offsets[0]:a.row_offsets[1]].sum() == 19.0


@pytest.mark.parametrize("dims,coef", [((8, 8, 8), (1, 1, 1)), ((9, 5, 7), (1, 1, 100)), ((32, 32, 32), (1, 1, 1))])
def test_stencil7_assembly_bitwise(cs, port, dims, coef):
    sysd = cs.stencil7(cs.PoissonSpec(*dims), coef)
    o = port.stencil7(*dims, coef=coef)
    assert _same(sysd.a.row_offsets, o.rowptr)
    assert _same(sysd.a.col_indices, o.col)
    assert _same(sysd.a.values, o.val)


def test_upload_roundtrip(cs, port):
    o = port.poisson27(6, 5, 4)
    p = cs.DeviceProblem.from_csr(_csr(cs, o))
    back = p.to_csr()
    assert _same(back.row_offsets, o.rowptr) and _same(back.col_indices, o.col)
    assert _same(back.values, o.val)


@pytest.mark.parametrize("gen", ["p27_64", "p7_32", "random"])
def test_spmv_bitwise(cs, port, gen):
    """csr.cpp:111-124: row-serial, stored order, no FMA -> identical bits."""
    rng = np.random.default_rng(1)
    if gen == "p27_64":
        o = port.poisson27(64)
    elif gen == "p7_32":
        o = port.stencil7(32)
    else:  # random sparse rows with random values, some empty rows
        n = 5000
        lens = rng.integers(0, 40, n)
        lens[::97] = 0
        rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        ci = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lens]).astype(np.int64)
        from oracle.oracle import Csr
        o = Csr(n, rp, ci, rng.standard_normal(rp[-1]))
    x = rng.standard_normal(o.n)
    y = cs.spmv(_csr(cs, o), x)
    assert _same(y, port.spmv(o, x))


@pytest.mark.parametrize("s", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("precond", [0, 1])
def test_mpk_bitwise(cs, port, s, precond):
    """mpk.cpp:26-71: fused SpMV + lincomb3 + Jacobi epilogue == reference."""
    o = port.poisson27(12, 10, 9)
    r = np.random.default_rng(s).standard_normal(o.n)
    lo, hi = (0.05, 1.6) if precond else (1.0, 40.0)
    m = cs.JacobiPreconditioner(_csr(cs, o)) if precond else cs.IdentityPreconditioner()
    res = cs.mpk_chebyshev(_csr(cs, o), r, s, m, cs.ChebyshevParams.from_interval(lo, hi))
    z, p = port.mpk(o, r, s, lo, hi, precond)
    assert _same(np.asfortranarray(res.z).T, z)
    assert _same(np.asfortranarray(res.p).T, p)


def test_mpk_spec_example(cs):
    """diag(1,3), lambda=[1,3], r=[1,1], s=3."""
    a = cs.CsrMatrix.diagonal_matrix([1.0, 3.0])
    res = cs.mpk_chebyshev(a, [1.0, 1.0], 3, cs.IdentityPreconditioner(),
                           cs.ChebyshevParams.from_interval(1.0, 3.0))
    assert res.z.T.tolist() == [[1, 1], [-1, 1], [1, 1]]
    assert res.p.T.tolist() == [[1, 1], [1, 3], [-1, 3], [1, 3]]


def test_mpk_basis_breakdown(cs):
    a = cs.CsrMatrix.diagonal_matrix([1.0, 1e308])
    with pytest.raises(cs.BasisBreakdownError) as e:
        cs.mpk_chebyshev(a, [1.0, 1e308], 3, cs.IdentityPreconditioner(),
                         cs.ChebyshevParams.from_interval(1.0, 3.0))
    assert e.value.column >= 1


def test_random_vector_bitwise(cs, port):
    assert _same(cs.random_vector(100003, 1234), port.random_vector(100003, 1234))


@pytest.mark.parametrize("ku,kv", [(4, 4), (8, 1), (12, 12), (3, 7)])
def test_block_gram(cs, port, ku, kv):
    rng = np.random.default_rng(ku * 31 + kv)
    n = 70001
    u, v = rng.standard_normal((ku, n)), rng.standard_normal((kv, n))
    g_ref = port.block_gram(u, v)
    g_dev = cs.block_gram(u.T, v.T, mode="reference")
    assert _same(g_dev, g_ref)
    g_fast = cs.block_gram(u.T, v.T, mode="fast")
    np.testing.assert_allclose(g_fast, g_ref, rtol=1e-11, atol=1e-11 * np.abs(g_ref).max())


def test_block_update_bitwise(cs, port):
    rng = np.random.default_rng(3)
    n, m, k = 10007, 6, 5
    y, x, c = rng.standard_normal((k, n)), rng.standard_normal((m, n)), rng.standard_normal((m, k))
    out = cs.block_update(y.T, x.T, c)
    assert _same(np.asfortranarray(out).T, port.block_update(y, x, c))


def test_assemble_gram_bitwise(cs, port):
    rng = np.random.default_rng(4)
    n, k = 5000, 6
    q = rng.standard_normal((k, n))
    aq = q + 0.01 * rng.standard_normal((k, n))
    g = cs.assemble_gram(q.T, aq.T)
    assert _same(g.w, port.assemble_gram(q, aq))
    with pytest.raises(cs.NotSpdError):
        cs.assemble_gram(q.T, -q.T)


def test_fgs_spec_examples(cs):
    """SPEC.md:296-299."""
    g = cs.gram_from_matrix(np.array([[1.0, 0.5], [0.5, 1.0]]))
    r = cs.fgs_solve(g, np.array([1.0, 0.0]), cs.FgsConfig(nu=1))
    assert r.x[:, 0].tolist() == [1.0, -0.5] and r.rel_residual == 0.25
    r = cs.fgs_solve(g, np.array([1.0, 0.0]), cs.FgsConfig(nu=50))
    assert r.x[:, 0].tolist() == [1.3333333333333333, -0.66666666666666663]
    r = cs.fgs_solve(g, np.zeros(2), cs.FgsConfig(nu=3))
    assert r.x.tolist() == [[0.0], [0.0]] and r.rel_residual == 0.0


@pytest.mark.parametrize("s,k,nu", [(4, 1, 30), (8, 8, 30), (12, 12, 2), (16, 3, 7), (64, 64, 3)])
def test_fgs_and_cholesky_bitwise(cs, port, s, k, nu):
    rng = np.random.default_rng(s * 100 + k)
    b = rng.standard_normal((s, s))
    w = b @ b.T + s * np.eye(s)
    w = 0.5 * (w + w.T)
    rhs = rng.standard_normal((s, k))
    r = cs.fgs_solve(cs.gram_from_matrix(w), rhs, cs.FgsConfig(nu=nu))
    x_o, d_o = port.fgs_solve(w, rhs, nu)
    assert _same(r.x, x_o) and r.rel_residual == d_o
    assert _same(cs.small_cholesky_solve(w, rhs), port.cholesky_solve(w, rhs))


def test_small_errors(cs):
    with pytest.raises(cs.NotSpdError):
        cs.small_cholesky_solve(np.array([[1.0, 2.0], [2.0, 1.0]]), np.ones(2))
    with pytest.raises(cs.InvalidMatrixError):
        cs.fgs_solve(cs.gram_from_matrix(np.array([[1.0, 0.5], [0.4, 1.0]])), np.ones(2))
    with pytest.raises(cs.NotSpdError):
        cs.fgs_solve(cs.gram_from_matrix(np.array([[0.0, 0.0], [0.0, 1.0]])), np.ones(2))


def test_tridiag_eigvals(cs, port):
    rng = np.random.default_rng(5)
    d, e = rng.uniform(0.1, 2.0, 40), rng.uniform(0.01, 0.5, 39)
    ev = cs.tridiag_eigvals(d, e)
    t = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    np.testing.assert_allclose(ev, np.linalg.eigvalsh(t), rtol=1e-13, atol=1e-14)
    np.testing.assert_allclose(ev, port.tridiag_eigvals(d, e), rtol=1e-13, atol=1e-14)


@pytest.mark.parametrize("gen,precond", [("p27_32", 1), ("p27_16", 0), ("p7_32", 1)])
def test_lanczos_interval(cs, port, gen, precond):
    """spectral.cpp:60-132: device Lanczos vs the CPU oracle's interval."""
    o = {"p27_32": lambda: port.poisson27(32), "p27_16": lambda: port.poisson27(16),
         "p7_32": lambda: port.stencil7(32)}[gen]()
    lo, hi = port.estimate_interval(o, precond)
    m = cs.JacobiPreconditioner(_csr(cs, o)) if precond else cs.IdentityPreconditioner()
    e_ref = cs.estimate_interval(_csr(cs, o), m, mode="reference")
    assert abs(e_ref.lambda_min / lo - 1) < 1e-12 and abs(e_ref.lambda_max / hi - 1) < 1e-13
    e_fast = cs.estimate_interval(_csr(cs, o), m, mode="fast")
    assert abs(e_fast.lambda_min / lo - 1) < 1e-9 and abs(e_fast.lambda_max / hi - 1) < 1e-11
