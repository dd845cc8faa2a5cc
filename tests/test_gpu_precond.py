"""Pluggable device preconditioners against the reference.

The reference solver accepts any ``const Preconditioner&`` (precond.hpp:12-23,
solver.cpp:78-80). Two device kinds beyond identity/Jacobi plug into the same
solve path:

* block Jacobi -- parity partner: a block-Jacobi SUBCLASS of the reference's own
  Preconditioner compiled into oracle/_ref (ref_capi.cpp BlockJacobiRef), run by
  the unmodified reference pcg_s_solve / estimate_interval / pcg_solve;
* a device plugin (DevicePreconditioner: the caller enqueues out = M^-1 in on the
  solve stream) -- here a torch kernel computing the Jacobi scaling, which must
  reproduce the built-in Jacobi solve bit for bit.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL_X = 1e-8


def _csr(cs, o):
    return cs.CsrMatrix(o.n, o.rowptr, o.col, o.val)


@pytest.mark.parametrize("bs,stencil,n,s", [(4, 27, 16, 4), (2, 7, 20, 4), (8, 27, 14, 8),
                                            (3, 27, 13, 4)])
def test_block_jacobi_reference_mode_bitwise(cs, port, ref, bs, stencil, n, s):
    o = port.poisson27(n) if stencil == 27 else port.stencil7(n)
    a = _csr(cs, o)
    m = cs.BlockJacobiPreconditioner(a, bs)
    lam = ref.estimate_interval(o, 100 + bs)
    x_r, r_r = ref.pcg_s_solve(o, s=s, tol=1e-8, spectrum=lam, precond=100 + bs, max_outer=2000)
    cfg = cs.SolverConfig(s=s, tol=1e-8, max_outer=2000, mode="reference",
                          spectrum=cs.SpectrumEstimate(*lam))
    res = cs.pcg_s_solve(a, np.ones(o.n), np.zeros(o.n), m, cfg)
    assert res.report.outer_iters == r_r.outer_iters
    assert res.x.tobytes() == x_r.tobytes()
    assert res.report.rel_residual.tobytes() == r_r.rel_residual.tobytes()
    assert res.report.delta_alpha.tobytes() == r_r.delta_alpha.tobytes()
    # device Lanczos with the block-Jacobi M inner product
    p = cs.DeviceProblem.from_csr(a).set_precond(m)
    est = p.estimate_interval(40, 1234, "reference")
    assert abs(est.lambda_min / lam[0] - 1) < 1e-10 and abs(est.lambda_max / lam[1] - 1) < 1e-10
    # fast algebra: same count +-1, x within 1e-8
    fast = p.pcg_s_solve(cfg=cs.SolverConfig(s=s, tol=1e-8, max_outer=2000))
    assert abs(fast.report.outer_iters - r_r.outer_iters) <= 1
    assert np.linalg.norm(fast.x - x_r) / np.linalg.norm(x_r) <= TOL_X
    # classical PCG with the same preconditioner: reference order bitwise
    x_c, r_c = ref.pcg_solve(o, tol=1e-8, max_iter=2000, precond=100 + bs)
    pc = p.pcg_solve(tol=1e-8, max_iter=2000, mode="reference")
    assert pc.report.outer_iters == r_c.outer_iters
    assert pc.x.tobytes() == x_c.tobytes()
    pcf = p.pcg_solve(tol=1e-8, max_iter=2000)
    assert abs(pcf.report.outer_iters - r_c.outer_iters) <= 1
    p.close()


def test_block_jacobi_mpk_and_errors(cs, port, ref):
    o = port.poisson27(10)
    a = _csr(cs, o)
    m = cs.BlockJacobiPreconditioner(a, 4)
    r = np.random.default_rng(3).standard_normal(o.n)
    z_r, p_r = ref.mpk(o, r, 5, 0.05, 1.6, precond=104)
    res = cs.mpk_chebyshev(a, r, 5, m, cs.ChebyshevParams.from_interval(0.05, 1.6))
    assert np.asfortranarray(res.z).T.tobytes() == z_r.tobytes()
    assert np.asfortranarray(res.p).T.tobytes() == p_r.tobytes()
    # a non-SPD diagonal block is refused like the reference ctor (NotSpdError)
    bad = cs.CsrMatrix(o.n, o.rowptr, o.col, np.where(o.col == np.repeat(
        np.arange(o.n), np.diff(o.rowptr)), -1.0, o.val))
    with pytest.raises(cs.NotSpdError):
        cs.DeviceProblem.from_csr(bad).set_precond(cs.BlockJacobiPreconditioner(bad, 4))
    with pytest.raises(cs.InvalidArgumentError):
        cs.BlockJacobiPreconditioner(a, 17)


class _Ptr:
    """__cuda_array_interface__ view of a raw device pointer (torch.as_tensor)."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None}


def test_device_plugin_matches_builtin_jacobi(cs, port):
    """A DevicePreconditioner doing out = (1/a_ii) * in with a torch kernel on the
    solve stream is the Jacobi preconditioner: every solve path (Lanczos, MPK,
    the fast update pass, classical PCG) gives the built-in Jacobi's bits."""
    import torch
    o = port.poisson27(18, 16, 14)
    a = _csr(cs, o)
    d = torch.tensor(cs.DeviceProblem.from_csr(a).set_precond("jacobi").inv_diag(), device="cuda")
    calls = []

    class TorchJacobi(cs.DevicePreconditioner):
        def device_apply(self, in_ptr, out_ptr, n, stream):
            calls.append(n)
            with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
                x = torch.as_tensor(_Ptr(in_ptr, n), device="cuda")
                y = torch.as_tensor(_Ptr(out_ptr, n), device="cuda")
                torch.mul(d, x, out=y)

    for mode in ("reference", "fast"):
        pj = cs.DeviceProblem.from_csr(a).set_precond("jacobi")
        pp = cs.DeviceProblem.from_csr(a).set_precond(TorchJacobi())
        cfg = cs.SolverConfig(s=4, tol=1e-8, max_outer=500, mode=mode)
        rj, rp = pj.pcg_s_solve(cfg=cfg), pp.pcg_s_solve(cfg=cfg)
        lp, lj = rp.report.spectrum_used.lambda_min, rj.report.spectrum_used.lambda_min
        if mode == "reference":
            assert lp == lj
        else:  # built-in Jacobi takes the G-only Lanczos, a general M the (v, g) one
            assert abs(lp / lj - 1) < 1e-9
        if mode == "reference":
            assert rp.report.outer_iters == rj.report.outer_iters
            assert rp.x.tobytes() == rj.x.tobytes()
        else:  # general M takes the reference MPK epilogue, built-in Jacobi the fused one
            assert abs(rp.report.outer_iters - rj.report.outer_iters) <= 1
            assert np.linalg.norm(rp.x - rj.x) / np.linalg.norm(rj.x) < 1e-8
        cj, cp = pj.pcg_solve(tol=1e-8, max_iter=500, mode=mode), pp.pcg_solve(
            tol=1e-8, max_iter=500, mode=mode)
        assert cp.report.outer_iters == cj.report.outer_iters
        if mode == "reference":
            assert cp.x.tobytes() == cj.x.tobytes()
        pj.close()
        pp.close()
    assert calls and all(c == o.n for c in calls)

    class Failing(cs.DevicePreconditioner):
        def device_apply(self, in_ptr, out_ptr, n, stream):
            raise RuntimeError("boom")

    with pytest.raises(cs.Error):
        cs.DeviceProblem.from_csr(a).set_precond(Failing()).pcg_s_solve(
            cfg=cs.SolverConfig(s=4, tol=1e-8))
