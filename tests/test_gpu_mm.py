"""Matrix Market -> device path on one GPU: a general
(locally shuffled, non-stencil-ordered) SPD operator goes file -> host parse
-> SELL upload and must give bitwise reference-mode solves and SpMVs against
the oracle, through both the Python mirror and the C++ drop-in reader."""
import numpy as np
import pytest

from tools.mgpu_check import shuffled

pytestmark = pytest.mark.gpu


def test_mm_file_to_device_solve_bitwise(cs, port, tmp_path):
    o = shuffled(port.poisson27(18, 16, 14), seed=3)
    path = str(tmp_path / "a.mtx")
    cs.write_matrix_market(path, cs.CsrMatrix(o.n, o.rowptr, o.col, o.val))
    p = cs.DeviceProblem.read_matrix_market(path, True).set_precond("jacobi")
    loc = p.to_csr()
    assert loc.col_indices.tobytes() == o.col.tobytes() and loc.values.tobytes() == o.val.tobytes()
    x = np.random.default_rng(1).standard_normal(o.n)
    assert p.spmv(x).tobytes() == port.spmv(o, x).tobytes()
    lam = port.estimate_interval(o, 1)
    x_o, r_o = port.pcg_s_solve(o, s=4, nu=30, tol=1e-8, spectrum=lam, max_outer=500)
    res = p.pcg_s_solve(cfg=cs.SolverConfig(s=4, tol=1e-8, max_outer=500, mode="reference",
                                            spectrum=cs.SpectrumEstimate(*lam)))
    assert res.report.outer_iters == r_o.outer_iters
    assert res.x.tobytes() == x_o.tobytes()
    # the C++/Python host reader feeds the same bytes as the direct device reader
    a = cs.read_matrix_market(path, True)
    res2 = cs.pcg_s_solve(a, np.ones(a.n), np.zeros(a.n), cs.JacobiPreconditioner(a),
                          cs.SolverConfig(s=4, tol=1e-8, max_outer=500, mode="reference",
                                          spectrum=cs.SpectrumEstimate(*lam)))
    assert res2.x.tobytes() == x_o.tobytes()
