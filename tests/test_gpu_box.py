"""Plane-streaming box SpMV (spmv.cu sell_box_kernel).

27-point classes whose table is a 3x3x3 box in natural ordering are applied
plane by plane from shared memory. The kernel must give the CDIA row sums bit
for bit: the SpMV equals the CPU oracle, and fast-algebra solves (the fused
MPK epilogues) are bitwise the same with the kernel switched off
(CS_SPMV_BOX=0: gather kernels). Shapes cover several T-row columns per
plane, partial columns, planes not a multiple of 32 rows, and thin grids."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPES = [(64, 64, 40), (70, 50, 13), (40, 36, 30), (5, 4, 7), (128, 96, 9), (33, 20, 11)]


def _solve(cs, p, lam, box):
    old = os.environ.get("CS_SPMV_BOX")
    os.environ["CS_SPMV_BOX"] = "1" if box else "0"
    try:
        r = p.pcg_s_solve(cfg=cs.SolverConfig(s=8, tol=1e-8, max_outer=3000, spectrum=lam))
        y = p.spmv(np.arange(p.n_local, dtype=np.float64) % 7 - 3.0)
        return r.x.tobytes(), r.report.outer_iters, y.tobytes()
    finally:
        if old is None:
            os.environ.pop("CS_SPMV_BOX", None)
        else:
            os.environ["CS_SPMV_BOX"] = old


@pytest.mark.parametrize("dims", SHAPES)
def test_box_spmv_bitwise_and_solve_identical(cs, port, dims):
    o = port.poisson27(*dims)
    x = np.random.default_rng(11).standard_normal(o.n)
    want = port.spmv(o, x)
    p = cs.DeviceProblem.generate("poisson27", *dims).set_precond("jacobi")
    try:
        assert p.cdia_classes >= 1
        os.environ.pop("CS_SPMV_BOX", None)
        assert p.spmv(x).tobytes() == want.tobytes()
        lam = cs.SpectrumEstimate(*port.estimate_interval(o, 1))
        on = _solve(cs, p, lam, True)
        off = _solve(cs, p, lam, False)
        assert on[1] == off[1], (on[1], off[1])
        assert on[0] == off[0], "box-kernel solve differs from the gather-kernel solve"
        assert on[2] == off[2]
    finally:
        p.close()
