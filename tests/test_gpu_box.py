"""Plane-streaming box SpMV (spmv.cu sell_box_kernel).

27-point classes whose table is a 3x3x3 box in natural ordering are applied
plane by plane from shared memory. In the reference order the kernel must give the
CDIA row sums bit for bit: the SpMV equals the CPU oracle, and fast-algebra
solves are bitwise the same with the kernel switched off (CS_SPMV_BOX=0: gather
kernels) when its separable variant is off (CS_BOX_SEP=0); with it (the
default for the fast MPK kinds) the solution agrees to 1e-8. Shapes cover several T-row columns per
plane, partial columns, planes not a multiple of 32 rows, and thin grids."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPES = [(64, 64, 40), (70, 50, 13), (40, 36, 30), (5, 4, 7), (128, 96, 9), (33, 20, 11),
          (16, 40, 12), (256, 9, 7)]


def _solve(cs, p, lam, box, sep=True, nobits=True, variant=0, vstrip=True, sepk=True, ws=True):
    env = {"CS_SPMV_BOX": "1" if box else "0", "CS_BOX_SEP": "1" if sep else "0",
           "CS_BOX_NOBITS": "1" if nobits else "0", "CS_BOX_VSTRIP": "1" if vstrip else "0",
           "CS_BOX_SEPK": "1" if sepk else "0", "CS_BOX_WS": "1" if ws else "0"}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        r = p.pcg_s_solve(cfg=cs.SolverConfig(s=8, tol=1e-8, max_outer=3000, spectrum=lam,
                                              variant=variant))
        y = p.spmv(np.arange(p.n_local, dtype=np.float64) % 7 - 3.0)
        return r.x, r.report.outer_iters, y.tobytes()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


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
        exact = _solve(cs, p, lam, True, sep=False)
        off = _solve(cs, p, lam, False)
        assert exact[1] == off[1], (exact[1], off[1])
        assert exact[0].tobytes() == off[0].tobytes(), "box solve differs from the gather solve"
        assert exact[2] == off[2]
        # default: the fast MPK kinds take the separable plane sums on these
        # geometric classes (another rounding of the same row sums): same x to 1e-8
        sep = _solve(cs, p, lam, True)
        assert sep[2] == off[2]  # plain SpMV stays in the exact order
        assert abs(sep[1] - off[1]) <= max(2, off[1] // 20), (sep[1], off[1])
        assert np.linalg.norm(sep[0] - off[0]) / np.linalg.norm(off[0]) <= 1e-8
        # face bits from the plane index and one plane per column (no participation
        # stream) vs from the stream: the same arithmetic, bit for bit -- in both
        # residual schedules (the true residual runs its b - A x through the kernel)
        # and the vertical-strip row mapping (line sums shared by a thread's R
        # consecutive lines, where the line length divides the block) vs the
        # strided mapping: the same sums in the same order
        for variant in (256, 128):
            a = _solve(cs, p, lam, True, nobits=True, variant=variant)
            b = _solve(cs, p, lam, True, nobits=False, variant=variant)
            assert a[1] == b[1] and a[0].tobytes() == b[0].tobytes(), (variant, a[1], b[1])
            for nb in (True, False):
                c = _solve(cs, p, lam, True, nobits=nb, variant=variant, vstrip=False)
                assert c[1] == a[1] and c[0].tobytes() == a[0].tobytes(), (variant, nb)
            # the compile-time specialised planar kernel (with and without its
            # producer warp) vs the general kernel's separable path
            for sepk, ws in ((False, True), (True, False)):
                c = _solve(cs, p, lam, True, variant=variant, sepk=sepk, ws=ws)
                assert c[1] == a[1] and c[0].tobytes() == a[0].tobytes(), (variant, sepk, ws)
    finally:
        p.close()
