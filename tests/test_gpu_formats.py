"""Every device storage format gives the same bits.

The conversion SELL-32 -> SELL-32P -> SELL-32PU -> CDIA is chosen per slice
from the matrix; environment switches force the earlier formats:
CS_SELL_EXPLICIT=1 (explicit int32 columns everywhere), CS_SELL_VALUES=1
(pattern slices keep their value slots), CS_SELL_CDIA=0 (uniform tables, no
constant-diagonal classes). For each format: the SpMV equals the CPU oracle
bit for bit, and a fast-algebra solve is bitwise identical to the default
format's (same spectrum injected; exact-order box kernel, CS_BOX_SEP=0)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FORMATS = {
    "explicit": {"CS_SELL_EXPLICIT": "1"},
    "pattern_values": {"CS_SELL_VALUES": "1"},
    "uniform_tables": {"CS_SELL_CDIA": "0"},
    "cdia": {},
}
CASES = [("poisson27", (32, 32, 32), None), ("poisson27", (33, 17, 9), None),
         ("poisson7", (24, 24, 24), None), ("aniso7", (20, 18, 16), (1.0, 1.0, 100.0))]


def _generate(cs, kind, dims, coef, env):
    old = {k: os.environ.get(k) for k in ("CS_SELL_EXPLICIT", "CS_SELL_VALUES", "CS_SELL_CDIA")}
    try:
        for k in old:
            os.environ.pop(k, None)
        os.environ.update(env)
        return cs.DeviceProblem.generate(kind, *dims, coef or (1.0, 1.0, 1.0)).set_precond("jacobi")
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _oracle(port, kind, dims, coef):
    if kind == "poisson27":
        return port.poisson27(*dims)
    return port.stencil7(*dims, coef=coef or (1.0, 1.0, 1.0))


@pytest.mark.parametrize("kind,dims,coef", CASES)
def test_formats_spmv_and_solve_bitwise(cs, port, kind, dims, coef, monkeypatch):
    # the exact-order kernels (the box kernel's separable fast variant is another
    # rounding; tests/test_gpu_box.py bounds it)
    monkeypatch.setenv("CS_BOX_SEP", "0")
    o = _oracle(port, kind, dims, coef)
    x = np.random.default_rng(5).standard_normal(o.n)
    want = port.spmv(o, x)
    sols = {}
    for name, env in FORMATS.items():
        p = _generate(cs, kind, dims, coef, env)
        try:
            if name == "cdia":
                assert p.cdia_classes >= 1, "stencils convert to constant-diagonal classes"
            if name == "explicit":
                assert p.pattern_slices == 0
            if name == "pattern_values":
                assert p.uniform_slices == 0 and p.pattern_slices > 0
            y = p.spmv(x)
            assert y.tobytes() == want.tobytes(), name
            lam = cs.SpectrumEstimate(*port.estimate_interval(o, 1))
            r = p.pcg_s_solve(cfg=cs.SolverConfig(s=4, tol=1e-8, max_outer=2000, spectrum=lam))
            sols[name] = (r.x.tobytes(), r.report.outer_iters)
        finally:
            p.close()
    ref = sols["cdia"]
    for name, v in sols.items():
        assert v == ref, f"{name} differs from the CDIA solve"


def test_shuffled_operator_stays_explicit(cs, port):
    """A reordered operator (rows shuffled inside windows, columns renumbered)
    has slices whose 32 rows share few relative offsets: the conversion must keep
    them as explicit SELL-32 (a uniform table would be ~800 entries walked one by
    one per warp: 5x slower, profiles/r02h_irregular_spmv_128.txt) -- and the
    SpMV stays bitwise the oracle's."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "tools"))
    from irregular_bench import permuted
    o = port.poisson27(24, 24, 24)
    a = cs.CsrMatrix(o.n, o.rowptr, o.col, o.val)
    rp, col, val = permuted(a, 4096)
    p = cs.DeviceProblem.from_csr(cs.CsrMatrix(o.n, rp, col, val))
    try:
        assert p.uniform_slices == 0 and p.cdia_classes == 0, (p.uniform_slices, p.cdia_classes)
        assert p.device_bytes / p.nnz_local < 14.0  # explicit: 8 B value + 4 B column (+ slice padding)
        from oracle.oracle import Csr
        q = Csr(o.n, rp, col, val)
        x = np.random.default_rng(5).standard_normal(o.n)
        assert p.spmv(x).tobytes() == port.spmv(q, x).tobytes()
    finally:
        p.close()
