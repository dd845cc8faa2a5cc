"""CPU-only: the C-ABI library loads, exports every symbol include/chebstep_gpu.h
declares, its host-only entries (partitioning, halo maps, tridiagonal
eigenvalues) work without a GPU, and compute entries fail loudly -- there is
no CPU fallback."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "chebstep_gpu.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(cs_[a-z0-9_]+)\s*\(", txt)))


def test_header_symbols_exported():
    import paper_2603_09790_b200 as cs
    lib = ctypes.CDLL(cs.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    from paper_2603_09790_b200 import _lib
    assert set(declared_symbols()) <= set(_lib.SIGNATURES)


def test_library_is_sm100a():
    import paper_2603_09790_b200 as cs
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", cs.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_partition_rows():
    import paper_2603_09790_b200 as cs
    plane, nz = 64, 10
    for P in (1, 2, 3, 4, 8, 10):
        spans = [cs.partition_rows(plane * nz, plane, P, r) for r in range(P)]
        assert spans[0][0] == 0 and spans[-1][1] == plane * nz
        for (b0, e0), (b1, e1) in zip(spans, spans[1:]):
            assert e0 == b1
        assert all((e - b) % plane == 0 and e > b for b, e in spans)
        sizes = [(e - b) // plane for b, e in spans]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(cs.InvalidArgumentError):
        cs.partition_rows(plane * nz, plane, 11, 0)


def test_halo_map_matches_planes(port):
    """General-CSR halo map on z-slabs of the 27-point operator == the plane layout
    the device generator uses (lower ghost plane, then upper), columns remapped with
    the in-row order untouched."""
    import paper_2603_09790_b200 as cs
    nx, ny, nz, P = 7, 5, 9, 3
    o = port.poisson27(nx, ny, nz)
    plane = nx * ny
    for r in range(P):
        b, e = cs.partition_rows(o.n, plane, P, r)
        rp = o.rowptr[b:e + 1] - o.rowptr[b]
        cg = o.col[o.rowptr[b]:o.rowptr[e]]
        ghosts, cl = cs.halo_map_csr(b, e, rp, cg)
        want = []
        if b > 0:
            want += list(range(b - plane, b))
        if e < o.n:
            want += list(range(e, e + plane))
        assert ghosts.tolist() == want
        back = np.where(cl < e - b, cl + b, ghosts[np.maximum(cl - (e - b), 0)])
        assert back.tolist() == cg.tolist()


def test_tridiag_eigvals_host_only(port):
    import paper_2603_09790_b200 as cs
    rng = np.random.default_rng(2)
    d, e = rng.uniform(0.1, 3, 40), rng.uniform(0.001, 0.6, 39)
    ev = cs.tridiag_eigvals(d, e)
    t = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    np.testing.assert_allclose(ev, np.linalg.eigvalsh(t), rtol=1e-13, atol=1e-14)


def test_compute_entries_fail_without_gpu():
    import paper_2603_09790_b200 as cs
    if cs.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(cs.CudaError):
        cs.Context(0)
    with pytest.raises(cs.CudaError):
        cs.spmv(cs.CsrMatrix.identity(4), np.ones(4))


def test_product_does_not_import_oracle():
    """The product package never references the test oracle."""
    pkg = os.path.join(ROOT, "paper_2603_09790_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "cs_oracle" not in txt and "libchebstep_ref" not in txt, f


def test_python_constants_match_header():
    """Every CS_VAR_* / CS_MODE_* / CS_PRECOND_* value the Python mirror uses is
    the header's (the schedule bits are checked by the GPU solver tests)."""
    import re
    from paper_2603_09790_b200 import _lib as L
    hdr = open(os.path.join(ROOT, "include", "chebstep_gpu.h")).read()
    defs = dict(re.findall(r"#define\s+(CS_VAR_\w+)\s+(\d+)", hdr))
    assert defs, "no CS_VAR_* in the header"
    for name, val in defs.items():
        assert getattr(L, name) == int(val), name
