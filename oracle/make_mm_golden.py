"""make_mm_golden.py -- TEST INFRASTRUCTURE ONLY. Generates
tests/golden/mm_cases.json: Matrix Market inputs (as text) with the result of
the UNMODIFIED reference reader (oracle/_ref: chebstep::read_matrix_market,
problems.cpp:55-109) -- either the CSR it returns or the error code + message
it throws -- plus CSR validation cases (csr.cpp:58-110) and the reference
writer's exact output (problems.cpp:111-127).

    make -C oracle all && python oracle/make_mm_golden.py
"""
from __future__ import annotations

import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle.oracle import Csr, Oracle, OracleError  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden", "mm_cases.json")
HDR = "%%MatrixMarket matrix coordinate real symmetric\n"

READ_CASES = [
    # name, text, require_spd
    ("tridiag", HDR + "3 3 5\n1 1 2\n2 1 -1\n2 2 2\n3 2 -1\n3 3 2\n", True),
    ("shuffled_comments_blank_crlf",
     HDR + "% a comment\n\n3 3 5\r\n3 3 2.5e0\r\n% inside\n2 1 -1\n\n1 1 +2\n3 2 -.5\n2 2 2.\n", True),
    ("upper_triangle_given", HDR + "2 2 3\n1 1 4\n1 2 1\n2 2 4\n", True),
    ("uppercase_header", "%%MatrixMarket MATRIX Coordinate REAL Symmetric\n2 2 2\n1 1 1\n2 2 1\n",
     False),
    ("trailing_tokens_ignored", HDR + "2 2 2\n1 1 1 extra stuff\n2 2 3 4 5\n", False),
    ("garbage_after_declared_entries", HDR + "2 2 2\n1 1 1\n2 2 1\nthis is not an entry\n", False),
    ("hex_prefix_reads_zero", HDR + "2 2 2\n1 1 0x1p3\n2 2 1\n", False),
    ("exponent_forms", HDR + "3 3 3\n1 1 1E-3\n2 2 -2.5e+10\n3 3 4.9e-324\n", False),
    ("empty_file", "", False),
    ("bad_banner", "%MatrixMarket matrix coordinate real symmetric\n1 1 1\n1 1 1\n", False),
    ("array_format", "%%MatrixMarket matrix array real symmetric\n1 1 1\n1 1 1\n", False),
    ("complex_field", "%%MatrixMarket matrix coordinate complex symmetric\n1 1 1\n1 1 1 0\n", False),
    ("general_symmetry", "%%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 1\n", False),
    ("no_size_line", HDR + "% only comments\n", False),
    ("bad_size_line", HDR + "3 x 3\n", False),
    ("non_square", HDR + "3 4 1\n1 1 1\n", False),
    ("zero_entries", HDR + "3 3 0\n", False),
    ("missing_value", HDR + "2 2 2\n1 1\n2 2 1\n", False),
    ("nan_value", HDR + "2 2 2\n1 1 nan\n2 2 1\n", False),
    ("inf_value", HDR + "2 2 2\n1 1 inf\n2 2 1\n", False),
    ("overflow_value", HDR + "2 2 2\n1 1 1e400\n2 2 1\n", False),
    ("dangling_exponent", HDR + "2 2 2\n1 1 1e\n2 2 1\n", False),
    ("blank_line_with_spaces", HDR + "2 2 2\n1 1 1\n   \n2 2 1\n", False),
    ("index_zero", HDR + "2 2 2\n0 1 1\n2 2 1\n", False),
    ("index_too_large", HDR + "2 2 2\n1 1 1\n3 2 1\n", False),
    ("fewer_entries", HDR + "3 3 3\n1 1 1\n2 2 1\n", False),
    ("duplicate_mirror", HDR + "2 2 4\n1 1 1\n2 1 5\n1 2 5\n2 2 1\n", False),
    ("duplicate_same", HDR + "2 2 3\n1 1 1\n1 1 2\n2 2 1\n", False),
    ("spd_missing_diagonal", HDR + "2 2 2\n1 1 1\n2 1 1\n", True),
    ("spd_nonpositive_diagonal", HDR + "2 2 2\n1 1 1\n2 2 0\n", True),
    ("spd_ok_not_required", HDR + "2 2 2\n1 1 -1\n2 2 0\n", False),
]


def csr_dict(a: Csr) -> dict:
    return {"n": a.n, "rowptr": a.rowptr.tolist(), "col": a.col.tolist(),
            "val_hex": [float(v).hex() for v in a.val]}


def run_read(ref: Oracle, text: str, spd: bool) -> dict:
    with tempfile.NamedTemporaryFile("w", suffix=".mtx", delete=False, newline="") as f:
        f.write(text)
        path = f.name
    try:
        return {"ok": csr_dict(ref.mm_read(path, spd))}
    except OracleError as e:
        return {"error": {"code": e.code, "msg": e.msg.replace(path, "<path>")}}
    finally:
        os.unlink(path)


def validation_cases():
    c = []
    ok = Csr(2, np.array([0, 2, 4]), np.array([0, 1, 0, 1]), np.array([2.0, -1.0, -1.0, 2.0]))
    c.append(("sym_ok", ok))
    c.append(("rowptr0", Csr(2, np.array([1, 2, 4]), np.array([0, 1, 0, 1]), np.ones(4))))
    c.append(("decreasing", Csr(3, np.array([0, 2, 1, 3]), np.array([0, 1, 2]), np.ones(3))))
    c.append(("col_range", Csr(2, np.array([0, 1, 2]), np.array([0, 2]), np.ones(2))))
    c.append(("unsorted", Csr(2, np.array([0, 2, 3]), np.array([1, 0, 1]), np.ones(3))))
    c.append(("repeated_col", Csr(2, np.array([0, 2, 3]), np.array([0, 0, 1]), np.ones(3))))
    c.append(("nonfinite", Csr(2, np.array([0, 1, 2]), np.array([0, 1]), np.array([1.0, np.inf]))))
    c.append(("missing_counterpart", Csr(2, np.array([0, 2, 3]), np.array([0, 1, 1]), np.ones(3))))
    c.append(("counterpart_differs", Csr(2, np.array([0, 2, 4]), np.array([0, 1, 0, 1]),
                                         np.array([2.0, -1.0, -1.5, 2.0]))))
    c.append(("no_diag", Csr(2, np.array([0, 1, 2]), np.array([1, 0]), np.ones(2))))
    c.append(("neg_diag", Csr(2, np.array([0, 1, 2]), np.array([0, 1]), np.array([1.0, -0.0]))))
    return c


def main():
    ref = Oracle("ref")
    out = {"source": "oracle/_ref (unmodified reference read/write_matrix_market, validate_*)",
           "read": [], "validate": [], "write": []}
    for name, text, spd in READ_CASES:
        out["read"].append({"name": name, "text": text, "require_spd": spd,
                            "expect": run_read(ref, text, spd)})
    for name, a in validation_cases():
        res = {}
        for check in (0, 1, 2):
            try:
                ref.csr_validate(a, check)
                res[str(check)] = None
            except OracleError as e:
                res[str(check)] = {"code": e.code, "msg": e.msg}
        out["validate"].append({"name": name, "csr": {"n": a.n, "rowptr": a.rowptr.tolist(),
                                                      "col": a.col.tolist(),
                                                      "val_hex": [float(v).hex() for v in a.val]},
                                "expect": res})
    rng = np.random.default_rng(7)
    vals = np.array([1.0 / 3.0, -0.0, 5e-324, 1e300, -2.5, 123456789.125, 0.1, 1e-5])
    a = Csr(4, np.array([0, 2, 5, 7, 9]), np.array([0, 1, 0, 1, 3, 2, 3, 1, 3]),
            rng.choice(vals, 9))
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "w.mtx")
        ref.mm_write(p, a)
        out["write"].append({"name": "awkward_values", "csr": csr_dict(a),
                             "text": open(p).read()})
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
