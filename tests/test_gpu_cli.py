"""The `chebstep` CLI (reference src/cli.cpp:184-305) on the
device path: file names, CSV schema lines and headers, JSON summary schemas
and keys, exit codes; values equal to the Python mirror's solve of the same
problem (same device arithmetic) and to the reference library within the
spectrum-estimate rounding (the CLI runs its own Lanczos, as the reference's
does)."""
import csv
import json
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2603_09790_b200", "bin", "chebstep")

SOLVE_KEYS = {"schema", "problem", "method", "converged", "outer_iters", "final_rel_residual",
              "counts", "model_flops", "inexact", "config", "spectrum"}


def run(*args):
    return subprocess.run([BIN, *map(str, args)], capture_output=True, text=True, timeout=600)


def read_csv(path):
    with open(path) as f:
        lines = f.read().splitlines()
    return lines[0], lines[1], [r for r in csv.reader(lines[2:])]


def test_cli_usage_codes(cs):
    assert run().returncode == 64
    assert run("solve", "--poisson", 4, 4).returncode == 64
    assert run("solve").returncode == 64  # neither --poisson nor --matrix
    assert run("solve", "--poisson", 4, 4, 4, "--gram", "lu").returncode == 64
    assert run("solve", "--poisson", 4, 4, 4, "--s", "x").returncode == 64
    assert run("solve", "--help").returncode == 0
    assert run("perf-model").returncode == 64


def test_cli_solve_csv_and_json(cs, port, tmp_path):
    out = tmp_path / "s"
    r = run("solve", "--poisson", 12, 12, 12, "--precond", "jacobi", "--s", 4, "--tol", "1e-8",
            "--mode", "reference", "--out", out)
    assert r.returncode == 0, r.stderr
    schema, header, rows = read_csv(out / "solve_history.csv")
    assert schema == "# chebstep-csv v1 solve-history"
    assert header == "k,rel_res,delta_alpha,delta_beta"
    summ = json.load(open(out / "solve_summary.json"))
    assert set(summ) == SOLVE_KEYS
    assert summ["schema"] == "chebstep-solve-summary/1" and summ["problem"] == "poisson-12x12x12"
    assert summ["method"] == "pcgs-fgs"
    assert summ["config"] == {"s": 4, "gram": "fgs", "nu": 30, "tol": 1e-8, "max_outer": 500,
                              "precond": "jacobi", "seed": 1234}
    text = open(out / "solve_summary.json").read()
    assert '"tol": 1e-08' in text and text.startswith('{\n  "config": {\n    "gram": "fgs"')
    # same device arithmetic through the Python mirror: identical numbers
    o = port.poisson27(12)
    a = cs.CsrMatrix(o.n, o.rowptr, o.col, o.val)
    res = cs.pcg_s_solve(a, np.ones(o.n), np.zeros(o.n), cs.JacobiPreconditioner(a),
                         cs.SolverConfig(s=4, tol=1e-8, mode="reference"))
    rep = res.report
    assert len(rows) == rep.outer_iters + 1 == summ["outer_iters"] + 1
    assert [float(r[1]) for r in rows] == list(rep.rel_residual)
    assert rows[0][2] == "" and rows[0][3] == "" and rows[-1][3] == ""
    assert [float(r[2]) for r in rows[1:]] == list(rep.delta_alpha)
    assert summ["counts"] == {"spmv": rep.spmv_count, "precond": rep.precond_count,
                              "allreduce": rep.allreduce_count}
    # the reference library on the same problem (its own Lanczos / dsterf)
    from oracle.oracle import Oracle
    try:
        ref = Oracle("ref")
    except FileNotFoundError:
        return
    _, rr = ref.pcg_s_solve(o, s=4, tol=1e-8, precond=1)
    assert summ["outer_iters"] == rr.outer_iters
    assert summ["spectrum"]["lambda_min"] == pytest.approx(rr.lambda_min, rel=1e-10)
    np.testing.assert_allclose([float(r[1]) for r in rows], rr.rel_residual, rtol=1e-6)
    # --format json: histories inside the summary, no CSV
    out2 = tmp_path / "j"
    r = run("solve", "--poisson", 12, 12, 12, "--precond", "jacobi", "--s", 4, "--tol", "1e-8",
            "--mode", "reference", "--format", "json", "--out", out2)
    assert r.returncode == 0
    s2 = json.load(open(out2 / "solve_summary.json"))
    assert s2["history"]["rel_residual"] == list(rep.rel_residual)
    assert not (out2 / "solve_history.csv").exists()


def test_cli_not_converged_exit_2(cs, tmp_path):
    r = run("solve", "--poisson", 16, 16, 16, "--max-outer", 1, "--out", tmp_path)
    assert r.returncode == 2
    assert json.load(open(tmp_path / "solve_summary.json"))["converged"] is False


def test_cli_compare(cs, tmp_path):
    r = run("compare", "--poisson", 10, 10, 10, "--precond", "jacobi", "--tol", "1e-8",
            "--s", 2, 4, "--out", tmp_path)
    assert r.returncode == 0, r.stderr
    schema, header, rows = read_csv(tmp_path / "compare.csv")
    assert schema == "# chebstep-csv v1 compare-history" and header == "method,s,k,rel_res"
    summ = json.load(open(tmp_path / "compare_summary.json"))
    assert summ["schema"] == "chebstep-compare-summary/1"
    runs = [(x["method"], x["s"]) for x in summ["runs"]]
    assert runs == [("pcg", 1), ("pcgs-cholesky", 2), ("pcgs-cholesky", 4), ("pcgs-fgs", 2),
                    ("pcgs-fgs", 4)]
    assert all(set(x) == {"method", "s", "converged", "iters", "final_rel_residual"}
               for x in summ["runs"])
    assert len(rows) == sum(x["iters"] + 1 for x in summ["runs"])


def test_cli_gram_analysis_matches_reference(cs, tmp_path):
    from oracle.oracle import Oracle
    try:
        ref, port = Oracle("ref"), Oracle("port")
    except FileNotFoundError:
        pytest.skip("reference oracle not built")
    r = run("gram-analysis", "--poisson", 10, 10, 10, "--precond", "jacobi", "--s", 4,
            "--tol", "1e-8", "--mode", "reference", "--out", tmp_path)
    assert r.returncode == 0, r.stderr
    schema, header, rows = read_csv(tmp_path / "gram_analysis.csv")
    assert schema == "# chebstep-csv v1 gram-analysis"
    assert header == ("k,rel_res,delta_alpha,delta_beta,kappa_w,fgs_spectral_norm,"
                      "fgs_spectral_radius,structure_dev")
    o = port.poisson27(10)
    _, rep, hk = ref.pcg_s_solve_hooks(o, s=4, tol=1e-8, collect_gram=True)
    assert len(rows) == rep.outer_iters
    np.testing.assert_allclose([float(x[4]) for x in rows], hk["kappa"], rtol=1e-6)
    _, _, ents = read_csv(tmp_path / "gram_matrices.csv")
    assert len(ents) == rep.outer_iters * 16
    w1 = np.array([float(e[3]) for e in ents[:16]]).reshape(4, 4)
    np.testing.assert_allclose(w1, hk["gram"][0], rtol=1e-9)
    import ctypes as C
    f = ref.lib.ref_fgs_rate_normalized
    f.argtypes = [C.c_int, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    for k, w in enumerate(hk["gram"][:5]):
        a, b = C.c_double(), C.c_double()
        wf = np.asfortranarray(w)
        f(4, wf.ctypes.data, C.byref(a), C.byref(b))
        assert float(rows[k][5]) == pytest.approx(a.value, rel=1e-6)
        assert float(rows[k][6]) == pytest.approx(b.value, rel=1e-6)


def test_cli_matrix_market_input(cs, port, tmp_path):
    o = port.poisson27(9, 8, 7)
    path = tmp_path / "small.mtx"
    cs.write_matrix_market(str(path), cs.CsrMatrix(o.n, o.rowptr, o.col, o.val))
    r = run("solve", "--matrix", path, "--precond", "jacobi", "--tol", "1e-8", "--out", tmp_path)
    assert r.returncode == 0, r.stderr
    summ = json.load(open(tmp_path / "solve_summary.json"))
    assert summ["problem"] == "small.mtx" and summ["converged"]
    r = run("solve", "--matrix", tmp_path / "missing.mtx", "--out", tmp_path)
    assert r.returncode == 1 and "cannot open" in r.stderr
