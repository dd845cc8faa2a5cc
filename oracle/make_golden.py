"""make_golden.py -- TEST INFRASTRUCTURE ONLY. Generates tests/golden/*.json
from the compiled, unmodified reference library (oracle/_ref, built by
oracle/Makefile from /root/reference/proj/src). Run in the development
container (where /root/reference exists):

    make -C oracle all && python oracle/make_golden.py

Fixtures are small (hashes + short histories); tests/test_oracle.py pins the C
restatement to them and the GPU tests compare against the restatement.
Long-running golden outer counts (64^3 .. 256^3, from oracle/_ref/ref_probe)
are merged from --probe-json files into outer_counts.json.
"""
from __future__ import annotations

import argparse
import glob
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle.oracle import Csr, Oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")


def h(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def problem(port, name):
    kind, n = name.split("_")
    n = int(n)
    return port.poisson27(n) if kind == "p27" else port.stencil7(n)


SOLVES = [
    # name, s, nu, gram, tol, precond
    ("p27_16", 4, 30, "fgs", 1e-6, 0),
    ("p27_16", 4, 30, "cholesky", 1e-6, 0),
    ("p27_16", 2, 30, "fgs", 1e-6, 0),
    ("p27_16", 6, 30, "fgs", 1e-6, 0),
    ("p27_8", 4, 30, "fgs", 1e-6, 0),
    ("p27_8", 4, 30, "cholesky", 1e-6, 0),
    ("p7_32", 4, 2, "fgs", 1e-8, 1),
    ("p27_32", 8, 30, "fgs", 1e-8, 1),
    ("p27_32", 12, 30, "fgs", 1e-8, 1),
    ("p27_32", 4, 30, "cholesky", 1e-8, 1),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--probe-json", nargs="*", default=[])
    args = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    ref, port = Oracle("ref"), Oracle("port")

    # ---- KATs (SPEC.md examples, evaluated by the reference binary)
    kats = {}
    a = ref.poisson27(4)
    kats["poisson27_4"] = {"nnz": a.nnz, "row0_len": int(a.rowptr[1]), "row0_sum": float(a.val[:a.rowptr[1]].sum()),
                           "rowptr_sha": h(a.rowptr), "col_sha": h(a.col), "val_sha": h(a.val)}
    for n in (16, 33):
        a = ref.poisson27(n, n + 1, n - 1)
        kats[f"poisson27_{n}x{n+1}x{n-1}"] = {"nnz": a.nnz, "rowptr_sha": h(a.rowptr),
                                             "col_sha": h(a.col), "val_sha": h(a.val)}
    d = Csr(2, np.array([0, 1, 2]), np.array([0, 1]), np.array([1.0, 3.0]))
    z, p = ref.mpk(d, np.array([1.0, 1.0]), 3, 1.0, 3.0, precond=0)
    kats["mpk_diag13"] = {"z": z.tolist(), "p": p.tolist()}
    w = np.array([[1.0, 0.5], [0.5, 1.0]])
    for nu in (1, 50):
        x, dl = ref.fgs_solve(w, np.array([1.0, 0.0]), nu)
        kats[f"fgs_2x2_nu{nu}"] = {"x": x[:, 0].tolist(), "delta": dl}
    r = np.random.default_rng(7).standard_normal(5000)
    kats["random_vector_1234"] = {"n": 5000, "sha": h(ref.random_vector(5000, 1234)),
                                  "head": ref.random_vector(4, 1234).tolist()}
    a = ref.poisson27(12, 10, 9)
    r = np.random.default_rng(11).standard_normal(a.n)
    kats["spmv_p27_12x10x9_rng11"] = {"sha": h(ref.spmv(a, r))}
    for s, pc in ((5, 1), (3, 0)):
        z, p = ref.mpk(a, r, s, 0.05 if pc else 1.0, 1.6 if pc else 40.0, precond=pc)
        kats[f"mpk_p27_12x10x9_s{s}_pc{pc}"] = {"z_sha": h(z), "p_sha": h(p)}
    rng = np.random.default_rng(3)
    q = rng.standard_normal((6, 4000))
    aq = q + 0.01 * rng.standard_normal((6, 4000))
    kats["assemble_gram_rng3"] = {"w_sha": h(ref.assemble_gram(q, aq))}
    kats["block_gram_rng3"] = {"g_sha": h(ref.block_gram(q, aq))}
    c = rng.standard_normal((6, 6))
    kats["block_update_rng3"] = {"sha": h(ref.block_update(aq, q, c))}
    b = rng.standard_normal((8, 8))
    w8 = b @ b.T + 8 * np.eye(8)
    w8 = 0.5 * (w8 + w8.T)
    rhs = rng.standard_normal((8, 8))
    x, dl = ref.fgs_solve(w8, rhs, 30)
    kats["fgs_8x8_rng3"] = {"x_sha": h(x), "delta": dl}
    kats["chol_8x8_rng3"] = {"x_sha": h(ref.cholesky_solve(w8, rhs))}
    with open(os.path.join(OUT, "kats.json"), "w") as f:
        json.dump(kats, f, indent=1)

    # ---- spectra (Lanczos 40 steps, seed 1234, dsterf)
    spectra = {}
    for name in ("p27_16", "p27_32", "p7_32", "p27_8"):
        o = problem(port, name)
        for pc in (0, 1):
            spectra[f"{name}_pc{pc}"] = list(ref.estimate_interval(o, pc))
    with open(os.path.join(OUT, "spectra.json"), "w") as f:
        json.dump(spectra, f, indent=1)

    # ---- solves with the reference spectrum injected
    solves = {}
    for name, s, nu, gram, tol, pc in SOLVES:
        o = problem(port, name)
        lam = tuple(spectra[f"{name}_pc{pc}"])
        key = f"{name}_s{s}_nu{nu}_{gram}_tol{tol:g}_pc{pc}"
        try:
            x, rp = ref.pcg_s_solve(o, s=s, nu=nu, gram=gram, tol=tol, spectrum=lam, precond=pc,
                                    max_outer=5000)
            solves[key] = {"spectrum": list(lam), "outer_iters": rp.outer_iters,
                           "converged": rp.converged, "spmv_count": rp.spmv_count,
                           "precond_count": rp.precond_count, "allreduce_count": rp.allreduce_count,
                           "local_update_flops": rp.local_update_flops,
                           "gram_solve_flops": rp.gram_solve_flops,
                           "rel_residual_sha": h(rp.rel_residual),
                           "delta_alpha_sha": h(rp.delta_alpha), "delta_beta_sha": h(rp.delta_beta),
                           "rel_residual_tail": rp.rel_residual[-3:].tolist(),
                           "x_sha": h(x), "x_sum": float(x.sum()), "x_norm": float(np.linalg.norm(x))}
        except Exception as e:  # breakdown cases are goldens too
            solves[key] = {"spectrum": list(lam), "error": getattr(e, "code", -1),
                           "payload": getattr(e, "payload", -1), "msg": str(e)}
        # classical PCG comparator
    for name in ("p27_32", "p7_32"):
        o = problem(port, name)
        x, rp = ref.pcg_solve(o, tol=1e-8, max_iter=5000)
        solves[f"{name}_pcg_tol1e-08_pc1"] = {"outer_iters": rp.outer_iters, "x_sha": h(x),
                                              "rel_residual_sha": h(rp.rel_residual)}
    with open(os.path.join(OUT, "solves.json"), "w") as f:
        json.dump(solves, f, indent=1)

    # ---- long-run outer counts from ref_probe JSON lines
    path = os.path.join(OUT, "outer_counts.json")
    table = json.load(open(path)) if os.path.exists(path) else {}
    for pj in args.probe_json:
        for fn in glob.glob(pj):
            for line in open(fn):
                line = line.strip()
                if not line.startswith("{"):
                    continue
                d = json.loads(line)
                n = d["N"]
                key = (f"p{d['stencil']}_{n}x{n}x{n}_s{d['s']}_nu{d['nu']}_{d['precond']}_"
                       f"{d['tol']:.0e}".replace("e-0", "e-0"))
                if d["method"] == "pcg":
                    key = f"p{d['stencil']}_{n}x{n}x{n}_pcg_{d['precond']}_{d['tol']:.0e}"
                elif d["method"] == "pcgs-cholesky":
                    key += "_cholesky"
                table[key] = {k: d[k] for k in ("outer_iters", "converged", "spmv_count",
                                                "lambda_min", "lambda_max", "final_rel_residual",
                                                "max_delta_alpha", "x_sum", "x_norm",
                                                "t_lanczos_s", "t_solve_s")}
                table[key]["source"] = "oracle/_ref/ref_probe (unmodified reference, 1 core)"
    with open(path, "w") as f:
        json.dump(table, f, indent=1, sort_keys=True)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
