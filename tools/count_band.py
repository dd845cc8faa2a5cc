"""Outer-count sensitivity of the s-step solve at BASELINE scale.

    python tools/count_band.py [--cases p27:128:8,p27:256:8] [--out profiles/r02_count_band.json]

For each case (stencil:N:s, nu = 30, Jacobi, tol 1e-8, b = 1, x0 = 0) every run
uses the SAME spectrum (the reference's golden lambda where one exists, else
this device's Lanczos), so only the arithmetic differs:

  reference band  reference algebra (explicit W, b1, b2; serial reductions) with
                  lambda exact, lambda * (1 -+ 1e-13), lambda * (1 -+ 1e-12)
                  (SURVEY App. B.1), and with tree reductions (App. B.2);
  attribution     the fast one-allreduce algebra as shipped, then with each
                  non-reference rounding switched back in turn (CS_VAR_*):
                  explicit W_k per outer, reference FGS sequence, reference MPK
                  epilogue, and all three.

Every run records the outer count, the final recurrence residual and
||x - x_ref|| / ||x_ref|| against the exact-lambda reference-algebra x.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def golden_lambda(kind, n, s):
    with open(os.path.join(ROOT, "tests", "golden", "outer_counts.json")) as f:
        g = json.load(f)
    key = f"{'p27' if kind == 'poisson27' else 'p7'}_{n}x{n}x{n}_s{s}_nu30_jacobi_1e-08"
    if key in g:
        return g[key]["lambda_min"], g[key]["lambda_max"], g[key]["outer_iters"], g[key].get("x_norm")
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="p27:128:8,p27:96:8,p27:128:4,p7:256:4,p27:256:8")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_count_band.json"))
    ap.add_argument("--skip-ref", action="store_true", help="no serial reference-algebra runs")
    ap.add_argument("--ref-only", action="store_true",
                    help="only the exact-lambda serial reference run (for rel_x_vs_ref)")
    ap.add_argument("--variants", default="")
    ap.add_argument("--tree-band", action="store_true",
                    help="reference band with tree reductions (fast) instead of serial chains")
    a = ap.parse_args()
    import paper_2603_09790_b200 as cs
    from paper_2603_09790_b200 import _lib as L

    ctx = cs.Context(0)
    cs.set_default_context(ctx)
    results = []
    if os.path.exists(a.out):
        with open(a.out) as f:
            results = json.load(f).get("runs", [])
    for case in a.cases.split(","):
        st, n, s = case.split(":")
        n, s = int(n), int(s)
        kind = "poisson27" if st == "p27" else "poisson7"
        p = cs.DeviceProblem.generate(kind, n, n, n)
        p.set_precond("jacobi")
        gl = golden_lambda(kind, n, s)
        if gl:
            lo, hi, gcount, gnorm = gl
            lam_src = "golden (reference library)"
        else:
            est = p.estimate_interval(40, 1234, "fast")
            lo, hi, gcount, gnorm = est.lambda_min, est.lambda_max, None, None
            lam_src = "device Lanczos (fast)"
        print(f"== {case}: lambda [{lo!r}, {hi!r}] ({lam_src}), golden outer {gcount}", flush=True)

        def run(label, mode, variant=0, eps=0.0):
            spec = cs.SpectrumEstimate(lo * (1 + eps), hi * (1 - eps), "injected", 0.9, 1.1)
            cfg = cs.SolverConfig(s=s, tol=1e-8, max_outer=20000, mode=mode, variant=variant,
                                  spectrum=spec)
            t0 = time.time()
            res = p.pcg_s_solve(cfg=cfg)
            dt = time.time() - t0
            r = res.report
            return {"case": case, "label": label, "mode": mode, "variant": variant, "eps": eps,
                    "outer": r.outer_iters, "converged": bool(r.converged),
                    "final_rel": r.rel_residual[-1], "max_delta_alpha": max(r.delta_alpha),
                    "x_norm": float(np.linalg.norm(res.x)), "wall_s": round(dt, 2),
                    "t_solve_ms": round(r.t_solve_ms, 2),
                    "ms_per_outer": round(r.t_solve_ms / max(r.outer_iters, 1), 4),
                    "golden_outer": gcount}, res.x

        xref = None
        runs = []

        def add(label, mode, variant=0, eps=0.0):
            nonlocal xref
            d, x = run(label, mode, variant, eps)
            if xref is None and mode == "reference" and eps == 0.0 and variant == 0:
                xref = x
            if xref is not None:
                d["rel_x_vs_ref"] = float(np.linalg.norm(x - xref) / np.linalg.norm(xref))
            runs.append(d)
            print(json.dumps(d), flush=True)

        if a.tree_band:  # reference algebra, tree reductions, lambda perturbed
            for eps in (0.0, 1e-13, -1e-13, 1e-12, -1e-12, 1e-11, -1e-11, 1e-10, -1e-10, 1e-9,
                        -1e-9):
                add(f"reference-tree lambda*(1{'-' if eps >= 0 else '+'}{abs(eps):g})", "reference",
                    L.CS_VAR_TREE, eps)
        elif a.ref_only:
            add("reference", "reference")
        elif not a.skip_ref:
            add("reference", "reference")
            for eps in (1e-13, -1e-13, 1e-12, -1e-12):
                add(f"reference lambda*(1{'-' if eps > 0 else '+'}{abs(eps):g})", "reference", 0, eps)
            add("reference, tree reductions", "reference", L.CS_VAR_TREE)
        variants = [("fast, stored P (round 1)", L.CS_VAR_P_STORED),
                    ("fast shipped", 0),
                    ("fast + explicit W", L.CS_VAR_EXPLICIT_W),
                    ("fast + reference FGS", L.CS_VAR_REF_FGS),
                    ("fast + reference MPK", L.CS_VAR_REF_MPK),
                    ("fast + explicit W + ref FGS + ref MPK",
                     L.CS_VAR_EXPLICIT_W | L.CS_VAR_REF_FGS | L.CS_VAR_REF_MPK),
                    ("fast, stored P + explicit W", L.CS_VAR_P_STORED | L.CS_VAR_EXPLICIT_W),
                    ("fast, true residual", L.CS_VAR_TRUE_R),
                    ("fast, recursive residual", L.CS_VAR_RECUR_R)]
        if a.variants:
            keep = set(a.variants.split(","))
            variants = [v for v in variants if str(v[1]) in keep]
        for label, var in variants:
            add(label, "fast", var)
        results = [r for r in results if r["case"] != case] + runs
        with open(a.out, "w") as f:
            json.dump({"lambda_note": "golden lambda injected where the reference has one",
                       "runs": results}, f, indent=1)
        p.close()


if __name__ == "__main__":
    main()
