"""Small end-to-end workload for compute-sanitizer (memcheck / synccheck / racecheck).

    compute-sanitizer --tool memcheck python tools/sanitize_case.py
    compute-sanitizer --tool racecheck python tools/sanitize_case.py --quick

Covers the hot kernels on a 27-point 64^3 problem (the plane-streaming box
SpMV with its cp.async.bulk/mbarrier ring, the fused MPK epilogues, the DMMA
pack reduction, the fused update pass, the single-CTA Gram step, the Lanczos
kernels) plus the streamed CSR upload and the gather SpMV of an irregular
matrix. Prints one line per stage; any sanitizer error is reported by the tool.
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="fewer outer iterations (racecheck is slow)")
    a = ap.parse_args()
    import paper_2603_09790_b200 as cs
    from paper_2603_09790_b200 import _lib as L

    ctx = cs.Context(0)
    cs.set_default_context(ctx)
    mo = 2 if a.quick else 6
    p = cs.DeviceProblem.generate("poisson27", 64, 64, 64).set_precond("jacobi")
    print("problem: cdia classes", p.cdia_classes, flush=True)
    for var in (0, L.CS_VAR_EXPLICIT_W):
        r = p.pcg_s_solve(cfg=cs.SolverConfig(s=8, tol=1e-8, max_outer=mo, variant=var))
        print(f"fast solve variant {var}: outer {r.report.outer_iters}", flush=True)
    r = p.pcg_s_solve(cfg=cs.SolverConfig(s=4, tol=1e-8, max_outer=2, mode="reference",
                                          lanczos_steps=4))
    print("reference solve: outer", r.report.outer_iters, flush=True)
    rp = p.pcg_solve(tol=1e-8, max_iter=5)
    print("classical pcg: iters", rp.report.outer_iters, flush=True)
    y = p.spmv(np.ones(p.n_local))
    print("spmv ok", float(y.sum()), flush=True)
    # irregular matrix through the streamed host-CSR upload (small chunks: several stages)
    os.environ["CS_UPLOAD_CHUNK_NNZ"] = "4096"
    rng = np.random.default_rng(1)
    n = 3000
    rows = [[] for _ in range(n)]
    for i in range(n):
        rows[i].append((i, 8.0))
        for j in rng.choice(n, 3, replace=False):
            if j != i:
                rows[i].append((int(j), -0.5))
                rows[int(j)].append((i, -0.5))
    rp_, ci, va = [0], [], []
    for i in range(n):
        d = {}
        for j, v in rows[i]:
            d[j] = d.get(j, 0.0) + v
        for j in sorted(d):
            ci.append(j)
            va.append(d[j])
        rp_.append(len(ci))
    A = cs.CsrMatrix(n, np.array(rp_, np.int64), np.array(ci, np.int64), np.array(va))
    res = cs.pcg_s_solve(A, np.ones(n), np.zeros(n), cs.JacobiPreconditioner(A),
                         cs.SolverConfig(s=4, tol=1e-8, max_outer=mo))
    print("irregular csr solve: outer", res.report.outer_iters, flush=True)
    p.close()
    print("sanitize case done", flush=True)


if __name__ == "__main__":
    main()
