"""Profiling driver (used under ncu): device-resident 27-pt Poisson solve.

    python tools/profile_solve.py [--n 256] [--s 8] [--solves 1] [--max-outer M]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_09790_b200 as cs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--s", type=int, default=8)
ap.add_argument("--stencil", default="poisson27")
ap.add_argument("--solves", type=int, default=1)
ap.add_argument("--max-outer", type=int, default=50000)
ap.add_argument("--mode", default="fast")
a = ap.parse_args()
p = cs.DeviceProblem.generate(a.stencil, a.n, a.n, a.n).set_precond("jacobi")
cfg = cs.SolverConfig(s=a.s, tol=1e-8, max_outer=a.max_outer, mode=a.mode)
for _ in range(a.solves):
    r = p.pcg_s_solve(cfg=cfg)
    print(f"outer={r.report.outer_iters} launches={r.report.kernel_launches} "
          f"t_solve_ms={r.report.t_solve_ms:.1f} t_lanczos_ms={r.report.t_lanczos_ms:.1f}")
if a.solves >= 1:
    ctx = cs.default_context()
    ctx.reset_timing()
    ctx.set_timing(True)
    r = p.pcg_s_solve(cfg=cfg)
    ctx.set_timing(False)
    t = ctx.timing()
    mat = p.device_bytes
    n = p.n_local
    per = {k: (round(v[0], 3), v[1], round(v[0] / max(v[1], 1), 4)) for k, v in t.items() if v[1]}
    print("timed solve: outer", r.report.outer_iters, "phases (ms, launches, ms/launch):", per)
    sp = t["spmv"]
    print(f"matrix {mat/1e9:.3f} GB ({mat/p.nnz_local:.2f} B/nnz); spmv avg {sp[0]/sp[1]:.4f} ms "
          f"-> {(mat + 24*n)/(sp[0]/sp[1]/1e3)/1e9:.0f} GB/s (mat+3 vectors)")
