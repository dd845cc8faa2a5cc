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
