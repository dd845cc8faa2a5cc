"""Time the SpMV-family kernels alone on a device-generated problem.

    python tools/spmv_micro.py [--n 256] [--stencil poisson27]
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_09790_b200 as cs  # noqa: E402
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--stencil", default="poisson27")
ap.add_argument("--kinds", default="plain,mpk_ref,mpk_fast,pack8,update8")
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
p = cs.DeviceProblem.generate(a.stencil, a.n, a.n, a.n).set_precond("jacobi")
n, mat = p.n_local, p.device_bytes
v = 8 * n
res = {}
print(f"format: slices={p.slices} pattern={p.pattern_slices} uniform={p.uniform_slices} "
      f"table_entries={p.pattern_entries} bytes={mat}")
for kind, byts in (("plain", mat + 2 * v), ("mpk_ref", mat + 7 * v), ("mpk_fast", mat + 5 * v),
                   ("pack8", (18 if os.environ.get("CS_BENCH_PZ") else 25) * v),
                   ("update8", (45 if os.environ.get("CS_BENCH_PZ") else 54) * v)):
    if kind not in a.kinds.split(","):
        continue
    ms = p.bench_spmv(kind, a.reps)
    res[kind] = (round(ms, 4), round(byts / (ms / 1e3) / 1e9))
print(f"{os.environ.get('CS_LIB', 'default')} {a.stencil} {a.n}^3 mat {mat/p.nnz_local:.2f} B/nnz "
      f"explicit={bool(os.environ.get('CS_SELL_EXPLICIT'))} values={bool(os.environ.get('CS_SELL_VALUES'))}: " +
      " ".join(f"{k}={v[0]}ms/{v[1]}GB/s" for k, v in res.items()))
