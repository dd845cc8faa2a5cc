"""SpMV / solve throughput on an IRREGULAR operator.

    python tools/irregular_bench.py [N] [--window W]

The 27-point Poisson N^3 operator under a random symmetric permutation
P A P^T (rows shuffled inside windows of W rows, columns renumbered and
re-sorted per row, as a reordered Matrix Market input would arrive) is uploaded
through the general CSR path (`DeviceProblem.from_csr`: SELL-32 slices, pattern
/ uniform-value compression where slices still share offsets -- no CDIA class,
no box kernel). One fast-mode solve runs with per-launch CUDA events; the SpMV
phase is reported against its stored-format bytes (the SELL arrays once, x read,
the MPK epilogue vectors) and against the 12 B/nnz + 16 B/row CSR figure of
SURVEY 8(d). The natural-order operator is timed the same way for comparison.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def permuted(a, window, seed=7):
    """P A P^T with rows shuffled inside windows (vectorised)."""
    rng = np.random.default_rng(seed)
    n = a.n
    perm = np.arange(n)
    for s in range(0, n, window):
        rng.shuffle(perm[s:s + window])
    inv = np.empty_like(perm)
    inv[perm] = np.arange(n)
    rp = np.asarray(a.row_offsets)
    lens = np.diff(rp)
    rows_old = np.repeat(np.arange(n), lens)
    rows_new = inv[rows_old]
    cols_new = inv[np.asarray(a.col_indices)]
    order = np.lexsort((cols_new, rows_new))
    new_rp = np.concatenate([[0], np.cumsum(np.bincount(rows_new, minlength=n))]).astype(np.int64)
    return new_rp, cols_new[order].astype(np.int64), np.asarray(a.values)[order]


def measure(cs, ctx, p, s, label):
    import torch
    nl = p.n_local
    dev = torch.device("cuda", 0)
    b = torch.ones(nl, dtype=torch.float64, device=dev)
    x0 = torch.zeros(nl, dtype=torch.float64, device=dev)
    x = torch.empty(nl, dtype=torch.float64, device=dev)
    cfg = cs.SolverConfig(s=s, tol=1e-8, max_outer=50000)
    p.pcg_s_solve_device(b.data_ptr(), x0.data_ptr(), x.data_ptr(), cfg)  # warm-up
    ctx.reset_timing()
    ctx.set_timing(True)
    t0 = time.perf_counter()
    rep = p.pcg_s_solve_device(b.data_ptr(), x0.data_ptr(), x.data_ptr(), cfg)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ctx.set_timing(False)
    ph = ctx.timing()
    v = 8 * nl
    # every SpMV of the solve: the stored SELL arrays once + x read + y/z written
    # (+ the epilogue's z_{q-2}); counted per launch family as in bench.py
    nspmv = rep.spmv_count + 40  # + the Lanczos SpMVs
    mat = p.device_bytes
    alg = nspmv * (mat + 3 * v)
    spmv_ms = ph["spmv"][0]
    out = {"label": label, "n": nl, "nnz": p.nnz_local, "format": {
        "slices": p.slices, "pattern_slices": p.pattern_slices,
        "uniform_slices": p.uniform_slices, "cdia_classes": p.cdia_classes,
        "bytes": mat, "bytes_per_nnz": mat / p.nnz_local},
        "outer": rep.outer_iters, "t_solve_ms": rep.t_solve_ms, "wall_s": wall,
        "spmv_launch_family_ms": spmv_ms, "spmv_count": nspmv,
        "spmv_ms_each": spmv_ms / nspmv,
        "spmv_GBps_stored": alg / (spmv_ms / 1e3) / 1e9,
        "spmv_GBps_csr12": nspmv * (12 * p.nnz_local + 16 * nl) / (spmv_ms / 1e3) / 1e9,
        "phases_ms": {k: round(t[0], 2) for k, t in ph.items()}}
    print(json.dumps(out), flush=True)
    return out


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 128
    window = int(sys.argv[sys.argv.index("--window") + 1]) if "--window" in sys.argv else 4096
    import paper_2603_09790_b200 as cs
    ctx = cs.Context(0)
    cs.set_default_context(ctx)
    g = cs.DeviceProblem.generate("poisson27", n, n, n).set_precond("jacobi")
    a = g.to_csr()
    measure(cs, ctx, g, 8, f"27-pt {n}^3 natural order (generated: CDIA / box kernel)")
    g.close()
    nat = cs.DeviceProblem.from_csr(a).set_precond("jacobi")
    measure(cs, ctx, nat, 8, f"27-pt {n}^3 natural order, uploaded CSR")
    nat.close()
    rp, col, val = permuted(a, window)
    q = cs.DeviceProblem.from_csr(cs.CsrMatrix(a.n, rp, col, val)).set_precond("jacobi")
    measure(cs, ctx, q, 8, f"27-pt {n}^3 rows shuffled in windows of {window} (irregular)")
    q.close()


if __name__ == "__main__":
    main()
