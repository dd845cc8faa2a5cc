"""Phase breakdown of the e2e solve (host CSR -> host x) with CS_TRACE=1.

    CS_TRACE=1 python tools/e2e_trace.py [N] [--pinned]

The reference-facing entry with the host int64 CSR in pageable numpy memory
(what a reference caller passes), or page-locked with --pinned; prints the
library's per-phase trace lines (stderr) and the raw host->device bandwidth of
one value array, pageable and pinned, for comparison with the upload phase.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_09790_b200 as cs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 256
pinned_mode = "--pinned" in sys.argv
p = cs.DeviceProblem.generate("poisson27", n, n, n).set_precond("jacobi")
a = p.to_csr()
p.close()


def pinned(arr):
    t = torch.empty(arr.size, dtype={np.int64: torch.int64, np.float64: torch.float64}[arr.dtype.type],
                    pin_memory=True)
    t.numpy()[:] = arr
    return t


if pinned_mode:
    keep = [pinned(a.row_offsets), pinned(a.col_indices), pinned(a.values)]
    a = cs.CsrMatrix(a.n, keep[0].numpy(), keep[1].numpy(), keep[2].numpy())
b, x0 = np.ones(a.n), np.zeros(a.n)
cfg = cs.SolverConfig(s=8, tol=1e-8, max_outer=50000)
m = cs.JacobiPreconditioner(a)
for i in range(5):
    t0 = time.perf_counter()
    r = cs.pcg_s_solve(a, b, x0, m, cfg)
    print(f"e2e {time.perf_counter()-t0:.3f} s outer {r.report.outer_iters} "
          f"t_solve {r.report.t_solve_ms:.0f} t_lz {r.report.t_lanczos_ms:.0f}", flush=True)
vals = a.values
d = torch.empty(vals.size, dtype=torch.float64, device="cuda")
for label, src in (("pageable", torch.from_numpy(vals)), ("pinned", pinned(vals[: 1 << 27]))):
    for i in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d[: src.numel()].copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"{label} h2d {src.numel()*8/1e9:.2f} GB {dt*1e3:.1f} ms "
              f"{src.numel()*8/dt/1e9:.1f} GB/s", flush=True)
