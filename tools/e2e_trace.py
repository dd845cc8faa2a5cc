import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_09790_b200 as cs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
p = cs.DeviceProblem.generate("poisson27", n, n, n).set_precond("jacobi")
a = p.to_csr()
def pinned(arr):
    t = torch.empty(arr.size, dtype={np.int64: torch.int64, np.float64: torch.float64}[arr.dtype.type], pin_memory=True)
    t.numpy()[:] = arr
    return t
keep = [pinned(a.row_offsets), pinned(a.col_indices), pinned(a.values)]
ah = cs.CsrMatrix(a.n, keep[0].numpy(), keep[1].numpy(), keep[2].numpy())
b, x0 = pinned(np.ones(a.n)), pinned(np.zeros(a.n))
cfg = cs.SolverConfig(s=8, tol=1e-8, max_outer=50000)
m = cs.JacobiPreconditioner(ah)
for i in range(3):
    t0 = time.perf_counter()
    r = cs.pcg_s_solve(ah, b.numpy(), x0.numpy(), m, cfg)
    print(f"e2e {time.perf_counter()-t0:.3f} s outer {r.report.outer_iters} t_solve {r.report.t_solve_ms:.0f} t_lz {r.report.t_lanczos_ms:.0f}", flush=True)
# raw pinned H2D bandwidth of the value array, for comparison with the upload phase
d = torch.empty(keep[2].numel(), dtype=torch.float64, device="cuda")
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    d.copy_(keep[2], non_blocking=True); torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"pinned h2d {keep[2].numel()*8/1e9:.2f} GB {dt*1e3:.1f} ms {keep[2].numel()*8/dt/1e9:.1f} GB/s", flush=True)
