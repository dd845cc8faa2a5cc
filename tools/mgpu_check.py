"""Multi-GPU parity driver (torchrun, one process per GPU), used by
tests/test_gpu_multi.py:

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/mgpu_check.py --grid 48

Each rank owns a z-slab of a global 27-point (or 7-point) grid generated on
its GPU. Checks, per rank, against the CPU oracle (test infrastructure):
  * partitioned assembly: local rows with global columns == the oracle's rows, bitwise;
  * ghost list == the neighbour planes;
  * distributed SpMV (NCCL halo exchange + SELL kernel) == oracle rows, bitwise;
  * distributed fast-mode PCG-S (one NCCL allreduce per outer iteration, halo
    planes by NVLink peer stores): outer count within +-1 of the oracle, x
    within 1e-8 relative, and bitwise equal to the same solve with the NCCL halo;
  * classical PCG on the same slabs.
Rank 0 prints one JSON line with every verdict.
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def shuffled(o, seed):
    """P A P^T for a permutation that shuffles rows inside windows of 4096 and
    swaps a few rows across the whole range: an irregular but partly local
    halo. Rows stay sorted by column (reference CsrMatrix invariant)."""
    from oracle.oracle import Csr
    rng = np.random.default_rng(seed)
    perm = np.arange(o.n)
    for s in range(0, o.n, 4096):
        rng.shuffle(perm[s:s + 4096])
    for _ in range(16):
        i, j = rng.integers(0, o.n, 2)
        perm[i], perm[j] = perm[j], perm[i]
    inv = np.empty_like(perm)
    inv[perm] = np.arange(o.n)
    lens = np.diff(o.rowptr)[perm]
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    col = np.empty_like(o.col)
    val = np.empty_like(o.val)
    for i in range(o.n):
        a0, a1 = o.rowptr[perm[i]], o.rowptr[perm[i] + 1]
        c = inv[o.col[a0:a1]]
        k = np.argsort(c, kind="stable")
        col[rp[i]:rp[i + 1]] = c[k]
        val[rp[i]:rp[i + 1]] = o.val[a0:a1][k]
    return Csr(o.n, rp, col, val)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=48)
    ap.add_argument("--nz", type=int, default=0)
    ap.add_argument("--s", type=int, default=4)
    ap.add_argument("--stencil", default="poisson27")
    ap.add_argument("--variant", type=int, default=0, help="CS_VAR_* bits of the fast solves")
    ap.add_argument("--mm", action="store_true",
                    help="general CSR path: a locally shuffled operator read from a Matrix "
                         "Market file (irregular, owner-grouped halo)")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    rank, world, local = (int(os.environ[k]) for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    import paper_2603_09790_b200 as cs
    from oracle.oracle import Oracle
    ctx = cs.Context(local)
    cs.set_default_context(ctx)
    obj = [cs.Context.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx.comm_init(world, rank, obj[0])
    n, nz = a.grid, a.nz or a.grid
    port = Oracle("port")
    o = port.poisson27(n, n, nz) if a.stencil == "poisson27" else port.stencil7(n, n, nz)
    if a.mm:
        o = shuffled(o, seed=7)
        path = os.path.join(os.environ.get("MGPU_TMP", "/tmp"), f"mgpu_{n}_{nz}_{a.stencil}.mtx")
        if rank == 0:
            cs.write_matrix_market(path, cs.CsrMatrix(o.n, o.rowptr, o.col, o.val))
        dist.barrier()
        p = cs.DeviceProblem.read_matrix_market(path, True, ctx=ctx).set_precond("jacobi")
    else:
        p = cs.DeviceProblem.generate(a.stencil, n, n, nz, ctx=ctx).set_precond("jacobi")
    b0, e0 = p.row_begin, p.row_begin + p.n_local
    res = {"rank": rank, "rows": [b0, e0], "n_ghost": p.n_ghost}
    loc = p.to_csr()
    rp = o.rowptr[b0:e0 + 1] - o.rowptr[b0]
    res["assembly_bitwise"] = bool(
        loc.row_offsets.tobytes() == rp.tobytes()
        and loc.col_indices.tobytes() == o.col[o.rowptr[b0]:o.rowptr[e0]].tobytes()
        and loc.values.tobytes() == o.val[o.rowptr[b0]:o.rowptr[e0]].tobytes())
    if a.mm:
        cols = o.col[o.rowptr[b0]:o.rowptr[e0]]
        want = np.unique(cols[(cols < b0) | (cols >= e0)]).tolist()
    else:
        plane = n * n
        want = (list(range(b0 - plane, b0)) if b0 > 0 else []) + \
            (list(range(e0, e0 + plane)) if e0 < o.n else [])
    res["ghosts_ok"] = p.ghosts().tolist() == want
    xg = np.random.default_rng(3).standard_normal(o.n)
    y = p.spmv(xg[b0:e0])
    res["spmv_bitwise"] = bool(y.tobytes() == port.spmv(o, xg)[b0:e0].tobytes())
    # distributed fast-mode solve vs the oracle
    x_o, r_o = port.pcg_s_solve(o, s=a.s, tol=1e-8, max_outer=5000)
    sol = p.pcg_s_solve(cfg=cs.SolverConfig(s=a.s, tol=1e-8, max_outer=5000, variant=a.variant))
    parts = [None] * world
    dist.all_gather_object(parts, (b0, sol.x))
    x = np.concatenate([v for _, v in sorted(parts, key=lambda t: t[0])])
    res["outer"] = [sol.report.outer_iters, r_o.outer_iters]
    res["outer_ok"] = abs(sol.report.outer_iters - r_o.outer_iters) <= 1
    res["x_rel"] = float(np.linalg.norm(x - x_o) / np.linalg.norm(x_o))
    res["allreduces"] = sol.report.device_allreduces
    res["halo_mode"] = p.halo_mode
    res["schedule"] = sol.report.schedule
    # the same solve with the peer halo but the NCCL allreduce, and with the NCCL
    # halo: the halo transport must not change a bit; the fused peer-memory
    # allreduce (rank-order sums) is another rounding of the same block -> x to 1e-8
    spec = sol.report.spectrum_used
    os.environ["CS_P2P_ALLREDUCE"] = "0"
    sol_a = p.pcg_s_solve(cfg=cs.SolverConfig(s=a.s, tol=1e-8, max_outer=5000, spectrum=spec,
                                              variant=a.variant))
    res["schedule_nccl_allreduce"] = sol_a.report.schedule
    os.environ["CS_P2P_HALO"] = "0"
    sol_n = p.pcg_s_solve(cfg=cs.SolverConfig(s=a.s, tol=1e-8, max_outer=5000, spectrum=spec,
                                              variant=a.variant))
    os.environ.pop("CS_P2P_HALO")
    os.environ.pop("CS_P2P_ALLREDUCE")
    res["halo_mode_off"] = p.halo_mode
    res["transport_bitwise"] = bool(sol_n.x.tobytes() == sol_a.x.tobytes()
                                    and sol_n.report.outer_iters == sol_a.report.outer_iters)
    res["fused_allreduce_x_rel"] = float(np.linalg.norm(sol.x - sol_a.x) /
                                         max(np.linalg.norm(sol_a.x), 1e-300))
    res["fused_allreduce_outer"] = [sol.report.outer_iters, sol_a.report.outer_iters]
    res["lambda_rel"] = abs(sol.report.spectrum_used.lambda_min / r_o.lambda_min - 1)
    pc = p.pcg_solve(tol=1e-8, max_iter=5000)
    xp, rpcg = port.pcg_solve(o, tol=1e-8, max_iter=5000)
    parts = [None] * world
    dist.all_gather_object(parts, (b0, pc.x))
    x2 = np.concatenate([v for _, v in sorted(parts, key=lambda t: t[0])])
    res["pcg_iters"] = [pc.report.outer_iters, rpcg.outer_iters]
    res["pcg_x_rel"] = float(np.linalg.norm(x2 - xp) / np.linalg.norm(xp))
    allres = [None] * world
    dist.all_gather_object(allres, res)
    if rank == 0:
        print("MGPU " + json.dumps(allres), flush=True)
    p.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
