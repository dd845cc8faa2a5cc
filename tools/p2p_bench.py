"""Halo-transport micro-benchmarks under torchrun (one rank per GPU):

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/p2p_bench.py [--n 256]

Per rank: the fast MPK step on the slab without any halo (mpk_fast), the
peer-memory z_0 push kernel alone (p2p_push) and one MPK step through the
peer-memory halo (p2p_mpk: interior + release, wait + boundary)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--reps", type=int, default=50)
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    rank, world, local = (int(os.environ[k]) for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    import paper_2603_09790_b200 as cs
    ctx = cs.Context(local)
    cs.set_default_context(ctx)
    obj = [cs.Context.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx.comm_init(world, rank, obj[0])
    p = cs.DeviceProblem.generate("poisson27", a.n, a.n, a.n, ctx=ctx).set_precond("jacobi")
    p.pcg_s_solve(cfg=cs.SolverConfig(s=8, tol=1e-8, max_outer=2))
    res = {"rank": rank, "halo": p.halo_mode, "n_local": p.n_local}
    for k in ("mpk_fast", "p2p_push", "p2p_mpk", "p2p_mpk"):
        dist.barrier()
        res[k] = round(p.bench_spmv(k, a.reps) * 1e3, 2)  # us
    if os.environ.get("CS_TIMING_TRACE"):
        for k in ("mpk_fast", "plain"):
            dist.barrier()
            ctx.reset_timing()
            ctx.set_timing(True)
            p.bench_spmv(k, 1)
            ctx.set_timing(False)
            ctx.timing()
            print(f"rank {rank} traced {k}", file=sys.stderr, flush=True)
    out = [None] * world
    dist.all_gather_object(out, res)
    if rank == 0:
        print("P2P " + json.dumps(out), flush=True)
    p.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
