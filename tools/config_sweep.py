"""BASELINE.json configs 2-5 as measurement sweeps (one JSON line per run).

    python tools/config_sweep.py --config 3 [--n 512] [--svals 4,8,12]
    python tools/config_sweep.py --config 4 [--n 384] [--nu 1,2,3,4]
    torchrun --nproc-per-node N tools/config_sweep.py --config 5 [--stencil 7,27]

config 2: 27-pt 256^3, s=8 single GPU, s-step PCG vs classical PCG
config 3: 27-pt 512^3 (strong scaling over the ranks this runs on), s sweep
config 4: anisotropic 7-point diffusion (1:1:100) 384^3, s=8, FGS sweeps nu sweep:
          outer counts, delta_alpha / delta_beta maxima, breakdowns (stability study)
config 5: weak scaling, 256^3 per GPU (z-stacked), 7- and 27-point: solve time and
          reductions per second, s-step PCG vs classical PCG

Timing: CUDA events on the solve stream (report t_solve_ms / t_lanczos_ms), max over
ranks. Every solve is device-resident (device-generated operator, b = 1, x0 = 0).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True, choices=[2, 3, 4, 5])
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--svals", default="", help="comma-separated s values")
    ap.add_argument("--nu", default="")
    ap.add_argument("--stencil", default="27")
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--max-outer", type=int, default=20000)
    ap.add_argument("--no-pcg", action="store_true")
    a = ap.parse_args()
    import torch
    rank, world, local = (int(os.environ.get(k, d)) for k, d in
                          (("RANK", 0), ("WORLD_SIZE", 1), ("LOCAL_RANK", 0)))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2603_09790_b200 as cs
    ctx = cs.Context(local)
    cs.set_default_context(ctx)
    if world > 1:
        obj = [cs.Context.unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(obj, src=0)
        ctx.comm_init(world, rank, obj[0])
    dev = torch.device("cuda", local)

    runs = []  # (kind, nx, ny, nz, coef, s, nu)
    if a.config == 2:
        n = a.n or 256
        runs = [("poisson27", n, n, n, None, int(s), 30) for s in (a.svals or "8").split(",")]
    elif a.config == 3:
        n = a.n or 512
        runs = [("poisson27", n, n, n, None, int(s), 30) for s in (a.svals or "4,8,12").split(",")]
    elif a.config == 4:
        n = a.n or 384
        runs = [("aniso7", n, n, n, (1.0, 1.0, 100.0), int(a.svals or 8), int(nu))
                for nu in (a.nu or "1,2,3,4").split(",")]
    else:
        n = a.n or 256
        runs = [("poisson27" if st == "27" else "poisson7", n, n, n * world, None,
                 int(a.svals or 8), 30) for st in a.stencil.split(",")]

    prob_key, prob = None, None
    for kind, nx, ny, nz, coef, s, nu in runs:
        key = (kind, nx, ny, nz, coef)
        if key != prob_key:
            if prob is not None:
                prob.close()
            prob = cs.DeviceProblem.generate(kind, nx, ny, nz, coef or (1.0, 1.0, 1.0),
                                             ctx=ctx).set_precond("jacobi")
            prob_key = key
        nl = prob.n_local
        b = torch.ones(nl, dtype=torch.float64, device=dev)
        x0 = torch.zeros(nl, dtype=torch.float64, device=dev)
        x = torch.empty(nl, dtype=torch.float64, device=dev)
        cfg = cs.SolverConfig(s=s, tol=a.tol, max_outer=a.max_outer, fgs=cs.FgsConfig(nu=nu))
        try:
            prob.pcg_s_solve_device(b.data_ptr(), x0.data_ptr(), x.data_ptr(), cfg)  # warm-up
            rep = prob.pcg_s_solve_device(b.data_ptr(), x0.data_ptr(), x.data_ptr(), cfg)
            err = None
        except cs.Error as e:  # breakdowns are results of the stability study
            rep, err = None, f"{type(e).__name__}: {e}"
        line = {"config": a.config, "workload": f"{kind} {nx}x{ny}x{nz}", "coef": coef,
                "s": s, "nu": nu, "n_gpus": world, "n_global": prob.n_global,
                "halo": prob.halo_mode if world > 1 else "none"}
        if rep is not None:
            t = ctx.allreduce_max(rep.t_solve_ms)
            tl = ctx.allreduce_max(rep.t_lanczos_ms)
            line.update({
                "converged": rep.converged, "outer_iters": rep.outer_iters,
                "final_rel_residual": float(rep.rel_residual[-1]),
                # t_solve excludes the spectrum estimate; the solve time is both
                "t_solve_ms": t, "t_lanczos_ms": tl, "t_total_ms": t + tl,
                "t_outer_ms": t / max(rep.outer_iters, 1),
                "gdof_s": prob.n_global / ((t + tl) / 1e3) / 1e9,
                "allreduces": rep.device_allreduces,
                "reductions_per_s": rep.device_allreduces / ((t + tl) / 1e3),
                "max_delta_alpha": float(max(rep.delta_alpha)) if len(rep.delta_alpha) else None,
                "max_delta_beta": float(max(rep.delta_beta)) if len(rep.delta_beta) else None,
                "lambda": [rep.spectrum_used.lambda_min, rep.spectrum_used.lambda_max]})
        else:
            line["error"] = err
        if not a.no_pcg and a.config in (2, 3, 5) and s == int((a.svals or "8").split(",")[0]):
            rp = prob.pcg_solve_device(b.data_ptr(), x0.data_ptr(), x.data_ptr(), tol=a.tol,
                                       max_iter=200000)
            tp = ctx.allreduce_max(rp.t_solve_ms)
            line["pcg"] = {"iters": rp.outer_iters, "t_solve_ms": tp,
                           "gdof_s": prob.n_global / (tp / 1e3) / 1e9,
                           "reductions_per_s": 2 * rp.outer_iters / (tp / 1e3)}
        if rank == 0:
            print(json.dumps(line), flush=True)
    prob.close()
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
