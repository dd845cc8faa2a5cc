#!/usr/bin/env python
"""bench.py -- headline benchmark of the B200 Chebyshev s-step PCG solve path.

Metric (BASELINE.json): s-step PCG solve time to 1e-8 as GDOF/s
(GDOF/s := n_global / t_solve / 1e9, one "step" = one complete pcg_s_solve:
Lanczos spectrum estimate + setup + outer iterations to ||r||/||b|| <= 1e-8).

Workload (BASELINE configs[1], weak-scaled for N>1 as configs[4]): 27-point
Poisson 256^3 per GPU (global 256 x 256 x 256N, z-stacked), s=8, FGS nu=30,
Jacobi, b=1, x0=0, fast (one-allreduce) algebra. Inputs are device-generated
and HBM-resident when the timed region starts (`value`); `e2e` repeats the
solve through the reference-facing C-ABI entry with HOST buffers (the host CSR
upload + SELL conversion + solve + x download inside the timed region).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Rank 0 prints ONE JSON line. `--impl reference` times the reference CPU
implementation (oracle/_ref, the unmodified reference library compiled from
/root/reference, or the C restatement when absent) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "s-step PCG solve time to 1e-8 (GDOF/s)"
UNIT = "GDOF/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--grid", type=int, default=512,
                    help="grid edge (default 512: BASELINE configs[2], the north-star 27-pt 512^3)")
    ap.add_argument("--stencil", type=int, default=27, choices=[7, 27])
    ap.add_argument("--s", type=int, default=8)
    ap.add_argument("--nu", type=int, default=30)
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--mode", default="fast", choices=["fast", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the n^3 grid split into z-slabs over N GPUs (default); "
                         "weak: n^3 per GPU, global n x n x nN")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-pcg", action="store_true")
    ap.add_argument("--variant", type=int, default=0, help="CS_VAR_* bits (A/B runs)")
    return ap.parse_args()


# ------------------------------------------------------------------------------ helpers

def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


class Clocks:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        rows = []
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) >= 9:
                rows.append(p)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        loaded = [v for v in sm if v > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


def nnz_of(stencil, nx, ny, nz):
    f = lambda m: 3 * m - 2 if m > 1 else 1  # noqa: E731
    if stencil == 27:
        return f(nx) * f(ny) * f(nz)
    n = nx * ny * nz
    return n + 2 * ((nx - 1) * ny * nz + nx * (ny - 1) * nz + nx * ny * (nz - 1))


def spmv_alg_bytes(mat_bytes, n, s, outer, lanczos_steps, mode="fast", jacobi=True,
                   diag_stream=True, pz=False, tr=False, mat_fast=None, rz=False):
    """Algorithmic bytes of every SpMV-phase kernel of one solve:
    the matrix in the format actually stored (SELL-32P: FP64 value slots +
    per-slice column/pattern/meta bytes; CDIA: 32-bit participation words) read
    once, x read once, each output written once, plus the epilogue vectors of
    each MPK step. mat_fast: the matrix bytes of the fast kinds (separable box
    SpMV on planar classes: no participation words, 0), default mat_bytes.
    tr: the true-residual schedule's r = b - A x, z_0 = M^-1 r once per outer."""
    mf = mat_bytes if mat_fast is None else mat_fast
    v = 8 * n
    b_spmv = mat_bytes + 2 * v                       # y = A x
    b_resid = mat_bytes + 3 * v                      # r = b - A x
    b_dot = mf + 2 * v                               # Lanczos t = A v (+ v.t)
    j = v if jacobi and diag_stream else 0          # D^-1 read by the epilogue
    if mode == "fast":                               # z_q = 2a D^-1 p_q - 2s z_{q-1} - z_{q-2}
        b_first = mf + 3 * v + j                     # x, p, z (+ D^-1)
        b_mid = mf + 4 * v + j                       # x, p, z_{q-2}, z (+ D^-1)
    else:                                            # reference zp recurrence (+ D^-1 vector)
        b_first = mat_bytes + 2 * v + v + j + (v if jacobi else 0) + v
        b_mid = mat_bytes + 2 * v + 2 * v + j + (v if jacobi else 0) + v
    b_last = b_spmv
    per_mpk = b_last if s == 1 else b_first + (s - 2) * b_mid + b_last
    setup_mpk = per_mpk  # the setup MPK always stores P (it becomes AQ_1)
    if pz and mode == "fast":  # no p_q written; the last step writes z_s (a mid-type step)
        per_mpk = (b_first - v) if s == 1 else (b_first - v) + (s - 1) * (b_mid - v)
    if tr and mode == "fast":  # x, b read; r (unless formed from z_0 by the pack), z_0 written
        per_mpk += mf + (3 if rz else 4) * v + j
    # setup MPK + one (speculative) MPK per outer iteration (fast algebra)
    return b_resid + lanczos_steps * b_dot + outer * per_mpk + setup_mpk, b_spmv


def update_vectors(s, pz, tr, diag_stream):
    """Vectors the fast update pass moves per row. Recursive
    residual: Q, Z, AQ, P (PZ: z_s, + D^-1 unless uniform), x, r read; Q, AQ,
    x, r, z_0 written. True residual: Q, Z, x read; Q, x written."""
    if tr:
        return 3 * s + 2
    return (5 if pz else 6) * s + (6 if diag_stream else 5)


def outer_bytes_format(mat_bytes, n, s, diag_stream=True, pz=False, tr=False, mat_fast=None,
                       rz=False):
    """Per-outer algorithmic bytes of the fast schedule in the stored format:
    s SpMV/MPK steps + packed reduction 8n(3s+1) + update pass 8n(6s+6).
    PZ schedule (P derived from Z): MPK steps write no p (the last writes z_s),
    pack 8n(2s+2), update 8n(5s+6). True residual: update 8n(3s+2) + one
    residual SpMV (x, b read; r, z_0 written)."""
    mf = mat_bytes if mat_fast is None else mat_fast
    v = 8 * n
    j = v if diag_stream else 0
    if pz:
        mpk = (mf + 2 * v + j) + (s - 1) * (mf + 3 * v + j)
        if tr:
            mpk += mf + (3 if rz else 4) * v + j
        return mpk + v * (2 * s + (1 if rz else 2)) + v * update_vectors(s, pz, tr, diag_stream)
    mpk = (mf + 3 * v + j) + (s - 2) * (mf + 4 * v + j) + (mat_bytes + 2 * v) \
        if s > 1 else mat_bytes + 2 * v
    return mpk + v * (3 * s + 1) + v * update_vectors(s, pz, False, diag_stream)


def outer_bytes(nnz, n, s):
    """B_outer(s) = s*B_spmv + 8n(14s+3) (Jacobi, 12 B/nnz CSR/SELL)."""
    return s * (12 * nnz + 16 * n) + 8 * n * (14 * s + 3)


# ------------------------------------------------------------------------------ CPU baseline

def golden_run(stencil, n, s, nu, world):
    """The reference's outer count and spectrum for this workload: the compiled
    reference (ref_probe) where it could run here, else the GPU's reference-
    algebra mode (the reference's operation order; bitwise equal to it wherever
    both ran), recorded in tests/golden/outer_counts.json with its source."""
    try:
        with open(os.path.join(ROOT, "tests", "golden", "outer_counts.json")) as f:
            table = json.load(f)
        key = f"p{stencil}_{n}x{n}x{n * world}_s{s}_nu{nu}_jacobi_1e-08"
        return table.get(key)
    except (OSError, ValueError):
        return None


def cpu_sample(args, lam, world=1, lanczos=True):
    """Bounded CPU sample of the same workload on one host core: the reference
    on a grid x grid x nzs slab of the same operator with the same spectrum.
    Per-outer time = t(max_outer=2) - t(max_outer=1) of pcg_s_solve; the
    Lanczos estimate (40 steps, the solve's own first phase) timed once on the
    same slab. Both are linear in n and are scaled to the full grid."""
    from oracle import oracle as orc
    kind = "ref" if orc.available("ref") else "port"
    o = orc.Oracle(kind)
    try:
        os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
    except (AttributeError, OSError):
        pass
    nxy = args.grid
    nzs = max(2, (1 << 21) // (nxy * nxy))  # ~2M rows: 8 planes at 512^2, 32 at 256^2
    if args.stencil == 27:
        a = o.poisson27(nxy, nxy, nzs)
    else:
        a = orc.Oracle("port").stencil7(nxy, nxy, nzs)
    scale = nxy * world / nzs if args.scaling == "weak" else nxy / nzs
    t = []
    for mo in (1, 2):
        t0 = time.perf_counter()
        o.pcg_s_solve(a, s=args.s, nu=args.nu, tol=args.tol, max_outer=mo, spectrum=lam,
                      precond=1)
        t.append(time.perf_counter() - t0)
    per_outer = max(t[1] - t[0], 1e-9) * scale
    t_lz = 0.0
    if lanczos:
        t0 = time.perf_counter()
        o.estimate_interval(a, 1, 40, 1234)
        t_lz = (time.perf_counter() - t0) * scale
    return {"kind": "reference" if kind == "ref" else "port", "cores": 1,
            "per_outer_s": per_outer, "lanczos_s": t_lz,
            "sample": (f"reference pcg_s_solve on a {nxy}x{nxy}x{nzs} slab of the same operator, "
                       f"same s/nu/spectrum: t(max_outer=2)-t(max_outer=1) = {t[1]-t[0]:.3f} s; "
                       f"Lanczos (40 steps) on the slab {t_lz / scale:.3f} s; both scaled "
                       f"x{scale:g} to the full grid; 1 of {os.cpu_count()} host cores (the "
                       "reference is single-threaded)")}


# ------------------------------------------------------------------------------ reference arm

def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    n = args.grid
    wz = world if args.scaling == "weak" else 1
    n_global = n * n * n * wz
    g = golden_run(args.stencil, n, args.s, args.nu, wz)
    if g:
        outer, lam, src = g["outer_iters"], (g["lambda_min"], g["lambda_max"]), g["source"]
    else:  # no recorded run for this grid: 27-pt Jacobi interval of 128^3
        outer, lam, src = 1000, (0.0023051621745818554, 1.5204622252319928), "assumed"
    vals = []
    smp = cpu_sample(args, lam, wz, lanczos=True)
    t_lz = smp["lanczos_s"]
    for i in range(args.warmup + args.steps):
        if i > 0:
            smp = cpu_sample(args, lam, wz, lanczos=False)
        if i >= args.warmup:
            vals.append(n_global / (t_lz + outer * smp["per_outer_s"]) / 1e9)
    v = statistics.median(vals)
    t_step = n_global / v / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (27-point Poisson, b=1, x0=0)",
            "config": {"workload": f"{args.stencil}-pt Poisson {n}x{n}x{n*wz}, s={args.s}, "
                       f"nu={args.nu}, Jacobi, tol {args.tol:g}",
                       "outer_iters": outer, "outer_iters_source": src,
                       "lambda": list(lam), "extrapolated": True,
                       "timing": "each step = one bounded slab sample (one host core); solve time "
                                 "= Lanczos + outer_iters x per-outer, scaled to the full grid"},
            "ms_per_step": t_step * 1e3,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": smp["kind"],
                             "sample": smp["sample"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------ our arm

def run_ours(args):
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2603_09790_b200 as cs

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    ctx = cs.Context(local)
    cs.set_default_context(ctx)
    if world > 1:
        obj = [cs.Context.unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(obj, src=0)
        ctx.comm_init(world, rank, obj[0])
    n = args.grid
    nz = n * world if args.scaling == "weak" else n
    kind = "poisson27" if args.stencil == 27 else "poisson7"
    prob = cs.DeviceProblem.generate(kind, n, n, nz, ctx=ctx).set_precond("jacobi")
    nl, ng = prob.n_local, prob.n_global
    dev = torch.device("cuda", local)
    b = torch.ones(nl, dtype=torch.float64, device=dev)
    x0 = torch.zeros(nl, dtype=torch.float64, device=dev)
    x = torch.empty(nl, dtype=torch.float64, device=dev)
    cfg = cs.SolverConfig(s=args.s, tol=args.tol, max_outer=50000, fgs=cs.FgsConfig(nu=args.nu),
                          mode=args.mode, variant=args.variant)
    torch.cuda.synchronize()

    def step():
        return prob.pcg_s_solve_device(b.data_ptr(), x0.data_ptr(), x.data_ptr(), cfg)

    for _ in range(args.warmup):
        rep = step()
    ext = torch.cuda.ExternalStream(ctx.stream(), device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = Clocks(local)
    barrier()
    # (1) the headline: K solves, no per-launch instrumentation
    l0 = ctx.launches()
    clocks.start()
    e0.record(ext)
    reps = [step() for _ in range(args.steps)]
    e1.record(ext)
    e1.synchronize()
    clk = clocks.stop()
    launches = ctx.launches() - l0
    t_ms = e0.elapsed_time(e1)
    t_max = ctx.allreduce_max(t_ms)
    barrier()
    # (2) one more solve with CUDA events around every launch: per-phase kernel
    # times for the roofline (instrumentation overhead reported)
    ctx.reset_timing()
    ctx.set_timing(True)
    e0.record(ext)
    reps_t = [step()]  # one instrumented solve: the per-phase split, not the headline
    e1.record(ext)
    e1.synchronize()
    ctx.set_timing(False)
    t_inst = e0.elapsed_time(e1)
    barrier()
    phases = ctx.timing()
    rep = reps[-1]
    value = ng * args.steps / (t_max / 1e3) / 1e9
    ms_step = t_max / args.steps

    # roofline per hot kernel family, the dominant one as "roofline"
    nnz_l = prob.nnz_local
    # matrix bytes one SpMV streams: CDIA reads only the 32-bit participation
    # words (its tables are kernel parameters); other formats their SELL arrays
    mat = 4 * 32 * prob.slices if prob.cdia_classes > 0 else prob.device_bytes
    dstream = not prob.cdia_uniform_diag  # CDIA: 1/a_ii is a kernel constant
    pz = bool(rep.schedule & 1)  # CS_SCHED_P_FROM_Z
    tr = bool(rep.schedule & 4)  # CS_SCHED_TRUE_R
    rz = bool(rep.schedule & 8)  # CS_SCHED_R_FROM_Z0
    # planar CDIA classes: the separable fast kinds read no participation words
    mat_f = 0 if (prob.cdia_planar and args.mode == "fast") else mat
    alg, b_spmv = spmv_alg_bytes(mat, nl, args.s, rep.outer_iters, cfg.lanczos_steps, args.mode,
                                 diag_stream=dstream, pz=pz, tr=tr, mat_fast=mat_f, rz=rz)
    v8 = 8 * nl
    outers_t = sum(r.outer_iters for r in reps_t)
    upd_vec = update_vectors(args.s, pz, tr, dstream)
    alg_phase = {
        "spmv": sum(spmv_alg_bytes(mat, nl, args.s, r.outer_iters, cfg.lanczos_steps,
                                   args.mode, diag_stream=dstream, pz=pz, tr=tr,
                                   mat_fast=mat_f, rz=rz)[0] for r in reps_t),
        # recursive residual: Q, Z, AQ, P (PZ: Z + z_s instead of P), x, r (+ D^-1
        # unless uniform) read; Q, AQ, x, r, z_0 written. True residual: Q, Z, x
        # read; Q, x written
        "update": outers_t * v8 * upd_vec,
        # Q, Z, P, r read once (PZ: Q, Z, z_s, r); one launch per outer + the setup one
        "reduce": outers_t * v8 * ((2 * args.s + (1 if rz else 2)) if pz else (3 * args.s + 1))
        + len(reps_t) * v8 * (3 * args.s + 1),
    }
    names = {"spmv": ("sell_boxsep_kernel<kMpk*/kResidF> (planar 27-point class: separable plane "
                      "sums over bulk-copied plane stages, producer warp + mbarrier ring, fused "
                      "MPK / residual epilogue)" if prob.cdia_planar and args.mode == "fast" else
                      "sell_box_kernel<kMpk*> (plane-streaming FP64 SpMV over the 3x3x3 constant-"
                      "diagonal class: bulk-copied plane stages, fused MPK epilogue; gather "
                      "kernels for other classes)"),
             "update": ("update_tr_kernel<s,beta> (Q, x update pass; r from the residual SpMV)"
                        if tr else "update_kernel<s,beta,xr,z0> (Q, AQ, x, r, z_0 update pass)"),
             "reduce": "pack_kernel<s> (packed Gram/projection block, DMMA)"}
    peak, peak_src = measured_peak()
    trf = ncu_traffic() or {}
    kern = {}
    for ph, byts in alg_phase.items():
        ms = phases[ph][0]
        if ms <= 0:
            continue
        ach = byts / (ms / 1e3) / 1e9
        t = trf.get(ph) or {}
        kern[ph] = {"kernel": names[ph], "ms_per_solve": ms / len(reps_t),
                    "share_of_step": ms / t_inst if t_inst > 0 else None,
                    "achieved": ach, "frac": ach / peak,
                    "alg_bytes_per_solve": byts / len(reps_t),
                    "traffic": t.get("bytes_per_launch"),
                    "traffic_alg_per_launch": t.get("alg_bytes_per_launch")}
    dom = max(kern, key=lambda k: kern[k]["ms_per_solve"])
    d = kern[dom]
    roof = {"kernel": d["kernel"], "bound": "hbm", "achieved": d["achieved"], "peak": peak,
            "unit": "GB/s", "frac": d["frac"], "traffic": d["traffic"],
            "traffic_alg_per_launch": d["traffic_alg_per_launch"], "peak_source": peak_src,
            "share_of_step": d["share_of_step"],
            "measured": "CUDA events around every launch of one instrumented solve run right "
                        "after the timed region (instrumentation overhead %.1f%%)" %
                        (100 * (t_inst / len(reps_t) / (t_ms / args.steps) - 1) if t_ms > 0 else 0),
            "kernels": kern,
            "alg_bytes_per_spmv": b_spmv,
            "matrix_bytes": mat, "matrix_bytes_per_nnz": mat / nnz_l,
            "survey_B_spmv_12B_per_nnz": 12 * nnz_l + 16 * nl}
    # whole-solve bandwidth against B_outer
    solve_outer_ms = rep.t_solve_ms / max(rep.outer_iters, 1)
    b_out = outer_bytes_format(mat, nl, args.s, dstream, pz, tr, mat_f, rz)
    b_survey = outer_bytes(nnz_l, nl, args.s)
    solve_level = {"t_outer_ms": solve_outer_ms, "B_outer_GB": b_out / 1e9,
                   "achieved_GBps": b_out / (solve_outer_ms / 1e3) / 1e9,
                   "frac_of_peak": b_out / (solve_outer_ms / 1e3) / 1e9 / peak,
                   "survey_B_outer_GB_12B_per_nnz": b_survey / 1e9,
                   "survey_roofline_ms_at_peak": b_survey / peak / 1e6,
                   "t_lanczos_ms": rep.t_lanczos_ms, "t_solve_ms": rep.t_solve_ms}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (device-generated 27-point Poisson, b=1, x0=0)",
            "config": {"workload": f"{args.stencil}-pt Poisson global {n}x{n}x{nz} "
                       f"({'strong' if args.scaling == 'strong' else 'weak'} scaling, "
                       f"{nz // world} z-planes per GPU), s={args.s}, nu={args.nu}, Jacobi, "
                       f"tol {args.tol:g}, {args.mode} algebra",
                       "n_global": ng, "nnz_local": nnz_l, "outer_iters": rep.outer_iters,
                       "converged": rep.converged,
                       "final_rel_residual": float(rep.rel_residual[-1]),
                       "lambda": [rep.spectrum_used.lambda_min, rep.spectrum_used.lambda_max],
                       "allreduces_per_solve": rep.device_allreduces,
                       "l2": "inputs > L2 (matrix %.1f GB/GPU vs 126 MB L2); no flush" %
                             (prob.device_bytes / 1e9),
                       "parallelism": f"z-slab row partition x{world}",
                       "halo": prob.halo_mode,
                       "matrix_format": {"slices": prob.slices,
                                         "pattern_slices": prob.pattern_slices,
                                         "uniform_value_slices": prob.uniform_slices,
                                         "table_entries": prob.pattern_entries,
                                         "cdia_classes": prob.cdia_classes,
                                         "cdia_uniform_diag": bool(prob.cdia_uniform_diag),
                                         "bytes": prob.device_bytes}},
            "gpu_launches": launches,
            "roofline": roof,
            "solve_roofline": solve_level,
            "phases_ms": {k: round(v[0], 3) for k, v in phases.items()},
            "clocks": clk}

    # classical PCG on the same GPUs (configs[1] "vs classical PCG")
    if not args.no_pcg:
        rp = prob.pcg_solve_device(b.data_ptr(), x0.data_ptr(), x.data_ptr(), tol=args.tol,
                                   max_iter=100000)
        t_pcg = ctx.allreduce_max(rp.t_solve_ms)
        line["pcg"] = {"gdof_s": ng / (t_pcg / 1e3) / 1e9, "iters": rp.outer_iters,
                       "t_solve_ms": t_pcg, "allreduces_per_solve": 2 * rp.outer_iters,
                       "reductions_per_s_pcgs": rep.device_allreduces / (ms_step / 1e3),
                       "reductions_per_s_pcg": 2 * rp.outer_iters / (t_pcg / 1e3)}
    # e2e through the reference-facing C-ABI entry with host buffers (the N=1 CSR
    # path releases the device-resident problem first: HBM for the upload)
    del b, x0, x
    if not args.no_e2e:
        line["e2e"] = e2e(args, cs, ctx, prob, world, torch)
    if rank == 0 and world == 1 and not args.no_cpu:
        lam = (rep.spectrum_used.lambda_min, rep.spectrum_used.lambda_max)
        smp = cpu_sample(args, lam)
        g = golden_run(args.stencil, args.grid, args.s, args.nu, 1)
        outer, src = ((g["outer_iters"], g["source"]) if g else
                      (rep.outer_iters, "this GPU run (no recorded reference count)"))
        v = ng / (smp["lanczos_s"] + outer * smp["per_outer_s"]) / 1e9
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": smp["cores"],
                                "kind": smp["kind"], "extrapolated": True,
                                "sample": smp["sample"] + f"; solve = Lanczos + {outer} outer "
                                f"iterations ({src})"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    prob.close()
    barrier()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def host_mem_available():
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def e2e(args, cs, ctx, prob, world, torch):
    """The same solve through the reference-facing entry with HOST buffers in
    PAGEABLE memory (what a reference caller passes: std::vector / numpy), every
    host<->device byte inside the timed region.

    N=1 and the host can hold the reference's int64 CSR (+ headroom):
      cs_pcg_s_solve_csr = chebstep::pcg_s_solve(const CsrMatrix&, b, x0, M, cfg):
      streamed CSR upload overlapped with the SELL-32 fill, CDIA conversion,
      Jacobi setup, Lanczos, solve, x download.
    Otherwise (e.g. 27-pt 512^3: 58.8 GB of int64 CSR) the device-resident-
      problem overload cs_pcg_s_solve with host b / x0 -> host x."""
    import numpy as np
    nl, ng = prob.n_local, prob.n_global
    cfg = cs.SolverConfig(s=args.s, tol=args.tol, max_outer=50000, fgs=cs.FgsConfig(nu=args.nu),
                          mode=args.mode, variant=args.variant)
    nnz = prob.nnz_local
    csr_bytes = 8 * (nl + 1) + 16 * nnz
    avail = host_mem_available()
    use_csr = world == 1 and avail > 1.5 * csr_bytes + 32 * nl
    if use_csr:
        a = prob.to_csr()  # numpy (pageable) int64 CSR, the reference layout
        prob.close()       # its workspace + Lanczos basis (126 GB at 512^3) leave HBM
        torch.cuda.empty_cache()
        bh, x0h = np.ones(nl), np.zeros(nl)
        m = cs.JacobiPreconditioner(a)
        call = lambda: cs.pcg_s_solve(a, bh, x0h, m, cfg, ctx=ctx)  # noqa: E731
        h2d = csr_bytes + 16 * nl
        entry = ("cs_pcg_s_solve_csr: pageable host int64 CSR + b + x0 -> host x (streamed "
                 "upload, SELL/CDIA conversion, Jacobi, Lanczos, solve, download)")
    else:
        bh, x0h = np.ones(nl), np.zeros(nl)
        call = lambda: prob.pcg_s_solve(bh, x0h, cfg)  # noqa: E731
        h2d = 16 * nl
        entry = ("cs_pcg_s_solve: device-resident problem, pageable host b + x0 -> host x" +
                 (f" (host MemAvailable {avail / 1e9:.0f} GB cannot hold the {csr_bytes / 1e9:.1f} "
                  "GB int64 CSR)" if world == 1 else ""))
    call()  # warm-up
    ts = []
    res = None
    for _ in range(args.e2e_steps):
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        res = call()
        ts.append(ctx.allreduce_max(time.perf_counter() - t0))
    dt = statistics.median(ts)
    return {"value": ng / dt / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": 8 * nl, "steps": args.e2e_steps, "entry": entry,
            "ms_per_step": dt * 1e3, "ms_per_step_all": [round(t * 1e3, 1) for t in ts],
            "statistic": "median over steps, wall clock (host buffers), max over ranks",
            "outer_iters": res.report.outer_iters}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
