"""Multi-GPU parity (needs >= 2 GPUs; skipped otherwise): runs
tools/mgpu_check.py under torchrun, one rank per GPU, z-slab partition with
the NVLink peer-memory halo (and the NCCL halo, bitwise the same) and one NCCL
allreduce per outer iteration."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.parametrize("stencil,n,nz,mm,variant", [("poisson27", 40, 48, False, 256),
                                                     ("poisson27", 40, 48, False, 128),
                                                     ("poisson7", 32, 40, False, 0),
                                                     ("poisson27", 24, 32, True, 0)])
def test_multi_gpu_parity(stencil, n, nz, mm, variant, tmp_path):
    """variant 256 / 128: the recursive / true-residual fast schedule (the true
    residual moves x's boundary planes by peer stores from the update pass and
    z_0's from the residual SpMV)."""
    ng = _gpus()
    if ng < 2:
        pytest.skip("needs >= 2 GPUs")
    world = ng  # every GPU of the box (2, 4 or 8 ranks)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + n + 7 * mm + variant % 7),
           os.path.join(ROOT, "tools", "mgpu_check.py"), "--grid", str(n), "--nz", str(nz),
           "--stencil", stencil, "--variant", str(variant)] + (["--mm"] if mm else [])
    env = dict(os.environ, MGPU_TMP=str(tmp_path))
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    line = [l for l in out.stdout.splitlines() if l.startswith("MGPU ")]
    assert line, out.stdout[-3000:] + out.stderr[-3000:]
    res = json.loads(line[0][5:])
    assert len(res) == world
    for r in res:
        assert r["assembly_bitwise"] and r["ghosts_ok"] and r["spmv_bitwise"], r
        if mm:
            assert r["n_ghost"] > 0, r
        assert r["outer_ok"], r
        assert r["transport_bitwise"], r
        assert r["fused_allreduce_x_rel"] <= 1e-8, r
        assert abs(r["fused_allreduce_outer"][0] - r["fused_allreduce_outer"][1]) <= 1, r
        assert r["halo_mode"] == ("nccl" if mm else "nvlink-p2p"), r
        # PZ schedules over the peer halo: the per-outer allreduce runs inside the
        # pack over peer memory (CS_SCHED_P2P_ALLREDUCE), off with CS_P2P_ALLREDUCE=0
        if not mm:
            assert bool(r["schedule"] & 16) and not r["schedule_nccl_allreduce"] & 16, r
        assert r["halo_mode_off"] == "nccl", r
        assert r["x_rel"] <= 1e-8, r
        assert abs(r["pcg_iters"][0] - r["pcg_iters"][1]) <= 1 and r["pcg_x_rel"] <= 1e-8, r
        assert r["lambda_rel"] < 1e-9, r
