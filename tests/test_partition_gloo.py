"""CPU-only multi-process test of the N>1 host logic with the gloo backend:
world_size 2 and 3 ranks each take their z-slab of the 27-point operator
(cs_partition_rows), build the halo map (cs_halo_map_csr), exchange ghost
values with point-to-point gloo messages exactly as the GPU path exchanges
ghost planes, and run a distributed SpMV and a distributed dot product in the
reference row order. The result must be BITWISE the single-address-space
reference SpMV (row order is partition-invariant) and the global sum must
match to rounding."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, dims, out_q):
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2603_09790_b200 as cs
    from oracle.oracle import Oracle
    port_o = Oracle("port")
    nx, ny, nz = dims
    o = port_o.poisson27(nx, ny, nz)
    plane = nx * ny
    b, e = cs.partition_rows(o.n, plane, world, rank)
    rp = o.rowptr[b:e + 1] - o.rowptr[b]
    cg = o.col[o.rowptr[b]:o.rowptr[e]]
    vals = o.val[o.rowptr[b]:o.rowptr[e]]
    ghosts, cl = cs.halo_map_csr(b, e, rp, cg)
    nloc = e - b
    x_glob = np.random.default_rng(5).standard_normal(o.n)
    x = np.zeros(nloc + ghosts.size)
    x[:nloc] = x_glob[b:e]
    # halo exchange: my first plane -> rank-1 (its upper ghosts), my last -> rank+1
    lo_cnt = plane if b > 0 else 0
    reqs = []
    send_lo = torch.from_numpy(x[:plane].copy())
    send_hi = torch.from_numpy(x[nloc - plane:nloc].copy())
    recv_lo = torch.zeros(plane, dtype=torch.float64)
    recv_hi = torch.zeros(plane, dtype=torch.float64)
    if rank > 0:
        reqs += [dist.isend(send_lo, rank - 1), dist.irecv(recv_lo, rank - 1)]
    if rank < world - 1:
        reqs += [dist.isend(send_hi, rank + 1), dist.irecv(recv_hi, rank + 1)]
    for r in reqs:
        r.wait()
    if rank > 0:
        x[nloc:nloc + plane] = recv_lo.numpy()
    if rank < world - 1:
        x[nloc + lo_cnt:nloc + lo_cnt + plane] = recv_hi.numpy()
    # row-serial SpMV in stored order (csr.cpp:116-121)
    y = np.zeros(nloc)
    for i in range(nloc):
        acc = 0.0
        for k in range(rp[i], rp[i + 1]):
            acc = acc + vals[k] * x[cl[k]]
        y[i] = acc
    y_ref = port_o.spmv(o, x_glob)[b:e]
    ok_spmv = y.tobytes() == y_ref.tobytes()
    # distributed dot: local serial partial + allreduce
    part = torch.tensor([float(np.dot(y, x[:nloc]))], dtype=torch.float64)
    dist.all_reduce(part)
    glob = float(np.dot(port_o.spmv(o, x_glob), x_glob))
    ok_dot = abs(part.item() - glob) <= 1e-12 * abs(glob)
    spans = [None] * world
    dist.all_gather_object(spans, (b, e))
    out_q.put((rank, ok_spmv, ok_dot, spans, ghosts.tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,dims", [(2, (6, 5, 8)), (3, (4, 7, 9))])
def test_distributed_spmv_gloo(world, dims):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    res.sort()
    for rank, ok_spmv, ok_dot, spans, ghosts in res:
        assert ok_spmv, f"rank {rank}: distributed SpMV differs from the reference"
        assert ok_dot, f"rank {rank}: distributed dot differs"
    spans = res[0][3]
    n = dims[0] * dims[1] * dims[2]
    assert spans[0][0] == 0 and spans[-1][1] == n
    assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))


def _worker_mm(rank, world, port, path, out_q):
    """General-CSR path: Matrix Market file -> cs_partition_rows(plane=1) ->
    cs_halo_map_csr -> owner-grouped request/reply halo (the protocol of
    runtime.cu plan_general_halo: counts, then global row ids, then values)."""
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2603_09790_b200 as cs
    from oracle.oracle import Csr, Oracle
    a = cs.read_matrix_market(path, True)
    b, e = cs.partition_rows(a.n, 1, world, rank)
    rp = a.row_offsets[b:e + 1] - a.row_offsets[b]
    cg = a.col_indices[a.row_offsets[b]:a.row_offsets[e]]
    vals = a.values[a.row_offsets[b]:a.row_offsets[e]]
    ghosts, cl = cs.halo_map_csr(b, e, rp, cg)
    spans = [cs.partition_rows(a.n, 1, world, q) for q in range(world)]
    owner = np.searchsorted([s[1] for s in spans], ghosts, side="right")
    rcnt = np.bincount(owner, minlength=world).astype(np.int64)
    scnt = torch.zeros(world, dtype=torch.int64)
    for q in range(world):  # counts: all-to-all by point-to-point
        if q == rank:
            continue
        reqs = [dist.isend(torch.tensor([rcnt[q]]), q), dist.irecv(t := torch.zeros(1, dtype=torch.int64), q)]
        for r in reqs:
            r.wait()
        scnt[q] = t[0]
    roff = np.concatenate([[0], np.cumsum(rcnt)])
    want = {}
    for q in range(world):
        if q == rank:
            continue
        reqs, got = [], torch.zeros(int(scnt[q]), dtype=torch.int64)
        if rcnt[q]:
            reqs.append(dist.isend(torch.from_numpy(ghosts[roff[q]:roff[q + 1]].copy()), q))
        if scnt[q]:
            reqs.append(dist.irecv(got, q))
        for r in reqs:
            r.wait()
        want[q] = got.numpy() - b
    x_glob = np.random.default_rng(9).standard_normal(a.n)
    x = np.concatenate([x_glob[b:e], np.zeros(ghosts.size)])
    for q in range(world):
        if q == rank:
            continue
        reqs, buf = [], torch.zeros(int(rcnt[q]), dtype=torch.float64)
        if scnt[q]:
            reqs.append(dist.isend(torch.from_numpy(x[want[q]].copy()), q))
        if rcnt[q]:
            reqs.append(dist.irecv(buf, q))
        for r in reqs:
            r.wait()
        x[e - b + roff[q]:e - b + roff[q + 1]] = buf.numpy()
    nloc = e - b
    y = np.zeros(nloc)
    for i in range(nloc):
        acc = 0.0
        for k in range(rp[i], rp[i + 1]):
            acc = acc + vals[k] * x[cl[k]]
        y[i] = acc
    o = Csr(a.n, a.row_offsets, a.col_indices, a.values)
    ok = y.tobytes() == Oracle("port").spmv(o, x_glob)[b:e].tobytes()
    out_q.put((rank, ok, int(ghosts.size)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_general_csr_halo(world, tmp_path):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2603_09790_b200 as cs
    from oracle.oracle import Oracle
    from tools.mgpu_check import shuffled
    o = shuffled(Oracle("port").poisson27(12, 11, 10), seed=4)
    path = str(tmp_path / "g.mtx")
    cs.write_matrix_market(path, cs.CsrMatrix(o.n, o.rowptr, o.col, o.val))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_mm, args=(r, world, port, path, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(60)
    assert all(ok for _, ok, _ in res), res
    assert all(g > 0 for _, _, g in res), res
