"""World-size-2 CPU (gloo) checks of the N > 1 host logic: every rank builds its own slab
(decomposePar analogue), the 128-byte unique-id broadcast used to bootstrap NCCL, the halo pairing
convention across real processes (reading Z22), and the bench's max-over-ranks timing.  A
distributed Jacobi-PCG driven by the oracle's SpMV + gloo point-to-point/allreduce must reproduce
the single-domain oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import meshgen
import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _halo(parts, g, xs_local, world):
    """Exchange operand values at interface cells with gloo send/recv (pairing by list order)."""
    me = parts[g]
    reqs, recv = [], []
    for itf in me.interfaces:
        buf = torch.from_numpy(np.ascontiguousarray(xs_local[itf.faceCells]))
        reqs.append(dist.isend(buf, dst=itf.neighbRank))
        rb = torch.empty(len(itf.faceCells), dtype=torch.float64)
        reqs.append(dist.irecv(rb, src=itf.neighbRank))
        recv.append(rb)
    for r in reqs:
        r.wait()
    return [r.numpy() for r in recv]


def _amul(parts, g, x, world):
    y = oracle.amul(parts[g], x)
    for itf, xn in zip(parts[g].interfaces, _halo(parts, g, x, world)):
        oracle.iface_update(y, itf.faceCells, itf.coeffs, xn)
    return y


def _gsum(v):
    t = torch.tensor(v, dtype=torch.float64)
    dist.all_reduce(t)
    return t.numpy()


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # unique-id bootstrap as bench.py / dist_worker.py do it
        uid = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        assert uid[0] == bytes(range(128))
        g = meshgen.hex_laplacian(10, 9, 12, conductance_sigma=0.5, seed=4, dirichlet=dict(x0=1.0))
        parts = meshgen.slab_partition(g, world)
        bnd = meshgen.slab_bounds(g.nCells, world)
        lo, hi = int(bnd[rank]), int(bnd[rank + 1])
        # distributed SpMV
        xg = np.random.default_rng(2).uniform(-1, 1, g.nCells)
        y = _amul(parts, rank, xg[lo:hi].copy(), world)
        # distributed Jacobi-PCG (SURVEY §8(c) c2 order, 2 reductions per iteration)
        b = g.b[lo:hi]
        rD = 1.0 / parts[rank].diag
        x = np.zeros(hi - lo)
        r = b - _amul(parts, rank, x, world)
        nb = np.sqrt(_gsum([b @ b])[0])
        p = np.zeros_like(x)
        rho_old = None
        it = 0
        for k in range(1000):
            z = rD * r
            rho = _gsum([z @ r])[0]
            p = z if k == 0 else z + (rho / rho_old) * p
            qv = _amul(parts, rank, p, world)
            alpha = rho / _gsum([p @ qv])[0]
            x = x + alpha * p
            r = r - alpha * qv
            it = k + 1
            if np.sqrt(_gsum([r @ r])[0]) / nb < 1e-10:
                break
            rho_old = rho
        # max-over-ranks timing reduction as in bench.py
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out = [None] * world
        dist.all_gather_object(out, (y, x, it, float(t.item())))
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_two_ranks(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = meshgen.hex_laplacian(10, 9, 12, conductance_sigma=0.5, seed=4, dirichlet=dict(x0=1.0))
    xg = np.random.default_rng(2).uniform(-1, 1, g.nCells)
    yo = oracle.amul(g, xg)
    y = np.concatenate([o[0] for o in out])
    assert np.linalg.norm(y - yo) <= 1e-12 * np.linalg.norm(yo)
    st, xo, oit, ores = oracle.pcg(g, g.b, tol=1e-10, maxIter=1000)
    x = np.concatenate([o[1] for o in out])
    assert {o[2] for o in out} == {oit}
    assert np.linalg.norm(x - xo) <= 1e-9 * np.linalg.norm(xo)
    assert all(o[3] == float(world) for o in out)
