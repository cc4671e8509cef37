"""Multi-process host logic of the z-slab partition on CPU (gloo, world size 2 and 3).

The GPU driver (gdp_dist.cu) is exercised bit-for-bit by the loopback tests; here the same
schedule is modelled with numpy on real processes: each rank owns planes [z0, z0+nzl),
exchanges one ghost plane with each neighbour before every red-black half-sweep (send first
plane down / last plane up, as comm_halo_parts does), colours cells by GLOBAL (x+y+z) parity,
and forms exact per-plane sums by a one-hot sum-allreduce.  The result must equal the
single-process sweep bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1310_0041_b200 as gdp

W = (1.0, 1.0, 0.1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _halfsweep(x, b, z0, nzg, color, lo, hi):
    """RB Gauss-Seidel half-sweep in correction form on a slab with ghost planes (float32)."""
    nz, ny, nx = x.shape
    f = np.float32
    xp = np.concatenate([lo[None] if lo is not None else x[:1], x, hi[None] if hi is not None else x[-1:]])
    zz, yy, xx = np.meshgrid(np.arange(nz) + z0, np.arange(ny), np.arange(nx), indexing="ij")
    mask = ((xx + yy + zz) & 1) == color
    c = xp[1:-1]
    s = np.zeros_like(c)
    D = np.zeros_like(c)

    def link(nb, have, w):
        nonlocal s, D
        s = s + np.where(have, f(w) * (c - nb), f(0))
        D = D + np.where(have, f(w), f(0))
    link(np.pad(c, ((0, 0), (0, 0), (1, 0)), mode="edge")[:, :, :-1], xx > 0, W[0])
    link(np.pad(c, ((0, 0), (0, 0), (0, 1)), mode="edge")[:, :, 1:], xx < nx - 1, W[0])
    link(np.pad(c, ((0, 0), (1, 0), (0, 0)), mode="edge")[:, :-1], yy > 0, W[1])
    link(np.pad(c, ((0, 0), (0, 1), (0, 0)), mode="edge")[:, 1:], yy < ny - 1, W[1])
    link(xp[:-2], zz > 0, W[2])
    link(xp[2:], zz < nzg - 1, W[2])
    r = b - s
    new = (c + r / np.where(D > 0, D, f(1))).astype(f)
    return np.where(mask, new, c).astype(f)


def _worker(rank, world, port, nz, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(1)
    ny, nx = 9, 11
    X = rng.random((nz, ny, nx)).astype(np.float32)
    B = (rng.random((nz, ny, nx)) - 0.5).astype(np.float32)
    z0, nzl = gdp.partition(nz, world)[rank]
    x = X[z0:z0 + nzl].copy()
    b = B[z0:z0 + nzl]
    for hs in range(6):
        lo = hi = None
        reqs = []
        lo_t = torch.zeros(ny, nx)
        hi_t = torch.zeros(ny, nx)
        if rank > 0:
            reqs.append(dist.isend(torch.from_numpy(x[0].copy()), rank - 1))
            reqs.append(dist.irecv(lo_t, rank - 1))
        if rank < world - 1:
            reqs.append(dist.isend(torch.from_numpy(x[-1].copy()), rank + 1))
            reqs.append(dist.irecv(hi_t, rank + 1))
        for r_ in reqs:
            r_.wait()
        if rank > 0:
            lo = lo_t.numpy()
        if rank < world - 1:
            hi = hi_t.numpy()
        x = _halfsweep(x, b, z0, nz, hs & 1, lo, hi)
    # exact per-plane sums: one non-zero contributor per element
    planes = torch.zeros(nz, dtype=torch.float64)
    planes[z0:z0 + nzl] = torch.from_numpy(x.astype(np.float64).sum(axis=(1, 2)))
    dist.all_reduce(planes)
    gathered = [torch.zeros(nz, ny, nx) for _ in range(world)] if rank == 0 else None
    full = torch.zeros(nz, ny, nx)
    full[z0:z0 + nzl] = torch.from_numpy(x)
    dist.all_reduce(full)
    if rank == 0:
        ref = X.copy()
        for hs in range(6):
            ref = _halfsweep(ref, B, 0, nz, hs & 1, None, None)
        q.put((np.array_equal(full.numpy(), ref),
               np.array_equal(planes.numpy(), ref.astype(np.float64).sum(axis=(1, 2)))))
    dist.destroy_process_group()
    del gathered


@pytest.mark.parametrize("world,nz", [(2, 8), (3, 10)])
def test_slab_halo_schedule_matches_single_process(world, nz):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nz, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    same_x, same_planes = q.get(timeout=5)
    assert same_x and same_planes


def test_partition_tiles_stack():
    for nz, w in ((128, 8), (33, 3), (5, 5), (12, 5)):
        p = gdp.partition(nz, w)
        assert p[0][0] == 0 and sum(n for _, n in p) == nz
        assert all(p[i][0] + p[i][1] == p[i + 1][0] for i in range(w - 1))
        assert max(n for _, n in p) - min(n for _, n in p) <= 1


def _uid_worker(rank, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    t = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        t = torch.frombuffer(bytearray(gdp.get_unique_id()), dtype=torch.uint8).clone()
    dist.broadcast(t, 0)
    q.put((rank, bytes(t.numpy())))
    dist.destroy_process_group()


def test_unique_id_broadcast_over_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_uid_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    a, b = q.get(timeout=5), q.get(timeout=5)
    assert a[1] == b[1] and len(a[1]) == 128 and any(a[1])
