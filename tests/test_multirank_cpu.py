"""Multi-rank host logic on CPU (gloo, world_size 2 and 3).

The library's row-slab decomposition (sw2d_partition) and per-step halo plan
(sw2d_halo_plan, the plan its NCCL and virtual-rank exchanges execute) are
driven here by real torch.distributed processes over gloo: every rank steps
its slab plus the 2 halo rows on each side with the CPU oracle, exchanges the
halo rows the plan names with its neighbours, and the gathered owned rows must
equal the single-grid oracle bitwise (the dependency cone of one step is 2
rows).  A wrong row, direction or count in the plan
breaks bitwise equality within a few steps.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import sw2d_inputs as si
from paper_1711_04471_b200 import sw2d

P = dict(si.PARAMS)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cfg():
    return dict(si.config("c3"), nx=97, ny=61, sigma=4.0, seed=21)


HALO = 4  # SW2D_HALO_ROWS (include/sw2d.h)


def _exchange(arrs, plan, rank):
    """Send/recv HALO storage rows per field with the neighbours (the plan)."""
    reqs, landing = [], []
    for side, peer in ((0, rank - 1), (1, rank + 1)):
        snd, rcv = plan[2 * side], plan[2 * side + 1]
        if snd < 0:
            continue
        for a in arrs:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(a[snd:snd + HALO])),
                                   peer))
            buf = torch.empty((HALO, a.shape[1]), dtype=torch.float32)
            reqs.append(dist.irecv(buf, peer))
            landing.append((a, rcv, buf))
    for r in reqs:
        r.wait()
    for a, rcv, buf in landing:
        a[rcv:rcv + HALO] = buf.numpy()


def _worker(rank, world, port, nsteps, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = _cfg()
        ny, nx = cfg["ny"], cfg["nx"]
        j0, nrows = sw2d.sw2d_partition(ny, world, rank)
        plan = sw2d.sw2d_halo_plan(ny, world, rank)
        # storage rows 0..nrows+2H-1 <-> global rows j0-H .. j0+nrows+H-1
        st = [np.zeros((nrows + 2 * HALO, nx), np.float32) for _ in range(4)]
        own = si.generate(cfg, j0=j0, nrows=nrows)
        for a, o in zip(st, own):
            a[HALO:nrows + HALO] = o
        hz, e, u, v = st
        _exchange([hz], plan, rank)                  # static hzero halo, once
        s_lo = 0 if plan[1] >= 0 else HALO           # window: storage rows in the grid
        s_hi = nrows + 2 * HALO if plan[3] >= 0 else nrows + HALO
        for _ in range(nsteps):
            _exchange([e, u, v], plan, rank)         # state-n halos
            w = oracle.run(P, hz[s_lo:s_hi], e[s_lo:s_hi], u[s_lo:s_hi], v[s_lo:s_hi], 1)
            for a, b in zip((e, u, v), w):
                a[s_lo:s_hi] = b
        sl = slice(HALO, nrows + HALO)
        owned = torch.from_numpy(np.stack([e[sl], u[sl], v[sl]]))
        sizes = [sw2d.sw2d_partition(ny, world, r)[1] for r in range(world)]
        if rank == 0:
            parts = [owned] + [torch.empty((3, n, nx), dtype=torch.float32) for n in sizes[1:]]
            for r in range(1, world):
                dist.recv(parts[r], r)
            full = torch.cat(parts, dim=1).numpy()
            np.save(result_path, full)
        else:
            dist.send(owned, 0)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slabs_with_halo_plan_equal_single_grid(world, tmp_path):
    nsteps = 40
    path = str(tmp_path / "full.npy")
    mp.spawn(_worker, args=(world, _free_port(), nsteps, path), nprocs=world, join=True)
    got = np.load(path)
    cfg = _cfg()
    want = oracle.run(P, *si.generate(cfg), nsteps)
    for name, g, w in zip(("eta", "u", "v"), got, want):
        bad = np.argwhere(g != w)
        assert len(bad) == 0, f"{name} differs first at {tuple(bad[0])} with {world} ranks"
    assert np.max(np.abs(want[1])) > 0


def test_halo_plan_is_symmetric():
    """What a rank sends north is what its north neighbour receives from the
    south, and the rows are owned rows / halo rows."""
    for ny, world in [(16, 2), (61, 3), (1000, 8), (16384 * 8, 8)]:
        for r in range(world):
            j0, n = sw2d.sw2d_partition(ny, world, r)
            p = sw2d.sw2d_halo_plan(ny, world, r)
            if r > 0:
                assert p[0] == HALO and p[1] == 0
            else:
                assert p[0] == p[1] == -1
            if r < world - 1:
                assert p[2] == n and p[3] == n + HALO
                # the north neighbour's first owned storage row holds global row j0 + n
                assert sw2d.sw2d_partition(ny, world, r + 1)[0] == j0 + n
            else:
                assert p[2] == p[3] == -1
