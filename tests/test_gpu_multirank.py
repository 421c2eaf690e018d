"""Real multi-GPU parity (skipped on boxes with fewer than two GPUs).

One process per GPU over torch.distributed (NCCL), as bench.py runs: every
rank creates an sw2d handle on its own device with a shared ncclUniqueId,
steps its row slab with the library's halo exchange (NCCL send/recv or fused
P2P stores over NVLink), and the gathered slabs plus the per-step
diagnostics must equal the single-grid oracle (fields bitwise).  On a 1-GPU
box the NCCL machinery is covered by test_single_rank_nccl_machinery and the
decomposition by the virtual-rank tests.
"""
import os
import socket

import numpy as np
import pytest

import oracle
import sw2d_inputs as si
from paper_1711_04471_b200 import sw2d

pytestmark = pytest.mark.gpu
P = dict(si.PARAMS)


def _ngpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cfg():
    return dict(si.config("c3"), nx=333, ny=260, sigma=12.0, seed=77)


def _worker(rank, world, port, nsteps, halo, out_dir, boot=0):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        obj = [sw2d.sw2d_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        cfg = _cfg()
        nx, ny = cfg["nx"], cfg["ny"]
        j0, nrows = sw2d.sw2d_partition(ny, world, rank)
        st = si.generate(cfg, j0=j0, nrows=nrows)
        mask = (1 << sw2d.SW2D_RED_N) - 1
        p = sw2d.make_params(nx, ny, cfg["dx"], cfg["dy"], cfg["dt"], cfg["g"], cfg["eps"],
                             cfg["hmin"], reduce_every_step=mask, history_len=nsteps)
        h = sw2d.sw2d_create(p, sw2d.make_dist(rank, world, rank, 0, obj[0], halo, boot))
        try:
            if boot == sw2d.SW2D_BOOT_EXTERNAL:   # no NCCL: the blobs travel over torch
                blobs = [None] * world
                dist.all_gather_object(blobs, sw2d.sw2d_p2p_export(h))
                sw2d.sw2d_p2p_import(h, blobs)
            sw2d.sw2d_set_state(h, *st)
            sw2d.sw2d_step(h, nsteps)
            e, u, v, w = sw2d.get_state(h, nx)
            hist = np.stack([sw2d.sw2d_reduce_history(h, op, nsteps)
                             for op in range(sw2d.SW2D_RED_N)], axis=1)
        finally:
            sw2d.sw2d_destroy(h)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), j0=j0, e=e, u=u, v=v, w=w, hist=hist)
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(_ngpus() < 2, reason="needs two GPUs (one process per GPU)")
@pytest.mark.parametrize("halo,boot", [(sw2d.SW2D_HALO_NCCL, sw2d.SW2D_BOOT_NCCL),
                                       (sw2d.SW2D_HALO_P2P, sw2d.SW2D_BOOT_NCCL),
                                       (sw2d.SW2D_HALO_P2P, sw2d.SW2D_BOOT_EXTERNAL)])
def test_two_real_ranks_bitwise(halo, boot, tmp_path):
    import torch.multiprocessing as mp
    world, nsteps = 2, 37
    mp.spawn(_worker, args=(world, _free_port(), nsteps, halo, str(tmp_path), boot),
             nprocs=world, join=True)
    cfg = _cfg()
    st = si.generate(cfg)
    want = oracle.run(P, *st, nsteps, history=True)
    ww = oracle.wet(P, st[0], want[0])
    parts = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    for name, idx in (("e", 0), ("u", 1), ("v", 2)):
        got = np.concatenate([q[name] for q in parts])
        assert np.array_equal(got, want[idx]), f"{name} differs across the slab split"
    assert np.array_equal(np.concatenate([q["w"] for q in parts]), ww)
    for q in parts:  # every rank holds the global (allreduced) records
        hist = q["hist"]
        for op in range(oracle.NRED):
            g, w = hist[:, op], want[3][:, op]
            if op in (oracle.VOLUME, oracle.SUM_ETA):
                assert np.all(np.abs(g - w) <= 1e-5 * np.maximum(np.abs(w), 1e-12))
            else:
                assert np.array_equal(g, w)
