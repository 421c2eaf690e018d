"""Real ranks on ONE B200: the P2P transport between processes.

2 and 3 processes share cuda:0, one rank each (one process per rank, as on a
multi-GPU box), with no NCCL anywhere (SW2D_BOOT_EXTERNAL): every rank
exports its peer blob (CUDA IPC handles of its state buffers and sync buffer),
gloo all-gathers the blobs, and sw2d_p2p_import maps the peers — within one
device CUDA IPC maps another process's allocation just as it maps a peer
GPU's.  What runs is exactly the multi-GPU P2P path:

* the boundary launches' remote stores into the neighbours' halo rows,
* the cuStreamWaitValue32 / cuStreamWriteValue32 halo signals (monotone
  counters: a second sw2d_set_state on the same handles must not race the
  neighbours' last signals of the previous run — ADVICE r01 #2),
* the record exchange that replaces the allreduce (each
  rank stores its partial record into every peer's slot and folds the slots
  in rank order), with history rings shorter than the run,
* sw2d_reduce through the same exchange.

No kernel spins on another rank: every cross-rank wait is a stream memory
operation (a front-end semaphore wait, like an IPC event), so the ranks'
kernels need not be co-resident.  Each run's gathered fields and wet masks
must equal the single-grid oracle bitwise, every rank's per-step records must
be identical and within 1e-5 (sums) / exact (max, min, count) of the oracle's.
"""
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

import oracle
import sw2d_inputs as si
from paper_1711_04471_b200 import sw2d

pytestmark = pytest.mark.gpu
P = dict(si.PARAMS)
ALL = (1 << sw2d.SW2D_RED_N) - 1
TIMEOUT_S = 240


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cfg(nx, ny):
    return dict(si.config("c3"), nx=nx, ny=ny, sigma=max(2.0, min(nx, ny) / 20), seed=77)


def _worker(rank, world, port, out_dir, nx, ny, runs, history_len, mask):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        cfg = _cfg(nx, ny)
        j0, nrows = sw2d.sw2d_partition(ny, world, rank)
        st = si.generate(cfg, j0=j0, nrows=nrows)
        p = sw2d.make_params(nx, ny, cfg["dx"], cfg["dy"], cfg["dt"], cfg["g"], cfg["eps"],
                             cfg["hmin"], reduce_every_step=mask, history_len=history_len)
        h = sw2d.sw2d_create(p, sw2d.make_dist(rank, world, 0, 0, None, sw2d.SW2D_HALO_P2P,
                                               sw2d.SW2D_BOOT_EXTERNAL))
        try:
            blobs = [None] * world
            dist.all_gather_object(blobs, sw2d.sw2d_p2p_export(h))
            sw2d.sw2d_p2p_import(h, blobs)
            plan = sw2d.sw2d_plan(h)
            for i, chunks in enumerate(runs):
                sw2d.sw2d_set_state(h, *st)
                for c in chunks:
                    sw2d.sw2d_step(h, c)
                n = sum(chunks)
                e, u, v, w = sw2d.get_state(h, nx)
                keep = min(n, history_len)
                hist = np.stack([sw2d.sw2d_reduce_history(h, op, keep) if mask >> op & 1
                                 else np.zeros(keep) for op in range(sw2d.SW2D_RED_N)], axis=1)
                red = np.array([sw2d.sw2d_reduce(h, op) for op in range(sw2d.SW2D_RED_N)])
                np.savez(os.path.join(out_dir, f"run{i}_rank{rank}.npz"), j0=j0, e=e, u=u, v=v,
                         w=w, hist=hist, red=red, plan=plan, launches=sw2d.sw2d_launch_count(h))
        finally:
            sw2d.sw2d_destroy(h)
    finally:
        dist.destroy_process_group()


def _run_procs(world, out_dir, nx, ny, runs, history_len, mask):
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker,
                         args=(r, world, port, str(out_dir), nx, ny, runs, history_len, mask))
             for r in range(world)]
    for pr in procs:
        pr.start()
    try:
        for pr in procs:
            pr.join(TIMEOUT_S)
        hung = [r for r, pr in enumerate(procs) if pr.is_alive()]
        assert not hung, f"ranks {hung} did not finish within {TIMEOUT_S} s"
        codes = [pr.exitcode for pr in procs]
        assert codes == [0] * world, f"rank exit codes {codes}"
    finally:
        for pr in procs:
            if pr.is_alive():
                pr.kill()
                pr.join(10)


def _check(world, out_dir, nx, ny, runs, history_len, mask):
    cfg = _cfg(nx, ny)
    st = si.generate(cfg)
    for i, chunks in enumerate(runs):
        n = sum(chunks)
        want = oracle.run(P, *st, n, history=True)
        ww = oracle.wet(P, st[0], want[0])
        parts = [np.load(out_dir / f"run{i}_rank{r}.npz") for r in range(world)]
        where = f"run {i} ({chunks}), {world} ranks, history_len {history_len}"
        assert "halo=p2p" in str(parts[0]["plan"]), str(parts[0]["plan"])
        for name, idx in (("e", 0), ("u", 1), ("v", 2)):
            got = np.concatenate([q[name] for q in parts])
            bad = np.argwhere(got != want[idx])
            assert bad.size == 0, f"{where}: {name} differs first at {tuple(bad[0])}"
        assert np.array_equal(np.concatenate([q["w"] for q in parts]), ww), f"{where}: wet"
        keep = min(n, history_len)
        ref = want[3][n - keep:]
        h0 = parts[0]["hist"]
        for q in parts[1:]:  # every rank folds the same slots in the same order
            assert np.array_equal(q["hist"], h0), f"{where}: ranks' records differ"
            assert np.array_equal(q["red"], parts[0]["red"]), f"{where}: sw2d_reduce differs"
        for op in range(oracle.NRED):
            if not mask >> op & 1:
                continue
            g, w = h0[:, op], ref[:, op]
            if op in (oracle.VOLUME, oracle.SUM_ETA):
                assert np.all(np.abs(g - w) <= 1e-5 * np.maximum(np.abs(w), 1e-12)), (where, op)
            else:
                assert np.array_equal(g, w), (where, oracle.RED_NAMES[op], g, w)
        red_want = oracle.reduce(P, st[0], *want[:3])
        red = parts[0]["red"]
        for op in range(oracle.NRED):
            if op in (oracle.VOLUME, oracle.SUM_ETA):
                assert abs(red[op] - red_want[op]) <= 1e-5 * max(abs(red_want[op]), 1e-12)
            else:
                assert red[op] == red_want[op], (where, oracle.RED_NAMES[op])


@pytest.mark.parametrize("world,history_len,mask", [
    (2, 1, ALL),       # ring of one record: every pass's two records share a slot
    (2, 0, 1 << sw2d.SW2D_RED_VOLUME),
    (3, 3, ALL),
    (3, 0, 0),         # no per-step records: halos and sw2d_reduce only
])
def test_p2p_real_ranks_share_one_gpu_bitwise(world, history_len, mask, tmp_path):
    nx, ny = 333, 130
    # two runs on the same handles (the second set_state follows the first
    # run's last signals); odd chunks give one-step passes; 130 steps take the
    # 64-record exchange ring around twice
    runs = [[37], [5, 1, 64, 60]]
    hl = history_len or 1024
    _run_procs(world, tmp_path, nx, ny, runs, hl, mask)
    _check(world, tmp_path, nx, ny, runs, hl, mask)


def test_p2p_import_rejects_mismatched_blobs():
    """A blob set that does not describe this grid / rank order is refused
    (checked before any IPC mapping: one process suffices)."""
    p = sw2d.make_params(64, 40)
    h = sw2d.sw2d_create(p, sw2d.make_dist(0, 2, 0, 0, None, sw2d.SW2D_HALO_P2P,
                                           sw2d.SW2D_BOOT_EXTERNAL))
    try:
        mine = sw2d.sw2d_p2p_export(h)
        with pytest.raises(sw2d.Sw2dError) as ei:
            sw2d.sw2d_p2p_import(h, [mine, mine])   # rank 1's slot holds rank 0's blob
        assert ei.value.code == sw2d.SW2D_EINVAL
        with pytest.raises(sw2d.Sw2dError) as ei:
            sw2d.sw2d_p2p_import(h, [mine])          # wrong length
        assert ei.value.code == sw2d.SW2D_EINVAL
        st = si.generate(_cfg(64, 40), j0=0, nrows=20)
        with pytest.raises(sw2d.Sw2dError) as ei:
            sw2d.sw2d_set_state(h, *st)             # peers not mapped yet
        assert ei.value.code == sw2d.SW2D_ESTATE
    finally:
        sw2d.sw2d_destroy(h)
    with pytest.raises(sw2d.Sw2dError) as ei:   # no NCCL means P2P halos only
        sw2d.sw2d_create(p, sw2d.make_dist(0, 2, 0, 0, None, sw2d.SW2D_HALO_NCCL,
                                           sw2d.SW2D_BOOT_EXTERNAL))
    assert ei.value.code == sw2d.SW2D_EINVAL
