"""Host<->device transfer probe for the e2e path (bench.py `e2e`): times
sw2d_set_state (H2D from pinned memory), sw2d_get_state (D2H to pinned
memory) and sw2d_step(100) on C5, alone and overlapped (two handles, two host
threads), plus raw cudaMemcpyAsync H2D / D2H / both at once of the same
bytes, to see which transfer bounds e2e.

    python tools/xfer_probe.py [--nx 16384 --ny 16384]
"""
import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import sw2d_inputs as si  # noqa: E402
from paper_1711_04471_b200 import sw2d  # noqa: E402


def wall(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=16384)
    ap.add_argument("--ny", type=int, default=16384)
    a = ap.parse_args()
    cfg = dict(si.config("c5", 1), nx=a.nx, ny=a.ny)
    nx, ny = a.nx, a.ny
    torch.cuda.set_device(0)
    host = [torch.empty((ny, nx), dtype=torch.float32, pin_memory=True) for _ in range(4)]
    si.generate(cfg, out=tuple(t.numpy() for t in host))
    outs = [torch.empty((ny, nx), dtype=torch.float32, pin_memory=True) for _ in range(3)]
    p = sw2d.make_params(nx, ny, reduce_every_step=1 << sw2d.SW2D_RED_VOLUME, history_len=100)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    h1 = sw2d.sw2d_create(p, None, s1)
    h2 = sw2d.sw2d_create(p, None, s2)
    res = {}
    try:
        sw2d.sw2d_set_state(h1, *host)
        sw2d.sw2d_set_state(h2, *host)
        res["set_state_s"] = wall(lambda: sw2d.sw2d_set_state(h1, *host))
        res["get_state_s"] = wall(lambda: sw2d.sw2d_get_state(h2, *outs))
        res["step100_s"] = wall(lambda: (sw2d.sw2d_step(h1, 100), sw2d.sw2d_sync(h1)))

        def both():
            t = threading.Thread(target=lambda: sw2d.sw2d_get_state(h2, *outs))
            t.start()
            sw2d.sw2d_set_state(h1, *host)
            t.join()
        res["set_and_get_overlapped_s"] = wall(both)
        # raw copies of the same bytes
        dev = torch.empty(4 * ny * nx, dtype=torch.float32, device="cuda")
        dev2 = torch.empty(3 * ny * nx, dtype=torch.float32, device="cuda")
        hin = torch.empty(4 * ny * nx, dtype=torch.float32, pin_memory=True)
        hout = torch.empty(3 * ny * nx, dtype=torch.float32, pin_memory=True)
        res["raw_h2d_16B_s"] = wall(lambda: dev.copy_(hin, non_blocking=True))
        res["raw_d2h_12B_s"] = wall(lambda: hout.copy_(dev2, non_blocking=True))

        def raw_both():
            with torch.cuda.stream(s1):
                dev.copy_(hin, non_blocking=True)
            with torch.cuda.stream(s2):
                hout.copy_(dev2, non_blocking=True)
        res["raw_both_s"] = wall(raw_both)
        gb_in, gb_out = 16 * nx * ny / 1e9, 12 * nx * ny / 1e9
        res["raw_h2d_GBps"] = gb_in / res["raw_h2d_16B_s"]
        res["raw_d2h_GBps"] = gb_out / res["raw_d2h_12B_s"]
        res["set_state_GBps"] = gb_in / res["set_state_s"]
        res["get_state_GBps"] = gb_out / res["get_state_s"]
        # bench.py's pipelined e2e loop with per-call timestamps
        s3 = torch.cuda.Stream()
        h3 = sw2d.sw2d_create(p, None, s3)
        hs, sts = [h1, h2, h3], [s1, s2, s3]
        sw2d.sw2d_set_state(h3, *host)
        K = 8
        done = [torch.cuda.Event() for _ in range(K)]
        enq = [threading.Event() for _ in range(K)]
        freed = [threading.Event() for _ in range(K)]
        outs3 = [[torch.empty((ny, nx), dtype=torch.float32, pin_memory=True) for _ in range(3)]
                 for _ in range(3)]
        hist = [__import__("numpy").empty(100) for _ in range(3)]
        tr = []
        t0 = time.perf_counter()

        def up():
            for k in range(K):
                b = k % 3
                if k >= 3:
                    freed[k - 3].wait()
                ta = time.perf_counter()
                sw2d.sw2d_set_state(hs[b], *host)
                tb = time.perf_counter()
                if k > 0:
                    sts[b].wait_event(done[k - 1])
                sw2d.sw2d_step(hs[b], 100)
                done[k].record(sts[b])
                enq[k].set()
                tr.append(("up", k, ta - t0, tb - t0))

        def down():
            for k in range(K):
                enq[k].wait()
                ta = time.perf_counter()
                sw2d.sw2d_get_state(hs[k % 3], *outs3[k % 3])
                tb = time.perf_counter()
                sw2d.sw2d_reduce_history(hs[k % 3], sw2d.SW2D_RED_VOLUME, 100, hist[k % 3])
                freed[k].set()
                tr.append(("down", k, ta - t0, tb - t0))
        th = [threading.Thread(target=up), threading.Thread(target=down)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        torch.cuda.synchronize()
        res["pipeline_s_per_problem"] = (time.perf_counter() - t0) / K
        res["trace"] = sorted(tr, key=lambda x: x[2])
        sw2d.sw2d_destroy(h3)
    finally:
        sw2d.sw2d_destroy(h1)
        sw2d.sw2d_destroy(h2)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
