"""Quick timing of the SOR kernel (NEXT-4) for tuning: per-iteration device
time with CUDA events on the handle's stream, for several z-chunk sizes.
usage: python tools/sor_time.py [config ...] [--kz 0,8,16] [--iters N]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import sor_inputs as so  # noqa: E402
from paper_1711_04471_b200 import sor3d  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="*", default=["sor300", "sor1024"])
ap.add_argument("--kz", default="0")
ap.add_argument("--iters", type=int, default=0)
ap.add_argument("--every", type=int, default=0)
ap.add_argument("--shape", default="", help="nx,ny,nz override (seeded like sor_s1)")
a = ap.parse_args()
if a.shape:
    nx, ny, nz = (int(v) for v in a.shape.split(","))
    so.CONFIGS["shape"] = dict(nx=nx, ny=ny, nz=nz, iters=50, seed=7, desc="custom")
    a.configs = ["shape"]
for name in a.configs:
    cfg = so.config(name)
    p0, rhs = so.generate(cfg)
    n = a.iters or cfg["iters"]
    for kz in [int(x) for x in a.kz.split(",")]:
        os.environ["SOR3D_KZ"] = str(kz)
        s = torch.cuda.Stream()
        h = sor3d.sor3d_create(sor3d.make_params(cfg["nx"], cfg["ny"], cfg["nz"], **so.params()),
                               stream=s)
        sor3d.sor3d_set(h, p0, rhs)
        sor3d.sor3d_iterate(h, 5, a.every)
        sor3d.sor3d_sync(h)
        best = 1e30
        for rep in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            sor3d.sor3d_iterate(h, n, a.every)
            e1.record(s)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) / 1e3)
        cells = so.cells(cfg)
        per = best / n
        print(f"{name} kz={kz} {sor3d.sor3d_plan(h)}\n   {n} iters: {best*1e3:.3f} ms, "
              f"{per*1e6:.2f} us/iter, {cells*n/best:.3e} cell-iter/s, "
              f"{12*cells/per/1e9:.0f} GB/s (12 B/cell)", flush=True)
        sor3d.sor3d_destroy(h)
