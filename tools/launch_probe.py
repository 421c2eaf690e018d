"""Host cost of enqueuing steps vs device time per step (tiny grid)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1711_04471_b200 import sw2d
s = torch.cuda.Stream()
for nx, ny in ((32, 8), (500, 500)):
    hz = np.full((ny, nx), 10.0, np.float32); e = np.zeros_like(hz)
    h = sw2d.sw2d_create(sw2d.make_params(nx, ny), None, s)
    sw2d.sw2d_set_state(h, hz, e)
    sw2d.sw2d_step(h, 200); sw2d.sw2d_sync(h)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    t0 = time.perf_counter(); sw2d.sw2d_step(h, 2000); t1 = time.perf_counter()
    b.record(s); sw2d.sw2d_sync(h)
    print(f"{nx}x{ny}: host enqueue {(t1 - t0) / 2000 * 1e6:.2f} us/step, device {a.elapsed_time(b) / 2000 * 1000:.2f} us/step", flush=True)
    sw2d.sw2d_destroy(h)
