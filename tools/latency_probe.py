"""Per-step time of tiny grids: one warp marching ny rows (SW2D_MIN_ROWS large)
-> fixed launch cost + per-row iteration latency."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1711_04471_b200 import sw2d
torch.cuda.init()
s = torch.cuda.Stream()
for ny in (4, 8, 16, 32, 64, 128, 256):
    nx = 32
    hz = np.full((ny, nx), 10.0, np.float32); e = np.zeros_like(hz)
    h = sw2d.sw2d_create(sw2d.make_params(nx, ny), None, s)
    sw2d.sw2d_set_state(h, hz, e)
    sw2d.sw2d_step(h, 200); sw2d.sw2d_sync(h)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s); sw2d.sw2d_step(h, 2000); b.record(s); sw2d.sw2d_sync(h)
    print(f"kind {os.environ.get('SW2D_STEP_KERNEL','auto')} ny {ny:4d}: {a.elapsed_time(b) / 2000 * 1000:.2f} us/step", flush=True)
    sw2d.sw2d_destroy(h)
# empty kernel launch rate for reference
x = torch.zeros(1, device="cuda")
with torch.cuda.stream(s):
    for _ in range(100): x.add_(1)
    a.record(s)
    for _ in range(2000): x.add_(1)
    b.record(s)
torch.cuda.synchronize()
print(f"torch add_ launch: {a.elapsed_time(b) / 2000 * 1000:.2f} us")
