"""Print the step-kernel launch plan of a handle (GPU box): occupancy, grid."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_1711_04471_b200 import sw2d
for nx, ny, red in [(16384, 16384, 1), (8192, 8192, 0), (500, 500, 0)]:
    h = sw2d.sw2d_create(sw2d.make_params(nx, ny, reduce_every_step=red))
    print(nx, ny, red, "ok")
    sw2d.sw2d_destroy(h)
