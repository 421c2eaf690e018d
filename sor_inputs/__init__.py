"""sor_inputs — seeded synthetic inputs for the NEXT-4 SOR Poisson workload
(shared by the oracle side and the CUDA side; holds none of the method's
arithmetic: it makes right-hand sides and initial guesses, nothing that
relaxes them).

Recipe (DESIGN.md §13 "Input recipe"): the UFLES pressure equation's
right-hand side is the divergence of the predicted velocity field over a
building-resolving urban domain, smooth in the open air
with sharp sources and sinks at obstacles.  Synthetic stand-in:

* grid spacings dx = dy = 4 m (300 cells over the paper's 1.2 km,
  PAPER.md:427-429), dz = 2 m (reading S6), omega = 1.5 (reading S5);
* rhs = sum over 12 seeded blobs of a_b exp(-|x - c_b|^2 / (2 s_b^2)) (cell
  units; centres uniform in the box, widths 2..8 cells, amplitudes +-1
  uniform) plus white noise uniform in [-0.05, 0.05);
* p0 = white noise uniform in [-0.01, 0.01) (a warm start: the previous
  time step's pressure);
* every random number comes from splitmix64 over a counter: blob b uses the
  stream of seed ^ b, cell noise uses the hash of (seed, field, flat index),
  so any value is a pure function of (config, index), computed in float64
  and rounded once to float32.
"""
from __future__ import annotations

import numpy as np

CONFIGS = {
    "sor_s1": dict(nx=37, ny=29, nz=11, iters=20, seed=11,
                   desc="SOR 37x29x11 (ragged tiles), 20 iterations"),
    "sor_s2": dict(nx=130, ny=70, nz=40, iters=10, seed=12,
                   desc="SOR 130x70x40 (several tiles and z-chunks), 10 iterations"),
    "sor300": dict(nx=300, ny=300, nz=90, iters=50, seed=1711044716,
                   desc="UFLES press shape: 300x300x90, 50 SOR iterations "
                        "(PAPER.md:427-428)"),
    "sor1024": dict(nx=1024, ny=1024, nz=256, iters=10, seed=1711044717,
                    desc="SOR 1024x1024x256 (larger than L2: HBM-bound study), "
                         "10 iterations"),
}
PARAMS = dict(dx=4.0, dy=4.0, dz=2.0, omega=1.5)
NBLOB = 12
_M64 = np.uint64((1 << 64) - 1)


def _mix(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _uniform(seed: int, field: int, idx: np.ndarray) -> np.ndarray:
    """Uniform [0, 1) doubles: splitmix64 of counter seed*2^8+field, idx."""
    with np.errstate(over="ignore"):
        key = np.uint64(((seed << 8) + field) & ((1 << 64) - 1))
        z = _mix(key * np.uint64(0x9E3779B97F4A7C15) + idx.astype(np.uint64)
                 * np.uint64(0x9E3779B97F4A7C15) + np.uint64(0x632BE59BD9B4E019))
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / (1 << 53))


def config(name: str) -> dict:
    c = dict(CONFIGS[name])
    c["name"] = name
    return c


def params(cfg: dict | None = None) -> dict:
    return dict(PARAMS)


def _blobs(cfg):
    nx, ny, nz = cfg["nx"], cfg["ny"], cfg["nz"]
    u = _uniform(cfg["seed"], 1, np.arange(NBLOB * 5))
    u = u.reshape(NBLOB, 5)
    return [(u[b, 0] * nx, u[b, 1] * ny, u[b, 2] * nz, 2.0 + 6.0 * u[b, 3], 2.0 * u[b, 4] - 1.0)
            for b in range(NBLOB)]


def generate(cfg: dict, k0: int = 0, nk: int | None = None):
    """(p0, rhs) float32 [nk][ny][nx] for planes [k0, k0+nk) (0-based)."""
    nx, ny, nz = cfg["nx"], cfg["ny"], cfg["nz"]
    nk = nz - k0 if nk is None else nk
    z = np.arange(k0, k0 + nk, dtype=np.float64)[:, None, None] + 1.0
    y = np.arange(ny, dtype=np.float64)[None, :, None] + 1.0
    x = np.arange(nx, dtype=np.float64)[None, None, :] + 1.0
    rhs = np.zeros((nk, ny, nx), np.float64)
    for (cx, cy, cz, s, a) in _blobs(cfg):
        rhs += a * (np.exp(-(x - cx) ** 2 / (2 * s * s)) * np.exp(-(y - cy) ** 2 / (2 * s * s))
                    * np.exp(-(z - cz) ** 2 / (2 * s * s)))
    flat = (np.arange(k0 * ny * nx, (k0 + nk) * ny * nx, dtype=np.int64)).reshape(nk, ny, nx)
    rhs += 0.1 * _uniform(cfg["seed"], 2, flat) - 0.05
    p0 = 0.02 * _uniform(cfg["seed"], 3, flat) - 0.01
    return p0.astype(np.float32), rhs.astype(np.float32)


def cells(cfg: dict) -> int:
    return cfg["nx"] * cfg["ny"] * cfg["nz"]
