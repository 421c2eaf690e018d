"""sw2d_inputs — seeded synthetic inputs for the 2DSW step (shared by both arms).

This module is the ONLY code shared by the oracle side and the CUDA side.  It
holds none of the method's arithmetic: it makes bathymetry, an initial
free-surface bump and the model parameters, nothing that steps the model.

Recipe:

* Model parameters follow the paper's 2DSW runs: dx = dy = 1 m, dt = 0.01 s
  ("spatial resolution of 1 m and a time step of 0.01 s");
  g = 9.81, Shapiro eps = 0.05, hmin = 0.05 m (readings R7, R10).
* Cell centre coordinates, 1-based cell indices j (rows, y) and k (cols, x):
  x = (k - (nx+1)/2) dx, y = (j - (ny+1)/2) dy.
* ``flat``: H0 = 10 m everywhere (C1, C2: the paper's flat 500x500 shape).
* ``bowl``: H0 = 10 (1 - x^2/Rx^2 - y^2/Ry^2) - sum_i 13 exp(-d_i^2 / (2 s^2)),
  Rx = 0.45 nx dx, Ry = 0.45 ny dy, s = min(nx, ny) dx / 170; 16 island
  centres uniform in the 0.8-scaled ellipse, drawn with splitmix64(seed) by
  rejection in the unit disk.  An island term is included only where
  d_i < 8 s (its value beyond is < 2e-13 m).  Land outside the ellipse and the
  island tops are dry; the slopes are an active shoreline.
* Initial state: eta = -min(0, H0) (rest; land cells have h = 0), plus the
  Gaussian bump A * exp(-(j-jc)^2/(2 sig^2)) * exp(-(k-kc)^2/(2 sig^2)) (cell
  units, evaluated in double in that order) added where H0 >= hmin; u = v = 0.
  For ``bowl`` the bump centre is the grid centre plus a seeded offset uniform
  in the 0.3-scaled ellipse.
* Everything is computed in float64 and rounded once to float32, and every
  value is a pure function of (config, seed, j, k), so any row slab or window
  can be generated on its own (each rank makes its own slab).
"""
from __future__ import annotations

import numpy as np

PARAMS = dict(dx=1.0, dy=1.0, dt=0.01, g=9.81, eps=0.05, hmin=0.05)

# BASELINE.json "configs" (C1..C5); steps are the configs' step counts.
CONFIGS = {
    "c1": dict(nx=100, ny=100, kind="flat", amp=0.5, sigma=5.0, seed=0,
               steps=1000,
               desc="2DSW 100x100 grid, 1000 steps, single Gaussian eta bump, "
                    "closed basin"),
    "c2": dict(nx=500, ny=500, kind="flat", amp=0.5, sigma=25.0, seed=0,
               steps=10000,
               desc="2DSW 500x500 grid matching the paper's 2DSW run shape, "
                    "10k steps, 1 B200"),
    "c3": dict(nx=8192, ny=8192, kind="bowl", amp=0.5, sigma=128.0,
               seed=1711044713, steps=1000,
               desc="2DSW 8192x8192 with wet/dry bathymetry, 1 B200 roofline "
                    "study"),
    "c4": dict(nx=32768, ny=32768, kind="bowl", amp=0.5, sigma=512.0,
               seed=1711044714, steps=1000,
               desc="2DSW 32768x32768 row-decomposed over 2/4/8 B200 with "
                    "NVLink halo exchange (strong scaling)"),
    "c5": dict(nx=16384, ny=16384, kind="bowl", amp=0.5, sigma=256.0,
               seed=1711044715, steps=1000, per_gpu_rows=16384,
               desc="2DSW weak scaling: 16384x16384 per GPU at 1/2/4/8 B200 "
                    "with per-step global-volume reduction"),
    # the paper's other 2DSW sizes, for the small-grid study
    "p1000": dict(nx=1000, ny=1000, kind="flat", amp=0.5, sigma=50.0, seed=0, steps=10000,
                  desc="2DSW 1000x1000 (paper size), flat basin, 10k steps"),
    "p2000": dict(nx=2000, ny=2000, kind="flat", amp=0.5, sigma=100.0, seed=0, steps=10000,
                  desc="2DSW 2000x2000 (paper size), flat basin, 10k steps"),
}

_M64 = (1 << 64) - 1


class SplitMix64:
    """splitmix64 (Steele, Lea, Flood 2014) — the counter-based seed stream."""

    def __init__(self, seed: int):
        self.state = seed & _M64

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)

    def uniform(self) -> float:
        return (self.next() >> 11) * (1.0 / (1 << 53))

    def disk(self):
        while True:
            a = 2.0 * self.uniform() - 1.0
            b = 2.0 * self.uniform() - 1.0
            if a * a + b * b < 1.0:
                return a, b


def config(name: str, nranks: int = 1) -> dict:
    """The named config with its global grid; c5 grows ny with the rank count
    (weak scaling: 16384 rows per GPU)."""
    cfg = dict(CONFIGS[name])
    cfg["name"] = name
    if name == "c5":
        cfg["ny"] = cfg["per_gpu_rows"] * int(nranks)
    cfg.update(PARAMS)
    return cfg


def _layout(cfg):
    """Island centres and bump centre (in metres / cell units) for a config."""
    nx, ny, dx, dy = cfg["nx"], cfg["ny"], cfg["dx"], cfg["dy"]
    jc, kc = (ny + 1) / 2.0, (nx + 1) / 2.0
    islands = []
    if cfg["kind"] == "bowl":
        rx, ry = 0.45 * nx * dx, 0.45 * ny * dy
        rng = SplitMix64(cfg["seed"])
        for _ in range(16):
            a, b = rng.disk()
            islands.append((0.8 * rx * a, 0.8 * ry * b))
        a, b = rng.disk()
        kc += 0.3 * rx * a / dx
        jc += 0.3 * ry * b / dy
    return islands, jc, kc


def generate(cfg: dict, j0: int = 0, nrows: int | None = None, k0: int = 0,
             ncols: int | None = None, out=None, chunk_rows: int = 1024):
    """(hzero, eta, u, v) float32 [nrows][ncols] for the window of 0-based
    rows [j0, j0+nrows) and cols [k0, k0+ncols) of the config's global grid.

    ``out``: optional 4-tuple of preallocated float32 arrays (e.g. pinned host
    buffers) to fill instead of allocating."""
    nx, ny = cfg["nx"], cfg["ny"]
    nrows = ny - j0 if nrows is None else nrows
    ncols = nx - k0 if ncols is None else ncols
    if not (0 <= j0 and j0 + nrows <= ny and 0 <= k0 and k0 + ncols <= nx):
        raise ValueError("window outside the grid")
    if out is None:
        out = tuple(np.empty((nrows, ncols), np.float32) for _ in range(4))
    hz, eta, u, v = out
    u[...] = 0.0
    v[...] = 0.0
    dx, dy, hmin = cfg["dx"], cfg["dy"], np.float32(cfg["hmin"])
    islands, jc, kc = _layout(cfg)
    kk = np.arange(k0 + 1, k0 + ncols + 1, dtype=np.float64)   # 1-based k
    x = (kk - (nx + 1) / 2.0) * dx
    sig = cfg["sigma"]
    gx = np.exp(-((kk - kc) ** 2) / (2.0 * sig * sig))
    amp = cfg["amp"]
    if cfg["kind"] == "bowl":
        rx, ry = 0.45 * nx * dx, 0.45 * ny * dy
        s = min(nx, ny) * dx / 170.0
        cut = 8.0 * s
        bx = 1.0 - (x * x) / (rx * rx)
    for r0 in range(0, nrows, chunk_rows):
        r1 = min(nrows, r0 + chunk_rows)
        jj = np.arange(j0 + r0 + 1, j0 + r1 + 1, dtype=np.float64)  # 1-based j
        if cfg["kind"] == "flat":
            h0d = np.full((r1 - r0, ncols), 10.0)
        else:
            y = (jj - (ny + 1) / 2.0) * dy
            h0d = 10.0 * (bx[None, :] - ((y * y) / (ry * ry))[:, None])
            for (xi, yi) in islands:
                # rows / cols of this chunk within the cut radius
                ra = np.searchsorted(y, yi - cut, side="left")
                rb = np.searchsorted(y, yi + cut, side="right")
                ca = np.searchsorted(x, xi - cut, side="left")
                cb = np.searchsorted(x, xi + cut, side="right")
                if ra >= rb or ca >= cb:
                    continue
                d2 = ((x[ca:cb] - xi) ** 2)[None, :] + ((y[ra:rb] - yi) ** 2)[:, None]
                term = 13.0 * np.exp(-d2 / (2.0 * s * s))
                term[d2 >= cut * cut] = 0.0
                h0d[ra:rb, ca:cb] -= term
        h0 = h0d.astype(np.float32)
        hz[r0:r1] = h0
        gy = amp * np.exp(-((jj - jc) ** 2) / (2.0 * sig * sig))
        bump = gy[:, None] * gx[None, :]
        rest = -np.minimum(np.float32(0.0), h0).astype(np.float64)
        e = np.where(h0 >= hmin, rest + bump, rest)
        eta[r0:r1] = e.astype(np.float32)
    return hz, eta, u, v


def model_params(cfg: dict) -> dict:
    """The scalar model parameters of a config (dx, dy, dt, g, eps, hmin)."""
    return {k: cfg[k] for k in ("dx", "dy", "dt", "g", "eps", "hmin")}


def cells(cfg: dict) -> int:
    return int(cfg["nx"]) * int(cfg["ny"])

