"""oracle — TEST INFRASTRUCTURE ONLY: the CPU parity oracles of the 2DSW step
and (NEXT-4) of red-black SOR for the Poisson equation.

Plain single-threaded C11 (``oracle/sw2d_ref.c``, ``oracle/sor_ref.c``),
loaded with ctypes.  The 2DSW oracle follows arXiv 1711.04471 §6.2
(time loop -> predictor ``dyn`` -> first-order Shapiro
filter ``shapiro`` -> velocity update) with the textbook scheme and readings
listed in DESIGN.md §3; the SOR oracle follows the UFLES
``press`` solver of §6.3 with the readings
S1-S9 of DESIGN.md §13.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package.  It shares
no code with ``paper_1711_04471_b200`` and never imports it.

Pins: ``tests/test_oracle_pins.py`` (2DSW: invariants, closed forms, hand
examples) and ``tests/test_sor_oracle_pins.py`` (SOR: hand example, dense
solve, O(h^2) manufactured solution, exact polynomial residual, Gauss-Seidel
property).  Parity unpinned by the paper: the 2DSW blocked-face velocity rule
(reading R4) and operation order (R12), and the SOR operation order (S4);
they are pinned only by the DESIGN.md readings.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sw2d_ref.c")
_SOR_SRC = os.path.join(_HERE, "sor_ref.c")   # NEXT-4: red-black SOR Poisson
_LIB = os.path.join(_HERE, "libsw2d_ref.so")

# reduction slots (sw2d_ref.h)
VOLUME, SUM_ETA, MAX_ETA, MIN_ETA, MAX_ABS_U, MAX_ABS_V, WET_COUNT = range(7)
NRED = 7
RED_NAMES = ("VOLUME", "SUM_ETA", "MAX_ETA", "MIN_ETA", "MAX_ABS_U",
             "MAX_ABS_V", "WET_COUNT")

CFLAGS = ["-std=c11", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
          "-fno-fast-math", "-Wall", "-Wextra"]


def build(force: bool = False) -> str:
    """Compile libsw2d_ref.so (gcc, no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or (
            os.path.getmtime(_LIB) < max(os.path.getmtime(_SRC), os.path.getmtime(_SOR_SRC),
                                         os.path.getmtime(_SRC[:-1] + "h"))):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, _SOR_SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Params(ctypes.Structure):
    _fields_ = [("dx", ctypes.c_float), ("dy", ctypes.c_float),
                ("dt", ctypes.c_float), ("g", ctypes.c_float),
                ("eps", ctypes.c_float), ("hmin", ctypes.c_float)]


class _SorParams(ctypes.Structure):
    _fields_ = [("dx", ctypes.c_float), ("dy", ctypes.c_float), ("dz", ctypes.c_float),
                ("omega", ctypes.c_float)]


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        fp = ctypes.POINTER(ctypes.c_float)
        dp = ctypes.POINTER(ctypes.c_double)
        i64 = ctypes.c_int64
        lib.sw2d_ref_run.argtypes = [ctypes.POINTER(_Params), i64, i64, fp, fp,
                                     fp, fp, i64, dp]
        lib.sw2d_ref_reduce.argtypes = [ctypes.POINTER(_Params), i64, i64, fp,
                                        fp, fp, fp, dp]
        lib.sw2d_ref_wet.argtypes = [ctypes.POINTER(_Params), i64, i64, fp, fp,
                                     ctypes.POINTER(ctypes.c_uint8)]
        lib.sor_ref_run.argtypes = [ctypes.POINTER(_SorParams), i64, i64, i64, fp, fp, i64, dp]
        lib.sor_ref_residual.argtypes = [ctypes.POINTER(_SorParams), i64, i64, i64, fp, fp, dp]
        for f in (lib.sw2d_ref_run, lib.sw2d_ref_reduce, lib.sw2d_ref_wet, lib.sor_ref_run,
                  lib.sor_ref_residual):
            f.restype = ctypes.c_int
        _lib = lib
    return _lib


def _params(p) -> _Params:
    return _Params(float(p["dx"]), float(p["dy"]), float(p["dt"]),
                   float(p["g"]), float(p["eps"]), float(p["hmin"]))


def _f32(a):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def run(params, hzero, eta, u, v, nsteps: int, history: bool = False):
    """Advance the state ``nsteps`` steps; returns (eta, u, v[, hist]).

    Inputs are 2-D float32 arrays [ny][nx] (copied; the caller's are not
    modified).  ``hist`` is [nsteps][7] float64: the diagnostics after each
    step."""
    ny, nx = np.shape(hzero)
    hz, hzp = _f32(hzero)
    e, ep = _f32(np.array(eta, dtype=np.float32, copy=True))
    uu, up = _f32(np.array(u, dtype=np.float32, copy=True))
    vv, vp = _f32(np.array(v, dtype=np.float32, copy=True))
    hist = np.zeros((max(nsteps, 0), NRED), np.float64) if history else None
    hp = hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if history else None
    prm = _params(params)
    rc = _load().sw2d_ref_run(ctypes.byref(prm), nx, ny, hzp, ep, up, vp,
                              int(nsteps), hp)
    if rc != 0:
        raise ValueError("sw2d_ref_run: invalid arguments")
    return (e, uu, vv, hist) if history else (e, uu, vv)


def reduce(params, hzero, eta, u, v) -> np.ndarray:
    """The seven diagnostics (VOLUME, SUM_ETA, MAX_ETA, MIN_ETA, MAX_ABS_U,
    MAX_ABS_V, WET_COUNT) of a state, as float64[7]."""
    ny, nx = np.shape(hzero)
    out = np.zeros(NRED, np.float64)
    keep = [_f32(a)[0] for a in (hzero, eta, u, v)]  # held for the call
    args = [k.ctypes.data_as(ctypes.POINTER(ctypes.c_float)) for k in keep]
    prm = _params(params)
    rc = _load().sw2d_ref_reduce(ctypes.byref(prm), nx, ny, *args,
                                 out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    if rc != 0:
        raise ValueError("sw2d_ref_reduce: invalid arguments")
    return out


def wet(params, hzero, eta) -> np.ndarray:
    """uint8 wet mask !(hzero + eta < hmin)."""
    ny, nx = np.shape(hzero)
    hz, hzp = _f32(hzero)
    e, ep = _f32(eta)
    out = np.zeros((ny, nx), np.uint8)
    prm = _params(params)
    rc = _load().sw2d_ref_wet(ctypes.byref(prm), nx, ny, hzp, ep,
                              out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)))
    if rc != 0:
        raise ValueError("sw2d_ref_wet: invalid arguments")
    return out


# --- NEXT-4: red-black SOR for the Poisson equation (oracle/sor_ref.c) -------

def _sor_params(p) -> _SorParams:
    return _SorParams(float(p["dx"]), float(p["dy"]), float(p["dz"]), float(p["omega"]))


def sor_run(params, p, rhs, n: int, history: bool = False):
    """n red-black SOR iterations from p (float32 [nz][ny][nx], copied) for
    Lap(p) = rhs with zero Dirichlet ghosts; returns p (and, with history,
    [n][2] float64: L2 and Linf of the residual after each iteration)."""
    nz, ny, nx = np.shape(rhs)
    pp, ptr = _f32(np.array(p, dtype=np.float32, copy=True))
    rr, rptr = _f32(rhs)
    hist = np.zeros((max(n, 0), 2), np.float64) if history else None
    hp = hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if history else None
    prm = _sor_params(params)
    if _load().sor_ref_run(ctypes.byref(prm), nx, ny, nz, ptr, rptr, int(n), hp) != 0:
        raise ValueError("sor_ref_run: invalid arguments")
    return (pp, hist) if history else pp


def sor_residual(params, p, rhs) -> np.ndarray:
    """[L2, Linf] of r = rhs - Lap(p)."""
    nz, ny, nx = np.shape(rhs)
    pp, ptr = _f32(p)
    rr, rptr = _f32(rhs)
    out = np.zeros(2, np.float64)
    prm = _sor_params(params)
    if _load().sor_ref_residual(ctypes.byref(prm), nx, ny, nz, ptr, rptr,
                                out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))) != 0:
        raise ValueError("sor_ref_residual: invalid arguments")
    return out
