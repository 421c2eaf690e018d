"""Thin Python binding of the C ABI in ``include/sor3d.h`` (ctypes): the
red-black SOR Poisson solver of SURVEY.md §8(f) NEXT-4 (the UFLES "press"
subroutine, arXiv 1711.04471 §6.3).

Argument marshalling only: every iteration runs in the CUDA kernels of
``libsw2d.so`` (the same library as the 2DSW step).  The functions keep the C
names.  Arrays may be numpy arrays or torch tensors (host or CUDA),
C-contiguous float32 [nz][ny][nx].  A non-zero status raises ``Sor3dError``.
No fallback: if the library is missing every call raises.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import sw2d as _sw2d

SOR3D_OK, SOR3D_EINVAL, SOR3D_ENOMEM, SOR3D_ECUDA, SOR3D_ESTATE = 0, -1, -2, -3, -5

#: every symbol include/sor3d.h declares (checked by tests/test_abi.py)
SYMBOLS = ("sor3d_abi_version", "sor3d_create", "sor3d_set", "sor3d_iterate",
           "sor3d_residual", "sor3d_residual_history", "sor3d_history_count",
           "sor3d_get", "sor3d_sync", "sor3d_launch_count", "sor3d_plan",
           "sor3d_destroy", "sor3d_last_error")


class Sor3dError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{msg} (status {code})")
        self.code = code


class sor3d_params(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int64), ("ny", ctypes.c_int64), ("nz", ctypes.c_int64),
                ("dx", ctypes.c_float), ("dy", ctypes.c_float), ("dz", ctypes.c_float),
                ("omega", ctypes.c_float), ("history_len", ctypes.c_int32)]


_lib = None


def load():
    """The loaded library with the sor3d_* signatures set (raises if missing)."""
    global _lib
    if _lib is not None:
        return _lib
    lib = _sw2d.load()
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    sig = {
        "sor3d_abi_version": ([], ctypes.c_int),
        "sor3d_create": ([ctypes.POINTER(sor3d_params), vp, ctypes.POINTER(vp)], ctypes.c_int),
        "sor3d_set": ([vp, vp, vp], ctypes.c_int),
        "sor3d_iterate": ([vp, i64, i64], ctypes.c_int),
        "sor3d_residual": ([vp, vp], ctypes.c_int),
        "sor3d_residual_history": ([vp, vp, i64], ctypes.c_int),
        "sor3d_history_count": ([vp], ctypes.c_int64),
        "sor3d_get": ([vp, vp], ctypes.c_int),
        "sor3d_sync": ([vp], ctypes.c_int),
        "sor3d_launch_count": ([vp], ctypes.c_int64),
        "sor3d_plan": ([vp], ctypes.c_char_p),
        "sor3d_destroy": ([vp], None),
        "sor3d_last_error": ([vp], ctypes.c_char_p),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def _check(rc: int, h=None):
    if rc != SOR3D_OK:
        raise Sor3dError(rc, load().sor3d_last_error(h).decode() or f"status {rc}")


def make_params(nx, ny, nz, dx=1.0, dy=1.0, dz=1.0, omega=1.5, history_len=0) -> sor3d_params:
    return sor3d_params(int(nx), int(ny), int(nz), float(dx), float(dy), float(dz),
                        float(omega), int(history_len))


def sor3d_abi_version() -> int:
    return load().sor3d_abi_version()


def sor3d_create(params: sor3d_params, stream=None):
    """Opaque handle; ``stream`` as in sw2d_create (None: library-owned)."""
    if stream is not None and hasattr(stream, "cuda_stream"):
        stream = stream.cuda_stream
    if stream is not None and int(stream) == 0:
        stream = 1  # cudaStreamLegacy; NULL means "own stream"
    h = ctypes.c_void_p()
    _check(load().sor3d_create(ctypes.byref(params),
                               ctypes.c_void_p(stream) if stream is not None else None,
                               ctypes.byref(h)))
    return h


def sor3d_set(h, p, rhs) -> None:
    _check(load().sor3d_set(h, _sw2d._ptr(p), _sw2d._ptr(rhs)), h)


def sor3d_iterate(h, n: int, residual_every: int = 0) -> None:
    _check(load().sor3d_iterate(h, int(n), int(residual_every)), h)


def sor3d_residual(h) -> np.ndarray:
    out = np.zeros(2, np.float64)
    _check(load().sor3d_residual(h, ctypes.c_void_p(out.ctypes.data)), h)
    return out


def sor3d_residual_history(h, n: int) -> np.ndarray:
    out = np.zeros((int(n), 2), np.float64)
    _check(load().sor3d_residual_history(h, ctypes.c_void_p(out.ctypes.data), int(n)), h)
    return out


def sor3d_history_count(h) -> int:
    return int(load().sor3d_history_count(h))


def sor3d_get(h, p) -> None:
    _check(load().sor3d_get(h, _sw2d._ptr(p, writable=True)), h)


def sor3d_sync(h) -> None:
    _check(load().sor3d_sync(h), h)


def sor3d_launch_count(h) -> int:
    return int(load().sor3d_launch_count(h))


def sor3d_plan(h) -> str:
    return load().sor3d_plan(h).decode()


def sor3d_destroy(h) -> None:
    if h:
        load().sor3d_destroy(h)


def sor3d_last_error(h=None) -> str:
    return load().sor3d_last_error(h).decode()


def get(h, nx: int, ny: int, nz: int) -> np.ndarray:
    """Download p into a new numpy array [nz][ny][nx]."""
    p = np.empty((nz, ny, nx), np.float32)
    sor3d_get(h, p)
    return p
