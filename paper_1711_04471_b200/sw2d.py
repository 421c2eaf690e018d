"""Thin Python binding of the C ABI in ``include/sw2d.h`` (ctypes).

Argument marshalling only: every step of the 2DSW path runs in the CUDA
kernels of ``libsw2d.so``.  The functions keep the C names.  Arrays may be
numpy arrays or torch tensors (host or CUDA), C-contiguous, float32 (uint8 for
the wet mask), shaped [nrows][nx].  A non-zero status raises ``Sw2dError``.

There is no fallback: if ``libsw2d.so`` is missing or fails to load, every
call raises.  Build it with ``python -m paper_1711_04471_b200._build``.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_LIB_PATH = os.environ.get("SW2D_LIBRARY") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libsw2d.so")   # SW2D_LIBRARY: debug build

SW2D_OK, SW2D_EINVAL, SW2D_ENOMEM, SW2D_ECUDA, SW2D_ENCCL, SW2D_ESTATE, \
    SW2D_EUNSUPPORTED = 0, -1, -2, -3, -4, -5, -6
SW2D_BC_CLOSED = 0
(SW2D_RED_VOLUME, SW2D_RED_SUM_ETA, SW2D_RED_MAX_ETA, SW2D_RED_MIN_ETA,
 SW2D_RED_MAX_ABS_U, SW2D_RED_MAX_ABS_V, SW2D_RED_WET_COUNT) = range(7)
SW2D_RED_N = 7
SW2D_VARIANT_FUSED = 0
SW2D_VARIANT_PAPER = 1
SW2D_HALO_NCCL, SW2D_HALO_P2P = 0, 1
SW2D_BOOT_NCCL, SW2D_BOOT_EXTERNAL = 0, 1
SW2D_P2P_BLOB_BYTES = 1024

#: every symbol include/sw2d.h declares (checked by tests/test_abi.py)
SYMBOLS = ("sw2d_abi_version", "sw2d_partition", "sw2d_halo_plan", "sw2d_nccl_unique_id",
           "sw2d_create", "sw2d_p2p_export", "sw2d_p2p_import",
           "sw2d_local_rows", "sw2d_local_shape", "sw2d_set_state", "sw2d_step",
           "sw2d_run_snapshots", "sw2d_reduce", "sw2d_reduce_history", "sw2d_get_state",
           "sw2d_sync", "sw2d_plan",
           "sw2d_launch_count", "sw2d_destroy", "sw2d_strerror",
           "sw2d_last_error")


class Sw2dError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{msg} (status {code})")
        self.code = code


class sw2d_params(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int64), ("ny", ctypes.c_int64),
                ("dx", ctypes.c_float), ("dy", ctypes.c_float),
                ("dt", ctypes.c_float), ("g", ctypes.c_float),
                ("eps", ctypes.c_float), ("hmin", ctypes.c_float),
                ("bc", ctypes.c_int32), ("reduce_every_step", ctypes.c_uint32),
                ("variant", ctypes.c_int32), ("history_len", ctypes.c_int32)]


class sw2d_dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("nranks", ctypes.c_int32),
                ("device", ctypes.c_int32), ("virtual_ranks", ctypes.c_int32),
                ("halo_mode", ctypes.c_int32), ("nccl_id", ctypes.c_ubyte * 128),
                ("bootstrap", ctypes.c_int32)]


_lib = None


def load(path: str = _LIB_PATH):
    """Load libsw2d.so (raises if it is missing: no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: build it with "
                           "`python -m paper_1711_04471_b200._build`")
    lib = ctypes.CDLL(path)
    vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
    p64 = ctypes.POINTER(ctypes.c_int64)
    sig = {
        "sw2d_abi_version": ([], ctypes.c_int),
        "sw2d_partition": ([i64, i32, i32, p64, p64], ctypes.c_int),
        "sw2d_halo_plan": ([i64, i32, i32, p64], ctypes.c_int),
        "sw2d_nccl_unique_id": ([vp], ctypes.c_int),
        "sw2d_create": ([ctypes.POINTER(sw2d_params), ctypes.POINTER(sw2d_dist), vp,
                         ctypes.POINTER(vp)], ctypes.c_int),
        "sw2d_p2p_export": ([vp, vp, ctypes.c_size_t], ctypes.c_int),
        "sw2d_p2p_import": ([vp, vp, ctypes.c_size_t], ctypes.c_int),
        "sw2d_local_rows": ([vp, p64, p64], ctypes.c_int),
        "sw2d_local_shape": ([vp, p64, p64], ctypes.c_int),
        "sw2d_set_state": ([vp, vp, vp, vp, vp], ctypes.c_int),
        "sw2d_step": ([vp, i64], ctypes.c_int),
        "sw2d_run_snapshots": ([vp, i64, i64, vp, i64], ctypes.c_int),
        "sw2d_reduce": ([vp, ctypes.c_int, ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
        "sw2d_reduce_history": ([vp, ctypes.c_int, vp, i64], ctypes.c_int),
        "sw2d_get_state": ([vp, vp, vp, vp, vp], ctypes.c_int),
        "sw2d_sync": ([vp], ctypes.c_int),
        "sw2d_launch_count": ([vp], ctypes.c_int64),
        "sw2d_plan": ([vp], ctypes.c_char_p),
        "sw2d_destroy": ([vp], None),
        "sw2d_strerror": ([ctypes.c_int], ctypes.c_char_p),
        "sw2d_last_error": ([vp], ctypes.c_char_p),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def _check(rc: int, h=None):
    if rc != SW2D_OK:
        lib = load()
        detail = lib.sw2d_last_error(h).decode() or lib.sw2d_strerror(rc).decode()
        raise Sw2dError(rc, detail)


def _ptr(a, dtype=np.float32, writable=False, need=None):
    """Pointer of a C-contiguous numpy array / torch tensor (host or CUDA)
    holding at least `need` elements (the C side reads / writes that many)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):  # torch.Tensor
        import torch
        want = {np.float32: torch.float32, np.float64: torch.float64,
                np.uint8: torch.uint8}[dtype]
        if a.dtype != want or not a.is_contiguous():
            raise TypeError(f"tensor must be contiguous {want}")
        size = a.numel()
        ptr = a.data_ptr()
    else:
        if not isinstance(a, np.ndarray) or a.dtype != dtype or not a.flags.c_contiguous:
            raise TypeError(f"array must be a C-contiguous numpy {np.dtype(dtype).name} array")
        if writable and not a.flags.writeable:
            raise TypeError("output array is read-only")
        size = a.size
        ptr = a.ctypes.data
    if need is not None and size < need:
        raise ValueError(f"array holds {size} elements, the call needs {need}")
    return ctypes.c_void_p(ptr)


def _cells(h) -> int:
    """Elements of one [nrows][nx] field of the rows the handle holds."""
    n, nx = sw2d_local_shape(h)
    return n * nx


def make_params(nx, ny, dx=1.0, dy=1.0, dt=0.01, g=9.81, eps=0.05, hmin=0.05,
                reduce_every_step=0, history_len=0, variant=SW2D_VARIANT_FUSED,
                bc=SW2D_BC_CLOSED) -> sw2d_params:
    return sw2d_params(int(nx), int(ny), float(dx), float(dy), float(dt), float(g),
                       float(eps), float(hmin), int(bc), int(reduce_every_step),
                       int(variant), int(history_len))


def make_dist(rank=0, nranks=1, device=-1, virtual_ranks=0, nccl_id=None,
              halo_mode=0, bootstrap=SW2D_BOOT_NCCL) -> sw2d_dist:
    d = sw2d_dist(int(rank), int(nranks), int(device), int(virtual_ranks), int(halo_mode))
    if nccl_id is not None:
        ctypes.memmove(d.nccl_id, bytes(nccl_id), 128)
    d.bootstrap = int(bootstrap)
    return d


# --- the ABI, same names ---------------------------------------------------

def sw2d_abi_version() -> int:
    return load().sw2d_abi_version()


def sw2d_partition(ny: int, nranks: int, rank: int):
    j0, n = ctypes.c_int64(), ctypes.c_int64()
    _check(load().sw2d_partition(int(ny), int(nranks), int(rank),
                                 ctypes.byref(j0), ctypes.byref(n)))
    return j0.value, n.value


def sw2d_halo_plan(ny: int, nranks: int, rank: int):
    """(send_south, recv_south, send_north, recv_north) first storage rows of
    the SW2D_HALO_ROWS-row halo messages of `rank` (-1: no neighbour)."""
    out = (ctypes.c_int64 * 4)()
    rc = load().sw2d_halo_plan(int(ny), int(nranks), int(rank), out)
    if rc < 0:
        _check(rc)
    return tuple(int(x) for x in out)


def sw2d_nccl_unique_id() -> bytes:
    buf = (ctypes.c_ubyte * 128)()
    _check(load().sw2d_nccl_unique_id(buf))
    return bytes(buf)


def sw2d_create(params: sw2d_params, dist: sw2d_dist | None = None, stream=None):
    """Returns an opaque handle (ctypes.c_void_p).  ``stream``: a CUDA stream
    handle (int / torch.cuda.Stream) to enqueue on (0 = the legacy default
    stream), or None for a library-owned stream."""
    if stream is not None and hasattr(stream, "cuda_stream"):
        stream = stream.cuda_stream
    if stream is not None and int(stream) == 0:
        stream = 1  # the legacy default stream (cudaStreamLegacy); NULL means "own stream"
    h = ctypes.c_void_p()
    rc = load().sw2d_create(ctypes.byref(params),
                            ctypes.byref(dist) if dist is not None else None,
                            ctypes.c_void_p(stream) if stream is not None else None,
                            ctypes.byref(h))
    _check(rc)
    return h


def sw2d_p2p_export(h) -> bytes:
    """This rank's peer blob (SW2D_P2P_BLOB_BYTES bytes) for sw2d_p2p_import."""
    buf = (ctypes.c_ubyte * SW2D_P2P_BLOB_BYTES)()
    _check(load().sw2d_p2p_export(h, buf, SW2D_P2P_BLOB_BYTES), h)
    return bytes(buf)


def sw2d_p2p_import(h, blobs) -> None:
    """``blobs``: every rank's blob in rank order (a list of bytes, or their
    concatenation)."""
    data = b"".join(blobs) if isinstance(blobs, (list, tuple)) else bytes(blobs)
    buf = (ctypes.c_ubyte * len(data)).from_buffer_copy(data)
    _check(load().sw2d_p2p_import(h, buf, len(data)), h)


def sw2d_local_rows(h):
    j0, n = ctypes.c_int64(), ctypes.c_int64()
    _check(load().sw2d_local_rows(h, ctypes.byref(j0), ctypes.byref(n)), h)
    return j0.value, n.value


def sw2d_local_shape(h):
    """(nrows, nx) of the [nrows][nx] host-visible arrays of this handle."""
    n, nx = ctypes.c_int64(), ctypes.c_int64()
    _check(load().sw2d_local_shape(h, ctypes.byref(n), ctypes.byref(nx)), h)
    return n.value, nx.value


def sw2d_set_state(h, hzero, eta, u=None, v=None) -> None:
    c = _cells(h)
    _check(load().sw2d_set_state(h, _ptr(hzero, need=c), _ptr(eta, need=c), _ptr(u, need=c),
                                 _ptr(v, need=c)), h)


def sw2d_step(h, nsteps: int) -> None:
    _check(load().sw2d_step(h, int(nsteps)), h)


def sw2d_run_snapshots(h, nsteps: int, every: int, out_eta) -> None:
    """Run nsteps; out_eta [nsnap][nrows][nx] float32 receives eta after every
    `every` steps (nsnap = nsteps // every)."""
    nsnap = int(nsteps) // int(every) if every else -1
    out = _ptr(out_eta, writable=True, need=max(nsnap, 0) * _cells(h))
    _check(load().sw2d_run_snapshots(h, int(nsteps), int(every), out, nsnap), h)


def sw2d_reduce(h, op: int) -> float:
    out = ctypes.c_double()
    _check(load().sw2d_reduce(h, int(op), ctypes.byref(out)), h)
    return out.value


def sw2d_reduce_history(h, op: int, n: int, out=None) -> np.ndarray:
    out = np.empty(int(n), np.float64) if out is None else out
    _check(load().sw2d_reduce_history(h, int(op), _ptr(out, np.float64, True, need=int(n)),
                                      int(n)), h)
    return out


def sw2d_get_state(h, eta=None, u=None, v=None, wet=None) -> None:
    c = _cells(h)
    _check(load().sw2d_get_state(h, _ptr(eta, writable=True, need=c),
                                 _ptr(u, writable=True, need=c), _ptr(v, writable=True, need=c),
                                 _ptr(wet, np.uint8, True, need=c)), h)


def sw2d_sync(h) -> None:
    _check(load().sw2d_sync(h), h)


def sw2d_launch_count(h) -> int:
    return int(load().sw2d_launch_count(h))


def sw2d_plan(h) -> str:
    return load().sw2d_plan(h).decode()


def sw2d_destroy(h) -> None:
    if h:
        load().sw2d_destroy(h)


def sw2d_strerror(code: int) -> str:
    return load().sw2d_strerror(int(code)).decode()


def sw2d_last_error(h=None) -> str:
    return load().sw2d_last_error(h).decode()


# --- convenience -----------------------------------------------------------

def get_state(h, nx: int, wet: bool = True):
    """Allocate numpy outputs and download (eta, u, v, wet) of the local rows."""
    _, n = sw2d_local_rows(h)
    e = np.empty((n, nx), np.float32)
    u = np.empty((n, nx), np.float32)
    v = np.empty((n, nx), np.float32)
    w = np.empty((n, nx), np.uint8) if wet else None
    sw2d_get_state(h, e, u, v, w)
    return (e, u, v, w) if wet else (e, u, v)
