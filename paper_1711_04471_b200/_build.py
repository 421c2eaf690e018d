"""Build of the CUDA C-ABI library ``libsw2d.so`` (sm_100a, in-tree).

``python -m paper_1711_04471_b200._build`` or ``__graft_entry__.build()``.
nvcc cross-compiles for sm_100a without a GPU.  ``--fmad=false`` backs up the
kernels' explicit ``__f*_rn`` intrinsics: no multiply-add is ever contracted,
so the step's arithmetic is the oracle's, operation for operation.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsw2d.so")
DEBUG_LIB = os.path.join(PKG, "libsw2d_dbg.so")   # device bounds checks (SW2D_DEBUG_BOUNDS)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_include() -> str:
    cands = []
    try:
        import nvidia.nccl  # type: ignore
        cands += [os.path.join(p, "include") for p in nvidia.nccl.__path__]
    except Exception:
        pass
    cands.append("/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/include")
    for c in cands:
        if os.path.exists(os.path.join(c, "nccl.h")):
            return c
    raise RuntimeError("nccl.h not found (needed for NCCL types)")


FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "--fmad=false", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
    "-Xcompiler", "-fPIC,-O2,-Wall",
    "-shared",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [
        os.path.join(ROOT, "include", "sw2d.h"), os.path.join(ROOT, "include", "sor3d.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, extra=(), debug: bool = False,
          out: str | None = None) -> str:
    """Build libsw2d.so (or `out`: an A/B variant built with `extra` flags)."""
    variant = out is not None
    out = out or (DEBUG_LIB if debug else LIB)
    if debug:
        extra = (*extra, "-DSW2D_DEBUG_BOUNDS")
    elif not force and not variant and not _stale():
        return LIB
    tmp = out + f".tmp{os.getpid()}"
    objdir = out + f".obj{os.getpid()}"
    os.makedirs(objdir, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", _nccl_include()]
    compile_flags = [f for f in FLAGS if f != "-shared"]
    jobs = []
    for src in sources():   # one nvcc per translation unit, in parallel, then link
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        jobs.append([NVCC, *compile_flags, *extra, *inc, "-c", src, "-o", obj])
    try:
        procs = []
        for cmd in jobs:
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            procs.append((cmd, subprocess.Popen(cmd)))
        for cmd, pr in procs:
            if pr.wait() != 0:
                raise subprocess.CalledProcessError(pr.returncode, cmd)
        link = [NVCC, *FLAGS, *extra, *[c[-1] for c in jobs], "-o", tmp, "-ldl"]
        subprocess.check_call(link)
        os.replace(tmp, out)
    finally:
        for f in glob.glob(os.path.join(objdir, "*.o")):
            os.remove(f)
        os.rmdir(objdir)
    return out


if __name__ == "__main__":
    # python -m paper_1711_04471_b200._build [-v] [--ptxas] [--debug]
    #        [--out path -DFLAG=1 ...]   (A/B variants: extra nvcc flags after --out)
    v = "-v" in sys.argv
    extra = ["-Xptxas", "-v"] if "--ptxas" in sys.argv else []
    out = None
    if "--out" in sys.argv:
        i = sys.argv.index("--out")
        out = sys.argv[i + 1]
        extra += [a for a in sys.argv[i + 2:] if a.startswith("-D")]
    print(build(force=True, verbose=v, extra=extra, debug="--debug" in sys.argv, out=out))
