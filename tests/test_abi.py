"""C-ABI library checks that need no GPU: it builds/loads, exports every
symbol include/sw2d.h declares, and its pure host logic (slab partition,
status strings) behaves as the header states."""
import os
import re

import pytest

from paper_1711_04471_b200 import sw2d

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "sw2d.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sw2d_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1711_04471_b200 import _build
    _build.build()
    return sw2d.load()


def test_exports_every_declared_symbol(lib):
    declared = _declared_symbols()
    assert len(declared) >= 15
    assert sorted(declared) == sorted(sw2d.SYMBOLS)
    for name in declared:
        assert hasattr(lib, name), name


def test_abi_version(lib):
    src = open(os.path.join(ROOT, "include", "sw2d.h")).read()
    declared = int(re.search(r"#define SW2D_ABI_VERSION (\d+)", src).group(1))
    assert sw2d.sw2d_abi_version() == declared


def test_built_for_sm100a(lib):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", sw2d._LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


_PROBE_DEFINES = (("-DSW2D_EXACT_FMA=0", "-DSW2D_F32X2_MIN_RED=0"),
                  ("-DSW2D_EXACT_FMA=0", "-DSW2D_PACKED_MUL=0"))
_probe_cache = {}


def _probe_cmd(red, defines, cubin):
    from paper_1711_04471_b200 import _build
    cmd = [_build.NVCC, *[f for f in _build.FLAGS if f not in ("-shared",)],
           "-Xcompiler", "-fPIC", f"-DPROBE_RED={red}", *defines,
           "-I", os.path.join(ROOT, "include"), "-I", _build.CSRC, "-cubin", "-o", cubin,
           os.path.join(ROOT, "tools", "cta2_probe.cu")]
    return [c for c in cmd if c != "-Xcompiler,-fPIC,-O2,-Wall"]


def _probe_sass(red, *defines):
    """SASS of sw2d_step_cta2<red, 0> alone (tools/cta2_probe.cu), built with the
    library's flags plus `defines`.  The first call builds every (red, defines)
    pair the tests use at once, in parallel (each takes tens of seconds)."""
    import subprocess
    import tempfile
    if not _probe_cache:
        with tempfile.TemporaryDirectory() as d:
            jobs = {}
            for r in (0, 1, 2):
                for k, defs in enumerate(_PROBE_DEFINES):
                    cubin = os.path.join(d, f"probe_{r}_{k}.cubin")
                    jobs[(r, defs)] = (cubin, subprocess.Popen(
                        _probe_cmd(r, defs, cubin), stdout=subprocess.PIPE,
                        stderr=subprocess.PIPE))
            for key, (cubin, proc) in jobs.items():
                out, err = proc.communicate()
                assert proc.returncode == 0, err.decode()[-2000:]
                _probe_cache[key] = subprocess.run(
                    ["/usr/local/cuda/bin/cuobjdump", "-sass", cubin],
                    capture_output=True, text=True).stdout
    sass = _probe_cache[(red, tuple(defines))]
    funcs = [f for f in re.split(r"\n\s+Function : ", sass)[1:]
             if "sw2d_step_cta2" in f.split("\n", 1)[0]]
    assert len(funcs) == 1
    return funcs[0]


@pytest.mark.parametrize("red", [0, 1, 2])
def test_step_kernel_fuses_no_rounded_product(red):
    """Bitwise parity needs every rounded product rounded before its add
    (R24).  ptxas 12.9 contracts mul.rn.f32x2 + add.rn.f32x2
    into FFMA2 even under --fmad=false, so the packed products are written as
    fma.rn.f32x2 with a -0 addend held in a kernel parameter (Coef::nz); the
    only other fused multiply-adds are the exact wet-flag products
    (sel(w, x) + y, SW2D_EXACT_FMA).  With those built as mul + add
    (SW2D_EXACT_FMA=0) every FFMA2 of the two-step kernel must be a product
    with a scalar-broadcast addend (the -0) and no negated operand, and no
    scalar FFMA may remain: ptxas fused nothing on its own.  (The GPU parity
    tests, bitwise against the oracle, are the final word.)  With the products scalar too
    (SW2D_PACKED_MUL=0) there is no fused multiply-add at all."""
    f = _probe_sass(red, "-DSW2D_EXACT_FMA=0", "-DSW2D_F32X2_MIN_RED=0")
    assert not re.search(r"\bFFMA\b", f), "scalar FFMA: a contracted mul + add"
    addends = re.findall(r"\bFFMA2\s+[^;]*,\s*(-?R\d+(?:\.reuse)?\.F32\S*)\s*;", f)
    n = len(re.findall(r"\bFFMA2\b", f))
    assert n > 0, "packed products missing"
    assert len(addends) == n, "an FFMA2 whose addend is not a scalar broadcast"
    # a product with a -0 addend negates nothing; the one add with a broadcast
    # constant in the step (1 - q*s) is a subtraction, so contracting it (or
    # any e - t*c) would show a negated operand
    for m in re.finditer(r"\bFFMA2\s+([^;]*);", f):
        assert "-R" not in m.group(1), m.group(0)
    g = _probe_sass(red, "-DSW2D_EXACT_FMA=0", "-DSW2D_PACKED_MUL=0")
    assert not re.search(r"\bFFMA2?\b", g), "fused multiply-add with scalar products"


def test_step_kernels_pack_adds(lib):
    import subprocess
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", sw2d._LIB_PATH],
                          capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", sass)[1:]
    steps = [f for f in funcs if "sw2d_step" in f.split("\n", 1)[0]]
    assert steps, "no sw2d_step kernels found in the SASS"
    assert any(re.search(r"\bFADD2\b", f) for f in steps), "packed adds missing"
    assert any(re.search(r"\bFFMA2\b", f) for f in steps), "packed products missing"


@pytest.mark.parametrize("ny,p",[(10, 1), (17, 2), (100, 3), (16384 * 8, 8), (16, 2)])
def test_partition_balanced_and_covering(lib, ny, p):
    rows = [sw2d.sw2d_partition(ny, p, r) for r in range(p)]
    assert rows[0][0] == 0
    for (j0, n), (j1, _) in zip(rows, rows[1:]):
        assert j0 + n == j1
    assert rows[-1][0] + rows[-1][1] == ny
    sizes = [n for _, n in rows]
    assert max(sizes) - min(sizes) <= 1


def test_partition_rejects(lib):
    for args in [(15, 2, 0), (10, 0, 0), (10, 2, 2), (10, 2, -1), (0, 1, 0)]:
        with pytest.raises(sw2d.Sw2dError) as ei:
            sw2d.sw2d_partition(*args)
        assert ei.value.code == sw2d.SW2D_EINVAL


def test_strerror(lib):
    assert sw2d.sw2d_strerror(0) == "ok"
    assert sw2d.sw2d_strerror(sw2d.SW2D_ESTATE) == "state not set"
    assert sw2d.sw2d_strerror(-99) == "unknown status"


def test_create_validates_params_before_touching_the_gpu(lib):
    bad = [dict(dx=0.0), dict(dt=float("nan")), dict(eps=1.5), dict(hmin=-1.0),
           dict(g=-9.81), dict(nx=0)]
    for b in bad:
        kw = dict(nx=8, ny=8)
        kw.update(b)
        with pytest.raises(sw2d.Sw2dError) as ei:
            sw2d.sw2d_create(sw2d.make_params(**kw))
        assert ei.value.code == sw2d.SW2D_EINVAL
    with pytest.raises(sw2d.Sw2dError) as ei:
        sw2d.sw2d_create(sw2d.make_params(8, 8, bc=1))
    assert ei.value.code == sw2d.SW2D_EUNSUPPORTED


def test_nccl_unique_id_host_only(lib):
    uid = sw2d.sw2d_nccl_unique_id()
    assert len(uid) == 128


# --- NEXT-4: include/sor3d.h ---------------------------------------------------

def _declared_sor3d():
    src = open(os.path.join(ROOT, "include", "sor3d.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sor3d_[a-z_]+)\s*\(", src)))


def test_sor3d_exports_every_declared_symbol(lib):
    from paper_1711_04471_b200 import sor3d
    declared = _declared_sor3d()
    assert len(declared) >= 12
    assert declared == sorted(sor3d.SYMBOLS)
    for name in declared:
        assert hasattr(lib, name), name
    src = open(os.path.join(ROOT, "include", "sor3d.h")).read()
    assert sor3d.sor3d_abi_version() == int(
        re.search(r"#define SOR3D_ABI_VERSION (\d+)", src).group(1))


def test_sor3d_create_validates_params_before_touching_the_gpu(lib):
    from paper_1711_04471_b200 import sor3d
    for b in [dict(nx=0), dict(nz=-3), dict(dx=0.0), dict(dz=float("inf")), dict(omega=2.0),
              dict(omega=0.0), dict(history_len=-1), dict(ny=(1 << 20) + 1)]:
        kw = dict(nx=8, ny=8, nz=8)
        kw.update(b)
        with pytest.raises(sor3d.Sor3dError) as ei:
            sor3d.sor3d_create(sor3d.make_params(**kw))
        assert ei.value.code == sor3d.SOR3D_EINVAL
    assert sor3d.sor3d_launch_count(None) == -1
    assert sor3d.sor3d_history_count(None) == -1
