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


def test_step_kernels_have_no_fused_multiply_add(lib):
    """Bitwise parity needs every product rounded before its add (DESIGN.md
    §7, packed FP32 adds): ptxas 12.9 contracts a packed f32x2 mul feeding a
    packed add into FFMA2 even under --fmad=false, so check the SASS of the
    2DSW step kernels for any FFMA / FFMA2."""
    import subprocess
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", sw2d._LIB_PATH],
                          capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", sass)[1:]
    steps = [f for f in funcs if "sw2d_step" in f.split("\n", 1)[0]]
    assert steps, "no sw2d_step kernels found in the SASS"
    for f in steps:
        name = f.split("\n", 1)[0].strip()
        assert not re.search(r"\bFFMA2?\b", f), f"fused multiply-add in {name}"
    assert any(re.search(r"\bFADD2\b", f) for f in steps), "packed adds missing"


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
