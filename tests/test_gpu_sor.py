"""GPU parity of the NEXT-4 red-black SOR solver (include/sor3d.h) against the
CPU oracle (oracle/sor_ref.c), through the C ABI.

Bar: p bitwise equal to the oracle after every tested
iteration count (same binary32 operations in the same order, no FMA); the
residual Linf exact (a max of identical fp32 values) and L2 within 1e-12
relative (fp64 sums of identical squares in another order).  Sizes: ragged
tiles (60 x 28 columns per CTA; 60 x 12 with SOR3D_ROWS=16) and z-chunks, degenerate 1-cell axes, chunk
overrides, and the paper's full 300 x 300 x 90 x 50 iterations (the oracle
runs it in ~10 s) — the launch configuration bench.py times.
"""
import numpy as np
import pytest

import oracle
import sor_inputs as so
from paper_1711_04471_b200 import sor3d

pytestmark = pytest.mark.gpu
L2_RTOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    sor3d.load()


def _case(nx, ny, nz, seed=5):
    cfg = dict(so.config("sor_s1"), nx=nx, ny=ny, nz=nz, seed=seed)
    return so.generate(cfg)


def gpu_sor(prm, p0, rhs, n, every=0, kz=None, monkeypatch=None):
    nz, ny, nx = rhs.shape
    if kz is not None:
        monkeypatch.setenv("SOR3D_KZ", str(kz))
    h = sor3d.sor3d_create(sor3d.make_params(nx, ny, nz, **prm))
    try:
        sor3d.sor3d_set(h, p0, rhs)
        sor3d.sor3d_iterate(h, n, every)
        p = sor3d.get(h, nx, ny, nz)
        nrec = sor3d.sor3d_history_count(h)
        hist = sor3d.sor3d_residual_history(h, nrec) if nrec else np.zeros((0, 2))
        launches = sor3d.sor3d_launch_count(h)
        plan = sor3d.sor3d_plan(h)
    finally:
        sor3d.sor3d_destroy(h)
    return p, hist, launches, plan


def check_hist(got, want):
    assert got.shape == want.shape, (got.shape, want.shape)
    np.testing.assert_array_equal(got[:, 1], want[:, 1])          # Linf exact
    np.testing.assert_allclose(got[:, 0], want[:, 0], rtol=L2_RTOL, atol=0)


def assert_bitwise(got, want, where):
    if not np.array_equal(got.view(np.uint32), want.view(np.uint32)):
        bad = np.argwhere(got.view(np.uint32) != want.view(np.uint32))
        k, j, i = bad[0]
        raise AssertionError(f"{where}: {len(bad)} cells differ, first (k={k}, j={j}, i={i}): "
                             f"gpu {got[k, j, i]!r} oracle {want[k, j, i]!r}")


P = so.params()


@pytest.mark.parametrize("name", ["sor_s1", "sor_s2"])
def test_small_configs_bitwise_with_history(name):
    cfg = so.config(name)
    p0, rhs = so.generate(cfg)
    n = cfg["iters"]
    want, wh = oracle.sor_run(P, p0, rhs, n, history=True)
    got, gh, launches, _ = gpu_sor(P, p0, rhs, n, every=1)
    assert_bitwise(got, want, name)
    check_hist(gh, wh)
    assert launches == n + 1   # one per iteration + the final residual-only pass


def test_paper_size_300x300x90_50_iterations():
    """The paper's UFLES press configuration, full field."""
    cfg = so.config("sor300")
    p0, rhs = so.generate(cfg)
    want, wh = oracle.sor_run(P, p0, rhs, 50, history=True)
    got, gh, launches, plan = gpu_sor(P, p0, rhs, 50, every=1)
    assert_bitwise(got, want, "sor300")
    check_hist(gh, wh)


@pytest.mark.parametrize("shape", [(1, 1, 1), (1, 7, 5), (9, 1, 3), (4, 5, 1), (60, 12, 2),
                                   (61, 13, 3), (59, 11, 4), (121, 25, 9), (2, 2, 2),
                                   (200, 3, 2), (3, 100, 2)])
def test_edge_shapes(shape):
    nx, ny, nz = shape
    p0, rhs = _case(nx, ny, nz)
    want, wh = oracle.sor_run(P, p0, rhs, 7, history=True)
    got, gh, _, _ = gpu_sor(P, p0, rhs, 7, every=1)
    assert_bitwise(got, want, f"{shape}")
    check_hist(gh, wh)


@pytest.mark.parametrize("kz", [1, 2, 3, 5, 64])
def test_z_chunks(kz, monkeypatch):
    """Chunk boundaries inside the march (the 2-plane overlap of each chunk)."""
    p0, rhs = _case(70, 20, 13)
    want = oracle.sor_run(P, p0, rhs, 6)
    got, _, _, plan = gpu_sor(P, p0, rhs, 6, kz=kz, monkeypatch=monkeypatch)
    assert f"z-chunk {min(kz, 13)}" in plan
    assert_bitwise(got, want, f"kz={kz}")


@pytest.mark.parametrize("prm", [dict(dx=1.0, dy=1.0, dz=1.0, omega=1.0),
                                 dict(dx=0.5, dy=3.0, dz=1.7, omega=1.9),
                                 dict(dx=4.0, dy=4.0, dz=2.0, omega=0.7)])
def test_parameters(prm):
    p0, rhs = _case(67, 31, 10, seed=9)
    want, wh = oracle.sor_run(prm, p0, rhs, 9, history=True)
    got, gh, _, _ = gpu_sor(prm, p0, rhs, 9, every=1)
    assert_bitwise(got, want, str(prm))
    check_hist(gh, wh)


@pytest.mark.parametrize("n,every", [(10, 3), (10, 5), (1, 1), (7, 100), (0, 1)])
def test_residual_every(n, every):
    p0, rhs = _case(41, 17, 6)
    want, wh = oracle.sor_run(P, p0, rhs, n, history=True)
    got, gh, launches, _ = gpu_sor(P, p0, rhs, n, every=every)
    assert_bitwise(got, want, f"n={n}")
    rows = [t - 1 for t in range(1, n + 1) if t % every == 0 or t == n]
    check_hist(gh, wh[rows] if rows else np.zeros((0, 2)))
    assert launches == n + (1 if n else 0)


def test_residual_of_state_and_device_pointers():
    import torch
    p0, rhs = _case(90, 40, 12)
    nz, ny, nx = rhs.shape
    h = sor3d.sor3d_create(sor3d.make_params(nx, ny, nz, **P))
    try:
        sor3d.sor3d_set(h, torch.from_numpy(p0).cuda(), torch.from_numpy(rhs).cuda())
        r0 = sor3d.sor3d_residual(h)
        w0 = oracle.sor_residual(P, p0, rhs)
        assert r0[1] == w0[1] and abs(r0[0] - w0[0]) <= L2_RTOL * w0[0]
        sor3d.sor3d_iterate(h, 4)
        out = torch.empty((nz, ny, nx), dtype=torch.float32, device="cuda")
        sor3d.sor3d_get(h, out)
        want = oracle.sor_run(P, p0, rhs, 4)
        assert_bitwise(out.cpu().numpy(), want, "device pointers")
        r = sor3d.sor3d_residual(h)
        w = oracle.sor_residual(P, want, rhs)
        assert r[1] == w[1] and abs(r[0] - w[0]) <= L2_RTOL * w[0]
        # set again resets the state and the history
        sor3d.sor3d_set(h, p0, rhs)
        assert sor3d.sor3d_history_count(h) == 0
        sor3d.sor3d_iterate(h, 4, 2)
        assert_bitwise(sor3d.get(h, nx, ny, nz), want, "after re-set")
        assert sor3d.sor3d_history_count(h) == 2
    finally:
        sor3d.sor3d_destroy(h)


def test_history_ring_wraps():
    p0, rhs = _case(33, 14, 5)
    want, wh = oracle.sor_run(P, p0, rhs, 12, history=True)
    nz, ny, nx = rhs.shape
    h = sor3d.sor3d_create(sor3d.make_params(nx, ny, nz, history_len=5, **P))
    try:
        sor3d.sor3d_set(h, p0, rhs)
        sor3d.sor3d_iterate(h, 12, 1)
        assert sor3d.sor3d_history_count(h) == 12
        check_hist(sor3d.sor3d_residual_history(h, 5), wh[7:])
        with pytest.raises(sor3d.Sor3dError):
            sor3d.sor3d_residual_history(h, 6)
    finally:
        sor3d.sor3d_destroy(h)


def test_errors():
    h = sor3d.sor3d_create(sor3d.make_params(8, 8, 8))
    try:
        with pytest.raises(sor3d.Sor3dError) as ei:
            sor3d.sor3d_iterate(h, 1)
        assert ei.value.code == sor3d.SOR3D_ESTATE
        p0, rhs = _case(8, 8, 8)
        rhs[3, 2, 1] = np.nan
        with pytest.raises(sor3d.Sor3dError) as ei:
            sor3d.sor3d_set(h, p0, rhs)
        assert ei.value.code == sor3d.SOR3D_EINVAL
        with pytest.raises(sor3d.Sor3dError) as ei:
            sor3d.sor3d_iterate(h, 1)
        assert ei.value.code == sor3d.SOR3D_ESTATE
        rhs[3, 2, 1] = 0.0
        sor3d.sor3d_set(h, p0, rhs)
        with pytest.raises(sor3d.Sor3dError) as ei:
            sor3d.sor3d_iterate(h, -1)
        assert ei.value.code == sor3d.SOR3D_EINVAL
    finally:
        sor3d.sor3d_destroy(h)


def test_deterministic_residual():
    p0, rhs = _case(150, 60, 20)
    a = gpu_sor(P, p0, rhs, 5, every=1)[1]
    b = gpu_sor(P, p0, rhs, 5, every=1)[1]
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("rows", [16, 32])
def test_cta_rows_variants(rows, monkeypatch):
    """Both CTA shapes (64 x 16 and 64 x 32 extended tiles) are bitwise."""
    monkeypatch.setenv("SOR3D_ROWS", str(rows))
    p0, rhs = _case(131, 45, 17)
    want, wh = oracle.sor_run(P, p0, rhs, 5, history=True)
    got, gh, _, plan = gpu_sor(P, p0, rhs, 5, every=1)
    assert f"64x{rows}" in plan
    assert_bitwise(got, want, f"rows={rows}")
    check_hist(gh, wh)


def test_create_rejects_grids_beyond_32bit_offsets():
    """The kernel addresses its streams with 32-bit element offsets: padded
    arrays of 2^31 elements or more are refused before any allocation."""
    with pytest.raises(sor3d.Sor3dError) as ei:
        sor3d.sor3d_create(sor3d.make_params(2048, 2048, 2048))
    assert ei.value.code == sor3d.SOR3D_EINVAL
    assert "2^31" in str(ei.value)
