"""Pins of the NEXT-4 oracle (oracle/sor_ref.c): red-black SOR for the Poisson
equation, the UFLES "press" solver of arXiv 1711.04471 §6.3 (PAPER.md:399-401,
418, 427-428).  The paper prints no equations or values; the pins are a
hand-computed example (tests/golden/), the exact discrete solution of small
systems (dense linear algebra), the second-order convergence of a
manufactured solution, an exact residual of a polynomial state and the
Gauss-Seidel property of the red-black ordering."""
import math
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
P1 = dict(dx=1.0, dy=1.0, dz=1.0, omega=1.5)


def _golden(name):
    vals = {}
    for line in open(os.path.join(GOLDEN, name)):
        line = line.split("#")[0].split()
        if line:
            vals[line[0]] = [float(x) for x in line[1:]]
    return vals


def test_golden_3x1x1_two_iterations():
    """Hand computation: red cell i=2 then black cells i=1,3, twice, and the
    residual after the first iteration (catches a wrong colour, ordering,
    relaxation form, stencil weight or residual sign)."""
    g = _golden("golden_sor_3x1x1.txt")
    rhs = np.array(g["rhs"], np.float32).reshape(1, 1, 3)
    p0 = np.zeros_like(rhs)
    p1, h1 = oracle.sor_run(P1, p0, rhs, 1, history=True)
    np.testing.assert_allclose(p1.ravel(), g["p_after_1"], rtol=1e-6)
    np.testing.assert_allclose(h1[0], [g["residual_after_1"][0], g["residual_after_1"][1]],
                               rtol=1e-6)
    p2 = oracle.sor_run(P1, p0, rhs, 2)
    np.testing.assert_allclose(p2.ravel(), g["p_after_2"], rtol=1e-6)


def _dense_laplacian(nx, ny, nz, dx, dy, dz):
    n = nx * ny * nz
    A = np.zeros((n, n))
    idx = lambda k, j, i: (k * ny + j) * nx + i  # noqa: E731
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                r = idx(k, j, i)
                A[r, r] = -2 / dx**2 - 2 / dy**2 - 2 / dz**2
                for (dk, dj, di, h) in ((0, 0, 1, dx), (0, 0, -1, dx), (0, 1, 0, dy),
                                        (0, -1, 0, dy), (1, 0, 0, dz), (-1, 0, 0, dz)):
                    kk, jj, ii = k + dk, j + dj, i + di
                    if 0 <= kk < nz and 0 <= jj < ny and 0 <= ii < nx:
                        A[r, idx(kk, jj, ii)] = 1 / h**2
    return A


@pytest.mark.parametrize("omega", [1.0, 1.5, 1.8])
def test_converges_to_exact_discrete_solution(omega):
    """SOR's fixed point is the solution of the discrete system (dense solve);
    anisotropic spacings (catches dx/dy/dz mix-ups)."""
    rng = np.random.default_rng(3)
    nx, ny, nz = 6, 5, 4
    p = dict(dx=1.0, dy=0.7, dz=1.3, omega=omega)
    rhs = rng.uniform(-1, 1, (nz, ny, nx)).astype(np.float32)
    A = _dense_laplacian(nx, ny, nz, p["dx"], p["dy"], p["dz"])
    exact = np.linalg.solve(A, rhs.astype(np.float64).ravel()).reshape(nz, ny, nx)
    got, hist = oracle.sor_run(p, np.zeros_like(rhs), rhs, 400, history=True)
    assert np.max(np.abs(got - exact)) <= 1e-4 * np.max(np.abs(exact))
    assert hist[-1, 0] < 1e-3 * hist[0, 0]


def test_manufactured_solution_second_order():
    """p* = sin(pi x/X) sin(pi y/Y) sin(pi z/Z) with its continuous Laplacian as
    rhs: the converged discrete solution errs by O(h^2) (ratio ~4 per halving)."""
    errs = []
    for n in (7, 15):
        X = 1.0
        h = X / (n + 1)
        p = dict(dx=h, dy=h, dz=h, omega=1.6)
        x = np.arange(1, n + 1) * h
        sx = np.sin(math.pi * x / X)
        star = np.einsum("k,j,i->kji", sx, sx, sx)
        rhs = (-3 * math.pi**2 * star).astype(np.float32)
        got = oracle.sor_run(p, np.zeros_like(rhs), rhs, 600)
        errs.append(np.max(np.abs(got - star)))
    ratio = errs[0] / errs[1]
    assert 3.0 < ratio < 5.0, (errs, ratio)


def test_residual_exact_for_a_polynomial():
    """The second difference of a quadratic is exact: for
    p = x(X-x) y(Y-y) z(Z-z), which vanishes on the ghost nodes, Lap(p) is known
    in closed form and the residual of rhs = Lap(p) is roundoff only (catches a
    wrong residual sign, diagonal term or weight)."""
    nx, ny, nz = 9, 7, 5
    dx, dy, dz = 0.5, 0.25, 1.0
    X, Y, Z = (nx + 1) * dx, (ny + 1) * dy, (nz + 1) * dz
    x = np.arange(1, nx + 1) * dx
    y = np.arange(1, ny + 1) * dy
    z = np.arange(1, nz + 1) * dz
    fx, fy, fz = x * (X - x), y * (Y - y), z * (Z - z)
    p = np.einsum("k,j,i->kji", fz, fy, fx)
    lap = -2 * (np.einsum("k,j,i->kji", fz, fy, np.ones(nx)) +
                np.einsum("k,j,i->kji", fz, np.ones(ny), fx) +
                np.einsum("k,j,i->kji", np.ones(nz), fy, fx))
    prm = dict(dx=dx, dy=dy, dz=dz, omega=1.0)
    l2, linf = oracle.sor_residual(prm, p.astype(np.float32), lap.astype(np.float32))
    assert linf <= 1e-5 * np.max(np.abs(lap)), linf
    l2w, _ = oracle.sor_residual(prm, p.astype(np.float32), (lap + 1.0).astype(np.float32))
    assert abs(l2w - math.sqrt(nx * ny * nz)) < 1e-3


def test_red_black_gauss_seidel_property():
    """With omega = 1 the black sweep solves every black cell's equation given
    its (red) neighbours: after one iteration the black cells' residual is
    roundoff, the red cells' is not."""
    rng = np.random.default_rng(9)
    nx, ny, nz = 8, 6, 5
    p = dict(dx=1.0, dy=1.0, dz=1.0, omega=1.0)
    rhs = rng.uniform(-1, 1, (nz, ny, nx)).astype(np.float32)
    got = oracle.sor_run(p, np.zeros_like(rhs), rhs, 1).astype(np.float64)
    pad = np.pad(got, 1)
    lap = (pad[1:-1, 1:-1, 2:] + pad[1:-1, 1:-1, :-2] + pad[1:-1, 2:, 1:-1] +
           pad[1:-1, :-2, 1:-1] + pad[2:, 1:-1, 1:-1] + pad[:-2, 1:-1, 1:-1] - 6 * got)
    r = rhs - lap
    kk, jj, ii = np.indices((nz, ny, nx)) + 1
    black = (kk + jj + ii) % 2 == 1
    assert np.max(np.abs(r[black])) < 1e-5
    assert np.max(np.abs(r[~black])) > 1e-2


def test_sor_inputs_are_pure_functions_of_index():
    """The shared input generator (no method arithmetic): any plane range
    equals the same planes of the full generation (so any slab can be made on
    its own), and the paper-shaped config has the stated shape."""
    import sor_inputs as so
    cfg = so.config("sor_s2")
    p0, rhs = so.generate(cfg)
    p1, r1 = so.generate(cfg, k0=13, nk=9)
    assert np.array_equal(p0[13:22], p1) and np.array_equal(rhs[13:22], r1)
    c = so.config("sor300")
    assert (c["nx"], c["ny"], c["nz"], c["iters"]) == (300, 300, 90, 50)
    assert np.all(np.isfinite(rhs)) and np.abs(p0).max() <= 0.01
