"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Element by element on the same seeded inputs (sw2d_inputs), at sizes the
oracle finishes in seconds that span several warp strips (120 columns),
several row segments and ragged tails; the full BASELINE sizes (C3 8192^2,
C5 16384^2 in bench.py's launch configuration) on sampled windows the oracle
computes exactly from the initial state, plus properties that hold at any
size.  The bar (north_star): fields within 1e-5 of max |field| after 100
steps — we require bitwise (same operation order, no FMA) —
reductions 1e-5 relative (max/min/count exact), wet masks bit-exact.
"""
import numpy as np
import pytest

import oracle
import sw2d_inputs as si
from paper_1711_04471_b200 import sw2d
from _parity import assert_state_equal, check_reductions, gpu_run, oracle_run

pytestmark = pytest.mark.gpu

P = dict(si.PARAMS)
ALL = (1 << sw2d.SW2D_RED_N) - 1


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    sw2d.load()


def _bowl(nx, ny, seed=3, sigma=None):
    cfg = dict(si.config("c3"), nx=nx, ny=ny, seed=seed,
               sigma=sigma if sigma else max(2.0, min(nx, ny) / 16))
    return cfg, si.generate(cfg)


# --- full-field parity at oracle-sized grids ------------------------------

@pytest.mark.parametrize("nsteps", [1, 100, 1000])
def test_c1_bitwise(nsteps):
    cfg = si.config("c1")
    st = si.generate(cfg)
    want = oracle_run(P, st, nsteps)
    got, _, red, _ = gpu_run(P, st, nsteps)
    assert_state_equal(got, want, where=f"C1 after {nsteps} steps")
    check_reductions(red, oracle.reduce(P, st[0], *want[:3]))


@pytest.mark.parametrize("nx,ny", [(517, 389), (241, 600), (120, 121), (1000, 37)])
def test_wetdry_bowl_bitwise_ragged(nx, ny):
    """Several 120-column strips with a ragged last strip, several row
    segments with a ragged last one, shorelines and islands."""
    cfg, st = _bowl(nx, ny)
    want = oracle_run(P, st, 100)
    got, _, red, _ = gpu_run(P, st, 100)
    assert_state_equal(got, want, where=f"bowl {nx}x{ny}, 100 steps")
    check_reductions(red, oracle.reduce(P, st[0], *want[:3]))


def test_c2_paper_shape_bitwise():
    cfg = si.config("c2")
    st = si.generate(cfg)
    want = oracle_run(P, st, 100)
    got, _, _, _ = gpu_run(P, st, 100)
    assert_state_equal(got, want, where="C2 500x500, 100 steps")


@pytest.mark.parametrize("nx,ny", [(1, 1), (1, 9), (9, 1), (2, 3), (3, 3), (4, 4),
                                   (5, 130), (119, 2), (121, 8), (240, 17)])
def test_degenerate_and_tiny_grids(nx, ny):
    rng = np.random.default_rng(nx * 1000 + ny)
    hz = rng.uniform(-1.0, 3.0, (ny, nx)).astype(np.float32)
    e = np.where(hz < 0, -hz, rng.uniform(-0.2, 0.4, (ny, nx))).astype(np.float32)
    u = rng.uniform(-0.3, 0.3, (ny, nx)).astype(np.float32)
    v = rng.uniform(-0.3, 0.3, (ny, nx)).astype(np.float32)
    st = (hz, e, u, v)
    want = oracle_run(P, st, 25)
    got, _, red, _ = gpu_run(P, st, 25)
    assert_state_equal(got, want, where=f"random {nx}x{ny}")
    check_reductions(red, oracle.reduce(P, hz, *want[:3]))


def test_golden_examples_through_the_abi():
    """The hand-computed 3x3 example (tests/golden) on the GPU."""
    hz = np.full((3, 3), 10.0, np.float32)
    e = np.zeros((3, 3), np.float32)
    e[1, 1] = 1.0
    z = np.zeros_like(hz)
    got, _, _, _ = gpu_run(P, (hz, e, z, z), 1)
    assert abs(float(got[0][1, 1]) - 0.90953375) < 1e-6
    assert abs(float(got[0][0, 1]) - 0.0223467875) < 1e-7
    assert abs(float(got[1][1, 1]) - 0.0981) < 1e-7


def test_lake_at_rest_bitwise_gpu():
    rng = np.random.default_rng(5)
    hz = rng.uniform(-2.0, 10.0, (300, 257)).astype(np.float32)
    hz[rng.random(hz.shape) < 0.1] = np.float32(0.02)
    hz[5, 7] = np.float32(P["hmin"])
    e = (-np.minimum(np.float32(0.0), hz)).astype(np.float32)
    z = np.zeros_like(hz)
    got, _, _, _ = gpu_run(P, (hz, e, z, z), 500)
    np.testing.assert_array_equal(got[0], e)
    assert np.all(got[1] == 0) and np.all(got[2] == 0)


# --- chunking, determinism, reductions ------------------------------------

def test_step_chunking_is_invisible():
    cfg, st = _bowl(300, 250)
    a, _, _, _ = gpu_run(P, st, 60)
    b, _, _, _ = gpu_run(P, st, 60, chunks=[1, 7, 0, 22, 30])
    assert_state_equal(a, b, where="chunked vs one call")


def test_determinism_run_to_run():
    cfg, st = _bowl(700, 333)
    a, ha, ra, _ = gpu_run(P, st, 50, reduce_mask=ALL)
    b, hb, rb, _ = gpu_run(P, st, 50, reduce_mask=ALL)
    assert_state_equal(a, b, where="run twice")
    for op in ha:
        np.testing.assert_array_equal(ha[op], hb[op])
    assert ra == rb


@pytest.mark.parametrize("mask", [ALL, 1 << sw2d.SW2D_RED_VOLUME,
                                  (1 << sw2d.SW2D_RED_MAX_ABS_U) | (1 << sw2d.SW2D_RED_WET_COUNT)])
def test_fused_per_step_reductions(mask):
    """The fused epilogue's per-step diagnostics against the oracle's
    per-step history (sums 1e-5 relative; max/min/count exact); fields stay
    bitwise whatever the reduction level."""
    cfg, st = _bowl(389, 277)
    want = oracle_run(P, st, 40, history=True)
    got, hist, _, _ = gpu_run(P, st, 40, reduce_mask=mask)
    assert_state_equal(got, want[:4], where="with fused reductions")
    ohist = want[4]
    for op, series in hist.items():
        for n in range(40):
            row = np.zeros(oracle.NRED)
            row[op] = series[n]
            ref = np.zeros(oracle.NRED)
            ref[op] = ohist[n, op]
            check_reductions(row, ref)


# --- virtual ranks: the multi-GPU decomposition on one device -------------

@pytest.mark.parametrize("halo", [sw2d.SW2D_HALO_NCCL, sw2d.SW2D_HALO_P2P])
@pytest.mark.parametrize("nranks", [2, 3, 5, 8])
def test_virtual_ranks_bitwise_equal_single(nranks, halo):
    """Row slabs with a 2-row halo exchanged every step reproduce the
    single-slab result bitwise (the per-cell arithmetic does not depend on
    the slab), and the decomposed diagnostics agree.  HALO_NCCL moves the
    halos with device copies between steps (the NCCL path's plan); HALO_P2P
    has the boundary launches store their rows straight into the neighbour
    slabs (the fused path real ranks run over NVLink)."""
    cfg, st = _bowl(263, 97)
    one, h1, r1, _ = gpu_run(P, st, 80, reduce_mask=ALL)
    many, hm, rm, _ = gpu_run(P, st, 80, reduce_mask=ALL,
                              dist=sw2d.make_dist(0, nranks, virtual_ranks=1, halo_mode=halo))
    assert_state_equal(many, one, where=f"{nranks} virtual ranks")
    want = oracle_run(P, st, 80)
    assert_state_equal(many, want, where=f"{nranks} virtual ranks vs oracle")
    check_reductions(rm, r1)


# --- error contract --------------------------------------------------------

def test_status_codes():
    p = sw2d.make_params(16, 16)
    h = sw2d.sw2d_create(p)
    try:
        with pytest.raises(sw2d.Sw2dError) as ei:
            sw2d.sw2d_step(h, 1)
        assert ei.value.code == sw2d.SW2D_ESTATE
        with pytest.raises(sw2d.Sw2dError) as ei:
            sw2d.sw2d_reduce(h, 0)
        assert ei.value.code == sw2d.SW2D_ESTATE
        hz = np.full((16, 16), 10.0, np.float32)
        e = np.zeros_like(hz)
        e[3, 4] = np.nan
        with pytest.raises(sw2d.Sw2dError) as ei:
            sw2d.sw2d_set_state(h, hz, e)
        assert ei.value.code == sw2d.SW2D_EINVAL
        e[3, 4] = 0.0
        sw2d.sw2d_set_state(h, hz, e)          # recovers: EINVAL is not sticky
        sw2d.sw2d_step(h, 3)
        with pytest.raises(sw2d.Sw2dError) as ei:
            sw2d.sw2d_reduce_history(h, 0, 1)  # op not in reduce_every_step
        assert ei.value.code == sw2d.SW2D_EINVAL
        with pytest.raises(sw2d.Sw2dError):
            sw2d.sw2d_step(h, -1)
    finally:
        sw2d.sw2d_destroy(h)
    with pytest.raises(sw2d.Sw2dError) as ei:
        sw2d.sw2d_create(sw2d.make_params(16, 15), sw2d.make_dist(0, 2, virtual_ranks=1))
    assert ei.value.code == sw2d.SW2D_EINVAL


def test_wall_faces_ignored_on_input_and_zero_on_output():
    cfg, st = _bowl(130, 60)
    hz, e, u, v = [a.copy() for a in st]
    u[:, -1] = 5.0     # east wall faces
    v[-1, :] = -5.0    # north wall faces
    got, _, _, _ = gpu_run(P, (hz, e, u, v), 0)
    assert np.all(got[1][:, -1] == 0) and np.all(got[2][-1, :] == 0)
    want = oracle_run(P, (hz, e, u, v), 10)
    got, _, _, _ = gpu_run(P, (hz, e, u, v), 10)
    assert_state_equal(got, want, where="wall faces on input")


def test_torch_device_buffers():
    """set/get state from CUDA tensors (UVA) equals the host path."""
    import torch
    cfg, st = _bowl(200, 150)
    dev = [torch.from_numpy(a).cuda() for a in st]
    p = sw2d.make_params(200, 150)
    h = sw2d.sw2d_create(p, None, torch.cuda.current_stream())
    try:
        sw2d.sw2d_set_state(h, *dev)
        sw2d.sw2d_step(h, 30)
        out = [torch.empty_like(dev[0]) for _ in range(3)]
        sw2d.sw2d_get_state(h, *out)
        torch.cuda.synchronize()
    finally:
        sw2d.sw2d_destroy(h)
    want = oracle_run(P, st, 30)
    assert_state_equal([o.cpu().numpy() for o in out] + [None], want, where="torch buffers")


# --- full BASELINE sizes: sampled windows + properties ---------------------

def _window_parity(cfg, got, nsteps, centers, size=48):
    """Oracle on windows of the initial state with a margin of 2*nsteps+2
    cells (the step's dependency cone is 2 cells per step; cells farther than
    that from a window edge that is not a real wall are exact)."""
    nx, ny = cfg["nx"], cfg["ny"]
    m = 2 * nsteps + 2
    for (jc, kc) in centers:
        j0 = min(max(jc - size // 2, 0), ny - size)
        k0 = min(max(kc - size // 2, 0), nx - size)
        wj0, wk0 = max(j0 - m, 0), max(k0 - m, 0)
        wj1, wk1 = min(j0 + size + m, ny), min(k0 + size + m, nx)
        st = si.generate(cfg, j0=wj0, nrows=wj1 - wj0, k0=wk0, ncols=wk1 - wk0)
        want = oracle_run(P, st, nsteps)
        sl = (slice(j0 - wj0, j0 - wj0 + size), slice(k0 - wk0, k0 - wk0 + size))
        sub = [g[j0:j0 + size, k0:k0 + size] for g in got]
        assert_state_equal(sub, [w[sl] for w in want],
                           where=f"window at ({j0},{k0}) after {nsteps} steps")


def _full_size_run(cfg, nsteps, mask):
    nx, ny = cfg["nx"], cfg["ny"]
    st = si.generate(cfg)
    p = sw2d.make_params(nx, ny, reduce_every_step=mask, history_len=nsteps)
    h = sw2d.sw2d_create(p)
    try:
        sw2d.sw2d_set_state(h, *st)
        v0 = sw2d.sw2d_reduce(h, sw2d.SW2D_RED_VOLUME)
        sw2d.sw2d_step(h, nsteps)
        got = sw2d.get_state(h, nx)
        hist = sw2d.sw2d_reduce_history(h, sw2d.SW2D_RED_VOLUME, nsteps) if mask else None
        red = [sw2d.sw2d_reduce(h, op) for op in range(sw2d.SW2D_RED_N)]
    finally:
        sw2d.sw2d_destroy(h)
    return st, got, v0, hist, red


def _sample_centers(cfg, got):
    nx, ny = cfg["nx"], cfg["ny"]
    e = got[0]
    # corners, edge midpoints, centre, the bump peak, a shoreline cell
    w = got[3]
    shore = np.argwhere(w[ny // 2, :-1] != w[ny // 2, 1:])
    sk = int(shore[0][0]) if len(shore) else nx // 3
    peak = np.unravel_index(np.argmax(np.abs(e)), e.shape)
    return [(0, 0), (0, nx - 1), (ny - 1, 0), (ny - 1, nx - 1), (ny // 2, 0),
            (0, nx // 2), (ny // 2, nx // 2), (int(peak[0]), int(peak[1])), (ny // 2, sk)]


def test_c3_full_size_sampled_parity():
    cfg = si.config("c3")
    n = 100
    st, got, v0, _, red = _full_size_run(cfg, n, 0)
    _window_parity(cfg, got, n, _sample_centers(cfg, got))
    assert abs(red[sw2d.SW2D_RED_VOLUME] - v0) <= 1e-6 * v0


def test_c5_bench_configuration_sampled_parity():
    """bench.py's launch configuration: C5 16384^2 on one GPU with the
    per-step VOLUME reduction fused."""
    cfg = si.config("c5", 1)
    n = 30
    st, got, v0, hist, red = _full_size_run(cfg, n, 1 << sw2d.SW2D_RED_VOLUME)
    _window_parity(cfg, got, n, _sample_centers(cfg, got), size=32)
    assert np.max(np.abs(hist - v0)) <= 1e-6 * v0
    # fused (per-quad fp32 partials, then fp64) vs standalone (fp64 per cell)
    # VOLUME: measured 2e-9 apart on C5; the north_star bar for sums is 1e-5
    assert abs(hist[-1] - red[sw2d.SW2D_RED_VOLUME]) <= 1e-7 * v0


# --- the paper-shaped unfused variant (NEXT-1): same parity bar ------------

@pytest.mark.parametrize("nx,ny,n", [(100, 100, 100), (517, 389, 100), (1, 9, 25), (9, 1, 25),
                                     (3, 3, 1)])
def test_paper_variant_bitwise(nx, ny, n):
    if (nx, ny) == (100, 100):
        st = si.generate(si.config("c1"))
    else:
        st = _bowl(nx, ny)[1] if min(nx, ny) > 8 else _random_state(nx, ny)
    want = oracle_run(P, st, n, history=True)
    got, hist, red, launches = gpu_run(P, st, n, reduce_mask=ALL,
                                       variant=sw2d.SW2D_VARIANT_PAPER)
    assert_state_equal(got, want[:4], where=f"paper variant {nx}x{ny}")
    check_reductions(red, oracle.reduce(P, st[0], *want[:3]))
    for op, series in hist.items():
        for k in range(n):
            row = np.zeros(oracle.NRED)
            row[op] = series[k]
            ref = np.zeros(oracle.NRED)
            ref[op] = want[4][k, op]
            check_reductions(row, ref)
    assert launches >= 3 * n


def test_paper_variant_rejects_ranks():
    with pytest.raises(sw2d.Sw2dError) as ei:
        sw2d.sw2d_create(sw2d.make_params(64, 64, variant=sw2d.SW2D_VARIANT_PAPER),
                         sw2d.make_dist(0, 2, virtual_ranks=1))
    assert ei.value.code == sw2d.SW2D_EUNSUPPORTED


def _random_state(nx, ny):
    rng = np.random.default_rng(nx * 7919 + ny)
    hz = rng.uniform(-1.0, 3.0, (ny, nx)).astype(np.float32)
    e = np.where(hz < 0, -hz, rng.uniform(-0.2, 0.4, (ny, nx))).astype(np.float32)
    u = rng.uniform(-0.3, 0.3, (ny, nx)).astype(np.float32)
    v = rng.uniform(-0.3, 0.3, (ny, nx)).astype(np.float32)
    return hz, e, u, v


def test_c4_max_size_single_gpu_sampled_parity():
    """The largest BASELINE grid, C4 32768^2 (30 GB of state), on one GPU:
    inputs built on the device chunk by chunk, state uploaded from CUDA
    memory (UVA), sampled windows checked against the oracle."""
    import torch
    cfg = si.config("c4")
    nx, ny, n = cfg["nx"], cfg["ny"], 6
    dev = [torch.empty((ny, nx), dtype=torch.float32, device="cuda") for _ in range(4)]
    step = 2048
    for j0 in range(0, ny, step):
        part = si.generate(cfg, j0=j0, nrows=min(step, ny - j0))
        for d, a in zip(dev, part):
            d[j0:j0 + a.shape[0]].copy_(torch.from_numpy(a))
    p = sw2d.make_params(nx, ny)
    h = sw2d.sw2d_create(p, None, torch.cuda.current_stream())
    try:
        sw2d.sw2d_set_state(h, *dev)
        v0 = sw2d.sw2d_reduce(h, sw2d.SW2D_RED_VOLUME)
        sw2d.sw2d_step(h, n)
        out = [torch.empty_like(dev[0]) for _ in range(3)]
        wet = torch.empty((ny, nx), dtype=torch.uint8, device="cuda")
        sw2d.sw2d_get_state(h, *out, wet)
        v1 = sw2d.sw2d_reduce(h, sw2d.SW2D_RED_VOLUME)
    finally:
        sw2d.sw2d_destroy(h)
    del dev
    size, m = 32, 2 * n + 2
    centers = [(0, 0), (ny - 1, nx - 1), (ny // 2, nx // 2), (ny // 3, 2 * nx // 3),
               (0, nx // 2), (ny - 1, 17)]
    for (jc, kc) in centers:
        j0 = min(max(jc - size // 2, 0), ny - size)
        k0 = min(max(kc - size // 2, 0), nx - size)
        wj0, wk0 = max(j0 - m, 0), max(k0 - m, 0)
        wj1, wk1 = min(j0 + size + m, ny), min(k0 + size + m, nx)
        st = si.generate(cfg, j0=wj0, nrows=wj1 - wj0, k0=wk0, ncols=wk1 - wk0)
        want = oracle_run(P, st, n)
        sl = (slice(j0 - wj0, j0 - wj0 + size), slice(k0 - wk0, k0 - wk0 + size))
        sub = [t[j0:j0 + size, k0:k0 + size].cpu().numpy() for t in (*out, wet)]
        assert_state_equal(sub, [w[sl] for w in want], where=f"C4 window ({j0},{k0})")
    assert abs(v1 - v0) <= 1e-6 * v0


# --- periodic output (NEXT-3) ----------------------------------------------

@pytest.mark.parametrize("dist", [None, "virtual3"])
def test_snapshots_equal_oracle_states(dist):
    """sw2d_run_snapshots delivers eta after every `every` steps (copies
    overlapped with the following steps); each snapshot equals the oracle's
    state at that step bitwise, and the final state is that of nsteps."""
    import torch
    cfg, st = _bowl(301, 203)
    ny, nx = st[0].shape
    nsteps, every = 40, 7
    nsnap = nsteps // every
    out = torch.empty((nsnap, ny, nx), dtype=torch.float32, pin_memory=True)
    d = sw2d.make_dist(0, 3, virtual_ranks=1) if dist else None
    h = sw2d.sw2d_create(sw2d.make_params(nx, ny), d)
    try:
        sw2d.sw2d_set_state(h, *st)
        sw2d.sw2d_run_snapshots(h, nsteps, every, out)
        final = sw2d.get_state(h, nx)
    finally:
        sw2d.sw2d_destroy(h)
    cur = st
    for k in range(nsnap):
        e, u, v = oracle.run(P, cur[0], cur[1], cur[2], cur[3], every)
        cur = (cur[0], e, u, v)
        np.testing.assert_array_equal(out[k].numpy(), e)
    e, u, v = oracle.run(P, cur[0], cur[1], cur[2], cur[3], nsteps - nsnap * every)
    assert_state_equal(final[:3] + (None,), (e, u, v, None), where="after snapshots")


# --- kernel variants forced on oracle-sized grids --------------------------

@pytest.mark.parametrize("kind,two", [("1", "1"), ("1", "0"), ("2", "1"), ("2", "0")])
@pytest.mark.parametrize("nx,ny,n", [(517, 389, 41), (241, 600, 30), (120, 121, 7), (9, 13, 5),
                                     (57, 70, 9), (113, 33, 12)])
def test_kernel_kinds_bitwise(kind, two, nx, ny, n, monkeypatch):
    """Every step-kernel kind on the same grids (the size heuristic picks
    only one of them per grid): the CTA/TMA kernel with two steps per launch
    (and an odd step count), one step per launch, and the
    small-grid kernels with two steps (56-column strips: 57 and 113 columns
    end one column into a strip) and one step per launch — all bitwise equal
    to the oracle, with all fused per-step diagnostics."""
    monkeypatch.setenv("SW2D_STEP_KERNEL", kind)
    monkeypatch.setenv("SW2D_TWO_STEP", two)
    st = _bowl(nx, ny)[1] if min(nx, ny) > 8 else _random_state(nx, ny)
    want = oracle_run(P, st, n, history=True)
    got, hist, red, _ = gpu_run(P, st, n, reduce_mask=ALL)
    assert_state_equal(got, want[:4], where=f"kind {kind} two {two} {nx}x{ny}")
    check_reductions(red, oracle.reduce(P, st[0], *want[:3]))
    for op, series in hist.items():
        for k in range(n):
            row = np.zeros(oracle.NRED)
            row[op] = series[k]
            ref = np.zeros(oracle.NRED)
            ref[op] = want[4][k, op]
            check_reductions(row, ref)
    got2, _, _, _ = gpu_run(P, st, n, chunks=[1, n - 1])
    assert_state_equal(got2, want[:4], where=f"kind {kind} two {two} chunked")


@pytest.mark.parametrize("halo", [sw2d.SW2D_HALO_NCCL, sw2d.SW2D_HALO_P2P])
@pytest.mark.parametrize("two", ["1", "0"])
@pytest.mark.parametrize("nranks,n", [(2, 31), (3, 8), (5, 17)])
def test_virtual_ranks_kinds_bitwise(nranks, n, two, halo, monkeypatch):
    """Row slabs with the CTA kernel (forced), one or two steps per launch,
    NCCL-plan device copies or fused P2P halo stores: bitwise equal to the
    oracle, diagnostics folded over all slabs, odd step counts included."""
    monkeypatch.setenv("SW2D_STEP_KERNEL", "1")
    monkeypatch.setenv("SW2D_TWO_STEP", two)
    cfg, st = _bowl(263, 97)
    want = oracle_run(P, st, n, history=True)
    got, hist, red, _ = gpu_run(P, st, n, reduce_mask=ALL,
                                dist=sw2d.make_dist(0, nranks, virtual_ranks=1, halo_mode=halo))
    assert_state_equal(got, want[:4], where=f"{nranks} slabs two={two} halo={halo}")
    check_reductions(red, oracle.reduce(P, st[0], *want[:3]))
    for op, series in hist.items():
        for k in range(n):
            row = np.zeros(oracle.NRED)
            row[op] = series[k]
            ref = np.zeros(oracle.NRED)
            ref[op] = want[4][k, op]
            check_reductions(row, ref)


@pytest.mark.parametrize("kind", ["1", "2"])
def test_graph_replay_both_parities(kind, monkeypatch):
    """Long sw2d_step calls replay captured CUDA graphs (one per starting
    buffer parity); chunks that start on either parity and leave remainders
    equal the oracle bitwise."""
    monkeypatch.setenv("SW2D_STEP_KERNEL", kind)
    cfg, st = _bowl(300, 170)
    n = 1 + 64 + 129 + 70
    want = oracle_run(P, st, n)
    got, _, _, launches = gpu_run(P, st, n, chunks=[1, 64, 129, 70])
    assert_state_equal(got, want, where=f"graphs kind {kind}")


def _history_run(st, chunks, mask, history_len, dist=None):
    hz, e, u, v = st
    ny, nx = hz.shape
    p = sw2d.make_params(nx, ny, P["dx"], P["dy"], P["dt"], P["g"], P["eps"], P["hmin"],
                         reduce_every_step=mask, history_len=history_len)
    h = sw2d.sw2d_create(p, dist)
    try:
        sw2d.sw2d_set_state(h, hz, e, u, v)
        for n in chunks:
            sw2d.sw2d_step(h, n)
        out = sw2d.get_state(h, nx)
        k = min(sum(chunks), history_len)
        hist = {op: sw2d.sw2d_reduce_history(h, op, k)
                for op in range(sw2d.SW2D_RED_N) if mask & (1 << op)}
    finally:
        sw2d.sw2d_destroy(h)
    return out, hist


def _check_history(hist, want_hist, n):
    k = len(next(iter(hist.values())))
    for op, series in hist.items():
        for t in range(k):
            row = np.zeros(oracle.NRED)
            row[op] = series[t]
            ref = np.zeros(oracle.NRED)
            ref[op] = want_hist[n - k + t, op]
            check_reductions(row, ref)


@pytest.mark.parametrize("kind,history_len", [("1", 300), ("2", 300), ("2", 37), ("1", 64)])
def test_graph_replay_with_per_step_diagnostics(kind, history_len, monkeypatch):
    """Graphs also replay with per-step diagnostics: the history slot of each
    record is found on the device (a step counter that advances with the
    records), so every step's record lands in its ring slot — also when the
    ring wraps (history_len 37, 64) and chunks start on either parity."""
    monkeypatch.setenv("SW2D_STEP_KERNEL", kind)
    cfg, st = _bowl(300, 170)
    n = 1 + 64 + 129 + 70
    want = oracle_run(P, st, n, history=True)
    got, hist = _history_run(st, [1, 64, 129, 70], ALL, history_len)
    assert_state_equal(got, want[:4], where=f"graphs+diagnostics kind {kind}")
    _check_history(hist, want[4], n)


def test_graph_replay_diagnostics_virtual_ranks():
    """Three virtual slabs (several launches per step share one record) in
    replayed graphs with per-step diagnostics."""
    cfg, st = _bowl(250, 120)
    n = 2 + 64 + 66
    want = oracle_run(P, st, n, history=True)
    got, hist = _history_run(st, [2, 64, 66], ALL, 200,
                             dist=sw2d.make_dist(0, 3, virtual_ranks=1))
    assert_state_equal(got, want[:4], where="virtual ranks, graphs + diagnostics")
    _check_history(hist, want[4], n)


# --- tests of the tests: fault injection and mapping permutation -------------

def test_fault_injection_skipped_halo_fails_parity(monkeypatch):
    """SW2D_FAULT_SKIP_HALO drops one halo exchange between virtual slabs: the
    parity check must catch it (it would pass a checker that compares a slab
    only with itself)."""
    cfg, st = _bowl(240, 96)
    n = 12
    want = oracle_run(P, st, n)
    dist = sw2d.make_dist(0, 3, virtual_ranks=1)
    got, _, _, _ = gpu_run(P, st, n, dist=dist)
    assert_state_equal(got, want, where="no fault")
    monkeypatch.setenv("SW2D_FAULT_SKIP_HALO", "4")
    monkeypatch.setenv("SW2D_GRAPHS", "0")
    bad, _, _, _ = gpu_run(P, st, n, dist=dist)
    with pytest.raises(AssertionError):
        assert_state_equal(bad, want, where="skipped halo at step 4")


@pytest.mark.parametrize("env", [dict(SW2D_STEP_KERNEL="1", SW2D_MIN_ROWS="1"),
                                 dict(SW2D_STEP_KERNEL="1", SW2D_CTAS_PER_SM="1"),
                                 dict(SW2D_STEP_KERNEL="1", SW2D_MIN_ROWS="64"),
                                 dict(SW2D_STEP_KERNEL="2", SW2D_MIN_ROWS2="1"),
                                 dict(SW2D_STEP_KERNEL="2", SW2D_MIN_ROWS2="40"),
                                 dict(SW2D_STEP_KERNEL="1", SW2D_GRAPHS="0")])
def test_mapping_permutations_bitwise(env, monkeypatch):
    """Map soundness (SPEC's permutation check, adapted): other segmentations
    of the grid into CTAs/warps, and graphs off, give bitwise the same
    fields — every cell's arithmetic is independent of the mapping."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    cfg, st = _bowl(700, 300)
    want = oracle_run(P, st, 66)
    got, _, _, _ = gpu_run(P, st, 66)
    assert_state_equal(got, want, where=str(env))


@pytest.mark.parametrize("nx,ny,n,ctas", [(700, 300, 41, ""), (700, 300, 41, "23"),
                                          (2000, 389, 30, ""), (2000, 389, 7, "61"),
                                          (1921, 64, 12, "6"), (600, 9, 5, "")])
@pytest.mark.parametrize("mask", [ALL, 1 << sw2d.SW2D_RED_VOLUME, 0])
def test_even_split_bitwise(nx, ny, n, ctas, mask, monkeypatch):
    """The two-step kernel's even split of group-rows over CTAs (SW2D_SK=2
    forces it; the planner picks it on HBM-sized grids such as C3/C5): CTAs
    whose share spans two column groups of different widths, shares of a few
    rows, CTAs with no rows (600x9 over 148 CTAs) — bitwise equal to the
    oracle with all, one (VOLUME: the pipelined pair) or no per-step
    diagnostics, odd step counts included."""
    monkeypatch.setenv("SW2D_STEP_KERNEL", "1")
    monkeypatch.setenv("SW2D_SK", "2")
    if ctas:
        monkeypatch.setenv("SW2D_SK_CTAS", ctas)
    st = _bowl(nx, ny)[1]
    want = oracle_run(P, st, n, history=True)
    got, hist, red, _ = gpu_run(P, st, n, reduce_mask=mask)
    assert_state_equal(got, want[:4], where=f"even split {nx}x{ny} ctas {ctas or 'sms'}")
    check_reductions(red, oracle.reduce(P, st[0], *want[:3]))
    for op, series in (hist or {}).items():
        for k in range(n):
            row = np.zeros(oracle.NRED)
            row[op] = series[k]
            ref = np.zeros(oracle.NRED)
            ref[op] = want[4][k, op]
            check_reductions(row, ref)


@pytest.mark.parametrize("nx,ny,want", [(16384, 16384, "even-rows"), (8192, 8192, "even-rows"),
                                         (2000, 2000, "grid")])
def test_even_split_planner_choice(nx, ny, want):
    """The planner takes the even row split where it shortens the busiest
    CTA's rows (C5, C3: 20 / 10 column groups leave SMs idle in the group x
    segment grid) and keeps the grid where the split's extra streamed rows
    would cost more (2000^2: 3 groups, ~40 rows per CTA)."""
    h = sw2d.sw2d_create(sw2d.make_params(nx, ny), None)
    try:
        assert ("split=%s" % want) in sw2d.sw2d_plan(h), sw2d.sw2d_plan(h)
        if want == "even-rows":
            import torch
            sms = torch.cuda.get_device_properties(0).multi_processor_count
            assert ("split=even-rows:%d" % sms) in sw2d.sw2d_plan(h), sw2d.sw2d_plan(h)
    finally:
        sw2d.sw2d_destroy(h)


def test_even_split_uses_every_sm_with_real_ranks(monkeypatch):
    """With real ranks (here the NCCL machinery forced on one rank) the even
    split still uses one CTA per SM on every SM: the bands follow the
    interior launch and the NCCL exchange kernels run on a highest-priority
    stream (the 4 reserved SMs cost 2.7% on every rank)."""
    import torch
    monkeypatch.setenv("SW2D_FORCE_NCCL", "1")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    uid = sw2d.sw2d_nccl_unique_id()
    h = sw2d.sw2d_create(sw2d.make_params(16384, 16384), sw2d.make_dist(0, 1, 0, 0, uid))
    try:
        assert ("split=even-rows:%d" % sms) in sw2d.sw2d_plan(h), sw2d.sw2d_plan(h)
    finally:
        sw2d.sw2d_destroy(h)


@pytest.mark.parametrize("halo", [sw2d.SW2D_HALO_NCCL, sw2d.SW2D_HALO_P2P])
def test_even_split_virtual_ranks_bitwise(halo, monkeypatch):
    """Even split inside each slab's interior launch, with the halo-band
    launches of three virtual ranks (NCCL-plan copies or P2P stores)."""
    monkeypatch.setenv("SW2D_STEP_KERNEL", "1")
    monkeypatch.setenv("SW2D_SK", "2")
    monkeypatch.setenv("SW2D_GRAPHS", "0")
    st = _bowl(700, 300)[1]
    want = oracle_run(P, st, 19)
    got, _, _, _ = gpu_run(P, st, 19, dist=sw2d.make_dist(0, 3, 0, 1, halo_mode=halo))
    assert_state_equal(got, want, where=f"even split, 3 virtual ranks, halo {halo}")


@pytest.mark.parametrize("halo", [sw2d.SW2D_HALO_NCCL, sw2d.SW2D_HALO_P2P])
@pytest.mark.parametrize("history_len", [1, 3, 0])
def test_single_rank_nccl_machinery(halo, history_len, monkeypatch):
    """One real rank with the NCCL path forced on (SW2D_FORCE_NCCL): the
    library's NCCL communicator, comm stream, grouped halo exchange (no
    peers), the per-step records' out-of-place allreduce (NCCL mode) or slot
    exchange (P2P mode, here with itself) and, in P2P mode, the blob
    all-gather all run on the GPU; fields stay bitwise and every kept
    per-step record equals the oracle's — also with history rings shorter
    than the run (1 and 3 records for 23 steps: ADVICE r01 #1) and over 150
    steps (the 64-record exchange ring wraps).  Real ranks sharing the GPU:
    tests/test_gpu_p2p_procs.py."""
    monkeypatch.setenv("SW2D_FORCE_NCCL", "1")
    cfg, st = _bowl(300, 200)
    hz, e, u, v = st
    uid = sw2d.sw2d_nccl_unique_id()
    p = sw2d.make_params(300, 200, P["dx"], P["dy"], P["dt"], P["g"], P["eps"], P["hmin"],
                         reduce_every_step=ALL, history_len=history_len)
    h = sw2d.sw2d_create(p, sw2d.make_dist(0, 1, 0, 0, uid, halo))
    try:
        for chunks in ([23], [7, 1, 80, 62]):
            n = sum(chunks)
            want = oracle_run(P, st, n, history=True)
            sw2d.sw2d_set_state(h, hz, e, u, v)
            for c in chunks:
                sw2d.sw2d_step(h, c)
            got = sw2d.get_state(h, 300)
            keep = min(n, history_len or 1024)
            hist = {op: sw2d.sw2d_reduce_history(h, op, keep) for op in range(sw2d.SW2D_RED_N)}
            red = [sw2d.sw2d_reduce(h, op) for op in range(sw2d.SW2D_RED_N)]
            assert_state_equal(got, want[:4], where=f"forced NCCL, halo {halo}, {chunks}")
            check_reductions(red, oracle.reduce(P, st[0], *want[:3]))
            for k in range(keep):
                check_reductions([hist[op][k] for op in range(sw2d.SW2D_RED_N)],
                                 want[4][n - keep + k])
    finally:
        sw2d.sw2d_destroy(h)


def test_legacy_default_stream_long_run():
    """A handle on the legacy default stream (binding: stream=0) takes long
    sw2d_step calls without graph capture (that stream cannot be captured)."""
    cfg, st = _bowl(200, 150)
    hz, e, u, v = st
    n = 130
    want = oracle_run(P, st, n)
    p = sw2d.make_params(200, 150, P["dx"], P["dy"], P["dt"], P["g"], P["eps"], P["hmin"],
                         reduce_every_step=1 << sw2d.SW2D_RED_VOLUME, history_len=n)
    h = sw2d.sw2d_create(p, None, 0)
    try:
        sw2d.sw2d_set_state(h, hz, e, u, v)
        sw2d.sw2d_step(h, n)
        got = sw2d.get_state(h, 200)
    finally:
        sw2d.sw2d_destroy(h)
    assert_state_equal(got, want, where="legacy stream")


# --- persistent cooperative kernel for the paper's small grids (NEXT-2) ------

@pytest.mark.parametrize("k", ["1", "2", "3", "4"])
@pytest.mark.parametrize("nx,ny,n,shape", [(100, 100, 100, None), (500, 500, 100, None),
                                           (263, 97, 51, "0"), (57, 300, 20, "1"),
                                           (1, 9, 25, None), (9, 1, 25, None), (3, 3, 7, None),
                                           (1000, 1000, 16, None), (130, 61, 33, "2"),
                                           (700, 90, 12, "3"), (333, 140, 17, "4"),
                                           (200, 257, 22, "5")])
def test_persistent_kernel_bitwise(nx, ny, n, shape, k, monkeypatch):
    """One cooperative launch advances the whole grid: every CTA keeps its
    tile in shared memory, K steps per block, neighbour tiles synchronised by
    per-tile counters (no grid barrier, no relaunch).  Bitwise equal to the
    oracle on ragged grids and degenerate ones, with all per-step
    diagnostics (deferred fold), chunked calls continuing the counters."""
    monkeypatch.setenv("SW2D_PERSIST", "1")
    monkeypatch.setenv("SW2D_PERSIST_K", k)
    if shape:
        if k in ("3", "4") and shape in ("0", "3"):
            pytest.skip("K = 3, 4: 16 shared rows leave a tile shorter than its apron")
        monkeypatch.setenv("SW2D_PERSIST_SHAPE", shape)
    h = sw2d.sw2d_create(sw2d.make_params(nx, ny, reduce_every_step=ALL, history_len=n))
    try:   # the persistent kernel with K steps per block is what runs (1000^2:
        # more tiles than co-resident CTAs, the planner falls back to the row march)
        plan = sw2d.sw2d_plan(h)
        if nx * ny <= 500 * 500:
            assert "kernel=persist steps_per_block=%s " % k in plan, plan
        else:
            assert "kernel=persist" not in plan or "steps_per_block=%s " % k in plan, plan
    finally:
        sw2d.sw2d_destroy(h)
    st = (si.generate(si.config("c1")) if (nx, ny) == (100, 100) else
          si.generate(si.config("c2")) if (nx, ny) == (500, 500) else
          _bowl(nx, ny)[1] if min(nx, ny) > 8 else _random_state(nx, ny))
    want = oracle_run(P, st, n, history=True)
    got, hist, red, launches = gpu_run(P, st, n, reduce_mask=ALL)
    assert_state_equal(got, want[:4], where=f"persistent K={k} {nx}x{ny}")
    check_reductions(red, oracle.reduce(P, st[0], *want[:3]))
    _check_history(hist, want[4], n)
    got2, _, _, _ = gpu_run(P, st, n, chunks=[1, n // 2, n - 1 - n // 2])
    assert_state_equal(got2, want[:4], where=f"persistent K={k} chunked")


def test_persistent_kernel_is_the_small_grid_plan(monkeypatch):
    """With SW2D_PERSIST=1 the planner picks the persistent kernel for the
    paper's sizes on one GPU without ranks, the row-march kernels otherwise."""
    monkeypatch.setenv("SW2D_PERSIST", "1")
    h = sw2d.sw2d_create(sw2d.make_params(500, 500))
    try:
        assert "kernel=persist" in sw2d.sw2d_plan(h), sw2d.sw2d_plan(h)
    finally:
        sw2d.sw2d_destroy(h)
    for dist in (sw2d.make_dist(0, 2, virtual_ranks=1), None):
        nx = 500 if dist is not None else 8192
        h = sw2d.sw2d_create(sw2d.make_params(nx, 500), dist)
        try:
            assert "kernel=persist" not in sw2d.sw2d_plan(h), sw2d.sw2d_plan(h)
        finally:
            sw2d.sw2d_destroy(h)


@pytest.mark.parametrize("history_len", [1, 37, 300])
def test_persistent_kernel_long_run_history(history_len, monkeypatch):
    """C2-shaped run over several red chunks (64 steps per launch with
    diagnostics) with the ring shorter and longer than the run."""
    monkeypatch.setenv("SW2D_PERSIST", "1")
    st = si.generate(si.config("c2"))
    n = 257
    want = oracle_run(P, st, n, history=True)
    got, hist = _history_run(st, [3, 254], ALL, history_len)
    assert_state_equal(got, want[:4], where=f"persistent long run, history {history_len}")
    _check_history(hist, want[4], n)


def test_persistent_kernels_of_two_handles_interleave_safely():
    """Two small-grid handles on their own streams, stepped back to back
    without synchronisation: their persistent launches are ordered (one
    device-wide event), so neither waits on CTAs the other keeps from
    starting; both equal the oracle."""
    st = si.generate(si.config("c1"))
    want = oracle_run(P, st, 150)
    hs = []
    try:
        for _ in range(2):
            h = sw2d.sw2d_create(sw2d.make_params(100, 100, reduce_every_step=1, history_len=8))
            assert "kernel=persist" in sw2d.sw2d_plan(h), sw2d.sw2d_plan(h)
            sw2d.sw2d_set_state(h, *st)
            hs.append(h)
        for chunk in (64, 86):
            for h in hs:
                sw2d.sw2d_step(h, chunk)
        for h in hs:
            assert_state_equal(sw2d.get_state(h, 100), want, where="two handles")
    finally:
        for h in hs:
            sw2d.sw2d_destroy(h)


@pytest.mark.parametrize("rows", ["2", "5", "6", "7", "8", "11", "13"])
@pytest.mark.parametrize("mask", [ALL, 0])
def test_interior_row_loop_segment_lengths(rows, mask, monkeypatch):
    """The two-step kernel runs a segment's first rows and last rows with the
    row tests and the rows between without them (interior row
    loop): segments of 2 .. 13 output rows put every transition (no interior,
    one iteration of it, tails of 0-2 rows) at many places of the grid,
    including the north / south walls — bitwise equal to the oracle, with and
    without the per-step diagnostics."""
    monkeypatch.setenv("SW2D_STEP_KERNEL", "1")
    monkeypatch.setenv("SW2D_SK", "0")
    monkeypatch.setenv("SW2D_MIN_ROWS", rows)
    st = _bowl(250, 257)[1]
    n = 20
    want = oracle_run(P, st, n, history=True)
    got, hist, red, _ = gpu_run(P, st, n, reduce_mask=mask)
    assert_state_equal(got, want[:4], where=f"segments of {rows} rows")
    if mask:
        check_reductions(red, oracle.reduce(P, st[0], *want[:3]))
        _check_history(hist, want[4], n)


@pytest.mark.parametrize("tag", ["0", "1"])
@pytest.mark.parametrize("nx,ny,n,k,shape", [(100, 100, 61, "2", None), (500, 500, 40, "3", None),
                                             (263, 97, 51, "2", "0"), (333, 140, 17, "3", "4"),
                                             (130, 61, 33, "1", "2"), (3, 3, 7, "2", None)])
def test_persistent_kernel_handshakes_bitwise(nx, ny, n, k, shape, tag, monkeypatch):
    """Both handshakes between the persistent kernel's tiles — per-tile step
    counters, and the ring as tagged 8-byte words polled directly (the
    default where every SM holds one CTA) — forced on plans of one and of
    several CTAs per SM: bitwise equal to the oracle with all diagnostics,
    over chunked calls (the tags continue across launches)."""
    monkeypatch.setenv("SW2D_PERSIST", "1")
    monkeypatch.setenv("SW2D_PERSIST_K", k)
    monkeypatch.setenv("SW2D_PERSIST_TAGGED", tag)
    if shape:
        monkeypatch.setenv("SW2D_PERSIST_SHAPE", shape)
    h = sw2d.sw2d_create(sw2d.make_params(nx, ny, reduce_every_step=ALL, history_len=n))
    try:
        plan = sw2d.sw2d_plan(h)
        assert "kernel=persist" in plan, plan
        assert ("handshake=tagged" if tag == "1" else "handshake=counters") in plan, plan
    finally:
        sw2d.sw2d_destroy(h)
    st = (si.generate(si.config("c1")) if (nx, ny) == (100, 100) else
          si.generate(si.config("c2")) if (nx, ny) == (500, 500) else
          _bowl(nx, ny)[1] if min(nx, ny) > 8 else _random_state(nx, ny))
    want = oracle_run(P, st, n, history=True)
    got, hist, red, _ = gpu_run(P, st, n, reduce_mask=ALL, chunks=[1, n // 2, n - 1 - n // 2])
    assert_state_equal(got, want[:4], where=f"persistent K={k} handshake {tag} {nx}x{ny}")
    check_reductions(red, oracle.reduce(P, st[0], *want[:3]))
    _check_history(hist, want[4], n)
