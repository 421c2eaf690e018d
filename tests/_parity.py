"""Parity helpers for the GPU tests: run both arms on the same seeded inputs
and report the first divergence (field, (j, k), both values)."""
from __future__ import annotations

import numpy as np

import oracle
from paper_1711_04471_b200 import sw2d

FIELDS = ("eta", "u", "v", "wet")


def first_divergence(name, got, want, tol_rel=0.0):
    """None if equal (values: +0 == -0; tol_rel relative to max |want|),
    else a one-line report of the first differing element."""
    got = np.asarray(got)
    want = np.asarray(want)
    assert got.shape == want.shape, (name, got.shape, want.shape)
    if tol_rel == 0.0:
        bad = got != want
    else:
        scale = max(float(np.max(np.abs(want))), 1e-30)
        bad = np.abs(got.astype(np.float64) - want.astype(np.float64)) > tol_rel * scale
    if not np.any(bad):
        return None
    j, k = np.argwhere(bad)[0]
    return (f"{name}: {int(bad.sum())} of {bad.size} differ; first at (j={j}, k={k}): "
            f"gpu={got[j, k]!r} oracle={want[j, k]!r}")


def assert_state_equal(got, want, tol_rel=0.0, where=""):
    msgs = []
    for name, g, w in zip(FIELDS, got, want):
        if g is None or w is None:
            continue
        m = first_divergence(name, g, w, 0.0 if name == "wet" else tol_rel)
        if m:
            msgs.append(m)
    assert not msgs, where + "\n" + "\n".join(msgs)


def oracle_run(params, state, nsteps, history=False):
    hz, e, u, v = state
    out = oracle.run(params, hz, e, u, v, nsteps, history=history)
    w = oracle.wet(params, hz, out[0])
    return (out[0], out[1], out[2], w) + ((out[3],) if history else ())


def gpu_run(params, state, nsteps, reduce_mask=0, dist=None, chunks=None,
            variant=sw2d.SW2D_VARIANT_FUSED):
    """Create a handle, upload, step (optionally in chunks), download."""
    hz, e, u, v = state
    ny, nx = hz.shape
    p = sw2d.make_params(nx, ny, params["dx"], params["dy"], params["dt"],
                         params["g"], params["eps"], params["hmin"],
                         reduce_every_step=reduce_mask,
                         history_len=max(nsteps, 1), variant=variant)
    h = sw2d.sw2d_create(p, dist)
    try:
        sw2d.sw2d_set_state(h, hz, e, u, v)
        for n in (chunks or [nsteps]):
            sw2d.sw2d_step(h, n)
        out = sw2d.get_state(h, nx)
        hist = None
        if reduce_mask:
            hist = {op: sw2d.sw2d_reduce_history(h, op, nsteps)
                    for op in range(sw2d.SW2D_RED_N) if reduce_mask & (1 << op)}
        red = [sw2d.sw2d_reduce(h, op) for op in range(sw2d.SW2D_RED_N)]
        launches = sw2d.sw2d_launch_count(h)
    finally:
        sw2d.sw2d_destroy(h)
    return out, hist, red, launches


def check_reductions(got, want, rel=1e-5):
    """Sums within rel (north_star 1e-5); max/min/count exact."""
    for op in range(oracle.NRED):
        g, w = float(got[op]), float(want[op])
        if op in (oracle.VOLUME, oracle.SUM_ETA):
            assert abs(g - w) <= rel * max(abs(w), 1e-12), (oracle.RED_NAMES[op], g, w)
        else:
            assert g == w, (oracle.RED_NAMES[op], g, w)
