#!/usr/bin/env python
"""bench.py — 2DSW cell-updates/s on B200 (BASELINE.json metric) + roofline.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...    (one rank per GPU)

Workload: BASELINE.json configs[4], C5 — the weak
scaling run, 16384 x 16384 cells per GPU (global nx = 16384, ny = 16384 N),
wet/dry bowl with islands, closed basin, dx = dy = 1 m, dt = 0.01 s, with the
per-step global-volume reduction fused into the step.  It is the one config
that spans 1/2/4/8 B200 and whose state (7.5 GB per GPU) is far larger than
L2, as the "% of HBM roofline" half of the metric needs.  One bench step =
one sw2d_step(T) call = T = 100 model time steps (the paper's time loop,
PAPER.md:369-385); value = global cells * T * K / time.

`value`: device-resident state, CUDA events on the handle's stream around K
bench steps, barrier + synchronize on both sides, max over ranks.
`e2e`: the same metric through the public C ABI with host buffers: every
bench step uploads the state from pinned host memory (sw2d_set_state), runs
T steps and reads the T per-step volumes back (sw2d_reduce_history).
`--impl reference`: the CPU oracle (oracle/, single-threaded C) timed on a
bounded sample of the same workload (rank 0 only).

`--workload sor300|sor1024`: the paper's second
workload, red-black SOR for the UFLES pressure Poisson equation
 through include/sor3d.h: one bench step = one
sor3d_iterate(50) call (the paper's 50 SOR iterations per time step) with the
residual folded every iteration; metric SOR cell-iterations/s.  L2 is flushed
(a 512 MB write) before every timed step, each step timed by its own events.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import sw2d_inputs as si  # noqa: E402

METRIC = "2DSW cell-updates/s at 1/2/4/8 B200; % of HBM roofline"
UNIT = "cell-updates/s"
BYTES_PER_CELL = 28          # fused step: read eta,u,v,hzero (16 B) + write eta,u,v (12 B)
PAPER_BYTES_PER_CELL = 75   # paper-shaped variant: 21 + 20 + 34 B over its 3 map kernels
FALLBACK_HBM_GBS = 6650.0    # B200_PROFILING.md fallback (only if MEASURED_PEAKS.json is absent)
E2E_HANDLES = int(os.environ.get("SW2D_E2E_HANDLES", "3"))   # e2e pipeline depth (one GPU)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["c5", "c3", "c2", "c1", "c4", "p1000", "p2000",
                                           "sor300", "sor1024"], default="c5")
    ap.add_argument("--sor-iters", type=int, default=None,
                    help="SOR iterations per bench step (default: the config's, 50 for sor300)")
    ap.add_argument("--sor-residual-every", type=int, default=1,
                    help="SOR residual fold every N iterations (0: none)")
    ap.add_argument("--substeps", type=int, default=None,
                    help="model time steps per bench step (default 100; c2: 10000)")
    ap.add_argument("--reduce", choices=["default", "none", "volume", "all"], default="default",
                    help="per-step fused diagnostics (default: VOLUME for c5, none otherwise)")
    ap.add_argument("--variant", choices=["fused", "paper"], default="fused",
                    help="paper: the paper-shaped 3-map-kernel step (NEXT-1, comparison)")
    ap.add_argument("--halo", choices=["nccl", "p2p"], default="nccl",
                    help="N>1 halo exchange: NCCL send/recv, or fused P2P stores (IPC)")
    ap.add_argument("--snapshots", action="store_true",
                    help="also time sw2d_run_snapshots: eta to pinned host memory once per "
                         "bench step, the copy overlapped with the next steps (NEXT-3)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true",
                    help="short run for ncu: no e2e / cpu baseline / clocks")
    return ap.parse_args()


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def l2_peak():
    """The L2 roofline's peak: the best copy bandwidth over L2-resident
    footprints (<= 64 MB) measured by tools/l2_bw.cu on a B200
    (profiles/r02_l2_peak.json), or (None, why)."""
    p = os.path.join(ROOT, "profiles", "r02_l2_peak.json")
    try:
        with open(p) as f:
            d = json.load(f)
        best = max(r["gbs"] for r in d["results"]
                   if r["kind"] == "copy" and r["footprint_mb"] <= 64)
        return float(best), ("measured: tools/l2_bw.cu copy kernel, L2-resident footprint "
                             "(profiles/r02_l2_peak.json)")
    except Exception as e:  # noqa: BLE001
        return None, "no L2 measurement (%s)" % type(e).__name__


def _ncu_summary():
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def ncu_traffic(workload, kernel):
    """DRAM bytes per launch of `kernel` on `workload` from the committed ncu
    capture (profiles/ncu_summary.json), or None."""
    d = _ncu_summary().get(workload, {}).get(kernel, {})
    return d.get("dram_bytes_per_launch")


def ncu_instr_per_cell_step(workload, kernel):
    """Thread-instructions per cell-step of `kernel` on `workload` from the
    committed ncu capture, with the capture's name, or (None, None)."""
    d = _ncu_summary().get(workload, {}).get(kernel, {})
    if "thread_instr_per_cell_step" in d:
        return d["thread_instr_per_cell_step"], d.get("capture", "profiles/ncu_summary.json")
    return None, None


def max_sm_mhz():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["sm_max_mhz"])
    except Exception:
        return 1965.0


class Clocks:
    """nvidia-smi sampling of SM clocks and throttle reasons during a region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, val in zip(names, f[3:7]):
                if val.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_info():
    """Host CPU model and core count (the oracle runs on one of them)."""
    model = platform.processor() or platform.machine()
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu": model, "of_cores": os.cpu_count()}


class OneCore:
    """Pin this process to one core while the single-threaded oracle runs."""

    def __enter__(self):
        self.saved = None
        try:
            self.saved = os.sched_getaffinity(0)
            os.sched_setaffinity(0, {min(self.saved)})
        except (AttributeError, OSError):
            self.saved = None
        return self

    def __exit__(self, *a):
        if self.saved is not None:
            os.sched_setaffinity(0, self.saved)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def default_substeps(workload):
    return 10000 if workload in ("c2", "p1000", "p2000") else 100


# ---------------------------------------------------------------------------
# reference arm: the CPU oracle on a bounded sample of the same workload
# ---------------------------------------------------------------------------

def oracle_sample(cfg, target_s=4.0):
    """A band of rows from the middle of the workload's grid (full width),
    run as its own closed basin; sized for about target_s seconds per sample."""
    import oracle
    nx, ny = cfg["nx"], cfg["ny"]
    rows = int(max(4, min(ny, 256)))
    j0 = max(0, ny // 2 - rows // 2)
    st = si.generate(cfg, j0=j0, nrows=rows)
    params = si.model_params(cfg)
    t = time.perf_counter()
    oracle.run(params, *st, 1)
    per_step = max(time.perf_counter() - t, 1e-6)
    steps = int(max(1, min(1000, target_s / per_step)))
    desc = (f"rows [{j0},{j0 + rows}) x all {nx} cols of {cfg['name']} run as a closed "
            f"basin, {steps} steps per sample (single-threaded C oracle)")
    return params, st, steps, rows * nx, desc


def run_reference(args, cfg, ws, rank):
    if rank != 0:
        return
    import oracle
    params, st, steps, cells, desc = oracle_sample(cfg)
    times = []
    with OneCore():
        for _ in range(max(args.warmup, 0)):
            oracle.run(params, *st, steps)
        for _ in range(args.steps):
            t = time.perf_counter()
            oracle.run(params, *st, steps)
            times.append(time.perf_counter() - t)
    tot = sum(times)
    value = cells * steps * args.steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(cfg, args, ws),
        "cpu_baseline": dict({"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                              "sample": desc}, **cpu_info()),
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(cfg, args, ws):
    return {
        "workload": f"{cfg['name']}: {cfg['desc']}",
        "nx": cfg["nx"], "ny": cfg["ny"], "cells_per_gpu": cfg["nx"] * cfg["ny"] // ws,
        "substeps_per_step": args.substeps, "dx": cfg["dx"], "dt": cfg["dt"],
        "reduce_every_step": args.reduce if args.reduce != "default" else
        ("VOLUME" if cfg["name"] == "c5" else "none"),
        "parallelism": f"row slabs x{ws}" if ws > 1 else "1 GPU",
        "l2": "inputs larger than L2 (state >> 126 MB), no flush"
        if cfg["nx"] * cfg["ny"] // ws * BYTES_PER_CELL > 1e9 else
        "L2-resident working set (launch/latency-bound; no L2 flush)",
    }


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args, cfg, ws, rank, local):
    import torch
    import torch.distributed as dist

    from paper_1711_04471_b200 import sw2d

    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    nx, ny = cfg["nx"], cfg["ny"]
    j0, nrows = sw2d.sw2d_partition(ny, ws, rank)
    T = args.substeps
    mask = (1 << sw2d.SW2D_RED_VOLUME) if cfg["name"] == "c5" else 0
    if args.reduce != "default":
        mask = {"none": 0, "volume": 1 << sw2d.SW2D_RED_VOLUME,
                "all": (1 << sw2d.SW2D_RED_N) - 1}[args.reduce]

    # inputs for this rank's slab, in pinned host memory
    host = [torch.empty((nrows, nx), dtype=torch.float32, pin_memory=True) for _ in range(4)]
    si.generate(cfg, j0=j0, nrows=nrows, out=tuple(t.numpy() for t in host))

    uid = None
    if ws > 1:
        obj = [sw2d.sw2d_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    elif os.environ.get("SW2D_FORCE_NCCL", "0") != "0":
        uid = sw2d.sw2d_nccl_unique_id()   # one real rank with the NCCL machinery (A/B)
    stream = torch.cuda.Stream()          # the handle's stream; events are recorded on it
    torch.cuda.set_stream(stream)
    p = sw2d.make_params(nx, ny, cfg["dx"], cfg["dy"], cfg["dt"], cfg["g"], cfg["eps"],
                         cfg["hmin"], reduce_every_step=mask, history_len=max(T, 1),
                         variant=sw2d.SW2D_VARIANT_PAPER if args.variant == "paper"
                         else sw2d.SW2D_VARIANT_FUSED)
    halo = sw2d.SW2D_HALO_P2P if args.halo == "p2p" else sw2d.SW2D_HALO_NCCL
    h = sw2d.sw2d_create(p, sw2d.make_dist(rank, ws, local, 0, uid, halo), stream)

    def barrier():
        if ws > 1:
            dist.barrier()

    def max_over_ranks(x):
        if ws == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    try:
        sw2d.sw2d_set_state(h, *host)
        for _ in range(args.warmup):
            sw2d.sw2d_step(h, T)
        sw2d.sw2d_sync(h)

        # --- value: state resident in HBM -------------------------------
        l0 = sw2d.sw2d_launch_count(h)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with Clocks(local) as clk:
            barrier()
            torch.cuda.synchronize()
            ev0.record(stream)
            for _ in range(args.steps):
                sw2d.sw2d_step(h, T)
            ev1.record(stream)
            sw2d.sw2d_sync(h)
            torch.cuda.synchronize()
            barrier()
        ms = max_over_ranks(ev0.elapsed_time(ev1))
        launches = sw2d.sw2d_launch_count(h) - l0
        value = nx * ny * T * args.steps / (ms * 1e-3)

        # roofline of the step kernel.  One launch advances `spl` model steps
        # (2: the two-step kernel on one slab; 1: one step; at N>1 interior +
        # boundary launches per step are timed together).
        red_lvl = 0 if not mask else (1 if mask < 4 else 2)
        launches_per_step = launches / (T * args.steps)
        plan = dict(kv.split("=") for kv in sw2d.sw2d_plan(h).split())
        persist = plan.get("kernel") == "persist"
        pk = int(plan.get("steps_per_block", "0"))
        if persist:
            # K steps per shared-memory block; the bytes are those of the
            # two-step pass (14 B/cell-step), whatever K, so that the small-grid
            # kernels compare on one scale
            spl = 2
        else:
            spl = int(plan.get("steps_per_launch", "1")) if args.variant == "fused" else 1
        t_launch_s = ms * 1e-3 / (T * args.steps) * spl
        cells_local = nrows * nx
        bpc = BYTES_PER_CELL if args.variant == "fused" else PAPER_BYTES_PER_CELL
        alg_bytes = bpc * cells_local            # state in + state out, per launch
        hbm_achieved = alg_bytes / t_launch_s / 1e9
        peak, peak_src = hbm_peak()
        if persist:
            kname = "sw2d_persist<%d, %s, %s, %d, %s>" % (
                pk, plan["warps"], plan["rows_per_thread"], red_lvl,
                "true" if plan.get("handshake") == "tagged" else "false")
        elif plan.get("kernel") == "small":
            kname = ("sw2d_step_small2<%d>" if spl == 2 else "sw2d_step_small<%d>") % red_lvl
        elif spl == 2:
            kname = "sw2d_step_cta2<%d>" % red_lvl
        else:
            kname = "sw2d_step_cta<%d, 0>" % red_lvl
        if args.variant != "fused":
            kname = "paper_momentum + paper_continuity + paper_shapiro_update (per step)"
        # The binding ceiling is HBM: a launch moves the state once in and once
        # out (28 B/cell) whatever number of model steps it advances, i.e. 14
        # B/cell-step for the two-step kernel.  `achieved` =
        # those bytes / the launch's average duration, from the CUDA events
        # around the timed region (the handle's stream) divided by the
        # launches in it (the graphs' tiny set_dstep / ring_scatter kernels
        # included, so it slightly understates the step kernel).
        roof = {"bound": "hbm", "achieved": hbm_achieved, "peak": peak, "unit": "GB/s",
                "frac": hbm_achieved / peak, "peak_source": peak_src,
                "traffic": ncu_traffic(cfg["name"], kname) if args.variant == "fused" else None,
                "algorithmic_bytes_per_launch": alg_bytes,
                "algorithmic_bytes_per_cell_step": bpc / spl, "model_steps_per_launch": spl,
                "kernel": kname, "launches_per_model_step": launches_per_step,
                "plan": sw2d.sw2d_plan(h)}
        if persist or plan.get("kernel") == "small":
            # Small grids (state in L2, the persistent kernel or the small-grid
            # graphs): the same algorithmic bytes — what a two-step pass must
            # move in and out, 14 B/cell-step — can only come from L2, so the
            # roofline is L2's measured copy bandwidth (tools/l2_bw.cu); the
            # HBM figures move to hbm_view.
            # (The persistent kernel keeps its tile in shared memory and moves
            # only the tile rings through L2, so this bounds the regime, not
            # the kernel's own traffic: a low frac = latency-bound.)
            l2, l2_src = l2_peak()
            if l2:
                hv = {k: roof[k] for k in ("bound", "achieved", "peak", "unit", "frac",
                                           "peak_source", "traffic")}
                roof.update(bound="l2", peak=l2, frac=hbm_achieved / l2, peak_source=l2_src,
                            traffic=None, hbm_view=hv)
            roof["us_per_model_step"] = ms * 1e3 / (T * args.steps)
        if persist:   # one launch runs many blocks of K steps
            roof["algorithmic_bytes_per_two_steps"] = roof.pop("algorithmic_bytes_per_launch")
            roof.pop("model_steps_per_launch")
            roof["model_steps_per_block"] = pk
            roof["launches_per_model_step"] = launches_per_step
        # the survey's single-step budget (28 B per cell-STEP):
        # above 1 here because two steps share one HBM pass
        roof["survey_28B_frac"] = value / ws * BYTES_PER_CELL / 1e9 / peak
        ipc, ipc_src = ncu_instr_per_cell_step(cfg["name"], kname)
        if ipc:
            # the other ceiling: instruction issue, 4 warp-instr/clk/SM x 32
            # lanes x SMs x max SM clock, at ncu's thread-instructions per
            # cell-step for this kernel on this workload
            sm_hz = max_sm_mhz() * 1e6
            sms = torch.cuda.get_device_properties(local).multi_processor_count
            issue_peak = 4 * 32 * sms * sm_hz / 1e12
            ach = ipc * (cells_local * spl / t_launch_s) / 1e12
            roof["issue_view"] = {
                "bound": "alu", "achieved": ach, "peak": issue_peak, "unit": "Tinstr/s",
                "frac": ach / issue_peak, "thread_instr_per_cell_step": ipc, "ncu": ipc_src,
                "peak_source": "4 warp-instructions/clk/SM x 32 x %d SMs x %.0f MHz "
                               "(B200_PROFILING.md / B300_MICROARCH.md issue model)"
                               % (sms, sm_hz / 1e6)}

        # --- periodic output overlapped with compute (optional) ------------
        snaps = None
        if args.snapshots:
            snapbuf = torch.empty((1, nrows, nx), dtype=torch.float32, pin_memory=True)
            barrier()
            torch.cuda.synchronize()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            for _ in range(args.steps):
                sw2d.sw2d_run_snapshots(h, T, T, snapbuf)
            s1.record(stream)
            torch.cuda.synchronize()
            sms = max_over_ranks(s0.elapsed_time(s1))
            snaps = {"value": nx * ny * T * args.steps / (sms * 1e-3), "unit": UNIT,
                     "every": T, "d2h_bytes_per_step": 4 * cells_local,
                     "path": "sw2d_run_snapshots(T, every=T) per bench step, pinned host"}

        # --- e2e: host buffers through the C ABI ----------------------------
        # Every bench step is one independent problem through the public API:
        # sw2d_set_state from pinned host memory (16 B/cell H2D), sw2d_step(T),
        # then the result back to pinned host memory — the state eta, u, v
        # (sw2d_get_state, 12 B/cell D2H) and the T per-step volumes
        # (sw2d_reduce_history).  Wall clock around the whole loop, synchronized
        # on both sides.  One GPU: SW2D_E2E_HANDLES (default 3) handles on as
        # many streams, pipelined the way a user runs a stream of problems —
        # problem k+1 uploads and problem k-1 downloads (two host threads; the
        # calls block) while problem k computes; the computes are serialised by
        # events, so compute never overlaps compute.  Several ranks: one
        # handle, serial.
        e2e = None
        if not args.no_e2e and not args.profile:
            nbuf = E2E_HANDLES if ws == 1 else 1   # (several ranks: one handle, serial)
            out_state = [[torch.empty((nrows, nx), dtype=torch.float32, pin_memory=True)
                          for _ in range(3)] for _ in range(nbuf)]
            out_hist = [np.empty(max(T, 1), np.float64) for _ in range(nbuf)]

            def read_back(hh, b):
                sw2d.sw2d_get_state(hh, *out_state[b])
                if mask:
                    sw2d.sw2d_reduce_history(hh, sw2d.SW2D_RED_VOLUME, T, out_hist[b])
                else:
                    out_hist[b][0] = sw2d.sw2d_reduce(hh, sw2d.SW2D_RED_VOLUME)

            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                sw2d.sw2d_set_state(h, *host)
                sw2d.sw2d_step(h, T)
                read_back(h, 0)
            sw2d.sw2d_sync(h)
            torch.cuda.synchronize()
            wall_serial = max_over_ranks(time.perf_counter() - t0)
            barrier()
            ref_eta = out_state[0][0].clone()
            wall, how = wall_serial, "serial, one handle"
            if ws == 1:
                import threading
                nh = E2E_HANDLES
                streams = [stream] + [torch.cuda.Stream() for _ in range(nh - 1)]
                hs = [h] + [sw2d.sw2d_create(p, sw2d.make_dist(rank, ws, local, 0, uid, halo), st)
                            for st in streams[1:]]
                try:
                    for hh in hs[1:]:   # warm the other handles (graphs, plan)
                        sw2d.sw2d_set_state(hh, *host)
                        sw2d.sw2d_step(hh, T)
                        sw2d.sw2d_sync(hh)
                    torch.cuda.synchronize()
                    done = [torch.cuda.Event() for _ in range(args.steps)]
                    enq = [threading.Event() for _ in range(args.steps)]
                    freed = [threading.Event() for _ in range(args.steps)]
                    err = []

                    def uploader():
                        try:
                            for k in range(args.steps):
                                b = k % nh
                                if k >= nh:
                                    freed[k - nh].wait()
                                sw2d.sw2d_set_state(hs[b], *host)
                                if k > 0:   # computes run one after another
                                    streams[b].wait_event(done[k - 1])
                                sw2d.sw2d_step(hs[b], T)
                                done[k].record(streams[b])
                                enq[k].set()
                        except Exception as ex:   # surface in the main thread
                            err.append(ex)
                            for e_ in enq:
                                e_.set()

                    def downloader():
                        try:
                            for k in range(args.steps):
                                enq[k].wait()
                                if err:
                                    return
                                read_back(hs[k % nh], k % nh)
                                freed[k].set()
                        except Exception as ex:
                            err.append(ex)
                            for f_ in freed:
                                f_.set()

                    t0 = time.perf_counter()
                    th = [threading.Thread(target=uploader), threading.Thread(target=downloader)]
                    for t_ in th:
                        t_.start()
                    for t_ in th:
                        t_.join()
                    torch.cuda.synchronize()
                    wall = time.perf_counter() - t0
                    if err:
                        raise err[0]
                    how = (f"pipelined: {nh} handles on {nh} streams, upload / compute / "
                           "download")
                    last = (args.steps - 1) % nh
                    assert torch.equal(out_state[last][0], ref_eta), "e2e: handles disagree"
                finally:
                    for hh in hs[1:]:
                        sw2d.sw2d_destroy(hh)
            e2e = {"value": nx * ny * T * args.steps / wall, "unit": UNIT,
                   "h2d_bytes_per_step": 16 * cells_local,
                   "d2h_bytes_per_step": 12 * cells_local + (8 * T if mask else 8),
                   "ms_per_step": 1e3 * wall / args.steps, "wall_s": wall,
                   "path": "sw2d_set_state(pinned host hzero, eta, u, v) + sw2d_step(T) + "
                           "sw2d_get_state(pinned host eta, u, v) + sw2d_reduce_history(VOLUME, "
                           "T) per bench step, wall clock; " + how,
                   "serial": {"value": nx * ny * T * args.steps / wall_serial,
                              "ms_per_step": 1e3 * wall_serial / args.steps,
                              "wall_s": wall_serial}}
    finally:
        sw2d.sw2d_destroy(h)

    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return

    cpu = None
    if ws == 1 and not args.no_cpu_baseline and not args.profile:
        import oracle
        params, st, steps, cells, desc = oracle_sample(cfg, target_s=12.0)
        with OneCore():
            t = time.perf_counter()
            oracle.run(params, *st, steps)
            dt_s = time.perf_counter() - t
        cpu = dict({"value": cells * steps / dt_s, "unit": UNIT, "cores": 1, "kind": "oracle",
                    "sample": desc, "seconds": dt_s}, **cpu_info())

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (seeded bowl + islands + Gaussian bump)",
        "config": workload_config(cfg, args, ws),
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
        "clocks": clk.summary(), "gpu_launches": launches,
    }
    if snaps is not None:
        line["snapshots"] = snaps
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# NEXT-4: red-black SOR (include/sor3d.h)
# ---------------------------------------------------------------------------

SOR_METRIC = "SOR cell-iterations/s (red-black 7-point Poisson, UFLES press shape)"
SOR_UNIT = "cell-iterations/s"
SOR_BYTES_PER_CELL = 12      # one fused iteration: read p, rhs (8 B) + write p (4 B)
SOR_RES_BYTES_PER_CELL = 8   # the trailing residual-only pass: read p, rhs


def sor_config(cfg, args, n, every):
    return {
        "workload": f"{cfg['name']}: {cfg['desc']}",
        "nx": cfg["nx"], "ny": cfg["ny"], "nz": cfg["nz"], "iterations_per_step": n,
        "residual_every": every, "omega": 1.5, "dx": 4.0, "dz": 2.0,
        "parallelism": "1 GPU (replicas only: independent solves per GPU)",
        "l2": "L2 flushed (512 MB write) before every timed step; each step timed alone",
    }


def run_sor_reference(args, cfg, rank):
    if rank != 0:
        return
    import oracle
    import sor_inputs as so
    p0, rhs = so.generate(cfg)
    prm = so.params()
    n = min(args.sor_iters or cfg["iters"], 10)
    hist = args.sor_residual_every > 0
    times = []
    with OneCore():
        for _ in range(max(args.warmup, 0)):
            oracle.sor_run(prm, p0, rhs, 1, history=hist)
        for _ in range(args.steps):
            t = time.perf_counter()
            oracle.sor_run(prm, p0, rhs, n, history=hist)
            times.append(time.perf_counter() - t)
    tot = sum(times)
    cells = so.cells(cfg)
    value = cells * n * args.steps / tot
    desc = (f"the full {cfg['nx']}x{cfg['ny']}x{cfg['nz']} grid, {n} iterations per step "
            f"(residual every iteration: {hist}), single-threaded C oracle")
    print(json.dumps({
        "impl": "reference", "metric": SOR_METRIC, "value": value, "unit": SOR_UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": sor_config(cfg, args, n, args.sor_residual_every),
        "cpu_baseline": dict({"value": value, "unit": SOR_UNIT, "cores": 1, "kind": "oracle",
                              "sample": desc}, **cpu_info()),
        "e2e": {"value": value, "unit": SOR_UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


def run_sor_ours(args, cfg, ws, rank, local):
    """Replicas only: every rank solves its own copy (no data-path exchange)."""
    import torch
    import torch.distributed as dist

    import sor_inputs as so
    from paper_1711_04471_b200 import sor3d

    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    nx, ny, nz = cfg["nx"], cfg["ny"], cfg["nz"]
    cells = nx * ny * nz
    n = args.sor_iters or cfg["iters"]
    every = args.sor_residual_every
    nrec = 0 if every <= 0 else len([t for t in range(1, n + 1) if t % every == 0 or t == n])
    p0, rhs = so.generate(cfg)
    hp0 = torch.from_numpy(p0).pin_memory()
    hrhs = torch.from_numpy(rhs).pin_memory()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    h = sor3d.sor3d_create(sor3d.make_params(nx, ny, nz, **so.params(),
                                             history_len=max(nrec, 1)), stream)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        if ws > 1:
            dist.barrier()

    def max_over_ranks(x):
        if ws == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed_steps(body):
        tot = 0.0
        for _ in range(args.steps):
            flush.fill_(1)                      # L2 flush, outside the timed region
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            body()
            e1.record(stream)
            e1.synchronize()
            tot += e0.elapsed_time(e1)
        return tot

    try:
        sor3d.sor3d_set(h, hp0, hrhs)
        for _ in range(args.warmup):
            sor3d.sor3d_iterate(h, n, every)
        sor3d.sor3d_sync(h)
        l0 = sor3d.sor3d_launch_count(h)
        with Clocks(local) as clk:
            barrier()
            torch.cuda.synchronize()
            ms = timed_steps(lambda: sor3d.sor3d_iterate(h, n, every))
            torch.cuda.synchronize()
            barrier()
        ms = max_over_ranks(ms)
        launches = sor3d.sor3d_launch_count(h) - l0
        value = ws * cells * n * args.steps / (ms * 1e-3)
        step_s = ms * 1e-3 / args.steps
        alg = cells * (SOR_BYTES_PER_CELL * n + (SOR_RES_BYTES_PER_CELL if every > 0 else 0))
        peak, peak_src = hbm_peak()
        kname = "sor_iter<32, %d, 1, %d>" % (1 if every > 0 else 0,
                                           1 if "L2 hints" in sor3d.sor3d_plan(h) else 0)
        ach = alg / step_s / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": ach / peak, "peak_source": peak_src,
                "traffic": ncu_traffic(cfg["name"], kname), "kernel": kname,
                "algorithmic_bytes_per_step": alg,
                "algorithmic_bytes_per_cell_iteration": SOR_BYTES_PER_CELL,
                "launches_per_step": launches / args.steps, "plan": sor3d.sor3d_plan(h)}

        e2e = None
        if not args.no_e2e and not args.profile:
            hist = np.empty((max(nrec, 1), 2), np.float64)
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()

            def e2e_body():
                sor3d.sor3d_set(h, hp0, hrhs)
                sor3d.sor3d_iterate(h, n, every)
                if nrec:
                    hist[:] = sor3d.sor3d_residual_history(h, nrec)
                else:
                    sor3d.sor3d_residual(h)
            ems = max_over_ranks(timed_steps(e2e_body))
            e2e = {"value": ws * cells * n * args.steps / (ems * 1e-3), "unit": SOR_UNIT,
                   "h2d_bytes_per_step": 8 * cells, "d2h_bytes_per_step": 16 * max(nrec, 1),
                   "ms_per_step": ems / args.steps, "wall_s": time.perf_counter() - t0,
                   "path": "sor3d_set(pinned host p, rhs) + sor3d_iterate(n, every) + "
                           "sor3d_residual_history per bench step"}
    finally:
        sor3d.sor3d_destroy(h)
    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return
    cpu = None
    if ws == 1 and not args.no_cpu_baseline and not args.profile:
        import oracle
        ns = 10
        with OneCore():
            t = time.perf_counter()
            oracle.sor_run(so.params(), p0, rhs, ns, history=every > 0)
            dt_s = time.perf_counter() - t
        cpu = dict({"value": cells * ns / dt_s, "unit": SOR_UNIT, "cores": 1, "kind": "oracle",
                    "sample": f"the full grid, {ns} iterations (residual every iteration: "
                              f"{every > 0}), single-threaded C oracle", "seconds": dt_s},
                   **cpu_info())
    print(json.dumps({
        "metric": SOR_METRIC, "value": value, "unit": SOR_UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded Gaussian sources + noise, sor_inputs)",
        "config": sor_config(cfg, args, n, every), "roofline": roof, "cpu_baseline": cpu,
        "e2e": e2e, "clocks": clk.summary(), "gpu_launches": launches,
    }), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    ws, rank, local = dist_env()
    if args.workload.startswith("sor"):
        import sor_inputs as so
        cfg = so.config(args.workload)
        if args.impl == "reference":
            run_sor_reference(args, cfg, rank)
        else:
            run_sor_ours(args, cfg, ws, rank, local)
        return
    if args.substeps is None:
        args.substeps = default_substeps(args.workload)
    cfg = si.config(args.workload, ws if args.workload == "c5" else 1)
    if args.impl == "reference":
        run_reference(args, cfg, ws, rank)
        return
    run_ours(args, cfg, ws, rank, local)


if __name__ == "__main__":
    main()
