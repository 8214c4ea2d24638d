#!/usr/bin/env python
"""bench.py — LSKUM fixed-point iteration on B200: device-timed point-iterations/s.

Workload (BASELINE.json configs[1]): NACA 0012, M=0.85, alpha=1 deg, ~160K
points, second order with 3 inner derivative sweeps, CFL 0.5.  The cloud is
this repo's synthetic NACA 0012 O-cloud (520 surface points x 308 rings, far
field at 20 chords; lskum_b200_cloud_generate_naca0012), with the surface ring
held at the free stream (kind outer): the reference has no wall flux and its
split stencils on a curved wall are singular or unstable (gap 5),
so this is the NACA point distribution both codes can run.  State: the free
stream lskum_run initialises — an exact fixed point with the full arithmetic
cost.  `--cloud rect` uses the reference's jittered rectangle instead.  The
`large` block repeats the measurement on a ~10M-point cloud (configs[3]).

One step = one fixed-point iteration (3 sweeps, flux, update, residue tree).
`value` times K steps with CUDA events on the engine's stream, with the L2
flushed (384 MB overwrite) before every step: each step is one CUDA graph
[flush, start event, iteration, end event], so the events bracket the cold-L2
iteration and not the flush or the graph launch; `e2e` times lskum_run through the
C ABI from host buffers (upload, K iterations, copy-back of the 21-slot store).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
COUNTS_PATH = os.path.join(ROOT, "profiles", "flux_ncu_counts.json")
METRIC = "point-iterations/sec (device-timed) at 1/2/4/8 B200; % HBM roofline"
UNIT = "point-iterations/s"

# Algorithmic bytes per point: one derivative sweep reads
# x,y (16) q (32) qx,qy (64) offsets (8) ids (4k) and writes qx,qy (64):
# 184 + 4k; the fused flux+dt+update+q+residue pass moves 217 + 4k.
def sweep_bytes(k):
    return 184 + 4 * k


def flux_bytes(k):
    return 217 + 4 * k


def iteration_bytes(k, order, inner):
    return (inner * sweep_bytes(k) if order == 2 else 0) + flux_bytes(k) - (64 if order == 1 else 0)


# ---------------------------------------------------------------------------
def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--cloud", choices=["naca", "rect"], default="naca",
                    help="naca: synthetic NACA 0012 O-cloud (surface held, see DESIGN.md); "
                         "rect: the reference's jittered rectangle")
    ap.add_argument("--side", type=int, default=400, help="rect cloud is side x side points")
    ap.add_argument("--naca", default="520x308", help="NACA cloud n_wall x n_rings (per GPU)")
    ap.add_argument("--order", type=int, default=2)
    ap.add_argument("--inner", type=int, default=3)
    ap.add_argument("--mach", type=float, default=0.85)
    ap.add_argument("--aoa", type=float, default=1.0)
    ap.add_argument("--fp-mode", default="fast")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-steady", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline sample target")
    ap.add_argument("--large-side", type=int, default=3163,
                    help="side of the >=10M-point rect cloud measured alongside (configs[3]); 0 = skip")
    ap.add_argument("--large-naca", default="4000x2500", help="NACA size of the >=10M-point cloud")
    ap.add_argument("--large-steps", type=int, default=10)
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the GPU works."""

    FIELDS = ("clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), float(parts[2]), parts[3:]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        loaded = [r for r in rows if r[2] >= 50.0] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in loaded for i, v in enumerate(r[3]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(loaded)}


def load_counts():
    try:
        with open(COUNTS_PATH) as f:
            return json.load(f)
    except OSError:
        return {}


def hbm_peak():
    try:
        with open(PEAKS_PATH) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# CPU baseline: the reference's own implementation (oracle/_ref/liblskum.so,
# built from /root/reference by oracle/Makefile) through its C ABI, on all host
# cores (parts = workers = nproc).  Falls back to the plain-C port when the
# reference build is absent.  Test/baseline infrastructure only.
def reference_lib():
    so = os.path.join(ROOT, "oracle", "_ref", "liblskum.so")
    if not os.path.exists(so):
        return None
    L = ctypes.CDLL(so)
    vp = ctypes.c_void_p
    L.lskum_cloud_read_file.argtypes = [ctypes.c_char_p, ctypes.POINTER(vp)]
    L.lskum_config_create.argtypes = [ctypes.POINTER(vp)]
    L.lskum_config_set.argtypes = [vp, ctypes.c_char_p, ctypes.c_char_p]
    L.lskum_run.argtypes = [vp, vp, ctypes.POINTER(vp)]
    L.lskum_result_total_seconds.argtypes = [vp]
    L.lskum_result_total_seconds.restype = ctypes.c_double
    L.lskum_result_destroy.argtypes = [vp]
    L.lskum_cloud_destroy.argtypes = [vp]
    L.lskum_config_destroy.argtypes = [vp]
    L.lskum_last_error.restype = ctypes.c_char_p
    return L


def reference_run(L, cloud_h, a, iters, threads):
    cfg = ctypes.c_void_p()
    L.lskum_config_create(ctypes.byref(cfg))
    for k, v in (("mach", a.mach), ("aoa", a.aoa), ("order", a.order), ("inner", a.inner),
                 ("cfl", 0.5), ("iters", iters), ("parts", threads), ("workers", threads),
                 ("layout", "soa"), ("residual_mode", "fused")):
        assert L.lskum_config_set(cfg, k.encode(), str(v).encode()) == 0
    res = ctypes.c_void_p()
    t0 = time.perf_counter()
    rc = L.lskum_run(cloud_h, cfg, ctypes.byref(res))
    wall = time.perf_counter() - t0
    if rc != 0:
        raise RuntimeError(L.lskum_last_error().decode())
    secs = L.lskum_result_total_seconds(res)
    L.lskum_result_destroy(res)
    L.lskum_config_destroy(cfg)
    return secs, wall


def reference_cloud(L, cloud):
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "bench.grid")
        cloud.write_file(path)  # same grid file feeds both sides
        h = ctypes.c_void_p()
        if L.lskum_cloud_read_file(path.encode(), ctypes.byref(h)) != 0:
            raise RuntimeError(L.lskum_last_error().decode())
    return h


def cpu_baseline(cloud, a, target_s):
    """Bounded sample of the same workload on the host cores."""
    n = cloud.n
    threads = os.cpu_count() or 1
    L = reference_lib()
    if L is not None:
        h = reference_cloud(L, cloud)
        s1, _ = reference_run(L, h, a, 2, threads)
        iters = int(max(2, min(500, target_s / max(s1 / 2, 1e-6))))
        secs, _ = reference_run(L, h, a, iters, threads)
        L.lskum_cloud_destroy(h)
        return {"value": n * iters / secs, "unit": UNIT, "cores": threads, "kind": "reference",
                "sample": f"{iters} iterations of the {n}-point cloud, lskum_run of oracle/_ref/liblskum.so "
                          f"(parts=workers={threads}, soa, fused), reference loop timer"}
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import pyoracle as P
    g = cloud.geometry()
    c = P.Cloud(g["x"], g["y"], g["kind"], g["nx"], g["ny"], g["off"], g["nbr"])
    t0 = time.perf_counter()
    P.orc_run(c, mach=a.mach, aoa=a.aoa, iters=1, order=a.order, inner=a.inner)
    one = time.perf_counter() - t0
    iters = int(max(1, min(200, target_s / max(one, 1e-6))))
    t0 = time.perf_counter()
    P.orc_run(c, mach=a.mach, aoa=a.aoa, iters=iters, order=a.order, inner=a.inner)
    dt = time.perf_counter() - t0
    return {"value": n * iters / dt, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{iters} iterations of the {n}-point cloud, oracle/lskum_oracle.c (1 thread)"}


def naca_dims(spec, scale=1.0):
    nw, nr = (int(v) for v in spec.lower().split("x"))
    f = math.sqrt(scale)
    nw = max(16, 2 * int(round(nw * f / 2)))
    return nw, max(3, int(round(nr * f)))


def make_cloud(L, a, scale=1.0, large=False):
    """The workload cloud for `scale` GPUs (weak scaling: points grow with scale)."""
    if a.cloud == "naca":
        nw, nr = naca_dims(a.large_naca if large else a.naca, scale)
        return L.Cloud.generate_naca0012(nw, nr, 20.0, 0.0, 7, 8, frozen_wall=True), f"{nw}x{nr}"
    side = int(round((a.large_side if large else a.side) * math.sqrt(scale)))
    return L.Cloud.generate_rect(side, side, 0.1, 7, 8), f"{side}x{side}"


def workload_text(a, dims, large=False):
    if a.cloud == "naca":
        size = "~10M points, BASELINE configs[3]" if large else "~160K points/GPU, BASELINE configs[1]"
        return (f"synthetic NACA 0012 O-cloud {dims} (n_wall x n_rings, far field 20 chords, kNN k=8; "
                f"surface points held at the free stream because the reference has no wall flux); {size}; "
                f"M={a.mach}, AoA={a.aoa}, order {a.order}, {a.inner} inner sweeps; free-stream state")
    size = "~10M points, BASELINE configs[3] size" if large else "stand-in for BASELINE configs[1] (~160K/GPU)"
    return (f"rect {dims} (reference generator, jitter 0.1, seed 7, k 8), {size}; M={a.mach}, AoA={a.aoa}, "
            f"order {a.order}, {a.inner} inner sweeps; free-stream state")


def rooflines(L, counts, n, n_flux, k, order, inner, step_ms, sweep_ms, flux_ms, device=0, domains=1):
    """Flux kernel against the measured DFMA peak (dynamic FP64 flops per point
    from ncu), sweep and whole iteration against the measured HBM copy peak."""
    fp64_peak = L.fp64_peak_tflops(device)
    flops_pt = counts.get("flux_fp64_flops_per_point")
    n_flux_dom = n_flux / domains
    achieved = flops_pt * n_flux_dom / (flux_ms * 1e-3) / 1e12 if (flops_pt and flux_ms > 0) else None
    traffic = counts.get("flux_dram_bytes_per_point")
    hbm, hbm_kind = hbm_peak()
    sweep_gbs = sweep_bytes(k) * (n / domains) / (sweep_ms * 1e-3) / 1e9 if sweep_ms else None
    iter_gbs = iteration_bytes(k, order, inner) * n / (step_ms * 1e-3) / 1e9 / domains
    inst = counts.get("flux_fp64_thread_inst_per_point") or {}
    inst_pt = sum(inst.get(k, 0.0) for k in ("dfma", "dadd", "dmul"))
    pipe = inst_pt * n_flux_dom / (flux_ms * 1e-3) / (fp64_peak * 1e12 / 2) if (inst_pt and flux_ms > 0) else None
    flux = {"bound": "fp64", "kernel": "k_flux_ws (fast flux residual: split-stencil weights, cp.async staged)",
            "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
            "frac": achieved / fp64_peak if achieved else None,
            "fp64_pipe_frac": pipe,
            "fp64_pipe_note": "FP64 instructions (DFMA+DADD+DMUL, ncu) per second over the DFMA instruction peak "
                              "(peak TFLOP/s / 2): DADD/DMUL occupy a full pipe slot for one flop",
            "traffic": traffic * n_flux_dom if traffic else None,
            "traffic_unit": "bytes per launch (ncu dram__bytes_read+write)",
            "peak_source": "DFMA microbenchmark on this GPU (lskum_b200_fp64_peak)",
            "flops_source": f"ncu dynamic 2*DFMA+DADD+DMUL = {flops_pt:.0f} per point "
                            "(profiles/flux_ncu_counts.json)" if flops_pt else None,
            "launch_ms": flux_ms}
    hbmr = {"bound": "hbm", "kernel": "k_sweep2 (derivative sweep)", "achieved": sweep_gbs, "peak": hbm,
            "unit": "GB/s", "frac": sweep_gbs / hbm if sweep_gbs else None,
            "algorithmic_bytes_per_point": sweep_bytes(k), "launch_ms": sweep_ms, "peak_source": hbm_kind,
            "iteration_achieved_gbs_per_gpu": iter_gbs, "iteration_frac": iter_gbs / hbm,
            "iteration_bytes_per_point": iteration_bytes(k, order, inner)}
    return flux, hbmr


def large_run(L, a, counts):
    """The >=10M-point cloud (BASELINE configs[3] size; roofline
    fractions are quoted there), same session machinery, L2 flushed per step."""
    cloud, dims = make_cloud(L, a, large=True)
    n = cloud.n
    k = cloud.nnz // n
    n_flux = int(np.count_nonzero(cloud.geometry()["kind"] != 2))
    cfg = L.Config(mach=a.mach, aoa=a.aoa, order=a.order, inner=a.inner, cfl=0.5, fp_mode=a.fp_mode,
                   iters=a.large_steps, device=0)
    step_ms, sweep_ms, flux_ms = [], [], []
    with ClockSampler(0) as clocks, L.Session(cloud, cfg, capacity=2 * a.large_steps + 3) as sess:
        for _ in range(3):
            sess.step_flushed()
        for _ in range(a.large_steps):
            step_ms.append(sess.step_flushed())
        for _ in range(a.large_steps):  # per-kernel events: separate steps (their event nodes lengthen a step)
            sess.step_flushed(kernel_events=True)
            sw, fl = sess.event_ms()
            sweep_ms.append(sw)
            flux_ms.append(fl)
    total = sum(step_ms)
    flux, hbmr = rooflines(L, counts, n, n_flux, k, a.order, a.inner, total / a.large_steps,
                           statistics.mean(sweep_ms) if a.order == 2 else None, statistics.mean(flux_ms))
    return {"workload": workload_text(a, dims, large=True),
            "n_points": n, "value": n * a.large_steps / (total * 1e-3), "unit": UNIT,
            "ms_per_step": total / a.large_steps, "steps": a.large_steps, "warmup": 3,
            "roofline": flux, "roofline_hbm": hbmr, "clocks": clocks.summary(),
            "l2": "flushed before every timed step (384 MB overwrite); working set ~3 GB > L2"}


# BASELINE.json configs as NACA 0012 O-clouds (n_wall x n_rings): the sizes
# the configs name, with their Mach numbers and angles of attack.
CONFIG_SIZES = [("configs[0] ~40K, M=0.63 AoA=2", "260x154", 0.63, 2.0),
                ("configs[1] ~160K, M=0.85 AoA=1", "520x308", 0.85, 1.0),
                ("configs[2] ~625K, M=1.2 AoA=0", "1000x625", 1.2, 0.0),
                ("configs[3] ~10M, M=0.85 AoA=1", "4000x2500", 0.85, 1.0),
                ("configs[4] ~40M, M=0.85 AoA=1", "8000x5000", 0.85, 1.0)]


def sizes_run(L, a, iters=40):
    """Device-timed throughput at every BASELINE config size, order 2 and 1
    (back-to-back iterations in captured graphs, after 10 warm-up iterations)."""
    out = []
    for label, spec, mach, aoa in CONFIG_SIZES:
        nw, nr = (int(v) for v in spec.split("x"))
        cloud = L.Cloud.generate_naca0012(nw, nr, 20.0, 0.0, 7, 8, frozen_wall=True)
        row = {"config": label, "cloud": f"NACA 0012 {spec}", "n_points": cloud.n}
        for order in (2, 1):
            cfg = L.Config(mach=mach, aoa=aoa, order=order, inner=a.inner, cfl=0.5, fp_mode=a.fp_mode,
                           iters=iters + 10, device=0)
            with L.Session(cloud, cfg, capacity=iters + 10) as sess:
                sess.iterate(10)
                ms = sess.iterate(iters)
            row[f"order{order}"] = {"value": cloud.n * iters / (ms * 1e-3), "ms_per_iteration": ms / iters}
        out.append(row)
    return {"unit": UNIT, "what": f"{iters} back-to-back iterations per size (no L2 flush), free stream; "
                                   "surface held (frozen NACA variant)", "rows": out}


def config_block(a, n, extra=None):
    c = {"workload": workload_text(a, a.dims),
         "n_points": n, "stencil": "kNN k=8 (exact, bit-identical to the reference's build_stencils)",
         "order": a.order, "inner": a.inner, "mach": a.mach, "aoa_deg": a.aoa, "cfl": 0.5,
         "fp_mode": a.fp_mode, "l2": "flushed before every timed step (384 MB overwrite in the same CUDA graph, ahead of the step's start event)",
         "parallelism": f"rcb{a.gpus}" if a.gpus > 1 else "single-domain"}
    if extra:
        c.update(extra)
    return c


# ---------------------------------------------------------------------------
def run_reference_arm(a):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_2403_13287_b200 import lskum as LB
    cloud, a.dims = make_cloud(LB, a, max(a.gpus, world))  # same cloud as the b200 arm
    n = cloud.n
    L = reference_lib()
    threads = os.cpu_count() or 1
    if L is None:
        base = cpu_baseline(cloud, a, a.cpu_seconds)
        value, kind, sample = base["value"], base["kind"], base["sample"]
    else:
        h = reference_cloud(L, cloud)
        if a.warmup > 0:
            reference_run(L, h, a, a.warmup, threads)
        secs, wall = reference_run(L, h, a, a.steps, threads)
        L.lskum_cloud_destroy(h)
        value, kind = n * a.steps / secs, "reference"
        sample = (f"{a.steps} iterations (after {a.warmup} warm-up) of the {n}-point cloud through the "
                  f"reference lskum_run (oracle/_ref/liblskum.so), parts=workers={threads}")
    out = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
           "steps": a.steps, "warmup": a.warmup, "ms_per_step": n / value * 1e3,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": config_block(a, n),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads if kind == "reference" else 1,
                            "kind": kind, "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def run_b200_arm(a):
    from paper_2403_13287_b200 import lskum as L
    world, rank, local = dist_env()
    gpus = max(a.gpus, world)
    if world > 1:
        return run_b200_ranks(a, L, world, rank, local)
    # weak scaling: ~160K points per GPU (both cloud dimensions grow with sqrt(gpus))
    cloud, a.dims = make_cloud(L, a, gpus)
    n = cloud.n
    k = cloud.nnz // n
    n_flux = int(sum(1 for v in cloud.geometry()["kind"] if v != 2))
    cfg = L.Config(mach=a.mach, aoa=a.aoa, order=a.order, inner=a.inner, cfl=0.5, fp_mode=a.fp_mode,
                   iters=a.steps, device=0, gpus=gpus)
    steady_iters = 0
    with ClockSampler(0) as clocks:
        sess = L.Session(cloud, cfg, capacity=a.warmup + 2 * a.steps + 4000)
        for _ in range(a.warmup):
            sess.step_flushed()
        step_ms, sweep_ms, flux_ms = [], [], []
        for _ in range(a.steps):
            step_ms.append(sess.step_flushed())
        for _ in range(a.steps):  # per-kernel events: separate steps (their event nodes lengthen a step)
            sess.step_flushed(kernel_events=True)
            sw, fl = sess.event_ms()
            sweep_ms.append(sw)
            flux_ms.append(fl)
        launches = sess.info()["launches_per_iter"]
        steady = None
        if not a.no_steady:
            per = max(statistics.median(step_ms), 1e-3)
            steady_iters = int(min(3900, max(20, 1500.0 / per)))
            steady_ms = sess.iterate(steady_iters)
            steady = n * steady_iters / (steady_ms * 1e-3)
        residues = sess.residues()
        sess.close()
    clk = clocks.summary()
    total_ms = sum(step_ms)
    value = n * a.steps / (total_ms * 1e-3)

    # e2e through the drop-in C ABI (lskum_run) from host buffers.  Cold: a
    # fresh cloud handle built from host arrays (outside the timer), so the
    # timed call screens the stencils, uploads the geometry (H2D), sets up the
    # device domain, initialises the free stream, runs K iterations and copies
    # the 21-slot store back (D2H).  Warm: a second lskum_run on that handle
    # (lskum_run keeps the cloud's device domain resident between calls).
    g = cloud.geometry()
    e2e_cfg = L.Config(mach=a.mach, aoa=a.aoa, order=a.order, inner=a.inner, cfl=0.5,
                       fp_mode=a.fp_mode, iters=a.steps, device=0, gpus=gpus)
    L.run(L.Cloud.from_arrays(g["x"], g["y"], g["kind"], g["nx"], g["ny"], g["off"], g["nbr"]),
          e2e_cfg).close()  # context and module load
    e2e_cloud = L.Cloud.from_arrays(g["x"], g["y"], g["kind"], g["nx"], g["ny"], g["off"], g["nbr"])
    t0 = time.perf_counter()
    res = L.run(e2e_cloud, e2e_cfg)
    e2e_wall = time.perf_counter() - t0
    res.close()
    t0 = time.perf_counter()
    res = L.run(e2e_cloud, e2e_cfg)
    e2e_warm = time.perf_counter() - t0
    res.close()
    nnz = e2e_cloud.nnz
    h2d = n * (16 + 16 + 1 + 1) + 4 * (n + 1) + 4 * nnz  # xy, normals, kind, part, offsets, ids
    d2h = n * 21 * 8 + 8 * a.steps                       # 21-slot store + residue history

    # rooflines
    counts = load_counts()
    sweep_avg = statistics.mean(sweep_ms) if a.order == 2 else None
    flux_roof, hbm_roof = rooflines(L, counts, n, n_flux, k, a.order, a.inner, total_ms / a.steps, sweep_avg,
                                    statistics.mean(flux_ms), 0, gpus)
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": gpus, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": total_ms / a.steps, "higher_is_better": True,
        "scaling": "weak" if gpus > 1 else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (free-stream state on a generated cloud)",
        "config": config_block(a, n, {"parallelism": f"rcb{gpus} device domains, peer-memory halos"
                                      if gpus > 1 else "single-domain"}),
        "e2e": {"value": n * a.steps / e2e_wall, "unit": UNIT,
                "h2d_bytes_per_step": int(h2d / a.steps), "d2h_bytes_per_step": int(d2h / a.steps),
                "what": "wall time of lskum_run (C ABI) on a fresh cloud handle: stencil screening, geometry "
                        f"H2D, device setup, free-stream init, {a.steps} iterations, copy-back of the 21-slot "
                        "store (D2H)",
                "warm": {"value": n * a.steps / e2e_warm, "h2d_bytes_per_step": 0,
                         "d2h_bytes_per_step": int(d2h / a.steps),
                         "what": "second lskum_run on the same cloud handle: geometry, weights and graphs "
                                 "stay resident; free stream initialised on the device"}},
        "gpu_launches": launches * a.steps,
        "gpu_launches_note": f"{launches} kernels per iteration (all domains) x {a.steps}; "
                             f"plus {a.steps * gpus} L2-flush kernels between steps",
        "roofline": flux_roof,
        "roofline_hbm": hbm_roof,
        "steady_state": {"value": steady, "iterations": steady_iters,
                         "what": "same session, back-to-back iterations, no L2 flush"},
        "clocks": clk,
        "final_residue": float(residues[-1]) if len(residues) else None,
    }
    if (a.large_side > 0 if a.cloud == "rect" else a.large_naca != "0") and gpus == 1:
        out["large"] = large_run(L, a, counts)
        out["sizes"] = sizes_run(L, a)
    if not a.no_cpu_baseline and gpus == 1:
        out["cpu_baseline"] = cpu_baseline(cloud, a, a.cpu_seconds)
    print(json.dumps(out), flush=True)


def run_b200_ranks(a, L, world, rank, local):
    """torchrun: one process per GPU, each running its RCB piece (RankSession).

    Halo exchange and the residue tree are device-to-device over CUDA IPC
    (NVLink peer memory), ordered by device-side progress counters; the gloo
    group only carries setup, per-step barriers and the max-over-ranks timing.
    """
    import numpy as np
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo")
    ndev = max(1, torch.cuda.device_count())
    device = local % ndev
    a.gpus = world
    cloud, a.dims = make_cloud(L, a, world)
    n = cloud.n
    k = cloud.nnz // n
    n_flux = int(sum(1 for v in cloud.geometry()["kind"] if v != 2))
    cfg = L.Config(mach=a.mach, aoa=a.aoa, order=a.order, inner=a.inner, cfl=0.5, fp_mode=a.fp_mode,
                   iters=a.steps)
    step_ms, sweep_ms, flux_ms = [], [], []
    with ClockSampler(device) as clocks:
        sess = L.RankSession(cloud, cfg, rank, world, device, capacity=a.warmup + a.steps + 4000)
        for _ in range(a.warmup):
            sess.flush_l2()
            dist.barrier()
            sess.iterate(1)
        for _ in range(a.steps):
            sess.flush_l2()
            dist.barrier()
            step_ms.append(sess.iterate(1))
            sw, fl = sess.event_ms()
            sweep_ms.append(sw)
            flux_ms.append(fl)
        launches = sess.info()["launches_per_iter"]
        residues = sess.residues()
        sess.close()
    # e2e: host arrays -> this rank's piece on its GPU -> K iterations -> copy-back
    e2e_cloud, _ = make_cloud(L, a, world)
    dist.barrier()
    t0 = time.perf_counter()
    with L.RankSession(e2e_cloud, cfg, rank, world, device, capacity=a.steps) as es:
        es.iterate(a.steps)
        es.download()
    e2e_wall = time.perf_counter() - t0
    mine = {"step_ms": step_ms, "sweep_ms": statistics.mean(sweep_ms) if a.order == 2 else None,
            "flux_ms": statistics.mean(flux_ms), "e2e_wall": e2e_wall, "launches": launches,
            "clocks": clocks.summary()}
    everyone = [None] * world
    dist.all_gather_object(everyone, mine)
    if rank == 0:
        step_max = np.max(np.array([e["step_ms"] for e in everyone]), axis=0)  # max over ranks, per step
        total_ms = float(step_max.sum())
        value = n * a.steps / (total_ms * 1e-3)
        e2e_wall = max(e["e2e_wall"] for e in everyone)
        flux_avg = max(e["flux_ms"] for e in everyone)
        counts = load_counts()
        sweep_avg = max(e["sweep_ms"] for e in everyone) if a.order == 2 else None
        flux_roof, hbm_roof = rooflines(L, counts, n, n_flux, k, a.order, a.inner, total_ms / a.steps, sweep_avg,
                                        flux_avg, device, world)
        nnz = e2e_cloud.nnz
        h2d = n * (16 + 16 + 1 + 1 + 32) + 4 * (n + 1) + 4 * nnz
        d2h = n * 21 * 8 + 8 * a.steps
        clk = everyone[0]["clocks"]
        clk["reasons"] = sorted({r for e in everyone for r in e["clocks"]["reasons"]})
        launches = sum(e["launches"] for e in everyone)
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": total_ms / a.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (free-stream state on a generated cloud)",
            "config": config_block(a, n, {"parallelism": f"rcb{world}: one process per GPU, CUDA-IPC peer-memory "
                                                         "halos, device-side progress counters"}),
            "e2e": {"value": n * a.steps / e2e_wall, "unit": UNIT,
                    "h2d_bytes_per_step": int(h2d / a.steps), "d2h_bytes_per_step": int(d2h / a.steps),
                    "what": "max over ranks of RankSession create (screening, upload of the rank's piece), "
                            f"{a.steps} iterations, copy-back of owned points"},
            "gpu_launches": launches * a.steps,
            "gpu_launches_note": f"{launches} kernels per iteration summed over ranks (compute, halo, "
                                 f"signal, wait) x {a.steps}; plus {a.steps * world} L2-flush kernels",
            "roofline": flux_roof,
            "roofline_hbm": hbm_roof,
            "clocks": clk,
            "final_residue": float(residues[-1]) if len(residues) else None,
        }
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def main():
    a = parse()
    if a.impl == "reference":
        run_reference_arm(a)
    else:
        run_b200_arm(a)


if __name__ == "__main__":
    main()
