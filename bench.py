#!/usr/bin/env python
"""bench.py — LSKUM fixed-point iteration on B200: device-timed point-iterations/s.

Workload (BASELINE.json configs[4], the largest single-GPU configuration and
the strong-scaling one): a synthetic NACA 0012 O-cloud of 40,000,000 points
(8000 surface points x 5000 rings, far field at 20 chords, exact kNN k=8 — the
reference's build_stencils, bit for bit), M 0.85, alpha 1 deg, second order
with 3 inner derivative sweeps, CFL 0.5.  The surface ring is held at the free
stream (kind outer): the reference has no wall flux and its split stencils on
a curved wall are singular or unstable, so this is the NACA
point distribution both codes can run.  State: the free stream lskum_run
initialises — an exact fixed point with the full arithmetic cost.

One step = one fixed-point iteration over the whole cloud (3 sweeps, flux,
update, residue).  `value` times K steps with CUDA events on the engine's
stream, with the L2 flushed (384 MB overwrite) before every step (the working
set, ~13 GB, is far larger than L2 anyway): each step is one CUDA graph
[flush, start event, iteration, end event].  `e2e` times lskum_run through
the C ABI from host buffers (stencil screening, geometry upload, K
iterations, copy-back of the 21-slot store).  `--gpus N` is STRONG scaling:
the same 40M-point cloud split into N RCB pieces, one process per GPU
(torchrun; a plain `--gpus N` call re-launches itself under torchrun).

The reference arm (`--impl reference`) runs the reference's own lskum_run
(oracle/_ref/liblskum.so, built from /root/reference by oracle/Makefile) on the
same cloud, written as a grid file by a child process and parsed by the
reference's reader, on all host cores.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import socket
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


# BASELINE.json configs as NACA 0012 O-clouds (n_wall x n_rings): the sizes
# the configs name, with their Mach numbers and angles of attack.
CONFIG_SIZES = [("configs[0] ~40K, M=0.63 AoA=2", "260x154", 0.63, 2.0),
                ("configs[1] ~160K, M=0.85 AoA=1", "520x308", 0.85, 1.0),
                ("configs[2] ~625K, M=1.2 AoA=0", "1000x625", 1.2, 0.0),
                ("configs[3] ~10M, M=0.85 AoA=1", "4000x2500", 0.85, 1.0),
                ("configs[4] ~40M, M=0.85 AoA=1", "8000x5000", 0.85, 1.0)]


# ---------------------------------------------------------------------------
def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--naca", default="8000x5000", help="NACA 0012 cloud n_wall x n_rings (whole job)")
    ap.add_argument("--config-label", default="configs[4]")
    ap.add_argument("--order", type=int, default=2)
    ap.add_argument("--inner", type=int, default=3)
    ap.add_argument("--mach", type=float, default=0.85)
    ap.add_argument("--aoa", type=float, default=1.0)
    ap.add_argument("--fp-mode", default="fast")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sizes", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--ref-iters", type=int, default=3,
                    help="reference iterations per timed lskum_run on the workload cloud (bounded sample)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    return world, rank, local, local_world


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


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


def naca_dims(spec):
    nw, nr = (int(v) for v in spec.lower().split("x"))
    return nw, nr


def workload_text(a):
    nw, nr = naca_dims(a.naca)
    return (f"synthetic NACA 0012 O-cloud {nw}x{nr} (n_wall x n_rings, far field 20 chords, kNN k=8; surface "
            f"points held at the free stream because the reference has no wall flux); {nw * nr:,} points, "
            f"BASELINE {a.config_label}; M={a.mach}, AoA={a.aoa}, order {a.order}, {a.inner} inner sweeps; "
            "free-stream state")


def config_block(a, n, extra=None):
    c = {"workload": workload_text(a),
         "n_points": n, "stencil": "kNN k=8 (exact, bit-identical to the reference's build_stencils)",
         "order": a.order, "inner": a.inner, "mach": a.mach, "aoa_deg": a.aoa, "cfl": 0.5,
         "fp_mode": a.fp_mode,
         "l2": "flushed before every timed step (384 MB overwrite in the same CUDA graph, ahead of the step's "
               "start event); working set ~330 B/point, far larger than the 126 MB L2",
         "parallelism": "single-domain"}
    if extra:
        c.update(extra)
    return c


# ---------------------------------------------------------------------------
# The reference's own implementation (oracle/_ref, built from /root/reference
# by oracle/Makefile) — the CPU baseline and the reference arm.  Test/baseline
# infrastructure only; the product path never touches oracle/.
def reference_lib():
    so = os.path.join(ROOT, "oracle", "_ref", "liblskum.so")
    if not os.path.exists(so):
        return None
    L = ctypes.CDLL(so)
    vp = ctypes.c_void_p
    L.lskum_cloud_read_file.argtypes = [ctypes.c_char_p, ctypes.POINTER(vp)]
    L.lskum_cloud_n_points.argtypes = [vp]
    L.lskum_config_create.argtypes = [ctypes.POINTER(vp)]
    L.lskum_config_set.argtypes = [vp, ctypes.c_char_p, ctypes.c_char_p]
    L.lskum_run.argtypes = [vp, vp, ctypes.POINTER(vp)]
    L.lskum_result_total_seconds.argtypes = [vp]
    L.lskum_result_total_seconds.restype = ctypes.c_double
    L.lskum_result_iterations.argtypes = [vp]
    L.lskum_result_destroy.argtypes = [vp]
    L.lskum_cloud_destroy.argtypes = [vp]
    L.lskum_config_destroy.argtypes = [vp]
    L.lskum_last_error.restype = ctypes.c_char_p
    return L


def write_grid_in_child(a, path):
    """The workload cloud as a grid file (the reference's format), written by a
    child process so the process that times the reference never maps this
    repo's library."""
    nw, nr = naca_dims(a.naca)
    code = ("import sys; sys.path.insert(0, %r); from paper_2403_13287_b200 import lskum as L; "
            "L.Cloud.generate_naca0012(%d, %d, 20.0, 0.0, 7, 8, frozen_wall=True).write_file(%r)"
            % (ROOT, nw, nr, path))
    subprocess.run([sys.executable, "-c", code], check=True)


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
    L.lskum_config_destroy(cfg)
    if rc != 0:
        raise RuntimeError(L.lskum_last_error().decode())
    secs = L.lskum_result_total_seconds(res)
    L.lskum_result_destroy(res)
    return secs, wall


def reference_measure(a, iters):
    """The reference's lskum_run on the workload cloud: `iters` iterations on
    all host cores, timed by the reference's own loop timer
    (runtime.cpp:237-271: the iteration loop only — setup, validation and
    partitioning excluded, as the reference measures itself)."""
    L = reference_lib()
    if L is None:
        return None
    threads = os.cpu_count() or 1
    with tempfile.TemporaryDirectory(dir="/dev/shm" if os.path.isdir("/dev/shm") else None) as d:
        path = os.path.join(d, "workload.grid")
        write_grid_in_child(a, path)
        h = ctypes.c_void_p()
        t0 = time.perf_counter()
        if L.lskum_cloud_read_file(path.encode(), ctypes.byref(h)) != 0:
            raise RuntimeError(L.lskum_last_error().decode())
        parse_s = time.perf_counter() - t0
    n = L.lskum_cloud_n_points(h)
    secs, wall = reference_run(L, h, a, iters, threads)
    L.lskum_cloud_destroy(h)
    return {"value": n * iters / secs, "unit": UNIT, "cores": threads, "kind": "reference", "cpu": cpu_model(),
            "sample": f"{iters} iterations of the {n:,}-point workload cloud through the reference's lskum_run "
                      f"(oracle/_ref/liblskum.so, built from /root/reference/proj; parts=workers={threads}, soa, "
                      f"fused), reference loop timer {secs:.2f} s; the cloud read from the same grid file by the "
                      f"reference's parser ({parse_s:.1f} s); lskum_run wall incl. validation and partitioning "
                      f"{wall:.1f} s",
            "n_points": n, "seconds": secs}


def run_reference_arm(a):
    world, rank, _, _ = dist_env()
    if rank != 0:
        return
    base = reference_measure(a, max(1, min(a.steps, a.ref_iters)))
    nw, nr = naca_dims(a.naca)
    if base is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/liblskum.so not built"}), flush=True)
        return
    n = base["n_points"]
    value = base["value"]
    out = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
           "steps": a.steps, "warmup": a.warmup, "ms_per_step": n / value * 1e3,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": config_block(a, n, {"parallelism": f"{base['cores']} host threads"}),
           "cpu_baseline": {k: base[k] for k in ("value", "unit", "cores", "kind", "cpu", "sample")},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "note": f"each step is one full iteration over the {n:,}-point cloud; {base['sample'].split(';')[0]} "
                   "(a bounded sample: one reference iteration at this size takes seconds)"}
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------------------
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
            "peak_source": "DFMA microbenchmark on this GPU (lskum_b200_fp64_peak); MEASURED_PEAKS.json has no FP64 "
                           "entry",
            "flops_source": f"ncu dynamic 2*DFMA+DADD+DMUL = {flops_pt:.0f} per point "
                            "(profiles/flux_ncu_counts.json)" if flops_pt else None,
            "launch_ms": flux_ms}
    hbmr = {"bound": "hbm", "kernel": "k_sweep_tile (derivative sweep: stencil unions of 128-point tiles staged in "
                                      "shared memory by TMA bulk copies)", "achieved": sweep_gbs, "peak": hbm,
            "unit": "GB/s", "frac": sweep_gbs / hbm if sweep_gbs else None,
            "algorithmic_bytes_per_point": sweep_bytes(k), "launch_ms": sweep_ms, "peak_source": hbm_kind,
            "iteration_achieved_gbs_per_gpu": iter_gbs, "iteration_frac": iter_gbs / hbm,
            "iteration_bytes_per_point": iteration_bytes(k, order, inner)}
    return flux, hbmr


def make_cloud(L, a):
    nw, nr = naca_dims(a.naca)
    return L.Cloud.generate_naca0012(nw, nr, 20.0, 0.0, 7, 8, frozen_wall=True)


def sizes_run(L, a, big=None, iters=30):
    """Device-timed throughput at every BASELINE config size, order 2 and 1
    (back-to-back iterations in captured graphs, after 10 warm-up iterations)."""
    out = []
    for label, spec, mach, aoa in CONFIG_SIZES:
        nw, nr = naca_dims(spec)
        cloud = big if (big is not None and big.n == nw * nr) else \
            L.Cloud.generate_naca0012(nw, nr, 20.0, 0.0, 7, 8, frozen_wall=True)
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


def relaunch_under_torchrun(a):
    """`bench.py --gpus N` (N > 1) outside torchrun: one process per GPU."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.run(cmd).returncode)


def run_b200_arm(a):
    world, rank, local, local_world = dist_env()
    if world > 1:
        return run_b200_ranks(a, world, rank, local, local_world)
    if a.gpus > 1:
        return relaunch_under_torchrun(a)
    from paper_2403_13287_b200 import lskum as L
    t_setup = time.perf_counter()
    cloud = make_cloud(L, a)
    n = cloud.n
    k = cloud.nnz // n
    g = cloud.geometry()
    n_flux = int(np.count_nonzero(g["kind"] != 2))
    cfg = L.Config(mach=a.mach, aoa=a.aoa, order=a.order, inner=a.inner, cfl=0.5, fp_mode=a.fp_mode,
                   iters=a.steps, device=0)
    with ClockSampler(0) as clocks:
        sess = L.Session(cloud, cfg, capacity=a.warmup + 2 * a.steps + 4)
        setup_s = time.perf_counter() - t_setup
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
        residues = sess.residues()
        sess.close()
    clk = clocks.summary()
    total_ms = sum(step_ms)
    value = n * a.steps / (total_ms * 1e-3)

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": total_ms / a.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (free-stream state on a generated cloud)",
        "config": config_block(a, n),
        "gpu_launches": launches * a.steps,
        "gpu_launches_note": f"{launches} kernels per iteration x {a.steps}; plus {a.steps} L2-flush kernels "
                             "between steps",
    }
    counts = load_counts()
    flux_roof, hbm_roof = rooflines(L, counts, n, n_flux, k, a.order, a.inner, total_ms / a.steps,
                                    statistics.mean(sweep_ms) if a.order == 2 else None, statistics.mean(flux_ms))
    out["roofline"] = flux_roof
    out["roofline_hbm"] = hbm_roof
    out["clocks"] = clk
    out["final_residue"] = float(residues[-1]) if len(residues) else None
    out["setup_s"] = setup_s

    if not a.no_e2e:
        # e2e through the drop-in C ABI (lskum_run) from host buffers.  Cold: a
        # fresh cloud handle built from host arrays (outside the timer), so the
        # timed call screens the stencils, uploads the geometry (H2D), sets up
        # the device domain, initialises the free stream, runs K iterations and
        # copies the 21-slot store back (D2H).  Warm: a second lskum_run on that
        # handle (the cloud's device domain stays resident between calls).
        arrays = (g["x"], g["y"], g["kind"], g["nx"], g["ny"], g["off"], g["nbr"])
        e2e_cfg = L.Config(mach=a.mach, aoa=a.aoa, order=a.order, inner=a.inner, cfl=0.5,
                           fp_mode=a.fp_mode, iters=a.steps, device=0)
        # process warm-up outside the timer: CUDA context, module load and the
        # grow-only pinned staging the copies run through (a same-size run on
        # another handle), so the timed copies start from pinned host memory
        warm = L.Cloud.from_arrays(*arrays)
        L.run(warm, e2e_cfg).close()
        warm.close()
        e2e_cloud = L.Cloud.from_arrays(*arrays)
        t0 = time.perf_counter()
        res = L.run(e2e_cloud, e2e_cfg)
        e2e_wall = time.perf_counter() - t0
        res.close()
        t0 = time.perf_counter()
        res = L.run(e2e_cloud, e2e_cfg)
        e2e_warm = time.perf_counter() - t0
        res.close()
        e2e_cloud.close()
        nnz = cloud.nnz
        # what lskum_run moves H2D for this cloud (engine Domain: straight from the
        # cloud's pinned arrays): x and y, kinds, stencil ids; uniform stencils'
        # offsets are generated on the device, normals only sent for wall points
        # (none here), partition ids only when non-zero (one partition)
        h2d = n * (8 + 8 + 1) + 4 * nnz
        d2h = n * 21 * 8 + 8 * a.steps                       # 21-slot store + residue history
        out["e2e"] = {"value": n * a.steps / e2e_wall, "unit": UNIT,
                      "h2d_bytes_per_step": int(h2d / a.steps), "d2h_bytes_per_step": int(d2h / a.steps),
                      "what": "wall time of lskum_run (C ABI) on a fresh cloud handle: stencil screening, geometry "
                              f"H2D, device setup, free-stream init, {a.steps} iterations, copy-back of the 21-slot "
                              "store (D2H)",
                      "warm": {"value": n * a.steps / e2e_warm, "h2d_bytes_per_step": 0,
                               "d2h_bytes_per_step": int(d2h / a.steps),
                               "what": "second lskum_run on the same cloud handle: geometry, weights and graphs "
                                       "stay resident; free stream initialised on the device"}}
    if not a.no_sizes:
        out["sizes"] = sizes_run(L, a, big=cloud)
    cloud.close()
    if not a.no_cpu_baseline:
        base = reference_measure(a, max(1, min(a.steps, a.ref_iters)))
        if base is not None:
            out["cpu_baseline"] = {k: base[k] for k in ("value", "unit", "cores", "kind", "cpu", "sample")}
    print(json.dumps(out), flush=True)


def run_b200_ranks(a, world, rank, local, local_world):
    """torchrun: one process per GPU, each running its RCB piece of the SAME
    cloud (strong scaling; RankSession).

    Halo exchange is device-to-device over CUDA IPC (NVLink peer memory),
    ordered by device-side progress counters; the residue is each rank's exact
    fixed-point partial, summed by rank 0's residue kernel over peer memory.
    The gloo group only carries setup, per-step barriers and the max-over-ranks
    timing.
    """
    # the host's cores are shared by the ranks of this node (setup work only)
    os.environ.setdefault("LSKUM_HOST_THREADS", str(max(1, (os.cpu_count() or 1) // max(1, local_world))))
    import torch
    import torch.distributed as dist

    from paper_2403_13287_b200 import lskum as L

    dist.init_process_group("gloo")
    ndev = max(1, torch.cuda.device_count())
    device = local % ndev
    a.gpus = world
    t_setup = time.perf_counter()
    cloud = make_cloud(L, a)
    n = cloud.n
    k = cloud.nnz // n
    n_flux = int(np.count_nonzero(cloud.geometry()["kind"] != 2))
    cfg = L.Config(mach=a.mach, aoa=a.aoa, order=a.order, inner=a.inner, cfl=0.5, fp_mode=a.fp_mode,
                   iters=a.steps)
    step_ms, sweep_ms, flux_ms = [], [], []
    with ClockSampler(device) as clocks:
        sess = L.RankSession(cloud, cfg, rank, world, device, capacity=a.warmup + a.steps + 4)
        setup_s = time.perf_counter() - t_setup
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
    e2e_wall = None
    if not a.no_e2e:
        # e2e: host arrays -> this rank's piece on its GPU -> K iterations -> copy-back
        cloud.reset_store(0)
        dist.barrier()
        t0 = time.perf_counter()
        with L.RankSession(cloud, cfg, rank, world, device, capacity=a.steps) as es:
            es.iterate(a.steps)
            es.download()
        e2e_wall = time.perf_counter() - t0
    nnz = cloud.nnz
    cloud.close()
    mine = {"step_ms": step_ms, "sweep_ms": statistics.mean(sweep_ms) if a.order == 2 else None,
            "flux_ms": statistics.mean(flux_ms), "e2e_wall": e2e_wall, "launches": launches,
            "clocks": clocks.summary(), "setup_s": setup_s}
    everyone = [None] * world
    dist.all_gather_object(everyone, mine)
    if rank == 0:
        step_max = np.max(np.array([e["step_ms"] for e in everyone]), axis=0)  # max over ranks, per step
        total_ms = float(step_max.sum())
        value = n * a.steps / (total_ms * 1e-3)
        flux_avg = max(e["flux_ms"] for e in everyone)
        counts = load_counts()
        sweep_avg = max(e["sweep_ms"] for e in everyone) if a.order == 2 else None
        flux_roof, hbm_roof = rooflines(L, counts, n, n_flux, k, a.order, a.inner, total_ms / a.steps, sweep_avg,
                                        flux_avg, device, world)
        h2d = n * (16 + 16 + 1 + 2 + 32) + 4 * (n + 1) + 4 * nnz
        d2h = n * 21 * 8 + 8 * a.steps
        clk = dict(everyone[0]["clocks"])
        clk["reasons"] = sorted({r for e in everyone for r in e["clocks"]["reasons"]})
        clk["per_rank_sm_mhz"] = [e["clocks"]["sm_mhz"] for e in everyone]
        launches = sum(e["launches"] for e in everyone)
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": total_ms / a.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (free-stream state on a generated cloud)",
            "config": config_block(a, n, {"parallelism": f"rcb{world}: the same cloud in {world} RCB pieces, one "
                                                         "process per GPU, CUDA-IPC peer-memory halos, device-side "
                                                         "progress counters, exact per-rank residue partials"}),
            "gpu_launches": launches * a.steps,
            "gpu_launches_note": f"{launches} kernels per iteration summed over ranks (compute, halo, "
                                 f"signal, wait) x {a.steps}; plus {a.steps * world} L2-flush kernels",
            "roofline": flux_roof,
            "roofline_hbm": hbm_roof,
            "clocks": clk,
            "per_rank_ms_per_step": [statistics.mean(e["step_ms"]) for e in everyone],
            "final_residue": float(residues[-1]) if len(residues) else None,
            "setup_s": max(e["setup_s"] for e in everyone),
        }
        if e2e_wall is not None:
            wall = max(e["e2e_wall"] for e in everyone)
            out["e2e"] = {"value": n * a.steps / wall, "unit": UNIT,
                          "h2d_bytes_per_step": int(h2d / a.steps), "d2h_bytes_per_step": int(d2h / a.steps),
                          "what": "max over ranks of RankSession create (screening, upload of the rank's piece), "
                                  f"{a.steps} iterations, copy-back of owned points"}
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
