"""A/B timing of library builds (kernel variants) on one cloud (profiling aid).

  python scripts/ab_kernels.py [--naca 4000x2500] [--reps 3] lib1.so lib2.so:VAR=value,VAR2=v ...
Each build runs in its own process (LSKUM_B200_LIB): a free-stream session on
the NACA cloud, 10 warm-up iterations, then per rep: 20 cold-L2 steps with
kernel events (first sweep, flux) and 40 back-to-back iterations.  Prints one
JSON line per build and rep (builds interleaved, so drift hits all alike).
"""
import argparse, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys, json, statistics, os
sys.path.insert(0, %(root)r)
from paper_2403_13287_b200 import lskum as L
nw, nr = %(nw)d, %(nr)d
c = L.Cloud.generate_naca0012(nw, nr, 20.0, 0.0, 7, 8, frozen_wall=True)
cfg = L.Config(mach=0.85, aoa=1.0, order=%(order)d, iters=200, fp_mode=%(fp)r)
s = L.Session(c, cfg, capacity=200)
s.iterate(10)
sw, fl, st = [], [], []
for _ in range(20):
    st.append(s.step_flushed(kernel_events=True))
    a, b = s.event_ms()
    sw.append(a); fl.append(b)
ms = s.iterate(40)
print(json.dumps({"lib": os.environ.get("LSKUM_B200_LIB"), "env": {k: v for k, v in os.environ.items() if k.startswith("LSKUM_") and k != "LSKUM_B200_LIB"}, "n": c.n, "sweep_ms": statistics.median(sw),
                  "flux_ms": statistics.median(fl), "step_ms_events": statistics.median(st),
                  "iter_ms": ms / 40, "kernels": [(k, round(v * 1e3 / max(n, 1), 4)) for k, v, n in s.kernels()]}))
'''

ap = argparse.ArgumentParser()
ap.add_argument("--naca", default="4000x2500")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--order", type=int, default=2)
ap.add_argument("--fp", default="fast")
ap.add_argument("libs", nargs="+")
a = ap.parse_args()
nw, nr = (int(v) for v in a.naca.split("x"))
code = CHILD % {"root": ROOT, "nw": nw, "nr": nr, "order": a.order, "fp": a.fp}
for rep in range(a.reps):
    for spec in a.libs:
        lib, _, extra = spec.partition(":")
        env = dict(os.environ, LSKUM_B200_LIB=os.path.abspath(lib))
        for kv in filter(None, extra.split(",")):
            k, v = kv.split("=", 1)
            env[k] = v
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else json.dumps({"lib": spec, "err": out.stderr[-500:]})
        print(line, flush=True)
