"""Cost of the flux's rare-path deferral on flows that take the rare paths
(profiling aid): free stream at the given Mach numbers on the NACA cloud,
iteration time with the deferral on (default) and off, in child processes.

  python scripts/defer_cost.py [n_wall x n_rings] [mach ...]
"""
import json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json
sys.path.insert(0, %(root)r)
from paper_2403_13287_b200 import lskum as L
nw, nr = %(nw)d, %(nr)d
c = L.Cloud.generate_naca0012(nw, nr, 20.0, 0.0, 7, 8, frozen_wall=True)
out = {}
for mach in %(machs)r:
    s = L.Session(c, L.Config(mach=mach, aoa=1.0, order=2, iters=20, cfl=0.1), capacity=20)
    try:
        s.iterate(2)
        ms = s.iterate(5)
        out[str(mach)] = round(ms / 5, 4)
    except L.LskumError as e:
        out[str(mach)] = str(e)[:80]
    s.close()
print(json.dumps(out))
'''
spec = sys.argv[1] if len(sys.argv) > 1 else "4000x2500"
machs = [float(m) for m in sys.argv[2:]] or [0.85, 1.2, 1.6, 2.0]
nw, nr = (int(v) for v in spec.split("x"))
code = CHILD % {"root": ROOT, "nw": nw, "nr": nr, "machs": machs}
for defer in ("1", "0"):
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, LSKUM_FLUX_DEFER=defer),
                       capture_output=True, text=True)
    print(json.dumps({"LSKUM_FLUX_DEFER": defer, "ms_per_iteration": json.loads(r.stdout.strip().splitlines()[-1])
                      if r.returncode == 0 else r.stderr[-400:]}), flush=True)
