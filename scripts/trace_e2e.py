"""Host-phase trace of lskum_run (LSKUM_TRACE=1): where the end-to-end time goes.

  python scripts/trace_e2e.py [n_wall x n_rings] [iters]
Runs lskum_run on a fresh cloud handle (cold: screening, geometry upload,
setup) and then again on the same handle (warm)."""
import os, sys, time
os.environ.setdefault("LSKUM_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_13287_b200 import lskum as L
spec = sys.argv[1] if len(sys.argv) > 1 else "520x308"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
nw, nr = (int(v) for v in spec.split("x"))
base = L.Cloud.generate_naca0012(nw, nr, 20.0, 0.0, 7, 8, frozen_wall=True)
g = base.geometry()
cfg = L.Config(mach=0.85, aoa=1.0, iters=iters)
L.run(L.Cloud.from_arrays(g["x"], g["y"], g["kind"], g["nx"], g["ny"], g["off"], g["nbr"]), cfg).close()
for rep in range(2):
    c = L.Cloud.from_arrays(g["x"], g["y"], g["kind"], g["nx"], g["ny"], g["off"], g["nbr"])
    for kind in ("cold", "warm"):
        print(f"--- {kind} run {rep}", file=sys.stderr, flush=True)
        t0 = time.perf_counter()
        r = L.run(c, cfg)
        print(f"{kind} run {rep}: wall {time.perf_counter() - t0:.4f} s, device loop {r.total_seconds:.4f} s",
              file=sys.stderr, flush=True)
        r.close()
