"""Repeated cold lskum_run on fresh 40M cloud handles (profiling aid): the
spread of the end-to-end time across handles, with the pinned-memory options
of the environment (LSKUM_PINNED_CLOUD / LSKUM_PINNED_STORE).

  python scripts/e2e_reps.py [n_wall x n_rings] [reps]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_13287_b200 import lskum as L
spec = sys.argv[1] if len(sys.argv) > 1 else "8000x5000"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
nw, nr = (int(v) for v in spec.split("x"))
base = L.Cloud.generate_naca0012(nw, nr, 20.0, 0.0, 7, 8, frozen_wall=True)
g = base.geometry()
base.close()
arrays = (g["x"], g["y"], g["kind"], g["nx"], g["ny"], g["off"], g["nbr"])
cfg = L.Config(mach=0.85, aoa=1.0, iters=20)
tag = f"cloud={os.environ.get('LSKUM_PINNED_CLOUD', '1')} store={os.environ.get('LSKUM_PINNED_STORE', '1')}"
for rep in range(reps):
    t0 = time.perf_counter()
    c = L.Cloud.from_arrays(*arrays)
    t1 = time.perf_counter()
    r = L.run(c, cfg)
    t2 = time.perf_counter()
    r.close()
    r = L.run(c, cfg)
    t3 = time.perf_counter()
    r.close()
    c.close()
    t4 = time.perf_counter()
    print(f"{tag} rep {rep}: create {t1 - t0:.3f} s, cold run {t2 - t1:.4f} s, warm run {t3 - t2:.4f} s, "
          f"close {t4 - t3:.3f} s", flush=True)
