"""Host-phase trace of lskum_run (LSKUM_TRACE=1): where the end-to-end time goes."""
import os, sys, time
os.environ.setdefault("LSKUM_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_13287_b200 import lskum as L
spec = sys.argv[1] if len(sys.argv) > 1 else "520x308"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
nw, nr = (int(v) for v in spec.split("x"))
c = L.Cloud.generate_naca0012(nw, nr, 20.0, 0.0, 7, 8, frozen_wall=True)
cfg = L.Config(mach=0.85, aoa=1.0, iters=iters)
for rep in range(3):
    t0 = time.perf_counter()
    r = L.run(c, cfg)
    print(f"run {rep}: wall {time.perf_counter() - t0:.4f} s, device loop {r.total_seconds:.4f} s", flush=True)
    r.close()
