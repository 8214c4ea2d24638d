"""Host-phase trace of lskum_run (LSKUM_TRACE=1): where the end-to-end time goes."""
import os, sys, time
os.environ.setdefault("LSKUM_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_13287_b200 import lskum as L
side = int(sys.argv[1]) if len(sys.argv) > 1 else 400
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
c = L.Cloud.generate_rect(side, side, 0.1, 7, 8)
cfg = L.Config(mach=0.85, aoa=1.0, iters=iters)
for rep in range(3):
    t0 = time.perf_counter()
    r = L.run(c, cfg)
    print(f"run {rep}: wall {time.perf_counter() - t0:.4f} s, device loop {r.total_seconds:.4f} s", flush=True)
    r.close()
