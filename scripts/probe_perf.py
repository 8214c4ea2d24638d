"""Quick device-timing probe: free-stream sessions at several cloud sizes."""
import sys, time, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_13287_b200 import lskum as L

sizes = [int(a) for a in sys.argv[1:]] or [200, 400, 790, 2000]
for side in sizes:
    for order in [int(o) for o in os.environ.get("PROBE_ORDERS", "2,1").split(",")]:
        t0 = time.time()
        c = L.Cloud.generate_rect(side, side, 0.1, 7, 8)
        tg = time.time() - t0
        cfg = L.Config(mach=0.85, aoa=1.0, order=order, iters=60, fp_mode=os.environ.get("PROBE_FP", "fast"))
        s = L.Session(c, cfg, capacity=60)
        s.iterate(10)
        ms = s.iterate(40)
        n = c.n
        k = s.kernels()
        print(json.dumps({"side": side, "n": n, "order": order, "fp": os.environ.get("PROBE_FP", "fast"), "lanes": os.environ.get("LSKUM_SWEEP_LANES", "2"), "gen_s": round(tg, 2),
                          "ms_per_it": ms / 40, "pt_it_s": n * 40 / (ms * 1e-3),
                          "kernels": [(a, round(b * 1e3 / max(cn, 1), 4), cn) for a, b, cn in k]}), flush=True)
        s.close()
