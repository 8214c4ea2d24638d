"""Quick device-timing probe: free-stream sessions at several cloud sizes.

  python scripts/probe_perf.py [side ...]            rect side x side clouds
  PROBE_NACA=4000x2500 python scripts/probe_perf.py   NACA 0012 O-clouds (n_wall x n_rings, comma list)
  PROBE_FLUSH=1 ...                                    flush L2 before every timed iteration
"""
import sys, time, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_13287_b200 import lskum as L

clouds = []
if os.environ.get("PROBE_NACA"):
    for spec in os.environ["PROBE_NACA"].split(","):
        nw, nr = (int(v) for v in spec.split("x"))
        clouds.append((spec, lambda nw=nw, nr=nr: L.Cloud.generate_naca0012(nw, nr, 20.0, 0.0, 7, 8, frozen_wall=True)))
else:
    for side in [int(a) for a in sys.argv[1:]] or [200, 400, 790, 2000]:
        clouds.append((side, lambda side=side: L.Cloud.generate_rect(side, side, 0.1, 7, 8)))
for label, make in clouds:
    for order in [int(o) for o in os.environ.get("PROBE_ORDERS", "2,1").split(",")]:
        t0 = time.time()
        c = make()
        tg = time.time() - t0
        cfg = L.Config(mach=0.85, aoa=1.0, order=order, iters=60, fp_mode=os.environ.get("PROBE_FP", "fast"),
                       chunk=int(os.environ.get("PROBE_CHUNK", "16")))
        s = L.Session(c, cfg, capacity=60)
        s.iterate(10)
        if os.environ.get("PROBE_FLUSH"):  # L2 flushed before every iteration (bench.py's headline timing)
            ms = 0.0
            for _ in range(40):
                ms += s.step_flushed()
        else:
            ms = s.iterate(40)
        n = c.n
        k = s.kernels()
        print(json.dumps({"cloud": label, "n": n, "order": order, "fp": os.environ.get("PROBE_FP", "fast"),
                          "gen_s": round(tg, 2), "ms_per_it": ms / 40, "pt_it_s": n * 40 / (ms * 1e-3),
                          "kernels": [(a, round(b * 1e3 / max(cn, 1), 4), cn) for a, b, cn in k]}), flush=True)
        s.close()
