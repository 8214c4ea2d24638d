import sys, os, numpy as np
sys.path.insert(0, "/root/repo")
from paper_2403_13287_b200 import lskum as L
c = L.Cloud.generate_naca0012(520, 308, 20.0, 0.0, 7, 8, frozen_wall=True)
for chunk in (1, 16):
    for rep in range(2):
        r = L.run(c, L.Config(mach=0.85, aoa=1.0, iters=60, chunk=chunk))
        w = r.wall_ms()
        print(chunk, "device loop ms/it", r.total_seconds * 1e3 / 60, "median span ms", float(np.median(w[5:])), flush=True)
        r.close()
