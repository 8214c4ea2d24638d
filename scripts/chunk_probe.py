import sys, time
sys.path.insert(0, "/root/repo")
from paper_2403_13287_b200 import lskum as L
base = L.Cloud.generate_naca0012(520, 308, 20.0, 0.0, 7, 8, frozen_wall=True)
g = base.geometry()
L.run(L.Cloud.from_arrays(g["x"], g["y"], g["kind"], g["nx"], g["ny"], g["off"], g["nbr"]), L.Config(iters=5)).close()
for chunk in (2, 4, 10, 16, 50):
    cold, warm, dev = [], [], []
    for rep in range(3):
        c = L.Cloud.from_arrays(g["x"], g["y"], g["kind"], g["nx"], g["ny"], g["off"], g["nbr"])
        cfg = L.Config(mach=0.85, aoa=1.0, iters=50, chunk=chunk)
        t0 = time.perf_counter(); r = L.run(c, cfg); cold.append(time.perf_counter() - t0); r.close()
        t0 = time.perf_counter(); r = L.run(c, cfg); warm.append(time.perf_counter() - t0); dev.append(r.total_seconds); r.close()
    print(f"chunk {chunk:2d}: cold {min(cold)*1e3:.3f} ms  warm {min(warm)*1e3:.3f} ms  device loop {min(dev)*1e3:.3f} ms", flush=True)
