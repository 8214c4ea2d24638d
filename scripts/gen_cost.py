import time, sys, os
sys.path.insert(0, ".")
from paper_2403_13287_b200 import lskum as L
for rep in range(2):
    t = time.perf_counter(); c = L.Cloud.generate_naca0012(8000, 5000, 20.0, 0.0, 7, 8, frozen_wall=True)
    t1 = time.perf_counter(); c.close(); t2 = time.perf_counter()
    print(os.environ.get("LSKUM_PINNED_CLOUD", "1"), os.environ.get("LSKUM_PINNED_STORE", "1"), "gen %.2f close %.2f" % (t1 - t, t2 - t1), flush=True)
