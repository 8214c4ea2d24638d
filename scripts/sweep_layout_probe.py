"""Writes a NACA cloud's neighbour table for scripts/sweep_layout_probe.cu,
builds and runs it (on the GPU box).

  python scripts/sweep_layout_probe.py [n_wall x n_rings]
"""
import os, subprocess, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_13287_b200 import lskum as L

spec = sys.argv[1] if len(sys.argv) > 1 else "4000x2500"
nw, nr = (int(v) for v in spec.split("x"))
c = L.Cloud.generate_naca0012(nw, nr, 20.0, 0.0, 7, 8, frozen_wall=True)
g = c.geometry()
assert np.all(np.diff(g["off"]) == 8)
with open("/tmp/sweep_geo.bin", "wb") as f:
    np.array([c.n], np.int32).tofile(f)
    g["nbr"].astype(np.int32).tofile(f)
    np.stack([g["x"], g["y"]], 1).astype(np.float64).tofile(f)
here = os.path.dirname(os.path.abspath(__file__))
subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-o", "/tmp/sweep_layout_probe",
                os.path.join(here, "sweep_layout_probe.cu")], check=True)
subprocess.run(["/tmp/sweep_layout_probe", "/tmp/sweep_geo.bin"], check=True)
