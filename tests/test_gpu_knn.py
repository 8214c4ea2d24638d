"""GPU kNN queries (engine k_knn on attach_knn's 2-d tree), GPU tests.

The generators' stencils are the reference's build_stencils (cloud.cpp:137-237):
the exact k nearest by (d^2, id), ids ascending — pinned against the reference
on small clouds by test_naca.py / test_oracle_pinning.py through the host
kd-tree.  Above 64K points the tree is queried on the GPU; the stencils must be
identical to the host queries (LSKUM_GPU_KNN=0, in a child process) on a
graded NACA O-cloud, a jittered rectangle and an exact lattice (equal distances:
the id tie-break decides).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2403_13287_b200 import lskum as L

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MAKERS = {
    "naca": "L.Cloud.generate_naca0012(900, 400, 20.0, 0.0, 7, 8, frozen_wall=True)",
    "rect_jitter": "L.Cloud.generate_rect(500, 400, 0.3, 11, 8)",
    "lattice": "L.Cloud.generate_rect(400, 300, 0.0, 1, 8)",
    "naca_k6": "L.Cloud.generate_naca0012(600, 300, 20.0, 0.05, 3, 6)",
}


@pytest.mark.parametrize("case", sorted(MAKERS))
def test_gpu_knn_equals_host_knn(case, tmp_path):
    c = eval(MAKERS[case])
    assert c.n >= 1 << 16
    g = c.geometry()
    out = str(tmp_path / "host.npy")
    code = (f"import sys, numpy as np\nsys.path.insert(0, {ROOT!r})\n"
            f"from paper_2403_13287_b200 import lskum as L\nc = {MAKERS[case]}\n"
            f"np.save({out!r}, c.geometry()['nbr'])\n")
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, LSKUM_GPU_KNN="0"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert np.array_equal(g["nbr"], np.load(out))
