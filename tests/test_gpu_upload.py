"""Geometry upload and copy-back paths of lskum_run (GPU tests).

Large clouds keep their per-point arrays in pinned host memory (HostAlloc,
host/core.hpp) and the engine uploads them with DMAs straight from those
arrays; with LSKUM_PINNED_CLOUD=0 (heap arrays) the same geometry goes through
pinned staging in point chunks.  The copy-back packs the 21-slot store on the
device and copies it in point chunks on two streams; with LSKUM_ZERO_COPY=1 the
pack kernel writes the pinned store directly.  Whatever the path, the results
must be bitwise the same: a 10M-point run (direct upload, chunked copy-back) is
compared with the same run in a child process on heap arrays (staged upload)
with the zero-copy store, in both store layouts.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2403_13287_b200 import lskum as L

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys
import numpy as np
sys.path.insert(0, {root!r})
sys.path.insert(0, {tests!r})
from paper_2403_13287_b200 import lskum as L
from test_gpu_upload import case
res, f = case({layout})
np.save({out!r} + "_res.npy", res)
np.save({out!r} + "_f.npy", f)
'''


def case(layout):
    c = L.Cloud.generate_naca0012(4000, 2500, 20.0, 0.0, 7, 8, frozen_wall=True)
    c.reset_store(0)
    g = c.geometry()
    a = np.radians(1.0)
    prim = np.tile([1.0, 0.85 * np.cos(a), 0.85 * np.sin(a), 1.0 / 1.4], (c.n, 1))
    w = 0.02 * np.exp(-((g["x"] + 0.5) ** 2 + (g["y"] - 0.3) ** 2) / 0.02)
    prim[:, 0] *= 1.0 + w
    prim[:, 3] *= 1.0 + w
    c.set_primitives(prim)
    res = L.run_fixed_point(c, L.Config(mach=0.85, aoa=1.0, iters=3, order=2, inner=3, cfl=0.5, layout=layout))
    return res.residues(), c.fields()


@pytest.mark.parametrize("layout", ["aos", "soa"])
def test_direct_upload_and_chunked_copy_back_are_bitwise_the_staged_paths(layout, tmp_path):
    res, f = case(layout)
    out = str(tmp_path / "heap")
    code = CHILD.format(root=ROOT, tests=os.path.join(ROOT, "tests"), layout=repr(layout), out=out)
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, LSKUM_PINNED_CLOUD="0", LSKUM_ZERO_COPY="1"),
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    assert np.array_equal(res, np.load(out + "_res.npy"))
    assert np.array_equal(f, np.load(out + "_f.npy"))
    assert np.any(f[:, 8:16] != 0.0) and np.all(np.isfinite(f))


def test_fresh_handles_reuse_the_device_scratch_bitwise():
    """The copy-back's packed store and the screening buffers live in grow-only
    per-device scratch shared by the process's domains (engine.cu ScratchLease):
    a smaller cloud after a larger one, then the larger again, each on a fresh
    handle, give the same bits as the first run of that size."""
    def run(nw, nr):
        c = L.Cloud.generate_naca0012(nw, nr, 20.0, 0.0, 7, 8, frozen_wall=True)
        c.reset_store(0)
        g = c.geometry()
        a = np.radians(1.0)
        prim = np.tile([1.0, 0.85 * np.cos(a), 0.85 * np.sin(a), 1.0 / 1.4], (c.n, 1))
        prim[:, 0] *= 1.0 + 0.02 * np.exp(-((g["x"] + 0.5) ** 2 + (g["y"] - 0.3) ** 2) / 0.02)
        c.set_primitives(prim)
        res = L.run_fixed_point(c, L.Config(mach=0.85, aoa=1.0, iters=3, order=2, inner=3, cfl=0.5))
        out = (res.residues(), c.fields())
        c.close()
        return out

    big1 = run(1000, 625)
    small = run(400, 200)
    big2 = run(1000, 625)
    assert np.array_equal(big1[0], big2[0]) and np.array_equal(big1[1], big2[1])
    assert small[1].shape[0] == 80000 and np.all(np.isfinite(small[1]))
