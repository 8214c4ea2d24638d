"""Tiled derivative sweep (engine dev/tiles.cuh), GPU tests.

The tiled sweep stages each tile's stencil union in shared memory with bulk
copies and gathers from there; tiles that do not fit the plan (too many id
intervals, too many staged points) are gathered from global memory by the same
kernel.  The per-point arithmetic is shared with the untiled sweep (k_sweep2,
kernels.cuh sweep_point8), so whole runs must be BITWISE those of the untiled
sweep (LSKUM_SWEEP_TILE=0, run in a child process) in both arithmetic modes —
on the BASELINE NACA clouds (every tile staged), on a cloud whose second half
is shuffled (staged and global tiles mixed) and on RCM / Hilbert device orders.
The untiled sweep itself is pinned to the reference by the per-kernel and
whole-run parity tests (test_gpu_kernels.py, test_gpu_parity_configs.py).
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2403_13287_b200 import lskum as L

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MACH, AOA = 0.85, 1.0


def naca(nw, nr):
    return L.Cloud.generate_naca0012(nw, nr, 20.0, 0.0, 7, 8, frozen_wall=True)


def bumped(c, amp=0.02):
    g = c.geometry()
    a = np.radians(AOA)
    prim = np.tile([1.0, MACH * np.cos(a), MACH * np.sin(a), 1.0 / 1.4], (c.n, 1))
    r2 = (g["x"] + 0.5) ** 2 + (g["y"] - 0.3) ** 2
    w = amp * np.exp(-r2 / 0.02)
    prim[:, 0] *= 1.0 + w
    prim[:, 3] *= 1.0 + w
    return prim


def half_shuffled(c, seed=3):
    """The cloud with the ids of its second half randomly relabelled (stencil
    order kept): tiles there gather from global memory, the first half stages."""
    g = c.geometry()
    n = c.n
    order = np.arange(n)
    order[n // 2:] = n // 2 + np.random.default_rng(seed).permutation(n - n // 2)
    inv = np.empty(n, dtype=np.int64)
    inv[order] = np.arange(n)
    off = g["off"]
    cnt = np.diff(off)[order]
    noff = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
    src = np.arange(noff[-1]) + np.repeat(off[:-1][order] - noff[:-1], cnt)
    nbr = inv[g["nbr"][src]].astype(np.int32)
    return L.Cloud.from_arrays(g["x"][order], g["y"][order], g["kind"][order], g["nx"][order],
                               g["ny"][order], noff, nbr)


CHILD = r'''
import sys, json
import numpy as np
sys.path.insert(0, %(root)r)
sys.path.insert(0, %(tests)r)
from paper_2403_13287_b200 import lskum as L
from test_gpu_tiles import *
c = {maker}
c.set_primitives(bumped(c))
res = L.run_fixed_point(c, L.Config(mach=MACH, aoa=AOA, iters={iters}, order=2, inner=3, cfl=0.5,
                                    fp_mode={fp!r}, reorder={reorder!r}))
np.save({out!r} + "_res.npy", res.residues())
np.save({out!r} + "_f.npy", c.fields())
'''


def untiled(maker, iters, fp, reorder, tmp_path):
    out = str(tmp_path / "untiled")
    code = (CHILD % {"root": ROOT, "tests": os.path.join(ROOT, "tests")}).format(
        maker=maker, iters=iters, fp=fp, reorder=reorder, out=out)
    env = dict(os.environ, LSKUM_SWEEP_TILE="0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out + "_res.npy"), np.load(out + "_f.npy")


def tiled(c, iters, fp, reorder):
    c.set_primitives(bumped(c))
    cfg = L.Config(mach=MACH, aoa=AOA, iters=iters, order=2, inner=3, cfl=0.5, fp_mode=fp, reorder=reorder)
    s = L.Session(c, cfg, capacity=iters, from_state=True)
    tiles = s.tiles()
    s.close()
    c.set_primitives(bumped(c))
    res = L.run_fixed_point(c, cfg)
    return tiles, res.residues(), c.fields()


@pytest.mark.parametrize("dims", [(250, 160), (520, 308), (1000, 625), (4000, 2500)])
def test_tile_plan_stages_the_naca_clouds(dims):
    c = naca(*dims)
    s = L.Session(c, L.Config(mach=MACH, aoa=AOA, order=2, iters=1), capacity=1)
    staged, total = s.tiles()
    s.close()
    assert total == (c.n + 127) // 128  # default tile shape: 128 points
    # a few tiles at the trailing edge, where kNN stencils reach several rings
    # out, exceed the stage and are gathered from global memory
    assert staged >= 0.97 * total, (staged, total)


@pytest.mark.parametrize("fp", ["fast", "strict"])
@pytest.mark.parametrize("case", [
    ("naca(1000, 625)", "none", 4),
    ("half_shuffled(naca(400, 200))", "none", 4),
    ("naca(400, 200)", "rcm", 3),
    ("naca(400, 200)", "hilbert", 3),
])
def test_tiled_sweep_is_bitwise_the_untiled_sweep(case, fp, tmp_path):
    maker, reorder, iters = case
    c = eval(maker)
    tiles, res, f = tiled(c, iters, fp, reorder)
    want_res, want_f = untiled(maker, iters, fp, reorder, tmp_path)
    assert tiles[1] > 0
    if maker.startswith("half"):
        assert 0 < tiles[0] < tiles[1], tiles  # both tile kinds ran
    assert np.array_equal(res, want_res)
    assert np.array_equal(f, want_f)
    assert np.any(f[:, 8:16] != 0.0)  # derivatives were exercised
