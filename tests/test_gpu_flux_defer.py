"""Rare-path deferral of the staged flux kernel (GPU tests).

k_flux_ws<.., DEFER> evaluates every pair without the rare fallbacks — the
libdevice erf above |s| = 1.5 (a local normal Mach number above ~1.8), the
exponential outside its range, the invalid-state and singular-split failure
checks — and lists the points whose evaluation needed one; k_flux_redo then
recomputes exactly those points with the fallbacks in place (kernels.cuh).
A supersonic flow takes the erf fallback on every pair, so every point goes
through the redo list.  Checked here: against the oracle (the reference's
algorithm, kinetic.cpp:38-111) within the 1e-12 / 1e-10 tolerances, and
bitwise against runs with the fallbacks inline (LSKUM_FLUX_DEFER=0, child
process) on NACA and rectangle clouds at M = 2 and 2.5.  The failure paths
through the redo list are covered by the abort parity tests
(test_gpu_runs.py, test_gpu_parity_configs.py), which run with deferral on.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import pyoracle as P
from conftest import rel_err
from paper_2403_13287_b200 import lskum as L

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("order", [1, 2])
def test_supersonic_flux_through_the_redo_list_matches_oracle(order):
    mach, aoa = 2.5, 3.0
    c = P.orc_generate_rect(24, 24, 0.1, 5, 8)
    prim0 = P.center_bump(c, mach=mach, aoa=aoa)
    want = P.orc_run(c, mach=mach, aoa=aoa, iters=5, order=order, prim0=prim0)
    assert want.code == 0, want.msg
    pc = L.Cloud.from_arrays(c.x, c.y, c.kind, c.nx, c.ny, c.off, c.nbr)
    pc.reset_store(0)
    pc.set_primitives(prim0)
    res = L.run_fixed_point(pc, L.Config(mach=mach, aoa=aoa, iters=5, inner=3, cfl=0.5, order=order))
    f = pc.fields()
    assert res.iterations == 5
    assert rel_err(f[:, 0:4], want.store[:, 0:4]) <= 1e-12
    live = c.kind != 2
    assert rel_err(f[live, 16:20], want.store[live, 16:20]) <= 1e-10
    r, w = np.asarray(res.residues()), np.asarray(want.residue)
    assert float(np.max(np.abs(r - w) / np.abs(w))) <= 1e-10


CHILD = r'''
import sys
import numpy as np
sys.path.insert(0, {root!r})
sys.path.insert(0, {tests!r})
sys.path.insert(0, {oracle!r})
from test_gpu_flux_defer import supersonic
res, f = supersonic({maker!r}, {mach}, {iters})
np.save({out!r} + "_res.npy", res)
np.save({out!r} + "_f.npy", f)
'''


def supersonic(maker, mach, iters):
    if maker.startswith("naca"):
        nw, nr = (int(v) for v in maker[4:].split("x"))
        c = L.Cloud.generate_naca0012(nw, nr, 20.0, 0.0, 7, 8, frozen_wall=True)
        xc, yc = -0.5, 0.3
    else:
        nx, ny = (int(v) for v in maker[4:].split("x"))
        c = L.Cloud.generate_rect(nx, ny, 0.0, 0, 8)  # unjittered: zero-offset pairs too
        xc, yc = 0.5, 0.5
    c.reset_store(0)
    g = c.geometry()
    a = np.radians(1.0)
    prim = np.tile([1.0, mach * np.cos(a), mach * np.sin(a), 1.0 / 1.4], (c.n, 1))
    w = 0.05 * np.exp(-((g["x"] - xc) ** 2 + (g["y"] - yc) ** 2) / 0.02)
    prim[:, 0] *= 1.0 + w
    prim[:, 3] *= 1.0 + w
    c.set_primitives(prim)
    res = L.run_fixed_point(c, L.Config(mach=mach, aoa=1.0, iters=iters, order=2, inner=3, cfl=0.5))
    return res.residues(), c.fields()


@pytest.mark.parametrize("maker,mach,iters", [("naca1000x625", 2.0, 3), ("naca400x200", 2.0, 5),
                                              ("rect60x40", 2.5, 5)])
def test_deferred_rare_paths_are_bitwise_the_inline_fallbacks(maker, mach, iters, tmp_path):
    res, f = supersonic(maker, mach, iters)
    out = str(tmp_path / "inline")
    code = CHILD.format(root=ROOT, tests=os.path.join(ROOT, "tests"), oracle=os.path.join(ROOT, "oracle"),
                        maker=maker, mach=mach, iters=iters, out=out)
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, LSKUM_FLUX_DEFER="0"),
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    assert np.array_equal(res, np.load(out + "_res.npy"))
    assert np.array_equal(f, np.load(out + "_f.npy"))
    assert np.any(f[:, 16:20] != 0.0) and np.all(np.isfinite(f))


def _supersonic_naca_arrays(nw, nr, mach):
    c = L.Cloud.generate_naca0012(nw, nr, 20.0, 0.0, 7, 8, frozen_wall=True)
    g = c.geometry()
    c.close()
    a = np.radians(1.0)
    prim = np.tile([1.0, mach * np.cos(a), mach * np.sin(a), 1.0 / 1.4], (len(g["x"]), 1))
    w = 0.05 * np.exp(-((g["x"] + 0.5) ** 2 + (g["y"] - 0.3) ** 2) / 0.02)
    prim[:, 0] *= 1.0 + w
    prim[:, 3] *= 1.0 + w
    return (g["x"], g["y"], g["kind"], g["nx"], g["ny"], g["off"], g["nbr"]), prim


def _single(arrays, prim, iters, **cfg):
    pc = L.Cloud.from_arrays(*arrays)
    pc.reset_store(0)
    pc.set_primitives(prim)
    res = L.run_fixed_point(pc, L.Config(iters=iters, **cfg))
    return pc, res.residues()


@pytest.mark.parametrize("gpus", [2, 4])
def test_redo_pass_in_multi_domain_runs_is_bitwise_single_domain(gpus):
    """Several domains on the device (MultiRun): each domain's flux pass lists
    and redoes its own supersonic points; the run equals the one-domain run."""
    arrays, prim = _supersonic_naca_arrays(400, 200, 2.0)
    cfg = dict(mach=2.0, aoa=1.0, order=2, inner=3, cfl=0.5)
    one, r1 = _single(arrays, prim, 6, **cfg)
    many, rn = _single(arrays, prim, 6, gpus=gpus, **cfg)
    assert np.array_equal(rn, r1)
    assert many.fields_equal(one)


@pytest.mark.parametrize("world", [2, 4])
def test_redo_pass_in_rank_runs_is_bitwise_single_domain(world):
    """One process per rank, interior and boundary flux passes (each followed
    by its redo pass) on supersonic flow: bitwise the one-domain run."""
    import rank_worker as W

    arrays, prim = _supersonic_naca_arrays(400, 200, 2.0)
    cfg = dict(mach=2.0, aoa=1.0, order=2, inner=3, cfl=0.5)
    one, r1 = _single(arrays, prim, 6, **cfg)
    want_f = one.fields()
    out = W.launch(W.run_rank, world, arrays, prim, cfg, [2, 4], 0)
    assert all(v[0] == "ok" for v in out), out
    assert np.array_equal(out[0][1], r1)
    owned, _ = L.partition(L.Cloud.from_arrays(*arrays), world)
    for r, v in enumerate(out):
        assert np.array_equal(v[2][owned[r]], want_f[owned[r]]), r
