"""Rare-path deferral of the staged flux kernel (GPU tests).

k_flux_ws<.., DEFER> evaluates every pair without the rare fallbacks — the
libdevice erf above |s| = 1.5 (a local normal Mach number above ~1.8), the
exponential outside its range, the invalid-state and singular-split failure
checks — and flags the points whose evaluation needed one; k_flux_redo then
recomputes exactly those points with the fallbacks in place (kernels.cuh).
By default a run defers only when its initial state has at most 1% of its
points near the rare paths (Domain::probe_defer), so a supersonic flow runs
with the fallbacks inline; LSKUM_FLUX_DEFER=2 forces the deferral, and a
supersonic flow then sends every point through the redo.  Checked here, with
the forced deferral in child processes: against the oracle (the reference's
algorithm, kinetic.cpp:38-111) within the 1e-12 / 1e-10 tolerances, and
bitwise against the inline fallbacks (this process, where the probe turns the
deferral off) on NACA and rectangle clouds at M = 2 and 2.5, in one-domain,
multi-domain and one-process-per-rank runs.  The failure paths through the
redo are covered by the abort parity tests (test_gpu_runs.py,
test_gpu_parity_configs.py), whose subsonic runs defer.
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

CHILD = r'''
import sys
import numpy as np
sys.path.insert(0, {root!r})
sys.path.insert(0, {tests!r})
sys.path.insert(0, {oracle!r})
import test_gpu_flux_defer as T
res, f = getattr(T, {fn!r})(*{args!r})
np.save({out!r} + "_res.npy", res)
np.save({out!r} + "_f.npy", f)
'''


def forced(fn, args, tmp_path):
    """fn(*args) -> (residues, fields) in a child with the deferral forced on."""
    out = str(tmp_path / fn)
    code = CHILD.format(root=ROOT, tests=os.path.join(ROOT, "tests"), oracle=os.path.join(ROOT, "oracle"),
                        fn=fn, args=tuple(args), out=out)
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, LSKUM_FLUX_DEFER="2"),
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out + "_res.npy"), np.load(out + "_f.npy")


def rect_supersonic(order):
    mach, aoa = 2.5, 3.0
    c = P.orc_generate_rect(24, 24, 0.1, 5, 8)
    prim0 = P.center_bump(c, mach=mach, aoa=aoa)
    pc = L.Cloud.from_arrays(c.x, c.y, c.kind, c.nx, c.ny, c.off, c.nbr)
    pc.reset_store(0)
    pc.set_primitives(prim0)
    res = L.run_fixed_point(pc, L.Config(mach=mach, aoa=aoa, iters=5, inner=3, cfl=0.5, order=order))
    return res.residues(), pc.fields()


@pytest.mark.parametrize("order", [1, 2])
def test_supersonic_flux_through_the_redo_matches_oracle(order, tmp_path):
    mach, aoa = 2.5, 3.0
    c = P.orc_generate_rect(24, 24, 0.1, 5, 8)
    prim0 = P.center_bump(c, mach=mach, aoa=aoa)
    want = P.orc_run(c, mach=mach, aoa=aoa, iters=5, order=order, prim0=prim0)
    assert want.code == 0, want.msg
    r, f = forced("rect_supersonic", (order,), tmp_path)
    assert len(r) == 5
    assert rel_err(f[:, 0:4], want.store[:, 0:4]) <= 1e-12
    live = c.kind != 2
    assert rel_err(f[live, 16:20], want.store[live, 16:20]) <= 1e-10
    w = np.asarray(want.residue)
    assert float(np.max(np.abs(np.asarray(r) - w) / np.abs(w))) <= 1e-10


def supersonic(maker, mach, iters, gpus=1):
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
    res = L.run_fixed_point(c, L.Config(mach=mach, aoa=1.0, iters=iters, order=2, inner=3, cfl=0.5, gpus=gpus))
    return res.residues(), c.fields()


@pytest.mark.parametrize("maker,mach,iters", [("naca1000x625", 2.0, 3), ("naca400x200", 2.0, 5),
                                              ("rect60x40", 2.5, 5)])
def test_deferred_rare_paths_are_bitwise_the_inline_fallbacks(maker, mach, iters, tmp_path):
    res, f = supersonic(maker, mach, iters)  # here: the probe keeps the fallbacks inline
    want_res, want_f = forced("supersonic", (maker, mach, iters), tmp_path)
    assert np.array_equal(res, want_res)
    assert np.array_equal(f, want_f)
    assert np.any(f[:, 16:20] != 0.0) and np.all(np.isfinite(f))


@pytest.mark.parametrize("gpus", [2, 4])
def test_redo_pass_in_multi_domain_runs_is_bitwise_single_domain(gpus, tmp_path):
    """Several domains on the device (MultiRun), each flagging and redoing its
    own supersonic points: bitwise the one-domain run with inline fallbacks."""
    r1, f1 = supersonic("naca400x200", 2.0, 6)
    rn, fn = forced("supersonic", ("naca400x200", 2.0, 6, gpus), tmp_path)
    assert np.array_equal(rn, r1)
    assert np.array_equal(fn, f1)


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


@pytest.mark.parametrize("world", [2, 4])
def test_redo_pass_in_rank_runs_is_bitwise_single_domain(world, monkeypatch):
    """One process per rank (the deferral forced in the ranks), interior and
    boundary flux passes each followed by its redo: bitwise the one-domain run."""
    import rank_worker as W

    arrays, prim = _supersonic_naca_arrays(400, 200, 2.0)
    cfg = dict(mach=2.0, aoa=1.0, order=2, inner=3, cfl=0.5)
    one = L.Cloud.from_arrays(*arrays)
    one.reset_store(0)
    one.set_primitives(prim)
    r1 = L.run_fixed_point(one, L.Config(iters=6, **cfg)).residues()
    want_f = one.fields()
    monkeypatch.setenv("LSKUM_FLUX_DEFER", "2")  # inherited by the spawned ranks
    out = W.launch(W.run_rank, world, arrays, prim, cfg, [2, 4], 0)
    assert all(v[0] == "ok" for v in out), out
    assert np.array_equal(out[0][1], r1)
    owned, _ = L.partition(L.Cloud.from_arrays(*arrays), world)
    for r, v in enumerate(out):
        assert np.array_equal(v[2][owned[r]], want_f[owned[r]]), r


@pytest.mark.parametrize("mach,want", [(0.85, 7), (1.2, 7), (2.0, 6)])
def test_probe_defers_only_flows_that_rarely_need_the_fallbacks(mach, want):
    """The run's initial state decides: a subsonic/transonic/low-supersonic free
    stream defers (7 kernels per iteration: 3 sweeps, flux, redo, update,
    residue), M = 2 keeps the fallbacks inline (no redo pass)."""
    c = L.Cloud.generate_naca0012(400, 200, 20.0, 0.0, 7, 8, frozen_wall=True)
    with L.Session(c, L.Config(mach=mach, aoa=1.0, order=2, iters=2), capacity=2) as s:
        s.iterate(2)
        assert s.info()["launches_per_iter"] == want
