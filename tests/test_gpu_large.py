"""Properties checked at the BASELINE cloud sizes (GPU tests).

The oracle only finishes small clouds in seconds, so at 0.6-10M points the
GPU path is checked through size-independent properties of the algorithm:
the free stream is an exact fixed point (residual and residue exactly 0, the
state bitwise unchanged), runs are deterministic, iterating in pieces equals
one run, multi-domain runs equal the single-domain run bitwise, and a local
perturbation stays local (one iteration moves only the perturbed points' stencil
closure).  Sizes: configs[2] (~625K points) everywhere, configs[3] (10M) for
the fixed point and determinism.
"""
import math

import numpy as np
import pytest

from paper_2403_13287_b200 import lskum as L

pytestmark = pytest.mark.gpu

MACH, AOA = 0.85, 1.0


def naca(nw, nr):
    return L.Cloud.generate_naca0012(nw, nr, 20.0, 0.0, 7, 8, frozen_wall=True)


def free_stream(n):
    a = math.radians(AOA)
    return np.tile([1.0, MACH * math.cos(a), MACH * math.sin(a), 1.0 / 1.4], (n, 1))


def bumped(c, amp=0.02):
    """Free stream + a Gaussian density/pressure bump ahead of the section."""
    g = c.geometry()
    prim = free_stream(c.n)
    r2 = (g["x"] + 0.5) ** 2 + (g["y"] - 0.3) ** 2
    w = amp * np.exp(-r2 / 0.02)
    prim[:, 0] *= 1.0 + w
    prim[:, 3] *= 1.0 + w
    return prim


def run(c, prim, iters, **cfg):
    c.reset_store(0)
    c.set_primitives(prim)
    res = L.run_fixed_point(c, L.Config(mach=MACH, aoa=AOA, iters=iters, order=2, inner=3, cfl=0.5, **cfg))
    return res.residues(), c.fields()


@pytest.mark.parametrize("dims", [(1000, 625), (4000, 2500)])
def test_free_stream_is_an_exact_fixed_point_at_scale(dims):
    c = naca(*dims)
    prim = free_stream(c.n)
    res, f = run(c, prim, 3)
    assert np.all(res == 0.0)
    assert np.array_equal(f[:, 0:4], prim)  # primitives bitwise unchanged
    assert np.all(f[:, 8:20] == 0.0)        # derivatives and residuals exactly zero


@pytest.mark.parametrize("dims", [(1000, 625), (4000, 2500)])
def test_runs_are_deterministic_at_scale(dims):
    c = naca(*dims)
    prim = bumped(c)
    r1, f1 = run(c, prim, 4)
    r2, f2 = run(naca(*dims), prim, 4)
    assert np.all(np.isfinite(r1)) and r1[0] > 0.0
    assert np.array_equal(r1, r2) and np.array_equal(f1, f2)


def test_pieces_and_domains_equal_one_run_at_scale():
    c = naca(1000, 625)
    prim = bumped(c)
    r_one, f_one = run(c, prim, 6)
    # the same 6 iterations in pieces of a device session
    c2 = naca(1000, 625)
    c2.reset_store(0)
    c2.set_primitives(prim)
    with L.Session(c2, L.Config(mach=MACH, aoa=AOA, iters=6, order=2, inner=3, cfl=0.5), capacity=6,
                   from_state=True) as s:
        s.iterate(2)
        s.iterate(4)
        r_pieces = s.residues()
        s.download()
    assert np.array_equal(r_pieces, r_one)
    assert np.array_equal(c2.fields(), f_one)
    # four RCB device domains with peer-memory halos
    r_dom, f_dom = run(naca(1000, 625), prim, 6, gpus=4)
    assert np.array_equal(r_dom, r_one) and np.array_equal(f_dom, f_one)


def test_a_local_perturbation_stays_local():
    """After one iteration only points within the 5-hop stencil closure of the
    bump (3 sweeps + flux + update) can differ from the free stream."""
    c = naca(1000, 625)
    g = c.geometry()
    prim = free_stream(c.n)
    p0 = int(np.argmin((g["x"] + 0.5) ** 2 + (g["y"] - 0.3) ** 2))
    prim[p0, 0] *= 1.01
    _, f = run(c, prim, 1)
    # 5-hop reverse closure (points whose stencils reach p0 within 5 hops)
    off, nbr = g["off"], g["nbr"]
    reach = np.zeros(c.n, dtype=bool)
    reach[p0] = True
    src = np.repeat(np.arange(c.n), np.diff(off))
    for _ in range(5):
        reach = reach | np.bincount(src[reach[nbr]], minlength=c.n).astype(bool)
    moved = np.any(f[:, 0:4] != free_stream(c.n), axis=1)
    assert moved[p0] and moved.sum() > 1
    assert not np.any(moved & ~reach)
