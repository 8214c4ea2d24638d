"""Synthetic NACA 0012 O-cloud generator (no reference
counterpart, the reference's generators are cloud.cpp:323-425).

CPU tests: geometry of the section and far field, kNN stencils bit-exact with
the reference's build_stencils (cloud.cpp:137-237, through oracle/_ref when
built), validation identical to the reference's validate_cloud, the frozen
surface variant validating cleanly, and the config spec.  GPU test: a frozen
NACA cloud runs and matches the oracle like the rectangle fixtures.
"""
import math
import os

import numpy as np
import pytest

import pyoracle as P
from conftest import rel_err
from paper_2403_13287_b200 import lskum as L

NW, NR = 160, 80


def y_t(x, t=0.12):
    return 5 * t * (0.2969 * np.sqrt(x) - 0.1260 * x - 0.3516 * x**2 + 0.2843 * x**3 - 0.1036 * x**4)


@pytest.fixture(scope="module")
def naca():
    return L.Cloud.generate_naca0012(NW, NR, 20.0, 0.0, 7, 8, frozen_wall=True)


def test_section_and_far_field(naca):
    g = naca.geometry()
    assert naca.n == NW * NR
    x, y = g["x"], g["y"]
    sx, sy = x[:NW], y[:NW]
    assert (sx[0], sy[0]) == (1.0, 0.0) and (sx[NW // 2], sy[NW // 2]) == (0.0, 0.0)
    np.testing.assert_allclose(np.abs(sy), y_t(sx), rtol=1e-13, atol=1e-15)
    assert np.all(sy[1:NW // 2] > 0) and np.all(sy[NW // 2 + 1:] < 0)  # TE -> upper -> LE -> lower
    seg = np.hypot(np.diff(np.r_[sx, sx[0]]), np.diff(np.r_[sy, sy[0]]))
    assert seg.max() / seg.min() < 1.05  # equal arc length (chords of a fine arc table)
    fx, fy = x[-NW:], y[-NW:]
    np.testing.assert_allclose(np.hypot(fx - 0.5, fy), 20.0, rtol=1e-13)
    k = g["kind"]
    assert np.all(k[:NW] == 2) and np.all(k[-NW:] == 2)
    np.testing.assert_allclose(np.hypot(g["nx"][-NW:], g["ny"][-NW:]), 1.0, rtol=1e-14)


def test_wall_normals_point_into_the_body():
    c = L.Cloud.generate_naca0012(NW, NR, 20.0, 0.05, 3, 8)
    g = c.geometry()
    assert np.all(g["kind"][:NW] == 1)
    nx, ny = g["nx"][:NW], g["ny"][:NW]
    np.testing.assert_allclose(np.hypot(nx, ny), 1.0, rtol=1e-14)
    # a step along the normal from a surface point lands inside the section
    px, py = g["x"][:NW] + 1e-4 * nx, g["y"][:NW] + 1e-4 * ny
    inside = (px > 0) & (px < 1) & (np.abs(py) < y_t(np.clip(px, 0, 1)))
    assert inside.mean() > 0.95  # all but the cusp at the trailing edge


def test_frozen_surface_validates(naca):
    v = naca.validate()
    assert v["n_defective"] == 0 and v["min_stencil_size"] == 8


@pytest.mark.skipif(not P.have_ref(), reason="reference build (oracle/_ref) absent")
def test_stencils_bit_exact_with_reference_knn():
    c = L.Cloud.generate_naca0012(NW, NR, 20.0, 0.1, 5, 8)
    g = c.geometry()
    r = P.ref_knn(g["x"], g["y"], 8)
    assert np.array_equal(r.off, g["off"]) and np.array_equal(r.nbr, g["nbr"])


@pytest.mark.skipif(not P.have_ref(), reason="reference build (oracle/_ref) absent")
@pytest.mark.parametrize("frozen", [False, True])
def test_validation_matches_reference(frozen):
    c = L.Cloud.generate_naca0012(NW, NR, 20.0, 0.05, 5, 8, frozen_wall=frozen)
    g = c.geometry()
    pc = P.Cloud(g["x"], g["y"], g["kind"], g["nx"], g["ny"], g["off"], g["nbr"])
    want = P.ref_validate(pc)
    got = c.validate()
    assert got["n_defective"] == want["n_defective"]
    assert got["h_ref"] == want["h_ref"] and got["det_tol"] == want["det_tol"]
    assert np.array_equal(np.sort(c.defective_ids()), np.sort(want["defective"]))
    if frozen:
        assert want["n_defective"] == 0


def test_config_spec(tmp_path):
    with L.Config(generate=f"naca0012:{NW}x{NR}:frozen", outer_radius="20", seed="7") as cfg:
        c = L.Cloud.from_config(cfg)
    ref = L.Cloud.generate_naca0012(NW, NR, 20.0, 0.0, 7, 8, frozen_wall=True)
    a, b = c.geometry(), ref.geometry()
    for key in ("x", "y", "kind", "nbr"):
        assert np.array_equal(a[key], b[key]), key
    path = str(tmp_path / "naca.grid")
    c.write_file(path)
    back = L.Cloud.read_file(path)
    assert np.array_equal(back.geometry()["x"], a["x"]) and np.array_equal(back.geometry()["nbr"], a["nbr"])


def test_rejects_bad_arguments():
    for args in [(15, 10), (161, 10), (160, 2)]:
        with pytest.raises(L.LskumError):
            L.Cloud.generate_naca0012(*args)
    with pytest.raises(L.LskumError):
        L.Cloud.generate_naca0012(160, 80, 1.5)


@pytest.mark.gpu
@pytest.mark.parametrize("order,iters", [(1, 60), (2, 20)])
@pytest.mark.parametrize("mach,aoa", [(0.63, 2.0), (0.85, 1.0), (1.2, 0.0)])  # BASELINE configs[0..2]
def test_frozen_naca_run_matches_oracle(naca, order, iters, mach, aoa):
    g = naca.geometry()
    c = P.Cloud(g["x"], g["y"], g["kind"], g["nx"], g["ny"], g["off"], g["nbr"])
    prim0 = P.center_bump(c, mach=mach, aoa=aoa)
    want = P.orc_run(c, mach=mach, aoa=aoa, iters=iters, order=order, prim0=prim0)
    assert want.code == 0, want.msg
    pc = L.Cloud.from_arrays(c.x, c.y, c.kind, c.nx, c.ny, c.off, c.nbr)
    pc.reset_store(0)
    pc.set_primitives(prim0)
    res = L.run_fixed_point(pc, L.Config(mach=mach, aoa=aoa, iters=iters, order=order, inner=3, cfl=0.5))
    got = res.residues()
    assert float(np.max(np.abs(got - want.residue) / np.abs(want.residue))) <= 1e-10
    assert rel_err(pc.fields()[:, 0:4], want.store[:, 0:4]) <= 1e-12


def test_frozen_trailing_edge_points_are_valid_boundary_points(tmp_path):
    """Interior points behind the sharp trailing edge whose split stencils fail
    validation are held (kind outer) and carry a unit normal, as the grid
    format requires of boundary points (reference cloud.cpp:470-477)."""
    nw, nr = 520, 308
    c = L.Cloud.generate_naca0012(nw, nr, 20.0, 0.0, 7, 8, frozen_wall=True)
    g = c.geometry()
    held = np.nonzero(g["kind"][nw:-nw] == 2)[0] + nw
    assert len(held) > 0 and np.all(g["x"][held] > 0.99)  # all just behind the trailing edge
    np.testing.assert_allclose(np.hypot(g["nx"][held], g["ny"][held]), 1.0, rtol=1e-14)
    path = str(tmp_path / "naca.grid")
    c.write_file(path)
    assert L.Cloud.read_file(path).validate()["n_defective"] == 0


@pytest.mark.gpu
@pytest.mark.parametrize("gamma", [1.4, 1.3, 5.0 / 3.0])
def test_gas_constant_paths_match_oracle(naca, gamma):
    """The density power 2/(gamma-1): 5 (gamma 1.4, the compile-time
    specialised flux kernel), 6.67 (gamma 1.3, logarithm path) and 3
    (gamma 5/3, integer power) against the oracle."""
    g = naca.geometry()
    c = P.Cloud(g["x"], g["y"], g["kind"], g["nx"], g["ny"], g["off"], g["nbr"])
    prim0 = P.center_bump(c, mach=0.85, aoa=1.0)
    want = P.orc_run(c, mach=0.85, aoa=1.0, gamma=gamma, iters=15, order=2, prim0=prim0)
    assert want.code == 0, want.msg
    pc = L.Cloud.from_arrays(c.x, c.y, c.kind, c.nx, c.ny, c.off, c.nbr)
    pc.reset_store(0)
    pc.set_primitives(prim0)
    res = L.run_fixed_point(pc, L.Config(mach=0.85, aoa=1.0, gamma=gamma, iters=15, order=2, inner=3, cfl=0.5))
    got = res.residues()
    assert float(np.max(np.abs(got - want.residue) / np.abs(want.residue))) <= 1e-10
    assert rel_err(pc.fields()[:, 0:4], want.store[:, 0:4]) <= 1e-12
