"""Surface force coefficients (new: the reference has Cp only,
bench.cpp:101-105, so this is checked against closed-form integrals rather
than the reference)."""
import math

import numpy as np
import pytest

from paper_2403_13287_b200 import lskum as L

GAMMA = 1.4


def with_pressure(c, p):
    n = c.n
    prim = np.tile([1.0, 0.0, 0.0, 1.0 / GAMMA], (n, 1))
    prim[:, 3] = p
    c.reset_store(0)
    c.set_primitives(prim)
    return c


def test_uniform_pressure_gives_no_force():
    c = L.Cloud.generate_naca0012(200, 20, 20.0, 0.0, 3, 8)
    with_pressure(c, np.full(c.n, 1.0 / GAMMA + 0.3))
    with L.Config(mach="0.7", aoa="3.0") as cfg:
        f = c.surface_forces(cfg)
    assert abs(f["cl"]) < 1e-13 and abs(f["cd"]) < 1e-13 and abs(f["cm"]) < 1e-13
    assert f["chord"] == pytest.approx(1.0, abs=1e-12)


@pytest.mark.parametrize("aoa", [0.0, 7.0, 90.0])
def test_linear_pressure_on_a_cylinder_is_exact(aoa):
    """p = p_inf + g y on the polygon through the unit circle's wall points:
    F = -int Cp n ds = -(g / (M^2/2)) (0, area) exactly (the panel rule is exact
    for linear pressure), chord 2; rotated into the free-stream frame."""
    nt, mach, gr = 128, 0.5, 0.02
    c = L.Cloud.generate_annulus(nt, 6, 5.0, 0.0, 1, 8)
    y = c.geometry()["y"]
    with_pressure(c, 1.0 / GAMMA + gr * y)
    g = c.geometry()
    wx, wy = g["x"][:nt], g["y"][:nt]
    area = 0.5 * abs(np.sum(wx * np.roll(wy, -1) - np.roll(wx, -1) * wy))
    fy = -gr / (0.5 * mach * mach) * area
    a = math.radians(aoa)
    chord = wx.max() - wx.min()
    with L.Config(mach=str(mach), aoa=str(aoa)) as cfg:
        f = c.surface_forces(cfg)
    assert f["chord"] == pytest.approx(chord, rel=1e-15)
    assert f["cl"] == pytest.approx(fy * math.cos(a) / chord, rel=1e-12, abs=1e-14)
    assert f["cd"] == pytest.approx(fy * math.sin(a) / chord, rel=1e-12, abs=1e-14)


def test_explicit_loop_equals_wall_points_and_orientation_free():
    c = L.Cloud.generate_naca0012(160, 20, 20.0, 0.0, 3, 8)
    rng = np.random.default_rng(4)
    with_pressure(c, 1.0 / GAMMA + 0.05 * rng.standard_normal(c.n))
    with L.Config(mach="0.8", aoa="2.0") as cfg:
        f0 = c.surface_forces(cfg)
        loop = np.arange(160, dtype=np.int32)
        f1 = c.surface_forces(cfg, loop)
        f2 = c.surface_forces(cfg, loop[::-1].copy())  # clockwise: same body, same force
    for k in ("cl", "cd", "cm"):
        assert f0[k] == f1[k]
        assert f2[k] == pytest.approx(f1[k], rel=1e-12, abs=1e-15)


def test_symmetric_section_without_incidence_has_no_lift():
    c = L.Cloud.generate_naca0012(200, 20, 20.0, 0.0, 3, 8)
    y = c.geometry()["y"]
    with_pressure(c, 1.0 / GAMMA + 0.1 * y * y)  # symmetric in y
    with L.Config(mach="0.6", aoa="0.0") as cfg:
        f = c.surface_forces(cfg)
    assert abs(f["cl"]) < 1e-14 and abs(f["cm"]) < 1e-14


def test_rejects_bad_input():
    c = L.Cloud.generate_rect(10, 10, 0.0, 1, 8)  # no wall points
    with L.Config(mach="0.5") as cfg:
        with pytest.raises(L.LskumError):
            c.surface_forces(cfg)
        with pytest.raises(L.LskumError):
            c.surface_forces(cfg, [0, 1, 10**6])
