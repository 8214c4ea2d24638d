"""End-to-end parity of the GPU fixed-point loop against the reference (GPU tests).

Goldens in tests/golden/ come from the reference build itself
(tests/golden/make_golden.py).  Tolerances follow SURVEY.md 8(c):
order 1: residue <= 1e-10 relative, state <= 1e-12 (scale-aware) at 100
iterations; order 2: residue <= 1e-10 over 20 iterations and <= 1e-9 at 30,
same abort iteration and code (the reference's determinism contract,
tests/acceptance.cpp:249-313).  Free stream, layouts, split4, partitions and
sessions are checked bitwise.
"""
import math
import os

import numpy as np
import pytest

import pyoracle as P
from conftest import rel_err
from paper_2403_13287_b200 import lskum as L

pytestmark = pytest.mark.gpu


def product_cloud(c) -> L.Cloud:
    return L.Cloud.from_arrays(c.x, c.y, c.kind, c.nx, c.ny, c.off, c.nbr)


def bump_run(c, prim0, iters, order=2, **cfg):
    pc = product_cloud(c)
    pc.reset_store(0)
    pc.set_primitives(prim0)
    conf = L.Config(mach=0.63, aoa=2.0, iters=iters, inner=3, cfl=0.5, order=order, **cfg)
    res = L.run_fixed_point(pc, conf)
    return pc, res


def rel_seq(got, want):
    return float(np.max(np.abs(np.asarray(got) - np.asarray(want)) / np.abs(np.asarray(want))))


@pytest.mark.parametrize("fp_mode", ["strict", "fast"])
def test_order1_bump_100_iterations(bump_cloud_arrays, golden, fp_mode):
    c, prim0 = bump_cloud_arrays
    g, _ = golden
    pc, res = bump_run(c, prim0, 100, order=1, fp_mode=fp_mode)
    assert res.iterations == 100
    assert rel_seq(res.residues(), g["o1_residue100"]) <= 1e-10
    f = pc.fields()
    want = g["o1_store100"]
    assert rel_err(f[:, 0:4], want[:, 0:4]) <= 1e-12
    assert rel_err(f[:, 4:8], want[:, 4:8]) <= 1e-12
    assert np.all(f[:, 8:16] == 0.0)  # order 1 never publishes derivatives
    assert rel_err(f[:, 16:20], want[:, 16:20]) <= 1e-10
    assert rel_err(f[:, 20:21], want[:, 20:21]) <= 1e-12


@pytest.mark.parametrize("fp_mode", ["strict", "fast"])
def test_order2_bump_prefix(bump_cloud_arrays, golden, fp_mode):
    c, prim0 = bump_cloud_arrays
    g, _ = golden
    pc, res = bump_run(c, prim0, 30, fp_mode=fp_mode)
    r = res.residues()
    assert rel_seq(r[:20], g["o2_residue30"][:20]) <= 1e-10
    assert rel_seq(r, g["o2_residue30"]) <= 1e-9
    f = pc.fields()
    assert rel_err(f[:, 0:4], g["o2_store30"][:, 0:4]) <= 1e-9
    # SURVEY 8(c) golden point value
    assert np.allclose(f[820, 0:4], [0.99116092878983286, 0.61300448906736682,
                                     0.033032774308643181, 0.698440501891747], rtol=1e-9, atol=0)


@pytest.mark.parametrize("parts", [1, 8])
def test_order2_bump_aborts_like_reference(bump_cloud_arrays, golden, parts):
    c, prim0 = bump_cloud_arrays
    _, meta = golden
    want = meta["o2_abort"] if parts == 1 else meta[f"o2_abort_parts{parts}"]
    with pytest.raises(L.LskumError) as e:
        bump_run(c, prim0, 2000, parts=parts)
    assert e.value.status == want["code"]
    got, exp = e.value.message, want["message"]
    assert got.split(":")[0] == exp.split(":")[0] == "iteration 35"
    assert got == exp


def test_free_stream_is_a_fixed_point(golden):
    """Reference test_capi.cpp:112-178 and acceptance check 5."""
    with L.Config(generate="16x16", jitter="0.05", seed="9", iters="10") as cfg:
        cloud = L.Cloud.from_config(cfg)
        assert cloud.n == 256
        res = L.run(cloud, cfg)
        assert res.iterations == 10
        assert res.residue(1) == 0.0 and res.final_residue == 0.0 and res.final_log10_rel == 0.0
        with pytest.raises(L.LskumError):
            res.residue(0)
        with pytest.raises(L.LskumError):
            res.residue(11)
        assert res.rdp > 0.0 and res.total_seconds > 0.0
        names = [k[0] for k in res.kernels()]
        assert "flux_residual" in names
        assert all(k[1] >= 0.0 and k[2] >= 0.0 for k in res.kernels())
        prefix = "/tmp/lskum_b200_test/run/out"
        res.write_outputs(cloud, prefix)
        for ext in (".residue.csv", ".solution.dat", ".bench.csv"):
            assert os.path.exists(prefix + ext)
        p = cloud.primitive(0)
        assert p[0] == 1.0 and p[3] == pytest.approx(1.0 / 1.4)
        with pytest.raises(L.LskumError):
            cloud.primitive(256)


def test_free_stream_fields_match_reference(bump_cloud_arrays, golden):
    c, _ = bump_cloud_arrays
    g, _ = golden
    pc = product_cloud(c)
    res = L.run(pc, L.Config(iters=10))
    assert np.all(res.residues() == 0.0)
    f, want = pc.fields(), g["fs_store10"]
    for lo, hi in ((0, 4), (8, 21)):  # everything except q is bitwise
        assert np.array_equal(f[:, lo:hi], want[:, lo:hi])
    assert rel_err(f[:, 4:8], want[:, 4:8]) <= 1e-14


def test_layouts_split4_parts_are_bitwise_invariant(bump_cloud_arrays):
    c, prim0 = bump_cloud_arrays
    base, rb = bump_run(c, prim0, 25)
    for variant in (dict(layout="soa"), dict(residual_mode="split4"), dict(parts=4, workers=4),
                    dict(parts=8, layout="soa", residual_mode="split4"), dict(chunk=3)):
        other, ro = bump_run(c, prim0, 25, **variant)
        assert np.array_equal(ro.residues(), rb.residues()), variant
        assert other.fields_equal(base), variant


def test_order1_differs_from_order2(bump_cloud_arrays):
    c, prim0 = bump_cloud_arrays
    a, _ = bump_run(c, prim0, 25, order=1)
    b, _ = bump_run(c, prim0, 25, order=2)
    assert np.max(np.abs(a.fields()[:, 0] - b.fields()[:, 0])) > 1e-8


def test_session_pieces_equal_one_run(bump_cloud_arrays):
    c, prim0 = bump_cloud_arrays
    whole, rw = bump_run(c, prim0, 30)
    pc = product_cloud(c)
    pc.set_primitives(prim0)
    cfg = L.Config(iters=30)
    with L.Session(pc, cfg, capacity=30, from_state=True) as s:
        for n in (7, 13, 10):
            assert s.iterate(n) > 0.0
        assert np.array_equal(s.residues(), rw.residues())
        s.download()
        names = [k[0] for k in s.kernels()]
        assert names[:2] == ["q_variables", "q_derivatives"] and "flux_residual" in names
        # 3 sweeps, flux (+ the redo pass of its rare-path points for stencils <= 8), update, exact residue
        assert s.info()["launches_per_iter"] == (7 if np.diff(c.off).max() <= 8 else 6)
    assert pc.fields_equal(whole)


def test_defective_cloud_rejected_before_iterating():
    x = [0.1 * i for i in range(5)]
    nbr = [j for i in range(5) for j in range(5) if j != i]
    pc = L.Cloud.from_arrays(x, [0.0] * 5, np.zeros(5, np.uint8), np.zeros(5), np.zeros(5),
                             np.arange(0, 21, 4, dtype=np.int64), nbr)
    with pytest.raises(L.LskumError) as e:
        L.run(pc, L.Config(iters=3))
    assert e.value.status == L.ERR_VALIDATION and "defective" in e.value.message


@pytest.mark.parametrize("cfg", [dict(order=1), dict(order=2)])
def test_200sq_matches_reference_history(cfg, golden):
    """200^2 order-1 1000-iteration history; order 2 on the 30-iteration prefix."""
    _, meta = golden
    c = P.orc_generate_rect(200, 200, 0.1, 7, 8)
    prim0 = P.center_bump(c)
    if cfg["order"] == 1:
        pc, res = bump_run(c, prim0, 1000, order=1)
        r = res.residues()
        assert abs(r[0] / meta["rect200_o1_1000"]["res1"] - 1) <= 1e-10
        assert abs(r[-1] / meta["rect200_o1_1000"]["res1000"] - 1) <= 1e-9
    else:
        want = P.orc_run(c, iters=20, order=2, prim0=prim0)
        pc, res = bump_run(c, prim0, 20, order=2)
        assert rel_seq(res.residues(), want.residue) <= 1e-10
        assert rel_err(pc.fields()[:, :4], want.store[:, :4]) <= 1e-10


@pytest.mark.parametrize("gpus", [2, 3, 4, 8])
def test_multi_domain_halo_engine_is_bitwise_single_domain(bump_cloud_arrays, gpus):
    """gpus=N splits the cloud into N RCB device domains (on distinct GPUs when
    present, else sharing one) with peer-memory halo gathers; per-point
    arithmetic and the residue tree are unchanged, so results are bitwise those
    of the single-domain run (the reference's invariance across partitions,
    tests/test_runtime.cpp:250-289)."""
    c, prim0 = bump_cloud_arrays
    base, rb = bump_run(c, prim0, 25)
    for order in (2, 1):
        if order == 1:
            base, rb = bump_run(c, prim0, 25, order=1)
        other, ro = bump_run(c, prim0, 25, order=order, gpus=gpus)
        assert np.array_equal(ro.residues(), rb.residues()), (gpus, order)
        assert other.fields_equal(base), (gpus, order)


@pytest.mark.parametrize("gpus,parts", [(4, 1), (8, 8), (4, 8), (3, 2)])
def test_multi_domain_abort_matches_reference(bump_cloud_arrays, golden, gpus, parts):
    c, prim0 = bump_cloud_arrays
    _, meta = golden
    want = meta["o2_abort"] if parts == 1 else meta[f"o2_abort_parts{parts}"]
    with pytest.raises(L.LskumError) as e:
        bump_run(c, prim0, 2000, gpus=gpus, parts=parts)
    assert (e.value.status, e.value.message) == (want["code"], want["message"])


def test_multi_domain_session_pieces_equal_single_run(bump_cloud_arrays):
    c, prim0 = bump_cloud_arrays
    whole, rw = bump_run(c, prim0, 20)
    pc = product_cloud(c)
    pc.set_primitives(prim0)
    with L.Session(pc, L.Config(iters=20, gpus=3), capacity=20, from_state=True) as s:
        for n in (5, 15):
            s.iterate(n)
        assert np.array_equal(s.residues(), rw.residues())
        s.download()
    assert pc.fields_equal(whole)


def _grid_cloud():
    """20x20 unjittered rectangle: many pairs with a zero x or y offset, which
    belong to both half stencils of that axis (kernels.cpp:32-35)."""
    return P.orc_generate_rect(20, 20, 0.0, 11, 8)


@pytest.mark.parametrize("fp_mode", ["strict", "fast"])
@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("cloud", ["bump", "grid"])
def test_solver_flux_residual_matches_oracle(bump_cloud_arrays, cloud, order, fp_mode):
    """The solver loop's flux kernel (fast mode: geometry-only split-stencil
    weights, k_flux_w) against the oracle after one iteration: residual slot
    and updated primitives within the reference's 1e-12 oracle tolerance."""
    if cloud == "bump":
        c, prim0 = bump_cloud_arrays
    else:
        c = _grid_cloud()
        prim0 = P.center_bump(c)
    want = P.orc_run(c, iters=1, order=order, prim0=prim0)
    assert want.code == 0, want.msg
    pc, res = bump_run(c, prim0, 1, order=order, fp_mode=fp_mode)
    f = pc.fields()
    live = c.kind != 2
    assert np.abs(want.store[live, 16:20]).max() > 1e-4
    assert rel_err(f[live, 16:20], want.store[live, 16:20]) <= 1e-12
    assert rel_err(f[:, 0:4], want.store[:, 0:4]) <= 1e-12
    assert rel_seq(res.residues(), want.residue) <= 1e-10


def test_cached_domain_reruns_match_fresh_clouds(bump_cloud_arrays):
    """lskum_run keeps the cloud's device domain between calls (geometry,
    weights, buffers, graphs).  A sequence of runs with changing order, fp
    mode, CFL, partition count, chunking and iteration count on ONE cloud must
    give bitwise the results of the same runs on fresh clouds."""
    c, prim0 = bump_cloud_arrays
    cached = product_cloud(c)
    seq = [dict(order=2, iters=12), dict(order=1, iters=30), dict(order=2, iters=12, fp_mode="strict"),
           dict(order=2, iters=7, cfl=0.4, parts=8), dict(order=2, iters=30, chunk=5),
           dict(order=2, iters=60), dict(order=2, iters=12)]  # 60: aborts at 35 like the reference
    for cfg in seq:
        iters = cfg.pop("iters")
        conf = L.Config(mach=0.63, aoa=2.0, iters=iters, inner=3, **dict(dict(cfl=0.5), **cfg))
        out = []
        for cloud in (cached, product_cloud(c)):
            cloud.reset_store(0)
            cloud.set_primitives(prim0)
            try:
                out.append((L.run_fixed_point(cloud, conf).residues(), cloud.fields()))
            except L.LskumError as e:
                out.append((e.message, cloud.fields()))
        (r1, f1), (r2, f2) = out
        assert (r1 == r2) if isinstance(r1, str) else np.array_equal(r1, r2), cfg
        assert np.array_equal(f1, f2), cfg


@pytest.mark.parametrize("which", ["rect", "annulus", "naca_wall", "naca_frozen", "grid"])
def test_device_screening_equals_host(which):
    """validate_cloud on the device (lskum_run's screening) == the host
    screening, itself pinned to the reference: report and defective ids."""
    if which == "rect":
        c = L.Cloud.generate_rect(60, 50, 0.1, 3, 8)
    elif which == "annulus":
        c = L.Cloud.generate_annulus(64, 12, 6.0, 0.1, 5, 8)
    elif which == "naca_wall":
        c = L.Cloud.generate_naca0012(160, 60, 20.0, 0.05, 5, 8)
    elif which == "naca_frozen":
        c = L.Cloud.generate_naca0012(160, 60, 20.0, 0.0, 5, 8, frozen_wall=True)
    else:
        c = L.Cloud.generate_rect(30, 30, 0.0, 1, 8)
    want = c.validate()
    got, ids = c.validate_device(0)
    for key in ("n_points", "n_defective", "n_wall_isolated", "min_stencil_size", "h_ref", "det_tol"):
        assert got[key] == want[key], key
    assert np.array_equal(ids, c.defective_ids())
    if which in ("naca_wall", "annulus"):
        assert want["n_defective"] + want["n_wall_isolated"] > 0  # the check is not vacuous
