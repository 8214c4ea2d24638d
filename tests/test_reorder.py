"""Locality permutation of the device numbering (config key `reorder`).

SURVEY section 7 step 6: the device may hold the points in a locality order
(Hilbert curve, or reverse Cuthill-McKee — what reorder=auto uses for a
poorly ordered cloud), ids only — each point keeps its stencil order, residue summands are
indexed by original id, failures carry original ids and the store comes back
in original order.  So every run must be bitwise the unpermuted run, and an
abort must carry the same message (the reference's first-failure order).

CPU: the host side (mode parsing, the auto decision's gather metric, the
orders).  GPU: bitwise invariance of runs, aborts and the screening gate
under reorder=hilbert/rcm, and auto on a shuffled cloud.
"""
import numpy as np
import pytest

from paper_2403_13287_b200 import lskum as L


def shuffled(c: L.Cloud, seed: int = 1) -> L.Cloud:
    """The same cloud with its point ids randomly relabelled (each stencil
    keeps its order) — what a point file from another tool may look like."""
    g = c.geometry()
    n = c.n
    order = np.random.default_rng(seed).permutation(n)
    inv = np.empty(n, dtype=np.int64)
    inv[order] = np.arange(n)
    off = g["off"]
    cnt = np.diff(off)[order]
    noff = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
    src = np.arange(noff[-1]) + np.repeat(off[:-1][order] - noff[:-1], cnt)
    nbr = inv[g["nbr"][src]].astype(np.int32)
    return L.Cloud.from_arrays(g["x"][order], g["y"][order], g["kind"][order], g["nx"][order],
                               g["ny"][order], noff, nbr)


def naca(nw=120, nr=40):
    return L.Cloud.generate_naca0012(nw, nr, 20.0, 0.0, 7, 8, frozen_wall=True)


# ---------------------------------------------------------------- CPU
def test_reorder_config_key():
    for v in ("none", "hilbert", "rcm", "auto"):
        assert L.Config(reorder=v).get("reorder") == v
    assert L.Config().get("reorder") == "auto"
    with pytest.raises(L.LskumError) as e:
        L.Config(reorder="rcm2")
    assert e.value.status == L.ERR_CONFIG


def test_auto_keeps_a_well_ordered_cloud():
    loc = naca().locality("auto")
    assert not loc["permuted"]
    assert 0.0 < loc["lines_before"] < 3.0  # ring order: ~1.9 lines per point
    assert loc["lines_after"] == 0.0  # no locality order even computed


def test_auto_reorders_a_shuffled_cloud():
    loc = shuffled(naca()).locality("auto")
    assert loc["permuted"]
    assert loc["lines_before"] > 6.0 and loc["lines_after"] < 3.0


def test_explicit_modes():
    c = naca()
    assert c.locality("hilbert")["permuted"]
    rcm = c.locality("rcm")
    assert rcm["permuted"] and rcm["lines_after"] < 3.0
    none = c.locality("none")
    assert not none["permuted"] and none["lines_before"] == 0.0


# ---------------------------------------------------------------- GPU
def product_cloud(c) -> L.Cloud:
    return L.Cloud.from_arrays(c.x, c.y, c.kind, c.nx, c.ny, c.off, c.nbr)


def bump_run(c, prim0, iters, order=2, **cfg):
    pc = product_cloud(c)
    pc.reset_store(0)
    pc.set_primitives(prim0)
    conf = L.Config(mach=0.63, aoa=2.0, iters=iters, inner=3, cfl=0.5, order=order, **cfg)
    return pc, L.run_fixed_point(pc, conf)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["hilbert", "rcm"])
@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("fp_mode", ["fast", "strict"])
def test_locality_numbering_is_bitwise_invariant(bump_cloud_arrays, mode, order, fp_mode):
    c, prim0 = bump_cloud_arrays
    base, rb = bump_run(c, prim0, 25, order=order, fp_mode=fp_mode, reorder="none")
    perm, rp = bump_run(c, prim0, 25, order=order, fp_mode=fp_mode, reorder=mode)
    assert np.array_equal(rp.residues(), rb.residues())
    assert perm.fields_equal(base)


@pytest.mark.gpu
@pytest.mark.parametrize("parts", [1, 8])
def test_locality_numbering_aborts_like_reference(bump_cloud_arrays, golden, parts):
    c, prim0 = bump_cloud_arrays
    _, meta = golden
    want = meta["o2_abort"] if parts == 1 else meta[f"o2_abort_parts{parts}"]
    with pytest.raises(L.LskumError) as e:
        bump_run(c, prim0, 2000, parts=parts, reorder="rcm" if parts == 1 else "hilbert")
    assert (e.value.status, e.value.message) == (want["code"], want["message"])


@pytest.mark.gpu
def test_shuffled_cloud_auto_equals_unpermuted():
    c = shuffled(naca())
    runs = []
    for mode in ("none", "auto"):
        cc = L.Cloud.from_arrays(**{k: v for k, v in c.geometry().items()})
        r = L.run(cc, L.Config(mach=0.85, aoa=1.0, iters=40, order=2, reorder=mode))
        runs.append((r.residues(), cc))
    assert np.array_equal(runs[0][0], runs[1][0])
    assert runs[1][1].fields_equal(runs[0][1])


@pytest.mark.gpu
def test_screening_gate_reports_cloud_ids_under_permutation():
    """lskum_run's device screening on a permuted domain names the same first
    defective point as the unpermuted one (ids mapped back to the cloud)."""
    msgs = []
    for mode in ("none", "hilbert"):
        c = L.Cloud.generate_naca0012(160, 60, 20.0, 0.05, 5, 8)
        if c.validate()["n_defective"] == 0:
            pytest.skip("generator produced no defective stencil")
        with pytest.raises(L.LskumError) as e:
            L.run(c, L.Config(iters=3, reorder=mode))
        msgs.append((e.value.status, e.value.message))
    assert msgs[0] == msgs[1] and msgs[0][0] == L.ERR_VALIDATION


@pytest.mark.gpu
def test_session_on_permuted_domain_equals_run(bump_cloud_arrays):
    c, prim0 = bump_cloud_arrays
    whole, rw = bump_run(c, prim0, 30, reorder="hilbert")
    pc = product_cloud(c)
    pc.set_primitives(prim0)
    with L.Session(pc, L.Config(iters=30, reorder="hilbert"), capacity=30, from_state=True) as s:
        for n in (7, 13, 10):
            s.iterate(n)
        assert np.array_equal(s.residues(), rw.residues())
        s.download()
    assert pc.fields_equal(whole)


@pytest.mark.gpu
@pytest.mark.parametrize("gpus", [2, 4])
def test_multi_domain_locality_numbering_is_bitwise(bump_cloud_arrays, gpus):
    """Multi-domain runs order each domain's owned points by the cloud's
    locality order (reorder=rcm/hilbert/auto); results stay bitwise those of
    the single-domain run in cloud order."""
    c, prim0 = bump_cloud_arrays
    base, rb = bump_run(c, prim0, 25, reorder="none")
    for mode in ("rcm", "hilbert"):
        other, ro = bump_run(c, prim0, 25, gpus=gpus, reorder=mode)
        assert np.array_equal(ro.residues(), rb.residues()), mode
        assert other.fields_equal(base), mode


@pytest.mark.gpu
def test_ranks_on_shuffled_cloud_use_locality_numbering():
    """Per-rank domains of a shuffled cloud (reorder=auto -> RCM inside each
    RCB piece) give the single-domain run's bits."""
    import rank_worker as W

    c = shuffled(naca(80, 30))
    g = c.geometry()
    arrays = (g["x"], g["y"], g["kind"], g["nx"], g["ny"], g["off"], g["nbr"])
    assert c.locality("auto")["permuted"]
    pc = L.Cloud.from_arrays(*arrays)
    pc.reset_store(0)
    cfg = dict(mach=0.85, aoa=1.0, iters=8, inner=3, cfl=0.5, order=2)
    rng = np.random.default_rng(3)  # perturbed free stream: a non-trivial transient
    prim0 = np.tile([1.0, 0.85, 0.01, 1.0 / 1.4], (c.n, 1))
    prim0[:, [0, 3]] *= 1.0 + 1e-4 * rng.standard_normal((c.n, 2))
    pc.set_primitives(prim0)
    want = L.run_fixed_point(pc, L.Config(reorder="none", **cfg))
    out = W.launch(W.run_rank, 2, arrays, prim0, dict(cfg, reorder="auto"), [3, 5], 0)
    assert all(v[0] == "ok" for v in out), out
    assert np.array_equal(out[0][1], want.residues()) and want.residues()[-1] > 0.0
    owned, _ = L.partition(L.Cloud.from_arrays(*arrays), 2)
    for r, v in enumerate(out):
        assert np.array_equal(v[2][owned[r]], pc.fields()[owned[r]]), r
