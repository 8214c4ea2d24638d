"""One process per GPU (torchrun-style ranks) — bench.py's N>1 path.

CPU (gloo, world_size 2): the host logic every rank runs on its own —
the RCB maps that decide who owns which point agree bit for bit across
processes, and a failing setup raises the same agreed error on every rank
instead of leaving one blocked in the exchange.

GPU: the ranks share the box's single B200 (the driver grants one), each
process holding its own CUDA context and mapping its peers' q/dq buffers,
progress counters and rank 0's residue array through CUDA IPC.  Results must
be bitwise those of the single-domain run — the reference's invariance of the
iteration under partitioning (tests/test_runtime.cpp:250-289) — and an abort
must carry the reference's message on every rank.
"""
import numpy as np
import pytest

import rank_worker as W


def arrays_of(c):
    return (c.x, c.y, c.kind, c.nx, c.ny, c.off, c.nbr)


def test_rank_maps_agree_across_processes(bump_cloud_arrays):
    c, _ = bump_cloud_arrays
    out = W.launch(W.host_maps, 2, arrays_of(c), 4)
    for v in out:
        assert v[0] == "ok" and v[1], "ranks derived different RCB maps"
    owned = out[0][2]
    allp = np.sort(np.concatenate(owned))
    assert np.array_equal(allp, np.arange(len(c.x)))  # a partition of the points


def test_rank_setup_failure_is_agreed(bump_cloud_arrays):
    import torch

    if torch.cuda.is_available():
        pytest.skip("checks the no-device path")
    c, _ = bump_cloud_arrays
    out = W.launch(W.create_without_device, 2, arrays_of(c))
    assert all(v[0] == "err" for v in out)
    assert out[0][1:] == out[1][1:]


def test_first_failure_is_min_stage_then_key_owner_message():
    """The error every rank raises is the smallest (stage, key) record, in the
    words of the rank owning the failing point (reference wording)."""
    from paper_2403_13287_b200 import lskum as L

    N = L.NO_ERROR
    owner_msg = "iteration 3: flux reconstruction failed on edge (7, 9): q-state with q3 >= 0 (q3=0.1)"
    recs = [(6, "iteration 3: failure at point 7 owned by another rank", 40, 5, 0),
            (6, owner_msg, 40, 5, 1),
            (5, "iteration 3: later-stage failure", 41, 1, 1),
            (6, "the run failed on another rank", N, N, 0)]
    assert L.first_failure(recs) == (6, owner_msg)
    # a lower stage wins over a lower key
    assert L.first_failure([(5, "a", 38, 9, 1), (6, "b", 39, 0, 1)]) == (5, "a")
    assert L.first_failure([(0, "", N, N, 0), (0, "", N, N, 0)]) is None
    assert L.first_failure([(0, "", N, N, 0), (1, "setup", N, N, 0)]) == (1, "setup")


def _single(c, prim0, iters, **cfg):
    from paper_2403_13287_b200 import lskum as L

    pc = L.Cloud.from_arrays(*arrays_of(c))
    pc.reset_store(0)
    pc.set_primitives(prim0)
    res = L.run_fixed_point(pc, L.Config(**cfg, iters=iters))
    return pc.fields(), res.residues()


BASE = dict(mach=0.63, aoa=2.0, inner=3, cfl=0.5)


@pytest.mark.gpu
@pytest.mark.parametrize("world,order", [(2, 2), (3, 2), (2, 1)])
def test_ranks_bitwise_single_domain(bump_cloud_arrays, world, order):
    c, prim0 = bump_cloud_arrays
    cfg = dict(BASE, order=order)
    want_f, want_r = _single(c, prim0, 20, **cfg)
    out = W.launch(W.run_rank, world, arrays_of(c), prim0, cfg, [7, 13], 0)
    assert all(v[0] == "ok" for v in out), out
    assert np.array_equal(out[0][1], want_r)
    from paper_2403_13287_b200 import lskum as L

    owned, _ = L.partition(L.Cloud.from_arrays(*arrays_of(c)), world)
    for r, v in enumerate(out):
        f = v[2]
        assert np.array_equal(f[owned[r]], want_f[owned[r]]), r
        assert v[3]["launches_per_iter"] > 0
    assert all(len(v[1]) == 0 for v in out[1:])  # residues live on rank 0


@pytest.mark.gpu
@pytest.mark.parametrize("overlap", ["0", "1"])
def test_ranks_overlap_switch_is_bitwise(bump_cloud_arrays, monkeypatch, overlap):
    """Interior/boundary split on (default) and off give the same bits."""
    monkeypatch.setenv("LSKUM_RANK_OVERLAP", overlap)  # inherited by the spawned ranks
    c, prim0 = bump_cloud_arrays
    cfg = dict(BASE, order=2)
    want_f, want_r = _single(c, prim0, 30, **cfg)
    out = W.launch(W.run_rank, 4, arrays_of(c), prim0, cfg, [1, 11, 18], 0)
    assert all(v[0] == "ok" for v in out), out
    assert np.array_equal(out[0][1], want_r)
    from paper_2403_13287_b200 import lskum as L

    owned, _ = L.partition(L.Cloud.from_arrays(*arrays_of(c)), 4)
    for r, v in enumerate(out):
        assert np.array_equal(v[2][owned[r]], want_f[owned[r]]), r


@pytest.mark.gpu
@pytest.mark.parametrize("world,parts", [(2, 1), (4, 8)])
def test_ranks_abort_matches_reference(bump_cloud_arrays, golden, world, parts):
    c, prim0 = bump_cloud_arrays
    _, meta = golden
    want = meta["o2_abort"] if parts == 1 else meta[f"o2_abort_parts{parts}"]
    out = W.launch(W.run_rank, world, arrays_of(c), prim0, dict(BASE, order=2, parts=parts), [2000], 0)
    for v in out:
        assert v[0] == "err", v
        assert (v[1], v[2]) == (want["code"], want["message"])
