"""Pin the CPU oracle (oracle/lskum_oracle.c) before trusting it (CPU tests).

1. against the committed golden fixtures produced by the reference itself
   (tests/golden/make_golden.py -> bump40.npz, golden.json): bitwise;
2. against the reference build (oracle/_ref/liblskum_refshim.so) when it is
   present: bitwise, on fresh inputs;
3. against the reference's own known-answer tests (tests/test_kinetic.cpp,
   tests/test_kernels.cpp, tests/test_bench_config.cpp, test_output.txt).
"""
import hashlib
import math

import numpy as np
import pytest

import pyoracle as P


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module")
def orc_bump(bump_cloud_arrays):
    return bump_cloud_arrays


def test_generator_and_knn_match_golden(golden):
    g, meta = golden
    c = P.orc_generate_rect(40, 40, 0.1, 7, 8)
    for k in ("x", "y", "kind", "nx", "ny", "off", "nbr"):
        assert np.array_equal(getattr(c, k), g[k]), k
    for key, (nx, ny, jit, seed, k) in {"rect_61x47_j0.2_s11_k12": (61, 47, 0.2, 11, 12)}.items():
        r = P.orc_generate_rect(nx, ny, jit, seed, k)
        assert digest(r.x, r.y, r.kind, r.nx, r.ny, r.off, r.nbr) == meta[key]
    a = P.orc_generate_annulus(128, 16, 10.0, 0.1, 5, 9)
    assert digest(a.x, a.y, a.kind, a.nx, a.ny, a.off, a.nbr) == meta["annulus_128x16_k9"]


def test_mt19937_64_known_answer():
    # std::mt19937_64 default seed 5489: the 10000th draw is 9981545732273789042
    # (C++ standard [rand.predef]).
    assert int(P.orc_mt_draws(5489, 10000)[-1]) == 9981545732273789042


def test_order2_prefix_and_abort_match_golden(orc_bump, golden):
    c, prim0 = orc_bump
    g, meta = golden
    r = P.orc_run(c, iters=30, order=2, prim0=prim0)
    assert r.code == 0
    assert np.array_equal(r.residue, g["o2_residue30"])
    assert np.array_equal(r.store, g["o2_store30"])
    # SURVEY 8(c) quoted values (measured on the reference)
    assert r.residue[0] == 6.9654492363047232e-06
    assert r.residue[29] == 4.5538658675122872e-04
    a = P.orc_run(c, iters=2000, order=2, prim0=prim0)
    assert (a.code, a.msg) == (meta["o2_abort"]["code"], meta["o2_abort"]["message"])
    assert a.msg == ("iteration 35: flux reconstruction failed on edge (673, 712): "
                     "q-state with q3 >= 0 (q3=0.053609)")  # test_output.txt:25


def test_order1_matches_golden(orc_bump, golden):
    c, prim0 = orc_bump
    g, _ = golden
    r = P.orc_run(c, iters=100, order=1, prim0=prim0)
    assert np.array_equal(r.residue, g["o1_residue100"])
    assert np.array_equal(r.store, g["o1_store100"])
    assert r.residue[0] == 7.5677835945780028e-06 and r.residue[99] == 5.4982373502215492e-07


def test_free_stream_golden(orc_bump, golden):
    c, _ = orc_bump
    g, _ = golden
    r = P.orc_run(c, iters=10, order=2)
    assert np.all(r.residue == 0.0)
    assert np.array_equal(r.store, g["fs_store10"])


def test_validation_and_partitions_match_golden(orc_bump, golden):
    c, _ = orc_bump
    g, meta = golden
    v = P.orc_validate(c)
    for k, want in meta["validate_bump40"].items():
        assert v[k] == want, k
    a = P.orc_generate_annulus(64, 8, 10.0, 0.1, 3, 8)
    va = P.orc_validate(a)
    assert va["n_defective"] == meta["validate_annulus64x8"]["n_defective"]
    assert va["defective"].tolist() == meta["validate_annulus64x8"]["defective"]
    for parts in (2, 3, 4, 8):
        loc, gh = P.orc_partition(c, parts)
        owner = np.zeros(c.n, np.int32)
        for p, l in enumerate(loc):
            owner[l] = p
        assert np.array_equal(owner, g[f"part{parts}_owner"])
        assert [len(x) for x in gh] == g[f"part{parts}_ghost_counts"].tolist()
        assert np.array_equal(np.concatenate(gh), g[f"part{parts}_ghosts"])


def test_reduce_golden(golden):
    g, meta = golden
    assert P.orc_reduce(g["reduce_in"]) == meta["reduce_out"]
    v = g["reduce_in"]

    def pairwise(lo, hi):  # tests/test_runtime.cpp:25-30
        if hi == lo:
            return 0.0
        if hi - lo == 1:
            return v[lo]
        mid = lo + (hi - lo) // 2
        return pairwise(lo, mid) + pairwise(mid, hi)

    assert P.orc_reduce(v) == pairwise(0, len(v))
    assert P.orc_reduce(np.ones(10000)) == 10000.0
    assert P.orc_reduce(np.zeros(0)) == 0.0


def test_kinetic_known_answers(golden):
    g, _ = golden
    st = g["kin_states"]
    for i in range(len(st)):
        assert np.array_equal(P.orc_kinetic("q_from_prim", st[i])[1], g["kin_q_from_prim"][i])
        assert np.array_equal(P.orc_kinetic("cons_from_prim", st[i])[1], g["kin_cons_from_prim"][i])
        for axis in (0, 1):
            for minus in (0, 1):
                got = P.orc_kinetic("kfvs", st[i], axis=axis, minus=minus)[1]
                assert np.array_equal(got, g[f"kin_kfvs_{axis}{minus}"][i])
    # tests/test_kinetic.cpp:18-29, :83-90
    rc, q = P.orc_kinetic("q_from_prim", [1.0, 0.0, 0.0, 1.0])
    assert q[0] == pytest.approx(2.5 * math.log(0.5), rel=1e-14) and q[3] == pytest.approx(-1.0, rel=1e-15)
    rc, f = P.orc_kinetic("kfvs", [1.0, 0.0, 0.0, 1.0], axis=0, minus=0)
    assert f[0] == pytest.approx(0.3989422804, rel=1e-9) and f[1] == pytest.approx(0.5, rel=1e-15)
    assert f[3] == pytest.approx(3.0 / math.sqrt(2.0 * math.pi), rel=1e-12)
    # invalid states (tests/test_kinetic.cpp:62-67)
    assert P.orc_kinetic("q_from_prim", [-1.0, 0, 0, 1.0])[0] == 6
    assert P.orc_kinetic("prim_from_q", [0.0, 0, 0, 0.5])[0] == 6
    assert P.orc_kinetic("prim_from_cons", [1.0, 3.0, 0.0, 1.0])[0] == 6


def test_split_flux_identity():
    """plus + minus == full flux (tests/test_kinetic.cpp:92-107, acceptance check 1)."""
    rng = np.random.default_rng(13)
    worst = 0.0
    for _ in range(2000):
        rho, p = rng.uniform(0.2, 3.0, 2)
        mach, th = rng.uniform(0, 3.0), rng.uniform(0, 2 * math.pi)
        a = math.sqrt(1.4 * p / rho)
        s = [rho, mach * a * math.cos(th), mach * a * math.sin(th), p]
        for axis in (0, 1):
            full = P.orc_kinetic("full_flux", s, axis=axis)[1]
            plus = P.orc_kinetic("kfvs", s, axis=axis, minus=0)[1]
            minus = P.orc_kinetic("kfvs", s, axis=axis, minus=1)[1]
            worst = max(worst, float(np.max(np.abs(plus + minus - full) / np.maximum(np.abs(full), 1.0))))
    assert worst <= 1e-12


@pytest.mark.skipif(not P.have_ref(), reason="reference build absent (oracle/_ref)")
def test_oracle_is_bitwise_the_reference_on_fresh_inputs():
    for (nx, ny, jit, seed) in ((23, 31, 0.15, 99), (16, 16, 0.08, 5)):
        cr = P.ref_generate_rect(nx, ny, jit, seed, 8)
        co = P.orc_generate_rect(nx, ny, jit, seed, 8)
        for k in ("x", "y", "kind", "nx", "ny", "off", "nbr"):
            assert np.array_equal(getattr(cr, k), getattr(co, k))
        prim0 = P.center_bump(cr, mach=0.85, aoa=1.0)
        for order in (1, 2):
            r = P.ref_run(cr, mach=0.85, aoa=1.0, iters=25, order=order, prim0=prim0)
            o = P.orc_run(co, mach=0.85, aoa=1.0, iters=25, order=order, prim0=prim0)
            assert (r.code, r.msg) == (o.code, o.msg)
            assert np.array_equal(r.residue, o.residue) and np.array_equal(r.store, o.store)
    rng = np.random.default_rng(5)
    for n in (0, 1, 7, 4097):
        v = rng.normal(size=n)
        assert P.ref_reduce(v) == P.orc_reduce(v)
