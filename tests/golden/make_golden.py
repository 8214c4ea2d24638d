"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Runs the unmodified reference core (oracle/_ref/liblskum_refshim.so, compiled
from /root/reference/proj/src by oracle/Makefile) on the reference's own test
fixtures (tests/support.hpp:45-70: 40x40 cloud, jitter 0.1, seed 7, k 8,
M 0.63, alpha 2, CFL 0.5, n_inner 3, +5% Gaussian bump) and stores small
input/output vectors.  Re-run with:  python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import pyoracle as P  # noqa: E402


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    P.build_oracle()
    assert P.have_ref(), "reference shim not built (needs /root/reference)"
    meta = {}
    c = P.ref_generate_rect(40, 40, 0.1, 7, 8)
    prim0 = P.center_bump(c)
    arrays = dict(x=c.x, y=c.y, kind=c.kind, nx=c.nx, ny=c.ny, off=c.off, nbr=c.nbr, prim0=prim0)

    # order 2: 30-iteration prefix + the full run's abort (tests/acceptance.cpp:223-313)
    r30 = P.ref_run(c, iters=30, order=2, prim0=prim0)
    assert r30.code == 0
    arrays["o2_residue30"] = r30.residue
    arrays["o2_store30"] = r30.store
    ra = P.ref_run(c, iters=2000, order=2, prim0=prim0)
    meta["o2_abort"] = {"code": ra.code, "message": ra.msg, "iterations_completed": int(len(ra.residue))}
    for parts in (2, 4, 8):
        rp = P.ref_run(c, iters=2000, order=2, prim0=prim0, parts=parts, workers=1)
        meta[f"o2_abort_parts{parts}"] = {"code": rp.code, "message": rp.msg}
    # order 1: 100 iterations
    r1 = P.ref_run(c, iters=100, order=1, prim0=prim0)
    assert r1.code == 0
    arrays["o1_residue100"] = r1.residue
    arrays["o1_store100"] = r1.store
    # free stream
    rf = P.ref_run(c, iters=10, order=2)
    arrays["fs_residue10"] = rf.residue
    arrays["fs_store10"] = rf.store

    # validation + partitions
    v = P.ref_validate(c)
    meta["validate_bump40"] = {k: (float(v[k]) if isinstance(v[k], float) else int(v[k]))
                               for k in ("n_defective", "n_wall_isolated", "min_stencil_size",
                                         "h_ref", "det_tol")}
    for parts in (2, 3, 4, 8):
        loc, gh = P.ref_partition(c, parts)
        arrays[f"part{parts}_owner"] = np.concatenate(
            [np.full(len(l), p, np.int32) for p, l in enumerate(loc)])[np.argsort(np.concatenate(loc))]
        arrays[f"part{parts}_ghost_counts"] = np.array([len(g) for g in gh], np.int64)
        arrays[f"part{parts}_ghosts"] = np.concatenate(gh).astype(np.int32)
    a = P.ref_generate_annulus(64, 8, 10.0, 0.1, 3, 8)
    va = P.ref_validate(a)
    meta["validate_annulus64x8"] = {"n_defective": int(va["n_defective"]),
                                    "defective": va["defective"].tolist(),
                                    "n_wall_isolated": int(va["n_wall_isolated"]),
                                    "det_tol": float(va["det_tol"])}
    # larger generated clouds: digests of the generator + kNN output
    for (nx, ny, jit, seed, k) in ((200, 200, 0.1, 7, 8), (61, 47, 0.2, 11, 12)):
        g = P.ref_generate_rect(nx, ny, jit, seed, k)
        meta[f"rect_{nx}x{ny}_j{jit}_s{seed}_k{k}"] = digest(g.x, g.y, g.kind, g.nx, g.ny, g.off, g.nbr)
    g = P.ref_generate_annulus(128, 16, 10.0, 0.1, 5, 9)
    meta["annulus_128x16_k9"] = digest(g.x, g.y, g.kind, g.nx, g.ny, g.off, g.nbr)
    # 200^2 order-1 run, 1000 iterations, as quoted in SURVEY 8(c)
    c2 = P.ref_generate_rect(200, 200, 0.1, 7, 8)
    r2 = P.ref_run(c2, iters=1000, order=1, prim0=P.center_bump(c2), parts=8, workers=8)
    meta["rect200_o1_1000"] = {"res1": float(r2.residue[0]), "res1000": float(r2.residue[-1])}
    # deterministic reduce
    rng = np.random.default_rng(17)
    vals = rng.uniform(-1, 1, 1000)
    arrays["reduce_in"] = vals
    meta["reduce_out"] = float(P.ref_reduce(vals))
    # kinetic KATs over random states (tests/support.hpp:27-35 ranges)
    st = np.stack([rng.uniform(0.2, 3.0, 500), rng.uniform(-2, 2, 500), rng.uniform(-2, 2, 500),
                   rng.uniform(0.2, 3.0, 500)], axis=1)
    arrays["kin_states"] = st
    outs = {}
    for op in ("q_from_prim", "cons_from_prim"):
        outs[op] = np.array([P.ref_kinetic(op, s)[1] for s in st])
    for axis in (0, 1):
        for minus in (0, 1):
            outs[f"kfvs_{axis}{minus}"] = np.array([P.ref_kinetic("kfvs", s, axis=axis, minus=minus)[1]
                                                    for s in st])
    for k2, v2 in outs.items():
        arrays["kin_" + k2] = v2
    np.savez_compressed(os.path.join(HERE, "bump40.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print(json.dumps(meta, indent=1)[:2000])


if __name__ == "__main__":
    main()
