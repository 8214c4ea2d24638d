"""How much does point order matter?  The NACA O-cloud as generated (ring by
ring), randomly shuffled, and in Hilbert-curve order; the permutation is
applied to the cloud itself (ids relabelled, each stencil keeps its order).

  python scripts/order_probe.py [n_wall x n_rings ...]
"""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_13287_b200 import lskum as L


def hilbert_key(x, y, bits=16):
    """Hilbert index of points scaled to a 2^bits grid (vectorised d2xy inverse)."""
    n = 1 << bits
    xi = ((x - x.min()) / max(np.ptp(x), 1e-300) * (n - 1)).astype(np.int64)
    yi = ((y - y.min()) / max(np.ptp(y), 1e-300) * (n - 1)).astype(np.int64)
    d = np.zeros_like(xi)
    s = n >> 1
    while s > 0:
        rx = ((xi & s) > 0).astype(np.int64)
        ry = ((yi & s) > 0).astype(np.int64)
        d += s * s * ((3 * rx) ^ ry)
        # rotate
        m = ry == 0
        flip = m & (rx == 1)
        xi = np.where(flip, s - 1 - xi, xi)
        yi = np.where(flip, s - 1 - yi, yi)
        xi2 = np.where(m, yi, xi)
        yi2 = np.where(m, xi, yi)
        xi, yi = xi2, yi2
        s >>= 1
    return d


def permuted(g, order):
    """Cloud whose point k is g's point order[k]."""
    n = len(order)
    inv = np.empty(n, dtype=np.int64)
    inv[order] = np.arange(n)
    off = g["off"]
    cnt = np.diff(off)[order]
    noff = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
    idx = np.concatenate([np.arange(off[p], off[p + 1]) for p in order]) if n < 0 else None
    # vectorised gather of each point's stencil in its original order
    starts = off[:-1][order]
    rep = np.repeat(starts - noff[:-1], cnt)
    src = np.arange(noff[-1]) + rep
    nbr = inv[g["nbr"][src]].astype(np.int32)
    return L.Cloud.from_arrays(g["x"][order], g["y"][order], g["kind"][order], g["nx"][order], g["ny"][order],
                               noff, nbr)


specs = sys.argv[1:] or ["520x308", "4000x2500"]
for spec in specs:
    nw, nr = (int(v) for v in spec.split("x"))
    base = L.Cloud.generate_naca0012(nw, nr, 20.0, 0.0, 7, 8, frozen_wall=True)
    g = base.geometry()
    n = base.n
    rng = np.random.default_rng(1)
    import scipy.sparse as sp
    from scipy.sparse.csgraph import reverse_cuthill_mckee
    A = sp.csr_matrix((np.ones(len(g["nbr"])), g["nbr"], g["off"]), shape=(n, n))
    rcm = np.asarray(reverse_cuthill_mckee((A + A.T).tocsr(), symmetric_mode=True))
    for label, order in [("generated", np.arange(n)), ("shuffled", rng.permutation(n)),
                         ("hilbert", np.argsort(hilbert_key(g["x"], g["y"]), kind="stable")),
                         ("rcm", rcm)]:
        c = base if label == "generated" else permuted(g, order)
        cfg = L.Config(mach=0.85, aoa=1.0, order=2, iters=60, reorder="none")
        s = L.Session(c, cfg, capacity=60)
        s.iterate(10)
        ms = s.iterate(40) / 40
        k = {a: b / max(cn, 1) * 1e3 for a, b, cn in s.kernels()}
        print(json.dumps({"cloud": spec, "order": label, "ms_per_it": round(ms, 4),
                          "sweep_ms": round(k["q_derivatives"], 4), "flux_ms": round(k["flux_residual"], 4),
                          "update_ms": round(k["state_update"], 4)}), flush=True)
        s.close()
