"""ctypes bindings for the ORACLE side (test infrastructure only).

Two CPU checkers live behind this module:

* ``orc``  — the plain-C restatement ``oracle/lskum_oracle.c`` (always buildable,
  travels to the GPU box as source and is compiled there by ``make -C oracle``);
* ``ref``  — the unmodified reference core compiled from /root/reference by
  ``oracle/Makefile`` into ``oracle/_ref/liblskum_refshim.so`` (present only when
  the reference was available at build time).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline legs
import this module.  The product (``paper_2403_13287_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
ORC_SO = os.path.join(REF_DIR, "liblskum_oracle_c.so")
REF_SO = os.path.join(REF_DIR, "liblskum_refshim.so")
REF_CAPI_SO = os.path.join(REF_DIR, "liblskum.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")

NSLOT = 21


@dataclass
class Cloud:
    x: np.ndarray
    y: np.ndarray
    kind: np.ndarray
    nx: np.ndarray
    ny: np.ndarray
    off: np.ndarray
    nbr: np.ndarray

    @property
    def n(self) -> int:
        return int(self.x.shape[0])

    def args(self):
        return (self.n, self.x, self.y, self.kind, self.nx, self.ny, self.off, self.nbr)


def build_oracle() -> None:
    """Compile the C restatement (and the reference shim when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_orc = None
_ref = None


def orc_lib():
    global _orc
    if _orc is None:
        if not os.path.exists(ORC_SO) or os.path.getmtime(ORC_SO) < os.path.getmtime(
            os.path.join(HERE, "lskum_oracle.c")
        ):
            subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
        _orc = C.CDLL(ORC_SO)
        _setup_orc(_orc)
    return _orc


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not have_ref():
            raise FileNotFoundError(REF_SO)
        _ref = C.CDLL(REF_SO)
        _setup_ref(_ref)
    return _ref


# --------------------------------------------------------------------------- C oracle
class _OrcCloud(C.Structure):
    _fields_ = [
        ("n", C.c_int32),
        ("x", C.c_void_p), ("y", C.c_void_p), ("nx", C.c_void_p), ("ny", C.c_void_p),
        ("kind", C.c_void_p), ("off", C.c_void_p), ("nbr", C.c_void_p),
    ]


class _OrcStatus(C.Structure):
    _fields_ = [("code", C.c_int), ("iteration", C.c_int), ("point", C.c_int),
                ("nb", C.c_int), ("msg", C.c_char * 320)]


class _OrcConfig(C.Structure):
    _fields_ = [("mach", C.c_double), ("aoa_deg", C.c_double), ("gamma", C.c_double),
                ("cfl", C.c_double), ("iters", C.c_int), ("n_inner", C.c_int),
                ("order", C.c_int)]


class _OrcValidation(C.Structure):
    _fields_ = [("n_defective", C.c_int32), ("n_wall_isolated", C.c_int32),
                ("min_stencil_size", C.c_int32), ("h_ref", C.c_double),
                ("det_tol", C.c_double)]


class _OrcOwned(C.Structure):
    _fields_ = [("n", C.c_int32), ("nnz", C.c_int64),
                ("x", C.POINTER(C.c_double)), ("y", C.POINTER(C.c_double)),
                ("nx", C.POINTER(C.c_double)), ("ny", C.POINTER(C.c_double)),
                ("kind", C.POINTER(C.c_uint8)), ("off", C.POINTER(C.c_int64)),
                ("nbr", C.POINTER(C.c_int32))]


def _setup_orc(L):
    L.orc_run.argtypes = [C.POINTER(_OrcCloud), C.POINTER(_OrcConfig), _dp, _dp,
                          C.POINTER(C.c_int), C.POINTER(_OrcStatus)]
    L.orc_reduce.restype = C.c_double
    L.orc_reduce.argtypes = [_dp, C.c_int64, C.c_int64]
    L.orc_generate_rect.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                    C.c_double, C.c_double, C.c_uint64, C.c_int,
                                    C.POINTER(_OrcOwned)]
    L.orc_generate_annulus.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_uint64,
                                       C.c_int, C.POINTER(_OrcOwned)]
    L.orc_mt_draws.argtypes = [C.c_uint64, C.c_int, np.ctypeslib.ndpointer(dtype=np.uint64)]
    L.orc_validate.argtypes = [C.POINTER(_OrcCloud), C.POINTER(_OrcValidation), _i32p]
    L.orc_partition.argtypes = [C.POINTER(_OrcCloud), C.c_int, _i32p, _i64p, _i32p, C.c_int64]
    for name in ("orc_q_from_prim", "orc_prim_from_q", "orc_cons_from_prim", "orc_prim_from_cons"):
        getattr(L, name).argtypes = [_dp, C.c_double, _dp, C.POINTER(_OrcStatus)]
    L.orc_full_flux.argtypes = [_dp, C.c_int, C.c_double, _dp, C.POINTER(_OrcStatus)]
    L.orc_kfvs_flux.argtypes = [_dp, C.c_int, C.c_int, C.c_double, _dp, C.POINTER(_OrcStatus)]
    L.orc_q_variables.argtypes = [C.POINTER(_OrcCloud), _dp, C.c_double, C.POINTER(_OrcStatus)]
    L.orc_q_derivatives.argtypes = [C.POINTER(_OrcCloud), _dp, C.c_double, _dp,
                                    C.POINTER(_OrcStatus)]
    L.orc_publish.argtypes = [C.POINTER(_OrcCloud), _dp, _dp]
    L.orc_flux_fused.argtypes = [C.POINTER(_OrcCloud), _dp, C.c_double, C.c_double,
                                 C.POINTER(_OrcStatus)]
    L.orc_flux_direction.argtypes = [C.POINTER(_OrcCloud), _dp, C.c_double, C.c_double,
                                     C.c_int, C.c_int, C.c_int, C.POINTER(_OrcStatus)]
    L.orc_timestep.argtypes = [C.POINTER(_OrcCloud), _dp, C.c_double, C.c_double]
    L.orc_state_update.argtypes = [C.POINTER(_OrcCloud), _dp, C.c_double, C.POINTER(_OrcStatus)]


def _orc_cloud(c: Cloud) -> _OrcCloud:
    return _OrcCloud(c.n, c.x.ctypes.data, c.y.ctypes.data, c.nx.ctypes.data,
                     c.ny.ctypes.data, c.kind.ctypes.data, c.off.ctypes.data,
                     c.nbr.ctypes.data)


def _from_owned(o: _OrcOwned) -> Cloud:
    n, nnz = o.n, o.nnz
    cp = lambda p, cnt, dt: np.ctypeslib.as_array(p, shape=(cnt,)).astype(dt, copy=True)
    return Cloud(cp(o.x, n, np.float64), cp(o.y, n, np.float64), cp(o.kind, n, np.uint8),
                 cp(o.nx, n, np.float64), cp(o.ny, n, np.float64), cp(o.off, n + 1, np.int64),
                 cp(o.nbr, nnz, np.int32))


def orc_generate_rect(nx, ny, jitter, seed, k, bounds=(0.0, 1.0, 0.0, 1.0)) -> Cloud:
    L = orc_lib()
    o = _OrcOwned()
    rc = L.orc_generate_rect(nx, ny, *bounds, jitter, seed, k, C.byref(o))
    if rc:
        raise ValueError(f"orc_generate_rect failed: {rc}")
    c = _from_owned(o)
    L.orc_free_cloud(C.byref(o))
    return c


def orc_generate_annulus(nt, nr, r_outer, jitter, seed, k) -> Cloud:
    L = orc_lib()
    o = _OrcOwned()
    rc = L.orc_generate_annulus(nt, nr, r_outer, jitter, seed, k, C.byref(o))
    if rc:
        raise ValueError(f"orc_generate_annulus failed: {rc}")
    c = _from_owned(o)
    L.orc_free_cloud(C.byref(o))
    return c


def orc_mt_draws(seed: int, count: int) -> np.ndarray:
    out = np.zeros(count, dtype=np.uint64)
    orc_lib().orc_mt_draws(seed, count, out)
    return out


def orc_reduce(v: np.ndarray) -> float:
    v = np.ascontiguousarray(v, dtype=np.float64)
    return orc_lib().orc_reduce(v, 0, v.shape[0])


@dataclass
class RunOut:
    code: int
    msg: str
    store: np.ndarray  # n x 21 AoS
    residue: np.ndarray  # completed iterations
    iteration: int = 0
    point: int = -1
    nb: int = -1
    seconds: float = 0.0


def orc_run(c: Cloud, mach=0.63, aoa=2.0, gamma=1.4, iters=10, inner=3, cfl=0.5, order=2,
            prim0=None) -> RunOut:
    L = orc_lib()
    store = np.zeros((c.n, NSLOT))
    if prim0 is None:
        import math
        a = aoa * math.pi / 180.0
        store[:, 0] = 1.0
        store[:, 1] = mach * math.cos(a)
        store[:, 2] = mach * math.sin(a)
        store[:, 3] = 1.0 / gamma
    else:
        store[:, 0:4] = prim0
    cfg = _OrcConfig(mach, aoa, gamma, cfl, iters, inner, order)
    res = np.zeros(max(iters, 1))
    nd = C.c_int(0)
    st = _OrcStatus()
    oc = _orc_cloud(c)
    rc = L.orc_run(C.byref(oc), C.byref(cfg), store.reshape(-1), res, C.byref(nd), C.byref(st))
    return RunOut(rc, st.msg.decode(), store, res[: nd.value].copy(), st.iteration, st.point, st.nb)


def orc_validate(c: Cloud):
    L = orc_lib()
    v = _OrcValidation()
    bad = np.zeros(max(c.n, 1), dtype=np.int32)
    oc = _orc_cloud(c)
    L.orc_validate(C.byref(oc), C.byref(v), bad)
    return dict(n_defective=v.n_defective, n_wall_isolated=v.n_wall_isolated,
                min_stencil_size=v.min_stencil_size, h_ref=v.h_ref, det_tol=v.det_tol,
                defective=bad[: v.n_defective].copy())


def orc_partition(c: Cloud, n_parts: int):
    L = orc_lib()
    owner = np.zeros(c.n, dtype=np.int32)
    goff = np.zeros(n_parts + 1, dtype=np.int64)
    cap = int(c.off[-1]) + 1
    ghosts = np.zeros(cap, dtype=np.int32)
    oc = _orc_cloud(c)
    rc = L.orc_partition(C.byref(oc), n_parts, owner, goff, ghosts, cap)
    if rc:
        raise ValueError(f"orc_partition failed: {rc}")
    locals_ = [np.nonzero(owner == p)[0].astype(np.int32) for p in range(n_parts)]
    gl = [ghosts[goff[p]:goff[p + 1]].copy() for p in range(n_parts)]
    return locals_, gl


def orc_kernel(which: str, c: Cloud, store: np.ndarray, gamma=1.4, cfl=0.5, det_tol=0.0,
               scratch=None, axis=0, minus=0, first=1):
    """Run one reference phase (restated) over all points, in place on `store` (n x 21)."""
    L = orc_lib()
    oc = _orc_cloud(c)
    st = _OrcStatus()
    flat = store.reshape(-1)
    rc = 0
    if which == "q_variables":
        rc = L.orc_q_variables(C.byref(oc), flat, gamma, C.byref(st))
    elif which == "q_derivatives":
        rc = L.orc_q_derivatives(C.byref(oc), flat, det_tol, scratch.reshape(-1), C.byref(st))
    elif which == "publish":
        L.orc_publish(C.byref(oc), flat, scratch.reshape(-1))
    elif which == "flux_fused":
        rc = L.orc_flux_fused(C.byref(oc), flat, gamma, det_tol, C.byref(st))
    elif which == "flux_direction":
        rc = L.orc_flux_direction(C.byref(oc), flat, gamma, det_tol, axis, minus, first,
                                  C.byref(st))
    elif which == "timestep":
        L.orc_timestep(C.byref(oc), flat, gamma, cfl)
    elif which == "state_update":
        rc = L.orc_state_update(C.byref(oc), flat, gamma, C.byref(st))
    else:
        raise KeyError(which)
    return rc, st.msg.decode()


def orc_kinetic(op: str, v, gamma=1.4, axis=0, minus=0):
    L = orc_lib()
    a = np.ascontiguousarray(v, dtype=np.float64)
    out = np.zeros(4)
    st = _OrcStatus()
    if op == "full_flux":
        rc = L.orc_full_flux(a, axis, gamma, out, C.byref(st))
    elif op == "kfvs":
        rc = L.orc_kfvs_flux(a, axis, minus, gamma, out, C.byref(st))
    else:
        rc = getattr(L, "orc_" + op)(a, gamma, out, C.byref(st))
    return rc, out


# --------------------------------------------------------------------------- reference shim
def _setup_ref(L):
    cl = [C.c_int32, _dp, _dp, _u8p, _dp, _dp, _i64p, _i32p]
    L.refshim_kernel.argtypes = [C.c_int] + cl + [_dp, C.c_double, C.c_double, C.c_double,
                                                  _dp, C.c_int, C.c_int, C.c_int, C.c_char_p,
                                                  C.c_int]
    L.refshim_validate.argtypes = cl + [_i32p, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                        C.POINTER(C.c_int32), C.POINTER(C.c_double),
                                        C.POINTER(C.c_double), _dp, _dp]
    L.refshim_partition.argtypes = cl + [C.c_int, _i32p, _i32p, _i32p, C.c_int64]
    L.refshim_reduce.restype = C.c_double
    L.refshim_reduce.argtypes = [_dp, C.c_int64]
    L.refshim_run.argtypes = cl + [C.c_double, C.c_double, C.c_double, C.c_int, C.c_int,
                                   C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.c_void_p, _dp, _dp, C.POINTER(C.c_int),
                                   C.POINTER(C.c_double), C.c_char_p, C.c_int]
    L.refshim_generate_rect.restype = C.c_void_p
    L.refshim_generate_rect.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                        C.c_double, C.c_double, C.c_uint64, C.c_int]
    L.refshim_generate_annulus.restype = C.c_void_p
    L.refshim_generate_annulus.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double,
                                           C.c_uint64, C.c_int]
    L.refshim_knn.restype = C.c_void_p
    L.refshim_knn.argtypes = [C.c_int32, _dp, _dp, C.c_int]
    L.refshim_cloud_sizes.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int64)]
    L.refshim_cloud_get.argtypes = [C.c_void_p, _dp, _dp, _u8p, _dp, _dp, _i64p, _i32p]
    L.refshim_cloud_free.argtypes = [C.c_void_p]
    L.refshim_kinetic.argtypes = [C.c_int, _dp, _dp, C.c_int, C.c_int, C.c_double]


def _ref_take(h) -> Cloud:
    L = ref_lib()
    if not h:
        raise ValueError("reference generator failed")
    n = C.c_int32()
    nnz = C.c_int64()
    L.refshim_cloud_sizes(h, C.byref(n), C.byref(nnz))
    n, nnz = n.value, nnz.value
    c = Cloud(np.zeros(n), np.zeros(n), np.zeros(n, np.uint8), np.zeros(n), np.zeros(n),
              np.zeros(n + 1, np.int64), np.zeros(nnz, np.int32))
    L.refshim_cloud_get(h, c.x, c.y, c.kind, c.nx, c.ny, c.off, c.nbr)
    L.refshim_cloud_free(h)
    return c


def ref_generate_rect(nx, ny, jitter, seed, k, bounds=(0.0, 1.0, 0.0, 1.0)) -> Cloud:
    return _ref_take(ref_lib().refshim_generate_rect(nx, ny, *bounds, jitter, seed, k))


def ref_knn(x, y, k) -> Cloud:
    """The reference's build_stencils on the given points (kinds/normals zero)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    return _ref_take(ref_lib().refshim_knn(len(x), x, y, k))


def ref_generate_annulus(nt, nr, r_outer, jitter, seed, k) -> Cloud:
    return _ref_take(ref_lib().refshim_generate_annulus(nt, nr, r_outer, jitter, seed, k))


_KERNEL_IDS = {"q_variables": 0, "q_derivatives": 1, "publish": 2, "flux_fused": 3,
               "flux_direction": 4, "timestep": 5, "state_update": 6}


def ref_kernel(which: str, c: Cloud, store: np.ndarray, gamma=1.4, cfl=0.5, det_tol=0.0,
               scratch=None, axis=0, minus=0, first=1):
    L = ref_lib()
    if scratch is None:
        scratch = np.zeros(c.n * 8)
    err = C.create_string_buffer(512)
    rc = L.refshim_kernel(_KERNEL_IDS[which], *c.args(), store.reshape(-1), gamma, cfl,
                          det_tol, scratch.reshape(-1), axis, minus, first, err, 512)
    return rc, err.value.decode()


def ref_validate(c: Cloud):
    L = ref_lib()
    bad = np.zeros(max(c.n, 1), dtype=np.int32)
    nd, nw, ms = C.c_int32(), C.c_int32(), C.c_int32()
    h, t = C.c_double(), C.c_double()
    fd = np.zeros(c.n)
    sd = np.zeros(4 * c.n)
    L.refshim_validate(*c.args(), bad, C.byref(nd), C.byref(nw), C.byref(ms), C.byref(h),
                       C.byref(t), fd, sd)
    return dict(n_defective=nd.value, n_wall_isolated=nw.value, min_stencil_size=ms.value,
                h_ref=h.value, det_tol=t.value, defective=bad[: nd.value].copy(),
                full_det=fd, split_det=sd.reshape(c.n, 4))


def ref_partition(c: Cloud, n_parts: int):
    L = ref_lib()
    owner = np.zeros(c.n, dtype=np.int32)
    gc = np.zeros(n_parts, dtype=np.int32)
    cap = int(c.off[-1]) + 1
    ghosts = np.zeros(cap, dtype=np.int32)
    rc = L.refshim_partition(*c.args(), n_parts, owner, gc, ghosts, cap)
    if rc:
        raise ValueError(f"refshim_partition failed: {rc}")
    locals_ = [np.nonzero(owner == p)[0].astype(np.int32) for p in range(n_parts)]
    off = np.concatenate([[0], np.cumsum(gc)])
    gl = [ghosts[off[p]:off[p + 1]].copy() for p in range(n_parts)]
    return locals_, gl


def ref_reduce(v: np.ndarray) -> float:
    v = np.ascontiguousarray(v, dtype=np.float64)
    return ref_lib().refshim_reduce(v, v.shape[0])


def ref_run(c: Cloud, mach=0.63, aoa=2.0, gamma=1.4, iters=10, inner=3, cfl=0.5, order=2,
            layout=0, mode=0, parts=1, workers=1, prim0=None) -> RunOut:
    L = ref_lib()
    store = np.zeros(c.n * NSLOT)
    res = np.zeros(max(iters, 1))
    nd = C.c_int(0)
    secs = C.c_double(0.0)
    err = C.create_string_buffer(512)
    p0 = None
    if prim0 is not None:
        p0 = np.ascontiguousarray(prim0, dtype=np.float64).reshape(-1)
    rc = L.refshim_run(*c.args(), mach, aoa, gamma, iters, inner, cfl, order, layout, mode,
                       parts, workers, None if p0 is None else p0.ctypes.data, store, res,
                       C.byref(nd), C.byref(secs), err, 512)
    return RunOut(rc, err.value.decode(), store.reshape(c.n, NSLOT), res[: nd.value].copy(),
                  seconds=secs.value)


_KIN = {"q_from_prim": 0, "prim_from_q": 1, "cons_from_prim": 2, "prim_from_cons": 3,
        "full_flux": 4, "kfvs": 5}


def ref_kinetic(op: str, v, gamma=1.4, axis=0, minus=0):
    a = np.ascontiguousarray(v, dtype=np.float64)
    out = np.zeros(4)
    rc = ref_lib().refshim_kinetic(_KIN[op], a, out, axis, minus, gamma)
    return rc, out


# --------------------------------------------------------------------------- fixtures
def center_bump(c: Cloud, mach=0.63, aoa=2.0, gamma=1.4, amplitude=0.05, sigma=0.1):
    """Free stream + the reference's +5% Gaussian bump (tests/support.hpp:45-56)."""
    import math
    a = aoa * math.pi / 180.0
    prim = np.empty((c.n, 4))
    prim[:, 0] = 1.0
    prim[:, 1] = mach * math.cos(a)
    prim[:, 2] = mach * math.sin(a)
    prim[:, 3] = 1.0 / gamma
    # per point, in the reference's operation order (no vectorised reassociation)
    for i in range(c.n):
        dx = c.x[i] - 0.5
        dy = c.y[i] - 0.5
        f = 1.0 + amplitude * math.exp(-(dx * dx + dy * dy) / (2.0 * sigma * sigma))
        prim[i, 0] *= f
        prim[i, 3] *= f
    return prim
