"""Host layer of liblskum_b200.so on CPU (no GPU needed): generators, kNN,
screening, bisection, grid files, config, metrics and C-ABI error conventions,
checked against the reference goldens / reference build and the reference's
own unit-test expectations (tests/test_cloud.cpp, test_bench_config.cpp,
test_capi.cpp, test_runtime.cpp)."""
import ctypes
import hashlib
import os
import re
import subprocess

import numpy as np
import pytest

import pyoracle as P
from paper_2403_13287_b200 import lskum as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def digest(g):
    h = hashlib.sha256()
    for k in ("x", "y", "kind", "nx", "ny", "off", "nbr"):
        h.update(np.ascontiguousarray(g[k]).tobytes())
    return h.hexdigest()


# ------------------------------------------------------------------ C-ABI surface
def declared_functions():
    names = set()
    for path in (os.path.join(ROOT, "include", "lskum", "lskum.h"), os.path.join(ROOT, "include", "lskum_b200.h")):
        text = open(path).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"\b(lskum_\w+)\s*\(", text):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol():
    names = declared_functions()
    assert len(names) >= 35 + 29
    lib = ctypes.CDLL(L.build_library())
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    # the drop-in header declares exactly the reference's 35 entry points
    ref_h = "/root/reference/proj/include/lskum/lskum.h"
    ours = {n for n in names if not n.startswith("lskum_b200")}
    assert len(ours) == 35
    if os.path.exists(ref_h):
        text = re.sub(r"/\*.*?\*/", "", open(ref_h).read(), flags=re.S)
        assert ours == set(re.findall(r"\b(lskum_\w+)\s*\(", text))


def test_library_is_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_status_and_metric_helpers():
    assert [L.status_name(i) for i in range(8)] == L.STATUS_NAMES
    assert L.status_name(42) == "unknown"
    assert L.version() == "1.0.0"
    assert L.rdp(466.0, 10000, 10000000) == pytest.approx(4.66e-9, rel=1e-12)
    assert abs(L.relative_performance(0.679, 0.466) - 1.457) < 0.001
    assert abs(L.relative_performance(0.641, 0.466) - 1.378) < 0.003
    with pytest.raises(L.LskumError) as e:
        L.rdp(1.0, 0, 10)
    assert e.value.status == L.ERR_ARGUMENT
    with pytest.raises(L.LskumError):
        L.relative_performance(1.0, 0.0)
    lib = L.lib()
    assert lib.lskum_rdp(1.0, 10, 10, None) == L.ERR_ARGUMENT
    assert lib.lskum_cloud_read_file(None, None) == L.ERR_ARGUMENT
    assert L.last_error() == "null argument"


# ------------------------------------------------------------------ generators / kNN
def test_generators_match_reference(golden):
    g, meta = golden
    c = L.Cloud.generate_rect(40, 40, 0.1, 7, 8).geometry()
    for k in ("x", "y", "kind", "nx", "ny", "off", "nbr"):
        assert np.array_equal(c[k], g[k]), k
    assert digest(L.Cloud.generate_rect(200, 200, 0.1, 7, 8).geometry()) == meta["rect_200x200_j0.1_s7_k8"]
    assert digest(L.Cloud.generate_rect(61, 47, 0.2, 11, 12).geometry()) == meta["rect_61x47_j0.2_s11_k12"]
    assert digest(L.Cloud.generate_annulus(128, 16, 10.0, 0.1, 5, 9).geometry()) == meta["annulus_128x16_k9"]


def test_knn_bucket_path_equals_brute_force():
    """tests/test_cloud.cpp:110-126: 3600 points, k=9 through the bucket grid."""
    g = L.Cloud.generate_rect(60, 60, 0.25, 3, 9).geometry()
    x, y = g["x"], g["y"]
    for p in range(0, 3600, 97):
        d2 = (x - x[p]) * (x - x[p]) + (y - y[p]) * (y - y[p])
        d2[p] = np.inf
        order = np.lexsort((np.arange(3600), d2))[:9]
        assert np.array_equal(np.sort(order), g["nbr"][g["off"][p]:g["off"][p + 1]])


def test_generator_argument_errors():
    for args in ((3, 10, 0.1, 1, 8), (10, 10, 0.5, 1, 8), (6, 6, 0.0, 0, 2), (6, 6, 0.0, 0, 36)):
        with pytest.raises(L.LskumError) as e:
            L.Cloud.generate_rect(*args)
        assert e.value.status == L.ERR_ARGUMENT
    assert L.Cloud.generate_rect(6, 6, 0.0, 0, 35).nnz == 36 * 35
    with pytest.raises(L.LskumError):
        L.Cloud.generate_annulus(4, 8)
    with pytest.raises(L.LskumError):
        L.Cloud.generate_annulus(16, 8, outer_radius=0.5)


# ------------------------------------------------------------------ screening / bisection
def test_validation_matches_reference(golden):
    _, meta = golden
    v = L.Cloud.generate_rect(40, 40, 0.1, 7, 8).validate()
    for k, want in meta["validate_bump40"].items():
        key = "min_stencil_size" if k == "min_stencil_size" else k
        assert v[key] == want, k
    a = L.Cloud.generate_annulus(64, 8, 10.0, 0.1, 3, 8)
    va = a.validate()
    assert va["n_defective"] == meta["validate_annulus64x8"]["n_defective"]
    assert va["det_tol"] == meta["validate_annulus64x8"]["det_tol"]
    assert a.defective_ids().tolist() == meta["validate_annulus64x8"]["defective"]


def test_lopsided_point_is_defective():
    """tests/test_cloud.cpp:160-178."""
    x = [0.1 * i for i in range(6)]
    y = [0.0 if i == 0 else 0.01 * (1 if i % 2 else -1) for i in range(6)]
    nbr = [j for i in range(6) for j in range(6) if j != i]
    c = L.Cloud.from_arrays(x, y, np.zeros(6, np.uint8), np.zeros(6), np.zeros(6),
                            np.arange(0, 31, 5, dtype=np.int64), nbr)
    assert c.validate()["n_defective"] > 0
    assert 0 in c.defective_ids().tolist()


def test_run_rejects_defective_cloud_before_touching_the_gpu(tmp_path):
    """tests/test_capi.cpp:240-262 (runs on CPU: the screening gate precedes device work)."""
    flat = tmp_path / "flat.grid"
    lines = ["4"] + [f"{i} {0.1 * i} 0 0 0 0 3 " + " ".join(str(j) for j in range(4) if j != i) for i in range(4)]
    flat.write_text("\n".join(lines) + "\n")
    c = L.Cloud.read_file(str(flat))
    v = c.validate()
    assert v["n_defective"] == 4
    assert c.defective_ids().tolist()[:2] == [0, 1]
    with pytest.raises(L.LskumError) as e:
        L.run(c, L.Config(iters=3))
    assert e.value.status == L.ERR_VALIDATION and "defective" in e.value.message
    with pytest.raises(L.LskumError) as e:
        L.Cloud.from_config(L.Config())
    assert e.value.status == L.ERR_CONFIG


def test_annulus_generate_config_is_rejected():
    """CLI smoke test cli_validate_defective: annulus:64x8 fails validation (exit 2)."""
    cfg = L.Config(generate="annulus:64x8", jitter="0.1", seed="3", iters="2")
    c = L.Cloud.from_config(cfg)
    with pytest.raises(L.LskumError) as e:
        L.run(c, cfg)
    assert e.value.status == L.ERR_VALIDATION


def test_partitions_match_reference(golden):
    g, _ = golden
    c = L.Cloud.generate_rect(40, 40, 0.1, 7, 8)
    for parts in (2, 3, 4, 8):
        loc, gh = L.partition(c, parts)
        owner = np.zeros(c.n, np.int32)
        for p, l in enumerate(loc):
            owner[l] = p
            assert abs(len(l) - c.n / parts) <= 1.0
        assert np.array_equal(owner, g[f"part{parts}_owner"])
        assert [len(x) for x in gh] == g[f"part{parts}_ghost_counts"].tolist()
        assert np.array_equal(np.concatenate(gh), g[f"part{parts}_ghosts"])
    with pytest.raises(L.LskumError):
        L.partition(c, 0)
    with pytest.raises(L.LskumError):
        L.partition(c, c.n + 1)


def test_partitions_match_reference_on_large_cloud():
    pc = P.orc_generate_rect(120, 90, 0.2, 4, 8)
    c = L.Cloud.from_arrays(pc.x, pc.y, pc.kind, pc.nx, pc.ny, pc.off, pc.nbr)
    for parts in (5, 8):
        a, b = L.partition(c, parts)
        a2, b2 = P.orc_partition(pc, parts)
        assert all(np.array_equal(u, v) for u, v in zip(a, a2))
        assert all(np.array_equal(u, v) for u, v in zip(b, b2))


# ------------------------------------------------------------------ grid files
def test_grid_file_round_trip_is_exact(tmp_path):
    c = L.Cloud.generate_rect(12, 12, 0.1, 9, 8)
    path = str(tmp_path / "g.grid")
    c.write_file(path)
    back = L.Cloud.read_file(path)
    a, b = c.geometry(), back.geometry()
    for k in a:
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.skipif(not os.path.exists(P.REF_CAPI_SO), reason="reference build absent")
def test_grid_file_bytes_match_reference_writer(tmp_path):
    ref = ctypes.CDLL(P.REF_CAPI_SO)
    h = ctypes.c_void_p()
    assert ref.lskum_cloud_generate_annulus(48, 6, ctypes.c_double(10.0), ctypes.c_double(0.1),
                                            ctypes.c_uint64(3), 8, ctypes.byref(h)) == 0
    rp = str(tmp_path / "ref.grid")
    assert ref.lskum_cloud_write_file(h, rp.encode()) == 0
    ref.lskum_cloud_destroy(h)
    mp = str(tmp_path / "ours.grid")
    L.Cloud.generate_annulus(48, 6, 10.0, 0.1, 3, 8).write_file(mp)
    assert open(rp, "rb").read() == open(mp, "rb").read()


@pytest.mark.parametrize("text,needle", [
    ("", "header"),
    ("abc\n", "header"),
    ("1\n0 0 0 7 0 0 3 1 2 3\n", "kind"),
    ("4\n0 0 0 0 0 0 2 1 2\n", "stencil too small"),
    ("4\n0 0 0 0 0 0 3 1 2 9\n", "neighbor id out of range"),
    ("2\n0 0 0 0 0 0 3 1 1 1\n1 1 0 0 0 0 3 0 0 0\n2 2 0 0 0 0 3 0 0 0\n", "record count mismatch"),
    ("2\n0 0 0 0 0 0 3 1 1 1\n", "record count mismatch"),
    ("1\n5 0 0 0 0 0 3 0 0 0\n", "ascending"),
    ("1\n0 0 0 1 0.5 0.5 3 0 0 0\n", "unit length"),
])
def test_grid_parse_errors_name_the_line(tmp_path, text, needle):
    p = tmp_path / "bad.grid"
    p.write_text(text)
    with pytest.raises(L.LskumError) as e:
        L.Cloud.read_file(str(p))
    assert e.value.status == L.ERR_PARSE
    assert needle in e.value.message and "line" in e.value.message


@pytest.mark.skipif(not os.path.exists(P.REF_CAPI_SO), reason="reference build absent")
@pytest.mark.parametrize("text", [
    "", "abc\n", "1\n0 0 0 7 0 0 3 1 2 3\n", "4\n0 0 0 0 0 0 2 1 2\n", "2\n0 0 0 0 0 0 3 1 1 1\n",
    "1\n0 0 0 1 0.5 0.5 3 0 0 0\n", "3\n0 0 0 0 0 0 3 1 2 2\n\n1 1 0 0 0 0 3 0 2 2\n2 0 1 0 0 0 3 0 1 1 7\n",
])
def test_parse_messages_equal_reference(tmp_path, text):
    ref = ctypes.CDLL(P.REF_CAPI_SO)
    ref.lskum_last_error.restype = ctypes.c_char_p
    p = tmp_path / "t.grid"
    p.write_text(text)
    h = ctypes.c_void_p()
    rc = ref.lskum_cloud_read_file(str(p).encode(), ctypes.byref(h))
    msg = ref.lskum_last_error().decode()
    with pytest.raises(L.LskumError) as e:
        L.Cloud.read_file(str(p))
    assert (e.value.status, e.value.message) == (rc, msg)


def test_missing_grid_is_io_error():
    with pytest.raises(L.LskumError) as e:
        L.Cloud.read_file("/nonexistent/nope.grid")
    assert e.value.status == L.ERR_IO and "nope.grid" in e.value.message


# ------------------------------------------------------------------ config
def test_config_entries_round_trip():
    c = L.Config()
    entries = {"mach": "0.85", "aoa": "-1.25", "gamma": "1.67", "iters": "500", "inner": "2",
               "cfl": "0.4", "order": "1", "layout": "soa", "residual_mode": "split4", "parts": "4",
               "workers": "2", "out_prefix": "runs/a", "generate": "32x16", "jitter": "0.1",
               "seed": "42", "knn": "10", "outer_radius": "7.5", "fp_mode": "strict", "chunk": "8",
               "device": "0", "gpus": "1"}
    for k, v in entries.items():
        c.set(k, v)
    reals = {"mach", "aoa", "gamma", "cfl", "jitter", "outer_radius"}
    for k, v in entries.items():
        got = c.get(k)
        assert (float(got) == float(v) and got == "%.17g" % float(v)) if k in reals else got == v, k
    c.set("bounds", "-1, 1, -0.5, 0.5")
    assert c.get("bounds") == "-1,1,-0.5,0.5"
    c.validate()
    for k, v in (("no_such_key", "1"), ("mach", "fast"), ("iters", "12.5"), ("layout", "csr"),
                 ("residual_mode", "split3"), ("bounds", "0,1,0"), ("fp_mode", "sloppy"), ("mach", "1e999")):
        with pytest.raises(L.LskumError) as e:
            c.set(k, v)
        assert e.value.status == L.ERR_CONFIG
    with pytest.raises(L.LskumError) as e:
        c.get("nope")
    assert e.value.status == L.ERR_CONFIG
    buf = ctypes.create_string_buffer(2)
    assert L.lib().lskum_config_get(c._h, b"mach", buf, 2) == L.ERR_ARGUMENT
    for k, v in (("mach", "-0.1"), ("gamma", "1.0"), ("iters", "-1"), ("inner", "0"), ("cfl", "0"),
                 ("order", "3"), ("parts", "0"), ("workers", "0")):
        bad = L.Config().set(k, v)
        with pytest.raises(L.LskumError) as e:
            bad.validate()
        assert e.value.status == L.ERR_CONFIG, k


def test_config_files(tmp_path):
    p = tmp_path / "solver.cfg"
    p.write_text("# study\n\n  mach = 0.5  \niters=7 # trailing comment\n\tlayout\t=\tsoa\n")
    c = L.Config().load(str(p))
    assert (c.get("mach"), c.get("iters"), c.get("layout")) == ("0.5", "7", "soa")
    p.write_text("mach 0.5\n")
    with pytest.raises(L.LskumError) as e:
        L.Config().load(str(p))
    assert e.value.status == L.ERR_CONFIG and ":1:" in e.value.message
    with pytest.raises(L.LskumError) as e:
        L.Config().load(str(tmp_path / "missing.cfg"))
    assert e.value.status == L.ERR_IO and "missing.cfg" in e.value.message


@pytest.mark.skipif(not os.path.exists(P.REF_CAPI_SO), reason="reference build absent")
def test_config_rendering_equals_reference():
    ref = ctypes.CDLL(P.REF_CAPI_SO)
    h = ctypes.c_void_p()
    ref.lskum_config_create(ctypes.byref(h))
    ours = L.Config()
    for k, v in (("mach", "0.1"), ("aoa", "3.3333333333333335"), ("seed", "18446744073709551615"),
                 ("bounds", "0.1,0.7,-3,1e-3"), ("jitter", "1e-300")):
        r1 = ref.lskum_config_set(h, k.encode(), v.encode())
        try:
            ours.set(k, v)
            r2 = 0
        except L.LskumError as e:
            r2 = e.value.status if hasattr(e, "value") else e.status
        assert r1 == r2, k
    for k in ("mach", "aoa", "gamma", "iters", "inner", "cfl", "order", "layout", "residual_mode", "parts",
              "workers", "out_prefix", "grid", "generate", "jitter", "seed", "knn", "bounds", "outer_radius"):
        buf = ctypes.create_string_buffer(512)
        assert ref.lskum_config_get(h, k.encode(), buf, 512) == 0
        assert ours.get(k) == buf.value.decode(), k
    ref.lskum_config_destroy(h)


# ------------------------------------------------------------------ no silent CPU path
def test_solver_needs_the_gpu_and_says_so():
    if L.device_count() > 0:
        pytest.skip("a CUDA device is present")
    c = L.Cloud.generate_rect(16, 16, 0.05, 9, 8)
    with pytest.raises(L.LskumError) as e:
        L.run(c, L.Config(iters=2))
    assert "CUDA" in e.value.message
