"""A C program compiled against include/lskum/lskum.h, linked once against
this repo's liblskum_b200.so and once against the reference's own liblskum.so
(oracle/_ref, built from /root/reference/proj/src/capi/lskum_capi.cpp by
oracle/Makefile).  The transcripts and the output files the two write
(.residue.csv, .solution.dat, .bench.csv, .surface.csv; reference
bench.cpp:107-183) must agree: statuses, messages, kernel rows and counts
exactly; numbers within the SURVEY.md 8(c) tolerances.  This is the relink a
reference user does, exercised end to end.
"""
import os
import shutil
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "capi", "consumer.c")
PRODUCT_DIR = os.path.join(ROOT, "paper_2403_13287_b200")
REF_DIR = os.path.join(ROOT, "oracle", "_ref")
have_ref = os.path.exists(os.path.join(REF_DIR, "liblskum.so"))


def build(tmp, libdir, lib, name):
    exe = os.path.join(tmp, name)
    subprocess.run(["gcc", "-std=c11", "-O1", "-Wall", "-Wextra", "-Werror", f"-I{ROOT}/include", SRC,
                    f"-L{libdir}", f"-l{lib}", f"-Wl,-rpath,{libdir}", "-o", exe], check=True)
    return exe


def run(exe, out):
    os.makedirs(out, exist_ok=True)
    p = subprocess.run([exe, out], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr
    return [ln for ln in p.stdout.splitlines() if ln]


def test_consumer_compiles_and_links_against_both_libraries(tmp_path):
    exe = build(str(tmp_path), PRODUCT_DIR, "lskum_b200", "consumer_b200")
    undefined = subprocess.run(["nm", "-D", "--undefined-only", exe], capture_output=True, text=True).stdout
    assert "lskum_run" in undefined and "lskum_result_kernel_name" in undefined
    ldd = subprocess.run(["ldd", exe], capture_output=True, text=True).stdout
    assert "liblskum_b200.so" in ldd
    if have_ref:
        build(str(tmp_path), REF_DIR, "lskum", "consumer_ref")


def close(a, b, rel):
    a, b = np.asarray(a, float), np.asarray(b, float)
    scale = np.maximum(np.abs(b), 1.0)
    return bool(np.all(np.abs(a - b) <= rel * scale))


def compare_transcripts(got, want):
    assert len(got) == len(want), (len(got), len(want))
    for g, w in zip(got, want):
        kind = w[0]
        assert g[0] == kind, (g, w)
        if kind == "E":
            assert g == w
        elif kind == "N":
            gt, wt = g.split(), w.split()
            assert gt[1] == wt[1]
            assert close([float(v) for v in gt[2:]], [float(v) for v in wt[2:]], 1e-10), (g, w)
        else:  # timings
            assert g.split()[1] == w.split()[1] and float(g.split()[2]) > 0.0


def read_csv(path):
    with open(path) as f:
        return [ln.rstrip("\n").split(",") for ln in f]


def compare_outputs(gdir, wdir):
    names = sorted(os.listdir(wdir))
    outs = [n for n in names if n.endswith((".csv", ".dat"))]
    assert sorted(n for n in os.listdir(gdir) if n.endswith((".csv", ".dat"))) == outs
    assert any(n.endswith(".surface.csv") for n in outs)
    for n in outs:
        g, w = os.path.join(gdir, n), os.path.join(wdir, n)
        if n.endswith(".residue.csv"):
            gr, wr = read_csv(g), read_csv(w)
            assert gr[0] == wr[0] == ["iter", "residue", "log10rel", "wall_ms"]
            assert [r[0] for r in gr] == [r[0] for r in wr]
            assert close([float(r[1]) for r in gr[1:]], [float(r[1]) for r in wr[1:]], 1e-10), n
            assert close([float(r[2]) for r in gr[1:]], [float(r[2]) for r in wr[1:]], 1e-9), n
        elif n.endswith(".bench.csv"):
            gr, wr = read_csv(g), read_csv(w)
            assert [r[0] for r in gr] == [r[0] for r in wr], n  # kernel rows + total
        elif n.endswith(".surface.csv"):
            gr, wr = read_csv(g), read_csv(w)
            assert gr[0] == wr[0] == ["arc_position", "cp"]
            assert [r[0] for r in gr] == [r[0] for r in wr]  # arc positions: same text
            assert close([float(r[1]) for r in gr[1:]], [float(r[1]) for r in wr[1:]], 1e-9), n
        else:  # solution.dat: ids and coordinates as text, primitives numerically
            with open(g) as f:
                gl = f.read().splitlines()
            with open(w) as f:
                wl = f.read().splitlines()
            assert gl[0] == wl[0] and len(gl) == len(wl)
            gs = [ln.split() for ln in gl[1:]]
            ws = [ln.split() for ln in wl[1:]]
            assert [r[:3] for r in gs] == [r[:3] for r in ws]
            gv = np.array([[float(v) for v in r[3:]] for r in gs])
            wv = np.array([[float(v) for v in r[3:]] for r in ws])
            assert close(gv, wv, 1e-10), n


@pytest.mark.gpu
@pytest.mark.skipif(not have_ref, reason="reference build (oracle/_ref) absent")
def test_consumer_transcript_and_outputs_match_the_reference(tmp_path):
    tmp = str(tmp_path)
    ours = run(build(tmp, PRODUCT_DIR, "lskum_b200", "consumer_b200"), os.path.join(tmp, "b200"))
    ref = run(build(tmp, REF_DIR, "lskum", "consumer_ref"), os.path.join(tmp, "ref"))
    assert ref[-1] == "E done"
    compare_transcripts(ours, ref)
    compare_outputs(os.path.join(tmp, "b200"), os.path.join(tmp, "ref"))
    shutil.rmtree(tmp, ignore_errors=True)
