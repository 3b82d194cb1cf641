"""The C++ drop-in (include/hz_b200.hpp + include/seistomo_compat): an
UNCHANGED seistomo caller (tests/dropin/sec33_composition.cpp, written
against the reference's public headers only) compiles against the B200
library, and on the GPU its results equal the same source compiled against
the reference (oracle/_ref/sec33_ref, oracle/Makefile): grid / attenuation /
point_source / to_csr / mass bitwise, one V-cycle to 1e-12, block_fgmres and
the W-BiCGSTAB facade solve to the solution tolerance, sensitivity pieces
bitwise / 1e-13."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "dropin", "sec33_composition.cpp")
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "sec33_ref")
PKG = os.path.join(ROOT, "paper_1607_00968_b200")


def build_ours(out):
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include", "seistomo_compat"),
           "-I", os.path.join(ROOT, "include"), SRC, "-L", PKG, "-l:libhz_b200.so", f"-Wl,-rpath,{PKG}", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def read_results(path):
    out = {}
    with open(path, "rb") as f:
        while True:
            tag = f.read(8)
            if not tag:
                break
            cnt = int(np.frombuffer(f.read(8), np.int64)[0])
            out[tag.decode().strip()] = np.frombuffer(f.read(8 * cnt), np.float64).copy()
    return out


def test_unchanged_seistomo_caller_compiles_against_dropin(tmp_path):
    build_ours(str(tmp_path / "sec33_ours"))


def test_reference_build_of_the_same_caller_runs():
    if not os.path.exists(REF_BIN):
        pytest.skip("oracle/_ref/sec33_ref not built (make -C oracle)")
    out = os.path.join("/tmp", f"sec33_ref_{os.getpid()}.bin")
    r = subprocess.run([REF_BIN, out], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    res = read_results(out)
    assert res["R_fgmres"][1] == 1.0 and res["R_bicg"][1] == 1.0


def _cplx(a):
    return a.view(np.complex128)


@pytest.mark.gpu
def test_dropin_caller_matches_reference_build(tmp_path):
    assert os.path.exists(REF_BIN), "oracle/_ref/sec33_ref missing: build() compiles it where /root/reference exists"
    ours = build_ours(str(tmp_path / "sec33_ours"))
    r1 = subprocess.run([REF_BIN, str(tmp_path / "ref.bin")], capture_output=True, text=True, timeout=600)
    assert r1.returncode == 0, r1.stderr
    r2 = subprocess.run([ours, str(tmp_path / "ours.bin")], capture_output=True, text=True, timeout=600)
    assert r2.returncode == 0, r2.stderr
    ref = read_results(str(tmp_path / "ref.bin"))
    got = read_results(str(tmp_path / "ours.bin"))
    assert sorted(ref) == sorted(got)
    # setup pieces: bitwise
    for tag in ("ramp", "mass", "gfactor", "nodes", "B", "csr_rp", "csr_ci", "csr_v", "sens_rhs"):
        assert np.array_equal(ref[tag], got[tag]), tag
    so_r, so_g = ref["sens_out"], got["sens_out"]
    assert np.max(np.abs(so_r - so_g)) <= 1e-13 * np.max(np.abs(so_r))
    # one V(2,2) cycle from zero: <= 1e-12 normwise
    c_r, c_g = _cplx(ref["cycle"]), _cplx(got["cycle"])
    assert np.linalg.norm(c_g - c_r) <= 1e-12 * np.linalg.norm(c_r)
    k = 4
    for X, R, cyc_tol in (("X_fgmres", "R_fgmres", 0.05), ("X_bicg", "R_bicg", 0.15)):
        xr, xg = _cplx(ref[X]).reshape(-1, k), _cplx(got[X]).reshape(-1, k)
        rr, rg = ref[R], got[R]
        assert rr[1] == 1.0 and rg[1] == 1.0, (X, rr[:2], rg[:2])
        assert np.all(rg[2 + k:2 + 2 * k] <= 1e-6)
        assert abs(rg[0] - rr[0]) <= max(2, cyc_tol * rr[0]), (X, rr[0], rg[0])
        for j in range(k):
            err = np.linalg.norm(xg[:, j] - xr[:, j]) / np.linalg.norm(xr[:, j])
            assert err <= 1e-5, (X, j, err)
