"""CPU tier: the C-ABI library (the product) builds, loads, exports every
entry point include/hz_b200.h declares, and fails loudly -- never falls back
to a CPU path -- when no CUDA device is visible."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hz_b200.h")


def header_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"HZ_API\s+[\w\s\*]+?\b(hz_\w+)\s*\(", txt)))


def test_header_declares_and_library_exports_every_symbol():
    from paper_1607_00968_b200 import _native
    syms = header_symbols()
    assert len(syms) >= 25
    assert sorted(_native.EXPORTS) == syms
    lib = _native.lib()
    for s in syms:
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(hz_\w+)", out))
    assert set(syms) <= exported
    # nothing but the C ABI is exported
    assert {e for e in exported if e.startswith("hz_")} == set(syms)


def test_library_is_sm100a_cuda():
    from paper_1607_00968_b200 import _native
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_options_default_mirror_reference():
    """HelmholtzSolveOptions defaults (inc/helmholtz_solver.hpp:14-24)."""
    from paper_1607_00968_b200 import _native
    o = _native.hz_options()
    _native.lib().hz_options_default(C.byref(o))
    assert (o.method, o.tol, o.max_cycles, o.nlevels, o.shift_factor) == (0, 1e-6, 200, 3, 0.2)
    assert (o.cycle_kind, o.pre, o.post, o.jacobi_weight, o.k_inner) == (1, 2, 2, 0.8, 2)
    assert (o.fgmres_restart, o.dense_threshold, o.precond_precision, o.rhs_block) == (5, 3000, 0, 0)
    assert _native.lib().hz_abi_version() == 2


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="only meaningful without a GPU")
def test_no_cpu_fallback_without_device():
    import paper_1607_00968_b200 as hz
    from paper_1607_00968_b200 import configs
    assert hz.device_count() == 0
    cfg = configs.small_problem(2, (17, 17, 1))
    with pytest.raises(hz.CudaError):
        hz.HelmholtzProblem.from_config(cfg)


def test_python_mirror_validates_before_the_device():
    import paper_1607_00968_b200 as hz
    with pytest.raises(hz.ValidationError):
        hz.HelmholtzSolveOptions(method="Nope").to_c()
    with pytest.raises(hz.ValidationError):
        hz.HelmholtzSolveOptions(precond_precision="c32").to_c()
    with pytest.raises(hz.ValidationError):
        hz.HelmholtzSolveOptions(rhs_block=-1).to_c()
    with pytest.raises(hz.ValidationError):
        hz.HelmholtzProblem(2, (17, 17), (1.0, 1.0), np.ones(10), 1.0,
                            hz.AttenuationField(0.0, np.zeros(10)))


def test_cpp_header_compiles():
    """The header-only C++ drop-in (include/hz_b200.hpp) compiles with g++."""
    src = os.path.join(ROOT, "include", "hz_b200.hpp")
    if not os.path.exists(src):
        pytest.skip("no C++ header")
    r = subprocess.run(["g++", "-std=c++17", "-fsyntax-only", "-x", "c++", src, "-I", os.path.join(ROOT, "include")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_library_has_no_undefined_internal_symbols():
    """Every hz:: template the library uses is instantiated in it (a missing
    explicit instantiation only shows up as a load failure on the GPU box)."""
    import shutil
    import subprocess
    from paper_1607_00968_b200 import _native
    if not shutil.which("nm"):
        pytest.skip("nm not available")
    out = subprocess.run(["nm", "-C", "--undefined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    missing = [ln for ln in out.splitlines() if "hz::" in ln]
    assert not missing, missing
