"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, and exports every
symbol include/diffpd_b200.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "diffpd_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pd_[a-z_A-Z0-9]+)\s*\(", src)))


def test_library_builds_and_exports_header_symbols():
    import paper_2101_05917_b200 as pdb
    from paper_2101_05917_b200 import _lib
    lib_path = pdb.build()
    lib = ctypes.CDLL(lib_path)
    declared = _declared()
    assert set(declared) == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    # sm_100a code object present
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_create_fails_loudly_without_gpu_or_on_bad_input():
    import numpy as np
    import paper_2101_05917_b200 as pdb
    from pd_inputs import grid_mesh
    rest, hex8 = grid_mesh((2, 1, 1), 0.01)
    with pytest.raises(pdb.PDError) as e:
        pdb.Simulator(rest, hex8, 0.01, youngs=1e5, poisson=0.7, density=1e3, h=0.01)
    assert "poisson" in str(e.value)
    bad = hex8.copy()
    bad[0, 1] = bad[0, 0]
    with pytest.raises(pdb.PDError):
        pdb.Simulator(rest, bad, 0.01, youngs=1e5, poisson=0.45, density=1e3, h=0.01)


def test_native_plan_factorisation():
    # Host setup (ND ordering + supernodal Cholesky of A_s) solves A_s x = A_s v to 1e-10 via the
    # same tile/block schedule the GPU uses (tests/native/plan_check.cpp; no GPU involved).
    exe = "/tmp/diffpd_plan_check"
    subprocess.run(["g++", "-O2", "-std=c++17", "-fopenmp", "-o", exe,
                    os.path.join(ROOT, "tests", "native", "plan_check.cpp"),
                    os.path.join(ROOT, "paper_2101_05917_b200", "csrc", "setup.cpp")], check=True)
    for args in (["4", "2", "2"], ["8", "4", "4"], ["20", "20", "4", "0"], ["24", "12", "12", "0"],
                 ["20", "20", "4", "0", "1"], ["6", "4", "3", "0", "1"], ["8", "4", "4", "1", "1"]):
        r = subprocess.run([exe] + args, capture_output=True, text=True)
        assert r.returncode == 0, r.stdout + r.stderr
        # the K3 v4 warp-range schedule, at the GPU's warp count and at an odd one
        for warps in ("1184", "37"):
            r = subprocess.run([exe] + args, capture_output=True, text=True,
                               env=dict(os.environ, PLAN_V="4", PLAN_WARPS=warps))
            assert r.returncode == 0, r.stdout + r.stderr
