"""CPU checks of the C-ABI boundary: libhmg.so loads, exports every function
declared in include/hmg.h, and rejects invalid arguments (naming them)
before any device work."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1605_00492_b200 import build
    build.build()
    from paper_1605_00492_b200 import load_library
    return load_library()


def declared_functions():
    src = open(os.path.join(ROOT, "include", "hmg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hmg_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_survey_entry_points():
    names = declared_functions()
    for n in ("hmg_build_hierarchy", "hmg_apply_helmholtz", "hmg_line_smooth", "hmg_restrict",
              "hmg_prolong_add", "hmg_vcycle", "hmg_pcg_solve", "hmg_free_hierarchy", "hmg_last_error"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    for n in declared_functions():
        assert hasattr(lib, n), f"libhmg.so does not export {n}"


def _build(lib, *args):
    h = ctypes.c_void_p()
    lam = args[5]
    ptr = lam.ctypes.data_as(ctypes.c_void_p) if lam is not None else None
    code = lib.hmg_build_hierarchy(args[0], args[1], args[2], args[3], args[4], ptr, args[6], ctypes.byref(h))
    return code, lib.hmg_last_error().decode()


@pytest.mark.parametrize("args,name", [
    ((11, 0, 8, 0.01, 1e-4), "fine_ref"),
    ((2, 3, 8, 0.01, 1e-4), "coarsest_ref"),
    ((2, -1, 8, 0.01, 1e-4), "coarsest_ref"),
    ((2, 0, 0, 0.01, 1e-4), "nlayers"),
    ((2, 0, 8, 0.0, 1e-4), "thickness"),
    ((2, 0, 8, float("nan"), 1e-4), "thickness"),
    ((2, 0, 8, 0.01, -1.0), "w2"),
])
def test_build_rejects_invalid_arguments(lib, args, name):
    lam = np.ones((8, 320))
    code, msg = _build(lib, *args, lam, 0)
    assert code == 1 and msg.startswith(name), msg


@pytest.mark.parametrize("bad", [0.0, -1.0, float("nan"), float("inf")])
def test_build_rejects_bad_coefficients(lib, bad):
    lam = np.ones((8, 320))
    lam[3, 17] = bad
    code, msg = _build(lib, 2, 0, 8, 0.01, 1e-4, lam, 0)
    assert code == 1 and "lam_host" in msg and str(3 * 320 + 17) in msg


def test_null_arguments(lib):
    code, msg = _build(lib, 2, 0, 8, 0.01, 1e-4, None, 0)
    assert code == 1 and "lam_host" in msg
    assert lib.hmg_apply_helmholtz(None, 0, None, None, None) == 1
    assert "h" in lib.hmg_last_error().decode()
    assert lib.hmg_free_hierarchy(None) == 0


def test_no_cpu_fallback_in_product_package():
    """The product package never imports the oracle or computes on the CPU."""
    pkg = os.path.join(ROOT, "paper_1605_00492_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            src = open(os.path.join(pkg, f)).read()
            assert "import oracle" not in src and "from oracle" not in src
