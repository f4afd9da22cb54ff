"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, and
exports every symbol include/aim.h declares (no compute calls without a GPU),
and the binding declares a signature for each."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "aim.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(aim_[a-z_]+)\s*\(", src)))


def test_header_declares_boundary():
    names = header_functions()
    for f in ("aim_plan_create", "aim_matvec", "aim_gmres", "aim_plan_destroy", "aim_plan_info", "aim_last_error"):
        assert f in names


def test_library_builds_and_exports_all_symbols():
    from paper_1712_02443_b200 import build, _lib
    lib_path = build.build()
    assert os.path.exists(lib_path)
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (aim_[a-z_]+)$", out, flags=re.M))
    missing = [f for f in header_functions() if f not in exported]
    assert not missing, missing
    lib = _lib.load()
    declared = {n for n, _, _ in _lib.SIGNATURES}
    assert set(header_functions()) == declared
    for f in header_functions():
        assert hasattr(lib, f)


def test_library_is_sm100a():
    from paper_1712_02443_b200 import build
    lib_path = build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_path], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_last_error_and_arg_checks_without_gpu():
    """Argument validation happens before any device call."""
    import ctypes
    from paper_1712_02443_b200 import _lib
    lib = _lib.load()
    out = ctypes.c_void_p()
    st = lib.aim_plan_create(None, 0, None, 0, None, 0, 1.0, 0.1, 2, 0.3, 0, None, ctypes.byref(out))
    assert st == -1 and b"NULL" in lib.aim_last_error()
    import numpy as np
    v = np.zeros((3, 3)); t = np.zeros((2, 3), np.int32); r = np.zeros((1, 4), np.int32)
    st = lib.aim_plan_create(v.ctypes.data, 3, t.ctypes.data, 2, r.ctypes.data, 1, -1.0, 0.1, 2, 0.3, 0, None,
                             ctypes.byref(out))
    assert st == -1
    st = lib.aim_plan_create(v.ctypes.data, 3, t.ctypes.data, 2, r.ctypes.data, 1, 1.0, 0.1, 9, 0.3, 0, None,
                             ctypes.byref(out))
    assert st == -1
    assert lib.aim_matvec(None, None, None, 1, None) == -1


def test_product_does_not_import_oracle():
    """The product path never reaches the oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_1712_02443_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                s = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", s).replace("oracle/", ""), f
