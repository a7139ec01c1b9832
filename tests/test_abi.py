"""CPU checks of the boundary: libhelm.so loads without a GPU, exports every entry point
include/helm.h declares, and the ctypes structs match the C layout (compiled with gcc)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_1703_09268_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "helm.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\**\s*([a-z_][a-z0-9_]*)\s*\(", src, flags=re.M)
    return sorted(set(n for n in names if n.startswith(("helm_", "fwi_"))))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for n in ("helm_setup", "helm_apply", "helm_solve", "fwi_misfit_grad"):
        assert n in names


def test_library_loads_and_exports_every_symbol():
    lib = _lib.load()
    for n in declared_functions():
        assert hasattr(lib, n), n
        assert n in _lib.SIGNATURES, f"binding lacks {n}"
    assert b"sm_100a" in lib.helm_version()


def test_bad_arguments_fail_before_any_device_work():
    lib = _lib.load()
    g = _lib.HelmGrid()
    g.ndim = 5
    h = ctypes.c_void_p()
    st = lib.helm_setup(ctypes.byref(g), None, 1.0, None, 1, 1, None, None, ctypes.byref(h))
    assert st == _lib.HELM_ERR_ARG and h.value is None
    assert b"ndim" in lib.helm_last_error()


def test_ctypes_layout_matches_c(tmp_path):
    prog = tmp_path / "sz.c"
    prog.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "helm.h"\nint main(){'
                    'printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu\\n", sizeof(helm_grid), offsetof(helm_grid,h),'
                    'offsetof(helm_grid,pml), sizeof(helm_pml), sizeof(helm_mlopts), sizeof(helm_solve_opts),'
                    'sizeof(helm_solve_report), offsetof(helm_solve_report,bytes_alg), offsetof(helm_grid,stencil));'
                    ' return 0;}')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(prog), "-o", str(exe)])
    got = [int(v) for v in subprocess.check_output([str(exe)]).split()]
    want = [ctypes.sizeof(_lib.HelmGrid), _lib.HelmGrid.h.offset, _lib.HelmGrid.pml.offset,
            ctypes.sizeof(_lib.HelmPml), ctypes.sizeof(_lib.HelmMlOpts), ctypes.sizeof(_lib.HelmSolveOpts),
            ctypes.sizeof(_lib.HelmSolveReport), _lib.HelmSolveReport.bytes_alg.offset, _lib.HelmGrid.stencil.offset]
    assert got == want


def test_no_oracle_import_in_product():
    """The product path never imports the oracle."""
    pkg = os.path.join(ROOT, "paper_1703_09268_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                s = open(os.path.join(dp, f)).read()
                assert "import oracle" not in s and "from oracle" not in s, f
