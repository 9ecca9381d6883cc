"""CPU checks of the C-ABI boundary: the in-tree library builds, loads without a GPU, and exports
every entry point include/hjb.h declares (no compute calls here)."""
import ctypes
import os
import re

from paper_1605_04821_b200 import _lib, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "hjb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hjb_[a-z_0-9]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    path = build.build()
    lib = ctypes.CDLL(path)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.hjb_version() == 1


def test_defaults_without_gpu():
    lib = _lib.load()
    p = _lib.SolveParams()
    lib.hjb_solve_params_default(2, ctypes.byref(p))
    assert p.krylov_rtol == 1e-12 and p.use_mg == 1 and p.mg.nu_pre == 2 and p.mg.omega == 1.0
    # creating a grid without a device fails with a status code, never a crash
    d = _lib.GridDesc(dim=2, P=2, K=4, Q=0, n=9, lo=-1, hi=1, rank=0, nranks=1, nccl_id=None,
                      stream=None, device=0)
    h = ctypes.c_void_p()
    code = lib.hjb_grid_create(ctypes.byref(d), ctypes.byref(h))
    assert code in (0, 5)
    if code == 0:
        lib.hjb_grid_destroy(h)
    d.dim = 5
    assert lib.hjb_grid_create(ctypes.byref(d), ctypes.byref(h)) == 1
