"""Nonlinear-residual certificate of an implicit step over EVERY interior row (oracle, plain C).

    R(U) = max_j | U_j - U^{n-1}_j - dt min_a H^a_j(U) |         (derivation D1)
    ||U - U*||_inf <= R(U) / (1 - dt max c)                       (D6)

`oracle/certify.c` restates oracle.scheme / oracle.howard row by row in C (OpenMP over rows) so that
the certificate covers all 2.7e8 rows of BASELINE cfg4 in seconds per step on the host cores
(SURVEY §8c-7).  It is pinned against the numpy oracle (tests/test_oracle_certify.py) and by D6 on
tiny grids.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py); shares no code with the GPU path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "certify.c")
LIB = os.path.join(HERE, "libcertify.so")


class _Problem(C.Structure):
    _fields_ = [("d", C.c_int32), ("P", C.c_int32), ("K", C.c_int32), ("Q", C.c_int32), ("n", C.c_int64),
                ("lo", C.c_double), ("hi", C.c_double), ("dt", C.c_double),
                ("sigma_dir", C.c_void_p), ("b_dir", C.c_void_p), ("c_ctrl", C.c_void_p),
                ("f_basis", C.c_void_p), ("f_ctrl", C.c_void_p)]


class _Arrays(C.Structure):
    _fields_ = [("U", C.c_void_p), ("u_off", C.c_int64), ("Uprev", C.c_void_p),
                ("sigma_scale", C.c_void_p), ("sigma_node", C.c_void_p), ("b_scale", C.c_void_p),
                ("b_node", C.c_void_p), ("c_node", C.c_void_p), ("f_feat", C.c_void_p),
                ("f_off", C.c_int64), ("f_ld", C.c_int64)]


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.run(["gcc", "-O3", "-fopenmp", "-ffp-contract=off", "-std=gnu99", "-shared", "-fPIC",
                        "-o", LIB, SRC, "-lm"], check=True)
    return LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.orc_residual_rows.restype = C.c_double
        _lib.orc_residual_rows.argtypes = [C.POINTER(_Problem), C.POINTER(_Arrays), C.c_int64, C.c_int64,
                                           C.c_void_p, C.c_void_p]
    return _lib


def _c(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def residual_rows(prob, t, dt, r0, r1, U, u_off, Uprev, fields, f_off, f_ld, policy=None, Rrow=None):
    """Low level: max R_j over interior nodes of slowest-axis rows [r0, r1).
    U[g - u_off] must exist for every endpoint cell of those rows (the rows +- the stencil reach);
    Uprev[g - f_off] and field planes fields[name][k, g - f_off] (plane stride f_ld) on the rows.
    Optional outputs policy (uint8) / Rrow (float64) indexed g - f_off."""
    fb, fc = prob.f_tables(t)
    sd, bd, cc = prob.control_tables()
    keep = [sd, bd, cc, fb, fc]
    pb = _Problem(prob.d, prob.P, prob.K, prob.Q, prob.n, prob.lo, prob.hi, dt,
                  sd.ctypes.data, bd.ctypes.data, cc.ctypes.data, fb.ctypes.data, fc.ctypes.data)
    arrs = {}
    for k in ("sigma_scale", "sigma_node", "b_scale", "b_node", "c_node", "f_feat"):
        v = fields.get(k) if fields is not None else None
        arrs[k] = _c(v)
    for a in (U, Uprev):
        assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    ar = _Arrays(U.ctypes.data, u_off, Uprev.ctypes.data,
                 *[None if arrs[k] is None else arrs[k].ctypes.data
                   for k in ("sigma_scale", "sigma_node", "b_scale", "b_node", "c_node", "f_feat")],
                 f_off, f_ld)
    keep.append(arrs)
    pp = None if policy is None else policy.ctypes.data
    rp = None if Rrow is None else Rrow.ctypes.data
    r = _load().orc_residual_rows(C.byref(pb), C.byref(ar), r0, r1, pp, rp)
    del keep
    return r


def residual(prob, U_full, Uprev_full, t, dt, fields_full=None, with_policy=False):
    """R(U) over every interior row of a problem held as full-grid numpy arrays (fields evaluated on
    the full grid unless given).  Returns max R, or (max R, policy [N], R [N]) with_policy."""
    if fields_full is None:
        fields_full = prob.fields(prob.all_idx())
    U = np.ascontiguousarray(U_full, dtype=np.float64)
    Up = np.ascontiguousarray(Uprev_full, dtype=np.float64)
    pol = np.zeros(prob.N, dtype=np.uint8) if with_policy else None
    Rr = np.zeros(prob.N) if with_policy else None
    r = residual_rows(prob, t, dt, 1, prob.n - 1, U, 0, Up, fields_full, 0, prob.N, pol, Rr)
    return (r, pol, Rr) if with_policy else r
