"""Thin Python binding of libhjb (include/hjb.h): argument marshalling only.

Every operation of the hot path runs in the sm_100a kernels behind the C-ABI; torch is used only
to own device memory and to hand over the current CUDA stream.  There is no CPU fallback: if the
library (or a CUDA device) is missing, construction raises.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import check


def _ptr(t):
    """Raw pointer of a torch tensor / numpy array / None (no copies, no conversions)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        if not t.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return t.ctypes.data
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return t.data_ptr()


def _host_f64(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return a


class HJBGrid:
    """Handle on one grid (one rank).  Arrays passed in must follow `layout` (see hjb.h)."""

    def __init__(self, dim: int, P: int, K: int, Q: int, n: int, lo: float, hi: float,
                 device: int = 0, stream=None, rank: int = 0, nranks: int = 1, halo: int = 0,
                 comm: str = "nccl", comm_id: bytes = None):
        """nranks > 1: slab `rank` of a decomposed grid (hjb_partition).  comm = "nccl" (one process
        per GPU; comm_id = the 128-byte id from comm_unique_id() on rank 0, broadcast by the caller)
        or "threads" (TEST-ONLY: ranks are threads of one process; comm_id = any shared 128-byte key).
        Every call is then collective."""
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("HJBGrid needs a CUDA device (B200); there is no CPU fallback")
        self.lib = _lib.load()
        self.device = device
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self._stream = stream
        self._id = None
        if nranks > 1:
            if comm_id is None or len(comm_id) != 128:
                raise ValueError("nranks > 1 needs a 128-byte comm_id")
            self._id = C.create_string_buffer(bytes(comm_id), 128)
        d = _lib.GridDesc(dim=dim, P=P, K=K, Q=Q, n=n, lo=lo, hi=hi, rank=rank, nranks=nranks,
                          nccl_id=C.cast(self._id, C.c_void_p) if self._id is not None else None,
                          stream=stream.cuda_stream, device=device, halo=halo,
                          comm=_lib.HJB_COMM_THREADS if comm == "threads" else _lib.HJB_COMM_NCCL)
        h = C.c_void_p()
        check(self.lib.hjb_grid_create(C.byref(d), C.byref(h)))
        self.h = h
        self.rank, self.nranks = rank, nranks
        self.dim, self.P, self.K, self.Q, self.n = dim, P, K, Q, n
        self._keep = {}

    # ------------------------------------------------------------------ lifetime
    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            check(self.lib.hjb_grid_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ------------------------------------------------------------------ layout
    def layout(self) -> dict:
        lay = _lib.Layout()
        check(self.lib.hjb_grid_query(self.h, C.byref(lay)))
        return {f: getattr(lay, f) for f, _ in lay._fields_}

    # ------------------------------------------------------------------ coefficients
    def set_coeffs(self, sigma_dir, b_dir, c_ctrl, f_basis=None, f_ctrl=None, *, sigma_scale=None,
                   sigma_node=None, b_scale=None, b_node=None, c_node=None, f_feat=None):
        tabs = [_host_f64(sigma_dir), _host_f64(b_dir), _host_f64(c_ctrl),
                None if f_basis is None else _host_f64(f_basis),
                None if f_ctrl is None else _host_f64(f_ctrl)]
        c = _lib.Coeffs(*[_ptr(t) for t in tabs],
                        *[_ptr(t) for t in (sigma_scale, sigma_node, b_scale, b_node, c_node, f_feat)])
        check(self.lib.hjb_set_coeffs(self.h, C.byref(c)))
        # the library retains the device field pointers: keep the tensors alive
        self._keep = dict(sigma_scale=sigma_scale, sigma_node=sigma_node, b_scale=b_scale,
                          b_node=b_node, c_node=c_node, f_feat=f_feat)

    def set_source(self, f_basis, f_ctrl=None):
        fb = _host_f64(f_basis)
        fc = None if f_ctrl is None else _host_f64(f_ctrl)
        check(self.lib.hjb_set_source(self.h, _ptr(fb), _ptr(fc)))

    # ------------------------------------------------------------------ hot path
    def policy_update(self, dt, U, U_prev, policy, F):
        st = _lib.PiStats()
        check(self.lib.hjb_policy_update(self.h, dt, _ptr(U), _ptr(U_prev), _ptr(policy), _ptr(F),
                                         C.byref(st)))
        return {"changed": st.changed, "R_max": st.R_max}

    def apply(self, dt, policy, x, y):
        check(self.lib.hjb_apply(self.h, dt, _ptr(policy), _ptr(x), _ptr(y)))

    @staticmethod
    def mg_params(dim, **kw):
        p = _lib.MgParams()
        _lib.load().hjb_mg_params_default(dim, C.byref(p))
        for k, v in kw.items():
            setattr(p, k, v)
        return p

    @staticmethod
    def solve_params(dim, mg=None, **kw):
        p = _lib.SolveParams()
        _lib.load().hjb_solve_params_default(dim, C.byref(p))
        for k, v in kw.items():
            setattr(p, k, v)
        if mg:
            for k, v in mg.items():
                setattr(p.mg, k, v)
        return p

    def mg_setup(self, dt, policy, **mg):
        p = self.mg_params(self.dim, **mg)
        check(self.lib.hjb_mg_setup(self.h, dt, _ptr(policy), C.byref(p)))
        return self.layout()["n_levels"]

    def mg_apply(self, b, x):
        check(self.lib.hjb_mg_apply(self.h, _ptr(b), _ptr(x)))

    def solve(self, dt, policy, F, x, mg=None, **kw):
        p = self.solve_params(self.dim, mg, **kw)
        st = _lib.SolveStats()
        check(self.lib.hjb_solve(self.h, dt, _ptr(policy), _ptr(F), _ptr(x), C.byref(p), C.byref(st)))
        return {"iters": st.iters, "rres": st.rres, "rres_inf": st.rres_inf}

    def step(self, dt, U_prev, U, policy=None, psi=None, mg=None, raise_on_error=True, **kw):
        p = self.solve_params(self.dim, mg, **kw)
        st = _lib.StepStats()
        code = self.lib.hjb_step(self.h, dt, _ptr(U_prev), _ptr(U), _ptr(policy), _ptr(psi),
                                 C.byref(p), C.byref(st))
        out = st.as_dict()
        out["status"] = _lib.STATUS.get(code, code)
        if raise_on_error:
            check(code)
        return out

    def set_boundary_samples(self, refine=0, samples=None):
        """Exact-psi boundary mode (hjb_set_boundary_samples); samples=None: interpolation mode."""
        check(self.lib.hjb_set_boundary_samples(self.h, int(refine), _ptr(samples)))
        self._keep_bsamp = samples

    def cfl_rate(self, policy=None) -> float:
        """Positivity rate max (sum_p (A_p+B_p)/(2dx) - c) of Proposition CFL (hjb_cfl_rate)."""
        r = C.c_double()
        check(self.lib.hjb_cfl_rate(self.h, _ptr(policy), C.byref(r)))
        return r.value

    # ------------------------------------------------------------------ instrumentation
    def profile_reset(self, time_kernels: bool = False):
        check(self.lib.hjb_profile_reset(self.h, 1 if time_kernels else 0))

    def profile_read(self) -> dict:
        pr = _lib.Profile()
        check(self.lib.hjb_profile_read(self.h, C.byref(pr)))
        return pr.as_dict()
