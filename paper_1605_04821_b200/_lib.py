"""ctypes declarations mirroring include/hjb.h (argument marshalling only)."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhjb.so")

HJB_MAX_PI_LOG = 64

STATUS = {0: "HJB_OK", 1: "HJB_ERR_INVALID_ARG", 2: "HJB_ERR_UNSUPPORTED", 3: "HJB_ERR_STATE",
          4: "HJB_ERR_OOM", 5: "HJB_ERR_CUDA", 6: "HJB_ERR_NCCL", 7: "HJB_ERR_NOT_CONVERGED",
          8: "HJB_ERR_BREAKDOWN", 9: "HJB_ERR_NONFINITE"}

# every symbol include/hjb.h declares (checked by tests/test_abi.py)
EXPORTS = ["hjb_last_error", "hjb_version", "hjb_grid_create", "hjb_grid_query", "hjb_grid_destroy",
           "hjb_set_coeffs", "hjb_set_source", "hjb_policy_update", "hjb_apply",
           "hjb_mg_params_default", "hjb_mg_setup", "hjb_mg_apply", "hjb_solve_params_default",
           "hjb_solve", "hjb_step", "hjb_profile_reset", "hjb_profile_read",
           "hjb_partition", "hjb_halo_plan", "hjb_comm_unique_id", "hjb_cfl_rate",
           "hjb_set_boundary_samples"]

HJB_COMM_NCCL, HJB_COMM_THREADS = 0, 1

KERNEL_CLASSES = ["search", "apply", "resid", "smooth", "transfer", "coarse", "vector", "reduce",
                  "boundary", "mg_coarse", "nested"]
HJB_KC_COUNT = len(KERNEL_CLASSES)


class GridDesc(C.Structure):
    _fields_ = [("dim", C.c_int32), ("P", C.c_int32), ("K", C.c_int32), ("Q", C.c_int32),
                ("n", C.c_int64), ("lo", C.c_double), ("hi", C.c_double),
                ("rank", C.c_int32), ("nranks", C.c_int32), ("nccl_id", C.c_void_p),
                ("stream", C.c_void_p), ("device", C.c_int32), ("halo", C.c_int64), ("comm", C.c_int32)]


class Layout(C.Structure):
    _fields_ = [("n", C.c_int64), ("row_elems", C.c_int64), ("row0", C.c_int64), ("row1", C.c_int64),
                ("halo", C.c_int64), ("local_row0", C.c_int64), ("local_rows", C.c_int64),
                ("local_elems", C.c_int64), ("n_interior", C.c_int64), ("n_boundary", C.c_int64),
                ("n_levels", C.c_int32), ("h", C.c_double), ("k", C.c_double)]


class HaloMsg(C.Structure):
    _fields_ = [("peer", C.c_int32), ("send_row", C.c_int64), ("recv_row", C.c_int64), ("rows", C.c_int64)]


class Coeffs(C.Structure):
    _fields_ = [(f, C.c_void_p) for f in ("sigma_dir", "b_dir", "c_ctrl", "f_basis", "f_ctrl",
                                         "sigma_scale", "sigma_node", "b_scale", "b_node", "c_node",
                                         "f_feat")]


class PiStats(C.Structure):
    _fields_ = [("changed", C.c_int64), ("R_max", C.c_double)]


class MgParams(C.Structure):
    _fields_ = [("nu_pre", C.c_int32), ("nu_post", C.c_int32), ("omega", C.c_double),
                ("coarse_max_n", C.c_int32), ("coarse_k_mode", C.c_int32), ("max_levels", C.c_int32),
                ("gather_n", C.c_int32), ("gamma", C.c_int32), ("gamma_min_nodes", C.c_int32),
                ("coarse_op", C.c_int32), ("precision", C.c_int32)]


class SolveParams(C.Structure):
    _fields_ = [("krylov_rtol", C.c_double), ("krylov_maxit", C.c_int32), ("use_mg", C.c_int32),
                ("tol_pi", C.c_double), ("max_pi", C.c_int32), ("mg", MgParams),
                ("pi_forcing", C.c_double), ("guess", C.c_int32), ("krylov_rtol_inf", C.c_double),
                ("theta", C.c_double), ("solver", C.c_int32), ("nested_coarsen", C.c_int32),
                ("nested_min_n", C.c_int32), ("nested_increment", C.c_int32)]

HJB_GUESS_PREV, HJB_GUESS_GIVEN, HJB_GUESS_EXTRAPOLATE, HJB_GUESS_NESTED = 0, 1, 2, 3


class SolveStats(C.Structure):
    _fields_ = [("iters", C.c_int32), ("rres", C.c_double), ("rres_inf", C.c_double)]


class StepStats(C.Structure):
    _fields_ = [("pi_iters", C.c_int32), ("krylov_iters_total", C.c_int32),
                ("krylov_iters", C.c_int32 * HJB_MAX_PI_LOG), ("changed", C.c_int64 * HJB_MAX_PI_LOG),
                ("R", C.c_double * HJB_MAX_PI_LOG), ("final_R", C.c_double), ("final_rres", C.c_double),
                ("ms_search", C.c_double), ("ms_setup", C.c_double), ("ms_solve", C.c_double),
                ("n_levels", C.c_int32), ("final_rres_inf", C.c_double),
                ("nested_pi_iters", C.c_int32), ("ms_nested", C.c_double)]

    def as_dict(self):
        k = self.pi_iters
        m = min(k + 1, HJB_MAX_PI_LOG)
        return dict(pi_iters=k, krylov_iters_total=self.krylov_iters_total,
                    krylov_iters=list(self.krylov_iters[:k]), changed=list(self.changed[:m]),
                    R=list(self.R[:m]), final_R=self.final_R, final_rres=self.final_rres,
                    ms_search=self.ms_search, ms_setup=self.ms_setup, ms_solve=self.ms_solve,
                    n_levels=self.n_levels, final_rres_inf=self.final_rres_inf,
                    nested_pi_iters=self.nested_pi_iters, ms_nested=self.ms_nested)


class Profile(C.Structure):
    _fields_ = [("launches", C.c_int64 * HJB_KC_COUNT), ("calls", C.c_int64 * HJB_KC_COUNT),
                ("ms", C.c_double * HJB_KC_COUNT),
                ("bytes", C.c_double * HJB_KC_COUNT), ("flops", C.c_double * HJB_KC_COUNT),
                ("nodes", C.c_double * HJB_KC_COUNT), ("total_launches", C.c_int64),
                ("timed", C.c_int32), ("graph_launches", C.c_int64), ("graph_kernels", C.c_int64)]

    def as_dict(self):
        per = {k: dict(launches=self.launches[i], calls=self.calls[i], ms=self.ms[i], bytes=self.bytes[i],
                       flops=self.flops[i], nodes=self.nodes[i])
               for i, k in enumerate(KERNEL_CLASSES)}
        return dict(classes=per, total_launches=self.total_launches, timed=bool(self.timed),
                    graph_launches=self.graph_launches, graph_kernels=self.graph_kernels)


_lib = None


def load(path: str = None):
    """Load libhjb.so.  Raises (loudly) if it is missing: there is no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    # HJB_LIB selects an alternative in-tree build (kernel A/B experiments, tools/)
    path = path or os.environ.get("HJB_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise RuntimeError(f"libhjb.so not found at {path}: build it with "
                           "`python -m paper_1605_04821_b200.build` (no CPU fallback exists)")
    lib = C.CDLL(path)
    vp, i32, i64, d = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    sig = {
        "hjb_last_error": (C.c_char_p, []),
        "hjb_version": (i32, []),
        "hjb_grid_create": (i32, [C.POINTER(GridDesc), C.POINTER(vp)]),
        "hjb_grid_query": (i32, [vp, C.POINTER(Layout)]),
        "hjb_grid_destroy": (i32, [vp]),
        "hjb_set_coeffs": (i32, [vp, C.POINTER(Coeffs)]),
        "hjb_set_source": (i32, [vp, vp, vp]),
        "hjb_policy_update": (i32, [vp, d, vp, vp, vp, vp, C.POINTER(PiStats)]),
        "hjb_apply": (i32, [vp, d, vp, vp, vp]),
        "hjb_mg_params_default": (None, [i32, C.POINTER(MgParams)]),
        "hjb_mg_setup": (i32, [vp, d, vp, C.POINTER(MgParams)]),
        "hjb_mg_apply": (i32, [vp, vp, vp]),
        "hjb_solve_params_default": (None, [i32, C.POINTER(SolveParams)]),
        "hjb_solve": (i32, [vp, d, vp, vp, vp, C.POINTER(SolveParams), C.POINTER(SolveStats)]),
        "hjb_step": (i32, [vp, d, vp, vp, vp, vp, C.POINTER(SolveParams), C.POINTER(StepStats)]),
        "hjb_profile_reset": (i32, [vp, i32]),
        "hjb_profile_read": (i32, [vp, C.POINTER(Profile)]),
        "hjb_partition": (i32, [i32, i64, i32, i32, i64, C.POINTER(Layout)]),
        "hjb_comm_unique_id": (i32, [vp]),
        "hjb_cfl_rate": (i32, [vp, vp, C.POINTER(d)]),
        "hjb_set_boundary_samples": (i32, [vp, i32, vp]),
        "hjb_halo_plan": (i32, [i32, i64, i32, i32, i64, HaloMsg * 2, C.POINTER(i32)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


class HJBError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


def check(code: int):
    if code != 0:
        raise HJBError(code, load().hjb_last_error().decode(errors="replace"))


def partition(dim: int, n: int, nranks: int, rank: int, halo: int) -> dict:
    """Host-only slab layout of `rank` (hjb_partition); raises HJBError on invalid input."""
    lay = Layout()
    check(load().hjb_partition(dim, n, nranks, rank, halo, C.byref(lay)))
    return {f: getattr(lay, f) for f, _ in lay._fields_}


def halo_plan(dim: int, n: int, nranks: int, rank: int, halo: int) -> list:
    """Host-only halo messages of `rank` (hjb_halo_plan)."""
    msgs = (HaloMsg * 2)()
    cnt = C.c_int32()
    check(load().hjb_halo_plan(dim, n, nranks, rank, halo, msgs, C.byref(cnt)))
    return [dict(peer=m.peer, send_row=m.send_row, recv_row=m.recv_row, rows=m.rows) for m in msgs[:cnt.value]]


def comm_unique_id() -> bytes:
    """128-byte ncclUniqueId (rank 0 creates it, the caller broadcasts it)."""
    buf = C.create_string_buffer(128)
    check(load().hjb_comm_unique_id(buf))
    return buf.raw
