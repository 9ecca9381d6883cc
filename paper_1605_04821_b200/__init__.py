"""B200-native implicit semi-Lagrangian HJB step (arXiv:1605.04821): C-ABI library libhjb.so
(sm_100a CUDA kernels, fp64) and its thin Python binding."""
from .api import HJBGrid  # noqa: F401
from ._lib import HJBError, load  # noqa: F401

__all__ = ["HJBGrid", "HJBError", "load"]
