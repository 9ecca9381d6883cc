"""Seeded synthetic inputs shared by the oracle and the GPU harness (no method arithmetic)."""
from .problems import (Problem, bj_config, problem_A, problem_B, lisl_laplacian,  # noqa: F401
                       random_vector, eta)
from . import noise  # noqa: F401
