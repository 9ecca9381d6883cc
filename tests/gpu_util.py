"""Helpers for the GPU parity tests: build/load libhjb and put a synth problem on the device."""
import numpy as np


def require_gpu():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("GPU test selected but no CUDA device is visible (no fallback exists)")
    from paper_1605_04821_b200 import build
    build.build()
    return torch


def to_dev(a, torch):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def setup(p, from_host=True):
    """(grid, fields) with fields computed in numpy (identical inputs to the oracle's)."""
    from synth.device import grid_for
    return grid_for(p, device=0, from_host=from_host)


def row_scale(p, policy_full, x_full, dt, idx, fields=None):
    """Rounding scale |A||x| of each row (SURVEY reading xvi): |x_j| + dt (sum_i l_ji (|x_i|+|x_j|)
    + |c_j x_j|), from the oracle's l_hat rows."""
    from oracle.scheme import Geometry, lhat_rows, node_coefficients
    geo = Geometry.of(p)
    sig, b, c = node_coefficients(p, idx, policy_full[idx], fields)
    cols, vals, _ = lhat_rows(geo, geo.node_x(idx), sig, b)
    xa = np.abs(x_full)
    return xa[idx] + dt * (np.sum(vals * (xa[cols] + xa[idx][:, None]), axis=1) + np.abs(c) * xa[idx])
