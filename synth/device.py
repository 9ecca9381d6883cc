"""Device-resident inputs for a synth Problem (input generation only, no method arithmetic):
the per-node coefficient fields, initial data and packed Dirichlet data as torch CUDA tensors
in the single-rank layout of include/hjb.h (full grid, lexicographic, x1 fastest)."""
from __future__ import annotations

import numpy as np


def node_fields(p, device="cuda", from_host=False):
    """Per-node fields as contiguous float64 device tensors.
    from_host=True evaluates them in numpy (bitwise identical to what the oracle sees) and
    copies; otherwise they are evaluated by torch on the device (large grids)."""
    import torch
    if from_host:
        f = p.fields(p.all_idx())
        return {k: torch.from_numpy(np.ascontiguousarray(v)).to(device) for k, v in f.items()}
    idx = torch.arange(p.N, device=device, dtype=torch.int64)
    f = p.fields(idx)
    return {k: v.contiguous() for k, v in f.items()}


def grid_for(p, device=0, from_host=None, t0=None):
    """Create an HJBGrid for problem p and upload tables + fields; returns (grid, fields)."""
    import torch
    from paper_1605_04821_b200 import HJBGrid
    if from_host is None:
        from_host = p.N <= (1 << 22)
    dev = torch.device("cuda", device)
    g = HJBGrid(p.d, p.P, p.K, p.Q, p.n, p.lo, p.hi, device=device)
    fields = node_fields(p, dev, from_host)
    sd, bd, cc = p.control_tables()
    fb, fc = p.f_tables(p.dt if t0 is None else t0)
    g.set_coeffs(sd, bd, cc, fb, fc, **fields)
    return g, fields


def initial_values(p, device="cuda", from_host=None):
    import torch
    if from_host is None:
        from_host = p.N <= (1 << 22)
    if from_host:
        return torch.from_numpy(np.ascontiguousarray(p.g(p.all_idx()))).to(device)
    return p.g(torch.arange(p.N, device=device, dtype=torch.int64)).contiguous()


def packed_psi(p, t, device="cuda"):
    """Dirichlet data psi(t) at the boundary nodes in lexicographic order (hjb.h packed layout)."""
    import torch
    b = p.boundary_idx()
    return torch.from_numpy(np.ascontiguousarray(p.psi(t, b))).to(device)
