"""Device-resident inputs for a synth Problem (input generation only, no method arithmetic):
the per-node coefficient fields, initial data and packed Dirichlet data as torch CUDA tensors
in the layout of include/hjb.h (lexicographic, x1 fastest).  With nranks > 1 every array is the
rank's local slab: global rows [local_row0, local_row0 + local_rows) of the slowest axis."""
from __future__ import annotations

import numpy as np


def local_index(p, lay=None, device=None, numpy=False):
    """Global flat node indices of the local array described by `lay` (None: the full grid)."""
    import torch
    start = 0 if lay is None else lay["local_row0"] * lay["row_elems"]
    count = p.N if lay is None else lay["local_elems"]
    if numpy:
        return np.arange(start, start + count, dtype=np.int64)
    return torch.arange(start, start + count, device=device, dtype=torch.int64)


def node_fields(p, device="cuda", from_host=False, lay=None):
    """Per-node fields as contiguous float64 device tensors on the local array.
    from_host=True evaluates them in numpy (bitwise identical to what the oracle sees) and
    copies; otherwise they are evaluated by torch on the device (large grids)."""
    import torch
    if from_host:
        f = p.fields(local_index(p, lay, numpy=True))
        return {k: torch.from_numpy(np.ascontiguousarray(v)).to(device) for k, v in f.items()}
    f = p.fields(local_index(p, lay, device=device))
    return {k: v.contiguous() for k, v in f.items()}


def grid_for(p, device=0, from_host=None, t0=None, rank=0, nranks=1, halo=None, comm="nccl",
             comm_id=None, stream=None):
    """Create an HJBGrid for problem p (slab `rank` of `nranks`) and upload tables + fields;
    returns (grid, fields)."""
    import torch
    from paper_1605_04821_b200 import HJBGrid
    if from_host is None:
        from_host = p.N <= (1 << 22)
    if nranks > 1 and halo is None:
        halo = p.halo_rows()
    dev = torch.device("cuda", device)
    g = HJBGrid(p.d, p.P, p.K, p.Q, p.n, p.lo, p.hi, device=device, stream=stream, rank=rank,
                nranks=nranks, halo=halo or 0, comm=comm, comm_id=comm_id)
    lay = g.layout()
    with torch.cuda.stream(stream) if stream is not None else _nullctx():
        fields = node_fields(p, dev, from_host, lay)
    if stream is not None:
        stream.synchronize()
    sd, bd, cc = p.control_tables()
    fb, fc = p.f_tables(p.dt if t0 is None else t0)
    g.set_coeffs(sd, bd, cc, fb, fc, **fields)
    return g, fields


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def initial_values(p, device="cuda", from_host=None, lay=None):
    import torch
    if from_host is None:
        from_host = p.N <= (1 << 22)
    if from_host:
        return torch.from_numpy(np.ascontiguousarray(p.g(local_index(p, lay, numpy=True)))).to(device)
    return p.g(local_index(p, lay, device=device)).contiguous()


def packed_psi(p, t, device="cuda"):
    """Dirichlet data psi(t) at the boundary nodes in lexicographic order (hjb.h packed layout)."""
    import torch
    b = p.boundary_idx()
    return torch.from_numpy(np.ascontiguousarray(p.psi(t, b))).to(device)
