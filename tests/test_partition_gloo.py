"""Multi-rank host logic on CPU (gloo, world_size 2): the library's slab partition (hjb_partition)
tiles the interior rows, and its halo plan (hjb_halo_plan) + halo width rule give every owned row
all the data its stencil reads.  Each rank holds ONLY its local slab (rows outside it are NaN),
fills its halos by exchanging exactly the rows the plan names (gloo send/recv, the same messages
the NCCL path sends), then evaluates the oracle operator at its owned rows: the result must equal
the single-grid oracle bit for bit and contain no NaN.  A halo one row too small must fail."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1605_04821_b200 import _lib
from synth import bj_config, random_vector

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cfg, n, K, halo_delta, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.scheme import Geometry, apply_operator
        p = bj_config(cfg, n=n, K=K)
        H = p.halo_rows() + halo_delta
        lay = _lib.partition(p.d, p.n, world, rank, H)
        re = lay["row_elems"]
        # tiling of the interior rows across ranks
        rows = torch.tensor([lay["row0"], lay["row1"]], dtype=torch.int64)
        allr = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allr, rows)
        ok_tiling = allr[0][0].item() == 1 and allr[-1][1].item() == p.n - 1 and all(
            allr[q][1].item() == allr[q + 1][0].item() for q in range(world - 1))
        # global data (seeded; identical on every rank) and the local slab view
        x_glob = random_vector(p)
        pol_glob = np.random.default_rng(7).integers(0, p.K, size=p.N)
        lo, lr = lay["local_row0"], lay["local_rows"]
        local = np.full(lr * re, np.nan)
        own0, own1 = lay["row0"], lay["row1"]
        # owned rows and any Dirichlet boundary rows inside the local window are known locally
        for r in range(lo, lo + lr):
            if own0 <= r < own1 or r == 0 or r == p.n - 1:
                local[(r - lo) * re:(r - lo + 1) * re] = x_glob[r * re:(r + 1) * re]
        # halo exchange exactly as planned (send to lower first, then upper: matching order)
        reqs = []
        for m in _lib.halo_plan(p.d, p.n, world, rank, H):
            snd = torch.from_numpy(local[(m["send_row"] - lo) * re:(m["send_row"] - lo + m["rows"]) * re].copy())
            rcv = torch.empty(m["rows"] * re, dtype=torch.float64)
            reqs.append((dist.isend(snd, m["peer"]), dist.irecv(rcv, m["peer"]), rcv, m))
        for s_, r_, rcv, m in reqs:
            s_.wait()
            r_.wait()
            a = (m["recv_row"] - lo) * re
            local[a:a + m["rows"] * re] = rcv.numpy()
        # evaluate the operator at owned rows using ONLY the local slab
        x_view = np.full(p.N, np.nan)
        x_view[lo * re:(lo + lr) * re] = local
        geo = Geometry.of(p)
        inter = geo.interior_idx()
        slow = inter // re
        mine = inter[(slow >= own0) & (slow < own1)]
        y_loc = apply_operator(p, pol_glob, x_view, p.dt, idx=mine)
        y_ref = apply_operator(p, pol_glob, x_glob, p.dt, idx=mine)
        res = [ok_tiling, int(mine.size), bool(np.isnan(y_loc).any()),
               bool(np.array_equal(y_loc, y_ref))]
        out[rank] = res
    finally:
        dist.destroy_process_group()


def _run(cfg, n, K, halo_delta=0, world=2):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, n, K, halo_delta, out)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(240)
        assert pr.exitcode == 0, f"worker exit {pr.exitcode}"
    return [out[r] for r in range(world)]


@pytest.mark.parametrize("cfg,n,K", [(0, 33, 16), (2, 129, 7), (3, 21, 96)])
def test_slab_halo_gloo(cfg, n, K):
    res = _run(cfg, n, K if cfg != 3 else None)
    p = bj_config(cfg, n=n, K=K if cfg != 3 else None)
    assert sum(r[1] for r in res) == p.N_interior        # every interior row owned exactly once
    for ok_tiling, cnt, has_nan, equal in res:
        assert ok_tiling and not has_nan and equal


def test_halo_one_row_short_is_detected():
    res = _run(0, 33, 16, halo_delta=-1)
    assert any(r[2] for r in res)                         # some owned row reads an unfilled row


def test_partition_rejects_thin_slabs():
    from paper_1605_04821_b200 import HJBError
    with pytest.raises(HJBError):
        _lib.partition(2, 33, 8, 0, 5)                    # 31 rows / 8 ranks < 5 halo rows
    lay = _lib.partition(2, 33, 1, 0, 7)
    assert lay["halo"] == 0 and lay["local_rows"] == 33 and lay["n_interior"] == 31 * 31
