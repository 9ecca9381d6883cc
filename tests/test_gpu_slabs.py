"""Slab decomposition on one GPU: R ranks as host threads of this process (HJB_COMM_THREADS, the
test-only backend: halos by device copies ordered with CUDA events, no kernel waits on another).
Everything above the exchange -- partition, halo widths, per-level ownership, the gather level,
rank-ordered reductions, the collective call sequence of hjb_step -- is the code the NCCL path runs.

  * operator apply and control search on slabs are BIT-IDENTICAL to the single-rank result
    (same per-node arithmetic, halos carry exact copies);
  * full implicit steps on slabs match the CPU oracle within the NS tolerance (1e-8 ||u||_inf).
"""
import os
import threading

import numpy as np
import pytest

from gpu_util import require_gpu, to_dev
from oracle.howard import howard_step
from synth import bj_config, random_vector

pytestmark = pytest.mark.gpu


def _run_ranks(R, body):
    """Run body(rank, key) in R threads; re-raise the first error."""
    key = os.urandom(128)
    out, errs = [None] * R, [None] * R

    def work(r):
        try:
            out[r] = body(r, key)
        except BaseException as e:  # noqa: BLE001
            errs[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    for e in errs:
        if e is not None:
            raise e
    return out


def _assemble(p, parts):
    """Owned rows of every rank -> one full-grid array (boundary rows from the edge ranks)."""
    full = np.full(p.N, np.nan)
    for lay, loc in parts:
        re, lo = lay["row_elems"], lay["local_row0"]
        r0, r1 = lay["row0"], lay["row1"]
        if r0 == 1:
            r0 = 0
        if r1 == p.n - 1:
            r1 = p.n
        full[r0 * re:r1 * re] = loc[(r0 - lo) * re:(r1 - lo) * re]
    return full


def _slab_apply_and_search(p, R):
    torch = require_gpu()
    from synth.device import grid_for, local_index
    x = random_vector(p)
    pol = np.random.default_rng(7).integers(0, p.K, size=p.N).astype(np.uint8)
    Uprev = p.g(p.all_idx())
    U = Uprev + 0.05 * np.random.default_rng(11).uniform(-1, 1, size=p.N)

    def body(r, key):
        st = torch.cuda.Stream()
        g, fields = grid_for(p, 0, from_host=True, rank=r, nranks=R, comm="threads", comm_id=key, stream=st)
        lay = g.layout()
        li = local_index(p, lay, numpy=True)
        with torch.cuda.stream(st):
            xd, pd = to_dev(x[li], torch), to_dev(pol[li], torch)
            y = torch.zeros(lay["local_elems"], dtype=torch.float64, device="cuda")
            Ud, Upd = to_dev(U[li], torch), to_dev(Uprev[li], torch)
            pol2 = torch.zeros(lay["local_elems"], dtype=torch.uint8, device="cuda")
            F = torch.zeros(lay["local_elems"], dtype=torch.float64, device="cuda")
        st.synchronize()
        g.apply(p.dt, pd, xd, y)
        stt = g.policy_update(p.dt, Ud, Upd, pol2, F)
        st.synchronize()
        res = (lay, y.cpu().numpy(), pol2.cpu().numpy().astype(np.float64), F.cpu().numpy(), stt)
        g.close()
        return res

    return _run_ranks(R, body)


@pytest.mark.parametrize("cfg,n,K,R", [(0, 33, 16, 2), (2, 129, 7, 3), (3, 17, None, 2)])
def test_slab_apply_and_search_bitwise(cfg, n, K, R):
    torch = require_gpu()
    from synth.device import grid_for
    p = bj_config(cfg, n=n, K=K)
    parts = _slab_apply_and_search(p, R)
    # single-rank reference on the same inputs
    g, _ = grid_for(p, 0, from_host=True)
    x = random_vector(p)
    pol = np.random.default_rng(7).integers(0, p.K, size=p.N).astype(np.uint8)
    y = torch.zeros(p.N, dtype=torch.float64, device="cuda")
    g.apply(p.dt, to_dev(pol, torch), to_dev(x, torch), y)
    Uprev = p.g(p.all_idx())
    U = Uprev + 0.05 * np.random.default_rng(11).uniform(-1, 1, size=p.N)
    pol2 = torch.zeros(p.N, dtype=torch.uint8, device="cuda")
    F = torch.zeros(p.N, dtype=torch.float64, device="cuda")
    st1 = g.policy_update(p.dt, to_dev(U, torch), to_dev(Uprev, torch), pol2, F)
    torch.cuda.synchronize()
    inter = ~p.is_boundary(p.all_idx())
    ya = _assemble(p, [(q[0], q[1]) for q in parts])
    pa = _assemble(p, [(q[0], q[2]) for q in parts])
    Fa = _assemble(p, [(q[0], q[3]) for q in parts])
    assert np.array_equal(ya[inter], y.cpu().numpy()[inter])
    assert np.array_equal(pa[inter], pol2.cpu().numpy()[inter].astype(np.float64))
    assert np.array_equal(Fa[inter], F.cpu().numpy()[inter])
    for q in parts:                                   # reductions agree on every rank
        assert q[4]["changed"] == st1["changed"] and q[4]["R_max"] == st1["R_max"]


def _slab_march(p, R, steps, **kw):
    torch = require_gpu()
    from synth.device import grid_for, initial_values, packed_psi

    def body(r, key):
        st = torch.cuda.Stream()
        g, fields = grid_for(p, 0, from_host=True, rank=r, nranks=R, comm="threads", comm_id=key, stream=st)
        lay = g.layout()
        with torch.cuda.stream(st):
            U = initial_values(p, lay=lay).contiguous()
            U2 = torch.empty_like(U)
            pol = torch.zeros(lay["local_elems"], dtype=torch.uint8, device="cuda")
        stats = []
        for s in range(1, steps + 1):
            t = s * p.dt
            fb, fc = p.f_tables(t)
            g.set_source(fb, fc)
            with torch.cuda.stream(st):
                psi = packed_psi(p, t)
            st.synchronize()
            stats.append(g.step(p.dt, U, U2, pol, psi, **kw))
            U, U2 = U2, U
        st.synchronize()
        res = (lay, U.cpu().numpy(), stats)
        g.close()
        return res

    return _run_ranks(R, body)


@pytest.mark.parametrize("name,cfg,n,K,R,steps,mg", [
    ("cfg0_R2", 0, 33, 16, 2, 2, {}),
    ("cfg2_257_R3_slab_coarse_levels", 2, 257, 8, 3, 1, {"gather_n": 33}),
    ("cfg2_257_R2_wcycle_on_slab_levels", 2, 257, 8, 2, 1, {"gather_n": 33, "gamma": 2, "gamma_min_nodes": 0}),
    ("cfg3_17_R2", 3, 17, None, 2, 1, {}),
])
def test_slab_step_matches_oracle(name, cfg, n, K, R, steps, mg):
    p = bj_config(cfg, n=n, K=K)
    parts = _slab_march(p, R, steps, mg=mg, pi_forcing=1e-2)
    Ug = _assemble(p, [(q[0], q[1]) for q in parts])
    Uo = p.g(p.all_idx())
    for s in range(1, steps + 1):
        Uo, _, _ = howard_step(p, Uo, s * p.dt, p.dt)
    err = np.abs(Ug - Uo).max() / max(1.0, np.abs(Uo).max())
    assert err <= 1e-8, (name, err, parts[0][2][-1])
    # every rank took the same decisions (collective sequence in lockstep)
    for q in parts[1:]:
        assert [st["pi_iters"] for st in q[2]] == [st["pi_iters"] for st in parts[0][2]]
        assert [st["krylov_iters_total"] for st in q[2]] == [st["krylov_iters_total"] for st in parts[0][2]]
    if mg.get("gather_n") == 33 and "gamma" not in mg:
        assert parts[0][2][-1]["n_levels"] >= 4


def test_wcycle_revisit_is_rank_independent():
    """the W-cycle revisit is decided on a coarse level's GLOBAL interior count, so every
    rank count takes the same branch.  gamma_min_nodes = 127^2 (the 129^2 level of n = 257) sits
    exactly at the global count: a per-rank count (~127^2 / R) would skip the revisit for R > 1
    (and desynchronise the collectives across ranks).  Identical Krylov counts for R = 1, 2, 3."""
    p = bj_config(2, n=257, K=8)
    mg = {"gather_n": 33, "gamma": 2, "gamma_min_nodes": 127 * 127}
    counts = []
    for R in (1, 2, 3):
        parts = _slab_march(p, R, 1, mg=mg, pi_forcing=1e-2)
        counts.append([st["krylov_iters"] for st in parts[0][2]])
        for q in parts[1:]:
            assert [st["krylov_iters"] for st in q[2]] == counts[-1]
    assert counts[0] == counts[1] == counts[2], counts
