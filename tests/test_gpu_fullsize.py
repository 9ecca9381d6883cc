"""Parity at BASELINE.json's FULL sizes, in the launch configuration bench.py times (single rank,
the library's own launch shapes), on SAMPLED outputs the oracle computes one by one:

  * operator apply (random x ~ U[-1,1], seed 43; random policy): sampled rows incl. every corner /
    edge-adjacent region, row-wise <= 1e-12 (reading xvi);
  * control search at U0: sampled rows, policy identical unless near-tie, F within 1e-12;
  * one full implicit step (hjb_step with bench.py's solver settings): the oracle's nonlinear
    residual R_j(U_gpu) at sampled rows is at the solver tolerance -- by D6 this bounds
    |U_gpu - U*| (a property that holds at any size).
cfg2 (2049^2, K = 64), cfg3 (129^3, K = 96, trilinear) and cfg4 (16385^2, K = 32, 2.7e8 unknowns).
"""
import numpy as np
import pytest

from gpu_util import require_gpu
from oracle.howard import control_search, hamiltonian
from oracle.scheme import Geometry, apply_operator, lhat_rows, node_coefficients
from synth import bj_config, random_vector

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _sample_interior(p, m, seed=5):
    """m random interior nodes plus the nodes nearest every corner and face midpoint."""
    rng = np.random.default_rng(seed)
    n = p.n
    pts = [rng.integers(1, n - 1, size=m) for _ in range(p.d)]
    special = [1, 2, n // 2, n - 3, n - 2]
    grid = np.array(np.meshgrid(*([special] * p.d), indexing="ij")).reshape(p.d, -1)
    mi = [np.concatenate([pts[k], grid[k]]) for k in range(p.d)]
    idx = np.zeros_like(mi[0])
    for k in reversed(range(p.d)):
        idx = idx * n + mi[k]
    return np.unique(idx.astype(np.int64))


@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_fullsize_apply_sampled(cfg):
    torch = require_gpu()
    from synth.device import grid_for
    p = bj_config(cfg)
    g, _ = grid_for(p, device=0)
    dev_idx = torch.arange(p.N, device="cuda")
    x = random_vector(p, idx=dev_idx).contiguous()                      # seed 43, identical to numpy
    pol = (torch.remainder(dev_idx * 2654435761, p.K)).to(torch.uint8)   # deterministic mixed policy
    y = torch.empty_like(x)
    g.apply(p.dt, pol, x, y)
    torch.cuda.synchronize()
    idx = _sample_interior(p, 3000)
    xh = x.cpu().numpy()
    polh = pol.cpu().numpy().astype(np.int64)
    yo = apply_operator(p, polh, xh, p.dt, idx=idx)
    yg = y.cpu().numpy()[idx]
    geo = Geometry.of(p)
    sig, b, c = node_coefficients(p, idx, polh[idx])
    cols, vals, _ = lhat_rows(geo, geo.node_x(idx), sig, b)
    xa = np.abs(xh)
    scale = xa[idx] + p.dt * (np.sum(vals * (xa[cols] + xa[idx][:, None]), axis=1) + np.abs(c) * xa[idx])
    # NS: "operator apply <= 1e-12 relative in max-norm"
    assert np.abs(yg - yo).max() <= 1e-12 * np.abs(yo).max()
    # row-wise (reading xvi): the rounding scale of a row plus the oracle's own coordinate rounding:
    # it forms z = lo + i h + mu y and (z - lo)/h in physical units, which carries an absolute error
    # of ~(n-1) eps cells in the fraction s at large n (the grid-unit GPU path has ~|o| eps)
    tol = 1e-12 + 4.0 * (p.n - 1) * np.finfo(float).eps
    err = np.abs(yg - yo) / scale
    print(f"cfg{cfg}: row-wise apply error / rounding scale: max {err.max():.3e} (tolerance {tol:.3e}); "
          f"max-norm relative {np.abs(yg - yo).max() / np.abs(yo).max():.3e}")
    assert err.max() <= tol, (err.max(), tol)


@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_fullsize_search_and_step_sampled(cfg):
    torch = require_gpu()
    from synth.device import grid_for, initial_values, packed_psi
    p = bj_config(cfg)
    g, _ = grid_for(p, device=0)
    U0 = initial_values(p).contiguous()
    pol = torch.zeros(p.N, dtype=torch.uint8, device="cuda")
    F = torch.zeros(p.N, dtype=torch.float64, device="cuda")
    g.policy_update(p.dt, U0, U0, pol, F)
    torch.cuda.synchronize()
    idx = _sample_interior(p, 1500)
    U0h = U0.cpu().numpy()
    sr = control_search(p, U0h, U0h, p.dt, p.dt, idx=idx)
    pg = pol.cpu().numpy()[idx].astype(np.int64)
    decisive = sr.ties == 1
    assert np.array_equal(pg[decisive], sr.policy[decisive])
    Hg, _, _ = hamiltonian(p, idx, pg, U0h, p.dt, p.fields(idx))
    assert np.all(Hg - sr.H <= 1e-12 * sr.scale)
    Fg = F.cpu().numpy()[idx]
    assert np.abs(Fg[decisive] - sr.F[decisive]).max(initial=0.0) <= 1e-12 * max(1.0, np.abs(sr.F).max())
    # one implicit step with bench.py's settings, then the oracle's residual certificate
    fb, fc = p.f_tables(p.dt)
    g.set_source(fb, fc)
    U1 = torch.empty_like(U0)
    st = g.step(p.dt, U0, U1, pol, packed_psi(p, p.dt))
    torch.cuda.synchronize()
    U1h = U1.cpu().numpy()
    sr1 = control_search(p, U1h, U0h, p.dt, p.dt, idx=idx)
    # R_j = |U_j - U^{n-1}_j - dt min_a H^a_j(U)|: the GPU stopped at R <= 1e-10 or at an exactly
    # evaluated stable policy (rres <= 1e-12); allow the rounding scale of the recomputation
    bound = max(st["final_R"], 1e-10) + 1e-12 * p.dt * sr1.scale + 1e-12 * (1 + np.abs(U1h[idx]))
    assert np.all(sr1.R <= 2 * bound), (sr1.R.max(), st)
    # boundary rows hold psi exactly
    bidx = p.boundary_idx()
    assert np.array_equal(U1h[bidx], p.psi(p.dt, bidx))
