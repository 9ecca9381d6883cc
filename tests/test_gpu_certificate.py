"""Full-grid certificates of GPU marches at BASELINE sizes (VERDICT r1 "next" 1).

The GPU marches a config with bench.py's exact solver settings (library defaults: inexact early
policy evaluations, W-cycle on the large levels, extrapolated initial iterate from the second step
on).  After a step the C oracle (oracle/certify.c, pinned in test_oracle_certify.py) evaluates the
nonlinear residual
    R_n = max_j | U^n_j - U^{n-1}_j - dt min_a H^a_j(U^n) |
of the GPU's pair (U^{n-1}, U^n) over EVERY interior row.  By D6 the exact step solution U* from the
GPU's U^{n-1} satisfies ||U^n - U*||_inf <= R_n / (1 - dt max c) <= R_n (c = -0.1), and the implicit
step map is non-expansive in the max-norm (M-matrix, A^{-1} >= 0, row sums >= 1), so the GPU march
is within sum_n R_n of the oracle's exact march from u*(0).  The NS tolerance is 1e-8 ||u||_inf.

  cfg2 (2049^2, K = 64, 16 steps): every step certified on every row.
  cfg3 (129^3, K = 96, 16 steps): every step certified on every row.
  cfg4 (16385^2, K = 32, 8 steps, 2.7e8 unknowns): the final step on every row (~1e10 (node,
      control) pairs: ~2 min on the box's 16 host cores), every other step on 20 000 sampled rows
      (the nodes nearest every corner and face included).
"""
import os
import time

import numpy as np
import pytest

from gpu_util import require_gpu
from oracle import certify
from synth import bj_config

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

TOL = 1e-8


def _march(p, on_step):
    """March p over its n_steps with bench.py's settings; on_step(s, U_prev_dev, U_dev, stats)."""
    torch = require_gpu()
    from paper_1605_04821_b200 import _lib
    from synth.device import grid_for, initial_values, packed_psi
    g, fields = grid_for(p, device=0)
    U = initial_values(p).contiguous()
    U2 = torch.empty_like(U)
    pol = torch.zeros(p.N, dtype=torch.uint8, device="cuda")
    for s in range(1, p.n_steps + 1):
        t = s * p.dt
        fb, fc = p.f_tables(t)
        g.set_source(fb, fc)
        st = g.step(p.dt, U, U2, pol, packed_psi(p, t),
                    guess=_lib.HJB_GUESS_EXTRAPOLATE if s >= 2 else _lib.HJB_GUESS_PREV)
        torch.cuda.synchronize()
        on_step(s, U, U2, st, fields)
        U, U2 = U2, U
    g.close()


def _certify_rows(p, t, Uprev_h, U_h, fields, r0, r1, chunk_rows):
    """max R over interior rows [r0, r1) in row blocks (fields copied to host per block)."""
    re = p.n ** (p.d - 1)
    H = p.halo_rows() + 1
    Rmax = 0.0
    for a in range(r0, r1, chunk_rows):
        b = min(r1, a + chunk_rows)
        w0, w1 = max(0, a - H), min(p.n, b + H)
        sl = slice(a * re, b * re)
        fw = {k: np.ascontiguousarray(v[..., sl].cpu().numpy()) for k, v in fields.items()}
        R = certify.residual_rows(p, t, p.dt, a, b, U_h[w0 * re:w1 * re], w0 * re, Uprev_h[sl], fw,
                                  a * re, (b - a) * re)
        Rmax = max(Rmax, R)
    return Rmax


def _sample_rows_R(p, t, Uprev_h, U_h, fields, m=20000, seed=9):
    """R_j on m random interior nodes (+ corners / face midpoints) via the numpy oracle."""
    from oracle.howard import control_search
    rng = np.random.default_rng(seed)
    n = p.n
    special = [1, 2, n // 2, n - 3, n - 2]
    pts = [np.concatenate([rng.integers(1, n - 1, size=m),
                           np.array(np.meshgrid(*([special] * p.d), indexing="ij")).reshape(p.d, -1)[k]])
           for k in range(p.d)]
    idx = np.zeros_like(pts[0])
    for k in reversed(range(p.d)):
        idx = idx * n + pts[k]
    idx = np.unique(idx.astype(np.int64))
    sr = control_search(p, U_h, Uprev_h, t, p.dt, idx=idx)
    return float(sr.R.max())


@pytest.mark.parametrize("cfg", [2, 3])
def test_march_certified_every_step_every_row(cfg):
    p = bj_config(cfg)
    Rs, norms = [], []

    def on_step(s, U, U2, st, fields):
        Uph, Uh = U.cpu().numpy(), U2.cpu().numpy()
        R = _certify_rows(p, s * p.dt, Uph, Uh, fields, 1, p.n - 1, 256 if p.d == 2 else 32)
        Rs.append(R)
        norms.append(np.abs(Uh).max())
        assert R <= TOL * max(1.0, norms[-1]), (s, R, st)

    t0 = time.time()
    _march(p, on_step)
    assert sum(Rs) <= TOL * max(1.0, max(norms)), Rs
    print(f"cfg{cfg}: R per step {['%.1e' % r for r in Rs]} (sum {sum(Rs):.2e}), {time.time() - t0:.0f} s, "
          f"{os.cpu_count()} host cpus")


def test_march_certified_cfg4():
    p = bj_config(4)
    Rs = []

    def on_step(s, U, U2, st, fields):
        Uph, Uh = U.cpu().numpy(), U2.cpu().numpy()
        t = s * p.dt
        if s < p.n_steps:
            R = _sample_rows_R(p, t, Uph, Uh, fields)
        else:
            t0 = time.time()
            R = _certify_rows(p, t, Uph, Uh, fields, 1, p.n - 1, 2048)
            print(f"cfg4 final-step certificate over {p.N_interior} rows: R = {R:.3e} in "
                  f"{time.time() - t0:.0f} s on {os.cpu_count()} host cpus")
        Rs.append(R)
        assert R <= TOL * max(1.0, float(np.abs(Uh).max())), (s, R, st)

    _march(p, on_step)
    print("cfg4 R per step:", ["%.1e" % r for r in Rs])
