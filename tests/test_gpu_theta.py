"""theta-scheme on the GPU (eq. FullScheme, Proposition
CFL P:437-441) through the C-ABI (hjb_step with hjb_solve_params.theta, hjb_cfl_rate):

  * parity with the oracle's theta-march (oracle.howard.march(theta=...)) on the same inputs:
    explicit Euler (theta = 0, no solve: rounding only) and theta = 1/2 (policy iteration, solves
    to 1e-12; NS tolerance 1e-8 ||u||_inf);
  * the positivity rate of Proposition CFL against the oracle's cfl_rate;
  * the errors PAPER.md prints for Problems A / B (tests/golden/paper_theta_tables.json) at the grid
    sizes the oracle cannot reach in a test (161^2 .. 641^2): explicit truncated steps incl. the CFL
    blow-ups (dt = dx/4 from N_x = 321; two-sided overstepping on the shifted domain), implicit
    steps at every step size -- the GPU reproduction of Tables 1, 1-B, shifted, 4 and 4-B.
"""
import json
import math
import os

import numpy as np
import pytest

from gpu_util import require_gpu, setup, to_dev
from oracle.howard import cfl_rate, control_search, march
from oracle.scheme import Geometry
from synth import bj_config, problem_A, problem_B

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_theta_tables.json")))
MK = {"A": lambda nx: problem_A(nx), "B": lambda nx: problem_B(nx),
      "A_shifted": lambda nx: problem_A(nx, shift=7 * math.pi / 8)}


def gpu_march(p, n_steps, theta, from_host=True):
    """theta-march on the GPU with the library defaults; returns (U full grid, per-step stats) or
    (None, stats) if the march stopped on a non-finite value (the CFL blow-up)."""
    torch = require_gpu()
    from paper_1605_04821_b200 import HJBError, _lib
    from synth.device import packed_psi
    g, _ = setup(p, from_host=from_host)
    dt = p.T / n_steps
    U = to_dev(p.g(p.all_idx()), torch)
    U2 = torch.empty_like(U)
    pol = torch.zeros(p.N, dtype=torch.uint8, device="cuda")
    stats = []
    try:
        for s in range(1, n_steps + 1):
            fb, fc = p.f_tables((s - 1) * dt + theta * dt)      # f at t_{n-1} + theta dt
            g.set_source(fb, fc)
            stats.append(g.step(dt, U, U2, pol, packed_psi(p, s * dt), theta=theta,
                                guess=_lib.HJB_GUESS_PREV))
            U, U2 = U2, U
        torch.cuda.synchronize()
        out = U.cpu().numpy()
        if not np.all(np.isfinite(out)):
            out = None
    except HJBError as e:
        if "NONFINITE" not in str(e):
            raise
        out = None
    g.close()
    return out, stats


@pytest.mark.parametrize("name,mk,theta,steps", [
    ("probA_41_explicit", lambda: problem_A(41), 0.0, 9),
    ("probB_41_explicit", lambda: problem_B(41), 0.0, 9),
    ("probA_shift_41_explicit", lambda: problem_A(41, shift=7 * math.pi / 8), 0.0, 21),
    ("probA_41_theta_half", lambda: problem_A(41), 0.5, 4),
    ("cfg2_65_K8_theta_half", lambda: bj_config(2, n=65, K=8), 0.5, 2),
    ("cfg3_9_explicit", lambda: bj_config(3, n=9), 0.0, 3),
])
def test_theta_march_parity(name, mk, theta, steps):
    p = mk()
    Ug, st = gpu_march(p, steps, theta)
    Uo, _, _ = march(p, n_steps=steps, theta=theta)
    scale = max(1.0, np.abs(Uo).max())
    tol = 1e-11 if theta == 0.0 else 1e-8            # explicit: rounding only; else solves to 1e-12
    assert Ug is not None
    assert np.abs(Ug - Uo).max() <= tol * scale, (name, np.abs(Ug - Uo).max(), st[-1])


def test_cfl_rate_matches_oracle():
    torch = require_gpu()
    p = problem_A(81)
    g, _ = setup(p)
    r_all = g.cfl_rate(None)
    ro, _ = cfl_rate(p)
    assert abs(r_all - ro) <= 1e-10 * ro, (r_all, ro)
    U = p.u_exact(0.25, p.all_idx())
    inter = Geometry.of(p).interior_idx()
    pol = np.zeros(p.N, dtype=np.int64)
    pol[inter] = control_search(p, U, U, 0.25, 0.01).policy
    r_pol = g.cfl_rate(to_dev(pol.astype(np.uint8), torch))
    ro_pol, _ = cfl_rate(p, policy=pol)
    assert abs(r_pol - ro_pol) <= 1e-10 * ro_pol and r_pol <= r_all
    g.close()


def _steps(p, col):
    dx = (p.hi - p.lo) / (p.n - 1)
    dt = {0: p.T, 1: dx / 4, 2: dx ** 1.5, 3: dx ** 2}[col]
    return int(math.ceil(p.T / dt - 1e-12))


TABLE_CASES = [
    # explicit (theta = 0): Tables 1 / 1-B / shifted
    ("explicit", "A", 161, 0), ("explicit", "A", 321, 0), ("explicit", "A", 641, 0),
    ("explicit", "A", 161, 1), ("explicit", "A", 321, 1), ("explicit", "A", 321, 2), ("explicit", "A", 641, 2),
    ("explicit", "B", 321, 0), ("explicit", "B", 321, 1), ("explicit", "B", 641, 2),
    ("explicit", "A_shifted", 161, 1), ("explicit", "A_shifted", 321, 3), ("explicit", "A_shifted", 641, 0),
    # implicit (theta = 1): Tables 4 / 4-B
    ("implicit", "A", 321, 0), ("implicit", "A", 641, 0), ("implicit", "A", 161, 1), ("implicit", "A", 321, 2),
    ("implicit", "B", 321, 0),
    # Table 4-B at N_x = 641 (dt = T) and 161 (dt = dx^1.5) is NOT reproduced within 5 %: measured
    # 1.713e-3 vs 1.53e-3 and 8.63e-3 vs 6.37e-3 (r02); the oracle agrees with the GPU
    # (321, dt = T: oracle 3.1693e-3, GPU 3.169e-3, paper 3.04e-3).  Problem B ties every control at u*
    # and the printed rates of that table are irregular (1.50, 0.86, 1.36).
]


@pytest.mark.slow
@pytest.mark.parametrize("scheme,prob,nx,col", TABLE_CASES)
def test_paper_theta_tables_gpu(scheme, prob, nx, col):
    p = MK[prob](nx)
    U, _ = gpu_march(p, _steps(p, col), 0.0 if scheme == "explicit" else 1.0)
    gold = GOLD[f"{scheme}_{prob}"][str(nx)][col]
    if gold is None or gold > 1.0:                 # the paper's blown-up explicit march
        assert U is None or np.abs(U - p.u_exact(p.T, p.all_idx())).max() > 1e3
        return
    assert U is not None
    err = float(np.abs(U - p.u_exact(p.T, p.all_idx())).max())
    print(f"{scheme} {prob} N_x={nx} column {GOLD['columns'][col]}: error {err:.3e} (paper {gold:.2e})")
    assert abs(err / gold - 1) <= 0.05, (err, gold)
