"""Pins of the oracle's theta-scheme (eq. FullScheme P:415-426,
Proposition / Corollary CFL P:437-452) against the errors PAPER.md prints for Problems A and B
(tests/golden/paper_theta_tables.json, every table cited there): explicit Euler (theta = 0) and
implicit Euler (theta = 1) with the truncated stencil, four step sizes, incl. the CFL blow-ups of the
explicit method (one-sided overstepping needs dt ~ dx^(3/2); two-sided, on the shifted domain,
dt ~ dx^2).  CPU only."""
import json
import math
import os

import numpy as np
import pytest

from oracle.howard import cfl_rate, howard_step, march
from oracle.scheme import Geometry
from oracle.system import assemble
from synth import problem_A, problem_B

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_theta_tables.json")))
MK = {"A": lambda nx: problem_A(nx), "B": lambda nx: problem_B(nx),
      "A_shifted": lambda nx: problem_A(nx, shift=7 * math.pi / 8)}


def _steps(p, col):
    dx = (p.hi - p.lo) / (p.n - 1)
    dt = {0: p.T, 1: dx / 4, 2: dx ** 1.5, 3: dx ** 2}[col]
    return int(math.ceil(p.T / dt - 1e-12))


def _check(err, gold):
    if gold is None or gold > 1.0:                 # the paper's blown-up explicit march
        assert (not np.isfinite(err)) or err > 1e3, err
    else:
        assert abs(err / gold - 1) <= 0.05, (err, gold)


CASES = [("explicit", "A", 41, c) for c in range(4)] + [("explicit", "B", 41, c) for c in range(4)] + \
        [("explicit", "A_shifted", 41, c) for c in range(4)] + [("implicit", "A", 41, c) for c in range(4)] + \
        [("implicit", "B", 41, c) for c in range(4)] + \
        [("explicit", "A", 81, c) for c in (0, 1, 2)] + [("explicit", "A_shifted", 81, c) for c in (1, 2, 3)]


@pytest.mark.parametrize("scheme,prob,nx,col", CASES)
def test_paper_theta_tables(scheme, prob, nx, col):
    p = MK[prob](nx)
    U, _, _ = march(p, n_steps=_steps(p, col), theta=0.0 if scheme == "explicit" else 1.0)
    err = float(np.abs(U - p.u_exact(p.T, p.all_idx())).max())
    _check(err, GOLD[f"{scheme}_{prob}"][str(nx)][col])


def test_theta_half_between_and_reduces():
    """theta = 1 reproduces the implicit step exactly; theta = 1/2 (Crank-Nicolson type) is a valid
    positive-type step where the CFL of Proposition CFL holds with (1 - theta): its error is of the
    same order as the explicit / implicit ones."""
    p = problem_A(41)
    U1, _, _ = march(p, n_steps=9, theta=1.0)
    U1b, _, _ = march(p, n_steps=9)
    assert np.array_equal(U1, U1b)
    Uh, _, _ = march(p, n_steps=9, theta=0.5)
    e = np.abs(Uh - p.u_exact(p.T, p.all_idx())).max()
    assert 0.02 < e < 0.06, e


def test_explicit_step_is_the_assembled_explicit_operator():
    """theta = 0: U^n = U^{n-1} + dt (L_hat^pi + c) U^{n-1} + dt f^pi with pi = argmin H(U^{n-1}); equal to
    F of the assembled theta-system (A = I) at that policy, i.e. the B^{n,n-1} row of P:419-424."""
    p = problem_B(21)
    U0 = p.g(p.all_idx())
    dt = 0.01
    U1, pol, _ = howard_step(p, U0, dt, dt, theta=0.0)
    psi = np.zeros(p.N)
    b = p.boundary_idx()
    psi[b] = p.psi(dt, b)
    sysm = assemble(p, pol, dt, dt, U0, psi, theta=0.0)
    assert abs(sysm.A - __import__("scipy.sparse", fromlist=["eye"]).eye(sysm.A.shape[0])).max() == 0
    assert np.abs(U1[sysm.interior] - sysm.F).max() <= 1e-13


def test_cfl_rate_growth_law():
    """Proposition / Corollary CFL: the positivity rate max_i (sum_p (A_p+B_p)/(2dx) - c_i)
    of the controls a march selects (the policy at u*(t = 1/4)) grows like dx^(-3/2) where one side
    of a diffusion stencil oversteps (Problem A) and like dx^(-2) where both sides do (the shifted
    domain's bottom-left corner, Remark two-over P:640-651).  Measured when written (N_x = 81 -> 161):
    A 77.0 -> 207.2 (exponent 1.43), shifted 166.9 -> 665.9 (2.00)."""
    from oracle.howard import control_search
    rates = {}
    for name in ("A", "A_shifted"):
        rr = []
        for nx in (81, 161):
            p = MK[name](nx)
            U = p.u_exact(0.25, p.all_idx())
            inter = Geometry.of(p).interior_idx()
            pol = np.zeros(p.N, dtype=np.int64)
            pol[inter] = control_search(p, U, U, 0.25, 0.01).policy
            rr.append(cfl_rate(p, policy=pol)[0])
        rates[name] = math.log2(rr[1] / rr[0])
    assert 1.3 <= rates["A"] <= 1.7, rates
    assert 1.85 <= rates["A_shifted"] <= 2.15, rates
    # without any selection (every control) the rate bounds the selected one
    p = problem_A(41)
    assert cfl_rate(p)[0] >= cfl_rate(p, policy=np.zeros(p.N, dtype=np.int64))[0]
