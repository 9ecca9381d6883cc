"""Pins of the C certificate oracle (oracle/certify.c): it must agree with the numpy oracle's
brute-force control search (oracle.howard.control_search, itself pinned in test_oracle_*.py) row by
row on every interior node -- R_j within the rounding scale, the argmin identical wherever the
minimum is decisive -- on configs that exercise every branch (truncated rows, per-node scale and
offset fields, 3D, exact ties), and must satisfy the D6 error bound against an exact discrete
solution.  CPU only."""
import numpy as np
import pytest

from oracle import certify
from oracle.howard import control_search, howard_step
from oracle.scheme import Geometry
from synth import bj_config, problem_A, problem_B

CASES = [
    ("cfg0_33", lambda: bj_config(0)),
    ("cfg2_65_K8_noise_truncation", lambda: bj_config(2, n=65, K=8)),
    ("cfg3_9", lambda: bj_config(3, n=9)),
    ("problemA_41_sigma_node", lambda: problem_A(41)),
    ("problemB_41_ties", lambda: problem_B(41)),
]


@pytest.mark.parametrize("name,mk", CASES, ids=[c[0] for c in CASES])
def test_certificate_matches_numpy_oracle(name, mk):
    p = mk()
    inter = Geometry.of(p).interior_idx()
    rng = np.random.default_rng(3)
    Up = p.g(p.all_idx())
    U = Up.copy()
    U[inter] += 0.01 * rng.uniform(-1, 1, inter.size)
    t, dt = p.dt, p.dt
    sr = control_search(p, U, Up, t, dt)
    R, pol, Rr = certify.residual(p, U, Up, t, dt, with_policy=True)
    assert R == pytest.approx(sr.R.max(), rel=1e-12, abs=1e-13)
    tol = 1e-12 * (1.0 + dt * sr.scale)
    assert np.all(np.abs(Rr[inter] - sr.R) <= tol)
    decisive = sr.ties == 1
    assert np.array_equal(pol[inter][decisive], sr.policy[decisive])
    if name.startswith("problemB"):
        assert (~decisive).sum() > 0          # ties exercised


def test_certificate_d6_bound():
    """D6: ||U - U*||_inf <= R(U) / (1 - dt c_max) with U* the exact step solution (c = -0.1)."""
    p = bj_config(2, n=33, K=8)
    dt = p.dt
    U0 = p.g(p.all_idx())
    Ustar, _, _ = howard_step(p, U0, dt, dt, tol_pi=0.0)
    inter = Geometry.of(p).interior_idx()
    rng = np.random.default_rng(4)
    for amp in (1e-3, 1e-7):
        U = Ustar.copy()
        U[inter] += amp * rng.uniform(-1, 1, size=inter.size)
        R = certify.residual(p, U, U0, dt, dt)
        err = np.abs(U - Ustar).max()
        assert err <= R / (1 + 0.1 * dt) * (1 + 1e-9) + 1e-14
        assert R <= 50 * err                   # and it is not vacuous
    assert certify.residual(p, Ustar, U0, dt, dt) <= 1e-10


def test_certificate_row_blocks_compose():
    """Row-block calls (as the full-size GPU tests make them, with offset windows) give the same
    per-row values as one call over the whole grid."""
    p = bj_config(2, n=65, K=8)
    Up = p.g(p.all_idx())
    U = Up + 0.01 * np.random.default_rng(5).uniform(-1, 1, p.N)
    ff = p.fields(p.all_idx())
    _, _, Rfull = certify.residual(p, U, Up, p.dt, p.dt, fields_full=ff, with_policy=True)
    n = p.n
    H = p.halo_rows()
    for r0, r1 in ((1, 20), (20, 41), (41, n - 1)):
        w0, w1 = max(0, r0 - H), min(n, r1 + H)
        Uw = np.ascontiguousarray(U[w0 * n:w1 * n])
        sl = slice(r0 * n, r1 * n)
        fw = {k: np.ascontiguousarray(v[..., sl]) for k, v in ff.items()}
        Rr = np.zeros((r1 - r0) * n)
        R = certify.residual_rows(p, p.dt, p.dt, r0, r1, Uw, w0 * n, np.ascontiguousarray(Up[sl]), fw,
                                  r0 * n, (r1 - r0) * n, Rrow=Rr)
        own = Rfull[sl]
        m = own > 0
        assert np.array_equal(Rr[m], own[m]) and R == own.max()
