"""Pins of the multigrid components (SURVEY §8(c) "MG (preconditioner only)"):
prolongation exact on bilinear functions, full weighting reproduces constants, the Galerkin coarse
operator of the 5-point Laplacian is the classical 9-point stencil, V(1,1) Gauss-Seidel on the
5-point Laplacian contracts by <= 0.2, and the LISL sigma = 2I model degrades at even
levels (no interpolation).  CPU only."""
import numpy as np
import scipy.sparse as sp

from oracle.multigrid import galerkin_hierarchy, prolongation, stationary_rho, vcycle
from oracle.system import assemble
from synth import lisl_laplacian


def _grid(n):
    x = np.linspace(0.0, 1.0, n)
    X1, X2 = np.meshgrid(x[1:-1], x[1:-1], indexing="xy")     # x1 fastest after ravel
    return X1.ravel(), X2.ravel()


def test_prolongation_exact_on_bilinear_functions():
    nc = 17
    P = prolongation(nc)
    f = lambda a, b: 0.3 + 1.7 * a - 0.9 * b + 2.3 * a * b  # noqa: E731
    xc1, xc2 = _grid(nc)
    xf1, xf2 = _grid(2 * nc - 1)
    pf = P @ f(xc1, xc2)
    h = 1.0 / (2 * nc - 2)
    deep = (xf1 > 1.5 * h) & (xf1 < 1 - 1.5 * h) & (xf2 > 1.5 * h) & (xf2 < 1 - 1.5 * h)
    assert np.abs(pf[deep] - f(xf1, xf2)[deep]).max() < 1e-14     # every parent an interior node


def test_full_weighting_reproduces_constants():
    nc = 17
    P = prolongation(nc)
    R = P.T / 4.0
    rc = R @ np.ones(P.shape[0])
    xc1, xc2 = _grid(nc)
    hc = 1.0 / (nc - 1)
    deep = (xc1 > 1.5 * hc) & (xc1 < 1 - 1.5 * hc) & (xc2 > 1.5 * hc) & (xc2 < 1 - 1.5 * hc)
    assert np.abs(rc[deep] - 1.0).max() < 1e-15


def _five_point(n):
    m = n - 2
    T = sp.diags([-np.ones(m - 1), 2 * np.ones(m), -np.ones(m - 1)], [-1, 0, 1])
    I = sp.eye(m)
    return (sp.kron(I, T) + sp.kron(T, I)).tocsr() * (n - 1) ** 2


def test_galerkin_of_five_point_laplacian_is_nine_point_stencil():
    """Textbook: with bilinear P and full weighting R = P^T/4, the Galerkin operator R A_h P of the
    5-point Laplacian is the classical 9-point stencil (1/(4 H^2)) [-1 -2 -1; -2 12 -2; -1 -2 -1],
    H = 2h, at every deep coarse node."""
    n = 33
    A = _five_point(n)
    lv = galerkin_hierarchy(A, n, coarsest_n=17)
    Ac = lv[1][0].toarray()
    nc = 17
    H = 1.0 / (nc - 1)
    m = nc - 2
    j = (m // 2) * m + m // 2                      # a deep coarse row
    row = Ac[j].reshape(m, m)
    c1, c0 = m // 2, m // 2
    st = row[c1 - 1:c1 + 2, c0 - 1:c0 + 2] * (4 * H * H)
    assert np.allclose(st, [[-1, -2, -1], [-2, 12, -2], [-1, -2, -1]], atol=1e-10), st
    assert abs(row.sum() - st.sum() / (4 * H * H)) < 1e-8 * abs(row).max()   # nothing else in the row


def test_vcycle_gauss_seidel_five_point_contracts():
    """V(1,1) on the 2D 5-point Laplacian 65^2 contracts by rho <= 0.2."""
    n = 65
    lv = galerkin_hierarchy(_five_point(n), n)
    b = np.ones((n - 2) ** 2)
    rho, k = stationary_rho(lv, b, nu1=1, nu2=1, smoother="gs")
    assert rho <= 0.2, (rho, k)


def _lisl_laplacian_matrix(sig, ell):
    p = lisl_laplacian(sig, ell)
    z = np.zeros(p.N)
    sysm = assemble(p, np.zeros(p.N, dtype=np.int64), 1.0, 1.0, z, z)
    return (sysm.A - sp.eye(sysm.A.shape[0])).tocsr(), p.n          # = -L_hat (c = 0, dt = 1)


def test_lisl_sigma2_even_level_degrades():
    """P:954-962 / S:493: for the LISL Laplacian with sigma = 2I the steps land on nodes at even levels
    (no interpolation) and Galerkin GMG V(1,1)-GS converges markedly slower there than at the odd
    level below; sigma = sqrt(5) I (always interpolated) does not show the jump.  Measured when
    written: sigma = 2: l = 7 rho 0.063, l = 8 rho 0.366; sqrt 5: l = 7 0.056, l = 8 0.093."""
    r = {}
    for sig in (2.0, 5 ** 0.5):
        for ell in (7, 8):
            A, n = _lisl_laplacian_matrix(sig, ell)
            lv = galerkin_hierarchy(A, n)
            r[(sig, ell)] = stationary_rho(lv, np.ones(A.shape[0]), nu1=1, nu2=1, smoother="gs")[0]
    assert r[(2.0, 8)] > 3 * r[(2.0, 7)], r
    assert r[(5 ** 0.5, 8)] < 0.5 * r[(2.0, 8)], r


def test_jacobi_vcycle_is_a_convergent_preconditioner():
    """Damped Jacobi (the library's smoother, omega = 1) V(2,2) with Galerkin coarse operators on an
    implicit LISL system (M-matrix, row sums >= 1): the stationary iteration converges."""
    from synth import bj_config
    p = bj_config(2, n=65, K=8)
    rng = np.random.default_rng(3)
    pol = rng.integers(0, p.K, size=p.N)
    z = np.zeros(p.N)
    A = assemble(p, pol, p.dt, p.dt, z, z).A
    lv = galerkin_hierarchy(A, p.n)
    rho, k = stationary_rho(lv, np.ones(A.shape[0]), nu1=2, nu2=2, smoother="jacobi")
    assert rho < 0.5 and k < 40, (rho, k)


def test_galerkin_w_cycle_needs_damping():
    """Reading xxix: on Galerkin coarse operators (not M-matrices) the W-cycle with coarse Jacobi
    damping 0.8 diverges while 0.6 contracts strongly (cfg2 model, 257^2, greedy policy at U0)."""
    from oracle.howard import control_search
    from oracle.scheme import Geometry
    from synth import bj_config
    p = bj_config(2, n=257)
    U0 = p.g(p.all_idx())
    inter = Geometry.of(p).interior_idx()
    pol = np.zeros(p.N, dtype=np.int64)
    pol[inter] = control_search(p, U0, U0, p.dt, p.dt).policy
    z = np.zeros(p.N)
    lv = galerkin_hierarchy(assemble(p, pol, p.dt, p.dt, z, z).A, p.n)
    b = np.ones(inter.size)
    rho6, _ = stationary_rho(lv, b, nu1=2, nu2=2, omega=1.0, omega_coarse=0.6, gamma=2, maxit=40)
    assert rho6 < 0.2, rho6
