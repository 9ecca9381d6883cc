"""Pins for the oracle's stencil layer against values the paper and mathematics fix
(not against the oracle itself).  CPU only."""
import math

import numpy as np
import pytest

from oracle.scheme import (Geometry, drift_weights, interp_weights, lhat_rows, node_coefficients,
                           stencil_pairs, truncation_mu, truncation_weights, apply_operator)
from synth import bj_config, lisl_laplacian, noise, problem_A, problem_B, random_vector


# ------------------------------------------------------------------ input generator
def test_splitmix64_reference_value():
    # splitmix64 with state 0: first output is 0xE220A8397B1DCDAF (the generator's published
    # first value); pins the counter generator both sides draw from.
    assert int(noise.splitmix64_np(np.array([0], dtype=np.uint64))[0]) == 0xE220A8397B1DCDAF


def test_noise_numpy_torch_identical():
    torch = pytest.importorskip("torch")
    idx = np.arange(0, 5000, 7)
    a = noise.uniform_pm1_np(42, 3, idx)
    b = noise.uniform_pm1_torch(42, 3, torch.from_numpy(idx)).numpy()
    assert np.array_equal(a, b)
    assert a.min() >= -1 and a.max() < 1 and abs(a.mean()) < 0.05


# ------------------------------------------------------------------ truncation
def test_mu_worked_examples():
    # Omega=[0,1], x=15/16, y=+1/4 -> mu=1/4; 2D x=(15/16,1/2), y=(1/4,1/4) -> 1/4
    geo = Geometry(2, 17, 0.0, 1.0)
    x = np.array([[15 / 16, 0.5], [15 / 16, 0.5], [0.5, 0.5]])
    y = np.array([[0.25, 0.0], [0.25, 0.25], [0.1, -0.2]])
    mu, bind = truncation_mu(geo, x, y)
    assert mu == pytest.approx([0.25, 0.25, 1.0], abs=1e-15)
    assert bind[0, 0] and not bind[0, 1] and not bind[2].any()


def test_weights_worked_examples():
    # SPEC S:177-178, re-derived from eq. (eqn_Ap)/(eqn_APp1): mu+=1/4, mu-=1 -> A=6.4, B=1.6;
    # drift mu=1/2 -> A=B=2; no overstep -> A=B=1.
    A, B = truncation_weights(np.array([0.25, 1.0]), np.array([1.0, 1.0]))
    assert A == pytest.approx([6.4, 1.0]) and B == pytest.approx([1.6, 1.0])
    Ad, Bd = drift_weights(np.array([0.5]))
    assert Ad[0] == pytest.approx(2.0) and Bd[0] == pytest.approx(2.0)


@pytest.mark.parametrize("mk", [lambda: problem_A(81), lambda: bj_config(2, n=129),
                                lambda: bj_config(3, n=17)])
def test_consistency_conditions_all_nodes(mk):
    """eqs. (AB1)-(AB2) and (AB_drift), hold exactly (to rounding) at every interior node
    and control: A y+ + B y- = 0, A y+y+^T + B y-y-^T = 2dx sigma sigma^T, (A+B) y_d = 2dx b,
    and A, B >= 1 (Corollary a)."""
    p = mk()
    geo = Geometry.of(p)
    idx = geo.interior_idx()
    x = geo.node_x(idx)
    fields = p.fields(idx)
    for a in range(0, p.K, max(1, p.K // 8)):
        sig, b, _ = node_coefficients(p, idx, np.full(idx.size, a), fields)
        pairs = stencil_pairs(geo, x, sig, b)
        scale = geo.dx * np.max(np.sum(sig ** 2, axis=2))
        for q, (zp, A, zm, B) in enumerate(pairs[:-1]):
            yp, ym = zp - x, zm - x
            assert np.all(A >= 1 - 1e-14) and np.all(B >= 1 - 1e-14)
            first = A[:, None] * yp + B[:, None] * ym
            assert np.abs(first).max() <= 1e-12 * math.sqrt(scale) * A.max()
            second = (A[:, None, None] * yp[:, :, None] * yp[:, None, :]
                      + B[:, None, None] * ym[:, :, None] * ym[:, None, :])
            target = 2 * geo.dx * sig[:, q, :, None] * sig[:, q, None, :]
            assert np.abs(second - target).max() <= 1e-10 * scale
            # every truncated endpoint lies on the closed domain (case B cannot occur)
            assert zp.min() >= geo.lo and zp.max() <= geo.hi and zm.min() >= geo.lo and zm.max() <= geo.hi
        zd, Ad, _, Bd = pairs[-1]
        assert np.abs((Ad + Bd)[:, None] * (zd - x) - 2 * geo.dx * b).max() <= 1e-12 * max(1.0, np.abs(b).max())


def test_truncation_growth_law():
    """Corollary b: one-sided truncation gives A ~ dx^{-1/2}; the untruncated side -> 2."""
    vals = []
    for nx in (41, 81, 161):
        p = problem_A(nx)
        geo = Geometry.of(p)
        idx = geo.interior_idx()
        x = geo.node_x(idx)
        sig, b, _ = node_coefficients(p, idx, np.zeros(idx.size, dtype=int))
        (zp, A, zm, B) = stencil_pairs(geo, x, sig, b)[0]
        dist = np.linalg.norm(zm - x, axis=1)
        full = np.isclose(dist, geo.k * np.linalg.norm(sig[:, 0, :], axis=1))
        one_sided = (A > 1.0) & full
        vals.append(A[one_sided].max() * math.sqrt(geo.dx))
        # node adjacent to the boundary: B (untruncated side) close to 2
        k = np.argmax(A * full)
        assert 1.5 < B[k] <= 2.0
    assert max(vals) / min(vals) < 1.6      # A * sqrt(dx) bounded above and below


# ------------------------------------------------------------------ interpolation
def test_interp_worked_example_and_properties():
    geo = Geometry(2, 2, 0.0, 1.0)
    cols, w = interp_weights(geo, np.array([[0.25, 0.5]]))
    got = dict(zip(cols[0].tolist(), w[0].tolist()))
    # weights (0.375, 0.125, 0.375, 0.125) on vertices in lexicographic node order
    assert [got[i] for i in range(4)] == pytest.approx([0.375, 0.125, 0.375, 0.125])
    rng = np.random.default_rng(0)
    for d in (2, 3):
        geo = Geometry(d, 9, -1.0, 1.0)
        z = rng.uniform(-1, 1, size=(2000, d))
        z[:5] = 1.0                                        # upper face (reading vii)
        cols, w = interp_weights(geo, z)
        assert np.all(w >= 0) and np.abs(w.sum(1) - 1).max() < 1e-14
        xn = geo.node_x(np.arange(9 ** d))
        g = rng.normal(size=d)
        aff = xn @ g + 0.3
        assert np.abs((w * aff[cols]).sum(1) - (z @ g + 0.3)).max() < 1e-13
        # w_i(x_j) = delta_ij
        cols, w = interp_weights(geo, xn)
        assert np.abs((w * (cols == np.arange(9 ** d)[:, None])).sum(1) - 1).max() < 1e-14


# ------------------------------------------------------------------ the operator
@pytest.mark.parametrize("cfg", [0, 2, 3])
def test_constants_annihilated(cfg):
    """L_hat[1] = 0 (partition of unity) => (A 1)_j = 1 - dt c_j at every interior row,
    i.e. the full row sum is 1 - dt c >= 1."""
    p = bj_config(cfg, n=17)
    rng = np.random.default_rng(1)
    pol = rng.integers(0, p.K, size=p.N)
    y = apply_operator(p, pol, np.ones(p.N), dt=0.37)
    assert np.abs(y - (1 + 0.37 * 0.1)).max() < 1e-11


def _quad_check(p, phi, Hmat, grad, rtol=1e-11):
    geo = Geometry.of(p)
    idx = geo.interior_idx()
    x = geo.node_x(idx)
    fields = p.fields(idx)
    xn = geo.node_x(np.arange(p.N))
    phi_full = phi(xn)
    for a in range(0, p.K, max(1, p.K // 4)):
        sig, b, _ = node_coefficients(p, idx, np.full(idx.size, a), fields)
        cols, vals, rowsum = lhat_rows(geo, x, sig, b)
        L = np.sum(vals * (phi_full[cols] - phi(x)[:, None]), axis=1)
        # drift endpoint never truncated here (|dx b| < dx <= distance to the boundary)
        exact = (0.5 * np.einsum("mpi,ij,mpj->m", sig, Hmat, sig)
                 + np.einsum("mi,mi->m", b, grad(x))
                 + 0.5 * geo.dx * np.einsum("mi,ij,mj->m", b, Hmat, b))
        assert np.abs(L - exact).max() <= rtol * rowsum.max() * np.abs(phi_full).max()


def test_quadratic_cross_terms_exact_incl_truncated_rows():
    """D5 (derived from P:309-316 + multilinear exactness on x_i x_j): for phi with zero pure
    second derivatives the truncated LISL operator reproduces 1/2 sum_p s_p^T H s_p + b.grad phi
    + (dx/2) b^T H b exactly at EVERY interior node, truncated rows included."""
    p2 = bj_config(0, n=33)
    _quad_check(p2, lambda x: x[:, 0] * x[:, 1] + 0.3 * x[:, 0] - 0.2 * x[:, 1],
                np.array([[0, 1.0], [1.0, 0]]), lambda x: np.stack([x[:, 1] + 0.3, x[:, 0] - 0.2], 1))
    p3 = bj_config(3, n=17)
    H3 = np.array([[0, 1.0, 1.0], [1.0, 0, 1.0], [1.0, 1.0, 0]])
    _quad_check(p3, lambda x: x[:, 0] * x[:, 1] + x[:, 1] * x[:, 2] + x[:, 0] * x[:, 2],
                H3, lambda x: x @ H3)


def test_quadratic_squares_node_landing():
    """with sigma = 2I and even level, every step lands on a node (no interpolation),
    so L_hat[x1^2 + x2^2] = 1/2 sum_p sigma_p^T H sigma_p = 2 sigma^2 = 8 at every interior node,
    truncated ones included (truncated endpoints sit on boundary nodes)."""
    p = lisl_laplacian(2.0, 6)
    geo = Geometry.of(p)
    idx = geo.interior_idx()
    x = geo.node_x(idx)
    sig, b, _ = node_coefficients(p, idx, np.zeros(idx.size, dtype=int))
    xn = geo.node_x(np.arange(p.N))
    phi = (xn ** 2).sum(1)
    cols, vals, _ = lhat_rows(geo, x, sig, b)
    L = np.sum(vals * (phi[cols] - phi[idx][:, None]), axis=1)
    assert np.abs(L - 8.0).max() < 1e-9


def test_quadratic_interpolation_bias_closed_form():
    """Axis-aligned sigma = (s,0), k s/dx = r not integer: I_dx(x1^2)(x + r dx) - (x + r dx)^2
    = f (1-f) dx^2 with f = r - floor(r) (linear interpolation of a parabola), so at untruncated
    nodes L_hat[x1^2] = s^2 + f (1 - f) dx (P:736-740 stencil form)."""
    s = 1.37
    p = lisl_laplacian(s, 8)
    p.sigma_dir[:] = 0
    p.sigma_dir[0, 0, 0] = s
    geo = Geometry.of(p)
    idx = geo.interior_idx()
    x = geo.node_x(idx)
    sig, b, _ = node_coefficients(p, idx, np.zeros(idx.size, dtype=int))
    r = geo.k * s / geo.dx
    f = r - math.floor(r)
    inner = (x[:, 0] - r * geo.dx > 0) & (x[:, 0] + r * geo.dx < 1)
    xn = geo.node_x(np.arange(p.N))
    phi = xn[:, 0] ** 2
    cols, vals, _ = lhat_rows(geo, x, sig, b)
    L = np.sum(vals * (phi[cols] - phi[idx][:, None]), axis=1)
    assert np.abs(L[inner] - (s * s + f * (1 - f) * geo.dx)).max() < 1e-9
    assert inner.sum() > 0.5 * inner.size


def test_one_dimensional_closed_form_matrix():
    """for constant sigma in 1D, the LISL matrix is L_SL = gamma L^m + (1-gamma) L^{m+1}
    with m = floor(sigma/sqrt dx), gamma = (m+1) - sigma/sqrt dx, i.e. l_hat_{j,j+-m} = gamma/(2dx),
    l_hat_{j,j+-(m+1)} = (1-gamma)/(2dx) at nodes whose stencil does not overstep."""
    sigma = 2.3
    p = lisl_laplacian(sigma, 8)
    p.sigma_dir[:] = 0
    p.sigma_dir[0, 0, 0] = sigma                      # diffusion along x1 only
    geo = Geometry.of(p)
    m = math.floor(sigma / math.sqrt(geo.dx))
    gamma = (m + 1) - sigma / math.sqrt(geo.dx)
    # the paper's matrix on one grid line (dx = 1 normalisation): L^m has 2 on the diagonal, -1 at +-m
    Nline = p.n
    def Lm(mm):
        M = 2 * np.eye(Nline)
        M -= np.eye(Nline, k=mm) + np.eye(Nline, k=-mm)
        return M
    LSL = gamma * Lm(m) + (1 - gamma) * Lm(m + 1)
    row2 = p.n // 2
    line = np.arange(m + 2, p.n - m - 2)             # nodes whose stencil stays inside
    idx = row2 * p.n + line
    x = geo.node_x(idx)
    sig, b, _ = node_coefficients(p, idx, np.zeros(idx.size, dtype=int))
    cols, vals, _ = lhat_rows(geo, x, sig, b)
    for r, j in enumerate(line):
        full = np.zeros(p.N)
        np.add.at(full, cols[r], vals[r])
        got = full[row2 * p.n: (row2 + 1) * p.n].copy()
        assert full.sum() - got.sum() < 1e-12 * full.sum()     # nothing off the grid line
        got[j] -= full.sum()          # l_hat row -> operator row sum_i l_ji (phi_i - phi_j)
        assert np.abs(got - (-LSL[j] / (2 * geo.dx))).max() < 1e-9 / geo.dx


def test_exact_psi_mode_quadratic_closed_form():
    """Exact-psi boundary mode (Remark rhs; NEXT-2): a truncated endpoint takes psi(z), so
    for a quadratic phi = 1/2 x^T H x + g.x the truncated LISL row is D5 with the interpolation bias
    of the UNtruncated endpoints only:
        L_hat[phi](x_j) = 1/2 sum_p s_p^T H s_p + b.(H x_j + g) + (mu_d dx/2) b^T H b
                          + sum_{e untruncated} w_e sum_i (H_ii/2) s_{e,i}(1 - s_{e,i}) dx^2
    (the consistency identities D4 make a truncated pair exact given exact endpoint values).  The
    interpolation mode differs at truncated rows (face interpolation of a curved psi)."""
    import math as _m
    from oracle.scheme import interp_weights, lhat_apply, stencil_pairs
    p = bj_config(0, n=33)
    geo = Geometry.of(p)
    idx = geo.interior_idx()
    x = geo.node_x(idx)
    alpha = np.full(idx.size, 3)
    sig, b, _ = node_coefficients(p, idx, alpha)
    Hm = np.array([[1.4, -0.4], [-0.4, 2.6]])
    gv = np.array([0.2, -0.1])
    phi_of = lambda X: 0.5 * np.einsum("mi,ij,mj->m", X, Hm, X) + X @ gv  # noqa: E731
    phi = phi_of(geo.node_x(np.arange(p.N)))
    L_ex = lhat_apply(geo, idx, sig, b, phi, exact_psi=phi_of)
    L_in = lhat_apply(geo, idx, sig, b, phi)
    expect = 0.5 * np.einsum("mpi,ij,mpj->m", sig, Hm, sig) + np.einsum("mi,mi->m", b, x @ Hm + gv)
    trunc_any = np.zeros(idx.size, dtype=bool)
    for (zp, A, zm, B, tp, tm) in stencil_pairs(geo, x, sig, b, with_masks=True):
        for z, W, tr in ((zp, A, tp), (zm, B, tm)):
            t = (z - geo.lo) / geo.dx
            s = t - np.clip(np.floor(t), 0, geo.n - 2)
            bias = (W / (2 * geo.dx)) * np.sum(0.5 * np.diag(Hm)[None, :] * s * (1 - s), axis=1) * geo.dx ** 2
            expect = expect + np.where(tr, 0.0, bias)
            trunc_any |= tr
    # drift: (mu_d dx / 2) b^T H b (mu_d = 1: never truncated in cfg0)
    expect = expect + 0.5 * geo.dx * np.einsum("mi,ij,mj->m", b, Hm, b)
    assert np.abs(L_ex - expect).max() < 1e-9 * max(1.0, np.abs(expect).max()), np.abs(L_ex - expect).max()
    assert trunc_any.sum() > 0 and np.abs(L_in - L_ex)[trunc_any].max() > 1e-6
    assert np.abs(L_in - L_ex)[~trunc_any].max() <= 1e-12 * np.abs(L_in).max()   # same value, other summation order
