"""Geometric multigrid with Galerkin coarse operators (oracle).

PAPER.md:932-937: "the smoother is Gauss-Seidel, the prolongation operator bilinear interpolation,
the restriction the transpose of the prolongation, and the coarse grid operator is constructed using
the Galerkin principle".  Grids have 2^l + 1 nodes per dimension; unknowns are interior nodes
(lexicographic, x1 fastest); the coarse boundary is Dirichlet (zero correction).

    P        bilinear interpolation from the coarse interior to the fine interior
    R        P^T / 4 (full weighting; the scale cancels in the correction P (R A P)^-1 R)
    A_{l+1}  R A_l P

Cycles: V(nu1, nu2) with damped Jacobi (the GPU library's smoother, for its parity tests) or
lexicographic Gauss-Seidel (the paper's), exact coarsest solve.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def prolongation_1d(nc: int) -> sp.csr_matrix:
    """Linear interpolation from the nc - 2 coarse interior nodes to the 2 nc - 3 fine interior nodes
    of a uniform grid (fine node i: even -> coarse i/2, odd -> the mean of its two neighbours);
    coarse boundary nodes carry 0 (Dirichlet)."""
    nf = 2 * nc - 1
    rows, cols, vals = [], [], []
    for i in range(1, nf - 1):
        if i % 2 == 0:
            parents = [(i // 2, 1.0)]
        else:
            parents = [(i // 2, 0.5), (i // 2 + 1, 0.5)]
        for I, w in parents:
            if 1 <= I <= nc - 2:
                rows.append(i - 1)
                cols.append(I - 1)
                vals.append(w)
    return sp.csr_matrix((vals, (rows, cols)), shape=(nf - 2, nc - 2))


def prolongation(nc: int, d: int = 2) -> sp.csr_matrix:
    """Tensor-product (bi/tri)linear prolongation on the interior, x1 fastest."""
    p1 = prolongation_1d(nc)
    P = p1
    for _ in range(d - 1):
        P = sp.kron(p1, P)
    return P.tocsr()


def galerkin_hierarchy(A: sp.csr_matrix, n: int, d: int = 2, coarsest_n: int = 9):
    """[(A_l, P_l, d)]: A_0 = A on n^d nodes, A_{l+1} = R A_l P_l with R = P_l^T / 2^d, coarsening
    while n > coarsest_n (n = 2^l + 1); P of the coarsest level is None."""
    levels = [[A.tocsr(), None, d]]
    nn = n
    while nn > coarsest_n and (nn - 1) % 2 == 0:
        nc = (nn - 1) // 2 + 1
        P = prolongation(nc, d)
        Ac = ((P.T @ levels[-1][0] @ P) / (2 ** d)).tocsr()
        levels[-1][1] = P
        levels.append([Ac, None, d])
        nn = nc
    return levels


def vcycle(levels, b, nu1=2, nu2=2, omega=1.0, smoother="jacobi", lvl=0, omega_coarse=None, gamma=1):
    """x = M^-1 b: one V(nu1, nu2) cycle from x = 0 (damped Jacobi with omega on the finest level and
    omega_coarse (default omega) below, or forward lexicographic Gauss-Seidel), full-weighting
    restriction R = P^T / 2^d, prolongation P, exact solve on the coarsest level."""
    A, P, d = levels[lvl]
    if lvl > 0 and omega_coarse is not None:
        omega = omega_coarse
    if P is None:
        return spla.spsolve(A.tocsc(), b)
    D = A.diagonal()
    if smoother == "jacobi":
        step = lambda x: x + omega * (b - A @ x) / D  # noqa: E731
    else:
        L = sp.tril(A, format="csr")
        U = sp.triu(A, k=1, format="csr")
        step = lambda x: spla.spsolve_triangular(L, b - U @ x, lower=True)  # noqa: E731
    x = np.zeros_like(b)
    for _ in range(nu1):
        x = step(x)
    rc = (P.T @ (b - A @ x)) / (2 ** d)
    oc = omega if omega_coarse is None else omega_coarse
    ec = vcycle(levels, rc, nu1, nu2, oc, smoother, lvl + 1, omega_coarse, gamma)
    Ac = levels[lvl + 1][0]
    for _ in range(gamma - 1):             # W-cycle: refine the coarse correction (cycle index gamma)
        if levels[lvl + 1][1] is None:
            break
        ec = ec + vcycle(levels, rc - Ac @ ec, nu1, nu2, oc, smoother, lvl + 1, omega_coarse, gamma)
    x = x + P @ ec
    for _ in range(nu2):
        x = step(x)
    return x


def stationary_rho(levels, b, tol=1e-6, maxit=200, **kw):
    """rho = (r_k / r_0)^(1/k) of the stationary MG iteration x += M^-1 (b - A x) from x = 0 until
    ||r_k||_2 <= tol ||b||_2 (the paper's residual reduction factor)."""
    A = levels[0][0]
    x = np.zeros_like(b)
    r0 = np.linalg.norm(b)
    k = 0
    rn = r0
    while rn > tol * r0 and k < maxit:
        x = x + vcycle(levels, b - A @ x, **kw)
        rn = np.linalg.norm(b - A @ x)
        k += 1
    return (rn / r0) ** (1.0 / max(k, 1)), k
