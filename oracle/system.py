"""Assembly of the implicit (theta = 1) positive-type system for a fixed policy, and its solve
(oracle).  P:103-127 (positive type), P:415-426 (eq. FullScheme and its B coefficients),
P:147-156 (nonlinear system, M-matrix, policy evaluation).

Unknowns are the interior nodes; Dirichlet values psi at boundary nodes are moved to the
right-hand side (reading ix: boundary rows are identities with rhs psi, eliminated here).

For theta = 1 the coefficients of eq. (FullScheme) are
    B^{n,n}_{jj}   = 1 + dt ( sum_p (A_p + B_p)/(2dx) - l_hat_jj - c_j )
    B^{n,n}_{ji}   = dt l_hat_ji          (i != j)
    B^{n,n-1}_{jj} = 1,  B^{n,n-1}_{ji} = 0
and the row reads  B_jj U_j - sum_{i!=j} B_ji U_i - U^{n-1}_j - dt f_j = 0.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .scheme import Geometry, lhat_rows, node_coefficients, source_term


class System:
    """A^pi (CSR over interior unknowns, interior ordering = lexicographic) and F^pi."""

    def __init__(self, A, F, interior, geo):
        self.A, self.F, self.interior, self.geo = A, F, interior, geo


def assemble(prob, policy_full, dt, t, U_prev_full, psi_full, fields=None, k_scale=1.0, theta=1.0,
             exact_psi=False):
    """Assemble A^pi, F^pi of the theta-scheme, eq. (FullScheme), for the policy pi:
        A^pi = I - theta dt (L_hat^pi + c^pi)                               (interior rows)
        F^pi = U^{n-1} + (1 - theta) dt (L_hat^pi + c^pi)[U^{n-1}] + dt f^pi
               + theta dt sum_{i in dOmega} l_hat_ji psi_i(t_n)
    (B^{n,n} and B^{n,n-1} of P:419-424 with time-independent sigma, b).  c and f are evaluated at
    t_{n-1} + theta dt; t is t_n.  U_prev_full holds psi(t_{n-1}) on the boundary.
    policy_full: control index per full-grid node (only interior entries used).  theta = 1 is the
    implicit Euler system of the paper's experiments (reading x).  exact_psi: the exact-psi boundary
    mode (Remark rhs): a truncated endpoint contributes psi(t_n, z) (psi(t_{n-1}, z) in the
    explicit part) to F instead of the interpolation of nodal boundary values (prob.psi_at)."""
    geo = Geometry.of(prob, k_scale)
    interior = geo.interior_idx()
    m = interior.size
    if fields is None:
        fields = prob.fields(interior)
    alpha = np.asarray(policy_full)[interior]
    sig, b, c = node_coefficients(prob, interior, alpha, fields)
    x = geo.node_x(interior)
    t_theta = t - dt + theta * dt
    if exact_psi:
        cols, vals, rowsum, bsum = lhat_rows(geo, x, sig, b, exact_psi=lambda z: prob.psi_at(t, z))
    else:
        cols, vals, rowsum = lhat_rows(geo, x, sig, b)
        bsum = np.zeros(m)

    # position of each full-grid node in the interior unknown vector (-1 for boundary)
    pos = np.full(prob.N, -1, dtype=np.int64)
    pos[interior] = np.arange(m)
    rows = np.repeat(np.arange(m), cols.shape[1])
    cflat, vflat = cols.ravel(), vals.ravel()
    cpos = pos[cflat]

    is_self = cflat == np.repeat(interior, cols.shape[1])
    l_jj = np.bincount(rows[is_self], weights=vflat[is_self], minlength=m)
    diag = 1.0 + theta * dt * (rowsum - l_jj - c)               # B^{n,n}_jj

    off = (~is_self) & (cpos >= 0)                              # interior off-diagonals
    A = sp.coo_matrix((np.concatenate([-theta * dt * vflat[off], diag]),
                       (np.concatenate([rows[off], np.arange(m)]),
                        np.concatenate([cpos[off], np.arange(m)]))), shape=(m, m)).tocsr()
    A.sum_duplicates()

    f = source_term(prob, t_theta, alpha, fields)
    bnd = cpos < 0                                              # couplings to boundary nodes
    F = U_prev_full[interior] + dt * f
    F = F + np.bincount(rows[bnd], weights=theta * dt * vflat[bnd] * psi_full[cflat[bnd]], minlength=m)
    F = F + theta * dt * bsum
    if theta < 1.0:                                             # B^{n,n-1} U^{n-1}: explicit part
        if exact_psi:
            cp, vp, rp, bp = lhat_rows(geo, x, sig, b, exact_psi=lambda z: prob.psi_at(t - dt, z))
            Lprev = np.sum(vp * U_prev_full[cp], axis=1) + bp - rp * U_prev_full[interior]
        else:
            Lprev = np.sum(vals * (U_prev_full[cols] - U_prev_full[interior][:, None]), axis=1)
        F = F + (1.0 - theta) * dt * (Lprev + c * U_prev_full[interior])
    return System(A, F, interior, geo)


def solve(system: System, x0=None, rtol=1e-13, direct_limit=70_000):
    """Policy evaluation A^pi X = F^pi.  Sparse direct (SuperLU) up to
    `direct_limit` unknowns, else ILU-preconditioned GMRES to ||F - AX||_2 <= rtol ||F||_2.
    The true residual is recomputed and returned."""
    A, F = system.A, system.F
    if A.shape[0] <= direct_limit:
        X = spla.splu(A.tocsc(), permc_spec="COLAMD").solve(F)
    else:
        ilu = spla.spilu(A.tocsc(), drop_tol=1e-5, fill_factor=20)
        M = spla.LinearOperator(A.shape, ilu.solve)
        X, info = spla.gmres(A, F, x0=x0, rtol=rtol, atol=0.0, M=M, restart=100, maxiter=200)
        if info != 0:
            raise RuntimeError(f"oracle gmres did not converge (info={info})")
    r = F - A @ X
    return X, float(np.linalg.norm(r) / max(np.linalg.norm(F), 1e-300))


def dense_solve(system: System):
    """Tiny-grid reference: numpy dense LU (LAPACK gesv)."""
    return np.linalg.solve(system.A.toarray(), system.F)
