"""Aggregation-based algebraic multigrid (oracle).

PAPER.md:171-176 and P:1162-1164: "aggregation based methods ... as preconditioners of a Krylov
method, and part of an enhanced multigrid cycle" (the K-cycle: "at each coarse level the solution to
the residual equation is computed using a number of Krylov subspace iterations"), aggregates "formed
using heuristic criteria following coupling in the strongest direction", GCR as the outer Krylov
method, one Gauss-Seidel pre- and post-smoothing step; the theory needs an
M-matrix with non-negative row and column sums, which makes the symmetric part A + A^T an M-matrix
with non-negative row sums -- so couplings are measured on the symmetric part.

    pairwise matching   node i (unaggregated, in index order) pairs with the unaggregated j of most
                        negative symmetrised coupling (a_ij + a_ji)/2 if it is strong:
                        -(a_ij + a_ji)/2 >= beta * max_k -(a_ik + a_ki)/2; else it stays single
    double pairwise     two matching passes (the second on the pair-aggregated matrix): aggregates
                        of at most 4 nodes, P = 0/1 aggregate indicator, A_c = P^T A P
    K-cycle             level l: GS pre-smoothing, residual, the coarse system solved by 2 flexible
                        CG/GCR iterations preconditioned by the K-cycle of level l+1 (exact on the
                        coarsest), prolongation, GS post-smoothing
    stop coarsening     at <= max(stop_n, N^(1/3)) unknowns

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def pairwise_matching(A: sp.csr_matrix, beta: float = 0.25):
    """agg[i] = aggregate index of node i (pairs or singletons), in index order of the leaders."""
    n = A.shape[0]
    S = ((A + A.T) * 0.5).tocsr()
    agg = -np.ones(n, dtype=np.int64)
    na = 0
    indptr, indices, data = S.indptr, S.indices, S.data
    for i in range(n):
        if agg[i] >= 0:
            continue
        row = slice(indptr[i], indptr[i + 1])
        cols, vals = indices[row], data[row]
        off = cols != i
        strongest = max(0.0, float((-vals[off]).max(initial=0.0)))
        best, bj = 0.0, -1
        for c, v in zip(cols, vals):
            if c == i or agg[c] >= 0:
                continue
            if -v > best:
                best, bj = -v, c
        if bj >= 0 and best >= beta * strongest and best > 0.0:
            agg[i] = agg[bj] = na
        else:
            agg[i] = na
        na += 1
    return agg, na


def indicator(agg, na):
    n = agg.size
    return sp.csr_matrix((np.ones(n), (np.arange(n), agg)), shape=(n, na))


def double_pairwise(A: sp.csr_matrix, beta: float = 0.25):
    """Two pairwise passes: P = P1 P2 (aggregates of <= 4 nodes), A_c = P^T A P."""
    a1, n1 = pairwise_matching(A, beta)
    P1 = indicator(a1, n1)
    A1 = (P1.T @ A @ P1).tocsr()
    a2, n2 = pairwise_matching(A1, beta)
    P = (P1 @ indicator(a2, n2)).tocsr()
    return P, (P.T @ A @ P).tocsr()


def hierarchy(A: sp.csr_matrix, stop_n: int = 64, beta: float = 0.25, max_levels: int = 20):
    """[(A_l, P_l)] with P of the coarsest level None."""
    N1 = A.shape[0]
    stop = max(stop_n, int(round(N1 ** (1.0 / 3.0))))
    levels = [[A.tocsr(), None]]
    while levels[-1][0].shape[0] > stop and len(levels) < max_levels:
        P, Ac = double_pairwise(levels[-1][0], beta)
        if Ac.shape[0] >= levels[-1][0].shape[0]:       # no coarsening possible (e.g. diagonal matrix)
            break
        levels[-1][1] = P
        levels.append([Ac, None])
    return levels


def complexities(levels):
    """(grid complexity c_G = sum N_l / N_1, algebraic complexity c_A = sum nnz_l / nnz_1)."""
    N = [L[0].shape[0] for L in levels]
    Z = [L[0].nnz for L in levels]
    return sum(N) / N[0], sum(Z) / Z[0]


def _gs(A, b, x, lower=True):
    """One forward (lower) or backward Gauss-Seidel sweep."""
    if lower:
        L = sp.tril(A, format="csr")
        return spla.spsolve_triangular(L, b - sp.triu(A, k=1, format="csr") @ x, lower=True)
    U = sp.triu(A, format="csr")
    return spla.spsolve_triangular(U, b - sp.tril(A, k=-1, format="csr") @ x, lower=False)


def kcycle(levels, b, lvl=0, inner=2):
    """x = B_l^{-1} b: the K-cycle of level l (one GS pre- and post-smoothing step)."""
    A, P = levels[lvl]
    if P is None:
        return spla.spsolve(A.tocsc(), b)
    x = _gs(A, b, np.zeros_like(b), lower=True)
    rc = P.T @ (b - A @ x)
    Ac = levels[lvl + 1][0]
    if levels[lvl + 1][1] is None:
        ec = spla.spsolve(Ac.tocsc(), rc)
    else:
        ec = fgcr(Ac, rc, lambda v: kcycle(levels, v, lvl + 1, inner), maxit=inner, rtol=0.0)[0]
    x = x + P @ ec
    return _gs(A, b, x, lower=False)


def fgcr(A, b, prec, x0=None, rtol=1e-6, maxit=200, restart=10):
    """Flexible GCR (right preconditioning; P:1163 GCR for AGMG): returns (x, iterations, ||r||/||b||)."""
    x = np.zeros_like(b) if x0 is None else x0.copy()
    r = b - A @ x
    bn = np.linalg.norm(b)
    it = 0
    Z, AZ = [], []
    while it < maxit:
        if bn > 0 and np.linalg.norm(r) <= rtol * bn:
            break
        z = prec(r)
        az = A @ z
        for zz, aa in zip(Z, AZ):           # orthogonalise A z against the previous A z's
            h = az @ aa
            az = az - h * aa
            z = z - h * zz
        nrm = np.linalg.norm(az)
        if nrm == 0.0:
            break
        az, z = az / nrm, z / nrm
        g = r @ az
        x = x + g * z
        r = r - g * az
        Z.append(z)
        AZ.append(az)
        if len(Z) >= restart:
            Z, AZ = [], []
        it += 1
    return x, it, (np.linalg.norm(r) / bn if bn > 0 else 0.0)


def rho(levels, b, tol=1e-6, maxit=200):
    """Residual reduction factor (r_k / r_0)^(1/k) of K-cycle-preconditioned GCR to tol."""
    A = levels[0][0]
    x, k, rel = fgcr(A, b, lambda v: kcycle(levels, v), rtol=tol, maxit=maxit)
    return rel ** (1.0 / max(k, 1)), k
