"""Policy iteration (Howard) for the implicit step and time marching (oracle).

P:147-158: the nonlinear system max_a (A^a_i X - F^a_i) = 0 (eq. nonlinear_sys), row-wise
maximisation by linear search over a finite control set, then a linear solve at the fixed
policy.  For theta = 1 (derivation D1):
    (A^a U)_j - F^a_j = U_j - U^{n-1}_j - dt H^a_j(U),   H^a_j(U) = L_hat^a[U](x_j) + c^a_j U_j + f^a_j
so argmax_a of the row residual is argmin_a H^a_j (the inf of eq. 1.1).

Readings: lowest index on exact ties (iii/iv); initial policy = greedy at U^{n-1}
with boundary psi(t_n); stop when the policy is unchanged or R <= tol_pi, max_pi = 50.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .scheme import Geometry, lhat_rows, node_coefficients, source_term
from .system import assemble, solve

NEAR_TIE_REL = 1e-12


@dataclass
class SearchResult:
    policy: np.ndarray          # [N_I] argmin control (lowest index on exact ties)
    H: np.ndarray               # [N_I] min_a H^a_j
    F: np.ndarray               # [N_I] U^{n-1}_j + dt f^{a_j}_j
    R: np.ndarray               # [N_I] |U_j - U^{n-1}_j - dt min_a H^a_j|
    scale: np.ndarray           # [N_I] S_j = sum of |terms| of H at the argmin (rounding scale)
    second_gap: np.ndarray      # [N_I] H(second best) - H(best)  (inf if K == 1)
    ties: np.ndarray = field(default=None)  # [N_I] number of controls within 1e-12 S_j of the min


def hamiltonian(prob, idx, alpha, U_full, t, fields, k_scale=1.0, exact_psi=None):
    """H^a_j(U) = L_hat^a[U](x_j) + c^a_j U_j + f^a_j for one control per node (eq. Lhat),
    plus S_j = sum of |terms| (near-tie scale, reading iv).  exact_psi (z -> psi(z)): truncated
    endpoints take the Dirichlet value (Remark rhs)."""
    geo = Geometry.of(prob, k_scale)
    sig, b, c = node_coefficients(prob, idx, alpha, fields)
    x = geo.node_x(idx)
    Uj = U_full[idx]
    f = source_term(prob, t, alpha, fields)
    if exact_psi is None:
        cols, vals, _ = lhat_rows(geo, x, sig, b)
        diff = U_full[cols] - Uj[:, None]
        L = np.sum(vals * diff, axis=1)
        S = np.sum(vals * (np.abs(U_full[cols]) + np.abs(Uj)[:, None]), axis=1)
    else:
        cols, vals, rowsum, bsum = lhat_rows(geo, x, sig, b, exact_psi=exact_psi)
        L = np.sum(vals * U_full[cols], axis=1) + bsum - rowsum * Uj
        S = np.sum(vals * np.abs(U_full[cols]), axis=1) + np.abs(bsum) + rowsum * np.abs(Uj)
    H = L + c * Uj + f
    S = S + np.abs(c * Uj) + np.abs(f)
    return H, S, f


def control_search(prob, U_full, U_prev_full, t, dt, fields=None, idx=None, k_scale=1.0,
                   chunk=1 << 18, exact_psi=None):
    """Exhaustive linear search over the discrete control set (footnote P:156):
    for every interior j and every a in index order evaluate H^a_j(U) from its definition and
    keep the lowest-index argmin."""
    geo = Geometry.of(prob, k_scale)
    if idx is None:
        idx = geo.interior_idx()
    idx = np.asarray(idx, dtype=np.int64)
    outs = []
    for s in range(0, idx.size, chunk):
        sub = idx[s:s + chunk]
        fl = prob.fields(sub) if fields is None else {k: (v[..., s:s + chunk]) for k, v in fields.items()}
        m = sub.size
        best = np.full(m, np.inf)
        second = np.full(m, np.inf)
        arg = np.zeros(m, dtype=np.int64)
        Sbest = np.zeros(m)
        fbest = np.zeros(m)
        Hall = np.empty((prob.K, m))
        Sall = np.empty((prob.K, m))
        for a in range(prob.K):
            H, S, f = hamiltonian(prob, sub, np.full(m, a), U_full, t, fl, k_scale, exact_psi)
            Hall[a], Sall[a] = H, S
            better = H < best                      # strict: lowest index wins exact ties
            second = np.where(better, best, np.minimum(second, H))
            best = np.where(better, H, best)
            arg = np.where(better, a, arg)
            Sbest = np.where(better, S, Sbest)
            fbest = np.where(better, f, fbest)
        ties = np.sum(Hall - best[None, :] <= NEAR_TIE_REL * Sbest[None, :], axis=0)
        Uj, Upj = U_full[sub], U_prev_full[sub]
        outs.append(SearchResult(policy=arg, H=best, F=Upj + dt * fbest,
                                 R=np.abs(Uj - Upj - dt * best), scale=Sbest,
                                 second_gap=second - best, ties=ties))
    cat = lambda k: np.concatenate([getattr(o, k) for o in outs])  # noqa: E731
    return SearchResult(policy=cat("policy"), H=cat("H"), F=cat("F"), R=cat("R"),
                        scale=cat("scale"), second_gap=cat("second_gap"), ties=cat("ties"))


@dataclass
class StepStats:
    pi_iters: int = 0
    changed: list = field(default_factory=list)
    residuals: list = field(default_factory=list)
    solve_rres: list = field(default_factory=list)


def howard_step(prob, U_prev_full, t, dt, fields=None, tol_pi=None, max_pi=50, k_scale=1.0,
                policy0=None, solve_kw=None, theta=1.0, exact_psi=False):
    """One step t_{n-1} -> t_n = t of the theta-scheme (eq. FullScheme) by policy
    iteration.  The row residual of control a is (derivation D1 with theta)
        (A^a U - F^a)_j = U_j - U^{n-1}_j - dt H^a_j(V),   V = theta U + (1 - theta) U^{n-1},
    (L_hat and c are linear in their argument), so the policy improvement is the control search at V
    with f at t_{n-1} + theta dt.  theta = 0 (explicit Euler) needs no solve: U^n = U^{n-1} + dt
    min_a H^a(U^{n-1}) at every interior node, boundary psi(t_n).  exact_psi: the exact-psi boundary
    mode of Remark rhs: truncated endpoints take psi(z) (for V: theta psi(t_n, z) +
    (1 - theta) psi(t_{n-1}, z)), prob.psi_at.
    Returns (U^n on the full grid, policy on the full grid, StepStats)."""
    geo = Geometry.of(prob, k_scale)
    interior = geo.interior_idx()
    if fields is None:
        fields = prob.fields(interior)
    tol_pi = prob.tol_pi if tol_pi is None else tol_pi
    bidx = prob.boundary_idx()
    psi_full = np.zeros(prob.N)
    psi_full[bidx] = prob.psi(t, bidx)
    t_theta = t - dt + theta * dt
    pol_full = np.zeros(prob.N, dtype=np.int64)
    stats = StepStats()
    tp = t - dt
    ex_v = (lambda z: theta * prob.psi_at(t, z) + (1.0 - theta) * prob.psi_at(tp, z)) if exact_psi else None
    if theta == 0.0:                              # explicit Euler: one control search at U^{n-1}
        sr = control_search(prob, U_prev_full, U_prev_full, t_theta, dt, fields=fields, idx=interior,
                            k_scale=k_scale, exact_psi=ex_v)
        U = U_prev_full.copy()
        U[interior] = U_prev_full[interior] + dt * sr.H
        U[bidx] = psi_full[bidx]
        pol_full[interior] = sr.policy
        stats.pi_iters = 1
        return U, pol_full, stats
    U = U_prev_full.copy()
    U[bidx] = psi_full[bidx]                      # a1: Dirichlet rows are identities
    if policy0 is not None:
        pol_full[interior] = policy0
    have_policy = False
    for it in range(1, max_pi + 1):
        V = theta * U + (1.0 - theta) * U_prev_full
        sr = control_search(prob, V, U_prev_full, t_theta, dt, fields=fields, idx=interior, k_scale=k_scale,
                            exact_psi=ex_v)
        R = np.abs(U[interior] - U_prev_full[interior] - dt * sr.H)      # = sr.R when theta = 1
        changed = int(np.sum(sr.policy != pol_full[interior]))
        stats.changed.append(changed)
        stats.residuals.append(float(R.max(initial=0.0)))
        if have_policy and (changed == 0 or R.max(initial=0.0) <= tol_pi):
            break
        pol_full[interior] = sr.policy
        have_policy = True
        sysm = assemble(prob, pol_full, dt, t, U_prev_full, psi_full, fields=fields, k_scale=k_scale,
                        theta=theta, exact_psi=exact_psi)
        X, rres = solve(sysm, x0=U[interior], **(solve_kw or {}))
        stats.solve_rres.append(rres)
        U[interior] = X
        stats.pi_iters = it
    return U, pol_full, stats


def march(prob, n_steps=None, fields=None, k_scale=1.0, theta=1.0, **kw):
    """theta-scheme march U^0 = g, U^n = step(U^{n-1}) to T in n_steps uniform steps."""
    n_steps = n_steps or prob.n_steps
    dt = prob.T / n_steps
    idx = prob.all_idx()
    U = prob.g(idx).astype(np.float64)
    geo = Geometry.of(prob, k_scale)
    if fields is None:
        fields = prob.fields(geo.interior_idx())
    hist = []
    pol = None
    for s in range(1, n_steps + 1):
        U, pol, st = howard_step(prob, U, s * dt, dt, fields=fields, k_scale=k_scale, theta=theta, **kw)
        hist.append(st)
        if not np.all(np.isfinite(U)):
            break                                  # an unstable explicit march (CFL violated)
    return U, pol, hist


def cfl_rate(prob, fields=None, k_scale=1.0, policy=None):
    """max over interior nodes i (and controls a) of  sum_p (A^a_p + B^a_p)/(2 dx) - c^a_i, the rate in
    the positivity (CFL) condition of Proposition CFL (eq. CFL_trunc):
        (1 - theta) dt [ sum_p (A_p + B_p)/(2 dx) - c ] <= 1   for all a, i
    (the sum runs over the M = P + 1 pairs incl. the drift pair).  policy (full-grid control index):
    the rate of those controls only (the condition is sufficient; a march only applies the controls
    it selects).  Returns (rate, (node, control) of the max).  Truncated rows make it grow like
    dx^{-3/2} (one side oversteps) or dx^{-2} (both sides), Corollary CFL."""
    geo = Geometry.of(prob, k_scale)
    interior = geo.interior_idx()
    if fields is None:
        fields = prob.fields(interior)
    x = geo.node_x(interior)
    best, arg = -np.inf, (None, None)
    ctrls = [None] if policy is not None else range(prob.K)
    for a in ctrls:
        al = np.asarray(policy)[interior] if a is None else np.full(interior.size, a)
        sig, b, c = node_coefficients(prob, interior, al, fields)
        _, _, rowsum = lhat_rows(geo, x, sig, b)
        r = rowsum - c
        j = int(np.argmax(r))
        if r[j] > best:
            best, arg = float(r[j]), (int(interior[j]), int(al[j]))
    return best, arg
