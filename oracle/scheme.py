"""Scheme 2 LISL stencil with consistency-preserving boundary truncation (oracle).

Written step by step from PAPER.md in the paper's notation:
  * steps y^{a,+-}_p = +- sqrt(dx) sigma^a_p (p <= P), y^{a,+-}_{P+1} = dx b^a, M = P+1
  * truncation  y_hat = mu y,  mu = largest value in (0,1] keeping x + mu y in closed Omega
  * weights A_p = 2/(mu+^2 + mu+ mu-), B_p = 2/(mu-^2 + mu- mu+); drift A = B = 1/mu
  * multilinear interpolation I_dx, w_j >= 0, sum w = 1, w_i(x_j) = delta_ij
  * l_hat_{j,i} = sum_p [A_p w_i(x_j + y_hat+_p) + B_p w_i(x_j + y_hat-_p)] / (2 dx)
  * L_hat[phi](x_j) = sum_i l_hat_{j,i} (phi_i - phi_j)                                       (eq. Lhat)

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import itertools
import math

import numpy as np


class Geometry:
    """Uniform Cartesian grid on [lo, hi]^d with n nodes per dimension."""

    def __init__(self, d: int, n: int, lo: float, hi: float, k_scale: float = 1.0):
        self.d, self.n, self.lo, self.hi = d, n, float(lo), float(hi)
        self.dx = (self.hi - self.lo) / (n - 1)
        self.k = k_scale * math.sqrt(self.dx)            # k = sqrt(dx)

    @classmethod
    def of(cls, prob, k_scale: float = 1.0):
        return cls(prob.d, prob.n, prob.lo, prob.hi, k_scale)

    def node_x(self, idx):
        """x_j = lo + i*dx per dimension, i1 fastest."""
        idx = np.asarray(idx, dtype=np.int64)
        out = np.empty((idx.size, self.d))
        r = idx.copy()
        for i in range(self.d):
            out[:, i] = self.lo + (r % self.n).astype(np.float64) * self.dx
            r //= self.n
        return out

    def multi(self, idx):
        idx = np.asarray(idx, dtype=np.int64)
        out = []
        r = idx.copy()
        for _ in range(self.d):
            out.append(r % self.n)
            r //= self.n
        return out

    def flat(self, mi):
        f = np.zeros_like(mi[0])
        for i in reversed(range(self.d)):
            f = f * self.n + mi[i]
        return f

    def interior_idx(self):
        ax = np.arange(1, self.n - 1)
        grids = np.meshgrid(*([ax] * self.d), indexing="ij")
        # lexicographic with x1 fastest: iterate the last dimension slowest
        mi = [g.transpose(*reversed(range(self.d))).ravel() for g in grids]
        return self.flat(mi)

    def is_boundary(self, idx):
        mi = self.multi(idx)
        b = np.zeros(np.asarray(idx).shape, dtype=bool)
        for i in mi:
            b |= (i == 0) | (i == self.n - 1)
        return b


# ------------------------------------------------------------------ truncation
def truncation_mu(geo: Geometry, x: np.ndarray, y: np.ndarray):
    """mu = min{ mu >= 0 : x + mu y in dOmega } capped at 1, i.e. the largest mu in (0,1] such that
    x + [0, mu] y stays in closed Omega (equal on boxes, reading vi).
    Returns (mu [m], binding face per dimension as a bool mask [m, d])."""
    m, d = x.shape
    face_t = np.full((m, d), np.inf)
    pos, neg = y > 0, y < 0
    face_t[pos] = (geo.hi - x[pos]) / y[pos]
    face_t[neg] = (geo.lo - x[neg]) / y[neg]
    mu = np.minimum(1.0, face_t.min(axis=1))
    binding = (face_t <= mu[:, None]) & (mu[:, None] < 1.0)
    return mu, binding


def truncated_endpoint(geo: Geometry, x, y, mu, binding):
    """x + y_hat with y_hat = mu y; the binding coordinate is put exactly on the
    face x_i = lo or hi (reading: face snapping), all coordinates kept in [lo, hi]."""
    z = x + mu[:, None] * y
    face = np.where(y > 0, geo.hi, geo.lo)
    z = np.where(binding, face, z)
    return np.clip(z, geo.lo, geo.hi)


def truncation_weights(mu_plus, mu_minus):
    """Scheme 2 diffusion weights, eq. (eqn_Ap), P:298-302:
    A = 2/(mu+^2 + mu+ mu-),  B = 2/(mu-^2 + mu- mu+)."""
    A = 2.0 / (mu_plus ** 2 + mu_plus * mu_minus)
    B = 2.0 / (mu_minus ** 2 + mu_minus * mu_plus)
    return A, B


def drift_weights(mu):
    """Scheme 2 drift weights, eq. (eqn_APp1): A = B = 1/mu."""
    return 1.0 / mu, 1.0 / mu


# ------------------------------------------------------------------ interpolation
def interp_weights(geo: Geometry, z: np.ndarray):
    """Multilinear interpolation I_dx: the 2^d vertices of the cell containing z with
    tensor-product weights.  Cell index clamped to [0, n-2] so z on the upper face uses the
    last cell with local coordinate 1 (reading vii).  Returns (idx [m, 2^d], w [m, 2^d])."""
    m, d = z.shape
    t = (z - geo.lo) / geo.dx
    c = np.clip(np.floor(t), 0, geo.n - 2).astype(np.int64)
    s = t - c
    cols, ws = [], []
    for bits in itertools.product((0, 1), repeat=d):
        mi = [c[:, i] + bits[i] for i in range(d)]
        w = np.ones(m)
        for i in range(d):
            w = w * (s[:, i] if bits[i] else 1.0 - s[:, i])
        cols.append(geo.flat(mi))
        ws.append(w)
    return np.stack(cols, axis=1), np.stack(ws, axis=1)


# ------------------------------------------------------------------ coefficients
def node_coefficients(prob, idx, alpha, fields=None):
    """sigma^a_p(x_j), b^a(x_j), c^a(x_j) from the affine-separable coefficient model of synth/
    (problem data).  alpha: control index per node."""
    if fields is None:
        fields = prob.fields(np.asarray(idx, dtype=np.int64))
    alpha = np.asarray(alpha, dtype=np.int64)
    sig = prob.sigma_dir[alpha].copy()                    # [m, P, d]
    if "sigma_scale" in fields:
        sig = sig * np.asarray(fields["sigma_scale"]).T[:, :, None]
    if "sigma_node" in fields:
        sig = sig + np.asarray(fields["sigma_node"]).transpose(2, 0, 1)
    b = prob.b_dir[alpha].copy()                           # [m, d]
    if "b_scale" in fields:
        b = b * np.asarray(fields["b_scale"])[:, None]
    if "b_node" in fields:
        b = b + np.asarray(fields["b_node"]).T
    c = prob.c_ctrl[alpha].copy()
    if "c_node" in fields:
        c = c + np.asarray(fields["c_node"])
    return sig, b, c


def source_term(prob, t, alpha, fields):
    """f^a(t, x_j) = f_ctrl[a] + sum_q f_basis[a,q] f_feat[q](x_j) (problem data)."""
    fb, fc = prob.f_tables(t)
    alpha = np.asarray(alpha, dtype=np.int64)
    ff = np.asarray(fields["f_feat"])                      # [Q, m]
    return fc[alpha] + np.einsum("mq,qm->m", fb[alpha], ff)


# ------------------------------------------------------------------ the truncated LISL row
def stencil_pairs(geo: Geometry, x, sig, b, with_masks=False):
    """The M = P+1 Scheme-2 pairs at nodes x, each truncated.
    Returns a list of pairs (z_plus, A, z_minus, B) with A, B the finite-difference weights of
    eq. (TruncScheme); with_masks: (z_plus, A, z_minus, B, trunc_plus, trunc_minus), the
    masks of the endpoints whose ray was truncated (mu < 1: they lie on dOmega)."""
    m, d = x.shape
    P = sig.shape[1]
    pairs = []
    for p in range(P):
        y_plus = geo.k * sig[:, p, :]                      # +sqrt(dx) sigma_p
        y_minus = -geo.k * sig[:, p, :]
        mu_p, bind_p = truncation_mu(geo, x, y_plus)
        mu_m, bind_m = truncation_mu(geo, x, y_minus)
        A, B = truncation_weights(mu_p, mu_m)
        pp = (truncated_endpoint(geo, x, y_plus, mu_p, bind_p), A,
              truncated_endpoint(geo, x, y_minus, mu_m, bind_m), B)
        pairs.append(pp + (mu_p < 1.0, mu_m < 1.0) if with_masks else pp)
    # drift pair p = P+1: y+ = y- = dx b (both signs equal), A = B = 1/mu
    y_d = geo.dx * b
    mu_d, bind_d = truncation_mu(geo, x, y_d)
    A, B = drift_weights(mu_d)
    z_d = truncated_endpoint(geo, x, y_d, mu_d, bind_d)
    pairs.append((z_d, A, z_d, B) + ((mu_d < 1.0, mu_d < 1.0) if with_masks else ()))
    return pairs


def lhat_rows(geo: Geometry, x, sig, b, exact_psi=None):
    """Rows of l_hat for nodes x:
        l_hat_{j,i} = sum_p [A_p w_i(x_j + y_hat+_p) + B_p w_i(x_j + y_hat-_p)] / (2 dx)
    Returns (cols [m, E], vals [m, E], rowsum [m]) with duplicates not merged, and
    rowsum = sum_p (A_p + B_p)/(2 dx).
    exact_psi (a function z [m, d] -> psi(z)): the exact-psi boundary mode of Remark rhs
    (NEXT-2): a truncated endpoint (on dOmega) takes the Dirichlet value psi(z) instead of
    the interpolation of the nodal boundary values; its interpolation entries are dropped from
    (cols, vals) and returned as a fourth output, the row's sum_e w_e psi(z_e) [m]."""
    cols, vals = [], []
    rowsum = np.zeros(x.shape[0])
    bsum = np.zeros(x.shape[0])
    for (zp, A, zm, B, tp, tm) in stencil_pairs(geo, x, sig, b, with_masks=True):
        for z, W, tr in ((zp, A, tp), (zm, B, tm)):
            iz, wz = interp_weights(geo, z)
            w = W[:, None] * wz / (2.0 * geo.dx)
            if exact_psi is not None and tr.any():
                w = np.where(tr[:, None], 0.0, w)
                bsum[tr] += W[tr] / (2.0 * geo.dx) * exact_psi(z[tr])
            cols.append(iz)
            vals.append(w)
        rowsum += (A + B) / (2.0 * geo.dx)
    out = (np.concatenate(cols, axis=1), np.concatenate(vals, axis=1), rowsum)
    return out + (bsum,) if exact_psi is not None else out


def lhat_apply(geo: Geometry, idx, sig, b, phi_full, exact_psi=None):
    """L_hat[phi](x_j) = sum_i l_hat_{j,i} (phi_i - phi_j)  (eq. Lhat), with phi given
    on the full grid (boundary nodes hold their values: interpolate-at-boundary mode), or
    with exact_psi the truncated endpoints taking psi(z) (Remark rhs)."""
    x = geo.node_x(idx)
    phi_j = phi_full[np.asarray(idx)]
    if exact_psi is None:
        cols, vals, _ = lhat_rows(geo, x, sig, b)
        return np.sum(vals * (phi_full[cols] - phi_j[:, None]), axis=1)
    cols, vals, rowsum, bsum = lhat_rows(geo, x, sig, b, exact_psi)
    # sum over non-truncated entries of w (phi_i - phi_j) + sum over truncated endpoints w (psi - phi_j)
    return np.sum(vals * phi_full[cols], axis=1) + bsum - rowsum * phi_j


def apply_operator(prob, policy_full, x_full, dt, idx=None, fields=None, k_scale=1.0, exact_psi=None):
    """Matrix-free (A^pi x)_j for interior rows j (theta = 1):
        (A x)_j = x_j - dt [ L_hat[x](x_j) + c_j x_j ]
    Boundary entries of x are used as given.  Returns values at idx (default: all interior)."""
    geo = Geometry.of(prob, k_scale)
    if idx is None:
        idx = geo.interior_idx()
    idx = np.asarray(idx, dtype=np.int64)
    sig, b, c = node_coefficients(prob, idx, np.asarray(policy_full)[idx], fields)
    L = lhat_apply(geo, idx, sig, b, x_full, exact_psi)
    return x_full[idx] - dt * (L + c * x_full[idx])
