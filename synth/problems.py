"""Seeded synthetic HJB problems: the BASELINE.json configs, the paper's Problems A/B and
the LISL-Laplacian model problem, expressed in the affine-separable coefficient model that
the C-ABI (include/hjb.h) and the oracle both consume.

INPUT GENERATION ONLY. Nothing here evaluates the numerical method (no stencil, no
interpolation, no truncation, no solve). It evaluates the *problem data* of the PDE
u_t - inf_a { L^a u + c^a u + f^a } = 0: the coefficients at grid nodes,
the manufactured source f, the initial data g and the Dirichlet data psi.

Coefficient model (per node x, control a; PAPER.md:37-41 with sigma in R^{d x P}):
    sigma^a_p(x) = sigma_scale[p](x) * sigma_dir[a,p,:] + sigma_node[p,:](x)
    b^a(x)       = b_scale(x) * b_dir[a,:] + b_node[:](x)
    c^a(x)       = c_node(x) + c_ctrl[a]
    f^a(t, x)    = f_ctrl(t)[a] + sum_q f_basis(t)[a,q] * f_feat[q](x)
Absent node fields default to 1 (scales) or 0 (offsets).

Grid: n nodes per dimension on [lo, hi]^d, h = (hi - lo)/(n - 1), x_i = lo + i*h,
flat index lexicographic with x1 fastest.

Every field evaluator takes flat node indices and an array namespace `xp` (numpy or torch),
so the same definitions build small CPU problems (oracle) and 2.7e8-node device arrays (GPU).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import noise

NOISE_SEED = 42        # SURVEY §8c-xv / S:654
NOISE_AMP = 0.05       # BASELINE.json configs[2]: "seeded uniform noise of amplitude 0.05"


def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


def _xp_of(a):
    if _is_torch(a):
        import torch
        return torch
    return np


@dataclass
class Problem:
    name: str
    d: int
    P: int
    K: int
    Q: int
    n: int
    lo: float
    hi: float
    T: float
    n_steps: int
    sigma_dir: np.ndarray                 # [K, P, d]
    b_dir: np.ndarray                     # [K, d]
    c_ctrl: np.ndarray                    # [K]
    _fields: Callable                     # (idx, xp) -> dict of node fields
    _f_tables: Callable                   # t -> (f_basis [K,Q], f_ctrl [K])
    _u_exact: Optional[Callable] = None   # (t, idx, xp) -> values
    _u_at: Optional[Callable] = None      # (t, [x_1..x_d] coordinate arrays, xp) -> values
    _g: Optional[Callable] = None         # (idx, xp) -> values (default u_exact(0))
    _psi: Optional[Callable] = None       # (t, idx, xp) -> values (default u_exact(t))
    tol_pi: float = 1e-10
    krylov_rtol: float = 1e-12
    meta: dict = field(default_factory=dict)

    # ---------------------------------------------------------------- geometry
    @property
    def h(self) -> float:
        return (self.hi - self.lo) / (self.n - 1)

    @property
    def N(self) -> int:
        return self.n ** self.d

    @property
    def N_interior(self) -> int:
        return (self.n - 2) ** self.d

    @property
    def dt(self) -> float:
        return self.T / self.n_steps

    def all_idx(self, xp=np, device=None):
        if xp is np:
            return np.arange(self.N, dtype=np.int64)
        return xp.arange(self.N, dtype=xp.int64, device=device)

    def multi_index(self, idx):
        """Per-dimension node indices (i1 fastest)."""
        n = self.n
        out = []
        r = idx
        for _ in range(self.d):
            out.append(r % n)
            r = r // n
        return out

    def coords(self, idx):
        xp = _xp_of(idx)
        h = self.h
        return [self.lo + (i.to(xp.float64) if xp is not np else i.astype(np.float64)) * h
                for i in self.multi_index(idx)]

    def is_boundary(self, idx):
        mi = self.multi_index(idx)
        b = (mi[0] == 0) | (mi[0] == self.n - 1)
        for i in mi[1:]:
            b = b | (i == 0) | (i == self.n - 1)
        return b

    def boundary_idx(self):
        """Boundary node flat indices in lexicographic order (the packed psi layout of hjb.h)."""
        n = self.n
        full = np.arange(n, dtype=np.int64)
        ring = np.concatenate([full, (np.arange(1, n - 1, dtype=np.int64)[:, None] * n
                                      + np.array([0, n - 1])).ravel(), (n - 1) * n + full])
        if self.d == 2:
            return ring
        plane = np.arange(n * n, dtype=np.int64)
        mid = (np.arange(1, n - 1, dtype=np.int64)[:, None] * n * n + ring[None, :]).ravel()
        return np.concatenate([plane, mid, (n - 1) * n * n + plane])

    # ---------------------------------------------------------------- data
    def fields(self, idx):
        return self._fields(idx, _xp_of(idx))

    def f_tables(self, t: float):
        fb, fc = self._f_tables(t)
        return np.ascontiguousarray(fb, dtype=np.float64), np.ascontiguousarray(fc, dtype=np.float64)

    def u_exact(self, t, idx):
        if self._u_exact is None:
            return None
        return self._u_exact(t, idx, _xp_of(idx))

    def psi_at(self, t, X):
        """Dirichlet data psi(t, z) at arbitrary boundary points z (X: [m, d] coordinates), for the
        exact-psi boundary mode (PAPER.md Remark rhs); psi = u_exact on dOmega here."""
        X = np.asarray(X, dtype=np.float64)
        return self._u_at(t, [X[:, i] for i in range(self.d)], np)

    def g(self, idx):
        if self._g is not None:
            return self._g(idx, _xp_of(idx))
        return self._u_exact(0.0, idx, _xp_of(idx))

    def psi(self, t, idx):
        if self._psi is not None:
            return self._psi(t, idx, _xp_of(idx))
        return self._u_exact(t, idx, _xp_of(idx))

    def halo_rows(self, k_scale: float = 1.0) -> int:
        """Halo rows a slab needs: floor(max |offset| along the slowest axis, in cells) + 1 (an
        endpoint at i + o reads rows floor(i+o) and floor(i+o)+1), from the problem data (the
        library re-checks it on the device in hjb_set_coeffs)."""
        f = self.fields(self.all_idx()) if self.N <= (1 << 22) else self.fields(
            np.arange(0, self.N, max(1, self.N // (1 << 20)), dtype=np.int64))
        ax = self.d - 1
        sc = np.abs(np.asarray(f["sigma_scale"])).max(axis=1) if "sigma_scale" in f else np.ones(self.P)
        sn = np.abs(np.asarray(f["sigma_node"])[:, ax]).max(axis=1) if "sigma_node" in f else np.zeros(self.P)
        bs = np.abs(np.asarray(f["b_scale"])).max() if "b_scale" in f else 1.0
        bn = np.abs(np.asarray(f["b_node"])[ax]).max() if "b_node" in f else 0.0
        kh = k_scale * math.sqrt(self.h) / self.h
        reach = max(kh * (sc[p] * np.abs(self.sigma_dir[:, p, ax]).max() + sn[p]) for p in range(self.P))
        reach = max(reach, bs * np.abs(self.b_dir[:, ax]).max() + bn)
        return int(math.floor(reach * (1 + 1e-12))) + 1

    def control_tables(self):
        return (np.ascontiguousarray(self.sigma_dir, dtype=np.float64),
                np.ascontiguousarray(self.b_dir, dtype=np.float64),
                np.ascontiguousarray(self.c_ctrl, dtype=np.float64))


# =================================================================== noise fields
def eta(p: Problem, field_id: int, idx):
    """Smoothed noise eta in [-1,1]: average of i.i.d. U[-1,1] over the node and its in-domain
    axis neighbours (5-point filter in 2D, 7-point in 3D) -- SURVEY §8c-xv reading."""
    xp = _xp_of(idx)
    mi = p.multi_index(idx)
    stride = [p.n ** k for k in range(p.d)]

    def draw(j):
        if xp is np:
            return noise.uniform_pm1_np(NOISE_SEED, field_id, j)
        return noise.uniform_pm1_torch(NOISE_SEED, field_id, j)

    acc = draw(idx)
    cnt = xp.ones_like(acc)
    for k in range(p.d):
        for sgn in (-1, 1):
            nb = mi[k] + sgn
            ok = (nb >= 0) & (nb <= p.n - 1)
            j = xp.where(ok, idx + sgn * stride[k], idx)
            v = draw(j)
            acc = acc + xp.where(ok, v, xp.zeros_like(v))
            cnt = cnt + (ok.astype(np.float64) if xp is np else ok.to(xp.float64))
    return acc / cnt


# =================================================================== 2D rotated model
def _rot2(theta):
    c, s = math.cos(theta), math.sin(theta)
    return np.array([[c, -s], [s, c]])


def rotated_2d(name: str, n: int, K: int, s: tuple, beta: float, n_steps: int,
               noisy: bool, T: float = 1.0, c: float = -0.1) -> Problem:
    """BASELINE.json configs 0,1,2,4: sigma^th = R(th) diag(s1,s2), b = beta (cos th, sin th),
    c = -0.1, u* = (1+t) sin(pi x1/2) cos(pi x2/2),
    f^th = u*_t - L^th u* - c u* + (th - th*(x))^2, th*(x) = pi|x1| mod pi  on [-1,1]^2.
    With noise (cfg2/4): s_p(x) = s_p (1 + 0.05 eta_p(x)), beta(x) = beta (1 + 0.05 eta_3(x))."""
    d, P = 2, 2
    thetas = np.array([j * math.pi / K for j in range(K)])
    sigma_dir = np.zeros((K, P, d))
    b_dir = np.zeros((K, d))
    for a, th in enumerate(thetas):
        R = _rot2(th)
        for q in range(P):
            sigma_dir[a, q, :] = s[q] * R[:, q]
        b_dir[a, :] = beta * np.array([math.cos(th), math.sin(th)])
    c_ctrl = np.full(K, c)
    hp = math.pi / 2

    def phi_parts(x1, x2, xp):
        S1, C1 = xp.sin(hp * x1), xp.cos(hp * x1)
        S2, C2 = xp.sin(hp * x2), xp.cos(hp * x2)
        return S1, C1, S2, C2

    def fields(idx, xp):
        x1, x2 = p.coords(idx)
        S1, C1, S2, C2 = phi_parts(x1, x2, xp)
        phi = S1 * C2
        H11 = -(hp ** 2) * phi
        H22 = -(hp ** 2) * phi
        H12 = -(hp ** 2) * C1 * S2
        G1 = hp * C1 * C2
        G2 = -hp * S1 * S2
        out = {}
        if noisy:
            e1, e2, e3 = eta(p, 0, idx), eta(p, 1, idx), eta(p, 2, idx)
            sc1 = 1.0 + NOISE_AMP * e1
            sc2 = 1.0 + NOISE_AMP * e2
            bsc = 1.0 + NOISE_AMP * e3
            out["sigma_scale"] = xp.stack([sc1, sc2])
            out["b_scale"] = bsc
            s1sq, s2sq = (s[0] * sc1) ** 2, (s[1] * sc2) ** 2
            bet = beta * bsc
        else:
            s1sq = xp.full_like(phi, s[0] ** 2)
            s2sq = xp.full_like(phi, s[1] ** 2)
            bet = xp.full_like(phi, beta)
        thstar = xp.remainder(math.pi * xp.abs(x1), math.pi)
        # tr(a^th H) = 1/2 sum_p s_p^2 (R e_p)^T H (R e_p)
        #  = 1/4 (s1^2+s2^2)(H11+H22) + 1/4 (s1^2-s2^2)(H11-H22) cos2th + 1/2 (s1^2-s2^2) H12 sin2th
        feats = [
            phi,                                      # basis 1 - c(1+t)   (u*_t - c u*)
            0.25 * (s1sq + s2sq) * (H11 + H22),        # basis -(1+t)
            0.25 * (s1sq - s2sq) * (H11 - H22),        # basis -(1+t) cos 2th
            0.5 * (s1sq - s2sq) * H12,                 # basis -(1+t) sin 2th
            bet * G1,                                  # basis -(1+t) cos th
            bet * G2,                                  # basis -(1+t) sin th
            thstar,                                    # basis -2 th
            thstar * thstar,                           # basis 1
        ]
        out["f_feat"] = xp.stack(feats)
        return out

    def f_tables(t):
        fb = np.zeros((K, 8))
        for a, th in enumerate(thetas):
            fb[a] = [1.0 - c * (1.0 + t), -(1.0 + t), -(1.0 + t) * math.cos(2 * th),
                     -(1.0 + t) * math.sin(2 * th), -(1.0 + t) * math.cos(th),
                     -(1.0 + t) * math.sin(th), -2.0 * th, 1.0]
        return fb, thetas ** 2

    def u_at(t, x, xp):
        return (1.0 + t) * xp.sin(hp * x[0]) * xp.cos(hp * x[1])

    def u_exact(t, idx, xp):
        return u_at(t, p.coords(idx), xp)

    p = Problem(name=name, d=d, P=P, K=K, Q=8, n=n, lo=-1.0, hi=1.0, T=T, n_steps=n_steps,
                sigma_dir=sigma_dir, b_dir=b_dir, c_ctrl=c_ctrl, _fields=fields,
                _f_tables=f_tables, _u_exact=u_exact, _u_at=u_at,
                meta=dict(thetas=thetas, s=s, beta=beta, noisy=noisy, c=c))
    return p


# =================================================================== 3D rotated model
def _rot_zy(ph, th):
    cz, sz = math.cos(ph), math.sin(ph)
    cy, sy = math.cos(th), math.sin(th)
    Rz = np.array([[cz, -sz, 0], [sz, cz, 0], [0, 0, 1.0]])
    Ry = np.array([[cy, 0, sy], [0, 1.0, 0], [-sy, 0, cy]])
    return Rz @ Ry


def rotated_3d(name: str, n: int, n_phi: int = 12, n_vt: int = 8, s=(1.0, 0.4, 0.1),
               beta: float = 0.1, n_steps: int = 16, T: float = 1.0, c: float = -0.1) -> Problem:
    """BASELINE.json configs[3] with SURVEY §8c-xiv reading: R = R_z(phi) R_y(vt),
    phi_a = a pi/12, vt_b = b pi/8, alpha = 8a + b; sigma_p = s_p R e_p; b = 0.1 R e1;
    u* = (1+t) prod cos(pi x_i / 2); penalty (phi-phi*)^2 + (vt-vt*)^2,
    phi* = pi|x1| mod pi, vt* = pi|x2| mod pi."""
    d, P = 3, 3
    K = n_phi * n_vt
    sigma_dir = np.zeros((K, P, d))
    b_dir = np.zeros((K, d))
    angles = []
    for a in range(n_phi):
        for b in range(n_vt):
            ph, vt = a * math.pi / n_phi, b * math.pi / n_vt
            R = _rot_zy(ph, vt)
            k = n_vt * a + b
            angles.append((ph, vt))
            for q in range(P):
                sigma_dir[k, q, :] = s[q] * R[:, q]
            b_dir[k, :] = beta * R[:, 0]
    c_ctrl = np.full(K, c)
    hp = math.pi / 2
    pairs = [(0, 0), (1, 1), (2, 2), (0, 1), (0, 2), (1, 2)]

    def fields(idx, xp):
        x = p.coords(idx)
        Cs = [xp.cos(hp * xi) for xi in x]
        Ss = [xp.sin(hp * xi) for xi in x]
        phi = Cs[0] * Cs[1] * Cs[2]
        H = {}
        for (i, j) in pairs:
            if i == j:
                H[(i, j)] = -(hp ** 2) * phi
            else:
                k = 3 - i - j
                H[(i, j)] = (hp ** 2) * Ss[i] * Ss[j] * Cs[k]
        G = []
        for i in range(3):
            o = [Cs[j] for j in range(3) if j != i]
            G.append(-hp * Ss[i] * o[0] * o[1])
        phstar = xp.remainder(math.pi * xp.abs(x[0]), math.pi)
        vtstar = xp.remainder(math.pi * xp.abs(x[1]), math.pi)
        feats = [phi] + [H[pq] for pq in pairs] + G + [phstar, vtstar, phstar ** 2 + vtstar ** 2]
        return {"f_feat": xp.stack(feats)}

    def f_tables(t):
        fb = np.zeros((K, 13))
        fc = np.zeros(K)
        for k, (ph, vt) in enumerate(angles):
            sd = sigma_dir[k]                      # [P, d] rows are sigma_p
            row = [1.0 - c * (1.0 + t)]
            for (i, j) in pairs:
                a_ij = 0.5 * sum(sd[q, i] * sd[q, j] for q in range(P))
                row.append(-(1.0 + t) * a_ij * (1.0 if i == j else 2.0))
            for i in range(3):
                row.append(-(1.0 + t) * b_dir[k, i])
            row += [-2.0 * ph, -2.0 * vt, 1.0]
            fb[k] = row
            fc[k] = ph * ph + vt * vt
        return fb, fc

    def u_at(t, x, xp):
        return (1.0 + t) * xp.cos(hp * x[0]) * xp.cos(hp * x[1]) * xp.cos(hp * x[2])

    def u_exact(t, idx, xp):
        return u_at(t, p.coords(idx), xp)

    p = Problem(name=name, d=d, P=P, K=K, Q=13, n=n, lo=-1.0, hi=1.0, T=T, n_steps=n_steps,
                sigma_dir=sigma_dir, b_dir=b_dir, c_ctrl=c_ctrl, _fields=fields,
                _f_tables=f_tables, _u_exact=u_exact, _u_at=u_at,
                meta=dict(angles=angles, s=s, beta=beta, c=c))
    return p


# =================================================================== BASELINE.json configs
def bj_config(i: int, n: Optional[int] = None, K: Optional[int] = None,
              n_steps: Optional[int] = None) -> Problem:
    """BASELINE.json configs[i]; n/K/n_steps override for reduced-size parity runs."""
    if i == 0:
        return rotated_2d("cfg0", n or 33, K or 16, (1.0, 0.3), 0.2, n_steps or 8, noisy=False)
    if i == 1:
        return rotated_2d("cfg1", n or 257, K or 32, (1.0, 0.1), 0.2, n_steps or 32, noisy=False)
    if i == 2:
        return rotated_2d("cfg2", n or 2049, K or 64, (1.5, 0.05), 0.2, n_steps or 16, noisy=True)
    if i == 3:
        return rotated_3d("cfg3", n or 129, n_steps=n_steps or 16)
    if i == 4:
        return rotated_2d("cfg4", n or 16385, K or 32, (1.5, 0.05), 0.2, n_steps or 8, noisy=True)
    raise ValueError(i)


# =================================================================== paper problems
def problem_A(nx: int, n_alpha: int = 40, T: float = 0.5, n_steps: int = 1, shift: float = 0.0) -> Problem:
    """PAPER.md:465-471 (Problem A): u = (3/2 - t) sin x1 sin x2 on [-pi,pi]^2, b = alpha,
    sigma = sqrt2 (sin(x1+x2), cos(x1+x2)), c = 0, unit-circle controls
    alpha_i = (cos 2 pi i/N, sin 2 pi i/N).  shift = 7 pi/8: the shifted domain
    [-pi/8, 15 pi/8]^2 of Remark two-over, psi = u on its boundary (not zero)."""
    K = n_alpha
    d, P = 2, 1
    sigma_dir = np.zeros((K, P, d))
    b_dir = np.array([[math.cos(2 * math.pi * i / K), math.sin(2 * math.pi * i / K)] for i in range(K)])
    r2 = math.sqrt(2.0)

    def fields(idx, xp):
        x1, x2 = p.coords(idx)
        s12, c12 = xp.sin(x1 + x2), xp.cos(x1 + x2)
        sn = xp.stack([xp.stack([r2 * s12, r2 * c12])])          # [P=1, d, m]
        ss = xp.sin(x1) * xp.sin(x2)
        br = xp.sqrt(xp.cos(x1) ** 2 * xp.sin(x2) ** 2 + xp.sin(x1) ** 2 * xp.cos(x2) ** 2) \
            - 2.0 * s12 * c12 * xp.cos(x1) * xp.cos(x2)
        return {"sigma_node": sn, "f_feat": xp.stack([ss, br])}

    def f_tables(t):
        fb = np.tile(np.array([0.5 - t, 1.5 - t]), (K, 1))
        return fb, np.zeros(K)

    def u_at(t, x, xp):
        return (1.5 - t) * xp.sin(x[0]) * xp.sin(x[1])

    def u_exact(t, idx, xp):
        return u_at(t, p.coords(idx), xp)

    p = Problem(name=f"problemA_{nx}" + (f"_shift{shift:g}" if shift else ""), d=d, P=P, K=K, Q=2, n=nx,
                lo=-math.pi + shift, hi=math.pi + shift, T=T,
                n_steps=n_steps, sigma_dir=sigma_dir, b_dir=b_dir, c_ctrl=np.zeros(K),
                _fields=fields, _f_tables=f_tables, _u_exact=u_exact, _u_at=u_at)
    return p


def problem_B(nx: int, n_alpha: int = 40, T: float = 0.5, n_steps: int = 1) -> Problem:
    """PAPER.md:473-479 (Problem B): u = (2 - t) sin x1 sin x2, sigma = sqrt2 alpha, b = c = 0,
    f = (1-t) sin x1 sin x2 - 2 a1 a2 (2-t) cos x1 cos x2."""
    K = n_alpha
    d, P = 2, 1
    al = np.array([[math.cos(2 * math.pi * i / K), math.sin(2 * math.pi * i / K)] for i in range(K)])
    sigma_dir = (math.sqrt(2.0) * al)[:, None, :]
    b_dir = np.zeros((K, d))

    def fields(idx, xp):
        x1, x2 = p.coords(idx)
        return {"f_feat": xp.stack([xp.sin(x1) * xp.sin(x2), xp.cos(x1) * xp.cos(x2)])}

    def f_tables(t):
        fb = np.stack([np.full(K, 1.0 - t), -2.0 * al[:, 0] * al[:, 1] * (2.0 - t)], axis=1)
        return fb, np.zeros(K)

    def u_at(t, x, xp):
        return (2.0 - t) * xp.sin(x[0]) * xp.sin(x[1])

    def u_exact(t, idx, xp):
        return u_at(t, p.coords(idx), xp)

    p = Problem(name=f"problemB_{nx}", d=d, P=P, K=K, Q=2, n=nx, lo=-math.pi, hi=math.pi, T=T,
                n_steps=n_steps, sigma_dir=sigma_dir, b_dir=b_dir, c_ctrl=np.zeros(K),
                _fields=fields, _f_tables=f_tables, _u_exact=u_exact, _u_at=u_at)
    return p


def lisl_laplacian(sigma: float, ell: int, d: int = 2, T: float = 1e6) -> Problem:
    """PAPER.md:932-937 model: LISL discretisation of -1/2 div(sigma sigma^T grad) with
    sigma = sigma*I on [0,1]^d, homogeneous Dirichlet, one control, no drift, c = f = 0.
    Used through the implicit system I - dt L with a very large dt (dt -> infinity
    approaches the pure LISL Laplacian)."""
    K, P = 1, d
    sigma_dir = (sigma * np.eye(d))[None, :, :]
    n = 2 ** ell + 1

    def fields(idx, xp):
        return {"f_feat": xp.stack([xp.zeros_like(p.coords(idx)[0])])}

    def f_tables(t):
        return np.zeros((1, 1)), np.zeros(1)

    def zero(t, idx, xp):
        return xp.zeros_like(p.coords(idx)[0])

    p = Problem(name=f"lisl_lap_{sigma:g}_{ell}", d=d, P=P, K=K, Q=1, n=n, lo=0.0, hi=1.0, T=T,
                n_steps=1, sigma_dir=sigma_dir, b_dir=np.zeros((1, d)), c_ctrl=np.zeros(1),
                _fields=fields, _f_tables=f_tables, _u_exact=None,
                _g=lambda idx, xp: zero(0, idx, xp), _psi=zero,
                _u_at=lambda t, x, xp: xp.zeros_like(x[0]))
    return p


def random_vector(p: Problem, seed: int = 43, idx=None):
    """Seeded apply-test vector x ~ U[-1,1] over the full grid (seed 43)."""
    if idx is None:
        idx = p.all_idx()
    if _is_torch(idx):
        return noise.uniform_pm1_torch(seed, 0, idx)
    return noise.uniform_pm1_np(seed, 0, idx)


def face_samples(p: Problem, t: float, refine: int):
    """psi(t, .) sampled on every face of dOmega at spacing h / refine (input data of the exact-psi
    boundary mode, include/hjb.h hjb_set_boundary_samples): face f = 2 d + side (side 0: x_d = lo,
    1: x_d = hi); along-face axes in increasing order, the first fastest; M = refine (n - 1) + 1 samples
    per axis.  Returns a float64 array [2 d][M^(d-1)]."""
    M = refine * (p.n - 1) + 1
    s = np.linspace(p.lo, p.hi, M)
    out = []
    for d in range(p.d):
        for side in (0, 1):
            others = [e for e in range(p.d) if e != d]
            grids = np.meshgrid(*([s] * len(others)), indexing="ij")   # first other axis slowest
            cols = {}
            for k, e in enumerate(others):
                cols[e] = grids[k].T.ravel() if len(others) == 2 else grids[k].ravel()
            X = np.zeros((M ** len(others), p.d))
            for e in others:
                X[:, e] = cols[e]
            X[:, d] = p.lo if side == 0 else p.hi
            out.append(p.psi_at(t, X))
    return np.stack(out)
