"""Diagnostics (not the product path): how many preconditioner applications does the policy
evaluation need with the library's BiCGSTAB vs a right-preconditioned GMRES(m) prototype built
from the same C-ABI calls (hjb_apply, hjb_mg_apply) and torch vector algebra, and what is the
contraction factor of the V-cycle used as a stationary iteration.

    python tools/krylov_study.py --cfg 2 [--m 40] [--eta 0.03]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from synth import bj_config  # noqa: E402
from synth.device import grid_for, initial_values  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=2)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--m", type=int, default=40)
ap.add_argument("--eta", type=float, default=0.03)
ap.add_argument("--nu", type=int, default=2)
ap.add_argument("--omega", type=float, default=None)
ap.add_argument("--kmode", type=int, default=None)
ap.add_argument("--no-gmres", action="store_true")
ap.add_argument("--exact-only", action="store_true")
args = ap.parse_args()

p = bj_config(args.cfg, n=args.n)
g, _ = grid_for(p, device=0)
U0 = initial_values(p).contiguous()
pol = torch.zeros(p.N, dtype=torch.uint8, device="cuda")
F = torch.zeros(p.N, dtype=torch.float64, device="cuda")
g.policy_update(p.dt, U0, U0, pol, F)
mask = torch.ones(p.N, dtype=torch.float64, device="cuda")
mask[torch.from_numpy(p.boundary_idx()).cuda()] = 0.0
mg = {"nu_pre": args.nu, "nu_post": args.nu}
if args.omega is not None:
    mg["omega"] = args.omega
if args.kmode is not None:
    mg["coarse_k_mode"] = args.kmode
g.mg_setup(p.dt, pol, **mg)
torch.cuda.synchronize()
print(f"{p.name} n={p.n} K={p.K} N={p.N}", flush=True)


def A(x):
    y = torch.empty_like(x)
    g.apply(p.dt, pol, x, y)
    return y * mask


def M(b):
    x = torch.zeros_like(b)
    g.mg_apply(b, x)
    return x * mask


Fi = F * mask
fn = Fi.norm().item()
r0 = Fi - A(U0)
r0n = r0.norm().item()
print(f"||F|| = {fn:.3e}  ||r0||/||F|| = {r0n / fn:.3e}", flush=True)

# stationary V-cycle iteration on the error equation
x = torch.zeros_like(r0)
res = [r0n]
for k in range(8):
    r = r0 - A(x)
    x = x + M(r)
    res.append((r0 - A(x)).norm().item())
rates = [res[i + 1] / res[i] for i in range(len(res) - 1)]
print("stationary V-cycle residual ratios:", " ".join(f"{q:.3f}" for q in rates), flush=True)

cases = (("eta", max(1e-12 * fn, args.eta * r0n)), ("exact", 1e-12 * fn))
for tol_name, tol in cases[1:] if args.exact_only else cases:
    # library BiCGSTAB
    xb = U0.clone()
    torch.cuda.synchronize()
    t0 = time.time()
    rt = tol / fn
    st = g.solve(p.dt, pol, F, xb, mg=mg, krylov_rtol=max(rt, 1e-14), krylov_maxit=500)
    torch.cuda.synchronize()
    tb = time.time() - t0
    print(f"[{tol_name}] BiCGSTAB: iters={st['iters']} precond={2 * st['iters']} rres={st['rres']:.2e} "
          f"{tb * 1e3:.1f} ms", flush=True)
    if args.no_gmres:
        continue
    # GMRES(m), right preconditioned, classical Gram-Schmidt with one re-orthogonalisation
    torch.cuda.synchronize()
    t0 = time.time()
    xg = U0.clone()
    nprec = 0
    tot = 0
    for cyc in range(10):
        r = Fi - A(xg) if cyc else r0.clone()
        beta = r.norm().item()
        if beta <= tol:
            break
        m = args.m
        V = torch.empty((m + 1, p.N), dtype=torch.float64, device="cuda")
        V[0] = r / beta
        Hm = np.zeros((m + 1, m))
        cs, sn = np.zeros(m), np.zeros(m)
        gv = np.zeros(m + 1)
        gv[0] = beta
        j_done = 0
        for j in range(m):
            w = A(M(V[j]))
            nprec += 1
            h = V[:j + 1] @ w
            w -= V[:j + 1].T @ h
            h2 = V[:j + 1] @ w
            w -= V[:j + 1].T @ h2
            hcol = (h + h2).cpu().numpy()
            hn = w.norm().item()
            Hm[:j + 1, j] = hcol
            Hm[j + 1, j] = hn
            for i in range(j):
                a, b = Hm[i, j], Hm[i + 1, j]
                Hm[i, j], Hm[i + 1, j] = cs[i] * a + sn[i] * b, -sn[i] * a + cs[i] * b
            d = np.hypot(Hm[j, j], Hm[j + 1, j])
            cs[j], sn[j] = Hm[j, j] / d, Hm[j + 1, j] / d
            Hm[j, j], Hm[j + 1, j] = d, 0.0
            gv[j + 1] = -sn[j] * gv[j]
            gv[j] = cs[j] * gv[j]
            j_done = j + 1
            if hn > 0:
                V[j + 1] = w / hn
            if abs(gv[j + 1]) <= tol:
                break
        y = np.linalg.solve(np.triu(Hm[:j_done, :j_done]), gv[:j_done])
        z = V[:j_done].T @ torch.from_numpy(y).cuda()
        xg = xg + M(z)
        nprec += 1
        tot += j_done
        del V
    torch.cuda.synchronize()
    tg = time.time() - t0
    tr = (Fi - A(xg)).norm().item()
    print(f"[{tol_name}] GMRES({args.m}): iters={tot} precond={nprec} rres={tr / fn:.2e} (target {tol / fn:.2e}) "
          f"{tg * 1e3:.1f} ms (torch vector algebra)", flush=True)
