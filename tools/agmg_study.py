"""Aggregation AMG (solver = 1) vs BiCGSTAB + geometric multigrid (solver = 0) on a BASELINE config:
the exact evaluation of the greedy policy at U0 (iterations, setup + solve time), then a short march
with each solver (ms per step, Krylov iterations per policy iteration).

    python tools/agmg_study.py --cfg 2 [--steps 3]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1605_04821_b200 import _lib  # noqa: E402
from synth import bj_config  # noqa: E402
from synth.device import grid_for, initial_values, packed_psi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=2)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--steps", type=int, default=3)
args = ap.parse_args()
p = bj_config(args.cfg, n=args.n)
g, fields = grid_for(p, device=0)
U0 = initial_values(p).contiguous()
pol = torch.zeros(p.N, dtype=torch.uint8, device="cuda")
F = torch.zeros(p.N, dtype=torch.float64, device="cuda")
fb, fc = p.f_tables(p.dt)
g.set_source(fb, fc)
g.policy_update(p.dt, U0, U0, pol, F)
for solver in (0, 1):
    if solver == 0:
        g.mg_setup(p.dt, pol)
    x = U0.clone()
    torch.cuda.synchronize()
    t0 = time.time()
    st = g.solve(p.dt, pol, F, x, solver=solver)
    torch.cuda.synchronize()
    print(f"cfg{args.cfg} n={p.n} solver={'AGMG+GCR' if solver else 'GMG+BiCGSTAB'}: exact policy solve "
          f"{st['iters']} iterations (rres {st['rres']:.1e}, rres_inf {st['rres_inf']:.1e}), "
          f"{(time.time() - t0) * 1e3:.1f} ms incl. setup", flush=True)
for solver in (0, 1):
    U = initial_values(p).contiguous()
    U2 = torch.empty_like(U)
    pl = torch.zeros(p.N, dtype=torch.uint8, device="cuda")
    for s in range(1, args.steps + 1):
        t = s * p.dt
        g.set_source(*p.f_tables(t))
        torch.cuda.synchronize()
        t0 = time.time()
        st = g.step(p.dt, U, U2, pl, packed_psi(p, t), solver=solver,
                    guess=_lib.HJB_GUESS_EXTRAPOLATE if s >= 2 else _lib.HJB_GUESS_PREV)
        torch.cuda.synchronize()
        print(f"  solver={solver} step {s}: {(time.time() - t0) * 1e3:.0f} ms, PI {st['pi_iters']}, "
              f"Krylov {st['krylov_iters']}, final rres {st['final_rres']:.1e}", flush=True)
        U, U2 = U2, U
g.close()
