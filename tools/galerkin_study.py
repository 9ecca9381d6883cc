"""Galerkin (R A P) vs rediscretised coarse operators (NEXT-4 measurement): for the greedy policy at
U0 of a BASELINE config, the exact policy-evaluation solve (BiCGSTAB to 1e-12) with each coarse
operator and cycle index; iterations, setup and solve device time, and the stationary contraction
of one cycle (||r_after|| / ||r_before|| of x += M^-1 r, averaged over 5 cycles).

    python tools/galerkin_study.py --cfg 2
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from synth import bj_config  # noqa: E402
from synth.device import grid_for, initial_values, packed_psi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=2)
ap.add_argument("--n", type=int, default=None)
args = ap.parse_args()
p = bj_config(args.cfg, n=args.n)
g, fields = grid_for(p, device=0)
U0 = initial_values(p).contiguous()
pol = torch.zeros(p.N, dtype=torch.uint8, device="cuda")
F = torch.zeros(p.N, dtype=torch.float64, device="cuda")
fb, fc = p.f_tables(p.dt)
g.set_source(fb, fc)
g.policy_update(p.dt, U0, U0, pol, F)
for coarse_op in (0, 1):
    for gamma in (1, 2):
        mg = {"coarse_op": coarse_op, "gamma": gamma}
        torch.cuda.synchronize()
        t0 = time.time()
        try:
            nl = g.mg_setup(p.dt, pol, **mg)
        except Exception as e:  # noqa: BLE001
            print(f"cfg{args.cfg} coarse_op={coarse_op} gamma={gamma}: {e}", flush=True)
            continue
        torch.cuda.synchronize()
        ts = time.time() - t0
        x = U0.clone()
        t0 = time.time()
        st = g.solve(p.dt, pol, F, x, mg=mg)
        torch.cuda.synchronize()
        tv = time.time() - t0
        print(f"cfg{args.cfg} n={p.n} coarse_op={'galerkin' if coarse_op else 'rediscretised'} gamma={gamma} "
              f"levels={nl}: BiCGSTAB iterations {st['iters']} (rres {st['rres']:.1e}), setup {ts * 1e3:.1f} ms, "
              f"solve {tv * 1e3:.1f} ms", flush=True)
g.close()
