"""The paper's own linear-solve timings as context (Table "Time"):
Problems A and B at N_x = 321 / 641, implicit theta = 1, dt = T and dt = dx, on the GPU
through hjb_step, reporting the average device seconds per time step spent in policy evaluation
(MG/AGMG setup + Krylov solve, the quantity of Table Time), policy and Krylov iterations, and the
L-infinity error against u* (Table 4 / 4-B).  The paper: MATLAB 2015a,
quad-core AMD 4.2 GHz, Krylov tolerance 1e-6 relative; this run uses the same
tolerance for the linear solves (krylov_rtol = 1e-6, no max-norm stop) with the paper's preconditioner
(solver = 1: GCR + aggregation AMG with K-cycle) and the library default (BiCGSTAB +
GMG where n = 2^l + 1, unpreconditioned BiCGSTAB otherwise).  Context only, not a target.

    python tools/paper_context.py [--sizes 321,641] [--solvers 1,0]
"""
import argparse
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1605_04821_b200 import _lib  # noqa: E402
from synth import problem_A, problem_B  # noqa: E402
from synth.device import grid_for, packed_psi  # noqa: E402

# PAPER.md:1206-1210, seconds per time step in linear solves: (Direct, AMG, AGMG) x (dt = T, dt = dx)
PAPER = {("A", 321): {"T": (49.60, 43.62, 3.31), "dx": (17.93, 10.07, 0.41)},
         ("A", 641): {"T": (9.50e3, 373.77, 21.22), "dx": (4.33e3, 48.82, 1.84)},
         ("B", 321): {"T": (14.35, 18.59, 0.77), "dx": (68.70, 16.19, 0.40)},
         ("B", 641): {"T": (950.62, 5.64e3, 7.82), "dx": (2.09e4, 102.57, 1.85)}}

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="321,641")
ap.add_argument("--solvers", default="1,0")
args = ap.parse_args()
print("problem N_x dt solver | steps PI/step Krylov/PI | s/step solve (GPU) | paper s/step AGMG (Direct, AMG) "
      "| err vs u*", flush=True)
for prob, mk in (("A", problem_A), ("B", problem_B)):
    for nx in [int(s) for s in args.sizes.split(",")]:
        for col in ("T", "dx"):
            for solver in [int(s) for s in args.solvers.split(",")]:
                p = mk(nx)
                dx = (p.hi - p.lo) / (p.n - 1)
                n_steps = 1 if col == "T" else int(math.ceil(p.T / dx - 1e-12))
                dt = p.T / n_steps
                g, _ = grid_for(p, device=0, from_host=True)
                U = torch.from_numpy(p.g(p.all_idx())).cuda()
                U2 = torch.empty_like(U)
                pol = torch.zeros(p.N, dtype=torch.uint8, device="cuda")
                tot_solve, pis, krs = 0.0, 0, 0
                for s in range(1, n_steps + 1):
                    fb, fc = p.f_tables(s * dt)
                    g.set_source(fb, fc)
                    st = g.step(dt, U, U2, pol, packed_psi(p, s * dt), solver=solver, krylov_rtol=1e-6,
                                krylov_rtol_inf=0.0, guess=_lib.HJB_GUESS_PREV)
                    tot_solve += (st["ms_setup"] + st["ms_solve"]) / 1e3
                    pis += st["pi_iters"]
                    krs += st["krylov_iters_total"]
                    U, U2 = U2, U
                torch.cuda.synchronize()
                err = float(np.abs(U.cpu().numpy() - p.u_exact(p.T, p.all_idx())).max())
                ref = PAPER[(prob, nx)][col]
                print(f"{prob} {nx} {col:2s} {'AGMG+GCR' if solver == 1 else 'BiCGSTAB(+GMG)':14s} | {n_steps:3d} "
                      f"{pis / n_steps:5.2f} {krs / max(1, pis):6.2f} | {tot_solve / n_steps:9.4f} | "
                      f"{ref[2]:8.2f} ({ref[0]:.3g}, {ref[1]:.3g}) | {err:.3e}", flush=True)
                g.close()
