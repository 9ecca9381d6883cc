"""Policy-iteration trace of one march (diagnostics): per step, per PI iteration the changed count,
the nonlinear residual R and the Krylov iterations; optional solver settings.

    python tools/pi_study.py --cfg 4 [--steps 3] [--pi-forcing 0.01]
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
ap.add_argument("--cfg", type=int, default=4)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--pi-forcing", type=float, default=None)
args = ap.parse_args()
p = bj_config(args.cfg, n=args.n)
g, fields = grid_for(p, device=0)
U = initial_values(p).contiguous()
U2 = torch.empty_like(U)
pol = torch.zeros(p.N, dtype=torch.uint8, device="cuda")
kw = {} if args.pi_forcing is None else {"pi_forcing": args.pi_forcing}
for s in range(1, args.steps + 1):
    t = s * p.dt
    fb, fc = p.f_tables(t)
    g.set_source(fb, fc)
    torch.cuda.synchronize()
    t0 = time.time()
    guess = _lib.HJB_GUESS_EXTRAPOLATE if s >= 2 else _lib.HJB_GUESS_PREV
    st = g.step(p.dt, U, U2, pol, packed_psi(p, t), guess=guess, **kw)
    torch.cuda.synchronize()
    el = time.time() - t0
    print(f"step {s}: {el * 1e3:.0f} ms pi={st['pi_iters']} krylov={st['krylov_iters']} "
          f"changed={st['changed']} R={['%.1e' % r for r in st['R']]} "
          f"ms search/setup/solve={st['ms_search']:.0f}/{st['ms_setup']:.0f}/{st['ms_solve']:.0f}", flush=True)
    U, U2 = U2, U
