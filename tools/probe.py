"""Quick timing/iteration probe of hjb_step on a BASELINE config (diagnostics, not the bench)."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from synth import bj_config
from synth.device import grid_for, initial_values, packed_psi

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=1)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--K", type=int, default=None)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--nu", type=int, default=2)
ap.add_argument("--omega", type=float, default=1.0)
ap.add_argument("--kmode", type=int, default=0)
ap.add_argument("--eta", type=float, default=0.0)
ap.add_argument("--profile", action="store_true")
args = ap.parse_args()
p = bj_config(args.cfg, n=args.n, K=args.K)
t0 = time.time()
g, fields = grid_for(p, device=0)
U = initial_values(p).contiguous(); U2 = torch.empty_like(U)
pol = torch.zeros(p.N, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
print(f"{p.name} n={p.n} K={p.K} N_I={p.N_interior} setup {time.time()-t0:.1f}s", flush=True)
for s in range(1, args.steps + 1):
    t = s * p.dt
    fb, fc = p.f_tables(t); g.set_source(fb, fc)
    psi = packed_psi(p, t)
    torch.cuda.synchronize(); t1 = time.time()
    if args.profile: g.profile_reset(True)
    st = g.step(p.dt, U, U2, pol, psi, mg=dict(nu_pre=args.nu, nu_post=args.nu, omega=args.omega, coarse_k_mode=args.kmode), raise_on_error=False, pi_forcing=args.eta)
    torch.cuda.synchronize(); el = time.time() - t1
    U, U2 = U2, U
    err = (U - p.u_exact(t, torch.arange(p.N, device="cuda"))).abs().max().item()
    print(json.dumps(dict(step=s, wall_s=round(el, 4), err_vs_ustar=err, **st)), flush=True)
    print(f"  unknowns*steps/s = {p.N_interior/el:.3e}", flush=True)
    if args.profile:
        pr = g.profile_read()
        for k, v in pr["classes"].items():
            if v["launches"]:
                gbs = v["bytes"] / max(v["ms"], 1e-9) / 1e6
                print(f"  {k:9s} launches={v['launches']:6d} ms={v['ms']:10.3f} GB/s={gbs:8.1f} "
                      f"TF/s={v['flops'] / max(v['ms'], 1e-9) / 1e9:7.3f}", flush=True)
