"""Kernel-level timing of the hot kernels on a BASELINE config (diagnostics, not the bench):
fine-level operator apply (hjb_apply), one V-cycle (hjb_mg_apply), control search
(hjb_policy_update), with the library's per-class event timing and algorithmic bytes/flops.

    python tools/opbench.py --cfg 4 [--reps 20]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from synth import bj_config, random_vector  # noqa: E402
from synth.device import grid_for, initial_values  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=4)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--only", default="apply,vcycle,search")
ap.add_argument("--policy", default="greedy", choices=["greedy", "zero", "random"])
args = ap.parse_args()
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "MEASURED_PEAKS.json"))) if os.path.exists("MEASURED_PEAKS.json") else {"hbm_gbs": 6454.0}
p = bj_config(args.cfg, n=args.n)
t0 = time.time()
g, fields = grid_for(p, device=0)
U0 = initial_values(p).contiguous()
x = random_vector(p, idx=torch.arange(p.N, device="cuda")).contiguous()
pol = torch.zeros(p.N, dtype=torch.uint8, device="cuda")
F = torch.zeros(p.N, dtype=torch.float64, device="cuda")
g.policy_update(p.dt, U0, U0, pol, F)          # a realistic (smooth) policy: greedy at U0
if args.policy == "zero":
    pol.zero_()
elif args.policy == "random":
    pol.copy_(torch.remainder(torch.arange(p.N, device="cuda") * 2654435761, p.K).to(torch.uint8))
y = torch.empty_like(x)
torch.cuda.synchronize()
print(f"{p.name} n={p.n} K={p.K} N={p.N} setup {time.time() - t0:.1f}s", flush=True)


def report(tag, reps):
    pr = g.profile_read()
    for k, v in pr["classes"].items():
        if v["launches"] and v["ms"] > 0:
            gbs = v["bytes"] / (v["ms"] / 1e3) / 1e9
            calls = v.get("calls") or v["launches"]
            print(f"  [{tag}] {k:9s} calls={calls:5d} launches={v['launches']:5d} ms/call={v['ms'] / calls:9.4f} "
                  f"GB/s={gbs:8.1f} ({gbs / peaks['hbm_gbs']:.3f} of HBM) TF/s={v['flops'] / (v['ms'] / 1e3) / 1e12:7.3f}",
                  flush=True)


only = args.only.split(",")
if "apply" in only:
    for _ in range(3):
        g.apply(p.dt, pol, x, y)
    g.profile_reset(True)
    for _ in range(args.reps):
        g.apply(p.dt, pol, x, y)
    report("apply", args.reps)
if "vcycle" in only:
    g.mg_setup(p.dt, pol)
    g.mg_apply(x, y)
    g.profile_reset(True)
    for _ in range(max(1, args.reps // 4)):
        g.mg_apply(x, y)
    report("vcycle", args.reps // 4)
    # whole cycles without per-kernel events (graph replay on one rank), CUDA events on the stream
    g.profile_reset(False)
    for prec in (0, 1):
        g.mg_setup(p.dt, pol, precision=prec)
        g.mg_apply(x, y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(1, args.reps // 2)
        e0.record()
        for _ in range(reps):
            g.mg_apply(x, y)
        e1.record()
        torch.cuda.synchronize()
        print(f"  [vcycle] precision={prec} (0 fp64, 1 fp32): {e0.elapsed_time(e1) / reps:.3f} ms per cycle "
              f"(untimed kernels, {reps} cycles)", flush=True)
if "search" in only:
    g.profile_reset(True)
    for _ in range(max(1, args.reps // 10)):
        g.policy_update(p.dt, U0, U0, pol, F)
    report("search", args.reps // 10)
