#!/usr/bin/env python
"""Benchmark of the hot path: implicit semi-Lagrangian HJB steps (arXiv:1605.04821) on B200.

One "step" = one implicit Euler step t_{n-1} -> t_n solved by policy iteration through the C-ABI
(`hjb_step`: control search + GMG-preconditioned BiCGSTAB per policy iteration), i.e. every row
of SURVEY.md §8(a) once.  Metric (BASELINE.json): unknowns*steps/s = N_I * K / time.
Steps follow the config's own schedule (cfg4: T = 1 in 8 implicit steps): step s of the run is step
((s-1) mod n_steps) + 1 of a march, which restarts from g = u*(0) after n_steps, so every timed
step lies in t in (0, T] (warm-up + timed steps may span several marches).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl b200|reference]

Prints ONE JSON line (rank 0).  Timing: W untimed warm-up steps, then exactly K steps bracketed by
a barrier + cuda synchronize on both sides, each step timed with CUDA events on the library's
stream (L2 flushed before every timed step by writing a 256 MiB buffer, outside the events),
max over ranks.  `roofline` is the dominant kernel class's algorithmic bytes / its summed
event-timed device time over the timed region (library instrumentation, hjb_profile_*).
`e2e` repeats the timed steps through the same C-ABI call with pinned HOST buffers (host<->device
copies inside the timed region).  `cpu_baseline` (rank 0, N=1) times the CPU oracle on a bounded
sample (one full oracle step of the same coefficient model on a reduced grid).
`--impl reference` times that oracle alone (the CPU reference arm of this tier).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "implicit SL steps: unknowns·steps/s, fraction of HBM/FP64 roofline, 1/2/4/8 B200"
UNIT = "unknowns·steps/s"
CONFIG_IDX = {"cfg0": 0, "cfg1": 1, "cfg2": 2, "cfg3": 3, "cfg4": 4}
DEFAULT_CONFIG = "cfg4"
ORACLE_SAMPLE_N = 129          # cpu_baseline / reference-arm sample grid (same coefficient model)
HBM_FALLBACK_GBS = 6650.0      # B200_PROFILING.md fallback, used only without MEASURED_PEAKS.json
FP64_NOMINAL_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # 148 SMs x 64 DFMA/clk x 2 x 1.965 GHz


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIG_IDX))
    ap.add_argument("--n", type=int, default=None, help="override grid size (diagnostics only)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-time-kernels", action="store_true",
                    help="do not event-time kernel classes (roofline then null)")
    ap.add_argument("--json-out", default=None)
    ap.add_argument("--pi-forcing", type=float, default=None, help="solver setting (default: library's)")
    ap.add_argument("--nu", type=int, default=None, help="V(nu,nu) smoothing sweeps (default: library's 2)")
    ap.add_argument("--nu-pre", type=int, default=None, help="pre-smoothing sweeps (overrides --nu)")
    ap.add_argument("--nu-post", type=int, default=None, help="post-smoothing sweeps (overrides --nu)")
    ap.add_argument("--gamma", type=int, default=None, help="multigrid cycle index (default: library's 2)")
    ap.add_argument("--gamma-min", type=int, default=None, help="min coarse-level nodes for a revisit")
    ap.add_argument("--mg-precision", type=int, default=None, choices=[0, 1],
                    help="multigrid cycle vectors: 0 = fp64, 1 = fp32 (default: library's)")
    ap.add_argument("--nested-upto", type=int, default=1,
                    help="steps 1..K of a march start from the nested coarse solve (HJB_GUESS_NESTED); "
                         "later steps extrapolate in time; 0 = never nested")
    ap.add_argument("--nested-min-n", type=int, default=None, help="HJB_GUESS_NESTED: smallest nested grid")
    ap.add_argument("--nested-coarsen", type=int, default=None, help="HJB_GUESS_NESTED: 2^m coarsening per axis")
    ap.add_argument("--nested-increment", type=int, default=None,
                    help="HJB_GUESS_NESTED: 1 = U_prev + prolonged coarse increment")
    ap.add_argument("--stats-jsonl", default=None,
                    help="write one JSON line of hjb_step_stats per timed step (SURVEY §5 metrics)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": HBM_FALLBACK_GBS}, "fallback"


def fp64_peak():
    """Measured fp64 FMA peak (profiles/fp64_peak.json, tools/fp64_peak.cu) else nominal."""
    path = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["tflops"]), "measured (profiles/fp64_peak.json)"
    return FP64_NOMINAL_TFLOPS, "nominal 148 SMs x 64 DFMA/clk x 2 x 1.965 GHz"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [c.strip() for c in r]
            if len(r) < 9:
                continue
            try:
                sm.append(float(r[1]))
                smax.append(float(r[2]))
            except ValueError:
                continue
            for nm, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU oracle
def oracle_sample(cfg_idx: int, n: int = ORACLE_SAMPLE_N):
    """One full oracle implicit step (policy iteration, SuperLU solves) of the same coefficient model
    on an n^d grid, single-threaded.  Returns (unknowns*steps/s, seconds, description)."""
    from threadpoolctl import threadpool_limits

    from oracle.howard import howard_step
    from synth import bj_config
    p = bj_config(cfg_idx, n=n if cfg_idx != 3 else min(n, 17))
    U0 = p.g(p.all_idx())
    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        howard_step(p, U0, p.dt, p.dt)
        el = time.perf_counter() - t0
    desc = (f"one oracle implicit step (Howard + SuperLU, 1 thread) of the {p.name} coefficient model "
            f"on {p.n}^{p.d} ({p.N_interior} unknowns, K={p.K}, dt={p.dt:g})")
    return p.N_interior / el, el, desc


def run_reference(args):
    rank, world, _ = dist_env()
    if world > 1 and rank != 0:
        return
    cfg = CONFIG_IDX[args.config]
    for _ in range(args.warmup):
        oracle_sample(cfg, n=17 if cfg != 3 else 9)
    vals, secs = [], []
    desc = ""
    for _ in range(args.steps):
        v, s, desc = oracle_sample(cfg)
        vals.append(v)
        secs.append(s)
    tot = sum(secs)
    from synth import bj_config
    p = bj_config(cfg, n=ORACLE_SAMPLE_N if cfg != 3 else 17)
    value = p.N_interior * args.steps / tot
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"{args.config} coefficient model, oracle sample on {p.n}^{p.d}"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line, args)


def emit(line, args):
    s = json.dumps(line)
    print(s, flush=True)
    if args.json_out:
        with open(args.json_out, "w") as f:
            f.write(s + "\n")


# ----------------------------------------------------------------------------- GPU arm
def run_b200(args):
    import numpy as np
    import torch

    from paper_1605_04821_b200 import build as libbuild
    rank, world, local = dist_env()
    if world != args.gpus and "WORLD_SIZE" in os.environ:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (there is no CPU fallback)")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if rank == 0:
        libbuild.build()
    if dist is not None:
        dist.barrier()
    from paper_1605_04821_b200 import _lib
    from synth import bj_config
    from synth.device import grid_for, initial_values, packed_psi

    cfg = CONFIG_IDX[args.config]
    p = bj_config(cfg, n=args.n)
    dev = torch.device("cuda", local)
    comm_id = None
    if dist is not None:                      # slab decomposition over the ranks (NCCL)
        obj = [_lib.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm_id = obj[0]
    g, fields = grid_for(p, device=local, rank=rank, nranks=world, comm="nccl", comm_id=comm_id)
    lay = g.layout()
    nI = p.N_interior                          # whole-job unknowns (all ranks)
    U = initial_values(p, device=dev, lay=lay).contiguous()
    U2 = torch.empty_like(U)
    pol = torch.zeros(lay["local_elems"], dtype=torch.uint8, device=dev)

    def bar():
        if dist is not None:
            dist.barrier()

    def allmax(v):
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # 256 MiB > 126 MB L2
    stream = torch.cuda.current_stream(dev)
    total = args.warmup + args.steps
    # per-step inputs of one march (problem data, generated before the timed region)
    ns = p.n_steps
    psis = [packed_psi(p, s * p.dt, device=dev) for s in range(1, ns + 1)]
    srcs = [p.f_tables(s * p.dt) for s in range(1, ns + 1)]
    U0 = U.clone()                             # g = u*(0): every march starts here

    skw = {} if args.pi_forcing is None else {"pi_forcing": args.pi_forcing}
    mgkw = {} if args.nu is None else {"nu_pre": args.nu, "nu_post": args.nu}
    if args.nu_pre is not None:
        mgkw["nu_pre"] = args.nu_pre
    if args.nu_post is not None:
        mgkw["nu_post"] = args.nu_post
    if args.gamma is not None:
        mgkw["gamma"] = args.gamma
    if args.gamma_min is not None:
        mgkw["gamma_min_nodes"] = args.gamma_min
    if args.mg_precision is not None:
        mgkw["precision"] = args.mg_precision

    def step_of(s):          # step index within its march (1..n_steps)
        return (s - 1) % ns + 1

    if args.nested_min_n is not None:
        skw["nested_min_n"] = args.nested_min_n
    if args.nested_coarsen is not None:
        skw["nested_coarsen"] = args.nested_coarsen
    if args.nested_increment is not None:
        skw["nested_increment"] = args.nested_increment

    def guess_of(si):        # initial iterate of step si (the fixed point does not depend on it)
        if si <= args.nested_upto:
            return _lib.HJB_GUESS_NESTED
        return _lib.HJB_GUESS_EXTRAPOLATE if si >= 2 else _lib.HJB_GUESS_PREV

    def do_step(s, Uin, Uout, polbuf):
        # march restart: U^0 = g (a device copy, part of the step's setup a1).  Initial iterate:
        # linear extrapolation 2 U^{n-1} - U^{n-2} once two steps exist (Uout holds U^{n-2}:
        # ping-pong buffers); the fixed point does not depend on it (DESIGN.md xxiv)
        si = step_of(s)
        if si == 1:
            Uin.copy_(U0)
        fb, fc = srcs[si - 1]
        g.set_source(fb, fc)
        return g.step(p.dt, Uin, Uout, polbuf, psis[si - 1], mg=mgkw, guess=guess_of(si), **skw)

    stats = []
    for s in range(1, args.warmup + 1):
        do_step(s, U, U2, pol)
        U, U2 = U2, U
    torch.cuda.synchronize()
    # state at the start of the timed region: the e2e pass replays exactly these steps
    snap = None if args.no_e2e else (U.cpu().pin_memory(), U2.cpu().pin_memory(), pol.cpu().pin_memory())
    dsnap = None if args.no_time_kernels else (U.clone(), U2.clone(), pol.clone())
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    # the timed region runs without per-kernel events (they cost ~5 % of a step and keep the
    # multigrid's level-0 cycle out of its CUDA graph); the per-class breakdown comes from a profiled
    # replay of the same steps afterwards
    g.profile_reset(time_kernels=False)
    clk = ClockSampler(local)
    bar()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    for i, s in enumerate(range(args.warmup + 1, total + 1)):
        flush.zero_()
        ev[i][0].record(stream)
        stats.append(do_step(s, U, U2, pol))
        ev[i][1].record(stream)
        U, U2 = U2, U
    torch.cuda.synchronize()
    bar()
    wall = time.perf_counter() - wall0
    clocks = clk.stop()
    prof_timed = g.profile_read()
    ms_steps = [a.elapsed_time(b) for a, b in ev]
    if args.stats_jsonl and rank == 0:
        write_stats_jsonl(args.stats_jsonl, stats, ms_steps,
                          [step_of(s) * p.dt for s in range(args.warmup + 1, total + 1)], nI)
    Ufinal = U.clone()
    prof = prof_timed
    replay_steps = 0
    if dsnap is not None:       # profiled replay (per-kernel events) of the timed steps' first march part
        Ur, U2r, polr = dsnap
        replay_steps = min(args.steps, p.n_steps)
        g.profile_reset(time_kernels=True)
        ev_r0, ev_r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev_r0.record(stream)
        for s in range(args.warmup + 1, args.warmup + replay_steps + 1):
            do_step(s, Ur, U2r, polr)
            Ur, U2r = U2r, Ur
        ev_r1.record(stream)
        torch.cuda.synchronize()
        prof = g.profile_read()
        ms_replay = ev_r0.elapsed_time(ev_r1)
        del Ur, U2r, polr, dsnap
    ms_total = allmax(sum(ms_steps))          # device time, max over ranks
    value = nI * args.steps / (ms_total / 1e3)
    # solution sanity vs the manufactured solution (not a parity claim; parity is in tests/)
    t_end = step_of(total) * p.dt
    from synth.device import local_index
    li = local_index(p, lay, device=dev)
    own = ~p.is_boundary(li)
    r_own = (li // lay["row_elems"] >= lay["row0"]) & (li // lay["row_elems"] < lay["row1"])
    diff = (Ufinal - p.u_exact(t_end, li)).abs()
    err = allmax(diff[own & r_own].max().item() if world > 1 else diff.max().item())

    # --------------------------------------------------------------- roofline (dominant class)
    peaks, peak_src = measured_peaks()
    cls = prof["classes"]
    # the nested coarse grids' work (HJB_GUESS_NESTED) is one class of other grids' kernels: not a
    # roofline candidate (its share of the step is reported in time_share_by_class)
    timed = {k: v for k, v in cls.items() if v["ms"] > 0 and k != "nested"}
    roof = None
    roof_search = None
    if timed:
        dom = max(timed, key=lambda k: timed[k]["ms"])
        c = timed[dom]
        per_launch_ms = c["ms"] / max(1, c["calls"] or c["launches"])   # per application
        if dom == "search":
            pk, src = fp64_peak()
            ach = c["nodes"] * search_flops_per_node(p) / (c["ms"] / 1e3) / 1e12
            roof = {"bound": "alu", "kernel": dom, "achieved": ach, "peak": pk, "unit": "TFLOP/s",
                    "frac": ach / pk, "traffic": traffic_for(dom, args.config, c),
                    "peak_source": src, "launch_ms": per_launch_ms,
                    "flops_per_node": search_flops_per_node(p),
                    "flop_count": "SURVEY §8(d): K[(2P+1) 2^d 2 + 2Q + 4], Q = 6 (2D) / 13 (3D) basis "
                                  "terms of D8 (the library's own count uses the config's Q)"}
        else:
            ach = c["bytes"] / (c["ms"] / 1e3) / 1e9
            pk = float(peaks["hbm_gbs"])
            roof = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": pk, "unit": "GB/s",
                    "frac": ach / pk, "traffic": traffic_for(dom, args.config, c),
                    "peak_source": f"{peak_src} copy bandwidth (MEASURED_PEAKS.json)",
                    "launch_ms": per_launch_ms,
                    "algorithmic_bytes_per_launch": c["bytes"] / max(1, c["calls"] or c["launches"]),
                    "note": "per application of the fine-level operator class (one application = the "
                            "deep-rectangle kernel + boundary-layer strips)"}
        if "search" in timed and dom != "search":
            c = timed["search"]
            pk, src = fp64_peak()
            ach = c["nodes"] * search_flops_per_node(p) / (c["ms"] / 1e3) / 1e12
            roof_search = {"bound": "alu", "achieved": ach, "peak": pk, "unit": "TFLOP/s",
                           "frac": ach / pk, "peak_source": src,
                           "flops_per_node": search_flops_per_node(p),
                           "launch_ms": c["ms"] / max(1, c["calls"] or c["launches"])}
    denom = ms_replay if replay_steps else ms_total
    shares = {k: round(v["ms"] / denom, 4) for k, v in cls.items() if v["ms"] > 0}
    if shares:   # launches over < 16384 nodes are not event-timed (library: kTimeMinNodes) + host gaps
        shares["untimed_small_launches_and_gaps"] = round(max(0.0, 1.0 - sum(shares.values())), 4)
    hbm_frac = {k: (v["bytes"] / (v["ms"] / 1e3) / 1e9) / float(peaks["hbm_gbs"])
                for k, v in cls.items() if v["ms"] > 0 and k not in ("search", "nested")}

    # --------------------------------------------------------------- e2e through host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(g, p, args, snap, stream, srcs, psis, nI, dev, lay, bar, allmax, skw, mgkw, U0, step_of,
                      guess_of)

    pis = [st["pi_iters"] for st in stats]
    kr = [st["krylov_iters_total"] for st in stats]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_total / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args.config, p), "n": p.n, "d": p.d, "K": p.K,
                   "unknowns": nI, "dt": p.dt, "n_steps_per_march": p.n_steps,
                   "parallelism": f"slab{world}", "l2": "256 MiB L2 flush before every timed step; "
                   "working set > L2"},
        "roofline": roof, "roofline_search": roof_search,
        "hbm_frac_by_class": hbm_frac, "time_share_by_class": shares,
        "ms_per_step_spread": {"min": min(ms_steps), "median": statistics.median(ms_steps),
                               "max": max(ms_steps), "all": [round(x, 2) for x in ms_steps]},
        "t_range": [round((step_of(args.warmup + 1) - 1) * p.dt, 6), round(p.T, 6)]
        if args.steps >= ns else [round((step_of(s) - 1) * p.dt, 6) for s in (args.warmup + 1, total)],
        "march": f"T = {p.T:g} in {ns} implicit steps; restart from u*(0) after step {ns}",
        "pi_per_step": pis, "krylov_per_step": kr,
        "nested_pi_per_step": [st["nested_pi_iters"] for st in stats],
        "nested_ms_per_step": [round(st["ms_nested"], 2) for st in stats],
        "initial_iterate": (f"steps 1..{args.nested_upto} of a march: nested coarse solve (HJB_GUESS_NESTED); "
                            "later: 2 U^{n-1} - U^{n-2}") if args.nested_upto > 0 else
                           "step 1: U^{n-1}; later: 2 U^{n-1} - U^{n-2}",
        "mg_cycles_per_pi": (2 * sum(kr) / max(1, sum(pis))),
        "krylov_iters_per_pi": sum(kr) / max(1, sum(pis)), "pi_iters_per_step": sum(pis) / len(pis),
        "levels": stats[-1]["n_levels"], "final_rres": max(st["final_rres"] for st in stats),
        "final_rres_inf": max(st["final_rres_inf"] for st in stats),
        "final_R": max(st["final_R"] for st in stats),
        "max_err_vs_ustar": err, "wall_s_timed": wall,
        "gpu_launches": int(prof_timed["total_launches"]), "graph_launches": int(prof_timed["graph_launches"]),
        "host_launch_calls_per_step": (int(prof_timed["total_launches"]) - int(prof_timed["graph_kernels"])
                                       + int(prof_timed["graph_launches"])) / args.steps,
        "profiled_replay": None if not replay_steps else {
            "steps": replay_steps, "ms_per_step": ms_replay / replay_steps,
            "note": "roofline, hbm_frac_by_class and time_share_by_class come from this replay of the first "
                    "timed steps from the same state with per-kernel CUDA events on (the timed region runs "
                    "without them)"},
        "clocks": clocks, "e2e": e2e,
    }
    if not args.no_cpu_baseline and rank == 0 and world == 1:
        v, s, desc = oracle_sample(cfg)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc,
                                "seconds": s, "host_cpus": os.cpu_count(),
                                "fullsize_sample": oracle_fullsize_sample(p, U, pol)}
    if rank == 0:
        emit(line, args)
    g.close()


def search_flops_per_node(p):
    """K [(2P+1) 2^d 2 + 2Q + 4] algorithmic fp64 flops per node of the control search,
    with Q = 6 (2D) / 13 (3D) source basis terms (derivation D8)."""
    q = 6 if p.d == 2 else 13
    return p.K * ((2 * p.P + 1) * (1 << p.d) * 2 + 2 * q + 4)


def oracle_fullsize_sample(p, U, pol, m=1 << 15):
    """SURVEY §8(d) oracle baseline at the FULL config size: the oracle's brute-force control search
    and matrix-free apply on m sampled interior rows of the real grid (1 thread), as rows/s."""
    import numpy as np
    from threadpoolctl import threadpool_limits

    from oracle.howard import control_search
    from oracle.scheme import apply_operator
    rng = np.random.default_rng(11)
    mi = [rng.integers(1, p.n - 1, size=m) for _ in range(p.d)]
    idx = np.zeros(m, dtype=np.int64)
    for k in reversed(range(p.d)):
        idx = idx * p.n + mi[k]
    Uh = U.cpu().numpy()
    polh = pol.cpu().numpy().astype(np.int64)
    fields = p.fields(idx)
    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        control_search(p, Uh, Uh, p.dt, p.dt, fields=fields, idx=idx)
        ts = time.perf_counter() - t0
        t0 = time.perf_counter()
        apply_operator(p, polh, Uh, p.dt, idx=idx, fields=fields)
        ta = time.perf_counter() - t0
    return {"search_rows_per_s": m / ts, "apply_rows_per_s": m / ta, "rows": m, "cores": 1,
            "search_s": ts, "apply_s": ta,
            "sample": f"oracle control search (K={p.K}) and apply on {m} random interior rows of the "
                      f"full {p.n}^{p.d} grid, 1 thread"}


def workload_name(cfg, p):
    return {"cfg0": "BASELINE configs[0]", "cfg1": "BASELINE configs[1]", "cfg2": "BASELINE configs[2]",
            "cfg3": "BASELINE configs[3]", "cfg4": "BASELINE configs[4] (largest grid, 1 GPU)"}[cfg] + \
        f": d={p.d}, {p.n}^{p.d} grid, K={p.K}"


def traffic_for(cls, config, c):
    """DRAM bytes per launch of this class from a committed ncu --set full summary
    (profiles/ncu_traffic.json: bytes per node of the captured launch x this run's nodes/launch)."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    e = d.get(config, {}).get(cls)
    if not e:
        return None
    return e["dram_bytes_per_node"] * c["nodes"] / max(1, c["calls"] or c["launches"])


def write_stats_jsonl(path, stats, ms_steps, ts, nI):
    """Per-step metrics, one JSON object per line (SURVEY §5 "Metrics / logging")."""
    with open(path, "w") as f:
        for st, ms, t in zip(stats, ms_steps, ts):
            k = st["pi_iters"]
            f.write(json.dumps({
                "t": round(t, 12), "ms": round(ms, 3), "unknowns_steps_per_s": nI / (ms / 1e3),
                "pi_iters": k, "krylov_iters": st["krylov_iters"], "mg_cycles": 2 * st["krylov_iters_total"],
                "changed": st["changed"], "R": st["R"], "final_R": st["final_R"],
                "final_rres": st["final_rres"], "final_rres_inf": st["final_rres_inf"],
                "nested_pi_iters": st["nested_pi_iters"], "ms_nested": st["ms_nested"],
                "ms_search": st["ms_search"], "ms_setup": st["ms_setup"], "ms_solve": st["ms_solve"],
                "status": st.get("status")}) + "\n")


def run_e2e(g, p, args, snap, stream, srcs, psis, nI, dev, lay, bar, allmax, skw, mgkw, U0, step_of, guess_of):
    """The SAME K steps as the timed region (replayed from its starting state) through hjb_step with
    pinned HOST buffers: each step copies U_prev, the policy and psi host->device and U + policy
    device->host inside the timed region (inside the call).  A march restart passes a pinned host
    copy of g = u*(0) (prepared before the timed region, one per restart) as U_prev."""
    import torch
    N = lay["local_elems"]
    Uh_prev, Uh, polh = snap          # U^{W}, U^{W-1}, policy at the start of the timed region
    psih = [x.cpu().pin_memory() for x in psis]
    Uh_np, Uhp_np, pol_np = Uh.numpy(), Uh_prev.numpy(), polh.numpy()
    psi_np = [x.numpy() for x in psih]
    base = args.warmup
    n_e2e = args.steps
    restarts = [s for s in range(base + 1, base + n_e2e + 1) if step_of(s) == 1]
    u0h = {s: U0.cpu().pin_memory().numpy() for s in restarts}
    bar()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    t0 = time.perf_counter()
    from paper_1605_04821_b200 import _lib
    for i in range(n_e2e):
        s = base + i + 1
        si = step_of(s)
        if si == 1:
            Uhp_np = u0h[s]
        fb, fc = srcs[si - 1]
        g.set_source(fb, fc)
        g.step(p.dt, Uhp_np, Uh_np, pol_np, psi_np[si - 1], mg=mgkw, **skw, guess=guess_of(si))
        Uhp_np, Uh_np = Uh_np, Uhp_np
    ev1.record(stream)
    torch.cuda.synchronize()
    bar()
    wall = time.perf_counter() - t0
    ms = allmax(ev0.elapsed_time(ev1))
    nb = psis[0].numel()
    return {"value": nI * n_e2e / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": 8 * N + N + 8 * nb,
            "d2h_bytes_per_step": 8 * N + N, "steps": n_e2e, "wall_s": wall,
            "path": "hjb_step C-ABI with pinned host U_prev/U/policy/psi"}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
