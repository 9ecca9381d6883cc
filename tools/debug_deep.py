"""Debug: deep vs general operator apply on cfg1 -- where and how much do they differ?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from synth import bj_config, random_vector
from synth.device import grid_for

p = bj_config(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
rng = np.random.default_rng(11)
Uprev = p.g(p.all_idx()); U = Uprev + 0.05 * rng.uniform(-1, 1, size=p.N)
x = random_vector(p)
out = {}
for mode in ("general", "deep"):
    os.environ.pop("HJB_NO_DEEP", None)
    if mode == "general":
        os.environ["HJB_NO_DEEP"] = "1"
    g, _ = grid_for(p, 0, from_host=True)
    pol = torch.zeros(p.N, dtype=torch.uint8, device="cuda"); F = torch.zeros(p.N, dtype=torch.float64, device="cuda")
    g.policy_update(p.dt, torch.from_numpy(U).cuda(), torch.from_numpy(Uprev).cuda(), pol, F)
    y = torch.zeros(p.N, dtype=torch.float64, device="cuda")
    g.apply(p.dt, pol, torch.from_numpy(x).cuda(), y)
    torch.cuda.synchronize()
    out[mode] = (pol.cpu().numpy(), y.cpu().numpy())
    g.close()
d = out["general"][1] - out["deep"][1]
bad = np.nonzero(d)[0]
print("policies equal:", np.array_equal(out["general"][0], out["deep"][0]))
print("differing entries:", bad.size, "of", p.N)
if bad.size:
    i0, i1 = bad % p.n, bad // p.n
    print("i0 range", i0.min(), i0.max(), "i1 range", i1.min(), i1.max())
    rel = np.abs(d[bad]) / np.maximum(1e-300, np.abs(out["general"][1][bad]))
    print("max rel", rel.max(), "median rel", np.median(rel))
    print("examples", [(int(a), int(b), out["general"][1][k], out["deep"][1][k]) for a, b, k in list(zip(i0, i1, bad))[:8]])
