"""BASELINE configs[3] at full size on one GPU: 3D layered model 200^3 + PML 20 (240^3
extended), h = 25 m, f = 6 Hz, 64 surface sources, 40,000 receivers. Generates d_obs at the
true model (FORW_MODEL, rtol 1e-8), then times one misfit + gradient evaluation (128 solves,
rtol 1e-6) and prints solves/s, outer cycles, the library's algorithmic bytes and the
per-level kernel breakdown.

    python scripts/cfg4_run.py [--max-rhs 16] [--dtype c128|c64] [--n 200]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1703_09268_b200 import api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--max-rhs", type=int, default=16)
ap.add_argument("--dtype", default="c128")
ap.add_argument("--n", type=int, default=200)
ap.add_argument("--nsrc", type=int, default=64)
a = ap.parse_args()
t0 = time.perf_counter()
p = synth.cfg4(n=a.n)
p = p.with_(src=p.src[:a.nsrc])
grid = api.Grid.of(p)
pml = api.Pml(v_ref=4500.0)
dt = api.C64 if a.dtype == "c64" else api.C128
tg = time.perf_counter() - t0
torch.cuda.synchronize()
t1 = time.perf_counter()
d, repf = api.fwi_forward(grid, p.m_true, p.freqs, p.src, p.rec, pml, api.C128, api.SolveOpts(rtol=1e-8),
                          max_rhs=a.max_rhs)
torch.cuda.synchronize()
tf = time.perf_counter() - t1
api.profile(True, 5)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
fg, rep = api.fwi_misfit_grad(grid, p.m, p.freqs, p.src, p.rec, d, pml, dt, api.SolveOpts(rtol=1e-6),
                              max_rhs=a.max_rhs)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
levels = {}
for lv in range(4):
    pr = api.profile_read(lv)
    row = {k: {"est_ms": round(v["ms"] * v["launches"] / v["sampled"], 1),
               "GBps": round(v["bytes"] / max(v["ms"], 1e-9) / 1e6, 1), "launches": v["launches"],
               "us_per_launch": round(1e3 * v["ms"] / v["sampled"], 1)} for k, v in pr.items() if v["sampled"]}
    if row:
        levels[lv] = row
api.profile(False, 1)
fgh = fg.cpu().numpy()
nsolve = len(rep)
byts = sum(r["bytes_alg"] for r in rep)
out = {"workload": f"cfg4 {a.n}^3 + PML {p.pml[0][0]}, 64 sources, 6 Hz, {a.dtype}, max_rhs {a.max_rhs}",
       "gen_s": round(tg, 1), "forward_data_s": round(tf, 1), "eval_s": round(ms / 1e3, 2),
       "solves": nsolve, "solves_per_s": round(nsolve / (ms / 1e3), 3),
       "cycles": {"min": min(r["outer_cycles"] for r in rep), "max": max(r["outer_cycles"] for r in rep),
                  "mean": round(float(np.mean([r["outer_cycles"] for r in rep])), 2)},
       "all_converged": all(r["converged"] for r in rep), "f": float(fgh[0]), "g_norm": float(np.linalg.norm(fgh[1:])),
       "alg_bytes": byts, "achieved_GBps": round(byts / (ms / 1e3) / 1e9, 1), "levels": levels}
print(json.dumps(out))
