"""Per-level / per-class launches and time of ONE outer FGMRES cycle on cfg2 (5 Hz) with B
identical RHS (none converges): where the fixed per-cycle cost goes.

    python scripts/cycle_profile.py [B ...]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1703_09268_b200 import api  # noqa: E402

p = synth.cfg2(freqs=(5.0,))
grid, pml = api.Grid.of(p), api.Pml(v_ref=3000.0)
w = 2 * np.pi * 5.0
for B in [int(x) for x in sys.argv[1:]] or [1, 150]:
    op = api.helm_setup(grid, p.m, w, pml, api.C128, max_rhs=B)
    Bq = torch.zeros(B, p.n_ext, dtype=torch.complex128, device="cuda")
    nx = p.next[0]
    node = int(p.src[25])
    Bq[:, (node // p.n[0] + 20) * nx + node % p.n[0] + 20] = 1.0 / p.h**2
    X = torch.empty_like(Bq)
    so = api.SolveOpts(rtol=1e-14, max_outer=2)
    api.helm_solve(op, Bq, X, opts=so)
    torch.cuda.synchronize()
    api.profile(True, 1)
    n0 = api.launch_count() if hasattr(api, "launch_count") else 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    api.helm_solve(op, Bq, X, opts=so)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 2
    out = {"B": B, "ms_per_cycle": round(ms, 2), "levels": {}}
    tot_l = 0
    for lv in range(4):
        pr = api.profile_read(lv)
        row = {k: [v["launches"] // 2, round(v["ms"] / 2, 2)] for k, v in pr.items() if v["launches"]}
        if row:
            out["levels"][lv] = row
            tot_l += sum(v[0] for v in row.values())
    out["launches_per_cycle"] = tot_l
    api.profile(False, 1)
    print(json.dumps(out))
    del op
