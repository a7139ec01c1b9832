"""How much of the cfg2 evaluation is the convergence tail? (1) per-RHS outer-cycle counts of
the bench's joint forward batch (150 RHS, 3 frequencies); (2) time per outer cycle t(B) with B
active RHS (B copies of one source, max_outer = 4, rtol tiny so none converges); (3) the batch
time predicted as sum over cycles c of t(nact(c)) vs the ideal sum(cycles) * t(150) / 150.

    python scripts/batch_tail.py
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1703_09268_b200 import api  # noqa: E402

p = synth.cfg2()
grid, pml = api.Grid.of(p), api.Pml(v_ref=3000.0)
d, rep = api.fwi_forward(grid, p.m_true, p.freqs, p.src, p.rec, pml, api.C128, api.SolveOpts(rtol=1e-6), max_rhs=150)
cyc = np.array([r["outer_cycles"] for r in rep])
out = {"cycles_hist": np.bincount(cyc).tolist(), "mean": float(cyc.mean()), "max": int(cyc.max())}
w = 2 * np.pi * 5.0
tb = {}
for B in (1, 2, 5, 10, 20, 40, 75, 150):
    op = api.helm_setup(grid, p.m, w, pml, api.C128, max_rhs=B)
    Bq = torch.zeros(B, p.n_ext, dtype=torch.complex128, device="cuda")
    nx = p.next[0]
    node = int(p.src[25])
    ix, iz = node % p.n[0], node // p.n[0]
    Bq[:, (iz + 20) * nx + ix + 20] = 1.0 / p.h**2
    X = torch.empty_like(Bq)
    so = api.SolveOpts(rtol=1e-14, max_outer=4)
    api.helm_solve(op, Bq, X, opts=so)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    api.helm_solve(op, Bq, X, opts=so)
    e1.record()
    torch.cuda.synchronize()
    tb[B] = e0.elapsed_time(e1) / 4
    del op
out["t_cycle_ms"] = tb
Bs = np.array(sorted(tb))
ts = np.array([tb[b] for b in Bs])
nact = [(cyc > c).sum() for c in range(cyc.max())]
pred = sum(float(np.interp(n, Bs, ts)) for n in nact if n > 0)
ideal = cyc.sum() * tb[150] / 150
out.update({"nact_per_cycle": [int(n) for n in nact], "pred_batch_ms": pred, "ideal_ms": ideal,
            "tail_overhead": pred / ideal - 1})
print(json.dumps(out))
