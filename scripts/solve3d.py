"""Timed 3D preconditioned solve for A/B of the plane kernels: cfg4's layered model at n^3
(+ PML 10), 6 Hz, the first b sources in one batched helm_solve (rtol 1e-6), one warm-up
solve then `reps` timed ones (CUDA events). Prints one JSON line with ms per solve batch,
outer cycles, algorithmic bytes rate and the per-level kernel-class breakdown.

    python scripts/solve3d.py [n=96] [b=8] [c128|c64] [reps=2]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1703_09268_b200 import api  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 96
b = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dt = api.C64 if (len(sys.argv) > 3 and sys.argv[3] == "c64") else api.C128
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
p = synth.cfg4(n=n)
w = 2 * np.pi * p.freqs[0]
op = api.helm_setup(api.Grid.of(p), p.m, w, api.Pml(v_ref=4500.0), dt, max_rhs=b)
td = torch.complex128 if dt == api.C128 else torch.complex64
B = torch.zeros(b, p.n_ext, dtype=td, device="cuda")
nx, ny, nz = p.next
for s in range(b):
    node = int(p.src[s])
    ix, iy, iz = node % p.n[0], (node // p.n[0]) % p.n[1], node // (p.n[0] * p.n[1])
    B[s, ((iz + p.pml[2][0]) * ny + iy + p.pml[1][0]) * nx + ix + p.pml[0][0]] = 1.0 / p.h**3
X = torch.empty_like(B)
rep = api.helm_solve(op, B, X, opts=api.SolveOpts(rtol=1e-6))
torch.cuda.synchronize()
api.profile(True, 3)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    rep = api.helm_solve(op, B, X, opts=api.SolveOpts(rtol=1e-6))
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
levels = {}
for lv in range(4):
    pr = api.profile_read(lv)
    row = {k: [round(v["ms"] * v["launches"] / v["sampled"] / reps, 2), round(v["bytes"] / max(v["ms"], 1e-9) / 1e6)]
           for k, v in pr.items() if v["sampled"]}
    if row:
        levels[lv] = row
api.profile(False, 1)
byts = sum(r["bytes_alg"] for r in rep)
print(json.dumps({"n": n, "b": b, "dtype": "c64" if dt == api.C64 else "c128", "lib": os.environ.get("HELM_LIB_VARIANT", "cur"),
                  "ms": round(ms, 2), "cycles": [r["outer_cycles"] for r in rep],
                  "converged": all(r["converged"] for r in rep), "GBps": round(byts / (ms / 1e3) / 1e9),
                  "levels": levels}))
