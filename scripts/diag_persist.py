"""Diagnostic: medium3d solves with the persistent coarse V-cycle (HELM_PERSIST=1) — outer
cycles and residuals per RHS, c128 and c64 (same case as tests/test_gpu_paths.py)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from oracle import discretize as D  # noqa: E402
from oracle.solve import rel_residual  # noqa: E402
from paper_1703_09268_b200 import api  # noqa: E402
from tests.test_gpu_operator import medium3d  # noqa: E402

p = medium3d()
w = 2 * np.pi * p.freqs[0]
pml = D.PmlParams(v_ref=float(np.max(1 / np.sqrt(p.m))) * 1.1)
H = D.helmholtz_matrix(p, w, pml)
out = {"env": {k: v for k, v in os.environ.items() if k.startswith("HELM_")}}
for name, dt, td in (("c128", api.C128, torch.complex128), ("c64", api.C64, torch.complex64)):
    op = api.helm_setup(api.Grid.of(p), p.m, w, api.Pml(pml.R, pml.power, pml.v_ref), dt, max_rhs=3)
    b = np.zeros((3, p.n_ext), np.complex128)
    b[np.arange(3), [p.n_ext // 2, p.n_ext // 3, p.n_ext // 5]] = 1.0
    X = torch.empty(3, p.n_ext, dtype=td, device="cuda")
    rep = api.helm_solve(op, torch.from_numpy(b).to(td).cuda(), X, opts=api.SolveOpts(rtol=1e-6))
    Xh = X.cpu().numpy().astype(np.complex128)
    out[name] = {"cycles": [r["outer_cycles"] for r in rep], "rel": [r["rel_residual"] for r in rep],
                 "oracle_rel": [rel_residual(H, Xh[r], b[r]) for r in range(3)]}
print(json.dumps(out))
