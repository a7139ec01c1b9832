"""BASELINE configs[2] (cfg3): 3D constant velocity 64^3 + PML 10, 8 Hz, preconditioned FGMRES to
rel. residual 1e-6 — device time of one solve (1 RHS, centred source) and of the 8-source batch
(CUDA events, after one untimed solve). One JSON line."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1703_09268_b200 import api  # noqa: E402

out = {"env": {k: v for k, v in os.environ.items() if k.startswith("HELM_")}}
hbm = 6548.2
for name, p, vref in (("single", synth.cfg3(), 2000.0), ("batch8", synth.cfg3_batch(8), 2000.0),
                      ("table3_5x6", synth.table3(5, 6), 2000.0)):
    w = 2 * np.pi * p.freqs[0]
    b = len(p.src)
    pml = p.pml[0][0]
    for dt, tag in ((api.C128, "c128"), (api.C64, "c64")):
        op = api.helm_setup(api.Grid.of(p), p.m, w, api.Pml(v_ref=vref), dt, max_rhs=b)
        td = torch.complex128 if dt == api.C128 else torch.complex64
        B = torch.zeros(b, p.n_ext, dtype=td, device="cuda")
        nx, ny, nz = p.next
        for s, node in enumerate(p.src):
            node = int(node)
            ix, iy, iz = node % p.n[0], (node // p.n[0]) % p.n[1], node // (p.n[0] * p.n[1])
            B[s, ((iz + pml) * ny + iy + pml) * nx + ix + pml] = 1.0 / p.h**3
        X = torch.empty_like(B)
        api.helm_solve(op, B, X)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = api.launch_count()
        e0.record()
        rep = api.helm_solve(op, B, X)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        byts = sum(r["bytes_alg"] for r in rep)
        out[f"{name}_{tag}"] = {"ms": round(ms, 2), "solves_per_s": round(b / (ms / 1e3), 1),
                                "cycles": [r["outer_cycles"] for r in rep],
                                "rel_res_max": max(r["rel_residual"] for r in rep),
                                "launches": api.launch_count() - l0,
                                "alg_GBps": round(byts / (ms / 1e3) / 1e9, 1),
                                "hbm_frac": round(byts / (ms / 1e3) / 1e9 / hbm, 4)}
        del op
print(json.dumps(out))
