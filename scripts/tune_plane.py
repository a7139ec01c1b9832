"""Per-level kernel timings (back-to-back launches, helm_probe_kernel) for tuning the plane
kernel's ring depth / occupancy. Run under different HELM_PLANE_OCC / HELM_PLANE_S.

    python scripts/tune_plane.py [cfg2|cfg3|mv256] [c128|c64]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1703_09268_b200 import api  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
dt = api.C64 if (len(sys.argv) > 2 and sys.argv[2] == "c64") else api.C128
nrhs_arg = int(sys.argv[3]) if len(sys.argv) > 3 else 0
if what == "cfg2":
    p, f, vref, nrhs = synth.cfg2(freqs=(5.0,)), 5.0, 3000.0, nrhs_arg or 50
elif what == "cfg3":
    p, f, vref, nrhs = synth.cfg3_batch(8), 8.0, 2000.0, 8
else:
    p, f, vref, nrhs = synth.cfg5(256), 6.0, 4500.0, 1
op = api.helm_setup(api.Grid.of(p), p.m, 2 * np.pi * f, api.Pml(v_ref=vref), dt, max_rhs=nrhs)
levels = op.levels()
Sc, Sr = (16, 8) if dt == api.C128 else (8, 4)
out = {"case": what, "nrhs": nrhs, "variant": os.environ.get("HELM_LIB_VARIANT", "cur"), "dtype": "c128" if dt == api.C128 else "c64", "env": {k: v for k, v in os.environ.items() if k.startswith("HELM_")},
       "rows": []}
kinds = [(0, 0, 2), (1, 0, 3), (3, 0, 2), (3, 1, 4), (3, 2, 5), (3, 3, 6), (4, 4, 6), (2, 2, 5), (10, 5, 7), (11, 2, 5), (11, 4, 7), (12, 0, 1)]
for l, (nx, ny, nz) in enumerate(levels):
    N = nx * ny * nz
    for kind, nv, nvec in kinds:
        if l == len(levels) - 1 and kind in (2, 11):
            continue
        try:
            ms = api.probe_kernel(op, l, kind, nv, nrhs, reps=40)
        except Exception as e:  # noqa: BLE001
            out["rows"].append({"level": l, "kind": kind, "nv": nv, "err": str(e)[:80]})
            continue
        by = N * nrhs * (nvec * Sc + (Sr if kind <= 4 else 0))
        out["rows"].append({"level": l, "kind": kind, "nv": nv, "us": round(ms * 1e3, 2),
                            "GBps": round(by / (ms * 1e-3) / 1e9, 1)})
# whole V-cycles per level (host-synchronised)
for l in range(len(levels) - 1):
    nx, ny, nz = levels[l]
    b = torch.randn(nrhs, nx * ny * nz, dtype=op.tdtype, device="cuda")
    z = torch.empty_like(b)
    api.helm_vcycle(op, b, z, level=l)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 3 if l == 0 else 10
    for _ in range(reps):
        api.helm_vcycle(op, b, z, level=l)
    torch.cuda.synchronize()
    out["rows"].append({"level": l, "vcycle_ms": round((time.perf_counter() - t0) / reps * 1e3, 3)})
print(json.dumps(out))
