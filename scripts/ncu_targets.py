"""Small, deterministic launch sequences for ncu captures.

    python scripts/ncu_targets.py matvec [N] [c128|c64] [b]   # 4 x helm_apply on cfg5
    python scripts/ncu_targets.py cfg2                       # one cfg2 forward solve batch (5 Hz)
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1703_09268_b200 import api  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "matvec"
if what == "matvec":
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    dt = sys.argv[3] if len(sys.argv) > 3 else "c128"
    b = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    p = synth.cfg5(N)
    dtype = api.C128 if dt == "c128" else api.C64
    op = api.helm_setup(api.Grid.of(p), p.m, 2 * np.pi * 6.0, api.Pml(v_ref=4500.0), dtype, max_rhs=b,
                        mlopts=api.MlOpts(levels=0))
    td = torch.complex128 if dtype == api.C128 else torch.complex64
    x = torch.randn(b, p.n_ext, dtype=td, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
    y = torch.empty_like(x)
    for _ in range(4):
        api.helm_apply(op, x, y)
    torch.cuda.synchronize()
elif what == "cfg2":
    p = synth.cfg2(freqs=(5.0,))
    w = 2 * np.pi * 5.0
    op = api.helm_setup(api.Grid.of(p), p.m, w, api.Pml(v_ref=3000.0), api.C128, max_rhs=50)
    B = torch.zeros(50, p.n_ext, dtype=torch.complex128, device="cuda")
    nx = p.next[0]
    for s, node in enumerate(p.src):
        ix, iz = node % p.n[0], node // p.n[0]
        B[s, (iz + 20) * nx + ix + 20] = 1.0 / p.h**2
    X = torch.empty_like(B)
    api.helm_solve(op, B, X, opts=api.SolveOpts(max_outer=1))
    torch.cuda.synchronize()
elif what == "probe":
    # python scripts/ncu_targets.py probe cfg2|mv256 level kind nv  (5 launches of one kernel)
    case, level, kind, nv = sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
    if case == "cfg2":
        p, f, vref, nrhs = synth.cfg2(freqs=(5.0,)), 5.0, 3000.0, 50
    elif case == "cfg2_150":
        p, f, vref, nrhs = synth.cfg2(freqs=(5.0,)), 5.0, 3000.0, 150
    elif case.startswith("cfg4_"):   # cfg4 full size, nrhs = the suffix (bench: 8)
        p, f, vref, nrhs = synth.cfg4(), 6.0, 4500.0, int(case.split("_")[1])
    else:
        p, f, vref, nrhs = synth.cfg5(256), 6.0, 4500.0, 1
    dt = api.C64 if os.environ.get("PROBE_DTYPE") == "c64" else api.C128
    op = api.helm_setup(api.Grid.of(p), p.m, 2 * np.pi * f, api.Pml(v_ref=vref), dt, max_rhs=nrhs)
    print(api.probe_kernel(op, level, kind, nv, nrhs, reps=int(os.environ.get("PROBE_REPS", "4"))))
    torch.cuda.synchronize()
print("ok")
