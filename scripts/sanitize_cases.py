"""Small hot-path invocations for compute-sanitizer (memcheck / racecheck / synccheck):
cfg1 (2D march kernels), tiny3d (3D plane kernels, TMA stages, split-ring fused steps),
cfg3 single source and the 8-source batch (3D, one outer FGMRES cycle each, the second
and later V-cycles replayed from CUDA graphs), both precisions, forward and adjoint.

    compute-sanitizer --tool memcheck python scripts/sanitize_cases.py [case ...]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1703_09268_b200 import api  # noqa: E402


def solve(p, vref, dtype, nrhs, max_outer, adjoint):
    w = 2 * np.pi * p.freqs[0]
    op = api.helm_setup(api.Grid.of(p), p.m, w, api.Pml(v_ref=vref), dtype, max_rhs=nrhs)
    td = api.TORCH_DTYPE[dtype]
    b = torch.zeros(nrhs, p.n_ext, dtype=td)
    for r in range(nrhs):
        b[r, (p.n_ext // (r + 2)) | 1] = 1.0
    b = b.cuda()
    x = torch.empty_like(b)
    rep = api.helm_solve(op, b, x, adjoint=adjoint, opts=api.SolveOpts(rtol=1e-6, max_outer=max_outer))
    y = torch.empty_like(b)
    api.helm_apply(op, x, y, adjoint)
    torch.cuda.synchronize()
    return rep


CASES = {
    "cfg1": lambda: [solve(synth.cfg1(), 2000.0, dt, 1, 3, adj) for dt in (api.C128, api.C64) for adj in (0, 1)],
    "tiny3d": lambda: [solve(synth.tiny3d(n=(45, 37, 29)), 3000.0, dt, 3, 3, adj) for dt in (api.C128, api.C64)
                       for adj in (0, 1)],
    "cfg3": lambda: [solve(synth.cfg3(), 2000.0, api.C128, 1, 1, 0)],
    "cfg3b8": lambda: [solve(synth.cfg3_batch(8), 2000.0, api.C64, 8, 1, 1)],
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        reps = CASES[n]()
        print(n, "ok", flush=True)
