"""Wall time of one level-0 V-cycle (cfg2 shape) vs the GPU time of its kernels.

    python scripts/vcycle_gap.py [nrhs] [reps]   -> prints wall ms per V-cycle and launches
Run once plainly, then under `ncu --metrics gpu__time_duration.sum` with -s/-c selecting one
V-cycle's launches; the gap fraction = 1 - sum(kernel ms) / wall ms.
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

nrhs = int(sys.argv[1]) if len(sys.argv) > 1 else 50
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
p = synth.cfg2(freqs=(5.0,))
op = api.helm_setup(api.Grid.of(p), p.m, 2 * np.pi * 5.0, api.Pml(v_ref=3000.0), api.C128, max_rhs=nrhs)
b = torch.randn(nrhs, p.n_ext, dtype=torch.complex128, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
z = torch.empty_like(b)
api.helm_vcycle(op, b, z)
torch.cuda.synchronize()
l0 = api.launch_count()
t0 = time.perf_counter()
for _ in range(reps):
    api.helm_vcycle(op, b, z)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / reps
print(json.dumps({"nrhs": nrhs, "wall_ms": wall * 1e3, "launches_per_vcycle": (api.launch_count() - l0) / reps}))
