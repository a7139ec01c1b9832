"""Per-kernel bandwidth table of the hot-path kernels on one level of an op (CUDA events,
`reps` back-to-back launches through helm_probe_kernel): algorithmic bytes (SURVEY d.2,
DESIGN §6) / average launch time, per (level, kernel).

    python scripts/probe_table.py [cfg4|cfg3|cfg2] [nrhs] [c128|c64] [levels...]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1703_09268_b200 import api  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dts = sys.argv[3] if len(sys.argv) > 3 else "c128"
lvls = [int(v) for v in sys.argv[4:]] or [0, 1, 2]
if case == "cfg4":
    p, f, vref = synth.cfg4(), 6.0, 4500.0
elif case == "cfg3":
    p, f, vref = synth.cfg3(), 8.0, 2000.0
else:
    p, f, vref = synth.cfg2(freqs=(5.0,)), 5.0, 3000.0
dt = api.C64 if dts == "c64" else api.C128
Sc, Sr = (8, 4) if dt == api.C64 else (16, 8)
op = api.helm_setup(api.Grid.of(p), p.m, 2 * np.pi * f, api.Pml(v_ref=vref), dt, max_rhs=nrhs)
dims = op.levels()
hbm = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))[
    "hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6548.2
kinds = [("matvec", 0, 0, 2 * Sc + Sr), ("resid", 1, 0, 3 * Sc + Sr)]
kinds += [(f"arnoldi{j}", 3, j, (2 if j == 0 else j + 3) * Sc + Sr) for j in range(4)]
# the last step stores V_4 only with HELM_LASTV=1 (3D; the solution update reforms it otherwise)
kinds += [("arnoldi4_last", 4, 4, (6 if os.environ.get("HELM_LASTV", "0") != "0" else 5) * Sc + Sr),
          ("solupdate5", 10, 5, 7 * Sc)]
kinds += [(f"fgmres{j + 1}", 2, j, (3 + j) * Sc + Sr) for j in (0, 2, 4)] + [("update2", 11, 2, 5 * Sc)]
for l in lvls:
    if l >= len(dims):
        continue
    N = int(np.prod(dims[l]))
    for name, kind, nv, per in kinds:
        if kind == 10 and l == len(dims) - 1:
            pass
        ms = api.probe_kernel(op, l, kind, nv, nrhs, reps=20)
        gbs = per * N * nrhs / (ms / 1e3) / 1e9
        print(json.dumps({"case": case, "dtype": dts, "nrhs": nrhs, "level": l, "dims": dims[l], "kernel": name,
                          "us": round(ms * 1e3, 1), "GBps": round(gbs, 1), "frac": round(gbs / hbm, 3)}), flush=True)
