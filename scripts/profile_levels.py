"""Per-level, per-kernel-class device time of one cfg2 FWI evaluation (diagnostic).

    python scripts/profile_levels.py [--dtype c128|c64] [--freq 5] [--nsrc 50]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1703_09268_b200 import api  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="c128")
    ap.add_argument("--freq", type=float, default=0.0, help="one frequency (0 = the cfg2 set 3,5,7 Hz)")
    ap.add_argument("--nsrc", type=int, default=50)
    ap.add_argument("--max-rhs", type=int, default=0)
    ap.add_argument("--stride", type=int, default=1)
    a = ap.parse_args()
    p = synth.cfg2(nsrc=a.nsrc, freqs=(a.freq,) if a.freq > 0 else (3.0, 5.0, 7.0))
    mr = a.max_rhs if a.max_rhs > 0 else a.nsrc * len(p.freqs)
    grid = api.Grid.of(p)
    pml = api.Pml(v_ref=3000.0)
    dt = api.C64 if a.dtype == "c64" else api.C128
    d, _ = api.fwi_forward(grid, p.m_true, p.freqs, p.src, p.rec, pml, api.C128, api.SolveOpts(rtol=1e-8), max_rhs=mr)
    api.fwi_misfit_grad(grid, p.m, p.freqs, p.src, p.rec, d, pml, dt, max_rhs=mr)   # warm
    torch.cuda.synchronize()
    api.profile(True, a.stride)
    t0 = time.perf_counter()
    fg, rep = api.fwi_misfit_grad(grid, p.m, p.freqs, p.src, p.rec, d, pml, dt, max_rhs=mr)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    out = {"wall_s": wall, "cycles": sorted({r["outer_cycles"] for r in rep}), "levels": {}}
    tot = 0.0
    for lvl in range(5):
        pr = api.profile_read(lvl)
        row = {}
        for k, v in pr.items():
            if v["launches"]:
                est = v["ms"] * v["launches"] / max(v["sampled"], 1)
                tot += est
                row[k] = {"launches": v["launches"], "est_ms": round(est, 2),
                          "avg_us": round(1e3 * v["ms"] / max(v["sampled"], 1), 2),
                          "GBps": round(v["bytes"] / max(v["ms"], 1e-9) / 1e6, 1)}
        if row:
            out["levels"][lvl] = row
    out["gpu_est_s"] = tot / 1e3
    api.profile(False, 1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
