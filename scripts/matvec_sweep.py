"""a2 bandwidth sweep on BASELINE configs[4] (cfg5): N^3 in {128,256,384,512}, c64/c128,
RHS batch 1/4/16, unit-variance random input generated on the device (seed 1).
Timing: CUDA events on the launching stream, 3 warm-ups, median and best of 10, rotating
buffer sets whose total exceeds 2 x L2 (d.3). Prints one JSON line per case."""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1703_09268_b200 import api  # noqa: E402

HBM = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else 6650.0


def run(N, dt, b, adjoint=0, reps=10, stencil="std2"):
    p = synth.cfg5(N).with_(stencil=stencil)
    dtype = api.C128 if dt == "c128" else api.C64
    op = api.helm_setup(api.Grid.of(p), p.m, 2 * np.pi * 6.0, api.Pml(v_ref=4500.0), dtype, max_rhs=b,
                        mlopts=api.MlOpts(levels=0))
    td = torch.complex128 if dtype == api.C128 else torch.complex64
    sc, sr = (16, 8) if dtype == api.C128 else (8, 4)
    vec = p.n_ext * b * sc
    sets = max(1, min(4, int(np.ceil(2 * 2 * 126e6 / (2 * vec)))))
    g = torch.Generator(device="cuda").manual_seed(1)
    xs = [torch.randn(b, p.n_ext, dtype=td, device="cuda", generator=g) for _ in range(sets)]
    ys = [torch.empty_like(xs[0]) for _ in range(sets)]
    for i in range(3):
        api.helm_apply(op, xs[i % sets], ys[i % sets], adjoint)
    torch.cuda.synchronize()
    ts = []
    for i in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        api.helm_apply(op, xs[i % sets], ys[i % sets], adjoint)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    api.profile(True, 1)   # the kernel alone (library events around the launch on its stream)
    for i in range(reps):
        api.helm_apply(op, xs[i % sets], ys[i % sets], adjoint)
    torch.cuda.synchronize()
    pr = api.profile_read()["stencil"]
    api.profile(False, 1)
    tk = pr["ms"] / max(1, pr["sampled"]) / 1e3
    t = statistics.median(ts)
    bytes_ = p.n_ext * (2 * sc * b + sr)
    out = {"N": N, "dtype": dt, "b": b, "adjoint": adjoint, "stencil": stencil, "ms_median": t * 1e3, "ms_best": min(ts) * 1e3,
           "gpts": p.n_ext * b / t / 1e9, "GBps": bytes_ / t / 1e9, "frac_measured": bytes_ / t / 1e9 / HBM,
           "frac_8TBs": bytes_ / t / 8e12, "alg_bytes": bytes_, "ms_kernel": tk * 1e3, "gpts_kernel": p.n_ext * b / tk / 1e9,
           "frac_measured_kernel": bytes_ / tk / 1e9 / HBM, "frac_8TBs_kernel": bytes_ / tk / 8e12}
    del xs, ys, op
    torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", default="128,256,384,512")
    ap.add_argument("--dtype", default="c128,c64")
    ap.add_argument("--b", default="1,4,16")
    ap.add_argument("--stencil", default="std2")
    a = ap.parse_args()
    for N in [int(v) for v in a.N.split(",")]:
        for dt in a.dtype.split(","):
            for b in [int(v) for v in a.b.split(",")]:
                if N == 512 and b == 16 and dt == "c128":
                    pass
                print(json.dumps(run(N, dt, b, stencil=a.stencil)), flush=True)
