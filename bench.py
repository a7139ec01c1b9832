#!/usr/bin/env python
"""bench.py — one JSON line for the driver.

A step = one full pass of the hot path: fwi_misfit_grad over this
rank's shots of BASELINE configs[1] (2D FWI, 401x201 + PML 20, 50 shots x 3 frequencies,
401 receivers) = 300 preconditioned solves (150 forward + 150 adjoint), then one NCCL
all_reduce of [f || g]. Weak scaling: rank r fires its own 50 shots (x = 4 + 8k + r), so the
per-GPU work is fixed as N grows; at N = 1 the workload is exactly configs[1].

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--dtype c128|c64] [--workload cfg2|cfg3]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Helmholtz matvec Gpts/s and % HBM roofline; preconditioned solves/s per GPU at 1/2/4/8"
FALLBACK_HBM = 6650.0


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


# ----------------------------------------------------------------------------- workload
def workload(name: str, rank: int):
    import synth
    if name == "cfg2":
        p = synth.cfg2()
        n = p.n
        src = synth.node_id(4 + 8 * np.arange(50) + (rank % 8), 0, 2, n)
        desc = ("cfg2 (BASELINE configs[1]): 2D FWI misfit+gradient, 401x201 interior + PML 20 "
                "(441x241 ext), h=10 m, v 1500-4000 m/s + 8 seeded blobs, 50 shots x {3,5,7} Hz, 401 receivers")
        return p.with_(src=src), desc, 3000.0 * 1.0
    if name == "cfg3":
        p = synth.cfg3_batch(8)
        desc = "cfg3 batch: 3D constant 64^3 + PML 10 (84^3 ext), 8 sources, f=8 Hz (forward solves only)"
        return p, desc, 2000.0
    raise SystemExit(f"unknown workload {name}")


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int):
        self.dev, self.rows, self.proc = dev, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.dev)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for nm, v in zip(names, r[2:6]):
                    if v.lower() in ("active", "1", "yes"):
                        reasons.add(nm)
            except (ValueError, IndexError):
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- our arm
def run_ours(args, rank, size, dev):
    import torch
    import torch.distributed as dist

    from paper_1703_09268_b200 import api
    from paper_1703_09268_b200 import dist as hdist

    prob, desc, vref = workload(args.workload, rank)
    dtype = api.C64 if args.dtype == "c64" else api.C128
    grid = api.Grid.of(prob)
    pml = api.Pml(v_ref=vref)
    opts = api.SolveOpts(rtol=1e-6)
    nsrc = len(prob.src)
    # joint (source, frequency) batches: by default one batch holds every pair
    max_rhs = args.max_rhs if args.max_rhs > 0 else nsrc * len(prob.freqs)
    stream = torch.cuda.current_stream()

    # observed data from the true model (untimed): Listing 1 FORW_MODEL on this rank's shots
    d_obs, _ = api.fwi_forward(grid, prob.m_true, prob.freqs, prob.src, prob.rec, pml, api.C128,
                               api.SolveOpts(rtol=1e-8), max_rhs=max_rhs)
    fg = torch.empty(1 + grid.n_interior, dtype=torch.float64, device="cuda")

    def step(fg_out, host_roundtrip=False):
        fg2, rep = api.fwi_misfit_grad(grid, prob.m, prob.freqs, prob.src, prob.rec, d_obs, pml, dtype, opts,
                                       max_rhs=max_rhs, fg=fg_out)
        if size > 1:
            dist.all_reduce(fg2, op=dist.ReduceOp.SUM)
        if host_roundtrip:
            return fg2.cpu(), rep
        return fg2, rep

    reps = None
    for _ in range(args.warmup):
        _, reps = step(fg)
    solves_per_step = 2 * nsrc * len(prob.freqs)

    def timed(k, host_roundtrip=False, profile=False):
        if size > 1:
            dist.barrier()
        torch.cuda.synchronize()
        if profile:
            api.profile(True, args.probe_stride)
        l0 = api.launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rep = None
        for _ in range(k):
            _, rep = step(fg, host_roundtrip)
        e1.record(stream)
        torch.cuda.synchronize()
        launches = api.launch_count() - l0
        ms = e0.elapsed_time(e1)
        if size > 1:
            t = torch.tensor([ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            dist.barrier()
        return ms, launches, rep

    with ClockSampler(dev) as clk:
        ms, launches, reps = timed(args.steps)
    # kernel-class shares and the live roofline of the dominant class: one more step with
    # every `probe_stride`-th launch bracketed by CUDA events (not part of `value`)
    timed(1, profile=True)
    prof = api.profile_read()
    prof_lv = {lv: api.profile_read(lv) for lv in range(4)}
    api.profile(False, 1)
    ms_e2e, _, _ = timed(max(1, min(args.steps, 2)), host_roundtrip=True)
    k_e2e = max(1, min(args.steps, 2))

    value = solves_per_step * size * args.steps / (ms / 1e3)
    e2e_value = solves_per_step * size * k_e2e / (ms_e2e / 1e3)
    hbm, peak_kind = peaks()

    # shares of device time per kernel class, and the dominant (class, level) pair: its live
    # roofline is algorithmic bytes / event-timed duration over its sampled launches
    est = {}
    for name, p in prof.items():
        if p["sampled"]:
            est[name] = p["ms"] * p["launches"] / p["sampled"]
    total_est = sum(est.values()) or 1.0
    kernel_shares = {k: round(v / total_est, 3) for k, v in sorted(est.items(), key=lambda kv: -kv[1])}
    cl = {}
    for lv, pr in prof_lv.items():
        for name, p in pr.items():
            if p["sampled"]:
                cl[(name, lv)] = p
    def est_ms(p):
        return p["ms"] * p["launches"] / p["sampled"]
    roof = None
    level_shares = {}
    for (name, lv), p in cl.items():
        level_shares.setdefault(f"L{lv}", 0.0)
        level_shares[f"L{lv}"] += est_ms(p) / total_est
    level_shares = {k: round(v, 3) for k, v in sorted(level_shares.items())}
    if cl:
        (dname, dlv), p = max(cl.items(), key=lambda kv: est_ms(kv[1]))
        achieved = p["bytes"] / (p["ms"] / 1e3) / 1e9
        tr = traffic_for(f"{dname}@L{dlv}")
        roof = {"kernel": f"{dname} (fused GMRES Arnoldi step, k_march2d MODE 3/4) at level {dlv}" if dname == "arnoldi"
                else f"{dname} at level {dlv}", "bound": "hbm", "achieved": round(achieved, 1), "peak": hbm,
                "unit": "GB/s", "frac": round(achieved / hbm, 4),
                "traffic": round(tr["ratio"] * p["bytes"] / p["sampled"]) if tr else None,
                "traffic_note": tr.get("note") if tr else None,
                "peak_kind": peak_kind, "share_of_step": round(est_ms(p) / total_est, 3),
                "avg_launch_us": round(1e3 * p["ms"] / p["sampled"], 2),
                "alg_bytes_per_launch": round(p["bytes"] / p["sampled"]), "sampled_launches": p["sampled"]}
        cls_all = prof[dname]
        roof["class_all_levels"] = {"achieved": round(cls_all["bytes"] / (cls_all["ms"] / 1e3) / 1e9, 1),
                                    "share_of_step": kernel_shares.get(dname)}

    cycles = [r["outer_cycles"] for r in (reps or [])]
    # whole-step algorithmic HBM bytes counted by the library (every executed kernel, SURVEY d.2)
    step_bytes = sum(r["bytes_alg"] for r in (reps or []))
    solve_roof = {"alg_bytes_per_step": step_bytes, "achieved_GBps": round(step_bytes / (ms / args.steps / 1e3) / 1e9, 1),
                  "frac": round(step_bytes / (ms / args.steps / 1e3) / 1e9 / peaks()[0], 4)}
    h2d = 8 * grid.n_interior + 16 * d_obs.size + 8 * (nsrc + len(prob.rec)) + 16 * len(prob.freqs)
    d2h = 8 * (1 + grid.n_interior)
    out = {
        "metric": METRIC, "value": round(value, 3), "unit": "solves/s", "n_gpus": size, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": "c128" if dtype == api.C128 else "c64 (mixed: c128 outer FGMRES)",
        "data": "synthetic (seeded generators, synth/)",
        "config": {"workload": desc, "solves_per_step_per_gpu": solves_per_step, "rtol": opts.rtol,
                   "precond": "ML-GMRES (3,5,3,5), 3 grids, outer FGMRES(5)", "max_rhs": max_rhs,
                   "batching": "joint (source, frequency) batches of max_rhs RHS (P:141)",
                   "l2": "no flush: working set %.1f GB > 126 MB L2" % (ws_bytes(grid, dtype, max_rhs) / 1e9),
                   "parallelism": f"dp{size} (source shards, one fp64 NCCL all_reduce per step)",
                   "outer_cycles_last_step": {"min": min(cycles), "max": max(cycles)} if cycles else None},
        "e2e": {"value": round(e2e_value, 3), "unit": "solves/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": int(launches),
        "roofline": roof,
        "kernel_shares": kernel_shares,
        "level_shares": level_shares,
        "solve_roofline": solve_roof,
        "clocks": clk.summary(),
    }
    return out, prob


def ws_bytes(grid, dtype, max_rhs):
    sc = 16 if dtype == 1 else 8
    return 24 * grid.n_ext * max_rhs * sc


def traffic_for(key):
    """DRAM traffic / algorithmic bytes of a (class, level) pair from the committed ncu --set full
    capture (profiles/ncu_traffic.json, written from the capture's dram__bytes_read.sum +
    dram__bytes_write.sum of the same kernels), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(key)
    except Exception:
        return None


def matvec_probe(dtype_name="c128", N=256, nrhs=1, reps=10):
    """a2 alone on BASELINE configs[4] (cfg5 N^3): Gpts/s with 3 rotating buffer sets > 2 x L2."""
    import torch

    import synth
    from paper_1703_09268_b200 import api
    p = synth.cfg5(N)
    dtype = api.C128 if dtype_name == "c128" else api.C64
    op = api.helm_setup(api.Grid.of(p), p.m, 2 * np.pi * 6.0, api.Pml(v_ref=4500.0), dtype, max_rhs=nrhs,
                        mlopts=api.MlOpts(levels=0))   # operator only: no solver workspace
    td = torch.complex128 if dtype == api.C128 else torch.complex64
    g = torch.Generator(device="cuda").manual_seed(1)
    n_ext = p.n_ext
    sets = max(3, int(np.ceil(2 * 126e6 / (2 * n_ext * nrhs * (16 if dtype == api.C128 else 8)))) + 1)
    xs = [torch.randn(nrhs, n_ext, dtype=td, device="cuda", generator=g) for _ in range(sets)]
    ys = [torch.empty_like(xs[0]) for _ in range(sets)]
    for i in range(3):
        api.helm_apply(op, xs[i % sets], ys[i % sets])
    torch.cuda.synchronize()
    times = []
    for i in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        api.helm_apply(op, xs[i % sets], ys[i % sets])
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    t = statistics.median(times) / 1e3
    sc, sr = (16, 8) if dtype == api.C128 else (8, 4)
    gpts = n_ext * nrhs / t / 1e9
    gbs = n_ext * (2 * sc * nrhs + sr) / t / 1e9
    hbm, _ = peaks()
    return {"workload": f"cfg5 {N}^3 {dtype_name} b={nrhs}", "gpts": round(gpts, 2), "gb_s": round(gbs, 1),
            "hbm_frac": round(gbs / hbm, 4), "ms": round(t * 1e3, 4), "best_ms": round(min(times), 4)}


# ----------------------------------------------------------------------------- oracle arm
def oracle_step(prob, d, fi, pml):
    """One bounded sample of the workload on the host: the oracle's misfit+gradient for one
    frequency over all shots (LU factorization + forward and adjoint triangular solves)."""
    from oracle import fwi
    p1 = prob.with_(freqs=(prob.freqs[fi],))
    t0 = time.perf_counter()
    fwi.misfit_grad(p1, pml, d[fi:fi + 1])
    return time.perf_counter() - t0, 2 * len(prob.src)


def cpu_baseline(prob, pml_o, d=None):
    from oracle import fwi
    if d is None:
        d = fwi.forward_data(prob.with_(freqs=(prob.freqs[1],)), pml_o, prob.m_true)
        fi = 0
        p = prob.with_(freqs=(prob.freqs[1],))
    else:
        fi, p = 1, prob
    dt, n = oracle_step(p, d, fi, pml_o)
    return {"value": round(n / dt, 4), "unit": "solves/s", "cores": 1, "kind": "oracle",
            "sample": f"oracle (scipy SuperLU, 1 thread) misfit+gradient of {p.name} at {p.freqs[fi]} Hz over "
                      f"{len(prob.src)} shots = {n} solves in {dt:.1f} s"}


def run_reference(args, rank, size):
    if rank != 0:
        return None
    from oracle import discretize as D
    from oracle import fwi
    prob, desc, vref = workload(args.workload, 0)
    pml_o = D.PmlParams(v_ref=vref)
    d = fwi.forward_data(prob, pml_o, prob.m_true)
    steps = []
    total = args.warmup + args.steps
    for i in range(total):
        dt, n = oracle_step(prob, d, i % len(prob.freqs), pml_o)
        if i >= args.warmup:
            steps.append((dt, n))
    t = sum(s[0] for s in steps)
    n = sum(s[1] for s in steps)
    value = n / t
    return {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "solves/s", "n_gpus": size,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * t / args.steps, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (seeded generators, synth/)",
        "config": {"workload": desc + " — each step one frequency (100 solves) of it",
                   "solves_per_step_per_gpu": 2 * len(prob.src)},
        "cpu_baseline": {"value": round(value, 4), "unit": "solves/s", "cores": 1, "kind": "oracle",
                         "sample": "oracle misfit+gradient, one frequency x 50 shots per step (SuperLU, 1 thread)"},
        "e2e": {"value": round(value, 4), "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


# ----------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dtype", default="c128", choices=["c128", "c64"])
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--max-rhs", type=int, default=0, help="RHS per joint batch (0 = all pairs)")
    ap.add_argument("--probe-stride", type=int, default=7)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-matvec", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    size = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        out = run_reference(args, rank, size)
        if out is not None:
            print(json.dumps(out), flush=True)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if size > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    out, prob = run_ours(args, rank, size, local)
    if rank == 0:
        if size == 1 and not args.no_matvec:
            out["matvec"] = {k: matvec_probe(*k_) for k, k_ in
                             (("c128_b1_256", ("c128", 256, 1)), ("c128_b1_512", ("c128", 512, 1)),
                              ("c128_b4_256", ("c128", 256, 4)), ("c64_b4_256", ("c64", 256, 4)))}
        if size == 1 and not args.no_cpu_baseline:
            from oracle import discretize as D
            out["cpu_baseline"] = cpu_baseline(prob, D.PmlParams(v_ref=3000.0))
        print(json.dumps(out), flush=True)
    if size > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
