"""Write the cfg3 (BASELINE configs[2]) reference solutions used by tests/test_gpu_cfg3.py.

Calls only oracle/ and synth/ (SURVEY c.2 step 3 "otherwise"): the oracle's ML-GMRES mirror
(oracle/mlgmres.py, the oracle's own accelerator for 3D sizes where LU is infeasible) solves
H u = q and H^H v = q to a true relative residual <= 1e-10 (fields solved to 1e-10),
and every field is certified by the oracle's own assembled H (c.2 step 6). With --cross-check
the single forward field is also solved by unpreconditioned GMRES(100) to 1e-10
(oracle.solve.gmres_solve, ~10 min) and the two references are compared.

Stored (tests/golden/cfg3/): the single-source forward and adjoint fields in full, rounded
to complex64 (adds <= 6e-8 relative error, far below the 1e-5 parity bar), and for the
8-source batch (synth.cfg3_batch) each field on 5 z-planes (both PML edges, two interior
planes and its own source plane), also complex64; meta.json records residuals, rounding errors and timings.

    python scripts/make_cfg3_reference.py [--cross-check] [--procs 8]
"""
import argparse
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tests", "golden", "cfg3")
VREF = 2000.0


def _solve(args):
    kind, s, adjoint = args
    import synth
    from oracle import discretize as D
    from oracle import fwi, mlgmres
    from oracle.solve import rel_residual
    p = synth.cfg3() if kind == "single" else synth.cfg3_batch(8)
    w = 2 * np.pi * p.freqs[0]
    pml = D.PmlParams(v_ref=VREF)
    hier = mlgmres.Hierarchy(p, w, pml)
    q = fwi.source_matrix(p, w, p.src[s:s + 1])[:, 0]
    t0 = time.perf_counter()
    u, cycles, rel = mlgmres.solve(hier, q, rtol=1e-10, adjoint=adjoint, max_outer=40)
    dt = time.perf_counter() - t0
    H = D.helmholtz_matrix(p, w, pml)
    cert = rel_residual(H, u, q, adjoint=adjoint)
    return kind, s, adjoint, u, {"cycles": int(cycles), "rel_residual": float(cert), "solve_s": round(dt, 1)}


FIXED_PLANES = (0, 36, 59, 83)      # both PML edges and two interior planes of the 84^3 grid


def planes_for(p):
    """Per RHS: the fixed planes plus the plane of its own source (padded to 5 with z = 47)."""
    out = []
    for node in p.src:
        ps = set(FIXED_PLANES) | {int(node) // (p.n[0] * p.n[1]) + p.pml[2][0]}
        if len(ps) < 5:
            ps.add(47)
        out.append(sorted(ps))
    return np.array(out, np.int64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cross-check", action="store_true")
    ap.add_argument("--procs", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    import synth
    os.makedirs(OUT, exist_ok=True)
    jobs = [("single", 0, False), ("single", 0, True)] + [("batch", s, adj) for adj in (False, True) for s in range(8)]
    with mp.get_context("fork").Pool(a.procs) as pool:
        res = pool.map(_solve, jobs)
    meta = {"how": "oracle/mlgmres.py solve (ML-GMRES mirror, FGMRES(5) outer) to rtol 1e-10, certified by "
                   "oracle.solve.rel_residual with oracle.discretize.helmholtz_matrix; stored rounded to complex64",
            "rtol": 1e-10, "pml_v_ref": VREF, "fields": {}}
    pb = synth.cfg3_batch(8)
    planes = planes_for(pb)
    Nx, Ny, Nz = pb.next
    slabs = {False: np.zeros((8, planes.shape[1], Ny, Nx), np.complex64),
             True: np.zeros((8, planes.shape[1], Ny, Nx), np.complex64)}
    u_single = None
    for kind, s, adj, u, info in res:
        u64 = u.astype(np.complex64)
        info["rounded_rel_err"] = float(np.linalg.norm(u64.astype(np.complex128) - u) / np.linalg.norm(u))
        name = f"{kind}_{'adj' if adj else 'fwd'}" + (f"_{s}" if kind == "batch" else "")
        meta["fields"][name] = info
        if kind == "single":
            np.save(os.path.join(OUT, f"single_{'adj' if adj else 'fwd'}.npy"), u64.reshape(Nz, Ny, Nx))
            if not adj:
                u_single = u
        else:
            slabs[adj][s] = u64.reshape(Nz, Ny, Nx)[planes[s]]
    np.savez(os.path.join(OUT, "batch8_slabs.npz"), z_planes=planes, fwd=slabs[False], adj=slabs[True])
    if a.cross_check:
        from oracle import discretize as D
        from oracle import fwi
        from oracle.solve import gmres_solve
        p = synth.cfg3()
        w = 2 * np.pi * p.freqs[0]
        H = D.helmholtz_matrix(p, w, D.PmlParams(v_ref=VREF))
        q = fwi.source_matrix(p, w, p.src)[:, 0]
        t0 = time.perf_counter()
        ug = gmres_solve(H, q, rtol=1e-10, restart=100, maxiter=100)
        meta["gmres_cross_check"] = {"field": "single_fwd", "solver": "oracle.solve.gmres_solve GMRES(100), rtol 1e-10",
                                     "rel_diff": float(np.linalg.norm(ug - u_single) / np.linalg.norm(ug)),
                                     "solve_s": round(time.perf_counter() - t0, 1)}
    with open(os.path.join(OUT, "meta.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(json.dumps(meta, indent=1))


if __name__ == "__main__":
    main()
