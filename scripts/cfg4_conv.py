"""Convergence diagnosis of BASELINE configs[3] (cfg4): outer FGMRES cycles of the forward and
adjoint solves for a given PML width and hierarchy depth.

Forward RHS: the first `nsrc` surface point sources q = e_s / h^3 (D7). Adjoint RHS: seeded
unit-variance complex noise on the receiver plane (z = 2, every interior node), the shape of
-P_r^T r. Prints one JSON line: cycles per RHS, solve times, points per wavelength per level.

    python scripts/cfg4_conv.py [--n 200] [--pml 10] [--levels 3] [--nsrc 8] [--dtype c128]
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

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=200)
ap.add_argument("--pml", type=int, default=10)
ap.add_argument("--levels", type=int, default=3)
ap.add_argument("--nsrc", type=int, default=8)
ap.add_argument("--dtype", default="c128")
ap.add_argument("--model", default="m0", choices=["m0", "mtrue"])
ap.add_argument("--max-outer", type=int, default=80)
a = ap.parse_args()

p = synth.cfg4(n=a.n, pml=a.pml)
grid = api.Grid.of(p)
f = p.freqs[0]
w = 2 * np.pi * f
dt = api.C64 if a.dtype == "c64" else api.C128
m = p.m if a.model == "m0" else p.m_true
op = api.helm_setup(grid, m, w, api.Pml(v_ref=4500.0), dt, max_rhs=a.nsrc, mlopts=api.MlOpts(levels=a.levels))
levels = op.levels()
Nx, Ny, Nz = p.next
td = api.TORCH_DTYPE[dt]
B = torch.zeros(a.nsrc, Nz, Ny, Nx, dtype=td)
for s, node in enumerate(p.src[:a.nsrc]):
    ix, iy, iz = node % p.n[0], (node // p.n[0]) % p.n[1], node // (p.n[0] * p.n[1])
    B[s, iz + a.pml, iy + a.pml, ix + a.pml] = 1.0 / p.h**3
A = torch.zeros_like(B)
rng = np.random.default_rng(1)
noise = (rng.standard_normal((a.nsrc, p.n[1], p.n[0])) + 1j * rng.standard_normal((a.nsrc, p.n[1], p.n[0]))) * np.sqrt(0.5)
A[:, 2 + a.pml, a.pml:a.pml + p.n[1], a.pml:a.pml + p.n[0]] = torch.from_numpy(noise).to(td)
B, A = B.cuda(), A.cuda()
X = torch.empty_like(B)
opts = api.SolveOpts(rtol=1e-6, max_outer=a.max_outer)
out = {"n": a.n, "pml": a.pml, "levels": a.levels, "levels_dims": levels, "dtype": a.dtype, "model": a.model,
       "nsrc": a.nsrc}
for name, rhs, adj in (("forward", B, 0), ("adjoint", A, 1)):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = api.helm_solve(op, rhs, X, adjoint=adj, opts=opts)
    torch.cuda.synchronize()
    out[name] = {"cycles": [r["outer_cycles"] for r in rep], "converged": all(r["converged"] for r in rep),
                 "s": round(time.perf_counter() - t0, 2), "rel": max(r["rel_residual"] for r in rep)}
# points per wavelength per level at v_min / v_max (h_l = 2^l h)
vmin, vmax = 1500.0 * 0.95, 4500.0 * 1.05
out["ppw"] = [{"level": l, "h": p.h * 2**l, "ppw_vmin": round(vmin / f / (p.h * 2**l), 2),
               "ppw_vmax": round(vmax / f / (p.h * 2**l), 2)} for l in range(len(levels))]
out["pml_wavelengths"] = {"vmin": round(a.pml * p.h / (1500.0 / f), 2), "vmax": round(a.pml * p.h / (4500.0 / f), 2)}
print(json.dumps(out), flush=True)
