"""Diagnose the deep-2D joint-batch case: matvec and solve parity on a 2D grid with
nz_ext = 1000, and misfit/gradient per frequency vs the oracle."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from oracle import discretize as D, fwi
from oracle.solve import LU
from paper_1703_09268_b200 import api
nz = int(sys.argv[1]) if len(sys.argv) > 1 else 960
p = synth.tiny2d(nx=40, nz=nz, pml=20, nsrc=2).with_(freqs=(6.0, 8.0, 10.0, 12.0))
pml = D.PmlParams(v_ref=3000.0)
out = {"nz_ext": p.next[2]}
def rel(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))
w = 2 * np.pi * 12.0
H = D.helmholtz_matrix(p, w, pml)
op = api.helm_setup(api.Grid.of(p), p.m, w, api.Pml(v_ref=3000.0), api.C128, max_rhs=2)
x = synth.random_complex((2, p.n_ext), 1)
y = torch.empty(2, p.n_ext, dtype=torch.complex128, device="cuda")
api.helm_apply(op, torch.from_numpy(x).cuda(), y)
out["apply"] = rel(y.cpu().numpy()[0], H @ x[0])
q = fwi.source_matrix(p, w, p.src)
X = torch.empty(2, p.n_ext, dtype=torch.complex128, device="cuda")
for adj in (0, 1):
    rep = api.helm_solve(op, torch.from_numpy(np.ascontiguousarray(q.T)).cuda(), X, adjoint=adj, opts=api.SolveOpts(rtol=1e-8, max_outer=200))
    U = LU(H).solve(q, adjoint=bool(adj)).T
    out[f"solve{adj}"] = [rel(X.cpu().numpy()[r], U[r]) for r in range(2)]
    out[f"cyc{adj}"] = [r["outer_cycles"] for r in rep]
d = fwi.forward_data(p, pml, p.m_true)
for fi in range(4):
    p1 = p.with_(freqs=(p.freqs[fi],))
    f_ref, g_ref = fwi.misfit_grad(p1, pml, d[fi:fi+1])
    fg, rep = api.fwi_misfit_grad(api.Grid.of(p1), p1.m, p1.freqs, p1.src, p1.rec, d[fi:fi+1], api.Pml(v_ref=3000.0),
                                  api.C128, api.SolveOpts(rtol=1e-8, max_outer=200), max_rhs=8)
    fg = fg.cpu().numpy()
    out[f"freq{fi}"] = {"f": abs(fg[0] - f_ref) / f_ref, "g": rel(fg[1:], g_ref.ravel())}
f_ref, g_ref = fwi.misfit_grad(p, pml, d)
for mr in (2, 4, 6, 8):
    fg, rep = api.fwi_misfit_grad(api.Grid.of(p), p.m, p.freqs, p.src, p.rec, d, api.Pml(v_ref=3000.0), api.C128,
                                  api.SolveOpts(rtol=1e-8, max_outer=200), max_rhs=mr)
    fg = fg.cpu().numpy()
    out[f"joint_maxrhs{mr}"] = {"f": abs(fg[0] - f_ref) / f_ref, "g": rel(fg[1:], g_ref.ravel())}
print(json.dumps(out))
