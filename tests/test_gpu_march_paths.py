"""GPU parity of the 2D march kernel's two ring feeds, each in a fresh process (the switch is
read once per process): the TMA-fed ring (complex128: one elected lane per warp issues the
strip rows of every operand and m on a per-slot mbarrier; default for three or more streamed
operands on large levels, HELM_MARCH_TMA=2 everywhere) and the per-lane cp.async ring
(HELM_MARCH_TMA=0; always used for complex64, whose strips start at an odd, 8-B aligned point). On the ragged 2D grid of test_gpu_operator (medium2d) each must match the
assembled oracle H / H^H (c128 <= 1e-12, c64 <= 1e-5) for STD2 and the paper's 9-point
stencil (R34), give a certified preconditioned solve (rel. residual <= 1e-6 by the oracle's
H), and misfit / gradient on tiny2d that match the oracle's LU evaluation (<= 1e-5)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, numpy as np, torch
import synth
from oracle import discretize as D
from oracle import fwi
from oracle.solve import rel_residual
from paper_1703_09268_b200 import api
from tests.test_gpu_operator import medium2d
out = {}
for st in ("std2", "opt"):
    p = medium2d().with_(stencil=st)
    w = 2 * np.pi * p.freqs[0]
    pml = D.PmlParams(v_ref=float(np.max(1 / np.sqrt(p.m))) * 1.1)
    H = D.helmholtz_matrix(p, w, pml)
    for name, dt, td in (("c128", api.C128, torch.complex128), ("c64", api.C64, torch.complex64)):
        op = api.helm_setup(api.Grid.of(p), p.m, w, api.Pml(pml.R, pml.power, pml.v_ref), dt, max_rhs=3)
        x = synth.random_complex((3, p.n_ext), 1)
        for adj in (0, 1):
            A = D.helmholtz_adjoint_matrix(H) if adj else H
            y = torch.empty(3, p.n_ext, dtype=td, device="cuda")
            api.helm_apply(op, torch.from_numpy(x.astype(np.complex128)).to(td).cuda(), y, adj)
            yg = y.cpu().numpy().astype(np.complex128)
            xr = x.astype(np.complex64).astype(np.complex128) if name == "c64" else x
            out[f"{st}_{name}_apply{adj}"] = max(float(np.linalg.norm(yg[r] - A @ xr[r]) / np.linalg.norm(A @ xr[r]))
                                                 for r in range(3))
        b = np.zeros((3, p.n_ext), np.complex128)
        b[np.arange(3), [p.n_ext // 2, p.n_ext // 3, p.n_ext // 5]] = 1.0
        X = torch.empty(3, p.n_ext, dtype=td, device="cuda")
        rep = api.helm_solve(op, torch.from_numpy(b).to(td).cuda(), X, opts=api.SolveOpts(rtol=1e-6))
        Xh = X.cpu().numpy().astype(np.complex128)
        out[f"{st}_{name}_solve"] = max(rel_residual(H, Xh[r], b[r]) for r in range(3))
        out[f"{st}_{name}_conv"] = all(r["converged"] for r in rep)
p = synth.tiny2d()
pml = D.PmlParams(v_ref=3000.0)
d = fwi.forward_data(p, pml, p.m_true)
fg, _ = api.fwi_misfit_grad(api.Grid.of(p), p.m, p.freqs, p.src, p.rec, d, api.Pml(v_ref=pml.v_ref), api.C128,
                            api.SolveOpts(rtol=1e-8), max_rhs=4)
f_ref, g_ref = fwi.misfit_grad(p, pml, d)
fg = fg.cpu().numpy()
out["f"] = abs(fg[0] - f_ref) / f_ref
out["g"] = float(np.linalg.norm(fg[1:] - g_ref.ravel()) / np.linalg.norm(g_ref))
print(json.dumps(out))
"""


@pytest.mark.parametrize("env", [{}, {"HELM_MARCH_TMA": "2"}, {"HELM_MARCH_TMA": "0"}],
                         ids=["default_rule", "tma_ring_always", "cpasync_ring"])
def test_march_feeds_match_oracle(env):
    e = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""), **env)
    r = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=e, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for st in ("std2", "opt"):
        for adj in (0, 1):
            assert res[f"{st}_c128_apply{adj}"] <= 1e-12, res
            assert res[f"{st}_c64_apply{adj}"] <= 1e-5, res
        assert res[f"{st}_c128_conv"] and res[f"{st}_c128_solve"] <= 1e-6 * (1 + 1e-3), res
        assert res[f"{st}_c64_conv"] and res[f"{st}_c64_solve"] <= 2e-6, res
    assert res["f"] <= 1e-5 and res["g"] <= 1e-5, res
