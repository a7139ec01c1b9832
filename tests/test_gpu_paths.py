"""GPU parity of the alternative 3D stage-fill paths, each in a fresh process (the switches are
read once per process): per-thread cp.async instead of TMA (HELM_TMA=0), TMA tiles with m and
the z coefficients by cp.async (HELM_TMA_MZ=0), and two rows per thread for the matvec
(HELM_PLANE_PY=2), the split ring for the last fused Arnoldi step (HELM_SPLIT=1; also with one
row per thread, HELM_SPLIT_PY=1) or for every fused step (HELM_SPLIT=2), also with three formed slots (two barriers per
plane, HELM_SPLIT_OCC=4) or two raw stages (HELM_SPLIT_D=2), and coarse V-cycles as kernel
one grid-synchronous launch instead of a launch sequence (HELM_PERSIST=1; the level-1
V-cycle is also compared with the numpy mirror, <= 1e-12, and must take <= 2 launches), and
32 x 16 matvec tiles (HELM_MATVEC_BY=16), and the round-1 single ring that keeps plane z-1 in
shared memory (HELM_PREV=0) or keeps it in registers in every mode including the matvec
(HELM_PREV=2), and the fused steps' per-item ring fills (HELM_CONT=0) against the default
continuous ring across a CTA's items, also with items shorter than the ring (HELM_PLANE_NZC=9:
3-4 planes per item; =40: one plane per item, so the ring spans several items), the last
fused step storing V_{k-1} (HELM_LASTV=1) instead of the solution update reforming it, and
the per-warp reduction tail (HELM_CTA_RED=0) instead of one slot per CTA, and the fused steps
with two rows per thread everywhere (HELM_FUSED_PY1=99) or one row for the last step too
(HELM_FUSED_PY1_LAST=1). Each must match the assembled oracle H (c128 <= 1e-12, c64 <= 1e-5) for
helm_apply forward / adjoint on a ragged multi-tile grid, and give a certified solve."""
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
from oracle.solve import rel_residual
from paper_1703_09268_b200 import api
from tests.test_gpu_operator import medium3d
p = medium3d()
w = 2 * np.pi * p.freqs[0]
pml = D.PmlParams(v_ref=float(np.max(1 / np.sqrt(p.m))) * 1.1)
H = D.helmholtz_matrix(p, w, pml)
out = {}
for name, dt, td in (("c128", api.C128, torch.complex128), ("c64", api.C64, torch.complex64)):
    op = api.helm_setup(api.Grid.of(p), p.m, w, api.Pml(pml.R, pml.power, pml.v_ref), dt, max_rhs=3)
    x = synth.random_complex((3, p.n_ext), 1)
    for adj in (0, 1):
        A = D.helmholtz_adjoint_matrix(H) if adj else H
        y = torch.empty(3, p.n_ext, dtype=td, device="cuda")
        api.helm_apply(op, torch.from_numpy(x.astype(np.complex128)).to(td).cuda(), y, adj)
        yg = y.cpu().numpy().astype(np.complex128)
        xr = x.astype(np.complex64).astype(np.complex128) if name == "c64" else x
        out[f"{name}_apply{adj}"] = max(float(np.linalg.norm(yg[r] - A @ xr[r]) / np.linalg.norm(A @ xr[r])) for r in range(3))
    b = np.zeros((3, p.n_ext), np.complex128)
    b[np.arange(3), [p.n_ext // 2, p.n_ext // 3, p.n_ext // 5]] = 1.0
    X = torch.empty(3, p.n_ext, dtype=td, device="cuda")
    rep = api.helm_solve(op, torch.from_numpy(b).to(td).cuda(), X, opts=api.SolveOpts(rtol=1e-6))
    Xh = X.cpu().numpy().astype(np.complex128)
    out[f"{name}_solve"] = max(rel_residual(H, Xh[r], b[r]) for r in range(3))
    out[f"{name}_conv"] = all(r["converged"] for r in rep)
# level-1 V-cycle (coarsest GMRES below it) vs the mirror, complex128
from oracle import mlgmres
op = api.helm_setup(api.Grid.of(p), p.m, w, api.Pml(pml.R, pml.power, pml.v_ref), api.C128, max_rhs=2)
hier = mlgmres.Hierarchy(p, w, pml)
n1 = int(np.prod(hier.shapes[1]))
b1 = synth.random_complex((2, n1), 2)
z1 = torch.zeros(2, n1, dtype=torch.complex128, device="cuda")
l0 = api.launch_count()
api.helm_vcycle(op, torch.from_numpy(b1).cuda(), z1, level=1, adjoint=1)
out["vcycle1_launches"] = api.launch_count() - l0
zg = z1.cpu().numpy()
out["vcycle1"] = max(float(np.linalg.norm(zg[r] - mlgmres.vcycle(hier, 1, b1[r], adjoint=True)) /
                          np.linalg.norm(zg[r])) for r in range(2))
print(json.dumps(out))
"""


@pytest.mark.parametrize("env", [{"HELM_TMA": "0"}, {"HELM_TMA_MZ": "0"}, {"HELM_PLANE_PY": "2"},
                                 {"HELM_SPLIT": "1"}, {"HELM_SPLIT": "1", "HELM_SPLIT_PY": "1"}, {"HELM_SPLIT": "2"}, {"HELM_SPLIT": "2", "HELM_SPLIT_OCC": "4"},
                                 {"HELM_SPLIT": "2", "HELM_SPLIT_D": "2"}, {"HELM_PERSIST": "1"}, {"HELM_MATVEC_BY": "16"}, {"HELM_PREV": "0"}, {"HELM_PREV": "2"},
                                 {"HELM_CONT": "0"}, {"HELM_PLANE_NZC": "9"}, {"HELM_PLANE_NZC": "40"},
                                 {"HELM_LASTV": "1"}, {"HELM_CTA_RED": "0"}, {"HELM_FUSED_PY1": "99"},
                                 {"HELM_FUSED_PY1_LAST": "1"}],
                         ids=["cpasync", "tma_tiles_only", "py2", "split_last_step", "split_last_step_one_row", "split_all", "split_nf3", "split_d2",
                              "persistent_vcycle", "matvec_by16", "ring_without_register_plane",
                              "register_plane_every_mode", "per_item_ring", "cont_ring_short_items",
                              "cont_ring_one_plane_items", "last_basis_vector_stored", "per_warp_reduction",
                              "fused_steps_two_rows", "fused_steps_one_row_last_step_too"])
def test_alternative_stage_paths_match_oracle(env):
    e = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""), **env)
    r = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for adj in (0, 1):
        assert res[f"c128_apply{adj}"] <= 1e-12, res
        assert res[f"c64_apply{adj}"] <= 1e-5, res
    assert res["c128_conv"] and res["c128_solve"] <= 1e-6 * (1 + 1e-3), res
    assert res["c64_conv"] and res["c64_solve"] <= 2e-6, res
    assert res["vcycle1"] <= 1e-12, res
    if env.get("HELM_PERSIST") == "1":
        assert res["vcycle1_launches"] <= 2, res
