"""GPU: early stopping inside an outer FGMRES cycle ("the Arnoldi estimate is allowed
only for early stopping inside a cycle"; convergence is decided on the TRUE residual).

Each variant runs in a fresh process (HELM_EARLY is read once per process). Batches mix RHS of
different difficulty (point sources, a smooth random RHS, a scaled copy and a zero RHS) so that
they leave their cycles at different inner steps, forward and adjoint, 2D and 3D, c128 and c64.
Checked against the oracle's assembled H and its LU (unique solution): certified true residual,
point-source solutions <= 2e-5 from LU (random RHS <= 5e-5: only ||H^-1|| bounds the error
at a residual of 1e-6, in either schedule), never more level-0 matvecs or cycles than full cycles take, and the
full-cycle schedule (HELM_EARLY=0) still certifies."""
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
from oracle.solve import LU, rel_residual
from paper_1703_09268_b200 import api
from tests.test_gpu_operator import medium2d
out = {}
# 3D: 39 x 29 x 25 extended points (two x tiles, four y tile rows, ragged tails; small enough
# for a quick oracle LU — the plane kernel's paths have their own parity tests)
for pname, p in (("2d", medium2d()), ("3d", synth.tiny3d(n=(29, 19, 15), pml=5))):
    w = 2 * np.pi * p.freqs[0]
    pml = D.PmlParams(v_ref=float(np.max(1 / np.sqrt(p.m))) * 1.1)
    H = D.helmholtz_matrix(p, w, pml)
    lu = LU(H)
    nb = 5
    b = np.zeros((nb, p.n_ext), np.complex128)
    b[0, p.n_ext // 2] = 1.0
    b[1, p.n_ext // 3] = 1.0
    b[2] = synth.random_complex((p.n_ext,), 5)
    b[3] = 1e6 * b[0] + 1e3 * synth.random_complex((p.n_ext,), 6)   # scale invariance of the stop rule
    # b[4] = 0
    for name, dt, td in (("c128", api.C128, torch.complex128), ("c64", api.C64, torch.complex64)):
        op = api.helm_setup(api.Grid.of(p), p.m, w, api.Pml(pml.R, pml.power, pml.v_ref), dt, max_rhs=nb)
        for adj in (0, 1):
            U = lu.solve(b[:4].T, adjoint=bool(adj)).T
            X = torch.full((nb, p.n_ext), 3.0 - 2j, dtype=td, device="cuda")
            rep = api.helm_solve(op, torch.from_numpy(b).to(td).cuda(), X, adjoint=adj, opts=api.SolveOpts(rtol=1e-6))
            Xh = X.cpu().numpy().astype(np.complex128)
            A = D.helmholtz_adjoint_matrix(H) if adj else H
            bq = b.astype(np.complex64).astype(np.complex128) if name == "c64" else b
            key = f"{pname}_{name}_{adj}"
            out[key] = {
                "conv": all(r["converged"] for r in rep),
                "res": max(rel_residual(A, Xh[r], bq[r]) for r in range(4)),
                "err": [float(np.linalg.norm(Xh[r] - U[r]) / np.linalg.norm(U[r])) for r in range(4)],
                "zero": bool(np.all(Xh[4] == 0)) and rep[4]["outer_cycles"] == 0,
                "cycles": [r["outer_cycles"] for r in rep],
                "mv0": [r["matvecs"][0] for r in rep],
            }
print(json.dumps(out))
"""


def _run(env):
    e = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""), **env)
    r = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=e, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.fixture(scope="module")
def runs():
    """(default factor, full cycles, factor 0.98): the default (0.5) may never trigger on grids
    this small, 0.98 exercises the early-exit path itself."""
    return _run({}), _run({"HELM_EARLY": "0"}), _run({"HELM_EARLY_PCT": "98"})


def test_early_stop_solutions_are_certified(runs):
    for res in runs:
        for key, v in res.items():
            tol_res = 1e-6 * (1 + 1e-3) if "c128" in key else 2e-6
            assert v["conv"] and v["zero"], (key, v)
            assert v["res"] <= tol_res, (key, v)
            # A certified residual of rtol = 1e-6 bounds the error only through ||H^-1||: measured
            # error / residual ratios are 4-11 for point sources and up to 17 for the random
            # full-spectrum RHS, in EVERY schedule (medium3d, full cycles, adjoint point source:
            # residual 9.7e-7, error 1.05e-5; profiles/r02/ab_r2z), so the bars here are 2e-5 and
            # 5e-5; the north star's 1e-5 on f, g and the BASELINE configs is checked where it is
            # stated (test_gpu_fwi, test_gpu_solve, test_gpu_fullsize).
            assert max(v["err"][:2]) <= 2e-5, (key, v)
            assert max(v["err"][2:]) <= 5e-5, (key, v)


def test_early_stop_never_costs_more(runs):
    default, full, p98 = runs
    for early in (default, p98):
        for key in full:
            for r in range(4):
                assert early[key]["cycles"][r] <= full[key]["cycles"][r] + 1, (key, early[key], full[key])
                # a cycle cut short may need one more short cycle, never more level-0 matvecs
                # than one extra inner step plus the extra true-residual check
                assert early[key]["mv0"][r] <= full[key]["mv0"][r] + 8, (key, early[key], full[key])
    saved = sum(full[key]["mv0"][r] - p98[key]["mv0"][r] for key in full for r in range(4))
    assert saved > 0, (p98, full)   # the early exit was taken somewhere
