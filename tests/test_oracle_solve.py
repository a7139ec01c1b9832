"""Pins of oracle/solve.py's iterative path (c.2 step 3 "otherwise"):
unpreconditioned GMRES(restart) to 1e-10 equals the sparse LU solution (an independent
direct method) forward and adjoint, and a solve that cannot reach the tolerance raises
instead of returning silently. Also pins the cfg3 reference files in tests/golden/cfg3/
(written by scripts/make_cfg3_reference.py from oracle/ only) by their metadata and, cheaply,
by the oracle's own residual on the stored single-source field."""
import json
import os

import numpy as np
import pytest

import synth
from oracle import discretize as D
from oracle import fwi, mlgmres
from oracle.solve import LU, NotConverged, gmres_solve, rel_residual

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cfg3")


@pytest.mark.parametrize("adjoint", [False, True])
def test_gmres_solve_equals_lu_tiny3d(adjoint):
    p = synth.tiny3d()
    w = 2 * np.pi * p.freqs[0]
    H = D.helmholtz_matrix(p, w, D.default_pml(p.m))
    q = fwi.source_matrix(p, w, p.src[:1])[:, 0]
    u_lu = LU(H).solve(q, adjoint=adjoint)
    u = gmres_solve(H, q, rtol=1e-10, restart=100, adjoint=adjoint, maxiter=400)
    assert rel_residual(H, u, q, adjoint=adjoint) <= 1e-10 * (1 + 1e-6)
    assert np.linalg.norm(u - u_lu) / np.linalg.norm(u_lu) < 1e-8


def test_gmres_solve_adjoint_is_not_forward():
    """H is not complex-symmetric in the PML (D6): the adjoint solve differs from conj of the
    forward one, so a solver that ignored `adjoint` would fail the test above."""
    p = synth.tiny3d()
    w = 2 * np.pi * p.freqs[0]
    H = D.helmholtz_matrix(p, w, D.default_pml(p.m))
    q = fwi.source_matrix(p, w, p.src[:1])[:, 0]
    uf = gmres_solve(H, q, rtol=1e-10, maxiter=400)
    ua = gmres_solve(H, q, rtol=1e-10, adjoint=True, maxiter=400)
    assert np.linalg.norm(ua - uf) > 1e-3 * np.linalg.norm(uf)


def test_gmres_solve_raises_when_not_converged():
    p = synth.tiny3d()
    w = 2 * np.pi * p.freqs[0]
    H = D.helmholtz_matrix(p, w, D.default_pml(p.m))
    q = fwi.source_matrix(p, w, p.src[:1])[:, 0]
    with pytest.raises(NotConverged):
        gmres_solve(H, q, rtol=1e-10, restart=5, maxiter=2)


def test_cfg3_reference_files_are_certified():
    """The stored cfg3 references: metadata says every field was certified by the oracle's own
    residual at <= 1e-10 (mirror ML-GMRES solve, c.2 step 6) and the single forward field was
    cross-checked against the unpreconditioned GMRES path; the stored (complex64-rounded)
    single forward field still has a residual at the complex64 rounding level."""
    meta = json.load(open(os.path.join(GOLD, "meta.json")))
    assert meta["rtol"] <= 1e-10
    for k, v in meta["fields"].items():
        assert v["rel_residual"] <= 1e-10, k
    if "gmres_cross_check" in meta:
        assert meta["gmres_cross_check"]["rel_diff"] <= 1e-8
    p = synth.cfg3()
    w = 2 * np.pi * p.freqs[0]
    H = D.helmholtz_matrix(p, w, D.PmlParams(v_ref=2000.0))
    u = np.load(os.path.join(GOLD, "single_fwd.npy")).astype(np.complex128).ravel()
    q = fwi.source_matrix(p, w, p.src)[:, 0]
    assert rel_residual(H, u, q) <= 1e-6           # c64 rounding alone gives ~3e-7 here
    assert meta["fields"]["single_fwd"]["rounded_rel_err"] <= 1e-7


def test_mirror_solver_adjoint_at_tight_tolerance():
    """The mirror's solve at 1e-10 (the cfg3 reference path) equals LU on the adjoint too."""
    p = synth.tiny3d(n=(15, 13, 11))
    w = 2 * np.pi * p.freqs[0]
    hier = mlgmres.Hierarchy(p, w, D.default_pml(p.m))
    q = fwi.source_matrix(p, w, p.src[:1])[:, 0]
    u_lu = LU(hier.H[0]).solve(q, adjoint=True)
    u, _, rel = mlgmres.solve(hier, q, rtol=1e-10, adjoint=True)
    assert rel <= 1e-10 and np.linalg.norm(u - u_lu) / np.linalg.norm(u_lu) < 1e-8
