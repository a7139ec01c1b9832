"""GPU parity of a3-a6/a8 through the C ABI: level transfers vs the mirror's P and R, one
V-cycle vs the numpy mirror (same fixed counts, c.4: <= 1e-12 c128), and full FGMRES +
ML-GMRES solves vs LU (rel-L2 <= 1e-5 at rel-residual 1e-6, R24) incl. adjoint, batched,
mixed c64, zero right-hand side."""
import numpy as np
import pytest
import torch

import synth
from oracle import discretize as D
from oracle import fwi, green, mlgmres
from oracle.solve import LU, rel_residual
from paper_1703_09268_b200 import api

from .helpers import rel, to_dev, to_host

pytestmark = pytest.mark.gpu


def _setup(p, dtype=api.C128, nrhs=1, vref=None):
    w = 2 * np.pi * p.freqs[0]
    pml = D.default_pml(p.m) if vref is None else D.PmlParams(v_ref=vref)
    op = api.helm_setup(api.Grid.of(p), p.m, w, api.Pml(pml.R, pml.power, pml.v_ref), dtype, max_rhs=nrhs)
    return op, w, pml


@pytest.mark.parametrize("make", [synth.tiny2d, synth.tiny3d, synth.cfg1])
def test_transfers_match_mirror(make):
    p = make()
    op, w, pml = _setup(p, nrhs=2)
    hier = mlgmres.Hierarchy(p, w, pml)
    for l in range(len(hier.P)):
        nf, nc = hier.P[l].shape
        r = synth.random_complex((2, nf), 1)
        out = torch.zeros(2, nc, dtype=torch.complex128, device="cuda")
        api.helm_transfer(op, to_dev(r), out, level=l, prolong=False)
        ref = np.stack([hier.R[l] @ r[i] for i in range(2)])
        assert rel(to_host(out), ref) <= 1e-14
        xc = synth.random_complex((2, nc), 3)
        xf = synth.random_complex((2, nf), 4)
        t = to_dev(xf)
        api.helm_transfer(op, to_dev(xc), t, level=l, prolong=True)
        ref = np.stack([xf[i] + hier.P[l] @ xc[i] for i in range(2)])
        assert rel(to_host(t), ref) <= 1e-14


@pytest.mark.parametrize("make,adjoint", [(synth.tiny2d, 0), (synth.tiny2d, 1), (synth.tiny3d, 0),
                                          (synth.cfg1, 0), (synth.cfg1, 1)])
def test_vcycle_matches_mirror(make, adjoint):
    p = make()
    op, w, pml = _setup(p, nrhs=2)
    hier = mlgmres.Hierarchy(p, w, pml)
    b = synth.random_complex((2, p.n_ext), 1)
    z = torch.zeros(2, p.n_ext, dtype=torch.complex128, device="cuda")
    api.helm_vcycle(op, to_dev(b), z, level=0, adjoint=adjoint)
    zg = to_host(z)
    for r in range(2):
        ref = mlgmres.vcycle(hier, 0, b[r], adjoint=bool(adjoint))
        assert rel(zg[r], ref) <= 1e-12


@pytest.mark.parametrize("make,adjoint,nrhs", [(synth.tiny2d, 0, 2), (synth.tiny3d, 1, 2), (synth.cfg1, 0, 1),
                                                (synth.cfg1, 1, 3)])
def test_coarse_vcycle_matches_mirror(make, adjoint, nrhs):
    """The V-cycle at the second-to-last level (coarsest GMRES below it), same fixed counts as
    the mirror (the grid-synchronous single-launch variant is checked in test_gpu_paths)."""
    p = make()
    op, w, pml = _setup(p, nrhs=nrhs)
    hier = mlgmres.Hierarchy(p, w, pml)
    n1 = int(np.prod(hier.shapes[1]))
    b = synth.random_complex((nrhs, n1), 2)
    z = torch.zeros(nrhs, n1, dtype=torch.complex128, device="cuda")
    api.helm_vcycle(op, to_dev(b), z, level=1, adjoint=adjoint)
    zg = to_host(z)
    for r in range(nrhs):
        assert rel(zg[r], mlgmres.vcycle(hier, 1, b[r], adjoint=bool(adjoint))) <= 1e-12


@pytest.mark.parametrize("dtype", [api.C128, api.C64])
def test_cfg1_solve_matches_lu_and_green(dtype):
    """Config 1 (BASELINE configs[0]): vs LU <= 1e-5, certificate <= 1e-6, vs -(i/4)H0 <= 1.5 %."""
    p = synth.cfg1()
    op, w, pml = _setup(p, dtype)
    H = D.helmholtz_matrix(p, w, pml)
    q = fwi.source_matrix(p, w, p.src)[:, 0]
    u_lu = LU(H).solve(q)
    td = torch.complex128 if dtype == api.C128 else torch.complex64
    x = torch.zeros(1, p.n_ext, dtype=td, device="cuda")
    rep = api.helm_solve(op, to_dev(q, td), x)
    u = to_host(x)[0]
    assert rep[0]["converged"] and rep[0]["rel_residual"] <= 1e-6
    assert rel(u, u_lu) <= 1e-5
    if dtype == api.C128:
        assert rel_residual(H, u, q) <= 1e-6 * (1 + 1e-3)
    assert green.green_error(p, u, 2000.0, 5.0, int(p.src[0])) < 0.015
    assert rep[0]["outer_cycles"] <= 3


@pytest.mark.parametrize("adjoint", [0, 1])
def test_batched_solves_match_lu(adjoint):
    p = synth.tiny3d(nsrc=3)
    op, w, pml = _setup(p, nrhs=4)
    H = D.helmholtz_matrix(p, w, pml)
    Q = fwi.source_matrix(p, w, p.src)
    B = np.concatenate([Q.T, np.zeros((1, p.n_ext))])          # 4th RHS is zero
    U = LU(H).solve(Q, adjoint=bool(adjoint)).T
    x = torch.full((4, p.n_ext), 7.0 + 1j, dtype=torch.complex128, device="cuda")
    rep = api.helm_solve(op, to_dev(B), x, adjoint=adjoint)
    xg = to_host(x)
    for r in range(3):
        assert rep[r]["converged"], rep[r]
        assert rel(xg[r], U[r]) <= 1e-5
    assert np.all(xg[3] == 0) and rep[3]["converged"] and rep[3]["outer_cycles"] == 0


def test_unpreconditioned_gmres_path():
    p = synth.tiny2d()
    op, w, pml = _setup(p)
    H = D.helmholtz_matrix(p, w, pml)
    q = fwi.source_matrix(p, w, p.src[:1])[:, 0]
    x = torch.zeros(1, p.n_ext, dtype=torch.complex128, device="cuda")
    rep = api.helm_solve(op, to_dev(q), x, opts=api.SolveOpts(precond=0, max_outer=2000))
    assert rep[0]["converged"]
    assert rel(to_host(x)[0], LU(H).solve(q)) <= 1e-5


def test_workspace_within_paper_bound():
    """the solve keeps at most 26 vectors of the finest size per RHS."""
    p = synth.cfg3()
    op, w, pml = _setup(p)
    assert op.workspace_vectors() <= 26


@pytest.mark.parametrize("make", [synth.tiny2d, synth.tiny3d])
def test_solves_are_bitwise_reproducible(make):
    """R30: every reduction is fixed-order fp64 and the level-0 V-cycle replays a captured
    CUDA graph after its first live run — repeated solves give bitwise identical results."""
    p = make()
    op, w, pml = _setup(p, nrhs=len(p.src))
    Q = fwi.source_matrix(p, w, p.src)
    b = to_dev(np.ascontiguousarray(Q.T))
    xs = []
    for _ in range(3):
        x = torch.zeros_like(b)
        rep = api.helm_solve(op, b, x)
        assert all(r["converged"] for r in rep)
        xs.append(to_host(x))
    assert np.array_equal(xs[0], xs[1]) and np.array_equal(xs[1], xs[2])
