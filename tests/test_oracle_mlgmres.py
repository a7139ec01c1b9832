"""Pins of the ML-GMRES mirror (D13-D14): grid rule, P/R identities, memory formula
(P:295-301), and that FGMRES+V-cycle reproduces the LU solution (the definition)."""
import numpy as np
import pytest

import synth
from oracle import discretize as D
from oracle import fwi, mlgmres
from oracle.solve import LU


@pytest.mark.parametrize("N,chain", [(84, [42, 21]), (220, [110, 55]), (441, [221, 111]),
                                     (241, [121, 61]), (141, [71, 36]), (97, [49, 25])])
def test_coarse_sizes(N, chain):
    """S:314 (97 -> 49 -> 25) and SURVEY c.4 level sizes."""
    out = []
    for _ in chain:
        N = mlgmres.coarse_size(N)
        out.append(N)
    assert out == chain


def test_prolongation_reproduces_constants_and_restriction_is_scaled_adjoint():
    Nf = 11  # odd: every fine node has its coarse neighbours in range
    P = mlgmres.prolongation_1d(Nf)
    assert np.allclose(P @ np.ones(P.shape[1]), 1.0)
    # tensor-product R = 2^-d P^T dot test through the hierarchy
    p = synth.tiny3d()
    hier = mlgmres.Hierarchy(p, 2 * np.pi * 8, D.PmlParams(v_ref=2500.0))
    xc = synth.random_complex(hier.P[0].shape[1], 1)
    yf = synth.random_complex(hier.P[0].shape[0], 3)
    a = np.vdot(yf, hier.P[0] @ xc)
    b = np.vdot(hier.R[0] @ yf, xc) * 2.0**3
    assert abs(a - b) <= 1e-14 * abs(a)
    # linear fields are reproduced exactly on odd grids away from the far ghost
    x = np.arange(mlgmres.coarse_size(Nf), dtype=float) * 2.0
    assert np.allclose((P @ x)[:-1], np.arange(Nf - 1, dtype=float))


def test_full_weighting_preserves_constants():
    W = mlgmres.full_weighting_1d(10)
    assert np.allclose(W @ np.full(10, 3.5), 3.5)
    p = synth.const_problem("c", 3, (9, 8, 7), 10.0, 2, 1700.0, 5.0)
    hier = mlgmres.Hierarchy(p, 2 * np.pi * 5, D.default_pml(p.m))
    for me in hier.m_ext:
        assert np.allclose(me, 1 / 1700.0**2, rtol=1e-15)


def test_coarse_operator_is_rediscretized_laplacian():
    """No PML, omega^2 m = 0: level-1 operator = 5-point Laplacian with spacing 2h."""
    p = synth.const_problem("c", 2, (9, 9), 5.0, 0, 1700.0, 5.0).with_(m=np.zeros((9, 1, 9)))
    hier = mlgmres.Hierarchy(p, 1.0, D.PmlParams(v_ref=1.0), opts=mlgmres.MlOpts(levels=2))
    A = hier.H[1].toarray()
    h2 = (2 * 5.0) ** 2
    Nc = 5
    k = 2 * Nc + 2            # interior coarse node (2,2)
    assert np.isclose(A[k, k], -4 / h2) and np.isclose(A[k, k + 1], 1 / h2) and np.isclose(A[k, k + Nc], 1 / h2)


def test_peak_memory_formula():
    """'our preconditioner requires at most 26 vectors'; S:331 (1,1,1,1), k_i=1 -> 14."""
    assert mlgmres.peak_vectors(5, 5, 5) == 26
    assert mlgmres.peak_vectors(1, 1, 1) == 14


@pytest.mark.parametrize("make,adjoint", [(synth.cfg1, False), (synth.tiny2d, False),
                                          (synth.tiny2d, True), (synth.tiny3d, False),
                                          (synth.tiny3d, True)])
def test_mlgmres_solution_equals_lu(make, adjoint):
    p = make()
    w = 2 * np.pi * p.freqs[0]
    pml = D.default_pml(p.m)
    hier = mlgmres.Hierarchy(p, w, pml)
    q = fwi.source_matrix(p, w, p.src[:1])[:, 0]
    u_lu = LU(hier.H[0]).solve(q, adjoint=adjoint)
    u, cycles, rel = mlgmres.solve(hier, q, rtol=1e-10, adjoint=adjoint)
    assert rel <= 1e-10
    assert np.linalg.norm(u - u_lu) / np.linalg.norm(u_lu) < 1e-8
    assert cycles <= 8


def test_vcycle_homogeneous_and_zero():
    """GMRES from 0 is scale-equivariant, so the V-cycle is positively homogeneous (§7 notes)."""
    p = synth.tiny2d()
    hier = mlgmres.Hierarchy(p, 2 * np.pi * 9, D.default_pml(p.m))
    b = synth.random_complex(p.n_ext, 1)
    z1 = mlgmres.vcycle(hier, 0, b)
    z2 = mlgmres.vcycle(hier, 0, 3.7 * b)
    assert np.linalg.norm(z2 - 3.7 * z1) <= 1e-12 * np.linalg.norm(z2)
    assert np.all(mlgmres.vcycle(hier, 0, np.zeros_like(b)) == 0)


def test_cfg1_expected_outer_cycles():
    """[probe] STD2 config 1 converges to 1e-6 in 2 outer FGMRES(5) cycles (parity unpinned vs
    the paper's 27-pt Table 3)."""
    p = synth.cfg1()
    w = 2 * np.pi * 5.0
    hier = mlgmres.Hierarchy(p, w, D.default_pml(p.m))
    q = fwi.source_matrix(p, w, p.src)[:, 0]
    _, cycles, rel = mlgmres.solve(hier, q, rtol=1e-6)
    assert cycles == 2 and rel <= 1e-6
