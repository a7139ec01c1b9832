"""Oracle solves pinned to physics: analytic Green's functions (§6.1), the
library Hankel function, second-order refinement, the sign reading R2."""
import numpy as np
import pytest
from scipy.special import hankel1

import synth
from oracle import discretize as D
from oracle import fwi, green, mlgmres
from oracle.solve import LU, rel_residual


def test_hankel_library_value():
    """J0(1) = 0.76520, Y0(1) = 0.08826 => H0^(1)(1) = J0 + i Y0."""
    z = hankel1(0, 1.0)
    assert abs(z.real - 0.76520) < 5e-6 and abs(z.imag - 0.08826) < 5e-6


def _solve_point(p, f):
    w = 2 * np.pi * f
    H = D.helmholtz_matrix(p, w, D.default_pml(p.m))
    q = fwi.source_matrix(p, w, p.src)[:, 0]
    u = LU(H).solve(q)
    assert rel_residual(H, u, q) < 1e-10
    return u


def test_cfg1_green_2d():
    """Config 1 vs -(i/4) H0^(1)(kappa r) at r >= 1 lambda (c.4: <= 1.5 %); the opposite
    sign is off by ~2 (R2)."""
    p = synth.cfg1()
    u = _solve_point(p, 5.0)
    err = green.green_error(p, u, 2000.0, 5.0, int(p.src[0]))
    assert err < 0.015
    assert green.green_error(p, -u, 2000.0, 5.0, int(p.src[0])) > 1.5


def test_second_order_refinement():
    """Halving h (same physical domain and PML) divides the Green's error by ~4."""
    errs = []
    for h, n, w in ((20.0, 51, 10), (10.0, 101, 20)):
        p = synth.const_problem("r", 2, (n, n), h, w, 2000.0, 5.0, [(n // 2, 0, n // 2)])
        u = _solve_point(p, 5.0)
        errs.append(green.green_error(p, u, 2000.0, 5.0, int(p.src[0])))
    ratio = errs[0] / errs[1]
    assert 3.0 < ratio < 5.0, errs


@pytest.mark.slow
def test_green_3d_with_mirror_solver():
    """3D constant (12.5 ppw) vs -e^{i kappa r}/(4 pi r) at r >= 1 lambda (c.4: <= 15 %), solved
    by the oracle's ML-GMRES mirror to 1e-8 and certified by the true residual; the paper's
    printed (+) sign is off by ~2 (R2)."""
    p = synth.const_problem("g3", 3, (40, 40, 40), 20.0, 8, 2000.0, 8.0, [(20, 20, 20)])
    w = 2 * np.pi * 8.0
    hier = mlgmres.Hierarchy(p, w, D.default_pml(p.m))
    q = fwi.source_matrix(p, w, p.src)[:, 0]
    u, cycles, rel = mlgmres.solve(hier, q, rtol=1e-8)
    assert rel_residual(hier.H[0], u, q) <= 1e-8 * (1 + 1e-6)
    err = green.green_error(p, u, 2000.0, 8.0, int(p.src[0]))
    assert err < 0.15, err
    assert green.green_error(p, -u, 2000.0, 8.0, int(p.src[0])) > 1.5
