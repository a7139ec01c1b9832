"""Pins of the off-grid Kaiser-windowed sinc oracle (oracle/interp.py; SURVEY §8(f) rank 4,
PAPER P:139, readings R33): on-node points reduce to the on-node delta of D7/D8 (so the whole
off-grid evaluation equals fwi.forward_data / fwi.misfit_grad there), a constant is reproduced
exactly, a band-limited field is sampled far better than by linear interpolation (a high-order
interpolant, which a dropped window, a mis-scaled sinc or a wrong axis would break), and the
off-grid gradient matches a central difference of the off-grid misfit."""
import numpy as np
import pytest

import synth
from oracle import discretize as D
from oracle import fwi
from oracle import interp as I


def _coords_of_nodes(p, ids):
    ix, iy, iz = ids % p.n[0], (ids // p.n[0]) % p.n[1], ids // (p.n[0] * p.n[1])
    return np.stack([ix * p.h, iy * p.h, iz * p.h], axis=1).astype(np.float64)


def _offgrid(p, n, seed):
    rng = np.random.default_rng(seed)
    c = np.zeros((n, 3))
    for a in range(3):
        if p.n[a] > 1:
            c[:, a] = rng.uniform(1.0 * p.h, (p.n[a] - 2) * p.h, size=n)
    return c


@pytest.mark.parametrize("make", [synth.tiny2d, synth.tiny3d])
def test_on_node_points_are_the_on_node_delta(make):
    p = make()
    P = I.interp_matrix(p, _coords_of_nodes(p, p.rec)).toarray()
    E = np.zeros_like(P)
    E[np.arange(len(p.rec)), D.interior_to_ext_index(p, p.rec)] = 1.0
    assert np.abs(P - E).max() <= 1e-12


def test_on_node_evaluation_equals_the_node_oracle():
    p = synth.tiny2d()
    pml = D.PmlParams(v_ref=3000.0)
    sx, rx = _coords_of_nodes(p, p.src), _coords_of_nodes(p, p.rec)
    d_node = fwi.forward_data(p, pml, p.m_true)
    d_off = I.forward_data(p, pml, sx, rx, p.m_true)
    assert np.abs(d_off - d_node).max() <= 1e-12 * np.abs(d_node).max()
    f0, g0 = fwi.misfit_grad(p, pml, d_node)
    f1, g1 = I.misfit_grad(p, pml, d_node, sx, rx)
    assert abs(f1 - f0) <= 1e-12 * f0 and np.linalg.norm(g1 - g0) <= 1e-12 * np.linalg.norm(g0)


@pytest.mark.parametrize("make", [synth.tiny2d, synth.tiny3d])
def test_constant_reproduction_and_support(make):
    p = make()
    P = I.interp_matrix(p, _offgrid(p, 20, 1))
    assert np.abs(np.asarray(P.sum(axis=1)).ravel() - 1.0).max() <= 1e-14
    assert np.diff(P.indptr).max() <= (2 * I.HALF_WIDTH + 1) ** p.ndim


def test_band_limited_sampling_is_high_order():
    """cos(k . x) at 8 points per wavelength: the windowed sinc error is <= 1e-2 and at least
    10x below bilinear interpolation's (error ~ (k h)^2 / 8 ~ 8e-2)."""
    p = synth.const_problem("il", 2, (60, 50), 10.0, 8, 2000.0, 5.0)
    kx, kz = 2 * np.pi / (8 * p.h) * np.cos(0.3), 2 * np.pi / (8 * p.h) * np.sin(0.3)
    Nx, _, Nz = p.next
    ex = (np.arange(Nx) - p.pml[0][0]) * p.h
    ez = (np.arange(Nz) - p.pml[2][0]) * p.h
    field = np.cos(kz * ez[:, None] + kx * ex[None, :]).ravel()
    c = _offgrid(p, 50, 7)
    c[:, 0] = np.clip(c[:, 0], 6 * p.h, (p.n[0] - 7) * p.h)
    c[:, 2] = np.clip(c[:, 2], 6 * p.h, (p.n[2] - 7) * p.h)
    exact = np.cos(kx * c[:, 0] + kz * c[:, 2])
    err_sinc = np.abs(I.interp_matrix(p, c) @ field - exact).max()
    fx, fz = c[:, 0] / p.h, c[:, 2] / p.h
    i0, k0 = np.floor(fx).astype(int), np.floor(fz).astype(int)
    ax, az = fx - i0, fz - k0
    F = field.reshape(Nz, Nx)
    L = lambda i, k: F[k + p.pml[2][0], i + p.pml[0][0]]  # noqa: E731
    lin = ((1 - ax) * (1 - az) * L(i0, k0) + ax * (1 - az) * L(i0 + 1, k0) + (1 - ax) * az * L(i0, k0 + 1)
           + ax * az * L(i0 + 1, k0 + 1))
    err_lin = np.abs(lin - exact).max()
    assert err_sinc <= 1e-2 and err_sinc * 10 <= err_lin, (err_sinc, err_lin)


def test_offgrid_gradient_matches_directional_difference():
    p = synth.tiny2d()
    pml = D.PmlParams(v_ref=3000.0)
    sx, rx = _offgrid(p, 2, 3), _offgrid(p, 9, 4)
    d = I.forward_data(p, pml, sx, rx, p.m_true)
    _, g = I.misfit_grad(p, pml, d, sx, rx)
    dm = np.ones_like(p.m) * 1e-9
    t = 1e-2
    fd = (I.misfit_grad(p, pml, d, sx, rx, p.m + t * dm)[0] - I.misfit_grad(p, pml, d, sx, rx, p.m - t * dm)[0]) / (2 * t)
    assert abs(fd - np.sum(g * dm)) <= 1e-6 * abs(fd)


def test_points_outside_the_interior_are_rejected():
    p = synth.tiny2d()
    with pytest.raises(ValueError):
        I.interp_matrix(p, [[-1.0, 0.0, 10.0]])
    with pytest.raises(ValueError):
        I.interp_matrix(p, [[10.0, 5.0, 10.0]])
