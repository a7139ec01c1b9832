"""Analytic free-space Green's functions (ORACLE — test infrastructure only).

§6.1 PAPER.md P:339-345 with the sign reading R2/R3 of SURVEY.md §8(c):
Eq. (1) has a +delta source and the e^{-i omega t} convention, so
  G_2D = -(i/4) H_0^(1)(kappa r),      G_3D = -e^{i kappa r} / (4 pi r),
kappa = 2 pi f / v0. (The paper prints +e^{i kappa r}/(4 pi r), the -delta form.)
"""
from __future__ import annotations

import numpy as np
from scipy.special import hankel1


def green_2d(r, kappa):
    return -0.25j * hankel1(0, kappa * np.asarray(r, np.float64))


def green_3d(r, kappa):
    r = np.asarray(r, np.float64)
    return -np.exp(1j * kappa * r) / (4.0 * np.pi * r)


def distance_field(prob, src_id: int) -> np.ndarray:
    """|x - x_s| on the extended grid (Nz, Ny, Nx) from the source node."""
    nx, ny, nz = prob.n
    Nx, Ny, Nz = prob.next
    sx, sy, sz = src_id % nx, (src_id // nx) % ny, src_id // (nx * ny)
    x = (np.arange(Nx) - prob.pml[0][0] - sx) * prob.h
    y = (np.arange(Ny) - prob.pml[1][0] - sy) * prob.h
    z = (np.arange(Nz) - prob.pml[2][0] - sz) * prob.h
    Z, Y, X = np.meshgrid(z, y, x, indexing="ij")
    return np.sqrt(X**2 + Y**2 + Z**2)


def interior_mask(prob) -> np.ndarray:
    Nx, Ny, Nz = prob.next
    msk = np.zeros((Nz, Ny, Nx), bool)
    (xl, _), (yl, _), (zl, _) = prob.pml
    nx, ny, nz = prob.n
    msk[zl:zl + nz, yl:yl + ny, xl:xl + nx] = True
    return msk


def green_error(prob, u_ext: np.ndarray, v0: float, f: float, src_id: int, rmin_wavelengths=1.0):
    """Relative L2 error of u vs the analytic G on interior nodes with r >= rmin * lambda (c.2 step 5)."""
    kappa = 2.0 * np.pi * f / v0
    lam = v0 / f
    r = distance_field(prob, src_id)
    sel = interior_mask(prob) & (r >= rmin_wavelengths * lam)
    G = green_2d(r[sel], kappa) if prob.ndim == 2 else green_3d(r[sel], kappa)
    u = u_ext.reshape(r.shape)[sel]
    return float(np.linalg.norm(u - G) / np.linalg.norm(G))
