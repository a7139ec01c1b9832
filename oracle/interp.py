"""Off-grid sources and receivers by Kaiser-windowed sinc interpolation (ORACLE — test
infrastructure only).

PAPER.md P:139: "In order to discretize the delta source function, we use Kaiser-windowed sinc
interpolation [47]" — without parameters. Readings (R33):
  * 1D weight of grid node k for a point at fractional grid position t (t = x / h):
        w_k = sinc(t - k) I0(b sqrt(1 - ((t - k)/r)^2)) / I0(b)    for |t - k| <= r, else 0,
    sinc(x) = sin(pi x)/(pi x); b = 6.31, r = 4 grid points;
  * the weights of each axis are divided by their sum, so that a constant field is reproduced
    exactly (S:121 asks for 1e-6; the raw window misses by up to 4e-4) — a point on a node
    still gets weight 1 there and 0 elsewhere, i.e. the on-node delta of D7/D8;
  * multi-dimensional weights are tensor products of the 1D ones; taps falling outside
    the extended grid are dropped before the normalisation;
  * coordinates are physical, relative to interior node (0, 0, 0): x = i h; points must lie in
    the interior box; 2D problems use (x, 0, z).
P_r = interp_matrix(rec); the source for point s is q_s = S(omega) P_s^T e_s / h^d (D7 with the
delta replaced by its interpolant).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .discretize import PmlParams, extension_matrix, helmholtz_matrix
from .solve import LU

KAISER_B = 6.31
HALF_WIDTH = 4


def kaiser_sinc_1d(t: float, n_ext: int, lo: int, b: float = KAISER_B, r: int = HALF_WIDTH):
    """Extended-grid nodes and normalised weights of one axis for interior grid position t."""
    k = np.arange(int(np.ceil(t - r)), int(np.floor(t + r)) + 1)
    d = t - k
    w = np.sinc(d) * np.i0(b * np.sqrt(np.clip(1.0 - (d / r) ** 2, 0.0, None))) / np.i0(b)
    e = k + lo
    keep = (e >= 0) & (e < n_ext)
    e, w = e[keep], w[keep]
    return e, w / w.sum()


def interp_matrix(prob, coords, b: float = KAISER_B, r: int = HALF_WIDTH) -> sp.csr_matrix:
    """Rows = points, columns = extended-grid nodes (x fastest): the sampling operator P."""
    coords = np.atleast_2d(np.asarray(coords, np.float64))
    Nx, Ny, Nz = prob.next
    rows, cols, vals = [], [], []
    for i, (x, y, z) in enumerate(coords):
        if prob.ndim == 2 and y != 0.0:
            raise ValueError(f"point {i}: 2D problems need y = 0")
        for a, (c, n) in enumerate(zip((x, y, z), prob.n)):
            if not (0.0 <= c <= (n - 1) * prob.h):
                raise ValueError(f"point {i} outside the interior along axis {a}")
        ex, wx = kaiser_sinc_1d(x / prob.h, Nx, prob.pml[0][0], b, r)
        if prob.ndim == 3:
            ey, wy = kaiser_sinc_1d(y / prob.h, Ny, prob.pml[1][0], b, r)
        else:
            ey, wy = np.zeros(1, int), np.ones(1)
        ez, wz = kaiser_sinc_1d(z / prob.h, Nz, prob.pml[2][0], b, r)
        idx = ((ez[:, None, None] * Ny + ey[None, :, None]) * Nx + ex[None, None, :]).ravel()
        w = (wz[:, None, None] * wy[None, :, None] * wx[None, None, :]).ravel()
        rows.append(np.full(idx.size, i))
        cols.append(idx)
        vals.append(w)
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(len(coords), prob.n_ext))


def source_matrix(prob, omega: float, src_xyz, weight: complex = 1.0, b=KAISER_B, r=HALF_WIDTH) -> np.ndarray:
    """Columns q_s = S(omega) P_s^T e_s / h^d, shape (N_ext, ns)."""
    Ps = interp_matrix(prob, src_xyz, b, r)
    return np.asarray((Ps.T * (weight / prob.h ** prob.ndim)).todense()).astype(np.complex128)


def forward_data(prob, pml: PmlParams, src_xyz, rec_xyz, m_int=None, weights=None) -> np.ndarray:
    """Listing 1 FORW_MODEL with off-grid P_s, P_r: d[f, s, k] = (P_r H_f^-1 q_s)_k."""
    Pr = interp_matrix(prob, rec_xyz)
    out = []
    for fi, f in enumerate(prob.freqs):
        w = 2.0 * np.pi * f
        S = 1.0 if weights is None else weights[fi]
        U = LU(helmholtz_matrix(prob, w, pml, m_int)).solve(source_matrix(prob, w, src_xyz, S))
        out.append((Pr @ U).T)
    return np.stack(out)


def misfit_grad(prob, pml: PmlParams, d_obs, src_xyz, rec_xyz, m_int=None, weights=None):
    """Listing 1 case OBJ with off-grid P_s, P_r (same steps as fwi.misfit_grad)."""
    Pr = interp_matrix(prob, rec_xyz)
    f = 0.0
    g_ext = np.zeros(prob.n_ext)
    for fi, fr in enumerate(prob.freqs):
        w = 2.0 * np.pi * fr
        S = 1.0 if weights is None else weights[fi]
        lu = LU(helmholtz_matrix(prob, w, pml, m_int))
        U = lu.solve(source_matrix(prob, w, src_xyz, S))
        res = Pr @ U - d_obs[fi].T
        f += 0.5 * float(np.sum(np.abs(res) ** 2))
        V = lu.solve(-(Pr.T @ res), adjoint=True)
        g_ext += np.sum(np.real(w**2 * np.conj(U) * V), axis=1)
    return f, (extension_matrix(prob).T @ g_ext).reshape(prob.m.shape)
