"""Reduced least-squares misfit and adjoint-state gradient (ORACLE — test infrastructure only).

Follows Listing 1 ``case OBJ`` and SURVEY.md §8(c) D7-D12:
  q_s      = S(omega) e_{node(s)} / h^d                              (D7, R12, R28)
  u        = H^-1 q_s                                                (Table 1 row u(m))
  f       += 1/2 || P_r u - d ||^2                                   (Eq. 2; phi P:57; D10)
  v        = H^-H ( -P_r^T (P_r u - d) )                             (Table 1 V(m); D11)
  g       += E^T sum_s Re(omega^2 conj(u) v)                         (Eq. 8, Table 1 grad f
                                                                      P:102, Listing 1; D12)
The PML reference velocity ``pml.v_ref`` must be fixed (independent of m) so
that H depends on m only through omega^2 diag(E m) (Eq. 7) — DESIGN.md R31.
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np

from .discretize import PmlParams, extension_matrix, helmholtz_matrix, interior_to_ext_index, mass_matrix, stencil_of
from .solve import LU


def _mass_h(prob, V: np.ndarray) -> np.ndarray:
    """A^H V with A of Eq. (7): identity for STD2, the mass distribution of R34 / R35
    for the "opt" stencils (the gradient T^* = omega^2 diag(conj u) A^H)."""
    if stencil_of(prob) == "std2":
        return V
    return mass_matrix(prob).conj().T @ V


def _mass(prob, X: np.ndarray) -> np.ndarray:
    """A X (T dm = omega^2 A (u .* E dm), Eq. 7)."""
    if stencil_of(prob) == "std2":
        return X
    return mass_matrix(prob) @ X


def source_matrix(prob, omega: float, src_ids: Sequence[int], weight: complex = 1.0) -> np.ndarray:
    """D7: columns q_s = S(omega) e_node(s) / h^d on the extended grid, shape (N_ext, ns)."""
    idx = interior_to_ext_index(prob, src_ids)
    Q = np.zeros((prob.n_ext, len(idx)), np.complex128)
    Q[idx, np.arange(len(idx))] = weight / prob.h ** prob.ndim
    return Q


def receivers(prob, U: np.ndarray) -> np.ndarray:
    """D8: (P_r u)_k = u(node(rec_k)); U is (N_ext, ns) -> (nrec, ns)."""
    return U[interior_to_ext_index(prob, prob.rec), :]


def receivers_adjoint(prob, R: np.ndarray) -> np.ndarray:
    """D8: P_r^T scatter-adds receiver values back onto the extended grid."""
    out = np.zeros((prob.n_ext, R.shape[1]), np.complex128)
    np.add.at(out, interior_to_ext_index(prob, prob.rec), R)
    return out


def forward_data(prob, pml: PmlParams, m_int=None, src_ids=None, weights=None) -> np.ndarray:
    """Listing 1 ``FORW_MODEL``: d[f, s, k] = (P_r H_f^-1 q_s)_k."""
    src_ids = prob.src if src_ids is None else src_ids
    out = []
    for fi, f in enumerate(prob.freqs):
        w = 2.0 * np.pi * f
        S = 1.0 if weights is None else weights[fi]
        H = helmholtz_matrix(prob, w, pml, m_int)
        U = LU(H).solve(source_matrix(prob, w, src_ids, S))
        out.append(receivers(prob, U).T)
    return np.stack(out)          # (nfreq, nsrc, nrec), receiver fastest


def misfit_grad(prob, pml: PmlParams, d_obs: np.ndarray, m_int=None, src_ids=None,
                weights=None, return_fields: bool = False):
    """Listing 1 ``case OBJ`` with LU solves: returns (f, g) with g on the interior grid.

    d_obs has shape (nfreq, nsrc, nrec) for the sources ``src_ids``."""
    m_int = prob.m if m_int is None else m_int
    src_ids = prob.src if src_ids is None else src_ids
    E = extension_matrix(prob)
    f = 0.0
    g_ext = np.zeros(prob.n_ext)
    fields = []
    for fi, fr in enumerate(prob.freqs):
        w = 2.0 * np.pi * fr
        S = 1.0 if weights is None else weights[fi]
        H = helmholtz_matrix(prob, w, pml, m_int)
        lu = LU(H)
        U = lu.solve(source_matrix(prob, w, src_ids, S))                 # u = H^-1 q
        r = receivers(prob, U) - d_obs[fi].T                             # P_r u - d
        f += 0.5 * float(np.sum(np.abs(r) ** 2))                          # Eq. (2)
        V = lu.solve(-receivers_adjoint(prob, r), adjoint=True)          # v = H^-H(-P_r^T r)
        g_ext += np.sum(np.real(w**2 * np.conj(U) * _mass_h(prob, V)), axis=1)   # Re(w^2 conj(u) A^H v)
        if return_fields:
            fields.append((U, V))
    g = E.T @ g_ext                                                      # E^T (R11)
    if return_fields:
        return f, g.reshape(prob.m.shape), fields
    return f, g.reshape(prob.m.shape)


# ----------------------------------------------------------------------------- SURVEY §8(f) rank 1
# Linearised modelling, its adjoint and the Gauss-Newton Hessian (Table 1, Table 2
# P:111-117; Listing 1 JACOBI_FORW / JACOBI_ADJ / HESS_GN P:167-180). With A of Eq. 7 (I for
# STD2, the mass distribution M for the R34 / R35 stencils):
#   T dm  = DH(m)[dm] u = omega^2 A (u (.) (E dm))
#   T^* z = E^T Re(omega^2 conj(u) (.) (A^H z))     (sum_srcs = to_phys * real)
#   J dm  = P_r Du[dm],  Du[dm] = -H^-1 T dm
#   J^H y = T^* H^-H (-P_r^T y)
#   H_GN dm = J^H J dm = T^* H^-H (-P_r^T P_r (-H^-1 T dm))
# (Listing 1 writes T(U)*dU in HESS_GN where Table 1 has T^*: the adjoint is used.)

def jacobian(prob, pml: PmlParams, dm: np.ndarray, m_int=None, src_ids=None, weights=None) -> np.ndarray:
    """Listing 1 JACOBI_FORW: d_lin[f, s, k] = (P_r (-H^-1 T dm))_k, shape (nfreq, nsrc, nrec)."""
    src_ids = prob.src if src_ids is None else src_ids
    dm_ext = extension_matrix(prob) @ np.asarray(dm, np.float64).ravel()
    out = []
    for fi, fr in enumerate(prob.freqs):
        w = 2.0 * np.pi * fr
        S = 1.0 if weights is None else weights[fi]
        lu = LU(helmholtz_matrix(prob, w, pml, m_int))
        U = lu.solve(source_matrix(prob, w, src_ids, S))
        dU = lu.solve(-(w**2) * _mass(prob, U * dm_ext[:, None]))
        out.append(receivers(prob, dU).T)
    return np.stack(out)


def jacobian_adjoint(prob, pml: PmlParams, y: np.ndarray, m_int=None, src_ids=None, weights=None) -> np.ndarray:
    """Listing 1 JACOBI_ADJ: g = E^T sum Re(omega^2 conj(u) H^-H(-P_r^T y)); y: (nfreq, nsrc, nrec)."""
    src_ids = prob.src if src_ids is None else src_ids
    g_ext = np.zeros(prob.n_ext)
    for fi, fr in enumerate(prob.freqs):
        w = 2.0 * np.pi * fr
        S = 1.0 if weights is None else weights[fi]
        lu = LU(helmholtz_matrix(prob, w, pml, m_int))
        U = lu.solve(source_matrix(prob, w, src_ids, S))
        V = lu.solve(-receivers_adjoint(prob, y[fi].T), adjoint=True)
        g_ext += np.sum(np.real(w**2 * np.conj(U) * _mass_h(prob, V)), axis=1)
    return (extension_matrix(prob).T @ g_ext).reshape(prob.m.shape)


def gn_hessian(prob, pml: PmlParams, dm: np.ndarray, m_int=None, src_ids=None, weights=None) -> np.ndarray:
    """Listing 1 HESS_GN (with T^*): three solves per (source, frequency) (Table 2)."""
    src_ids = prob.src if src_ids is None else src_ids
    dm_ext = extension_matrix(prob) @ np.asarray(dm, np.float64).ravel()
    g_ext = np.zeros(prob.n_ext)
    for fi, fr in enumerate(prob.freqs):
        w = 2.0 * np.pi * fr
        S = 1.0 if weights is None else weights[fi]
        lu = LU(helmholtz_matrix(prob, w, pml, m_int))
        U = lu.solve(source_matrix(prob, w, src_ids, S))
        dU = lu.solve(-(w**2) * _mass(prob, U * dm_ext[:, None]))
        V = lu.solve(-receivers_adjoint(prob, receivers(prob, dU)), adjoint=True)
        g_ext += np.sum(np.real(w**2 * np.conj(U) * _mass_h(prob, V)), axis=1)
    return (extension_matrix(prob).T @ g_ext).reshape(prob.m.shape)


def taylor_errors(fun, m, dm, g, ts):
    """§6.1: e0(t) = |f(m+t dm) - f(m)|, e1(t) = |f(m+t dm) - f(m) - t <g, dm>|."""
    f0 = fun(m)
    gd = float(np.sum(g * dm))
    e0, e1 = [], []
    for t in ts:
        ft = fun(m + t * dm)
        e0.append(abs(ft - f0))
        e1.append(abs(ft - f0 - t * gd))
    return np.array(e0), np.array(e1)
