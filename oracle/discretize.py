"""Discrete PML Helmholtz operator, assembled (ORACLE — test infrastructure only).

Implements SURVEY.md §8(c) c.1 D1-D6, which restate:
  * Eq. (1), PAPER.md P:61-63 — (nabla^2 + omega^2 m) u = S delta, m = slowness^2 (R1);
  * §3 P:67-71 — domain extended to Omega' with zero Dirichlet, model extended
    "in the normal direction", PML derivative d~_x = (1/eta(x)) d_x;
  * Eq. (7) P:633 — H = L + omega^2 A diag(m), A = I for the 5/7-point STD2 stencil (R4).
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np
import scipy.sparse as sp


@dataclasses.dataclass(frozen=True)
class PmlParams:
    """D3 / R5: quadratic ramp, sigma_max = (p+1) v_ref ln(1/R) / (2 L)."""
    R: float = 1e-4
    power: int = 2
    v_ref: float = 0.0          # <= 0: max velocity of the model (helm_setup default)


def default_pml(m: np.ndarray, v_ref: float = 0.0) -> PmlParams:
    return PmlParams(v_ref=float(v_ref) if v_ref > 0 else float(np.max(1.0 / np.sqrt(m))))


def ext_shape(prob) -> tuple:
    """Extended sizes (Nz, Ny, Nx) for a C-order [z][y][x] array (D1)."""
    Nx, Ny, Nz = prob.next
    return (Nz, Ny, Nx)


# ----------------------------------------------------------------------------- D3, D4
def pml_eta(xi, n_int, h0, w_lo, w_hi, omega, pml: PmlParams):
    """D3: eta(xi) = 1 + i sigma(xi)/omega (R3: e^{-i omega t}, outgoing e^{+i kappa r}).

    d(xi) = max(0, -xi) + max(0, xi - (n-1) h); sigma = sigma_max (d/L)^p with
    L = w h the PML thickness on that side; no clamping of d/L (D3)."""
    xi = np.asarray(xi, dtype=np.float64)
    L_int = (n_int - 1) * h0
    sigma = np.zeros_like(xi)
    for w, d in ((w_lo, np.maximum(0.0, -xi)), (w_hi, np.maximum(0.0, xi - L_int))):
        if w > 0:
            L = w * h0
            smax = (pml.power + 1) * pml.v_ref * np.log(1.0 / pml.R) / (2.0 * L)
            sigma = sigma + smax * (d / L) ** pml.power
    return 1.0 + 1j * sigma / omega


def tables_1d(N, n_int, h0, w_lo, w_hi, omega, pml: PmlParams, level: int = 0):
    """D4 (+D13 for coarse levels): 1D stretched second difference along one axis.

    Node i of level l sits at xi = (i 2^l - w_lo) h0 with spacing h = 2^l h0;
      up_i = 1/(h^2 eta_i eta_{i+1/2}),  lo_i = 1/(h^2 eta_i eta_{i-1/2}),
      dg_i = -(up_i + lo_i).
    Returns complex arrays (lo, dg, up) of length N."""
    h = h0 * 2.0 ** level
    i = np.arange(N, dtype=np.float64)
    xi = (i * 2.0 ** level - w_lo) * h0
    e0 = pml_eta(xi, n_int, h0, w_lo, w_hi, omega, pml)
    ep = pml_eta(xi + 0.5 * h, n_int, h0, w_lo, w_hi, omega, pml)
    em = pml_eta(xi - 0.5 * h, n_int, h0, w_lo, w_hi, omega, pml)
    up = 1.0 / (h * h * e0 * ep)
    lo = 1.0 / (h * h * e0 * em)
    dg = -(up + lo)
    return lo, dg, up


def adjoint_tables_1d(lo, dg, up):
    """D6 closed form: (T^H y)_i = conj(up_{i-1}) y_{i-1} + conj(dg_i) y_i + conj(lo_{i+1}) y_{i+1}.
    Used only to cross-check against the explicit conjugate transpose."""
    loH = np.zeros_like(lo)
    upH = np.zeros_like(up)
    loH[1:] = np.conj(up[:-1])
    upH[:-1] = np.conj(lo[1:])
    return loH, np.conj(dg), upH


def second_difference(lo, dg, up):
    """Sparse T_a with zero ghosts: row i = lo_i u_{i-1} + dg_i u_i + up_i u_{i+1}."""
    N = len(dg)
    return sp.diags([lo[1:], dg, up[:-1]], [-1, 0, 1], shape=(N, N), format="csr",
                    dtype=np.complex128)


# ----------------------------------------------------------------------------- D2
def interior_to_ext_index(prob, ids):
    """Interior linear node ids -> extended linear indices (D7/D8)."""
    nx, ny, nz = prob.n
    Nx, Ny, Nz = prob.next
    ids = np.asarray(ids, dtype=np.int64)
    ix = ids % nx
    iy = (ids // nx) % ny
    iz = ids // (nx * ny)
    return (ix + prob.pml[0][0]) + Nx * ((iy + prob.pml[1][0]) + Ny * (iz + prob.pml[2][0]))


def extension_matrix(prob) -> sp.csr_matrix:
    """D2: E, m_ext(i) = m(clamp(i_a - w_a^-, 0, n_a - 1)) per axis."""
    nx, ny, nz = prob.n
    Nx, Ny, Nz = prob.next
    cx = np.clip(np.arange(Nx) - prob.pml[0][0], 0, nx - 1)
    cy = np.clip(np.arange(Ny) - prob.pml[1][0], 0, ny - 1)
    cz = np.clip(np.arange(Nz) - prob.pml[2][0], 0, nz - 1)
    CZ, CY, CX = np.meshgrid(cz, cy, cx, indexing="ij")
    cols = (CX + nx * (CY + ny * CZ)).ravel()
    rows = np.arange(Nx * Ny * Nz)
    return sp.csr_matrix((np.ones(rows.size), (rows, cols)), shape=(Nx * Ny * Nz, nx * ny * nz))


def extend(prob, m_int: np.ndarray) -> np.ndarray:
    """m_ext = E m, returned with shape (Nz, Ny, Nx)."""
    return (extension_matrix(prob) @ np.asarray(m_int, np.float64).ravel()).reshape(ext_shape(prob))


# ----------------------------------------------------------------------------- R34 / R35
# The paper's higher-order stencils (2D "9pt optimal" [23], 3D "compact 27-pt" [60];
# coefficients not printed): DESIGN readings R34 (2D) / R35 (3D) define them as product forms
# of 1D operators, so that the PML enters through the same stretched tables T_a as STD2:
#   L = sum of consistent Laplacians (T_a along one axis times averages A_b along the others),
#   H = L + omega^2 M diag(E m)          (Eq. 7 with A = M)
# with A_a = (1/4, 1/2, 1/4) and E_a = (1/2, 0, 1/2) (zero ghosts, R7) and the weights
# below (derived by scripts/derive_opt_stencil.py: least-squares phase-velocity error over
# all directions and 4..inf points per wavelength, non-negative weights), copied from DESIGN.
OPT9 = dict(a=0.58547, c=0.63353, d=0.36647)                       # e = 1 - c - d = 0
OPT27 = dict(w1=0.36027, w2=0.46886, w3=0.17087, m1=0.47314, m2=0.50415, m3=0.02271)   # m4 = 0


def averaging_1d(N: int, w_off: float, w_mid: float) -> sp.csr_matrix:
    """Tridiagonal (w_off, w_mid, w_off) with zero ghosts: A_a = (1/4, 1/2, 1/4), E_a = (1/2, 0, 1/2)."""
    return sp.diags([np.full(N - 1, w_off), np.full(N, w_mid), np.full(N - 1, w_off)], [-1, 0, 1],
                    shape=(N, N), format="csr", dtype=np.complex128)


def _k3(Az, Ay, Ax):
    return sp.kron(Az, sp.kron(Ay, Ax))


def operator_from_tables(T, m_ext, omega: float, ndim: int, stencil: str = "std2") -> sp.csr_matrix:
    """H from the per-axis stretched second differences T = (Tx, Ty, Tz) (Ty None in 2D) and the
    extended model (C-order [z][y][x]): D5 for "std2", R34 / R35 for "opt"."""
    Tx, Ty, Tz = T
    Nx, Nz = Tx.shape[0], Tz.shape[0]
    Ny = Ty.shape[0] if ndim == 3 else 1
    Ix, Iy, Iz = (sp.identity(k, format="csr", dtype=np.complex128) for k in (Nx, Ny, Nz))
    m_diag = sp.diags(omega**2 * np.asarray(m_ext).ravel())
    if stencil == "std2":
        L = _k3(Iz, Iy, Tx) + _k3(Tz, Iy, Ix)
        if ndim == 3:
            L = L + _k3(Iz, Ty, Ix)
        return (L + m_diag).tocsr()
    if stencil != "opt":
        raise ValueError(f"unknown stencil {stencil!r}")
    Ax, Az = averaging_1d(Nx, 0.25, 0.5), averaging_1d(Nz, 0.25, 0.5)
    Ex, Ez = averaging_1d(Nx, 0.5, 0.0), averaging_1d(Nz, 0.5, 0.0)
    if ndim == 2:
        a, c, d = OPT9["a"], OPT9["c"], OPT9["d"]
        e = 1.0 - c - d
        L = a * (_k3(Iz, Iy, Tx) + _k3(Tz, Iy, Ix)) + (1 - a) * (_k3(Az, Iy, Tx) + _k3(Tz, Iy, Ax))
        M = c * _k3(Iz, Iy, Ix) + d / 2 * (_k3(Iz, Iy, Ex) + _k3(Ez, Iy, Ix)) + e * _k3(Ez, Iy, Ex)
        return (L + M @ m_diag).tocsr()
    Ay, Ey = averaging_1d(Ny, 0.25, 0.5), averaging_1d(Ny, 0.5, 0.0)
    w1, w2, w3 = OPT27["w1"], OPT27["w2"], OPT27["w3"]
    m1, m2, m3 = OPT27["m1"], OPT27["m2"], OPT27["m3"]
    m4 = 1.0 - m1 - m2 - m3
    L1 = _k3(Iz, Iy, Tx) + _k3(Iz, Ty, Ix) + _k3(Tz, Iy, Ix)
    L2 = 0.5 * (_k3(Iz, Ay, Tx) + _k3(Az, Iy, Tx) + _k3(Iz, Ty, Ax) + _k3(Az, Ty, Ix) + _k3(Tz, Iy, Ax) + _k3(Tz, Ay, Ix))
    L3 = _k3(Az, Ay, Tx) + _k3(Az, Ty, Ax) + _k3(Tz, Ay, Ax)
    L = w1 * L1 + w2 * L2 + w3 * L3
    M = (m1 * _k3(Iz, Iy, Ix) + m2 / 3 * (_k3(Iz, Iy, Ex) + _k3(Iz, Ey, Ix) + _k3(Ez, Iy, Ix))
         + m3 / 3 * (_k3(Iz, Ey, Ex) + _k3(Ez, Iy, Ex) + _k3(Ez, Ey, Ix)) + m4 * _k3(Ez, Ey, Ex))
    return (L + M @ m_diag).tocsr()


def mass_matrix(prob) -> sp.csr_matrix:
    """A of Eq. (7): I for STD2, the mass distribution M of R34 / R35 for "opt"."""
    Nx, Ny, Nz = prob.next
    zero = [sp.csr_matrix((k, k), dtype=np.complex128) for k in (Nx, Ny, Nz)]
    T = (zero[0], zero[1] if prob.ndim == 3 else None, zero[2])
    return operator_from_tables(T, np.ones(prob.n_ext), 1.0, prob.ndim, stencil_of(prob)).real.tocsr()


def stencil_of(prob) -> str:
    return getattr(prob, "stencil", "std2")


# ----------------------------------------------------------------------------- D5
def helmholtz_matrix(prob, omega: float, pml: PmlParams, m_int: Optional[np.ndarray] = None,
                     ) -> sp.csr_matrix:
    """D5: H = sum_a T_a (acting along axis a) + omega^2 diag(E m), C-order [z][y][x] (STD2);
    prob.stencil == "opt": R34 / R35 (operator_from_tables).

    2D problems (ndim == 2) have no y term (ny = 1 and no T_y)."""
    m_int = prob.m if m_int is None else m_int
    nx, ny, nz = prob.n
    Nx, Ny, Nz = prob.next
    (wxl, wxh), (wyl, wyh), (wzl, wzh) = prob.pml
    Tx = second_difference(*tables_1d(Nx, nx, prob.h, wxl, wxh, omega, pml))
    Tz = second_difference(*tables_1d(Nz, nz, prob.h, wzl, wzh, omega, pml))
    Ty = second_difference(*tables_1d(Ny, ny, prob.h, wyl, wyh, omega, pml)) if prob.ndim == 3 else None
    return operator_from_tables((Tx, Ty, Tz), extend(prob, m_int), omega, prob.ndim, stencil_of(prob))


def helmholtz_rows(prob, omega: float, pml: PmlParams, z_lo: int, z_hi: int,
                   m_int: Optional[np.ndarray] = None) -> sp.csr_matrix:
    """The rows of D5's H for the extended z-planes [z_lo, z_hi) (all x, y), shape
    (rows, N_ext): the same Kronecker sum as helmholtz_matrix with the z factor restricted
    to those planes, so large grids can be checked slab by slab without assembling H."""
    m_int = prob.m if m_int is None else m_int
    nx, ny, nz = prob.n
    Nx, Ny, Nz = prob.next
    (wxl, wxh), (wyl, wyh), (wzl, wzh) = prob.pml
    Tx = second_difference(*tables_1d(Nx, nx, prob.h, wxl, wxh, omega, pml))
    Tz = second_difference(*tables_1d(Nz, nz, prob.h, wzl, wzh, omega, pml))[z_lo:z_hi]
    Ix, Iy = (sp.identity(k, format="csr", dtype=np.complex128) for k in (Nx, Ny))
    Izr = sp.identity(Nz, format="csr", dtype=np.complex128)[z_lo:z_hi]
    L = sp.kron(Izr, sp.kron(Iy, Tx)) + sp.kron(Tz, sp.kron(Iy, Ix))
    if prob.ndim == 3:
        Ty = second_difference(*tables_1d(Ny, ny, prob.h, wyl, wyh, omega, pml))
        L = L + sp.kron(Izr, sp.kron(Ty, Ix))
    m_slab = extend(prob, m_int)[z_lo:z_hi].ravel()
    rows = np.arange(z_lo * Ny * Nx, z_hi * Ny * Nx)
    D = sp.csr_matrix((omega**2 * m_slab, (np.arange(rows.size), rows)), shape=(rows.size, Nx * Ny * Nz))
    return (L + D).tocsr()


def helmholtz_adjoint_matrix(H: sp.spmatrix) -> sp.csr_matrix:
    """H^H as the explicit conjugate transpose (c.2 step 2) — deliberately not D6."""
    return H.conj().T.tocsr()
