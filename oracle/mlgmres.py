"""Numpy mirror of the ML-GMRES preconditioner (ORACLE — test infrastructure only).

The converged solution of H u = q does not depend on the preconditioner; this
mirror exists (a) to check the GPU V-cycle map itself with the same fixed
counts and (b) as the oracle's own accelerator for 3D sizes where LU is
infeasible (its output is always certified by the true residual).

Follows PAPER.md §5:
  * Alg. 1, the standard V-cycle: smooth, residual, restrict, coarse
    solve, prolong + correct, smooth;
  * P:258 linear interpolation P and its adjoint as restriction (R21: R = 2^-d P^T);
  * P:272-276 / Fig. 3: smoother = GMRES [72] with identity
    preconditioner, coarse solver = FGMRES [71] preconditioned recursively by the
    same V-cycle; coarsest level GMRES unpreconditioned (R20);
  * P:284 memory vector (k_so, k_si, k_co, k_ci) = (3,5,3,5), outer FGMRES(5) to 1e-6;
  * P:295-301 peak-memory formula;
and SURVEY.md §8(c) D13 (hierarchy) and D14 (fixed counts, breakdown guard).
Gram-Schmidt is the modified (textbook Arnoldi) variant; least squares by
numpy ``lstsq`` on the (k+1) x k Hessenberg matrix.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Callable, List, Optional

import numpy as np
import scipy.sparse as sp

from .discretize import PmlParams, extend, operator_from_tables, second_difference, stencil_of, tables_1d

BREAKDOWN = 1e-14


@dataclasses.dataclass(frozen=True)
class MlOpts:
    levels: int = 3
    ks_o: int = 3
    ks_i: int = 5
    kc_o: int = 3
    kc_i: int = 5


def coarse_size(N: int) -> int:
    """D13: N^{l+1} = ceil(N^l / 2); coarse node j sits on fine node 2j."""
    return (N + 1) // 2


def prolongation_1d(Nf: int) -> sp.csr_matrix:
    """D13 / P:258 linear interpolation: fine 2j <- coarse j; fine 2j+1 <- (c_j + c_{j+1})/2,
    with the coarse ghost c_{Nc} = 0 (zero Dirichlet)."""
    Nc = coarse_size(Nf)
    rows, cols, vals = [], [], []
    for i in range(Nf):
        j = i // 2
        if i % 2 == 0:
            rows.append(i); cols.append(j); vals.append(1.0)
        else:
            rows.append(i); cols.append(j); vals.append(0.5)
            if j + 1 < Nc:
                rows.append(i); cols.append(j + 1); vals.append(0.5)
    return sp.csr_matrix((vals, (rows, cols)), shape=(Nf, Nc))


def full_weighting_1d(Nf: int) -> sp.csr_matrix:
    """S:340 / D13: normalized (1/4, 1/2, 1/4) over in-range fine nodes 2j-1, 2j, 2j+1."""
    Nc = coarse_size(Nf)
    W = sp.lil_matrix((Nc, Nf))
    for j in range(Nc):
        for i, w in ((2 * j - 1, 0.25), (2 * j, 0.5), (2 * j + 1, 0.25)):
            if 0 <= i < Nf:
                W[j, i] = w
    W = W.tocsr()
    s = np.asarray(W.sum(axis=1)).ravel()
    return sp.diags(1.0 / s) @ W


def _kron3(Az, Ay, Ax):
    return sp.kron(Az, sp.kron(Ay, Ax)).tocsr()


class Hierarchy:
    """D13: levels l = 0..L-1 sharing the physical PML; rediscretized operators."""

    def __init__(self, prob, omega: float, pml: PmlParams, m_int=None, opts: MlOpts = MlOpts()):
        self.prob, self.omega, self.pml, self.opts = prob, omega, pml, opts
        self.d = prob.ndim
        Nx, Ny, Nz = prob.next
        shapes = [(Nz, Ny, Nx)]
        m_ext = [extend(prob, prob.m if m_int is None else m_int)]
        P: List[sp.csr_matrix] = []
        W: List[sp.csr_matrix] = []
        for l in range(1, opts.levels):
            nz, ny, nx = shapes[-1]
            cz, cy, cx = coarse_size(nz), (coarse_size(ny) if self.d == 3 else 1), coarse_size(nx)
            Py = prolongation_1d(ny) if self.d == 3 else sp.identity(1, format="csr")
            Wy = full_weighting_1d(ny) if self.d == 3 else sp.identity(1, format="csr")
            P.append(_kron3(prolongation_1d(nz), Py, prolongation_1d(nx)))
            W.append(_kron3(full_weighting_1d(nz), Wy, full_weighting_1d(nx)))
            shapes.append((cz, cy, cx))
            m_ext.append((W[-1] @ m_ext[-1].ravel()).reshape(cz, cy, cx))
        self.shapes, self.m_ext, self.P = shapes, m_ext, P
        self.R = [(2.0 ** -self.d) * p.T.tocsr() for p in P]          # R21
        self.H = [self._operator(l) for l in range(opts.levels)]
        self.HH = [h.conj().T.tocsr() for h in self.H]

    def _operator(self, l: int) -> sp.csr_matrix:
        """D4-D5 at level l with (h_l, m_l, omega) (rediscretization)."""
        pr = self.prob
        Nz, Ny, Nx = self.shapes[l]
        (wxl, wxh), (wyl, wyh), (wzl, wzh) = pr.pml
        nx, ny, nz = pr.n
        Tx = second_difference(*tables_1d(Nx, nx, pr.h, wxl, wxh, self.omega, self.pml, l))
        Tz = second_difference(*tables_1d(Nz, nz, pr.h, wzl, wzh, self.omega, self.pml, l))
        Ty = second_difference(*tables_1d(Ny, ny, pr.h, wyl, wyh, self.omega, self.pml, l)) if self.d == 3 else None
        return operator_from_tables((Tx, Ty, Tz), self.m_ext[l], self.omega, self.d, stencil_of(pr))

    def op(self, l: int, adjoint: bool) -> Callable[[np.ndarray], np.ndarray]:
        A = self.HH[l] if adjoint else self.H[l]
        return lambda x: A @ x


def krylov(A, b, x0, ko: int, ki: int, M=None):
    """GMRES(ko, ki) (M None, P:274 smoother) or FGMRES(ko, ki) with right preconditioner M
    ([71]): ko restart cycles of ki Arnoldi steps, fixed counts (R19), MGS, breakdown
    guard h_{j+1,j} <= 1e-14 beta ends that cycle (D14)."""
    x = np.zeros_like(b) if x0 is None else x0.copy()
    for _ in range(ko):
        r = b - A(x)
        beta = np.linalg.norm(r)
        if beta == 0.0:
            break
        V = [r / beta]
        Z = []
        Hm = np.zeros((ki + 1, ki), np.complex128)
        k = ki
        for j in range(ki):
            z = M(V[j]) if M is not None else V[j]
            Z.append(z)
            w = A(z)
            for i in range(j + 1):
                Hm[i, j] = np.vdot(V[i], w)
                w = w - Hm[i, j] * V[i]
            Hm[j + 1, j] = np.linalg.norm(w)
            if Hm[j + 1, j].real <= BREAKDOWN * beta:
                k = j + 1
                break
            V.append(w / Hm[j + 1, j])
        e1 = np.zeros(k + 1, np.complex128)
        e1[0] = beta
        y = np.linalg.lstsq(Hm[:k + 1, :k], e1, rcond=None)[0]
        for i in range(k):
            x = x + y[i] * Z[i]
    return x


def vcycle(hier: Hierarchy, l: int, b: np.ndarray, adjoint: bool = False) -> np.ndarray:
    """Alg. 1 with the recursion of Fig. 3 and the fixed counts of D14."""
    o = hier.opts
    A = hier.op(l, adjoint)
    x = krylov(A, b, None, o.ks_o, o.ks_i)                          # pre-smooth from 0
    r = b - A(x)                                                     # residual
    rc = hier.R[l] @ r                                               # restrict
    Ac = hier.op(l + 1, adjoint)
    if l + 1 == o.levels - 1:
        xc = krylov(Ac, rc, None, o.kc_o, o.kc_i)                    # coarsest: GMRES
    else:
        xc = krylov(Ac, rc, None, o.kc_o, o.kc_i,
                    M=lambda v: vcycle(hier, l + 1, v, adjoint))    # FGMRES + V-cycle
    x = x + hier.P[l] @ xc                                           # prolong + correct
    return krylov(A, b, x, o.ks_o, o.ks_i)                           # post-smooth


def solve(hier: Hierarchy, b: np.ndarray, rtol: float = 1e-6, k_inner: int = 5,
          max_outer: int = 50, adjoint: bool = False, precond: bool = True):
    """Outer FGMRES(k_inner) restarted until the true residual <= rtol (R23), x0 = 0.
    Returns (x, outer_cycles, rel_residual)."""
    A = hier.op(0, adjoint)
    M = (lambda v: vcycle(hier, 0, v, adjoint)) if precond else None
    nb = np.linalg.norm(b)
    x = np.zeros_like(b)
    cycles = 0
    while True:
        rel = np.linalg.norm(b - A(x)) / nb
        if rel <= rtol or cycles >= max_outer:
            return x, cycles, float(rel)
        x = krylov(A, b, x, 1, k_inner, M)
        cycles += 1


def peak_vectors(k_i=5, ks_i=5, kc_i=5, dim=3) -> float:
    """P:299 peak memory in units of fine-grid vectors (R18); the coarsening factor is 2^d."""
    c = 2.0 ** dim
    return (2 * k_i + 6) + max(ks_i + 5, (2 * kc_i + 6) / c + max((ks_i + 5) / c, (2 * kc_i + 6) / c**2))
