"""Reference solves of H u = q (ORACLE — test infrastructure only).

SURVEY.md §8(c) c.2 step 3: the method's result is the solution of a linear
system (D9); the oracle computes it directly with sparse LU ("sparse LU
decomposition ... reused across multiple sources") where feasible, otherwise
with unpreconditioned GMRES [72] to a tight tolerance, and certifies any
solution with its true residual (c.2 step 6).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla
from threadpoolctl import threadpool_limits


class LU:
    """splu(H) (COLAMD); ``solve(Q)`` for H^-1 Q and ``solve(Q, adjoint=True)`` for H^-H Q."""

    def __init__(self, H: sp.spmatrix):
        # SuperLU's small dense kernels go through BLAS; a multi-threaded BLAS makes them
        # ~100x slower on this host, so the factorization runs single-threaded.
        with threadpool_limits(1):
            self.lu = spla.splu(sp.csc_matrix(H))

    def solve(self, Q: np.ndarray, adjoint: bool = False) -> np.ndarray:
        Q = np.asarray(Q, np.complex128)
        with threadpool_limits(1):
            return self.lu.solve(Q, trans="H" if adjoint else "N")


class NotConverged(RuntimeError):
    pass


def gmres_solve(H: sp.spmatrix, q: np.ndarray, rtol: float = 1e-10, restart: int = 100,
                adjoint: bool = False, maxiter: int = 200) -> np.ndarray:
    """c.2 step 3 "otherwise": unpreconditioned restarted GMRES(restart) [72], x0 = 0,
    to ||q - Hx|| <= rtol ||q|| (D9); H^H for adjoints (D6 via the explicit transpose).
    Raises NotConverged when scipy reports info != 0 or the TRUE residual misses rtol."""
    A = H.conj().T.tocsr() if adjoint else H
    x, info = spla.gmres(A, q, rtol=rtol, atol=0.0, restart=restart, maxiter=maxiter)
    res = float(np.linalg.norm(q - A @ x) / np.linalg.norm(q))
    if info != 0 or not res <= rtol * (1 + 1e-6):
        raise NotConverged(f"GMRES({restart}) did not reach rtol {rtol:g}: info {info}, true residual {res:.3e}")
    return x


def rel_residual(H: sp.spmatrix, x: np.ndarray, b: np.ndarray, adjoint: bool = False) -> float:
    """c.2 step 6: ||b - H x|| / ||b|| (one SpMV with the oracle's own H)."""
    A = H.conj().T if adjoint else H
    return float(np.linalg.norm(b - A @ x) / np.linalg.norm(b))
