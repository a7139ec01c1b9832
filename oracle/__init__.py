"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct numpy/scipy implementation of what the hot path
computes: the PML Helmholtz operator assembled as an explicit
sparse matrix, its solution by sparse LU / GMRES, the least-squares misfit and
the adjoint-state gradient, the analytic Green's functions, and a numpy mirror
of the ML-GMRES preconditioner (Alg. 1 / Fig. 3 of the paper).

Rules:
  * only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
    ``cpu_baseline`` / ``--impl reference`` legs may import anything here;
  * it shares no code, table or constant generator with the CUDA path
    (``paper_1703_09268_b200``) and never imports it;
  * fp64 / complex128 throughout;
  * every function cites the PAPER.md passage (``P:<line>``) or the SURVEY.md
    reading (``D<n>`` / ``R<n>`` of §8(c)) it implements.

Parity status: every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` against something other than itself (closed forms,
textbook special cases, analytic Green's functions, the paper's printed
numbers, brute force). The ML-GMRES mirror is pinned to LU solves and to its
own algebraic identities; its exact iteration counts vs the paper's Table 3 are
"parity unpinned" (27-pt stencil, R4).
"""
from threadpoolctl import threadpool_limits as _tpl

# The oracle runs single-threaded (SURVEY §8(d) d.4 "one process" baseline): a
# multi-threaded BLAS makes SuperLU and the mirror's small vector ops ~20-100x
# slower on these hosts.
_tpl(1)

from .discretize import (  # noqa: F401
    PmlParams, default_pml, extension_matrix, extend, helmholtz_matrix, tables_1d,
    adjoint_tables_1d, ext_shape, interior_to_ext_index,
)
