"""B200-native hot path of arXiv 1703.09268 (Da Silva & Herrmann): the per-source,
per-frequency PML Helmholtz solve (FGMRES + ML-GMRES) feeding the FWI misfit and gradient.

The product is libhelm.so (csrc/, C ABI in include/helm.h); this package is its thin
ctypes binding (api.py) plus the source-sharded multi-GPU driver (dist.py).
"""
from .api import (  # noqa: F401
    C64, C128, Grid, MlOpts, Pml, SolveOpts, HelmOp, helm_setup, helm_apply, helm_solve, helm_vcycle,
    helm_transfer, fwi_misfit_grad, fwi_forward,
)
