"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This package holds NO arithmetic of the method (no operator, no PML, no solve,
no misfit): only grids, velocity models, acquisition geometry and random
vectors, generated from fixed seeds. Both sides (``oracle/`` and the CUDA path
via ``paper_1703_09268_b200``) consume what it produces; neither imports the
other. Recipes follow SURVEY.md §8(d) d.1 and are restated in DESIGN.md §3.
"""
from .configs import (  # noqa: F401
    Problem, cfg1, cfg2, cfg3, cfg3_batch, cfg4, cfg4_replica, cfg5, tiny2d, tiny3d,
    const_problem, random_complex, random_real, node_id, table3_grid, table3, TABLE3_CELLS,
)
