"""Source-sharded multi-GPU evaluation (Fig. 2).

One process per GPU. Rank r of P owns sources [floor(r S / P), floor((r+1) S / P)) for every
frequency, runs fwi_misfit_grad on its shard (each rank holds the full model and builds
its own hierarchy), and the ranks combine [f || g] with ONE in-place fp64 all_reduce (NCCL
over NVLink on GPUs; gloo in the CPU tests). There is no other traffic: a single solve is
never split across GPUs (the paper prefers "a larger number of sources distributed to
multiple nodes rather than ... multiple nodes solving a single problem").
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple

import torch
import torch.distributed as dist


def world() -> Tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard(nsrc: int, rank: int, size: int) -> Tuple[int, int]:
    """Contiguous, disjoint, covering: rank r gets [floor(r S/P), floor((r+1) S/P))."""
    return (rank * nsrc) // size, ((rank + 1) * nsrc) // size


def misfit_grad_sharded(evaluate: Optional[Callable] = None, nsrc: int = 0, group=None, **kw):
    """Evaluate this rank's source shard and all-reduce [f || g] in place (fixed shard order,
    R30). ``evaluate(src_range=(s0, s1), **kw) -> (fg tensor, reports)`` defaults to
    api.fwi_misfit_grad (GPU); tests pass a CPU evaluator under gloo."""
    if evaluate is None:
        from .api import fwi_misfit_grad as evaluate
    rank, size = world()
    s0, s1 = shard(nsrc, rank, size)
    fg, rep = evaluate(src_range=(s0, s1), **kw)
    if size > 1:
        dist.all_reduce(fg, op=dist.ReduceOp.SUM, group=group)
    return fg, rep, (s0, s1)


def _reduce_sharded(evaluate: Callable, nsrc: int, group=None, **kw):
    rank, size = world()
    s0, s1 = shard(nsrc, rank, size)
    out, rep = evaluate(src_range=(s0, s1), **kw)
    if size > 1:
        dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    return out, rep, (s0, s1)


def jacobian_adjoint_sharded(evaluate: Optional[Callable] = None, nsrc: int = 0, group=None, **kw):
    """J^H y (Listing 1 JACOBI_ADJ) summed over source shards: same sharding and ONE all-reduce
    as misfit_grad_sharded; y holds the whole survey, each rank reads its sources."""
    if evaluate is None:
        from .api import fwi_jacobian_adjoint as evaluate
    return _reduce_sharded(evaluate, nsrc, group, **kw)


def gn_hessian_sharded(evaluate: Optional[Callable] = None, nsrc: int = 0, group=None, **kw):
    """J^H J dm (Listing 1 HESS_GN) summed over source shards with ONE all-reduce."""
    if evaluate is None:
        from .api import fwi_gn_hessian as evaluate
    return _reduce_sharded(evaluate, nsrc, group, **kw)


def jacobian_sharded(evaluate: Optional[Callable] = None, nsrc: int = 0, **kw):
    """J dm (Listing 1 JACOBI_FORW) for this rank's sources: data-parallel with no collective —
    each rank's d_lin[:, s0:s1] is its own output (the caller gathers if it needs the whole)."""
    if evaluate is None:
        from .api import fwi_jacobian as evaluate
    rank, size = world()
    s0, s1 = shard(nsrc, rank, size)
    d, rep = evaluate(src_range=(s0, s1), **kw)
    return d, rep, (s0, s1)
