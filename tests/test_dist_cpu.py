"""World-size-2 gloo test of the source-sharded driver on CPU: the all-reduced [f || g] over
shards equals the single-process result, with the oracle standing in for the GPU
evaluator (tests may call oracle/)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1703_09268_b200 import dist as hdist


def test_shards_cover_sources_exactly_once():
    for S in (1, 7, 50, 64):
        for P in (1, 2, 3, 4, 8):
            seen = []
            for r in range(P):
                s0, s1 = hdist.shard(S, r, P)
                seen += list(range(s0, s1))
            assert seen == list(range(S))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_eval(src_range, prob, pml, d):
    from oracle import fwi
    s0, s1 = src_range
    f, g = fwi.misfit_grad(prob, pml, d[:, s0:s1], src_ids=prob.src[s0:s1])
    return torch.from_numpy(np.concatenate([[f], g.ravel()])), None


def _worker(rank, size, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    import synth
    from oracle import discretize as D, fwi
    p = synth.tiny2d(nsrc=5)
    pml = D.PmlParams(v_ref=3000.0)
    d = fwi.forward_data(p, pml, p.m_true)
    fg, _, rng = hdist.misfit_grad_sharded(_oracle_eval, nsrc=len(p.src), prob=p, pml=pml, d=d)
    if rank == 0:
        torch.save(fg, out)
    dist.destroy_process_group()


def test_gloo_allreduce_equals_single_process(tmp_path):
    import synth
    from oracle import discretize as D, fwi
    out = str(tmp_path / "fg.pt")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    fg = torch.load(out).numpy()
    p = synth.tiny2d(nsrc=5)
    pml = D.PmlParams(v_ref=3000.0)
    d = fwi.forward_data(p, pml, p.m_true)
    f, g = fwi.misfit_grad(p, pml, d)
    assert abs(fg[0] - f) <= 1e-12 * f
    assert np.linalg.norm(fg[1:] - g.ravel()) <= 1e-12 * np.linalg.norm(g)
