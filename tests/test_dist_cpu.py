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


def _gn_eval(src_range, prob, pml, dm):
    from oracle import fwi
    s0, s1 = src_range
    return torch.from_numpy(fwi.gn_hessian(prob, pml, dm, src_ids=prob.src[s0:s1]).ravel()), None


def _jh_eval(src_range, prob, pml, y):
    from oracle import fwi
    s0, s1 = src_range
    return torch.from_numpy(fwi.jacobian_adjoint(prob, pml, y[:, s0:s1], src_ids=prob.src[s0:s1]).ravel()), None


def _worker_lin(rank, size, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    import synth
    from oracle import discretize as D
    p = synth.tiny2d(nsrc=5)
    pml = D.PmlParams(v_ref=3000.0)
    rng = np.random.default_rng(5)
    dm = rng.standard_normal(p.m.shape) * 1e-8
    y = rng.standard_normal((1, 5, len(p.rec))) + 1j * rng.standard_normal((1, 5, len(p.rec)))
    h, _, _ = hdist.gn_hessian_sharded(_gn_eval, nsrc=5, prob=p, pml=pml, dm=dm)
    g, _, _ = hdist.jacobian_adjoint_sharded(_jh_eval, nsrc=5, prob=p, pml=pml, y=y)
    if rank == 0:
        torch.save((h, g), out)
    dist.destroy_process_group()


def test_gloo_sharded_gn_and_jacobian_adjoint(tmp_path):
    """SURVEY §8(f) on the §8(e) sharding: all-reduced shards = the single-process oracle."""
    import synth
    from oracle import discretize as D, fwi
    out = str(tmp_path / "lin.pt")
    mp.spawn(_worker_lin, args=(2, _free_port(), out), nprocs=2, join=True)
    h, g = (t.numpy() for t in torch.load(out))
    p = synth.tiny2d(nsrc=5)
    pml = D.PmlParams(v_ref=3000.0)
    rng = np.random.default_rng(5)
    dm = rng.standard_normal(p.m.shape) * 1e-8
    y = rng.standard_normal((1, 5, len(p.rec))) + 1j * rng.standard_normal((1, 5, len(p.rec)))
    h_ref = fwi.gn_hessian(p, pml, dm).ravel()
    g_ref = fwi.jacobian_adjoint(p, pml, y).ravel()
    assert np.linalg.norm(h - h_ref) <= 1e-12 * np.linalg.norm(h_ref)
    assert np.linalg.norm(g - g_ref) <= 1e-12 * np.linalg.norm(g_ref)
