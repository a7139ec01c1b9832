"""GPU parity of a7-a9 through the C ABI: fwi_misfit_grad f and g vs the oracle (LU fields)
<= 1e-5 (north star), FORW_MODEL data, GPU Taylor test, zero residual at the
true model, source-shard additivity, empty shard."""
import numpy as np
import pytest

import synth
from oracle import discretize as D
from oracle import fwi
from paper_1703_09268_b200 import api

from .helpers import rel

pytestmark = pytest.mark.gpu

VREF = 3000.0


def _args(p, dtype=api.C128, rtol=1e-8, max_rhs=4, **kw):
    return dict(grid=api.Grid.of(p), freqs=p.freqs, src_node=p.src, rec_node=p.rec, pml=api.Pml(v_ref=VREF),
                dtype=dtype, opts=api.SolveOpts(rtol=rtol), max_rhs=max_rhs, **kw)


@pytest.mark.parametrize("make", [synth.tiny2d, synth.tiny3d])
def test_forward_data_matches_oracle(make):
    p = make()
    pml = D.PmlParams(v_ref=VREF)
    d_ref = fwi.forward_data(p, pml, p.m_true)
    d, rep = api.fwi_forward(m_slowness2=p.m_true, **_args(p))
    assert rel(d, d_ref) <= 1e-6


@pytest.mark.parametrize("make", [synth.tiny2d, synth.tiny3d])
@pytest.mark.parametrize("dtype", [api.C128, api.C64])
@pytest.mark.parametrize("rtol", [1e-6, 1e-8])
def test_misfit_grad_matches_oracle(make, dtype, rtol):
    p = make()
    pml = D.PmlParams(v_ref=VREF)
    d = fwi.forward_data(p, pml, p.m_true)
    f_ref, g_ref = fwi.misfit_grad(p, pml, d)
    fg, rep = api.fwi_misfit_grad(m_slowness2=p.m, d_obs=d, **_args(p, dtype, rtol=rtol, max_rhs=2))
    fg = fg.cpu().numpy()
    assert abs(fg[0] - f_ref) <= 1e-5 * f_ref
    assert rel(fg[1:], g_ref.ravel()) <= 1e-5
    assert all(r["converged"] for r in rep)


def test_gpu_taylor_test():
    """e0 = O(h), e1 = O(h^2) with the GPU's own f and g (fields solved to 1e-10)."""
    p = synth.tiny2d()
    pml = D.PmlParams(v_ref=VREF)
    d = fwi.forward_data(p, pml, p.m_true)
    a = _args(p, rtol=1e-10)

    def fg_at(m):
        return api.fwi_misfit_grad(m_slowness2=m, d_obs=d, **a)[0].cpu().numpy()

    base = fg_at(p.m)
    f0, g = base[0], base[1:].reshape(p.m.shape)
    dm = p.m_true - p.m
    ts = 2.0 ** -np.arange(2, 9)
    e0, e1 = [], []
    for t in ts:
        ft = fg_at(p.m + t * dm)[0]
        e0.append(abs(ft - f0))
        e1.append(abs(ft - f0 - t * np.sum(g * dm)))
    s0 = np.log2(np.array(e0[:-1]) / np.array(e0[1:]))
    s1 = np.log2(np.array(e1[:-1]) / np.array(e1[1:]))
    assert np.all(np.abs(s0 - 1) < 0.25), s0
    assert np.all(np.abs(s1 - 2) < 0.25), s1


def test_zero_residual_and_shards():
    p = synth.tiny2d(nsrc=5)
    pml = D.PmlParams(v_ref=VREF)
    d = fwi.forward_data(p, pml, p.m_true)
    fg_true = api.fwi_misfit_grad(m_slowness2=p.m_true, d_obs=d, **_args(p, rtol=1e-10))[0].cpu().numpy()
    fg0 = api.fwi_misfit_grad(m_slowness2=p.m, d_obs=d, **_args(p))[0].cpu().numpy()
    assert fg_true[0] <= 1e-10 * fg0[0]
    parts = [api.fwi_misfit_grad(m_slowness2=p.m, d_obs=d, src_range=r, **_args(p))[0].cpu().numpy()
             for r in ((0, 2), (2, 5), (5, 5))]
    assert np.all(parts[2] == 0)                       # empty shard: f = 0, g = 0
    tot = parts[0] + parts[1] + parts[2]
    assert abs(tot[0] - fg0[0]) <= 1e-9 * fg0[0]
    assert rel(tot[1:], fg0[1:]) <= 1e-9


@pytest.mark.parametrize("max_rhs", [1, 4, 9])
@pytest.mark.parametrize("dtype", [api.C128, api.C64])
def test_joint_frequency_batches_match_oracle(max_rhs, dtype):
    """Joint (source, frequency) batches: 3 sources x 3 frequencies in batches of
    1 (one operator each), 4 (batches spanning two frequencies) and 9 (all three operators in
    one batched solve, RHS converging at different cycles) give the oracle's f and g."""
    p = synth.tiny2d().with_(freqs=(6.0, 9.0, 12.0))
    pml = D.PmlParams(v_ref=VREF)
    d = fwi.forward_data(p, pml, p.m_true)
    f_ref, g_ref = fwi.misfit_grad(p, pml, d)
    fg, rep = api.fwi_misfit_grad(m_slowness2=p.m, d_obs=d, **_args(p, dtype, rtol=1e-8, max_rhs=max_rhs))
    fg = fg.cpu().numpy()
    assert len(rep) == 18 and all(r["converged"] for r in rep)
    assert abs(fg[0] - f_ref) <= 1e-5 * f_ref
    assert rel(fg[1:], g_ref.ravel()) <= 1e-5


def test_joint_batch_forward_data():
    p = synth.tiny3d().with_(freqs=(6.0, 8.0))
    pml = D.PmlParams(v_ref=VREF)
    d_ref = fwi.forward_data(p, pml, p.m_true)
    d, rep = api.fwi_forward(m_slowness2=p.m_true, **_args(p, max_rhs=4))
    assert rel(d, d_ref) <= 1e-6


@pytest.mark.parametrize("make", [synth.tiny2d, synth.tiny3d])
def test_graph_cache_survives_model_and_frequency_changes(make):
    """The captured V-cycle graphs are kept across fwi_* calls (keyed by the batch's omegas;
    the model is rewritten in place): alternating models and frequency sets on the cached op
    must give the oracle's f and g every time, and repeat bit for bit."""
    p = make()
    pml = D.PmlParams(v_ref=VREF)
    f0 = float(p.freqs[0])
    cases = [(p.m, (f0,)), (0.5 * (p.m + p.m_true), (f0,)), (p.m, (f0, 0.8 * f0)), (p.m_true * 1.03, (0.8 * f0,)),
             (p.m, (f0,)), (0.5 * (p.m + p.m_true), (f0,)), (p.m, (f0, 0.8 * f0))]
    fgs = []
    for i, (m, freqs) in enumerate(cases):
        q = p.with_(freqs=freqs)
        d = fwi.forward_data(q, pml, q.m_true)
        f_ref, g_ref = fwi.misfit_grad(q, pml, d, m_int=m)
        fg, rep = api.fwi_misfit_grad(m_slowness2=m, d_obs=d, **_args(q, rtol=1e-8, max_rhs=3))
        fg = fg.cpu().numpy().copy()
        assert all(r["converged"] for r in rep)
        assert abs(fg[0] - f_ref) <= 1e-5 * f_ref, (i, fg[0], f_ref)
        assert rel(fg[1:], g_ref.ravel()) <= 1e-5, i
        fgs.append(fg)
    for a, b in ((0, 4), (1, 5), (2, 6)):   # identical inputs: live, captured and replayed V-cycles agree bitwise
        assert np.array_equal(fgs[a], fgs[b]), (a, b)
