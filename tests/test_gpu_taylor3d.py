"""3D GPU Taylor tests of the gradient (§6.1: the paper's Taylor test is 3D,
fields solved to a relative residual of 1e-10), with the library's own f and g from
fwi_misfit_grad: e0(t) = |f(m + t dm) - f(m)| = O(t) and e1(t) = |f(m + t dm) - f(m) -
t <g, dm>| = O(t^2), checked as slopes 1 and 2 (+-0.25) over successive halvings.

* the cfg4 replica (24^3 + PML 6, same generator; observed data from the oracle's LU);
* cfg4 at FULL size (200^3 + PML 20, 6 Hz; the first two surface sources, all 40,000
  receivers; observed data = the GPU's own FORW_MODEL at the true model, rtol 1e-10 — an
  input of the test only: the expected values are the slopes, fixed by Taylor's theorem).
dm = m_true - m0 (the 5 % smoothed perturbation of the generator)."""
import numpy as np
import pytest

import synth
from oracle import discretize as D
from oracle import fwi
from paper_1703_09268_b200 import api

pytestmark = pytest.mark.gpu


def _taylor(p, d, ts, max_rhs, src_range=None):
    a = dict(grid=api.Grid.of(p), freqs=p.freqs, src_node=p.src, rec_node=p.rec, d_obs=d, pml=api.Pml(v_ref=4500.0),
             dtype=api.C128, opts=api.SolveOpts(rtol=1e-10, max_outer=200), max_rhs=max_rhs, src_range=src_range)

    def fg_at(m):
        fg, rep = api.fwi_misfit_grad(m_slowness2=m, **a)
        assert all(r["converged"] for r in rep)
        return fg.cpu().numpy()

    base = fg_at(p.m)
    f0, g = base[0], base[1:].reshape(p.m.shape)
    dm = p.m_true - p.m
    gdm = float(np.sum(g * dm))
    e0, e1 = [], []
    for t in ts:
        ft = fg_at(p.m + t * dm)[0]
        e0.append(abs(ft - f0))
        e1.append(abs(ft - f0 - t * gdm))
    s0 = np.log2(np.array(e0[:-1]) / np.array(e0[1:]))
    s1 = np.log2(np.array(e1[:-1]) / np.array(e1[1:]))
    return s0, s1, e0, e1


def test_taylor_3d_cfg4_replica():
    p = synth.cfg4_replica()
    pml = D.PmlParams(v_ref=4500.0)
    d = fwi.forward_data(p, pml, p.m_true)
    s0, s1, e0, e1 = _taylor(p, d, 2.0 ** -np.arange(2, 8), max_rhs=4)
    assert np.all(np.abs(s0 - 1) < 0.25), (s0, e0)
    assert np.all(np.abs(s1 - 2) < 0.25), (s1, e1)


def test_taylor_3d_cfg4_fullsize():
    p = synth.cfg4()
    p = p.with_(src=p.src[:2])
    d, rep = api.fwi_forward(api.Grid.of(p), p.m_true, p.freqs, p.src, p.rec, api.Pml(v_ref=4500.0), api.C128,
                             api.SolveOpts(rtol=1e-10, max_outer=200), max_rhs=2)
    assert all(r["converged"] for r in rep)
    s0, s1, e0, e1 = _taylor(p, d, 2.0 ** -np.arange(2, 6), max_rhs=2)
    assert np.all(np.abs(s0 - 1) < 0.25), (s0, e0)
    assert np.all(np.abs(s1 - 2) < 0.25), (s1, e1)
