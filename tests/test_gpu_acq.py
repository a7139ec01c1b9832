"""GPU parity of off-grid sources and receivers (Kaiser-windowed sinc,
PAPER P:139, DESIGN R33) through the C ABI: forward data and misfit / gradient vs the oracle
(oracle/interp.py, LU fields), densely packed receivers whose interpolation supports overlap,
on-node points identical to the node-id path, and rejection of points outside the interior."""
import numpy as np
import pytest

import synth
from oracle import discretize as D
from oracle import interp as I
from paper_1703_09268_b200 import api
from paper_1703_09268_b200._lib import HelmError

from .helpers import rel

pytestmark = pytest.mark.gpu

VREF = 3000.0


def _acq(p, seed=0, nrec=None):
    rng = np.random.default_rng(seed)
    ns = len(p.src)
    src = np.zeros((ns, 3))
    src[:, 0] = rng.uniform(2 * p.h, (p.n[0] - 3) * p.h, ns)
    src[:, 2] = rng.uniform(1.3 * p.h, 3.1 * p.h, ns)
    if p.ndim == 3:
        src[:, 1] = rng.uniform(2 * p.h, (p.n[1] - 3) * p.h, ns)
    nrec = nrec or (len(p.rec) if p.ndim == 2 else 24)
    rec = np.zeros((nrec, 3))
    rec[:, 0] = np.linspace(0.3 * p.h, (p.n[0] - 1.2) * p.h, nrec)   # ~0.7 h apart in 2D: supports overlap
    rec[:, 2] = 0.6 * p.h
    if p.ndim == 3:
        rec[:, 1] = rng.uniform(0.0, (p.n[1] - 1) * p.h, nrec)
    return src, rec


def _args(p, dtype=api.C128, rtol=1e-8, max_rhs=4):
    return dict(grid=api.Grid.of(p), freqs=p.freqs, pml=api.Pml(v_ref=VREF), dtype=dtype,
                opts=api.SolveOpts(rtol=rtol), max_rhs=max_rhs)


@pytest.mark.parametrize("make", [synth.tiny2d, synth.tiny3d])
def test_offgrid_forward_matches_oracle(make):
    p = make()
    sx, rx = _acq(p)
    ref = I.forward_data(p, D.PmlParams(v_ref=VREF), sx, rx, p.m_true)
    d, rep = api.fwi_forward_acq(m_slowness2=p.m_true, acq=api.Acq(sx, rx), **_args(p))
    assert all(r["converged"] for r in rep)
    assert rel(d, ref) <= 1e-6


@pytest.mark.parametrize("make", [synth.tiny2d, synth.tiny3d])
@pytest.mark.parametrize("dtype", [api.C128, api.C64])
def test_offgrid_misfit_grad_matches_oracle(make, dtype):
    p = make()
    sx, rx = _acq(p, 1)
    pml = D.PmlParams(v_ref=VREF)
    d = I.forward_data(p, pml, sx, rx, p.m_true)
    f_ref, g_ref = I.misfit_grad(p, pml, d, sx, rx)
    fg, rep = api.fwi_misfit_grad_acq(m_slowness2=p.m, acq=api.Acq(sx, rx), d_obs=d,
                                      **_args(p, dtype, rtol=1e-8 if dtype == api.C128 else 1e-6, max_rhs=2))
    fg = fg.cpu().numpy()
    assert all(r["converged"] for r in rep)
    assert abs(fg[0] - f_ref) <= 1e-5 * f_ref
    assert rel(fg[1:], g_ref.ravel()) <= 1e-5


def test_on_node_points_equal_the_node_path():
    p = synth.tiny2d()
    node_xyz = lambda ids: np.stack([ids % p.n[0] * p.h, 0 * ids, ids // p.n[0] * p.h], 1).astype(float)  # noqa: E731
    a = _args(p)
    d_node, _ = api.fwi_forward(m_slowness2=p.m_true, src_node=p.src, rec_node=p.rec, **a)
    d_acq, _ = api.fwi_forward_acq(m_slowness2=p.m_true, acq=api.Acq(node_xyz(p.src), node_xyz(p.rec)), **a)
    assert rel(d_acq, d_node) <= 1e-14
    fg_n, _ = api.fwi_misfit_grad(m_slowness2=p.m, src_node=p.src, rec_node=p.rec, d_obs=d_node, **a)
    fg_a, _ = api.fwi_misfit_grad_acq(m_slowness2=p.m, acq=api.Acq(node_xyz(p.src), node_xyz(p.rec)), d_obs=d_node, **a)
    # same fields; f is reduced in a different (fixed) order and the adjoint source carries
    # signed zeros around each receiver: agreement to rounding, not bitwise
    assert rel(fg_a.cpu().numpy(), fg_n.cpu().numpy()) <= 1e-12


def test_points_outside_are_rejected():
    p = synth.tiny2d()
    sx, rx = _acq(p)
    bad = rx.copy()
    bad[3, 0] = -0.5 * p.h
    with pytest.raises(HelmError, match="point 3"):
        api.fwi_forward_acq(m_slowness2=p.m, acq=api.Acq(sx, bad), **_args(p))
    bad = rx.copy()
    bad[0, 1] = 1.0
    with pytest.raises(HelmError, match="y = 0"):
        api.fwi_forward_acq(m_slowness2=p.m, acq=api.Acq(sx, bad), **_args(p))


def test_source_frequency_subset_matches_oracle():
    """Batch-mode subset: f, g over the selected (frequency, source) pairs equal the
    oracle's per-frequency sums over the selected sources; the full mask equals
    fwi_misfit_grad; an empty mask gives zeros."""
    from oracle import fwi
    p = synth.tiny2d(nsrc=4).with_(freqs=(7.0, 9.0))
    pml = D.PmlParams(v_ref=VREF)
    d = fwi.forward_data(p, pml, p.m_true)
    mask = np.array([[1, 0, 1, 1], [0, 1, 0, 1]], np.uint8)
    f_ref, g_ref = 0.0, np.zeros(p.m.shape)
    for fi, fr in enumerate(p.freqs):
        sel = np.flatnonzero(mask[fi])
        q = p.with_(freqs=(fr,))
        fpart, gpart = fwi.misfit_grad(q, pml, d[fi:fi + 1][:, sel], src_ids=p.src[sel])
        f_ref += fpart
        g_ref += gpart
    a = dict(grid=api.Grid.of(p), freqs=p.freqs, src_node=p.src, rec_node=p.rec, pml=api.Pml(v_ref=VREF),
             opts=api.SolveOpts(rtol=1e-8), max_rhs=3)
    fg, rep = api.fwi_misfit_grad_subset(m_slowness2=p.m, d_obs=d, pair_mask=mask, **a)
    fg = fg.cpu().numpy()
    assert len(rep) == 2 * int(mask.sum()) and all(r["converged"] for r in rep)
    assert abs(fg[0] - f_ref) <= 1e-5 * f_ref and rel(fg[1:], g_ref.ravel()) <= 1e-5
    full, _ = api.fwi_misfit_grad_subset(m_slowness2=p.m, d_obs=d, pair_mask=np.ones_like(mask), **a)
    ref_full, _ = api.fwi_misfit_grad(m_slowness2=p.m, d_obs=d, **a)
    assert rel(full.cpu().numpy(), ref_full.cpu().numpy()) <= 1e-12
    empty, rep0 = api.fwi_misfit_grad_subset(m_slowness2=p.m, d_obs=d, pair_mask=np.zeros_like(mask), **a)
    assert rep0 == [] and float(empty.abs().max()) == 0.0
