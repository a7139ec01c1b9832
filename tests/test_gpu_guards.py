"""Guards of the C ABI added in round 2:

* helm_setup warns (helm_last_error, status OK) when the finest grid has fewer than 4 points
  per wavelength at v_min;
* a cached fwi op (same geometry, reused across calls) still rejects a bad model or PML;
* 2D joint batches close before the march kernel's shared-memory z table overflows (deep
  grid x several frequencies): f, g still match the oracle; a grid too deep for even one
  operator fails with HELM_ERR_SHAPE instead of a CUDA launch error."""
import numpy as np
import pytest
import torch

import synth
from oracle import discretize as D
from oracle import fwi
from paper_1703_09268_b200 import _lib, api

from .helpers import rel

pytestmark = pytest.mark.gpu


def test_coarse_grid_warning():
    p = synth.tiny3d()
    lib = _lib.load()
    # 20 m spacing, v_min ~ 1700 m/s: 4 ppw at ~21 Hz; 40 Hz gives ~2 ppw
    api.helm_setup(api.Grid.of(p), p.m, 2 * np.pi * 40.0, api.Pml(v_ref=3000.0), api.C128, max_rhs=1)
    assert b"points per wavelength" in lib.helm_last_error()
    api.helm_setup(api.Grid.of(p), p.m, 2 * np.pi * 8.0, api.Pml(v_ref=3000.0), api.C128, max_rhs=1)
    assert b"points per wavelength" not in lib.helm_last_error()


def test_cached_fwi_op_validates_model_and_pml():
    p = synth.tiny2d()
    pml = D.PmlParams(v_ref=3000.0)
    d = fwi.forward_data(p, pml, p.m_true)
    a = dict(grid=api.Grid.of(p), freqs=p.freqs, src_node=p.src, rec_node=p.rec, d_obs=d, dtype=api.C128,
             opts=api.SolveOpts(rtol=1e-6), max_rhs=4)
    api.fwi_misfit_grad(m_slowness2=p.m, pml=api.Pml(v_ref=3000.0), **a)      # creates the cached op
    bad = p.m.copy()
    bad.flat[7] = np.nan
    with pytest.raises(_lib.HelmError) as e:
        api.fwi_misfit_grad(m_slowness2=bad, pml=api.Pml(v_ref=3000.0), **a)
    assert e.value.status == _lib.HELM_ERR_ARG
    with pytest.raises(_lib.HelmError) as e:
        api.fwi_misfit_grad(m_slowness2=p.m, pml=api.Pml(R=1.5, v_ref=3000.0), **a)
    assert e.value.status == _lib.HELM_ERR_ARG


def test_deep_2d_grid_splits_joint_batches():
    """nz_ext = 1000 complex128: 48 KB of z table per operator, so at most 3 operators fit next
    to the march ring; 4 frequencies in one call are split over two batched solves. (Solved to
    1e-10: the residual P_r u - d of this deep model's small blob is ~1e-3 of the direct wave at
    the receivers, so solve errors are amplified ~1e3 in f and g — at 1e-8 the oracle
    comparison measured 5e-7 / 4.7e-5 for every max_rhs, i.e. with or without the split.)"""
    p = synth.tiny2d(nx=40, nz=960, pml=20, nsrc=2).with_(freqs=(6.0, 8.0, 10.0, 12.0))
    pml = D.PmlParams(v_ref=3000.0)
    d = fwi.forward_data(p, pml, p.m_true)
    f_ref, g_ref = fwi.misfit_grad(p, pml, d)
    fg, rep = api.fwi_misfit_grad(api.Grid.of(p), p.m, p.freqs, p.src, p.rec, d, api.Pml(v_ref=3000.0), api.C128,
                                  api.SolveOpts(rtol=1e-10, max_outer=400), max_rhs=8)
    fg = fg.cpu().numpy()
    assert all(r["converged"] for r in rep)
    assert abs(fg[0] - f_ref) <= 1e-5 * f_ref
    assert rel(fg[1:], g_ref.ravel()) <= 1e-5


def test_too_deep_2d_grid_fails_cleanly():
    p = synth.tiny2d(nx=5, nz=6000, pml=2, nsrc=1)
    op = api.helm_setup(api.Grid.of(p), p.m, 2 * np.pi * 1.0, api.Pml(v_ref=3000.0), api.C128, max_rhs=1,
                        mlopts=api.MlOpts(levels=0))
    x = torch.zeros(1, p.n_ext, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    with pytest.raises(_lib.HelmError) as e:
        api.helm_apply(op, x, y)
    assert e.value.status == _lib.HELM_ERR_SHAPE
