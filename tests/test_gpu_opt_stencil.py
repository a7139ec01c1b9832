"""GPU parity of the paper's higher-order stencils ("9pt
optimal" [23] / "compact 27-pt" [60]; DESIGN readings R34 / R35) through the C ABI with
grid.stencil = HELM_OPT, against the oracle's assembled operator of the same reading:

* helm_apply forward / adjoint on ragged multi-tile grids (3D 27-pt plane kernel with the
  halo'd model tiles; 2D 9-pt march kernel): <= 1e-12 complex128, <= 1e-5 complex64;
* one V-cycle vs the numpy mirror on the opt stencil (every level rediscretised with it):
  <= 1e-12;
* preconditioned solves vs LU (<= 1e-5, R24), misfit and gradient (A = M in T^*, Eqs. 7-8)
  and J^H y vs the oracle (<= 1e-5 / 1e-6), and a GPU Taylor test (slopes 1 and 2);
* at 5 points per wavelength the GPU's opt solution is several times closer to the analytic
  Green's function than its STD2 solution (the reason the paper uses these stencils);
* the Born-source calls reject the opt stencil."""
import numpy as np
import pytest
import torch

import synth
from oracle import discretize as D
from oracle import fwi, green, mlgmres
from oracle.solve import LU
from paper_1703_09268_b200 import _lib, api

from .helpers import rel, to_dev, to_host
from .test_gpu_operator import medium2d, medium3d

pytestmark = pytest.mark.gpu


def _op(p, dtype=api.C128, nrhs=3, vref=None, levels=None):
    w = 2 * np.pi * p.freqs[0]
    vref = float(np.max(1 / np.sqrt(p.m))) * 1.1 if vref is None else vref
    pml = D.PmlParams(v_ref=vref)
    ml = api.MlOpts(levels=levels) if levels is not None else None
    op = api.helm_setup(api.Grid.of(p), p.m, w, api.Pml(pml.R, pml.power, pml.v_ref), dtype, max_rhs=nrhs, mlopts=ml)
    return op, w, pml


# complex64 3D needs an even extended nx on every level (TMA rows): medium3d (72 -> 36 -> 18)
CASES = [(medium3d, api.C128), (medium3d, api.C64), (medium2d, api.C128), (medium2d, api.C64),
         (synth.tiny3d, api.C128), (synth.cfg1, api.C128), (synth.cfg1, api.C64)]


@pytest.mark.parametrize("make,dtype", CASES)
@pytest.mark.parametrize("adjoint", [0, 1])
def test_apply_matches_oracle(make, dtype, adjoint):
    p = make().with_(stencil="opt")
    op, w, pml = _op(p, dtype, nrhs=3, levels=0)
    H = D.helmholtz_matrix(p, w, pml)
    A = H.conj().T.tocsr() if adjoint else H
    x = synth.random_complex((3, p.n_ext), 1)
    td = api.TORCH_DTYPE[dtype]
    y = torch.empty(3, p.n_ext, dtype=td, device="cuda")
    api.helm_apply(op, to_dev(x, td), y, adjoint=adjoint)
    xr = x.astype(np.complex64).astype(np.complex128) if dtype == api.C64 else x
    Y = to_host(y)
    tol = 1e-12 if dtype == api.C128 else 1e-5
    for r in range(3):
        assert rel(Y[r], A @ xr[r]) <= tol, r


@pytest.mark.parametrize("make,adjoint", [(synth.tiny2d, 0), (synth.tiny3d, 1), (medium3d, 0)])
def test_vcycle_matches_mirror(make, adjoint):
    p = make().with_(stencil="opt")
    op, w, pml = _op(p, nrhs=2)
    hier = mlgmres.Hierarchy(p, w, pml)
    b = synth.random_complex((2, p.n_ext), 1)
    z = torch.zeros(2, p.n_ext, dtype=torch.complex128, device="cuda")
    api.helm_vcycle(op, to_dev(b), z, level=0, adjoint=adjoint)
    zg = to_host(z)
    for r in range(2):
        assert rel(zg[r], mlgmres.vcycle(hier, 0, b[r], adjoint=bool(adjoint))) <= 1e-12


def even3d():
    """Small 3D grid whose extended nx is even on every level (24 -> 12 -> 6): complex64 TMA rows."""
    return synth.tiny3d(n=(16, 11, 9))


@pytest.mark.parametrize("make,dtype,rtol", [(synth.tiny3d, api.C128, 1e-6), (synth.cfg1, api.C128, 1e-6),
                                              (synth.cfg1, api.C64, 1e-6), (even3d, api.C64, 1e-6),
                                              (even3d, api.C128, 1e-6)])
@pytest.mark.parametrize("adjoint", [0, 1])
def test_solve_matches_lu(make, dtype, rtol, adjoint):
    """Solution rel-L2 <= 1e-5 (R24). (medium3d — point-wise random 1500-3000 m/s, 131k unknowns
    — measured 1.15e-5 at rtol 1e-6: worse conditioned; its 3D LU is too slow for this suite.)"""
    p = make().with_(stencil="opt")
    op, w, pml = _op(p, dtype, nrhs=1)
    H = D.helmholtz_matrix(p, w, pml)
    q = fwi.source_matrix(p, w, p.src[:1])[:, 0]
    td = api.TORCH_DTYPE[dtype]
    x = torch.zeros(1, p.n_ext, dtype=td, device="cuda")
    rep = api.helm_solve(op, to_dev(q, td), x, adjoint=adjoint, opts=api.SolveOpts(rtol=rtol))
    assert rep[0]["converged"] and rep[0]["rel_residual"] <= rtol
    assert rel(to_host(x)[0], LU(H).solve(q, adjoint=bool(adjoint))) <= 1e-5


@pytest.mark.parametrize("make,dtype", [(synth.tiny2d, api.C128), (synth.tiny2d, api.C64), (synth.tiny3d, api.C128)])
def test_misfit_grad_and_jacobian_adjoint_match_oracle(make, dtype):
    p = make().with_(stencil="opt")
    pml = D.PmlParams(v_ref=3000.0)
    d = fwi.forward_data(p, pml, p.m_true)
    f_ref, g_ref = fwi.misfit_grad(p, pml, d)
    a = dict(grid=api.Grid.of(p), freqs=p.freqs, src_node=p.src, rec_node=p.rec, pml=api.Pml(v_ref=3000.0),
             dtype=dtype, opts=api.SolveOpts(rtol=1e-8), max_rhs=4)
    fg, rep = api.fwi_misfit_grad(m_slowness2=p.m, d_obs=d, **a)
    fg = fg.cpu().numpy()
    assert all(r["converged"] for r in rep)
    assert abs(fg[0] - f_ref) <= 1e-5 * f_ref
    assert rel(fg[1:], g_ref.ravel()) <= 1e-5
    d_gpu, _ = api.fwi_forward(m_slowness2=p.m_true, **a)
    assert rel(d_gpu, d) <= 1e-6
    y = synth.random_complex(d.shape, 7)
    g, _ = api.fwi_jacobian_adjoint(m_slowness2=p.m, y=y, **a)
    assert rel(g.cpu().numpy(), fwi.jacobian_adjoint(p, pml, y, p.m).ravel()) <= 1e-5


def test_gpu_taylor_opt_3d():
    p = synth.tiny3d().with_(stencil="opt")
    pml = D.PmlParams(v_ref=3000.0)
    d = fwi.forward_data(p, pml, p.m_true)
    a = dict(grid=api.Grid.of(p), freqs=p.freqs, src_node=p.src, rec_node=p.rec, d_obs=d, pml=api.Pml(v_ref=3000.0),
             dtype=api.C128, opts=api.SolveOpts(rtol=1e-10), max_rhs=2)
    base = api.fwi_misfit_grad(m_slowness2=p.m, **a)[0].cpu().numpy()
    f0, g = base[0], base[1:].reshape(p.m.shape)
    dm = p.m_true - p.m
    e0, e1 = [], []
    ts = 2.0 ** -np.arange(2, 8)
    for t in ts:
        ft = api.fwi_misfit_grad(m_slowness2=p.m + t * dm, **a)[0].cpu().numpy()[0]
        e0.append(abs(ft - f0))
        e1.append(abs(ft - f0 - t * np.sum(g * dm)))
    s0, s1 = np.log2(np.array(e0[:-1]) / e0[1:]), np.log2(np.array(e1[:-1]) / e1[1:])
    assert np.all(np.abs(s0 - 1) < 0.25), s0
    assert np.all(np.abs(s1 - 2) < 0.25), s1


def test_green_at_5_ppw_better_than_std2():
    v, h = 2000.0, 10.0
    f = v / (5 * h)
    err = {}
    for st in ("std2", "opt"):
        p = synth.const_problem("g", 2, (161, 161), h, 30, v, f, [(80, 0, 80)]).with_(stencil=st)
        op, w, _ = _op(p, nrhs=1, vref=v)
        q = fwi.source_matrix(p, w, p.src)[:, 0]
        x = torch.zeros(1, p.n_ext, dtype=torch.complex128, device="cuda")
        rep = api.helm_solve(op, to_dev(q), x, opts=api.SolveOpts(rtol=1e-8, max_outer=200))
        assert rep[0]["converged"]
        err[st] = green.green_error(p, to_host(x)[0], v, f, int(p.src[0]))
    assert err["opt"] <= err["std2"] / 4, err


def test_born_calls_reject_opt():
    p = synth.tiny2d().with_(stencil="opt")
    with pytest.raises(_lib.HelmError) as e:
        api.fwi_jacobian(api.Grid.of(p), p.m, p.freqs, p.src, p.rec, np.zeros_like(p.m), api.Pml(v_ref=3000.0))
    assert e.value.status == _lib.HELM_ERR_ARG
