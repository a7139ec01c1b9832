"""GPU parity of SURVEY §8(f) rank 1 — Listing 1 JACOBI_FORW / JACOBI_ADJ / HESS_GN (P:167-180,
Table 1) — through the C ABI against the oracle's LU evaluation (oracle/fwi.py jacobian,
jacobian_adjoint, gn_hessian), plus properties that hold on the GPU side alone: the dot test
<J dm, y> = <dm, J^H y>, J^H (P_r u - d) = the gradient, GN dm = J^H (J dm), joint-batch and
source-shard invariance, the empty shard.

Tolerance: fields solved to rtol 1e-8 (c128) — each output is a linear functional of solves
with relative error <= cond-weighted 1e-8, so 1e-6 is loose for c128; the mixed c64 mode
(outer c128, D15) uses 1e-6 solves and 1e-4.
"""
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


def _dm(p, seed=7):
    rng = np.random.default_rng(seed)
    return 0.1 * np.abs(p.m).max() * rng.standard_normal(p.m.shape)


def _y(p, seed=8):
    rng = np.random.default_rng(seed)
    sh = (len(p.freqs), len(p.src), len(p.rec))
    return rng.standard_normal(sh) + 1j * rng.standard_normal(sh)


TOL = {api.C128: (1e-8, 1e-6), api.C64: (1e-6, 1e-4)}


@pytest.mark.parametrize("make", [synth.tiny2d, synth.tiny3d])
@pytest.mark.parametrize("dtype", [api.C128, api.C64])
def test_jacobian_matches_oracle(make, dtype):
    p = make()
    dm = _dm(p)
    ref = fwi.jacobian(p, D.PmlParams(v_ref=VREF), dm, p.m)
    rt, tol = TOL[dtype]
    d, rep = api.fwi_jacobian(m_slowness2=p.m, dm=dm, **_args(p, dtype, rtol=rt))
    assert len(rep) == 2 * len(p.freqs) * len(p.src) and all(r["converged"] for r in rep)
    assert rel(d, ref) <= tol


@pytest.mark.parametrize("make", [synth.tiny2d, synth.tiny3d])
@pytest.mark.parametrize("dtype", [api.C128, api.C64])
def test_jacobian_adjoint_matches_oracle(make, dtype):
    p = make()
    y = _y(p)
    ref = fwi.jacobian_adjoint(p, D.PmlParams(v_ref=VREF), y, p.m)
    rt, tol = TOL[dtype]
    g, rep = api.fwi_jacobian_adjoint(m_slowness2=p.m, y=y, **_args(p, dtype, rtol=rt))
    assert all(r["converged"] for r in rep)
    assert rel(g.cpu().numpy(), ref.ravel()) <= tol


@pytest.mark.parametrize("make", [synth.tiny2d, synth.tiny3d])
@pytest.mark.parametrize("dtype", [api.C128, api.C64])
def test_gn_hessian_matches_oracle(make, dtype):
    p = make()
    dm = _dm(p)
    ref = fwi.gn_hessian(p, D.PmlParams(v_ref=VREF), dm, p.m)
    rt, tol = TOL[dtype]
    h, rep = api.fwi_gn_hessian(m_slowness2=p.m, dm=dm, **_args(p, dtype, rtol=rt))
    assert len(rep) == 3 * len(p.freqs) * len(p.src) and all(r["converged"] for r in rep)
    assert rel(h.cpu().numpy(), ref.ravel()) <= tol


def test_gpu_dot_test():
    """<J dm, y>_R = <dm, J^H y> with the GPU's own J and J^H (solves to 1e-10)."""
    p = synth.tiny2d()
    dm, y = _dm(p), _y(p)
    a = _args(p, rtol=1e-10)
    Jdm, _ = api.fwi_jacobian(m_slowness2=p.m, dm=dm, **a)
    JHy, _ = api.fwi_jacobian_adjoint(m_slowness2=p.m, y=y, **a)
    lhs = np.real(np.vdot(y, Jdm))
    rhs = float(np.dot(dm.ravel(), JHy.cpu().numpy()))
    assert abs(lhs - rhs) <= 1e-7 * max(abs(lhs), abs(rhs))


def test_jacobian_adjoint_of_residual_is_gradient():
    """J^H (P_r u - d) = g of fwi_misfit_grad (Eq. 8 and JACOBI_ADJ describe one quantity)."""
    p = synth.tiny2d()
    pml = D.PmlParams(v_ref=VREF)
    d = fwi.forward_data(p, pml, p.m_true)
    a = _args(p, rtol=1e-10)
    u_rec, _ = api.fwi_forward(m_slowness2=p.m, **a)
    fg, _ = api.fwi_misfit_grad(m_slowness2=p.m, d_obs=d, **a)
    g, _ = api.fwi_jacobian_adjoint(m_slowness2=p.m, y=u_rec - d, **a)
    assert rel(g.cpu().numpy(), fg.cpu().numpy()[1:]) <= 1e-7


def test_gn_is_jh_of_j():
    p = synth.tiny3d()
    dm = _dm(p, 11)
    a = _args(p, rtol=1e-10)
    Jdm, _ = api.fwi_jacobian(m_slowness2=p.m, dm=dm, **a)
    JHJ, _ = api.fwi_jacobian_adjoint(m_slowness2=p.m, y=Jdm, **a)
    H, _ = api.fwi_gn_hessian(m_slowness2=p.m, dm=dm, **a)
    assert rel(H.cpu().numpy(), JHJ.cpu().numpy()) <= 1e-7


def test_joint_batch_and_shards_invariance():
    """One joint (source, frequency) batch of every pair, or 1-RHS batches, or source shards
    summed: same J^H y and GN dm (to solver tolerance)."""
    p = synth.tiny2d()
    y, dm = _y(p), _dm(p)
    npair = len(p.freqs) * len(p.src)
    g_all, _ = api.fwi_jacobian_adjoint(m_slowness2=p.m, y=y, **_args(p, rtol=1e-10, max_rhs=npair))
    g_one, _ = api.fwi_jacobian_adjoint(m_slowness2=p.m, y=y, **_args(p, rtol=1e-10, max_rhs=1))
    assert rel(g_all.cpu().numpy(), g_one.cpu().numpy()) <= 1e-8
    ns = len(p.src)
    parts = [api.fwi_gn_hessian(m_slowness2=p.m, dm=dm, src_range=r, **_args(p, rtol=1e-10))[0].cpu().numpy()
             for r in [(0, ns // 2), (ns // 2, ns)]]
    h, _ = api.fwi_gn_hessian(m_slowness2=p.m, dm=dm, **_args(p, rtol=1e-10))
    assert rel(parts[0] + parts[1], h.cpu().numpy()) <= 1e-8
    d_part, _ = api.fwi_jacobian(m_slowness2=p.m, dm=dm, src_range=(1, ns), **_args(p, rtol=1e-10))
    d_full, _ = api.fwi_jacobian(m_slowness2=p.m, dm=dm, **_args(p, rtol=1e-10))
    assert rel(d_part, d_full[:, 1:]) <= 1e-8


def test_empty_shard_and_zero_perturbation():
    p = synth.tiny2d()
    h, rep = api.fwi_gn_hessian(m_slowness2=p.m, dm=_dm(p), src_range=(2, 2), **_args(p))
    assert rep == [] and float(h.abs().max()) == 0.0
    d, _ = api.fwi_jacobian(m_slowness2=p.m, dm=np.zeros_like(p.m), **_args(p))
    assert np.all(d == 0)
