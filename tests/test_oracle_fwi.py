"""Oracle misfit / gradient pins: Taylor test (§6.1), zero residual at the true
model, source-sum linearity, and the E^T reading R11."""
import numpy as np

import synth
from oracle import discretize as D
from oracle import fwi


def _setup():
    p = synth.tiny2d()
    pml = D.PmlParams(v_ref=3000.0)          # fixed: H depends on m only via Eq. (7)
    d = fwi.forward_data(p, pml, p.m_true)
    return p, pml, d


def _slopes(e, ts):
    return np.log2(e[:-1] / e[1:])


def test_taylor_first_and_second_order():
    p, pml, d = _setup()
    f0, g = fwi.misfit_grad(p, pml, d)
    dm = p.m_true - p.m                      # physically meaningful direction
    ts = 2.0 ** -np.arange(2, 10)
    e0, e1 = fwi.taylor_errors(lambda m: fwi.misfit_grad(p, pml, d, m)[0], p.m, dm, g, ts)
    s0, s1 = _slopes(e0, ts), _slopes(e1, ts)
    assert np.all(np.abs(s0 - 1) < 0.25), s0         # O(h)   (P:318 line 1)
    assert np.all(np.abs(s1 - 2) < 0.25), s1         # O(h^2) (P:318 line 2)


def test_taylor_3d():
    """The paper's Taylor test is 3D (§6.1): the oracle's f, g on tiny3d (LU fields)
    give e0 slope 1 and e1 slope 2."""
    p = synth.tiny3d()
    pml = D.PmlParams(v_ref=3000.0)
    d = fwi.forward_data(p, pml, p.m_true)
    _, g = fwi.misfit_grad(p, pml, d)
    dm = p.m_true - p.m
    ts = 2.0 ** -np.arange(2, 9)
    e0, e1 = fwi.taylor_errors(lambda m: fwi.misfit_grad(p, pml, d, m)[0], p.m, dm, g, ts)
    assert np.all(np.abs(_slopes(e0, ts) - 1) < 0.25), _slopes(e0, ts)
    assert np.all(np.abs(_slopes(e1, ts) - 2) < 0.25), _slopes(e1, ts)


def test_interior_only_gradient_fails_taylor():
    """R11: restricting Re(w^2 conj(u) v) to the interior (instead of E^T) loses second order."""
    p, pml, d = _setup()
    _, g = fwi.misfit_grad(p, pml, d)
    # rebuild g without the E^T fold: interior samples of g_ext only
    w = 2 * np.pi * p.freqs[0]
    f, g_full, fields = fwi.misfit_grad(p, pml, d, return_fields=True)
    U, V = fields[0]
    gext = np.sum(np.real(w**2 * np.conj(U) * V), axis=1).reshape(D.ext_shape(p))
    (xl, _), _, (zl, _) = p.pml
    g_int = gext[zl:zl + p.n[2], :, xl:xl + p.n[0]]
    assert np.linalg.norm(g_int - g_full) / np.linalg.norm(g_full) > 1e-3
    dm = synth.random_real(p.m.shape, 2) * np.abs(p.m).max() * 0.05   # touches boundary cells
    ts = 2.0 ** -np.arange(4, 12)
    _, e1 = fwi.taylor_errors(lambda m: fwi.misfit_grad(p, pml, d, m)[0], p.m, dm, g_int, ts)
    assert np.median(_slopes(e1, ts)) < 1.5


def test_zero_residual_at_true_model():
    p, pml, d = _setup()
    f, g = fwi.misfit_grad(p, pml, d, p.m_true)
    f0, _ = fwi.misfit_grad(p, pml, d)
    assert f <= 1e-20 * max(f0, 1.0) + 1e-24
    assert np.abs(g).max() < 1e-10 * np.abs(fwi.misfit_grad(p, pml, d)[1]).max()


def test_source_sum_linearity():
    p, pml, d = _setup()
    fa, ga = fwi.misfit_grad(p, pml, d[:, :1], src_ids=p.src[:1])
    fb, gb = fwi.misfit_grad(p, pml, d[:, 1:], src_ids=p.src[1:])
    f, g = fwi.misfit_grad(p, pml, d)
    assert abs(fa + fb - f) <= 1e-12 * f
    assert np.linalg.norm(ga + gb - g) <= 1e-12 * np.linalg.norm(g)


def test_gradient_matches_directional_difference():
    """Central difference of f along a smooth direction agrees with <g, dm> to O(t^2)."""
    p, pml, d = _setup()
    _, g = fwi.misfit_grad(p, pml, d)
    dm = np.ones_like(p.m) * 1e-9
    t = 1e-2
    fp = fwi.misfit_grad(p, pml, d, p.m + t * dm)[0]
    fm = fwi.misfit_grad(p, pml, d, p.m - t * dm)[0]
    fd = (fp - fm) / (2 * t)
    assert abs(fd - np.sum(g * dm)) <= 1e-6 * abs(fd)


# ---------------------------------------------------------------- SURVEY §8(f) rank 1 pins
def _lin_setup():
    p = synth.tiny2d()
    pml = D.PmlParams(v_ref=3000.0)
    rng = np.random.default_rng(2)
    dm = rng.standard_normal(p.m.shape) * 0.05 * p.m
    return p, pml, dm


def test_jacobian_matches_central_differences_of_forward_modelling():
    """J dm = dF/dm [dm]: central differences of the (pinned) forward modelling converge to
    it at second order (an independent check of the linearisation, Table 1 row J)."""
    p, pml, dm = _lin_setup()
    J = fwi.jacobian(p, pml, dm)
    errs = []
    for t in (1e-2, 5e-3, 2.5e-3):
        fd = (fwi.forward_data(p, pml, p.m + t * dm) - fwi.forward_data(p, pml, p.m - t * dm)) / (2 * t)
        errs.append(np.linalg.norm(fd - J) / np.linalg.norm(J))
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert errs[-1] < 1e-4 and np.all(np.abs(rates - 2) < 0.3), (errs, rates)


def test_jacobian_adjoint_dot_test():
    """Table 5: <J dm, y> = <dm, J^H y> (paper: 1.9973e-9 at solver tol 1e-10; LU here)."""
    p, pml, dm = _lin_setup()
    rng = np.random.default_rng(5)
    y = (rng.standard_normal((len(p.freqs), len(p.src), len(p.rec)))
         + 1j * rng.standard_normal((len(p.freqs), len(p.src), len(p.rec))))
    lhs = np.real(np.vdot(y, fwi.jacobian(p, pml, dm)))
    rhs = float(np.sum(dm * fwi.jacobian_adjoint(p, pml, y)))
    assert abs(lhs - rhs) <= 1e-12 * max(abs(lhs), abs(rhs))


def test_jacobian_adjoint_of_residual_is_the_gradient():
    """grad f = J^H (P u - d) (Table 1: grad f = T^* V, V = -H^-H P^T grad phi)."""
    p, pml, _ = _lin_setup()
    d = fwi.forward_data(p, pml, p.m_true)
    f, g = fwi.misfit_grad(p, pml, d)
    r = fwi.forward_data(p, pml, p.m) - d
    assert np.linalg.norm(fwi.jacobian_adjoint(p, pml, r) - g) <= 1e-12 * np.linalg.norm(g)


def test_gauss_newton_is_jh_j_symmetric_psd():
    """H_GN dm = J^H J dm (Table 1), three solves per pair (Table 2); symmetric, PSD."""
    p, pml, dm = _lin_setup()
    dm2 = np.random.default_rng(7).standard_normal(p.m.shape) * 0.05 * p.m
    Hd = fwi.gn_hessian(p, pml, dm)
    assert np.linalg.norm(Hd - fwi.jacobian_adjoint(p, pml, fwi.jacobian(p, pml, dm))) <= 1e-12 * np.linalg.norm(Hd)
    a = float(np.sum(dm2 * Hd))
    b = float(np.sum(dm * fwi.gn_hessian(p, pml, dm2)))
    assert abs(a - b) <= 1e-11 * max(abs(a), abs(b))
    Jd = fwi.jacobian(p, pml, dm)
    assert abs(float(np.sum(dm * Hd)) - np.linalg.norm(Jd) ** 2) <= 1e-11 * np.linalg.norm(Jd) ** 2
