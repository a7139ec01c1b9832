"""R30: every reduction on the path is fixed-order fp64 (no float atomics), so whole evaluations
are bitwise reproducible run to run — misfit/gradient in a joint (source, frequency) batch
(2D and 3D, c128 and the c64 mixed mode), the off-grid path (transposed-gather adjoint
source) and the Gauss-Newton product."""
import numpy as np
import pytest

import synth
from oracle import discretize as D
from oracle import fwi
from paper_1703_09268_b200 import api

pytestmark = pytest.mark.gpu

VREF = 3000.0


def _a(p, dtype=api.C128):
    return dict(grid=api.Grid.of(p), freqs=p.freqs, pml=api.Pml(v_ref=VREF), dtype=dtype,
                opts=api.SolveOpts(rtol=1e-8 if dtype == api.C128 else 1e-6), max_rhs=len(p.src) * len(p.freqs))


@pytest.mark.parametrize("make", [synth.tiny2d, synth.tiny3d])
@pytest.mark.parametrize("dtype", [api.C128, api.C64])
def test_misfit_grad_bitwise_reproducible(make, dtype):
    p = make()
    d = fwi.forward_data(p, D.PmlParams(v_ref=VREF), p.m_true)
    runs = [api.fwi_misfit_grad(m_slowness2=p.m, src_node=p.src, rec_node=p.rec, d_obs=d, **_a(p, dtype))[0].cpu().numpy()
            for _ in range(2)]
    assert np.array_equal(runs[0], runs[1])


def test_offgrid_and_gn_bitwise_reproducible():
    p = synth.tiny2d()
    rng = np.random.default_rng(3)
    sx = np.stack([rng.uniform(2 * p.h, 30 * p.h, 3), np.zeros(3), rng.uniform(1.2 * p.h, 3 * p.h, 3)], 1)
    rx = np.stack([np.linspace(0.4 * p.h, 35 * p.h, 50), np.zeros(50), np.full(50, 0.7 * p.h)], 1)
    d = np.asarray(rng.standard_normal((1, 3, 50)) + 1j * rng.standard_normal((1, 3, 50)))
    acq = api.Acq(sx, rx)
    r = [api.fwi_misfit_grad_acq(m_slowness2=p.m, acq=acq, d_obs=d, **_a(p))[0].cpu().numpy() for _ in range(2)]
    assert np.array_equal(r[0], r[1])
    dm = rng.standard_normal(p.m.shape) * 1e-8
    h = [api.fwi_gn_hessian(m_slowness2=p.m, src_node=p.src, rec_node=p.rec, dm=dm, **_a(p))[0].cpu().numpy()
         for _ in range(2)]
    assert np.array_equal(h[0], h[1])
