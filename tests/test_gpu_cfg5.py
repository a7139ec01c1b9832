"""GPU matvec parity on BASELINE configs[4] (cfg5) at the sizes the bench reports, through the
C ABI (helm_apply), against the oracle's assembled operator (c.2 step 2):

* 128^3: the FULL oracle SpMV H @ x for b in {1, 4, 16} x {complex64, complex128}, forward,
  and the adjoint (H^H as the oracle's explicit conjugate transpose) at b = 4;
* 384^3 and 512^3 at b = 16 (the bench's largest launches: 512^3 x 16 RHS = 2^31 points, byte
  offsets beyond 2^34): sampled z-slabs (first, last, random interior planes) of the first,
  a middle and the LAST right-hand side vs the oracle's rows of H for those planes.

Tolerances (north star): rel-L2 <= 1e-12 (complex128), <= 1e-5 (complex64; the oracle
applies the exact operator to the same complex64-rounded input, D15). Inputs: unit-variance
complex normal x generated on the device from seed 1 (SURVEY d.1, cfg5 row)."""
import numpy as np
import pytest
import torch

import synth
from oracle import discretize as D
from paper_1703_09268_b200 import api

from .helpers import rel

pytestmark = pytest.mark.gpu

W = 2 * np.pi * 6.0
PML = D.PmlParams(v_ref=4500.0)
_P = {}


def _prob(N):
    if N not in _P:
        _P.clear()
        _P[N] = synth.cfg5(N)
    return _P[N]


def _apply(p, dtype, b, adjoint=0):
    op = api.helm_setup(api.Grid.of(p), p.m, W, api.Pml(v_ref=4500.0), dtype, max_rhs=b, mlopts=api.MlOpts(levels=0))
    x = torch.randn(b, p.n_ext, dtype=api.TORCH_DTYPE[dtype], device="cuda",
                    generator=torch.Generator(device="cuda").manual_seed(1))
    y = torch.empty_like(x)
    api.helm_apply(op, x, y, adjoint=adjoint)
    torch.cuda.synchronize()
    del op
    return x, y


@pytest.mark.parametrize("dtype", [api.C128, api.C64])
@pytest.mark.parametrize("b", [1, 4, 16])
def test_cfg5_128_full_spmv(dtype, b):
    p = _prob(128)
    x, y = _apply(p, dtype, b)
    H = D.helmholtz_matrix(p, W, PML)
    X = x.cpu().numpy().astype(np.complex128)
    Y = y.cpu().numpy().astype(np.complex128)
    tol = 1e-12 if dtype == api.C128 else 1e-5
    for r in range(b):
        assert rel(Y[r], H @ X[r]) <= tol, r


@pytest.mark.parametrize("dtype", [api.C128, api.C64])
def test_cfg5_128_full_adjoint(dtype):
    p = _prob(128)
    x, y = _apply(p, dtype, 4, adjoint=1)
    HH = D.helmholtz_matrix(p, W, PML).conj().T.tocsr()
    X = x.cpu().numpy().astype(np.complex128)
    Y = y.cpu().numpy().astype(np.complex128)
    tol = 1e-12 if dtype == api.C128 else 1e-5
    for r in range(4):
        assert rel(Y[r], HH @ X[r]) <= tol, r


@pytest.mark.parametrize("N", [384, 512])
@pytest.mark.parametrize("dtype", [api.C128, api.C64])
def test_cfg5_large_b16_sampled_slabs(N, dtype):
    b = 16
    p = _prob(N)
    x, y = _apply(p, dtype, b)
    Nx, Ny, Nz = p.next
    plane = Nx * Ny
    rng = np.random.default_rng(3)
    slabs = [0, Nz - 2] + sorted(rng.choice(np.arange(1, Nz - 3), 3, replace=False).tolist())
    tol = 1e-12 if dtype == api.C128 else 1e-5
    for z0 in slabs:
        z1 = z0 + 2
        lo, hi = max(z0 - 1, 0), min(z1 + 1, Nz)
        A = D.helmholtz_rows(p, W, PML, z0, z1)[:, lo * plane:hi * plane]
        for r in (0, b // 2, b - 1):
            xs = x[r, lo * plane:hi * plane].cpu().numpy().astype(np.complex128)
            ys = y[r, z0 * plane:z1 * plane].cpu().numpy().astype(np.complex128)
            assert rel(ys, A @ xs) <= tol, (z0, r)
    del x, y
    torch.cuda.empty_cache()
