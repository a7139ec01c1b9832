"""GPU parity of a1/a2 through the C ABI: tables and level models vs the oracle, helm_apply
forward / adjoint vs the assembled sparse H (c.4: <= 1e-12 c128, <= 1e-5 c64), GPU dot test."""
import numpy as np
import pytest
import torch

import synth
from oracle import discretize as D
from oracle import mlgmres
from paper_1703_09268_b200 import api
from paper_1703_09268_b200._lib import HelmError

from .helpers import rel, to_dev, to_host

pytestmark = pytest.mark.gpu


def medium3d():
    """Spans several 32x8 tiles and z-chunks with ragged tails in every axis."""
    rng = np.random.default_rng(0)
    p = synth.const_problem("m3", 3, (61, 37, 29), 15.0, 6, 2000.0, 11.0)
    v = 1500 + 1500 * rng.random(p.m.shape)
    return p.with_(m=1 / v**2, pml=((6, 5), (4, 7), (6, 3)))


def medium2d():
    rng = np.random.default_rng(1)
    p = synth.const_problem("m2", 2, (150, 83), 10.0, 12, 2000.0, 6.0)
    v = 1500 + 2000 * rng.random(p.m.shape)
    return p.with_(m=1 / v**2, pml=((12, 9), (0, 0), (5, 12)))


CASES = [synth.tiny2d, synth.tiny3d, medium3d, medium2d, synth.cfg1]


def _setup(p, dtype=api.C128, nrhs=3, f=None):
    f = p.freqs[0] if f is None else f
    w = 2 * np.pi * f
    pml = D.PmlParams(v_ref=float(np.max(1 / np.sqrt(p.m))) * 1.1)
    op = api.helm_setup(api.Grid.of(p), p.m, w, api.Pml(pml.R, pml.power, pml.v_ref), dtype, max_rhs=nrhs)
    return op, w, pml


@pytest.mark.parametrize("make", CASES)
def test_tables_and_models_match_oracle(make):
    p = make()
    op, w, pml = _setup(p)
    hier = mlgmres.Hierarchy(p, w, pml)
    levels = op.levels()
    assert [(s[2], s[1], s[0]) for s in levels] == [tuple(s) for s in hier.shapes]
    for l, (Nx, Ny, Nz) in enumerate(levels):
        for adj in (0, 1):
            tab, m = op.get_level(l, adj)
            for a, (N, n, (wl, wh)) in enumerate(zip((Nx, Ny, Nz), p.n, p.pml)):
                if a == 1 and p.ndim == 2:
                    assert np.all(tab[a, :, :N] == 0)
                    continue
                ref = D.tables_1d(N, n, p.h, wl, wh, w, pml, l)
                if adj:
                    ref = D.adjoint_tables_1d(*ref)
                for t in range(3):
                    scale = np.abs(ref[t]).max()
                    assert np.abs(tab[a, t, :N] - ref[t]).max() <= 1e-14 * scale, (l, adj, a, t)
            assert np.abs(m - hier.m_ext[l]).max() <= 1e-15 * np.abs(hier.m_ext[l]).max()


@pytest.mark.parametrize("make", CASES)
@pytest.mark.parametrize("adjoint", [0, 1])
def test_apply_c128_matches_sparse(make, adjoint):
    p = make()
    op, w, pml = _setup(p)
    H = D.helmholtz_matrix(p, w, pml)
    A = D.helmholtz_adjoint_matrix(H) if adjoint else H
    x = synth.random_complex((3, p.n_ext), 1)
    y = torch.empty(3, p.n_ext, dtype=torch.complex128, device="cuda")
    api.helm_apply(op, to_dev(x), y, adjoint)
    yg = to_host(y)
    for r in range(3):
        assert rel(yg[r], A @ x[r]) <= 1e-12


@pytest.mark.parametrize("make", CASES)
def test_apply_c64_matches_sparse(make):
    p = make()
    op, w, pml = _setup(p, api.C64)
    H = D.helmholtz_matrix(p, w, pml)
    x = synth.random_complex((3, p.n_ext), 1).astype(np.complex64)
    for adjoint in (0, 1):
        A = D.helmholtz_adjoint_matrix(H) if adjoint else H
        y = torch.empty(3, p.n_ext, dtype=torch.complex64, device="cuda")
        api.helm_apply(op, to_dev(x, torch.complex64), y, adjoint)
        yg = to_host(y)
        for r in range(3):
            assert rel(yg[r], A @ x[r].astype(np.complex128)) <= 1e-5


@pytest.mark.parametrize("make", [synth.tiny3d, medium2d])
def test_gpu_dot_test(make):
    """Table 5 on the GPU's own forward and adjoint kernels."""
    p = make()
    op, w, pml = _setup(p, nrhs=1)
    x = to_dev(synth.random_complex(p.n_ext, 1))
    yv = to_dev(synth.random_complex(p.n_ext, 3))
    Hx = torch.empty_like(x)
    HHy = torch.empty_like(yv)
    api.helm_apply(op, x, Hx, 0)
    api.helm_apply(op, yv, HHy, 1)
    a = torch.vdot(yv, Hx).item()
    b = torch.vdot(HHy, x).item()
    assert abs(a - b) / max(abs(a), abs(b)) < 1e-13


def test_errors_are_reported():
    p = synth.tiny2d()
    op, w, pml = _setup(p, nrhs=1)
    x = torch.zeros(2, p.n_ext, dtype=torch.complex128, device="cuda")
    y = torch.zeros_like(x)
    with pytest.raises(HelmError) as e:
        api.helm_apply(op, x, y, 0)          # nrhs = 2 > max_rhs = 1
    assert e.value.status == -2
    assert torch.all(y == 0)
