"""Pins of the oracle's discrete operator against closed forms,
textbook special cases and brute force — never against the oracle itself."""
import numpy as np
import pytest
import scipy.sparse as sp

import synth
from oracle import discretize as D


def _prob(ndim, n, pml, h=10.0, seed=0):
    rng = np.random.default_rng(seed)
    if ndim == 2:
        p = synth.const_problem("t", 2, (n[0], n[2]), h, pml, 2000.0, 7.0)
    else:
        p = synth.const_problem("t", 3, n, h, pml, 2000.0, 7.0)
    v = 1500.0 + 1000.0 * rng.random(p.m.shape)
    return p.with_(m=1.0 / v**2)


def test_interior_tables_are_textbook_second_difference():
    """eta = 1 in the interior: lo = up = 1/h^2, dg = -2/h^2 (D4 reduces to the 3-point Laplacian)."""
    N, n, w, h = 40, 24, 8, 12.5
    lo, dg, up = D.tables_1d(N, n, h, w, w, 2 * np.pi * 5, D.PmlParams(v_ref=2500.0))
    inner = slice(w + 1, w + n - 1)   # nodes whose half-neighbours are also interior
    assert np.allclose(lo[inner], 1 / h**2, rtol=0, atol=1e-18)
    assert np.allclose(up[inner], 1 / h**2, rtol=0, atol=1e-18)
    assert np.allclose(dg[inner], -2 / h**2, rtol=0, atol=1e-18)
    # PML nodes are damped: |eta| > 1 => |coef| < 1/h^2, and Im != 0
    assert np.all(np.abs(lo[:w]) < 1 / h**2) and np.all(np.abs(np.imag(lo[:w])) > 0)


def test_dirichlet_laplacian_spectrum():
    """No PML: T is the Dirichlet second difference, eigenvalues -(4/h^2) sin^2(k pi / (2(N+1)))."""
    N, h = 17, 3.0
    lo, dg, up = D.tables_1d(N, N, h, 0, 0, 1.0, D.PmlParams(v_ref=1.0))
    T = D.second_difference(lo, dg, up).toarray()
    ev = np.sort(np.linalg.eigvals(T).real)
    k = np.arange(1, N + 1)
    ref = np.sort(-(4 / h**2) * np.sin(k * np.pi / (2 * (N + 1))) ** 2)
    assert np.allclose(ev, ref, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("ndim", [2, 3])
def test_laplacian_annihilates_affine_fields(ndim):
    """omega^2 m = 0 and no PML: L (a + b.x) = 0 at nodes not adjacent to the ghosts."""
    p = _prob(ndim, (9, 8, 7), 0)
    p = p.with_(m=np.zeros_like(p.m))
    H = D.helmholtz_matrix(p, 1.0, D.PmlParams(v_ref=1.0))
    Nz, Ny, Nx = D.ext_shape(p)
    Z, Y, X = np.meshgrid(np.arange(Nz), np.arange(Ny), np.arange(Nx), indexing="ij")
    f = 0.7 + 1.3 * X - 0.4 * Z + (2.1 * Y if ndim == 3 else 0)
    y = (H @ f.ravel().astype(complex)).reshape(f.shape)
    sl = (slice(1, -1), slice(1, -1) if ndim == 3 else slice(None), slice(1, -1))
    assert np.max(np.abs(y[sl])) < 1e-12


def test_plane_wave_symbol_3d():
    """Interior plane wave e^{i k.x}: H u = (-(4/h^2) sum_a sin^2(k_a h/2) + omega^2 m) u."""
    p = synth.const_problem("t", 3, (12, 11, 10), 5.0, 3, 1800.0, 9.0)
    w = 2 * np.pi * 9.0
    H = D.helmholtz_matrix(p, w, D.default_pml(p.m))
    Nz, Ny, Nx = D.ext_shape(p)
    k = np.array([0.11, -0.07, 0.05])
    Z, Y, X = np.meshgrid(np.arange(Nz), np.arange(Ny), np.arange(Nx), indexing="ij")
    u = np.exp(1j * p.h * (k[0] * X + k[1] * Y + k[2] * Z))
    y = (H @ u.ravel()).reshape(u.shape)
    lam = -(4 / p.h**2) * np.sum(np.sin(k * p.h / 2) ** 2) + w**2 / 1800.0**2
    sl = (slice(4, -4),) * 3     # nodes whose whole stencil is interior (eta = 1)
    assert np.max(np.abs(y[sl] - lam * u[sl])) / abs(lam) < 1e-12


@pytest.mark.parametrize("ndim", [2, 3])
def test_affine_in_m(ndim):
    """Eq. (7) / S:177: H(m + dm) x - H(m) x = omega^2 (E dm) .* x exactly."""
    p = _prob(ndim, (11, 9, 8), 4)
    w = 2 * np.pi * 6.0
    pml = D.PmlParams(v_ref=2600.0)
    dm = synth.random_real(p.m.shape, 2) * 1e-8
    x = synth.random_complex(p.n_ext, 1)
    lhs = D.helmholtz_matrix(p, w, pml, p.m + dm) @ x - D.helmholtz_matrix(p, w, pml) @ x
    E = D.extension_matrix(p)
    rhs = w**2 * (E @ dm.ravel()) * x
    assert np.linalg.norm(lhs - rhs) / np.linalg.norm(rhs) < 1e-8   # cancellation of O(1e8) terms
    # and brute force: E replicates along the normal (clamp indices)
    Nz, Ny, Nx = D.ext_shape(p)
    me = D.extend(p, dm)
    for (k, j, i) in [(0, 0, 0), (Nz - 1, Ny - 1, Nx - 1), (3, 0 if ndim == 2 else 5, Nx - 2), (Nz // 2, Ny // 2, 1)]:
        kk = min(max(k - p.pml[2][0], 0), p.n[2] - 1)
        jj = min(max(j - p.pml[1][0], 0), p.n[1] - 1)
        ii = min(max(i - p.pml[0][0], 0), p.n[0] - 1)
        assert me[k, j, i] == dm[kk, jj, ii]


@pytest.mark.parametrize("ndim,nnz", [(2, 5), (3, 7)])
def test_impulse_support(ndim, nnz):
    """H e_k has 5 (2D) / 7 (3D) nonzeros, symmetric pattern around an interior k."""
    p = _prob(ndim, (9, 9, 9), 3)
    H = D.helmholtz_matrix(p, 2 * np.pi * 5, D.PmlParams(v_ref=2600.0))
    Nz, Ny, Nx = D.ext_shape(p)
    k = (Nz // 2) * Nx * Ny + (Ny // 2) * Nx + Nx // 2
    col = H[:, k].toarray().ravel()
    nzi = np.flatnonzero(col)
    assert len(nzi) == nnz
    assert sorted(nzi - k) == sorted({0, 1, -1, Nx, -Nx} | ({Nx * Ny, -Nx * Ny} if ndim == 3 else set()))


def test_adjoint_closed_form_matches_conjugate_transpose():
    """D6: the conjugate-transposed 1D tables reproduce H^H; H is NOT complex-symmetric in the PML."""
    p = _prob(3, (7, 6, 5), 4)
    w = 2 * np.pi * 8.0
    pml = D.PmlParams(v_ref=2600.0)
    H = D.helmholtz_matrix(p, w, pml)
    HH = D.helmholtz_adjoint_matrix(H)
    # rebuild H^H from D6 tables
    nx, ny, nz = p.n
    Nx, Ny, Nz = p.next
    mats = []
    for N, n, (wl, wh) in ((Nx, nx, p.pml[0]), (Ny, ny, p.pml[1]), (Nz, nz, p.pml[2])):
        mats.append(D.second_difference(*D.adjoint_tables_1d(*D.tables_1d(N, n, p.h, wl, wh, w, pml))))
    Ix, Iy, Iz = (sp.identity(k) for k in (Nx, Ny, Nz))
    HH6 = sp.kron(Iz, sp.kron(Iy, mats[0])) + sp.kron(Iz, sp.kron(mats[1], Ix)) + \
        sp.kron(mats[2], sp.kron(Iy, Ix)) + sp.diags(w**2 * D.extend(p, p.m).ravel())
    assert abs(HH - HH6).max() < 1e-12 * abs(H).max()
    assert abs(H - H.T).max() > 1e-6 * abs(H).max()


@pytest.mark.parametrize("ndim", [2, 3])
def test_dot_test(ndim):
    """Table 5: |<Hx,y> - <x,H^H y>| / max ~ 1e-15 (paper 2.9004e-15)."""
    p = _prob(ndim, (13, 10, 9), 5)
    H = D.helmholtz_matrix(p, 2 * np.pi * 7, D.PmlParams(v_ref=2600.0))
    x = synth.random_complex(p.n_ext, 1)
    y = synth.random_complex(p.n_ext, 3)
    a = np.vdot(y, H @ x)
    b = np.vdot(D.helmholtz_adjoint_matrix(H) @ y, x)
    assert abs(a - b) / max(abs(a), abs(b)) < 1e-13


def test_extension_identities():
    p = _prob(3, (6, 5, 4), 3)
    E = D.extension_matrix(p)
    # constant -> constant; restriction to the interior is the identity; pml=0 -> identity
    assert np.allclose(E @ np.ones(p.n_interior), 1.0)
    me = D.extend(p, p.m)
    (xl, _), (yl, _), (zl, _) = p.pml
    assert np.array_equal(me[zl:zl + 4, yl:yl + 5, xl:xl + 6], p.m)
    p0 = p.with_(pml=((0, 0),) * 3)
    assert (D.extension_matrix(p0) - sp.identity(p.n_interior)).nnz == 0
    # E^T sums each PML line into its boundary cell: column sums count replicas
    cs = np.asarray(E.sum(axis=0)).ravel().reshape(p.m.shape)
    assert cs[2, 2, 2] == 1 and cs[0, 0, 0] == (1 + 3) ** 3


@pytest.mark.parametrize("ndim", [2, 3])
def test_slab_rows_equal_full_assembly(ndim):
    """helmholtz_rows (used to check large grids slab by slab) = the pinned full D5 matrix
    restricted to those z-planes, exactly."""
    p = _prob(ndim, (11, 9, 10), 4)
    w, pml = 2 * np.pi * 6, D.PmlParams(v_ref=2500.0)
    H = D.helmholtz_matrix(p, w, pml)
    Nx, Ny, Nz = p.next
    for z0, z1 in ((0, 2), (5, 9), (Nz - 3, Nz)):
        Hs = D.helmholtz_rows(p, w, pml, z0, z1)
        ref = H[z0 * Ny * Nx:z1 * Ny * Nx]
        assert (Hs - ref).count_nonzero() == 0 or abs(Hs - ref).max() == 0.0
