"""Seeded synthetic problems.

Conventions (SURVEY.md §8 "Sizes used throughout"):
  * interior sizes ``n = (nx, ny, nz)``; 2D problems are (x, z) with ny = 1;
  * arrays are C-order ``[z][y][x]`` (x fastest);
  * the model input is slowness squared m = 1/v^2 [s^2/m^2];
  * sources / receivers are interior nodes given by linear ids
    ``ix + nx*(iy + ny*iz)`` (R13: on-node, so Kaiser-sinc reduces to a delta);
  * ``pml = ((wx-, wx+), (wy-, wy+), (wz-, wz+))`` in grid points.

Seeds: model 0, random vectors 1, Taylor perturbation 2 (d.1).
Nothing in this module computes any part of the Helmholtz method.
"""
from __future__ import annotations

import dataclasses
from typing import Optional, Sequence, Tuple

import numpy as np


@dataclasses.dataclass
class Problem:
    name: str
    ndim: int
    n: Tuple[int, int, int]                 # interior (nx, ny, nz)
    h: float
    pml: Tuple[Tuple[int, int], ...]        # per axis (lo, hi)
    m: np.ndarray                           # slowness^2, shape (nz, ny, nx), float64
    freqs: Tuple[float, ...]                # Hz
    src: np.ndarray                         # int64 interior node ids
    rec: np.ndarray                         # int64 interior node ids
    m_true: Optional[np.ndarray] = None     # model that generated observed data
    stencil: str = "std2"                    # discretisation: "std2" (5/7-pt) or "opt" (9/27-pt, R34/R35)

    @property
    def next(self) -> Tuple[int, int, int]:
        """Extended (PML-included) sizes per axis (x, y, z)."""
        return tuple(self.n[a] + self.pml[a][0] + self.pml[a][1] for a in range(3))

    @property
    def n_interior(self) -> int:
        return int(np.prod(self.n))

    @property
    def n_ext(self) -> int:
        return int(np.prod(self.next))

    def with_(self, **kw) -> "Problem":
        return dataclasses.replace(self, **kw)


def node_id(ix, iy, iz, n) -> np.ndarray:
    """Linear interior node id; every axis index must lie inside the interior (no wrap-around)."""
    nx, ny, nz = n
    ix, iy, iz = (np.asarray(v, np.int64) for v in (ix, iy, iz))
    for v, m, a in ((ix, nx, "x"), (iy, ny, "y"), (iz, nz, "z")):
        if v.size and (v.min() < 0 or v.max() >= m):
            raise ValueError(f"node index out of the interior along {a}: [{v.min()}, {v.max()}] vs n = {m}")
    return ix + nx * (iy + ny * iz)


def random_complex(shape, seed: int = 1, dtype=np.complex128) -> np.ndarray:
    """i.i.d. complex normal with unit variance: Re, Im ~ N(0, 1/2)."""
    rng = np.random.default_rng(seed)
    z = (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) * np.sqrt(0.5)
    return z.astype(dtype)


def random_real(shape, seed: int = 2) -> np.ndarray:
    return np.random.default_rng(seed).standard_normal(shape)


def const_problem(name, ndim, n_int, h, pml_w, v, f, src_ijk=None, rec_ijk=None) -> Problem:
    """Constant-velocity problem; ``pml_w`` is the PML width on every side."""
    if ndim == 2:
        nx, nz = n_int
        n = (nx, 1, nz)
        pml = ((pml_w, pml_w), (0, 0), (pml_w, pml_w))
    else:
        n = tuple(n_int)
        pml = ((pml_w, pml_w),) * 3
    m = np.full((n[2], n[1], n[0]), 1.0 / v**2)
    if src_ijk is None:
        src_ijk = [(n[0] // 2, n[1] // 2, n[2] // 2)]
    src = np.array([node_id(i, j, k, n) for (i, j, k) in src_ijk], np.int64)
    rec = (np.zeros(0, np.int64) if rec_ijk is None else
           np.array([node_id(i, j, k, n) for (i, j, k) in rec_ijk], np.int64))
    return Problem(name, ndim, n, float(h), pml, m, (float(f),), src, rec)


# ----------------------------------------------------------------------------- config 1
def cfg1() -> Problem:
    """2D constant: 101x101, h=10 m, v=2000 m/s, f=5 Hz, PML 20, source at (50,50)."""
    return const_problem("cfg1", 2, (101, 101), 10.0, 20, 2000.0, 5.0, [(50, 0, 50)])


# ----------------------------------------------------------------------------- config 2
def cfg2_model(nx=401, nz=201, h=10.0, seed=0):
    """v0(z) = 1500 + 2500 z/200 (z index), plus K=8 seeded Gaussian blobs (+-10%)."""
    rng = np.random.default_rng(seed)
    K = 8
    cx = rng.uniform(0.0, 4000.0, K)
    cz = rng.uniform(200.0, 1800.0, K)
    s = rng.uniform(100.0, 300.0, K)
    a = rng.uniform(-0.1, 0.1, K)
    zi = np.arange(nz, dtype=np.float64)
    v0 = 1500.0 + 2500.0 * zi / (nz - 1)
    X = np.arange(nx) * h
    Z = zi * h
    ZZ, XX = np.meshgrid(Z, X, indexing="ij")
    p = np.zeros((nz, nx))
    for k in range(K):
        p += a[k] * np.exp(-((XX - cx[k]) ** 2 + (ZZ - cz[k]) ** 2) / (2.0 * s[k] ** 2))
    p = np.clip(p, -0.1, 0.1)
    v0_2d = np.repeat(v0[:, None], nx, axis=1)
    vt = v0_2d * (1.0 + p)
    return v0_2d, vt


def cfg2(nsrc: int = 50, freqs=(3.0, 5.0, 7.0)) -> Problem:
    nx, nz, h = 401, 201, 10.0
    v0, vt = cfg2_model(nx, nz, h)
    n = (nx, 1, nz)
    src = node_id(4 + 8 * np.arange(nsrc), 0, 2, n)
    rec = node_id(np.arange(nx), 0, 2, n)
    m0 = (1.0 / v0**2)[:, None, :]
    mt = (1.0 / vt**2)[:, None, :]
    return Problem("cfg2", 2, n, h, ((20, 20), (0, 0), (20, 20)), m0, tuple(freqs),
                   src, rec, m_true=mt)


# ----------------------------------------------------------------------------- config 3
def cfg3() -> Problem:
    """3D constant: 64^3, h=20 m, v=2000, f=8 Hz, PML 10, centred source (32,32,32)."""
    return const_problem("cfg3", 3, (64, 64, 64), 20.0, 10, 2000.0, 8.0, [(32, 32, 32)])


def cfg3_batch(b: int = 8) -> Problem:
    """cfg3 throughput variant: b sources at seeded interior nodes >= 1 wavelength
    (12.5 points) from the PML."""
    p = cfg3()
    rng = np.random.default_rng(0)
    ijk = rng.integers(13, 64 - 13, size=(b, 3))
    return p.with_(name=f"cfg3b{b}", src=node_id(ijk[:, 0], ijk[:, 1], ijk[:, 2], p.n))


# ----------------------------------------------------------------------------- config 4 / 5
def layered_model(n: int, seed: int = 0, noise: float = 0.05):
    """5 layers 1500..4500 m/s in z, plus smoothed noise scaled to max|n| = noise."""
    from scipy.ndimage import gaussian_filter
    vl = np.array([1500.0, 2250.0, 3000.0, 3750.0, 4500.0])
    z = np.arange(n)
    layer = np.minimum((5 * z) // n, 4)
    v0 = np.broadcast_to(vl[layer][:, None, None], (n, n, n)).copy()
    rng = np.random.default_rng(seed)
    nz = gaussian_filter(rng.standard_normal((n, n, n)), sigma=4, mode="nearest")
    nz *= noise / np.abs(nz).max()
    return v0, v0 * (1.0 + nz)


def cfg4(n: int = 200, h: float = 25.0, pml: int = 20, nsrc_side: int = 8,
         src_pitch: int = 25, src_off: int = 12, f: float = 6.0, name="cfg4") -> Problem:
    """Layered 3D FWI problem (BASELINE configs[3]). PML width (R9, revised in round 2): 20
    points = one wavelength at the model's mean layer velocity (3000 m/s at 6 Hz, h = 25 m);
    10 points (one wavelength at v_min) is only 1/3 wavelength in the fast bottom layers and
    measured 13 / 17 forward / adjoint outer cycles against 5 / 5 at 20."""
    v0, vt = layered_model(n)
    N = (n, n, n)
    k = src_off + src_pitch * np.arange(nsrc_side)
    sx, sy = np.meshgrid(k, k, indexing="ij")
    src = node_id(sx.ravel(), sy.ravel(), 2, N)
    rx, ry = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    rec = np.sort(node_id(rx.ravel(), ry.ravel(), 2, N))
    return Problem(name, 3, N, h, ((pml, pml),) * 3, 1.0 / v0**2, (f,), src, rec,
                   m_true=1.0 / vt**2)


def cfg4_replica(n: int = 24, pml: int = 6) -> Problem:
    """Parity replica of cfg4 from the same generator: 4 sources at {n/4, 3n/4}^2 (n = 24:
    {6, 18}^2), n^2 receivers."""
    return cfg4(n=n, pml=pml, nsrc_side=2, src_pitch=n // 2, src_off=n // 4, name=f"cfg4r{n}")


def cfg5(N: int) -> Problem:
    """Matvec sweep: cfg4 generator at interior (N-20)^3 with PML 10 inside N^3 (R8)."""
    p = cfg4(n=N - 20, pml=10, nsrc_side=1, name=f"cfg5_{N}")
    return p.with_(rec=np.zeros(0, np.int64))


# ----------------------------------------------------------------------------- Table 3 grids
def table3_grid(n_lambda: int, n_ppw: int) -> int:
    """Grid points per axis incl. a one-wavelength PML per side: n_l n_ppw + 2 n_ppw + 1."""
    return n_lambda * n_ppw + 2 * n_ppw + 1


TABLE3_CELLS = [(nl, npw) for nl in (5, 10, 25, 40, 50) for npw in (6, 8, 10)]


def table3(n_lambda: int, n_ppw: int, v: float = 2000.0, f: float = 10.0) -> Problem:
    """Table 3's study: 3D constant velocity with n_lambda wavelengths per axis
    sampled at n_ppw points per wavelength, plus a PML of one wavelength (n_ppw points) on each
    side, centred point source. Scale-free: h = (v / f) / n_ppw; the interior has
    n_lambda n_ppw + 1 points per axis, the extended grid table3_grid(n_lambda, n_ppw)."""
    n = n_lambda * n_ppw + 1
    h = v / f / n_ppw
    return const_problem(f"table3_{n_lambda}_{n_ppw}", 3, (n, n, n), h, n_ppw, v, f, [(n // 2, n // 2, n // 2)])


# ----------------------------------------------------------------------------- tiny cases
def tiny2d(nx=37, nz=29, pml=7, h=10.0, f=9.0, nsrc=3, seed=0) -> Problem:
    """Small heterogeneous 2D problem used by fast tests (ragged sizes on purpose)."""
    rng = np.random.default_rng(seed)
    zi = np.arange(nz)[:, None]
    v = 1600.0 + 900.0 * zi / (nz - 1) + 60.0 * rng.standard_normal((nz, nx))
    v = np.clip(v, 1400.0, 2800.0)
    n = (nx, 1, nz)
    xs = np.linspace(3, nx - 4, nsrc).astype(int)
    src = node_id(xs, 0, 2, n)
    rec = node_id(np.arange(nx), 0, 1, n)
    vt = v * (1.0 + 0.05 * np.exp(-(((np.arange(nx)[None] - nx / 2) ** 2) + (zi - nz / 2) ** 2) / 30.0))
    return Problem("tiny2d", 2, n, h, ((pml, pml), (0, 0), (pml, pml)),
                   (1.0 / v**2)[:, None, :], (f,), src, rec, m_true=(1.0 / vt**2)[:, None, :])


def tiny3d(n=(13, 11, 9), pml=4, h=20.0, f=8.0, nsrc=2, seed=0) -> Problem:
    rng = np.random.default_rng(seed)
    nx, ny, nz = n
    v = 1800.0 + 300.0 * np.arange(nz)[:, None, None] / (nz - 1) + 40.0 * rng.standard_normal((nz, ny, nx))
    src = node_id(np.linspace(2, nx - 3, nsrc).astype(int), ny // 2, 1, n)
    rx, ry = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    rec = np.sort(node_id(rx.ravel(), ry.ravel(), 1, n))
    vt = v * 1.03
    return Problem("tiny3d", 3, tuple(n), h, ((pml, pml),) * 3, 1.0 / v**2, (f,), src, rec,
                   m_true=1.0 / vt**2)
