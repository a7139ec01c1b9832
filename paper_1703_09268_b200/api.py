"""Thin Python binding of include/helm.h with the same entry-point names.

Argument marshalling only: every numeric step runs in libhelm.so's CUDA kernels. torch
supplies device memory and the current CUDA stream (plumbing, not the product).
Complex device arrays are torch tensors of dtype complex64 / complex128 on the extended
grid, shape (nrhs, Nz, Ny, Nx) (or anything contiguous with that many elements).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib as L

C64, C128 = L.HELM_C64, L.HELM_C128
TORCH_DTYPE = {C64: torch.complex64, C128: torch.complex128}


STENCILS = {"std2": L.HELM_STD2, "opt": L.HELM_OPT}


@dataclasses.dataclass(frozen=True)
class Grid:
    """D1: interior sizes (nx, ny, nz) (ny = 1 in 2D), spacing h, PML ((xl,xh),(yl,yh),(zl,zh)),
    stencil "std2" (5/7-pt, D4-D5) or "opt" (9/27-pt, DESIGN R34/R35)."""
    ndim: int
    n: Tuple[int, int, int]
    h: float
    pml: Tuple[Tuple[int, int], ...]
    stencil: str = "std2"

    @staticmethod
    def of(p) -> "Grid":
        return Grid(int(p.ndim), tuple(int(v) for v in p.n), float(p.h), tuple(tuple(int(w) for w in a) for a in p.pml),
                    getattr(p, "stencil", "std2"))

    @property
    def next(self):
        return tuple(self.n[a] + self.pml[a][0] + self.pml[a][1] for a in range(3))

    @property
    def n_ext(self):
        return int(np.prod(self.next))

    @property
    def n_interior(self):
        return int(np.prod(self.n))

    def c(self) -> L.HelmGrid:
        g = L.HelmGrid()
        g.ndim = self.ndim
        for a in range(3):
            g.n[a] = self.n[a]
            g.pml[a][0], g.pml[a][1] = self.pml[a]
        g.h = self.h
        g.stencil = STENCILS[self.stencil]
        return g


@dataclasses.dataclass(frozen=True)
class Pml:
    R: float = 1e-4
    power: int = 2
    v_ref: float = 0.0

    def c(self) -> L.HelmPml:
        return L.HelmPml(self.R, self.power, self.v_ref)


@dataclasses.dataclass(frozen=True)
class Acq:
    """Off-grid acquisition (helm.h helm_acq, DESIGN R33): physical (x, y, z) of the source and
    receiver points relative to interior node 0 (y = 0 in 2D); Kaiser window b and half-width
    (<= 0: 6.31 and 4)."""
    src_xyz: np.ndarray
    rec_xyz: np.ndarray
    kaiser_b: float = 0.0
    half_width: int = 0

    def c(self):
        s = np.ascontiguousarray(self.src_xyz, np.float64).reshape(-1, 3)
        r = np.ascontiguousarray(self.rec_xyz, np.float64).reshape(-1, 3)
        st = L.HelmAcq(_dptr(s), _dptr(r), float(self.kaiser_b), int(self.half_width))
        return st, (s, r), len(s), len(r)


@dataclasses.dataclass(frozen=True)
class SolveOpts:
    k_inner: int = 5
    max_outer: int = 50
    rtol: float = 1e-6
    precond: int = 1

    def c(self) -> L.HelmSolveOpts:
        return L.HelmSolveOpts(self.k_inner, self.max_outer, self.rtol, self.precond)


@dataclasses.dataclass(frozen=True)
class MlOpts:
    levels: int = 3
    ks_o: int = 3
    ks_i: int = 5
    kc_o: int = 3
    kc_i: int = 5

    def c(self) -> L.HelmMlOpts:
        return L.HelmMlOpts(self.levels, self.ks_o, self.ks_i, self.kc_o, self.kc_i)


def _stream(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _i64ptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def _tptr(t: torch.Tensor):
    assert t.is_cuda and t.is_contiguous()
    return C.c_void_p(t.data_ptr())


class HelmOp:
    """Owning handle of a helm_op (helm_setup / helm_destroy)."""

    def __init__(self, handle, grid: Grid, dtype: int, max_rhs: int):
        self._h = handle
        self.grid, self.dtype, self.max_rhs = grid, dtype, max_rhs
        self.tdtype = TORCH_DTYPE[dtype]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and L is not None and L._lib is not None:   # not during interpreter teardown
            L._lib.helm_destroy(h)
        self._h = None

    @property
    def handle(self):
        return self._h

    def levels(self) -> List[Tuple[int, int, int]]:
        lib = L.load()
        n = C.c_int32()
        dims = np.zeros((4, 3), np.int64)
        L.check(lib.helm_levels(self._h, C.byref(n), _i64ptr(dims)))
        return [tuple(int(v) for v in dims[l]) for l in range(n.value)]

    def get_level(self, level: int, adjoint: int = 0):
        """Returns (tables[3 axes][3 = lo,dg,up][Nmax] complex128, m_ext (Nz,Ny,Nx) float64)."""
        lib = L.load()
        nx, ny, nz = self.levels()[level]
        nmax = max(nx, ny, nz)
        tab = np.zeros((3, 3, nmax), np.complex128)
        m = np.zeros((nz, ny, nx), np.float64)
        L.check(lib.helm_get_level(self._h, level, adjoint, nmax, tab.ctypes.data_as(C.POINTER(C.c_double)), _dptr(m)))
        return tab, m

    def workspace_vectors(self) -> float:
        return L.load().helm_workspace_vectors(self._h)

    def empty(self, nrhs: int = 1, level: int = 0) -> torch.Tensor:
        nx, ny, nz = self.levels()[level]
        return torch.empty((nrhs, nz, ny, nx), dtype=self.tdtype, device="cuda")


def helm_setup(grid: Grid, m_slowness2: np.ndarray, omega: float, pml: Pml = Pml(), dtype: int = C128,
               max_rhs: int = 1, mlopts: Optional[MlOpts] = None, stream=None) -> HelmOp:
    lib = L.load()
    m = np.ascontiguousarray(m_slowness2, dtype=np.float64)
    assert m.size == grid.n_interior
    g, p = grid.c(), pml.c()
    ml = mlopts.c() if mlopts is not None else None
    h = C.c_void_p()
    L.check(lib.helm_setup(C.byref(g), _dptr(m), float(omega), C.byref(p), dtype, max_rhs,
                           C.byref(ml) if ml is not None else None, _stream(stream), C.byref(h)))
    return HelmOp(h, grid, dtype, max_rhs)


def helm_apply(op: HelmOp, x: torch.Tensor, y: torch.Tensor, adjoint: int = 0, stream=None) -> torch.Tensor:
    nrhs = x.numel() // op.grid.n_ext
    assert x.dtype == op.tdtype and y.dtype == op.tdtype and y.numel() == x.numel()
    L.check(L.load().helm_apply(op.handle, adjoint, nrhs, _tptr(x), _tptr(y), _stream(stream)))
    return y


def helm_solve(op: HelmOp, b: torch.Tensor, x: torch.Tensor, adjoint: int = 0, opts: SolveOpts = SolveOpts(),
               stream=None) -> List[dict]:
    nrhs = b.numel() // op.grid.n_ext
    assert b.dtype == op.tdtype and x.dtype == op.tdtype and x.numel() == b.numel()
    rep = (L.HelmSolveReport * nrhs)()
    so = opts.c()
    L.check(L.load().helm_solve(op.handle, adjoint, nrhs, _tptr(b), _tptr(x), C.byref(so), rep, _stream(stream)))
    return [r.as_dict() for r in rep]


def helm_vcycle(op: HelmOp, b: torch.Tensor, z: torch.Tensor, level: int = 0, adjoint: int = 0, stream=None):
    nx, ny, nz = op.levels()[level]
    nrhs = b.numel() // (nx * ny * nz)
    L.check(L.load().helm_vcycle(op.handle, level, adjoint, nrhs, _tptr(b), _tptr(z), _stream(stream)))
    return z


def helm_transfer(op: HelmOp, inp: torch.Tensor, out: torch.Tensor, level: int = 0, prolong: bool = False,
                  stream=None):
    nx, ny, nz = op.levels()[level + (1 if prolong else 0)]
    nrhs = inp.numel() // (nx * ny * nz)
    L.check(L.load().helm_transfer(op.handle, level, int(prolong), nrhs, _tptr(inp), _tptr(out), _stream(stream)))
    return out


def _freq_args(freqs, weights):
    f = np.ascontiguousarray(freqs, np.float64)
    w = None if weights is None else np.ascontiguousarray(np.asarray(weights, np.complex128).view(np.float64))
    return f, w


def fwi_misfit_grad(grid: Grid, m_slowness2: np.ndarray, freqs: Sequence[float], src_node: np.ndarray,
                    rec_node: np.ndarray, d_obs: np.ndarray, pml: Pml, dtype: int = C128,
                    opts: SolveOpts = SolveOpts(), max_rhs: int = 16, src_range: Optional[Tuple[int, int]] = None,
                    weights=None, fg: Optional[torch.Tensor] = None, stream=None):
    """Listing 1 `case OBJ`: returns (fg, reports); fg[0] = f, fg[1:] = g (interior, x fastest),
    fp64 on the device. d_obs: host complex128 (nfreq, nsrc_total, nrec)."""
    lib = L.load()
    m = np.ascontiguousarray(m_slowness2, np.float64)
    src = np.ascontiguousarray(src_node, np.int64)
    rec = np.ascontiguousarray(rec_node, np.int64)
    d = np.ascontiguousarray(d_obs, np.complex128)
    f, w = _freq_args(freqs, weights)
    s0, s1 = (0, len(src)) if src_range is None else src_range
    if fg is None:
        fg = torch.empty(1 + grid.n_interior, dtype=torch.float64, device="cuda")
    nrep = len(f) * (s1 - s0) * 2
    rep = (L.HelmSolveReport * max(nrep, 1))()
    g, p, so = grid.c(), pml.c(), opts.c()
    L.check(lib.fwi_misfit_grad(C.byref(g), _dptr(m), len(f), _dptr(f), None if w is None else _dptr(w), len(src), s0, s1,
                                _i64ptr(src), len(rec), _i64ptr(rec), d.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)),
                                C.byref(p), dtype, C.byref(so), max_rhs, _tptr(fg), rep, _stream(stream)))
    return fg, [rep[i].as_dict() for i in range(nrep)]


def fwi_forward(grid: Grid, m_slowness2: np.ndarray, freqs: Sequence[float], src_node: np.ndarray,
                rec_node: np.ndarray, pml: Pml, dtype: int = C128, opts: SolveOpts = SolveOpts(), max_rhs: int = 16,
                src_range: Optional[Tuple[int, int]] = None, weights=None, stream=None):
    """Listing 1 `case FORW_MODEL`: returns (d (nfreq, ns, nrec) complex128 host, reports)."""
    lib = L.load()
    m = np.ascontiguousarray(m_slowness2, np.float64)
    src = np.ascontiguousarray(src_node, np.int64)
    rec = np.ascontiguousarray(rec_node, np.int64)
    f, w = _freq_args(freqs, weights)
    s0, s1 = (0, len(src)) if src_range is None else src_range
    d = np.zeros((len(f), s1 - s0, len(rec)), np.complex128)
    nrep = len(f) * (s1 - s0) * 2
    rep = (L.HelmSolveReport * max(nrep, 1))()
    g, p, so = grid.c(), pml.c(), opts.c()
    L.check(lib.fwi_forward(C.byref(g), _dptr(m), len(f), _dptr(f), None if w is None else _dptr(w), s0, s1,
                            _i64ptr(src), len(rec), _i64ptr(rec), C.byref(p), dtype, C.byref(so), max_rhs,
                            d.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)), rep, _stream(stream)))
    return d, [rep[i].as_dict() for i in range(0, nrep, 2)]


def _dp(a: np.ndarray):
    return a.view(np.float64).ctypes.data_as(C.POINTER(C.c_double))


def fwi_jacobian(grid: Grid, m_slowness2: np.ndarray, freqs: Sequence[float], src_node: np.ndarray,
                 rec_node: np.ndarray, dm: np.ndarray, pml: Pml, dtype: int = C128, opts: SolveOpts = SolveOpts(),
                 max_rhs: int = 16, src_range: Optional[Tuple[int, int]] = None, weights=None, stream=None):
    """Listing 1 JACOBI_FORW: returns (J dm as (nfreq, ns, nrec) complex128 host, reports [.., 2])."""
    lib = L.load()
    m = np.ascontiguousarray(m_slowness2, np.float64)
    dmv = np.ascontiguousarray(dm, np.float64)
    src = np.ascontiguousarray(src_node, np.int64)
    rec = np.ascontiguousarray(rec_node, np.int64)
    f, w = _freq_args(freqs, weights)
    s0, s1 = (0, len(src)) if src_range is None else src_range
    d = np.zeros((len(f), s1 - s0, len(rec)), np.complex128)
    nrep = len(f) * (s1 - s0) * 2
    rep = (L.HelmSolveReport * max(nrep, 1))()
    g, p, so = grid.c(), pml.c(), opts.c()
    L.check(lib.fwi_jacobian(C.byref(g), _dptr(m), len(f), _dptr(f), None if w is None else _dptr(w), s0, s1,
                             _i64ptr(src), len(rec), _i64ptr(rec), _dptr(dmv), C.byref(p), dtype, C.byref(so),
                             max_rhs, _dp(d), rep, _stream(stream)))
    return d, [rep[i].as_dict() for i in range(nrep)]


def fwi_jacobian_adjoint(grid: Grid, m_slowness2: np.ndarray, freqs: Sequence[float], src_node: np.ndarray,
                         rec_node: np.ndarray, y: np.ndarray, pml: Pml, dtype: int = C128,
                         opts: SolveOpts = SolveOpts(), max_rhs: int = 16,
                         src_range: Optional[Tuple[int, int]] = None, weights=None,
                         out: Optional[torch.Tensor] = None, stream=None):
    """Listing 1 JACOBI_ADJ: returns (J^H y as fp64 device (n_interior,), reports [.., 2]).
    y: host complex128 (nfreq, nsrc_total, nrec)."""
    lib = L.load()
    m = np.ascontiguousarray(m_slowness2, np.float64)
    src = np.ascontiguousarray(src_node, np.int64)
    rec = np.ascontiguousarray(rec_node, np.int64)
    yv = np.ascontiguousarray(y, np.complex128)
    f, w = _freq_args(freqs, weights)
    s0, s1 = (0, len(src)) if src_range is None else src_range
    if out is None:
        out = torch.empty(grid.n_interior, dtype=torch.float64, device="cuda")
    nrep = len(f) * (s1 - s0) * 2
    rep = (L.HelmSolveReport * max(nrep, 1))()
    g, p, so = grid.c(), pml.c(), opts.c()
    L.check(lib.fwi_jacobian_adjoint(C.byref(g), _dptr(m), len(f), _dptr(f), None if w is None else _dptr(w),
                                     len(src), s0, s1, _i64ptr(src), len(rec), _i64ptr(rec), _dp(yv), C.byref(p),
                                     dtype, C.byref(so), max_rhs, _tptr(out), rep, _stream(stream)))
    return out, [rep[i].as_dict() for i in range(nrep)]


def fwi_gn_hessian(grid: Grid, m_slowness2: np.ndarray, freqs: Sequence[float], src_node: np.ndarray,
                   rec_node: np.ndarray, dm: np.ndarray, pml: Pml, dtype: int = C128, opts: SolveOpts = SolveOpts(),
                   max_rhs: int = 16, src_range: Optional[Tuple[int, int]] = None, weights=None,
                   out: Optional[torch.Tensor] = None, stream=None):
    """Listing 1 HESS_GN: returns (J^H J dm as fp64 device (n_interior,), reports [.., 3])."""
    lib = L.load()
    m = np.ascontiguousarray(m_slowness2, np.float64)
    dmv = np.ascontiguousarray(dm, np.float64)
    src = np.ascontiguousarray(src_node, np.int64)
    rec = np.ascontiguousarray(rec_node, np.int64)
    f, w = _freq_args(freqs, weights)
    s0, s1 = (0, len(src)) if src_range is None else src_range
    if out is None:
        out = torch.empty(grid.n_interior, dtype=torch.float64, device="cuda")
    nrep = len(f) * (s1 - s0) * 3
    rep = (L.HelmSolveReport * max(nrep, 1))()
    g, p, so = grid.c(), pml.c(), opts.c()
    L.check(lib.fwi_gn_hessian(C.byref(g), _dptr(m), len(f), _dptr(f), None if w is None else _dptr(w), s0, s1,
                               _i64ptr(src), len(rec), _i64ptr(rec), _dptr(dmv), C.byref(p), dtype, C.byref(so),
                               max_rhs, _tptr(out), rep, _stream(stream)))
    return out, [rep[i].as_dict() for i in range(nrep)]


def fwi_misfit_grad_subset(grid: Grid, m_slowness2: np.ndarray, freqs: Sequence[float], src_node: np.ndarray,
                           rec_node: np.ndarray, d_obs: np.ndarray, pair_mask: np.ndarray, pml: Pml, dtype: int = C128,
                           opts: SolveOpts = SolveOpts(), max_rhs: int = 16,
                           src_range: Optional[Tuple[int, int]] = None, weights=None,
                           fg: Optional[torch.Tensor] = None, stream=None):
    """Listing 1 `case OBJ` over the (frequency, source) pairs with pair_mask[f, s] (the paper's
    batch-mode subset): (fg, reports of the selected pairs in frequency-major order)."""
    lib = L.load()
    m = np.ascontiguousarray(m_slowness2, np.float64)
    src = np.ascontiguousarray(src_node, np.int64)
    rec = np.ascontiguousarray(rec_node, np.int64)
    d = np.ascontiguousarray(d_obs, np.complex128)
    f, w = _freq_args(freqs, weights)
    mask = np.ascontiguousarray(pair_mask, np.uint8).reshape(len(f), len(src))
    s0, s1 = (0, len(src)) if src_range is None else src_range
    if fg is None:
        fg = torch.empty(1 + grid.n_interior, dtype=torch.float64, device="cuda")
    nrep = int(mask[:, s0:s1].astype(bool).sum()) * 2
    rep = (L.HelmSolveReport * max(nrep, 1))()
    g, p, so = grid.c(), pml.c(), opts.c()
    L.check(lib.fwi_misfit_grad_subset(C.byref(g), _dptr(m), len(f), _dptr(f), None if w is None else _dptr(w), len(src),
                                       s0, s1, _i64ptr(src), len(rec), _i64ptr(rec), _dp(d),
                                       mask.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(p), dtype, C.byref(so),
                                       max_rhs, _tptr(fg), rep, _stream(stream)))
    return fg, [rep[i].as_dict() for i in range(nrep)]


def fwi_misfit_grad_acq(grid: Grid, m_slowness2: np.ndarray, freqs: Sequence[float], acq: Acq, d_obs: np.ndarray,
                        pml: Pml, dtype: int = C128, opts: SolveOpts = SolveOpts(), max_rhs: int = 16,
                        src_range: Optional[Tuple[int, int]] = None, weights=None,
                        fg: Optional[torch.Tensor] = None, stream=None):
    """Listing 1 `case OBJ` with off-grid (Kaiser-sinc) sources and receivers: (fg, reports)."""
    lib = L.load()
    m = np.ascontiguousarray(m_slowness2, np.float64)
    d = np.ascontiguousarray(d_obs, np.complex128)
    f, w = _freq_args(freqs, weights)
    ac, keep, ns_tot, nrec = acq.c()
    s0, s1 = (0, ns_tot) if src_range is None else src_range
    if fg is None:
        fg = torch.empty(1 + grid.n_interior, dtype=torch.float64, device="cuda")
    nrep = len(f) * (s1 - s0) * 2
    rep = (L.HelmSolveReport * max(nrep, 1))()
    g, p, so = grid.c(), pml.c(), opts.c()
    L.check(lib.fwi_misfit_grad_acq(C.byref(g), _dptr(m), len(f), _dptr(f), None if w is None else _dptr(w), ns_tot, s0,
                                    s1, nrec, C.byref(ac), _dp(d), C.byref(p), dtype, C.byref(so), max_rhs, _tptr(fg),
                                    rep, _stream(stream)))
    del keep
    return fg, [rep[i].as_dict() for i in range(nrep)]


def fwi_forward_acq(grid: Grid, m_slowness2: np.ndarray, freqs: Sequence[float], acq: Acq, pml: Pml,
                    dtype: int = C128, opts: SolveOpts = SolveOpts(), max_rhs: int = 16,
                    src_range: Optional[Tuple[int, int]] = None, weights=None, stream=None):
    """Listing 1 `case FORW_MODEL` with off-grid sources and receivers: (d (nfreq, ns, nrec), reports)."""
    lib = L.load()
    m = np.ascontiguousarray(m_slowness2, np.float64)
    f, w = _freq_args(freqs, weights)
    ac, keep, ns_tot, nrec = acq.c()
    s0, s1 = (0, ns_tot) if src_range is None else src_range
    d = np.zeros((len(f), s1 - s0, nrec), np.complex128)
    nrep = len(f) * (s1 - s0) * 2
    rep = (L.HelmSolveReport * max(nrep, 1))()
    g, p, so = grid.c(), pml.c(), opts.c()
    L.check(lib.fwi_forward_acq(C.byref(g), _dptr(m), len(f), _dptr(f), None if w is None else _dptr(w), ns_tot, s0, s1,
                                nrec, C.byref(ac), C.byref(p), dtype, C.byref(so), max_rhs, _dp(d), rep,
                                _stream(stream)))
    del keep
    return d, [rep[i].as_dict() for i in range(0, nrep, 2)]


# ---------------------------------------------------------------------------- measurement
def profile(enable: bool, stride: int = 1):
    """Sample every `stride`-th launch of each kernel class with CUDA events on its stream."""
    L.check(L.load().helm_profile(int(enable), int(stride)))


def profile_read(level: int = -1) -> dict:
    lib = L.load()
    n = L.NCLASS
    la = np.zeros(n, np.int64)
    sa = np.zeros(n, np.int64)
    ms = np.zeros(n)
    by = np.zeros(n)
    L.check(lib.helm_profile_read(level, _i64ptr(la), _i64ptr(sa), _dptr(ms), _dptr(by)))
    return {L.CLASS_NAMES[c]: {"launches": int(la[c]), "sampled": int(sa[c]), "ms": float(ms[c]),
                               "bytes": float(by[c])} for c in range(n)}


def probe_kernel(op: HelmOp, level: int, kind: int, nv: int, nrhs: int, reps: int = 50, stream=None) -> float:
    """Average device ms per launch of one hot-path kernel (see helm.h helm_probe_kernel)."""
    ms = C.c_double()
    L.check(L.load().helm_probe_kernel(op.handle, level, kind, nv, nrhs, reps, C.byref(ms), _stream(stream)))
    return ms.value


def launch_count() -> int:
    return int(L.load().helm_launch_count())
