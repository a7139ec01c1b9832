// stencil.cuh — pipelined plane-streaming stencil for sm_100a (a2, and a3's projections).
//
// A CTA owns a BX x BY tile of "rows" and a z-range, and streams the planes z0-1 .. z1 of
// its input through an S-stage shared-memory ring filled by asynchronous copies (cp.async /
// LDGSTS; zero-fill implements the Dirichlet ghosts, R7): the tile plus its one-point halo,
// the model m and, per mode, the own-point operands (b for the residual, V_0..V_{NV-1} for
// the fused Gram-Schmidt projections). S-3 planes stay in flight while plane z is computed
// (Little's law: ~40 KB in flight per SM at ~800 ns keeps HBM streaming).
//   YC = true  (3D): rows are y (coupled by the stencil), one RHS per CTA.
//   YC = false (2D): rows are right-hand sides (uncoupled); the grid plane is one x-row,
//                    so every sync still covers BX*BY points.
// Each thread owns PY rows of one column; per-thread load slots (global offset, shared
// offset, static predicate) are computed once and advanced by one plane per step. PML
// enters only through the 1D tables (D4-D6).
//
// MODE 0: y = s H x              (s = lazy normalisation of x, per RHS)
// MODE 1: y = b - H x, ||y||     (starts a Krylov cycle: beta, v0 scale, g, kact)
// MODE 2: w = s H x and h_i = <V_i, w>, i < NV (fused CGS projections, fp64 sums)
#pragma once
#include "kernels.cuh"

template <int B> __device__ __forceinline__ void cpa(unsigned s, const void* gmem, bool pred) {
  const int sz = pred ? B : 0;
  if constexpr (B == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(s), "l"(gmem), "n"(B), "r"(sz) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N> __device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <typename R> struct PlaneArgs {
  Geo<R> g;
  const cx<R>* x;          // input (rhs-major)
  cx<R>* y;                // output
  const cx<R>* b;          // MODE 1
  VPtrs<R> V;              // MODE 2
  const double* xscale;    // MODE 0/2: per-RHS lazy scale of x (stride sstride) or null
  int sstride;
  const int* active;       // per-RHS outer mask or null
  const int* kact;         // skip RHS r if jstep >= kact[r] (null = never)
  int jstep;
  int nrhs, ntx, nty, zlen;
  KCtx ctx;
  RedBuf rb;
};

template <typename R, int BX, int BY, int NP>
struct PlaneSmem {
  static constexpr int XE = (BY + 2) * (BX + 2);    // halo tile elements
  static constexpr int PE = BY * BX;                 // own-point elements
  static constexpr size_t stage_bytes =
      ((XE * sizeof(cx<R>) + PE * sizeof(R) + NP * PE * sizeof(cx<R>)) + 127) / 128 * 128;
};

// Deterministic warp-level reduction into per-RHS slots: lane 0 of each contributing warp
// writes its NV partials to slot `slot`, bumps the RHS ticket; the warp that brings the
// ticket to `nslots` sums all slots in fixed order and returns true (all lanes) with the
// totals in tot[] (valid in every lane).
template <int NV>
__device__ __forceinline__ bool warp_slot_reduce(double2 (&v)[NV], double2* part, unsigned* ticket, int slot,
                                                 int nslots, double2 (&tot)[NV]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v[k].x += __shfl_xor_sync(0xffffffffu, v[k].x, o);
      v[k].y += __shfl_xor_sync(0xffffffffu, v[k].y, o);
    }
  unsigned last = 0;
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) part[(size_t)slot * NV + k] = v[k];
    __threadfence();
    last = atomicAdd(ticket, 1u) == (unsigned)(nslots - 1);
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return false;
  __threadfence();
#pragma unroll
  for (int k = 0; k < NV; ++k) tot[k] = make_double2(0.0, 0.0);
  for (int sl = lane; sl < nslots; sl += 32) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const double2 t = __ldcg(part + (size_t)sl * NV + k);
      tot[k].x += t.x;
      tot[k].y += t.y;
    }
  }
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      tot[k].x += __shfl_xor_sync(0xffffffffu, tot[k].x, o);
      tot[k].y += __shfl_xor_sync(0xffffffffu, tot[k].y, o);
    }
  if (lane == 0) *ticket = 0u;
  return true;
}

template <typename R, int BX, int BY, int PY, int S, int MODE, int NV, bool YC>
__global__ void __launch_bounds__(BX * BY / PY)
k_plane(const PlaneArgs<R> a) {
  using C = cx<R>;
  constexpr int NP = MODE == 1 ? 1 : (MODE == 2 ? NV : 0);
  constexpr int NVR = MODE == 1 ? 1 : (MODE == 2 ? NV : 1);   // reduced values per RHS
  using SM = PlaneSmem<R, BX, BY, NP>;
  constexpr int NT = BX * BY / PY;
  constexpr int RS = BY / PY;          // row stride between a thread's rows
  constexpr int XP = BX + 2;           // shared row pitch (elements)
  static_assert(YC || PY == 1, "2D (rows = RHS) uses one row per thread");
  static_assert(BX == 32, "one warp per tile row");
  extern __shared__ __align__(128) unsigned char smem[];

  const Geo<R>& g = a.g;
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const int tx = threadIdx.x % BX, ty0 = threadIdx.x / BX;
  int tile = blockIdx.x, r0 = 0;
  if constexpr (YC) {
    r0 = blockIdx.x % a.nrhs;
    tile = blockIdx.x / a.nrhs;
    if (a.active && !a.active[r0]) return;
    if (a.kact && a.jstep >= a.kact[r0]) return;
  }
  const int txb = tile % a.ntx, tyb = tile / a.ntx;
  const int ix = txb * BX + tx;
  const int z0 = blockIdx.y * a.zlen, z1 = min(z0 + a.zlen, nz);
  const long long N = g.N;
  const long long plane = YC ? (long long)nx * ny : (long long)nx;
  const C zero = mkc((R)0, (R)0);

  // ---- rows owned by this thread: spatial y (YC) or right-hand side (2D)
  int rowv[PY];          // y index (YC) or rhs index (2D)
  bool rok[PY];          // row exists, is active, and this lane's column is inside the grid
  bool ract = true;      // 2D: this warp's RHS row exists and is active (warp-uniform)
  R sc[PY];              // lazy scale of x for this row's RHS
  long long gofs[PY];    // global offset of (ix, row) at z = 0
#pragma unroll
  for (int k = 0; k < PY; ++k) {
    const int row = tyb * BY + ty0 + k * RS;
    rowv[k] = row;
    if constexpr (YC) {
      rok[k] = row < ny && ix < nx;
      gofs[k] = (long long)r0 * N + (long long)row * nx + ix;
      sc[k] = (MODE != 1 && a.xscale) ? (R)a.xscale[(long long)r0 * a.sstride] : (R)1;
    } else {
      bool ok = row < a.nrhs;
      if (ok && a.active && !a.active[row]) ok = false;
      if (ok && a.kact && a.jstep >= a.kact[row]) ok = false;
      ract = ok;
      rok[k] = ok && ix < nx;
      gofs[k] = (long long)min(row, a.nrhs - 1) * N + ix;
      sc[k] = (ok && MODE != 1 && a.xscale) ? (R)a.xscale[(long long)row * a.sstride] : (R)1;
    }
  }
  if constexpr (!YC) {
    if (!__syncthreads_or(ract ? 1 : 0)) return;
  }

  // ---- load slots: own points, x-halo, y-halo (YC) — fixed per thread, bumped per plane
  constexpr int NL = 2 * PY + (YC ? 2 : 0);
  long long lg[NL];
  unsigned ls[NL];
  bool lp[NL];
  int nl = 0;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem);
#pragma unroll
  for (int k = 0; k < PY; ++k) {
    const int sr = ty0 + k * RS + 1;
    lg[nl] = gofs[k]; ls[nl] = (unsigned)((sr * XP + tx + 1) * sizeof(C)); lp[nl] = rok[k]; ++nl;
  }
#pragma unroll
  for (int k = 0; k < PY; ++k) {
    const int sr = ty0 + k * RS + 1;
    if (tx == 0) { lg[nl] = gofs[k] - 1; ls[nl] = (unsigned)(sr * XP * sizeof(C)); lp[nl] = rok[k] && ix > 0; ++nl; }
    if (tx == BX - 1) { lg[nl] = gofs[k] + 1; ls[nl] = (unsigned)((sr * XP + BX + 1) * sizeof(C)); lp[nl] = rok[k] && ix + 1 < nx; ++nl; }
  }
  if constexpr (YC) {
    if (ty0 == 0) {
      lg[nl] = gofs[0] - nx; ls[nl] = (unsigned)((tx + 1) * sizeof(C)); lp[nl] = ix < nx && rowv[0] - 1 >= 0 && rowv[0] - 1 < ny; ++nl;
    }
    if (ty0 + (PY - 1) * RS == BY - 1) {
      lg[nl] = gofs[PY - 1] + nx; ls[nl] = (unsigned)(((BY + 1) * XP + tx + 1) * sizeof(C));
      lp[nl] = ix < nx && rowv[PY - 1] + 1 < ny; ++nl;
    }
  }
  const long long mofs0 = YC ? (long long)rowv[0] * nx + ix : (long long)ix;
  const unsigned m_s0 = (unsigned)(SM::XE * sizeof(C));
  const unsigned p_s0 = (unsigned)(SM::XE * sizeof(C) + SM::PE * sizeof(R));

  const int nq = z1 - z0 + 2;
  auto load = [&](int q) {
    if (q < nq) {
      const int z = z0 - 1 + q;
      const bool zin = z >= 0 && z < nz;
      const unsigned st = sbase + (unsigned)((q % S) * SM::stage_bytes);
      const long long zo = (long long)z * plane;
#pragma unroll
      for (int i = 0; i < NL; ++i)
        if (i < nl) {
          const bool p = lp[i] && zin;
          cpa<sizeof(C)>(st + ls[i], p ? a.x + lg[i] + zo : a.x, p);
        }
      if (q >= 1 && z < z1) {
#pragma unroll
        for (int k = 0; k < PY; ++k)
          if (rok[k]) {
            const int pr = (ty0 + k * RS) * BX + tx;
            cpa<sizeof(R)>(st + m_s0 + pr * sizeof(R), g.m + (YC ? mofs0 + (long long)k * RS * nx : mofs0) + zo, true);
            if constexpr (MODE == 1) cpa<sizeof(C)>(st + p_s0 + pr * sizeof(C), a.b + gofs[k] + zo, true);
            if constexpr (MODE == 2) {
#pragma unroll
              for (int v = 0; v < NV; ++v)
                cpa<sizeof(C)>(st + p_s0 + (v * SM::PE + pr) * sizeof(C), a.V.p[v] + gofs[k] + zo, true);
            }
          }
      }
    }
    cpa_commit();   // always commit (possibly empty) so group counting stays uniform
  };

  // ---- per-thread operator coefficients (1D tables; ghosts masked, R7)
  const C lox = (ix > 0 && ix < nx) ? g.lo[0][ix] : zero;
  const C upx = (ix < nx - 1) ? g.up[0][ix] : zero;
  const C dgx = ix < nx ? g.dg[0][ix] : zero;
  C loy[PY], upy[PY], dgy[PY];
#pragma unroll
  for (int k = 0; k < PY; ++k) {
    if constexpr (YC) {
      const int iy = rowv[k];
      loy[k] = (iy > 0 && iy < ny) ? g.lo[1][iy] : zero;
      upy[k] = (iy < ny - 1) ? g.up[1][iy] : zero;
      dgy[k] = iy < ny ? g.dg[1][iy] : zero;
    } else {
      loy[k] = upy[k] = dgy[k] = zero;
    }
  }
  double nrm = 0.0;
  double2 acc[NVR];
#pragma unroll
  for (int k = 0; k < NVR; ++k) acc[k] = make_double2(0.0, 0.0);

#pragma unroll
  for (int q = 0; q < S - 1; ++q) load(q);
  for (int z = z0; z < z1; ++z) {
    const int q = z - z0 + 1;
    cpa_wait<S - 4>();        // this thread's groups <= q+1 complete (committed: <= q+S-3)
    __syncthreads();          // ... for every thread; stage (q-2)%S is free again
    load(q + S - 2);          // S-3 planes in flight while plane z is computed
    const C* X0 = reinterpret_cast<const C*>(smem + ((q - 1) % S) * SM::stage_bytes);
    const C* X1 = reinterpret_cast<const C*>(smem + (q % S) * SM::stage_bytes);
    const C* X2 = reinterpret_cast<const C*>(smem + ((q + 1) % S) * SM::stage_bytes);
    const R* Ms = reinterpret_cast<const R*>(smem + (q % S) * SM::stage_bytes + m_s0);
    const C* Ps = reinterpret_cast<const C*>(smem + (q % S) * SM::stage_bytes + p_s0);
    const C lz = z > 0 ? g.lo[2][z] : zero, uz = z < nz - 1 ? g.up[2][z] : zero, dz = g.dg[2][z];
    const long long zo = (long long)z * plane;
#pragma unroll
    for (int k = 0; k < PY; ++k) {
      if (!rok[k]) continue;
      const int c = (ty0 + k * RS + 1) * XP + tx + 1;
      const int pr = (ty0 + k * RS) * BX + tx;
      const C cur = X1[c];
      const R wm = g.w2 * Ms[pr];
      // tree-shaped sum: four independent complex products, then two adds
      C t0 = cmul(mkc(dgx.x + dgy[k].x + dz.x + wm, dgx.y + dgy[k].y + dz.y), cur);
      C t1 = cfma(upx, X1[c + 1], cmul(lox, X1[c - 1]));
      C t2 = cfma(uz, X2[c], cmul(lz, X0[c]));
      if constexpr (YC) t0 = cfma(upy[k], X1[c + XP], cfma(loy[k], X1[c - XP], t0));
      const C hx = cadd(cadd(t0, t1), t2);
      C* yp = a.y + gofs[k] + zo;
      if constexpr (MODE == 0) {
        *yp = cscale(hx, sc[k]);
      } else if constexpr (MODE == 1) {
        const C rv = csub(Ps[pr], hx);
        *yp = rv;
        nrm += (double)rv.x * rv.x + (double)rv.y * rv.y;
      } else {
        const C w = cscale(hx, sc[k]);
        *yp = w;
        const double2 wd = to_d(w);
#pragma unroll
        for (int v = 0; v < NV; ++v) acc[v] = cdot_acc(acc[v], to_d(Ps[v * SM::PE + pr]), wd);
      }
    }
  }
  cpa_wait<0>();
  if constexpr (MODE != 0) {
    if constexpr (MODE == 1) acc[0] = make_double2(nrm, 0.0);
    // 3D: every warp of the CTA belongs to RHS r0 -> slots (tile, zchunk, warp)
    // 2D: warp w owns RHS rowv[0]              -> slots (x-tile, zchunk)
    int r, slot, nslots;
    if constexpr (YC) {
      r = r0;
      constexpr int WPB = NT / 32;
      slot = ((tile + a.ntx * a.nty * blockIdx.y) * WPB) + (threadIdx.x >> 5);
      nslots = a.ntx * a.nty * gridDim.y * WPB;
    } else {
      r = rowv[0];
      if (!ract) return;          // warp-uniform: one RHS row per warp
      slot = txb + a.ntx * blockIdx.y;
      nslots = a.ntx * gridDim.y;
    }
    double2 tot[NVR];
    if (warp_slot_reduce<NVR>(acc, a.rb.part + r * a.rb.pstride, a.rb.ticket + r, slot, nslots, tot)) {
      if ((threadIdx.x & 31) == 0) {
        if constexpr (MODE == 1) {
          const double beta = sqrt(tot[0].x);
          KCtx ctx = a.ctx;
          ctx.beta[r] = beta;
          ctx.scale[r * (HELM_KMAX + 1)] = beta > 0.0 ? 1.0 / beta : 0.0;
          for (int i = 0; i <= HELM_KMAX; ++i) ctx.g[r * (HELM_KMAX + 1) + i] = make_double2(i == 0 ? beta : 0.0, 0.0);
          ctx.kact[r] = beta > 0.0 ? ctx.k : 0;
        } else {
          const double* scl = a.ctx.scale + r * (HELM_KMAX + 1);
          double2* H = a.ctx.H + (long long)r * (HELM_KMAX + 1) * HELM_KMAX;
          for (int i = 0; i < NV; ++i) H[hidx(i, a.jstep)] = make_double2(tot[i].x * scl[i], tot[i].y * scl[i]);
        }
      }
    }
  }
}
