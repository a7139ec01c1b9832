// persist.cuh — one grid-synchronous (cooperative) launch per coarse V-cycle (sm_100a).
//
// Alg. 1 at the second-to-last level l with the coarsest level l+1 (Fig. 3
// recursion bottom, R20): pre-smooth GMRES(ks_o, ks_i) from 0, r = b - H_l x, restrict
// (R = 2^-d P^T, R21), coarsest GMRES(kc_o, kc_i) from 0, prolong + correct, post-smooth
// GMRES(ks_o, ks_i) from x (fixed counts, D14). On small coarse levels every one of the ~66
// kernels of this V-cycle is latency-bound (the fixed ~9-10 us per dependent kernel of
// DESIGN §6): here the dependent steps meet at grid barriers instead of kernel boundaries.
//
// Decomposition: cpr CTAs per active RHS, each owning a contiguous chunk of the level's
// points (recomputed per level). Neighbours come from global memory (these levels are L2
// resident). GMRES is classical Gram-Schmidt with two reductions per step (projections, then
// the norm of the updated vector: no Pythagoras), lazy normalisation, breakdown guard
// h_{j+1,j} <= 1e-14 beta (D14). Reductions are deterministic: every CTA writes fp64 block
// partials, and after the grid barrier every CTA of the RHS sums the cpr partials of its RHS
// in the same fixed order, so all CTAs hold identical Krylov scalars (kept in shared memory,
// no further broadcast). Every CTA executes the same number of grid barriers whatever its
// RHS's breakdown state.
#pragma once
#include <cooperative_groups.h>
#include "kernels.cuh"

template <typename R> struct PersistArgs {
  Geo<R> gf, gc;                 // operators of level l (fine) and l+1 (coarsest)
  const cx<R>* b;                // V-cycle input at level l
  cx<R>* x;                      // V-cycle output at level l
  cx<R>* SV[HELM_KMAX + 1];      // level-l basis (SV[0]: residual)
  cx<R>* SW;                     // level-l raw products
  cx<R>* FV[HELM_KMAX + 1];      // level-(l+1) basis
  cx<R>* FW;
  cx<R>* Fx;
  cx<R>* Fb;
  const int* active;             // compact active-RHS list (nact entries)
  int nact, cpr;                 // active RHS, CTAs per RHS (grid = nact * cpr)
  int ks_o, ks_i, kc_o, kc_i;
  int has_y;
  R fac;                         // 2^-d
  double2* part;                 // [grid][HELM_KMAX + 1] block partials
};

namespace persist {

// Vectors written inside this kernel are read through L2 only (ld.global.cg): a line another
// CTA wrote before the last grid barrier must not be served from this SM's L1.
template <typename T> __device__ __forceinline__ T ldv(const T* p) { return __ldcg(p); }

template <typename R>
__device__ __forceinline__ cx<R> apply_h(const Geo<R>& g, const OpTab<R>& T, const cx<R>* __restrict__ u,
                                         const R* __restrict__ m, long long p) {
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const long long pl = (long long)nx * ny;
  const int ix = (int)(p % nx), iy = (int)((p / nx) % ny), iz = (int)(p / pl);
  const cx<R> c = ldv(u + p);
  const cx<R> d = cadd(cadd(__ldg(T.dg[0] + ix), __ldg(T.dg[1] + iy)), __ldg(T.dg[2] + iz));
  cx<R> acc = cmul(mkc(d.x + T.w2 * __ldg(m + p), d.y), c);
  if (ix > 0) acc = cfma(__ldg(T.lo[0] + ix), ldv(u + p - 1), acc);
  if (ix < nx - 1) acc = cfma(__ldg(T.up[0] + ix), ldv(u + p + 1), acc);
  if (ny > 1) {
    if (iy > 0) acc = cfma(__ldg(T.lo[1] + iy), ldv(u + p - nx), acc);
    if (iy < ny - 1) acc = cfma(__ldg(T.up[1] + iy), ldv(u + p + nx), acc);
  }
  if (iz > 0) acc = cfma(__ldg(T.lo[2] + iz), ldv(u + p - pl), acc);
  if (iz < nz - 1) acc = cfma(__ldg(T.up[2] + iz), ldv(u + p + pl), acc);
  return acc;
}

// Krylov scalars of one RHS, replicated in every CTA of the RHS.
struct State {
  double scale[HELM_KMAX + 1];
  double2 H[(HELM_KMAX + 1) * HELM_KMAX];
  double cs[HELM_KMAX];
  double2 sn[HELM_KMAX];
  double2 g[HELM_KMAX + 1];
  double2 y[HELM_KMAX];
  double beta;
  int kact;
};

template <int NT> struct Block {
  double2 red[NT / 32][HELM_KMAX + 1];
  double2 tot[HELM_KMAX + 1];
};

// Sum nv fp64 complex values over the CTA (fixed order), write the CTA's partials, grid
// barrier, then sum this RHS's cpr partials in fixed order: tot[0..nv) in shared memory.
template <int NT>
__device__ void grid_reduce(cooperative_groups::grid_group& grid, Block<NT>& B, double2* v, int nv, double2* part,
                            int slot0, int cpr) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int k = 0; k < nv; ++k) {
    double2 s = v[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
      s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
    }
    if (lane == 0) B.red[w][k] = s;
  }
  __syncthreads();
  if (threadIdx.x < nv) {
    double2 s = make_double2(0.0, 0.0);
    for (int i = 0; i < NT / 32; ++i) s = make_double2(s.x + B.red[i][threadIdx.x].x, s.y + B.red[i][threadIdx.x].y);
    __stcg(part + (size_t)blockIdx.x * (HELM_KMAX + 1) + threadIdx.x, s);
  }
  grid.sync();
  if (threadIdx.x < nv) {
    double2 s = make_double2(0.0, 0.0);
    for (int c = 0; c < cpr; ++c) {
      const double2 t = __ldcg(part + (size_t)(slot0 + c) * (HELM_KMAX + 1) + threadIdx.x);
      s = make_double2(s.x + t.x, s.y + t.y);
    }
    B.tot[threadIdx.x] = s;
  }
  __syncthreads();
}

// Column j complete with h_{j+1,j} = hn (one thread): Givens rotations, residual estimate,
// lazy scale of v_{j+1}, breakdown guard (D14); the LS solve when the cycle's last column
// closes. Same algebra as kernels.cuh finalize_column / solve_ls.
__device__ inline void close_column(State& S, int j, double hn) {
  double2* H = S.H;
  for (int i = 0; i < j; ++i) {
    const double2 a = H[hidx(i, j)], bb = H[hidx(i + 1, j)];
    const double c = S.cs[i];
    const double2 sv = S.sn[i];
    H[hidx(i, j)] = cadd(make_double2(c * a.x, c * a.y), cmul(sv, bb));
    H[hidx(i + 1, j)] = csub(make_double2(c * bb.x, c * bb.y), cmul(cconj(sv), a));
  }
  const double2 a = H[hidx(j, j)];
  const double aa = sqrt(cabs2(a)), rr = sqrt(aa * aa + hn * hn);
  double c;
  double2 sv;
  if (rr == 0.0) { c = 1.0; sv = make_double2(0.0, 0.0); }
  else if (aa == 0.0) { c = 0.0; sv = make_double2(1.0, 0.0); }
  else { c = aa / rr; sv = make_double2(a.x / aa * hn / rr, a.y / aa * hn / rr); }
  S.cs[j] = c;
  S.sn[j] = sv;
  H[hidx(j, j)] = cadd(make_double2(c * a.x, c * a.y), make_double2(sv.x * hn, sv.y * hn));
  H[hidx(j + 1, j)] = make_double2(0.0, 0.0);
  const double2 gj = S.g[j];
  S.g[j + 1] = cmul(make_double2(-sv.x, sv.y), gj);
  S.g[j] = make_double2(c * gj.x, c * gj.y);
  if (hn <= 1e-14 * S.beta) {
    S.kact = j + 1;
    S.scale[j + 1] = 0.0;
  } else {
    S.scale[j + 1] = 1.0 / hn;
  }
}

__device__ inline void solve_ls(State& S) {
  const int k = S.kact;
  for (int i = HELM_KMAX - 1; i >= 0; --i) {
    if (i >= k) { S.y[i] = make_double2(0.0, 0.0); continue; }
    double2 t = S.g[i];
    for (int l = i + 1; l < k; ++l) t = csub(t, cmul(S.H[hidx(i, l)], S.y[l]));
    const double2 d = S.H[hidx(i, i)];
    S.y[i] = (d.x == 0.0 && d.y == 0.0) ? make_double2(0.0, 0.0) : cdiv(t, d);
  }
}

// Restarted GMRES(ko, ki) on one level for this CTA's RHS r: x <- (x0zero ? 0 : x) + the
// Krylov corrections; V[0..ki] basis, W raw products (all offset to RHS r).
template <typename R, int NT>
__device__ void gmres(cooperative_groups::grid_group& grid, Block<NT>& B, State& S, const Geo<R>& g,
                      const OpTab<R>& T, const cx<R>* b, cx<R>* x, bool x0zero, int ko, int ki, cx<R>* const* V,
                      cx<R>* W, long long p0, long long p1, double2* part, int slot0, int cpr) {
  using C = cx<R>;
  for (int cyc = 0; cyc < ko; ++cyc) {
    const bool zero = x0zero && cyc == 0;
    const C* v0 = zero ? b : V[0];
    double2 nr = make_double2(0.0, 0.0);
    for (long long p = p0 + threadIdx.x; p < p1; p += NT) {
      const C rv = zero ? ldv(b + p) : csub(ldv(b + p), apply_h(g, T, x, g.m, p));
      if (!zero) V[0][p] = rv;
      nr.x += (double)rv.x * rv.x + (double)rv.y * rv.y;
    }
    grid_reduce<NT>(grid, B, &nr, 1, part, slot0, cpr);
    if (threadIdx.x == 0) {
      const double beta = sqrt(B.tot[0].x);
      S.beta = beta;
      S.scale[0] = beta > 0.0 ? 1.0 / beta : 0.0;
      S.kact = beta > 0.0 ? ki : 0;
      for (int i = 0; i <= HELM_KMAX; ++i) S.g[i] = make_double2(i == 0 ? beta : 0.0, 0.0);
      for (int i = 0; i < (HELM_KMAX + 1) * HELM_KMAX; ++i) S.H[i] = make_double2(0.0, 0.0);
    }
    __syncthreads();
    for (int j = 0; j < ki; ++j) {
      const bool act = j < S.kact;                 // uniform over the RHS's CTAs
      const C* vj = j == 0 ? v0 : V[j];
      // w = H (s_j v_j); projections <s_i v_i, w>, i <= j
      double2 dt[HELM_KMAX + 1];
#pragma unroll
      for (int i = 0; i <= HELM_KMAX; ++i) dt[i] = make_double2(0.0, 0.0);
      if (act) {
        const R sj = (R)S.scale[j];
        R si[HELM_KMAX + 1];
#pragma unroll
        for (int i = 0; i <= HELM_KMAX; ++i) si[i] = i <= j ? (R)S.scale[i] : (R)0;
        for (long long p = p0 + threadIdx.x; p < p1; p += NT) {
          const C w = cscale(apply_h(g, T, vj, g.m, p), sj);
          W[p] = w;
          const double2 wd = to_d(w);
#pragma unroll
          for (int i = 0; i <= HELM_KMAX; ++i)
            if (i <= j) dt[i] = cdot_acc(dt[i], to_d(cscale(ldv((i == 0 ? v0 : V[i]) + p), si[i])), wd);
        }
      }
      grid_reduce<NT>(grid, B, dt, j + 1, part, slot0, cpr);
      if (threadIdx.x == 0 && act)
        for (int i = 0; i <= j; ++i) S.H[hidx(i, j)] = B.tot[i];
      __syncthreads();
      // v_{j+1} = w - sum_i h_ij s_i v_i (stored unnormalised), ||v_{j+1}||
      double2 n2 = make_double2(0.0, 0.0);
      if (act) {
        C cf[HELM_KMAX + 1];
#pragma unroll
        for (int i = 0; i <= HELM_KMAX; ++i) {
          const double2 h = i <= j ? S.H[hidx(i, j)] : make_double2(0.0, 0.0);
          cf[i] = mkc((R)(-h.x * S.scale[i]), (R)(-h.y * S.scale[i]));
        }
        for (long long p = p0 + threadIdx.x; p < p1; p += NT) {
          C w = W[p];
#pragma unroll
          for (int i = 0; i <= HELM_KMAX; ++i)
            if (i <= j) w = cfma(cf[i], ldv((i == 0 ? v0 : V[i]) + p), w);
          V[j + 1][p] = w;
          n2.x += (double)w.x * w.x + (double)w.y * w.y;
        }
      }
      grid_reduce<NT>(grid, B, &n2, 1, part, slot0, cpr);
      if (threadIdx.x == 0 && act) {
        close_column(S, j, sqrt(B.tot[0].x));
        if (j + 1 >= S.kact) solve_ls(S);
      }
      __syncthreads();
    }
    if (threadIdx.x == 0 && S.kact == 0) solve_ls(S);   // zero residual: y = 0
    __syncthreads();
    // x <- (zero ? 0 : x) + sum_{i < kact} y_i s_i v_i (own points only)
    C yl[HELM_KMAX];
    const int k = S.kact;
#pragma unroll
    for (int i = 0; i < HELM_KMAX; ++i) {
      const double2 yv = i < k ? S.y[i] : make_double2(0.0, 0.0);
      yl[i] = mkc((R)(yv.x * S.scale[i]), (R)(yv.y * S.scale[i]));
    }
    for (long long p = p0 + threadIdx.x; p < p1; p += NT) {
      C xv = zero ? mkc((R)0, (R)0) : x[p];
#pragma unroll
      for (int i = 0; i < HELM_KMAX; ++i)
        if (i < k) xv = cfma(yl[i], ldv((i == 0 ? v0 : V[i]) + p), xv);
      x[p] = xv;
    }
    grid.sync();   // x complete before the next residual reads neighbours
  }
}

}  // namespace persist

template <typename R, int NT>
__global__ void __launch_bounds__(NT) k_vcycle_persist(const __grid_constant__ PersistArgs<R> a) {
  namespace cg = cooperative_groups;
  using C = cx<R>;
  cg::grid_group grid = cg::this_grid();
  __shared__ persist::Block<NT> B;
  __shared__ persist::State S;
  const int ia = blockIdx.x / a.cpr, cir = blockIdx.x % a.cpr;
  const int r = a.active ? a.active[ia] : ia;
  const int slot0 = ia * a.cpr;
  const Geo<R>& gf = a.gf;
  const Geo<R>& gc = a.gc;
  const OpTab<R> Tf = op_tab(gf, r), Tc = op_tab(gc, r);
  const long long Nf = gf.N, Nc = gc.N;
  const long long f0 = Nf * cir / a.cpr, f1 = Nf * (cir + 1) / a.cpr;   // this CTA's fine points
  const long long c0 = Nc * cir / a.cpr, c1 = Nc * (cir + 1) / a.cpr;   // and coarse points
  const long long of = (long long)r * Nf, oc = (long long)r * Nc;
  C* Vf[HELM_KMAX + 1];
  C* Vc[HELM_KMAX + 1];
  for (int i = 0; i <= a.ks_i; ++i) Vf[i] = a.SV[i] + of;
  for (int i = 0; i <= a.kc_i; ++i) Vc[i] = a.FV[i] + oc;
  const C* b = a.b + of;
  C* x = a.x + of;
  // (1) pre-smooth from 0
  persist::gmres<R, NT>(grid, B, S, gf, Tf, b, x, true, a.ks_o, a.ks_i, Vf, a.SW + of, f0, f1, a.part, slot0, a.cpr);
  // (2) r = b - H x, restricted: r_c = 2^-d P^T r (the residual goes to SV[0])
  for (long long p = f0 + threadIdx.x; p < f1; p += NT)
    Vf[0][p] = csub(persist::ldv(b + p), persist::apply_h(gf, Tf, x, gf.m, p));
  grid.sync();
  {
    const int fx = gf.nx, fy = gf.ny, fz = gf.nz, cxn = gc.nx, cyn = gc.ny;
    const int hy = a.has_y;
    for (long long p = c0 + threadIdx.x; p < c1; p += NT) {
      const int jx = (int)(p % cxn), jy = (int)((p / cxn) % cyn), jz = (int)(p / ((long long)cxn * cyn));
      C acc = mkc((R)0, (R)0);
      for (int dz = -1; dz <= 1; ++dz) {
        const int iz = 2 * jz + dz;
        if (iz < 0 || iz >= fz) continue;
        const R wz = dz == 0 ? (R)1 : (R)0.5;
        for (int dy = -hy; dy <= hy; ++dy) {
          const int iy = hy ? 2 * jy + dy : 0;
          if (iy < 0 || iy >= fy) continue;
          const R wy = wz * (dy == 0 ? (R)1 : (R)0.5);
          for (int dx = -1; dx <= 1; ++dx) {
            const int ix = 2 * jx + dx;
            if (ix < 0 || ix >= fx) continue;
            const R w = wy * (dx == 0 ? (R)1 : (R)0.5);
            const C v = persist::ldv(Vf[0] + ((long long)iz * fy + iy) * fx + ix);
            acc.x += w * v.x;
            acc.y += w * v.y;
          }
        }
      }
      a.Fb[oc + p] = mkc(acc.x * a.fac, acc.y * a.fac);
    }
  }
  grid.sync();
  // (3) coarsest GMRES from 0
  persist::gmres<R, NT>(grid, B, S, gc, Tc, a.Fb + oc, a.Fx + oc, true, a.kc_o, a.kc_i, Vc, a.FW + oc, c0, c1, a.part,
                        slot0, a.cpr);
  // (4) x += P x_c
  {
    const int fx = gf.nx, fy = gf.ny, cxn = gc.nx, cyn = gc.ny, czn = gc.nz;
    const C* cin = a.Fx + oc;
    for (long long p = f0 + threadIdx.x; p < f1; p += NT) {
      const int ix = (int)(p % fx), iy = (int)((p / fx) % fy), iz = (int)(p / ((long long)fx * fy));
      int jx[2], jy[2], jz[2];
      R wx[2], wy[2], wz[2];
      int nxp, nyp, nzp;
      auto axis = [](int i, int nc, int* j, R* w, int& n) {
        if ((i & 1) == 0) { j[0] = i >> 1; w[0] = (R)1; n = 1; }
        else { j[0] = i >> 1; w[0] = (R)0.5; j[1] = (i >> 1) + 1; w[1] = (R)0.5; n = j[1] < nc ? 2 : 1; }
      };
      axis(ix, cxn, jx, wx, nxp);
      axis(iz, czn, jz, wz, nzp);
      if (a.has_y) axis(iy, cyn, jy, wy, nyp);
      else { jy[0] = 0; wy[0] = (R)1; nyp = 1; }
      C acc = mkc((R)0, (R)0);
      for (int u = 0; u < nzp; ++u)
        for (int v = 0; v < nyp; ++v)
          for (int w = 0; w < nxp; ++w) {
            const R wt = wz[u] * wy[v] * wx[w];
            const C c = persist::ldv(cin + ((long long)jz[u] * cyn + jy[v]) * cxn + jx[w]);
            acc.x += wt * c.x;
            acc.y += wt * c.y;
          }
      x[p] = cadd(x[p], acc);
    }
  }
  grid.sync();
  // (5) post-smooth from x
  persist::gmres<R, NT>(grid, B, S, gf, Tf, b, x, false, a.ks_o, a.ks_i, Vf, a.SW + of, f0, f1, a.part, slot0, a.cpr);
}
