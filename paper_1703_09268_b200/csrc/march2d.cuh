// march2d.cuh — register z-march stencil for 2D grids (a2, and a3's fused Arnoldi), sm_100a.
//
// In 2D the rows of a batch are independent right-hand sides and the stencil couples only
// x±1 and z±1 (D4-D5). One warp owns one x-strip of one RHS: lane l sits at x = x0 - 1 + l,
// lanes 1..30 produce outputs and lanes 0 / 31 only carry the strip's halo, so every lane
// loads exactly one point of every operand per plane (coalesced 512 B per warp, no extra
// halo requests), x-neighbours come from warp shuffles, z-neighbours from the register
// march, and the next P planes are prefetched into registers (plain 16-B loads; P planes x
// ~14 warps per SM keep ~50-100 KB in flight per SM). The level's z coefficients sit in
// shared memory (filled once per CTA); there is no barrier on the streaming path and every
// warp streams independently. Work items are (strip, z-chunk) pairs of one RHS,
// dealt round-robin to the RHS's warps; each warp reduces its projections in registers and
// the per-RHS slot reduction (warp_slot_reduce) finishes in fixed order.
//
// Modes as stencil.cuh: 0 y = s H x; 1 y = b - H x and ||y||; 2 y = s H x with <V_i, y>,
// i < NV; 3 fused GMRES step NV (form V_NV = s W - sum h s_i V_i on the fly, write V_NV and
// Y = H V_NV, dots <V_i, Y> i <= NV, ||V_NV||^2); 4 = 3 for the last step (Y not stored,
// ||Y||^2 reduced, last column by Pythagoras).
#pragma once
#include "stencil.cuh"

template <typename R> struct MarchArgs {
  Geo<R> g;
  const cx<R>* x;          // marched operand: x (MODE 0-2), V_0 or raw W (MODE 3/4)
  cx<R>* y;
  const cx<R>* b;          // MODE 1
  VPtrs<R> V;              // MODE 2: V_0..V_{NV-1} own points; MODE 3/4: the basis to form with
  cx<R>* vout;             // MODE 3/4, NV > 0: formed V_NV
  const double* xscale;    // MODE 0/2 lazy scale per RHS (stride sstride) or null
  int sstride;
  const int* active;        // compact list of the active RHS (null: all), nrhs entries
  const int* kact;
  int jskip, jstep;
  int nrhs;                 // active RHS processed by this launch
  int nstrip;              // strips of 30 outputs per row
  int wpr;                 // warps per RHS
  int nzc, zlen;           // z-chunks per strip
  KCtx ctx;
  RedBuf rb;
};

template <typename R, int MODE, int NV> struct MarchPlane {
  static constexpr int NB = (MODE == 2 || MODE >= 3) ? NV : 0;   // basis values per point
  cx<R> x;                 // marched operand (raw W for MODE 3/4, NV > 0)
  cx<R> v[NB > 0 ? NB : 1];
  cx<R> b;                 // MODE 1
  R m;
};

template <typename R, int MODE, int NV, int P>
__global__ void __launch_bounds__(128)
k_march2d(const MarchArgs<R> a) {
  using C = cx<R>;
  using PL = MarchPlane<R, MODE, NV>;
  constexpr int NB = PL::NB;
  constexpr bool FORM = MODE >= 3 && NV > 0;
  constexpr bool LAST = MODE == 4;
  constexpr int NVR = MODE == 1 ? 1 : (MODE == 2 ? NV : (MODE >= 3 ? NV + 3 : 1));
  const Geo<R>& g = a.g;
  const int nx = g.nx, nz = g.nz;
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int ia = gw / a.wpr, wi = gw % a.wpr;   // ia: index in the compact active-RHS list
  const int r = ia < a.nrhs ? (a.active ? a.active[ia] : ia) : 0;
  const long long N = g.N;
  const long long rb0 = (long long)r * N;
  const C zero = mkc((R)0, (R)0);
  // z coefficients of every operator of the level in shared memory (ghosts masked, R7):
  // nop x nz x 3 complex
  extern __shared__ __align__(16) unsigned char zsm[];
  C* zt = reinterpret_cast<C*>(zsm);
  for (int e = threadIdx.x; e < g.nop * nz; e += blockDim.x) {
    const int z = e % nz;
    zt[3 * e] = z > 0 ? g.lo[2][e] : zero;
    zt[3 * e + 1] = g.dg[2][e];
    zt[3 * e + 2] = z < nz - 1 ? g.up[2][e] : zero;
  }
  __syncthreads();
  if (ia >= a.nrhs) return;
  if (a.kact && a.jskip >= a.kact[r]) return;

  R sc = (R)1;
  if ((MODE == 0 || MODE == 2) && a.xscale) sc = (R)a.xscale[(long long)r * a.sstride];
  const OpTab<R> T = op_tab(g, r);
  const C* ztr = zt + 3 * (long long)(g.rop ? g.rop[r] : 0) * nz;
  R cw = (R)1;
  C cv[FORM ? NV : 1];
  if constexpr (FORM) {
    const double* s = a.ctx.scale + (long long)r * (HELM_KMAX + 1);
    const double2* H = a.ctx.H + (long long)r * (HELM_KMAX + 1) * HELM_KMAX;
    cw = (R)s[NV - 1];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const double2 h = H[hidx(i, NV - 1)];
      cv[i] = mkc((R)(-h.x * s[i]), (R)(-h.y * s[i]));
    }
  }

  double2 acc[NVR];
#pragma unroll
  for (int k = 0; k < NVR; ++k) acc[k] = make_double2(0.0, 0.0);
  double nrm = 0.0, ynrm = 0.0;

  const int nitems = a.nstrip * a.nzc;
  for (int it = wi; it < nitems; it += a.wpr) {
    const int strip = it % a.nstrip, zc = it / a.nstrip;
    const int z0 = zc * a.zlen, z1 = min(nz, z0 + a.zlen);
    const int x = strip * 30 - 1 + lane;
    const bool inx = x >= 0 && x < nx;
    const bool outp = lane >= 1 && lane <= 30 && inx;
    const long long xo = rb0 + (inx ? x : 0);
    const C lox = outp ? T.lo[0][x] : zero, upx = outp ? T.up[0][x] : zero, dgx = outp ? T.dg[0][x] : zero;

    // load one plane (z may be a ghost plane: zeros, R7)
    auto load = [&](int z, PL& p) {
      const bool ok = inx && z >= 0 && z < nz;
      const long long o = xo + (long long)z * nx;
      p.x = ok ? a.x[o] : zero;
#pragma unroll
      for (int i = 0; i < NB; ++i) p.v[i] = ok ? a.V.p[i][o] : zero;
      if constexpr (MODE == 1) p.b = ok ? a.b[o] : zero;
      p.m = ok ? g.m[x + (long long)z * nx] : (R)0;
    };
    auto formed = [&](const PL& p) -> C {
      if constexpr (FORM) {
        C v = cscale(p.x, cw);
#pragma unroll
        for (int i = 0; i < NV; ++i) v = cfma(cv[i], p.v[i], v);
        return v;
      } else {
        return p.x;
      }
    };

    // march state: formed operand at z-1, z, z+1 and the planes z, z+1 themselves
    PL pc, pn;            // planes z (current) and z+1
    PL q[P];              // prefetched planes z+2 .. z+1+P (ring, static index)
    {
      PL pm;
      load(z0 - 1, pm);
      load(z0, pc);
      load(z0 + 1, pn);
#pragma unroll
      for (int k = 0; k < P; ++k) load(z0 + 2 + k, q[k]);
      C fm = formed(pm), f0 = formed(pc), fp = formed(pn);
      for (int zb = z0; zb < z1; zb += P) {
#pragma unroll
        for (int k = 0; k < P; ++k) {
          const int z = zb + k;
          if (z < z1) {
            // ---- compute plane z
            C left = mkc(__shfl_up_sync(0xffffffffu, f0.x, 1), __shfl_up_sync(0xffffffffu, f0.y, 1));
            C right = mkc(__shfl_down_sync(0xffffffffu, f0.x, 1), __shfl_down_sync(0xffffffffu, f0.y, 1));
            const R wm = T.w2 * pc.m;
            const C lz = ztr[3 * z], dz = ztr[3 * z + 1], uz = ztr[3 * z + 2];
            C t0 = cmul(mkc(dgx.x + dz.x + wm, dgx.y + dz.y), f0);
            C t1 = cfma(upx, right, cmul(lox, left));
            C t2 = cfma(uz, fp, cmul(lz, fm));
            const C hx = cadd(cadd(t0, t1), t2);
            if (outp) {
              const long long o = xo + (long long)z * nx;
              if constexpr (MODE == 0) {
                a.y[o] = cscale(hx, sc);
              } else if constexpr (MODE == 1) {
                const C rv = csub(pc.b, hx);
                a.y[o] = rv;
                nrm += (double)rv.x * rv.x + (double)rv.y * rv.y;
              } else if constexpr (MODE == 2) {
                const C w = cscale(hx, sc);
                a.y[o] = w;
                const double2 wd = to_d(w);
#pragma unroll
                for (int i = 0; i < NV; ++i) acc[i] = cdot_acc(acc[i], to_d(pc.v[i]), wd);
              } else {
                const double2 hd = to_d(hx);
                if constexpr (LAST) ynrm += hd.x * hd.x + hd.y * hd.y;
                else a.y[o] = hx;
#pragma unroll
                for (int i = 0; i < NV; ++i) acc[i] = cdot_acc(acc[i], to_d(pc.v[i]), hd);
                acc[NV] = cdot_acc(acc[NV], to_d(f0), hd);
                if constexpr (NV > 0) {
                  a.vout[o] = f0;
                  nrm += (double)f0.x * f0.x + (double)f0.y * f0.y;
                }
              }
            }
            // ---- advance: z+1 becomes current, q[k] (plane z+2) is formed, refill q[k]
            fm = f0;
            f0 = fp;
            pc = pn;
            pn = q[k];
            fp = formed(pn);
            load(z + 2 + P, q[k]);
          }
        }
      }
    }
  }

  if constexpr (MODE != 0) {
    if constexpr (MODE == 1) acc[0] = make_double2(nrm, 0.0);
    if constexpr (MODE >= 3) acc[NV + 1] = make_double2(nrm, 0.0);
    if constexpr (MODE >= 3) acc[NV + 2] = make_double2(ynrm, 0.0);
    double2 tot[NVR];
    // partials indexed by the compact index (<= one wave of warps in total), ticket by RHS
    if (warp_slot_reduce<NVR>(acc, a.rb.part + (size_t)ia * a.wpr * NVR, a.rb.ticket + r, wi, a.wpr, tot)) {
      if (lane == 0) plane_epilogue<MODE, NV>(a.ctx, r, a.jstep, tot);
    }
  }
}

// ---------------------------------------------------------------------------------------
// 3D matvec y = s H x (a2, `helm_apply` and the cfg5 sweep) as a register z-march: one warp
// owns RY consecutive y-rows of a 30-point x-strip of one RHS (lanes 0 / 31 carry the x
// halo), loads the RY + 2 rows y0-1 .. y0+RY of every plane (the y halo rows: 1 + 2/RY reads
// per point from L2, one from HBM), takes x-neighbours by shuffle, y-neighbours from its own
// registers and z-neighbours from the march, and prefetches P planes. No shared memory
// beyond the z-table, no barriers. Items (y-block, strip, z-chunk) of one RHS are dealt to
// that RHS's warps round-robin with the y-block fastest (neighbouring blocks share halo rows
// in L2 at the same depth).
template <typename R> struct March3Args {
  Geo<R> g;
  const cx<R>* x;
  cx<R>* y;
  const double* xscale;
  int sstride;
  const int* active;        // compact list of the active RHS (null: all)
  int nrhs, nstrip, nyb, wpr, nzc, zlen;
};

template <typename R, int RY> struct M3Plane {
  cx<R> x[RY + 2];   // rows y0-1 .. y0+RY
  R m[RY];
};

template <typename R, int RY, int P>
__global__ void __launch_bounds__(128)
k_march3d(const March3Args<R> a) {
  using C = cx<R>;
  using PL = M3Plane<R, RY>;
  const Geo<R>& g = a.g;
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const long long plane = (long long)nx * ny;
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int ia = gw / a.wpr, wi = gw % a.wpr;
  const int r = ia < a.nrhs ? (a.active ? a.active[ia] : ia) : 0;
  const C zero = mkc((R)0, (R)0);
  extern __shared__ __align__(16) unsigned char zsm3[];
  C* zt = reinterpret_cast<C*>(zsm3);
  for (int e = threadIdx.x; e < g.nop * nz; e += blockDim.x) {
    const int z = e % nz;
    zt[3 * e] = z > 0 ? g.lo[2][e] : zero;
    zt[3 * e + 1] = g.dg[2][e];
    zt[3 * e + 2] = z < nz - 1 ? g.up[2][e] : zero;
  }
  __syncthreads();
  if (ia >= a.nrhs) return;
  const R sc = a.xscale ? (R)a.xscale[(long long)r * a.sstride] : (R)1;
  const OpTab<R> T = op_tab(g, r);
  const C* ztr = zt + 3 * (long long)(g.rop ? g.rop[r] : 0) * nz;
  const long long rb0 = (long long)r * g.N;

  const int nitems = a.nyb * a.nstrip * a.nzc;
  for (int it = wi; it < nitems; it += a.wpr) {
    const int yb = it % a.nyb, strip = (it / a.nyb) % a.nstrip, zc = it / (a.nyb * a.nstrip);
    const int z0 = zc * a.zlen, z1 = min(nz, z0 + a.zlen);
    const int y0 = yb * RY;
    const int x = strip * 30 - 1 + lane;
    const bool inx = x >= 0 && x < nx;
    const bool outx = lane >= 1 && lane <= 30 && inx;
    const C lox = outx ? T.lo[0][x] : zero, upx = outx ? T.up[0][x] : zero, dgx = outx ? T.dg[0][x] : zero;
    C loy[RY], upy[RY], dgy[RY];
    bool rowok[RY + 2];
#pragma unroll
    for (int k = 0; k < RY + 2; ++k) rowok[k] = (y0 - 1 + k) >= 0 && (y0 - 1 + k) < ny;
#pragma unroll
    for (int k = 0; k < RY; ++k) {
      const int yy = y0 + k;
      const bool ok = yy < ny;
      loy[k] = ok && yy > 0 ? T.lo[1][yy] : zero;
      upy[k] = ok && yy < ny - 1 ? T.up[1][yy] : zero;
      dgy[k] = ok ? T.dg[1][yy] : zero;
    }
    const long long xo = rb0 + (inx ? x : 0) + (long long)(y0 - 1) * nx;
    auto load = [&](int z, PL& p) {
      const bool zin = inx && z >= 0 && z < nz;
      const long long o = xo + (long long)z * plane;
#pragma unroll
      for (int k = 0; k < RY + 2; ++k) p.x[k] = (zin && rowok[k]) ? a.x[o + (long long)k * nx] : zero;
#pragma unroll
      for (int k = 0; k < RY; ++k) p.m[k] = (zin && rowok[k + 1]) ? g.m[o - rb0 + (long long)(k + 1) * nx] : (R)0;
    };
    PL pc, pn, q[P];    // full planes z, z+1 and the prefetched z+2 .. z+1+P
    C xm[RY];           // own rows at z-1
    {
      PL t;
      load(z0 - 1, t);
#pragma unroll
      for (int k = 0; k < RY; ++k) xm[k] = t.x[k + 1];
      load(z0, pc);
      load(z0 + 1, pn);
#pragma unroll
      for (int k = 0; k < P; ++k) load(z0 + 2 + k, q[k]);
    }
    for (int zb = z0; zb < z1; zb += P) {
#pragma unroll
      for (int j = 0; j < P; ++j) {
        const int z = zb + j;
        if (z < z1) {
          const C lz = ztr[3 * z], dz = ztr[3 * z + 1], uz = ztr[3 * z + 2];
#pragma unroll
          for (int k = 0; k < RY; ++k) {
            const C cur = pc.x[k + 1];
            const C left = mkc(__shfl_up_sync(0xffffffffu, cur.x, 1), __shfl_up_sync(0xffffffffu, cur.y, 1));
            const C right = mkc(__shfl_down_sync(0xffffffffu, cur.x, 1), __shfl_down_sync(0xffffffffu, cur.y, 1));
            const R wm = T.w2 * pc.m[k];
            C t0 = cmul(mkc(dgx.x + dgy[k].x + dz.x + wm, dgx.y + dgy[k].y + dz.y), cur);
            C t1 = cfma(upx, right, cmul(lox, left));
            C t2 = cfma(uz, pn.x[k + 1], cmul(lz, xm[k]));
            C t3 = cfma(upy[k], pc.x[k + 2], cmul(loy[k], pc.x[k]));
            const C hx = cadd(cadd(t0, t1), cadd(t2, t3));
            if (outx && rowok[k + 1]) a.y[xo + (long long)(k + 1) * nx + (long long)z * plane] = cscale(hx, sc);
          }
#pragma unroll
          for (int k = 0; k < RY; ++k) xm[k] = pc.x[k + 1];
          pc = pn;
          pn = q[j];
          load(z + 2 + P, q[j]);
        }
      }
    }
  }
}
