// march2d.cuh — register z-march stencil for 2D grids (a2, and a3's fused Arnoldi), sm_100a.
//
// In 2D the rows of a batch are independent right-hand sides and the stencil couples only
// x±1 and z±1 (D4-D5). One warp owns one x-strip of one RHS: lane l sits at x = x0 - 1 + l,
// lanes 1..30 produce outputs and lanes 0 / 31 only carry the strip's halo, so every lane
// loads exactly one point of every operand per plane (coalesced 512 B per warp, no extra
// halo requests), x-neighbours come from warp shuffles, z-neighbours from the register
// march, and the next S-2 planes are prefetched by cp.async into a per-lane shared-memory
// ring (each lane reads back only its own copies, so the ring needs no barrier; registers
// stay free for occupancy). The level's packed z coefficients are copied into shared
// memory once per CTA. There is no barrier on the streaming path and every warp streams
// independently (a variant carrying the z coefficients in the ring needed two warp barriers
// per plane and was 12 % slower end to end). Work items are (strip, z-chunk) pairs of one RHS,
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
  int nzc, zlen;           // z-chunks per strip and their length
  int S;                   // per-lane prefetch ring depth (planes)
  KCtx ctx;
  RedBuf rb;
  // TMA feed (complex128): tm[i] = operand i of the stage as [rhs][z][x] 8-byte words, box =
  // one 32-point strip row (x0-1 .. x0+30); tmm = m's 16-B pitched copy, box = 34 reals from
  // x0-2 (TMA box starts must be 16-B aligned). Out-of-bounds elements are zero-filled (R7).
  int tma;
  CUtensorMap tm[HELM_KMAX + 2];
  CUtensorMap tmm;
};

// Per-lane prefetch ring in shared memory: every lane only ever reads back what it copied
// itself (neighbours travel as formed values through shuffles), so the ring needs no
// barrier at all — cp.async.wait_group per lane is the whole synchronisation, and the
// registers stay free for occupancy. Stage layout (per warp): NX operand arrays of 32
// complex, then 32 reals of m.
template <typename R, int MODE, int NV, bool TM = false> struct MarchShape {
  static constexpr int NB = (MODE == 2 || MODE >= 3) ? NV : 0;    // basis operands
  static constexpr int NX = 1 + NB + (MODE == 1 ? 1 : 0);         // x/W, V_i, b
  // TMA: every box lands 128-B aligned; m is a 34-real box starting one point before the strip
  static constexpr int stage_bytes = TM ? (NX * 32 * (int)sizeof(cx<R>) + 34 * (int)sizeof(R) + 127) / 128 * 128
                                        : (32 * (NX * (int)sizeof(cx<R>) + (int)sizeof(R)) + 15) / 16 * 16;
  static constexpr int m_off = NX * 32 * (int)sizeof(cx<R>);
};

// One march pass over the (strip, z-chunk) items of RHS r owned by warp `wi` of `nw`: the
// streaming body of k_march2d. Accumulates this warp's partial projections / norms.
template <typename R, int MODE, int NV, int NVR, int ST = 0, bool TM = false>
__device__ __forceinline__ void march_pass(const Geo<R>& g, const OpTab<R>& T, const cx<R>* ztr, long long rb0,
                                           const cx<R>* xin, const cx<R>* bin, cx<R>* yout, cx<R>* vout,
                                           const cx<R>* const* Vp, R sc, R cw, const cx<R> (&cv)[(MODE >= 3 && NV > 0) ? NV : 1],
                                           int nstrip, int nzc, int zlen, int wi, int nw, int S, unsigned char* ring,
                                           unsigned ring_s, double2 (&acc)[NVR], double& nrm, double& ynrm,
                                           const MarchArgs<R>* ta = nullptr, int rhs = 0, unsigned mb_s = 0) {
  using C = cx<R>;
  using SH = MarchShape<R, MODE, NV, TM>;
  constexpr int NB = SH::NB, NX = SH::NX, SB = SH::stage_bytes;
  constexpr bool FORM = MODE >= 3 && NV > 0;
  constexpr bool LAST = MODE == 4;
  const int nx = g.nx, nz = g.nz;
  const int lane = threadIdx.x & 31;
  const C zero = mkc((R)0, (R)0);
  const int nitems = nstrip * nzc;
  unsigned par = 0;   // TMA: expected parity of each slot's mbarrier (persists across items)
  for (int it = wi; it < nitems; it += nw) {
    const int strip = it % nstrip, zc = it / nstrip;
    const int z0 = zc * zlen, z1 = min(nz, z0 + zlen);
    const int x = strip * 30 - 1 + lane;
    const bool inx = x >= 0 && x < nx;
    const bool outp = lane >= 1 && lane <= 30 && inx;
    const long long xo = rb0 + (inx ? x : 0);
    const C lox = outp ? T.lo[0][x] : zero, upx = outp ? T.up[0][x] : zero, dgx = outp ? T.dg[0][x] : zero;
    const C* src[NX];
    src[0] = xin + xo;
#pragma unroll
    for (int i = 0; i < NB; ++i) src[1 + i] = Vp[i] + xo;
    if constexpr (MODE == 1) src[NX - 1] = bin + xo;
    const R* msrc = g.m + (inx ? x : 0);

    // TMA: one elected lane issues the boxes of plane q into slot sl on the slot's mbarrier
    // (every lane tracks the slot parities); the slot's previous contents were read by the
    // generic proxy of every lane, hence the warp barrier before each refill (issue_tm callers)
    auto issue_tm = [&](int q, int sl) {
      if (q <= z1) {
        if (lane == 0) {
          fence_proxy_async();
          const unsigned bar = mb_s + 8 * sl, d = ring_s + (unsigned)(sl * SB);
          mbar_expect_tx(bar, (unsigned)(NX * 32 * sizeof(C) + 34 * sizeof(R)));
          constexpr int CR = (int)(sizeof(C) / 8);
#pragma unroll
          for (int i = 0; i < NX; ++i)
            tma_load3(d + (unsigned)(i * 32 * sizeof(C)), &ta->tm[i], bar, CR * (strip * 30 - 1), q, rhs);
          tma_load2(d + (unsigned)SH::m_off, &ta->tmm, bar, strip * 30 - 2, q);
        }
        par ^= 1u << sl;
      }
    };
    auto wait_tm = [&](int sl) { mbar_wait(mb_s + 8 * sl, ((par >> sl) & 1u) ^ 1u); };
    // plane q (may be a ghost plane: zero-filled, R7) into ring slot `sl`; one commit group
    auto issue = [&](int q, int sl) {
      if constexpr (TM) { issue_tm(q, sl); return; }
      if (q <= z1) {
        const bool ok = inx && q >= 0 && q < nz;
        const long long zo = ok ? (long long)q * nx : 0;
        const unsigned d = ring_s + (unsigned)(sl * SB);
#pragma unroll
        for (int i = 0; i < NX; ++i) cpa<sizeof(C)>(d + (unsigned)((i * 32 + lane) * sizeof(C)), src[i] + zo, ok);
        cpa<sizeof(R)>(d + (unsigned)(NX * 32 * sizeof(C) + lane * sizeof(R)), msrc + zo, ok);
      }
      cpa_commit();
    };
    auto opnd = [&](int sl, int i) -> C {
      return *reinterpret_cast<const C*>(ring + sl * SB + (i * 32 + lane) * sizeof(C));
    };
    auto formed = [&](int sl) -> C {
      C v = opnd(sl, 0);
      if constexpr (FORM) {
        v = cscale(v, cw);
#pragma unroll
        for (int i = 0; i < NV; ++i) v = cfma(cv[i], opnd(sl, 1 + i), v);
      }
      return v;
    };

    auto mval = [&](int sl) -> R {
      return *reinterpret_cast<const R*>(ring + sl * SB + SH::m_off + (lane + (TM ? 1 : 0)) * sizeof(R));
    };
    auto shu = [](C v) { return mkc(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1)); };
    auto shd = [](C v) { return mkc(__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1)); };

    // prologue: planes z0-1 .. z0+S-2 into slots 0 .. S-1 (slot of plane q: (q - z0 + 1) % S)
    for (int k = 0; k < S; ++k) issue(z0 - 1 + k, k);
    if constexpr (TM) { wait_tm(0); wait_tm(1); }
    else cpa_wait_n(S - 2);                 // planes z0-1, z0 landed
    C fm = formed(0);
    R mm = ST == 1 ? mval(0) : (R)0;        // OPT: the model of plane z-1 rides along in a register
    if constexpr (TM) __syncwarp();         // every lane is done with slot 0
    issue(z0 - 1 + S, 0);                   // slot of z0-1 is free again
    C f0 = formed(1);
    int s0 = 1;                             // slot of plane z
    for (int z = z0; z < z1; ++z) {
      const int s1 = s0 + 1 == S ? 0 : s0 + 1;
      if constexpr (TM) wait_tm(s1);
      else cpa_wait_n(S - 2);               // plane z+1 landed (planes up to z+S-1 issued)
      const C fp = formed(s1);
      // ---- compute plane z
      const C left = shu(f0), right = shd(f0);
      const R mz = mval(s0);
      const C lz = ztr[3 * z], dz = ztr[3 * z + 1], uz = ztr[3 * z + 2];
      C hx;
      if constexpr (ST == 1) {
        // R34 (2D "9pt optimal", P:204 [23]): coef(dx, dz) = tx[dx] G9[dz] + tz[dz] G9[dx], and
        // the mass distribution M (centre C9, edges D9/4, corners E9/4) of m u (Eq. 7, A = M)
        const R g0 = (R)optw::G9_0, g1 = (R)optw::G9_1;
        const C ul = shu(fm), ur = shd(fm), dl = shu(fp), dr = shd(fp);   // (x-1, z-1), (x+1, z-1), (x-1, z+1), (x+1, z+1)
        auto ax = [&](C t, R gz) { return mkc(t.x * gz, t.y * gz); };
        C acc = cmul(cadd(ax(dgx, g0), ax(dz, g0)), f0);                                  // (0, 0)
        acc = cfma(cadd(ax(lox, g0), ax(dz, g1)), left, acc);                              // (-1, 0)
        acc = cfma(cadd(ax(upx, g0), ax(dz, g1)), right, acc);                             // (+1, 0)
        acc = cfma(cadd(ax(dgx, g1), ax(lz, g0)), fm, acc);                                // (0, -1)
        acc = cfma(cadd(ax(dgx, g1), ax(uz, g0)), fp, acc);                                // (0, +1)
        acc = cfma(cadd(ax(lox, g1), ax(lz, g1)), ul, acc);                                // (-1, -1)
        acc = cfma(cadd(ax(upx, g1), ax(lz, g1)), ur, acc);                                // (+1, -1)
        acc = cfma(cadd(ax(lox, g1), ax(uz, g1)), dl, acc);                                // (-1, +1)
        acc = cfma(cadd(ax(upx, g1), ax(uz, g1)), dr, acc);                                // (+1, +1)
        // forward: M diag(m) u (neighbours' m); adjoint (tables of H^H): diag(m) M u (H^H =
        // L^H + omega^2 diag(m) M, M real symmetric)
        const bool adj = g.adj != 0;
        const R mp = mval(s1);
        const R mlft = adj ? (R)1 : __shfl_up_sync(0xffffffffu, mz, 1);
        const R mrgt = adj ? (R)1 : __shfl_down_sync(0xffffffffu, mz, 1);
        C ms = cscale(f0, (R)optw::MU9_0 * (adj ? (R)1 : mz));
        ms = cfma(mkc((R)optw::MU9_1 * mlft, (R)0), left, ms);
        ms = cfma(mkc((R)optw::MU9_1 * mrgt, (R)0), right, ms);
        ms = cfma(mkc((R)optw::MU9_1 * (adj ? (R)1 : mm), (R)0), fm, ms);
        ms = cfma(mkc((R)optw::MU9_1 * (adj ? (R)1 : mp), (R)0), fp, ms);
        if constexpr (optw::MU9_2 != 0.0) {
          const R mul = adj ? (R)1 : __shfl_up_sync(0xffffffffu, mm, 1), mur = adj ? (R)1 : __shfl_down_sync(0xffffffffu, mm, 1);
          const R mdl = adj ? (R)1 : __shfl_up_sync(0xffffffffu, mp, 1), mdr = adj ? (R)1 : __shfl_down_sync(0xffffffffu, mp, 1);
          ms = cfma(mkc((R)optw::MU9_2 * mul, (R)0), ul, ms);
          ms = cfma(mkc((R)optw::MU9_2 * mur, (R)0), ur, ms);
          ms = cfma(mkc((R)optw::MU9_2 * mdl, (R)0), dl, ms);
          ms = cfma(mkc((R)optw::MU9_2 * mdr, (R)0), dr, ms);
        }
        const R wm = adj ? T.w2 * mz : T.w2;
        hx = mkc(acc.x + wm * ms.x, acc.y + wm * ms.y);
        mm = mz;
      } else {
        const R wm = T.w2 * mz;
        C t0 = cmul(mkc(dgx.x + dz.x + wm, dgx.y + dz.y), f0);
        C t1 = cfma(upx, right, cmul(lox, left));
        C t2 = cfma(uz, fp, cmul(lz, fm));
        hx = cadd(cadd(t0, t1), t2);
      }
      if (outp) {
        const long long o = xo + (long long)z * nx;
        if constexpr (MODE == 0) {
          yout[o] = cscale(hx, sc);
        } else if constexpr (MODE == 1) {
          const C rv = csub(opnd(s0, NX - 1), hx);
          yout[o] = rv;
          nrm += (double)rv.x * rv.x + (double)rv.y * rv.y;
        } else if constexpr (MODE == 2) {
          const C w = cscale(hx, sc);
          yout[o] = w;
          const double2 wd = to_d(w);
#pragma unroll
          for (int i = 0; i < NV; ++i) acc[i] = cdot_acc(acc[i], to_d(opnd(s0, 1 + i)), wd);
        } else {
          const double2 hd = to_d(hx);
          if constexpr (LAST) ynrm += hd.x * hd.x + hd.y * hd.y;
          else yout[o] = hx;
#pragma unroll
          for (int i = 0; i < NV; ++i) acc[i] = cdot_acc(acc[i], to_d(opnd(s0, 1 + i)), hd);
          acc[NV] = cdot_acc(acc[NV], to_d(f0), hd);
          if constexpr (NV > 0) {
            vout[o] = f0;
            nrm += (double)f0.x * f0.x + (double)f0.y * f0.y;
          }
        }
      }
      // ---- advance: slot of plane z is free -> plane z+S
      if constexpr (TM) __syncwarp();
      issue(z + S, s0);
      fm = f0;
      f0 = fp;
      s0 = s1;
    }
    if constexpr (!TM) cpa_wait<0>();      // (TMA: every issued plane <= z1 was waited for)
    __syncwarp();
  }
}

// Forming coefficients of fused step NV (MODE 3/4): V_NV = cw W + sum_i cv_i V_i.
template <typename R, int NV>
__device__ __forceinline__ void form_coeffs(const KCtx& ctx, int r, R& cw, cx<R> (&cv)[NV > 0 ? NV : 1]) {
  if constexpr (NV > 0) {
    const double* s = ctx.scale + (long long)r * (HELM_KMAX + 1);
    const double2* H = ctx.H + (long long)r * (HELM_KMAX + 1) * HELM_KMAX;
    cw = (R)s[NV - 1];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const double2 h = H[hidx(i, NV - 1)];
      cv[i] = mkc((R)(-h.x * s[i]), (R)(-h.y * s[i]));
    }
  }
}

template <typename R, int MODE, int NV, int ST = 0, bool TM = false>
__global__ void __launch_bounds__(128)
k_march2d(const __grid_constant__ MarchArgs<R> a) {
  pdl_wait();
  pdl_trigger();
  using C = cx<R>;
  using SH = MarchShape<R, MODE, NV, TM>;
  constexpr int SB = SH::stage_bytes;
  constexpr bool FORM = MODE >= 3 && NV > 0;
  constexpr int NVR = MODE == 1 ? 1 : (MODE == 2 ? NV : (MODE >= 3 ? NV + 3 : 1));
  const Geo<R>& g = a.g;
  const int nz = g.nz, S = a.S;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gw = blockIdx.x * (blockDim.x >> 5) + wib;
  const int ia = gw / a.wpr, wi = gw % a.wpr;   // ia: index in the compact active-RHS list
  const int r = ia < a.nrhs ? (a.active ? a.active[ia] : ia) : 0;
  // z coefficients of every operator of the level (packed, ghosts masked, R7) in shared
  // memory: one contiguous copy per CTA
  extern __shared__ __align__(16) unsigned char msm[];
  // (cp.async: every element in flight at once — a load/store loop here cost several L2
  // round trips per launch, a fixed latency that dominated the small late-cycle batches)
  C* zt = reinterpret_cast<C*>(msm);
  {
    const unsigned zs = (unsigned)__cvta_generic_to_shared(zt);
    for (int e = threadIdx.x; e < 3 * g.nop * nz; e += blockDim.x) cpa<sizeof(C)>(zs + e * (unsigned)sizeof(C), g.zpk + e, true);
    cpa_commit();
    cpa_wait<0>();
  }
  __syncthreads();
  if (ia >= a.nrhs) return;
  if (a.kact && a.jskip >= a.kact[r]) return;
  const size_t zbytes = TM ? ((size_t)3 * g.nop * nz * sizeof(C) + 127) / 128 * 128
                           : ((size_t)3 * g.nop * nz * sizeof(C) + 15) / 16 * 16;
  unsigned char* ring = msm + zbytes + (size_t)wib * S * SB;
  const unsigned ring_s = (unsigned)__cvta_generic_to_shared(ring);
  // TMA: S mbarriers per warp after the four warps' rings
  const unsigned mb_s = (unsigned)__cvta_generic_to_shared(msm + zbytes + (size_t)4 * S * SB) + (unsigned)(wib * S * 8);
  if constexpr (TM) {
    if (lane == 0) {
      for (int k = 0; k < S; ++k) mbar_init(mb_s + 8 * k, 1);
      fence_mbar_init();
    }
    __syncwarp();
  }

  R sc = (R)1;
  if ((MODE == 0 || MODE == 2) && a.xscale) sc = (R)a.xscale[(long long)r * a.sstride];
  const OpTab<R> T = op_tab(g, r);
  const C* ztr = zt + 3 * (long long)(g.rop ? g.rop[r] : 0) * nz;   // this RHS's z table
  R cw = (R)1;
  C cv[FORM ? NV : 1];
  if constexpr (FORM) form_coeffs<R, NV>(a.ctx, r, cw, cv);

  double2 acc[NVR];
#pragma unroll
  for (int k = 0; k < NVR; ++k) acc[k] = make_double2(0.0, 0.0);
  double nrm = 0.0, ynrm = 0.0;
  // items (strip, z-chunk) of this RHS, strip fastest, dealt round-robin to its warps: warps
  // on neighbouring strips stream the same depth together, so the cache lines shared at
  // strip boundaries are read from HBM once (a balanced contiguous split lost up to 15 %)
  march_pass<R, MODE, NV, NVR, ST, TM>(g, T, ztr, (long long)r * g.N, a.x, a.b, a.y, a.vout, a.V.p, sc, cw, cv, a.nstrip,
                                   a.nzc, a.zlen, wi, a.wpr, S, ring, ring_s, acc, nrm, ynrm, &a, r, mb_s);

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
