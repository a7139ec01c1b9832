// stencil.cuh — pipelined plane-streaming stencil for sm_100a (a2, and a3's fused Arnoldi).
//
// Work decomposition. A "row tile" is BX x BY rows of the extended grid: (x, y) points of
// one RHS in 3D (YC = true), or 32 x-points of 8 right-hand sides in 2D (YC = false; rows
// are uncoupled RHS and the plane is one x-row). A work item is one row tile over one
// z-chunk of zlen planes. The grid is one resident wave: `groups` x `cpg` CTAs, a group
// being one RHS (3D) or one 8-RHS row group (2D); a group's items, ordered (z-chunk, tile)
// with the tile fastest, are dealt round-robin to its CTAs, so co-resident CTAs sweep
// neighbouring tiles at the same depth and their halos meet in L2 (the host picks the chunk
// count that minimises waves x (planes + 2 halo planes) per item). Each item streams the
// planes z0-1 .. z1 through an S-stage shared-memory ring filled by asynchronous copies
// (cp.async / LDGSTS; zero-fill implements the Dirichlet ghosts, R7): the tile plus its
// one-point halo for every halo'd operand, the model m, the per-plane z coefficients of the
// 1D tables and, per mode, the own-point operands; S-3 planes are in flight while plane z
// is computed. In 2D every warp owns its row of each stage and synchronises with the warp
// barrier only — no CTA-wide barrier on the streaming path. PML enters only through the
// 1D tables (D4-D6).
//
// MODE 0: y = s H x              (s = lazy normalisation of x, per RHS)
// MODE 1: y = b - H x, ||y||     (starts a Krylov cycle: beta, v0 scale, g, kact)
// MODE 2: w = s H x and h_i = <V_i, w>, i < NV (fused CGS projections, fp64 sums) — FGMRES
// MODE 3/4: fused Arnoldi step NV of unpreconditioned GMRES (lazy normalisation; 4 = last):
//           NV = 0: Y = H V_0,                          dots <V_0, Y>
//           NV > 0: V_NV = s_{NV-1} W - sum_{i<NV} h_{i,NV-1} s_i V_i formed on the fly
//                   (halo included) from the raw W = Y_{NV-1} and V_0..V_{NV-1};
//                   writes V_NV and Y = H V_NV; dots <V_i, Y>, i <= NV, and ||V_NV||^2.
//         The last CTA per RHS finalises column NV-1 (h_{NV,NV-1} = ||V_NV||, Givens,
//         breakdown guard) and stores column NV: h_{i,NV} = s_i s_NV <V_i, Y>.
#pragma once
#include <cuda.h>   // CUtensorMap (the map is encoded on the host through the driver entry point)
#include "kernels.cuh"

// ---- TMA + mbarrier (3D halo'd tiles): one elected thread issues cp.async.bulk.tensor per
// operand and stage; out-of-bounds box elements are zero-filled = the Dirichlet ghosts (R7).
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load4(unsigned dst, const CUtensorMap* map, unsigned bar, int c0, int c1, int c2,
                                          int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];\n" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load3(unsigned dst, const CUtensorMap* map, unsigned bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load2(unsigned dst, const CUtensorMap* map, unsigned bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }

template <int B> __device__ __forceinline__ void cpa(unsigned s, const void* gmem, bool pred) {
  const int sz = pred ? B : 0;
  if constexpr (B == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(s), "l"(gmem), "n"(B), "r"(sz) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N> __device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
// wait until at most n groups are pending (n is block-uniform; wait_group needs an immediate)
__device__ __forceinline__ void cpa_wait_n(int n) {
  switch (n) {
    case 0: cpa_wait<0>(); break;   case 1: cpa_wait<1>(); break;   case 2: cpa_wait<2>(); break;
    case 3: cpa_wait<3>(); break;   case 4: cpa_wait<4>(); break;   case 5: cpa_wait<5>(); break;
    case 6: cpa_wait<6>(); break;   case 7: cpa_wait<7>(); break;   case 8: cpa_wait<8>(); break;
    case 9: cpa_wait<9>(); break;   case 10: cpa_wait<10>(); break; default: cpa_wait<11>(); break;
  }
}

// 3D tiles couple the rows (y) of a CTA: block barrier. 2D rows are independent right-hand
// sides and each warp owns its row of every ring stage: warp barrier only.
template <bool YC> __device__ __forceinline__ void csync() {
  if constexpr (YC) __syncthreads(); else __syncwarp();
}

template <typename R> struct PlaneArgs {
  Geo<R> g;
  const cx<R>* x;          // halo'd input: x (MODE 0-2); V_0 (MODE 3, NV = 0) or raw W (MODE 3, NV > 0)
  cx<R>* y;                // output
  const cx<R>* b;          // MODE 1
  VPtrs<R> V;              // MODE 2: own-point V_0..V_{NV-1}; MODE 3: halo'd V_0..V_{NV-1}
  cx<R>* vout;             // MODE 3 (NV > 0): the formed V_NV is written here
  const double* xscale;    // MODE 0/2: per-RHS lazy scale of x (stride sstride) or null
  int sstride;
  const int* active;       // compact list of the active RHS (null: all); one group each
  const int* kact;         // skip RHS r if jskip >= kact[r] (null = never)
  int jskip;
  int jstep;               // Hessenberg column written (MODE 2, 3)
  int nrhs, ntx, nty;      // row tiles: ntx x nty per group (nty = 1 in 2D)
  int by;                  // tile rows (BY of the launched kernel; host bookkeeping)
  int cpg;                 // CTAs per group
  int nzc, zlen;           // z-chunks per tile and their length
  int S;                   // ring stages (>= 4; split-ring fused steps: raw stages D >= 2)
  int nf;                  // split-ring fused steps: formed slots (3: two barriers per plane, 4: one)
  int prev;                // single ring: plane z-1 from registers (S-2 planes in flight)
  int wlast;               // MODE 4 (NV > 0): store V_NV (0: not stored — the solution update reforms
                           // it from W and V_0..V_{NV-1} with the coefficients the epilogue saves)
  int ctared;              // reduction tail: one slot per CTA, summed by the last CTA (0: per warp)
  int cont;                // fused steps with TMA-only stages: one ring across the CTA's items
                           // (the next item's planes are in flight while this one finishes)
  int tma;                 // TMA stages (tm[0] = x / W, tm[1 + i] = V_i halo'd tiles; tmm = m, tmz = z
                           // coefficients) instead of per-thread cp.async
  CUtensorMap tm[HELM_KMAX + 1];
  CUtensorMap tmm, tmz;
  int tmq;                 // with tma: m and the z coefficients by TMA too (else per-thread cp.async)
  KCtx ctx;
  RedBuf rb;
};

template <typename R, int BX, int BY, int NX, int NP, bool YC, bool MREG = false, bool MH = false>
struct PlaneSmem {
  static constexpr int YH = YC ? 1 : 0;              // y-halo rows (3D only)
  // TMA boxes must start 16-B aligned along x (measured on B200: an unaligned start faults
  // with an illegal instruction, scripts/tma_probe.cu), so the tile's first interior column
  // sits XO = 16 B / element into the row: complex128 1, complex64 2 (one unused column)
  static constexpr int XO = (int)(16 / sizeof(cx<R>));
  static constexpr int XP = BX + 2 * XO;              // shared row pitch (elements)
  static constexpr int XE = (BY + 2 * YH) * XP;       // halo tile elements
  // tile stride in elements, padded to 128 B (TMA destinations must be 128-B aligned)
  static constexpr int XS = (int)(((XE * sizeof(cx<R>) + 127) / 128 * 128) / sizeof(cx<R>));
  static constexpr int PE = BY * BX;                 // own-point elements
  static constexpr size_t x_off = 0;
  // m is staged in the ring, except for the complex128 five-tile stages (the last Arnoldi
  // steps), where it is register-prefetched two planes ahead so that the stage fits two
  // CTAs per SM (measured: 3.3 -> 4.1 TB/s there; smaller stages are faster with m staged)
  // (MREG: m always register-prefetched — the split-ring fused steps below; MH: the OPT
  // stencils' mass distribution needs m at the 27 neighbours, so m is staged as a halo'd tile,
  // 16-B aligned box start XOm = 16 B / real before the interior like the complex tiles)
  static constexpr bool MR = !MREG && (MH || sizeof(cx<R>) != 16 || NX < 5);
  static constexpr int XOm = (int)(16 / sizeof(R));
  static constexpr int XPm = BX + 2 * XOm;
  static constexpr int MEm = (BY + 2 * YH) * XPm;
  static constexpr size_t m_bytes = MH ? ((size_t)MEm * sizeof(R) + 127) / 128 * 128 : (size_t)PE * sizeof(R);
  static constexpr size_t m_off = (size_t)NX * XS * sizeof(cx<R>);
  static constexpr size_t p_off = m_off + (MR ? m_bytes : 0);
  static constexpr size_t z_off = p_off + (size_t)NP * PE * sizeof(cx<R>);
  static constexpr int ZR = YC ? 1 : BY;               // z-coefficient rows (2D: one per warp)
  static constexpr size_t stage_bytes = (z_off + ZR * 4 * sizeof(cx<R>) + 127) / 128 * 128;
};

// Split-ring fused Arnoldi steps (MODE 3/4, NV > 0, TMA fills): the raw operands of a plane
// (halo'd tiles of W and V_0..V_{NV-1}) live in a D-stage TMA ring only until v_NV is formed
// from them; the formed halo'd tile (and the plane's z coefficients) go to one of NF = 4
// small "formed" slots that the stencil reads for planes z-1, z, z+1, and each thread keeps
// the own points of V_0..V_{NV-1} (the projection operands of plane z) in registers. A raw
// stage is refilled right after its plane is formed, so D-1 planes stay in flight instead of
// S-3 with full-size stages (the ncu capture of the old design: 1 plane in flight per CTA,
// 12 warps/SM, DRAM 44-51 % busy at level 1), and one CTA barrier per plane suffices.
template <typename R, int BX, int BY, bool YC> struct FormSlot {
  using SM1 = PlaneSmem<R, BX, BY, 1, 0, YC, true>;
  static constexpr size_t z_off = (size_t)SM1::XS * sizeof(cx<R>);
  static constexpr size_t bytes = (z_off + 4 * sizeof(cx<R>) + 127) / 128 * 128;
};

// MODE 4 = MODE 3 for the LAST step of a cycle: Y = H V_NV is not stored, and ||Y||^2 is
// reduced too, so that h_{NV+1,NV} = (s_NV^2 ||Y||^2 - sum_i |h_{i,NV}|^2)^{1/2}
// (Pythagoras on the orthonormal basis) finalises the last column without another pass
// over the data. V_{NV+1} itself is never needed; this h only enters the last Givens
// rotation (and the unused residual estimate), where its rounding is negligible.
template <int MODE, int NV> struct PlaneShape {
  static constexpr int NX = MODE >= 3 ? NV + 1 : 1;                       // halo'd tiles
  static constexpr int NP = MODE == 1 ? 1 : (MODE == 2 ? NV : 0);         // own-point operands
  static constexpr int NVR = MODE == 1 ? 1 : (MODE == 2 ? NV : (MODE >= 3 ? NV + 3 : 1));
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
  // four slots per lane per round, all loads issued before the adds (the sum over a lane's
  // slots was a chain of dependent L2 round trips: several us per launch at small batches);
  // the summation order is fixed by the slot index, so results stay bitwise reproducible
  int sl = lane;
  for (; sl + 96 < nslots; sl += 128) {
    double2 t[4][NV];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int k = 0; k < NV; ++k) t[u][k] = __ldcg(part + (size_t)(sl + 32 * u) * NV + k);
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        tot[k].x += t[u][k].x;
        tot[k].y += t[u][k].y;
      }
  }
  for (; sl < nslots; sl += 32) {
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

// Deterministic CTA-level reduction into per-RHS slots (3D plane kernel): the CTA's warps
// are summed in smem (fixed warp order) into ONE slot per CTA; the CTA that brings the ticket
// to `nslots` sums all slots with every thread (strided, four independent loads in flight per
// thread, then a fixed shuffle / warp tree). Versus one slot per warp summed by one warp
// (warp_slot_reduce) this is 4x fewer slots and 4x the readers: the tail of a launch is one
// or two L2 round trips instead of nslots/128 (measured: ~5 us per launch at 2,400 slots).
// `scratch` is shared memory free for reuse (the ring, after the last item). Returns true in
// every thread of the last CTA (false elsewhere); the totals tot[] are valid in thread 0.
template <int NV, int NT>
__device__ __forceinline__ bool cta_slot_reduce(double2 (&v)[NV], double2* part, unsigned* ticket, int slot, int nslots,
                                                double2 (&tot)[NV], double2* scratch) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned* flag = reinterpret_cast<unsigned*>(scratch + NW * NV);
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v[k].x += __shfl_xor_sync(0xffffffffu, v[k].x, o);
      v[k].y += __shfl_xor_sync(0xffffffffu, v[k].y, o);
    }
  __syncthreads();   // every thread is done with the ring that scratch aliases
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) scratch[warp * NV + k] = v[k];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double2 t = scratch[k];
      for (int w = 1; w < NW; ++w) { t.x += scratch[w * NV + k].x; t.y += scratch[w * NV + k].y; }
      part[(size_t)slot * NV + k] = t;
    }
    __threadfence();
    *flag = atomicAdd(ticket, 1u) == (unsigned)(nslots - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (!*flag) return false;
  __threadfence();
  double2 t[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) t[k] = make_double2(0.0, 0.0);
  int sl = threadIdx.x;
  for (; sl + 3 * NT < nslots; sl += 4 * NT) {
    double2 u[4][NV];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int k = 0; k < NV; ++k) u[q][k] = __ldcg(part + (size_t)(sl + q * NT) * NV + k);
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int k = 0; k < NV; ++k) { t[k].x += u[q][k].x; t[k].y += u[q][k].y; }
  }
  for (; sl < nslots; sl += NT)
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const double2 u = __ldcg(part + (size_t)sl * NV + k);
      t[k].x += u.x;
      t[k].y += u.y;
    }
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      t[k].x += __shfl_xor_sync(0xffffffffu, t[k].x, o);
      t[k].y += __shfl_xor_sync(0xffffffffu, t[k].y, o);
    }
  __syncthreads();   // thread 0's reads of the first scratch use are done
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) scratch[warp * NV + k] = t[k];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      tot[k] = scratch[k];
      for (int w = 1; w < NW; ++w) { tot[k].x += scratch[w * NV + k].x; tot[k].y += scratch[w * NV + k].y; }
    }
    *ticket = 0u;
  }
  return true;
}

// Per-RHS epilogue of the stencil modes, run by one lane of the last-arriving warp with the
// reduced totals: MODE 1 starts a Krylov cycle (beta = ||r||); MODE 2 stores projection
// column jstep; MODE 3/4 finalise column NV-1 with h_{NV,NV-1} = ||V_NV|| (D14 guard), store
// column NV and, for the last step, close it by Pythagoras.
template <int MODE, int NV, int NVR>
__device__ inline void plane_epilogue(const KCtx& ctx, int r, int jstep, const double2 (&tot)[NVR]) {
  const int K1 = HELM_KMAX + 1;
  constexpr bool LAST = MODE == 4;
  if constexpr (MODE == 1) {
    start_cycle(ctx, r, sqrt(tot[0].x));
  } else if constexpr (MODE == 2) {
    const double* scl = ctx.scale + r * K1;
    double2* H = ctx.H + (long long)r * K1 * HELM_KMAX;
    for (int i = 0; i < NV; ++i) H[hidx(i, jstep)] = make_double2(tot[i].x * scl[i], tot[i].y * scl[i]);
  } else if constexpr (MODE >= 3) {
    if constexpr (LAST && NV > 0) {
      // the forming coefficients of V_NV (column NV-1 is still unrotated here): the solution
      // update reforms V_NV from W and V_0..V_{NV-1} when this step does not store it
      const double* s = ctx.scale + r * K1;
      const double2* H = ctx.H + (long long)r * K1 * HELM_KMAX;
      double2* fc = ctx.fc + r * K1;
      for (int i = 0; i < NV; ++i) {
        const double2 h = H[hidx(i, NV - 1)];
        fc[i] = make_double2(-h.x * s[i], -h.y * s[i]);
      }
      fc[NV] = make_double2(s[NV - 1], 0.0);
    }
    // the lazy scales s_0..s_{NV-1} are loaded before finalize_column (which only writes
    // s_NV = 1/||V_NV||, or 0 on breakdown, i.e. when it leaves kact = NV): no dependent reload
    const double* scl = ctx.scale + r * K1;
    double sv[NV + 1];
#pragma unroll
    for (int i = 0; i < NV; ++i) sv[i] = scl[i];
    int kact = HELM_KMAX;
    if constexpr (NV > 0) {
      const double hn = sqrt(tot[NV + 1].x);
      kact = finalize_column(ctx, r, NV - 1, hn);
      sv[NV] = kact == NV ? 0.0 : 1.0 / hn;
    } else {
      sv[0] = scl[0];
      if constexpr (LAST) kact = ctx.kact[r];
    }
    const double sj = sv[NV];
    double2* H = ctx.H + (long long)r * K1 * HELM_KMAX;
    double hh = 0.0;
#pragma unroll
    for (int i = 0; i <= NV; ++i) {
      const double f = sv[i] * sj;
      const double2 h = make_double2(tot[i].x * f, tot[i].y * f);
      H[hidx(i, NV)] = h;
      hh += cabs2(h);
    }
    if constexpr (LAST) {
      if (NV < kact) {          // column NV is live (no breakdown above)
        const double w2 = sj * sj * tot[NV + 2].x;
        finalize_column(ctx, r, NV, sqrt(fmax(w2 - hh, 0.0)));
      }
    }
  }
}

// The launch's scalar epilogue runs in ONE thread and is a chain of dependent accesses to the
// RHS's Krylov state (Givens rotations, back substitution: ~1 us per rotation from L2,
// measured at cfg3). KStage: warp 0 of the last CTA copies that state into shared memory
// (independent loads, one round trip), lane 0 runs the epilogue on the copy through a KCtx
// view (generic pointers into shared memory, RHS index 0), and the warp writes it back.
struct KStage {
  static constexpr int K1 = HELM_KMAX + 1;
  // double2 units: H, sn, g, y, fc, then the reals scale, cs, beta and the int kact
  static constexpr int oH = 0, oSn = oH + K1 * HELM_KMAX, oG = oSn + HELM_KMAX, oY = oG + K1, oFc = oY + HELM_KMAX,
                       oReal = oFc + K1;
  static constexpr int nReal = K1 + HELM_KMAX + 1;   // scale, cs, beta (doubles)
  static constexpr int bytes = oReal * 16 + nReal * 8 + 16;
  __device__ static KCtx view(unsigned char* base, int k) {
    double2* d2 = reinterpret_cast<double2*>(base);
    double* d1 = reinterpret_cast<double*>(d2 + oReal);
    KCtx s{};
    s.H = d2 + oH; s.sn = d2 + oSn; s.g = d2 + oG; s.y = d2 + oY; s.fc = d2 + oFc;
    s.scale = d1; s.cs = d1 + K1; s.beta = d1 + K1 + HELM_KMAX;
    s.kact = reinterpret_cast<int*>(d1 + nReal);
    s.k = k;
    return s;
  }
  template <bool IN, typename T> __device__ static void cp(T* g, T* sm, int n, int lane) {
    for (int i = lane; i < n; i += 32) {
      if (IN) sm[i] = g[i];
      else g[i] = sm[i];
    }
  }
  template <bool IN> __device__ static void copy(const KCtx& g, int r, const KCtx& s, int lane) {
    cp<IN>(g.H + (long long)r * K1 * HELM_KMAX, s.H, K1 * HELM_KMAX, lane);
    cp<IN>(g.sn + r * HELM_KMAX, s.sn, HELM_KMAX, lane);
    cp<IN>(g.g + r * K1, s.g, K1, lane);
    cp<IN>(g.y + r * HELM_KMAX, s.y, HELM_KMAX, lane);
    cp<IN>(g.fc + r * K1, s.fc, K1, lane);
    cp<IN>(g.scale + r * K1, s.scale, K1, lane);
    cp<IN>(g.cs + r * HELM_KMAX, s.cs, HELM_KMAX, lane);
    cp<IN>(g.beta + r, s.beta, 1, lane);
    cp<IN>(g.kact + r, s.kact, 1, lane);
  }
};

// plane_epilogue on the shared-memory copy of RHS r's Krylov state; called by warp 0 (all
// lanes) of the last CTA, tot[] valid in lane 0; `sm` = KStage::bytes of free shared memory.
template <int MODE, int NV, int NVR>
__device__ __forceinline__ void plane_epilogue_staged(const KCtx& ctx, int r, int jstep, const double2 (&tot)[NVR],
                                                      unsigned char* sm) {
  const int lane = threadIdx.x & 31;
  const KCtx s = KStage::view(sm, ctx.k);
  KStage::copy<true>(ctx, r, s, lane);
  __syncwarp();
  if (lane == 0) plane_epilogue<MODE, NV>(s, 0, jstep, tot);
  __syncwarp();
  KStage::copy<false>(ctx, r, s, lane);
}

// DESIGN R35 (3D "compact 27-pt", P:204 [60]) at one point: L u + omega^2 M (m u) over the
// 27 neighbours of the halo'd tiles of planes z-1, z, z+1 (X*, complex; M*, the model), from
// the point's 1D table entries t_a = (lo, dg, up) (ghost entries already zero, R7) and the
// constant product-form weights (kernels.cuh optw).
// H^H = L^H + omega^2 diag(m) M (M real symmetric): with adj the mass term is m(centre) times
// the M-average of u (the tables are already H^H's, D6).
template <typename R>
__device__ __forceinline__ cx<R> opt27(const cx<R>* const (&X)[3], const R* const (&Mh)[3], int c, int cm, int XP,
                                       int XPm, const cx<R> (&tx)[3], const cx<R> (&ty)[3], const cx<R> (&tz)[3],
                                       R w2, bool adj) {
  using C = cx<R>;
  constexpr R G[3] = {(R)optw::G27_0, (R)optw::G27_1, (R)optw::G27_2};
  constexpr R MU[4] = {(R)optw::MU27_0, (R)optw::MU27_1, (R)optw::MU27_2, (R)optw::MU27_3};
  C acc = mkc((R)0, (R)0), ms = mkc((R)0, (R)0);
#pragma unroll
  for (int iz = 0; iz < 3; ++iz)
#pragma unroll
    for (int iy = 0; iy < 3; ++iy)
#pragma unroll
      for (int ix = 0; ix < 3; ++ix) {
        const int nx_ = ix != 1, ny_ = iy != 1, nz_ = iz != 1;
        const C u = X[iz][c + (iy - 1) * XP + (ix - 1)];
        // coefficient: tx[ix] G(dy, dz) + ty[iy] G(dx, dz) + tz[iz] G(dx, dy)
        const R gx = G[ny_ + nz_], gy = G[nx_ + nz_], gz = G[nx_ + ny_];
        const C cf = mkc(tx[ix].x * gx + ty[iy].x * gy + tz[iz].x * gz, tx[ix].y * gx + ty[iy].y * gy + tz[iz].y * gz);
        acc = cfma(cf, u, acc);
        const R mu = MU[nx_ + ny_ + nz_];
        if (mu != (R)0) ms = cfma(mkc(adj ? mu : mu * Mh[iz][cm + (iy - 1) * XPm + (ix - 1)], (R)0), u, ms);
      }
  const R wm = adj ? w2 * Mh[1][cm] : w2;
  return mkc(acc.x + wm * ms.x, acc.y + wm * ms.y);
}

template <typename R, int BX, int BY, int PY, int MODE, int NV, bool YC, bool SPLIT, int ST>
__device__ __forceinline__ void plane_body(const PlaneArgs<R>& a) {
  pdl_wait();
  pdl_trigger();
  using C = cx<R>;
  using Sh = PlaneShape<MODE, NV>;
  constexpr int NX = Sh::NX, NP = Sh::NP, NVR = Sh::NVR;
  using SM = PlaneSmem<R, BX, BY, NX, NP, YC, SPLIT, ST == 1>;
  using FS = FormSlot<R, BX, BY, YC>;
  static_assert(!SPLIT || (MODE >= 3 && NV > 0 && YC), "split ring: fused GMRES steps that form v_NV (3D)");
  static_assert(!(SPLIT && ST == 1), "the OPT stencil runs on the single ring");
  constexpr int YH = SM::YH;
  constexpr int NT = BX * BY / PY;
  constexpr int RS = BY / PY;          // row stride between a thread's rows
  constexpr int XP = SM::XP, XO = SM::XO;   // shared row pitch, first interior column
  constexpr bool FORM = MODE >= 3 && NV > 0;
  constexpr bool LAST = MODE == 4;
  static_assert(YC || PY == 1, "2D (rows = RHS) uses one row per thread");
  static_assert(BX == 32, "one warp per tile row");
  extern __shared__ __align__(128) unsigned char smem[];

  const Geo<R>& g = a.g;
  const int S = a.S;
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const int tx = threadIdx.x % BX, ty0 = threadIdx.x / BX;
  const int grp = blockIdx.x / a.cpg, cig = blockIdx.x % a.cpg;
  const long long N = g.N;
  const long long plane = YC ? (long long)nx * ny : (long long)nx;
  const C zero = mkc((R)0, (R)0);

  // ---- this CTA's RHS: entry grp of the compact active list
  static_assert(YC, "2D grids use the register march (march2d.cuh)");
  int rhs[PY];
  const bool ract = true;
  R sc = (R)1;           // lazy scale of x for this RHS (MODE 0 / 2)
  {
    const int r = a.active ? a.active[grp] : grp;
    if (a.kact && a.jskip >= a.kact[r]) return;
#pragma unroll
    for (int k = 0; k < PY; ++k) rhs[k] = r;
  }
  if ((MODE == 0 || MODE == 2) && a.xscale && ract) sc = (R)a.xscale[(long long)rhs[0] * a.sstride];
  const OpTab<R> T = op_tab(g, rhs[0]);

  // ---- MODE 3 forming coefficients of this thread's RHS: V_NV = cw W + sum_i cv_i V_i
  R cw = (R)1;
  C cv[FORM ? NV : 1];
  if constexpr (FORM) {
    const int r = rhs[0];
    const double* s = a.ctx.scale + (long long)r * (HELM_KMAX + 1);
    const double2* H = a.ctx.H + (long long)r * (HELM_KMAX + 1) * HELM_KMAX;
    cw = (R)s[NV - 1];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const double2 h = H[hidx(i, NV - 1)];
      cv[i] = mkc((R)(-h.x * s[i]), (R)(-h.y * s[i]));
    }
  }

  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem);
  // TMA: one mbarrier per ring stage, after the stages (stage addresses stay 128-B aligned)
  const unsigned mbase = sbase + (unsigned)(S * SM::stage_bytes + (SPLIT ? a.nf * FS::bytes : 0));
  const bool tma = a.tma != 0;
  if (tma) {
    if (threadIdx.x == 0) {
      for (int s2 = 0; s2 < S; ++s2) mbar_init(mbase + 8 * s2, 1);
      fence_mbar_init();
    }
    __syncthreads();
  }
  unsigned pbits = 0;      // parity of the next TMA fill of each stage
  // per-thread cp.async groups: everything without TMA; with TMA only MODE 1/2's own points
  const bool tmq = tma && a.tmq != 0;
  const bool cpa_on = !tmq || MODE == 1 || MODE == 2;
  const int zrow0 = (g.rop ? g.rop[rhs[0]] : 0) * nz;   // this RHS's rows of the z table
  double2 acc[NVR];
#pragma unroll
  for (int k = 0; k < NVR; ++k) acc[k] = make_double2(0.0, 0.0);
  double nrm = 0.0, ynrm = 0.0;

  // work items of this group: (z-chunk, tile), tile fastest, dealt round-robin to the
  // group's CTAs so that co-resident CTAs sweep neighbouring tiles at the same z (their
  // halos meet in L2)
  const int ntile = a.ntx * a.nty;
  const int nitems = ntile * a.nzc;

  // TMA fill of stage `stg` with plane z of tile `tile`: one elected thread issues the boxes
  // (halo'd tiles, m, the z row); every thread flips the stage's expected parity
  auto tma_fill = [&](int tile, int z, int stg) {
    if (threadIdx.x == 0) {
      const int txb = tile % a.ntx, tyb = tile / a.ntx;
      const unsigned st = sbase + (unsigned)(stg * SM::stage_bytes);
      fence_proxy_async();   // the stage's previous contents were read / formed by the generic proxy
      const unsigned bar = mbase + 8 * stg;
      // full boxes (OOB zero-filled): the halo'd tiles, m's own points, the z row
      mbar_expect_tx(bar, (unsigned)(NX * SM::XE * sizeof(C) +
                                     (tmq ? (SM::MR ? (ST == 1 ? SM::MEm : SM::PE) * sizeof(R) : 0) + 4 * sizeof(C)
                                          : 0)));
      constexpr int CR = (int)(sizeof(C) / 8);   // tensor element = one 8-byte word
#pragma unroll
      for (int t = 0; t < NX; ++t)
        tma_load4(st + (unsigned)(t * SM::XS * sizeof(C)), &a.tm[t], bar, CR * (txb * BX - XO), tyb * BY - YH, z,
                  rhs[0]);
      if (tmq) {
        if constexpr (ST == 1) tma_load3(st + (unsigned)SM::m_off, &a.tmm, bar, txb * BX - SM::XOm, tyb * BY - 1, z);
        else if constexpr (SM::MR) tma_load3(st + (unsigned)SM::m_off, &a.tmm, bar, txb * BX, tyb * BY, z);
        tma_load2(st + (unsigned)SM::z_off, &a.tmz, bar, 0, zrow0 + z);
      }
    }
    pbits ^= 1u << stg;
  };

  // Continuous ring (fused Arnoldi steps whose stages are filled by TMA alone): the CTA's
  // items form ONE stream of planes (z0-1 .. z1 of each item in turn) through the ring, so
  // the first planes of the next item are already in flight while this item's last planes
  // are computed (no ring refill bubble per item; measured at cfg4 level 1: 9 items per CTA).
  // The loader cursor (item, plane, stage) advances in the order the stages are freed.
  constexpr bool CONT_OK = MODE >= 3 && !SPLIT && ST == 0;
  const bool cont = CONT_OK && tma && tmq && a.prev != 0 && a.cont != 0;
  // (the item's tile, first plane and plane count are derived once per item: integer division
  // per plane in every thread cost 15 % more instructions, measured)
  int l_it = cig, l_q = 0, l_stg = 0, c_stg = 0, l_tile = 0, l_z = 0, l_nq = 0;
  auto loader_item = [&]() {
    if (l_it < nitems) {
      const int zc = l_it / ntile;
      l_tile = l_it - zc * ntile;
      l_z = zc * a.zlen - 1;
      l_nq = min(nz, zc * a.zlen + a.zlen) - zc * a.zlen + 2;
    }
  };
  auto loader_next = [&]() {
    if (l_it < nitems) {
      tma_fill(l_tile, l_z + l_q, l_stg);
      if (++l_q == l_nq) {
        l_q = 0;
        l_it += a.cpg;
        loader_item();
      }
    }
    l_stg = l_stg + 1 == S ? 0 : l_stg + 1;
  };
  if (cont) loader_item();
  if (cont && ract)
    for (int q = 0; q < S; ++q) loader_next();   // the first S planes of the stream

  for (int it = cig; it < (ract ? nitems : 0); it += a.cpg) {
    const int tile = it % ntile, zc = it / ntile;
    const int z0 = zc * a.zlen, z1 = min(nz, z0 + a.zlen);
    const int txb = tile % a.ntx, tyb = tile / a.ntx;
    const int ix = txb * BX + tx;

    int rowv[PY];
    bool rok[PY];
    long long gofs[PY];
#pragma unroll
    for (int k = 0; k < PY; ++k) {
      if constexpr (YC) {
        const int row = tyb * BY + ty0 + k * RS;
        rowv[k] = row;
        rok[k] = row < ny && ix < nx;
        gofs[k] = (long long)rhs[0] * N + (long long)row * nx + ix;
      } else {
        rowv[k] = 0;
        rok[k] = ract && ix < nx;
        gofs[k] = (long long)rhs[0] * N + ix;
      }
    }
    // load slots at fixed positions (static indexing keeps them in registers): own points
    // [0, PY), x-halo left [PY, 2PY), right [2PY, 3PY), y-halo low / high (YC); `lh` says
    // whether this thread issues the slot at all, `lp` whether it is in the grid (else the
    // copy zero-fills: the Dirichlet ghost).
    constexpr int NL = 3 * PY + (YC ? 2 : 0);
    long long lg[NL];
    unsigned ls[NL];
    bool lp[NL], lh[NL];
#pragma unroll
    for (int k = 0; k < PY; ++k) {
      const int sr = ty0 + k * RS + YH;
      lg[k] = gofs[k]; ls[k] = (unsigned)((sr * XP + tx + XO) * sizeof(C)); lp[k] = rok[k]; lh[k] = true;
      lg[PY + k] = gofs[k] - 1; ls[PY + k] = (unsigned)((sr * XP + XO - 1) * sizeof(C));
      lp[PY + k] = rok[k] && ix > 0; lh[PY + k] = tx == 0;
      lg[2 * PY + k] = gofs[k] + 1; ls[2 * PY + k] = (unsigned)((sr * XP + BX + XO) * sizeof(C));
      lp[2 * PY + k] = rok[k] && ix + 1 < nx; lh[2 * PY + k] = tx == BX - 1;
    }
    if constexpr (YC) {
      lg[3 * PY] = gofs[0] - nx; ls[3 * PY] = (unsigned)((tx + XO) * sizeof(C));
      lp[3 * PY] = ix < nx && rowv[0] - 1 >= 0 && rowv[0] - 1 < ny; lh[3 * PY] = ty0 == 0;
      lg[3 * PY + 1] = gofs[PY - 1] + nx; ls[3 * PY + 1] = (unsigned)(((BY + 1) * XP + tx + XO) * sizeof(C));
      lp[3 * PY + 1] = ix < nx && rowv[PY - 1] + 1 < ny; lh[3 * PY + 1] = ty0 + (PY - 1) * RS == BY - 1;
    }
    const long long mofs0 = YC ? (long long)rowv[0] * nx + ix : (long long)ix;

    const int nq = z1 - z0 + 2;
    auto load = [&](int q, int stg) {
      if (q < nq) {
        const int z = z0 - 1 + q;
        const bool zin = z >= 0 && z < nz;
        const unsigned st = sbase + (unsigned)(stg * SM::stage_bytes);
        const long long zo = (long long)z * plane;
        if (tma) {
          tma_fill(tile, z, stg);
        } else {
#pragma unroll
          for (int t = 0; t < NX; ++t) {
            const C* src = t == 0 ? a.x : a.V.p[t - 1];
#pragma unroll
            for (int i = 0; i < NL; ++i)
              if (lh[i]) {
                const bool p = lp[i] && zin;
                cpa<sizeof(C)>(st + (unsigned)(t * SM::XS * sizeof(C)) + ls[i], p ? src + lg[i] + zo : a.x, p);
              }
          }
        }
        if (cpa_on && q >= 1 && z < z1) {   // per-thread operands (none for MODE 0/3/4 with TMA)
          if (!tmq && (YC ? threadIdx.x : tx) < 3) {   // z coefficients of plane z: lo, dg, up (ghosts masked, R7)
            const int c3 = YC ? threadIdx.x : tx;
            const C* tz = c3 == 0 ? T.lo[2] : (c3 == 1 ? T.dg[2] : T.up[2]);
            const bool p = c3 == 1 || (c3 == 0 ? z > 0 : z < nz - 1);
            cpa<sizeof(C)>(st + (unsigned)(SM::z_off + ((YC ? 0 : ty0) * 4 + c3) * sizeof(C)), p ? tz + z : tz, p);
          }
#pragma unroll
          for (int k = 0; k < PY; ++k)
            if (rok[k]) {
              const int pr = (ty0 + k * RS) * BX + tx;
              if constexpr (SM::MR && ST == 0)
                if (!tmq)
                  cpa<sizeof(R)>(st + (unsigned)(SM::m_off + pr * sizeof(R)), g.m + (YC ? mofs0 + (long long)k * RS * nx : mofs0) + zo, true);
              if constexpr (MODE == 1) cpa<sizeof(C)>(st + (unsigned)(SM::p_off + pr * sizeof(C)), a.b + gofs[k] + zo, true);
              if constexpr (MODE == 2) {
#pragma unroll
                for (int v = 0; v < NV; ++v)
                  cpa<sizeof(C)>(st + (unsigned)(SM::p_off + (v * SM::PE + pr) * sizeof(C)), a.V.p[v] + gofs[k] + zo, true);
              }
            }
        }
      }
      if (cpa_on) cpa_commit();   // always commit (possibly empty) so group counting stays uniform
    };
    // MODE 3: turn the raw W tile of stage `q` into V_NV in place (halo included)
    auto form = [&](int stg) {
      if constexpr (FORM) {
        C* X = reinterpret_cast<C*>(smem + stg * SM::stage_bytes);
        auto f1 = [&](int e) {
          C v = cscale(X[e], cw);
#pragma unroll
          for (int i = 0; i < NV; ++i) v = cfma(cv[i], X[(i + 1) * SM::XS + e], v);
          X[e] = v;
        };
        if constexpr (YC) {
          for (int e = threadIdx.x; e < SM::XE; e += NT) f1(e);
        } else {
          const int rowe = ty0 * XP;
          f1(rowe + tx + XO);
          if (tx == 0) f1(rowe + XO - 1);
          if (tx == BX - 1) f1(rowe + BX + XO);
        }
      }
    };

    // per-thread operator coefficients along x (and y in 3D)
    const C lox = (ix > 0 && ix < nx) ? T.lo[0][ix] : zero;
    const C upx = (ix < nx - 1) ? T.up[0][ix] : zero;
    const C dgx = ix < nx ? T.dg[0][ix] : zero;
    C loy[PY], upy[PY], dgy[PY];
#pragma unroll
    for (int k = 0; k < PY; ++k) {
      if constexpr (YC) {
        const int iy = rowv[k];
        loy[k] = (iy > 0 && iy < ny) ? T.lo[1][iy] : zero;
        upy[k] = (iy < ny - 1) ? T.up[1][iy] : zero;
        dgy[k] = iy < ny ? T.dg[1][iy] : zero;
      } else {
        loy[k] = upy[k] = dgy[k] = zero;
      }
    }

    // model m of this thread's points: register-prefetched two planes ahead (complex128)
    R mr0[PY], mr1[PY], mr2[PY];
    auto ldm = [&](int zz, R (&dst)[PY]) {
#pragma unroll
      for (int k = 0; k < PY; ++k)
        dst[k] = (rok[k] && zz < z1) ? __ldg(g.m + (YC ? mofs0 + (long long)k * RS * nx : mofs0) + (long long)zz * plane)
                                     : (R)0;
    };
    // split ring: own points of V_0..V_{NV-1} of the plane being computed (vd) and of the
    // plane being formed (vn), captured from the raw stage before it is refilled
    constexpr int NVD = SPLIT ? NV : 1;
    C vd[PY][NVD], vn[PY][NVD];
    // single ring, STD2: plane z-1 enters only through the own-point z-neighbour term, so each
    // thread keeps it in registers (prevc) and its stage is refilled one plane earlier
    constexpr bool PREV_OK = !SPLIT && ST == 0;
    const bool PREV = PREV_OK && a.prev != 0;   // HELM_PREV=0: the round-1 ring (A/B)
    C prevc[PY];
    // plane z from the tiles of planes z-1, z, z+1 (X0, X1, X2; x/y halo in X1), m (Ms or
    // registers), the own-point operands (Ps) and the plane's z coefficients (Zt)
    auto compute = [&](int z, const C* X0, const C* X1, const C* X2, const R* Ms, const C* Ps, const C* Zt,
                       const R* Ms0 = nullptr, const R* Ms2 = nullptr) {
      const C lz = Zt[(YC ? 0 : ty0) * 4], dz = Zt[(YC ? 0 : ty0) * 4 + 1], uz = Zt[(YC ? 0 : ty0) * 4 + 2];
      const long long zo = (long long)z * plane;
#pragma unroll
      for (int k = 0; k < PY; ++k) {
        if (!rok[k]) continue;
        const int c = (ty0 + k * RS + YH) * XP + tx + XO;
        const int pr = (ty0 + k * RS) * BX + tx;
        const C cur = X1[c];
        C hx;
        if constexpr (ST == 1) {   // R35: the 27-point stencil with the mass distribution
          const int cm = (ty0 + k * RS + YH) * SM::XPm + tx + SM::XOm;
          const C* const Xs[3] = {X0, X1, X2};
          const R* const Mh[3] = {Ms0, Ms, Ms2};
          const C txa[3] = {lox, dgx, upx}, tya[3] = {loy[k], dgy[k], upy[k]}, tza[3] = {lz, dz, uz};
          hx = opt27<R>(Xs, Mh, c, cm, XP, SM::XPm, txa, tya, tza, T.w2, g.adj != 0);
        } else {
          const R wm = T.w2 * (SM::MR ? Ms[pr] : mr0[k]);
          // tree-shaped sum: four independent complex products, then two adds
          C t0 = cmul(mkc(dgx.x + dgy[k].x + dz.x + wm, dgx.y + dgy[k].y + dz.y), cur);
          C t1 = cfma(upx, X1[c + 1], cmul(lox, X1[c - 1]));
          C t2 = cfma(uz, X2[c], cmul(lz, PREV ? prevc[k] : X0[c]));
          if constexpr (YC) t0 = cfma(upy[k], X1[c + XP], cfma(loy[k], X1[c - XP], t0));
          hx = cadd(cadd(t0, t1), t2);
        }
        if constexpr (PREV_OK) prevc[k] = cur;   // plane z is the next plane's z-1
        C* yp = a.y + gofs[k] + zo;
        if constexpr (MODE == 0) {
          *yp = cscale(hx, sc);
        } else if constexpr (MODE == 1) {
          const C rv = csub(Ps[pr], hx);
          *yp = rv;
          nrm += (double)rv.x * rv.x + (double)rv.y * rv.y;
        } else if constexpr (MODE == 2) {
          const C w = cscale(hx, sc);
          *yp = w;
          const double2 wd = to_d(w);
#pragma unroll
          for (int v = 0; v < NV; ++v) acc[v] = cdot_acc(acc[v], to_d(Ps[v * SM::PE + pr]), wd);
        } else {
          const double2 hd = to_d(hx);
          if constexpr (LAST) ynrm += hd.x * hd.x + hd.y * hd.y;
          else *yp = hx;
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            if constexpr (SPLIT) acc[v] = cdot_acc(acc[v], to_d(vd[k][v]), hd);
            else acc[v] = cdot_acc(acc[v], to_d(X1[(v + 1) * SM::XS + c]), hd);
          }
          acc[NV] = cdot_acc(acc[NV], to_d(cur), hd);
          if constexpr (NV > 0) {
            if (!LAST || a.wlast) a.vout[gofs[k] + zo] = cur;
            nrm += (double)cur.x * cur.x + (double)cur.y * cur.y;
          }
        }
      }
      if constexpr (!SM::MR) {
#pragma unroll
        for (int k = 0; k < PY; ++k) { mr0[k] = mr1[k]; mr1[k] = mr2[k]; }
      }
    };

    if constexpr (SPLIT) {
      // ---- split ring (TMA tiles, m in registers): raw stage of plane q is q % S, formed
      // slot q % nf; plane q = z - z0 + 1
      const int NF = a.nf;
      const unsigned fb0 = (unsigned)(S * SM::stage_bytes);
      auto fslot = [&](int q) { return smem + fb0 + (unsigned)((q % NF) * FS::bytes); };
      auto form_split = [&](int q) {
        const int rs = q % S;
        const C* X = reinterpret_cast<const C*>(smem + rs * SM::stage_bytes);
        unsigned char* fp = fslot(q);
        C* F = reinterpret_cast<C*>(fp);
        for (int e = threadIdx.x; e < SM::XE; e += NT) {
          C v = cscale(X[e], cw);
#pragma unroll
          for (int i = 0; i < NV; ++i) v = cfma(cv[i], X[(i + 1) * SM::XS + e], v);
          F[e] = v;
        }
        if (threadIdx.x < 4)
          reinterpret_cast<C*>(fp + FS::z_off)[threadIdx.x] =
              reinterpret_cast<const C*>(smem + rs * SM::stage_bytes + SM::z_off)[threadIdx.x];
#pragma unroll
        for (int k = 0; k < PY; ++k) {
          const int c = (ty0 + k * RS + YH) * XP + tx + XO;
#pragma unroll
          for (int v = 0; v < NV; ++v) vn[k][v] = X[(v + 1) * SM::XS + c];
        }
      };
      auto wait_raw = [&](int q) {
        const int rs = q % S;
        mbar_wait(mbase + 8 * rs, ((pbits >> rs) & 1u) ^ 1u);
      };
      for (int q = 0; q < S; ++q) load(q, q);   // planes z0-1 .. z0+S-2 in flight
      ldm(z0, mr0);
      ldm(z0 + 1, mr1);
      for (int q = 0; q < 2; ++q) {             // form planes z0-1 and z0
        wait_raw(q);
        form_split(q);
        csync<YC>();
        load(q + S, q % S);
      }
#pragma unroll
      for (int k = 0; k < PY; ++k)
#pragma unroll
        for (int v = 0; v < NV; ++v) vd[k][v] = vn[k][v];
      for (int z = z0; z < z1; ++z) {
        const int q = z - z0 + 1, qn = q + 1;
        wait_raw(qn);
        if (NF == 3) csync<YC>();               // compute(z-1) is done with formed slot qn % 3
        form_split(qn);
        csync<YC>();                            // slot qn formed; raw stage qn consumed
        load(qn + S, qn % S);                   // S-1 planes in flight while plane z is computed
        ldm(z + 2, mr2);
        const unsigned char* f1 = fslot(q);
        compute(z, reinterpret_cast<const C*>(fslot(q - 1 + NF)), reinterpret_cast<const C*>(f1),
                reinterpret_cast<const C*>(fslot(qn)), nullptr, nullptr,
                reinterpret_cast<const C*>(f1 + FS::z_off));
#pragma unroll
        for (int k = 0; k < PY; ++k)
#pragma unroll
          for (int v = 0; v < NV; ++v) vd[k][v] = vn[k][v];
      }
    } else if (PREV) {
      // ---- single ring, plane z-1 in registers: the stage of plane q is q % S; at plane z the
      // stage of z-1 is free, so S-2 planes are in flight (the ncu stall profile of the fused
      // steps at cfg4 level 1 showed 20 % of warp time waiting for TMA stages with S-3 = 1)
      auto inc = [S](int x) { return x + 1 == S ? 0 : x + 1; };
      const int s_m1 = cont ? c_stg : 0;           // stage of plane z0-1
      if (!cont)
        for (int q = 0; q < S; ++q) load(q, q);    // planes z0-1 .. z0+S-2 (cont: already in flight)
      if constexpr (!SM::MR) { ldm(z0, mr0); ldm(z0 + 1, mr1); }
      if (cpa_on) cpa_wait_n(S - 1);               // plane z0-1 (this thread's copies)
      if (tma) mbar_wait(mbase + 8 * s_m1, ((pbits >> s_m1) & 1u) ^ 1u);
      csync<YC>();
      if constexpr (FORM) {
        form(s_m1);
        csync<YC>();
      }
      {
        const C* Xm = reinterpret_cast<const C*>(smem + s_m1 * SM::stage_bytes);
#pragma unroll
        for (int k = 0; k < PY; ++k) prevc[k] = rok[k] ? Xm[(ty0 + k * RS + YH) * XP + tx + XO] : zero;
      }
      int s_fr = s_m1, s_0 = inc(s_m1), s_p1 = inc(s_0);   // stages of planes z-1 (free), z, z+1
      for (int z = z0; z < z1; ++z) {
        const int q = z - z0 + 1;
        if (cpa_on) cpa_wait_n(S - 3);   // this thread's groups <= q+1 complete (committed: <= q+S-2)
        if (tma) {
          if (z == z0) mbar_wait(mbase + 8 * s_0, ((pbits >> s_0) & 1u) ^ 1u);
          mbar_wait(mbase + 8 * s_p1, ((pbits >> s_p1) & 1u) ^ 1u);
        }
        // forming needs no barrier before it: v_NV of plane z+1 goes into tile 0 of its own
        // (landed) stage, which no thread still in plane z-1 reads; the one barrier below both
        // publishes it and frees the stage of plane z-1 (every thread is past plane z-1)
        if constexpr (FORM) {
          if (z == z0) form(s_0);
          form(s_p1);
        }
        csync<YC>();
        if (cont) loader_next();         // the stream's next plane into the freed stage s_fr
        else load(q + S - 1, s_fr);      // S-2 planes in flight while plane z is computed
        const unsigned char* st1 = smem + s_0 * SM::stage_bytes;
        if constexpr (!SM::MR) ldm(z + 2, mr2);
        compute(z, nullptr, reinterpret_cast<const C*>(st1), reinterpret_cast<const C*>(smem + s_p1 * SM::stage_bytes),
                reinterpret_cast<const R*>(st1 + SM::m_off), reinterpret_cast<const C*>(st1 + SM::p_off),
                reinterpret_cast<const C*>(st1 + SM::z_off));
        s_fr = s_0;
        s_0 = s_p1;
        s_p1 = inc(s_p1);
      }
      if (cont) {
        // planes z1-1 and z1 (stages s_fr, s_0) are free once every thread is past compute(z1-1)
        csync<YC>();
        loader_next();
        loader_next();
        c_stg = s_p1;                    // the next item's plane z0'-1
      }
    } else {
      // ring stages are tracked incrementally (no division on the streaming path)
      auto inc = [S](int x) { return x + 1 == S ? 0 : x + 1; };
      int s_ld = 0;
      for (int q = 0; q < S - 1; ++q) { load(q, s_ld); s_ld = inc(s_ld); }
      int s_m1 = 0;             // stage of plane z-1
      if constexpr (!SM::MR) { ldm(z0, mr0); ldm(z0 + 1, mr1); }
      for (int z = z0; z < z1; ++z) {
        const int q = z - z0 + 1;
        if (cpa_on) cpa_wait_n(S - 4);   // this thread's groups <= q+1 complete (committed: <= q+S-3)
        if (tma) {                // ... and the TMA tiles of planes <= q+1 (stage s_m1 + 2)
          const int sw = inc(inc(s_m1));
          if (z == z0) {
            mbar_wait(mbase + 8 * s_m1, ((pbits >> s_m1) & 1u) ^ 1u);
            mbar_wait(mbase + 8 * inc(s_m1), ((pbits >> inc(s_m1)) & 1u) ^ 1u);
          }
          mbar_wait(mbase + 8 * sw, ((pbits >> sw) & 1u) ^ 1u);
        }
        csync<YC>();              // ... for every thread; stage (q-2)%S is free again
        load(q + S - 2, s_ld);    // S-3 planes in flight while plane z is computed
        s_ld = inc(s_ld);
        const int s_0 = inc(s_m1), s_p1 = inc(s_0);
        if constexpr (FORM) {
          if (z == z0) { form(s_m1); form(s_0); }
          form(s_p1);
          csync<YC>();
        }
        const unsigned char* st1 = smem + s_0 * SM::stage_bytes;
        if constexpr (!SM::MR) ldm(z + 2, mr2);
        compute(z, reinterpret_cast<const C*>(smem + s_m1 * SM::stage_bytes), reinterpret_cast<const C*>(st1),
                reinterpret_cast<const C*>(smem + s_p1 * SM::stage_bytes), reinterpret_cast<const R*>(st1 + SM::m_off),
                reinterpret_cast<const C*>(st1 + SM::p_off), reinterpret_cast<const C*>(st1 + SM::z_off),
                reinterpret_cast<const R*>(smem + s_m1 * SM::stage_bytes + SM::m_off),
                reinterpret_cast<const R*>(smem + s_p1 * SM::stage_bytes + SM::m_off));
        s_m1 = s_0;
      }
    }
    if (!cont) {
      cpa_wait<0>();
      csync<YC>();     // the next item's prologue reuses the ring
    }
  }

  if constexpr (MODE != 0) {
    if constexpr (MODE == 1) acc[0] = make_double2(nrm, 0.0);
    if constexpr (MODE >= 3) acc[NV + 1] = make_double2(nrm, 0.0);
    if constexpr (MODE >= 3) acc[NV + 2] = make_double2(ynrm, 0.0);
    // every thread of the CTA belongs to RHS rhs[0] -> one slot per CTA of the group
    // (a.ctared = 0: one slot per warp, summed by one warp — the round-2 tail, A/B)
    const int r = rhs[0];
    double2 tot[NVR];
    if (a.ctared) {
      // (the KStage copy sits 4 KB into the ring, clear of the reduction scratch)
      if (cta_slot_reduce<NVR, NT>(acc, a.rb.part + (size_t)grp * a.cpg * NVR, a.rb.ticket + r, cig, a.cpg, tot,
                                   reinterpret_cast<double2*>(smem)) &&
          threadIdx.x < 32)
        plane_epilogue_staged<MODE, NV>(a.ctx, r, a.jstep, tot, smem + 4096);
    } else {
      constexpr int WPB = NT / 32;
      const int slot = cig * WPB + (threadIdx.x >> 5);
      const int nslots = a.cpg * WPB;
      if (warp_slot_reduce<NVR>(acc, a.rb.part + (size_t)grp * nslots * NVR, a.rb.ticket + r, slot, nslots, tot)) {
        if ((threadIdx.x & 31) == 0) plane_epilogue<MODE, NV>(a.ctx, r, a.jstep, tot);
      }
    }
  }
}

// The plane kernel. k_plane_o2 is the same body compiled for two resident CTAs per SM
// (register cap 65536 / (2 NT)): the split-ring last step with one row per thread
// (HELM_SPLIT_PY=1). (An explicit minimum of one CTA in k_plane's bounds let ptxas take up to
// 255 registers: 128 -> 198 for the fused steps, measured — so k_plane keeps the bare bound.)
template <typename R, int BX, int BY, int PY, int MODE, int NV, bool YC, bool SPLIT = false, int ST = 0>
__global__ void __launch_bounds__(BX * BY / PY) k_plane(const __grid_constant__ PlaneArgs<R> a) {
  plane_body<R, BX, BY, PY, MODE, NV, YC, SPLIT, ST>(a);
}
template <typename R, int BX, int BY, int PY, int MODE, int NV, bool YC, bool SPLIT = false, int ST = 0>
__global__ void __launch_bounds__(BX * BY / PY, 2) k_plane_o2(const __grid_constant__ PlaneArgs<R> a) {
  plane_body<R, BX, BY, PY, MODE, NV, YC, SPLIT, ST>(a);
}
