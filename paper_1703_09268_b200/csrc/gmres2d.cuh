// gmres2d.cuh — per-RHS persistent GMRES(ko, ki) for the coarse levels of 2D problems
// (a4: the V-cycle smoothers and the coarsest solve of ML-GMRES, Alg. 1 P:260-270 with the
// fixed counts of R19-R20), sm_100a.
//
// On the coarse levels of a 2D batch (121 x 221 and 61 x 111 points per RHS for cfg2) every
// grid-wide kernel is short and its launch / ramp / grid-reduction floor dominates: a
// GMRES(3,5) there is 21 such launches. Here ONE CTA owns one active RHS and runs the whole
// restarted GMRES: cycle start (||b|| or r = b - H x), the ki fused Arnoldi steps (the same
// march_pass as k_march2d: form v_j on the fly, stencil, projections, norms; last column by
// Pythagoras), the Givens / least-squares epilogue, and the solution update — separated by
// block barriers, with fixed-order block reductions (warp shuffles, then one thread over the
// warp partials in warp order). Nothing but the RHS's own vectors is touched, so RHS run
// fully independently; the grid is the compact list of active RHS. Mathematically identical
// to the grid-wide sequence (same operations in a different summation order).
#pragma once
#include "march2d.cuh"

#define HELM_GMRES_CTA_KI 5     // largest inner dimension handled here (fused-step templates)
#define HELM_GMRES_WARPS 8

template <typename R> struct GmresArgs {
  Geo<R> g;
  const cx<R>* b;            // right-hand side (basis vector 0 of the first cycle when x0 = 0)
  cx<R>* x;                  // iterate (in/out; zeroed implicitly when x0zero)
  cx<R>* V[HELM_KMAX + 1];   // basis V[0..ki-1]; V[ki] and Wx: raw-product ping-pong
  cx<R>* Wx;
  const int* active;         // compact list of active RHS (nrhs entries)
  int nrhs;
  int ko, ki, x0zero;
  int nstrip, nzc, zlen, S;
  KCtx ctx;
};

// Fixed-order block reduction of NVR fp64 complex partials: warp shuffles, lane 0 -> smem,
// thread 0 sums the warps in order. The result is valid in thread 0 only.
template <int NVR>
__device__ __forceinline__ void block_reduce_fixed(double2 (&v)[NVR], double2* red /* [warps][NVR] */) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < NVR; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v[k].x += __shfl_xor_sync(0xffffffffu, v[k].x, o);
      v[k].y += __shfl_xor_sync(0xffffffffu, v[k].y, o);
    }
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NVR; ++k) red[w * NVR + k] = v[k];
  __syncthreads();
  if (threadIdx.x == 0)
#pragma unroll
    for (int k = 0; k < NVR; ++k) {
      double2 t = red[k];
      for (int i = 1; i < nw; ++i) t = make_double2(t.x + red[i * NVR + k].x, t.y + red[i * NVR + k].y);
      v[k] = t;
    }
}

template <typename R, int MODE, int NV>
__device__ __forceinline__ void gmres_step(const GmresArgs<R>& a, const OpTab<R>& T, const cx<R>* ztr, int r,
                                           const cx<R>* xin, cx<R>* yout, cx<R>* vout, const VPtrs<R>& Vp,
                                           unsigned char* ring, unsigned ring_s, double2* red) {
  using C = cx<R>;
  constexpr int NVR = NV + 3;
  R cw = (R)1;
  C cv[NV > 0 ? NV : 1];
  form_coeffs<R, NV>(a.ctx, r, cw, cv);
  double2 acc[NVR];
#pragma unroll
  for (int k = 0; k < NVR; ++k) acc[k] = make_double2(0.0, 0.0);
  double nrm = 0.0, ynrm = 0.0;
  march_pass<R, MODE, NV, NVR>(a.g, T, ztr, (long long)r * a.g.N, xin, nullptr, yout, vout, Vp.p, (R)1, cw, cv,
                               a.nstrip, a.nzc, a.zlen, threadIdx.x >> 5, blockDim.x >> 5, a.S, ring, ring_s,
                               acc, nrm, ynrm);
  acc[NV + 1] = make_double2(nrm, 0.0);
  acc[NV + 2] = make_double2(ynrm, 0.0);
  block_reduce_fixed<NVR>(acc, red);
  if (threadIdx.x == 0) plane_epilogue<MODE, NV>(a.ctx, r, NV, acc);
  __syncthreads();
}

template <typename R>
__global__ void __launch_bounds__(HELM_GMRES_WARPS * 32, 2)
k_gmres2d(const GmresArgs<R> a) {
  pdl_wait();
  pdl_trigger();
  using C = cx<R>;
  constexpr int K1 = HELM_KMAX + 1;
  constexpr int SBMAX = MarchShape<R, 3, HELM_GMRES_CTA_KI - 1>::stage_bytes;
  const Geo<R>& g = a.g;
  const int nz = g.nz;
  const int r = a.active ? a.active[blockIdx.x] : blockIdx.x;
  const long long N = g.N, rb0 = (long long)r * N;
  extern __shared__ __align__(16) unsigned char gsm[];
  C* zt = reinterpret_cast<C*>(gsm);
  for (int e = threadIdx.x; e < 3 * g.nop * nz; e += blockDim.x) zt[e] = g.zpk[e];
  const size_t zbytes = ((size_t)3 * g.nop * nz * sizeof(C) + 15) / 16 * 16;
  double2* red = reinterpret_cast<double2*>(gsm + zbytes);                       // [warps][KMAX+3]
  const size_t rbytes = (size_t)HELM_GMRES_WARPS * (HELM_KMAX + 3) * sizeof(double2);
  unsigned char* ring = gsm + zbytes + rbytes + (size_t)(threadIdx.x >> 5) * a.S * SBMAX;
  const unsigned ring_s = (unsigned)__cvta_generic_to_shared(ring);
  __syncthreads();
  const OpTab<R> T = op_tab(g, r);
  const C* ztr = zt + 3 * (long long)(g.rop ? g.rop[r] : 0) * nz;
  const KCtx& ctx = a.ctx;
  const int ki = a.ki;

  for (int cyc = 0; cyc < a.ko; ++cyc) {
    const bool first_zero = cyc == 0 && a.x0zero;
    // ---- cycle start: beta = ||r_0||, v_0 = r_0 / beta (lazy)
    const C* v0;
    {
      double2 acc[1] = {make_double2(0.0, 0.0)};
      if (first_zero) {
        const C* br = a.b + rb0;
        double s = 0.0;
        for (long long p = threadIdx.x; p < N; p += blockDim.x) {
          const C v = br[p];
          s += (double)v.x * v.x + (double)v.y * v.y;
        }
        acc[0].x = s;
        v0 = a.b;
      } else {
        double nrm = 0.0, ynrm = 0.0;
        const C cv0[1] = {mkc((R)0, (R)0)};
        march_pass<R, 1, 0, 1>(g, T, ztr, rb0, a.x, a.b, a.V[0], nullptr, nullptr, (R)1, (R)1, cv0, a.nstrip, a.nzc,
                               a.zlen, threadIdx.x >> 5, blockDim.x >> 5, a.S, ring, ring_s, acc, nrm, ynrm);
        acc[0] = make_double2(nrm, 0.0);
        v0 = a.V[0];
      }
      block_reduce_fixed<1>(acc, red);
      if (threadIdx.x == 0) start_cycle(ctx, r, sqrt(acc[0].x));
      __syncthreads();
    }
    // ---- ki fused Arnoldi steps (raw products ping-pong between V[ki] and Wx)
    VPtrs<R> Vp;
#pragma unroll
    for (int i = 0; i <= HELM_GMRES_CTA_KI; ++i) Vp.p[i] = i == 0 ? v0 : a.V[i];
    C* const wk = a.V[ki];
    for (int j = 0; j < ki; ++j) {
      if (j > 0 && j - 1 >= ctx.kact[r]) break;   // breakdown (D14) or zero RHS: cycle is over
      if (j == 0 && ctx.kact[r] == 0) break;
      const C* xin = j == 0 ? v0 : (((j - 1) & 1) ? a.Wx : wk);
      C* yout = (j & 1) ? a.Wx : wk;
      C* vout = j == 0 ? nullptr : a.V[j];
      const bool last = j == ki - 1;
      switch (j) {
        case 0: if (last) gmres_step<R, 4, 0>(a, T, ztr, r, xin, yout, vout, Vp, ring, ring_s, red);
                else gmres_step<R, 3, 0>(a, T, ztr, r, xin, yout, vout, Vp, ring, ring_s, red); break;
        case 1: if (last) gmres_step<R, 4, 1>(a, T, ztr, r, xin, yout, vout, Vp, ring, ring_s, red);
                else gmres_step<R, 3, 1>(a, T, ztr, r, xin, yout, vout, Vp, ring, ring_s, red); break;
        case 2: if (last) gmres_step<R, 4, 2>(a, T, ztr, r, xin, yout, vout, Vp, ring, ring_s, red);
                else gmres_step<R, 3, 2>(a, T, ztr, r, xin, yout, vout, Vp, ring, ring_s, red); break;
        case 3: if (last) gmres_step<R, 4, 3>(a, T, ztr, r, xin, yout, vout, Vp, ring, ring_s, red);
                else gmres_step<R, 3, 3>(a, T, ztr, r, xin, yout, vout, Vp, ring, ring_s, red); break;
        default: gmres_step<R, 4, 4>(a, T, ztr, r, xin, yout, vout, Vp, ring, ring_s, red); break;
      }
    }
    // ---- solution update x = (first ? 0 : x) + sum_{i < kact} y_i s_i V_i
    {
      const int k = ctx.kact[r];
      C yc[HELM_GMRES_CTA_KI];
      const double* sc = ctx.scale + r * K1;
#pragma unroll
      for (int i = 0; i < HELM_GMRES_CTA_KI; ++i) {
        const double2 yv = i < k ? ctx.y[r * HELM_KMAX + i] : make_double2(0.0, 0.0);
        const double s = i < k ? sc[i] : 0.0;
        yc[i] = mkc((R)(yv.x * s), (R)(yv.y * s));
      }
      C* xr = a.x + rb0;
      const C* vp[HELM_GMRES_CTA_KI];
#pragma unroll
      for (int i = 0; i < HELM_GMRES_CTA_KI; ++i) vp[i] = Vp.p[i] + rb0;
      for (long long p = threadIdx.x; p < N; p += blockDim.x) {
        C xv = first_zero ? mkc((R)0, (R)0) : xr[p];
#pragma unroll
        for (int i = 0; i < HELM_GMRES_CTA_KI; ++i)
          if (i < k) xv = cfma(yc[i], vp[i][p], xv);
        xr[p] = xv;
      }
      __syncthreads();
    }
  }
}
