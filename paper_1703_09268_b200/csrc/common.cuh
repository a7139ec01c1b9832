// common.cuh — complex arithmetic, per-RHS Krylov context and deterministic reductions
// shared by every kernel of libhelm (sm_100a). Nothing here is shared with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define HELM_KMAX 8          // largest inner Krylov dimension supported (k_i, k_si, k_ci)
#define HELM_RED_THREADS 256 // block size of the BLAS-1 / reduction kernels

template <typename R> struct cx_of;
template <> struct cx_of<float> { using t = float2; };
template <> struct cx_of<double> { using t = double2; };
template <typename R> using cx = typename cx_of<R>::t;

__host__ __device__ __forceinline__ float2 mkc(float a, float b) { return make_float2(a, b); }
__host__ __device__ __forceinline__ double2 mkc(double a, double b) { return make_double2(a, b); }

template <typename T> __device__ __forceinline__ T cadd(T a, T b) { return mkc(a.x + b.x, a.y + b.y); }
template <typename T> __device__ __forceinline__ T csub(T a, T b) { return mkc(a.x - b.x, a.y - b.y); }
template <typename T> __device__ __forceinline__ T cmul(T a, T b) {
  return mkc(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a*b + c
template <typename T> __device__ __forceinline__ T cfma(T a, T b, T c) {
  return mkc(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
template <typename T, typename S> __device__ __forceinline__ T cscale(T a, S s) {
  return mkc(a.x * s, a.y * s);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double cabs2(double2 a) { return a.x * a.x + a.y * a.y; }
__device__ __forceinline__ double2 to_d(float2 a) { return make_double2(a.x, a.y); }
__device__ __forceinline__ double2 to_d(double2 a) { return a; }
template <typename T> __device__ __forceinline__ T from_d(double2 a);
template <> __device__ __forceinline__ float2 from_d<float2>(double2 a) { return make_float2((float)a.x, (float)a.y); }
template <> __device__ __forceinline__ double2 from_d<double2>(double2 a) { return a; }
// conj(a) * b accumulated in fp64
__device__ __forceinline__ double2 cdot_acc(double2 acc, double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, fma(a.y, b.y, acc.x)), fma(a.x, b.y, fma(-a.y, b.x, acc.y)));
}
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  double d = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}

// Per-RHS scalars of one Krylov process (one per level and role). All fp64, device-resident
// so that whole cycles are stream-ordered with no host round trip (capturable as graphs).
struct KCtx {
  double* beta;    // [nrhs]          ||r0|| of the current cycle
  double* scale;   // [nrhs][KMAX+1]  lazy normalisation: v_i = scale_i * V_i(stored)
  double2* H;      // [nrhs][KMAX+1][KMAX] Hessenberg (rotated in place -> R)
  double* cs;      // [nrhs][KMAX]    Givens c (real)
  double2* sn;     // [nrhs][KMAX]    Givens s (complex)
  double2* g;      // [nrhs][KMAX+1]  rotated rhs beta e1
  int* kact;       // [nrhs]          active Krylov dimension (breakdown / zero rhs)
  double2* y;      // [nrhs][KMAX]    least-squares solution R y = g of the cycle (set when
                   //                 its last column closes; zero until then)
  double2* fc;     // [nrhs][KMAX+1]  forming coefficients of the last basis vector of the cycle,
                   //                 V_{k-1} = fc_{k-1} W + sum_{i<k-1} fc_i V_i (saved by the
                   //                 last fused step, which does not store V_{k-1}, 3D)
  int k;           // inner dimension of this process
  double* tol;     // [nrhs] or null: absolute residual-estimate tolerance for stopping INSIDE a
                   //                 cycle (R23: the Arnoldi estimate |g_{j+1}| may end a cycle
                   //                 early; convergence itself is decided on the true residual).
                   //                 Only the outer FGMRES sets it.
};

__device__ __forceinline__ int hidx(int i, int j) { return i * HELM_KMAX + j; }

// Programmatic dependent launch (sm_90+): the hot-path kernels are launched so that the next
// kernel's launch and block scheduling overlap this one's tail. Every such kernel calls
// pdl_wait() before touching memory (it returns once the preceding grid has completed and
// flushed) and pdl_trigger() to let its dependent launch early. Both are no-ops for a
// normal launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// ---------------------------------------------------------------- deterministic reductions
// Block-wide sum of NV fp64 complex values; fixed shuffle + fixed smem order (no atomics on
// data), result valid in thread 0.
template <int NV>
__device__ __forceinline__ void block_sum(double2 (&v)[NV], double2* sm /* [32][NV] */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v[k].x += __shfl_down_sync(0xffffffffu, v[k].x, o);
      v[k].y += __shfl_down_sync(0xffffffffu, v[k].y, o);
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) sm[warp * NV + k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double2 s = sm[k];
      for (int w = 1; w < nw; ++w) s = make_double2(s.x + sm[w * NV + k].x, s.y + sm[w * NV + k].y);
      v[k] = s;
    }
  }
  __syncthreads();
}

// Two-level deterministic grid reduction with a last-block ticket. Each block writes its
// partials part[blk*nv + k]; the last block to arrive for this RHS sums them over blocks in
// fixed order and returns true (all its threads) with the totals in `tot` (thread 0 valid
// after the call; broadcast through smem). The ticket is reset for graph replay.
template <int NV>
__device__ bool grid_sum_last(double2 (&v)[NV], int nv, double2* part, unsigned* ticket, int blk,
                              int nblk, double2* sm, double2* tot /* smem [NV] */) {
  block_sum<NV>(v, sm);
  __shared__ unsigned s_last;
  if (threadIdx.x == 0) {
    for (int k = 0; k < nv; ++k) part[(size_t)blk * nv + k] = v[k];
    __threadfence();
    unsigned t = atomicAdd(ticket, 1u);
    s_last = (t == (unsigned)(nblk - 1));
  }
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  // sum partials over blocks in fixed order: thread t handles blocks t, t+bd, ...
  double2 acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = make_double2(0.0, 0.0);
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) {
    const volatile double2* pb = part + (size_t)b * nv;
#pragma unroll
    for (int k = 0; k < NV; ++k)
      if (k < nv) {
        acc[k].x += pb[k].x;
        acc[k].y += pb[k].y;
      }
  }
  block_sum<NV>(acc, sm);
  if (threadIdx.x == 0) {
    for (int k = 0; k < nv; ++k) tot[k] = acc[k];
    *ticket = 0u;
  }
  __syncthreads();
  return true;
}
