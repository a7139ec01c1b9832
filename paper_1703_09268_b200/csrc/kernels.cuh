// kernels.cuh — sm_100a kernels of the Helmholtz hot path.
// Layout: complex interleaved, [rhs][z][y][x] with x fastest on the PML-extended grid.
// Every reduction is fp64 and deterministic (fixed-order block + last-block ticket).
#pragma once
#include "common.cuh"

// ----------------------------------------------------------------------------- geometry
// One geometry, `nop` operators: the batch of a joint (source, frequency) evaluation
// (Fig. 2) shares grid and model; operator o = frequency omega_o has its own 1D
// tables (stored op-major: table o of axis a starts at o * N_a) and omega_o^2. RHS r uses
// operator rop[r] (rop == null: operator 0).
#define HELM_MAXOP 16
template <typename R> struct Geo {
  int nx, ny, nz;          // extended sizes of this level
  long long N;             // nx*ny*nz
  const R* m;              // level model (slowness^2), extended
  int nop;                 // operators sharing this geometry
  const int* rop;          // per-RHS operator index, or null
  R w2[HELM_MAXOP];        // omega_o^2
  const cx<R>* lo[3];      // 1D tables (H or H^H), axis 0=x,1=y,2=z, nop tables each
  const cx<R>* dg[3];
  const cx<R>* up[3];
  const cx<R>* zpk;        // packed z coefficients [op][z][lo, dg, up] (ghosts masked, R7)
  int st;                  // stencil kind: 0 STD2 (D4-D5), 1 OPT (DESIGN R34 2D / R35 3D)
  int adj;                 // tables are H^H's (D6); OPT: the mass term is then diag(m) M, not M diag(m)
};

// ----------------------------------------------------------------------------- R34 / R35
// The paper's higher-order stencils (2D "9pt optimal" [23], 3D "compact 27-pt" [60])
// as the DESIGN readings define them: product forms of the stretched 1D tables T_a with the
// averages A = (1/4, 1/2, 1/4) and E = (1/2, 0, 1/2), H = L + omega^2 M diag(m) (Eq. 7 with
// A = M). Weights: DESIGN R34 / R35 (literal copies; scripts/derive_opt_stencil.py).
namespace optw {
constexpr double A9 = 0.58547, C9 = 0.63353, D9 = 0.36647, E9 = 1.0 - C9 - D9;
constexpr double W1 = 0.36027, W2 = 0.46886, W3 = 0.17087;
constexpr double M1 = 0.47314, M2 = 0.50415, M3 = 0.02271, M4 = 1.0 - M1 - M2 - M3;
// 2D: coef(dx, dz) = tx[dx] G9[dz] + tz[dz] G9[dx], G9 = a delta + (1 - a) A
constexpr double G9_0 = A9 + (1.0 - A9) / 2, G9_1 = (1.0 - A9) / 4;
// 3D: coef = tx[dx] G27(dy, dz) + ty[dy] G27(dx, dz) + tz[dz] G27(dx, dy),
// G27 = w1 delta delta + (w2/2)(A delta + delta A) + w3 A A, by number of nonzero offsets
constexpr double G27_0 = W1 + W2 / 2 + W3 / 4, G27_1 = W2 / 8 + W3 / 8, G27_2 = W3 / 16;
// mass weight of a neighbour by number of nonzero offsets (2D: centre, edge, corner)
constexpr double MU9_0 = C9, MU9_1 = D9 / 4, MU9_2 = E9 / 4;
constexpr double MU27_0 = M1, MU27_1 = M2 / 6, MU27_2 = M3 / 12, MU27_3 = M4 / 8;
}

// The 1D tables and omega^2 of RHS r's operator.
template <typename R> struct OpTab {
  const cx<R>*lo[3], *dg[3], *up[3];
  R w2;
};
template <typename R> __device__ __forceinline__ OpTab<R> op_tab(const Geo<R>& g, int r) {
  const int o = g.rop ? g.rop[r] : 0;
  OpTab<R> t;
  const long long n[3] = {g.nx, g.ny, g.nz};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    t.lo[a] = g.lo[a] + o * n[a];
    t.dg[a] = g.dg[a] + o * n[a];
    t.up[a] = g.up[a] + o * n[a];
  }
  t.w2 = g.w2[o];
  return t;
}

template <typename R> struct VPtrs { const cx<R>* p[HELM_KMAX + 1]; };

struct RedBuf {            // reduction scratch: partials per rhs + one ticket per rhs
  double2* part;
  unsigned* ticket;
  long long pstride;       // double2 entries per rhs
};

// ================================================================= Krylov scalars (device)
// Start a (re)started Krylov cycle of RHS r with ||r_0|| = beta: v_0 = r_0 / beta (lazy).
__device__ inline void start_cycle(const KCtx& ctx, int r, double beta) {
  constexpr int K1 = HELM_KMAX + 1;
  ctx.beta[r] = beta;
  ctx.scale[r * K1] = beta > 0.0 ? 1.0 / beta : 0.0;
  for (int i = 0; i <= HELM_KMAX; ++i) ctx.g[r * K1 + i] = make_double2(i == 0 ? beta : 0.0, 0.0);
  ctx.kact[r] = beta > 0.0 ? ctx.k : 0;
  for (int i = 0; i < HELM_KMAX; ++i) ctx.y[r * HELM_KMAX + i] = make_double2(0.0, 0.0);
}

// Back substitution R y = g over the cycle's kact columns (the rotated Hessenberg), once
// per RHS when the last column closes; the solution update then only reads y.
// (These scalar routines run in one thread at the tail of a launch: the 3D plane kernel
// stages the RHS's Krylov state in shared memory first, stencil.cuh KStage, so each
// dependent access is a shared-memory access, not an L2 round trip.)
__device__ inline void solve_ls(const KCtx& ctx, int r) {
  constexpr int K1 = HELM_KMAX + 1;
  const int k = ctx.kact[r];
  const double2* H = ctx.H + (long long)r * K1 * HELM_KMAX;
  const double2* gv = ctx.g + r * K1;
  double2 yv[HELM_KMAX];
  for (int i = HELM_KMAX - 1; i >= 0; --i) {
    if (i >= k) { yv[i] = make_double2(0.0, 0.0); continue; }
    double2 t = gv[i];
    for (int l = i + 1; l < k; ++l) t = csub(t, cmul(H[hidx(i, l)], yv[l]));
    const double2 d = H[hidx(i, i)];
    yv[i] = (d.x == 0.0 && d.y == 0.0) ? make_double2(0.0, 0.0) : cdiv(t, d);
  }
  for (int i = 0; i < HELM_KMAX; ++i) ctx.y[r * HELM_KMAX + i] = yv[i];
}

// Column j of the Hessenberg of RHS r is complete once h_{j+1,j} = hn is known: apply the
// previous Givens rotations to it, form rotation j, rotate g (residual estimate |g_{j+1}|),
// set the lazy scale of v_{j+1}, and apply the exact-breakdown guard (D14). Returns the
// RHS's active Krylov dimension afterwards.
__device__ inline int finalize_column(const KCtx& ctx, int r, int j, double hn) {
  constexpr int K1 = HELM_KMAX + 1;
  double2* H = ctx.H + (long long)r * K1 * HELM_KMAX;
  double* cs = ctx.cs + r * HELM_KMAX;
  double2* sn = ctx.sn + r * HELM_KMAX;
  double2* gv = ctx.g + r * K1;
  for (int i = 0; i < j; ++i) {   // previous rotations on column j
    const double2 a = H[hidx(i, j)], bb = H[hidx(i + 1, j)];
    const double c = cs[i];
    const double2 sv = sn[i];
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
  cs[j] = c; sn[j] = sv;
  H[hidx(j, j)] = cadd(make_double2(c * a.x, c * a.y), make_double2(sv.x * hn, sv.y * hn));
  H[hidx(j + 1, j)] = make_double2(0.0, 0.0);
  const double2 gj = gv[j];
  gv[j + 1] = cmul(make_double2(-sv.x, sv.y), gj);   // -conj(s) g_j
  gv[j] = make_double2(c * gj.x, c * gj.y);
  if (hn <= 1e-14 * ctx.beta[r]) {                    // breakdown guard (D14)
    ctx.kact[r] = j + 1;
    ctx.scale[r * K1 + j + 1] = 0.0;
  } else {
    ctx.scale[r * K1 + j + 1] = 1.0 / hn;
  }
  // early stop inside a cycle (R23): the residual estimate |g_{j+1}| of this RHS reached its
  // tolerance, so the cycle closes at j + 1 columns exactly like a breakdown (the host drops
  // the RHS from the cycle's remaining steps and the solution update reads j + 1 columns).
  if (ctx.tol && j + 1 < ctx.kact[r] && sqrt(cabs2(gv[j + 1])) <= ctx.tol[r]) {
    ctx.kact[r] = j + 1;
    ctx.scale[r * K1 + j + 1] = 0.0;
  }
  const int kact = ctx.kact[r];
  if (j + 1 >= kact) solve_ls(ctx, r);                // the cycle's last column closed
  return kact;
}

// ================================================================= a1: setup (D2-D4, D6, D13)
struct AxisPml {
  int N;            // nodes on this level
  int n_int;        // interior nodes (finest)
  int wlo, whi;     // PML widths (finest points)
  int level;        // coarsening level l (node i at xi = (i 2^l - wlo) h0)
  double h0, omega, R, power, vref;
};

__device__ inline double2 pml_eta(double xi, const AxisPml& a) {
  const double Lint = (a.n_int - 1) * a.h0;
  double sigma = 0.0;
  const double c = (a.power + 1.0) * a.vref * log(1.0 / a.R) * 0.5;
  if (a.wlo > 0) {
    const double L = a.wlo * a.h0, d = fmax(0.0, -xi);
    sigma += (c / L) * pow(d / L, a.power);
  }
  if (a.whi > 0) {
    const double L = a.whi * a.h0, d = fmax(0.0, xi - Lint);
    sigma += (c / L) * pow(d / L, a.power);
  }
  return make_double2(1.0, sigma / a.omega);   // eta = 1 + i sigma/omega (R3)
}

// D4: up_i = 1/(h^2 eta_i eta_{i+1/2}), lo_i = 1/(h^2 eta_i eta_{i-1/2}), dg = -(up+lo).
// Writes forward tables; the adjoint tables (D6) are derived by k_tables_adj.
__global__ void k_tables(AxisPml a, double2* lo, double2* dg, double2* up) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.N) return;
  const double s = (double)(1 << a.level);
  const double h = a.h0 * s;
  const double xi = ((double)i * s - a.wlo) * a.h0;
  const double2 e0 = pml_eta(xi, a), ep = pml_eta(xi + 0.5 * h, a), em = pml_eta(xi - 0.5 * h, a);
  const double2 one = make_double2(1.0 / (h * h), 0.0);
  double2 pu = make_double2(e0.x * ep.x - e0.y * ep.y, e0.x * ep.y + e0.y * ep.x);
  double2 pl = make_double2(e0.x * em.x - e0.y * em.y, e0.x * em.y + e0.y * em.x);
  double2 u = cdiv(one, pu), l = cdiv(one, pl);
  up[i] = u;
  lo[i] = l;
  dg[i] = make_double2(-(u.x + l.x), -(u.y + l.y));
}

// D6: (T^H y)_i = conj(up_{i-1}) y_{i-1} + conj(dg_i) y_i + conj(lo_{i+1}) y_{i+1}
__global__ void k_tables_adj(int N, const double2* lo, const double2* dg, const double2* up,
                             double2* loH, double2* dgH, double2* upH) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  loH[i] = i > 0 ? cconj(up[i - 1]) : make_double2(0.0, 0.0);
  dgH[i] = cconj(dg[i]);
  upH[i] = i < N - 1 ? cconj(lo[i + 1]) : make_double2(0.0, 0.0);
}

// D2: m_ext(i) = m(clamp(i_a - w_a^-, 0, n_a - 1)) (replication along the normal)
__global__ void k_extend(int Nx, int Ny, int Nz, int nx, int ny, int nz, int wx, int wy, int wz,
                         const double* __restrict__ m, double* __restrict__ me) {
  long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= (long long)Nx * Ny * Nz) return;
  int ix = p % Nx, iy = (p / Nx) % Ny, iz = p / ((long long)Nx * Ny);
  int cx_ = min(max(ix - wx, 0), nx - 1), cy = min(max(iy - wy, 0), ny - 1), cz = min(max(iz - wz, 0), nz - 1);
  me[p] = m[(long long)cz * nx * ny + (long long)cy * nx + cx_];
}

// D13: normalized full weighting (1/4, 1/2, 1/4) over in-range fine nodes, per axis.
__global__ void k_coarsen_model(int fx, int fy, int fz, int cxn, int cyn, int czn, int has_y,
                                const double* __restrict__ mf, double* __restrict__ mc) {
  long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= (long long)cxn * cyn * czn) return;
  int jx = p % cxn, jy = (p / cxn) % cyn, jz = p / ((long long)cxn * cyn);
  double s = 0.0, ws = 0.0;
  for (int dz = -1; dz <= 1; ++dz) {
    int iz = 2 * jz + dz;
    if (iz < 0 || iz >= fz) continue;
    double wz = dz == 0 ? 0.5 : 0.25;
    for (int dy = -has_y; dy <= has_y; ++dy) {
      int iy = has_y ? 2 * jy + dy : 0;
      if (iy < 0 || iy >= fy) continue;
      double wy = has_y ? (dy == 0 ? 0.5 : 0.25) : 1.0;
      for (int dx = -1; dx <= 1; ++dx) {
        int ix = 2 * jx + dx;
        if (ix < 0 || ix >= fx) continue;
        double w = wz * wy * (dx == 0 ? 0.5 : 0.25);
        s += w * mf[((long long)iz * fy + iy) * fx + ix];
        ws += w;
      }
    }
  }
  mc[p] = s / ws;
}

template <typename Tin, typename Tout>
__global__ void k_cast(long long n, const Tin* __restrict__ a, Tout* __restrict__ b) {
  long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) b[p] = (Tout)a[p];
}
// zpk[(o nz + z) ZS + {0,1,2}] = (lo_z (0 at z = 0), dg_z, up_z (0 at z = nz-1)) of operator o;
// ZS = 4 pads each entry with a zero (the 3D TMA copy moves whole 16-B multiples per plane)
template <typename T, int ZS = 3>
__global__ void k_zpack(int nz, int nop, const T* __restrict__ lo, const T* __restrict__ dg, const T* __restrict__ up,
                        T* __restrict__ zpk) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nz * nop) return;
  const int z = e % nz;
  T zero;
  zero.x = 0; zero.y = 0;
  zpk[ZS * e] = z > 0 ? lo[e] : zero;
  zpk[ZS * e + 1] = dg[e];
  zpk[ZS * e + 2] = z < nz - 1 ? up[e] : zero;
  if constexpr (ZS == 4) zpk[ZS * e + 3] = zero;
}

__global__ void k_cast_c(long long n, const double2* __restrict__ a, float2* __restrict__ b) {
  long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) b[p] = make_float2((float)a[p].x, (float)a[p].y);
}

// ================================================================= a3/a4: Krylov BLAS-1
// Cycle start from x0 = 0: r = b, v0 = b / ||b|| (lazy: scale only).
template <typename R>
__global__ void __launch_bounds__(HELM_RED_THREADS)
k_norm_start(long long N, const cx<R>* __restrict__ b, const int* __restrict__ active, KCtx ctx, RedBuf rb) {
  pdl_wait();
  pdl_trigger();
  const int r = active ? active[blockIdx.y] : blockIdx.y;   // compact list of active RHS
  const cx<R>* br = b + (long long)r * N;
  double s = 0.0;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < N; p += (long long)gridDim.x * blockDim.x) {
    cx<R> v = br[p];
    s += (double)v.x * v.x + (double)v.y * v.y;
  }
  __shared__ double2 sm[32];
  __shared__ double2 tot[1];
  double2 v[1] = {make_double2(s, 0.0)};
  if (grid_sum_last<1>(v, 1, rb.part + r * rb.pstride, rb.ticket + r, blockIdx.x, gridDim.x, sm, tot)) {
    if (threadIdx.x == 0) start_cycle(ctx, r, sqrt(tot[0].x));
  }
}

// out = (Tout)(s_r * in); zero if this Krylov step is past the active dimension.
template <typename Tin, typename Tout>
__global__ void k_copy_scale(long long N, const Tin* __restrict__ in, Tout* __restrict__ out,
                             const double* __restrict__ scale, int sstride, const int* __restrict__ kact,
                             int jstep, const int* __restrict__ active) {
  pdl_wait();
  pdl_trigger();
  const int r = active ? active[blockIdx.y] : blockIdx.y;   // compact list of active RHS
  const bool dead = kact && jstep >= kact[r];
  const double s = scale ? scale[(long long)r * sstride] : 1.0;
  const long long off = (long long)r * N;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < N; p += (long long)gridDim.x * blockDim.x) {
    double2 v = dead ? make_double2(0.0, 0.0) : to_d(in[off + p]);
    out[off + p] = from_d<Tout>(make_double2(v.x * s, v.y * s));
  }
}

// ================================================================= a5: level transfer (D13)
// r_c = 2^-d P^T r_f: coarse j gathers fine 2j (weight 1) and 2j+-1 (weight 1/2) per axis.
template <typename R>
__global__ void k_restrict(int fx, int fy, int fz, int cxn, int cyn, int czn, int has_y, R fac,
                           const cx<R>* __restrict__ in, cx<R>* __restrict__ out, const int* __restrict__ active) {
  pdl_wait();
  pdl_trigger();
  const int r = active ? active[blockIdx.y] : blockIdx.y;   // compact list of active RHS
  const long long Nc = (long long)cxn * cyn * czn, Nf = (long long)fx * fy * fz;
  const cx<R>* fin = in + (long long)r * Nf;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < Nc; p += (long long)gridDim.x * blockDim.x) {
    const int jx = p % cxn, jy = (p / cxn) % cyn, jz = p / ((long long)cxn * cyn);
    cx<R> acc = mkc((R)0, (R)0);
    for (int dz = -1; dz <= 1; ++dz) {
      const int iz = 2 * jz + dz;
      if (iz < 0 || iz >= fz) continue;
      const R wz = dz == 0 ? (R)1 : (R)0.5;
      for (int dy = -has_y; dy <= has_y; ++dy) {
        const int iy = has_y ? 2 * jy + dy : 0;
        if (iy < 0 || iy >= fy) continue;
        const R wy = wz * (dy == 0 ? (R)1 : (R)0.5);
        for (int dx = -1; dx <= 1; ++dx) {
          const int ix = 2 * jx + dx;
          if (ix < 0 || ix >= fx) continue;
          const R w = wy * (dx == 0 ? (R)1 : (R)0.5);
          const cx<R> v = fin[((long long)iz * fy + iy) * fx + ix];
          acc.x += w * v.x;
          acc.y += w * v.y;
        }
      }
    }
    out[(long long)r * Nc + p] = mkc(acc.x * fac, acc.y * fac);
  }
}

// x_f += P x_c: fine 2j <- c_j; fine 2j+1 <- (c_j + c_{j+1})/2 with c_{Nc} = 0, tensor product.
template <typename R>
__global__ void k_prolong_add(int fx, int fy, int fz, int cxn, int cyn, int czn, int has_y,
                              const cx<R>* __restrict__ in, cx<R>* __restrict__ out, const int* __restrict__ active) {
  pdl_wait();
  pdl_trigger();
  const int r = active ? active[blockIdx.y] : blockIdx.y;   // compact list of active RHS
  const long long Nc = (long long)cxn * cyn * czn, Nf = (long long)fx * fy * fz;
  const cx<R>* cin = in + (long long)r * Nc;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < Nf; p += (long long)gridDim.x * blockDim.x) {
    const int ix = p % fx, iy = (p / fx) % fy, iz = p / ((long long)fx * fy);
    int jx[2], jy[2], jz[2];
    R wx[2], wy[2], wz[2];
    int nxp, nyp, nzp;
    auto axis = [](int i, int nc, int* j, R* w, int& n) {
      if ((i & 1) == 0) { j[0] = i >> 1; w[0] = (R)1; n = 1; }
      else { j[0] = i >> 1; w[0] = (R)0.5; j[1] = (i >> 1) + 1; w[1] = (R)0.5; n = j[1] < nc ? 2 : 1; }
    };
    axis(ix, cxn, jx, wx, nxp);
    axis(iz, czn, jz, wz, nzp);
    if (has_y) axis(iy, cyn, jy, wy, nyp);
    else { jy[0] = 0; wy[0] = (R)1; nyp = 1; }
    cx<R> acc = mkc((R)0, (R)0);
    for (int a = 0; a < nzp; ++a)
      for (int bq = 0; bq < nyp; ++bq)
        for (int c = 0; c < nxp; ++c) {
          const R w = wz[a] * wy[bq] * wx[c];
          const cx<R> v = cin[((long long)jz[a] * cyn + jy[bq]) * cxn + jx[c]];
          acc.x += w * v.x;
          acc.y += w * v.y;
        }
    cx<R>* o = out + (long long)r * Nf + p;
    *o = cadd(*o, acc);
  }
}

// ================================================================= a7, a9: FWI kernels
// q_s = S(omega_s) e_node(s) / h^d (D7), one amplitude per RHS; B zeroed beforehand.
template <typename R>
__global__ void k_inject(int ns, long long N, const long long* __restrict__ src_ext, const double2* __restrict__ amp,
                         cx<R>* __restrict__ B) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < ns) B[(long long)s * N + src_ext[s]] = from_d<cx<R>>(amp[s]);
}

// r = P_r u - d (D8, D10); A = -P_r^T r (D11, receivers distinct); f += 1/2 ||r||^2 (fp64,
// deterministic: block partials + last-block ticket, then one sequential add into *f).
template <typename R>
__global__ void __launch_bounds__(HELM_RED_THREADS)
k_gather_residual(int ns, int nrec, long long N, const long long* __restrict__ rec_ext,
                  const double2* __restrict__ d, const cx<R>* __restrict__ U, cx<R>* __restrict__ A,
                  double* f, RedBuf rb) {
  double s = 0.0;
  const long long tot_n = (long long)ns * nrec;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < tot_n; q += (long long)gridDim.x * blockDim.x) {
    const int si = q / nrec, k = q % nrec;
    const long long e = rec_ext[k];
    const double2 u = to_d(U[(long long)si * N + e]);
    const double2 rv = csub(u, d[q]);
    A[(long long)si * N + e] = from_d<cx<R>>(make_double2(-rv.x, -rv.y));
    s += cabs2(rv);
  }
  __shared__ double2 sm[32];
  __shared__ double2 tot[1];
  double2 v[1] = {make_double2(s, 0.0)};
  if (grid_sum_last<1>(v, 1, rb.part, rb.ticket, blockIdx.x, gridDim.x, sm, tot)) {
    if (threadIdx.x == 0) *f += 0.5 * tot[0].x;
  }
}

// d[s][k] = (P_r u_s)_k (D8; Listing 1 FORW_MODEL P:164-165)
template <typename R>
__global__ void k_gather_data(int ns, int nrec, long long N, const long long* __restrict__ rec_ext,
                              const cx<R>* __restrict__ U, double2* __restrict__ d) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (long long)ns * nrec) return;
  const int si = q / nrec, k = q % nrec;
  d[q] = to_d(U[(long long)si * N + rec_ext[k]]);
}

// g_ext += sum_s Re(omega_s^2 conj(u_s) v_s) (Eq. 8, Listing 1), fp64, fixed
// RHS order (the batch's RHS may carry different frequencies).
template <typename R>
__global__ void k_grad(int ns, long long N, const double* __restrict__ w2, const cx<R>* __restrict__ U,
                       const cx<R>* __restrict__ V, double* __restrict__ gext) {
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < N; p += (long long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int s = 0; s < ns; ++s) {
      const double2 u = to_d(U[(long long)s * N + p]), v = to_d(V[(long long)s * N + p]);
      acc += w2[s] * (u.x * v.x + u.y * v.y);
    }
    gext[p] += acc;
  }
}

// OPT stencils (DESIGN R34 / R35): H = L + omega^2 M diag(m), so T^* z = Re(omega^2 conj(u) (M^H z))
// (Eqs. 7-8; M real symmetric): g_ext += sum_s Re(omega_s^2 conj(u_s) (M v_s)), the
// mass distribution gathered per point (ghosts zero, R7), fp64, fixed RHS order.
template <typename R>
__global__ void k_grad_opt(int ns, int nx, int ny, int nz, const double* __restrict__ w2, const cx<R>* __restrict__ U,
                           const cx<R>* __restrict__ V, double* __restrict__ gext) {
  const long long N = (long long)nx * ny * nz, pl = (long long)nx * ny;
  const bool d3 = ny > 1;
  const double mu3[4] = {optw::MU27_0, optw::MU27_1, optw::MU27_2, optw::MU27_3};
  const double mu2[3] = {optw::MU9_0, optw::MU9_1, optw::MU9_2};
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < N; p += (long long)gridDim.x * blockDim.x) {
    const int ix = (int)(p % nx), iy = (int)((p / nx) % ny), iz = (int)(p / pl);
    double acc = 0.0;
    for (int s = 0; s < ns; ++s) {
      const cx<R>* v = V + (long long)s * N;
      double mx = 0.0, my = 0.0;
      for (int dz = -1; dz <= 1; ++dz) {
        if (iz + dz < 0 || iz + dz >= nz) continue;
        for (int dy = d3 ? -1 : 0; dy <= (d3 ? 1 : 0); ++dy) {
          if (iy + dy < 0 || iy + dy >= ny) continue;
          for (int dx = -1; dx <= 1; ++dx) {
            if (ix + dx < 0 || ix + dx >= nx) continue;
            const int n = (dx != 0) + (dy != 0) + (dz != 0);
            const double mu = d3 ? mu3[n] : mu2[n];
            const double2 q = to_d(v[p + dz * pl + dy * nx + dx]);
            mx += mu * q.x;
            my += mu * q.y;
          }
        }
      }
      const double2 u = to_d(U[(long long)s * N + p]);
      acc += w2[s] * (u.x * mx + u.y * my);
    }
    gext[p] += acc;
  }
}

// g = E^T g_ext (D12, R11): each interior cell sums the extended nodes that replicate it
// (its PML line / face / corner box); written into fg[1 + i]; fg[0] = f.
// (f == null: model-space output only, g[p] = (E^T g_ext)_p without the leading f slot)
__global__ void k_fold(int Nx, int Ny, int Nz, int nx, int ny, int nz, int wx, int wy, int wz,
                       const double* __restrict__ gext, const double* __restrict__ f, double* __restrict__ fg) {
  long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (f && p == 0) fg[0] = *f;
  const int off = f ? 1 : 0;
  if (p >= (long long)nx * ny * nz) return;
  const int ix = p % nx, iy = (p / nx) % ny, iz = p / ((long long)nx * ny);
  auto range = [](int i, int n, int w, int Nn, int& a, int& b) {
    a = i == 0 ? 0 : i + w;
    b = i == n - 1 ? Nn - 1 : i + w;
  };
  int xa, xb, ya, yb, za, zb;
  range(ix, nx, wx, Nx, xa, xb);
  range(iy, ny, wy, Ny, ya, yb);
  range(iz, nz, wz, Nz, za, zb);
  double s = 0.0;
  for (int k = za; k <= zb; ++k)
    for (int j = ya; j <= yb; ++j)
      for (int i = xa; i <= xb; ++i) s += gext[((long long)k * Ny + j) * Nx + i];
  fg[off + p] = s;
}

// Born source of the linearised modelling (Table 1 T dm, Eq. 7 with A = I; Listing 1
// JACOBI_FORW / HESS_GN): B_s = -T dm = -omega_s^2 u_s (.) (E dm), dm_ext = E dm in fp64.
template <typename R>
__global__ void k_born_src(int ns, long long N, const double* __restrict__ w2, const cx<R>* __restrict__ U,
                           const double* __restrict__ dm_ext, cx<R>* __restrict__ B) {
  const long long tot = (long long)ns * N;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < tot; q += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(q / N);
    const long long p = q - (long long)s * N;
    const double2 u = to_d(U[q]);
    const double c = -w2[s] * dm_ext[p];
    B[q] = from_d<cx<R>>(make_double2(c * u.x, c * u.y));
  }
}

// Adjoint source from host data y (Listing 1 JACOBI_ADJ): A_s = -P_r^T y_s (receivers distinct; A zeroed).
template <typename R>
__global__ void k_scatter_neg(int ns, int nrec, long long N, const long long* __restrict__ rec_ext,
                              const double2* __restrict__ y, cx<R>* __restrict__ A) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (long long)ns * nrec) return;
  const int s = (int)(q / nrec), k = (int)(q % nrec);
  const double2 v = y[q];
  A[(long long)s * N + rec_ext[k]] = from_d<cx<R>>(make_double2(-v.x, -v.y));
}

// ================================================================= a3/a4 BLAS-1, templated
// NV = j+1 basis vectors known at compile time; 2 points per thread per iteration so every
// thread has 2*(NV+1) independent 16-byte loads in flight.
template <typename R, int NV>
__global__ void __launch_bounds__(HELM_RED_THREADS)
k_update_t(long long N, VPtrs<R> V, int j, cx<R>* __restrict__ w, const int* __restrict__ active, KCtx ctx,
           RedBuf rb) {
  pdl_wait();
  pdl_trigger();
  const int r = active ? active[blockIdx.y] : blockIdx.y;   // compact list of active RHS
  if (j >= ctx.kact[r]) return;
  const long long off = (long long)r * N;
  cx<R>* wr = w + off;
  cx<R> coef[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const double2 h = ctx.H[(long long)r * (HELM_KMAX + 1) * HELM_KMAX + hidx(i, j)];
    const double sc = ctx.scale[r * (HELM_KMAX + 1) + i];
    coef[i] = from_d<cx<R>>(make_double2(-h.x * sc, -h.y * sc));
  }
  const cx<R>* vp[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) vp[i] = V.p[i] + off;
  double s = 0.0;
  const long long gs = (long long)gridDim.x * blockDim.x;
  long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; p + gs < N; p += 2 * gs) {
    cx<R> w0 = wr[p], w1 = wr[p + gs];
    cx<R> a0[NV], a1[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) { a0[i] = vp[i][p]; a1[i] = vp[i][p + gs]; }
#pragma unroll
    for (int i = 0; i < NV; ++i) { w0 = cfma(coef[i], a0[i], w0); w1 = cfma(coef[i], a1[i], w1); }
    wr[p] = w0;
    wr[p + gs] = w1;
    s += (double)w0.x * w0.x + (double)w0.y * w0.y + (double)w1.x * w1.x + (double)w1.y * w1.y;
  }
  if (p < N) {
    cx<R> w0 = wr[p];
#pragma unroll
    for (int i = 0; i < NV; ++i) w0 = cfma(coef[i], vp[i][p], w0);
    wr[p] = w0;
    s += (double)w0.x * w0.x + (double)w0.y * w0.y;
  }
  __shared__ double2 sm[32];
  __shared__ double2 tot[1];
  double2 v[1] = {make_double2(s, 0.0)};
  if (grid_sum_last<1>(v, 1, rb.part + r * rb.pstride, rb.ticket + r, blockIdx.x, gridDim.x, sm, tot)) {
    if (threadIdx.x == 0) finalize_column(ctx, r, j, sqrt(tot[0].x));
  }
}

// x <- (init ? 0 : x) + sum_{i<kact} y_i z_i, R y = g by back substitution (per block).
// W != null (3D unpreconditioned GMRES, whose last fused step does not store z_{K-1}): when
// the cycle ran all K steps, z_{K-1} = fc_{K-1} W + sum_{i<K-1} fc_i z_i (the forming
// coefficients that step saved) is folded into the coefficients and W read in its place.
template <typename R, int K>
__global__ void __launch_bounds__(HELM_RED_THREADS)
k_solupdate_t(long long N, VPtrs<R> Z, const double* __restrict__ zscale, cx<R>* __restrict__ x, int init,
              const int* __restrict__ active, KCtx ctx, const cx<R>* __restrict__ W) {
  pdl_wait();
  pdl_trigger();
  const int r = active ? active[blockIdx.y] : blockIdx.y;   // compact list of active RHS
  __shared__ cx<R> yc[K];
  __shared__ int s_k;
  if (threadIdx.x == 0) {
    const int K1 = HELM_KMAX + 1;
    const int k = ctx.kact[r];
    double2 yd[K];
    for (int i = 0; i < K; ++i) {
      const double2 yv = ctx.y[r * HELM_KMAX + i];
      const double sc = (zscale && i < k) ? zscale[r * K1 + i] : 1.0;
      yd[i] = make_double2(yv.x * sc, yv.y * sc);
    }
    if (W && k == K && K > 1) {
      const double2* fc = ctx.fc + r * K1;
      const double2 yl = yd[K - 1];
      for (int i = 0; i < K - 1; ++i) yd[i] = cadd(yd[i], cmul(yl, fc[i]));
      yd[K - 1] = make_double2(yl.x * fc[K - 1].x, yl.y * fc[K - 1].x);
    }
    for (int i = 0; i < K; ++i) yc[i] = from_d<cx<R>>(yd[i]);
    s_k = k;
  }
  __syncthreads();
  const int k = s_k;
  if (k == 0 && !init) return;
  const long long off = (long long)r * N;
  cx<R>* xr = x + off;
  cx<R> yl[K];
  const cx<R>* zp[K];
#pragma unroll
  for (int i = 0; i < K; ++i) { yl[i] = yc[i]; zp[i] = Z.p[i] + off; }
  if (W && k == K) zp[K - 1] = W + off;
  const long long gs = (long long)gridDim.x * blockDim.x;
  long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; p + gs < N; p += 2 * gs) {
    cx<R> x0 = init ? mkc((R)0, (R)0) : xr[p];
    cx<R> x1 = init ? mkc((R)0, (R)0) : xr[p + gs];
    cx<R> a0[K], a1[K];
#pragma unroll
    for (int i = 0; i < K; ++i)
      if (i < k) { a0[i] = zp[i][p]; a1[i] = zp[i][p + gs]; }
#pragma unroll
    for (int i = 0; i < K; ++i)
      if (i < k) { x0 = cfma(yl[i], a0[i], x0); x1 = cfma(yl[i], a1[i], x1); }
    xr[p] = x0;
    xr[p + gs] = x1;
  }
  if (p < N) {
    cx<R> x0 = init ? mkc((R)0, (R)0) : xr[p];
#pragma unroll
    for (int i = 0; i < K; ++i)
      if (i < k) x0 = cfma(yl[i], zp[i][p], x0);
    xr[p] = x0;
  }
}

// ---------------------------------------------------------------------------------------
// Off-grid sources and receivers (Kaiser-windowed sinc, DESIGN R33; SURVEY
// §8(f) rank 4). P is a sparse row set built on the host: point p has taps [off[p], off[p+1])
// with extended-grid nodes node[t] and weights w[t] (tensor products of normalised 1D
// windowed-sinc weights). All sums run in a fixed order (bitwise reproducible, R30).

// q_b = amp_b P_s^T e_{src(b)} (B zeroed; the taps of one source are distinct nodes).
template <typename R>
__global__ void k_inject_taps(int nb, long long N, const long long* __restrict__ srcb, const int* __restrict__ off,
                              const long long* __restrict__ node, const double* __restrict__ w,
                              const double2* __restrict__ amp, cx<R>* __restrict__ B) {
  const int b = blockIdx.x;
  if (b >= nb) return;
  const int s = (int)srcb[b];
  const double2 a = amp[b];
  for (int t = off[s] + threadIdx.x; t < off[s + 1]; t += blockDim.x)
    B[(long long)b * N + node[t]] = from_d<cx<R>>(make_double2(a.x * w[t], a.y * w[t]));
}

// out[b][k] = (P_r u_b)_k - d[b][k]   (d may be null)
template <typename R>
__global__ void k_rec_gather(int nb, int nrec, long long N, const int* __restrict__ off, const long long* __restrict__ node,
                             const double* __restrict__ w, const cx<R>* __restrict__ U, const double2* __restrict__ d,
                             double2* __restrict__ out) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (long long)nb * nrec) return;
  const int b = (int)(q / nrec), k = (int)(q % nrec);
  const cx<R>* u = U + (long long)b * N;
  double sx = 0.0, sy = 0.0;
  for (int t = off[k]; t < off[k + 1]; ++t) {
    const double2 v = to_d(u[node[t]]);
    sx += w[t] * v.x;
    sy += w[t] * v.y;
  }
  if (d) { sx -= d[q].x; sy -= d[q].y; }
  out[q] = make_double2(sx, sy);
}

// *f += 1/2 sum |r_i|^2 over n entries: one 1024-thread block, fixed order.
__global__ void __launch_bounds__(1024) k_half_sumsq(long long n, const double2* __restrict__ r, double* f) {
  __shared__ double sm[1024];
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += 1024) s += r[i].x * r[i].x + r[i].y * r[i].y;
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int h = 512; h > 0; h >>= 1) {
    if (threadIdx.x < h) sm[threadIdx.x] += sm[threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) *f += 0.5 * sm[0];
}

// A_b = -P_r^T r_b as a gather over the touched nodes (rows of P_r^T: node[p], taps
// [off[p], off[p+1]) with receiver rec[t] and weight w[t]); A zeroed elsewhere.
template <typename R>
__global__ void k_rec_scatterT(int nb, int nnode, int nrec, long long N, const int* __restrict__ off,
                               const long long* __restrict__ node, const int* __restrict__ rec,
                               const double* __restrict__ w, const double2* __restrict__ r, cx<R>* __restrict__ A) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (long long)nb * nnode) return;
  const int b = (int)(q / nnode), p = (int)(q % nnode);
  double sx = 0.0, sy = 0.0;
  for (int t = off[p]; t < off[p + 1]; ++t) {
    const double2 v = r[(long long)b * nrec + rec[t]];
    sx += w[t] * v.x;
    sy += w[t] * v.y;
  }
  A[(long long)b * N + node[p]] = from_d<cx<R>>(make_double2(-sx, -sy));
}
