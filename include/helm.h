/*
 * helm.h — C ABI of libhelm.so, the B200 (sm_100a) hot path of arXiv 1703.09268:
 * the per-source, per-frequency PML Helmholtz solve (FGMRES + ML-GMRES) feeding the
 * least-squares misfit and its adjoint-state gradient.
 *
 * Citations: P:n = line n of the paper text,
 *            D<k>/R<k> = SURVEY.md §8(c) definitions / readings (restated in DESIGN.md).
 *
 * Conventions (every entry point):
 *  - Layout. Complex arrays are interleaved (re, im), C-order [rhs][z][y][x], x fastest,
 *    on the PML-EXTENDED grid (N_a = n_a + pml[a][0] + pml[a][1]). 2D problems are (x, z):
 *    ndim = 2, n[1] = 1, pml[1] = {0, 0}. Models are real, INTERIOR, x fastest.
 *  - Ownership. The caller owns every pointer argument. Host arrays are copied before the
 *    call returns. Device arrays are caller-allocated (cudaMalloc / torch) and must be
 *    8-byte aligned (16 for complex128). A helm_op owns its device copies of the model,
 *    the 1D PML tables, the level hierarchy, the Krylov workspace for max_rhs right-hand
 *    sides and its captured CUDA graphs; helm_destroy frees them.
 *  - Streams. Work is ordered on `cuda_stream` (cudaStream_t, NULL = legacy default).
 *    helm_apply is asynchronous. helm_setup, helm_solve, fwi_* return after completion.
 *  - Concurrency. One helm_op must not be used from two threads/streams at once.
 *  - Errors. A negative status means nothing was written to the outputs (argument and
 *    shape checks run before any work). CUDA / allocation failures return
 *    HELM_ERR_CUDA / HELM_ERR_OOM. helm_last_error() gives thread-local text for the last
 *    non-OK status (and for warnings, e.g. < 4 points per wavelength, with HELM_OK).
 *  - There is no CPU fallback: every numeric step runs in this library's CUDA kernels.
 */
#ifndef HELM_H
#define HELM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HELM_OK = 0,
  HELM_ERR_ARG = -1,    /* bad scalar argument / NULL pointer */
  HELM_ERR_SHAPE = -2,  /* sizes inconsistent (nrhs > max_rhs, grid too small, ...) */
  HELM_ERR_CUDA = -3,   /* CUDA runtime error (text in helm_last_error) */
  HELM_ERR_OOM = -4,    /* device allocation failed */
  HELM_ERR_STATE = -5   /* library / device not usable (no sm_100 device, ...) */
} helm_status;

/* D15 / R26. HELM_C128: everything complex128, fp64 reductions.
 * HELM_C64 ("mixed"): user-visible complex arrays are complex64; the stencil, the V-cycle
 * and the smoother / coarse Krylov bases run in complex64 with fp32 tables and model; the
 * outer FGMRES (its basis, iterate, true residual and matvec) runs in complex128 against
 * the fp64 operator, so solves reach the fp64 operator's rel-residual target. */
typedef enum { HELM_C64 = 0, HELM_C128 = 1 } helm_dtype;

/* D1. Interior grid; PML points per axis and side. */
typedef struct {
  int32_t ndim;        /* 2 (x,z) or 3 (x,y,z) */
  int64_t n[3];        /* interior points per axis, x first (n[1] = 1 in 2D) */
  double h;            /* uniform spacing [m], > 0 */
  int32_t pml[3][2];   /* PML points per axis per side (pml[1] = {0,0} in 2D) */
  int32_t stencil;     /* HELM_STD2 (0): 5-pt (2D) / 7-pt (3D), D4-D5 (R4). HELM_OPT (1): the paper's
                        * higher-order stencils ("9pt optimal" [23] / "compact 27-pt" [60]) as
                        * DESIGN R34 (2D 9-pt) / R35 (3D 27-pt): product forms of the same stretched
                        * 1D tables, H = L + omega^2 M diag(m) with the mass distribution M = A of
                        * Eq. (7). Every level of the hierarchy uses the same kind. OPT is
                        * supported by helm_apply, helm_solve, fwi_misfit_grad, fwi_forward and
                        * fwi_jacobian_adjoint; the Born-source calls (fwi_jacobian,
                        * fwi_gn_hessian) and off-grid acquisition return HELM_ERR_ARG for it. */
} helm_grid;
#define HELM_STD2 0
#define HELM_OPT 1

/* D3 / R5. sigma(d) = sigma_max (d/L)^power, sigma_max = (power+1) v_ref ln(1/R) / (2L),
 * eta = 1 + i sigma/omega (R3). v_ref <= 0 in helm_setup means "max velocity of m";
 * fwi_* require v_ref > 0 so that H depends on m only through omega^2 diag(E m) (Eq. 7). */
typedef struct { double R; int32_t power; double v_ref; } helm_pml;

/* §5: memory vector (k_so, k_si, k_co, k_ci) = (3,5,3,5), levels = 3 grids (R20).
 * levels = 0 builds an operator-only op (helm_apply only; no hierarchy or Krylov workspace). */
typedef struct { int32_t levels, ks_o, ks_i, kc_o, kc_i; } helm_mlopts;

/* outer FGMRES(k_inner) restarted until the TRUE ||b - Hx||/||b|| <= rtol per RHS
 * (R23), x0 = 0; precond 1 = ML-GMRES, 0 = none (plain restarted GMRES(k_inner)). A RHS
 * whose Arnoldi residual estimate reaches 0.5 rtol ||b|| inside a cycle closes that cycle at
 * the current column (R23's early stop); the true residual is then checked as always.
 * outer_cycles counts started cycles, full or cut short. */
typedef struct { int32_t k_inner, max_outer; double rtol; int32_t precond; } helm_solve_opts;

/* Per right-hand side. matvecs[l] = operator applications on level l (fine = 0);
 * bytes_alg = algorithmic HBM bytes the kernels of this solve moved for this RHS
 * (DESIGN.md §6 per-kernel formulas). Non-convergence is NOT an error: converged = 0. */
typedef struct {
  int32_t outer_cycles, converged;
  double rel_residual;
  int64_t matvecs[4];
  double bytes_alg;
} helm_solve_report;

/* Off-grid acquisition ("Kaiser-windowed sinc interpolation"; SURVEY §8(f) rank 4;
 * DESIGN R33). Coordinates are physical (grid units of h), relative to interior node (0,0,0),
 * host fp64 triples (x, y, z) — 2D grids need y = 0; every point must lie inside the interior
 * box [0, (n_a - 1) h] (else HELM_ERR_ARG naming the point). Rows of P: tensor products of 1D
 * weights sinc(t-k) I0(b sqrt(1-((t-k)/r)^2)) / I0(b), |t-k| <= r, each axis normalised to
 * sum 1 (an on-node point is the on-node delta). kaiser_b <= 0 selects 6.31, half_width <= 0
 * selects 4 (max 8). The source of point s is S(omega) P_s^T e_s / h^d. */
typedef struct {
  const double* src_xyz;   /* [nsrc_total][3] */
  const double* rec_xyz;   /* [nrec][3] */
  double kaiser_b;
  int32_t half_width;
} helm_acq;

typedef struct helm_op helm_op;   /* opaque */

/* a1 (Fig. 3). Builds, on the device: m_ext = E m (D2), the per
 * level / per axis complex 1D tables (lo, dg, up) of H and of H^H (D4, D6), the coarse
 * models by normalized full weighting and their tables (D13), and the Krylov workspace for
 * `max_rhs` right-hand sides. omega = 2 pi f [rad/s] > 0. mlopts NULL = defaults.
 * m_slowness2: host, interior, n[0]*n[1]*n[2] doubles, x fastest (R1: m = 1/v^2). */
helm_status helm_setup(const helm_grid* grid, const double* m_slowness2, double omega,
                       const helm_pml* pml, helm_dtype dtype, int32_t max_rhs,
                       const helm_mlopts* mlopts, void* cuda_stream, helm_op** out);

/* a2 (Eq. 1). y = H x (adjoint = 0) or y = H^H x (adjoint = 1) for
 * nrhs right-hand sides on the finest extended grid; x, y device, dtype of the op, must not
 * alias. H = sum_a T_a + omega^2 diag(E m) (D5; grid.stencil = HELM_OPT: R34 / R35),
 * zero Dirichlet ghosts (R7). Asynchronous on cuda_stream. */
helm_status helm_apply(helm_op* op, int32_t adjoint, int32_t nrhs, const void* x_dev,
                       void* y_dev, void* cuda_stream);

/* a3-a6 (+a8 with adjoint = 1). Solves H x = b (or H^H x = b) for nrhs independent RHS
 * (R27) with the paper's solver: outer FGMRES with k_inner = 5 inner iterations to a true
 * relative residual of rtol = 1e-6 (R23), right-preconditioned by the ML-GMRES cycle
 * of §5 (Alg. 1, recursion Fig. 3; counts (3,5,3,5) P:284; GMRES
 * smoothers P:274). b_dev, x_dev: device, extended grid, dtype of the op; x_dev is output
 * only (x0 = 0). report_host: NULL or an array of nrhs reports. Returns after
 * completion. Non-convergence within max_outer is not an error (converged = 0). */
helm_status helm_solve(helm_op* op, int32_t adjoint, int32_t nrhs, const void* b_dev,
                       void* x_dev, const helm_solve_opts* opts,
                       helm_solve_report* report_host, void* cuda_stream);

/* a1-a9 (Listing 1 `case OBJ`; Eq. 2; Eq. 8; D7-D12). For each
 * frequency and each source s in [src_begin, src_end):
 *   u = H^-1 q_s, q_s = S e_node(s)/h^d;  f += 1/2 ||P_r u - d||^2;
 *   v = H^-H(-P_r^T(P_r u - d));        g += E^T Re(omega^2 conj(u) v).
 * Sources are solved in batches of at most `max_rhs`. src_node / rec_node: host, interior
 * linear node ids (ix + nx*(iy + ny*iz)); receivers must be distinct. d_obs_reim: host
 * complex128 [nfreq][nsrc_total][nrec]. src_weight_reim: host complex128 [nfreq] or NULL
 * (S = 1). fg_dev: device fp64 [1 + n_interior], overwritten with f then g (interior, x
 * fastest); the multi-GPU sum is the caller's all_reduce over this buffer.
 * report_host: NULL or [nfreq][src_end - src_begin][2] (forward, adjoint). */
helm_status fwi_misfit_grad(const helm_grid* grid, const double* m_slowness2, int32_t nfreq,
                            const double* freq_hz, const double* src_weight_reim,
                            int32_t nsrc_total, int32_t src_begin, int32_t src_end,
                            const int64_t* src_node, int32_t nrec, const int64_t* rec_node,
                            const double* d_obs_reim, const helm_pml* pml, helm_dtype dtype,
                            const helm_solve_opts* opts, int32_t max_rhs, double* fg_dev,
                            helm_solve_report* report_host, void* cuda_stream);

/* Listing 1 `case FORW_MODEL`: d[f][s][k] = (P_r H_f^-1 q_s)_k for s in
 * [src_begin, src_end). d_host: host complex128 [nfreq][src_end - src_begin][nrec]. */
helm_status fwi_forward(const helm_grid* grid, const double* m_slowness2, int32_t nfreq,
                        const double* freq_hz, const double* src_weight_reim,
                        int32_t src_begin, int32_t src_end, const int64_t* src_node,
                        int32_t nrec, const int64_t* rec_node, const helm_pml* pml,
                        helm_dtype dtype, const helm_solve_opts* opts, int32_t max_rhs,
                        double* d_host, helm_solve_report* report_host, void* cuda_stream);

/* ---- the linearised operators of Listing 1 (Table 1) ------
 * With T dm = omega^2 u (E dm) (the Born source, D2/D5) and T^* z = E^T Re(omega^2 conj(u) z):
 *   J dm   = P_r du,  du = -H^-1 T dm                    (JACOBI_FORW, 2 solves per pair)
 *   J^H y  = T^* H^-H(-P_r^T y)                           (JACOBI_ADJ, 2 solves per pair)
 *   GN dm  = J^H J dm = T^* H^-H(-P_r^T P_r du)           (HESS_GN, 3 solves per pair, Table 2)
 * Same conventions as fwi_misfit_grad (host node ids, host data, joint (source, frequency)
 * batches of at most max_rhs). dm: host fp64 interior perturbation of m = slowness^2.
 * Reports: NULL or [nfreq][src_end - src_begin][2] (J, J^H: forward, second solve) or [..][3]
 * (GN: forward, born, adjoint). Errors as fwi_misfit_grad. */

/* d_host: host complex128 [nfreq][src_end - src_begin][nrec] = J dm for this shard's sources. */
helm_status fwi_jacobian(const helm_grid* grid, const double* m_slowness2, int32_t nfreq,
                         const double* freq_hz, const double* src_weight_reim,
                         int32_t src_begin, int32_t src_end, const int64_t* src_node,
                         int32_t nrec, const int64_t* rec_node, const double* dm,
                         const helm_pml* pml, helm_dtype dtype, const helm_solve_opts* opts,
                         int32_t max_rhs, double* d_host, helm_solve_report* report_host,
                         void* cuda_stream);

/* y_reim: host complex128 [nfreq][nsrc_total][nrec] (the whole survey; this shard reads
 * its own sources). g_dev: device fp64 [n_interior] = this shard's part of J^H y (all-reduce
 * across shards is the caller's). */
helm_status fwi_jacobian_adjoint(const helm_grid* grid, const double* m_slowness2, int32_t nfreq,
                                 const double* freq_hz, const double* src_weight_reim,
                                 int32_t nsrc_total, int32_t src_begin, int32_t src_end,
                                 const int64_t* src_node, int32_t nrec, const int64_t* rec_node,
                                 const double* y_reim, const helm_pml* pml, helm_dtype dtype,
                                 const helm_solve_opts* opts, int32_t max_rhs, double* g_dev,
                                 helm_solve_report* report_host, void* cuda_stream);

/* h_dev: device fp64 [n_interior] = this shard's part of J^H J dm. */
helm_status fwi_gn_hessian(const helm_grid* grid, const double* m_slowness2, int32_t nfreq,
                           const double* freq_hz, const double* src_weight_reim,
                           int32_t src_begin, int32_t src_end, const int64_t* src_node,
                           int32_t nrec, const int64_t* rec_node, const double* dm,
                           const helm_pml* pml, helm_dtype dtype, const helm_solve_opts* opts,
                           int32_t max_rhs, double* h_dev, helm_solve_report* report_host,
                           void* cuda_stream);

/* Batch-mode subset ("a set of source-frequency indices"):
 * fwi_misfit_grad over only the (frequency, source) pairs with pair_mask[f][s] != 0 (host
 * uint8 [nfreq][nsrc_total]; sources outside [src_begin, src_end) are ignored), evaluated in
 * joint batches in frequency-major order. report_host: NULL or [selected pairs][2] in that
 * order. An empty selection gives f = 0, g = 0. */
helm_status fwi_misfit_grad_subset(const helm_grid* grid, const double* m_slowness2, int32_t nfreq,
                                   const double* freq_hz, const double* src_weight_reim,
                                   int32_t nsrc_total, int32_t src_begin, int32_t src_end,
                                   const int64_t* src_node, int32_t nrec, const int64_t* rec_node,
                                   const double* d_obs_reim, const uint8_t* pair_mask,
                                   const helm_pml* pml, helm_dtype dtype, const helm_solve_opts* opts,
                                   int32_t max_rhs, double* fg_dev, helm_solve_report* report_host,
                                   void* cuda_stream);

/* ---- off-grid acquisition (helm_acq above): Listing 1 OBJ and FORW_MODEL with interpolated
 * P_s, P_r. Same arguments and outputs as fwi_misfit_grad / fwi_forward with the node-id
 * arrays replaced by `acq` (nsrc_total = number of source points, nrec = receiver points);
 * receivers need not be distinct nodes. */
helm_status fwi_misfit_grad_acq(const helm_grid* grid, const double* m_slowness2, int32_t nfreq,
                                const double* freq_hz, const double* src_weight_reim,
                                int32_t nsrc_total, int32_t src_begin, int32_t src_end,
                                int32_t nrec, const helm_acq* acq, const double* d_obs_reim,
                                const helm_pml* pml, helm_dtype dtype, const helm_solve_opts* opts,
                                int32_t max_rhs, double* fg_dev, helm_solve_report* report_host,
                                void* cuda_stream);
helm_status fwi_forward_acq(const helm_grid* grid, const double* m_slowness2, int32_t nfreq,
                            const double* freq_hz, const double* src_weight_reim,
                            int32_t nsrc_total, int32_t src_begin, int32_t src_end, int32_t nrec,
                            const helm_acq* acq, const helm_pml* pml, helm_dtype dtype,
                            const helm_solve_opts* opts, int32_t max_rhs, double* d_host,
                            helm_solve_report* report_host, void* cuda_stream);

/* ---- inspection entry points (same op; used by the parity tests) ---------------------- */

/* Number of levels and per-level extended sizes (x, y, z). dims_host: [levels][3]. */
helm_status helm_levels(const helm_op* op, int32_t* levels, int64_t* dims_host);

/* Copies level `level`'s 1D tables (complex128, [3 axes][3 = lo,dg,up][Nmax]) for H
 * (adjoint 0) or H^H (adjoint 1), and its model (fp64, extended, x fastest). */
helm_status helm_get_level(const helm_op* op, int32_t level, int32_t adjoint, int64_t nmax,
                           double* tables_host, double* m_host);

/* One ML-GMRES V-cycle z = M_l(b) at level `level` (Alg. 1 + Fig. 3 recursion, fixed
 * counts D14), b and z device arrays of the op's dtype on that level's grid. */
helm_status helm_vcycle(helm_op* op, int32_t level, int32_t adjoint, int32_t nrhs,
                        const void* b_dev, void* z_dev, void* cuda_stream);

/* Level transfer (D13): restrict (R = 2^-d P^T, fine level -> level+1) or prolong-add
 * (x_fine += P x_coarse), dtype of the op. */
helm_status helm_transfer(helm_op* op, int32_t level, int32_t prolong, int32_t nrhs,
                          const void* in_dev, void* out_dev, void* cuda_stream);

/* ---- measurement probes (bench.py) ---------------------------------------------------- */

/* Kernel classes: 0 stencil (y = H x), 1 stencil-residual (r = b - H x, ||r||), 2 norm,
 * 3 arnoldi (stencil + CGS projections; the fused GMRES step), 4 update (+norm, Givens),
 * 5 solution update, 6 copy/convert, 7 restrict, 8 prolong-add, 9 fwi (inject/gather/
 * gradient/fold), 10 setup, 11 vcycle_persist (a whole coarse V-cycle in one grid-synchronous
 * launch, counted at its finer level). */
#define HELM_NCLASS 12

/* When enable != 0, every `stride`-th launch of each class is bracketed by CUDA events
 * recorded on the stream it is launched on. Resets the accumulated statistics. */
helm_status helm_profile(int32_t enable, int32_t stride);

/* Per class (arrays of HELM_NCLASS) for grid level `level` (0 = finest .. 3; 4 = kernels
 * without a level; -1 = all): launches since the last helm_profile call, sampled launches,
 * summed device ms of the sampled launches, summed algorithmic bytes of the sampled
 * launches. Synchronizes on the recorded events. */
helm_status helm_profile_read(int32_t level, int64_t* launches, int64_t* sampled, double* ms,
                              double* bytes);

/* Average device ms per launch of `reps` back-to-back launches of one hot-path kernel on
 * the op's level workspace (contents overwritten): kind 0-4 = stencil modes (0 y = Hx,
 * 1 residual, 2 stencil + CGS projections, 3 fused GMRES step, 4 its last step; nv = step),
 * 10 = solution update (k = nv), 11 = CGS update (j = nv), 12 = norm. Tuning probe only. */
helm_status helm_probe_kernel(helm_op* op, int32_t level, int32_t kind, int32_t nv, int32_t nrhs,
                              int32_t reps, double* ms_per_launch, void* cuda_stream);

/* Total kernel launches issued by this library since it was loaded. */
int64_t     helm_launch_count(void);

/* Peak live workspace of a solve, in vectors of the finest size per RHS. */
double      helm_workspace_vectors(const helm_op* op);

void        helm_destroy(helm_op* op);
const char* helm_last_error(void);
const char* helm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HELM_H */
