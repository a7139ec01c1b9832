// helm.cu — host side of libhelm.so: the helm_op (device-resident model, 1D PML tables,
// level hierarchy, Krylov workspace), the FGMRES / ML-GMRES orchestration and the C ABI
// declared in include/helm.h. All numerics run in the kernels of kernels.cuh.
#include "helm.h"
#include "march2d.cuh"
#include "persist.cuh"
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <tuple>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <set>
#include <type_traits>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

struct HelmErr {
  helm_status st;
  std::string msg;
};

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw HelmErr{e_ == cudaErrorMemoryAllocation ? HELM_ERR_OOM : HELM_ERR_CUDA,       \
                    std::string(#call) + ": " + cudaGetErrorString(e_)};                  \
  } while (0)
#define CKL() CK(cudaGetLastError())
#define REQ(cond, st, msg) \
  do {                     \
    if (!(cond)) throw HelmErr{st, msg}; \
  } while (0)

constexpr int K1 = HELM_KMAX + 1;

// ------------------------------------------------------------------------------ probes
enum KClass { KC_STENCIL = 0, KC_RESID, KC_NORM, KC_DOTS, KC_UPDATE, KC_SOLUPD, KC_COPY, KC_RESTRICT,
              KC_PROLONG, KC_FWI, KC_SETUP, KC_PERSIST };
struct ProbeRec { int cls, level; cudaEvent_t a, b; double bytes; };
struct Prof {
  bool on = false;
  int stride = 1;
  long long launches[HELM_NCLASS][5] = {};   // [class][level 0..3, 4 = no level]
  long long sampled[HELM_NCLASS][5] = {};
  double ms[HELM_NCLASS][5] = {};
  double bytes[HELM_NCLASS][5] = {};
  int cur_level = 4;
  std::vector<ProbeRec> pending;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t cur_a = nullptr;
  bool cur_sampled = false;
};
Prof g_prof;
std::atomic<long long> g_launches{0};   // all threads (fwi evaluations may run concurrently)

cudaEvent_t prof_event() {
  if (!g_prof.pool.empty()) {
    cudaEvent_t e = g_prof.pool.back();
    g_prof.pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
// Launch counted but never timed (setup / FWI bookkeeping kernels).
inline void prof_count(int cls) {
  ++g_launches;
  if (g_prof.on) g_prof.launches[cls][4]++;
}
// Call immediately before a launch on stream st.
inline void prof_begin(int cls, cudaStream_t st, int level) {
  ++g_launches;
  if (!g_prof.on) return;
  g_prof.cur_level = level;
  g_prof.cur_sampled = (g_prof.launches[cls][level]++ % g_prof.stride) == 0;
  if (g_prof.cur_sampled) {
    g_prof.cur_a = prof_event();
    cudaEventRecord(g_prof.cur_a, st);
  }
}
// Call immediately after the launch, with its algorithmic bytes (all RHS).
inline void prof_end(int cls, cudaStream_t st, double bytes) {
  if (!g_prof.on || !g_prof.cur_sampled) return;
  cudaEvent_t b = prof_event();
  cudaEventRecord(b, st);
  g_prof.pending.push_back({cls, g_prof.cur_level, g_prof.cur_a, b, bytes});
  g_prof.cur_sampled = false;
}
void prof_drain() {
  for (auto& r : g_prof.pending) {
    cudaEventSynchronize(r.b);
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    g_prof.ms[r.cls][r.level] += t;
    g_prof.bytes[r.cls][r.level] += r.bytes;
    g_prof.sampled[r.cls][r.level] += 1;
    g_prof.pool.push_back(r.a);
    g_prof.pool.push_back(r.b);
  }
  g_prof.pending.clear();
}
constexpr int TARGET_BLOCKS = 148 * 8;   // 148 SMs x 8 resident 256-thread CTAs

int g_num_sms = 0;
int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  return g_num_sms;
}

template <typename T> T* dalloc(std::vector<void*>& keep, size_t n) {
  void* p = nullptr;
  if (n == 0) n = 1;
  CK(cudaMalloc(&p, n * sizeof(T)));
  keep.push_back(p);
  return static_cast<T*>(p);
}

struct LevelDev {
  int nx = 0, ny = 0, nz = 0;
  long long N = 0;
  double* m64 = nullptr;
  float* m32 = nullptr;
  double2* t64[2][3][3] = {};   // [adjoint][axis][lo,dg,up]
  float2* t32[2][3][3] = {};
  double2* z64[2] = {};         // packed z coefficients per adjoint (k_zpack)
  float2* z32[2] = {};
  // 3D only, for the TMA plane stages: z coefficients padded to 4 per plane, and m with its
  // row pitch nxq rounded up to a 16-B multiple
  double2* zq64[2] = {};
  float2* zq32[2] = {};
  double* mq64 = nullptr;
  float* mq32 = nullptr;
  int nxq = 0;
  int tiles = 0;
};

template <typename R> struct LevelWS {
  cx<R>* SV[K1] = {};   // smoother basis (GMRES), SV[0] also the V-cycle residual; SV[k] raw W
  cx<R>* SW = nullptr;  // second raw-W buffer of the fused GMRES steps (ping-pong with SV[k])
  cx<R>* VB = nullptr;  // V-cycle input copy (scaled basis vector of the caller)
  cx<R>* VX = nullptr;  // level-0 V-cycle output in mixed mode
  cx<R>* FV[K1] = {};   // coarse-solve basis at this level
  cx<R>* FW = nullptr;  // second raw-W buffer of the coarsest (unpreconditioned) GMRES
  cx<R>* FZ[HELM_KMAX] = {};
  cx<R>* Fx = nullptr;
  cx<R>* Fb = nullptr;
  KCtx ctxS{}, ctxC{};
};

}  // namespace

struct helm_op {
  helm_grid grid{};
  helm_pml pml{};
  helm_mlopts ml{};
  helm_dtype dtype = HELM_C128;
  int device = 0;              // CUDA device the op's memory lives on
  int max_rhs = 1;
  double omega = 0.0;          // = omegas[0]
  int nop = 1;                 // operators (frequencies) sharing the geometry (joint batches)
  double omegas[HELM_MAXOP] = {};
  int* rop_d = nullptr;        // per-RHS operator index (device, max_rhs)
  double vref = 0.0;
  int L = 1;
  int dim = 3;
  LevelDev lev[4];
  LevelWS<double> w64[4];
  LevelWS<float> w32[4];
  double2* OV[K1] = {};
  double2* OZ[HELM_KMAX] = {};
  double2* OX = nullptr;
  double2* OB = nullptr;
  KCtx ctxO{};
  int* active_d = nullptr;     // compact list of the active RHS indices (nact entries)
  std::vector<int> alist_dev;  // host mirror of what active_d holds (set_active skips re-uploads)
  int nact = 0;
  RedBuf rb{};
  double* m_int_d = nullptr;     // interior model (fp64)
  std::vector<void*> allocs;
  cudaStream_t st = nullptr;
  int k_inner = 5;
  // accounting (per RHS of the current solve)
  std::vector<int> act_h, alist_h;
  std::vector<double> bytes;
  std::vector<int64_t> mv[4];
  double ws_vectors = 0.0;
  bool apply_only = false;
  // captured level-0 V-cycles (CUDA graphs), keyed by (adjoint, batch size, active count) and
  // the operator signature `gsig` = the batch's omegas: the only values a captured kernel
  // carries BY VALUE besides the key (omega^2 per operator and the operator count); model,
  // tables, Krylov scalars, operator indices and the active list are device memory behind
  // fixed pointers, rewritten in place by op_set_model / build_tables. So graphs stay valid
  // across fwi_* calls and model updates and are only matched by signature.
  struct VGraph {
    int adj, nrhs, nact; cudaGraphExec_t exec; double bytes; long long mv[4]; long long launches;
    std::vector<double> sig;
  };
  std::vector<VGraph> vgraphs;
  std::vector<double> gsig;
  cudaStream_t cap_st = nullptr;   // private stream for graph capture (the caller's may be legacy)
  bool graphs_off = false;         // a capture failed: run V-cycles live from then on
  void clear_graphs() {
    for (auto& g : vgraphs) cudaGraphExecDestroy(g.exec);
    vgraphs.clear();
  }
  void trim_graphs() {             // bounded cache: drop the oldest half
    constexpr size_t cap = 256;
    if (vgraphs.size() < cap) return;
    const size_t drop = vgraphs.size() / 2;
    for (size_t i = 0; i < drop; ++i) cudaGraphExecDestroy(vgraphs[i].exec);
    vgraphs.erase(vgraphs.begin(), vgraphs.begin() + drop);
  }
  ~helm_op() {
    clear_graphs();
    if (cap_st) cudaStreamDestroy(cap_st);
    for (void* p : allocs) cudaFree(p);
  }
};

namespace {

// ------------------------------------------------------------------------------ accounting
double acct(helm_op* op, int level, double bytes_per_rhs, bool matvec, int nrhs) {
  double tot = 0.0;
  for (int r = 0; r < nrhs; ++r)
    if (op->act_h[r]) {
      op->bytes[r] += bytes_per_rhs;
      tot += bytes_per_rhs;
      if (matvec) op->mv[level][r] += 1;
    }
  return tot;
}

int blas_blocks(long long N, int nrhs) {
  long long want = (TARGET_BLOCKS + nrhs - 1) / nrhs;
  long long cap = (N + HELM_RED_THREADS - 1) / HELM_RED_THREADS;
  return (int)std::max(1LL, std::min(want, cap));
}

KCtx make_ctx(std::vector<void*>& keep, int nrhs, int k) {
  KCtx c{};
  c.beta = dalloc<double>(keep, nrhs);
  c.scale = dalloc<double>(keep, (size_t)nrhs * K1);
  c.H = dalloc<double2>(keep, (size_t)nrhs * K1 * HELM_KMAX);
  c.cs = dalloc<double>(keep, (size_t)nrhs * HELM_KMAX);
  c.sn = dalloc<double2>(keep, (size_t)nrhs * HELM_KMAX);
  c.g = dalloc<double2>(keep, (size_t)nrhs * K1);
  c.kact = dalloc<int>(keep, nrhs);
  c.y = dalloc<double2>(keep, (size_t)nrhs * HELM_KMAX);
  c.fc = dalloc<double2>(keep, (size_t)nrhs * K1);
  CK(cudaMemset(c.y, 0, sizeof(double2) * nrhs * HELM_KMAX));
  c.k = k;
  CK(cudaMemset(c.H, 0, sizeof(double2) * nrhs * K1 * HELM_KMAX));
  CK(cudaMemset(c.kact, 0, sizeof(int) * nrhs));
  return c;
}

template <typename R> Geo<R> geo(const helm_op* op, int l, int adj);
template <> Geo<double> geo<double>(const helm_op* op, int l, int adj) {
  const LevelDev& L = op->lev[l];
  Geo<double> g{};
  g.nx = L.nx; g.ny = L.ny; g.nz = L.nz; g.N = L.N;
  g.m = L.m64; g.nop = op->nop; g.rop = op->nop > 1 ? op->rop_d : nullptr;
  for (int o = 0; o < op->nop; ++o) g.w2[o] = op->omegas[o] * op->omegas[o];
  for (int a = 0; a < 3; ++a) { g.lo[a] = L.t64[adj][a][0]; g.dg[a] = L.t64[adj][a][1]; g.up[a] = L.t64[adj][a][2]; }
  g.zpk = L.z64[adj];
  g.st = op->grid.stencil;
  g.adj = adj;
  return g;
}
template <> Geo<float> geo<float>(const helm_op* op, int l, int adj) {
  const LevelDev& L = op->lev[l];
  Geo<float> g{};
  g.nx = L.nx; g.ny = L.ny; g.nz = L.nz; g.N = L.N;
  g.m = L.m32; g.nop = op->nop; g.rop = op->nop > 1 ? op->rop_d : nullptr;
  for (int o = 0; o < op->nop; ++o) g.w2[o] = (float)(op->omegas[o] * op->omegas[o]);
  for (int a = 0; a < 3; ++a) { g.lo[a] = L.t32[adj][a][0]; g.dg[a] = L.t32[adj][a][1]; g.up[a] = L.t32[adj][a][2]; }
  g.zpk = L.z32[adj];
  g.st = op->grid.stencil;
  g.adj = adj;
  return g;
}

// ------------------------------------------------------------------------------ launchers
template <int N = 1, typename F> void dispatch_k(int k, F&& f) {
  if constexpr (N <= HELM_KMAX) {
    if (k == N) { f(std::integral_constant<int, N>{}); return; }
    dispatch_k<N + 1>(k, f);
  } else {
    throw HelmErr{HELM_ERR_ARG, "Krylov dimension out of range"};
  }
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

// Opt-in dynamic shared memory: the limit is ONE setting per (kernel, device) shared by every
// host thread, so it is raised once per (kernel instantiation, device) to the device's
// opt-in maximum (227 KB on B200) and never lowered — no thread can shrink a limit another
// thread's launch relies on. Cheap after the first call (a set lookup).
std::mutex g_optin_mu;
std::set<std::pair<const void*, int>> g_optin_done;   // (kernel, device)
template <typename K> void ensure_smem_optin(K kern) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  const std::pair<const void*, int> key{reinterpret_cast<const void*>(kern), dev};
  std::lock_guard<std::mutex> lk(g_optin_mu);
  if (g_optin_done.count(key)) return;
  int optin = 0;
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
  g_optin_done.insert(key);
}
int smem_optin() {
  static const int v = [] {
    int dev = 0, o = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&o, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return o;
  }();
  return v;
}

// Hot-path launches use programmatic dependent launch (see common.cuh pdl_wait): the
// launch and block scheduling of each kernel overlap the tail of its predecessor.
// HELM_PDL=0 disables it (plain stream order).
template <typename... KArgs, typename... Args>
void pdl_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  static const bool on = env_int("HELM_PDL", 0) != 0;   // measured: slower on B200 here (opt-in)
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = on ? 1 : 0;
  CK(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

template <int N = 0, typename F> void dispatch_k0(int k, F&& f) {
  if constexpr (N < HELM_KMAX) {
    if (k == N) { f(std::integral_constant<int, N>{}); return; }
    dispatch_k0<N + 1>(k, f);
  } else {
    throw HelmErr{HELM_ERR_ARG, "Krylov step out of range"};
  }
}

// Plane-kernel configuration: 32x8 row tiles, one row per thread (3D: x,y of one RHS; 2D:
// 32 x-points x 8 right-hand sides). The ring depth S is a launch parameter: the largest
// S <= 12 whose ring fits the shared-memory budget of `occ_target` CTAs per SM (default 4;
// HELM_PLANE_OCC / HELM_PLANE_S override, for tuning).
// Rows per thread: 4 for the plain matvec (halves the per-plane fixed cost per point: measured
// +15-35 % on the cfg5 sweep, profiles/r01/matvec_py_ab.txt), 2 for MODE 1/2, 1 for the
// register-heavy Arnoldi steps.
#ifndef HELM_PY34
#define HELM_PY34 2   // Arnoldi steps: 2 rows per thread (3D solve A/B: c128 -2..4 %, c64 -15 %)
#endif
template <int MODE, bool YC> constexpr int plane_py() { return !YC ? 1 : (MODE == 0 ? 4 : (MODE < 3 ? 2 : HELM_PY34)); }

// Ring depth S = smem budget / (occupancy target x stage bytes). Measured on the cfg5 matvec
// (profiles/r01/matvec_occ_ab.txt): complex64 stages are half the bytes, and its kernels are
// issue-latency bound, so it wants more resident CTAs (8) over a deeper ring; complex128 4.
// The 64-thread matvec CTAs (PY = 4) want 12 (complex64) / 6 (complex128).
struct PlaneTune { int occ_target, s_fixed; };
template <typename R, int PY> const PlaneTune& plane_tune() {
  static const PlaneTune t{std::max(1, env_int("HELM_PLANE_OCC", PY == 4 ? (sizeof(R) == 4 ? 12 : 6) : (sizeof(R) == 4 ? 8 : 4))),
                           env_int("HELM_PLANE_S", 0)};
  return t;
}

// TMA tensor map of a batched complex vector [rhs][z][y][x] viewed as 8-byte words (x
// fastest), box = the 34 x 10 halo'd tile (x0-1 .. x0+32, y0-1 .. y0+8) of one plane of one
// RHS. Needs a 16-B aligned base and row pitch (always for complex128; even nx for
// complex64). Returns false when TMA is not used for the array.
PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

template <typename R>
bool make_tile_map(CUtensorMap* m, const void* base, int nx, int ny, int nz, int nrhs, int by = 8) {
  auto enc = tma_encoder();
  if (!enc || !base || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
  // the tensor element is an 8-byte word (one complex64, or half a complex128): TMA only
  // moves bytes, and 8-byte elements keep the 16-B row-pitch rule satisfiable for complex64
  const cuuint64_t ce = sizeof(cx<R>) / 8;
  if ((ce * (cuuint64_t)nx * 8) % 16) return false;
  cuuint64_t dims[4] = {ce * (cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz, (cuuint64_t)nrhs};
  cuuint64_t strides[3] = {ce * (cuuint64_t)nx * 8, ce * (cuuint64_t)nx * ny * 8, ce * (cuuint64_t)nx * ny * nz * 8};
  // box = the tile plus its x halo, starting 16-B aligned (PlaneSmem::XO): 34 complex128 or
  // 36 complex64 per row
  const cuuint32_t xo = (cuuint32_t)(16 / sizeof(cx<R>));
  cuuint32_t box[4] = {(cuuint32_t)((32 + 2 * xo) * ce), (cuuint32_t)(by + 2), 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  const CUresult rc = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void*>(base), dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return rc == CUDA_SUCCESS;
}

// TMA maps of the per-plane operands that are not halo'd: m (16-B pitched copy, box = the
// 32 x 8 own points of a tile) and the padded z-coefficient rows (box = one plane's 4 entries).
template <typename R>
bool make_m_map(CUtensorMap* m, const R* mq, int nxq, int ny, int nz, bool halo = false, int by = 8) {
  auto enc = tma_encoder();
  if (!enc || !mq) return false;
  cuuint64_t dims[3] = {(cuuint64_t)nxq, (cuuint64_t)ny, (cuuint64_t)nz};
  cuuint64_t strides[2] = {(cuuint64_t)nxq * sizeof(R), (cuuint64_t)nxq * ny * sizeof(R)};
  // own points (32 x 8), or for the OPT stencils' mass term the halo'd tile starting 16 B
  // before the interior (PlaneSmem::XOm) and one row above: (32 + 2 XOm) x 10
  const cuuint32_t xom = (cuuint32_t)(16 / sizeof(R));
  cuuint32_t box[3] = {halo ? 32 + 2 * xom : 32, (cuuint32_t)(halo ? by + 2 : by), 1};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(m, sizeof(R) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
             const_cast<R*>(mq), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
template <typename R>
bool make_z_map(CUtensorMap* m, const cx<R>* zq, int nz, int nop) {
  auto enc = tma_encoder();
  if (!enc || !zq) return false;
  const cuuint64_t w = 4 * sizeof(cx<R>) / 8;   // 8-byte words per plane row
  cuuint64_t dims[2] = {w, (cuuint64_t)nz * nop};
  cuuint64_t strides[1] = {w * 8};
  cuuint32_t box[2] = {(cuuint32_t)w, 1};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<cx<R>*>(zq), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// 2D march strips (march2d.cuh TMA feed): operand [rhs][z][x] as 8-byte words, box = one
// 32-point strip row; m's padded copy [z][xq], box = 34 reals (starting one point before the
// strip's first lane, 16-B aligned).
template <typename R>
bool make_strip_map(CUtensorMap* m, const void* base, int nx, int nz, int nrhs) {
  auto enc = tma_encoder();
  if (!enc || !base || (reinterpret_cast<uintptr_t>(base) & 15) || sizeof(cx<R>) != 16) return false;
  const cuuint64_t ce = sizeof(cx<R>) / 8;
  cuuint64_t dims[3] = {ce * (cuuint64_t)nx, (cuuint64_t)nz, (cuuint64_t)nrhs};
  cuuint64_t strides[2] = {ce * (cuuint64_t)nx * 8, ce * (cuuint64_t)nx * nz * 8};
  cuuint32_t box[3] = {(cuuint32_t)(32 * ce), 1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
template <typename R>
bool make_mstrip_map(CUtensorMap* m, const R* mq, int nxq, int nz) {
  auto enc = tma_encoder();
  if (!enc || !mq) return false;
  cuuint64_t dims[2] = {(cuuint64_t)nxq, (cuuint64_t)nz};
  cuuint64_t strides[1] = {(cuuint64_t)nxq * sizeof(R)};
  cuuint32_t box[2] = {34, 1};
  cuuint32_t es[2] = {1, 1};
  return enc(m, sizeof(R) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
             const_cast<R*>(mq), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
template <typename R> const R* level_mq(const LevelDev& L);
template <> const double* level_mq<double>(const LevelDev& L) { return L.mq64; }
template <> const float* level_mq<float>(const LevelDev& L) { return L.mq32; }
template <typename R> const cx<R>* level_zq(const LevelDev& L, int adj);
template <> const double2* level_zq<double>(const LevelDev& L, int adj) { return L.zq64[adj]; }
template <> const float2* level_zq<float>(const LevelDev& L, int adj) { return L.zq32[adj]; }

struct PlaneCfg { int S = 0, occ = 0, nf = 0; size_t smem = 0; };

// Split of a group's T tiles x nz planes over its CTAs (one resident wave of G CTAs over
// all groups): the z-chunk count minimising waves x (chunk planes + 2 halo planes).
struct PlaneSplit { int cpg, nzc, zlen; };
PlaneSplit plane_split(int groups, long long G, int T, int nz, int hw10 = 20) {
  const long long cpg0 = std::max(1LL, G / groups);
  long long best = -1;
  PlaneSplit r{1, 1, nz};
  for (int n = 1; n <= nz; ++n) {
    const int zl = (nz + n - 1) / n, nzc = (nz + zl - 1) / zl;
    if (nzc != n) continue;
    const long long items = (long long)T * nzc;
    const long long waves = (items + cpg0 - 1) / cpg0;
    const long long cost = waves * (10LL * zl + hw10);   // hw10: per-item overhead in tenths of a plane
    if (best < 0 || cost < best) { best = cost; r = PlaneSplit{(int)std::min(cpg0, items), nzc, zl}; }
  }
  return r;
}

// Launch with exactly one resident wave (groups x cpg CTAs, see stencil.cuh).
template <typename R, int MODE, int NV, bool YC, int PY = plane_py<MODE, YC>(), bool SPLIT = false, int ST = 0,
          int BY = 8>
void run_plane(PlaneArgs<R>& a, int groups, long long units, cudaStream_t st) {
  if constexpr (MODE == 0 && PY == 4 && ST == 0 && BY == 8) {   // A/B switches of the matvec
    static const bool py2 = env_int("HELM_PLANE_PY", 4) == 2;    // two rows per thread
    if (py2) { run_plane<R, MODE, NV, YC, 2>(a, groups, units, st); return; }
    if (a.by == 16) {                                             // launch_plane chose 16-row tiles
      run_plane<R, MODE, NV, YC, 4, false, 0, 16>(a, groups, units, st);
      return;
    }
  }
  using Sh = PlaneShape<MODE, NV>;
  constexpr int NT = 32 * BY / PY;
  constexpr size_t sb = PlaneSmem<R, 32, BY, Sh::NX, Sh::NP, YC, SPLIT, ST == 1>::stage_bytes;
  void (*kern)(PlaneArgs<R>) = nullptr;
  if constexpr (PY == 1 && MODE >= 3 && ST == 0) kern = k_plane_o2<R, 32, BY, PY, MODE, NV, YC, SPLIT, ST>;
  else kern = k_plane<R, 32, BY, PY, MODE, NV, YC, SPLIT, ST>;
  static const PlaneCfg cfg = [&] {
    PlaneCfg c;
    const PlaneTune& t = plane_tune<R, PY>();
    if constexpr (SPLIT) {
      // split-ring fused steps: D raw stages + nf formed slots per CTA at `occ` CTAs per SM
      // (default 2 complex128 / 3 complex64; HELM_SPLIT_OCC, HELM_SPLIT_D override)
      const size_t fb = FormSlot<R, 32, 8, YC>::bytes;
      const int occ_t = std::max(1, env_int("HELM_SPLIT_OCC", sizeof(R) == 8 ? 2 : 3));
      const long long budget = (long long)(smem_optin() - 1024) / occ_t;
      c.nf = 4;
      long long d = (budget - 4 * (long long)fb) / (long long)(sb + 8);
      if (d < 2) { c.nf = 3; d = (budget - 3 * (long long)fb) / (long long)(sb + 8); }
      const int dfix = env_int("HELM_SPLIT_D", 0);
      c.S = dfix >= 2 ? dfix : (int)std::max(2LL, std::min(12LL, d));
      c.smem = c.S * sb + c.nf * fb + 8 * c.S;
    } else {
      // the first fused step (one halo'd tile, S = 7 at the default target 4) is faster with a
      // shallower ring at 5 CTAs per SM: cfg4 level 0 701 -> 654 us (profiles/r02/ab_r2v)
      const int occ_t = (MODE == 3 && NV == 0 && !env_int("HELM_PLANE_OCC", 0) && sizeof(R) == 8) ? 5 : t.occ_target;
      c.S = t.s_fixed >= 4 ? std::min(t.s_fixed, 12) : (int)std::min<size_t>(12, (220 * 1024) / (occ_t * sb));
      c.S = std::max(c.S, 4);
      c.smem = c.S * sb + 8 * c.S;   // ring + one mbarrier per stage (TMA)
    }
    ensure_smem_optin(kern);
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.occ, kern, NT, c.smem));
    if (c.occ < 1) throw HelmErr{HELM_ERR_STATE, "plane kernel does not fit on an SM"};
    if (env_int("HELM_DEBUG", 0)) {
      cudaFuncAttributes fa{};
      cudaFuncGetAttributes(&fa, kern);
      std::fprintf(stderr, "[helm] plane R=%zu mode=%d nv=%d py=%d split=%d S=%d nf=%d smem=%zu regs=%d occ=%d\n", sizeof(R),
                   MODE, NV, PY, (int)SPLIT, c.S, c.nf, c.smem, fa.numRegs, c.occ);
    }
    return c;
  }();
  ensure_smem_optin(kern);   // this device (the cached configuration may come from another one)
  // plane z-1 in registers (stencil.cuh PREV): same-box A/B (profiles/r02/probe_prev_ab.txt) at
  // cfg4: residual and fused steps at level 1 +7-19 %, level-0 residual +23 %, level-0 steps
  // 1-2 -7 %. The configs[4] matvec (MODE 0), 24-cell sweep (profiles/r02/ab_r2u): complex64
  // gains at every size (512^3 b = 1: 0.69 -> 0.83 of measured HBM, 256^3 b = 4: 0.57 -> 0.65),
  // complex128 gains up to 256^3 (+PML; b = 4: 0.74 -> 0.89) and loses at 384^3-512^3
  // (0.85 -> 0.76), so MODE 0 uses it for complex64 and for grids of <= 24 M points.
  // HELM_PREV: 1 (default) as above, 2 every mode, 0 none.
  static const int prev_mode = env_int("HELM_PREV", 1);
  const bool mv_prev = sizeof(R) == 4 || a.g.N <= 24LL * 1000 * 1000;
  a.prev = prev_mode == 2 || (prev_mode == 1 && (MODE != 0 || mv_prev));
  // continuous ring across a CTA's items (fused steps with TMA-only stages; HELM_CONT=0: per-item
  // ring fills, the round-2 kernel). An item then costs its planes plus the two halo planes'
  // loads and forming, not a ring refill: HELM_CONT_HW10 = that overhead in tenths of a plane.
  static const int cont_on = env_int("HELM_CONT", 1);
  static const int cont_hw10 = env_int("HELM_CONT_HW10", 10);
  static const int ctared = env_int("HELM_CTA_RED", 1);   // CTA-level reduction tail (stencil.cuh)
  a.ctared = ctared;
  a.cont = (MODE >= 3 && !SPLIT && ST == 0 && cont_on && a.tma && a.tmq && a.prev) ? 1 : 0;
  PlaneSplit sp = plane_split(groups, (long long)num_sms() * cfg.occ, a.ntx * a.nty, a.g.nz, a.cont ? cont_hw10 : 20);
  static const int nzc_fix = env_int("HELM_PLANE_NZC", 0);   // tuning: force the z-chunk count
  if (nzc_fix > 0) {
    sp.zlen = (a.g.nz + nzc_fix - 1) / nzc_fix;
    sp.nzc = (a.g.nz + sp.zlen - 1) / sp.zlen;
    sp.cpg = (int)std::min<long long>(std::max(1LL, (long long)num_sms() * cfg.occ / groups), (long long)a.ntx * a.nty * sp.nzc);
  }
  a.cpg = sp.cpg; a.nzc = sp.nzc; a.zlen = sp.zlen;
  a.S = cfg.S;
  a.nf = cfg.nf;
  if (env_int("HELM_DEBUG", 0) > 1)
    std::fprintf(stderr, "[helm] plane launch mode=%d nv=%d split=%d cont=%d groups=%d cpg=%d nzc=%d zlen=%d tiles=%d\n", MODE,
                 NV, (int)SPLIT, a.cont, groups, sp.cpg, sp.nzc, sp.zlen, a.ntx * a.nty);
  const long long cpg = sp.cpg;
  pdl_launch(kern, dim3((unsigned)(groups * cpg)), dim3(NT), cfg.smem, st, a);
}

// Largest number of operators (frequencies) one 2D joint batch may hold: the march kernel
// keeps 3 z coefficients per plane and operator in shared memory next to a ring of at least
// 3 stages of its widest mode (the last fused GMRES step, HELM_KMAX basis tiles).
template <typename R> int march_max_ops(int nz) {
  const long long ring = 4LL * 3 * MarchShape<R, 4, HELM_KMAX - 1>::stage_bytes;
  const long long per_op = 3LL * nz * sizeof(cx<R>);
  return (int)std::max(0LL, std::min<long long>(HELM_MAXOP, (smem_optin() - ring - 16) / per_op));
}

// 2D: register z-march kernel (march2d.cuh), one warp per (RHS, 30-point strip, z-chunk)
// item; exactly one resident wave of warps, split evenly over the active right-hand sides.
// The per-lane cp.async ring holds S planes (S-2 in flight): S is the largest depth <= 16
// whose rings fit a shared-memory budget of ~220 KB / occ_target CTAs (5 by default: a
// shallower ring for up to 20 warps per SM; HELM_MARCH_OCC / HELM_MARCH_S override for tuning).
template <typename R, int MODE, int NV, int ST = 0, bool TM = false>
void run_march_t(MarchArgs<R>& a, cudaStream_t st);

// 2D march launch: the TMA-fed ring for complex128 when every operand map could be encoded
// (a.tma, set by launch_plane; HELM_MARCH_TMA=0: per-lane cp.async), else per-lane cp.async.
template <typename R, int MODE, int NV, int ST = 0>
void run_march(MarchArgs<R>& a, cudaStream_t st) {
  if constexpr (sizeof(R) == 8) {
    if (a.tma) { run_march_t<R, MODE, NV, ST, true>(a, st); return; }
  }
  run_march_t<R, MODE, NV, ST, false>(a, st);
}

template <typename R, int MODE, int NV, int ST, bool TM>
void run_march_t(MarchArgs<R>& a, cudaStream_t st) {
  auto kern = k_march2d<R, MODE, NV, ST, TM>;
  constexpr int SB = MarchShape<R, MODE, NV, TM>::stage_bytes;
  const size_t zbytes = TM ? ((size_t)3 * a.g.nz * a.g.nop * sizeof(cx<R>) + 127) / 128 * 128
                           : ((size_t)3 * a.g.nz * a.g.nop * sizeof(cx<R>) + 15) / 16 * 16;
  // bench A/B (march2d_variants_ab.txt): complex128 5 vs 4 = +3-5 %; complex64 (half the stage
  // bytes) 8 vs 5 = +8 % on the level-1 fused steps
  static const int occ_t = std::max(1, env_int("HELM_MARCH_OCC", sizeof(R) == 4 ? 8 : 5));
  static const int s_fix = env_int("HELM_MARCH_S", 0);
  int S = s_fix >= 3 ? s_fix : (int)(((220 * 1024) / occ_t - (long long)zbytes) / (4 * (SB + (TM ? 8 : 0))));
  S = std::max(3, std::min(S, 16));
  const size_t smem = zbytes + (size_t)4 * S * SB + (TM ? (size_t)4 * S * 8 : 0);
  // the z table of every operator of the batch lives in shared memory (fwi_run closes joint
  // batches before this limit, march_max_ops); a grid too deep for even one operator fails here
  REQ(smem <= (size_t)smem_optin(), HELM_ERR_SHAPE,
      "2D grid too deep for the march kernel: nz_ext x operators = " + std::to_string(a.g.nz * a.g.nop) +
          " z-table entries exceed shared memory");
  struct Cfg { size_t smem = 0; int occ = 0; };
  thread_local Cfg cache[4];   // small per-thread cache of (smem -> occupancy)
  ensure_smem_optin(kern);
  int occ = 0;
  for (auto& c : cache)
    if (c.smem == smem) { occ = c.occ; break; }
  if (!occ) {
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128, smem));
    if (occ < 1) throw HelmErr{HELM_ERR_STATE, "march kernel does not fit on an SM"};
    thread_local int next = 0;
    cache[next] = Cfg{smem, occ};
    next = (next + 1) % 4;
    if (env_int("HELM_DEBUG", 0)) {
      cudaFuncAttributes fa{};
      cudaFuncGetAttributes(&fa, kern);
      std::fprintf(stderr, "[helm] march2d R=%zu mode=%d nv=%d tma=%d S=%d smem=%zu regs=%d occ=%d warps/SM=%d\n",
                   sizeof(R), MODE, NV, (int)TM, S, smem, fa.numRegs, occ, occ * 4);
    }
  }
  a.S = S;
  const long long W = (long long)num_sms() * occ * 4;
  const int wpr = (int)std::max(1LL, W / a.nrhs);
  const int nz = a.g.nz;
  long long best = -1;
  int nzc_b = 1, zl_b = nz;
  // z-chunk count minimising rounds x (chunk + halo + ring fill) + the slot reduction of the
  // last-arriving warp (one L2 round trip per 128 warps of the RHS, worth ~red_w plane steps):
  // small late-cycle batches otherwise spread one RHS over thousands of 1-plane items
  static const int red_w = env_int("HELM_MARCH_RED", 8);   // bench A/B: 8 vs 0 = +3 %
  for (int n = 1; n <= nz; ++n) {
    const int zl = (nz + n - 1) / n, nzc = (nz + zl - 1) / zl;
    if (nzc != n) continue;
    const long long items = (long long)a.nstrip * nzc;
    const long long used = std::min<long long>(wpr, items);
    const long long cost = ((items + wpr - 1) / wpr) * (zl + 2 + S / 2) + red_w * ((used + 127) / 128);
    if (best < 0 || cost < best) { best = cost; nzc_b = nzc; zl_b = zl; }
  }
  static const int nzc_fix = env_int("HELM_MARCH_NZC", 0);   // tuning: force the z-chunk count
  if (nzc_fix > 0) { zl_b = (nz + nzc_fix - 1) / nzc_fix; nzc_b = (nz + zl_b - 1) / zl_b; }
  a.nzc = nzc_b; a.zlen = zl_b;
  a.wpr = (int)std::min<long long>(wpr, (long long)a.nstrip * nzc_b);
  if (env_int("HELM_DEBUG", 0) > 1)
    std::fprintf(stderr, "[helm] march2d nx=%d nz=%d nrhs=%d W=%lld wpr=%d nstrip=%d nzc=%d zlen=%d S=%d\n", a.g.nx, nz,
                 a.nrhs, W, a.wpr, a.nstrip, a.nzc, a.zlen, S);
  const long long warps = (long long)a.nrhs * a.wpr;
  pdl_launch(kern, dim3((unsigned)((warps + 3) / 4)), dim3(128), smem, st, a);
}

// Plane-streaming stencil (stencil.cuh). mode 0: y = s H x; 1: y = b - H x (+cycle start);
// 2: y = s H x with the fused projections h_ij = <V_i, y>, i < nv (nv = j + 1);
// 3: fused Arnoldi step nv of unpreconditioned GMRES (x = raw W or V_0, V = basis, vout);
// 4: its last step (Y not stored, the last column finalised by Pythagoras).
// Does the last fused Arnoldi step of a GMRES cycle store V_{k-1}? 2D (march kernel): yes.
// 3D: no (HELM_LASTV=1: yes, the round-2 schedule) — the solution update reforms it from
// W = Y_{k-2} and V_0..V_{k-2} with the forming coefficients the step's epilogue saves
// (KCtx::fc), one vector write less per restart cycle.
bool last_v_stored(const helm_op* op, int l) {
  static const bool lastv = env_int("HELM_LASTV", 0) != 0;
  return lastv || op->lev[l].ny == 1;
}

template <typename R>
void launch_plane(helm_op* op, int l, int adj, int mode, int nrhs, const cx<R>* x, cx<R>* y, const cx<R>* b,
                  const VPtrs<R>* V, int nv, const double* xscale, const int* kact, int j, const KCtx& ctx,
                  cx<R>* vout = nullptr) {
  if (!op->nact) return;
  const int cls = mode == 0 ? KC_STENCIL : (mode == 1 ? KC_RESID : KC_DOTS);
  const double Sc = sizeof(cx<R>), Sr = sizeof(R);
  double per;
  if (mode == 0) per = 2 * Sc + Sr;
  else if (mode == 1) per = 3 * Sc + Sr;
  else if (mode == 2) per = (2 + nv) * Sc + Sr;
  else if (mode == 3) per = (nv == 0 ? 2 : nv + 3) * Sc + Sr;
  else per = (nv == 0 ? 1 : nv + (last_v_stored(op, l) ? 2 : 1)) * Sc + Sr;   // last step: Y (3D: nor V_nv) not stored
  if (op->lev[l].ny == 1) {   // 2D: register z-march
    MarchArgs<R> m{};
    m.g = geo<R>(op, l, adj);
    m.x = x; m.y = y; m.b = b; m.vout = vout;
    if (V) m.V = *V;
    m.xscale = xscale; m.sstride = K1; m.active = op->active_d; m.kact = kact; m.jstep = j;
    m.jskip = mode >= 3 ? std::max(nv - 1, 0) : j;
    m.nrhs = op->nact; m.ctx = ctx; m.rb = op->rb;
    m.nstrip = (m.g.nx + 29) / 30;
    m.tma = 0;
    if constexpr (sizeof(R) == 8) {
      // TMA-fed march ring (complex128): strip rows of every streamed operand and m's padded
      // copy. Same-box A/B at cfg2 (profiles/r02/ab_r2x, 150 RHS): TMA wins with three or more
      // streamed operands on the large levels (level 0 fused steps 2-4 -5-7 %, FGMRES 5 -13 %)
      // and loses with one or two (matvec, residual, steps 0-1: +8-15 %; 126 vs 96 registers)
      // and on the small coarsest level. HELM_MARCH_TMA: 1 (default) that rule, 2 always, 0 never.
      static const int mtma = env_int("HELM_MARCH_TMA", 1);
      const LevelDev& Lv = op->lev[l];
      const int nb = (mode == 2 || mode >= 3) ? nv : 0;
      const int nxo = 1 + nb + (mode == 1 ? 1 : 0);
      const bool want = mtma == 2 || (mtma == 1 && nxo >= 3 && m.g.N * (long long)op->nact >= 2000000LL);
      if (want && Lv.mq64) {
        bool ok = make_strip_map<R>(&m.tm[0], x, m.g.nx, m.g.nz, nrhs);
        for (int i = 0; i < nb && ok; ++i) ok = make_strip_map<R>(&m.tm[1 + i], m.V.p[i], m.g.nx, m.g.nz, nrhs);
        if (mode == 1 && ok) ok = make_strip_map<R>(&m.tm[1 + nb], b, m.g.nx, m.g.nz, nrhs);
        ok = ok && make_mstrip_map<R>(&m.tmm, Lv.mq64, Lv.nxq, Lv.nz);
        m.tma = ok ? 1 : 0;
      }
    }
    prof_begin(cls, op->st, l);
    if (op->grid.stencil == HELM_OPT) {   // R34: the 9-point stencil
      if (mode == 0) run_march<R, 0, 0, 1>(m, op->st);
      else if (mode == 1) run_march<R, 1, 0, 1>(m, op->st);
      else if (mode == 2) dispatch_k(nv, [&](auto c) { run_march<R, 2, decltype(c)::value, 1>(m, op->st); });
      else if (mode == 3) dispatch_k0(nv, [&](auto c) { run_march<R, 3, decltype(c)::value, 1>(m, op->st); });
      else dispatch_k0(nv, [&](auto c) { run_march<R, 4, decltype(c)::value, 1>(m, op->st); });
    } else if (mode == 0) run_march<R, 0, 0>(m, op->st);
    else if (mode == 1) run_march<R, 1, 0>(m, op->st);
    else if (mode == 2) dispatch_k(nv, [&](auto c) { run_march<R, 2, decltype(c)::value>(m, op->st); });
    else if (mode == 3) dispatch_k0(nv, [&](auto c) { run_march<R, 3, decltype(c)::value>(m, op->st); });
    else dispatch_k0(nv, [&](auto c) { run_march<R, 4, decltype(c)::value>(m, op->st); });
    CKL();
    prof_end(cls, op->st, acct(op, l, per * m.g.N, true, nrhs));
    return;
  }
  PlaneArgs<R> a{};
  a.g = geo<R>(op, l, adj);
  a.x = x; a.y = y; a.b = b; a.vout = vout;
  if (V) a.V = *V;
  a.xscale = xscale; a.sstride = K1; a.active = op->active_d; a.kact = kact; a.jstep = j;
  a.jskip = mode >= 3 ? std::max(nv - 1, 0) : j;
  a.nrhs = nrhs; a.ctx = ctx; a.rb = op->rb;
  a.wlast = last_v_stored(op, l) ? 1 : 0;
  a.ntx = (a.g.nx + 31) / 32;
  // tile height: 8 rows; the plain matvec can use 16 (HELM_MATVEC_BY=16: half the y-halo
  // overhead per point, one CTA covers 32 x 16 points)
  static const int mv_by = env_int("HELM_MATVEC_BY", 8) == 16 ? 16 : 8;
  const int by = (mode == 0 && op->grid.stencil == HELM_STD2) ? mv_by : 8;
  a.nty = (a.g.ny + by - 1) / by;
  a.by = by;
  const int groups = op->nact;
  // TMA for the halo'd tiles when every halo'd operand can be described (HELM_TMA=0: cp.async)
  static const bool tma_on = env_int("HELM_TMA", 1) != 0;
  const bool opt = op->grid.stencil == HELM_OPT;
  a.tma = 0;
  if (tma_on || opt) {
    const int nxt = mode >= 3 ? nv + 1 : 1;
    bool ok = true;
    for (int t = 0; t < nxt && ok; ++t)
      ok = make_tile_map<R>(&a.tm[t], t == 0 ? (const void*)x : (const void*)a.V.p[t - 1], a.g.nx, a.g.ny, a.g.nz, nrhs,
                            by);
    a.tma = ok ? 1 : 0;
    static const bool tmq_on_env = env_int("HELM_TMA_MZ", 1) != 0;
    const bool tmq_on = tmq_on_env || opt;
    const LevelDev& Lv = op->lev[l];
    a.tmq = a.tma && tmq_on && make_m_map<R>(&a.tmm, level_mq<R>(Lv), Lv.nxq, Lv.ny, Lv.nz, opt, by) &&
            make_z_map<R>(&a.tmz, level_zq<R>(Lv, adj), Lv.nz, op->nop);
  }
  const long long units = (long long)a.ntx * a.nty * a.g.nz;
  if (opt) {   // R35: every mode of the plane kernel on the 27-point stencil (single ring, TMA)
    REQ(a.tma && a.tmq, HELM_ERR_SHAPE,
        "the OPT stencil needs TMA-describable rows on every level (complex64: even extended nx)");
    prof_begin(cls, op->st, l);
    // one row per thread (256-thread CTAs): the 27-point sum for 4 rows per thread needed 255
    // registers and 400 B of stack (measured 14 Gpts/s at 512^3 c128)
    if (mode == 0) run_plane<R, 0, 0, true, 1, false, 1>(a, groups, units, op->st);
    else if (mode == 1) run_plane<R, 1, 0, true, 1, false, 1>(a, groups, units, op->st);
    else if (mode == 2)
      dispatch_k(nv, [&](auto c) { run_plane<R, 2, decltype(c)::value, true, 1, false, 1>(a, groups, units, op->st); });
    else if (mode == 3) dispatch_k0(nv, [&](auto c) { run_plane<R, 3, decltype(c)::value, true, 1, false, 1>(a, groups, units, op->st); });
    else dispatch_k0(nv, [&](auto c) { run_plane<R, 4, decltype(c)::value, true, 1, false, 1>(a, groups, units, op->st); });
    CKL();
    prof_end(cls, op->st, acct(op, l, per * a.g.N, true, nrhs));
    return;
  }
  prof_begin(cls, op->st, l);
  if (mode == 0) run_plane<R, 0, 0, true>(a, groups, units, op->st);
  else if (mode == 1) run_plane<R, 1, 0, true>(a, groups, units, op->st);
  else if (mode == 2) dispatch_k(nv, [&](auto c) { run_plane<R, 2, decltype(c)::value, true>(a, groups, units, op->st); });
  else {
    // fused steps that form v_nv (nv > 0): split raw / formed rings (stencil.cuh FormSlot) when
    // every operand comes by TMA. Same-box A/B (profiles/r02/probe_split_ab.txt): with fewer,
    // deeper CTAs the split ring loses on steps 1-3 (the per-plane wait/form/compute chain of a
    // CTA is the limit, not bytes in flight) and won on the last complex128 step (NV = 4) while
    // that step stored V_4. Since the last step stores nothing (last_v_stored), the single ring
    // wins there too (profiles/r02/ab_r2q: cfg4 level 0 2334 -> 2001 us, level 1 325 -> 280 us,
    // level 2 64 -> 58 us). HELM_SPLIT: 0 (default) off, 1 the last complex128 step, 2 all.
    static const int split_mode = env_int("HELM_SPLIT", 0);
    const bool split = a.tma && a.tmq && nv > 0 &&
                       (split_mode == 2 || (split_mode == 1 && sizeof(R) == 8 && mode == 4 && nv >= 4));
    auto go = [&](auto c) {
      constexpr int NVc = decltype(c)::value;
      if constexpr (NVc > 0) {
        if (split) {
          if constexpr (NVc >= 4) {
            // one row per thread (256-thread CTAs, 2 per SM): twice the warps of the 2-row
            // split kernel for the last step's five-tile stages (HELM_SPLIT_PY=1, A/B)
            static const bool py1 = env_int("HELM_SPLIT_PY", 2) == 1;
            if (py1 && mode == 4) {
              run_plane<R, 4, NVc, true, 1, true>(a, groups, units, op->st);
              return;
            }
          }
          if (mode == 3) run_plane<R, 3, NVc, true, plane_py<3, true>(), true>(a, groups, units, op->st);
          else run_plane<R, 4, NVc, true, plane_py<4, true>(), true>(a, groups, units, op->st);
          return;
        }
      }
      if constexpr (NVc >= 3 && NVc <= 4) {
        // one row per thread (256-thread CTAs, <= 128 registers, two per SM) for the steps
        // with four or five halo'd tiles per stage, whose 2-row CTAs fit only two per SM
        // (8 warps). HELM_FUSED_PY1 = the first step NV that uses it (default 3), MODE 3 only
        // unless HELM_FUSED_PY1_LAST=1. Same-box A/B (profiles/r02/ab_r2s): step 3 at cfg4
        // level 1 253 -> 243 us, level 0 1897 -> 1861 us; the last step (stores nothing,
        // fewer operands per point) loses: 277 -> 292 us.
        static const int py1_from = env_int("HELM_FUSED_PY1", 3);
        static const bool py1_last = env_int("HELM_FUSED_PY1_LAST", 0) != 0;
        if (nv >= py1_from && (mode == 3 || py1_last)) {
          if (mode == 3) run_plane<R, 3, NVc, true, 1>(a, groups, units, op->st);
          else run_plane<R, 4, NVc, true, 1>(a, groups, units, op->st);
          return;
        }
      }
      if (mode == 3) run_plane<R, 3, NVc, true>(a, groups, units, op->st);
      else run_plane<R, 4, NVc, true>(a, groups, units, op->st);
    };
    dispatch_k0(nv, go);
  }
  CKL();
  prof_end(cls, op->st, acct(op, l, per * a.g.N, true, nrhs));
}

template <typename R>
void launch_stencil(helm_op* op, int l, int adj, int mode, int nrhs, const cx<R>* x, cx<R>* y,
                    const cx<R>* b, const double* xscale, const int* kact, int j, const KCtx& ctx) {
  launch_plane<R>(op, l, adj, mode, nrhs, x, y, b, nullptr, 0, xscale, kact, j, ctx);
}

template <typename R> VPtrs<R> vptrs(cx<R>* const* V, const cx<R>* v0, int n) {
  VPtrs<R> p{};
  for (int i = 0; i < n && i < K1; ++i) p.p[i] = (i == 0 && v0) ? v0 : V[i];
  return p;
}

template <typename R>
void launch_norm_start(helm_op* op, int l, int nrhs, const cx<R>* b, const KCtx& ctx) {
  const long long N = op->lev[l].N;
  if (!op->nact) return;
  dim3 grid(blas_blocks(N, op->nact), op->nact);
  prof_begin(KC_NORM, op->st, l);
  pdl_launch(k_norm_start<R>, grid, dim3(HELM_RED_THREADS), 0, op->st, N, b, (const int*)op->active_d, ctx, op->rb);
  CKL();
  prof_end(KC_NORM, op->st, acct(op, l, sizeof(cx<R>) * (double)N, false, nrhs));
}

template <typename R>
void launch_update(helm_op* op, int l, int nrhs, const VPtrs<R>& V, int j, cx<R>* w, const KCtx& ctx) {
  const long long N = op->lev[l].N;
  if (!op->nact) return;
  dim3 grid(blas_blocks(N, op->nact), op->nact);
  prof_begin(KC_UPDATE, op->st, l);
  dispatch_k(j + 1, [&](auto c) {
    pdl_launch(k_update_t<R, decltype(c)::value>, grid, dim3(HELM_RED_THREADS), 0, op->st, N, V, j, w,
               (const int*)op->active_d, ctx, op->rb);
  });
  CKL();
  prof_end(KC_UPDATE, op->st, acct(op, l, (j + 3.0) * sizeof(cx<R>) * N, false, nrhs));
}

template <typename R>
void launch_solupdate(helm_op* op, int l, int nrhs, const VPtrs<R>& Z, const double* zscale, cx<R>* x,
                      int init, int k, const KCtx& ctx, const cx<R>* W = nullptr) {
  const long long N = op->lev[l].N;
  if (!op->nact) return;
  dim3 grid(blas_blocks(N, op->nact), op->nact);
  prof_begin(KC_SOLUPD, op->st, l);
  dispatch_k(k, [&](auto c) {
    pdl_launch(k_solupdate_t<R, decltype(c)::value>, grid, dim3(HELM_RED_THREADS), 0, op->st, N, Z, zscale, x, init,
               (const int*)op->active_d, ctx, W);
  });
  CKL();
  prof_end(KC_SOLUPD, op->st, acct(op, l, (k + (init ? 1.0 : 2.0)) * sizeof(cx<R>) * N, false, nrhs));
}

template <typename Ti, typename To>
void launch_copy_scale(helm_op* op, int l, int nrhs, const Ti* in, To* out, const double* scale,
                       const int* kact, int j) {
  const long long N = op->lev[l].N;
  if (!op->nact) return;
  dim3 grid(blas_blocks(N, op->nact), op->nact);
  prof_begin(KC_COPY, op->st, l);
  pdl_launch(k_copy_scale<Ti, To>, grid, dim3(HELM_RED_THREADS), 0, op->st, N, in, out, scale, (int)K1, kact, j,
             (const int*)op->active_d);
  CKL();
  prof_end(KC_COPY, op->st, acct(op, l, (double)(sizeof(Ti) + sizeof(To)) * N, false, nrhs));
}

template <typename R>
void launch_restrict(helm_op* op, int l, int nrhs, const cx<R>* in, cx<R>* out) {
  const LevelDev &F = op->lev[l], &Cc = op->lev[l + 1];
  if (!op->nact) return;
  dim3 grid(blas_blocks(Cc.N, op->nact), op->nact);
  const R fac = (R)std::ldexp(1.0, -op->dim);
  prof_begin(KC_RESTRICT, op->st, l);
  pdl_launch(k_restrict<R>, grid, dim3(HELM_RED_THREADS), 0, op->st, F.nx, F.ny, F.nz, Cc.nx, Cc.ny, Cc.nz,
             (int)(op->dim == 3), fac, in, out, (const int*)op->active_d);
  CKL();
  prof_end(KC_RESTRICT, op->st, acct(op, l, sizeof(cx<R>) * (double)(F.N + Cc.N), false, nrhs));
}

template <typename R>
void launch_prolong_add(helm_op* op, int l, int nrhs, const cx<R>* in, cx<R>* out) {
  const LevelDev &F = op->lev[l], &Cc = op->lev[l + 1];
  if (!op->nact) return;
  dim3 grid(blas_blocks(F.N, op->nact), op->nact);
  prof_begin(KC_PROLONG, op->st, l);
  pdl_launch(k_prolong_add<R>, grid, dim3(HELM_RED_THREADS), 0, op->st, F.nx, F.ny, F.nz, Cc.nx, Cc.ny, Cc.nz,
             (int)(op->dim == 3), in, out, (const int*)op->active_d);
  CKL();
  prof_end(KC_PROLONG, op->st, acct(op, l, sizeof(cx<R>) * (double)(2 * F.N + Cc.N), false, nrhs));
}

// ------------------------------------------------------------------------------ Krylov
// One restarted GMRES (flex = false) / FGMRES (flex = true, right preconditioner M) process
// of `ko` cycles of `ki` Arnoldi steps on level l (fixed counts, R19; breakdown guard D14).
// GMRES steps are fused (stencil.cuh MODE 3/4): step j forms v_j from the previous raw
// product W and the basis while applying H, so there is no separate update pass; W
// ping-pongs between V[ki] and Wx; the last step closes the Hessenberg by Pythagoras.
// FGMRES keeps stencil+projections (MODE 2) + update (its v_{j+1} feeds the preconditioner).
template <typename R>
using Precond = std::function<void(const cx<R>* v, const double* vscale, const int* kact, int j, cx<R>* z)>;

template <typename R>
void krylov(helm_op* op, int l, int adj, int nrhs, KCtx& ctx, int ko, int ki, bool flex, const cx<R>* b,
            cx<R>* x, bool x0zero, cx<R>* const* V, cx<R>* const* Z, const Precond<R>& M, cx<R>* Wx = nullptr) {
  ctx.k = ki;
  for (int cyc = 0; cyc < ko; ++cyc) {
    const bool first_zero = (cyc == 0 && x0zero);
    const cx<R>* v0;
    if (first_zero) {
      launch_norm_start<R>(op, l, nrhs, b, ctx);
      v0 = b;
    } else {
      launch_stencil<R>(op, l, adj, 1, nrhs, x, V[0], b, nullptr, nullptr, 0, ctx);
      v0 = V[0];
    }
    if (!flex) {
      cx<R>* Wb[2] = {V[ki], Wx};
      for (int j = 0; j < ki; ++j) {
        VPtrs<R> Vp = vptrs<R>(V, v0, j);
        const cx<R>* xin = j == 0 ? v0 : Wb[(j - 1) & 1];
        launch_plane<R>(op, l, adj, j == ki - 1 ? 4 : 3, nrhs, xin, Wb[j & 1], nullptr, &Vp, j, nullptr, ctx.kact,
                        j, ctx, j == 0 ? nullptr : V[j]);
      }
      VPtrs<R> Vp = vptrs<R>(V, v0, ki);
      launch_solupdate<R>(op, l, nrhs, Vp, ctx.scale, x, first_zero, ki, ctx,
                          (ki >= 2 && !last_v_stored(op, l)) ? Wb[(ki - 2) & 1] : nullptr);
      continue;
    }
    for (int j = 0; j < ki; ++j) {
      VPtrs<R> Vp = vptrs<R>(V, v0, j + 1);
      M(Vp.p[j], ctx.scale + j, ctx.kact, j, Z[j]);
      launch_plane<R>(op, l, adj, 2, nrhs, Z[j], V[j + 1], nullptr, &Vp, j + 1, nullptr, ctx.kact, j, ctx);
      launch_update<R>(op, l, nrhs, Vp, j, V[j + 1], ctx);
    }
    VPtrs<R> Zp{};
    for (int i = 0; i < ki; ++i) Zp.p[i] = Z[i];
    launch_solupdate<R>(op, l, nrhs, Zp, nullptr, x, first_zero, ki, ctx);
  }
}

template <typename R> LevelWS<R>* wsets(helm_op* op);
template <> LevelWS<double>* wsets<double>(helm_op* op) { return op->w64; }
template <> LevelWS<float>* wsets<float>(helm_op* op) { return op->w32; }

// Algorithmic bytes of one persistent-kernel GMRES(ko, ki) on N points (its own schedule:
// per step a stencil+projection pass and an update+norm pass, then the solution update).
double persist_gmres_bytes(double N, int ko, int ki, bool x0zero, double Sc, double Sr) {
  double b = 0.0;
  for (int c = 0; c < ko; ++c) {
    const bool zero = x0zero && c == 0;
    b += zero ? Sc * N : (3 * Sc + Sr) * N;                         // r = b - H x, ||r||
    for (int j = 0; j < ki; ++j) b += (2.0 * (j + 3) * Sc + Sr) * N;  // both passes of step j
    b += (ki + (zero ? 1 : 2)) * Sc * N;                              // x update
  }
  return b;
}

// The V-cycle at the second-to-last level (l + 1 coarsest) as ONE cooperative launch
// (persist.cuh) when the level is small (HELM_PERSIST_MAXPTS points over the active RHS,
// default 2^21). OPT-IN (HELM_PERSIST=1): measured on the B200 (profiles/r02/persist_ab.txt)
// it issues 10x fewer launches but is not faster — cfg3 one solve 148 vs 137 ms, 8-source
// batch 306 vs 217 ms, cfg2 bench 31 vs 66 solves/s — because a grid barrier plus the
// dependent L2 round trips of a pass cost about what a graph-launched kernel boundary does
// (DESIGN §6, §11). Returns false when not applicable.
template <typename R>
bool vcycle_persist(helm_op* op, int l, int adj, int nrhs, const cx<R>* b, cx<R>* x) {
  static const int on = env_int("HELM_PERSIST", 0);
  static const long long maxpts = std::max(0, env_int("HELM_PERSIST_MAXPTS", 1 << 21));
  if (!on || op->nact == 0 || l + 1 != op->L - 1 || op->grid.stencil != HELM_STD2) return false;
  const LevelDev &F = op->lev[l], &Cc = op->lev[l + 1];
  if (F.N * (long long)op->nact > maxpts) return false;
  const helm_mlopts& o = op->ml;
  constexpr int NT = 256;
  auto kern = k_vcycle_persist<R, NT>;
  static const int per_sm = [&] {
    int v = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, NT, 0));
    return v;
  }();
  const long long G = (long long)per_sm * num_sms();
  if (per_sm < 1 || G < op->nact) return false;
  // CTAs per RHS: all co-resident CTAs, but no fewer than 4 x NT fine points per CTA
  const int cpr = (int)std::max(1LL, std::min(G / op->nact, (F.N + 4 * NT - 1) / (4 * NT)));
  LevelWS<R>* W = wsets<R>(op);
  PersistArgs<R> a{};
  a.gf = geo<R>(op, l, adj);
  a.gc = geo<R>(op, l + 1, adj);
  a.b = b; a.x = x;
  for (int i = 0; i <= o.ks_i; ++i) a.SV[i] = W[l].SV[i];
  a.SW = W[l].SW;
  for (int i = 0; i <= o.kc_i; ++i) a.FV[i] = W[l + 1].FV[i];
  a.FW = W[l + 1].FW; a.Fx = W[l + 1].Fx; a.Fb = W[l + 1].Fb;
  a.active = op->active_d; a.nact = op->nact; a.cpr = cpr;
  a.ks_o = o.ks_o; a.ks_i = o.ks_i; a.kc_o = o.kc_o; a.kc_i = o.kc_i;
  a.has_y = op->dim == 3; a.fac = (R)std::ldexp(1.0, -op->dim);
  a.part = op->rb.part;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(op->nact * cpr));
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = op->st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const double Sc = sizeof(cx<R>), Sr = sizeof(R);
  const double bytes = persist_gmres_bytes((double)F.N, o.ks_o, o.ks_i, true, Sc, Sr) +
                       persist_gmres_bytes((double)F.N, o.ks_o, o.ks_i, false, Sc, Sr) +
                       (3 * Sc + Sr) * F.N + Sc * (F.N + Cc.N) +                  // residual, restrict
                       persist_gmres_bytes((double)Cc.N, o.kc_o, o.kc_i, true, Sc, Sr) +
                       Sc * (2.0 * F.N + Cc.N);                                    // prolong + add
  prof_begin(KC_PERSIST, op->st, l);
  CK(cudaLaunchKernelEx(&cfg, kern, a));
  CKL();
  prof_end(KC_PERSIST, op->st, acct(op, l, bytes, false, nrhs));
  // matvec counts of the equivalent launch sequence: per GMRES(ko, ki) ko ki steps plus the
  // restart residuals, plus the V-cycle residual at level l
  for (int r = 0; r < nrhs; ++r)
    if (op->act_h[r]) {
      op->mv[l][r] += 2LL * o.ks_o * o.ks_i + (o.ks_o - 1) + o.ks_o + 1;
      op->mv[l + 1][r] += (long long)o.kc_o * o.kc_i + (o.kc_o - 1);
    }
  return true;
}

// Alg. 1 with the recursion of Fig. 3: x = M_l(b).
template <typename R>
void vcycle(helm_op* op, int l, int adj, int nrhs, const cx<R>* b, cx<R>* x) {
  if (vcycle_persist<R>(op, l, adj, nrhs, b, x)) return;
  LevelWS<R>* W = wsets<R>(op);
  const helm_mlopts& o = op->ml;
  // pre-smooth: GMRES(ks_o, ks_i) from 0 (R19)
  krylov<R>(op, l, adj, nrhs, W[l].ctxS, o.ks_o, o.ks_i, false, b, x, true, W[l].SV, nullptr, nullptr, W[l].SW);
  // residual and restriction (R = 2^-d P^T, R21)
  launch_stencil<R>(op, l, adj, 1, nrhs, x, W[l].SV[0], b, nullptr, nullptr, 0, W[l].ctxS);
  launch_restrict<R>(op, l, nrhs, W[l].SV[0], W[l + 1].Fb);
  // coarse solve (R20): coarsest GMRES, otherwise FGMRES preconditioned by V-cycle_{l+1}
  if (l + 1 == op->L - 1) {
    krylov<R>(op, l + 1, adj, nrhs, W[l + 1].ctxC, o.kc_o, o.kc_i, false, W[l + 1].Fb, W[l + 1].Fx, true,
              W[l + 1].FV, nullptr, nullptr, W[l + 1].FW);
  } else {
    Precond<R> M = [op, l, adj, nrhs, W](const cx<R>* v, const double* vs, const int* kact, int j, cx<R>* z) {
      launch_copy_scale<cx<R>, cx<R>>(op, l + 1, nrhs, v, W[l + 1].VB, vs, kact, j);
      vcycle<R>(op, l + 1, adj, nrhs, W[l + 1].VB, z);
    };
    krylov<R>(op, l + 1, adj, nrhs, W[l + 1].ctxC, o.kc_o, o.kc_i, true, W[l + 1].Fb, W[l + 1].Fx, true,
              W[l + 1].FV, W[l + 1].FZ, M);
  }
  launch_prolong_add<R>(op, l, nrhs, W[l + 1].Fx, x);
  // post-smooth: GMRES(ks_o, ks_i) from the current x
  krylov<R>(op, l, adj, nrhs, W[l].ctxS, o.ks_o, o.ks_i, false, b, x, false, W[l].SV, nullptr, nullptr, W[l].SW);
}

// ------------------------------------------------------------------------------ setup
void build_tables(helm_op* op) {
  const helm_grid& G = op->grid;
  for (int l = 0; l < op->L; ++l) {
    LevelDev& Lv = op->lev[l];
    const int Ns[3] = {Lv.nx, Lv.ny, Lv.nz};
    for (int a = 0; a < 3; ++a) {
      const int N = Ns[a];
      const int NT = N * op->nop;   // op-major: operator o's table at o * N
      if (a == 1 && op->dim == 2) {   // 2D: no y term (tables identically zero)
        for (int adj = 0; adj < 2; ++adj)
          for (int t = 0; t < 3; ++t) CK(cudaMemsetAsync(Lv.t64[adj][a][t], 0, sizeof(double2) * NT, op->st));
      } else {
        for (int o = 0; o < op->nop; ++o) {
          AxisPml ap{};
          ap.N = N; ap.n_int = (int)G.n[a]; ap.wlo = G.pml[a][0]; ap.whi = G.pml[a][1]; ap.level = l;
          ap.h0 = G.h; ap.omega = op->omegas[o]; ap.R = op->pml.R; ap.power = op->pml.power; ap.vref = op->vref;
          double2* T0[3] = {Lv.t64[0][a][0] + (size_t)o * N, Lv.t64[0][a][1] + (size_t)o * N, Lv.t64[0][a][2] + (size_t)o * N};
          double2* T1[3] = {Lv.t64[1][a][0] + (size_t)o * N, Lv.t64[1][a][1] + (size_t)o * N, Lv.t64[1][a][2] + (size_t)o * N};
          prof_count(KC_SETUP);
          k_tables<<<(N + 127) / 128, 128, 0, op->st>>>(ap, T0[0], T0[1], T0[2]);
          CKL();
          prof_count(KC_SETUP);
          k_tables_adj<<<(N + 127) / 128, 128, 0, op->st>>>(N, T0[0], T0[1], T0[2], T1[0], T1[1], T1[2]);
          CKL();
        }
      }
      if (op->dtype == HELM_C64)
        for (int adj = 0; adj < 2; ++adj)
          for (int t = 0; t < 3; ++t) {
            prof_count(KC_SETUP);
            k_cast_c<<<(NT + 127) / 128, 128, 0, op->st>>>(NT, Lv.t64[adj][a][t], Lv.t32[adj][a][t]);
            CKL();
          }
    }
    const int nzo = Lv.nz * op->nop;
    for (int adj = 0; adj < 2; ++adj) {
      prof_count(KC_SETUP);
      k_zpack<double2><<<(nzo + 127) / 128, 128, 0, op->st>>>(Lv.nz, op->nop, Lv.t64[adj][2][0], Lv.t64[adj][2][1],
                                                              Lv.t64[adj][2][2], Lv.z64[adj]);
      CKL();
      if (op->dtype == HELM_C64) {
        prof_count(KC_SETUP);
        k_zpack<float2><<<(nzo + 127) / 128, 128, 0, op->st>>>(Lv.nz, op->nop, Lv.t32[adj][2][0], Lv.t32[adj][2][1],
                                                               Lv.t32[adj][2][2], Lv.z32[adj]);
        CKL();
      }
      if (Lv.ny > 1) {
        prof_count(KC_SETUP);
        k_zpack<double2, 4><<<(nzo + 127) / 128, 128, 0, op->st>>>(Lv.nz, op->nop, Lv.t64[adj][2][0],
                                                                   Lv.t64[adj][2][1], Lv.t64[adj][2][2], Lv.zq64[adj]);
        CKL();
        if (op->dtype == HELM_C64) {
          prof_count(KC_SETUP);
          k_zpack<float2, 4><<<(nzo + 127) / 128, 128, 0, op->st>>>(Lv.nz, op->nop, Lv.t32[adj][2][0],
                                                                   Lv.t32[adj][2][1], Lv.t32[adj][2][2], Lv.zq32[adj]);
          CKL();
        }
      }
    }
  }
}

void build_models(helm_op* op) {
  const helm_grid& G = op->grid;
  LevelDev& L0 = op->lev[0];
  prof_count(KC_SETUP);
  k_extend<<<(unsigned)((L0.N + 255) / 256), 256, 0, op->st>>>(L0.nx, L0.ny, L0.nz, (int)G.n[0], (int)G.n[1], (int)G.n[2],
                                                               G.pml[0][0], G.pml[1][0], G.pml[2][0], op->m_int_d, L0.m64);
  CKL();
  for (int l = 1; l < op->L; ++l) {
    const LevelDev &F = op->lev[l - 1];
    LevelDev& Cc = op->lev[l];
    prof_count(KC_SETUP);
    k_coarsen_model<<<(unsigned)((Cc.N + 255) / 256), 256, 0, op->st>>>(F.nx, F.ny, F.nz, Cc.nx, Cc.ny, Cc.nz, op->dim == 3,
                                                                        F.m64, Cc.m64);
    CKL();
  }
  if (op->dtype == HELM_C64)
    for (int l = 0; l < op->L; ++l) {
      LevelDev& Lv = op->lev[l];
      prof_count(KC_SETUP);
      k_cast<double, float><<<(unsigned)((Lv.N + 255) / 256), 256, 0, op->st>>>(Lv.N, Lv.m64, Lv.m32);
      CKL();
    }
  for (int l = 0; l < op->L; ++l) {   // 16-B pitched copies of m for the TMA stages (3D) / strips (2D)
    LevelDev& Lv = op->lev[l];
    const size_t rows = (size_t)Lv.ny * Lv.nz;
    CK(cudaMemcpy2DAsync(Lv.mq64, sizeof(double) * Lv.nxq, Lv.m64, sizeof(double) * Lv.nx, sizeof(double) * Lv.nx, rows,
                         cudaMemcpyDeviceToDevice, op->st));
    if (op->dtype == HELM_C64)
      CK(cudaMemcpy2DAsync(Lv.mq32, sizeof(float) * Lv.nxq, Lv.m32, sizeof(float) * Lv.nx, sizeof(float) * Lv.nx, rows,
                           cudaMemcpyDeviceToDevice, op->st));
  }
}

template <typename R>
void alloc_ws(helm_op* op) {
  LevelWS<R>* W = wsets<R>(op);
  const helm_mlopts& o = op->ml;
  const int B = op->max_rhs;
  double vec = 0.0;  // live vectors in units of the finest size
  const double N0 = (double)op->lev[0].N;
  for (int l = 0; l < op->L; ++l) {
    const size_t n = (size_t)op->lev[l].N * B;
    const double f = op->lev[l].N / N0 * (sizeof(cx<R>) / 16.0);
    if (l < op->L - 1) {   // levels that run a V-cycle: smoother basis + input copy
      for (int i = 0; i <= o.ks_i; ++i) W[l].SV[i] = dalloc<cx<R>>(op->allocs, n);
      W[l].SW = dalloc<cx<R>>(op->allocs, n);
      W[l].VB = dalloc<cx<R>>(op->allocs, n);
      W[l].ctxS = make_ctx(op->allocs, B, o.ks_i);
      vec += (o.ks_i + 3) * f;
      if (l == 0) { W[l].VX = dalloc<cx<R>>(op->allocs, n); vec += f; }   // fixed V-cycle output (graphs)
    }
    if (l >= 1) {          // coarse solves
      for (int i = 0; i <= o.kc_i; ++i) W[l].FV[i] = dalloc<cx<R>>(op->allocs, n);
      const bool flex = (l < op->L - 1);
      if (flex)
        for (int i = 0; i < o.kc_i; ++i) W[l].FZ[i] = dalloc<cx<R>>(op->allocs, n);
      else
        W[l].FW = dalloc<cx<R>>(op->allocs, n);
      W[l].Fx = dalloc<cx<R>>(op->allocs, n);
      W[l].Fb = dalloc<cx<R>>(op->allocs, n);
      W[l].ctxC = make_ctx(op->allocs, B, o.kc_i);
      vec += ((o.kc_i + 1) + (flex ? o.kc_i : 1) + 2) * f;
    }
  }
  op->ws_vectors += vec;
}

void validate_grid(const helm_grid* g) {
  REQ(g, HELM_ERR_ARG, "grid is NULL");
  REQ(g->ndim == 2 || g->ndim == 3, HELM_ERR_ARG, "ndim must be 2 or 3");
  REQ(g->h > 0 && std::isfinite(g->h), HELM_ERR_ARG, "h must be > 0");
  for (int a = 0; a < 3; ++a) {
    REQ(g->n[a] >= 1, HELM_ERR_SHAPE, "n[a] must be >= 1");
    REQ(g->pml[a][0] >= 0 && g->pml[a][1] >= 0, HELM_ERR_ARG, "pml widths must be >= 0");
  }
  if (g->ndim == 2) REQ(g->n[1] == 1 && g->pml[1][0] == 0 && g->pml[1][1] == 0, HELM_ERR_SHAPE, "2D grids need n[1]=1, pml[1]={0,0}");
  else REQ(g->n[1] >= 2, HELM_ERR_SHAPE, "3D grids need n[1] >= 2");
  REQ(g->n[0] >= 2 && g->n[2] >= 2, HELM_ERR_SHAPE, "n[0], n[2] must be >= 2");
  REQ(g->stencil == HELM_STD2 || g->stencil == HELM_OPT, HELM_ERR_ARG, "stencil must be HELM_STD2 or HELM_OPT");
  for (int a = 0; a < 3; ++a) REQ(g->n[a] + g->pml[a][0] + g->pml[a][1] < (1LL << 30), HELM_ERR_SHAPE, "axis too large");
}

// Model and PML checks of helm_setup, also applied when a cached fwi op is reused.
void validate_model_pml(const helm_grid& g, const double* m, const helm_pml& P) {
  REQ(std::isfinite(P.R) && P.R > 0 && P.R < 1 && P.power >= 0 && std::isfinite(P.v_ref), HELM_ERR_ARG,
      "bad PML parameters");
  const size_t n_int = (size_t)g.n[0] * g.n[1] * g.n[2];
  for (size_t i = 0; i < n_int; ++i) REQ(m[i] > 0 && std::isfinite(m[i]), HELM_ERR_ARG, "m must be > 0 and finite");
}

void op_set_model(helm_op* op, const double* m_host) {
  // captured graphs stay valid: the models are rewritten in place (helm_op::VGraph)
  const helm_grid& G = op->grid;
  const size_t n_int = (size_t)G.n[0] * G.n[1] * G.n[2];
  CK(cudaMemcpyAsync(op->m_int_d, m_host, n_int * sizeof(double), cudaMemcpyHostToDevice, op->st));
  build_models(op);
}

void op_set_omegas(helm_op* op, const double* w, int n) {
  REQ(n >= 1 && n <= HELM_MAXOP, HELM_ERR_ARG, "too many operators in one batch");
  for (int o = 0; o < n; ++o) REQ(w[o] > 0 && std::isfinite(w[o]), HELM_ERR_ARG, "omega must be > 0");
  op->gsig.assign(w, w + n);   // captured kernels carry omega^2 and the operator count by value
  op->nop = n;
  for (int o = 0; o < n; ++o) op->omegas[o] = w[o];
  op->omega = w[0];
  build_tables(op);
}
void op_set_omega(helm_op* op, double omega) { op_set_omegas(op, &omega, 1); }

// RHS -> operator map of the next solves (joint (source, frequency) batches).
void op_set_rop(helm_op* op, const std::vector<int>& rop) {
  CK(cudaMemcpyAsync(op->rop_d, rop.data(), sizeof(int) * rop.size(), cudaMemcpyHostToDevice, op->st));
}

helm_op* op_create(const helm_grid* grid, const double* m, double omega, const helm_pml* pml, helm_dtype dtype,
                   int max_rhs, const helm_mlopts* mlo, cudaStream_t st, int k_inner) {
  validate_grid(grid);
  REQ(m, HELM_ERR_ARG, "m is NULL");
  REQ(omega > 0 && std::isfinite(omega), HELM_ERR_ARG, "omega must be > 0");
  REQ(dtype == HELM_C64 || dtype == HELM_C128, HELM_ERR_ARG, "bad dtype");
  REQ(max_rhs >= 1, HELM_ERR_ARG, "max_rhs must be >= 1");
  helm_mlopts o = mlo ? *mlo : helm_mlopts{3, 3, 5, 3, 5};
  const bool apply_only = o.levels == 0;   // operator-only op: helm_apply, no solver workspace
  if (apply_only) o.levels = 1;
  REQ(o.levels >= 1 && o.levels <= 4, HELM_ERR_ARG, "levels must be in [0,4]");
  REQ(o.ks_o >= 1 && o.ks_i >= 1 && o.kc_o >= 1 && o.kc_i >= 1, HELM_ERR_ARG, "Krylov counts must be >= 1");
  REQ(o.ks_i <= HELM_KMAX && o.kc_i <= HELM_KMAX && k_inner <= HELM_KMAX && k_inner >= 1, HELM_ERR_ARG,
      "inner Krylov dimension exceeds HELM_KMAX");
  helm_pml P = pml ? *pml : helm_pml{1e-4, 2, 0.0};
  validate_model_pml(*grid, m, P);
  const size_t n_int = (size_t)grid->n[0] * grid->n[1] * grid->n[2];
  double vref = P.v_ref;
  if (!(vref > 0)) {
    double mmin = m[0];
    for (size_t i = 1; i < n_int; ++i) mmin = std::min(mmin, m[i]);
    vref = 1.0 / std::sqrt(mmin);   // max velocity (R5 default)
  }
  int dev = 0, major = 0, minor = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  CK(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
  REQ(major == 10 && minor == 0, HELM_ERR_STATE, "libhelm is built for sm_100a (B200) only");

  std::unique_ptr<helm_op> op(new helm_op());
  op->device = dev;
  op->grid = *grid; op->pml = P; op->ml = o; op->dtype = dtype; op->max_rhs = max_rhs; op->omega = omega;
  op->vref = vref; op->st = st; op->dim = grid->ndim; op->k_inner = k_inner;
  // hierarchy sizes (D13): N -> ceil(N/2) on active axes, stop when an axis would be < 5
  int dims[4][3];
  dims[0][0] = (int)(grid->n[0] + grid->pml[0][0] + grid->pml[0][1]);
  dims[0][1] = (int)(grid->n[1] + grid->pml[1][0] + grid->pml[1][1]);
  dims[0][2] = (int)(grid->n[2] + grid->pml[2][0] + grid->pml[2][1]);
  int L = 1;
  while (L < o.levels) {
    int c[3] = {(dims[L - 1][0] + 1) / 2, op->dim == 3 ? (dims[L - 1][1] + 1) / 2 : 1, (dims[L - 1][2] + 1) / 2};
    if (c[0] < 5 || c[2] < 5 || (op->dim == 3 && c[1] < 5)) break;
    for (int a = 0; a < 3; ++a) dims[L][a] = c[a];
    ++L;
  }
  if (L < o.levels) g_err = "warning: grid too small for the requested depth; using " + std::to_string(L) + " levels";
  op->L = L;
  {   // fewer than 4 points per wavelength on the finest grid is a warning, not a
      // failure (readable via helm_last_error); depth is limited by ppw on coarse grids
    double mmax = m[0];
    for (size_t i = 1; i < n_int; ++i) mmax = std::max(mmax, m[i]);
    const double ppw = 2.0 * M_PI / (omega * std::sqrt(mmax)) / grid->h;
    if (ppw < 4.0) {
      char buf[160];
      std::snprintf(buf, sizeof buf, "warning: grid too coarse: %.2f points per wavelength at v_min (< 4)", ppw);
      g_err = g_err.empty() ? std::string(buf) : g_err + "; " + buf;
    }
  }
  for (int l = 0; l < L; ++l) {
    LevelDev& Lv = op->lev[l];
    Lv.nx = dims[l][0]; Lv.ny = dims[l][1]; Lv.nz = dims[l][2];
    Lv.N = (long long)Lv.nx * Lv.ny * Lv.nz;
    Lv.m64 = dalloc<double>(op->allocs, Lv.N);
    if (dtype == HELM_C64) Lv.m32 = dalloc<float>(op->allocs, Lv.N);
    const int Ns[3] = {Lv.nx, Lv.ny, Lv.nz};
    for (int adj = 0; adj < 2; ++adj)
      for (int a = 0; a < 3; ++a)
        for (int t = 0; t < 3; ++t) {
          Lv.t64[adj][a][t] = dalloc<double2>(op->allocs, (size_t)Ns[a] * HELM_MAXOP);
          if (dtype == HELM_C64) Lv.t32[adj][a][t] = dalloc<float2>(op->allocs, (size_t)Ns[a] * HELM_MAXOP);
        }
    for (int adj = 0; adj < 2; ++adj) {
      Lv.z64[adj] = dalloc<double2>(op->allocs, (size_t)3 * Lv.nz * HELM_MAXOP);
      if (dtype == HELM_C64) Lv.z32[adj] = dalloc<float2>(op->allocs, (size_t)3 * Lv.nz * HELM_MAXOP);
      if (Lv.ny > 1) {
        Lv.zq64[adj] = dalloc<double2>(op->allocs, (size_t)4 * Lv.nz * HELM_MAXOP);
        if (dtype == HELM_C64) Lv.zq32[adj] = dalloc<float2>(op->allocs, (size_t)4 * Lv.nz * HELM_MAXOP);
      }
    }
    {   // 16-B pitched copy of m: the 3D TMA m tiles, and (complex128) the 2D march strips
      Lv.nxq = (Lv.nx + 3) / 4 * 4;
      Lv.mq64 = dalloc<double>(op->allocs, (size_t)Lv.nxq * Lv.ny * Lv.nz);
      if (dtype == HELM_C64) Lv.mq32 = dalloc<float>(op->allocs, (size_t)Lv.nxq * Lv.ny * Lv.nz);
      // the row padding [nx, nxq) is read as the x = nx ghost's model by the OPT stencil's
      // halo'd m tile: keep it finite (zero)
      CK(cudaMemset(Lv.mq64, 0, sizeof(double) * (size_t)Lv.nxq * Lv.ny * Lv.nz));
      if (Lv.mq32) CK(cudaMemset(Lv.mq32, 0, sizeof(float) * (size_t)Lv.nxq * Lv.ny * Lv.nz));
    }
  }
  op->m_int_d = dalloc<double>(op->allocs, n_int);
  // reduction scratch: BLAS kernels use (KMAX+1) x blocks per RHS at stride pstride; the
  // plane kernels use (KMAX+2) x slots per RHS, <= max(2048/32 x SMs, 8 x max_rhs) slots total
  // (one resident wave of CTAs, one slot per warp, see run_plane).
  const long long pst = (long long)K1 * TARGET_BLOCKS;
  const long long plane_slots = std::max(64LL * num_sms(), 8LL * max_rhs) * (HELM_KMAX + 2);
  op->rb.pstride = pst;
  op->rb.part = dalloc<double2>(op->allocs, (size_t)std::max(pst * max_rhs, plane_slots));
  op->rb.ticket = dalloc<unsigned>(op->allocs, max_rhs);
  CK(cudaMemset(op->rb.ticket, 0, sizeof(unsigned) * max_rhs));
  op->active_d = dalloc<int>(op->allocs, max_rhs);
  op->rop_d = dalloc<int>(op->allocs, max_rhs);
  CK(cudaMemset(op->rop_d, 0, sizeof(int) * max_rhs));
  op->apply_only = apply_only;
  if (apply_only) {
    op->act_h.assign(max_rhs, 1);
    op->bytes.assign(max_rhs, 0.0);
    for (int l = 0; l < 4; ++l) op->mv[l].assign(max_rhs, 0);
    op_set_model(op.get(), m);
    op_set_omega(op.get(), omega);
    CK(cudaStreamSynchronize(st));
    return op.release();
  }
  // outer FGMRES (always complex128, D15) + V-cycle workspace in the V-cycle precision
  const size_t n0 = (size_t)op->lev[0].N * max_rhs;
  for (int i = 0; i <= k_inner; ++i) op->OV[i] = dalloc<double2>(op->allocs, n0);
  for (int i = 0; i < k_inner; ++i) op->OZ[i] = dalloc<double2>(op->allocs, n0);
  op->ctxO = make_ctx(op->allocs, max_rhs, k_inner);
  op->ctxO.tol = dalloc<double>(op->allocs, max_rhs);   // early stop inside an outer cycle (R23)
  CK(cudaMemset(op->ctxO.tol, 0, sizeof(double) * max_rhs));
  op->ws_vectors = 2 * k_inner + 1;
  if (dtype == HELM_C64) {
    op->OX = dalloc<double2>(op->allocs, n0);
    op->OB = dalloc<double2>(op->allocs, n0);
    op->ws_vectors += 2;
    alloc_ws<float>(op.get());
  } else {
    alloc_ws<double>(op.get());
  }
  op->act_h.assign(max_rhs, 1);
  op->bytes.assign(max_rhs, 0.0);
  for (int l = 0; l < 4; ++l) op->mv[l].assign(max_rhs, 0);
  op_set_model(op.get(), m);
  op_set_omega(op.get(), omega);
  CK(cudaStreamSynchronize(st));
  return op.release();
}

void reset_acct(helm_op* op, int nrhs) {
  std::fill(op->bytes.begin(), op->bytes.end(), 0.0);
  for (int l = 0; l < 4; ++l) std::fill(op->mv[l].begin(), op->mv[l].end(), 0);
  std::fill(op->act_h.begin(), op->act_h.end(), 0);
  std::fill(op->act_h.begin(), op->act_h.begin() + nrhs, 1);
}

// Upload the compact list of active RHS: kernels launch over these only, so RHS that have
// converged (or were never active) cost nothing and the whole GPU works on the rest.
void set_active(helm_op* op, int nrhs) {
  op->alist_h.clear();
  for (int r = 0; r < nrhs; ++r)
    if (op->act_h[r]) op->alist_h.push_back(r);
  op->nact = (int)op->alist_h.size();
  // an unchanged list is not uploaded again (a pageable host->device copy costs ~10 us of host
  // time per call: the whole launch cost of a small helm_apply)
  if (op->nact && op->alist_h != op->alist_dev) {
    CK(cudaMemcpyAsync(op->active_d, op->alist_h.data(), sizeof(int) * op->nact, cudaMemcpyHostToDevice, op->st));
    op->alist_dev = op->alist_h;
  }
}

// Level-0 V-cycle as a replayed CUDA graph: within a solve the launch sequence of a V-cycle
// depends only on (adjoint, batch size, number of active RHS) — every Krylov scalar and the
// active list live in device memory — so it is captured once per key and replayed (no
// per-kernel host launch cost, tighter device-side launches). The graph writes a fixed
// output buffer. Host-side accounting of the captured launches is recorded at capture and
// added per replay. HELM_GRAPHS=0, or an active kernel profiler, runs the V-cycle live.
template <typename R>
void vcycle0_graph(helm_op* op, int adj, int nrhs, const cx<R>* b, cx<R>* z) {
  static const bool on = env_int("HELM_GRAPHS", 1) != 0;
  if (!on || g_prof.on || op->graphs_off || op->nact == 0) { vcycle<R>(op, 0, adj, nrhs, b, z); return; }
  for (auto& g : op->vgraphs)
    if (g.adj == adj && g.nrhs == nrhs && g.nact == op->nact && g.sig == op->gsig) {
      CK(cudaGraphLaunch(g.exec, op->st));
      for (int r = 0; r < nrhs; ++r)
        if (op->act_h[r]) {
          op->bytes[r] += g.bytes;
          for (int l = 0; l < 4; ++l) op->mv[l][r] += g.mv[l];
        }
      g_launches += g.launches;
      return;
    }
  vcycle<R>(op, 0, adj, nrhs, b, z);   // this call runs live; the next ones replay
  int r0 = 0;
  while (r0 < nrhs && !op->act_h[r0]) ++r0;
  const double b0 = op->bytes[r0];
  long long m0[4];
  for (int l = 0; l < 4; ++l) m0[l] = op->mv[l][r0];
  std::vector<double> bsave = op->bytes;
  std::vector<int64_t> msave[4];
  for (int l = 0; l < 4; ++l) msave[l] = op->mv[l];
  const long long l0 = g_launches;
  cudaGraph_t graph = nullptr;
  if (!op->cap_st) CK(cudaStreamCreateWithFlags(&op->cap_st, cudaStreamNonBlocking));
  cudaStream_t user_st = op->st;
  op->st = op->cap_st;   // capture on the private stream (nothing executes during capture)
  bool ok = cudaStreamBeginCapture(op->st, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
  if (ok) {
    try {
      vcycle<R>(op, 0, adj, nrhs, b, z);
    } catch (...) {
      ok = false;
    }
    cudaGraph_t g2 = nullptr;
    const cudaError_t e = cudaStreamEndCapture(op->st, &g2);
    if (!ok || e != cudaSuccess) {
      if (g2) cudaGraphDestroy(g2);
      ok = false;
    } else {
      graph = g2;
    }
  }
  cudaGetLastError();   // clear any capture error state
  op->st = user_st;
  if (!ok) {              // fall back to live V-cycles for this op
    op->bytes = bsave;
    for (int l = 0; l < 4; ++l) op->mv[l] = msave[l];
    g_launches = l0;
    op->graphs_off = true;
    return;
  }
  helm_op::VGraph vg{};
  vg.adj = adj; vg.nrhs = nrhs; vg.nact = op->nact;
  vg.bytes = op->bytes[r0] - b0;
  for (int l = 0; l < 4; ++l) vg.mv[l] = op->mv[l][r0] - m0[l];
  vg.launches = g_launches - l0;
  op->bytes = bsave;
  for (int l = 0; l < 4; ++l) op->mv[l] = msave[l];
  g_launches = l0;
  const cudaError_t e = cudaGraphInstantiate(&vg.exec, graph, 0);
  cudaGraphDestroy(graph);
  CK(e);
  vg.sig = op->gsig;
  op->trim_graphs();
  op->vgraphs.push_back(vg);
}

// ------------------------------------------------------------------------------ solve
// Outer FGMRES(k_inner) in complex128 against the fp64 operator (D15), restarted until the
// TRUE relative residual of every RHS is <= rtol (R23); converged RHS are masked out.
void solve_c128(helm_op* op, int adj, int nrhs, const double2* B, double2* X, const helm_solve_opts& so,
                helm_solve_report* rep) {
  const long long N = op->lev[0].N;
  reset_acct(op, nrhs);
  set_active(op, nrhs);
  CK(cudaMemsetAsync(X, 0, sizeof(double2) * N * nrhs, op->st));
  // Early stop inside a cycle (R23: "the Arnoldi estimate is allowed only for early stopping
  // inside a cycle"): when the residual estimate |g_{j+1}| of a RHS reaches 0.5 rtol ||b||
  // after inner step j, its cycle closes at j + 1 columns (finalize_column, as on a breakdown),
  // the RHS leaves the cycle's remaining steps, and the solution update reads j + 1 columns.
  // Convergence is still decided on the TRUE residual at the next cycle start. HELM_EARLY=0:
  // every cycle runs all k_inner steps.
  static const bool early = env_int("HELM_EARLY", 1) != 0;
  KCtx ctx = op->ctxO;
  ctx.k = op->k_inner;
  if (!early) ctx.tol = nullptr;
  std::vector<double> bn(nrhs), beta(nrhs), rel(nrhs, 1.0), tolh(nrhs, 0.0);
  std::vector<int> cycles(nrhs, 0), kact_h(nrhs, 0);
  launch_norm_start<double>(op, 0, nrhs, B, ctx);
  CK(cudaMemcpyAsync(bn.data(), ctx.beta, sizeof(double) * nrhs, cudaMemcpyDeviceToHost, op->st));
  CK(cudaStreamSynchronize(op->st));
  if (early) {
    // HELM_EARLY_PCT: the factor in percent (default 50; measured in profiles/r02/ab_r2z,
    // gpu_tests_r2aa: at 98 exit residuals sit at 0.9-1.0 rtol and the north star's 1e-5 bar on
    // f fails on tiny2d (1.6e-5); at 50 every parity test holds its bar)
    static const double fac = 0.01 * std::min(100, std::max(1, env_int("HELM_EARLY_PCT", 50)));
    for (int r = 0; r < nrhs; ++r) tolh[r] = fac * so.rtol * bn[r];
    CK(cudaMemcpyAsync(ctx.tol, tolh.data(), sizeof(double) * nrhs, cudaMemcpyHostToDevice, op->st));
  }
  const bool precond = so.precond != 0 && op->L >= 2;
  Precond<double> M;
  if (precond) {
    if (op->dtype == HELM_C128) {
      M = [op, adj, nrhs](const double2* v, const double* vs, const int* kact, int j, double2* z) {
        launch_copy_scale<double2, double2>(op, 0, nrhs, v, op->w64[0].VB, vs, kact, j);
        vcycle0_graph<double>(op, adj, nrhs, op->w64[0].VB, op->w64[0].VX);
        launch_copy_scale<double2, double2>(op, 0, nrhs, op->w64[0].VX, z, nullptr, nullptr, 0);
      };
    } else {
      M = [op, adj, nrhs](const double2* v, const double* vs, const int* kact, int j, double2* z) {
        launch_copy_scale<double2, float2>(op, 0, nrhs, v, op->w32[0].VB, vs, kact, j);
        vcycle0_graph<float>(op, adj, nrhs, op->w32[0].VB, op->w32[0].VX);
        launch_copy_scale<float2, double2>(op, 0, nrhs, op->w32[0].VX, z, nullptr, nullptr, 0);
      };
    }
  }
  for (int cyc = 0;; ++cyc) {
    const double2* v0;
    if (cyc == 0) {
      beta = bn;
      v0 = B;
    } else {
      launch_stencil<double>(op, 0, adj, 1, nrhs, X, op->OV[0], B, nullptr, nullptr, 0, ctx);
      CK(cudaMemcpyAsync(beta.data(), ctx.beta, sizeof(double) * nrhs, cudaMemcpyDeviceToHost, op->st));
      CK(cudaStreamSynchronize(op->st));
      v0 = op->OV[0];
    }
    int nact = 0;
    for (int r = 0; r < nrhs; ++r) {
      if (!op->act_h[r]) continue;
      rel[r] = bn[r] > 0 ? beta[r] / bn[r] : 0.0;
      if (rel[r] <= so.rtol || cycles[r] >= so.max_outer) op->act_h[r] = 0;
      else ++nact;
    }
    if (!nact) break;
    set_active(op, nrhs);
    const int ki = op->k_inner;
    const std::vector<int> cyc_act = op->act_h;   // the cycle's RHS (the solution update runs over these)
    bool shrunk = false;
    for (int j = 0; j < ki; ++j) {
      VPtrs<double> Vp = vptrs<double>(op->OV, v0, j + 1);
      const double2* zj;
      const double* zs;
      if (precond) {
        M(Vp.p[j], ctx.scale + j, ctx.kact, j, op->OZ[j]);
        zj = op->OZ[j];
        zs = nullptr;
      } else {
        zj = Vp.p[j];
        zs = ctx.scale + j;
      }
      launch_plane<double>(op, 0, adj, 2, nrhs, zj, op->OV[j + 1], nullptr, &Vp, j + 1, zs, ctx.kact, j, ctx);
      launch_update<double>(op, 0, nrhs, Vp, j, op->OV[j + 1], ctx);
      if (early && j + 1 < ki) {
        // RHS whose cycle closed at column j (estimate reached, or breakdown) sit out the rest
        CK(cudaMemcpyAsync(kact_h.data(), ctx.kact, sizeof(int) * nrhs, cudaMemcpyDeviceToHost, op->st));
        CK(cudaStreamSynchronize(op->st));
        int still = 0;
        bool changed = false;
        for (int r = 0; r < nrhs; ++r) {
          if (!op->act_h[r]) continue;
          if (kact_h[r] <= j + 1) { op->act_h[r] = 0; changed = true; }
          else ++still;
        }
        shrunk = shrunk || changed;
        if (!still) break;
        if (changed) set_active(op, nrhs);
      }
    }
    if (shrunk) {
      op->act_h = cyc_act;
      set_active(op, nrhs);
    }
    if (precond) {
      VPtrs<double> Zp{};
      for (int i = 0; i < ki; ++i) Zp.p[i] = op->OZ[i];
      launch_solupdate<double>(op, 0, nrhs, Zp, nullptr, X, 0, ki, ctx);
    } else {
      VPtrs<double> Vp = vptrs<double>(op->OV, v0, ki);
      launch_solupdate<double>(op, 0, nrhs, Vp, ctx.scale, X, 0, ki, ctx);
    }
    for (int r = 0; r < nrhs; ++r)
      if (op->act_h[r]) cycles[r]++;
  }
  CK(cudaStreamSynchronize(op->st));
  if (rep)
    for (int r = 0; r < nrhs; ++r) {
      rep[r].outer_cycles = cycles[r];
      rep[r].rel_residual = rel[r];
      rep[r].converged = rel[r] <= so.rtol;
      for (int l = 0; l < 4; ++l) rep[r].matvecs[l] = op->mv[l][r];
      rep[r].bytes_alg = op->bytes[r];
    }
}

helm_solve_opts default_solve_opts(const helm_op* op) { return helm_solve_opts{op->k_inner, 50, 1e-6, 1}; }

void check_solve_opts(const helm_op* op, const helm_solve_opts& so) {
  REQ(so.k_inner == op->k_inner, HELM_ERR_ARG, "opts.k_inner must equal the op's k_inner (5)");
  REQ(so.max_outer >= 0 && so.rtol > 0 && so.rtol < 1, HELM_ERR_ARG, "bad solve options");
}

void solve_any(helm_op* op, int adj, int nrhs, const void* b, void* x, const helm_solve_opts& so, helm_solve_report* rep) {
  const long long N = op->lev[0].N;
  if (op->dtype == HELM_C128) {
    solve_c128(op, adj, nrhs, (const double2*)b, (double2*)x, so, rep);
  } else {
    std::fill(op->act_h.begin(), op->act_h.end(), 1);
    set_active(op, nrhs);
    launch_copy_scale<float2, double2>(op, 0, nrhs, (const float2*)b, op->OB, nullptr, nullptr, 0);
    solve_c128(op, adj, nrhs, op->OB, op->OX, so, rep);
    std::fill(op->act_h.begin(), op->act_h.end(), 1);
    set_active(op, nrhs);
    launch_copy_scale<double2, float2>(op, 0, nrhs, op->OX, (float2*)x, nullptr, nullptr, 0);
    if (rep)   // the two c64 <-> c128 conversions around the outer solve
      for (int r = 0; r < nrhs; ++r) rep[r].bytes_alg += 2.0 * 24.0 * N;
    CK(cudaStreamSynchronize(op->st));
  }
}

// ------------------------------------------------------------------------------ FWI
struct FwiBufs {
  void *U = nullptr, *V = nullptr, *Bq = nullptr, *A = nullptr;
  double2* d = nullptr;
  long long *src_ext = nullptr, *rec_ext = nullptr;
  double *gext = nullptr, *f = nullptr;
  std::vector<void*> keep;
  ~FwiBufs() { for (void* p : keep) cudaFree(p); }
};

std::vector<long long> to_ext(const helm_grid& G, const int64_t* ids, int n) {
  std::vector<long long> e(n);
  const long long nx = G.n[0], ny = G.n[1], nz = G.n[2];
  const long long Nx = nx + G.pml[0][0] + G.pml[0][1], Ny = ny + G.pml[1][0] + G.pml[1][1];
  for (int i = 0; i < n; ++i) {
    REQ(ids[i] >= 0 && ids[i] < nx * ny * nz, HELM_ERR_ARG, "node id out of the interior");
    long long ix = ids[i] % nx, iy = (ids[i] / nx) % ny, iz = ids[i] / (nx * ny);
    e[i] = (ix + G.pml[0][0]) + Nx * ((iy + G.pml[1][0]) + Ny * (iz + G.pml[2][0]));
  }
  return e;
}

// Off-grid points (helm_acq): Kaiser-windowed sinc rows of P (DESIGN R33) built on
// the host — 1D weights sinc(t-k) I0(b sqrt(1-((t-k)/r)^2)) / I0(b), |t-k| <= r, normalised per
// axis after dropping taps outside the extended grid, tensor product over the axes.
struct TapRows {
  std::vector<int> off{0};
  std::vector<long long> node;
  std::vector<double> w;
};
static double sinc_pi(double x) { return x == 0.0 ? 1.0 : std::sin(M_PI * x) / (M_PI * x); }
static void ks_axis(double t, int n_ext, int lo, double b, int r, std::vector<long long>& e, std::vector<double>& w) {
  e.clear(); w.clear();
  double sum = 0.0;
  const double i0b = std::cyl_bessel_i(0.0, b);
  for (long long k = (long long)std::ceil(t - r); k <= (long long)std::floor(t + r); ++k) {
    const long long ek = k + lo;
    if (ek < 0 || ek >= n_ext) continue;
    const double d = t - (double)k, q = 1.0 - (d / r) * (d / r);
    const double wk = sinc_pi(d) * std::cyl_bessel_i(0.0, b * std::sqrt(std::max(q, 0.0))) / i0b;
    e.push_back(ek); w.push_back(wk); sum += wk;
  }
  for (double& x : w) x /= sum;
}
static TapRows build_taps(const helm_grid& G, const double* xyz, int npts, double b, int r) {
  TapRows T;
  const int Ne[3] = {(int)(G.n[0] + G.pml[0][0] + G.pml[0][1]), (int)(G.n[1] + G.pml[1][0] + G.pml[1][1]),
                     (int)(G.n[2] + G.pml[2][0] + G.pml[2][1])};
  std::vector<long long> e[3];
  std::vector<double> w[3];
  for (int p = 0; p < npts; ++p) {
    for (int a = 0; a < 3; ++a) {
      const double c = xyz[3 * p + a];
      if (a == 1 && G.ndim == 2) {
        REQ(c == 0.0, HELM_ERR_ARG, "2D acquisition points need y = 0");
        e[1].assign(1, 0); w[1].assign(1, 1.0);
        continue;
      }
      REQ(std::isfinite(c) && c >= 0.0 && c <= (double)(G.n[a] - 1) * G.h, HELM_ERR_ARG,
          "acquisition point " + std::to_string(p) + " outside the interior along axis " + std::to_string(a));
      ks_axis(c / G.h, Ne[a], (int)G.pml[a][0], b, r, e[a], w[a]);
    }
    for (size_t kz = 0; kz < e[2].size(); ++kz)
      for (size_t ky = 0; ky < e[1].size(); ++ky)
        for (size_t kx = 0; kx < e[0].size(); ++kx) {
          T.node.push_back((e[2][kz] * Ne[1] + e[1][ky]) * Ne[0] + e[0][kx]);
          T.w.push_back(w[2][kz] * w[1][ky] * w[0][kx]);
        }
    T.off.push_back((int)T.node.size());
  }
  return T;
}
// Rows of P^T: touched nodes in increasing order, each with its (point, weight) taps in
// increasing point order — the adjoint source is then a deterministic gather.
struct TapRowsT {
  std::vector<int> off{0}, pt;
  std::vector<long long> node;
  std::vector<double> w;
};
static TapRowsT transpose_taps(const TapRows& T) {
  std::vector<std::tuple<long long, int, double>> e;
  for (int p = 0; p + 1 < (int)T.off.size(); ++p)
    for (int t = T.off[p]; t < T.off[p + 1]; ++t) e.emplace_back(T.node[t], p, T.w[t]);
  std::sort(e.begin(), e.end());
  TapRowsT R;
  for (size_t i = 0; i < e.size(); ++i) {
    if (i > 0 && std::get<0>(e[i]) != std::get<0>(e[i - 1])) R.off.push_back((int)i);
    if (i == 0 || std::get<0>(e[i]) != std::get<0>(e[i - 1])) R.node.push_back(std::get<0>(e[i]));
    R.pt.push_back(std::get<1>(e[i]));
    R.w.push_back(std::get<2>(e[i]));
  }
  R.off.push_back((int)e.size());
  if (e.empty()) R.off.assign(1, 0);
  return R;
}
template <typename T> T* upload(std::vector<void*>& keep, const std::vector<T>& v, cudaStream_t st) {
  T* d = dalloc<T>(keep, std::max<size_t>(v.size(), 1));
  if (!v.empty()) CK(cudaMemcpyAsync(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, st));
  return d;
}

// Listing 1's PDEfunc modes over this rank's (frequency, source) pairs:
//   OBJ     f = sum 1/2 |P_r u - d|^2 and g = T^* V (2 solves per pair)
//   FORW    d = P_r u (1 solve)
//   JAC     d_lin = P_r Du[dm], Du[dm] = -H^-1 T dm (2 solves)
//   JACADJ  g = T^* H^-H (-P_r^T y) (2 solves)
//   GN      g = T^* H^-H (-P_r^T P_r Du[dm]) (3 solves, Table 2)
// The pairs are processed in joint batches of up to max_rhs right-hand sides (frequency-major
// order): each batch is ONE batched solve per stage whose RHS may use different frequencies
// (per-RHS operator tables, Geo::rop) — the paper's data parallelism over the joint (source,
// frequency) index set (Fig. 2) inside one GPU.
enum FwiMode { FW_OBJ = 0, FW_FORW, FW_JAC, FW_JACADJ, FW_GN };

template <typename R>
void fwi_run(helm_op* op, const helm_grid& G, FwiMode mode, int nfreq, const double* freq, const double* sw,
             int nsrc_total, int s_begin, int s_end, const int64_t* src, int nrec, const int64_t* rec,
             const double* dobs /* OBJ: d_obs, JACADJ: y; host [nfreq][nsrc_total][nrec] */,
             const double* dm /* JAC, GN: host interior */, const helm_solve_opts& so, double* out /* OBJ: [f|g],
             JACADJ/GN: g */, helm_solve_report* rep, double* d_out /* FORW, JAC: host [nfreq][ns][nrec] */,
             cudaStream_t st, const helm_acq* acq = nullptr /* off-grid points instead of src / rec nodes */,
             const uint8_t* mask = nullptr /* [nfreq][nsrc_total]: the (frequency, source) pairs to evaluate */) {
  using C = cx<R>;
  FwiBufs fb;
  const long long N = op->lev[0].N;
  const int B = op->max_rhs;
  const int ns = s_end - s_begin;
  const bool grad = mode == FW_OBJ || mode == FW_JACADJ || mode == FW_GN;
  const bool born = mode == FW_JAC || mode == FW_GN;
  const int rs = mode == FW_GN ? 3 : 2;   // report stride per pair
  fb.U = dalloc<C>(fb.keep, (size_t)N * B);
  fb.Bq = dalloc<C>(fb.keep, (size_t)N * B);
  void* dU = born ? dalloc<C>(fb.keep, (size_t)N * B) : nullptr;
  if (grad) {
    fb.V = dalloc<C>(fb.keep, (size_t)N * B);
    fb.A = dalloc<C>(fb.keep, (size_t)N * B);
    fb.gext = dalloc<double>(fb.keep, N);
    fb.f = dalloc<double>(fb.keep, 1);
    CK(cudaMemsetAsync(fb.gext, 0, sizeof(double) * N, st));
    CK(cudaMemsetAsync(fb.f, 0, sizeof(double), st));
  }
  double* dm_ext = nullptr;
  if (born) {   // dm_ext = E dm (D2)
    const long long nint = G.n[0] * G.n[1] * G.n[2];
    double* dm_int = dalloc<double>(fb.keep, nint);
    dm_ext = dalloc<double>(fb.keep, N);
    CK(cudaMemcpyAsync(dm_int, dm, sizeof(double) * nint, cudaMemcpyHostToDevice, st));
    const LevelDev& L0 = op->lev[0];
    prof_count(KC_FWI);
    k_extend<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(L0.nx, L0.ny, L0.nz, (int)G.n[0], (int)G.n[1], (int)G.n[2],
                                                          G.pml[0][0], G.pml[1][0], G.pml[2][0], dm_int, dm_ext);
    CKL();
  }
  fb.d = dalloc<double2>(fb.keep, (size_t)B * std::max(nrec, 1));
  double2* amp_d = dalloc<double2>(fb.keep, B);
  double* w2_d = dalloc<double>(fb.keep, B);
  long long* srcb_d = dalloc<long long>(fb.keep, B);
  const bool offg = acq != nullptr;
  std::vector<long long> sext, rext;
  // off-grid: P_s rows of this shard's sources, P_r rows and P_r^T rows on the device
  int *ps_off = nullptr, *pr_off = nullptr, *prt_off = nullptr, *prt_pt = nullptr, nprt = 0;
  long long *ps_node = nullptr, *pr_node = nullptr, *prt_node = nullptr;
  double *ps_w = nullptr, *pr_w = nullptr, *prt_w = nullptr;
  double2* rres = nullptr;
  if (offg) {
    const double kb = acq->kaiser_b > 0 ? acq->kaiser_b : 6.31;
    const int kr = acq->half_width > 0 ? acq->half_width : 4;
    REQ(kr <= 8, HELM_ERR_ARG, "half_width must be <= 8");
    const TapRows Ps = build_taps(G, acq->src_xyz + 3 * (size_t)s_begin, ns, kb, kr);
    const TapRows Pr = build_taps(G, acq->rec_xyz, nrec, kb, kr);
    const TapRowsT PrT = transpose_taps(Pr);
    ps_off = upload(fb.keep, Ps.off, st); ps_node = upload(fb.keep, Ps.node, st); ps_w = upload(fb.keep, Ps.w, st);
    pr_off = upload(fb.keep, Pr.off, st); pr_node = upload(fb.keep, Pr.node, st); pr_w = upload(fb.keep, Pr.w, st);
    prt_off = upload(fb.keep, PrT.off, st); prt_node = upload(fb.keep, PrT.node, st);
    prt_pt = upload(fb.keep, PrT.pt, st); prt_w = upload(fb.keep, PrT.w, st);
    nprt = (int)PrT.node.size();
    rres = dalloc<double2>(fb.keep, (size_t)B * std::max(nrec, 1));
    CK(cudaStreamSynchronize(st));   // the host tap vectors go out of scope
  } else {
    sext = to_ext(G, src + s_begin, ns);
    rext = to_ext(G, rec, nrec);
    std::vector<long long> sr = rext;
    std::sort(sr.begin(), sr.end());
    REQ(std::adjacent_find(sr.begin(), sr.end()) == sr.end(), HELM_ERR_ARG, "receivers must be distinct nodes");
  }
  fb.rec_ext = dalloc<long long>(fb.keep, std::max(nrec, 1));
  if (nrec && !offg) CK(cudaMemcpyAsync(fb.rec_ext, rext.data(), sizeof(long long) * nrec, cudaMemcpyHostToDevice, st));
  const unsigned gq = (unsigned)((B * (long long)std::max(nrec, 1) + 255) / 256);
  auto rec_gather = [&](int nb, const void* Uf, const double2* d, double2* o) {   // o = P_r u - d
    prof_count(KC_FWI);
    k_rec_gather<R><<<gq, 256, 0, st>>>(nb, nrec, N, pr_off, pr_node, pr_w, (const C*)Uf, d, o);
    CKL();
  };
  auto rec_scatterT = [&](int nb, const double2* r) {   // A = -P_r^T r
    if (!nprt) return;
    prof_count(KC_FWI);
    k_rec_scatterT<R><<<(unsigned)((nb * (long long)nprt + 255) / 256), 256, 0, st>>>(nb, nprt, nrec, N, prt_off,
                                                                                   prt_node, prt_pt, prt_w, r, (C*)fb.A);
    CKL();
  };
  const double hd = std::pow(G.h, (double)G.ndim);
  std::vector<helm_solve_report> rtmp(B);
  std::vector<double2> amp_h(B), dbat((size_t)B * std::max(nrec, 1));
  std::vector<double> w2_h(B), wop;
  std::vector<long long> srcb_h(B);
  std::vector<int> rop_h(B), fi_h(B), si_h(B);
  // the (frequency, source) pairs of this call, frequency-major: all of this shard's, or the
  // ones `mask` selects (the paper's batch-mode subset interface)
  std::vector<int> pf, ps;
  for (int f = 0; f < nfreq; ++f)
    for (int s = 0; s < ns; ++s)
      if (!mask || mask[(size_t)f * nsrc_total + s_begin + s]) { pf.push_back(f); ps.push_back(s); }
  const long long npairs = (long long)pf.size();
  long long p0 = 0;
  auto put_rep = [&](int nb, int k) {   // reports in pair order
    if (rep)
      for (int b = 0; b < nb; ++b) rep[(size_t)(p0 + b) * rs + k] = rtmp[b];
  };
  auto gather_out = [&](int nb, const void* Ufield) {   // d_out[f][s][:] = P_r field
    if (!nrec) return;
    if (offg) {
      rec_gather(nb, Ufield, nullptr, fb.d);
    } else {
      prof_count(KC_FWI);
      k_gather_data<R><<<(unsigned)((nb * (long long)nrec + 255) / 256), 256, 0, st>>>(nb, nrec, N, fb.rec_ext,
                                                                                  (const C*)Ufield, fb.d);
      CKL();
    }
    CK(cudaMemcpyAsync(dbat.data(), fb.d, sizeof(double2) * nb * nrec, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int b = 0; b < nb; ++b)
      std::memcpy(d_out + 2 * (((size_t)fi_h[b] * ns + si_h[b]) * nrec), &dbat[(size_t)b * nrec], sizeof(double2) * nrec);
  };
  // operators one joint batch may hold: HELM_MAXOP, and in 2D what the march kernel's
  // shared-memory z table takes (deep 2D grids x many frequencies)
  const int max_ops = op->dim == 2 ? march_max_ops<R>(op->lev[0].nz) : HELM_MAXOP;
  REQ(max_ops >= 1, HELM_ERR_SHAPE, "2D grid too deep for the march kernel (nz_ext = " +
                                        std::to_string(op->lev[0].nz) + ")");
  int nb = 0;
  for (p0 = 0; p0 < npairs; p0 += nb) {
    // the batch: up to B pairs in order, closed early before a (max_ops + 1)-th frequency
    nb = 0;
    for (int nf = 0, lf = -1; nb < B && p0 + nb < npairs; ++nb) {
      if (pf[p0 + nb] != lf) {
        if (nf == max_ops) break;
        ++nf;
        lf = pf[p0 + nb];
      }
    }
    // the batch's operators (distinct frequencies, in order) and per-RHS data
    wop.clear();
    int last_f = -1;
    for (int b = 0; b < nb; ++b) {
      const int fi = pf[p0 + b], si = ps[p0 + b];
      if (fi != last_f) { wop.push_back(2.0 * M_PI * freq[fi]); last_f = fi; }
      fi_h[b] = fi; si_h[b] = si; rop_h[b] = (int)wop.size() - 1;
      const double2 S = sw ? make_double2(sw[2 * fi], sw[2 * fi + 1]) : make_double2(1.0, 0.0);
      amp_h[b] = make_double2(S.x / hd, S.y / hd);
      w2_h[b] = wop.back() * wop.back();
      srcb_h[b] = offg ? si : sext[si];
    }
    REQ((int)wop.size() <= max_ops, HELM_ERR_STATE, "joint batch holds too many operators");
    op_set_omegas(op, wop.data(), (int)wop.size());
    op_set_rop(op, rop_h);
    CK(cudaMemcpyAsync(amp_d, amp_h.data(), sizeof(double2) * nb, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(w2_d, w2_h.data(), sizeof(double) * nb, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(srcb_d, srcb_h.data(), sizeof(long long) * nb, cudaMemcpyHostToDevice, st));
    // a7: inject q = S(omega) e_s / h^d
    CK(cudaMemsetAsync(fb.Bq, 0, sizeof(C) * N * nb, st));
    prof_count(KC_FWI);
    if (offg)   // q = S(omega) P_s^T e_s / h^d
      k_inject_taps<R><<<nb, 256, 0, st>>>(nb, N, srcb_d, ps_off, ps_node, ps_w, amp_d, (C*)fb.Bq);
    else
      k_inject<R><<<(nb + 127) / 128, 128, 0, st>>>(nb, N, srcb_d, amp_d, (C*)fb.Bq);
    CKL();
    // forward solves u = H^-1 q
    solve_any(op, 0, nb, fb.Bq, fb.U, so, rtmp.data());
    put_rep(nb, 0);
    if (mode == FW_FORW) { gather_out(nb, fb.U); continue; }
    if (born) {   // Du[dm] = -H^-1 T dm
      prof_count(KC_FWI);
      k_born_src<R><<<TARGET_BLOCKS, 256, 0, st>>>(nb, N, w2_d, (const C*)fb.U, dm_ext, (C*)fb.Bq);
      CKL();
      solve_any(op, 0, nb, fb.Bq, dU, so, rtmp.data());
      put_rep(nb, 1);
      if (mode == FW_JAC) { gather_out(nb, dU); continue; }
    }
    // adjoint source: OBJ: -P_r^T (P_r u - d) (+ f); JACADJ: -P_r^T y; GN: -P_r^T P_r Du[dm]
    if (mode != FW_GN && nrec) {
      for (int b = 0; b < nb; ++b)
        std::memcpy(&dbat[(size_t)b * nrec], dobs + 2 * (((size_t)fi_h[b] * nsrc_total + s_begin + si_h[b]) * nrec),
                    sizeof(double2) * nrec);
      CK(cudaMemcpyAsync(fb.d, dbat.data(), sizeof(double2) * nb * nrec, cudaMemcpyHostToDevice, st));
    }
    CK(cudaMemsetAsync(fb.A, 0, sizeof(C) * N * nb, st));
    if (nrec && offg) {
      if (mode == FW_JACADJ) {
        rec_scatterT(nb, fb.d);                                  // -P_r^T y
      } else if (mode == FW_GN) {
        rec_gather(nb, dU, nullptr, rres);                       // P_r Du
        rec_scatterT(nb, rres);
      } else {
        rec_gather(nb, fb.U, fb.d, rres);                        // r = P_r u - d
        prof_count(KC_FWI);
        k_half_sumsq<<<1, 1024, 0, st>>>((long long)nb * nrec, rres, fb.f);
        CKL();
        rec_scatterT(nb, rres);
      }
    } else if (nrec) {
      if (mode == FW_JACADJ) {
        prof_count(KC_FWI);
        k_scatter_neg<R><<<(unsigned)((nb * (long long)nrec + 255) / 256), 256, 0, st>>>(nb, nrec, N, fb.rec_ext, fb.d,
                                                                                    (C*)fb.A);
        CKL();
      } else {
        if (mode == FW_GN) CK(cudaMemsetAsync(fb.d, 0, sizeof(double2) * nb * nrec, st));   // "data" = 0
        dim3 gg(std::max(1, std::min(TARGET_BLOCKS, (nb * nrec + 255) / 256)));
        prof_count(KC_FWI);
        k_gather_residual<R><<<gg, HELM_RED_THREADS, 0, st>>>(nb, nrec, N, fb.rec_ext, fb.d,
                                                                (const C*)(mode == FW_GN ? dU : fb.U), (C*)fb.A, fb.f,
                                                                op->rb);
        CKL();
      }
    }
    // a8: adjoint solves
    solve_any(op, 1, nb, fb.A, fb.V, so, rtmp.data());
    put_rep(nb, rs - 1);
    // a9: g_ext += sum_b Re(omega_b^2 conj(u_b) (A^H v_b)), A = I (STD2) or M (OPT, Eq. 7)
    prof_count(KC_FWI);
    if (G.stencil == HELM_OPT)
      k_grad_opt<R><<<blas_blocks(N, 1), 256, 0, st>>>(nb, op->lev[0].nx, op->lev[0].ny, op->lev[0].nz, w2_d,
                                                      (const C*)fb.U, (const C*)fb.V, fb.gext);
    else
      k_grad<R><<<blas_blocks(N, 1), 256, 0, st>>>(nb, N, w2_d, (const C*)fb.U, (const C*)fb.V, fb.gext);
    CKL();
  }
  if (grad) {
    const long long nint = G.n[0] * G.n[1] * G.n[2];
    prof_count(KC_FWI);
    k_fold<<<(unsigned)((nint + 255) / 256), 256, 0, st>>>(op->lev[0].nx, op->lev[0].ny, op->lev[0].nz, (int)G.n[0],
                                                           (int)G.n[1], (int)G.n[2], G.pml[0][0], G.pml[1][0],
                                                           G.pml[2][0], fb.gext, mode == FW_OBJ ? fb.f : nullptr, out);
    CKL();
  }
  CK(cudaStreamSynchronize(st));
}

// One cached op per thread for fwi_*: the device workspace is reused across calls with the
// same geometry, dtype and batch size; model, hierarchy and tables are rebuilt every call.
thread_local helm_op* g_fwi_op = nullptr;

helm_op* fwi_op(const helm_grid* grid, const double* m, double omega, const helm_pml* pml, helm_dtype dtype,
                int max_rhs, cudaStream_t st) {
  helm_op* o = g_fwi_op;
  auto same = [](const helm_grid& a, const helm_grid& b) {
    if (a.ndim != b.ndim || a.h != b.h || a.stencil != b.stencil) return false;
    for (int i = 0; i < 3; ++i)
      if (a.n[i] != b.n[i] || a.pml[i][0] != b.pml[i][0] || a.pml[i][1] != b.pml[i][1]) return false;
    return true;
  };
  int dev = 0;
  CK(cudaGetDevice(&dev));
  if (o && o->device == dev && o->dtype == dtype && o->max_rhs == max_rhs && same(o->grid, *grid)) {
    validate_model_pml(*grid, m, *pml);
    o->st = st;
    o->pml = *pml;
    o->vref = pml->v_ref;
    op_set_model(o, m);
    op_set_omega(o, omega);
    return o;
  }
  delete g_fwi_op;
  g_fwi_op = nullptr;
  g_fwi_op = op_create(grid, m, omega, pml, dtype, max_rhs, nullptr, st, 5);
  return g_fwi_op;
}

helm_status wrap(const std::function<void()>& f) {
  try {
    f();
    return HELM_OK;
  } catch (const HelmErr& e) {
    g_err = e.msg;
    return e.st;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return HELM_ERR_OOM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HELM_ERR_STATE;
  }
}

void* level_ptr_check(const helm_op* op, int level) {
  REQ(op, HELM_ERR_ARG, "op is NULL");
  REQ(level >= 0 && level < op->L, HELM_ERR_ARG, "level out of range");
  return nullptr;
}

// Measurement probe: `reps` back-to-back launches of one hot-path kernel on the op's level
// workspace (CUDA events on the stream; average ms per launch). kind 0-4 = plane modes
// (nv = Krylov step), 10 = solution update (k = nv), 11 = CGS update (j = nv), 12 = norm.
template <typename R>
double probe_run(helm_op* op, int level, int kind, int nv, int nrhs, int reps) {
  LevelWS<R>* W = wsets<R>(op);
  LevelWS<R>& w = W[level];
  const bool sm = level < op->L - 1;
  cx<R>* const* V = sm ? w.SV : w.FV;
  cx<R>* Wx = sm ? w.SW : (w.FW ? w.FW : w.Fx);
  KCtx& ctx = sm ? w.ctxS : w.ctxC;
  REQ(V[0] && Wx, HELM_ERR_STATE, "no workspace on this level");
  const int k = sm ? op->ml.ks_i : op->ml.kc_i;
  REQ(nv >= 0 && (nv < k || (kind == 10 && nv == k)), HELM_ERR_ARG, "nv out of range");
  const long long N = op->lev[level].N;
  for (int i = 0; i <= k; ++i) CK(cudaMemsetAsync(V[i], 0x3f, sizeof(cx<R>) * N * nrhs, op->st));
  CK(cudaMemsetAsync(Wx, 0x3f, sizeof(cx<R>) * N * nrhs, op->st));
  ctx.k = k;
  launch_norm_start<R>(op, level, nrhs, V[0], ctx);
  VPtrs<R> Vp = vptrs<R>(V, V[0], std::max(nv, 1));
  VPtrs<R> Vq = vptrs<R>(V, V[0], nv + 1);
  auto one = [&] {
    if (kind <= 4)
      launch_plane<R>(op, level, 0, kind, nrhs, Wx, V[k], V[1], kind == 2 ? &Vq : &Vp, kind == 2 ? nv + 1 : nv,
                      nullptr, ctx.kact, nv, ctx, kind >= 3 && nv > 0 ? V[nv] : nullptr);
    else if (kind == 10) launch_solupdate<R>(op, level, nrhs, Vp, ctx.scale, Wx, 0, std::max(nv, 1), ctx);
    else if (kind == 11) launch_update<R>(op, level, nrhs, Vq, nv, V[k], ctx);
    else launch_norm_start<R>(op, level, nrhs, V[0], ctx);
  };
  one();
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, op->st));
  for (int i = 0; i < reps; ++i) one();
  CK(cudaEventRecord(e1, op->st));
  CK(cudaEventSynchronize(e1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return ms / reps;
}

}  // namespace

// ================================================================================ C ABI
extern "C" {

helm_status helm_setup(const helm_grid* grid, const double* m, double omega, const helm_pml* pml, helm_dtype dtype,
                       int32_t max_rhs, const helm_mlopts* mlopts, void* stream, helm_op** out) {
  return wrap([&] {
    REQ(out, HELM_ERR_ARG, "out is NULL");
    g_err.clear();
    *out = op_create(grid, m, omega, pml, dtype, max_rhs, mlopts, (cudaStream_t)stream, 5);
  });
}

helm_status helm_apply(helm_op* op, int32_t adjoint, int32_t nrhs, const void* x, void* y, void* stream) {
  return wrap([&] {
    REQ(op && x && y, HELM_ERR_ARG, "NULL argument");
    REQ(nrhs >= 1 && nrhs <= op->max_rhs, HELM_ERR_SHAPE, "nrhs must be in [1, max_rhs]");
    REQ(adjoint == 0 || adjoint == 1, HELM_ERR_ARG, "adjoint must be 0 or 1");
    REQ(x != y, HELM_ERR_ARG, "x and y must not alias");
    op->st = (cudaStream_t)stream;
    reset_acct(op, nrhs);
    std::fill(op->act_h.begin(), op->act_h.begin() + nrhs, 1);
    set_active(op, nrhs);
    if (op->dtype == HELM_C128)
      launch_stencil<double>(op, 0, adjoint, 0, nrhs, (const double2*)x, (double2*)y, nullptr, nullptr, nullptr, 0, op->ctxO);
    else
      launch_stencil<float>(op, 0, adjoint, 0, nrhs, (const float2*)x, (float2*)y, nullptr, nullptr, nullptr, 0, op->ctxO);
  });
}

helm_status helm_solve(helm_op* op, int32_t adjoint, int32_t nrhs, const void* b, void* x, const helm_solve_opts* opts,
                       helm_solve_report* rep, void* stream) {
  return wrap([&] {
    REQ(op && b && x, HELM_ERR_ARG, "NULL argument");
    REQ(nrhs >= 1 && nrhs <= op->max_rhs, HELM_ERR_SHAPE, "nrhs must be in [1, max_rhs]");
    REQ(adjoint == 0 || adjoint == 1, HELM_ERR_ARG, "adjoint must be 0 or 1");
    REQ(b != x, HELM_ERR_ARG, "b and x must not alias");
    REQ(!op->apply_only, HELM_ERR_STATE, "operator-only op (mlopts.levels = 0) cannot solve");
    helm_solve_opts so = opts ? *opts : default_solve_opts(op);
    check_solve_opts(op, so);
    op->st = (cudaStream_t)stream;
    solve_any(op, adjoint, nrhs, b, x, so, rep);
  });
}

static helm_status fwi_common(FwiMode mode, const helm_grid* grid, const double* m, int32_t nfreq,
                              const double* freq, const double* sw, int32_t nsrc_total, int32_t s_begin, int32_t s_end,
                              const int64_t* src, int32_t nrec, const int64_t* rec, const double* dobs,
                              const double* dm, const helm_pml* pml, helm_dtype dtype, const helm_solve_opts* opts,
                              int32_t max_rhs, double* out, helm_solve_report* rep, double* d_out, void* stream,
                              const helm_acq* acq = nullptr, const uint8_t* mask = nullptr) {
  return wrap([&] {
    validate_grid(grid);
    REQ(m && freq && pml && (src || acq), HELM_ERR_ARG, "NULL argument");
    if (acq) REQ(acq->src_xyz && (acq->rec_xyz || nrec == 0), HELM_ERR_ARG, "acq points NULL");
    REQ(nfreq >= 1, HELM_ERR_ARG, "nfreq must be >= 1");
    for (int i = 0; i < nfreq; ++i) REQ(freq[i] > 0, HELM_ERR_ARG, "frequencies must be > 0");
    REQ(pml->v_ref > 0, HELM_ERR_ARG, "fwi requires pml.v_ref > 0 (fixed PML, R31)");
    REQ(0 <= s_begin && s_begin <= s_end && s_end <= nsrc_total, HELM_ERR_ARG, "bad source range");
    REQ(nrec >= 0 && (nrec == 0 || rec || acq), HELM_ERR_ARG, "bad receivers");
    REQ(max_rhs >= 1, HELM_ERR_ARG, "max_rhs must be >= 1");
    if (mode == FW_OBJ || mode == FW_JACADJ) REQ(out && (dobs || nrec == 0), HELM_ERR_ARG, "output / data NULL");
    if (mode == FW_GN) REQ(out && dm, HELM_ERR_ARG, "output / dm NULL");
    if (mode == FW_JAC) REQ(d_out && dm, HELM_ERR_ARG, "d_out / dm NULL");
    if (mode == FW_FORW) REQ(d_out, HELM_ERR_ARG, "d_out NULL");
    if (grid->stencil == HELM_OPT)   // the Born source T dm = omega^2 M (u dm) and the off-grid
                                     // acquisition are implemented for STD2 only (helm.h)
      REQ(mode != FW_JAC && mode != FW_GN && !acq, HELM_ERR_ARG,
          "the OPT stencil supports fwi_misfit_grad, fwi_forward and fwi_jacobian_adjoint only");
    const cudaStream_t st = (cudaStream_t)stream;
    helm_op* op = fwi_op(grid, m, 2.0 * M_PI * freq[0], pml, dtype, max_rhs, st);
    helm_solve_opts so = opts ? *opts : default_solve_opts(op);
    check_solve_opts(op, so);
    const long long nint = grid->n[0] * grid->n[1] * grid->n[2];
    if (s_end == s_begin) {   // empty shard: zero outputs
      if (mode == FW_OBJ) CK(cudaMemsetAsync(out, 0, sizeof(double) * (1 + nint), st));
      if (mode == FW_JACADJ || mode == FW_GN) CK(cudaMemsetAsync(out, 0, sizeof(double) * nint, st));
      CK(cudaStreamSynchronize(st));
      return;
    }
    if (dtype == HELM_C128)
      fwi_run<double>(op, *grid, mode, nfreq, freq, sw, nsrc_total, s_begin, s_end, src, nrec, rec, dobs, dm, so, out,
                      rep, d_out, st, acq, mask);
    else
      fwi_run<float>(op, *grid, mode, nfreq, freq, sw, nsrc_total, s_begin, s_end, src, nrec, rec, dobs, dm, so, out,
                     rep, d_out, st, acq, mask);
  });
}

helm_status fwi_misfit_grad(const helm_grid* grid, const double* m, int32_t nfreq, const double* freq,
                            const double* sw, int32_t nsrc_total, int32_t s_begin, int32_t s_end, const int64_t* src,
                            int32_t nrec, const int64_t* rec, const double* dobs, const helm_pml* pml,
                            helm_dtype dtype, const helm_solve_opts* opts, int32_t max_rhs, double* fg,
                            helm_solve_report* rep, void* stream) {
  return fwi_common(FW_OBJ, grid, m, nfreq, freq, sw, nsrc_total, s_begin, s_end, src, nrec, rec, dobs, nullptr, pml,
                    dtype, opts, max_rhs, fg, rep, nullptr, stream);
}

helm_status fwi_forward(const helm_grid* grid, const double* m, int32_t nfreq, const double* freq, const double* sw,
                        int32_t s_begin, int32_t s_end, const int64_t* src, int32_t nrec, const int64_t* rec,
                        const helm_pml* pml, helm_dtype dtype, const helm_solve_opts* opts, int32_t max_rhs,
                        double* d_host, helm_solve_report* rep, void* stream) {
  if (!d_host) { g_err = "d_host is NULL"; return HELM_ERR_ARG; }
  return fwi_common(FW_FORW, grid, m, nfreq, freq, sw, s_end, s_begin, s_end, src, nrec, rec, nullptr, nullptr, pml,
                    dtype, opts, max_rhs, nullptr, rep, d_host, stream);
}

helm_status fwi_misfit_grad_subset(const helm_grid* grid, const double* m, int32_t nfreq, const double* freq,
                                   const double* sw, int32_t nsrc_total, int32_t s_begin, int32_t s_end,
                                   const int64_t* src, int32_t nrec, const int64_t* rec, const double* dobs,
                                   const uint8_t* pair_mask, const helm_pml* pml, helm_dtype dtype,
                                   const helm_solve_opts* opts, int32_t max_rhs, double* fg, helm_solve_report* rep,
                                   void* stream) {
  if (!pair_mask) { g_err = "pair_mask is NULL"; return HELM_ERR_ARG; }
  return fwi_common(FW_OBJ, grid, m, nfreq, freq, sw, nsrc_total, s_begin, s_end, src, nrec, rec, dobs, nullptr, pml,
                    dtype, opts, max_rhs, fg, rep, nullptr, stream, nullptr, pair_mask);
}

helm_status fwi_misfit_grad_acq(const helm_grid* grid, const double* m, int32_t nfreq, const double* freq,
                                const double* sw, int32_t nsrc_total, int32_t s_begin, int32_t s_end, int32_t nrec,
                                const helm_acq* acq, const double* dobs, const helm_pml* pml, helm_dtype dtype,
                                const helm_solve_opts* opts, int32_t max_rhs, double* fg, helm_solve_report* rep,
                                void* stream) {
  if (!acq) { g_err = "acq is NULL"; return HELM_ERR_ARG; }
  return fwi_common(FW_OBJ, grid, m, nfreq, freq, sw, nsrc_total, s_begin, s_end, nullptr, nrec, nullptr, dobs, nullptr,
                    pml, dtype, opts, max_rhs, fg, rep, nullptr, stream, acq);
}

helm_status fwi_forward_acq(const helm_grid* grid, const double* m, int32_t nfreq, const double* freq, const double* sw,
                            int32_t nsrc_total, int32_t s_begin, int32_t s_end, int32_t nrec, const helm_acq* acq,
                            const helm_pml* pml, helm_dtype dtype, const helm_solve_opts* opts, int32_t max_rhs,
                            double* d_host, helm_solve_report* rep, void* stream) {
  if (!acq || !d_host) { g_err = "acq / d_host is NULL"; return HELM_ERR_ARG; }
  return fwi_common(FW_FORW, grid, m, nfreq, freq, sw, nsrc_total, s_begin, s_end, nullptr, nrec, nullptr, nullptr,
                    nullptr, pml, dtype, opts, max_rhs, nullptr, rep, d_host, stream, acq);
}

helm_status fwi_jacobian(const helm_grid* grid, const double* m, int32_t nfreq, const double* freq, const double* sw,
                         int32_t s_begin, int32_t s_end, const int64_t* src, int32_t nrec, const int64_t* rec,
                         const double* dm, const helm_pml* pml, helm_dtype dtype, const helm_solve_opts* opts,
                         int32_t max_rhs, double* d_host, helm_solve_report* rep, void* stream) {
  if (!d_host || !dm) { g_err = "d_host / dm is NULL"; return HELM_ERR_ARG; }
  return fwi_common(FW_JAC, grid, m, nfreq, freq, sw, s_end, s_begin, s_end, src, nrec, rec, nullptr, dm, pml, dtype,
                    opts, max_rhs, nullptr, rep, d_host, stream);
}

helm_status fwi_jacobian_adjoint(const helm_grid* grid, const double* m, int32_t nfreq, const double* freq,
                                 const double* sw, int32_t nsrc_total, int32_t s_begin, int32_t s_end,
                                 const int64_t* src, int32_t nrec, const int64_t* rec, const double* y,
                                 const helm_pml* pml, helm_dtype dtype, const helm_solve_opts* opts, int32_t max_rhs,
                                 double* g_dev, helm_solve_report* rep, void* stream) {
  return fwi_common(FW_JACADJ, grid, m, nfreq, freq, sw, nsrc_total, s_begin, s_end, src, nrec, rec, y, nullptr, pml,
                    dtype, opts, max_rhs, g_dev, rep, nullptr, stream);
}

helm_status fwi_gn_hessian(const helm_grid* grid, const double* m, int32_t nfreq, const double* freq, const double* sw,
                           int32_t s_begin, int32_t s_end, const int64_t* src, int32_t nrec, const int64_t* rec,
                           const double* dm, const helm_pml* pml, helm_dtype dtype, const helm_solve_opts* opts,
                           int32_t max_rhs, double* h_dev, helm_solve_report* rep, void* stream) {
  return fwi_common(FW_GN, grid, m, nfreq, freq, sw, s_end, s_begin, s_end, src, nrec, rec, nullptr, dm, pml, dtype,
                    opts, max_rhs, h_dev, rep, nullptr, stream);
}

helm_status helm_levels(const helm_op* op, int32_t* levels, int64_t* dims) {
  return wrap([&] {
    REQ(op && levels, HELM_ERR_ARG, "NULL argument");
    *levels = op->L;
    if (dims)
      for (int l = 0; l < op->L; ++l) {
        dims[3 * l] = op->lev[l].nx; dims[3 * l + 1] = op->lev[l].ny; dims[3 * l + 2] = op->lev[l].nz;
      }
  });
}

helm_status helm_get_level(const helm_op* op, int32_t level, int32_t adjoint, int64_t nmax, double* tables,
                           double* m_host) {
  return wrap([&] {
    level_ptr_check(op, level);
    REQ(adjoint == 0 || adjoint == 1, HELM_ERR_ARG, "adjoint must be 0 or 1");
    const LevelDev& Lv = op->lev[level];
    const int Ns[3] = {Lv.nx, Lv.ny, Lv.nz};
    REQ(nmax >= *std::max_element(Ns, Ns + 3), HELM_ERR_SHAPE, "nmax smaller than the largest axis");
    CK(cudaStreamSynchronize(op->st));
    if (tables) {
      std::memset(tables, 0, sizeof(double) * 2 * 9 * nmax);
      for (int a = 0; a < 3; ++a)
        for (int t = 0; t < 3; ++t)
          CK(cudaMemcpy(tables + 2 * ((size_t)(a * 3 + t) * nmax), Lv.t64[adjoint][a][t], sizeof(double2) * Ns[a],
                        cudaMemcpyDeviceToHost));
    }
    if (m_host) CK(cudaMemcpy(m_host, Lv.m64, sizeof(double) * Lv.N, cudaMemcpyDeviceToHost));
  });
}

helm_status helm_vcycle(helm_op* op, int32_t level, int32_t adjoint, int32_t nrhs, const void* b, void* z, void* stream) {
  return wrap([&] {
    level_ptr_check(op, level);
    REQ(!op->apply_only, HELM_ERR_STATE, "operator-only op");
    REQ(level < op->L - 1, HELM_ERR_ARG, "no V-cycle on the coarsest level");
    REQ(b && z && b != z, HELM_ERR_ARG, "bad vectors");
    REQ(nrhs >= 1 && nrhs <= op->max_rhs, HELM_ERR_SHAPE, "nrhs must be in [1, max_rhs]");
    op->st = (cudaStream_t)stream;
    reset_acct(op, nrhs);
    set_active(op, nrhs);
    if (op->dtype == HELM_C128) {
      launch_copy_scale<double2, double2>(op, level, nrhs, (const double2*)b, op->w64[level].VB, nullptr, nullptr, 0);
      vcycle<double>(op, level, adjoint, nrhs, op->w64[level].VB, (double2*)z);
    } else {
      launch_copy_scale<float2, float2>(op, level, nrhs, (const float2*)b, op->w32[level].VB, nullptr, nullptr, 0);
      vcycle<float>(op, level, adjoint, nrhs, op->w32[level].VB, (float2*)z);
    }
    CK(cudaStreamSynchronize(op->st));
  });
}

helm_status helm_transfer(helm_op* op, int32_t level, int32_t prolong, int32_t nrhs, const void* in, void* out,
                          void* stream) {
  return wrap([&] {
    level_ptr_check(op, level);
    REQ(level < op->L - 1, HELM_ERR_ARG, "no coarser level");
    REQ(in && out && in != out, HELM_ERR_ARG, "bad vectors");
    REQ(nrhs >= 1 && nrhs <= op->max_rhs, HELM_ERR_SHAPE, "nrhs must be in [1, max_rhs]");
    op->st = (cudaStream_t)stream;
    reset_acct(op, nrhs);
    set_active(op, nrhs);
    if (op->dtype == HELM_C128) {
      if (prolong) launch_prolong_add<double>(op, level, nrhs, (const double2*)in, (double2*)out);
      else launch_restrict<double>(op, level, nrhs, (const double2*)in, (double2*)out);
    } else {
      if (prolong) launch_prolong_add<float>(op, level, nrhs, (const float2*)in, (float2*)out);
      else launch_restrict<float>(op, level, nrhs, (const float2*)in, (float2*)out);
    }
  });
}

helm_status helm_probe_kernel(helm_op* op, int32_t level, int32_t kind, int32_t nv, int32_t nrhs, int32_t reps,
                              double* ms_per_launch, void* stream) {
  return wrap([&] {
    level_ptr_check(op, level);
    REQ(!op->apply_only, HELM_ERR_STATE, "operator-only op");
    REQ(nrhs >= 1 && nrhs <= op->max_rhs && reps >= 1 && ms_per_launch, HELM_ERR_ARG, "bad probe arguments");
    op->st = (cudaStream_t)stream;
    reset_acct(op, nrhs);
    set_active(op, nrhs);
    *ms_per_launch = op->dtype == HELM_C128 ? probe_run<double>(op, level, kind, nv, nrhs, reps)
                                            : probe_run<float>(op, level, kind, nv, nrhs, reps);
  });
}

helm_status helm_profile(int32_t enable, int32_t stride) {
  return wrap([&] {
    REQ(stride >= 1, HELM_ERR_ARG, "stride must be >= 1");
    prof_drain();
    g_prof.on = enable != 0;
    g_prof.stride = stride;
    for (int c = 0; c < HELM_NCLASS; ++c)
      for (int l = 0; l < 5; ++l) {
        g_prof.launches[c][l] = g_prof.sampled[c][l] = 0;
        g_prof.ms[c][l] = g_prof.bytes[c][l] = 0.0;
      }
  });
}

helm_status helm_profile_read(int32_t level, int64_t* launches, int64_t* sampled, double* ms, double* bytes) {
  return wrap([&] {
    REQ(level >= -1 && level <= 4, HELM_ERR_ARG, "level must be in [-1, 4]");
    prof_drain();
    for (int c = 0; c < HELM_NCLASS; ++c) {
      long long la = 0, sa = 0;
      double m = 0, b = 0;
      for (int l = 0; l < 5; ++l)
        if (level < 0 || l == level) {
          la += g_prof.launches[c][l]; sa += g_prof.sampled[c][l]; m += g_prof.ms[c][l]; b += g_prof.bytes[c][l];
        }
      if (launches) launches[c] = la;
      if (sampled) sampled[c] = sa;
      if (ms) ms[c] = m;
      if (bytes) bytes[c] = b;
    }
  });
}

int64_t helm_launch_count(void) { return g_launches; }

double helm_workspace_vectors(const helm_op* op) { return op ? op->ws_vectors : 0.0; }

void helm_destroy(helm_op* op) {
  if (op == g_fwi_op) return;   // the cached FWI op is owned by the library
  delete op;
}

const char* helm_last_error(void) { return g_err.c_str(); }
const char* helm_version(void) { return "libhelm 0.1 (sm_100a)"; }

}  // extern "C"
