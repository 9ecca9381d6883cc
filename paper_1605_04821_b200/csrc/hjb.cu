// hjb.cu -- C-ABI of libhjb (include/hjb.h): handle management, coefficient upload, and the
// host orchestration of policy iteration / BiCGSTAB / geometric multigrid.  All arithmetic on
// grid data runs in the kernels of hjb_kernels.cuh; the host only sequences launches and reads a
// few scalars (Krylov convergence, policy-iteration stopping) through pinned memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "hjb.h"
#include "hjb_kernels.cuh"

using namespace hjb;

static thread_local std::string g_err;

static hjb_status fail(hjb_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define CK(call)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      return fail(e_ == cudaErrorMemoryAllocation ? HJB_ERR_OOM : HJB_ERR_CUDA,                   \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                            \
  } while (0)
#define CKL()                                                                                     \
  do {                                                                                            \
    cudaError_t e_ = cudaGetLastError();                                                          \
    if (e_ != cudaSuccess) return fail(HJB_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(e_)); \
  } while (0)
#define TRY(x)                     \
  do {                             \
    hjb_status s_ = (x);           \
    if (s_ != HJB_OK) return s_;   \
  } while (0)

static constexpr int kMaxBlocks = 148 * 16;  // partial-sum slots: 16 resident 128-thread CTAs per SM

struct Level {
  LevelDev L{};
  int64_t elems = 0;          // local elements of a grid array on this level
  double* tmp = nullptr;      // smoother ping-pong
  double* res = nullptr;      // residual before restriction
  double* x = nullptr;        // coarse levels: correction
  double* b = nullptr;        // coarse levels: restricted rhs
  uint8_t* pol = nullptr;     // coarse levels: injected policy
  double* fields = nullptr;   // coarse levels: injected field planes
  CoefDev C{};
  double* Ainv = nullptr;     // coarsest level dense inverse
};

struct hjb_grid {
  hjb_grid_desc desc{};
  int D = 2, P = 1, K = 1, Q = 0;
  int64_t n = 0;
  double lo = 0, hi = 1, h = 0, k = 0;
  cudaStream_t st = nullptr;
  LevelDev L0{};
  int64_t N = 0, n_interior = 0, n_boundary = 0;
  // coefficients
  double* d_tab = nullptr;  // sigma_dir | b_dir | c_ctrl | f_basis | f_ctrl
  CoefDev C0{};
  bool have_coeffs = false;
  // Krylov workspace
  double *r = nullptr, *rhat = nullptr, *p = nullptr, *v = nullptr, *s = nullptr, *t = nullptr;
  double *phat = nullptr, *shat = nullptr, *F = nullptr;
  double* partial = nullptr;
  double* red = nullptr;
  KScal* S = nullptr;
  KScal* hS = nullptr;     // pinned mirror
  double* hred = nullptr;  // pinned mirror of red
  uint8_t* pol_int = nullptr;
  // staging for host pointers
  double *stage_prev = nullptr, *stage_U = nullptr, *stage_psi = nullptr;
  uint8_t* stage_pol = nullptr;
  // multigrid
  std::vector<Level> levels;
  hjb_mg_params mgp{};
  bool mg_ready = false;
  const uint8_t* mg_pol0 = nullptr;
  double mg_dt = 0.0;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  // instrumentation (hjb_profile_*)
  static constexpr int kSlots = 256;
  bool prof_timing = false;
  cudaEvent_t pev[2 * kSlots] = {};
  int pcls[kSlots] = {};
  int npend = 0;
  hjb_profile prof{};
  int nplanes0 = 0;  // per-node coefficient planes read by the operator (sigma/b/c fields)
  int sms = 148;
  int nblk_last = 1;  // CTAs of the last dims() launch (partials to reduce)
};

// ---------------------------------------------------------------------------- instrumentation
static void prof_drain(hjb_grid* g) {
  if (g->npend == 0) return;
  cudaEventSynchronize(g->pev[2 * g->npend - 1]);
  for (int i = 0; i < g->npend; ++i) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, g->pev[2 * i], g->pev[2 * i + 1]) == cudaSuccess) g->prof.ms[g->pcls[i]] += ms;
  }
  g->npend = 0;
}
static void prof_pre(hjb_grid* g, int) {
  if (!g->prof_timing) return;
  if (g->npend == hjb_grid::kSlots) prof_drain(g);
  cudaEventRecord(g->pev[2 * g->npend], g->st);
}
static void prof_post(hjb_grid* g, int cls, double nodes, double bytes, double flops) {
  g->prof.launches[cls] += 1;
  g->prof.total_launches += 1;
  g->prof.nodes[cls] += nodes;
  g->prof.bytes[cls] += bytes;
  g->prof.flops[cls] += flops;
  if (!g->prof_timing) return;
  cudaEventRecord(g->pev[2 * g->npend + 1], g->st);
  g->pcls[g->npend] = cls;
  g->npend += 1;
}
// LAUNCH(class, nodes, algorithmic bytes, algorithmic flops, kernel<<<...>>>(...))
#define LAUNCH(CLS, NODES, BYTES, FLOPS, ...)                              \
  do {                                                                     \
    prof_pre(g, CLS);                                                      \
    __VA_ARGS__;                                                           \
    prof_post(g, CLS, (double)(NODES), (double)(BYTES), (double)(FLOPS));  \
  } while (0)

// ---------------------------------------------------------------------------- small helpers
// 2D launch over the owned interior of level L: x covers an x1 line, y strides over lines.  All
// CTAs are made co-resident (occupancy x SMs) so the lines in flight form one band that moves
// through the grid and the +-reach rows it gathers from stay in L2.
static int occupancy_of(const void* fn) {
  static std::map<const void*, int> cache;
  auto it = cache.find(fn);
  if (it != cache.end()) return it->second;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kTX, 0) != cudaSuccess || occ < 1) occ = 1;
  cache[fn] = occ;
  return occ;
}
static dim3 dims(hjb_grid* g, const LevelDev& L, const void* fn) {
  const int gx = std::max(1, (L.nI + kTX - 1) / kTX);
  const int64_t cap = std::min<int64_t>((int64_t)occupancy_of(fn) * g->sms, kMaxBlocks);
  const int gy = (int)std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(L.nrows, 65535), cap / gx));
  g->nblk_last = gx * gy;
  return dim3(gx, gy);
}
static int nblocks1d(int64_t work) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, kMaxBlocks));
}

static bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

static hjb_status dalloc(void** p, size_t bytes) {
  CK(cudaMalloc(p, bytes));
  return HJB_OK;
}

static LevelDev make_level(int D, int64_t n, double lo, double hi, double k, double k2, int rank, int nranks) {
  LevelDev L{};
  L.n = (int)n;
  L.nI = (int)(n - 2);
  L.nrows = 1;
  for (int d = 0; d < D - 1; ++d) L.nrows *= (int)(n - 2);
  L.row_elems = 1;
  for (int d = 0; d < D - 1; ++d) L.row_elems *= n;
  // single rank: owned interior rows 1..n-2 of the slowest axis, local array = whole grid
  (void)rank;
  (void)nranks;
  L.local_row0 = 0;
  L.local_rows = n;
  L.row_first = 1;
  int64_t own = 1;
  for (int d = 0; d < D; ++d) own *= (n - 2);
  L.n_own = own;
  L.h = (hi - lo) / (double)(n - 1);
  L.nm1 = (double)(n - 1);
  L.kh = k / L.h;
  L.k2h = k2 / L.h;
  L.inv_2k2 = 1.0 / (2.0 * k2);
  L.inv_k2 = 1.0 / k2;
  return L;
}

static double host_finalize(hjb_grid* g, int nblk, unsigned maxmask, int which, hjb_status* err,
                            double* second = nullptr) {
  LAUNCH(HJB_KC_REDUCE, nblk, 16.0 * nblk, 2.0 * nblk,
         k_finalize<<<1, 1024, 0, g->st>>>(g->partial, nblk, g->red, maxmask, g->S, which));
  cudaMemcpyAsync(g->hred, g->red, 2 * sizeof(double), cudaMemcpyDeviceToHost, g->st);
  cudaError_t e = cudaStreamSynchronize(g->st);
  if (e != cudaSuccess) {
    *err = fail(HJB_ERR_CUDA, std::string("sync: ") + cudaGetErrorString(e));
    return NAN;
  }
  *err = HJB_OK;
  if (second) *second = g->hred[1];
  return g->hred[0];
}

// ---------------------------------------------------------------------------- dimension dispatch
template <int D>
static void launch_operator(hjb_grid* g, const LevelDev& L, const CoefDev& C, int mode, int ndot, double dt,
                            double omega, const uint8_t* pol, const double* x, const double* b, double* y,
                            const double* u) {
  cudaStream_t st = g->st;
  const int cls = mode == OP_APPLY ? HJB_KC_APPLY : (mode == OP_RESID ? HJB_KC_RESID : HJB_KC_SMOOTH);
  const double nodes = (double)L.n_own;
  const double bpn = 1.0 + 8.0 + (mode != OP_JACOBI0 ? 8.0 : 0.0) + (mode != OP_APPLY ? 8.0 : 0.0) +
                     (ndot >= 1 ? 8.0 : 0.0) + 8.0 * g->nplanes0;
  const double fpn = (2.0 * g->P + 1.0) * (1 << D) * 2.0 + 4.0 + 2.0 * ndot;
#define OPL(M, ND) LAUNCH(cls, nodes, nodes * bpn, nodes * fpn, \
    k_operator<D, M, ND><<<dims(g, L, (const void*)k_operator<D, M, ND>), kTX, 0, st>>>(L, C, dt, omega, pol, x, b, y, u, g->partial))
  if (mode == OP_APPLY) {
    if (ndot == 0) OPL(OP_APPLY, 0);
    else if (ndot == 1) OPL(OP_APPLY, 1);
    else OPL(OP_APPLY, 2);
  } else if (mode == OP_RESID) {
    if (ndot == 0) OPL(OP_RESID, 0);
    else OPL(OP_RESID, 2);
  } else if (mode == OP_JACOBI) {
    OPL(OP_JACOBI, 0);
  } else {
    OPL(OP_JACOBI0, 0);
  }
#undef OPL
}

static void op(hjb_grid* g, const LevelDev& L, const CoefDev& C, int mode, int ndot, double dt, double omega,
               const uint8_t* pol, const double* x, const double* b, double* y, const double* u) {
  if (g->D == 2) launch_operator<2>(g, L, C, mode, ndot, dt, omega, pol, x, b, y, u);
  else launch_operator<3>(g, L, C, mode, ndot, dt, omega, pol, x, b, y, u);
}

// ---------------------------------------------------------------------------- API: misc
extern "C" const char* hjb_last_error(void) { return g_err.c_str(); }
extern "C" int32_t hjb_version(void) { return HJB_VERSION; }

extern "C" void hjb_mg_params_default(int32_t dim, hjb_mg_params* o) {
  if (!o) return;
  o->nu_pre = 2;
  o->nu_post = 2;
  o->omega = 1.0;
  o->coarse_max_n = (dim == 3) ? 5 : 9;
  o->coarse_k_mode = 0;
  o->max_levels = 32;
}

extern "C" void hjb_solve_params_default(int32_t dim, hjb_solve_params* o) {
  if (!o) return;
  o->krylov_rtol = 1e-12;
  o->krylov_maxit = 2000;
  o->use_mg = 1;
  o->tol_pi = 1e-10;
  o->max_pi = 50;
  hjb_mg_params_default(dim, &o->mg);
  o->pi_forcing = 0.0;
}

// ---------------------------------------------------------------------------- API: grid
static void free_levels(hjb_grid* g) {
  for (size_t i = 0; i < g->levels.size(); ++i) {
    Level& l = g->levels[i];
    cudaFree(l.tmp);
    cudaFree(l.res);
    if (i > 0) {
      cudaFree(l.x);
      cudaFree(l.b);
      cudaFree(l.pol);
      cudaFree(l.fields);
    }
    cudaFree(l.Ainv);
  }
  g->levels.clear();
  g->mg_ready = false;
}

extern "C" hjb_status hjb_grid_destroy(hjb_grid_t g) {
  if (!g) return fail(HJB_ERR_INVALID_ARG, "null handle");
  cudaSetDevice(g->desc.device);
  if (g->st) cudaStreamSynchronize(g->st);
  free_levels(g);
  double* bufs[] = {g->d_tab, g->r, g->rhat, g->p, g->v, g->s, g->t, g->phat, g->shat, g->F,
                    g->partial, g->red, g->stage_prev, g->stage_U, g->stage_psi};
  for (double* b : bufs) cudaFree(b);
  cudaFree(g->S);
  cudaFree(g->pol_int);
  cudaFree(g->stage_pol);
  cudaFreeHost(g->hS);
  cudaFreeHost(g->hred);
  for (auto& e : g->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : g->pev)
    if (e) cudaEventDestroy(e);
  delete g;
  return HJB_OK;
}

extern "C" hjb_status hjb_grid_create(const hjb_grid_desc* d, hjb_grid_t* out) {
  if (!d || !out) return fail(HJB_ERR_INVALID_ARG, "null desc/out");
  *out = nullptr;
  if (d->dim != 2 && d->dim != 3) return fail(HJB_ERR_INVALID_ARG, "dim must be 2 or 3");
  if (d->P < 1 || d->P > d->dim) return fail(HJB_ERR_INVALID_ARG, "P must be in [1, dim]");
  if (d->K < 1 || d->K > HJB_MAX_K) return fail(HJB_ERR_INVALID_ARG, "K must be in [1,255]");
  if (d->Q < 0 || d->Q > HJB_MAX_Q) return fail(HJB_ERR_INVALID_ARG, "Q must be in [0,16]");
  if (d->n < 3) return fail(HJB_ERR_INVALID_ARG, "n must be >= 3");
  if (!(d->hi > d->lo)) return fail(HJB_ERR_INVALID_ARG, "hi must be > lo");
  if (d->nranks != 1 || d->rank != 0)
    return fail(HJB_ERR_UNSUPPORTED, "nranks > 1: slab decomposition is not enabled in this build");
  int64_t tot = 1;
  for (int i = 0; i < d->dim; ++i) tot *= d->n;
  // local arrays are indexed with 32-bit offsets; one x1 line must fit the partial-sum slots
  if (tot >= (1LL << 31) || (d->n - 2) > (int64_t)kTX * kMaxBlocks)
    return fail(HJB_ERR_INVALID_ARG, "grid too large for one rank (local arrays must hold < 2^31 nodes)");
  CK(cudaSetDevice(d->device));
  hjb_grid* g = new hjb_grid();
  g->desc = *d;
  g->D = d->dim;
  g->P = d->P;
  g->K = d->K;
  g->Q = d->Q;
  g->n = d->n;
  g->lo = d->lo;
  g->hi = d->hi;
  g->h = (d->hi - d->lo) / (double)(d->n - 1);
  g->k = std::sqrt(g->h);  // k = sqrt(dx)
  g->st = (cudaStream_t)d->stream;
  cudaDeviceGetAttribute(&g->sms, cudaDevAttrMultiProcessorCount, d->device);
  if (g->sms < 1) g->sms = 148;
  g->L0 = make_level(g->D, g->n, g->lo, g->hi, g->k, g->h, 0, 1);
  g->N = g->L0.local_rows * g->L0.row_elems;
  g->n_interior = g->L0.n_own;
  g->n_boundary = tot - g->n_interior;
  const size_t vb = (size_t)g->N * sizeof(double);
  double** vecs[] = {&g->r, &g->rhat, &g->p, &g->v, &g->s, &g->t, &g->phat, &g->shat, &g->F};
  hjb_status s = HJB_OK;
  for (double** pv : vecs) {
    if ((s = dalloc((void**)pv, vb)) != HJB_OK) {
      hjb_grid_destroy(g);
      return s;
    }
    cudaMemsetAsync(*pv, 0, vb, g->st);
  }
  if ((s = dalloc((void**)&g->partial, (size_t)kMaxBlocks * 2 * sizeof(double))) != HJB_OK ||
      (s = dalloc((void**)&g->red, 4 * sizeof(double))) != HJB_OK ||
      (s = dalloc((void**)&g->S, sizeof(KScal))) != HJB_OK ||
      (s = dalloc((void**)&g->pol_int, (size_t)g->N)) != HJB_OK) {
    hjb_grid_destroy(g);
    return s;
  }
  cudaMemsetAsync(g->pol_int, 0, (size_t)g->N, g->st);
  if (cudaMallocHost((void**)&g->hS, sizeof(KScal)) != cudaSuccess ||
      cudaMallocHost((void**)&g->hred, 4 * sizeof(double)) != cudaSuccess) {
    hjb_grid_destroy(g);
    return fail(HJB_ERR_OOM, "pinned alloc");
  }
  for (auto& e : g->ev) cudaEventCreate(&e);
  for (auto& e : g->pev) cudaEventCreate(&e);
  cudaError_t e = cudaStreamSynchronize(g->st);
  if (e != cudaSuccess) {
    hjb_grid_destroy(g);
    return fail(HJB_ERR_CUDA, cudaGetErrorString(e));
  }
  hjb_mg_params_default(g->D, &g->mgp);
  *out = g;
  return HJB_OK;
}

// ---------------------------------------------------------------------------- API: partition
static int64_t ipow(int64_t b, int e) {
  int64_t r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

extern "C" hjb_status hjb_partition(int32_t dim, int64_t n, int32_t nranks, int32_t rank, int64_t halo,
                                    hjb_layout* o) {
  if (!o) return fail(HJB_ERR_INVALID_ARG, "null out");
  if (dim != 2 && dim != 3) return fail(HJB_ERR_INVALID_ARG, "dim must be 2 or 3");
  if (n < 3) return fail(HJB_ERR_INVALID_ARG, "n must be >= 3");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(HJB_ERR_INVALID_ARG, "bad rank/nranks");
  const int64_t nI = n - 2;
  if (nranks == 1) halo = 0;
  else if (halo < 1) return fail(HJB_ERR_INVALID_ARG, "halo must be >= 1 when nranks > 1");
  const int64_t r0 = 1 + (rank * nI) / nranks, r1 = 1 + ((rank + 1) * nI) / nranks;
  for (int q = 0; q < nranks; ++q) {
    const int64_t own = (((int64_t)q + 1) * nI) / nranks - ((int64_t)q * nI) / nranks;
    if (own < std::max<int64_t>(1, halo))
      return fail(HJB_ERR_INVALID_ARG, "too many ranks: every rank must own >= halo interior rows");
  }
  const int64_t lr0 = nranks == 1 ? 0 : std::max<int64_t>(0, r0 - halo);
  const int64_t lr1 = nranks == 1 ? n : std::min<int64_t>(n, r1 + halo);
  o->n = n;
  o->row_elems = ipow(n, dim - 1);
  o->row0 = r0;
  o->row1 = r1;
  o->halo = halo;
  o->local_row0 = lr0;
  o->local_rows = lr1 - lr0;
  o->local_elems = o->local_rows * o->row_elems;
  o->n_interior = (r1 - r0) * ipow(nI, dim - 1);
  o->n_boundary = ipow(n, dim) - ipow(nI, dim);
  o->n_levels = 0;
  o->h = 0.0;
  o->k = 0.0;
  return HJB_OK;
}

extern "C" hjb_status hjb_halo_plan(int32_t dim, int64_t n, int32_t nranks, int32_t rank, int64_t halo,
                                    hjb_halo_msg out[2], int32_t* count) {
  if (!out || !count) return fail(HJB_ERR_INVALID_ARG, "null out");
  hjb_layout me;
  TRY(hjb_partition(dim, n, nranks, rank, halo, &me));
  *count = 0;
  if (nranks == 1) return HJB_OK;
  if (rank > 0) {  // lower neighbour: send my first `halo` owned rows, receive its last ones
    out[*count] = hjb_halo_msg{rank - 1, me.row0, me.row0 - halo, halo};
    ++*count;
  }
  if (rank + 1 < nranks) {  // upper neighbour: send my last `halo` owned rows, receive its first ones
    out[*count] = hjb_halo_msg{rank + 1, me.row1 - halo, me.row1, halo};
    ++*count;
  }
  return HJB_OK;
}

extern "C" hjb_status hjb_grid_query(hjb_grid_t g, hjb_layout* o) {
  if (!g || !o) return fail(HJB_ERR_INVALID_ARG, "null handle/out");
  o->n = g->n;
  o->row_elems = g->L0.row_elems;
  o->row0 = 0;
  o->row1 = g->n;
  o->halo = 0;
  o->local_row0 = g->L0.local_row0;
  o->local_rows = g->L0.local_rows;
  o->local_elems = g->N;
  o->n_interior = g->n_interior;
  o->n_boundary = g->n_boundary;
  o->n_levels = (int32_t)g->levels.size();
  o->h = g->h;
  o->k = g->k;
  return HJB_OK;
}

// ---------------------------------------------------------------------------- API: coefficients
static hjb_status upload_tables(hjb_grid* g, const double* sigma_dir, const double* b_dir, const double* c_ctrl,
                                const double* f_basis, const double* f_ctrl) {
  const int D = g->D, K = g->K, P = g->P, Q = g->Q;
  const size_t nsd = (size_t)K * P * D, nbd = (size_t)K * D, nc = K, nfb = (size_t)K * Q, nfc = K;
  const size_t tot = nsd + nbd + nc + nfb + nfc;
  std::vector<double> h(tot, 0.0);
  if (sigma_dir) std::memcpy(h.data(), sigma_dir, nsd * sizeof(double));
  if (b_dir) std::memcpy(h.data() + nsd, b_dir, nbd * sizeof(double));
  if (c_ctrl) std::memcpy(h.data() + nsd + nbd, c_ctrl, nc * sizeof(double));
  if (f_basis && Q > 0) std::memcpy(h.data() + nsd + nbd + nc, f_basis, nfb * sizeof(double));
  if (f_ctrl) std::memcpy(h.data() + nsd + nbd + nc + nfb, f_ctrl, nfc * sizeof(double));
  if (!g->d_tab) TRY(dalloc((void**)&g->d_tab, tot * sizeof(double)));
  CK(cudaMemcpyAsync(g->d_tab, h.data(), tot * sizeof(double), cudaMemcpyHostToDevice, g->st));
  CK(cudaStreamSynchronize(g->st));  // h is a stack temporary
  g->C0.sigma_dir = g->d_tab;
  g->C0.b_dir = g->d_tab + nsd;
  g->C0.c_ctrl = g->d_tab + nsd + nbd;
  g->C0.f_basis = g->d_tab + nsd + nbd + nc;
  g->C0.f_ctrl = g->d_tab + nsd + nbd + nc + nfb;
  return HJB_OK;
}

extern "C" hjb_status hjb_set_coeffs(hjb_grid_t g, const hjb_coeffs* c) {
  if (!g || !c) return fail(HJB_ERR_INVALID_ARG, "null handle/coeffs");
  if (!c->sigma_dir || !c->b_dir || !c->c_ctrl) return fail(HJB_ERR_INVALID_ARG, "sigma_dir/b_dir/c_ctrl required");
  if (g->Q > 0 && (!c->f_basis || !c->f_feat)) return fail(HJB_ERR_INVALID_ARG, "Q > 0 needs f_basis and f_feat");
  const double* fields[] = {c->sigma_scale, c->sigma_node, c->b_scale, c->b_node, c->c_node, c->f_feat};
  for (const double* f : fields)
    if (f && !is_device_ptr(f)) return fail(HJB_ERR_INVALID_ARG, "coefficient fields must be device pointers");
  CK(cudaSetDevice(g->desc.device));
  TRY(upload_tables(g, c->sigma_dir, c->b_dir, c->c_ctrl, c->f_basis, c->f_ctrl));
  g->C0.sigma_scale = c->sigma_scale;
  g->C0.sigma_node = c->sigma_node;
  g->C0.b_scale = c->b_scale;
  g->C0.b_node = c->b_node;
  g->C0.c_node = c->c_node;
  g->C0.f_feat = c->f_feat;
  g->C0.ld = g->N;
  g->C0.K = g->K;
  g->C0.P = g->P;
  g->C0.Q = g->Q;
  g->nplanes0 = (c->sigma_scale ? g->P : 0) + (c->sigma_node ? g->P * g->D : 0) + (c->b_scale ? 1 : 0) +
                (c->b_node ? g->D : 0) + (c->c_node ? 1 : 0);
  g->have_coeffs = true;
  g->mg_ready = false;
  return HJB_OK;
}

extern "C" hjb_status hjb_set_source(hjb_grid_t g, const double* f_basis, const double* f_ctrl) {
  if (!g) return fail(HJB_ERR_INVALID_ARG, "null handle");
  if (!g->have_coeffs) return fail(HJB_ERR_STATE, "hjb_set_source before hjb_set_coeffs");
  const int K = g->K, Q = g->Q;
  std::vector<double> h((size_t)K * Q + K, 0.0);
  if (f_basis && Q > 0) std::memcpy(h.data(), f_basis, (size_t)K * Q * sizeof(double));
  if (f_ctrl) std::memcpy(h.data() + (size_t)K * Q, f_ctrl, (size_t)K * sizeof(double));
  CK(cudaMemcpyAsync((void*)g->C0.f_basis, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, g->st));
  CK(cudaStreamSynchronize(g->st));
  return HJB_OK;
}

// ---------------------------------------------------------------------------- policy improvement
static hjb_status policy_update_dev(hjb_grid* g, double dt, const double* U, const double* Uprev, uint8_t* pol,
                                    double* F, hjb_pi_stats* out) {
  const double nodes = (double)g->L0.n_own;
  const double bpn = 8.0 + 8.0 + 1.0 + 1.0 + 8.0 + 8.0 * g->Q + 8.0 * g->nplanes0;
  const double fpn = g->K * ((2.0 * g->P + 1.0) * (1 << g->D) * 2.0 + 2.0 * g->Q + 4.0);
  if (g->D == 2) LAUNCH(HJB_KC_SEARCH, nodes, nodes * bpn, nodes * fpn,
                        k_search<2><<<dims(g, g->L0, (const void*)k_search<2>), kTX, 0, g->st>>>(g->L0, g->C0, dt, U, Uprev, pol, F, g->partial));
  else LAUNCH(HJB_KC_SEARCH, nodes, nodes * bpn, nodes * fpn,
              k_search<3><<<dims(g, g->L0, (const void*)k_search<3>), kTX, 0, g->st>>>(g->L0, g->C0, dt, U, Uprev, pol, F, g->partial));
  CKL();
  hjb_status err;
  double changed = 0.0;
  const double R = host_finalize(g, g->nblk_last, 0x1u, SC_NONE, &err, &changed);
  if (err != HJB_OK) return err;
  if (out) {
    out->R_max = R;
    out->changed = (int64_t)changed;
  }
  if (!std::isfinite(R)) return fail(HJB_ERR_NONFINITE, "non-finite nonlinear residual");
  return HJB_OK;
}

static hjb_status check_dt(hjb_grid* g, double dt) {
  if (!(dt > 0.0) || !std::isfinite(dt)) return fail(HJB_ERR_INVALID_ARG, "dt must be > 0");
  if (!g->have_coeffs) return fail(HJB_ERR_STATE, "call hjb_set_coeffs first");
  return HJB_OK;
}

extern "C" hjb_status hjb_policy_update(hjb_grid_t g, double dt, const double* U, const double* U_prev,
                                        uint8_t* policy, double* F, hjb_pi_stats* out) {
  if (!g || !U || !U_prev || !policy || !F) return fail(HJB_ERR_INVALID_ARG, "null argument");
  TRY(check_dt(g, dt));
  CK(cudaSetDevice(g->desc.device));
  return policy_update_dev(g, dt, U, U_prev, policy, F, out);
}

// ---------------------------------------------------------------------------- apply
extern "C" hjb_status hjb_apply(hjb_grid_t g, double dt, const uint8_t* policy, const double* x, double* y) {
  if (!g || !policy || !x || !y) return fail(HJB_ERR_INVALID_ARG, "null argument");
  TRY(check_dt(g, dt));
  CK(cudaSetDevice(g->desc.device));
  if (x != y) CK(cudaMemcpyAsync(y, x, (size_t)g->N * sizeof(double), cudaMemcpyDeviceToDevice, g->st));
  else return fail(HJB_ERR_INVALID_ARG, "x and y must not alias");
  op(g, g->L0, g->C0, OP_APPLY, 0, dt, 0.0, policy, x, nullptr, y, nullptr);
  CKL();
  return HJB_OK;
}

// ---------------------------------------------------------------------------- multigrid
static hjb_status build_levels(hjb_grid* g, const hjb_mg_params* mp) {
  free_levels(g);
  const int D = g->D;
  int64_t n = g->n;
  g->levels.push_back(Level());
  g->levels[0].L = g->L0;
  g->levels[0].elems = g->N;
  g->levels[0].C = g->C0;
  auto interior_count = [&](int64_t nn) {
    int64_t c = 1;
    for (int d = 0; d < D; ++d) c *= (nn - 2);
    return c;
  };
  while ((int)g->levels.size() < mp->max_levels) {
    const bool small = interior_count(n) <= 160 && n <= std::max<int64_t>(mp->coarse_max_n, 3);
    if (small) break;
    if ((n - 1) % 2 != 0 || n < 5) {
      if (interior_count(n) > 160) {
        free_levels(g);
        return fail(HJB_ERR_UNSUPPORTED, "multigrid needs n = 2^l + 1 (coarsest interior <= 160 unknowns)");
      }
      break;
    }
    const int64_t nc = (n - 1) / 2 + 1;
    Level l;
    const double hc = (g->hi - g->lo) / (double)(nc - 1);
    const double kc = (mp->coarse_k_mode == 1) ? std::sqrt(hc) : g->k;
    const double k2c = (mp->coarse_k_mode == 1) ? hc : g->h;
    l.L = make_level(D, nc, g->lo, g->hi, kc, k2c, 0, 1);
    l.elems = l.L.local_rows * l.L.row_elems;
    g->levels.push_back(l);
    n = nc;
  }
  if (interior_count(g->levels.back().L.n) > 160) {
    free_levels(g);
    return fail(HJB_ERR_UNSUPPORTED, "coarsest level too large for the dense solve (needs n = 2^l + 1)");
  }
  // field planes present on the fine level (f_feat is not needed below level 0)
  int nplanes = 0;
  if (g->C0.sigma_scale) nplanes += g->P;
  if (g->C0.sigma_node) nplanes += g->P * D;
  if (g->C0.b_scale) nplanes += 1;
  if (g->C0.b_node) nplanes += D;
  if (g->C0.c_node) nplanes += 1;
  for (size_t i = 0; i < g->levels.size(); ++i) {
    Level& l = g->levels[i];
    const size_t vb = (size_t)l.elems * sizeof(double);
    TRY(dalloc((void**)&l.tmp, vb));
    TRY(dalloc((void**)&l.res, vb));
    CK(cudaMemsetAsync(l.tmp, 0, vb, g->st));
    CK(cudaMemsetAsync(l.res, 0, vb, g->st));
    if (i > 0) {
      TRY(dalloc((void**)&l.x, vb));
      TRY(dalloc((void**)&l.b, vb));
      TRY(dalloc((void**)&l.pol, (size_t)l.elems));
      CK(cudaMemsetAsync(l.x, 0, vb, g->st));
      CK(cudaMemsetAsync(l.b, 0, vb, g->st));
      CK(cudaMemsetAsync(l.pol, 0, (size_t)l.elems, g->st));
      if (nplanes > 0) TRY(dalloc((void**)&l.fields, (size_t)nplanes * vb));
      CoefDev C = g->C0;
      C.ld = l.elems;
      C.f_feat = nullptr;
      double* q = l.fields;
      if (g->C0.sigma_scale) { C.sigma_scale = q; q += (size_t)g->P * l.elems; }
      if (g->C0.sigma_node) { C.sigma_node = q; q += (size_t)g->P * D * l.elems; }
      if (g->C0.b_scale) { C.b_scale = q; q += l.elems; }
      if (g->C0.b_node) { C.b_node = q; q += (size_t)D * l.elems; }
      if (g->C0.c_node) { C.c_node = q; q += l.elems; }
      l.C = C;
    }
  }
  Level& lc = g->levels.back();
  TRY(dalloc((void**)&lc.Ainv, (size_t)lc.L.n_own * lc.L.n_own * sizeof(double)));
  g->mgp = *mp;
  return HJB_OK;
}

template <int D>
static hjb_status inject_all(hjb_grid* g) {
  for (size_t i = 1; i < g->levels.size(); ++i) {
    Level& lf = g->levels[i - 1];
    Level& lc = g->levels[i];
    const uint8_t* pf = (i == 1) ? g->mg_pol0 : lf.pol;
    const int nb = nblocks1d(lc.elems);
    LAUNCH(HJB_KC_TRANSFER, lc.elems, 2.0 * lc.elems, 0, k_inject_u8<D><<<nb, 256, 0, g->st>>>(lf.L, lc.L, pf, lc.pol));
    struct FP { const double* f; double* c; int np; };
    const FP fps[] = {{lf.C.sigma_scale, (double*)lc.C.sigma_scale, g->P},
                      {lf.C.sigma_node, (double*)lc.C.sigma_node, g->P * D},
                      {lf.C.b_scale, (double*)lc.C.b_scale, 1},
                      {lf.C.b_node, (double*)lc.C.b_node, D},
                      {lf.C.c_node, (double*)lc.C.c_node, 1}};
    for (const FP& f : fps)
      if (f.f)
        LAUNCH(HJB_KC_TRANSFER, lc.elems, 16.0 * f.np * lc.elems, 0,
               k_inject_f64<D><<<nb, 256, 0, g->st>>>(lf.L, lc.L, f.f, lf.C.ld, f.c, lc.C.ld, f.np));
    CKL();
  }
  Level& lc = g->levels.back();
  const int64_t Nc = lc.L.n_own;
  const uint8_t* pc = (g->levels.size() == 1) ? g->mg_pol0 : lc.pol;
  CK(cudaMemsetAsync(lc.Ainv, 0, (size_t)Nc * Nc * sizeof(double), g->st));
  LAUNCH(HJB_KC_COARSE, Nc, 8.0 * Nc * Nc, 0,
         k_coarse_assemble<D><<<(int)((Nc + 127) / 128), 128, 0, g->st>>>(lc.L, lc.C, g->mg_dt, pc, lc.Ainv));
  CKL();
  const size_t smem = (size_t)Nc * Nc * sizeof(double);
  if (smem > 48 * 1024) CK(cudaFuncSetAttribute(k_coarse_invert, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  LAUNCH(HJB_KC_COARSE, Nc, 16.0 * Nc * Nc, 2.0 * Nc * Nc * Nc, k_coarse_invert<<<1, 1024, smem, g->st>>>(lc.Ainv, (int)Nc));
  CKL();
  return HJB_OK;
}

extern "C" hjb_status hjb_mg_setup(hjb_grid_t g, double dt, const uint8_t* policy, const hjb_mg_params* mp) {
  if (!g || !policy) return fail(HJB_ERR_INVALID_ARG, "null argument");
  TRY(check_dt(g, dt));
  CK(cudaSetDevice(g->desc.device));
  hjb_mg_params def;
  hjb_mg_params_default(g->D, &def);
  const hjb_mg_params* p = mp ? mp : &def;
  if (p->nu_pre < 1 || p->nu_post < 0 || !(p->omega > 0.0) || p->omega > 1.0 || p->max_levels < 1)
    return fail(HJB_ERR_INVALID_ARG, "bad multigrid parameters");
  const bool rebuild = g->levels.empty() || std::memcmp(&g->mgp, p, sizeof(hjb_mg_params)) != 0 ||
                       g->levels[0].C.ld != g->C0.ld;
  if (rebuild) TRY(build_levels(g, p));
  g->levels[0].C = g->C0;
  // refresh field pointers of level 0 (set_coeffs may have changed them)
  g->mg_pol0 = policy;
  g->mg_dt = dt;
  if (g->D == 2) TRY(inject_all<2>(g));
  else TRY(inject_all<3>(g));
  g->mg_ready = true;
  return HJB_OK;
}

// V(nu_pre, nu_post) from x = 0 on level l: out = M_l^{-1} b
template <int D>
static hjb_status vcycle(hjb_grid* g, size_t l, const double* b, double* out) {
  Level& lv = g->levels[l];
  const uint8_t* pol = (l == 0) ? g->mg_pol0 : lv.pol;
  const LevelDev& L = lv.L;
  cudaStream_t st = g->st;
  if (l + 1 == g->levels.size()) {
    const int Nc = (int)L.n_own;
    LAUNCH(HJB_KC_COARSE, Nc, 8.0 * Nc * Nc + 16.0 * Nc, 2.0 * Nc * Nc,
           k_coarse_solve<D><<<1, 256, Nc * sizeof(double), st>>>(L, lv.Ainv, b, out));
    CKL();
    return HJB_OK;
  }
  const double dt = g->mg_dt, om = g->mgp.omega;
  const int npre = g->mgp.nu_pre, npost = g->mgp.nu_post;
  double* bufs[2] = {out, lv.tmp};
  int cur = ((npre - 1 + npost) % 2 == 0) ? 0 : 1;  // so the last sweep lands in `out`
  launch_operator<D>(g, L, lv.C, OP_JACOBI0, 0, dt, om, pol, nullptr, b, bufs[cur], nullptr);
  for (int k = 1; k < npre; ++k) {
    launch_operator<D>(g, L, lv.C, OP_JACOBI, 0, dt, om, pol, bufs[cur], b, bufs[1 - cur], nullptr);
    cur = 1 - cur;
  }
  launch_operator<D>(g, L, lv.C, OP_RESID, 0, dt, 0.0, pol, bufs[cur], b, lv.res, nullptr);
  Level& lc = g->levels[l + 1];
  LAUNCH(HJB_KC_TRANSFER, L.n_own, 8.0 * (L.n_own + lc.L.n_own), 18.0 * lc.L.n_own,
         k_restrict<D><<<dims(g, lc.L, (const void*)k_restrict<D>), kTX, 0, st>>>(L, lc.L, lv.res, lc.b));
  CKL();
  TRY(vcycle<D>(g, l + 1, lc.b, lc.x));
  LAUNCH(HJB_KC_TRANSFER, L.n_own, 16.0 * L.n_own + 8.0 * lc.L.n_own, 4.0 * L.n_own,
         k_prolong_add<D><<<dims(g, L, (const void*)k_prolong_add<D>), kTX, 0, st>>>(L, lc.L, lc.x, bufs[cur]));
  for (int k = 0; k < npost; ++k) {
    launch_operator<D>(g, L, lv.C, OP_JACOBI, 0, dt, om, pol, bufs[cur], b, bufs[1 - cur], nullptr);
    cur = 1 - cur;
  }
  CKL();
  if (bufs[cur] != out) return fail(HJB_ERR_STATE, "internal: V-cycle buffer parity");
  return HJB_OK;
}

static hjb_status precond(hjb_grid* g, bool use_mg, const double* b, double* x) {
  if (!use_mg) {
    const double nn = (double)g->L0.n_own;
    if (g->D == 2) LAUNCH(HJB_KC_VECTOR, nn, 16.0 * nn, 0, k_copy_interior<2><<<dims(g, g->L0, (const void*)k_copy_interior<2>), kTX, 0, g->st>>>(g->L0, b, x));
    else LAUNCH(HJB_KC_VECTOR, nn, 16.0 * nn, 0, k_copy_interior<3><<<dims(g, g->L0, (const void*)k_copy_interior<3>), kTX, 0, g->st>>>(g->L0, b, x));
    CKL();
    return HJB_OK;
  }
  return g->D == 2 ? vcycle<2>(g, 0, b, x) : vcycle<3>(g, 0, b, x);
}

extern "C" hjb_status hjb_mg_apply(hjb_grid_t g, const double* b, double* x) {
  if (!g || !b || !x) return fail(HJB_ERR_INVALID_ARG, "null argument");
  if (!g->mg_ready) return fail(HJB_ERR_STATE, "call hjb_mg_setup first");
  CK(cudaSetDevice(g->desc.device));
  return precond(g, true, b, x);
}

// ---------------------------------------------------------------------------- BiCGSTAB
template <int D>
static hjb_status norms_dev(hjb_grid* g, const double* v, double* n2, double* ninf) {
  LAUNCH(HJB_KC_VECTOR, g->L0.n_own, 8.0 * g->L0.n_own, 3.0 * g->L0.n_own,
         k_norms<D><<<dims(g, g->L0, (const void*)k_norms<D>), kTX, 0, g->st>>>(g->L0, v, g->partial));
  const int nb = g->nblk_last;
  CKL();
  hjb_status err;
  *n2 = std::sqrt(host_finalize(g, nb, 0x2u, SC_NONE, &err, ninf));
  return err;
}

template <int D>
// eta > 0: inexact policy evaluation, stop at ||r||_2 <= max(rtol ||F||_2, eta ||r_0||_2)
static hjb_status bicgstab(hjb_grid* g, double dt, const uint8_t* pol, const double* F, double* x,
                           const hjb_solve_params* sp, hjb_solve_stats* out, double eta = 0.0) {
  const LevelDev& L = g->L0;
  const CoefDev& C = g->C0;
  cudaStream_t st = g->st;
  const bool mg = sp->use_mg != 0;
  if (mg && (!g->mg_ready || g->mg_pol0 != pol || g->mg_dt != dt))
    return fail(HJB_ERR_STATE, "hjb_mg_setup must be called with the same policy and dt before solving");
  double bn2, bninf;
  TRY(norms_dev<D>(g, F, &bn2, &bninf));
  double tol = sp->krylov_rtol * bn2;
  int it = 0;
  hjb_status err = HJB_OK;
  double rr = 0.0;
  bool converged = false;
  for (int restart = 0; restart < 4 && !converged; ++restart) {
    // r = F - A x ; rhat = r ; p = r
    launch_operator<D>(g, L, C, OP_RESID, 0, dt, 0.0, pol, x, F, g->r, nullptr);
    LAUNCH(HJB_KC_VECTOR, L.n_own, 24.0 * L.n_own, 2.0 * L.n_own,
           k_bicg_init<D><<<dims(g, L, (const void*)k_bicg_init<D>), kTX, 0, st>>>(L, g->r, g->rhat, g->p, g->partial));
    CKL();
    rr = host_finalize(g, g->nblk_last, 0u, SC_INIT, &err);
    if (err != HJB_OK) return err;
    if (!std::isfinite(rr)) return fail(HJB_ERR_NONFINITE, "non-finite residual");
    if (restart == 0 && eta > 0.0) tol = std::max(tol, eta * std::sqrt(rr));
    if (std::sqrt(rr) <= tol) { converged = true; break; }
    bool restart_needed = false;
    int inner = 0;
    while (it < sp->krylov_maxit) {
      if (inner > 0)
        LAUNCH(HJB_KC_VECTOR, L.n_own, 32.0 * L.n_own, 4.0 * L.n_own,
               k_bicg_p<D><<<dims(g, L, (const void*)k_bicg_p<D>), kTX, 0, st>>>(L, g->S, g->r, g->p, g->v));
      TRY(precond(g, mg, g->p, g->phat));
      launch_operator<D>(g, L, C, OP_APPLY, 1, dt, 0.0, pol, g->phat, nullptr, g->v, g->rhat);
      { const int nb = g->nblk_last; LAUNCH(HJB_KC_REDUCE, nb, 16.0 * nb, 2.0 * nb, k_finalize<<<1, 1024, 0, st>>>(g->partial, nb, g->red, 0u, g->S, SC_AFTER_V)); }
      LAUNCH(HJB_KC_VECTOR, L.n_own, 24.0 * L.n_own, 4.0 * L.n_own,
             k_bicg_s<D><<<dims(g, L, (const void*)k_bicg_s<D>), kTX, 0, st>>>(L, g->S, g->r, g->v, g->s, g->partial));
      TRY(precond(g, mg, g->s, g->shat));
      launch_operator<D>(g, L, C, OP_APPLY, 2, dt, 0.0, pol, g->shat, nullptr, g->t, g->s);
      { const int nb = g->nblk_last; LAUNCH(HJB_KC_REDUCE, nb, 16.0 * nb, 2.0 * nb, k_finalize<<<1, 1024, 0, st>>>(g->partial, nb, g->red, 0u, g->S, SC_AFTER_T)); }
      LAUNCH(HJB_KC_VECTOR, L.n_own, 64.0 * L.n_own, 10.0 * L.n_own,
             k_bicg_x<D><<<dims(g, L, (const void*)k_bicg_x<D>), kTX, 0, st>>>(L, g->S, x, g->phat, g->shat, g->s, g->t, g->r, g->rhat, g->partial));
      { const int nb = g->nblk_last; LAUNCH(HJB_KC_REDUCE, nb, 16.0 * nb, 2.0 * nb, k_finalize<<<1, 1024, 0, st>>>(g->partial, nb, g->red, 0u, g->S, SC_AFTER_R)); }
      CKL();
      CK(cudaMemcpyAsync(g->hS, g->S, sizeof(KScal), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      ++it;
      ++inner;
      rr = g->hS->rr;
      if (!std::isfinite(rr)) return fail(HJB_ERR_NONFINITE, "non-finite residual in BiCGSTAB");
      if (std::sqrt(rr) <= tol) break;
      if (g->hS->breakdown) { restart_needed = true; break; }
    }
    // true residual check (recursive residual drifts, SURVEY hard part 5)
    launch_operator<D>(g, L, C, OP_RESID, 0, dt, 0.0, pol, x, F, g->r, nullptr);
    double tr2, trinf;
    TRY(norms_dev<D>(g, g->r, &tr2, &trinf));
    if (out) {
      out->iters = it;
      out->rres = bn2 > 0 ? tr2 / bn2 : tr2;
      out->rres_inf = bninf > 0 ? trinf / bninf : trinf;
    }
    if (tr2 <= tol) { converged = true; break; }
    if (it >= sp->krylov_maxit) break;
    (void)restart_needed;
  }
  if (out && converged && it == 0) {
    out->iters = 0;
    out->rres = bn2 > 0 ? std::sqrt(rr) / bn2 : 0.0;
    out->rres_inf = 0.0;
  }
  if (!converged) return fail(HJB_ERR_NOT_CONVERGED, "BiCGSTAB did not reach the tolerance");
  return HJB_OK;
}

extern "C" hjb_status hjb_solve(hjb_grid_t g, double dt, const uint8_t* policy, const double* F, double* x,
                                const hjb_solve_params* p, hjb_solve_stats* out) {
  if (!g || !policy || !F || !x) return fail(HJB_ERR_INVALID_ARG, "null argument");
  TRY(check_dt(g, dt));
  CK(cudaSetDevice(g->desc.device));
  hjb_solve_params def;
  hjb_solve_params_default(g->D, &def);
  const hjb_solve_params* sp = p ? p : &def;
  return g->D == 2 ? bicgstab<2>(g, dt, policy, F, x, sp, out) : bicgstab<3>(g, dt, policy, F, x, sp, out);
}

// ---------------------------------------------------------------------------- step
extern "C" hjb_status hjb_step(hjb_grid_t g, double dt, const double* U_prev, double* U, uint8_t* policy,
                               const double* psi, const hjb_solve_params* p, hjb_step_stats* out) {
  if (!g || !U_prev || !U) return fail(HJB_ERR_INVALID_ARG, "null argument");
  TRY(check_dt(g, dt));
  CK(cudaSetDevice(g->desc.device));
  hjb_solve_params def;
  hjb_solve_params_default(g->D, &def);
  const hjb_solve_params* sp = p ? p : &def;
  cudaStream_t st = g->st;
  const size_t vb = (size_t)g->N * sizeof(double);
  // stage host buffers (e2e path)
  const bool h_prev = !is_device_ptr(U_prev), h_U = !is_device_ptr(U);
  const bool h_pol = policy && !is_device_ptr(policy), h_psi = psi && !is_device_ptr(psi);
  const double* dprev = U_prev;
  double* dU = U;
  uint8_t* dpol = policy ? policy : g->pol_int;
  const double* dpsi = psi;
  if (h_prev) {
    if (!g->stage_prev) TRY(dalloc((void**)&g->stage_prev, vb));
    CK(cudaMemcpyAsync(g->stage_prev, U_prev, vb, cudaMemcpyHostToDevice, st));
    dprev = g->stage_prev;
  }
  if (h_U) {
    if (!g->stage_U) TRY(dalloc((void**)&g->stage_U, vb));
    dU = g->stage_U;
  }
  if (h_pol) {
    if (!g->stage_pol) TRY(dalloc((void**)&g->stage_pol, (size_t)g->N));
    CK(cudaMemcpyAsync(g->stage_pol, policy, (size_t)g->N, cudaMemcpyHostToDevice, st));
    dpol = g->stage_pol;
  }
  if (h_psi) {
    if (!g->stage_psi) TRY(dalloc((void**)&g->stage_psi, (size_t)g->n_boundary * sizeof(double)));
    CK(cudaMemcpyAsync(g->stage_psi, psi, (size_t)g->n_boundary * sizeof(double), cudaMemcpyHostToDevice, st));
    dpsi = g->stage_psi;
  }
  // a1: U <- U_prev with boundary psi(t_n)
  if (dU != dprev) CK(cudaMemcpyAsync(dU, dprev, vb, cudaMemcpyDeviceToDevice, st));
  if (dpsi) {
    const int nbb = (int)std::min<int64_t>((g->n_boundary + 255) / 256, 4096);
    const double nbd = (double)g->n_boundary;
    if (g->D == 2) LAUNCH(HJB_KC_BOUNDARY, nbd, 16.0 * nbd, 0, k_scatter_psi<2><<<nbb, 256, 0, st>>>(g->L0, g->n_boundary, dpsi, dU));
    else LAUNCH(HJB_KC_BOUNDARY, nbd, 16.0 * nbd, 0, k_scatter_psi<3><<<nbb, 256, 0, st>>>(g->L0, g->n_boundary, dpsi, dU));
    CKL();
  }
  hjb_step_stats S{};
  float ms;
  hjb_status result = HJB_OK;
  bool last_exact = true;  // the last policy evaluation reached krylov_rtol
  for (int it = 1; it <= sp->max_pi; ++it) {
    hjb_pi_stats pis{};
    cudaEventRecord(g->ev[0], st);
    TRY(policy_update_dev(g, dt, dU, dprev, dpol, g->F, &pis));
    cudaEventRecord(g->ev[1], st);
    cudaEventSynchronize(g->ev[1]);
    cudaEventElapsedTime(&ms, g->ev[0], g->ev[1]);
    S.ms_search += ms;
    const int slot = std::min(it - 1, HJB_MAX_PI_LOG - 1);
    S.changed[slot] = pis.changed;
    S.R[slot] = pis.R_max;
    S.final_R = pis.R_max;
    // stop: nonlinear residual certificate (any iterate), or a stable policy whose evaluation was exact
    if (it > 1 && (pis.R_max <= sp->tol_pi || (pis.changed == 0 && last_exact))) break;
    if (it == sp->max_pi) { result = fail(HJB_ERR_NOT_CONVERGED, "policy iteration hit max_pi"); break; }
    const bool settled = (it > 1 && pis.changed == 0);  // only reached after an inexact solve
    cudaEventRecord(g->ev[0], st);
    if (sp->use_mg && !(settled && g->mg_ready && g->mg_pol0 == dpol && g->mg_dt == dt))
      TRY(hjb_mg_setup(g, dt, dpol, &sp->mg));
    cudaEventRecord(g->ev[1], st);
    hjb_solve_stats ss{};
    // inexact Howard: while the policy still changes, evaluate it only to eta * ||r_0||
    const double eta = settled ? 0.0 : sp->pi_forcing;
    hjb_status s = g->D == 2 ? bicgstab<2>(g, dt, dpol, g->F, dU, sp, &ss, eta)
                             : bicgstab<3>(g, dt, dpol, g->F, dU, sp, &ss, eta);
    last_exact = (ss.rres <= sp->krylov_rtol);
    cudaEventRecord(g->ev[2], st);
    cudaEventSynchronize(g->ev[2]);
    cudaEventElapsedTime(&ms, g->ev[0], g->ev[1]);
    S.ms_setup += ms;
    cudaEventElapsedTime(&ms, g->ev[1], g->ev[2]);
    S.ms_solve += ms;
    S.pi_iters = it;
    S.krylov_iters[slot] = ss.iters;
    S.krylov_iters_total += ss.iters;
    S.final_rres = ss.rres;
    if (s != HJB_OK) { result = s; break; }
  }
  S.n_levels = (int32_t)g->levels.size();
  if (h_U) CK(cudaMemcpyAsync(U, dU, vb, cudaMemcpyDeviceToHost, st));
  if (h_pol) CK(cudaMemcpyAsync(policy, dpol, (size_t)g->N, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (out) *out = S;
  return result;
}

// ---------------------------------------------------------------------------- API: instrumentation
extern "C" hjb_status hjb_profile_reset(hjb_grid_t g, int32_t time_kernels) {
  if (!g) return fail(HJB_ERR_INVALID_ARG, "null handle");
  CK(cudaSetDevice(g->desc.device));
  prof_drain(g);
  g->prof = hjb_profile{};
  g->prof_timing = time_kernels != 0;
  g->prof.timed = g->prof_timing ? 1 : 0;
  return HJB_OK;
}

extern "C" hjb_status hjb_profile_read(hjb_grid_t g, hjb_profile* out) {
  if (!g || !out) return fail(HJB_ERR_INVALID_ARG, "null handle/out");
  CK(cudaSetDevice(g->desc.device));
  prof_drain(g);
  CK(cudaStreamSynchronize(g->st));
  *out = g->prof;
  return HJB_OK;
}
