// hjb.cu -- C-ABI of libhjb (include/hjb.h): handle management, coefficient upload, slab
// decomposition, and the host orchestration of policy iteration / BiCGSTAB / geometric multigrid.
// All arithmetic on grid data runs in the kernels of hjb_kernels.cuh; the host only sequences
// launches, halo exchanges and all-gathers (hjb_comm.h), and reads a few scalars (Krylov
// convergence, policy-iteration stopping) through pinned memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "hjb.h"
#include "hjb_comm.h"
#include "hjb_kernels.cuh"
#include "hjb_tma.cuh"
#include "hjb_win.cuh"
#include "hjb_search2.cuh"
#include "hjb_galerkin.cuh"
#include "hjb_agmg.cuh"
#include "hjb_nested.cuh"
#include <cub/device/device_scan.cuh>

namespace hjb {
struct WinPlan {
  bool ok = false;
  WinGeom geom{};
  SkipRect box{0, 0, 0, 0, 0, 0};
  size_t smem = 0;
  int grid = 0;
};
static const void* win_fn(int D, int P, bool gen) {
#define WF(DD, PP) (gen ? (const void*)k_search_win<DD, PP, true> : (const void*)k_search_win<DD, PP, false>)
  if (D == 2) return P == 1 ? WF(2, 1) : WF(2, 2);
  return P == 1 ? WF(3, 1) : P == 2 ? WF(3, 2) : WF(3, 3);
#undef WF
}
}  // namespace hjb


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
    if (e_ != cudaSuccess)                                                                        \
      return fail(HJB_ERR_CUDA, std::string("launch (hjb.cu:") + std::to_string(__LINE__) + "): " +  \
                                    cudaGetErrorString(e_));                                      \
  } while (0)
#define TRY(x)                     \
  do {                             \
    hjb_status s_ = (x);           \
    if (s_ != HJB_OK) return s_;   \
  } while (0)

static constexpr int kMaxBlocks = 148 * 16;  // partial-sum slots: 16 resident 128-thread CTAs per SM

// One multigrid level.  Level 0 is the fine grid.  "Slab" levels are decomposed like the fine grid
// (owned rows [r0, r1) of the slowest axis + H halo rows); "replicated" levels (at and below the
// gather level, nranks > 1 only) hold the full grid on every rank and are computed redundantly.
struct Level {
  LevelDev L{};
  int64_t elems = 0;              // local elements of a grid array on this level
  bool replicated = false;
  int64_t H = 0;                  // halo rows (slab levels, nranks > 1)
  std::vector<int64_t> r0s, r1s;  // slab levels: owned rows of every rank
  double* tmp = nullptr;          // smoother ping-pong
  double* res = nullptr;          // residual before restriction
  double* x = nullptr;            // coarse levels: correction
  double* b = nullptr;            // coarse levels: restricted rhs
  uint8_t* pol = nullptr;         // coarse levels: injected policy
  double* fields = nullptr;       // coarse levels: injected field planes
  CoefDev C{};
  double* Ainv = nullptr;         // coarsest level dense inverse
  double* dg = nullptr;           // smoothed levels: the diagonal of A (per policy, hjb_mg_setup)
  double* r2 = nullptr;           // W-cycle (gamma > 1): coarse residual / correction of a revisit
  double* e2 = nullptr;
  int* gcol = nullptr;            // Galerkin coarse operator (levels >= 1): ELL [kGalW][elems]
  double* gval = nullptr;
};

struct hjb_grid {
  hjb_grid_desc desc{};
  int D = 2, P = 1, K = 1, Q = 0;
  int64_t n = 0;
  double lo = 0, hi = 1, h = 0, k = 0;
  cudaStream_t st = nullptr;
  hjb_layout lay{};               // this rank's slab
  int R = 1, rank = 0;
  std::unique_ptr<Comm> comm;
  std::vector<int64_t> r0s, r1s;  // fine owned rows of every rank
  LevelDev L0{};
  int64_t N = 0, n_interior = 0, n_boundary = 0;
  // coefficients
  double* d_tab = nullptr;  // sigma_dir | b_dir | c_ctrl | f_basis | f_ctrl
  CoefDev C0{};
  bool have_coeffs = false;
  double reach_diff = 0.0, reach_drift = 0.0;  // max |offset| along the slowest axis, cells (level 0)
  // Krylov workspace
  double *r = nullptr, *rhat = nullptr, *p = nullptr, *v = nullptr, *s = nullptr, *t = nullptr;
  double *phat = nullptr, *shat = nullptr, *F = nullptr;
  double* partial = nullptr;
  double* red = nullptr;      // [0..1] result, [2..3] this rank's partial result
  double* red_all = nullptr;  // [nranks][2] gathered
  KScal* S = nullptr;
  KScal* hS = nullptr;        // pinned mirror
  double* hred = nullptr;     // pinned mirror of red
  uint8_t* pol_int = nullptr;
  double* scratch = nullptr;  // const-input copy for halo exchange (nranks > 1)
  // staging for host pointers
  double *stage_prev = nullptr, *stage_U = nullptr, *stage_psi = nullptr;
  uint8_t* stage_pol = nullptr;
  // gather-level staging (nranks > 1)
  void* gsend = nullptr;
  void* grecv = nullptr;
  size_t gbytes = 0;
  // multigrid
  std::vector<Level> levels;
  hjb_mg_params mgp{};
  bool mg_ready = false;
  const uint8_t* mg_pol0 = nullptr;
  double mg_dt = 0.0;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  // instrumentation (hjb_profile_*)
  // ring of per-launch event pairs; when it is full the OLDER half is drained (long finished: the
  // host runs at most a queue depth ahead), so timing never stalls the launch pipeline
  static constexpr int kSlots = 4096;
  bool prof_timing = false;
  cudaEvent_t pev[2 * kSlots] = {};
  int pcls[kSlots] = {};
  int phead = 0, npend = 0;
  hjb_profile prof{};
  int nplanes0 = 0;  // per-node coefficient planes read by the operator (sigma/b/c fields)
  int sms = 148;
  int nblk_last = 1;  // CTAs of the last dims() launch (partials to reduce)
  // deep rectangles (2D): per-rank scale-field ranges and per-axis endpoint reach
  std::vector<double> h_sd, h_bd;  // host copies of sigma_dir / b_dir
  std::vector<double> h_cc, h_fc, h_fb;  // host copies of c_ctrl / f_ctrl / f_basis (k_search_deep2 tables)
  double* d_rng = nullptr;    // [scmin_p, scmax_p]_p, [bsmin, bsmax]
  bool reach_ok = false;      // per-axis reach known (scale fields only): deep rectangles enabled
  bool tma_ok = false;        // TMA-windowed search tiles (k_search_tma)
  TmaGeom tma{};
  size_t tma_smem = 0;
  int tma_grid = 0;
  bool use_dg = true;          // smoother reads the stored diagonal (Level::dg)
  bool mg_f32 = false;         // the cycle's vectors in fp32 (hjb_mg_params.precision = 1, not Galerkin)
  int mg_gamma = 1;            // cycle index on levels owning >= gamma_min nodes (hjb_mg_params)
  int nu_coarse = 0;           // > 0: smoothing sweeps on levels >= 1 (experiment knob HJB_NU_COARSE)
  int64_t gamma_min = 0;       // revisit a coarse level only if it has >= gamma_min owned nodes
  WinPlan win_deep, win_full;  // shared-memory window search (k_search_win) over the deep box /
                               // over the whole interior (general geometry)
  double rdiff_ax[3] = {0, 0, 0}, rdrift_ax[3] = {0, 0, 0};
  double* rng_part = nullptr; // k_field_ranges block partials
  double2* upair = nullptr;   // (U_i, U_{i+1}) pair copy of the searched U (k_search_deep2)
  double4* uquad = nullptr;   // cell-corner copy of the searched U (k_search_deep2<..., QUADS>)
  // certified search skipping inside hjb_step (k_search_deep2<..., GAP>)
  float* gap = nullptr;             // [N] per-node lower bound of H_second - H_best
  double* uold[2] = {nullptr, nullptr};  // U at the previous search of the step (ping-pong)
  int uold_cur = 0;
  unsigned long long* d_gapred = nullptr;  // k_gap_delta maxima (+ the skipped-CTA counter)
  bool gap_on = false;      // the next policy_update_dev scans with gap bookkeeping
  bool gap_valid = false;   // gap / uold describe the previous search of this step
  double gap_G = 0.0, gap_D = 0.0, gap_umax = 0.0;  // cell-difference / max |dU| / max |U| bounds
  bool gap_first = true;    // the next GAP scan is a full one (bskip < 0)
  int64_t gap_skipped = 0, gap_ctas = 0;  // diagnostics (HJB_SKIP_DEBUG)
  bool search3 = false;       // k_search_deep3 on the deep rectangle (opt-in, HJB_SEARCH3=1)
  bool search2p = false;      // k_search_deep2p (software-pipelined) on the deep rectangle (opt-in)
  // halo exchange overlapped with the rows that do not read halos (nranks > 1, halo_begin): the
  // exchange runs on xst; the operator launches the inner band first, waits on xev[1], then the
  // edge bands
  cudaStream_t xst = nullptr;
  cudaEvent_t xev[2] = {nullptr, nullptr};
  struct {
    bool pending = false;
    int64_t H = 0;
    bool lo = false, hi = false;  // a neighbour below / above (its halo rows are in flight)
  } ovl;
  // nested iteration (HJB_GUESS_NESTED, hjb_nested.cuh): the same problem on the grid coarsened
  // 2^child_m times per axis, its fields injected from this grid's
  hjb_grid* child = nullptr;
  int child_m = 0;
  bool child_dirty = true;    // fields / tables changed since the last injection
  double* child_fields = nullptr;
  double* child_U = nullptr;
  double* child_prev = nullptr;
  uint8_t* child_pol = nullptr;
  double* vtheta = nullptr;   // theta U + (1-theta) U_prev (theta-scheme search argument)
  bool galerkin = false;      // coarse operators by the Galerkin product (hjb_mg_params.coarse_op)
  int* gb_col = nullptr;      // B = A P scratch of the Galerkin setup (ELL [kGalWB][elems_0])
  double* gb_val = nullptr;
  int* d_flag = nullptr;      // device overflow flag
  // aggregation AMG (hjb_solve_params.solver = 1; hjb_agmg.cuh)
  struct AgLevel {
    int64_t N = 0;
    int* col = nullptr;
    double* val = nullptr;
    double* dg = nullptr;
    int* agg = nullptr;   // this level -> next (not on the coarsest)
    int* mem = nullptr;   // members (<= 4) of the next level's aggregates: [4][N_next]
    double *x = nullptr, *b = nullptr, *r = nullptr, *t = nullptr, *z[2] = {nullptr, nullptr},
           *az[2] = {nullptr, nullptr};
    double* Ainv = nullptr;   // the coarsest level's dense inverse (points into ag_dense)
    int64_t cap = 0;          // capacity of the N-sized arrays (levels are pooled across setups)
    int64_t cap_agg = 0, cap_mem = 0;
  };
  std::vector<AgLevel> ag;
  std::vector<AgLevel> ag_pool;   // released levels, reused by the next setup (no cudaMalloc/Free,
                                  // which synchronise the device, on the per-policy setup path)
  double* ag_dense = nullptr;     // kAgDenseMax^2 dense inverse of the coarsest level
  int* ag_agg1c = nullptr;        // pass-1 copies of the pairwise matching (sized for level 0)
  int* ag_mem1c = nullptr;
  const uint8_t* ag_pol = nullptr;
  double ag_dt = 0.0;
  bool ag_ready = false;
  int* ag_i[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};  // setup scratch
  void* ag_cub = nullptr;
  size_t ag_cub_bytes = 0;
  double* ag_sc = nullptr;    // K-cycle inner GCR scalars on the device, 8 per level
  double* ag_Z[16] = {};      // outer FGCR directions (compact)
  double* ag_AZ[16] = {};
  const double* bsamp = nullptr;  // exact-psi mode: face samples of psi (caller-owned, retained)
  int brefine = 0;
  bool drift_reg = false;     // deep drift endpoints stay within one cell of the node (|offset| < 1)
  double h_rng[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // host copy of d_rng (scale-field ranges)
  // CUDA graphs of the multigrid tail: the cycle from level graph_level down (levels owning <=
  // kGraphMaxNodes nodes, launch-latency bound) is captured once per hierarchy and replayed
  struct SubGraph {
    size_t level;
    const void* b;   // the captured cycle's right-hand side / output (fp64 or fp32 vectors)
    const void* out;
    const uint8_t* pol0;
    cudaGraphExec_t exec;
    int64_t launches;
  };
  std::vector<SubGraph> graphs;
  size_t graph_level = (size_t)-1;
  double graph_dt = 0.0;          // dt / omega baked into the captured kernels' parameters
  bool capturing = false;
  int64_t cap_launches = 0;
  cudaStream_t cap_st = nullptr;  // private capture stream (the legacy default stream cannot capture)
};

static void agmg_free(hjb_grid* g);

// ---------------------------------------------------------------------------- instrumentation
// accumulate the `m` oldest pending launches
static void prof_drain_oldest(hjb_grid* g, int m) {
  if (m <= 0) return;
  const int K = hjb_grid::kSlots;
  cudaEventSynchronize(g->pev[2 * ((g->phead + m - 1) % K) + 1]);
  for (int i = 0; i < m; ++i) {
    const int k = (g->phead + i) % K;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, g->pev[2 * k], g->pev[2 * k + 1]) == cudaSuccess) g->prof.ms[g->pcls[k]] += ms;
  }
  g->phead = (g->phead + m) % K;
  g->npend -= m;
}
static void prof_drain(hjb_grid* g) { prof_drain_oldest(g, g->npend); }
// With per-launch timing on, launches over fewer than kTimeMinNodes nodes (the small multigrid
// levels, launch-latency bound) are not timed -- two event records each would add ~10 % to a W-cycle
// step -- and their bytes / flops / nodes are left out so every class total stays the timed subset;
// their device time is the unattributed remainder.  nodes <= 0: accounted by the caller, always timed.
constexpr double kTimeMinNodes = 16384.0;
static bool prof_timed(const hjb_grid* g, double nodes) {
  return g->prof_timing && !g->capturing && (nodes <= 0.0 || nodes >= kTimeMinNodes);
}
static void prof_pre(hjb_grid* g, int, double nodes) {
  if (!prof_timed(g, nodes)) return;
  if (g->npend == hjb_grid::kSlots) prof_drain_oldest(g, hjb_grid::kSlots / 2);
  cudaEventRecord(g->pev[2 * ((g->phead + g->npend) % hjb_grid::kSlots)], g->st);
}
static void prof_post(hjb_grid* g, int cls, double nodes, double bytes, double flops) {
  if (g->capturing) {  // recorded into a graph: counted at every replay instead
    g->cap_launches += 1;
    return;
  }
  g->prof.launches[cls] += 1;
  g->prof.total_launches += 1;
  if (g->prof_timing && !prof_timed(g, nodes)) return;
  g->prof.nodes[cls] += nodes;
  g->prof.bytes[cls] += bytes;
  g->prof.flops[cls] += flops;
  if (!g->prof_timing) return;
  const int k = (g->phead + g->npend) % hjb_grid::kSlots;
  cudaEventRecord(g->pev[2 * k + 1], g->st);
  g->pcls[k] = cls;
  g->npend += 1;
}
// LAUNCH(class, nodes, algorithmic bytes, algorithmic flops, kernel<<<...>>>(...))
#define LAUNCH(CLS, NODES, BYTES, FLOPS, ...)                              \
  do {                                                                     \
    prof_pre(g, CLS, (double)(NODES));                                     \
    __VA_ARGS__;                                                           \
    prof_post(g, CLS, (double)(NODES), (double)(BYTES), (double)(FLOPS));  \
  } while (0)

// ---------------------------------------------------------------------------- small helpers
// 2D launch over the owned interior of level L: x covers an x1 line, y strides over lines.  All
// CTAs are made co-resident (occupancy x SMs) so the lines in flight form one band that moves
// through the grid and the +-reach rows it gathers from stay in L2.
// A kernel's dynamic shared-memory limit is a process-wide attribute of the function: raise it once
// to the device's opt-in maximum (setting it to one grid's requirement would make another grid's
// larger launch fail -- two handles with different window plans in one process).
static cudaError_t allow_smem(const void* fn) {
  static std::mutex mu;
  static std::map<const void*, bool> done;
  std::lock_guard<std::mutex> lock(mu);
  if (done[fn]) return cudaSuccess;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa{};
  cudaError_t e = cudaFuncGetAttributes(&fa, fn);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
  if (e == cudaSuccess) done[fn] = true;
  return e;
}

static int occupancy_of(const void* fn, size_t smem = 0, int block = kTX) {
  // shared by every handle; thread-rank grids (HJB_COMM_THREADS) call it concurrently
  static std::mutex mu;
  static std::map<std::pair<const void*, size_t>, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_pair(fn, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int occ = 0;
#ifdef HJB_L1MAX
  cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 0);  // maximal L1
#endif
  if (smem > 48 * 1024) allow_smem(fn);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, block, smem) != cudaSuccess || occ < 1) occ = 1;
  cache[key] = occ;
  return occ;
}
static dim3 dims(hjb_grid* g, const LevelDev& L, const void* fn, int bx = kBX, size_t smem = 0) {
  const int by = kTX / bx;
  const int gx = std::max(1, (L.nI + bx - 1) / bx);
  const int64_t cap = std::min<int64_t>((int64_t)occupancy_of(fn, smem) * g->sms, kMaxBlocks);
  const int64_t rows = std::min<int64_t>(std::max((L.nrows + by - 1) / by, 1), 65535);
  const int gy = (int)std::max<int64_t>(1, std::min<int64_t>(rows, cap / gx));
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

static int64_t ipow(int64_t b, int e) {
  int64_t r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

// level geometry: owned interior rows [r0, r1) of the slowest axis, local rows [lr0, lr1)
static LevelDev make_level(int D, int64_t n, double lo, double hi, double k, double k2, int64_t r0, int64_t r1,
                           int64_t lr0, int64_t lr1) {
  LevelDev L{};
  L.n = (int)n;
  L.nI = (int)(n - 2);
  L.nrows = (int)((r1 - r0) * ipow(n - 2, D - 2));
  L.row_elems = ipow(n, D - 1);
  L.local_row0 = lr0;
  L.local_rows = lr1 - lr0;
  L.row_first = r0;
  L.n_own = (int64_t)L.nrows * L.nI;
  L.h = (hi - lo) / (double)(n - 1);
  L.nm1 = (double)(n - 1);
  L.kh = k / L.h;
  L.k2h = k2 / L.h;
  L.inv_2k2 = 1.0 / (2.0 * k2);
  L.inv_k2 = 1.0 / k2;
  L.pf_rows = 0;
  L.local_elems = (int)(L.local_rows * L.row_elems);
  return L;
}
static LevelDev full_level(int D, int64_t n, double lo, double hi, double k, double k2) {
  return make_level(D, n, lo, hi, k, k2, 1, n - 1, 0, n);
}

// ---------------------------------------------------------------------------- communication
// halo exchange of `rows` rows each side of a slab-level array x (no-op for one rank / replicated)
static void halo_end(hjb_grid* g);
// (esz: element size -- 8 for fp64 arrays, 4 for the fp32 cycle vectors)
static hjb_status halo_exchange(hjb_grid* g, const Level& lv, void* xv, int64_t rows, size_t esz = sizeof(double)) {
  if (g->R == 1 || lv.replicated || rows <= 0) return HJB_OK;
  char* x = static_cast<char*>(xv);
  if (g->st != g->xst) halo_end(g);
  const int64_t re = lv.L.row_elems, lr0 = lv.L.local_row0;
  const int64_t r0 = lv.r0s[g->rank], r1 = lv.r1s[g->rank];
  Msg m[2];
  int nm = 0;
  const size_t bytes = (size_t)(rows * re) * esz;
  const int64_t e = (int64_t)esz;
  if (g->rank > 0) m[nm++] = Msg{g->rank - 1, x + (r0 - lr0) * re * e, x + (r0 - rows - lr0) * re * e, bytes};
  if (g->rank + 1 < g->R) m[nm++] = Msg{g->rank + 1, x + (r1 - rows - lr0) * re * e, x + (r1 - lr0) * re * e, bytes};
  std::string err;
  if (g->comm->exchange(g->st, m, nm, &err) != cudaSuccess)
    return fail(g->desc.comm == HJB_COMM_NCCL ? HJB_ERR_NCCL : HJB_ERR_CUDA, "halo exchange: " + err);
  return HJB_OK;
}

// the stream waits for a halo exchange started by halo_begin
static void halo_end(hjb_grid* g) {
  if (!g->ovl.pending) return;
  cudaStreamWaitEvent(g->st, g->xev[1], 0);
  g->ovl.pending = false;
}

// Start the halo exchange of x on the exchange stream and return: the next launch_operator runs
// the rows that read no halo row while the rows travel, then waits (halo_end) and runs the edge
// rows.  Falls back to the blocking exchange without a second stream or while capturing a graph.
static hjb_status halo_begin(hjb_grid* g, const Level& lv, void* x, int64_t rows, size_t esz = sizeof(double)) {
  if (g->R == 1 || lv.replicated || rows <= 0) return HJB_OK;
  halo_end(g);
  if (!g->xst || g->capturing) return halo_exchange(g, lv, x, rows, esz);
  cudaEventRecord(g->xev[0], g->st);                // x is final on the compute stream
  cudaStreamWaitEvent(g->xst, g->xev[0], 0);
  cudaStream_t st = g->st;
  g->st = g->xst;  // the exchange is enqueued on the exchange stream
  const hjb_status r = halo_exchange(g, lv, x, rows, esz);
  g->st = st;
  if (r != HJB_OK) return r;
  cudaEventRecord(g->xev[1], g->xst);
  g->ovl.pending = true;
  g->ovl.H = rows;
  g->ovl.lo = g->rank > 0;
  g->ovl.hi = g->rank + 1 < g->R;
  return HJB_OK;
}

// reduce the block partials of the last dims() launch to red[0..1] on the device (several ranks:
// per-rank results all-gathered and combined in rank order), then the BiCGSTAB scalar update
static hjb_status reduce_dev(hjb_grid* g, int nblk, unsigned maxmask, int which) {
  if (g->R == 1) {
    LAUNCH(HJB_KC_REDUCE, nblk, 16.0 * nblk, 2.0 * nblk,
           k_finalize<<<1, 1024, 0, g->st>>>(g->partial, nblk, g->red, maxmask, g->S, which));
    CKL();
    return HJB_OK;
  }
  LAUNCH(HJB_KC_REDUCE, nblk, 16.0 * nblk, 2.0 * nblk,
         k_finalize<<<1, 1024, 0, g->st>>>(g->partial, nblk, g->red + 2, maxmask, g->S, SC_NONE));
  CKL();
  std::string err;
  if (g->comm->allgather(g->st, g->red + 2, g->red_all, 2 * sizeof(double), &err) != cudaSuccess)
    return fail(HJB_ERR_NCCL, "allgather: " + err);
  LAUNCH(HJB_KC_REDUCE, g->R, 16.0 * g->R, 2.0 * g->R,
         k_combine<<<1, 32, 0, g->st>>>(g->red_all, g->R, g->red, maxmask, g->S, which));
  CKL();
  return HJB_OK;
}

static double host_finalize(hjb_grid* g, int nblk, unsigned maxmask, int which, hjb_status* err,
                            double* second = nullptr) {
  *err = reduce_dev(g, nblk, maxmask, which);
  if (*err != HJB_OK) return NAN;
  cudaMemcpyAsync(g->hred, g->red, 2 * sizeof(double), cudaMemcpyDeviceToHost, g->st);
  cudaError_t e = cudaStreamSynchronize(g->st);
  if (e != cudaSuccess) {
    *err = fail(HJB_ERR_CUDA, std::string("sync: ") + cudaGetErrorString(e));
    return NAN;
  }
  if (second) *second = g->hred[1];
  return g->hred[0];
}

// copy rows [J0_q, J1_q) of a full-grid array from every rank to every rank (gather level)
static hjb_status gather_rows(hjb_grid* g, void* full, size_t elem, int64_t row_elems,
                              const std::vector<int64_t>& J0, const std::vector<int64_t>& J1) {
  int64_t maxr = 0;
  for (int q = 0; q < g->R; ++q) maxr = std::max(maxr, J1[q] - J0[q]);
  const size_t chunk = (size_t)(maxr * row_elems) * elem;
  if (chunk == 0) return HJB_OK;
  if (chunk > g->gbytes) {
    cudaFree(g->gsend);
    cudaFree(g->grecv);
    g->gsend = g->grecv = nullptr;
    TRY(dalloc(&g->gsend, chunk));
    TRY(dalloc(&g->grecv, chunk * g->R));
    g->gbytes = chunk;
  }
  const int me = g->rank;
  const size_t mine = (size_t)((J1[me] - J0[me]) * row_elems) * elem;
  if (mine)
    CK(cudaMemcpyAsync(g->gsend, (char*)full + (size_t)(J0[me] * row_elems) * elem, mine,
                       cudaMemcpyDeviceToDevice, g->st));
  std::string err;
  if (g->comm->allgather(g->st, g->gsend, g->grecv, chunk, &err) != cudaSuccess)
    return fail(HJB_ERR_NCCL, "gather level: " + err);
  for (int q = 0; q < g->R; ++q) {
    const size_t b = (size_t)((J1[q] - J0[q]) * row_elems) * elem;
    if (q != me && b)
      CK(cudaMemcpyAsync((char*)full + (size_t)(J0[q] * row_elems) * elem, (char*)g->grecv + q * chunk, b,
                         cudaMemcpyDeviceToDevice, g->st));
  }
  return HJB_OK;
}

// L2 prefetch distance of a level: its widest reach in rows + 2 (HJB_NO_PREFETCH: off)
static int prefetch_rows(hjb_grid* g, const LevelDev& L) {
#ifdef HJB_NO_PREFETCH
  return 0;
#else
  const double rd = g->reach_diff * (L.kh / g->L0.kh), rb = g->reach_drift * (L.k2h / g->L0.k2h);
  return (int)std::floor(std::max(rd, rb)) + 2;
#endif
}

// every owned interior node of level L as a box
static SkipRect full_box(hjb_grid* g, const LevelDev& L) {
  if (g->D == 2) return SkipRect{0, L.nI, 0, L.nrows, 0, 1};
  return SkipRect{0, L.nI, 0, L.nrows / L.nI, 0, L.nI};
}

// box (loop coordinates) of level L whose nodes have every endpoint of every control strictly
// inside the domain (empty when unknown, e.g. with per-node sigma/b offset fields)
static SkipRect deep_rect(hjb_grid* g, const LevelDev& L) {
  SkipRect r{0, 0, 0, 0, 0, 0};
  if (!g->reach_ok) return r;
  const int D = g->D, n = L.n;
  int m[3];
  for (int d = 0; d < D; ++d) {
    const double rr = std::max(g->rdiff_ax[d] * (L.kh / g->L0.kh), g->rdrift_ax[d] * (L.k2h / g->L0.k2h));
    m[d] = (int)std::floor(rr + 1e-6) + 1;  // i in [m, n-1-m]
  }
  const int c0 = m[0] - 1, c1 = n - 1 - m[0];
  const int slow = D - 1;
  const int planes = (D == 2) ? L.nrows : L.nrows / L.nI;
  const int zlo = std::max<int>(m[slow], (int)L.row_first), zhi = std::min<int>(n - 1 - m[slow], (int)L.row_first + planes - 1);
  if (c1 <= c0 || zhi < zlo) return r;
  r = SkipRect{c0, c1, zlo - (int)L.row_first, zhi + 1 - (int)L.row_first, 0, 1};
  if (D == 3) {
    r.y0 = m[1] - 1;
    r.y1 = n - 1 - m[1];
    if (r.y1 <= r.y0) return SkipRect{0, 0, 0, 0, 0, 0};
  }
  return r;
}

// `outer` minus `inner` as up to 6 boxes (slowest axis slabs, then y slabs, then x slabs), so each
// piece gets its own launch shape (a thin strip launched over the whole grid would leave the work
// to a handful of CTAs)
static int ring_strips(const SkipRect& o, const SkipRect& in, SkipRect* out) {
  int k = 0;
  const bool empty = in.c1 <= in.c0 || in.r1 <= in.r0 || in.y1 <= in.y0;
  if (empty) {
    out[k++] = o;
    return k;
  }
  if (in.r0 > o.r0) out[k++] = SkipRect{o.c0, o.c1, o.r0, in.r0, o.y0, o.y1};
  if (o.r1 > in.r1) out[k++] = SkipRect{o.c0, o.c1, in.r1, o.r1, o.y0, o.y1};
  if (in.y0 > o.y0) out[k++] = SkipRect{o.c0, o.c1, in.r0, in.r1, o.y0, in.y0};
  if (o.y1 > in.y1) out[k++] = SkipRect{o.c0, o.c1, in.r0, in.r1, in.y1, o.y1};
  if (in.c0 > o.c0) out[k++] = SkipRect{o.c0, in.c0, in.r0, in.r1, in.y0, in.y1};
  if (o.c1 > in.c1) out[k++] = SkipRect{in.c1, o.c1, in.r0, in.r1, in.y0, in.y1};
  return k;
}
static LevelDev shape_of(const LevelDev& L, const SkipRect& r) {
  LevelDev S = L;
  S.nI = r.c1 - r.c0;
  S.nrows = (r.r1 - r.r0) * (r.y1 - r.y0);
  return S;
}

// the fine-level coefficients for kernels whose argument is U itself: with the exact-psi mode the
// truncated endpoints read psi from the face samples (Remark rhs)
static CoefDev coef_u(const hjb_grid* g) {
  CoefDev C = g->C0;
  if (g->bsamp) {
    C.bsamp = g->bsamp;
    C.brefine = g->brefine;
    C.bM = (int)(g->brefine * (g->n - 1) + 1);
  }
  return C;
}

// ---------------------------------------------------------------------------- dimension dispatch
// V: element type of x, b, y, u (float only for the multigrid modes of the fp32 cycle); given
// explicitly (the pointer arguments do not deduce it: nullptr is a valid x / b / u)
template <typename T>
struct nodeduce { using type = T; };
template <int D, typename V = double>
static void launch_operator(hjb_grid* g, const LevelDev& L, const CoefDev& C, int mode, int ndot, double dt,
                            double omega, const uint8_t* pol, const typename nodeduce<V>::type* x,
                            const typename nodeduce<V>::type* b, typename nodeduce<V>::type* y,
                            const typename nodeduce<V>::type* u, bool fine = true) {
  cudaStream_t st = g->st;
  const int cls = mode == OP_DIAG ? HJB_KC_COARSE  // multigrid setup
                  : !fine ? HJB_KC_MG_COARSE
                          : (mode == OP_APPLY ? HJB_KC_APPLY : (mode == OP_RESID ? HJB_KC_RESID : HJB_KC_SMOOTH));
  const double nodes = (double)L.n_own;
  const bool gathers = mode != OP_JACOBI0 && mode != OP_DIAG;
  const double vs = (double)sizeof(V);
  const double bpn = 1.0 + vs + (gathers ? vs : 0.0) + (mode != OP_APPLY && mode != OP_DIAG ? vs : 0.0) +
                     (ndot >= 1 || mode == OP_JACOBI_D ? vs : 0.0) + 8.0 * g->nplanes0;
  const double fpn = (2.0 * g->P + 1.0) * (1 << D) * 2.0 + 4.0 + 2.0 * ndot;
  const size_t tsm = (size_t)g->K * (g->P * D + D + 1) * sizeof(double);  // control tables in smem
  // the deep rectangle of this level (2D): lean fast-path kernel there, general kernel on the
  // boundary-layer strips around it (small levels: one general launch)
  const SkipRect full = full_box(g, L);
  SkipRect rect = deep_rect(g, L);
  // small levels: one launch; 3D: the box + 6 slabs measured slower than one general launch
  // (cfg3 step 89 -> 114 ms), so the operator keeps the general kernel there
  if ((int64_t)L.nI * L.nrows < (1 << 16) || g->D == 3) rect = SkipRect{0, 0, 0, 0, 0, 0};
  const bool has_deep = rect.c1 > rect.c0 && rect.r1 > rect.r0;
  SkipRect strips[6];
  const int ns = ring_strips(full, rect, strips);
  // pieces in launch order: with a halo exchange in flight (halo_begin), first every piece's band of
  // slab rows that reads no halo row, then (after the exchange) the edge bands
  SkipRect pc[2][3 * 7];
  bool pdeep[2][3 * 7];
  int npc[2] = {0, 0};
  {
    int64_t lo = 0, hi = 1 << 30;  // slab-axis rows (loop coordinates) reading no halo row
    const bool split = g->ovl.pending;
    if (split) {
      const int64_t rows_own = D == 2 ? L.nrows : L.nrows / std::max(1, L.nI);
      lo = g->ovl.lo ? g->ovl.H : 0;
      hi = rows_own - (g->ovl.hi ? g->ovl.H : 0);
      if (hi <= lo) {  // a thin slab: no inner band
        halo_end(g);
        lo = 0;
        hi = 1 << 30;
      }
    }
    auto add = [&](int ph, const SkipRect& r, int64_t a, int64_t b, bool deep) {
      SkipRect q = r;
      q.r0 = (int)std::max<int64_t>(r.r0, a);
      q.r1 = (int)std::min<int64_t>(r.r1, b);
      if (q.r1 > q.r0 && q.c1 > q.c0) {
        pc[ph][npc[ph]] = q;
        pdeep[ph][npc[ph]++] = deep;
      }
    };
    for (int k = 0; k <= ns; ++k) {
      const bool deep = (k == ns);
      if (deep && !has_deep) break;
      const SkipRect& r = deep ? rect : strips[k];
      add(0, r, lo, hi, deep);
      if (g->ovl.pending) {
        add(1, r, 0, lo, deep);
        add(1, r, hi, 1 << 30, deep);
      }
    }
  }
#define OPL1(PP, M, ND, DP, RR)                                                                             \
  do {                                                                                                      \
    const LevelDev LL = shape_of(L, RR);                                                                    \
    const double nn = (double)LL.nI * LL.nrows;                                                             \
    LAUNCH(cls, nn, nn * bpn, nn * fpn,                                                                     \
           k_operator<D, PP, M, ND, DP, V><<<dims(g, LL, (const void*)k_operator<D, PP, M, ND, DP, V>, kBX, tsm), \
                                         dim3(kBX, kBY), tsm, st>>>(L, C, dt, omega, pol, x, b, y, u,       \
                                                                    g->partial + 2 * nb, RR));              \
    nb += g->nblk_last;                                                                                     \
  } while (0)
#define OPLP(PP, M, ND)                                           \
  do {                                                            \
    int nb = 0;                                                   \
    for (int ph = 0; ph < 2; ++ph) {                              \
      if (ph == 1) halo_end(g);                                   \
      for (int k = 0; k < npc[ph]; ++k) {                         \
        if (pdeep[ph][k]) OPL1(PP, M, ND, true, pc[ph][k]);       \
        else OPL1(PP, M, ND, false, pc[ph][k]);                   \
      }                                                           \
    }                                                             \
    g->nblk_last = nb;                                            \
  } while (0)
#define OPL(M, ND)                                                                                          \
  do {                                                                                                      \
    if (g->P == 1) OPLP(1, M, ND);                                                                          \
    else if (g->P == 2) OPLP(2, M, ND);                                                                     \
    else OPLP((D > 2 ? 3 : 2), M, ND);                                                                      \
  } while (0)
  if (!g->capturing && (!g->prof_timing || nodes >= kTimeMinNodes)) g->prof.calls[cls] += 1;  // timed subset
  if constexpr (!std::is_same<V, double>::value) {  // fp32 cycle: the multigrid modes only
    if (mode == OP_RESID) OPL(OP_RESID, 0);
    else if (mode == OP_JACOBI) OPL(OP_JACOBI, 0);
    else if (mode == OP_JACOBI_D) OPL(OP_JACOBI_D, 0);
    else if (mode == OP_DIAG) OPL(OP_DIAG, 0);
    else OPL(OP_JACOBI0, 0);
  } else if (mode == OP_APPLY) {
    if (ndot == 0) OPL(OP_APPLY, 0);
    else if (ndot == 1) OPL(OP_APPLY, 1);
    else OPL(OP_APPLY, 2);
  } else if (mode == OP_RESID) {
    if (ndot == 0) OPL(OP_RESID, 0);
    else OPL(OP_RESID, 2);
  } else if (mode == OP_JACOBI) {
    OPL(OP_JACOBI, 0);
  } else if (mode == OP_JACOBI_D) {
    OPL(OP_JACOBI_D, 0);
  } else if (mode == OP_DIAG) {
    OPL(OP_DIAG, 0);
  } else {
    OPL(OP_JACOBI0, 0);
  }
#undef OPL
#undef OPLP
#undef OPL1
  (void)nodes;
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
  o->gather_n = (dim == 3) ? 33 : 129;
  o->gamma = (dim == 3) ? 1 : 2;  // 3D: the V-cycle already contracts by <= 0.45 (W measured slower)
  o->gamma_min_nodes = 131072;
  o->coarse_op = 0;  // rediscretised coarse operators (NS); 1 = Galerkin R A P (NEXT-4)
  o->precision = 1;  // fp32 cycle vectors (preconditioner only, reading xxxi); 0 = fp64
}

extern "C" void hjb_solve_params_default(int32_t dim, hjb_solve_params* o) {
  if (!o) return;
  o->krylov_rtol = 1e-12;
  o->krylov_maxit = 2000;
  o->use_mg = 1;
  o->tol_pi = 1e-10;
  o->max_pi = 50;
  hjb_mg_params_default(dim, &o->mg);
  o->pi_forcing = 0.01;  // with the W-cycle (solves are cheap): 3 PI per step at cfg4 (DESIGN.md §3 xxii)
  o->guess = HJB_GUESS_PREV;
  o->krylov_rtol_inf = 1e-9;  // SURVEY §8c-xvii secondary stop (reading xvii)
  o->theta = 1.0;             // implicit Euler (the paper's experiments)
  o->solver = 0;              // BiCGSTAB + geometric multigrid (1: GCR + aggregation AMG, NEXT-1)
  o->nested_coarsen = 2;      // HJB_GUESS_NESTED: 4x coarser per axis ...
  o->nested_min_n = 513;      // ... while the coarse grid keeps n >= 513
  o->nested_increment = 0;    // prolong the coarse solution (1: U_prev + the prolonged coarse increment)
}

// ---------------------------------------------------------------------------- API: partition
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

extern "C" hjb_status hjb_comm_unique_id(void* out128) {
  if (!out128) return fail(HJB_ERR_INVALID_ARG, "null out");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(HJB_ERR_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
  std::memcpy(out128, &id, sizeof(id));
  return HJB_OK;
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
    cudaFree(l.dg);
    cudaFree(l.r2);
    cudaFree(l.e2);
    cudaFree(l.gcol);
    cudaFree(l.gval);
  }
  g->levels.clear();
  cudaFree(g->gb_col);
  cudaFree(g->gb_val);
  g->gb_col = nullptr;
  g->gb_val = nullptr;
  g->mg_ready = false;
  for (auto& sg : g->graphs) cudaGraphExecDestroy(sg.exec);
  g->graphs.clear();
  g->graph_level = (size_t)-1;
}

extern "C" hjb_status hjb_grid_destroy(hjb_grid_t g) {
  if (!g) return fail(HJB_ERR_INVALID_ARG, "null handle");
  cudaSetDevice(g->desc.device);
  if (g->st) cudaStreamSynchronize(g->st);
  if (g->child) hjb_grid_destroy(g->child);
  cudaFree(g->child_fields);
  cudaFree(g->child_U);
  cudaFree(g->child_prev);
  cudaFree(g->child_pol);
  free_levels(g);
  double* bufs[] = {g->d_tab, g->r, g->rhat, g->p, g->v, g->s, g->t, g->phat, g->shat, g->F,
                    g->partial, g->red, g->red_all, g->scratch, g->stage_prev, g->stage_U, g->stage_psi};
  for (double* b : bufs) cudaFree(b);
  cudaFree(g->gsend);
  cudaFree(g->grecv);
  cudaFree(g->d_rng);
  cudaFree(g->rng_part);
  cudaFree(g->upair);
  cudaFree(g->uquad);
  cudaFree(g->gap);
  cudaFree(g->uold[0]);
  cudaFree(g->uold[1]);
  cudaFree(g->d_gapred);
  cudaFree(g->vtheta);
  cudaFree(g->d_flag);
  agmg_free(g);
  if (g->cap_st) cudaStreamDestroy(g->cap_st);
  if (g->xst) cudaStreamDestroy(g->xst);
  for (auto& e : g->xev)
    if (e) cudaEventDestroy(e);
  cudaFree(g->S);
  cudaFree(g->pol_int);
  cudaFree(g->stage_pol);
  cudaFreeHost(g->hS);
  cudaFreeHost(g->hred);
  for (auto& e : g->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : g->pev)
    if (e) cudaEventDestroy(e);
  g->comm.reset();
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
  if (d->nranks < 1 || d->rank < 0 || d->rank >= d->nranks) return fail(HJB_ERR_INVALID_ARG, "bad rank/nranks");
  if (d->nranks > 1 && !d->nccl_id) return fail(HJB_ERR_INVALID_ARG, "nranks > 1 needs nccl_id (128 bytes)");
  if (d->nranks > 1 && d->comm != HJB_COMM_NCCL && d->comm != HJB_COMM_THREADS)
    return fail(HJB_ERR_INVALID_ARG, "unknown comm backend");
  hjb_layout lay;
  TRY(hjb_partition(d->dim, d->n, d->nranks, d->rank, d->halo, &lay));
  // local arrays are indexed with 32-bit offsets; one x1 line must fit the partial-sum slots
  if (lay.local_elems >= (1LL << 31) || (d->n - 2) > (int64_t)std::min(kBX, kSBX) * kMaxBlocks)
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
  g->R = d->nranks;
  g->rank = d->rank;
  g->lay = lay;
  cudaDeviceGetAttribute(&g->sms, cudaDevAttrMultiProcessorCount, d->device);
  if (g->sms < 1) g->sms = 148;
  for (int q = 0; q < g->R; ++q) {
    hjb_layout lq;
    hjb_partition(d->dim, d->n, d->nranks, q, d->halo, &lq);
    g->r0s.push_back(lq.row0);
    g->r1s.push_back(lq.row1);
  }
  g->L0 = make_level(g->D, g->n, g->lo, g->hi, g->k, g->h, lay.row0, lay.row1, lay.local_row0,
                     lay.local_row0 + lay.local_rows);
  g->N = lay.local_elems;
  g->n_interior = lay.n_interior;
  g->n_boundary = lay.n_boundary;
  if (g->R > 1) {
    std::string err;
    bool ok;
    if (d->comm == HJB_COMM_THREADS) {
      auto* c = new ThreadComm();
      g->comm.reset(c);
      ok = ThreadComm::init(c, d->nccl_id, d->rank, d->nranks, &err);
    } else {
      auto* c = new NcclComm();
      g->comm.reset(c);
      ok = NcclComm::init(c, d->nccl_id, d->rank, d->nranks, &err);
    }
    if (!ok) {
      hjb_grid_destroy(g);
      return fail(HJB_ERR_NCCL, err);
    }
  }
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
  if ((s = dalloc((void**)&g->partial, (size_t)kMaxBlocks * 8 * sizeof(double))) != HJB_OK ||
      (s = dalloc((void**)&g->red, 4 * sizeof(double))) != HJB_OK ||
      (s = dalloc((void**)&g->red_all, (size_t)2 * g->R * sizeof(double))) != HJB_OK ||
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
  if (g->R > 1 && !getenv("HJB_NO_OVERLAP")) {
    cudaStreamCreateWithFlags(&g->xst, cudaStreamNonBlocking);
    for (auto& e : g->xev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  }
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

extern "C" hjb_status hjb_grid_query(hjb_grid_t g, hjb_layout* o) {
  if (!g || !o) return fail(HJB_ERR_INVALID_ARG, "null handle/out");
  *o = g->lay;
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
  g->h_sd.assign(h.begin(), h.begin() + nsd);
  g->h_bd.assign(h.begin() + nsd, h.begin() + nsd + nbd);
  g->h_cc.assign(h.begin() + nsd + nbd, h.begin() + nsd + nbd + nc);
  g->h_fb.assign(h.begin() + nsd + nbd + nc, h.begin() + nsd + nbd + nc + nfb);
  g->h_fc.assign(h.begin() + nsd + nbd + nc + nfb, h.begin() + tot);
  return HJB_OK;
}

// ---------------------------------------------------------------------------- TMA tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn tma_encoder() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
    cudaGetLastError();
  }
  return fn;
}

// {2n, local_rows/2} pair-row view of a level-0 grid array (see hjb_tma.cuh), box bw x bh
static bool encode_pair_view(hjb_grid* g, const double* U, CUtensorMap* map) {
  EncodeTiledFn enc = tma_encoder();
  if (!enc) return false;
  const cuuint64_t n = (cuuint64_t)g->n;
  const cuuint64_t dims[2] = {2 * n, (cuuint64_t)(g->L0.local_rows / 2)};
  const cuuint64_t strides[1] = {2 * n * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)g->tma.bw, (cuuint32_t)g->tma.bh};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)U, dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ---------------------------------------------------------------------------- deep rectangles
// Per-rank ranges of the per-node scale fields -> per-axis reach of every control's endpoints ->
// the rectangle of nodes none of whose endpoints can be truncated (2D, no sigma/b offset fields).
// deep_rect() scales it to each multigrid level; the lean kernels run there.
// shared-memory window search (hjb_win.cuh): choose the tile of `box` (the fine level's deep box, or
// with gen the whole interior) whose window [tile - m, tile + m] fits in shared memory at the least
// staging + idle-thread cost
static hjb_status setup_win(hjb_grid* g, const SkipRect& dr, bool gen, WinPlan* plan) {
  const int D = g->D, P = g->P, K = g->K;
  *plan = WinPlan{};
  if (dr.c1 <= dr.c0 || dr.r1 <= dr.r0 || dr.y1 <= dr.y0) return HJB_OK;
  int m[3] = {0, 0, 0}, ex[3] = {1, 1, 1};
  for (int d = 0; d < D; ++d) m[d] = (int)std::floor(std::max(g->rdiff_ax[d], g->rdrift_ax[d]) + 1e-6) + 1;
  ex[0] = dr.c1 - dr.c0;
  ex[1] = D == 2 ? dr.r1 - dr.r0 : dr.y1 - dr.y0;
  ex[2] = D == 3 ? dr.r1 - dr.r0 : 1;
  const int ntab = ((K * (P * D + D + 2 + g->Q) + 15) / 16) * 16;
  const size_t cmb = (size_t)(kWinS - 1) * kWinNodes * (2 * sizeof(double) + sizeof(int));  // merge buffers
  const size_t limit = 227 * 1024 - 1024 - cmb;  // opt-in maximum less static shared memory
  const double loads = (double)K * (2 * P + 1) * (1 << D);  // shared-memory gathers per node
  static const int T0[] = {32, 64, 128}, T1[] = {1, 2, 4, 8, 16, 32, 64}, T2[] = {1, 2, 3, 4, 6, 8};
  double best = INFINITY;
  WinGeom W{};
  for (int t0 : T0)
    for (int t1 : T1)
      for (int t2 : T2) {
        if (D == 2 && t2 != 1) continue;
        const int t[3] = {t0, t1, t2};
        const int nodes = t0 * t1 * t2;
        if (nodes < kWinNodes) continue;
        int w[3], nt[3];
        double vol = 1.0, slots = 1.0, cov = 1.0;
        for (int d = 0; d < 3; ++d) {
          w[d] = t[d] + 2 * m[d];
          nt[d] = (ex[d] + t[d] - 1) / t[d];
          vol *= w[d];
          slots *= (double)nt[d] * t[d];
          cov *= ex[d];
        }
        if ((ntab + vol) * sizeof(double) > limit) continue;
        const double ntiles = (double)nt[0] * nt[1] * nt[2];
        // idle threads in partial tiles, window staging (~4 gathers per staged double), and fewer
        // tiles than SMs
        double cost = (slots / cov) * (1.0 + 4.0 * vol / nodes / loads);
        if (ntiles < g->sms) cost *= (double)g->sms / ntiles;
        if (cost < best) {
          best = cost;
          for (int d = 0; d < 3; ++d) {
            W.t[d] = t[d];
            W.m[d] = m[d];
            W.w[d] = w[d];
            W.nt[d] = nt[d];
          }
          W.ntiles = nt[0] * nt[1] * nt[2];
          W.tab = ntab;
        }
      }
  if (!std::isfinite(best)) return HJB_OK;
  const size_t smem = ((size_t)W.tab + (size_t)W.w[0] * W.w[1] * W.w[2]) * sizeof(double) + cmb;
  const void* fn = win_fn(D, P, gen);
  CK(allow_smem(fn));
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kWinNT, smem) != cudaSuccess || occ < 1) {
    cudaGetLastError();
    return HJB_OK;
  }
  plan->geom = W;
  plan->box = dr;
  plan->smem = smem;
  plan->grid = std::min(W.ntiles, std::min(occ * g->sms, kMaxBlocks));
  plan->ok = true;
  return HJB_OK;
}

static hjb_status setup_deep(hjb_grid* g) {
  g->reach_ok = false;
  g->win_deep = WinPlan{};
  g->win_full = WinPlan{};
#ifdef HJB_NO_DEEP
  return HJB_OK;
#endif
  if (g->C0.sigma_node || g->C0.b_node || getenv("HJB_NO_DEEP")) return HJB_OK;
  const int P = g->P, D = g->D, K = g->K;
  const LevelDev& L = g->L0;
  if (L.nrows <= 0) return HJB_OK;
  // per-rank ranges of the scale fields
  const int nv = 2 * P + 2;
  if (!g->rng_part) TRY(dalloc((void**)&g->rng_part, (size_t)kMaxBlocks * 8 * sizeof(double)));
  if (!g->d_rng) TRY(dalloc((void**)&g->d_rng, 8 * sizeof(double)));
#define FRNG(DD, PP) \
  k_field_ranges<DD, PP><<<dims(g, L, (const void*)k_field_ranges<DD, PP>), dim3(kBX, kBY), 0, g->st>>>(L, g->C0, g->rng_part)
  if (D == 2) {
    if (P == 1) FRNG(2, 1);
    else FRNG(2, 2);
  } else {
    if (P == 1) FRNG(3, 1);
    else if (P == 2) FRNG(3, 2);
    else FRNG(3, 3);
  }
#undef FRNG
  CKL();
  const int nb = g->nblk_last;
  std::vector<double> part((size_t)nb * nv);
  CK(cudaMemcpyAsync(part.data(), g->rng_part, part.size() * sizeof(double), cudaMemcpyDeviceToHost, g->st));
  CK(cudaStreamSynchronize(g->st));
  std::vector<double> mx(nv, -INFINITY);
  for (int b = 0; b < nb; ++b)
    for (int k = 0; k < nv; ++k) mx[k] = std::max(mx[k], part[(size_t)b * nv + k]);
  double rng[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int k = 0; k < P + 1; ++k) {
    rng[2 * k] = -mx[2 * k];
    rng[2 * k + 1] = mx[2 * k + 1];
  }
  for (int k = 0; k < nv; ++k)
    if (!std::isfinite(rng[k])) return HJB_OK;
  std::memcpy(g->h_rng, rng, sizeof(rng));
  CK(cudaMemcpyAsync(g->d_rng, rng, nv * sizeof(double), cudaMemcpyHostToDevice, g->st));
  CK(cudaStreamSynchronize(g->st));
  // reach per axis over all controls / endpoints (diffusion and drift separately: they scale
  // differently across multigrid levels)
  for (int d = 0; d < 3; ++d) g->rdiff_ax[d] = g->rdrift_ax[d] = 0.0;
  for (int a = 0; a < K; ++a)
    for (int e = 0; e <= P; ++e)
      for (int d = 0; d < D; ++d) {
        const double c = (e < P) ? L.kh * g->h_sd[(a * P + e) * D + d] : L.k2h * g->h_bd[a * D + d];
        const double f0 = rng[2 * e], f1 = rng[2 * e + 1];
        const double o0 = c * f0, o1 = c * f1;
        const double r = std::max(std::fabs(o0), std::fabs(o1));
        double& rr = (e < P) ? g->rdiff_ax[d] : g->rdrift_ax[d];
        rr = std::max(rr, r);
      }
  g->reach_ok = true;
  g->drift_reg = g->rdrift_ax[0] < 1.0 - 1e-9 && g->rdrift_ax[1] < 1.0 - 1e-9;
  // TMA-windowed search tiles inside the deep rectangle of the fine level (single tensor map view)
  g->tma_ok = false;
#ifndef HJB_NO_TMA
  // opt-in (HJB_TMA=1): measured slower than the direct deep kernel at cfg2/cfg4
  if (D == 2 && getenv("HJB_TMA") && !getenv("HJB_NO_TMA")) {
    double jit[2] = {0, 0};
    for (int a = 0; a < K; ++a)
      for (int e = 0; e <= P; ++e)
        for (int d = 0; d < D; ++d) {
          const double c = (e < P) ? L.kh * g->h_sd[(a * P + e) * D + d] : L.k2h * g->h_bd[a * D + d];
          jit[d] = std::max(jit[d], std::fabs(c * rng[2 * e + 1] - c * rng[2 * e]));
        }
    const SkipRect dr = deep_rect(g, L);
    TmaGeom T{};
    T.bw = (kWX - 1 + (int)std::ceil(jit[0] + 2e-6) + 3 + 1 + 1) & ~1;  // +1: aligned box start
    const int bwy = kWY - 1 + (int)std::ceil(jit[1] + 2e-6) + 3;
    T.bh = (bwy + 1) / 2 + 1;
    T.slot = ((T.bw * T.bh + 15) / 16) * 16;
    T.ntx = (dr.c1 - dr.c0) / kWX;
    // every pair-row a window needs must exist in the {2n, local_rows/2} view
    const int reach_y = (int)std::floor(std::max(g->rdiff_ax[1], g->rdrift_ax[1]) + 1e-6) + 2;
    const int pair_rows = (int)(L.local_rows / 2);
    int rmax = dr.r1;  // exclusive, loop coordinates
    while (rmax > dr.r0 && (int)L.row_first + rmax - 1 + reach_y - (int)L.local_row0 >= 2 * pair_rows) --rmax;
    T.nty = (rmax - dr.r0) / kWY;
    T.tiles = SkipRect{dr.c0, dr.c0 + T.ntx * kWX, dr.r0, dr.r0 + T.nty * kWY};
    const int E = 2 * P + 1;
    const size_t ntab = (size_t)K * (P * D + D + 2 + g->Q);
    const size_t smem = (ntab + (size_t)2 * E * 2 * T.slot) * sizeof(double) + 128;
    if (T.ntx > 0 && T.nty > 0 && T.bw <= 256 && T.bh <= 256 && smem <= 200 * 1024 && tma_encoder()) {
      const void* fn = P == 1 ? (const void*)k_search_tma<1> : (const void*)k_search_tma<2>;
      CK(allow_smem(fn));
      int occ = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kWT, smem) == cudaSuccess && occ >= 1) {
        g->tma = T;
        g->tma_smem = smem;
        g->tma_grid = std::min(T.ntx * T.nty, std::min(occ * g->sms, kMaxBlocks));
        g->tma_ok = true;
      }
    }
  }
#endif
  // HJB_WIN=0: direct kernels; =1: window over the deep box only (+ general strips); =2: window over
  // the whole interior where it fits, else over the deep box.  Default 2 in 2D, 1 in 3D (measured:
  // the general geometry in the 3D window kernel spills at 128 registers)
  const char* wenv = getenv("HJB_WIN");
  const int wmode = wenv ? atoi(wenv) : (D == 2 ? 2 : 1);
  if (wmode >= 1 && !g->tma_ok) {
    TRY(setup_win(g, deep_rect(g, L), false, &g->win_deep));
    if (wmode >= 2) TRY(setup_win(g, full_box(g, L), true, &g->win_full));
  }
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
  g->child_dirty = true;
  g->mg_ready = false;
  for (auto& sg : g->graphs) cudaGraphExecDestroy(sg.exec);  // captured kernels hold field pointers
  g->graphs.clear();
  {  // widest stencil offset: halo check (several ranks) and the L2 prefetch distance
    const double nodes = (double)g->L0.n_own;
    if (g->D == 2)
      LAUNCH(HJB_KC_BOUNDARY, nodes, nodes * 8.0 * (1 + g->nplanes0), 0,
             k_reach<2><<<dims(g, g->L0, (const void*)k_reach<2>), dim3(kBX, kBY), 0, g->st>>>(g->L0, g->C0, g->partial));
    else
      LAUNCH(HJB_KC_BOUNDARY, nodes, nodes * 8.0 * (1 + g->nplanes0), 0,
             k_reach<3><<<dims(g, g->L0, (const void*)k_reach<3>), dim3(kBX, kBY), 0, g->st>>>(g->L0, g->C0, g->partial));
    CKL();
    hjb_status err;
    double rb = 0.0;
    const double rd = host_finalize(g, g->nblk_last, 0x3u, SC_NONE, &err, &rb);
    if (err != HJB_OK) return err;
    g->reach_diff = rd;
    g->reach_drift = rb;
    const int64_t need = (int64_t)std::floor(std::max(rd, rb) * (1.0 + 1e-12)) + 1;
    g->L0.pf_rows = prefetch_rows(g, g->L0);
    TRY(setup_deep(g));
    if (g->R > 1 && need > g->lay.halo) {
      g->have_coeffs = false;
      return fail(HJB_ERR_INVALID_ARG, "halo too small for these coefficients: need " + std::to_string(need) +
                                           " rows, grid has " + std::to_string(g->lay.halo));
    }
  }
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
  g->h_fb.assign(h.begin(), h.begin() + (size_t)K * Q);
  g->h_fc.assign(h.begin() + (size_t)K * Q, h.end());
  return HJB_OK;
}

// the fine level as a Level (before hjb_mg_setup built the hierarchy)
static const Level& fine_level(hjb_grid* g, Level& tmp) {
  if (!g->levels.empty()) return g->levels[0];
  tmp.L = g->L0;
  tmp.replicated = false;
  tmp.H = g->lay.halo;
  tmp.r0s = g->r0s;
  tmp.r1s = g->r1s;
  return tmp;
}

static hjb_status halo_begin(hjb_grid* g, const Level& lv, void* x, int64_t rows, size_t esz);
// a const caller array whose halo rows must be filled: copy into scratch first (nranks > 1); the
// exchange is left in flight (halo_begin) for the launch_operator that follows
static hjb_status halo_input(hjb_grid* g, const double* x, const double** out) {
  *out = x;
  if (g->R == 1) return HJB_OK;
  if (!g->scratch) TRY(dalloc((void**)&g->scratch, (size_t)g->N * sizeof(double)));
  CK(cudaMemcpyAsync(g->scratch, x, (size_t)g->N * sizeof(double), cudaMemcpyDeviceToDevice, g->st));
  Level tmp;
  TRY(halo_begin(g, fine_level(g, tmp), g->scratch, g->lay.halo));
  *out = g->scratch;
  return HJB_OK;
}

// ---------------------------------------------------------------------------- policy improvement
// k_search_deep2 (hjb_search2.cuh): 2D, no offset fields, the control tables fit the parameter
// structs, Q in {1,2,8}, scale fields of one sign over the rank (zero steps and the drift quadrant are
// per-control facts), drift endpoints within one cell, table entries either 0 or far from underflow
static bool search2_ok(hjb_grid* g) {
  const int P = g->P, Q = g->Q, K = g->K;
  const int S = 2 * P + 4 + Q + P + 7;  // STabLayout<P, Q>::S
  if (g->D != 2 || !(Q == 1 || Q == 2 || Q == 8) || K * S > kSTabN || K > 256) return false;
  if (g->C0.sigma_node || g->C0.b_node || !g->reach_ok || !g->drift_reg) return false;
  for (int p = 0; p < P; ++p)
    if (!(g->h_rng[2 * p] > 0.0)) return false;     // min sigma scale > 0
  if (!(g->h_rng[2 * P] > 0.0)) return false;       // min b scale > 0
  for (double v : g->h_sd)
    if (v != 0.0 && std::fabs(v) < 1e-200) return false;
  for (double v : g->h_bd)
    if (v != 0.0 && std::fabs(v) < 1e-200) return false;
  return true;
}

template <int P, int Q, bool STRIP, bool QUADS = false, int KU = 0, bool GAP = false>
static void search2_launch(hjb_grid* g, const LevelDev& LL, double dt, const double* U, const double* Uprev,
                           uint8_t* pol, double* F, const SkipRect& rect, const STab& tab, const STabQuad& quad,
                           int* nblk, const GapArgs& ga = GapArgs{}) {
  const void* fn = (const void*)k_search_deep2<P, Q, STRIP, QUADS, KU, GAP>;
  const int64_t tiles = (int64_t)((LL.nI + kSBX - 1) / kSBX) * ((LL.nrows + kS2Y - 1) / kS2Y);
  const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, std::min<int64_t>((int64_t)occupancy_of(fn, 0, kS2T) * g->sms, kMaxBlocks)));
  LAUNCH(HJB_KC_SEARCH, 0, 0, 0,
         k_search_deep2<P, Q, STRIP, QUADS, KU, GAP><<<nb, dim3(kSBX, kS2Y), 0, g->st>>>(
             g->L0, STRIP ? coef_u(g) : g->C0, dt, U, g->upair, g->uquad, Uprev, pol, F, g->partial + 2 * *nblk, rect,
             tab, quad, ga));
  if (GAP) g->gap_ctas += nb > 0 ? (int64_t)((LL.nI + kSBX - 1) / kSBX) * ((LL.nrows + kS2Y - 1) / kS2Y) : 0;
  *nblk += nb;
}

// the deep rectangle with the software-pipelined k_search_deep2p
template <int P, int Q>
static hjb_status search2p_launch(hjb_grid* g, const LevelDev& LL, double dt, const double* U, const double* Uprev,
                                  uint8_t* pol, double* F, const SkipRect& rect, const STab& tab, const STabQuad& quad,
                                  int* nblk) {
  const void* fn = (const void*)k_search_deep2p<P, Q>;
  const int64_t tiles = (int64_t)((LL.nI + kSBX - 1) / kSBX) * ((LL.nrows + kS2Y - 1) / kS2Y);
  const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, std::min<int64_t>((int64_t)occupancy_of(fn, 0, kS2T) * g->sms, kMaxBlocks)));
  LAUNCH(HJB_KC_SEARCH, 0, 0, 0,
         k_search_deep2p<P, Q><<<nb, dim3(kSBX, kS2Y), 0, g->st>>>(g->L0, g->C0, dt, U, Uprev, pol, F,
                                                                   g->partial + 2 * *nblk, rect, tab, quad));
  *nblk += nb;
  return HJB_OK;
}

// the deep rectangle with k_search_deep3 (node-local bracket staged in shared memory)
template <int P, int Q>
static hjb_status search3_launch(hjb_grid* g, const LevelDev& LL, double dt, const double* U, const double* Uprev,
                                 uint8_t* pol, double* F, const SkipRect& rect, const STab& tab, const STabQuad& quad,
                                 int* nblk) {
  const void* fn = (const void*)k_search_deep3<P, Q>;
  const size_t smem = (size_t)g->K * kS2T * sizeof(double);
  CK(allow_smem(fn));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kS2T, smem));
  const int64_t tiles = (int64_t)((LL.nI + kSBX - 1) / kSBX) * ((LL.nrows + kS2Y - 1) / kS2Y);
  const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, std::min<int64_t>((int64_t)std::max(1, occ) * g->sms, kMaxBlocks)));
  LAUNCH(HJB_KC_SEARCH, 0, 0, 0,
         k_search_deep3<P, Q><<<nb, dim3(kSBX, kS2Y), smem, g->st>>>(g->L0, g->C0, dt, U, g->uquad, Uprev, pol, F,
                                                                     g->partial + 2 * *nblk, rect, tab, quad));
  *nblk += nb;
  return HJB_OK;
}

template <int P, int Q>
static void search2_tables(hjb_grid* g, STab& tab, STabQuad& quad) {
  using T = STabLayout<P, Q>;
  const double* sd = g->h_sd.data();
  const double* bd = g->h_bd.data();
  const double inv_2k2 = g->L0.inv_2k2, inv_k2 = g->L0.inv_k2;
  for (int a = 0; a < g->K; ++a) {
    double* t = tab.v + a * T::S;
    double wsum = 0.0;
    for (int p = 0; p < P; ++p) {
      t[T::SD + 2 * p] = sd[(a * P + p) * 2];
      t[T::SD + 2 * p + 1] = sd[(a * P + p) * 2 + 1];
      const bool nz = sd[(a * P + p) * 2] != 0.0 || sd[(a * P + p) * 2 + 1] != 0.0;
      t[T::W + p] = nz ? inv_2k2 : 0.0;
      wsum += 2.0 * t[T::W + p];
    }
    t[T::BD] = bd[a * 2];
    t[T::BD + 1] = bd[a * 2 + 1];
    t[T::WD] = (bd[a * 2] != 0.0 || bd[a * 2 + 1] != 0.0) ? inv_k2 : 0.0;
    t[T::WSUM] = wsum + t[T::WD];
    t[T::C] = g->h_cc[a];
    t[T::FC] = g->h_fc[a];
    for (int q = 0; q < Q; ++q) t[T::FB + q] = g->h_fb[(size_t)a * Q + q];
    quad.v[a] = (bd[a * 2] < 0.0 ? 1 : 0) | (bd[a * 2 + 1] < 0.0 ? 2 : 0);
    t[T::CMW] = t[T::C] - t[T::WSUM];
    t[T::DQ] = bd[a * 2] < 0.0 ? 1.0 : 0.0;
    t[T::DQ + 1] = bd[a * 2 + 1] < 0.0 ? 1.0 : 0.0;
    t[T::ABD] = std::fabs(bd[a * 2]);
    t[T::ABD + 1] = std::fabs(bd[a * 2 + 1]);
  }
}

// the deep rectangle (strips = nullptr) or the boundary-layer strips around it (ns boxes)
// this search's skip bound and rounding margins (k_search_deep2<..., GAP>) from the control tables:
//   |H^a_j(U) - H^a_j(U_old)| <= sum_e w_e |I dU(z_e) - dU_j| + |c^a| |dU_j|
// and a multilinear interpolant moves by at most G per cell along either axis (G = max |dU_i' - dU_i|
// over grid edges), so |I dU(z_e) - dU_j| <= G (|o_e,1| + |o_e,2|) with o_e the endpoint offsets in
// cells, bounded by the scale-field maxima (DESIGN.md §6 "Certified search skipping")
template <int P, int Q>
static GapArgs gap_args(hjb_grid* g, const STab& tab) {
  using T = STabLayout<P, Q>;
  GapArgs ga{};
  ga.gap = g->gap;
  ga.nskip = reinterpret_cast<int*>(g->d_gapred + 3);
  const double eps = 2.220446049250313e-16;
  const double G = g->gap_G + 4.0 * eps * g->gap_umax, Dm = g->gap_D + 2.0 * eps * g->gap_umax;
  const double bsmax = g->h_rng[2 * P + 1];
  double B = 0.0, wc = 0.0, fc = 0.0;
  for (int q = 0; q < 8; ++q) ga.fbmax[q] = 0.0;
  for (int a = 0; a < g->K; ++a) {
    const double* t = tab.v + a * T::S;
    double b = std::fabs(t[T::C]) * Dm;
    for (int p = 0; p < P; ++p)
      b += 2.0 * t[T::W + p] * G * g->L0.kh * g->h_rng[2 * p + 1] *
           (std::fabs(t[T::SD + 2 * p]) + std::fabs(t[T::SD + 2 * p + 1]));
    b += t[T::WD] * G * g->L0.k2h * bsmax * (std::fabs(t[T::BD]) + std::fabs(t[T::BD + 1]));
    // second bound: every tap is a convex combination of dU values, so |I dU(z_e) - dU_j| <= 2 max|dU|;
    // it wins when dU is rough at the cell scale (G ~ max|dU|: the late searches of a step)
    const double b2 = (2.0 * t[T::WSUM] + std::fabs(t[T::C])) * Dm;
    B = std::max(B, std::min(b, b2));
    wc = std::max(wc, 2.0 * t[T::WSUM] + std::fabs(t[T::C]));
    fc = std::max(fc, std::fabs(t[T::FC]));
    for (int q = 0; q < Q && q < 8; ++q) ga.fbmax[q] = std::max(ga.fbmax[q], std::fabs(t[T::FB + q]));
  }
  ga.bskip = g->gap_first ? -1.0 : B * (1.0 + 1e-9);
  ga.gmargin = 128.0 * eps * wc * g->gap_umax;
  ga.fcmax = fc;
  return ga;
}

static hjb_status launch_search2(hjb_grid* g, double dt, const double* U, const double* Uprev, uint8_t* pol,
                                 double* F, const SkipRect& rect, int* nblk, const SkipRect* strips = nullptr,
                                 int ns = 0) {
  static thread_local STab tab;       // 24 KB + 1 KB: kernel parameters, not on the stack
  static thread_local STabQuad quad;
  const LevelDev LL = shape_of(g->L0, rect);
#define S2(PP, QQ)                                                                                 \
  do {                                                                                             \
    search2_tables<PP, QQ>(g, tab, quad);                                                          \
    if (!strips && g->search2p)                                                                    \
      TRY((search2p_launch<PP, QQ>(g, LL, dt, U, Uprev, pol, F, rect, tab, quad, nblk)));          \
    else if (!strips && g->uquad && g->search3)                                                    \
      TRY((search3_launch<PP, QQ>(g, LL, dt, U, Uprev, pol, F, rect, tab, quad, nblk)));           \
    else if (!strips && g->uquad && g->K == 32 && PP == 2 && getenv("HJB_KUNROLL"))                \
      search2_launch<PP, QQ, false, true, 32>(g, LL, dt, U, Uprev, pol, F, rect, tab, quad, nblk); \
    else if (!strips && g->uquad)                                                                  \
      search2_launch<PP, QQ, false, true>(g, LL, dt, U, Uprev, pol, F, rect, tab, quad, nblk);     \
    else if (!strips && g->gap_on)                                                                 \
      search2_launch<PP, QQ, false, false, 0, true>(g, LL, dt, U, Uprev, pol, F, rect, tab, quad,  \
                                                    nblk, gap_args<PP, QQ>(g, tab));               \
    else if (!strips)                                                                              \
      search2_launch<PP, QQ, false>(g, LL, dt, U, Uprev, pol, F, rect, tab, quad, nblk);           \
    for (int k = 0; k < ns; ++k) {                                                                 \
      const LevelDev LS = shape_of(g->L0, strips[k]);                                              \
      if (LS.nI > 0 && LS.nrows > 0)                                                               \
        search2_launch<PP, QQ, true>(g, LS, dt, U, Uprev, pol, F, strips[k], tab, quad, nblk);     \
    }                                                                                              \
  } while (0)
  const int P = g->P, Q = g->Q;
  if (P == 1) {
    if (Q == 1) S2(1, 1); else if (Q == 2) S2(1, 2); else S2(1, 8);
  } else {
    if (Q == 1) S2(2, 1); else if (Q == 2) S2(2, 2); else S2(2, 8);
  }
#undef S2
  CKL();
  return HJB_OK;
}

// U's halo rows must already be exchanged
// Certified search skipping, called before each search of hjb_step's policy iteration (first: the
// step's first search, a full scan that records the gaps).  One pass of k_gap_delta gives max |U|,
// max |dU| and the largest cell difference of dU = U - U_old, and snapshots U as the next U_old.
static hjb_status gap_prepare(hjb_grid* g, const double* U, bool first) {
  g->gap_on = false;
  // opt-in (HJB_SKIP=1): measured slower at cfg4 (1708 vs 1600 ms per step, profiles/r02_s_*): the GAP
  // scan costs +25 % per full search and the grid-wide bound certifies too few CTAs
  const char* skip_env = getenv("HJB_SKIP");
  if (!skip_env || atoi(skip_env) == 0 || g->R != 1 || g->D != 2 || g->C0.c_node || getenv("HJB_NO_SKIP") || getenv("HJB_QUADS") ||
      getenv("HJB_SEARCH3") || getenv("HJB_SEARCH2P") || getenv("HJB_KUNROLL") || !search2_ok(g)) {
    g->gap_valid = false;
    return HJB_OK;
  }
  const size_t N = (size_t)g->N;
  if (!g->gap) {
    TRY(dalloc((void**)&g->gap, N * sizeof(float)));
    TRY(dalloc((void**)&g->uold[0], N * sizeof(double)));
    TRY(dalloc((void**)&g->uold[1], N * sizeof(double)));
    TRY(dalloc((void**)&g->d_gapred, 4 * sizeof(unsigned long long)));
  }
  first = first || !g->gap_valid;
  CK(cudaMemsetAsync(g->d_gapred, 0, 4 * sizeof(unsigned long long), g->st));
  const double* uo = first ? nullptr : g->uold[g->uold_cur];
  double* un = g->uold[first ? g->uold_cur : 1 - g->uold_cur];
  const double nn = (double)N;
  // a streaming pass: counted with the vector kernels (not in the search's flop roofline)
  LAUNCH(HJB_KC_VECTOR, nn, (first ? 16.0 : 24.0) * nn, 6.0 * nn,
         k_gap_delta<<<(int)std::min<int64_t>(((int64_t)N + 255) / 256, (int64_t)g->sms * 8), 256, 0, g->st>>>(
             U, uo, un, g->L0.n, (int64_t)N, g->d_gapred));
  CKL();
  double m[3];
  CK(cudaMemcpyAsync(m, g->d_gapred, 3 * sizeof(double), cudaMemcpyDeviceToHost, g->st));
  CK(cudaStreamSynchronize(g->st));
  if (!first) g->uold_cur = 1 - g->uold_cur;
  g->gap_umax = m[0];
  g->gap_D = m[1];
  g->gap_G = m[2];
  g->gap_first = first;
  g->gap_on = std::isfinite(m[0]) && std::isfinite(m[1]) && std::isfinite(m[2]);
  if (!g->gap_on) g->gap_valid = false;
  return HJB_OK;
}

static hjb_status policy_update_dev(hjb_grid* g, double dt, const double* U, const double* Uprev, uint8_t* pol,
                                    double* F, hjb_pi_stats* out) {
  halo_end(g);  // the search kernels take no row split: U's halo rows must have arrived
  const double nodes = (double)g->L0.n_own;
  const double bpn = 8.0 + 8.0 + 1.0 + 1.0 + 8.0 + 8.0 * g->Q + 8.0 * g->nplanes0;
  const double fpn = g->K * ((2.0 * g->P + 1.0) * (1 << g->D) * 2.0 + 2.0 * g->Q + 4.0);
  const size_t tsm = (size_t)g->K * (g->P * g->D + g->D + 2 + g->Q) * sizeof(double);
  // deep rectangle (2D): lean fast-path kernel there (TMA-windowed tiles inside it), general
  // kernel on the boundary-layer strips
  const SkipRect full = full_box(g, g->L0);
  const SkipRect rect = deep_rect(g, g->L0);
  const bool has_deep = rect.c1 > rect.c0 && rect.r1 > rect.r0;
  int nblk = 0;
  CUtensorMap umap;
  const bool use_tma = has_deep && g->tma_ok && ((uintptr_t)U & 15) == 0 && encode_pair_view(g, U, &umap);
  const SkipRect tiles = use_tma ? g->tma.tiles : SkipRect{0, 0, 0, 0};
  SkipRect gstrips[6], dstrips[6];
  // shared-memory window kernels: over the whole interior (no strips), or over the deep box
  // the whole-interior window (general geometry) has no exact-psi path: the general kernel takes the
  // strips in that mode
  const WinPlan* wp = use_tma ? nullptr : (g->win_full.ok && !g->bsamp) ? &g->win_full
                                        : (has_deep && g->win_deep.ok) ? &g->win_deep : nullptr;
  const CoefDev CU = coef_u(g);
  const bool win_all = wp == &g->win_full;
  int ngs = win_all ? 0 : ring_strips(full, rect, gstrips);
  // 2D deep rectangle without a window / TMA plan: the L1-lean k_search_deep2 (hjb_search2.cuh)
  const bool deep2 = g->D == 2 && has_deep && !wp && !use_tma && search2_ok(g) && !getenv("HJB_NO_SEARCH2");
  const int nds = (has_deep && !wp && !deep2) ? ring_strips(rect, tiles, dstrips) : 0;
  // with k_search_deep2 the boundary strips take its STRIP variant (HJB_NO_STRIP2: the general kernel)
  const bool strip2 = deep2 && !getenv("HJB_NO_STRIP2");
  if (!deep2 || g->uquad) g->gap_on = false;  // gap bookkeeping lives in the plain deep2 kernel only
  SkipRect s2strips[6];
  int ns2 = 0;
  if (strip2) {
    for (int k = 0; k < ngs; ++k) s2strips[ns2++] = gstrips[k];
    ngs = 0;
  }
#define SRCH1(DD, PP, DP, RR)                                                                                 \
  do {                                                                                                        \
    const LevelDev LL = shape_of(g->L0, RR);                                                                  \
    if (LL.nI > 0 && LL.nrows > 0) {                                                                          \
      LAUNCH(HJB_KC_SEARCH, 0, 0, 0,                                                                          \
             k_search<DD, PP, DP><<<dims(g, LL, (const void*)k_search<DD, PP, DP>, kSBX, tsm),                \
                                    dim3(kSBX, kSBY), tsm, g->st>>>(g->L0, CU, dt, U, Uprev, pol, F,          \
                                                                    g->partial + 2 * nblk, RR));             \
      nblk += g->nblk_last;                                                                                   \
    }                                                                                                         \
  } while (0)
#define SRCH(DD, PP)                                          \
  do {                                                        \
    for (int k = 0; k < ngs; ++k) SRCH1(DD, PP, false, gstrips[k]); \
    for (int k = 0; k < nds; ++k) SRCH1(DD, PP, true, dstrips[k]);  \
  } while (0)
  if (g->D == 2) {
    if (g->P == 1) SRCH(2, 1);
    else SRCH(2, 2);
  } else {
    if (g->P == 1) SRCH(3, 1);
    else if (g->P == 2) SRCH(3, 2);
    else SRCH(3, 3);
  }
#undef SRCH
#undef SRCH1
  CKL();
  g->prof.calls[HJB_KC_SEARCH] += 1;
  g->prof.nodes[HJB_KC_SEARCH] += nodes;  // algorithmic totals of the whole search (all launches)
  g->prof.bytes[HJB_KC_SEARCH] += nodes * bpn;
  g->prof.flops[HJB_KC_SEARCH] += nodes * fpn;
  if (wp) {  // the tiles' neighbourhoods of U staged in shared memory
#define WIN(DD, PP)                                                                                         \
  do {                                                                                                      \
    if (win_all)                                                                                            \
      LAUNCH(HJB_KC_SEARCH, 0, 0, 0,                                                                        \
             k_search_win<DD, PP, true><<<wp->grid, kWinNT, wp->smem, g->st>>>(                             \
                 g->L0, g->C0, dt, U, Uprev, pol, F, g->partial + 2 * nblk, wp->box, wp->geom));            \
    else                                                                                                    \
      LAUNCH(HJB_KC_SEARCH, 0, 0, 0,                                                                        \
             k_search_win<DD, PP, false><<<wp->grid, kWinNT, wp->smem, g->st>>>(                            \
                 g->L0, g->C0, dt, U, Uprev, pol, F, g->partial + 2 * nblk, wp->box, wp->geom));            \
  } while (0)
    if (g->D == 2) {
      if (g->P == 1) WIN(2, 1);
      else WIN(2, 2);
    } else {
      if (g->P == 1) WIN(3, 1);
      else if (g->P == 2) WIN(3, 2);
      else WIN(3, 3);
    }
#undef WIN
    CKL();
    nblk += wp->grid;
  }
  if (deep2) {
#if HJB_SEARCH2_PAIRS
    if (!g->upair) TRY(dalloc((void**)&g->upair, (size_t)g->N * sizeof(double2)));
    const int64_t ne = g->N;
    LAUNCH(HJB_KC_SEARCH, 0, 0, 0,
           k_make_pairs<<<(int)std::min<int64_t>((ne + 255) / 256, (int64_t)g->sms * 8), 256, 0, g->st>>>(U, g->upair, ne));
    CKL();
#endif
    // opt-in variants (measured at cfg4): 256-bit corner-copy taps (HJB_QUADS=1) and the
    // hoisted node-local bracket in shared memory (HJB_SEARCH3=1, needs the corner copy)
    g->search3 = getenv("HJB_SEARCH3") && (size_t)g->K * kS2T * sizeof(double) <= 200 * 1024;
    g->search2p = !g->search3 && !getenv("HJB_QUADS") && getenv("HJB_SEARCH2P");  // opt-in (slower)
    if (getenv("HJB_QUADS") || g->search3) {  // cell-corner copy of U for the 256-bit tap loads
      if (!g->uquad) TRY(dalloc((void**)&g->uquad, (size_t)g->N * sizeof(double4)));
      const int64_t ne = g->N;
      LAUNCH(HJB_KC_SEARCH, 0, 0, 0,
             k_make_quads<<<(int)std::min<int64_t>((ne + 255) / 256, (int64_t)g->sms * 8), 256, 0, g->st>>>(
                 U, g->uquad, (int)g->L0.n, ne));
      CKL();
    }
    TRY(launch_search2(g, dt, U, Uprev, pol, F, rect, &nblk));
    if (ns2 > 0) TRY(launch_search2(g, dt, U, Uprev, pol, F, rect, &nblk, s2strips, ns2));
  }
  if (use_tma) {  // deep tiles: windows staged in shared memory by TMA (partials after the others')
    if (g->P == 1)
      LAUNCH(HJB_KC_SEARCH, 0, 0, 0, k_search_tma<1><<<g->tma_grid, kWT, g->tma_smem, g->st>>>(
                                         g->L0, g->C0, dt, U, Uprev, pol, F, g->partial + 2 * nblk, g->tma, g->d_rng, umap));
    else
      LAUNCH(HJB_KC_SEARCH, 0, 0, 0, k_search_tma<2><<<g->tma_grid, kWT, g->tma_smem, g->st>>>(
                                         g->L0, g->C0, dt, U, Uprev, pol, F, g->partial + 2 * nblk, g->tma, g->d_rng, umap));
    CKL();
    nblk += g->tma_grid;
  }
  hjb_status err;
  double changed = 0.0;
  const double R = host_finalize(g, nblk, 0x1u, SC_NONE, &err, &changed);
  if (err != HJB_OK) return err;
  if (g->gap_on) {  // the scan kept the gaps: the next search of the step may skip
    unsigned long long ns = 0;
    CK(cudaMemcpy(&ns, g->d_gapred + 3, sizeof(ns), cudaMemcpyDeviceToHost));
    g->gap_skipped += (int64_t)(ns & 0xffffffffu);
    if (getenv("HJB_SKIP_DEBUG"))
      fprintf(stderr, "[hjb] search: %s, max|U| %.3e max|dU| %.3e G %.3e, skipped CTAs %lld (total so far %lld / %lld)\n",
              g->gap_first ? "full scan" : "gap-certified", g->gap_umax, g->gap_D, g->gap_G,
              (long long)(ns & 0xffffffffu), (long long)g->gap_skipped, (long long)g->gap_ctas);
    g->gap_valid = true;
    g->gap_on = false;
  } else {
    g->gap_valid = false;
  }
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
  const double* Ux;
  TRY(halo_input(g, U, &Ux));
  return policy_update_dev(g, dt, Ux, U_prev, policy, F, out);
}

// ---------------------------------------------------------------------------- apply
extern "C" hjb_status hjb_apply(hjb_grid_t g, double dt, const uint8_t* policy, const double* x, double* y) {
  if (!g || !policy || !x || !y) return fail(HJB_ERR_INVALID_ARG, "null argument");
  TRY(check_dt(g, dt));
  CK(cudaSetDevice(g->desc.device));
  if (x == y) return fail(HJB_ERR_INVALID_ARG, "x and y must not alias");
  CK(cudaMemcpyAsync(y, x, (size_t)g->N * sizeof(double), cudaMemcpyDeviceToDevice, g->st));
  const double* xx;
  TRY(halo_input(g, x, &xx));
  if (g->D == 2) launch_operator<2>(g, g->L0, g->C0, OP_APPLY, 0, dt, 0.0, policy, xx, nullptr, y, nullptr);
  else launch_operator<3>(g, g->L0, g->C0, OP_APPLY, 0, dt, 0.0, policy, xx, nullptr, y, nullptr);
  CKL();
  return HJB_OK;
}

// ---------------------------------------------------------------------------- multigrid
static int64_t level_halo(hjb_grid* g, const LevelDev& L) {
  // reach in this level's cells scales with kh, k2h relative to the fine level (same fields)
  const double rd = g->reach_diff * (L.kh / g->L0.kh), rb = g->reach_drift * (L.k2h / g->L0.k2h);
  return (int64_t)std::floor(std::max(rd, rb) * (1.0 + 1e-12)) + 1;
}

constexpr int64_t kGraphMaxNodes = 70000;  // 257^2 and below (measured: ~4 us of launch per kernel)

static hjb_status build_levels(hjb_grid* g, const hjb_mg_params* mp) {
  free_levels(g);
  g->mg_f32 = mp->precision == 1 && mp->coarse_op == 0;
  const int D = g->D;
  int64_t n = g->n;
  {
    Level l0;
    l0.L = g->L0;
    l0.elems = g->N;
    l0.C = g->C0;
    l0.H = g->lay.halo;
    l0.r0s = g->r0s;
    l0.r1s = g->r1s;
    g->levels.push_back(l0);
  }
  auto interior_count = [&](int64_t nn) { return ipow(nn - 2, D); };
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
    const Level& lf = g->levels.back();
    const int64_t nc = (n - 1) / 2 + 1;
    Level l;
    const double hc = (g->hi - g->lo) / (double)(nc - 1);
    // SL steps on the coarse level: 0 = the fine k (and drift step h); 1 = the scheme's own rule
    // k_l = sqrt(h_l) (measured: more Krylov iterations at cfg2 and cfg4)
    const double kc = (mp->coarse_k_mode == 1) ? std::sqrt(hc) : g->k;
    const double k2c = (mp->coarse_k_mode == 1) ? hc : g->h;
    l.L = full_level(D, nc, g->lo, g->hi, kc, k2c);
    l.replicated = (g->R > 1) && lf.replicated;
    if (g->R > 1 && !lf.replicated) {
      // coarse row J is owned by the rank owning fine row 2J: J in [ceil(r0/2), ceil(r1/2))
      std::vector<int64_t> c0(g->R), c1(g->R);
      for (int q = 0; q < g->R; ++q) {
        c0[q] = (lf.r0s[q] + 1) / 2;
        c1[q] = (lf.r1s[q] + 1) / 2;
      }
      const int64_t H = level_halo(g, l.L);
      bool thin = nc <= mp->gather_n;
      for (int q = 0; q < g->R; ++q) thin |= (c1[q] - c0[q]) < std::max<int64_t>(H, 1);
      if (thin) {
        l.replicated = true;
      } else {
        l.r0s = c0;
        l.r1s = c1;
        l.H = H;
        const int64_t r0 = c0[g->rank], r1 = c1[g->rank];
        l.L = make_level(D, nc, g->lo, g->hi, kc, k2c, r0, r1, std::max<int64_t>(0, r0 - H),
                         std::min<int64_t>(nc, r1 + H));
      }
    }
    l.elems = l.L.local_rows * l.L.row_elems;
    g->levels.push_back(l);
    n = nc;
  }
  if (interior_count(g->levels.back().L.n) > 160) {
    free_levels(g);
    return fail(HJB_ERR_UNSUPPORTED, "coarsest level too large for the dense solve (needs n = 2^l + 1)");
  }
  if (g->R > 1 && (g->levels.size() == 1 || !g->levels.back().replicated)) {
    free_levels(g);
    return fail(HJB_ERR_UNSUPPORTED, "multigrid on several ranks: the coarsest level must be gathered");
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
    if (i + 1 < g->levels.size()) {
      TRY(dalloc((void**)&l.dg, vb));
      CK(cudaMemsetAsync(l.dg, 0, vb, g->st));
    }
    if (i > 0) {
      TRY(dalloc((void**)&l.x, vb));
      TRY(dalloc((void**)&l.b, vb));
      TRY(dalloc((void**)&l.pol, (size_t)l.elems));
      CK(cudaMemsetAsync(l.x, 0, vb, g->st));
      CK(cudaMemsetAsync(l.b, 0, vb, g->st));
      CK(cudaMemsetAsync(l.pol, 0, (size_t)l.elems, g->st));
      if (nplanes > 0) {
        TRY(dalloc((void**)&l.fields, (size_t)nplanes * vb));
        CK(cudaMemsetAsync(l.fields, 0, (size_t)nplanes * vb, g->st));
      }
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
  if (g->mg_f32) {  // level 0's fp32 right-hand side and iterate (the caller's vectors are fp64)
    Level& l0 = g->levels[0];
    const size_t vb = (size_t)l0.elems * sizeof(float);
    TRY(dalloc((void**)&l0.x, vb));
    TRY(dalloc((void**)&l0.b, vb));
    CK(cudaMemsetAsync(l0.x, 0, vb, g->st));
    CK(cudaMemsetAsync(l0.b, 0, vb, g->st));
  }
  TRY(dalloc((void**)&lc.Ainv, (size_t)lc.L.n_own * lc.L.n_own * sizeof(double)));
  g->mgp = *mp;
  // graph tail: the first level (>= 1) owning <= kGraphMaxNodes interior nodes whose whole sub-cycle
  // runs without communication (one rank, or replicated levels) and is not revisited by a W-cycle
  g->graph_level = (size_t)-1;
  if (!getenv("HJB_NO_GRAPHS"))
    for (size_t l = 1; l < g->levels.size(); ++l) {
      const Level& lv = g->levels[l];
      const bool no_comm = g->R == 1 || lv.replicated;
      const bool revisited = mp->gamma > 1 && ipow(lv.L.n - 2, g->D) >= mp->gamma_min_nodes;
      if (no_comm && !revisited && lv.L.n_own <= kGraphMaxNodes) { g->graph_level = l; break; }
    }
  return HJB_OK;
}

// coarse rows of the first replicated level computed by each rank (from its last slab level)
static void transition_rows(hjb_grid* g, const Level& lf, std::vector<int64_t>& J0, std::vector<int64_t>& J1) {
  J0.resize(g->R);
  J1.resize(g->R);
  for (int q = 0; q < g->R; ++q) {
    J0[q] = (lf.r0s[q] + 1) / 2;
    J1[q] = (lf.r1s[q] + 1) / 2;
  }
}

template <int D>
static hjb_status inject_all(hjb_grid* g) {
  for (size_t i = 1; i < g->levels.size(); ++i) {
    Level& lf = g->levels[i - 1];
    Level& lc = g->levels[i];
    const uint8_t* pf = (i == 1) ? g->mg_pol0 : lf.pol;
    const int nb = nblocks1d(lc.elems);
    // fine rows whose policy / field values are valid on this rank
    const bool fslab = g->R > 1 && !lf.replicated;
    const int64_t fr_lo = fslab ? lf.r0s[g->rank] : 0;
    const int64_t fr_hi = fslab ? lf.r1s[g->rank] : lf.L.n;
    LAUNCH(HJB_KC_TRANSFER, lc.elems, 2.0 * lc.elems, 0,
           k_inject_u8<D><<<nb, 256, 0, g->st>>>(lf.L, lc.L, pf, lc.pol, fr_lo, fr_hi));
    struct FP { const double* f; double* c; int np; };
    const FP fps[] = {{lf.C.sigma_scale, (double*)lc.C.sigma_scale, g->P},
                      {lf.C.sigma_node, (double*)lc.C.sigma_node, g->P * D},
                      {lf.C.b_scale, (double*)lc.C.b_scale, 1},
                      {lf.C.b_node, (double*)lc.C.b_node, D},
                      {lf.C.c_node, (double*)lc.C.c_node, 1}};
    for (const FP& f : fps)
      if (f.f)
        LAUNCH(HJB_KC_TRANSFER, lc.elems, 16.0 * f.np * lc.elems, 0,
               k_inject_f64<D><<<nb, 256, 0, g->st>>>(lf.L, lc.L, f.f, lf.C.ld, f.c, lc.C.ld, f.np, fr_lo, fr_hi));
    CKL();
    if (lc.replicated && fslab) {  // gather level: every rank gets the full coarse data
      std::vector<int64_t> J0, J1;
      transition_rows(g, lf, J0, J1);
      const int64_t re = lc.L.row_elems;
      TRY(gather_rows(g, lc.pol, 1, re, J0, J1));
      for (const FP& f : fps)
        if (f.f)
          for (int k = 0; k < f.np; ++k) TRY(gather_rows(g, f.c + (size_t)k * lc.C.ld, 8, re, J0, J1));
    }
  }
  Level& lc = g->levels.back();
  const int64_t Nc = lc.L.n_own;
  const uint8_t* pc = (g->levels.size() == 1) ? g->mg_pol0 : lc.pol;
  CK(cudaMemsetAsync(lc.Ainv, 0, (size_t)Nc * Nc * sizeof(double), g->st));
  LAUNCH(HJB_KC_COARSE, Nc, 8.0 * Nc * Nc, 0,
         k_coarse_assemble<D><<<(int)((Nc + 127) / 128), 128, 0, g->st>>>(lc.L, lc.C, g->mg_dt, pc, lc.Ainv));
  CKL();
  const size_t smem = (size_t)Nc * Nc * sizeof(double);
  if (smem > 48 * 1024) CK(allow_smem((const void*)k_coarse_invert));
  LAUNCH(HJB_KC_COARSE, Nc, 16.0 * Nc * Nc, 2.0 * Nc * Nc * Nc, k_coarse_invert<<<1, 1024, smem, g->st>>>(lc.Ainv, (int)Nc));
  CKL();
  return HJB_OK;
}

// Galerkin coarse operators A_{l+1} = R A_l P for every coarse level (2D, one rank), their diagonals,
// and the coarsest level's dense inverse from its Galerkin rows (hjb_galerkin.cuh; NEXT-4)
static hjb_status galerkin_setup(hjb_grid* g, double dt, const uint8_t* policy) {
  if (g->D != 2 || g->R != 1)
    return fail(HJB_ERR_UNSUPPORTED, "Galerkin coarse operators: 2D on one rank only");
  if (!g->d_flag) TRY(dalloc((void**)&g->d_flag, sizeof(int)));
  CK(cudaMemsetAsync(g->d_flag, 0, sizeof(int), g->st));
  const size_t eb0 = (size_t)g->levels[0].elems;
  if (!g->gb_col) {
    TRY(dalloc((void**)&g->gb_col, (size_t)kGalWB * eb0 * sizeof(int)));
    TRY(dalloc((void**)&g->gb_val, (size_t)kGalWB * eb0 * sizeof(double)));
  }
  for (size_t l = 1; l < g->levels.size(); ++l) {
    Level& lv = g->levels[l];
    if (!lv.gcol) {
      TRY(dalloc((void**)&lv.gcol, (size_t)kGalW * lv.elems * sizeof(int)));
      TRY(dalloc((void**)&lv.gval, (size_t)kGalW * lv.elems * sizeof(double)));
      CK(cudaMemsetAsync(lv.gcol, 0xff, (size_t)kGalW * lv.elems * sizeof(int), g->st));
    }
  }
  for (size_t l = 0; l + 1 < g->levels.size(); ++l) {
    Level& lf = g->levels[l];
    Level& lc = g->levels[l + 1];
    const int64_t nf = (int64_t)lf.L.nI * lf.L.nrows, ncr = (int64_t)lc.L.nI * lc.L.nrows;
    const int bf = (int)std::min<int64_t>((nf + 127) / 128, (int64_t)g->sms * 16);
    const int bc = (int)std::min<int64_t>((ncr + 127) / 128, (int64_t)g->sms * 16);
    CK(cudaMemsetAsync(g->gb_col, 0xff, (size_t)kGalWB * lf.elems * sizeof(int), g->st));
    if (l == 0) {
      if (g->P == 1)
        LAUNCH(HJB_KC_COARSE, nf, 0, 0, k_gal_b_fine<1><<<bf, 128, 0, g->st>>>(lf.L, g->C0, dt, policy, lc.L.n, g->gb_col, g->gb_val, g->d_flag));
      else
        LAUNCH(HJB_KC_COARSE, nf, 0, 0, k_gal_b_fine<2><<<bf, 128, 0, g->st>>>(lf.L, g->C0, dt, policy, lc.L.n, g->gb_col, g->gb_val, g->d_flag));
    } else {
      LAUNCH(HJB_KC_COARSE, nf, 0, 0, k_gal_b_ell<<<bf, 128, 0, g->st>>>(lf.L, lf.gcol, lf.gval, lc.L.n, g->gb_col, g->gb_val, g->d_flag));
    }
    LAUNCH(HJB_KC_COARSE, ncr, 0, 0, k_gal_rb<<<bc, 128, 0, g->st>>>(lf.L, lc.L, g->gb_col, g->gb_val, lc.gcol, lc.gval, g->d_flag));
    CKL();
    if (l + 2 < g->levels.size())
      LAUNCH(HJB_KC_COARSE, ncr, 0, 0, k_gal_diag<<<bc, 128, 0, g->st>>>(lc.L, lc.gcol, lc.gval, lc.dg));
    CKL();
  }
  Level& lc = g->levels.back();
  const int64_t Nc = lc.L.n_own;
  if (g->levels.size() > 1) {
    CK(cudaMemsetAsync(lc.Ainv, 0, (size_t)Nc * Nc * sizeof(double), g->st));
    LAUNCH(HJB_KC_COARSE, Nc, 0, 0, k_gal_dense<<<(int)((Nc + 127) / 128), 128, 0, g->st>>>(lc.L, lc.gcol, lc.gval, lc.Ainv));
    const size_t smem = (size_t)Nc * Nc * sizeof(double);
    if (smem > 48 * 1024) CK(allow_smem((const void*)k_coarse_invert));
    LAUNCH(HJB_KC_COARSE, Nc, 16.0 * Nc * Nc, 2.0 * Nc * Nc * Nc, k_coarse_invert<<<1, 1024, smem, g->st>>>(lc.Ainv, (int)Nc));
    CKL();
  }
  int flag = 0;
  CK(cudaMemcpyAsync(&flag, g->d_flag, sizeof(int), cudaMemcpyDeviceToHost, g->st));
  CK(cudaStreamSynchronize(g->st));
  if (flag) return fail(HJB_ERR_UNSUPPORTED, "Galerkin coarse operator row wider than the ELL width (96)");
  return HJB_OK;
}

extern "C" hjb_status hjb_mg_setup(hjb_grid_t g, double dt, const uint8_t* policy, const hjb_mg_params* mp) {
  if (!g || !policy) return fail(HJB_ERR_INVALID_ARG, "null argument");
  TRY(check_dt(g, dt));
  CK(cudaSetDevice(g->desc.device));
  hjb_mg_params def;
  hjb_mg_params_default(g->D, &def);
  hjb_mg_params q = mp ? *mp : def;
  if (const char* e = getenv("HJB_MG_PRECISION")) q.precision = atoi(e);  // A/B knob
  const hjb_mg_params* p = &q;
  if (p->precision < 0 || p->precision > 1) return fail(HJB_ERR_INVALID_ARG, "bad multigrid precision");
  if (p->nu_pre < 1 || p->nu_post < 0 || !(p->omega > 0.0) || p->omega > 1.0 || p->max_levels < 1 ||
      p->gamma < 1 || p->gamma > 3 || p->gamma_min_nodes < 0 || p->coarse_op < 0 || p->coarse_op > 1)
    return fail(HJB_ERR_INVALID_ARG, "bad multigrid parameters");
  const bool rebuild = g->levels.empty() || std::memcmp(&g->mgp, p, sizeof(hjb_mg_params)) != 0 ||
                       g->levels[0].C.ld != g->C0.ld;
  if (rebuild) TRY(build_levels(g, p));
  g->levels[0].C = g->C0;  // refresh field pointers of level 0 (set_coeffs may have changed them)
  g->levels[0].L.pf_rows = g->L0.pf_rows;
  for (size_t i = 1; i < g->levels.size(); ++i) g->levels[i].L.pf_rows = prefetch_rows(g, g->levels[i].L);
  g->mg_pol0 = policy;
  g->mg_dt = dt;
  if (dt != g->graph_dt || getenv("HJB_NU_COARSE")) {  // captured graphs hold dt as a kernel parameter
    for (auto& sg : g->graphs) cudaGraphExecDestroy(sg.exec);
    g->graphs.clear();
    g->graph_dt = dt;
  }
  if (g->D == 2) TRY(inject_all<2>(g));
  else TRY(inject_all<3>(g));
  g->galerkin = p->coarse_op == 1;
  if (g->galerkin) TRY(galerkin_setup(g, dt, policy));
  // the diagonal of every smoothed level's operator (the smoother reads it instead of recomputing
  // the self weights; HJB_NO_DIAG=1 recomputes them in every sweep -- bit-identical either way)
  g->use_dg = !getenv("HJB_NO_DIAG");
  g->mg_gamma = p->gamma;
  g->gamma_min = p->gamma_min_nodes;
  g->nu_coarse = getenv("HJB_NU_COARSE") ? std::max(0, atoi(getenv("HJB_NU_COARSE"))) : 0;
  if (g->mg_gamma > 1)
    for (size_t l = 1; l + 1 < g->levels.size(); ++l) {
      Level& lv = g->levels[l];
      if (ipow(lv.L.n - 2, g->D) < g->gamma_min) continue;  // global count: same on every rank
      const size_t vb = (size_t)lv.elems * sizeof(double);
      if (!lv.r2) {
        TRY(dalloc((void**)&lv.r2, vb));
        TRY(dalloc((void**)&lv.e2, vb));
        CK(cudaMemsetAsync(lv.r2, 0, vb, g->st));
        CK(cudaMemsetAsync(lv.e2, 0, vb, g->st));
      }
    }
  if (g->galerkin) g->use_dg = true;  // the Galerkin smoother reads the stored diagonal
  if (g->use_dg)
    for (size_t l = 0; l + 1 < g->levels.size(); ++l) {
      if (g->galerkin && l >= 1) continue;  // from the Galerkin rows (galerkin_setup)
      Level& lv = g->levels[l];
      const uint8_t* pol = (l == 0) ? g->mg_pol0 : lv.pol;
      if (g->mg_f32) {
        float* dg = reinterpret_cast<float*>(lv.dg);
        if (g->D == 2) launch_operator<2, float>(g, lv.L, lv.C, OP_DIAG, 0, dt, 0.0, pol, nullptr, nullptr, dg, nullptr, l == 0);
        else launch_operator<3, float>(g, lv.L, lv.C, OP_DIAG, 0, dt, 0.0, pol, nullptr, nullptr, dg, nullptr, l == 0);
      } else if (g->D == 2) {
        launch_operator<2>(g, lv.L, lv.C, OP_DIAG, 0, dt, 0.0, pol, nullptr, nullptr, lv.dg, nullptr, l == 0);
      } else {
        launch_operator<3>(g, lv.L, lv.C, OP_DIAG, 0, dt, 0.0, pol, nullptr, nullptr, lv.dg, nullptr, l == 0);
      }
    }
  CKL();
  g->mg_ready = true;
  return HJB_OK;
}

// Jacobi damping of level l: Galerkin coarse operators are not M-matrices (positive off-diagonals,
// rows not diagonally dominant: measured at cfg2 513^2), where omega = 1 diverges (stationary
// V(2,2) rho 1.6) and 0.6 contracts in V- and W-cycles (0.092 / 0.028; 0.8 diverges in the W-cycle):
// min(omega, 0.6) there (reading xxix)
static double level_omega(const hjb_grid* g, size_t l) {
  return (g->galerkin && l >= 1) ? std::min(g->mgp.omega, kGalOmega) : g->mgp.omega;
}

// one residual (OP_RESID: y = b - A x) or damped-Jacobi sweep (OP_JACOBI / OP_JACOBI_D) on level l:
// the matrix-free rediscretised operator, or on Galerkin levels (l >= 1) the stored R A P rows
template <typename V>
static V* lvec(double* p) { return reinterpret_cast<V*>(p); }

template <int D, typename V = double>
static void level_sweep(hjb_grid* g, size_t l, int mode, const V* x, const V* b, V* y) {
  Level& lv = g->levels[l];
  const uint8_t* pol = (l == 0) ? g->mg_pol0 : lv.pol;
  const double dt = g->mg_dt, om = level_omega(g, l);
  if constexpr (std::is_same<V, double>::value) if (g->galerkin && l >= 1) {
    halo_end(g);
    const int64_t nn = (int64_t)lv.L.nI * lv.L.nrows;
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>((nn + 127) / 128, (int64_t)g->sms * 16));
    const double bytes = (8.0 * 3 + 12.0 * kGalW) * nn;
    if (mode == OP_RESID)
      LAUNCH(HJB_KC_MG_COARSE, nn, bytes, 2.0 * kGalW * nn,
             k_gal_sweep<false><<<nb, 128, 0, g->st>>>(lv.L, lv.gcol, lv.gval, x, b, lv.dg, 0.0, y));
    else
      LAUNCH(HJB_KC_MG_COARSE, nn, bytes + 8.0 * nn, 2.0 * kGalW * nn,
             k_gal_sweep<true><<<nb, 128, 0, g->st>>>(lv.L, lv.gcol, lv.gval, x, b, lv.dg, om, y));
    return;
  }
  launch_operator<D, V>(g, lv.L, lv.C, mode, 0, dt, mode == OP_RESID ? 0.0 : om, pol, x, b, y,
                        mode == OP_JACOBI_D ? lvec<V>(lv.dg) : nullptr, l == 0);
}

// V(nu_pre, nu_post) from x = 0 on level l: out = M_l^{-1} b
template <int D, typename V = double>
static hjb_status vcycle(hjb_grid* g, size_t l, const V* b, V* out) {
  // the whole cycle as one graph (one rank, no per-kernel timing), else its launch-bound tail
  const bool whole = l == 0 && g->R == 1 && !g->prof_timing && g->graph_level != (size_t)-1;
  if ((whole || l == g->graph_level) && !g->capturing) {
    hjb_grid::SubGraph* sg = nullptr;
    for (auto& x : g->graphs)
      if (x.level == l && x.b == b && x.out == out && x.pol0 == g->mg_pol0) sg = &x;
    if (!sg) {  // capture the sub-cycle once on the private stream (kernels recorded, not run)
      if (!g->cap_st) CK(cudaStreamCreateWithFlags(&g->cap_st, cudaStreamNonBlocking));
      cudaStream_t keep = g->st;
      g->cap_launches = 0;
      g->st = g->cap_st;
      g->capturing = true;
      cudaGraph_t graph = nullptr;
      cudaError_t e = cudaStreamBeginCapture(g->st, cudaStreamCaptureModeThreadLocal);
      hjb_status st = (e == cudaSuccess) ? vcycle<D, V>(g, l, b, out) : HJB_ERR_CUDA;
      cudaError_t e2 = cudaStreamEndCapture(g->st, &graph);
      g->capturing = false;
      g->st = keep;
      if (e != cudaSuccess || e2 != cudaSuccess || st != HJB_OK) {
        if (graph) cudaGraphDestroy(graph);
        return st != HJB_OK ? st : fail(HJB_ERR_CUDA, "multigrid graph capture failed");
      }
      cudaGraphExec_t exec = nullptr;
      e = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      if (e != cudaSuccess) return fail(HJB_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
      const int64_t nl = g->cap_launches;
      g->graphs.push_back(hjb_grid::SubGraph{l, b, out, g->mg_pol0, exec, nl});
      sg = &g->graphs.back();
    }
    CK(cudaGraphLaunch(sg->exec, g->st));
    g->prof.total_launches += sg->launches;
    g->prof.launches[HJB_KC_MG_COARSE] += sg->launches;
    g->prof.graph_launches += 1;
    g->prof.graph_kernels += sg->launches;
    return HJB_OK;
  }
  Level& lv = g->levels[l];
  const uint8_t* pol = (l == 0) ? g->mg_pol0 : lv.pol;
  const LevelDev& L = lv.L;
  cudaStream_t st = g->st;
  const bool fine = (l == 0);
  if (l + 1 == g->levels.size()) {
    const int Nc = (int)L.n_own;
    LAUNCH(HJB_KC_COARSE, Nc, 8.0 * Nc * Nc + 2.0 * sizeof(V) * Nc, 2.0 * Nc * Nc,
           k_coarse_solve<D, V><<<1, 256, Nc * sizeof(double), st>>>(L, lv.Ainv, b, out));
    CKL();
    return HJB_OK;
  }
  const double dt = g->mg_dt, om = level_omega(g, l);
  const int npre = (l > 0 && g->nu_coarse > 0) ? g->nu_coarse : g->mgp.nu_pre;
  const int npost = (l > 0 && g->nu_coarse > 0) ? g->nu_coarse : g->mgp.nu_post;
  const double vs = (double)sizeof(V);
  V* bufs[2] = {out, lvec<V>(lv.tmp)};
  V* res = lvec<V>(lv.res);
  int cur = ((npre - 1 + npost) % 2 == 0) ? 0 : 1;  // so the last sweep lands in `out`
  const int jmode = g->use_dg ? OP_JACOBI_D : OP_JACOBI;
  if (g->use_dg) {
    const double nn = (double)L.n_own;
    if (!g->capturing && (!g->prof_timing || nn >= kTimeMinNodes)) g->prof.calls[fine ? HJB_KC_SMOOTH : HJB_KC_MG_COARSE] += 1;
    LAUNCH(fine ? HJB_KC_SMOOTH : HJB_KC_MG_COARSE, nn, 3.0 * vs * nn, 2.0 * nn,
           k_jacobi0_diag<D, V><<<dims(g, L, (const void*)k_jacobi0_diag<D, V>), dim3(kBX, kBY), 0, st>>>(
               L, om, b, lvec<V>(lv.dg), bufs[cur]));
    CKL();
  } else {
    launch_operator<D, V>(g, L, lv.C, OP_JACOBI0, 0, dt, om, pol, nullptr, b, bufs[cur], nullptr, fine);
  }
  for (int k = 1; k < npre; ++k) {
    TRY(halo_begin(g, lv, bufs[cur], lv.H, sizeof(V)));
    level_sweep<D, V>(g, l, jmode, bufs[cur], b, bufs[1 - cur]);
    cur = 1 - cur;
  }
  TRY(halo_begin(g, lv, bufs[cur], lv.H, sizeof(V)));
  level_sweep<D, V>(g, l, OP_RESID, bufs[cur], b, res);
  Level& lc = g->levels[l + 1];
  V* const cb = lvec<V>(lc.b);
  V* const cx = lvec<V>(lc.x);
  TRY(halo_exchange(g, lv, res, 1, sizeof(V)));
  if (lc.replicated && !lv.replicated) {
    // gather level: restrict my coarse rows into the full coarse array, then all-gather them
    std::vector<int64_t> J0, J1;
    transition_rows(g, lv, J0, J1);
    LevelDev view = lc.L;
    view.row_first = J0[g->rank];
    view.nrows = (int)((J1[g->rank] - J0[g->rank]) * ipow(lc.L.n - 2, D - 2));
    view.n_own = (int64_t)view.nrows * view.nI;
    if (view.nrows > 0)
      LAUNCH(HJB_KC_TRANSFER, L.n_own, vs * (L.n_own + view.n_own), 18.0 * view.n_own,
             k_restrict<D, V, V><<<dims(g, view, (const void*)k_restrict<D, V, V>), dim3(kBX, kBY), 0, st>>>(L, view, res, cb));
    CKL();
    TRY(gather_rows(g, cb, sizeof(V), lc.L.row_elems, J0, J1));
  } else {
    LAUNCH(HJB_KC_TRANSFER, L.n_own, vs * (L.n_own + lc.L.n_own), 18.0 * lc.L.n_own,
           k_restrict<D, V, V><<<dims(g, lc.L, (const void*)k_restrict<D, V, V>), dim3(kBX, kBY), 0, st>>>(L, lc.L, res, cb));
    CKL();
  }
  TRY((vcycle<D, V>(g, l + 1, cb, cx)));
  // revisit decided on the level's GLOBAL interior count, so every rank takes the same branch
  const int gamma = (ipow(lc.L.n - 2, D) >= g->gamma_min) ? g->mg_gamma : 1;
  for (int k = 1; k < gamma && l + 2 < g->levels.size(); ++k) {  // W-cycle: revisit the coarse level
    const uint8_t* pc = lc.pol;
    TRY(halo_begin(g, lc, cx, lc.H, sizeof(V)));
    (void)pc;
    level_sweep<D, V>(g, l + 1, OP_RESID, cx, cb, lvec<V>(lc.r2));
    TRY((vcycle<D, V>(g, l + 1, lvec<V>(lc.r2), lvec<V>(lc.e2))));
    const double nc = (double)lc.L.n_own;
    LAUNCH(HJB_KC_VECTOR, nc, 3.0 * vs * nc, nc,
           k_add_interior<D, V><<<dims(g, lc.L, (const void*)k_add_interior<D, V>), dim3(kBX, kBY), 0, st>>>(lc.L, lvec<V>(lc.e2), cx));
    CKL();
  }
  TRY(halo_exchange(g, lc, cx, 1, sizeof(V)));
  LAUNCH(HJB_KC_TRANSFER, L.n_own, 2.0 * vs * L.n_own + vs * lc.L.n_own, 4.0 * L.n_own,
         k_prolong_add<D, V, V><<<dims(g, L, (const void*)k_prolong_add<D, V, V>), dim3(kBX, kBY), 0, st>>>(L, lc.L, cx, bufs[cur]));
  for (int k = 0; k < npost; ++k) {
    TRY(halo_begin(g, lv, bufs[cur], lv.H, sizeof(V)));
    level_sweep<D, V>(g, l, jmode, bufs[cur], b, bufs[1 - cur]);
    cur = 1 - cur;
  }
  CKL();
  if (bufs[cur] != out) return fail(HJB_ERR_STATE, "internal: V-cycle buffer parity");
  return HJB_OK;
}

// x = M^{-1} b with the fp32 cycle: b rounded to fp32 on entry, the result widened on exit
template <int D>
static hjb_status precond_f32(hjb_grid* g, const double* b, double* x) {
  Level& l0 = g->levels[0];
  float* b32 = reinterpret_cast<float*>(l0.b);
  float* x32 = reinterpret_cast<float*>(l0.x);
  const double nn = (double)g->L0.n_own;
  LAUNCH(HJB_KC_VECTOR, nn, 12.0 * nn, 0,
         k_copy_interior<D, double, float><<<dims(g, g->L0, (const void*)k_copy_interior<D, double, float>),
                                             dim3(kBX, kBY), 0, g->st>>>(g->L0, b, b32));
  TRY((vcycle<D, float>(g, 0, b32, x32)));
  LAUNCH(HJB_KC_VECTOR, nn, 12.0 * nn, 0,
         k_copy_interior<D, float, double><<<dims(g, g->L0, (const void*)k_copy_interior<D, float, double>),
                                             dim3(kBX, kBY), 0, g->st>>>(g->L0, x32, x));
  CKL();
  return HJB_OK;
}

static hjb_status precond(hjb_grid* g, bool use_mg, const double* b, double* x) {
  if (!use_mg) {
    const double nn = (double)g->L0.n_own;
    if (g->D == 2)
      LAUNCH(HJB_KC_VECTOR, nn, 16.0 * nn, 0,
             k_copy_interior<2><<<dims(g, g->L0, (const void*)k_copy_interior<2>), dim3(kBX, kBY), 0, g->st>>>(g->L0, b, x));
    else
      LAUNCH(HJB_KC_VECTOR, nn, 16.0 * nn, 0,
             k_copy_interior<3><<<dims(g, g->L0, (const void*)k_copy_interior<3>), dim3(kBX, kBY), 0, g->st>>>(g->L0, b, x));
    CKL();
    return HJB_OK;
  }
  if (g->mg_f32) return g->D == 2 ? precond_f32<2>(g, b, x) : precond_f32<3>(g, b, x);
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
         k_norms<D><<<dims(g, g->L0, (const void*)k_norms<D>), dim3(kBX, kBY), 0, g->st>>>(g->L0, v, g->partial));
  const int nb = g->nblk_last;
  CKL();
  hjb_status err;
  *n2 = std::sqrt(host_finalize(g, nb, 0x2u, SC_NONE, &err, ninf));
  return err;
}

// eta > 0: inexact policy evaluation, stop at ||r||_2 <= max(rtol ||F||_2, eta ||r_0||_2).
// x's halo rows are exchanged here (x is the caller's in/out array).
template <int D>
static hjb_status bicgstab(hjb_grid* g, double dt, const uint8_t* pol, const double* F, double* x,
                           const hjb_solve_params* sp, hjb_solve_stats* out, double eta = 0.0) {
  const LevelDev& L = g->L0;
  const CoefDev& C = g->C0;
  const CoefDev CUx = coef_u(g);  // residuals of x = U (exact-psi mode: psi at truncated endpoints)
  cudaStream_t st = g->st;
  Level tmpl;
  const Level& lv0 = fine_level(g, tmpl);
  const int64_t H = g->lay.halo;
  const bool mg = sp->use_mg != 0;
  if (mg && (!g->mg_ready || g->mg_pol0 != pol || g->mg_dt != dt))
    return fail(HJB_ERR_STATE, "hjb_mg_setup must be called with the same policy and dt before solving");
  double bn2, bninf;
  TRY(norms_dev<D>(g, F, &bn2, &bninf));
  double tol = sp->krylov_rtol * bn2;
  // secondary max-norm stop of an exact evaluation (reading xvii): ||r||_inf <= rtol_inf ||F||_inf
  const double tol_inf = (eta > 0.0 || !(sp->krylov_rtol_inf > 0.0)) ? INFINITY : sp->krylov_rtol_inf * bninf;
  int it = 0;
  hjb_status err = HJB_OK;
  double rr = 0.0;
  bool converged = false, broke = false, early = false;
  double tol_iter = tol;  // target of the recursive residual (tightened if the max-norm stop fails)
  for (int restart = 0; restart < 6 && !converged; ++restart) {
    // r = F - A x ; rhat = r ; p = r
    TRY(halo_begin(g, lv0, x, H));
    launch_operator<D>(g, L, CUx, OP_RESID, 0, dt, 0.0, pol, x, F, g->r, nullptr);
    LAUNCH(HJB_KC_VECTOR, L.n_own, 24.0 * L.n_own, 2.0 * L.n_own,
           k_bicg_init<D><<<dims(g, L, (const void*)k_bicg_init<D>), dim3(kBX, kBY), 0, st>>>(L, g->r, g->rhat, g->p, g->partial));
    CKL();
    rr = host_finalize(g, g->nblk_last, 0u, SC_INIT, &err);
    if (err != HJB_OK) return err;
    if (!std::isfinite(rr)) return fail(HJB_ERR_NONFINITE, "non-finite residual");
    if (restart == 0 && eta > 0.0) tol = tol_iter = std::max(tol, eta * std::sqrt(rr));
    if (std::sqrt(rr) <= tol && tol_inf == INFINITY) { converged = early = true; break; }
    int inner = 0;
    broke = false;
    while (it < sp->krylov_maxit && std::sqrt(rr) > tol_iter) {
      if (inner > 0)
        LAUNCH(HJB_KC_VECTOR, L.n_own, 32.0 * L.n_own, 4.0 * L.n_own,
               k_bicg_p<D><<<dims(g, L, (const void*)k_bicg_p<D>), dim3(kBX, kBY), 0, st>>>(L, g->S, g->r, g->p, g->v));
      TRY(precond(g, mg, g->p, g->phat));
      TRY(halo_begin(g, lv0, g->phat, H));
      launch_operator<D>(g, L, C, OP_APPLY, 1, dt, 0.0, pol, g->phat, nullptr, g->v, g->rhat);
      TRY(reduce_dev(g, g->nblk_last, 0u, SC_AFTER_V));
      LAUNCH(HJB_KC_VECTOR, L.n_own, 24.0 * L.n_own, 4.0 * L.n_own,
             k_bicg_s<D><<<dims(g, L, (const void*)k_bicg_s<D>), dim3(kBX, kBY), 0, st>>>(L, g->S, g->r, g->v, g->s, g->partial));
      TRY(precond(g, mg, g->s, g->shat));
      TRY(halo_begin(g, lv0, g->shat, H));
      launch_operator<D>(g, L, C, OP_APPLY, 2, dt, 0.0, pol, g->shat, nullptr, g->t, g->s);
      TRY(reduce_dev(g, g->nblk_last, 0u, SC_AFTER_T));
      LAUNCH(HJB_KC_VECTOR, L.n_own, 64.0 * L.n_own, 10.0 * L.n_own,
             k_bicg_x<D><<<dims(g, L, (const void*)k_bicg_x<D>), dim3(kBX, kBY), 0, st>>>(L, g->S, x, g->phat, g->shat, g->s,
                                                                               g->t, g->r, g->rhat, g->partial));
      TRY(reduce_dev(g, g->nblk_last, 0u, SC_AFTER_R));
      CK(cudaMemcpyAsync(g->hS, g->S, sizeof(KScal), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      ++it;
      ++inner;
      rr = g->hS->rr;
      // a breakdown keeps every coefficient finite (alpha = 0 / omega = 0 steps, scal_update), so x
      // is valid here: restart from it
      if (g->hS->breakdown) { broke = true; break; }
      if (!std::isfinite(rr)) return fail(HJB_ERR_NONFINITE, "non-finite residual in BiCGSTAB");
    }
    // true residual check (recursive residual drifts, SURVEY hard part 5) in both norms
    TRY(halo_begin(g, lv0, x, H));
    launch_operator<D>(g, L, CUx, OP_RESID, 0, dt, 0.0, pol, x, F, g->r, nullptr);
    double tr2, trinf;
    TRY(norms_dev<D>(g, g->r, &tr2, &trinf));
    if (!std::isfinite(tr2)) return fail(HJB_ERR_NONFINITE, "non-finite true residual");
    if (out) {
      out->iters = it;
      out->rres = bn2 > 0 ? tr2 / bn2 : tr2;
      out->rres_inf = bninf > 0 ? trinf / bninf : trinf;
    }
    if (tr2 <= tol && trinf <= tol_inf) { converged = true; break; }
    // tighten the 2-norm target in proportion to the max-norm excess (or the drift of the recursion)
    if (trinf > tol_inf) tol_iter = std::min(tol_iter, 0.5 * tr2 * (tol_inf / trinf));
    else tol_iter = std::min(tol_iter, 0.5 * tol * (tol / std::max(tr2, tol)));
    if (it >= sp->krylov_maxit) break;
  }
  if (out && early) {
    out->iters = 0;
    out->rres = bn2 > 0 ? std::sqrt(rr) / bn2 : 0.0;
    out->rres_inf = 0.0;
  }
  if (!converged && broke) return fail(HJB_ERR_BREAKDOWN, "BiCGSTAB breakdown in its last restart");
  if (!converged) return fail(HJB_ERR_NOT_CONVERGED, "BiCGSTAB did not reach the tolerance");
  return HJB_OK;
}

// ---------------------------------------------------------------------------- aggregation AMG
// (PAPER.md:171-176, 1162-1164): setup per policy, K-cycle preconditioned
// flexible GCR on the correction equation A e = F - A U (compact interior vectors)
constexpr int kAgRestart = 10;
constexpr double kAgOmega = 0.67;   // Jacobi damping of the K-cycle smoother (the paper uses GS)

// the levels of the current hierarchy go back to the pool (their buffers are reused)
static void agmg_release_levels(hjb_grid* g) {
  for (auto& l : g->ag) {
    l.Ainv = nullptr;
    g->ag_pool.push_back(l);
  }
  g->ag.clear();
  g->ag_ready = false;
}
static void agmg_free_levels(hjb_grid* g) {
  agmg_release_levels(g);
  for (auto& l : g->ag_pool) {
    cudaFree(l.col); cudaFree(l.val); cudaFree(l.dg); cudaFree(l.agg); cudaFree(l.mem);
    cudaFree(l.x); cudaFree(l.b); cudaFree(l.r); cudaFree(l.t);
    for (int k = 0; k < 2; ++k) { cudaFree(l.z[k]); cudaFree(l.az[k]); }
  }
  g->ag_pool.clear();
}
static void agmg_free(hjb_grid* g) {
  agmg_free_levels(g);
  cudaFree(g->ag_dense);
  cudaFree(g->ag_sc);
  g->ag_sc = nullptr;
  cudaFree(g->ag_agg1c);
  cudaFree(g->ag_mem1c);
  g->ag_dense = nullptr;
  g->ag_agg1c = g->ag_mem1c = nullptr;
  for (auto& p : g->ag_i) { cudaFree(p); p = nullptr; }
  cudaFree(g->ag_cub);
  g->ag_cub = nullptr;
  for (int k = 0; k < 16; ++k) { cudaFree(g->ag_Z[k]); cudaFree(g->ag_AZ[k]); g->ag_Z[k] = g->ag_AZ[k] = nullptr; }
}

static int ag_blocks(int64_t n, int bs = 256) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + bs - 1) / bs, (int64_t)148 * 32));
}

static hjb_status ag_alloc_level(hjb_grid* g, hjb_grid::AgLevel& l, int64_t N) {
  // the smallest pooled level that fits
  int best = -1;
  for (int i = 0; i < (int)g->ag_pool.size(); ++i)
    if (g->ag_pool[i].cap >= N && (best < 0 || g->ag_pool[i].cap < g->ag_pool[best].cap)) best = i;
  if (best >= 0) {
    l = g->ag_pool[best];
    g->ag_pool.erase(g->ag_pool.begin() + best);
    l.N = N;
    l.Ainv = nullptr;
    CK(cudaMemsetAsync(l.col, 0xff, (size_t)kAgW * N * sizeof(int), g->st));
    return HJB_OK;
  }
  l = hjb_grid::AgLevel{};
  l.N = N;
  l.cap = N;
  TRY(dalloc((void**)&l.col, (size_t)kAgW * N * sizeof(int)));
  TRY(dalloc((void**)&l.val, (size_t)kAgW * N * sizeof(double)));
  TRY(dalloc((void**)&l.dg, (size_t)N * sizeof(double)));
  double** vs[] = {&l.x, &l.b, &l.r, &l.t, &l.z[0], &l.z[1], &l.az[0], &l.az[1]};
  for (double** v : vs) TRY(dalloc((void**)v, (size_t)N * sizeof(double)));
  CK(cudaMemsetAsync(l.col, 0xff, (size_t)kAgW * N * sizeof(int), g->st));
  return HJB_OK;
}

// one pairwise matching pass on A (N rows): agg [N], mem [2][Nc] (g->ag_i[4] / [5] are sized N)
static hjb_status ag_pairwise(hjb_grid* g, int64_t N, const int* col, const double* val, int* agg, int* mem,
                              int64_t* Nc) {
  int *state = g->ag_i[0], *cand = g->ag_i[1], *flag = g->ag_i[2], *id = g->ag_i[3];
  CK(cudaMemsetAsync(state, 0xff, (size_t)N * sizeof(int), g->st));
  const int nb = ag_blocks(N, 128);
  unsigned long long* winner = (unsigned long long*)g->ag_i[2];  // flag/id scratch: 2 ints per node
  for (int round = 0; round < 6; ++round) {
    CK(cudaMemsetAsync(winner, 0, (size_t)N * sizeof(unsigned long long), g->st));
    LAUNCH(HJB_KC_COARSE, N, 0, 0, k_ag_candidates<<<nb, 128, 0, g->st>>>(N, col, val, state, cand, 0.25, round));
    LAUNCH(HJB_KC_COARSE, N, 0, 0, k_ag_propose<<<nb, 128, 0, g->st>>>(N, col, val, state, cand, winner));
    LAUNCH(HJB_KC_COARSE, N, 0, 0, k_ag_accept<<<nb, 128, 0, g->st>>>(N, winner, state));
  }
  LAUNCH(HJB_KC_COARSE, N, 0, 0, k_ag_singles<<<nb, 128, 0, g->st>>>(N, state));
  CKL();
  LAUNCH(HJB_KC_COARSE, N, 0, 0, k_ag_leader_flags<<<ag_blocks(N), 256, 0, g->st>>>(N, state, flag));
  size_t need = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, need, flag, id, (int)N, g->st);
  if (need > g->ag_cub_bytes) {
    cudaFree(g->ag_cub);
    TRY(dalloc(&g->ag_cub, need));
    g->ag_cub_bytes = need;
  }
  CK(cub::DeviceScan::ExclusiveSum(g->ag_cub, need, flag, id, (int)N, g->st));
  int last[2];
  CK(cudaMemcpyAsync(&last[0], id + N - 1, sizeof(int), cudaMemcpyDeviceToHost, g->st));
  CK(cudaMemcpyAsync(&last[1], flag + N - 1, sizeof(int), cudaMemcpyDeviceToHost, g->st));
  CK(cudaStreamSynchronize(g->st));
  *Nc = (int64_t)last[0] + last[1];
  CK(cudaMemsetAsync(mem, 0xff, (size_t)2 * *Nc * sizeof(int), g->st));
  LAUNCH(HJB_KC_COARSE, N, 0, 0, k_ag_number<<<ag_blocks(N), 256, 0, g->st>>>(N, state, id, agg, mem, *Nc));
  CKL();
  return HJB_OK;
}

template <int D>
static hjb_status agmg_setup(hjb_grid* g, double dt, const uint8_t* pol) {
  if (g->R != 1) return fail(HJB_ERR_UNSUPPORTED, "aggregation AMG: one rank only");
  agmg_release_levels(g);
  const int64_t N0 = g->L0.n_own;
  if (!g->d_flag) TRY(dalloc((void**)&g->d_flag, sizeof(int)));
  CK(cudaMemsetAsync(g->d_flag, 0, sizeof(int), g->st));
  if (!g->ag_i[0])
    for (auto& p : g->ag_i) TRY(dalloc((void**)&p, (size_t)N0 * 2 * sizeof(int)));
  g->ag.emplace_back();
  TRY(ag_alloc_level(g, g->ag.back(), N0));
  {
    auto& l0 = g->ag.back();
    const int nb = ag_blocks(N0, 128);
#define AGF(PP) LAUNCH(HJB_KC_COARSE, N0, 0, 0, k_ag_fine<D, PP><<<nb, 128, 0, g->st>>>(g->L0, g->C0, dt, pol, l0.col, l0.val, l0.dg, g->d_flag))
    if (g->P == 1) AGF(1);
    else if (g->P == 2) AGF(2);
    else AGF((D > 2 ? 3 : 2));
#undef AGF
    CKL();
    int flag = 0;
    CK(cudaMemcpyAsync(&flag, g->d_flag, sizeof(int), cudaMemcpyDeviceToHost, g->st));
    CK(cudaStreamSynchronize(g->st));
    if (flag) return fail(HJB_ERR_UNSUPPORTED, "aggregation AMG: a fine row wider than the ELL width (96)");
  }
  const int64_t stop = std::max<int64_t>(64, (int64_t)std::cbrt((double)N0));
  while (g->ag.back().N > stop && g->ag.size() < 20) {
    auto& lf = g->ag.back();
    const int64_t N = lf.N;
    // pass 1 on A_l
    int *agg1 = g->ag_i[4], *mem1 = g->ag_i[5];
    int64_t N1 = 0;
    TRY(ag_pairwise(g, N, lf.col, lf.val, agg1, mem1, &N1));
    hjb_grid::AgLevel tmp;
    TRY(ag_alloc_level(g, tmp, N1));
    LAUNCH(HJB_KC_COARSE, N1, 0, 0, k_ag_coarse<<<ag_blocks(N1, 128), 128, 0, g->st>>>(N, lf.col, lf.val, agg1, N1, mem1, 2,
                                                                                     tmp.col, tmp.val, tmp.dg, g->d_flag));
    // pass 2 on A_1 (the scratch of pass 1 moves into fresh buffers first)
    if (!g->ag_agg1c) {
      TRY(dalloc((void**)&g->ag_agg1c, (size_t)N0 * sizeof(int)));
      TRY(dalloc((void**)&g->ag_mem1c, (size_t)2 * N0 * sizeof(int)));
    }
    int *agg1c = g->ag_agg1c, *mem1c = g->ag_mem1c;
    CK(cudaMemcpyAsync(agg1c, agg1, (size_t)N * sizeof(int), cudaMemcpyDeviceToDevice, g->st));
    CK(cudaMemcpyAsync(mem1c, mem1, (size_t)2 * N1 * sizeof(int), cudaMemcpyDeviceToDevice, g->st));
    int64_t N2 = 0;
    TRY(ag_pairwise(g, N1, tmp.col, tmp.val, g->ag_i[4], g->ag_i[5], &N2));
    hjb_grid::AgLevel lc;
    TRY(ag_alloc_level(g, lc, N2));
    LAUNCH(HJB_KC_COARSE, N2, 0, 0, k_ag_coarse<<<ag_blocks(N2, 128), 128, 0, g->st>>>(N1, tmp.col, tmp.val, g->ag_i[4], N2,
                                                                                     g->ag_i[5], 2, lc.col, lc.val, lc.dg, g->d_flag));
    if (lf.cap_agg < N) {
      cudaFree(lf.agg);
      TRY(dalloc((void**)&lf.agg, (size_t)N * sizeof(int)));
      lf.cap_agg = N;
    }
    if (lf.cap_mem < 4 * N2) {
      cudaFree(lf.mem);
      TRY(dalloc((void**)&lf.mem, (size_t)4 * N2 * sizeof(int)));
      lf.cap_mem = 4 * N2;
    }
    CK(cudaMemsetAsync(lf.mem, 0xff, (size_t)4 * N2 * sizeof(int), g->st));
    LAUNCH(HJB_KC_COARSE, N, 0, 0, k_ag_compose<<<ag_blocks(std::max(N, N2)), 256, 0, g->st>>>(N, agg1c, g->ag_i[4], lf.agg, N1,
                                                                                             mem1c, g->ag_i[5], N2, lf.mem));
    CKL();
    int ovf = 0;  // a coarse row wider than the ELL width (kAgW): stop coarsening above this level
    CK(cudaMemcpyAsync(&ovf, g->d_flag, sizeof(int), cudaMemcpyDeviceToHost, g->st));
    CK(cudaStreamSynchronize(g->st));
    g->ag_pool.push_back(tmp);  // the pass-1 operator is not kept
    if (ovf || N2 * 10 >= N * 7) {  // overflow, or coarsening below 1.43x: the level just built is dropped
      if (ovf) CK(cudaMemsetAsync(g->d_flag, 0, sizeof(int), g->st));
      g->ag_pool.push_back(lc);
      break;
    }
    g->ag.push_back(lc);
  }
  auto& lc = g->ag.back();
  if (lc.N > kAgDenseMax) {
    // aggregation stalled above the dense size (e.g. Problem A at 321^2 with dt = dx): the coarsest
    // level is solved approximately by damped-Jacobi sweeps (the outer GCR is flexible)
    lc.Ainv = nullptr;
    g->ag_pol = pol;
    g->ag_dt = dt;
    g->ag_ready = true;
    return HJB_OK;
  }
  if (!g->ag_dense) TRY(dalloc((void**)&g->ag_dense, (size_t)kAgDenseMax * kAgDenseMax * sizeof(double)));
  lc.Ainv = g->ag_dense;
  CK(cudaMemsetAsync(lc.Ainv, 0, (size_t)lc.N * lc.N * sizeof(double), g->st));
  LAUNCH(HJB_KC_COARSE, lc.N, 0, 0, k_ag_dense<<<ag_blocks(lc.N), 256, 0, g->st>>>(lc.N, lc.col, lc.val, lc.Ainv));
  LAUNCH(HJB_KC_COARSE, lc.N, 0, 0, k_ag_invert<<<1, 1024, 0, g->st>>>(lc.Ainv, (int)lc.N));
  CKL();
  int flag = 0;
  CK(cudaMemcpyAsync(&flag, g->d_flag, sizeof(int), cudaMemcpyDeviceToHost, g->st));
  CK(cudaStreamSynchronize(g->st));
  if (flag) return fail(HJB_ERR_UNSUPPORTED, "aggregation AMG: a row wider than the ELL width (96)");
  g->ag_pol = pol;
  g->ag_dt = dt;
  g->ag_ready = true;
  return HJB_OK;
}

// dot products of compact vectors through the library's reduction path: returns (x.y, y.y)
static hjb_status ag_dot(hjb_grid* g, int64_t N, const double* x, const double* y, double* xy, double* yy) {
  const int nb = std::min(ag_blocks(N), kMaxBlocks);
  LAUNCH(HJB_KC_VECTOR, N, 16.0 * N, 4.0 * N, k_ag_dot2<<<nb, 256, 0, g->st>>>(N, x, y, g->partial));
  CKL();
  hjb_status err;
  *xy = host_finalize(g, nb, 0u, SC_NONE, &err, yy);
  return err;
}

static hjb_status ag_kcycle(hjb_grid* g, size_t l, const double* b, double* x);

// 2 flexible GCR iterations on level c (x0 = 0), preconditioned by its K-cycle: the K-cycle's
// coarse-grid solve ("a number of Krylov subspace iterations")
// HJB_AG_DEVICE=1: the scalars stay on the device (k_ag_scal / k_ag_axpy_dev), no host round trip
// inside the cycle, but without Notay's adaptive rule (stop after one iteration if it reduced the
// residual 4x), which needs the residual on the host: both iterations always.
static hjb_status ag_inner(hjb_grid* g, size_t c, const double* b, double* x) {
  auto& L = g->ag[c];
  const int64_t N = L.N;
  const int nb = ag_blocks(N);
  CK(cudaMemsetAsync(x, 0, (size_t)N * sizeof(double), g->st));
  CK(cudaMemcpyAsync(L.r, b, (size_t)N * sizeof(double), cudaMemcpyDeviceToDevice, g->st));
  if (getenv("HJB_AG_DEVICE")) {  // opt-in: measured slower (no adaptive skip below level 1 doubles
                                  // the launch-bound coarse visits; tools/paper_context.py)
    if (!g->ag_sc) TRY(dalloc((void**)&g->ag_sc, (size_t)8 * 32 * sizeof(double)));
    const int base = 8 * (int)std::min<size_t>(c, 31);
    const int nbd = std::min(ag_blocks(N), kMaxBlocks);
    for (int it = 0; it < 2; ++it) {
      TRY(ag_kcycle(g, c, L.r, L.z[it]));
      LAUNCH(HJB_KC_MG_COARSE, N, 0, 0, k_ag_spmv<<<nb, 256, 0, g->st>>>(N, L.col, L.val, L.z[it], L.az[it]));
      if (it == 1) {  // orthogonalise against the (normalised) first direction
        LAUNCH(HJB_KC_VECTOR, N, 16.0 * N, 4.0 * N, k_ag_dot2<<<nbd, 256, 0, g->st>>>(N, L.az[0], L.az[1], g->partial));
        LAUNCH(HJB_KC_REDUCE, nbd, 0, 0, k_ag_scal<<<1, 256, 0, g->st>>>(g->partial, nbd, g->ag_sc, base, 0));
        LAUNCH(HJB_KC_VECTOR, N, 0, 0, k_ag_axpy_dev<<<nb, 256, 0, g->st>>>(N, g->ag_sc, base, L.az[0], L.az[1]));
        LAUNCH(HJB_KC_VECTOR, N, 0, 0, k_ag_axpy_dev<<<nb, 256, 0, g->st>>>(N, g->ag_sc, base, L.z[0], L.z[1]));
      }
      LAUNCH(HJB_KC_VECTOR, N, 16.0 * N, 4.0 * N, k_ag_dot2<<<nbd, 256, 0, g->st>>>(N, L.az[it], L.az[it], g->partial));
      LAUNCH(HJB_KC_REDUCE, nbd, 0, 0, k_ag_scal<<<1, 256, 0, g->st>>>(g->partial, nbd, g->ag_sc, base + 1, 1));
      LAUNCH(HJB_KC_VECTOR, N, 0, 0, k_ag_scale_dev<<<nb, 256, 0, g->st>>>(N, g->ag_sc, base + 1, L.az[it]));
      LAUNCH(HJB_KC_VECTOR, N, 0, 0, k_ag_scale_dev<<<nb, 256, 0, g->st>>>(N, g->ag_sc, base + 1, L.z[it]));
      LAUNCH(HJB_KC_VECTOR, N, 16.0 * N, 4.0 * N, k_ag_dot2<<<nbd, 256, 0, g->st>>>(N, L.az[it], L.r, g->partial));
      LAUNCH(HJB_KC_REDUCE, nbd, 0, 0, k_ag_scal<<<1, 256, 0, g->st>>>(g->partial, nbd, g->ag_sc, base + 2, 2));
      LAUNCH(HJB_KC_VECTOR, N, 0, 0, k_ag_axpy_dev<<<nb, 256, 0, g->st>>>(N, g->ag_sc, base + 2, L.z[it], x));
      LAUNCH(HJB_KC_VECTOR, N, 0, 0, k_ag_axpy_dev<<<nb, 256, 0, g->st>>>(N, g->ag_sc, base + 3, L.az[it], L.r));
    }
    CKL();
    return HJB_OK;
  }
  for (int it = 0; it < 2; ++it) {
    TRY(ag_kcycle(g, c, L.r, L.z[it]));
    LAUNCH(HJB_KC_MG_COARSE, N, 0, 0, k_ag_spmv<<<nb, 256, 0, g->st>>>(N, L.col, L.val, L.z[it], L.az[it]));
    if (it == 1) {
      double h, unused;
      TRY(ag_dot(g, N, L.az[0], L.az[1], &h, &unused));
      LAUNCH(HJB_KC_VECTOR, N, 0, 0, k_ag_axpby<<<nb, 256, 0, g->st>>>(N, -h, L.az[0], 1.0, L.az[1]));
      LAUNCH(HJB_KC_VECTOR, N, 0, 0, k_ag_axpby<<<nb, 256, 0, g->st>>>(N, -h, L.z[0], 1.0, L.z[1]));
    }
    double unused, nn;
    TRY(ag_dot(g, N, L.az[it], L.az[it], &unused, &nn));
    const double nrm = std::sqrt(nn);
    if (!(nrm > 0.0)) break;
    LAUNCH(HJB_KC_VECTOR, N, 0, 0, k_ag_axpby<<<nb, 256, 0, g->st>>>(N, 0.0, L.az[it], 1.0 / nrm, L.az[it]));
    LAUNCH(HJB_KC_VECTOR, N, 0, 0, k_ag_axpby<<<nb, 256, 0, g->st>>>(N, 0.0, L.z[it], 1.0 / nrm, L.z[it]));
    double gam, rr;
    TRY(ag_dot(g, N, L.az[it], L.r, &gam, &rr));
    LAUNCH(HJB_KC_VECTOR, N, 0, 0, k_ag_axpby<<<nb, 256, 0, g->st>>>(N, gam, L.z[it], 1.0, x));
    LAUNCH(HJB_KC_VECTOR, N, 0, 0, k_ag_axpby<<<nb, 256, 0, g->st>>>(N, -gam, L.az[it], 1.0, L.r));
    // K-cycle's adaptive rule (Notay): one inner iteration suffices if it reduced the residual 4x
    if (it == 0 && rr - gam * gam <= 0.0625 * rr) break;
  }
  CKL();
  return HJB_OK;
}

// x = B_l^{-1} b: K-cycle of level l (one damped-Jacobi pre- and post-smoothing step)
static hjb_status ag_kcycle(hjb_grid* g, size_t l, const double* b, double* x) {
  auto& L = g->ag[l];
  const int64_t N = L.N;
  const int nb = ag_blocks(N);
  if (l + 1 == g->ag.size()) {
    if (L.Ainv) {
      LAUNCH(HJB_KC_COARSE, N, 0, 0, k_ag_dense_solve<<<(int)((N + 127) / 128), 128, 0, g->st>>>((int)N, L.Ainv, b, x));
    } else {  // no dense inverse (stalled aggregation): kAgCoarseSweeps damped-Jacobi sweeps from 0
      CK(cudaMemsetAsync(L.t, 0, (size_t)N * sizeof(double), g->st));
      double* in = L.t;
      double* outp = x;
      for (int k = 0; k < kAgCoarseSweeps; ++k) {
        LAUNCH(HJB_KC_COARSE, N, 0, 0, k_ag_sweep<true><<<nb, 256, 0, g->st>>>(N, L.col, L.val, L.dg, in, b, kAgOmega, outp));
        std::swap(in, outp);
      }
      if (in != x) CK(cudaMemcpyAsync(x, in, (size_t)N * sizeof(double), cudaMemcpyDeviceToDevice, g->st));
    }
    CKL();
    return HJB_OK;
  }
  auto& C = g->ag[l + 1];
  CK(cudaMemsetAsync(L.t, 0, (size_t)N * sizeof(double), g->st));
  LAUNCH(HJB_KC_MG_COARSE, N, 0, 0, k_ag_sweep<true><<<nb, 256, 0, g->st>>>(N, L.col, L.val, L.dg, L.t, b, kAgOmega, x));
  LAUNCH(HJB_KC_MG_COARSE, N, 0, 0, k_ag_sweep<false><<<nb, 256, 0, g->st>>>(N, L.col, L.val, L.dg, x, b, 0.0, L.t));
  LAUNCH(HJB_KC_TRANSFER, C.N, 0, 0, k_ag_restrict<<<ag_blocks(C.N), 256, 0, g->st>>>(C.N, L.mem, 4, L.t, C.b));
  if (l + 2 == g->ag.size()) TRY(ag_kcycle(g, l + 1, C.b, C.x));
  else TRY(ag_inner(g, l + 1, C.b, C.x));
  LAUNCH(HJB_KC_TRANSFER, N, 0, 0, k_ag_prolong<<<nb, 256, 0, g->st>>>(N, L.agg, C.x, x));
  CK(cudaMemcpyAsync(L.t, x, (size_t)N * sizeof(double), cudaMemcpyDeviceToDevice, g->st));
  LAUNCH(HJB_KC_MG_COARSE, N, 0, 0, k_ag_sweep<true><<<nb, 256, 0, g->st>>>(N, L.col, L.val, L.dg, L.t, b, kAgOmega, x));
  CKL();
  return HJB_OK;
}

// U += e with A e = F - A U solved by K-cycle-preconditioned flexible GCR(10) to
// ||F - A U||_2 <= max(rtol ||F||_2, eta ||r_0||_2) (and the max-norm stop of an exact evaluation)
template <int D>
static hjb_status agmg_solve(hjb_grid* g, double dt, const uint8_t* pol, const double* F, double* U,
                             const hjb_solve_params* sp, hjb_solve_stats* out, double eta) {
  if (!g->ag_ready || g->ag_pol != pol || g->ag_dt != dt) TRY(agmg_setup<D>(g, dt, pol));
  auto& L0 = g->ag[0];
  const int64_t N = L0.N;
  const int nb = ag_blocks(N);
  for (int k = 0; k < kAgRestart; ++k)
    if (!g->ag_Z[k]) {
      TRY(dalloc((void**)&g->ag_Z[k], (size_t)N * sizeof(double)));
      TRY(dalloc((void**)&g->ag_AZ[k], (size_t)N * sizeof(double)));
    }
  Level tmpl;
  const Level& lv0 = fine_level(g, tmpl);
  double bn2, bninf;
  TRY(norms_dev<D>(g, F, &bn2, &bninf));
  double tol = sp->krylov_rtol * bn2;
  const double tol_inf = (eta > 0.0 || !(sp->krylov_rtol_inf > 0.0)) ? INFINITY : sp->krylov_rtol_inf * bninf;
  int it = 0;
  bool converged = false;
  for (int restart = 0; restart < 6 && !converged; ++restart) {
    // r = F - A U (matrix-free, the boundary data included); compact copy
    TRY(halo_exchange(g, lv0, U, g->lay.halo));
    launch_operator<D>(g, g->L0, coef_u(g), OP_RESID, 0, dt, 0.0, pol, U, F, g->r, nullptr);
    double r2, rinf;
    TRY(norms_dev<D>(g, g->r, &r2, &rinf));
    if (!std::isfinite(r2)) return fail(HJB_ERR_NONFINITE, "non-finite residual");
    if (restart == 0 && eta > 0.0) tol = std::max(tol, eta * r2);
    if (out) {
      out->iters = it;
      out->rres = bn2 > 0 ? r2 / bn2 : r2;
      out->rres_inf = bninf > 0 ? rinf / bninf : rinf;
    }
    if (r2 <= tol && rinf <= tol_inf) { converged = true; break; }
    const double tol_it = (rinf > tol_inf) ? std::min(tol, 0.5 * r2 * (tol_inf / rinf)) : tol;
    LAUNCH(HJB_KC_VECTOR, N, 16.0 * N, 0, k_ag_gather<D><<<dims(g, g->L0, (const void*)k_ag_gather<D>), dim3(kBX, kBY), 0, g->st>>>(g->L0, g->r, L0.r));
    CK(cudaMemsetAsync(L0.x, 0, (size_t)N * sizeof(double), g->st));
    double rn = r2;
    int m = 0;
    while (it < sp->krylov_maxit && rn > tol_it) {
      TRY(ag_kcycle(g, 0, L0.r, g->ag_Z[m]));
      LAUNCH(HJB_KC_APPLY, N, 0, 0, k_ag_spmv<<<nb, 256, 0, g->st>>>(N, L0.col, L0.val, g->ag_Z[m], g->ag_AZ[m]));
      for (int k = 0; k < m; ++k) {
        double h, unused;
        TRY(ag_dot(g, N, g->ag_AZ[k], g->ag_AZ[m], &h, &unused));
        LAUNCH(HJB_KC_VECTOR, N, 0, 0, k_ag_axpby<<<nb, 256, 0, g->st>>>(N, -h, g->ag_AZ[k], 1.0, g->ag_AZ[m]));
        LAUNCH(HJB_KC_VECTOR, N, 0, 0, k_ag_axpby<<<nb, 256, 0, g->st>>>(N, -h, g->ag_Z[k], 1.0, g->ag_Z[m]));
      }
      double unused, nn;
      TRY(ag_dot(g, N, g->ag_AZ[m], g->ag_AZ[m], &unused, &nn));
      const double nrm = std::sqrt(nn);
      if (!(nrm > 0.0) || !std::isfinite(nrm)) break;
      LAUNCH(HJB_KC_VECTOR, N, 0, 0, k_ag_axpby<<<nb, 256, 0, g->st>>>(N, 0.0, g->ag_AZ[m], 1.0 / nrm, g->ag_AZ[m]));
      LAUNCH(HJB_KC_VECTOR, N, 0, 0, k_ag_axpby<<<nb, 256, 0, g->st>>>(N, 0.0, g->ag_Z[m], 1.0 / nrm, g->ag_Z[m]));
      double gam, rr;
      TRY(ag_dot(g, N, g->ag_AZ[m], L0.r, &gam, &rr));
      LAUNCH(HJB_KC_VECTOR, N, 0, 0, k_ag_axpby<<<nb, 256, 0, g->st>>>(N, gam, g->ag_Z[m], 1.0, L0.x));
      LAUNCH(HJB_KC_VECTOR, N, 0, 0, k_ag_axpby<<<nb, 256, 0, g->st>>>(N, -gam, g->ag_AZ[m], 1.0, L0.r));
      rn = std::sqrt(std::max(0.0, rr - gam * gam));
      ++it;
      if (++m == kAgRestart) m = 0;
    }
    LAUNCH(HJB_KC_VECTOR, N, 16.0 * N, 0, k_ag_scatter_add<D><<<dims(g, g->L0, (const void*)k_ag_scatter_add<D>), dim3(kBX, kBY), 0, g->st>>>(g->L0, L0.x, U));
    CKL();
    if (it >= sp->krylov_maxit) {
      TRY(halo_exchange(g, lv0, U, g->lay.halo));
      launch_operator<D>(g, g->L0, coef_u(g), OP_RESID, 0, dt, 0.0, pol, U, F, g->r, nullptr);
      TRY(norms_dev<D>(g, g->r, &r2, &rinf));
      if (out) { out->iters = it; out->rres = bn2 > 0 ? r2 / bn2 : r2; out->rres_inf = bninf > 0 ? rinf / bninf : rinf; }
      converged = r2 <= tol && rinf <= tol_inf;
      break;
    }
  }
  if (!converged) return fail(HJB_ERR_NOT_CONVERGED, "AGMG-preconditioned GCR did not reach the tolerance");
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
  if (sp->solver == 1)
    return g->D == 2 ? agmg_solve<2>(g, dt, policy, F, x, sp, out, 0.0) : agmg_solve<3>(g, dt, policy, F, x, sp, out, 0.0);
  return g->D == 2 ? bicgstab<2>(g, dt, policy, F, x, sp, out) : bicgstab<3>(g, dt, policy, F, x, sp, out);
}

// ---------------------------------------------------------------------------- theta-scheme
// y = A'_{dt'} x for the fine level (x's halos exchanged on a scratch copy when several ranks)
static hjb_status apply_fine(hjb_grid* g, double dtp, const uint8_t* pol, const double* x, double* y) {
  const double* xx;
  TRY(halo_input(g, x, &xx));
  if (g->D == 2) launch_operator<2>(g, g->L0, g->C0, OP_APPLY, 0, dtp, 0.0, pol, xx, nullptr, y, nullptr);
  else launch_operator<3>(g, g->L0, g->C0, OP_APPLY, 0, dtp, 0.0, pol, xx, nullptr, y, nullptr);
  CKL();
  return HJB_OK;
}

static hjb_status theta_rhs(hjb_grid* g, const double* up, const double* y, double* out) {
  const double nn = (double)g->L0.n_own;
  if (g->D == 2)
    LAUNCH(HJB_KC_VECTOR, nn, 32.0 * nn, 2.0 * nn,
           k_theta_rhs<2><<<dims(g, g->L0, (const void*)k_theta_rhs<2>), dim3(kBX, kBY), 0, g->st>>>(g->L0, g->F, up, y, out));
  else
    LAUNCH(HJB_KC_VECTOR, nn, 32.0 * nn, 2.0 * nn,
           k_theta_rhs<3><<<dims(g, g->L0, (const void*)k_theta_rhs<3>), dim3(kBX, kBY), 0, g->st>>>(g->L0, g->F, up, y, out));
  CKL();
  return HJB_OK;
}

// One theta-step (theta < 1) after hjb_step's staging (dU holds the initial iterate with psi(t_n)
// on its boundary; dprev holds U^{n-1} with psi(t_{n-1})).  theta = 0: explicit Euler.
static hjb_status theta_step(hjb_grid* g, double dt, const double* dprev, double* dU, uint8_t* dpol,
                             const hjb_solve_params* sp, hjb_step_stats* S) {
  const double th = sp->theta;
  Level tmpl;
  const Level& lv0 = fine_level(g, tmpl);
  const int64_t ne = g->N;
  cudaStream_t st = g->st;
  float ms;
  if (th == 0.0) {
    // search at U^{n-1}: policy argmin_a H^a(U^{n-1}), F = U^{n-1} + dt f^pi; then
    // U^n = F + U^{n-1} - A'_dt U^{n-1} = U^{n-1} + dt (L^pi + c) U^{n-1} + dt f^pi (interior)
    const double* up;
    TRY(halo_input(g, dprev, &up));
    hjb_pi_stats pis{};
    cudaEventRecord(g->ev[0], st);
    TRY(policy_update_dev(g, dt, up, dprev, dpol, g->F, &pis));
    cudaEventRecord(g->ev[1], st);
    TRY(apply_fine(g, dt, dpol, dprev, g->v));
    TRY(theta_rhs(g, dprev, g->v, dU));
    cudaEventRecord(g->ev[2], st);
    CK(cudaEventSynchronize(g->ev[2]));
    cudaEventElapsedTime(&ms, g->ev[0], g->ev[1]);
    S->ms_search += ms;
    cudaEventElapsedTime(&ms, g->ev[1], g->ev[2]);
    S->ms_solve += ms;
    S->pi_iters = 1;
    S->changed[0] = pis.changed;
    S->R[0] = S->final_R = 0.0;  // explicit: the step is its own solution
    return HJB_OK;
  }
  if (!g->vtheta) TRY(dalloc((void**)&g->vtheta, (size_t)ne * sizeof(double)));
  hjb_status result = HJB_OK;
  bool last_exact = true;
  const int nb1 = (int)std::min<int64_t>((ne + 255) / 256, (int64_t)g->sms * 8);
  for (int it = 1; it <= sp->max_pi; ++it) {
    hjb_pi_stats pis{};
    cudaEventRecord(g->ev[0], st);
    // search at V = theta U + (1 - theta) U^{n-1} (row residual U - U^{n-1} - dt H(V), D1 with theta)
    LAUNCH(HJB_KC_VECTOR, (double)ne, 24.0 * ne, 3.0 * ne, k_theta_mix<<<nb1, 256, 0, st>>>(th, dU, dprev, g->vtheta, ne));
    CKL();
    TRY(halo_exchange(g, lv0, g->vtheta, g->lay.halo));
    TRY(policy_update_dev(g, dt, g->vtheta, dprev, dpol, g->F, &pis));
    // F_theta = U^{n-1} + (1-theta) dt (L^pi + c) U^{n-1} + dt f^pi ; R = ||F_theta - A_{theta dt} U||_inf
    TRY(apply_fine(g, (1.0 - th) * dt, dpol, dprev, g->v));
    TRY(theta_rhs(g, dprev, g->v, g->F));
    TRY(halo_exchange(g, lv0, dU, g->lay.halo));
    if (g->D == 2) launch_operator<2>(g, g->L0, g->C0, OP_RESID, 0, th * dt, 0.0, dpol, dU, g->F, g->r, nullptr);
    else launch_operator<3>(g, g->L0, g->C0, OP_RESID, 0, th * dt, 0.0, dpol, dU, g->F, g->r, nullptr);
    double r2, Rinf;
    TRY(g->D == 2 ? norms_dev<2>(g, g->r, &r2, &Rinf) : norms_dev<3>(g, g->r, &r2, &Rinf));
    cudaEventRecord(g->ev[1], st);
    CK(cudaEventSynchronize(g->ev[1]));
    cudaEventElapsedTime(&ms, g->ev[0], g->ev[1]);
    S->ms_search += ms;
    const int slot = std::min(it - 1, HJB_MAX_PI_LOG - 1);
    S->changed[slot] = pis.changed;
    S->R[slot] = Rinf;
    S->final_R = Rinf;
    if (!std::isfinite(Rinf)) return fail(HJB_ERR_NONFINITE, "non-finite theta-scheme residual");
    if (it > 1 && (Rinf <= sp->tol_pi || (pis.changed == 0 && last_exact))) break;
    if (it == sp->max_pi) { result = fail(HJB_ERR_NOT_CONVERGED, "policy iteration hit max_pi"); break; }
    const bool settled = (it > 1 && pis.changed == 0);
    cudaEventRecord(g->ev[0], st);
    if (sp->use_mg && !(settled && g->mg_ready && g->mg_pol0 == dpol && g->mg_dt == th * dt))
      TRY(hjb_mg_setup(g, th * dt, dpol, &sp->mg));
    cudaEventRecord(g->ev[1], st);
    hjb_solve_stats ss{};
    const double eta = (settled || g->K == 1) ? 0.0 : sp->pi_forcing;
    hjb_status s2 = g->D == 2 ? bicgstab<2>(g, th * dt, dpol, g->F, dU, sp, &ss, eta)
                              : bicgstab<3>(g, th * dt, dpol, g->F, dU, sp, &ss, eta);
    last_exact = (ss.rres <= sp->krylov_rtol) && (!(sp->krylov_rtol_inf > 0.0) || ss.rres_inf <= sp->krylov_rtol_inf);
    cudaEventRecord(g->ev[2], st);
    CK(cudaEventSynchronize(g->ev[2]));
    cudaEventElapsedTime(&ms, g->ev[0], g->ev[1]);
    S->ms_setup += ms;
    cudaEventElapsedTime(&ms, g->ev[1], g->ev[2]);
    S->ms_solve += ms;
    S->pi_iters = it;
    S->krylov_iters[slot] = ss.iters;
    S->krylov_iters_total += ss.iters;
    S->final_rres = ss.rres;
    S->final_rres_inf = ss.rres_inf;
    if (s2 != HJB_OK) { result = s2; break; }
  }
  return result;
}

extern "C" hjb_status hjb_set_boundary_samples(hjb_grid_t g, int32_t refine, const double* samples) {
  if (!g) return fail(HJB_ERR_INVALID_ARG, "null handle");
  if (!samples) {
    g->bsamp = nullptr;
    g->brefine = 0;
    return HJB_OK;
  }
  if (refine < 1 || refine * (g->n - 1) + 1 < 4) return fail(HJB_ERR_INVALID_ARG, "refine must be >= 1 (>= 4 samples per axis)");
  if (!is_device_ptr(samples)) return fail(HJB_ERR_INVALID_ARG, "samples must be a device array");
  g->bsamp = samples;
  g->brefine = refine;
  return HJB_OK;
}

extern "C" hjb_status hjb_cfl_rate(hjb_grid_t g, const uint8_t* policy, double* rate) {
  if (!g || !rate) return fail(HJB_ERR_INVALID_ARG, "null argument");
  if (!g->have_coeffs) return fail(HJB_ERR_STATE, "call hjb_set_coeffs first");
  if (policy && !is_device_ptr(policy)) return fail(HJB_ERR_INVALID_ARG, "policy must be a device array");
  CK(cudaSetDevice(g->desc.device));
  const LevelDev& L = g->L0;
#define CFL(DD, PP)                                                                                       \
  LAUNCH(HJB_KC_BOUNDARY, 0, 0, 0,                                                                        \
         k_cfl<DD, PP><<<dims(g, L, (const void*)k_cfl<DD, PP>), dim3(kBX, kBY), 0, g->st>>>(L, g->C0, policy, \
                                                                                            g->partial))
  if (g->D == 2) {
    if (g->P == 1) CFL(2, 1);
    else CFL(2, 2);
  } else {
    if (g->P == 1) CFL(3, 1);
    else if (g->P == 2) CFL(3, 2);
    else CFL(3, 3);
  }
#undef CFL
  CKL();
  hjb_status err;
  *rate = host_finalize(g, g->nblk_last, 0x1u, SC_NONE, &err);
  return err;
}

// ---------------------------------------------------------------------------- step
static hjb_status implicit_pi(hjb_grid* g, double dt, const double* dprev, double* dU, uint8_t* dpol,
                              const hjb_solve_params* sp, hjb_step_stats& S);
static hjb_status nested_guess(hjb_grid* g, double dt, const double* dprev, double* dU, const hjb_solve_params* sp,
                               hjb_step_stats* S);

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
  const bool alias = (U == U_prev) && !h_prev;  // in-place step on device memory
  uint8_t* dpol = policy ? policy : g->pol_int;
  const double* dpsi = psi;
  if (h_prev || alias) {
    // host U_prev is staged; a device U_prev that is also the output U is copied first, else the
    // first solve would overwrite U^{n-1} and every later F = U^{n-1} + dt f would be wrong
    if (!g->stage_prev) TRY(dalloc((void**)&g->stage_prev, vb));
    CK(cudaMemcpyAsync(g->stage_prev, U_prev, vb, h_prev ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
    dprev = g->stage_prev;
  }
  if (sp->guess < HJB_GUESS_PREV || sp->guess > HJB_GUESS_NESTED)
    return fail(HJB_ERR_INVALID_ARG, "unknown initial-guess mode");
  // an in-place step has no U^{n-2} or caller's guess: it starts from U_prev (nested: refined from there)
  const int guess = (U == U_prev && sp->guess != HJB_GUESS_NESTED) ? HJB_GUESS_PREV : sp->guess;
  if (h_U) {
    if (!g->stage_U) TRY(dalloc((void**)&g->stage_U, vb));
    dU = g->stage_U;
    if (guess == HJB_GUESS_GIVEN || guess == HJB_GUESS_EXTRAPOLATE)
      CK(cudaMemcpyAsync(dU, U, vb, cudaMemcpyHostToDevice, st));
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
  // a1: initial iterate (U_prev, the caller's guess, or the linear extrapolation 2 U_prev - U^{n-2}),
  // then boundary entries psi(t_n)
  if ((guess == HJB_GUESS_PREV || guess == HJB_GUESS_NESTED) && dU != dprev) {
    CK(cudaMemcpyAsync(dU, dprev, vb, cudaMemcpyDeviceToDevice, st));
  } else if (guess == HJB_GUESS_EXTRAPOLATE) {
    const double nn = (double)g->L0.n_own;
    if (g->D == 2)
      LAUNCH(HJB_KC_VECTOR, nn, 24.0 * nn, 2.0 * nn,
             k_extrapolate<2><<<dims(g, g->L0, (const void*)k_extrapolate<2>), dim3(kBX, kBY), 0, st>>>(g->L0, dprev, dU));
    else
      LAUNCH(HJB_KC_VECTOR, nn, 24.0 * nn, 2.0 * nn,
             k_extrapolate<3><<<dims(g, g->L0, (const void*)k_extrapolate<3>), dim3(kBX, kBY), 0, st>>>(g->L0, dprev, dU));
    CKL();
  }
  if (dpsi) {
    const int nbb = (int)std::min<int64_t>((g->n_boundary + 255) / 256, 4096);
    const double nbd = (double)g->n_boundary;
    if (g->D == 2)
      LAUNCH(HJB_KC_BOUNDARY, nbd, 16.0 * nbd, 0, k_scatter_psi<2><<<nbb, 256, 0, st>>>(g->L0, g->n_boundary, dpsi, dU));
    else
      LAUNCH(HJB_KC_BOUNDARY, nbd, 16.0 * nbd, 0, k_scatter_psi<3><<<nbb, 256, 0, st>>>(g->L0, g->n_boundary, dpsi, dU));
    CKL();
  }
  Level tmpl;
  const Level& lv0 = fine_level(g, tmpl);
  hjb_step_stats S{};
  float ms;
  hjb_status result = HJB_OK;
  if (!(sp->theta >= 0.0 && sp->theta <= 1.0)) return fail(HJB_ERR_INVALID_ARG, "theta must be in [0, 1]");
  if (sp->theta < 1.0 && g->bsamp)
    return fail(HJB_ERR_UNSUPPORTED, "the exact-psi boundary mode supports theta = 1 only");
  if (sp->theta < 1.0) {
    result = theta_step(g, dt, dprev, dU, dpol, sp, &S);
    S.n_levels = (int32_t)g->levels.size();
    if (h_U) CK(cudaMemcpyAsync(U, dU, vb, cudaMemcpyDeviceToHost, st));
    if (h_pol) CK(cudaMemcpyAsync(policy, dpol, (size_t)g->N, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (out) *out = S;
    return result;
  }
  if (guess == HJB_GUESS_NESTED) {
    cudaEventRecord(g->ev[3], st);
    TRY(nested_guess(g, dt, dprev, dU, sp, &S));
    cudaEventRecord(g->ev[2], st);
    CK(cudaEventSynchronize(g->ev[2]));
    cudaEventElapsedTime(&ms, g->ev[3], g->ev[2]);
    S.ms_nested += ms;
  }
  result = implicit_pi(g, dt, dprev, dU, dpol, sp, S);
  S.n_levels = (int32_t)g->levels.size();
  if (h_U) CK(cudaMemcpyAsync(U, dU, vb, cudaMemcpyDeviceToHost, st));
  if (h_pol) CK(cudaMemcpyAsync(policy, dpol, (size_t)g->N, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (out) *out = S;
  return result;
}

// The Howard loop of an implicit step from the iterate dU (psi(t_n) on its
// boundary): policy improvement, stop test, policy evaluation, repeat.
static hjb_status implicit_pi(hjb_grid* g, double dt, const double* dprev, double* dU, uint8_t* dpol,
                              const hjb_solve_params* sp, hjb_step_stats& S) {
  cudaStream_t st = g->st;
  Level tmpl;
  const Level& lv0 = fine_level(g, tmpl);
  float ms;
  hjb_status result = HJB_OK;
  bool last_exact = true;  // the last policy evaluation reached krylov_rtol
  for (int it = 1; it <= sp->max_pi; ++it) {
    hjb_pi_stats pis{};
    cudaEventRecord(g->ev[0], st);
    TRY(halo_exchange(g, lv0, dU, g->lay.halo));
    // the step's first search is the plain scan (the GAP scan is ~25 % slower); the second one records
    // the gaps, from the third on CTAs may skip
    if (it == 1) {
      g->gap_on = false;
      g->gap_valid = false;
    } else {
      TRY(gap_prepare(g, dU, false));
    }
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
    if (sp->solver == 0 && sp->use_mg && !(settled && g->mg_ready && g->mg_pol0 == dpol && g->mg_dt == dt))
      TRY(hjb_mg_setup(g, dt, dpol, &sp->mg));
    if (sp->solver == 1 && !(settled && g->ag_ready && g->ag_pol == dpol && g->ag_dt == dt))
      TRY(g->D == 2 ? agmg_setup<2>(g, dt, dpol) : agmg_setup<3>(g, dt, dpol));
    cudaEventRecord(g->ev[1], st);
    hjb_solve_stats ss{};
    // inexact Howard: while the policy still changes, evaluate it only to eta * ||r_0||
    const double eta = (settled || g->K == 1) ? 0.0 : sp->pi_forcing;  // K = 1: the policy is final
    hjb_status s = sp->solver == 1 ? (g->D == 2 ? agmg_solve<2>(g, dt, dpol, g->F, dU, sp, &ss, eta)
                                                : agmg_solve<3>(g, dt, dpol, g->F, dU, sp, &ss, eta))
                   : g->D == 2 ? bicgstab<2>(g, dt, dpol, g->F, dU, sp, &ss, eta)
                               : bicgstab<3>(g, dt, dpol, g->F, dU, sp, &ss, eta);
    last_exact = (ss.rres <= sp->krylov_rtol) && (!(sp->krylov_rtol_inf > 0.0) || ss.rres_inf <= sp->krylov_rtol_inf);
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
    S.final_rres_inf = ss.rres_inf;
    if (s != HJB_OK) { result = s; break; }
  }
  return result;
}

// ---------------------------------------------------------------------------- nested iteration
// The coarse grid of HJB_GUESS_NESTED (created on first use; fields re-injected after set_coeffs),
// or nullptr when nesting does not apply (reading xxx).
static hjb_status nested_child(hjb_grid* g, const hjb_solve_params* sp, hjb_grid** out) {
  *out = nullptr;
  const int m = sp->nested_coarsen;
  if (m < 1 || m > 8 || g->R > 1 || g->bsamp || !g->have_coeffs) return HJB_OK;
  const int64_t f = 1LL << m;
  if ((g->n - 1) % f != 0) return HJB_OK;
  const int64_t nc = (g->n - 1) / f + 1;
  if (nc < std::max<int64_t>(5, sp->nested_min_n)) return HJB_OK;
  const int D = g->D;
  int64_t Nc = nc;
  for (int d = 1; d < D; ++d) Nc *= nc;
  const int np_sig = g->C0.sigma_scale ? g->P : 0, np_sn = g->C0.sigma_node ? g->P * D : 0,
            np_bs = g->C0.b_scale ? 1 : 0, np_bn = g->C0.b_node ? D : 0, np_c = g->C0.c_node ? 1 : 0,
            np_f = (g->Q > 0 && g->C0.f_feat) ? g->Q : 0;
  const int nplanes = np_sig + np_sn + np_bs + np_bn + np_c + np_f;
  if (g->child && g->child_m != m) {
    hjb_grid_destroy(g->child);
    g->child = nullptr;
    cudaFree(g->child_fields);
    cudaFree(g->child_U);
    cudaFree(g->child_prev);
    cudaFree(g->child_pol);
    g->child_fields = g->child_U = g->child_prev = nullptr;
    g->child_pol = nullptr;
  }
  if (!g->child) {
    hjb_grid_desc d = g->desc;
    d.n = nc;
    d.rank = 0;
    d.nranks = 1;
    d.nccl_id = nullptr;
    d.halo = 0;
    TRY(hjb_grid_create(&d, &g->child));
    g->child_m = m;
    g->child_dirty = true;
    if (nplanes > 0) TRY(dalloc((void**)&g->child_fields, (size_t)nplanes * Nc * sizeof(double)));
    TRY(dalloc((void**)&g->child_U, (size_t)Nc * sizeof(double)));
    TRY(dalloc((void**)&g->child_prev, (size_t)Nc * sizeof(double)));
    TRY(dalloc((void**)&g->child_pol, (size_t)Nc));
    CK(cudaMemsetAsync(g->child_pol, 0, (size_t)Nc, g->st));
  }
  hjb_grid* c = g->child;
  c->prof_timing = g->prof_timing;
  c->prof.timed = g->prof.timed;
  if (g->child_dirty) {
    const int nb = (int)std::min<int64_t>((Nc + 255) / 256, (int64_t)g->sms * 8);
    double* dst = g->child_fields;
    auto inj = [&](const double* src, int np) -> const double* {
      if (!src || np == 0) return nullptr;
      double* o = dst;
      if (D == 2)
        LAUNCH(HJB_KC_TRANSFER, Nc, 16.0 * np * Nc, 0,
               k_nest_inject<2><<<nb, 256, 0, g->st>>>(g->n, nc, (int)f, src, g->N, o, Nc, np));
      else
        LAUNCH(HJB_KC_TRANSFER, Nc, 16.0 * np * Nc, 0,
               k_nest_inject<3><<<nb, 256, 0, g->st>>>(g->n, nc, (int)f, src, g->N, o, Nc, np));
      dst += (size_t)np * Nc;
      return o;
    };
    hjb_coeffs cc{};
    cc.sigma_dir = g->h_sd.data();
    cc.b_dir = g->h_bd.data();
    cc.c_ctrl = g->h_cc.data();
    cc.f_basis = g->Q > 0 ? g->h_fb.data() : nullptr;
    cc.f_ctrl = g->h_fc.data();
    cc.sigma_scale = inj(g->C0.sigma_scale, np_sig);
    cc.sigma_node = inj(g->C0.sigma_node, np_sn);
    cc.b_scale = inj(g->C0.b_scale, np_bs);
    cc.b_node = inj(g->C0.b_node, np_bn);
    cc.c_node = inj(g->C0.c_node, np_c);
    cc.f_feat = inj(g->C0.f_feat, np_f);
    CKL();
    TRY(hjb_set_coeffs(c, &cc));
    g->child_dirty = false;
  }
  TRY(hjb_set_source(c, g->Q > 0 ? g->h_fb.data() : nullptr, g->h_fc.data()));  // f at t_n
  *out = c;
  return HJB_OK;
}

// dU (in: the iterate with psi(t_n) on its boundary) <- the prolonged solution of the step on the
// nested coarse grid (itself started from its own nested grid), interior entries only
static hjb_status nested_guess(hjb_grid* g, double dt, const double* dprev, double* dU, const hjb_solve_params* sp,
                               hjb_step_stats* S) {
  hjb_grid* c;
  TRY(nested_child(g, sp, &c));
  if (!c) return HJB_OK;
  TRY(check_dt(c, dt));
  const int64_t f = 1LL << g->child_m, nc = c->n;
  const int64_t Nc = c->N;
  const int nb = (int)std::min<int64_t>((Nc + 255) / 256, (int64_t)g->sms * 8);
  const int D = g->D;
  if (D == 2) {
    LAUNCH(HJB_KC_TRANSFER, Nc, 16.0 * Nc, 0, k_nest_inject<2><<<nb, 256, 0, g->st>>>(g->n, nc, (int)f, dU, g->N, g->child_U, Nc, 1));
    LAUNCH(HJB_KC_TRANSFER, Nc, 16.0 * Nc, 0, k_nest_inject<2><<<nb, 256, 0, g->st>>>(g->n, nc, (int)f, dprev, g->N, g->child_prev, Nc, 1));
  } else {
    LAUNCH(HJB_KC_TRANSFER, Nc, 16.0 * Nc, 0, k_nest_inject<3><<<nb, 256, 0, g->st>>>(g->n, nc, (int)f, dU, g->N, g->child_U, Nc, 1));
    LAUNCH(HJB_KC_TRANSFER, Nc, 16.0 * Nc, 0, k_nest_inject<3><<<nb, 256, 0, g->st>>>(g->n, nc, (int)f, dprev, g->N, g->child_prev, Nc, 1));
  }
  CKL();
  hjb_step_stats Sc{};
  TRY(nested_guess(c, dt, g->child_prev, g->child_U, sp, &Sc));
  const hjb_status r = implicit_pi(c, dt, g->child_prev, g->child_U, g->child_pol, sp, Sc);
  if (r != HJB_OK && r != HJB_ERR_NOT_CONVERGED) return r;  // an unconverged coarse iterate is still a guess
  S->nested_pi_iters += Sc.pi_iters + Sc.nested_pi_iters;
  const int64_t Nf = g->N;
  const int nbf = (int)std::min<int64_t>((Nf + 255) / 256, (int64_t)g->sms * 8);
  if (sp->nested_increment) {  // U^{n-1} + P (U_c^n - U_c^{n-1})
    if (D == 2)
      LAUNCH(HJB_KC_TRANSFER, Nf, 16.0 * Nf + 16.0 * Nc, 0,
             k_nest_prolong_inc<2><<<nbf, 256, 0, g->st>>>(g->n, nc, (int)f, g->child_U, g->child_prev, dprev, dU));
    else
      LAUNCH(HJB_KC_TRANSFER, Nf, 16.0 * Nf + 16.0 * Nc, 0,
             k_nest_prolong_inc<3><<<nbf, 256, 0, g->st>>>(g->n, nc, (int)f, g->child_U, g->child_prev, dprev, dU));
  } else if (D == 2) {
    LAUNCH(HJB_KC_TRANSFER, Nf, 8.0 * Nf + 8.0 * Nc, 0, k_nest_prolong<2><<<nbf, 256, 0, g->st>>>(g->n, nc, (int)f, g->child_U, dU));
  } else {
    LAUNCH(HJB_KC_TRANSFER, Nf, 8.0 * Nf + 8.0 * Nc, 0, k_nest_prolong<3><<<nbf, 256, 0, g->st>>>(g->n, nc, (int)f, g->child_U, dU));
  }
  CKL();
  return HJB_OK;
}

// ---------------------------------------------------------------------------- API: instrumentation
extern "C" hjb_status hjb_profile_reset(hjb_grid_t g, int32_t time_kernels) {
  if (!g) return fail(HJB_ERR_INVALID_ARG, "null handle");
  CK(cudaSetDevice(g->desc.device));
  prof_drain(g);
  g->prof = hjb_profile{};
  g->prof_timing = time_kernels != 0;
  g->prof.timed = g->prof_timing ? 1 : 0;
  if (g->child) TRY(hjb_profile_reset(g->child, time_kernels));
  return HJB_OK;
}

extern "C" hjb_status hjb_profile_read(hjb_grid_t g, hjb_profile* out) {
  if (!g || !out) return fail(HJB_ERR_INVALID_ARG, "null handle/out");
  CK(cudaSetDevice(g->desc.device));
  prof_drain(g);
  CK(cudaStreamSynchronize(g->st));
  *out = g->prof;
  if (g->child) {  // the nested coarse solves: one class of this grid's profile (their own grid's
                   // work, kept apart from the per-kernel roofline classes of this grid)
    hjb_profile c;
    TRY(hjb_profile_read(g->child, &c));
    for (int k = 0; k < HJB_KC_COUNT; ++k) {
      out->launches[HJB_KC_NESTED] += c.launches[k];
      out->ms[HJB_KC_NESTED] += c.ms[k];
      out->bytes[HJB_KC_NESTED] += c.bytes[k];
      out->flops[HJB_KC_NESTED] += c.flops[k];
    }
    out->calls[HJB_KC_NESTED] += c.calls[HJB_KC_SEARCH];
    out->nodes[HJB_KC_NESTED] += c.nodes[HJB_KC_SEARCH];
    out->total_launches += c.total_launches;
    out->graph_launches += c.graph_launches;
    out->graph_kernels += c.graph_kernels;
  }
  return HJB_OK;
}
