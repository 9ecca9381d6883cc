/*
 * hjb.h -- C-ABI of libhjb: the B200-native hot path of the implicit semi-Lagrangian
 * (LISL, Scheme 2 with boundary truncation) discretisation of the HJB equation
 *
 *     u_t - inf_a { L^a u + c^a u + f^a } = 0  in (0,T] x Omega,  u(0,.) = g,  u = psi on dOmega
 *     L^a u = tr[a^a D^2 u] + b^a . Du,   a^a = 1/2 sigma^a sigma^a^T,  sigma^a in R^{d x P}
 *                                                          (arXiv:1605.04821)
 *
 * one implicit Euler step (theta = 1) solved by policy iteration: a per-node
 * exhaustive control search, then a GMG-preconditioned BiCGSTAB solve of the policy system.
 * All arithmetic is fp64 and runs in sm_100a kernels; there is no CPU fallback.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  Grid:    Omega = [lo,hi]^d, d in {2,3}, n nodes per dimension including the boundary,
 *           h = (hi-lo)/(n-1), node x_i = lo + i*h.  Flat index lexicographic, x1 fastest.
 *  Layout:  every per-node array ("grid array") is a DEVICE array of hjb_layout.local_elems
 *           fp64 (or u8) elements holding the local slab rows [local_row0, local_row0+local_rows)
 *           of the slowest axis; with nranks == 1 this is simply the full n^d grid.
 *  Boundary: Dirichlet nodes are identity rows (reading ix in DESIGN.md); their values in U are
 *           psi(t_n) and the stencil interpolates them (truncated endpoints land on dOmega,
 *           PAPER.md:216-227, interpolate-at-boundary mode of PAPER.md:387-432).
 *  Streams: all work is enqueued on desc.stream (a cudaStream_t, 0 = legacy default).  Calls
 *           that return statistics synchronise that stream.
 *  Host buffers: hjb_step accepts host (pageable or pinned) pointers for U_prev/U/policy/psi
 *           and stages them through device memory inside the call (used by the e2e benchmark).
 *  Errors:  every call returns an hjb_status, never aborts; hjb_last_error() gives a message
 *           (thread-local, valid until the next call on that thread).
 *  Ownership: the handle and all workspaces (Krylov vectors, multigrid levels) are owned by the
 *           library from hjb_grid_create until hjb_grid_destroy.  Caller arrays stay caller-owned;
 *           hjb_set_coeffs RETAINS the device field pointers (not copied) until the next
 *           hjb_set_coeffs or hjb_grid_destroy.
 */
#ifndef HJB_H
#define HJB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HJB_VERSION 1
#define HJB_MAX_K 255
#define HJB_MAX_Q 16
#define HJB_MAX_PI_LOG 64

typedef struct hjb_grid* hjb_grid_t;

typedef enum {
  HJB_OK = 0,
  HJB_ERR_INVALID_ARG = 1,   /* null handle/pointer, d not in {2,3}, P > d, K not in [1,255],
                                Q > 16, n < 3, hi <= lo, dt <= 0, dt*max(c) >= 1 */
  HJB_ERR_UNSUPPORTED = 2,   /* multigrid on n != 2^l+1, nranks > 1 without NCCL support     */
  HJB_ERR_STATE = 3,         /* apply/search/step before hjb_set_coeffs; solve before mg_setup */
  HJB_ERR_OOM = 4,
  HJB_ERR_CUDA = 5,
  HJB_ERR_NCCL = 6,
  HJB_ERR_NOT_CONVERGED = 7, /* Krylov or policy iteration hit max iterations; U holds the best iterate */
  HJB_ERR_BREAKDOWN = 8,     /* BiCGSTAB (r_hat, v) == 0, rho == 0 or omega == 0 in the last of
                                its restarts (x is never updated with a non-finite coefficient) */
  HJB_ERR_NONFINITE = 9      /* NaN/Inf in a residual */
} hjb_status;

const char* hjb_last_error(void);
int32_t hjb_version(void);

/* ------------------------------------------------------------------------------ grid */
typedef struct {
  int32_t dim;         /* d in {2,3}                                                          */
  int32_t P;           /* columns of sigma, 1 <= P <= d                                       */
  int32_t K;           /* number of discrete controls, 1..255 (policy stored as uint8)        */
  int32_t Q;           /* number of source features f_feat, 0..16                             */
  int64_t n;           /* nodes per dimension incl. boundary, >= 3                            */
  double lo, hi;       /* Omega = [lo,hi]^d                                                   */
  int32_t rank;        /* slab decomposition along the slowest axis: this rank ...           */
  int32_t nranks;      /* ... of nranks (see hjb_partition)                                  */
  const void* nccl_id; /* nranks > 1: 128 bytes, the ncclUniqueId (comm = HJB_COMM_NCCL, created
                          by rank 0 and broadcast by the caller) or any group key shared by the
                          ranks (comm = HJB_COMM_THREADS)                                      */
  void* stream;        /* cudaStream_t                                                        */
  int32_t device;      /* CUDA device ordinal                                                 */
  int64_t halo;        /* nranks > 1: halo rows per side (>= floor(max reach in rows) + 1)   */
  int32_t comm;        /* HJB_COMM_NCCL (default) or HJB_COMM_THREADS                         */
} hjb_grid_desc;

/* Communication backends for nranks > 1.  With nranks > 1 EVERY call on a grid is collective:
 * all ranks must make the same calls in the same order.                                       */
#define HJB_COMM_NCCL 0     /* one process per GPU, NCCL over NVLink/NVSwitch (production)    */
#define HJB_COMM_THREADS 1  /* TEST-ONLY: ranks are host threads of one process on one device;
                               halos by device copies ordered with CUDA events               */

typedef struct {
  int64_t n;            /* nodes per dimension                                                */
  int64_t row_elems;    /* elements per slab row = n^(d-1)                                    */
  int64_t row0, row1;   /* owned rows [row0,row1) of the slowest axis (global indices)        */
  int64_t halo;         /* halo rows held on each side (0 when nranks == 1)                   */
  int64_t local_row0;   /* global row of local row 0 (= row0 - halo)                          */
  int64_t local_rows;   /* rows in every grid array                                           */
  int64_t local_elems;  /* local_rows * row_elems: length of every grid array                 */
  int64_t n_interior;   /* interior unknowns owned by this rank                               */
  int64_t n_boundary;   /* boundary nodes of the full grid (length of the packed psi array)   */
  int32_t n_levels;     /* multigrid levels after hjb_mg_setup (0 before)                     */
  double h, k;          /* mesh width and SL step k = sqrt(h)                   */
} hjb_layout;

/* Slab decomposition (host-only, no GPU needed; the same functions hjb_grid_create uses).
 * The n-2 interior rows of the slowest axis are split into nranks contiguous blocks,
 * rank r owning interior rows [1 + floor(r (n-2)/R), 1 + floor((r+1)(n-2)/R)).  Local arrays
 * hold the owned rows plus `halo` rows on each side, clipped to [0, n): the Dirichlet rows 0 and
 * n-1 live in the halo region of the first/last rank.  Every rank must own >= halo rows (so a halo
 * comes from one neighbour), else HJB_ERR_INVALID_ARG.  halo must be >= floor(max |offset| of a
 * stencil endpoint along the slowest axis, in cells) + 1 (the interpolation cell of an endpoint at
 * row i + o spans rows floor(i+o) .. floor(i+o)+1); hjb_set_coeffs checks this on the device.
 * nranks == 1: one slab, halo ignored (0).                                                      */
hjb_status hjb_partition(int32_t dim, int64_t n, int32_t nranks, int32_t rank, int64_t halo,
                         hjb_layout* out);

typedef struct {
  int32_t peer;        /* neighbour rank                                                       */
  int64_t send_row;    /* first GLOBAL row sent to peer (owned rows of this rank)              */
  int64_t recv_row;    /* first GLOBAL row received from peer (lands in this rank's halo)      */
  int64_t rows;        /* rows per message (= halo)                                           */
} hjb_halo_msg;

/* The halo messages of `rank` (0, 1 or 2: to rank-1 and rank+1), in that order. */
hjb_status hjb_halo_plan(int32_t dim, int64_t n, int32_t nranks, int32_t rank, int64_t halo,
                         hjb_halo_msg out[2], int32_t* count);

/* A fresh ncclUniqueId (128 bytes) for nranks > 1 with HJB_COMM_NCCL: rank 0 calls this and the
 * caller broadcasts the bytes to every rank (e.g. torch.distributed.broadcast_object_list).     */
hjb_status hjb_comm_unique_id(void* out128);

/* Create a grid handle; allocates the Krylov workspace (about 10 grid arrays).  With nranks > 1
 * this is collective (it initialises the communicator).                                        */
hjb_status hjb_grid_create(const hjb_grid_desc* desc, hjb_grid_t* out);
hjb_status hjb_grid_query(hjb_grid_t g, hjb_layout* out);
hjb_status hjb_grid_destroy(hjb_grid_t g);

/* ------------------------------------------------------------------------ coefficients
 * Affine-separable coefficient model (covers PAPER.md Problems A/B and every BASELINE config):
 *   sigma^a_p(x) = sigma_scale[p](x) * sigma_dir[a][p][:] + sigma_node[p][:](x)
 *   b^a(x)       = b_scale(x) * b_dir[a][:] + b_node[:](x)
 *   c^a(x)       = c_node(x) + c_ctrl[a]            (dt * max c < 1 is required)
 *   f^a(x)       = f_ctrl[a] + sum_q f_basis[a][q] * f_feat[q](x)
 * Tables (sigma_dir [K][P][d], b_dir [K][d], c_ctrl [K], f_basis [K][Q], f_ctrl [K] or NULL)
 * are HOST arrays, copied.  Fields are DEVICE grid arrays (plane stride = local_elems), NULL =
 * absent (scales default to 1, offsets to 0); they are retained, not copied.  Only the owned
 * entries of a field are read.                                                              */
typedef struct {
  const double* sigma_dir;
  const double* b_dir;
  const double* c_ctrl;
  const double* f_basis;
  const double* f_ctrl;
  const double* sigma_scale; /* [P][local_elems] */
  const double* sigma_node;  /* [P][d][local_elems] */
  const double* b_scale;     /* [local_elems] */
  const double* b_node;      /* [d][local_elems] */
  const double* c_node;      /* [local_elems] */
  const double* f_feat;      /* [Q][local_elems] */
} hjb_coeffs;

hjb_status hjb_set_coeffs(hjb_grid_t g, const hjb_coeffs* c);
/* Replace only the (time-dependent) source tables f_basis [K][Q] and f_ctrl [K] (host). */
hjb_status hjb_set_source(hjb_grid_t g, const double* f_basis, const double* f_ctrl);

/* --------------------------------------------------------------------- policy improvement
 * For every owned interior node j and every control a (in index order) evaluate
 *   H^a_j(U) = L_hat^a[U](x_j) + c^a_j U_j + f^a_j          (eq. Lhat)
 * and take the lowest-index argmin, which is the row-wise argmax of the positive-type residual
 * max_a (A^a U - F^a)_j (derivation D1 in DESIGN.md).  Writes
 *   policy[j] (in: previous policy, out: new), F[j] = U_prev_j + dt f^{policy_j}_j,
 * and returns R = max_j |U_j - U_prev_j - dt min_a H^a_j| and the number of changed entries.
 * U must hold psi on boundary nodes.  Non-interior entries of policy/F are not written.     */
typedef struct {
  int64_t changed;   /* nodes whose policy changed */
  double R_max;      /* nonlinear residual max_j |max_a (A^a U - F^a)_j| */
} hjb_pi_stats;

hjb_status hjb_policy_update(hjb_grid_t g, double dt, const double* U, const double* U_prev,
                             uint8_t* policy, double* F, hjb_pi_stats* out);

/* ---------------------------------------------------------------- policy operator apply
 * y = A^pi x matrix-free (theta = 1):
 *   (A x)_j = x_j - dt [ sum_e w_e (I x(z_e) - x_j) + c^{pi_j}_j x_j ]   at interior nodes,
 *   y_j = x_j at boundary nodes (identity rows).
 * w_e = A_p/(2h), B_p/(2h) for the 2P truncated diffusion endpoints and 1/(mu_d h) for the drift
 * endpoint.  x is read on the full local grid (boundary values as given).   */
hjb_status hjb_apply(hjb_grid_t g, double dt, const uint8_t* policy, const double* x, double* y);

/* ------------------------------------------------------------------------ multigrid
 * Geometric multigrid for A^pi (NS: damped Jacobi smoother, full-weighting restriction,
 * bilinear/trilinear prolongation, coarse operators REDISCRETISED from the injected policy;
 * PAPER.md:932-937 is the paper's Galerkin variant).  Requires n = 2^l + 1.                   */
typedef struct {
  int32_t nu_pre, nu_post;   /* smoothing sweeps (default 2, 2)                               */
  double omega;              /* Jacobi damping in (0,1] (default 1.0; Gershgorin-safe)        */
  int32_t coarse_max_n;      /* coarsen while n > coarse_max_n (default 9 in 2D, 5 in 3D)    */
  int32_t coarse_k_mode;     /* 0: coarse levels keep the fine SL step k (default);
                                1: k_l = sqrt(h_l) (the scheme's own rule on each level)      */
  int32_t max_levels;        /* cap on levels (default 32)                                     */
  int32_t gather_n;          /* nranks > 1: levels with n <= gather_n (or slabs thinner than
                                their halo) are replicated on every rank after an all-gather
                                (default 129 in 2D, 33 in 3D; BASELINE cfg4 "129^2 on one GPU") */
  int32_t gamma;             /* cycle index on the large levels: 1 = V-cycle, 2 = W-cycle (the
                                coarse correction of level l is refined by gamma - 1 further
                                cycles on the residual of level l+1); default 2 in 2D, 1 in 3D */
  int32_t gamma_min_nodes;   /* revisit level l+1 only if it owns >= gamma_min_nodes interior
                                nodes (smaller levels are launch-latency bound: plain V there);
                                default 131072                                                */
  int32_t coarse_op;         /* 0: coarse operators rediscretised on each level with the injected
                                policy (NS, default); 1: Galerkin A_{l+1} = R A_l P (PAPER.md:935,
                                "constructed using the Galerkin principle"),
                                stored ELL (<= 96 entries per row), 2D on one rank only
                                (HJB_ERR_UNSUPPORTED otherwise)                               */
  int32_t precision;         /* element type of the cycle's vectors: 0 = fp64, 1 = fp32 (default)
                                (iterates, right-hand sides, residuals and the stored diagonal of
                                every level in fp32; geometry, weights and row sums in fp64;
                                b converted on entry, M^{-1} b returned in fp64).  The cycle is
                                only the preconditioner: BiCGSTAB's residuals, stopping tests and
                                iterate stay fp64 (reading xxxi).  coarse_op = 0
                                only (the Galerkin cycle runs in fp64).  Measured at cfg4: one
                                cycle 66.6 -> 57.2 ms, the same Krylov iteration counts.       */
} hjb_mg_params;

void hjb_mg_params_default(int32_t dim, hjb_mg_params* out);
hjb_status hjb_mg_setup(hjb_grid_t g, double dt, const uint8_t* policy, const hjb_mg_params* p);
/* x = M^{-1} b: one (nu_pre, nu_post) cycle of index gamma from x = 0 (interior entries; boundary
   of x = 0). */
hjb_status hjb_mg_apply(hjb_grid_t g, const double* b, double* x);

/* --------------------------------------------------------------------------- solve
 * Policy evaluation A^pi X = F: right-preconditioned BiCGSTAB with one
 * V-cycle per preconditioner application, from x (in: initial guess with boundary = psi,
 * out: solution), stopping at ||F - A X||_2 <= rtol ||F||_2 over interior rows (BJ cfg1).     */
typedef struct {
  double krylov_rtol;        /* 1e-12 */
  int32_t krylov_maxit;      /* 2000 */
  int32_t use_mg;            /* 1 = GMG preconditioner, 0 = none */
  double tol_pi;             /* policy-iteration stop: R <= tol_pi (1e-10) */
  int32_t max_pi;            /* 50 */
  hjb_mg_params mg;
  double pi_forcing;         /* inexact policy iteration (hjb_step only): while the policy still
                                changes, each policy evaluation stops at ||r||_2 <= max(krylov_rtol
                                ||F||_2, pi_forcing ||r_0||_2); a policy found stable after an
                                inexact evaluation is re-evaluated exactly before the step ends, so
                                the fixed point is unchanged (DESIGN.md §3 reading xxii).
                                0 = exact evaluation every iteration (the paper's Howard loop);
                                default 0.01 (with the W-cycle measured best at cfg4 among
                                0 / 0.003 / 0.01 / 0.03 / 0.1: 2071 / 1466 / 1441 / 1696 / 1700 ms). */
  int32_t guess;             /* hjb_step's initial iterate (the fixed point does not depend on it):
                                HJB_GUESS_PREV (default): U_prev, as the paper's time march;
                                HJB_GUESS_GIVEN: U as passed by the caller;
                                HJB_GUESS_EXTRAPOLATE: U holds U^{n-2} on entry and the iterate is
                                2 U_prev - U^{n-2} (linear extrapolation in time, DESIGN.md xxiv);
                                HJB_GUESS_NESTED: nested iteration -- the same step is first solved
                                on the grid coarsened 2^nested_coarsen times per axis (own h and
                                k = sqrt(h); fields, U_prev and psi(t_n) injected from
                                coincident nodes; recursively nested while the next grid keeps
                                n >= nested_min_n) and its solution, prolonged multilinearly, is
                                the iterate (reading xxx).  Needs (n-1) divisible by
                                2^nested_coarsen, one rank, the interpolation boundary mode and
                                theta = 1; otherwise it falls back to HJB_GUESS_PREV.
                                Boundary entries are always set to psi(t_n) (if given).         */
  double krylov_rtol_inf;    /* secondary stop of an EXACT evaluation: also ||F - A X||_inf <=
                                krylov_rtol_inf ||F||_inf (default 1e-9; 0 = off).  The 2-norm rule
                                alone bounds ||r||_inf only by sqrt(N) krylov_rtol ||F||_2 (SURVEY
                                §8c-xvii; reading xvii).  Inexact evaluations (pi_forcing)
                                use the 2-norm rule only.                                       */
  double theta;              /* hjb_step's time scheme (eq. FullScheme):
                                1 = implicit Euler (default, the paper's experiments); 0 = explicit
                                Euler: U^n = U^{n-1} + dt min_a H^a(U^{n-1}), one control search and
                                one apply, no solve; 0 < theta < 1: policy iteration on
                                (I - theta dt (L^pi + c)) U = U^{n-1} + (1-theta) dt (L^pi + c) U^{n-1}
                                + dt f^pi, each policy from the search at theta U + (1-theta) U^{n-1}
                                (reading xxvi).  f must be set at t_{n-1} + theta dt
                                (P:124).  theta < 1 needs the CFL condition of Proposition CFL
                                (P:437-441), see hjb_cfl_rate; it is not enforced.               */
  int32_t solver;            /* policy evaluation: 0 = right-preconditioned BiCGSTAB with geometric
                                multigrid (default); 1 = flexible GCR(10) preconditioned by
                                aggregation AMG (SURVEY §8(f)
                                NEXT-1): the assembled operator, double pairwise aggregation,
                                K-cycle with 2 inner GCR iterations per coarse level.  One rank;
                                the setup is redone per policy.  Same stopping rules.           */
  int32_t nested_coarsen;    /* HJB_GUESS_NESTED: 2^nested_coarsen coarsening per axis (default 2) */
  int32_t nested_min_n;      /* HJB_GUESS_NESTED: nest only onto grids with n >= nested_min_n
                                (default 513)                                                   */
  int32_t nested_increment;  /* HJB_GUESS_NESTED: 0 = the prolonged coarse solution (default);
                                1 = U_prev + the prolonged coarse time increment U_c^n - U_c^{n-1}
                                (keeps the fine grid's U_prev, takes only the change from the
                                coarse step)                                                    */
} hjb_solve_params;

#define HJB_GUESS_PREV 0
#define HJB_GUESS_GIVEN 1
#define HJB_GUESS_EXTRAPOLATE 2
#define HJB_GUESS_NESTED 3

typedef struct {
  int32_t iters;             /* BiCGSTAB iterations */
  double rres;               /* final true relative residual ||F - A X||_2 / ||F||_2 */
  double rres_inf;           /* ||F - A X||_inf / ||F||_inf */
} hjb_solve_stats;

void hjb_solve_params_default(int32_t dim, hjb_solve_params* out);
hjb_status hjb_solve(hjb_grid_t g, double dt, const uint8_t* policy, const double* F, double* x,
                     const hjb_solve_params* p, hjb_solve_stats* out);

/* ---------------------------------------------------------------------------- step
 * One implicit Euler step t_{n-1} -> t_n = t_{n-1} + dt by policy iteration:
 *   U <- initial iterate (hjb_solve_params.guess; default U_prev) with boundary entries psi(t_n)
 *   (psi_packed: the n_boundary boundary values in lexicographic order; NULL keeps U's boundary
 *   entries), then repeat
 *     policy improvement (hjb_policy_update) -> stop if it > 1 and (changed == 0 or R <= tol_pi)
 *     -> mg setup -> BiCGSTAB solve of A^pi U = F^pi from the current U.
 * The initial policy is the greedy policy at U_prev (reading iii).  f must already be
 * at t_n (hjb_set_source).  policy may be NULL (internal buffer).  Pointers may be host.      */
typedef struct {
  int32_t pi_iters;                          /* policy evaluations (linear solves) performed */
  int32_t krylov_iters_total;
  int32_t krylov_iters[HJB_MAX_PI_LOG];      /* per policy iteration */
  int64_t changed[HJB_MAX_PI_LOG];           /* policy changes seen by each search */
  double R[HJB_MAX_PI_LOG];                  /* nonlinear residual seen by each search */
  double final_R;
  double final_rres;                         /* true relative residual of the last solve */
  double ms_search, ms_setup, ms_solve;      /* device time per phase (CUDA events) */
  int32_t n_levels;
  double final_rres_inf;                     /* ||F - A X||_inf / ||F||_inf of the last solve */
  int32_t nested_pi_iters;                   /* HJB_GUESS_NESTED: policy iterations on the coarser
                                                grids (all nesting levels) */
  double ms_nested;                          /* device time of the nested coarse solves */
} hjb_step_stats;

/* U may alias U_prev (in-place step): U_prev is then copied to an internal buffer first.    */
hjb_status hjb_step(hjb_grid_t g, double dt, const double* U_prev, double* U, uint8_t* policy,
                    const double* psi_packed, const hjb_solve_params* p, hjb_step_stats* out);

/* Exact-psi boundary mode (PAPER.md Remark rhs): a truncated
 * stencil endpoint lies on dOmega; by default (reading i) it takes the multilinear interpolation of
 * the nodal boundary values psi(t_n) held in U.  With samples != NULL it takes psi(t_n, z) itself,
 * reconstructed from samples of psi on the faces at spacing h / refine by cubic (2D) / bicubic (3D)
 * Lagrange interpolation along the face (error O((h/refine)^4): below fp64 rounding for the BJ
 * grids with refine >= 64 in 2D).  samples: DEVICE array, retained (the caller refreshes its
 * contents for every t_n), layout [2 d][M^(d-1)], M = refine (n - 1) + 1, face 2 d + side (side 0:
 * x_d = lo, 1: x_d = hi), along-face axes in increasing order, the first fastest.  Affects the
 * control search (hjb_policy_update, hjb_step) and the residuals of U (hjb_solve, hjb_step); the
 * system matrix is unchanged (a truncated endpoint couples to boundary nodes only).  theta = 1 only.
 * samples == NULL: back to interpolation.                                                      */
hjb_status hjb_set_boundary_samples(hjb_grid_t g, int32_t refine, const double* samples);

/* Positivity (CFL) rate of Proposition CFL (eq. CFL_trunc): the largest
 *   sum_{p=1}^{P+1} (A^a_p + B^a_p) / (2 dx) - c^a_j
 * over owned interior nodes j (truncated weights included, so it grows like dx^{-3/2} / dx^{-2}
 * where one / both sides of a stencil overstep, Corollary CFL P:444-452) and over the control of
 * each node (policy != NULL, device array) or over every control (policy == NULL).  A theta-step
 * is of positive type if (1 - theta) dt * rate <= 1 and theta dt max c <= 1.  Collective (max over
 * ranks).                                                                                       */
hjb_status hjb_cfl_rate(hjb_grid_t g, const uint8_t* policy, double* rate);

/* ------------------------------------------------------------------- instrumentation
 * Every kernel launch of the library is counted per class.  With time_kernels != 0 each launch
 * over >= 16384 nodes (and every control search) is also bracketed by CUDA events on the grid's
 * stream and its device time summed per class (the events add ~2 us of host work per launch; off
 * by default); smaller launches -- the launch-latency-bound small multigrid levels -- are then
 * counted in `launches` only, not in calls / bytes / flops / nodes, so every class total is the
 * timed subset and their device time is the unattributed remainder.  `bytes` is the ALGORITHMIC
 * HBM traffic of the launches (the per-node formulas of DESIGN.md §6 times the nodes each launch
 * processed), `flops` the algorithmic fp64 operations, so that bytes/ms and
 * flops/ms are roofline numerators.  Counters are per handle; reset clears them.              */
typedef enum {
  HJB_KC_SEARCH = 0,    /* control search (policy improvement)                               */
  HJB_KC_APPLY = 1,     /* y = A x on the fine level (Krylov operator, hjb_apply)            */
  HJB_KC_RESID = 2,     /* r = b - A x on the fine level                                     */
  HJB_KC_SMOOTH = 3,    /* damped-Jacobi sweeps on the fine level                            */
  HJB_KC_TRANSFER = 4,  /* restriction, prolongation, policy/field injection                 */
  HJB_KC_COARSE = 5,    /* coarsest-level dense assemble / invert / solve                    */
  HJB_KC_VECTOR = 6,    /* BiCGSTAB vector updates with fused dot products, norms, copies    */
  HJB_KC_REDUCE = 7,    /* fixed-order reduction of block partials + Krylov scalar update    */
  HJB_KC_BOUNDARY = 8,  /* Dirichlet data scatter, halo check                                */
  HJB_KC_MG_COARSE = 9, /* residual / Jacobi sweeps on coarse multigrid levels               */
  HJB_KC_NESTED = 10,   /* everything the nested coarse grids of HJB_GUESS_NESTED launched      */
  HJB_KC_COUNT = 11
} hjb_kernel_class;

typedef struct {
  int64_t launches[HJB_KC_COUNT];   /* kernel launches (one operator application may be several:
                                       the deep-rectangle kernel + boundary-layer strips)        */
  int64_t calls[HJB_KC_COUNT];      /* logical applications (operator sweeps, searches, ...)      */
  double ms[HJB_KC_COUNT];
  double bytes[HJB_KC_COUNT];
  double flops[HJB_KC_COUNT];
  double nodes[HJB_KC_COUNT];
  int64_t total_launches;   /* kernels executed (a replayed graph counts every kernel it holds) */
  int32_t timed;            /* 1 if ms[] was collected */
  int64_t graph_launches;   /* cudaGraphLaunch calls of the captured multigrid tail:
                               the cycle from the first level owning <= 70000 nodes down is captured
                               once per hierarchy and replayed; its kernels are untimed             */
  int64_t graph_kernels;    /* kernels executed inside those graph replays (host launch calls =
                               total_launches - graph_kernels + graph_launches)                   */
} hjb_profile;

hjb_status hjb_profile_reset(hjb_grid_t g, int32_t time_kernels);
hjb_status hjb_profile_read(hjb_grid_t g, hjb_profile* out);   /* synchronises the stream */

#ifdef __cplusplus
}
#endif
#endif /* HJB_H */
