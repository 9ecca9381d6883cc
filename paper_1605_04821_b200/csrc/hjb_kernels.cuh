// hjb_kernels.cuh -- __global__ kernels of the hot path (sm_100a, fp64).
#pragma once
#include <type_traits>

#include "hjb_device.cuh"

namespace hjb {

// every owned interior node of level L with (BX x BY) blocks
#define FOR_INTERIOR_B(L, BX, BY)                                                            \
  for (int row = blockIdx.y * (BY) + threadIdx.y; row < (L).nrows; row += gridDim.y * (BY)) \
    for (int col = blockIdx.x * (BX) + threadIdx.x; col < (L).nI; col += gridDim.x * (BX))

// every owned interior node of level L: (col, row) -> x1 index 1+col, line `row`
#define FOR_INTERIOR(L)                                                       \
  for (int row = blockIdx.y * kBY + threadIdx.y; row < (L).nrows; row += gridDim.y * kBY) \
    for (int col = blockIdx.x * kBX + threadIdx.x; col < (L).nI; col += gridDim.x * kBX)

// ================================================================== operator-family kernel
enum OpMode : int {
  OP_APPLY = 0,    // y = A x                    (+ optional dots with y)
  OP_RESID = 1,    // y = b - A x                (+ optional dots)
  OP_JACOBI = 2,   // y = x + omega (b - A x) / D
  OP_JACOBI0 = 3,  // y = omega b / D            (x = 0; geometry only, no gathers)
  OP_DIAG = 4,     // y = D = 1 + dt (sum_e w_e - self - c)   (MG setup: stored per level)
  OP_JACOBI_D = 5, // OP_JACOBI with D read from the stored diagonal (passed as u): no self weights
};

// NDOT: 0, 1 -> partial[0] = sum y*u ; 2 -> partial[0] = sum y*u, partial[1] = sum y*y
#ifndef HJB_OP_MINB
#define HJB_OP_MINB 4   // <= 128 registers: 16 resident warps per SM (measured best, profiles/r01_v3)
#endif
#ifndef HJB_OP_ILP
#define HJB_OP_ILP 1
#endif
#ifndef HJB_SEARCH_MINB
#define HJB_SEARCH_MINB 3  // general search: 168 registers (spills only in the truncation path): cfg3 -5 %
#endif
// Every node of the rectangle `it` (loop coordinates).  DEEP: `it` lies in the deep rectangle (all
// endpoints of every control strictly inside the box) -> the lean fast path, no truncation code.
#ifndef HJB_OP_DEEP_MINB
#define HJB_OP_DEEP_MINB 6  // lean deep kernels fit 80 registers: 24 resident warps (cfg4 sweep -17 %)
#endif
// residual sweeps and the Krylov applies with fused dot products spill at 80 registers: 96 (5 CTAs)
// for those (cfg4 fine residual 8.3 -> 7.4 ms, coarse sweeps -5 %); Jacobi and the plain apply keep 80
template <int MODE, int NDOT>
constexpr int op_deep_minb() { return (MODE == OP_RESID || NDOT > 0) ? HJB_OP_DEEP_MINB - 1 : HJB_OP_DEEP_MINB; }
// fp32 cycle vectors (hjb_mg_params.precision = 1): half the registers per gathered corner
#ifndef HJB_OP_DEEP_MINB_F32
#define HJB_OP_DEEP_MINB_F32 7  // 72 registers, 28 resident warps: cfg4 step 1605 -> 1563 ms (8: 1575; r02_t)
#endif
template <int MODE, int NDOT, typename V>
constexpr int op_deep_minb_v() {
  return std::is_same<V, double>::value ? op_deep_minb<MODE, NDOT>()
                                        : ((MODE == OP_JACOBI_D || MODE == OP_JACOBI || MODE == OP_JACOBI0)
                                               ? HJB_OP_DEEP_MINB_F32 : op_deep_minb<MODE, NDOT>());
}
// V: element type of x, b, y and the stored diagonal u (double; float for the fp32 multigrid
// vectors of hjb_mg_params.precision = 1 -- geometry and accumulation stay fp64)
template <int D, int P, int MODE, int NDOT, bool DEEP, typename V = double>
__global__ void __launch_bounds__(kTX, (DEEP && D == 2) ? op_deep_minb_v<MODE, NDOT, V>() : HJB_OP_MINB) k_operator(LevelDev L, CoefDev C, double dt, double omega,
                                                  const uint8_t* __restrict__ pol,
                                                  const V* __restrict__ x,
                                                  const V* __restrict__ b, V* __restrict__ y,
                                                  const V* __restrict__ u, double* partial,
                                                  SkipRect it) {
  constexpr bool GATHER = (MODE != OP_JACOBI0 && MODE != OP_DIAG);
  constexpr bool SELF = (MODE == OP_JACOBI || MODE == OP_JACOBI0 || MODE == OP_DIAG);
  constexpr int E = 2 * P + 1;
  constexpr bool XJ = GATHER;
  constexpr bool BJ = (MODE != OP_APPLY && MODE != OP_DIAG);
  extern __shared__ double tab[];
  stage_tables<D, P, false>(C, tab);
  const double* tsd = tab;
  const double* tbd = tab + C.K * P * D;
  const double* tcc = tbd + C.K * D;
  double dots[2] = {0.0, 0.0};
  const int nk = box_lines(it);
  // DEEP: ILP nodes per thread per pass (rows row, row + stride, ...): their loads and gathers are
  // in flight together (HJB_OP_ILP, default 1)
  constexpr int U = DEEP ? HJB_OP_ILP : 1;
  const int rstride = gridDim.y * kBY;
  auto pass = [&](int k0, int col, bool active) {
    NodeIn<D, P> in[U];
    bool ok[U];
    int rows[U];
#pragma unroll
    for (int v = 0; v < U; ++v) {
      ok[v] = active && k0 + v * rstride < nk;
      rows[v] = ok[v] ? box_row<D>(L, it, k0 + v * rstride) : 0;
      if (ok[v]) fetch_node<D, P, XJ, BJ, V>(L, C, pol, x, b, col, rows[v], in[v]);
    }
    Node<D> nd[U];
    Tap<D> taps[U][E];
    double wsum[U];
#pragma unroll
    for (int v = 0; v < U; ++v) {
      if (!ok[v]) continue;
      node_from<D, P>(L, col, rows[v], in[v], nd[v]);
      const int a = in[v].a;
      if (DEEP) {
        double o[P + 1][D];
        row_offsets<D, P>(L, tsd + a * P * D, tbd + a * D, nd[v], o);
        wsum[v] = row_geometry_fast<D, P>(L, nd[v], o, taps[v]);
      } else {
        wsum[v] = row_taps<D, P>(L, tsd + a * P * D, tbd + a * D, nd[v], taps[v]);
      }
    }
    double vals[U][E];
    if (GATHER) {
#pragma unroll
      for (int v = 0; v < U; ++v)
        if (ok[v])
#pragma unroll
          for (int e = 0; e < E; ++e) vals[v][e] = (DEEP || MODE != OP_RESID) ? tap_value<D>(L, x, taps[v][e])
                                                                           : tap_value_u<D>(L, C, x, taps[v][e]);
    }
#pragma unroll
    for (int v = 0; v < U; ++v) {
      if (!ok[v]) continue;
      double acc = 0.0, self = 0.0;
      if (GATHER) {
#pragma unroll
        for (int e = 0; e < E; ++e) acc = fma(taps[v][e].w, vals[v][e], acc);
      }
      if (SELF) {
#pragma unroll
        for (int e = 0; e < E; ++e) self += tap_self<D>(nd[v], taps[v][e]);
      }
      const double c = nd[v].cn + tcc[in[v].a];
      double out;
      if (MODE == OP_JACOBI0) {
        const double diag = 1.0 + dt * (wsum[v] - self - c);
        out = omega * in[v].bj / diag;
      } else if (MODE == OP_DIAG) {
        out = 1.0 + dt * (wsum[v] - self - c);
      } else {
        const double xj = in[v].xj;
        const double Ax = xj - dt * (acc - wsum[v] * xj + c * xj);
        if (MODE == OP_APPLY) {
          out = Ax;
        } else if (MODE == OP_RESID) {
          out = in[v].bj - Ax;
        } else {
          const double diag = (MODE == OP_JACOBI_D) ? (double)__ldg(u + nd[v].loc) : 1.0 + dt * (wsum[v] - self - c);
          out = xj + omega * (in[v].bj - Ax) / diag;
        }
      }
      y[nd[v].loc] = (V)out;
      if (NDOT >= 1 && MODE != OP_JACOBI_D) dots[0] = fma(out, (double)__ldg(u + nd[v].loc), dots[0]);
      if (NDOT >= 2) dots[1] = fma(out, out, dots[1]);
    }
  };
  // the general kernel (boundary-layer strips, small levels) walks its box as one packed index over
  // the (line, column) pairs, so that every lane has a node: the x1 strips are only reach-wide (4..143
  // columns on the cfg4 levels, against 128 lanes per CTA line)
  const int width = it.c1 - it.c0;
  if (!DEEP) {
    const int npk = nk * width;  // < 2^31: local arrays hold < 2^31 nodes
    const int step = gridDim.x * gridDim.y * kBX * kBY;
    for (int q = (blockIdx.y * gridDim.x + blockIdx.x) * (kBX * kBY) + threadIdx.y * kBX + threadIdx.x; q < npk;
         q += step) {
      const int k0 = q / width;
      pass(k0, it.c0 + (q - k0 * width), true);
    }
  } else {
    const int col = it.c0 + blockIdx.x * kBX + threadIdx.x;
    const bool active = col < it.c1;
    for (int k0 = blockIdx.y * kBY + threadIdx.y; k0 < nk; k0 += rstride * U) pass(k0, col, active);
  }
  if (NDOT > 0) block_reduce_store<2>(dots, partial);
}

// ================================================================== control search
// For every owned interior node: H^a = acc_a - wsum_a U_j + c^a U_j + f^a for all a (lowest-index
// argmin), policy/F outputs, partials: [max R, changed count].
// Every node of the rectangle `it` (loop coordinates).  DEEP: `it` lies in the deep rectangle -> the
// lean fast path.
#ifndef HJB_SEARCH_DEEP_MINB
#define HJB_SEARCH_DEEP_MINB 4  // 128 registers, no spills: cfg4 search 178 -> 156 ms
#endif
template <int D, int P, bool DEEP>
__global__ void __launch_bounds__(kTX, DEEP ? (D == 2 ? HJB_SEARCH_DEEP_MINB : 3) : HJB_SEARCH_MINB) k_search(LevelDev L, CoefDev C, double dt,
                                                const double* __restrict__ U,
                                                const double* __restrict__ Uprev,
                                                uint8_t* __restrict__ pol, double* __restrict__ F,
                                                double* partial, SkipRect it) {
  constexpr int E = 2 * P + 1;
  extern __shared__ double tab[];
  stage_tables<D, P, true>(C, tab);
  const double* tsd = tab;
  const double* tbd = tab + C.K * P * D;
  const double* tcc = tbd + C.K * D;
  const double* tfc = tcc + C.K;
  const double* tfb = tfc + C.K;
  double red[2] = {0.0, 0.0};
  const int nk = box_lines(it);
  // the general kernel (and any box narrower than a warp) walks its box as one packed index over
  // the (line, column) pairs, so every lane has a node: the boundary-layer strips along x1 are only
  // reach-wide (e.g. 8 of 32 lanes at cfg3)
  const int width = it.c1 - it.c0;
  auto node_work = [&](int k, int col) {
    const int row = box_row<D>(L, it, k);
    Node<D> nd;
    node_at<D>(L, col, row, nd);
    load_fields<D>(C, nd);
    prefetch_ahead(L, U, nd.loc, col);
    double feat[kMaxQ];
#pragma unroll
    for (int q = 0; q < kMaxQ; ++q) feat[q] = (q < C.Q) ? __ldg(C.f_feat + q * C.ld + nd.loc) : 0.0;
    const double Uj = __ldg(U + nd.loc);
    double best = INFINITY, fbest = 0.0;
    int arg = 0;
    // H^a_j = sum_e w_e I U(z_e) - wsum U_j + c^a_j U_j + f^a_j
    auto tail = [&](int a, double acc, double wsum, double& f) {
      f = tfc[a];
      const double* fb = tfb + a * C.Q;
#pragma unroll
      for (int q = 0; q < kMaxQ; ++q)
        if (q < C.Q) f = fma(fb[q], feat[q], f);
      const double c = nd.cn + tcc[a];
      return (acc - wsum * Uj) + c * Uj + f;
    };
    int a = 0;
    for (; a < C.K; ++a) {
      Tap<D> taps[E];
      double wsum;
      if (DEEP) {
        double o[P + 1][D];
        row_offsets<D, P>(L, tsd + a * P * D, tbd + a * D, nd, o);
        wsum = row_geometry_fast<D, P>(L, nd, o, taps);
      } else {
        wsum = row_taps<D, P>(L, tsd + a * P * D, tbd + a * D, nd, taps);
      }
      double vals[E];
#pragma unroll
      for (int e = 0; e < E; ++e) vals[e] = DEEP ? tap_value<D>(L, U, taps[e]) : tap_value_u<D>(L, C, U, taps[e]);
      double acc = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) acc = fma(taps[e].w, vals[e], acc);
      double f;
      const double H = tail(a, acc, wsum, f);
      if (H < best) {  // strict: lowest index wins exact ties (reading iv)
        best = H;
        arg = a;
        fbest = f;
      }
    }
    const double Up = __ldg(Uprev + nd.loc);
    const double R = fabs(Uj - Up - dt * best);
    const int old = pol[nd.loc];
    pol[nd.loc] = (uint8_t)arg;
    F[nd.loc] = fma(dt, fbest, Up);
    red[0] = fmax(red[0], (R == R) ? R : INFINITY);  // NaN -> inf (reported NONFINITE)
    red[1] += (old != arg) ? 1.0 : 0.0;
  };
  if (!DEEP || width < kSBX) {
    const int npk = nk * width;  // < 2^31: local arrays hold < 2^31 nodes
    const int gstride = gridDim.x * gridDim.y * kSBX * kSBY;
    for (int q = (blockIdx.y * gridDim.x + blockIdx.x) * (kSBX * kSBY) + threadIdx.y * kSBX + threadIdx.x; q < npk;
         q += gstride) {
      const int k = q / width;
      node_work(k, it.c0 + (q - k * width));
    }
  } else {
    for (int k = blockIdx.y * kSBY + threadIdx.y; k < nk; k += gridDim.y * kSBY)
      for (int col = it.c0 + blockIdx.x * kSBX + threadIdx.x; col < it.c1; col += gridDim.x * kSBX) node_work(k, col);
  }
  block_reduce_store<2>(red, partial, 0x1u);
}

// per-rank ranges of the per-node scale fields: [min sc_p, max sc_p]_p, [min bs, max bs] as
// block partials of maxima of (-min, max) pairs
template <int D, int P>
__global__ void __launch_bounds__(kTX) k_field_ranges(LevelDev L, CoefDev C, double* part) {
  double v[2 * P + 2];
#pragma unroll
  for (int k = 0; k < 2 * P + 2; ++k) v[k] = -INFINITY;
  FOR_INTERIOR(L) {
    Node<D> nd;
    node_at<D>(L, col, row, nd);
    load_fields<D>(C, nd);
#pragma unroll
    for (int p = 0; p < P; ++p) {
      v[2 * p] = fmax(v[2 * p], -nd.sc[p]);
      v[2 * p + 1] = fmax(v[2 * p + 1], nd.sc[p]);
    }
    v[2 * P] = fmax(v[2 * P], -nd.bs);
    v[2 * P + 1] = fmax(v[2 * P + 1], nd.bs);
  }
#pragma unroll
  for (int k = 0; k < 2 * P + 2; ++k) v[k] = warp_max(v[k]);
  __shared__ double sm[2 * P + 2][kTX / 32];
  const int tid = threadIdx.y * blockDim.x + threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < 2 * P + 2; ++k) sm[k][wid] = v[k];
  __syncthreads();
  if (tid == 0) {
    for (int k = 0; k < 2 * P + 2; ++k) {
      double m = -INFINITY;
      for (int w = 0; w < kTX / 32; ++w) m = fmax(m, sm[k][w]);
      part[(blockIdx.y * gridDim.x + blockIdx.x) * (2 * P + 2) + k] = m;
    }
  }
}

// ================================================================== Krylov vector kernels
// Device-resident BiCGSTAB scalars (right preconditioning).
struct KScal {
  double rho, rho_old, alpha, omega;
  double rhat_v, ts, tt, rr, ss;
  double bnorm2;
  int breakdown;
};

enum ScalOp : int { SC_NONE = 0, SC_INIT = 1, SC_AFTER_V = 2, SC_AFTER_T = 3, SC_AFTER_R = 4 };

__device__ __forceinline__ void scal_update(KScal* S, const double* red, int which) {
  if (which == SC_INIT) {          // red[0] = (r,r)
    S->rho = red[0]; S->rho_old = 1.0; S->alpha = 1.0; S->omega = 1.0; S->rr = red[0]; S->breakdown = 0;
  } else if (which == SC_AFTER_V) {  // red[0] = (rhat, v)
    S->rhat_v = red[0];
    if (red[0] == 0.0 || !(red[0] == red[0])) S->breakdown = 1;
    // on breakdown alpha = 0 keeps x finite: the half step is skipped and the omega step that
    // follows is a plain minimal-residual step; the host then restarts from x
    S->alpha = S->breakdown == 1 ? 0.0 : S->rho / red[0];
  } else if (which == SC_AFTER_T) {  // red = [(t,s), (t,t)]
    S->ts = red[0]; S->tt = red[1];
    S->omega = (red[1] > 0.0) ? red[0] / red[1] : 0.0;
    if (S->omega == 0.0) S->breakdown = 2;
  } else if (which == SC_AFTER_R) {  // red = [(rhat,r), (r,r)]
    S->rho_old = S->rho; S->rho = red[0]; S->rr = red[1];
    if (red[0] == 0.0 || !(red[1] == red[1])) S->breakdown = 3;
  }
}

// fixed-order deterministic reduction of nblk x 2 partials by one block (bit k of maxmask: max),
// then the BiCGSTAB scalar update `which` (no host round trip).
__global__ void __launch_bounds__(1024) k_finalize(const double* __restrict__ partial, int nblk, double* out,
                                                 unsigned maxmask, KScal* S, int which) {
  __shared__ double sm[2][1024];
  double v[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const bool mx = (maxmask >> k) & 1u;
    v[k] = mx ? -INFINITY : 0.0;
    for (int i = threadIdx.x; i < nblk; i += blockDim.x) {
      const double q = partial[i * 2 + k];
      v[k] = mx ? fmax(v[k], q) : v[k] + q;
    }
    sm[k][threadIdx.x] = v[k];
  }
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const bool mx = (maxmask >> k) & 1u;
        sm[k][threadIdx.x] = mx ? fmax(sm[k][threadIdx.x], sm[k][threadIdx.x + st]) : sm[k][threadIdx.x] + sm[k][threadIdx.x + st];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double red[2] = {sm[0][0], sm[1][0]};
    out[0] = red[0];
    out[1] = red[1];
    if (which != SC_NONE) scal_update(S, red, which);
  }
}

// multi-rank: combine the per-rank reductions gathered as all[q][2] (fixed rank order: bitwise
// repeatable for a given rank count), then the BiCGSTAB scalar update `which`
__global__ void k_combine(const double* __restrict__ all, int nranks, double* out, unsigned maxmask, KScal* S,
                          int which) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double red[2];
  for (int k = 0; k < 2; ++k) {
    const bool mx = (maxmask >> k) & 1u;
    double v = mx ? -INFINITY : 0.0;
    for (int q = 0; q < nranks; ++q) v = mx ? fmax(v, all[2 * q + k]) : v + all[2 * q + k];
    red[k] = v;
  }
  out[0] = red[0];
  out[1] = red[1];
  if (which != SC_NONE) scal_update(S, red, which);
}

// largest stencil offset along the slowest axis in cells over owned nodes and all controls:
// partial [max diffusion |o|, max drift |o|]  (halo check of hjb_set_coeffs)
template <int D>
__global__ void __launch_bounds__(kTX) k_reach(LevelDev L, CoefDev C, double* partial) {
  double red[2] = {0.0, 0.0};
  FOR_INTERIOR(L) {
    Node<D> nd;
    node_at<D>(L, col, row, nd);
    load_fields<D>(C, nd);
    for (int a = 0; a < C.K; ++a) {
      for (int p = 0; p < C.P; ++p) {
        const double o = L.kh * fma(nd.sc[p], __ldg(C.sigma_dir + (a * C.P + p) * D + D - 1), nd.sn[p][D - 1]);
        red[0] = fmax(red[0], fabs(o));
      }
      const double ob = L.k2h * fma(nd.bs, __ldg(C.b_dir + a * D + D - 1), nd.bn[D - 1]);
      red[1] = fmax(red[1], fabs(ob));
    }
  }
  block_reduce_store<2>(red, partial, 0x3u);
}

// r_hat = r, p = r ; partial: (r,r)
template <int D>
__global__ void __launch_bounds__(kTX) k_bicg_init(LevelDev L, const double* __restrict__ r,
                                                       double* __restrict__ rhat, double* __restrict__ p,
                                                       double* partial) {
  double red[2] = {0.0, 0.0};
  FOR_INTERIOR(L) {
    const int j = interior_offset<D>(L, col, row);
    const double v = r[j];
    rhat[j] = v;
    p[j] = v;
    red[0] = fma(v, v, red[0]);
  }
  block_reduce_store<2>(red, partial);
}

// p = r + beta (p - omega v),  beta = (rho/rho_old)(alpha/omega)
template <int D>
__global__ void __launch_bounds__(kTX) k_bicg_p(LevelDev L, const KScal* __restrict__ S,
                                                    const double* __restrict__ r, double* __restrict__ p,
                                                    const double* __restrict__ v) {
  const double beta = (S->rho / S->rho_old) * (S->alpha / S->omega);
  const double om = S->omega;
  FOR_INTERIOR(L) {
    const int j = interior_offset<D>(L, col, row);
    p[j] = fma(beta, fma(-om, v[j], p[j]), r[j]);
  }
}

// s = r - alpha v ; partial (s,s)
template <int D>
__global__ void __launch_bounds__(kTX) k_bicg_s(LevelDev L, const KScal* __restrict__ S,
                                                    const double* __restrict__ r, const double* __restrict__ v,
                                                    double* __restrict__ s, double* partial) {
  const double al = S->alpha;
  double red[2] = {0.0, 0.0};
  FOR_INTERIOR(L) {
    const int j = interior_offset<D>(L, col, row);
    const double sv = fma(-al, v[j], r[j]);
    s[j] = sv;
    red[0] = fma(sv, sv, red[0]);
  }
  block_reduce_store<2>(red, partial);
}

// x += alpha phat + omega shat ; r = s - omega t ; partials (rhat, r), (r, r)
template <int D>
__global__ void __launch_bounds__(kTX) k_bicg_x(LevelDev L, const KScal* __restrict__ S,
                                                    double* __restrict__ x, const double* __restrict__ phat,
                                                    const double* __restrict__ shat,
                                                    const double* __restrict__ s, const double* __restrict__ tv,
                                                    double* __restrict__ r, const double* __restrict__ rhat,
                                                    double* partial) {
  const double al = S->alpha, om = S->omega;
  double red[2] = {0.0, 0.0};
  FOR_INTERIOR(L) {
    const int j = interior_offset<D>(L, col, row);
    x[j] = fma(om, shat[j], fma(al, phat[j], x[j]));
    const double rv = fma(-om, tv[j], s[j]);
    r[j] = rv;
    red[0] = fma(rhat[j], rv, red[0]);
    red[1] = fma(rv, rv, red[1]);
  }
  block_reduce_store<2>(red, partial);
}

// squared 2-norm and max-norm partials of a vector over owned interior nodes
template <int D>
__global__ void __launch_bounds__(kTX) k_norms(LevelDev L, const double* __restrict__ v, double* partial) {
  double red[2] = {0.0, 0.0};
  FOR_INTERIOR(L) {
    const double a = v[interior_offset<D>(L, col, row)];
    red[0] = fma(a, a, red[0]);
    red[1] = fmax(red[1], (a == a) ? fabs(a) : INFINITY);
  }
  block_reduce_store<2>(red, partial, 0x2u);
}

// initial guess U <- 2 U_prev - U  (U holds U^{n-2} on entry: linear extrapolation in time)
template <int D>
__global__ void __launch_bounds__(kTX) k_extrapolate(LevelDev L, const double* __restrict__ up,
                                                     double* __restrict__ u) {
  FOR_INTERIOR(L) {
    const int j = interior_offset<D>(L, col, row);
    u[j] = fma(2.0, up[j], -u[j]);
  }
}

// ================================================================== theta-scheme
// V = theta U + (1 - theta) U_prev over every local element (boundary and halo entries included):
// the argument of the policy search of the theta-scheme (DESIGN.md §3 reading xxvi)
__global__ void __launch_bounds__(256) k_theta_mix(double theta, const double* __restrict__ u,
                                                   const double* __restrict__ up, double* __restrict__ v,
                                                   int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = fma(theta, u[i], (1.0 - theta) * up[i]);
}

// out = F + U_prev - y at interior nodes, with F = U_prev + dt f^pi (the search's output) and
// y = A'_{(1-theta) dt} U_prev = U_prev - (1-theta) dt (L^pi + c) U_prev: the theta-scheme right-hand
// side U_prev + (1-theta) dt (L^pi + c) U_prev + dt f^pi (B^{n,n-1} of P:419-424); theta = 0: U^n
template <int D>
__global__ void __launch_bounds__(kTX) k_theta_rhs(LevelDev L, const double* __restrict__ F,
                                                   const double* __restrict__ up, const double* __restrict__ y,
                                                   double* __restrict__ out) {
  FOR_INTERIOR(L) {
    const int j = interior_offset<D>(L, col, row);
    out[j] = F[j] + (up[j] - y[j]);
  }
}

// positivity (CFL) rate of Proposition CFL: max over owned interior nodes of
// sum_e w_e - c^a_j (= sum_p (A_p+B_p)/(2dx) - c, the M = P+1 pairs incl. the drift pair) for the
// node's control (pol != null) or over every control (pol == null); partial [max, 0]
template <int D, int P>
__global__ void __launch_bounds__(kTX, HJB_SEARCH_MINB) k_cfl(LevelDev L, CoefDev C, const uint8_t* __restrict__ pol,
                                                             double* partial) {
  double red[2] = {-INFINITY, 0.0};
  FOR_INTERIOR(L) {
    Node<D> nd;
    node_at<D>(L, col, row, nd);
    load_fields<D>(C, nd);
    const int a0 = pol ? (int)pol[nd.loc] : 0, a1 = pol ? a0 + 1 : C.K;
    for (int a = a0; a < a1; ++a) {
      Tap<D> taps[2 * P + 1];
      const double wsum = row_geometry<D, P>(L, C.sigma_dir + a * P * D, C.b_dir + a * D, nd, taps);
      red[0] = fmax(red[0], wsum - (nd.cn + C.c_ctrl[a]));
    }
  }
  block_reduce_store<2>(red, partial, 0x1u);
}

// first smoothing sweep from x = 0 with the stored diagonal: y = omega b / D (the arithmetic of
// k_operator<..., OP_JACOBI0>, without its per-node geometry)
template <int D, typename V = double>
__global__ void __launch_bounds__(kTX) k_jacobi0_diag(LevelDev L, double omega, const V* __restrict__ b,
                                                      const V* __restrict__ dg, V* __restrict__ y) {
  FOR_INTERIOR(L) {
    const int j = interior_offset<D>(L, col, row);
    y[j] = (V)(omega * (double)__ldg(b + j) / (double)__ldg(dg + j));
  }
}

template <int D, typename V = double>
__global__ void __launch_bounds__(kTX) k_add_interior(LevelDev L, const V* __restrict__ a,
                                                          V* __restrict__ y) {
  FOR_INTERIOR(L) {
    const int j = interior_offset<D>(L, col, row);
    y[j] += a[j];
  }
}

// b = a at the interior nodes (with a type conversion: the fp32 multigrid's entry and exit)
template <int D, typename VA = double, typename VB = double>
__global__ void __launch_bounds__(kTX) k_copy_interior(LevelDev L, const VA* __restrict__ a,
                                                           VB* __restrict__ b) {
  FOR_INTERIOR(L) {
    const int j = interior_offset<D>(L, col, row);
    b[j] = (VB)a[j];
  }
}

// ================================================================== boundary data
// scatter the packed boundary values (lexicographic order of boundary nodes) into U
template <int D>
__global__ void k_scatter_psi(LevelDev L, int64_t nb, const double* __restrict__ psi, double* __restrict__ U) {
  const int64_t n = L.n;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nb; q += (int64_t)gridDim.x * blockDim.x) {
    int64_t i[3] = {0, 0, 0};
    if (D == 2) {
      if (q < n) { i[0] = q; i[1] = 0; }
      else if (q < n + 2 * (n - 2)) { const int64_t r = q - n; i[1] = 1 + r / 2; i[0] = (r & 1) ? n - 1 : 0; }
      else { i[1] = n - 1; i[0] = q - n - 2 * (n - 2); }
    } else {
      const int64_t plane = n * n, ring = 4 * n - 4;
      if (q < plane) { i[2] = 0; i[1] = q / n; i[0] = q % n; }
      else if (q < plane + (n - 2) * ring) {
        const int64_t r = q - plane;
        i[2] = 1 + r / ring;
        const int64_t w = r % ring;
        if (w < n) { i[1] = 0; i[0] = w; }
        else if (w < n + 2 * (n - 2)) { const int64_t v = w - n; i[1] = 1 + v / 2; i[0] = (v & 1) ? n - 1 : 0; }
        else { i[1] = n - 1; i[0] = w - n - 2 * (n - 2); }
      } else {
        const int64_t r = q - plane - (n - 2) * ring;
        i[2] = n - 1; i[1] = r / n; i[0] = r % n;
      }
    }
    const int64_t slow = i[D - 1];
    if (slow < L.local_row0 || slow >= L.local_row0 + L.local_rows) continue;
    int64_t loc = (slow - L.local_row0);
    for (int d = D - 2; d >= 0; --d) loc = loc * n + i[d];
    U[loc] = psi[q];
  }
}

// ================================================================== certified search skipping
// One pass over the whole local grid (interior and boundary): out[0] = max |U|, out[1] = max |dU|,
// out[2] = max over grid edges of |dU_i' - dU_i| (i' the neighbour along x1 or x2), dU = U - uo;
// un = U (the next search's U_old; uo == nullptr: only max |U| and the copy).  Non-negative doubles
// order like their bit patterns, so the maxima are atomicMax on the 64-bit words.
__global__ void __launch_bounds__(256) k_gap_delta(const double* __restrict__ U, const double* __restrict__ uo,
                                                   double* __restrict__ un, int64_t n, int64_t N,
                                                   unsigned long long* __restrict__ out) {
  double m[3] = {0.0, 0.0, 0.0};
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
    const double u = U[j];
    un[j] = u;
    m[0] = fmax(m[0], fabs(u));
    if (uo) {
      const double d = u - uo[j];
      m[1] = fmax(m[1], fabs(d));
      if ((j % n) != n - 1) m[2] = fmax(m[2], fabs((U[j + 1] - uo[j + 1]) - d));
      if (j + n < N) m[2] = fmax(m[2], fabs((U[j + n] - uo[j + n]) - d));
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double v = m[k];
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out + k, (unsigned long long)__double_as_longlong(v));
  }
}

// ================================================================== multigrid transfers
// full weighting r_f -> b_c at coarse interior nodes (weights 1/4,1/2,1/4 per dim)
template <int D, typename VF = double, typename VC = double>
__global__ void __launch_bounds__(kTX) k_restrict(LevelDev Lf, LevelDev Lc, const VF* __restrict__ rf,
                                                      VC* __restrict__ bc) {
  FOR_INTERIOR(Lc) {
    Node<D> nd;
    node_at<D>(Lc, col, row, nd);
    double acc = 0.0;
    if (D == 2) {
      const int64_t base = (int64_t)(2 * nd.i[1] - Lf.local_row0) * Lf.n + 2 * nd.i[0];
#pragma unroll
      for (int o2 = -1; o2 <= 1; ++o2) {
        const double w2 = o2 == 0 ? 0.5 : 0.25;
#pragma unroll
        for (int o1 = -1; o1 <= 1; ++o1) {
          const double w1 = o1 == 0 ? 0.5 : 0.25;
          acc = fma(w1 * w2, (double)__ldg(rf + base + o2 * Lf.n + o1), acc);
        }
      }
    } else {
      const int64_t nf = Lf.n;
      const int64_t base = ((int64_t)(2 * nd.i[2] - Lf.local_row0) * nf + 2 * nd.i[1]) * nf + 2 * nd.i[0];
#pragma unroll
      for (int o3 = -1; o3 <= 1; ++o3) {
        const double w3 = o3 == 0 ? 0.5 : 0.25;
#pragma unroll
        for (int o2 = -1; o2 <= 1; ++o2) {
          const double w2 = o2 == 0 ? 0.5 : 0.25;
#pragma unroll
          for (int o1 = -1; o1 <= 1; ++o1) {
            const double w1 = o1 == 0 ? 0.5 : 0.25;
            acc = fma(w1 * w2 * w3, (double)__ldg(rf + base + (o3 * nf + o2) * nf + o1), acc);
          }
        }
      }
    }
    bc[nd.loc] = (VC)acc;
  }
}

// x_f += P e_c (multilinear prolongation) at fine interior nodes
template <int D, typename VC = double, typename VF = double>
__global__ void __launch_bounds__(kTX) k_prolong_add(LevelDev Lf, LevelDev Lc, const VC* __restrict__ ec,
                                                         VF* __restrict__ xf) {
  FOR_INTERIOR(Lf) {
    Node<D> nd;
    node_at<D>(Lf, col, row, nd);
    int c0[D], c1[D];
    double w1[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      c0[d] = nd.i[d] >> 1;
      const bool odd = nd.i[d] & 1;
      c1[d] = odd ? c0[d] + 1 : c0[d];
      w1[d] = odd ? 0.5 : 0.0;
    }
    double acc = 0.0;
    const int64_t nc = Lc.n;
#pragma unroll
    for (int m = 0; m < (1 << D); ++m) {
      double w = 1.0;
      int cc[D];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const bool hi = (m >> d) & 1;
        cc[d] = hi ? c1[d] : c0[d];
        w *= hi ? w1[d] : (1.0 - w1[d]);
      }
      if (w == 0.0) continue;
      int64_t loc = (int64_t)(cc[D - 1] - Lc.local_row0);
#pragma unroll
      for (int d = D - 2; d >= 0; --d) loc = loc * nc + cc[d];
      acc = fma(w, (double)__ldg(ec + loc), acc);
    }
    xf[nd.loc] = (VF)((double)xf[nd.loc] + acc);
  }
}

// inject the policy from level f to level c (coarse node J <- fine node 2J), every local coarse node
// whose fine node lies in the fine rows [fr_lo, fr_hi) (the rows whose values are valid there)
template <int D>
__global__ void k_inject_u8(LevelDev Lf, LevelDev Lc, const uint8_t* __restrict__ pf, uint8_t* __restrict__ pc,
                            int64_t fr_lo, int64_t fr_hi) {
  const int64_t nloc = Lc.local_rows * Lc.row_elems;
  const int64_t nc = Lc.n, nf = Lf.n;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nloc; q += (int64_t)gridDim.x * blockDim.x) {
    int64_t i[3];
    int64_t r = q;
#pragma unroll
    for (int d = 0; d < D - 1; ++d) { i[d] = r % nc; r /= nc; }
    const int64_t gfr = 2 * (r + Lc.local_row0);
    if (gfr < fr_lo || gfr >= fr_hi) continue;
    const int64_t fr = gfr - Lf.local_row0;
    if (fr < 0 || fr >= Lf.local_rows) continue;
    int64_t loc = fr;
#pragma unroll
    for (int d = D - 2; d >= 0; --d) loc = loc * nf + 2 * i[d];
    pc[q] = pf[loc];
  }
}

// inject nplanes fp64 field planes (plane strides ldf / ldc)
template <int D>
__global__ void k_inject_f64(LevelDev Lf, LevelDev Lc, const double* __restrict__ ff, int64_t ldf,
                             double* __restrict__ fc, int64_t ldc, int nplanes, int64_t fr_lo, int64_t fr_hi) {
  const int64_t nloc = Lc.local_rows * Lc.row_elems;
  const int64_t nc = Lc.n, nf = Lf.n;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nloc; q += (int64_t)gridDim.x * blockDim.x) {
    int64_t i[3];
    int64_t r = q;
#pragma unroll
    for (int d = 0; d < D - 1; ++d) { i[d] = r % nc; r /= nc; }
    const int64_t gfr = 2 * (r + Lc.local_row0);
    if (gfr < fr_lo || gfr >= fr_hi) continue;
    const int64_t fr = gfr - Lf.local_row0;
    if (fr < 0 || fr >= Lf.local_rows) continue;
    int64_t loc = fr;
#pragma unroll
    for (int d = D - 2; d >= 0; --d) loc = loc * nf + 2 * i[d];
    for (int k = 0; k < nplanes; ++k) fc[k * ldc + q] = ff[k * ldf + loc];
  }
}

// ================================================================== coarsest level (dense)
// interior node t (0..n_own) of a single-rank level -> (col, row)
template <int D>
__device__ __forceinline__ void coarse_node(const LevelDev& L, int t, Node<D>& nd) {
  const int row = t / L.nI;
  node_at<D>(L, t - row * L.nI, row, nd);
}

// assemble the dense interior matrix of the coarsest level: A[j][i] (row-major, Nc x Nc), the same
// truncated Scheme-2 row as row_eval (general path for every endpoint)
template <int D>
__global__ void k_coarse_assemble(LevelDev L, CoefDev C, double dt, const uint8_t* __restrict__ pol,
                                  double* __restrict__ A) {
  const int Nc = (int)L.n_own;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < Nc; t += gridDim.x * blockDim.x) {
    Node<D> nd;
    coarse_node<D>(L, t, nd);
    load_fields<D>(C, nd);
    const int a = pol[nd.loc];
    double* row = A + (int64_t)t * Nc;
    double wsum = 0.0;
    const int nI = L.nI;
    auto add_tap = [&](const double* o, double mu, int bd, double w) {
      int c[D];
      double s[D];
      cell_general<D>(L, nd, o, mu, bd, c, s);
#pragma unroll
      for (int m = 0; m < (1 << D); ++m) {
        double ww = w;
        int col = 0;
        bool interior = true;
#pragma unroll
        for (int d = D - 1; d >= 0; --d) {
          const bool hi = (m >> d) & 1;
          const int id = c[d] + (hi ? 1 : 0);
          ww *= hi ? s[d] : (1.0 - s[d]);
          interior &= (id >= 1 && id <= L.n - 2);
          col = col * nI + (id - 1);
        }
        if (interior && ww != 0.0) row[col] -= dt * ww;
      }
    };
    const double* sd = C.sigma_dir + a * C.P * D;
    for (int p = 0; p < C.P; ++p) {
      double o[D], om[D];
      bool nz = false;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        o[d] = L.kh * fma(nd.sc[p], sd[p * D + d], nd.sn[p][d]);
        om[d] = -o[d];
        nz |= (o[d] != 0.0);
      }
      if (!nz) continue;
      int bp, bm;
      const double mup = ray_mu<D>(L, nd, o, bp);
      const double mum = ray_mu<D>(L, nd, om, bm);
      double Aw = 1.0, Bw = 1.0;
      if (bp >= 0 || bm >= 0) {
        const double sum = mup + mum;
        Aw = 2.0 / (mup * sum);
        Bw = 2.0 / (mum * sum);
      }
      wsum += (Aw + Bw) * L.inv_2k2;
      add_tap(o, mup, bp, Aw * L.inv_2k2);
      add_tap(om, mum, bm, Bw * L.inv_2k2);
    }
    {
      double o[D];
      bool nz = false;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        o[d] = L.k2h * fma(nd.bs, C.b_dir[a * D + d], nd.bn[d]);
        nz |= (o[d] != 0.0);
      }
      if (nz) {
        int bdim;
        const double mu = ray_mu<D>(L, nd, o, bdim);
        const double w = (bdim >= 0) ? L.inv_k2 / mu : L.inv_k2;
        wsum += w;
        add_tap(o, mu, bdim, w);
      }
    }
    const double c = nd.cn + C.c_ctrl[a];
    row[t] += 1.0 + dt * (wsum - c);
  }
}

// in-place Gauss-Jordan inverse (no pivoting: the interior matrix is strictly row diagonally
// dominant, row sums >= 1 - dt c > 0), single block, matrix in shared memory (Nc <= 160).
__global__ void k_coarse_invert(double* __restrict__ A, int Nc) {
  extern __shared__ double M[];
  __shared__ double colk[160];
  const int NN = Nc * Nc;
  for (int e = threadIdx.x; e < NN; e += blockDim.x) M[e] = A[e];
  __syncthreads();
  for (int k = 0; k < Nc; ++k) {
    const double piv = M[k * Nc + k];
    __syncthreads();
    for (int j = threadIdx.x; j < Nc; j += blockDim.x) {
      const double v = (j == k) ? 1.0 : M[k * Nc + j];
      M[k * Nc + j] = v / piv;
    }
    for (int i = threadIdx.x; i < Nc; i += blockDim.x) colk[i] = (i == k) ? 0.0 : M[i * Nc + k];
    __syncthreads();
    for (int e = threadIdx.x; e < NN; e += blockDim.x) {
      const int i = e / Nc, j = e - i * Nc;
      if (i == k) continue;
      const double base = (j == k) ? 0.0 : M[e];
      M[e] = fma(-colk[i], M[k * Nc + j], base);
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < NN; e += blockDim.x) A[e] = M[e];
}

// x_c = Ainv b_c on the coarsest interior
template <int D, typename V = double>
__global__ void k_coarse_solve(LevelDev L, const double* __restrict__ Ainv, const V* __restrict__ b,
                               V* __restrict__ x) {
  extern __shared__ double bs[];
  const int Nc = (int)L.n_own;
  for (int t = threadIdx.x; t < Nc; t += blockDim.x) {
    const int row = t / L.nI;
    bs[t] = (double)b[interior_offset<D>(L, t - row * L.nI, row)];
  }
  __syncthreads();
  for (int t = threadIdx.x; t < Nc; t += blockDim.x) {
    double acc = 0.0;
    const double* rowp = Ainv + (int64_t)t * Nc;
    for (int i = 0; i < Nc; ++i) acc = fma(rowp[i], bs[i], acc);
    const int row = t / L.nI;
    x[interior_offset<D>(L, t - row * L.nI, row)] = (V)acc;
  }
}

}  // namespace hjb
