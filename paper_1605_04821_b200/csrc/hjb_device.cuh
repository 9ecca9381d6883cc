// hjb_device.cuh -- sm_100a device code for the implicit LISL/HJB hot path (fp64).
//
// Scheme (arXiv:1605.04821): Scheme 2 steps y+-_p = +-k sigma_p, y_{P+1} = k^2 b (PAPER.md:95-96,
// k = sqrt(h)), truncated to the box with mu = largest value in (0,1] keeping the segment in
// closed Omega, weights A = 2/(mu+^2+mu+mu-), B = 2/(mu-^2+mu-mu+), drift
// A = B = 1/mu, multilinear interpolation.  Row of the implicit system
// (theta = 1):
//     (A x)_j = x_j - dt [ sum_e w_e (I x(z_e) - x_j) + c_j x_j ],  w_e = {A,B}/(2k^2), 1/(mu_d k^2)
// and its diagonal D_j = 1 + dt (sum_e w_e - sum_e w_e w_j(z_e) - c_j).
//
// Geometry is done in GRID UNITS: a node is its integer multi-index i, a step y becomes the offset
// o = y/h in cells, an endpoint is t = i + mu o and its cell is floor(t) (clamped to n-2) with
// fraction s = t - floor(t).  This is the oracle's physical-coordinate formula (z - lo)/h divided
// through by h; the two differ only by rounding (~1e-16 relative in s), and every decision on the
// way (inside/outside, cell choice) is continuous in the result (SURVEY hard part 4).
//
// Everything is recomputed on the fly per (node, control): no per-policy matrix is stored.
// Thread mapping: a 2D launch, threads along x1 (coalesced; for x-independent sigma the endpoints
// of a warp are consecutive nodes), blocks striding over interior rows so the +-reach rows in
// flight form a band that stays L2-resident.
#pragma once
#include <cassert>
#include <cstdint>
#include <cuda_runtime.h>

// HJB_CHECK=1 (tools/build_variant.sh check -DHJB_CHECK=1): device-side bounds assertions on every
// gather (compute-sanitizer is closed on this GPU pool)
#ifdef HJB_CHECK
#define HJB_ASSERT(c) assert(c)
#else
#define HJB_ASSERT(c) ((void)0)
#endif

namespace hjb {

#ifndef HJB_TX
#define HJB_TX 128
#endif
constexpr int kTX = HJB_TX;  // threads per block of the 2D grid kernels
#ifndef HJB_BX
#define HJB_BX 128
#endif
constexpr int kBX = HJB_BX;        // block extent along x1 (consecutive nodes per row)
constexpr int kBY = kTX / kBX;     // interior lines per block
#ifndef HJB_SBX
#define HJB_SBX 32
#endif
constexpr int kSBX = HJB_SBX;      // control search: 32 x 4 blocks (4 adjacent lines share the
constexpr int kSBY = kTX / kSBX;   // same control's gather rows -> L1 reuse across warps)
constexpr int kMaxP = 3;
constexpr int kMaxQ = 16;

// ----------------------------------------------------------------------------- level geometry
struct LevelDev {
  int n;               // nodes per dimension on this level
  int nI;              // n - 2 interior nodes per dimension
  int nrows;           // owned interior lines along x1 (n_own / nI)
  int64_t row_elems;   // n^(D-1)
  int64_t local_row0;  // global slowest-axis row of local row 0
  int64_t local_rows;  // rows held in a local array
  int64_t row_first;   // first owned interior row (global, slowest axis)
  int64_t n_own;       // owned interior nodes
  double h, nm1;       // mesh width; n - 1
  double kh;           // diffusion step in cells: k / h (k = sqrt(h_fine) by default)
  double k2h;          // drift step in cells: k^2 / h
  double inv_2k2, inv_k2;
  int pf_rows;         // L2 prefetch distance along the slowest axis (max reach + 2; 0 = off)
  int local_elems;     // local_rows * row_elems
};

// L2 prefetch of the grid line `pf_rows` slowest-axis rows ahead of node j: the leading edge of
// the gather band, which would otherwise miss L2 (one line per 16 lanes)
// load used for the interpolation gathers (A/B knob for the cache operator: 0 = ld.global.nc,
// 1 = ld.global.ca, 2 = ld.global.cg)
#ifndef HJB_GLD_MODE
#define HJB_GLD_MODE 0
#endif
#if HJB_GLD_MODE == 1
#define HJB_GLD(p) __ldca(p)
#elif HJB_GLD_MODE == 2
#define HJB_GLD(p) __ldcg(p)
#else
#define HJB_GLD(p) __ldg(p)
#endif

__device__ __forceinline__ void prefetch_ahead(const LevelDev& L, const double* v, int j, int col) {
  if (L.pf_rows <= 0 || (col & 15) != 0) return;
  const long long a = (long long)j + (long long)L.pf_rows * L.row_elems;
  if (a < L.local_elems) asm volatile("prefetch.global.L2 [%0];" ::"l"(v + a));
}

// ----------------------------------------------------------------------------- coefficients
struct CoefDev {
  const double* sigma_dir;  // [K][P][D]
  const double* b_dir;      // [K][D]
  const double* c_ctrl;     // [K]
  const double* f_basis;    // [K][Q]
  const double* f_ctrl;     // [K]
  const double* sigma_scale;  // [P][ld] or null
  const double* sigma_node;   // [P][D][ld] or null
  const double* b_scale;      // [ld] or null
  const double* b_node;       // [D][ld] or null
  const double* c_node;       // [ld] or null
  const double* f_feat;       // [Q][ld] or null
  int64_t ld;
  int K, P, Q;
  // exact-psi boundary mode (Remark rhs; hjb_set_boundary_samples): psi sampled on the
  // faces at spacing h / brefine, bM samples per along-face axis; null = interpolation mode.  Set
  // only in the CoefDev passed where the argument is U itself (search, residual of U).
  const double* bsamp = nullptr;
  int brefine = 0, bM = 0;
};

template <int D>
struct Node {
  int i[D];          // global multi-index
  double fi[D];      // i as double
  double dist[D];    // min(i, n-1-i): an offset |o| <= dist keeps both i+o and i-o in the box
  int loc;           // local linear offset (local arrays hold < 2^31 elements)
  double sc[kMaxP];  // sigma scale per column
  double sn[kMaxP][D];
  double bs, bn[D], cn;
};

// interior line `row` (0..nrows), column `col` (0..nI) -> node
template <int D>
__device__ __forceinline__ void node_at(const LevelDev& L, int col, int row, Node<D>& nd) {
  nd.i[0] = 1 + col;
  if (D == 2) {
    nd.i[1] = (int)L.row_first + row;
    nd.loc = (nd.i[1] - (int)L.local_row0) * L.n + nd.i[0];
  } else {
    const int r2 = row / L.nI;
    nd.i[1] = 1 + (row - r2 * L.nI);
    nd.i[D - 1] = (int)L.row_first + r2;
    nd.loc = ((nd.i[D - 1] - (int)L.local_row0) * L.n + nd.i[1]) * L.n + nd.i[0];
  }
#pragma unroll
  for (int d = 0; d < D; ++d) {
    nd.fi[d] = (double)nd.i[d];
    const int m = min(nd.i[d], L.n - 1 - nd.i[d]);
    nd.dist[d] = (double)m;
  }
}

template <int D>
__device__ __forceinline__ int interior_offset(const LevelDev& L, int col, int row) {
  if (D == 2) return ((int)L.row_first + row - (int)L.local_row0) * L.n + 1 + col;
  const int r2 = row / L.nI;
  return (((int)L.row_first + r2 - (int)L.local_row0) * L.n + 1 + (row - r2 * L.nI)) * L.n + 1 + col;
}

template <int D>
__device__ __forceinline__ void load_fields(const CoefDev& C, Node<D>& nd) {
  const int64_t j = nd.loc;
#pragma unroll
  for (int p = 0; p < kMaxP; ++p) {
    nd.sc[p] = 1.0;
#pragma unroll
    for (int d = 0; d < D; ++d) nd.sn[p][d] = 0.0;
    if (p < C.P) {
      if (C.sigma_scale) nd.sc[p] = __ldg(C.sigma_scale + p * C.ld + j);
      if (C.sigma_node) {
#pragma unroll
        for (int d = 0; d < D; ++d) nd.sn[p][d] = __ldg(C.sigma_node + (p * D + d) * C.ld + j);
      }
    }
  }
  nd.bs = C.b_scale ? __ldg(C.b_scale + j) : 1.0;
#pragma unroll
  for (int d = 0; d < D; ++d) nd.bn[d] = C.b_node ? __ldg(C.b_node + d * C.ld + j) : 0.0;
  nd.cn = C.c_node ? __ldg(C.c_node + j) : 0.0;
}

// per-node streamed inputs of the operator kernels, loaded one line ahead (software pipelining:
// the next line's loads are in flight while this line's gathers run)
template <int D, int P>
struct NodeIn {
  double sc[P], sn[P][D], bs, bn[D], cn;
  double xj, bj;
  int a;
};

template <int D, int P, bool XJ, bool BJ, typename V = double>
__device__ __forceinline__ void fetch_node(const LevelDev& L, const CoefDev& C, const uint8_t* __restrict__ pol,
                                           const V* __restrict__ x, const V* __restrict__ b, int col,
                                           int row, NodeIn<D, P>& in) {
  const int j = interior_offset<D>(L, col, row);
#pragma unroll
  for (int p = 0; p < P; ++p) {
    in.sc[p] = C.sigma_scale ? __ldg(C.sigma_scale + p * C.ld + j) : 1.0;
#pragma unroll
    for (int d = 0; d < D; ++d) in.sn[p][d] = C.sigma_node ? __ldg(C.sigma_node + (p * D + d) * C.ld + j) : 0.0;
  }
  in.bs = C.b_scale ? __ldg(C.b_scale + j) : 1.0;
#pragma unroll
  for (int d = 0; d < D; ++d) in.bn[d] = C.b_node ? __ldg(C.b_node + d * C.ld + j) : 0.0;
  in.cn = C.c_node ? __ldg(C.c_node + j) : 0.0;
  in.a = __ldg(pol + j);
  in.xj = XJ ? (double)__ldg(x + j) : 0.0;
  in.bj = BJ ? (double)__ldg(b + j) : 0.0;
}

template <int D, int P>
__device__ __forceinline__ void node_from(const LevelDev& L, int col, int row, const NodeIn<D, P>& in, Node<D>& nd) {
  node_at<D>(L, col, row, nd);
#pragma unroll
  for (int p = 0; p < kMaxP; ++p) {
    nd.sc[p] = p < P ? in.sc[p < P ? p : 0] : 1.0;
#pragma unroll
    for (int d = 0; d < D; ++d) nd.sn[p][d] = p < P ? in.sn[p < P ? p : 0][d] : 0.0;
  }
  nd.bs = in.bs;
#pragma unroll
  for (int d = 0; d < D; ++d) nd.bn[d] = in.bn[d];
  nd.cn = in.cn;
}

// ----------------------------------------------------------------------------- cells
// floor split of t = i + o for an UNTRUNCATED offset: c = i + floor(o), s = o - floor(o), via
// round-to-nearest by the 1.5*2^52 magic constant (no fp64<->int conversion instructions).
// box of nodes in loop coordinates: col = i0 - 1 in [c0, c1); slab rows (2D: i1 - row_first, 3D:
// planes i2 - row_first) in [r0, r1); 3D only: y = i1 - 1 in [y0, y1) (2D: y0 = 0, y1 = 1).  Its
// k-th line is  row = (y0 + k % ny) + Y (r0 + k / ny),  ny = y1 - y0, Y = nI (3D) or 1 (2D).
struct SkipRect {
  int c0, c1, r0, r1;
  int y0 = 0, y1 = 1;
};

template <int D>
__device__ __forceinline__ int box_row(const LevelDev& L, const SkipRect& b, int k) {
  const int ny = b.y1 - b.y0;
  if (D == 2 || ny == 1) return (D == 3 ? b.y0 : 0) + (D == 3 ? L.nI : 1) * (b.r0 + k);
  const int z = k / ny;
  return b.y0 + (k - z * ny) + L.nI * (b.r0 + z);
}
__device__ __forceinline__ int box_lines(const SkipRect& b) { return (b.r1 - b.r0) * (b.y1 - b.y0); }

struct Split {
  int c;
  double s;
};
__device__ __forceinline__ void split_pm(double o, int i, int nm2, Split& p, Split& m) {
  const double magic = 6755399441055744.0;  // 1.5 * 2^52
  const double big = o + magic;
  const int r = __double2loint(big);          // rint(o) as an integer
  const double rf = big - magic;              // rint(o)
  const double f = o - rf;                    // in [-0.5, 0.5]
  // +o: floor = r - (f < 0)
  const bool neg = f < 0.0;
  p.c = i + r - (neg ? 1 : 0);
  p.s = neg ? f + 1.0 : f;
  // -o: rint(-o) = -r, fraction -f; floor = -r - (-f < 0)
  const bool pos = f > 0.0;
  m.c = i - r - (pos ? 1 : 0);
  m.s = pos ? 1.0 - f : -f;
  if (p.c > nm2) { p.c = nm2; p.s = 1.0; }  // endpoint exactly on the upper face
  if (m.c > nm2) { m.c = nm2; m.s = 1.0; }
}

__device__ __forceinline__ void split_p(double o, int i, int nm2, Split& p) {
  const double magic = 6755399441055744.0;
  const double big = o + magic;
  const int r = __double2loint(big);
  const double f = o - (big - magic);
  const bool neg = f < 0.0;
  p.c = i + r - (neg ? 1 : 0);
  p.s = neg ? f + 1.0 : f;
  if (p.c > nm2) { p.c = nm2; p.s = 1.0; }
}

// untruncated +-o pair in one dimension from one floor: +o -> (i + fl, o - fl); -o -> (i - fl - [s != 0],
// 1 - s or 0).  Used by the general path's untruncated case and by the fast path alike, so the two
// give bit-identical cells and fractions.
__device__ __forceinline__ void pair_split(double o, int i, int& cp, double& sp, int& cm, double& sm) {
  const double fl = floor(o);
  const int fi = (int)fl;
  sp = o - fl;
  const bool frac = sp != 0.0;
  cp = i + fi;
  cm = i - fi - (frac ? 1 : 0);
  sm = frac ? 1.0 - sp : 0.0;
}
__device__ __forceinline__ void single_split(double o, int i, int& c, double& s) {
  const double fl = floor(o);
  c = i + (int)fl;
  s = o - fl;
}

// general (possibly truncated) endpoint t = i + mu o, binding coordinate snapped onto the face
template <int D>
__device__ __forceinline__ void cell_general(const LevelDev& L, const Node<D>& nd, const double* o, double mu,
                                             int bd, int* c, double* s) {
#pragma unroll
  for (int d = 0; d < D; ++d) {
    double t = fma(mu, o[d], nd.fi[d]);
    t = fmin(fmax(t, 0.0), L.nm1);
    if (d == bd) t = (o[d] > 0.0) ? L.nm1 : 0.0;
    double fl = floor(t);
    int ci = (int)fl;
    if (ci > L.n - 2) { ci = L.n - 2; fl = (double)ci; }
    c[d] = ci;
    s[d] = t - fl;
  }
}

// truncation of the ray i + [0,1] o: mu = largest value in (0,1] keeping it in [0, n-1]^D
// (PAPER.md:224, 291-293); bd = binding dimension (-1 if untruncated).
template <int D>
__device__ __forceinline__ double ray_mu(const LevelDev& L, const Node<D>& nd, const double* o, int& bd) {
  double mu = 1.0;
  bd = -1;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const double room_hi = L.nm1 - nd.fi[d];
    if (o[d] > room_hi) {
      const double t = room_hi / o[d];
      if (t < mu) { mu = t; bd = d; }
    } else if (o[d] < -nd.fi[d]) {
      const double t = -nd.fi[d] / o[d];
      if (t < mu) { mu = t; bd = d; }
    }
  }
  return mu;
}

// ----------------------------------------------------------------------------- interpolation
// multilinear interpolation from the corner p of the tap's cell, strides sy (next x2 line) and sz
// (next x3 plane); LDG = the load (global: the read-only path, shared memory: plain loads).  One
// arithmetic order for every caller, so global and shared-memory gathers agree bit for bit.
template <int D, bool SMEM>
__device__ __forceinline__ double interp_at(const double* __restrict__ p, int sy, int sz, const double* s) {
#define HJB_LD(q) (SMEM ? *(q) : HJB_GLD(q))
  if (D == 2) {
    const double v00 = HJB_LD(p), v10 = HJB_LD(p + 1);
    const double v01 = HJB_LD(p + sy), v11 = HJB_LD(p + sy + 1);
    const double a = fma(s[0], v10 - v00, v00);
    const double b = fma(s[0], v11 - v01, v01);
    return fma(s[1], b - a, a);
  } else {
    const double v000 = HJB_LD(p), v100 = HJB_LD(p + 1);
    const double v010 = HJB_LD(p + sy), v110 = HJB_LD(p + sy + 1);
    const double v001 = HJB_LD(p + sz), v101 = HJB_LD(p + sz + 1);
    const double v011 = HJB_LD(p + sz + sy), v111 = HJB_LD(p + sz + sy + 1);
    const double a0 = fma(s[0], v100 - v000, v000);
    const double b0 = fma(s[0], v110 - v010, v010);
    const double a1 = fma(s[0], v101 - v001, v001);
    const double b1 = fma(s[0], v111 - v011, v011);
    const double p0 = fma(s[1], b0 - a0, a0);
    const double p1 = fma(s[1], b1 - a1, a1);
    return fma(s[2], p1 - p0, p0);
  }
#undef HJB_LD
}

template <int D>
__device__ __forceinline__ double gather_interp(const LevelDev& L, const double* __restrict__ v, const int* c,
                                                const double* s) {
  const int base = D == 2 ? (c[1] - (int)L.local_row0) * L.n + c[0]
                          : ((c[2] - (int)L.local_row0) * L.n + c[1]) * L.n + c[0];
  return interp_at<D, false>(v + base, L.n, L.n * L.n, s);
}

// multilinear weight of node i (multi-index) in the cell (c, s); 0 if not a vertex
template <int D>
__device__ __forceinline__ double self_weight(const int* i, const int* c, const double* s) {
  double w = 1.0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    if (i[d] == c[d]) w *= (1.0 - s[d]);
    else if (i[d] == c[d] + 1) w *= s[d];
    else return 0.0;
  }
  return w;
}

// ----------------------------------------------------------------------------- one row
// acc  = sum_e w_e I v(z_e)       (only if GATHER)
// wsum = sum_e w_e                (= sum_p (A_p+B_p)/(2k^2) + 1/(mu_d k^2))
// self = sum_e w_e w_j(z_e)       (only if SELF: l_hat_jj of P:399-401)
template <int D, bool GATHER, bool SELF>
__device__ __forceinline__ void row_eval(const LevelDev& L, const CoefDev& C, const Node<D>& nd, int a,
                                         const double* __restrict__ v, double& acc, double& wsum,
                                         double& self) {
  acc = 0.0;
  wsum = 0.0;
  self = 0.0;
  const double* sd = C.sigma_dir + a * C.P * D;
  const int nm2 = L.n - 2;
#pragma unroll
  for (int p = 0; p < kMaxP; ++p) {
    if (p >= C.P) break;
    double o[D];
    bool nz = false, inside = true;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      o[d] = L.kh * fma(nd.sc[p], __ldg(sd + p * D + d), nd.sn[p][d]);
      nz |= (o[d] != 0.0);
      inside &= (fabs(o[d]) <= nd.dist[d]);
    }
    if (!nz) continue;  // zero step: its two terms cancel exactly
    if (inside) {
      // untruncated pair (A = B = 1): endpoints i +- o
      int cp[D], cm[D];
      double sp[D], sm[D];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        Split P_, M_;
        split_pm(o[d], nd.i[d], nm2, P_, M_);
        cp[d] = P_.c; sp[d] = P_.s;
        cm[d] = M_.c; sm[d] = M_.s;
      }
      wsum += 2.0 * L.inv_2k2;
      if (GATHER) acc = fma(L.inv_2k2, gather_interp<D>(L, v, cp, sp) + gather_interp<D>(L, v, cm, sm), acc);
      if (SELF) self = fma(L.inv_2k2, self_weight<D>(nd.i, cp, sp) + self_weight<D>(nd.i, cm, sm), self);
      continue;
    }
    double om[D];
#pragma unroll
    for (int d = 0; d < D; ++d) om[d] = -o[d];
    int bp, bm;
    const double mup = ray_mu<D>(L, nd, o, bp);
    const double mum = ray_mu<D>(L, nd, om, bm);
    double A = 1.0, B = 1.0;
    if (bp >= 0 || bm >= 0) {
      const double sum = mup + mum;
      A = 2.0 / (mup * sum);
      B = 2.0 / (mum * sum);
    }
    const double wA = A * L.inv_2k2, wB = B * L.inv_2k2;
    wsum += wA + wB;
    int c[D];
    double s[D];
    cell_general<D>(L, nd, o, mup, bp, c, s);
    if (GATHER) acc = fma(wA, gather_interp<D>(L, v, c, s), acc);
    if (SELF) self = fma(wA, self_weight<D>(nd.i, c, s), self);
    cell_general<D>(L, nd, om, mum, bm, c, s);
    if (GATHER) acc = fma(wB, gather_interp<D>(L, v, c, s), acc);
    if (SELF) self = fma(wB, self_weight<D>(nd.i, c, s), self);
  }
  // drift pair: y_{P+1} = k^2 b, both endpoints equal, A = B = 1/mu (total weight 2/(mu 2k^2))
  {
    const double* bd_ = C.b_dir + a * D;
    double o[D];
    bool nz = false, inside = true;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      o[d] = L.k2h * fma(nd.bs, __ldg(bd_ + d), nd.bn[d]);
      nz |= (o[d] != 0.0);
      inside &= (fabs(o[d]) <= nd.dist[d]);
    }
    if (nz && inside) {  // untruncated drift endpoint (mu = 1)
      int c[D];
      double s[D];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        Split P_;
        split_p(o[d], nd.i[d], nm2, P_);
        c[d] = P_.c; s[d] = P_.s;
      }
      wsum += L.inv_k2;
      if (GATHER) acc = fma(L.inv_k2, gather_interp<D>(L, v, c, s), acc);
      if (SELF) self = fma(L.inv_k2, self_weight<D>(nd.i, c, s), self);
    } else if (nz) {
      int bdim;
      const double mu = ray_mu<D>(L, nd, o, bdim);
      int c[D];
      double s[D];
      cell_general<D>(L, nd, o, mu, bdim, c, s);
      const double w = (bdim >= 0) ? L.inv_k2 / mu : L.inv_k2;
      wsum += w;
      if (GATHER) acc = fma(w, gather_interp<D>(L, v, c, s), acc);
      if (SELF) self = fma(w, self_weight<D>(nd.i, c, s), self);
    }
  }
}

// ----------------------------------------------------------------------------- two-phase row
// The hot kernels evaluate a row in two phases: (1) the geometry of ALL 2P+1 endpoints (fp64, no
// memory traffic beyond the control tables), (2) all 2^d (2P+1) gathers issued back to back, so
// their L2 latencies overlap instead of serialising endpoint by endpoint.
template <int D>
struct Tap {
  int c[D];      // cell (lowest corner), global multi-index
  double s[D];   // fractions in the cell
  double w;      // weight w_e (0 for a skipped zero step)
  int face = -1; // truncated endpoint: its face of dOmega, 2 d + (upper side); -1 otherwise
};

template <int D>
__device__ __forceinline__ int tap_base(const LevelDev& L, const Tap<D>& t) {
  if (D == 2) return (t.c[1] - (int)L.local_row0) * L.n + t.c[0];
  return ((t.c[2] - (int)L.local_row0) * L.n + t.c[1]) * L.n + t.c[0];
}

template <int D>
__device__ __forceinline__ double tap_value(const LevelDev& L, const double* __restrict__ v, const Tap<D>& t) {
  HJB_ASSERT(tap_base<D>(L, t) >= 0 &&
             tap_base<D>(L, t) + (D == 2 ? L.n + 1 : L.n * L.n + L.n + 1) < L.local_elems);
  return interp_at<D, false>(v + tap_base<D>(L, t), L.n, L.n * L.n, t.s);
}

// fp32 multigrid vectors (hjb_mg_params.precision = 1): the cell corners are fp32, the fractions
// (fp64 geometry) rounded once to fp32, the multilinear combination in fp32 -- a preconditioner
// approximation, never part of a residual the solver stops on (reading xxxi)
template <int D>
__device__ __forceinline__ double interp_at_f32(const float* __restrict__ p, int sy, int sz, const double* sd) {
  const float s0 = (float)sd[0], s1 = (float)sd[1];
  if (D == 2) {
    const float v00 = __ldg(p), v10 = __ldg(p + 1);
    const float v01 = __ldg(p + sy), v11 = __ldg(p + sy + 1);
    const float a = fmaf(s0, v10 - v00, v00);
    const float b = fmaf(s0, v11 - v01, v01);
    return (double)fmaf(s1, b - a, a);
  } else {
    const float s2 = (float)sd[D > 2 ? 2 : 0];
    const float v000 = __ldg(p), v100 = __ldg(p + 1);
    const float v010 = __ldg(p + sy), v110 = __ldg(p + sy + 1);
    const float v001 = __ldg(p + sz), v101 = __ldg(p + sz + 1);
    const float v011 = __ldg(p + sz + sy), v111 = __ldg(p + sz + sy + 1);
    const float a0 = fmaf(s0, v100 - v000, v000);
    const float b0 = fmaf(s0, v110 - v010, v010);
    const float a1 = fmaf(s0, v101 - v001, v001);
    const float b1 = fmaf(s0, v111 - v011, v011);
    const float p0 = fmaf(s1, b0 - a0, a0);
    const float p1 = fmaf(s1, b1 - a1, a1);
    return (double)fmaf(s2, p1 - p0, p0);
  }
}

template <int D>
__device__ __forceinline__ double tap_value(const LevelDev& L, const float* __restrict__ v, const Tap<D>& t) {
  HJB_ASSERT(tap_base<D>(L, t) >= 0 &&
             tap_base<D>(L, t) + (D == 2 ? L.n + 1 : L.n * L.n + L.n + 1) < L.local_elems);
  return interp_at_f32<D>(v + tap_base<D>(L, t), L.n, L.n * L.n, t.s);
}

// cubic Lagrange weights at x for nodes 0, 1, 2, 3
__device__ __forceinline__ void cubic_weights(double x, double* w) {
  const double a = x - 1.0, b = x - 2.0, c = x - 3.0;
  w[0] = -a * b * c / 6.0;
  w[1] = x * b * c / 2.0;
  w[2] = -x * a * c / 2.0;
  w[3] = x * a * b / 6.0;
}

// psi(z) at a truncated endpoint on face t.face (exact-psi mode): cubic (2D) / bicubic (3D) Lagrange
// interpolation of the face samples, the 4 samples nearest to z per along-face axis (one-sided at the
// ends); along-face position z_e = c_e + s_e grid units = (c_e + s_e) brefine sample units
template <int D>
__device__ __forceinline__ double face_value(const CoefDev& C, const Tap<D>& t) {
  const int bd = t.face >> 1;
  const int M = C.bM;
  const double* F = C.bsamp + (int64_t)t.face * (D == 2 ? M : (int64_t)M * M);
  int k0[2];
  double w[2][4];
  int e = 0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    if (d == bd) continue;
    const double q = ((double)t.c[d] + t.s[d]) * C.brefine;
    int k = (int)floor(q) - 1;
    k = max(0, min(k, M - 4));
    k0[e] = k;
    cubic_weights(q - k, w[e]);
    ++e;
  }
  if (D == 2) {
    double v = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) v = fma(w[0][i], __ldg(F + k0[0] + i), v);
    return v;
  }
  double v = 0.0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    double r = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) r = fma(w[0][i], __ldg(F + (int64_t)(k0[1] + j) * M + k0[0] + i), r);
    v = fma(w[1][j], r, v);
  }
  return v;
}

// tap value on a vector v that is U itself: exact-psi mode (C.bsamp) replaces the interpolation of the
// nodal boundary values at a truncated endpoint by psi(z)
template <int D>
__device__ __forceinline__ double tap_value_u(const LevelDev& L, const CoefDev& C, const double* __restrict__ v,
                                              const Tap<D>& t) {
  if (C.bsamp != nullptr && t.face >= 0) return face_value<D>(C, t);
  return tap_value<D>(L, v, t);
}

// fp32 multigrid vectors are corrections with homogeneous boundary data: no face samples
template <int D>
__device__ __forceinline__ double tap_value_u(const LevelDev& L, const CoefDev&, const float* __restrict__ v,
                                              const Tap<D>& t) {
  return tap_value<D>(L, v, t);
}

// endpoints of control a at node nd: taps[2p] = +sigma_p, taps[2p+1] = -sigma_p, taps[2P] = drift.
// Returns wsum = sum_e w_e.
template <int D, int P>
__device__ __forceinline__ double row_geometry(const LevelDev& L, const double* sd, const double* bd_,
                                               const Node<D>& nd, Tap<D>* taps) {
  double wsum = 0.0;
  const int nm2 = L.n - 2;
#pragma unroll
  for (int p = 0; p < P; ++p) {
    double o[D];
    bool nz = false, inside = true;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      o[d] = L.kh * fma(nd.sc[p], sd[p * D + d], nd.sn[p][d]);
      nz |= (o[d] != 0.0);
      inside &= (fabs(o[d]) <= nd.dist[d]);
    }
    Tap<D>& tp = taps[2 * p];
    Tap<D>& tm = taps[2 * p + 1];
    if (inside) {  // untruncated pair (A = B = 1); a zero step gets weight 0 (its terms cancel)
#pragma unroll
      for (int d = 0; d < D; ++d) {
        pair_split(o[d], nd.i[d], tp.c[d], tp.s[d], tm.c[d], tm.s[d]);
        // |o| == dist: the endpoint sits on the upper face -> last cell with fraction 1
        if (tp.c[d] > nm2) { tp.c[d] = nm2; tp.s[d] = 1.0; }
        if (tm.c[d] > nm2) { tm.c[d] = nm2; tm.s[d] = 1.0; }
      }
      const double w = nz ? L.inv_2k2 : 0.0;
      tp.w = w;
      tm.w = w;
      wsum += 2.0 * w;
    } else {
      double om[D];
#pragma unroll
      for (int d = 0; d < D; ++d) om[d] = -o[d];
      int bp, bm;
      const double mup = ray_mu<D>(L, nd, o, bp);
      const double mum = ray_mu<D>(L, nd, om, bm);
      double A = 1.0, B = 1.0;
      if (bp >= 0 || bm >= 0) {
        const double sum = mup + mum;
        A = 2.0 / (mup * sum);
        B = 2.0 / (mum * sum);
      }
      tp.w = A * L.inv_2k2;
      tm.w = B * L.inv_2k2;
      wsum += tp.w + tm.w;
      cell_general<D>(L, nd, o, mup, bp, tp.c, tp.s);
      cell_general<D>(L, nd, om, mum, bm, tm.c, tm.s);
      tp.face = bp >= 0 ? 2 * bp + (o[bp] > 0.0 ? 1 : 0) : -1;
      tm.face = bm >= 0 ? 2 * bm + (om[bm] > 0.0 ? 1 : 0) : -1;
    }
  }
  {  // drift pair: y_{P+1} = k^2 b, both endpoints equal, A = B = 1/mu (total weight 2/(mu 2k^2))
    double o[D];
    bool nz = false, inside = true;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      o[d] = L.k2h * fma(nd.bs, bd_[d], nd.bn[d]);
      nz |= (o[d] != 0.0);
      inside &= (fabs(o[d]) <= nd.dist[d]);
    }
    Tap<D>& t = taps[2 * P];
    if (inside) {
#pragma unroll
      for (int d = 0; d < D; ++d) {
        single_split(o[d], nd.i[d], t.c[d], t.s[d]);
        if (t.c[d] > nm2) { t.c[d] = nm2; t.s[d] = 1.0; }
      }
      t.w = nz ? L.inv_k2 : 0.0;
    } else {
      int bdim;
      const double mu = ray_mu<D>(L, nd, o, bdim);
      cell_general<D>(L, nd, o, mu, bdim, t.c, t.s);
      t.w = (bdim >= 0) ? L.inv_k2 / mu : L.inv_k2;
      t.face = bdim >= 0 ? 2 * bdim + (o[bdim] > 0.0 ? 1 : 0) : -1;
    }
    wsum += t.w;
  }
  return wsum;
}

// ---- fast path: every endpoint strictly inside the box (no truncation; A = B = 1, mu_d = 1).
// Offsets o (cells) of the 2P diffusion steps and the drift step, as the general path forms them.
template <int D, int P>
__device__ __forceinline__ void row_offsets(const LevelDev& L, const double* sd, const double* bd,
                                            const Node<D>& nd, double (&o)[P + 1][D]) {
#pragma unroll
  for (int p = 0; p < P; ++p)
#pragma unroll
    for (int d = 0; d < D; ++d) o[p][d] = L.kh * fma(nd.sc[p], sd[p * D + d], nd.sn[p][d]);
#pragma unroll
  for (int d = 0; d < D; ++d) o[P][d] = L.k2h * fma(nd.bs, bd[d], nd.bn[d]);
}

// |o| < dist strictly: i +- o lies in the open box, so no endpoint is truncated and every cell
// index stays within [0, n-2] without clamping
template <int D, int P>
__device__ __forceinline__ bool offsets_inside(const Node<D>& nd, const double (&o)[P + 1][D]) {
  bool in = true;
#pragma unroll
  for (int p = 0; p <= P; ++p)
#pragma unroll
    for (int d = 0; d < D; ++d) in &= fabs(o[p][d]) < nd.dist[d];
  return in;
}

// cells and fractions of all endpoints from one floor per (step, dimension): +o -> (i + fl, o - fl),
// -o -> (i - fl - [s != 0], 1 - s or 0); zero steps get weight 0 (their two terms cancel)
template <int D, int P>
__device__ __forceinline__ double row_geometry_fast(const LevelDev& L, const Node<D>& nd,
                                                    const double (&o)[P + 1][D], Tap<D>* taps) {
  double wsum = 0.0;
#pragma unroll
  for (int p = 0; p < P; ++p) {
    bool nz = false;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      pair_split(o[p][d], nd.i[d], taps[2 * p].c[d], taps[2 * p].s[d], taps[2 * p + 1].c[d], taps[2 * p + 1].s[d]);
      nz |= (o[p][d] != 0.0);
    }
    const double w = nz ? L.inv_2k2 : 0.0;
    taps[2 * p].w = w;
    taps[2 * p + 1].w = w;
    wsum += 2.0 * w;
  }
  bool nz = false;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    single_split(o[P][d], nd.i[d], taps[2 * P].c[d], taps[2 * P].s[d]);
    nz |= (o[P][d] != 0.0);
  }
  taps[2 * P].w = nz ? L.inv_k2 : 0.0;
  return wsum + taps[2 * P].w;
}

// geometry of control a (table rows sd, bd) at node nd: fast path when the whole warp is untruncated
template <int D, int P>
__device__ __forceinline__ double row_taps(const LevelDev& L, const double* sd, const double* bd,
                                           const Node<D>& nd, Tap<D>* taps) {
  double o[P + 1][D];
  row_offsets<D, P>(L, sd, bd, nd, o);
  if (__all_sync(__activemask(), offsets_inside<D, P>(nd, o))) return row_geometry_fast<D, P>(L, nd, o, taps);
  return row_geometry<D, P>(L, sd, bd, nd, taps);
}

// the control tables in shared memory: sigma_dir [K][P][D] | b_dir [K][D] | c_ctrl [K]
// (| f_ctrl [K] | f_basis [K][Q] with SRC)
template <int D, int P, bool SRC>
__device__ __forceinline__ void stage_tables(const CoefDev& C, double* tab) {
  const int nsd = C.K * P * D, nbd = C.K * D;
  const int tid = threadIdx.y * blockDim.x + threadIdx.x, nt = blockDim.x * blockDim.y;
  for (int e = tid; e < nsd; e += nt) tab[e] = __ldg(C.sigma_dir + e);
  for (int e = tid; e < nbd; e += nt) tab[nsd + e] = __ldg(C.b_dir + e);
  for (int e = tid; e < C.K; e += nt) tab[nsd + nbd + e] = __ldg(C.c_ctrl + e);
  if (SRC) {
    for (int e = tid; e < C.K; e += nt) tab[nsd + nbd + C.K + e] = __ldg(C.f_ctrl + e);
    for (int e = tid; e < C.K * C.Q; e += nt) tab[nsd + nbd + 2 * C.K + e] = __ldg(C.f_basis + e);
  }
  __syncthreads();
}

template <int D>
__device__ __forceinline__ double tap_self(const Node<D>& nd, const Tap<D>& t) {
  return t.w * self_weight<D>(nd.i, t.c, t.s);
}

// ----------------------------------------------------------------------------- reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ int block_linear() { return blockIdx.y * gridDim.x + blockIdx.x; }

// block-reduce NV values (sum, or max if MAXMASK bit set) and write partial[block*NV + k]
template <int NV, int NT = kTX>
__device__ __forceinline__ void block_reduce_store(double (&val)[NV], double* partial, unsigned maxmask = 0u) {
  constexpr int NW = NT / 32;
  __shared__ double sm[NV][NW];
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double v = ((maxmask >> k) & 1u) ? warp_max(val[k]) : warp_sum(val[k]);
    if (lane == 0) sm[k][wid] = v;
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const bool mx = (maxmask >> k) & 1u;
      double v = lane < NW ? sm[k][lane] : (mx ? -INFINITY : 0.0);
      v = mx ? warp_max(v) : warp_sum(v);
      if (lane == 0) partial[block_linear() * NV + k] = v;
    }
  }
}

}  // namespace hjb
