// hjb_device.cuh -- sm_100a device code for the implicit LISL/HJB hot path.
//
// Scheme (arXiv:1605.04821): Scheme 2 steps y+-_p = +-k sigma_p, y_{P+1} = k^2 b (PAPER.md:95-96,
// k = sqrt(h)), truncated to the box with mu = largest value in (0,1] keeping the segment in
// closed Omega, weights A = 2/(mu+^2+mu+mu-), B = 2/(mu-^2+mu-mu+), drift
// A = B = 1/mu, multilinear interpolation.  Row of the implicit system
// (theta = 1):
//     (A x)_j = x_j - dt [ sum_e w_e (I x(z_e) - x_j) + c_j x_j ],  w_e = {A,B}/(2k^2), 1/(mu_d k^2)
// and its diagonal D_j = 1 + dt (sum_e w_e - sum_e w_e w_j(z_e) - c_j).
//
// Everything is recomputed on the fly per (node, control): no per-policy matrix is stored.
// Thread mapping: one thread per interior node, consecutive threads = consecutive x1 (coalesced
// gathers: for x-independent sigma the endpoints of a warp are consecutive nodes), grid-stride over
// the owned interior in row order so the +-reach rows in flight stay L2-resident.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hjb {

constexpr int kThreads = 256;
constexpr int kMaxP = 3;
constexpr int kMaxQ = 16;

// ----------------------------------------------------------------------------- level geometry
struct LevelDev {
  int n;               // nodes per dimension on this level
  int nI;              // n - 2 interior nodes per dimension
  int64_t row_elems;   // n^(D-1)
  int64_t local_row0;  // global slowest-axis row of local row 0
  int64_t local_rows;  // rows held in a local array
  int64_t row_first;   // first owned interior row (global, slowest axis)
  int64_t n_own;       // owned interior nodes
  double lo, hi, h, inv_h;
  double k;            // SL diffusion step scale (k = sqrt(h_fine) by default)
  double k2;           // drift step scale and denominator (= h on the fine level, exactly)
  double inv_2k2, inv_k2;
};

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
};

template <int D>
struct NodeCtx {
  int i[D];          // global multi-index
  double x[D];       // coordinates
  int64_t loc;       // local linear offset
  double sc[kMaxP];  // sigma scale per column
  double sn[kMaxP][D];
  double bs, bn[D], cn;
};

// interior flat index t -> node
template <int D>
__device__ __forceinline__ void node_from_interior(const LevelDev& L, int64_t t, NodeCtx<D>& nd) {
  const int64_t nI = L.nI;
  if (D == 2) {
    int64_t r = t / nI;
    nd.i[0] = 1 + (int)(t - r * nI);
    nd.i[1] = (int)(L.row_first + r);
    nd.loc = (int64_t)(nd.i[1] - L.local_row0) * L.n + nd.i[0];
  } else {
    int64_t r = t / nI;
    nd.i[0] = 1 + (int)(t - r * nI);
    int64_t r2 = r / nI;
    nd.i[1] = 1 + (int)(r - r2 * nI);
    nd.i[2] = (int)(L.row_first + r2);
    nd.loc = ((int64_t)(nd.i[2] - L.local_row0) * L.n + nd.i[1]) * L.n + nd.i[0];
  }
#pragma unroll
  for (int d = 0; d < D; ++d) nd.x[d] = L.lo + (double)nd.i[d] * L.h;
}

template <int D>
__device__ __forceinline__ void load_fields(const CoefDev& C, NodeCtx<D>& nd) {
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

// ----------------------------------------------------------------------------- truncation
// mu = largest value in (0,1] with x + [0,mu] y inside [lo,hi]^D;
// bd = binding dimension (-1 if untruncated).
template <int D>
__device__ __forceinline__ double ray_mu(const LevelDev& L, const double* x, const double* y, int& bd) {
  double mu = 1.0;
  bd = -1;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const double z = x[d] + y[d];
    if (z > L.hi) {
      const double t = (L.hi - x[d]) / y[d];
      if (t < mu) { mu = t; bd = d; }
    } else if (z < L.lo) {
      const double t = (L.lo - x[d]) / y[d];
      if (t < mu) { mu = t; bd = d; }
    }
  }
  return mu;
}

// endpoint z = x + s*mu*y with the binding coordinate put exactly on the face (reading: snap)
template <int D>
__device__ __forceinline__ void endpoint(const LevelDev& L, const double* x, const double* y, double smu,
                                         int bd, double* z) {
#pragma unroll
  for (int d = 0; d < D; ++d) {
    double v = fma(smu, y[d], x[d]);
    v = fmin(fmax(v, L.lo), L.hi);
    if (d == bd) v = (smu * y[d] > 0.0) ? L.hi : L.lo;
    z[d] = v;
  }
}

// ----------------------------------------------------------------------------- interpolation
// cell of z: c = clamp(floor((z-lo)/h), 0, n-2), s = (z-lo)/h - c (reading vii)
template <int D>
__device__ __forceinline__ void cell_of(const LevelDev& L, const double* z, int* c, double* s) {
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const double t = (z[d] - L.lo) * L.inv_h;
    int ci = (int)floor(t);
    ci = ci < 0 ? 0 : (ci > L.n - 2 ? L.n - 2 : ci);
    c[d] = ci;
    s[d] = t - (double)ci;
  }
}

template <int D>
__device__ __forceinline__ double gather_interp(const LevelDev& L, const double* __restrict__ v, const int* c,
                                                const double* s) {
  if (D == 2) {
    const double* p = v + ((int64_t)(c[1] - L.local_row0) * L.n + c[0]);
    const double v00 = __ldg(p), v10 = __ldg(p + 1);
    const double v01 = __ldg(p + L.n), v11 = __ldg(p + L.n + 1);
    const double a = fma(s[0], v10 - v00, v00);
    const double b = fma(s[0], v11 - v01, v01);
    return fma(s[1], b - a, a);
  } else {
    const int64_t n = L.n, nn = n * n;
    const double* p = v + (((int64_t)(c[2] - L.local_row0) * n + c[1]) * n + c[0]);
    const double v000 = __ldg(p), v100 = __ldg(p + 1);
    const double v010 = __ldg(p + n), v110 = __ldg(p + n + 1);
    const double v001 = __ldg(p + nn), v101 = __ldg(p + nn + 1);
    const double v011 = __ldg(p + nn + n), v111 = __ldg(p + nn + n + 1);
    const double a0 = fma(s[0], v100 - v000, v000);
    const double b0 = fma(s[0], v110 - v010, v010);
    const double a1 = fma(s[0], v101 - v001, v001);
    const double b1 = fma(s[0], v111 - v011, v011);
    const double p0 = fma(s[1], b0 - a0, a0);
    const double p1 = fma(s[1], b1 - a1, a1);
    return fma(s[2], p1 - p0, p0);
  }
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
__device__ __forceinline__ void row_eval(const LevelDev& L, const CoefDev& C, const NodeCtx<D>& nd, int a,
                                         const double* __restrict__ v, double& acc, double& wsum,
                                         double& self) {
  acc = 0.0;
  wsum = 0.0;
  self = 0.0;
  const double* sd = C.sigma_dir + (int64_t)a * C.P * D;
#pragma unroll
  for (int p = 0; p < kMaxP; ++p) {
    if (p >= C.P) break;
    double y[D];
    bool nz = false;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      y[d] = L.k * fma(nd.sc[p], __ldg(sd + p * D + d), nd.sn[p][d]);
      nz |= (y[d] != 0.0);
    }
    if (!nz) continue;  // zero step: its two terms cancel exactly
    double ym[D];
#pragma unroll
    for (int d = 0; d < D; ++d) ym[d] = -y[d];
    int bp, bm;
    const double mup = ray_mu<D>(L, nd.x, y, bp);
    const double mum = ray_mu<D>(L, nd.x, ym, bm);
    double A = 1.0, B = 1.0;
    if (bp >= 0 || bm >= 0) {
      const double sum = mup + mum;
      A = 2.0 / (mup * sum);
      B = 2.0 / (mum * sum);
    }
    double zp[D], zm[D];
    endpoint<D>(L, nd.x, y, mup, bp, zp);
    endpoint<D>(L, nd.x, y, -mum, bm, zm);
    const double wA = A * L.inv_2k2, wB = B * L.inv_2k2;
    wsum += wA + wB;
    int c[D];
    double s[D];
    cell_of<D>(L, zp, c, s);
    if (GATHER) acc = fma(wA, gather_interp<D>(L, v, c, s), acc);
    if (SELF) self = fma(wA, self_weight<D>(nd.i, c, s), self);
    cell_of<D>(L, zm, c, s);
    if (GATHER) acc = fma(wB, gather_interp<D>(L, v, c, s), acc);
    if (SELF) self = fma(wB, self_weight<D>(nd.i, c, s), self);
  }
  // drift pair: y_{P+1} = k^2 b, both endpoints equal, A = B = 1/mu (total weight 2/(mu 2k^2))
  {
    const double* bd_ = C.b_dir + (int64_t)a * D;
    double y[D];
    bool nz = false;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      y[d] = L.k2 * fma(nd.bs, __ldg(bd_ + d), nd.bn[d]);
      nz |= (y[d] != 0.0);
    }
    if (nz) {
      int bdim;
      const double mu = ray_mu<D>(L, nd.x, y, bdim);
      double z[D];
      endpoint<D>(L, nd.x, y, mu, bdim, z);
      const double w = (bdim >= 0) ? L.inv_k2 / mu : L.inv_k2;
      wsum += w;
      int c[D];
      double s[D];
      cell_of<D>(L, z, c, s);
      if (GATHER) acc = fma(w, gather_interp<D>(L, v, c, s), acc);
      if (SELF) self = fma(w, self_weight<D>(nd.i, c, s), self);
    }
  }
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

// block-reduce NV values (sum, or max if MAXMASK bit set) and write partial[blockIdx.x*NV + k]
template <int NV>
__device__ __forceinline__ void block_reduce_store(double (&val)[NV], double* partial, unsigned maxmask = 0u) {
  __shared__ double sm[NV][kThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
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
      double v = lane < (kThreads / 32) ? sm[k][lane] : (mx ? -INFINITY : 0.0);
      v = mx ? warp_max(v) : warp_sum(v);
      if (lane == 0) partial[blockIdx.x * NV + k] = v;
    }
  }
}

}  // namespace hjb
