// hjb_galerkin.cuh -- Galerkin coarse operators for the geometric multigrid (
// "the prolongation operator bilinear interpolation, the restriction the
// transpose of the prolongation, and the coarse grid operator is constructed using the Galerkin
// principle").  2D, one rank.
//
//   A_{l+1} = R A_l P,  P = bilinear prolongation from the coarse interior (zero Dirichlet coarse
//   boundary), R = P^T / 4 (full weighting; the 1/4 cancels in the coarse correction P A^-1 R).
//
// Two passes per level, each a plain sparse product with a per-row merge of duplicate columns:
//   B = A_l P   (fine rows: level 0 matrix-free from the scheme's row geometry, levels >= 1 from the
//                ELL arrays of A_l), then A_{l+1} = R B (coarse rows: 9 fine rows each).
// Merging uses a small open-addressing table in thread-local memory filled in a fixed order, so the
// sums are deterministic (bitwise repeatable).  Coarse operators are stored ELL, column-major
// ([slot][node], column = local linear index on the level grid, -1 = empty), interior rows only.
#pragma once
#include "hjb_device.cuh"

namespace hjb {

constexpr int kGalW = 96;   // ELL width of a coarse operator row
constexpr int kGalWB = 96;  // ELL width of a row of B = A P
constexpr int kGalHash = 256;
constexpr double kGalOmega = 0.6;  // Jacobi damping cap on Galerkin levels (reading xxix)

struct RowAcc {  // per-thread accumulator of (column, value) pairs
  int key[kGalHash];
  double val[kGalHash];
  int order[kGalHash];  // insertion order of the occupied slots
  int cnt;
};

__device__ __forceinline__ void acc_init(RowAcc& A) {
  for (int i = 0; i < kGalHash; ++i) A.key[i] = -1;
  A.cnt = 0;
}
// returns false on overflow
__device__ __forceinline__ bool acc_add(RowAcc& A, int col, double v) {
  unsigned h = ((unsigned)col * 2654435761u) & (kGalHash - 1);
  for (int probe = 0; probe < kGalHash; ++probe) {
    const int s = (h + probe) & (kGalHash - 1);
    if (A.key[s] == col) {
      A.val[s] += v;
      return true;
    }
    if (A.key[s] < 0) {
      A.key[s] = col;
      A.val[s] = v;
      A.order[A.cnt++] = s;
      return true;
    }
  }
  return false;
}

// coarse parents of a fine index i (0..nf-1) along one axis: up to 2 (index, weight); coarse boundary
// parents (0, nc-1) are dropped (zero Dirichlet correction)
__device__ __forceinline__ int parents(int i, int nc, int* pc, double* pw) {
  int k = 0;
  if ((i & 1) == 0) {
    const int c = i >> 1;
    if (c >= 1 && c <= nc - 2) { pc[k] = c; pw[k] = 1.0; ++k; }
  } else {
    const int c0 = i >> 1, c1 = c0 + 1;
    if (c0 >= 1 && c0 <= nc - 2) { pc[k] = c0; pw[k] = 0.5; ++k; }
    if (c1 >= 1 && c1 <= nc - 2) { pc[k] = c1; pw[k] = 0.5; ++k; }
  }
  return k;
}

// add a * P[i, :] for fine node (i0, i1) to the accumulator (coarse columns on the coarse grid n_c)
__device__ __forceinline__ bool add_prolonged(RowAcc& A, int i0, int i1, int nc, double a) {
  int p0[2], p1[2];
  double w0[2], w1[2];
  const int k0 = parents(i0, nc, p0, w0), k1 = parents(i1, nc, p1, w1);
  bool ok = true;
  for (int b = 0; b < k1; ++b)
    for (int c = 0; c < k0; ++c) ok &= acc_add(A, p1[b] * nc + p0[c], a * (w1[b] * w0[c]));
  return ok;
}

// write the accumulator as one ELL row (slots in insertion order); false on overflow
__device__ __forceinline__ bool acc_store(const RowAcc& A, int W, int64_t ld, int64_t row, int* cols, double* vals) {
  if (A.cnt > W) return false;
  for (int k = 0; k < W; ++k) {
    if (k < A.cnt) {
      const int s = A.order[k];
      cols[k * ld + row] = A.key[s];
      vals[k * ld + row] = A.val[s];
    } else {
      cols[k * ld + row] = -1;
      vals[k * ld + row] = 0.0;
    }
  }
  return true;
}

// B = A_0 P for the fine level (matrix-free rows of the implicit operator A = I - dt (L_hat + c) with
// the policy; interior columns only: boundary nodes are Dirichlet data, not unknowns).  B rows are
// stored at the fine row's local index; columns are coarse local indices.
template <int P>
__global__ void __launch_bounds__(128) k_gal_b_fine(LevelDev Lf, CoefDev C, double dt, const uint8_t* __restrict__ pol,
                                                   int nc, int* __restrict__ bcol, double* __restrict__ bval,
                                                   int* __restrict__ overflow) {
  constexpr int D = 2, E = 2 * P + 1;
  const int64_t ld = (int64_t)Lf.local_rows * Lf.row_elems;
  RowAcc A;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < (int64_t)Lf.nI * Lf.nrows;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(q / Lf.nI), col = (int)(q - (int64_t)row * Lf.nI);
    Node<D> nd;
    node_at<D>(Lf, col, row, nd);
    load_fields<D>(C, nd);
    const int a = pol[nd.loc];
    Tap<D> taps[E];
    const double wsum = row_geometry<D, P>(Lf, C.sigma_dir + a * P * D, C.b_dir + a * D, nd, taps);
    const double c = nd.cn + C.c_ctrl[a];
    acc_init(A);
    bool ok = true;
    // diagonal part 1 + dt (wsum - c); the self weights come back through the corner loop below
    ok &= add_prolonged(A, nd.i[0], nd.i[1], nc, 1.0 + dt * (wsum - c));
    for (int e = 0; e < E; ++e) {
      if (taps[e].w == 0.0) continue;
      for (int m = 0; m < 4; ++m) {
        const int hx = m & 1, hy = m >> 1;
        const int j0 = taps[e].c[0] + hx, j1 = taps[e].c[1] + hy;
        if (j0 < 1 || j0 > Lf.n - 2 || j1 < 1 || j1 > Lf.n - 2) continue;  // boundary corner: data
        const double wc = (hx ? taps[e].s[0] : 1.0 - taps[e].s[0]) * (hy ? taps[e].s[1] : 1.0 - taps[e].s[1]);
        if (wc == 0.0) continue;
        ok &= add_prolonged(A, j0, j1, nc, -dt * taps[e].w * wc);
      }
    }
    if (!ok || !acc_store(A, kGalWB, ld, nd.loc, bcol, bval)) atomicExch(overflow, 1);
  }
}

// B = A_l P for a coarse level l >= 1 stored ELL (columns: local indices on the level grid n_l)
__global__ void __launch_bounds__(128) k_gal_b_ell(LevelDev Lf, const int* __restrict__ acol,
                                                  const double* __restrict__ aval, int nc, int* __restrict__ bcol,
                                                  double* __restrict__ bval, int* __restrict__ overflow) {
  const int64_t ld = (int64_t)Lf.local_rows * Lf.row_elems;
  RowAcc A;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < (int64_t)Lf.nI * Lf.nrows;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(q / Lf.nI), col = (int)(q - (int64_t)row * Lf.nI);
    const int loc = (1 + row) * Lf.n + 1 + col;
    acc_init(A);
    bool ok = true;
    for (int k = 0; k < kGalW; ++k) {
      const int j = acol[k * ld + loc];
      if (j < 0) break;
      const int j1 = j / Lf.n, j0 = j - j1 * Lf.n;
      ok &= add_prolonged(A, j0, j1, nc, aval[k * ld + loc]);
    }
    if (!ok || !acc_store(A, kGalWB, ld, loc, bcol, bval)) atomicExch(overflow, 1);
  }
}

// A_{l+1} = R B: coarse row (I0, I1) sums the B rows of the fine interior nodes (2 I + d), d in
// {-1,0,1}^2, weighted (1/4, 1/2, 1/4) per axis (the full weighting of k_restrict)
__global__ void __launch_bounds__(128) k_gal_rb(LevelDev Lf, LevelDev Lc, const int* __restrict__ bcol,
                                               const double* __restrict__ bval, int* __restrict__ ccol,
                                               double* __restrict__ cval, int* __restrict__ overflow) {
  const int64_t ldf = (int64_t)Lf.local_rows * Lf.row_elems, ldc = (int64_t)Lc.local_rows * Lc.row_elems;
  RowAcc A;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < (int64_t)Lc.nI * Lc.nrows;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(q / Lc.nI), col = (int)(q - (int64_t)row * Lc.nI);
    const int I0 = 1 + col, I1 = 1 + row;
    acc_init(A);
    bool ok = true;
    for (int d1 = -1; d1 <= 1; ++d1)
      for (int d0 = -1; d0 <= 1; ++d0) {
        const int j0 = 2 * I0 + d0, j1 = 2 * I1 + d1;
        if (j0 < 1 || j0 > Lf.n - 2 || j1 < 1 || j1 > Lf.n - 2) continue;
        const double r = (d0 == 0 ? 0.5 : 0.25) * (d1 == 0 ? 0.5 : 0.25);
        const int64_t jl = (int64_t)j1 * Lf.n + j0;
        for (int k = 0; k < kGalWB; ++k) {
          const int c = bcol[k * ldf + jl];
          if (c < 0) break;
          ok &= acc_add(A, c, r * bval[k * ldf + jl]);
        }
      }
    const int64_t loc = (int64_t)I1 * Lc.n + I0;
    if (!ok || !acc_store(A, kGalW, ldc, loc, ccol, cval)) atomicExch(overflow, 1);
  }
}

// the diagonal of an ELL level (the smoother's D)
__global__ void __launch_bounds__(128) k_gal_diag(LevelDev L, const int* __restrict__ acol,
                                                 const double* __restrict__ aval, double* __restrict__ dg) {
  const int64_t ld = (int64_t)L.local_rows * L.row_elems;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < (int64_t)L.nI * L.nrows;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(q / L.nI), col = (int)(q - (int64_t)row * L.nI);
    const int loc = (1 + row) * L.n + 1 + col;
    double d = 0.0;
    for (int k = 0; k < kGalW; ++k) {
      const int j = acol[k * ld + loc];
      if (j < 0) break;
      if (j == loc) d += aval[k * ld + loc];
    }
    dg[loc] = d;
  }
}

// y = b - A x (RESID) or y = x + omega (b - A x) / D (JACOBI, D = dg) on an ELL level
template <bool JAC>
__global__ void __launch_bounds__(128) k_gal_sweep(LevelDev L, const int* __restrict__ acol,
                                                  const double* __restrict__ aval, const double* __restrict__ x,
                                                  const double* __restrict__ b, const double* __restrict__ dg,
                                                  double omega, double* __restrict__ y) {
  const int64_t ld = (int64_t)L.local_rows * L.row_elems;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < (int64_t)L.nI * L.nrows;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(q / L.nI), col = (int)(q - (int64_t)row * L.nI);
    const int loc = (1 + row) * L.n + 1 + col;
    double ax = 0.0;
    for (int k = 0; k < kGalW; ++k) {
      const int j = __ldg(acol + k * ld + loc);
      if (j < 0) break;
      HJB_ASSERT(j < ld);
      ax = fma(__ldg(aval + k * ld + loc), __ldg(x + j), ax);
    }
    const double r = __ldg(b + loc) - ax;
    y[loc] = JAC ? fma(omega, r / __ldg(dg + loc), __ldg(x + loc)) : r;
  }
}

// dense interior matrix of the coarsest level from its ELL rows (interior numbering t = row*nI + col)
__global__ void k_gal_dense(LevelDev L, const int* __restrict__ acol, const double* __restrict__ aval,
                            double* __restrict__ Ad) {
  const int64_t ld = (int64_t)L.local_rows * L.row_elems;
  const int Nc = L.nI * L.nrows;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < Nc; t += gridDim.x * blockDim.x) {
    const int row = t / L.nI, col = t - row * L.nI;
    const int loc = (1 + row) * L.n + 1 + col;
    for (int k = 0; k < kGalW; ++k) {
      const int j = acol[k * ld + loc];
      if (j < 0) break;
      const int j1 = j / L.n, j0 = j - j1 * L.n;
      Ad[(int64_t)t * Nc + (j1 - 1) * L.nI + (j0 - 1)] += aval[k * ld + loc];
    }
  }
}

}  // namespace hjb
