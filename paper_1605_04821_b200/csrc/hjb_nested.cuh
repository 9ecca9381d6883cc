// hjb_nested.cuh -- nested iteration for the initial iterate of an implicit step (DESIGN.md reading
// xxx).  Policy iteration converges from any initial iterate to the unique
// discrete solution of the step (M-matrix, Howard); the paper starts from U^{n-1}
// (reading iii).  HJB_GUESS_NESTED starts instead from the same step solved on the grid coarsened
// 2^m times per axis (the paper's scheme on that grid: its own h and k = sqrt(h)), with the
// coefficient fields, U^{n-1} and psi(t_n) injected from coincident fine nodes, prolonged
// multilinearly to the fine interior.  Only the number of policy iterations changes.
#pragma once
#include "hjb_device.cuh"

namespace hjb {

// dst[k][q] = src[k][f * q] for every coarse node q of the full grid (one rank: no halo rows),
// nplanes planes with strides ldf (fine) and ldc (coarse)
template <int D>
__global__ void k_nest_inject(int64_t nf, int64_t nc, int f, const double* __restrict__ src, int64_t ldf,
                              double* __restrict__ dst, int64_t ldc, int nplanes) {
  int64_t total = nc;
  for (int d = 1; d < D; ++d) total *= nc;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = q, loc = 0, stride = 1;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int64_t i = r % nc;
      r /= nc;
      loc += (int64_t)f * i * stride;
      stride *= nf;
    }
    for (int k = 0; k < nplanes; ++k) dst[k * ldc + q] = __ldg(src + k * ldf + loc);
  }
}

// Uf_j = (multilinear interpolation of Uc)(x_j) at every fine INTERIOR node j (boundary entries of Uf,
// psi(t_n), are left as they are).  Fine node I lies at coarse coordinate I / f.
template <int D>
__global__ void k_nest_prolong(int64_t nf, int64_t nc, int f, const double* __restrict__ Uc,
                               double* __restrict__ Uf) {
  int64_t total = nf;
  for (int d = 1; d < D; ++d) total *= nf;
  const double inv_f = 1.0 / (double)f;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = q;
    int64_t c0[D];
    double s[D];
    bool interior = true;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int64_t i = r % nf;
      r /= nf;
      interior &= (i > 0 && i < nf - 1);
      c0[d] = i / f;
      s[d] = (double)(i - c0[d] * f) * inv_f;
      if (c0[d] > nc - 2) {  // only the last boundary node (not interior): keep indices in range
        c0[d] = nc - 2;
        s[d] = 1.0;
      }
    }
    if (!interior) continue;
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m < (1 << D); ++m) {
      double w = 1.0;
      int64_t loc = 0, stride = 1;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const bool hi = (m >> d) & 1;
        w *= hi ? s[d] : 1.0 - s[d];
        loc += (c0[d] + (hi ? 1 : 0)) * stride;
        stride *= nc;
      }
      if (w != 0.0) acc = fma(w, __ldg(Uc + loc), acc);
    }
    Uf[q] = acc;
  }
}

// increment form: Uf_j = Uprev_j + (multilinear interpolation of Uc - Uc_prev)(x_j) at every fine
// INTERIOR node (the coarse step's time increment added to the fine U^{n-1})
template <int D>
__global__ void k_nest_prolong_inc(int64_t nf, int64_t nc, int f, const double* __restrict__ Uc,
                                   const double* __restrict__ Ucp, const double* __restrict__ Uprev,
                                   double* __restrict__ Uf) {
  int64_t total = nf;
  for (int d = 1; d < D; ++d) total *= nf;
  const double inv_f = 1.0 / (double)f;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = q;
    int64_t c0[D];
    double s[D];
    bool interior = true;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int64_t i = r % nf;
      r /= nf;
      interior &= (i > 0 && i < nf - 1);
      c0[d] = i / f;
      s[d] = (double)(i - c0[d] * f) * inv_f;
      if (c0[d] > nc - 2) {
        c0[d] = nc - 2;
        s[d] = 1.0;
      }
    }
    if (!interior) continue;
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m < (1 << D); ++m) {
      double w = 1.0;
      int64_t loc = 0, stride = 1;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const bool hi = (m >> d) & 1;
        w *= hi ? s[d] : 1.0 - s[d];
        loc += (c0[d] + (hi ? 1 : 0)) * stride;
        stride *= nc;
      }
      if (w != 0.0) acc = fma(w, __ldg(Uc + loc) - __ldg(Ucp + loc), acc);
    }
    Uf[q] = __ldg(Uprev + q) + acc;
  }
}

}  // namespace hjb
