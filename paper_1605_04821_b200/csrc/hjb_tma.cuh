// hjb_tma.cuh -- the control search on 2D deep-interior tiles with TMA-staged windows (sm_100a).
//
// A CTA takes a tile of kWX x kWY nodes all of whose endpoints, for every control, are strictly
// inside the box (no truncation).  For each control a, the cells the tile's 2P+1 endpoints touch
// lie in 2P+1 windows (tile span + the jitter of the per-node scale fields); one thread loads them
// global -> shared with cp.async.bulk.tensor (TMA) into one of two stages while the CTA evaluates
// H^a from the other stage (double buffering across controls, completion on mbarriers), so every
// gather of the search is a shared-memory load.
//
// Row pitch: the grid has n (odd) doubles per row, which a TMA tensor map cannot describe (global
// strides must be multiples of 16 bytes).  The map therefore views the array as PAIRS of rows
// ({2n, rows/2}, stride 16 n bytes): local row 2y' is x in [0, n) of pair-row y', local row 2y'+1
// is x in [n, 2n).  Each window is two boxes, its even and its odd rows.  The first element of a
// box must be 16-byte aligned (an odd FLOAT64 start coordinate is an illegal instruction on the
// B200, tools/tma_test.cu), so each box starts at the even element at or just before the window.
#pragma once
#include <cuda.h>  // CUtensorMap (type only; the encoder is fetched through cudaGetDriverEntryPoint)

#include "hjb_device.cuh"

namespace hjb {

constexpr int kWX = 32, kWY = 8, kWT = kWX * kWY;

struct TmaGeom {
  int bw, bh;        // box: bw doubles x bh pair-rows (one parity of a window)
  int slot;          // doubles per box slot in shared memory (128-byte multiple)
  int ntx, nty;      // tiles
  SkipRect tiles;    // tile rectangle in (col, row) loop coordinates
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_arrive(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  for (long long spin = 0; !done; ++spin) {
    if (spin > (1LL << 28)) __trap();  // a lost transaction: fail loudly instead of hanging
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"((uint64_t)map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// window origin (global cells) of endpoint e of control a for the tile whose first node is (ix0, iy0):
// every endpoint of the tile lies in [ix0 + omin, ix0 + kWX - 1 + omax] (+1 for the interpolation),
// omin/omax from the per-rank ranges rng = [scmin_p, scmax_p]_p, [bsmin, bsmax]
template <int P>
__device__ __forceinline__ void win_origin(const LevelDev& L, const double* sd, const double* bd, int e,
                                           const double* rng, int ix0, int iy0, int& wx0, int& wy0) {
  double lo[2];
#pragma unroll
  for (int d = 0; d < 2; ++d) {
    double c, f0, f1;
    if (e < 2 * P) {
      const int p = e >> 1;
      c = L.kh * ((e & 1) ? -sd[p * 2 + d] : sd[p * 2 + d]);
      f0 = rng[2 * p];
      f1 = rng[2 * p + 1];
    } else {
      c = L.k2h * bd[d];
      f0 = rng[2 * P];
      f1 = rng[2 * P + 1];
    }
    lo[d] = fmin(c * f0, c * f1) - 1e-6;
  }
  wx0 = ix0 + (int)floor(lo[0]);
  wy0 = iy0 + (int)floor(lo[1]);
}

#ifndef HJB_TMA_MINB
#define HJB_TMA_MINB 2   // <= 128 registers: two CTAs per SM overlap each other's TMA waits
#endif
template <int P>
__global__ void __launch_bounds__(kWT, HJB_TMA_MINB) k_search_tma(LevelDev L, CoefDev C, double dt,
                                                       const double* __restrict__ U,
                                                       const double* __restrict__ Uprev,
                                                       uint8_t* __restrict__ pol, double* __restrict__ F,
                                                       double* partial, TmaGeom W, const double* __restrict__ rng_g,
                                                       const __grid_constant__ CUtensorMap umap) {
  constexpr int D = 2, E = 2 * P + 1;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ int org[2][E][4];  // x origin (cells) of the even / odd box, first even / odd pair-row
  __shared__ double rng[2 * P + 2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // control tables (stage_tables<SRC> layout): sigma_dir | b_dir | c_ctrl | f_ctrl | f_basis
  const int ntab = C.K * (P * D + D + 2 + C.Q);
  for (int e = tid; e < C.K * P * D; e += kWT) sm[e] = __ldg(C.sigma_dir + e);
  for (int e = tid; e < C.K * D; e += kWT) sm[C.K * P * D + e] = __ldg(C.b_dir + e);
  for (int e = tid; e < C.K; e += kWT) {
    sm[C.K * (P * D + D) + e] = __ldg(C.c_ctrl + e);
    sm[C.K * (P * D + D + 1) + e] = __ldg(C.f_ctrl + e);
  }
  for (int e = tid; e < C.K * C.Q; e += kWT) sm[C.K * (P * D + D + 2) + e] = __ldg(C.f_basis + e);
  if (tid < 2 * P + 2) rng[tid] = rng_g[tid];
  const double* tsd = sm;
  const double* tbd = sm + C.K * P * D;
  const double* tcc = tbd + C.K * D;
  const double* tfc = tcc + C.K;
  const double* tfb = tfc + C.K;
  // [2 stages][E][2 parities][slot]; TMA destinations must be 128-byte aligned and the dynamic
  // shared window starts after the static variables, so align explicitly (+128 B in the launch)
  double* boxes = (double*)(((uintptr_t)(sm + ntab) + 127) & ~(uintptr_t)127);
  // the descriptor must stay in the parameter space: take its address here, at kernel scope (a
  // by-reference lambda capture of the parameter may materialise a local-memory copy, which TMA
  // cannot use)
  const CUtensorMap* const mp = &umap;
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)mp) : "memory");
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t uses[2] = {0u, 0u};
  const int lx = tid % kWX, ly = tid / kWX;
  const int lr0 = (int)L.local_row0;
  const int n = L.n;
  double red[2] = {0.0, 0.0};

  // thread 0: load the 2(2P+1) boxes of control a for the tile at (ix0, iy0) into stage st
  auto issue = [&, mp](int a, int st, int ix0, int iy0) {
    if (tid != 0) return;
    const double* sd = tsd + a * P * D;
    const double* bd = tbd + a * D;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of the stage done
    mbar_expect_arrive(&bars[st], (uint32_t)(E * 2 * W.bw * W.bh * 8));
#pragma unroll
    for (int e = 0; e < E; ++e) {
      int wx0, wy0;
      win_origin<P>(L, sd, bd, e, rng, ix0, iy0, wx0, wy0);
      const int r0 = wy0 - lr0;
      const int ye = (r0 + 1) >> 1, yo = r0 >> 1;
      const int xe = wx0 - (wx0 & 1), xo = wx0 - ((n + wx0) & 1);  // 16-byte aligned box starts
      org[st][e][0] = xe;
      org[st][e][1] = xo;
      org[st][e][2] = ye;
      org[st][e][3] = yo;
      double* b0 = boxes + (size_t)((st * E + e) * 2) * W.slot;
      tma_load_2d(b0, mp, xe, ye, &bars[st]);
      tma_load_2d(b0 + W.slot, mp, n + xo, yo, &bars[st]);
    }
  };

  const int ntiles = W.ntx * W.nty;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int ty = t / W.ntx, tx = t - ty * W.ntx;
    const int col = W.tiles.c0 + tx * kWX + lx, row = W.tiles.r0 + ty * kWY + ly;
    const int ix0 = 1 + W.tiles.c0 + tx * kWX, iy0 = (int)L.row_first + W.tiles.r0 + ty * kWY;
    Node<D> nd;
    node_at<D>(L, col, row, nd);
    load_fields<D>(C, nd);
    double feat[kMaxQ];
#pragma unroll
    for (int q = 0; q < kMaxQ; ++q) feat[q] = (q < C.Q) ? __ldg(C.f_feat + q * C.ld + nd.loc) : 0.0;
    const double Uj = __ldg(U + nd.loc);
    double best = INFINITY, fbest = 0.0;
    int arg = 0;
    __syncthreads();  // the previous tile is done with both stages
    issue(0, 0, ix0, iy0);
    if (C.K > 1) issue(1, 1, ix0, iy0);
    for (int a = 0; a < C.K; ++a) {
      const int st = a & 1;
      mbar_wait(&bars[st], uses[st] & 1u);
      uses[st] += 1;
      double o[P + 1][D];
      row_offsets<D, P>(L, tsd + a * P * D, tbd + a * D, nd, o);
      Tap<D> taps[E];
      const double wsum = row_geometry_fast<D, P>(L, nd, o, taps);
      double acc = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int r = taps[e].c[1] - lr0;        // local row of the cell's lower edge
        const int q = r & 1, yq = r >> 1;        // its parity box and pair-row
        const int r1 = r + 1, q1 = r1 & 1, y1 = r1 >> 1;
        const double* bx = boxes + (size_t)((st * E + e) * 2) * W.slot;
        const double* p0 = bx + q * W.slot + (yq - org[st][e][2 + q]) * W.bw + (taps[e].c[0] - org[st][e][q]);
        const double* p1 = bx + q1 * W.slot + (y1 - org[st][e][2 + q1]) * W.bw + (taps[e].c[0] - org[st][e][q1]);
        const double v00 = p0[0], v10 = p0[1], v01 = p1[0], v11 = p1[1];
        const double aa = fma(taps[e].s[0], v10 - v00, v00);
        const double bb = fma(taps[e].s[0], v11 - v01, v01);
        acc = fma(taps[e].w, fma(taps[e].s[1], bb - aa, aa), acc);
      }
      double f = tfc[a];
      const double* fb = tfb + a * C.Q;
#pragma unroll
      for (int q = 0; q < kMaxQ; ++q)
        if (q < C.Q) f = fma(fb[q], feat[q], f);
      const double c = nd.cn + tcc[a];
      const double H = (acc - wsum * Uj) + c * Uj + f;
      if (H < best) {  // strict: lowest index wins exact ties (reading iv)
        best = H;
        arg = a;
        fbest = f;
      }
      __syncthreads();  // every thread is done with stage st
      if (a + 2 < C.K) issue(a + 2, st, ix0, iy0);
    }
    const double Up = __ldg(Uprev + nd.loc);
    const double R = fabs(Uj - Up - dt * best);
    const int old = pol[nd.loc];
    pol[nd.loc] = (uint8_t)arg;
    F[nd.loc] = fma(dt, fbest, Up);
    red[0] = fmax(red[0], (R == R) ? R : INFINITY);
    red[1] += (old != arg) ? 1.0 : 0.0;
  }
  __shared__ double rs[2][kWT / 32];
  double v0 = warp_max(red[0]), v1 = warp_sum(red[1]);
  if (lane == 0) {
    rs[0][warp] = v0;
    rs[1][warp] = v1;
  }
  __syncthreads();
  if (warp == 0) {
    v0 = lane < kWT / 32 ? rs[0][lane] : -INFINITY;
    v1 = lane < kWT / 32 ? rs[1][lane] : 0.0;
    v0 = warp_max(v0);
    v1 = warp_sum(v1);
    if (lane == 0) {
      partial[blockIdx.x * 2] = v0;
      partial[blockIdx.x * 2 + 1] = v1;
    }
  }
}

}  // namespace hjb
