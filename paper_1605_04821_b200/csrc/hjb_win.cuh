// hjb_win.cuh -- the control search over the deep box with the tile's neighbourhood of U staged in
// shared memory (sm_100a).
//
// Every endpoint of every control of a deep node i lies within m_d cells of i along axis d (the
// per-axis reach, from the scale-field ranges; DESIGN.md §6 "deep rectangles"), and its
// interpolation cell corner within [i - m, i + m - 1].  A CTA takes a tile of T0 x T1 (x T2) nodes,
// copies the window [tile - m, tile + m] of U into shared memory ONCE, and then evaluates all K
// controls of all its nodes with shared-memory gathers: the window is reused K (2P+1) 2^d times per
// node.  Where the reach is small relative to a tile (3D, and the moderate 2D grids) this replaces
// L1/L2-latency-bound global gathers by shared-memory loads; at cfg4 (143-cell reach) the window
// does not fit and the direct deep kernel runs.  Geometry and arithmetic are those of
// k_search<D, P, true> (same helpers, same interpolation order), so results are bit-identical.
#pragma once
#include "hjb_device.cuh"

namespace hjb {

#ifndef HJB_WIN_NT
#define HJB_WIN_NT 512
#endif
#ifndef HJB_WIN_SPLIT
#define HJB_WIN_SPLIT 2
#endif
// threads per CTA; each node's K controls are split over kWinS threads (warps alternate control
// ranges, so the lanes of a warp are consecutive x nodes on the same control): more warps share one
// window, which is what hides the latency of the dependent geometry -> gather -> compare chain
constexpr int kWinNT = HJB_WIN_NT, kWinS = HJB_WIN_SPLIT, kWinNodes = kWinNT / kWinS;
#ifndef HJB_WIN_UNROLL
#define HJB_WIN_UNROLL 1
#endif
constexpr int kWinUnroll = HJB_WIN_UNROLL;  // controls interleaved per thread (A/B knob)

struct WinGeom {  // tiling of a box of nodes (loop coordinates, SkipRect) for k_search_win
  int t[3];    // tile extent per axis (x, then the 2D row / 3D y axis, then 3D planes; 2D: t[2] = 1)
  int m[3];    // window margin per axis (cells; m[2] = 0 in 2D)
  int w[3];    // window extent t + 2m
  int nt[3];   // tiles per axis over the deep box
  int ntiles;
  int tab;     // doubles of control tables at the start of shared memory (window follows)
};

// GEN = false: tiles of the deep box, lean untruncated geometry (k_search<D, P, true>'s);
// GEN = true: tiles of the whole interior, the general geometry with the warp vote (k_search<D, P,
// false>'s): truncated endpoints lie on the faces, still inside the window.
template <int D, int P, bool GEN>
__global__ void __launch_bounds__(kWinNT, 1) k_search_win(LevelDev L, CoefDev C, double dt,
                                                          const double* __restrict__ U,
                                                          const double* __restrict__ Uprev,
                                                          uint8_t* __restrict__ pol, double* __restrict__ F,
                                                          double* partial, SkipRect box, WinGeom wg) {
  constexpr int E = 2 * P + 1;
  extern __shared__ double tab[];
  stage_tables<D, P, true>(C, tab);
  const double* tsd = tab;
  const double* tbd = tab + C.K * P * D;
  const double* tcc = tbd + C.K * D;
  const double* tfc = tcc + C.K;
  const double* tfb = tfc + C.K;
  double* win = tab + wg.tab;
  // control-range merge buffers (kWinS > 1), behind the window
  double* cmb_h = win + wg.w[0] * wg.w[1] * wg.w[2];
  double* cmb_f = cmb_h + (kWinS - 1) * kWinNodes;
  int* cmb_a = (int*)(cmb_f + (kWinS - 1) * kWinNodes);
  const int tid = threadIdx.x;
  const int W0 = wg.w[0], W1 = wg.w[1], W01 = W0 * W1;
  const int nodes = wg.t[0] * wg.t[1] * wg.t[2];
  const int nlines = W1 * (D == 3 ? wg.w[2] : 1);
  double red[2] = {0.0, 0.0};
  for (int t = blockIdx.x; t < wg.ntiles; t += gridDim.x) {
    const int tx = t % wg.nt[0], tyz = t / wg.nt[0];
    const int ty = tyz % wg.nt[1], tz = tyz / wg.nt[1];
    // tile origin in loop coordinates (col; 2D slab row | 3D y; 3D slab plane) and in global cells
    const int col0 = box.c0 + tx * wg.t[0];
    const int a1 = (D == 2 ? box.r0 : box.y0) + ty * wg.t[1];
    const int a2 = box.r0 + tz * wg.t[2];
    int wo[3];
    wo[0] = 1 + col0 - wg.m[0];
    wo[1] = (D == 2 ? (int)L.row_first + a1 : 1 + a1) - wg.m[1];
    wo[2] = (D == 3 ? (int)L.row_first + a2 : 0) - wg.m[2];
    __syncthreads();  // the previous tile's gathers are done
    for (int ln = tid >> 5; ln < nlines; ln += kWinNT / 32) {
      const int l2 = (D == 3) ? ln / W1 : 0;
      const int gy = wo[1] + (ln - l2 * W1), gz = wo[2] + l2;
      bool ok;
      int base;
      if (D == 2) {
        ok = gy >= (int)L.local_row0 && gy < (int)(L.local_row0 + L.local_rows);
        base = (gy - (int)L.local_row0) * L.n;
      } else {
        ok = gy >= 0 && gy < L.n && gz >= (int)L.local_row0 && gz < (int)(L.local_row0 + L.local_rows);
        base = ((gz - (int)L.local_row0) * L.n + gy) * L.n;
      }
      double* dst = win + ln * W0;
      for (int x = tid & 31; x < W0; x += 32) {
        const int gx = wo[0] + x;
        dst[x] = (ok && gx >= 0 && gx < L.n) ? __ldg(U + base + gx) : 0.0;
      }
    }
    __syncthreads();
    const int sub = (tid >> 5) % kWinS;                        // control range of this thread
    const int slot = ((tid >> 5) / kWinS) * 32 + (tid & 31);     // node slot in a pass
    const int a_lo = (sub * C.K) / kWinS, a_hi = ((sub + 1) * C.K) / kWinS;
    for (int q0 = 0; q0 < nodes; q0 += kWinNodes) {
      const int q = q0 + slot;
      const int qx = q % wg.t[0], qr = q / wg.t[0];
      const int qy = qr % wg.t[1], qz = qr / wg.t[1];
      const int col = col0 + qx;
      bool valid = q < nodes && col < box.c1;
      int row = 0;
      if (D == 2) {
        valid = valid && a1 + qy < box.r1;
        row = a1 + qy;
      } else {
        valid = valid && a1 + qy < box.y1 && a2 + qz < box.r1;
        row = (a1 + qy) + L.nI * (a2 + qz);
      }
      Node<D> nd;
      double best = INFINITY, fbest = 0.0, Uj = 0.0;
      int arg = a_lo;
      if (valid) {
        node_at<D>(L, col, row, nd);
        load_fields<D>(C, nd);
        double feat[kMaxQ];
#pragma unroll
        for (int k = 0; k < kMaxQ; ++k) feat[k] = (k < C.Q) ? __ldg(C.f_feat + k * C.ld + nd.loc) : 0.0;
        Uj = __ldg(U + nd.loc);
#pragma unroll kWinUnroll
        for (int a = a_lo; a < a_hi; ++a) {
          Tap<D> taps[E];
          double wsum;
          if (GEN) {
            wsum = row_taps<D, P>(L, tsd + a * P * D, tbd + a * D, nd, taps);
          } else {
            double o[P + 1][D];
            row_offsets<D, P>(L, tsd + a * P * D, tbd + a * D, nd, o);
            wsum = row_geometry_fast<D, P>(L, nd, o, taps);
          }
          double vals[E];
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int off = (taps[e].c[0] - wo[0]) + W0 * (taps[e].c[1] - wo[1]) +
                            (D == 3 ? W01 * (taps[e].c[D - 1] - wo[2]) : 0);
            vals[e] = interp_at<D, true>(win + off, W0, W01, taps[e].s);
          }
          double acc = 0.0;
#pragma unroll
          for (int e = 0; e < E; ++e) acc = fma(taps[e].w, vals[e], acc);
          // H^a_j = sum_e w_e I U(z_e) - wsum U_j + c^a_j U_j + f^a_j  (as k_search)
          double f = tfc[a];
          const double* fb = tfb + a * C.Q;
#pragma unroll
          for (int k = 0; k < kMaxQ; ++k)
            if (k < C.Q) f = fma(fb[k], feat[k], f);
          const double c = nd.cn + tcc[a];
          const double H = (acc - wsum * Uj) + c * Uj + f;
          if (H < best) {  // strict: lowest index wins exact ties (reading iv)
            best = H;
            arg = a;
            fbest = f;
          }
        }
      }
      if (kWinS > 1) {
        // merge the control ranges in index order: a later range wins only with a strictly smaller
        // minimum, which is the sequential strict-less scan's result (lowest index on exact ties)
        __syncthreads();
        if (valid && sub > 0) {
          cmb_h[(sub - 1) * kWinNodes + slot] = best;
          cmb_f[(sub - 1) * kWinNodes + slot] = fbest;
          cmb_a[(sub - 1) * kWinNodes + slot] = arg;
        }
        __syncthreads();
        if (valid && sub == 0)
          for (int r = 0; r < kWinS - 1; ++r) {
            const double h = cmb_h[r * kWinNodes + slot];
            if (h < best) {
              best = h;
              arg = cmb_a[r * kWinNodes + slot];
              fbest = cmb_f[r * kWinNodes + slot];
            }
          }
      }
      if (valid && sub == 0) {
        const double Up = __ldg(Uprev + nd.loc);
        const double R = fabs(Uj - Up - dt * best);
        const int old = pol[nd.loc];
        pol[nd.loc] = (uint8_t)arg;
        F[nd.loc] = fma(dt, fbest, Up);
        red[0] = fmax(red[0], (R == R) ? R : INFINITY);
        red[1] += (old != arg) ? 1.0 : 0.0;
      }
    }
  }
  block_reduce_store<2, kWinNT>(red, partial, 0x1u);
}

}  // namespace hjb
