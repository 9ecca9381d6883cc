// hjb_search2.cuh -- the 2D deep-rectangle control search, restructured for the L1 data pipe
// (sm_100a).  Policy improvement of PAPER.md:147-156 (exhaustive linear search over the discrete
// control set, footnote P:156): for every deep node j and every control a, in index order,
//     H^a_j(U) = sum_e w_e I U(z_e) - (sum_e w_e) U_j + c^a_j U_j + f^a_j
// with the lowest-index argmin (reading iv).  Same geometry, same operands, same arithmetic order as
// k_search<2, P, true> (hjb_kernels.cuh) up to the rounding of equivalent formulations (the offset
// k sigma formed as (k sc) sd, the minus endpoint interpolated from the far corner, per-control
// weight sums): identical policies except at near-ties, F and R within rounding
// (tests/test_gpu_parity.py::test_deep_kernels_match_general).
//
// What bounds k_search<2, P, true> at BASELINE cfg4 (ncu, profiles/r01_v9_ncu_full_search_cfg4.md and
// DESIGN.md §6): the L1 data pipe (l1tex__data_pipe_lsu_wavefronts 71-83 % of peak): 20 scattered
// 8-byte gathers per (node, control) at ~4.2 wavefronts each, plus ~24 shared-memory wavefronts
// for the control tables.  This kernel removes both costs:
//   * the control tables live in the kernel PARAMETER space (a __grid_constant__ struct, constant
//     bank 0): a warp-uniform index a is served by the constant cache, not the L1 data pipe;
//   * each bilinear tap reads two 16-byte pairs (U_i, U_{i+1}) of rows c1 and c1+1 from a pair copy
//     UP[i] = (U[i], U[i+1]) built once per search (k_make_pairs): 2 LDG.128 instead of 4 LDG.64;
//   * the drift endpoint of the deep rectangle stays within one cell of the node (|h b^a / h| < 1,
//     checked on the host from the scale-field ranges), so its four taps come from the node's 3x3
//     neighbourhood of U held in registers (the quadrant is per control): no gathers at all;
//   * per (node, control) one floor per offset component serves both endpoints of a pair (the minus
//     endpoint is interpolated from the far corner of its cell), addresses are 32-bit offsets from the
//     node, and the weights / weight sum of the untruncated stencil are per-control table entries.
#pragma once
#include "hjb_device.cuh"

namespace hjb {

constexpr int kSTabN = 3072;  // doubles of control tables passed as a kernel parameter (24 KB)
struct STab {
  double v[kSTabN];  // per control a, stride P*2 + 2 + 2 + Q: sigma_dir [P][2] | b_dir [2] | c | f_ctrl | f_basis [Q]
};

// UP[i] = (U[i], U[i+1]) for every local element (the last one pairs with 0)
__global__ void __launch_bounds__(256) k_make_pairs(const double* __restrict__ U, double2* __restrict__ UP, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double a = __ldg(U + i);
    const double b = (i + 1 < n) ? __ldg(U + i + 1) : 0.0;
    UP[i] = make_double2(a, b);
  }
}

// Q4[i] = (U[i], U[i+1], U[i+n], U[i+n+1]): the four corners of the cell whose lower-left node is i,
// 32 bytes, so one 256-bit load (LDG.E.ENL2.256 on sm_100a) fetches a whole bilinear tap.  Entries
// whose corners leave the local array hold 0 (never read: deep nodes' cells are interior).
__global__ void __launch_bounds__(256) k_make_quads(const double* __restrict__ U, double4* __restrict__ Q4, int n,
                                                    int64_t ne) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ne; i += (int64_t)gridDim.x * blockDim.x) {
    const double a = __ldg(U + i);
    const double b = (i + 1 < ne) ? __ldg(U + i + 1) : 0.0;
    const double c = (i + n < ne) ? __ldg(U + i + n) : 0.0;
    const double d = (i + n + 1 < ne) ? __ldg(U + i + n + 1) : 0.0;
    double4* q = Q4 + i;
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(q), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
  }
}

// one 256-bit read-only load of a cell's four corners
__device__ __forceinline__ double4 ld_quad(const double4* q) {
  double4 r;
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(q));
  return r;
}
__device__ __forceinline__ const double4* quad_at(const double4* base, int off) {
  const double4* r;
  asm("mad.wide.s32 %0, %1, 32, %2;" : "=l"(r) : "r"(off), "l"(base));
  return r;
}

// bilinear value from the pairs (v00, v10) of row c1 and (v01, v11) of row c1+1 at fractions s
__device__ __forceinline__ double interp_pairs(const double2 lo, const double2 hi, double s0, double s1) {
  const double a = fma(s0, lo.y - lo.x, lo.x);
  const double b = fma(s0, hi.y - hi.x, hi.x);
  return fma(s1, b - a, a);
}
// the same bilinear value measured from the far corner: the cell's fractions are 1 - s0, 1 - s1
// (the minus endpoint x - o of an untruncated pair sits at (i - fl - 1) + (1 - s) per axis when
// x + o sits at (i + fl) + s, so it reuses the plus endpoint's s -- no separate split, and no
// special case at s = 0, where it reads the corner v11 exactly)
__device__ __forceinline__ double interp_pairs_mirror(const double2 lo, const double2 hi, double s0, double s1) {
  const double a = fma(-s0, lo.y - lo.x, lo.y);
  const double b = fma(-s0, hi.y - hi.x, hi.y);
  return fma(-s1, b - a, b);
}

// base + 16 off as one wide multiply-add (IMAD.WIDE) instead of a sign-extend + shift-add pair
__device__ __forceinline__ const double2* pair_at(const double2* base, int off) {
  const double2* r;
  asm("mad.wide.s32 %0, %1, 16, %2;" : "=l"(r) : "r"(off), "l"(base));
  return r;
}

// floor split of an offset o (|o| < 2^31): fl as an integer and the fraction s = o - fl (exact)
__device__ __forceinline__ void split_floor(double o, int& fl, double& s) {
  const double f = floor(o);
  s = o - f;
  fl = __double2loint(f + 6755399441055744.0);  // 1.5 * 2^52: the integer in the low word (no F2I)
}

// per-control uniform data of the parameter-space table, after the P*2 + 2 + 2 + Q scheme doubles:
//   w_p (P) | w_drift | wsum   -- the weights of the untruncated stencil (zero steps -> 0)
template <int P, int Q>
struct STabLayout {
  static constexpr int SD = 0, BD = 2 * P, C = 2 * P + 2, FC = 2 * P + 3, FB = 2 * P + 4, W = 2 * P + 4 + Q,
                       WD = W + P, WSUM = W + P + 1,
                       CMW = W + P + 2,  // c_ctrl - wsum (the diagonal part of H without c_node)
                       DQ = W + P + 3,   // [2] drift cell offset: 1 where the drift step is negative
                       ABD = W + P + 5,  // [2] |b_dir|: the drift step's magnitude per axis
                       S = W + P + 7;
};
// certified search skipping (k_search_deep2<..., GAP>): per-node gap bounds and this search's bound
struct GapArgs {
  float* gap;          // [N] lower bound of H_second - H_best per node (fp32, rounded down)
  double bskip;        // bound of |H^a_j(U) - H^a_j(U_old)| over all a, j; < 0: full scan everywhere
  double gmargin;      // rounding margin, U part: 4 * 32 eps (2 wsum + |c|)_max max|U|
  double fcmax;        // max_a |f_ctrl^a|
  double fbmax[8];     // max_a |f_basis^a_q|
  int* nskip;          // device counter of skipped CTAs
};
struct STabQuad {
  int v[256];  // drift endpoint quadrant per control: bit 0 = cell left of the node (x), bit 1 = below (y)
};

#ifndef HJB_SEARCH2_PAIRS
#define HJB_SEARCH2_PAIRS 0  // 1: 16-byte gathers from a pair copy (measured slower at cfg4:
                             // 2x the gather footprint, 102 vs 38 GB DRAM); 0: 8-byte gathers from U
#endif
// the two values (U_c, U_{c+1}) of the cell row at offset off from the node
#ifndef HJB_S2_PAIRSUM
#define HJB_S2_PAIRSUM 0  // 1: pair-summed corners, drift fraction by FMA, 2-op diagonal (12 fewer fp64
                          // operations per (node, control); measured slower at cfg4: 124 vs 107 ms)
#endif
#ifndef HJB_S2_EXP
#define HJB_S2_EXP 0  // bound experiments (tools/build_variant.sh): 1 = no gathers (tap
                      // values synthesised from the offsets); 2 = gathers kept, interpolation dropped
#endif
__device__ __forceinline__ double2 cell_row(const double2* up, const double* u, int off) {
#if HJB_S2_EXP == 1
  return make_double2(__hiloint2double(0x3ff00000, off), __hiloint2double(0x3ff00000, off + 1));
#endif
#if HJB_SEARCH2_PAIRS
  return __ldg(pair_at(up, off));
#else
  return make_double2(__ldg(u + off), __ldg(u + off + 1));
#endif
}

#ifndef HJB_SEARCH2_SYNC
#define HJB_SEARCH2_SYNC 8  // __syncthreads every 8 controls: the CTA's 4 lines stay in lockstep and
                            // share gathered lines in L1 (cfg4 search 135 -> 109 ms; 0 = off)
#endif
#ifndef HJB_S2Y
#define HJB_S2Y 4
#endif
constexpr int kS2Y = HJB_S2Y;         // lines per CTA (x: 32 consecutive nodes per warp)
constexpr int kS2T = 32 * kS2Y;       // threads per CTA
#ifndef HJB_SEARCH2_UNROLL
#define HJB_SEARCH2_UNROLL 1
#endif
constexpr int kS2Unroll = HJB_SEARCH2_UNROLL;  // controls per unrolled loop body (A/B knob)

#ifndef HJB_SUPER_COLS
#define HJB_SUPER_COLS 16
#endif
constexpr int kSuperCols = HJB_SUPER_COLS;  // tile columns per super-column (16 x 32 = 512 nodes)

#ifndef HJB_SEARCH2_MINB
#define HJB_SEARCH2_MINB 4
#endif
// Deep nodes only (every endpoint of every control strictly inside the box), no sigma/b offset
// fields, scale fields of one sign (so a control's zero steps and drift quadrant are per-control
// facts: host-checked), drift endpoints within one cell of the node.
// STRIP: a boundary-layer strip of the deep rectangle's ring: per control, a warp whose endpoints are
// all strictly inside runs the lean arithmetic above; otherwise the control takes the general
// truncated geometry (row_geometry, exact-psi aware) for the whole warp
// QUADS (deep rectangle only): the taps come from the corner copy Q4 (k_make_quads), one 256-bit load
// per endpoint, and an untruncated pair is combined before interpolating: the minus endpoint's cell
// is the plus endpoint's mirrored through the node and its fractions are 1 - s, so
//   I(x+o) + I(x-o) = bilinear(s; P00 + M11, P10 + M01, P01 + M10, P11 + M00)
// (P = the plus cell's corners, M = the minus cell's): 4 loads instead of 16 per (node, control) and
// 11 instead of 14 fp64 operations per pair.
// KU > 0: the control loop is fully unrolled for exactly KU = C.K controls, so every control-table
// entry is a constant-bank operand of its instruction (no LDC per entry).
// GAP (policy iteration inside hjb_step, deep rectangle, one rank): certified search skipping.
// gap[j] holds a lower bound of H_second - H_best at node j (fp32, rounded down) from the previous
// search of the step.  Between two searches H^a_j(U) changes by at most bskip for every a (the host
// bound from the per-axis cell differences of dU = U - U_old, DESIGN.md §6 "Certified search
// skipping"), so when gap[j] > 2 bskip + gmargin (gmargin: the rounding of both evaluations) the
// argmin at j cannot change.  A CTA whose nodes all pass that test evaluates only the current
// control of each node (F, R from it: bit-identical to the full scan, whose minimum it is) and
// lowers the stored gaps by 2 bskip; otherwise the CTA scans all K controls and stores fresh gaps.
// bskip < 0: full scan everywhere (the step's first search).
template <int P, int Q, bool STRIP = false, bool QUADS = false, int KU = 0, bool GAP = false>
__global__ void __launch_bounds__(kS2T, HJB_SEARCH2_MINB) k_search_deep2(LevelDev L, CoefDev C, double dt,
                                                                        const double* __restrict__ U,
                                                                        const double2* __restrict__ UP,
                                                                        const double4* __restrict__ Q4,
                                                                        const double* __restrict__ Uprev,
                                                                        uint8_t* __restrict__ pol,
                                                                        double* __restrict__ F, double* partial,
                                                                        SkipRect it, const __grid_constant__ STab tab,
                                                                        const __grid_constant__ STabQuad quad,
                                                                        const GapArgs ga) {
  using T = STabLayout<P, Q>;
  double red[2] = {0.0, 0.0};
  const int nk = box_lines(it);
  const int n = L.n;
  // tiles of kSBX columns x kS2Y lines, ordered so that the CTAs running at one time cover a compact
  // patch: super-columns of kSuperCols tile columns, walked top to bottom, left to right.  The
  // patch's gather window (+-reach rows and columns around it) then stays in L2; a full-width band
  // of lines (the operator kernels' order) with 16-byte pairs and a 143-row reach does not
  // (measured at cfg4: 229 GB of DRAM reads per search, L2 hit rate 47 %).
  const int tx = (it.c1 - it.c0 + kSBX - 1) / kSBX, ty = (nk + kS2Y - 1) / kS2Y;
  const int ntiles = tx * ty;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int sc = t / (kSuperCols * ty);               // super-column
    const int scw = min(kSuperCols, tx - sc * kSuperCols);
    const int tl = t - sc * kSuperCols * ty;            // tile within the super-column, row-major
    const int trow = tl / scw, tcol = sc * kSuperCols + (tl - trow * scw);
    const int k0 = trow * kS2Y + threadIdx.y;
    const int col0 = it.c0 + tcol * kSBX + threadIdx.x;
    const bool valid = k0 < nk && col0 < it.c1;
    // a lane past the box edge repeats the tile's first node (results dropped), so that every thread
    // of the CTA runs the control loop (HJB_SEARCH2_SYNC keeps the lines in lockstep)
    const int k = valid ? k0 : trow * kS2Y, col = valid ? col0 : it.c0 + tcol * kSBX;
    if (HJB_SEARCH2_SYNC > 0 || valid) {
      const int row = box_row<2>(L, it, k);
      Node<2> nd;
      node_at<2>(L, col, row, nd);
      load_fields<2>(C, nd);
      prefetch_ahead(L, U, nd.loc, col);
      double feat[Q > 0 ? Q : 1];
#pragma unroll
      for (int q = 0; q < Q; ++q) feat[q] = __ldg(C.f_feat + q * C.ld + nd.loc);
      const double Uj = __ldg(U + nd.loc);
      double nb[3][3];  // U at (i0 + c - 1, i1 + r - 1): nb[r][c]  (the drift endpoint's cells)
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) nb[r][c] = (r == 1 && c == 1) ? Uj : __ldg(U + nd.loc + (r - 1) * n + (c - 1));
      // one-sided differences of the 3x3 neighbourhood (index 0: towards -1, 1: towards +1)
      double ddx[2], ddy[2], ddxy[2][2];  // ddxy[y side][x side]
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        ddx[q] = nb[1][2 * q] - Uj;
        ddy[q] = nb[2 * q][1] - Uj;
      }
#pragma unroll
      for (int qy = 0; qy < 2; ++qy)
#pragma unroll
        for (int qx = 0; qx < 2; ++qx) ddxy[qy][qx] = (nb[2 * qy][2 * qx] - nb[1][2 * qx]) - (nb[2 * qy][1] - Uj);
      double ksc[P];
#pragma unroll
      for (int p = 0; p < P; ++p) ksc[p] = L.kh * nd.sc[p];
      const double kbs = L.k2h * nd.bs;
      const double2* up = UP + nd.loc;       // pairs of the node's row ...
      const double2* upn = up + n;           // ... and of the next row (one base per row: one
                                             // wide multiply-add per load address)
      const double* u0 = U + nd.loc;
      const double* u1 = u0 + n;
      const double4* q4 = Q4 + nd.loc;
      double best = INFINITY, fbest = 0.0, best2 = INFINITY;
      int arg = 0;
      // GAP: the CTA-uniform skip decision (lanes past the box edge vote yes)
      int a_lo = 0, a_hi = KU > 0 ? KU : C.K;
      bool skip = false;
      float gj = 0.0f;
      double gmarg = 0.0;
      if constexpr (GAP) {
        // rounding margin of this node: 4 E_j, E_j <= 32 eps S_j, S_j = sum of |terms| of any H^a_j:
        // ga.gmargin covers the U terms (2 wsum + |c|) max|U|, the f terms are bounded per node
        double fs = ga.fcmax;
#pragma unroll
        for (int q = 0; q < Q; ++q) fs = fma(ga.fbmax[q], fabs(feat[q]), fs);
        gmarg = ga.gmargin + 128.0 * 2.220446049250313e-16 * fs;
        gj = valid ? ga.gap[nd.loc] : 0.0f;
        const bool ok = ga.bskip >= 0.0 && (double)gj > 2.0 * ga.bskip + gmarg;
        skip = __syncthreads_and(ok || !valid) != 0;
        if (skip) {
          a_lo = pol[nd.loc];
          a_hi = a_lo + 1;
          if (threadIdx.x == 0 && threadIdx.y == 0) atomicAdd(ga.nskip, 1);
        }
      }
#pragma unroll(KU > 0 ? KU : kS2Unroll)
      for (int a = a_lo; a < a_hi; ++a) {
#if HJB_SEARCH2_SYNC
        if (!GAP || !skip) {
          __syncwarp();
          if ((a & (HJB_SEARCH2_SYNC - 1)) == 0) __syncthreads();  // keep the CTA's 4 lines in lockstep
        }
#endif
        const double* t = tab.v + a * T::S;
        if (STRIP) {
          bool inside = true;
#pragma unroll
          for (int p = 0; p < P; ++p)
            inside &= fabs(ksc[p] * t[T::SD + 2 * p]) < nd.dist[0] && fabs(ksc[p] * t[T::SD + 2 * p + 1]) < nd.dist[1];
          inside &= fabs(kbs * t[T::BD]) < nd.dist[0] && fabs(kbs * t[T::BD + 1]) < nd.dist[1];
          if (!__all_sync(__activemask(), inside)) {
            Tap<2> taps[2 * P + 1];
            const double wsum = row_geometry<2, P>(L, t + T::SD, t + T::BD, nd, taps);
            double acc = 0.0;
#pragma unroll
            for (int e = 0; e < 2 * P + 1; ++e) acc = fma(taps[e].w, tap_value_u<2>(L, C, U, taps[e]), acc);
            double f = t[T::FC];
#pragma unroll
            for (int q = 0; q < Q; ++q) f = fma(t[T::FB + q], feat[q], f);
            const double H = (acc - wsum * Uj) + (nd.cn + t[T::C]) * Uj + f;
            if (H < best) {
              best = H;
              arg = a;
              fbest = f;
            }
            continue;
          }
        }
        double acc = 0.0;
        if constexpr (QUADS) {
#pragma unroll
          for (int p = 0; p < P; ++p) {
            int fl0, fl1;
            double s0, s1;
            split_floor(ksc[p] * t[T::SD + 2 * p], fl0, s0);
            split_floor(ksc[p] * t[T::SD + 2 * p + 1], fl1, s1);
            const int off = fl1 * n + fl0;
            const int offm = -off - n - 1;
            HJB_ASSERT(nd.loc + off >= 0 && nd.loc + off + n + 1 < L.local_elems);
            HJB_ASSERT(nd.loc + offm >= 0 && nd.loc + offm + n + 1 < L.local_elems);
            const double4 pq = ld_quad(quad_at(q4, off)), mq = ld_quad(quad_at(q4, offm));
            const double a00 = pq.x + mq.w, a10 = pq.y + mq.z, a01 = pq.z + mq.y, a11 = pq.w + mq.x;
            const double lo = fma(s0, a10 - a00, a00), hi = fma(s0, a11 - a01, a01);
            acc = fma(t[T::W + p], fma(s1, hi - lo, lo), acc);
          }
        } else if (HJB_S2_PAIRSUM && HJB_S2_EXP == 0 && HJB_SEARCH2_PAIRS == 0) {
          // f first, then the taps: H = (c_node + c_a - wsum_a) U_j + f + sum of taps (two fp64
          // operations for the diagonal part); each untruncated pair summed corner by corner before
          // one bilinear interpolation (the minus endpoint's cell mirrored through the node, fractions
          // 1 - s): 11 instead of 14 operations per pair
          double f = t[T::FC];
#pragma unroll
          for (int q = 0; q < Q; ++q) f = fma(t[T::FB + q], feat[q], f);
          acc = f;
#pragma unroll
          for (int p = 0; p < P; ++p) {
            int fl0, fl1;
            double s0, s1;
            split_floor(ksc[p] * t[T::SD + 2 * p], fl0, s0);
            split_floor(ksc[p] * t[T::SD + 2 * p + 1], fl1, s1);
            const int off = fl1 * n + fl0;
            const int offm = -off - n - 1;
            HJB_ASSERT(nd.loc + off >= 0 && nd.loc + off + n + 1 < L.local_elems);
            HJB_ASSERT(nd.loc + offm >= 0 && nd.loc + offm + n + 1 < L.local_elems);
            const double p00 = __ldg(u0 + off), p10 = __ldg(u0 + off + 1);
            const double p01 = __ldg(u1 + off), p11 = __ldg(u1 + off + 1);
            const double m00 = __ldg(u0 + offm), m10 = __ldg(u0 + offm + 1);
            const double m01 = __ldg(u1 + offm), m11 = __ldg(u1 + offm + 1);
            const double a00 = p00 + m11, a10 = p10 + m01, a01 = p01 + m10, a11 = p11 + m00;
            const double lo = fma(s0, a10 - a00, a00), hi = fma(s0, a11 - a01, a01);
            acc = fma(t[T::W + p], fma(s1, hi - lo, lo), acc);
          }
          {  // drift endpoint within one cell: its cell offset is a per-control fact (DQ)
            const double s0 = fma(kbs, t[T::BD], t[T::DQ]), s1 = fma(kbs, t[T::BD + 1], t[T::DQ + 1]);
            double dv;
            switch (quad.v[a]) {
              case 0: dv = interp_pairs(make_double2(nb[1][1], nb[1][2]), make_double2(nb[2][1], nb[2][2]), s0, s1); break;
              case 1: dv = interp_pairs(make_double2(nb[1][0], nb[1][1]), make_double2(nb[2][0], nb[2][1]), s0, s1); break;
              case 2: dv = interp_pairs(make_double2(nb[0][1], nb[0][2]), make_double2(nb[1][1], nb[1][2]), s0, s1); break;
              default: dv = interp_pairs(make_double2(nb[0][0], nb[0][1]), make_double2(nb[1][0], nb[1][1]), s0, s1); break;
            }
            acc = fma(t[T::WD], dv, acc);
          }
          const double H = fma(nd.cn + t[T::CMW], Uj, acc);
          if (H < best) {  // strict: lowest index wins exact ties (reading iv)
            best = H;
            arg = a;
            fbest = f;
          }
          continue;
        } else {
#pragma unroll
        for (int p = 0; p < P; ++p) {
          int fl0, fl1;
          double s0, s1;
          split_floor(ksc[p] * t[T::SD + 2 * p], fl0, s0);
          split_floor(ksc[p] * t[T::SD + 2 * p + 1], fl1, s1);
          const int off = fl1 * n + fl0;          // plus endpoint's cell corner, relative to the node
          const int offm = -off - n - 1;          // minus endpoint's cell corner (i - fl - 1)
          HJB_ASSERT(nd.loc + off >= 0 && nd.loc + off + n + 1 < L.local_elems);
          HJB_ASSERT(nd.loc + offm >= 0 && nd.loc + offm + n + 1 < L.local_elems);
          const double2 p0 = cell_row(up, u0, off), p1 = cell_row(upn, u1, off);
          const double2 m0 = cell_row(up, u0, offm), m1 = cell_row(upn, u1, offm);
          const double w = t[T::W + p];
#if HJB_S2_EXP == 2
          acc += ((p0.x + p1.y) + (m0.x + m1.y)) + ((p0.y + p1.x) + (m0.y + m1.x)) + w * (s0 + s1);
#else
          acc = fma(w, interp_pairs(p0, p1, s0, s1), acc);
          acc = fma(w, interp_pairs_mirror(m0, m1, s0, s1), acc);
#endif
        }
        }
        {  // drift endpoint: within one cell of the node, its quadrant is a per-control fact; the
           // bilinear value measured from the node, I = U_j + |o0| Dx + |o1| (Dy + |o0| Dxy), with the
           // quadrant's one-sided differences formed once per node (7 instead of 13 fp64 operations)
          const double o0 = kbs * t[T::ABD], o1 = kbs * t[T::ABD + 1];
          double dx, dy, dxy;
          switch (quad.v[a]) {
            case 0: dx = ddx[1]; dy = ddy[1]; dxy = ddxy[1][1]; break;
            case 1: dx = ddx[0]; dy = ddy[1]; dxy = ddxy[1][0]; break;
            case 2: dx = ddx[1]; dy = ddy[0]; dxy = ddxy[0][1]; break;
            default: dx = ddx[0]; dy = ddy[0]; dxy = ddxy[0][0]; break;
          }
          const double dv = Uj + fma(o0, dx, o1 * fma(o0, dxy, dy));
          acc = fma(t[T::WD], dv, acc);
        }
        double f = t[T::FC];
#pragma unroll
        for (int q = 0; q < Q; ++q) f = fma(t[T::FB + q], feat[q], f);
        const double cc = nd.cn + t[T::C];
        const double H = (acc - t[T::WSUM] * Uj) + cc * Uj + f;
        if (H < best) {  // strict: lowest index wins exact ties (reading iv)
          if constexpr (GAP) best2 = best;
          best = H;
          arg = a;
          fbest = f;
        } else if constexpr (GAP) {
          best2 = fmin(best2, H);
        }
      }
      if constexpr (GAP) {
        if (valid) {
          // skipped: the bound carried forward; scanned: the fresh gap less the rounding margin
          const double gn = skip ? (double)gj - 2.0 * ga.bskip : (best2 - best) - gmarg;
          ga.gap[nd.loc] = __double2float_rd(fmax(gn, 0.0));
        }
      }
      if (valid) {
        const double Up = __ldg(Uprev + nd.loc);
        const double R = fabs(Uj - Up - dt * best);
        const int old = pol[nd.loc];
        pol[nd.loc] = (uint8_t)arg;
        F[nd.loc] = fma(dt, fbest, Up);
        red[0] = fmax(red[0], (R == R) ? R : INFINITY);  // NaN -> inf (reported NONFINITE)
        red[1] += (old != arg) ? 1.0 : 0.0;
      }
    }
  }
  block_reduce_store<2, kS2T>(red, partial, 0x1u);
}


// ------------------------------------------------------------------------------------------------
// k_search_deep2p: k_search_deep2 (8-byte taps, same arithmetic, bit-identical results) with the
// control loop software-pipelined: the geometry and the 16 tap loads of control a+1 are issued
// before control a is combined, so each warp keeps two controls' gathers in flight.  What bounds
// k_search_deep2 is latency (70 of its 107 ms at cfg4 remain with the gathers
// removed; 16 warps per SM at 128 registers): one control's loads (~16, some of them L2 misses) are
// waited on before its arithmetic, which no other warp fully covers.  Here the loads of the next
// control overlap the arithmetic of the current one, at the cost of more registers (3 CTAs per SM).
// Measured at cfg4 (opt-in HJB_SEARCH2P=1): 148 ms against 115 ms for k_search_deep2 on the same box
// (168 registers, 12 warps per SM); capped at 128 registers it spills (200 ms).
#ifndef HJB_SEARCH2P_MINB
#define HJB_SEARCH2P_MINB 3
#endif
template <int P>
struct S2Geom {
  int off[P];
  double s0[P], s1[P];
};
template <int P, int Q>
__global__ void __launch_bounds__(kS2T, HJB_SEARCH2P_MINB) k_search_deep2p(LevelDev L, CoefDev C, double dt,
                                                                          const double* __restrict__ U,
                                                                          const double* __restrict__ Uprev,
                                                                          uint8_t* __restrict__ pol,
                                                                          double* __restrict__ F, double* partial,
                                                                          SkipRect it, const __grid_constant__ STab tab,
                                                                          const __grid_constant__ STabQuad quad) {
  using T = STabLayout<P, Q>;
  double red[2] = {0.0, 0.0};
  const int nk = box_lines(it);
  const int n = L.n;
  const int K = C.K;
  const int tx = (it.c1 - it.c0 + kSBX - 1) / kSBX, ty = (nk + kS2Y - 1) / kS2Y;
  const int ntiles = tx * ty;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int sc = t / (kSuperCols * ty);
    const int scw = min(kSuperCols, tx - sc * kSuperCols);
    const int tl = t - sc * kSuperCols * ty;
    const int trow = tl / scw, tcol = sc * kSuperCols + (tl - trow * scw);
    const int k0 = trow * kS2Y + threadIdx.y;
    const int col0 = it.c0 + tcol * kSBX + threadIdx.x;
    const bool valid = k0 < nk && col0 < it.c1;
    const int k = valid ? k0 : trow * kS2Y, col = valid ? col0 : it.c0 + tcol * kSBX;
    const int row = box_row<2>(L, it, k);
    Node<2> nd;
    node_at<2>(L, col, row, nd);
    load_fields<2>(C, nd);
    prefetch_ahead(L, U, nd.loc, col);
    double feat[Q > 0 ? Q : 1];
#pragma unroll
    for (int q = 0; q < Q; ++q) feat[q] = __ldg(C.f_feat + q * C.ld + nd.loc);
    const double Uj = __ldg(U + nd.loc);
    double nb[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) nb[r][c] = (r == 1 && c == 1) ? Uj : __ldg(U + nd.loc + (r - 1) * n + (c - 1));
    double ksc[P];
#pragma unroll
    for (int p = 0; p < P; ++p) ksc[p] = L.kh * nd.sc[p];
    const double kbs = L.k2h * nd.bs;
    const double* u0 = U + nd.loc;
    const double* u1 = u0 + n;
    double best = INFINITY, fbest = 0.0;
    int arg = 0;
    auto geom = [&](int a, S2Geom<P>& g) {
      const double* tb = tab.v + a * T::S;
#pragma unroll
      for (int p = 0; p < P; ++p) {
        int fl0, fl1;
        split_floor(ksc[p] * tb[T::SD + 2 * p], fl0, g.s0[p]);
        split_floor(ksc[p] * tb[T::SD + 2 * p + 1], fl1, g.s1[p]);
        g.off[p] = fl1 * n + fl0;
      }
    };
    auto gather = [&](const S2Geom<P>& g, double (&v)[P][8]) {
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const int off = g.off[p], offm = -off - n - 1;
        HJB_ASSERT(nd.loc + off >= 0 && nd.loc + off + n + 1 < L.local_elems);
        HJB_ASSERT(nd.loc + offm >= 0 && nd.loc + offm + n + 1 < L.local_elems);
        v[p][0] = __ldg(u0 + off);
        v[p][1] = __ldg(u0 + off + 1);
        v[p][2] = __ldg(u1 + off);
        v[p][3] = __ldg(u1 + off + 1);
        v[p][4] = __ldg(u0 + offm);
        v[p][5] = __ldg(u0 + offm + 1);
        v[p][6] = __ldg(u1 + offm);
        v[p][7] = __ldg(u1 + offm + 1);
      }
    };
    auto combine = [&](int a, const S2Geom<P>& g, const double (&v)[P][8]) {
      const double* tb = tab.v + a * T::S;
      double acc = 0.0;
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const double w = tb[T::W + p];
        acc = fma(w, interp_pairs(make_double2(v[p][0], v[p][1]), make_double2(v[p][2], v[p][3]), g.s0[p], g.s1[p]), acc);
        acc = fma(w, interp_pairs_mirror(make_double2(v[p][4], v[p][5]), make_double2(v[p][6], v[p][7]), g.s0[p], g.s1[p]),
                  acc);
      }
      {
        const double o0 = kbs * tb[T::BD], o1 = kbs * tb[T::BD + 1];
        const double s0 = o0 - floor(o0), s1 = o1 - floor(o1);
        double dv;
        switch (quad.v[a]) {
          case 0: dv = interp_pairs(make_double2(nb[1][1], nb[1][2]), make_double2(nb[2][1], nb[2][2]), s0, s1); break;
          case 1: dv = interp_pairs(make_double2(nb[1][0], nb[1][1]), make_double2(nb[2][0], nb[2][1]), s0, s1); break;
          case 2: dv = interp_pairs(make_double2(nb[0][1], nb[0][2]), make_double2(nb[1][1], nb[1][2]), s0, s1); break;
          default: dv = interp_pairs(make_double2(nb[0][0], nb[0][1]), make_double2(nb[1][0], nb[1][1]), s0, s1); break;
        }
        acc = fma(tb[T::WD], dv, acc);
      }
      double f = tb[T::FC];
#pragma unroll
      for (int q = 0; q < Q; ++q) f = fma(tb[T::FB + q], feat[q], f);
      const double cc = nd.cn + tb[T::C];
      const double H = (acc - tb[T::WSUM] * Uj) + cc * Uj + f;
      if (H < best) {  // strict: lowest index wins exact ties (reading iv)
        best = H;
        arg = a;
        fbest = f;
      }
    };
    S2Geom<P> g0, g1;
    double v0[P][8], v1[P][8];
    geom(0, g0);
    gather(g0, v0);
    for (int a = 0; a < K; a += 2) {
#if HJB_SEARCH2_SYNC
      if ((a & (HJB_SEARCH2_SYNC - 1)) == 0) __syncthreads();  // the CTA's 4 lines in lockstep
#endif
      const bool two = a + 1 < K;
      if (two) {
        geom(a + 1, g1);
        gather(g1, v1);
      }
      combine(a, g0, v0);
      if (two) {
        if (a + 2 < K) {
          geom(a + 2, g0);
          gather(g0, v0);
        }
        combine(a + 1, g1, v1);
      }
    }
    if (valid) {
      const double Up = __ldg(Uprev + nd.loc);
      const double R = fabs(Uj - Up - dt * best);
      const int old = pol[nd.loc];
      pol[nd.loc] = (uint8_t)arg;
      F[nd.loc] = fma(dt, fbest, Up);
      red[0] = fmax(red[0], (R == R) ? R : INFINITY);  // NaN -> inf (reported NONFINITE)
      red[1] += (old != arg) ? 1.0 : 0.0;
    }
  }
  block_reduce_store<2, kS2T>(red, partial, 0x1u);
}

// ------------------------------------------------------------------------------------------------
// k_search_deep3: k_search_deep2 with the node-local part of every H^a hoisted out of the gather loop.
// What bounds k_search_deep2 at cfg4 is latency (ncu r02_o: 16 resident warps per SM at 128
// registers, issue 41 % active; each warp's control iteration waits ~1800 cycles on its dependent
// gathers).  Per (node, control) H^a_j splits into
//   H^a_j = sum_p w_p [I U(x + o_p) + I U(x - o_p)]                 (the gathers: two pairs)
//         + [ f^a_j + w_d I U(x + o_d) + (c^a_j - wsum^a) U_j ]      (node-local: no gathers)
// The bracket needs the node's features and its 3x3 neighbourhood (drift endpoint within one cell)
// but no memory traffic: a prologue evaluates it for all K controls into shared memory (one slot per
// thread and control), so the gather loop holds neither the features nor the neighbourhood in
// registers (fewer registers -> more resident warps to hide the gather latency) and issues only the
// pair taps (256-bit corner loads) plus one shared-memory read per control.  f at the argmin (for
// F) is re-evaluated once per node after the loop.  Same formulas, different summation order:
// identical policies except at near-ties (test_deep_kernels_match_general).
#ifndef HJB_SEARCH3_MINB
#define HJB_SEARCH3_MINB 6
#endif
template <int P, int Q>
__global__ void __launch_bounds__(kS2T, HJB_SEARCH3_MINB) k_search_deep3(LevelDev L, CoefDev C, double dt,
                                                                        const double* __restrict__ U,
                                                                        const double4* __restrict__ Q4,
                                                                        const double* __restrict__ Uprev,
                                                                        uint8_t* __restrict__ pol,
                                                                        double* __restrict__ F, double* partial,
                                                                        SkipRect it, const __grid_constant__ STab tab,
                                                                        const __grid_constant__ STabQuad quad) {
  using T = STabLayout<P, Q>;
  extern __shared__ double sbase[];  // [K][kS2T]: the node-local bracket of H^a
  const int tid = threadIdx.y * kSBX + threadIdx.x;
  double red[2] = {0.0, 0.0};
  const int nk = box_lines(it);
  const int n = L.n;
  const int K = C.K;
  const int tx = (it.c1 - it.c0 + kSBX - 1) / kSBX, ty = (nk + kS2Y - 1) / kS2Y;
  const int ntiles = tx * ty;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int sc = t / (kSuperCols * ty);
    const int scw = min(kSuperCols, tx - sc * kSuperCols);
    const int tl = t - sc * kSuperCols * ty;
    const int trow = tl / scw, tcol = sc * kSuperCols + (tl - trow * scw);
    const int k0 = trow * kS2Y + threadIdx.y;
    const int col0 = it.c0 + tcol * kSBX + threadIdx.x;
    const bool valid = k0 < nk && col0 < it.c1;
    const int k = valid ? k0 : trow * kS2Y, col = valid ? col0 : it.c0 + tcol * kSBX;
    const int row = box_row<2>(L, it, k);
    Node<2> nd;
    node_at<2>(L, col, row, nd);
    load_fields<2>(C, nd);
    prefetch_ahead(L, U, nd.loc, col);
    const double Uj = __ldg(U + nd.loc);
    const double kbs = L.k2h * nd.bs;
    {  // prologue: the node-local bracket for every control
      double feat[Q > 0 ? Q : 1];
#pragma unroll
      for (int q = 0; q < Q; ++q) feat[q] = __ldg(C.f_feat + q * C.ld + nd.loc);
      double nb[3][3];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) nb[r][c] = (r == 1 && c == 1) ? Uj : __ldg(U + nd.loc + (r - 1) * n + (c - 1));
      for (int a = 0; a < K; ++a) {
        const double* tb = tab.v + a * T::S;
        const double o0 = kbs * tb[T::BD], o1 = kbs * tb[T::BD + 1];
        const double s0 = o0 - floor(o0), s1 = o1 - floor(o1);
        double dv;
        switch (quad.v[a]) {
          case 0: dv = interp_pairs(make_double2(nb[1][1], nb[1][2]), make_double2(nb[2][1], nb[2][2]), s0, s1); break;
          case 1: dv = interp_pairs(make_double2(nb[1][0], nb[1][1]), make_double2(nb[2][0], nb[2][1]), s0, s1); break;
          case 2: dv = interp_pairs(make_double2(nb[0][1], nb[0][2]), make_double2(nb[1][1], nb[1][2]), s0, s1); break;
          default: dv = interp_pairs(make_double2(nb[0][0], nb[0][1]), make_double2(nb[1][0], nb[1][1]), s0, s1); break;
        }
        double f = tb[T::FC];
#pragma unroll
        for (int q = 0; q < Q; ++q) f = fma(tb[T::FB + q], feat[q], f);
        const double cw = (nd.cn + tb[T::C]) - tb[T::WSUM];
        sbase[a * kS2T + tid] = fma(cw, Uj, fma(tb[T::WD], dv, f));
      }
    }
    double ksc[P];
#pragma unroll
    for (int p = 0; p < P; ++p) ksc[p] = L.kh * nd.sc[p];
    const double4* q4 = Q4 + nd.loc;
    double best = INFINITY;
    int arg = 0;
    for (int a = 0; a < K; ++a) {
#if HJB_SEARCH2_SYNC
      if ((a & (HJB_SEARCH2_SYNC - 1)) == 0) __syncthreads();  // the CTA's 4 lines in lockstep
#endif
      const double* tb = tab.v + a * T::S;
      double acc = sbase[a * kS2T + tid];
#pragma unroll
      for (int p = 0; p < P; ++p) {
        int fl0, fl1;
        double s0, s1;
        split_floor(ksc[p] * tb[T::SD + 2 * p], fl0, s0);
        split_floor(ksc[p] * tb[T::SD + 2 * p + 1], fl1, s1);
        const int off = fl1 * n + fl0;
        const int offm = -off - n - 1;
        HJB_ASSERT(nd.loc + off >= 0 && nd.loc + off + n + 1 < L.local_elems);
        HJB_ASSERT(nd.loc + offm >= 0 && nd.loc + offm + n + 1 < L.local_elems);
        const double4 pq = ld_quad(quad_at(q4, off)), mq = ld_quad(quad_at(q4, offm));
        const double a00 = pq.x + mq.w, a10 = pq.y + mq.z, a01 = pq.z + mq.y, a11 = pq.w + mq.x;
        const double lo = fma(s0, a10 - a00, a00), hi = fma(s0, a11 - a01, a01);
        acc = fma(tb[T::W + p], fma(s1, hi - lo, lo), acc);
      }
      if (acc < best) {  // strict: lowest index wins exact ties (reading iv)
        best = acc;
        arg = a;
      }
    }
    if (valid) {
      const double* tb = tab.v + arg * T::S;
      double fbest = tb[T::FC];
#pragma unroll
      for (int q = 0; q < Q; ++q) fbest = fma(tb[T::FB + q], __ldg(C.f_feat + q * C.ld + nd.loc), fbest);
      const double Up = __ldg(Uprev + nd.loc);
      const double R = fabs(Uj - Up - dt * best);
      const int old = pol[nd.loc];
      pol[nd.loc] = (uint8_t)arg;
      F[nd.loc] = fma(dt, fbest, Up);
      red[0] = fmax(red[0], (R == R) ? R : INFINITY);  // NaN -> inf (reported NONFINITE)
      red[1] += (old != arg) ? 1.0 : 0.0;
    }
  }
  block_reduce_store<2, kS2T>(red, partial, 0x1u);
}

}  // namespace hjb
