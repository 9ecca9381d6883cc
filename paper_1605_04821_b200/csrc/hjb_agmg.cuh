// hjb_agmg.cuh -- aggregation-based algebraic multigrid (PAPER.md:171-176,
// 1162-1164): the fine policy operator assembled on the interior unknowns (compact numbering), double
// pairwise aggregation on the symmetric part's strongest negative couplings (parallel proposal
// matching), 0/1 aggregate transfers, coarse operators P^T A P, and the kernels of the K-cycle.
//
// Matching (per pass): node i's candidate is the unaggregated j maximising s_ij = -(a_ij + a_ji)/2
// with s_ij >= beta * max_k s_ik (beta = 0.25) and s_ij > 0 (lowest index on ties); i proposes to
// j, j keeps its strongest proposer; proposers and acceptors are the two colours of a hash bit,
// alternating per round, so every accepted proposal is a pair; six rounds, then the rest stay
// single (measured on cfg2 129^2: 89 % of the nodes paired).  (The oracle,
// oracle/agmg.py, matches greedily in index order: the aggregates differ, the solve does not.)
// Storage: ELL, column-major ([slot][row]), compact interior indices, -1 = empty.
#pragma once
#include "hjb_device.cuh"
#include "hjb_galerkin.cuh"

namespace hjb {

constexpr int kAgW = 96;  // ELL width of every AGMG level (fine: <= 1 + 4 (2P+1) entries per row)

template <int D>
__device__ __forceinline__ int compact_of(const LevelDev& L, const int* i) {
  return D == 2 ? (i[1] - 1) * L.nI + (i[0] - 1) : ((i[2] - 1) * L.nI + (i[1] - 1)) * L.nI + (i[0] - 1);
}

// fine operator A = I - dt (L_hat^pi + c^pi) on the interior unknowns (boundary couplings are data);
// row t = compact index of the node
template <int D, int P>
__global__ void __launch_bounds__(128) k_ag_fine(LevelDev L, CoefDev C, double dt, const uint8_t* __restrict__ pol,
                                                int* __restrict__ col, double* __restrict__ val,
                                                double* __restrict__ diag, int* __restrict__ overflow) {
  constexpr int E = 2 * P + 1;
  const int64_t N = (int64_t)L.nI * L.nrows;
  RowAcc A;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < N; q += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(q / L.nI), c0 = (int)(q - (int64_t)row * L.nI);
    Node<D> nd;
    node_at<D>(L, c0, row, nd);
    load_fields<D>(C, nd);
    const int a = pol[nd.loc];
    Tap<D> taps[E];
    const double wsum = row_geometry<D, P>(L, C.sigma_dir + a * P * D, C.b_dir + a * D, nd, taps);
    const double cc = nd.cn + C.c_ctrl[a];
    acc_init(A);
    bool ok = acc_add(A, (int)q, 1.0 + dt * (wsum - cc));
    for (int e = 0; e < E; ++e) {
      if (taps[e].w == 0.0) continue;
      for (int m = 0; m < (1 << D); ++m) {
        int j[3];
        double wc = 1.0;
        bool interior = true;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const int h = (m >> d) & 1;
          j[d] = taps[e].c[d] + h;
          wc *= h ? taps[e].s[d] : 1.0 - taps[e].s[d];
          interior &= (j[d] >= 1 && j[d] <= L.n - 2);
        }
        if (!interior || wc == 0.0) continue;
        ok &= acc_add(A, compact_of<D>(L, j), -dt * taps[e].w * wc);
      }
    }
    double dg = 0.0;
    for (int k = 0; k < A.cnt; ++k)
      if (A.key[A.order[k]] == (int)q) dg = A.val[A.order[k]];
    diag[q] = dg;
    if (!ok || !acc_store(A, kAgW, N, q, col, val)) atomicExch(overflow, 1);
  }
}

// a_ji by scanning row j
__device__ __forceinline__ double ell_entry(const int* __restrict__ col, const double* __restrict__ val, int64_t N,
                                            int j, int i) {
  for (int k = 0; k < kAgW; ++k) {
    const int c = col[k * N + j];
    if (c < 0) break;
    if (c == i) return val[k * N + j];
  }
  return 0.0;
}

// the proposer colour of a node: a hash bit (about half of any neighbourhood has the other colour)
__device__ __forceinline__ int ag_color(int64_t i) { return (int)((((uint64_t)i * 2654435761ull) >> 7) & 1ull); }

// one matching round: cand[i] for every unaggregated proposer i (colour == round parity), among the
// unaggregated neighbours of the other colour
__global__ void __launch_bounds__(128) k_ag_candidates(int64_t N, const int* __restrict__ col,
                                                      const double* __restrict__ val, const int* __restrict__ state,
                                                      int* __restrict__ cand, double beta, int round) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    if (state[i] >= 0 || ag_color(i) != (round & 1)) { cand[i] = -1; continue; }
    double strongest = 0.0, best = 0.0;
    int bj = -1;
    for (int k = 0; k < kAgW; ++k) {
      const int j = col[k * N + i];
      if (j < 0) break;
      if (j == (int)i) continue;
      const double s = -0.5 * (val[k * N + i] + ell_entry(col, val, N, j, (int)i));
      strongest = fmax(strongest, s);
      if (state[j] < 0 && ag_color(j) != (round & 1) && (s > best || (s == best && s > 0.0 && j < bj))) {
        best = s;
        bj = j;
      }
    }
    cand[i] = (bj >= 0 && best > 0.0 && best >= beta * strongest) ? bj : -1;
  }
}

// proposal round: every unaggregated i with a candidate j proposes to j; j keeps the strongest
// proposer (ties: lowest index) -- a 64-bit atomicMax on (strength as float bits, ~i)
__global__ void __launch_bounds__(128) k_ag_propose(int64_t N, const int* __restrict__ col, const double* __restrict__ val,
                                                   const int* __restrict__ state, const int* __restrict__ cand,
                                                   unsigned long long* __restrict__ winner) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    if (state[i] >= 0) continue;
    const int j = cand[i];
    if (j < 0) continue;
    double aij = 0.0;
    for (int k = 0; k < kAgW; ++k) {
      const int c = col[k * N + i];
      if (c < 0) break;
      if (c == j) aij = val[k * N + i];
    }
    const float s = (float)(-0.5 * (aij + ell_entry(col, val, N, j, (int)i)));
    const unsigned long long key = ((unsigned long long)__float_as_uint(fmaxf(s, 0.0f)) << 32) |
                                   (unsigned long long)(0xFFFFFFFFu - (unsigned)i);
    atomicMax(winner + j, key);
  }
}

// accept: every acceptor j (the other colour) pairs with its strongest proposer i; a proposer
// proposed once, so no node joins two pairs; leader = min(i, j)
__global__ void __launch_bounds__(128) k_ag_accept(int64_t N, const unsigned long long* __restrict__ winner,
                                                  int* __restrict__ state) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
    if (winner[j] == 0ull || state[j] >= 0) continue;
    const int i = (int)(0xFFFFFFFFu - (unsigned)(winner[j] & 0xFFFFFFFFull));
    const int lead = min(i, (int)j);
    state[i] = lead;
    state[j] = lead;
  }
}

// nodes left alone after the last round (an accepted acceptor is set by its proposer)
__global__ void __launch_bounds__(128) k_ag_singles(int64_t N, int* __restrict__ state) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    if (state[i] < 0) state[i] = (int)i;
}

__global__ void __launch_bounds__(256) k_ag_leader_flags(int64_t N, const int* __restrict__ state, int* __restrict__ flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = (state[i] == (int)i) ? 1 : 0;
}

// agg[i] = id of i's leader (ids = exclusive scan of the leader flags); members of each aggregate
__global__ void __launch_bounds__(256) k_ag_number(int64_t N, const int* __restrict__ state, const int* __restrict__ id,
                                                  int* __restrict__ agg, int* __restrict__ mem, int64_t Nc) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const int a = id[state[i]];
    agg[i] = a;
    mem[(state[i] == (int)i ? 0 : 1) * Nc + a] = (int)i;
  }
}

// compose two passes: agg = agg2[agg1], members (<= 4) of the final aggregates
__global__ void __launch_bounds__(256) k_ag_compose(int64_t N, const int* __restrict__ agg1, const int* __restrict__ agg2,
                                                   int* __restrict__ agg, int64_t N1, const int* __restrict__ mem1,
                                                   const int* __restrict__ mem2, int64_t Nc, int* __restrict__ mem) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    agg[i] = agg2[agg1[i]];
  for (int64_t I = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; I < Nc; I += (int64_t)gridDim.x * blockDim.x) {
    int k = 0;
    for (int a = 0; a < 2; ++a) {
      const int m = mem2[a * Nc + I];
      if (m < 0) continue;
      for (int b = 0; b < 2; ++b) {
        const int f = mem1[b * N1 + m];
        if (f >= 0) mem[(k++) * Nc + I] = f;
      }
    }
  }
}

// coarse row I = sum over the members i of row i with columns mapped through agg (P^T A P)
__global__ void __launch_bounds__(128) k_ag_coarse(int64_t Nf, const int* __restrict__ fcol, const double* __restrict__ fval,
                                                  const int* __restrict__ agg, int64_t Nc, const int* __restrict__ mem,
                                                  int nmem, int* __restrict__ ccol, double* __restrict__ cval,
                                                  double* __restrict__ cdiag, int* __restrict__ overflow) {
  RowAcc A;
  for (int64_t I = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; I < Nc; I += (int64_t)gridDim.x * blockDim.x) {
    acc_init(A);
    bool ok = true;
    for (int mm = 0; mm < nmem; ++mm) {
      const int i = mem[mm * Nc + I];
      if (i < 0) continue;
      for (int k = 0; k < kAgW; ++k) {
        const int j = fcol[k * Nf + i];
        if (j < 0) break;
        ok &= acc_add(A, agg[j], fval[k * Nf + i]);
      }
    }
    double dg = 0.0;
    for (int k = 0; k < A.cnt; ++k)
      if (A.key[A.order[k]] == (int)I) dg = A.val[A.order[k]];
    cdiag[I] = dg;
    if (!ok || !acc_store(A, kAgW, Nc, I, ccol, cval)) atomicExch(overflow, 1);
  }
}

// y = b - A x (JAC = false) or y = x + omega (b - A x) / D
template <bool JAC>
__global__ void __launch_bounds__(256) k_ag_sweep(int64_t N, const int* __restrict__ col, const double* __restrict__ val,
                                                 const double* __restrict__ dg, const double* __restrict__ x,
                                                 const double* __restrict__ b, double omega, double* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    double ax = 0.0;
    for (int k = 0; k < kAgW; ++k) {
      const int j = __ldg(col + k * N + i);
      if (j < 0) break;
      ax = fma(__ldg(val + k * N + i), __ldg(x + j), ax);
    }
    const double r = __ldg(b + i) - ax;
    y[i] = JAC ? fma(omega, r / __ldg(dg + i), __ldg(x + i)) : r;
  }
}

// y = A x
__global__ void __launch_bounds__(256) k_ag_spmv(int64_t N, const int* __restrict__ col, const double* __restrict__ val,
                                                const double* __restrict__ x, double* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    double ax = 0.0;
    for (int k = 0; k < kAgW; ++k) {
      const int j = __ldg(col + k * N + i);
      if (j < 0) break;
      ax = fma(__ldg(val + k * N + i), __ldg(x + j), ax);
    }
    y[i] = ax;
  }
}

// rc[I] = sum of r over the members of aggregate I (P^T r)
__global__ void __launch_bounds__(256) k_ag_restrict(int64_t Nc, const int* __restrict__ mem, int nmem,
                                                    const double* __restrict__ r, double* __restrict__ rc) {
  for (int64_t I = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; I < Nc; I += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int m = 0; m < nmem; ++m) {
      const int i = mem[m * Nc + I];
      if (i >= 0) s += r[i];
    }
    rc[I] = s;
  }
}

// x += P e (x_i += e_{agg(i)})
__global__ void __launch_bounds__(256) k_ag_prolong(int64_t N, const int* __restrict__ agg, const double* __restrict__ e,
                                                   double* __restrict__ x) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    x[i] += e[agg[i]];
}

// y = a x + b y ; partial sums of (y, z) if z
__global__ void __launch_bounds__(256) k_ag_axpby(int64_t N, double a, const double* __restrict__ x, double b,
                                                 double* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = fma(a, x[i], b * y[i]);
}

// block partials [sum x.y, sum y.y] of compact vectors (256 threads)
__global__ void __launch_bounds__(256) k_ag_dot2(int64_t N, const double* __restrict__ x, const double* __restrict__ y,
                                                double* partial) {
  double red[2] = {0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    red[0] = fma(x[i], y[i], red[0]);
    red[1] = fma(y[i], y[i], red[1]);
  }
  block_reduce_store<2, 256>(red, partial);
}

// K-cycle inner GCR scalars on the device (no host round trip inside the cycle): one block reduces
// the nb block partials of k_ag_dot2 in a fixed order and stores
//   op 0: s[slot] = -x.y            (minus the projection coefficient h)
//   op 1: s[slot] = 1 / sqrt(y.y)   (0 for a zero vector: the direction then adds nothing)
//   op 2: s[slot] = x.y, s[slot+1] = -x.y, s[slot+2] = y.y   (gamma, -gamma, r.r)
__global__ void __launch_bounds__(256) k_ag_scal(const double* __restrict__ partial, int nb, double* s, int slot,
                                                int op) {
  __shared__ double sm[2][256];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < nb; i += 256) {
    a += partial[2 * i];
    b += partial[2 * i + 1];
  }
  sm[0][threadIdx.x] = a;
  sm[1][threadIdx.x] = b;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      sm[0][threadIdx.x] += sm[0][threadIdx.x + w];
      sm[1][threadIdx.x] += sm[1][threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double xy = sm[0][0], yy = sm[1][0];
    if (op == 0) {
      s[slot] = -xy;
    } else if (op == 1) {
      s[slot] = yy > 0.0 ? 1.0 / sqrt(yy) : 0.0;
    } else {
      s[slot] = xy;
      s[slot + 1] = -xy;
      s[slot + 2] = yy;
    }
  }
}

// y += s[slot] x  /  y *= s[slot]  (coefficients from k_ag_scal)
__global__ void __launch_bounds__(256) k_ag_axpy_dev(int64_t N, const double* __restrict__ s, int slot,
                                                    const double* __restrict__ x, double* __restrict__ y) {
  const double a = s[slot];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = fma(a, x[i], y[i]);
}
__global__ void __launch_bounds__(256) k_ag_scale_dev(int64_t N, const double* __restrict__ s, int slot,
                                                     double* __restrict__ y) {
  const double a = s[slot];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    y[i] *= a;
}

// coarsest level: dense matrix from ELL (compact rows), then x = Ainv b
__global__ void k_ag_dense(int64_t N, const int* __restrict__ col, const double* __restrict__ val, double* __restrict__ Ad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    for (int k = 0; k < kAgW; ++k) {
      const int j = col[k * N + i];
      if (j < 0) break;
      Ad[i * N + j] += val[k * N + i];
    }
}
// in-place Gauss-Jordan inverse in global memory (one block; no pivoting: the coarse matrices are
// M-matrices with non-negative row sums and positive diagonals), N <= kAgDenseMax
constexpr int kAgDenseMax = 1024;
constexpr int kAgCoarseSweeps = 24;  // coarsest level without a dense inverse (stalled aggregation)
__global__ void __launch_bounds__(1024) k_ag_invert(double* __restrict__ M, int N) {
  __shared__ double colk[kAgDenseMax];
  for (int k = 0; k < N; ++k) {
    const double piv = M[(int64_t)k * N + k];
    __syncthreads();
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
      const double v = (j == k) ? 1.0 : M[(int64_t)k * N + j];
      M[(int64_t)k * N + j] = v / piv;
    }
    for (int i = threadIdx.x; i < N; i += blockDim.x) colk[i] = (i == k) ? 0.0 : M[(int64_t)i * N + k];
    __syncthreads();
    for (int64_t e = threadIdx.x; e < (int64_t)N * N; e += blockDim.x) {
      const int i = (int)(e / N), j = (int)(e - (int64_t)i * N);
      if (i == k) continue;
      const double base = (j == k) ? 0.0 : M[e];
      M[e] = fma(-colk[i], M[(int64_t)k * N + j], base);
    }
    __syncthreads();
  }
}

__global__ void k_ag_dense_solve(int N, const double* __restrict__ Ainv, const double* __restrict__ b, double* __restrict__ x) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < N; ++j) s = fma(Ainv[(int64_t)i * N + j], b[j], s);
    x[i] = s;
  }
}

// grid array (interior) <-> compact vector
template <int D>
__global__ void __launch_bounds__(kTX) k_ag_gather(LevelDev L, const double* __restrict__ g, double* __restrict__ c) {
  FOR_INTERIOR(L) { c[(int64_t)row * L.nI + col] = g[interior_offset<D>(L, col, row)]; }
}
template <int D>
__global__ void __launch_bounds__(kTX) k_ag_scatter_add(LevelDev L, const double* __restrict__ c, double* __restrict__ g) {
  FOR_INTERIOR(L) { g[interior_offset<D>(L, col, row)] += c[(int64_t)row * L.nI + col]; }
}

}  // namespace hjb
