/* certify.c -- ORACLE (test infrastructure, NOT product code): the nonlinear-residual certificate
 * of one implicit step, in plain C so it covers every row of the BASELINE grids.
 *
 * Only tests/ (via oracle/certify.py) may load this.  It shares no code with the CUDA path
 * (paper_1605_04821_b200/); it restates, row by row, the numpy oracle of oracle/scheme.py and
 * oracle/howard.py, which follow the paper:
 *
 *   steps   y^{a,+-}_p = +- sqrt(dx) sigma^a_p(x_j), p <= P;  drift y_{P+1} = dx b^a(x_j)
 *   mu      = largest value in (0,1] keeping x_j + mu y in closed Omega
 *           (binding coordinates snapped onto the face, all clipped to [lo,hi]: DESIGN reading i, vi)
 *   weights A_p = 2/(mu+^2 + mu+ mu-), B_p = 2/(mu-^2 + mu- mu+); drift A = B = 1/mu
 *   interp  multilinear from the cell c = clip(floor((z-lo)/dx), 0, n-2), s = (z-lo)/dx - c
 *   L_hat^a[U](x_j) = sum_e A_e/(2dx) sum_i w_i(z_e) (U_i - U_j)                          (eq. Lhat)
 *   H^a_j(U) = L_hat^a[U](x_j) + c^a_j U_j + f^a_j
 *   R_j(U)   = | U_j - U^{n-1}_j - dt min_a H^a_j(U) |  = | max_a (A^a U - F^a)_j |        (D1)
 * and by D6 ||U - U*||_inf <= max_j R_j / (1 - dt max c) for the exact solution U*
 * of the step, whatever U is.  The coefficient model is the affine-separable one of include/hjb.h
 * and synth/problems.py (problem data, not method):
 *   sigma^a_p = sigma_scale_p sigma_dir[a][p] + sigma_node_p,  b^a = b_scale b_dir[a] + b_node,
 *   c^a = c_ctrl[a] + c_node,  f^a = f_ctrl[a] + sum_q f_basis[a][q] f_feat_q.
 *
 * The one shortcut against the numpy text: an endpoint x + y that already lies in the closed box
 * has mu = 1 (no face parameter below 1), so its face parameters are not formed -- the same value.
 *
 * Build: gcc -O3 -fopenmp -ffp-contract=off -shared -fPIC (oracle/certify.py does it).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

typedef struct {
  int32_t d, P, K, Q;
  int64_t n;
  double lo, hi, dt;
  const double* sigma_dir; /* [K][P][d] */
  const double* b_dir;     /* [K][d]    */
  const double* c_ctrl;    /* [K]       */
  const double* f_basis;   /* [K][Q]    */
  const double* f_ctrl;    /* [K] or NULL */
} orc_problem;

typedef struct {
  const double* U;      /* U[g - u_off] for global flat index g (must cover every endpoint cell) */
  int64_t u_off;
  const double* Uprev;  /* Uprev[g - f_off] on the certified rows                               */
  const double *sigma_scale, *sigma_node, *b_scale, *b_node, *c_node, *f_feat; /* planes, NULL = absent */
  int64_t f_off, f_ld;  /* field element of node g: plane[k * f_ld + g - f_off]                   */
} orc_arrays;

/* truncation of the ray x + [0,1] y: mu and the binding mask */
#define INL static inline __attribute__((always_inline))
INL double trunc_mu(const int d, const orc_problem* pb, const double* x, const double* y, int* bind) {
  int inside = 1;
  for (int i = 0; i < d; ++i) {
    const double z = x[i] + y[i];
    if (z < pb->lo || z > pb->hi) inside = 0;
    bind[i] = 0;
  }
  if (inside) return 1.0;
  double ft[3], mu = 1.0;
  for (int i = 0; i < d; ++i) {
    ft[i] = INFINITY;
    if (y[i] > 0) ft[i] = (pb->hi - x[i]) / y[i];
    else if (y[i] < 0) ft[i] = (pb->lo - x[i]) / y[i];
    if (ft[i] < mu) mu = ft[i];
  }
  for (int i = 0; i < d; ++i) bind[i] = (ft[i] <= mu) && (mu < 1.0);
  return mu;
}

/* x + mu y, binding coordinates on the face, clipped to [lo,hi] (oracle truncated_endpoint) */
INL void endpoint(const int d, const orc_problem* pb, const double* x, const double* y, double mu, const int* bind,
                     double* z) {
  for (int i = 0; i < d; ++i) {
    double v = x[i] + mu * y[i];
    if (bind[i]) v = (y[i] > 0) ? pb->hi : pb->lo;
    if (v < pb->lo) v = pb->lo;
    if (v > pb->hi) v = pb->hi;
    z[i] = v;
  }
}

/* sum_i w_i(z) (U_i - U_j) over the 2^d vertices of z's cell */
INL double interp_diff(const int d, const orc_problem* pb, const orc_arrays* ar, const double* z, double Uj,
                       double inv_dx) {
  const int64_t n = pb->n;
  int64_t c[3];
  double s[3];
  for (int i = 0; i < d; ++i) {
    const double t = (z[i] - pb->lo) * inv_dx;   /* (z - lo)/dx */
    double fl = floor(t);
    if (fl < 0) fl = 0;
    if (fl > (double)(n - 2)) fl = (double)(n - 2);
    c[i] = (int64_t)fl;
    s[i] = t - fl;
  }
  double acc = 0.0;
  for (int m = 0; m < (1 << d); ++m) {
    double w = 1.0;
    int64_t g = 0;
    for (int i = d - 1; i >= 0; --i) {
      const int hi = (m >> i) & 1;
      w *= hi ? s[i] : 1.0 - s[i];
      g = g * n + c[i] + hi;
    }
    acc += w * (ar->U[g - ar->u_off] - Uj);
  }
  return acc;
}

/* H^a_j(U) at node g (multi-index mi, coordinates x) for control a */
INL double hamiltonian(const int d, const orc_problem* pb, const orc_arrays* ar, int64_t g, const double* x, int a, double Uj,
                          double dx, double k) {
  const int P = pb->P;
  const double inv_dx = 1.0 / dx, inv_2dx = 1.0 / (2.0 * dx);
  const int64_t fi = g - ar->f_off, ld = ar->f_ld;
  double L = 0.0;
  for (int p = 0; p < P; ++p) {
    const double sc = ar->sigma_scale ? ar->sigma_scale[p * ld + fi] : 1.0;
    double yp[3], ym[3];
    for (int i = 0; i < d; ++i) {
      double sg = pb->sigma_dir[(a * P + p) * d + i] * sc;
      if (ar->sigma_node) sg = sg + ar->sigma_node[(p * d + i) * ld + fi];
      yp[i] = k * sg;
      ym[i] = -k * sg;
    }
    int bp[3], bm[3];
    const double mup = trunc_mu(d, pb, x, yp, bp), mum = trunc_mu(d, pb, x, ym, bm);
    double A = 1.0, B = 1.0;    /* = 2/(1 + 1) when neither endpoint is truncated */
    if (mup < 1.0 || mum < 1.0) {
      A = 2.0 / (mup * mup + mup * mum);
      B = 2.0 / (mum * mum + mum * mup);
    }
    double zp[3], zm[3];
    endpoint(d, pb, x, yp, mup, bp, zp);
    endpoint(d, pb, x, ym, mum, bm, zm);
    L += A * inv_2dx * interp_diff(d, pb, ar, zp, Uj, inv_dx);
    L += B * inv_2dx * interp_diff(d, pb, ar, zm, Uj, inv_dx);
  }
  {  /* drift pair: y+ = y- = dx b, A = B = 1/mu, one endpoint counted twice */
    const double bs = ar->b_scale ? ar->b_scale[fi] : 1.0;
    double y[3];
    for (int i = 0; i < d; ++i) {
      double bv = pb->b_dir[a * d + i] * bs;
      if (ar->b_node) bv = bv + ar->b_node[i * ld + fi];
      y[i] = dx * bv;
    }
    int bd[3];
    const double mu = trunc_mu(d, pb, x, y, bd);
    double z[3];
    endpoint(d, pb, x, y, mu, bd, z);
    L += 2.0 * ((mu < 1.0 ? 1.0 / mu : 1.0) * inv_2dx) * interp_diff(d, pb, ar, z, Uj, inv_dx);
  }
  const double c = pb->c_ctrl[a] + (ar->c_node ? ar->c_node[fi] : 0.0);
  double f = pb->f_ctrl ? pb->f_ctrl[a] : 0.0;
  for (int q = 0; q < pb->Q; ++q) f += pb->f_basis[a * pb->Q + q] * ar->f_feat[q * ld + fi];
  return L + c * Uj + f;
}

/* R_j at node g (multi-index mi) of a d-dimensional grid; *arg = the lowest-index argmin */
INL double node_R(const int d, const orc_problem* pb, const orc_arrays* ar, const int64_t* mi, int* arg) {
  const int64_t n = pb->n;
  const double dx = (pb->hi - pb->lo) / (double)(n - 1);
  const double k = sqrt(dx);
  int64_t g = 0;
  for (int i = d - 1; i >= 0; --i) g = g * n + mi[i];
  double x[3];
  for (int i = 0; i < d; ++i) x[i] = pb->lo + (double)mi[i] * dx;
  const double Uj = ar->U[g - ar->u_off];
  double best = INFINITY;
  *arg = 0;
  for (int a = 0; a < pb->K; ++a) {
    const double H = hamiltonian(d, pb, ar, g, x, a, Uj, dx, k);
    if (H < best) { best = H; *arg = a; }   /* strict: lowest index on exact ties (reading iv) */
  }
  const double R = fabs(Uj - ar->Uprev[g - ar->f_off] - pb->dt * best);
  return (R != R) ? INFINITY : R;
}
/* the dimension as a literal, so the per-endpoint loops unroll */
static double node_R2(const orc_problem* pb, const orc_arrays* ar, const int64_t* mi, int* arg) {
  return node_R(2, pb, ar, mi, arg);
}
static double node_R3(const orc_problem* pb, const orc_arrays* ar, const int64_t* mi, int* arg) {
  return node_R(3, pb, ar, mi, arg);
}

/* max_j R_j(U) over the interior nodes of rows [r0, r1) of the slowest axis; optional argmin policy
 * (policy[g - f_off]) and per-row R (Rrow[g - f_off]).  Returns max R (NaN propagates as +inf). */
double orc_residual_rows(const orc_problem* pb, const orc_arrays* ar, int64_t r0, int64_t r1, uint8_t* policy,
                         double* Rrow) {
  const int d = pb->d;
  const int64_t n = pb->n;
  const int64_t per_row = (d == 2) ? (n - 2) : (n - 2) * (n - 2);
  const int64_t total = (r1 - r0) * per_row;
  double Rmax = 0.0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(max : Rmax)
  for (int64_t q = 0; q < total; ++q) {
    const int64_t row = r0 + q / per_row, rem = q % per_row;
    int64_t mi[3];
    mi[0] = 1 + rem % (n - 2);
    if (d == 3) mi[1] = 1 + rem / (n - 2);
    mi[d - 1] = row;
    int arg;
    const double R = (d == 2) ? node_R2(pb, ar, mi, &arg) : node_R3(pb, ar, mi, &arg);
    int64_t g = 0;
    for (int i = d - 1; i >= 0; --i) g = g * n + mi[i];
    if (policy) policy[g - ar->f_off] = (uint8_t)arg;
    if (Rrow) Rrow[g - ar->f_off] = R;
    if (R > Rmax) Rmax = R;
  }
  return Rmax;
}
