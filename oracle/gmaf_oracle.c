/*
 * gmaf_oracle.c -- TEST INFRASTRUCTURE ONLY (see gmaf_oracle.h).
 *
 * Plain single-threaded C11, FP64, compiled with -O2 -ffp-contract=off
 * -fno-fast-math so that every expression below is evaluated exactly in the
 * written order with no FMA contraction.  Loops are written in the paper's
 * order and notation; no blocking, fusion or reordering.
 */
#include "gmaf_oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ------------------------------------------------------------------ grid */

int orc_check_grid(const orc_grid* g) {
  if (!g) return ORC_E_INVALID_ARG;
  if (g->n_theta < 4 || g->n_y < 4) return ORC_E_INVALID_MESH;
  if (!(g->R_k > 0.0) || !(g->R_c > g->R_k) || !(g->mu > 0.0)) return ORC_E_INVALID_ARG;
  if (g->tex_n_theta > 0 || g->tex_n_y > 0) {
    if (g->tex_n_theta <= 0 || g->tex_n_y <= 0 || g->tex_band_rows <= 0 ||
        g->tex_band_rows > g->n_y || g->tex_fill_den <= 0 || g->tex_fill_num < 0 ||
        g->tex_fill_num > g->tex_fill_den || g->tex_depth < 0.0)
      return ORC_E_INVALID_ARG;
    /* MeshTooCoarse: fewer than 2 nodes per texture pitch in either direction */
    if (g->n_theta < 2 * g->tex_n_theta || g->tex_band_rows < 2 * g->tex_n_y)
      return ORC_E_MESH_TOO_COARSE;
  }
  return ORC_OK;
}

/* O2 texture mask (Fig. 10; R-A7): integer arithmetic only. */
int orc_texture_mask(const orc_grid* g, int32_t i, int32_t j) {
  if (g->tex_n_theta <= 0 || g->tex_n_y <= 0) return 0;
  if (j < 0 || j >= g->tex_band_rows) return 0;     /* ghost row -1 and rows above the band */
  int64_t nt = g->n_theta, B = g->tex_band_rows;
  int64_t N = g->tex_fill_num, D = g->tex_fill_den;
  int64_t ci = ((int64_t)i * (int64_t)g->tex_n_theta) % nt;
  int64_t cj = ((int64_t)j * (int64_t)g->tex_n_y) % B;
  return (D * ci < N * nt) && (D * cj < N * B);
}

/* ------------------------------------------------------------ thickness */

/* O3 (Eq. 2.3) and O4 (chain rule through e-dot, Eq. 2.2). */
int orc_thickness(const orc_grid* g, const orc_cond* c, double* h, double* hdot, double* bad) {
  int rc = orc_check_grid(g);
  if (rc != ORC_OK) return rc;
  const int32_t nt = g->n_theta, ny = g->n_y;
  const double dtheta = (2.0 * M_PI) / (double)nt;
  const double dy = c->L_F / (double)(ny + 1);
  const double sl = (c->e[2] - c->e[0]) / c->L_F;       /* (e3-e1)/L_F */
  const double tl = (c->e[3] - c->e[1]) / c->L_F;       /* (e4-e2)/L_F */
  const double sld = (c->edot[2] - c->edot[0]) / c->L_F;
  const double tld = (c->edot[3] - c->edot[1]) / c->L_F;
  int status = ORC_OK;
  for (int32_t j = -1; j <= ny; ++j) {
    const double y = (double)(j + 1) * dy;
    for (int32_t i = 0; i < nt; ++i) {
      const double th = (double)i * dtheta;
      const double ct = cos(th), st = sin(th);
      const double a = (g->R_c * ct - sl * y) - c->e[0];
      const double b = (g->R_c * st - tl * y) - c->e[1];
      const double r = sqrt(a * a + b * b);
      const double ht = orc_texture_mask(g, i, j) ? g->tex_depth : 0.0;
      const double hv = (r - g->R_k) + ht;
      const double ad = -(sld * y + c->edot[0]);
      const double bd = -(tld * y + c->edot[1]);
      const double hd = (a * ad + b * bd) / r;
      const size_t idx = (size_t)(j + 1) * (size_t)nt + (size_t)i;
      if (h) h[idx] = hv;
      if (hdot) hdot[idx] = hd;
      if (hv < g->h_min && status == ORC_OK) {
        status = ORC_E_NONPOSITIVE_THICKNESS;
        if (bad) { bad[0] = (double)i; bad[1] = (double)j; bad[2] = hv; }
      }
    }
  }
  return status;
}

/* ------------------------------------------------------------- assembly */

/* O5 (Eqs. 2.4-2.7; R-A1..A6).  A = -(discrete div g grad), SPD. */
int orc_assemble(const orc_grid* g, const orc_cond* c, double* AP, double* AE, double* AN, double* S) {
  const int32_t nt = g->n_theta, ny = g->n_y;
  const size_t nrow = (size_t)(ny + 2) * (size_t)nt;
  double* h = (double*)malloc(nrow * sizeof(double));
  double* hd = (double*)malloc(nrow * sizeof(double));
  double* gg = (double*)malloc(nrow * sizeof(double));
  if (!h || !hd || !gg) { free(h); free(hd); free(gg); return ORC_E_INVALID_ARG; }
  int rc = orc_thickness(g, c, h, hd, NULL);
  if (rc != ORC_OK) { free(h); free(hd); free(gg); return rc; }

  const double dtheta = (2.0 * M_PI) / (double)nt;
  const double dy = c->L_F / (double)(ny + 1);
  const double dx = g->R_k * dtheta;
  const double rx = dy / dx, ry = dx / dy;
  const double twelve_mu = 12.0 * g->mu;
#define H(i, j) h[(size_t)((j) + 1) * (size_t)nt + (size_t)(i)]
#define HD(i, j) hd[(size_t)((j) + 1) * (size_t)nt + (size_t)(i)]
#define G(i, j) gg[(size_t)((j) + 1) * (size_t)nt + (size_t)(i)]
  for (size_t q = 0; q < nrow; ++q) gg[q] = ((h[q] * h[q]) * h[q]) / twelve_mu;

  for (int32_t j = 0; j < ny; ++j) {
    for (int32_t i = 0; i < nt; ++i) {
      const int32_t iE = (i + 1) % nt, iW = (i + nt - 1) % nt;
      /* harmonic face conductances (R-A4) */
      const double gP = G(i, j), gE = G(iE, j), gW = G(iW, j), gN = G(i, j + 1), gS = G(i, j - 1);
      const double ge = ((2.0 * gP) * gE) / (gP + gE);
      const double gw = ((2.0 * gW) * gP) / (gW + gP);   /* = ge(iW, j) */
      const double gn = ((2.0 * gP) * gN) / (gP + gN);
      const double gs = ((2.0 * gS) * gP) / (gS + gP);   /* = gn(i, j-1) */
      const double aE = ge * rx, aW = gw * rx, aN = gn * ry, aS = gs * ry;
      const size_t k = (size_t)j * (size_t)nt + (size_t)i;
      AP[k] = ((aW + aE) + aS) + aN;
      AE[k] = -aE;                                       /* i = nt-1: wrap band A_EB (Eq. 2.7) */
      AN[k] = (j < ny - 1) ? -aN : 0.0;
      /* source: wedge (both sliding components, R-A1), squeeze (R-A5) */
      const double t1 = ((c->U_theta * 0.5) * ((H(iE, j) - H(iW, j)) * 0.5)) * dy;
      const double t2 = ((c->U_y * 0.5) * ((H(i, j + 1) - H(i, j - 1)) * 0.5)) * dx;
      const double t3 = (HD(i, j) * dx) * dy;
      double s = -((t1 + t2) + t3);
      if (j == 0) s = s + aS * c->p_in;                  /* Dirichlet fold, "linear transform" P:53 */
      if (j == ny - 1) s = s + aN * c->p_out;
      S[k] = s;
    }
  }
#undef H
#undef HD
#undef G
  free(h); free(hd); free(gg);
  return ORC_OK;
}

/* ------------------------------------------------------------ operators */

/* Coefficient of the stencil neighbour, from the 3 stored symmetric bands. */
static double aw_coef(int32_t nt, const double* AE, int32_t i, int32_t j) {  /* A_W(i,j) */
  return AE[(size_t)j * nt + (size_t)((i + nt - 1) % nt)];
}
static double as_coef(int32_t nt, const double* AN, int32_t i, int32_t j) {  /* A_S(i,j) */
  return (j > 0) ? AN[(size_t)(j - 1) * nt + (size_t)i] : 0.0;
}

/* Eq. 2.4: y_P = A_P x_P + A_E x_E + A_W x_W + A_S x_S + A_N x_N (summed W, E, S, N). */
void orc_spmv(int32_t nt, int32_t ny, const double* AP, const double* AE, const double* AN,
              const double* x, double* y) {
  for (int32_t j = 0; j < ny; ++j)
    for (int32_t i = 0; i < nt; ++i) {
      const size_t k = (size_t)j * nt + i;
      const int32_t iE = (i + 1) % nt, iW = (i + nt - 1) % nt;
      double s = AP[k] * x[k];
      s += aw_coef(nt, AE, i, j) * x[(size_t)j * nt + iW];
      s += AE[k] * x[(size_t)j * nt + iE];
      if (j > 0) s += as_coef(nt, AN, i, j) * x[k - nt];
      if (j < ny - 1) s += AN[k] * x[k + nt];
      y[k] = s;
    }
}

/* O6: ASSOR-II two-step apply (Eqs. 3.5-3.6), natural ordering idx = i + nt*j
 * (Eq. 3.8).  L(i,j) = {W if i>=1; E-wrap if i=nt-1; S if j>=1};
 * U(i,j) = {E if i<=nt-2; W-wrap if i=0; N if j<=ny-2}  (R-A12). */
static void assor2_apply(int32_t nt, int32_t ny, const double* AP, const double* AE, const double* AN,
                         double omega, const double* r, double* z) {
  const size_t n = (size_t)nt * ny;
  double* w = (double*)malloc(n * sizeof(double));
  double* v = (double*)malloc(n * sizeof(double));
  for (size_t k = 0; k < n; ++k) w[k] = r[k] / AP[k];               /* w = D^-1 r */
  for (int32_t j = 0; j < ny; ++j)                                   /* v = (I - w D^-1 L) w */
    for (int32_t i = 0; i < nt; ++i) {
      const size_t k = (size_t)j * nt + i;
      double s = 0.0;
      if (i >= 1) s += AE[k - 1] * w[k - 1];                         /* W */
      if (i == nt - 1) s += AE[k] * w[(size_t)j * nt];               /* E-wrap (lower) */
      if (j >= 1) s += AN[k - nt] * w[k - nt];                       /* S */
      v[k] = w[k] - (omega / AP[k]) * s;
    }
  const double c = (2.0 - omega) * omega;
  for (int32_t j = 0; j < ny; ++j)                                   /* z = c (I - w D^-1 L^T) v */
    for (int32_t i = 0; i < nt; ++i) {
      const size_t k = (size_t)j * nt + i;
      double s = 0.0;
      if (i == 0) s += AE[(size_t)j * nt + (nt - 1)] * v[(size_t)j * nt + (nt - 1)]; /* W-wrap (upper) */
      if (i <= nt - 2) s += AE[k] * v[k + 1];                        /* E */
      if (j <= ny - 2) s += AN[k] * v[k + nt];                       /* N */
      z[k] = c * (v[k] - (omega / AP[k]) * s);
    }
  free(w); free(v);
}

/* ASSOR-I (Eq. 3.2): z_i = w(2-w) r_i / (D_i + w^2 sum_{k<i} L_ik^2 / D_k). */
static void assor1_apply(int32_t nt, int32_t ny, const double* AP, const double* AE, const double* AN,
                         double omega, const double* r, double* z) {
  const double c = omega * (2.0 - omega);
  for (int32_t j = 0; j < ny; ++j)
    for (int32_t i = 0; i < nt; ++i) {
      const size_t k = (size_t)j * nt + i;
      double s = 0.0;
      if (i >= 1) s += (AE[k - 1] * AE[k - 1]) / AP[k - 1];
      if (i == nt - 1) s += (AE[k] * AE[k]) / AP[(size_t)j * nt];
      if (j >= 1) s += (AN[k - nt] * AN[k - nt]) / AP[k - nt];
      z[k] = (c * r[k]) / (AP[k] + (omega * omega) * s);
    }
}

/* SSOR (Eq. 2.9), applied EXACTLY by elimination -- the sequential triangular solves
 * the paper rejects for the GPU, which is why it is oracle-only:
 *   M = (D + w L) D^-1 (D + w L)^T / (w (2 - w))        (Eq. 2.9 at w = 1; Eq. 3.3 for w != 1)
 *   z = M^-1 r:  (D + w L) y = r   (forward, natural order idx = i + nt*j, Eq. 3.8)
 *                (D + w L^T) z' = D y   (backward),   z = w (2 - w) z'.
 * L is the strictly lower triangle of A in the natural ordering: W (i >= 1), the E-wrap of
 * column nt-1 and S (j >= 1); L^T holds E (i <= nt-2), the W-wrap of column 0 and N (R-A12). */
static void ssor_apply(int32_t nt, int32_t ny, const double* AP, const double* AE, const double* AN,
                       double omega, const double* r, double* z) {
  const size_t n = (size_t)nt * ny;
  double* y = (double*)malloc(n * sizeof(double));
  for (int32_t j = 0; j < ny; ++j)                                   /* forward: (D + w L) y = r */
    for (int32_t i = 0; i < nt; ++i) {
      const size_t k = (size_t)j * nt + i;
      double s = 0.0;
      if (i >= 1) s += AE[k - 1] * y[k - 1];                         /* W */
      if (i == nt - 1) s += AE[k] * y[(size_t)j * nt];               /* E-wrap: column 0 precedes */
      if (j >= 1) s += AN[k - nt] * y[k - nt];                       /* S */
      y[k] = (r[k] - omega * s) / AP[k];
    }
  for (int32_t j = ny - 1; j >= 0; --j)                              /* backward: (D + w L^T) z' = D y */
    for (int32_t i = nt - 1; i >= 0; --i) {
      const size_t k = (size_t)j * nt + i;
      double s = 0.0;
      if (i <= nt - 2) s += AE[k] * z[k + 1];                        /* E */
      if (i == 0) s += AE[(size_t)j * nt + (nt - 1)] * z[(size_t)j * nt + (nt - 1)]; /* W-wrap */
      if (j <= ny - 2) s += AN[k] * z[k + nt];                       /* N */
      z[k] = (AP[k] * y[k] - omega * s) / AP[k];
    }
  const double c = omega * (2.0 - omega);
  for (size_t k = 0; k < n; ++k) z[k] = c * z[k];
  free(y);
}

void orc_precond_apply(int32_t nt, int32_t ny, const double* AP, const double* AE, const double* AN,
                       int32_t precond, double omega, const double* r, double* z) {
  const size_t n = (size_t)nt * ny;
  switch (precond) {
    case ORC_PRECOND_SSOR: ssor_apply(nt, ny, AP, AE, AN, omega, r, z); break;
    case ORC_PRECOND_JACOBI: for (size_t k = 0; k < n; ++k) z[k] = r[k] / AP[k]; break;  /* Eq. 2.8 */
    case ORC_PRECOND_ASSOR2: assor2_apply(nt, ny, AP, AE, AN, omega, r, z); break;
    case ORC_PRECOND_ASSOR1: assor1_apply(nt, ny, AP, AE, AN, omega, r, z); break;
    default: for (size_t k = 0; k < n; ++k) z[k] = r[k]; break;
  }
}

int orc_expand_dense(int32_t nt, int32_t ny, const double* AP, const double* AE, const double* AN,
                     double* A) {
  const size_t n = (size_t)nt * ny;
  if (n > 4096) return ORC_E_INVALID_ARG;
  memset(A, 0, n * n * sizeof(double));
  for (int32_t j = 0; j < ny; ++j)
    for (int32_t i = 0; i < nt; ++i) {
      const size_t k = (size_t)j * nt + i;
      const size_t kE = (size_t)j * nt + (size_t)((i + 1) % nt);
      A[k * n + k] += AP[k];
      A[k * n + kE] += AE[k];      /* E (wrap at i = nt-1) */
      A[kE * n + k] += AE[k];      /* its symmetric W entry */
      if (j < ny - 1) { A[k * n + k + nt] += AN[k]; A[(k + nt) * n + k] += AN[k]; }
    }
  return ORC_OK;
}

/* Eq. 3.4 literally: M^-1 = (2-w) w D^-1 (I - w L^T D^-1) D (I - w D^-1 L) D^-1. */
int orc_assor2_dense(int32_t nt, int32_t ny, const double* AP, const double* AE, const double* AN,
                     double omega, double* Minv) {
  const size_t n = (size_t)nt * ny;
  if (n > 4096) return ORC_E_INVALID_ARG;
  double* A = (double*)malloc(n * n * sizeof(double));
  double* X = (double*)malloc(n * n * sizeof(double));   /* (I - w D^-1 L) D^-1 */
  double* Y = (double*)malloc(n * n * sizeof(double));   /* D^-1 (I - w L^T D^-1) D */
  orc_expand_dense(nt, ny, AP, AE, AN, A);
  for (size_t a = 0; a < n; ++a)
    for (size_t b = 0; b < n; ++b) {
      const double L_ab = (b < a) ? A[a * n + b] : 0.0;             /* strictly lower */
      const double LT_ab = (a < b) ? A[b * n + a] : 0.0;            /* (L^T)_ab = L_ba */
      const double Iab = (a == b) ? 1.0 : 0.0;
      X[a * n + b] = (Iab - omega * L_ab / AP[a]) / AP[b];
      Y[a * n + b] = (Iab - omega * LT_ab / AP[b]) * AP[b] / AP[a];
    }
  const double c = (2.0 - omega) * omega;
  for (size_t a = 0; a < n; ++a)
    for (size_t b = 0; b < n; ++b) {
      double s = 0.0;
      for (size_t m = 0; m < n; ++m) s += Y[a * n + m] * X[m * n + b];
      Minv[a * n + b] = c * s;
    }
  free(A); free(X); free(Y);
  return ORC_OK;
}

/* Textbook Cholesky A = L L^T, then forward/back substitution (O9). */
int orc_cholesky_solve(int32_t n, double* A, const double* b, double* x) {
  for (int32_t j = 0; j < n; ++j) {
    double d = A[(size_t)j * n + j];
    for (int32_t k = 0; k < j; ++k) d -= A[(size_t)j * n + k] * A[(size_t)j * n + k];
    if (!(d > 0.0)) return ORC_E_BREAKDOWN;
    const double ljj = sqrt(d);
    A[(size_t)j * n + j] = ljj;
    for (int32_t i = j + 1; i < n; ++i) {
      double s = A[(size_t)i * n + j];
      for (int32_t k = 0; k < j; ++k) s -= A[(size_t)i * n + k] * A[(size_t)j * n + k];
      A[(size_t)i * n + j] = s / ljj;
    }
  }
  double* yv = (double*)malloc((size_t)n * sizeof(double));
  for (int32_t i = 0; i < n; ++i) {
    double s = b[i];
    for (int32_t k = 0; k < i; ++k) s -= A[(size_t)i * n + k] * yv[k];
    yv[i] = s / A[(size_t)i * n + i];
  }
  for (int32_t i = n - 1; i >= 0; --i) {
    double s = yv[i];
    for (int32_t k = i + 1; k < n; ++k) s -= A[(size_t)k * n + i] * x[k];
    x[i] = s / A[(size_t)i * n + i];
  }
  free(yv);
  return ORC_OK;
}

/* ------------------------------------------------------------------ PCG */

static double dot(size_t n, const double* a, const double* b) {
  double s = 0.0;
  for (size_t k = 0; k < n; ++k) s += a[k] * b[k];
  return s;
}

/* O7: Table 1 with r0 = S - A p0 (R-A9) on A_G p_G = S_G (Eq. 3.7);
 * synchronized stop ||r||/||S_G|| <= tol (Eq. 3.9, recursive residual R-A10). */
int orc_pcg_joint(int32_t nt, int32_t ny, int32_t K,
                  const double* AP, const double* AE, const double* AN, const double* S,
                  double* p, double tol, double omega, int32_t precond, int32_t coupling,
                  int32_t max_iter, int32_t warm, orc_stats* st, double* history, double* cond_rel) {
  if (nt < 4 || ny < 4 || K < 1 || max_iter < 0) return ORC_E_INVALID_ARG;
  const size_t n = (size_t)nt * ny, N = n * (size_t)K;
  double* r = (double*)malloc(N * sizeof(double));
  double* z = (double*)malloc(N * sizeof(double));
  double* u = (double*)malloc(N * sizeof(double));
  double* v = (double*)malloc(N * sizeof(double));
  double* dk = (double*)calloc((size_t)K, sizeof(double));
  double* dk2 = (double*)calloc((size_t)K, sizeof(double));
  double* uvk = (double*)calloc((size_t)K, sizeof(double));
  double* Sk = (double*)calloc((size_t)K, sizeof(double));
#define BLK(ptr, k) ((ptr) + (size_t)(k) * n)
  /* step 1-2 */
  if (!warm) memset(p, 0, N * sizeof(double));
  for (int32_t k = 0; k < K; ++k) {
    orc_spmv(nt, ny, BLK(AP, k), BLK(AE, k), BLK(AN, k), BLK(p, k), BLK(v, k));
    for (size_t q = 0; q < n; ++q) BLK(r, k)[q] = BLK(S, k)[q] - BLK(v, k)[q];
    orc_precond_apply(nt, ny, BLK(AP, k), BLK(AE, k), BLK(AN, k), precond, omega, BLK(r, k), BLK(z, k));
    for (size_t q = 0; q < n; ++q) BLK(u, k)[q] = BLK(z, k)[q];
    dk[k] = dot(n, BLK(r, k), BLK(z, k));
    Sk[k] = dot(n, BLK(S, k), BLK(S, k));
  }
  double d = 0.0, SS = 0.0, rr = 0.0;
  for (int32_t k = 0; k < K; ++k) { d += dk[k]; SS += Sk[k]; }
  for (int32_t k = 0; k < K; ++k) rr += dot(n, BLK(r, k), BLK(r, k));
  const double nS = sqrt(SS);
  int status = ORC_OK, converged = 0, it = 0;
  double rel = (nS > 0.0) ? sqrt(rr) / nS : 0.0;
  if (history) history[0] = rel;
  if (nS == 0.0) {                       /* S_G = 0 -> p = 0 (O7) */
    memset(p, 0, N * sizeof(double));
    converged = 1;
  } else if (rel <= tol) {
    converged = 1;
  }
  for (int32_t j = 0; !converged && j < max_iter; ++j) {
    /* step 3: v = A u, alpha = d / (u.v) */
    double uv = 0.0;
    for (int32_t k = 0; k < K; ++k) {
      orc_spmv(nt, ny, BLK(AP, k), BLK(AE, k), BLK(AN, k), BLK(u, k), BLK(v, k));
      uvk[k] = dot(n, BLK(u, k), BLK(v, k));
      uv += uvk[k];
    }
    if (coupling == ORC_COUPLED) {
      if (!(uv > 0.0)) { status = ORC_E_BREAKDOWN; break; }
      const double alpha = d / uv;
      for (size_t q = 0; q < N; ++q) p[q] = p[q] + alpha * u[q];   /* step 4 */
      for (size_t q = 0; q < N; ++q) r[q] = r[q] - alpha * v[q];   /* step 5 */
    } else {
      int bad = 0;
      for (int32_t k = 0; k < K; ++k) {
        double ak = 0.0;
        if (dk[k] != 0.0) { if (!(uvk[k] > 0.0)) { bad = 1; break; } ak = dk[k] / uvk[k]; }
        for (size_t q = 0; q < n; ++q) BLK(p, k)[q] = BLK(p, k)[q] + ak * BLK(u, k)[q];
        for (size_t q = 0; q < n; ++q) BLK(r, k)[q] = BLK(r, k)[q] - ak * BLK(v, k)[q];
      }
      if (bad) { status = ORC_E_BREAKDOWN; break; }
    }
    /* step 6: synchronized global convergence (Eq. 3.9) */
    rr = 0.0;
    for (int32_t k = 0; k < K; ++k) rr += dot(n, BLK(r, k), BLK(r, k));
    rel = sqrt(rr) / nS;
    it = j + 1;
    if (history) history[it] = rel;
    if (rel <= tol) { converged = 1; break; }
    /* step 7-8 */
    double d2 = 0.0;
    for (int32_t k = 0; k < K; ++k) {
      orc_precond_apply(nt, ny, BLK(AP, k), BLK(AE, k), BLK(AN, k), precond, omega, BLK(r, k), BLK(z, k));
      dk2[k] = dot(n, BLK(r, k), BLK(z, k));
      d2 += dk2[k];
    }
    /* step 9 */
    if (coupling == ORC_COUPLED) {
      if (!(d2 > 0.0)) { status = ORC_E_BREAKDOWN; break; }
      const double beta = d2 / d;
      for (size_t q = 0; q < N; ++q) u[q] = z[q] + beta * u[q];
      d = d2;
    } else {
      int bad = 0;
      for (int32_t k = 0; k < K; ++k) {
        double bk = 0.0;
        if (dk[k] != 0.0) { if (dk2[k] < 0.0) { bad = 1; break; } bk = dk2[k] / dk[k]; }
        for (size_t q = 0; q < n; ++q) BLK(u, k)[q] = BLK(z, k)[q] + bk * BLK(u, k)[q];
        dk[k] = dk2[k];
      }
      if (bad) { status = ORC_E_BREAKDOWN; break; }
    }
  }
  if (status == ORC_OK && !converged) status = ORC_E_NO_CONVERGENCE;
  /* true residual at exit */
  double tr = 0.0;
  for (int32_t k = 0; k < K; ++k) {
    orc_spmv(nt, ny, BLK(AP, k), BLK(AE, k), BLK(AN, k), BLK(p, k), BLK(v, k));
    double tk = 0.0, rk = 0.0;
    for (size_t q = 0; q < n; ++q) {
      const double e = BLK(S, k)[q] - BLK(v, k)[q];
      tk += e * e;
    }
    rk = dot(n, BLK(r, k), BLK(r, k));
    tr += tk;
    if (cond_rel) cond_rel[k] = (Sk[k] > 0.0) ? sqrt(rk) / sqrt(Sk[k]) : 0.0;
  }
  if (st) {
    st->iterations = it;
    st->converged = converged;
    st->status = status;
    st->rel_residual = rel;
    st->true_rel_residual = (nS > 0.0) ? sqrt(tr) / nS : 0.0;
  }
#undef BLK
  free(r); free(z); free(u); free(v); free(dk); free(dk2); free(uvk); free(Sk);
  return status;
}

/* Test hook for the restart branch of the single-reduction recurrence (R-A32): restart when
 * den <= thresh * delta'.  thresh = 0 (the default) is the method itself (restart only when the
 * denominator has lost its sign); thresh >= 1 restarts at EVERY iteration (den < delta' always,
 * since beta gamma'/alpha > 0), which turns the recurrence into preconditioned steepest descent --
 * the form tests/test_oracle_pcg.py pins it against.  The count of restarts taken by the last
 * orc_pcg_joint_sr call is returned by orc_sr_restarts(). */
static double g_sr_restart_thresh = 0.0;
static int32_t g_sr_restarts = 0;
void orc_sr_set_restart_threshold(double thresh) { g_sr_restart_thresh = thresh; }
int32_t orc_sr_restarts(void) { return g_sr_restarts; }

/* O7-S3: the same PCG (Table 1) written with a single global reduction per
 * iteration (Chronopoulos & Gear's reformulation; SURVEY 8(c) O7 "S3 mode",
 * 8(e)): the search direction pd and s = A pd are updated as in Table 1 steps
 * 3-5/9, but alpha is obtained from gamma = r.z and delta = z.(A z) of the SAME
 * iterate, alpha_{j+1} = gamma_{j+1} / (delta_{j+1} - beta_{j+1} gamma_{j+1} / alpha_j),
 * which equals d / (u.A u) of Table 1 in exact arithmetic.  One (gamma, delta, r.r)
 * reduction per iteration is what the single-pass GPU schedule computes. */
int orc_pcg_joint_sr(int32_t nt, int32_t ny, int32_t K,
                     const double* AP, const double* AE, const double* AN, const double* S,
                     double* p, double tol, double omega, int32_t precond, int32_t coupling,
                     int32_t max_iter, int32_t warm, orc_stats* st, double* history, double* cond_rel) {
  if (nt < 4 || ny < 4 || K < 1 || max_iter < 0) return ORC_E_INVALID_ARG;
  const size_t n = (size_t)nt * ny, N = n * (size_t)K;
  double* r = (double*)malloc(N * sizeof(double));
  double* z = (double*)malloc(N * sizeof(double));
  double* w = (double*)malloc(N * sizeof(double));
  double* pd = (double*)calloc(N, sizeof(double));
  double* sv = (double*)malloc(N * sizeof(double));
  double* gk = (double*)calloc((size_t)K, sizeof(double));
  double* dk = (double*)calloc((size_t)K, sizeof(double));
  double* ak = (double*)calloc((size_t)K, sizeof(double));
  double* bk = (double*)calloc((size_t)K, sizeof(double));
  double* Sk = (double*)calloc((size_t)K, sizeof(double));
#define BLK(ptr, k) ((ptr) + (size_t)(k) * n)
  if (!warm) memset(p, 0, N * sizeof(double));
  g_sr_restarts = 0;
  double SS = 0.0, rr = 0.0;
  for (int32_t k = 0; k < K; ++k) {
    orc_spmv(nt, ny, BLK(AP, k), BLK(AE, k), BLK(AN, k), BLK(p, k), BLK(sv, k));
    for (size_t q = 0; q < n; ++q) BLK(r, k)[q] = BLK(S, k)[q] - BLK(sv, k)[q];
    orc_precond_apply(nt, ny, BLK(AP, k), BLK(AE, k), BLK(AN, k), precond, omega, BLK(r, k), BLK(z, k));
    orc_spmv(nt, ny, BLK(AP, k), BLK(AE, k), BLK(AN, k), BLK(z, k), BLK(w, k));
    gk[k] = dot(n, BLK(r, k), BLK(z, k));
    dk[k] = dot(n, BLK(z, k), BLK(w, k));
    Sk[k] = dot(n, BLK(S, k), BLK(S, k));
  }
  for (int32_t k = 0; k < K; ++k) SS += Sk[k];
  for (int32_t k = 0; k < K; ++k) rr += dot(n, BLK(r, k), BLK(r, k));
  const double nS = sqrt(SS);
  int status = ORC_OK, converged = 0, it = 0;
  double rel = (nS > 0.0) ? sqrt(rr) / nS : 0.0;
  if (history) history[0] = rel;
  double gam = 0.0, alpha = 0.0, beta = 0.0;
  if (nS == 0.0) { memset(p, 0, N * sizeof(double)); converged = 1; }
  else if (rel <= tol) converged = 1;
  else {
    if (coupling == ORC_COUPLED) {
      double dl = 0.0;
      for (int32_t k = 0; k < K; ++k) { gam += gk[k]; dl += dk[k]; }
      if (!(dl > 0.0)) status = ORC_E_BREAKDOWN;
      alpha = gam / dl;
    } else {
      for (int32_t k = 0; k < K; ++k) {
        ak[k] = 0.0;
        if (gk[k] != 0.0) { if (!(dk[k] > 0.0)) status = ORC_E_BREAKDOWN; ak[k] = gk[k] / dk[k]; }
      }
    }
  }
  for (int32_t j = 0; status == ORC_OK && !converged && j < max_iter; ++j) {
    for (int32_t k = 0; k < K; ++k) {
      const double a = (coupling == ORC_COUPLED) ? alpha : ak[k];
      const double b = (coupling == ORC_COUPLED) ? beta : bk[k];
      for (size_t q = 0; q < n; ++q) BLK(pd, k)[q] = BLK(z, k)[q] + b * BLK(pd, k)[q];   /* step 9 */
      orc_spmv(nt, ny, BLK(AP, k), BLK(AE, k), BLK(AN, k), BLK(pd, k), BLK(sv, k));    /* step 3 */
      for (size_t q = 0; q < n; ++q) BLK(p, k)[q] = BLK(p, k)[q] + a * BLK(pd, k)[q];  /* step 4 */
      for (size_t q = 0; q < n; ++q) BLK(r, k)[q] = BLK(r, k)[q] - a * BLK(sv, k)[q];  /* step 5 */
    }
    rr = 0.0;
    for (int32_t k = 0; k < K; ++k) rr += dot(n, BLK(r, k), BLK(r, k));
    rel = sqrt(rr) / nS;
    it = j + 1;
    if (history) history[it] = rel;
    if (rel <= tol) { converged = 1; break; }                                            /* step 6 */
    for (int32_t k = 0; k < K; ++k) {                                                    /* step 7-8 */
      orc_precond_apply(nt, ny, BLK(AP, k), BLK(AE, k), BLK(AN, k), precond, omega, BLK(r, k), BLK(z, k));
      orc_spmv(nt, ny, BLK(AP, k), BLK(AE, k), BLK(AN, k), BLK(z, k), BLK(w, k));
    }
    if (coupling == ORC_COUPLED) {
      double g2 = 0.0, d2 = 0.0;
      for (int32_t k = 0; k < K; ++k) { g2 += dot(n, BLK(r, k), BLK(z, k)); d2 += dot(n, BLK(z, k), BLK(w, k)); }
      if (!(g2 > 0.0)) { status = ORC_E_BREAKDOWN; break; }
      beta = g2 / gam;
      const double den = d2 - beta * g2 / alpha;
      if (den > g_sr_restart_thresh * d2) alpha = g2 / den;
      else if (d2 > 0.0) { beta = 0.0; alpha = g2 / d2; ++g_sr_restarts; }   /* restart along z (R-A32) */
      else { status = ORC_E_BREAKDOWN; break; }
      gam = g2;
    } else {
      for (int32_t k = 0; k < K; ++k) {
        const double g2 = dot(n, BLK(r, k), BLK(z, k)), d2 = dot(n, BLK(z, k), BLK(w, k));
        if (gk[k] == 0.0 || ak[k] == 0.0) { ak[k] = 0.0; bk[k] = 0.0; gk[k] = g2; continue; }
        if (g2 < 0.0) { status = ORC_E_BREAKDOWN; break; }
        bk[k] = g2 / gk[k];
        const double den = d2 - bk[k] * g2 / ak[k];
        if (den > g_sr_restart_thresh * d2) ak[k] = (g2 == 0.0) ? 0.0 : g2 / den;
        else if (d2 > 0.0) { bk[k] = 0.0; ak[k] = g2 / d2; ++g_sr_restarts; }   /* restart along z (R-A32) */
        else { status = ORC_E_BREAKDOWN; break; }
        gk[k] = g2;
      }
    }
  }
  if (status == ORC_OK && !converged) status = ORC_E_NO_CONVERGENCE;
  double tr = 0.0;
  for (int32_t k = 0; k < K; ++k) {
    orc_spmv(nt, ny, BLK(AP, k), BLK(AE, k), BLK(AN, k), BLK(p, k), BLK(sv, k));
    double tk = 0.0;
    for (size_t q = 0; q < n; ++q) { const double e = BLK(S, k)[q] - BLK(sv, k)[q]; tk += e * e; }
    tr += tk;
    if (cond_rel) cond_rel[k] = (Sk[k] > 0.0) ? sqrt(dot(n, BLK(r, k), BLK(r, k))) / sqrt(Sk[k]) : 0.0;
  }
  if (st) {
    st->iterations = it; st->converged = converged; st->status = status; st->rel_residual = rel;
    st->true_rel_residual = (nS > 0.0) ? sqrt(tr) / nS : 0.0;
  }
#undef BLK
  free(r); free(z); free(w); free(pd); free(sv); free(gk); free(dk); free(ak); free(bk); free(Sk);
  return status;
}

/* Asynchronous strategy (Eq. 3.10): per-block Krylov processes,
 * each frozen at its own convergence. */
int orc_pcg_async(int32_t nt, int32_t ny, int32_t K,
                  const double* AP, const double* AE, const double* AN, const double* S,
                  double* p, double tol, double omega, int32_t precond, int32_t max_iter,
                  int32_t* iters_k, orc_stats* st) {
  const size_t n = (size_t)nt * ny;
  int status = ORC_OK, all_conv = 1, maxit = 0;
  for (int32_t k = 0; k < K; ++k) {
    orc_stats sk;
    int rc = orc_pcg_joint(nt, ny, 1, AP + k * n, AE + k * n, AN + k * n, S + k * n, p + k * n,
                           tol, omega, precond, ORC_COUPLED, max_iter, 0, &sk, NULL, NULL);
    if (iters_k) iters_k[k] = sk.iterations;
    if (sk.iterations > maxit) maxit = sk.iterations;
    if (!sk.converged) all_conv = 0;
    if (rc != ORC_OK && status == ORC_OK) status = rc;
  }
  if (st) { st->iterations = maxit; st->converged = all_conv; st->status = status;
            st->rel_residual = 0.0; st->true_rel_residual = 0.0; }
  return status;
}

/* ----------------------------------------------------------- quadrature */

/* O8 (Sec. 2.4-III; R-A14): per surface element between nodes,
 * pressure traction -p n and Couette-Poiseuille wall shear on the piston,
 * moments about the bottom centre (0,0,0).  Sum in (j, i) order. */
int orc_wrench(const orc_grid* g, const orc_cond* c, const double* p, double* w) {
  const int32_t nt = g->n_theta, ny = g->n_y;
  const size_t nrow = (size_t)(ny + 2) * (size_t)nt;
  double* h = (double*)malloc(nrow * sizeof(double));
  int rc = orc_thickness(g, c, h, NULL, NULL);
  if (rc != ORC_OK) { free(h); return rc; }
  const double dtheta = (2.0 * M_PI) / (double)nt;
  const double dy = c->L_F / (double)(ny + 1);
  const double dx = g->R_k * dtheta;
  const double dA = dx * dy;
  double acc[12];
  for (int q = 0; q < 12; ++q) acc[q] = 0.0;
  for (int32_t j = -1; j <= ny - 1; ++j) {
    const double y0 = (double)(j + 1) * dy, y1 = (double)(j + 2) * dy;
    const double yc = (y0 + y1) * 0.5;
    for (int32_t i = 0; i < nt; ++i) {
      const int32_t i1 = (i + 1) % nt;
      /* corner pressures; ghost rows carry the Dirichlet data */
      const double p00 = (j < 0) ? c->p_in : p[(size_t)j * nt + i];
      const double p10 = (j < 0) ? c->p_in : p[(size_t)j * nt + i1];
      const double p01 = (j + 1 >= ny) ? c->p_out : p[(size_t)(j + 1) * nt + i];
      const double p11 = (j + 1 >= ny) ? c->p_out : p[(size_t)(j + 1) * nt + i1];
      const double h00 = h[(size_t)(j + 1) * nt + i], h10 = h[(size_t)(j + 1) * nt + i1];
      const double h01 = h[(size_t)(j + 2) * nt + i], h11 = h[(size_t)(j + 2) * nt + i1];
      const double pb = (((p00 + p10) + p01) + p11) * 0.25;
      const double hb = (((h00 + h10) + h01) + h11) * 0.25;
      const double dpdx = ((p10 + p11) - (p00 + p01)) / (2.0 * dx);
      const double dpdy = ((p01 + p11) - (p00 + p10)) / (2.0 * dy);
      const double thc = ((double)i + 0.5) * dtheta;
      const double cc = cos(thc), sc = sin(thc);
      const double rxv = g->R_k * cc, ryv = g->R_k * sc, rzv = yc;
      /* pressure traction on the piston */
      const double fx = -pb * cc * dA, fy = -pb * sc * dA, fz = 0.0;
      acc[0] += fx; acc[1] += fy; acc[2] += fz;
      acc[3] += ryv * fz - rzv * fy;
      acc[4] += rzv * fx - rxv * fz;
      acc[5] += rxv * fy - ryv * fx;
      /* viscous shear on the piston: tau = -(h/2) grad p - mu U / h */
      const double tth = -(hb * 0.5) * dpdx - (g->mu * c->U_theta) / hb;
      const double ty = -(hb * 0.5) * dpdy - (g->mu * c->U_y) / hb;
      const double sx = -tth * sc * dA, sy = tth * cc * dA, sz = ty * dA;
      acc[6] += sx; acc[7] += sy; acc[8] += sz;
      acc[9] += ryv * sz - rzv * sy;
      acc[10] += rzv * sx - rxv * sz;
      acc[11] += rxv * sy - ryv * sx;
    }
  }
  for (int q = 0; q < 12; ++q) w[q] = acc[q];
  free(h);
  return ORC_OK;
}
