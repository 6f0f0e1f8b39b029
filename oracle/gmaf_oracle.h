/*
 * gmaf_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded FP64 CPU oracle for the GMAF hot path
 * (arXiv 2511.06824): film thickness (Eq. 2.3), FVM assembly (Eqs. 2.4-2.7),
 * PCG (Table 1, sign fixed) with Jacobi (Eq. 2.8) / exact SSOR (Eq. 2.9) / ASSOR-I (Eq. 3.2) /
 * ASSOR-II (Eqs. 3.4-3.6) on the joint block-diagonal system (Eqs. 3.7-3.9),
 * a dense Cholesky reference, and the force/moment quadrature (Sec. 2.4-III).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
 * --impl reference) may load this library.  It shares no code, header,
 * table or constant generator with the CUDA product library; both consume
 * the same seeded inputs from gmaf_inputs/.
 *
 * Citations "P:n" are PAPER.md line numbers; "S:n" SPEC.md lines; "R-Ax"
 * are the readings listed in DESIGN.md section 3.
 *
 * Parity pins: every function is pinned by tests/test_oracle_*.py; the only
 * "parity unpinned" quantity is the absolute physical force of Figs. 4/6
 * (needs the unpublished Fig. 9 waveform and viscosity), see DESIGN.md.
 */
#ifndef GMAF_ORACLE_H
#define GMAF_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORC_OK = 0,
  ORC_E_INVALID_ARG = -1,
  ORC_E_INVALID_MESH = -2,        /* n_theta<4 or n_y<4 */
  ORC_E_MESH_TOO_COARSE = -3,     /* <2 nodes per texture pitch */
  ORC_E_NONPOSITIVE_THICKNESS = -4, /* h < h_min */
  ORC_E_BREAKDOWN = -5,           /* u.v <= 0 or d <= 0 */
  ORC_E_NO_CONVERGENCE = -6       /* max_iter reached, best iterate kept */
};

enum { ORC_PRECOND_NONE = 0, ORC_PRECOND_JACOBI = 1, ORC_PRECOND_ASSOR2 = 2, ORC_PRECOND_ASSOR1 = 3,
       ORC_PRECOND_SSOR = 4 /* exact SSOR, Eq. 2.9 (omega = 1) / Eq. 3.3 (omega != 1); oracle only */ };
enum { ORC_COUPLED = 0, ORC_LOCKSTEP = 1 };

typedef struct {
  int32_t n_theta, n_y;          /* unknown nodes; theta periodic; ghost rows y=0, y=L_F */
  double R_k, R_c;               /* m, Table 8 */
  double mu;                     /* Pa.s (R-A8) */
  double h_min;                  /* m, guard */
  int32_t tex_n_theta, tex_n_y;  /* dimple counts, 0,0 = smooth (Fig. 10) */
  int32_t tex_band_rows;         /* dimples occupy rows [0, band) */
  int32_t tex_fill_num, tex_fill_den; /* dimple fraction of pitch per direction */
  double tex_depth;              /* m, 20e-6 */
} orc_grid;

typedef struct {
  double e[4], edot[4];          /* eccentricity and rate (Table 8) */
  double L_F;                    /* coupling length, m */
  double U_theta, U_y;           /* sliding speed of piston vs bore, m/s (R-A1) */
  double p_in, p_out;            /* Dirichlet pressures at y=0, y=L_F, Pa */
} orc_cond;

typedef struct {
  int32_t iterations, converged, status;
  double rel_residual;           /* recursive, Eq. 3.9 with r_j (R-A10) */
  double true_rel_residual;      /* ||S - A p|| / ||S|| at exit */
} orc_stats;

/* O2 texture mask T(i,j) in {0,1}; i in [0,n_theta), j in [-1,n_y] (ghost rows never textured). */
int  orc_texture_mask(const orc_grid* g, int32_t i, int32_t j);
/* Validate mesh and texture resolution; returns ORC_OK or an error code. */
int  orc_check_grid(const orc_grid* g);

/* O3/O4: h and dh/dt on rows j=-1..n_y (layout [(n_y+2)][n_theta], row r = j+1).
 * Either output may be NULL.  Returns ORC_E_NONPOSITIVE_THICKNESS if any h < h_min
 * (and writes the offending (i,j,h) to bad[3] if bad != NULL). */
int  orc_thickness(const orc_grid* g, const orc_cond* c, double* h, double* hdot, double* bad);

/* O5: bands A_P, A_E, A_N and source S, each [n_y][n_theta]. */
int  orc_assemble(const orc_grid* g, const orc_cond* c, double* AP, double* AE, double* AN, double* S);

/* y = A x for one condition's bands (Eq. 2.4 with the wrap of Eq. 2.7). */
void orc_spmv(int32_t nt, int32_t ny, const double* AP, const double* AE, const double* AN,
              const double* x, double* y);

/* z = M^{-1} r for one condition: precond NONE / JACOBI / ASSOR2 (two-step, O6) / ASSOR1 /
 * SSOR (exact triangular solves, Eq. 2.9 at omega = 1). */
void orc_precond_apply(int32_t nt, int32_t ny, const double* AP, const double* AE, const double* AN,
                       int32_t precond, double omega, const double* r, double* z);

/* Eq. 3.4 as a dense n x n matrix (row-major), n = nt*ny <= 4096, for algebra pins. */
int  orc_assor2_dense(int32_t nt, int32_t ny, const double* AP, const double* AE, const double* AN,
                      double omega, double* Minv);
/* Expand the DIA bands to a dense row-major matrix (O9). n <= 4096. */
int  orc_expand_dense(int32_t nt, int32_t ny, const double* AP, const double* AE, const double* AN,
                      double* A);
/* Dense Cholesky solve A x = b (A SPD, row-major, overwritten by its factor).  Returns
 * ORC_E_BREAKDOWN if a pivot is <= 0. */
int  orc_cholesky_solve(int32_t n, double* A, const double* b, double* x);

/* O7: PCG (Table 1, sign fixed R-A9) on the joint block-diagonal system of K conditions
 * (Eq. 3.7), bands/vectors laid out [K][n_y][n_theta] (Eq. 3.8, block offset k*n).
 * coupling = ORC_COUPLED (global alpha/beta) or ORC_LOCKSTEP (per-k alpha_k/beta_k);
 * both stop on the global test of Eq. 3.9.  p is in/out (warm start if warm != 0,
 * else zeroed).  history (optional, length max_iter+1) receives ||r_j||/||S_G||.
 * cond_rel (optional, K) receives per-condition ||r_k||/||S_k|| at exit. */
int  orc_pcg_joint(int32_t nt, int32_t ny, int32_t K,
                   const double* AP, const double* AE, const double* AN, const double* S,
                   double* p, double tol, double omega, int32_t precond, int32_t coupling,
                   int32_t max_iter, int32_t warm, orc_stats* st, double* history, double* cond_rel);

/* O7-S3: Table 1 with one global reduction per iteration (Chronopoulos-Gear alpha
 * recurrence); same arguments as orc_pcg_joint.  This is the schedule
 * the single-pass GPU kernel follows, so iterates can be compared step by step.  Its alpha
 * denominator delta' - beta gamma'/alpha (> 0 in exact arithmetic) can lose its sign to
 * cancellation on a stagnating direction; the iteration then restarts along z (beta = 0,
 * alpha = gamma'/delta', an exact line search) instead of failing (DESIGN.md R-A32). */
int  orc_pcg_joint_sr(int32_t nt, int32_t ny, int32_t K,
                      const double* AP, const double* AE, const double* AN, const double* S,
                      double* p, double tol, double omega, int32_t precond, int32_t coupling,
                      int32_t max_iter, int32_t warm, orc_stats* st, double* history, double* cond_rel);

/* Test hook of the R-A32 restart branch (see gmaf_oracle.c): restart when den <= thresh * delta'
 * (default 0 = the method); orc_sr_restarts() = restarts taken by the last orc_pcg_joint_sr. */
void orc_sr_set_restart_threshold(double thresh);
int32_t orc_sr_restarts(void);

/* Asynchronous strategy (Eq. 3.10, NEXT-2): per-block PCG, block frozen once
 * ||r_k||/||S_k|| <= tol.  iters_k (K) receives per-block iteration counts. */
int  orc_pcg_async(int32_t nt, int32_t ny, int32_t K,
                   const double* AP, const double* AE, const double* AN, const double* S,
                   double* p, double tol, double omega, int32_t precond, int32_t max_iter,
                   int32_t* iters_k, orc_stats* st);

/* O8: force/moment of the oil film on the piston for one condition.
 * p: [n_y][n_theta] interior pressure.  w[12] = Fp_xyz, Mp_xyz, Fs_xyz, Ms_xyz. */
int  orc_wrench(const orc_grid* g, const orc_cond* c, const double* p, double* w);

#ifdef __cplusplus
}
#endif
#endif
