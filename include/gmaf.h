/*
 * gmaf.h -- C ABI of libgmaf, the B200-native (sm_100a) hot path of GMAF
 * (arXiv 2511.06824): the joint multi-working-condition pressure solve of one
 * Picard step.
 *
 *   gmaf_thickness  -> film thickness h(e) and rate dh/dt (Eq. 2.3, PAPER.md:45;
 *                      Eq. 2.2), h_min guard
 *   gmaf_assemble   -> FVM 5-point Reynolds system A_k p_k = S_k for K conditions
 *                      (Eqs. 2.4-2.7), symmetric DIA bands A_P, A_E, A_N
 *   gmaf_solve      -> PCG (Table 1; sign of r0 fixed, DESIGN.md R-A9) with the
 *                      ASSOR-II preconditioner (Eqs. 3.4-3.6) on the joint
 *                      block-diagonal system (Eq. 3.7) under the synchronized
 *                      global convergence test (Eq. 3.9)
 *   gmaf_integrate  -> force and moment of the oil film from normal pressure and
 *                      viscous shear for every condition (Sec. 2.4-III)
 *
 * Conventions (all entry points):
 *  - Every call returns a gmaf_status: 0 = OK, < 0 = error.  No C++ exception
 *    or abort crosses the ABI.  gmaf_last_error(ctx) gives a one-line reason.
 *  - Host pointers are caller-owned and only read/written during the call.
 *  - The caller owns the DEVICE workspace (e.g. a torch uint8 CUDA tensor of
 *    gmaf_workspace_bytes() bytes); it must outlive the context.  The library
 *    owns its CUDA graphs, events and pinned staging buffers.
 *  - All device work is enqueued on the caller's stream given at create.
 *    gmaf_thickness, gmaf_solve, gmaf_integrate and gmaf_get synchronize that
 *    stream before returning (they return host data); gmaf_assemble does not.
 *  - Call order: thickness -> assemble -> solve -> integrate; otherwise
 *    GMAF_E_STATE.  A new gmaf_thickness restarts the sequence (warm start
 *    reuses p from the previous solve).
 *  - One context per host thread.  FP64 throughout.
 *  - Device layout of every field: [K][n_y][n_theta], theta contiguous, global
 *    index i + n_theta*j + n*k with n = n_theta*n_y (Eq. 3.8).
 */
#ifndef GMAF_H
#define GMAF_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GMAF_OK = 0,
  GMAF_E_INVALID_ARG = -1,
  GMAF_E_INVALID_MESH = -2,          /* n_theta < 4 or n_y < 4, or (n_y + 16) n_theta >= 2^31 (32-bit row offsets) */
  GMAF_E_MESH_TOO_COARSE = -3,       /* < 2 nodes per dimple pitch */
  GMAF_E_NONPOSITIVE_THICKNESS = -4, /* h < h_min somewhere */
  GMAF_E_BREAKDOWN = -5,             /* u.v <= 0 or r.z <= 0: not SPD */
  GMAF_E_NO_CONVERGENCE = -6,        /* max_iter reached; the last iterate is kept in p */
  GMAF_E_STATE = -7,                 /* call order violated */
  GMAF_E_WORKSPACE = -8,             /* workspace NULL, too small or misaligned (256 B) */
  GMAF_E_CUDA = -9,                  /* a CUDA runtime error; see gmaf_last_error */
  GMAF_E_NCCL = -10,                 /* a collective failed (world > 1) */
  GMAF_E_SINGULAR = -11              /* Picard driver: the 4x4 update system is singular */
} gmaf_status;

enum { GMAF_PRECOND_NONE = 0,
       GMAF_PRECOND_JACOBI = 1,   /* D^-1 (Eq. 2.8) */
       GMAF_PRECOND_ASSOR2 = 2,   /* two-step ASSOR-II (Eqs. 3.4-3.6), the paper's choice */
       GMAF_PRECOND_ASSOR1 = 3 }; /* diagonal ASSOR-I (Eq. 3.2); single-pass schedule only */
enum { GMAF_COUPLED = 0,   /* one Krylov process on A_G: global alpha, beta (Eq. 3.9) */
       GMAF_LOCKSTEP = 1,  /* per-condition alpha_k, beta_k, same global stop test (R-A11) */
       GMAF_ASYNC = 2      /* asynchronous strategy (Eq. 3.10): per-condition processes, each
                              frozen once ||r_k||/||S_k|| <= tol (its CTAs stop loading); single-pass
                              schedule, one rank */ };
enum { GMAF_FIELD_P = 0, GMAF_FIELD_H = 1, GMAF_FIELD_HDOT = 2, GMAF_FIELD_AP = 3,
       GMAF_FIELD_AE = 4, GMAF_FIELD_AN = 5, GMAF_FIELD_S = 6, GMAF_FIELD_R = 7 };
enum { GMAF_SHARD_CONDITIONS = 0,       /* condition blocks; NCCL allgather per iteration (needs an id) */
       GMAF_SHARD_CONDITIONS_P2P = 1,    /* condition blocks; gather fused into the kernel, peer memory */
       GMAF_SHARD_ROWS_P2P = 2 };        /* row slabs of all K conditions; halo rows + sums over peer
                                            memory (SURVEY 8(e) partitioning of C3); see gmaf_slab */
/* Iteration schedule: both run the Table-1 method to the same rtol.
 * SINGLE: one fused kernel and one global (gamma, delta, r.r) reduction per iteration
 *         (Chronopoulos-Gear alpha recurrence; needs an even n_theta) -- the default;
 * TABLE1: two fused kernels per iteration with Table 1's two reductions (u.v, then r.r/r.z). */
enum { GMAF_SCHEDULE_TABLE1 = 0, GMAF_SCHEDULE_SINGLE = 1 };

/* Mesh and texture, shared by all K conditions; copied at create. */
typedef struct {
  int32_t n_theta, n_y;          /* unknown nodes; theta periodic; Dirichlet ghost rows at y = 0 and
                                    y = L_F are not counted (DESIGN.md R-A3) */
  double  R_k, R_c;              /* piston and bore radius, m (Table 8) */
  double  mu;                    /* viscosity, Pa.s (not in the paper; R-A8) */
  double  h_min;                 /* thickness guard, m */
  int32_t tex_n_theta, tex_n_y;  /* dimple counts; 0,0 = smooth (Fig. 10: 60x10, 60x20) */
  int32_t tex_band_rows;         /* dimples occupy unknown rows [0, band) from y = 0 */
  int32_t tex_fill_num, tex_fill_den; /* dimple fraction of the pitch in each direction */
  double  tex_depth;             /* m (20e-6) */
} gmaf_grid;

/* One working condition (Eqs. 2.17-2.19 build the 9 of one Picard step). */
typedef struct {
  double e[4], edot[4];          /* eccentricity (m) and its rate (m/s) */
  double L_F;                    /* coupling length, m */
  double U_theta, U_y;           /* sliding velocity of the piston relative to the bore, m/s */
  double p_in, p_out;            /* Dirichlet pressures at y = 0 and y = L_F, Pa */
} gmaf_condition;

/* Multi-GPU description (condition sharding).  dist == NULL, or world == 1
 * with nccl_unique_id == NULL: a single-rank context that needs no NCCL at all.  Otherwise
 * the K conditions are sharded over the ranks in contiguous blocks (the first K % world ranks
 * own one more); every rank calls every entry point with the same arguments (all K
 * conditions to gmaf_thickness), and each solve iteration performs ONE ncclAllGather of the
 * packed per-condition sums so that Eq. 3.9 and alpha/beta are evaluated identically on all
 * ranks.  nccl_unique_id points at the 128-byte ncclUniqueId made by gmaf_nccl_unique_id on
 * rank 0 and broadcast by the caller (e.g. over torch.distributed); gmaf_create is then a
 * collective call.  Requires world <= K and the single-pass schedule (even n_theta >= 12).
 * gmaf_get / gmaf_field_ptr accept only this rank's conditions; gmaf_integrate returns all K. */
typedef struct {
  int32_t rank, world;
  const void* nccl_unique_id;
  int32_t shard;                 /* GMAF_SHARD_CONDITIONS (NCCL), GMAF_SHARD_CONDITIONS_P2P or
                                    GMAF_SHARD_ROWS_P2P (row slabs, see gmaf_slab); a
                                    world > 1 context without an NCCL id is peer to peer */
} gmaf_dist;

typedef struct {
  int32_t iterations;            /* number of alpha-updates (Table 1 step 4) */
  int32_t converged;             /* 1 if Eq. 3.9 was met */
  int32_t status;                /* gmaf_status of the solve */
  int32_t precond;
  int32_t schedule;              /* GMAF_SCHEDULE_* used */
  int32_t pad;
  double  rel_residual;          /* recursive ||r||/||S_G|| at exit (R-A10) */
  double  true_rel_residual;     /* ||S_G - A_G p_G|| / ||S_G|| at exit */
  double  solve_ms;              /* device time of the solve (CUDA events) */
} gmaf_solve_stats;

/* Per-kernel device time accumulated since create or the last reset, measured
 * inside the kernels with %globaltimer (first CTA start -> last CTA end). */
typedef struct {
  char    name[24];
  int64_t launches;
  double  total_ms;
  double  bytes_per_launch;      /* algorithmic DRAM bytes per launch */
} gmaf_kernel_timing;

typedef struct gmaf_ctx gmaf_ctx;

/* Device workspace bytes needed for this grid, K conditions and distribution.
 * Returns 0 on invalid arguments.  The coefficient bands are stored once per DISTINCT matrix
 * (conditions with bitwise-equal e and L_F share one: Eq. 2.3 has no e-dot, so the 9
 * conditions of Eqs. 2.17-2.19 need 5): gmaf_workspace_bytes sizes them for K, the worst case;
 * gmaf_workspace_bytes_m for at most max_matrices (<= 0 or > K: K).  gmaf_create derives the
 * capacity from ws_bytes, and gmaf_thickness fails with GMAF_E_WORKSPACE if the conditions need
 * more distinct sets than that. */
size_t gmaf_workspace_bytes(const gmaf_grid* grid, int32_t K, const gmaf_dist* dist);
size_t gmaf_workspace_bytes_m(const gmaf_grid* grid, int32_t K, int32_t max_matrices, const gmaf_dist* dist);

/* Create a context.  d_workspace: device pointer (256-byte aligned) of ws_bytes >=
 * gmaf_workspace_bytes(); cuda_stream: a cudaStream_t (NULL = legacy default stream).
 * dist may be NULL (world = 1).  Errors: INVALID_ARG, INVALID_MESH, MESH_TOO_COARSE,
 * WORKSPACE, CUDA, NCCL. */
gmaf_status gmaf_create(const gmaf_grid* grid, int32_t K, const gmaf_dist* dist,
                        void* d_workspace, size_t ws_bytes, void* cuda_stream, gmaf_ctx** out);
gmaf_status gmaf_destroy(gmaf_ctx* ctx);

/* Upload the K conditions (host array, all K on every rank) and check h >= h_min on
 * every node of rows -1..n_y (synchronous).  Error: NONPOSITIVE_THICKNESS (nothing
 * downstream may run until a valid call). */
gmaf_status gmaf_thickness(gmaf_ctx* ctx, const gmaf_condition* conds);

/* Assemble A_P, A_E, A_N (one set per distinct e, Eq. 2.3 has no e-dot) and S for all
 * K conditions, bitwise equal to the oracle's evaluation order.
 * Asynchronous. */
gmaf_status gmaf_assemble(gmaf_ctx* ctx);

/* Solve A_G p_G = S_G.  tol = epsilon_PCG of Eq. 3.9 (relative); omega in (0,2);
 * precond GMAF_PRECOND_*; coupling GMAF_COUPLED or GMAF_LOCKSTEP; max_iter >= 0;
 * warm_start != 0 starts from the current p (else p0 = 0).  out: host stats (may be
 * NULL); cond_rel_residual: host array of K (may be NULL) receiving ||r_k||/||S_k||.
 * Errors: BREAKDOWN, NO_CONVERGENCE (p holds the last iterate), STATE, CUDA, NCCL. */
gmaf_status gmaf_solve(gmaf_ctx* ctx, double tol, double omega, int32_t precond, int32_t coupling,
                       int32_t max_iter, int32_t warm_start, gmaf_solve_stats* out,
                       double* cond_rel_residual);

/* Force and moment for every condition: host wrench[K*12], per k
 * [Fp_x,Fp_y,Fp_z, Mp_x,Mp_y,Mp_z, Fs_x,Fs_y,Fs_z, Ms_x,Ms_y,Ms_z] in N and N.m, X along
 * theta = 0, Y along theta = 90 deg, Z along the piston axis from the bottom, moments
 * about the bottom centre (DESIGN.md R-A14). */
gmaf_status gmaf_integrate(gmaf_ctx* ctx, double* wrench);

/* Copy one field of condition k to host_out: P, S, R, AP, AE, AN are [n_y][n_theta];
 * H and HDOT are [n_y+2][n_theta] (rows -1..n_y). */
gmaf_status gmaf_get(gmaf_ctx* ctx, int32_t field, int32_t k, double* host_out);

/* Device pointer of a field of condition k (P, S, R, AP, AE, AN), for zero-copy use. */
gmaf_status gmaf_field_ptr(gmaf_ctx* ctx, int32_t field, int32_t k, void** dptr);

/* Kernel timing (see gmaf_kernel_timing); n = capacity of out; *count receives the
 * number of entries.  gmaf_reset_kernel_times zeroes the accumulators. */
gmaf_status gmaf_kernel_times(gmaf_ctx* ctx, gmaf_kernel_timing* out, int32_t n, int32_t* count);
gmaf_status gmaf_reset_kernel_times(gmaf_ctx* ctx);

/* Run n_iter PCG iterations unconditionally (no convergence test; throughput mode of
 * SURVEY 8(d)) after a solve's init; used by the benchmark.  Stats as gmaf_solve. */
gmaf_status gmaf_solve_fixed(gmaf_ctx* ctx, double omega, int32_t precond, int32_t n_iter,
                             gmaf_solve_stats* out);

/* Choose the iteration schedule for subsequent solves (GMAF_SCHEDULE_*).  SINGLE with an
 * odd n_theta returns INVALID_ARG. */
gmaf_status gmaf_set_schedule(gmaf_ctx* ctx, int32_t schedule);

/* Per-condition iteration counts of the last solve (host int32[K]): the freeze iteration of
 * each condition under GMAF_ASYNC, the common count otherwise. */
gmaf_status gmaf_cond_iterations(gmaf_ctx* ctx, int32_t* out);

/* ---------------------------------------------------------------------------------------
 * Picard driver (Sec. 2.3, Eqs. 2.10-2.22): the iteration the
 * 9 working conditions exist for.  The paper defines the iteration, not the loads: the
 * generalized forces F1..F4 (Eq. 2.11) and the external / inertial load models are
 * DESIGN.md readings R-A28..R-A31.  Host code around the device path: every pressure solve
 * and force integral runs in the kernels above.
 * ------------------------------------------------------------------------------------- */
enum { GMAF_PICARD_SIMPLIFIED = 0,   /* Eqs. 2.20-2.22: drop dF/de, backward difference for e */
       GMAF_PICARD_GENERAL = 1 };    /* Eq. 2.12 with both Jacobians + the same backward difference */

typedef struct {
  double m_k, m_G;    /* piston and slipper mass, kg (Table 8: 0.128, 0.0259) */
  double R_b;         /* cylinder-block pitch radius, m (Table 8: 4.05e-2) */
  double beta;        /* swashplate inclination, rad (Table 8: 10 deg) */
  double omega_s;     /* shaft speed, rad/s (Table 8: 600 rpm) */
  double R_k;         /* piston radius, m (the bottom face pi R_k^2 carries p_in) */
} gmaf_pump;

typedef struct {
  double F[4];                 /* total general force F_E + F_I + F_O at (e, edot) (Eqs. 2.10-2.11), N */
  double F_oil[4], F_ext[4], F_inertial[4];
  double J_e[16], J_edot[16];  /* row-major dF_i/de_j (Eq. 2.13) and dF_i/d(edot)_j (Eq. 2.14) */
  double e_next[4], edot_next[4];   /* the update (scheme) */
  double wrench[12];           /* oil-film wrench of the base condition (gmaf_integrate layout) */
  int32_t pcg_iterations;      /* of the joint solve */
  int32_t pad;
} gmaf_picard_iterate;

/* Generalized forces of one state (host only, no context): F_oil4 from an oil-film wrench
 * (gmaf_integrate layout, R-A28: rigid-body virtual work of the two axis points at y = 0 and
 * y = L_F), F_ext4 the swashplate reaction to p_in on the piston bottom (R-A29) and F_in4 the
 * inertial load (R-A30) at shaft angle phi (rad).  Any output may be NULL.  Errors: INVALID_ARG. */
gmaf_status gmaf_general_forces(const gmaf_pump* pump, const gmaf_condition* cond, double phi,
                                const double* wrench12, double* F_oil4, double* F_ext4, double* F_in4);

/* One Picard iteration on a context created with K = 9 (world 1): the 9 conditions of
 * Eqs. 2.17-2.19 around `state` (e = e^(k), edot = edot^(k), plus the load case), ONE joint
 * thickness -> assemble -> solve -> integrate, the 9 general forces, the finite-difference
 * Jacobians (Eqs. 2.13-2.14, steps de and dedot; Table 8: 1e-9 m, 1e-8 m/s) and the update
 * for time step dt (R-A31): SIMPLIFIED e' = e - dt J_edot^-1 F, edot' = edot - J_edot^-1 F
 * (Eqs. 2.21-2.22); GENERAL (dt J_e + J_edot) d = -F, edot' = edot + d, e' = e + dt d.
 * tol/omega/max_iter/warm_start as gmaf_solve (ASSOR-II, coupled).  Errors: those of the
 * device calls, SINGULAR, INVALID_ARG (K != 9, dt <= 0, unknown scheme). */
gmaf_status gmaf_picard_iteration(gmaf_ctx* ctx, const gmaf_pump* pump, const gmaf_condition* state,
                                  double phi, double dt, int32_t scheme, double de, double dedot,
                                  double tol, double omega, int32_t max_iter, int32_t warm_start,
                                  gmaf_picard_iterate* out);

/* One time step t_l -> t_l + dt of the Picard time march (Sec. 2.3): starts from
 * e = e_l + dt edot_l, edot = edot_l (so e - e_l = dt edot holds at every iterate) and
 * iterates gmaf_picard_iteration until ||F|| <= eps_dyn * max(||F_E||, 1 N) (R-A31) or
 * max_picard iterations.  state: in = (e_l, edot_l, load case of t_l + dt), out = the state
 * whose force met the test (or the last iterate).  n_picard, residual (||F|| / scale) and
 * pcg_iterations (summed) may be NULL.  Returns NO_CONVERGENCE if max_picard was reached. */
gmaf_status gmaf_picard_step(gmaf_ctx* ctx, const gmaf_pump* pump, gmaf_condition* state, double phi,
                             double dt, int32_t scheme, double de, double dedot, double eps_dyn,
                             int32_t max_picard, double tol, double omega, int32_t max_iter,
                             int32_t* n_picard, double* residual, int32_t* pcg_iterations);

/* Peer-to-peer condition sharding (no NCCL).  A context created with
 * dist.world > 1 and dist.nccl_unique_id == NULL owns a small device exchange buffer; every rank
 * exports its CUDA IPC handle (64 bytes) with gmaf_p2p_handle, the caller all-gathers the handles
 * in rank order (e.g. over torch.distributed) and passes the world*64 bytes to gmaf_p2p_connect
 * (before the first solve).  The per-iteration reduction then runs on the device inside the
 * solve's CUDA graph: after each iteration kernel one CTA pushes the rank's per-condition sums
 * into every rank's buffer over NVLink, waits for all ranks (a solve whose peer never arrives
 * fails with GMAF_E_CUDA after 10 s), evaluates Eq. 3.9 / alpha / beta in global condition order
 * and sets the graph's WHILE condition -- no NCCL, no host round trip.  Ranks of one node only
 * (<= 8), K <= 256.  Errors: STATE (not a peer-to-peer context / already connected), CUDA. */
gmaf_status gmaf_p2p_handle(gmaf_ctx* ctx, void* out);
gmaf_status gmaf_p2p_connect(gmaf_ctx* ctx, const void* handles);

/* Row-slab sharding (dist.shard = GMAF_SHARD_ROWS_P2P; SURVEY 8(e) "row slabs with NVLink halo
 * exchange").  The 5-point stencil is local in y (Eqs. 2.4-2.7), so the joint
 * system of all K conditions is split into contiguous blocks of unknown rows: rank r owns rows
 * [y0, y1) of every condition (the first n_y % world ranks one row more) and stores SLAB_HALO = 4
 * halo rows on each side -- the y dependency radius of one single-pass iteration (A M^-1 A M^-1).
 * Connection as for GMAF_SHARD_CONDITIONS_P2P (gmaf_p2p_handle / gmaf_p2p_connect).  Inside the
 * solve's CUDA graph, after every iteration kernel, a multi-CTA kernel stores the 4 boundary rows
 * of r and of the search direction straight into the neighbours' inboxes over NVLink and then
 * gathers every rank's per-condition sums (gamma_k, delta_k, r.r_k, S.S_k), summed in rank order
 * so the scalars of Eq. 3.9 are bitwise the same on all ranks; the next iteration kernel streams
 * its halo rows from the inbox.  The converged p is exchanged once more for the true residual and
 * the quadrature.  gmaf_integrate returns all K wrenches (per-rank cell sums added in rank order);
 * gmaf_get writes only the own rows [y0, y1) of host_out (n_theta*n_y doubles; other rows are not
 * touched) and gmaf_field_ptr points at row y0 of the own rows.  Requires world <= 8, K <= 256,
 * n_y >= 8*world, an even n_theta >= 12.  Reports this context's own rows (all rows at world 1).
 * Errors: INVALID_ARG (null pointer). */
gmaf_status gmaf_slab(const gmaf_ctx* ctx, int32_t* y0, int32_t* y1);

/* The row partition itself, without a context (no GPU needed): own rows [y0, y1) and stored rows
 * [yb, ye) (own rows + up to 4 halo rows per side inside the domain) of `rank` among `world`
 * slabs of n_y unknown rows.  Errors: INVALID_ARG (null pointer, world outside 1..8, rank outside
 * 0..world-1, or a slab thinner than 8 rows). */
gmaf_status gmaf_slab_rows(int32_t n_y, int32_t world, int32_t rank, int32_t* y0, int32_t* y1,
                           int32_t* yb, int32_t* ye);

/* Launch configuration of this context's iteration kernel, for tests and
 * the benchmark: strip width tw (output columns per CTA), rows per chunk th, strips and chunks
 * per condition, CTAs per launch (n_strips * n_chunks * K_local), the schedule that solves use
 * (GMAF_SCHEDULE_*) and whether the single-pass solve runs as ONE persistent launch (1: all
 * iterations in one cooperative kernel with a grid barrier per iteration; 0: one kernel per
 * iteration inside the CUDA graph's WHILE loop).  Errors: INVALID_ARG (null pointer). */
typedef struct {
  int32_t tw, th, n_strips, n_chunks, n_ctas, schedule, persistent, pad;
} gmaf_tiles;
gmaf_status gmaf_tile_config(const gmaf_ctx* ctx, gmaf_tiles* out);

/* Load-balance diagnostics of the persistent solve: with the environment variable GMAF_DIAG set at
 * gmaf_create, the persistent kernel records the %globaltimer (ns) at which each CTA arrives at
 * the grid barrier of each of the first 32 iterations of a solve; this copies them to out
 * (uint64 [iteration][CTA], CTA b = tile * K + condition, tile = chunk * n_strips + strip) and
 * sets *count (0 without GMAF_DIAG or without the persistent path).  Errors: INVALID_ARG. */
gmaf_status gmaf_cta_arrivals(gmaf_ctx* ctx, uint64_t* out, int32_t n, int32_t* count);

/* Make a new ncclUniqueId (128 bytes) into out (NCCL is loaded at run time).  Errors: NCCL. */
gmaf_status gmaf_nccl_unique_id(void* out);

const char* gmaf_last_error(const gmaf_ctx* ctx);
const char* gmaf_version(void);

#ifdef __cplusplus
}
#endif
#endif
