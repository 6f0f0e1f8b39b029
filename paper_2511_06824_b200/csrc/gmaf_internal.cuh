// gmaf_internal.cuh -- device-side data structures and kernel launchers of libgmaf.
// Not part of the ABI (see include/gmaf.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gmaf {

// Per-condition parameters.  Every derived scalar is computed on the host with the
// same IEEE operations, in the same order, as the thickness/assembly definition
// (DESIGN.md sec. 5), so that device thickness and bands are bitwise reproducible.
struct CondParams {
  double e[4], edot[4];
  double LF, Ut, Uy, pin, pout;
  double dy;      // L_F / (n_y + 1)
  double dx;      // R_k * dtheta
  double rx, ry;  // dy/dx, dx/dy
  double sl, tl;  // (e3-e1)/L_F, (e4-e2)/L_F
  double sld, tld;// (edot3-edot1)/L_F, (edot4-edot2)/L_F
  int32_t mat;    // index of the distinct coefficient set used by this condition
  int32_t pad;
};

struct GridParams {
  int32_t nt, ny;
  double Rk, Rc, mu, hmin, twelve_mu, dtheta;
  int32_t tex_nt, tex_ny, tex_band, tex_num, tex_den;
  double tex_depth;
  // Row slab of this context.  The fields of condition (or coefficient set)
  // k hold the stored rows [yb, yb + ns/nt) -- the owned rows [y0, y1) plus up to SLAB_HALO
  // halo rows on each side -- and are addressed with GLOBAL row indices through fofs().  One
  // rank: y0 = yb = 0, y1 = ny, ns = nt*ny.
  int32_t y0, y1, yb;
  int32_t diag;     // 1: the persistent kernel records per-CTA grid-barrier arrival times (gmaf_cta_arrivals)
  long long ns;
};

constexpr int SLAB_HALO = 4;
constexpr int kDiagIters = 32;   // iterations whose per-CTA arrival times are recorded (diag mode)
constexpr int kMaxTilesPerCondition = 148 * 16;   // partials region: 4 K kMaxTilesPerCondition doubles
// diag mode: the arrival stamps occupy the END of the partials region (the per-launch, persistent
// and true-residual partial sums use its beginning)
__host__ __device__ __forceinline__ long long diag_offset(int K, int nblk) {
  return (long long)4 * K * kMaxTilesPerCondition - (long long)kDiagIters * nblk;
}   // halo rows per side: the y dependency radius of A M^-1 A M^-1

// Offset of (condition k, global row 0, column 0) in a [K][stored rows][nt] field.
__host__ __device__ __forceinline__ long long fofs(const GridParams& g, int k) {
  return (long long)k * g.ns - (long long)g.yb * g.nt;
}

// Kernel kinds for the in-kernel %globaltimer accounting.
enum KernelKind { KK_THICK = 0, KK_ASSEMBLE, KK_INIT, KK_PHASE_A, KK_PHASE_B, KK_TRUERES, KK_QUAD,
                  KK_SR_INIT, KK_SR_ITER,
                  KK_SR_TAIL,   // serial tail of k_sr ITER (last CTA: reduction + scalar stage), inside KK_SR_ITER;
                                // persistent k_srp: grid barrier complete -> scalars ready (CTA 0)
                  KK_SR_WAIT,   // persistent k_srp: CTA 0's arrival at the grid barrier -> barrier complete
                  KK_COUNT };

struct Timing {
  unsigned long long t_start[KK_COUNT];   // min start of the current launch (ULLONG_MAX = idle)
  unsigned long long total_ns[KK_COUNT];
  unsigned long long launches[KK_COUNT];
};

// Solver state resident on the device.  The host writes the parameter block before a
// graph launch; kernels update the rest; the host reads it back after the solve.
struct SolverState {
  // parameters
  double tol, omega;
  int32_t coupling, max_iter, fixed_iters, pad0;
  // global scalars
  double d;           // coupled: sum_k r.z
  double nS;          // ||S_G||
  double rel;         // recursive ||r||/||S_G||
  double true_rel;
  int32_t iter, done, converged, status;
  int32_t zero_p, pad1, pad2, pad3;
};

// Per-condition scalar arrays (length K each) carved next to SolverState.
struct CondScalars {
  double* alpha;   // [K]
  double* beta;    // [K]
  double* dk;      // [K] r_k.z_k
  double* Sk;      // [K] S_k.S_k
  double* rrk;     // [K] r_k.r_k
  double* uvk;     // [K]
  double* ttk;     // [K] true residual^2
  int32_t* itk;    // [K] iterations of condition k (asynchronous strategy, Eq. 3.10)
  int32_t* frz;    // [K] 1 once condition k met its own test (asynchronous strategy)
};

// Multi-rank state (world > 0 only for a condition-sharded context).
constexpr int kMaxP2P = 8;                 // ranks of one node in peer-to-peer mode
struct DistPtrs {
  int32_t world, rank, kofs, kmax_local;   // ranks own contiguous condition blocks
  double* packed_local;                    // [4][kmax_local] this rank's per-condition sums
  double* packed_all;                      // [world][4][kmax_local] after the allgather
  // peer-to-peer mode (no NCCL): every rank owns one exchange buffer, IPC-mapped by all ranks,
  // layout [2*world flags u64][2*world*xs doubles]; the gathers run inside the kernels
  int32_t p2p, xs, kglob, pad;
  char* peer[kMaxP2P];                     // exchange buffer of rank r (peer[rank] = own)
  unsigned long long* seq;                 // gathers issued so far (the same sequence on every rank)
  double* rr_all;                          // [kglob] r.r_k of every condition (last iteration)
  double* ss_all;                          // [kglob] S.S_k of every condition (init)
  // row-slab mode (every rank holds all K conditions, rows [y0, y1)): halo inboxes in the own
  // exchange buffer, [2 slots][2 sides][2 vectors][K][SLAB_HALO rows][nt]; side 0 = the rows
  // below y0 (written by rank-1), side 1 = the rows from y1 up (written by rank+1).  Slot = parity
  // of the gather stamp that published them.
  int32_t rows, pad2;
  double* halo_in[kMaxP2P];                // inbox of rank r (halo_in[rank] = own)
};

// Inbox element (slot, side, vector, condition k, halo row ri, column 0).
__host__ __device__ __forceinline__ long long halo_ofs(int slot, int side, int vec, int K, int k, int ri, int nt) {
  return ((((long long)(slot * 2 + side) * 2 + vec) * K + k) * SLAB_HALO + ri) * nt;
}

struct DevPtrs {
  const double* ct; const double* st;      // cos/sin(i dtheta)
  const double* cth; const double* sth;    // cos/sin((i+1/2) dtheta)
  const CondParams* cp;                    // [K]
  double* AP; double* AE; double* AN;      // [M][n]
  double* S; double* p;                    // [K][n]
  double* r[2]; double* u[2];              // [K][n] ping-pong (halo reads never race with writes)
  double* scratch;                         // [(n_y+2) n_theta] field readback
  const double* zero_row; const double* one_row;  // constant rows: TMA sources for out-of-range rows
  double* partials;                        // [4][K][n_cta_max]
  double* wrench_part;                     // [K][n_cta_q][12]
  double* wrench;                          // [K][12]
  SolverState* st_;
  CondScalars cs;
  unsigned int* counters;                  // [8] last-CTA counters
  Timing* timing;
  unsigned long long* guard;               // [4]: flag, k, i|j, h bits
  int32_t* mat_rep;                        // [M] representative condition of each matrix
  DistPtrs dist;
};

// Marching-tile configuration of the PCG kernels.
struct TileCfg {
  int32_t tw;        // output columns per strip (threads = tw + 2*HALO)
  int32_t th;        // output rows per chunk
  int32_t n_strips, n_chunks, n_tiles;  // tiles per condition
};

constexpr int HALO = 3;   // theta halo columns on each side (ASSOR-II + SpMV + seam)

// ---- launchers (geometry.cu) ----
cudaError_t launch_thickness_guard(const GridParams& g, const DevPtrs& d, int K, cudaStream_t s);
cudaError_t launch_assemble(const GridParams& g, const DevPtrs& d, int K, cudaStream_t s);
cudaError_t launch_field(const GridParams& g, const DevPtrs& d, int field, int k, cudaStream_t s);
cudaError_t launch_quadrature(const GridParams& g, const DevPtrs& d, int K, cudaStream_t s,
                              int* n_cta_out);

// ---- launchers (pcg.cu) ----
// precond: 0 none, 1 jacobi, 2 assor2.  cond_handle: graph conditional handle or 0.
cudaError_t launch_init(const GridParams& g, const DevPtrs& d, const TileCfg& t, int K, int precond,
                        bool warm, unsigned long long cond_handle, cudaStream_t s);
// parity = iteration index mod 2: phase A reads u[1-parity], writes u[parity], reads r[parity];
// phase B reads u[parity], r[parity] and writes r[1-parity].
cudaError_t launch_phase_a(const GridParams& g, const DevPtrs& d, const TileCfg& t, int K,
                           int precond, int parity, unsigned long long cond_handle, cudaStream_t s);
cudaError_t launch_phase_b(const GridParams& g, const DevPtrs& d, const TileCfg& t, int K,
                           int precond, int parity, unsigned long long cond_handle, cudaStream_t s);
cudaError_t launch_true_residual(const GridParams& g, const DevPtrs& d, const TileCfg& t, int K,
                                 cudaStream_t s);
// warm-start pre-pass: r0 = S - A p0 into r[out_parity] (no preconditioner, no graph condition)
cudaError_t launch_residual_init(const GridParams& g, const DevPtrs& d, const TileCfg& t, int K, int out_parity,
                                 cudaStream_t s);

cudaError_t launch_true_scalar(const DevPtrs& d, int world, cudaStream_t s);

// ---- launchers (sr.cu): single-pass schedule, one kernel + one reduction per iteration ----
constexpr int SR_HALO_COLS = 4;
cudaError_t launch_sr_init(const GridParams& g, const DevPtrs& d, const TileCfg& t, int K, int precond,
                           bool warm, unsigned long long cond_handle, cudaStream_t s);
cudaError_t launch_sr_iter(const GridParams& g, const DevPtrs& d, const TileCfg& t, int K, int precond,
                           int parity, unsigned long long cond_handle, cudaStream_t s);
cudaError_t launch_sr_fixup(const GridParams& g, const DevPtrs& d, int K, cudaStream_t s);
// multi-rank: scalars from the gathered per-condition sums (one CTA)
cudaError_t launch_sr_scalar(const DevPtrs& d, bool init, int Kglob, int Klocal, int kofs, int world,
                             cudaStream_t s);
cudaError_t configure_sr_kernels(const TileCfg& t, int K);
int sr_ctas_per_sm(const TileCfg& t);
// persistent single-pass solve (one rank): every iteration in one cooperative launch with a grid
// barrier per iteration and the scalar stage evaluated redundantly in every CTA (sr.cu k_srp)
cudaError_t launch_sr_persistent(const GridParams& g, const DevPtrs& d, const TileCfg& t, int K, int precond,
                                 cudaStream_t s);
int srp_ctas_per_sm(const TileCfg& t, int K, int Kall);
bool srp_fits(const TileCfg& t, int K, int Kall);
// peer-to-peer mode: gather n doubles per rank from src into packed_all-style dst [world][n]
// (one thread; a timeout marks the solve failed, GMAF_E_CUDA)
cudaError_t launch_p2p_gather(const DevPtrs& d, const double* src, int n, double* dst, cudaStream_t s);
// peer-to-peer mode: gather of the packed per-condition sums + the scalar stage (Eq. 3.9, alpha,
// beta) + the graph WHILE condition, one CTA, after every init / iteration kernel
cudaError_t launch_p2p_scalar(const DevPtrs& d, bool init, int Klocal, unsigned long long h, cudaStream_t s);
// row-slab mode: after every init / iteration kernel, push the boundary rows
// of (r_{i+1}, pd_i) into the neighbours' inboxes + gather the per-condition sums, summed over
// the ranks in rank order, + the scalar stage (multi-CTA; the last CTA gathers)
cudaError_t launch_p2p_rows(const GridParams& g, const DevPtrs& d, bool init, int parity, int K,
                            unsigned long long h, cudaStream_t s);
// row-slab mode: one-off exchange of field v's halo rows (push, stamp-only gather, unpack)
cudaError_t launch_slab_exchange(const GridParams& g, const DevPtrs& d, double* v, int K, cudaStream_t s);
// row-slab mode with DistPtrs.rows == 2: unpack an iteration's halo vectors into the fields
cudaError_t launch_slab_unpack2(const GridParams& g, const DevPtrs& d, bool init, int parity, int K,
                                cudaStream_t s);

// ---- host accessors (gmaf_api.cu) for the Picard driver (picard.cu) ----
}  // namespace gmaf
struct gmaf_ctx;
namespace gmaf {
int ctx_conditions(const gmaf_ctx* c);
int ctx_world(const gmaf_ctx* c);
}  // namespace gmaf
