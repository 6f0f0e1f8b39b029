// sr.cu -- single-pass PCG-ASSOR-II iteration on sm_100a: ONE kernel and ONE global
// reduction per iteration (schedule "SINGLE").
//
// The method is Table 1 (sign of r0 fixed) with the ASSOR-II two-step
// preconditioner (Eqs. 3.5-3.6) on the joint system (Eq. 3.7) and the synchronized
// global test (Eq. 3.9).  Its scalars come from Chronopoulos & Gear's single-reduction
// recurrence (oracle orc_pcg_joint_sr):
//
//   pd_i    = z_i + beta_i pd_{i-1}            (Table 1 step 9)
//   s_i     = A pd_i                            (step 3, recomputed, not stored)
//   x      += alpha_i pd_i                      (step 4, applied two iterations at a time)
//   r_{i+1} = r_i - alpha_i s_i                 (step 5)
//   z_{i+1} = M^-1 r_{i+1}, w = A z_{i+1}       (step 7, recomputed from r, not stored)
//   gamma = r.z, delta = z.w, r.r  -> ONE fixed-order reduction -> test (step 6),
//   beta = gamma'/gamma, alpha = gamma'/(delta' - beta gamma'/alpha)   (step 8)
//
// HBM traffic per DOF and iteration: r (read+write), pd (read+write), x (read+write every
// other iteration) = 40 B, plus the 3 coefficient bands of the DISTINCT matrices (shared
// through L2 by the conditions with equal e).
//
// Tiling.  Strip s of a condition owns output columns [s*TW - TW/2, (s+1)*TW - TW/2) (mod
// n_theta: the periodic seam lies in the MIDDLE of strip 0, so no strip edge is within 6
// columns of it and a halo of HALO = 4 columns -- the dependency radius of A M^-1 A M^-1
// away from the seam -- suffices), one thread per column PAIR, marching over a chunk of
// rows.  Rows are streamed by the TMA engine (cp.async.bulk) from a dedicated producer
// warp: r, pd, x into a 4-slot ring (consumed in one step), A_P, A_E, A_N into an 8-slot
// ring (alive for 5 steps), one full mbarrier per step, empty mbarriers per ring.  Derived
// rows (w, v1, pd, w2, v2, z2) live in 2-slot shared rings for theta-neighbour reads;
// own-column history in registers.  The row loop is unrolled by 8 so every ring slot is a
// compile-time index.  Two compute-warp barriers per row.  Stage lags (rows behind the
// load row jl):
//   A(0) load, D^-1, w      B(0) v1 = (I - wD^-1L) w        C(1) z, pd
//   D(2) s = A pd, r, x, w2 E(2) v2                         F(3) z2, gamma
//   G(4) delta = z2' A z2 (quadratic form)
#include <cstdint>
#include <cstdlib>
#include "sr_common.cuh"

namespace gmaf {

constexpr int SR_HALO = 4;      // theta halo (columns) on each side (seam kept mid-strip)
constexpr int SR_YLO = 4;       // rows loaded below the chunk
constexpr int SR_YHI = 4;       // rows loaded above the chunk
constexpr int SR_LAG = 4;       // the delta stage trails the load by 4 rows
constexpr int SR_VSLOTS = 4;    // TMA ring of vector rows (r, pd, x), consumed in one step
constexpr int SR_CSLOTS = 8;    // TMA ring of coefficient rows (AP, AE, AN), alive 5 steps
constexpr int SR_UNROLL = 8;    // row-loop unroll = coefficient-ring period

__host__ __device__ inline size_t sr_smem_bytes(int nl) {
  // vector slots + coefficient slots + 6 derived rings (2 each) + mbarriers
  return (size_t)(SR_VSLOTS * 3 + SR_CSLOTS * 3 + 12) * nl * sizeof(double) +
         (SR_CSLOTS + SR_VSLOTS + SR_CSLOTS) * sizeof(uint64_t) + 64;
}

// Per-thread geometry of one (strip, row chunk, condition) tile, recomputed by each role.
struct SrGeo {
  int NTC, NCT, NL, tid, tl, k, i0, j0, j1, gl, gr, im, ip, jbase, nsteps, m;
  bool is_producer, out, seamL, seamR, seamWarp, lcoef;
  long long fk;
};

// TWC > 0: the strip width as a compile-time constant (= t.tw; the persistent single-rank kernel
// of the common widths): every shared-memory ring address is then a per-thread base plus an
// immediate, which frees the registers and integer instructions of the runtime carve-up.
template <int TWC = 0>
__device__ __forceinline__ SrGeo sr_geo(const GridParams& g, const DevPtrs& d, const TileCfg& t, int K) {
  SrGeo q;
  const int tw = TWC > 0 ? TWC : t.tw;
  // warps 0 .. NCT/32-1 compute (one thread per column pair); the last warp streams rows (TMA)
  q.NTC = tw / 2 + SR_HALO;               // column pairs
  q.NCT = (q.NTC + 31) & ~31;             // compute threads (whole warps; idle lanes alias the last pair)
  q.NL = 2 * q.NTC;                       // loaded columns = tw + 2*HALO
  q.tid = threadIdx.x;
  q.is_producer = q.tid >= q.NCT;
  q.tl = min(q.tid, q.NTC - 1);
  q.k = blockIdx.x % K;
  const int tile = blockIdx.x / K;
  const int strip = tile % t.n_strips, chunk = tile / t.n_strips;
  const int nt = g.nt;
  // strip s owns [s tw - soff, (s+1) tw - soff): the seam (column 0) lies at local column
  // soff + HALO of strip 0, >= 6 columns from both edges.  With 512-column strips it is placed in
  // compute warp 6 (pair 198): warps map to the SM sub-partitions round-robin, and sub-partition 0
  // already carries three compute warps (0, 4 and the halo warp 8) while 2 and 3 carry two -- the
  // seam warp's extra wrap terms go where there are spare issue slots
  // (a function of the width alone, compile-time or not: every kernel variant tiles a context
  // identically, so their per-CTA partial sums -- and hence their scalars -- are bitwise equal)
  const int soff = tw == 512 ? 392 : tw / 2;
  q.i0 = strip * tw - soff;                         // first output column (may be negative: mod nt)
  q.j0 = g.y0 + chunk * t.th;
  q.j1 = min(q.j0 + t.th, g.y1);                    // own rows [y0, y1)
  const int cl = 2 * q.tl;
  int gl = (q.i0 - SR_HALO + cl) % nt;
  if (gl < 0) gl += nt;
  q.gl = gl;
  q.gr = gl + 1;                           // gl is even and nt is even: the pair never wraps
  // output pair: inside [HALO, HALO + TW) and, for the last (ragged) strip, before strip 0's
  // start + nt, i.e. its output index counted from strip 0's start is < nt
  const int o = q.i0 + cl - SR_HALO + soff;         // output index counted from strip 0's start
  q.out = (q.tid < q.NTC) && (cl >= SR_HALO) && (cl < SR_HALO + tw) && (o < nt);
  // ASSOR split on the periodic ring (R-A12): only a pair holding column 0 on its left or
  // column nt-1 on its right sees the wraps; every other pair uses the plain formulas.
  q.seamL = (q.gl == 0);
  q.seamR = (q.gr == nt - 1);
  q.seamWarp = false;                      // set by the compute role (warp vote)
  q.im = max(cl - 1, 0);                   // scalar index of the left neighbour of the pair
  q.ip = min(cl + 2, q.NL - 1);            // scalar index of the right neighbour of the pair
  // the left neighbour's A_E comes by shuffle, except in lane 0 and in idle lanes (which must
  // reproduce the last real pair exactly, since they write the same ring slots)
  q.lcoef = (q.tid & 31) == 0 || q.tid >= q.NTC;
  q.fk = fofs(g, q.k);                     // field base of condition k (global row indexing)
  q.m = d.cp[q.k].mat;
  q.jbase = q.j0 - SR_YLO;
  // steps jl = jbase .. jbase + nsteps - 1; the real ones end at j1 + LAG - 1, the rest pad to
  // a whole number of unrolled blocks (their rows read as zero rows)
  q.nsteps = ((q.j1 + SR_LAG - q.jbase) + SR_UNROLL - 1) & ~(SR_UNROLL - 1);
  return q;
}

// Shared-memory carve-up of the single-pass kernels (NL doubles per row).
struct SrSmem {
  double *vstage, *cring, *ringW, *ringV, *ringP, *ringW2, *ringV2, *ringU2;
  uint32_t full0, emptyv0, emptyc0;
};
__device__ __forceinline__ SrSmem sr_smem(double* smem_raw, int NL) {
  SrSmem s;
  s.vstage = smem_raw;                               // [4][3][NL]  r, pd, x rows
  s.cring = s.vstage + SR_VSLOTS * 3 * NL;           // [8][3][NL]  AP, AE, AN rows
  s.ringW = s.cring + SR_CSLOTS * 3 * NL;            // [2][NL] each
  s.ringV = s.ringW + 2 * NL;
  s.ringP = s.ringV + 2 * NL;
  s.ringW2 = s.ringP + 2 * NL;
  s.ringV2 = s.ringW2 + 2 * NL;
  s.ringU2 = s.ringV2 + 2 * NL;
  uint64_t* bars = reinterpret_cast<uint64_t*>(s.ringU2 + 2 * NL);
  s.full0 = smem_addr(bars);                         // [8] one per step mod 8
  s.emptyv0 = s.full0 + 8 * SR_CSLOTS;               // [4]
  s.emptyc0 = s.emptyv0 + 8 * SR_VSLOTS;             // [8]
  return s;
}

__device__ __forceinline__ void sr_init_barriers(const SrGeo& q, const SrSmem& s) {
  if (q.tid == 0) {
    for (int b = 0; b < SR_CSLOTS; ++b) mbar_init(s.full0 + 8 * b, 1);
    for (int b = 0; b < SR_VSLOTS; ++b) mbar_init(s.emptyv0 + 8 * b, q.NCT / 32);
    for (int b = 0; b < SR_CSLOTS; ++b) mbar_init(s.emptyc0 + 8 * b, q.NCT / 32);
    mbar_fence_init();
  }
  for (int i = q.tid; i < 12 * q.NL; i += blockDim.x) s.ringW[i] = 0.0;
}

// ------------------------------------------------------------------ TMA producer warp
// Streams steps [s_lo, s_hi) of one tile pass.  gstep0 = steps this CTA streamed in earlier
// passes (a multiple of 8): the ring slots and mbarrier phases continue across the passes of the
// persistent kernel.  Lane a < 6 streams array a: 0 r, 1 pd_{i-1}, 2 x (or S), 3 AP, 4 AE, 5 AN.
template <int MODE>
__device__ __forceinline__ void sr_produce(const GridParams& g, const DevPtrs& d, const SrGeo& q,
                                           const SrSmem& s, int K, int parity, uint32_t gstep0, int s_lo,
                                           int s_hi, int islot_in = -1) {
  constexpr bool ITER = (MODE == SR_ITER_EVEN || MODE == SR_ITER_ODD);
  constexpr bool XUPD = (MODE == SR_ITER_ODD);
  constexpr bool USE_PD = ITER;
  constexpr bool USE_X = XUPD || (MODE == SR_INIT_WARM);
  const int nt = g.nt, ny = g.ny, NL = q.NL;
  const long long fk = q.fk;
  // ITER: r_i = R[parity], pd_{i-1} = PD[1-parity].  INIT: r_0 = S (cold) or R[1] (warm).
  const double* rin = ITER ? d.r[parity] + fk : (MODE == SR_INIT_COLD ? d.S + fk : d.r[1] + fk);
  const int lane = q.tid - q.NCT;
  const bool vec = lane < 3;
  const double* srcp = lane == 0 ? rin
                     : lane == 1 ? d.u[1 - parity] + fk
                     : lane == 2 ? ((MODE == SR_INIT_WARM) ? d.S + fk : d.p + fk)
                     : lane == 3 ? d.AP + fofs(g, q.m)
                     : lane == 4 ? d.AE + fofs(g, q.m)
                                 : d.AN + fofs(g, q.m);
  const double* constrow = lane == 3 ? d.one_row : d.zero_row;
  const bool used = lane < 6 && (lane != 1 || USE_PD) && (lane != 2 || USE_X);
  const int lag = lane == 1 ? 1 : (lane == 2 ? 2 : 0);
  const int j0 = q.j0, j1 = q.j1, jbase = q.jbase;
  int lo = jbase, hi = min(j1 + SR_YHI, ny);                         // rows really read
  if (lane == 1) { lo = j0 - SR_YLO + 1; hi = min(j1 + SR_YHI - 1, ny); }
  if (lane == 2) { lo = j0; hi = j1; }
  if (lo < 0) lo = 0;
  int g0 = (q.i0 - SR_HALO) % nt;
  if (g0 < 0) g0 += nt;
  const int len0 = min(NL, nt - g0);                  // first segment (the seam splits a row)
  const uint32_t bytes = (uint32_t)NL * 8u * (uint32_t)(4 + (USE_PD ? 1 : 0) + (USE_X ? 1 : 0));
  const uint32_t dst0 = smem_addr(vec ? s.vstage + lane * NL : s.cring + (lane - 3) * NL);
  const uint32_t dstride = (uint32_t)(3 * NL * 8);    // bytes between slots
  // row-slab mode: an iteration's r and pd rows outside the own slab come from the inbox the
  // neighbours pushed them into (slot = parity of the last gather stamp)
  const bool inbox = ITER && lane < 2 && d.dist.rows == 1;
  const double* ibase = inbox ? d.dist.halo_in[d.dist.rank] : nullptr;
  // (the persistent kernel passes the slot: its own gathers advance the stamp during the launch)
  const int islot = !inbox ? 0 : islot_in >= 0 ? islot_in : (int)(*d.dist.seq & 1ull);
  for (int step = s_lo; step < s_hi; ++step) {
    const uint32_t gs = gstep0 + (uint32_t)step;
    const int sv = (int)(gs & (SR_VSLOTS - 1)), sc = (int)(gs & (SR_CSLOTS - 1));
    if (gs >= SR_VSLOTS) mbar_wait_sleep(s.emptyv0 + 8 * sv, ((gs / SR_VSLOTS) - 1) & 1);
    if (gs >= SR_CSLOTS) mbar_wait_sleep(s.emptyc0 + 8 * sc, ((gs / SR_CSLOTS) - 1) & 1);
    const uint32_t bar = s.full0 + 8 * sc;
#ifdef GMAF_EXPERIMENT_NOTMA
    // timing-only experiment (wrong results): no row is streamed, the rings keep stale data
    if (lane == 0) mbar_arrive(bar);
    __syncwarp();
    if (false) {
#else
    if (lane == 0) mbar_arrive_expect_tx(bar, bytes);
    __syncwarp();
    if (used) {
#endif
      const int row = jbase + step - lag;
      const uint32_t dst = dst0 + (uint32_t)(vec ? sv : sc) * dstride;
      if (row >= lo && row < hi) {
        const double* rowp = srcp + (long long)row * nt;
        if (inbox && (row < g.y0 || row >= g.y1)) {
          const int side = row < g.y0 ? 0 : 1;
          rowp = ibase + halo_ofs(islot, side, lane, K, q.k, side ? row - g.y1 : row - (g.y0 - SLAB_HALO), nt);
        }
        bulk_g2s(dst, rowp + g0, (uint32_t)len0 * 8u, bar);
        int done = len0;
        while (done < NL) {                              // wrapped remainder (small n_theta loops)
          const int len = min(NL - done, nt);
          bulk_g2s(dst + (uint32_t)done * 8u, rowp, (uint32_t)len * 8u, bar);
          done += len;
        }
      } else {
        bulk_g2s(dst, constrow, (uint32_t)NL * 8u, bar);
      }
    }
  }
}

// -------------------------------------------------------------------- compute warps
// One pass of the 7-stage row pipeline over the tile (all nsteps steps).  Accumulates the
// per-thread gamma, delta, r.r and S.S partials into acc.
// SEAM selects how the row loop treats the periodic seam (the wrap terms of R-A12):
//   SEAM_NONE  -- no seam code (a warp without a seam pair, in the split variant);
//   SEAM_FIXED -- the warp holding the seam pairs: corrections as selects, no divergent branches;
//   SEAM_CHECK -- one loop for every warp, the seam warp branching into the corrections.
// All three evaluate the same expressions for every column, so results are bitwise identical: a
// seam column's L/U sums are formed directly from its own terms (as Eqs. 3.5-3.6 state them for
// the natural ordering), not as the plain sums plus and minus a correction.
enum { SEAM_NONE = 0, SEAM_FIXED = 1, SEAM_CHECK = 2 };

// Timing-only instrumentation (-DGMAF_STEP_PROBE, never in the product build; scripts/probe_steps.py):
// per CTA and warp, clock() sums of the row step's intervals [top -> TMA data ready -> before
// barrier 1 -> after it -> before barrier 2 -> after it -> next top], read with gmaf_debug_step_probe.
#ifdef GMAF_STEP_PROBE
__device__ unsigned int g_step_probe[2048 * 16 * 8];
#define STEP_PROBE(i) { const unsigned int tn_ = (unsigned int)clock(); pc_[i] += tn_ - tprev_; tprev_ = tn_; }
#else
#define STEP_PROBE(i)
#endif
template <int PC, int MODE, int SEAM, bool ROT>
__device__ __forceinline__ void sr_compute_loop(const GridParams& g, const DevPtrs& d, const SrGeo& q, const SrSmem& s,
                                           int parity, double alpha, double alpha_prev, double beta, double omega,
                                           uint32_t gstep0, double& acc_rr, double& acc_g, double& acc_d,
                                           double& acc_s) {
  constexpr bool ITER = (MODE == SR_ITER_EVEN || MODE == SR_ITER_ODD);
  constexpr bool XUPD = (MODE == SR_ITER_ODD);         // x += a_{i-1} pd_{i-1} + a_i pd_i
  constexpr bool USE_PD = ITER;                         // pd_{-1} = 0 is stored by the init
  constexpr bool USE_X = XUPD || (MODE == SR_INIT_WARM);  // a warm init streams S in the x slot
  const int nt = g.nt, NL = q.NL, NTC = q.NTC, NCT = q.NCT, tl = q.tl, im = q.im, ip = q.ip;
  const int j0 = q.j0, j1 = q.j1, jbase = q.jbase, gl = q.gl;
  const unsigned nown = (unsigned)(j1 - j0);             // own rows [j0, j1)
  const bool out = q.out, seamL = q.seamL, seamR = q.seamR, lcoef = q.lcoef;
  const bool seamWarp = SEAM == SEAM_FIXED ||
                        (SEAM == SEAM_CHECK && __any_sync(0xffffffffu, (q.seamL || q.seamR) && q.tid < NCT));

  // output pointers at this thread's column pair; a row offset is 32-bit (row * n_theta < 2^31,
  // checked at create), so every store address is one IMAD + one wide IMAD
  double* rout = (ITER ? d.r[1 - parity] : d.r[0]) + q.fk + gl;
  double* pdout = (ITER ? d.u[parity] : d.u[1]) + q.fk + gl;
  double* x = d.p + q.fk + gl;
  const double c2 = (2.0 - omega) * omega;
  const double romega = 1.0 / omega;
  const double* vstage = s.vstage;
  const double* cring = s.cring;

  // own-column history in registers (suffix = lag in rows behind the load row);
  // coefficient rows are read from the 8-slot ring at their lag
  D2 oD1{0, 0}, oD2{0, 0}, oD3{0, 0};
  D2 r1{0, 0}, r2{0, 0}, pdo2{0, 0}, pd2{0, 0}, pd3{0, 0}, rn3{0, 0}, u2_4{0, 0};
  // ROT: coefficient rows past their first use stay in registers (rotated like the vector history):
  // A_E of rows jl-1..jl-4, A_N of rows jl-2..jl-4 and the left neighbour's A_E of rows jl-1,
  // jl-2 -- each shared-memory coefficient row is then read once per step (A_P at lags 2 and 4
  // excepted), which takes 7 of the 12 coefficient loads (28 of ~118 shared wavefronts per warp
  // and row) off the shared-memory pipe.  Needs the registers the compile-time strip width frees
  // (TWC > 0); the runtime-width kernels re-read the rows from the ring instead.
  D2 cE1{0, 0}, cE2{0, 0}, cE3{0, 0}, cE4{0, 0}, cN2{0, 0}, cN3{0, 0}, cN4{0, 0};
  double cE1m = 0.0, cE2m = 0.0;
  const bool lane0 = (q.tid & 31) == 0;
#ifdef GMAF_STEP_PROBE
  unsigned int pc_[6] = {0, 0, 0, 0, 0, 0};
  unsigned int tprev_ = (unsigned int)clock();
#endif
  for (int blk = 0; blk < q.nsteps; blk += SR_UNROLL) {
    const uint32_t gblk = gstep0 + (uint32_t)blk;
    const uint32_t cpar = (gblk / SR_UNROLL) & 1u;                   // phase of the per-step barriers
#pragma unroll
    for (int u = 0; u < SR_UNROLL; ++u) {
      const int jl = jbase + blk + u;
      const int sv = u & (SR_VSLOTS - 1);
      // coefficient rows at lag L live in slot (u - L) & 7; arrays AP=0, AE=1, AN=2
      const double* c0 = cring + (((u + 8) & 7) * 3) * NL;
      const double* c1 = cring + (((u + 7) & 7) * 3) * NL;
      const double* c2r = cring + (((u + 6) & 7) * 3) * NL;
      const double* c3 = cring + (((u + 5) & 7) * 3) * NL;
      const double* c4 = cring + (((u + 4) & 7) * 3) * NL;
      double* w_0 = s.ringW + (u & 1) * NL;
      const double* w_1 = s.ringW + ((u + 1) & 1) * NL;
      double* v_0 = s.ringV + (u & 1) * NL;
      const double* v_1 = s.ringV + ((u + 1) & 1) * NL;
      double* p_1 = s.ringP + ((u + 1) & 1) * NL;
      const double* p_2 = s.ringP + (u & 1) * NL;
      double* w2_2 = s.ringW2 + (u & 1) * NL;
      const double* w2_3 = s.ringW2 + ((u + 1) & 1) * NL;
      double* v2_2 = s.ringV2 + (u & 1) * NL;
      const double* v2_3 = s.ringV2 + ((u + 1) & 1) * NL;
      double* u2_3r = s.ringU2 + ((u + 1) & 1) * NL;
      const double* u2_4r = s.ringU2 + (u & 1) * NL;

      // ---- (A) row jl: streamed data, D^-1, w = D^-1 r
      STEP_PROBE(5);
      mbar_wait(s.full0 + 8 * u, cpar);
      STEP_PROBE(0);
      const double* vs = vstage + sv * 3 * NL;
      const D2 r0 = ld2(vs, tl);
      const D2 pdo1 = USE_PD ? ld2(vs + NL, tl) : D2{0, 0};
      const D2 x2 = USE_X ? ld2(vs + 2 * NL, tl) : D2{0, 0};
      __syncwarp();
      if (lane0) mbar_arrive(s.emptyv0 + 8 * sv);            // this warp is done with vector slot sv
      const D2 AP0 = ld2(c0, tl);
      const D2 AE0 = ld2(c0 + NL, tl);
      const D2 AN1 = ld2(c1 + 2 * NL, tl);
      const D2 w1 = rld(w_1, tl, NTC);
      const double ae0m = left_of(AE0.r, c0 + NL, im, lcoef);   // A_E(jl) left of the pair
      D2 iD0{fast_rcp(AP0.l), fast_rcp(AP0.r)};
      if constexpr (PC == SPC_ASSOR1) {
        // ASSOR-I (Eq. 3.2): the preconditioner is the diagonal c / Dt with
        // Dt_i = D_i + omega^2 sum_{k in L(i)} L_ik^2 / D_k, L = {W, E-wrap at n_theta-1, S}
        // (R-A12); it enters the pipeline exactly like Jacobi's D^-1
        const D2 AP1 = ld2(c1, tl);
        const double apl = left_of(AP0.r, c0, im, lcoef), ael = ae0m;
        double sl = dmul(dmul(ael, ael), fast_rcp(apl));
        double sr = dmul(dmul(AE0.l, AE0.l), iD0.l);
        if (SEAM != SEAM_NONE && seamWarp) {
          if (seamL) sl = 0.0;                                           // column 0: no W in L
          if (seamR) sr = dadd(sr, dmul(dmul(AE0.r, AE0.r), fast_rcp(c0[ip])));   // column nt-1: E-wrap
        }
        sl = dadd(sl, dmul(dmul(AN1.l, AN1.l), fast_rcp(AP1.l)));
        sr = dadd(sr, dmul(dmul(AN1.r, AN1.r), fast_rcp(AP1.r)));
        const double o2 = dmul(omega, omega);
        iD0 = {dmul(c2, fast_rcp(fma(o2, sl, AP0.l))), dmul(c2, fast_rcp(fma(o2, sr, AP0.r)))};
      }
      const D2 oD0{dmul(omega, iD0.l), dmul(omega, iD0.r)};
      D2 w0;
      if constexpr (PC == SPC_NONE) w0 = r0; else w0 = {dmul(r0.l, iD0.l), dmul(r0.r, iD0.r)};
      rst(w_0, tl, NTC, w0);
      STEP_PROBE(1);
      row_bar<SEAM != SEAM_CHECK>(NCT);                                         // barrier 1: w(jl) complete
      STEP_PROBE(2);

      // ---- (B) v1(jl) = w - (omega/D) sum_L A w  (Eq. 3.5);  (C) z(jl-1), pd(jl-1)
      D2 z1;
      if constexpr (PC == SPC_ASSOR2) {
        const double w0m = rleft(w_0, tl, NTC);
        const D2 v11 = rld(v_1, tl, NTC);
        const double v1p = rright(v_1, tl);
        const D2 AEm1 = ROT ? cE1 : ld2(c1 + NL, tl);
        // the seam warp (which paces its CTA at every row barrier, and the seam strip the grid)
        // loads its wrap operands together with the plain ones and applies them as selects
        double wE = 0.0, aW = 0.0, vW = 0.0;
        if constexpr (SEAM == SEAM_FIXED) {
          wE = rright(w_0, tl);                                 // w(jl) right of the pair (column 0 for nt-1)
          aW = c1[NL + im];                                     // A_E(jl-1) left of the pair (nt-1 for column 0)
          vW = rleft(v_1, tl, NTC);                             // v1(jl-1) left of the pair
        }
        // plain pair: L = {W, S}, U = {E, N}
        D2 sL{fma(ae0m, w0m, dmul(AN1.l, w1.l)), fma(AE0.l, w0.l, dmul(AN1.r, w1.r))};
        if constexpr (SEAM == SEAM_FIXED) {
          sL.l = seamL ? dmul(AN1.l, w1.l) : sL.l;              // column 0: W is the wrap (in U)
          sL.r = seamR ? fma(AE0.r, wE, sL.r) : sL.r;           // column nt-1: E-wrap is in L
        } else if (SEAM == SEAM_CHECK && seamWarp) {
          if (seamL) sL.l = dmul(AN1.l, w1.l);                  // column 0: W is the wrap (in U)
          if (seamR) sL.r = fma(AE0.r, rright(w_0, tl), sL.r);  // column nt-1: E-wrap is in L
        }
        const D2 v10{fma(-oD0.l, sL.l, w0.l), fma(-oD0.r, sL.r, w0.r)};
        rst(v_0, tl, NTC, v10);
        D2 sU{fma(AN1.l, v10.l, dmul(AEm1.l, v11.r)), fma(AN1.r, v10.r, dmul(AEm1.r, v1p))};
        if constexpr (SEAM == SEAM_FIXED) {
          sU.l = seamL ? fma(aW, vW, sU.l) : sU.l;              // column 0: the W-wrap is in U
          sU.r = seamR ? dmul(AN1.r, v10.r) : sU.r;             // column nt-1: no E in U
        } else if (SEAM == SEAM_CHECK && seamWarp) {
          if (seamL) sU.l = fma(c1[NL + im], rleft(v_1, tl, NTC), sU.l);   // column 0: the W-wrap is in U
          if (seamR) sU.r = dmul(AN1.r, v10.r);                 // column nt-1: no E in U
        }
        z1 = {dmul(c2, fma(-oD1.l, sU.l, v11.l)), dmul(c2, fma(-oD1.r, sU.r, v11.r))};
      } else {
        z1 = w1;                                            // D^-1 r (Jacobi) or r (none)
      }
      const D2 pd1 = USE_PD ? D2{fma(beta, pdo1.l, z1.l), fma(beta, pdo1.r, z1.r)} : z1;   // step 9
      rst(p_1, tl, NTC, pd1);
      // row jl-k is stored / summed only if the pair is an output pair and the row is one of the
      // chunk's own rows: predicated stores and selects (no branches in the row loop)
      stg2_if(out && (unsigned)(jl - 1 - j0) < nown, pdout + (jl - 1) * nt, ITER ? pd1 : D2{0, 0});   // INIT: pd_{-1} = 0
      // ---- (D) s(jl-2) = A pd, r_{i+1} = r_i - alpha s, x, w2 = D^-1 r_{i+1}
      D2 rn2;
      const D2 AEm2 = ROT ? cE2 : ld2(c2r + NL, tl);
      const D2 AN3 = ROT ? cN3 : ld2(c3 + 2 * NL, tl);
      const double ae2m = ROT ? cE2m : left_of(AEm2.r, c2r + NL, im, lcoef);
      {
        const D2 AP2 = ld2(c2r, tl);
        const D2 AN2 = ROT ? cN2 : ld2(c2r + 2 * NL, tl);
        // s = A pd, the term of the row computed in this step (pd1) added last
        D2 sv{fma(ae2m, rleft(p_2, tl, NTC), dmul(AP2.l, pd2.l)), fma(AEm2.l, pd2.l, dmul(AP2.r, pd2.r))};
        sv = {fma(AEm2.l, pd2.r, sv.l), fma(AEm2.r, rright(p_2, tl), sv.r)};
        sv = {fma(AN3.l, pd3.l, sv.l), fma(AN3.r, pd3.r, sv.r)};
        sv = {fma(AN2.l, pd1.l, sv.l), fma(AN2.r, pd1.r, sv.r)};
        rn2 = {fma(-alpha, sv.l, r2.l), fma(-alpha, sv.r, r2.r)};   // step 5 (INIT: alpha = 0)
      }
      {
        const bool p2 = out && (unsigned)(jl - 2 - j0) < nown;
        const int q2 = (jl - 2) * nt;
        stg2_if(p2, rout + q2, rn2);
        const double trr = dadd(acc_rr, fma(rn2.l, rn2.l, dmul(rn2.r, rn2.r)));
        acc_rr = p2 ? trr : acc_rr;
        if (XUPD) stg2_if(p2, x + q2, D2{dadd(x2.l, fma(alpha_prev, pdo2.l, dmul(alpha, pd2.l))),      // step 4
                                         dadd(x2.r, fma(alpha_prev, pdo2.r, dmul(alpha, pd2.r)))});
        if (MODE == SR_INIT_COLD) {
          stg2_if(p2, x + q2, D2{0, 0});
          const double ts = dadd(acc_s, fma(r2.l, r2.l, dmul(r2.r, r2.r)));
          acc_s = p2 ? ts : acc_s;
        }
        if (MODE == SR_INIT_WARM) {   // x2 holds S here
          const double ts = dadd(acc_s, fma(x2.l, x2.l, dmul(x2.r, x2.r)));
          acc_s = p2 ? ts : acc_s;
        }
      }
      D2 wz;
      if constexpr (PC == SPC_NONE) wz = rn2;
      else wz = {dmul(dmul(rn2.l, oD2.l), romega), dmul(dmul(rn2.r, oD2.r), romega)};
      rst(w2_2, tl, NTC, wz);
      STEP_PROBE(3);
      row_bar<SEAM != SEAM_CHECK>(NCT);                                         // barrier 2: w2(jl-2) complete
      STEP_PROBE(4);

      // ---- (E) v2(jl-2)   (F) z2(jl-3), gamma   (G) A z2 at jl-4, delta
      D2 u2_3;
      if constexpr (PC == SPC_ASSOR2) {
        const D2 w23 = rld(w2_3, tl, NTC);
        const double wz2m = rleft(w2_2, tl, NTC);
        const D2 v23 = rld(v2_3, tl, NTC);
        const double v23p = rright(v2_3, tl);
        const D2 AEm3 = ROT ? cE3 : ld2(c3 + NL, tl);
        double wE2 = 0.0, aW2 = 0.0, vW2 = 0.0;
        if constexpr (SEAM == SEAM_FIXED) {
          wE2 = rright(w2_2, tl);
          aW2 = c3[NL + im];
          vW2 = rleft(v2_3, tl, NTC);
        }
        D2 sL{fma(ae2m, wz2m, dmul(AN3.l, w23.l)), fma(AEm2.l, wz.l, dmul(AN3.r, w23.r))};
        if constexpr (SEAM == SEAM_FIXED) {
          sL.l = seamL ? dmul(AN3.l, w23.l) : sL.l;
          sL.r = seamR ? fma(AEm2.r, wE2, sL.r) : sL.r;
        } else if (SEAM == SEAM_CHECK && seamWarp) {
          if (seamL) sL.l = dmul(AN3.l, w23.l);
          if (seamR) sL.r = fma(AEm2.r, rright(w2_2, tl), sL.r);
        }
        const D2 v22{fma(-oD2.l, sL.l, wz.l), fma(-oD2.r, sL.r, wz.r)};
        rst(v2_2, tl, NTC, v22);
        D2 sU{fma(AN3.l, v22.l, dmul(AEm3.l, v23.r)), fma(AN3.r, v22.r, dmul(AEm3.r, v23p))};
        if constexpr (SEAM == SEAM_FIXED) {
          sU.l = seamL ? fma(aW2, vW2, sU.l) : sU.l;
          sU.r = seamR ? dmul(AN3.r, v22.r) : sU.r;
        } else if (SEAM == SEAM_CHECK && seamWarp) {
          if (seamL) sU.l = fma(c3[NL + im], rleft(v2_3, tl, NTC), sU.l);
          if (seamR) sU.r = dmul(AN3.r, v22.r);
        }
        u2_3 = {dmul(c2, fma(-oD3.l, sU.l, v23.l)), dmul(c2, fma(-oD3.r, sU.r, v23.r))};
      } else {
        u2_3 = rld(w2_3, tl, NTC);
      }
      u2_3r[tl] = u2_3.l;                                  // only the right-neighbour read (delta) remains
      {   // gamma
        const double tg = dadd(acc_g, fma(rn3.l, u2_3.l, dmul(rn3.r, u2_3.r)));
        acc_g = (out && (unsigned)(jl - 3 - j0) < nown) ? tg : acc_g;
      }
      {
        // delta = z2' A z2 as the quadratic form (A symmetric): each owned row j adds its
        // diagonal term and its east and north couplings, i.e. every edge once, at its
        // west / south end -- no w = A z2 vector, one coefficient row (lag 4)
        const D2 AP4 = ld2(c4, tl);
        const D2 AEm4 = ROT ? cE4 : ld2(c4 + NL, tl);
        const D2 AN4 = ROT ? cN4 : ld2(c4 + 2 * NL, tl);
        const double ql = fma(AP4.l, u2_4.l, dmul(2.0, fma(AN4.l, u2_3.l, dmul(AEm4.l, u2_4.r))));
        const double qr = fma(AP4.r, u2_4.r, dmul(2.0, fma(AN4.r, u2_3.r, dmul(AEm4.r, rright(u2_4r, tl)))));
        const double td = dadd(acc_d, fma(u2_4.l, ql, dmul(u2_4.r, qr)));
        acc_d = (out && (unsigned)(jl - 4 - j0) < nown) ? td : acc_d;
      }
      __syncwarp();
      // coefficient row jl-4 done (in the persistent kernel the first 4 steps of a pass release
      // the last 4 rows of the previous pass)
      if (lane0 && gblk + (uint32_t)u >= 4u) mbar_arrive(s.emptyc0 + 8 * ((u + 4) & 7));
      // rotate the histories (register renaming across the unrolled steps)
      u2_4 = u2_3;
      rn3 = rn2;
      pd3 = pd2; pd2 = pd1;
      pdo2 = pdo1;
      r2 = r1; r1 = r0;
      oD3 = oD2; oD2 = oD1; oD1 = oD0;
      if constexpr (ROT) {
        cE4 = cE3; cE3 = cE2; cE2 = cE1; cE1 = AE0;
        cN4 = cN3; cN3 = cN2; cN2 = AN1;
        cE2m = cE1m; cE1m = ae0m;
      }
    }
  }
#ifdef GMAF_STEP_PROBE
  if (lane0 && blockIdx.x < 2048)
    for (int i = 0; i < 6; ++i) atomicAdd(&g_step_probe[(blockIdx.x * 16 + (q.tid >> 5)) * 8 + i], pc_[i]);
#endif
}

// The compute role.  SPLIT: the warp holding the seam runs the SEAM_FIXED row loop and every
// other warp the SEAM_NONE one (warp-uniform choice, once per pass): the plain warps carry no
// seam code, and the seam warp no divergent branches -- worth ~4% at long row chunks (C3), but
// the two loops cost instruction-cache refills at every pass, which short chunks (row slabs of
// 128 rows) do not amortize.  !SPLIT: one SEAM_CHECK loop for all warps.
template <int PC, int MODE, bool SPLIT, int TWC = 0>
__device__ __forceinline__ void sr_compute(const GridParams& g, const DevPtrs& d, const SrGeo& q, const SrSmem& s,
                                           int parity, double alpha, double alpha_prev, double beta, double omega,
                                           uint32_t gstep0, double& acc_rr, double& acc_g, double& acc_d,
                                           double& acc_s) {
  if constexpr (SPLIT) {
    const bool seamWarp = __any_sync(0xffffffffu, (q.seamL || q.seamR) && q.tid < q.NCT);
    if (seamWarp)
      sr_compute_loop<PC, MODE, SEAM_FIXED, false>(g, d, q, s, parity, alpha, alpha_prev, beta, omega, gstep0, acc_rr, acc_g,
                                            acc_d, acc_s);
    else
      sr_compute_loop<PC, MODE, SEAM_NONE, false>(g, d, q, s, parity, alpha, alpha_prev, beta, omega, gstep0, acc_rr, acc_g,
                                           acc_d, acc_s);
  } else {
    sr_compute_loop<PC, MODE, SEAM_CHECK, (TWC > 0)>(g, d, q, s, parity, alpha, alpha_prev, beta, omega, gstep0, acc_rr, acc_g,
                                          acc_d, acc_s);
  }
}

template <int PC, int MODE, int TWC = 0>
__global__ void __maxnreg__(168)
k_sr(GridParams g, DevPtrs d, TileCfg t, int K, int parity, unsigned long long hcond, int use_cond) {
  extern __shared__ __align__(128) double smem_raw[];
  constexpr bool ITER = (MODE == SR_ITER_EVEN || MODE == SR_ITER_ODD);
  constexpr bool INIT = !ITER;
  SolverState* st = d.st_;
  if (ITER && st->done) return;
  timing_begin(d.timing, ITER ? KK_SR_ITER : KK_SR_INIT);
  const SrGeo q = sr_geo<TWC>(g, d, t, K);
  const SrSmem s = sr_smem(smem_raw, q.NL);
  sr_init_barriers(q, s);
  __syncthreads();

  double acc_rr = 0, acc_g = 0, acc_d = 0, acc_s = 0;
  // asynchronous strategy: a frozen condition's CTAs only join the reduction
  const bool frozen = ITER && st->coupling == 2 && d.cs.frz[q.k] != 0;
  if (frozen) {
  } else if (q.is_producer) {
    sr_produce<MODE>(g, d, q, s, K, parity, 0u, 0, q.nsteps);
  } else {
    const double alpha = ITER ? d.cs.alpha[q.k] : 0.0;
    const double alpha_prev = ITER ? d.cs.uvk[q.k] : 0.0;   // uvk holds alpha_{i-1} here
    const double beta = ITER ? d.cs.beta[q.k] : 0.0;
    sr_compute<PC, MODE, false, TWC>(g, d, q, s, parity, alpha, alpha_prev, beta, st->omega, 0u, acc_rr, acc_g, acc_d, acc_s);
  }

  // ---- per-CTA partials, then the scalar stage (last CTA, fixed order)
  double v[4] = {acc_rr, acc_g, acc_d, acc_s};
  // the whole dynamic shared memory (48 NL doubles) is dead now: the reduction scratch needs
  // 4 (blockDim + 32) and 4 K doubles (the host keeps K <= 12 NL on this schedule)
  sr_finish<ITER, INIT>(d, v, smem_raw, K, q.k, t.n_tiles, blockIdx.x / K, hcond, use_cond, q.NCT / 32);
}

static int sr_pairs(const TileCfg& t) { return t.tw / 2 + SR_HALO; }
// compute warps (column pairs rounded up to whole warps) + one TMA producer warp
static int sr_threads(const TileCfg& t) { return ((sr_pairs(t) + 31) & ~31) + 32; }

// ------------------------------------------------------------ persistent iteration kernel
// k_srp runs ALL iterations of a solve in one launch (one CTA per tile, every CTA resident: a
// cooperative launch).  Per iteration the CTA runs the same row pipeline as k_sr, then
//   * its per-thread partials are reduced by a fixed warp-shuffle tree + warps in order,
//   * thread 0 publishes them and arrives on a grid barrier (a monotonically increasing
//     counter: release add, acquire spin),
//   * EVERY CTA sums the per-CTA partials of every condition in CTA order (the same loads in the
//     same order everywhere) and runs the scalar stage (Eq. 3.9, alpha, beta; R-A24, R-A32) on its
//     own shared-memory copy of the solver state -- so every CTA holds bitwise the same scalars
//     and no CTA waits for a serial last-CTA tail or a kernel boundary;
//   * meanwhile the producer warp, released by the same grid barrier, already streams the first
//     rows of the next iteration (their data does not depend on the scalars).
// CTA 0 writes the state and the per-condition scalars back to global memory at exit.
// One rank only (row slabs / condition sharding keep the per-launch kernels + exchange kernels).
constexpr int kCtrGridBar = 14;   // d.counters slot of the grid barrier (zeroed before the launch)

__host__ __device__ inline size_t srp_align(size_t x) { return (x + 15) & ~(size_t)15; }
// extra dynamic shared memory after the rings: state copy, [4K] sums, [4 Kall] sums over the
// ranks (multi-rank: Kall = all conditions of the joint system), [4][32] warp partials,
// [4][nblk] per-CTA partials, 7 K doubles + 2 K ints of per-condition scalars, the flags
__host__ __device__ inline size_t srp_extra_bytes(int K, int nblk, int Kall) {
  return srp_align(sizeof(SolverState)) + srp_align((size_t)4 * K * 8) + srp_align((size_t)4 * Kall * 8) + 4 * 32 * 8 +
         srp_align((size_t)4 * nblk * 8) + srp_align((size_t)7 * K * 8) + srp_align((size_t)2 * K * 4) + 16 + 32 + 16;
}
__host__ __device__ inline size_t srp_smem_bytes(int nl, int K, int nblk, int Kall) {
  return srp_align(sr_smem_bytes(nl)) + srp_extra_bytes(K, nblk, Kall);
}

__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned int* p, unsigned int v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
constexpr long long kGridBarTimeoutNs = 20000000000ll;   // 20 s: a CTA that never arrives fails the solve
// spin until the grid barrier counter reaches target; false on timeout
__device__ __forceinline__ bool grid_wait(const unsigned int* ctr, unsigned int target) {
  if (ld_acquire_u32(ctr) >= target) return true;
  const unsigned long long t0 = globaltimer();
  while (ld_acquire_u32(ctr) < target)
    if ((long long)(globaltimer() - t0) > kGridBarTimeoutNs) return false;
  return true;
}

struct SrpShared {
  SolverState* st;
  double* red;      // [4K] per-condition sums [rr | gamma | delta | S.S]
  double* red2;     // [4 Kall] the sums the scalar stage takes (multi-rank: over all ranks)
  double* wpart;    // [4][32] per-warp partials
  double* pbuf;     // [4K][ncta] the per-CTA partials of one iteration
  CondScalars cs;   // CTA-private per-condition scalars
  volatile int* ready;   // [0]: iterations whose scalars are ready; [1]: failure flag
  unsigned long long* tim;   // [4] CTA 0's timing accumulators
  unsigned long long* seqbase;   // multi-rank: gathers issued before this launch
};
__device__ __forceinline__ SrpShared srp_shared(double* smem_raw, int NL, int K, int nblk, int Kall) {
  char* b = reinterpret_cast<char*>(smem_raw) + srp_align(sr_smem_bytes(NL));
  SrpShared x;
  x.st = reinterpret_cast<SolverState*>(b);
  b += srp_align(sizeof(SolverState));
  x.red = reinterpret_cast<double*>(b);
  b += srp_align((size_t)4 * K * 8);
  x.red2 = reinterpret_cast<double*>(b);
  b += srp_align((size_t)4 * Kall * 8);
  x.wpart = reinterpret_cast<double*>(b);
  b += 4 * 32 * 8;
  x.pbuf = reinterpret_cast<double*>(b);
  b += srp_align((size_t)4 * nblk * 8);
  double* a = reinterpret_cast<double*>(b);
  x.cs.alpha = a; x.cs.beta = a + K; x.cs.dk = a + 2 * K; x.cs.Sk = a + 3 * K; x.cs.rrk = a + 4 * K;
  x.cs.uvk = a + 5 * K; x.cs.ttk = a + 6 * K;
  b += srp_align((size_t)7 * K * 8);
  x.cs.itk = reinterpret_cast<int32_t*>(b); x.cs.frz = x.cs.itk + K;
  b += srp_align((size_t)2 * K * 4);
  x.ready = reinterpret_cast<volatile int*>(b);
  x.tim = reinterpret_cast<unsigned long long*>(b + 16);
  x.seqbase = reinterpret_cast<unsigned long long*>(b + 48);
  return x;
}

// Multi-rank (peer-to-peer): the same kernel on every rank.  Row slabs
// (d.dist.rows == 1): after its pass a CTA whose chunk touches the slab edge stores its output
// columns of the 4 boundary rows of r_{i+1} and pd_i straight into the neighbour's inbox over
// NVLink (slot = parity of the next gather stamp); after the local grid barrier, warp 0 of CTA 0
// pushes the rank's per-condition sums into every rank's exchange buffer and posts its stamp
// (release, system scope); EVERY CTA then waits for all ranks' stamps in its own buffer, reads
// the blocks, adds them over the ranks in rank order (row slabs) or places them in global
// condition order (condition sharding) and runs the same scalar stage -- bitwise the same
// scalars on every CTA of every rank.  The producers of edge chunks stream their halo rows from
// the inbox once the stamps (which also publish the halos) are in.
template <int PC, bool SPLIT, bool DIST, int TWC = 0>
__global__ void __maxnreg__(168) k_srp(GridParams g, DevPtrs d, TileCfg t, int K) {
  extern __shared__ __align__(128) double smem_raw[];
  if (d.st_->done) return;                   // the init already converged (or failed)
  constexpr bool dist = DIST;                // peer-to-peer multi-rank context (d.dist.world > 0)
  const int Kall = dist && d.dist.rows != 1 ? d.dist.kglob : K;
  const SrGeo q = sr_geo<TWC>(g, d, t, K);
  const SrSmem s = sr_smem(smem_raw, q.NL);
  const SrpShared x = srp_shared(smem_raw, q.NL, K, (int)gridDim.x, Kall);
  sr_init_barriers(q, s);
  // CTA-private copies of the solver state and of the per-condition scalars
  for (int i = q.tid; i < K; i += blockDim.x) {
    x.cs.alpha[i] = d.cs.alpha[i]; x.cs.beta[i] = d.cs.beta[i]; x.cs.dk[i] = d.cs.dk[i];
    x.cs.Sk[i] = d.cs.Sk[i]; x.cs.rrk[i] = d.cs.rrk[i]; x.cs.uvk[i] = d.cs.uvk[i]; x.cs.ttk[i] = d.cs.ttk[i];
    x.cs.itk[i] = d.cs.itk[i]; x.cs.frz[i] = d.cs.frz[i];
    x.red[3 * K + i] = 0.0;                  // the S.S sums: not formed in the iterations
  }
  if (q.tid == 0) {
    *x.st = *d.st_;
    x.ready[0] = 0;
    x.ready[1] = 0;
    *x.seqbase = dist ? *d.dist.seq : 0ull;   // nobody gathers before every CTA has passed barrier 0
  }
  __syncthreads();
  const int it0 = x.st->iter;                // iteration count at entry (0 after the init)
  const bool async = x.st->coupling == 2;
  const int nblk = gridDim.x, ncta = t.n_tiles, cta = blockIdx.x / K;
  unsigned int* gbar = d.counters + kCtrGridBar;
  const bool rows = dist && d.dist.rows == 1 && d.dist.world > 1;
  uint32_t gstep = 0;                        // row steps this CTA streamed / consumed so far

  if (q.is_producer) {
    // ------------------------------------------------ producer: stream every iteration
    const int lane = q.tid - q.NCT;
    // a chunk at a slab edge streams halo rows from the inbox: it needs the gather (whose
    // stamps publish them), the others only the local grid barrier
    const bool edge = rows && ((q.jbase < g.y0 && d.dist.rank > 0) ||
                               (q.j1 + SR_YLO > g.y1 && d.dist.rank < d.dist.world - 1));
    for (int it = 0;; ++it) {
      const int parity = (it0 + it) & 1;
      const int islot = (int)((*x.seqbase + (unsigned long long)it) & 1ull);
      int pre = 0;
      if (it > 0) {
        // the rows of iteration it were written by all CTAs (and neighbours) in iteration it-1
        bool ok = true;
        if (lane == 0)
          ok = edge ? p2p_stamps_wait(d.dist, *x.seqbase + (unsigned long long)it) : grid_wait(gbar, (unsigned)(it * nblk));
        ok = __shfl_sync(0xffffffffu, ok, 0);
        if (!ok) break;
        fence_proxy_async_global();          // generic-proxy / peer stores -> TMA (async-proxy) reads
        if (!async) {                        // prefetch 4 steps while the scalars are computed
          pre = 4;
          if (parity) sr_produce<SR_ITER_ODD>(g, d, q, s, K, 1, gstep, 0, pre, islot);
          else sr_produce<SR_ITER_EVEN>(g, d, q, s, K, 0, gstep, 0, pre, islot);
        }
        while (x.ready[0] < it && x.ready[1] == 0) __nanosleep(32);
      }
      __syncwarp();
      __threadfence_block();                 // the state written before the flag, read after it
      const bool stop = x.ready[1] != 0 || *reinterpret_cast<volatile int32_t*>(&x.st->done) != 0;
      if (stop) {
        // drain the prefetched steps (TMA writes into this CTA's shared memory) before exiting
        if (lane == 0)
          for (int b = 0; b < pre; ++b) mbar_wait(s.full0 + 8 * ((gstep + b) & 7), (gstep / SR_UNROLL) & 1u);
        break;
      }
      if (async && *reinterpret_cast<volatile int32_t*>(&x.cs.frz[q.k]) != 0) continue;   // frozen: no rows
      if (parity) sr_produce<SR_ITER_ODD>(g, d, q, s, K, 1, gstep, pre, q.nsteps, islot);
      else sr_produce<SR_ITER_EVEN>(g, d, q, s, K, 0, gstep, pre, q.nsteps, islot);
      gstep += (uint32_t)q.nsteps;
    }
    return;
  }

  // ------------------------------------------------------ compute warps
  const int NCT = q.NCT, nw = NCT >> 5;
  const bool timed = blockIdx.x == 0 && q.tid == 0;
  // CTA 0's timing accumulators live in shared memory (registers are the hot loop's)
  volatile unsigned long long* tim = x.tim;   // [0] start, [1] tail, [2] wait, [3] arrival
  if (timed) { tim[0] = globaltimer(); tim[1] = 0ull; tim[2] = 0ull; }
  const double omega = x.st->omega;
  for (int it = 0;; ++it) {
    const int parity = (it0 + it) & 1;
    double a_rr = 0.0, a_g = 0.0, a_d = 0.0, a_s = 0.0;
    if (!(async && x.cs.frz[q.k])) {
      const double alpha = x.cs.alpha[q.k], alpha_prev = x.cs.uvk[q.k], beta = x.cs.beta[q.k];
      if (parity) sr_compute<PC, SR_ITER_ODD, SPLIT, TWC>(g, d, q, s, 1, alpha, alpha_prev, beta, omega, gstep, a_rr, a_g, a_d, a_s);
      else sr_compute<PC, SR_ITER_EVEN, SPLIT, TWC>(g, d, q, s, 0, alpha, alpha_prev, beta, omega, gstep, a_rr, a_g, a_d, a_s);
      gstep += (uint32_t)q.nsteps;
    }
    // field stores of this iteration -> visible to the other CTAs' TMA reads after the barrier:
    // a proxy fence per thread; the gpu-scope ordering comes from thread 0's fence + release after
    // the CTA barrier below, which is cumulative over the writes the barrier ordered before it (the
    // scheme of cooperative groups' grid sync: only the arriving thread fences)
    fence_proxy_async_global();
    if (rows) {
      // row slabs: this CTA's output columns of the rows it owns among the 4 boundary rows of each
      // slab edge (r_{i+1} and pd_i) go straight into the neighbour's inbox (the next gather's
      // stamp publishes them); a ragged last chunk may own only part of an edge band
      const int rank = d.dist.rank, world = d.dist.world;
      const int lo_a = max(q.j0, g.y0), lo_b = min(q.j1, g.y0 + SLAB_HALO);          // band below
      const int hi_a = max(q.j0, g.y1 - SLAB_HALO), hi_b = min(q.j1, g.y1);          // band above
      const bool lo_edge = rank > 0 && lo_a < lo_b, hi_edge = rank < world - 1 && hi_a < hi_b;
      if (lo_edge || hi_edge) {
        compute_bar(NCT);                    // every thread's row stores precede the copies
        const int slot = (int)((*x.seqbase + (unsigned long long)it + 1ull) & 1ull);
        if (q.out) {
          for (int side = 0; side < 2; ++side) {
            if (side == 0 ? !lo_edge : !hi_edge) continue;
            double* inbox = d.dist.halo_in[side == 0 ? rank - 1 : rank + 1];
            const int ra = side == 0 ? lo_a : hi_a, rb = side == 0 ? lo_b : hi_b;
            const int rbase = side == 0 ? g.y0 : g.y1 - SLAB_HALO;
            for (int vec = 0; vec < 2; ++vec) {
              const double* src = (vec == 0 ? d.r[1 - parity] : d.u[parity]) + q.fk;
              for (int row = ra; row < rb; ++row) {
                const double2 v = __ldcg(reinterpret_cast<const double2*>(src + (long long)row * g.nt + q.gl));
                *reinterpret_cast<double2*>(inbox + halo_ofs(slot, 1 - side, vec, K, q.k, row - rbase, g.nt) + q.gl) = v;
              }
            }
          }
          __threadfence_system();
        }
      }
    }
    // fixed-order block reduction (the same as k_sr's, so both give bitwise the same partials)
    double v[3] = {a_rr, a_g, a_d};
    warp_tree_sum<3>(v, x.wpart);
    compute_bar(NCT);
    const unsigned int target = (unsigned)((it + 1) * nblk);
    double* part = d.partials + (size_t)(it & 1) * 4 * K * ncta;   // parity buffers
    if (q.tid == 0) {
      if (timed) tim[3] = globaltimer();
      // load-balance diagnostics: this CTA's arrival at the grid barrier (at the end of the
      // partials region; gmaf_cta_arrivals)
      if (g.diag && it < kDiagIters)
        reinterpret_cast<unsigned long long*>(d.partials + diag_offset(K, nblk))[it * nblk + blockIdx.x] = globaltimer();
      warps_in_order<3>(v, x.wpart, nw);
      for (int c = 0; c < 3; ++c) part[(size_t)(c * K + q.k) * ncta + cta] = v[c];
      // the release add publishes the partials and (cumulatively, after the CTA barrier) the
      // CTA's field stores; the acquire spin orders every later read -- no separate fences
      red_release_add(gbar, 1u);
      if (!grid_wait(gbar, target)) x.ready[1] = 1;
    }
    compute_bar(NCT);
    if (x.ready[1]) break;
    const unsigned long long t_bar = timed ? globaltimer() : 0ull;
    if (timed) tim[2] = tim[2] + (t_bar - tim[3]);
    // per-condition sums over the CTAs in CTA order (identical in every CTA): every partial is
    // loaded at once (one L2 round trip), then each (q, k) row is summed in CTA order
    {   // (the S.S column is not summed in the iterations: red[3K, 4K) stays zero)
      // stored CTA-major ([cta][row]) so that the per-row sums below read consecutive banks
      const int np = 3 * K * ncta, nrow = 3 * K;
#pragma unroll 4
      for (int i = q.tid; i < np; i += NCT) {
        const int row = i / ncta, b = i - row * ncta;
        x.pbuf[b * nrow + row] = __ldcg(part + i);
      }
    }
    compute_bar(NCT);
    double* red = x.red;
    for (int i = q.tid; i < 3 * K; i += NCT) {
      double a = 0.0;
      for (int b = 0; b < ncta; ++b) a += x.pbuf[b * (3 * K) + i];   // CTA order
      red[i] = a;
    }
    compute_bar(NCT);
    int kofs = 0;
    if (dist) {
      // warp 0 of CTA 0 pushes this rank's sums to every rank (peer memory, release stamp);
      // every CTA waits for all ranks' stamps itself and reads the blocks from its own buffer
      const int km = d.dist.kmax_local;
      const unsigned long long stamp = *x.seqbase + (unsigned long long)it + 1ull;
      if (blockIdx.x == 0 && q.tid < 32) {
        for (int i = q.tid; i < 4 * km; i += 32) {
          const int qq = i / km, kk = i - qq * km;
          d.dist.packed_local[i] = kk < K ? red[qq * K + kk] : 0.0;
        }
        __syncwarp();
        p2p_push(d.dist, d.dist.packed_local, 4 * km, stamp);
      }
      if (q.tid == 0 && !p2p_stamps_wait(d.dist, stamp)) x.ready[1] = 2;
      compute_bar(NCT);
      if (x.ready[1]) break;
      const int W = d.dist.world;
      if (d.dist.rows == 1) {
        // row slabs: every rank holds all K conditions; add the ranks' sums in rank order
        for (int i = q.tid; i < 4 * K; i += NCT) {
          const int qq = i / K, kk = i - qq * K;
          double a = 0.0;
          for (int r = 0; r < W; ++r) a += p2p_block(d.dist, stamp, r, qq * km + kk);
          x.red2[i] = a;
        }
      } else {
        // condition sharding: the ranks' blocks in global condition order
        kofs = d.dist.kofs;
        for (int kg = q.tid; kg < Kall; kg += NCT) {
          int r, kl;
          dist_owner(kg, Kall, W, &r, &kl);
          for (int qq = 0; qq < 4; ++qq) x.red2[qq * Kall + kg] = p2p_block(d.dist, stamp, r, qq * km + kl);
        }
      }
      compute_bar(NCT);
      if (blockIdx.x == 0)
        for (int kg = q.tid; kg < Kall; kg += NCT) d.dist.rr_all[kg] = x.red2[kg];
      red = x.red2;
    }
    if (q.tid == 0) {
      sr_scalar_stage<false>(x.cs, x.st, red, Kall, K, kofs, 0, 0ull, stage_prefetch(x.cs, x.st));
      __threadfence_block();
      x.ready[0] = it + 1;                  // the producer may go on (or stop)
    }
    compute_bar(NCT);
    if (timed) tim[1] = tim[1] + (globaltimer() - t_bar);
    if (x.st->done) break;
  }
  // CTA 0 writes the solver state and the per-condition scalars back
  if (blockIdx.x == 0) {
    for (int i = q.tid; i < K; i += NCT) {
      d.cs.alpha[i] = x.cs.alpha[i]; d.cs.beta[i] = x.cs.beta[i]; d.cs.dk[i] = x.cs.dk[i];
      d.cs.Sk[i] = x.cs.Sk[i]; d.cs.rrk[i] = x.cs.rrk[i]; d.cs.uvk[i] = x.cs.uvk[i];
      d.cs.itk[i] = x.cs.itk[i]; d.cs.frz[i] = x.cs.frz[i];
    }
    if (q.tid == 0) {
      SolverState st = *x.st;
      if (x.ready[1]) { st.done = 1; st.status = -9; }   // GMAF_E_CUDA: barrier or peer timeout
      *d.st_ = st;
      const unsigned long long t1 = globaltimer();
      const int iters = st.iter - it0;
      atomicAdd(&d.timing->total_ns[KK_SR_ITER], t1 - tim[0]);
      atomicAdd(&d.timing->launches[KK_SR_ITER], (unsigned long long)(iters > 0 ? iters : 0));
      atomicAdd(&d.timing->total_ns[KK_SR_TAIL], (unsigned long long)tim[1]);
      atomicAdd(&d.timing->launches[KK_SR_TAIL], (unsigned long long)(iters > 0 ? iters : 0));
      atomicAdd(&d.timing->total_ns[KK_SR_WAIT], (unsigned long long)tim[2]);
      atomicAdd(&d.timing->launches[KK_SR_WAIT], (unsigned long long)(iters > 0 ? iters : 0));
    }
  }
}

// conditions the scalar stage sees: all of the joint system when condition-sharded
static int srp_kall(const DevPtrs& d, int K) { return d.dist.world > 0 && d.dist.rows != 1 ? d.dist.kglob : K; }

// The split seam variant (see sr_compute): off by default.  With the seam warp and the other
// warps in different loops, the row barriers must be one shared out-of-line bar.sync (an
// .aligned barrier may not be reached from different instructions; compute-sanitizer synccheck
// flags it), and the calls cost more than the split saves (C3: 260 vs 250 us per iteration on
// the same box).  GMAF_SEAM_SPLIT=1 selects it for experiments.
bool srp_split_seam(const TileCfg& t) {
  (void)t;
  if (const char* e = std::getenv("GMAF_SEAM_SPLIT")) return std::atoi(e) != 0;
  return false;
}

#ifdef GMAF_STEP_PROBE
extern "C" int gmaf_debug_step_probe(unsigned int* out, int n, int reset) {
  if (n > 2048 * 16 * 8) n = 2048 * 16 * 8;
  if (cudaMemcpyFromSymbol(out, g_step_probe, (size_t)n * 4) != cudaSuccess) return -1;
  if (reset) {
    static unsigned int zeros[2048 * 16 * 8];
    if (cudaMemcpyToSymbol(g_step_probe, zeros, sizeof(zeros)) != cudaSuccess) return -1;
  }
  return n;
}
#endif

cudaError_t launch_sr_persistent(const GridParams& g, const DevPtrs& d, const TileCfg& t, int K, int precond,
                                 cudaStream_t s) {
  const bool split = srp_split_seam(t);
  const bool dist = d.dist.world > 0;
  cudaError_t e = cudaMemsetAsync(d.counters + kCtrGridBar, 0, sizeof(unsigned int), s);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(t.n_tiles * K);
  cfg.blockDim = dim3(sr_threads(t));
  cfg.dynamicSmemBytes = srp_smem_bytes(2 * sr_pairs(t), K, t.n_tiles * K, srp_kall(d, K));
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;   // every CTA resident (the grid barrier needs it)
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  switch (precond) {
    case SPC_ASSOR2:
      // (the multi-rank kernel keeps one loop: with the split loops it spills in the row loop)
      if (dist) {
        if (t.tw == 512) return cudaLaunchKernelEx(&cfg, k_srp<SPC_ASSOR2, false, true, 512>, g, d, t, K);
        if (t.tw == 256) return cudaLaunchKernelEx(&cfg, k_srp<SPC_ASSOR2, false, true, 256>, g, d, t, K);
        return cudaLaunchKernelEx(&cfg, k_srp<SPC_ASSOR2, false, true>, g, d, t, K);
      }
      if (split) return cudaLaunchKernelEx(&cfg, k_srp<SPC_ASSOR2, true, false>, g, d, t, K);
      if (t.tw == 512) return cudaLaunchKernelEx(&cfg, k_srp<SPC_ASSOR2, false, false, 512>, g, d, t, K);
      if (t.tw == 256) return cudaLaunchKernelEx(&cfg, k_srp<SPC_ASSOR2, false, false, 256>, g, d, t, K);
      return cudaLaunchKernelEx(&cfg, k_srp<SPC_ASSOR2, false, false>, g, d, t, K);
    // the comparison preconditioners (paper studies, NEXT-4) get the compile-time widths on one
    // rank too, so that their per-iteration times are comparable with ASSOR-II's
    case SPC_ASSOR1:
      if (dist) return cudaLaunchKernelEx(&cfg, k_srp<SPC_ASSOR1, false, true>, g, d, t, K);
      if (t.tw == 512) return cudaLaunchKernelEx(&cfg, k_srp<SPC_ASSOR1, false, false, 512>, g, d, t, K);
      if (t.tw == 256) return cudaLaunchKernelEx(&cfg, k_srp<SPC_ASSOR1, false, false, 256>, g, d, t, K);
      return cudaLaunchKernelEx(&cfg, k_srp<SPC_ASSOR1, false, false>, g, d, t, K);
    case SPC_JACOBI:
      if (dist) return cudaLaunchKernelEx(&cfg, k_srp<SPC_JACOBI, false, true>, g, d, t, K);
      if (t.tw == 512) return cudaLaunchKernelEx(&cfg, k_srp<SPC_JACOBI, false, false, 512>, g, d, t, K);
      if (t.tw == 256) return cudaLaunchKernelEx(&cfg, k_srp<SPC_JACOBI, false, false, 256>, g, d, t, K);
      return cudaLaunchKernelEx(&cfg, k_srp<SPC_JACOBI, false, false>, g, d, t, K);
    default:
      if (dist) return cudaLaunchKernelEx(&cfg, k_srp<SPC_NONE, false, true>, g, d, t, K);
      if (t.tw == 512) return cudaLaunchKernelEx(&cfg, k_srp<SPC_NONE, false, false, 512>, g, d, t, K);
      if (t.tw == 256) return cudaLaunchKernelEx(&cfg, k_srp<SPC_NONE, false, false, 256>, g, d, t, K);
      return cudaLaunchKernelEx(&cfg, k_srp<SPC_NONE, false, false>, g, d, t, K);
  }
}

// resident CTAs per SM of the persistent kernel with K conditions (0: it does not fit)
int srp_ctas_per_sm(const TileCfg& t, int K, int Kall) {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_srp<SPC_ASSOR2, false, true>, sr_threads(t),
                                                    srp_smem_bytes(2 * sr_pairs(t), K, t.n_tiles * K, Kall)) != cudaSuccess)
    return 0;
  return n;
}

// Multi-rank scalar stage: one CTA, after the allgather of every rank's packed sums
// (rank-major = condition-major since ranks own contiguous condition blocks).
template <bool INIT>
__global__ void k_sr_scalar(DevPtrs d, int Kglob, int Klocal, int kofs, int world) {
  if (!INIT && d.st_->done) return;
  extern __shared__ double sh[];       // [4][Kglob]
  const int km = d.dist.kmax_local;
  for (int kg = threadIdx.x; kg < Kglob; kg += blockDim.x) {
    int r, kl;
    dist_owner(kg, Kglob, world, &r, &kl);
    const double* src = d.dist.packed_all + (long long)r * 4 * km;
    for (int q = 0; q < 4; ++q) sh[q * Kglob + kg] = src[q * km + kl];
  }
  __syncthreads();
  if (threadIdx.x == 0) sr_scalar_stage<INIT>(d, sh, Kglob, Klocal, kofs, 0, 0ull);
}

// Peer-to-peer allgather as its own (one-warp) kernel: the true-residual and wrench gathers.
__global__ void k_p2p_gather(DevPtrs d, const double* src, int n, double* dst) {
  if (!p2p_gather(d.dist, src, n, dst) && threadIdx.x == 0) { d.st_->done = 1; d.st_->status = -9; }
}

cudaError_t launch_p2p_gather(const DevPtrs& d, const double* src, int n, double* dst, cudaStream_t s) {
  k_p2p_gather<<<1, 32, 0, s>>>(d, src, n, dst);
  return cudaGetLastError();
}

// x += alpha_{it-1} pd_{it-1} when the iteration count is odd (the last x update of the
// two-at-a-time scheme is still pending).  Elementwise, reads the device iteration count.
__global__ void k_sr_fixup(GridParams g, DevPtrs d, int K) {   // K = local conditions
  const bool async = d.st_->coupling == 2;     // asynchronous: each condition has its own count
  if (!async && (d.st_->iter & 1) == 0) return;
  const long long n = (long long)(g.y1 - g.y0) * g.nt;   // own rows
  const double* pd = d.u[0];   // pd_{it-1}, it-1 even -> parity 0
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n * K;
       q += (long long)gridDim.x * blockDim.x) {
    const int kk = (int)(q / n);
    const long long o = fofs(g, kk) + (long long)g.y0 * g.nt + (q - (long long)kk * n);
    const int it = async ? d.cs.itk[kk] : d.st_->iter;
    if (it & 1) d.p[o] = d.p[o] + d.cs.uvk[kk] * pd[o];
  }
}

// --------------------------------------------------------------------- launchers

template <typename KernelT>
static cudaError_t sr_launch(KernelT kern, const GridParams& g, const DevPtrs& d, const TileCfg& t, int K,
                             int parity, unsigned long long h, int use, cudaStream_t s) {
  const int threads = sr_threads(t);
  kern<<<dim3(t.n_tiles * K), threads, sr_smem_bytes(2 * sr_pairs(t)), s>>>(g, d, t, K, parity, h, use);
  return cudaGetLastError();
}

template <int MODE>
static cudaError_t sr_launch_mode(int precond, const GridParams& g, const DevPtrs& d, const TileCfg& t, int K,
                                  int parity, unsigned long long h, cudaStream_t s) {
  const int use = h != 0ull;
  switch (precond) {
    case SPC_ASSOR2:   // compile-time strip widths for the common meshes (sr_geo TWC)
      if (t.tw == 512) return sr_launch(k_sr<SPC_ASSOR2, MODE, 512>, g, d, t, K, parity, h, use, s);
      if (t.tw == 256) return sr_launch(k_sr<SPC_ASSOR2, MODE, 256>, g, d, t, K, parity, h, use, s);
      return sr_launch(k_sr<SPC_ASSOR2, MODE>, g, d, t, K, parity, h, use, s);
    case SPC_ASSOR1: return sr_launch(k_sr<SPC_ASSOR1, MODE>, g, d, t, K, parity, h, use, s);
    case SPC_JACOBI: return sr_launch(k_sr<SPC_JACOBI, MODE>, g, d, t, K, parity, h, use, s);
    default: return sr_launch(k_sr<SPC_NONE, MODE>, g, d, t, K, parity, h, use, s);
  }
}

cudaError_t launch_sr_init(const GridParams& g, const DevPtrs& d, const TileCfg& t, int K, int precond,
                           bool warm, unsigned long long h, cudaStream_t s) {
  if (warm) return sr_launch_mode<SR_INIT_WARM>(precond, g, d, t, K, 1, h, s);
  return sr_launch_mode<SR_INIT_COLD>(precond, g, d, t, K, 1, h, s);
}

// iteration i = 2m + parity: odd iterations also apply the pending x update
cudaError_t launch_sr_iter(const GridParams& g, const DevPtrs& d, const TileCfg& t, int K, int precond,
                           int parity, unsigned long long h, cudaStream_t s) {
  if (parity & 1) return sr_launch_mode<SR_ITER_ODD>(precond, g, d, t, K, parity, h, s);
  return sr_launch_mode<SR_ITER_EVEN>(precond, g, d, t, K, parity, h, s);
}

// Peer-to-peer mode: right after every init / iteration kernel (same CUDA graph), one CTA
// gathers all ranks' packed per-condition sums over NVLink peer memory and runs the scalar stage
// in global condition order -- bitwise the same on every rank -- and sets the WHILE condition.
// (Fusing this tail into k_sr itself was measured 30% slower: the extra code costs the hot loop
// registers; the separate 1-CTA kernel costs ~1%.)
template <bool INIT>
__global__ void k_p2p_scalar(DevPtrs d, int Klocal, unsigned long long hcond, int use_cond) {
  __shared__ double sh[4 * 256];
  if (!INIT && d.st_->done) return;
  const int km = d.dist.kmax_local, Kg = d.dist.kglob, lane = threadIdx.x;   // one warp
  if (!p2p_gather(d.dist, d.dist.packed_local, 4 * km, d.dist.packed_all)) {
    if (lane == 0) {
      d.st_->done = 1;
      d.st_->status = -9;                                 // GMAF_E_CUDA: a peer never arrived
      if (use_cond) cudaGraphSetConditional((cudaGraphConditionalHandle)hcond, 0u);
    }
    return;
  }
  for (int kg = lane; kg < Kg; kg += 32) {                // lanes in parallel (no dependent chain)
    int r, kl;
    dist_owner(kg, Kg, d.dist.world, &r, &kl);
    const double* srcp = d.dist.packed_all + (long long)r * 4 * km;
    for (int q = 0; q < 4; ++q) sh[q * Kg + kg] = srcp[q * km + kl];
    d.dist.rr_all[kg] = sh[kg];
    if (INIT) d.dist.ss_all[kg] = sh[3 * Kg + kg];
  }
  __syncwarp();
  if (lane == 0) sr_scalar_stage<INIT>(d, sh, Kg, Klocal, d.dist.kofs, use_cond, hcond);
}

// ------------------------------------------------- row-slab exchange
// Every rank holds all K conditions on the rows [y0, y1).  Push the SLAB_HALO boundary rows of
// nv vectors of every condition into the neighbours' inboxes (slot = parity of the NEXT gather
// stamp): own rows [y0, y0+H) go to rank-1 (its side 1), rows [y1-H, y1) to rank+1 (its side
// 0).  16-byte stores to peer memory over NVLink, then a system-scope fence, so that the stamp
// the following gather posts also publishes the halos.
constexpr int kCtrSlabRows = KK_COUNT + 1, kCtrSlabPush = KK_COUNT + 2;   // last-CTA counters

__device__ __forceinline__ void slab_push(const GridParams& g, const DevPtrs& d, const double* v0,
                                          const double* v1, int nv, int K) {
  const DistPtrs& dd = d.dist;
  const int slot = (int)((*dd.seq + 1ull) & 1ull);
  const int nt2 = g.nt / 2;
  // rows to send: [side][vec][k][ri], sides without a neighbour skipped; one CTA per row
  const int s0 = dd.rank > 0 ? 0 : 1, s1 = dd.rank < dd.world - 1 ? 2 : 1;
  const int per_side = nv * K * SLAB_HALO;
  for (int q = blockIdx.x; q < (s1 - s0) * per_side; q += gridDim.x) {
    const int side = s0 + q / per_side;                            // 0: to rank-1, 1: to rank+1
    const int e = q % per_side;
    const int ri = e % SLAB_HALO, k = (e / SLAB_HALO) % K, vec = e / (SLAB_HALO * K);
    const int row = side == 0 ? g.y0 + ri : g.y1 - SLAB_HALO + ri;
    const double2* src = reinterpret_cast<const double2*>((vec == 0 ? v0 : v1) + fofs(g, k) + (long long)row * g.nt);
    double2* dst = reinterpret_cast<double2*>(dd.halo_in[side == 0 ? dd.rank - 1 : dd.rank + 1] +
                                              halo_ofs(slot, 1 - side, vec, K, k, ri, g.nt));
    for (int c2 = threadIdx.x; c2 < nt2; c2 += blockDim.x) dst[c2] = src[c2];
  }
  // every thread that stored to a peer fences its OWN stores at system scope (a fence by one
  // thread after a CTA barrier does not drain the other warps' outstanding stores); then
  // last_cta_arrive chains the CTAs to the thread that posts the stamp
  __threadfence_system();
}

// The rank's per-condition sums of all ranks, summed in rank order (bitwise the same on every
// rank), then the scalar stage and the WHILE condition.  One warp.
template <bool INIT>
__device__ void slab_scalars(const DevPtrs& d, int K, unsigned long long hcond, int use_cond) {
  __shared__ double sh[4 * 256];
  const int km = d.dist.kmax_local, lane = threadIdx.x & 31;
  if (!p2p_gather(d.dist, d.dist.packed_local, 4 * km, d.dist.packed_all)) {
    if (lane == 0) {
      d.st_->done = 1;
      d.st_->status = -9;                                 // GMAF_E_CUDA: a peer never arrived
      if (use_cond) cudaGraphSetConditional((cudaGraphConditionalHandle)hcond, 0u);
    }
    return;
  }
  for (int i = lane; i < 4 * K; i += 32) {                // (q, k) pairs in parallel, ranks in order
    const int q = i / K, k = i - q * K;
    double s = 0.0;
    for (int r = 0; r < d.dist.world; ++r) s += d.dist.packed_all[(long long)r * 4 * km + q * km + k];
    sh[i] = s;
    if (q == 0) d.dist.rr_all[k] = s;
    if (INIT && q == 3) d.dist.ss_all[k] = s;
  }
  __syncwarp();
  if (lane == 0) sr_scalar_stage<INIT>(d, sh, K, K, 0, use_cond, hcond);
}

// After every init / iteration kernel of a row-slab solve (same CUDA graph): push the halos of
// the two vectors the next iteration reads across slab edges (r_{i+1}, pd_i; init: r_0, pd_-1),
// then the last CTA gathers the sums and runs the scalar stage.  The next k_sr streams those
// halo rows from the own inbox (TMA), so the exchange costs no extra pass over the fields.
template <bool INIT>
__global__ void k_p2p_rows(GridParams g, DevPtrs d, int parity, int K, unsigned long long hcond, int use_cond) {
  if (!INIT && d.st_->done) return;
  const double* va = INIT ? d.r[0] : d.r[1 - parity];
  const double* vb = INIT ? d.u[1] : d.u[parity];
  slab_push(g, d, va, vb, 2, K);
  if (!last_cta_arrive(&d.counters[kCtrSlabRows], gridDim.x)) return;
  if (threadIdx.x < 32) slab_scalars<INIT>(d, K, hcond, use_cond);
}

// One-off halo exchange of one field (the solution before a warm start / the true residual /
// the quadrature; the warm-start residual): push, a gather that only carries the stamp, then
// k_slab_unpack copies the inbox into the field's halo rows.
__global__ void k_slab_push(GridParams g, DevPtrs d, const double* v, int K) {
  slab_push(g, d, v, v, 1, K);
  if (!last_cta_arrive(&d.counters[kCtrSlabPush], gridDim.x)) return;
  if (threadIdx.x < 32 && !p2p_gather(d.dist, d.dist.packed_local, 0, d.dist.packed_all) && threadIdx.x == 0) {
    d.st_->done = 1;
    d.st_->status = -9;
  }
}

__global__ void k_slab_unpack(GridParams g, DevPtrs d, double* v, int K) {
  const DistPtrs& dd = d.dist;
  const int slot = (int)(*dd.seq & 1ull);
  const int nt2 = g.nt / 2;
  const int s0 = dd.rank > 0 ? 0 : 1, s1 = dd.rank < dd.world - 1 ? 2 : 1;
  const int per_side = K * SLAB_HALO;
  for (int q = blockIdx.x; q < (s1 - s0) * per_side; q += gridDim.x) {
    const int side = s0 + q / per_side;                            // 0: rows below y0, 1: from y1 up
    const int ri = (q % per_side) % SLAB_HALO, k = (q % per_side) / SLAB_HALO;
    const int row = side == 0 ? g.y0 - SLAB_HALO + ri : g.y1 + ri;
    const double2* src = reinterpret_cast<const double2*>(dd.halo_in[dd.rank] + halo_ofs(slot, side, 0, K, k, ri, g.nt));
    double2* dst = reinterpret_cast<double2*>(v + fofs(g, k) + (long long)row * g.nt);
    for (int c2 = threadIdx.x; c2 < nt2; c2 += blockDim.x) dst[c2] = src[c2];
  }
}

// Row-slab variant that unpacks an iteration's two halo vectors into the fields' halo rows
// (DistPtrs.rows == 2): the next k_sr then streams every row from the fields.
__global__ void k_slab_unpack2(GridParams g, DevPtrs d, double* v0, double* v1, int K) {
  const DistPtrs& dd = d.dist;
  if (d.st_->done) return;
  const int slot = (int)(*dd.seq & 1ull);
  const int nt2 = g.nt / 2;
  const int s0 = dd.rank > 0 ? 0 : 1, s1 = dd.rank < dd.world - 1 ? 2 : 1;
  const int per_side = 2 * K * SLAB_HALO;
  for (int q = blockIdx.x; q < (s1 - s0) * per_side; q += gridDim.x) {
    const int side = s0 + q / per_side;
    const int e = q % per_side;
    const int ri = e % SLAB_HALO, k = (e / SLAB_HALO) % K, vec = e / (SLAB_HALO * K);
    const int row = side == 0 ? g.y0 - SLAB_HALO + ri : g.y1 + ri;
    const double2* src = reinterpret_cast<const double2*>(dd.halo_in[dd.rank] + halo_ofs(slot, side, vec, K, k, ri, g.nt));
    double2* dst = reinterpret_cast<double2*>((vec ? v1 : v0) + fofs(g, k) + (long long)row * g.nt);
    for (int c2 = threadIdx.x; c2 < nt2; c2 += blockDim.x) dst[c2] = src[c2];
  }
}

// CTAs of the exchange kernels: one per halo row to send (at most 2 per SM); one for a single
// rank (nothing to push, only the gather).
static int slab_blocks(const GridParams& g, const DevPtrs& d, int K, int nv) {
  (void)g;
  if (d.dist.world <= 1) return 1;
  const int rows = 2 * nv * K * SLAB_HALO;
  return rows < 296 ? rows : 296;
}

cudaError_t launch_p2p_rows(const GridParams& g, const DevPtrs& d, bool init, int parity, int K,
                            unsigned long long h, cudaStream_t s) {
  const int use = h != 0ull;
  if (init) k_p2p_rows<true><<<slab_blocks(g, d, K, 2), 256, 0, s>>>(g, d, parity, K, h, use);
  else k_p2p_rows<false><<<slab_blocks(g, d, K, 2), 256, 0, s>>>(g, d, parity, K, h, use);
  return cudaGetLastError();
}

cudaError_t launch_slab_unpack2(const GridParams& g, const DevPtrs& d, bool init, int parity, int K,
                                cudaStream_t s) {
  double* v0 = init ? d.r[0] : d.r[1 - parity];
  double* v1 = init ? d.u[1] : d.u[parity];
  k_slab_unpack2<<<slab_blocks(g, d, K, 2), 256, 0, s>>>(g, d, v0, v1, K);
  return cudaGetLastError();
}

cudaError_t launch_slab_exchange(const GridParams& g, const DevPtrs& d, double* v, int K, cudaStream_t s) {
  k_slab_push<<<slab_blocks(g, d, K, 1), 256, 0, s>>>(g, d, v, K);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_slab_unpack<<<slab_blocks(g, d, K, 1), 256, 0, s>>>(g, d, v, K);
  return cudaGetLastError();
}

cudaError_t launch_p2p_scalar(const DevPtrs& d, bool init, int Klocal, unsigned long long h, cudaStream_t s) {
  const int use = h != 0ull;
  if (init) k_p2p_scalar<true><<<1, 32, 0, s>>>(d, Klocal, h, use);   // one warp
  else k_p2p_scalar<false><<<1, 32, 0, s>>>(d, Klocal, h, use);
  return cudaGetLastError();
}

cudaError_t launch_sr_fixup(const GridParams& g, const DevPtrs& d, int K, cudaStream_t s) {
  const long long work = (long long)g.nt * (g.y1 - g.y0) * K;
  long long blocks = (work + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_sr_fixup<<<(int)blocks, 256, 0, s>>>(g, d, K);
  return cudaGetLastError();
}

cudaError_t launch_sr_scalar(const DevPtrs& d, bool init, int Kglob, int Klocal, int kofs, int world,
                             cudaStream_t s) {
  const size_t sm = (size_t)4 * Kglob * sizeof(double);
  if (init) k_sr_scalar<true><<<1, 128, sm, s>>>(d, Kglob, Klocal, kofs, world);
  else k_sr_scalar<false><<<1, 128, sm, s>>>(d, Kglob, Klocal, kofs, world);
  return cudaGetLastError();
}

template <typename KernelT>
static cudaError_t sr_set(KernelT kern, int) {
  return raise_smem_cap(kern);
}

template <int MODE>
static cudaError_t sr_set_modes(int bytes) {
  cudaError_t e = sr_set(k_sr<SPC_ASSOR2, MODE>, bytes);
  if (e == cudaSuccess) e = sr_set(k_sr<SPC_ASSOR2, MODE, 512>, bytes);
  if (e == cudaSuccess) e = sr_set(k_sr<SPC_ASSOR2, MODE, 256>, bytes);
  if (e == cudaSuccess) e = sr_set(k_sr<SPC_ASSOR1, MODE>, bytes);
  if (e == cudaSuccess) e = sr_set(k_sr<SPC_JACOBI, MODE>, bytes);
  if (e == cudaSuccess) e = sr_set(k_sr<SPC_NONE, MODE>, bytes);
  return e;
}

// The dynamic shared-memory cap is a process-wide attribute of each kernel while the sizes differ
// per context (strip width, K): every kernel is raised once to the device's opt-in maximum (the
// cap only bounds a launch; occupancy follows the bytes actually requested), so a context created
// later can never lower the cap under an earlier one.  Fails if this context needs
// more than the device offers.
cudaError_t configure_sr_kernels(const TileCfg& t, int K) {
  const int cap = smem_optin_max();
  if (cap <= 0) return cudaErrorInvalidValue;
  if ((long long)sr_smem_bytes(2 * sr_pairs(t)) > cap - 1024) return cudaErrorInvalidValue;
  static unsigned done = 0u;   // host-side, once per device (the attribute is process-global)
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cudaErrorInvalidValue;
  if (done & (1u << dev)) return cudaSuccess;
  cudaError_t e = sr_set_modes<SR_ITER_EVEN>(cap);
  if (e == cudaSuccess) e = sr_set_modes<SR_ITER_ODD>(cap);
  if (e == cudaSuccess) e = sr_set_modes<SR_INIT_COLD>(cap);
  if (e == cudaSuccess) e = sr_set_modes<SR_INIT_WARM>(cap);
  if (e == cudaSuccess) e = sr_set(k_srp<SPC_ASSOR2, true, false>, cap);
  if (e == cudaSuccess) e = sr_set(k_srp<SPC_ASSOR2, false, false>, cap);
  if (e == cudaSuccess) e = sr_set(k_srp<SPC_ASSOR2, false, false, 512>, cap);
  if (e == cudaSuccess) e = sr_set(k_srp<SPC_ASSOR2, false, false, 256>, cap);
  if (e == cudaSuccess) e = sr_set(k_srp<SPC_ASSOR1, false, false>, cap);
  if (e == cudaSuccess) e = sr_set(k_srp<SPC_JACOBI, false, false>, cap);
  if (e == cudaSuccess) e = sr_set(k_srp<SPC_NONE, false, false>, cap);
  if (e == cudaSuccess) e = sr_set(k_srp<SPC_ASSOR1, false, false, 512>, cap);
  if (e == cudaSuccess) e = sr_set(k_srp<SPC_JACOBI, false, false, 512>, cap);
  if (e == cudaSuccess) e = sr_set(k_srp<SPC_NONE, false, false, 512>, cap);
  if (e == cudaSuccess) e = sr_set(k_srp<SPC_ASSOR1, false, false, 256>, cap);
  if (e == cudaSuccess) e = sr_set(k_srp<SPC_JACOBI, false, false, 256>, cap);
  if (e == cudaSuccess) e = sr_set(k_srp<SPC_NONE, false, false, 256>, cap);
  if (e == cudaSuccess) e = sr_set(k_srp<SPC_ASSOR2, false, true>, cap);
  if (e == cudaSuccess) e = sr_set(k_srp<SPC_ASSOR2, false, true, 512>, cap);
  if (e == cudaSuccess) e = sr_set(k_srp<SPC_ASSOR2, false, true, 256>, cap);
  if (e == cudaSuccess) e = sr_set(k_srp<SPC_ASSOR1, false, true>, cap);
  if (e == cudaSuccess) e = sr_set(k_srp<SPC_JACOBI, false, true>, cap);
  if (e == cudaSuccess) e = sr_set(k_srp<SPC_NONE, false, true>, cap);
  (void)K;
  if (e == cudaSuccess) done |= 1u << dev;
  return e;
}

// whether the persistent kernel fits this context (its extra shared memory grows with K)
bool srp_fits(const TileCfg& t, int K, int Kall) {
  return (long long)srp_smem_bytes(2 * sr_pairs(t), K, t.n_tiles * K, Kall) <= smem_optin_max() - 1024;
}

int sr_ctas_per_sm(const TileCfg& t) {
  int n = 0;
  const int threads = sr_threads(t);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_sr<SPC_ASSOR2, SR_ITER_ODD>, threads,
                                                    sr_smem_bytes(2 * sr_pairs(t))) != cudaSuccess)
    return 1;
  return n;
}

}  // namespace gmaf
