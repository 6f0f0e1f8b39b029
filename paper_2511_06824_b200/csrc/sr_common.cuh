// sr_common.cuh -- pieces shared by the two single-reduction PCG-ASSOR-II iteration kernels
// (today sr.cu; kept apart so a second iteration kernel can share them):
// PTX wrappers (mbarrier, TMA bulk copy, named barrier), column-pair helpers, the Table-1 /
// Chronopoulos-Gear scalar stage and the per-launch reduction tail.
#pragma once
#include <cstdint>
#include "device_common.cuh"
#include "gmaf_internal.cuh"

namespace gmaf {

enum { SR_ITER_EVEN = 0, SR_ITER_ODD = 3, SR_INIT_COLD = 1, SR_INIT_WARM = 2,
       SR_ITER_ANY = 4 /* either parity, decided at run time (persistent kernel) */ };
enum { SPC_NONE = 0, SPC_JACOBI = 1, SPC_ASSOR2 = 2, SPC_ASSOR1 = 3 };   // = GMAF_PRECOND_*

// ------------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// consumers: spin on try_wait (the data is normally already there)
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try(bar, parity)) {
  }
}
// producer: back off so a waiting producer does not steal issue slots from the compute warps
#ifndef GMAF_PRODUCER_SLEEP_NS
#define GMAF_PRODUCER_SLEEP_NS 128
#endif
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
  while (!mbar_try(bar, parity)) __nanosleep(GMAF_PRODUCER_SLEEP_NS);
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
// named barrier 1 over the compute warps only (the producer warp never joins it)
__device__ __forceinline__ void compute_bar(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}
// timing-only experiment (wrong results): the row pipeline's two barriers per row compiled out
#ifdef GMAF_EXPERIMENT_NOBAR
template <bool SHARED = false>
__device__ __forceinline__ void row_bar(int) { __syncwarp(); }
#else
// SHARED: the split seam loops (different barrier instructions in the seam warp and the others)
// use the NON-aligned form barrier.sync, which PTX allows to be reached from different
// instructions (bar.sync = barrier.sync.aligned requires the same instruction in every thread)
__device__ __forceinline__ void compute_bar_unaligned(int nthreads) {
  asm volatile("barrier.sync 1, %0;" ::"r"(nthreads) : "memory");
}
template <bool SHARED = false>
__device__ __forceinline__ void row_bar(int nthreads) {
  if constexpr (SHARED) compute_bar_unaligned(nthreads);
  else compute_bar(nthreads);
}
#endif
// 1/a to full double precision without the IEEE-division slow path: rcp.approx (MUFU)
// + one third-order Newton step (the solve does not need a correctly rounded D^-1).
__device__ __forceinline__ double fast_rcp(double a) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
  // one third-order Newton step r (1 + e + e^2), e = 1 - a r: the ~2^-22 approximation
  // becomes ~2^-66 in 3 dependent FMAs (two second-order steps need 4)
  const double e = fma(-a, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

// Explicitly rounded products and sums: every kernel variant (per-launch, persistent, compile-time
// or runtime strip width, seam variants) must round the same expressions the same way, so the row
// pipeline spells out each multiply, add and fused multiply-add instead of leaving the contraction
// of a*b + c*d to the compiler (which may contract differently in differently shaped kernels).
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

struct D2 { double l, r; };
__device__ __forceinline__ D2 ld2(const double* base, int t) {
  const double2 v = reinterpret_cast<const double2*>(base)[t];
  return {v.x, v.y};
}
__device__ __forceinline__ void st2(double* base, int t, D2 v) {
  reinterpret_cast<double2*>(base)[t] = make_double2(v.l, v.r);
}
// Derived rings use a split layout [even columns | odd columns] (NTC doubles each) so that
// the theta neighbours of a pair are contiguous across lanes (2 wavefronts, no conflicts).
__device__ __forceinline__ void rst(double* base, int t, int ntc, D2 v) { base[t] = v.l; base[ntc + t] = v.r; }
__device__ __forceinline__ D2 rld(const double* base, int t, int ntc) { return {base[t], base[ntc + t]}; }
__device__ __forceinline__ double rleft(const double* base, int t, int ntc) { return base[ntc + t - 1]; }
__device__ __forceinline__ double rright(const double* base, int t) { return base[t + 1]; }
// value of the pair to the left (its right column) of a coefficient row: a warp shuffle of the
// register copy, or the shared-memory element where the shuffle cannot supply it
__device__ __forceinline__ double left_of(double own_r, const double* row, int im, bool from_smem) {
  const double v = __shfl_up_sync(0xffffffffu, own_r, 1);
  return from_smem ? row[im] : v;
}
__device__ __forceinline__ void stg2(double* p, D2 v) {   // 16-byte global store (pairs are aligned)
  *reinterpret_cast<double2*>(p) = make_double2(v.l, v.r);
}
// the same store predicated on p (one predicated instruction, no branch); not ordered against other
// memory operations by the compiler -- the row loop's outputs are read only after the grid barrier
// (or the kernel boundary), whose fences are asm statements with memory clobbers
__device__ __forceinline__ void stg2_if(bool p, double* ptr, D2 v) {
  asm volatile(
      "{\n"
      ".reg .pred q;\n"
      "setp.ne.b32 q, %0, 0;\n"
      "@q st.global.v2.f64 [%1], {%2, %3};\n"
      "}\n" ::"r"((int)p),
      "l"(ptr), "d"(v.l), "d"(v.r));
}

// Table-1 scalars from the per-condition sums (fixed k order): convergence test (Eq. 3.9),
// alpha/beta of the single-reduction recurrence (coupled: global; lockstep: per condition).
// red = [rr | gamma | delta | S.S] x Kall.  Local conditions kofs .. kofs+Klocal-1 receive their
// alpha/beta in cs (indexed locally).  One thread.
// Asynchronous strategy (Eq. 3.10): every condition is its own Krylov process
// (per-condition alpha_k, beta_k) frozen at its own test ||r_k||/||S_k|| <= tol; the solve ends
// when all are frozen.  A frozen condition's CTAs no longer stream or compute (device mask, no
// host round trip -- the cost the paper's implementation paid).  One rank (Kall == Klocal).
template <bool INIT>
__device__ void sr_scalar_async(const CondScalars& cs, SolverState* st, const double* red, int K) {
  const double* rrk = red;
  const double* gk = red + K;
  const double* dk = red + 2 * K;
  const double* ssk = red + 3 * K;
  bool bad = false;
  if (INIT) {
    double SS = 0.0;
    for (int k = 0; k < K; ++k) SS += ssk[k];
    st->nS = sqrt(SS);
    st->iter = 0; st->status = 0; st->converged = 0; st->done = 0; st->zero_p = (st->nS == 0.0);
    for (int k = 0; k < K; ++k) {
      cs.Sk[k] = ssk[k]; cs.rrk[k] = rrk[k]; cs.itk[k] = 0;
      const double relk = ssk[k] > 0.0 ? sqrt(rrk[k]) / sqrt(ssk[k]) : 0.0;
      cs.frz[k] = (ssk[k] == 0.0 || relk <= st->tol) ? 1 : 0;
      double a0 = 0.0;
      if (!cs.frz[k] && gk[k] != 0.0) { if (!(dk[k] > 0.0)) bad = true; a0 = gk[k] / dk[k]; }
      cs.alpha[k] = a0; cs.beta[k] = 0.0; cs.uvk[k] = 0.0; cs.dk[k] = gk[k];
    }
  } else {
    st->iter += 1;
    for (int k = 0; k < K; ++k) {
      if (cs.frz[k]) continue;
      cs.itk[k] += 1;
      cs.rrk[k] = rrk[k];
      cs.uvk[k] = cs.alpha[k];                       // alpha used this iteration
      const double relk = cs.Sk[k] > 0.0 ? sqrt(rrk[k]) / sqrt(cs.Sk[k]) : 0.0;
      if (relk <= st->tol) { cs.frz[k] = 1; continue; }
      const double aold = cs.alpha[k], gold = cs.dk[k];
      double a = 0.0, b = 0.0;
      if (gold != 0.0 && aold != 0.0) {
        if (gk[k] < 0.0) bad = true;
        b = gk[k] / gold;
        const double den = dk[k] - b * gk[k] / aold;
        if (den > 0.0) a = (gk[k] == 0.0) ? 0.0 : gk[k] / den;
        else if (dk[k] > 0.0) { b = 0.0; a = gk[k] / dk[k]; }   // restart (R-A32)
        else bad = true;
      }
      cs.alpha[k] = a; cs.beta[k] = b; cs.dk[k] = gk[k];
    }
  }
  double rr = 0.0;
  int live = 0;
  for (int k = 0; k < K; ++k) { rr += cs.rrk[k]; live += cs.frz[k] ? 0 : 1; }
  st->rel = st->nS > 0.0 ? sqrt(rr) / st->nS : 0.0;
  if (live == 0) { st->done = 1; st->converged = 1; }
  else if (st->iter >= st->max_iter) { st->done = 1; st->status = -6; }
  if (bad && !st->done) { st->done = 1; st->status = -5; }
}

// Solver-state snapshot for the scalar stage, loaded early (overlapped with the partial-sum loads
// of the serial tail): the stage itself then makes no dependent global round trip.
struct StageIn { SolverState s; double aold0; };
__device__ __forceinline__ StageIn stage_prefetch(const CondScalars& cs, const SolverState* st) {
  StageIn in;
  in.s = *st;
  in.aold0 = cs.alpha[0];
  return in;
}
__device__ __forceinline__ StageIn stage_prefetch(const DevPtrs& d) { return stage_prefetch(d.cs, d.st_); }

// Executed by ONE THREAD on the critical path of every iteration (a warp-parallel version, with
// lanes evaluating the scalars redundantly and storing the per-condition arrays lane-parallel,
// was reverted: lanes read alpha[0] and the state while lane 0 was writing them, which corrupted
// the lockstep scalars for K = 2, 3 -- DESIGN.md sec. 9).  cs / st are the per-condition arrays
// and the solver state: global memory (d.cs, d.st_) for the per-launch kernels, CTA-private
// shared-memory copies in the persistent kernel.
template <bool INIT>
__device__ void sr_scalar_stage(const CondScalars& cs, SolverState* st, const double* red, int Kall, int Klocal,
                                int kofs, int use_cond, unsigned long long hcond, const StageIn& in) {
  // one thread on the critical path of every iteration: work on the register snapshot, write the
  // state back once
  SolverState s = in.s;
  const double aold0 = in.aold0;
  if (s.coupling == 2) {
    sr_scalar_async<INIT>(cs, st, red, Kall);
    if (use_cond && st->done) cudaGraphSetConditional((cudaGraphConditionalHandle)hcond, 0u);
    return;
  }
  const double* rrk = red;
  const double* gk = red + Kall;
  const double* dk = red + 2 * Kall;
  const double* ssk = red + 3 * Kall;
  double rr = 0.0;
  for (int kk = 0; kk < Kall; ++kk) rr += rrk[kk];
  for (int kl = 0; kl < Klocal; ++kl) cs.rrk[kl] = rrk[kofs + kl];
  bool bad = false;
  if (INIT) {
    double SS = 0.0;
    for (int kk = 0; kk < Kall; ++kk) SS += ssk[kk];
    for (int kl = 0; kl < Klocal; ++kl) cs.Sk[kl] = ssk[kofs + kl];
    s.nS = sqrt(SS);
    s.iter = 0; s.status = 0; s.converged = 0; s.done = 0; s.zero_p = 0;
    if (s.nS == 0.0) {
      s.rel = 0.0; s.done = 1; s.converged = 1; s.zero_p = 1;
    } else {
      s.rel = sqrt(rr) / s.nS;
      if (s.fixed_iters == 0 && s.rel <= s.tol) { s.done = 1; s.converged = 1; }
      else if (s.max_iter <= 0) { s.done = 1; s.status = -6; }
    }
    if (!s.done) {
      if (s.coupling == 0) {
        double gg = 0.0, dd = 0.0;
        for (int kk = 0; kk < Kall; ++kk) { gg += gk[kk]; dd += dk[kk]; }
        if (!(dd > 0.0)) bad = true;
        const double a0 = gg / dd;
        for (int kl = 0; kl < Klocal; ++kl) { cs.alpha[kl] = a0; cs.beta[kl] = 0.0; cs.uvk[kl] = 0.0; }
        s.d = gg;
      } else {
        for (int kk = 0; kk < Kall; ++kk)
          if (gk[kk] != 0.0 && !(dk[kk] > 0.0)) bad = true;
        for (int kl = 0; kl < Klocal; ++kl) {
          const int kk = kofs + kl;
          cs.alpha[kl] = gk[kk] != 0.0 ? gk[kk] / dk[kk] : 0.0;
          cs.beta[kl] = 0.0; cs.uvk[kl] = 0.0; cs.dk[kl] = gk[kk];
        }
      }
#if defined(GMAF_EXPERIMENT_NOTMA) || defined(GMAF_EXPERIMENT_NOBAR)
      bad = false;
#endif
      if (bad) { s.done = 1; s.status = -5; }
    }
  } else {
    s.iter += 1;
    s.rel = sqrt(rr) / s.nS;
    if (s.fixed_iters > 0) {
      if (s.iter >= s.fixed_iters) s.done = 1;
    } else if (s.rel <= s.tol) {
      s.done = 1; s.converged = 1;
    } else if (s.iter >= s.max_iter) {
      s.done = 1; s.status = -6;
    }
    if (!s.done || s.fixed_iters > 0) {
      if (s.coupling == 0) {
        double g2 = 0.0, d2 = 0.0;
        for (int kk = 0; kk < Kall; ++kk) { g2 += gk[kk]; d2 += dk[kk]; }
        double b = g2 / s.d;
        const double den = d2 - b * g2 / aold0;
        // Chronopoulos-Gear denominator: > 0 in exact arithmetic, lost to cancellation near a
        // stagnating direction -> restart along z (beta = 0, exact line search, R-A32)
        double a = 0.0;
        if (!(g2 > 0.0)) bad = true;
        else if (den > 0.0) a = g2 / den;
        else if (d2 > 0.0) { b = 0.0; a = g2 / d2; }
        else bad = true;
        for (int kl = 0; kl < Klocal; ++kl) { cs.uvk[kl] = aold0; cs.alpha[kl] = a; cs.beta[kl] = b; }
        s.d = g2;
      } else {
        for (int kk = 0; kk < Kall; ++kk)
          if (gk[kk] < 0.0) bad = true;
        for (int kl = 0; kl < Klocal; ++kl) {
          const int kk = kofs + kl;
          const double aold = cs.alpha[kl], gold = cs.dk[kl];
          cs.uvk[kl] = aold;                                   // alpha used this iteration
          double a = 0.0, b = 0.0;
          if (gold != 0.0 && aold != 0.0) {
            b = gk[kk] / gold;
            const double den = dk[kk] - b * gk[kk] / aold;
            if (den > 0.0) a = (gk[kk] == 0.0) ? 0.0 : gk[kk] / den;
            else if (dk[kk] > 0.0) { b = 0.0; a = gk[kk] / dk[kk]; }   // restart (R-A32)
            else bad = true;
          }
          cs.alpha[kl] = a; cs.beta[kl] = b; cs.dk[kl] = gk[kk];
        }
      }
#if defined(GMAF_EXPERIMENT_NOTMA) || defined(GMAF_EXPERIMENT_NOBAR)
      bad = false;   // timing-only builds: wrong data, run every fixed iteration anyway
#endif
      if (bad && !s.done) { s.done = 1; s.status = -5; }
    } else {
      for (int kl = 0; kl < Klocal; ++kl) cs.uvk[kl] = cs.alpha[kl];   // alpha used this iteration
    }
  }
  *st = s;
  // the WHILE handle defaults to 1 at every graph launch: write it only to stop the loop
  if (use_cond && s.done) cudaGraphSetConditional((cudaGraphConditionalHandle)hcond, 0u);
}

template <bool INIT>
__device__ __forceinline__ void sr_scalar_stage(const DevPtrs& d, const double* red, int Kall, int Klocal,
                                                int kofs, int use_cond, unsigned long long hcond, const StageIn& in) {
  sr_scalar_stage<INIT>(d.cs, d.st_, red, Kall, Klocal, kofs, use_cond, hcond, in);
}
template <bool INIT>
__device__ __forceinline__ void sr_scalar_stage(const DevPtrs& d, const double* red, int Kall, int Klocal,
                                                int kofs, int use_cond, unsigned long long hcond) {
  sr_scalar_stage<INIT>(d.cs, d.st_, red, Kall, Klocal, kofs, use_cond, hcond, stage_prefetch(d));
}


// ---------------------------------------------------------------- multi-rank helpers
// rank and local index of global condition kg (contiguous blocks; the first Kglob % world ranks
// hold one more)
__device__ __forceinline__ void dist_owner(int kg, int Kglob, int world, int* r, int* kl) {
  const int base = Kglob / world, extra = Kglob % world;
  if (kg < extra * (base + 1)) { *r = kg / (base + 1); *kl = kg % (base + 1); }
  else { *r = extra + (kg - extra * (base + 1)) / base; *kl = (kg - extra * (base + 1)) % base; }
}

constexpr long long kP2PTimeoutNs = 10000000000ll;   // 10 s: a peer that never arrives fails the solve

// Peer-to-peer allgather, executed by ONE WARP (all 32 lanes call it; the result is warp-uniform):
// push n doubles of src into slot `rank` of every rank's exchange buffer over NVLink (IPC-mapped
// peer memory, lanes in parallel), publish a monotonically increasing stamp with release
// semantics at system scope (lane r to rank r), wait for every rank's stamp in the own buffer
// (lane r polls rank r), and copy the gathered blocks to dst [world][n].  All ranks issue the same
// sequence of gathers, so their stamps agree; two parity slots keep a rank that runs one gather
// ahead from overwriting a block a slower rank still reads.  Returns false on timeout.
__device__ __forceinline__ bool p2p_gather(const DistPtrs& dd, const double* src, int n, double* dst) {
  const int lane = threadIdx.x & 31;
  const int W = dd.world;
  unsigned long long stamp = 0ull;
  if (lane == 0) {
    stamp = *dd.seq + 1ull;
    *dd.seq = stamp;
  }
  stamp = __shfl_sync(0xffffffffu, stamp, 0);
  const int par = (int)(stamp & 1ull);
  for (int i = lane; i < W * n; i += 32) {
    const int r = i / n, q = i - r * n;
    double* slot = reinterpret_cast<double*>(dd.peer[r] + 2 * W * 8) + ((long long)par * W + dd.rank) * dd.xs;
    *reinterpret_cast<volatile double*>(slot + q) = src[q];
  }
  __threadfence_system();
  __syncwarp();
  bool ok = true;
  if (lane < W) {
    unsigned long long* fl = reinterpret_cast<unsigned long long*>(dd.peer[lane]) + par * W + dd.rank;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(fl), "l"(stamp) : "memory");
    const unsigned long long* my = reinterpret_cast<const unsigned long long*>(dd.peer[dd.rank]) + par * W + lane;
    const unsigned long long t0 = globaltimer();
    for (;;) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(my) : "memory");
      if (v >= stamp) break;
      if ((long long)(globaltimer() - t0) > kP2PTimeoutNs) { ok = false; break; }
    }
  }
  // lane x reads every rank's block, but only lane r acquired rank r's stamp: the warp barrier
  // (bar.warp.sync orders memory among its lanes) plus a system-scope acquire-release fence by
  // every lane orders all the data reads below after all the stamp acquires
  __syncwarp();
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  if (!__all_sync(0xffffffffu, ok)) return false;
  const volatile double* data = reinterpret_cast<const volatile double*>(dd.peer[dd.rank] + 2 * W * 8);
  for (int i = lane; i < W * n; i += 32) {
    const int r = i / n, q = i - r * n;
    dst[i] = data[((long long)par * W + r) * dd.xs + q];
  }
  __syncwarp();
  return true;
}

// Fixed-order CTA sum of NV per-thread values over the first nw warps (the compute warps): an
// xor butterfly in every warp (every lane ends with bitwise the same warp sum: each level adds
// the same two partial sums), lane 0 parks it in wbuf[q*32 + warp], then thread 0 adds the warps
// in order.  The per-launch k_sr and the persistent k_srp both use it, so their per-CTA partials
// -- and hence their scalars -- are bitwise identical.  Warps >= nw must not call it; the caller
// separates the wbuf write from the read with a barrier over the nw warps.
template <int NV>
__device__ __forceinline__ void warp_tree_sum(double (&v)[NV], double* wbuf) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1)
#pragma unroll
    for (int c = 0; c < NV; ++c) v[c] += __shfl_xor_sync(0xffffffffu, v[c], m);
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int c = 0; c < NV; ++c) wbuf[c * 32 + (threadIdx.x >> 5)] = v[c];
}
template <int NV>
__device__ __forceinline__ void warps_in_order(double (&v)[NV], const double* wbuf, int nw) {
#pragma unroll
  for (int c = 0; c < NV; ++c) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += wbuf[c * 32 + w];
    v[c] = s;
  }
}

// The two halves of p2p_gather for the persistent kernel, where ONE warp pushes and EVERY CTA
// waits for and reads the gathered blocks itself (no second hop through a local broadcast).
// p2p_push: this rank's n doubles into slot `rank` of every rank's buffer (parity slot of
// `stamp`), then the stamp with release semantics at system scope; advances *dd.seq.  One warp.
__device__ __forceinline__ void p2p_push(const DistPtrs& dd, const double* src, int n, unsigned long long stamp) {
  const int lane = threadIdx.x & 31;
  const int W = dd.world;
  const int par = (int)(stamp & 1ull);
  for (int i = lane; i < W * n; i += 32) {
    const int r = i / n, qi = i - r * n;
    double* slot = reinterpret_cast<double*>(dd.peer[r] + 2 * W * 8) + ((long long)par * W + dd.rank) * dd.xs;
    *reinterpret_cast<volatile double*>(slot + qi) = src[qi];
  }
  // no per-lane system fence: the warp barrier orders every lane's block stores before lane r's
  // release store of the stamp, and a release is cumulative (it publishes the writes that
  // happen before it in causality order, the other lanes' included)
  __syncwarp();
  if (lane < W) {
    unsigned long long* fl = reinterpret_cast<unsigned long long*>(dd.peer[lane]) + par * W + dd.rank;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(fl), "l"(stamp) : "memory");
  }
  if (lane == 0) *dd.seq = stamp;
}
// p2p_stamps_wait: every rank's stamp >= `stamp` in the own buffer (acquire, system scope); one
// thread, followed by a barrier of the threads that read the blocks.  false on timeout.
__device__ __forceinline__ bool p2p_stamps_wait(const DistPtrs& dd, unsigned long long stamp) {
  const int par = (int)(stamp & 1ull);
  const unsigned long long t0 = globaltimer();
  for (int r = 0; r < dd.world; ++r) {
    const unsigned long long* fl = reinterpret_cast<const unsigned long long*>(dd.peer[dd.rank]) + par * dd.world + r;
    for (;;) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(fl) : "memory");
      if (v >= stamp) break;
      if ((long long)(globaltimer() - t0) > kP2PTimeoutNs) return false;
    }
  }
  return true;   // the caller's CTA barrier orders its threads' block reads after these acquires
}
// element qi of rank r's block of the gather `stamp`, from the own exchange buffer
__device__ __forceinline__ double p2p_block(const DistPtrs& dd, unsigned long long stamp, int r, int qi) {
  const int par = (int)(stamp & 1ull);
  const double* data = reinterpret_cast<const double*>(dd.peer[dd.rank] + 2 * dd.world * 8);
  return __ldcg(data + ((long long)par * dd.world + r) * dd.xs + qi);
}

// Per-CTA partials -> fixed-order per-condition sums in the last CTA -> the scalar stage
// (multi-rank: the packed sums for the allgather).  Every thread of the CTA calls it; `red`
// is dead shared memory of >= max(4 * (blockDim + 32), 4 * K) doubles.
template <bool ITER, bool INIT>
__device__ void sr_finish(const DevPtrs& d, double (&v)[4], double* red, int K, int k, int ncta, int cta,
                          unsigned long long hcond, int use_cond, int ncompute_warps) {
  const int tid = threadIdx.x;
  __syncthreads();                                   // the rings are dead: red may alias them
  if ((tid >> 5) < ncompute_warps) warp_tree_sum<4>(v, red);
  __syncthreads();
  if (tid == 0) warps_in_order<4>(v, red, ncompute_warps);
  if (tid == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) d.partials[(long long)(q * K + k) * ncta + cta] = v[q];
  }
  if (last_cta_arrive(&d.counters[ITER ? KK_SR_ITER : KK_SR_INIT], gridDim.x)) {
    const unsigned long long t_tail = (ITER && tid == 0) ? globaltimer() : 0ull;
    // thread 0 prefetches what the scalar stage and the timing need (overlaps the loads below)
    StageIn in{};
    unsigned long long t_start0 = 0ull;
    if (tid == 0) {
      in = stage_prefetch(d);
      t_start0 = d.timing->t_start[ITER ? KK_SR_ITER : KK_SR_INIT];
    }
    // per-condition sums in CTA order: [rr | gamma | delta | S.S] x K; all loads of a sum in
    // flight at once (one L2 round trip on this serial tail), adds in CTA order
    for (int q = tid; q < 4 * K; q += blockDim.x) {
      const double* srcp = d.partials + (long long)q * ncta;
      double sum = 0.0;
#pragma unroll 32
      for (int b = 0; b < ncta; ++b) sum += __ldcg(srcp + b);
      red[q] = sum;
    }
    __syncthreads();
    if (d.dist.world == 0 && tid == 0) sr_scalar_stage<INIT>(d, red, K, K, 0, use_cond, hcond, in);
    if (tid == 0) {
      if (d.dist.world > 0) {
        // multi-rank: publish this rank's per-condition sums
        const int km = d.dist.kmax_local;
        for (int q = 0; q < 4; ++q)
          for (int kk = 0; kk < km; ++kk) d.dist.packed_local[q * km + kk] = kk < K ? red[q * K + kk] : 0.0;
        // NCCL mode: the allgather + k_sr_scalar follow on the stream; peer-to-peer mode:
        // k_p2p_scalar follows in the same graph
      }
      timing_end(d.timing, ITER ? KK_SR_ITER : KK_SR_INIT, t_start0);
      if (ITER) {   // the serial tail: all other CTAs have finished when the last one arrives
        atomicAdd(&d.timing->total_ns[KK_SR_TAIL], globaltimer() - t_tail);
        atomicAdd(&d.timing->launches[KK_SR_TAIL], 1ull);
      }
    }
  }
}

}  // namespace gmaf
