// pcg.cu -- the PCG-ASSOR-II iteration of the joint K-condition system (Table 1,
// PAPER.md:73-83, sign of r0 fixed; Eqs. 3.5-3.6 two-step ASSOR; Eq. 3.9 synchronized
// convergence) as two fused, y-marching stencil kernels per iteration on sm_100a.
//
// Tiling: a CTA owns a strip of TW output columns (plus HALO = 3
// columns on each side, one thread per loaded column) of one condition k and marches
// over a chunk of TH output rows.  Rows are streamed once from HBM; row neighbours
// (j-1, j+1) live in registers, theta neighbours in a 4-slot shared-memory ring.  The
// per-CTA partial dot products are reduced in a fixed order by the last CTA to finish,
// which also computes alpha/beta and the global convergence test and drives the CUDA
// graph's WHILE node.  Every result is deterministic run to run.
//
//   phase A (Table 1 steps 7-9 + 3): z = M^-1 r (recomputed), u = z + beta u,
//            v = A u (not stored), partial u.v  ->  alpha
//   phase B (steps 4-6 + 7-8):      p += alpha u, r -= alpha A u (A u recomputed),
//            partial r.r, z = M^-1 r (recomputed), partial r.z -> test, beta
#include <cstdint>
#include "device_common.cuh"
#include "gmaf_internal.cuh"

namespace gmaf {

enum { PC_NONE = 0, PC_JACOBI = 1, PC_ASSOR2 = 2 };
enum { MODE_ITER = 0, MODE_INIT_COLD = 1, MODE_INIT_WARM = 2, MODE_TRUERES = 3 };

struct TileCtx {
  int k, i0, j0, j1, tl, gc, tm, tp;
  bool out_col, w0col, endcol;
};

__device__ __forceinline__ TileCtx tile_ctx(const GridParams& g, const TileCfg& t, int K) {
  TileCtx c;
  c.k = blockIdx.x % K;
  const int tile = blockIdx.x / K;
  const int strip = tile % t.n_strips, chunk = tile / t.n_strips;
  c.i0 = strip * t.tw;
  c.j0 = g.y0 + chunk * t.th;          // own rows [y0, y1) (all rows on one rank)
  c.j1 = min(c.j0 + t.th, g.y1);
  c.tl = threadIdx.x;
  int gc = (c.i0 - HALO + c.tl) % g.nt;
  if (gc < 0) gc += g.nt;
  c.gc = gc;
  c.tm = max(c.tl - 1, 0);
  c.tp = min(c.tl + 1, (int)blockDim.x - 1);
  c.out_col = (c.tl >= HALO) && (c.tl < HALO + t.tw) && (c.i0 + c.tl - HALO < g.nt);
  c.w0col = (gc == 0);            // its W neighbour is the wrap: belongs to U (R-A12)
  c.endcol = (gc == g.nt - 1);    // its E neighbour is the wrap: belongs to L
  return c;
}

// Shared ring: 4 slots x {AE, first-stage (w), second-stage (v1), vector (u)}.
struct Ring {
  double* ae; double* w; double* v; double* u; int nl;
  __device__ __forceinline__ double& AE(int row, int t) { return ae[(row & 3) * nl + t]; }
  __device__ __forceinline__ double& W(int row, int t) { return w[(row & 3) * nl + t]; }
  __device__ __forceinline__ double& V(int row, int t) { return v[(row & 3) * nl + t]; }
  __device__ __forceinline__ double& U(int row, int t) { return u[(row & 3) * nl + t]; }
};

__device__ __forceinline__ Ring make_ring(double* smem) {
  Ring r;
  r.nl = blockDim.x;
  r.ae = smem;
  r.w = smem + 4 * r.nl;
  r.v = smem + 8 * r.nl;
  r.u = smem + 12 * r.nl;
  for (int q = threadIdx.x; q < 16 * r.nl; q += blockDim.x) smem[q] = 0.0;
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------- scalar stage
// Executed by the last CTA of each kernel: fixed-order reduction of the per-CTA
// partials partials[q][k][cta], then the Table-1 scalars.
__device__ void reduce_partials(const DevPtrs& d, int nq, int K, int ncta, double* out /*smem nq*K*/) {
  for (int t = threadIdx.x; t < nq * K; t += blockDim.x) {
    const double* src = d.partials + (long long)t * ncta;
    double s = 0.0;
    for (int b = 0; b < ncta; ++b) s += __ldcg(src + b);
    out[t] = s;
  }
  __syncthreads();
}

// The WHILE handle's default value (1) is applied at every graph launch, so the condition is
// only ever written to stop the loop: no device-runtime call on a continuing iteration.
__device__ __forceinline__ void set_cond(bool use, unsigned long long h, bool keep_going) {
  if (use && !keep_going) cudaGraphSetConditional((cudaGraphConditionalHandle)h, 0u);
}

// ------------------------------------------------------------------ phase A
template <int PC>
__global__ void __launch_bounds__(288, 3)
k_phase_a(GridParams g, DevPtrs d, TileCfg t, int K, int parity, unsigned long long hcond, int use_cond) {
  extern __shared__ double smem[];
  SolverState* st = d.st_;
  if (st->done) return;
  timing_begin(d.timing, KK_PHASE_A);
  Ring R = make_ring(smem);
  const TileCtx c = tile_ctx(g, t, K);
  const int m = d.cp[c.k].mat;
  const double* __restrict__ AP = d.AP + fofs(g, m);
  const double* __restrict__ AE = d.AE + fofs(g, m);
  const double* __restrict__ AN = d.AN + fofs(g, m);
  const double* __restrict__ r = d.r[parity] + fofs(g, c.k);
  const double* __restrict__ uold = d.u[1 - parity] + fofs(g, c.k);
  double* __restrict__ u = d.u[parity] + fofs(g, c.k);
  const bool first = (st->iter == 0);
  const double beta = first ? 0.0 : d.cs.beta[c.k];
  const double omega = st->omega;
  const double c2 = (2.0 - omega) * omega;

  // own-column history (rows jl-1, jl-2, jl-3); out-of-range rows are (AP=1, rest 0)
  double AP1 = 1.0, AP2 = 1.0, AE1 = 0.0, AE2 = 0.0, AN1 = 0.0, AN2 = 0.0, AN3 = 0.0;
  double w1 = 0.0, v1 = 0.0, uo1 = 0.0, u2 = 0.0, u3 = 0.0;
  double acc = 0.0;
  for (int jl = c.j0 - 2; jl <= c.j1 + 1; ++jl) {
    double r0 = 0.0, uo0 = 0.0, AP0 = 1.0, AE0 = 0.0, AN0 = 0.0;
    if (jl >= 0 && jl < g.ny) {
      const long long q = (long long)jl * g.nt + c.gc;
      r0 = r[q]; AP0 = AP[q]; AE0 = AE[q]; AN0 = AN[q];
      if (!first) uo0 = uold[q];
    }
    const double inv0 = 1.0 / AP0;
    R.AE(jl, c.tl) = AE0;
    double z1;   // z at row jl-1
    if constexpr (PC == PC_ASSOR2) {
      const double w0 = r0 * inv0;                    // D^-1 r
      R.W(jl, c.tl) = w0;
      __syncthreads();   // the only barrier per row (4-slot ring)
      // v1(jl) = w - (omega/D) * sum_{L} A w   (Eq. 3.5)
      double sL = AN1 * w1;                            // S
      if (c.gc >= 1) sL += R.AE(jl, c.tm) * R.W(jl, c.tm);   // W
      if (c.endcol) sL += AE0 * R.W(jl, c.tp);               // E-wrap
      const double v0 = w0 - (omega * inv0) * sL;
      R.V(jl, c.tl) = v0;
      // z(jl-1) = c2 (v1 - (omega/D) sum_{U} A v1)   (Eq. 3.6); V(jl-1) was written last row
      double sU = AN1 * v0;                            // N
      if (!c.endcol) sU += AE1 * R.V(jl - 1, c.tp);           // E
      if (c.w0col) sU += R.AE(jl - 1, c.tm) * R.V(jl - 1, c.tm);  // W-wrap
      z1 = c2 * (v1 - (omega / AP1) * sU);
      w1 = w0; v1 = v0;
    } else if constexpr (PC == PC_JACOBI) {
      __syncthreads();
      z1 = w1;            // w1 holds D^-1 r of row jl-1
      w1 = r0 * inv0;
    } else {
      __syncthreads();
      z1 = w1;
      w1 = r0;
    }
    const double un1 = first ? z1 : z1 + beta * uo1;   // Table 1 step 9
    if (c.out_col && jl - 1 >= c.j0 && jl - 1 < c.j1) u[(long long)(jl - 1) * g.nt + c.gc] = un1;
    R.U(jl - 1, c.tl) = un1;
    // v(jl-2) = A u (Eq. 2.4), summed P, W, E, S, N; U(jl-2) was written last row
    double vv = AP2 * u2;
    vv += R.AE(jl - 2, c.tm) * R.U(jl - 2, c.tm);
    vv += AE2 * R.U(jl - 2, c.tp);
    vv += AN3 * u3;
    vv += AN2 * un1;
    if (c.out_col && jl - 2 >= c.j0 && jl - 2 < c.j1) acc += u2 * vv;
    u3 = u2; u2 = un1; uo1 = uo0;
    AP2 = AP1; AP1 = AP0; AE2 = AE1; AE1 = AE0; AN3 = AN2; AN2 = AN1; AN1 = AN0;
  }
  double v[1] = {acc};
  block_sum<1>(v, smem);
  const int ncta = t.n_tiles;
  const int cta = blockIdx.x / K;
  if (threadIdx.x == 0) d.partials[(long long)c.k * ncta + cta] = v[0];
  if (last_cta_arrive(&d.counters[KK_PHASE_A], gridDim.x)) {
    double* red = smem;   // K values
    reduce_partials(d, 1, K, ncta, red);
    if (threadIdx.x == 0) {
      bool bad = false;
      if (st->coupling == 0) {
        double uv = 0.0, dd = 0.0;
        for (int k = 0; k < K; ++k) { uv += red[k]; d.cs.uvk[k] = red[k]; }
        dd = st->d;
        if (!(uv > 0.0)) bad = true;
        const double alpha = dd / uv;
        for (int k = 0; k < K; ++k) d.cs.alpha[k] = alpha;
      } else {
        for (int k = 0; k < K; ++k) {
          d.cs.uvk[k] = red[k];
          double a = 0.0;
          if (d.cs.dk[k] != 0.0) {
            if (!(red[k] > 0.0)) bad = true;
            a = d.cs.dk[k] / red[k];
          }
          d.cs.alpha[k] = a;
        }
      }
      if (bad) {
        st->done = 1; st->status = -5; st->converged = 0;
        set_cond(use_cond, hcond, false);
      }
      timing_end(d.timing, KK_PHASE_A);
    }
  }
}

// -------------------------------------------------------------- phase B / init
template <int PC, int MODE>
__global__ void __launch_bounds__(288, 3)
k_phase_b(GridParams g, DevPtrs d, TileCfg t, int K, int parity, unsigned long long hcond, int use_cond) {
  extern __shared__ double smem[];
  SolverState* st = d.st_;
  constexpr bool ITER = (MODE == MODE_ITER);
  constexpr bool INIT = (MODE == MODE_INIT_COLD || MODE == MODE_INIT_WARM);
  constexpr bool TRUE_RES = (MODE == MODE_TRUERES);
  constexpr bool USE_U = (MODE != MODE_INIT_COLD);   // u := p for warm init / true residual
  constexpr bool NEED_Z = ITER || INIT;
  constexpr int KIND = ITER ? KK_PHASE_B : (INIT ? KK_INIT : KK_TRUERES);
  if (ITER && st->done) return;
  timing_begin(d.timing, KIND);
  Ring R = make_ring(smem);
  const TileCtx c = tile_ctx(g, t, K);
  const int m = d.cp[c.k].mat;
  const double* __restrict__ AP = d.AP + fofs(g, m);
  const double* __restrict__ AE = d.AE + fofs(g, m);
  const double* __restrict__ AN = d.AN + fofs(g, m);
  // ITER: r -= alpha A u.   INIT/TRUERES: r := S - A p  (u := p, alpha := 1).
  const double* __restrict__ rin = ITER ? d.r[parity] + fofs(g, c.k) : d.S + fofs(g, c.k);
  double* __restrict__ rout = (ITER ? d.r[1 - parity] : d.r[parity]) + fofs(g, c.k);
  const double* __restrict__ uin = ITER ? d.u[parity] + fofs(g, c.k) : d.p + fofs(g, c.k);
  double* __restrict__ p = d.p + fofs(g, c.k);
  const double alpha = ITER ? d.cs.alpha[c.k] : 1.0;
  const double omega = st->omega;
  const double c2 = (2.0 - omega) * omega;

  double AP1 = 1.0, AP2 = 1.0, AE1 = 0.0, AE2 = 0.0, AN1 = 0.0, AN2 = 0.0;
  double u1 = 0.0, u2 = 0.0, r1 = 0.0, p1 = 0.0, w1 = 0.0, v1 = 0.0, rn1 = 0.0;
  double acc_rr = 0.0, acc_rz = 0.0, acc_ss = 0.0;
  for (int jl = c.j0 - 2; jl <= c.j1 + 1; ++jl) {
    double u0 = 0.0, AP0 = 1.0, AE0 = 0.0, AN0 = 0.0, r0 = 0.0, p0 = 0.0;
    const bool in_rng = (jl >= 0 && jl < g.ny);
    const bool out_row0 = c.out_col && jl >= c.j0 && jl < c.j1;
    if (in_rng) {
      const long long q = (long long)jl * g.nt + c.gc;
      AP0 = AP[q]; AE0 = AE[q]; AN0 = AN[q];
      if (USE_U) u0 = uin[q];
      if (jl >= c.j0 - 1 && jl <= c.j1) r0 = rin[q];
      if (ITER && out_row0) p0 = p[q];
    }
    R.AE(jl, c.tl) = AE0;
    R.U(jl, c.tl) = u0;
    // s(jl-1) = A u at row jl-1 (row jl-1 of the ring was completed before last barrier)
    double s = 0.0;
    if constexpr (USE_U) {
      s = AP1 * u1;
      s += R.AE(jl - 1, c.tm) * R.U(jl - 1, c.tm);
      s += AE1 * R.U(jl - 1, c.tp);
      s += AN2 * u2;
      s += AN1 * u0;
    }
    const double rn = r1 - alpha * s;                  // Table 1 step 5 (or r0 = S - A p0)
    const bool out_row1 = c.out_col && jl - 1 >= c.j0 && jl - 1 < c.j1;
    if (out_row1) {
      const long long q1 = (long long)(jl - 1) * g.nt + c.gc;
      if (ITER) { rout[q1] = rn; p[q1] = p1 + alpha * u1; }   // step 4
      if (INIT) { rout[q1] = rn; if (MODE == MODE_INIT_COLD) p[q1] = 0.0; }
      acc_rr += rn * rn;
      if (INIT) acc_ss += r1 * r1;
    }
    double z2 = 0.0;     // z at row jl-2
    if constexpr (NEED_Z) {
      const double inv1 = 1.0 / AP1;
      if constexpr (PC == PC_ASSOR2) {
        const double w0 = rn * inv1;                   // w(jl-1)
        R.W(jl - 1, c.tl) = w0;
        __syncthreads();   // the only barrier per row
        double sL = AN2 * w1;                          // S: A_S(jl-1) = AN(jl-2)
        if (c.gc >= 1) sL += R.AE(jl - 1, c.tm) * R.W(jl - 1, c.tm);
        if (c.endcol) sL += AE1 * R.W(jl - 1, c.tp);
        const double v0 = w0 - (omega * inv1) * sL;   // v1(jl-1)
        R.V(jl - 1, c.tl) = v0;
        double sU = AN2 * v0;                          // N of row jl-2: AN(jl-2) * v1(jl-1)
        if (!c.endcol) sU += AE2 * R.V(jl - 2, c.tp);
        if (c.w0col) sU += R.AE(jl - 2, c.tm) * R.V(jl - 2, c.tm);
        z2 = c2 * (v1 - (omega / AP2) * sU);
        w1 = w0; v1 = v0;
      } else if constexpr (PC == PC_JACOBI) {
        __syncthreads();
        z2 = w1;
        w1 = rn * inv1;
      } else {
        __syncthreads();
        z2 = w1;
        w1 = rn;
      }
      if (c.out_col && jl - 2 >= c.j0 && jl - 2 < c.j1) acc_rz += rn1 * z2;
    } else {
      __syncthreads();
    }
    rn1 = rn;
    u2 = u1; u1 = u0; r1 = r0; p1 = p0;
    AP2 = AP1; AP1 = AP0; AE2 = AE1; AE1 = AE0; AN2 = AN1; AN1 = AN0;
  }
  double v[3] = {acc_rr, acc_rz, acc_ss};
  block_sum<3>(v, smem);
  const int ncta = t.n_tiles;
  const int cta = blockIdx.x / K;
  if (threadIdx.x == 0) {
    d.partials[(long long)(0 * K + c.k) * ncta + cta] = v[0];
    d.partials[(long long)(1 * K + c.k) * ncta + cta] = v[1];
    d.partials[(long long)(2 * K + c.k) * ncta + cta] = v[2];
  }
  if (last_cta_arrive(&d.counters[KIND], gridDim.x)) {
    double* red = smem;
    reduce_partials(d, 3, K, ncta, red);
    if (threadIdx.x == 0) {
      const double* rrk = red;
      const double* rzk = red + K;
      const double* ssk = red + 2 * K;
      double rr = 0.0;
      for (int k = 0; k < K; ++k) { rr += rrk[k]; }
      if (TRUE_RES) {
        for (int k = 0; k < K; ++k) d.cs.ttk[k] = rrk[k];
        st->true_rel = (st->nS > 0.0) ? sqrt(rr) / st->nS : 0.0;
        if (d.dist.world > 0)   // multi-rank: publish ||S_k - A_k p_k||^2; k_true_scalar sums all ranks
          for (int k = 0; k < d.dist.kmax_local; ++k) d.dist.packed_local[k] = k < K ? rrk[k] : 0.0;
      } else if (INIT) {
        double SS = 0.0, dd = 0.0;
        for (int k = 0; k < K; ++k) {
          d.cs.Sk[k] = ssk[k]; d.cs.rrk[k] = rrk[k]; d.cs.dk[k] = rzk[k];
          SS += ssk[k]; dd += rzk[k];
        }
        st->d = dd;
        st->nS = sqrt(SS);
        st->iter = 0;
        st->status = 0;
        st->converged = 0;
        st->done = 0;
        st->zero_p = 0;
        if (st->nS == 0.0) {
          st->rel = 0.0; st->done = 1; st->converged = 1; st->zero_p = 1;
        } else {
          st->rel = sqrt(rr) / st->nS;
          if (st->fixed_iters == 0 && st->rel <= st->tol) { st->done = 1; st->converged = 1; }
          else if (st->max_iter <= 0) { st->done = 1; st->status = -6; }
        }
        set_cond(use_cond, hcond, st->done == 0);
      } else {  // ITER
        for (int k = 0; k < K; ++k) d.cs.rrk[k] = rrk[k];
        st->iter += 1;
        st->rel = sqrt(rr) / st->nS;
        if (st->fixed_iters > 0) {
          if (st->iter >= st->fixed_iters) st->done = 1;
        } else if (st->rel <= st->tol) {
          st->done = 1; st->converged = 1;
        } else if (st->iter >= st->max_iter) {
          st->done = 1; st->status = -6;
        }
        if (!st->done || st->fixed_iters > 0) {
          bool bad = false;
          if (st->coupling == 0) {
            double d2 = 0.0;
            for (int k = 0; k < K; ++k) { d2 += rzk[k]; }
            if (!(d2 > 0.0)) bad = true;
            const double b = d2 / st->d;
            for (int k = 0; k < K; ++k) { d.cs.beta[k] = b; d.cs.dk[k] = rzk[k]; }
            st->d = d2;
          } else {
            for (int k = 0; k < K; ++k) {
              double b = 0.0;
              if (d.cs.dk[k] != 0.0) { if (rzk[k] < 0.0) bad = true; b = rzk[k] / d.cs.dk[k]; }
              d.cs.beta[k] = b; d.cs.dk[k] = rzk[k];
            }
          }
          if (bad && !st->done) { st->done = 1; st->status = -5; }
        }
        set_cond(use_cond, hcond, st->done == 0);
      }
      timing_end(d.timing, KIND);
    }
  }
}

// ------------------------------------------------------------------- launchers
static size_t ring_bytes(const TileCfg& t) {
  const int nl = t.tw + 2 * HALO;
  size_t b = (size_t)16 * nl * sizeof(double);
  const size_t red = (size_t)3 * (nl + 32) * sizeof(double);
  return b > red ? b : red;
}

static size_t tile_smem(const TileCfg& t, int K) {
  size_t sm = ring_bytes(t);
  // the last-CTA reduction reuses shared memory for 3*K doubles
  if (sm < (size_t)3 * K * sizeof(double)) sm = (size_t)3 * K * sizeof(double);
  return sm;
}

template <typename KernelT>
static cudaError_t launch_tiles(KernelT kern, const GridParams& g, const DevPtrs& d, const TileCfg& t,
                                int K, int parity, unsigned long long h, int use, cudaStream_t s) {
  const int threads = t.tw + 2 * HALO;
  kern<<<dim3(t.n_tiles * K), threads, tile_smem(t, K), s>>>(g, d, t, K, parity, h, use);
  return cudaGetLastError();
}

template <typename KernelT>
static cudaError_t set_smem(KernelT kern, int) {
  return raise_smem_cap(kern);
}

// Called once per context, outside any stream capture.
cudaError_t configure_pcg_kernels(const TileCfg& t, int K) {
  // raised once to the device's opt-in maximum (see configure_sr_kernels)
  const int sm = smem_optin_max();
  if (sm <= 0 || (long long)tile_smem(t, K) > sm) return cudaErrorInvalidValue;
  static unsigned done = 0u;   // once per device
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cudaErrorInvalidValue;
  if (done & (1u << dev)) return cudaSuccess;
  cudaError_t e = cudaSuccess;
#define GMAF_SET(...) if (e == cudaSuccess) e = set_smem(__VA_ARGS__, sm)
  GMAF_SET(k_phase_a<PC_ASSOR2>); GMAF_SET(k_phase_a<PC_JACOBI>); GMAF_SET(k_phase_a<PC_NONE>);
  GMAF_SET(k_phase_b<PC_ASSOR2, MODE_ITER>); GMAF_SET(k_phase_b<PC_JACOBI, MODE_ITER>);
  GMAF_SET(k_phase_b<PC_NONE, MODE_ITER>);
  GMAF_SET(k_phase_b<PC_ASSOR2, MODE_INIT_COLD>); GMAF_SET(k_phase_b<PC_JACOBI, MODE_INIT_COLD>);
  GMAF_SET(k_phase_b<PC_NONE, MODE_INIT_COLD>);
  GMAF_SET(k_phase_b<PC_ASSOR2, MODE_INIT_WARM>); GMAF_SET(k_phase_b<PC_JACOBI, MODE_INIT_WARM>);
  GMAF_SET(k_phase_b<PC_NONE, MODE_INIT_WARM>);
  GMAF_SET(k_phase_b<PC_NONE, MODE_TRUERES>);
#undef GMAF_SET
  if (e == cudaSuccess) done |= 1u << dev;
  return e;
}

cudaError_t launch_init(const GridParams& g, const DevPtrs& d, const TileCfg& t, int K, int precond,
                        bool warm, unsigned long long h, cudaStream_t s) {
  const int use = h != 0ull;
  if (warm) {
    if (precond == PC_ASSOR2) return launch_tiles(k_phase_b<PC_ASSOR2, MODE_INIT_WARM>, g, d, t, K, 0, h, use, s);
    if (precond == PC_JACOBI) return launch_tiles(k_phase_b<PC_JACOBI, MODE_INIT_WARM>, g, d, t, K, 0, h, use, s);
    return launch_tiles(k_phase_b<PC_NONE, MODE_INIT_WARM>, g, d, t, K, 0, h, use, s);
  }
  if (precond == PC_ASSOR2) return launch_tiles(k_phase_b<PC_ASSOR2, MODE_INIT_COLD>, g, d, t, K, 0, h, use, s);
  if (precond == PC_JACOBI) return launch_tiles(k_phase_b<PC_JACOBI, MODE_INIT_COLD>, g, d, t, K, 0, h, use, s);
  return launch_tiles(k_phase_b<PC_NONE, MODE_INIT_COLD>, g, d, t, K, 0, h, use, s);
}

cudaError_t launch_phase_a(const GridParams& g, const DevPtrs& d, const TileCfg& t, int K,
                           int precond, int parity, unsigned long long h, cudaStream_t s) {
  const int use = h != 0ull;
  if (precond == PC_ASSOR2) return launch_tiles(k_phase_a<PC_ASSOR2>, g, d, t, K, parity, h, use, s);
  if (precond == PC_JACOBI) return launch_tiles(k_phase_a<PC_JACOBI>, g, d, t, K, parity, h, use, s);
  return launch_tiles(k_phase_a<PC_NONE>, g, d, t, K, parity, h, use, s);
}

cudaError_t launch_phase_b(const GridParams& g, const DevPtrs& d, const TileCfg& t, int K,
                           int precond, int parity, unsigned long long h, cudaStream_t s) {
  const int use = h != 0ull;
  if (precond == PC_ASSOR2) return launch_tiles(k_phase_b<PC_ASSOR2, MODE_ITER>, g, d, t, K, parity, h, use, s);
  if (precond == PC_JACOBI) return launch_tiles(k_phase_b<PC_JACOBI, MODE_ITER>, g, d, t, K, parity, h, use, s);
  return launch_tiles(k_phase_b<PC_NONE, MODE_ITER>, g, d, t, K, parity, h, use, s);
}

cudaError_t launch_residual_init(const GridParams& g, const DevPtrs& d, const TileCfg& t, int K, int out_parity,
                                 cudaStream_t s) {
  return launch_tiles(k_phase_b<PC_NONE, MODE_INIT_WARM>, g, d, t, K, out_parity, 0ull, 0, s);
}

cudaError_t launch_true_residual(const GridParams& g, const DevPtrs& d, const TileCfg& t, int K,
                                 cudaStream_t s) {
  return launch_tiles(k_phase_b<PC_NONE, MODE_TRUERES>, g, d, t, K, 0, 0ull, 0, s);
}

// Multi-rank true residual: sum of every rank's ||S_k - A_k p_k||^2 in condition order.
__global__ void k_true_scalar(DevPtrs d, int world) {
  if (threadIdx.x != 0) return;
  const int km = d.dist.kmax_local;
  double rr = 0.0;
  for (int r = 0; r < world; ++r)
    for (int k = 0; k < km; ++k) rr += d.dist.packed_all[(long long)r * km + k];
  d.st_->true_rel = (d.st_->nS > 0.0) ? sqrt(rr) / d.st_->nS : 0.0;
}

cudaError_t launch_true_scalar(const DevPtrs& d, int world, cudaStream_t s) {
  k_true_scalar<<<1, 32, 0, s>>>(d, world);
  return cudaGetLastError();
}

// Resident CTAs per SM of the dominant iteration kernel (phase B, ASSOR-II).
int pcg_ctas_per_sm(const TileCfg& t, int K) {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_phase_b<PC_ASSOR2, MODE_ITER>, t.tw + 2 * HALO,
                                                    tile_smem(t, K)) != cudaSuccess)
    return 1;
  return n;
}

}  // namespace gmaf
