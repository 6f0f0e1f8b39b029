// geometry.cu -- film thickness (Eq. 2.3), FVM assembly (Eqs. 2.4-2.7) and the
// force/moment quadrature (Sec. 2.4-III) for K working conditions on sm_100a.
//
// Compiled with --fmad=false: every product and sum below is rounded separately,
// in the order written, so thickness, bands and source are bitwise reproducible
// against any IEEE evaluation of the same expressions.  CUDA's
// double '/' and sqrt are IEEE round-to-nearest; cos/sin come from host tables.
#include <cstdint>
#include "device_common.cuh"
#include "gmaf_internal.cuh"

namespace gmaf {

// Dimple mask (Fig. 10; DESIGN.md R-A7): integer arithmetic only.
__device__ __forceinline__ bool texture_mask(const GridParams& g, int i, int j) {
  if (g.tex_nt <= 0 || g.tex_ny <= 0) return false;
  if (j < 0 || j >= g.tex_band) return false;
  const long long nt = g.nt, B = g.tex_band, N = g.tex_num, D = g.tex_den;
  const long long ci = ((long long)i * (long long)g.tex_nt) % nt;
  const long long cj = ((long long)j * (long long)g.tex_ny) % B;
  return (D * ci < N * nt) && (D * cj < N * B);
}

// Eq. 2.3 at node (i, j), j in [-1, n_y]; also returns the rate (Eq. 2.2, chain rule).
struct Film { double h, hd; };

__device__ __forceinline__ Film film(const GridParams& g, const CondParams& c, const double* ct,
                                     const double* st, int i, int j, bool want_rate) {
  const double y = (double)(j + 1) * c.dy;
  const double a = (g.Rc * ct[i] - c.sl * y) - c.e[0];
  const double b = (g.Rc * st[i] - c.tl * y) - c.e[1];
  const double r = sqrt(a * a + b * b);
  const double ht = texture_mask(g, i, j) ? g.tex_depth : 0.0;
  Film f;
  f.h = (r - g.Rk) + ht;
  f.hd = 0.0;
  if (want_rate) {
    const double ad = -(c.sld * y + c.edot[0]);
    const double bd = -(c.tld * y + c.edot[1]);
    f.hd = (a * ad + b * bd) / r;
  }
  return f;
}

__device__ __forceinline__ double conductance(const GridParams& g, double h) {
  return ((h * h) * h) / g.twelve_mu;       // g = h^3 / (12 mu)
}

__device__ __forceinline__ double harmonic(double ga, double gb) {
  return ((2.0 * ga) * gb) / (ga + gb);
}

// ------------------------------------------------------------------ thickness guard
__global__ void k_thickness_guard(GridParams g, DevPtrs d, int K) {
  timing_begin(d.timing, KK_THICK);
  const long long rows = (long long)(g.ny + 2);
  const long long per_k = rows * g.nt;
  const long long total = per_k * K;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(q / per_k);
    const long long rem = q - (long long)k * per_k;
    const int j = (int)(rem / g.nt) - 1;
    const int i = (int)(rem % g.nt);
    const Film f = film(g, d.cp[k], d.ct, d.st, i, j, false);
    if (!(f.h >= g.hmin)) {
      if (atomicCAS(&d.guard[0], 0ull, 1ull) == 0ull) {
        d.guard[1] = (unsigned long long)k;
        d.guard[2] = ((unsigned long long)(unsigned)i << 32) | (unsigned long long)(unsigned)(j + 1);
        d.guard[3] = (unsigned long long)__double_as_longlong(f.h);
      }
    }
  }
  if (last_cta_arrive(&d.counters[KK_THICK], gridDim.x) && threadIdx.x == 0)
    timing_end(d.timing, KK_THICK);
}

// ------------------------------------------------------------------ assembly (G1)
// One thread per (i, j, k).  Bands are written once per distinct coefficient set
// (by its representative condition); S for every condition.
__global__ void k_assemble(GridParams g, DevPtrs d, int K) {
  timing_begin(d.timing, KK_ASSEMBLE);
  // the stored rows of this context (all rows on one rank; own rows + halo rows on a slab)
  const long long n = g.ns;
  const long long total = n * K;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(q / n);
    const long long idx = q - (long long)k * n;
    const int j = g.yb + (int)(idx / g.nt);
    const int i = (int)(idx % g.nt);
    const CondParams& c = d.cp[k];
    const int iE = (i + 1 == g.nt) ? 0 : i + 1;
    const int iW = (i == 0) ? g.nt - 1 : i - 1;
    const Film fP = film(g, c, d.ct, d.st, i, j, true);
    const double hE = film(g, c, d.ct, d.st, iE, j, false).h;
    const double hW = film(g, c, d.ct, d.st, iW, j, false).h;
    const double hN = film(g, c, d.ct, d.st, i, j + 1, false).h;
    const double hS = film(g, c, d.ct, d.st, i, j - 1, false).h;
    const double gP = conductance(g, fP.h), gE = conductance(g, hE), gW = conductance(g, hW);
    const double gN = conductance(g, hN), gS = conductance(g, hS);
    const double ge = harmonic(gP, gE);
    const double gw = harmonic(gW, gP);   // == ge(iW, j) bit for bit
    const double gn = harmonic(gP, gN);
    const double gs = harmonic(gS, gP);   // == gn(i, j-1) bit for bit
    const double aE = ge * c.rx, aW = gw * c.rx, aN = gn * c.ry, aS = gs * c.ry;
    if (d.mat_rep[c.mat] == k) {
      const long long o = (long long)c.mat * n + idx;   // = fofs(g, mat) + j*nt + i
      d.AP[o] = ((aW + aE) + aS) + aN;
      d.AE[o] = -aE;
      d.AN[o] = (j < g.ny - 1) ? -aN : 0.0;
    }
    const double t1 = ((c.Ut * 0.5) * ((hE - hW) * 0.5)) * c.dy;
    const double t2 = ((c.Uy * 0.5) * ((hN - hS) * 0.5)) * c.dx;
    const double t3 = (fP.hd * c.dx) * c.dy;
    double s = -((t1 + t2) + t3);
    if (j == 0) s = s + aS * c.pin;
    if (j == g.ny - 1) s = s + aN * c.pout;
    d.S[(long long)k * n + idx] = s;
  }
  if (last_cta_arrive(&d.counters[KK_ASSEMBLE], gridDim.x) && threadIdx.x == 0)
    timing_end(d.timing, KK_ASSEMBLE);
}

// ---------------------------------------------------------------- field readback
__global__ void k_field(GridParams g, DevPtrs d, int field, int k) {
  const long long total = (long long)(g.ny + 2) * g.nt;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(q / g.nt) - 1, i = (int)(q % g.nt);
    const Film f = film(g, d.cp[k], d.ct, d.st, i, j, true);
    d.scratch[q] = (field == 1) ? f.h : f.hd;
  }
}

// -------------------------------------------------------------- quadrature (G5)
// Cells (i, j), j in [-1, n_y-1], between node rows j and j+1 (ghost rows carry
// p_in / p_out).  Pressure traction -p n and Couette-Poiseuille wall shear on the
// piston; moments about the bottom centre (DESIGN.md R-A14).
constexpr int QUAD_THREADS = 256;

__global__ void __launch_bounds__(QUAD_THREADS) k_quadrature(GridParams g, DevPtrs d, int K) {
  __shared__ double red[12 * (QUAD_THREADS + 32)];
  timing_begin(d.timing, KK_QUAD);
  const int k = blockIdx.y;
  const CondParams& c = d.cp[k];
  const double* p = d.p + fofs(g, k);
  // this context's cells: j + 1 in [y0, y1), plus the top ghost cell j = n_y - 1 on the last slab
  // (all n_y + 1 cell rows on one rank); row y0 - 1 of a slab is its exchanged halo row
  const int cj0 = g.y0 - 1;
  const long long cells = (long long)(g.y1 - g.y0 + (g.y1 == g.ny ? 1 : 0)) * g.nt;
  const double dA = c.dx * c.dy;
  double acc[12];
#pragma unroll
  for (int q = 0; q < 12; ++q) acc[q] = 0.0;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < cells;
       q += (long long)gridDim.x * blockDim.x) {
    const int j = cj0 + (int)(q / g.nt), i = (int)(q % g.nt);
    const int i1 = (i + 1 == g.nt) ? 0 : i + 1;
    const double p00 = (j < 0) ? c.pin : p[(long long)j * g.nt + i];
    const double p10 = (j < 0) ? c.pin : p[(long long)j * g.nt + i1];
    const double p01 = (j + 1 >= g.ny) ? c.pout : p[(long long)(j + 1) * g.nt + i];
    const double p11 = (j + 1 >= g.ny) ? c.pout : p[(long long)(j + 1) * g.nt + i1];
    const double h00 = film(g, c, d.ct, d.st, i, j, false).h;
    const double h10 = film(g, c, d.ct, d.st, i1, j, false).h;
    const double h01 = film(g, c, d.ct, d.st, i, j + 1, false).h;
    const double h11 = film(g, c, d.ct, d.st, i1, j + 1, false).h;
    const double pb = (((p00 + p10) + p01) + p11) * 0.25;
    const double hb = (((h00 + h10) + h01) + h11) * 0.25;
    const double dpdx = ((p10 + p11) - (p00 + p01)) / (2.0 * c.dx);
    const double dpdy = ((p01 + p11) - (p00 + p10)) / (2.0 * c.dy);
    const double y0 = (double)(j + 1) * c.dy, y1 = (double)(j + 2) * c.dy;
    const double yc = (y0 + y1) * 0.5;
    const double cc = d.cth[i], sc = d.sth[i];
    const double rx = g.Rk * cc, ry = g.Rk * sc, rz = yc;
    const double fx = -pb * cc * dA, fy = -pb * sc * dA;
    acc[0] += fx; acc[1] += fy;
    acc[3] += -rz * fy;
    acc[4] += rz * fx;
    acc[5] += rx * fy - ry * fx;
    const double tth = -(hb * 0.5) * dpdx - (g.mu * c.Ut) / hb;
    const double ty = -(hb * 0.5) * dpdy - (g.mu * c.Uy) / hb;
    const double sx = -tth * sc * dA, sy = tth * cc * dA, sz = ty * dA;
    acc[6] += sx; acc[7] += sy; acc[8] += sz;
    acc[9] += ry * sz - rz * sy;
    acc[10] += rz * sx - rx * sz;
    acc[11] += rx * sy - ry * sx;
  }
  block_sum<12>(acc, red);
  const int ncta = gridDim.x;
  if (threadIdx.x == 0) {
    double* dst = d.wrench_part + ((long long)k * ncta + blockIdx.x) * 12;
#pragma unroll
    for (int q = 0; q < 12; ++q) dst[q] = acc[q];
  }
  if (last_cta_arrive(&d.counters[KK_QUAD], gridDim.x * gridDim.y)) {
    for (int t = threadIdx.x; t < 12 * K; t += blockDim.x) {
      const int kk = t / 12, q = t % 12;
      double s = 0.0;
      for (int b = 0; b < ncta; ++b) s += __ldcg(&d.wrench_part[((long long)kk * ncta + b) * 12 + q]);
      d.wrench[kk * 12 + q] = s;
    }
    if (threadIdx.x == 0) timing_end(d.timing, KK_QUAD);
  }
}

// ------------------------------------------------------------------- launchers
static int grid_for(long long work, int threads, int cap) {
  long long b = (work + threads - 1) / threads;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

cudaError_t launch_thickness_guard(const GridParams& g, const DevPtrs& d, int K, cudaStream_t s) {
  const long long work = (long long)(g.ny + 2) * g.nt * K;
  k_thickness_guard<<<grid_for(work, 256, 148 * 16), 256, 0, s>>>(g, d, K);
  return cudaGetLastError();
}

cudaError_t launch_assemble(const GridParams& g, const DevPtrs& d, int K, cudaStream_t s) {
  const long long work = g.ns * K;
  k_assemble<<<grid_for(work, 256, 148 * 16), 256, 0, s>>>(g, d, K);
  return cudaGetLastError();
}

cudaError_t launch_field(const GridParams& g, const DevPtrs& d, int field, int k, cudaStream_t s) {
  const long long work = (long long)(g.ny + 2) * g.nt;
  k_field<<<grid_for(work, 256, 148 * 8), 256, 0, s>>>(g, d, field, k);
  return cudaGetLastError();
}

int quad_ctas_per_condition(const GridParams& g, int K) {
  const long long cells = (long long)(g.y1 - g.y0 + 1) * g.nt;
  int per_k = grid_for(cells, QUAD_THREADS, 1 << 20);
  const int target = (148 * 8 + K - 1) / K;   // ~8 CTAs per SM in total
  if (per_k > target) per_k = target;
  return per_k < 1 ? 1 : per_k;
}

cudaError_t launch_quadrature(const GridParams& g, const DevPtrs& d, int K, cudaStream_t s,
                              int* n_cta_out) {
  const int per_k = quad_ctas_per_condition(g, K);
  if (n_cta_out) *n_cta_out = per_k;
  k_quadrature<<<dim3(per_k, K), QUAD_THREADS, 0, s>>>(g, d, K);
  return cudaGetLastError();
}

}  // namespace gmaf
