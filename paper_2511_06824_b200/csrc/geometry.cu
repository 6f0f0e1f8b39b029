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
// 32-bit unsigned arithmetic: the host rejects meshes whose products could reach 2^32
// (check_grid), so the same integers as the oracle's int64 evaluation, without 64-bit divisions.
__device__ __forceinline__ bool texture_mask(const GridParams& g, int i, int j) {
  if (g.tex_nt <= 0 || g.tex_ny <= 0) return false;
  if (j < 0 || j >= g.tex_band) return false;
  const unsigned nt = (unsigned)g.nt, B = (unsigned)g.tex_band, N = (unsigned)g.tex_num, D = (unsigned)g.tex_den;
  const unsigned ci = ((unsigned)i * (unsigned)g.tex_nt) % nt;
  const unsigned cj = ((unsigned)j * (unsigned)g.tex_ny) % B;
  return ((unsigned long long)D * ci < (unsigned long long)N * nt) &&
         ((unsigned long long)D * cj < (unsigned long long)N * B);
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
// One thread per (column i, chunk of ASM_ROWS stored rows, condition k), marching up the column:
// the thickness and conductance of the rows below and at the node are carried from the previous
// row, so per node it evaluates the film at (i, j+1) and at the two theta neighbours (3 instead of
// 5); every value is the same expression as before, so the bands stay bitwise.  Bands are written
// once per distinct coefficient set (by its representative condition); S for every condition.
constexpr int ASM_ROWS = 16;

__global__ void k_assemble(GridParams g, DevPtrs d, int K) {
  timing_begin(d.timing, KK_ASSEMBLE);
  // the stored rows of this context (all rows on one rank; own rows + halo rows on a slab)
  const int srows = (int)(g.ns / g.nt);
  const int nchunks = (srows + ASM_ROWS - 1) / ASM_ROWS;
  const long long per_k = (long long)g.nt * nchunks;
  const long long total = per_k * K;
  const long long n = g.ns;
  for (long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x; w < total;
       w += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(w / per_k);
    const long long rem = w - (long long)k * per_k;
    const int i = (int)(rem % g.nt), ch = (int)(rem / g.nt);
    const int ja = g.yb + ch * ASM_ROWS, jb = min(ja + ASM_ROWS, g.yb + srows);
    const CondParams& c = d.cp[k];
    const int iE = (i + 1 == g.nt) ? 0 : i + 1;
    const int iW = (i == 0) ? g.nt - 1 : i - 1;
    const bool rep = d.mat_rep[c.mat] == k;
    double hS = film(g, c, d.ct, d.st, i, ja - 1, false).h;
    Film fP = film(g, c, d.ct, d.st, i, ja, true);
    double gS = conductance(g, hS), gP = conductance(g, fP.h);
    for (int j = ja; j < jb; ++j) {
      const Film fN = film(g, c, d.ct, d.st, i, j + 1, true);
      const double hE = film(g, c, d.ct, d.st, iE, j, false).h;
      const double hW = film(g, c, d.ct, d.st, iW, j, false).h;
      const double hN = fN.h;
      const double gN = conductance(g, hN);
      const long long idx = (long long)(j - g.yb) * g.nt + i;
      if (rep) {
        // the bands: only the representative condition of a coefficient set needs them
        const double gE = conductance(g, hE), gW = conductance(g, hW);
        const double ge = harmonic(gP, gE);
        const double gw = harmonic(gW, gP);   // == ge(iW, j) bit for bit
        const double gn = harmonic(gP, gN);
        const double gs = harmonic(gS, gP);   // == gn(i, j-1) bit for bit
        const double aE = ge * c.rx, aW = gw * c.rx, aN = gn * c.ry, aS = gs * c.ry;
        const long long o = (long long)c.mat * n + idx;   // = fofs(g, mat) + j*nt + i
        d.AP[o] = ((aW + aE) + aS) + aN;
        d.AE[o] = -aE;
        d.AN[o] = (j < g.ny - 1) ? -aN : 0.0;
      }
      const double t1 = ((c.Ut * 0.5) * ((hE - hW) * 0.5)) * c.dy;
      const double t2 = ((c.Uy * 0.5) * ((hN - hS) * 0.5)) * c.dx;
      const double t3 = (fP.hd * c.dx) * c.dy;
      double sv = -((t1 + t2) + t3);
      if (j == 0) sv = sv + (harmonic(gS, gP) * c.ry) * c.pin;          // Dirichlet fold, aS p_in
      if (j == g.ny - 1) sv = sv + (harmonic(gP, gN) * c.ry) * c.pout;  // aN p_out
      d.S[(long long)k * n + idx] = sv;
      hS = fP.h; gS = gP;
      fP = fN; gP = gN;
    }
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
constexpr int QUAD_ROWS = 32;    // cell rows per thread (a column marches over them)

__device__ __forceinline__ double node_p(const CondParams& c, const double* p, int ny, int nt, int i, int j) {
  return j < 0 ? c.pin : (j >= ny ? c.pout : p[(long long)j * nt + i]);
}

// One thread per (column i, chunk of QUAD_ROWS cell rows): it marches up its column carrying the
// node values h and p of the lower cell row, so each node's thickness is evaluated once per
// thread (2 per cell instead of 4).
__global__ void __launch_bounds__(QUAD_THREADS) k_quadrature(GridParams g, DevPtrs d, int K) {
  __shared__ double red[12 * (QUAD_THREADS + 32)];
  timing_begin(d.timing, KK_QUAD);
  const int k = blockIdx.y;
  const CondParams& c = d.cp[k];
  const double* p = d.p + fofs(g, k);
  // this context's cells: j + 1 in [y0, y1), plus the top ghost cell j = n_y - 1 on the last slab
  // (all n_y + 1 cell rows on one rank); row y0 - 1 of a slab is its exchanged halo row
  const int cj0 = g.y0 - 1;
  const int crows = g.y1 - g.y0 + (g.y1 == g.ny ? 1 : 0);
  const int nchunks = (crows + QUAD_ROWS - 1) / QUAD_ROWS;
  const long long columns = (long long)g.nt * nchunks;
  const double dA = c.dx * c.dy;
  double acc[12];
#pragma unroll
  for (int q = 0; q < 12; ++q) acc[q] = 0.0;
  for (long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x; w < columns;
       w += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(w % g.nt), ch = (int)(w / g.nt);
    const int i1 = (i + 1 == g.nt) ? 0 : i + 1;
    const int ja = cj0 + ch * QUAD_ROWS, jb = min(ja + QUAD_ROWS, cj0 + crows);
    const double cc = d.cth[i], sc = d.sth[i];
    const double rx = g.Rk * cc, ry = g.Rk * sc;
    double p00 = node_p(c, p, g.ny, g.nt, i, ja), p10 = node_p(c, p, g.ny, g.nt, i1, ja);
    double h00 = film(g, c, d.ct, d.st, i, ja, false).h, h10 = film(g, c, d.ct, d.st, i1, ja, false).h;
    for (int j = ja; j < jb; ++j) {
      const double p01 = node_p(c, p, g.ny, g.nt, i, j + 1), p11 = node_p(c, p, g.ny, g.nt, i1, j + 1);
      const double h01 = film(g, c, d.ct, d.st, i, j + 1, false).h;
      const double h11 = film(g, c, d.ct, d.st, i1, j + 1, false).h;
      const double pb = (((p00 + p10) + p01) + p11) * 0.25;
      const double hb = (((h00 + h10) + h01) + h11) * 0.25;
      const double dpdx = ((p10 + p11) - (p00 + p01)) / (2.0 * c.dx);
      const double dpdy = ((p01 + p11) - (p00 + p10)) / (2.0 * c.dy);
      const double y0 = (double)(j + 1) * c.dy, y1 = (double)(j + 2) * c.dy;
      const double rz = (y0 + y1) * 0.5;
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
      p00 = p01; p10 = p11; h00 = h01; h10 = h11;
    }
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
  const long long work = (long long)g.nt * ((g.ns / g.nt + ASM_ROWS - 1) / ASM_ROWS) * K;
  k_assemble<<<grid_for(work, 256, 148 * 16), 256, 0, s>>>(g, d, K);
  return cudaGetLastError();
}

cudaError_t launch_field(const GridParams& g, const DevPtrs& d, int field, int k, cudaStream_t s) {
  const long long work = (long long)(g.ny + 2) * g.nt;
  k_field<<<grid_for(work, 256, 148 * 8), 256, 0, s>>>(g, d, field, k);
  return cudaGetLastError();
}

int quad_ctas_per_condition(const GridParams& g, int K) {
  const long long columns = (long long)((g.y1 - g.y0 + 1 + QUAD_ROWS - 1) / QUAD_ROWS) * g.nt;
  int per_k = grid_for(columns, QUAD_THREADS, 1 << 20);
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
