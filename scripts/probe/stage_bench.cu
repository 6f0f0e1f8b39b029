// Micro-benchmark of the single-thread scalar stage (sr_scalar_stage<false>, coupled, K = 9) that
// sits on the serial tail of every k_sr iteration: cycles per call, and the same for pieces.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2511_06824_b200/csrc/sr_common.cuh"
using namespace gmaf;

__global__ void k_bench(DevPtrs d, double* red, int K, long long* out) {
  __shared__ double sh[4 * 64];
  for (int i = threadIdx.x; i < 4 * K; i += blockDim.x) sh[i] = red[i];
  __syncthreads();
  if (threadIdx.x != 0) return;
  long long tc0 = clock64();
  d.st_->done = 0;
  sr_scalar_stage<false>(d, sh, K, K, 0, 0, 0ull);   // first (cold instruction cache) call
  long long tc1 = clock64();
  out[4] = tc1 - tc0;
  long long t0 = clock64();
  for (int it = 0; it < 100; ++it) {
    d.st_->done = 0;
    sr_scalar_stage<false>(d, sh, K, K, 0, 0, 0ull);
  }
  long long t1 = clock64();
  // pieces: snapshot load + store back
  for (int it = 0; it < 100; ++it) { SolverState s = *d.st_; s.iter += 1; *d.st_ = s; }
  long long t2 = clock64();
  double acc = 1.0;
  for (int it = 0; it < 100; ++it) { acc = sqrt(acc + sh[it & 7]) / (acc + 3.0); acc = acc / (acc + 1.0); }
  long long t3 = clock64();
  out[0] = (t1 - t0) / 100; out[1] = (t2 - t1) / 100; out[2] = (t3 - t2) / 100; out[3] = (long long)acc;
}

int main() {
  const int K = 9;
  DevPtrs d{};
  SolverState* st; double* cs; double* red; long long* out;
  cudaMalloc(&st, sizeof(SolverState)); cudaMalloc(&cs, 9 * K * 8); cudaMalloc(&red, 4 * K * 8); cudaMalloc(&out, 64);
  SolverState h{}; h.tol = 1e-30; h.omega = 1.6; h.coupling = 0; h.max_iter = 1 << 30; h.d = 1.0; h.nS = 1.0;
  cudaMemcpy(st, &h, sizeof(h), cudaMemcpyHostToDevice);
  double hr[4 * K]; for (int i = 0; i < 4 * K; ++i) hr[i] = 1.0 + i;
  cudaMemcpy(red, hr, sizeof(hr), cudaMemcpyHostToDevice);
  double ones[9 * K]; for (int i = 0; i < 9 * K; ++i) ones[i] = 1.0;
  cudaMemcpy(cs, ones, sizeof(ones), cudaMemcpyHostToDevice);
  d.st_ = st;
  d.cs.alpha = cs; d.cs.beta = cs + K; d.cs.dk = cs + 2 * K; d.cs.Sk = cs + 3 * K; d.cs.rrk = cs + 4 * K;
  d.cs.uvk = cs + 5 * K; d.cs.ttk = cs + 6 * K; d.cs.itk = (int*)(cs + 7 * K); d.cs.frz = d.cs.itk + K;
  k_bench<<<1, 32>>>(d, red, K, out);
  long long ho[5];
  cudaMemcpy(ho, out, sizeof(ho), cudaMemcpyDeviceToHost);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("cycles/call: stage %lld (first, cold: %lld)  snapshot+writeback %lld  sqrt+2div %lld  (clock %d kHz: stage %.2f us, cold %.2f us)\n",
         ho[0], ho[4], ho[1], ho[2], clk, ho[0] / (clk * 1e-3), ho[4] / (clk * 1e-3));
  return cudaGetLastError() != cudaSuccess;
}
