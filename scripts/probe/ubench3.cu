// Post-barrier shared-load bursts (the row pipeline's phase shape) on B200: NW warps per CTA, one
// CTA per SM; per iteration each warp does bar.sync, NL independent 8-byte shared loads of
// neighbour values, a dependent DFMA chain over them, and NS 8-byte stores.  Cycles per iteration
// against NL (does the burst of loads after the barrier set the phase length?).
#include <cstdio>
#include <cuda_runtime.h>

template <int NL, int NS, bool BAR>
__global__ void k_phase(double* out, int n, long long* cyc) {
  extern __shared__ double ring[];   // [NL + NS][1024]
  const int t = threadIdx.x, nt = blockDim.x;
  for (int i = t; i < (NL + NS) * 1024; i += nt) ring[i] = 1e-3 * (i & 7);
  __syncthreads();
  double x = 1.0;
  const long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
    if (BAR) asm volatile("bar.sync 1, %0;" ::"r"(nt) : "memory");
    double v[NL];
#pragma unroll
    for (int k = 0; k < NL; ++k) v[k] = ring[k * 1024 + ((t + 1 + k) & 1023)];
#pragma unroll
    for (int k = 0; k < NL; ++k) x = fma(v[k], 0.5, x * 0.999);
#pragma unroll
    for (int k = 0; k < NS; ++k) ring[(NL + k) * 1024 + t] = x + k;
  }
  const long long t1 = clock64();
  out[blockIdx.x * nt + t] = x;
  if (t == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int NL, int NS, bool BAR>
void run(double* d, long long* c, int warps) {
  const int n = 2000;
  const size_t sm = (size_t)(NL + NS) * 1024 * 8;
  cudaFuncSetAttribute(k_phase<NL, NS, BAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_phase<NL, NS, BAR><<<148, 32 * warps, sm>>>(d, n, c);
  k_phase<NL, NS, BAR><<<148, 32 * warps, sm>>>(d, n, c);
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("warps %2d loads %2d stores %d bar %d: %7.1f cycles per phase (%s)\n", warps, NL, NS, BAR, h / (double)n,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 1 << 24);
  cudaMalloc(&c, 4096 * 8);
  for (int w : {1, 9}) {
    run<1, 2, true>(d, c, w);
    run<4, 2, true>(d, c, w);
    run<8, 2, true>(d, c, w);
    run<16, 2, true>(d, c, w);
    run<8, 2, false>(d, c, w);
  }
  return 0;
}
