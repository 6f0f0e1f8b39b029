// FP64 dependent-chain latency under load on B200: W warps per SM (one CTA per SM), each thread
// running ILP independent chains of dependent DFMAs; reports cycles per chain link.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench2 ubench2.cu && ./ubench2
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void k_chain(double* out, double a, double b, int n, long long* cyc) {
  double x[ILP];
#pragma unroll
  for (int c = 0; c < ILP; ++c) x[c] = threadIdx.x * 1e-3 + c;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < ILP; ++c) x[c] = fma(x[c], a, b);
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < ILP; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
// a shared-memory round trip in the chain: x -> STS -> LDS (other lane) -> DFMA, W warps
__global__ void k_lds_chain(double* out, int n, long long* cyc) {
  extern __shared__ double sh[];
  double x = threadIdx.x * 1e-3;
  sh[threadIdx.x] = x;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    const double v = sh[threadIdx.x ^ 1];
    x = fma(v, 0.5, x);
    sh[threadIdx.x] = x;
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int ILP>
void run(double* d, long long* c, int warps) {
  const int n = 500;
  k_chain<ILP><<<148, 32 * warps>>>(d, 0.999, 1e-3, n, c);
  k_chain<ILP><<<148, 32 * warps>>>(d, 0.999, 1e-3, n, c);
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DFMA chains: %2d warps/SM, ILP %d: %.2f cycles per link, %.1f lane-FMA/cycle/SM\n", warps, ILP,
         h / (8.0 * n), 8.0 * n * ILP * 32 * warps / h);
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 1 << 26);
  cudaMalloc(&c, 4096 * 8);
  for (int w : {1, 4, 8, 10, 12, 16}) { run<1>(d, c, w); run<2>(d, c, w); run<4>(d, c, w); }
  for (int w : {1, 4, 10, 16}) {
    const int n = 500;
    k_lds_chain<<<148, 32 * w, 32 * w * 8>>>(d, n, c);
    k_lds_chain<<<148, 32 * w, 32 * w * 8>>>(d, n, c);
    long long h;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("LDS->DFMA->STS chain, %2d warps/SM: %.2f cycles per link\n", w, h / (double)n);
  }
  return 0;
}
