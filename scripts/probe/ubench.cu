// Micro-benchmarks of the latencies that bound the single-pass iteration kernel on B200
// (DESIGN.md sec. 6): dependent DFMA / DMUL chains, shared-memory load-to-use, named-barrier
// round trips with 10 warps, and FP64 issue throughput with independent chains.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench ubench.cu && ./ubench
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma_chain(double* out, double a, double b, int n, long long* cyc) {
  double x = threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) x = fma(x, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_dmul_chain(double* out, double a, int n, long long* cyc) {
  double x = threadIdx.x * 1e-3 + 1.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) x = x * a;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
// ILP chains per thread, many warps: FP64 throughput per SM
template <int C>
__global__ void k_dfma_tput(double* out, double a, double b, int n, long long* cyc) {
  double x[C];
#pragma unroll
  for (int c = 0; c < C; ++c) x[c] = threadIdx.x * 1e-3 + c;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < C; ++c) x[c] = fma(x[c], a, b);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
// shared-memory load to use: pointer chase through shared memory
__global__ void k_lds_chase(int* out, int n, long long* cyc) {
  __shared__ int buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = (i + 33) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) p = buf[p];
  long long t1 = clock64();
  out[threadIdx.x] = p;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
// shared double load -> DFMA -> shared store chain (the row pipeline's pattern)
__global__ void k_lds_dfma(double* out, int n, long long* cyc) {
  __shared__ double buf[64];
  buf[threadIdx.x] = 1.0;
  __syncwarp();
  double x = 0.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    const double v = buf[(threadIdx.x + i) & 31];
    x = fma(v, x, 0.25);
    buf[threadIdx.x] = x;
    __syncwarp();
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
// named barrier round trip with nthreads threads (all arrive together)
__global__ void k_bar(int n, long long* cyc) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) asm volatile("bar.sync 1, %0;" ::"r"((int)blockDim.x) : "memory");
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
// barrier + a dependent store/load exchange through shared memory between neighbours
__global__ void k_bar_xchg(double* out, int n, long long* cyc) {
  __shared__ double ring[2][1024];
  double x = threadIdx.x;
  ring[0][threadIdx.x] = x;
  ring[1][threadIdx.x] = x;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    const int s = i & 1;
    ring[s][threadIdx.x] = x;
    asm volatile("bar.sync 1, %0;" ::"r"((int)blockDim.x) : "memory");
    x = fma(ring[s][(threadIdx.x + 1) % blockDim.x], 0.5, x * 0.25);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
// cluster barrier round trip (arrive.release + wait.acquire) with 4-CTA clusters
__global__ void __cluster_dims__(4, 1, 1) k_cluster_bar(int n, long long* cyc) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* dout;
  long long* dc;
  int* iout;
  cudaMalloc(&dout, 1 << 24);
  cudaMalloc(&iout, 1 << 20);
  cudaMalloc(&dc, 4096 * 8);
  long long c[512];
  const int n = 1000;
  k_dfma_chain<<<1, 32>>>(dout, 0.999, 1e-3, n, dc);
  k_dfma_chain<<<1, 32>>>(dout, 0.999, 1e-3, n, dc);
  cudaMemcpy(c, dc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", c[0] / (16.0 * n));
  k_dmul_chain<<<1, 32>>>(dout, 0.999, n, dc);
  k_dmul_chain<<<1, 32>>>(dout, 0.999, n, dc);
  cudaMemcpy(c, dc, 8, cudaMemcpyDeviceToHost);
  printf("DMUL dependent latency: %.2f cycles\n", c[0] / (16.0 * n));
  for (int warps : {4, 8, 16, 32}) {
    k_dfma_tput<8><<<148, 32 * warps>>>(dout, 0.999, 1e-3, n, dc);
    k_dfma_tput<8><<<148, 32 * warps>>>(dout, 0.999, 1e-3, n, dc);
    cudaMemcpy(c, dc, 8, cudaMemcpyDeviceToHost);
    const double fl = 8.0 * 8 * n * 32 * warps;   // DFMA lanes per SM
    printf("DFMA throughput, %2d warps x 8 chains: %.1f lane-FMA/cycle/SM\n", warps, fl / c[0]);
  }
  k_lds_chase<<<1, 32>>>(iout, n, dc);
  k_lds_chase<<<1, 32>>>(iout, n, dc);
  cudaMemcpy(c, dc, 8, cudaMemcpyDeviceToHost);
  printf("LDS.32 pointer-chase latency: %.2f cycles\n", c[0] / (double)n);
  k_lds_dfma<<<1, 32>>>(dout, n, dc);
  k_lds_dfma<<<1, 32>>>(dout, n, dc);
  cudaMemcpy(c, dc, 8, cudaMemcpyDeviceToHost);
  printf("LDS.64 -> DFMA -> STS -> syncwarp loop: %.2f cycles\n", c[0] / (double)n);
  for (int t : {64, 128, 288, 320, 512}) {
    k_bar<<<1, t>>>(n, dc);
    k_bar<<<1, t>>>(n, dc);
    cudaMemcpy(c, dc, 8, cudaMemcpyDeviceToHost);
    printf("bar.sync round trip, %3d threads: %.2f cycles\n", t, c[0] / (double)n);
    k_bar_xchg<<<1, t>>>(dout, n, dc);
    k_bar_xchg<<<1, t>>>(dout, n, dc);
    cudaMemcpy(c, dc, 8, cudaMemcpyDeviceToHost);
    printf("STS -> bar.sync -> LDS -> DFMA exchange, %3d threads: %.2f cycles\n", t, c[0] / (double)n);
  }
  k_cluster_bar<<<4, 288>>>(n, dc);
  k_cluster_bar<<<4, 288>>>(n, dc);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(c, dc, 8, cudaMemcpyDeviceToHost);
  printf("cluster barrier (4 CTAs x 288 threads): %.2f cycles (%s)\n", c[0] / (double)n, cudaGetErrorString(e));
  return 0;
}
