// device_common.cuh -- small device helpers shared by the libgmaf kernels:
// %globaltimer kernel accounting, the last-CTA-done pattern and block reductions.
#pragma once
#include <cuda_runtime.h>
#include "gmaf_internal.cuh"

namespace gmaf {

// the device's opt-in maximum of dynamic shared memory per block (host)
inline int smem_optin_max() {
  static int v = -1;
  if (v < 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
      v = 0;
  }
  return v;
}

// Raise a kernel's dynamic shared-memory cap to the device's opt-in maximum minus its static
// shared memory (their sum may not exceed the opt-in limit).
template <typename KernelT>
inline cudaError_t raise_smem_cap(KernelT kern) {
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, kern);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              smem_optin_max() - (int)a.sharedSizeBytes);
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// First thread of every CTA lowers the launch start stamp.
__device__ __forceinline__ void timing_begin(Timing* T, int kind) {
  if (threadIdx.x == 0) atomicMin(&T->t_start[kind], globaltimer());
}

// Called by one thread of the last CTA of a launch.  One dependent load (the start stamp); the
// accumulations are fire-and-forget reductions (RED), so the serial tail of a launch does not wait.
__device__ __forceinline__ void timing_end(Timing* T, int kind, unsigned long long t0) {
  const unsigned long long t = globaltimer();
  if (t0 != ~0ull && t > t0) atomicAdd(&T->total_ns[kind], t - t0);
  atomicAdd(&T->launches[kind], 1ull);
  T->t_start[kind] = ~0ull;
}
__device__ __forceinline__ void timing_end(Timing* T, int kind) { timing_end(T, kind, T->t_start[kind]); }

// Returns true in exactly one CTA: the last one to arrive.  All partial results the
// CTA wrote before the call are visible to the last CTA (fence + atomic).  The counter
// is re-armed for the next launch.
__device__ __forceinline__ bool last_cta_arrive(unsigned int* counter, unsigned int n_ctas) {
  __shared__ int am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int prev = atomicAdd(counter, 1u);
    am_last = (prev == n_ctas - 1u);
    if (am_last) *counter = 0u;
  }
  __syncthreads();
  if (am_last) __threadfence();
  return am_last != 0;
}

// Deterministic block sum that tolerates a partial last warp (blockDim need not be a
// multiple of 32): every thread parks its values in shared memory, one thread per warp
// sums its warp's slots in lane order, thread 0 sums the warps in order.  All threads of
// the block must call it; the result is valid in thread 0.  smem: >= NV*(blockDim+32).
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* smem) {
  const int nt = blockDim.x, tid = threadIdx.x;
  const int nwarps = (nt + 31) >> 5;
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) smem[q * nt + tid] = v[q];
  __syncthreads();
  double* ws = smem + NV * nt;
  if (tid < nwarps) {
    const int lo = tid * 32, hi = min(lo + 32, nt);
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double s = 0.0;
      for (int t = lo; t < hi; ++t) s += smem[q * nt + t];
      ws[q * 32 + tid] = s;
    }
  }
  __syncthreads();
  if (tid == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double s = 0.0;
      for (int w = 0; w < nwarps; ++w) s += ws[q * 32 + w];
      v[q] = s;
    }
  }
}

}  // namespace gmaf
