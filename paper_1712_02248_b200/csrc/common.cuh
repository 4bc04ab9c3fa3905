// common.cuh -- shared device helpers for the cnmf-b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cuda/atomic>

namespace cnmf {

constexpr int kWarp = 32;


__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ int warp_or(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v |= __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide fp64 sum in a fixed order (warp tree, then warp 0 over the
// per-warp sums).  Every thread receives the result.  `red` needs
// blockDim.x/32 doubles of shared memory.
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < nw; ++i) t += red[i];
  return t;
}

// Sense-free generation barrier over all CTAs of a cooperative launch.
// bar[0] = arrival count, bar[1] = generation.  Release/acquire at gpu
// scope orders every global write before the barrier with every read after.
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    cuda::atomic_ref<unsigned, cuda::thread_scope_device> count(bar[0]);
    cuda::atomic_ref<unsigned, cuda::thread_scope_device> gen(bar[1]);
    const unsigned my_gen = gen.load(cuda::memory_order_relaxed);
    __threadfence();
    const unsigned arrived = count.fetch_add(1u, cuda::memory_order_acq_rel);
    if (arrived == nblocks - 1) {
      count.store(0u, cuda::memory_order_relaxed);
      gen.store(my_gen + 1u, cuda::memory_order_release);
    } else {
      while (gen.load(cuda::memory_order_acquire) == my_gen) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

}  // namespace cnmf
