// common.cuh -- shared device helpers for the cnmf-b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cuda/atomic>

#include <atomic>

namespace cnmf {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is a per-device setting:
// each call site keeps one bit per device in `done` (a second context on
// another device of the same process sets it there too).
inline void smem_attr_once(std::atomic<unsigned>& done, const void* fn, int bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned bit = 1u << (dev & 31);
  if (!(done.load(std::memory_order_acquire) & bit)) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    done.fetch_or(bit, std::memory_order_acq_rel);
  }
}

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

__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// Epoch-tagged all-to-all exchange for a cooperative launch (replaces a
// counter barrier + a separate partial read).  Every CTA writes its payload
// with plain stores, then publish() release-stores the epoch into its own
// tag; wait_all() polls all G tags with acquire loads.  Tags and payloads are
// double-buffered by epoch parity: a CTA can only publish epoch e+2 after all
// CTAs published e+1, i.e. after everyone finished reading epoch e.
__device__ __forceinline__ void xchg_publish(unsigned long long* tags, int cta,
                                             unsigned long long epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_acq_rel_gpu();
    st_release_u64(tags + cta, epoch);
  }
}
__device__ __forceinline__ void xchg_wait(const unsigned long long* tags, int G,
                                          unsigned long long epoch) {
  if (threadIdx.x < 32) {
    // Each lane checks all of its (<= 8) tags per round with relaxed loads
    // issued together (one L2 round trip per round, no L1 invalidation), then
    // one acquire fence once every tag shows the epoch.
    for (;;) {
      bool ready = true;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int b = threadIdx.x + 32 * i;
        if (b < G && ld_relaxed_u64(tags + b) < epoch) ready = false;
      }
      if (__all_sync(0xffffffffu, ready)) break;
      __nanosleep(20);
    }
    fence_acq_rel_gpu();
  }
  __syncthreads();
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
