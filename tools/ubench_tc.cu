// ubench_tc.cu -- cycles per tcgen05.mma.kind::tf32 (M=128, K=8) issued back to
// back by one thread, by N, number of independent accumulator chains, and A
// operand source (tensor memory vs shared memory).  Operand contents are
// irrelevant (zeros).  One CTA per SM, all SMs busy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_tc tools/ubench_tc.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_tf32(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
}

template <int N, int CHAINS, bool ATMEM, bool WARP = false>
__global__ void __launch_bounds__(128, 1) bench(int rounds, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  if (WARP ? warp == 0 : threadIdx.x == 0) {
    constexpr uint32_t id = idesc_tf32(N);
    const uint64_t bd = desc(base, 4096, 512, 1);            // MN-major B
    const uint64_t ad = desc(base + 65536, 16, 1024, 2);     // K-major A (SS mode)
    const uint32_t a_t = tm + 384;                           // A in TMEM (TS mode)
    long long t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
#pragma unroll
      for (int i = 0; i < 12; ++i) {
        const uint32_t d = tm + (i % CHAINS) * N;
        if (WARP) {  // converged warp, one elected lane issues inside the asm
          if (ATMEM)
            asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                         "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                         "r"(a_t), "l"(bd + (uint64_t)(i * 64)), "r"(id), "r"(1u)
                         : "memory");
          else
            asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                         "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                         "l"(ad), "l"(bd + (uint64_t)(i * 64)), "r"(id), "r"(1u)
                         : "memory");
        } else if (ATMEM)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                       "r"(a_t), "l"(bd), "r"(id), "r"(1u)
                       : "memory");
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                       "l"(ad), "l"(bd), "r"(id), "r"(1u)
                       : "memory");
      }
    }
    if (!WARP || (threadIdx.x & 31) == 0)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&bar))
                   : "memory");
    asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(
                     smem_u32(&bar))
                 : "memory");
    long long t1 = clock64();
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
  }
}

template <int N, int CHAINS, bool ATMEM, bool WARP = false>
void run(long long* d_out) {
  const int smem = 140 * 1024;
  cudaFuncSetAttribute(bench<N, CHAINS, ATMEM, WARP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int rounds = 2000;
  bench<N, CHAINS, ATMEM, WARP><<<148, 128, smem>>>(10, d_out);
  bench<N, CHAINS, ATMEM, WARP><<<148, 128, smem>>>(rounds, d_out);
  long long c = 0;
  cudaError_t e = cudaMemcpy(&c, d_out, 8, cudaMemcpyDeviceToHost);
  const double per = (double)c / (rounds * 12.0);
  const double floor = 128.0 * N / 256.0;
  printf("%s N=%3d chains=%d A=%s: %6.1f cyc/MMA (floor %5.1f) -> %5.1f%% %s\n", WARP ? "warp  " : "thread", N, CHAINS, ATMEM ? "tmem" : "smem",
         per, floor, 100.0 * floor / per, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  run<32, 1, true>(d);  run<32, 1, true, true>(d);  run<32, 1, false, true>(d);
  run<64, 1, true>(d);  run<64, 1, true, true>(d);  run<64, 1, false, true>(d);
  run<96, 1, true>(d);  run<96, 1, true, true>(d);  run<96, 1, false, true>(d);
  run<128, 1, true, true>(d); run<192, 1, true, true>(d); run<192, 1, false, true>(d);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
