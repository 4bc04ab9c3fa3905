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

template <int N, int CHAINS, bool ATMEM, bool WARP = false, bool VARY = false, int BG = 0, int COMMITS = 0>
__global__ void __launch_bounds__(128, 1) bench(int rounds, long long* out, const float* gsrc) {
  __shared__ volatile int stop;
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t cbar[4];
  __shared__ uint32_t tbase;
  const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&cbar[i])));
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
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (BG == 4 && warp == 1) {
    // background bulk copies global -> shared (64 KB region at +131072), 4 x 16 KB
    // in flight, like the kernel's X stream
    __shared__ __align__(8) uint64_t tbar[4];
    if ((threadIdx.x & 31) == 0) {
      for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&tbar[i])));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      uint32_t ph[4] = {0, 0, 0, 0};
      long long it = 0;
      for (int i = 0; i < 4; ++i) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16384;" ::"r"(smem_u32(&tbar[i])) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];" ::"r"(base + 131072 + i * 16384),
                     "l"(gsrc + ((blockIdx.x * 64 + it++ * 4096) & ((1 << 26) - 1))), "r"(smem_u32(&tbar[i])) : "memory");
      }
      while (!stop) {
        for (int i = 0; i < 4 && !stop; ++i) {
          asm volatile("{\n\t.reg .pred p;\nW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W2;\n\t}" ::"r"(smem_u32(&tbar[i])), "r"(ph[i]) : "memory");
          ph[i] ^= 1;
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16384;" ::"r"(smem_u32(&tbar[i])) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];" ::"r"(base + 131072 + i * 16384),
                       "l"(gsrc + ((blockIdx.x * 4096 + it++ * 4096) & ((1 << 26) - 1))), "r"(smem_u32(&tbar[i])) : "memory");
        }
      }
      for (int i = 0; i < 4; ++i)
        asm volatile("{\n\t.reg .pred p;\nW3:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W3;\n\t}" ::"r"(smem_u32(&tbar[i])), "r"(ph[i]) : "memory");
    }
  }
  if (BG && BG < 4 && warp >= 1) {
    // background load on warps 1..3 until warp 0 finishes: 1 = tcgen05.st (32 cols
    // per warp into cols 448..479 of its lane quarter), 2 = ld.shared.v4 streaming,
    // 3 = tcgen05.ld of 32 cols
    const uint32_t q = warp & 3;
    uint32_t v[32];
    for (int j = 0; j < 32; ++j) v[j] = j;
    float acc = 0.f;
    int it = 0;
    while (!stop) {
      if (BG == 1) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tm + (q << 21) + 448),
                     "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
                     "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      } else if (BG == 2) {
        float4 t;
        const uint32_t a = base + (((threadIdx.x * 16) + it * 4096) & 0x1FFFF);
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(t.x), "=f"(t.y), "=f"(t.z), "=f"(t.w) : "r"(a) : "memory");
        acc += t.x + t.w;
      } else if (BG == 3) {
        uint32_t h[32];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                     : "=r"(h[0]), "=r"(h[1]), "=r"(h[2]), "=r"(h[3]), "=r"(h[4]), "=r"(h[5]), "=r"(h[6]), "=r"(h[7]), "=r"(h[8]), "=r"(h[9]), "=r"(h[10]), "=r"(h[11]), "=r"(h[12]), "=r"(h[13]), "=r"(h[14]), "=r"(h[15]),
                       "=r"(h[16]), "=r"(h[17]), "=r"(h[18]), "=r"(h[19]), "=r"(h[20]), "=r"(h[21]), "=r"(h[22]), "=r"(h[23]), "=r"(h[24]), "=r"(h[25]), "=r"(h[26]), "=r"(h[27]), "=r"(h[28]), "=r"(h[29]), "=r"(h[30]), "=r"(h[31])
                     : "r"(tm + (q << 21) + 448));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        acc += __uint_as_float(h[0] ^ h[31]);
      }
      ++it;
    }
    if (acc == 12345.f) out[1] = it;
  }
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
                         "r"(a_t + (VARY ? (uint32_t)((i % 8) * 8) : 0u)),
                         "l"(bd + (uint64_t)(VARY ? (((r % 6) * 24576 + (i % 4) * 1024 + (i / 4 % 2) * 12288) >> 4) : i * 64)),
                         "r"(id), "r"(1u)
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
      for (int c = 0; c < COMMITS; ++c)  // like the kernel: commits after every 12 MMAs
        asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                     "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(&cbar[c])) : "memory");
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
    stop = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
  }
}

static float* g_src = nullptr;
template <int N, int CHAINS, bool ATMEM, bool WARP = false, bool VARY = false, int BG = 0, int COMMITS = 0>
void run(long long* d_out) {
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(bench<N, CHAINS, ATMEM, WARP, VARY, BG, COMMITS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int rounds = 2000;
  bench<N, CHAINS, ATMEM, WARP, VARY, BG, COMMITS><<<148, 128, smem>>>(10, d_out, g_src);
  bench<N, CHAINS, ATMEM, WARP, VARY, BG, COMMITS><<<148, 128, smem>>>(rounds, d_out, g_src);
  long long c = 0;
  cudaError_t e = cudaMemcpy(&c, d_out, 8, cudaMemcpyDeviceToHost);
  const double per = (double)c / (rounds * 12.0);
  const double floor = 128.0 * N / 256.0;
  printf("commits%d bg%d %s%s N=%3d chains=%d A=%s: %6.1f cyc/MMA (floor %5.1f) -> %5.1f%% %s\n", COMMITS, BG, WARP ? "warp  " : "thread", VARY ? " vary" : "     ", N, CHAINS, ATMEM ? "tmem" : "smem",
         per, floor, 100.0 * floor / per, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  cudaMalloc(&g_src, (size_t)4 << 28);
  run<128, 1, true, true, true, 0, 2>(d); run<128, 1, true, true, true, 4, 2>(d);
  run<96, 1, true, true, true, 0, 2>(d); run<96, 1, true, true, true, 4, 2>(d);
  run<80, 1, true, true, true, 0, 2>(d); run<80, 1, true, true, true, 4, 2>(d);
  run<80, 2, true, true, true, 0, 2>(d);
  run<64, 1, true, true, true, 0, 2>(d); run<64, 1, true, true, true, 4, 2>(d);
  run<48, 1, true, true, true, 0, 2>(d); run<48, 1, true, true, true, 4, 2>(d);
  run<32, 1, true, true, true, 0, 2>(d); run<32, 1, true, true, true, 4, 2>(d);
  run<256, 1, true, true, true, 0, 2>(d); run<256, 1, false, true, false, 0, 2>(d);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
