// tc_f16_check.cu -- layout check for tcgen05.mma.kind::f16 as the X-stream
// kernel would use it: A (128 x 32 fp16, two K=16 steps) written to tensor
// memory by tcgen05.st (two fp16 per 32-bit column, even k in the low half),
// B (32 x N fp16, MN-major) in shared memory with the TMA-style SWIZZLE_128B
// layout (64-element atoms x 8 K-rows), fp32 accumulation; D read back and
// compared with a CPU product.  One CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc_f16_check tools/tc_f16_check.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>

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
__host__ __device__ constexpr uint32_t idesc_f16(int n, bool b_mn) {
  return (1u << 4) | (0u << 7) | (0u << 10) | ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(n >> 3) << 17) |
         ((128u >> 4) << 24);
}

constexpr int N = 128;  // two 64-column atoms
constexpr int K = 32;

// B element (k, n) in the SW128 MN-major layout: atom a = n / 64 holds
// K rows of 128 B (64 halves); row k of atom a at a * (K * 128) + k * 128;
// the 16-byte chunk c = (n % 64) / 8 is stored at chunk c ^ (k % 8).
__host__ __device__ inline int b_off(int k, int n) {
  const int a = n / 64, nn = n % 64, c = nn / 8, w = nn % 8;
  return a * (K * 128) + k * 128 + (((c ^ (k & 7)) * 16) + w * 2);
}

__global__ void kern(const __half* a, const __half* b, float* d, uint32_t lbo, uint32_t sbo, int mode) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* sb = smem_raw + (sbase - smem_u32(smem_raw));
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < K * N; e += blockDim.x) {
    const int k = e / N, n = e % N;
    *reinterpret_cast<__half*>(sb + b_off(k, n)) = b[k * N + n];
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  // A: row r = 32 * warp + lane; columns 128 + (k / 2), low half = even k
  {
    const int r = 32 * warp + lane;
    uint32_t v[16];
    for (int j = 0; j < 16; ++j) {
      const __half lo = a[r * K + 2 * j], hi = a[r * K + 2 * j + 1];
      v[j] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
    }
    const uint32_t ta = tm + ((uint32_t)(32 * warp) << 16) + 128;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) {
    const uint32_t id = idesc_f16(N, true);
    for (int ks = 0; ks < K / 16; ++ks) {
      const uint64_t bd = desc(sbase + ks * 2 * 1024, lbo, sbo, 2);
      const uint32_t at = tm + 128 + 8 * ks;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm),
                   "r"(at), "l"(bd), "r"(id), "r"(ks)
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  {
    const int r = 32 * warp + lane;
    for (int c = 0; c < N; c += 32) {
      uint32_t h[32];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(h[0]), "=r"(h[1]), "=r"(h[2]), "=r"(h[3]), "=r"(h[4]), "=r"(h[5]), "=r"(h[6]), "=r"(h[7]),
            "=r"(h[8]), "=r"(h[9]), "=r"(h[10]), "=r"(h[11]), "=r"(h[12]), "=r"(h[13]), "=r"(h[14]), "=r"(h[15]),
            "=r"(h[16]), "=r"(h[17]), "=r"(h[18]), "=r"(h[19]), "=r"(h[20]), "=r"(h[21]), "=r"(h[22]), "=r"(h[23]),
            "=r"(h[24]), "=r"(h[25]), "=r"(h[26]), "=r"(h[27]), "=r"(h[28]), "=r"(h[29]), "=r"(h[30]), "=r"(h[31])
          : "r"(tm + ((uint32_t)(32 * warp) << 16) + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int j = 0; j < 32; ++j) d[r * N + c + j] = __uint_as_float(h[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
  }
}

int main(int argc, char** argv) {
  std::vector<__half> a(128 * K), b(K * N);
  std::vector<float> af(128 * K), bf(K * N);
  srand(7);
  for (int i = 0; i < 128 * K; ++i) { af[i] = (float)((rand() % 17) - 8) / 8.f; a[i] = __float2half(af[i]); }
  for (int i = 0; i < K * N; ++i) { bf[i] = (float)((rand() % 13) - 6) / 4.f; b[i] = __float2half(bf[i]); }
  __half *da, *db; float* dd;
  cudaMalloc(&da, a.size() * 2); cudaMalloc(&db, b.size() * 2); cudaMalloc(&dd, 128 * N * 4);
  cudaMemcpy(da, a.data(), a.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size() * 2, cudaMemcpyHostToDevice);
  const uint32_t cands[][2] = {{K * 128, 1024}, {1024, K * 128}, {K * 128, 512}, {16, 1024}};
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (auto& c : cands) {
    cudaMemset(dd, 0, 128 * N * 4);
    kern<<<1, 128, 64 * 1024>>>(da, db, dd, c[0], c[1], 0);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> d(128 * N);
    cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost);
    double worst = 0; int bad = 0;
    for (int r = 0; r < 128; ++r)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)af[r * K + k] * bf[k * N + n];
        const double err = fabs(ref - d[r * N + n]);
        worst = fmax(worst, err);
        bad += err > 1e-3;
      }
    printf("LBO %u SBO %u: %s, worst |err| %.3g, bad %d of %d, d[0]=%g d[1]=%g d[64]=%g\n", c[0], c[1],
           cudaGetErrorString(e), worst, bad, 128 * N, d[0], d[1], d[64]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
