// tc_i8_check.cu -- layout check for tcgen05.mma.kind::i8 as the exact
// (Ozaki-sliced) X-stream kernel uses it: A (128 x K int8) written to tensor
// memory by tcgen05.st (four int8 per 32-bit column, k ascending from the low
// byte; 8 columns per K = 32 step), B (N x K int8, K-major) in shared memory
// in the TMA SWIZZLE_128B layout (rows of 128 B, 8-row groups 1 KB apart, the
// 16-byte chunk c of row n at chunk c ^ (n % 8)), int32 accumulation in
// tensor memory; D read back and compared with a CPU integer product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc_i8_check tools/tc_i8_check.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
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
// kind::i8: D s32 (2 << 4), A and B signed 8-bit (1 << 7, 1 << 10), K-major
__host__ __device__ constexpr uint32_t idesc_i8(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
}

constexpr int N = 80;
constexpr int K = 128;  // four K = 32 steps: one 128-byte swizzle row

__host__ __device__ inline int b_off(int n, int k) {
  return (n / 8) * 1024 + (n % 8) * 128 + ((((k / 16) ^ (n % 8)) * 16) + (k % 16));
}

__global__ void kern(const int8_t* a, const int8_t* b, int* d) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* sb = smem_raw + (sbase - smem_u32(smem_raw));
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < N * K; e += blockDim.x) {
    const int n = e / K, k = e % K;
    sb[b_off(n, k)] = (uint8_t)b[n * K + k];
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
  {  // A: row r = 32 * warp + lane; columns 128 + k / 4, byte k % 4
    const int r = 32 * warp + lane;
    uint32_t v[32];
    for (int j = 0; j < 32; ++j) {
      uint32_t w = 0;
      for (int u = 0; u < 4; ++u) w |= (uint32_t)(uint8_t)a[r * K + 4 * j + u] << (8 * u);
      v[j] = w;
    }
    const uint32_t ta = tm + ((uint32_t)(32 * warp) << 16) + 128;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
        "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
        "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) {
    const uint32_t id = idesc_i8(N);
    for (int ks = 0; ks < K / 32; ++ks) {
      const uint64_t bd = desc(sbase + ks * 32, 16, 1024, 2);
      const uint32_t at = tm + 128 + 8 * ks;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm),
                   "r"(at), "l"(bd), "r"(id), "r"(ks)
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  {
    const int r = 32 * warp + lane;
    for (int c = 0; c < N; c += 16) {
      uint32_t h[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(h[0]), "=r"(h[1]), "=r"(h[2]), "=r"(h[3]), "=r"(h[4]), "=r"(h[5]), "=r"(h[6]), "=r"(h[7]),
            "=r"(h[8]), "=r"(h[9]), "=r"(h[10]), "=r"(h[11]), "=r"(h[12]), "=r"(h[13]), "=r"(h[14]), "=r"(h[15])
          : "r"(tm + ((uint32_t)(32 * warp) << 16) + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int j = 0; j < 16; ++j) d[r * N + c + j] = (int)h[j];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
  }
}

int main() {
  std::vector<int8_t> a(128 * K), b(N * K);
  srand(7);
  for (auto& v : a) v = (int8_t)((rand() % 129) - 64);
  for (auto& v : b) v = (int8_t)((rand() % 129) - 64);
  int8_t *da, *db;
  int* dd;
  cudaMalloc(&da, a.size());
  cudaMalloc(&db, b.size());
  cudaMalloc(&dd, 128 * N * 4);
  cudaMemcpy(da, a.data(), a.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size(), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaMemset(dd, 0, 128 * N * 4);
  kern<<<1, 128, 64 * 1024>>>(da, db, dd);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<int> d(128 * N);
  cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int r = 0; r < 128; ++r)
    for (int n = 0; n < N; ++n) {
      int ref = 0;
      for (int k = 0; k < K; ++k) ref += (int)a[r * K + k] * (int)b[n * K + k];
      bad += ref != d[r * N + n];
      if (ref != d[r * N + n] && bad <= 4) printf("  d[%d][%d] = %d, want %d\n", r, n, d[r * N + n], ref);
    }
  printf("kind::i8 TS, K-major SW128 B: %s, %d of %d entries wrong\n", cudaGetErrorString(e), bad, 128 * N);
  return bad != 0 || e != cudaSuccess;
}
