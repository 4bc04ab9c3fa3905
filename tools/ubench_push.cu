// Microbenchmark: the per-column norm all-reduce of the HALS kernels, two
// protocols, cycles per all-reduce on CTA 0's clock (cooperative launch, one
// CTA of 256 threads per SM):
//   (a) counter: tagged partial into one shared array, relaxed arrive on a
//       monotonic counter, warp poll of the counter, batched tagged read of
//       the G partials (hals_common.cuh allreduce_fused as committed);
//   (b) push: every CTA stores its tagged partial into all G CTAs' PRIVATE
//       arrays and polls only its own array's tags -- no counter, one L2
//       store latency plus one load round trip after the last arrival.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/ubench_push tools/ubench_push.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double wsum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ void st_relaxed(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ double ld_relaxed(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ bool tag_neg(unsigned long long nr) { return ((nr >> 1) & 1ULL) == 0; }

__device__ __forceinline__ double sum_tagged(const double* p, int G, int lane, bool neg) {
  double v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int b = lane + 32 * i;
    v[i] = b < G ? ld_relaxed(p + b) : (neg ? -0.0 : 0.0);
  }
  for (;;) {
    bool stale = false;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int b = lane + 32 * i;
      if (b < G && (signbit(v[i]) != 0) != neg) {
        stale = true;
        v[i] = ld_relaxed(p + b);
      }
    }
    if (!__any_sync(0xffffffffu, stale)) break;
  }
  double t = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) t += fabs(v[i]);
  return wsum(t);
}

// work: busy cycles between all-reduces (stands for the column update), so
// the CTAs do not arrive in lock step
template <int kMode>
__global__ void __launch_bounds__(256, 1)
    ar_kernel(double* slots, unsigned* ctr, int iters, int work, double* out, long long* cyc) {
  const int G = gridDim.x, cta = blockIdx.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __shared__ double red8[8], s_out;
  double acc = 0.0;
  unsigned long long nr = 0, ep = 0;
  const long long t0 = clock64();
  long long spent = 0;
  for (int it = 0; it < iters; ++it) {
    if (work) {
      const long long w0 = clock64();
      while (clock64() - w0 < work + ((cta * 7 + it) & 63)) {
      }
    }
    const long long a0 = clock64();
    double v = 1.0 + 1e-3 * (double)((threadIdx.x + cta + it) & 15);
    v = wsum(v);
    if (lane == 0) red8[wid] = v;
    __syncthreads();
    ++ep;
    if (wid == 0) {
      const bool neg = tag_neg(nr);
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) t += red8[w];
      const double tv = neg ? -t : t;
      double tot;
      if (kMode == 0) {
        double* slot = slots + (nr & 1ULL) * G;
        if (lane == 0) {
          st_relaxed(slot + cta, tv);
          asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        }
        unsigned c;
        const unsigned target = (unsigned)(ep * (unsigned long long)G);
        do {
          asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(ctr) : "memory");
        } while (__any_sync(0xffffffffu, (int)(c - target) < 0));
        tot = sum_tagged(slot, G, lane, neg);
      } else {
        // private arrays: [buffer][destination][source], 256 doubles per row
        double* base = slots + (nr & 1ULL) * (size_t)G * 256;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int dst = lane + 32 * i;
          if (dst < G) st_relaxed(base + (size_t)dst * 256 + cta, tv);
        }
        tot = sum_tagged(base + (size_t)cta * 256, G, lane, neg);
      }
      if (lane == 0) s_out = tot;
    }
    ++nr;
    __syncthreads();
    acc += s_out;
    spent += clock64() - a0;
  }
  if (threadIdx.x == 0) {
    cyc[2 * cta] = clock64() - t0;
    cyc[2 * cta + 1] = spent;
    out[cta] = acc;
  }
}

int main() {
  double* slots;
  unsigned* ctr;
  double* out;
  long long* cyc;
  const size_t slot_bytes = 2 * 256 * 256 * sizeof(double);
  cudaMalloc(&slots, slot_bytes);
  cudaMalloc(&ctr, 64);
  cudaMalloc(&out, 8 * 256);
  cudaMalloc(&cyc, 16 * 256);
  int iters = 4000;
  long long h[512];
  double ho[256];
  for (int G : {16, 148})
    for (int work : {0, 2000}) {
      for (int mode = 0; mode < 2; ++mode) {
        cudaMemset(slots, 0, slot_bytes);
        cudaMemset(ctr, 0, 64);
        void* args[] = {&slots, &ctr, &iters, &work, &out, &cyc};
        cudaError_t e = mode == 0 ? cudaLaunchCooperativeKernel((void*)ar_kernel<0>, G, 256, args, 0, 0)
                                  : cudaLaunchCooperativeKernel((void*)ar_kernel<1>, G, 256, args, 0, 0);
        cudaDeviceSynchronize();
        cudaMemcpy(h, cyc, 16 * G, cudaMemcpyDeviceToHost);
        cudaMemcpy(ho, out, 8 * G, cudaMemcpyDeviceToHost);
        bool same = true;
        for (int g = 1; g < G; ++g) same = same && ho[g] == ho[0];
        printf("%-8s G=%3d work=%4d: %6.0f cycles per all-reduce (in-call %6.0f)  sum %.6f %s (%s)\n",
               mode == 0 ? "counter" : "push", G, work, (double)h[0] / iters - work - 32,
               (double)h[1] / iters, ho[0], same ? "identical on every CTA" : "MISMATCH",
               cudaGetErrorString(e));
      }
    }
  return 0;
}
