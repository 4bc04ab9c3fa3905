// Microbenchmark: deterministic fp64 all-reduce variants across the CTAs of a
// cooperative launch on sm_100a (cycles per all-reduce, CTA 0's clock).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double wsum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// (a) LL slots written with atom.exch (goes straight to L2)
__global__ void ll_exch(unsigned long long* slots, int iters, double* out, long long* cyc) {
  const int G = gridDim.x, cta = blockIdx.x;
  __shared__ double s_total;
  double acc = 0;
  long long t0 = clock64();
  for (int it = 1; it <= iters; ++it) {
    unsigned long long* sl = slots + (it & 1) * G * 2;
    const double v = cta + it;
    if (threadIdx.x == 0) {
      unsigned long long bits = (unsigned long long)__double_as_longlong(v);
      atomicExch(sl + 2 * cta, ((unsigned long long)(unsigned)it << 32) | (bits >> 32));
      atomicExch(sl + 2 * cta + 1, ((unsigned long long)(unsigned)it << 32) | (bits & 0xffffffffULL));
    }
    if (threadIdx.x < 32) {
      double part = 0;
      for (int b = threadIdx.x; b < G; b += 32) {
        unsigned long long w0, w1;
        do {
          asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w0) : "l"(sl + 2 * b) : "memory");
          asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w1) : "l"(sl + 2 * b + 1) : "memory");
        } while ((unsigned)(w0 >> 32) != (unsigned)it || (unsigned)(w1 >> 32) != (unsigned)it);
        part += __longlong_as_double((long long)(((w0 & 0xffffffffULL) << 32) | (w1 & 0xffffffffULL)));
      }
      part = wsum(part);
      if (threadIdx.x == 0) s_total = part;
    }
    __syncthreads();
    acc += s_total;
  }
  if (threadIdx.x == 0) { cyc[cta] = clock64() - t0; out[cta] = acc; }
}
// (b) counter barrier (atomicAdd arrive, spin on counter) then read partials
__global__ void bar_read(unsigned* ctr, double* part, int iters, double* out, long long* cyc) {
  const int G = gridDim.x, cta = blockIdx.x;
  __shared__ double s_total;
  double acc = 0;
  long long t0 = clock64();
  for (int it = 1; it <= iters; ++it) {
    double* pp = part + (it & 1) * G;
    if (threadIdx.x == 0) {
      pp[cta] = cta + it;
      __threadfence();
      atomicAdd(ctr, 1u);
      const unsigned target = (unsigned)it * G;
      unsigned v;
      do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while (v < target);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      double s = 0;
      for (int b = threadIdx.x; b < G; b += 32) s += __ldcg(pp + b);
      s = wsum(s);
      if (threadIdx.x == 0) s_total = s;
    }
    __syncthreads();
    acc += s_total;
  }
  if (threadIdx.x == 0) { cyc[cta] = clock64() - t0; out[cta] = acc; }
}
// (c) last arriver reduces in fixed order and publishes an LL result word pair
__global__ void last_reduces(unsigned* ctr, double* part, unsigned long long* res, int iters, double* out, long long* cyc) {
  const int G = gridDim.x, cta = blockIdx.x;
  __shared__ double s_total;
  __shared__ int s_last;
  double acc = 0;
  long long t0 = clock64();
  for (int it = 1; it <= iters; ++it) {
    double* pp = part + (it & 1) * G;
    unsigned long long* rr = res + (it & 1) * 2;
    if (threadIdx.x == 0) {
      pp[cta] = cta + it;
      __threadfence();
      const unsigned old = atomicAdd(ctr, 1u);
      s_last = (old == (unsigned)it * G - 1);
    }
    __syncthreads();
    if (s_last && threadIdx.x < 32) {
      __threadfence();
      double s = 0;
      for (int b = threadIdx.x; b < G; b += 32) s += __ldcg(pp + b);
      s = wsum(s);
      if (threadIdx.x == 0) {
        unsigned long long bits = (unsigned long long)__double_as_longlong(s);
        atomicExch(rr, ((unsigned long long)(unsigned)it << 32) | (bits >> 32));
        atomicExch(rr + 1, ((unsigned long long)(unsigned)it << 32) | (bits & 0xffffffffULL));
      }
    }
    if (threadIdx.x == 0) {
      unsigned long long w0, w1;
      do {
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w0) : "l"(rr) : "memory");
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w1) : "l"(rr + 1) : "memory");
      } while ((unsigned)(w0 >> 32) != (unsigned)it || (unsigned)(w1 >> 32) != (unsigned)it);
      s_total = __longlong_as_double((long long)(((w0 & 0xffffffffULL) << 32) | (w1 & 0xffffffffULL)));
    }
    __syncthreads();
    acc += s_total;
  }
  if (threadIdx.x == 0) { cyc[cta] = clock64() - t0; out[cta] = acc; }
}

int main() {
  unsigned long long* slots; double* out; long long* cyc; unsigned* ctr; double* part; unsigned long long* res;
  cudaMalloc(&slots, 8 * 1024); cudaMalloc(&out, 8 * 1024); cudaMalloc(&cyc, 8 * 1024);
  cudaMalloc(&ctr, 64); cudaMalloc(&part, 8 * 1024); cudaMalloc(&res, 64);
  int iters = 2000;
  long long h[256];
  for (int G : {4, 40, 148}) {
    cudaMemset(slots, 0, 8 * 1024);
    void* a1[] = {&slots, &iters, &out, &cyc};
    cudaLaunchCooperativeKernel((void*)ll_exch, G, 256, a1, 0, 0);
    cudaMemcpy(h, cyc, 8 * G, cudaMemcpyDeviceToHost);
    printf("LL atom.exch   G=%3d: %6.0f cycles\n", G, (double)h[0] / iters);
    cudaMemset(ctr, 0, 64);
    void* a2[] = {&ctr, &part, &iters, &out, &cyc};
    cudaLaunchCooperativeKernel((void*)bar_read, G, 256, a2, 0, 0);
    cudaMemcpy(h, cyc, 8 * G, cudaMemcpyDeviceToHost);
    printf("barrier+read   G=%3d: %6.0f cycles\n", G, (double)h[0] / iters);
    cudaMemset(ctr, 0, 64); cudaMemset(res, 0, 64);
    void* a3[] = {&ctr, &part, &res, &iters, &out, &cyc};
    cudaLaunchCooperativeKernel((void*)last_reduces, G, 256, a3, 0, 0);
    cudaMemcpy(h, cyc, 8 * G, cudaMemcpyDeviceToHost);
    printf("last-reduces   G=%3d: %6.0f cycles (%s)\n", G, (double)h[0] / iters, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
