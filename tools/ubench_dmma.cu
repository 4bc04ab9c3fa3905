// Microbenchmark: sm_100a throughput of the FP64 tensor-core MMA
// (mma.sync.aligned.m8n8k4.row.col.f64) against DFMA, per SM.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_kernel(int iters, double* out) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[4][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 4; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c[t][0]), "+d"(c[t][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
  for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * p.multiProcessorCount * 1024);
  for (int warps : {4, 8, 16}) {
    const int iters = 20000;
    dmma_kernel<<<p.multiProcessorCount, 32 * warps>>>(10, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    dmma_kernel<<<p.multiProcessorCount, 32 * warps>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 256 * 4 * (double)iters * warps * p.multiProcessorCount;
    printf("DMMA m8n8k4, %d warps/SM: %.1f TFLOP/s (%s)\n", warps, flops / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
