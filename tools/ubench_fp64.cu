// Microbenchmark: sm_100a throughput of DFMA, FFMA and F2F.F64.F32 (cycles per
// warp-instruction per SM), used to pick the HALS kernels' arithmetic mix.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_k(double* out, int iters) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 1.0000001, c = 1e-9;
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void ffma_k(float* out, int iters) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const float b = 1.0000001f, c = 1e-9f;
  for (int i = 0; i < iters; ++i) {
    a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
    a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void f2f_k(double* out, const float* in, int iters) {
  float x0 = in[threadIdx.x & 7], x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += (double)x0 + (double)x1 + (double)x2 + (double)x3;
    x0 += 1.f; x1 += 1.f; x2 += 1.f; x3 += 1.f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* dout; float* fout; float* fin;
  cudaMalloc(&dout, 1 << 24); cudaMalloc(&fout, 1 << 24); cudaMalloc(&fin, 1024);
  cudaMemset(fin, 0, 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = nsm * 4, threads = 512, iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(e0); dfma_k<<<blocks, threads>>>(dout, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double n = (double)blocks * threads * iters * 8;
    if (rep) printf("DFMA: %.1f TFLOP/s, %.1f DFMA/clk/SM (clk %.0f MHz)\n", 2 * n / ms / 1e9, n / (ms * 1e-3) / nsm / (clk * 1e3), clk / 1e3);
    cudaEventRecord(e0); ffma_k<<<blocks, threads>>>(fout, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("FFMA: %.1f TFLOP/s, %.1f FFMA/clk/SM\n", 2 * n / ms / 1e9, n / (ms * 1e-3) / nsm / (clk * 1e3));
    cudaEventRecord(e0); f2f_k<<<blocks, threads>>>(dout, fin, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double nc = (double)blocks * threads * iters * 4;
    if (rep) printf("F2F.F64.F32 (+DADD): %.1f conv/clk/SM\n", nc / (ms * 1e-3) / nsm / (clk * 1e3));
  }
  return 0;
}
