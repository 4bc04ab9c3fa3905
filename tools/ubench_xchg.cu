// Microbenchmark: latency of one fp64 all-reduce across CTAs on sm_100a.
//  (1) LL slots in global memory (64-bit words carrying 32 data bits + epoch),
//      cooperative launch of G CTAs;
//  (2) one thread-block cluster of C CTAs exchanging through DSMEM with
//      barrier.cluster.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void ll_kernel(unsigned long long* slots, int iters, double* out, long long* cyc) {
  const int G = gridDim.x, cta = blockIdx.x;
  __shared__ double s_total;
  double acc = 0;
  long long t0 = clock64();
  for (int it = 1; it <= iters; ++it) {
    unsigned long long* sl = slots + (it & 1) * G * 2;
    const double v = cta + it;
    if (threadIdx.x == 0) {
      unsigned long long bits = (unsigned long long)__double_as_longlong(v);
      unsigned long long w0 = ((unsigned long long)(unsigned)it << 32) | (bits >> 32);
      unsigned long long w1 = ((unsigned long long)(unsigned)it << 32) | (bits & 0xffffffffULL);
      asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(sl + 2 * cta), "l"(w0), "l"(w1) : "memory");
    }
    if (threadIdx.x < 32) {
      double part = 0;
      for (int b = threadIdx.x; b < G; b += 32) {
        unsigned long long w0, w1;
        for (;;) {
          asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(sl + 2 * b) : "memory");
          if ((unsigned)(w0 >> 32) == (unsigned)it && (unsigned)(w1 >> 32) == (unsigned)it) break;
        }
        part += __longlong_as_double((long long)(((w0 & 0xffffffffULL) << 32) | (w1 & 0xffffffffULL)));
      }
      for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (threadIdx.x == 0) s_total = part;
    }
    __syncthreads();
    acc += s_total;
  }
  if (threadIdx.x == 0) { cyc[cta] = clock64() - t0; out[cta] = acc; }
}

__global__ void gridsync_kernel(int iters, long long* cyc) {
  cg::grid_group g = cg::this_grid();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) g.sync();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

__global__ void cluster_kernel(int iters, double* out, long long* cyc) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double slot[2];
  const int C = cl.num_blocks(), me = cl.block_rank();
  double acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (threadIdx.x == 0) slot[it & 1] = me + it;
    cl.sync();
    if (threadIdx.x < 32) {
      double part = 0;
      for (int b = threadIdx.x; b < C; b += 32) part += *cl.map_shared_rank(&slot[it & 1], b);
      for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (threadIdx.x == 0) acc += part;
    }
  }
  if (threadIdx.x == 0) { cyc[blockIdx.x] = clock64() - t0; out[blockIdx.x] = acc; }
}

int main() {
  unsigned long long* slots; double* out; long long* cyc;
  cudaMalloc(&slots, 8 * 1024); cudaMalloc(&out, 8 * 1024); cudaMalloc(&cyc, 8 * 1024);
  const int iters = 2000;
  long long h[256];
  for (int G : {4, 16, 40, 79, 148}) {
    cudaMemset(slots, 0, 8 * 1024);
    int it = iters;
    void* args[] = {&slots, &it, &out, &cyc};
    cudaLaunchCooperativeKernel((void*)ll_kernel, G, 256, args, 0, 0);
    cudaMemcpy(h, cyc, 8 * G, cudaMemcpyDeviceToHost);
    printf("LL allreduce  G=%3d: %6.0f cycles/round  (%s)\n", G, (double)h[0] / iters,
           cudaGetErrorString(cudaGetLastError()));
    void* a2[] = {&it, &cyc};
    cudaLaunchCooperativeKernel((void*)gridsync_kernel, G, 256, a2, 0, 0);
    cudaMemcpy(h, cyc, 8 * G, cudaMemcpyDeviceToHost);
    printf("cg grid.sync  G=%3d: %6.0f cycles/round\n", G, (double)h[0] / iters);
  }
  cudaFuncSetAttribute(cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int C : {2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = C; cfg.blockDim = 1024;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, cluster_kernel, iters, out, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 8 * C, cudaMemcpyDeviceToHost);
    printf("cluster DSMEM C=%3d: %6.0f cycles/round  (%s)\n", C, (double)h[0] / iters, cudaGetErrorString(e));
  }
  return 0;
}
