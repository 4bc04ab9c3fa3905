// Microbenchmark: cooperative launch with 16-CTA clusters on sm_100a and the
// latency of a cluster-wide fp64 all-reduce through distributed shared memory
// (each CTA stores its partial into every CTA's slot array, cluster barrier,
// each CTA sums the 16 slots in a fixed order).
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void __cluster_dims__(1, 1, 1) dummy() {}

template <int CS>
__global__ void __launch_bounds__(256, 1) kern(int iters, double* out, long long* cyc) {
  __shared__ double slots[2][16];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  double v = 1.0 + rank;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    double* buf = slots[it & 1];
    if (threadIdx.x < CS) {
      double* remote = cl.map_shared_rank(buf, threadIdx.x);
      remote[rank] = v;
    }
    cl.sync();
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < CS; ++r) s += buf[r];
    v = s * 1e-3 + 1.0;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    out[blockIdx.x] = v;
    cyc[blockIdx.x] = (t1 - t0) / iters;
  }
}

int main() {
  int dev = 0;
  cudaSetDevice(dev);
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, dev);
  for (int cs : {8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 200 * 1024;  // one CTA per SM
    cfg.attrs = at;
    cfg.numAttrs = 2;
    void (*k)(int, double*, long long*) = cs == 8 ? kern<8> : kern<16>;
    if (cs == 16) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    int ncl = 0;
    cfg.gridDim = dim3(cs);
    cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, (void*)k, &cfg);
    printf("cluster %d: max active clusters %d (%s)\n", cs, ncl, cudaGetErrorString(e));
    cfg.gridDim = dim3(cs * ncl);
    double* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(double) * 4096);
    cudaMalloc(&cyc, sizeof(long long) * 4096);
    e = cudaLaunchKernelEx(&cfg, k, 1000, out, cyc);
    cudaError_t e2 = cudaDeviceSynchronize();
    static long long h[4096];
    cudaMemcpy(h, cyc, sizeof(long long) * cs * ncl, cudaMemcpyDeviceToHost);
    printf("  grid %d: launch %s sync %s, cycles per all-reduce: cta0 %lld, last %lld\n",
           cs * ncl, cudaGetErrorString(e), cudaGetErrorString(e2), h[0], h[cs * ncl - 1]);
  }
  return 0;
}
