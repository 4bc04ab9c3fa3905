// Debug harness for the tcgen05 X-stream kernel: tiny NN/TN cases with the
// kernel's smem/TMEM dumps (xstream_tc_set_debug).  Not part of the product.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_1712_02248_b200/csrc/kernels.h"
using namespace cnmf;
int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 128, n = argc > 2 ? atoi(argv[2]) : 32, lp = 32;
  const bool tn = argc > 3 && atoi(argv[3]);
  std::vector<float> x((size_t)m * n), s((size_t)(tn ? m : n) * lp);
  for (size_t i = 0; i < x.size(); ++i) x[i] = (float)((i % 7) + 1) / 8.0f;
  for (size_t i = 0; i < s.size(); ++i) s[i] = (float)((i % 5) + 1) / 4.0f;
  float *dx, *ds, *dy, *dw, *dbg;
  const int64_t orow = tn ? n : m;
  cudaMalloc(&dx, x.size() * 4); cudaMalloc(&ds, s.size() * 4); cudaMalloc(&dy, orow * lp * 4);
  cudaMalloc(&dw, xstream_tc_ws_floats(m, n, lp, 148) * 4); cudaMalloc(&dbg, 1 << 20);
  cudaMemset(dbg, 0, 1 << 20); cudaMemset(dy, 0, orow * lp * 4);
  const float mode = argc > 4 ? (float)atof(argv[4]) : 0.f;
  cudaMemcpy(dbg + 65535, &mode, 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(ds, s.data(), s.size() * 4, cudaMemcpyHostToDevice);
  xstream_tc_set_debug(dbg);
  const bool ok = launch_xs_tc(tn, dx, n, m, n, ds, lp, dy, dw, 148, 0);
  cudaError_t e = cudaDeviceSynchronize();
  printf("launched=%d err=%s\n", ok, cudaGetErrorString(e));
  std::vector<float> y(orow * lp), d(1 << 18);
  cudaMemcpy(y.data(), dy, y.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(d.data(), dbg, 1 << 20, cudaMemcpyDeviceToHost);
  // reference
  double maxerr = 0, maxref = 0;
  for (int64_t r = 0; r < orow; ++r)
    for (int c = 0; c < lp; ++c) {
      double acc = 0;
      if (!tn) for (int k = 0; k < n; ++k) acc += (double)x[r * n + k] * s[(size_t)k * lp + c];
      else for (int k = 0; k < m; ++k) acc += (double)x[(size_t)k * n + r] * s[(size_t)k * lp + c];
      maxerr = std::max(maxerr, std::abs(acc - y[r * lp + c]));
      maxref = std::max(maxref, std::abs(acc));
      if (r < 2 && c < 4) printf("y[%ld][%d] = %g (ref %g)\n", (long)r, c, y[r * lp + c], acc);
    }
  printf("max abs err %g (max |ref| %g)\n", maxerr, maxref);
  printf("smem x stage[0..8]:"); for (int i = 0; i < 8; ++i) printf(" %g", d[i]); printf("\n");
  printf("smem b stage[0..8]:"); for (int i = 0; i < 8; ++i) printf(" %g", d[1024 + i]); printf("\n");
  printf("tmem row0 hi[0..4] lo-part[0..4]:"); for (int i = 0; i < 4; ++i) printf(" %g", d[2048 + i]);
  printf(" |"); for (int i = 0; i < 4; ++i) printf(" %g", d[2048 + 16 + i]); printf("\n");
  printf("tmem row5 hi[0..4]:"); for (int i = 0; i < 4; ++i) printf(" %g", d[2048 + 5 * 32 + i]); printf("\n");
  unsigned* u = reinterpret_cast<unsigned*>(d.data());
  printf("mma: d=%08x adesc=%08x_%08x bdesc=%08x_%08x idesc=%08x xa=%08x tmem_base(epi)=%08x\n",
         u[16384], u[16386], u[16385], u[16388], u[16387], u[16389], u[16390], u[16392]);
  int nz = 0;
  for (int cc = 0; cc < 512; ++cc) if (d[20480 + cc] != 0.f) { if (nz < 8) printf("  lane0 col %d = %g\n", cc, d[20480 + cc]); ++nz; }
  printf("non-zero lane-0 columns: %d\n", nz);
  return 0;
}
