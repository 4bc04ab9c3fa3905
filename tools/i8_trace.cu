// i8_trace.cu -- per-K-block event timeline of CTA 0 of the int8-sliced exact
// contraction (needs the I8_TRACE build of the library).  Debug tool.
//   bash tools/build_variant.sh i8trace "-DI8_TRACE"
//   nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/i8_trace tools/i8_trace.cu \
//        -Lpaper_1712_02248_b200/build_var/i8trace -lcnmf_b200
//   LD_LIBRARY_PATH=paper_1712_02248_b200/build_var/i8trace tools/i8_trace m n lp tn small_int
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_1712_02248_b200/csrc/kernels.h"
using namespace cnmf;
int main(int argc, char** argv) {
  const int64_t m = atoll(argv[1]), n = atoll(argv[2]);
  const int lp = atoi(argv[3]);
  const bool tn = argc > 4 && atoi(argv[4]) != 0, small_int = argc > 5 && atoi(argv[5]) != 0;
  const int64_t kdim = tn ? m : n, rows_out = tn ? n : m;
  std::vector<float> x(m * n);
  std::vector<double> s(kdim * lp);
  for (size_t i = 0; i < x.size(); ++i) x[i] = (float)((i * 2654435761u) % 1000) * (small_int ? 1.f : 1e-3f);
  for (size_t i = 0; i < s.size(); ++i) s[i] = (double)((i * 40503u) % 2000) / 1000.0 - 1.0;
  float* dx; double *ds, *dy; void* dw; int* sx; unsigned long long* dbg;
  cudaMalloc(&dx, x.size() * 4); cudaMalloc(&ds, s.size() * 8); cudaMalloc(&dy, rows_out * lp * 8);
  cudaMalloc(&dw, xs_i8_ws_bytes(m, n, lp, 148)); cudaMalloc(&sx, xs_i8_sx_ints(m, n) * 4);
  cudaMalloc(&dbg, 8 * 4096 * 8);
  cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(ds, s.data(), s.size() * 8, cudaMemcpyHostToDevice);
  if (small_int) cudaMemset(sx, 0, (m + n) * 4);
  else launch_xs_i8_prepare_x(dx, n, m, n, sx, 148, 0);
  launch_xs_i8(tn, dx, n, m, n, ds, lp, dy, dw, sx, 148, 0, small_int);  // warm
  cudaMemset(dbg, 0, 8 * 4096 * 8);
  xs_i8_set_debug(dbg);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const bool ok = launch_xs_i8(tn, dx, n, m, n, ds, lp, dy, dw, sx, 148, 0, small_int);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<unsigned long long> t(8 * 4096);
  cudaMemcpy(t.data(), dbg, t.size() * 8, cudaMemcpyDeviceToHost);
  int nb = 0; while (nb < 4096 && t[6 * 4096 + nb]) ++nb;
  printf("ok %d (%s): %.1f us (whole contraction), %.0f GB/s of X; CTA0 traced blocks %d\n", (int)ok,
         cudaGetErrorString(err), ms * 1e3, 4.0 * m * n / (ms * 1e-3) / 1e9, nb);
  const unsigned long long t0 = t[0];
  printf("blk    Xiss   gotX   digs   slot   stTM  mmaIn mmaIss | Xlat  digs slotw  stTM  st>mma issue  dMMA\n");
  double sum[7] = {0, 0, 0, 0, 0, 0, 0}; int cnt = 0;
  for (int b = 8; b < nb - 8; ++b) {
    auto T = [&](int ev) { return (long long)(t[ev * 4096 + b] - t0); };
    const long long d[7] = {T(1) - T(0), T(2) - T(1), T(3) - T(2), T(4) - T(3), T(5) - T(4), T(6) - T(5),
                            T(6) - (long long)(t[6 * 4096 + b - 1] - t0)};
    for (int i = 0; i < 7; ++i) sum[i] += (double)d[i];
    ++cnt;
    if (b >= nb / 2 - 8 && b < nb / 2 + 8)
      printf("%4d %6lld %6lld %6lld %6lld %6lld %6lld %6lld | %5lld %5lld %5lld %5lld %5lld %5lld %5lld\n", b, T(0), T(1),
             T(2), T(3), T(4), T(5), T(6), d[0], d[1], d[2], d[3], d[4], d[5], d[6]);
  }
  if (cnt)
    printf("mean over %d blocks: X latency %.0f, digits %.0f, slot wait %.0f, TMEM store %.0f, store->MMA %.0f, MMA issue %.0f, block period %.0f cycles\n",
           cnt, sum[0] / cnt, sum[1] / cnt, sum[2] / cnt, sum[3] / cnt, sum[4] / cnt, sum[5] / cnt, sum[6] / cnt);
  return 0;
}
