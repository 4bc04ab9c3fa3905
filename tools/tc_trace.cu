// tc_trace.cu -- per-K-block event timeline of CTA 0 of the tcgen05 X-stream
// kernel (needs the TC_TRACE build of the library).  Debug tool.
//   LD_LIBRARY_PATH=paper_1712_02248_b200/build_var/trace tools/tc_trace m n lp
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_1712_02248_b200/csrc/kernels.h"
using namespace cnmf;
int main(int argc, char** argv) {
  const int64_t m = atoll(argv[1]), n = atoll(argv[2]);
  const int lp = atoi(argv[3]);
  std::vector<float> x(m * n), s(n * lp);
  for (size_t i = 0; i < x.size(); ++i) x[i] = (float)((i * 2654435761u) % 1000) / 1000.f;
  for (size_t i = 0; i < s.size(); ++i) s[i] = (float)((i * 40503u) % 2000) / 1000.f - 1.f;
  float *dx, *ds, *dy, *dw, *dbg;
  cudaMalloc(&dx, x.size() * 4); cudaMalloc(&ds, s.size() * 4); cudaMalloc(&dy, m * lp * 4);
  cudaMalloc(&dw, xstream_tc_ws_floats(m, n, lp, 148) * 4); cudaMalloc(&dbg, 12 * 4096 * 8);
  cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(ds, s.data(), s.size() * 4, cudaMemcpyHostToDevice);
  launch_xs_tc(false, dx, n, m, n, ds, lp, dy, dw, 148, 0);  // warm
  cudaMemset(dbg, 0, 12 * 4096 * 8);
  xstream_tc_set_debug(dbg);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  launch_xs_tc(false, dx, n, m, n, ds, lp, dy, dw, 148, 0);
  cudaEventRecord(e1);
  cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<unsigned long long> t(12 * 4096);
  cudaMemcpy(t.data(), dbg, t.size() * 8, cudaMemcpyDeviceToHost);
  int nb = 0; while (nb < 4096 && t[5 * 4096 + nb]) ++nb;
  printf("%.1f us, %.0f GB/s; CTA0 blocks %d\n", ms * 1e3, 4.0 * m * n / (ms * 1e-3) / 1e9, nb);
  const unsigned long long t0 = t[0];
  printf("blk    Xiss   gotX   slot   done  mmaA   mmaIn mmaIss   Siss | Xlat slotw sttm  A->B  Slat  dMMA\n");
  for (int b = std::max(0, nb / 2 - 12); b < std::min(nb, nb / 2 + 12); ++b) {
    auto T = [&](int ev) { return (long long)(t[ev * 4096 + b] - t0); };
    printf("%4d %6lld %6lld %6lld %6lld %6lld %6lld %6lld %6lld | %5lld %5lld %5lld %5lld %5lld %5lld\n", b, T(0), T(1), T(2), T(3), T(7), T(4), T(5), T(6),
           T(1) - T(0), T(2) - T(1), T(3) - T(2), T(4) - T(7), T(4) - T(6), b ? T(5) - (long long)(t[5 * 4096 + b - 1] - t0) : 0);
  }
  // averages over the steady state
  double a[5] = {0, 0, 0, 0, 0}; int cnt = 0;
  for (int b = nb / 4; b < 3 * nb / 4; ++b, ++cnt) {
    a[0] += (double)(t[1 * 4096 + b] - t[0 * 4096 + b]);
    a[1] += (double)(t[2 * 4096 + b] - t[1 * 4096 + b]);
    a[2] += (double)(t[3 * 4096 + b] - t[2 * 4096 + b]);
    a[3] += (double)(t[4 * 4096 + b] - t[3 * 4096 + b]);
    a[4] += (double)(t[5 * 4096 + b] - t[5 * 4096 + b - 1]);
  }
  printf("steady-state means (cycles): X latency %.0f, split waits A slot %.0f, split store %.0f, handoff to MMA %.0f, MMA issue interval %.0f\n",
         a[0] / cnt, a[1] / cnt, a[2] / cnt, a[3] / cnt, a[4] / cnt);
  // per-quarter split completion relative to the MMA's view of opready
  double qd[4] = {0, 0, 0, 0};
  for (int b = nb / 4; b < 3 * nb / 4; ++b)
    for (int q = 0; q < 4; ++q) qd[q] += (double)((long long)t[7 * 4096 + b] - (long long)t[(8 + q) * 4096 + b]);
  printf("MMA sees opready minus split quarter done (cycles): q0 %.0f q1 %.0f q2 %.0f q3 %.0f\n",
         qd[0] / cnt, qd[1] / cnt, qd[2] / cnt, qd[3] / cnt);
  return 0;
}
