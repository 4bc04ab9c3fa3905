// tc_units.cu -- checks every split-K partial (unit = split x 128-row tile) of
// the tcgen05 X-stream kernel against a CPU fp64 reference, over repeated
// launches, and reports wrong units with their CTA and position in the CTA's
// schedule.  Debug harness, not part of the product.
//   usage: CNMF_TC_KCHUNK=64 tools/tc_units m n lp [trials]
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cstring>
#include <algorithm>
#include <cuda_runtime.h>
#include "../paper_1712_02248_b200/csrc/kernels.h"
using namespace cnmf;
int main(int argc, char** argv) {
  const int64_t m = atoi(argv[1]), n = atoi(argv[2]);
  const int lp = atoi(argv[3]), trials = argc > 4 ? atoi(argv[4]) : 3;
  const int L = (lp + 31) & ~31;
  const char* kc_env = getenv("CNMF_TC_KCHUNK");
  const int64_t kc = kc_env ? atoll(kc_env) : 0;
  if (!kc) { printf("set CNMF_TC_KCHUNK\n"); return 1; }
  const int64_t nsplit = (n + kc - 1) / kc, ntiles = (m + 127) / 128;
  std::vector<float> x(m * n), s(n * lp);
  uint64_t st = 12345;
  auto rnd = [&]() { st = st * 6364136223846793005ULL + 1442695040888963407ULL; return (float)((st >> 40) & 0xFFFFFF) / 16777216.0f; };
  for (auto& v : x) v = rnd();
  for (auto& v : s) v = rnd() * 2.f - 1.f;
  // reference partials [split][row][lp]
  std::vector<double> ref(nsplit * m * lp, 0.0);
  for (int64_t sp = 0; sp < nsplit; ++sp)
    for (int64_t r = 0; r < m; ++r) {
      double* o = &ref[(sp * m + r) * lp];
      for (int64_t k = sp * kc; k < std::min(n, (sp + 1) * kc); ++k) {
        const double xv = x[r * n + k];
        for (int c = 0; c < lp; ++c) o[c] += xv * s[k * lp + c];
      }
    }
  float *dx, *ds, *dy, *dw;
  const size_t wsf = xstream_tc_ws_floats(m, n, lp, 148);
  cudaMalloc(&dx, x.size() * 4); cudaMalloc(&ds, s.size() * 4); cudaMalloc(&dy, m * lp * 4);
  cudaMalloc(&dw, wsf * 4);
  cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(ds, s.data(), s.size() * 4, cudaMemcpyHostToDevice);
  const int64_t units = nsplit * ntiles, grid = std::min<int64_t>(units, 148);
  std::vector<float> parts(nsplit * m * lp);
  for (int t = 0; t < trials; ++t) {
    cudaMemset(dw, 0xFF, wsf * 4);  // NaN fill: unwritten partials show up
    const bool ok = launch_xs_tc(false, dx, n, m, n, ds, lp, dy, dw, 148, 0);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(parts.data(), dw + 2 * n * L, parts.size() * 4, cudaMemcpyDeviceToHost);
    int bad_units = 0, printed = 0;
    for (int64_t sp = 0; sp < nsplit; ++sp)
      for (int64_t tl = 0; tl < ntiles; ++tl) {
        int bad_rows = 0, first = -1; double worst = 0;
        for (int64_t r = tl * 128; r < std::min(m, tl * 128 + 128); ++r) {
          double en = 0, rn = 0;
          for (int c = 0; c < lp; ++c) {
            const double g = parts[(sp * m + r) * lp + c], rv = ref[(sp * m + r) * lp + c];
            en += (g - rv) * (g - rv); rn += rv * rv;
          }
          const double rel = std::sqrt(en / std::max(rn, 1e-30));
          if (!(rel < 1e-4)) { ++bad_rows; if (first < 0) first = (int)(r - tl * 128); worst = std::max(worst, rel); }
        }
        if (bad_rows) {
          ++bad_units;
          const int64_t u = sp * ntiles + tl;
          if (printed++ < 6) {
            printf("  trial %d unit %ld (split %ld tile %ld) cta %ld pos %ld: %d bad rows, first row %d, worst rel %.2e\n", t, (long)u,
                   (long)sp, (long)tl, (long)(u % grid), (long)(u / grid), bad_rows, first, worst);
            // least-squares decomposition of the error onto the unit's 24
            // per-k-step product terms (x_hi s_hi, x_hi s_lo, x_lo s_hi)
            const int64_t r = tl * 128 + first;
            const float* g = &parts[(sp * m + r) * lp];
            const double* rf = &ref[(sp * m + r) * lp];
            auto rna = [](float v) { uint32_t u; memcpy(&u, &v, 4); u = (u + 0x1000u) & 0xFFFFE000u; float o; memcpy(&o, &u, 4); return o; };
            const int64_t k0 = sp * kc, k1 = std::min(n, (sp + 1) * kc);
            const int nst = (int)((k1 - k0) / 8), nb = 3 * nst;
            std::vector<double> B((size_t)nb * lp, 0.0), e(lp);
            for (int c = 0; c < lp; ++c) e[c] = g[c] - rf[c];
            for (int st8 = 0; st8 < nst; ++st8)
              for (int k = 0; k < 8; ++k) {
                const int64_t kk = k0 + st8 * 8 + k;
                const float xv = x[r * n + kk], xh = rna(xv), xl = rna(xv - xh);
                for (int c = 0; c < lp; ++c) {
                  const float sv = s[kk * lp + c], sh = rna(sv), sl = rna(sv - sh);
                  B[(size_t)(3 * st8 + 0) * lp + c] += (double)xh * sh;
                  B[(size_t)(3 * st8 + 1) * lp + c] += (double)xh * sl;
                  B[(size_t)(3 * st8 + 2) * lp + c] += (double)xl * sh;
                }
              }
            // normal equations (nb x nb), Gaussian elimination
            std::vector<double> A((size_t)nb * nb), y(nb);
            for (int i = 0; i < nb; ++i) {
              for (int j = 0; j < nb; ++j) { double v = 0; for (int c = 0; c < lp; ++c) v += B[(size_t)i * lp + c] * B[(size_t)j * lp + c]; A[(size_t)i * nb + j] = v; }
              double v = 0; for (int c = 0; c < lp; ++c) v += B[(size_t)i * lp + c] * e[c]; y[i] = v;
            }
            for (int i = 0; i < nb; ++i) {
              int piv = i; for (int j = i + 1; j < nb; ++j) if (std::fabs(A[(size_t)j * nb + i]) > std::fabs(A[(size_t)piv * nb + i])) piv = j;
              for (int j = 0; j < nb; ++j) std::swap(A[(size_t)i * nb + j], A[(size_t)piv * nb + j]); std::swap(y[i], y[piv]);
              for (int j = i + 1; j < nb; ++j) { const double f = A[(size_t)j * nb + i] / A[(size_t)i * nb + i]; for (int q = i; q < nb; ++q) A[(size_t)j * nb + q] -= f * A[(size_t)i * nb + q]; y[j] -= f * y[i]; }
            }
            std::vector<double> cf(nb);
            for (int i = nb - 1; i >= 0; --i) { double v = y[i]; for (int q = i + 1; q < nb; ++q) v -= A[(size_t)i * nb + q] * cf[q]; cf[i] = v / A[(size_t)i * nb + i]; }
            double res = 0, en = 0;
            for (int c = 0; c < lp; ++c) { double v = e[c]; for (int i = 0; i < nb; ++i) v -= cf[i] * B[(size_t)i * lp + c]; res += v * v; en += e[c] * e[c]; }
            printf("    row %ld: fit residual %.2e; coefficients (k-step: hh hl lh):", (long)r, std::sqrt(res / en));
            for (int st8 = 0; st8 < nst; ++st8) printf(" [%d: %+.2f %+.2f %+.2f]", st8, cf[3 * st8], cf[3 * st8 + 1], cf[3 * st8 + 2]);
            printf("\n");
            const char* what = "lsq"; long a1 = 0, a2 = 0; double best = res / en;
            // another unit's partial for the same TMEM lane?
            {
              double bres = 1e300, balpha = 0; long bu = -1;
              for (int64_t sp2 = 0; sp2 < nsplit; ++sp2)
                for (int64_t tl2 = 0; tl2 < ntiles; ++tl2) {
                  const int64_t r2 = tl2 * 128 + (r % 128);
                  if (r2 >= m) continue;
                  const double* P = &ref[(sp2 * m + r2) * lp];
                  double pp = 0, pe = 0; for (int c = 0; c < lp; ++c) { pp += P[c] * P[c]; pe += P[c] * e[c]; }
                  const double al = pe / pp; double rr = 0;
                  for (int c = 0; c < lp; ++c) { const double v = e[c] - al * P[c]; rr += v * v; }
                  if (rr < bres) { bres = rr; balpha = al; bu = (long)(sp2 * ntiles + tl2); }
                }
              printf("    best other-unit match: unit %ld (cta %ld pos %ld) alpha %+.3f residual %.2e\n", bu, (long)(bu % grid), (long)(bu / grid), balpha, std::sqrt(bres / en));
            }
            // one k-step (8 K values) of row r replaced by 8 values of a same-lane row from any k-step?
            {
              double bres = 1e300; long bj = -1, br = -1, bk = -1;
              for (int j = 0; j < nst; ++j) {
                const int64_t kj = k0 + 8 * j;
                for (int64_t tl2 = 0; tl2 < ntiles; ++tl2) {
                  const int64_t r2 = tl2 * 128 + (r % 128);
                  if (r2 >= m) continue;
                  for (int64_t k2 = 0; k2 + 8 <= n; k2 += 8) {
                    double rr = 0;
                    for (int c = 0; c < lp; ++c) {
                      double d = 0;
                      for (int k = 0; k < 8; ++k) d += ((double)x[r2 * n + k2 + k] - (double)x[r * n + kj + k]) * s[(kj + k) * lp + c];
                      const double v = e[c] - d; rr += v * v;
                    }
                    if (rr < bres) { bres = rr; bj = j; br = (long)r2; bk = (long)k2; }
                  }
                }
              }
              printf("    best k-step substitution: k-step %ld of the unit <- row %ld k %ld..+8 (unit K start %ld), residual %.2e\n", bj, br, bk, (long)k0, std::sqrt(bres / en));
            }
            printf("    row %ld: best explanation %s (kblock %ld <- %ld) residual %.3e\n", (long)r, what, a1, a2, std::sqrt(best));
          }
        }
      }
    printf("trial %d: launched=%d err=%s bad units %d of %ld\n", t, ok, cudaGetErrorString(e), bad_units, (long)units);
  }
  return 0;
}
