// synth.cu -- synthetic X for the BASELINE.json configurations (bench
// harness; not on the solver path).  Same counter streams as the oracle's
// orc_synth_x (oracle/cnmf_oracle.c): W0 (d x r) stream 1, H0 (r x n) stream
// 2, |N(0,1)| noise stream 3, Gamma draws streams 4/5, Poisson stream 6;
// X = fp32( sum_r W0[i,r] H0[r,j] in fp64 without FMA contraction + noise ).
// Each shard generates only its own columns, so X is identical at any GPU
// count.
#include "common.cuh"
#include "kernels.h"

namespace cnmf {

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t synth_key(uint64_t seed, uint64_t stream) {
  return splitmix64(seed ^ splitmix64(stream * 0xD1B54A32D192ED03ULL));
}
__device__ __forceinline__ double synth_u(uint64_t key, uint64_t index) {
  return (double)(splitmix64(key + index) >> 11) * 0x1.0p-53;
}
__device__ __forceinline__ double synth_normal(uint64_t key, uint64_t pair) {
  const double u1 = 1.0 - synth_u(key, 2 * pair);
  const double u2 = synth_u(key, 2 * pair + 1);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}
__device__ double synth_gamma(uint64_t key, uint64_t index, double shape) {
  const double a = shape < 1.0 ? shape + 1.0 : shape;
  const double dd = a - 1.0 / 3.0, cc = 1.0 / sqrt(9.0 * dd);
  const uint64_t base = index * 64;
  double g = dd;
  for (uint64_t t = 0; t < 20; ++t) {
    const double z = synth_normal(key, base + 3 * t);
    const double v0 = 1.0 + cc * z;
    if (v0 <= 0.0) continue;
    const double v = v0 * v0 * v0;
    const double u = 1.0 - synth_u(key, 2 * (base + 3 * t + 1));
    if (log(u) < 0.5 * z * z + dd - dd * v + dd * log(v)) {
      g = dd * v;
      break;
    }
  }
  if (shape < 1.0) g *= pow(1.0 - synth_u(key, 2 * (base + 63)), 1.0 / shape);
  return g;
}
__device__ double synth_poisson(uint64_t key, uint64_t index, double lam) {
  const uint64_t base = index * 256;
  if (lam <= 0.0) return 0.0;
  if (lam < 30.0) {
    const double lim = exp(-lam);
    double p = 1.0;
    uint64_t k = 0;
    for (;;) {
      p *= 1.0 - synth_u(key, base + k);
      if (p <= lim || k >= 255) break;
      ++k;
    }
    return (double)k;
  }
  const double slam = sqrt(lam), loglam = log(lam);
  const double b = 0.931 + 2.53 * slam, a = -0.059 + 0.02483 * b;
  const double invalpha = 1.1239 + 1.1328 / (b - 3.4), vr = 0.9277 - 3.6224 / (b - 2);
  for (uint64_t t = 0; t < 127; ++t) {
    const double u = synth_u(key, base + 2 * t) - 0.5;
    const double v = 1.0 - synth_u(key, base + 2 * t + 1);
    const double us = 0.5 - fabs(u);
    const double kk = floor((2 * a / us + b) * u + lam + 0.43);
    if (us >= 0.07 && v <= vr) return kk;
    if (kk < 0 || (us < 0.013 && v > us)) continue;
    if (log(v) + log(invalpha) - log(a / (us * us) + b) <= -lam + kk * loglam - lgamma(kk + 1))
      return kk;
  }
  return floor(lam + 0.5);
}
__device__ double factor_entry(uint64_t seed, uint64_t stream, uint64_t index, int kind) {
  if (kind == 0) return synth_u(synth_key(seed, stream), index);
  if (kind == 1) return -log(1.0 - synth_u(synth_key(seed, stream), index));
  return synth_gamma(synth_key(seed, stream + 3), index, 0.3);
}

__global__ void factors_kernel(int64_t d, int64_t n, int rank, int kind, uint64_t seed,
                               int64_t col_lo, int64_t ncols, double* __restrict__ w0,
                               double* __restrict__ h0) {
  const int64_t tot = d * rank + (int64_t)rank * ncols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (e < d * rank) {
      w0[e] = factor_entry(seed, 1, (uint64_t)e, kind);
    } else {
      const int64_t f = e - d * rank, r = f / ncols, j = f - r * ncols;
      h0[f] = factor_entry(seed, 2, (uint64_t)(r * n + col_lo + j), kind);
    }
  }
}

__global__ void x_kernel(int64_t d, int64_t n, int rank, int noise_kind, double sigma,
                         uint64_t seed, int64_t col_lo, int64_t ncols, int64_t ldx,
                         const double* __restrict__ w0, const double* __restrict__ h0,
                         float* __restrict__ x) {
  const uint64_t knoise = synth_key(seed, 3), kpois = synth_key(seed, 6);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < d * ldx;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / ldx, j = e - i * ldx;
    if (j >= ncols) {
      x[e] = 0.f;
      continue;
    }
    double acc = 0.0;
    for (int r = 0; r < rank; ++r) acc = __dadd_rn(acc, __dmul_rn(w0[i * rank + r], h0[r * ncols + j]));
    const uint64_t gidx = (uint64_t)(i * n + col_lo + j);
    if (noise_kind == 1) acc = __dadd_rn(acc, __dmul_rn(sigma, fabs(synth_normal(knoise, gidx))));
    if (noise_kind == 2) acc = synth_poisson(kpois, gidx, acc);
    x[e] = (float)acc;
  }
}

}  // namespace

size_t synth_scratch_doubles(int64_t d, int64_t ncols, int rank) {
  return (size_t)(d * rank + (int64_t)rank * ncols);
}

void launch_synth_x(int64_t d, int64_t n, int rank, int factor_kind, int noise_kind, double sigma,
                    uint64_t seed, int64_t col_lo, int64_t col_hi, int64_t ldx, float* x,
                    double* scratch, cudaStream_t s) {
  const int64_t ncols = col_hi - col_lo;
  double* w0 = scratch;
  double* h0 = scratch + d * rank;
  note_launches(1);
  factors_kernel<<<148 * 8, 256, 0, s>>>(d, n, rank, factor_kind, seed, col_lo, ncols, w0, h0);
  note_launches(1);
  x_kernel<<<148 * 16, 256, 0, s>>>(d, n, rank, noise_kind, sigma, seed, col_lo, ncols, ldx, w0,
                                    h0, x);
}

}  // namespace cnmf
