// rng.cu -- the reference's seeded variate streams, generated on the device.
//
// Reference: cnmf::Rng (proj/include/cnmf/rng.hpp:13-60) = std::mt19937_64
// plus fixed mappings:  uniform = (u64 >> 11) * 2^-53;  uniform_positive
// rejects exact 0;  normal = Box-Muller (cos first, sin cached as spare).
// gaussian_sketch (proj/src/compression.cpp:11-16) fills row-major from a
// fresh Rng(seed); initialize (proj/src/solvers.cpp:206-211, 314-325) fills A
// then B row-major with uniform_positive.
//
// MT19937-64 is sequential, so one warp owns one engine and emits its raw
// 64-bit stream 156 words per step.  The
// mapping kernels are then fully parallel: normal e uses words 2*(e/2) and
// 2*(e/2)+1 and uniform e uses word e, EXCEPT after a word whose 53-bit
// uniform is exactly 0 (probability 2^-53 per draw), where the reference
// rejects and re-draws.  The fast mappings detect that case and set a flag;
// the host then re-runs the exact sequential mapping (single thread) so the
// stream stays identical to the reference in every case.
#include "common.cuh"
#include "kernels.h"

namespace cnmf {

namespace {

constexpr int kN = 312, kM = 156;
constexpr uint64_t kUM = 0xFFFFFFFF80000000ULL, kLM = 0x7FFFFFFFULL;
constexpr uint64_t kMatA = 0xB5026F5AA96619E9ULL;

__device__ __forceinline__ uint64_t mix(uint64_t a, uint64_t b) {
  const uint64_t y = (a & kUM) | (b & kLM);
  return (y >> 1) ^ ((y & 1ULL) ? kMatA : 0ULL);
}
__device__ __forceinline__ uint64_t temper(uint64_t z) {
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= z >> 43;
  return z;
}

// One warp per engine.  The engine is run as its linear recurrence
//   x[p + 312] = x[p + 156] ^ mix(x[p], x[p + 1])
// over a 312-word shared-memory ring (slot p % 312): the 156 words
// x[N .. N+155] depend only on x[N-312 .. N-1], so each step computes them in
// parallel (about five per lane), reads before writes, two __syncwarp()s per
// step and no block barrier.  Output word t is temper(x[312 + t]), exactly the
// std::mt19937_64 sequence (first twist after seeding).
__global__ void __launch_bounds__(32) mt_stream_kernel(MtJobs jobs) {
  const MtJob job = jobs.job[blockIdx.x];
  __shared__ uint64_t x[kN];
  const int lane = threadIdx.x;
  if (lane == 0) {
    x[0] = job.seed;
    for (int i = 1; i < kN; ++i)
      x[i] = 6364136223846793005ULL * (x[i - 1] ^ (x[i - 1] >> 62)) + (uint64_t)i;
  }
  __syncwarp();
  constexpr int kPer = (kM + 31) / 32;  // 5 words per lane per step
  const uint64_t nsteps = (job.nwords + kM - 1) / kM;
  int base = 0;  // (N - 312) % 312 for the current step, N = 312 + 156 * step
  for (uint64_t step = 0; step < nsteps; ++step) {
    uint64_t v[kPer];
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
      const int i = lane + 32 * r;
      if (i < kM) {
        const int j = base + i;  // < 312 + 156
        const int s0 = j >= kN ? j - kN : j;
        const int s1 = j + 1 >= kN ? j + 1 - kN : j + 1;
        const int s2 = j + kM >= kN ? j + kM - kN : j + kM;
        v[r] = x[s2] ^ mix(x[s0], x[s1]);
      }
    }
    __syncwarp();
    const uint64_t out0 = step * kM;
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
      const int i = lane + 32 * r;
      if (i < kM) {
        const int j = base + i;
        x[j >= kN ? j - kN : j] = v[r];
        if (out0 + i < job.nwords) job.out[out0 + i] = temper(v[r]);
      }
    }
    __syncwarp();
    base = base + kM >= kN ? base + kM - kN : base + kM;
  }
}

__device__ __forceinline__ double u53(uint64_t w) { return (double)(w >> 11) * 0x1.0p-53; }

// normal e -> out[(e / cols) * ld + e % cols]
__global__ void normal_map_kernel(const uint64_t* __restrict__ words, uint64_t count, int cols,
                                  int ld, float* __restrict__ out, int* __restrict__ flag) {
  const uint64_t npairs = (count + 1) / 2;
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < npairs;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const double u1 = u53(words[2 * p]);
    const double u2 = u53(words[2 * p + 1]);
    if (u1 == 0.0) *flag = 1;
    const double radius = sqrt(-2.0 * log(u1));
    const double angle = 2.0 * 3.141592653589793238462643383279502884 * u2;
    double s, c;
    sincos(angle, &s, &c);
    const uint64_t e0 = 2 * p, e1 = 2 * p + 1;
    out[(e0 / cols) * ld + e0 % cols] = (float)(radius * c);
    if (e1 < count) out[(e1 / cols) * ld + e1 % cols] = (float)(radius * s);
  }
}

// Exact sequential Box-Muller over the stream (zero-rejection path).
__global__ void normal_exact_kernel(const uint64_t* __restrict__ words, uint64_t nwords,
                                    uint64_t count, int cols, int ld, float* __restrict__ out,
                                    int* __restrict__ flag) {
  if (threadIdx.x != 0 || blockIdx.x != 0 || *flag == 0) return;
  uint64_t pos = 0;
  for (uint64_t e = 0; e < count; e += 2) {
    double u1 = 0.0;
    while (u1 == 0.0) {
      if (pos >= nwords) { *flag = 2; return; }
      u1 = u53(words[pos++]);
    }
    if (pos >= nwords) { *flag = 2; return; }
    const double u2 = u53(words[pos++]);
    const double radius = sqrt(-2.0 * log(u1));
    const double angle = 2.0 * 3.141592653589793238462643383279502884 * u2;
    double s, c;
    sincos(angle, &s, &c);
    out[(e / cols) * ld + e % cols] = (float)(radius * c);
    if (e + 1 < count) out[((e + 1) / cols) * ld + (e + 1) % cols] = (float)(radius * s);
  }
  *flag = 3;  // served by the exact path
}

// uniform_positive e (A then B, both row-major d x k / n x k in the
// reference) -> column-major device factors A_cm[c*d + i], B_cm[c*n + i].
__global__ void uniform_init_kernel(const uint64_t* __restrict__ words, uint64_t d, uint64_t n,
                                    int k, double* __restrict__ a_cm, double* __restrict__ b_cm,
                                    int* __restrict__ flag) {
  const uint64_t na = d * k, total = (d + n) * k;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const double u = u53(words[e]);
    if (u == 0.0) *flag = 1;
    if (e < na)
      a_cm[(e % k) * d + e / k] = u;
    else
      b_cm[((e - na) % k) * n + (e - na) / k] = u;
  }
}

__global__ void uniform_init_exact_kernel(const uint64_t* __restrict__ words, uint64_t nwords,
                                          uint64_t d, uint64_t n, int k, double* __restrict__ a_cm,
                                          double* __restrict__ b_cm, int* __restrict__ flag,
                                          uint64_t* __restrict__ consumed) {
  if (threadIdx.x != 0 || blockIdx.x != 0 || *flag == 0) return;
  const uint64_t na = d * k, total = (d + n) * k;
  uint64_t pos = 0;
  for (uint64_t e = 0; e < total; ++e) {
    double u = 0.0;
    while (u == 0.0) {
      if (pos >= nwords) { *flag = 2; return; }
      u = u53(words[pos++]);
    }
    if (e < na)
      a_cm[(e % k) * d + e / k] = u;
    else
      b_cm[((e - na) % k) * n + (e - na) / k] = u;
  }
  *consumed = pos;
  *flag = 3;
}

}  // namespace

void launch_mt_streams(const MtJobs& jobs, int njobs, cudaStream_t s) {
  note_launches(1);
  mt_stream_kernel<<<njobs, 32, 0, s>>>(jobs);
}

void launch_normal_map(const uint64_t* words, uint64_t count, int cols, int ld, float* out,
                       int* flag, int nsm, cudaStream_t s) {
  const uint64_t npairs = (count + 1) / 2;
  const int blocks = (int)std::min<uint64_t>((npairs + 255) / 256, (uint64_t)nsm * 8);
  note_launches(1);
  normal_map_kernel<<<blocks > 0 ? blocks : 1, 256, 0, s>>>(words, count, cols, ld, out, flag);
}

void launch_normal_exact(const uint64_t* words, uint64_t nwords, uint64_t count, int cols, int ld,
                         float* out, int* flag, cudaStream_t s) {
  note_launches(1);
  normal_exact_kernel<<<1, 32, 0, s>>>(words, nwords, count, cols, ld, out, flag);
}

void launch_uniform_init(const uint64_t* words, uint64_t d, uint64_t n, int k, double* a_cm,
                         double* b_cm, int* flag, int nsm, cudaStream_t s) {
  const uint64_t total = (d + n) * (uint64_t)k;
  const int blocks = (int)std::min<uint64_t>((total + 255) / 256, (uint64_t)nsm * 8);
  note_launches(1);
  uniform_init_kernel<<<blocks > 0 ? blocks : 1, 256, 0, s>>>(words, d, n, k, a_cm, b_cm, flag);
}

void launch_uniform_init_exact(const uint64_t* words, uint64_t nwords, uint64_t d, uint64_t n,
                               int k, double* a_cm, double* b_cm, int* flag, uint64_t* consumed,
                               cudaStream_t s) {
  note_launches(1);
  uniform_init_exact_kernel<<<1, 32, 0, s>>>(words, nwords, d, n, k, a_cm, b_cm, flag, consumed);
}

}  // namespace cnmf
