// rng.cu -- the reference's seeded variate streams, generated on the device.
//
// Reference: cnmf::Rng (proj/include/cnmf/rng.hpp:13-60) = std::mt19937_64
// plus fixed mappings:  uniform = (u64 >> 11) * 2^-53;  uniform_positive
// rejects exact 0;  normal = Box-Muller (cos first, sin cached as spare).
// gaussian_sketch (proj/src/compression.cpp:11-16) fills row-major from a
// fresh Rng(seed); initialize (proj/src/solvers.cpp:206-211, 314-325) fills A
// then B row-major with uniform_positive.
//
// MT19937-64 is sequential, so one CTA owns one engine and emits its raw
// 64-bit stream 312 words per twist (156 threads, two words each).  The
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

// One 312-word twist of the state in shared memory, in place (blockDim >=
// 156; threads >= 156 only take part in the barriers).  Before: mt holds
// x_p .. x_p+311; after: x_p+312 .. x_p+623.
__device__ __forceinline__ void mt_twist(uint64_t* mt, int t) {
  uint64_t o0 = 0, o1 = 0, o156 = 0, o157 = 0, o311 = 0;
  if (t < kM) {
    o0 = mt[t];
    o1 = mt[t + 1];
    o156 = mt[t + kM];
    if (t + kM + 1 < kN) o157 = mt[t + kM + 1];
    if (t == 0) o311 = mt[kN - 1];
  }
  __syncthreads();
  if (t < kM) {
    const uint64_t nt = o156 ^ mix(o0, o1);  // i = t       (uses old values)
    mt[t] = nt;
    if (t + kM < kN - 1) mt[t + kM] = nt ^ mix(o156, o157);  // i = t+156 (new mt[i-156])
  }
  __syncthreads();
  if (t == 0) mt[kN - 1] = mt[kM - 1] ^ mix(o311, mt[0]);  // i = 311 (new mt[0], mt[155])
  __syncthreads();
}

__device__ __forceinline__ void mt_seed(uint64_t* mt, uint64_t seed, int t) {
  if (t == 0) {
    mt[0] = seed;
    for (int i = 1; i < kN; ++i)
      mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
  }
  __syncthreads();
}

// One CTA per engine; blockDim.x == 160 (156 active in the twist).  Output
// word t is temper(x_312+t) (raw = 1: x_312+t itself).
__global__ void __launch_bounds__(160) mt_stream_kernel(MtJobs jobs, int raw) {
  const MtJob job = jobs.job[blockIdx.x];
  __shared__ uint64_t mt[kN];
  const int t = threadIdx.x;
  mt_seed(mt, job.seed, t);
  const uint64_t nblocks = (job.nwords + kN - 1) / kN;
  for (uint64_t blk = 0; blk < nblocks; ++blk) {
    mt_twist(mt, t);
    if (t < kM) {
      const uint64_t base = blk * kN;
      const uint64_t w0 = mt[t], w1 = mt[t + kM];
      if (base + t < job.nwords) job.out[base + t] = raw ? w0 : temper(w0);
      if (base + t + kM < job.nwords) job.out[base + t + kM] = raw ? w1 : temper(w1);
    }
    __syncthreads();  // next twist reads after this block's outputs are taken
  }
}

// ---- jump-ahead (parallel segments of one stream) -------------------------
// Segment k of the output stream starts at output kJ, whose raw word is
// x_312+kJ.  Its 312 starting words x_312+kJ+w = XOR over the set bits i of
// c_k = x^(kJ) mod phi of x_312+i+w (mt_jump.cpp), i.e. a GF(2) convolution
// of the raw prefix x_312 .. x_312+19967+311 with c_k.  CTA b builds the
// state of segment k = b + 1 from the prefix held in shared memory.
constexpr int kJumpPoly = 312;                  // words per polynomial (19968 bits)
constexpr int kJumpPrefix = 64 * kJumpPoly + kN;  // raw words the convolution reads

// Segment k's starting state = sum over the set bits of its jump polynomial
// of the prefix shifted by the bit's position (GF(2), XOR).  The CTA first
// lists the polynomial's set-bit positions in shared memory (a block scan of
// the words' popcounts), then each of kJumpGroups thread groups of 312 XORs
// its share of the list with four independent accumulators; the groups'
// partials are combined at the end.  XOR is exact and order-free: bitwise
// the serial result.  (Peeling bits with ffs in a per-word while loop made
// every step wait on the previous one: 480 us per CTA.)
constexpr int kJumpGroups = 3;
constexpr int kJumpThreads = kN * kJumpGroups;
size_t jump_state_smem() {
  return sizeof(uint64_t) * (kJumpPrefix + kJumpGroups * kN) + sizeof(uint16_t) * 64 * kJumpPoly;
}
// `parts` CTAs share one segment (block b: segment b / parts + 1, part
// b % parts), each XORing a slice of the position list into the zeroed
// state with atomicXor -- so short streams fill the GPU too.
__global__ void __launch_bounds__(kJumpThreads) mt_jump_state_kernel(
    const uint64_t* __restrict__ prefix, const uint64_t* __restrict__ polys,
    uint64_t* __restrict__ states, int parts) {
  extern __shared__ uint64_t pre[];  // kJumpPrefix words, kJumpGroups x kN partials, positions
  uint64_t* part = pre + kJumpPrefix;
  uint16_t* pos = reinterpret_cast<uint16_t*>(part + kJumpGroups * kN);
  __shared__ int wsum[kJumpThreads / 32];
  __shared__ int npos;
  const int seg = blockIdx.x / parts, prt = blockIdx.x - seg * parts;
  const int k = seg + 1, tid = threadIdx.x;
  const int grp = tid / kN, w = tid - grp * kN;
  const int lane = tid & 31, wid = tid >> 5;
  for (int e = tid; e < kJumpPrefix; e += blockDim.x) pre[e] = prefix[e];
  // set-bit positions of c_k in ascending order: thread t < 312 owns word t
  const uint64_t word = tid < kJumpPoly ? polys[(size_t)k * kJumpPoly + tid] : 0ull;
  const int cnt = __popcll(word);
  int incl = cnt;  // inclusive scan: warps, then the warp totals
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  if (tid == 0) {
    int run = 0;
    for (int i = 0; i < kJumpThreads / 32; ++i) {
      const int t = wsum[i];
      wsum[i] = run;
      run += t;
    }
    npos = run;
  }
  __syncthreads();
  int off = wsum[wid] + incl - cnt;
  for (uint64_t bits = word; bits; bits &= bits - 1) pos[off++] = (uint16_t)(64 * tid + __ffsll(bits) - 1);
  __syncthreads();
  const int n = npos;
  const int p0 = prt * n / parts, p1 = (prt + 1) * n / parts;  // this CTA's slice
  const int i0 = p0 + grp * (p1 - p0) / kJumpGroups, i1 = p0 + (grp + 1) * (p1 - p0) / kJumpGroups;
  uint64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  int i = i0;
  for (; i + 3 < i1; i += 4) {
    a0 ^= pre[pos[i] + w];
    a1 ^= pre[pos[i + 1] + w];
    a2 ^= pre[pos[i + 2] + w];
    a3 ^= pre[pos[i + 3] + w];
  }
  for (; i < i1; ++i) a0 ^= pre[pos[i] + w];
  uint64_t acc = (a0 ^ a1) ^ (a2 ^ a3);
  part[grp * kN + w] = acc;
  __syncthreads();
  if (grp == 0) {
#pragma unroll
    for (int g = 1; g < kJumpGroups; ++g) acc ^= part[g * kN + w];
    atomicXor(reinterpret_cast<unsigned long long*>(states + (size_t)seg * kN + w),
              (unsigned long long)acc);
  }
}

// CTA k emits outputs [kJ, min((k + 1) J, nwords)): the segment's starting
// words (segment 0: the prefix itself), tempered, then twists onward.
__global__ void __launch_bounds__(160) mt_segment_kernel(const uint64_t* __restrict__ prefix,
                                                         const uint64_t* __restrict__ states,
                                                         uint64_t J, uint64_t nwords,
                                                         uint64_t* __restrict__ out) {
  __shared__ uint64_t mt[kN];
  const int t = threadIdx.x, k = blockIdx.x;
  const uint64_t s0 = (uint64_t)k * J;
  if (s0 >= nwords) return;
  const uint64_t cnt = min(J, nwords - s0);
  const uint64_t* src = k == 0 ? prefix : states + (size_t)(k - 1) * kN;
  for (int e = t; e < kN; e += blockDim.x) mt[e] = src[e];
  __syncthreads();
  for (uint64_t base = 0; base < cnt; base += kN) {
    if (base) mt_twist(mt, t);
    if (t < kM) {
      if (base + t < cnt) out[s0 + base + t] = temper(mt[t]);
      if (base + t + kM < cnt) out[s0 + base + t + kM] = temper(mt[t + kM]);
    }
    __syncthreads();
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

// reinit_column (solvers.cpp:28-31) from the run stream: rows_total values
// uniform_positive() * 1e-3 taken from words[*pos ...]; entries [off, off +
// count) land in col.  The map kernel assumes no rejected (exact zero)
// draw in the window and flags one; the exact kernel then redoes the window
// sequentially with the reference's rejection, and always advances *pos.
__global__ void redraw_map_kernel(const uint64_t* __restrict__ words, const uint64_t* __restrict__ pos,
                                  uint64_t rows_total, uint64_t off, uint64_t count,
                                  double* __restrict__ col, int* __restrict__ flag) {
  const uint64_t p0 = *pos;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < rows_total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double u = u53(words[p0 + i]);
    if (u == 0.0) *flag = 1;
    if (i >= off && i < off + count) col[i - off] = u * 1e-3;
  }
}

__global__ void redraw_exact_kernel(const uint64_t* __restrict__ words, uint64_t nwords,
                                    uint64_t* __restrict__ pos, uint64_t rows_total, uint64_t off,
                                    uint64_t count, double* __restrict__ col, int* __restrict__ flag) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  uint64_t p = *pos;
  if (*flag == 0) {
    *pos = p + rows_total;
    return;
  }
  for (uint64_t i = 0; i < rows_total; ++i) {
    double u = 0.0;
    while (u == 0.0) {
      if (p >= nwords) { *flag = 2; return; }
      u = u53(words[p++]);
    }
    if (i >= off && i < off + count) col[i - off] = u * 1e-3;
  }
  *pos = p;
  *flag = 0;
}

}  // namespace

void launch_mt_streams(const MtJobs& jobs, int njobs, cudaStream_t s) {
  note_launches(1);
  mt_stream_kernel<<<njobs, 160, 0, s>>>(jobs, 0);
}

// nwords outputs of Rng(seed) in K = ceil(nwords / J) parallel segments;
// polys: K x 312 words (x^(kJ) mod phi, k = 0 .. K-1) on the device;
// ws: 312 * (64 + 2) + 312 * K words of scratch.
void launch_mt_jump(uint64_t seed, uint64_t nwords, uint64_t J, int K, const uint64_t* polys,
                    uint64_t* ws, uint64_t* out, cudaStream_t s) {
  uint64_t* prefix = ws;                   // kJumpPrefix raw words
  uint64_t* states = ws + kJumpPrefix + 8;  // (K - 1) x 312
  MtJobs jobs{};
  jobs.job[0] = MtJob{seed, (uint64_t)kJumpPrefix, prefix};
  note_launches(1);
  mt_stream_kernel<<<1, 160, 0, s>>>(jobs, 1);
  if (K > 1) {
    const int smem = (int)jump_state_smem();
    static std::atomic<unsigned> attr{0u};
    smem_attr_once(attr, (const void*)(mt_jump_state_kernel), smem);
    note_launches(1);
    const int parts = std::max(1, 148 / (K - 1));  // about one wave of CTAs
    cudaMemsetAsync(states, 0, sizeof(uint64_t) * kN * (K - 1), s);
    mt_jump_state_kernel<<<(K - 1) * parts, kJumpThreads, smem, s>>>(prefix, polys, states, parts);
  }
  note_launches(1);
  mt_segment_kernel<<<K, 160, 0, s>>>(prefix, states, J, nwords, out);
}
size_t mt_jump_ws_words(int K) { return (size_t)kJumpPrefix + 8 + (size_t)kN * (K > 1 ? K - 1 : 1); }

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

void launch_redraw_fill(const uint64_t* words, uint64_t nwords, uint64_t* pos, uint64_t rows_total,
                        uint64_t off, uint64_t count, double* col, int* flag, int nsm,
                        cudaStream_t s) {
  const int blocks = (int)std::min<uint64_t>((rows_total + 255) / 256, (uint64_t)nsm * 4);
  note_launches(2);
  redraw_map_kernel<<<blocks > 0 ? blocks : 1, 256, 0, s>>>(words, pos, rows_total, off, count,
                                                             col, flag);
  redraw_exact_kernel<<<1, 32, 0, s>>>(words, nwords, pos, rows_total, off, count, col, flag);
}

}  // namespace cnmf
