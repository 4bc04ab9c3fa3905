// dense.cu -- the uncompressed solvers' contractions and the multiplicative
// updates.
//
// Reference call sites:
//   fasthals_step / hals_step   solvers.cpp:96-187  p = X B, X^T A; g = B^T B, A^T A
//   mu_step                     solvers.cpp:55-64, 327-330
//   mu_rp_step                  solvers.cpp:69-93 (semi_nmf_half), 337-346
//
// Precision.  The uncompressed updates feed X B and X^T A straight into the
// column sweeps every iteration, and FastHALS trajectories amplify a relative
// perturbation of those products ~1e3x over 100 iterations (measured with a
// NumPy model of fasthals_step: 1e-7 per-entry noise -> 1.2e-4 trajectory
// deviation at 600 x 400, k = 16).  The tensor-core 3xTF32 stream is ~1e-6
// accurate, so these contractions run in fp64 on the CUDA cores (X converted
// exactly from fp32, fp64 accumulation), with split-K partials reduced in a
// fixed order: bitwise reproducible.  At k >= 10 this is fp64-FMA bound, not
// HBM bound (2 k flops per 4-byte X element vs ~4.7 flop/B machine balance).
#include "common.cuh"
#include "kernels.h"

namespace cnmf {

namespace {

constexpr int kBK = 32;    // reduction depth per stage (8 MMA k-steps of 4)
constexpr int kXT = 256;   // threads per X-stream CTA (8 warps: 4 row groups x 2 column halves)
// Up to LP = 96: two cp.async stages and two CTAs per SM (<= 128 registers):
// the range finder's fp64 passes at C3 take 107.5 ms vs 119-121 ms with one
// CTA of three or four stages (tools/rf_kappa.py; the second CTA hides the
// other's barriers).  Wider tiles keep one CTA of three stages (their 64+
// accumulator doubles do not fit 128 registers).
template <int LP> struct Xs64Occ {
  static constexpr int kStages = LP <= 96 ? 2 : 3;
  static constexpr int kMinBlocks = LP <= 96 ? 2 : 1;
};
constexpr int kNNS = kBK + 4;   // NN X-tile row stride (floats): conflict-free fragment reads
constexpr int kXBM = 128;  // output rows per CTA
constexpr int kTNS = kXBM + 8;  // TN X-tile row stride (floats)

template <int LP>
struct Xs64Shape {
  static constexpr int BM = kXBM;
  static constexpr int TN = LP / 16;        // 8-column MMA tiles per warp (half the columns)
  static constexpr int SLD = LP + 2;        // S-tile row stride (doubles)
  static constexpr int XF = (kXBM * kNNS > kBK * kTNS) ? kXBM * kNNS : kBK * kTNS;  // floats
  static constexpr size_t stage_bytes = sizeof(float) * XF + sizeof(double) * kBK * SLD;
  static constexpr int NS = Xs64Occ<LP>::kStages;
  static constexpr size_t smem = NS * stage_bytes;
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src), "r"(src_bytes)
               : "memory");
}

// fp32 -> fp64 on the integer pipe (exact for zero and normal numbers; the
// FP64 conversion unit issues at 1/4 the DFMA rate).  Subnormal inputs take
// the F2F path.
__device__ __forceinline__ double f2d_int(float f) {
  const uint32_t u = __float_as_uint(f), a = u & 0x7fffffffu;
  if (a < 0x00800000u && a != 0u) return (double)f;
  const uint32_t hi = (u & 0x80000000u) | (a ? (a >> 3) + 0x38000000u : 0u);
  return __hiloint2double((int)hi, (int)(u << 29));
}

// FP64 tensor-core MMA, D (8 x 8) += A (8 x 4, row) B (4 x 8, col): lane
// (g = lane / 4, t = lane % 4) supplies A[g][t], B[t][g] and holds D[g][2t],
// D[g][2t + 1] (tools/ubench_dmma.cu).
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// out[s][r][c] (s = blockIdx.y split) = sum over the split's K range of
// op(X)[r][k] S[k][c]; op(X) = X (NN: r < m, K = n) or X^T (TN: r < n, K = m).
// On the FP64 tensor cores: warp (wm, wn) owns rows 32 wm .. 32 wm + 31 and
// columns wn LP/2 .. of the CTA's 128 x LP tile as 4 x LP/16 MMA tiles; per
// k-step it loads one A value per m-tile (fp32, widened on the integer pipe)
// and one B value per n-tile -- two operand registers per 256 FMAs, where a
// SIMT fp64 tile moved 2.5 bytes of shared memory per FMA.  X (fp32) and S
// (fp64) stream through a 3-stage cp.async ring.
template <bool kTN, int LP>
__global__ void __launch_bounds__(kXT, Xs64Occ<LP>::kMinBlocks) xs64_kernel(const float* __restrict__ x, int64_t ldx,
                                                      int64_t m, int64_t n,
                                                      const double* __restrict__ s,
                                                      double* __restrict__ out, int64_t kchunk,
                                                      const int* __restrict__ halt) {
  if (halt && *(volatile const int*)halt) return;  // queued behind a HALS halt
  using Sh = Xs64Shape<LP>;
  constexpr int TN = Sh::TN, SLD = Sh::SLD;
  extern __shared__ __align__(16) unsigned char xs64_smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int wm = warp & 3, wn = warp >> 2;
  const int64_t out_rows = kTN ? n : m, K = kTN ? m : n;
  const int64_t row0 = (int64_t)blockIdx.x * kXBM;
  const int64_t kbeg = (int64_t)blockIdx.y * kchunk, kend = min(K, kbeg + kchunk);
  double* dst = out + (int64_t)blockIdx.y * out_rows * LP;
  auto xbuf = [&](int b) { return reinterpret_cast<float*>(xs64_smem + b * Sh::stage_bytes); };
  auto sbuf = [&](int b) {
    return reinterpret_cast<double*>(xs64_smem + b * Sh::stage_bytes + sizeof(float) * Sh::XF);
  };

  auto issue = [&](int64_t k0, int b) {
    float* xs = xbuf(b);
    for (int e = tid; e < kXBM * kBK / 4; e += kXT) {  // 16-byte chunks of X
      const float* src = x;
      int bytes = 0;
      float* d;
      if (!kTN) {  // row e / 8, k quad e % 8
        const int r = e >> 3, q = e & 7;
        const int64_t gr = row0 + r, gk = k0 + 4 * q;
        d = xs + r * kNNS + 4 * q;
        if (gr < m && gk < kend) {
          src = x + gr * ldx + gk;
          bytes = (int)(4 * (kend - gk < 4 ? kend - gk : 4));
        }
      } else {     // k row e / 32, column quad e % 32
        const int kk = e >> 5, c4 = e & 31;
        const int64_t gk = k0 + kk, gr = row0 + 4 * c4;
        d = xs + kk * kTNS + 4 * c4;
        if (gk < kend && gr < n) {
          src = x + gk * ldx + gr;
          bytes = (int)(4 * (n - gr < 4 ? n - gr : 4));
        }
      }
      cp_async16(d, src, bytes);
    }
    double* ss = sbuf(b);
    for (int e = tid; e < kBK * LP / 2; e += kXT) {  // 16-byte chunks of S
      const int kk = e / (LP / 2), c2 = e % (LP / 2);
      const int64_t gk = k0 + kk;
      cp_async16(ss + kk * SLD + 2 * c2, gk < kend ? s + gk * LP + 2 * c2 : s, gk < kend ? 16 : 0);
    }
  };

  double acc[4][TN][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int64_t nst = (kend - kbeg + kBK - 1) / kBK;
#pragma unroll
  constexpr int kNS = Sh::NS;
  for (int p = 0; p < kNS - 1; ++p) {
    if (p < nst) issue(kbeg + p * kBK, p);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int64_t st = 0; st < nst; ++st) {
    asm volatile("cp.async.wait_group %0;" ::"n"(kNS - 2) : "memory");
    __syncthreads();  // stage st visible to all; stage st - 1 fully consumed
    if (st + kNS - 1 < nst) issue(kbeg + (st + kNS - 1) * kBK, (int)((st + kNS - 1) % kNS));
    asm volatile("cp.async.commit_group;" ::: "memory");
    const int b = (int)(st % kNS);
    const float* xs = xbuf(b);
    const double* sb = sbuf(b) + wn * (LP / 2) + g;
#pragma unroll
    for (int ks = 0; ks < kBK / 4; ++ks) {
      const int kk = 4 * ks + t4;
      double av[4], bv[TN];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = 32 * wm + 8 * i + g;
        av[i] = f2d_int(kTN ? xs[kk * kTNS + r] : xs[r * kNNS + kk]);
      }
#pragma unroll
      for (int j = 0; j < TN; ++j) bv[j] = sb[kk * SLD + 8 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) dmma(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = row0 + 32 * wm + 8 * i + g;
    if (r < out_rows)
#pragma unroll
      for (int j = 0; j < TN; ++j)
        *reinterpret_cast<double2*>(dst + r * LP + wn * (LP / 2) + 8 * j + 2 * t4) =
            make_double2(acc[i][j][0], acc[i][j][1]);
  }
}

__global__ void reduce_splits64_kernel(const double* __restrict__ part, int splits, int64_t total,
                                       double* __restrict__ out, const int* __restrict__ halt) {
  if (halt && *(volatile const int*)halt) return;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < splits; ++q) s += part[(int64_t)q * total + e];
    out[e] = s;
  }
}

// Per-CTA partial Gram of a k-column fp64 factor with element (r, a) at
// f[a cs + r rs] (column-major k x rows: cs = rows, rs = 1; row-major
// rows x k: cs = 1, rs = k): part[cta][a][b] = sum over the CTA's rows
// (ascending) of F(r, a) F(r, b); 4 x 4 tiles of the upper triangle, up to 3
// tiles per thread (k <= 128).
constexpr int kGR = 32;  // rows per stage
__global__ void __launch_bounds__(256) gram_cm_kernel(const double* __restrict__ f, int64_t rows,
                                                      int k, int64_t cs, int64_t rs,
                                                      int64_t rows_per_cta,
                                                      double* __restrict__ part,
                                                      const int* __restrict__ halt) {
  if (halt && *(volatile const int*)halt) return;
  extern __shared__ __align__(16) double gst[];
  const int k4 = (k + 3) & ~3, nb4 = k4 >> 2, nb = nb4 * (nb4 + 1) / 2;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta, r1 = min(rows, r0 + rows_per_cta);
  double acc[3][16];
  int bi[3], bj[3];
#pragma unroll
  for (int u = 0; u < 3; ++u) {
    int b = threadIdx.x + 256 * u, i = 0;
    if (b < nb) {
      while (b >= nb4 - i) {
        b -= nb4 - i;
        ++i;
      }
    }
    bi[u] = i;
    bj[u] = i + b;
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[u][e] = 0.0;
  }
  for (int64_t s0 = r0; s0 < r1; s0 += kGR) {
    __syncthreads();
    for (int e = threadIdx.x; e < kGR * k4; e += 256) {
      const int c = e / kGR, rr = e % kGR;
      const int64_t r = s0 + rr;
      gst[rr * k4 + c] = (c < k && r < r1) ? f[(int64_t)c * cs + r * rs] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      if (threadIdx.x + 256 * u >= nb) break;
      for (int rr = 0; rr < kGR; ++rr) {
        double xv[4], yv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          xv[i] = gst[rr * k4 + 4 * bi[u] + i];
          yv[i] = gst[rr * k4 + 4 * bj[u] + i];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[u][4 * i + j] = fma(xv[i], yv[j], acc[u][4 * i + j]);
      }
    }
  }
  double* out = part + (int64_t)blockIdx.x * k * k;
#pragma unroll
  for (int u = 0; u < 3; ++u) {
    if (threadIdx.x + 256 * u >= nb) break;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int a = 4 * bi[u] + i, b = 4 * bj[u] + j;
        if (a < k && b < k) {
          out[a * k + b] = acc[u][4 * i + j];
          out[b * k + a] = acc[u][4 * i + j];
        }
      }
  }
}

// column-major k x rows fp64 -> row-major rows x lp fp64, zero-padded columns
__global__ void cm_to_rm_pad64_kernel(const double* __restrict__ f, int64_t rows, int k, int lp,
                                      double* __restrict__ out, const int* __restrict__ halt) {
  if (halt && *(volatile const int*)halt) return;
  const int64_t total = rows * lp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / lp;
    const int c = (int)(e - r * lp);
    out[e] = c < k ? f[(int64_t)c * rows + r] : 0.0;
  }
}

// Multiplicative update of a column-major k x rows factor T (one thread per
// row, every column against the OLD row: the denominator T g is formed before
// any entry changes, solvers.cpp:60-63):
//   semi = 0: t_j *= num_j / ((T g)_j + 1e-12)                   (mu_update_half)
//   semi = 1: t_j *= sqrt((num_j^+ + (T g^-)_j) /
//                         (num_j^- + (T g^+)_j + 1e-12))         (semi_nmf_half)
// num: row-major rows x ldn fp64.  The new factor goes to t_out.
__global__ void mu_update_kernel(const double* __restrict__ t_in, int64_t rows, int k,
                                 const double* __restrict__ num, int ldn,
                                 const double* __restrict__ g, int semi,
                                 double* __restrict__ t_out) {
  extern __shared__ double mu_g[];
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) mu_g[e] = g[e];
  __syncthreads();
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    for (int j = 0; j < k; ++j) {
      double pos = 0.0, neg = 0.0;
      for (int c = 0; c < k; ++c) {  // matmul order: c ascending (matrix.cpp:105-116)
        const double tv = t_in[(int64_t)c * rows + r], gv = mu_g[c * k + j];
        if (!semi) {
          pos += tv * gv;
        } else {
          if (gv > 0.0) pos += tv * gv;
          else neg += tv * (-gv);
        }
      }
      const double t = t_in[(int64_t)j * rows + r], nv = num[r * ldn + j];
      double v;
      if (!semi) {
        v = t * (nv / (pos + 1e-12));
      } else {
        const double numer = (nv > 0.0 ? nv : 0.0) + neg;
        const double denom = (nv < 0.0 ? -nv : 0.0) + pos + 1e-12;
        v = t * sqrt(numer / denom);
      }
      t_out[(int64_t)j * rows + r] = v;
    }
  }
}

// out[r][j] = sum_{q < l} in[r][q] m[q][j]: a rows x lp fp32 view times an
// lp x k fp64 matrix (rows >= l of m unused), fp64, q ascending.
__global__ void rows_small64_kernel(const float* __restrict__ in, int64_t rows, int l, int lp,
                                    const double* __restrict__ m, int k, double* __restrict__ out,
                                    int ldo) {
  extern __shared__ double rs_m[];
  for (int e = threadIdx.x; e < l * k; e += blockDim.x) rs_m[e] = m[e];
  __syncthreads();
  const int64_t total = rows * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / k;
    const int j = (int)(e - r * k);
    const float* row = in + r * lp;
    double s = 0.0;
    for (int q = 0; q < l; ++q) s = fma((double)row[q], rs_m[q * k + j], s);
    out[r * ldo + j] = s;
  }
}

// Split-K plan: fewest waves per unit of K work, cost(s) = ceil(tiles s / nsm) / s
// (+ a small charge per split for the partial-sum traffic).
int64_t xs64_splits(int64_t tiles, int64_t K, int nsm) {
  int64_t best = 1;
  double best_cost = 1e300;
  const int64_t smax = std::max<int64_t>(1, std::min<int64_t>(64, K / (4 * kBK)));
  for (int64_t sp = 1; sp <= smax; ++sp) {
    const double cost = (double)((tiles * sp + nsm - 1) / nsm) / (double)sp + 0.002 * (double)sp;
    if (cost < best_cost) {
      best_cost = cost;
      best = sp;
    }
  }
  return best;
}

template <bool kTN, int LP>
void xs64_launch(const float* x, int64_t ldx, int64_t m, int64_t n, const double* s, double* out,
                 double* ws, int nsm, cudaStream_t st, const int* halt) {
  using Sh = Xs64Shape<LP>;
  const int64_t out_rows = kTN ? n : m, K = kTN ? m : n;
  const int64_t tiles = (out_rows + Sh::BM - 1) / Sh::BM;
  int64_t splits = xs64_splits(tiles, K, nsm);
  const int64_t kchunk = ((K + splits - 1) / splits + kBK - 1) / kBK * kBK;
  splits = (K + kchunk - 1) / kchunk;
  static std::atomic<unsigned> attr{0u};
  smem_attr_once(attr, (const void*)(xs64_kernel<kTN, LP>), (int)Sh::smem);
  double* dst = splits > 1 ? ws : out;
  note_launches(1);
  xs64_kernel<kTN, LP><<<dim3((unsigned)tiles, (unsigned)splits), kXT, Sh::smem, st>>>(
      x, ldx, m, n, s, dst, kchunk, halt);
  if (splits > 1) {
    const int64_t total = out_rows * LP;
    note_launches(1);
    reduce_splits64_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 8 * nsm), 256, 0,
                             st>>>(ws, (int)splits, total, out, halt);
  }
}

template <bool kTN>
void xs64_dispatch(const float* x, int64_t ldx, int64_t m, int64_t n, const double* s, int lp,
                   double* out, double* ws, int nsm, cudaStream_t st, const int* halt) {
  switch (lp) {
    case 16: xs64_launch<kTN, 16>(x, ldx, m, n, s, out, ws, nsm, st, halt); break;
    case 32: xs64_launch<kTN, 32>(x, ldx, m, n, s, out, ws, nsm, st, halt); break;
    case 48: xs64_launch<kTN, 48>(x, ldx, m, n, s, out, ws, nsm, st, halt); break;
    case 64: xs64_launch<kTN, 64>(x, ldx, m, n, s, out, ws, nsm, st, halt); break;
    case 80: xs64_launch<kTN, 80>(x, ldx, m, n, s, out, ws, nsm, st, halt); break;
    case 96: xs64_launch<kTN, 96>(x, ldx, m, n, s, out, ws, nsm, st, halt); break;
    case 112: xs64_launch<kTN, 112>(x, ldx, m, n, s, out, ws, nsm, st, halt); break;
    case 128: xs64_launch<kTN, 128>(x, ldx, m, n, s, out, ws, nsm, st, halt); break;
    default: break;  // callers pad to a multiple of 16 <= 128
  }
}

// One 32-row stage per CTA where the k x k tiles leave most threads idle
// (small k: the per-CTA work is a short dependent chain, so spread the rows);
// one CTA per SM at most once every thread owns a tile.
int gram_grid(int64_t rows, int k, int nsm) {
  const int nb4 = (k + 3) / 4, nb = nb4 * (nb4 + 1) / 2;
  const int64_t cap = nb >= 128 ? nsm : 4 * (int64_t)nsm;
  return (int)std::max<int64_t>(1, std::min<int64_t>(cap, (rows + 31) / 32));
}

}  // namespace

size_t xs64_ws_doubles(int64_t m, int64_t n, int lp, int nsm) {
  // split-K partials of either orientation, with the launch's own plan
  const int64_t bm = kXBM;
  size_t most = 0;
  for (int tn = 0; tn < 2; ++tn) {
    const int64_t rows = tn ? n : m, K = tn ? m : n;
    const int64_t tiles = (rows + bm - 1) / bm;
    int64_t sp = xs64_splits(tiles, K, nsm);
    const int64_t kchunk = ((K + sp - 1) / sp + kBK - 1) / kBK * kBK;
    sp = (K + kchunk - 1) / kchunk;
    if (sp > 1) most = std::max(most, (size_t)(sp * rows * lp));
  }
  return std::max<size_t>(most, 1);
}

void launch_xs64_nn(const float* x, int64_t ldx, int64_t m, int64_t n, const double* s, int lp,
                    double* out, double* ws, int nsm, cudaStream_t st, const int* halt) {
  xs64_dispatch<false>(x, ldx, m, n, s, lp, out, ws, nsm, st, halt);
}

void launch_xs64_tn(const float* x, int64_t ldx, int64_t m, int64_t n, const double* t, int lp,
                    double* out, double* ws, int nsm, cudaStream_t st, const int* halt) {
  xs64_dispatch<true>(x, ldx, m, n, t, lp, out, ws, nsm, st, halt);
}

size_t gram_cm_ws_doubles(int64_t rows, int k, int nsm) {
  return (size_t)gram_grid(rows, k, nsm) * k * k;
}

void launch_gram_cm(const double* f_cm, int64_t rows, int k, double* g, double* ws, int nsm,
                    cudaStream_t st, bool row_major, const int* halt) {
  const int grid = gram_grid(rows, k, nsm);
  const int64_t per = (rows + grid - 1) / grid;
  const int k4 = (k + 3) & ~3;
  note_launches(2);
  gram_cm_kernel<<<grid, 256, sizeof(double) * kGR * k4, st>>>(
      f_cm, rows, k, row_major ? 1 : rows, row_major ? k : 1, per, ws, halt);
  reduce_splits64_kernel<<<(k * k + 255) / 256, 256, 0, st>>>(ws, grid, (int64_t)k * k, g, halt);
}

void launch_cm_to_rm_pad64(const double* f_cm, int64_t rows, int k, int lp, double* out,
                           int nsm, cudaStream_t st, const int* halt) {
  const int64_t total = rows * lp;
  note_launches(1);
  cm_to_rm_pad64_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 8 * nsm), 256, 0,
                          st>>>(f_cm, rows, k, lp, out, halt);
}

void launch_mu_update(const double* t_in, int64_t rows, int k, const double* num, int ldn,
                      const double* g, int semi, double* t_out, int nsm, cudaStream_t st) {
  static std::atomic<unsigned> attr{0u};
  smem_attr_once(attr, (const void*)(mu_update_kernel), (int)(sizeof(double) * 128 * 128));
  note_launches(1);
  mu_update_kernel<<<(unsigned)std::min<int64_t>((rows + 127) / 128, 8 * nsm), 128,
                     sizeof(double) * k * k, st>>>(t_in, rows, k, num, ldn, g, semi, t_out);
}

void launch_rows_small64(const float* in, int64_t rows, int l, int lp, const double* m, int k,
                         double* out, int ldo, int nsm, cudaStream_t st) {
  const int64_t total = rows * k;
  static std::atomic<unsigned> attr{0u};
  smem_attr_once(attr, (const void*)(rows_small64_kernel), (int)(sizeof(double) * 128 * 128));
  note_launches(1);
  rows_small64_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 8 * nsm), 256,
                        sizeof(double) * l * k, st>>>(in, rows, l, lp, m, k, out, ldo);
}

}  // namespace cnmf
