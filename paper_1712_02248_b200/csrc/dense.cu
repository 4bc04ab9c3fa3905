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

constexpr int kBK = 8;     // reduction depth per stage
constexpr int kXT = 256;   // threads per X-stream CTA

template <int LP>
struct Xs64Shape {
  static constexpr int CG = LP / 16;        // 16-column groups
  static constexpr int RS = kXT / CG;       // row stride between a thread's 4 rows
  static constexpr int BM = 4 * RS;         // output rows per CTA
  static constexpr int XF4 = (2 * BM + kXT - 1) / kXT;  // X float4 per thread per stage
  static constexpr size_t smem = sizeof(double) * 2 * kBK * (BM + LP);
};

// out[s][r][c] (s = blockIdx.y split) = sum over the split's K range of
// op(X)[r][k] S[k][c]; op(X) = X (NN: r < m, K = n) or X^T (TN: r < n, K = m).
// Thread tile: rows rg + RS i (i < 4) x columns 16 cg .. 16 cg + 15 (threads
// beyond RS * CG only load).  X staged as fp64 [kBK][BM], S as [kBK][LP];
// both double-buffered through registers, one barrier per stage.
template <bool kTN, int LP>
__global__ void __launch_bounds__(kXT, 1) xs64_kernel(const float* __restrict__ x, int64_t ldx,
                                                      int64_t m, int64_t n,
                                                      const double* __restrict__ s,
                                                      double* __restrict__ out, int64_t kchunk) {
  using Sh = Xs64Shape<LP>;
  constexpr int CG = Sh::CG, RS = Sh::RS, BM = Sh::BM, XF4 = Sh::XF4;
  constexpr int SD2 = kBK * LP / 2;  // double2 of S per stage
  constexpr int SPT = (SD2 + kXT - 1) / kXT;
  extern __shared__ __align__(16) double xs64_smem[];
  double* Xs = xs64_smem;                // [2][kBK][BM]
  double* Ss = xs64_smem + 2 * kBK * BM;  // [2][kBK][LP]
  const int tid = threadIdx.x, cg = tid % CG, rg = tid / CG;
  const bool computes = rg < RS;
  const int64_t out_rows = kTN ? n : m, K = kTN ? m : n;
  const int64_t row0 = (int64_t)blockIdx.x * BM;
  const int64_t kbeg = (int64_t)blockIdx.y * kchunk, kend = min(K, kbeg + kchunk);
  double* dst = out + (int64_t)blockIdx.y * out_rows * LP;

  float4 px[XF4];
  double2 ps[SPT];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int u = 0; u < XF4; ++u) {
      const int e = tid + kXT * u;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (e < 2 * BM) {
        if (!kTN) {  // row e / 2, k offset 4 (e % 2)
          const int64_t gr = row0 + (e >> 1), gk = k0 + 4 * (e & 1);
          if (gr < m && gk < kend) {
            const float* src = x + gr * ldx + gk;
            if (gk + 3 < kend) {
              v = __ldg(reinterpret_cast<const float4*>(src));
            } else {
              v.x = src[0];
              if (gk + 1 < kend) v.y = src[1];
              if (gk + 2 < kend) v.z = src[2];
            }
          }
        } else {     // k offset e / (BM / 4), rows 4 (e % (BM / 4)) ..
          const int64_t gk = k0 + e / (BM / 4), gr = row0 + 4 * (e % (BM / 4));
          if (gk < kend && gr < n) {
            const float* src = x + gk * ldx + gr;
            if (gr + 3 < n) {
              v = __ldg(reinterpret_cast<const float4*>(src));
            } else {
              v.x = src[0];
              if (gr + 1 < n) v.y = src[1];
              if (gr + 2 < n) v.z = src[2];
            }
          }
        }
      }
      px[u] = v;
    }
#pragma unroll
    for (int u = 0; u < SPT; ++u) {
      const int e = tid + kXT * u;
      const int kk = e / (LP / 2), c2 = e % (LP / 2);
      const int64_t gk = k0 + kk;
      ps[u] = (e < SD2 && gk < kend) ? __ldg(reinterpret_cast<const double2*>(s + gk * LP) + c2)
                                     : make_double2(0.0, 0.0);
    }
  };
  auto store = [&](int buf) {
    double* xb = Xs + buf * kBK * BM;
#pragma unroll
    for (int u = 0; u < XF4; ++u) {
      const int e = tid + kXT * u;
      if (e < 2 * BM) {
        if (!kTN) {
          const int r = e >> 1, k4 = 4 * (e & 1);
          xb[(k4 + 0) * BM + r] = px[u].x;
          xb[(k4 + 1) * BM + r] = px[u].y;
          xb[(k4 + 2) * BM + r] = px[u].z;
          xb[(k4 + 3) * BM + r] = px[u].w;
        } else {
          const int kk = e / (BM / 4), c = 4 * (e % (BM / 4));
          double2* d2 = reinterpret_cast<double2*>(xb + kk * BM + c);
          d2[0] = make_double2(px[u].x, px[u].y);
          d2[1] = make_double2(px[u].z, px[u].w);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < SPT; ++u) {
      const int e = tid + kXT * u;
      if (e < SD2) reinterpret_cast<double2*>(Ss + buf * kBK * LP)[e] = ps[u];
    }
  };

  double acc[4][16];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int c = 0; c < 16; ++c) acc[i][c] = 0.0;

  const int64_t nst = (kend - kbeg + kBK - 1) / kBK;
  if (nst > 0) load(kbeg);
  for (int64_t st = 0; st < nst; ++st) {
    const int buf = (int)(st & 1);
    store(buf);
    __syncthreads();  // also orders this store after every read of buf two stages ago
    if (st + 1 < nst) load(kbeg + (st + 1) * kBK);
    if (computes) {
      const double* xb = Xs + buf * kBK * BM + rg;
      const double* sb = Ss + buf * kBK * LP + 16 * cg;
#pragma unroll
      for (int kk = 0; kk < kBK; ++kk) {
        double xv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) xv[i] = xb[kk * BM + RS * i];
#pragma unroll
        for (int c2 = 0; c2 < 8; ++c2) {
          const double2 sv = reinterpret_cast<const double2*>(sb + kk * LP)[c2];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            acc[i][2 * c2] = fma(xv[i], sv.x, acc[i][2 * c2]);
            acc[i][2 * c2 + 1] = fma(xv[i], sv.y, acc[i][2 * c2 + 1]);
          }
        }
      }
    }
  }
  if (computes) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t r = row0 + rg + RS * i;
      if (r < out_rows) {
        double2* o = reinterpret_cast<double2*>(dst + r * LP + 16 * cg);
#pragma unroll
        for (int c2 = 0; c2 < 8; ++c2) o[c2] = make_double2(acc[i][2 * c2], acc[i][2 * c2 + 1]);
      }
    }
  }
}

__global__ void reduce_splits64_kernel(const double* __restrict__ part, int splits, int64_t total,
                                       double* __restrict__ out) {
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
                                                      double* __restrict__ part) {
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
                                      double* __restrict__ out) {
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

template <bool kTN, int LP>
void xs64_launch(const float* x, int64_t ldx, int64_t m, int64_t n, const double* s, double* out,
                 double* ws, int nsm, cudaStream_t st) {
  using Sh = Xs64Shape<LP>;
  const int64_t out_rows = kTN ? n : m, K = kTN ? m : n;
  const int64_t tiles = (out_rows + Sh::BM - 1) / Sh::BM;
  // one wave of one CTA per SM (the kernel is fp64-FMA bound with 8 warps)
  int64_t splits = std::max<int64_t>(1, ((int64_t)nsm + tiles - 1) / tiles);
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, K / (4 * kBK)));
  const int64_t kchunk = ((K + splits - 1) / splits + kBK - 1) / kBK * kBK;
  splits = (K + kchunk - 1) / kchunk;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(xs64_kernel<kTN, LP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Sh::smem);
    attr = true;
  }
  double* dst = splits > 1 ? ws : out;
  note_launches(1);
  xs64_kernel<kTN, LP><<<dim3((unsigned)tiles, (unsigned)splits), kXT, Sh::smem, st>>>(
      x, ldx, m, n, s, dst, kchunk);
  if (splits > 1) {
    const int64_t total = out_rows * LP;
    note_launches(1);
    reduce_splits64_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 8 * nsm), 256, 0,
                             st>>>(ws, (int)splits, total, out);
  }
}

template <bool kTN>
void xs64_dispatch(const float* x, int64_t ldx, int64_t m, int64_t n, const double* s, int lp,
                   double* out, double* ws, int nsm, cudaStream_t st) {
  switch (lp) {
    case 16: xs64_launch<kTN, 16>(x, ldx, m, n, s, out, ws, nsm, st); break;
    case 32: xs64_launch<kTN, 32>(x, ldx, m, n, s, out, ws, nsm, st); break;
    case 48: xs64_launch<kTN, 48>(x, ldx, m, n, s, out, ws, nsm, st); break;
    case 64: xs64_launch<kTN, 64>(x, ldx, m, n, s, out, ws, nsm, st); break;
    case 80: xs64_launch<kTN, 80>(x, ldx, m, n, s, out, ws, nsm, st); break;
    case 96: xs64_launch<kTN, 96>(x, ldx, m, n, s, out, ws, nsm, st); break;
    case 112: xs64_launch<kTN, 112>(x, ldx, m, n, s, out, ws, nsm, st); break;
    case 128: xs64_launch<kTN, 128>(x, ldx, m, n, s, out, ws, nsm, st); break;
    default: break;  // callers pad to a multiple of 16 <= 128
  }
}

int gram_grid(int64_t rows, int nsm) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(nsm, (rows + 255) / 256));
}

}  // namespace

size_t xs64_ws_doubles(int64_t m, int64_t n, int lp, int nsm) {
  // split-K partials: splits <= ceil(nsm / tiles), so splits * rows <=
  // (nsm + tiles) * BM <= nsm * 1024 + rows + 1024
  const int64_t rows = std::max(m, n);
  return (size_t)(((int64_t)nsm * 1024 + rows + 1024) * lp);
}

void launch_xs64_nn(const float* x, int64_t ldx, int64_t m, int64_t n, const double* s, int lp,
                    double* out, double* ws, int nsm, cudaStream_t st) {
  xs64_dispatch<false>(x, ldx, m, n, s, lp, out, ws, nsm, st);
}

void launch_xs64_tn(const float* x, int64_t ldx, int64_t m, int64_t n, const double* t, int lp,
                    double* out, double* ws, int nsm, cudaStream_t st) {
  xs64_dispatch<true>(x, ldx, m, n, t, lp, out, ws, nsm, st);
}

size_t gram_cm_ws_doubles(int64_t rows, int k, int nsm) {
  return (size_t)gram_grid(rows, nsm) * k * k;
}

void launch_gram_cm(const double* f_cm, int64_t rows, int k, double* g, double* ws, int nsm,
                    cudaStream_t st, bool row_major) {
  const int grid = gram_grid(rows, nsm);
  const int64_t per = (rows + grid - 1) / grid;
  const int k4 = (k + 3) & ~3;
  note_launches(2);
  gram_cm_kernel<<<grid, 256, sizeof(double) * kGR * k4, st>>>(
      f_cm, rows, k, row_major ? 1 : rows, row_major ? k : 1, per, ws);
  reduce_splits64_kernel<<<(k * k + 255) / 256, 256, 0, st>>>(ws, grid, (int64_t)k * k, g);
}

void launch_cm_to_rm_pad64(const double* f_cm, int64_t rows, int k, int lp, double* out,
                           int nsm, cudaStream_t st) {
  const int64_t total = rows * lp;
  note_launches(1);
  cm_to_rm_pad64_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 8 * nsm), 256, 0,
                          st>>>(f_cm, rows, k, lp, out);
}

void launch_mu_update(const double* t_in, int64_t rows, int k, const double* num, int ldn,
                      const double* g, int semi, double* t_out, int nsm, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(mu_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(double) * 128 * 128));
    attr = true;
  }
  note_launches(1);
  mu_update_kernel<<<(unsigned)std::min<int64_t>((rows + 127) / 128, 8 * nsm), 128,
                     sizeof(double) * k * k, st>>>(t_in, rows, k, num, ldn, g, semi, t_out);
}

void launch_rows_small64(const float* in, int64_t rows, int l, int lp, const double* m, int k,
                         double* out, int ldo, int nsm, cudaStream_t st) {
  const int64_t total = rows * k;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(rows_small64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(double) * 128 * 128));
    attr = true;
  }
  note_launches(1);
  rows_small64_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 8 * nsm), 256,
                        sizeof(double) * l * k, st>>>(in, rows, l, lp, m, k, out, ldo);
}

}  // namespace cnmf
