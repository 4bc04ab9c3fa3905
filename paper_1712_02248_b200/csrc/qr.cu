// qr.cu -- orthonormal bases for the range finders.
//
// Reference: thin_qr (proj/src/qr.cpp:10-75), Householder with a
// rank-deficiency floor of 1e-12 ||M||_F, called after every application of X
// or X^T in range_finder_impl (proj/src/compression.cpp:32-40).  Only the
// SPAN of Q enters FastHALS-RP (the step depends on L L^T and R^T R only,
// solvers.cpp:421-443), so the device uses CholeskyQR2:
//   G1 = Y^T Y (fp64) -> R1 = chol(G1) -> Q1 = Y R1^-1 -> G2 = Q1^T Q1 -> Q = Q1 R2^-1.
// The first Gram must be fp64 (cond(Y) reaches ~1e5, so cond(G1) ~ 1e10).
// When a Cholesky pivot shows Y numerically rank deficient, a single-CTA
// fp64 Householder QR with the reference's floor and completion rule
// replaces the result (rare path: exactly low-rank test data).
#include "common.cuh"
#include "kernels.h"

#include <functional>
#include <vector>

namespace cnmf {

namespace {

constexpr int kGramRows = 64;

struct QrWs {
  double* part;    // [grid][lp*lp]
  double* g;       // lp x lp
  double* rinv64;  // lp x lp
  float* rinv;     // lp x lp
  float* q1;       // rows x lp
  int* flag;
  double* hw;      // rows x lp (Householder working copy / Q)
  double* hv;      // rows x lp (reflectors)
  float* xs_ws;    // split-K scratch for the apply step
};

int gram_grid(int64_t rows, int nsm) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(nsm, (rows + kGramRows - 1) / kGramRows));
}

QrWs carve(void* ws, int64_t rows, int lp, int nsm) {
  QrWs w;
  char* p = static_cast<char*>(ws);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) & ~size_t(255);
    return r;
  };
  const int grid = gram_grid(rows, nsm);
  w.part = (double*)take(sizeof(double) * grid * lp * lp);
  w.g = (double*)take(sizeof(double) * lp * lp);
  w.rinv64 = (double*)take(sizeof(double) * lp * lp);
  w.rinv = (float*)take(sizeof(float) * lp * lp);
  w.q1 = (float*)take(sizeof(float) * rows * lp);
  w.flag = (int*)take(sizeof(int) * 4);
  w.hw = (double*)take(sizeof(double) * rows * lp);
  w.hv = (double*)take(sizeof(double) * rows * lp);
  w.xs_ws = (float*)take(sizeof(float) * xstream_ws_floats(rows, lp, lp, nsm));
  return w;
}

// Per-CTA fp64 partial of Y^T Y over its row chunks; upper-triangle 4x4
// blocks, thread t owns blocks t, t+256, t+512.
__global__ void __launch_bounds__(256) gram_kernel(const float* __restrict__ y, int64_t rows,
                                                   int l, int lp, double* __restrict__ part) {
  extern __shared__ __align__(16) float ys[];  // kGramRows x (lp + 4)
  const int lps = lp + 4;
  const int nbl = (l + 3) >> 2, nb = nbl * (nbl + 1) / 2;
  int bi[3], bj[3];
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    int b = threadIdx.x + 256 * t;
    bi[t] = -1;
    bj[t] = -1;
    if (b < nb) {
      int i = 0;
      while (b >= nbl - i) {
        b -= nbl - i;
        ++i;
      }
      bi[t] = i;
      bj[t] = i + b;
    }
  }
  double acc[3][16];
#pragma unroll
  for (int t = 0; t < 3; ++t)
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[t][e] = 0.0;
  const int64_t nchunks = (rows + kGramRows - 1) / kGramRows;
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int64_t r0 = ch * kGramRows;
    const int nr = (int)((rows - r0) < kGramRows ? (rows - r0) : kGramRows);
    __syncthreads();
    for (int e = threadIdx.x; e < kGramRows * (lp / 4); e += 256) {
      const int r = e / (lp / 4), c4 = e - r * (lp / 4);
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < nr) v = *reinterpret_cast<const float4*>(y + (r0 + r) * lp + 4 * c4);
      *reinterpret_cast<float4*>(ys + r * lps + 4 * c4) = v;
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      if (bi[t] < 0) continue;
      for (int r = 0; r < nr; ++r) {
        const float4 a = *reinterpret_cast<const float4*>(ys + r * lps + 4 * bi[t]);
        const float4 b = *reinterpret_cast<const float4*>(ys + r * lps + 4 * bj[t]);
        const double av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[t][4 * i + j] = fma(av[i], bv[j], acc[t][4 * i + j]);
      }
    }
  }
  double* dst = part + (int64_t)blockIdx.x * lp * lp;
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    if (bi[t] < 0) continue;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dst[(4 * bi[t] + i) * lp + 4 * bj[t] + j] = acc[t][4 * i + j];
  }
}

// G[a][b] (a <= b < l) = fixed-order sum of partials (lanes over CTAs, then
// a warp tree), mirrored; zero outside l x l.  One warp per entry.
__global__ void gram_reduce_kernel(const double* __restrict__ part, int grid, int l, int lp,
                                   double* __restrict__ g) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int e = w; e < lp * lp; e += nw) {
    const int a = e / lp, b = e - a * lp;
    double s = 0.0;
    if (a < l && b < l) {
      const int lo = min(a, b), hi = max(a, b);
      for (int c = lane; c < grid; c += 32) s += part[(int64_t)c * lp * lp + lo * lp + hi];
      s = warp_sum(s);
    }
    if (lane == 0) g[e] = s;
  }
}

// Cholesky G = R^T R (R upper) and R^-1 in one CTA of 1024 threads (fp64,
// shared memory), ONE elimination sweep with one barrier per column.
// Symmetric Gaussian elimination G = L D L^T (L unit lower, D the pivots)
// gives R = D^1/2 L^T, hence R^-1 = L^-T D^-1/2, and L^-1 is what the same row
// operations make of the identity.  Row a of the workspace holds both: its
// strict lower part (columns < a) the row of M -> L^-1 (unit diagonal
// implicit), its upper part (columns >= a) the row of the trailing G.  At
// step j every row a > j takes f_a = G[j][a] / p_j times row j off both parts:
// columns < j of M, M[a][j] = -f_a, columns >= a of G.  A warp owns a row, its
// lanes the columns (l <= 128: four per lane).
// Afterwards R^-1[i][c] = M[c][i] / sqrt(p_c).  The previous version ran the
// factorisation and a right-looking back substitution as two sweeps of l
// barriers each on 128 threads: 389 us per call at l = 120, 40 us at l = 36
// (profiles/r02_c4_launch_summary.txt).
// flag |= 1 when a pivot is non-positive or below 1e-13 of its original
// diagonal (Y numerically rank deficient at fp32 resolution -> Householder).
constexpr int kCholThreads = 1024;
__global__ void __launch_bounds__(kCholThreads) chol_inv_kernel(const double* __restrict__ g, int l,
                                                                int lp, double* __restrict__ rinv64,
                                                                float* __restrict__ rinv,
                                                                int* __restrict__ flag) {
  extern __shared__ double gs[];
  const int ls = l | 1;
  double* diag0 = gs + l * ls;
  double* rdi = diag0 + l;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  for (int e = tid; e < l * l; e += nt) {
    const int a = e / l, b = e - a * l;
    gs[a * ls + b] = b >= a ? g[a * lp + b] : 0.0;
  }
  for (int e = tid; e < l; e += nt) diag0[e] = g[e * lp + e];
  for (int e = tid; e < lp * lp; e += nt) {  // padding and the lower triangle stay zero
    rinv[e] = 0.f;
    rinv64[e] = 0.0;
  }
  __syncthreads();
  for (int j = 0; j < l; ++j) {
    const double* rowj = gs + j * ls;
    const double piv = rowj[j];
    if (!(piv > 1e-13 * diag0[j]) || !(piv > 0.0)) {  // uniform across the CTA
      if (tid == 0) *flag = 1;
      return;
    }
    const double ip = __drcp_rn(piv);
    // lane t owns columns t + 32 u of every row: row j's values are loaded
    // once per step (M[j][j] = 1 is implicit -- its slot holds the pivot),
    // and a row a > j updates columns <= j (M) and >= a (G).  Two rows per
    // pass, loads before stores, so the shared-memory latencies overlap.
    double vj[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int b = lane + 32 * u;
      vj[u] = b == j ? 1.0 : (b < l ? rowj[b] : 0.0);
    }
    for (int a0 = j + 1 + warp; a0 < l; a0 += 2 * nw) {
      const int a1 = a0 + nw;
      const bool two = a1 < l;
      double* row0 = gs + a0 * ls;
      double* row1 = gs + (two ? a1 : a0) * ls;
      const double f0 = rowj[a0] * ip, f1 = two ? rowj[a1] * ip : 0.0;
      double v0[4], v1[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int b = lane + 32 * u;
        v0[u] = (b <= j || (b >= a0 && b < l)) ? row0[b] : 0.0;
        v1[u] = (two && (b <= j || (b >= a1 && b < l))) ? row1[b] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int b = lane + 32 * u;
        if (b <= j || (b >= a0 && b < l)) row0[b] = fma(-f0, vj[u], v0[u]);
        if (two && (b <= j || (b >= a1 && b < l))) row1[b] = fma(-f1, vj[u], v1[u]);
      }
    }
    __syncthreads();
  }
  for (int j = tid; j < l; j += nt) rdi[j] = 1.0 / sqrt(gs[j * ls + j]);
  __syncthreads();
  for (int e = tid; e < l * l; e += nt) {
    const int c = e / l, i = e - c * l;  // consecutive threads walk row c of M
    if (i > c) continue;
    const double v = i == c ? rdi[c] : gs[c * ls + i] * rdi[c];
    rinv[i * lp + c] = (float)v;
    rinv64[i * lp + c] = v;
  }
}

// Householder QR with the reference's semantics (qr.cpp:10-75), fp64, one
// CTA; runs only when the Cholesky path flagged the input.
__global__ void __launch_bounds__(1024) householder_kernel(const float* __restrict__ y,
                                                           int64_t rows, int l, int lp,
                                                           double* __restrict__ w,
                                                           double* __restrict__ v,
                                                           float* __restrict__ q,
                                                           const int* __restrict__ flag) {
  if (*flag == 0) return;
  __shared__ double red[32];
  __shared__ unsigned char skip[128];
  const int tid = threadIdx.x, nt = blockDim.x;
  double s = 0.0;
  for (int64_t e = tid; e < rows * l; e += nt) {
    const double t = y[(e / l) * lp + e % l];
    w[e] = t;
    v[e] = 0.0;
    s += t * t;
  }
  const double floor_ = 1e-12 * sqrt(block_sum(s, red));
  for (int j = 0; j < l; ++j) {
    s = 0.0;
    for (int64_t i = j + tid; i < rows; i += nt) s += w[i * l + j] * w[i * l + j];
    const double normx = sqrt(block_sum(s, red));
    if (normx < floor_) {
      for (int64_t i = j + tid; i < rows; i += nt) w[i * l + j] = 0.0;
      if (tid == 0) skip[j] = 1;
      __syncthreads();
      continue;
    }
    if (tid == 0) skip[j] = 0;
    const double wjj = w[(int64_t)j * l + j];
    const double alpha = wjj >= 0.0 ? -normx : normx;
    s = 0.0;
    for (int64_t i = j + tid; i < rows; i += nt) {
      const double t = w[i * l + j] - (i == j ? alpha : 0.0);
      v[i * l + j] = t;
      s += t * t;
    }
    const double vn = sqrt(block_sum(s, red));
    for (int64_t i = j + tid; i < rows; i += nt) v[i * l + j] /= vn;
    __syncthreads();
    for (int c = j; c < l; ++c) {
      s = 0.0;
      for (int64_t i = j + tid; i < rows; i += nt) s += v[i * l + j] * w[i * l + c];
      const double proj = 2.0 * block_sum(s, red);
      for (int64_t i = j + tid; i < rows; i += nt) w[i * l + c] -= proj * v[i * l + j];
      __syncthreads();
    }
  }
  // Q = H_0 ... H_{l-1} applied to the identity slice (reverse order).
  for (int64_t e = tid; e < rows * l; e += nt) w[e] = ((e / l) == (e % l)) ? 1.0 : 0.0;
  __syncthreads();
  for (int jj = l - 1; jj >= 0; --jj) {
    if (skip[jj]) continue;
    for (int c = 0; c < l; ++c) {
      s = 0.0;
      for (int64_t i = jj + tid; i < rows; i += nt) s += v[i * l + jj] * w[i * l + c];
      const double proj = 2.0 * block_sum(s, red);
      for (int64_t i = jj + tid; i < rows; i += nt) w[i * l + c] -= proj * v[i * l + jj];
      __syncthreads();
    }
  }
  for (int64_t e = tid; e < rows * lp; e += nt) {
    const int64_t r = e / lp;
    const int c = (int)(e % lp);
    q[e] = c < l ? (float)w[r * l + c] : 0.f;
  }
}

// Column signs s that turn an orthonormal factor M with positive R diagonal
// (CholeskyQR2's) into the reference's Householder factor M diag(s)
// (qr.cpp:35: alpha_j = -sign(w_jj) |x_j|, R_jj = alpha_j).  Householder's
// Q depends only on the nested column spans of its input (right-multiplying
// by any nonsingular upper-triangular T rescales each step's column by T_jj
// and leaves every reflector I - 2 v v^T unchanged), so Q_house(Y) =
// Q_house(M) = M diag(s).  For orthonormal M the reduced columns stay unit
// and mutually orthogonal, so each step touches only the top l x l block:
// w = T_jj, alpha = -sign(w), |v|^2 = 2 (1 + |w|), and for c > j
// T_rc += 2 alpha T_jc (T_rj - alpha delta_rj) / |v|^2.  One CTA, fp64.
__global__ void __launch_bounds__(256) householder_signs_kernel(const float* __restrict__ q, int l,
                                                                int lp, float* __restrict__ sgn) {
  extern __shared__ double hs_t[];
  double* coef = hs_t + l * l;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < l * l; e += nt) hs_t[e] = q[(e / l) * lp + e % l];
  __syncthreads();
  for (int j = 0; j < l; ++j) {
    const double w = hs_t[j * l + j];
    const double alpha = w >= 0.0 ? -1.0 : 1.0;
    const double inv = 1.0 / (2.0 * (1.0 + fabs(w)));
    for (int c = j + 1 + tid; c < l; c += nt) coef[c] = 2.0 * alpha * hs_t[j * l + c] * inv;
    if (tid == 0) sgn[j] = (float)alpha;
    __syncthreads();
    const int m = l - j - 1;
    for (int e = tid; e < (l - j) * m; e += nt) {
      const int r = j + e / m, c = j + 1 + e % m;
      hs_t[r * l + c] += coef[c] * (hs_t[r * l + j] - (r == j ? alpha : 0.0));
    }
    __syncthreads();
  }
}

__global__ void scale_cols_kernel(float* __restrict__ q, int64_t rows, int l, int lp,
                                  const float* __restrict__ sgn) {
  const int64_t total = rows * lp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % lp);
    if (c < l) q[e] *= sgn[c];
  }
}

void gram(const float* y, int64_t rows, int l, int lp, const QrWs& w, int nsm,
          cudaStream_t st) {
  const int grid = gram_grid(rows, nsm);
  const size_t smem = sizeof(float) * kGramRows * (lp + 4);
  note_launches(1);
  gram_kernel<<<grid, 256, smem, st>>>(y, rows, l, lp, w.part);
  note_launches(1);
  gram_reduce_kernel<<<(lp * lp + 7) / 8, 256, 0, st>>>(w.part, grid, l, lp, w.g);
}


// Q = Y R^-1 in fp64 on the FP64 tensor cores (m8n8k4 DMMA): Y fp32 (rows x
// lp, widened exactly), R^-1 fp64 (lp x lp, upper triangular, zero padded)
// staged in shared memory, Q rounded to fp32 once.  CholeskyQR's R^-1 spans
// the sketch's condition number (~1e4-1e5 at C3), so the products' rounding
// is amplified by it in the small singular directions of Y: through the
// 3xTF32 X-stream kernel (fp32 R^-1, ~1e-6 relative error) the range finder's
// basis missed the reference's span by up to 1e-3 at C3 and the FastHALS-RP
// trajectory by 5e-4 (tools/proj_swap.py: fp64 projectors with the device's
// own compressed views track the reference within 8e-6).
// One warp per 8-row tile, all column tiles in registers (lp <= 128).
template <typename In, typename Out>
__global__ void __launch_bounds__(256) apply_rinv64_kernel(const In* __restrict__ y,
                                                           int64_t rows, int l, int lp,
                                                           const double* __restrict__ rinv,
                                                           Out* __restrict__ q) {
  extern __shared__ double rs[];  // lp x (lp + 4)
  const int rsd = lp + 4;
  for (int e = threadIdx.x; e < lp * lp; e += blockDim.x) rs[(e / lp) * rsd + e % lp] = rinv[e];
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  const int nct = (l + 7) >> 3;
  const int64_t ntiles = (rows + 7) / 8;
  for (int64_t tI = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); tI < ntiles;
       tI += (int64_t)gridDim.x * 8) {
    const int64_t r = tI * 8 + g;
    const In* yr = y + (r < rows ? r : 0) * lp + t4;
    double acc[16][2];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll 4
    for (int kk = 0; kk < l; kk += 4) {
      const double a = (kk + t4 < lp && r < rows) ? (double)__ldg(yr + kk) : 0.0;
      const double* bp = rs + (kk + t4) * rsd + g;
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < nct && j * 8 + 8 > kk) {  // R^-1 is upper triangular: tiles left of kk are zero
          const double b = bp[j * 8];
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(acc[j][0]), "+d"(acc[j][1])
                       : "d"(a), "d"(b));
        }
    }
    if (r < rows) {
      Out* qr_ = q + r * lp;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int c = j * 8 + 2 * t4;
        if (c < lp) {
          qr_[c] = c < l ? (Out)acc[j][0] : (Out)0;
          if (c + 1 < lp) qr_[c + 1] = c + 1 < l ? (Out)acc[j][1] : (Out)0;
        }
      }
    }
  }
}

template <typename In, typename Out>
void apply_rinv64(const In* y, int64_t rows, int l, int lp, const double* rinv64, Out* q,
                  int nsm, cudaStream_t st) {
  const int smem = (int)(sizeof(double) * lp * (lp + 4));
  static std::atomic<unsigned> attr{0u};
  smem_attr_once(attr, (const void*)(apply_rinv64_kernel<In, Out>), (int)(sizeof(double) * 128 * 132));
  const int64_t ntiles = (rows + 7) / 8;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((ntiles + 7) / 8, nsm));
  note_launches(1);
  apply_rinv64_kernel<In, Out><<<grid, 256, smem, st>>>(y, rows, l, lp, rinv64, q);
}

__global__ void f64_to_f32_kernel(const double* __restrict__ a, int64_t total, float* __restrict__ b,
                                  const int* __restrict__ only_if) {
  if (only_if && *only_if == 0) return;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x)
    b[e] = (float)a[e];
}
__global__ void f32_to_f64_kernel(const float* __restrict__ a, int64_t total, double* __restrict__ b,
                                  const int* __restrict__ only_if) {
  if (only_if && *only_if == 0) return;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x)
    b[e] = (double)a[e];
}
int conv_grid(int64_t total, int nsm) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, (int64_t)nsm * 8));
}

void chol_inv(int l, int lp, const QrWs& w, cudaStream_t st) {
  const size_t smem = sizeof(double) * (l * (l | 1) + 3 * l);
  static std::atomic<unsigned> attr{0u};
  smem_attr_once(attr, (const void*)(chol_inv_kernel), (int)(sizeof(double) * (128 * 129 + 3 * 128)));
  note_launches(1);
  chol_inv_kernel<<<1, kCholThreads, smem, st>>>(w.g, l, lp, w.rinv64, w.rinv, w.flag);
}

}  // namespace

size_t qr_ws_bytes(int64_t rows, int lp, int nsm) {
  const int grid = gram_grid(rows, nsm);
  auto r = [](size_t b) { return (b + 255) & ~size_t(255); };
  return r(sizeof(double) * grid * lp * lp) + 2 * r(sizeof(double) * lp * lp) +
         r(sizeof(float) * lp * lp) + r(sizeof(float) * rows * lp) + r(16) +
         2 * r(sizeof(double) * rows * lp) + r(sizeof(float) * xstream_ws_floats(rows, lp, lp, nsm)) +
         1024;
}

// CholeskyQR2 of a ROW-SHARDED matrix (each rank holds `rows` rows of Y):
// the fp64 Gram of the local rows is completed by the caller's in-place sum
// all-reduce across ranks (two lp x lp Gram all-reduces
// per QR); R^-1 is then identical on every rank and applied locally.  No
// Householder fallback here: *flag_out (device int) is set when a pivot
// broke down and the caller gathers Y for the replicated path.
void launch_thin_qr_dist(const float* y, int64_t rows, int l, int lp, float* q, void* ws, int nsm,
                         cudaStream_t st, const std::function<void(double*, size_t)>& allreduce_g,
                         int** flag_out, int passes) {
  const QrWs w = carve(ws, rows, lp, nsm);
  cudaMemsetAsync(w.flag, 0, sizeof(int), st);
  gram(y, rows, l, lp, w, nsm, st);
  allreduce_g(w.g, (size_t)lp * lp);
  chol_inv(l, lp, w, st);
  if (passes >= 2) {
    apply_rinv64(y, rows, l, lp, w.rinv64, w.q1, nsm, st);
    gram(w.q1, rows, l, lp, w, nsm, st);
    allreduce_g(w.g, (size_t)lp * lp);
    chol_inv(l, lp, w, st);
    apply_rinv64(w.q1, rows, l, lp, w.rinv64, q, nsm, st);
  } else {
    apply_rinv64(y, rows, l, lp, w.rinv64, q, nsm, st);
  }
  *flag_out = w.flag;
}

void launch_thin_qr(const float* y, int64_t rows, int l, int lp, float* q, void* ws, int nsm,
                    cudaStream_t st, int passes) {
  const QrWs w = carve(ws, rows, lp, nsm);
  cudaMemsetAsync(w.flag, 0, sizeof(int), st);
  gram(y, rows, l, lp, w, nsm, st);
  chol_inv(l, lp, w, st);
  if (passes >= 2) {
    apply_rinv64(y, rows, l, lp, w.rinv64, w.q1, nsm, st);
    gram(w.q1, rows, l, lp, w, nsm, st);
    chol_inv(l, lp, w, st);
    apply_rinv64(w.q1, rows, l, lp, w.rinv64, q, nsm, st);
  } else {
    apply_rinv64(y, rows, l, lp, w.rinv64, q, nsm, st);
  }
  note_launches(1);
  householder_kernel<<<1, 1024, 0, st>>>(y, rows, l, lp, w.hw, w.hv, q, w.flag);
}

// CholeskyQR(2) of an fp64 rows x lp matrix into an fp64 basis (the range
// finder's fp64 path, engine.cpp): fp64 Gram (dense.cu launch_gram_cm), the
// same Cholesky / inverse and fp64 DMMA application; on a breakdown the
// Householder kernel runs on the fp32 rounding of y (device-side flag).
size_t qr64_ws_bytes(int64_t rows, int lp, int nsm) {
  return qr_ws_bytes(rows, lp, nsm) + sizeof(double) * (gram_cm_ws_doubles(rows, lp, nsm) + 64);
}
void launch_thin_qr64(const double* y, int64_t rows, int l, int lp, double* q, void* ws, int nsm,
                      cudaStream_t st, int passes) {
  const QrWs w = carve(ws, rows, lp, nsm);
  double* gws = reinterpret_cast<double*>(static_cast<char*>(ws) + qr_ws_bytes(rows, lp, nsm));
  double* q1 = w.hw;  // rows x lp doubles (the Householder working copy when it runs)
  cudaMemsetAsync(w.flag, 0, sizeof(int), st);
  launch_gram_cm(y, rows, lp, w.g, gws, nsm, st, true);
  chol_inv(l, lp, w, st);
  if (passes >= 2) {
    apply_rinv64(y, rows, l, lp, w.rinv64, q1, nsm, st);
    launch_gram_cm(q1, rows, lp, w.g, gws, nsm, st, true);
    chol_inv(l, lp, w, st);
    apply_rinv64(q1, rows, l, lp, w.rinv64, q, nsm, st);
  } else {
    apply_rinv64(y, rows, l, lp, w.rinv64, q, nsm, st);
  }
  // breakdown (rank deficiency): Householder on fp32 y, result widened
  const int64_t total = rows * lp;
  note_launches(3);
  f64_to_f32_kernel<<<conv_grid(total, nsm), 256, 0, st>>>(y, total, w.q1, w.flag);
  householder_kernel<<<1, 1024, 0, st>>>(w.q1, rows, l, lp, w.hw, w.hv, w.xs_ws, w.flag);
  f32_to_f64_kernel<<<conv_grid(total, nsm), 256, 0, st>>>(w.xs_ws, total, q, w.flag);
}

// Condition estimate of the last CholeskyQR's input: max_j r_jj / min_j r_jj
// of its R (from R^-1's diagonal in the workspace).  Synchronises `st`.
double qr_kappa_estimate(const void* ws, int64_t rows, int l, int lp, int nsm, cudaStream_t st) {
  const QrWs w = carve(const_cast<void*>(ws), rows, lp, nsm);
  std::vector<double> dg(l);
  if (cudaMemcpy2DAsync(dg.data(), sizeof(double), w.rinv64, sizeof(double) * (lp + 1),
                        sizeof(double), l, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return 0.0;
  double mx = 0.0, mn = 1e308;
  for (double v : dg) {
    if (!(v > 0.0)) return 1e308;  // breakdown
    mx = std::max(mx, 1.0 / v);
    mn = std::min(mn, 1.0 / v);
  }
  return mx / mn;
}

// Row-sharded fp64 CholeskyQR(2): local fp64 Grams summed by allreduce_g;
// *flag_out is set on a breakdown (the caller falls back, sharded.inc).
void launch_thin_qr64_dist(const double* y, int64_t rows, int l, int lp, double* q, void* ws,
                           int nsm, cudaStream_t st,
                           const std::function<void(double*, size_t)>& allreduce_g,
                           int** flag_out, int passes) {
  const QrWs w = carve(ws, rows, lp, nsm);
  double* gws = reinterpret_cast<double*>(static_cast<char*>(ws) + qr_ws_bytes(rows, lp, nsm));
  double* q1 = w.hw;
  cudaMemsetAsync(w.flag, 0, sizeof(int), st);
  launch_gram_cm(y, rows, lp, w.g, gws, nsm, st, true);
  allreduce_g(w.g, (size_t)lp * lp);
  chol_inv(l, lp, w, st);
  if (passes >= 2) {
    apply_rinv64(y, rows, l, lp, w.rinv64, q1, nsm, st);
    launch_gram_cm(q1, rows, lp, w.g, gws, nsm, st, true);
    allreduce_g(w.g, (size_t)lp * lp);
    chol_inv(l, lp, w, st);
    apply_rinv64(q1, rows, l, lp, w.rinv64, q, nsm, st);
  } else {
    apply_rinv64(y, rows, l, lp, w.rinv64, q, nsm, st);
  }
  *flag_out = w.flag;
}

void launch_f64_to_f32(const double* a, int64_t total, float* b, int nsm, cudaStream_t st) {
  note_launches(1);
  f64_to_f32_kernel<<<conv_grid(total, nsm), 256, 0, st>>>(a, total, b, nullptr);
}
void launch_f32_to_f64(const float* a, int64_t total, double* b, int nsm, cudaStream_t st) {
  note_launches(1);
  f32_to_f64_kernel<<<conv_grid(total, nsm), 256, 0, st>>>(a, total, b, nullptr);
}

void launch_householder_signs(float* q, int64_t rows, int l, int lp, float* sgn, int nsm,
                              cudaStream_t st) {
  const size_t smem = sizeof(double) * (l * l + l);
  static std::atomic<unsigned> attr{0u};
  smem_attr_once(attr, (const void*)(householder_signs_kernel), (int)(sizeof(double) * (128 * 128 + 128)));
  note_launches(2);
  householder_signs_kernel<<<1, 256, smem, st>>>(q, l, lp, sgn);
  const int64_t total = rows * lp;
  const int grid = (int)std::min<int64_t>((total + 255) / 256, 4 * nsm);
  scale_cols_kernel<<<grid, 256, 0, st>>>(q, rows, l, lp, sgn);
}

}  // namespace cnmf
