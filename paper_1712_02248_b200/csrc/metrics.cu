// metrics.cu -- objective, input scan, Gini and layout helpers.
//
// Reference: reconstruction_error dense form (proj/src/metrics.cpp:61-77,
// 1/2 sum (x_ij - a_i . b_j)^2, direct residual); check_data
// (proj/src/solvers.cpp:47-52); gini (metrics.cpp:104-121).
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"
#include "kernels.h"

namespace cnmf {

namespace {

constexpr int kTile = 64;

// One warp per row (lanes over the row's float4 chunks): the check_data flag
// (solvers.cpp:47-52), ||X||^2 partials per block, and -- when rexp is given
// -- the row's exponent for the X-stream kernel's fp16 path (row max scaled
// into [2^14, 2^15)) plus `wide` when a row's smallest nonzero magnitude is
// below 2^-30 of its max.  One read of X serves the validation and the
// scaling.  inexact |= 1 when some element is not exactly a tf32 value (the
// X-stream kernel's two-product mode needs every element exact).
__global__ void __launch_bounds__(256) check_data_kernel(const float* __restrict__ x, int64_t ldx,
                                                         int64_t d, int64_t n,
                                                         int* __restrict__ flag,
                                                         double* __restrict__ part,
                                                         int8_t* __restrict__ rexp,
                                                         int* __restrict__ wide,
                                                         int* __restrict__ inexact,
                                                         int* __restrict__ nonint) {
  __shared__ double red[8];
  double s = 0.0;
  int bad = 0;
  unsigned low = 0u;
  int frac = 0;  // some element is not an integer below 2^26 (the int8-sliced contractions
                 // take such an X unscaled: xstream_i8.cu)
  const int lane = threadIdx.x & 31;
  const int64_t n4 = (n + 3) / 4;
  const bool vec = (ldx % 4) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < d; i += warps) {
    const float* row = x + i * ldx;
    float mx = 0.f, mn = INFINITY;
    for (int64_t c = lane; c < n4; c += 32) {
      const int64_t j = 4 * c;
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      if (vec && j + 3 < n) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(row + j));
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
      } else {
        for (int q = 0; q < 4 && j + q < n; ++q) v[q] = __ldg(row + j + q);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (!(v[q] >= 0.f) || !isfinite(v[q])) bad = 1;
        low |= __float_as_uint(v[q]);
        frac |= (v[q] != truncf(v[q])) ? 1 : 0;  // (the magnitude bounds: from mx, per row)
        s += (double)v[q] * (double)v[q];
        mx = fmaxf(mx, v[q]);
        if (v[q] > 0.f) mn = fminf(mn, v[q]);
      }
    }
    frac |= !(mx < 67108864.f) ? 1 : 0;  // this lane's elements of the row
    frac |= !(mx < 8192.f) ? 2 : 0;
    if (rexp) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      }
      if (lane == 0) {
        int e = 0;
        if (mx > 0.f && isfinite(mx)) {
          frexpf(mx, &e);
          e = max(-126, min(126, 15 - e));
        }
        rexp[i] = (int8_t)e;
        if (mx > 0.f && mn < mx * 0x1.0p-30f) atomicOr(wide, 1);
      }
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) *flag = 1;
  if (__syncthreads_or((low & 0x1FFFu) != 0u) && threadIdx.x == 0 && inexact) *inexact = 1;
  // bit 0: some element is not an integer below 2^26; bit 1: some element >= 8192
  if (nonint) {
    const int f1 = __syncthreads_or(frac & 1), f2 = __syncthreads_or(frac & 2);
    if (threadIdx.x == 0 && (f1 || f2)) atomicOr(nonint, (f1 ? 1 : 0) | (f2 ? 2 : 0));
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void sum_partials_kernel(const double* __restrict__ part, int count,
                                    double* __restrict__ out, double scale) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < count; ++i) s += part[i];
    *out = scale * s;
  }
}

// 1/2 ||X - A B^T||^2: CTA c takes 64x64 tiles c, c+G, ...; fp32 dot
// products over k, fp64 residual squares, fixed-order reductions.
__global__ void __launch_bounds__(256) recon_error_kernel(const float* __restrict__ x, int64_t ldx,
                                                          int64_t d, int64_t n,
                                                          const double* __restrict__ a_cm,
                                                          const double* __restrict__ b_cm, int k,
                                                          double* __restrict__ part) {
  extern __shared__ __align__(16) float sm[];
  float* As = sm;              // k x 64
  float* Bs = sm + k * kTile;  // k x 64
  __shared__ double red[8];
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const int64_t tr = (d + kTile - 1) / kTile, tc = (n + kTile - 1) / kTile;
  double s = 0.0;
  for (int64_t t = blockIdx.x; t < tr * tc; t += gridDim.x) {
    const int64_t i0 = (t / tc) * kTile, j0 = (t % tc) * kTile;
    __syncthreads();
    for (int e = tid; e < k * kTile; e += 256) {
      const int c = e >> 6, r = e & 63;
      As[e] = (i0 + r < d) ? (float)a_cm[(int64_t)c * d + i0 + r] : 0.f;
      Bs[e] = (j0 + r < n) ? (float)b_cm[(int64_t)c * n + j0 + r] : 0.f;
    }
    __syncthreads();
    float pred[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) pred[i][j] = 0.f;
    for (int c = 0; c < k; ++c) {
      const float4 a = *reinterpret_cast<const float4*>(As + c * kTile + ty * 4);
      float b[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[c * kTile + tx + 16 * j];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        pred[0][j] = fmaf(a.x, b[j], pred[0][j]);
        pred[1][j] = fmaf(a.y, b[j], pred[1][j]);
        pred[2][j] = fmaf(a.z, b[j], pred[2][j]);
        pred[3][j] = fmaf(a.w, b[j], pred[3][j]);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t gi = i0 + ty * 4 + i;
      if (gi >= d) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t gj = j0 + tx + 16 * j;
        if (gj < n) {
          const double diff = (double)__ldg(x + gi * ldx + gj) - (double)pred[i][j];
          s = fma(diff, diff, s);
        }
      }
    }
  }
  s = block_sum(s, red);
  if (tid == 0) part[blockIdx.x] = s;
}

__global__ void gini_partial_kernel(const double* __restrict__ sorted,
                                    const double* __restrict__ orig, int64_t count,
                                    double* __restrict__ part) {
  __shared__ double red[8];
  double acc = 0.0, tot = 0.0;
  const double m = (double)count;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    acc += (2.0 * (double)(i + 1) - m - 1.0) * sorted[i];
    tot += orig[i];
  }
  acc = block_sum(acc, red);
  tot = block_sum(tot, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = acc;
    part[2 * blockIdx.x + 1] = tot;
  }
}

__global__ void gini_final_kernel(const double* __restrict__ part, int nb, int64_t count,
                                  double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double acc = 0.0, tot = 0.0;
  for (int i = 0; i < nb; ++i) {
    acc += part[2 * i];
    tot += part[2 * i + 1];
  }
  // metrics.cpp:104-121; an all-zero B has no coefficient (NaN in run()).
  *out = (tot == 0.0 || count == 0) ? __longlong_as_double(0x7ff8000000000000LL)
                                    : acc / ((double)count * tot);
}

__global__ void cm_to_rm_kernel(const double* __restrict__ cm, int64_t rows, int k,
                                float* __restrict__ rm) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * k;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / k;
    const int c = (int)(e - i * k);
    rm[e] = (float)cm[(int64_t)c * rows + i];
  }
}

__global__ void rm_to_cm_kernel(const float* __restrict__ rm, int64_t rows, int k,
                                double* __restrict__ cm) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * k;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / rows, i = e - c * rows;
    cm[e] = rm[i * k + c];
  }
}

__global__ void pad_cols_kernel(const float* __restrict__ src, int64_t rows, int l,
                                float* __restrict__ dst, int lp) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * lp;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / lp;
    const int c = (int)(e - r * lp);
    dst[e] = c < l ? src[r * l + c] : 0.f;
  }
}

__global__ void unpad_cols_kernel(const float* __restrict__ src, int64_t rows, int lp,
                                  float* __restrict__ dst, int l) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * l;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / l;
    const int c = (int)(e - r * l);
    dst[e] = src[r * lp + c];
  }
}

__global__ void transpose_kernel(const float* __restrict__ src, int64_t rows, int64_t cols,
                                 int64_t lds, float* __restrict__ dst, int64_t ldd) {
  __shared__ float t[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    t[i][threadIdx.x] = (r < rows && c < cols) ? src[r * lds + c] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (c < cols && r < rows) dst[c * ldd + r] = t[threadIdx.x][i];
  }
}

int blocks_for(int64_t work, int nsm) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, (int64_t)nsm * 8));
}

}  // namespace

static unsigned long long g_launches = 0;
void note_launches(int n) { __atomic_fetch_add(&g_launches, (unsigned long long)n, __ATOMIC_RELAXED); }
uint64_t launch_count() { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

size_t metrics_ws_bytes(int64_t, int64_t, int nsm) { return sizeof(double) * (nsm * 16 + 64); }

void launch_check_data(const float* x, int64_t ldx, int64_t d, int64_t n, int* flag,
                       double* norm_sq, void* ws, int nsm, cudaStream_t st, int8_t* rexp,
                       int* wide, int* inexact, int* nonint) {
  const int grid = nsm * 4;
  double* part = static_cast<double*>(ws);
  note_launches(1);
  check_data_kernel<<<grid, 256, 0, st>>>(x, ldx, d, n, flag, part, rexp, wide, inexact, nonint);
  note_launches(1);
  sum_partials_kernel<<<1, 32, 0, st>>>(part, grid, norm_sq, 1.0);
}

void launch_recon_error(const float* x, int64_t ldx, int64_t d, int64_t n, const double* a_cm,
                        const double* b_cm, int k, double* out, void* ws, int nsm,
                        cudaStream_t st) {
  const int64_t tiles = ((d + kTile - 1) / kTile) * ((n + kTile - 1) / kTile);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)nsm * 4));
  const size_t smem = sizeof(float) * 2 * k * kTile;
  static std::atomic<unsigned> attr{0u};
  smem_attr_once(attr, (const void*)(recon_error_kernel), (int)(sizeof(float) * 2 * 128 * kTile));
  double* part = static_cast<double*>(ws);
  note_launches(1);
  recon_error_kernel<<<grid, 256, smem, st>>>(x, ldx, d, n, a_cm, b_cm, k, part);
  note_launches(1);
  sum_partials_kernel<<<1, 32, 0, st>>>(part, grid, out, 0.5);
}

size_t gini_ws_bytes(int64_t count) {
  size_t temp = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, temp, (const double*)nullptr, (double*)nullptr,
                                 (int)count);
  return temp + sizeof(double) * count + sizeof(double) * 2 * 1024 + 1024;
}

void launch_gini(const double* b_cm, int64_t count, double* out, void* ws, size_t ws_bytes,
                 cudaStream_t st) {
  char* p = static_cast<char*>(ws);
  double* part = reinterpret_cast<double*>(p);
  double* sorted = reinterpret_cast<double*>(p + sizeof(double) * 2 * 1024);
  char* temp = p + sizeof(double) * 2 * 1024 + ((sizeof(double) * count + 255) & ~size_t(255));
  size_t temp_bytes = ws_bytes - (size_t)(temp - p);
  cub::DeviceRadixSort::SortKeys(temp, temp_bytes, b_cm, sorted, (int)count, 0, 64, st);
  const int nb = (int)std::min<int64_t>(1024, std::max<int64_t>(1, (count + 255) / 256));
  note_launches(1);
  gini_partial_kernel<<<nb, 256, 0, st>>>(sorted, b_cm, count, part);
  note_launches(1);
  gini_final_kernel<<<1, 32, 0, st>>>(part, nb, count, out);
}

void launch_cm_to_rm(const double* cm, int64_t rows, int k, float* rm, cudaStream_t st) {
  note_launches(1);
  cm_to_rm_kernel<<<blocks_for(rows * k, 148), 256, 0, st>>>(cm, rows, k, rm);
}
void launch_rm_to_cm(const float* rm, int64_t rows, int k, double* cm, cudaStream_t st) {
  note_launches(1);
  rm_to_cm_kernel<<<blocks_for(rows * k, 148), 256, 0, st>>>(rm, rows, k, cm);
}
void launch_pad_cols(const float* src, int64_t rows, int l, float* dst, int lp, cudaStream_t st) {
  note_launches(1);
  pad_cols_kernel<<<blocks_for(rows * lp, 148), 256, 0, st>>>(src, rows, l, dst, lp);
}
void launch_unpad_cols(const float* src, int64_t rows, int lp, float* dst, int l,
                       cudaStream_t st) {
  note_launches(1);
  unpad_cols_kernel<<<blocks_for(rows * l, 148), 256, 0, st>>>(src, rows, lp, dst, l);
}
void launch_transpose(const float* src, int64_t rows, int64_t cols, int64_t lds, float* dst,
                      int64_t ldd, cudaStream_t st) {
  const dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
  note_launches(1);
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(src, rows, cols, lds, dst, ldd);
}

}  // namespace cnmf
