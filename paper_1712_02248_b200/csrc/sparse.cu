// sparse.cu -- CSR input for every solver.
//
// Reference: SparseMatrix (proj/include/cnmf/matrix.hpp:34-44), its products
// matmul(SparseMatrix, DenseMatrix) (proj/src/matrix.cpp:156-189), the
// sparse reconstruction error (proj/src/metrics.cpp:79-102) and
// run(SparseMatrix, ...) (proj/src/solvers.cpp:515-517): run_impl is the same
// template, so only the X contractions, check_data, ||X||^2 and the
// objective differ from the dense path.
//
// X is held as CSR (row offsets int64, column indices int32, fp32 values)
// plus the CSR of X^T built once on the host, so both orientations are
// row-gather products with no atomics: out[r][:] = sum_p v_p S[col_p][:],
// one warp per output row, nonzeros in ascending order, fp64 accumulation --
// bitwise reproducible.  The gathered S rows (n x lp or d x lp) stay in L2.
#include "common.cuh"
#include "kernels.h"

namespace cnmf {

namespace {

template <typename SIn, typename Out>
__global__ void __launch_bounds__(256) csr_spmm_kernel(const int64_t* __restrict__ rp,
                                                       const int32_t* __restrict__ ci,
                                                       const float* __restrict__ v, int64_t rows,
                                                       const SIn* __restrict__ s, int lds, int l,
                                                       Out* __restrict__ out, int ldo,
                                                       const int* __restrict__ halt) {
  if (halt && *(volatile const int*)halt) return;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < rows; r += nwarps) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    const int64_t p0 = rp[r], p1 = rp[r + 1];
    for (int64_t base = p0; base < p1; base += 32) {
      // the warp loads 32 nonzeros at once, then walks them in order
      const int64_t pe = base + lane;
      const int32_t cl = pe < p1 ? __ldg(ci + pe) : 0;
      const float vl = pe < p1 ? __ldg(v + pe) : 0.f;
      const int cnt = (int)(p1 - base < 32 ? p1 - base : 32);
      for (int t = 0; t < cnt; ++t) {
        const int32_t col = __shfl_sync(0xffffffffu, cl, t);
        const double val = (double)__shfl_sync(0xffffffffu, vl, t);
        const SIn* srow = s + (int64_t)col * lds;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = lane + 32 * u;
          if (c < l) acc[u] = fma(val, (double)__ldg(srow + c), acc[u]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = lane + 32 * u;
      if (c < ldo) out[r * ldo + c] = c < l ? (Out)acc[u] : (Out)0;
    }
  }
}

// Per-row cross term sum_p v_p (a_r . b_col_p) of the sparse objective
// (metrics.cpp:84-93), a warp per row, then block partials in a fixed order.
__global__ void __launch_bounds__(256) csr_cross_kernel(const int64_t* __restrict__ rp,
                                                        const int32_t* __restrict__ ci,
                                                        const float* __restrict__ v, int64_t d,
                                                        int64_t n, const double* __restrict__ a_cm,
                                                        const double* __restrict__ b_cm, int k,
                                                        double* __restrict__ part) {
  __shared__ double wsum[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double mine = 0.0;  // lane 0 of each warp: its rows' cross terms, rows ascending
  for (int64_t r = blockIdx.x * 8 + w; r < d; r += (int64_t)gridDim.x * 8) {
    double row = 0.0;  // nonzeros of the row in lane-strided order, then a fixed butterfly
    for (int64_t p = rp[r] + lane; p < rp[r + 1]; p += 32) {
      const int64_t col = ci[p];
      double pred = 0.0;
      for (int c = 0; c < k; ++c) pred = fma(a_cm[(int64_t)c * d + r], b_cm[(int64_t)c * n + col], pred);
      row = fma((double)v[p], pred, row);
    }
    row = warp_sum(row);
    if (lane == 0) mine += row;
  }
  if (lane == 0) wsum[w] = mine;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < 8; ++i) t += wsum[i];
    part[blockIdx.x] = t;
  }
}

// check_data on the stored values (solvers.cpp:47-52) and ||X||^2
__global__ void __launch_bounds__(256) csr_check_kernel(const float* __restrict__ v, int64_t nnz,
                                                        int* __restrict__ flag,
                                                        double* __restrict__ part) {
  __shared__ double red[32];
  double s = 0.0;
  bool bad = false;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nnz;
       p += (int64_t)gridDim.x * blockDim.x) {
    const float x = v[p];
    if (!(x >= 0.f) || !isfinite(x)) bad = true;
    s = fma((double)x, (double)x, s);
  }
  if (bad) atomicOr(flag, 1);
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void sum_parts_kernel(const double* __restrict__ part, int count, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) s += part[i];  // fixed strided order
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

// 0.5 |X|^2 - cross + 0.5 trace((A^T A)(B^T B)), clamped at zero (metrics.cpp:95-101)
__global__ void sparse_objective_kernel(const double* __restrict__ xnorm,
                                        const double* __restrict__ cross_part, int ncross,
                                        const double* __restrict__ ata,
                                        const double* __restrict__ btb, int k,
                                        double* __restrict__ out) {
  __shared__ double red[32];
  double cr = 0.0;
  for (int i = threadIdx.x; i < ncross; i += blockDim.x) cr += cross_part[i];
  cr = block_sum(cr, red);
  double q = 0.0;
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    const int r = e / k, c = e - r * k;
    q = fma(ata[r * k + c], btb[c * k + r], q);
  }
  q = block_sum(q, red);
  if (threadIdx.x == 0) {
    const double err = 0.5 * *xnorm - cr + 0.5 * q;
    *out = err > 0.0 ? err : 0.0;
  }
}

int spmm_grid(int64_t rows, int nsm) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((rows + 7) / 8, 16 * (int64_t)nsm));
}

}  // namespace

void launch_csr_spmm_f32(const CsrView& x, bool transpose, const float* s, int lds, int l,
                         float* out, int ldo, int nsm, cudaStream_t st) {
  const int64_t* rp = transpose ? x.t_rp : x.rp;
  const int32_t* ci = transpose ? x.t_ci : x.ci;
  const float* v = transpose ? x.t_v : x.v;
  const int64_t rows = transpose ? x.n : x.d;
  note_launches(1);
  csr_spmm_kernel<float, float><<<spmm_grid(rows, nsm), 256, 0, st>>>(rp, ci, v, rows, s, lds, l,
                                                                     out, ldo, nullptr);
}

void launch_csr_spmm_f64(const CsrView& x, bool transpose, const double* s, int lds, int l,
                         double* out, int ldo, int nsm, cudaStream_t st, const int* halt) {
  const int64_t* rp = transpose ? x.t_rp : x.rp;
  const int32_t* ci = transpose ? x.t_ci : x.ci;
  const float* v = transpose ? x.t_v : x.v;
  const int64_t rows = transpose ? x.n : x.d;
  note_launches(1);
  csr_spmm_kernel<double, double><<<spmm_grid(rows, nsm), 256, 0, st>>>(rp, ci, v, rows, s, lds,
                                                                       l, out, ldo, halt);
}

size_t csr_metrics_ws_doubles(int nsm) { return (size_t)16 * nsm + 8; }

void launch_csr_check(const CsrView& x, int* flag, double* norm_sq, double* ws, int nsm,
                      cudaStream_t st) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((x.nnz + 255) / 256, 4 * (int64_t)nsm));
  note_launches(2);
  csr_check_kernel<<<grid, 256, 0, st>>>(x.v, x.nnz, flag, ws);
  sum_parts_kernel<<<1, 256, 0, st>>>(ws, grid, norm_sq);
}

void launch_csr_objective(const CsrView& x, const double* a_cm, const double* b_cm, int k,
                          const double* xnorm, const double* ata, const double* btb, double* out,
                          double* ws, int nsm, cudaStream_t st) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((x.d + 7) / 8, 16 * (int64_t)nsm));
  note_launches(2);
  csr_cross_kernel<<<grid, 256, 0, st>>>(x.rp, x.ci, x.v, x.d, x.n, a_cm, b_cm, k, ws);
  sparse_objective_kernel<<<1, 256, 0, st>>>(xnorm, ws, grid, ata, btb, k, out);
}

}  // namespace cnmf
