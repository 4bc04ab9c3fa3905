// hals.cu -- FastHALS-RP iterations as one persistent cooperative kernel.
//
// Reference: fasthals_rp_step, proj/src/solvers.cpp:414-456 (A half 419-439,
// B half 440-455), the B update forms 480-509, and the dead-component redraw
// path 424-428 / 435 / 445-449 / 452 (reinit_column 28-31,
// refresh_cross_products 133-144, normalize_column 39-45).
//
// One CTA per SM.  CTA b owns a contiguous block of A rows and of B rows.
// Per iteration:
//   A half: g = B-check^T B-check (grid-distributed) | h = X-check B-check for
//           the CTA's rows | k sequential column updates of the CTA's A rows
//           held in shared memory, each followed by a grid-wide fp64 norm
//           (one grid barrier per column) | A-hat = L^T A (per-CTA partials,
//           fixed-order reduction).
//   B half: w = A-hat^T A-hat | p = X-hat^T A-hat and the k column updates,
//           both row-local (no barrier between columns) | zero-column check |
//           B-check = R B (partials + fixed-order reduction).
// Every cross-CTA sum is reduced in a fixed order, so the run is bitwise
// reproducible.  A dead or emptied component cannot be redrawn on the device
// (the reference draws it from the run's host Rng), so the kernel halts at
// exactly the reference's event point, records it in HaltInfo, and the host
// draws the column, uploads it and resumes (engine.cpp).
#include "common.cuh"
#include "kernels.h"

namespace cnmf {

namespace {

constexpr int kThreads = 256;
constexpr int kChunkB = 64;  // B rows per sweep chunk (4 threads per row)
constexpr double kDead = 1e-12;  // solvers.cpp:19

struct HalsArgs {
  HalsState st;
  int normalize_a;
  double alpha, beta;
  int it_begin, it_end, start_half, start_col;
  int skip_dead;       // column whose dead check is skipped once (just redrawn), or -1
  int rows_a, rows_b;  // rows per CTA
};

__host__ __device__ inline int64_t align4(int64_t v) { return (v + 3) & ~int64_t(3); }

// out(r, c) = sum_{l'} In[r, l'] * M[l', c] for r < nrows, c < k.
// In: global rows with leading dimension lp; M: shared lp x k (row-major).
template <typename Out>
__device__ void rows_times_small(const float* __restrict__ in, int nrows, int lp, int k,
                                 const float* __restrict__ M, float* stage, Out out) {
  const int lpp = lp + 1;
  const int r = threadIdx.x & 31, cg = threadIdx.x >> 5;
  for (int r0 = 0; r0 < nrows; r0 += 32) {
    __syncthreads();
    for (int e = threadIdx.x; e < 32 * lp; e += kThreads) {
      const int rr = e / lp, cc = e - rr * lp;
      stage[rr * lpp + cc] = (r0 + rr < nrows) ? in[(int64_t)(r0 + rr) * lp + cc] : 0.f;
    }
    __syncthreads();
    float acc[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) acc[t] = 0.f;
    for (int q = 0; q < lp; ++q) {
      const float xv = stage[r * lpp + q];
      const float* mrow = M + q * k;
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int c = cg + 8 * t;
        if (c < k) acc[t] = fmaf(xv, mrow[c], acc[t]);
      }
    }
    if (r0 + r < nrows) {
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int c = cg + 8 * t;
        if (c < k) out(r0 + r, c, acc[t]);
      }
    }
  }
  __syncthreads();
}

// Per-CTA partial P[l', c] = sum_r In[r, l'] * F(r, c), written as fp64 to
// part (lp x k).  Thread t owns 4x4 output blocks t, t+256, t+512, t+768.
template <typename FAcc>
__device__ void small_partial(const float* __restrict__ in, int nrows, int l, int lp, int k,
                              FAcc F, float* stage, double* __restrict__ part) {
  const int lpp = lp + 1;
  const int nbl = (l + 3) >> 2, nbc = (k + 3) >> 2, nb = nbl * nbc;
  float acc[4][16];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[t][i] = 0.f;
  for (int r0 = 0; r0 < nrows; r0 += 32) {
    __syncthreads();
    for (int e = threadIdx.x; e < 32 * lp; e += kThreads) {
      const int rr = e / lp, cc = e - rr * lp;
      stage[rr * lpp + cc] = (r0 + rr < nrows) ? in[(int64_t)(r0 + rr) * lp + cc] : 0.f;
    }
    __syncthreads();
    const int rmax = min(32, nrows - r0);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int b = threadIdx.x + kThreads * t;
      if (b >= nb) break;
      const int bl = b / nbc, bc = b - bl * nbc;
      for (int rr = 0; rr < rmax; ++rr) {
        float xi[4], fj[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) xi[i] = stage[rr * lpp + 4 * bl + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) fj[j] = (4 * bc + j < k) ? F(r0 + rr, 4 * bc + j) : 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[t][4 * i + j] = fmaf(xi[i], fj[j], acc[t][4 * i + j]);
      }
    }
  }
  for (int e = threadIdx.x; e < lp * k; e += kThreads) part[e] = 0.0;
  __syncthreads();
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int b = threadIdx.x + kThreads * t;
    if (b >= nb) break;
    const int bl = b / nbc, bc = b - bl * nbc;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int li = 4 * bl + i, cj = 4 * bc + j;
        if (li < l && cj < k) part[li * k + cj] = (double)acc[t][4 * i + j];
      }
  }
}

// Fixed-order sum of the grid's per-CTA partials into dst (lp x k).
__device__ void reduce_partials(const double* __restrict__ part, int G, int n_el,
                                double* __restrict__ dst) {
  const int gt = blockIdx.x * kThreads + threadIdx.x, gs = gridDim.x * kThreads;
  for (int e = gt; e < n_el; e += gs) {
    double s = 0.0;
    for (int b = 0; b < G; ++b) s += part[(int64_t)b * n_el + e];
    dst[e] = s;
  }
}

// gram[a*k+b] = sum_{l' < l} M[l'*k+a] * M[l'*k+b], fp64, grid-distributed.
__device__ void gram_small(const double* __restrict__ M, int l, int k, double* __restrict__ gram) {
  const int gt = blockIdx.x * kThreads + threadIdx.x, gs = gridDim.x * kThreads;
  for (int e = gt; e < k * k; e += gs) {
    const int a = e / k, b = e - a * k;
    double s = 0.0;
    for (int q = 0; q < l; ++q) s += M[q * k + a] * M[q * k + b];
    gram[e] = s;
  }
}

__global__ void __launch_bounds__(kThreads, 1) hals_kernel(const HalsArgs p) {
  extern __shared__ __align__(16) float smem[];
  __shared__ double red[kThreads / 32];
  __shared__ double s_total;
  __shared__ int zf[128];

  const HalsState& S = p.st;
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
  const int k = S.k, lp = S.lp, l = S.l, kp1 = k + 1, lpp = lp + 1;
  const int64_t d = S.d, n = S.n;
  const int64_t a_lo = min(d, (int64_t)cta * p.rows_a), a_hi = min(d, a_lo + p.rows_a);
  const int64_t b_lo = min(n, (int64_t)cta * p.rows_b), b_hi = min(n, b_lo + p.rows_b);
  const int na = (int)(a_hi - a_lo), nbr = (int)(b_hi - b_lo);
  const int nel = lp * k;

  // A-half shared layout
  float* As = smem;                                       // rows_a x kp1
  float* U = As + align4((int64_t)p.rows_a * kp1);        // max(lp*k, k*k)
  float* stageA = U + align4(max(lp * k, k * k));         // 32 x lpp
  // B-half shared layout
  float* Ah = smem;                                       // lp x k
  float* Ws = Ah + align4(lp * k);                        // k x k
  float* Bs = Ws + align4(k * k);                         // kChunkB x kp1
  float* stageB = Bs + align4(kChunkB * kp1);             // 32 x (max(lpp, kp1))

  int half = p.start_half, col0 = p.start_col, skip = p.skip_dead;
  for (int it = p.it_begin; it < p.it_end; ++it) {
    if (half == 0) {
      // ---- A half: g, h, sweep, A-hat --------------------------------
      gram_small(S.bchk, l, k, S.g);
      grid_barrier(S.bar, G);
      for (int e = tid; e < lp * k; e += kThreads) U[e] = (float)S.bchk[e];
      for (int e = tid; e < na * k; e += kThreads) {
        const int c = e / na, r = e - c * na;
        As[r * kp1 + c] = S.a[(int64_t)c * d + a_lo + r];
      }
      __syncthreads();
      rows_times_small(S.xc + a_lo * lp, na, lp, k, U, stageA,
                       [&](int r, int c, float v) { S.h[(int64_t)c * d + a_lo + r] = v; });
      for (int e = tid; e < k * k; e += kThreads) U[e] = (float)S.g[e];
      int jd = k;
      // solvers.cpp:424 checks g_jj once per column; a column redrawn for
      // this check is not re-checked (the reference uses `if`, not `while`).
      for (int j = col0; j < k; ++j)
        if (j != skip && S.g[j * k + j] < kDead) { jd = j; break; }
      skip = -1;
      __syncthreads();
      const int q = tid & 3, rsub = tid >> 2;
      for (int j = col0; j < jd; ++j) {
        const float gjj = (float)S.g[j * k + j];
        double nrm = 0.0;
        for (int r0 = 0; r0 < na; r0 += kThreads / 4) {
          const int r = r0 + rsub;
          float s = 0.f;
          if (r < na)
            for (int c = q; c < k; c += 4) s = fmaf(As[r * kp1 + c], U[c * k + j], s);
          s += __shfl_xor_sync(0xffffffffu, s, 1);
          s += __shfl_xor_sync(0xffffffffu, s, 2);
          if (r < na && q == 0) {
            float v = As[r * kp1 + j] + (S.h[(int64_t)j * d + a_lo + r] - s) / gjj;
            v = v > 0.f ? v : 0.f;
            As[r * kp1 + j] = v;
            nrm += (double)v * (double)v;
          }
        }
        const double cta_nrm = block_sum(nrm, red);
        if (tid == 0) S.npart[(int64_t)j * G + cta] = cta_nrm;
        grid_barrier(S.bar, G);
        if (tid == 0) {
          double t = 0.0;
          for (int b = 0; b < G; ++b) t += S.npart[(int64_t)j * G + b];
          s_total = t;
        }
        __syncthreads();
        const double total = s_total;
        if (total == 0.0) {  // column emptied: host redraws a_j (solvers.cpp:435)
          for (int e = tid; e < na * k; e += kThreads) {
            const int c = e / na, r = e - c * na;
            S.a[(int64_t)c * d + a_lo + r] = As[r * kp1 + c];
          }
          if (cta == 0 && tid == 0) *S.halt = HaltInfo{1, it + 1, 0, j, kEvZeroA, {0, 0, 0}};
          return;
        }
        if (p.normalize_a) {
          const float nv = (float)sqrt(total);
          for (int r = tid; r < na; r += kThreads) As[r * kp1 + j] = As[r * kp1 + j] / nv;
        }
        __syncthreads();
      }
      for (int e = tid; e < na * k; e += kThreads) {
        const int c = e / na, r = e - c * na;
        S.a[(int64_t)c * d + a_lo + r] = As[r * kp1 + c];
      }
      if (jd < k) {  // dead B column: host redraws b_jd (solvers.cpp:424-428)
        if (cta == 0 && tid == 0) *S.halt = HaltInfo{1, it + 1, 0, jd, kEvDeadB, {0, 0, 0}};
        return;
      }
      small_partial(S.lm + a_lo * lp, na, l, lp, k,
                    [&](int r, int c) { return As[r * kp1 + c]; }, stageA,
                    S.part + (int64_t)cta * nel);
      grid_barrier(S.bar, G);
      reduce_partials(S.part, G, nel, S.ahat);
      grid_barrier(S.bar, G);
      half = 1;
      col0 = 0;
    }
    // ---- B half: w, p, sweep, zero check, B-check ------------------------
    gram_small(S.ahat, l, k, S.w);
    grid_barrier(S.bar, G);
    for (int e = tid; e < lp * k; e += kThreads) Ah[e] = (float)S.ahat[e];
    for (int e = tid; e < k * k; e += kThreads) Ws[e] = (float)S.w[e];
    if (tid < 128) zf[tid] = 0;
    int jd = k;
    for (int j = col0; j < k; ++j)
      if (j != skip && S.w[j * k + j] < kDead) { jd = j; break; }
    skip = -1;
    __syncthreads();
    const bool constrained = !(p.alpha == 0.0 && p.beta == 0.0);
    const float alpha = (float)p.alpha, beta = (float)p.beta;
    for (int c0 = 0; c0 < nbr; c0 += kChunkB) {
      const int nr = min(kChunkB, nbr - c0);
      __syncthreads();
      for (int e = tid; e < nr * k; e += kThreads) {
        const int c = e / nr, r = e - c * nr;
        const int64_t gi = (int64_t)c * n + b_lo + c0 + r;
        const float v = S.b[gi];
        Bs[r * kp1 + c] = v;
        S.bold[gi] = v;
      }
      // p rows for this chunk, written into the stage tail as [r][c] (kp1 stride)
      float* Ps = stageB + 32 * max(lpp, kp1);
      rows_times_small(S.xht + (b_lo + c0) * lp, nr, lp, k, Ah, stageB,
                       [&](int r, int c, float v) { Ps[r * kp1 + c] = v; });
      const int q = tid & 3, r = tid >> 2;
      for (int j = col0; j < jd; ++j) {
        const float wjj = Ws[j * k + j];
        float s = 0.f;
        if (r < nr)
          for (int c = q; c < k; c += 4) s = fmaf(Bs[r * kp1 + c], Ws[c * k + j], s);
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        if (r < nr && q == 0) {
          const float bij = Bs[r * kp1 + j], pij = Ps[r * kp1 + j];
          float v = constrained ? (bij * wjj + pij - s - alpha) / (wjj + beta)
                                : bij + (pij - s) / wjj;
          v = v > 0.f ? v : 0.f;
          Bs[r * kp1 + j] = v;
          if (v != 0.f) zf[j] = 1;
        }
        __syncwarp();
      }
      __syncthreads();
      for (int e = tid; e < nr * k; e += kThreads) {
        const int c = e / nr, rr = e - c * nr;
        S.b[(int64_t)c * n + b_lo + c0 + rr] = Bs[rr * kp1 + c];
      }
    }
    __syncthreads();
    if (tid < k) S.zflag[(int64_t)cta * k + tid] = zf[tid];
    grid_barrier(S.bar, G);
    int j0 = k;
    for (int j = col0; j < jd; ++j) {
      int any = 0;
      for (int b = 0; b < G && !any; ++b) any = S.zflag[(int64_t)b * k + j];
      if (!any) { j0 = j; break; }
    }
    if (j0 < jd) {  // b_j0 emptied: roll later columns back, host redraws (solvers.cpp:452)
      for (int c = j0 + 1; c < jd; ++c)
        for (int r = tid; r < nbr; r += kThreads) {
          const int64_t gi = (int64_t)c * n + b_lo + r;
          S.b[gi] = S.bold[gi];
        }
      if (cta == 0 && tid == 0) *S.halt = HaltInfo{1, it + 1, 1, j0, kEvZeroB, {0, 0, 0}};
      return;
    }
    if (jd < k) {  // dead A column: host redraws a_jd (solvers.cpp:445-449)
      if (cta == 0 && tid == 0) *S.halt = HaltInfo{1, it + 1, 1, jd, kEvDeadA, {0, 0, 0}};
      return;
    }
    {
      float* Fs = stageB + 32 * max(lpp, kp1);  // 32 x kp1 staged B rows
      const int nbl = (l + 3) >> 2, nbc = (k + 3) >> 2, nb = nbl * nbc;
      float acc[4][16];
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[t][i] = 0.f;
      for (int r0 = 0; r0 < nbr; r0 += 32) {
        const int rmax = min(32, nbr - r0);
        __syncthreads();
        for (int e = tid; e < 32 * lp; e += kThreads) {
          const int rr = e / lp, cc = e - rr * lp;
          stageB[rr * lpp + cc] = rr < rmax ? S.rt[(b_lo + r0 + rr) * lp + cc] : 0.f;
        }
        for (int e = tid; e < 32 * k; e += kThreads) {
          const int c = e >> 5, rr = e & 31;
          Fs[rr * kp1 + c] = rr < rmax ? S.b[(int64_t)c * n + b_lo + r0 + rr] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int b = tid + kThreads * t;
          if (b >= nb) break;
          const int bl = b / nbc, bc = b - bl * nbc;
          for (int rr = 0; rr < rmax; ++rr) {
            float xi[4], fj[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) xi[i] = stageB[rr * lpp + 4 * bl + i];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
              fj[jj] = (4 * bc + jj < k) ? Fs[rr * kp1 + 4 * bc + jj] : 0.f;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int jj = 0; jj < 4; ++jj)
                acc[t][4 * i + jj] = fmaf(xi[i], fj[jj], acc[t][4 * i + jj]);
          }
        }
      }
      double* part = S.part + (int64_t)cta * nel;
      for (int e = tid; e < nel; e += kThreads) part[e] = 0.0;
      __syncthreads();
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int b = tid + kThreads * t;
        if (b >= nb) break;
        const int bl = b / nbc, bc = b - bl * nbc;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const int li = 4 * bl + i, cj = 4 * bc + jj;
            if (li < l && cj < k) part[li * k + cj] = (double)acc[t][4 * i + jj];
          }
      }
    }
    grid_barrier(S.bar, G);
    reduce_partials(S.part, G, nel, S.bchk);
    grid_barrier(S.bar, G);
    half = 0;
    col0 = 0;
  }
  if (cta == 0 && tid == 0) *S.halt = HaltInfo{0, p.it_end, 0, 0, 0, {0, 0, 0}};
}

size_t hals_smem_bytes(const HalsState& st, int rows_a) {
  const int k = st.k, lp = st.lp, kp1 = k + 1, lpp = lp + 1;
  const int64_t a_half = align4((int64_t)rows_a * kp1) + align4(std::max(lp * k, k * k)) +
                         32 * lpp;
  const int64_t b_half = align4(lp * k) + align4(k * k) + align4(kChunkB * kp1) +
                         32 * std::max(lpp, kp1) + 32 * kp1 + (int64_t)kChunkB * kp1;
  return (size_t)std::max(a_half, b_half) * sizeof(float);
}

// Column-wise compress_factor_a / compress_factor_b (compression.cpp:90-96):
// one CTA per (l', c) output, fixed-order fp64 sum over the rows.
__global__ void compress_factor_kernel(const float* __restrict__ basis, int64_t rows, int lp,
                                       const float* __restrict__ f_cm, int k, int column,
                                       int l, double* __restrict__ out) {
  __shared__ double red[32];
  const int li = blockIdx.x;
  const int c = column >= 0 ? column : blockIdx.y;
  double s = 0.0;
  if (li < l)
    for (int64_t i = threadIdx.x; i < rows; i += blockDim.x)
      s += (double)basis[i * lp + li] * (double)f_cm[(int64_t)c * rows + i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) out[li * k + c] = li < l ? s : 0.0;
}

__global__ void normalize_column_kernel(float* __restrict__ a_cm, int64_t d, int j) {
  __shared__ double red[32];
  float* col = a_cm + (int64_t)j * d;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < d; i += blockDim.x) s += (double)col[i] * (double)col[i];
  s = block_sum(s, red);
  if (s == 0.0) return;
  const float nv = (float)sqrt(s);
  for (int64_t i = threadIdx.x; i < d; i += blockDim.x) col[i] = col[i] / nv;
}

}  // namespace

size_t hals_part_doubles(int grid, int lp, int k) { return (size_t)grid * lp * k; }

static int rows_per_cta(int64_t rows, int grid) { return (int)((rows + grid - 1) / grid); }

int hals_grid(const HalsState& st, int nsm) {
  // Fewest CTAs that still cover the rows with a shared-memory A block; at
  // small sizes fewer CTAs make the per-column grid barrier cheaper.
  int grid = (int)std::min<int64_t>(nsm, std::max<int64_t>(1, (st.d + 127) / 128));
  grid = std::max(grid, (int)std::min<int64_t>(nsm, (st.n + 255) / 256));
  while (grid < nsm && hals_smem_bytes(st, rows_per_cta(st.d, grid)) > 220 * 1024) ++grid;
  return grid;
}

cudaError_t launch_hals(const HalsState& st, int normalize_a, double alpha, double beta,
                        int it_begin, int it_end, int start_half, int start_col, int skip_dead,
                        int grid, cudaStream_t s) {
  HalsArgs a;
  a.st = st;
  a.normalize_a = normalize_a;
  a.alpha = alpha;
  a.beta = beta;
  a.it_begin = it_begin;
  a.it_end = it_end;
  a.start_half = start_half;
  a.start_col = start_col;
  a.skip_dead = skip_dead;
  a.rows_a = rows_per_cta(st.d, grid);
  a.rows_b = rows_per_cta(st.n, grid);
  const size_t smem = hals_smem_bytes(st, a.rows_a);
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  cudaError_t e =
      cudaFuncSetAttribute(hals_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  void* args[] = {&a};
  note_launches(1);
  return cudaLaunchCooperativeKernel((const void*)hals_kernel, dim3(grid), dim3(kThreads), args,
                                     smem, s);
}

void launch_compress_factors(const HalsState& st, int which, int column, cudaStream_t s) {
  const dim3 grid(st.lp, column >= 0 ? 1 : st.k);
  note_launches(1);
  if (which == 0)
    compress_factor_kernel<<<grid, 256, 0, s>>>(st.lm, st.d, st.lp, st.a, st.k, column, st.l,
                                                st.ahat);
  else
    compress_factor_kernel<<<grid, 256, 0, s>>>(st.rt, st.n, st.lp, st.b, st.k, column, st.l,
                                                st.bchk);
}

void launch_normalize_column(float* a_cm, int64_t d, int j, cudaStream_t s) {
  note_launches(1);
  normalize_column_kernel<<<1, 1024, 0, s>>>(a_cm, d, j);
}

}  // namespace cnmf
