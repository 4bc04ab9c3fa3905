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
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "hals_common.cuh"
#include "kernels.h"

namespace cnmf {

namespace {

using namespace hals_detail;
constexpr int kNB = 8;        // columns per block of the blocked sweeps
constexpr int kRB = 3;        // B rows per thread per pass of the B sweep
// A rows per thread: the A sweep keeps its rows' block state in registers
// across the per-column grid all-reduces, so the kernel is instantiated for
// up to 3 (rows per CTA <= 768) or 6 (<= 1536) rows per thread.
constexpr int kMaxRPTLarge = 6;
constexpr double kDead = 1e-12;  // solvers.cpp:19

// Precision.  The HALS state (A, B, h = X-check B-check, p = X-hat^T A-hat,
// A-hat, B-check, g, w) is fp64 like the reference's; only the compressed
// views and projectors (X-check, X-hat^T, L, R^T) are fp32.  Measured on the
// C2 configuration: the trajectory passes through a locally unstable stretch
// (iterations ~5-20) that amplifies per-iteration rounding ~5x per
// iteration, so fp32 state or fp32 accumulation moves it by 1e-4 while fp64
// state keeps it at the compression's 1e-6.  fp32 operands are converted
// once when staged (F2F.F64.F32 issues at 1/4 the DFMA rate,
// tools/ubench_fp64.cu).

struct HalsArgs {
  HalsState st;
  int normalize_a;
  double alpha, beta;
  int it_begin, it_end, start_half, start_col;
  int skip_dead;       // column whose dead check is skipped once (just redrawn), or -1
  int products_valid;  // the first half's products (h, g or p, w) are current (ZeroA / ZeroB resume)
  int rows_a, rows_b;  // rows per CTA
  int a_dmma;          // A-sweep block products on the DMMA path (shared memory permitting)
  unsigned long long epoch0;
};

// ---- streamed products ----------------------------------------------------
// The row products (rows_times_small) and the partials (small_partial)
// stream the CTA's rows of an fp32 matrix (ld lp) through 3-deep cp.async
// rings and multiply on the FP64 tensor cores (m8n8k4 DMMA, fp32 operands
// widened in registers); see each routine for its warp tiling.
constexpr int kSR = 64;                 // rows per stage



// FP64 tensor-core MMA, D (8 x 8) += A (8 x 4, row) B (4 x 8, col): lane
// (g = lane / 4, t = lane % 4) supplies A[g][t] and B[t][g] and holds
// D[g][2t], D[g][2t + 1] (tools/ubench_dmma.cu: 37 TFLOP/s, the DFMA rate,
// from two operand registers per 256 FMAs instead of shared-memory-bound
// register tiles).
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
// 16-byte global -> shared copy; src_bytes = 0 zero-fills the destination
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src), "r"(src_bytes)
               : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// out(r, c) = sum_{q < kdim} In[r, q] M[q, c] (fp64) for r < nrows, c < k.
// M: shared fp64 (lp x k).  The fp32 rows stream through a ring of kRing raw
// 64-row stages filled by cp.async (several stages in flight per SM: the
// one-stage register prefetch left the phase latency-bound far below both
// HBM and DMMA rates), row stride lp + 4 floats (conflict-free A fragments).
// On the FP64 tensor cores: a warp item is two 8-column tiles of M times 4 of
// the stage's 8 row tiles (eight accumulator chains; each A fragment is
// widened from fp32 once and used for both column tiles; at k = 50 the 8
// items cover the 8 warps in one round).
constexpr int kRing = 3;
__host__ __device__ constexpr int rts_stage_floats(int lp) { return kSR * (lp + 4); }
template <typename Out>
__device__ void rows_times_small(const float* __restrict__ in, int nrows, int lp, int kdim, int k,
                                 const double* __restrict__ M, float* ring, Out out) {
  const int lps = lp + 4, sfl = rts_stage_floats(lp);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int nct = (k + 7) >> 3, nqs = (kdim + 3) >> 2;
  const int ncp = (nct + 1) >> 1;  // column-tile pairs
  const int nitems = 2 * ncp;      // (column-tile pair, row-tile half)
  const int nst = (nrows + kSR - 1) / kSR;
  const int q4 = lp >> 2, nchunk = kSR * q4;
  auto issue = [&](int st) {  // always commits a group (empty past the end)
    if (st < nst) {
      float* dst = ring + (st % kRing) * sfl;
      const int r0 = st * kSR;
      for (int e = threadIdx.x; e < nchunk; e += kThreads) {
        const int rr = e / q4, c4 = e - rr * q4;
        const bool ok = r0 + rr < nrows;
        cp_async16(dst + rr * lps + 4 * c4, in + (int64_t)(ok ? r0 + rr : 0) * lp + 4 * c4, ok ? 16 : 0);
      }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int i = 0; i < kRing - 1; ++i) issue(i);
  for (int st = 0; st < nst; ++st) {
    cp_async_wait<kRing - 2>();  // this thread's copies of stage st have landed
    __syncthreads();             // everyone's have; the slot refilled below is free
    issue(st + kRing - 1);
    const float* stg = ring + (st % kRing) * sfl;
    const int r0 = st * kSR;
    for (int it = warp; it < nitems; it += kThreads / 32) {
      const int cp = it >> 1, rh = it & 1;
      // this lane's B-fragment columns in the pair's two tiles
      const int cb0 = cp * 16 + g, cb1 = cb0 + 8;
      const bool bok0 = cb0 < k, bok1 = cb1 < k;
      const double* bp0 = M + t4 * k + (bok0 ? cb0 : 0);
      const double* bp1 = M + t4 * k + (bok1 ? cb1 : 0);
      double acc[2][4][2];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[h][i][0] = acc[h][i][1] = 0.0;
      const float* a0 = stg + (rh * 32 + g) * lps + t4;
#pragma unroll 2
      for (int qs = 0; qs < nqs; ++qs) {
        const double b0 = bok0 ? bp0[4 * qs * k] : 0.0;
        const double b1 = bok1 ? bp1[4 * qs * k] : 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double av = (double)a0[i * 8 * lps + 4 * qs];  // widened once, used twice
          dmma(acc[0][i][0], acc[0][i][1], av, b0);
          dmma(acc[1][i][0], acc[1][i][1], av, b1);
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c0 = cp * 16 + h * 8 + 2 * t4;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = r0 + rh * 32 + i * 8 + g;
          if (r < nrows) {
            if (c0 < k) out(r, c0, acc[h][i][0]);
            if (c0 + 1 < k) out(r, c0 + 1, acc[h][i][1]);
          }
        }
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();
}

// Per-CTA partial P[l', c] = sum_r In[r, l'] * F[c][row0 + r] (fp64, rows in
// ascending order) into part (global lp x k, rows >= l zero).  In: fp32 rows
// (ld lp), register-prefetched like rows_times_small; F: column-major fp64
// state (ld ldf), copied by cp.async into a double-buffered row-major stage
// (fst: 2 x kSR x (k + 1)).  8 x 8 output tiles on the FP64 tensor cores
// (dmma), up to 8 per warp accumulating in registers across all stages
// (several passes when l x k needs more tiles than that).

// Stages of the partial products: kSRP rows of the fp32 input (row stride
// lps_partial: A-fragment reads conflict-free) and of the column-major fp64
// factor (per column kSRP + 4 doubles), kRing deep, both filled by cp.async.
constexpr int kSRP = 32;
constexpr int kFS = kSRP + 4;
__host__ __device__ constexpr int lps_partial(int lp) { return lp + (8 - lp % 32 + 32) % 32; }
__host__ __device__ constexpr int64_t partial_stage_bytes(int lp, int k) {
  return (int64_t)kSRP * lps_partial(lp) * 4 + (int64_t)k * kFS * 8;
}

template <int kTPW>  // 8 x 8 output tiles per warp per pass over the rows
__device__ __noinline__ void small_partial_t(const float* __restrict__ in, int nrows, int l, int lp, int k,
                                const double* __restrict__ F, int64_t ldf, double* ringd,
                                double* __restrict__ part) {
  const int lps = lps_partial(lp);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int nlt = (l + 7) >> 3, nct = (k + 7) >> 3, ntile = nlt * nct;
  const int nst = (nrows + kSRP - 1) / kSRP;
  const int q4 = lp >> 2, nchunk = kSRP * q4;
  const int64_t sbytes = partial_stage_bytes(lp, k);
  char* ring = reinterpret_cast<char*>(ringd);
  auto xst = [&](int st) { return reinterpret_cast<float*>(ring + (st % kRing) * sbytes); };
  auto fst = [&](int st) {
    return reinterpret_cast<double*>(ring + (st % kRing) * sbytes + (int64_t)kSRP * lps * 4);
  };
  auto issue = [&](int st) {  // always commits a group (empty past the end)
    if (st < nst) {
      const int r0 = st * kSRP;
      float* xd = xst(st);
      for (int e = threadIdx.x; e < nchunk; e += kThreads) {
        const int rr = e / q4, c4 = e - rr * q4;
        const bool ok = r0 + rr < nrows;
        cp_async16(xd + rr * lps + 4 * c4, in + (int64_t)(ok ? r0 + rr : 0) * lp + 4 * c4, ok ? 16 : 0);
      }
      double* fd = fst(st);
      for (int e = threadIdx.x; e < kSRP * k; e += kThreads) {  // coalesced along each column
        const int c = e / kSRP, rr = e - c * kSRP;
        if (r0 + rr < nrows) cp_async8(fd + c * kFS + rr, F + (int64_t)c * ldf + r0 + rr);
        else fd[c * kFS + rr] = 0.0;
      }
    }
    cp_async_commit();
  };
  for (int p0 = 0; p0 < ntile; p0 += kTPW * (kThreads / 32)) {
    double acc[kTPW][2];
    // per-tile fragment offsets, computed once per pass (an integer division
    // per tile per stage showed up as 3% of the C4 kernel's stall samples)
    int xoff[kTPW], foff[kTPW];
#pragma unroll
    for (int u = 0; u < kTPW; ++u) {
      acc[u][0] = acc[u][1] = 0.0;
      const int tI = p0 + warp + (kThreads / 32) * u;
      const int l0 = (tI / nct) * 8, c0 = (tI % nct) * 8;
      xoff[u] = t4 * lps + l0 + g;
      foff[u] = c0 + g < k ? (c0 + g) * kFS + t4 : -1;
    }
    __syncthreads();  // previous users of the ring are done
#pragma unroll
    for (int i = 0; i < kRing - 1; ++i) issue(i);
    for (int st = 0; st < nst; ++st) {
      cp_async_wait<kRing - 2>();
      __syncthreads();  // stage st visible to all; the slot refilled below is free
      issue(st + kRing - 1);
      const float* xs = xst(st);
      const double* fs = fst(st);
      // stages are zero-filled past nrows: a fixed trip count
#pragma unroll
      for (int u = 0; u < kTPW; ++u) {
        const int tI = p0 + warp + (kThreads / 32) * u;
        if (tI >= ntile) break;  // warp-uniform
        const bool bok = foff[u] >= 0;
        const float* xa = xs + xoff[u];
        const double* fb = fs + (bok ? foff[u] : t4);
#pragma unroll
        for (int rs = 0; rs < kSRP; rs += 4) {
          const double av = (double)xa[rs * lps];      // A[g][t] = In[rs + t][l0 + g]
          const double bv = bok ? fb[rs] : 0.0;        // B[t][g] = F[rs + t][c0 + g]
          dmma(acc[u][0], acc[u][1], av, bv);
        }
      }
    }
    cp_async_wait<0>();
#pragma unroll
    for (int u = 0; u < kTPW; ++u) {
      const int tI = p0 + warp + (kThreads / 32) * u;
      if (tI >= ntile) break;
      const int li = (tI / nct) * 8 + g, c = (tI % nct) * 8 + 2 * t4;
      if (li < l) {
        if (c < k) part[li * k + c] = acc[u][0];
        if (c + 1 < k) part[li * k + c + 1] = acc[u][1];
      }
    }
  }
  for (int e = l * k + threadIdx.x; e < lp * k; e += kThreads) part[e] = 0.0;
  __syncthreads();
}

// Register-blocked variant: the 8 warps form a wl x wc grid over the l x k
// tile grid, each warp owning a BL x BC block of 8 x 8 output tiles for the
// whole row stream.  Per k-step a warp loads BL A fragments (fp32 -> fp64)
// and BC B fragments for BL * BC DMMAs (C4: 4 x 7 tiles, 11 shared loads per
// 28 DMMAs; the one-tile-per-item form above needed two loads per DMMA and
// was shared-memory bound: short-scoreboard stalls on its fragment loads were
// the C4 kernel's second hottest lines).  One pass over the rows for any
// l, k <= 128.
template <int BL, int BC>
__device__ __noinline__ void small_partial_blk(const float* __restrict__ in, int nrows, int l,
                                               int lp, int k, const double* __restrict__ F,
                                               int64_t ldf, double* ringd, double* __restrict__ part,
                                               int wc) {
  const int lps = lps_partial(lp);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int nlt = (l + 7) >> 3, nct = (k + 7) >> 3;
  const int wi = warp / wc, wj = warp - wi * wc;
  const int lt0 = wi * BL, ct0 = wj * BC;
  const int nst = (nrows + kSRP - 1) / kSRP;
  const int q4 = lp >> 2, nchunk = kSRP * q4;
  const int64_t sbytes = partial_stage_bytes(lp, k);
  char* ring = reinterpret_cast<char*>(ringd);
  auto xst = [&](int st) { return reinterpret_cast<float*>(ring + (st % kRing) * sbytes); };
  auto fst = [&](int st) {
    return reinterpret_cast<double*>(ring + (st % kRing) * sbytes + (int64_t)kSRP * lps * 4);
  };
  auto issue = [&](int st) {  // always commits a group (empty past the end)
    if (st < nst) {
      const int r0 = st * kSRP;
      float* xd = xst(st);
      for (int e = threadIdx.x; e < nchunk; e += kThreads) {
        const int rr = e / q4, c4 = e - rr * q4;
        const bool ok = r0 + rr < nrows;
        cp_async16(xd + rr * lps + 4 * c4, in + (int64_t)(ok ? r0 + rr : 0) * lp + 4 * c4, ok ? 16 : 0);
      }
      double* fd = fst(st);
      for (int e = threadIdx.x; e < kSRP * k; e += kThreads) {  // coalesced along each column
        const int c = e / kSRP, rr = e - c * kSRP;
        if (r0 + rr < nrows) cp_async8(fd + c * kFS + rr, F + (int64_t)c * ldf + r0 + rr);
        else fd[c * kFS + rr] = 0.0;
      }
    }
    cp_async_commit();
  };
  // fragment offsets: A[g][t] = In[rs + t][l0 + g], B[t][g] = F[c0 + g][rs + t];
  // tiles past the grid read row/column 0 and are never stored
  int xo[BL], fo[BC];
#pragma unroll
  for (int i = 0; i < BL; ++i) {
    const int lt = lt0 + i;
    xo[i] = t4 * lps + (lt < nlt ? lt * 8 + g : 0);
  }
#pragma unroll
  for (int j = 0; j < BC; ++j) {
    const int c = (ct0 + j) * 8 + g;
    fo[j] = (c < k ? c : 0) * kFS + t4;
  }
  double acc[BL][BC][2];
#pragma unroll
  for (int i = 0; i < BL; ++i)
#pragma unroll
    for (int j = 0; j < BC; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const bool active = lt0 < nlt && ct0 < nct;  // warp-uniform
  __syncthreads();  // previous users of the ring are done
#pragma unroll
  for (int i = 0; i < kRing - 1; ++i) issue(i);
  for (int st = 0; st < nst; ++st) {
    cp_async_wait<kRing - 2>();
    __syncthreads();  // stage st visible to all; the slot refilled below is free
    issue(st + kRing - 1);
    if (!active) continue;
    const float* xs = xst(st);
    const double* fs = fst(st);
#pragma unroll 2
    for (int rs = 0; rs < kSRP; rs += 4) {
      double av[BL], bv[BC];
#pragma unroll
      for (int i = 0; i < BL; ++i) av[i] = (double)xs[xo[i] + rs * lps];
#pragma unroll
      for (int j = 0; j < BC; ++j) bv[j] = fs[fo[j] + rs];
#pragma unroll
      for (int i = 0; i < BL; ++i)
#pragma unroll
        for (int j = 0; j < BC; ++j) dmma(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
    }
  }
  cp_async_wait<0>();
  if (active) {
#pragma unroll
    for (int i = 0; i < BL; ++i)
#pragma unroll
      for (int j = 0; j < BC; ++j) {
        const int li = (lt0 + i) * 8 + g, c = (ct0 + j) * 8 + 2 * t4;
        if (lt0 + i < nlt && ct0 + j < nct && li < l) {
          if (c < k) part[li * k + c] = acc[i][j][0];
          if (c + 1 < k) part[li * k + c + 1] = acc[i][j][1];
        }
      }
  }
  for (int e = l * k + threadIdx.x; e < lp * k; e += kThreads) part[e] = 0.0;
  __syncthreads();
}

// Per-warp block shapes (BL x BC tiles) and the 8-warp grid (wl x wc) they
// imply, cheapest first by fragment loads per DMMA.
__device__ void small_partial(const float* __restrict__ in, int nrows, int l, int lp, int k,
                              const double* __restrict__ F, int64_t ldf, double* ring,
                              double* __restrict__ part) {
  const int nlt = (l + 7) >> 3, nct = (k + 7) >> 3;
  auto fits = [&](int wl, int bl, int bc) {  // wl x (8 / wl) warps of bl x bc tiles
    return (nlt + wl - 1) / wl <= bl && (nct + 8 / wl - 1) / (8 / wl) <= bc;
  };
  if (fits(4, 2, 2)) small_partial_blk<2, 2>(in, nrows, l, lp, k, F, ldf, ring, part, 2);
  else if (fits(2, 4, 2)) small_partial_blk<4, 2>(in, nrows, l, lp, k, F, ldf, ring, part, 4);
  else if (fits(4, 3, 4)) small_partial_blk<3, 4>(in, nrows, l, lp, k, F, ldf, ring, part, 2);
  else if (fits(2, 5, 2)) small_partial_blk<5, 2>(in, nrows, l, lp, k, F, ldf, ring, part, 4);
  else if (fits(4, 4, 4)) small_partial_blk<4, 4>(in, nrows, l, lp, k, F, ldf, ring, part, 2);
  else if (fits(2, 6, 4)) small_partial_blk<6, 4>(in, nrows, l, lp, k, F, ldf, ring, part, 4);
  else if (fits(4, 4, 7)) small_partial_blk<4, 7>(in, nrows, l, lp, k, F, ldf, ring, part, 2);
  else if (fits(4, 4, 8)) small_partial_blk<4, 8>(in, nrows, l, lp, k, F, ldf, ring, part, 2);
  else {
    const int ntile = nlt * nct;
    if (ntile <= 8 * (kThreads / 32))
      small_partial_t<8>(in, nrows, l, lp, k, F, ldf, ring, part);
    else
      small_partial_t<16>(in, nrows, l, lp, k, F, ldf, ring, part);
  }
}

// Block-wide staging copy dst[e] = f(e) for e < total with eight loads in
// flight per thread before any store (a plain strided loop waits one L2
// round trip per element: ~30k cycles for a 100 x 112 Gram, measured by ncu
// as the top long-scoreboard stall of the C4 kernel).
template <typename F>
__device__ __forceinline__ void stage8(double* __restrict__ dst, int total, F f) {
  for (int e0 = threadIdx.x; e0 < total; e0 += 8 * kThreads) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * kThreads;
      v[u] = e < total ? f(e) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * kThreads;
      if (e < total) dst[e] = v[u];
    }
  }
}

// Gram of a final lp x k fp64 matrix M (rows >= l are zero), fp64:
// out[a*k+b] = sum_{l'<l} M[l',a] M[l',b], into this CTA's scratch.  `st` is
// free shared memory for l4 x k8 doubles.  8 x 8 tiles of the upper triangle
// on the FP64 tensor cores (two fragment loads per DMMA), mirrored.
__device__ __noinline__ void gram_to_scratch(const double* __restrict__ M, int l, int k, double* st,
                                double* __restrict__ out) {
  const int k8 = (k + 7) & ~7, l4 = (l + 3) & ~3;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  __syncthreads();
  stage8(st, l4 * k8, [&](int e) {
    const int r = e / k8, c = e - r * k8;
    return (r < l && c < k) ? __ldcg(M + r * k + c) : 0.0;
  });
  __syncthreads();
  const int nkt = k8 >> 3, ntri = nkt * (nkt + 1) / 2, nqs = l4 >> 2;
  for (int tI = warp; tI < ntri; tI += kThreads / 32) {
    int ai = 0, rem = tI;
    while (rem >= nkt - ai) {
      rem -= nkt - ai;
      ++ai;
    }
    const int bi = ai + rem;
    double d0 = 0.0, d1 = 0.0;
    const double* pa = st + t4 * k8 + ai * 8 + g;
    const double* pb = st + t4 * k8 + bi * 8 + g;
#pragma unroll 4
    for (int qs = 0; qs < nqs; ++qs) dmma(d0, d1, pa[4 * qs * k8], pb[4 * qs * k8]);
    const int a = ai * 8 + g, c = bi * 8 + 2 * t4;
    const double v[2] = {d0, d1};
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int cc = c + j;
      if (a < k && cc < k && (ai < bi || a <= cc)) {
        out[a * k + cc] = v[j];
        out[cc * k + a] = v[j];
      }
    }
  }
  __syncthreads();
}

// g / w in shared memory: k x kg, row stride kg = k rounded up to 8 with zero
// padding, so a block's 8 coefficients of one row are two aligned 32-byte
// halves (four 16-byte vector loads, broadcast across the warp).
// Row stride of g / w in shared memory: k rounded up to 16, plus 4 (== 4 mod
// 16 doubles: the DMMA B fragments of the A-sweep block product are
// conflict-free); rows k .. k4 - 1 are zero.
__host__ __device__ constexpr int gram_stride(int k) { return ((k + 15) & ~15) + 4; }
__device__ __forceinline__ void load_gram(double* gw, const double* __restrict__ src, int k, int kg,
                                          bool cg) {
  const int k4 = (k + 3) & ~3;
  stage8(gw, k4 * kg, [&](int e) {
    const int r = e / kg, c = e - r * kg;
    return (r < k && c < k) ? (cg ? __ldcg(src + r * k + c) : src[r * k + c]) : 0.0;
  });
}

// ---- A-sweep block product on the FP64 tensor cores ---------------------
// acc(r, t) = sum_c A[r][c] g[c][jb + t] for the CTA's rows, t < 8 NT: the
// product every column block of the A sweep starts from (solvers.cpp:429,
// the running A g_j).  A is read from L2 (column-major state) as DMMA A
// fragments, g from shared memory; the results go to shared memory (row
// stride 8 NT + 1), from where each thread takes its rows.  Replaces a SIMT
// loop that re-read every A row per block with 4 loads in flight per thread
// (latency-bound: the hottest line of the C4 kernel's ncu profile).
template <int NT>
__device__ __noinline__ void a_block_dmma(const double* __restrict__ a, int64_t d, int64_t a_lo,
                                          int na, int k, const double* __restrict__ gw, int kg,
                                          int jb, double* __restrict__ accs) {
  constexpr int NBS = 8 * NT + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t4 = lane & 3;
  const int k4 = (k + 3) & ~3;
  const int npair = (na + 15) >> 4;
  for (int pI = warp; pI < npair; pI += kThreads / 32) {
    const int r0 = pI * 16, ra = r0 + g, rb = r0 + 8 + g;
    const double* pa = a + a_lo + (ra < na ? ra : 0) + (int64_t)t4 * d;
    const double* pb = a + a_lo + (rb < na ? rb : 0) + (int64_t)t4 * d;
    const double* wp = gw + t4 * kg + jb + g;
    double acc[2][NT][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int h = 0; h < NT; ++h) acc[i][h][0] = acc[i][h][1] = 0.0;
#pragma unroll 5
    for (int c = 0; c < k4; c += 4) {
      const bool okc = c + t4 < k;
      const double a0 = (okc && ra < na) ? __ldcg(pa + (int64_t)c * d) : 0.0;
      const double a1 = (okc && rb < na) ? __ldcg(pb + (int64_t)c * d) : 0.0;
#pragma unroll
      for (int h = 0; h < NT; ++h) {
        const double wv = wp[c * kg + 8 * h];
        dmma(acc[0][h][0], acc[0][h][1], a0, wv);
        dmma(acc[1][h][0], acc[1][h][1], a1, wv);
      }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int h = 0; h < NT; ++h) {
        double* dst = accs + (r0 + 8 * i + g) * NBS + 8 * h + 2 * t4;
        dst[0] = acc[i][h][0];
        dst[1] = acc[i][h][1];
      }
  }
}
// Shared memory of the DMMA A-sweep product (doubles), next to g.
__host__ __device__ constexpr int64_t a_dmma_doubles(int rows_a, int nb) {
  return (int64_t)((rows_a + 15) & ~15) * (nb + 1);
}
template <int N>
__device__ __forceinline__ void loadn(const double* p, double (&v)[N]) {
  const double2* q = reinterpret_cast<const double2*>(p);
#pragma unroll
  for (int u = 0; u < N / 2; ++u) {
    const double2 t = q[u];
    v[2 * u] = t.x;
    v[2 * u + 1] = t.y;
  }
}
__device__ __forceinline__ void load8(const double* p, double (&v)[8]) {
  const double2* q = reinterpret_cast<const double2*>(p);
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const double2 t = q[u];
    v[2 * u] = t.x;
    v[2 * u + 1] = t.y;
  }
}

// ---- B sweep on the FP64 tensor cores ------------------------------------
// The B half's column updates are row-local (solvers.cpp:444-451, the B update
// forms 480-509): every row of B runs its own k-step Gauss-Seidel chain
// against w.  Each warp takes 16-row strips of the CTA's rows in turn, stages
// the strip's k columns in shared memory (column-major, stride kBsStr), and
// sweeps it in 16-column blocks:
//   * block product acc = B_strip w[:, block] as m8n8k4 DMMAs (two 8-row x
//     two 8-column tiles, chain over all k columns with the current values:
//     columns before the block already updated, the block's own still old);
//   * in-block chain: lane (g, t4) of the accumulator layout holds row g's
//     columns {2t4, 2t4+1, 8+2t4, 9+2t4}, so column t of the block is owned
//     by lane t4 = (t % 8) / 2 of each 4-lane row group; the owner's new value
//     and delta are broadcast in the group (shuffle), and every lane folds the
//     delta into its later columns' accumulators (acc_u += delta w_ju).
// w sits in shared memory (row stride kgs = 16-padded k + 4: conflict-free
// fragments), the strip rows are read once from L2/HBM and written once.
// The SIMT sweep it replaces re-read every B row from L2 once per 16-column
// block and ran ~18% of the DFMA peak (profiles/r01_hals_c3_summary.md).
constexpr int kBsRows = 16;  // rows per warp strip
constexpr int kBsStr = 20;   // strip column stride (doubles, == 4 mod 16)
__host__ __device__ constexpr int bs_kgs(int k) { return ((k + 15) & ~15) + 4; }
__host__ __device__ constexpr int64_t bs_smem_doubles(int k) {
  return (int64_t)((k + 3) & ~3) * bs_kgs(k) + (int64_t)(kThreads / 32) * ((k + 3) & ~3) * kBsStr;
}
// Static shared memory of hals_kernel is ~2.4 KB; the DMMA sweep is used
// when its dynamic share fits next to it (k <= 100).
__host__ __device__ constexpr bool bs_dmma_fits(int k) {
  return bs_smem_doubles(k) * 8 + 4096 <= 227 * 1024;
}

template <bool kConstrained>
__device__ __noinline__ void b_sweep_dmma(const HalsState& S, const double* __restrict__ ws,
                                          const double* __restrict__ s_diag,
                                          const double* __restrict__ s_winv, double* strips,
                                          const double* __restrict__ bcur, double* __restrict__ bnxt,
                                          int64_t b_lo, int nbr, int col0, int jd, double alpha,
                                          unsigned* zmask) {
  const int k = S.k, k4 = (k + 3) & ~3, kgs = bs_kgs(k);
  const int64_t n = S.n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3, grp = lane & ~3;
  double* bs = strips + (int64_t)warp * k4 * kBsStr;
  const int nstrip = (nbr + kBsRows - 1) / kBsRows;
  for (int si = warp; si < nstrip; si += kThreads / 32) {
    const int r0 = si * kBsRows, nr = min(kBsRows, nbr - r0);
    const int64_t rbase = b_lo + r0;
    __syncwarp();  // the previous strip's write-back reads are done
    // Columns < col0 were updated by an earlier launch and carried into bcur
    // by the caller's resume convention; the rest are the old B.
    for (int e = lane; e < k4 * kBsRows; e += 32) {
      const int c = e >> 4, rr = e & 15;
      double* dst = bs + c * kBsStr + rr;
      if (c < k && rr < nr) cp_async8(dst, bcur + (int64_t)c * n + rbase + rr);
      else *dst = 0.0;
    }
    cp_async_commit();
    cp_async_wait_all();
    __syncwarp();
    unsigned zm0 = 0u, zm1 = 0u, zm2 = 0u, zm3 = 0u;  // lane 0: non-zero columns
    for (int jb = col0 & ~15; jb < jd; jb += 16) {
      const int t0 = max(col0 - jb, 0), nbj = min(16, jd - jb);
      if (t0 >= nbj) continue;
      // p of this lane's accumulator entries (issued before the chain)
      double pv[2][2][2];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int c = jb + 8 * h + 2 * t4 + e, r = 8 * i + g;
            pv[i][h][e] = (c < k && r < nr) ? __ldcg(S.p + (int64_t)c * n + rbase + r) : 0.0;
          }
      double acc[2][2][2];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int h = 0; h < 2; ++h) acc[i][h][0] = acc[i][h][1] = 0.0;
      const double* ap = bs + t4 * kBsStr + g;  // A[g][t] = B[8i + g][c + t]
      const double* wp = ws + t4 * kgs + jb + g;  // B[t][g] = w[c + t][jb + 8h + g]
#pragma unroll 5
      for (int c = 0; c < k4; c += 4) {
        const double a0 = ap[c * kBsStr], a1 = ap[c * kBsStr + 8];
        const double w0 = wp[c * kgs], w1 = wp[c * kgs + 8];
        dmma(acc[0][0][0], acc[0][0][1], a0, w0);
        dmma(acc[0][1][0], acc[0][1][1], a0, w1);
        dmma(acc[1][0][0], acc[1][0][1], a1, w0);
        dmma(acc[1][1][0], acc[1][1][1], a1, w1);
      }
      // in-block chain; bit t of nzb: this lane owns a non-zero entry of column jb + t
      unsigned nzb = 0u;
      auto chain = [&](auto full_c) {
        constexpr bool kFull = decltype(full_c)::value;  // all 16 columns, from the first
        const double* wrow = ws + jb * kgs + jb + 2 * t4;
        double2 wr0 = *reinterpret_cast<const double2*>(wrow + (kFull ? 0 : t0) * kgs);
        double2 wr1 = *reinterpret_cast<const double2*>(wrow + (kFull ? 0 : t0) * kgs + 8);
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          if constexpr (!kFull) {
            if (t < t0) continue;
            if (t >= nbj) break;
          }
          const int j = jb + t, hh = t >> 3, ee = t & 1, ow = grp | ((t & 7) >> 1);
          const bool owner = t4 == ((t & 7) >> 1);
          const double wjj = s_diag[j], winv = s_winv[j];
          // row j of w for this lane's columns; the next row is loaded while
          // this step's chain runs
          const double wv[2][2] = {{(2 * t4 > t) ? wr0.x : 0.0, (2 * t4 + 1 > t) ? wr0.y : 0.0},
                                   {(8 + 2 * t4 > t) ? wr1.x : 0.0, (9 + 2 * t4 > t) ? wr1.y : 0.0}};
          if (t + 1 < 16) {
            wr0 = *reinterpret_cast<const double2*>(wrow + (t + 1) * kgs);
            wr1 = *reinterpret_cast<const double2*>(wrow + (t + 1) * kgs + 8);
          }
          bool nz = false;
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int r = 8 * i + g;
            const double bo = bs[j * kBsStr + r];
            const double sv = acc[i][hh][ee], pp = pv[i][hh][ee];
            // solvers.cpp:480-490 (unconstrained) / 502-508 (constrained); the
            // division is a multiplication by the precomputed reciprocal
            const double v = kConstrained ? (bo * wjj + pp - sv - alpha) * winv : bo + (pp - sv) * winv;
            const double vf = v > 0.0 ? v : 0.0;
            const double dl = __shfl_sync(0xffffffffu, vf - bo, ow);
            if (owner && r < nr) {
              bs[j * kBsStr + r] = vf;
              nz |= vf != 0.0;
            }
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int e = 0; e < 2; ++e) acc[i][h][e] = fma(dl, wv[h][e], acc[i][h][e]);
          }
          nzb |= nz ? (1u << t) : 0u;
        }
      };
      if (t0 == 0 && nbj == 16) chain(std::true_type{});
      else chain(std::false_type{});
      const unsigned nzw = __reduce_or_sync(0xffffffffu, nzb) << (jb & 16);
      const int wq = jb >> 5;
      zm0 |= wq == 0 ? nzw : 0u;
      zm1 |= wq == 1 ? nzw : 0u;
      zm2 |= wq == 2 ? nzw : 0u;
      zm3 |= wq == 3 ? nzw : 0u;
    }
    if (lane == 0) {
      if (zm0) atomicOr(&zmask[0], zm0);
      if (zm1) atomicOr(&zmask[1], zm1);
      if (zm2) atomicOr(&zmask[2], zm2);
      if (zm3) atomicOr(&zmask[3], zm3);
    }
    __syncwarp();
    for (int e = lane; e < k * kBsRows; e += 32) {
      const int c = e >> 4, rr = e & 15;
      if (rr < nr) bnxt[(int64_t)c * n + rbase + rr] = bs[c * kBsStr + rr];
    }
  }
}

// An emptied A column served inside the kernel (reinit_column + the norm of
// normalize_column, solvers.cpp:28-31,40-45,435-436): row i of the column
// takes the run stream's word pos + i as uniform_positive() * kReinitScale,
// written unnormalised to S.a; one norm all-reduce follows, which also carries
// "some word was a rejected draw" (uniform_positive redraws an exact zero,
// probability 2^-53 per word) as +inf.  Returns 0 when the stream's next d
// words are not on the device (nothing done), 1 when served (s_red holds the
// squared norm and its inverse root; *s_pos and S.pos advanced, S.pos[1]
// counted), 2 when a rejected draw leaves the event to the host (the
// all-reduce was run: the caller advances ep and nr for 1 and 2).
__device__ __noinline__ int serve_zero_a(const HalsState& S, int G, int cta, unsigned long long ep,
                                         unsigned long long nr, int j, int64_t a_lo, int na,
                                         unsigned long long* s_pos, double* red8, double* s_red) {
  const unsigned long long p0 = *s_pos;
  if (p0 + (unsigned long long)S.d + 64ULL > S.nwords) return 0;
  double n2 = 0.0;
  bool bad = false;
  for (int r = threadIdx.x; r < na; r += kThreads) {
    const double u = (double)(__ldcg(S.words + p0 + (unsigned long long)(a_lo + r)) >> 11) * 0x1.0p-53;
    bad |= u == 0.0;
    const double v = u * 1e-3;  // kReinitScale
    S.a[(int64_t)j * S.d + a_lo + r] = v;
    n2 = fma(v, v, n2);
  }
  const double tot = allreduce_fused(S, G, cta, ep, nr, bad ? INFINITY : n2, red8, s_red);
  if (!(tot < INFINITY)) return 2;
  if (threadIdx.x == 0) {
    *s_pos = p0 + (unsigned long long)S.d;
    if (cta == 0) {
      S.pos[0] = p0 + (unsigned long long)S.d;
      S.pos[1] += 1ULL;
    }
  }
  return 1;
}

// RPT: A rows per thread; NB: columns per sweep block (16 halves the sweeps'
// re-reads of A and B -- one pass over all k columns per block -- where the
// registers allow it; the 6-row instance keeps 8).
// kInl: an emptied A column is served inside the kernel (serve_zero_a).  The
// call's register constraints slow the steady-state sweep by ~5%, so the host
// uses this instance only for a run's first iterations, where the events
// cluster (engine.cpp run_hals), and the plain one for the rest.
template <int RPT, int NB, bool kInl>
__global__ void __launch_bounds__(kThreads, 1) hals_kernel(const HalsArgs p) {
  extern __shared__ __align__(16) double smem[];
  __shared__ double red8[kThreads / 32];
  __shared__ double s_total;
  __shared__ unsigned zmask[4];
  __shared__ double s_diag[128];  // g_jj / w_jj (divisors and dead checks)
  __shared__ double s_ginv[128];  // 1 / g_jj (A half)
  __shared__ double s_red[2];     // norm all-reduce: total, 1/sqrt(total)
  __shared__ long long s_prof[21];
  __shared__ unsigned long long s_rng_pos;

  const HalsState& S = p.st;
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
  const int k = S.k, lp = S.lp, l = S.l, kp1 = k + 1, lpp = lp + 1, kg = gram_stride(k);
  const int64_t d = S.d, n = S.n;
  const int64_t a_lo = min(d, (int64_t)cta * p.rows_a), a_hi = min(d, a_lo + p.rows_a);
  const int64_t b_lo = min(n, (int64_t)cta * p.rows_b), b_hi = min(n, b_lo + p.rows_b);
  const int na = (int)(a_hi - a_lo), nbr = (int)(b_hi - b_lo);
  const int nel = lp * k;
  double* gsc = S.gsc + (int64_t)cta * k * k;
  double* wsc = S.wsc + (int64_t)cta * k * k;

  // shared layout: products use [M lp*k | stage 64*lpp]; sweeps use [g or w k*k];
  // partials use [stage 32*lpp | fst 32*kp1] (+ group reduction aliasing it)
  double* Ms = smem;
  float* ring64 = reinterpret_cast<float*>(smem + lp * k);  // rows_times_small stages
  double* gw = smem;

  const bool prof = S.prof != nullptr && cta == 0;
  long long t_last = 0;
  if (prof && tid == 0) {
    for (int i = 0; i < 21; ++i) s_prof[i] = 0;
    t_last = clock64();
  }
#define HALS_PROF(id)                 \
  if (prof && tid == 0) {             \
    const long long now_ = clock64(); \
    s_prof[id] += now_ - t_last;      \
    t_last = now_;                    \
  }
  if (S.dense && __ldcg(&S.halt->halted)) return;  // queued behind a halt: no-op
  unsigned long long ep = p.epoch0;
  unsigned long long nr = S.nr0;  // norm all-reduces so far (slot tags)
  // The run stream's position: read once per launch (before this CTA's first
  // grid exchange, hence before CTA 0 can have advanced it) and advanced by
  // every CTA alike at each redraw served in-kernel (serve_zero_a).
  if (tid == 0) s_rng_pos = (S.words != nullptr && !S.dense) ? __ldcg(S.pos) : 0ULL;
  bool have_g = false, have_w = false;
  // resumed after an emptied column (ZeroA / ZeroB: the redraw changed A or B
  // only, not B-check or A-hat): the halted launch's h, g (A half) or p, w
  // (B half) are still current in global memory -- skip recomputing them
  bool reuse = p.products_valid != 0;
  double* bcur = S.b;  // B as of the start of the B half
  double* bnxt = S.bold;
  int half = p.start_half, col0 = p.start_col, skip = p.skip_dead;
  const int rpt = (na + kThreads - 1) / kThreads;  // <= RPT (launch_hals)

  for (int it = p.it_begin; it < p.it_end; ++it) {
    if (half == 0) {
      // ================= A half (solvers.cpp:419-439) =====================
      if (S.dense) {  // p = X B, g = B^T B prepared by the host (solvers.cpp:154-155)
        load_gram(gw, S.gd, k, kg, true);
      } else {
        if (!reuse) {
          if (!have_g) gram_to_scratch(S.bchk, l, k, smem, gsc);
          // h = X-check B-check for this CTA's rows (solvers.cpp:421)
          stage8(Ms, lp * k, [&](int e) { return __ldcg(S.bchk + e); });
          HALS_PROF(0);
          rows_times_small(S.xc + a_lo * lp, na, lp, l, k, Ms, ring64,
                           [&](int r, int c, double v) { S.h[(int64_t)c * d + a_lo + r] = v; });
        }
        reuse = false;
        load_gram(gw, gsc, k, kg, false);
      }
      __syncthreads();
      for (int e = tid; e < k; e += kThreads) {
        s_diag[e] = gw[e * kg + e];
        s_ginv[e] = 1.0 / gw[e * kg + e];
      }
      __syncthreads();
      HALS_PROF(1);
      // solvers.cpp:424 checks g_jj once per column; a column redrawn for
      // this check is not re-checked (the reference uses `if`, not `while`).
      int jd = k;
      for (int j = col0; j < k; ++j)
        if (j != skip && s_diag[j] < kDead) { jd = j; break; }
      skip = -1;
      // Blocked column sweep (solvers.cpp:423-437).  Thread owns rows
      // tid + 256 i.  Blocks are 8-aligned columns [jb, jb + 8) (the first
      // one starts at col0 after a resume).  Per block: acc = A g[:, block]
      // with the current A; when a column is final its delta is folded into
      // the block's later accumulators (the reference's running A g_j, with
      // the same fp64 operation order as summing the deltas per column).
      // One all-reduce per column for the norm.
      for (int jb = col0 & ~(NB - 1); jb < jd; jb += NB) {
        const int t0 = max(col0 - jb, 0), nbj = min(NB, jd - jb);
        if (t0 >= nbj) continue;  // resumed at col0 == jd: nothing left in this block
        double acc[RPT][NB];
        if (p.a_dmma) {
          double* accs = smem + (int64_t)((k + 3) & ~3) * kg;
          __syncthreads();  // the previous block's A updates are written
          a_block_dmma<NB / 8>(S.a, d, a_lo, na, k, gw, kg, jb, accs);
          __syncthreads();
#pragma unroll
          for (int i = 0; i < RPT; ++i) {
            const int r = tid + kThreads * i;
            const bool ok = i < rpt && r < na;
#pragma unroll
            for (int t = 0; t < NB; ++t) acc[i][t] = ok ? accs[r * (NB + 1) + t] : 0.0;
          }
        } else {
#pragma unroll
        for (int i = 0; i < RPT; ++i)
#pragma unroll
          for (int t = 0; t < NB; ++t) acc[i][t] = 0.0;
        for (int c0 = 0; c0 < k; c0 += 4) {  // 4 columns of A in flight per row
          double av4[RPT][4];
#pragma unroll
          for (int i = 0; i < RPT; ++i) {
            const int r = tid + kThreads * i;
            const bool ok = i < rpt && r < na;
#pragma unroll
            for (int cc = 0; cc < 4; ++cc)
              av4[i][cc] = (ok && c0 + cc < k) ? __ldcg(S.a + (int64_t)(c0 + cc) * d + a_lo + r) : 0.0;
          }
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            if (c0 + cc >= k) break;
            double gv[NB];  // padded columns (>= k) are zero
            loadn<NB>(gw + (c0 + cc) * kg + jb, gv);
#pragma unroll
            for (int i = 0; i < RPT; ++i)
#pragma unroll
              for (int t = 0; t < NB; ++t) acc[i][t] = fma(av4[i][cc], gv[t], acc[i][t]);
          }
        }
        }
        double hv[RPT], av[RPT];
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          const int r = tid + kThreads * i;
          const bool ok = i < rpt && r < na;
          const int j = jb + t0;
          hv[i] = ok ? (S.dense ? __ldcg(S.hd + (a_lo + r) * lp + j)
                                : __ldcg(S.h + (int64_t)j * d + a_lo + r))
                     : 0.0;
          av[i] = ok ? __ldcg(S.a + (int64_t)j * d + a_lo + r) : 0.0;
        }
        HALS_PROF(2);
#pragma unroll
        for (int t = 0; t < NB; ++t) {
          if (t < t0) continue;
          if (t >= nbj) break;
          const int j = jb + t;
          const double ginv = s_ginv[j];
          double nrm = 0.0, vv[RPT];
#pragma unroll
          for (int i = 0; i < RPT; ++i) {
            vv[i] = 0.0;
            const int r = tid + kThreads * i;
            if (i < rpt && r < na) {  // solvers.cpp:430-434
              const double v = av[i] + (hv[i] - acc[i][t]) * ginv;
              vv[i] = v > 0.0 ? v : 0.0;
              nrm = fma(vv[i], vv[i], nrm);
            }
          }
          // prefetch the next column's h and a while the norm is reduced
          double hn[RPT], an[RPT];
#pragma unroll
          for (int i = 0; i < RPT; ++i) {
            const int r = tid + kThreads * i;
            const bool ok = i < rpt && r < na && t + 1 < nbj;
            hn[i] = ok ? (S.dense ? __ldcg(S.hd + (a_lo + r) * lp + j + 1)
                                  : __ldcg(S.h + (int64_t)(j + 1) * d + a_lo + r))
                       : 0.0;
            an[i] = ok ? __ldcg(S.a + (int64_t)(j + 1) * d + a_lo + r) : 0.0;
          }
          HALS_PROF(2);
          const double total = allreduce_fused(S, G, cta, ep, nr, nrm, red8, s_red);
          HALS_PROF(3);
          if (total == 0.0) {  // column emptied: a_j is redrawn (solvers.cpp:435)
            // served in-kernel from the run stream when possible (serve_zero_a)
            int sv = 0;
            if constexpr (kInl) {
              if (S.words != nullptr && !S.dense)
                sv = serve_zero_a(S, G, cta, ep, nr, j, a_lo, na, &s_rng_pos, red8, s_red);
            }
            if (sv != 0) {  // it ran one norm all-reduce
              ++ep;
              ++nr;
            }
            if (sv == 1) {
#pragma unroll
              for (int i = 0; i < RPT; ++i) {
                const int r = tid + kThreads * i;
                vv[i] = (i < rpt && r < na) ? __ldcg(S.a + (int64_t)j * d + a_lo + r) : 0.0;
              }
            } else {  // the host redraws a_j and relaunches at column j + 1
#pragma unroll
              for (int i = 0; i < RPT; ++i) {
                const int r = tid + kThreads * i;
                if (i < rpt && r < na) S.a[(int64_t)j * d + a_lo + r] = 0.0;
              }
              if (cta == 0 && tid == 0) {
                *S.halt = HaltInfo{1, it + 1, 0, j, kEvZeroA, bcur == S.bold, ep};
                S.halt->last_nr = nr;
              }
              return;
            }
          }
          const double inv_nrm = s_red[1];
          double gr[NB];  // row j of g: the later columns' coefficients of a_j
          loadn<NB>(gw + j * kg + jb, gr);
#pragma unroll
          for (int i = 0; i < RPT; ++i) {
            const int r = tid + kThreads * i;
            if (i < rpt && r < na) {  // solvers.cpp:436
              const double nf = p.normalize_a ? vv[i] * inv_nrm : vv[i];
              S.a[(int64_t)j * d + a_lo + r] = nf;
              const double dlt = nf - av[i];
#pragma unroll
              for (int u = 0; u < NB; ++u)
                if (u > t) acc[i][u] = fma(dlt, gr[u], acc[i][u]);
            }
            hv[i] = hn[i];
            av[i] = an[i];
          }
        }
      }
      __syncthreads();
      if (jd < k) {  // dead B column: host redraws b_jd (solvers.cpp:424-428)
        if (cta == 0 && tid == 0) {
          *S.halt = HaltInfo{1, it + 1, 0, jd, kEvDeadB, bcur == S.bold, ep};
          S.halt->last_nr = nr;
        }
        return;
      }
      if (S.dense) {  // one half per launch
        if (cta == 0 && tid == 0) {
          *S.halt = HaltInfo{0, it + 1, 0, 0, 0, bcur == S.bold, ep};
          S.halt->last_nr = nr;
          if (prof)
            for (int i = 0; i < 21; ++i) S.prof[i] += s_prof[i];
        }
        return;
      }
      // A-hat = L^T A (solvers.cpp:438): partials, exchange, slice reduce, exchange
      small_partial(S.lm + a_lo * lp, na, l, lp, k, S.a + a_lo, d, smem,
                    S.part + (int64_t)cta * nel);
      HALS_PROF(4);
      exchange_fast(S, G, ep);
      HALS_PROF(5);
      slice_reduce(S.part, G, nel, S.ahat);
      HALS_PROF(6);
      exchange_fast(S, G, ep);
      HALS_PROF(7);
      gram_to_scratch(S.ahat, l, k, smem, wsc);  // w = A-hat^T A-hat (solvers.cpp:443)
      HALS_PROF(8);
      have_w = true;
      half = 1;
      col0 = 0;
    }
    // ================== B half (solvers.cpp:440-455) =======================
    if (S.dense) {  // p = X^T A, w = A^T A prepared by the host (solvers.cpp:175-176)
      load_gram(gw, S.wd, k, kg, true);
    } else {
      if (!reuse) {
        if (!have_w) gram_to_scratch(S.ahat, l, k, smem, wsc);
        // p = X-hat^T A-hat for this CTA's rows (solvers.cpp:442)
        stage8(Ms, lp * k, [&](int e) { return __ldcg(S.ahat + e); });
        rows_times_small(S.xht + b_lo * lp, nbr, lp, l, k, Ms, ring64,
                         [&](int r, int c, double v) { S.p[(int64_t)c * n + b_lo + r] = v; });
      }
      reuse = false;
      if (!bs_dmma_fits(k)) load_gram(gw, wsc, k, kg, false);  // (the DMMA sweep stages its own)
    }
    if (tid < 4) zmask[tid] = 0u;
    __syncthreads();
    if (!S.dense && bs_dmma_fits(k))
      for (int e = tid; e < k; e += kThreads) s_diag[e] = wsc[e * k + e];
    else
      for (int e = tid; e < k; e += kThreads) s_diag[e] = gw[e * kg + e];
    __syncthreads();
    int jd = k;
    for (int j = col0; j < k; ++j)
      if (j != skip && s_diag[j] < kDead) { jd = j; break; }
    skip = -1;
    HALS_PROF(9);
    // columns before col0 were updated by an earlier launch: carry them over
    for (int c = 0; c < col0; ++c)
      for (int r = tid; r < nbr; r += kThreads)
        bnxt[(int64_t)c * n + b_lo + r] = bcur[(int64_t)c * n + b_lo + r];
    const bool constrained = !(p.alpha == 0.0 && p.beta == 0.0);
    if (!S.dense && bs_dmma_fits(k)) {
      // w in the DMMA sweep's layout (row stride kgs, rows/columns zero-padded)
      const int k4 = (k + 3) & ~3, kgs = bs_kgs(k);
      double* ws = smem;
      __syncthreads();  // everyone is done with the product stage / gw copy
      stage8(ws, k4 * kgs, [&](int e) {
        const int r = e / kgs, c = e - r * kgs;
        return (r < k && c < k) ? wsc[r * k + c] : 0.0;
      });
      for (int e = tid; e < k; e += kThreads)
        s_ginv[e] = constrained ? 1.0 / (wsc[e * k + e] + p.beta) : 1.0 / wsc[e * k + e];
      __syncthreads();
      if (constrained)
        b_sweep_dmma<true>(S, ws, s_diag, s_ginv, smem + (int64_t)k4 * kgs, bcur, bnxt, b_lo, nbr,
                           col0, jd, p.alpha, zmask);
      else
        b_sweep_dmma<false>(S, ws, s_diag, s_ginv, smem + (int64_t)k4 * kgs, bcur, bnxt, b_lo, nbr,
                            col0, jd, 0.0, zmask);
    } else {
    // Rows are independent: kRB rows per thread per pass (rows rb0 + tid +
    // 256 i), 8-aligned column blocks as in the A half, deltas folded into
    // the block's later accumulators, zero-column flags by warp ballot.
    // (RB = 1 when the CTA has at most 256 rows: no idle row slots)
    auto b_sweep = [&](auto rb_const) {
      constexpr int RB = decltype(rb_const)::value;
      for (int rb0 = 0; rb0 < nbr; rb0 += kThreads * RB) {  // CTA-uniform trip count
        int64_t gr[RB];
        bool okr[RB];
  #pragma unroll
        for (int i = 0; i < RB; ++i) {
          const int r = rb0 + tid + kThreads * i;
          okr[i] = r < nbr;
          gr[i] = b_lo + (okr[i] ? r : 0);
        }
        for (int jb = col0 & ~(NB - 1); jb < jd; jb += NB) {
          const int t0 = max(col0 - jb, 0), nbj = min(NB, jd - jb);
          if (t0 >= nbj) continue;  // resumed at col0 == jd: nothing left in this block
          const int jbe = jb + t0;  // columns < jbe already live in bnxt
          double acc[RB][NB];
  #pragma unroll
          for (int i = 0; i < RB; ++i)
  #pragma unroll
            for (int t = 0; t < NB; ++t) acc[i][t] = 0.0;
          // software-pipelined: the next 4 columns' loads are in flight while
          // the current 4 are multiplied (the loop was latency-bound)
          double bv4[RB][4], bvn[RB][4];
          auto load4 = [&](int c0, double (&dst)[RB][4]) {
  #pragma unroll
            for (int i = 0; i < RB; ++i)
  #pragma unroll
              for (int cc = 0; cc < 4; ++cc) {
                const int c = c0 + cc;
                dst[i][cc] = (okr[i] && c < k) ? __ldcg((c < jbe ? bnxt : bcur) + (int64_t)c * n + gr[i]) : 0.0;
              }
          };
          load4(0, bv4);
          for (int c0 = 0; c0 < k; c0 += 4) {
            if (c0 + 4 < k) load4(c0 + 4, bvn);
  #pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
              if (c0 + cc >= k) break;
              double gv[NB];
              loadn<NB>(gw + (c0 + cc) * kg + jb, gv);
  #pragma unroll
              for (int i = 0; i < RB; ++i)
  #pragma unroll
                for (int t = 0; t < NB; ++t) acc[i][t] = fma(bv4[i][cc], gv[t], acc[i][t]);
            }
  #pragma unroll
            for (int i = 0; i < RB; ++i)
  #pragma unroll
              for (int cc = 0; cc < 4; ++cc) bv4[i][cc] = bvn[i][cc];
          }
          // b and p of the next column are loaded one step ahead: the column
          // chain waits on arithmetic only
          double bb[RB], pb[RB];
          auto load_bp = [&](int j, double (&bo)[RB], double (&po)[RB]) {
  #pragma unroll
            for (int i = 0; i < RB; ++i) {
              const bool ok = okr[i] && j < jb + nbj;
              bo[i] = ok ? __ldcg(bcur + (int64_t)j * n + gr[i]) : 0.0;
              po[i] = ok ? (S.dense ? __ldcg(S.pd + gr[i] * lp + j) : __ldcg(S.p + (int64_t)j * n + gr[i]))
                         : 0.0;
            }
          };
          load_bp(jbe, bb, pb);
  #pragma unroll
          for (int t = 0; t < NB; ++t) {
            if (t < t0) continue;
            if (t >= nbj) break;
            const int j = jb + t;
            const double wjj = s_diag[j];
            double bn[RB], pn[RB];
            load_bp(j + 1, bn, pn);
            double grow[NB];
            loadn<NB>(gw + j * kg + jb, grow);
            bool nz = false;
  #pragma unroll
            for (int i = 0; i < RB; ++i) {
              const double s = acc[i][t];
              const double bij = bb[i];
              const double pij = pb[i];
              const double v = constrained ? (bij * wjj + pij - s - p.alpha) / (wjj + p.beta)  // 502-508
                                           : bij + (pij - s) / wjj;                            // 480-490
              const double vf = v > 0.0 ? v : 0.0;
              if (okr[i]) {
                bnxt[(int64_t)j * n + gr[i]] = vf;
                nz |= vf != 0.0;
              }
              const double dlt = vf - bij;
  #pragma unroll
              for (int u = 0; u < NB; ++u)
                if (u > t) acc[i][u] = fma(dlt, grow[u], acc[i][u]);
              bb[i] = bn[i];
              pb[i] = pn[i];
            }
            const unsigned bal = __ballot_sync(0xffffffffu, nz);
            if ((tid & 31) == 0 && bal) atomicOr(&zmask[j >> 5], 1u << (j & 31));
          }
        }
      }
    };
    if (nbr <= kThreads) b_sweep(std::integral_constant<int, 1>{});
    else b_sweep(std::integral_constant<int, kRB>{});
    }
    __syncthreads();
    HALS_PROF(10);
    if (tid < 4) S.zpart[cta * 4 + tid] = zmask[tid];
    // B-check partial = R_rows B_rows, published together with the zero flags
    if (!S.dense)
      small_partial(S.rt + b_lo * lp, nbr, l, lp, k, bnxt + b_lo, n, smem,
                    S.part + (int64_t)cta * nel);
    HALS_PROF(11);
    exchange_fast(S, G, ep);
    HALS_PROF(12);
    if (tid < 4) zmask[tid] = 0u;
    __syncthreads();
    for (int e = tid; e < G * 4; e += kThreads) {
      const unsigned v = __ldcg(S.zpart + e);
      if (v) atomicOr(&zmask[e & 3], v);
    }
    __syncthreads();
    if (S.sharded) {
      // this rank's B-check partial; the host all-reduces it with the other
      // ranks' and decides zero columns on the global mask.  bcur keeps the
      // old B for a host-side rollback.
      for (int c = jd; c < k; ++c)  // columns from a dead A column on were not reached
        for (int r = tid; r < nbr; r += kThreads) {
          const int64_t gi = (int64_t)c * n + b_lo + r;
          bnxt[gi] = bcur[gi];
        }
      slice_reduce(S.part, G, nel, S.bchk);
      exchange_fast(S, G, ep);
      if (cta == 0 && tid < 4) S.zpart[4 * G + tid] = zmask[tid];
      if (cta == 0 && tid == 0) { *S.halt = HaltInfo{1, it + 1, 1, jd, kEvShard, bnxt == S.bold, ep}; S.halt->last_nr = nr; }
      return;
    }
    int j0 = k;
    for (int j = col0; j < jd; ++j)
      if (!(zmask[j >> 5] & (1u << (j & 31)))) { j0 = j; break; }
    if (j0 < jd || jd < k) {
      // The new B lives in bnxt.  Columns after an emptied b_j0 were computed
      // against the zero column, and columns from jd on were never reached:
      // both keep their old values from bcur.
      const int from = j0 < jd ? j0 + 1 : jd;
      for (int c = from; c < k; ++c)
        for (int r = tid; r < nbr; r += kThreads) {
          const int64_t gi = (int64_t)c * n + b_lo + r;
          bnxt[gi] = bcur[gi];
        }
      if (cta == 0 && tid == 0) {
        // pad = 1 tells the host the current B is the second buffer
        *S.halt = j0 < jd ? HaltInfo{1, it + 1, 1, j0, kEvZeroB, bnxt == S.bold, ep}
                          : HaltInfo{1, it + 1, 1, jd, kEvDeadA, bnxt == S.bold, ep};
          S.halt->last_nr = nr;
      }
      return;
    }
    HALS_PROF(13);
    if (!S.dense) {
      slice_reduce(S.part, G, nel, S.bchk);
      HALS_PROF(14);
      exchange_fast(S, G, ep);
      HALS_PROF(15);
      gram_to_scratch(S.bchk, l, k, smem, gsc);  // g for the next A half (solvers.cpp:422)
      HALS_PROF(16);
      have_g = true;
    }
    double* tb = bcur;
    bcur = bnxt;
    bnxt = tb;
    half = 0;
    col0 = 0;
  }
  if (cta == 0 && tid == 0) {
    *S.halt = HaltInfo{0, p.it_end, 0, 0, 0, bcur == S.bold, ep};
    S.halt->last_nr = nr;
    if (prof)
      for (int i = 0; i < 21; ++i) S.prof[i] += s_prof[i];
  }
#undef HALS_PROF
}

// Shared memory (bytes): the max over phases.
// g plus the DMMA A-sweep product buffer (bytes), for block width nb
static size_t a_dmma_smem(const HalsState& st, int rows_a, int nb) {
  const int64_t k4 = (st.k + 3) & ~3;
  return (size_t)(k4 * gram_stride(st.k) + a_dmma_doubles(rows_a, nb)) * sizeof(double);
}
size_t hals_smem_bytes(const HalsState& st, int /*rows_a*/) {
  const int64_t k = st.k, lp = st.lp, l = st.l, kp1 = k + 1, lpp = lp + 1;
  const int64_t k4 = (k + 3) & ~3;
  const int64_t prod = lp * k + (kRing * (int64_t)rts_stage_floats((int)lp) + 1) / 2;
  const int64_t sweep = ((k + 3) & ~3) * gram_stride((int)k);
  const int64_t part = (kRing * partial_stage_bytes((int)lp, (int)k) + 7) / 8;  // cp.async ring
  const int64_t gram = ((l + 3) & ~3) * ((k + 7) & ~7);
  const int64_t bsw = (!st.dense && bs_dmma_fits((int)k)) ? bs_smem_doubles((int)k) : 0;
  return (size_t)std::max(std::max(std::max(prod, sweep), std::max(part, gram)), bsw) *
         sizeof(double);
}

// Column-wise compress_factor_a / compress_factor_b (compression.cpp:90-96):
// one CTA per (l', c) output, fixed-order fp64 sum over the rows.
__global__ void compress_factor_kernel(const float* __restrict__ basis, int64_t rows, int lp,
                                       const double* __restrict__ f_cm, int k, int column,
                                       int l, double* __restrict__ out) {
  __shared__ double red[32];
  const int li = blockIdx.x;
  const int c = column >= 0 ? column : blockIdx.y;
  double s = 0.0;
  if (li < l)
    for (int64_t i = threadIdx.x; i < rows; i += blockDim.x)
      s += (double)basis[i * lp + li] * f_cm[(int64_t)c * rows + i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) out[li * k + c] = li < l ? s : 0.0;
}

// All columns at once (run start): CTA c takes a contiguous block of rows,
// streams it in 32-row stages through shared memory (the basis rows and the
// factor's column segments, both read coalesced exactly once) and keeps a
// register tile of the lp x k output per thread -- l' = lane + 32 a, column =
// warp + 8 b: the basis values are conflict-free loads, the factor values
// warp-wide broadcasts, 4 x 16 fp64 FMAs per 20 shared loads.  Per-CTA
// partials in `part`, summed over the CTAs in a fixed order by
// compress_factor_reduce_kernel.  The one-CTA-per-output kernel above read
// the basis with stride lp once per column: 3.3 ms per factor at C4.
constexpr int kCfRows = 32, kCfA = 4, kCfB = 16;  // lp <= 128, k <= 128
__global__ void __launch_bounds__(256) compress_factor_tile_kernel(
    const float* __restrict__ basis, int64_t rows, int lp, const double* __restrict__ f_cm, int k,
    int64_t rows_per_cta, double* __restrict__ part) {
  __shared__ float bs[kCfRows][128];   // row reads / writes walk consecutive words
  __shared__ double fs[128][kCfRows];  // read as warp-wide broadcasts (48 KB static in all)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta, r1 = min(rows, r0 + rows_per_cta);
  double acc[kCfA][kCfB];
#pragma unroll
  for (int a = 0; a < kCfA; ++a)
#pragma unroll
    for (int b = 0; b < kCfB; ++b) acc[a][b] = 0.0;
  for (int64_t s0 = r0; s0 < r1; s0 += kCfRows) {
    const int nr = (int)min((int64_t)kCfRows, r1 - s0);
    __syncthreads();
    for (int e = threadIdx.x; e < kCfRows * 128; e += 256) {
      const int r = e >> 7, c = e & 127;
      bs[r][c] = (r < nr && c < lp) ? basis[(s0 + r) * lp + c] : 0.f;
    }
    for (int e = threadIdx.x; e < 128 * kCfRows; e += 256) {
      const int c = e >> 5, r = e & 31;
      fs[c][r] = (r < nr && c < k) ? f_cm[(int64_t)c * rows + s0 + r] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int r = 0; r < kCfRows; ++r) {
      double bv[kCfA];
#pragma unroll
      for (int a = 0; a < kCfA; ++a) bv[a] = (double)bs[r][lane + 32 * a];
#pragma unroll
      for (int b = 0; b < kCfB; ++b) {
        const double fv = fs[warp + 8 * b][r];
#pragma unroll
        for (int a = 0; a < kCfA; ++a) acc[a][b] = fma(bv[a], fv, acc[a][b]);
      }
    }
  }
  double* out = part + (int64_t)blockIdx.x * lp * k;
#pragma unroll
  for (int a = 0; a < kCfA; ++a)
#pragma unroll
    for (int b = 0; b < kCfB; ++b) {
      const int li = lane + 32 * a, c = warp + 8 * b;
      if (li < lp && c < k) out[li * k + c] = acc[a][b];
    }
}

__global__ void compress_factor_reduce_kernel(const double* __restrict__ part, int ctas, int lp, int k,
                                              int l, double* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= lp * k) return;
  double s = 0.0;
  for (int c = 0; c < ctas; ++c) s += part[(int64_t)c * lp * k + e];
  out[e] = e / k < l ? s : 0.0;
}

__global__ void normalize_column_kernel(double* __restrict__ a_cm, int64_t d, int j) {
  __shared__ double red[32];
  double* col = a_cm + (int64_t)j * d;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < d; i += blockDim.x) s += col[i] * col[i];
  s = block_sum(s, red);
  if (s == 0.0) return;
  const double nv = sqrt(s);
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
                        unsigned long long epoch0, int grid, cudaStream_t s, int products_valid) {
  HalsArgs a;
  a.products_valid = products_valid;
  a.st = st;
  a.normalize_a = normalize_a;
  a.alpha = alpha;
  a.beta = beta;
  a.it_begin = it_begin;
  a.it_end = it_end;
  a.start_half = start_half;
  a.start_col = start_col;
  a.skip_dead = skip_dead;
  a.epoch0 = epoch0;
  a.rows_a = rows_per_cta(st.d, grid);
  a.rows_b = rows_per_cta(st.n, grid);
  size_t smem = hals_smem_bytes(st, a.rows_a);
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  // rows per thread of the A sweep (register-resident across the column chain)
  const int rpt = (a.rows_a + kThreads - 1) / kThreads;
  if (rpt > kMaxRPTLarge) return cudaErrorInvalidConfiguration;
  const bool large = rpt > 3 || std::getenv("CNMF_HALS_RPT6") != nullptr;  // env: tests only
  // DMMA block products in the A sweep where g and the product buffer fit
  // next to the kernel's static shared memory (CNMF_HALS_ASIMT: comparisons)
  const size_t adm = a_dmma_smem(st, a.rows_a, large ? 8 : 16);
  // Measured: C4 (k = 100) A sweep 344k -> 267k cycles per iteration; at
  // C3 (k = 50, 676 rows per SM) the SIMT loop is faster (163k vs 197k), so
  // the tensor-core product is taken from k > 64.
  a.a_dmma = adm + 4096 <= 227 * 1024 && st.k > 64 && std::getenv("CNMF_HALS_ASIMT") == nullptr;
  if (a.a_dmma) smem = std::max(smem, adm);
  const bool inl = st.words != nullptr && !st.dense;  // in-kernel service of emptied A columns
  const void* fn = large ? (inl ? (const void*)hals_kernel<kMaxRPTLarge, 8, true>
                                : (const void*)hals_kernel<kMaxRPTLarge, 8, false>)
                         : (inl ? (const void*)hals_kernel<3, 16, true> : (const void*)hals_kernel<3, 16, false>);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  void* args[] = {&a};
  note_launches(1);
  return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kThreads), args, smem, s);
}

void launch_compress_factors(const HalsState& st, int which, int column, cudaStream_t s) {
  if (column < 0 && st.part_ctas > 0 && st.lp <= 128 && st.k <= 128) {
    const float* basis = which == 0 ? st.lm : st.rt;
    const int64_t rows = which == 0 ? st.d : st.n;
    const int64_t per = ((rows + st.part_ctas - 1) / st.part_ctas + kCfRows - 1) / kCfRows * kCfRows;
    const int ctas = (int)std::max<int64_t>(1, (rows + per - 1) / per);
    note_launches(2);
    compress_factor_tile_kernel<<<ctas, 256, 0, s>>>(basis, rows, st.lp, which == 0 ? st.a : st.b, st.k,
                                                     per, st.part);
    compress_factor_reduce_kernel<<<(st.lp * st.k + 255) / 256, 256, 0, s>>>(
        st.part, ctas, st.lp, st.k, st.l, which == 0 ? st.ahat : st.bchk);
    return;
  }
  const dim3 grid(st.lp, column >= 0 ? 1 : st.k);
  note_launches(1);
  if (which == 0)
    compress_factor_kernel<<<grid, 256, 0, s>>>(st.lm, st.d, st.lp, st.a, st.k, column, st.l,
                                                st.ahat);
  else
    compress_factor_kernel<<<grid, 256, 0, s>>>(st.rt, st.n, st.lp, st.b, st.k, column, st.l,
                                                st.bchk);
}

void launch_normalize_column(double* a_cm, int64_t d, int j, cudaStream_t s) {
  note_launches(1);
  normalize_column_kernel<<<1, 1024, 0, s>>>(a_cm, d, j);
}

}  // namespace cnmf
