// hals_resident.cu -- FastHALS-RP iterations with every operand resident in
// shared memory (configurations whose per-CTA rows fit, e.g. BASELINE C1/C2).
//
// Same algorithm, precision, halting protocol and exchange primitives as the
// streaming kernel in hals.cu (reference: fasthals_rp_step,
// proj/src/solvers.cpp:414-456).  At launch each CTA loads its rows of
// X-check, L (A side) and X-hat^T, R^T (B side) as fp64 plus its fp64 rows
// of A and B; every product, sweep and partial then runs from shared memory
// and the only global traffic is the per-column norm all-reduce and the
// A-hat / B-check partials.  A and B are written back when the launch ends
// or halts.
#include <cstdlib>

#include "common.cuh"
#include "hals_common.cuh"
#include "kernels.h"

namespace cnmf {

namespace {

using namespace hals_detail;
constexpr int kNB = 8;           // columns per block of the blocked sweeps
constexpr double kDead = 1e-12;  // solvers.cpp:19

struct ResArgs {
  HalsState st;
  int normalize_a;
  double alpha, beta;
  int it_begin, it_end, start_half, start_col, skip_dead;
  int rows_a, rows_b;
  unsigned long long epoch0;
};

struct ResLayout {  // offsets in doubles
  int64_t xc, lm, as, hs, xh, rt, bs0, bs1, ps, gw, ms, red, total;
};

__host__ __device__ inline ResLayout res_layout(int rows_a, int rows_b, int lp, int k) {
  const int64_t lpp = lp + 1, kp1 = k + 1;
  ResLayout L;
  int64_t o = 0;
  L.xc = o; o += rows_a * lpp;
  L.lm = o; o += rows_a * lpp;
  L.as = o; o += rows_a * kp1;
  L.hs = o; o += rows_a * kp1;
  L.xh = o; o += rows_b * lpp;
  L.rt = o; o += rows_b * lpp;
  L.bs0 = o; o += rows_b * kp1;
  L.bs1 = o; o += rows_b * kp1;
  L.ps = o; o += rows_b * kp1;
  L.gw = o; o += (int64_t)k * k;
  L.ms = o; o += lpp * k;
  L.red = o; o += 16 * kThreads;
  L.total = o;
  return L;
}

// fp32 global rows (ld lp) -> fp64 shared rows (stride lp + 1)
__device__ void load_rows(const float* __restrict__ src, int nrows, int lp, double* dst) {
  const int lpp = lp + 1, q4 = lp >> 2;
  for (int e = threadIdx.x; e < nrows * q4; e += kThreads) {
    const int r = e / q4, c4 = e - r * q4;
    const float4 v = __ldg(reinterpret_cast<const float4*>(src + (int64_t)r * lp) + c4);
    double* d = dst + r * lpp + 4 * c4;
    d[0] = v.x;
    d[1] = v.y;
    d[2] = v.z;
    d[3] = v.w;
  }
}

// out[r][c] = sum_q X[r][q] M[q][c] (all shared fp64); X stride lpp, M lp x k
// (stride k), out stride kp1.  2x4 register tiles.
__device__ void prod_rows(const double* X, int nrows, int lp, int kdim, const double* M, int k,
                          double* out) {
  const int lpp = lp + 1, kp1 = k + 1;
  const int rg = (nrows + 1) >> 1, cgn = (k + 3) >> 2, tiles = rg * cgn;
  for (int tI = threadIdx.x; tI < tiles; tI += kThreads) {
    const int r0 = 2 * (tI / cgn), c0 = 4 * (tI % cgn);
    const bool r1ok = r0 + 1 < nrows;
    double acc[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
    const double* x0 = X + r0 * lpp;
    const double* x1 = X + (r1ok ? r0 + 1 : r0) * lpp;
#pragma unroll 4
    for (int q = 0; q < kdim; ++q) {
      const double a0 = x0[q], a1 = x1[q];
      const double* m = M + q * k + c0;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const double mv = c0 + t < k ? m[t] : 0.0;
        acc[0][t] = fma(a0, mv, acc[0][t]);
        acc[1][t] = fma(a1, mv, acc[1][t]);
      }
    }
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (c0 + t < k) {
        out[r0 * kp1 + c0 + t] = acc[0][t];
        if (r1ok) out[(r0 + 1) * kp1 + c0 + t] = acc[1][t];
      }
  }
  __syncthreads();
}

// part[l'][c] = sum_r X[r][l'] F[r][c] over nrows shared rows (fp64, rows in
// ascending order) into global part (lp x k, rows >= l zero).  2 x 2 output
// blocks, one per thread, each summing all rows itself: no cross-thread
// reduction, two independent accumulator chains per output (even / odd rows,
// added at the end in a fixed order).
__device__ void partial_rows(const double* X, const double* F, int nrows, int l, int lp, int k,
                             double* /*red*/, double* __restrict__ part) {
  const int lpp = lp + 1, kp1 = k + 1;
  const int nbl = (l + 1) >> 1, nbc = (k + 1) >> 1, nb = nbl * nbc;
  for (int b = threadIdx.x; b < nb; b += kThreads) {
    const int l0 = 2 * (b / nbc), c0 = 2 * (b - (b / nbc) * nbc);
    const int l1 = min(l0 + 1, l - 1), c1 = min(c0 + 1, k - 1);
    double a[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
    int r = 0;
    for (; r + 1 < nrows; r += 2) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double* xr = X + (r + h) * lpp;
        const double* fr = F + (r + h) * kp1;
        const double x0 = xr[l0], x1 = xr[l1], f0 = fr[c0], f1 = fr[c1];
        a[h][0] = fma(x0, f0, a[h][0]);
        a[h][1] = fma(x0, f1, a[h][1]);
        a[h][2] = fma(x1, f0, a[h][2]);
        a[h][3] = fma(x1, f1, a[h][3]);
      }
    }
    if (r < nrows) {
      const double* xr = X + r * lpp;
      const double* fr = F + r * kp1;
      a[0][0] = fma(xr[l0], fr[c0], a[0][0]);
      a[0][1] = fma(xr[l0], fr[c1], a[0][1]);
      a[0][2] = fma(xr[l1], fr[c0], a[0][2]);
      a[0][3] = fma(xr[l1], fr[c1], a[0][3]);
    }
    part[l0 * k + c0] = a[0][0] + a[1][0];
    if (c0 + 1 < k) part[l0 * k + c0 + 1] = a[0][1] + a[1][1];
    if (l0 + 1 < l) {
      part[(l0 + 1) * k + c0] = a[0][2] + a[1][2];
      if (c0 + 1 < k) part[(l0 + 1) * k + c0 + 1] = a[0][3] + a[1][3];
    }
  }
  for (int e = l * k + threadIdx.x; e < lp * k; e += kThreads) part[e] = 0.0;
}

// MS <- M (global fp64 lp x k, stride k in shared), then GW = MS^T MS over
// the first l rows (fp64): one upper-triangle entry per thread, rows in
// ascending order, mirrored.
__device__ void load_and_gram(const double* __restrict__ M, int l, int lp, int k, double* ms,
                              double* gw) {
  __syncthreads();
  for (int e = threadIdx.x; e < lp * k; e += kThreads) ms[e] = __ldcg(M + e);
  __syncthreads();
  const int ntri = k * (k + 1) / 2;
  for (int e = threadIdx.x; e < ntri; e += kThreads) {
    int a = 0, rem = e;
    while (rem >= k - a) {
      rem -= k - a;
      ++a;
    }
    const int c = a + rem;
    double s0 = 0.0, s1 = 0.0;
    int r = 0;
    for (; r + 1 < l; r += 2) {
      s0 = fma(ms[r * k + a], ms[r * k + c], s0);
      s1 = fma(ms[(r + 1) * k + a], ms[(r + 1) * k + c], s1);
    }
    if (r < l) s0 = fma(ms[r * k + a], ms[r * k + c], s0);
    const double v = s0 + s1;
    gw[a * k + c] = v;
    gw[c * k + a] = v;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads, 1) hals_resident_kernel(const ResArgs p) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double red8[kThreads / 32];
  __shared__ double s_red[2];      // all-reduce total, 1/sqrt(total)
  __shared__ double s_ginv[128];   // 1/g_jj or 1/w_jj of the current half
  __shared__ unsigned zmask[4];
  __shared__ unsigned s_zw[4 * (kThreads / 32)];
  __shared__ long long s_prof[21];

  const HalsState& S = p.st;
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
  const int k = S.k, lp = S.lp, l = S.l, kp1 = k + 1;
  const int64_t d = S.d, n = S.n;
  const int64_t a_lo = min(d, (int64_t)cta * p.rows_a), a_hi = min(d, a_lo + p.rows_a);
  const int64_t b_lo = min(n, (int64_t)cta * p.rows_b), b_hi = min(n, b_lo + p.rows_b);
  const int na = (int)(a_hi - a_lo), nbr = (int)(b_hi - b_lo);
  const int nel = lp * k;
  const ResLayout L = res_layout(p.rows_a, p.rows_b, lp, k);
  double *XC = sm + L.xc, *LM = sm + L.lm, *AS = sm + L.as, *HS = sm + L.hs;
  double *XH = sm + L.xh, *RT = sm + L.rt, *PS = sm + L.ps, *GW = sm + L.gw, *MS = sm + L.ms;
  double *RED = sm + L.red;
  double* bsc = sm + L.bs0;  // B as of the start of the B half
  double* bsn = sm + L.bs1;

  const bool prof = S.prof != nullptr && cta == 0;
  long long t_last = 0;
  if (prof && tid == 0) {
    for (int i = 0; i < 21; ++i) s_prof[i] = 0;
    t_last = clock64();
  }
#define RES_PROF(id)                  \
  if (prof && tid == 0) {             \
    const long long now_ = clock64(); \
    s_prof[id] += now_ - t_last;      \
    t_last = now_;                    \
  }

  // ---- prologue: rows of the compressed views, projectors and state ----
  load_rows(S.xc + a_lo * lp, na, lp, XC);
  load_rows(S.lm + a_lo * lp, na, lp, LM);
  load_rows(S.xht + b_lo * lp, nbr, lp, XH);
  load_rows(S.rt + b_lo * lp, nbr, lp, RT);
  for (int e = tid; e < na * k; e += kThreads) {
    const int c = e / na, r = e - c * na;
    AS[r * kp1 + c] = S.a[(int64_t)c * d + a_lo + r];
  }
  for (int e = tid; e < nbr * k; e += kThreads) {
    const int c = e / nbr, r = e - c * nbr;
    bsc[r * kp1 + c] = S.b[(int64_t)c * n + b_lo + r];
  }
  __syncthreads();

  auto write_back = [&](const double* bsrc) {
    __syncthreads();
    for (int e = tid; e < na * k; e += kThreads) {
      const int c = e / na, r = e - c * na;
      S.a[(int64_t)c * d + a_lo + r] = AS[r * kp1 + c];
    }
    for (int e = tid; e < nbr * k; e += kThreads) {
      const int c = e / nbr, r = e - c * nbr;
      S.b[(int64_t)c * n + b_lo + r] = bsrc[r * kp1 + c];
    }
  };

  unsigned long long ep = p.epoch0;
  unsigned long long nr = S.nr0;  // norm all-reduces so far (slot tags)
  bool have_g = false, have_w = false;
  int half = p.start_half, col0 = p.start_col, skip = p.skip_dead;
  const bool constrained = !(p.alpha == 0.0 && p.beta == 0.0);

  for (int it = p.it_begin; it < p.it_end; ++it) {
    if (half == 0) {
      // ================= A half (solvers.cpp:419-439) =====================
      if (!have_g) load_and_gram(S.bchk, l, lp, k, MS, GW);  // g (422)
      else {
        __syncthreads();
        for (int e = tid; e < lp * k; e += kThreads) MS[e] = __ldcg(S.bchk + e);
        __syncthreads();
      }
      prod_rows(XC, na, lp, l, MS, k, HS);  // h = X-check B-check (421)
      RES_PROF(1);
      int jd = k;
      for (int j = col0; j < k; ++j)
        if (j != skip && GW[j * k + j] < kDead) { jd = j; break; }
      skip = -1;
      // reciprocal divisors: one multiply on the per-column critical path
      // (differs from the reference's division by at most one rounding)
      for (int e = tid; e < k; e += kThreads) s_ginv[e] = 1.0 / GW[e * k + e];
      __syncthreads();
      const int r = tid;  // one A row per thread (rows_a <= 256)
      const bool live = r < na;
      for (int jb = col0; jb < jd; jb += kNB) {
        const int nbj = min(kNB, jd - jb);
        double acc[kNB], dl[kNB];
#pragma unroll
        for (int t = 0; t < kNB; ++t) {
          acc[t] = 0.0;
          dl[t] = 0.0;
        }
        if (live)
          for (int c = 0; c < k; ++c) {
            const double a = AS[r * kp1 + c];
#pragma unroll
            for (int t = 0; t < kNB; ++t)
              if (t < nbj) acc[t] = fma(a, GW[c * k + jb + t], acc[t]);
          }
        RES_PROF(2);
#pragma unroll
        for (int t = 0; t < kNB; ++t) {
          if (t >= nbj) break;
          const int j = jb + t;
          double v = 0.0, aold = 0.0;
          if (live) {  // solvers.cpp:430-434
            double s = acc[t];
#pragma unroll
            for (int u = 0; u < kNB; ++u)
              if (u < t) s = fma(dl[u], GW[(jb + u) * k + j], s);
            aold = AS[r * kp1 + j];
            v = aold + (HS[r * kp1 + j] - s) * s_ginv[j];
            v = v > 0.0 ? v : 0.0;
          }
          RES_PROF(2);
          const double total = allreduce_fused(S, G, cta, ep, nr, v * v, red8, s_red, prof ? s_prof + 17 : nullptr);
          RES_PROF(3);
          if (total == 0.0) {  // column emptied: host redraws a_j (solvers.cpp:435)
            if (live) AS[r * kp1 + j] = 0.0;
            write_back(bsc);
            if (cta == 0 && tid == 0) { *S.halt = HaltInfo{1, it + 1, 0, j, kEvZeroA, 0, ep}; S.halt->last_nr = nr; }
            return;
          }
          if (live) {  // solvers.cpp:436
            const double nf = p.normalize_a ? v * s_red[1] : v;
            AS[r * kp1 + j] = nf;
            dl[t] = nf - aold;
          }
        }
      }
      __syncthreads();
      if (jd < k) {  // dead B column: host redraws b_jd (solvers.cpp:424-428)
        write_back(bsc);
        if (cta == 0 && tid == 0) { *S.halt = HaltInfo{1, it + 1, 0, jd, kEvDeadB, 0, ep}; S.halt->last_nr = nr; }
        return;
      }
      partial_rows(LM, AS, na, l, lp, k, RED, S.part + (int64_t)cta * nel);  // A-hat (438)
      RES_PROF(4);
      exchange_fast(S, G, ep);
      RES_PROF(5);
      slice_reduce(S.part, G, nel, S.ahat);
      exchange_fast(S, G, ep);
      RES_PROF(7);
      load_and_gram(S.ahat, l, lp, k, MS, GW);  // w (443); MS keeps A-hat for p
      RES_PROF(8);
      have_w = true;
      half = 1;
      col0 = 0;
    } else if (!have_w) {
      load_and_gram(S.ahat, l, lp, k, MS, GW);
    }
    // ================== B half (solvers.cpp:440-455) =======================
    prod_rows(XH, nbr, lp, l, MS, k, PS);  // p = X-hat^T A-hat (442)
    for (int e = tid; e < 4 * (kThreads / 32); e += kThreads) s_zw[e] = 0u;
    for (int e = tid; e < k; e += kThreads)
      s_ginv[e] = 1.0 / (constrained ? GW[e * k + e] + p.beta : GW[e * k + e]);
    __syncthreads();
    int jd = k;
    for (int j = col0; j < k; ++j)
      if (j != skip && GW[j * k + j] < kDead) { jd = j; break; }
    skip = -1;
    RES_PROF(9);
    if ((tid & ~31) < nbr) {  // warps holding B rows (one row per thread)
      const int r = tid;
      const bool live = r < nbr;
      const int rr = live ? r : 0;
      unsigned zw0 = 0u, zw1 = 0u, zw2 = 0u, zw3 = 0u;  // columns with a non-zero entry in this warp
      if (live)
        for (int c = 0; c < col0; ++c) bsn[r * kp1 + c] = bsc[r * kp1 + c];
      for (int jb = col0; jb < jd; jb += kNB) {
        const int nbj = min(kNB, jd - jb);
        double acc[kNB], dl[kNB];
#pragma unroll
        for (int t = 0; t < kNB; ++t) {
          acc[t] = 0.0;
          dl[t] = 0.0;
        }
        for (int c = 0; c < k; ++c) {  // columns < jb already live in bsn
          const double bv = c < jb ? bsn[rr * kp1 + c] : bsc[rr * kp1 + c];
#pragma unroll
          for (int t = 0; t < kNB; ++t)
            if (t < nbj) acc[t] = fma(bv, GW[c * k + jb + t], acc[t]);
        }
#pragma unroll
        for (int t = 0; t < kNB; ++t) {
          if (t >= nbj) break;
          const int j = jb + t;
          double sacc = acc[t];
#pragma unroll
          for (int u = 0; u < kNB; ++u)
            if (u < t) sacc = fma(dl[u], GW[(jb + u) * k + j], sacc);
          const double wjj = GW[j * k + j];
          const double bij = bsc[rr * kp1 + j], pij = PS[rr * kp1 + j];
          const double v = constrained ? (bij * wjj + pij - sacc - p.alpha) * s_ginv[j]  // 502-508
                                       : bij + (pij - sacc) * s_ginv[j];                  // 480-490
          const double vf = v > 0.0 ? v : 0.0;
          if (live) bsn[r * kp1 + j] = vf;
          dl[t] = vf - bij;
          if (__ballot_sync(0xffffffffu, live && vf != 0.0)) {
            const unsigned bit = 1u << (j & 31);
            if ((j >> 5) == 0) zw0 |= bit;
            else if ((j >> 5) == 1) zw1 |= bit;
            else if ((j >> 5) == 2) zw2 |= bit;
            else zw3 |= bit;
          }
        }
      }
      if (live)
        for (int c = jd; c < k; ++c) bsn[r * kp1 + c] = bsc[r * kp1 + c];
      if ((tid & 31) == 0) {
        const int w = tid >> 5;
        s_zw[4 * w + 0] = zw0;
        s_zw[4 * w + 1] = zw1;
        s_zw[4 * w + 2] = zw2;
        s_zw[4 * w + 3] = zw3;
      }
    }
    __syncthreads();
    if (tid < 4) {
      unsigned m = 0u;
      for (int w = 0; w < kThreads / 32; ++w) m |= s_zw[4 * w + tid];
      zmask[tid] = m;
    }
    RES_PROF(10);
    // zero-column flags: one OR per CTA into S.zpart[0..3] (reset by CTA 0
    // after the next exchange, and by the launcher), published by the exchange
    if (tid < 4 && zmask[tid]) atomicOr(S.zpart + tid, zmask[tid]);
    partial_rows(RT, bsn, nbr, l, lp, k, RED, S.part + (int64_t)cta * nel);  // B-check (454)
    RES_PROF(11);
    exchange_fast(S, G, ep);
    RES_PROF(12);
    if (tid < 4) zmask[tid] = __ldcg(S.zpart + tid);
    __syncthreads();
    if (S.sharded) {
      // this rank's B-check partial; the host all-reduces it with the other
      // ranks' and decides zero columns on the global mask
      slice_reduce(S.part, G, nel, S.bchk);
      exchange_fast(S, G, ep);
      if (cta == 0 && tid < 4) {
        S.zpart[4 * G + tid] = zmask[tid];
        S.zpart[tid] = 0u;
      }
      for (int e = tid; e < nbr * k; e += kThreads) {  // old B for a host-side rollback
        const int c = e / nbr, r = e - c * nbr;
        S.bold[(int64_t)c * n + b_lo + r] = bsc[r * kp1 + c];
      }
      write_back(bsn);
      if (cta == 0 && tid == 0) { *S.halt = HaltInfo{1, it + 1, 1, jd, kEvShard, 0, ep}; S.halt->last_nr = nr; }
      return;
    }
    int j0 = k;
    for (int j = col0; j < jd; ++j)
      if (!(zmask[j >> 5] & (1u << (j & 31)))) { j0 = j; break; }
    if (j0 < jd || jd < k) {
      // columns after an emptied b_j0 were computed against the zero column:
      // they keep their old values (columns from jd on already do)
      if (j0 < jd && tid < nbr)
        for (int c = j0 + 1; c < jd; ++c) bsn[tid * kp1 + c] = bsc[tid * kp1 + c];
      write_back(bsn);
      if (cta == 0 && tid == 0) {
        *S.halt = j0 < jd ? HaltInfo{1, it + 1, 1, j0, kEvZeroB, 0, ep}
                          : HaltInfo{1, it + 1, 1, jd, kEvDeadA, 0, ep};
        S.halt->last_nr = nr;
      }
      return;
    }
    RES_PROF(13);
    slice_reduce(S.part, G, nel, S.bchk);
    exchange_fast(S, G, ep);
    if (cta == 0 && tid < 4) S.zpart[tid] = 0u;  // every CTA has read the flags
    RES_PROF(15);
    load_and_gram(S.bchk, l, lp, k, MS, GW);  // g for the next A half (422)
    RES_PROF(16);
    have_g = true;
    double* tb = bsc;
    bsc = bsn;
    bsn = tb;
    half = 0;
    col0 = 0;
  }
  write_back(bsc);
  if (cta == 0 && tid == 0) {
    *S.halt = HaltInfo{0, p.it_end, 0, 0, 0, 0, ep};
    S.halt->last_nr = nr;
    if (prof)
      for (int i = 0; i < 21; ++i) S.prof[i] += s_prof[i];
  }
#undef RES_PROF
}

}  // namespace

int hals_resident_grid(const HalsState& st, int nsm) {
  if (const char* e = std::getenv("CNMF_RES_GRID")) {  // experiments only (tools/)
    const int g = std::atoi(e);
    const int ra = (int)((st.d + g - 1) / g), rb = (int)((st.n + g - 1) / g);
    if (g >= 1 && g <= nsm && ra <= kThreads && rb <= kThreads &&
        res_layout(ra, rb, st.lp, st.k).total * (int64_t)sizeof(double) <= 220 * 1024)
      return g;
  }
  for (int g = std::max(1, (int)((std::max(st.d, st.n) + kThreads - 1) / kThreads)); g <= nsm;
       ++g) {
    const int ra = (int)((st.d + g - 1) / g), rb = (int)((st.n + g - 1) / g);
    if (ra > kThreads || rb > kThreads) continue;
    if (res_layout(ra, rb, st.lp, st.k).total * (int64_t)sizeof(double) <= 220 * 1024) {
      // prefer the full chip (more DFMA lanes) when that still fits
      const int ra2 = (int)((st.d + nsm - 1) / nsm), rb2 = (int)((st.n + nsm - 1) / nsm);
      if (res_layout(ra2, rb2, st.lp, st.k).total * (int64_t)sizeof(double) <= 220 * 1024)
        return nsm;
      return g;
    }
  }
  return 0;  // does not fit: use the streaming kernel
}

cudaError_t launch_hals_resident(const HalsState& st, int normalize_a, double alpha, double beta,
                                 int it_begin, int it_end, int start_half, int start_col,
                                 int skip_dead, unsigned long long epoch0, int grid,
                                 cudaStream_t s) {
  ResArgs a;
  a.st = st;
  a.normalize_a = normalize_a;
  a.alpha = alpha;
  a.beta = beta;
  a.it_begin = it_begin;
  a.it_end = it_end;
  a.start_half = start_half;
  a.start_col = start_col;
  a.skip_dead = skip_dead;
  a.rows_a = (int)((st.d + grid - 1) / grid);
  a.rows_b = (int)((st.n + grid - 1) / grid);
  a.epoch0 = epoch0;
  const size_t smem = (size_t)res_layout(a.rows_a, a.rows_b, st.lp, st.k).total * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(hals_resident_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(st.zpart, 0, 4 * sizeof(unsigned), s);  // zero-column flag words
  if (e != cudaSuccess) return e;
  void* args[] = {&a};
  note_launches(1);
  return cudaLaunchCooperativeKernel((const void*)hals_resident_kernel, dim3(grid),
                                     dim3(kThreads), args, smem, s);
}

}  // namespace cnmf
