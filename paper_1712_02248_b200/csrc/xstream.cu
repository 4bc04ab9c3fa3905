// xstream.cu -- the X-streaming contractions of the compression half.
//
// Reference call sites (all dense `matmul`, proj/src/matrix.cpp:94-154):
//   X * S     (NN, matrix.cpp:105-116) from range_finder_impl
//             (proj/src/compression.cpp:33,37,39) and compress_right (:82-84,
//             as X * (R^T) with R^T held row-major n x l)
//   X^T * T   (TN, matrix.cpp:129-140) from range_finder_impl (:32,38,39)
//             and compress_left (:73-75, stored transposed: X-hat^T = X^T L)
//
// One X pass per call; every X element is read once from HBM (128-bit loads,
// coalesced along rows), staged in shared memory and reused for all lp
// output columns from registers.  Split-K partials are reduced in a fixed
// order, so results are bitwise reproducible run to run.
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "kernels.h"

namespace cnmf {

namespace {

constexpr int kBM = 64;   // output rows per CTA
constexpr int kBK = 32;   // reduction depth per stage
constexpr int kAPad = 4;  // smem row padding for the staged X tile

template <bool kTN, int LP>
__global__ void __launch_bounds__(256) xs_kernel(const float* __restrict__ x, int64_t ldx,
                                                 int64_t m, int64_t n,
                                                 const float* __restrict__ s,
                                                 float* __restrict__ out, int64_t kchunk) {
  constexpr int TNC = LP / 16;
  extern __shared__ __align__(16) float xs_smem[];
  float(*As)[kBK][kBM + kAPad] = reinterpret_cast<float(*)[kBK][kBM + kAPad]>(xs_smem);
  float(*Bs)[kBK][LP] = reinterpret_cast<float(*)[kBK][LP]>(xs_smem + 2 * kBK * (kBM + kAPad));

  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const int64_t out_rows = kTN ? n : m;
  const int64_t K = kTN ? m : n;
  const int64_t row0 = (int64_t)blockIdx.x * kBM;
  const int64_t kbeg = (int64_t)blockIdx.y * kchunk;
  const int64_t kend = min(K, kbeg + kchunk);
  float* dst = out + (int64_t)blockIdx.y * out_rows * LP;

  float4 ra[2];
  float4 rb[(8 * LP + 255) / 256];

  auto load_tile = [&](int64_t k0) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int idx = tid + i * 256;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (!kTN) {
        const int r = idx >> 3, k4 = idx & 7;
        const int64_t gr = row0 + r, gk = k0 + 4 * k4;
        if (gr < m && gk < kend) {
          const float* src = x + gr * ldx + gk;
          if (gk + 3 < kend) {
            v = __ldg(reinterpret_cast<const float4*>(src));
          } else {  // ragged tail: never read past column kend - 1
            v.x = __ldg(src);
            if (gk + 1 < kend) v.y = __ldg(src + 1);
            if (gk + 2 < kend) v.z = __ldg(src + 2);
          }
        }
      } else {
        const int kk = idx >> 4, c4 = idx & 15;
        const int64_t gk = k0 + kk, gc = row0 + 4 * c4;
        if (gk < kend && gc < n) {
          const float* src = x + gk * ldx + gc;
          if (gc + 3 < n) {
            v = __ldg(reinterpret_cast<const float4*>(src));
          } else {
            v.x = __ldg(src);
            if (gc + 1 < n) v.y = __ldg(src + 1);
            if (gc + 2 < n) v.z = __ldg(src + 2);
          }
        }
      }
      ra[i] = v;
    }
#pragma unroll
    for (int i = 0; i < (8 * LP + 255) / 256; ++i) {
      const int idx = tid + i * 256;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (idx < 8 * LP) {
        const int kk = idx / (LP / 4), j4 = idx % (LP / 4);
        const int64_t gk = k0 + kk;
        if (gk < kend) v = __ldg(reinterpret_cast<const float4*>(s + gk * LP + 4 * j4));
      }
      rb[i] = v;
    }
  };
  auto store_tile = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int idx = tid + i * 256;
      if (!kTN) {
        const int r = idx >> 3, k4 = idx & 7;
        As[buf][4 * k4 + 0][r] = ra[i].x;
        As[buf][4 * k4 + 1][r] = ra[i].y;
        As[buf][4 * k4 + 2][r] = ra[i].z;
        As[buf][4 * k4 + 3][r] = ra[i].w;
      } else {
        const int kk = idx >> 4, c4 = idx & 15;
        *reinterpret_cast<float4*>(&As[buf][kk][4 * c4]) = ra[i];
      }
    }
#pragma unroll
    for (int i = 0; i < (8 * LP + 255) / 256; ++i) {
      const int idx = tid + i * 256;
      if (idx < 8 * LP) {
        const int kk = idx / (LP / 4), j4 = idx % (LP / 4);
        *reinterpret_cast<float4*>(&Bs[buf][kk][4 * j4]) = rb[i];
      }
    }
  };

  float acc[4][TNC];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < TNC; ++j) acc[i][j] = 0.f;

  if (kbeg < kend) {
    load_tile(kbeg);
    store_tile(0);
    __syncthreads();
    int buf = 0;
    for (int64_t k0 = kbeg; k0 < kend; k0 += kBK) {
      const bool more = k0 + kBK < kend;
      if (more) load_tile(k0 + kBK);
#pragma unroll 8
      for (int kk = 0; kk < kBK; ++kk) {
        const float4 a = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
        float b[TNC];
#pragma unroll
        for (int j = 0; j < TNC; ++j) b[j] = Bs[buf][kk][tx + 16 * j];
#pragma unroll
        for (int j = 0; j < TNC; ++j) {
          acc[0][j] = fmaf(a.x, b[j], acc[0][j]);
          acc[1][j] = fmaf(a.y, b[j], acc[1][j]);
          acc[2][j] = fmaf(a.z, b[j], acc[2][j]);
          acc[3][j] = fmaf(a.w, b[j], acc[3][j]);
        }
      }
      if (more) {
        store_tile(buf ^ 1);
        __syncthreads();
        buf ^= 1;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = row0 + ty * 4 + i;
    if (r < out_rows) {
#pragma unroll
      for (int j = 0; j < TNC; ++j) dst[r * LP + tx + 16 * j] = acc[i][j];
    }
  }
}

__global__ void split_reduce_kernel(const float4* __restrict__ part, int splits, int64_t total4,
                                    float4* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total4;
       e += (int64_t)gridDim.x * blockDim.x) {
    float4 acc = part[e];
    for (int s = 1; s < splits; ++s) {
      const float4 v = part[(int64_t)s * total4 + e];
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    out[e] = acc;
  }
}

struct SplitPlan {
  int64_t kchunk;
  int splits;
  int tiles;
};

SplitPlan plan(int64_t out_rows, int64_t K, int nsm) {
  SplitPlan p;
  p.tiles = (int)((out_rows + kBM - 1) / kBM);
  const int64_t kblocks = (K + kBK - 1) / kBK;
  const int64_t target = (int64_t)nsm * 3;
  int64_t splits = (target + p.tiles - 1) / p.tiles;
  splits = std::max<int64_t>(1, std::min<int64_t>(splits, kblocks));
  const int64_t per = (kblocks + splits - 1) / splits;
  p.kchunk = std::max<int64_t>(1, per) * kBK;
  p.splits = (int)((K + p.kchunk - 1) / p.kchunk);
  if (p.splits < 1) p.splits = 1;
  return p;
}

template <bool kTN>
void dispatch(const float* x, int64_t ldx, int64_t m, int64_t n, const float* s, int lp,
              float* out, float* ws, int nsm, cudaStream_t st) {
  const int64_t out_rows = kTN ? n : m;
  const SplitPlan p = plan(out_rows, kTN ? m : n, nsm);
  float* dst = p.splits > 1 ? ws : out;
  dim3 grid(p.tiles, p.splits);
  switch (lp) {
#define CNMF_XS_CASE(LPV)                                                              \
  case LPV: {                                                                           \
    const int smem = (int)sizeof(float) * 2 * kBK * (kBM + kAPad + LPV);                \
    static std::atomic<unsigned> attr{0u};                                              \
    smem_attr_once(attr, (const void*)(xs_kernel<kTN, LPV>), smem);                     \
    note_launches(1);                                                                   \
    xs_kernel<kTN, LPV><<<grid, 256, smem, st>>>(x, ldx, m, n, s, dst, p.kchunk);       \
    break;                                                                              \
  }
    CNMF_XS_CASE(16)
    CNMF_XS_CASE(32)
    CNMF_XS_CASE(48)
    CNMF_XS_CASE(64)
    CNMF_XS_CASE(80)
    CNMF_XS_CASE(96)
    CNMF_XS_CASE(112)
    CNMF_XS_CASE(128)
#undef CNMF_XS_CASE
    default: return;
  }
  if (p.splits > 1) {
    const int64_t total4 = out_rows * lp / 4;
    const int blocks = (int)std::min<int64_t>((total4 + 255) / 256, (int64_t)nsm * 8);
    note_launches(1);
    split_reduce_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<const float4*>(ws), p.splits,
                                                total4, reinterpret_cast<float4*>(out));
  }
}

}  // namespace

size_t xstream_ws_floats(int64_t m, int64_t n, int lp, int nsm) {
  const SplitPlan a = plan(m, n, nsm), b = plan(n, m, nsm);
  const int64_t fa = a.splits > 1 ? (int64_t)a.splits * m * lp : 0;
  const int64_t fb = b.splits > 1 ? (int64_t)b.splits * n * lp : 0;
  return std::max<size_t>((size_t)std::max<int64_t>(std::max(fa, fb), 4),
                          xstream_tc_ws_floats(m, n, lp, nsm));
}

// The tcgen05 kernel (xstream_tc.cu) is the production path; this SIMT kernel
// serves shapes outside its envelope and CNMF_XS=simt (A/B comparisons).
static bool use_tc() {
  static const int mode = [] {
    const char* e = std::getenv("CNMF_XS");
    return (e && std::string(e) == "simt") ? 0 : 1;
  }();
  return mode == 1;
}

void launch_xs_nn(const float* x, int64_t ldx, int64_t m, int64_t n, const float* s, int lp,
                  float* y, float* ws, int nsm, cudaStream_t st, const int8_t* rexp, bool x_exact) {
  if (use_tc() && launch_xs_tc(false, x, ldx, m, n, s, lp, y, ws, nsm, st, rexp, x_exact)) return;
  dispatch<false>(x, ldx, m, n, s, lp, y, ws, nsm, st);
}

void launch_xs_tn(const float* x, int64_t ldx, int64_t m, int64_t n, const float* t, int lp,
                  float* z, float* ws, int nsm, cudaStream_t st, const int8_t* rexp, bool x_exact) {
  if (use_tc() && launch_xs_tc(true, x, ldx, m, n, t, lp, z, ws, nsm, st, rexp, x_exact)) return;
  dispatch<true>(x, ldx, m, n, t, lp, z, ws, nsm, st);
}

}  // namespace cnmf
