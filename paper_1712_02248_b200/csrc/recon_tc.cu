// recon_tc.cu -- the objective 1/2 ||X - A B^T||_F^2 on the 5th-generation
// tensor cores (reference: reconstruction_error, proj/src/metrics.cpp:61-77,
// the direct-residual form; the run evaluates it every error_interval
// iterations, solvers.cpp:223-229,262-283).
//
// One X pass.  For a 128-row x 64-column tile of X the prediction
// P = A_tile B_tile^T (K = k, padded to KR, a multiple of 8) is computed by
// tcgen05 kind::tf32 MMAs in the 3xTF32 split (a_hi b_hi + a_hi b_lo +
// a_lo b_hi, fp32 accumulation in tensor memory, K <= 128 so the chain is
// short), then the epilogue reads the X tile from shared memory, forms the
// fp32 residual x - p and accumulates its square in fp64.  The residual's
// relative error is ~1e-6 |x| / |x - p|, so the sum of squares is exact to
// far below the 1e-4 trajectory bar (the expanded form
// would lose ~4 digits; this one does not).
//
// Operands (prepared by re_split_kernel from the fp64 column-major state):
//   A_hi, A_lo   d_pad x KR fp32 row-major -> tensor memory (lane = tile row,
//                column = k), loaded once per work unit by the epilogue warps;
//   Bt_hi, Bt_lo KR x n_pad fp32 row-major -> MN-major SMEM operand by TMA
//                (the layout of the X contractions' S operand, xstream_tc.cu);
//   X            TMA boxes of 32 columns x 128 rows, SWIZZLE_128B.
// Warp roles (192 threads): 0-3 epilogue + A loader, 4 TMA producer, 5 MMA
// issuer (+ TMEM allocation).  Persistent CTAs walk (row tile, column chunk)
// units; per-CTA fp64 partials are reduced in a fixed order (deterministic).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace cnmf {
namespace {

using namespace tc;

constexpr int kM = 128;           // tile rows (MMA M, TMEM lanes)
constexpr int kN = 64;            // tile columns (MMA N)
constexpr int kThreadsRE = 192;   // warps 0-3 epilogue, 4 TMA, 5 MMA
constexpr int kWarpTMA = 4, kWarpMMA = 5;
constexpr int kXS = 3;            // X stages
constexpr int kBS = 2;            // B stages
constexpr uint32_t kXBytes = kM * kN * 4;  // 32 KB: two 16 KB boxes of 32 columns

struct ReArgs {
  int64_t d, n;
  const float* ahi;  // d_pad x KR
  const float* alo;
  int kr;            // K padded to a multiple of 8 (<= 128)
  int nks;           // MMA k-steps = kr / 8
  int ntr;           // row tiles
  int nct;           // column tiles (of kN)
  int nchunks;       // column chunks per row tile
  double* part;      // [gridDim.x]
};

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float (&v)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
      : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&h)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(h[0]), "=r"(h[1]), "=r"(h[2]), "=r"(h[3]), "=r"(h[4]), "=r"(h[5]), "=r"(h[6]),
        "=r"(h[7]), "=r"(h[8]), "=r"(h[9]), "=r"(h[10]), "=r"(h[11]), "=r"(h[12]), "=r"(h[13]),
        "=r"(h[14]), "=r"(h[15]), "=r"(h[16]), "=r"(h[17]), "=r"(h[18]), "=r"(h[19]),
        "=r"(h[20]), "=r"(h[21]), "=r"(h[22]), "=r"(h[23]), "=r"(h[24]), "=r"(h[25]),
        "=r"(h[26]), "=r"(h[27]), "=r"(h[28]), "=r"(h[29]), "=r"(h[30]), "=r"(h[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(kThreadsRE, 1)
    recon_tc_kernel(const __grid_constant__ CUtensorMap map_x,
                    const __grid_constant__ CUtensorMap map_bh,
                    const __grid_constant__ CUtensorMap map_bl, const ReArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
  __shared__ __align__(8) uint64_t xfull[kXS], xempty[kXS], bfull[kBS], bempty[kBS];
  __shared__ __align__(8) uint64_t acc_full[2], acc_empty[2], a_ready;
  __shared__ uint32_t tmem_base;
  __shared__ double red[4];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kr = args.kr, nks = args.nks;
  const uint32_t atom_bytes = (uint32_t)kr * 128;     // one 32-column MN atom of KR K-rows
  const uint32_t bhalf = 2 * atom_bytes;              // b_hi (or b_lo) of a 64-column tile
  const uint32_t xoff = 0, boff = kXS * kXBytes;
  auto x_addr = [&](int s) { return sbase + xoff + s * kXBytes; };
  auto b_addr = [&](int b) { return sbase + boff + b * 2 * bhalf; };
  // two accumulator buffers of [main a_hi b_hi | corrections a_hi b_lo + a_lo b_hi]:
  // the tensor core's fp32 accumulation rounds toward zero, so the small
  // corrections get their own chain and the main chain is only nks long
  const uint32_t kAccCols = 4 * kN, a_hi_col = kAccCols, a_lo_col = kAccCols + kr;
  const uint32_t tmem_cols = (kAccCols + 2 * kr) <= 256 ? 256u : 512u;  // <= 512 for kr <= 128

  if (threadIdx.x == 0) {
    for (int s = 0; s < kXS; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], 4);
    }
    for (int s = 0; s < kBS; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&bempty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);
    }
    mbar_init(&a_ready, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == kWarpMMA) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;

  const int units = args.ntr * args.nchunks;
  const int per_chunk = (args.nct + args.nchunks - 1) / args.nchunks;
  // unit u: column chunk u / ntr, row tile u % ntr (CTAs running at the same
  // time sweep the same B tiles: L2 reuse)
  auto unit_cols = [&](int u, int& c0, int& c1) {
    const int ch = u / args.ntr;
    c0 = ch * per_chunk;
    c1 = min(args.nct, c0 + per_chunk);
  };
  auto tma = [&](uint32_t dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
  };

  double total = 0.0;
  if (warp == kWarpTMA) {
    if (lane == 0) {
      int s = 0, b = 0;
      uint32_t xph = 0, bph = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int c0, c1;
        unit_cols(u, c0, c1);
        const int row0 = (u % args.ntr) * kM;
        for (int ct = c0; ct < c1; ++ct) {
          const int col0 = ct * kN;
          mbar_wait(&bempty[b], bph ^ 1);
          mbar_expect_tx(&bfull[b], 2 * bhalf);
          tma(b_addr(b), &map_bh, &bfull[b], col0, 0);
          tma(b_addr(b) + atom_bytes, &map_bh, &bfull[b], col0 + 32, 0);
          tma(b_addr(b) + bhalf, &map_bl, &bfull[b], col0, 0);
          tma(b_addr(b) + bhalf + atom_bytes, &map_bl, &bfull[b], col0 + 32, 0);
          if (++b == kBS) {
            b = 0;
            bph ^= 1;
          }
          mbar_wait(&xempty[s], xph ^ 1);
          mbar_expect_tx(&xfull[s], kXBytes);
          tma(x_addr(s), &map_x, &xfull[s], col0, row0);
          tma(x_addr(s) + kXBytes / 2, &map_x, &xfull[s], col0 + 32, row0);
          if (++s == kXS) {
            s = 0;
            xph ^= 1;
          }
        }
      }
    }
  } else if (warp == kWarpMMA) {
    // per k-step: a_hi b_hi, a_hi b_lo, a_lo b_hi into one accumulator
    const uint32_t idesc = idesc_tf32(kN, false, true);
    int b = 0, ab = 0;
    uint32_t bph = 0, aph = 0, uph = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      int c0, c1;
      unit_cols(u, c0, c1);
      mbar_wait_warp(&a_ready, uph);  // this unit's A tile is in tensor memory
      uph ^= 1;
      for (int ct = c0; ct < c1; ++ct) {
        mbar_wait_warp(&acc_empty[ab], aph ^ 1);
        mbar_wait_warp(&bfull[b], bph);
        tc_fence_after();
        const uint32_t dcol = tmem + ab * 2 * kN;  // [main | corrections]
        const uint64_t bh = desc_mn(b_addr(b), atom_bytes);
        const uint64_t bl = desc_mn(b_addr(b) + bhalf, atom_bytes);
        for (int ks = 0; ks < nks; ++ks) {
          const uint64_t koff = (uint64_t)(ks * 1024 >> 4);
          const uint32_t acc = ks > 0 ? 1u : 0u;
          mma_ts_elect(dcol, tmem + a_hi_col + 8 * ks, bh + koff, idesc, acc);
          mma_ts_elect(dcol + kN, tmem + a_hi_col + 8 * ks, bl + koff, idesc, acc);
          mma_ts_elect(dcol + kN, tmem + a_lo_col + 8 * ks, bh + koff, idesc, 1u);
        }
        commit_elect(&bempty[b]);
        commit_elect(&acc_full[ab]);
        if (++b == kBS) {
          b = 0;
          bph ^= 1;
        }
        if (++ab == 2) {
          ab = 0;
          aph ^= 1;
        }
      }
    }
  } else {
    // ---------------- epilogue warps 0..3 (tile rows 32 q .. 32 q + 31) -------
    const int q = warp, r = 32 * q + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(32 * q) << 16);
    int s = 0, ab = 0;
    uint32_t xph = 0, aph = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      int c0, c1;
      unit_cols(u, c0, c1);
      // A tile rows -> tensor memory (a_hi | a_lo).  Every MMA of the
      // previous unit has completed: its last accumulator was consumed below.
      {
        const int64_t row = (int64_t)(u % args.ntr) * kM + r;
        const float4* ph = reinterpret_cast<const float4*>(args.ahi + row * kr);
        const float4* pl = reinterpret_cast<const float4*>(args.alo + row * kr);
        for (int c = 0; c < kr; c += 8) {
          float vh[8], vl[8];
          const float4 h0 = __ldg(ph + c / 4), h1 = __ldg(ph + c / 4 + 1);
          const float4 l0 = __ldg(pl + c / 4), l1 = __ldg(pl + c / 4 + 1);
          vh[0] = h0.x; vh[1] = h0.y; vh[2] = h0.z; vh[3] = h0.w;
          vh[4] = h1.x; vh[5] = h1.y; vh[6] = h1.z; vh[7] = h1.w;
          vl[0] = l0.x; vl[1] = l0.y; vl[2] = l0.z; vl[3] = l0.w;
          vl[4] = l1.x; vl[5] = l1.y; vl[6] = l1.z; vl[7] = l1.w;
          tmem_st8(lane_base + a_hi_col + c, vh);
          tmem_st8(lane_base + a_lo_col + c, vl);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_ready);
      }
      for (int ct = c0; ct < c1; ++ct) {
        mbar_wait_warp(&acc_full[ab], aph);
        mbar_wait_warp(&xfull[s], xph);
        tc_fence_after();
        double t0 = 0.0, t1 = 0.0;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t p[32], pc[32];
          tmem_ld32(lane_base + ab * 2 * kN + 32 * hh, p);
          tmem_ld32(lane_base + ab * 2 * kN + kN + 32 * hh, pc);
#pragma unroll
          for (int j = 0; j < 32; ++j)
            p[j] = __float_as_uint(__uint_as_float(p[j]) + __uint_as_float(pc[j]));
          // X box hh: row r is 128 B, 16 B chunk c at (c ^ (r & 7)) (SWIZZLE_128B)
          const uint32_t rowa = x_addr(s) + hh * (kXBytes / 2) + r * 128;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            float4 xv;
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                         : "=f"(xv.x), "=f"(xv.y), "=f"(xv.z), "=f"(xv.w)
                         : "r"(rowa + ((c ^ (r & 7)) << 4))
                         : "memory");
            const float e0 = xv.x - __uint_as_float(p[4 * c]);
            const float e1 = xv.y - __uint_as_float(p[4 * c + 1]);
            const float e2 = xv.z - __uint_as_float(p[4 * c + 2]);
            const float e3 = xv.w - __uint_as_float(p[4 * c + 3]);
            t0 = fma((double)e0, (double)e0, t0);
            t1 = fma((double)e1, (double)e1, t1);
            t0 = fma((double)e2, (double)e2, t0);
            t1 = fma((double)e3, (double)e3, t1);
          }
        }
        total += t0 + t1;
        // the X stage may be refilled only after its values were consumed
        // (an mbarrier arrive does not wait for in-flight shared loads)
        asm volatile("" ::"d"(t0), "d"(t1));
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&acc_empty[ab]);
          mbar_arrive(&xempty[s]);
        }
        if (++ab == 2) {
          ab = 0;
          aph ^= 1;
        }
        if (++s == kXS) {
          s = 0;
          xph ^= 1;
        }
      }
    }
  }
  // fixed-order CTA sum: lanes (butterfly), then the four epilogue warps
  if (warp < 4) {
    total = warp_sum(total);
    if (lane == 0) red[warp] = total;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) args.part[blockIdx.x] = (red[0] + red[1]) + (red[2] + red[3]);
  if (warp == kWarpMMA) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(tmem_cols));
  }
}

// fp64 column-major factors -> the 3xTF32 operands: A_hi/A_lo (d_pad x kr,
// row-major) and Bt_hi/Bt_lo (kr x n_pad, row-major), zero padded.
__global__ void re_split_kernel(const double* __restrict__ a_cm, const double* __restrict__ b_cm,
                                int64_t d, int64_t n, int k, int kr, int64_t d_pad, int64_t n_pad,
                                float* __restrict__ ahi, float* __restrict__ alo,
                                float* __restrict__ bhi, float* __restrict__ blo) {
  const int64_t na = d_pad * kr, total = na + (int64_t)kr * n_pad;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    float* dh;
    float* dl;
    int64_t o;
    if (e < na) {  // e = c * d_pad + i (coalesced reads of column c)
      const int64_t c = e / d_pad, i = e - c * d_pad;
      if (c < k && i < d) v = a_cm[c * d + i];
      dh = ahi;
      dl = alo;
      o = i * kr + c;
    } else {
      const int64_t f = e - na, c = f / n_pad, j = f - c * n_pad;
      if (c < k && j < n) v = b_cm[c * n + j];
      dh = bhi;
      dl = blo;
      o = f;
    }
    const float hi = __uint_as_float(rna_tf32_bits((float)v));
    const float lo = __uint_as_float(rna_tf32_bits((float)(v - (double)hi)));
    dh[o] = hi;
    dl[o] = lo;
  }
}

__global__ void re_sum_kernel(const double* __restrict__ part, int count, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < count; ++i) s += part[i];
    *out = 0.5 * s;
  }
}

}  // namespace

size_t recon_tc_ws_bytes(int64_t d, int64_t n, int k, int nsm) {
  const int64_t kr = (k + 7) & ~7;
  const int64_t d_pad = (d + kM - 1) / kM * kM, n_pad = (n + kN - 1) / kN * kN;
  return sizeof(float) * 2 * (d_pad * kr + kr * n_pad) + sizeof(double) * (nsm + 64) + 256;
}

bool launch_recon_tc(const float* x, int64_t ldx, int64_t d, int64_t n, const double* a_cm,
                     const double* b_cm, int k, double* out, void* ws, int nsm, cudaStream_t st) {
  if (k < 1 || k > 128 || (ldx % 4) != 0 || (reinterpret_cast<uintptr_t>(x) & 15)) {
    if (std::getenv("CNMF_RECON_DEBUG")) std::fprintf(stderr, "recon_tc: shape not taken\n");
    return false;
  }
  const int kr = (k + 7) & ~7;
  const int64_t d_pad = (d + kM - 1) / kM * kM, n_pad = (n + kN - 1) / kN * kN;
  float* ahi = static_cast<float*>(ws);
  float* alo = ahi + d_pad * kr;
  float* bhi = alo + d_pad * kr;
  float* blo = bhi + (int64_t)kr * n_pad;
  double* part = reinterpret_cast<double*>(
      (reinterpret_cast<uintptr_t>(blo + (int64_t)kr * n_pad) + 255) & ~uintptr_t(255));
  const int64_t tot = (d_pad + n_pad) * kr;
  if (std::getenv("CNMF_RECON_DEBUG")) {
    const cudaError_t e0 = cudaGetLastError();
    if (e0 != cudaSuccess) std::fprintf(stderr, "recon_tc: pending error %s\n", cudaGetErrorString(e0));
  }
  note_launches(1);
  re_split_kernel<<<(int)std::min<int64_t>((tot + 255) / 256, (int64_t)nsm * 8), 256, 0, st>>>(
      a_cm, b_cm, d, n, k, kr, d_pad, n_pad, ahi, alo, bhi, blo);
  CUtensorMap mx, mh, ml;
  bool ok = make_map(&mx, x, d, n, ldx, 32, kM, CU_TENSOR_MAP_SWIZZLE_128B) &&
            make_map(&mh, bhi, kr, n_pad, n_pad, 32, kr, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) &&
            make_map(&ml, blo, kr, n_pad, n_pad, 32, kr, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  if (!ok) {
    if (std::getenv("CNMF_RECON_DEBUG")) std::fprintf(stderr, "recon_tc: tensor map encode failed\n");
    return false;
  }
  ReArgs a;
  a.d = d;
  a.n = n;
  a.ahi = ahi;
  a.alo = alo;
  a.kr = kr;
  a.nks = kr / 8;
  a.ntr = (int)(d_pad / kM);
  a.nct = (int)(n_pad / kN);
  // enough units for ~8 per SM (load balance), at least 4 column tiles each
  int nch = 1;
  while ((int64_t)a.ntr * nch < (int64_t)nsm * 8 && a.nct / (nch * 2) >= 4) nch *= 2;
  a.nchunks = nch;
  a.part = part;
  const int units = a.ntr * a.nchunks;
  const int grid = std::min(units, nsm);
  // X stages + B stages of (b_hi | b_lo) x two 32-column atoms of kr K-rows
  const int smem = (int)(kXS * kXBytes + kBS * 2 * 2 * (uint32_t)kr * 128 + 1024);
  // per call: the attribute is per device, and cheap to set
  if (cudaFuncSetAttribute(recon_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
      cudaSuccess)
    return false;
  note_launches(1);
  recon_tc_kernel<<<grid, kThreadsRE, smem, st>>>(mx, mh, ml, a);
  if (const cudaError_t e = cudaGetLastError(); e != cudaSuccess) {
    if (std::getenv("CNMF_RECON_DEBUG"))
    {
      cudaFuncAttributes fa{};
      cudaFuncGetAttributes(&fa, recon_tc_kernel);
      int occ = -1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, recon_tc_kernel, kThreadsRE, smem);
      std::fprintf(stderr,
                   "recon_tc: launch failed: %s (grid %d smem %d kr %d units %d; maxdyn %d "
                   "static %zu regs %d occ %d)\n",
                   cudaGetErrorString(e), grid, smem, kr, units, fa.maxDynamicSharedSizeBytes,
                   fa.sharedSizeBytes, fa.numRegs, occ);
    }
    return false;
  }
  note_launches(1);
  re_sum_kernel<<<1, 32, 0, st>>>(part, grid, out);
  return true;
}

}  // namespace cnmf
