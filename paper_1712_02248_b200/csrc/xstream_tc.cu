// xstream_tc.cu -- the X-streaming contractions on the 5th-generation tensor
// cores (tcgen05, kind::tf32, 3xTF32 split, accumulators in TMEM, operands
// staged by TMA).
//
// Reference call sites: dense matmul NN (proj/src/matrix.cpp:105-116) and TN
// (129-140) from range_finder_impl / compress_left / compress_right
// (proj/src/compression.cpp:23-84).  Same contract as xstream.cu:
//   NN  Y (m x lp) = X (m x n) S (n x lp)     A = X tile, K-major (SW128)
//   TN  Z (n x lp) = X^T T (m x lp)           A = X tile, MN-major (SW128)
// B (S or T, row-major K x lp) is always an MN-major operand, so X is read by
// TMA exactly as stored -- no transposes anywhere.
//
// 3xTF32: x = x_hi + x_lo with x_hi = rna_tf32(x), x_lo = rna_tf32(x - x_hi),
// computed in shared memory by split warps (x_hi rewritten in place);
// s = s_hi + s_lo pre-split once per call.  Per k-step two MMAs:
//   D[:, 0:2L] += x_hi * [s_hi | s_lo]      (N = 2L, one read of x_hi)
//   D[:, 0:L]  += x_lo * s_hi
// and the epilogue adds D[:, 0:L] + D[:, L:2L].  fp32 accumulation in TMEM.
//
// Warp roles (320 threads): warps 0..3 epilogue (TMEM -> registers ->
// global), warp 4 TMA producer, warp 5 MMA issuer (also allocates TMEM),
// warps 6..9 split x_hi / x_lo.  Persistent CTAs walk (tile, k-split) units.
// The tensor core's fp32 accumulation error grows with the chain length, so
// every 4 K-blocks (16 k-steps) the accumulator is drained into per-row fp32
// running sums in the epilogue's registers while the second TMEM buffer
// takes the next chunk.  Split-K partials are reduced in a fixed order.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <string>
#include <utility>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace cnmf {

namespace {

using namespace tc;

constexpr int kBM = 128;     // output rows per unit (MMA M)
constexpr int kBK = 32;      // K elements per stage (4 MMA k-steps of 8)
constexpr int kThreadsTC = 352;  // warps 0-3 epilogue, 4 X TMA, 5 MMA, 6-9 split, 10 S TMA
constexpr int kWarpTMA = 4, kWarpMMA = 5, kWarpSplit0 = 6, kWarpBTMA = 10;
#ifdef TC_DRAIN
constexpr int kDrain = TC_DRAIN;
#else
constexpr int kDrain = 4;         // K-blocks per drain (16 k-steps x 3 MMAs per accumulation chain)
#endif
// The fp16 path drains every K-block: its K = 16 MMAs grow the accumulation
// error faster (tools/f16_accuracy.py); with drains every 2 / 4 blocks the C2
// trajectory with forced fp16 deviates 1.3e-4 / 2.6e-4 from the reference,
// every block 1e-5 (tests/test_gpu_f16.py), at ~8% of the fp16 speed-up.
#ifdef TC_DRAIN16
constexpr int kDrain16 = TC_DRAIN16;
#else
constexpr int kDrain16 = 4;
#endif
constexpr int kXBytes = kBM * kBK * 4;  // 16 KB per stage (x_hi), same for x_lo

// Operand splits of the X-stream kernel:
//   kTF32  3xTF32: x = x_hi + x_lo (tf32, 22 of fp32's 24 bits), 3 products;
//   kF16   fp16 hi / lo with power-of-two row / column scaling (opt-in);
//   kBF9   BF16x9: x = x0 + x1 + x2 and s = s0 + s1 + s2 in bf16 -- EXACT
//          for fp32 (8 + 8 + 8 significant bits, fp32's exponent range, no
//          scaling) -- and all nine products, so the only rounding is the
//          fp32 accumulation.  The 3xTF32 split drops x's last two bits:
//          to the range finder that is a perturbation of the DATA (d X S
//          with d X ~ 2^-23 |X| entrywise, structured like X), which moves
//          the noise-level singular subspaces the sketch resolves; at C3 it
//          left the range finder's basis ~1e-4 from the reference's span and
//          the FastHALS-RP trajectory 5e-4 from the reference's
//          (tools/proj_swap.py: fp64 projectors with this kernel's own
//          views track it within 8e-6).  Rounding S only re-draws the sketch
//          (harmless), so x's exactness is what matters.
//          The x0 s0 products accumulate in their own chain (L <= 96), so the
//          small terms are not rounded against the large ones.
//   kX1    X exact in tf32 (every element's low 13 mantissa bits zero, e.g.
//          count data: check_data / launch_x_tf32_exact decide per X): x_lo
//          = 0, so 3xTF32 reduces to x s_hi + x s_lo -- the same products,
//          here summed in two accumulator chains (x s_hi and x s_lo apart,
//          added in the epilogue) -- and the MMA reads X straight from the
//          TMA stage (both operands from shared memory, no split warps, no
//          tensor-memory operand stores: the limiter of the kTF32 kernel,
//          DESIGN 3.1).
constexpr int kTF32 = 0, kF16 = 1, kBF9 = 2, kX1 = 3;

// Instruction descriptor: kind::f16 with fp16 A and B, fp32 accumulate,
// M = 128 (layouts checked by tools/tc_f16_check.cu); bf16 sets the A / B
// type fields (bits 7 and 10).
__host__ __device__ constexpr uint32_t idesc_f16(int n, bool b_mn, bool bf16 = false) {
  return (1u << 4) | (bf16 ? (1u << 7) | (1u << 10) : 0u) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
}
__device__ __forceinline__ void mma16_ts_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "{\n\t.reg .u32 ln;\n\tmov.u32 ln, %%laneid;\n\tsetp.eq.u32 e, ln, 0;\n\t}\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// 2^e as a float, e in [-126, 127]
__device__ __forceinline__ float exp2i(int e) { return __int_as_float((127 + e) << 23); }

struct TcArgs {
  int64_t rows_out;  // output rows (m for NN, n for TN)
  int64_t kdim;      // reduction length (n for NN, m for TN)
  int64_t kchunk;    // K per split (multiple of kBK)
  int ntiles, nsplit, lp;
  float* out;        // [nsplit][rows_out][lp] or the final output when nsplit == 1
  float* dbg;        // optional debug dump (tools/tc_debug.cu), null in production
  int nmma;          // MMA N = lp rounded up to 16 (<= L): padding columns are not computed
  // fp16 path only: per-row exponents of X (NN: output rows; TN: the K index),
  // applied as exact 2^e scalings, and the per-output-column unscale factors
  const int8_t* rexp;
  const float* cscale;
};


// Shared-memory rings: X stages (TMA -> split warps) and S stages (TMA ->
// MMA: s_hi | s_lo).  The split warps write x_hi / x_lo straight into tensor
// memory (tcgen05.st), and the MMA reads its A operand from there, so X costs
// one TMA write plus one LDS pass of shared-memory bandwidth (the v2 kernel's
// shared-memory operand slots cost four more and made it smem-bound).  An X
// stage is released as soon as the split warps have read it.
template <int L, int kMode = kTF32> struct TcRings {
  // fp16 / bf16 S stages are LH halves wide: 64-element SWIZZLE_128B atoms
  static constexpr bool kHalf = kMode == kF16 || kMode == kBF9;
  static constexpr int LH = (L + 63) & ~63;
  static constexpr int kBBytes = kHalf ? kBK * LH * 2 : kBK * L * 4;  // one S piece per K-block
  static constexpr int kPieces = kMode == kBF9 ? 3 : 2;               // S pieces per stage
  static constexpr int kBudget = 225 * 1024;
  // Both operands arrive with ~1.5-2k cycles of latency (X from HBM, S from
  // L2, re-requested only when a stage frees), so the budget is split to keep
  // several K-blocks of each in flight.
#ifdef TC_XSTAGES
  static constexpr int kXStages = TC_XSTAGES;
#else
  static constexpr int kXStages = kMode == kX1 ? (L <= 64 ? 8 : (L <= 96 ? 6 : 5))
                                               : (L <= 32 ? 8 : (L <= 64 ? 6 : (L <= 96 ? 5 : 4)));
#endif
  static constexpr int kBFit = (kBudget - kXStages * kXBytes) / (kPieces * kBBytes);
#ifdef TC_BSTAGES
  static constexpr int kBStages = TC_BSTAGES;
#else
  static constexpr int kBStages = kBFit > 8 ? 8 : kBFit;
#endif
  static constexpr int kXOff = 0;
  static constexpr int kBOff = kXStages * kXBytes;
  static constexpr int kBytes = kBOff + kBStages * kPieces * kBBytes;
  // Tensor memory: two accumulator buffers of L columns (double-buffered
  // drain), then the A slots of 64 columns (x_hi: 32, x_lo: 32; lane = tile
  // row, column = k).
  // fp16: the small correction products (x_hi s_lo + x_lo s_hi) accumulate
  // in a second accumulator, so the big one's rounding cannot swamp them;
  // the epilogue folds the two (L <= 96: 2 x 2L accumulator columns + 4
  // operand slots of 32 fill the 512 TMEM columns)
  // kX1 issues x [s_hi | s_lo] as ONE N = L + nmma MMA per k-step: with both
  // operands in shared memory the MMAs are bound by shared-memory reads (4 KB
  // of A + 4 KB of B per N = 128 k-step, i.e. the SM's 128 B/clk for its 64
  // cycles), and the merged MMA reads x once for both products (C4: NN 70.8 ->
  // 77.6%, TN 71.0 -> 77.4% of HBM).  The two products land in separate
  // accumulator columns (all 512 TMEM columns at L = 128) and the epilogue
  // adds them.  -DTC_X1_NOMERGE keeps the two-MMA form (comparisons).
#ifdef TC_X1_NOMERGE
  static constexpr bool kMerge = false;
#else
  static constexpr bool kMerge = kMode == kX1;
#endif
  static constexpr int kChains = kMode == kF16 ? 2 : ((kMode == kBF9 && L <= 96) || kMerge ? 2 : 1);
  static constexpr int kAccCols = kChains * L;
  static constexpr int kAOff = 2 * kAccCols;
  // A operand slot per K-block: tf32 x_hi | x_lo 32 + 32 columns; fp16 two
  // halves per column, 16 + 16
  // bf16x3: three halves-pairs of 16 columns
  static constexpr int kASlot = kMode == kF16 ? 32 : (kMode == kBF9 ? 48 : 64);
  static constexpr int kOpFit = (512 - kAOff) / kASlot;
#ifdef TC_OPSTAGES
  static constexpr int kOpStages = TC_OPSTAGES;
#else
  static constexpr int kOpStages = kOpFit > 4 ? 4 : (kOpFit < 1 ? 1 : kOpFit);  // kX1 uses none
#endif
  static constexpr uint32_t kTmemNeed = kAOff + (kMode == kX1 ? 0 : kOpStages * kASlot);
  static constexpr uint32_t kTmemCols =
      kTmemNeed <= 32 ? 32 : (kTmemNeed <= 64 ? 64 : (kTmemNeed <= 128 ? 128 : (kTmemNeed <= 256 ? 256 : 512)));
};

__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a)
               : "memory");  // must not sink below the mbarrier arrive that frees the stage
  return v;
}
__device__ __forceinline__ float lds32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
// TC_TRACE builds (tools only): per-K-block event times of CTA 0 into args.dbg
// as uint64 [event][block]: 0 X issue, 1 split got X, 2 split got A slot,
// 3 split done, 4 MMA got operands, 5 MMA issued, 6 S issue, 7 MMA got A slot.
#ifdef TC_TRACE
#define TC_EV(ev, blk)                                                              \
  do {                                                                              \
    const int blk_ = (blk);                                                         \
    if (blockIdx.x == 0 && args.dbg && blk_ < 4096)                                 \
      reinterpret_cast<unsigned long long*>(args.dbg)[(ev) * 4096 + blk_] = clock64(); \
  } while (0)
#else
#define TC_EV(ev, blk) \
  do {                 \
  } while (0)
#endif

template <bool kTN, int L, int kMode>  // L = padded width (multiple of 32, <= 128)
__global__ void __launch_bounds__(kThreadsTC, 1)
    xs_tc_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_bh,
                 const __grid_constant__ CUtensorMap map_bl, const __grid_constant__ CUtensorMap map_b2,
                 const TcArgs args) {
  using R = TcRings<L, kMode>;
  constexpr bool kIsF16 = kMode == kF16, kIsBF9 = kMode == kBF9, kIsX1 = kMode == kX1;
  constexpr int kDr = kIsF16 ? kDrain16 : kDrain;  // K-blocks per accumulator drain
  constexpr int kSX = R::kXStages, kSO = R::kOpStages, kSB = R::kBStages;
  constexpr uint32_t kTmemCols = R::kTmemCols;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
  __shared__ __align__(8) uint64_t xfull[kSX], xempty[kSX], opready[kSO], opempty[kSO];
  __shared__ __align__(8) uint64_t bfull[kSB], bempty[kSB], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSX; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], kIsX1 ? 1 : 4);  // kX1: released by the MMA commit
    }
    for (int s = 0; s < kSO; ++s) {
      mbar_init(&opready[s], 4);
      mbar_init(&opempty[s], 1);
    }
    for (int s = 0; s < kSB; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&bempty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == kWarpMMA) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;

  const int units = args.ntiles * args.nsplit;
  auto x_addr = [&](int s) { return sbase + R::kXOff + s * kXBytes; };
  auto b_addr = [&](int b) { return sbase + R::kBOff + b * R::kPieces * R::kBBytes; };  // [s_hi | s_lo (| s2)]
  auto unit_k = [&](int u, int64_t& k0, int64_t& k1) {
    const int split = u / args.ntiles;
    k0 = (int64_t)split * args.kchunk;
    k1 = min(args.kdim, k0 + args.kchunk);
  };
  auto tma = [&](uint32_t dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
  };

  if (warp == kWarpTMA) {
    // ---------------- X producer ----------------
    // NN: one 32 (k) x 128 (rows) box, SWIZZLE_128B (conflict-free row reads;
    // for kX1 the K-major SW128 A operand as it stands);
    // TN: one 128 (rows of Z = columns of X) x 32 (k) box, no swizzle; kX1:
    // four 32 x 32 boxes in the MN-major SW128/32 B-atom operand layout (the
    // same as S's).
    if (lane == 0) {
      int nblk = 0;
      int s = 0;
      uint32_t ph = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int64_t k0, k1;
        unit_k(u, k0, k1);
        const int row0 = (u % args.ntiles) * kBM;
        for (int64_t kk = k0; kk < k1; kk += kBK) {
          mbar_wait(&xempty[s], ph ^ 1);
          TC_EV(0, nblk++);
          mbar_expect_tx(&xfull[s], kXBytes);
          if (!kTN) {
            tma(x_addr(s), &map_x, &xfull[s], (int)kk, row0);
          } else if constexpr (kIsX1) {
#pragma unroll
            for (int a = 0; a < kBM / 32; ++a)
              tma(x_addr(s) + a * (kBK * 128), &map_x, &xfull[s], row0 + 32 * a, (int)kk);
          } else {
            tma(x_addr(s), &map_x, &xfull[s], row0, (int)kk);
          }
          if (++s == kSX) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == kWarpBTMA) {
    // ---------------- S producer (L2-resident small operand) ----------------
    // This kernel is a programmatic dependent launch behind the S split
    // kernel: everything else (TMEM, barriers, the X stream into the ring and
    // the X splits) starts while the split runs; only S waits for it.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (lane == 0) {
      int nblk = 0;
      int b = 0;
      uint32_t ph = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int64_t k0, k1;
        unit_k(u, k0, k1);
        for (int64_t kk = k0; kk < k1; kk += kBK) {
          mbar_wait(&bempty[b], ph ^ 1);
          TC_EV(6, nblk++);
          mbar_expect_tx(&bfull[b], R::kPieces * R::kBBytes);
          if constexpr (R::kHalf) {  // 64-half atoms of 32 K-rows x 128 B
#pragma unroll
            for (int a = 0; a < R::LH / 64; ++a) {
              tma(b_addr(b) + a * (kBK * 128), &map_bh, &bfull[b], 64 * a, (int)kk);
              tma(b_addr(b) + (R::LH / 64 + a) * (kBK * 128), &map_bl, &bfull[b], 64 * a, (int)kk);
              if constexpr (kIsBF9)
                tma(b_addr(b) + (2 * (R::LH / 64) + a) * (kBK * 128), &map_b2, &bfull[b], 64 * a, (int)kk);
            }
          } else {
#pragma unroll
            for (int a = 0; a < L / 32; ++a) {
              tma(b_addr(b) + a * (kBK * 128), &map_bh, &bfull[b], 32 * a, (int)kk);
              tma(b_addr(b) + (L / 32 + a) * (kBK * 128), &map_bl, &bfull[b], 32 * a, (int)kk);
            }
          }
          if (++b == kSB) {
            b = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == kWarpMMA) {
    // ---------------- MMA issuer ----------------
    // Per k-step three MMAs into one accumulator: x_hi s_hi, x_hi s_lo,
    // x_lo s_hi (A from tensor memory).  Every kDrain K-blocks the
    // accumulator goes to the epilogue (which sums the chunks in registers)
    // and the other buffer takes over: the tensor core's fp32 accumulation
    // error grows with the chain length (tools/tc_precision.py).
    {  // the whole warp walks the schedule; the elected leader issues
      int nblk = 0;
      const uint32_t idesc = idesc_tf32(args.nmma, false, true);
      constexpr uint32_t kLoOff = (L / 32) * (kBK * 128);
      int o = 0, b = 0, ab = 0, xs = 0;
      uint32_t oph = 0, bph = 0, aph = 0, xph = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int64_t k0, k1;
        unit_k(u, k0, k1);
        for (int64_t g0 = k0; g0 < k1; g0 += (int64_t)kDr * kBK) {
          const int64_t g1 = min(k1, g0 + (int64_t)kDr * kBK);
          mbar_wait_warp(&acc_empty[ab], aph ^ 1);
          tc_fence_after();
          const uint32_t d = tmem + ab * R::kAccCols;
          uint32_t acc = 0;
          for (int64_t kk = g0; kk < g1; kk += kBK) {
            if constexpr (kIsX1) {
              // X straight from its TMA stage: x s_hi then x s_lo per k-step
              // (kTF32's order with its zero x_lo s_hi product dropped).
              // K-major SW128 (NN): 8-row groups 1 KB apart, a k-step is 32 B
              // into the swizzle atom; MN-major (TN): as S.
              mbar_wait_warp(&xfull[xs], xph);
              mbar_wait_warp(&bfull[b], bph);
              if (lane == 0) TC_EV(4, nblk);
              tc_fence_after();
              const uint32_t idx = idesc_tf32(args.nmma, kTN, true);
              const uint64_t ax = kTN ? desc_mn(x_addr(xs), kBK * 128) : smem_desc(x_addr(xs), 16, 1024, 2);
              const uint64_t bh = desc_mn(b_addr(b), kBK * 128);
              const uint64_t bl = desc_mn(b_addr(b) + kLoOff, kBK * 128);
#pragma unroll
              for (int ks = 0; ks < kBK / 8; ++ks) {
                const uint64_t koff = (uint64_t)(ks * 1024 >> 4);
                const uint64_t aoff = kTN ? koff : (uint64_t)(ks * 32 >> 4);
                if constexpr (R::kMerge) {
                  // s_hi's L columns and s_lo's atoms are contiguous in the stage:
                  // one N = L + nmma MMA, the two products in separate columns
                  mma_ss_elect(d, ax + aoff, bh + koff, idesc_tf32(L + args.nmma, kTN, true), acc);
                } else {
                  mma_ss_elect(d, ax + aoff, bh + koff, idx, acc);
                  mma_ss_elect(d, ax + aoff, bl + koff, idx, 1u);
                }
                acc = 1u;
              }
              commit_elect(&xempty[xs]);  // X stage and S stage free once these MMAs complete
              commit_elect(&bempty[b]);
              if (lane == 0) TC_EV(5, nblk);
              ++nblk;
              if (++xs == kSX) {
                xs = 0;
                xph ^= 1;
              }
              if (++b == kSB) {
                b = 0;
                bph ^= 1;
              }
              continue;
            }
            mbar_wait(&opready[o], oph);
            if (lane == 0) TC_EV(7, nblk);
            mbar_wait_warp(&bfull[b], bph);
            if (lane == 0) TC_EV(4, nblk);
            tc_fence_after();
            const uint32_t ahi = tmem + R::kAOff + R::kASlot * o;
            if constexpr (kIsBF9) {
              // two K = 16 steps of all nine products x_i s_j; A: 8 columns
              // (16 bf16) per step, x1 16 and x2 32 columns after x0; B pieces
              // kP bytes apart.  x0 s0 -> chain 0, the rest -> chain 1 (one
              // chain when L > 96: TMEM)
              constexpr uint32_t kP = (R::LH / 64) * (kBK * 128);
              const uint32_t idb = idesc_f16(args.nmma, true, true);
              const uint32_t dc = R::kChains == 2 ? d + L : d;
#pragma unroll
              for (int ks = 0; ks < kBK / 16; ++ks) {
                uint64_t bd[3];
#pragma unroll
                for (int j = 0; j < 3; ++j) bd[j] = smem_desc(b_addr(b) + j * kP + ks * 2048, kBK * 128, 1024, 2);
                const uint32_t a0 = ahi + 8 * ks, a1 = a0 + 16, a2 = a0 + 32;
                mma16_ts_elect(d, a0, bd[0], idb, acc);
                mma16_ts_elect(dc, a0, bd[1], idb, R::kChains == 2 ? acc : 1u);
                mma16_ts_elect(dc, a1, bd[0], idb, 1u);
                mma16_ts_elect(dc, a0, bd[2], idb, 1u);
                mma16_ts_elect(dc, a1, bd[1], idb, 1u);
                mma16_ts_elect(dc, a2, bd[0], idb, 1u);
                mma16_ts_elect(dc, a1, bd[2], idb, 1u);
                mma16_ts_elect(dc, a2, bd[1], idb, 1u);
                mma16_ts_elect(dc, a2, bd[2], idb, 1u);
                acc = 1u;
              }
            } else if constexpr (kIsF16) {
              // two K = 16 steps: x_hi s_hi, x_hi s_lo, x_lo s_hi; A: 8 columns
              // (16 halves) per step, x_lo 16 columns after x_hi; B: SWIZZLE_128B
              // MN-major, 8-row groups 1 KB apart, atoms kBK x 128 B apart
              constexpr uint32_t kLo16 = (R::LH / 64) * (kBK * 128);
              const uint32_t id16 = idesc_f16(args.nmma, true);
#pragma unroll
              for (int ks = 0; ks < kBK / 16; ++ks) {
                const uint64_t bh = smem_desc(b_addr(b) + ks * 2048, kBK * 128, 1024, 2);
                const uint64_t bl = smem_desc(b_addr(b) + kLo16 + ks * 2048, kBK * 128, 1024, 2);
                mma16_ts_elect(d, ahi + 8 * ks, bh, id16, acc);            // main
                mma16_ts_elect(d + L, ahi + 8 * ks, bl, id16, acc);        // corrections
                mma16_ts_elect(d + L, ahi + 16 + 8 * ks, bh, id16, 1u);
                acc = 1u;
              }
            } else {
            // descriptor address field is addr >> 4 in the low bits: k-step
            // offsets (1 KB) are added to the base descriptors directly
            const uint64_t bh = desc_mn(b_addr(b), kBK * 128);
            const uint64_t bl = desc_mn(b_addr(b) + kLoOff, kBK * 128);
#pragma unroll
            for (int ks = 0; ks < kBK / 8; ++ks) {
              const uint64_t koff = (uint64_t)(ks * 1024 >> 4);
              mma_ts_elect(d, ahi + 8 * ks, bh + koff, idesc, acc);
              mma_ts_elect(d, ahi + 8 * ks, bl + koff, idesc, 1u);
              mma_ts_elect(d, ahi + 32 + 8 * ks, bh + koff, idesc, 1u);
              acc = 1u;
            }
            }
            commit_elect(&opempty[o]);  // A slot and S stage free once these MMAs complete
            commit_elect(&bempty[b]);
            if (lane == 0) TC_EV(5, nblk);
            ++nblk;
            if (++o == kSO) {
              o = 0;
              oph ^= 1;
            }
            if (++b == kSB) {
              b = 0;
              bph ^= 1;
            }
          }
          commit_elect(&acc_full[ab]);
          if (++ab == 2) {
            ab = 0;
            aph ^= 1;
          }
        }
      }
    }
  } else if (!kIsX1 && warp >= kWarpSplit0 && warp < kWarpSplit0 + 4) {
    // ---------------- split warps: X stage -> (x_hi, x_lo) in tensor memory ----
    // Warp w may only access TMEM lanes 32 (w % 4) .. +31: it owns those tile
    // rows; each thread splits its row's 32 K values.
    const int q = warp & 3;
    const int r = 32 * q + lane;  // tile row (TMEM lane)
    int nblk = 0;
    int s = 0, o = 0;
    uint32_t xph = 0, oph = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      int64_t k0, k1;
      unit_k(u, k0, k1);
      float row_scale = 1.f;  // NN fp16: 2^e of this thread's X row
      int ecur[8], enxt[8];   // TN fp16: packed int8 exponents of the block's K rows
      // rexp is zero-padded to a multiple of 4 bytes past the rows (xs_rexp_bytes)
      auto load_e = [&](int64_t kb, int (&dst)[8]) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          dst[j] = kb + 4 * j < args.kdim ? __ldg(reinterpret_cast<const int*>(args.rexp + kb) + j) : 0;
      };
      if constexpr (kIsF16 && !kTN) {
        const int64_t row = (int64_t)(u % args.ntiles) * kBM + r;
        row_scale = row < args.rows_out ? exp2i(args.rexp[row]) : 1.f;
      }
      if constexpr (kIsF16 && kTN) load_e(k0, ecur);
      for (int64_t kk = k0; kk < k1; kk += kBK) {
        if constexpr (kIsF16 && kTN) {
          if (kk + kBK < k1) load_e(kk + kBK, enxt);
        }
        mbar_wait_warp(&xfull[s], xph);
        if (q == 0 && lane == 0) TC_EV(1, nblk);
        float v[32];
        if (!kTN) {  // SWIZZLE_128B K-major: 16 B chunk c of row r at chunk c ^ (r & 7)
          const uint32_t row = x_addr(s) + r * 128;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 t = lds128(row + ((c ^ (r & 7)) << 4));
            v[4 * c] = t.x;
            v[4 * c + 1] = t.y;
            v[4 * c + 2] = t.z;
            v[4 * c + 3] = t.w;
          }
        } else {  // unswizzled [k][128]: lanes read consecutive words
#pragma unroll
          for (int kq = 0; kq < 32; ++kq) v[kq] = lds32(x_addr(s) + kq * (kBM * 4) + r * 4);
        }
        uint32_t hi[32], lo[32];
        if constexpr (kIsBF9) {
          // exact three-way bf16 split: words 0..15 x0 pairs, 16..31 x1 pairs
          // (in hi), x2 pairs in lo[0..15] (even k in the low half)
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const __nv_bfloat162 p0 = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
            const float2 f0 = __bfloat1622float2(p0);
            const float r0 = v[2 * j] - f0.x, r1 = v[2 * j + 1] - f0.y;
            const __nv_bfloat162 p1 = __floats2bfloat162_rn(r0, r1);
            const float2 f1 = __bfloat1622float2(p1);
            const __nv_bfloat162 p2 = __floats2bfloat162_rn(r0 - f1.x, r1 - f1.y);
            hi[j] = *reinterpret_cast<const uint32_t*>(&p0);
            hi[16 + j] = *reinterpret_cast<const uint32_t*>(&p1);
            lo[j] = *reinterpret_cast<const uint32_t*>(&p2);
          }
        } else if constexpr (kIsF16) {
          // exact power-of-two scaling into fp16's normal range, then the
          // hi / lo fp16 split: words 0..15 = x_hi pairs, 16..31 = x_lo pairs
          // (even k in the low half)
          if constexpr (!kTN) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] *= row_scale;
          } else {
            // the block's 32 K-row exponents were loaded one block ahead
#pragma unroll
            for (int j = 0; j < 32; j += 4)
#pragma unroll
              for (int u = 0; u < 4; ++u) v[j + u] *= exp2i((int)(int8_t)(ecur[j >> 2] >> (8 * u)));
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const __half2 h = __floats2half2_rn(v[2 * j], v[2 * j + 1]);
            const float2 hf = __half22float2(h);
            const __half2 l2 = __floats2half2_rn(v[2 * j] - hf.x, v[2 * j + 1] - hf.y);
            hi[j] = *reinterpret_cast<const uint32_t*>(&h);
            hi[16 + j] = *reinterpret_cast<const uint32_t*>(&l2);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) tf32_split_bits(v[j], hi[j], lo[j]);
        }
        mbar_wait_warp(&opempty[o], oph ^ 1);
        if (q == 0 && lane == 0) TC_EV(2, nblk);
        tc_fence_after();
        {
          const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + R::kAOff + R::kASlot * o;
          if constexpr (kIsBF9) {
            tmem_st32(ta, hi);
            tmem_st16(ta + 32, lo);
          } else if constexpr (kIsF16) {
            tmem_st32(ta, hi);
          } else {
            tmem_st32(ta, hi);
            tmem_st32(ta + 32, lo);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&opready[o]);
        // The X stage is released only here, after tcgen05.st has consumed
        // the registers its values were loaded into: an mbarrier arrive does
        // not wait for in-flight ld.shared, and the compiler is free to sink
        // register arithmetic below it, so releasing right after the loads let
        // the next TMA overwrite rows before their last chunks were read
        // (tools/tc_units.cu found block b computed with block b + kXStages).
        if (lane == 0) mbar_arrive(&xempty[s]);
        if (q == 0 && lane == 0) TC_EV(3, nblk);
        if (lane == 0) TC_EV(8 + q, nblk);  // per-quarter split done (tools/tc_trace.cu)
        if constexpr (kIsF16 && kTN) {
#pragma unroll
          for (int j = 0; j < 8; ++j) ecur[j] = enxt[j];
        }
        ++nblk;
        if (++s == kSX) {
          s = 0;
          xph ^= 1;
        }
        if (++o == kSO) {
          o = 0;
          oph ^= 1;
        }
      }
    }
  } else if (warp < 4) {
    // ---------------- epilogue (warps 0..3): TMEM chunks -> registers -> global
    const int q = warp;  // TMEM lane quarter this warp may access
    int ab = 0;
    uint32_t aph = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      int64_t k0, k1;
      unit_k(u, k0, k1);
      const int tile = u % args.ntiles, split = u / args.ntiles;
#ifdef TC_EPI64  // experiment: fp64 running sums in the epilogue (spills; precision tests only)
      double run[L];
#else
      float run[L];
#endif
#pragma unroll
      for (int c = 0; c < L; ++c) run[c] = 0.f;
      for (int64_t g0 = k0; g0 < k1; g0 += (int64_t)kDr * kBK) {
        mbar_wait_warp(&acc_full[ab], aph);
        tc_fence_after();
        const uint32_t base = tmem + ab * R::kAccCols + ((uint32_t)(32 * q) << 16);
#pragma unroll
        for (int c = 0; c < R::kAccCols; c += 32) {
          uint32_t h[32];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
              "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
              : "=r"(h[0]), "=r"(h[1]), "=r"(h[2]), "=r"(h[3]), "=r"(h[4]), "=r"(h[5]), "=r"(h[6]),
                "=r"(h[7]), "=r"(h[8]), "=r"(h[9]), "=r"(h[10]), "=r"(h[11]), "=r"(h[12]),
                "=r"(h[13]), "=r"(h[14]), "=r"(h[15]), "=r"(h[16]), "=r"(h[17]), "=r"(h[18]),
                "=r"(h[19]), "=r"(h[20]), "=r"(h[21]), "=r"(h[22]), "=r"(h[23]), "=r"(h[24]),
                "=r"(h[25]), "=r"(h[26]), "=r"(h[27]), "=r"(h[28]), "=r"(h[29]), "=r"(h[30]),
                "=r"(h[31])
              : "r"(base + c));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 32; ++j) run[(c + j) % L] += __uint_as_float(h[j]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[ab]);
        if (++ab == 2) {
          ab = 0;
          aph ^= 1;
        }
      }
      const int64_t row = (int64_t)tile * kBM + 32 * q + lane;
      if (row < args.rows_out) {
        float* dst = args.out + ((int64_t)split * args.rows_out + row) * args.lp;
        if constexpr (kIsF16) {  // undo the power-of-two scalings (exact)
          const float rs = kTN ? 1.f : exp2i(-(int)args.rexp[row]);
#pragma unroll
          for (int c = 0; c < L; c += 4)
            if (c < args.lp) {
              const float4 cs = __ldg(reinterpret_cast<const float4*>(args.cscale + c));
              *reinterpret_cast<float4*>(dst + c) = make_float4(run[c] * rs * cs.x, run[c + 1] * rs * cs.y,
                                                                run[c + 2] * rs * cs.z, run[c + 3] * rs * cs.w);
            }
        } else {
#pragma unroll
          for (int c = 0; c < L; c += 4)
            if (c < args.lp)
              *reinterpret_cast<float4*>(dst + c) =
                  make_float4((float)run[c], (float)run[c + 1], (float)run[c + 2], (float)run[c + 3]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kWarpMMA) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTmemCols));
  }
}

// s (rows x lp) -> s_hi, s_lo (rows x L, zero padded): tf32 round-to-nearest
// split so the tensor core's truncation of the operands is exact.
__global__ void split_tf32_kernel(const float* __restrict__ s, int64_t rows, int lp, int L,
                                  float* __restrict__ hi, float* __restrict__ lo) {
  asm volatile("griddepcontrol.launch_dependents;");
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * L;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / L;
    const int c = (int)(e - r * L);
    const float v = c < lp ? s[r * lp + c] : 0.f;
    uint32_t h, l2;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(v));
    const float rem = v - __uint_as_float(h);
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l2) : "f"(rem));
    hi[e] = __uint_as_float(h);
    lo[e] = __uint_as_float(l2);
  }
}

// s (rows x lp) -> s0, s1, s2 bf16 (rows x LH, zero padded), s = s0 + s1 + s2
// exactly (BF16x9 path).  Triggers the dependent contraction at once.
__global__ void split_bf9_kernel(const float* __restrict__ s, int64_t rows, int lp, int LH,
                                 __nv_bfloat16* __restrict__ s0, __nv_bfloat16* __restrict__ s1,
                                 __nv_bfloat16* __restrict__ s2) {
  asm volatile("griddepcontrol.launch_dependents;");
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * LH;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / LH;
    const int c = (int)(e - r * LH);
    const float v = c < lp ? s[r * lp + c] : 0.f;
    const __nv_bfloat16 b0 = __float2bfloat16_rn(v);
    const float r1 = v - __bfloat162float(b0);
    const __nv_bfloat16 b1 = __float2bfloat16_rn(r1);
    s0[e] = b0;
    s1[e] = b1;
    s2[e] = __float2bfloat16_rn(r1 - __bfloat162float(b1));
  }
}

// fp16 path: per-column max |s'| of s' = s * 2^-rexp[row] (TN; s' = s for
// NN), as float bits (non-negative floats order like unsigned ints).
__global__ void s_colmax_kernel(const float* __restrict__ s, int64_t rows, int lp,
                                const int8_t* __restrict__ rexp, unsigned* __restrict__ cmax) {
  const int c = threadIdx.x;
  if (c >= lp) return;
  float m = 0.f;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    float v = fabsf(s[r * lp + c]);
    if (rexp) v *= exp2i(-(int)rexp[r]);
    m = fmaxf(m, v);
  }
  atomicMax(cmax + c, __float_as_uint(m));
}

// Column exponent f with max * 2^f in [2^14, 2^15) (fp16's normal range with
// one binade of headroom), clamped to the float exponent range.
__device__ __forceinline__ int col_exponent(unsigned bits) {
  if (bits == 0u) return 0;
  int e;
  frexpf(__uint_as_float(bits), &e);
  return max(-126, min(126, 15 - e));
}

// s' (rows x lp) -> s_hi, s_lo fp16 (rows x LH, zero padded), scaled by 2^f
// per column; cscale[c] = 2^-f.  Triggers the dependent contraction at once.
__global__ void split_f16_kernel(const float* __restrict__ s, int64_t rows, int lp, int LH,
                                 const int8_t* __restrict__ rexp, const unsigned* __restrict__ cmax,
                                 __half* __restrict__ hi, __half* __restrict__ lo,
                                 float* __restrict__ cscale) {
  asm volatile("griddepcontrol.launch_dependents;");
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * LH;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / LH;
    const int c = (int)(e - r * LH);
    float v = 0.f;
    if (c < lp) {
      v = s[r * lp + c];
      if (rexp) v *= exp2i(-(int)rexp[r]);
      v *= exp2i(col_exponent(cmax[c]));
    }
    const __half h = __float2half_rn(v);
    hi[e] = h;
    lo[e] = __float2half_rn(v - __half2float(h));
  }
  if (blockIdx.x == 0)
    for (int c = threadIdx.x; c < LH; c += blockDim.x)
      cscale[c] = c < lp ? exp2i(-col_exponent(cmax[c])) : 0.f;
}

// Per-row exponents of X for the fp16 path (NN rows / TN K index): row max
// scaled into [2^14, 2^15); `wide` is set when a row's smallest nonzero
// magnitude is below 2^-30 of its max (fp16's subnormal range would cost
// accuracy there: the caller then keeps the 3xTF32 path).
__global__ void x_rowexp_kernel(const float* __restrict__ x, int64_t ldx, int64_t d, int64_t n,
                                int8_t* __restrict__ rexp, int* __restrict__ wide) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < d; i += warps) {
    const float* row = x + i * ldx;
    float mx = 0.f, mn = INFINITY;
    for (int64_t j = lane; j < n; j += 32) {
      const float v = fabsf(__ldg(row + j));
      mx = fmaxf(mx, v);
      if (v > 0.f) mn = fminf(mn, v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    if (lane == 0) {
      rexp[i] = (int8_t)max(-126, min(126, mx > 0.f ? 15 - [&] { int e; frexpf(mx, &e); return e; }() : 0));
      if (mx > 0.f && mn < mx * 0x1.0p-30f) atomicOr(wide, 1);
    }
  }
}

__global__ void tc_split_reduce_kernel(const float4* __restrict__ part, int splits, int64_t total4,
                                       float4* __restrict__ out) {
  // programmatic dependent launch behind xs_tc_kernel: launched while its
  // last CTAs drain, reads the partials only once it has completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
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

float* g_tc_debug = nullptr;

struct TcPlan {
  int ntiles, nsplit;
  int64_t kchunk;
};

TcPlan tc_plan(int64_t rows_out, int64_t kdim, int nsm) {
  TcPlan p;
  p.ntiles = (int)((rows_out + kBM - 1) / kBM);
  const int64_t kblocks = (kdim + kBK - 1) / kBK;
  if (const char* e = std::getenv("CNMF_TC_KCHUNK")) {  // experiments only
    p.kchunk = std::max<int64_t>(kBK, (std::atoll(e) / kBK) * kBK);
    p.nsplit = (int)((kdim + p.kchunk - 1) / p.kchunk);
    return p;
  }
  // Choose the K-split count that minimises the makespan of the persistent
  // grid: ceil(units / G) rounds of ceil(kblocks / nsplit) K-blocks each, plus
  // the partial-output traffic of extra splits (write + reduce read, in
  // K-block equivalents: 128 rows x lp x 8 B per split vs 16 KB per K-block).
  int64_t best_ns = 1;
  double best = 1e300;
  for (int64_t ns = 1; ns <= std::min<int64_t>(64, kblocks); ++ns) {
    const int64_t per = (kblocks + ns - 1) / ns;
    const int64_t units = (int64_t)p.ntiles * ((kblocks + per - 1) / per);
    const int64_t rounds = (units + nsm - 1) / nsm;
    const double cost = (double)rounds * (double)per + (ns > 1 ? (double)ns * (double)p.ntiles / nsm * 4.5 : 0.0) + 2.0 * rounds;
    if (cost < best - 1e-9) {
      best = cost;
      best_ns = ns;
    }
  }
  const int64_t per = (kblocks + best_ns - 1) / best_ns;
  p.kchunk = per * kBK;
  p.nsplit = (int)((kdim + p.kchunk - 1) / p.kchunk);
  return p;
}

template <bool kTN, int L, int kMode>
cudaError_t run_tc(const CUtensorMap& mx, const CUtensorMap& mh, const CUtensorMap& ml,
                   const CUtensorMap& m2, const TcArgs& a, int grid, cudaStream_t st) {
  constexpr int smem = TcRings<L, kMode>::kBytes + 1024;
  static std::atomic<unsigned> attr{0u};
  smem_attr_once(attr, (const void*)(xs_tc_kernel<kTN, L, kMode>), smem);
  note_launches(1);
  return launch_pdl(xs_tc_kernel<kTN, L, kMode>, dim3(grid), dim3(kThreadsTC), (size_t)smem, st, mx,
                    mh, ml, m2, a);
}

}  // namespace

void xstream_tc_set_debug(float* dbg) { g_tc_debug = dbg; }

// floats per K row of the split S operand: tf32 hi + lo (2L), or three bf16
// pieces of LH halves (BF16x9)
static int64_t s_piece_floats(int L) {
  const int LH = (L + 63) & ~63;
  return std::max<int64_t>(2 * L, (3 * LH + 1) / 2);
}

size_t xstream_tc_ws_floats(int64_t m, int64_t n, int lp, int nsm) {
  const int L = (lp + 31) & ~31;
  const TcPlan a = tc_plan(m, n, nsm), b = tc_plan(n, m, nsm);
  const int64_t parts = std::max<int64_t>((int64_t)a.nsplit * m * lp, (int64_t)b.nsplit * n * lp);
  return (size_t)(parts + std::max(m, n) * s_piece_floats(L) + 512 + 64);
}

// The production operand split is 3xTF32: the kernel now serves the
// compressed views only (the range finder runs in fp64, engine.cpp), whose
// tf32-level error moves the C3 trajectory by < 1e-5 (tools/proj_swap.py).
// CNMF_XS=bf9 selects BF16x9 (1.9e-7 vs 9.8e-7 relative error at C3, but
// 46% / 40% of HBM at C3 / C4 against 66% / 58%), CNMF_XS=f16 the scaled
// fp16 path (rexp).
static int xs_tc_mode(const int8_t* rexp) {
  if (rexp) return kF16;
  static const int m = [] {
    const char* e = std::getenv("CNMF_XS");
    return (e && std::string(e) == "bf9") ? kBF9 : kTF32;
  }();
  return m;
}

// CNMF_XS_EXACT=0 keeps the three-product kernel for tf32-exact X
// (comparisons only: the results are bitwise the same).
static bool xs_exact_enabled() {
  const char* e = std::getenv("CNMF_XS_EXACT");
  return !(e && std::string(e) == "0");
}

// flag |= 1 when some element of X has a nonzero low 13 mantissa bits, i.e.
// is not exactly a tf32 value (kX1 needs every element exact).
__global__ void x_tf32_exact_kernel(const float* __restrict__ x, int64_t ldx, int64_t d, int64_t n,
                                    int* __restrict__ flag) {
  unsigned any = 0u;
  const int64_t n4 = n / 4;
  for (int64_t i = blockIdx.y; i < d; i += gridDim.y) {
    const float* row = x + i * ldx;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n4; c += (int64_t)gridDim.x * blockDim.x) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(row) + c);
      any |= v.x | v.y | v.z | v.w;
    }
    if (blockIdx.x == 0 && threadIdx.x < (n & 3)) any |= __float_as_uint(__ldg(row + 4 * n4 + threadIdx.x));
  }
  if (__syncthreads_or((any & 0x1FFFu) != 0u) && threadIdx.x == 0) atomicOr(flag, 1);
}

void launch_x_tf32_exact(const float* x, int64_t ldx, int64_t d, int64_t n, int* flag, int nsm,
                         cudaStream_t st) {
  if ((ldx % 4) != 0 || (reinterpret_cast<uintptr_t>(x) & 15)) {  // outside the kernel's envelope
    cudaMemsetAsync(flag, 0xFF, sizeof(int), st);
    return;
  }
  note_launches(1);
  const int gx = (int)std::max<int64_t>(1, std::min<int64_t>((n / 4 + 255) / 256, 8));
  const int gy = (int)std::max<int64_t>(1, std::min<int64_t>(d, (int64_t)nsm * 8 / gx));
  x_tf32_exact_kernel<<<dim3(gx, gy), 256, 0, st>>>(x, ldx, d, n, flag);
}

size_t xs_rexp_bytes(int64_t rows) { return (size_t)((rows + 3) / 4 * 4 + 64); }

void launch_x_rowexp(const float* x, int64_t ldx, int64_t d, int64_t n, int8_t* rexp, int* wide,
                     int nsm, cudaStream_t st) {
  cudaMemsetAsync(rexp, 0, xs_rexp_bytes(d), st);  // the padding must read as exponent 0
  note_launches(1);
  x_rowexp_kernel<<<(int)std::max<int64_t>(1, std::min<int64_t>((d + 7) / 8, (int64_t)nsm * 16)), 256,
                    0, st>>>(x, ldx, d, n, rexp, wide);
}

// rexp != nullptr selects the fp16 hi/lo path (per-row power-of-two scaling
// of X, per-column scaling of S): half the tensor-memory operand bytes and
// half the MMA time of 3xTF32 at the same 22-bit operand precision.
bool launch_xs_tc(bool tn, const float* x, int64_t ldx, int64_t m, int64_t n, const float* s,
                  int lp, float* out, float* ws, int nsm, cudaStream_t st, const int8_t* rexp,
                  bool x_exact) {
  const int L = (lp + 31) & ~31;
  if (L > 128 || (ldx % 4) != 0 || (reinterpret_cast<uintptr_t>(x) & 15)) return false;
  int mode = xs_tc_mode(rexp);
  if (mode == kF16 && L > 96) mode = kTF32;  // two accumulators fit TMEM up to L = 96
  if (mode == kTF32 && x_exact && xs_exact_enabled()) mode = kX1;
  const bool f16 = mode == kF16, bf9 = mode == kBF9, x1 = mode == kX1;
  const int LH = (L + 63) & ~63;
  const int64_t rows_out = tn ? n : m, kdim = tn ? m : n;
  const TcPlan p = tc_plan(rows_out, kdim, nsm);
  const int64_t pf = s_piece_floats(L);
  float* hi = ws;
  float* lo = ws + kdim * (int64_t)L;
  unsigned* cmax = reinterpret_cast<unsigned*>(ws + kdim * pf);
  float* cscale = ws + kdim * pf + 256;
  float* parts = ws + kdim * pf + 512;
  __half* hi16 = reinterpret_cast<__half*>(hi);
  __half* lo16 = reinterpret_cast<__half*>(lo);
  __nv_bfloat16* b16[3] = {reinterpret_cast<__nv_bfloat16*>(ws),
                           reinterpret_cast<__nv_bfloat16*>(ws) + kdim * LH,
                           reinterpret_cast<__nv_bfloat16*>(ws) + 2 * kdim * LH};
  if (bf9) {
    note_launches(1);
    split_bf9_kernel<<<std::min<int64_t>((kdim * LH + 255) / 256, nsm * 8), 256, 0, st>>>(
        s, kdim, lp, LH, b16[0], b16[1], b16[2]);
  } else if (f16) {
    if (cudaMemsetAsync(cmax, 0, sizeof(unsigned) * 128, st) != cudaSuccess) return false;
    note_launches(2);
    s_colmax_kernel<<<(int)std::max<int64_t>(1, std::min<int64_t>(kdim, (int64_t)nsm * 2)), 128, 0, st>>>(
        s, kdim, lp, tn ? rexp : nullptr, cmax);
    split_f16_kernel<<<std::min<int64_t>((kdim * LH + 255) / 256, nsm * 8), 256, 0, st>>>(
        s, kdim, lp, LH, tn ? rexp : nullptr, cmax, hi16, lo16, cscale);
  } else {
    note_launches(1);
    split_tf32_kernel<<<std::min<int64_t>((kdim * L + 255) / 256, nsm * 8), 256, 0, st>>>(
        s, kdim, lp, L, hi, lo);
  }
  CUtensorMap mx, mh, ml, m2;
  // X: NN boxes 32 (k) x 128 (rows), 128 B swizzle; TN boxes 128 x 32 (k), unswizzled.
  // S hi / lo: MN-major operand atoms: tf32 32 x 32 boxes, 128 B swizzle with
  // 32 B atoms; fp16 64 x 32 boxes, 128 B swizzle.
  // kX1 TN: 32 x 32 boxes in the MN-major operand layout (as S).
  bool ok = tn ? (x1 ? make_map(&mx, x, m, n, ldx, 32, kBK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)
                     : make_map(&mx, x, m, n, ldx, kBM, kBK, CU_TENSOR_MAP_SWIZZLE_NONE))
               : make_map(&mx, x, m, n, ldx, kBK, kBM, CU_TENSOR_MAP_SWIZZLE_128B);
  if (bf9)
    ok = ok && make_map(&mh, b16[0], kdim, LH, LH, 64, kBK, CU_TENSOR_MAP_SWIZZLE_128B, true) &&
         make_map(&ml, b16[1], kdim, LH, LH, 64, kBK, CU_TENSOR_MAP_SWIZZLE_128B, true) &&
         make_map(&m2, b16[2], kdim, LH, LH, 64, kBK, CU_TENSOR_MAP_SWIZZLE_128B, true);
  else if (f16)
    ok = ok && make_map(&mh, hi16, kdim, LH, LH, 64, kBK, CU_TENSOR_MAP_SWIZZLE_128B, true) &&
         make_map(&ml, lo16, kdim, LH, LH, 64, kBK, CU_TENSOR_MAP_SWIZZLE_128B, true);
  else
    ok = ok && make_map(&mh, hi, kdim, L, L, 32, kBK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) &&
         make_map(&ml, lo, kdim, L, L, 32, kBK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  if (!ok) return false;
  if (!bf9) m2 = mh;  // unused by the other modes
  TcArgs a;
  a.rows_out = rows_out;
  a.kdim = kdim;
  a.kchunk = p.kchunk;
  a.ntiles = p.ntiles;
  a.nsplit = p.nsplit;
  a.lp = lp;
  a.out = p.nsplit > 1 ? parts : out;
  a.dbg = g_tc_debug;
  a.nmma = (lp + 15) & ~15;
  a.rexp = rexp;
  a.cscale = cscale;
  const int units = p.ntiles * p.nsplit;
  const int grid = std::min(units, nsm);
  cudaError_t e;
#define XS_CASE(TN, LL)                                                                       \
  case (TN ? 1000 : 0) + LL:                                                                  \
    e = bf9 ? run_tc<TN, LL, kBF9>(mx, mh, ml, m2, a, grid, st)                               \
            : (f16 && LL <= 96) ? run_tc<TN, (LL <= 96 ? LL : 96), kF16>(mx, mh, ml, m2, a, grid, st) \
            : x1                ? run_tc<TN, LL, kX1>(mx, mh, ml, m2, a, grid, st)           \
                                : run_tc<TN, LL, kTF32>(mx, mh, ml, m2, a, grid, st);        \
    break;
  switch ((tn ? 1000 : 0) + L) {
    XS_CASE(false, 32) XS_CASE(false, 64) XS_CASE(false, 96) XS_CASE(false, 128)
    XS_CASE(true, 32) XS_CASE(true, 64) XS_CASE(true, 96) XS_CASE(true, 128)
    default: return false;
  }
#undef XS_CASE
  if (e != cudaSuccess) return false;
  if (p.nsplit > 1) {
    const int64_t total4 = rows_out * lp / 4;
    note_launches(1);
    if (launch_pdl(tc_split_reduce_kernel,
                   dim3((int)std::min<int64_t>((total4 + 255) / 256, (int64_t)nsm * 8)), dim3(256),
                   0, st, reinterpret_cast<const float4*>(parts), p.nsplit, total4,
                   reinterpret_cast<float4*>(out)) != cudaSuccess)
      return false;
  }
  return true;
}

}  // namespace cnmf
