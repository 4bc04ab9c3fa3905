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
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace cnmf {

namespace {

constexpr int kBM = 128;     // output rows per unit (MMA M)
constexpr int kBK = 32;      // K elements per stage (4 MMA k-steps of 8)
constexpr int kThreadsTC = 352;  // warps 0-3 epilogue, 4 X TMA, 5 MMA, 6-9 split, 10 S TMA
constexpr int kWarpTMA = 4, kWarpMMA = 5, kWarpSplit0 = 6, kWarpBTMA = 10;
constexpr int kDrain = 4;         // K-blocks (16 MMA k-steps) per TMEM accumulation chain
constexpr int kXBytes = kBM * kBK * 4;  // 16 KB per stage (x_hi), same for x_lo

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Shared-memory matrix descriptor (sm_100, version 1).  K-major operands use
// SWIZZLE_128B (layout 2: 8 rows x 128 B atoms, 16 B granules); MN-major
// 32-bit operands must use SWIZZLE_128B_BASE32B (layout 1: 4 K-rows x 128 B
// atoms, 32 B granules) -- with plain SWIZZLE_128B an MN-major kind::tf32 MMA
// is a silent no-op on B200 (measured with tools/tc_debug.cu).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout = 2) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;        // version
  d |= (uint64_t)layout << 61;   // layout type
  return d;
}
// MN-major operand: atoms of 32 elements along MN (one 128 B row) x 4 K-rows;
// MN atoms `lbo` bytes apart, 4-row groups 512 B apart.
__device__ __forceinline__ uint64_t desc_mn(uint32_t addr, uint32_t lbo) {
  return smem_desc(addr, lbo, 512, 1);
}
// Instruction descriptor: kind::tf32, fp32 accumulate, M = 128.
__host__ __device__ constexpr uint32_t idesc_tf32(int n, bool a_mn, bool b_mn) {
  return (1u << 4)                       // D format F32
         | (2u << 7)                     // A format TF32
         | (2u << 10)                    // B format TF32
         | ((a_mn ? 1u : 0u) << 15)      // A major
         | ((b_mn ? 1u : 0u) << 16)      // B major
         | ((uint32_t)(n >> 3) << 17)    // N >> 3
         | ((uint32_t)(kBM >> 4) << 24); // M >> 4
}

struct TcArgs {
  int64_t rows_out;  // output rows (m for NN, n for TN)
  int64_t kdim;      // reduction length (n for NN, m for TN)
  int64_t kchunk;    // K per split (multiple of kBK)
  int ntiles, nsplit, lp;
  float* out;        // [nsplit][rows_out][lp] or the final output when nsplit == 1
  float* dbg;        // optional debug dump (tools/tc_debug.cu), null in production
};

// x -> (x_hi, x_lo) = (rna_tf32(x), rna_tf32(x - x_hi)); both exactly
// representable in tf32, so the tensor core's operand conversion is exact.
__device__ __forceinline__ void tf32_split(float x, float& hi, float& lo) {
  uint32_t h, l;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  hi = __uint_as_float(h);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(x - hi));
  lo = __uint_as_float(l);
}

// Shared-memory rings (bytes): X stages (TMA -> split warps), operand slots
// (split warps -> MMA: x_hi, x_lo) and S slots (TMA -> MMA: s_hi, s_lo).  An X
// stage is released as soon as the split warps have read it, so the TMA
// producer runs kXStages * 16 KB ahead of the consumers instead of being held
// through the MMA (the first version kept <= 32 KB of X in flight per SM).
template <int L> struct TcRings {
  static constexpr int kBBytes = kBK * L * 4;               // s_hi or s_lo per K-block
  static constexpr int kOpStages = 2;
  static constexpr int kBStages = 3;
  static constexpr int kBudget = 225 * 1024;
  static constexpr int kXStages =
      (kBudget - kOpStages * 2 * kXBytes - kBStages * 2 * kBBytes) / kXBytes > 8
          ? 8
          : (kBudget - kOpStages * 2 * kXBytes - kBStages * 2 * kBBytes) / kXBytes;
  static constexpr int kXOff = 0;
  static constexpr int kOpOff = kXStages * kXBytes;
  static constexpr int kBOff = kOpOff + kOpStages * 2 * kXBytes;
  static constexpr int kBytes = kBOff + kBStages * 2 * kBBytes;
};

__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

template <bool kTN, int L>  // L = padded width (multiple of 32, <= 128)
__global__ void __launch_bounds__(kThreadsTC, 1)
    xs_tc_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_bh,
                 const __grid_constant__ CUtensorMap map_bl, const TcArgs args) {
  using R = TcRings<L>;
  constexpr int kSX = R::kXStages, kSO = R::kOpStages, kSB = R::kBStages;
  constexpr int kAccCols = 2 * L;  // per accumulator buffer
  constexpr uint32_t kTmemCols = 4 * L <= 32 ? 32 : (4 * L <= 64 ? 64 : (4 * L <= 128 ? 128 : (4 * L <= 256 ? 256 : 512)));

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
  __shared__ __align__(8) uint64_t xfull[kSX], xempty[kSX], opready[kSO], opempty[kSO];
  __shared__ __align__(8) uint64_t bfull[kSB], bempty[kSB], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSX; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], 4);
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
  auto hi_addr = [&](int o) { return sbase + R::kOpOff + o * 2 * kXBytes; };
  auto lo_addr = [&](int o) { return sbase + R::kOpOff + o * 2 * kXBytes + kXBytes; };
  auto b_addr = [&](int b) { return sbase + R::kBOff + b * 2 * R::kBBytes; };  // [s_hi | s_lo]
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
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int64_t k0, k1;
        unit_k(u, k0, k1);
        const int row0 = (u % args.ntiles) * kBM;
        for (int64_t kk = k0; kk < k1; kk += kBK) {
          mbar_wait(&xempty[s], ph ^ 1);
          mbar_expect_tx(&xfull[s], kXBytes);
          if (!kTN) {
            tma(x_addr(s), &map_x, &xfull[s], (int)kk, row0);
          } else {
#pragma unroll
            for (int a = 0; a < kBM / 32; ++a)
              tma(x_addr(s) + a * (kBK * 128), &map_x, &xfull[s], row0 + 32 * a, (int)kk);
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
    if (lane == 0) {
      int b = 0;
      uint32_t ph = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int64_t k0, k1;
        unit_k(u, k0, k1);
        for (int64_t kk = k0; kk < k1; kk += kBK) {
          mbar_wait(&bempty[b], ph ^ 1);
          mbar_expect_tx(&bfull[b], 2 * R::kBBytes);
#pragma unroll
          for (int a = 0; a < L / 32; ++a) {
            tma(b_addr(b) + a * (kBK * 128), &map_bh, &bfull[b], 32 * a, (int)kk);
            tma(b_addr(b) + (L / 32 + a) * (kBK * 128), &map_bl, &bfull[b], 32 * a, (int)kk);
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
    // Every kDrain K-blocks the accumulator is handed to the epilogue (which
    // sums the chunks in registers) and the other TMEM buffer takes over: the
    // tensor core's fp32 accumulation error grows with the chain length
    // (tools/tc_precision.py), so chains are kept to 16 k-steps.
    if (lane == 0) {
      constexpr uint32_t idesc_full = idesc_tf32(2 * L, kTN, true);
      constexpr uint32_t idesc_hi = idesc_tf32(L, kTN, true);
      int o = 0, b = 0, ab = 0;
      uint32_t oph = 0, bph = 0, aph = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int64_t k0, k1;
        unit_k(u, k0, k1);
        for (int64_t g0 = k0; g0 < k1; g0 += (int64_t)kDrain * kBK) {
          const int64_t g1 = min(k1, g0 + (int64_t)kDrain * kBK);
          mbar_wait(&acc_empty[ab], aph ^ 1);
          tc_fence_after();
          const uint32_t d = tmem + ab * kAccCols;
          uint32_t acc = 0;
          for (int64_t kk = g0; kk < g1; kk += kBK) {
            mbar_wait(&opready[o], oph);
            mbar_wait(&bfull[b], bph);
            tc_fence_after();
            const uint32_t xa = hi_addr(o), la = lo_addr(o), ba = b_addr(b);
#pragma unroll
            for (int ks = 0; ks < kBK / 8; ++ks) {
              const uint32_t aoff = kTN ? ks * 1024 : ks * 32;
              const uint64_t ahi = kTN ? desc_mn(xa + aoff, kBK * 128) : smem_desc(xa + aoff, 16, 1024);
              const uint64_t alo = kTN ? desc_mn(la + aoff, kBK * 128) : smem_desc(la + aoff, 16, 1024);
              const uint64_t bd = desc_mn(ba + ks * 1024, kBK * 128);
              tc_mma_tf32(d, ahi, bd, idesc_full, acc);
              tc_mma_tf32(d, alo, bd, idesc_hi, 1u);
              acc = 1u;
            }
            tc_commit(&opempty[o]);  // operand slot and S slot free once these MMAs complete
            tc_commit(&bempty[b]);
            if (++o == kSO) {
              o = 0;
              oph ^= 1;
            }
            if (++b == kSB) {
              b = 0;
              bph ^= 1;
            }
          }
          tc_commit(&acc_full[ab]);
          if (++ab == 2) {
            ab = 0;
            aph ^= 1;
          }
        }
      }
    }
  } else if (warp >= kWarpSplit0 && warp < kWarpSplit0 + 4) {
    // ---------------- split warps: X stage -> (x_hi, x_lo) operand slot ----
    const int t = threadIdx.x - 32 * kWarpSplit0;  // 0..127
    constexpr int kPer = kXBytes / 16 / 128;       // float4 per thread per stage (8)
    int s = 0, o = 0;
    uint32_t xph = 0, oph = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      int64_t k0, k1;
      unit_k(u, k0, k1);
      for (int64_t kk = k0; kk < k1; kk += kBK) {
        mbar_wait(&xfull[s], xph);
        float4 v[kPer];
#pragma unroll
        for (int i = 0; i < kPer; ++i) v[i] = lds128(x_addr(s) + 16 * (t + 128 * i));
        __syncwarp();
        if (lane == 0) mbar_arrive(&xempty[s]);  // the X stage can be refilled now
        mbar_wait(&opempty[o], oph ^ 1);
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
          float4 h, l;
          tf32_split(v[i].x, h.x, l.x);
          tf32_split(v[i].y, h.y, l.y);
          tf32_split(v[i].z, h.z, l.z);
          tf32_split(v[i].w, h.w, l.w);
          sts128(hi_addr(o) + 16 * (t + 128 * i), h);
          sts128(lo_addr(o) + 16 * (t + 128 * i), l);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&opready[o]);
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
      float run[L];
#pragma unroll
      for (int c = 0; c < L; ++c) run[c] = 0.f;
      for (int64_t g0 = k0; g0 < k1; g0 += (int64_t)kDrain * kBK) {
        mbar_wait(&acc_full[ab], aph);
        tc_fence_after();
        const uint32_t base = tmem + ab * kAccCols + ((uint32_t)(32 * q) << 16);
#pragma unroll
        for (int c = 0; c < L; c += 16) {
          uint32_t h[16], o[16];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(h[0]), "=r"(h[1]), "=r"(h[2]), "=r"(h[3]), "=r"(h[4]), "=r"(h[5]), "=r"(h[6]),
                "=r"(h[7]), "=r"(h[8]), "=r"(h[9]), "=r"(h[10]), "=r"(h[11]), "=r"(h[12]),
                "=r"(h[13]), "=r"(h[14]), "=r"(h[15])
              : "r"(base + c));
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(o[0]), "=r"(o[1]), "=r"(o[2]), "=r"(o[3]), "=r"(o[4]), "=r"(o[5]), "=r"(o[6]),
                "=r"(o[7]), "=r"(o[8]), "=r"(o[9]), "=r"(o[10]), "=r"(o[11]), "=r"(o[12]),
                "=r"(o[13]), "=r"(o[14]), "=r"(o[15])
              : "r"(base + L + c));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 16; ++j)
            run[c + j] += __uint_as_float(h[j]) + __uint_as_float(o[j]);
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
#pragma unroll
        for (int c = 0; c < L; c += 4)
          if (c < args.lp) *reinterpret_cast<float4*>(dst + c) = make_float4(run[c], run[c + 1], run[c + 2], run[c + 3]);
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

__global__ void tc_split_reduce_kernel(const float4* __restrict__ part, int splits, int64_t total4,
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

float* g_tc_debug = nullptr;

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2D fp32 row-major tensor (rows x cols, row pitch ld floats), 32 x box_rows
// boxes with 128-byte swizzle.
bool make_map(CUtensorMap* m, const float* base, int64_t rows, int64_t cols, int64_t ld,
              int box_rows, bool mn_major) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  const cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

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

template <bool kTN, int L>
cudaError_t run_tc(const CUtensorMap& mx, const CUtensorMap& mh, const CUtensorMap& ml,
                   const TcArgs& a, int grid, cudaStream_t st) {
  constexpr int smem = TcRings<L>::kBytes + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(xs_tc_kernel<kTN, L>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  note_launches(1);
  xs_tc_kernel<kTN, L><<<grid, kThreadsTC, smem, st>>>(mx, mh, ml, a);
  return cudaGetLastError();
}

}  // namespace

void xstream_tc_set_debug(float* dbg) { g_tc_debug = dbg; }

size_t xstream_tc_ws_floats(int64_t m, int64_t n, int lp, int nsm) {
  const int L = (lp + 31) & ~31;
  const TcPlan a = tc_plan(m, n, nsm), b = tc_plan(n, m, nsm);
  const int64_t parts = std::max<int64_t>((int64_t)a.nsplit * m * lp, (int64_t)b.nsplit * n * lp);
  return (size_t)(parts + 2 * std::max(m, n) * (int64_t)L + 64);
}

bool launch_xs_tc(bool tn, const float* x, int64_t ldx, int64_t m, int64_t n, const float* s,
                  int lp, float* out, float* ws, int nsm, cudaStream_t st) {
  const int L = (lp + 31) & ~31;
  if (L > 128 || (ldx % 4) != 0 || (reinterpret_cast<uintptr_t>(x) & 15)) return false;
  const int64_t rows_out = tn ? n : m, kdim = tn ? m : n;
  const TcPlan p = tc_plan(rows_out, kdim, nsm);
  float* hi = ws;
  float* lo = ws + kdim * (int64_t)L;
  float* parts = lo + kdim * (int64_t)L;
  note_launches(1);
  split_tf32_kernel<<<std::min<int64_t>((kdim * L + 255) / 256, nsm * 8), 256, 0, st>>>(
      s, kdim, lp, L, hi, lo);
  CUtensorMap mx, mh, ml;
  bool ok = tn ? make_map(&mx, x, m, n, ldx, kBK, true) : make_map(&mx, x, m, n, ldx, kBM, false);
  ok = ok && make_map(&mh, hi, kdim, L, L, kBK, true) && make_map(&ml, lo, kdim, L, L, kBK, true);
  if (!ok) return false;
  TcArgs a;
  a.rows_out = rows_out;
  a.kdim = kdim;
  a.kchunk = p.kchunk;
  a.ntiles = p.ntiles;
  a.nsplit = p.nsplit;
  a.lp = lp;
  a.out = p.nsplit > 1 ? parts : out;
  a.dbg = g_tc_debug;
  const int units = p.ntiles * p.nsplit;
  const int grid = std::min(units, nsm);
  cudaError_t e;
  switch ((tn ? 1000 : 0) + L) {
    case 32: e = run_tc<false, 32>(mx, mh, ml, a, grid, st); break;
    case 64: e = run_tc<false, 64>(mx, mh, ml, a, grid, st); break;
    case 96: e = run_tc<false, 96>(mx, mh, ml, a, grid, st); break;
    case 128: e = run_tc<false, 128>(mx, mh, ml, a, grid, st); break;
    case 1032: e = run_tc<true, 32>(mx, mh, ml, a, grid, st); break;
    case 1064: e = run_tc<true, 64>(mx, mh, ml, a, grid, st); break;
    case 1096: e = run_tc<true, 96>(mx, mh, ml, a, grid, st); break;
    case 1128: e = run_tc<true, 128>(mx, mh, ml, a, grid, st); break;
    default: return false;
  }
  if (e != cudaSuccess) return false;
  if (p.nsplit > 1) {
    const int64_t total4 = rows_out * lp / 4;
    note_launches(1);
    tc_split_reduce_kernel<<<(int)std::min<int64_t>((total4 + 255) / 256, (int64_t)nsm * 8), 256,
                             0, st>>>(reinterpret_cast<const float4*>(parts), p.nsplit, total4,
                                      reinterpret_cast<float4*>(out));
  }
  return true;
}

}  // namespace cnmf
