// hals_common.cuh -- grid-wide exchange primitives shared by the streaming
// (hals.cu) and shared-memory-resident (hals_resident.cu) FastHALS-RP kernels.
#pragma once

#include "common.cuh"
#include "kernels.h"

namespace cnmf {
namespace hals_detail {

constexpr int kThreads = 256;

// Grid-wide barrier with payload visibility: every CTA's global writes made
// before the call are visible to every CTA after it.  A monotonic arrival
// counter (reset per run; `ep` counts barriers) -- measured as the cheapest
// deterministic exchange on B200 (tools/ubench_allreduce.cu: ~2.9k cycles at
// 4 CTAs, ~4.1k at 148, including the read of the per-CTA partials).
__device__ __forceinline__ void exchange(const HalsState& S, int G, int /*cta*/,
                                         unsigned long long& ep) {
  ++ep;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(S.bar, 1u);
    const unsigned target = (unsigned)(ep * (unsigned long long)G);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(S.bar) : "memory");
    } while ((int)(v - target) < 0);
  }
  __syncthreads();
}

// All-reduce of one fp64 per CTA: partial -> barrier -> every CTA sums the G
// partials in the same fixed order (lanes, then a warp tree).  Partials are
// double-buffered by barrier parity.
__device__ __forceinline__ double allreduce(const HalsState& S, int G, int cta, unsigned long long& ep,
                            double v, double* s_out) {
  double* slot = S.npart + ((ep + 1) & 1ULL) * G;
  if (threadIdx.x == 0) slot[cta] = v;
  exchange(S, G, cta, ep);
  if (threadIdx.x < 32) {
    double t = 0.0;
    for (int b = threadIdx.x; b < G; b += 32) t += __ldcg(slot + b);
    t = warp_sum(t);
    if (threadIdx.x == 0) *s_out = t;
  }
  __syncthreads();
  return *s_out;
}

// After an exchange of per-CTA partials (G x nel doubles): CTA c reduces its
// slice of entries in a fixed order (lanes over CTAs, then a warp tree).
__device__ __forceinline__ void slice_reduce(const double* __restrict__ part, int G, int nel,
                             double* __restrict__ dst) {
  const int per = (nel + G - 1) / G;
  const int e0 = blockIdx.x * per, e1 = min(nel, e0 + per);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int e = e0 + wid; e < e1; e += kThreads / 32) {
    double s = 0.0;
#pragma unroll 5
    for (int b = lane; b < G; b += 32) s += __ldcg(part + (int64_t)b * nel + e);
    s = warp_sum(s);
    if (lane == 0) dst[e] = s;
  }
}


}  // namespace hals_detail
}  // namespace cnmf
