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
// Warp 0 polls the arrival counter with every lane (converged): a single
// lane spinning while its warp-mates wait at a barrier cost ~2x in detection
// latency (measured in the HALS kernel: 2.5k -> 1.2k cycles per all-reduce).
__device__ __forceinline__ void poll_counter_warp(const unsigned* bar, unsigned target) {
  unsigned c;
  do {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(bar) : "memory");
  } while (__any_sync(0xffffffffu, (int)(c - target) < 0));
}

__device__ __forceinline__ void poll_counter_warp_relaxed(const unsigned* bar, unsigned target) {
  unsigned c;
  do {
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(bar) : "memory");
  } while (__any_sync(0xffffffffu, (int)(c - target) < 0));
}

__device__ __forceinline__ void exchange(const HalsState& S, int G, int /*cta*/,
                                         unsigned long long& ep) {
  ++ep;
  __syncthreads();
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(S.bar, 1u);
    }
    poll_counter_warp(S.bar, (unsigned)(ep * (unsigned long long)G));
  }
  __syncthreads();
}

// 1/sqrt(x) for x > 0 to ~1 ulp (0 for x <= 0): hardware rsqrt seed + two
// fp64 Newton steps, far shorter than sqrt() followed by a division (the
// reference divides by sqrt; the difference is a rounding or two).
__device__ __forceinline__ double rsqrt_fp64(double x) {
  if (!(x > 0.0)) return 0.0;
  double y = rsqrt(x);  // MUFU-seeded, already close to fp64 precision
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}

// Sum of the G (<= 32 * 8 fast path) per-CTA doubles at p, by one warp, in a
// fixed order (lane-strided, then a butterfly).  All loads are issued before
// any is used: a runtime-trip-count loop would serialise them into G / 32
// L2 round trips (measured ~3k cycles at G = 148).
__device__ __forceinline__ double warp_sum_partials(const double* __restrict__ p, int G, int lane) {
  double t = 0.0;
  if (G <= 256) {
    double v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int b = lane + 32 * i;
      v[i] = b < G ? __ldcg(p + b) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) t += v[i];
  } else {
    for (int b = lane; b < G; b += 32) t += __ldcg(p + b);
  }
  return warp_sum(t);
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
    const double t = warp_sum_partials(slot, G, threadIdx.x);
    if (threadIdx.x == 0) *s_out = t;
  }
  __syncthreads();
  return *s_out;
}

// Arrival on the grid counter with release semantics for everything the
// block wrote before (callers synchronised the block first).
__device__ __forceinline__ void arrive_release(unsigned* bar) {
#ifdef HALS_FENCE_ATOMIC
  __threadfence();
  atomicAdd(bar, 1u);
#else
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
#endif
}

// Tagged slots for the per-column norm all-reduce: the partial (>= 0) is
// stored with its sign bit set on every other use of its buffer, so one
// 64-bit store carries both the value and its freshness and the arrival
// needs no release fence (the counter only says "everyone has written";
// a reader that still sees last use's sign re-reads that slot).  Buffer and
// tag follow nr, the count of these all-reduces in the run (carried across
// launches in HaltInfo::last_nr / HalsState::nr0), NOT the barrier epoch:
// other grid barriers between two uses must not make a buffer's next use
// carry its previous tag.  Use nr goes to buffer nr & 1 with the tag flipped
// every second use, so consecutive uses of one buffer always differ; the
// first use of each buffer is the negative one, which the zeroed slots
// never match.
__device__ __forceinline__ bool tag_neg(unsigned long long nr) { return ((nr >> 1) & 1ULL) == 0; }

__device__ __forceinline__ void st_tagged(double* slot, double v, bool neg) {
  const double t = neg ? -v : v;
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(slot), "d"(t) : "memory");
}

__device__ __forceinline__ double ld_relaxed(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}

// Sum of the G tagged partials (fixed order, as warp_sum_partials), waiting
// for every slot to carry this use's tag.
__device__ __forceinline__ double warp_sum_tagged(const double* __restrict__ p, int G, int lane,
                                                  bool neg) {
  double t = 0.0;
  for (int b0 = 0; b0 < G; b0 += 256) {
    double v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int b = b0 + lane + 32 * i;
      v[i] = b < G ? ld_relaxed(p + b) : (neg ? -0.0 : 0.0);
    }
    for (;;) {
      bool stale = false;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int b = b0 + lane + 32 * i;
        if (b < G && (signbit(v[i]) != 0) != neg) {
          stale = true;
          v[i] = ld_relaxed(p + b);
        }
      }
      if (!__any_sync(0xffffffffu, stale)) break;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) t += fabs(v[i]);
  }
  return warp_sum(t);
}

__device__ __forceinline__ void arrive_relaxed(unsigned* bar) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
}

// Block + grid all-reduce of one fp64 per thread with two __syncthreads:
// warp sums -> red8 -> warp 0 sums the warp partials, lane 0 publishes the
// CTA partial, arrives on the monotonic counter with a release add (no
// separate __threadfence), polls with acquire loads; warp 0 then sums the G
// CTA partials (lanes over CTAs in a fixed order, then a butterfly), so every
// CTA computes the bitwise-identical total.  Lane 0 also stores 1/sqrt(total)
// (0 when total == 0) into s_out[1] so callers normalise with one multiply.
// Partials are double-buffered by use parity: a CTA can only write use
// nr + 2's slot after every CTA arrived at use nr + 1, i.e. finished reading
// use nr.
__device__ __forceinline__ double allreduce_fused(const HalsState& S, int G, int cta,
                                                  unsigned long long& ep, unsigned long long& nr,
                                                  double v,
                                                  double* red8, double* s_out,
                                                  long long* prof = nullptr) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  long long t0 = 0, t1 = 0, t2 = 0, t3 = 0;
  if (prof && threadIdx.x == 0) t0 = clock64();
  v = warp_sum(v);
  if (lane == 0) red8[wid] = v;
  __syncthreads();
  ++ep;
  if (wid == 0) {
    if (prof && lane == 0) t1 = clock64();
    double* slot = S.npart + (nr & 1ULL) * G;
    const bool neg = tag_neg(nr);
    if (lane == 0) {
      double t = 0.0;  // CTA partial: the warp partials in a fixed order
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) t += red8[w];
      st_tagged(slot + cta, t, neg);
      arrive_relaxed(S.bar);
      if (prof) t2 = clock64();
    }
    // every lane polls (no divergent spin + reconvergence), then reads; the
    // tags, not acquire ordering, vouch for the slot values
    poll_counter_warp_relaxed(S.bar, (unsigned)(ep * (unsigned long long)G));
    if (prof && lane == 0) t3 = clock64();
    const double tot = warp_sum_tagged(slot, G, lane, neg);
    if (lane == 0) {
      s_out[0] = tot;
      s_out[1] = rsqrt_fp64(tot);
      if (prof) {
        const long long t4 = clock64();
        prof[0] += t1 - t0;  // local reduction + first barrier
        prof[1] += t2 - t1;  // warp-0 sum, publish, arrive
        prof[2] += t3 - t2;  // poll until all CTAs arrived
        prof[3] += t4 - t3;  // read partials, sum, 1/sqrt
      }
    }
  }
  ++nr;
  __syncthreads();
  return s_out[0];
}

// Grid barrier with payload visibility (release add + acquire poll), the
// cheaper form of exchange() for callers that already synchronised the block.
__device__ __forceinline__ void exchange_fast(const HalsState& S, int G, unsigned long long& ep) {
  ++ep;
  __syncthreads();
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) arrive_release(S.bar);
    poll_counter_warp(S.bar, (unsigned)(ep * (unsigned long long)G));
  }
  __syncthreads();
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
    if (G <= 256) {
      double v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int b = lane + 32 * i;
        v[i] = b < G ? __ldcg(part + (int64_t)b * nel + e) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) s += v[i];
    } else {
      for (int b = lane; b < G; b += 32) s += __ldcg(part + (int64_t)b * nel + e);
    }
    s = warp_sum(s);
    if (lane == 0) dst[e] = s;
  }
}


}  // namespace hals_detail
}  // namespace cnmf
