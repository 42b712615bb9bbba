// Device helpers shared by the scan / rescore kernels.
#pragma once

#include <cuda_fp16.h>
#include <math.h>
#include <stdint.h>

#include "mc_internal.cuh"

namespace mc {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ uint4 ld_stream16(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Physical ring slot of live-local row i.
__device__ __forceinline__ long long ring_slot(const RingState& st, long long i) {
  long long s = st.head + i;
  return s >= st.cap ? s - st.cap : s;
}

// Global append position of live-local row i on shard (G, g).
__device__ __forceinline__ long long global_pos(const RingState& st, long long i, ShardMap sm) {
  return (st.jhead + i) * (long long)sm.G + sm.g;
}

// Inverse: live-local row of global position p (p must belong to this shard and be live).
__device__ __forceinline__ long long local_row(const RingState& st, long long p, ShardMap sm) {
  return (p - sm.g) / sm.G - st.jhead;
}

// Knuth TwoSum: s + e == a + b exactly.  Symmetric in (a, b).
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  double z = s - a;
  e = (a - (s - z)) + (b - z);
}

__device__ __forceinline__ void dot2_step(double a, double b, double& s, double& c) {
  const double p = a * b;
  const double ep = fma(a, b, -p);
  double t, et;
  two_sum(s, p, t, et);
  s = t;
  c += ep + et;
}

// Compensated (Ogita-Rump-Oishi Dot2) float64 dot product of one row with q
// over n elements (n a multiple of 64, rows and q zero-padded), one warp.
// Lane l owns elements 2l, 2l+1 of every 64-element block j.  Block j feeds
// chain j % 4 (four independent error-free accumulation chains, so the
// dependent latency is a quarter of a single chain's); blocks are visited in
// increasing order and the chains are combined in a fixed tree, then the
// butterfly.  All loads of a 1024-element batch are issued before the first
// product.  The lane->element map, chain map and trees are fixed, so every
// lane returns the same bits and identical rows always score identically
// (exact ties stay exact) — on every path that rescores (scan tails, merge,
// exhaustive rescan).
__device__ __forceinline__ double warp_dot64(const double* __restrict__ row, const double* __restrict__ q, int n,
                                             int lane) {
  double s[4] = {0.0, 0.0, 0.0, 0.0}, c[4] = {0.0, 0.0, 0.0, 0.0};
  for (int base = 0; base < n; base += 1024) {
    double2 a[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int i = base + 64 * j + 2 * lane;
      a[j] = i < n ? __ldg(reinterpret_cast<const double2*>(row + i)) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int i = base + 64 * j + 2 * lane;
      if (i < n) {
        const double2 b = *reinterpret_cast<const double2*>(q + i);
        dot2_step(a[j].x, b.x, s[j & 3], c[j & 3]);
        dot2_step(a[j].y, b.y, s[j & 3], c[j & 3]);
      }
    }
  }
  double t, et;
  two_sum(s[0], s[1], t, et);
  s[0] = t;
  c[0] = (c[0] + c[1]) + et;
  two_sum(s[2], s[3], t, et);
  s[2] = t;
  c[2] = (c[2] + c[3]) + et;
  two_sum(s[0], s[2], t, et);
  double sum = t, comp = (c[0] + c[2]) + et;
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    const double s2 = __shfl_xor_sync(FULL, sum, off);
    const double c2 = __shfl_xor_sync(FULL, comp, off);
    two_sum(sum, s2, t, et);
    sum = t;
    comp = (comp + c2) + et;
  }
  // Inf/NaN products poison the compensation term; the plain sum then carries
  // the same (order-independent) Inf/NaN a naive summation would produce.
  return isfinite(sum) ? sum + comp : sum;
}

// Kept as a name for the small-batch scans (n <= 1024: one load batch).
__device__ __forceinline__ double warp_dot64_1k(const double* __restrict__ row, const double* __restrict__ q, int n,
                                                int lane) {
  return warp_dot64(row, q, n, lane);
}

__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
  for (int off = 16; off; off >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, off));
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(FULL, v, off);
  return v;
}

// Per-row int8 scale: s >= max|e| / 127 (rounded up, so |e / s| <= 127 and
// rint never leaves [-127, 127]); a zero row gets s = 1.
__device__ __forceinline__ float int8_scale(double amax) {
  return amax > 0.0 ? __double2float_ru(amax / 127.0) : 1.0f;
}
__device__ __forceinline__ int8_t int8_quant(double v, float s) {
  return (int8_t)__double2int_rn(v / (double)s);
}

// One warp writes every device copy of a float64 row (zero-padded to Dp) into
// ring slot `slot` (k_append's work, used by the fused scans for the few rows
// appended since the last lookup).  Returns the row's int8 scale.
static __device__ __noinline__ float write_row_all(const double* __restrict__ src, long long slot, const RingBufs& rb,
                                            int Dp, int lane) {
  double amax = 0.0, l1 = 0.0;
  for (int i = lane; i < Dp; i += 32) {
    const double v = src[i];
    amax = fmax(amax, fabs(v));
    l1 += fabs(v);
  }
  amax = warp_max_d(amax);
  l1 = warp_sum_d(l1);
  const float s = int8_scale(amax);
  // row pointers in registers: through the reference every store below could alias rb,
  // and the compiler would reload its fields from the caller's stack each iteration
  double* const d64 = rb.r64 + (size_t)slot * Dp;
  __half* const d16 = rb.r16 + (size_t)slot * Dp;
  int8_t* const d8 = rb.r8 + (size_t)slot * rb.p8;
  float2* const dq = rb.rq + slot;
  for (int i = lane; i < Dp; i += 32) {
    const double v = src[i];
    d64[i] = v;
    d16[i] = __double2half(v);
    d8[i] = int8_quant(v, s);
  }
  if (lane == 0) *dq = make_float2(s, __double2float_ru(l1 * (1.0 + 1e-12)));
  return s;
}

// Composite order of (similarity, position): larger similarity wins; equal
// similarities go to the larger (newer) position — cache.py:255-256.  NaN
// ranks above everything (np.argmax returns the first NaN of the reversed
// view, i.e. the newest NaN).
__device__ __forceinline__ bool better(double a, long long pa, double b, long long pb) {
  bool na = isnan(a), nb = isnan(b);
  if (na || nb) {
    if (na && nb) return pa > pb;
    return na;
  }
  if (a != b) return a > b;
  return pa > pb;
}

// Running best / runner-up tracker over float64 candidates.
struct Best2 {
  double s;
  long long p;
  double s2;  // best similarity among candidates other than (s, p)
  int ties;   // candidates with similarity bit-equal to s (>= 1 once set)

  __device__ __forceinline__ void init() {
    s = -INFINITY;
    p = -1;
    s2 = -INFINITY;
    ties = 0;
  }
  __device__ __forceinline__ void add(double v, long long pv) {
    if (pv < 0) return;
    if (p < 0 || better(v, pv, s, p)) {
      if (p >= 0) s2 = fmax(s2, s);
      ties = (p >= 0 && v == s) ? ties + 1 : 1;
      s = v;
      p = pv;
    } else {
      s2 = fmax(s2, v);
      if (v == s) ties++;
    }
  }
  __device__ __forceinline__ void merge(const Best2& o) {
    if (o.p < 0) return;
    if (p < 0) {
      *this = o;
      return;
    }
    if (better(o.s, o.p, s, p)) {
      int t = (o.s == s) ? o.ties + ties : o.ties;
      s2 = fmax(fmax(s2, s), o.s2);
      s = o.s;
      p = o.p;
      ties = t;
    } else {
      if (o.s == s) ties += o.ties;
      s2 = fmax(fmax(s2, o.s), o.s2);
    }
  }
  __device__ __forceinline__ void shfl_merge(int off) {
    Best2 o;
    o.s = __shfl_xor_sync(FULL, s, off);
    o.p = __shfl_xor_sync(FULL, p, off);
    o.s2 = __shfl_xor_sync(FULL, s2, off);
    o.ties = __shfl_xor_sync(FULL, ties, off);
    merge(o);
  }
};

}  // namespace mc
