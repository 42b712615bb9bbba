// Certified float64 merge + decision epilogue as device functions, shared by
// the standalone merge kernel (rescore.cu, tensor-core path) and the fused
// tail of the GEMV scan (scan_gemv.cu, last CTA to finish).
//
// Certificate.  For one query, with delta the rigorous
// bound on |approx - exact| (query units) of the scan that produced the lists:
//   M   = max approximate score over all chunk lists
//   rescore in float64 every listed row with approx >= M - 2 delta  -> s_c
//   every listed row below that has exact < M - delta <= s_c, and
//   every chunk floor F (largest score the chunk did not list) must satisfy
//   F + delta < s_c, or the query is flagged for the exhaustive rescan.
// Decision (cache.py:255-260, :112-117): newest among equal maxima, miss iff
// best < tau_0 (NaN is a hit, as `nan < tau` is false in numpy), k = the
// largest k_j with best >= tau_j.
#pragma once

#include "mc_device.cuh"

namespace mc {

constexpr int MERGE_THREADS = 256;
constexpr int MERGE_WARPS = MERGE_THREADS / 32;

constexpr int MERGE_CAND = 512;  // candidate capacity; more forces the exhaustive rescan

struct MergeScratch {
  double shd[MERGE_WARPS];
  float shf[MERGE_WARPS];
  Best2 shb[MERGE_WARPS];
  long long cand[MERGE_CAND];  // positions to rescore in float64
  int n_cand;
  int fail;
};

template <typename T>
__device__ __forceinline__ T block_sum(T v, T* sh) {
#pragma unroll
  for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(FULL, v, off);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  T t = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
  return t;
}

__device__ __forceinline__ float block_max(float v, float* sh) {
#pragma unroll
  for (int off = 16; off; off >>= 1) v = fmaxf(v, __shfl_xor_sync(FULL, v, off));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  float t = -INFINITY;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = fmaxf(t, sh[w]);
  return t;
}

// Block-wide merge of per-thread trackers.  `warp_uniform`: every lane of a
// warp already holds the same tracker (warp-cooperative rescoring), so the
// lanes must not be merged with each other — that would count each tie twice.
__device__ __forceinline__ Best2 block_best(Best2 b, Best2* sh, bool warp_uniform) {
  if (!warp_uniform) {
#pragma unroll
    for (int off = 16; off; off >>= 1) b.shfl_merge(off);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[warp] = b;
  __syncthreads();
  Best2 t;
  t.init();
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t.merge(sh[w]);
  return t;
}

// ||q||_2 and ||q||_1 of a float64 row held in shared memory (fixed order),
// rounded up so they bound the true norms.
__device__ __forceinline__ void q_norms(const double* sq, int D, double* sh, double& n2, double& n1) {
  double a = 0.0, c = 0.0;
  for (int i = threadIdx.x; i < D; i += blockDim.x) {
    a += sq[i] * sq[i];
    c += fabs(sq[i]);
  }
  a = block_sum(a, sh);
  c = block_sum(c, sh);
  n2 = sqrt(a) * (1.0 + 1e-15);
  n1 = c * (1.0 + 1e-15);
}

// Load query row q (global, length D, zero-padded to Dp) into shared memory.
__device__ __forceinline__ void load_query(const double* __restrict__ q, int D, int Dp, double* sq) {
  for (int i = threadIdx.x; i < Dp; i += blockDim.x) sq[i] = i < D ? q[i] : 0.0;
  __syncthreads();
}

// Certified merge of one query's chunk lists (whole CTA, blockDim == MERGE_THREADS).
// `scale` turns list scores into query units.  Returns the record in every thread.
static __device__ mc_record merge_one(const RingState& st, const double* __restrict__ ring64, int D, int Dp,
                               const double* sq, const float* __restrict__ ps, const long long* __restrict__ pp,
                               const float* __restrict__ pf, int n_chunks, double scale, double eps_rel,
                               double eps_a1, ShardMap sm, MergeScratch& ms) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double n2, n1;
  q_norms(sq, D, ms.shd, n2, n1);
  // Non-finite or extreme-magnitude queries leave the scan's error model; the
  // exhaustive float64 scan answers them instead.
  const bool exotic = !(n1 <= 1e30) || !(n2 >= 1e-30);
  const double delta = eps_rel * n2 + eps_a1 * n1;

  // One pass over the lists (and the floors) into registers: the max, the compaction and
  // the certificate below reuse them instead of re-reading global memory.
  const int ne = n_chunks * KP;
  constexpr int PER = 4;  // entries per thread kept in registers; longer lists re-read the rest
  float es[PER];
  long long ep[PER];
  float m = -INFINITY;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int e = threadIdx.x + k * (int)blockDim.x;
    es[k] = -INFINITY;
    ep[k] = -1;
    if (e < ne) {
      ep[k] = pp[e];
      es[k] = ps[e];
    }
  }
  float fmx = -INFINITY;  // largest finite-or-inf floor of this thread's chunks (fmaxf skips NaN)
  for (int c = threadIdx.x; c < n_chunks; c += blockDim.x) fmx = fmaxf(fmx, pf[c]);
#pragma unroll
  for (int k = 0; k < PER; ++k)
    if (ep[k] >= 0) m = fmaxf(m, es[k]);
  for (int e = threadIdx.x + PER * (int)blockDim.x; e < ne; e += blockDim.x)
    if (pp[e] >= 0) m = fmaxf(m, ps[e]);
  m = block_max(m, ms.shf);
  const double M = (double)m * scale;
  const double thr = M - 2.0 * delta - 1e-9;

  // Compact the candidates (thread-parallel, the lists are L2-hot after the max pass) ...
  if (threadIdx.x == 0) {
    ms.n_cand = 0;
    ms.fail = 0;
  }
  __syncthreads();
  auto admit = [&](long long p, float sc) {
    if (p >= 0 && (double)sc * scale >= thr) {
      const int i = atomicAdd(&ms.n_cand, 1);
      if (i < MERGE_CAND)
        ms.cand[i] = p;
      else
        ms.fail = 1;
    }
  };
#pragma unroll
  for (int k = 0; k < PER; ++k) admit(ep[k], es[k]);
  for (int e = threadIdx.x + PER * (int)blockDim.x; e < ne; e += blockDim.x) admit(pp[e], ps[e]);
  __syncthreads();
  // ... then one warp per candidate computes its float64 similarity.
  const int n_cand = min(ms.n_cand, MERGE_CAND);
  Best2 best;
  best.init();
  for (int i = warp; i < n_cand; i += MERGE_WARPS) {
    const long long p = ms.cand[i];
    const long long slot = ring_slot(st, local_row(st, p, sm));
    best.add(warp_dot64(ring64 + (size_t)slot * Dp, sq, Dp, lane), p);
  }
  best = block_best(best, ms.shb, true);

  // every chunk's floor must lie below the best (monotone in the floor: test the largest)
  if (fmx > -INFINITY && !((double)fmx * scale + delta < best.s)) atomicOr(&ms.fail, 1);
  __syncthreads();
  mc_record r;
  r.sim = best.s;
  r.second = best.s2;
  r.pos = best.p;
  r.flags = (best.ties >= 2 ? MC_FLAG_TIE : 0u) | (ms.fail || best.p < 0 ? FLAG_NEED_FALLBACK : 0u) |
            (exotic ? FLAG_NEED_EXHAUSTIVE : 0u);
  r.reserved = 0;
  __syncthreads();  // ms is reused by the next call
  return r;
}

// Decision for one query from its merged best (cache.py:255-260 + select_k), plus the serving
// decision the callers derive from it: steps = T - k (engine.py:38-45, service_time), route =
// hit / miss queue (scheduler.py:80-89) and sigma[k] (noise_reentry_level, cache.py:325-334).
__device__ __forceinline__ OutRec decide(const Best2& best, unsigned fl, long long base, const Thresholds& thr) {
  OutRec o;
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  o.steps = thr.total_steps;
  o.route = 0;
  o.sigma = qnan;
  if (best.p < 0) {
    o.live = -1;
    o.sim = qnan;
    o.k = 0;
    o.flags = MC_FLAG_EMPTY | (fl & (FLAG_NEED_FALLBACK | FLAG_NEED_EXHAUSTIVE));
    return o;
  }
  o.live = best.p - base;
  o.sim = best.s;
  const double s = best.s;
  unsigned f = fl;
  if (!(s < thr.taus[0])) f |= MC_FLAG_HIT;  // cache.py:258 — `best < tau` is the miss test
  int k = 0, jk = -1;
  for (int j = 0; j < thr.n; ++j) {
    if (s >= thr.taus[j]) {  // cache.py:112-117
      k = thr.ks[j];
      jk = j;
    }
    if (fabs(s - thr.taus[j]) < AMBIG) f |= MC_FLAG_NEAR_TAU;
  }
  o.k = k;
  if (best.ties >= 2) f |= MC_FLAG_TIE;
  if (best.s2 != s && s - best.s2 < AMBIG) f |= MC_FLAG_NEAR_TIE;
  o.flags = f;
  if (f & MC_FLAG_HIT) {
    o.route = 1;
    o.steps = thr.total_steps - k;  // a NaN best is a hit with no k: every step runs
    if (thr.has_sigma && jk >= 0) o.sigma = thr.sigma[jk];
  }
  return o;
}

__device__ __forceinline__ Best2 record_best(const mc_record& r) {
  Best2 b;
  b.init();
  if (r.pos >= 0) {
    b.s = r.sim;
    b.p = r.pos;
    b.s2 = r.second;
    b.ties = (r.flags & MC_FLAG_TIE) ? 2 : 1;
  }
  return b;
}

// k_finalize's decision for a single shard's record (G = 1, base = jhead).
__device__ __forceinline__ OutRec decide_one(const mc_record& r, long long base, const Thresholds& thr) {
  Best2 best;
  best.init();
  unsigned fl = 0;
  if (r.pos < 0) {
    if (r.flags != 0xffffffffu) fl |= r.flags & FLAG_NEED_ANY;
  } else {
    fl |= r.flags & (MC_FLAG_FALLBACK | MC_FLAG_NONFINITE | FLAG_NEED_ANY);
    best.merge(record_best(r));
  }
  return decide(best, fl, base, thr);
}

}  // namespace mc
