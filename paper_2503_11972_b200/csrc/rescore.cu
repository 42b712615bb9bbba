// K4 — certified float64 rescoring, exhaustive fallback, and the decision epilogue.
//
// The scans (scan_gemv.cu / scan_tc.cu) return, per query and per chunk of
// live rows, the K' best *approximate* scores plus the largest score the
// chunk dropped (its floor).  With delta = the rigorous bound on
// |approx - exact| for this query and path:
//   1. M  = max approximate score (query units).
//   2. Every listed row with approx >= M - 2 delta is rescored in float64
//      (compensated dot, warp_dot64) against the fp64 master -> best s_c.
//      Any row with approx < M - 2 delta has exact < M - delta <= s_c.
//   3. Certificate: every chunk floor F satisfies F + delta < s_c, so no
//      dropped row can reach (or tie) s_c.  Otherwise the query is flagged
//      and the host runs k_exact_scan (all rows, filter approx >= s_c - delta',
//      float64 for the survivors).
// The decision (k_finalize) restates cache.py:255-260 + select_k (:112-117):
// newest among equal maxima, miss iff best < tau_0 (NaN counts as a hit, as in
// numpy), k = largest k_j with best >= tau_j.
#include "mc_device.cuh"

namespace mc {

constexpr int MERGE_THREADS = 256;
constexpr int MERGE_WARPS = MERGE_THREADS / 32;

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
__device__ Best2 block_best(Best2 b, Best2* sh, bool warp_uniform) {
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

// ||q||_2 and ||q||_1 of a float64 row held in shared memory (fixed order).
__device__ void q_norms(const double* sq, int D, double* sh, double& n2, double& n1) {
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

__global__ void __launch_bounds__(MERGE_THREADS)
    k_merge(const RingState* __restrict__ d_state, const double* __restrict__ ring64, int D, int Dp,
            const double* __restrict__ q64, const float* __restrict__ part_s, const long long* __restrict__ part_p,
            const float* __restrict__ part_floor, int n_chunks, const double* __restrict__ qscale, double eps_rel,
            double eps_a1, mc_record* __restrict__ rec, ShardMap sm) {
  extern __shared__ double sq[];  // [Dp]
  __shared__ double shd[MERGE_WARPS];
  __shared__ float shf[MERGE_WARPS];
  __shared__ Best2 shb[MERGE_WARPS];
  __shared__ int sh_fail;
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const RingState st = *d_state;
  for (int i = threadIdx.x; i < D; i += blockDim.x) sq[i] = q64[(size_t)b * Dp + i];
  if (threadIdx.x == 0) sh_fail = 0;
  __syncthreads();
  double n2, n1;
  q_norms(sq, D, shd, n2, n1);
  // Non-finite or extreme-magnitude queries leave the fp16/fp32 scan's error
  // model; they are answered by the exhaustive float64 scan instead.
  const bool exotic = !(n1 <= 1e30) || !(n2 >= 1e-30);
  const double scale = qscale ? qscale[b] : 1.0;
  const double delta = eps_rel * n2 + eps_a1 * n1;

  const int ne = n_chunks * KP;
  const float* ps = part_s + (size_t)b * ne;
  const long long* pp = part_p + (size_t)b * ne;
  float m = -INFINITY;
  for (int e = threadIdx.x; e < ne; e += blockDim.x)
    if (pp[e] >= 0) m = fmaxf(m, ps[e]);
  m = block_max(m, shf);
  const double M = (double)m * scale;
  const double thr = M - 2.0 * delta - 1e-9;

  Best2 best;
  best.init();
  for (int e = warp; e < ne; e += MERGE_WARPS) {
    const long long p = pp[e];
    if (p < 0 || (double)ps[e] * scale < thr) continue;  // warp-uniform
    const long long slot = ring_slot(st, local_row(st, p, sm));
    const double v = warp_dot64(ring64 + (size_t)slot * Dp, sq, D, lane);
    best.add(v, p);
  }
  best = block_best(best, shb, true);

  const float* pf = part_floor + (size_t)b * n_chunks;
  int fail = 0;
  for (int c = threadIdx.x; c < n_chunks; c += blockDim.x) {
    const float f = pf[c];
    if (f > -INFINITY && !((double)f * scale + delta < best.s)) fail = 1;
  }
  if (fail) atomicOr(&sh_fail, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    mc_record r;
    r.sim = best.s;
    r.second = best.s2;
    r.pos = best.p;
    r.flags = (best.ties >= 2 ? MC_FLAG_TIE : 0u) | (sh_fail || best.p < 0 ? FLAG_NEED_FALLBACK : 0u) |
              (exotic ? FLAG_NEED_EXHAUSTIVE : 0u);
    r.reserved = 0;
    rec[b] = r;
  }
}

cudaError_t launch_merge(const RingState* d_state, const double* ring64, int D, int Dp, const double* q64, int B,
                         const Partials& part, const double* qscale, double eps_rel, double eps_a1, mc_record* rec,
                         ShardMap sm, cudaStream_t s) {
  const size_t smem = (size_t)Dp * sizeof(double);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_merge<<<B, MERGE_THREADS, smem, s>>>(d_state, ring64, D, Dp, q64, part.s, part.p, part.floor_, part.n_chunks,
                                         qscale, eps_rel, eps_a1, rec, sm);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Exhaustive exact rescan, driven by the merge record's flags:
//   FLAG_NEED_FALLBACK   -> filtered: approx >= rec.sim - delta' - 1e-9, then float64
//   FLAG_NEED_EXHAUSTIVE -> every row in float64 (non-finite / extreme queries;
//                           NaN ordered as numpy's argmax)
// Queries without either flag cost one flag test per CTA.
__device__ __forceinline__ int rescan_mode(unsigned f) {
  return (f & FLAG_NEED_EXHAUSTIVE) ? 2 : ((f & FLAG_NEED_FALLBACK) ? 1 : 0);
}

constexpr int EXACT_THREADS = 256;
constexpr int EXACT_WARPS = EXACT_THREADS / 32;

__global__ void __launch_bounds__(EXACT_THREADS)
    k_exact_scan(const __half* __restrict__ ring16, const double* __restrict__ ring64,
                 const RingState* __restrict__ d_state, int D, int Dp, const double* __restrict__ q64, int B,
                 const mc_record* __restrict__ rec,
                 mc_record* __restrict__ scratch, double eps_rel, double eps_a1, ShardMap sm) {
  extern __shared__ double sq[];  // [Dp] float64 query
  __shared__ double shd[EXACT_WARPS];
  __shared__ Best2 shb[EXACT_WARPS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const RingState st = *d_state;
  const long long n = st.count;
  const int n16 = Dp >> 3;
  for (int b = 0; b < B; ++b) {
    const int md = rescan_mode(rec[b].flags);
    if (md == 0) continue;  // block-uniform
    __syncthreads();
    for (int i = threadIdx.x; i < Dp; i += blockDim.x) sq[i] = q64[(size_t)b * Dp + i];
    __syncthreads();
    double n2 = 0, n1 = 0;
    double thr = -INFINITY;
    if (md == 1) {
      q_norms(sq, D, shd, n2, n1);
      thr = rec[b].sim - (eps_rel * n2 + eps_a1 * n1) - 1e-9;
    }
    Best2 best;
    best.init();
    for (long long row = (long long)blockIdx.x * EXACT_WARPS + warp; row < n;
         row += (long long)gridDim.x * EXACT_WARPS) {
      const long long slot = ring_slot(st, row);
      bool take = (md == 2);
      if (!take) {
        const __half* src = ring16 + (size_t)slot * Dp;
        float acc = 0.f;
        for (int c = lane; c < n16; c += 32) {
          const uint4 v = ld_stream16(src + c * 8);
          const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float2 f = __half22float2(h[t]);
            acc = fmaf(f.x, (float)sq[c * 8 + 2 * t], acc);
            acc = fmaf(f.y, (float)sq[c * 8 + 2 * t + 1], acc);
          }
        }
#pragma unroll
        for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(FULL, acc, off);
        take = (double)acc >= thr;
      }
      if (take) best.add(warp_dot64(ring64 + (size_t)slot * Dp, sq, D, lane), global_pos(st, row, sm));
    }
    best = block_best(best, shb, true);
    if (threadIdx.x == 0) {
      mc_record r;
      r.sim = best.s;
      r.second = best.s2;
      r.pos = best.p;
      r.flags = (unsigned)best.ties;  // tie count carried to the reduce
      r.reserved = 0;
      scratch[(size_t)b * gridDim.x + blockIdx.x] = r;
    }
  }
}

__global__ void k_exact_reduce(const mc_record* __restrict__ scratch, int nparts, mc_record* __restrict__ rec) {
  const int b = blockIdx.x;
  const int md = rescan_mode(rec[b].flags);
  if (md == 0) return;
  __shared__ Best2 shb[EXACT_WARPS];
  Best2 best;
  best.init();
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) {
    const mc_record r = scratch[(size_t)b * nparts + i];
    if (r.pos < 0) continue;
    Best2 o;
    o.s = r.sim;
    o.p = r.pos;
    o.s2 = r.second;
    o.ties = (int)r.flags;
    best.merge(o);
  }
  best = block_best(best, shb, false);
  if (threadIdx.x == 0) {
    mc_record r;
    r.sim = best.s;
    r.second = best.s2;
    r.pos = best.p;
    r.flags = (best.ties >= 2 ? MC_FLAG_TIE : 0u) | (md == 2 ? MC_FLAG_NONFINITE : MC_FLAG_FALLBACK);
    r.reserved = 0;
    rec[b] = r;
  }
}

int exact_grid(int sm_count) { return 2 * sm_count; }

cudaError_t launch_exact_rescan(const __half* ring16, const double* ring64, const RingState* d_state, int D, int Dp,
                                const double* q64, int B, mc_record* rec,
                                mc_record* scratch, int grid, double eps_rel_gemv, double eps_a1, ShardMap sm,
                                cudaStream_t s) {
  const size_t smem = (size_t)Dp * sizeof(double);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_exact_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_exact_scan<<<grid, EXACT_THREADS, smem, s>>>(ring16, ring64, d_state, D, Dp, q64, B, rec, scratch,
                                                 eps_rel_gemv, eps_a1, sm);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_exact_reduce<<<B, EXACT_THREADS, 0, s>>>(scratch, grid, rec);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Decision epilogue: merge G shard records per query, then cache.py:255-260.
__global__ void k_finalize(const mc_record* __restrict__ rec, int G, int B, long long p0,
                           const RingState* __restrict__ d_state, Thresholds thr, OutRec* __restrict__ out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  Best2 best;
  best.init();
  unsigned fl = 0;
  for (int g = 0; g < G; ++g) {
    const mc_record r = rec[(size_t)g * B + b];
    if (r.pos < 0) {  // empty shard (or unanswered query: keep its rescan request)
      if (r.flags != 0xffffffffu) fl |= r.flags & FLAG_NEED_ANY;
      continue;
    }
    fl |= r.flags & (MC_FLAG_FALLBACK | MC_FLAG_NONFINITE | FLAG_NEED_ANY);
    Best2 o;
    o.s = r.sim;
    o.p = r.pos;
    o.s2 = r.second;
    o.ties = (r.flags & MC_FLAG_TIE) ? 2 : 1;
    best.merge(o);
  }
  OutRec o;
  if (best.p < 0) {
    o.live = -1;
    o.sim = __longlong_as_double(0x7ff8000000000000ll);
    o.k = 0;
    o.flags = MC_FLAG_EMPTY | (fl & (FLAG_NEED_FALLBACK | FLAG_NEED_EXHAUSTIVE));
  } else {
    const long long base = p0 >= 0 ? p0 : d_state->jhead;
    o.live = best.p - base;
    o.sim = best.s;
    const double s = best.s;
    unsigned f = fl;
    if (!(s < thr.taus[0])) f |= MC_FLAG_HIT;  // cache.py:258 — `best < tau` is the miss test
    int k = 0;
    for (int j = 0; j < thr.n; ++j) {
      if (s >= thr.taus[j]) k = thr.ks[j];  // cache.py:112-117
      if (fabs(s - thr.taus[j]) < AMBIG) f |= MC_FLAG_NEAR_TAU;
    }
    o.k = k;
    if (best.ties >= 2) f |= MC_FLAG_TIE;
    if (best.s2 != s && s - best.s2 < AMBIG) f |= MC_FLAG_NEAR_TIE;
    o.flags = f;
  }
  out[b] = o;
}

cudaError_t launch_finalize(const mc_record* rec, int G, int B, long long p0, const RingState* d_state,
                            Thresholds thr, OutRec* out, cudaStream_t s) {
  k_finalize<<<(B + 127) / 128, 128, 0, s>>>(rec, G, B, p0, d_state, thr, out);
  return cudaGetLastError();
}

}  // namespace mc
