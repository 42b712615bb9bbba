// K4 — certified float64 rescoring (standalone, for the tensor-core scan),
// the exhaustive fallback, and the shard-merging decision epilogue.
//
// The certificate and the decision rules live in merge.cuh; the GEMV scan
// runs the same code fused into its last CTA.
#include "merge.cuh"

namespace mc {

__global__ void __launch_bounds__(MERGE_THREADS)
    k_merge(const RingState* __restrict__ d_state, const double* __restrict__ ring64, int D, int Dp,
            const double* __restrict__ q64, const float* __restrict__ part_s, const long long* __restrict__ part_p,
            const float* __restrict__ part_floor, int n_chunks, const double* __restrict__ qscale, double eps_rel,
            double eps_a1, mc_record* __restrict__ rec, ShardMap sm, Thresholds thr, OutRec* __restrict__ out) {
  extern __shared__ __align__(16) double sq[];  // [Dp]
  __shared__ MergeScratch ms;
  const int b = blockIdx.x;
  const RingState st = *d_state;
  load_query(q64 + (size_t)b * Dp, D, Dp, sq);
  // Programmatic dependent launch: the query and the ring state were written before the
  // scan's prep kernel started; the candidate lists are read only after the scan is done.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // the next step's query prep may be placed now (it waits for this grid before writing)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const mc_record r = merge_one(st, ring64, D, Dp, sq, part_s + (size_t)b * n_chunks * KP,
                                part_p + (size_t)b * n_chunks * KP, part_floor + (size_t)b * n_chunks, n_chunks,
                                qscale ? qscale[b] : 1.0, eps_rel, eps_a1, sm, ms);
  if (threadIdx.x == 0) {
    rec[b] = r;
    if (out) out[b] = decide_one(r, st.jhead, thr);  // single shard: k_finalize's decision, fused
  }
}

cudaError_t launch_merge(const RingState* d_state, const double* ring64, int D, int Dp, const double* q64, int B,
                         const Partials& part, const double* qscale, double eps_rel, double eps_a1, mc_record* rec,
                         ShardMap sm, const Thresholds* thr, OutRec* out, cudaStream_t s) {
  const size_t smem = (size_t)Dp * sizeof(double);
  if (smem > 32 * 1024) {  // dynamic + the kernel's static smem may pass the 48 KB default
    cudaError_t e = cudaFuncSetAttribute(k_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(B);
  cfg.blockDim = dim3(MERGE_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // griddepcontrol.wait in k_merge
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_merge, d_state, ring64, D, Dp, q64, (const float*)part.s, (const long long*)part.p,
                            (const float*)part.floor_, part.n_chunks, qscale, eps_rel, eps_a1, rec, sm,
                            out ? *thr : Thresholds{}, out);
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
                 const mc_record* __restrict__ rec, mc_record* __restrict__ scratch, double eps_rel, double eps_a1,
                 ShardMap sm) {
  extern __shared__ __align__(16) double sq[];  // [Dp] float64 query
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
    load_query(q64 + (size_t)b * Dp, D, Dp, sq);
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
      if (take) best.add(warp_dot64(ring64 + (size_t)slot * Dp, sq, Dp, lane), global_pos(st, row, sm));
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
                                const double* q64, int B, mc_record* rec, mc_record* scratch, int grid,
                                double eps_rel_gemv, double eps_a1, ShardMap sm, cudaStream_t s) {
  const size_t smem = (size_t)Dp * sizeof(double);
  if (smem > 32 * 1024) {  // dynamic + the kernel's static smem may pass the 48 KB default
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
// Decision epilogue over G shard records per query (shard-major), then
// cache.py:255-260.  p0 < 0 means "read jhead from d_state" (single GPU).
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
    best.merge(record_best(r));
  }
  out[b] = decide(best, fl, p0 >= 0 ? p0 : d_state->jhead, thr);
}

cudaError_t launch_finalize(const mc_record* rec, int G, int B, long long p0, const RingState* d_state,
                            Thresholds thr, OutRec* out, cudaStream_t s) {
  k_finalize<<<(B + 127) / 128, 128, 0, s>>>(rec, G, B, p0, d_state, thr, out);
  return cudaGetLastError();
}

}  // namespace mc
