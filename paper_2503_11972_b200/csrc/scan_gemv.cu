// K2 — batch-1..4 GEMV scan over the fp16 ring (HBM-bound path), with the
// certified merge and the decision fused into the last CTA to finish.
//
// Replaces the OpenBLAS dgemv of cache.py:254 for small batches.  Each warp
// owns a contiguous run of live rows and streams R rows at a time with
// 16-byte `ld.global.nc.L1::no_allocate` loads (R * NJ loads in flight per
// lane, ~150 KB per SM), converts fp16 -> fp32, FMAs against the fp32 query
// held in registers and reduces with a 5-step xor butterfly (every lane ends
// with the same bits).  Scores never leave registers: each warp keeps a
// sorted top-K' over lanes 0..K'-1, admitting only scores above both the
// K'-th kept score and (running max - margin), where margin > 2 delta.
//
// Certified rescoring, per CTA.  A score x pruned by the margin rule has
// exact(x) <= x + delta < runmax - delta <= exact(running-max row), so it can
// never be (or tie) the best.  Each CTA therefore rescores in float64 only its
// listed rows within 2 delta (+1e-9) of its approximate maximum — every row
// it skips is strictly below a rescored one — and publishes one exact record
// (best, runner-up, ties) plus `ovf`, the largest score a full warp list had
// to drop while it was still within the margin.  Certificate: ovf + delta <
// the global exact best, else the exhaustive rescan answers (rescore.cu).
//
// Fused tail: every CTA bumps a device counter after writing its record; the
// last one reduces the records of each query (Best2 merge + certificate) and
// writes the decision, so one launch does scan + rescoring + epilogue.
//
// Algorithmic bytes per lookup batch: count * Dp * 2 (the fp16 ring) + Dp * 8 per query.
#include "merge.cuh"

namespace mc {

constexpr int GEMV_THREADS = 256;
constexpr int GEMV_WARPS = GEMV_THREADS / 32;

__device__ __forceinline__ void fma8(float& acc, const uint4& v, const float* q) {
  const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const float2 f = __half22float2(h[t]);
    acc = fmaf(f.x, q[2 * t], acc);
    acc = fmaf(f.y, q[2 * t + 1], acc);
  }
}

struct GemvTail {
  unsigned* counter;      // zero between launches; the last CTA resets it
  const double* ring64;   // float64 master (rescoring)
  int D;
  double eps_rel, eps_a1;
  Thresholds thr;
  mc_record* rec;         // per-query merged record (rescan requests live in its flags)
  OutRec* out;            // per-query decision (nullptr: records only, e.g. a shard's local answer)
};

template <int NJ, int NB, int R>
__global__ void __launch_bounds__(GEMV_THREADS, (NJ * NB > 12) ? 1 : 2)
    k_gemv_scan(const __half* __restrict__ ring16, const RingState* __restrict__ d_state, int Dp,
                const double* __restrict__ q64, int nb, CtaRec* __restrict__ cta, int b0, float margin_rel,
                ShardMap sm, GemvTail tail) {
  extern __shared__ __align__(16) double sq[];  // [Dp] float64 query (rescoring)
  __shared__ float sh_s[NB][GEMV_WARPS * KP];
  __shared__ long long sh_p[NB][GEMV_WARPS * KP];
  __shared__ float sh_run[NB][GEMV_WARPS];
  __shared__ float sh_ovf[NB][GEMV_WARPS];
  __shared__ MergeScratch ms;
  __shared__ int sh_last;

  const RingState st = *d_state;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int n16 = Dp >> 3;  // 16-byte chunks per row

  // Query in fp32 registers: lane owns chunks lane + 32*j; admission margin per
  // query = 2.02 delta (delta = eps_rel ||q||_2 + eps_a1 ||q||_1) + fp32 slack.
  // A non-finite query gives a NaN margin: nothing is admitted, and the tail
  // routes it to the exhaustive float64 scan.
  float q[NB][NJ][8];
  float margin[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    float a2 = 0.f, a1 = 0.f;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int c = lane + 32 * j;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const float x = (b < nb && c < n16) ? (float)q64[(size_t)b * Dp + c * 8 + t] : 0.f;
        q[b][j][t] = x;
        a2 = fmaf(x, x, a2);
        a1 += fabsf(x);
      }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      a2 += __shfl_xor_sync(FULL, a2, off);
      a1 += __shfl_xor_sync(FULL, a1, off);
    }
    margin[b] = 2.02f * (float)(tail.eps_rel * sqrt((double)a2) + tail.eps_a1 * (double)a1) * 1.001f +
                margin_rel * sqrtf(a2);
  }

  // Per-warp sorted top-K': lane k < KP holds the k-th best (score, pos).
  float ls[NB], wmin[NB], runmax[NB], ovf[NB];
  long long lp[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    ls[b] = -INFINITY;
    lp[b] = -1;
    wmin[b] = -INFINITY;
    runmax[b] = -INFINITY;
    ovf[b] = -INFINITY;
  }

  const long long n = st.count;
  const long long n_warps = (long long)gridDim.x * GEMV_WARPS;
  const long long per = (n + n_warps - 1) / n_warps;
  const long long r0 = ((long long)blockIdx.x * GEMV_WARPS + warp) * per;
  const long long r1 = min(n, r0 + per);

  for (long long base = r0; base < r1; base += R) {
    uint4 v[R][NJ];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const long long row = base + r;
      if (row < r1) {
        const __half* src = ring16 + (size_t)ring_slot(st, row) * Dp;
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          const int c = lane + 32 * j;
          v[r][j] = (c < n16) ? ld_stream16(src + c * 8) : make_uint4(0, 0, 0, 0);
        }
      } else {
#pragma unroll
        for (int j = 0; j < NJ; ++j) v[r][j] = make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const long long row = base + r;
      if (row >= r1) break;  // warp-uniform
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < NJ; ++j) fma8(acc, v[r][j], q[b][j]);
#pragma unroll
        for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(FULL, acc, off);
        if (b >= nb) continue;
        // acc, wmin, runmax are identical in every lane: the branches are warp-uniform
        runmax[b] = fmaxf(runmax[b], acc);
        const float lo = runmax[b] - margin[b];
        if (acc > fmaxf(wmin[b], lo)) {
          const long long last_p = __shfl_sync(FULL, lp[b], KP - 1);
          if (last_p >= 0) ovf[b] = fmaxf(ovf[b], wmin[b]);  // evicted from a full list
          const unsigned ahead = __ballot_sync(FULL, lane < KP && ls[b] >= acc);
          const int at = __popc(ahead);
          const float up_s = __shfl_up_sync(FULL, ls[b], 1);
          const long long up_p = __shfl_up_sync(FULL, lp[b], 1);
          if (lane == at) {
            ls[b] = acc;
            lp[b] = global_pos(st, row, sm);
          } else if (lane > at && lane < KP) {
            ls[b] = up_s;
            lp[b] = up_p;
          }
          wmin[b] = __shfl_sync(FULL, ls[b], KP - 1);
        } else if (acc > lo) {
          ovf[b] = fmaxf(ovf[b], acc);  // within the margin but the list is full
        }
      }
    }
  }

  // ---------------------------------------------------------------- CTA rescoring
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    if (lane < KP) {
      sh_s[b][warp * KP + lane] = ls[b];
      sh_p[b][warp * KP + lane] = lp[b];
    }
    if (lane == 0) {
      sh_run[b][warp] = runmax[b];
      sh_ovf[b][warp] = ovf[b];
    }
  }
  for (int b = 0; b < nb; ++b) {
    load_query(q64 + (size_t)b * Dp, tail.D, Dp, sq);  // ends with __syncthreads
    double n2, n1;
    q_norms(sq, tail.D, ms.shd, n2, n1);
    const double delta = tail.eps_rel * n2 + tail.eps_a1 * n1;
    float mc = -INFINITY, ov = -INFINITY;
#pragma unroll
    for (int w = 0; w < GEMV_WARPS; ++w) {
      mc = fmaxf(mc, sh_run[b][w]);
      ov = fmaxf(ov, sh_ovf[b][w]);
    }
    const double thr = (double)mc - 2.0 * delta - 1e-9;
    Best2 best;
    best.init();
    for (int e = warp; e < GEMV_WARPS * KP; e += GEMV_WARPS) {
      const long long p = sh_p[b][e];
      if (p < 0 || (double)sh_s[b][e] < thr) continue;  // warp-uniform
      const long long slot = ring_slot(st, local_row(st, p, sm));
      best.add(warp_dot64(tail.ring64 + (size_t)slot * Dp, sq, Dp, lane), p);
    }
    best = block_best(best, ms.shb, true);
    if (threadIdx.x == 0) {
      CtaRec r;
      r.s = best.s;
      r.s2 = best.s2;
      r.p = best.p;
      r.ovf = ov;
      r.ties = best.ties;
      cta[(size_t)(b0 + b) * gridDim.x + blockIdx.x] = r;
    }
  }

  if (!tail.counter) return;
  // ---------------------------------------------------------------- fused tail
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) sh_last = atomicAdd(tail.counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!sh_last) return;
  __threadfence();
  for (int b = 0; b < nb; ++b) {
    const int gb = b0 + b;
    load_query(q64 + (size_t)b * Dp, tail.D, Dp, sq);
    double n2, n1;
    q_norms(sq, tail.D, ms.shd, n2, n1);
    const bool exotic = !(n1 <= 1e30) || !(n2 >= 1e-30);
    const double delta = tail.eps_rel * n2 + tail.eps_a1 * n1;
    Best2 best;
    best.init();
    float ov = -INFINITY;
    for (int c = threadIdx.x; c < (int)gridDim.x; c += blockDim.x) {
      const CtaRec r = cta[(size_t)gb * gridDim.x + c];
      ov = fmaxf(ov, r.ovf);
      if (r.p < 0) continue;
      Best2 o;
      o.s = r.s;
      o.p = r.p;
      o.s2 = r.s2;
      o.ties = r.ties;
      best.merge(o);
    }
    best = block_best(best, ms.shb, false);
    ov = block_max(ov, ms.shf);
    if (threadIdx.x == 0) {
      const bool fail = best.p < 0 || !(ov == -INFINITY || (double)ov + delta < best.s);
      mc_record r;
      r.sim = best.s;
      r.second = best.s2;
      r.pos = best.p;
      r.flags = (best.ties >= 2 ? MC_FLAG_TIE : 0u) | (fail ? FLAG_NEED_FALLBACK : 0u) |
                (exotic ? FLAG_NEED_EXHAUSTIVE : 0u);
      r.reserved = 0;
      tail.rec[gb] = r;
      if (tail.out) tail.out[gb] = decide(record_best(r), r.flags & FLAG_NEED_ANY, st.jhead, tail.thr);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *tail.counter = 0u;
}

int gemv_grid(int sm_count) { return 2 * sm_count; }

// Rows streamed per warp iteration: ~18 16-byte loads in flight per lane per query.
constexpr int rows_for(int NJ, int NB) {
  const int r = 18 / (NJ * NB);
  return r < 1 ? 1 : (r > 8 ? 8 : r);
}

template <int NJ, int NB>
static cudaError_t launch_one(const __half* ring16, const RingState* d_state, int Dp, const double* q64, int nb,
                              CtaRec* cta, int b0, int grid, float margin_rel, ShardMap sm, const GemvTail& tail,
                              cudaStream_t s) {
  constexpr int R = rows_for(NJ, NB);
  auto kern = k_gemv_scan<NJ, NB, R>;
  const size_t smem = (size_t)Dp * sizeof(double);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  kern<<<grid, GEMV_THREADS, smem, s>>>(ring16, d_state, Dp, q64, nb, cta, b0, margin_rel, sm, tail);
  return cudaGetLastError();
}

template <int NJ>
static cudaError_t launch_nj(const __half* ring16, const RingState* d_state, int Dp, const double* q64, int nb,
                             CtaRec* cta, int b0, int grid, float margin_rel, ShardMap sm, const GemvTail& tail,
                             cudaStream_t s) {
  if (nb == 1) return launch_one<NJ, 1>(ring16, d_state, Dp, q64, nb, cta, b0, grid, margin_rel, sm, tail, s);
  if (nb == 2) return launch_one<NJ, 2>(ring16, d_state, Dp, q64, nb, cta, b0, grid, margin_rel, sm, tail, s);
  return launch_one<NJ, 4>(ring16, d_state, Dp, q64, nb, cta, b0, grid, margin_rel, sm, tail, s);
}

cudaError_t launch_gemv_scan(const __half* ring16, const RingState* d_state, int D, int Dp, const double* q64,
                             int nb, CtaRec* cta, int b0, int grid, ShardMap sm, unsigned* counter,
                             const double* ring64, const Thresholds& thr, mc_record* rec, OutRec* out,
                             cudaStream_t s) {
  const int nj = (Dp / 8 + 31) / 32;
  if (nb < 1 || nb > 4) return cudaErrorInvalidValue;
  GemvTail tail{counter, ring64, D, gemv_eps_rel(Dp), eps_abs1(), thr, rec, out};
  const float mrel = 1e-6f;  // slack for the fp32 arithmetic of the admission test
  switch (nj) {
    case 1: return launch_nj<1>(ring16, d_state, Dp, q64, nb, cta, b0, grid, mrel, sm, tail, s);
    case 2: return launch_nj<2>(ring16, d_state, Dp, q64, nb, cta, b0, grid, mrel, sm, tail, s);
    case 3: return launch_nj<3>(ring16, d_state, Dp, q64, nb, cta, b0, grid, mrel, sm, tail, s);
    case 4: return launch_nj<4>(ring16, d_state, Dp, q64, nb, cta, b0, grid, mrel, sm, tail, s);
    case 5: case 6: return launch_nj<6>(ring16, d_state, Dp, q64, nb, cta, b0, grid, mrel, sm, tail, s);
    case 7: case 8: return launch_nj<8>(ring16, d_state, Dp, q64, nb, cta, b0, grid, mrel, sm, tail, s);
    default:
      if (nj <= 12) return launch_nj<12>(ring16, d_state, Dp, q64, nb, cta, b0, grid, mrel, sm, tail, s);
      if (nj <= 16) return launch_nj<16>(ring16, d_state, Dp, q64, nb, cta, b0, grid, mrel, sm, tail, s);
      return cudaErrorInvalidValue;
  }
}

// fp32 accumulation depth of one GEMV score: NJ*8 sequential FMAs + 5 butterfly adds.
double gemv_eps_rel(int Dp) {
  const int nj = (Dp / 8 + 31) / 32;
  const double u16 = ldexp(1.0, -11), u32 = ldexp(1.0, -24);
  const double n_acc = nj * 8 + 5;
  // |e16 - e| <= u16 |e|, |q32 - q| <= u32 |q|, products of unit-ish vectors,
  // accumulation gamma_n <= 1.01 n u32; sum |e||q| <= ||e|| ||q|| <= (1+1e-6) ||q||.
  const double rel = (1.0 + 1e-6) * ((u16 + u32 + u16 * u32) * (1.0 + 1.01 * n_acc * u32) + 1.01 * n_acc * u32);
  return 1.25 * rel;  // safety factor
}

// Absolute term per unit of ||q||_1: fp16 subnormal rounding (half spacing 2^-25).
double eps_abs1() { return 1.25 * ldexp(1.0, -25); }

}  // namespace mc
