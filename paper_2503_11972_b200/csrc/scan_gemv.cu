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
#include <cstdlib>

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
  unsigned* gmax;         // [b0 + b] running max approx score (orderable key); zero between launches
  const double* ring64;   // float64 master (rescoring)
  int D;
  double eps_rel, eps_a1;
  Thresholds thr;
  mc_record* rec;         // per-query merged record (rescan requests live in its flags)
  OutRec* out;            // per-query decision (nullptr: records only, e.g. a shard's local answer)
  unsigned long long* timing;  // optional [4]: min start, max scan end, max rescoring end, tail end (ns)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Pending FIFO appends folded into the scan (replaces k_append for small flushes):
// stage rows [0, n) (float64, stride Dp, zero padded) belong to ring slots
// (first_slot + i) mod C; the warp that scans a pending row converts it exactly
// as k_append would and writes both ring copies.
struct GemvAppend {
  const double* stage;
  long long n;
  long long first_slot;
  RingBufs rb;
  RingState* d_state;  // receives the new window (block 0)
};

// One 16-byte chunk (8 values) of a pending row as the fp16 scan sees it.
__device__ __forceinline__ uint4 pending_chunk16(const double* __restrict__ srow, int c) {
  __align__(16) __half hv[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) hv[t] = __double2half(srow[c * 8 + t]);
  return *reinterpret_cast<const uint4*>(hv);
}

__device__ __forceinline__ unsigned ticket_acq_rel(unsigned* counter) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(counter) : "memory");
  return old;
}

__device__ __forceinline__ unsigned order_key(float f) {
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float order_val(unsigned k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

template <int NJ, int NB, int R>
__global__ void __launch_bounds__(GEMV_THREADS, (NJ * NB > 12) ? 1 : 2)
    k_gemv_scan(const __half* __restrict__ ring16, const RingState st, int Dp, const double* __restrict__ q64,
                int nb, CtaRec* __restrict__ cta, int b0, float margin_rel, ShardMap sm, GemvTail tail,
                GemvAppend app) {
  extern __shared__ __align__(16) double sq[];  // [nb][Dp] float64 queries (rescoring), filled by warp 0
  __shared__ float sh_s[NB][GEMV_WARPS * KP];
  __shared__ long long sh_p[NB][GEMV_WARPS * KP];
  __shared__ float sh_run[NB][GEMV_WARPS];
  __shared__ float sh_ovf[NB][GEMV_WARPS];
  __shared__ float sh_gmax[NB];
  __shared__ MergeScratch ms;
  __shared__ int sh_last;

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int n16 = Dp >> 3;  // 16-byte chunks per row
  if (blockIdx.x == 0 && threadIdx.x == 0 && app.d_state) *app.d_state = st;
  if (tail.timing && threadIdx.x == 0) atomicMin(tail.timing + 0, gtimer());

  const long long n = st.count;
  const long long n_warps = (long long)gridDim.x * GEMV_WARPS;
  const long long per = (n + n_warps - 1) / n_warps;
  const long long r0 = ((long long)blockIdx.x * GEMV_WARPS + warp) * per;
  const long long r1 = min(n, r0 + per);
  const long long n_pend = min(app.n, n);      // pending rows still live: the newest n_pend
  const long long pend0 = n - n_pend;          // live-local index of the first of them
  const long long pend_skip = app.n - n_pend;  // stage rows already evicted

  // One batch of R rows: 16-byte loads (lane owns chunks lane + 32 j).  A pending
  // row comes from the stage (float64 -> fp16 RN, as k_append) and is written back.
  auto load_batch = [&](long long base, uint4 (&v)[R][NJ]) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const long long row = base + r;
      if (row < r1 && row < pend0) {
        const __half* src = ring16 + (size_t)ring_slot(st, row) * Dp;
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          const int c = lane + 32 * j;
          v[r][j] = (c < n16) ? ld_stream16(src + c * 8) : make_uint4(0, 0, 0, 0);
        }
      } else if (row < r1) {  // pending row (rare, warp-uniform)
        const double* srow = app.stage + (size_t)(pend_skip + row - pend0) * Dp;
        write_row_all(srow, ring_slot(st, row), app.rb, Dp, lane);
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          const int c = lane + 32 * j;
          v[r][j] = (c < n16) ? pending_chunk16(srow, c) : make_uint4(0, 0, 0, 0);
        }
      } else {
#pragma unroll
        for (int j = 0; j < NJ; ++j) v[r][j] = make_uint4(0, 0, 0, 0);
      }
    }
  };

  // First batch in flight before the query loads, so both latencies overlap.
  uint4 v[R][NJ];
  load_batch(r0, v);

  // Query in fp32 registers; delta (= eps_rel ||q||_2 + eps_a1 ||q||_1, float64)
  // and the admission margin 2.02 delta + fp32 slack per query.  A non-finite
  // query gives a NaN margin: nothing is admitted, and the tail routes it to
  // the exhaustive float64 scan.
  float q[NB][NJ][8];
  float margin[NB];
  double delta[NB];
  bool exotic[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    double a2 = 0.0, a1 = 0.0;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int c = lane + 32 * j;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const double x = (b < nb && c < n16 && c * 8 + t < tail.D) ? q64[(size_t)b * Dp + c * 8 + t] : 0.0;
        if (warp == 0 && b < nb && c < n16) sq[(size_t)b * Dp + c * 8 + t] = x;
        q[b][j][t] = (float)x;
        a2 = fma(x, x, a2);
        a1 += fabs(x);
      }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      a2 += __shfl_xor_sync(FULL, a2, off);
      a1 += __shfl_xor_sync(FULL, a1, off);
    }
    // Rounded up past any summation-order difference with the host/merge norms.
    const double n2 = sqrt(a2) * (1.0 + 1e-12), n1 = a1 * (1.0 + 1e-12);
    exotic[b] = !(n1 <= 1e30) || !(n2 >= 1e-30);
    delta[b] = tail.eps_rel * n2 + tail.eps_a1 * n1;
    margin[b] = (float)(2.02 * delta[b]) + margin_rel * (float)n2;
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

  for (long long base = r0; base < r1; base += R) {
    if (base != r0) load_batch(base, v);
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
  if (tail.timing && lane == 0) atomicMax(tail.timing + 1, gtimer());
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
  __syncthreads();
  // Publish this CTA's approximate maxima; a CTA more than 2 delta below the
  // running global maximum holds no row that can reach (or tie within 1e-9)
  // the certified best, so it skips the float64 rescoring.
  if (threadIdx.x < nb) {
    const int b = threadIdx.x;
    float mc = -INFINITY;
#pragma unroll
    for (int w = 0; w < GEMV_WARPS; ++w) mc = fmaxf(mc, sh_run[b][w]);
    const unsigned mine = order_key(mc);
    const unsigned old = atomicMax(tail.gmax + b0 + b, mine);
    sh_gmax[b] = order_val(old > mine ? old : mine);
  }
  __syncthreads();
  for (int b = 0; b < nb; ++b) {
    float mc = -INFINITY, ov = -INFINITY;
#pragma unroll
    for (int w = 0; w < GEMV_WARPS; ++w) {
      mc = fmaxf(mc, sh_run[b][w]);
      ov = fmaxf(ov, sh_ovf[b][w]);
    }
    const double d2 = 2.0 * delta[b] + 1e-9;
    Best2 best;
    best.init();
    if (mc > -INFINITY && (double)mc >= (double)sh_gmax[b] - d2) {  // block-uniform
      const double thr = (double)mc - d2;
      for (int e = warp; e < GEMV_WARPS * KP; e += GEMV_WARPS) {
        const long long p = sh_p[b][e];
        if (p < 0 || (double)sh_s[b][e] < thr) continue;  // warp-uniform
        const long long l = local_row(st, p, sm);
        // a row appended by this launch is read from the stage (the ring copy
        // was written in this kernel and is not visible to the read-only path)
        const double* row = l >= pend0 ? app.stage + (size_t)(pend_skip + l - pend0) * Dp
                                        : tail.ring64 + (size_t)ring_slot(st, l) * Dp;
        best.add(warp_dot64(row, sq + (size_t)b * Dp, Dp, lane), p);
      }
      best = block_best(best, ms.shb, true);
    }
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

  if (tail.timing && threadIdx.x == 0) atomicMax(tail.timing + 2, gtimer());
  if (!tail.counter) return;
  // ---------------------------------------------------------------- fused tail
  // Thread 0 wrote this CTA's records; its acq_rel ticket releases them and, on
  // the last CTA, acquires everyone else's (then bar.sync shares that view).
  if (threadIdx.x == 0) sh_last = ticket_acq_rel(tail.counter) == gridDim.x - 1;
  __syncthreads();
  if (!sh_last) return;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    if (b >= nb) break;
    const int gb = b0 + b;
    const double dl = delta[b];
    Best2 best;
    best.init();
    float ov = -INFINITY;
    for (int c = threadIdx.x; c < (int)gridDim.x; c += blockDim.x) {
      CtaRec r;
      const CtaRec* src = cta + (size_t)gb * gridDim.x + c;
      r.s = __ldcg(&src->s);
      r.s2 = __ldcg(&src->s2);
      r.p = __ldcg(&src->p);
      r.ovf = __ldcg(&src->ovf);
      r.ties = __ldcg(&src->ties);
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
      const bool fail = best.p < 0 || !(ov == -INFINITY || (double)ov + dl + 1e-9 < best.s);
      mc_record r;
      r.sim = best.s;
      r.second = best.s2;
      r.pos = best.p;
      r.flags = (best.ties >= 2 ? MC_FLAG_TIE : 0u) | (fail ? FLAG_NEED_FALLBACK : 0u) |
                (exotic[b] ? FLAG_NEED_EXHAUSTIVE : 0u);
      r.reserved = 0;
      tail.rec[gb] = r;
      if (tail.out) tail.out[gb] = decide(record_best(r), r.flags & FLAG_NEED_ANY, st.jhead, tail.thr);
      tail.gmax[gb] = 0u;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *tail.counter = 0u;
    if (tail.timing) tail.timing[3] = gtimer();
  }
}

int gemv_grid(int sm_count) { return 2 * sm_count; }

// MC_GEMV_TIMING=1: every GEMV launch records phase timestamps (measurement only).
static unsigned long long* g_timing = nullptr;
unsigned long long* gemv_timing_buffer() {
  static bool init = false;
  if (!init) {
    init = true;
    const char* e = getenv("MC_GEMV_TIMING");
    if (e && atoi(e) && cudaMalloc(&g_timing, (8 + 12 * 512) * sizeof(unsigned long long)) == cudaSuccess) {
      cudaMemset(g_timing, 0, (8 + 12 * 512) * sizeof(unsigned long long));
      const unsigned long long init8[8] = {~0ull, 0, 0, 0, 0, 0, 0, 0};
      cudaMemcpy(g_timing, init8, sizeof init8, cudaMemcpyHostToDevice);
    }
  }
  return g_timing;
}

// Rows streamed per warp iteration: ~18 16-byte loads in flight per lane per query.
constexpr int rows_for(int NJ, int NB) {
  const int r = 18 / (NJ * NB);
  return r < 1 ? 1 : (r > 8 ? 8 : r);
}

template <int NJ, int NB>
static cudaError_t launch_one(const __half* ring16, const RingState& st, int Dp, const double* q64, int nb,
                              CtaRec* cta, int b0, int grid, float margin_rel, ShardMap sm, const GemvTail& tail,
                              const GemvAppend& app, cudaStream_t s) {
  constexpr int R = rows_for(NJ, NB);
  auto kern = k_gemv_scan<NJ, NB, R>;
  const size_t smem = (size_t)NB * Dp * sizeof(double);
  if (smem > 32 * 1024) {  // dynamic + the kernel's static smem may pass the 48 KB default
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  kern<<<grid, GEMV_THREADS, smem, s>>>(ring16, st, Dp, q64, nb, cta, b0, margin_rel, sm, tail, app);
  return cudaGetLastError();
}

template <int NJ>
static cudaError_t launch_nj(const __half* ring16, const RingState& st, int Dp, const double* q64, int nb,
                             CtaRec* cta, int b0, int grid, float margin_rel, ShardMap sm, const GemvTail& tail,
                             const GemvAppend& app, cudaStream_t s) {
  if (nb == 1) return launch_one<NJ, 1>(ring16, st, Dp, q64, nb, cta, b0, grid, margin_rel, sm, tail, app, s);
  if (nb == 2) return launch_one<NJ, 2>(ring16, st, Dp, q64, nb, cta, b0, grid, margin_rel, sm, tail, app, s);
  return launch_one<NJ, 4>(ring16, st, Dp, q64, nb, cta, b0, grid, margin_rel, sm, tail, app, s);
}

unsigned long long* gemv_timing_buffer();

cudaError_t launch_gemv_scan(const __half* ring16, const RingState& st, int D, int Dp, const double* q64, int nb,
                             CtaRec* cta, int b0, int grid, ShardMap sm, unsigned* counter, unsigned* gmax,
                             const double* ring64, const Thresholds& thr, mc_record* rec, OutRec* out,
                             const GemvAppendArgs& a, cudaStream_t s) {
  const int nj = (Dp / 8 + 31) / 32;
  if (nb < 1 || nb > 4) return cudaErrorInvalidValue;
  GemvTail tail{counter, gmax, ring64, D, gemv_eps_rel(Dp), eps_abs1(), thr, rec, out, gemv_timing_buffer()};
  GemvAppend app{a.stage, a.n, a.first_slot, a.rb, a.d_state};
  const float mrel = 1e-6f;  // slack for the fp32 arithmetic of the admission test
#define MC_GEMV_CASE(NJV) return launch_nj<NJV>(ring16, st, Dp, q64, nb, cta, b0, grid, mrel, sm, tail, app, s)
  switch (nj) {
    case 1: MC_GEMV_CASE(1);
    case 2: MC_GEMV_CASE(2);
    case 3: MC_GEMV_CASE(3);
    case 4: MC_GEMV_CASE(4);
    case 5: case 6: MC_GEMV_CASE(6);
    case 7: case 8: MC_GEMV_CASE(8);
    default:
      if (nj <= 12) MC_GEMV_CASE(12);
      if (nj <= 16) MC_GEMV_CASE(16);
      return cudaErrorInvalidValue;
  }
#undef MC_GEMV_CASE
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
