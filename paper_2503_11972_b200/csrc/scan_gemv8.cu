// K2q — batch-1..4 scan over the int8 ring copy (HBM-bound path, half the
// bytes of the fp16 scan), with the same fused certified merge as K2.
//
// Storage: ring row e is kept as int8 ê = rint(e / s_e) with a per-row scale
// s_e >= max|e|/127 (rounded up) and L1_e >= ||e||_1 (rq[slot] = (s_e, L1_e)).
// The query is quantised per lookup the same way (s_q, q̂).  A row's score is
// the exact int32 dot Σ ê_i q̂_i (dp4a) times s_e s_q, with the rigorous bound
//   |e·q - s_e s_q Σ ê_i q̂_i| <= ½ s_q ||e||_1 + ½ s_e s_q ||q̂||_1 = delta_e
// (|e_i - s_e ê_i| <= s_e/2, |q_i - s_q q̂_i| <= s_q/2), so each row carries an
// upper bound u = approx + delta_e and a lower bound l = approx - delta_e.
//
// Certificate (as K2, with per-row bounds).  A warp tracks lo = max l; a row
// with u < lo - 1e-9 is strictly (>= 1e-9) below the row that set lo and is
// pruned.  Kept rows go to a sorted top-K' by u; rows a full list drops raise
// `ovf` (max u dropped).  Each CTA rescores in float64 its listed rows with
// u >= lo_cta - 1e-9, unless its best u is below the running global lo
// (atomicMax).  The last CTA merges the per-CTA exact records; certificate:
// ovf + 1e-9 < best, else the exhaustive rescan (rescore.cu) answers.
//
// Loads: a group of G rows is G * N16 16-byte chunks, a multiple of 32; lane l
// takes chunks l, l+32, ... so every warp load is 512 contiguous bytes even
// when a row is not a multiple of 512 bytes (e.g. 768-dim rows).
//
// Pending appends (rows added since the last lookup) are not in the int8 scan:
// CTA 0 writes them to every ring copy and scores them exactly (float64, from
// the stage) in its rescoring phase.
//
// Algorithmic bytes per launch: count * (Dp + 8) + nb * Dp * 8.
#include <cstdlib>

#include "merge.cuh"

namespace mc {

constexpr int G8_THREADS = 256;
constexpr int G8_WARPS = G8_THREADS / 32;

__device__ __forceinline__ unsigned key_of(float f) {
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float val_of(unsigned k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

__device__ __forceinline__ int dp16(const uint4& a, const uint4& b, int acc) {
  acc = __dp4a((int)a.x, (int)b.x, acc);
  acc = __dp4a((int)a.y, (int)b.y, acc);
  acc = __dp4a((int)a.z, (int)b.z, acc);
  return __dp4a((int)a.w, (int)b.w, acc);
}

struct Gemv8Tail {
  unsigned* counter;
  unsigned* gmax;  // [b0 + b] running max of lo (orderable key); zero between launches
  int D;
  Thresholds thr;
  mc_record* rec;
  OutRec* out;
  unsigned long long* timing;  // optional phase stamps (MC_GEMV_TIMING=1)
  const QPrep* prep;           // [nb] per-query quantisation (host-computed, in the envelope)
  const int8_t* q8;            // [nb][Dp] q̂
};

unsigned long long* gemv_timing_buffer();

__device__ __forceinline__ unsigned long long gtimer8() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct Gemv8Append {
  const double* stage;
  long long n;
  RingState* d_state;
};

template <int N16, int LOADS>
struct Geom {
  static constexpr int gcd(int a, int b) { return b ? gcd(b, a % b) : a; }
  static constexpr int G = 32 / gcd(N16, 32);        // rows per group
  static constexpr int LPG = G * N16 / 32;           // 16-byte loads per lane per group
  static constexpr int RG0 = LOADS / LPG > 0 ? LOADS / LPG : 1;
  static constexpr int RG = RG0 * G > 32 ? 32 / G : RG0;  // groups per batch (<= 32 rows)
  static constexpr int ROWS = RG * G;
};

template <int N16, int NB>
__global__ void __launch_bounds__(G8_THREADS, NB == 1 ? 2 : 1)
    k_gemv8_scan(RingBufs rb, const RingState st, const double* __restrict__ q64, int nb, CtaRec* __restrict__ cta,
                 int b0, ShardMap sm, Gemv8Tail tail, Gemv8Append app) {
  using Gm = Geom<N16, 12>;  // ~12 16-byte loads in flight per lane (2 CTAs / SM measured best)
  constexpr int G = Gm::G, LPG = Gm::LPG, RG = Gm::RG, ROWS = Gm::ROWS;
  constexpr int Dp = N16 * 16;
  extern __shared__ __align__(16) double sq[];  // [nb][Dp] float64 queries (rescoring)
  __shared__ float sh_u[NB][G8_WARPS * KP];
  __shared__ long long sh_p[NB][G8_WARPS * KP];
  __shared__ double sh_lo[NB][G8_WARPS];
  __shared__ float sh_ovf[NB][G8_WARPS];
  __shared__ float sh_g[NB];
  __shared__ MergeScratch ms;
  __shared__ int sh_last;
  __shared__ uint4 sh_qc[NB > 1 ? NB : 1][N16];  // q̂ chunks (read per use when NB > 1)

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  if (blockIdx.x == 0 && threadIdx.x == 0 && app.d_state) *app.d_state = st;
  if (tail.timing && threadIdx.x == 0) atomicMin(tail.timing + 0, gtimer8());

  const long long n = st.count;
  const long long n_pend = min(app.n, n);
  const long long pend0 = n - n_pend;  // rows [pend0, n) are scored exactly by CTA 0
  const long long n_warps = (long long)gridDim.x * G8_WARPS;
  const long long per = (pend0 + n_warps - 1) / n_warps;
  const long long r0 = ((long long)blockIdx.x * G8_WARPS + warp) * per;
  const long long r1 = min(pend0, r0 + per);

  // ---- batch loads (issued before the query prologue to overlap the latencies)
  auto load_batch = [&](long long base, uint4 (&v)[RG][LPG], float2& rq) {
#pragma unroll
    for (int g = 0; g < RG; ++g)
#pragma unroll
      for (int j = 0; j < LPG; ++j) {
        const int f = lane + 32 * j;
        const long long row = base + g * G + f / N16;
        v[g][j] = row < r1 ? ld_stream16(rb.r8 + (size_t)ring_slot(st, row) * rb.p8 + (f % N16) * 16)
                           : make_uint4(0, 0, 0, 0);
      }
    const long long row = base + lane;
    rq = (lane < ROWS && row < r1) ? __ldg(rb.rq + ring_slot(st, row)) : make_float2(0.f, 0.f);
  };
  uint4 v[RG][LPG];
  float2 rq;
  load_batch(r0, v, rq);

  // ---- query side: q̂ chunks + scalars quantised by the host (quantize_query)
  uint4 qr[LPG];
  double sq8[NB], q1[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const QPrep pq = b < nb ? tail.prep[b] : QPrep{0.0, 0.0, 0.0, 0.f, 0};
    sq8[b] = pq.s;
    q1[b] = pq.q1;
    const uint4* qc = reinterpret_cast<const uint4*>(tail.q8 + (size_t)b * Dp);
    if constexpr (NB == 1) {
#pragma unroll
      for (int j = 0; j < LPG; ++j) qr[j] = qc[(lane + 32 * j) % N16];
    } else {
      if (warp == 0)
        for (int col = lane; col < N16; col += 32) sh_qc[b][col] = b < nb ? qc[col] : make_uint4(0, 0, 0, 0);
    }
  }
  if constexpr (NB > 1) __syncthreads();

  // ---- per-warp state: sorted top-K' by upper bound u over lanes 0..K'-1
  // gk: the best known global lower bound (some row's l, possibly another warp's;
  // published / refreshed through the gmax word whenever this warp's lo passes it)
  float lu[NB], wmin[NB], ovf[NB], gk[NB];
  long long lp[NB];
  double lo[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    lu[b] = -INFINITY;
    lp[b] = -1;
    wmin[b] = -INFINITY;
    ovf[b] = -INFINITY;
    lo[b] = -INFINITY;
    gk[b] = -INFINITY;
  }

  for (long long base = r0; base < r1; base += ROWS) {
    if (base != r0) load_batch(base, v, rq);
#pragma unroll
    for (int g = 0; g < RG; ++g) {
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        int part[G];
#pragma unroll
        for (int t = 0; t < G; ++t) part[t] = 0;
#pragma unroll
        for (int j = 0; j < LPG; ++j) {
          const int rg = (lane + 32 * j) / N16;
          uint4 qv;
          if constexpr (NB == 1)
            qv = qr[j];
          else
            qv = sh_qc[b][(lane + 32 * j) % N16];
          const int d = dp16(v[g][j], qv, 0);
#pragma unroll
          for (int t = 0; t < G; ++t) part[t] += (rg == t) ? d : 0;
        }
#pragma unroll
        for (int t = 0; t < G; ++t) {
#pragma unroll
          for (int off = 16; off; off >>= 1) part[t] += __shfl_xor_sync(FULL, part[t], off);
        }
        if (b >= nb) continue;
#pragma unroll
        for (int t = 0; t < G; ++t) {
          const long long row = base + g * G + t;
          if (row >= r1) break;  // warp-uniform
          const float2 e = make_float2(__shfl_sync(FULL, rq.x, g * G + t), __shfl_sync(FULL, rq.y, g * G + t));
          const double approx = (double)part[t] * ((double)e.x * sq8[b]);
          const double dl = (0.5 * sq8[b] * (double)e.y + 0.5 * (double)e.x * q1[b]) * (1.0 + 1e-9) + 1e-12;
          const double u = approx + dl, l = approx - dl;
          lo[b] = fmax(lo[b], l);
          if (u < fmax(lo[b], (double)gk[b]) - 1e-9) continue;  // strictly below a row with l >= that
          const float uf = __double2float_ru(u);
          if (uf > wmin[b]) {
            const long long last_p = __shfl_sync(FULL, lp[b], KP - 1);
            if (last_p >= 0) ovf[b] = fmaxf(ovf[b], wmin[b]);  // evicted from a full list
            const unsigned ahead = __ballot_sync(FULL, lane < KP && lu[b] >= uf);
            const int at = __popc(ahead);
            const float up_u = __shfl_up_sync(FULL, lu[b], 1);
            const long long up_p = __shfl_up_sync(FULL, lp[b], 1);
            if (lane == at) {
              lu[b] = uf;
              lp[b] = global_pos(st, row, sm);
            } else if (lane > at && lane < KP) {
              lu[b] = up_u;
              lp[b] = up_p;
            }
            wmin[b] = __shfl_sync(FULL, lu[b], KP - 1);
          } else {
            ovf[b] = fmaxf(ovf[b], uf);  // kept by the bound but the list is full
          }
        }
      }
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const float lf = __double2float_rd(lo[b]);
      if (b < nb && lf > gk[b]) {  // warp-uniform: share this warp's bound, learn the global one
        float g = lf;
        if (lane == 0) {
          const unsigned mine = key_of(lf);
          const unsigned old = atomicMax(tail.gmax + b0 + b, mine);
          g = val_of(old > mine ? old : mine);
        }
        gk[b] = __shfl_sync(FULL, g, 0);
      }
    }
  }

  // ---------------------------------------------------------------- CTA rescoring
  if (tail.timing && lane == 0) atomicMax(tail.timing + 1, gtimer8());
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    if (lane < KP) {
      sh_u[b][warp * KP + lane] = lu[b];
      sh_p[b][warp * KP + lane] = lp[b];
    }
    if (lane == 0) {
      sh_lo[b][warp] = lo[b];
      sh_ovf[b][warp] = ovf[b];
    }
  }
  __syncthreads();
  if (threadIdx.x < nb) {
    const int b = threadIdx.x;
    double lc = -INFINITY;
#pragma unroll
    for (int w = 0; w < G8_WARPS; ++w) lc = fmax(lc, sh_lo[b][w]);
    const unsigned mine = key_of(__double2float_rd(lc));
    const unsigned old = atomicMax(tail.gmax + b0 + b, mine);
    sh_g[b] = val_of(old > mine ? old : mine);
  }
  __syncthreads();
  for (int b = 0; b < nb; ++b) {
    double lc = -INFINITY;
    float umax = -INFINITY, ov = -INFINITY;
#pragma unroll
    for (int w = 0; w < G8_WARPS; ++w) {
      lc = fmax(lc, sh_lo[b][w]);
      ov = fmaxf(ov, sh_ovf[b][w]);
      umax = fmaxf(umax, sh_u[b][w * KP]);
    }
    Best2 best;
    best.init();
    const bool scan_part = umax > -INFINITY && (double)umax >= (double)sh_g[b] - 1e-9;
    const bool pend_part = blockIdx.x == 0 && n_pend > 0;
    if (scan_part || pend_part) {  // block-uniform
      load_query(q64 + (size_t)b * Dp, tail.D, Dp, sq + (size_t)b * Dp);
      if (scan_part) {
        const double thr = fmax(lc, (double)sh_g[b]) - 1e-9;
        for (int e = warp; e < G8_WARPS * KP; e += G8_WARPS) {
          const long long p = sh_p[b][e];
          if (p < 0 || (double)sh_u[b][e] < thr) continue;  // warp-uniform
          const long long slot = ring_slot(st, local_row(st, p, sm));
          best.add(warp_dot64(rb.r64 + (size_t)slot * Dp, sq + (size_t)b * Dp, Dp, lane), p);
        }
      }
      if (pend_part) {  // rows appended since the last lookup: write every copy, score exactly
        for (long long i = warp; i < n_pend; i += G8_WARPS) {
          const double* srow = app.stage + (size_t)(app.n - n_pend + i) * Dp;
          const long long row = pend0 + i;
          if (b == 0) write_row_all(srow, ring_slot(st, row), rb, Dp, lane);
          best.add(warp_dot64(srow, sq + (size_t)b * Dp, Dp, lane), global_pos(st, row, sm));
        }
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

  if (tail.timing && threadIdx.x == 0) atomicMax(tail.timing + 2, gtimer8());
  if (!tail.counter) return;
  // ---------------------------------------------------------------- fused tail
  if (threadIdx.x == 0) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(tail.counter) : "memory");
    sh_last = old == gridDim.x - 1;
  }
  __syncthreads();
  if (!sh_last) return;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    if (b >= nb) break;
    const int gb = b0 + b;
    const bool exotic = tail.prep[b].exotic != 0;
    Best2 best;
    best.init();
    float ov = -INFINITY;
    for (int c = threadIdx.x; c < (int)gridDim.x; c += blockDim.x) {
      const CtaRec* src = cta + (size_t)gb * gridDim.x + c;
      CtaRec r;
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
      const bool fail = best.p < 0 || !(ov == -INFINITY || (double)ov + 1e-9 < best.s);
      mc_record r;
      r.sim = best.s;
      r.second = best.s2;
      r.pos = best.p;
      r.flags = (best.ties >= 2 ? MC_FLAG_TIE : 0u) | (fail ? FLAG_NEED_FALLBACK : 0u) |
                (exotic ? FLAG_NEED_EXHAUSTIVE : 0u);
      r.reserved = 0;
      tail.rec[gb] = r;
      if (tail.out) tail.out[gb] = decide(record_best(r), r.flags & FLAG_NEED_ANY, st.jhead, tail.thr);
      tail.gmax[gb] = 0u;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *tail.counter = 0u;
    if (tail.timing) tail.timing[3] = gtimer8();
  }
}

template <int N16>
static cudaError_t launch8(const RingBufs& rb, const RingState& st, const double* q64, int nb, CtaRec* cta, int b0,
                           int grid, ShardMap sm, const Gemv8Tail& tail, const Gemv8Append& app, cudaStream_t s) {
  const size_t smem = (size_t)(nb == 1 ? 1 : 4) * N16 * 16 * sizeof(double);
  if (nb == 1) {
    k_gemv8_scan<N16, 1><<<grid, G8_THREADS, smem, s>>>(rb, st, q64, nb, cta, b0, sm, tail, app);
  } else {
    auto kern = k_gemv8_scan<N16, 4>;
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    kern<<<grid, G8_THREADS, smem, s>>>(rb, st, q64, nb, cta, b0, sm, tail, app);
  }
  return cudaGetLastError();
}

// Dimensions whose row groups need at most 8 loads per lane (Dp/64 in 1..8, 10,
// 12, 14, 16); others use the fp16 GEMV.
bool gemv8_supported(int Dp) {
  if (Dp % 64 != 0 || Dp < 64 || Dp > 1024) return false;
  const int k = Dp / 64;
  return k <= 8 || k % 2 == 0;
}

cudaError_t launch_gemv8_scan(const RingBufs& rb, const RingState& st, int D, int Dp, const double* q64, int nb,
                              CtaRec* cta, int b0, int grid, ShardMap sm, unsigned* counter, unsigned* gmax,
                              const Thresholds& thr, mc_record* rec, OutRec* out, const GemvAppendArgs& a,
                              const QPrep* prep, const int8_t* q8, cudaStream_t s) {
  if (nb < 1 || nb > 4 || !gemv8_supported(Dp)) return cudaErrorInvalidValue;
  Gemv8Tail tail{counter, gmax, D, thr, rec, out, gemv_timing_buffer(), prep, q8};
  Gemv8Append app{a.stage, a.n, a.d_state};
#define MC_G8(K) \
  case K: return launch8<K * 4>(rb, st, q64, nb, cta, b0, grid, sm, tail, app, s)
  switch (Dp / 64) {
    MC_G8(1); MC_G8(2); MC_G8(3); MC_G8(4); MC_G8(5); MC_G8(6); MC_G8(7); MC_G8(8);
    MC_G8(10); MC_G8(12); MC_G8(14); MC_G8(16);
    default: return cudaErrorInvalidValue;
  }
#undef MC_G8
}

}  // namespace mc
