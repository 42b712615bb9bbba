// K2s — batch-1..4 scan over the int8 ring copy, streamed through TMA.
//
// The default small-batch path (C2: 100k x 768, B = 1).  It replaces the
// `_buf[_lo:_hi] @ q` dgemv of cache.py:254 for the filtering pass and keeps
// the certified float64 decision of K2q (scan_gemv8.cu), with the same error
// model and the same CtaRec / last-CTA merge contract:
//
//   per row e:  approx = s_e s_q Σ ê_i q̂_i   (exact int32 dot, exact scaling)
//               delta_e = ½ s_q ||e||_1 + ½ s_e s_q ||q̂||_1  (rigorous bound)
//               l = approx - delta_e <= e·q <= u = approx + delta_e
//   a row with u < L - 1e-9, where L <= the exact score of some other row,
//   can neither be nor tie the best; every other row is rescored in float64.
//
// Layout of one CTA (one per SM, persistent over its row range):
//   warp 0      producer: one 1-D bulk copy (cp.async.bulk, TMA engine) of a
//               stage's 32*R contiguous ring rows plus one of their
//               (s_e, ||e||_1) pairs; nst stages in flight.  One large copy
//               per stage: the TMA engine's per-operation cost caps small
//               (4-8 KB) boxes well below HBM rate (scripts/tma_microbench.cu).
//   warps 1..8  consumers: warp w owns stage buffer w; lane = row, so the
//               int32 dot needs no cross-lane reduction.  Lane l walks its
//               row's 16-byte chunks starting at chunk l (rotated order): with
//               the row stride a multiple of 128 B, the 8 lanes of a shared-
//               memory phase then hit 8 distinct bank groups.  A row that
//               survives the bound is pushed to the warp's candidate queue.
//   warp 9      rescorer: pending appends (CTA 0), a pool member, then the CTA
//               record, the ticket and — in the last CTA — the merge and
//               the decision (cache.py:255-260, select_k :112-117).
//   warp 10     bound poller: while the CTA streams, folds the other CTAs'
//               bound into the CTA's and prefetches the leading candidate's
//               float64 row into L2.
// Rescoring is lazy: it starts when the CTA's scan is over, and then the
// rescorer and the eight consumer warps form a pool that claims candidates
// best-first (see `pool`).
// The lower bound L is shared three ways: per warp (registers), per CTA
// (shared-memory atomicMax on an order-preserving float key) and across
// CTAs (fire-and-forget atomicMax on 8 replicas of the global gmax word; the
// poller folds the global value back into the CTA's).
//
// Pending appends (rows added since the last lookup) are not in the int8
// copy yet: CTA 0's eager warp writes every ring copy and scores them exactly
// from the envelope at kernel start.
//
// Algorithmic bytes per launch: count * (P8 + 8) + nb * (9 * Dp + 40), P8 = Dp rounded up to 128.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "merge.cuh"
#include "sm100.cuh"

namespace mc {

#ifndef S8_CONSUMERS
#define S8_CONSUMERS 4
#endif
// Consumer warps (and stages in flight).  4 (default): a CTA of at most half the shared memory
// and registers of an SM, so two co-reside and a launch's scan starts on an SM while the
// previous launch's CTA there still rescores and merges (back-to-back C2 steps 16.2 -> 12.1 us,
// profiles/r02_consumers_ab.txt).  8: one CTA per SM, no overlap between launches.
constexpr int S8_CW = S8_CONSUMERS;
#ifdef S8_CTAS
constexpr int S8_CTAS_PER_SM = S8_CTAS;
#else
constexpr int S8_CTAS_PER_SM = S8_CONSUMERS <= 4 ? 2 : 1;
#endif
#ifndef S8_GRID_PER_SM
#define S8_GRID_PER_SM 1
#endif
// CTAs per SM in one launch's grid (S8_GRID_PER_SM = 2 with 4 consumers: two half-size CTAs per
// SM, so an SM frees half its room as soon as one of them retires).
int s8_grid(int sm_count) { return S8_GRID_PER_SM * sm_count; }
// A launch that cannot overlap a neighbouring lookup (a shard's local lookup: the exact-rescan
// and merge kernels sit between consecutive scans) fills every co-resident CTA slot instead:
// one 148-CTA launch alone streams a 1M-row window at ~5.2 TB/s, two CTAs per SM keep more
// bytes in flight.  The record buffers are sized for this grid.
int s8_grid_wide(int sm_count) { return S8_CTAS_PER_SM * sm_count; }
constexpr int S8_THREADS = (S8_CW + 4) * 32;   // producer + consumers + rescorer + bound poller + eager rescorer
constexpr int S8_EAGER = S8_CW + 1;            // S.best slot of the eager rescorer
constexpr int S8_QCAP = 128;                   // candidate queue entries per consumer warp
constexpr int S8_GSTRIDE = 128;                // gmax u64 words per query: S8_GREP replicas, 128 B apart
constexpr int S8_GREP = 8;                     // replicas of the global bound (spreads the hot line)
// Only the poller warp touches the global bound: a fence, an acquire/release
// or a bar.sync waits for the warp's outstanding global operations, and a
// red to a hot line can take microseconds — so the warps that synchronise
// (consumers, pool, rescorer) never have one in flight.  For the same reason
// measurement stamps go to shared memory and are written out at the end.
constexpr int S8_PUB0 = 32 - S8_GREP;          // poller lanes S8_PUB0.. own one replica each
// per-CTA measurement slots (MC_GEMV_TIMING=1), timing[8 + 8 * cta + k]
enum { S8T_SCAN = 0, S8T_POOL, S8T_R0, S8T_R1, S8T_POOLX, S8T_REC, S8T_PUSH, S8T_RESC };

__host__ __device__ constexpr int s8_rows_per_lane(int kb) { return kb >= 4 ? 1 : (kb == 1 ? 4 : 2); }

__device__ __forceinline__ unsigned s8_key(float f) {
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float s8_val(unsigned k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

__device__ __forceinline__ int dp16x(const uint4& a, const uint4& b, int acc) {
  acc = __dp4a((int)a.x, (int)b.x, acc);
  acc = __dp4a((int)a.y, (int)b.y, acc);
  acc = __dp4a((int)a.z, (int)b.z, acc);
  return __dp4a((int)a.w, (int)b.w, acc);
}

__device__ __forceinline__ int ld_acq_cta(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel_cta(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_vol_u32(const unsigned* p) { return *(const volatile unsigned*)p; }
__device__ __forceinline__ unsigned long long ld_relaxed_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long s8_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct S8Args {
  unsigned* counter;           // last-CTA ticket (zero between launches)
  // [(b0 + b) * S8_GSTRIDE + 16 r] global lower-bound replicas: (epoch << 32) | key.  A value
  // from an earlier launch's epoch is smaller than any of this launch's and is ignored when
  // read, so the words are never reset (a late atomic of a finished launch cannot leak into
  // the next one).
  unsigned long long* gmax;
  Thresholds thr;
  mc_record* rec;
  OutRec* out;
  unsigned long long* timing;  // optional phase stamps (MC_GEMV_TIMING=1)
  const QPrep* prep;           // [nb] per-query quantisation (host-computed, in the envelope)
  const int8_t* q8;            // [nb][Dp] q̂
  const double* stage;         // pending appends (float64, stride Dp)
  long long n_app;
  RingState* d_state;
  unsigned* done_seq;          // optional (host-mapped): set to `seq` after `out` is written (zero-copy result)
  unsigned seq;
  uint4* outp;                 // optional (host-mapped): packed decisions, one 16-byte store each (see below)
  unsigned epoch;              // this launch's tag on the gmax words (never 0)
  double* gq64;                // [Dp] L2 relay of the pending row (single-query launches, CTA 0)
  // Overlap with the previous launch on this ring (the next lookup's scan starts while the
  // previous grid's merge still runs; see the prologue): sync[0] = epoch whose pending rows
  // are written and visible, sync[1] = epoch whose CTA records the merger has read.  Records
  // alternate between two buffers by epoch parity, rec_par uint4 apart.  nullptr: no overlap.
  unsigned* sync;
  unsigned rec_par;
  unsigned overlap;  // 0: the previous kernel on the stream may be another path's (wait for it in full)
};
__device__ __forceinline__ unsigned ld_acquire_gpu_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// The single-query launch's inputs (no host->device copy before the kernel):
// the query and its int8 quantisation ride in the kernel parameter block
// (~9 KB; every CTA needs them); the pending row stays in mapped host memory
// and only CTA 0, which writes it into the ring, reads it (over PCIe, once,
// with every load in flight) into an L2 relay buffer.
#ifndef S8IN_DMAX
#define S8IN_DMAX 1024  // measurement knob: a smaller parameter block (valid only for Dp <= S8IN_DMAX)
#endif
struct S8In {
  QPrep prep;
  alignas(16) int8_t q8[S8IN_DMAX];
  alignas(16) double q64[S8IN_DMAX];  // the float64 query, zero-padded to Dp
  const double* hstage;          // host-mapped pending row (zero-padded to Dp), or nullptr
};
struct S8NoIn {
  int unused;
};

// A decision packed into two 16-byte stores (two PCIe writes, each read by the
// host with one 16-byte load):
//   [0] sim | live (int32) | k (8) flags (8: MC_FLAG_* bits 0-6, bit 7 = needs the
//       exhaustive path) seq (16)
//   [1] sigma | steps (int32) | route (8) 0 (8) seq (16)
// The sequence tag makes each record self-validating, so no system-scope fence
// has to separate the decisions from a completion word.
__device__ __forceinline__ uint4 pack_out(const OutRec& o, unsigned seq16) {
  const unsigned long long sb = (unsigned long long)__double_as_longlong(o.sim);
  const unsigned f8 = (o.flags & 0x7fu) | ((o.flags & FLAG_NEED_ANY) ? 0x80u : 0u);
  return make_uint4((unsigned)sb, (unsigned)(sb >> 32), (unsigned)o.live,
                    ((unsigned)o.k & 0xffu) | (f8 << 8) | (seq16 << 16));
}
__device__ __forceinline__ uint4 pack_out2(const OutRec& o, unsigned seq16) {
  const unsigned long long gb = (unsigned long long)__double_as_longlong(o.sigma);
  return make_uint4((unsigned)gb, (unsigned)(gb >> 32), (unsigned)o.steps, ((unsigned)o.route & 0xffu) | (seq16 << 16));
}

// Rows [r0, r1) (live-local) of one CTA, cut into stages of up to `rows`
// rows that never cross the physical end of the ring.
struct S8Work {
  long long r0, r1, w;  // w = first row that wraps to slot 0
  int ns1, ns, rows;
  __device__ void init(const RingState& st, long long n_scan, int cta, int grid, int rows_) {
    rows = rows_;
    r0 = n_scan * cta / grid;
    r1 = n_scan * (cta + 1) / grid;
    w = st.cap - st.head;
    const long long e1 = min(r1, max(r0, w));
    const long long b2 = max(r0, w);
    ns1 = (int)((e1 - r0 + rows - 1) / rows);
    ns = ns1 + (int)(r1 > b2 ? (r1 - b2 + rows - 1) / rows : 0);
  }
  // stage i -> first live row, row count, first physical slot
  __device__ void stage(int i, const RingState& st, long long& row0, int& n, long long& slot0) const {
    long long end;
    if (i < ns1) {
      row0 = r0 + (long long)i * rows;
      end = min(row0 + rows, min(r1, max(r0, w)));
    } else {
      row0 = max(r0, w) + (long long)(i - ns1) * rows;
      end = min(row0 + rows, r1);
    }
    n = (int)(end - row0);
    slot0 = row0 < w ? st.head + row0 : st.head + row0 - st.cap;
  }
};

// Shared state of one CTA (besides the dynamic stage buffers); sized for
// four queries, declared once at namespace scope so the out-of-line helpers
// below address it directly.
constexpr int NB = 4;
struct S8Smem {
  uint64_t full[S8_CW], empty[S8_CW];   // stage mbarriers
  float qu[S8_CW][S8_QCAP];             // candidate queues: upper bound (float, rounded up)
  long long qp[S8_CW][S8_QCAP];         //   global position << 2 | query
  int qc[S8_CW][S8_QCAP];               //   pool claim flags
  int qtail[S8_CW];
  float ovf[S8_CW][NB];                 // largest bound a full queue dropped
  unsigned bound[NB];                   // CTA lower bound (order-preserving float key)
  int done, pool_done;
  int q_ready;                          // sq64 (the float64 queries) is filled
  Best2 best[S8_CW + 2][NB];            // float64 best per pool warp, then the eager rescorer's
  unsigned long long t[8];              // measurement stamps (MC_GEMV_TIMING=1)
  unsigned long long c[4];              // pool cycle counts (MC_GEMV_TIMING=1)
};
__shared__ S8Smem g_s8;
#define S g_s8

// Per-launch constants of the cold paths (pool, pending rows, finish).
struct S8Ctx {
  RingBufs rb;
  RingState st;
  ShardMap sm;
  const double* sq64;  // shared memory: [NB][Dp] float64 queries
  int Dp, nb, ncw;
  bool timing;
};

__device__ __forceinline__ void s8_raise(unsigned* bound, int lane, double sc) {
  // an exact score is a lower bound for everyone (the poller publishes it)
  if (lane == 0 && !isnan(sc)) atomicMax(bound, s8_key(__double2float_rd(sc)));
}

// The cold paths below run once per launch.  They are out of line, so their
// code exists once (shared by the nine pool warps) and the instruction cache
// holds one copy.

// One out-of-line copy of the exact dot for every rescoring warp of the CTA
// (the pool, CTA 0's pending rows, the poller's warm-up).
__device__ __noinline__ double s8_dot(const double* row, const double* q, int n, int lane) {
  return warp_dot64(row, q, n, lane);
}

// One best-first pass over the (final) candidate queues, flattened by their
// prefix sums so the entries spread over the 32 lanes with independent
// loads.  Returns the queue index (w * S8_QCAP + i) of the live, unclaimed
// candidate with the largest upper bound, or -1.  `retire` marks candidates
// whose bound fell below the CTA's lower bound (false: a side-effect-free
// warm-up pass).  Inlined: an out-of-line call costs more here (measured, scripts/ab_c2.sh).
__device__ __forceinline__ int s8_pass(int ncw, bool retire) {
  const int lane = threadIdx.x & 31;
  int tails = 0;  // lane w < ncw: tail of queue w
  if (lane < ncw) tails = ld_acq_cta(&S.qtail[lane]);  // pairs with the pushing warp's st.release
  int start[S8_CW];
  int total = 0;
#pragma unroll
  for (int w = 0; w < S8_CW; ++w) {
    start[w] = total;
    total += w < ncw ? __shfl_sync(FULL, tails, w) : 0;
  }
  float bu = -INFINITY;
  int bi = -1;
  for (int f = lane; f < total; f += 32) {
    int w = 0, base = 0;
#pragma unroll
    for (int k = 1; k < S8_CW; ++k)
      if (k < ncw && f >= start[k]) {
        w = k;
        base = start[k];
      }
    const int i = f - base;
    const float u = *(volatile float*)&S.qu[w][i];
    const int claimed = *(volatile int*)&S.qc[w][i];
    const int b = (int)(S.qp[w][i] & 3);
    const float bnd = s8_val(ld_vol_u32(&S.bound[b]));
    if (u == -INFINITY || claimed) continue;
    if ((double)u < (double)bnd - 1e-9) {
      if (retire) S.qu[w][i] = -INFINITY;  // strictly below a row whose exact score is known to exceed it
      continue;
    }
    if (u > bu) {
      bu = u;
      bi = w * S8_QCAP + i;
    }
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    const float ou = __shfl_xor_sync(FULL, bu, off);
    const int oi = __shfl_xor_sync(FULL, bi, off);
    if (ou > bu || (ou == bu && oi > bi)) {
      bu = ou;
      bi = oi;
    }
  }
  return bi;
}

// CTA 0's eager warp: rows appended since the last lookup are not in the int8
// copy yet — write every ring copy and score them exactly (float64).
__device__ __forceinline__ void s8_pending(const S8Ctx x, const double* stage, long long n_app,
                                        long long n_pend, long long n_scan) {
  const int lane = threadIdx.x & 31;
  while (!*(volatile int*)&S.q_ready) {
  }
  for (long long i = 0; i < n_pend; ++i) {
    const double* srow = stage + (size_t)(n_app - n_pend + i) * x.Dp;
    const long long row = n_scan + i;
    write_row_all(srow, ring_slot(x.st, row), x.rb, x.Dp, lane);
    for (int b = 0; b < x.nb; ++b) {
      const double sc = s8_dot(srow, x.sq64 + (size_t)b * x.Dp, x.Dp, lane);
      if (lane == 0) S.best[S8_EAGER][b].add(sc, global_pos(x.st, row, x.sm));
      s8_raise(&S.bound[b], lane, sc);
    }
  }
  __syncwarp();
}

// Rescoring pool: the rescorer warp and the eight consumer warps, once every
// consumer is done (a hardware barrier: nothing spins beside the streaming
// warps).  Lazy: nothing is rescored while the CTA streams (those loads would
// queue behind the scan's, and the bound keeps rising).  Best-first: claim the
// live candidate with the largest upper bound and rescore it in float64; its
// exact score then prunes the rest.  Candidates whose bound fell below the
// CTA's lower bound are retired unscored.  Result: S.best[wid][*].
__device__ __forceinline__ void s8_pool(const S8Ctx x, int wid) {
  const int lane = threadIdx.x & 31;
  // barrier.sync (not bar.sync, the .aligned form): lanes may arrive unconverged after the
  // lane-0 bookkeeping above (compute-sanitizer synccheck)
  __syncwarp();
  asm volatile("barrier.sync 1, %0;" ::"n"((S8_CW + 1) * 32) : "memory");
  while (!*(volatile int*)&S.q_ready) {
  }
  if (x.timing && lane == 0) atomicMax(&S.t[S8T_POOL], s8_timer());
  const long long c_pool = clock64();
  bool first_pass = true;
  while (true) {
    const int bi = s8_pass(x.ncw, true);
    if (x.timing && first_pass && lane == 0) atomicMax(&S.c[0], (unsigned long long)(clock64() - c_pool));
    first_pass = false;
    if (bi < 0) break;  // nothing live and unclaimed is left (claimed ones finish with their claimer)
    const int w = bi / S8_QCAP, i = bi % S8_QCAP;
    int won = 0;
    if (lane == 0) won = atomicCAS(&S.qc[w][i], 0, 1) == 0;
    if (__shfl_sync(FULL, won, 0)) {
      const long long pb = S.qp[w][i];
      const int b = (int)(pb & 3);
      const long long p = pb >> 2;
      const long long slot = ring_slot(x.st, local_row(x.st, p, x.sm));
      const long long c_dot = clock64();
      if (x.timing && lane == 0) {
        atomicMin(&S.t[S8T_R0], s8_timer());
        atomicMin(&S.c[2], (unsigned long long)(c_dot - c_pool));
      }
      const double sc = s8_dot(x.rb.r64 + (size_t)slot * x.Dp, x.sq64 + (size_t)b * x.Dp, x.Dp, lane);
      if (lane == 0) {
        S.best[wid][b].add(sc, p);
        if (x.timing) {
          atomicMax(&S.t[S8T_R1], s8_timer());
          atomicMax(&S.c[3], (unsigned long long)(clock64() - c_dot));
          atomicAdd(&S.t[S8T_RESC], 1ull);
        }
      }
      s8_raise(&S.bound[b], lane, sc);
      __syncwarp();
      if (lane == 0) S.qu[w][i] = -INFINITY;
    }
    __syncwarp();
  }
  if (x.timing && lane == 0) atomicMax(&S.t[S8T_POOLX], s8_timer());
  __syncwarp();
  if (lane == 0) {
    __threadfence_block();
    atomicAdd(&S.pool_done, 1);
  }
}

// Per-CTA record of the streamed scan: two self-validating 16-byte words (each
// stored and loaded as one 16-byte access), tagged with the launch epoch:
//   [0] s (float64) | off (bits 0-29: global position - position of live row 0;
//       0x3fffffff = no candidate) + min(ties, 3) << 30 | epoch
//   [1] s2 (float64) | ovf (float bits) | epoch
// No ticket: one merger (CTA 0's rescorer) polls the records until every one
// carries this launch's epoch.  A word from an earlier launch never matches.
constexpr unsigned S8_NOOFF = 0x3fffffffu;
__device__ __forceinline__ uint4 ld_relaxed_v4(const uint4* p) {
  uint4 r;
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p)
               : "memory");
  return r;
}
__device__ __forceinline__ void st_v4(uint4* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// The rescorer after the pool: the CTA record and, in CTA 0, the merge of
// every CTA's record and the decision (cache.py:255-260, select_k :112-117),
// then the zero-copy result.
__device__ __forceinline__ void s8_finish(const S8Ctx x, const S8Args& a, const QPrep* prep, uint4* crec, int b0) {
  const int lane = threadIdx.x & 31;
  const int nb = x.nb;
  const unsigned tag = a.epoch;
  const long long pbase = global_pos(x.st, 0, x.sm);
  if (a.sync) crec += (size_t)(tag & 1u) * a.rec_par;  // this epoch's record buffer
  if (lane == 0)
    while (ld_acq_cta(&S.pool_done) != S8_CW + 2) {  // the pool warps (consumers + rescorer) and the eager rescorer
    }
  if (lane == 0 && a.sync)  // the launch two back used this buffer: its merger must be done reading it
    while ((int)(ld_acquire_gpu_u32(a.sync + 1) - (tag - 2u)) < 0) {
    }
  __syncwarp();
  for (int b = 0; b < nb; ++b) {
    Best2 m;
    m.init();
    float ov = -INFINITY;
    for (int w = 0; w <= S8_EAGER; ++w) m.merge(S.best[w][b]);
    for (int w = 0; w < x.ncw; ++w) ov = fmaxf(ov, S.ovf[w][b]);
    if (lane == 0) {
      const unsigned long long sb = (unsigned long long)__double_as_longlong(m.s);
      const unsigned long long s2b = (unsigned long long)__double_as_longlong(m.s2);
      const unsigned off = m.p < 0 ? S8_NOOFF : (unsigned)(m.p - pbase) | ((unsigned)min(m.ties, 3) << 30);
      uint4* dst = crec + ((size_t)(b0 + b) * gridDim.x + blockIdx.x) * 2;
      st_v4(dst, make_uint4((unsigned)sb, (unsigned)(sb >> 32), off, tag));
      st_v4(dst + 1, make_uint4((unsigned)s2b, (unsigned)(s2b >> 32), __float_as_uint(ov), tag));
    }
  }
  if (x.timing && lane == 0) S.t[S8T_REC] = s8_timer();
  __syncwarp();
  auto dump = [&]() {  // measurement stamps, written once this CTA is off the critical path
    if (x.timing && lane < 8) a.timing[8 + 8 * blockIdx.x + lane] = S.t[lane];
    if (x.timing && lane < 4) a.timing[8 + 8 * 512 + 4 * blockIdx.x + lane] = S.c[lane];
  };
  if (blockIdx.x != 0) {
    dump();
    return;
  }
  unsigned exotic = 0;
  if (lane < nb) exotic = prep[lane].exotic != 0 ? 1u : 0u;
  // Merge the per-CTA records with independent warp reductions (no chain of
  // Best2 merges): best = max s; among records at best: max position and the
  // summed tie counts; runner-up = max over the others' s and everyone's s2
  // (a second record at the best makes the runner-up equal to it, as in
  // Best2::merge).  Record similarities are finite here (exotic queries are
  // flagged for the exhaustive path).
  constexpr int PER = 10;  // records per lane: grid <= 320 (the host clamps it)
  for (int b = 0; b < nb; ++b) {
    const int gb = b0 + b;
    const uint4* src = crec + (size_t)gb * gridDim.x * 2;
    uint4 ra[PER], rb2[PER];
    unsigned ok = 0;  // bit k: record 32 k + lane seen
#pragma unroll
    for (int k = 0; k < PER; ++k)
      if (32 * k + lane >= (int)gridDim.x) ok |= 1u << k;
    while (true) {
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        if (!(ok >> k & 1u)) {
          const int c = 32 * k + lane;
          ra[k] = ld_relaxed_v4(src + 2 * c);
          rb2[k] = ld_relaxed_v4(src + 2 * c + 1);
          if (ra[k].w == tag && rb2[k].w == tag) ok |= 1u << k;
        }
      }
      if (__all_sync(FULL, ok == (1u << PER) - 1u)) break;
    }
    if (b == 0 && lane == 0 && x.timing) a.timing[4] = a.timing[5] = s8_timer();
    double rs[PER], rs2[PER];
    long long rp[PER];
    int rt[PER];
    float ro[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const bool in = 32 * k + lane < (int)gridDim.x;
      const unsigned off = in ? ra[k].z : S8_NOOFF;
      rs[k] = __longlong_as_double((long long)(((unsigned long long)ra[k].y << 32) | ra[k].x));
      rs2[k] = __longlong_as_double((long long)(((unsigned long long)rb2[k].y << 32) | rb2[k].x));
      ro[k] = in ? __uint_as_float(rb2[k].z) : -INFINITY;
      rp[k] = off == S8_NOOFF ? -1 : pbase + (long long)(off & S8_NOOFF);
      rt[k] = (int)(off >> 30);
      if (rp[k] < 0) rs[k] = rs2[k] = -INFINITY;
    }
    double bs = -INFINITY;
    float ov = -INFINITY;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      if (rp[k] >= 0) bs = fmax(bs, rs[k]);
      ov = fmaxf(ov, ro[k]);
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      bs = fmax(bs, __shfl_xor_sync(FULL, bs, off));
      ov = fmaxf(ov, __shfl_xor_sync(FULL, ov, off));
    }
    long long bp = -1;
    int nt = 0, neq = 0;
    double s2 = -INFINITY;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      if (rp[k] < 0) continue;
      if (rs[k] == bs) {
        bp = max(bp, rp[k]);
        nt += rt[k];
        ++neq;
      } else {
        s2 = fmax(s2, rs[k]);
      }
      s2 = fmax(s2, rs2[k]);
    }
    nt = __reduce_add_sync(FULL, (unsigned)nt);
    neq = __reduce_add_sync(FULL, (unsigned)neq);
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      bp = max(bp, __shfl_xor_sync(FULL, bp, off));
      s2 = fmax(s2, __shfl_xor_sync(FULL, s2, off));
    }
    if (neq >= 2) s2 = bs;
    const bool exo = __shfl_sync(FULL, exotic, b) != 0;
    if (b == 0 && lane == 0 && x.timing) a.timing[6] = s8_timer();
    if (lane == 0) {
      const bool fail = bp < 0 || !(ov == -INFINITY || (double)ov + 1e-9 < bs);
      mc_record r;
      r.sim = bs;
      r.second = s2;
      r.pos = bp;
      r.flags = (nt >= 2 ? MC_FLAG_TIE : 0u) | (fail ? FLAG_NEED_FALLBACK : 0u) | (exo ? FLAG_NEED_EXHAUSTIVE : 0u);
      r.reserved = 0;
      a.rec[gb] = r;
      const OutRec o = decide(record_best(r), r.flags & FLAG_NEED_ANY, x.st.jhead, a.thr);
      if (a.out) a.out[gb] = o;
      if (a.outp) {
        st_v4(a.outp + 2 * gb, pack_out(o, a.seq));
        st_v4(a.outp + 2 * gb + 1, pack_out2(o, a.seq));
      }
      if (b == 0 && x.timing) a.timing[7] = s8_timer();
    }
  }
  __syncwarp();
  if (lane == 0 && a.sync) st_release_gpu_u32(a.sync + 1, tag);  // every record of this launch is read
  if (lane == 0) {
    if (a.done_seq) {  // zero-copy result: the decisions, then the sequence word, over the system fabric
      __threadfence_system();
      *(volatile unsigned*)a.done_seq = a.seq;
    }
    if (x.timing) a.timing[3] = s8_timer();
  }
  dump();
}

template <int KB, int NBQ, bool IN>
__global__ void __launch_bounds__(S8_THREADS, S8_CTAS_PER_SM)
    k_stream8_scan(RingBufs rb, const RingState st, const double* __restrict__ q64_dev, int nb,
                   CtaRec* __restrict__ cta, int b0, ShardMap sm, S8Args a, int nst, int Dp,
                   const __grid_constant__ std::conditional_t<IN, S8In, S8NoIn> in) {
  // IN: this lookup's query, its quantisation and its pending row arrive in the
  // launch's parameter block (no host->device copy before the kernel)
  const double* q64 = q64_dev;
  const int8_t* q8p = a.q8;
  const QPrep* prepp = a.prep;
  const double* stagep = a.stage;
  if constexpr (IN) {
    q64 = in.q64;
    q8p = in.q8;
    prepp = &in.prep;
    stagep = in.hstage;  // CTA 0's poller reads it once; its eager warp then uses the relay (below)
  }
  constexpr int P8 = KB * 128;                // int8 row stride (Dp rounded up to 128)
  constexpr int R = s8_rows_per_lane(KB);
  constexpr int SROWS = 32 * R;               // rows per stage
  constexpr int NCH = P8 / 16;                // 16-byte chunks per int8 row (a multiple of 8)
  constexpr int SDATA = SROWS * P8;           // int8 bytes of a stage
  constexpr int RQS = SROWS + 2;              // (s, L1) entries per stage buffer (16-byte aligned copy)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stages = base;                                            // [nst][SDATA]
  float2* rqs = reinterpret_cast<float2*>(base + (size_t)nst * SDATA);  // [nst][RQS]
  int8_t* sq8 = reinterpret_cast<int8_t*>(rqs + (size_t)nst * RQS);     // [NBQ][P8]
  double* sq64 = reinterpret_cast<double*>(sq8 + NBQ * P8);              // [NBQ][Dp] float64 queries

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const long long n = st.count;
  const long long n_pend = min(a.n_app, n);
  const long long n_scan = n - n_pend;  // rows [n_scan, n) are scored exactly by CTA 0
  S8Work wk;
  wk.init(st, n_scan, blockIdx.x, gridDim.x, SROWS);
  const bool timing = a.timing != nullptr;

  // Programmatic dependent launch: the next lookup's grid may be scheduled as
  // soon as SMs free up; it runs its prologue (this block up to
  // griddepcontrol.wait) while this grid's last CTA still merges.
  if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; ++i) {
      mbar_init(&S.full[i], 1);
      mbar_init(&S.empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int b = 0; b < NBQ; ++b) S.bound[b] = s8_key(-INFINITY);
    S.done = 0;
    S.pool_done = 0;
    S.q_ready = IN ? 0 : 1;
    for (int k = 0; k < 8; ++k) S.t[k] = 0ull;
    S.t[S8T_R0] = ~0ull;
    for (int k = 0; k < 4; ++k) S.c[k] = k == 2 ? ~0ull : 0ull;
  }
  if (threadIdx.x < S8_CW) S.qtail[threadIdx.x] = 0;
  for (int i = threadIdx.x; i < (S8_CW + 2) * NB; i += blockDim.x) (&S.best[0][0])[i].init();
  for (int i = threadIdx.x; i < S8_CW * S8_QCAP; i += blockDim.x) (&S.qc[0][0])[i] = 0;
  if constexpr (!IN) {  // a parameter-block query is copied by the poller warp, off the prologue
    for (int i = threadIdx.x; i < NBQ * Dp; i += blockDim.x) sq64[i] = i < nb * Dp ? q64[i] : 0.0;
  }
  for (int i = threadIdx.x; i < NBQ * P8 / 16; i += blockDim.x) {  // q̂ (stride Dp) -> [NBQ][P8], zero-padded
    const int b = i / (P8 / 16), c = i % (P8 / 16);
    reinterpret_cast<uint4*>(sq8)[i] = (b < nb && c < Dp / 16)
                                           ? reinterpret_cast<const uint4*>(q8p + (size_t)b * Dp)[c]
                                           : make_uint4(0u, 0u, 0u, 0u);
  }
  // Everything above reads only this launch's inputs (host-staged queries) and
  // initialises shared memory; from here on the ring is touched.
  // With `sync`, this launch does not wait for the previous one on the ring to finish: it needs
  // only the rows that launch appended (its CTA 0 publishes sync[0] once they are written).
  // The previous launch's window survives the rows this one appends (<= PIPE_SLACK of them land
  // in spare slots), the bound words are epoch-tagged and the records alternate by epoch parity
  // (a record writer waits for sync[1]).  Otherwise: the full programmatic dependency.
  if (a.sync && a.overlap && a.n_app <= PIPE_SLACK) {
    if (threadIdx.x == 0)
      while ((int)(ld_acquire_gpu_u32(a.sync) - (a.epoch - 1u)) < 0) {
      }
  } else {
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0 && a.d_state) *a.d_state = st;
    if (timing) atomicMin(a.timing + 0, s8_timer());
  }
  __syncthreads();

  const int ncw = min(nst, S8_CW);
  const S8Ctx x{rb, st, sm, sq64, Dp, nb, ncw, timing};
  unsigned long long* const gq = a.gmax + (size_t)b0 * S8_GSTRIDE;  // this launch's queries

  if (warp == S8_CW + 3) {
    // ------------------------------------------------------------ eager rescorer
    // While the CTA streams, rescore (best-first, one at a time) the live
    // candidate with the largest upper bound: its exact score raises the bound
    // early and the pool after the scan mostly finds the CTA's best done.  It
    // checks `done` before each claim and never waits on global memory, so it
    // hands over within one exact dot once the scan is over.
    // CTA 0's eager warp first writes and scores the rows appended since the last lookup: off the
    // rescorer, whose pool barrier (and CTA 0's record, which the merge waits for) it would delay
    if (blockIdx.x == 0) {
      if (n_pend > 0) s8_pending(x, IN ? a.gq64 : stagep, a.n_app, n_pend, n_scan);
      __syncwarp();
      if (lane == 0 && a.sync) {  // the rows appended before this launch are in the ring
        __threadfence();
        st_release_gpu_u32(a.sync, a.epoch);
      }
    }
    while (!*(volatile int*)&S.q_ready) {
    }
    while (*(volatile int*)&S.done != S8_CW) {
      const int bi = s8_pass(ncw, false);
      if (bi < 0 || *(volatile int*)&S.done == S8_CW) {
        __nanosleep(200);
        continue;
      }
      const int w = bi / S8_QCAP, i = bi % S8_QCAP;
      int won = 0;
      if (lane == 0) won = atomicCAS(&S.qc[w][i], 0, 1) == 0;
      if (__shfl_sync(FULL, won, 0)) {
        const long long pb = S.qp[w][i];
        const int b = (int)(pb & 3);
        const long long p = pb >> 2;
        const long long slot = ring_slot(st, local_row(st, p, sm));
        const double sc = s8_dot(rb.r64 + (size_t)slot * Dp, sq64 + (size_t)b * Dp, Dp, lane);
        if (lane == 0) {
          S.best[S8_EAGER][b].add(sc, p);
          if (!isnan(sc)) atomicMax(&S.bound[b], s8_key(__double2float_rd(sc)));
          if (timing) atomicAdd(&S.t[S8T_RESC], 1ull);
        }
        __syncwarp();
        if (lane == 0) S.qu[w][i] = -INFINITY;
      }
      __syncwarp();
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      atomicAdd(&S.pool_done, 1);
    }
    return;
  }

  if (warp == S8_CW + 2) {
    // ------------------------------------------------------------ bound poller
    // Until the pool is done: carry the CTA's bound to the other CTAs (lane
    // S8_PUB0 + r owns replica r), fold theirs in (replica cta % S8_GREP), and
    // while the CTA streams pull the leading candidate's float64 row into L2
    // so its rescoring after the scan hits L2.  This warp never synchronises
    // (its global atomics stay off the other warps' fences and barriers).
    if constexpr (IN) {
#pragma unroll 4
      for (int i = lane; 2 * i < Dp; i += 32)  // the query, from the parameter block
        reinterpret_cast<double2*>(sq64)[i] = reinterpret_cast<const double2*>(q64)[i];
      if (blockIdx.x == 0 && stagep) {  // the pending row: one PCIe round trip (16 x 16 B per lane, Dp <= 1024)
        const double2* hs = reinterpret_cast<const double2*>(stagep);
        double2 vs[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int i = lane + 32 * k;
          vs[k] = 2 * i < Dp ? hs[i] : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (2 * (lane + 32 * k) < Dp) reinterpret_cast<double2*>(a.gq64)[lane + 32 * k] = vs[k];
      }
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        *(volatile int*)&S.q_ready = 1;
      }
    }
    int pf = -1;
    unsigned pub[NBQ];
#pragma unroll
    for (int b = 0; b < NBQ; ++b) pub[b] = 0u;
    while (*(volatile int*)&S.pool_done < S8_CW + 2) {
      unsigned gk = 0;
      if (lane >= S8_PUB0 && lane - S8_PUB0 < nb) {
        const unsigned long long g = ld_relaxed_gpu(gq + (lane - S8_PUB0) * S8_GSTRIDE + 16 * (blockIdx.x % S8_GREP));
        gk = (unsigned)(g >> 32) == a.epoch ? (unsigned)g : 0u;
      }
#pragma unroll
      for (int b = 0; b < NBQ; ++b) {
        const unsigned mine = ld_vol_u32(&S.bound[b]);
        if (b < nb && mine > pub[b]) {
          if (lane >= S8_PUB0)
            atomicMax(gq + b * S8_GSTRIDE + 16 * (lane - S8_PUB0), ((unsigned long long)a.epoch << 32) | mine);
          pub[b] = mine;
        }
      }
      if (*(volatile int*)&S.done != S8_CW) {
        const int bi = s8_pass(ncw, false);
        if (bi >= 0 && bi != pf) {
          pf = bi;
          const long long p = S.qp[bi / S8_QCAP][bi % S8_QCAP] >> 2;
          const char* row = reinterpret_cast<const char*>(rb.r64 + (size_t)ring_slot(st, local_row(st, p, sm)) * Dp);
          for (int off = lane * 128; off < Dp * 8; off += 32 * 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(row + off));
        }
      }
      if (gk && gk > ld_vol_u32(&S.bound[lane - S8_PUB0])) atomicMax(&S.bound[lane - S8_PUB0], gk);
      __syncwarp();
    }
    return;
  }

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      for (int i = 0; i < wk.ns; ++i) {
        const int buf = i % nst;
        mbar_wait(&S.empty[buf], ((i / nst) & 1) ^ 1);
        long long row0, slot0;
        int nr;
        wk.stage(i, st, row0, nr, slot0);
        const long long q0 = slot0 & ~1ll;    // (s, L1) pairs from a 16-byte aligned slot
        const uint32_t qbytes = (uint32_t)(((slot0 - q0) + nr + 1) / 2 * 16);
        const uint32_t dbytes = (uint32_t)nr * P8;
        mbar_expect_tx(&S.full[buf], dbytes + qbytes);
        bulk_load_hint(stages + (size_t)buf * SDATA, rb.r8 + (size_t)slot0 * P8, dbytes, &S.full[buf], pol);
        bulk_load_hint(rqs + (size_t)buf * RQS, rb.rq + q0, qbytes, &S.full[buf], pol);
      }
    }
    return;
  }

  if (warp > S8_CW) {
    // ------------------------------------------------------------ rescorer
    s8_pool(x, S8_CW);
    s8_finish(x, a, prepp, reinterpret_cast<uint4*>(cta), b0);
    return;
  }

  // -------------------------------------------------------------- consumers
  const int cw = warp - 1;
  double sq[NBQ], q1[NBQ];
#pragma unroll
  for (int b = 0; b < NBQ; ++b) {
    const QPrep pq = b < nb ? prepp[b] : QPrep{0.0, 0.0, 0.0, 0.f, 0};
    sq[b] = pq.s;
    q1[b] = pq.q1;
  }
  float lo[NBQ], ovf[NBQ];
#pragma unroll
  for (int b = 0; b < NBQ; ++b) {
    lo[b] = -INFINITY;
    ovf[b] = -INFINITY;
  }
  int tail = 0;
  if (cw < ncw) {
    for (int i = cw; i < wk.ns; i += ncw) {
      const int buf = i % nst;
      long long row0, slot0;
      int nr;
      wk.stage(i, st, row0, nr, slot0);
      mbar_wait(&S.full[buf], (i / nst) & 1);
      const uint8_t* sb = stages + (size_t)buf * SDATA;
      const int lrot = lane % NCH;    // first chunk of this lane (NCH may be 8 < 32 lanes)
      int acc[R][NBQ], acc2[R][NBQ];  // two chains per dot (exact integers: order is free)
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int b = 0; b < NBQ; ++b) acc[r][b] = acc2[r][b] = 0;
      // partially unrolled: each warp runs this loop only a few times per
      // launch, so a compact body keeps it resident in the instruction cache
#pragma unroll 8
      for (int j = 0; j < NCH; ++j) {
        int c = j + lrot;  // rotated chunk order (conflict-free, see the header)
        c = c >= NCH ? c - NCH : c;
        uint4 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = *reinterpret_cast<const uint4*>(sb + (r * 32 + lane) * P8 + c * 16);
#pragma unroll
        for (int b = 0; b < NBQ; ++b) {
          const uint4 qv = *reinterpret_cast<const uint4*>(sq8 + b * P8 + c * 16);
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (j & 1)
              acc2[r][b] = dp16x(v[r], qv, acc2[r][b]);
            else
              acc[r][b] = dp16x(v[r], qv, acc[r][b]);
          }
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int b = 0; b < NBQ; ++b) acc[r][b] += acc2[r][b];
      float2 e[R];
#pragma unroll
      for (int r = 0; r < R; ++r) e[r] = rqs[(size_t)buf * RQS + (slot0 & 1) + r * 32 + lane];
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.empty[buf]);

      // bounds: the warp's own, then the CTA's (which carries the global one)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const bool valid = r * 32 + lane < nr;
#pragma unroll
        for (int b = 0; b < NBQ; ++b) {
          if (b >= nb) break;
          const double approx = (double)acc[r][b] * ((double)e[r].x * sq[b]);
          const double dl = (0.5 * sq[b] * (double)e[r].y + 0.5 * (double)e[r].x * q1[b]) * (1.0 + 1e-9) + 1e-12;
          float lf = valid ? __double2float_rd(approx - dl) : -INFINITY;
#pragma unroll
          for (int off = 16; off; off >>= 1) lf = fmaxf(lf, __shfl_xor_sync(FULL, lf, off));
          float bnd = s8_val(ld_vol_u32(&S.bound[b]));
          if (lf > lo[b]) {
            lo[b] = lf;
            if (lf > bnd) {  // publish to the CTA (the poller carries it to the other CTAs)
              if (lane == 0) atomicMax(&S.bound[b], s8_key(lf));
              bnd = lf;
            }
          }
          const double u = approx + dl;
          const bool keep = valid && u >= (double)bnd - 1e-9;
          const unsigned m = __ballot_sync(FULL, keep);
          if (m) {
            const int idx = tail + __popc(m & ((1u << lane) - 1u));
            if (keep) {
              const float uf = __double2float_ru(u);
              if (idx < S8_QCAP) {
                S.qu[cw][idx] = uf;
                S.qp[cw][idx] = (global_pos(st, row0 + r * 32 + lane, sm) << 2) | b;
              } else {
                ovf[b] = fmaxf(ovf[b], uf);
              }
            }
            if (timing && lane == 0) atomicAdd(&S.t[S8T_PUSH], (unsigned long long)__popc(m));
            tail = min(tail + __popc(m), S8_QCAP);
            __syncwarp();
            if (lane == 0) st_rel_cta(&S.qtail[cw], tail);
          }
        }
      }
    }
  }
#pragma unroll
  for (int b = 0; b < NBQ; ++b) {
    float o = ovf[b];
#pragma unroll
    for (int off = 16; off; off >>= 1) o = fmaxf(o, __shfl_xor_sync(FULL, o, off));
    if (lane == 0) S.ovf[cw][b] = o;
  }
  __syncwarp();
  if (lane == 0) {
    __threadfence_block();
    atomicAdd(&S.done, 1);
    if (timing) atomicMax(&S.t[S8T_SCAN], s8_timer());
  }
  s8_pool(x, cw);
}

// ---------------------------------------------------------------- host side
struct S8Plan {
  int Dp = 0;
  int P8 = 0;
  int nst[2] = {0, 0};      // stages in flight (NB = 1, 4)
  size_t smem[2] = {0, 0};  // dynamic shared memory (NB = 1, 4)
};

bool stream8_supported(int Dp) { return Dp % 64 == 0 && Dp >= 64 && Dp <= 1024; }

static size_t s8_smem(int P8, int Dp, int nst, int NB) {
  const int rows = 32 * s8_rows_per_lane(P8 / 128);
  return 1024 + (size_t)nst * rows * P8 + (size_t)nst * (rows + 2) * 8 + (size_t)NB * P8 + (size_t)NB * Dp * 8;
}

// Stage count: as many (<= S8_CW) as fit next to the kernel's static shared memory.
static int s8_fit(int P8, int Dp, int NB, size_t static_smem, size_t optin) {
  int nst = S8_CW;
  while (nst > 1 && static_smem + s8_smem(P8, Dp, nst, NB) > optin) --nst;
  return nst;
}
template <int KB>
static cudaError_t s8_attr(S8Plan* p) {  // sizes the stages, raises the smem limit
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  if (S8_CTAS_PER_SM > 1) {  // keep S8_CTAS_PER_SM CTAs co-resident (1 KB per CTA is reserved)
    int per_sm = 0;
    if ((e = cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev)) != cudaSuccess)
      return e;
    optin = std::min(optin, per_sm / S8_CTAS_PER_SM - 1024);
  }
  cudaFuncAttributes fa1, fa4, fai;
  if ((e = cudaFuncGetAttributes(&fa1, k_stream8_scan<KB, 1, false>)) != cudaSuccess) return e;
  if ((e = cudaFuncGetAttributes(&fa4, k_stream8_scan<KB, 4, false>)) != cudaSuccess) return e;
  if ((e = cudaFuncGetAttributes(&fai, k_stream8_scan<KB, 1, true>)) != cudaSuccess) return e;
  p->nst[0] = s8_fit(p->P8, p->Dp, 1, std::max(fa1.sharedSizeBytes, fai.sharedSizeBytes), (size_t)optin);
  p->nst[1] = s8_fit(p->P8, p->Dp, 4, fa4.sharedSizeBytes, (size_t)optin);
  p->smem[0] = s8_smem(p->P8, p->Dp, p->nst[0], 1);
  p->smem[1] = s8_smem(p->P8, p->Dp, p->nst[1], 4);
  e = cudaFuncSetAttribute(k_stream8_scan<KB, 1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->smem[0]);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_stream8_scan<KB, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->smem[0]);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_stream8_scan<KB, 4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->smem[1]);
}

S8Plan* s8_plan_create(int8_t* ring8, float2* ringq, long long C, int Dp, int P8, char* err, int errlen) {
  (void)ring8;
  (void)ringq;
  (void)C;
  if (!stream8_supported(Dp) || P8 % 128 != 0 || P8 < Dp) {
    snprintf(err, errlen, "stream8 scan needs 64 | Dp <= 1024 and 128 | P8 (Dp=%d, P8=%d)", Dp, P8);
    return nullptr;
  }
  S8Plan* p = new S8Plan();
  p->Dp = Dp;
  p->P8 = P8;
  cudaError_t e;
  switch (P8 / 128) {
    case 1: e = s8_attr<1>(p); break;
    case 2: e = s8_attr<2>(p); break;
    case 3: e = s8_attr<3>(p); break;
    case 4: e = s8_attr<4>(p); break;
    case 5: e = s8_attr<5>(p); break;
    case 6: e = s8_attr<6>(p); break;
    case 7: e = s8_attr<7>(p); break;
    default: e = s8_attr<8>(p); break;
  }
  if (e != cudaSuccess) {
    snprintf(err, errlen, "cannot raise dynamic shared memory to %zu bytes: %s", p->smem[1], cudaGetErrorString(e));
    delete p;
    return nullptr;
  }
  return p;
}

void s8_plan_destroy(S8Plan* p) { delete p; }

template <int KB>
static cudaError_t s8_launch(const S8Plan* p, const RingBufs& rb, const RingState& st, const double* q64, int nb,
                             CtaRec* cta, int b0, int grid, ShardMap sm, const S8Args& a, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(S8_THREADS);
  cfg.dynamicSmemBytes = nb == 1 ? p->smem[0] : p->smem[1];
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // see griddepcontrol in the kernel
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const S8NoIn none{0};
  if (nb == 1)
    return cudaLaunchKernelEx(&cfg, k_stream8_scan<KB, 1, false>, rb, st, q64, nb, cta, b0, sm, a, p->nst[0], p->Dp,
                              none);
  return cudaLaunchKernelEx(&cfg, k_stream8_scan<KB, 4, false>, rb, st, q64, nb, cta, b0, sm, a, p->nst[1], p->Dp,
                            none);
}

template <int KB>
static cudaError_t s8_launch_in(const S8Plan* p, const RingBufs& rb, const RingState& st, CtaRec* cta, int grid,
                                ShardMap sm, const S8Args& a, const S8In& in, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(S8_THREADS);
  cfg.dynamicSmemBytes = p->smem[0];
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_stream8_scan<KB, 1, true>, rb, st, (const double*)nullptr, 1, cta, 0, sm, a,
                            p->nst[0], p->Dp, in);
}

size_t s8_in_bytes() { return sizeof(S8In); }

// One query whose float64 row, int8 quantisation and (<= 1) pending row ride
// in the kernel's parameter block: q64 / stage are HOST rows (D doubles), the
// quantisation is done here into the block.
cudaError_t launch_stream8_direct(const S8Plan* p, const RingBufs& rb, const RingState& st, int D, const double* q64,
                                  const double* stage_row, CtaRec* cta, int grid, ShardMap sm, unsigned* counter,
                                  unsigned long long* gmax, unsigned epoch, const Thresholds& thr, mc_record* rec,
                                  OutRec* out,
                                  RingState* d_state, unsigned* done_seq, unsigned seq, uint4* outp,
                                  void (*quantise)(const double*, int, int, QPrep*, int8_t*), double* gq64,
                                  unsigned* sync, unsigned rec_par, bool overlap, cudaStream_t s) {
  if (!p || p->Dp > S8IN_DMAX || grid > 320) return cudaErrorInvalidValue;
  static thread_local S8In in;
  const int Dp = p->Dp;
  memcpy(in.q64, q64, (size_t)D * sizeof(double));
  memset(in.q64 + D, 0, (size_t)(Dp - D) * sizeof(double));
  quantise(in.q64, D, Dp, &in.prep, in.q8);
  in.hstage = stage_row;
  S8Args a{counter, gmax, thr, rec, out, gemv_timing_buffer(), nullptr, nullptr, nullptr, stage_row ? 1 : 0, d_state,
           done_seq, seq, outp, epoch, gq64, sync, rec_par, overlap ? 1u : 0u};
  switch (p->P8 / 128) {
    case 1: return s8_launch_in<1>(p, rb, st, cta, grid, sm, a, in, s);
    case 2: return s8_launch_in<2>(p, rb, st, cta, grid, sm, a, in, s);
    case 3: return s8_launch_in<3>(p, rb, st, cta, grid, sm, a, in, s);
    case 4: return s8_launch_in<4>(p, rb, st, cta, grid, sm, a, in, s);
    case 5: return s8_launch_in<5>(p, rb, st, cta, grid, sm, a, in, s);
    case 6: return s8_launch_in<6>(p, rb, st, cta, grid, sm, a, in, s);
    case 7: return s8_launch_in<7>(p, rb, st, cta, grid, sm, a, in, s);
    case 8: return s8_launch_in<8>(p, rb, st, cta, grid, sm, a, in, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_stream8_scan(const S8Plan* p, const RingBufs& rb, const RingState& st, const double* q64, int nb,
                                CtaRec* cta, int b0, int grid, ShardMap sm, unsigned* counter,
                                unsigned long long* gmax, unsigned epoch, const Thresholds& thr, mc_record* rec, OutRec* out, const GemvAppendArgs& app,
                                const QPrep* prep, const int8_t* q8, unsigned* done_seq, unsigned seq,
                                uint4* outp, unsigned* sync, unsigned rec_par, bool overlap, cudaStream_t s) {
  if (!p || nb < 1 || nb > 4 || grid > 320) return cudaErrorInvalidValue;  // grid <= 320: the merger's records
  S8Args a{counter, gmax, thr, rec, out, gemv_timing_buffer(), prep, q8, app.stage, app.n, app.d_state, done_seq, seq,
           outp, epoch, nullptr, sync, rec_par, overlap ? 1u : 0u};
  switch (p->P8 / 128) {
    case 1: return s8_launch<1>(p, rb, st, q64, nb, cta, b0, grid, sm, a, s);
    case 2: return s8_launch<2>(p, rb, st, q64, nb, cta, b0, grid, sm, a, s);
    case 3: return s8_launch<3>(p, rb, st, q64, nb, cta, b0, grid, sm, a, s);
    case 4: return s8_launch<4>(p, rb, st, q64, nb, cta, b0, grid, sm, a, s);
    case 5: return s8_launch<5>(p, rb, st, q64, nb, cta, b0, grid, sm, a, s);
    case 6: return s8_launch<6>(p, rb, st, q64, nb, cta, b0, grid, sm, a, s);
    case 7: return s8_launch<7>(p, rb, st, q64, nb, cta, b0, grid, sm, a, s);
    case 8: return s8_launch<8>(p, rb, st, q64, nb, cta, b0, grid, sm, a, s);
    default: return cudaErrorInvalidValue;
  }
}

#undef S
}  // namespace mc
