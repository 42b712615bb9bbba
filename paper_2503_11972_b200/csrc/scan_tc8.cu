// K3q — batched lookups on int8 tensor cores (tcgen05 kind::i8, CTA pairs).
//
// The default path for B >= 5 (C3: 100k x 1024, B = 256).  It replaces B
// sequential `_buf[_lo:_hi] @ q` dgemv calls (cache.py:254) with one dense
// contraction over the int8 ring copy, S = Q̂ · R̂ᵀ (exact int32 in TMEM), and
// certifies candidates with the per-row bounds of the small-batch scans:
//
//   approx = s_e s_q Σ ê_i q̂_i,  delta = ½ s_q ||e||_1 + ½ s_e ||s_q q̂||_1
//   l = approx - delta <= e·q <= u = approx + delta
//
// Against the fp16 tensor-core scan (scan_tc.cu) both operands are half the
// bytes: the ring streams 1 KB per row instead of 2 KB at D = 1024, and the
// per-tile operand traffic into shared memory halves — that traffic, not the
// tensor pipe, bounds the fp16 kernel on this part.  int8 MMAs also run at
// twice the fp16 rate.
//
// Layout (cta_group::2, 192 threads per CTA, one CTA per SM):
//   warp 0     TMA producer: A = 128 quantised queries x 128 B, B = this
//              CTA's 128 slots x 128 B per K block (SWIZZLE_128B), 6 stages
//   warp 1     MMA issuer (leader CTA): 4 x tcgen05.mma.cta_group::2.kind::i8
//              M=256 N=256 K=32 per K block, int32 accumulators double-
//              buffered in TMEM (2 x 256 columns)
//   warps 2-5  epilogue: thread = query row (TMEM lane); per slot column the
//              certified interval [l, u] from the slot's (s_e, ||e||_1)
//              (staged per tile in shared memory) and the query's (s_q, q1);
//              a register top-K' by u with pruning u < max l (dominated rows)
//              and the largest admissible u not kept (the floor)
// Output per (query, CTA pair): K' (u, position), the floor and max l — the
// merge (k_merge8) rescoring every listed row with u >= max l in float64 and
// certifying floor < best.
//
// Algorithmic work per launch: 2 * Bp * n_live * P8 int8 ops; HBM bytes
// n_live * (P8 + 8) + Bp * P8.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "merge.cuh"
#include "sm100.cuh"

namespace mc {

constexpr int T8_BN = 256;                    // ring slots per N tile (per CTA pair)
constexpr int T8_BK = 128;                    // int8 per K block = one 128-byte swizzle row
constexpr int T8_UK = 32;                     // UMMA_K of kind::i8
constexpr int T8_STAGES = 6;
constexpr int T8_THREADS = 192;
constexpr int T8_A_BYTES = 128 * T8_BK;       // 16 KB: this CTA's 128 queries
constexpr int T8_B_BYTES = 128 * T8_BK;       // 16 KB: this CTA's half of the slot tile
constexpr int T8_RQ_BYTES = 2 * T8_BN * 8;    // double-buffered (s, L1) of a tile's slots
constexpr int T8_SMEM = T8_STAGES * (T8_A_BYTES + T8_B_BYTES) + T8_RQ_BYTES + 1024 + 256;
constexpr int T8_TMEM_COLS = 2 * T8_BN;
constexpr float T8_PRUNE = 1e-6f;             // slack of the domination test (float rounding)

// kind::i8 instruction descriptor: s8 x s8 -> s32, both K-major, M x N.
__host__ __device__ constexpr uint32_t umma_idesc_i8(int M, int N) {
  return (2u << 4)                      // D format s32
         | (1u << 7) | (1u << 10)       // A, B signed 8-bit
         | ((uint32_t)(N >> 3) << 17)   // N
         | ((uint32_t)(M >> 4) << 24);  // M
}

__device__ __forceinline__ void umma_i8_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                             uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc)
      : "memory");
}

struct T8Window {
  int first, n_live, n_total;
};

__device__ __forceinline__ T8Window t8_window(const RingState& st) {
  T8Window w;
  w.n_total = (int)((st.cap + T8_BN - 1) / T8_BN);
  if (st.count <= 0) {
    w.first = 0;
    w.n_live = 0;
  } else if (st.count >= st.cap) {
    w.first = 0;
    w.n_live = w.n_total;
  } else {
    w.first = (int)(st.head / T8_BN);
    const long long end = st.head + st.count;
    long long nl;
    if (end <= st.cap)
      nl = (end - 1) / T8_BN - w.first + 1;
    else
      nl = (w.n_total - w.first) + (end - st.cap - 1) / T8_BN + 1;
    w.n_live = nl < w.n_total ? (int)nl : w.n_total;
  }
  return w;
}

// Register top-K' by upper bound of one query over the slots a CTA pair scans.
// Rows with u < runl - T8_PRUNE (runl = the largest lower bound seen) are
// dominated and dropped silently; admissible rows a full list cannot keep
// raise `drop` (the floor), which the merge's certificate must clear.
struct TopK8 {
  float s[KP];
  int slot[KP];
  float mn, runl, drop;

  __device__ __forceinline__ void init() {
#pragma unroll
    for (int i = 0; i < KP; ++i) {
      s[i] = -INFINITY;
      slot[i] = -1;
    }
    mn = -INFINITY;
    runl = -INFINITY;
    drop = -INFINITY;
  }
  __device__ __forceinline__ void push(float v, int sl) {
    drop = fmaxf(drop, mn);
    bool done = false;
#pragma unroll
    for (int i = 0; i < KP; ++i) {
      const bool here = !done && s[i] == mn;
      s[i] = here ? v : s[i];
      slot[i] = here ? sl : slot[i];
      done |= here;
    }
    float m = s[0];
#pragma unroll
    for (int i = 1; i < KP; ++i) m = fminf(m, s[i]);
    mn = m;
  }
  // 32 consecutive slots' bounds (dead slots: u = l = -inf).
  __device__ __forceinline__ void scan32(const float (&u)[32], const float (&l)[32], int slot0) {
    float lm = l[0], um = u[0];
#pragma unroll
    for (int j = 1; j < 32; ++j) {
      lm = fmaxf(lm, l[j]);
      um = fmaxf(um, u[j]);
    }
    runl = fmaxf(runl, lm);
    const float live = runl - T8_PRUNE;
    if (um < live) return;  // every row dominated
    if (um <= mn) {         // admissible rows, none beats the list: the floor covers them
      drop = fmaxf(drop, um);
      return;
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (u[j] < live) continue;
      if (u[j] > mn)
        push(u[j], slot0 + j);
      else
        drop = fmaxf(drop, u[j]);
    }
  }
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(T8_THREADS, 1)
    k_tc8_scan_pair(const __grid_constant__ CUtensorMap q_map, const __grid_constant__ CUtensorMap ring_map,
                    const RingState* __restrict__ d_state, const float2* __restrict__ rq,
                    const float* __restrict__ qs, const float* __restrict__ qn1, int n_mp, int B, int n_kb,
                    float* __restrict__ part_s, long long* __restrict__ part_p, float* __restrict__ part_floor,
                    float* __restrict__ part_maxl, int n_chunks, ShardMap sm, int dbg) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smA = smem;
  uint8_t* smB = smem + T8_STAGES * T8_A_BYTES;
  float2* rqbuf = reinterpret_cast<float2*>(smB + T8_STAGES * T8_B_BYTES);  // [2][T8_BN]
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(rqbuf) + T8_RQ_BYTES);
  uint64_t* full = bars;                   // [S]  leader only: TMA bytes of both CTAs
  uint64_t* empty = bars + T8_STAGES;      // [S]  MMA commit, multicast to both CTAs
  uint64_t* tfull = bars + 2 * T8_STAGES;  // [2]  MMA commit, multicast to both CTAs
  uint64_t* tempty = tfull + 2;            // [2]  leader only: 4 epilogue warps x 2 CTAs
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int cid = blockIdx.x >> 1;
  const int n_clusters = gridDim.x >> 1;
  const RingState st = *d_state;
  const T8Window win = t8_window(st);
  const int m_pair = cid % n_mp;
  const int group = cid / n_mp;
  const int n_groups = n_clusters / n_mp;
  const int n_units = win.n_live > group ? (win.n_live - group + n_groups - 1) / n_groups : 0;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&q_map)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ring_map)) : "memory");
    for (int i = 0; i < T8_STAGES; ++i) {
      mbar_init(&full[i], 2);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(T8_TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      const uint32_t leader_full0 = mapa_shared(smem_u32(&full[0]), 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int u = 0; u < n_units; ++u) {
        const int t = (win.first + group + u * n_groups) % win.n_total;
        for (int kb = 0; kb < n_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (rank == 0)
            mbar_expect_tx(&full[stage], 2 * (T8_A_BYTES + T8_B_BYTES));
          else
            mbar_arrive_remote(leader_full0 + stage * 8);
          tma_load_2d_pair(smA + stage * T8_A_BYTES, &q_map, &full[stage], kb * T8_BK, m_pair * 256 + rank * 128);
          tma_load_2d_pair(smB + stage * T8_B_BYTES, &ring_map, &full[stage], kb * T8_BK, t * T8_BN + rank * 128);
          if (++stage == T8_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader only)
    if (rank == 0) {
      constexpr uint32_t idesc = umma_idesc_i8(256, T8_BN);
      int stage = 0;
      uint32_t phase = 0;
      for (int u = 0; u < n_units; ++u) {
        const int acc = u & 1;
        const uint32_t acc_phase = (u >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * T8_BN);
        for (int kb = 0; kb < n_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a0 = smem_u32(smA + stage * T8_A_BYTES);
            const uint32_t b0 = smem_u32(smB + stage * T8_B_BYTES);
#pragma unroll
            for (int k = 0; k < T8_BK / T8_UK; ++k)
              if (!(dbg & 2)) umma_i8_pair(d_tmem, umma_desc_sw128(a0 + k * T8_UK), umma_desc_sw128(b0 + k * T8_UK), idesc,
                           (kb | k) != 0);
            umma_commit_pair(&empty[stage]);
          }
          __syncwarp();
          if (++stage == T8_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (lane == 0) umma_commit_pair(&tfull[acc]);
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    const int et = (warp - 2) * 32 + lane;  // 0..127: this thread's share of the (s, L1) staging
    const int b = m_pair * 256 + (int)rank * 128 + row;
    const float sq = qs[b];   // padded rows: 0
    const float q1 = qn1[b];
    const uint32_t leader_tempty0 = mapa_shared(smem_u32(&tempty[0]), 0);
    TopK8 top;
    top.init();
    auto tile_slot0 = [&](int u) { return (long long)((win.first + group + u * n_groups) % win.n_total) * T8_BN; };
    auto fetch = [&](long long slot0, float2& r0, float2& r1) {
      const long long a = slot0 + et, c = slot0 + et + 128;
      r0 = a < st.cap ? __ldg(rq + a) : make_float2(0.f, 0.f);
      r1 = c < st.cap ? __ldg(rq + c) : make_float2(0.f, 0.f);
    };
    float2 n0 = make_float2(0.f, 0.f), n1 = n0;
    if (n_units > 0) fetch(tile_slot0(0), n0, n1);
    for (int u = 0; u < n_units; ++u) {
      const int acc = u & 1;
      const uint32_t acc_phase = (u >> 1) & 1;
      const long long slot0 = tile_slot0(u);
      float2* rb = rqbuf + acc * T8_BN;
      rb[et] = n0;
      rb[et + 128] = n1;
      asm volatile("bar.sync 2, 128;" ::: "memory");  // the four epilogue warps: this tile's (s, L1) staged
      if (u + 1 < n_units) fetch(tile_slot0(u + 1), n0, n1);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      long long l0 = slot0 - st.head;
      if (l0 < 0) l0 += st.cap;
      const bool all_live = (slot0 + T8_BN <= st.cap) && (l0 + T8_BN <= st.count);
#pragma unroll 1
      for (int c = 0; c < T8_BN / 32; ++c) {
        if (dbg & 4) break;  // bisection: no epilogue work
        float v[32];
        tmem_ld32(tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * T8_BN + c * 32), v);
        float uu[32], ll[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float2 e = rb[c * 32 + j];  // same address in every lane: a broadcast
          const float dot = (float)__float_as_int(v[j]);  // exact: |dot| <= 1024 * 127^2 < 2^24
          const float approx = dot * (e.x * sq);
          const float d = fmaf(0.5f * sq, e.y, 0.5f * e.x * q1);
          // float rounding of approx (2 ulp) and of d, u, l: a relative + absolute slack
          const float dd = fmaf(d, 1.0f + 1e-5f, fmaf(fabsf(approx), 1e-6f, 1e-6f));
          uu[j] = approx + dd;
          ll[j] = approx - dd;
        }
        if (!all_live) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const long long slot = slot0 + c * 32 + j;
            long long l = l0 + c * 32 + j;
            if (l >= st.cap) l -= st.cap;
            if (slot >= st.cap || l >= st.count) uu[j] = ll[j] = -INFINITY;
          }
        }
        top.scan32(uu, ll, (int)(slot0 + c * 32));
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(leader_tempty0 + acc * 8);
    }
    if (b < B) {
      const size_t o = (size_t)b * n_chunks + group;
#pragma unroll
      for (int i = 0; i < KP; ++i) {
        long long pos = -1;
        if (top.slot[i] >= 0) {
          long long l = (long long)top.slot[i] - st.head;
          if (l < 0) l += st.cap;
          pos = (st.jhead + l) * (long long)sm.G + sm.g;
        }
        part_s[o * KP + i] = top.s[i];
        part_p[o * KP + i] = pos;
      }
      part_floor[o] = top.drop;
      part_maxl[o] = top.runl;
    }
  }

  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(T8_TMEM_COLS)
                 : "memory");
  }
}

// Query quantisation for the int8 MMA: s = max|q| / 127 rounded up (so |q̂| <=
// 127), q̂ = rint(q / s), q1 = s * ||q̂||_1 rounded up.  Rows past B are zero.
__global__ void k_tc8_prep(const double* __restrict__ q64, int B, int D, int Dp, int P8, int8_t* __restrict__ q8,
                           float* __restrict__ qs, float* __restrict__ qn1) {
  __shared__ double red[32];
  __shared__ int redi[32];
  const int b = blockIdx.x;
  double amax = 0.0;
  if (b < B)
    for (int i = threadIdx.x; i < D; i += blockDim.x) amax = fmax(amax, fabs(q64[(size_t)b * Dp + i]));
#pragma unroll
  for (int off = 16; off; off >>= 1) amax = fmax(amax, __shfl_xor_sync(FULL, amax, off));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amax;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    bool finite = true;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      finite &= isfinite(red[w]) != 0;
      m = fmax(m, red[w]);
    }
    red[0] = (finite && m > 0.0 && m <= 1e30) ? (double)__double2float_ru(m / 127.0) : 0.0;
  }
  __syncthreads();
  const double s = red[0];
  int l1 = 0;
  for (int i = threadIdx.x; i < P8; i += blockDim.x) {
    const int v = (b < B && s > 0.0 && i < D) ? __double2int_rn(q64[(size_t)b * Dp + i] / s) : 0;
    q8[(size_t)b * P8 + i] = (int8_t)v;
    l1 += v < 0 ? -v : v;
  }
  l1 = __reduce_add_sync(FULL, l1);
  if ((threadIdx.x & 31) == 0) redi[threadIdx.x >> 5] = l1;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += redi[w];
    qs[b] = (float)s;
    qn1[b] = __double2float_ru((double)t * s);
  }
}

// Certified merge of one query's pair lists with per-row bounds: L = the
// largest lower bound any pair saw; every listed row with u >= L - T8_PRUNE is
// rescored in float64 (a row with u < L is strictly below the row that set
// L); certificate: every floor (largest admissible u a list dropped) lies
// strictly below the best exact score.
__global__ void __launch_bounds__(MERGE_THREADS)
    k_merge8(const RingState* __restrict__ d_state, const double* __restrict__ ring64, int D, int Dp,
             const double* __restrict__ q64, const float* __restrict__ part_s, const long long* __restrict__ part_p,
             const float* __restrict__ part_floor, const float* __restrict__ part_maxl, int n_chunks,
             mc_record* __restrict__ rec, ShardMap sm) {
  extern __shared__ __align__(16) double sq[];  // [Dp]
  __shared__ MergeScratch ms;
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const RingState st = *d_state;
  load_query(q64 + (size_t)b * Dp, D, Dp, sq);
  double n2, n1;
  q_norms(sq, D, ms.shd, n2, n1);
  const bool exotic = !(n1 <= 1e30) || !(n2 >= 1e-30);
  const float* ps = part_s + (size_t)b * n_chunks * KP;
  const long long* pp = part_p + (size_t)b * n_chunks * KP;
  float L = -INFINITY;
  for (int c = threadIdx.x; c < n_chunks; c += blockDim.x) L = fmaxf(L, part_maxl[(size_t)b * n_chunks + c]);
  L = block_max(L, ms.shf);
  const float thr = L - T8_PRUNE;
  if (threadIdx.x == 0) {
    ms.n_cand = 0;
    ms.fail = 0;
  }
  __syncthreads();
  const int ne = n_chunks * KP;
  for (int e = threadIdx.x; e < ne; e += blockDim.x) {
    const long long p = pp[e];
    if (p >= 0 && ps[e] >= thr) {
      const int i = atomicAdd(&ms.n_cand, 1);
      if (i < MERGE_CAND)
        ms.cand[i] = p;
      else
        ms.fail = 1;
    }
  }
  __syncthreads();
  const int n_cand = min(ms.n_cand, MERGE_CAND);
  Best2 best;
  best.init();
  for (int i = warp; i < n_cand; i += MERGE_WARPS) {
    const long long p = ms.cand[i];
    const long long slot = ring_slot(st, local_row(st, p, sm));
    best.add(warp_dot64(ring64 + (size_t)slot * Dp, sq, Dp, lane), p);
  }
  best = block_best(best, ms.shb, true);
  int fail = 0;
  for (int c = threadIdx.x; c < n_chunks; c += blockDim.x) {
    const float f = part_floor[(size_t)b * n_chunks + c];
    if (f > -INFINITY && !((double)f < best.s)) fail = 1;
  }
  if (fail) atomicOr(&ms.fail, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    mc_record r;
    r.sim = best.s;
    r.second = best.s2;
    r.pos = best.p;
    r.flags = (best.ties >= 2 ? MC_FLAG_TIE : 0u) | (ms.fail || best.p < 0 ? FLAG_NEED_FALLBACK : 0u) |
              (exotic ? FLAG_NEED_EXHAUSTIVE : 0u);
    r.reserved = 0;
    rec[b] = r;
  }
}

// ---------------------------------------------------------------- host side
struct Tc8Plan {
  int dbg = 0;  // MC_TC8_DEBUG bisection switches: 2 no MMA, 4 no epilogue (timing only)
  int8_t* q8 = nullptr;  // [Bcap][P8] quantised queries (the A operand)
  float* qs = nullptr;   // [Bcap] s_q
  float* q1 = nullptr;   // [Bcap] s_q ||q̂||_1
  CUtensorMap q_map, ring_map;
  int Bcap = 0, P8 = 0, Dp = 0, sm_count = 0;
};

static bool encode_i8(CUtensorMap* m, void* base, long long rows, int cols, char* err, int errlen) {
  auto enc = get_encode();
  if (!enc) {
    snprintf(err, errlen, "cuTensorMapEncodeTiled unavailable from the driver");
    return false;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols};
  cuuint32_t box[2] = {(cuuint32_t)T8_BK, 128};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    snprintf(err, errlen, "cuTensorMapEncodeTiled (int8) failed (%d) rows=%lld cols=%d", (int)r, rows, cols);
    return false;
  }
  return true;
}

void tc8_plan_destroy(Tc8Plan* p) {
  if (!p) return;
  cudaFree(p->q8);
  cudaFree(p->qs);
  cudaFree(p->q1);
  delete p;
}

bool tc8_supported(int P8) { return P8 % T8_BK == 0 && P8 >= T8_BK && P8 <= 1024; }

Tc8Plan* tc8_plan_create(int8_t* ring8, long long C, int Dp, int P8, int Bcap, int sm_count, char* err, int errlen) {
  if (!tc8_supported(P8)) {
    snprintf(err, errlen, "int8 tensor-core scan needs 128 | P8 <= 1024 (P8=%d)", P8);
    return nullptr;
  }
  Tc8Plan* p = new Tc8Plan();
  p->Bcap = (Bcap + 255) / 256 * 256;
  p->P8 = P8;
  p->Dp = Dp;
  p->sm_count = sm_count;
  if (const char* e = getenv("MC_TC8_DEBUG")) p->dbg = atoi(e);
  if (cudaMalloc(&p->q8, (size_t)p->Bcap * P8) != cudaSuccess ||
      cudaMalloc(&p->qs, (size_t)p->Bcap * sizeof(float)) != cudaSuccess ||
      cudaMalloc(&p->q1, (size_t)p->Bcap * sizeof(float)) != cudaSuccess) {
    snprintf(err, errlen, "cudaMalloc failed for the int8 query tile");
    tc8_plan_destroy(p);
    return nullptr;
  }
  if (!encode_i8(&p->q_map, p->q8, p->Bcap, P8, err, errlen) || !encode_i8(&p->ring_map, ring8, C, P8, err, errlen)) {
    tc8_plan_destroy(p);
    return nullptr;
  }
  if (cudaFuncSetAttribute(k_tc8_scan_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, T8_SMEM) != cudaSuccess) {
    snprintf(err, errlen, "cannot raise dynamic shared memory to %d bytes", T8_SMEM);
    tc8_plan_destroy(p);
    return nullptr;
  }
  return p;
}

int tc8_bcap(const Tc8Plan* p) { return p ? p->Bcap : 0; }

static int tc8_nm(int B) { return (B + 255) / 256; }

int tc8_chunks(const Tc8Plan* p, int B) { return (p->sm_count / 2) / tc8_nm(B); }

cudaError_t launch_tc8_scan(Tc8Plan* p, const double* q64, int B, int D, const RingState* d_state,
                            const float2* rq, const Partials& part, ShardMap sm, cudaStream_t s) {
  if (B < 1 || B > p->Bcap) return cudaErrorInvalidValue;
  const int nm = tc8_nm(B);
  const int groups = tc8_chunks(p, B);
  if (groups < 1 || groups > part.n_chunks || !part.maxl) return cudaErrorInvalidValue;
  k_tc8_prep<<<nm * 256, 128, 0, s>>>(q64, B, D, p->Dp, p->P8, p->q8, p->qs, p->q1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_tc8_scan_pair<<<2 * nm * groups, T8_THREADS, T8_SMEM, s>>>(p->q_map, p->ring_map, d_state, rq, p->qs, p->q1, nm,
                                                                 B, p->P8 / T8_BK, part.s, part.p, part.floor_,
                                                                 part.maxl, groups, sm, p->dbg);
  return cudaGetLastError();
}

cudaError_t launch_merge8(const RingState* d_state, const double* ring64, int D, int Dp, const double* q64, int B,
                          const Partials& part, mc_record* rec, ShardMap sm, cudaStream_t s) {
  const size_t smem = (size_t)Dp * sizeof(double);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_merge8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_merge8<<<B, MERGE_THREADS, smem, s>>>(d_state, ring64, D, Dp, q64, part.s, part.p, part.floor_, part.maxl,
                                          part.n_chunks, rec, sm);
  return cudaGetLastError();
}

}  // namespace mc
