// K3 — tensor-core scan for batched lookups (tcgen05 + TMEM + TMA, sm_100a).
//
// Replaces B sequential `_buf[_lo:_hi] @ q` dgemv calls (cache.py:254) with
// one dense contraction S = Q · Rᵀ over the fp16 ring:
//   A = queries  [Bp][Dp] fp16, K-major (q / ||q||, so every row is unit-scale)
//   B = ring     [C ][Dp] fp16, K-major (the ring rows as stored — no transpose)
//   D = scores   [128 queries][256 slots] fp32 in TMEM (double-buffered)
// Queries sit on UMMA M (one 128-row M tile per CTA), ring slots on UMMA N.
// Scores never reach HBM: the epilogue warps pull each accumulator out of
// TMEM (tcgen05.ld 32x32b: thread t <-> query row t) and keep a per-query
// register top-K' plus the largest dropped score (the chunk floor).  The
// per-CTA lists go to the same Partials the GEMV path writes, so the
// certified float64 merge (rescore.cu) is shared.
//
// Warp roles (192 threads, 1 CTA per SM, persistent):
//   warp 0    TMA producer  (one lane): A 128x64 + B 256x64 per K block
//   warp 1    MMA issuer    (one lane): 4 x tcgen05.mma 128x256x16 per K block;
//             also owns the TMEM allocation (512 columns = 2 accumulators)
//   warps 2-5 epilogue: TMEM lane quadrant (warp % 4), 32 queries each
//
// Schedule: grid = n_m * floor(SMs / n_m).  CTA c serves M tile (c % n_m) and
// every (grid / n_m)-th live N tile starting at c / n_m — the n_m CTAs that
// share an N tile run it at the same time, so the ring is read from HBM once
// and from L2 n_m times.  Live N tiles start at the tile holding `head` and
// wrap around the ring; slots outside the live window are masked in the
// epilogue.
//
// Algorithmic work per launch: 2 * Bp * n_live * Dp flops; HBM bytes
// n_live * Dp * 2 + Bp * Dp * 2.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "mc_device.cuh"
#include "sm100.cuh"

namespace mc {

constexpr int TC_BM = 128;      // queries per M tile (UMMA_M)
constexpr int TC_BN = 256;      // ring slots per N tile (UMMA_N)
constexpr int TC_BK = 64;       // fp16 per K block = one 128-byte swizzle row
constexpr int TC_UK = 16;       // UMMA_K for kind::f16
constexpr int TC_STAGES = 4;
constexpr int TC_THREADS = 192;
constexpr int TC_A_BYTES = TC_BM * TC_BK * 2;  // 16 KB
constexpr int TC_B_BYTES = TC_BN * TC_BK * 2;  // 32 KB
constexpr int TC_SMEM = TC_STAGES * (TC_A_BYTES + TC_B_BYTES) + 1024 /*align*/ + 256 /*barriers*/;
constexpr int TC_TMEM_COLS = 2 * TC_BN;  // two fp32 accumulators of 256 columns



// kind::f16 instruction descriptor: fp16 x fp16 -> fp32, both K-major, M x N.
__host__ __device__ constexpr uint32_t umma_idesc_f16(int M, int N) {
  return (1u << 4)                      // D format f32
         | (0u << 7) | (0u << 10)       // A, B format f16
         | ((uint32_t)(N >> 3) << 17)   // N
         | ((uint32_t)(M >> 4) << 24);  // M
}

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}


// ---------------------------------------------------------------- schedule
struct TileWindow {
  int first;    // physical N tile holding the oldest live slot
  int n_live;   // N tiles overlapping the live window
  int n_total;  // N tiles covering the ring
};

__device__ __forceinline__ TileWindow tile_window(const RingState& st) {
  TileWindow w;
  w.n_total = (int)((st.cap + TC_BN - 1) / TC_BN);
  if (st.count <= 0) {
    w.first = 0;
    w.n_live = 0;
  } else if (st.count >= st.cap) {
    w.first = 0;
    w.n_live = w.n_total;
  } else {
    w.first = (int)(st.head / TC_BN);
    const long long end = st.head + st.count;  // one past the newest slot, unwrapped
    long long nl;
    if (end <= st.cap)
      nl = (end - 1) / TC_BN - w.first + 1;
    else  // tiles first .. n_total-1, then 0 .. the tile of the newest wrapped slot
      nl = (w.n_total - w.first) + (end - st.cap - 1) / TC_BN + 1;
    w.n_live = nl < w.n_total ? (int)nl : w.n_total;
  }
  return w;
}

// Register top-K' of one query over the slots a CTA scans: unsorted, with
// the smallest kept score `mn`, the running maximum `runmax`, and the largest
// score not kept (`drop`, the chunk floor).  Admission needs v > mn and
// v > runmax - margin: with margin > 2 delta (delta = the scan's error bound
// in these units) nothing dropped can reach the certified best, so lists stay
// short and the merge's certificate holds; the merge re-checks it anyway.
// Slots stay 32-bit physical ring indices until the list is written out.
struct TopK {
  float s[KP];
  int slot[KP];
  float mn;
  float runmax;
  float drop;

  __device__ __forceinline__ void init() {
#pragma unroll
    for (int i = 0; i < KP; ++i) {
      s[i] = -INFINITY;
      slot[i] = -1;
    }
    mn = -INFINITY;
    runmax = -INFINITY;
    drop = -INFINITY;
  }
  // Precondition: v > mn.  Replaces one entry holding the minimum.
  __device__ __forceinline__ void push(float v, int sl) {
    drop = fmaxf(drop, mn);  // the evicted score (-inf while the list is filling)
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
  // 32 consecutive scores (non-live slots already set to -inf).
  __device__ __forceinline__ void scan32(const float (&v)[32], int slot0, float margin) {
    float m0 = fmaxf(v[0], v[1]), m1 = fmaxf(v[2], v[3]), m2 = fmaxf(v[4], v[5]), m3 = fmaxf(v[6], v[7]);
#pragma unroll
    for (int j = 8; j < 32; j += 8) {
      m0 = fmaxf(m0, fmaxf(v[j + 0], v[j + 1]));
      m1 = fmaxf(m1, fmaxf(v[j + 2], v[j + 3]));
      m2 = fmaxf(m2, fmaxf(v[j + 4], v[j + 5]));
      m3 = fmaxf(m3, fmaxf(v[j + 6], v[j + 7]));
    }
    const float cmax = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3));
    runmax = fmaxf(runmax, cmax);
    const float thr = fmaxf(mn, runmax - margin);
    if (cmax > thr) {  // a new or near maximum in this chunk
      // Elements at or below the chunk-start threshold can never be admitted (the
      // threshold only rises as pushes raise mn): fold them into drop at once, and walk
      // only the others, in slot order, through the sequential admission test.  Each lane
      // loops over its own few candidates instead of the warp predicating all 32 pushes.
      unsigned mask = 0;
      float dr = -INFINITY;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (v[j] > thr)
          mask |= 1u << j;
        else
          dr = fmaxf(dr, v[j]);
      }
      drop = fmaxf(drop, dr);
      while (mask) {
        const int j = __ffs(mask) - 1;
        mask &= mask - 1;
        const float x = pick32(v, j);
        if (x > fmaxf(mn, runmax - margin))
          push(x, slot0 + j);
        else
          drop = fmaxf(drop, x);
      }
    } else {
      drop = fmaxf(drop, cmax);
    }
  }
  // v[j] for a runtime j without local memory: a select tree on the bits of j.
  static __device__ __forceinline__ float pick32(const float (&v)[32], int j) {
    float a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = (j & 1) ? v[2 * i + 1] : v[2 * i];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = (j & 2) ? a[2 * i + 1] : a[2 * i];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = (j & 4) ? a[2 * i + 1] : a[2 * i];
#pragma unroll
    for (int i = 0; i < 2; ++i) a[i] = (j & 8) ? a[2 * i + 1] : a[2 * i];
    return (j & 16) ? a[1] : a[0];
  }
};

// ---------------------------------------------------------------- CTA-pair variant
// cta_group::2: a cluster of two CTAs on one TPC computes a 256-query x
// 256-slot tile per MMA.  CTA r loads queries [256 m + 128 r, +128) and ring
// slots [256 t + 128 r, +128) into its own shared memory; the leader (r = 0)
// issues tcgen05.mma.cta_group::2, which reads the B halves of both CTAs, and
// each CTA's TMEM receives the scores of its own 128 queries against all 256
// slots.  Per SM that is 32 KB of operands per K block instead of 48 KB, so a
// 6-stage ring fits and the tensor pipe is no longer starved.
constexpr int TP_STAGES = 6;
constexpr int TP_A_BYTES = 128 * TC_BK * 2;  // 16 KB: this CTA's 128 queries
constexpr int TP_B_BYTES = 128 * TC_BK * 2;  // 16 KB: this CTA's half of the slot tile
constexpr int TP_SMEM = TP_STAGES * (TP_A_BYTES + TP_B_BYTES) + 1024 + 256;
// The pair kernel runs eight epilogue warps (two per TMEM lane quadrant, each
// owning half of the 256 accumulator columns) so the top-K' filter keeps pace
// with the MMAs; the column halves' lists meet in shared memory at the end.
constexpr int TP_THREADS = 320;
constexpr int TP_X_BYTES = 128 * (2 * KP + 1) * 4;  // half 1's lists: s[KP], slot[KP], drop per query row
// Pair kernel stages: TQ_SUB 64-wide K blocks per stage (fewer barrier round trips per tile),
// TQ_STAGES deep; TQ_SUB x TQ_STAGES = 6 keeps the bytes in flight of the original 6 x 1.
constexpr int TQ_SUB = 2;
constexpr int TQ_STAGES = 3;
constexpr int TP_SMEM_PAIR = TQ_STAGES * TQ_SUB * (TP_A_BYTES + TP_B_BYTES) + 1024 + 256 + TP_X_BYTES;






__device__ __forceinline__ void umma_f16_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                              uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc)
      : "memory");
}


__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TP_THREADS, 1)
    k_tc_scan_pair(const __grid_constant__ CUtensorMap q_map, const __grid_constant__ CUtensorMap ring_map,
                   const __grid_constant__ CUtensorMap ring_map_q,
                   const RingState* __restrict__ d_state, int n_mp, int B, int n_kb, float* __restrict__ part_s,
                   long long* __restrict__ part_p, float* __restrict__ part_floor, int n_chunks, float margin,
                   ShardMap sm, int dbg, unsigned long long* __restrict__ tim) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // tim (MC_GEMV_TIMING=1, measurement only): per-cluster cycle sums at tim[8 + 12 * cluster + i]:
  // 0 MMA-issue loop, 1 MMA waits on full, 2 MMA waits on tempty, 3 units, 4 producer waits on
  // empty, 5 epilogue waits on tfull, 6 epilogue busy, 7 prologue (to griddepcontrol.wait done),
  // 8 MMA-issue loop in globaltimer ns
  const long long t_k0 = clock64();
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smA = smem;
  uint8_t* smB = smem + TQ_STAGES * TQ_SUB * TP_A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smB + TQ_STAGES * TQ_SUB * TP_B_BYTES);
  uint64_t* full = bars;                   // [S]  leader only: TMA bytes of both CTAs
  uint64_t* empty = bars + TQ_STAGES;      // [S]  MMA commit, multicast to both CTAs
  uint64_t* tfull = bars + 2 * TQ_STAGES;  // [2]  MMA commit, multicast to both CTAs
  uint64_t* tempty = tfull + 2;            // [2]  leader only: 4 epilogue warps x 2 CTAs
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int cid = blockIdx.x >> 1;
  const int n_clusters = gridDim.x >> 1;
  const RingState st = *d_state;
  const TileWindow win = tile_window(st);
  const int m_pair = cid % n_mp;
  const int group = cid / n_mp;
  const int n_groups = n_clusters / n_mp;
  // Slot tiles are dealt round-robin over the pair groups.  When the last round is at most
  // half full its tiles are split into 128-slot halves (N = 128 MMAs) over twice as many
  // groups, so no group runs a whole extra tile (C3: 391 tiles over 74 groups).
  const int n_rounds = win.n_live / n_groups, n_rem = win.n_live % n_groups;
  const bool split = n_rem > 0 && 2 * n_rem <= n_groups && !(dbg & 128);
  const int n_full = split ? n_rounds : (win.n_live > group ? (win.n_live - group + n_groups - 1) / n_groups : 0);
  const int n_units = n_full + ((split && group < 2 * n_rem) ? 1 : 0);
  const int n_kg = (n_kb + TQ_SUB - 1) / TQ_SUB;  // stages per unit
  // unit u -> physical tile t and half (-1: the whole 256-slot tile)
  auto unit = [&](int u, int& t, int& hsel) {
    if (u < n_full) {
      t = (win.first + group + u * n_groups) % win.n_total;
      hsel = -1;
    } else {
      t = (win.first + n_rounds * n_groups + (group >> 1)) % win.n_total;
      hsel = group & 1;
    }
  };

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&q_map)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ring_map)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ring_map_q)) : "memory");
    for (int i = 0; i < TQ_STAGES; ++i) {
      mbar_init(&full[i], 2);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 16);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TC_TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Programmatic dependent launch: everything above overlapped k_tc_prep; the
  // query operand it writes is read (by TMA) only after this point.  The ring
  // state was published by kernels that finished before k_tc_prep started.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // and the merge behind this kernel may be scheduled as CTAs retire (it waits for all of them)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  unsigned long long* tcl = tim ? tim + 8 + 12 * (size_t)cid : nullptr;
  if (tcl && rank == 0 && threadIdx.x == 0) atomicAdd(tcl + 7, (unsigned long long)(clock64() - t_k0));

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    // The whole warp walks the loop and lane 0 issues (no lane parked at the closing
    // cluster barrier while lane 0 loops).
    const uint32_t leader_full0 = mapa_shared(smem_u32(&full[0]), 0);
    int stage = 0;
    uint32_t phase = 0;
    long long tw_empty = 0;
    for (int u = 0; u < n_units; ++u) {
      int t, hsel;
      unit(u, t, hsel);
      const int bbytes = hsel < 0 ? TP_B_BYTES : TP_B_BYTES / 2;
      for (int kg = 0; kg < n_kg; ++kg) {
        const int ns = min(TQ_SUB, n_kb - kg * TQ_SUB);
        const long long w0 = tcl ? clock64() : 0;
        mbar_wait2(&empty[stage], phase ^ 1, dbg & 16);
        if (tcl) tw_empty += clock64() - w0;
        if (lane == 0) {
          if (rank == 0)
            mbar_expect_tx(&full[stage], (dbg & 1) ? 0 : 2 * ns * (TP_A_BYTES + bbytes));
          else
            mbar_arrive_remote(leader_full0 + stage * 8);
          if (!(dbg & 1))
            for (int sb = 0; sb < ns; ++sb) {
              const int kb = kg * TQ_SUB + sb;
              uint8_t* da = smA + (stage * TQ_SUB + sb) * TP_A_BYTES;
              uint8_t* db = smB + (stage * TQ_SUB + sb) * TP_B_BYTES;
              tma_load_2d_pair(da, &q_map, &full[stage], kb * TC_BK, m_pair * 256 + rank * 128);
              if (hsel < 0)
                tma_load_2d_pair(db, &ring_map, &full[stage], kb * TC_BK, ((dbg & 8) ? (t & 7) : t) * TC_BN + rank * 128);
              else  // this CTA's 64 slots of the half tile
                tma_load_2d_pair(db, &ring_map_q, &full[stage], kb * TC_BK, t * TC_BN + hsel * 128 + rank * 64);
            }
        }
        __syncwarp();
        if (++stage == TQ_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    if (tcl && rank == 0 && lane == 0) atomicAdd(tcl + 4, (unsigned long long)tw_empty);
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader only)
    if (rank == 0) {
      const long long tm0 = clock64();
      unsigned long long g0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
      long long tw_full = 0, tw_tempty = 0;
      constexpr uint32_t idesc_full = umma_idesc_f16(256, TC_BN);
      constexpr uint32_t idesc_half = umma_idesc_f16(256, TC_BN / 2);
      int stage = 0;
      uint32_t phase = 0;
      for (int u = 0; u < n_units; ++u) {
        int t_unused, hsel;
        unit(u, t_unused, hsel);
        const uint32_t idesc = hsel < 0 ? idesc_full : idesc_half;
        const int acc = u & 1;
        const uint32_t acc_phase = (u >> 1) & 1;
        long long w0 = tcl ? clock64() : 0;
        mbar_wait2(&tempty[acc], acc_phase ^ 1, dbg & 16);
        if (tcl) tw_tempty += clock64() - w0;
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * TC_BN);
        for (int kg = 0; kg < n_kg; ++kg) {
          const int ns = min(TQ_SUB, n_kb - kg * TQ_SUB);
          w0 = tcl ? clock64() : 0;
          mbar_wait2(&full[stage], phase, dbg & 16);
          if (tcl) tw_full += clock64() - w0;
          tc_fence_after();
          if (lane == 0) {
            for (int sb = 0; sb < ns; ++sb) {
              const int kb = kg * TQ_SUB + sb;
              const uint32_t a0 = smem_u32(smA + (stage * TQ_SUB + sb) * TP_A_BYTES);
              const uint32_t b0 = smem_u32(smB + (stage * TQ_SUB + sb) * TP_B_BYTES);
#pragma unroll
              for (int k = 0; k < TC_BK / TC_UK; ++k)
                if (!(dbg & 2))
                  umma_f16_pair(d_tmem, umma_desc_sw128(a0 + k * TC_UK * 2), umma_desc_sw128(b0 + k * TC_UK * 2),
                                idesc, (kb | k) != 0);
            }
            if (dbg & 32) {  // bisection only (valid with dbg & 2): plain arrives instead of the commit
              mbar_arrive(&empty[stage]);
              mbar_arrive_remote(mapa_shared(smem_u32(&empty[stage]), 1));
            } else {
              umma_commit_pair(&empty[stage]);
            }
          }
          __syncwarp();
          if (++stage == TQ_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (lane == 0) umma_commit_pair(&tfull[acc]);
        __syncwarp();
      }
      if (tcl && lane == 0) {
        atomicAdd(tcl + 0, (unsigned long long)(clock64() - tm0));
        atomicAdd(tcl + 1, (unsigned long long)tw_full);
        atomicAdd(tcl + 2, (unsigned long long)tw_tempty);
        atomicAdd(tcl + 3, (unsigned long long)n_units);
        unsigned long long g1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
        atomicAdd(tcl + 8, g1 - g0);  // ns of the MMA-issue loop (clock = tcl[0] / tcl[8])
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    // Warps 2..9: TMEM lane quadrant = warp % 4, column half = (warp - 2) / 4.
    const int quad = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row = quad * 32 + lane;
    const int b = m_pair * 256 + (int)rank * 128 + row;
    const uint32_t leader_tempty0 = mapa_shared(smem_u32(&tempty[0]), 0);
    TopK top;
    top.init();
    long long tw_tfull = 0;
    const long long te0 = clock64();
    for (int u = 0; u < n_units; ++u) {
      const int acc = u & 1;
      const uint32_t acc_phase = (u >> 1) & 1;
      int t, hsel;
      unit(u, t, hsel);
      const int width = hsel < 0 ? TC_BN : TC_BN / 2;  // accumulator columns of this unit
      const int nch = width / 64;                        // 32-column chunks per epilogue warp
      const long long slot0 = (long long)t * TC_BN + (hsel < 0 ? 0 : hsel * 128);
      const long long w0 = tcl ? clock64() : 0;
      mbar_wait(&tfull[acc], acc_phase);
      if (tcl) tw_tfull += clock64() - w0;
      tc_fence_after();
      long long l0 = slot0 - st.head;
      if (l0 < 0) l0 += st.cap;
      const bool all_live = (slot0 + width <= st.cap) && (l0 + width <= st.count);
      // nch (4, or 2 on a half tile) 32-column chunks per warp; chunk c+1's TMEM load overlaps chunk c's filter
      auto filter = [&](uint32_t (&r)[32], int c) {
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        if (!all_live) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const long long slot = slot0 + c * 32 + j;
            long long l = l0 + c * 32 + j;
            if (l >= st.cap) l -= st.cap;
            if (slot >= st.cap || l >= st.count) v[j] = -INFINITY;
          }
        }
        top.scan32(v, (int)(slot0 + c * 32), margin);
      };
      if (!(dbg & 4)) {
        const int c0 = half * nch;
        const uint32_t ta = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * TC_BN + c0 * 32);
        uint32_t rc[32], rn[32];
        tmem_ld32_async(ta, rc);
        tmem_wait_ld();
        tmem_pin(rc);
#pragma unroll 1
        for (int c = 0; c < nch; ++c) {  // one copy of the filter code (instruction cache)
          if (c + 1 < nch) tmem_ld32_async(ta + 32 * (c + 1), rn);
          filter(rc, c0 + c);
          tmem_wait_ld();
          tmem_pin(rn);
#pragma unroll
          for (int j = 0; j < 32; ++j) rc[j] = rn[j];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(leader_tempty0 + acc * 8);
    }
    if (tcl && rank == 0 && warp == 2 && lane == 0) {
      atomicAdd(tcl + 5, (unsigned long long)tw_tfull);
      atomicAdd(tcl + 6, (unsigned long long)(clock64() - te0 - tw_tfull));
    }
    // column half 1 hands its list to half 0 of the same query row
    float* xs = reinterpret_cast<float*>(bars + 32);  // [KP][128] scores (past the 256-byte barrier block)
    int* xp = reinterpret_cast<int*>(xs + KP * 128);  // [KP][128] slots
    float* xd = reinterpret_cast<float*>(xp + KP * 128);  // [128] drop
    if (half == 1) {
#pragma unroll
      for (int i = 0; i < KP; ++i) {
        xs[i * 128 + row] = top.s[i];
        xp[i * 128 + row] = top.slot[i];
      }
      xd[row] = top.drop;
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (half == 0) {
      top.drop = fmaxf(top.drop, xd[row]);
#pragma unroll
      for (int i = 0; i < KP; ++i) {
        const float v = xs[i * 128 + row];
        const int sl = xp[i * 128 + row];
        if (sl < 0) continue;
        if (v > top.mn)
          top.push(v, sl);
        else
          top.drop = fmaxf(top.drop, v);
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
      }
    }
  }

  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TC_TMEM_COLS)
                 : "memory");
  }
}

// q16[b] = fp16(q[b] / ||q[b]||), zero rows for b >= B and zero padding columns;
// qscale[b] = ||q[b]|| turns a scan score back into query units.
__global__ void __launch_bounds__(64) k_tc_prep(const double* __restrict__ q64, int B, int D, int Dp,
                                                 __half* __restrict__ q16, double* __restrict__ qscale) {
  // the pair scan (launched as a programmatic dependent) may start its prologue now
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // one warp per query row, two rows per CTA (B / 2 CTAs spread the 2 MB of C3 queries over
  // the SMs); 16-byte loads, all of a row's loads in flight at once, a warp reduction
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * 2 + (threadIdx.x >> 5);
  const double2* src = reinterpret_cast<const double2*>(q64 + (size_t)b * Dp);  // Dp: a multiple of 64
  const int n2 = Dp >> 1;
  double a = 0.0;
  if (b < B)
    for (int i = lane; i < n2; i += 32) {
      const double2 v = src[i];
      const double x0 = 2 * i < D ? v.x : 0.0, x1 = 2 * i + 1 < D ? v.y : 0.0;
      a = fma(x0, x0, a);
      a = fma(x1, x1, a);
    }
#pragma unroll
  for (int off = 16; off; off >>= 1) a += __shfl_xor_sync(FULL, a, off);
  const double n = sqrt(a);
  const bool ok = b < B && n > 0.0 && isfinite(n);
  const double inv = ok ? 1.0 / n : 0.0;
  // launched as a programmatic dependent of the previous step's merge, which still reads qscale:
  // write only once that grid is done (the query reads above overlap its tail)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int i = lane; i < n2; i += 32) {
    double2 v = make_double2(0.0, 0.0);
    if (ok) v = src[i];
    const double x0 = 2 * i < D ? v.x * inv : 0.0, x1 = 2 * i + 1 < D ? v.y * inv : 0.0;
    reinterpret_cast<__half2*>(q16 + (size_t)b * Dp)[i] = __halves2half2(__double2half(x0), __double2half(x1));
  }
  if (lane == 0 && b < B) qscale[b] = ok ? n : 0.0;
}

// ---------------------------------------------------------------- host side
struct TcPlan {
  __half* ring16 = nullptr;
  long long C = 0;
  int Dp = 0;
  int Bcap = 0;  // multiple of TC_BM
  int sm_count = 0;
  __half* q16 = nullptr;
  double* qscale = nullptr;
  CUtensorMap q_map;
  CUtensorMap ring_map_half;  // 128-slot boxes (CTA-pair kernel)
  CUtensorMap ring_map_q;     // 64-slot boxes (CTA-pair kernel, half-width tail tiles)
  int dbg = 0;  // MC_TC_DEBUG bisection switches: 1 no TMA, 2 no MMA, 4 no epilogue (timing only)
};

static bool encode_2d(CUtensorMap* m, void* base, long long rows, int cols, int box_rows, char* err, int errlen) {
  auto enc = get_encode();
  if (!enc) {
    snprintf(err, errlen, "cuTensorMapEncodeTiled unavailable from the driver");
    return false;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)TC_BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    snprintf(err, errlen, "cuTensorMapEncodeTiled failed (%d) rows=%lld cols=%d", (int)r, rows, cols);
    return false;
  }
  return true;
}

TcPlan* tc_plan_create(__half* ring16, long long C, int Dp, int Bcap, int sm_count, char* err, int errlen) {
  if (Dp % TC_BK != 0) {
    snprintf(err, errlen, "tensor-core scan needs Dp %% %d == 0 (Dp=%d)", TC_BK, Dp);
    return nullptr;
  }
  TcPlan* p = new TcPlan();
  p->ring16 = ring16;
  p->C = C;
  p->Dp = Dp;
  p->Bcap = (Bcap + 255) / 256 * 256;
  p->sm_count = sm_count;
  if (const char* e = getenv("MC_TC_DEBUG")) p->dbg = atoi(e);
  if (cudaMalloc(&p->q16, (size_t)p->Bcap * Dp * sizeof(__half)) != cudaSuccess ||
      cudaMalloc(&p->qscale, (size_t)p->Bcap * sizeof(double)) != cudaSuccess) {
    snprintf(err, errlen, "cudaMalloc failed for the query tile");
    tc_plan_destroy(p);
    return nullptr;
  }
  if (!encode_2d(&p->q_map, p->q16, p->Bcap, Dp, TC_BM, err, errlen) ||
      !encode_2d(&p->ring_map_half, ring16, C, Dp, 128, err, errlen) ||
      !encode_2d(&p->ring_map_q, ring16, C, Dp, 64, err, errlen)) {
    tc_plan_destroy(p);
    return nullptr;
  }
  if (cudaFuncSetAttribute(k_tc_scan_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, TP_SMEM_PAIR) != cudaSuccess) {
    snprintf(err, errlen, "cannot raise dynamic shared memory to %d bytes", TP_SMEM_PAIR);
    tc_plan_destroy(p);
    return nullptr;
  }
  return p;
}

void tc_plan_destroy(TcPlan* p) {
  if (!p) return;
  cudaFree(p->q16);
  cudaFree(p->qscale);
  delete p;
}

int tc_bcap(const TcPlan* p) { return p->Bcap; }

// M pairs (CTA pair, 256 queries) for B queries.
static int tc_nm(const TcPlan* p, int B) {
  (void)p;
  return (B + 255) / 256;
}

int tc_chunks(const TcPlan* p, int B) { return (p->sm_count / 2) / tc_nm(p, B); }  // one list per cluster

const double* tc_qscale(const TcPlan* p) { return p->qscale; }

double gemm_eps_rel(int Dp);

// Admission margin in normalised score units: > 2 delta / ||q|| for every
// query (delta / ||q|| <= eps_rel + eps_abs1 * ||q||_1 / ||q||_2 and
// ||q||_1 <= sqrt(D) ||q||_2), plus slack for the fp32 subtraction.
static float tc_margin(int Dp) {
  return (float)(2.0 * (gemm_eps_rel(Dp) + eps_abs1() * sqrt((double)Dp)) * 1.01 + 1e-6);
}

cudaError_t launch_tc_scan(TcPlan* p, const double* q64, int B, int D, const RingState* d_state,
                           const Partials& part, ShardMap sm, cudaStream_t s) {
  if (B < 1 || B > p->Bcap) return cudaErrorInvalidValue;
  const int nm = tc_nm(p, B);
  const int groups = tc_chunks(p, B);
  if (groups < 1 || groups > part.n_chunks) return cudaErrorInvalidValue;
  const int rows = nm * 256;
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((rows + 1) / 2);
    cfg.blockDim = dim3(64);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // griddepcontrol.wait in k_tc_prep
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_tc_prep, q64, B, D, p->Dp, p->q16, p->qscale);
    if (e != cudaSuccess) return e;
  }
  const float margin = tc_margin(p->Dp);
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * nm * groups);
    cfg.blockDim = dim3(TP_THREADS);
    cfg.dynamicSmemBytes = TP_SMEM_PAIR;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // see griddepcontrol in both kernels
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_tc_scan_pair, p->q_map, p->ring_map_half, p->ring_map_q, d_state, nm, B,
                              p->Dp / TC_BK,
                              part.s, part.p, part.floor_, groups, margin, sm, p->dbg, gemv_timing_buffer());
  }
  return cudaGetLastError();
}

// Error bound of a tensor-core score relative to ||q||_2: entries and the
// normalised query are both fp16-rounded (|de_i| <= u|e_i|, |dq_i| <= u|q_i|,
// so sum |e_i q_i| (2u + u^2) <= (2u + u^2)(1 + 1e-6)), plus fp16 subnormal
// rounding of q/||q|| (2^-25 per component, <= 2^-25 sqrt(Dp) in total), plus
// fp32 accumulation inside the tensor core, bounded as Dp + 16 sequential
// truncating adds (2 u32 each) of terms whose absolute sum is <= 1 + 1e-6.
double gemm_eps_rel(int Dp) {
  const double u16 = ldexp(1.0, -11), u32 = ldexp(1.0, -24);
  const double rounding = (2 * u16 + u16 * u16) * (1.0 + 1e-6);
  const double sub = ldexp(1.0, -25) * sqrt((double)Dp);
  const double accum = (Dp + 16) * 2.0 * u32 * (1.0 + rounding);
  return 1.25 * (rounding + sub + accum);
}

}  // namespace mc
