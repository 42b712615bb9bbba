// K2 — batch-1..4 GEMV scan over the fp16 ring (HBM-bound path).
//
// Replaces the OpenBLAS dgemv of cache.py:254 for small batches.  Each CTA
// owns a contiguous chunk of live rows; each warp streams R rows at a time
// with 16-byte `ld.global.nc.L1::no_allocate` loads (R*NJ loads in flight per
// lane), converts fp16 -> fp32, FMAs against the fp32 query held in
// registers, and reduces with a 5-step xor butterfly (every lane ends with
// the same bits).  Scores never leave registers: each warp keeps a sorted
// top-K' list spread over lanes 0..K'-1, then the CTA merges its 8 warp lists
// and writes one K' list + a "floor" (largest score it dropped, or -inf) —
// the data the certificate in rescore.cu needs.
//
// Algorithmic bytes per lookup: count * Dp * 2 (+ Dp * 8 for q).
#include "mc_device.cuh"

namespace mc {

constexpr int GEMV_THREADS = 256;
constexpr int GEMV_WARPS = GEMV_THREADS / 32;

__device__ __forceinline__ void fma8(float& acc, const uint4& v, const float* q) {
  const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    float2 f = __half22float2(h[t]);
    acc = fmaf(f.x, q[2 * t], acc);
    acc = fmaf(f.y, q[2 * t + 1], acc);
  }
}

template <int NJ, int NB, int R>
__global__ void __launch_bounds__(GEMV_THREADS, 2)
    k_gemv_scan(const __half* __restrict__ ring16, const RingState* __restrict__ d_state, int Dp,
                const double* __restrict__ q64, int nb, float* __restrict__ part_s, long long* __restrict__ part_p,
                float* __restrict__ part_floor, int n_chunks, int part_b0, ShardMap sm) {
  const RingState st = *d_state;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int n16 = Dp >> 3;  // 16-byte chunks per row

  // Query in fp32 registers: lane owns chunks lane + 32*j.
  float q[NB][NJ][8];
#pragma unroll
  for (int b = 0; b < NB; ++b)
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int c = lane + 32 * j;
#pragma unroll
      for (int t = 0; t < 8; ++t)
        q[b][j][t] = (b < nb && c < n16) ? (float)q64[(size_t)b * Dp + c * 8 + t] : 0.f;
    }

  // Per-warp sorted top-K': lane k < KP holds the k-th best (score, pos).
  float ls[NB];
  long long lp[NB];
  float wmin[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    ls[b] = -INFINITY;
    lp[b] = -1;
    wmin[b] = -INFINITY;
  }

  const long long n = st.count;
  const long long per = (n + gridDim.x - 1) / gridDim.x;
  const long long r0 = (long long)blockIdx.x * per;
  const long long r1 = min(n, r0 + per);

  for (long long base = r0 + (long long)warp * R; base < r1; base += (long long)GEMV_WARPS * R) {
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
      const long long pos = global_pos(st, row, sm);
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < NJ; ++j) fma8(acc, v[r][j], q[b][j]);
#pragma unroll
        for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(FULL, acc, off);
        if (b < nb && acc > wmin[b]) {  // warp-uniform: acc and wmin are identical in all lanes
          const unsigned ahead = __ballot_sync(FULL, lane < KP && ls[b] >= acc);
          const int at = __popc(ahead);
          const float up_s = __shfl_up_sync(FULL, ls[b], 1);
          const long long up_p = __shfl_up_sync(FULL, lp[b], 1);
          if (lane == at) {
            ls[b] = acc;
            lp[b] = pos;
          } else if (lane > at && lane < KP) {
            ls[b] = up_s;
            lp[b] = up_p;
          }
          wmin[b] = __shfl_sync(FULL, ls[b], KP - 1);
        }
      }
    }
  }

  // CTA merge of the 8 warp lists -> one K' list per query.
  __shared__ float sh_s[NB][GEMV_WARPS * KP];
  __shared__ long long sh_p[NB][GEMV_WARPS * KP];
#pragma unroll
  for (int b = 0; b < NB; ++b)
    if (lane < KP) {
      sh_s[b][warp * KP + lane] = ls[b];
      sh_p[b][warp * KP + lane] = lp[b];
    }
  __syncthreads();
  const long long seen = r1 > r0 ? r1 - r0 : 0;
  for (int b = 0; b < nb; ++b) {
    float* os = part_s + ((size_t)(part_b0 + b) * n_chunks + blockIdx.x) * KP;
    long long* op = part_p + ((size_t)(part_b0 + b) * n_chunks + blockIdx.x) * KP;
    if (threadIdx.x < GEMV_WARPS * KP) {
      const int e = threadIdx.x;
      const float s = sh_s[b][e];
      const long long p = sh_p[b][e];
      int rank = 0;
      for (int o = 0; o < GEMV_WARPS * KP; ++o) {
        const float so = sh_s[b][o];
        const long long po = sh_p[b][o];
        // strict total order on (score, pos, slot) so ranks are a permutation
        rank += (so > s) || (so == s && (po > p || (po == p && o < e)));
      }
      if (rank < KP) {
        os[rank] = s;
        op[rank] = p;
      }
      if (rank == KP - 1)
        part_floor[(size_t)(part_b0 + b) * n_chunks + blockIdx.x] = seen > KP ? s : -INFINITY;
    }
  }
}

int gemv_grid(int sm_count) { return 2 * sm_count; }

template <int NJ>
static cudaError_t launch_nj(const __half* ring16, const RingState* d_state, int Dp, const double* q64, int nb,
                             const Partials& part, int part_b0, int grid, ShardMap sm, cudaStream_t s) {
  constexpr int R1 = NJ <= 4 ? 4 : (NJ <= 8 ? 2 : 1);
  constexpr int R2 = NJ <= 4 ? 2 : 1;
  if (nb == 1)
    k_gemv_scan<NJ, 1, R1><<<grid, GEMV_THREADS, 0, s>>>(ring16, d_state, Dp, q64, nb, part.s, part.p, part.floor_,
                                                         part.n_chunks, part_b0, sm);
  else if (nb == 2)
    k_gemv_scan<NJ, 2, R2><<<grid, GEMV_THREADS, 0, s>>>(ring16, d_state, Dp, q64, nb, part.s, part.p, part.floor_,
                                                         part.n_chunks, part_b0, sm);
  else
    k_gemv_scan<NJ, 4, 1><<<grid, GEMV_THREADS, 0, s>>>(ring16, d_state, Dp, q64, nb, part.s, part.p, part.floor_,
                                                        part.n_chunks, part_b0, sm);
  return cudaGetLastError();
}

cudaError_t launch_gemv_scan(const __half* ring16, const RingState* d_state, int Dp, const double* q64, int nb,
                             const Partials& part, int part_b0, int grid, ShardMap sm, cudaStream_t s) {
  const int nj = (Dp / 8 + 31) / 32;
  if (nb < 1 || nb > 4) return cudaErrorInvalidValue;
  switch (nj) {
    case 1: return launch_nj<1>(ring16, d_state, Dp, q64, nb, part, part_b0, grid, sm, s);
    case 2: return launch_nj<2>(ring16, d_state, Dp, q64, nb, part, part_b0, grid, sm, s);
    case 3: return launch_nj<3>(ring16, d_state, Dp, q64, nb, part, part_b0, grid, sm, s);
    case 4: return launch_nj<4>(ring16, d_state, Dp, q64, nb, part, part_b0, grid, sm, s);
    case 5: case 6: return launch_nj<6>(ring16, d_state, Dp, q64, nb, part, part_b0, grid, sm, s);
    case 7: case 8: return launch_nj<8>(ring16, d_state, Dp, q64, nb, part, part_b0, grid, sm, s);
    default:
      if (nj <= 12) return launch_nj<12>(ring16, d_state, Dp, q64, nb, part, part_b0, grid, sm, s);
      if (nj <= 16) return launch_nj<16>(ring16, d_state, Dp, q64, nb, part, part_b0, grid, sm, s);
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
