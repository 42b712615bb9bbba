// K1 — FIFO ring maintenance (replaces cache.py:181-196's float64 `_buf`).
//
// Pending appends are staged host-side (the envelope) and copied in one H2D;
// this kernel writes each staged float64 row into every device copy of its
// ring slot — the float64 master, the round-to-nearest fp16 scan copy and the
// per-row-scaled int8 scan copy with its (scale, L1) pair — and publishes the
// new (head, count, jhead).  Small flushes skip it: the fused scans write the
// few rows appended since the last lookup themselves (write_row_all).
#include "mc_device.cuh"

namespace mc {

// One warp per staged row: float64 master, fp16 RN, int8 + (scale, L1).
__global__ void k_append(const double* __restrict__ stage, long long n, long long first_slot, long long C, int Dp,
                         RingBufs rb, RingState* d_state, RingState ns) {
  const int lane = threadIdx.x & 31;
  const long long w0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long r = w0; r < n; r += nw) {
    long long slot = first_slot + r;
    if (slot >= C) slot -= C;
    write_row_all(stage + (size_t)r * Dp, slot, rb, Dp, lane);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *d_state = ns;
}

__global__ void k_set_state(RingState* d_state, RingState ns) { *d_state = ns; }

// Stage rows are zero-padded to Dp (the envelope keeps padding columns zero).
cudaError_t launch_append(const double* stage, long long n, long long first_slot, const RingState& ns, int D,
                          int Dp, const RingBufs& rb, RingState* d_state, cudaStream_t s) {
  (void)D;
  if (n <= 0) {
    k_set_state<<<1, 1, 0, s>>>(d_state, ns);
  } else {
    const long long blocks = (n + 3) / 4;  // 4 warps per block
    const int grid = (int)(blocks < 4096 ? blocks : 4096);
    k_append<<<grid, 128, 0, s>>>(stage, n, first_slot, ns.cap, Dp, rb, d_state, ns);
  }
  return cudaGetLastError();
}

// f4 — on-device synthetic rows (measurement infrastructure for 1M-10M entry
// caches).  The generative model of the reference's
// generators (pkg/src/mixserve/workload.py:124-154, image_embedding +
// gen_queries): row r belongs to cluster c(r); its query is
// q = normalize(center_c + spread * g) and the cached image is
// e = normalize(beta * q + (1 - beta) * g'), g and g' standard-normal-like
// vectors.  Not numpy's PCG64 streams, so never used for golden parity: the
// parity tests read the generated float64 rows back (mc_read_rows) and run the
// oracle on exactly those bits.  Normals are Irwin-Hall(4) sums of counter-
// hashed uniforms (splitmix64), centred and scaled to unit variance.
__device__ __forceinline__ unsigned long long gen_mix(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ double gen_gauss(unsigned long long key) {
  const unsigned long long a = gen_mix(key), b = gen_mix(key ^ 0xD1B54A32D192ED03ull);
  const double u = (double)(a & 0xffffffffu) + (double)(a >> 32) + (double)(b & 0xffffffffu) + (double)(b >> 32);
  return (u * (1.0 / 4294967296.0) - 2.0) * 1.7320508075688772;
}

// One warp per generated row (D <= 1024: 32 elements per lane in registers).
__global__ void k_generate(long long n, long long first_slot, long long C, int D, int Dp, RingBufs rb,
                           const double* __restrict__ centers, int K, double spread, double beta,
                           unsigned long long seed, long long row0, RingState* d_state, RingState ns) {
  const int lane = threadIdx.x & 31;
  const long long w0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long r = w0; r < n; r += nw) {
    const unsigned long long grow = (unsigned long long)(row0 + r);
    const unsigned long long key = gen_mix(seed ^ gen_mix(grow));
    const int c = (int)(key % (unsigned long long)K);
    const double* ctr = centers + (size_t)c * Dp;
    double v[32];
    double ss = 0.0;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const int j = lane + 32 * k;
      v[k] = 0.0;
      if (j < D) {
        v[k] = ctr[j] + spread * gen_gauss(key * 0x100000001B3ull + 2ull * (unsigned long long)j);
        ss += v[k] * v[k];
      }
    }
    ss = warp_sum_d(ss);
    const double qn = sqrt(ss);
    double ss2 = 0.0;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const int j = lane + 32 * k;
      if (j < D) {
        v[k] = beta * (v[k] / qn) + (1.0 - beta) * gen_gauss(key * 0x100000001B3ull + 2ull * (unsigned long long)j + 1ull);
        ss2 += v[k] * v[k];
      }
    }
    ss2 = warp_sum_d(ss2);
    const double en = sqrt(ss2);
    long long slot = first_slot + r;
    if (slot >= C) slot -= C;
    double* d64 = rb.r64 + (size_t)slot * Dp;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const int j = lane + 32 * k;
      if (j < Dp) d64[j] = j < D ? v[k] / en : 0.0;
    }
    __syncwarp();
    write_row_all(d64, slot, rb, Dp, lane);  // every other copy (fp16, int8 + scale) from the float64 row
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *d_state = ns;
}

cudaError_t launch_generate(long long n, long long first_slot, const RingState& ns, int D, int Dp, const RingBufs& rb,
                            const double* centers, int K, double spread, double beta, unsigned long long seed,
                            long long row0, RingState* d_state, cudaStream_t s) {
  if (D > 1024) return cudaErrorInvalidValue;
  const long long blocks = (n + 7) / 8;  // 8 warps per block
  const int grid = (int)(blocks < 8 * 148 ? (blocks > 0 ? blocks : 1) : 8 * 148);
  k_generate<<<grid, 256, 0, s>>>(n, first_slot, ns.cap, D, Dp, rb, centers, K, spread, beta, seed, row0, d_state, ns);
  return cudaGetLastError();
}

// Measurement helper: one thread spinning for `ns` nanoseconds of device time (globaltimer).
__global__ void k_spin(long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while ((long long)(t - t0) < ns);
}

cudaError_t launch_spin(long long ns, cudaStream_t s) {
  k_spin<<<1, 1, 0, s>>>(ns);
  return cudaGetLastError();
}

// Measurement helper (mc_profile_steps): read a buffer larger than L2 so the
// next step starts with the ring evicted and L2 holding only clean lines (a
// write-based flush would leave ~126 MB of dirty lines to write back during
// the timed kernel).
__global__ void k_l2_flush(const uint4* __restrict__ p, size_t n16, unsigned* sink) {
  unsigned acc = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = ld_stream16(p + i);
    acc ^= v.x ^ v.w;
  }
  if (acc == 0x9e3779b9u) *sink = acc;
}

cudaError_t launch_l2_flush(void* buf, size_t bytes, cudaStream_t s) {
  k_l2_flush<<<4 * 148, 256, 0, s>>>(static_cast<const uint4*>(buf), bytes / 16, static_cast<unsigned*>(buf));
  return cudaGetLastError();
}

}  // namespace mc
