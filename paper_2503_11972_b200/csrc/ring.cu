// K1 — FIFO ring maintenance (replaces cache.py:181-196's float64 `_buf`).
//
// Pending appends are staged host-side and copied in one H2D per flush; this
// kernel writes each staged float64 row into its ring slot twice — the fp64
// master and the round-to-nearest fp16 scan copy (padding columns zeroed) —
// and publishes the new (head, count, jhead) so graph-captured scans read the
// current window from device memory.
#include "mc_device.cuh"

namespace mc {

__global__ void k_append(const double* __restrict__ stage, long long n, long long first_slot, long long C, int D,
                         int Dp, __half* __restrict__ ring16, double* __restrict__ ring64, RingState* d_state,
                         RingState ns) {
  for (long long r = blockIdx.x; r < n; r += gridDim.x) {
    long long slot = first_slot + r;
    if (slot >= C) slot -= C;
    const double* src = stage + (size_t)r * Dp;
    double* d64 = ring64 + (size_t)slot * Dp;
    __half* d16 = ring16 + (size_t)slot * Dp;
    for (int c = threadIdx.x; c < Dp; c += blockDim.x) {
      const double v = c < D ? src[c] : 0.0;
      d64[c] = v;
      d16[c] = __double2half(v);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *d_state = ns;
}

__global__ void k_set_state(RingState* d_state, RingState ns) { *d_state = ns; }

cudaError_t launch_append(const double* stage, long long n, long long first_slot, const RingState& ns, int D,
                          int Dp, __half* ring16, double* ring64, RingState* d_state, cudaStream_t s) {
  if (n <= 0) {
    k_set_state<<<1, 1, 0, s>>>(d_state, ns);
  } else {
    const int grid = (int)(n < 4096 ? n : 4096);
    k_append<<<grid, 128, 0, s>>>(stage, n, first_slot, ns.cap, D, Dp, ring16, ring64, d_state, ns);
  }
  return cudaGetLastError();
}

}  // namespace mc
