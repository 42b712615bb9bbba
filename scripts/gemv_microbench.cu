// Microbenchmark (measurement tooling, not product): the GEMV access pattern in isolation.
// rows x 768 fp16, warp reads R rows per batch (lane owns 16-byte chunks lane + 32 j), then
// (optionally) fp32 dot + butterfly.  Variants: order (0 per-warp contiguous, 1 grid-linear),
// CTAs per SM, R, compute on/off, software prefetch of the next batch.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint4 ldnc(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

template <int R, bool COMPUTE, bool PREFETCH>
__global__ void k(const __half* __restrict__ ring, long long n, int order, const float* __restrict__ qg, float* out) {
  constexpr int NJ = 3, DP = 768;
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  const long long w = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  float q[NJ][8];
#pragma unroll
  for (int j = 0; j < NJ; ++j)
#pragma unroll
    for (int t = 0; t < 8; ++t) q[j][t] = qg[(lane + 32 * j) * 8 + t];
  long long r0, r1, step;
  if (order == 0) {
    const long long per = (n + warps - 1) / warps;
    r0 = w * per;
    r1 = min(n, r0 + per);
    step = R;
  } else {
    r0 = w * R;
    r1 = n;
    step = warps * R;
  }
  float best = -1e30f;
  uint4 nx[R][NJ];
  if (PREFETCH && r0 < r1) {
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int j = 0; j < NJ; ++j)
        nx[r][j] = (r0 + r < r1) ? ldnc(ring + (size_t)(r0 + r) * DP + (lane + 32 * j) * 8) : make_uint4(0, 0, 0, 0);
  }
  for (long long base = r0; base < r1; base += step) {
    uint4 v[R][NJ];
    if (PREFETCH) {
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int j = 0; j < NJ; ++j) v[r][j] = nx[r][j];
      const long long nb = base + step;
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int j = 0; j < NJ; ++j)
          nx[r][j] = (nb + r < r1) ? ldnc(ring + (size_t)(nb + r) * DP + (lane + 32 * j) * 8) : make_uint4(0, 0, 0, 0);
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int j = 0; j < NJ; ++j)
          v[r][j] = (base + r < r1) ? ldnc(ring + (size_t)(base + r) * DP + (lane + 32 * j) * 8) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float acc = 0.f;
      if (COMPUTE) {
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          const __half2* h = reinterpret_cast<const __half2*>(&v[r][j]);
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float2 f = __half22float2(h[t]);
            acc = fmaf(f.x, q[j][2 * t], acc);
            acc = fmaf(f.y, q[j][2 * t + 1], acc);
          }
        }
#pragma unroll
        for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      } else {
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc += __uint_as_float(v[r][j].x ^ v[r][j].w);
      }
      best = fmaxf(best, acc);
    }
  }
  if (best == 123.f) out[0] = best;
}

template <int R, bool C, bool P>
float run(const __half* ring, long long n, int order, int cps, const float* q, float* out, void* flush, int sms) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int rep = 0; rep < 4; ++rep) {
    cudaMemsetAsync(flush, rep, 512 << 20);
    cudaEventRecord(a);
    k<R, C, P><<<sms * cps, 256>>>(ring, n, order, q, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep) best = fminf(best, ms);
  }
  return best * 1e3f;
}

int main() {
  const long long n = 100000;
  __half* ring;
  cudaMalloc(&ring, n * 768 * 2);
  cudaMemset(ring, 0, n * 768 * 2);
  float *q, *out;
  cudaMalloc(&q, 768 * 4);
  cudaMemset(q, 0, 768 * 4);
  cudaMalloc(&out, 4);
  void* flush;
  cudaMalloc(&flush, 512 << 20);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double mb = n * 768 * 2 / 1e6;
#define RUN(R, C, P, order, cps)                                                                      \
  {                                                                                                   \
    float us = run<R, C, P>(ring, n, order, cps, q, out, flush, sms);                               \
    printf("R=%d compute=%d prefetch=%d order=%d ctas/sm=%d: %.1f us  %.0f GB/s\n", R, C, P, order, cps, us, \
           mb / us * 1e3);                                                                            \
  }
  RUN(6, true, false, 0, 2) RUN(6, false, false, 0, 2) RUN(6, true, false, 1, 2) RUN(6, false, false, 1, 2)
  RUN(2, true, false, 0, 4) RUN(2, true, false, 1, 4) RUN(4, true, false, 0, 3) RUN(4, true, false, 1, 3)
  RUN(3, true, true, 0, 2) RUN(3, true, true, 1, 2) RUN(1, true, false, 1, 8) RUN(1, false, false, 1, 8)
  RUN(2, true, true, 1, 3) RUN(8, true, false, 1, 1) RUN(6, true, false, 1, 1)
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
