// Microbenchmark (measurement tooling, not product): tcgen05.mma issue rate on one B200, SS mode
// (both operands in shared memory, SW128 K-major), the shapes the C3 pair kernel uses.
//   mode 0: cta_group::2, M=256 N=256 K=16, one commit at the end (pure issue rate)
//   mode 1: cta_group::2, M=256 N=256, commit every `per` MMAs, the issuer waits for the commit
//           `lag` commits back (the pair kernel's stage pipeline without a producer)
//   mode 2: cta_group::1, M=128 N=256 K=16, one commit at the end
//   mode 3: cta_group::2, M=256 N=128 (the half-tile MMAs)
// One cluster of two CTAs per TPC (74 clusters), operands never reloaded (contents irrelevant).
// Prints cycles per MMA (leader clock64) and the chip-wide TFLOP/s from globaltimer.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2503_11972_b200/csrc -o scripts/mma_mb scripts/mma_microbench.cu -lcuda
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "sm100.cuh"

using namespace mc;

__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma1(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit1(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    k_mma(int mode, int n_mma, int per, int lag, long long* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* A = sm;              // 128 x 64 fp16, SW128 (16 KB)
  uint8_t* Bm = sm + 16384;     // 128 x 64 fp16 (16 KB)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 32768);  // [8]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool pair = mode != 2;
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 1) {
    if (pair) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "r"(512)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "r"(512)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const bool issuer = warp == 1 && lane == 0 && (!pair || rank == 0);
  if (issuer) {
    const uint32_t id = mode == 2 ? idesc_f16(128, 256) : mode == 3 ? idesc_f16(256, 128) : idesc_f16(256, 256);
    // descriptors once; a K step of 16 fp16 (32 bytes) adds 2 to the start-address field
    const uint64_t da0 = umma_desc_sw128(smem_u32(A)), db0 = umma_desc_sw128(smem_u32(Bm));
    const long long c0 = clock64();
    const uint64_t g0 = gtime();
    int ncommit = 0;
    const int n_grp = n_mma / 8;  // groups of 8 MMAs (one pair-kernel stage: two 64-wide K blocks)
    for (int g = 0; g < n_grp; ++g) {
      const uint32_t d = tmem + (uint32_t)(((g >> 3) & 1) * 256);
      if (pair) {
#pragma unroll
        for (int k = 0; k < 8; ++k) mma2(d, da0 + 2 * (k & 3), db0 + 2 * (k & 3), id, (g & 7) | k);
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) mma1(d, da0 + 2 * (k & 3), db0 + 2 * (k & 3), id, (g & 7) | k);
      }
      if (mode == 1) {
        umma_commit_pair(&bars[ncommit & 7]);
        ++ncommit;
        if (ncommit > lag) {  // wait for the commit `lag` back
          const int w = ncommit - 1 - lag;
          mbar_wait(&bars[w & 7], (w >> 3) & 1);
        }
      }
    }
    if (pair)
      umma_commit_pair(&bars[ncommit & 7]);
    else
      commit1(&bars[ncommit & 7]);
    // drain every outstanding commit in order
    for (int w = (mode == 1 ? (ncommit > lag ? ncommit - lag : 0) : ncommit); w <= ncommit; ++w)
      mbar_wait(&bars[w & 7], (w >> 3) & 1);
    const long long c1 = clock64();
    const uint64_t g1 = gtime();
    const int cl = blockIdx.x >> (pair ? 1 : 0);
    out[cl * 4 + 0] = c1 - c0;
    out[cl * 4 + 1] = (long long)(g1 - g0);
    out[cl * 4 + 2] = (long long)g0;
    out[cl * 4 + 3] = (long long)g1;
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 1) {
    if (pair)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

int main(int argc, char** argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 32768 + 1024 + 256;
  cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long* d_out;
  cudaMalloc(&d_out, sizeof(long long) * 4 * sms);
  long long* h = (long long*)malloc(sizeof(long long) * 4 * sms);
  struct Case { int mode, n, per, lag; const char* name; };
  const Case cases[] = {
      {0, 4096, 0, 0, "pair M256 N256, one commit"},
      {1, 4096, 8, 2, "pair M256 N256, commit/8 wait lag 2"},
      {1, 4096, 8, 1, "pair M256 N256, commit/8 wait lag 1"},
      {1, 4096, 8, 0, "pair M256 N256, commit/8 wait lag 0 (serialised)"},
      {3, 4096, 0, 0, "pair M256 N128, one commit"},
  };
  for (const Case& c : cases) {
    const int grid = (c.mode == 2) ? sms : 2 * (sms / 2);
    for (int rep = 0; rep < 3; ++rep) {
      k_mma<<<grid, 128, smem>>>(c.mode, c.n, c.per, c.lag, d_out);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("%s: %s\n", c.name, cudaGetErrorString(e));
        return 1;
      }
    }
    cudaMemcpy(h, d_out, sizeof(long long) * 4 * sms, cudaMemcpyDeviceToHost);
    const int nunits = c.mode == 2 ? grid : grid / 2;
    double cyc = 0, ns = 0;
    long long gmin = h[2], gmax = h[3];
    for (int i = 0; i < nunits; ++i) {
      cyc += h[i * 4];
      ns += h[i * 4 + 1];
      gmin = h[i * 4 + 2] < gmin ? h[i * 4 + 2] : gmin;
      gmax = h[i * 4 + 3] > gmax ? h[i * 4 + 3] : gmax;
    }
    cyc /= nunits;
    ns /= nunits;
    const double M = c.mode == 2 ? 128 : 256, N = c.mode == 3 ? 128 : 256;
    const double flops = 2.0 * M * N * 16 * c.n * nunits;
    printf("%-52s %7.1f cyc/MMA  clk %.0f MHz  %.0f TFLOP/s (span %.1f us)\n", c.name, cyc / c.n,
           cyc / ns * 1e3, flops / (double)(gmax - gmin) / 1e3, (gmax - gmin) / 1e3);
  }
  return 0;
}
