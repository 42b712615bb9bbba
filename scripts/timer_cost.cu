// Measurement tooling: cost of reading %globaltimer vs clock64 inside a kernel,
// and the latency of one 6 KB float64 row read (cold) by a warp.
#include <cstdio>
__global__ void k(unsigned long long* out, const double* row) {
  unsigned long long g0, g1;
  long long c0 = clock64();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  for (int i = 0; i < 100; ++i) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  long long c1 = clock64();
  double2 a[12];
  long long c2 = clock64();
  for (int j = 0; j < 12; ++j) a[j] = __ldg(reinterpret_cast<const double2*>(row + 64 * j + 2 * (threadIdx.x & 31)));
  double s = 0;
  for (int j = 0; j < 12; ++j) s += a[j].x + a[j].y;
  long long c3 = clock64();
  if (threadIdx.x == 0) {
    out[0] = c1 - c0;
    out[1] = g1 - g0;
    out[2] = c3 - c2;
    out[3] = (unsigned long long)s;
  }
}
int main() {
  unsigned long long* d;
  double* row;
  cudaMalloc(&d, 64);
  cudaMalloc(&row, 1 << 24);
  cudaMemset(row, 0, 1 << 24);
  unsigned long long h[4];
  for (int rep = 0; rep < 3; ++rep) {
    k<<<1, 32>>>(d, row + rep * 100000);
    cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("101 globaltimer reads: %llu cycles, %llu ns of globaltimer; cold 6KB warp row read: %llu cycles\n", h[0],
           h[1], h[2]);
  }
  return 0;
}
