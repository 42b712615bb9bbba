// Measurement tooling: host-side cost of the CUDA runtime calls on the lookup's submit path.
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_nop(int* p) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && p[0] == 12345) p[1] = 1;
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  char* h;
  char* d;
  cudaMallocHost(&h, 1 << 20);
  cudaMalloc(&d, 1 << 20);
  cudaEvent_t ev;
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  auto now = [] { return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  const int N = 2000;
  double t_cp = 0, t_ev = 0, t_l = 0, t_lx = 0;
  for (int i = 0; i < N + 50; ++i) {
    const double a = now();
    cudaMemcpyAsync(d, h, 13 * 1024, cudaMemcpyHostToDevice, s);
    const double b = now();
    cudaEventRecord(ev, s);
    const double c = now();
    k_nop<<<148, 384, 0, s>>>((int*)d);
    const double e = now();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(384);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_nop, (int*)d);
    const double f = now();
    cudaStreamSynchronize(s);
    if (i >= 50) {
      t_cp += b - a;
      t_ev += c - b;
      t_l += e - c;
      t_lx += f - e;
    }
  }
  printf("memcpyAsync 13 KB pinned %.2f us | eventRecord %.2f us | launch <<<>>> %.2f us | launchEx+PDL %.2f us\n",
         t_cp / N, t_ev / N, t_l / N, t_lx / N);
  return 0;
}
