// First DMA into freshly pinned host memory vs later DMAs (profiling aid):
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o /tmp/pfd scripts/pin_first_dma.cu && /tmp/pfd
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
static double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
int main() {
  const size_t sizes[] = {size_t(1) << 30, size_t(6720) << 20};
  char* d;
  cudaMalloc((void**)&d, sizes[1]);
  cudaFree(0);
  for (size_t n : sizes) {
    for (int rep = 0; rep < 2; ++rep) {
      char* h;
      double t0 = now_ms();
      cudaHostAlloc((void**)&h, n, cudaHostAllocPortable);
      double t1 = now_ms();
      cudaMemcpy(h, d, n, cudaMemcpyDeviceToHost);
      double t2 = now_ms();
      cudaMemcpy(h, d, n, cudaMemcpyDeviceToHost);
      double t3 = now_ms();
      cudaMemcpy(d, h, n, cudaMemcpyHostToDevice);
      double t4 = now_ms();
      cudaFreeHost(h);
      double t5 = now_ms();
      printf("%.2f GB: alloc %.1f ms, D2H#1 %.1f ms (%.1f GB/s), D2H#2 %.1f ms (%.1f GB/s), H2D %.1f ms, free %.1f ms\n",
             n / 1e9, t1 - t0, t2 - t1, n / (t2 - t1) / 1e6, t3 - t2, n / (t3 - t2) / 1e6, t4 - t3, t5 - t4);
    }
  }
  return 0;
}
