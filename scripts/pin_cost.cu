// Cost of pinning a 27 MB host store: cudaHostAlloc vs cudaHostRegister of an
// existing (touched) allocation, and the D2H rate straight into it.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o /tmp/pin_cost scripts/pin_cost.cu
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
static double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
int main() {
  const size_t N = 21ull * 160160 * 8;
  char* d;
  cudaMalloc((void**)&d, N);
  cudaFree(0);
  for (int rep = 0; rep < 4; ++rep) {
    double t0 = now_ms();
    char* h;
    cudaHostAlloc((void**)&h, N, 0);
    double t1 = now_ms();
    cudaMemcpy(h, d, N, cudaMemcpyDeviceToHost);
    double t2 = now_ms();
    cudaFreeHost(h);
    double t3 = now_ms();
    char* m = (char*)aligned_alloc(4096, N);
    memset(m, 0, N);
    double t4 = now_ms();
    cudaHostRegister(m, N, cudaHostRegisterDefault);
    double t5 = now_ms();
    cudaMemcpy(m, d, N, cudaMemcpyDeviceToHost);
    double t6 = now_ms();
    cudaHostUnregister(m);
    double t7 = now_ms();
    char* u = (char*)aligned_alloc(4096, N);
    double t8 = now_ms();
    cudaHostRegister(u, N, cudaHostRegisterDefault);  // untouched pages
    double t9 = now_ms();
    cudaHostUnregister(u);
    free(u);
    free(m);
    std::printf("hostalloc %.3f  d2h %.3f  freehost %.3f | memset %.3f register %.3f d2h %.3f unregister %.3f | register untouched %.3f\n",
                t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t6 - t5, t7 - t6, t9 - t8);
  }
}
