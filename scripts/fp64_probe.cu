// FP64 pipe probe (profiling aid): dependent-chain latency and throughput of
// DFMA on one SM for 1..8 independent chains per warp and 1..16 warps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/fp64_probe.cu -o /tmp/fp64_probe && /tmp/fp64_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void chains(double* out, int iters, double m, long long* cycles) {
  double v[C];
#pragma unroll
  for (int c = 0; c < C; ++c) v[c] = threadIdx.x * 1e-3 + c;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c) v[c] = fma(v[c], m, 1e-9);
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += v[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int C>
void run(int warps, double* out, long long* cyc) {
  const int iters = 4096;
  chains<C><<<1, 32 * warps>>>(out, iters, 0.999999, cyc);
  chains<C><<<1, 32 * warps>>>(out, iters, 0.999999, cyc);
  long long c = 0;
  cudaMemcpy(&c, cyc, sizeof c, cudaMemcpyDeviceToHost);
  const double per = double(c) / (double(iters) * C);
  printf("chains/warp %d warps/SM %2d: %6.2f cycles per DFMA per warp, SM rate %5.2f warp-DFMA/cycle\n", C, warps,
         per, warps / per);
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 1 << 12);
  for (int w : {1, 4, 8, 16}) {
    run<1>(w, out, cyc);
    run<2>(w, out, cyc);
    run<4>(w, out, cyc);
    run<8>(w, out, cyc);
  }
  return 0;
}
