// Derivative-sweep gather layout probe (standalone): the production layout
// (xy double2[n], q D4[n], dq 2xD4[n] per component pair) against one
// 128-byte record per point {q, dq pair 0, dq pair 1, xy, pad}, same
// arithmetic as k_sweep2's fast path, on a real neighbour table.
//   python scripts/sweep_layout_probe.py  (writes /tmp/sweep_geo.bin, builds, runs)
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

struct D4 {
  double a, b, c, d;
};

__device__ __forceinline__ double2 ld2(const double* p) {
  double2 v;
  asm("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void ld4d(const double* p, double2& lo, double2& hi) {
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(lo.x), "=d"(lo.y), "=d"(hi.x), "=d"(hi.y) : "l"(p));
}
__device__ __forceinline__ int4 ld_i4(const int* p) {
  int4 v;
  asm("ld.global.nc.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

// REC = false: xy / q / dq arrays.  REC = true: 16 doubles per point:
// [0..3] q, [4..7] dq pair 0, [8..11] dq pair 1, [12..13] xy.
template <bool REC>
__global__ void __launch_bounds__(256, 2) sweep(int n, const int* __restrict__ nbr, const double2* __restrict__ xy,
                                                const double* __restrict__ qd0, const double* __restrict__ dd0,
                                                double* __restrict__ out) {
  const int h = threadIdx.x & 1;
  const long long n2 = 2ll * n;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < n2; t += stride) {
    const int i = static_cast<int>(t >> 1);
    const int4 a0 = ld_i4(nbr + 8 * i), a1 = ld_i4(nbr + 8 * i + 4);
    const int nb[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
    double2 pi, qi, qxi, qyi;
    if (REC) {
      const double* r = qd0 + 16ll * i;
      pi = ld2(r + 12);
      qi = ld2(r + 2 * h);
      ld4d(r + 4 + 4 * h, qxi, qyi);
    } else {
      pi = xy[i];
      qi = ld2(qd0 + 4ll * i + 2 * h);
      ld4d(dd0 + 8ll * i + 4 * h, qxi, qyi);
    }
    double sxx = 0, sxy = 0, syy = 0, bx0 = 0, bx1 = 0, by0 = 0, by1 = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      double2 pn, qn, qxn, qyn;
      if (REC) {
        const double* r = qd0 + 16ll * nb[j];
        pn = ld2(r + 12);
        qn = ld2(r + 2 * h);
        ld4d(r + 4 + 4 * h, qxn, qyn);
      } else {
        pn = xy[nb[j]];
        qn = ld2(qd0 + 4ll * nb[j] + 2 * h);
        ld4d(dd0 + 8ll * nb[j] + 4 * h, qxn, qyn);
      }
      const double dx = pn.x - pi.x, dy = pn.y - pi.y;
      sxx += dx * dx;
      sxy += dx * dy;
      syy += dy * dy;
      const double df0 = fma(-0.5, fma(dx, qxn.x - qxi.x, dy * (qyn.x - qyi.x)), qn.x - qi.x);
      const double df1 = fma(-0.5, fma(dx, qxn.y - qxi.y, dy * (qyn.y - qyi.y)), qn.y - qi.y);
      bx0 += dx * df0;
      by0 += dy * df0;
      bx1 += dx * df1;
      by1 += dy * df1;
    }
    const double r = 1.0 / (sxx * syy - sxy * sxy);
    double* o = REC ? out + 16ll * i + 4 + 4 * h : out + 8ll * i + 4 * h;
    o[0] = (syy * bx0 - sxy * by0) * r;
    o[1] = (syy * bx1 - sxy * by1) * r;
    o[2] = (sxx * by0 - sxy * bx0) * r;
    o[3] = (sxx * by1 - sxy * bx1) * r;
  }
}

int main(int argc, char** argv) {
  FILE* f = std::fopen(argc > 1 ? argv[1] : "/tmp/sweep_geo.bin", "rb");
  if (!f) return 1;
  int n = 0;
  if (std::fread(&n, 4, 1, f) != 1) return 1;
  std::vector<int> nbr(8ull * n);
  std::vector<double> xy(2ull * n);
  if (std::fread(nbr.data(), 4, nbr.size(), f) != nbr.size()) return 1;
  if (std::fread(xy.data(), 8, xy.size(), f) != xy.size()) return 1;
  std::fclose(f);
  std::vector<double> q(4ull * n), dq(8ull * n), rec(16ull * n, 0.0);
  for (size_t k = 0; k < q.size(); ++k) q[k] = 0.001 * (k % 97);
  for (size_t k = 0; k < dq.size(); ++k) dq[k] = 0.0001 * (k % 89);
  for (int i = 0; i < n; ++i) {
    for (int c = 0; c < 4; ++c) rec[16ull * i + c] = q[4ull * i + c];
    for (int c = 0; c < 8; ++c) rec[16ull * i + 4 + c] = dq[8ull * i + c];
    rec[16ull * i + 12] = xy[2ull * i];
    rec[16ull * i + 13] = xy[2ull * i + 1];
  }
  int *dn;
  double *dxy, *dqv, *ddq, *drec, *dout, *drout;
  cudaMalloc(&dn, nbr.size() * 4);
  cudaMalloc(&dxy, xy.size() * 8);
  cudaMalloc(&dqv, q.size() * 8);
  cudaMalloc(&ddq, dq.size() * 8);
  cudaMalloc(&drec, rec.size() * 8);
  cudaMalloc(&dout, dq.size() * 8);
  cudaMalloc(&drout, rec.size() * 8);
  cudaMemcpy(dn, nbr.data(), nbr.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dxy, xy.data(), xy.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dqv, q.data(), q.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(ddq, dq.data(), dq.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(drec, rec.data(), rec.size() * 8, cudaMemcpyHostToDevice);
  int per_sm = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep<false>, 256, 0);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = std::min((2 * n + 255) / 256, per_sm * sms);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int variant = 0; variant < 2; ++variant) {
    for (int rep = 0; rep < 3; ++rep) {
      const int iters = 20;
      cudaEventRecord(e0);
      for (int k = 0; k < iters; ++k) {
        if (variant == 0)
          sweep<false><<<grid, 256>>>(n, dn, reinterpret_cast<double2*>(dxy), dqv, ddq, dout);
        else
          sweep<true><<<grid, 256>>>(n, dn, nullptr, drec, nullptr, drout);
      }
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      std::printf("%s: %.4f ms per sweep (%d points)\n", variant ? "128-byte records" : "arrays (production)",
                  ms / iters, n);
    }
  }
  std::printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
