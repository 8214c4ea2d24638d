// DMA rate into/out of pinned staging depending on how host threads touched
// the staging lines just before (regular stores, streaming stores, reads,
// reads + clflushopt).  Standalone probe for the e2e copy path:
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -Xcompiler -mclflushopt -o /tmp/dma_probe scripts/dma_probe.cu -lpthread
#include <cuda_runtime.h>
#include <emmintrin.h>
#include <immintrin.h>

#include <cstdio>
#include <cstring>
#include <functional>
#include <thread>
#include <vector>

static const size_t N = 21ull * 160160 * 8;  // bytes
static const int T = 16;

static void par(const std::function<void(size_t, size_t)>& f) {
  std::vector<std::thread> th;
  for (int k = 0; k < T; ++k) {
    size_t lo = (N * k / T) & ~size_t(63), hi = (N * (k + 1) / T) & ~size_t(63);
    if (k == T - 1) hi = N;
    th.emplace_back([&f, lo, hi] { f(lo, hi); });
  }
  for (auto& t : th) t.join();
}

static void nt_copy(char* dst, const char* src, size_t n) {
  size_t i = 0;
  for (; i + 64 <= n; i += 64) {
    __m128i a = _mm_loadu_si128((const __m128i*)(src + i));
    __m128i b = _mm_loadu_si128((const __m128i*)(src + i + 16));
    __m128i c = _mm_loadu_si128((const __m128i*)(src + i + 32));
    __m128i d = _mm_loadu_si128((const __m128i*)(src + i + 48));
    _mm_stream_si128((__m128i*)(dst + i), a);
    _mm_stream_si128((__m128i*)(dst + i + 16), b);
    _mm_stream_si128((__m128i*)(dst + i + 32), c);
    _mm_stream_si128((__m128i*)(dst + i + 48), d);
  }
  std::memcpy(dst + i, src + i, n - i);
  _mm_sfence();
}

static void flush(char* p, size_t n) {
  for (size_t i = 0; i < n; i += 64) _mm_clflushopt(p + i);
  _mm_sfence();
}

int main() {
  char *h, *d;
  cudaHostAlloc((void**)&h, N, 0);
  cudaMalloc((void**)&d, N);
  std::vector<char> src(N, 1), store(N, 2);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto dma = [&](bool d2h) {
    cudaEventRecord(e0, st);
    cudaMemcpyAsync(d2h ? (void*)h : (void*)d, d2h ? (void*)d : (void*)h, N,
                    d2h ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
  };
  struct Case {
    const char* name;
    std::function<void()> pre;
  };
  std::vector<Case> cases = {
      {"idle", [] {}},
      {"16 thr memcpy into staging", [&] { par([&](size_t a, size_t b) { std::memcpy(h + a, src.data() + a, b - a); }); }},
      {"16 thr NT copy into staging", [&] { par([&](size_t a, size_t b) { nt_copy(h + a, src.data() + a, b - a); }); }},
      {"16 thr memcpy + clflushopt", [&] {
         par([&](size_t a, size_t b) {
           std::memcpy(h + a, src.data() + a, b - a);
           flush(h + a, b - a);
         });
       }},
      {"16 thr read staging (memcpy out)", [&] { par([&](size_t a, size_t b) { std::memcpy(store.data() + a, h + a, b - a); }); }},
      {"16 thr read staging, NT store out", [&] { par([&](size_t a, size_t b) { nt_copy(store.data() + a, h + a, b - a); }); }},
      {"16 thr read + clflushopt staging", [&] {
         par([&](size_t a, size_t b) {
           std::memcpy(store.data() + a, h + a, b - a);
           flush(h + a, b - a);
         });
       }},
      {"16 thr NT out + clflushopt staging", [&] {
         par([&](size_t a, size_t b) {
           nt_copy(store.data() + a, h + a, b - a);
           flush(h + a, b - a);
         });
       }},
  };
  for (auto& c : cases) {
    for (int dir = 0; dir < 2; ++dir) {
      std::printf("%-36s %s:", c.name, dir ? "d2h" : "h2d");
      for (int r = 0; r < 5; ++r) {
        c.pre();
        std::printf(" %.3f", dma(dir == 1));
      }
      std::printf("\n");
    }
  }
  // cost of the host-side variants themselves
  auto wall = [](const std::function<void()>& f) {
    auto t0 = std::chrono::steady_clock::now();
    f();
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  };
  for (size_t k = 2; k < cases.size(); ++k) {
    double best = 1e9;
    for (int r = 0; r < 5; ++r) best = std::min(best, wall(cases[k].pre));
    std::printf("host cost %-36s %.3f ms\n", cases[k].name, best);
  }
  return 0;
}
