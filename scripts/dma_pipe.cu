// Chunked D2H through pinned staging + host copy-out into a pageable store:
// wall time of the whole pipeline for several chunk counts / copy-out styles.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -Xcompiler -mclflushopt -o /tmp/dma_pipe scripts/dma_pipe.cu -lpthread
#include <cuda_runtime.h>
#include <immintrin.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static const size_t N = 21ull * 160160 * 8;

static void nt_copy(char* dst, const char* src, size_t n) {
  size_t i = 0;
  for (; i + 64 <= n; i += 64) {
    __m128i a = _mm_load_si128((const __m128i*)(src + i));
    __m128i b = _mm_load_si128((const __m128i*)(src + i + 16));
    __m128i c = _mm_load_si128((const __m128i*)(src + i + 32));
    __m128i d = _mm_load_si128((const __m128i*)(src + i + 48));
    _mm_stream_si128((__m128i*)(dst + i), a);
    _mm_stream_si128((__m128i*)(dst + i + 16), b);
    _mm_stream_si128((__m128i*)(dst + i + 32), c);
    _mm_stream_si128((__m128i*)(dst + i + 48), d);
  }
  std::memcpy(dst + i, src + i, n - i);
  _mm_sfence();
}
// streaming (MOVNTDQA) loads from write-combined memory, NT stores out
__attribute__((target("sse4.1"))) static void nt_load_copy(char* dst, const char* src, size_t n) {
  size_t i = 0;
  for (; i + 64 <= n; i += 64) {
    __m128i a = _mm_stream_load_si128((__m128i*)(src + i));
    __m128i b = _mm_stream_load_si128((__m128i*)(src + i + 16));
    __m128i c = _mm_stream_load_si128((__m128i*)(src + i + 32));
    __m128i d = _mm_stream_load_si128((__m128i*)(src + i + 48));
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
  char *h, *d, *hwc;
  cudaHostAlloc((void**)&h, N, 0);
  cudaHostAlloc((void**)&hwc, N, cudaHostAllocWriteCombined);
  cudaMalloc((void**)&d, N);
  cudaMemset(d, 1, N);
  char* store = (char*)aligned_alloc(64, N);
  memset(store, 0, N);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const int T = 16;
  for (int mode = 0; mode < 6; ++mode) {
    char* hb = mode >= 4 ? hwc : h;
    for (int chunks : {1, 4, 8, 16, 32, 64}) {
      double best = 1e9, sum = 0;
      for (int rep = 0; rep < 7; ++rep) {
        std::vector<cudaEvent_t> ev(chunks);
        cudaDeviceSynchronize();
        auto t0 = std::chrono::steady_clock::now();
        for (int c = 0; c < chunks; ++c) {
          size_t lo = (N * c / chunks) & ~size_t(63), hi = c == chunks - 1 ? N : (N * (c + 1) / chunks) & ~size_t(63);
          cudaEventCreateWithFlags(&ev[c], cudaEventDisableTiming);
          cudaMemcpyAsync(hb + lo, d + lo, hi - lo, cudaMemcpyDeviceToHost, st);
          cudaEventRecord(ev[c], st);
        }
        std::atomic<int> next{0};
        auto work = [&] {
          for (;;) {
            int c = next.fetch_add(1);
            if (c >= chunks) return;
            size_t lo = (N * c / chunks) & ~size_t(63), hi = c == chunks - 1 ? N : (N * (c + 1) / chunks) & ~size_t(63);
            cudaEventSynchronize(ev[c]);
            if (mode == 0 || mode == 1) std::memcpy(store + lo, h + lo, hi - lo);
            else if (mode == 2 || mode == 3) nt_copy(store + lo, h + lo, hi - lo);
            else if (mode == 4) nt_load_copy(store + lo, hwc + lo, hi - lo);
            else std::memcpy(store + lo, hwc + lo, hi - lo);
            if (mode == 1 || mode == 3) flush(h + lo, hi - lo);
          }
        };
        std::vector<std::thread> th;
        for (int k = 0; k < std::min(T, chunks) - 1; ++k) th.emplace_back(work);
        work();
        for (auto& t : th) t.join();
        double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        for (auto e : ev) cudaEventDestroy(e);
        if (rep >= 2) { best = std::min(best, ms); sum += ms; }
      }
      const char* names[] = {"memcpy", "memcpy+flush", "NT", "NT+flush", "WC+ntload", "WC+memcpy"};
      std::printf("%-13s chunks %2d: best %.3f ms  mean %.3f ms\n", names[mode], chunks, best, sum / 5);
    }
  }
}
