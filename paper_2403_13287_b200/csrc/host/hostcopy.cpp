// hostcopy.cpp — host side of the pinned staging buffers.
//
// A DMA into or out of pinned staging runs 3-5x below the PCIe rate when the
// staging lines sit in the host's CPU caches, i.e. after the (multi-threaded)
// stores that fill it or the reads that drain it (measured on the B200 box:
// 27 MB in 2.2 ms instead of 0.48 ms; scripts/dma_probe.cu).  Staging is
// therefore filled with streaming stores, which bypass the caches, and its
// lines are flushed after the host has read them.
#include <algorithm>
#include <cstdint>
#include <cstring>

#include "core.hpp"

#if defined(__x86_64__)
#include <cpuid.h>
#include <immintrin.h>
#endif

namespace lskb {

#if defined(__x86_64__)
namespace {

bool has_clflushopt() {
  static const bool on = [] {
    unsigned a = 0, b = 0, c = 0, d = 0;
    if (!__get_cpuid_count(7, 0, &a, &b, &c, &d)) return false;
    return ((b >> 23) & 1u) != 0;
  }();
  return on;
}

__attribute__((target("clflushopt"))) void flush_opt(const char* p, const char* e) {
  for (; p < e; p += 64) _mm_clflushopt(const_cast<char*>(p));
}

}  // namespace

void flush_lines(const void* p, std::size_t bytes) {
  if (!bytes) return;
  const char* b = reinterpret_cast<const char*>(reinterpret_cast<std::uintptr_t>(p) & ~std::uintptr_t{63});
  const char* e = static_cast<const char*>(p) + bytes;
  if (has_clflushopt()) {
    flush_opt(b, e);
  } else {
    for (; b < e; b += 64) _mm_clflush(b);
  }
  _mm_sfence();
}

void stream_copy(void* dst, const void* src, std::size_t bytes) {
  char* d = static_cast<char*>(dst);
  const char* s = static_cast<const char*>(src);
  const std::size_t head = std::min<std::size_t>(bytes, (16 - (reinterpret_cast<std::uintptr_t>(d) & 15)) & 15);
  if (head) {
    std::memcpy(d, s, head);
    flush_lines(d, head);
    d += head, s += head, bytes -= head;
  }
  std::size_t i = 0;
  for (; i + 64 <= bytes; i += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 32));
    const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + i), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 48), e);
  }
  for (; i + 16 <= bytes; i += 16)
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + i), _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i)));
  if (i < bytes) {
    std::memcpy(d + i, s + i, bytes - i);
    flush_lines(d + i, bytes - i);
  }
  _mm_sfence();
}

void stream_pairs(double* dst, const double* a, const double* b, std::size_t n) {
  if (reinterpret_cast<std::uintptr_t>(dst) & 15) {
    for (std::size_t i = 0; i < n; ++i) dst[2 * i] = a[i], dst[2 * i + 1] = b[i];
    flush_lines(dst, 2 * n * sizeof(double));
    return;
  }
  for (std::size_t i = 0; i < n; ++i) _mm_stream_pd(dst + 2 * i, _mm_set_pd(b[i], a[i]));
  _mm_sfence();
}

#else

void flush_lines(const void*, std::size_t) {}
void stream_copy(void* dst, const void* src, std::size_t bytes) { std::memcpy(dst, src, bytes); }
void stream_pairs(double* dst, const double* a, const double* b, std::size_t n) {
  for (std::size_t i = 0; i < n; ++i) dst[2 * i] = a[i], dst[2 * i + 1] = b[i];
}

#endif

}  // namespace lskb
