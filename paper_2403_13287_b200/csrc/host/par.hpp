// par.hpp — minimal fork/join helper for host-side setup work (kNN, stencil
// screening, staging).  Results never depend on the thread count: every
// index is processed by exactly one thread with no cross-index reduction.
#pragma once

#include <algorithm>
#include <cstdint>
#include <thread>
#include <vector>

namespace lskb {

inline int host_threads() {
  const unsigned hw = std::thread::hardware_concurrency();
  return static_cast<int>(std::clamp<unsigned>(hw == 0 ? 1 : hw, 1, 64));
}

// Calls fn(lo, hi) over contiguous slices of [0, n).
template <class Fn>
void parallel_slices(std::int64_t n, Fn&& fn, std::int64_t min_per_thread = 4096) {
  const int t = static_cast<int>(std::min<std::int64_t>(host_threads(),
                                                        std::max<std::int64_t>(1, n / min_per_thread)));
  if (t <= 1) {
    fn(std::int64_t{0}, n);
    return;
  }
  std::vector<std::thread> pool;
  pool.reserve(t);
  for (int k = 0; k < t; ++k) {
    const std::int64_t lo = n * k / t, hi = n * (k + 1) / t;
    pool.emplace_back([&fn, lo, hi] { fn(lo, hi); });
  }
  for (auto& th : pool) th.join();
}

}  // namespace lskb
