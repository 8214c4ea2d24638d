// par.hpp — minimal fork/join helper for host-side setup work (kNN, stencil
// screening, staging, copy-back).  Results never depend on the thread count:
// every index is processed by exactly one thread with no cross-index reduction.
//
// The workers are created once per process and parked on a condition
// variable; a call hands them its slices and works on slices itself, so a
// call costs a wake-up, not host_threads() thread creations (which dominated
// lskum_run's staging and copy-back at ~160K points).  A call made while the
// pool is busy (a nested call, or a second host thread) runs its slices
// serially on the calling thread.
#pragma once

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <thread>
#include <vector>

namespace lskb {

// Host threads for setup work: all hardware threads (at most 64), or
// LSKUM_HOST_THREADS (one process per GPU shares the host between ranks).
inline int host_threads() {
  static const int n = [] {
    const char* e = std::getenv("LSKUM_HOST_THREADS");
    const int v = e ? std::atoi(e) : 0;
    if (v > 0) return std::clamp(v, 1, 64);
    const unsigned hw = std::thread::hardware_concurrency();
    return static_cast<int>(std::clamp<unsigned>(hw == 0 ? 1 : hw, 1, 64));
  }();
  return n;
}

class WorkPool {
 public:
  // Process-wide pool, never destroyed (workers stay parked until exit).
  static WorkPool& get() {
    static WorkPool* p = new WorkPool(host_threads() - 1);
    return *p;
  }
  int workers() const { return static_cast<int>(threads_.size()); }

  // Runs task(k) for every k in [0, tasks) on the workers and the caller.
  // Returns false without running anything when the pool is already busy.
  template <class Task>
  bool run(int tasks, Task& task) {
    std::unique_lock<std::mutex> busy(busy_, std::try_to_lock);
    if (!busy.owns_lock()) return false;
    Job job;
    job.ctx = &task;
    job.call = [](void* c, int k) { (*static_cast<Task*>(c))(k); };
    job.tasks = tasks;
    {
      std::lock_guard<std::mutex> lk(m_);
      job_ = &job;
      ++gen_;
    }
    cv_.notify_all();
    drain(job);
    while (job.done.load(std::memory_order_acquire) < tasks) std::this_thread::yield();
    {
      std::lock_guard<std::mutex> lk(m_);
      job_ = nullptr;  // late-waking workers find nothing to take
    }
    while (active_.load(std::memory_order_acquire) > 0) std::this_thread::yield();
    return true;
  }

 private:
  struct Job {
    void* ctx = nullptr;
    void (*call)(void*, int) = nullptr;
    int tasks = 0;
    std::atomic<int> next{0}, done{0};
  };

  explicit WorkPool(int n) {
    for (int k = 0; k < n; ++k) {
      threads_.emplace_back([this] { loop(); });
      threads_.back().detach();
    }
  }
  static void drain(Job& j) {
    for (;;) {
      const int k = j.next.fetch_add(1, std::memory_order_relaxed);
      if (k >= j.tasks) return;
      j.call(j.ctx, k);
      j.done.fetch_add(1, std::memory_order_release);
    }
  }
  void loop() {
    std::uint64_t seen = 0;
    for (;;) {
      Job* j = nullptr;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        j = job_;
        if (!j) continue;
        active_.fetch_add(1, std::memory_order_relaxed);
      }
      drain(*j);
      active_.fetch_sub(1, std::memory_order_release);
    }
  }

  std::mutex busy_, m_;
  std::condition_variable cv_;
  std::uint64_t gen_ = 0;
  Job* job_ = nullptr;
  std::atomic<int> active_{0};
  std::vector<std::thread> threads_;
};

// Calls fn(k) for k in [0, tasks) on the pool.
template <class Fn>
void parallel_tasks(int tasks, Fn&& fn) {
  if (tasks <= 1) {
    if (tasks == 1) fn(0);
    return;
  }
  auto task = [&](int k) { fn(k); };
  if (!WorkPool::get().run(tasks, task))
    for (int k = 0; k < tasks; ++k) fn(k);
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
  auto slice = [&](int k) { fn(n * k / t, n * (k + 1) / t); };
  if (!WorkPool::get().run(t, slice))
    for (int k = 0; k < t; ++k) slice(k);
}

}  // namespace lskb
