// engine.cu — device engine: memory, streams, CUDA graphs and kernel launches
// for the LSKUM fixed-point iteration on sm_100a.
//
// Replaces the reference's L3 runtime (/root/reference/proj/src/core/
// runtime.cpp:84-275): the WorkerPool fork/join per phase becomes stream
// order inside a captured CUDA graph of `chunk` iterations; the per-phase
// exceptions become a device error word (min-reduced key, see kernels.cuh)
// that the host polls asynchronously; per-phase wall timers become
// globaltimer-stamped device durations.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../engine.hpp"
#include "kernels.cuh"
#include "tiles.cuh"
#include "../host/par.hpp"

namespace lskb {

namespace {

using namespace lskd;

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    raise(Status::argument, std::string("CUDA failure in ") + what + ": " + cudaGetErrorString(e));
  }
}

// LSKUM_GRAPHS=0: iterations launched kernel by kernel instead of as
// captured CUDA graphs (single-domain runs).
bool graphs_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("LSKUM_GRAPHS");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

bool graph_upload() {
  static const bool on = [] {
    const char* e = std::getenv("LSKUM_GRAPH_UPLOAD");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

// LSKUM_TRACE only: waits for the stream so the trace line times its work.
// (LSKUM_TRACE_NOSYNC=1: host timestamps only, the pipeline left as it runs)
void trace_sync(cudaStream_t st, const char* what) {
  if (!tracing()) return;
  static const bool nosync = [] {
    const char* e = std::getenv("LSKUM_TRACE_NOSYNC");
    return e && std::atoi(e) == 1;
  }();
  if (!nosync) cudaStreamSynchronize(st);
  trace(what);
}

// Device buffers come from the device's stream-ordered memory pool
// (cudaMallocAsync), whose release threshold is raised once per device so
// memory freed by one run is reused by the next without driver round trips.
void ensure_pool(int device) {
  static bool done[64] = {};
  if (done[device & 63]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    unsigned long long keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  cudaGetLastError();
  done[device & 63] = true;
}

template <class T>
class DBuf {
 public:
  DBuf() = default;
  explicit DBuf(std::size_t count, cudaStream_t st = nullptr) { alloc(count, st); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void alloc(std::size_t count, cudaStream_t st = nullptr) {
    release();
    st_ = st;
    n_ = count;
    if (!count) return;
    if (st) ck(cudaMallocAsync(reinterpret_cast<void**>(&p_), count * sizeof(T), st), "cudaMallocAsync");
    else ck(cudaMalloc(reinterpret_cast<void**>(&p_), count * sizeof(T)), "cudaMalloc");
  }
  T* get() const { return p_; }
  std::size_t size() const { return n_; }

 private:
  void release() {
    if (!p_) return;
    if (st_) cudaFreeAsync(p_, st_);
    else cudaFree(p_);
    p_ = nullptr;
  }
  T* p_ = nullptr;
  std::size_t n_ = 0;
  cudaStream_t st_ = nullptr;
};

// Grow-only device scratch per device and slot for the large transient buffers
// of a run (the copy-back's packed store, the screening's keys and sort
// space), shared by the process's domains and allocated with plain cudaMalloc:
// measured at 40M points, taking a 6.7 GB buffer from the stream-ordered pool
// on a fresh domain's stream stalled a cold lskum_run by 5-550 ms (pool
// growth), while the pool-backed per-domain buffers of the same sizes did not.
// A lease holds the slot until the holder's stream work on it is synchronised.
enum : int { kScratchPack = 0, kScratchScreen = 1, kScratchSlots = 2 };
class ScratchLease {
 public:
  ScratchLease(int device, int slot, std::size_t bytes) : e_(entry(device, slot)), lk_(e_.m) {
    if (e_.bytes < bytes) {
      int prev = 0;
      ck(cudaGetDevice(&prev), "cudaGetDevice");
      ck(cudaSetDevice(device), "cudaSetDevice");  // the slot's device, whatever is current
      if (e_.p) ck(cudaFree(e_.p), "cudaFree(scratch)");
      e_.p = nullptr;
      e_.bytes = 0;
      ck(cudaMalloc(&e_.p, bytes), "cudaMalloc(scratch)");
      e_.bytes = bytes;
      ck(cudaSetDevice(prev), "cudaSetDevice");
    }
  }
  ScratchLease(const ScratchLease&) = delete;
  ScratchLease& operator=(const ScratchLease&) = delete;
  char* get() const { return static_cast<char*>(e_.p); }

 private:
  struct Entry {
    std::mutex m;
    void* p = nullptr;
    std::size_t bytes = 0;
  };
  static Entry& entry(int device, int slot) {
    static Entry tab[64][kScratchSlots];
    return tab[device & 63][slot];
  }
  Entry& e_;
  std::unique_lock<std::mutex> lk_;
};

// Small pinned host blocks (control words, poll slots) are recycled through a
// process-wide free list: cudaHostAlloc costs about a millisecond per call,
// which a fresh domain would otherwise pay several times.
class PinnedPool {
 public:
  static constexpr std::size_t kBlock = 4096;
  static void* take() {
    {
      std::lock_guard<std::mutex> g(mu());
      auto& f = free_list();
      if (!f.empty()) {
        void* p = f.back();
        f.pop_back();
        return p;
      }
    }
    void* p = nullptr;
    ck(cudaHostAlloc(&p, kBlock, 0), "cudaHostAlloc");
    return p;
  }
  static void give(void* p) {
    std::lock_guard<std::mutex> g(mu());
    free_list().push_back(p);
  }

 private:
  static std::mutex& mu() {
    static std::mutex m;
    return m;
  }
  static std::vector<void*>& free_list() {
    static std::vector<void*> f;
    return f;
  }
};

template <class T>
class HBuf {  // pinned host staging
 public:
  HBuf() = default;
  HBuf(const HBuf&) = delete;
  HBuf& operator=(const HBuf&) = delete;
  ~HBuf() { release(); }
  void alloc(std::size_t count) {
    release();
    if (!count) return;
    if (count * sizeof(T) <= PinnedPool::kBlock) {
      p_ = static_cast<T*>(PinnedPool::take());
      pooled_ = true;
    } else {
      ck(cudaHostAlloc(reinterpret_cast<void**>(&p_), count * sizeof(T), 0), "cudaHostAlloc");
    }
  }
  T* get() const { return p_; }

 private:
  void release() {
    if (!p_) return;
    if (pooled_) PinnedPool::give(p_);
    else cudaFreeHost(p_);
    p_ = nullptr;
    pooled_ = false;
  }
  T* p_ = nullptr;
  bool pooled_ = false;
};

// Grow-only pinned host staging, one per host thread (runs on different
// clouds may proceed concurrently from different threads).
class Staging {
 public:
  ~Staging() {
    if (p_) cudaFreeHost(p_);
  }
  void* get(std::size_t bytes) {
    if (bytes > cap_) {
      if (p_) cudaFreeHost(p_);
      p_ = nullptr;
      cap_ = 0;
      ck(cudaHostAlloc(&p_, bytes, 0), "cudaHostAlloc(staging)");
      cap_ = bytes;
    }
    return p_;
  }

 private:
  void* p_ = nullptr;
  std::size_t cap_ = 0;
};
thread_local Staging t_staging;

// Pinned host memory for large field stores (StoreBuffer) and large cloud
// arrays (HostAlloc, host/core.hpp): the copy-back DMAs straight into the
// cloud's store and the geometry upload straight from its arrays.  Freed
// blocks are kept for the next store / cloud of the same sizes (a cloud handle
// per run, as lskum_run users and the bench create them, then costs no page
// pinning).
class StorePool {
 public:
  static void* alloc(std::size_t bytes) {
    {
      std::lock_guard<std::mutex> g(mu());
      auto& f = free_blocks();
      for (auto it = f.begin(); it != f.end(); ++it)
        if (it->second == bytes) {
          void* p = it->first;
          f.erase(it);
          return p;
        }
    }
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
      cudaGetLastError();
      return nullptr;
    }
    void* p = nullptr;
    if (cudaHostAlloc(&p, bytes, cudaHostAllocPortable) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    return p;
  }
  // Freed blocks stay cached (most recent last) up to kKeepBytes, so the next
  // cloud / store of the same sizes reuses them instead of pinning anew
  // (cudaHostAlloc runs at ~1-2 GB/s); the oldest go back to the system.
  static constexpr std::size_t kKeepBytes = std::size_t{24} << 30;
  static void release(void* p, std::size_t bytes) {
    std::lock_guard<std::mutex> g(mu());
    auto& f = free_blocks();
    f.emplace_back(p, bytes);
    std::size_t total = 0;
    for (const auto& b : f) total += b.second;
    while (total > kKeepBytes && f.size() > 1) {
      total -= f.front().second;
      cudaFreeHost(f.front().first);
      f.erase(f.begin());
    }
  }

 private:
  static std::mutex& mu() {
    static std::mutex m;
    return m;
  }
  static std::vector<std::pair<void*, std::size_t>>& free_blocks() {
    static std::vector<std::pair<void*, std::size_t>> f;
    return f;
  }
};
const bool g_store_hooks = [] {
  store_hooks().alloc = &StorePool::alloc;
  store_hooks().release = &StorePool::release;
  return true;
}();

// Launch with programmatic stream serialisation (LSKUM_PDL=0: plain launches):
// inside a captured iteration the next kernel's launch overlaps this one's
// tail; every such kernel starts with pdl_enter() (kernels.cuh).  Measured on
// B200 at 160K points: 97.7 -> 96.1 us per order-2 iteration, 46.1 -> 44.4 us
// per order-1 iteration.
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("LSKUM_PDL");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

template <class... KArgs, class... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, std::size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  ck(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...), "cudaLaunchKernelEx");
}

int flux_width(int kmax) { return kmax <= 8 ? 8 : (kmax <= 16 ? 16 : 32); }

std::size_t flux_smem_bytes(int W, int kcap) {
  const int P = flux_points_per_block(W);
  return (static_cast<std::size_t>(P) * flux_stride(kcap) + static_cast<std::size_t>(P) * 16) * sizeof(double);
}

template <int W, bool S, int MB>
void flux_launch_t(const FluxArgs& a, std::size_t smem, cudaStream_t st) {
  static std::size_t configured[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (smem > configured[dev & 63]) {
    ck(cudaFuncSetAttribute(k_flux<W, S, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(smem)),
       "cudaFuncSetAttribute(k_flux)");
    configured[dev & 63] = smem;
  }
  const int P = flux_points_per_block(W);
  static int resident[64] = {};
  if (!resident[dev & 63]) {
    int per_sm = 0, sms = 0;
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_flux<W, S, MB>, W * P, smem), "occupancy");
    ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "attr");
    resident[dev & 63] = std::max(1, per_sm) * sms;
  }
  const int groups = (a.g.n + P - 1) / P;
  launch_pdl(k_flux<W, S, MB>, std::max(1, std::min(groups, resident[dev & 63])), W * P, smem, st, a);
}

// Derivative sweep launch: strict (bitwise) or FMA variant, resident blocks per
// SM from LSKUM_SWEEP_MINB (2 | 3 | 4, default 3), persistent grid.
// Default: 2 for the unrolled 8-point kernel (128 registers keep all eight
// gathers in flight), 3 for the generic loop.
int sweep_min_blocks(bool unrolled) {
  static int mb = [] {
    const char* e = std::getenv("LSKUM_SWEEP_MINB");
    const int v = e ? std::atoi(e) : 0;
    return (v >= 2 && v <= 4) ? v : 0;
  }();
  return mb ? mb : (unrolled ? 2 : 3);
}

// Sweep variant: LSKUM_SWEEP_LANES = 2 (default, k_sweep2) | 1 (k_sweep).
int sweep_lanes() {
  static int v = [] {
    const char* e = std::getenv("LSKUM_SWEEP_LANES");
    return (e && std::atoi(e) == 1) ? 1 : 2;
  }();
  return v;
}

// Unrolled sweep for uniform 8-point stencils (LSKUM_SWEEP_UNROLL=0 disables).
bool sweep_unrolled() {
  static int v = [] {
    const char* e = std::getenv("LSKUM_SWEEP_UNROLL");
    return (e && std::atoi(e) == 0) ? 0 : 1;
  }();
  return v != 0;
}

template <class K>
int resident_blocks(K kern, int slot) {
  static int resident[8][64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int& r = resident[slot & 7][dev & 63];
  if (!r) {
    int per_sm = 0, sms = 0;
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0), "occupancy");
    ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "attr");
    r = std::max(1, per_sm) * sms;
  }
  return r;
}

// The unrolled 8-point sweep in blocks of NT threads (MB resident per SM).
template <bool S, int MB, int NT>
void sweep8_launch(const Geo& g, const D4* q, const D4* dq_in, D4* dq_out, const Gas& gas, Ctl* ctl,
                   unsigned long long* it0, int sweep, cudaStream_t st) {
  static int resident[64] = {};  // per instantiation and device
  int dev = 0;
  cudaGetDevice(&dev);
  if (!resident[dev & 63]) {
    int per_sm = 0, sms = 0;
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sweep2<S, MB, 8, NT>, NT, 0), "occupancy");
    ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "attr");
    resident[dev & 63] = std::max(1, per_sm) * sms;
  }
  const int npts = g.list ? g.nlist : g.n;
  const int grid = std::max(1, std::min((2 * npts + NT - 1) / NT, resident[dev & 63]));
  launch_pdl(k_sweep2<S, MB, 8, NT>, grid, NT, 0, st, g, q, dq_in, dq_out, gas, ctl, it0, sweep);
}

// 128-thread blocks for the unrolled sweep (default; LSKUM_SWEEP_BLOCK=256:
// 256-thread blocks, 0.5% slower at 160K and 10M points).
bool sweep_small_blocks() {
  static const bool on = [] {
    const char* e = std::getenv("LSKUM_SWEEP_BLOCK");
    return !(e && std::atoi(e) == 256);
  }();
  return on;
}

template <bool S, int MB>
void sweep_launch_t(const Geo& g, const D4* q, const D4* dq_in, D4* dq_out, const Gas& gas, Ctl* ctl,
                    unsigned long long* it0, int sweep, cudaStream_t st) {
  const int slot = (S ? 4 : 0) + MB - 2;
  if (sweep_lanes() == 2 && g.kfix == 8 && sweep_unrolled()) {
    if (sweep_small_blocks()) sweep8_launch<S, 2 * MB, 128>(g, q, dq_in, dq_out, gas, ctl, it0, sweep, st);
    else sweep8_launch<S, MB, 256>(g, q, dq_in, dq_out, gas, ctl, it0, sweep, st);
  } else if (sweep_lanes() == 2) {
    const int npts = g.list ? g.nlist : g.n;
    const int grid = std::max(1, std::min((2 * npts + 255) / 256, resident_blocks(k_sweep2<S, MB>, slot)));
    launch_pdl(k_sweep2<S, MB, 0>, grid, 256, 0, st, g, q, dq_in, dq_out, gas, ctl, it0, sweep);
  } else {
    const int grid = std::max(1, std::min((g.n + 255) / 256, resident_blocks(k_sweep<S, MB>, slot)));
    launch_pdl(k_sweep<S, MB>, grid, 256, 0, st, g, q, dq_in, dq_out, gas, ctl, it0, sweep);
  }
}

void sweep_launch(bool strict, const Geo& g, const D4* q, const D4* dq_in, D4* dq_out, const Gas& gas, Ctl* ctl,
                  unsigned long long* it0, int sweep, cudaStream_t st) {
  const int mb = sweep_min_blocks(sweep_lanes() == 2 && g.kfix == 8 && sweep_unrolled());
  if (strict) {
    if (mb == 2) sweep_launch_t<true, 2>(g, q, dq_in, dq_out, gas, ctl, it0, sweep, st);
    else if (mb == 4) sweep_launch_t<true, 4>(g, q, dq_in, dq_out, gas, ctl, it0, sweep, st);
    else sweep_launch_t<true, 3>(g, q, dq_in, dq_out, gas, ctl, it0, sweep, st);
  } else {
    if (mb == 2) sweep_launch_t<false, 2>(g, q, dq_in, dq_out, gas, ctl, it0, sweep, st);
    else if (mb == 4) sweep_launch_t<false, 4>(g, q, dq_in, dq_out, gas, ctl, it0, sweep, st);
    else sweep_launch_t<false, 3>(g, q, dq_in, dq_out, gas, ctl, it0, sweep, st);
  }
}

// LSKUM_ZERO_COPY=1: the copy-back writes a pinned store directly from the
// pack kernel (no 21-slot device pack buffer: 6.7 GB at 40M points) instead of
// packing on the device and copying in chunks.  Off by default: the copy
// engines are faster (40M: 127 ms zero copy vs 119 ms packed + DMA).
bool zero_copy_store() {
  static int v = [] {
    const char* e = std::getenv("LSKUM_ZERO_COPY");
    return (e && std::atoi(e) == 1) ? 1 : 0;
  }();
  return v != 0;
}

// Tiled sweep (tiles.cuh) for uniform 8-point stencils.  LSKUM_SWEEP_TILE
// selects the tile shape: 128 (default) = tiles of 128 points, 256-thread
// blocks, 2 resident per SM, each with 2 stages of up to 480 staged points
// (2 x 55.9 KB); 64 = tiles of 64 points, 128-thread blocks, 4 per SM, 2
// stages of up to 216 points (2 x 25.3 KB); 0 = untiled sweep.  A ring
// cloud's tile stages ~3 x (TP + 4) points (its row and the rows above and below).
template <int TP>
struct TileShape;
template <>
struct TileShape<128> {
  static constexpr int MB = 2, smax = 480;
};
template <>
struct TileShape<64> {
  static constexpr int MB = 4, smax = 216;
};
int sweep_tile_p() {
  static int v = [] {
    const char* e = std::getenv("LSKUM_SWEEP_TILE");
    if (!e) return 128;
    const int t = std::atoi(e);
    return t == 0 ? 0 : (t == 64 ? 64 : 128);
  }();
  return v;
}

template <bool S, int TP, bool LIST>
void sweep_tile_launch_t(const Geo& g, const D4* q, const D4* dq_in, D4* dq_out, const Gas& gas, Ctl* ctl, int sweep,
                         const TilePlan* plan, const std::uint16_t* slot, int ntiles, const int* tlist,
                         cudaStream_t st) {
  constexpr int MB = TileShape<TP>::MB, smax = TileShape<TP>::smax;
  constexpr std::size_t smem = 2 * tile_stage_bytes(TP, smax);
  auto kern = k_sweep_tile<S, TP, MB, LIST>;
  static int resident[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!resident[dev & 63]) {
    ck(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
       "cudaFuncSetAttribute(k_sweep_tile)");
    int per_sm = 0, sms = 0;
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 2 * TP, smem), "occupancy");
    ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "attr");
    resident[dev & 63] = std::max(1, per_sm) * sms;
  }
  const int grid = std::max(1, std::min(ntiles, resident[dev & 63]));
  launch_pdl(kern, grid, 2 * TP, smem, st, g, q, dq_in, dq_out, gas, ctl, sweep, plan, slot, smax, ntiles, tlist);
}

template <bool S>
void sweep_tile_launch(int tp, const Geo& g, const D4* q, const D4* dq_in, D4* dq_out, const Gas& gas, Ctl* ctl,
                       int sweep, const TilePlan* plan, const std::uint16_t* slot, int ntiles, const int* tlist,
                       cudaStream_t st) {
  if (tp == 64) {
    if (tlist) sweep_tile_launch_t<S, 64, true>(g, q, dq_in, dq_out, gas, ctl, sweep, plan, slot, ntiles, tlist, st);
    else sweep_tile_launch_t<S, 64, false>(g, q, dq_in, dq_out, gas, ctl, sweep, plan, slot, ntiles, tlist, st);
  } else {
    if (tlist) sweep_tile_launch_t<S, 128, true>(g, q, dq_in, dq_out, gas, ctl, sweep, plan, slot, ntiles, tlist, st);
    else sweep_tile_launch_t<S, 128, false>(g, q, dq_in, dq_out, gas, ctl, sweep, plan, slot, ntiles, tlist, st);
  }
}

// Register/occupancy trade-off of the W=8 kernel: minimum resident blocks per
// SM (LSKUM_FLUX_MINB = 2 | 3, default 2: 128 registers, no spills).
int flux_min_blocks() {
  static int mb = [] {
    const char* e = std::getenv("LSKUM_FLUX_MINB");
    const int v = e ? std::atoi(e) : 2;
    return (v >= 2 && v <= 3) ? v : 2;
  }();
  return mb;
}

template <bool S>
void flux_launch_s(int W, const FluxArgs& a, std::size_t smem, cudaStream_t st) {
  if (W == 8) {
    const int mb = flux_min_blocks();
    if (mb == 2) flux_launch_t<8, S, 2>(a, smem, st);
    else flux_launch_t<8, S, 3>(a, smem, st);
  } else if (W == 16) {
    flux_launch_t<16, S, 2>(a, smem, st);
  } else {
    flux_launch_t<32, S, 1>(a, smem, st);
  }
}

void flux_launch(int W, bool strict, const FluxArgs& a, std::size_t smem, cudaStream_t st) {
  if (strict) flux_launch_s<true>(W, a, smem, st);
  else flux_launch_s<false>(W, a, smem, st);
}

// Fast-mode flux: the weighted kernel (LSKUM_FLUX_W=0 selects the per-iteration
// solve kernel k_flux instead).
bool flux_weighted() {
  static int v = [] {
    const char* e = std::getenv("LSKUM_FLUX_W");
    return (e && std::atoi(e) == 0) ? 0 : 1;
  }();
  return v != 0;
}

// Per-rank runs: interior/boundary overlap of the halo exchange
// (LSKUM_RANK_OVERLAP=0 disables).
bool overlap_enabled() {
  static int v = [] {
    const char* e = std::getenv("LSKUM_RANK_OVERLAP");
    return (e && std::atoi(e) == 0) ? 0 : 1;
  }();
  return v != 0;
}

// First order, fast mode: split fluxes evaluated once per point
// (LSKUM_POINT_FLUX=0 disables).
bool point_flux_enabled() {
  static int v = [] {
    const char* e = std::getenv("LSKUM_POINT_FLUX");
    return (e && std::atoi(e) == 0) ? 0 : 1;
  }();
  return v != 0;
}

// Staged variant for stencils of at most 8 (LSKUM_FLUX_STAGE=0 disables it).
bool flux_staged() {
  static int v = [] {
    const char* e = std::getenv("LSKUM_FLUX_STAGE");
    return (e && std::atoi(e) == 0) ? 0 : 1;
  }();
  return v != 0;
}

// Block shape of the staged flux kernel: LSKUM_FLUX_WS = "<warps>x<blocks/SM>"
// (default by size, both 16 warps/SM: 4x4 below 512K owned points — finer
// blocks balance the short 160K-point launch better — and 8x2 above, 0.8-1.6%
// faster from 625K to 10M points; 8x3, 4x5, 6x3 spill and are slower).
int flux_ws_shape(int n) {
  static int v = [] {
    const char* e = std::getenv("LSKUM_FLUX_WS");
    const std::string s = e ? e : "";
    if (s == "8x2") return 82;
    if (s == "8x3") return 83;
    if (s == "4x4") return 44;
    if (s == "4x5") return 45;
    if (s == "6x3") return 63;
    return 0;
  }();
  return v ? v : (n >= (1 << 19) ? 82 : 44);
}

// The staged flux kernel, instantiated for gamma = 1.4 (2/(gamma-1) = 5 at
// compile time: -2.8% flux time at 10M points) and for any gamma.
// Uniform 8-point stencils over all owned points: the k_flux_ws instantiation
// with compile-time stencil offsets (LSKUM_FLUX_U8=0 disables it).
bool flux_u8() {
  static int v = [] {
    const char* e = std::getenv("LSKUM_FLUX_U8");
    return (e && std::atoi(e) == 0) ? 0 : 1;
  }();
  return v != 0;
}

// Rare-path deferral of the staged flux kernel (k_flux_ws<.., DEFER>, then
// k_flux_redo over the points it flagged).  LSKUM_FLUX_DEFER: 1 (default)
// per run from the initial state (Domain::probe_defer), 0 never (fallback
// branches inside the staged kernel), 2 always (tests of the redo path).
int flux_defer_mode() {
  static int v = [] {
    const char* e = std::getenv("LSKUM_FLUX_DEFER");
    const int m = e ? std::atoi(e) : 1;
    return m < 0 || m > 2 ? 1 : m;
  }();
  return v;
}
bool flux_defer() { return flux_defer_mode() != 0; }

template <int MB, int NW, int HP, bool U8, bool DEFER>
void flux_ws_launch_k(const FluxArgs& a, const double2* w1, const double2* w2, const std::uint8_t* sing,
                      const FluxRedo& rd, cudaStream_t st) {
  constexpr std::size_t smem = static_cast<std::size_t>(2 * NW) * kFluxStageBytes;
  auto kern = k_flux_ws<MB, NW, HP, U8, DEFER>;
  static int resident[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!resident[dev & 63]) {
    ck(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
       "cudaFuncSetAttribute(k_flux_ws)");
    int per_sm = 0, sms = 0;
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NW * 32, smem), "occupancy");
    ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "attr");
    resident[dev & 63] = std::max(1, per_sm) * sms;
  }
  const int groups = ((a.g.list ? a.g.nlist : a.g.n) + 3) / 4;
  const int blocks = std::max(1, std::min((groups + NW - 1) / NW, resident[dev & 63]));
  launch_pdl(kern, blocks, NW * 32, smem, st, a, w1, w2, sing, rd);
  if constexpr (DEFER) {
    // one warp step per 4096 points, at most two blocks per SM
    const int steps = (a.g.n + kRedoPointsPer - 1) / kRedoPointsPer;
    static int sms[64] = {};
    if (!sms[dev & 63]) ck(cudaDeviceGetAttribute(&sms[dev & 63], cudaDevAttrMultiProcessorCount, dev), "attr");
    const int rblocks = std::max(1, std::min((steps + 7) / 8, 2 * sms[dev & 63]));
    launch_pdl(k_flux_redo, rblocks, 256, 0, st, a, w1, w2, sing, rd);
  }
}

template <int MB, int NW, int HP, bool U8>
void flux_ws_launch_d(const FluxArgs& a, const double2* w1, const double2* w2, const std::uint8_t* sing,
                      const FluxRedo* rd, cudaStream_t st) {
  if (rd) flux_ws_launch_k<MB, NW, HP, U8, true>(a, w1, w2, sing, *rd, st);
  else flux_ws_launch_k<MB, NW, HP, U8, false>(a, w1, w2, sing, FluxRedo{nullptr}, st);
}

template <int MB, int NW, int HP>
void flux_ws_launch_hp(const FluxArgs& a, const double2* w1, const double2* w2, const std::uint8_t* sing,
                       const FluxRedo* rd, cudaStream_t st) {
  if (a.g.kfix == 8 && !a.g.list && flux_u8()) flux_ws_launch_d<MB, NW, HP, true>(a, w1, w2, sing, rd, st);
  else flux_ws_launch_d<MB, NW, HP, false>(a, w1, w2, sing, rd, st);
}

template <int MB, int NW>
void flux_ws_launch(const FluxArgs& a, const double2* w1, const double2* w2, const std::uint8_t* sing,
                    const FluxRedo* rd, cudaStream_t st) {
  if (a.gas.half_pow == 5) flux_ws_launch_hp<MB, NW, 5>(a, w1, w2, sing, rd, st);
  else flux_ws_launch_hp<MB, NW, -1>(a, w1, w2, sing, rd, st);
}

// rd: the domain's redo list (null: no deferral).
void flux_w_launch(const FluxArgs& a, int kmax, const double2* w1, const double2* w2, const std::uint8_t* sing,
                   const FluxRedo* rd, cudaStream_t st) {
  const int groups = (a.g.n + 3) / 4;
  if (kmax <= 8 && flux_staged()) {
    if (!flux_defer()) rd = nullptr;
    switch (flux_ws_shape(a.g.n)) {
      case 83: flux_ws_launch<3, 8>(a, w1, w2, sing, rd, st); break;
      case 44: flux_ws_launch<4, 4>(a, w1, w2, sing, rd, st); break;
      case 45: flux_ws_launch<5, 4>(a, w1, w2, sing, rd, st); break;
      case 63: flux_ws_launch<3, 6>(a, w1, w2, sing, rd, st); break;
      case 82: flux_ws_launch<2, 8>(a, w1, w2, sing, rd, st); break;
      default: flux_ws_launch<4, 4>(a, w1, w2, sing, rd, st); break;
    }
    return;
  }
  const int blocks = std::max(1, std::min((groups + 7) / 8, resident_blocks(k_flux_w<2>, 7)));
  launch_pdl(k_flux_w<2>, blocks, 256, 0, st, a, w1, w2, sing);
}

// Depth of the per-block nodes of the residue tree: at most ~8 values per
// thread (256 threads per block), at most 8192 blocks (the final block folds
// up to 8 partials per thread, then 10 levels in shared memory).
int tree_depth(long long n) {
  int d = 0;
  while (d < 13 && (n >> (d + 8)) > 8) ++d;
  return d;
}

// ---- diagnostics: re-evaluates the failing item named by the error key ----
template <bool S>
__global__ void k_diagnose(Geo g, const D4* q, const D4* dq, const D4* prim, const double* uval,
                           const double* uwhich, Gas gas, unsigned long long key, int i, double* out) {
  const unsigned phase = key_phase(key);
  const unsigned dir = key_dir(key);
  const unsigned j = key_j(key);
  for (int t = 0; t < 6; ++t) out[t] = 0.0;
  if (phase == PH_RESIDUE) return;
  if (phase == PH_QVAR) {
    out[1] = prim[i].a;
    out[2] = prim[i].d;
    return;
  }
  if (phase == PH_UPDATE) {
    out[1] = uval[i];
    out[0] = uwhich[i];
    return;
  }
  const double2 pi = g.xy[i];
  if (phase == PH_SWEEP || j == kSolveSlot) {
    double sxx = 0.0, sxy = 0.0, syy = 0.0;
    int count = 0;
    for (int e = g.off[i]; e < g.off[i + 1]; ++e) {
      const double2 pn = g.xy[g.nbr[e]];
      const double dx = X::sub(pn.x, pi.x), dy = X::sub(pn.y, pi.y);
      if (phase == PH_FLUX) {
        const double dd = dir < 2 ? dx : dy;
        if (!((dir & 1) ? dd >= 0.0 : dd <= 0.0)) continue;
      }
      sxx = X::add(sxx, X::mul(dx, dx));
      sxy = X::add(sxy, X::mul(dx, dy));
      syy = X::add(syy, X::mul(dy, dy));
      ++count;
    }
    out[0] = 2.0;
    out[1] = X::sub(X::mul(sxx, syy), X::mul(sxy, sxy));
    out[2] = count;
    return;
  }
  const int nb = g.nbr[g.off[i] + j];
  const double2 pn = g.xy[nb];
  const double dx = X::sub(pn.x, pi.x), dy = X::sub(pn.y, pi.y);
  const D4 qi = q[i], qn = q[nb];
  D4 qxi, qyi, qxn, qyn;
  dq_load(dq, g.nloc, i, qxi, qyi);
  dq_load(dq, g.nloc, nb, qxn, qyn);
  double ti[4], tn[4];
  for (int c = 0; c < 4; ++c) {
    ti[c] = corrected<S>(comp(qi, c), comp(qxi, c), comp(qyi, c), dx, dy);
    tn[c] = corrected<S>(comp(qn, c), comp(qxn, c), comp(qyn, c), dx, dy);
  }
  out[3] = gidx(g, nb);
  if (!(ti[3] < 0.0)) {
    out[0] = 0.0;
    out[1] = ti[3];
    return;
  }
  if (!(tn[3] < 0.0)) {
    out[0] = 0.0;
    out[1] = tn[3];
    return;
  }
  double r, u1, u2, p;
  prim_from_q<S>(ti[0], ti[1], ti[2], ti[3], gas.inv_gm1, gas.gm1, r, u1, u2, p);
  out[0] = 1.0;
  if (!(r > 0.0) || !(p > 0.0)) {
    out[1] = r;
    out[2] = p;
    return;
  }
  prim_from_q<S>(tn[0], tn[1], tn[2], tn[3], gas.inv_gm1, gas.gm1, r, u1, u2, p);
  out[1] = r;
  out[2] = p;
}

// Resets this domain's timers, points it at the run's shared word and (for
// the domain that owns it) resets that word.
__global__ void k_ctl_init(Ctl* ctl, Shared* sh, int own_shared, int diag_iter, int spi, int upd_blocks,
                           int split4 = 0) {
  ctl->sh = sh;
  ctl->split4 = split4;
  ctl->diag_iter = diag_iter;
  ctl->spi = spi;
  ctl->upd_blocks = upd_blocks > 0 ? upd_blocks : 1;
  ctl->upd_done = 0;
  ctl->err_stage = kNoErr;
  ctl->err_key = kNoErr;
  if (own_shared) {
    sh->err_stage = kNoErr;
    sh->iter = 0;
  }
  for (int k = 0; k < KT_COUNT; ++k) {
    ctl->kt[k].t0 = ~0ull;
    ctl->kt[k].t1 = 0;
    ctl->kt[k].done = 0;
    ctl->kt[k].total_ns = 0;
    ctl->kt[k].launches = 0;
  }
}

__global__ void k_set_diag(Ctl* ctl, int diag_iter) { ctl->diag_iter = diag_iter; }

// Writes the 21-slot field store in the host FieldBlock's layout (AoS: point
// major; SoA: slot major), so the copy-back is one contiguous D2H transfer.
// Points [lo, hi) of n.
__global__ void k_pack_fields(int n, int lo, int hi, int soa, const D4* prim, const D4* q, const D4* dq,
                              long long dq_ps, const D4* res, const double* dt, const int* gid, double* out) {
  for (int i = lo + blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += gridDim.x * blockDim.x) {
    const int p = gid ? gid[i] : i;  // position in the store
    D4 qx, qy;
    dq_load(dq, dq_ps, i, qx, qy);
    const D4 v[5] = {prim[i], q[i], qx, qy, res[i]};
    double r[21];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      r[4 * k] = v[k].a;
      r[4 * k + 1] = v[k].b;
      r[4 * k + 2] = v[k].c;
      r[4 * k + 3] = v[k].d;
    }
    r[20] = dt[i];
    if (soa) {
#pragma unroll
      for (int k = 0; k < 21; ++k) out[static_cast<size_t>(k) * n + p] = r[k];
    } else {
#pragma unroll
      for (int k = 0; k < 21; ++k) out[static_cast<size_t>(p) * 21 + k] = r[k];
    }
  }
}

// The 21-slot store in the AoS layout written straight into pinned host memory
// (zero copy, no device pack buffer): a block gathers its 256 points' records
// in shared memory, then writes them as one contiguous run of 16-byte stores,
// so the writes reach the host as full PCIe transactions.
constexpr int kPackPts = 256;
__global__ void __launch_bounds__(kPackPts) k_pack_aos_host(int n, const D4* prim, const D4* q, const D4* dq,
                                                            long long dq_ps, const D4* res, const double* dt,
                                                            double* out) {
  __shared__ __align__(16) double tile[kPackPts * 21];
  for (long long p0 = static_cast<long long>(blockIdx.x) * kPackPts; p0 < n;
       p0 += static_cast<long long>(gridDim.x) * kPackPts) {
    const long long i = p0 + threadIdx.x;
    if (i < n) {
      D4 qx, qy;
      dq_load(dq, dq_ps, i, qx, qy);
      const D4 v[5] = {prim[i], q[i], qx, qy, res[i]};
      double* r = tile + threadIdx.x * 21;
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        r[4 * k] = v[k].a;
        r[4 * k + 1] = v[k].b;
        r[4 * k + 2] = v[k].c;
        r[4 * k + 3] = v[k].d;
      }
      r[20] = dt[i];
    }
    __syncthreads();
    const int pts = n - p0 < kPackPts ? static_cast<int>(n - p0) : kPackPts;
    const int chunks = pts * 21 * 8 / 16;  // whole 16-byte chunks
    const double2* src = reinterpret_cast<const double2*>(tile);
    double2* o = reinterpret_cast<double2*>(out + p0 * 21);
    for (int c = threadIdx.x; c < chunks; c += kPackPts) o[c] = src[c];
    if ((pts * 21) & 1) {  // an odd trailing double
      if (threadIdx.x == 0) out[p0 * 21 + pts * 21 - 1] = tile[pts * 21 - 1];
    }
    __syncthreads();
  }
}

// Scatters the primitives (slots 0-3 of a FieldBlock in either layout) into D4 records.
// ---- stencil screening on the device (reference validate_cloud,
// cloud.cpp:252-321; host twin: host/screen.cpp).  Same sums in the same
// order with separately rounded products and sums, so determinants, the
// defective set and the report are bitwise the reference's.
struct ScreenOut {
  unsigned long long n_finite;
  int n_defective, n_wall_isolated, min_size, pad;
};

// Nearest-neighbour distances as sortable keys (non-negative doubles order
// like their bit patterns; non-finite values sort last) + the finite count.
__global__ void k_screen_keys(int n, const double* mind, unsigned long long* keys, ScreenOut* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double d = mind[i];
  keys[i] = static_cast<unsigned long long>(__double_as_longlong(d));
  if (isfinite(d)) atomicAdd(&out->n_finite, 1ull);
}

__global__ void k_screen(Geo g, double tol, ScreenOut* out, int* defective, int cap) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= g.n) return;
  double fxx = 0.0, fxy = 0.0, fyy = 0.0, hxx[4] = {0, 0, 0, 0}, hxy[4] = {0, 0, 0, 0}, hyy[4] = {0, 0, 0, 0};
  int fc = 0, hc[4] = {0, 0, 0, 0}, walls = 0;
  const double2 pp = g.xy[p];
  for (int e = g.off[p]; e < g.off[p + 1]; ++e) {
    const int nb = g.nbr[e];
    const double2 pn = g.xy[nb];
    const double dx = X::sub(pn.x, pp.x), dy = X::sub(pn.y, pp.y);
    const double xx = X::mul(dx, dx), xy = X::mul(dx, dy), yy = X::mul(dy, dy);
    fxx = X::add(fxx, xx);
    fxy = X::add(fxy, xy);
    fyy = X::add(fyy, yy);
    ++fc;
    const bool in[4] = {dx >= 0.0, dx <= 0.0, dy >= 0.0, dy <= 0.0};
#pragma unroll
    for (int h = 0; h < 4; ++h)
      if (in[h]) {
        hxx[h] = X::add(hxx[h], xx);
        hxy[h] = X::add(hxy[h], xy);
        hyy[h] = X::add(hyy[h], yy);
        ++hc[h];
      }
    if (g.kind[nb] == KIND_WALL) ++walls;
  }
  bool bad = X::sub(X::mul(fxx, fyy), X::mul(fxy, fxy)) < tol || fc < 3;
  if (g.kind[p] != KIND_OUTER)
#pragma unroll
    for (int h = 0; h < 4; ++h)
      bad = bad || hc[h] == 0 || X::sub(X::mul(hxx[h], hyy[h]), X::mul(hxy[h], hxy[h])) < tol;
  if (bad) {
    const int slot = atomicAdd(&out->n_defective, 1);
    if (slot < cap) defective[slot] = p;
  }
  if (g.kind[p] == KIND_WALL && walls < 2) atomicAdd(&out->n_wall_isolated, 1);
  atomicMin(&out->min_size, fc);
}

// Derivative planes (plane stride ps) <-> the reference's scratch layout
// [qx0..3, qy0..3] per point: to_records = 1: plain -> planes, 0: planes -> plain.
__global__ void k_dq_layout(const D4* in, D4* out, long long n, long long ps, int to_records) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  if (to_records) {
    dq_store(out, ps, i, ld4(in + 2 * i), ld4(in + 2 * i + 1));
  } else {
    D4 qx, qy;
    dq_load(in, ps, i, qx, qy);
    st4(out + 2 * i, qx);
    st4(out + 2 * i + 1, qy);
  }
}

__global__ void k_fill_d4(D4* out, int n, D4 v) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = v;
}

__global__ void k_unpack_prim(int n, int soa, const double* in, D4* prim) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (soa)
      prim[i] = D4{in[i], in[static_cast<size_t>(n) + i], in[2 * static_cast<size_t>(n) + i],
                   in[3 * static_cast<size_t>(n) + i]};
    else
      prim[i] = D4{in[4 * static_cast<size_t>(i)], in[4 * static_cast<size_t>(i) + 1],
                   in[4 * static_cast<size_t>(i) + 2], in[4 * static_cast<size_t>(i) + 3]};
  }
}

// Overwrites a buffer larger than L2 (126 MB) so the next step starts cold.
__global__ void k_flush(double* buf, long long n, double v) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    buf[i] = v;
}

// DFMA throughput probe: 8 independent FMA chains per thread.
__global__ void __launch_bounds__(256) k_dfma_peak(double* out, int iters, double m, double c) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
  for (int t = 0; t < iters; ++t) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], m, c);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 1.2345) out[0] = s;  // keeps the chains live
}

std::string itos(long long v) { return std::to_string(v); }

}  // namespace

// ===========================================================================
// Domain: one device's share of the cloud and its solver state.  A domain owns
// points [0, n_own) in local numbering and keeps read-only halo copies of the
// points its stencils reach in [n_own, n_loc); with one domain n_own = n_loc = n
// and local ids are global ids.
struct GeomView {
  int n_own = 0, n_loc = 0;
  const double *x = nullptr, *y = nullptr, *nx = nullptr, *ny = nullptr;  // n_loc
  const Kind* kind = nullptr;                                             // n_loc
  const std::int64_t* off = nullptr;                                      // n_own + 1
  const std::int32_t* nbr = nullptr;                                      // local ids
  const std::uint16_t* part = nullptr;                                    // n_loc or null
  const std::int32_t* gid = nullptr;                                      // n_loc or null
  std::int64_t nnz = 0;
};

GeomView view_of(const LocalGeom& g) {
  GeomView v;
  v.n_own = g.n_own;
  v.n_loc = g.n_loc;
  v.x = g.x.data();
  v.y = g.y.data();
  v.nx = g.nx.data();
  v.ny = g.ny.data();
  v.kind = g.kind.data();
  v.off = g.off.data();
  v.nbr = g.nbr.data();
  v.part = g.part.data();
  v.gid = g.gid.data();
  v.nnz = static_cast<std::int64_t>(g.nbr.size());
  return v;
}

GeomView view_of(const PointSet& ps, const std::vector<std::uint16_t>& part) {
  GeomView v;
  v.n_own = v.n_loc = ps.n();
  v.x = ps.x.data();
  v.y = ps.y.data();
  v.nx = ps.nx.data();
  v.ny = ps.ny.data();
  v.kind = ps.kind.data();
  v.off = ps.off.data();
  v.nbr = ps.nbr.data();
  v.part = part.size() == static_cast<std::size_t>(ps.n()) ? part.data() : nullptr;
  v.nnz = ps.nnz();
  return v;
}

Gas make_gas(double gamma, double cfl, double det_tol) {
  Gas g{};
  g.gamma = gamma;
  g.gm1 = gamma - 1.0;
  g.inv_gm1 = 1.0 / (gamma - 1.0);
  g.ep_fac = g.inv_gm1 + 1.0;
  g.cfl = cfl;
  g.det_tol = det_tol;
  const double m = 2.0 / (gamma - 1.0);
  const double mr = std::nearbyint(m);
  g.half_pow = (std::fabs(m - mr) < 1e-9 && mr >= 1.0 && mr <= 40.0) ? static_cast<int>(mr) : -1;
  return g;
}

// Geometry upload from a cloud whose arrays live in pinned host memory
// (HostAlloc): the coordinates arrive as two planes and are interleaved here;
// uniform stencils get their offsets generated, others narrowed to int32.
__global__ void k_interleave(const double* a, const double* b, double2* out, long long n) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    out[i] = make_double2(a[i], b[i]);
}
__global__ void k_off_fill(int* off, long long n, int k, const std::int64_t* src) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i <= n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    off[i] = src ? static_cast<int>(src[i]) : static_cast<int>(i * k);
}

bool pinned_host(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

class Domain {
 public:
  // ipc: buffers that peers read (q, dq, the shared word, the residue array)
  // come from plain cudaMalloc so they can be exported as CUDA IPC handles.
  Domain(const GeomView& gv, int device, double gamma, double cfl, double det_tol, int capacity,
         bool ipc = false)
      : n_(gv.n_own), n_loc_(gv.n_loc), device_(device), ipc_(ipc), stream_holder_(device) {
    st_ = stream_holder_.st;
    ck(cudaEventCreate(&ev0_), "cudaEventCreate");
    ck(cudaEventCreate(&ev1_), "cudaEventCreate");
    for (auto& e : kev_) ck(cudaEventCreate(&e), "cudaEventCreate");
    for (auto& e : poll_ev_) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    trace("domain: stream and events");
    if (gv.nnz >= (1ll << 31)) raise(Status::argument, "stencil table exceeds 2^31 entries");
    gas_ = make_gas(gamma, cfl, det_tol);
    nnz_ = gv.nnz;
    d1_ = tree_depth(n_);
    n_res_ = n_;

    const std::size_t n = static_cast<std::size_t>(n_), nl = static_cast<std::size_t>(n_loc_);
    const std::size_t nnz = static_cast<std::size_t>(gv.nnz);
    ensure_pool(device);
    // geometry, packed on the host into pinned staging, then async copies
    const std::size_t b_xy = nl * sizeof(double2), b_off = (n + 1) * sizeof(int), b_nbr = nnz * sizeof(int);
    const std::size_t b_gid = gv.gid ? nl * sizeof(int) : 0;
    trace("domain: pool");
    // Pass 1 on the host threads (reads only): stencil sizes (kmax, uniform
    // size kfix), wall points (normals are only read for them) and non-zero
    // partition ids (only read on the failure path).
    const int tasks = std::max(1, std::min(host_threads(), static_cast<int>(nl >> 14)));
    const std::int64_t k0 = n ? gv.off[1] - gv.off[0] : 0;
    std::vector<std::int64_t> t_kmax(static_cast<std::size_t>(tasks), 1);
    std::vector<char> t_uniform(static_cast<std::size_t>(tasks), 1), t_walls(static_cast<std::size_t>(tasks), 0),
        t_parts(static_cast<std::size_t>(tasks), 0);
    parallel_tasks(tasks, [&](int t) {
      auto part_of = [&](std::size_t len, int k) { return len * static_cast<std::size_t>(k) / tasks; };
      const std::size_t lo = part_of(nl, t), hi = part_of(nl, t + 1);
      char walls = 0, parts = 0;
      for (std::size_t i = lo; i < hi; ++i) walls |= static_cast<std::uint8_t>(gv.kind[i]) == KIND_WALL;
      if (gv.part)
        for (std::size_t i = lo; i < hi; ++i) parts |= gv.part[i] != 0;
      t_walls[t] = walls;
      t_parts[t] = parts;
      const std::size_t olo = part_of(n, t), ohi = part_of(n, t + 1);
      std::int64_t km = 1;
      bool uni = true;
      for (std::size_t i = olo; i < ohi; ++i) {
        const std::int64_t e0 = gv.off[i], k = gv.off[i + 1] - e0;
        km = std::max(km, k);
        uni = uni && k == k0 && e0 == static_cast<std::int64_t>(i) * k0;
      }
      t_kmax[t] = km;
      t_uniform[t] = uni;
    });
    std::int64_t km = 1;
    bool uniform = true;
    for (int t = 0; t < tasks; ++t) {
      km = std::max(km, t_kmax[t]);
      uniform = uniform && t_uniform[t];
    }
    kmax_ = static_cast<int>(km);
    if (kmax_ > kMaxStencil)
      raise(Status::argument, "stencils of more than " + std::to_string(kMaxStencil) + " neighbours are not supported");
    kfix_ = uniform && k0 == km ? kmax_ : 0;
    W_ = flux_width(kmax_);
    smem_ = flux_smem_bytes(W_, kmax_);
    stride_ = flux_stride(kmax_);
    const bool any_wall = std::any_of(t_walls.begin(), t_walls.end(), [](char c) { return c != 0; });
    const bool any_part = std::any_of(t_parts.begin(), t_parts.end(), [](char c) { return c != 0; });
    trace("domain: scanned");
    xy_.alloc(nl, st_);
    nrm_.alloc(nl, st_);
    kind_.alloc(nl, st_);
    part_.alloc(nl, st_);
    off_.alloc(n + 1, st_);
    nbr_.alloc(std::max<std::size_t>(1, nnz), st_);
    mind_.alloc(n, st_);
    if (!any_wall) ck(cudaMemsetAsync(nrm_.get(), 0, b_xy, st_), "zero nrm");
    if (!any_part) {
      ck(cudaMemsetAsync(part_.get(), 0, nl * sizeof(std::uint16_t), st_), "zero part");
      part_host_.clear();  // empty = all partition ids 0
    }
    // Pass 2a: a single-domain cloud whose arrays are pinned (HostAlloc) is
    // copied straight from them — no staging.
    // (kinds, 1 B per point, may sit below HostAlloc's pinned threshold: they
    // go through a small staging copy)
    const bool direct = n == nl && !gv.gid && pinned_host(gv.x) && pinned_host(gv.y) &&
                        (kfix_ > 0 || pinned_host(gv.off)) && (nnz == 0 || pinned_host(gv.nbr)) &&
                        (!any_wall || (pinned_host(gv.nx) && pinned_host(gv.ny))) && !any_part;
    if (direct) {
      const int blocks = static_cast<int>(std::min<std::size_t>(4096, (nl + 255) / 256));
      DBuf<double> tx(std::max<std::size_t>(1, nl), st_), ty(std::max<std::size_t>(1, nl), st_);
      trace("domain: direct temporaries");
      auto planes = [&](const double* a, const double* b, double2* out, const char* what) {
        ck(cudaMemcpyAsync(tx.get(), a, nl * sizeof(double), cudaMemcpyHostToDevice, st_), what);
        ck(cudaMemcpyAsync(ty.get(), b, nl * sizeof(double), cudaMemcpyHostToDevice, st_), what);
        k_interleave<<<blocks, 256, 0, st_>>>(tx.get(), ty.get(), out, static_cast<long long>(nl));
        ck(cudaGetLastError(), "k_interleave");
      };
      planes(gv.x, gv.y, xy_.get(), "H2D x/y");
      if (nnz) ck(cudaMemcpyAsync(nbr_.get(), gv.nbr, b_nbr, cudaMemcpyHostToDevice, st_), "H2D nbr");
      if (pinned_host(gv.kind)) {
        ck(cudaMemcpyAsync(kind_.get(), gv.kind, nl, cudaMemcpyHostToDevice, st_), "H2D kind");
      } else {
        std::uint8_t* hk = static_cast<std::uint8_t*>(t_staging.get(nl));
        stream_copy(hk, gv.kind, nl);
        ck(cudaMemcpyAsync(kind_.get(), hk, nl, cudaMemcpyHostToDevice, st_), "H2D kind");
      }
      DBuf<std::int64_t> toff(kfix_ > 0 ? 1 : n + 1, st_);
      if (kfix_ == 0)
        ck(cudaMemcpyAsync(toff.get(), gv.off, (n + 1) * sizeof(std::int64_t), cudaMemcpyHostToDevice, st_), "H2D off");
      k_off_fill<<<blocks, 256, 0, st_>>>(off_.get(), static_cast<long long>(n), kfix_, kfix_ > 0 ? nullptr : toff.get());
      ck(cudaGetLastError(), "k_off_fill");
      if (any_wall) {
        ck(cudaStreamSynchronize(st_), "geometry planes");  // tx/ty are reused
        planes(gv.nx, gv.ny, nrm_.get(), "H2D nx/ny");
      }
      trace("domain: direct copies queued");
      ck(cudaStreamSynchronize(st_), "geometry upload");  // temporaries go back to the pool
      trace("domain: direct copies done");
    }
    // Pass 2: stage the geometry into pinned memory in point chunks (streaming
    // stores / flushed lines, so the DMA runs at PCIe rate, hostcopy.cpp) and
    // queue each chunk's copies as soon as it is staged — staging chunk c + 1
    // overlaps the DMA of chunk c.
    char* hs = direct ? nullptr : static_cast<char*>(t_staging.get(2 * b_xy + 3 * nl + b_off + b_nbr + b_gid + 64));
    double2* hxy = reinterpret_cast<double2*>(hs);
    double2* hnrm = hxy + nl;
    std::uint16_t* hpart = reinterpret_cast<std::uint16_t*>(hnrm + nl);
    std::uint8_t* hkind = reinterpret_cast<std::uint8_t*>(hpart + nl);
    int* hoff = reinterpret_cast<int*>(hs + ((2 * b_xy + 3 * nl + 15) & ~std::size_t{15}));
    int* hnbr = hoff + n + 1;
    int* hgid = hnbr + nnz;
    const int chunks = direct ? 0 : static_cast<int>(std::max<std::size_t>(1, std::min<std::size_t>(8, nl >> 20)));
    for (int c = 0; c < chunks; ++c) {
      const std::size_t lo = nl * c / chunks, hi = nl * (c + 1) / chunks;
      const std::size_t olo = std::min(lo, n), ohi = std::min(hi, n);
      const std::size_t elo = olo < n ? static_cast<std::size_t>(gv.off[olo]) : nnz;
      const std::size_t ehi = static_cast<std::size_t>(gv.off[ohi]);
      parallel_slices(static_cast<std::int64_t>(hi - lo), [&](std::int64_t a, std::int64_t b) {
        const std::size_t plo = lo + a, phi = lo + b, cnt = phi - plo;
        stream_pairs(reinterpret_cast<double*>(hxy + plo), gv.x + plo, gv.y + plo, cnt);
        if (any_wall) stream_pairs(reinterpret_cast<double*>(hnrm + plo), gv.nx + plo, gv.ny + plo, cnt);
        for (std::size_t i = plo; i < phi; ++i) hkind[i] = static_cast<std::uint8_t>(gv.kind[i]);
        flush_lines(hkind + plo, cnt);
        if (any_part) {
          for (std::size_t i = plo; i < phi; ++i) hpart[i] = gv.part[i];
          flush_lines(hpart + plo, cnt * sizeof(std::uint16_t));
        }
        const std::size_t qlo = std::min(plo, n), qhi = std::min(phi, n);
        for (std::size_t i = qlo; i < qhi; ++i) hoff[i] = static_cast<int>(gv.off[i]);
        if (qhi > qlo) flush_lines(hoff + qlo, (qhi - qlo) * sizeof(int));
        if (qhi > qlo) {
          const std::size_t blo = static_cast<std::size_t>(gv.off[qlo]) * sizeof(int),
                            bhi = static_cast<std::size_t>(gv.off[qhi]) * sizeof(int);
          stream_copy(reinterpret_cast<char*>(hnbr) + blo, reinterpret_cast<const char*>(gv.nbr) + blo, bhi - blo);
        }
      }, 1 << 14);
      if (c == chunks - 1) {
        hoff[n] = static_cast<int>(gv.off[n]);
        flush_lines(hoff + n, sizeof(int));
      }
      const std::size_t cnt = hi - lo;
      ck(cudaMemcpyAsync(xy_.get() + lo, hxy + lo, cnt * sizeof(double2), cudaMemcpyHostToDevice, st_), "H2D xy");
      if (any_wall)
        ck(cudaMemcpyAsync(nrm_.get() + lo, hnrm + lo, cnt * sizeof(double2), cudaMemcpyHostToDevice, st_), "H2D nrm");
      ck(cudaMemcpyAsync(kind_.get() + lo, hkind + lo, cnt, cudaMemcpyHostToDevice, st_), "H2D kind");
      if (any_part)
        ck(cudaMemcpyAsync(part_.get() + lo, hpart + lo, cnt * sizeof(std::uint16_t), cudaMemcpyHostToDevice, st_),
           "H2D part");
      const std::size_t offn = ohi - olo + (c == chunks - 1 ? 1 : 0);
      if (offn)
        ck(cudaMemcpyAsync(off_.get() + olo, hoff + olo, offn * sizeof(int), cudaMemcpyHostToDevice, st_), "H2D off");
      if (ehi > elo)
        ck(cudaMemcpyAsync(nbr_.get() + elo, hnbr + elo, (ehi - elo) * sizeof(int), cudaMemcpyHostToDevice, st_),
           "H2D nbr");
    }
    if (any_part) part_host_.assign(hpart, hpart + nl);
    trace("domain: staged, copies queued");
    if (gv.gid) {
      std::memcpy(hgid, gv.gid, b_gid);
      flush_lines(hgid, b_gid);
      gid_host_.assign(gv.gid, gv.gid + nl);
    }
    if (gv.gid) {
      gid_.alloc(nl, st_);
      ck(cudaMemcpyAsync(gid_.get(), hgid, b_gid, cudaMemcpyHostToDevice, st_), "H2D gid");
    }
    // state: q / dq carry halo slots; prim covers them for the first q_variables
    cudaStream_t shared_st = ipc ? nullptr : st_;
    prim_.alloc(nl, st_);
    q_[0].alloc(nl, shared_st);
    q_[1].alloc(nl, shared_st);
    dq_[0].alloc(2 * nl, shared_st);
    dq_[1].alloc(2 * nl, shared_st);
    res_.alloc(n, st_);
    dt_.alloc(n, st_);
    which_.alloc(n, st_);
    mag_.alloc(n, st_);
    mag_out_ = mag_.get();
    pval_.alloc(8192, st_);
    psz_.alloc(8192, st_);
    acc_.alloc(2 * kAccWords, shared_st);  // peers read it (root's residue)
    acc_tab_.p[0] = acc_.get();
    acc_ndom_ = 1;
    ctl_.alloc(1, st_);
    sh_.alloc(1, shared_st);
    // whole words defined (refresh_ctl copies them back, padding included)
    ck(cudaMemsetAsync(ctl_.get(), 0, sizeof(Ctl), st_), "memset ctl");
    ck(cudaMemsetAsync(sh_.get(), 0, sizeof(Shared), st_), "memset shared");
    shared_ = sh_.get();
    diag_.alloc(8, st_);
    capacity_ = std::max(capacity, 1);
    hist_.alloc(capacity_, st_);
    it0_.alloc(capacity_, st_);
    it1_.alloc(capacity_, st_);
    hpoll_.alloc(kPolls);
    hctl_.alloc(1);
    hsh_.alloc(1);
    trace("domain: allocated, copies queued");
    trace_sync(st_, "domain: copies done");
    DBuf<unsigned long long> zc(1, st_);
    ck(cudaMemsetAsync(zc.get(), 0, sizeof(unsigned long long), st_), "memset");
    k_min_dist<<<(n_ + 255) / 256, 256, 0, st_>>>(geo(), mind_.get(), zc.get());
    ck(cudaGetLastError(), "k_min_dist");
    k_ctl_init<<<1, 1, 0, st_>>>(ctl_.get(), shared_, 1, -1, 0, update_blocks());
    ck(cudaMemcpyAsync(&zero_pairs_, zc.get(), sizeof zero_pairs_, cudaMemcpyDeviceToHost, st_), "D2H zero pairs");
    ck(cudaStreamSynchronize(st_), "geometry upload");
  }

  ~Domain() {
    cudaSetDevice(device_);
    cudaStreamSynchronize(st_);  // nothing in flight before the buffers go back to the pool
    clear_graphs();
    cudaEventDestroy(ev0_);
    cudaEventDestroy(ev1_);
    for (auto& e : kev_) cudaEventDestroy(e);
    for (auto& e : poll_ev_) cudaEventDestroy(e);
    // the stream itself is released by stream_holder_ after every DBuf member
  }

  Geo geo() const {
    Geo g;
    g.xy = xy_.get();
    g.nrm = nrm_.get();
    g.kind = kind_.get();
    g.part = part_.get();
    g.off = off_.get();
    g.nbr = nbr_.get();
    g.mind = mind_.get();
    g.gid = gid_.get();
    g.n = n_;
    g.kfix = kfix_;
    g.nloc = n_loc_;
    return g;
  }

  // ---- multi-domain wiring ----
  // Use another domain's shared control word (error word, iteration counter).
  void use_shared(Shared* sh) { shared_ = sh; }
  Shared* shared() const { return shared_; }
  // Residue summands are written (by global id) into `mag` (the root's array).
  void use_mag(double* mag) { mag_out_ = mag; }
  // Root only: residue tree over n_total global ids.
  void set_residue_size(long long n_total) {
    n_res_ = n_total;
    d1_ = tree_depth(n_total);
    if (n_total != n_ || ipc_) {
      mag_.alloc(static_cast<std::size_t>(n_total), ipc_ ? nullptr : st_);
      mag_out_ = mag_.get();
    }
  }
  double* mag_buf() { return mag_.get(); }
  // Exact residue accumulators ([2][kAccWords]); the root sums every domain's.
  unsigned long long* acc_buf() { return acc_.get(); }
  void use_acc_tab(const AccTab& t, int ndom) {
    acc_tab_ = t;
    acc_ndom_ = ndom;
  }
  Shared* own_shared() { return sh_.get(); }
  int n_loc() const { return n_loc_; }
  int device() const { return device_; }
  int global_of(int local) const { return gid_host_.empty() ? local : gid_host_[local]; }
  // Local index of an owned cloud point (failure diagnostics; linear search).
  int local_of(long long global) const {
    if (gid_host_.empty()) return static_cast<int>(global);
    const auto it = std::find(gid_host_.begin(), gid_host_.begin() + n_, static_cast<int>(global));
    return it == gid_host_.begin() + n_ ? 0 : static_cast<int>(it - gid_host_.begin());
  }

  // ---- stencil screening (validate_cloud) on the device-resident geometry ----
  Screening screen() {
    ck(cudaSetDevice(device_), "cudaSetDevice");
    Screening out;
    const int n = n_;
    if (n <= 0) return out;
    if (tracing()) {
      cudaEventCreate(&ev_trace_);
      cudaEventRecord(ev_trace_, st_);
    }
    DBuf<ScreenOut> so(1, st_);
    ScreenOut init{0, 0, 0, 0x7FFFFFFF, 0};
    ck(cudaMemcpyAsync(so.get(), &init, sizeof init, cudaMemcpyHostToDevice, st_), "H2D screen");
    // keys, sorted keys, the sort's temporary space and the defect list in one scratch lease
    std::size_t tmp_bytes = 0;
    ck(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, static_cast<unsigned long long*>(nullptr),
                                      static_cast<unsigned long long*>(nullptr), n, 0, 64, st_),
       "sort size");
    auto up = [](std::size_t b) { return (b + 255) & ~static_cast<std::size_t>(255); };
    const std::size_t kb = up(static_cast<std::size_t>(n) * sizeof(unsigned long long));
    const std::size_t tb = up(std::max<std::size_t>(1, tmp_bytes));
    const std::size_t bb = up(static_cast<std::size_t>(n) * sizeof(int));
    ScratchLease scr(device_, kScratchScreen, 2 * kb + tb + bb);
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(scr.get());
    unsigned long long* sorted = reinterpret_cast<unsigned long long*>(scr.get() + kb);
    char* tmp = scr.get() + 2 * kb;
    int* bad = reinterpret_cast<int*>(scr.get() + 2 * kb + tb);
    trace_sync(st_, "screen: buffers");
    k_screen_keys<<<(n + 255) / 256, 256, 0, st_>>>(n, mind_.get(), keys, so.get());
    trace_sync(st_, "screen: keys");
    ck(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, keys, sorted, n, 0, 64, st_), "sort");
    trace_sync(st_, "screen: sorted");
    ScreenOut head{};
    ck(cudaMemcpyAsync(&head, so.get(), sizeof head, cudaMemcpyDeviceToHost, st_), "D2H screen");
    if (tracing()) {  // device time of the work queued so far vs the host's wait
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, st_);
      cudaEventSynchronize(e);
      float ms = 0.0f;
      cudaEventElapsedTime(&ms, ev_trace_, e);
      char buf[96];
      std::snprintf(buf, sizeof buf, "screen: device work since upload %.2f ms", ms);
      trace(buf);
      cudaEventDestroy(e);
    }
    ck(cudaStreamSynchronize(st_), "screen keys");
    if (head.n_finite > 0) {
      unsigned long long bits = 0;
      ck(cudaMemcpy(&bits, sorted + (head.n_finite - 1) / 2, sizeof bits, cudaMemcpyDeviceToHost), "D2H h_ref");
      std::memcpy(&out.h_ref, &bits, sizeof bits);
    }
    out.det_tol = 1e-12 * out.h_ref * out.h_ref * out.h_ref * out.h_ref;  // cloud.cpp:274
    const int cap = n;
    k_screen<<<(n + 255) / 256, 256, 0, st_>>>(geo(), out.det_tol, so.get(), bad, cap);
    ck(cudaGetLastError(), "k_screen");
    ck(cudaMemcpyAsync(&head, so.get(), sizeof head, cudaMemcpyDeviceToHost, st_), "D2H screen");
    ck(cudaStreamSynchronize(st_), "screen");
    out.n_defective = head.n_defective;
    out.n_wall_isolated = head.n_wall_isolated;
    out.min_stencil = head.min_size;
    out.defective.resize(static_cast<std::size_t>(head.n_defective));
    if (head.n_defective > 0) {
      ck(cudaMemcpy(out.defective.data(), bad, sizeof(int) * head.n_defective, cudaMemcpyDeviceToHost),
         "D2H defective");
      for (auto& p : out.defective) p = global_of(p);  // point ids of the cloud
      std::sort(out.defective.begin(), out.defective.end());
    }
    return out;
  }

  // ---- state transfer (FieldBlock <-> device records) ----
  // Uniform primitive state on owned and halo points (lskum_run's free stream).
  void fill_prim(const double (&v)[4]) {
    k_fill_d4<<<std::min<int>((n_loc_ + 255) / 256, 4096), 256, 0, st_>>>(prim_.get(), n_loc_,
                                                                          D4{v[0], v[1], v[2], v[3]});
    ck(cudaGetLastError(), "k_fill_d4");
  }

  void upload(const FieldBlock& f, bool full) {
    const std::size_t n = static_cast<std::size_t>(n_);
    if (!full && gid_host_.empty()) {
      // primitives only: 4 doubles per point through pinned staging (SoA: the
      // first 4n doubles of the block; AoS: gathered 4 of every 21)
      const bool soa = f.layout() == Layout::soa;
      double* h = static_cast<double*>(t_staging.get(4 * n * sizeof(double)));
      if (soa) {
        stream_copy(h, f.raw(), 4 * n * sizeof(double));
      } else {
        const double* src = f.raw();
        for (std::size_t i = 0; i < n; ++i) std::memcpy(h + 4 * i, src + 21 * i, 4 * sizeof(double));
        flush_lines(h, 4 * n * sizeof(double));
      }
      DBuf<double> tmp(4 * n, st_);
      ck(cudaMemcpyAsync(tmp.get(), h, 4 * n * sizeof(double), cudaMemcpyHostToDevice, st_), "H2D prim");
      k_unpack_prim<<<std::min<int>((n_ + 255) / 256, 4096), 256, 0, st_>>>(n_, soa ? 1 : 0, tmp.get(),
                                                                            prim_.get());
      ck(cudaGetLastError(), "k_unpack_prim");
      ck(cudaStreamSynchronize(st_), "upload");
      return;
    }
    if (!full) {
      // owned + halo primitives gathered by global id
      const std::size_t nl = static_cast<std::size_t>(n_loc_);
      D4* h = static_cast<D4*>(t_staging.get(nl * sizeof(D4)));
      for (std::size_t i = 0; i < nl; ++i) {
        const int p = gid_host_[i];
        h[i] = D4{f.at(p, slot::prim), f.at(p, slot::prim + 1), f.at(p, slot::prim + 2), f.at(p, slot::prim + 3)};
      }
      flush_lines(h, nl * sizeof(D4));
      ck(cudaMemcpyAsync(prim_.get(), h, nl * sizeof(D4), cudaMemcpyHostToDevice, st_), "H2D prim");
      ck(cudaStreamSynchronize(st_), "upload");
      return;
    }
    std::vector<D4> h(6 * n);
    D4* hp = h.data();
    for (std::size_t i = 0; i < n; ++i) {
      const int p = static_cast<int>(i);
      hp[i] = D4{f.at(p, slot::prim), f.at(p, slot::prim + 1), f.at(p, slot::prim + 2), f.at(p, slot::prim + 3)};
      hp[n + i] = D4{f.at(p, slot::q), f.at(p, slot::q + 1), f.at(p, slot::q + 2), f.at(p, slot::q + 3)};
      // derivative planes (dq_load/dq_store layout): qx records, then qy records
      hp[2 * n + i] = D4{f.at(p, slot::qx), f.at(p, slot::qx + 1), f.at(p, slot::qx + 2), f.at(p, slot::qx + 3)};
      hp[3 * n + i] = D4{f.at(p, slot::qy), f.at(p, slot::qy + 1), f.at(p, slot::qy + 2), f.at(p, slot::qy + 3)};
      hp[4 * n + i] =
          D4{f.at(p, slot::res), f.at(p, slot::res + 1), f.at(p, slot::res + 2), f.at(p, slot::res + 3)};
      reinterpret_cast<double*>(hp + 5 * n)[i] = f.at(p, slot::dt);
    }
    ck(cudaMemcpyAsync(prim_.get(), hp, n * sizeof(D4), cudaMemcpyHostToDevice, st_), "H2D prim");
    ck(cudaMemcpyAsync(q_[0].get(), hp + n, n * sizeof(D4), cudaMemcpyHostToDevice, st_), "H2D q");
    ck(cudaMemcpyAsync(dq_[0].get(), hp + 2 * n, n * sizeof(D4), cudaMemcpyHostToDevice, st_), "H2D qx");
    ck(cudaMemcpyAsync(dq_[0].get() + n_loc_, hp + 3 * n, n * sizeof(D4), cudaMemcpyHostToDevice, st_), "H2D qy");
    ck(cudaMemcpyAsync(res_.get(), hp + 4 * n, n * sizeof(D4), cudaMemcpyHostToDevice, st_), "H2D res");
    ck(cudaMemcpyAsync(dt_.get(), hp + 5 * n, n * sizeof(double), cudaMemcpyHostToDevice, st_), "H2D dt");
    ck(cudaStreamSynchronize(st_), "upload");
  }

  void download(FieldBlock& f, bool with_q, const D4* qsrc, const D4* dqsrc) {
    const std::size_t n = static_cast<std::size_t>(n_);
    if (with_q && (gid_host_.empty() || (n_loc_ == n_ && static_cast<std::size_t>(f.size()) == n))) {
      // pack on the device in the host layout (scattered to cloud order when
      // the domain is a permutation of the whole cloud), one D2H into the store
      const bool soa = f.layout() == Layout::soa;
      void* hdev = nullptr;
      if (f.pinned() && gid_host_.empty() && zero_copy_store() &&
          cudaHostGetDevicePointer(&hdev, f.raw(), 0) == cudaSuccess && hdev) {
        // pinned store in cloud order: the kernels write it directly (zero copy)
        double* out = static_cast<double*>(hdev);
        if (soa)  // 21 rows: consecutive points of a row are consecutive addresses
          k_pack_fields<<<std::min<int>((n_ + 255) / 256, 4096), 256, 0, st_>>>(
              n_, 0, n_, 1, prim_.get(), qsrc, dqsrc, static_cast<long long>(n_loc_), res_.get(), dt_.get(), nullptr,
              out);
        else
          k_pack_aos_host<<<std::min<int>((n_ + kPackPts - 1) / kPackPts, 2048), kPackPts, 0, st_>>>(
              n_, prim_.get(), qsrc, dqsrc, static_cast<long long>(n_loc_), res_.get(), dt_.get(), out);
        ck(cudaGetLastError(), "k_pack (zero copy)");
        ck(cudaStreamSynchronize(st_), "download");
        trace("download: stored (zero copy)");
        return;
      }
      cudaGetLastError();
      ScratchLease packed_lease(device_, kScratchPack, 21 * n * sizeof(double));
      double* const packed = reinterpret_cast<double*>(packed_lease.get());
      auto pack = [&](int lo, int hi) {
        k_pack_fields<<<std::max(1, std::min<int>((hi - lo + 255) / 256, 4096)), 256, 0, st_>>>(
            n_, lo, hi, soa ? 1 : 0, prim_.get(), qsrc, dqsrc, static_cast<long long>(n_loc_), res_.get(), dt_.get(),
            static_cast<const int*>(gid_.get()), packed);
        ck(cudaGetLastError(), "k_pack_fields");
      };
      if (f.pinned()) {  // the store is pinned: DMA straight into it
        if (gid_host_.empty()) {
          // cloud order: pack and copy in point chunks, so the packing of
          // chunk c + 1 overlaps the transfer of chunk c (SoA: 21 rows of the
          // chunk's points, one 2-D copy)
          // (the copies run on a second stream, each after its chunk's packing)
          const int chunks = static_cast<int>(std::max<std::size_t>(1, std::min<std::size_t>(8, n >> 20)));
          cudaStream_t cs = nullptr;
          ck(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "cudaStreamCreate");
          std::vector<cudaEvent_t> packed_ev(static_cast<std::size_t>(chunks));
          for (auto& e : packed_ev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
          cudaError_t err = cudaSuccess;
          for (int c = 0; c < chunks && err == cudaSuccess; ++c) {
            const int lo = static_cast<int>(n * c / chunks), hi = static_cast<int>(n * (c + 1) / chunks);
            pack(lo, hi);
            err = cudaEventRecord(packed_ev[c], st_);
            if (err == cudaSuccess) err = cudaStreamWaitEvent(cs, packed_ev[c], 0);
            if (err != cudaSuccess) break;
            if (soa)
              err = cudaMemcpy2DAsync(f.raw() + lo, n * sizeof(double), packed + lo, n * sizeof(double),
                                      (hi - lo) * sizeof(double), 21, cudaMemcpyDeviceToHost, cs);
            else
              err = cudaMemcpyAsync(f.raw() + 21ll * lo, packed + 21ll * lo, 21ll * (hi - lo) * sizeof(double),
                                    cudaMemcpyDeviceToHost, cs);
          }
          trace("download: chunks queued");
          const cudaError_t serr = cudaStreamSynchronize(cs);
          for (auto& e : packed_ev) cudaEventDestroy(e);
          cudaStreamDestroy(cs);
          ck(err, "D2H fields");
          ck(serr, "download (copy stream)");
        } else {
          pack(0, n_);
          ck(cudaMemcpyAsync(f.raw(), packed, 21 * n * sizeof(double), cudaMemcpyDeviceToHost, st_),
             "D2H fields");
        }
        ck(cudaStreamSynchronize(st_), "download");
        trace("download: stored (pinned store)");
        return;
      }
      pack(0, n_);
      trace_sync(st_, "download: packed");
      // through pinned staging (full-rate D2H) in chunks; host threads copy
      // each chunk into the store as soon as its transfer completes
      const std::size_t count = 21 * n, bytes = count * sizeof(double);
      double* h = static_cast<double*>(t_staging.get(bytes));
      double* dst = f.raw();
      const int chunks = static_cast<int>(std::max<std::size_t>(1, std::min<std::size_t>(16, bytes >> 21)));
      std::vector<cudaEvent_t> done(static_cast<std::size_t>(chunks));
      auto lo_of = [&](std::int64_t c) { return count * static_cast<std::size_t>(c) / static_cast<std::size_t>(chunks); };
      for (int c = 0; c < chunks; ++c) {
        const std::size_t lo = lo_of(c), hi = lo_of(c + 1);
        ck(cudaEventCreateWithFlags(&done[c], cudaEventDisableTiming), "cudaEventCreate");
        ck(cudaMemcpyAsync(h + lo, packed + lo, (hi - lo) * sizeof(double), cudaMemcpyDeviceToHost, st_),
           "D2H fields");
        ck(cudaEventRecord(done[c], st_), "cudaEventRecord");
      }
      trace("download: copies queued");
      std::atomic<int> sync_err{0};
      parallel_slices(chunks, [&](std::int64_t a, std::int64_t b) {
        for (std::int64_t c = a; c < b; ++c) {
          const cudaError_t e = cudaEventSynchronize(done[c]);
          if (e != cudaSuccess) {  // never copy stale staging bytes into the store
            int none = 0;
            sync_err.compare_exchange_strong(none, static_cast<int>(e));
            continue;
          }
          const std::size_t lo = lo_of(c), hi = lo_of(c + 1);
          std::memcpy(dst + lo, h + lo, (hi - lo) * sizeof(double));
          flush_lines(h + lo, (hi - lo) * sizeof(double));  // the next DMA into staging stays at full rate
        }
      }, 1);
      trace("download: copied out");
      if (sync_err.load() != 0) {
        for (cudaEvent_t e : done) cudaEventDestroy(e);
        ck(static_cast<cudaError_t>(sync_err.load()), "download (copy-back event)");
      }
      ck(cudaStreamSynchronize(st_), "download");
      trace("download: stored");
      for (cudaEvent_t e : done) cudaEventDestroy(e);
      return;
    }
    std::vector<D4> h(6 * n);
    D4* hp = h.data();
    ck(cudaMemcpyAsync(hp, prim_.get(), n * sizeof(D4), cudaMemcpyDeviceToHost, st_), "D2H prim");
    if (with_q) ck(cudaMemcpyAsync(hp + n, qsrc, n * sizeof(D4), cudaMemcpyDeviceToHost, st_), "D2H q");
    ck(cudaMemcpyAsync(hp + 2 * n, dqsrc, n * sizeof(D4), cudaMemcpyDeviceToHost, st_), "D2H qx");
    ck(cudaMemcpyAsync(hp + 3 * n, dqsrc + n_loc_, n * sizeof(D4), cudaMemcpyDeviceToHost, st_), "D2H qy");
    ck(cudaMemcpyAsync(hp + 4 * n, res_.get(), n * sizeof(D4), cudaMemcpyDeviceToHost, st_), "D2H res");
    ck(cudaMemcpyAsync(hp + 5 * n, dt_.get(), n * sizeof(double), cudaMemcpyDeviceToHost, st_), "D2H dt");
    ck(cudaStreamSynchronize(st_), "download");
    const double* dtp = reinterpret_cast<const double*>(hp + 5 * n);
    for (std::size_t i = 0; i < n; ++i) {
      const int p = global_of(static_cast<int>(i));
      const D4& s = hp[i];
      f.at(p, slot::prim) = s.a;
      f.at(p, slot::prim + 1) = s.b;
      f.at(p, slot::prim + 2) = s.c;
      f.at(p, slot::prim + 3) = s.d;
      if (with_q) {
        const D4& q = hp[n + i];
        f.at(p, slot::q) = q.a;
        f.at(p, slot::q + 1) = q.b;
        f.at(p, slot::q + 2) = q.c;
        f.at(p, slot::q + 3) = q.d;
      }
      const D4& qx = hp[2 * n + i];
      const D4& qy = hp[3 * n + i];
      const D4& r = hp[4 * n + i];
      for (int c = 0; c < 4; ++c) {
        f.at(p, slot::qx + c) = comp(qx, c);
        f.at(p, slot::qy + c) = comp(qy, c);
        f.at(p, slot::res + c) = comp(r, c);
      }
      f.at(p, slot::dt) = dtp[i];
    }
  }

  // ---- solver mode ----
  // Zeroes the once-per-run fields (runtime.cpp:216-224) and the control
  // block; with `own_shared` this domain also resets the run's shared word.
  void reset_run(int order, int inner, int fp_mode, int chunk, bool own_shared) {
    // captured graphs bake in the iteration's kernel sequence
    if (order != order_ || inner != inner_ || (fp_mode == 1) != strict_ || std::max(1, chunk) != chunk_)
      clear_graphs();
    order_ = order;
    inner_ = inner;
    strict_ = fp_mode == 1;
    chunk_ = std::max(1, chunk);
    if (!strict_ && flux_weighted()) ensure_weights();
    if (order == 2) ensure_tiles();
    if (!strict_ && order == 1 && point_flux_enabled() && !pf_.get()) {  // not inside a graph capture
      pf_.alloc(static_cast<std::size_t>(std::max(1, n_loc_)), st_);
      pfvalid_.alloc(static_cast<std::size_t>(std::max(1, n_loc_)), st_);
    }
    const std::size_t n = static_cast<std::size_t>(n_), nl = static_cast<std::size_t>(n_loc_);
    ck(cudaMemsetAsync(dq_[0].get(), 0, 2 * nl * sizeof(D4), st_), "zero dq");
    ck(cudaMemsetAsync(dq_[1].get(), 0, 2 * nl * sizeof(D4), st_), "zero dq");
    ck(cudaMemsetAsync(res_.get(), 0, n * sizeof(D4), st_), "zero res");
    ck(cudaMemsetAsync(dt_.get(), 0, n * sizeof(double), st_), "zero dt");
    ck(cudaMemsetAsync(acc_.get(), 0, 2 * kAccWords * sizeof(unsigned long long), st_), "zero acc");
    k_ctl_init<<<1, 1, 0, st_>>>(ctl_.get(), shared_, own_shared ? 1 : 0, -1, (order == 2 ? inner : 0) + 4,
                                 update_blocks(), split4_ ? 1 : 0);
    a_ = 0;
    b_ = 0;
    done_ = 0;
    total_ms_ = 0.0;
  }
  // The first iteration's q_variables over owned and halo points; later q
  // comes out of k_update.
  void first_q() {
    Geo g = geo();
    g.n = n_loc_;
    k_qvar<<<(n_loc_ + 255) / 256, 256, 0, st_>>>(g, prim_.get(), q_[0].get(), gas_, ctl_.get());
    ck(cudaGetLastError(), "k_qvar");
    probe_defer();
  }
  // Whether this run defers the flux's rare paths: only while few points take
  // them (measured at 10M points: deferral 3.65 vs 3.78 ms per iteration up to
  // M 1.6, but 10.7 vs 4.65 ms at M 2, where every point goes through the
  // redo).  Decided from the run's initial state; both choices give the same
  // bits.  Captured graphs bake the choice in.
  void probe_defer() {
    bool defer = false;
    if (!strict_ && weights_ && flux_defer_mode() == 2 && !any_sing_) {
      defer = true;
    } else if (!strict_ && weights_ && flux_defer() && !any_sing_ && n_ > 0) {
      DBuf<unsigned> cnt(1, st_);
      ck(cudaMemsetAsync(cnt.get(), 0, sizeof(unsigned), st_), "zero probe");
      k_defer_probe<<<std::min((n_ + 255) / 256, 4096), 256, 0, st_>>>(geo(), prim_.get(), cnt.get());
      ck(cudaGetLastError(), "k_defer_probe");
      unsigned h = 0;
      ck(cudaMemcpyAsync(&h, cnt.get(), sizeof h, cudaMemcpyDeviceToHost, st_), "D2H probe");
      ck(cudaStreamSynchronize(st_), "probe");
      defer = static_cast<long long>(h) * 100 <= static_cast<long long>(n_);  // <= 1% of the points
    }
    if (defer != defer_run_) clear_graphs();
    defer_run_ = defer;
  }
  void begin_run(int order, int inner, int fp_mode, int chunk) {
    reset_run(order, inner, fp_mode, chunk, true);
    trace("engine: run reset (weights)");
    first_q();
    ck(cudaStreamSynchronize(st_), "begin_run");
    refresh_ctl();
  }

  // Kernels of one launch_flux: the point fluxes + gather (order 1), or the
  // staged kernel + the redo pass of its rare-path points (DEFER), or one.
  int flux_launches() const {
    const bool pf = !strict_ && weights_ && order_ == 1 && point_flux_enabled() && pf_.get() && kmax_ <= 8;
    if (pf) return 2;
    const bool redo = !strict_ && weights_ && kmax_ <= 8 && flux_staged() && defer_run_;
    return redo ? 2 : 1;
  }
  int launches_per_iter() const { return (order_ == 2 ? inner_ : 0) + flux_launches() + 1 + (strict_ ? 2 : 1); }

  // Grid of k_update (persistent: at most the resident blocks); fixed per
  // domain, since the iteration index is derived from its completed blocks.
  int update_blocks() const {
    return std::max(1, std::min((n_ + 255) / 256, resident_blocks(k_update, 3)));
  }

  void clear_graphs() {
    for (auto& kv : graphs_) cudaGraphExecDestroy(kv.second);
    graphs_.clear();
  }

  // Reuse by a later run on the same geometry (the per-cloud engine cache):
  // gas constants, the error tie-break partition ids and the history
  // capacity may change; kernels captured with the old values are dropped.
  void reconfigure(double gamma, double cfl, double det_tol, const std::uint16_t* part, int capacity) {
    ck(cudaSetDevice(device_), "cudaSetDevice");
    const Gas g = make_gas(gamma, cfl, det_tol);
    if (g.gamma != gas_.gamma || g.cfl != gas_.cfl || g.det_tol != gas_.det_tol) {
      if (g.det_tol != gas_.det_tol) weights_ = false;
      gas_ = g;
      clear_graphs();
    }
    if (capacity > capacity_) {
      capacity_ = capacity;
      hist_.alloc(capacity_, st_);
      it0_.alloc(capacity_, st_);
      it1_.alloc(capacity_, st_);
      clear_graphs();
    }
    const std::size_t nl = static_cast<std::size_t>(n_loc_);
    if (!part && part_host_.empty()) return;  // one partition before and now (the common case)
    std::vector<std::uint16_t> hp(nl, 0);
    if (part)
      for (std::size_t i = 0; i < nl; ++i) hp[i] = part[gid_host_.empty() ? i : static_cast<std::size_t>(gid_host_[i])];
    const bool zero = std::all_of(hp.begin(), hp.end(), [](std::uint16_t v) { return v == 0; });
    if (zero && part_host_.empty()) return;
    if (zero) {
      part_host_.clear();
      ck(cudaMemsetAsync(part_.get(), 0, nl * sizeof(std::uint16_t), st_), "zero part");
    } else if (hp != part_host_) {
      part_host_ = hp;
      ck(cudaMemcpyAsync(part_.get(), part_host_.data(), nl * sizeof(std::uint16_t), cudaMemcpyHostToDevice, st_),
         "H2D part");
    }
    ck(cudaStreamSynchronize(st_), "part");
  }

  // Geometry-only split-stencil weights for the fast flux kernel (once per
  // domain); the zero-offset table w2 only exists when such pairs do.
  void ensure_weights() {
    if (weights_) return;
    const int blocks = (n_ + 255) / 256;
    const std::size_t nnz = static_cast<std::size_t>(std::max<std::int64_t>(1, nnz_));
    w1_.alloc(nnz, st_);
    psign_.alloc(nnz, st_);
    if (zero_pairs_) w2_.alloc(nnz, st_);  // counted by k_min_dist
    sing_.alloc(static_cast<std::size_t>(std::max(1, n_)), st_);
    const std::size_t nwords =
        static_cast<std::size_t>((std::max(1, n_) + kRedoPointsPer - 1) / kRedoPointsPer) * kRedoWordsPer;
    redo_bits_.alloc(nwords, st_);
    ck(cudaMemsetAsync(redo_bits_.get(), 0, nwords * sizeof(unsigned), st_), "zero redo bits");
    DBuf<unsigned> any(1, st_);
    ck(cudaMemsetAsync(any.get(), 0, sizeof(unsigned), st_), "zero any_sing");
    k_flux_weights<<<std::max(1, blocks), 256, 0, st_>>>(geo(), gas_.det_tol, w1_.get(), w2_.get(), sing_.get(),
                                                          psign_.get());
    ck(cudaGetLastError(), "k_flux_weights");
    k_flux_any_sing<<<std::max(1, blocks), 256, 0, st_>>>(geo(), sing_.get(), any.get());
    ck(cudaGetLastError(), "k_flux_any_sing");
    unsigned any_h = 0;
    ck(cudaMemcpyAsync(&any_h, any.get(), sizeof(unsigned), cudaMemcpyDeviceToHost, st_), "D2H any_sing");
    ck(cudaStreamSynchronize(st_), "weights");
    any_sing_ = any_h != 0;
    weights_ = true;
  }

  // Event record that also fires when captured into a graph (an external
  // event-record node); a plain captured cudaEventRecord only orders work.
  void record_ext(cudaEvent_t e) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    ck(cudaStreamIsCapturing(st_, &cs), "StreamIsCapturing");
    if (cs == cudaStreamCaptureStatusActive)
      ck(cudaEventRecordWithFlags(e, st_, cudaEventRecordExternal), "EventRecordExternal");
    else
      ck(cudaEventRecord(e, st_), "EventRecord");
  }

  // ---- building blocks of one iteration (also used by the multi-domain driver) ----
  // Derivative sweep s of the iteration (s = 0 stamps the iteration start).
  // list/nlist: a subset of the owned points (see Geo::list); only the
  // unrolled 8-point sweep and the staged flux kernel support it
  // (subsets_supported()).
  void launch_sweep(int a, int b, int s, const int* list = nullptr, int nlist = 0) {
    Geo g = geo();
    g.list = list;
    g.nlist = nlist;
    if (!list && tiles_) {
      launch_sweep_tiles(a, b, s, nullptr, ntiles_);
      return;
    }
    sweep_launch(strict_, g, q_[a].get(), dq_[b].get(), dq_[b ^ 1].get(), gas_, ctl_.get(),
                 s == 0 ? it0_.get() : nullptr, s, st_);
  }
  // Tiled sweep over the tiles tlist[0 .. ntl) (null: all ntl tiles).
  void launch_sweep_tiles(int a, int b, int s, const int* tlist, int ntl) {
    const Geo g = geo();
    if (strict_)
      sweep_tile_launch<true>(tile_p_, g, q_[a].get(), dq_[b].get(), dq_[b ^ 1].get(), gas_, ctl_.get(), s,
                              tplan_.get(), tslot_.get(), ntl, tlist, st_);
    else
      sweep_tile_launch<false>(tile_p_, g, q_[a].get(), dq_[b].get(), dq_[b ^ 1].get(), gas_, ctl_.get(), s,
                               tplan_.get(), tslot_.get(), ntl, tlist, st_);
  }
  bool tiled() const { return tiles_; }
  int tile_points() const { return tile_p_; }
  // Tile plan of the tiled sweep (geometry only, once per domain; uniform
  // 8-point stencils).  Returns the number of tiles that are staged.
  int ensure_tiles() {
    if (tiles_ || kfix_ != 8 || n_ <= 0 || sweep_tile_p() == 0) return tiles_staged_;
    tile_p_ = sweep_tile_p();
    ntiles_ = (n_ + tile_p_ - 1) / tile_p_;
    tplan_.alloc(static_cast<std::size_t>(ntiles_), st_);
    tslot_.alloc(static_cast<std::size_t>(n_) * 8, st_);
    if (tile_p_ == 64)
      k_tile_plan<64><<<ntiles_, 64, 0, st_>>>(geo(), TileShape<64>::smax, tplan_.get(), tslot_.get());
    else
      k_tile_plan<128><<<ntiles_, 128, 0, st_>>>(geo(), TileShape<128>::smax, tplan_.get(), tslot_.get());
    ck(cudaGetLastError(), "k_tile_plan");
    std::vector<TilePlan> h(static_cast<std::size_t>(ntiles_));
    ck(cudaMemcpyAsync(h.data(), tplan_.get(), h.size() * sizeof(TilePlan), cudaMemcpyDeviceToHost, st_), "D2H tiles");
    ck(cudaStreamSynchronize(st_), "tile plan");
    tiles_staged_ = static_cast<int>(std::count_if(h.begin(), h.end(), [](const TilePlan& t) { return t.nint > 0; }));
    trace("engine: tile plan");
    tiles_ = true;
    return tiles_staged_;
  }
  int tiles_staged() const { return tiles_staged_; }
  int tiles_total() const { return ntiles_; }
  bool subsets_supported() const {
    return !strict_ && weights_ && kmax_ <= 8 && kfix_ == 8 && flux_staged() && sweep_lanes() == 2 &&
           sweep_unrolled();
  }
  void launch_flux(int a, int b, bool stamp, const int* list = nullptr, int nlist = 0) {
    FluxArgs fa;
    fa.g = geo();
    fa.g.list = list;
    fa.g.nlist = nlist;
    fa.gas = gas_;
    fa.q = q_[a].get();
    fa.dq = dq_[b].get();
    fa.res = res_.get();
    fa.ctl = ctl_.get();
    fa.iter_t0 = stamp ? it0_.get() : nullptr;
    fa.kcap = kmax_;
    fa.stride = stride_;
    fa.mask = 0xF;
    fa.first = 1;
    if (!strict_ && weights_ && order_ == 1 && point_flux_enabled() && pf_.get() && kmax_ <= 8) {
      // first order: per-point split fluxes (owned and halo points), then the gather
      launch_pdl(k_point_flux, std::max(1, (n_loc_ + 255) / 256), 256, 0, st_, n_loc_,
                 static_cast<const D4*>(q_[a].get()), gas_, pf_.get(), pfvalid_.get(),
                 static_cast<const Ctl*>(ctl_.get()));
      const int groups = (n_ + 3) / 4;
      const int blocks = std::max(1, std::min((groups + 7) / 8, resident_blocks(k_flux1<2>, 7)));
      launch_pdl(k_flux1<2>, blocks, 256, 0, st_, fa, static_cast<const PointFlux*>(pf_.get()),
                 static_cast<const std::uint8_t*>(pfvalid_.get()), static_cast<const double2*>(w1_.get()),
                 static_cast<const double2*>(w2_.get()), static_cast<const std::uint8_t*>(sing_.get()),
                 static_cast<const std::uint8_t*>(psign_.get()));
    } else if (!strict_ && weights_) {
      const FluxRedo rd{redo_bits_.get()};
      flux_w_launch(fa, kmax_, w1_.get(), w2_.get(), sing_.get(), defer_run_ ? &rd : nullptr, st_);
    } else {
      flux_launch(W_, strict_, fa, smem_, st_);
    }
  }
  void launch_update(int a) {
    UpdateArgs ua;
    ua.g = geo();
    ua.gas = gas_;
    ua.q = q_[a].get();
    ua.res = res_.get();
    ua.prim = prim_.get();
    ua.q_next = q_[a ^ 1].get();
    ua.dt = dt_.get();
    ua.mag = mag_out_;
    ua.which = which_.get();
    ua.ctl = ctl_.get();
    ua.acc = strict_ ? nullptr : acc_.get();
    launch_pdl(k_update, update_blocks(), 256, 0, st_, ua);
  }
  void launch_residue() {
    if (!strict_) {
      launch_pdl(k_residue_exact, 1, 96, 0, st_, acc_tab_, acc_ndom_, n_res_, hist_.get(), it0_.get(), it1_.get(),
                 ctl_.get());
      return;
    }
    launch_pdl(k_tree_partial, 1 << d1_, kTreeThreads, 0, st_, static_cast<const double*>(mag_.get()), n_res_, d1_,
               pval_.get(), psz_.get(),
                                                      ctl_.get());
    launch_pdl(k_tree_final, 1, 1024, 0, st_, static_cast<const double*>(pval_.get()),
               static_cast<const long long*>(psz_.get()), d1_, n_res_, hist_.get(), it0_.get(), it1_.get(),
               ctl_.get());
  }
  // Halo gather of `planes` record planes per point (q: 1, dq: 2) from the
  // owners' buffers, as part of stage `sub` of the iteration (0: q; 1+s:
  // derivatives of sweep s).
  void launch_halo(D4* dst, int planes, const int* hdom, const int* hidx, const PeerTab& src, int sub,
                   bool skip_first = false) {
    const int nh = n_loc_ - n_;
    if (nh <= 0) return;
    k_halo<<<std::min((nh * planes + 255) / 256, 4096), 256, 0, st_>>>(dst, n_loc_, planes, n_, nh, hdom, hidx,
                                                                         src, ctl_.get(), sub, skip_first ? 1 : 0);
  }

  // One iteration starting at parity (a, b); `timed` brackets the first sweep
  // and the flux kernel with CUDA events (read back by last_event_ms()).
  void enqueue_iteration(int& a, int& b, bool timed) {
    if (order_ == 2) {
      for (int s = 0; s < inner_; ++s) {
        if (timed && s == 0) record_ext(kev_[0]);
        launch_sweep(a, b, s);
        if (timed && s == 0) record_ext(kev_[1]);
        b ^= 1;
      }
    }
    if (timed) record_ext(kev_[2]);
    launch_flux(a, b, order_ != 2);
    if (timed) record_ext(kev_[3]);
    launch_update(a);
    a ^= 1;
    launch_residue();
  }

  cudaGraphExec_t graph_for(int a, int b, int c) {
    const auto key = std::make_tuple(a, b, c);
    auto it = graphs_.find(key);
    if (it != graphs_.end()) return it->second;
    cudaGraph_t graph;
    ck(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal), "BeginCapture");
    int pa = a, pb = b;
    // no per-kernel event nodes (they lengthen the iteration); event_ms()
    // reads the events of step_flushed(kernel_events = true)
    for (int k = 0; k < c; ++k) enqueue_iteration(pa, pb, false);
    ck(cudaGetLastError(), "capture launches");
    ck(cudaStreamEndCapture(st_, &graph), "EndCapture");
    cudaGraphExec_t exec;
    ck(cudaGraphInstantiate(&exec, graph, 0), "GraphInstantiate");
    cudaGraphDestroy(graph);
    if (graph_upload()) ck(cudaGraphUpload(exec, st_), "GraphUpload");  // launch without a first-use upload
    graphs_[key] = exec;
    return exec;
  }

  void advance(int& a, int& b, int c) const {
    if (c & 1) a ^= 1;
    if (order_ == 2 && ((c * inner_) & 1)) b ^= 1;
  }

  // Iterations per graph launch for an n-iteration call: an even divisor of
  // n of at least chunk/2 when there is one (one graph, parities preserved,
  // fewer nodes to instantiate than chunk + remainder), else `chunk`.
  int run_chunk(int n) const {
    if (n <= chunk_) return n;
    for (int c = chunk_ & ~1; c >= std::max(2, chunk_ / 2); c -= 2)
      if (n % c == 0) return c;
    return chunk_;
  }

  void set_diag(int it) { k_set_diag<<<1, 1, 0, st_>>>(ctl_.get(), it); }

  // Runs up to n iterations; stops early on a device error.  Returns the
  // CUDA-event milliseconds around the enqueued work.
  double iterate(int n) {
    if (done_ + n > capacity_) raise(Status::argument, "session capacity exceeded");
    ck(cudaSetDevice(device_), "cudaSetDevice");
    set_diag(done_ + n - 1);
    const bool direct = !graphs_enabled();
    const int chunk = run_chunk(n);
    // First call with this chunking: the GPU runs the first chunk launched
    // kernel by kernel while the host instantiates the graphs for the rest
    // (instantiation ~0.35 ms at 160K points; later calls replay cached graphs).
    bool missing = false;
    {
      int a = a_, b = b_, left = n;
      while (left > 0) {
        const int c = std::min(chunk, left);
        missing = missing || !graphs_.count(std::make_tuple(a, b, c));
        advance(a, b, c);
        left -= c;
      }
    }
    const int pre = (!direct && missing && n > chunk) ? chunk : 0;
    ck(cudaEventRecord(ev0_, st_), "EventRecord");
    int left = n, issued = 0, waited = 0;
    bool failed = false;
    if (pre > 0) {
      for (int k = 0; k < pre; ++k) enqueue_iteration(a_, b_, false);
      left -= pre;
      failed = poll(issued, waited);
    }
    if (!direct) {
      int a = a_, b = b_, rest = left;
      while (rest > 0) {
        const int c = std::min(chunk, rest);
        graph_for(a, b, c);
        advance(a, b, c);
        rest -= c;
      }
    }
    trace("engine: graphs ready");
    while (left > 0 && !failed) {
      const int c = std::min(chunk, left);
      if (direct) {
        for (int k = 0; k < c; ++k) enqueue_iteration(a_, b_, k == c - 1);
      } else {
        ck(cudaGraphLaunch(graph_for(a_, b_, c), st_), "GraphLaunch");
        advance(a_, b_, c);
      }
      left -= c;
      if (left == 0) ck(cudaEventRecord(ev1_, st_), "EventRecord");
      failed = poll(issued, waited);
    }
    if (left > 0) ck(cudaEventRecord(ev1_, st_), "EventRecord");  // stopped early
    ck(cudaStreamSynchronize(st_), "iterate");
    float ms = 0.0f;
    ck(cudaEventElapsedTime(&ms, ev0_, ev1_), "EventElapsed");
    total_ms_ += ms;
    refresh_ctl();
    done_ = completed();
    return ms;
  }

  // One cold-L2 step (bench.py's timed steps): a graph of [L2 flush, event,
  // one iteration, event].  The events bracket the iteration inside the
  // graph, so the step's device time excludes the flush and the graph launch
  // (a one-iteration graph launched from the host costs ~20 us of GPU-side
  // start-up that back-to-back iterations never pay).
  // kernel_events: also bracket the first sweep and the flux kernel with
  // events (last_event_ms); event nodes between kernels lengthen the step.
  double step_flushed(bool kernel_events) {
    if (done_ + 1 > capacity_) raise(Status::argument, "session capacity exceeded");
    ck(cudaSetDevice(device_), "cudaSetDevice");
    if (!flush_.get()) flush_.alloc(static_cast<std::size_t>(48) << 20);  // 384 MB
    set_diag(done_);
    const auto key = std::make_tuple(a_, b_, kernel_events ? -2 : -1);
    auto it = graphs_.find(key);
    cudaGraphExec_t exec;
    if (it != graphs_.end()) {
      exec = it->second;
    } else {
      cudaGraph_t graph;
      ck(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal), "BeginCapture");
      k_flush<<<148 * 8, 256, 0, st_>>>(flush_.get(), static_cast<long long>(flush_.size()), 1.0);
      record_ext(ev0_);
      int pa = a_, pb = b_;
      enqueue_iteration(pa, pb, kernel_events);
      record_ext(ev1_);
      ck(cudaGetLastError(), "capture launches");
      ck(cudaStreamEndCapture(st_, &graph), "EndCapture");
      ck(cudaGraphInstantiate(&exec, graph, 0), "GraphInstantiate");
      cudaGraphDestroy(graph);
      graphs_[key] = exec;
    }
    ck(cudaGraphLaunch(exec, st_), "GraphLaunch");
    advance(a_, b_, 1);
    ck(cudaStreamSynchronize(st_), "step");
    float ms = 0.0f;
    ck(cudaEventElapsedTime(&ms, ev0_, ev1_), "EventElapsed");
    total_ms_ += ms;
    refresh_ctl();
    done_ = completed();
    return ms;
  }

  // Enqueues an async copy of the error word; waits on the oldest copy once
  // kPolls-1 are in flight.  True once an error has been observed.
  bool poll(int& issued, int& waited) {
    const int s = issued % kPolls;
    ck(cudaMemcpyAsync(hpoll_.get() + s, &shared_->err_stage, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                       st_),
       "poll copy");
    ck(cudaEventRecord(poll_ev_[s], st_), "poll event");
    ++issued;
    if (issued - waited >= kPolls - 1) {
      const int w = waited % kPolls;
      ck(cudaEventSynchronize(poll_ev_[w]), "poll sync");
      ++waited;
      return hpoll_.get()[w] != kNoErr;
    }
    return false;
  }

  void refresh_ctl() {
    ck(cudaMemcpyAsync(hctl_.get(), ctl_.get(), sizeof(Ctl), cudaMemcpyDeviceToHost, st_), "D2H ctl");
    ck(cudaMemcpyAsync(hsh_.get(), shared_, sizeof(Shared), cudaMemcpyDefault, st_), "D2H shared");
    ck(cudaStreamSynchronize(st_), "ctl");
  }

  bool failed() const { return hsh_.get()->err_stage != kNoErr; }
  // This domain's own failure record (valid after refresh_ctl).
  bool has_error() const { return hctl_.get()->err_stage != kNoErr; }
  unsigned long long err_stage() const { return hctl_.get()->err_stage; }
  unsigned long long err_key() const { return hctl_.get()->err_key; }
  int err_iter() const {
    const int spi = hctl_.get()->spi;
    const unsigned long long st = hctl_.get()->err_stage;
    return (st == kNoErr || spi <= 0) ? 0 : static_cast<int>(st / static_cast<unsigned>(spi));
  }
  const Shared& shared_host() const { return *hsh_.get(); }
  // Iterations completed without failure (valid after refresh_ctl): the
  // shared counter also advances past failed iterations, so it is capped at
  // the iteration of the run's first failing stage.
  int completed() const {
    const Shared& s = *hsh_.get();
    const int spi = hctl_.get()->spi;
    if (s.err_stage == kNoErr || spi <= 0) return s.iter;
    return std::min<long long>(s.iter, static_cast<long long>(s.err_stage / static_cast<unsigned>(spi)));
  }

  // CUDA-event times of the first sweep and the flux kernel of the last
  // iteration of the last graph replay (valid after iterate()).
  void last_event_ms(double& sweep_ms, double& flux_ms) const {
    float a = 0.0f, b = 0.0f;
    sweep_ms = flux_ms = 0.0;
    if (order_ == 2 && cudaEventElapsedTime(&a, kev_[0], kev_[1]) == cudaSuccess) sweep_ms = a;
    if (cudaEventElapsedTime(&b, kev_[2], kev_[3]) == cudaSuccess) flux_ms = b;
    cudaGetLastError();
  }

  // Overwrites 384 MB (> the 126 MB L2) on this domain's stream.  Stream
  // ordered, no host wait: the next step's kernels are queued behind it, so a
  // timed step starts on a cold L2 without an idle GPU waiting for its launch.
  void flush_l2() {
    if (!flush_.get()) flush_.alloc(static_cast<std::size_t>(48) << 20);  // 384 MB
    k_flush<<<148 * 8, 256, 0, st_>>>(flush_.get(), static_cast<long long>(flush_.size()), 1.0);
    ck(cudaGetLastError(), "flush");
  }

  // q / published dq read by 0-based iteration t (parities start at 0 per run).
  const D4* q_of_iter(int t) const { return q_[t & 1].get(); }
  const D4* dq_of_flux(int t) const { return order_ == 2 ? dq_[((t + 1) * inner_) & 1].get() : dq_[0].get(); }
  Fault fault_in_run(int local) {
    const int t = std::max(0, std::min(err_iter(), std::max(0, capacity_ - 1)));
    return fault(true, q_of_iter(t), dq_of_flux(t), local);
  }
  Fault fault_in_run() { return fault_in_run(-1); }

  // Builds the reference-format message for the recorded failure; `local` is
  // the failing point's local index (-1: the key's global id is local).
  Fault fault(bool with_iteration, const D4* qsrc, const D4* dqsrc, int local = -1) {
    return fault_for(err_key(), err_iter(), with_iteration, qsrc, dqsrc, local);
  }
  // Message for `key` (another domain's record when this domain owns the point).
  Fault fault_for(unsigned long long key, int err_it, bool with_iteration, const D4* qsrc, const D4* dqsrc,
                  int local = -1) {
    const unsigned phase = key_phase(key);
    const long long point = key_point(key);
    const int iter = err_it + 1;
    if (phase == PH_RESIDUE)
      return Fault(Status::positivity, "solver diverged at iteration " + itos(iter) + " (non-finite residue)");
    if (phase == PH_STALL) return Fault(Status::argument, "peer rank stopped making progress (wait timed out)");
    const int li = local >= 0 ? local : local_of(point);
    if (strict_)
      k_diagnose<true><<<1, 1, 0, st_>>>(geo(), qsrc, dqsrc, prim_.get(), dt_.get(), which_.get(), gas_, key, li,
                                         diag_.get());
    else
      k_diagnose<false><<<1, 1, 0, st_>>>(geo(), qsrc, dqsrc, prim_.get(), dt_.get(), which_.get(), gas_, key, li,
                                          diag_.get());
    double d[6];
    ck(cudaMemcpyAsync(d, diag_.get(), sizeof d, cudaMemcpyDeviceToHost, st_), "D2H diag");
    ck(cudaStreamSynchronize(st_), "diagnose");
    Status code = Status::positivity;
    std::string msg;
    if (phase == PH_QVAR) {
      msg = "invalid primitive state: rho=" + fmt_f(d[1]) + " p=" + fmt_f(d[2]);
    } else if (phase == PH_SWEEP) {
      code = Status::singular;
      msg = "full stencil of point " + itos(point) + ": singular least-squares stencil (det=" + fmt_f(d[1]) +
            ", n=" + itos(static_cast<long long>(d[2])) + ")";
    } else if (phase == PH_FLUX) {
      if (d[0] == 2.0) {
        code = Status::singular;
        msg = "split stencil of point " + itos(point) + ": singular least-squares stencil (det=" + fmt_f(d[1]) +
              ", n=" + itos(static_cast<long long>(d[2])) + ")";
      } else if (d[0] == 0.0) {
        msg = "flux reconstruction failed on edge (" + itos(point) + ", " + itos(static_cast<long long>(d[3])) +
              "): q-state with q3 >= 0 (q3=" + fmt_f(d[1]) + ")";
      } else {
        msg = "invalid primitive state: rho=" + fmt_f(d[1]) + " p=" + fmt_f(d[2]);
      }
    } else {  // PH_UPDATE
      msg = "state update lost positivity at point " + itos(point) + ": conserved state with " +
            (d[0] == 0.0 ? "non-positive density " : "non-positive pressure ") + fmt_f(d[1]);
    }
    if (with_iteration) msg = "iteration " + itos(iter) + ": " + msg;
    return Fault(code, msg);
  }

  // ---- accessors for the run/session drivers ----
  int n() const { return n_; }
  int done() const { return done_; }
  void set_done(int d) { done_ = d; }
  double total_ms() const { return total_ms_; }
  void add_ms(double ms) { total_ms_ += ms; }
  cudaStream_t stream() const { return st_; }
  const D4* q_read_last() const { return q_of_iter(std::max(0, done_ - 1)); }
  const D4* q_buf(int k) const { return q_[k].get(); }
  D4* q_buf(int k) { return q_[k].get(); }
  D4* dq_buf(int k) { return dq_[k].get(); }
  const D4* dq_cur() const { return done_ > 0 ? dq_of_flux(done_ - 1) : dq_[0].get(); }
  D4* prim() { return prim_.get(); }
  D4* res() { return res_.get(); }
  double* dt() { return dt_.get(); }
  double* mind() { return mind_.get(); }
  double* which() { return which_.get(); }
  Ctl* dctl() { return ctl_.get(); }
  const Gas& gas() const { return gas_; }
  int width() const { return W_; }
  int kmax() const { return kmax_; }
  std::size_t smem() const { return smem_; }
  void set_strict(bool s) { strict_ = s; }
  // residual_mode=split4: flux failures ordered direction-first (err_key).
  void set_split4(bool s) { split4_ = s; }
  int order() const { return order_; }
  int inner() const { return inner_; }

  std::vector<double> residues() const {
    std::vector<double> out(static_cast<std::size_t>(done_));
    if (done_ > 0)
      ck(cudaMemcpy(out.data(), hist_.get(), done_ * sizeof(double), cudaMemcpyDeviceToHost), "D2H hist");
    return out;
  }
  std::vector<double> wall_ms() const {
    std::vector<unsigned long long> t0(done_), t1(done_);
    std::vector<double> out(static_cast<std::size_t>(done_));
    if (done_ > 0) {
      ck(cudaMemcpy(t0.data(), it0_.get(), done_ * sizeof(unsigned long long), cudaMemcpyDeviceToHost), "D2H t0");
      ck(cudaMemcpy(t1.data(), it1_.get(), done_ * sizeof(unsigned long long), cudaMemcpyDeviceToHost), "D2H t1");
      for (int k = 0; k < done_; ++k) out[k] = t1[k] >= t0[k] ? (t1[k] - t0[k]) * 1e-6 : 0.0;
    }
    return out;
  }
  std::vector<KernelTime> kernel_times() const {
    // Device timer slots -> the reference's timer rows (runtime.cpp:144-190,
    // :257): q_variables, q_derivatives (all sweeps), flux_residual (or its
    // four split4 passes), timestep, state_update, residue.  Two rows are
    // attributed rather than timed separately: the time step is fused into
    // k_update (their time is split in proportion to the reference kernels'
    // algorithmic bytes, 97 : 105 B/pt), and the four split4
    // directions are one fused flux kernel (a quarter each; summarize() adds
    // the aggregate row as make_bench_report does, bench.cpp:72-99).
    double secs[5] = {0, 0, 0, 0, 0};
    std::int64_t cnt[5] = {0, 0, 0, 0, 0};
    for (int k = 0; k < KT_COUNT; ++k) {
      const KTimer& t = hctl_.get()->kt[k];
      const int r = k == KT_QVAR ? 0 : (k < KT_FLUX ? 1 : (k == KT_FLUX ? 2 : (k == KT_UPDATE ? 3 : 4)));
      secs[r] += t.total_ns * 1e-9;
      cnt[r] += static_cast<std::int64_t>(t.launches);
    }
    std::vector<KernelTime> out;
    if (cnt[0] > 0) out.push_back({"q_variables", secs[0], cnt[0]});
    if (cnt[1] > 0) out.push_back({"q_derivatives", secs[1], cnt[1]});
    if (cnt[2] > 0) {
      if (split4_) {
        for (const char* nm : {"flux_residual_xplus", "flux_residual_xminus", "flux_residual_yplus",
                               "flux_residual_yminus"})
          out.push_back({nm, secs[2] * 0.25, cnt[2]});
      } else {
        out.push_back({"flux_residual", secs[2], cnt[2]});
      }
    }
    if (cnt[3] > 0) {
      constexpr double kTimestepShare = 97.0 / (97.0 + 105.0);
      out.push_back({"timestep", secs[3] * kTimestepShare, cnt[3]});
      out.push_back({"state_update", secs[3] - secs[3] * kTimestepShare, cnt[3]});
    }
    if (cnt[4] > 0) out.push_back({"residue", secs[4], cnt[4]});
    static const bool per_sweep = std::getenv("LSKUM_KT_SWEEPS") != nullptr;  // probes: one line per sweep
    static const char* sweeps[] = {"sweep0", "sweep1", "sweep2", "sweep3", "sweep4", "sweep5", "sweep6", "sweep7+"};
    for (int k = KT_SWEEP; per_sweep && k < KT_FLUX; ++k) {
      const KTimer& t = hctl_.get()->kt[k];
      if (t.launches) out.push_back({sweeps[k - KT_SWEEP], t.total_ns * 1e-9, static_cast<std::int64_t>(t.launches)});
    }
    return out;
  }

 private:
  static constexpr int kPolls = 4;
  // Owns the stream; declared before the buffers so it is destroyed after them
  // (their stream-ordered frees are enqueued on it).
  struct StreamHolder {
    cudaStream_t st = nullptr;
    explicit StreamHolder(int device) {
      ck(cudaSetDevice(device), "cudaSetDevice");
      ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
    }
    ~StreamHolder() {
      if (st) {
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
      }
    }
  };
  int n_ = 0, n_loc_ = 0, device_ = 0;
  bool ipc_ = false;
  long long n_res_ = 0;
  StreamHolder stream_holder_;
  cudaStream_t st_ = nullptr;
  cudaEvent_t ev0_ = nullptr, ev1_ = nullptr, poll_ev_[kPolls] = {}, kev_[4] = {};
  DBuf<double> flush_;
  Gas gas_{};
  int kmax_ = 1, kfix_ = 0, W_ = 8, d1_ = 0;
  std::size_t smem_ = 0;
  int stride_ = 0;
  std::vector<int> gid_host_;
  std::vector<std::uint16_t> part_host_;
  DBuf<double2> xy_, nrm_;
  DBuf<std::uint8_t> kind_;
  DBuf<std::uint16_t> part_;
  DBuf<int> off_, nbr_, gid_;
  DBuf<double> mind_, dt_, which_, mag_, pval_, hist_, diag_;
  double* mag_out_ = nullptr;
  DBuf<long long> psz_;
  DBuf<unsigned long long> acc_;
  AccTab acc_tab_{};
  int acc_ndom_ = 1;
  DBuf<D4> prim_, q_[2], dq_[2], res_;
  std::int64_t nnz_ = 0;
  DBuf<double2> w1_, w2_;       // least-squares weights of the split stencils (fast mode)
  DBuf<TilePlan> tplan_;        // tile plan of the tiled sweep (tiles.cuh)
  DBuf<std::uint16_t> tslot_;
  int ntiles_ = 0, tiles_staged_ = 0, tile_p_ = 128;
  unsigned long long zero_pairs_ = 0;  // pairs with dx == 0 or dy == 0 (non-outer points)
  cudaEvent_t ev_trace_ = nullptr;     // LSKUM_TRACE: device-time reference of the screening
  bool tiles_ = false;
  DBuf<PointFlux> pf_;           // first order: split fluxes per point (owned + halo)
  DBuf<std::uint8_t> psign_;     // first order: half-stencil signs / zero offset per pair
  DBuf<std::uint8_t> pfvalid_;
  DBuf<std::uint8_t> sing_;     // first singular split direction per point
  DBuf<unsigned> redo_bits_;       // flux points whose evaluation took a rare path (k_flux_redo)
  bool any_sing_ = false;          // a live point has a singular split stencil: no deferral
  bool defer_run_ = false;         // this run defers the flux's rare paths (probe_defer)
  bool weights_ = false;
  DBuf<Ctl> ctl_;
  DBuf<Shared> sh_;
  Shared* shared_ = nullptr;
  DBuf<unsigned long long> it0_, it1_;
  HBuf<unsigned long long> hpoll_;
  HBuf<Ctl> hctl_;
  HBuf<Shared> hsh_;
  int capacity_ = 1;
  int order_ = 2, inner_ = 3, chunk_ = 16;
  bool strict_ = false;
  bool split4_ = false;
  int a_ = 0, b_ = 0, done_ = 0;
  double total_ms_ = 0.0;
  std::map<std::tuple<int, int, int>, cudaGraphExec_t> graphs_;
};

// ===========================================================================
namespace {

// A single-device domain of the whole cloud in the numbering `loc` chooses:
// the cloud's own order, or its locality permutation (reorder.cpp).
std::unique_ptr<Domain> cloud_domain(const PointSet& ps, const std::shared_ptr<const Locality>& loc,
                                     const std::vector<std::uint16_t>& part_of, int device, double gamma,
                                     double cfl, double det_tol, int capacity) {
  if (loc->order.empty())
    return std::make_unique<Domain>(view_of(ps, part_of), device, gamma, cfl, det_tol, capacity);
  const LocalGeom g = permuted_geom(ps, loc->order, part_of);
  trace("engine: locality permutation");
  return std::make_unique<Domain>(view_of(g), device, gamma, cfl, det_tol, capacity);
}

std::shared_ptr<const Locality> locality_of(const PointSet& ps, int reorder) {
  cloud_locality(ps, reorder);
  return ps.locality;
}

std::unique_ptr<Domain> open_domain(PointSet& ps, const EngineSpec& spec, int capacity) {
  auto d = cloud_domain(ps, locality_of(ps, spec.reorder), spec.part_of, spec.device, spec.gamma, spec.cfl,
                        spec.det_tol, capacity);
  trace("engine: geometry uploaded");
  d->upload(ps.fields, false);
  trace("engine: state uploaded");
  d->set_split4(spec.split4);
  d->begin_run(spec.order, spec.inner, spec.fp_mode, spec.chunk);
  return d;
}

// The cloud's cached single-device domain (PointSet::engine_cache), created on
// first use and reconfigured for later runs: repeated lskum_run calls on one
// cloud keep geometry, split-stencil weights, buffers and captured graphs
// resident instead of re-uploading and re-capturing them.
struct EngineCache {
  std::unique_ptr<Domain> dom;
  int device = -1;
  std::shared_ptr<const Locality> loc;  // device numbering the domain was built with
};

// The cached domain is reusable when it was built in the same numbering.
bool same_numbering(const EngineCache& c, const std::shared_ptr<const Locality>& loc) {
  return c.loc == loc || (c.loc && c.loc->order.empty() && loc->order.empty());
}


Domain& cached_domain(PointSet& ps, const EngineSpec& spec, int capacity) {
  auto* c = static_cast<EngineCache*>(ps.engine_cache.get());
  const std::shared_ptr<const Locality> loc = locality_of(ps, spec.reorder);
  if (c && c->device == spec.device && c->dom && same_numbering(*c, loc)) {
    c->dom->reconfigure(spec.gamma, spec.cfl, spec.det_tol, spec.part_of.empty() ? nullptr : spec.part_of.data(),
                        capacity);
    trace("engine: cached domain reconfigured");
  } else {
    ps.engine_cache.reset();  // release the old device's buffers first
    auto fresh = std::make_shared<EngineCache>();
    fresh->device = spec.device;
    fresh->loc = loc;
    fresh->dom = cloud_domain(ps, loc, spec.part_of, spec.device, spec.gamma, spec.cfl, spec.det_tol, capacity);
    trace("engine: geometry uploaded");
    ps.engine_cache = fresh;
    c = fresh.get();
  }
  Domain& d = *c->dom;
  if (spec.fs_device) d.fill_prim(spec.fs_prim);
  else d.upload(ps.fields, false);
  trace("engine: state uploaded");
  d.set_split4(spec.split4);
  d.begin_run(spec.order, spec.inner, spec.fp_mode, spec.chunk);
  return d;
}

}  // namespace

// lskum_run's stencil screening on the device: uploads the
// geometry into the cloud's resident domain (which the run then reuses) and
// screens it there.  The report is cached on the cloud like the host one.
Screening engine_screen(PointSet& ps, int device, double gamma, double cfl, int capacity, int reorder) {
  auto* c = static_cast<EngineCache*>(ps.engine_cache.get());
  const std::shared_ptr<const Locality> loc = locality_of(ps, reorder);
  if (!(c && c->device == device && c->dom && same_numbering(*c, loc))) {
    ps.engine_cache.reset();
    auto fresh = std::make_shared<EngineCache>();
    fresh->device = device;
    fresh->loc = loc;
    fresh->dom = cloud_domain(ps, loc, {}, device, gamma, cfl, 0.0, std::max(1, capacity));
    trace("engine: geometry uploaded");
    ps.engine_cache = fresh;
    c = fresh.get();
  }
  Screening scr = c->dom->screen();
  trace("engine: screened on device");
  return scr;
}

void engine_prescreen(PointSet& ps, const Settings& s) {
  if (ps.screening || s.gpus > 1) return;
  ps.screening = std::make_shared<const Screening>(engine_screen(ps, s.device, s.gamma, s.cfl, s.iters, s.reorder));
}

namespace {

// Copy-back of the reference's end-of-run store: prim (final), q of the last
// iteration, published qx/qy, flux_res and delta_t of the last iteration.
void copy_back(Domain& d, PointSet& ps, bool* written = nullptr) {
  const bool with_q = d.done() > 0;
  d.download(ps.fields, with_q, d.q_read_last(), d.dq_cur());
  if (written) *written = true;
}

}  // namespace

RunRecord engine_run(PointSet& ps, const EngineSpec& spec) {
  RunRecord rec;
  if (spec.iters == 0) {
    // No phase runs: only the once-per-run zeroing (runtime.cpp:216-224).
    for (std::int32_t i = 0; i < ps.n(); ++i) {
      for (int c = 0; c < 4; ++c) {
        ps.fields.at(i, slot::qx + c) = 0.0;
        ps.fields.at(i, slot::qy + c) = 0.0;
        ps.fields.at(i, slot::res + c) = 0.0;
      }
      ps.fields.at(i, slot::dt) = 0.0;
    }
    return rec;
  }
  Domain* d = nullptr;
  try {
    d = &cached_domain(ps, spec, spec.iters);
  } catch (const Fault&) {
    throw;
  } catch (...) {
    ps.engine_cache.reset();  // a device-side failure leaves the cached domain unusable
    throw;
  }
  trace("engine: domain open");
  if (d->failed()) {  // first q_variables
    copy_back(*d, ps, spec.store_written);
    throw d->fault_in_run();
  }
  d->iterate(spec.iters);
  trace("engine: iterated");
  if (d->failed()) {
    Fault f = d->fault_in_run();
    copy_back(*d, ps, spec.store_written);
    rec.abort_iteration = d->err_iter() + 1;
    throw f;
  }
  copy_back(*d, ps, spec.store_written);
  trace("engine: copied back");
  rec.iterations = d->done();
  rec.residue = d->residues();
  rec.wall_ms = d->wall_ms();
  rec.kernels = d->kernel_times();
  rec.total_seconds = d->total_ms() * 1e-3;
  const double first = rec.residue.empty() ? 0.0 : rec.residue.front();
  for (double r : rec.residue)
    rec.log10_rel.push_back((first > 0.0 && r > 0.0) ? std::log10(r / first) : 0.0);
  return rec;
}

// ===========================================================================
// Multi-domain run.  Per iteration, on every domain d (own stream, own device):
//   [t>0] wait residue(t-1) on the root   (iteration counter + residue buffer)
//   [t>0] gather q halo from owners        (after their update(t-1))
//   sweeps s: sweep -> gather dq halo       (after the owners' sweep s; a sweep
//             that overwrites a buffer readers gathered two stages ago waits
//             for their gather)
//   flux -> update (residue summands into the root's global-id array)
// and on the root: wait every update(t) -> midpoint-tree residue.
// Stencils keep their global order in local ids, so all per-point arithmetic
// and the residue tree are identical to the single-domain run.
namespace {

class EventRing {
 public:
  EventRing() = default;
  EventRing(const EventRing&) = delete;
  EventRing& operator=(const EventRing&) = delete;
  void create(int device, int n) {
    ck(cudaSetDevice(device), "cudaSetDevice");
    ev_.resize(static_cast<std::size_t>(n));
    for (auto& e : ev_) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
  }
  ~EventRing() {
    for (auto& e : ev_) cudaEventDestroy(e);
  }
  cudaEvent_t operator[](int k) const { return ev_[static_cast<std::size_t>(k) % ev_.size()]; }

 private:
  std::vector<cudaEvent_t> ev_;
};

void enable_peers(const std::vector<int>& devs) {
  for (int a : devs)
    for (int b : devs) {
      if (a == b) continue;
      int can = 0;
      ck(cudaDeviceCanAccessPeer(&can, a, b), "cudaDeviceCanAccessPeer");
      if (!can) raise(Status::argument, "devices " + itos(a) + " and " + itos(b) + " cannot access each other's memory");
      ck(cudaSetDevice(a), "cudaSetDevice");
      const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else ck(e, "cudaDeviceEnablePeerAccess");
    }
}


}  // namespace

class MultiRun {
 public:
  MultiRun(PointSet& ps, const EngineSpec& spec, const std::vector<LocalGeom>& geoms, int capacity)
      : ps_(ps), spec_(spec), geoms_(geoms), P_(static_cast<int>(geoms.size())) {
    if (P_ < 1 || P_ > kMaxDomains) raise(Status::config, "gpus must lie in [1, " + itos(kMaxDomains) + "]");
    const int ndev = engine_device_count();
    if (ndev < 1) raise(Status::argument, "no CUDA device");
    dev_.resize(static_cast<std::size_t>(P_));
    for (int d = 0; d < P_; ++d) dev_[d] = (spec.device + d) % ndev;
    {
      std::vector<int> uniq(dev_);
      std::sort(uniq.begin(), uniq.end());
      uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
      enable_peers(uniq);
    }
    src_.resize(P_);
    readers_.resize(P_);
    for (int d = 0; d < P_; ++d) {
      std::vector<int> sv(geoms[d].halo_dom.begin(), geoms[d].halo_dom.end());
      std::sort(sv.begin(), sv.end());
      sv.erase(std::unique(sv.begin(), sv.end()), sv.end());
      src_[d] = sv;
      for (int o : sv) readers_[o].push_back(d);
    }
    dom_.resize(P_);
    hdom_.resize(P_);
    hidx_.resize(P_);
    for (int d = 0; d < P_; ++d) {
      dom_[d] = std::make_unique<Domain>(view_of(geoms[d]), dev_[d], spec.gamma, spec.cfl, spec.det_tol, capacity);
      const std::size_t nh = geoms[d].halo_dom.size();
      ck(cudaSetDevice(dev_[d]), "cudaSetDevice");
      hdom_[d] = std::make_unique<DBuf<int>>(std::max<std::size_t>(1, nh));
      hidx_[d] = std::make_unique<DBuf<int>>(std::max<std::size_t>(1, nh));
      if (nh) {
        ck(cudaMemcpy(hdom_[d]->get(), geoms[d].halo_dom.data(), nh * sizeof(int), cudaMemcpyHostToDevice), "H2D hdom");
        ck(cudaMemcpy(hidx_[d]->get(), geoms[d].halo_idx.data(), nh * sizeof(int), cudaMemcpyHostToDevice), "H2D hidx");
      }
    }
    Domain& r = root();
    r.set_residue_size(ps.n());
    AccTab tab{};
    for (int d = 0; d < P_; ++d) tab.p[d] = dom_[d]->acc_buf();
    r.use_acc_tab(tab, P_);  // exact residue: the root sums every domain's digits
    for (int d = 1; d < P_; ++d) {
      dom_[d]->use_shared(r.shared());
      dom_[d]->use_mag(r.mag_buf());
    }
    for (int d = 0; d < P_; ++d) dom_[d]->upload(ps.fields, false);
    for (int d = 0; d < P_; ++d) dom_[d]->set_split4(spec.split4);
    r.reset_run(spec.order, spec.inner, spec.fp_mode, spec.chunk, true);
    ck(cudaStreamSynchronize(r.stream()), "root init");  // shared word initialised before others use it
    for (int d = 1; d < P_; ++d) dom_[d]->reset_run(spec.order, spec.inner, spec.fp_mode, spec.chunk, false);
    for (int d = 0; d < P_; ++d) dom_[d]->first_q();
    for (int d = 0; d < P_; ++d) ck(cudaStreamSynchronize(dom_[d]->stream()), "first q");
    ev_sw_ = std::vector<EventRing>(P_);
    ev_dqh_ = std::vector<EventRing>(P_);
    ev_upd_ = std::vector<EventRing>(P_);
    for (int d = 0; d < P_; ++d) {
      ev_sw_[d].create(dev_[d], 4);
      ev_dqh_[d].create(dev_[d], 4);
      ev_upd_[d].create(dev_[d], 2);
    }
    ev_res_.create(dev_[0], 2);
    ck(cudaSetDevice(dev_[0]), "cudaSetDevice");
    ck(cudaEventCreate(&t0_), "ev");
    ck(cudaEventCreate(&t1_), "ev");
    for (auto& e : kev_) ck(cudaEventCreate(&e), "ev");
    r.refresh_ctl();
  }
  ~MultiRun() {
    for (int d = 0; d < P_; ++d)
      if (dom_[d]) cudaStreamSynchronize(dom_[d]->stream());
    cudaEventDestroy(t0_);
    cudaEventDestroy(t1_);
    for (auto& e : kev_) cudaEventDestroy(e);
  }

  Domain& root() { return *dom_[0]; }
  void tiles(int* staged, int* total) const {
    for (const auto& d : dom_) {
      *staged += d->tiles_staged();
      *total += d->tiles_total();
    }
  }
  int launches_per_iter() const {
    return P_ * ((spec_.order == 2 ? 2 * spec_.inner : 0) + 2 + dom_[0]->flux_launches()) +
           (spec_.fp_mode == 1 ? 2 : 1);
  }

  // Enqueues n more iterations (stopping early on an error); returns the
  // CUDA-event ms on the root stream, which waits for every domain.
  double iterate(int n) {
    Domain& r = root();
    for (int d = 0; d < P_; ++d) {
      ck(cudaSetDevice(dev_[d]), "cudaSetDevice");
      dom_[d]->set_diag(t_ + n - 1);
    }
    ck(cudaSetDevice(dev_[0]), "cudaSetDevice");
    ck(cudaEventRecord(t0_, r.stream()), "EventRecord");
    for (int d = 1; d < P_; ++d) wait(d, t0_);  // all domains start after the stamp
    int issued = 0, waited = 0;
    bool failed = false;
    const int end = t_ + n;
    for (; t_ < end && !failed; ++t_) {
      failed = enqueue(t_, t_ == end - 1) || false;
      failed = r.poll(issued, waited);
    }
    ck(cudaSetDevice(dev_[0]), "cudaSetDevice");
    ck(cudaEventRecord(t1_, r.stream()), "EventRecord");
    for (int d = 0; d < P_; ++d) ck(cudaStreamSynchronize(dom_[d]->stream()), "multi-domain iterate");
    float ms = 0.0f;
    ck(cudaEventElapsedTime(&ms, t0_, t1_), "EventElapsed");
    r.refresh_ctl();
    const int done = r.completed();
    for (int d = 0; d < P_; ++d) dom_[d]->set_done(done);
    r.add_ms(ms);
    return ms;
  }

  bool failed() { return root().failed(); }

  // The run's failure: min (stage, key) over the domains' own records; the
  // message is built by the domain owning the failing point.
  int first_failing_domain() {
    int best = -1;
    for (int d = 0; d < P_; ++d) {
      dom_[d]->refresh_ctl();
      if (!dom_[d]->has_error()) continue;
      if (best < 0 || std::make_pair(dom_[d]->err_stage(), dom_[d]->err_key()) <
                          std::make_pair(dom_[best]->err_stage(), dom_[best]->err_key()))
        best = d;
    }
    return best;
  }
  int abort_iteration() {
    const int d = first_failing_domain();
    return d < 0 ? 0 : dom_[d]->err_iter() + 1;
  }
  Fault fault() {
    const int rec = first_failing_domain();
    if (rec < 0) return Fault(Status::argument, "multi-domain run failed without a failure record");
    const unsigned long long key = dom_[rec]->err_key();
    const int g = static_cast<int>(key_point(key));
    int owner = rec, local = -1;
    if (key_phase(key) < PH_RESIDUE) {
      for (int d = 0; d < P_; ++d) {
        const auto& own = geoms_[d].gid;
        const auto it = std::lower_bound(own.begin(), own.begin() + geoms_[d].n_own, g);
        if (it != own.begin() + geoms_[d].n_own && *it == g) {
          owner = d;
          local = static_cast<int>(it - own.begin());
          break;
        }
      }
    }
    Domain& o = *dom_[owner];
    const int t = std::max(0, dom_[rec]->err_iter());
    return o.fault_for(key, dom_[rec]->err_iter(), true, o.q_of_iter(t), o.dq_of_flux(t), local);
  }

  void download() {
    for (int d = 0; d < P_; ++d) copy_back(*dom_[d], ps_);
  }

  void flush_l2() {
    for (int d = 0; d < P_; ++d) dom_[d]->flush_l2();
  }

  void last_event_ms(double& sweep_ms, double& flux_ms) const {
    float a = 0.0f, b = 0.0f;
    sweep_ms = flux_ms = 0.0;
    if (spec_.order == 2 && cudaEventElapsedTime(&a, kev_[0], kev_[1]) == cudaSuccess) sweep_ms = a;
    if (cudaEventElapsedTime(&b, kev_[2], kev_[3]) == cudaSuccess) flux_ms = b;
    cudaGetLastError();
  }

 private:
  void wait(int d, cudaEvent_t e) { ck(cudaStreamWaitEvent(dom_[d]->stream(), e, 0), "StreamWaitEvent"); }
  PeerTab peers_q(int a) const {
    PeerTab tb{};
    for (int o = 0; o < P_; ++o) {
      tb.base[o] = dom_[o]->q_buf(a);
      tb.ps[o] = dom_[o]->n_loc();
    }
    return tb;
  }
  PeerTab peers_dq(int b) const {
    PeerTab tb{};
    for (int o = 0; o < P_; ++o) {
      tb.base[o] = dom_[o]->dq_buf(b);
      tb.ps[o] = dom_[o]->n_loc();
    }
    return tb;
  }

  bool enqueue(int t, bool timed) {
    const int a = t & 1;
    Domain& r = root();
    if (t > 0) {
      for (int d = 0; d < P_; ++d) {
        ck(cudaSetDevice(dev_[d]), "cudaSetDevice");
        for (int o : src_[d]) wait(d, ev_upd_[o][t - 1]);
        dom_[d]->launch_halo(dom_[d]->q_buf(a), 1, hdom_[d]->get(), hidx_[d]->get(), peers_q(a), 0);
      }
    }
    int bfin = 0;
    if (spec_.order == 2) {
      for (int s = 0; s < spec_.inner; ++s) {
        const int k = t * spec_.inner + s, b = k & 1;
        for (int d = 0; d < P_; ++d) {
          ck(cudaSetDevice(dev_[d]), "cudaSetDevice");
          if (s >= 2)
            for (int rd : readers_[d]) wait(d, ev_dqh_[rd][k - 2]);
          if (timed && s == 0 && d == 0) ck(cudaEventRecord(kev_[0], r.stream()), "EventRecord");
          dom_[d]->launch_sweep(a, b, s);
          if (timed && s == 0 && d == 0) ck(cudaEventRecord(kev_[1], r.stream()), "EventRecord");
          ck(cudaEventRecord(ev_sw_[d][k], dom_[d]->stream()), "EventRecord");
        }
        for (int d = 0; d < P_; ++d) {
          ck(cudaSetDevice(dev_[d]), "cudaSetDevice");
          for (int o : src_[d]) wait(d, ev_sw_[o][k]);
          dom_[d]->launch_halo(dom_[d]->dq_buf(b ^ 1), 2, hdom_[d]->get(), hidx_[d]->get(), peers_dq(b ^ 1), 1 + s);
          ck(cudaEventRecord(ev_dqh_[d][k], dom_[d]->stream()), "EventRecord");
        }
      }
      bfin = ((t + 1) * spec_.inner) & 1;
    }
    for (int d = 0; d < P_; ++d) {
      ck(cudaSetDevice(dev_[d]), "cudaSetDevice");
      if (timed && d == 0) ck(cudaEventRecord(kev_[2], r.stream()), "EventRecord");
      dom_[d]->launch_flux(a, bfin, spec_.order != 2);
      if (timed && d == 0) ck(cudaEventRecord(kev_[3], r.stream()), "EventRecord");
      // the root's residue of t-1 has read what update(t) overwrites (the
      // residue summands, or the accumulator of iteration t+1)
      if (t > 0) wait(d, ev_res_[t - 1]);
      dom_[d]->launch_update(a);
      ck(cudaEventRecord(ev_upd_[d][t], dom_[d]->stream()), "EventRecord");
    }
    ck(cudaSetDevice(dev_[0]), "cudaSetDevice");
    for (int d = 1; d < P_; ++d) wait(0, ev_upd_[d][t]);
    r.launch_residue();
    ck(cudaEventRecord(ev_res_[t], r.stream()), "EventRecord");
    ck(cudaGetLastError(), "multi-domain launches");
    return false;
  }

  PointSet& ps_;
  EngineSpec spec_;
  std::vector<LocalGeom> geoms_;
  int P_ = 0;
  std::vector<int> dev_;
  std::vector<std::vector<int>> src_, readers_;
  std::vector<std::unique_ptr<Domain>> dom_;
  std::vector<std::unique_ptr<DBuf<int>>> hdom_, hidx_;
  std::vector<EventRing> ev_sw_, ev_dqh_, ev_upd_;
  EventRing ev_res_;
  cudaEvent_t t0_ = nullptr, t1_ = nullptr, kev_[4] = {};
  int t_ = 0;
};

// ===========================================================================
// One process per GPU (torchrun ranks).  Every rank derives the same RCB
// decomposition and builds only its own domain.  Peers' q/dq buffers, the
// root's shared control word and residue array are mapped with CUDA IPC; the
// stage ordering that MultiRun gets from cross-stream events comes from
// monotonic 64-bit progress counters written with release semantics by
// k_signal and awaited with acquire loads by k_wait (device-side, so no host
// ordering between processes is needed).
namespace {

enum : int { FL_SW = 0, FL_DQH = 1, FL_UPD = 2, FL_RES = 3, FL_COUNT = 4 };

struct WaitList {
  const unsigned long long* ptr[kMaxDomains];
  int n;
};

// Progress counters: values are derived on the device from this domain's
// iteration index t (iter_of): value = t * mult + add, so one captured graph
// serves every iteration.
__device__ __forceinline__ unsigned long long iter_value(const Ctl* ctl, long long mult, long long add) {
  return static_cast<unsigned long long>(static_cast<long long>(iter_of(ctl)) * mult + add);
}

__global__ void k_signal(unsigned long long* flag, const Ctl* ctl, long long mult, long long add) {
  const unsigned long long v = iter_value(ctl, mult, add);
  __threadfence_system();
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(v) : "memory");
}

// Spins (acquire, system scope) until every listed counter reaches `target`.
// Gives up early only when a failure at a stage before `guard` (the stage of
// the kernel this wait protects) is recorded — that kernel and everything
// after it skip, so nothing is left to order — or after kStallNs, recording
// PH_STALL (stage 0) so the host raises instead of hanging the device.
constexpr unsigned long long kStallNs = 30ull * 1000 * 1000 * 1000;

// guard stage = t * spi + sub (sub may be negative: a stage of the previous
// iteration index, for waits placed after k_update).
__global__ void k_wait(WaitList w, long long mult, long long add, Ctl* ctl, int sub) {
  const int m = threadIdx.x;
  if (m >= w.n) return;
  const long long starget = static_cast<long long>(iter_of(ctl)) * mult + add;
  if (starget <= 0) return;  // counters start at 0
  const unsigned long long target = static_cast<unsigned long long>(starget);
  const unsigned long long guard = iter_value(ctl, ctl->spi, sub);
  const unsigned long long t0 = globaltimer();
  for (;;) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(w.ptr[m]) : "memory");
    if (v >= target) return;
    const unsigned long long first = min(ld_volatile(&ctl->sh->err_stage), ld_volatile(&ctl->err_stage));
    if (first != kNoErr && first < guard) return;
    if (globaltimer() - t0 > kStallNs) {
      atomicMin(&ctl->err_stage, 0ull);
      atomicMin(&ctl->err_key, static_cast<unsigned long long>(PH_STALL) << 61);
      atomicMin(&ctl->sh->err_stage, 0ull);
      return;
    }
    __nanosleep(256);
  }
}

struct RankBlob {
  int rank = 0, world = 0, device = 0, nloc = 0;  // nloc: plane stride of the rank's dq buffers
  cudaIpcMemHandle_t q[2], dq[2], flags, sh, mag, acc;
};

template <class T>
T* open_ipc(const cudaIpcMemHandle_t& h) {
  void* p = nullptr;
  ck(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  return static_cast<T*>(p);
}

}  // namespace

class RankRun {
 public:
  RankRun(PointSet& ps, const EngineSpec& spec, int rank, int world, int device, int capacity)
      : ps_(ps), spec_(spec), rank_(rank), world_(world), device_(device) {
    if (world < 1 || world > kMaxDomains || rank < 0 || rank >= world)
      raise(Status::argument, "rank/world out of range");
    geoms_ = decompose(ps, world, spec.part_of, spec.reorder);
    spi_ = (spec.order == 2 ? spec.inner : 0) + 4;
    const LocalGeom& g = geoms_[rank];
    dom_ = std::make_unique<Domain>(view_of(g), device, spec.gamma, spec.cfl, spec.det_tol, capacity, true);
    std::vector<int> srcs(g.halo_dom.begin(), g.halo_dom.end());
    std::sort(srcs.begin(), srcs.end());
    srcs.erase(std::unique(srcs.begin(), srcs.end()), srcs.end());
    src_ = srcs;
    for (int d = 0; d < world; ++d) {
      if (d == rank) continue;
      for (int o : geoms_[d].halo_dom)
        if (o == rank) {
          readers_.push_back(d);
          break;
        }
    }
    ck(cudaSetDevice(device), "cudaSetDevice");
    const std::size_t nh = g.halo_dom.size();
    hdom_.alloc(std::max<std::size_t>(1, nh));
    hidx_.alloc(std::max<std::size_t>(1, nh));
    if (nh) {
      ck(cudaMemcpy(hdom_.get(), g.halo_dom.data(), nh * sizeof(int), cudaMemcpyHostToDevice), "H2D hdom");
      ck(cudaMemcpy(hidx_.get(), g.halo_idx.data(), nh * sizeof(int), cudaMemcpyHostToDevice), "H2D hidx");
    }
    // owned points whose stencil reaches a halo slot (boundary) and the rest
    // (interior): interior work runs while the halo is in flight
    {
      std::vector<int> in, bd;
      for (std::int32_t i = 0; i < g.n_own; ++i) {
        bool touches = false;
        for (std::int64_t e = g.off[i]; e < g.off[i + 1] && !touches; ++e) touches = g.nbr[e] >= g.n_own;
        (touches ? bd : in).push_back(i);
      }
      n_interior_ = static_cast<int>(in.size());
      n_boundary_ = static_cast<int>(bd.size());
      interior_.alloc(std::max<std::size_t>(1, in.size()));
      boundary_.alloc(std::max<std::size_t>(1, bd.size()));
      if (!in.empty())
        ck(cudaMemcpy(interior_.get(), in.data(), in.size() * sizeof(int), cudaMemcpyHostToDevice), "H2D interior");
      if (!bd.empty())
        ck(cudaMemcpy(boundary_.get(), bd.data(), bd.size() * sizeof(int), cudaMemcpyHostToDevice), "H2D boundary");
    }
    flags_.alloc(FL_COUNT);
    ck(cudaMemset(flags_.get(), 0, FL_COUNT * sizeof(unsigned long long)), "zero flags");
    if (rank == 0) {
      dom_->set_residue_size(ps.n());
      dom_->set_split4(spec.split4);
      dom_->reset_run(spec.order, spec.inner, spec.fp_mode, spec.chunk, true);  // shared word
      ck(cudaStreamSynchronize(dom_->stream()), "root init");
    }
    ck(cudaEventCreate(&t0_), "ev");
    ck(cudaEventCreate(&t1_), "ev");
    for (auto& e : kev_) ck(cudaEventCreate(&e), "ev");
    blob_.rank = rank;
    blob_.world = world;
    blob_.device = device;
    blob_.nloc = dom_->n_loc();
    ck(cudaIpcGetMemHandle(&blob_.q[0], dom_->q_buf(0)), "IpcGetMemHandle q0");
    ck(cudaIpcGetMemHandle(&blob_.q[1], dom_->q_buf(1)), "IpcGetMemHandle q1");
    ck(cudaIpcGetMemHandle(&blob_.dq[0], dom_->dq_buf(0)), "IpcGetMemHandle dq0");
    ck(cudaIpcGetMemHandle(&blob_.dq[1], dom_->dq_buf(1)), "IpcGetMemHandle dq1");
    ck(cudaIpcGetMemHandle(&blob_.flags, flags_.get()), "IpcGetMemHandle flags");
    ck(cudaIpcGetMemHandle(&blob_.acc, dom_->acc_buf()), "IpcGetMemHandle acc");
    if (rank == 0) {
      ck(cudaIpcGetMemHandle(&blob_.sh, dom_->own_shared()), "IpcGetMemHandle shared");
      ck(cudaIpcGetMemHandle(&blob_.mag, dom_->mag_buf()), "IpcGetMemHandle mag");
    }
  }

  ~RankRun() {
    if (dom_) cudaStreamSynchronize(dom_->stream());
    for (auto& kv : graphs_) cudaGraphExecDestroy(kv.second);
    for (void* p : opened_) cudaIpcCloseMemHandle(p);
    cudaEventDestroy(t0_);
    cudaEventDestroy(t1_);
    for (auto& e : kev_) cudaEventDestroy(e);
  }

  const RankBlob& blob() const { return blob_; }

  // Maps every peer's buffers, uploads this rank's state and computes its
  // first q (owned and halo points).
  void connect(const std::vector<RankBlob>& blobs) {
    if (static_cast<int>(blobs.size()) != world_) raise(Status::argument, "need one blob per rank");
    ck(cudaSetDevice(device_), "cudaSetDevice");
    AccTab acc{};
    for (int o = 0; o < world_; ++o) {
      if (o == rank_) {
        acc.p[o] = dom_->acc_buf();
        for (int k = 0; k < 2; ++k) {
          qp_[k].base[o] = dom_->q_buf(k);
          dqp_[k].base[o] = dom_->dq_buf(k);
          qp_[k].ps[o] = dqp_[k].ps[o] = dom_->n_loc();
        }
        flag_[o] = flags_.get();
        continue;
      }
      const RankBlob& b = blobs[o];
      for (int k = 0; k < 2; ++k) {
        qp_[k].base[o] = open(open_ipc<D4>(b.q[k]));
        dqp_[k].base[o] = open(open_ipc<D4>(b.dq[k]));
        qp_[k].ps[o] = dqp_[k].ps[o] = b.nloc;
      }
      flag_[o] = open(open_ipc<unsigned long long>(b.flags));
      if (rank_ == 0) acc.p[o] = open(open_ipc<unsigned long long>(b.acc));
      if (o == 0) {
        dom_->use_shared(open(open_ipc<Shared>(b.sh)));
        dom_->use_mag(open(open_ipc<double>(b.mag)));
      }
    }
    if (rank_ == 0) dom_->use_acc_tab(acc, world_);
    dom_->upload(ps_.fields, false);
    dom_->set_split4(spec_.split4);
    if (rank_ != 0) dom_->reset_run(spec_.order, spec_.inner, spec_.fp_mode, spec_.chunk, false);
    split_tiles();
    dom_->first_q();
    ck(cudaStreamSynchronize(dom_->stream()), "first q");
    dom_->refresh_ctl();
  }

  // Runs up to n iterations in captured graphs of `chunk` iterations (flag
  // targets are derived on the device, so graphs are reused across chunks);
  // stops early on a device error.  Returns the CUDA-event ms of the work.
  double iterate(int n) {
    Domain& d = *dom_;
    ck(cudaSetDevice(device_), "cudaSetDevice");
    d.set_diag(t_ + n - 1);
    const int chunk = std::max(1, spec_.chunk);
    {
      int t = t_, left = n;
      while (left > 0) {
        const int c = std::min(chunk, left);
        graph_for(t, c);
        t += c;
        left -= c;
      }
    }
    ck(cudaEventRecord(t0_, d.stream()), "EventRecord");
    int issued = 0, waited = 0;
    bool failed = false;
    const int end = t_ + n;
    while (t_ < end && !failed) {
      const int c = std::min(chunk, end - t_);
      ck(cudaGraphLaunch(graph_for(t_, c), d.stream()), "GraphLaunch");
      t_ += c;
      failed = d.poll(issued, waited);
    }
    // Every rank returns only after the root's residue of its last iteration,
    // so all of them observe the same error word.
    if (rank_ != 0) wait_for(std::vector<int>{0}, FL_RES, 1, 0, 0);
    ck(cudaEventRecord(t1_, d.stream()), "EventRecord");
    ck(cudaStreamSynchronize(d.stream()), "rank iterate");
    float ms = 0.0f;
    ck(cudaEventElapsedTime(&ms, t0_, t1_), "EventElapsed");
    d.refresh_ctl();
    d.set_done(d.completed());
    d.add_ms(ms);
    return ms;
  }

  bool failed() { return dom_->failed(); }
  // This rank's own failure record (the Python driver takes the min over
  // ranks) and the message for it: built here when the failing point is
  // owned by this rank (or the failure is not point-specific).
  bool has_error() const { return dom_->has_error(); }
  unsigned long long err_stage() const { return dom_->err_stage(); }
  unsigned long long err_key() const { return dom_->err_key(); }
  bool owns_failure() const {
    if (!dom_->has_error()) return false;
    const unsigned long long key = dom_->err_key();
    if (key_phase(key) >= PH_RESIDUE) return true;
    const int g = static_cast<int>(key_point(key));
    const LocalGeom& lg = geoms_[rank_];
    return std::binary_search(lg.gid.begin(), lg.gid.begin() + lg.n_own, g);
  }
  Fault fault() {
    if (!dom_->has_error())
      return Fault(Status::positivity, "the run failed on another rank");
    const unsigned long long key = dom_->err_key();
    const unsigned phase = key_phase(key);
    const int g = static_cast<int>(key_point(key));
    if (!owns_failure())
      return Fault(phase == PH_SWEEP ? Status::singular : Status::positivity,
                   "iteration " + itos(dom_->err_iter() + 1) + ": failure at point " + itos(g) +
                       " owned by another rank");
    int local = -1;
    if (phase < PH_RESIDUE) {
      const LocalGeom& lg = geoms_[rank_];
      local = static_cast<int>(std::lower_bound(lg.gid.begin(), lg.gid.begin() + lg.n_own, g) - lg.gid.begin());
    }
    return dom_->fault_in_run(local);
  }
  Domain& dom() { return *dom_; }
  bool is_root() const { return rank_ == 0; }
  void download() { copy_back(*dom_, ps_); }
  void flush_l2() { dom_->flush_l2(); }
  // Kernels (compute, halo, signal, wait) this rank enqueued for its last iteration.
  int launches_per_iter() const { return launches_; }
  void last_event_ms(double& sweep_ms, double& flux_ms) const {
    float a = 0.0f, b = 0.0f;
    sweep_ms = flux_ms = 0.0;
    if (spec_.order == 2 && cudaEventElapsedTime(&a, kev_[0], kev_[1]) == cudaSuccess) sweep_ms = a;
    if (cudaEventElapsedTime(&b, kev_[2], kev_[3]) == cudaSuccess) flux_ms = b;
    cudaGetLastError();
  }

 private:
  template <class T>
  T* open(T* p) {
    opened_.push_back(p);
    return p;
  }
  void signal(int slot, long long mult, long long add) {
    k_signal<<<1, 1, 0, dom_->stream()>>>(flags_.get() + slot, dom_->dctl(), mult, add);
    ++launches_;
  }
  // Waits until the ranks' `slot` counters reach t * mult + add (t: this
  // domain's iteration index), guarding stage t * spi + sub (see k_wait).
  void wait_for(const std::vector<int>& ranks, int slot, long long mult, long long add, int sub) {
    if (ranks.empty()) return;
    WaitList w{};
    w.n = static_cast<int>(ranks.size());
    for (int m = 0; m < w.n; ++m) w.ptr[m] = flag_[ranks[m]] + slot;
    k_wait<<<1, 32, 0, dom_->stream()>>>(w, mult, add, dom_->dctl(), sub);
    ++launches_;
  }

  // Graph of c iterations starting at iteration t (parities from t).
  cudaGraphExec_t graph_for(int t, int c) {
    const int a = t & 1, b = spec_.order == 2 ? (t * spec_.inner) & 1 : 0;
    const auto key = std::make_tuple(a, b, c);
    auto it = graphs_.find(key);
    if (it != graphs_.end()) return it->second;
    cudaStream_t st = dom_->stream();
    cudaGraph_t graph;
    ck(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "BeginCapture");
    for (int k = 0; k < c; ++k) enqueue_iteration(t + k, k == c - 1);
    ck(cudaGetLastError(), "capture launches");
    ck(cudaStreamEndCapture(st, &graph), "EndCapture");
    cudaGraphExec_t exec;
    ck(cudaGraphInstantiate(&exec, graph, 0), "GraphInstantiate");
    cudaGraphDestroy(graph);
    graphs_[key] = exec;
    return exec;
  }

  // With a tile plan the sweeps' interior work runs tiled: the tiles none of
  // whose points reads a halo slot go to the tiled sweep (tile_in_) while the
  // halo is in flight; the points of the other tiles (bd_tiles_, a superset
  // of the boundary points) to the list sweep after it.
  void split_tiles() {
    if (!dom_->tiled() || tiles_split_) return;
    const LocalGeom& g = geoms_[rank_];
    const int tp = dom_->tile_points();
    std::vector<int> tin, bpts;
    for (std::int32_t t0 = 0; t0 < g.n_own; t0 += tp) {
      const std::int32_t t1 = std::min<std::int32_t>(g.n_own, t0 + tp);
      bool touches = false;
      for (std::int32_t i = t0; i < t1 && !touches; ++i)
        for (std::int64_t e = g.off[i]; e < g.off[i + 1] && !touches; ++e) touches = g.nbr[e] >= g.n_own;
      if (touches)
        for (std::int32_t i = t0; i < t1; ++i) bpts.push_back(i);
      else
        tin.push_back(t0 / tp);
    }
    n_tile_in_ = static_cast<int>(tin.size());
    n_bd_tiles_ = static_cast<int>(bpts.size());
    tile_in_.alloc(std::max<std::size_t>(1, tin.size()));
    bd_tiles_.alloc(std::max<std::size_t>(1, bpts.size()));
    if (!tin.empty())
      ck(cudaMemcpy(tile_in_.get(), tin.data(), tin.size() * sizeof(int), cudaMemcpyHostToDevice), "H2D tiles");
    if (!bpts.empty())
      ck(cudaMemcpy(bd_tiles_.get(), bpts.data(), bpts.size() * sizeof(int), cudaMemcpyHostToDevice), "H2D tiles");
    tiles_split_ = true;
  }

  // Second order with halo latency hidden behind interior work: each sweep and
  // the flux run first over the interior points (no halo reads), then wait for
  // the owners, gather the halo of the previous stage and finish the boundary
  // points.  Counters (global sweep index k = t * inner + s): FL_SW = k + 1
  // after sweep k; FL_DQH = j + 1 once sweep j's output halo is gathered;
  // FL_UPD = t + 1 after update(t); FL_RES = t + 1 after the root's residue(t).
  // Write-after-read guards: a sweep overwrites sweep k-2's output, so it waits
  // for its readers' FL_DQH >= k - 1; update(t) writes residue summands into
  // the root's array, so it waits for the root's FL_RES >= t.
  void enqueue_overlapped(int t, bool timed) {
    Domain& d = *dom_;
    const int a = t & 1;
    launches_ = 0;
    const long long inner = spec_.inner;
    const int* in = interior_.get();
    const int* bd = boundary_.get();
    for (int s = 0; s < spec_.inner; ++s) {
      const int b = (t * spec_.inner + s) & 1;
      wait_for(readers_, FL_DQH, inner, s - 1, 1 + s);
      if (timed && s == 0) d.record_ext(kev_[0]);
      if (tiles_split_) d.launch_sweep_tiles(a, b, s, tile_in_.get(), n_tile_in_);
      else d.launch_sweep(a, b, s, in, n_interior_);
      if (s == 0) {
        wait_for(src_, FL_UPD, 1, 0, 1);  // owners' q of iteration t
        d.launch_halo(d.q_buf(a), 1, hdom_.get(), hidx_.get(), qp_[a], 1, true);
      } else {
        wait_for(src_, FL_SW, inner, s, 1 + s);  // owners finished sweep k - 1
        d.launch_halo(d.dq_buf(b), 2, hdom_.get(), hidx_.get(), dqp_[b], 1 + s);
        signal(FL_DQH, inner, s);
      }
      if (tiles_split_) d.launch_sweep(a, b, s, bd_tiles_.get(), n_bd_tiles_);
      else d.launch_sweep(a, b, s, bd, n_boundary_);
      if (timed && s == 0) d.record_ext(kev_[1]);
      launches_ += 3;  // interior sweep, halo, boundary sweep
      signal(FL_SW, inner, s + 1);
    }
    const int bfin = ((t + 1) * spec_.inner) & 1;
    const int sub_fl = spi_ - 3;
    if (timed) d.record_ext(kev_[2]);
    d.launch_flux(a, bfin, false, in, n_interior_);
    wait_for(src_, FL_SW, inner, inner, sub_fl);  // owners finished the last sweep
    d.launch_halo(d.dq_buf(bfin), 2, hdom_.get(), hidx_.get(), dqp_[bfin], sub_fl);
    signal(FL_DQH, inner, inner);
    d.launch_flux(a, bfin, false, bd, n_boundary_);
    if (timed) d.record_ext(kev_[3]);
    wait_for(std::vector<int>{0}, FL_RES, 1, 0, spi_ - 2);  // root's residue(t-1) has read the summands
    d.launch_update(a);  // the device iteration index is t + 1 from here on
    launches_ += 2 + 2 * d.flux_launches();  // interior flux, halo, boundary flux, update
    signal(FL_UPD, 1, 0);
    if (rank_ == 0) {
      std::vector<int> all;
      for (int o = 1; o < world_; ++o) all.push_back(o);
      wait_for(all, FL_UPD, 1, 0, -1);
      d.launch_residue();
      launches_ += spec_.fp_mode == 1 ? 2 : 1;
      signal(FL_RES, 1, 0);
    }
    ck(cudaGetLastError(), "rank launches");
  }

  // One iteration; only the buffer parities depend on the host-side t (the
  // counters' targets follow the device iteration index).  Timed: CUDA
  // events around the first sweep and the flux kernel.
  void enqueue_iteration(int t, bool timed) {
    if (spec_.order == 2 && dom_->subsets_supported() && overlap_enabled()) return enqueue_overlapped(t, timed);
    Domain& d = *dom_;
    cudaStream_t st = d.stream();
    const int a = t & 1;
    launches_ = 0;
    const long long inner = spec_.inner;
    wait_for(std::vector<int>{0}, FL_RES, 1, 0, 0);  // root's residue of iteration t-1 done
    wait_for(src_, FL_UPD, 1, 0, 0);                   // owners' q of iteration t ready
    d.launch_halo(d.q_buf(a), 1, hdom_.get(), hidx_.get(), qp_[a], 0, true);
    ++launches_;
    int bfin = 0;
    if (spec_.order == 2) {
      for (int s = 0; s < spec_.inner; ++s) {
        const int b = (t * spec_.inner + s) & 1;
        if (s >= 2) wait_for(readers_, FL_DQH, inner, s - 1, 1 + s);  // readers gathered sweep k-2
        if (timed && s == 0) d.record_ext(kev_[0]);
        d.launch_sweep(a, b, s);
        launches_ += 2;  // sweep + dq halo
        if (timed && s == 0) d.record_ext(kev_[1]);
        signal(FL_SW, inner, s + 1);                  // = k + 1, k = t * inner + s
        wait_for(src_, FL_SW, inner, s + 1, 1 + s);
        d.launch_halo(d.dq_buf(b ^ 1), 2, hdom_.get(), hidx_.get(), dqp_[b ^ 1], 1 + s);
        signal(FL_DQH, inner, s + 1);
      }
      bfin = ((t + 1) * spec_.inner) & 1;
    }
    if (timed) d.record_ext(kev_[2]);
    d.launch_flux(a, bfin, spec_.order != 2);
    if (timed) d.record_ext(kev_[3]);
    d.launch_update(a);  // the device iteration index is t + 1 from here on
    launches_ += 1 + d.flux_launches();  // flux + update
    signal(FL_UPD, 1, 0);
    if (rank_ == 0) {
      std::vector<int> all;
      for (int o = 1; o < world_; ++o) all.push_back(o);
      wait_for(all, FL_UPD, 1, 0, -1);  // guard: the residue stage of iteration t
      d.launch_residue();
      launches_ += spec_.fp_mode == 1 ? 2 : 1;  // tree partial + final, or the exact sum
      signal(FL_RES, 1, 0);
    }
    ck(cudaGetLastError(), "rank launches");
  }

  PointSet& ps_;
  EngineSpec spec_;
  int rank_ = 0, world_ = 1, device_ = 0;
  std::vector<LocalGeom> geoms_;
  std::unique_ptr<Domain> dom_;
  std::vector<int> src_, readers_;
  DBuf<int> hdom_, hidx_;
  DBuf<int> interior_, boundary_;
  int n_interior_ = 0, n_boundary_ = 0;
  DBuf<int> tile_in_, bd_tiles_;  // interior tiles / points of the other tiles (split_tiles)
  int n_tile_in_ = 0, n_bd_tiles_ = 0;
  bool tiles_split_ = false;
  DBuf<unsigned long long> flags_;
  PeerTab qp_[2]{}, dqp_[2]{};
  unsigned long long* flag_[kMaxDomains] = {};
  std::vector<void*> opened_;
  RankBlob blob_{};
  cudaEvent_t t0_ = nullptr, t1_ = nullptr, kev_[4] = {};
  int t_ = 0, launches_ = 0, spi_ = 4;
  std::map<std::tuple<int, int, int>, cudaGraphExec_t> graphs_;
};

RankRun* rank_open(PointSet& ps, const EngineSpec& spec, int rank, int world, int device, int capacity) {
  return new RankRun(ps, spec, rank, world, device, capacity);
}
std::size_t rank_blob_bytes() { return sizeof(RankBlob); }
std::vector<unsigned char> rank_blob(const RankRun* r) {
  const unsigned char* p = reinterpret_cast<const unsigned char*>(&r->blob());
  return std::vector<unsigned char>(p, p + sizeof(RankBlob));
}
void rank_connect(RankRun* r, const std::vector<std::vector<unsigned char>>& blobs) {
  std::vector<RankBlob> bs(blobs.size());
  for (std::size_t i = 0; i < blobs.size(); ++i) {
    if (blobs[i].size() != sizeof(RankBlob)) raise(Status::argument, "malformed rank blob");
    std::memcpy(&bs[i], blobs[i].data(), sizeof(RankBlob));
  }
  r->connect(bs);
  if (r->failed()) throw r->fault();
}
double rank_iterate(RankRun* r, int n) {
  const double ms = r->iterate(n);
  if (r->failed()) throw r->fault();
  return ms;
}
std::vector<double> rank_residues(RankRun* r) { return r->is_root() ? r->dom().residues() : std::vector<double>(); }
void rank_download(RankRun* r) { r->download(); }
void rank_flush_l2(RankRun* r) { r->flush_l2(); }
void rank_event_ms(const RankRun* r, double* sweep_ms, double* flux_ms) { r->last_event_ms(*sweep_ms, *flux_ms); }
int rank_launches_per_iter(const RankRun* r) { return r->launches_per_iter(); }
void rank_error(const RankRun* r, unsigned long long* stage, unsigned long long* key, int* owns) {
  *stage = r->has_error() ? r->err_stage() : kNoErr;
  *key = r->has_error() ? r->err_key() : kNoErr;
  *owns = r->owns_failure() ? 1 : 0;
}
void rank_close(RankRun* r) { delete r; }

RunRecord engine_run_multi(PointSet& ps, const EngineSpec& spec, const std::vector<LocalGeom>& geoms) {
  if (spec.iters == 0) return engine_run(ps, spec);
  RunRecord rec;
  MultiRun m(ps, spec, geoms, spec.iters);
  trace("engine: domains open");
  if (m.failed()) throw m.fault();
  m.iterate(spec.iters);
  trace("engine: iterated");
  if (m.failed()) {
    Fault f = m.fault();
    rec.abort_iteration = m.abort_iteration();
    throw f;
  }
  m.download();
  trace("engine: copied back");
  Domain& r = m.root();
  rec.iterations = r.done();
  rec.residue = r.residues();
  rec.wall_ms = r.wall_ms();
  rec.kernels = r.kernel_times();
  rec.total_seconds = r.total_ms() * 1e-3;
  const double first = rec.residue.empty() ? 0.0 : rec.residue.front();
  for (double x : rec.residue) rec.log10_rel.push_back((first > 0.0 && x > 0.0) ? std::log10(x / first) : 0.0);
  return rec;
}

// ---- sessions (single domain, or a multi-domain run when spec.gpus > 1) ----
class Session {
 public:
  std::unique_ptr<Domain> dom;
  std::unique_ptr<MultiRun> multi;
  PointSet* ps = nullptr;
  Domain& head() { return multi ? multi->root() : *dom; }
  const Domain& head() const { return multi ? const_cast<MultiRun&>(*multi).root() : *dom; }
};

Session* session_open(PointSet& ps, const EngineSpec& spec, int capacity) {
  auto s = std::make_unique<Session>();
  s->ps = &ps;
  if (spec.gpus > 1) {
    s->multi = std::make_unique<MultiRun>(ps, spec, decompose(ps, spec.gpus, spec.part_of, spec.reorder), capacity);
    if (s->multi->failed()) throw s->multi->fault();
  } else {
    s->dom = open_domain(ps, spec, capacity);
    if (s->dom->failed()) throw s->dom->fault_in_run();
  }
  return s.release();
}

double session_iterate(Session* s, int n) {
  if (s->multi) {
    const double ms = s->multi->iterate(n);
    if (s->multi->failed()) throw s->multi->fault();
    return ms;
  }
  const double ms = s->dom->iterate(n);
  if (s->dom->failed()) throw s->dom->fault_in_run();
  return ms;
}

std::vector<double> session_residues(const Session* s) { return s->head().residues(); }
std::vector<KernelTime> session_kernels(const Session* s) { return s->head().kernel_times(); }
int session_launches_per_iter(const Session* s) {
  return s->multi ? s->multi->launches_per_iter() : s->dom->launches_per_iter();
}
void session_tiles(const Session* s, int* staged, int* total) {
  *staged = *total = 0;
  if (s->multi) {
    s->multi->tiles(staged, total);
  } else {
    *staged = s->dom->tiles_staged();
    *total = s->dom->tiles_total();
  }
}
std::uint64_t session_stream(const Session* s) { return reinterpret_cast<std::uint64_t>(s->head().stream()); }
void session_download(Session* s) {
  if (s->multi) s->multi->download();
  else copy_back(*s->dom, *s->ps);
}
void session_event_ms(const Session* s, double* sweep_ms, double* flux_ms) {
  if (s->multi) s->multi->last_event_ms(*sweep_ms, *flux_ms);
  else s->dom->last_event_ms(*sweep_ms, *flux_ms);
}
void session_flush_l2(Session* s) {
  if (s->multi) s->multi->flush_l2();
  else s->dom->flush_l2();
}
double session_step_flushed(Session* s, bool kernel_events) {
  if (s->multi) {
    s->multi->flush_l2();
    return session_iterate(s, 1);
  }
  const double ms = s->dom->step_flushed(kernel_events);
  if (s->dom->failed()) throw s->dom->fault_in_run();
  return ms;
}

// ---- exact kNN queries on attach_knn's 2-d tree (host/synth.cpp): one thread
// per point, in tree order (neighbouring threads walk similar paths).  The k
// best by (d^2, id) are kept sorted in registers; a subtree is skipped only
// when its box's lower bound exceeds the current k-th distance strictly, and
// distances and bounds are formed with separately rounded products and sums
// (no FMA) exactly as on the host — so the set is the host's, which is the
// reference's build_stencils set (cloud.cpp:137-237).
template <int K>
__global__ void __launch_bounds__(128) k_knn(const KdNode* __restrict__ nodes, const KdPt* __restrict__ pts, int n,
                                             std::int32_t* __restrict__ nbr) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const KdPt me = pts[t];
  const double px = me.x, py = me.y;
  double bd[K];
  int bi[K];
  int cnt = 0;
  auto bound = [&](const KdNode& b) {
    const double ex = px < b.x0 ? __dsub_rn(b.x0, px) : (px > b.x1 ? __dsub_rn(px, b.x1) : 0.0);
    const double ey = py < b.y0 ? __dsub_rn(b.y0, py) : (py > b.y1 ? __dsub_rn(py, b.y1) : 0.0);
    return __dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey));
  };
  int stack[96];
  int sp = 0;
  stack[sp++] = 0;
  while (sp > 0) {
    const KdNode b = nodes[stack[--sp]];
    if (cnt == K && bound(b) > bd[K - 1]) continue;
    if (b.left < 0) {
      for (int e = b.lo; e < b.hi; ++e) {
        const KdPt c = pts[e];
        if (c.id == me.id) continue;
        const double dx = __dsub_rn(c.x, px), dy = __dsub_rn(c.y, py);
        const double d2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
        if (cnt == K && !(d2 < bd[K - 1] || (d2 == bd[K - 1] && c.id < bi[K - 1]))) continue;
        int j = cnt < K ? cnt++ : K - 1;  // insertion into the sorted list
        while (j > 0 && (d2 < bd[j - 1] || (d2 == bd[j - 1] && c.id < bi[j - 1]))) {
          bd[j] = bd[j - 1];
          bi[j] = bi[j - 1];
          --j;
        }
        bd[j] = d2;
        bi[j] = c.id;
      }
      continue;
    }
    const double bl = bound(nodes[b.left]), br = bound(nodes[b.right]);
    if (sp + 2 > 96) __trap();  // depth far beyond any median-split tree of 2^31 points
    if (bl <= br) {  // nearer child last, so it is visited first
      stack[sp++] = b.right;
      stack[sp++] = b.left;
    } else {
      stack[sp++] = b.left;
      stack[sp++] = b.right;
    }
  }
  // ids ascending (the reference sorts each stencil)
  for (int a = 1; a < K; ++a) {
    const int v = bi[a];
    int j = a;
    while (j > 0 && bi[j - 1] > v) {
      bi[j] = bi[j - 1];
      --j;
    }
    bi[j] = v;
  }
  std::int32_t* out = nbr + static_cast<long long>(me.id) * K;
  for (int j = 0; j < K; ++j) out[j] = bi[j];
}

template <int K>
void knn_launch(const KdNode* nodes, const KdPt* pts, int n, std::int32_t* nbr, cudaStream_t st) {
  k_knn<K><<<(n + 127) / 128, 128, 0, st>>>(nodes, pts, n, nbr);
}

bool engine_knn(const std::vector<KdNode>& nodes, const std::vector<KdPt>& pts, int k, std::int32_t* nbr) {
  int count = 0;
  const bool supported = (k >= 3 && k <= 8) || k == 12 || k == 16;
  if (!supported || cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return false;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  ensure_pool(dev);
  const int n = static_cast<int>(pts.size());
  cudaStream_t st = nullptr;
  ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
  {
    DBuf<KdNode> dn(nodes.size(), st);
    DBuf<KdPt> dp(pts.size(), st);
    DBuf<std::int32_t> dnbr(static_cast<std::size_t>(n) * k, st);
    ck(cudaMemcpyAsync(dn.get(), nodes.data(), nodes.size() * sizeof(KdNode), cudaMemcpyHostToDevice, st), "H2D kd");
    ck(cudaMemcpyAsync(dp.get(), pts.data(), pts.size() * sizeof(KdPt), cudaMemcpyHostToDevice, st), "H2D kd");
    switch (k) {
      case 3: knn_launch<3>(dn.get(), dp.get(), n, dnbr.get(), st); break;
      case 4: knn_launch<4>(dn.get(), dp.get(), n, dnbr.get(), st); break;
      case 5: knn_launch<5>(dn.get(), dp.get(), n, dnbr.get(), st); break;
      case 6: knn_launch<6>(dn.get(), dp.get(), n, dnbr.get(), st); break;
      case 7: knn_launch<7>(dn.get(), dp.get(), n, dnbr.get(), st); break;
      case 8: knn_launch<8>(dn.get(), dp.get(), n, dnbr.get(), st); break;
      case 12: knn_launch<12>(dn.get(), dp.get(), n, dnbr.get(), st); break;
      case 16: knn_launch<16>(dn.get(), dp.get(), n, dnbr.get(), st); break;
      default: break;
    }
    ck(cudaGetLastError(), "k_knn");
    ck(cudaMemcpyAsync(nbr, dnbr.get(), static_cast<std::size_t>(n) * k * sizeof(std::int32_t), cudaMemcpyDeviceToHost,
                       st),
       "D2H knn");
    ck(cudaStreamSynchronize(st), "knn");
  }
  cudaStreamDestroy(st);
  return true;
}

__global__ void k_math_selftest(int fn, const double* in, long long n, double* ref, double* ours) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double x = in[i];
    if (fn == 0) {
      ref[i] = erf(x);
      ours[i] = lk_erf(x);
    } else if (fn == 1) {
      ref[i] = exp(x);
      ours[i] = lk_exp(x);
    } else {  // fast mode's polynomial erf
      const double xs[1] = {x};
      double o[1];
      erf_fast_n<1>(xs, o);
      ref[i] = erf(x);
      ours[i] = o[0];
    }
  }
}

void engine_math_selftest(int fn, const double* in, std::int64_t n, double* ref, double* ours) {
  if (n <= 0) return;
  DBuf<double> d_in(static_cast<std::size_t>(n)), d_ref(static_cast<std::size_t>(n)),
      d_ours(static_cast<std::size_t>(n));
  ck(cudaMemcpy(d_in.get(), in, n * sizeof(double), cudaMemcpyHostToDevice), "H2D selftest");
  k_math_selftest<<<1184, 256>>>(fn, d_in.get(), n, d_ref.get(), d_ours.get());
  ck(cudaGetLastError(), "selftest launch");
  ck(cudaMemcpy(ref, d_ref.get(), n * sizeof(double), cudaMemcpyDeviceToHost), "D2H selftest");
  ck(cudaMemcpy(ours, d_ours.get(), n * sizeof(double), cudaMemcpyDeviceToHost), "D2H selftest");
}

double engine_fp64_peak_tflops(int device) {
  ck(cudaSetDevice(device), "cudaSetDevice");
  int sms = 0;
  ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device), "attr");
  DBuf<double> out(1);
  const int blocks = sms * 8, threads = 256, iters = 8192;
  cudaEvent_t e0, e1;
  ck(cudaEventCreate(&e0), "ev");
  ck(cudaEventCreate(&e1), "ev");
  double best = 0.0;
  for (int rep = 0; rep < 4; ++rep) {
    ck(cudaEventRecord(e0), "ev");
    k_dfma_peak<<<blocks, threads>>>(out.get(), iters, 0.999999, 1e-7);
    ck(cudaEventRecord(e1), "ev");
    ck(cudaEventSynchronize(e1), "dfma");
    float ms = 0.0f;
    ck(cudaEventElapsedTime(&ms, e0, e1), "ev");
    const double flops = 2.0 * 8.0 * iters * static_cast<double>(blocks) * threads;
    if (rep > 0) best = std::max(best, flops / (ms * 1e-3) / 1e12);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return best;
}
void session_close(Session* s) { delete s; }

// ---- per-phase operators ----
void engine_op(PointSet& ps, Op op, const OpSpec& spec, double* scratch) {
  Domain d(view_of(ps, {}), spec.device, spec.gamma, spec.cfl, spec.det_tol, 1);
  d.set_strict(spec.fp_mode == 1);
  d.upload(ps.fields, true);
  k_ctl_init<<<1, 1, 0, d.stream()>>>(d.dctl(), d.shared(), 1, -1, 0, d.update_blocks());
  const Geo g = d.geo();
  const int n = ps.n();
  const int blocks = (n + 255) / 256;
  const std::size_t nn = static_cast<std::size_t>(n);
  cudaStream_t st = d.stream();
  // dq_[1] doubles as the scratch buffer of q_derivatives / publish.
  switch (op) {
    case Op::q_variables:
      k_qvar<<<blocks, 256, 0, st>>>(g, d.prim(), d.q_buf(0), d.gas(), d.dctl());
      break;
    case Op::q_derivatives:
      sweep_launch(spec.fp_mode == 1, g, d.q_buf(0), d.dq_buf(0), d.dq_buf(1), d.gas(), d.dctl(), nullptr, 0, st);
      break;
    case Op::publish:  // scratch is the reference's [qx0..3, qy0..3] per point
      ck(cudaMemcpyAsync(d.dq_buf(1), scratch, nn * 8 * sizeof(double), cudaMemcpyHostToDevice, st), "H2D scratch");
      k_dq_layout<<<static_cast<int>((nn + 255) / 256), 256, 0, st>>>(d.dq_buf(1), d.dq_buf(0),
                                                                     static_cast<long long>(nn), g.nloc, 1);
      break;
    case Op::flux_fused:
    case Op::flux_direction: {
      FluxArgs fa{};
      fa.g = g;
      fa.gas = d.gas();
      fa.q = d.q_buf(0);
      fa.dq = d.dq_buf(0);
      fa.res = d.res();
      fa.ctl = d.dctl();
      fa.kcap = d.kmax();
      fa.stride = flux_stride(d.kmax());
      fa.mask = op == Op::flux_fused ? 0xF : (1 << (spec.axis * 2 + spec.sign));
      fa.first = op == Op::flux_fused ? 1 : spec.first;
      flux_launch(d.width(), spec.fp_mode == 1, fa, d.smem(), st);
      break;
    }
    case Op::timestep:
      k_op_timestep<<<blocks, 256, 0, st>>>(g, d.prim(), d.dt(), d.gas());
      break;
    case Op::state_update:
      k_op_update<<<blocks, 256, 0, st>>>(g, d.prim(), d.res(), d.dt(), d.gas(), d.dctl(), d.which());
      break;
  }
  ck(cudaGetLastError(), "operator launch");
  ck(cudaStreamSynchronize(st), "operator");
  d.refresh_ctl();
  if (d.failed()) throw d.fault(false, d.q_buf(0), d.dq_buf(0));
  if (op == Op::q_derivatives) {
    DBuf<D4> plain(2 * nn, st);
    k_dq_layout<<<static_cast<int>((nn + 255) / 256), 256, 0, st>>>(d.dq_buf(1), plain.get(),
                                                                   static_cast<long long>(nn), g.nloc, 0);
    ck(cudaMemcpyAsync(scratch, plain.get(), nn * 8 * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H scratch");
    ck(cudaStreamSynchronize(st), "scratch");
    return;  // the store itself is untouched (reference kernels.hpp:30-35)
  }
  d.download(ps.fields, true, d.q_buf(0), d.dq_buf(0));
}

double engine_reduce(const double* v, std::int64_t n, int device) {
  ck(cudaSetDevice(device), "cudaSetDevice");
  if (n <= 0) return 0.0;
  DBuf<double> dv(static_cast<std::size_t>(n)), pv(8192), out(1);
  DBuf<long long> ps(8192);
  DBuf<Ctl> ctl(1);
  ck(cudaMemcpy(dv.get(), v, n * sizeof(double), cudaMemcpyHostToDevice), "H2D reduce");
  DBuf<Shared> sh(1);
  k_ctl_init<<<1, 1>>>(ctl.get(), sh.get(), 1, -1, 0, 1);
  const int d1 = tree_depth(n);
  k_tree_partial<<<1 << d1, kTreeThreads>>>(dv.get(), n, d1, pv.get(), ps.get(), ctl.get());
  k_tree_result<<<1, 1024>>>(pv.get(), ps.get(), d1, out.get());
  ck(cudaGetLastError(), "reduce launch");
  double r = 0.0;
  ck(cudaMemcpy(&r, out.get(), sizeof r, cudaMemcpyDeviceToHost), "D2H reduce");
  return r;
}

double engine_exact_sum(const double* v, std::int64_t n, int device) {
  ck(cudaSetDevice(device), "cudaSetDevice");
  DBuf<double> dv(static_cast<std::size_t>(std::max<std::int64_t>(1, n))), out(1);
  DBuf<unsigned long long> acc(kAccWords);
  ck(cudaMemset(acc.get(), 0, kAccWords * sizeof(unsigned long long)), "memset acc");
  if (n > 0) {
    ck(cudaMemcpy(dv.get(), v, n * sizeof(double), cudaMemcpyHostToDevice), "H2D exact sum");
    const int blocks = static_cast<int>(std::min<std::int64_t>((n + 255) / 256, 148 * 8));
    k_exact_sum_blocks<<<blocks, 256>>>(dv.get(), n, acc.get());
  }
  k_exact_sum_final<<<1, 1>>>(acc.get(), out.get());
  ck(cudaGetLastError(), "exact sum launch");
  double r = 0.0;
  ck(cudaMemcpy(&r, out.get(), sizeof r, cudaMemcpyDeviceToHost), "D2H exact sum");
  return r;
}

int engine_device_count() {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return c;
}

}  // namespace lskb
