// core.hpp — host-side model of the LSKUM problem (C++20).
//
// Native C++ counterpart of the reference's host layers L1/L4
// (/root/reference/proj/src/core/{cloud,layout,config,bench,error}.hpp):
// a columnar point set with CSR stencils, the 21-slot field block, the
// solver settings and the error type that crosses the C ABI as a status.
// The iteration itself lives on the GPU (../dev); this header is what the
// host side of the boundary hands to it.
#pragma once

#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace lskb {

// Status codes == LSKUM_ERR_* (reference error.hpp:9-17, lskum.h:18-27).
enum class Status : int {
  ok = 0,
  argument = 1,
  parse = 2,
  io = 3,
  validation = 4,
  singular = 5,
  positivity = 6,
  config = 7,
};

class Fault : public std::runtime_error {
 public:
  Fault(Status s, const std::string& what) : std::runtime_error(what), status_(s) {}
  Status status() const noexcept { return status_; }

 private:
  Status status_;
};

[[noreturn]] inline void raise(Status s, const std::string& what) { throw Fault(s, what); }

// Host-phase tracing to stderr when LSKUM_TRACE is set (setup cost analysis).
void trace(const char* what);
bool tracing();

// Pinned staging I/O (hostcopy.cpp): streaming stores into staging, and
// flushing staging lines after the host read them, keep the DMA at PCIe rate.
void flush_lines(const void* p, std::size_t bytes);
void stream_copy(void* dst, const void* src, std::size_t bytes);
void stream_pairs(double* dst, const double* a, const double* b, std::size_t n);  // dst[2i] = a[i], dst[2i+1] = b[i]

// %f rendering, as std::to_string(double) produces in the reference messages.
std::string fmt_f(double v);

enum class Kind : std::uint8_t { interior = 0, wall = 1, outer = 2 };
enum class Layout : std::uint8_t { aos = 0, soa = 1 };

// Slot map of the 21-double field record (reference layout.hpp:11-19).
namespace slot {
inline constexpr int prim = 0, q = 4, qx = 8, qy = 12, res = 16, dt = 20, count = 21;
}

// Per-point solver fields in one buffer; AoS or SoA differ only in strides
// (reference layout.hpp:24-48).  The GPU never sees this block directly: it
// is the staging/copy-back format behind lskum_cloud_primitive/fields_equal.
// std::allocator without value-initialisation of default-constructed elements.
template <class T>
struct NoInitAlloc : std::allocator<T> {
  NoInitAlloc() = default;
  template <class U>
  NoInitAlloc(const NoInitAlloc<U>&) noexcept {}
  template <class U>
  struct rebind {
    using other = NoInitAlloc<U>;
  };
  template <class U, class... A>
  void construct(U* p, A&&... a) {
    if constexpr (sizeof...(A) > 0) ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
    else ::new (static_cast<void*>(p)) U;
  }
};

// Storage of a field store.  Large stores (>= 64 MB) come from pinned host
// memory when the engine registered an allocator (store_pinned_hooks(), set by
// engine.cu; a process-wide pool keeps freed blocks for the next store of the
// same size), so the copy-back DMAs straight into the store instead of through
// staging and a host copy.  Falls back to ordinary memory (no device,
// LSKUM_PINNED_STORE=0).  Contents are not initialised.
struct StoreHooks {
  void* (*alloc)(std::size_t bytes) = nullptr;    // null on failure
  void (*release)(void* p, std::size_t bytes) = nullptr;
};
StoreHooks& store_hooks();
// Clouds keep their large arrays in pinned memory (LSKUM_PINNED_CLOUD=0: heap).
bool pinned_clouds();

// Allocator of a cloud's per-point arrays (coordinates, normals, kinds,
// stencil offsets and ids): blocks of 32 MB and more come from pinned host
// memory through store_hooks() (the engine's pool), so the geometry upload
// DMAs straight from the cloud's own arrays instead of through staging;
// smaller blocks, and every block when no device is present, from the heap.
// The pinned/heap decision is a function of the block size alone, so
// deallocate() takes the same path as allocate() did.
template <class T>
struct HostAlloc {
  using value_type = T;
  HostAlloc() = default;
  template <class U>
  HostAlloc(const HostAlloc<U>&) noexcept {}
  static constexpr std::size_t kPinnedMin = std::size_t{32} << 20;
  static bool pinned_block(std::size_t bytes) { return bytes >= kPinnedMin && store_hooks().alloc && pinned_clouds(); }
  T* allocate(std::size_t n) {
    const std::size_t bytes = n * sizeof(T);
    if (pinned_block(bytes)) {
      // a pinned block carries a 64-byte header: 1 = pinned, so a heap
      // fallback of the same size is released to the heap
      char* p = static_cast<char*>(store_hooks().alloc(bytes + 64));
      if (p) {
        *reinterpret_cast<std::uint64_t*>(p) = 1;
        return reinterpret_cast<T*>(p + 64);
      }
      char* h = static_cast<char*>(::operator new(bytes + 64));
      *reinterpret_cast<std::uint64_t*>(h) = 0;
      return reinterpret_cast<T*>(h + 64);
    }
    return static_cast<T*>(::operator new(bytes));
  }
  void deallocate(T* p, std::size_t n) noexcept {
    const std::size_t bytes = n * sizeof(T);
    if (pinned_block(bytes)) {
      char* b = reinterpret_cast<char*>(p) - 64;
      if (*reinterpret_cast<std::uint64_t*>(b) == 1) store_hooks().release(b, bytes + 64);
      else ::operator delete(b);
      return;
    }
    ::operator delete(p);
  }
  template <class U>
  bool operator==(const HostAlloc<U>&) const noexcept { return true; }
};
template <class T>
using HVec = std::vector<T, HostAlloc<T>>;

class StoreBuffer {
 public:
  StoreBuffer() = default;
  explicit StoreBuffer(std::size_t count) { allocate(count); }
  StoreBuffer(const StoreBuffer& o) : StoreBuffer(o.n_) {
    if (n_) std::memcpy(p_, o.p_, n_ * sizeof(double));
  }
  StoreBuffer(StoreBuffer&& o) noexcept : p_(o.p_), n_(o.n_), pinned_(o.pinned_) {
    o.p_ = nullptr;
    o.n_ = 0;
    o.pinned_ = false;
  }
  StoreBuffer& operator=(StoreBuffer o) noexcept {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    std::swap(pinned_, o.pinned_);
    return *this;
  }
  ~StoreBuffer() { release(); }
  double* data() { return p_; }
  const double* data() const { return p_; }
  std::size_t size() const { return n_; }
  bool pinned() const { return pinned_; }
  double& operator[](std::size_t i) { return p_[i]; }
  double operator[](std::size_t i) const { return p_[i]; }

 private:
  void allocate(std::size_t count);
  void release();
  double* p_ = nullptr;
  std::size_t n_ = 0;
  bool pinned_ = false;
};

class FieldBlock {
 public:
  FieldBlock() = default;
  FieldBlock(Layout layout, std::int32_t n);

  Layout layout() const { return layout_; }
  std::int32_t size() const { return n_; }
  double& at(std::int32_t p, int s) { return data_[index(p, s)]; }
  double at(std::int32_t p, int s) const { return data_[index(p, s)]; }
  std::size_t point_stride() const { return layout_ == Layout::aos ? slot::count : 1; }
  std::size_t slot_stride() const {
    return layout_ == Layout::aos ? 1 : static_cast<std::size_t>(n_);
  }
  double* raw() { return data_.data(); }
  const double* raw() const { return data_.data(); }
  // The store lives in pinned host memory (device copies may target it directly).
  bool pinned() const { return data_.pinned(); }

  // Point-major (AoS) export/import regardless of the layout.
  void export_aos(double* out) const;
  void import_aos(const double* in);

 private:
  std::size_t index(std::int32_t p, int s) const {
    return static_cast<std::size_t>(p) * point_stride() + static_cast<std::size_t>(s) * slot_stride();
  }
  Layout layout_ = Layout::aos;
  std::int32_t n_ = 0;
  // Allocated without value-initialisation; the constructor zero-fills it in
  // parallel (first touch spread over threads: hundreds of MB at 10M+ points).
  StoreBuffer data_;
};

// Bitwise comparison over every (point, slot) (reference layout.cpp:29-45).
bool fields_identical(const FieldBlock& a, const FieldBlock& b);

// Columnar point set + CSR stencils (reference cloud.hpp:37-74).
struct Screening;

struct Locality;

struct PointSet {
  HVec<double> x, y, nx, ny;
  HVec<Kind> kind;
  HVec<std::int64_t> off{0};  // n+1
  HVec<std::int32_t> nbr;     // ascending ids per point
  FieldBlock fields;

  std::int32_t n() const { return static_cast<std::int32_t>(x.size()); }
  std::int64_t nnz() const { return off.empty() ? 0 : off.back(); }
  std::int32_t degree(std::int32_t i) const {
    return static_cast<std::int32_t>(off[i + 1] - off[i]);
  }
  // Screening report of this (immutable) geometry, computed on first use.
  mutable std::shared_ptr<const Screening> screening;
  // Device numbering chosen by the last run's reorder mode (reorder.cpp).
  mutable std::shared_ptr<const Locality> locality;
  // Device-resident copy of this geometry kept between lskum_run calls (the
  // engine's single-device domain: geometry, weights, state buffers, CUDA
  // graphs); released with the cloud.
  mutable std::shared_ptr<void> engine_cache;

  bool has_wall() const;
  int max_degree() const;
  void reset_fields(Layout layout);
};

// One row of input, as produced by the readers and generators.
struct PointRow {
  double x = 0, y = 0, nx = 0, ny = 0;
  Kind kind = Kind::interior;
};

// Checks ids/stencils (reference cloud.cpp:42-83 semantics) and assembles.
PointSet assemble(std::vector<PointRow> rows, std::vector<std::int64_t> off,
                  std::vector<std::int32_t> nbr);

// ---- grid files (reference cloud.cpp:427-545 format) ----
PointSet read_grid_file(const std::string& path);
PointSet parse_grid_text(const char* text, std::size_t len);
void write_grid_file(const PointSet& ps, const std::string& path);

// ---- generators + kNN (reference cloud.cpp:137-237, 323-425) ----
struct Box {
  double xmin = 0.0, xmax = 1.0, ymin = 0.0, ymax = 1.0;
};
PointSet make_rect(int nx, int ny, const Box& box, double jitter, std::uint64_t seed, int k);
PointSet make_annulus(int n_theta, int n_rings, double r_outer, double jitter,
                      std::uint64_t seed, int k);
PointSet make_naca0012(int n_wall, int n_rings, double r_outer, double jitter, std::uint64_t seed, int k,
                       bool frozen_wall);
void attach_knn(PointSet& ps, int k);

// 2-d tree of attach_knn (synth.cpp), also queried on the GPU (engine_knn).
struct KdNode {
  double x0, x1, y0, y1;              // bounding box of points [lo, hi)
  std::int32_t lo, hi, left, right;   // leaf: left = right = -1
};
struct KdPt {
  double x, y;
  std::int32_t id, pad;
};

// ---- stencil screening (reference cloud.cpp:252-321) ----
struct Screening {
  double h_ref = 0.0, det_tol = 0.0;
  std::int32_t n_defective = 0, n_wall_isolated = 0, min_stencil = 0;
  std::vector<std::int32_t> defective;
};
Screening screen_stencils(const PointSet& ps);

// ---- recursive coordinate bisection (reference partition.cpp:12-80) ----
struct Piece {
  std::vector<std::int32_t> owned;   // ascending
  std::vector<std::int32_t> halo;    // ascending; stencil closure minus owned
};
std::vector<Piece> bisect_cloud(const PointSet& ps, int n_parts);

// ---- settings (reference config.hpp:12-57, config.cpp) ----
struct Settings {
  // solver
  double mach = 0.63, aoa = 2.0, gamma = 1.4, cfl = 0.5;
  int iters = 1000, inner = 3, order = 2;
  Layout layout = Layout::aos;
  int residual_split4 = 0;  // 0 fused, 1 split4
  int parts = 1, workers = 1;
  std::string out_prefix;
  // grid source
  std::string grid, generate;
  double jitter = 0.0;
  std::uint64_t seed = 0;
  int knn = 8;
  Box bounds;
  double outer_radius = 10.0;
  // B200 additions
  int device = 0, gpus = 1, fp_mode = 0, chunk = 16;
  int reorder = 2;  // kReorderAuto (none | hilbert | rcm | auto)

  void check() const;  // ErrorCode::config on bad values (reference config.cpp:47-56)
  void set(const std::string& key, const std::string& value);
  std::string get(const std::string& key) const;
  void load(const std::string& path);
};
PointSet acquire_points(const Settings& s);

// ---- locality permutation of the device numbering (reorder.cpp) ----
enum : int { kReorderNone = 0, kReorderHilbert = 1, kReorderAuto = 2, kReorderRcm = 3 };
struct Locality {
  int mode = kReorderNone;
  std::vector<std::int32_t> order;   // device index k -> point id; empty: identity
  double lines_before = 0.0, lines_after = 0.0;  // gather lines per point (sampled)
};
// Mean distinct 128-byte derivative-record lines touched by the neighbours of
// 16 consecutive points in the given order (empty: the cloud's own).
double gather_lines_per_point(const PointSet& ps, const std::vector<std::int32_t>& order);
std::vector<std::int32_t> hilbert_order(const PointSet& ps);
std::vector<std::int32_t> rcm_order(const PointSet& ps);
// The cloud's device numbering for `mode`, cached on the cloud.
const Locality& cloud_locality(const PointSet& ps, int mode);

// ---- run results / reports (reference runtime.hpp:29-47, bench.cpp) ----
struct KernelTime {
  std::string name;
  double seconds = 0.0;
  std::int64_t launches = 0;
};

struct RunRecord {
  int iterations = 0;
  std::vector<double> residue, log10_rel, wall_ms;
  std::vector<KernelTime> kernels;
  double total_seconds = 0.0;
  int abort_iteration = 0;
};

void freestream(PointSet& ps, double mach, double aoa_deg, double gamma);
double rate_of_data_processing(double seconds, std::int64_t iters, std::int64_t n);
double relative_rate(double rdp_test, double rdp_ref);
double pressure_coeff(double p, double mach, double gamma);
struct Forces {
  double cl = 0.0, cd = 0.0, cm = 0.0, chord = 0.0;
  std::int32_t points = 0;
};
Forces surface_forces(const PointSet& ps, const std::vector<std::int32_t>& loop, double mach, double aoa_deg,
                      double gamma);

struct KernelRow {
  std::string name;
  double seconds = 0.0, rdp = 0.0;
};
struct Report {
  int iterations = 0;
  std::int32_t n = 0;
  double total_seconds = 0.0, total_rdp = 0.0;
  std::vector<KernelRow> rows;
};
Report summarize(const RunRecord& run, std::int32_t n);
void write_run_outputs(const std::string& prefix, const PointSet& ps, const RunRecord& run,
                       const Report& rep, const Settings& s);

// Runs the fixed-point loop on the GPU from the primitives in ps.fields
// (reference run_fixed_point, runtime.cpp:195-275).  Throws Fault on failure
// with the reference's code and "iteration N: ..." message.
RunRecord solve_on_device(PointSet& ps, const Settings& s);
// lskum_run: reset the store to the configured layout + free stream + solve.
// Single-domain runs initialise the state on the device and leave the host
// store to the copy-back; on an early failure the host store gets the same
// reset + free stream the reference leaves (lskum_capi.cpp:209-220).
RunRecord solve_from_freestream(PointSet& ps, const Settings& s);

}  // namespace lskb
