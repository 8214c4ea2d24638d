// engine.hpp — the boundary between the C++ host layer and the CUDA engine.
//
// The host (host/*.cpp, g++) owns clouds, settings, validation and
// partitioning; the engine (dev/engine.cu, nvcc, sm_100a) owns device memory,
// streams, CUDA graphs and kernels.  Everything crossing this header is plain
// host data; device pointers never leave engine.cu.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "host/core.hpp"

namespace lskb {

struct EngineSpec {
  double gamma = 1.4, cfl = 0.5, det_tol = 0.0;
  int iters = 0, inner = 3, order = 2;
  int fp_mode = 0;  // 0 fast, 1 strict
  int split4 = 0;   // residual_mode=split4 (failure order: direction before partition)
  int chunk = 16;   // iterations per captured graph
  int device = 0;
  int gpus = 1;     // device domains (sessions; lskum_run decides in solve.cpp)
  int reorder = 0;  // single-device numbering: kReorderNone / Hilbert / Auto (reorder.cpp)
  // Partition of each point (reference error tie-break, runtime.cpp:115-118).
  std::vector<std::uint16_t> part_of;
  // lskum_run's free-stream initialisation done on the device (single-domain
  // runs): the host store is only written by the copy-back; store_written
  // reports whether that happened, so the caller can apply the host-side
  // initialisation the reference leaves behind when a run fails earlier.
  bool fs_device = false;
  double fs_prim[4] = {0.0, 0.0, 0.0, 0.0};
  bool* store_written = nullptr;
};

// Exact k nearest neighbours by (d^2, id) of every point, from attach_knn's
// 2-d tree, on the GPU: nbr[p * k ..] = the ids, ascending.  False when no
// device is usable or k is not one of 3..8, 12, 16 (the caller queries on the host).
bool engine_knn(const std::vector<KdNode>& nodes, const std::vector<KdPt>& pts, int k, std::int32_t* nbr);

// Stencil screening on the device into ps.screening (single-device runs; no-op
// when the report is cached or gpus > 1).
void engine_prescreen(PointSet& ps, const Settings& s);
// The same report computed on `device` (kept resident in the cloud's cache).
Screening engine_screen(PointSet& ps, int device, double gamma = 1.4, double cfl = 0.5, int capacity = 1,
                        int reorder = 0);

// Config check + stencil screening gate + bisection (host side of a run).
EngineSpec prepare_run(const PointSet& ps, const Settings& s);

// Fixed-point loop from the primitives in ps.fields; on return ps.fields holds
// the reference's final 21-slot store.  Throws Fault like run_fixed_point.
RunRecord engine_run(PointSet& ps, const EngineSpec& spec);

// One device domain of a multi-domain run: the points of one RCB piece in
// local numbering (owned [0, n_own), then halo [n_own, n_loc)), the local
// stencil table, and where each halo point lives (owner domain, its local
// index there).  Built on the host by decompose().
struct LocalGeom {
  std::int32_t n_own = 0, n_loc = 0;
  std::vector<double> x, y, nx, ny;      // n_loc
  std::vector<Kind> kind;                // n_loc
  std::vector<std::int64_t> off;         // n_own + 1
  std::vector<std::int32_t> nbr;         // local ids
  std::vector<std::uint16_t> part;       // n_loc: reference partition (error tie-break)
  std::vector<std::int32_t> gid;         // n_loc: local -> global id
  std::vector<std::int32_t> halo_dom;    // n_loc - n_own
  std::vector<std::int32_t> halo_idx;    // n_loc - n_own
};
std::vector<LocalGeom> decompose(const PointSet& ps, int n_domains, const std::vector<std::uint16_t>& part_of,
                                 int reorder = 0);
// The whole cloud as one domain in the given device order (reorder.cpp):
// point k of the domain is point order[k] of the cloud; no halo.
LocalGeom permuted_geom(const PointSet& ps, const std::vector<std::int32_t>& order,
                        const std::vector<std::uint16_t>& part_of);

// Multi-domain run: one Domain per RCB piece, devices assigned round-robin
// from spec.device; halos exchanged by peer-memory gathers; residue summed
// over global ids on the first domain (bitwise equal to engine_run).
RunRecord engine_run_multi(PointSet& ps, const EngineSpec& spec, const std::vector<LocalGeom>& geoms);

// Device-resident session (bench, ranks).
class Session;
Session* session_open(PointSet& ps, const EngineSpec& spec, int capacity);
double session_iterate(Session* s, int n);  // returns device ms; throws Fault
std::vector<double> session_residues(const Session* s);
std::vector<KernelTime> session_kernels(const Session* s);
int session_launches_per_iter(const Session* s);
void session_tiles(const Session* s, int* staged, int* total);  // tiled-sweep plan over all domains
std::uint64_t session_stream(const Session* s);
void session_download(Session* s);
void session_event_ms(const Session* s, double* sweep_ms, double* flux_ms);
void session_flush_l2(Session* s);
double session_step_flushed(Session* s, bool kernel_events);  // L2 flush + one iteration; device ms of the iteration
double engine_fp64_peak_tflops(int device);
// Evaluates libdevice erf/exp (fn 0/1) and the engine's constant-table replicas.
void engine_math_selftest(int fn, const double* in, std::int64_t n, double* ref, double* ours);
void session_close(Session* s);

// One process per GPU: this rank's domain of a `world`-way RCB run.  The
// opaque blob (CUDA IPC handles) is exchanged by the caller (e.g. an
// all_gather over torch.distributed) and passed back to rank_connect.
class RankRun;
RankRun* rank_open(PointSet& ps, const EngineSpec& spec, int rank, int world, int device, int capacity);
std::size_t rank_blob_bytes();
std::vector<unsigned char> rank_blob(const RankRun* r);
void rank_connect(RankRun* r, const std::vector<std::vector<unsigned char>>& blobs);
double rank_iterate(RankRun* r, int n);
std::vector<double> rank_residues(RankRun* r);
void rank_download(RankRun* r);
void rank_flush_l2(RankRun* r);
void rank_event_ms(const RankRun* r, double* sweep_ms, double* flux_ms);
int rank_launches_per_iter(const RankRun* r);
// This rank's failure record (stage, key; ~0 = none) and whether it owns the failing point.
void rank_error(const RankRun* r, unsigned long long* stage, unsigned long long* key, int* owns);
void rank_close(RankRun* r);

// Per-phase operators on the whole cloud (reference kernels.hpp:25-63).
enum class Op { q_variables, q_derivatives, publish, flux_fused, flux_direction, timestep,
                state_update };
struct OpSpec {
  double gamma = 1.4, cfl = 0.5, det_tol = 0.0;
  int fp_mode = 0;
  int axis = 0, sign = 0, first = 1;
  int device = 0;
};
void engine_op(PointSet& ps, Op op, const OpSpec& spec, double* scratch);
double engine_reduce(const double* v, std::int64_t n, int device);
// Correctly rounded sum of non-negative doubles (the fast-mode residue accumulator).
double engine_exact_sum(const double* v, std::int64_t n, int device);
int engine_device_count();

}  // namespace lskb
