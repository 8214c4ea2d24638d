/* lskum_b200.h — B200-specific extensions to the drop-in C ABI (lskum/lskum.h).
 *
 * The reference keeps part of its interface in C++ only (run_fixed_point,
 * the per-phase operators, partition_cloud).  Those are exposed here as plain
 * C so test harnesses, the bench and per-rank launchers can reach the same
 * boundaries without C++ types.  Each entry cites the reference interface it
 * mirrors.  All calls are synchronous; device memory never outlives the call
 * (sessions own theirs until lskum_b200_session_destroy).
 *
 * Extra config keys accepted by lskum_config_set (reference config.cpp:98-131
 * rejects unknown keys; these are additive):
 *   device=N          CUDA device ordinal for single-GPU runs (default 0)
 *   gpus=N            number of device domains (RCB parts on distinct devices
 *                     when available; default 1)
 *   fp_mode=fast|strict  strict = the reference's exact operation sequence in
 *                     the flux kernel; fast = deduplicated x/y reconstruction
 *                     (default fast).  Sweeps, time step, update and residue
 *                     are bitwise-reference in both modes.
 *   chunk=N           iterations per captured CUDA graph (default 16)
 */
#ifndef LSKUM_B200_H
#define LSKUM_B200_H

#include "lskum/lskum.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- backend / device info ---- */
const char* lskum_b200_backend(void);
int lskum_b200_device_count(int* out);

/* ---- clouds on plain arrays (PointCloud(records), reference cloud.hpp:42-74) ---- */
int lskum_b200_cloud_from_arrays(int32_t n, const double* x, const double* y,
                                 const uint8_t* kind, const double* nx, const double* ny,
                                 const int64_t* offsets, const int32_t* nbrs,
                                 lskum_cloud** out);
int lskum_b200_cloud_nnz(const lskum_cloud* cloud, int64_t* out);
/* Surface force coefficients from the cloud's current pressures (SURVEY
 * 8(f)-4; the reference has Cp only, bench.cpp:101-105): out = {Cl, Cd, Cm
 * about the quarter chord, chord}.  loop = surface point ids around the body
 * in order (n = 0: the wall points in id order); panels carry the mean Cp of
 * their end points; M and AoA from cfg. */
int lskum_b200_surface_forces(const lskum_cloud* cloud, const lskum_config* cfg, const int32_t* loop, int32_t n,
                              double out[4]);
/* validate_cloud (reference cloud.cpp:252-321) computed on `device` — the
 * screening lskum_run performs there; same report and
 * defective ids (ascending) as lskum_cloud_validate / _defective_ids. */
/* Device numbering a run with config key reorder = mode (0 none, 1 hilbert,
 * 2 auto, 3 rcm) uses: *permuted = 1 when the device holds the points in a
 * locality order (Hilbert curve, or reverse Cuthill-McKee for rcm and auto);
 * *lines_before / *lines_after = sampled 128-byte derivative-record lines the
 * neighbours of 16 consecutive points touch, per point, in the cloud's own
 * order and in the locality order (0 when not computed).
 * Host-only (no device needed); cached on the cloud. */
int lskum_b200_cloud_locality(lskum_cloud* cloud, int mode, double* lines_before, double* lines_after,
                              int* permuted);
int lskum_b200_cloud_validate_device(lskum_cloud* cloud, int device, lskum_validation* out, int32_t* ids,
                                     int32_t cap, int32_t* n_out);
/* Synthetic NACA 0012 O-cloud (no reference counterpart, the
 * reference's generators are cloud.cpp:323-425): n_wall surface points (even),
 * n_rings rings out to a far-field circle of radius outer_radius chords about
 * (0.5, 0); kNN stencils as lskum_cloud_generate_rect.  frozen_wall != 0 marks
 * the surface ring outer (held state) instead of wall.  Config spec:
 * generate=naca0012:<n_wall>x<n_rings>[:frozen]. */
int lskum_b200_cloud_generate_naca0012(int n_wall, int n_rings, double outer_radius, double jitter,
                                       uint64_t seed, int knn, int frozen_wall, lskum_cloud** out);
/* Any output pointer may be NULL. */
int lskum_b200_cloud_geometry(const lskum_cloud* cloud, double* x, double* y, uint8_t* kind,
                              double* nx, double* ny, int64_t* offsets, int32_t* nbrs);
/* PointCloud::reset_store (reference cloud.cpp:90-92); layout 0 = aos, 1 = soa. */
int lskum_b200_cloud_reset_store(lskum_cloud* cloud, int layout);
/* Whole 21-slot store as point-major (AoS) n*21 doubles, whatever the layout. */
int lskum_b200_cloud_get_fields(const lskum_cloud* cloud, double* aos);
int lskum_b200_cloud_set_fields(lskum_cloud* cloud, const double* aos);

/* ---- fixed-point driver (run_fixed_point, reference runtime.hpp:103) ----
 * Iterates from the primitives already in the cloud's store (no free-stream
 * reset) — the C++-host entry the reference tests call directly. */
int lskum_b200_run_fixed_point(lskum_cloud* cloud, const lskum_config* cfg,
                               lskum_result** out);
/* 1-based iteration at which a failed run aborted (0 if none / not applicable). */
int lskum_b200_result_abort_iteration(const lskum_result* result);
int lskum_b200_result_wall_ms(const lskum_result* result, int iteration, double* out);

/* ---- per-phase device operators (reference kernels.hpp:25-63) ----
 * Each runs one phase over every point of `cloud` on the GPU, reading and
 * writing the cloud's host field store (uploaded and downloaded around the
 * kernel).  Same error codes and messages as the reference phase. */
typedef struct {
  double gamma;   /* GasModel::gamma */
  double cfl;     /* KernelParams::cfl */
  double det_tol; /* KernelParams::det_tol */
  int fp_mode;    /* 0 = fast, 1 = strict (flux only) */
} lskum_b200_params;

int lskum_b200_op_q_variables(lskum_cloud* cloud, const lskum_b200_params* p);
/* scratch: n*8 doubles (qx[4], qy[4] per point), as q_derivatives_kernel. */
int lskum_b200_op_q_derivatives(lskum_cloud* cloud, const lskum_b200_params* p,
                                double* scratch);
int lskum_b200_op_publish(lskum_cloud* cloud, const double* scratch);
int lskum_b200_op_flux_residual(lskum_cloud* cloud, const lskum_b200_params* p);
/* axis 0/1 = x/y, sign 0/1 = plus/minus; first != 0 zeroes the accumulator. */
int lskum_b200_op_flux_direction(lskum_cloud* cloud, const lskum_b200_params* p, int axis,
                                 int sign, int first);
int lskum_b200_op_timestep(lskum_cloud* cloud, const lskum_b200_params* p);
int lskum_b200_op_state_update(lskum_cloud* cloud, const lskum_b200_params* p);
/* deterministic_reduce (reference reduce.hpp:11-17) evaluated on the device. */
int lskum_b200_reduce(const double* values, int64_t n, double* out);
/* Correctly rounded (nearest, ties to even) sum of non-negative doubles: the
   fast-mode residue accumulator (kernels.cuh acc_warp_add / acc_to_double). */
int lskum_b200_exact_sum(const double* values, int64_t n, double* out);

/* ---- partitioning (partition_cloud, reference partition.hpp:27) ----
 * owner[i] = part of point i; ghosts of part p are ghosts[ghost_off[p]..ghost_off[p+1]). */
int lskum_b200_partition(const lskum_cloud* cloud, int n_parts, int32_t* owner,
                         int64_t* ghost_off, int32_t* ghosts, int64_t ghost_cap);

/* ---- device-resident sessions (bench.py, per-rank launchers) ----
 * create: validate, free-stream initialise (unless from_state != 0), upload,
 *         build the CUDA graphs; capacity = max iterations over the session.
 * iterate: run n more iterations; *device_ms = CUDA-event time on the
 *          session's stream around exactly those iterations.
 * download: copy the 21-slot store back into the cloud. */
typedef struct lskum_b200_session lskum_b200_session;
int lskum_b200_session_create(lskum_cloud* cloud, const lskum_config* cfg, int capacity,
                              int from_state, lskum_b200_session** out);
int lskum_b200_session_iterate(lskum_b200_session* s, int n, double* device_ms);
int lskum_b200_session_residues(const lskum_b200_session* s, double* out, int cap,
                                int* n_out);
/* Per-kernel device seconds accumulated so far (globaltimer, per launch). */
int lskum_b200_session_kernel_count(const lskum_b200_session* s);
const char* lskum_b200_session_kernel_name(const lskum_b200_session* s, int index);
int lskum_b200_session_kernel_stats(const lskum_b200_session* s, int index, double* seconds,
                                    int64_t* launches);
/* Kernel launches per iteration and the CUDA stream (cudaStream_t as integer). */
int lskum_b200_session_info(const lskum_b200_session* s, int* launches_per_iter,
                            uint64_t* stream);
/* Tiled derivative sweep (engine tiles.cuh): tiles whose stencil union is
 * staged in shared memory, and all tiles, summed over the session's domains
 * (0/0: the run has no tile plan — first order, non-uniform stencils or
 * LSKUM_SWEEP_TILE=0). */
int lskum_b200_session_tiles(const lskum_b200_session* s, int* staged, int* total);
int lskum_b200_session_download(lskum_b200_session* s);
/* CUDA-event milliseconds of the first derivative sweep and of the flux
 * kernel of the latest lskum_b200_session_step_flushed(kernel_events = 1)
 * (events recorded inside the graph; multi-device sessions: latest iteration). */
int lskum_b200_session_event_ms(const lskum_b200_session* s, double* sweep_ms, double* flux_ms);
/* Overwrites a 384 MB scratch buffer on the session stream (cold-L2 steps). */
int lskum_b200_session_flush_l2(lskum_b200_session* s);
/* One cold-L2 step: the flush and one iteration in one CUDA graph;
 * *device_ms = CUDA-event time of the iteration (events inside the graph).
 * kernel_events != 0 also records the event_ms() events around the first
 * sweep and the flux kernel (which lengthens the step). */
int lskum_b200_session_step_flushed(lskum_b200_session* s, int kernel_events, double* device_ms);
/* Measured FP64 FMA throughput of `device` (TFLOP/s, DFMA = 2 flops). */
int lskum_b200_fp64_peak(int device, double* tflops);
void lskum_b200_session_destroy(lskum_b200_session* s);

/* ---- one process per GPU (torchrun ranks) ----
 * Every rank calls rank_create on the same cloud/config with its rank, the
 * world size and its CUDA device; the rank builds only its own RCB piece
 * (owned points + halo) in IPC-exportable memory.  The caller exchanges the
 * opaque blobs (rank_blob_size() bytes each, e.g. an all_gather) and passes
 * all `world` of them, in rank order, to rank_connect.  Stage ordering across
 * processes is device-side (release/acquire progress counters), so iterate
 * only enqueues and synchronises its own stream.  Residues are available on
 * rank 0; download fills this rank's owned points of the cloud's store.
 * rank_info: kernels enqueued per iteration and this rank's failure record:
 * the stage (iteration * (sweeps + 4) + phase slot) and ordering key of its
 * first failure (UINT64_MAX: none) and whether it owns the failing point.
 * The run's failure is the record with the smallest (stage, key) over the
 * ranks; the owning rank's lskum_last_error() text is the reference's. */
typedef struct lskum_b200_rank lskum_b200_rank;
int lskum_b200_rank_create(lskum_cloud* cloud, const lskum_config* cfg, int rank, int world,
                           int device, int capacity, int from_state, lskum_b200_rank** out);
int lskum_b200_rank_blob_size(void);
int lskum_b200_rank_blob(const lskum_b200_rank* r, void* out);
int lskum_b200_rank_connect(lskum_b200_rank* r, const void* blobs, int world);
int lskum_b200_rank_iterate(lskum_b200_rank* r, int n, double* device_ms);
int lskum_b200_rank_residues(const lskum_b200_rank* r, double* out, int cap, int* n_out);
int lskum_b200_rank_info(const lskum_b200_rank* r, int* launches_per_iter, uint64_t* err_stage,
                         uint64_t* err_key, int* owns_failure);
int lskum_b200_rank_download(lskum_b200_rank* r);
int lskum_b200_rank_event_ms(const lskum_b200_rank* r, double* sweep_ms, double* flux_ms);
int lskum_b200_rank_flush_l2(lskum_b200_rank* r);
void lskum_b200_rank_destroy(lskum_b200_rank* r);

/* ---- verification hook ----
 * Evaluates CUDA libdevice erf (fn 0, 2) / exp (fn 1) into ref[] and into ours[]
 * the engine's constant-table replicas used by the flux kernel (fn 0, 1: must be
 * bitwise equal) or fp_mode fast's polynomial erf (fn 2: a few ulps). */
int lskum_b200_math_selftest(int fn, const double* in, int64_t n, double* ref, double* ours);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* LSKUM_B200_H */
