// capi.cpp — extern "C" boundary: lskum.h (drop-in) and lskum_b200.h.
//
// Status/ownership conventions of the reference C API
// (src/capi/lskum_capi.cpp:15-37): C++ exceptions never cross; Fault maps to
// its status, any other std::exception to LSKUM_ERR_ARGUMENT; the message is
// kept in a thread_local string for lskum_last_error(); NULL arguments give
// LSKUM_ERR_ARGUMENT "null argument".
#include <algorithm>
#include <cstring>
#include <memory>
#include <new>
#include <string>

#include "../engine.hpp"
#include "core.hpp"
#include "lskum_b200.h"

namespace {

thread_local std::string t_last_error;

int fail(int status, const char* what) {
  t_last_error = what;
  return status;
}

template <class Fn>
int guard(Fn&& fn) {
  try {
    fn();
    t_last_error.clear();
    return LSKUM_OK;
  } catch (const lskb::Fault& f) {
    t_last_error = f.what();
    return static_cast<int>(f.status());
  } catch (const std::bad_alloc&) {
    t_last_error = "out of memory";
    return LSKUM_ERR_ARGUMENT;
  } catch (const std::exception& e) {
    t_last_error = e.what();
    return LSKUM_ERR_ARGUMENT;
  }
}

}  // namespace

struct lskum_cloud {
  lskb::PointSet ps;
};

struct lskum_config {
  lskb::Settings s;
};

struct lskum_result {
  lskb::RunRecord run;
  lskb::Report rep;
  lskb::Settings s;
};

struct lskum_b200_session {
  lskb::Session* session = nullptr;
  lskum_cloud* cloud = nullptr;
  std::vector<lskb::KernelTime> kernels;
  ~lskum_b200_session() {
    if (session) lskb::session_close(session);
  }
};

struct lskum_b200_rank {
  lskb::RankRun* run = nullptr;
  ~lskum_b200_rank() {
    if (run) lskb::rank_close(run);
  }
};

#define NONNULL(...)                                                    \
  do {                                                                  \
    const void* ptrs_[] = {__VA_ARGS__};                                \
    for (const void* p_ : ptrs_)                                        \
      if (!p_) return fail(LSKUM_ERR_ARGUMENT, "null argument");        \
  } while (0)

extern "C" {

// ---------------------------------------------------------------- clouds
int lskum_cloud_read_file(const char* path, lskum_cloud** out) {
  NONNULL(path, out);
  return guard([&] { *out = new lskum_cloud{lskb::read_grid_file(path)}; });
}

int lskum_cloud_write_file(const lskum_cloud* cloud, const char* path) {
  NONNULL(cloud, path);
  return guard([&] { lskb::write_grid_file(cloud->ps, path); });
}

int lskum_cloud_generate_rect(int nx, int ny, double jitter, uint64_t seed, int knn, lskum_cloud** out) {
  NONNULL(out);
  return guard([&] { *out = new lskum_cloud{lskb::make_rect(nx, ny, lskb::Box{}, jitter, seed, knn)}; });
}

int lskum_cloud_generate_annulus(int n_theta, int n_rings, double outer_radius, double jitter,
                                 uint64_t seed, int knn, lskum_cloud** out) {
  NONNULL(out);
  return guard([&] {
    *out = new lskum_cloud{lskb::make_annulus(n_theta, n_rings, outer_radius, jitter, seed, knn)};
  });
}

int lskum_b200_cloud_generate_naca0012(int n_wall, int n_rings, double outer_radius, double jitter,
                                       uint64_t seed, int knn, int frozen_wall, lskum_cloud** out) {
  NONNULL(out);
  return guard([&] {
    *out = new lskum_cloud{lskb::make_naca0012(n_wall, n_rings, outer_radius, jitter, seed, knn, frozen_wall != 0)};
  });
}

int lskum_cloud_from_config(const lskum_config* cfg, lskum_cloud** out) {
  NONNULL(cfg, out);
  return guard([&] { *out = new lskum_cloud{lskb::acquire_points(cfg->s)}; });
}

int32_t lskum_cloud_n_points(const lskum_cloud* cloud) { return cloud ? cloud->ps.n() : 0; }

int lskum_cloud_validate(const lskum_cloud* cloud, lskum_validation* out) {
  NONNULL(cloud, out);
  return guard([&] {
    const lskb::Screening s = lskb::screen_stencils(cloud->ps);
    out->n_points = cloud->ps.n();
    out->n_defective = s.n_defective;
    out->n_wall_isolated = s.n_wall_isolated;
    out->min_stencil_size = s.min_stencil;
    out->h_ref = s.h_ref;
    out->det_tol = s.det_tol;
  });
}

int lskum_b200_cloud_locality(lskum_cloud* cloud, int mode, double* lines_before, double* lines_after,
                              int* permuted) {
  NONNULL(cloud);
  if (mode < 0 || mode > 3) return fail(LSKUM_ERR_ARGUMENT, "reorder mode must be 0, 1, 2 or 3");
  return guard([&] {
    const lskb::Locality& loc = lskb::cloud_locality(cloud->ps, mode);
    if (lines_before) *lines_before = loc.lines_before;
    if (lines_after) *lines_after = loc.lines_after;
    if (permuted) *permuted = loc.order.empty() ? 0 : 1;
  });
}

int lskum_b200_cloud_validate_device(lskum_cloud* cloud, int device, lskum_validation* out, int32_t* ids,
                                     int32_t cap, int32_t* n_out) {
  if (!cloud || !out || !n_out || (cap > 0 && !ids)) return fail(LSKUM_ERR_ARGUMENT, "null argument");
  return guard([&] {
    const lskb::Screening s = lskb::engine_screen(cloud->ps, device);
    out->n_points = cloud->ps.n();
    out->n_defective = s.n_defective;
    out->n_wall_isolated = s.n_wall_isolated;
    out->min_stencil_size = s.min_stencil;
    out->h_ref = s.h_ref;
    out->det_tol = s.det_tol;
    *n_out = s.n_defective;
    const int32_t m = std::min<int32_t>(cap, static_cast<int32_t>(s.defective.size()));
    for (int32_t i = 0; i < m; ++i) ids[i] = s.defective[i];
  });
}

int lskum_cloud_defective_ids(const lskum_cloud* cloud, int32_t* ids, int32_t cap, int32_t* n_out) {
  if (!cloud || !n_out || (cap > 0 && !ids)) return fail(LSKUM_ERR_ARGUMENT, "null argument");
  return guard([&] {
    const lskb::Screening s = lskb::screen_stencils(cloud->ps);
    *n_out = s.n_defective;
    const int32_t m = std::min<int32_t>(cap, static_cast<int32_t>(s.defective.size()));
    for (int32_t i = 0; i < m; ++i) ids[i] = s.defective[i];
  });
}

int lskum_cloud_primitive(const lskum_cloud* cloud, int32_t point, double out[4]) {
  NONNULL(cloud, out);
  if (point < 0 || point >= cloud->ps.n()) return fail(LSKUM_ERR_ARGUMENT, "point id out of range");
  for (int c = 0; c < 4; ++c) out[c] = cloud->ps.fields.at(point, lskb::slot::prim + c);
  return LSKUM_OK;
}

int lskum_cloud_fields_equal(const lskum_cloud* a, const lskum_cloud* b, int* equal) {
  NONNULL(a, b, equal);
  return guard([&] { *equal = lskb::fields_identical(a->ps.fields, b->ps.fields) ? 1 : 0; });
}

void lskum_cloud_destroy(lskum_cloud* cloud) { delete cloud; }

// ---------------------------------------------------------------- config
int lskum_config_create(lskum_config** out) {
  NONNULL(out);
  *out = new lskum_config{};
  return LSKUM_OK;
}

int lskum_config_set(lskum_config* cfg, const char* key, const char* value) {
  NONNULL(cfg, key, value);
  return guard([&] { cfg->s.set(key, value); });
}

int lskum_config_get(const lskum_config* cfg, const char* key, char* buf, size_t cap) {
  NONNULL(cfg, key, buf);
  return guard([&] {
    const std::string v = cfg->s.get(key);
    if (cap < v.size() + 1) lskb::raise(lskb::Status::argument, std::string("buffer too small for ") + key);
    std::memcpy(buf, v.c_str(), v.size() + 1);
  });
}

int lskum_config_load(lskum_config* cfg, const char* path) {
  NONNULL(cfg, path);
  return guard([&] { cfg->s.load(path); });
}

int lskum_config_validate(const lskum_config* cfg) {
  NONNULL(cfg);
  return guard([&] { cfg->s.check(); });
}

void lskum_config_destroy(lskum_config* cfg) { delete cfg; }

// ---------------------------------------------------------------- solving
static int run_impl(lskum_cloud* cloud, const lskum_config* cfg, lskum_result** out, bool reinit) {
  NONNULL(cloud, cfg, out);
  return guard([&] {
    lskb::trace("run: enter");
    lskb::RunRecord run = reinit ? lskb::solve_from_freestream(cloud->ps, cfg->s)
                                 : lskb::solve_on_device(cloud->ps, cfg->s);
    lskb::Report rep = lskb::summarize(run, cloud->ps.n());
    lskb::trace("run: done");
    *out = new lskum_result{std::move(run), std::move(rep), cfg->s};
  });
}

int lskum_run(lskum_cloud* cloud, const lskum_config* cfg, lskum_result** out) {
  return run_impl(cloud, cfg, out, true);
}

int lskum_result_iterations(const lskum_result* r) { return r ? r->run.iterations : 0; }

int lskum_result_residue(const lskum_result* r, int iteration, double* out) {
  NONNULL(r, out);
  if (iteration < 1 || iteration > static_cast<int>(r->run.residue.size()))
    return fail(LSKUM_ERR_ARGUMENT, "iteration out of range");
  *out = r->run.residue[iteration - 1];
  return LSKUM_OK;
}

int lskum_result_final_residue(const lskum_result* r, double* out) {
  NONNULL(r, out);
  if (r->run.residue.empty()) return fail(LSKUM_ERR_ARGUMENT, "empty history");
  *out = r->run.residue.back();
  return LSKUM_OK;
}

int lskum_result_final_log10_rel(const lskum_result* r, double* out) {
  NONNULL(r, out);
  if (r->run.log10_rel.empty()) return fail(LSKUM_ERR_ARGUMENT, "empty history");
  *out = r->run.log10_rel.back();
  return LSKUM_OK;
}

double lskum_result_total_seconds(const lskum_result* r) { return r ? r->run.total_seconds : 0.0; }

int lskum_result_rdp(const lskum_result* r, double* out) {
  NONNULL(r, out);
  *out = r->rep.total_rdp;
  return LSKUM_OK;
}

int lskum_result_kernel_count(const lskum_result* r) { return r ? static_cast<int>(r->rep.rows.size()) : 0; }

const char* lskum_result_kernel_name(const lskum_result* r, int index) {
  if (!r || index < 0 || index >= static_cast<int>(r->rep.rows.size())) return nullptr;
  return r->rep.rows[index].name.c_str();
}

int lskum_result_kernel_seconds(const lskum_result* r, int index, double* out) {
  if (!r || !out || index < 0 || index >= static_cast<int>(r->rep.rows.size()))
    return fail(LSKUM_ERR_ARGUMENT, "bad kernel index");
  *out = r->rep.rows[index].seconds;
  return LSKUM_OK;
}

int lskum_result_kernel_rdp(const lskum_result* r, int index, double* out) {
  if (!r || !out || index < 0 || index >= static_cast<int>(r->rep.rows.size()))
    return fail(LSKUM_ERR_ARGUMENT, "bad kernel index");
  *out = r->rep.rows[index].rdp;
  return LSKUM_OK;
}

int lskum_result_write_outputs(const lskum_result* r, const lskum_cloud* cloud, const char* prefix) {
  NONNULL(r, cloud, prefix);
  return guard([&] { lskb::write_run_outputs(prefix, cloud->ps, r->run, r->rep, r->s); });
}

void lskum_result_destroy(lskum_result* r) { delete r; }

int lskum_b200_surface_forces(const lskum_cloud* cloud, const lskum_config* cfg, const int32_t* loop, int32_t n,
                              double out[4]) {
  if (!cloud || !cfg || !out || (n > 0 && !loop)) return fail(LSKUM_ERR_ARGUMENT, "null argument");
  return guard([&] {
    const std::vector<std::int32_t> ids(loop, loop + std::max<int32_t>(n, 0));
    const lskb::Forces f = lskb::surface_forces(cloud->ps, ids, cfg->s.mach, cfg->s.aoa, cfg->s.gamma);
    out[0] = f.cl;
    out[1] = f.cd;
    out[2] = f.cm;
    out[3] = f.chord;
  });
}

// ---------------------------------------------------------------- metrics / diagnostics
int lskum_rdp(double wall_seconds, int64_t iterations, int64_t n_points, double* out) {
  NONNULL(out);
  return guard([&] { *out = lskb::rate_of_data_processing(wall_seconds, iterations, n_points); });
}

int lskum_relative_performance(double rdp_test, double rdp_reference, double* out) {
  NONNULL(out);
  return guard([&] { *out = lskb::relative_rate(rdp_test, rdp_reference); });
}

const char* lskum_last_error(void) { return t_last_error.c_str(); }

const char* lskum_status_name(int status) {
  switch (status) {
    case LSKUM_OK: return "ok";
    case LSKUM_ERR_ARGUMENT: return "argument";
    case LSKUM_ERR_PARSE: return "parse";
    case LSKUM_ERR_IO: return "io";
    case LSKUM_ERR_VALIDATION: return "validation";
    case LSKUM_ERR_SINGULAR: return "singular";
    case LSKUM_ERR_POSITIVITY: return "positivity";
    case LSKUM_ERR_CONFIG: return "config";
    default: return "unknown";
  }
}

const char* lskum_version(void) { return "1.0.0"; }

// ================================================================ B200 extensions
const char* lskum_b200_backend(void) { return "cuda sm_100a"; }

int lskum_b200_device_count(int* out) {
  NONNULL(out);
  *out = lskb::engine_device_count();
  return LSKUM_OK;
}

int lskum_b200_cloud_from_arrays(int32_t n, const double* x, const double* y, const uint8_t* kind,
                                 const double* nx, const double* ny, const int64_t* offsets,
                                 const int32_t* nbrs, lskum_cloud** out) {
  NONNULL(x, y, kind, nx, ny, offsets, out);
  if (n <= 0) return fail(LSKUM_ERR_ARGUMENT, "point cloud needs at least one point");
  if (offsets[n] > 0 && !nbrs) return fail(LSKUM_ERR_ARGUMENT, "null argument");
  return guard([&] {
    std::vector<lskb::PointRow> rows(static_cast<std::size_t>(n));
    for (int32_t i = 0; i < n; ++i) {
      if (kind[i] > 2) lskb::raise(lskb::Status::argument, "unknown point kind at point " + std::to_string(i));
      rows[i] = lskb::PointRow{x[i], y[i], nx[i], ny[i], static_cast<lskb::Kind>(kind[i])};
    }
    std::vector<int64_t> off(offsets, offsets + n + 1);
    std::vector<int32_t> nb;
    if (nbrs) nb.assign(nbrs, nbrs + offsets[n]);
    *out = new lskum_cloud{lskb::assemble(std::move(rows), std::move(off), std::move(nb))};
  });
}

int lskum_b200_cloud_nnz(const lskum_cloud* cloud, int64_t* out) {
  NONNULL(cloud, out);
  *out = cloud->ps.nnz();
  return LSKUM_OK;
}

int lskum_b200_cloud_geometry(const lskum_cloud* cloud, double* x, double* y, uint8_t* kind, double* nx,
                              double* ny, int64_t* offsets, int32_t* nbrs) {
  NONNULL(cloud);
  const lskb::PointSet& ps = cloud->ps;
  const std::size_t n = static_cast<std::size_t>(ps.n());
  if (x) std::memcpy(x, ps.x.data(), n * sizeof(double));
  if (y) std::memcpy(y, ps.y.data(), n * sizeof(double));
  if (nx) std::memcpy(nx, ps.nx.data(), n * sizeof(double));
  if (ny) std::memcpy(ny, ps.ny.data(), n * sizeof(double));
  if (kind)
    for (std::size_t i = 0; i < n; ++i) kind[i] = static_cast<uint8_t>(ps.kind[i]);
  if (offsets) std::memcpy(offsets, ps.off.data(), (n + 1) * sizeof(int64_t));
  if (nbrs) std::memcpy(nbrs, ps.nbr.data(), ps.nbr.size() * sizeof(int32_t));
  return LSKUM_OK;
}

int lskum_b200_cloud_reset_store(lskum_cloud* cloud, int layout) {
  NONNULL(cloud);
  if (layout != 0 && layout != 1) return fail(LSKUM_ERR_ARGUMENT, "layout must be 0 (aos) or 1 (soa)");
  return guard([&] { cloud->ps.reset_fields(layout ? lskb::Layout::soa : lskb::Layout::aos); });
}

int lskum_b200_cloud_get_fields(const lskum_cloud* cloud, double* aos) {
  NONNULL(cloud, aos);
  cloud->ps.fields.export_aos(aos);
  return LSKUM_OK;
}

int lskum_b200_cloud_set_fields(lskum_cloud* cloud, const double* aos) {
  NONNULL(cloud, aos);
  cloud->ps.fields.import_aos(aos);
  return LSKUM_OK;
}

int lskum_b200_run_fixed_point(lskum_cloud* cloud, const lskum_config* cfg, lskum_result** out) {
  return run_impl(cloud, cfg, out, false);
}

int lskum_b200_result_abort_iteration(const lskum_result* r) { return r ? r->run.abort_iteration : 0; }

int lskum_b200_result_wall_ms(const lskum_result* r, int iteration, double* out) {
  NONNULL(r, out);
  if (iteration < 1 || iteration > static_cast<int>(r->run.wall_ms.size()))
    return fail(LSKUM_ERR_ARGUMENT, "iteration out of range");
  *out = r->run.wall_ms[iteration - 1];
  return LSKUM_OK;
}

static int op_impl(lskum_cloud* cloud, const lskum_b200_params* p, lskb::Op op, double* scratch,
                   int axis = 0, int sign = 0, int first = 1) {
  NONNULL(cloud, p);
  return guard([&] {
    lskb::OpSpec spec;
    spec.gamma = p->gamma;
    spec.cfl = p->cfl;
    spec.det_tol = p->det_tol;
    spec.fp_mode = p->fp_mode;
    spec.axis = axis;
    spec.sign = sign;
    spec.first = first;
    lskb::engine_op(cloud->ps, op, spec, scratch);
  });
}

int lskum_b200_op_q_variables(lskum_cloud* c, const lskum_b200_params* p) {
  return op_impl(c, p, lskb::Op::q_variables, nullptr);
}
int lskum_b200_op_q_derivatives(lskum_cloud* c, const lskum_b200_params* p, double* scratch) {
  NONNULL(scratch);
  return op_impl(c, p, lskb::Op::q_derivatives, scratch);
}
int lskum_b200_op_publish(lskum_cloud* c, const double* scratch) {
  NONNULL(scratch);
  const lskum_b200_params p{1.4, 0.5, 0.0, 0};
  return op_impl(c, &p, lskb::Op::publish, const_cast<double*>(scratch));
}
int lskum_b200_op_flux_residual(lskum_cloud* c, const lskum_b200_params* p) {
  return op_impl(c, p, lskb::Op::flux_fused, nullptr);
}
int lskum_b200_op_flux_direction(lskum_cloud* c, const lskum_b200_params* p, int axis, int sign, int first) {
  if ((axis != 0 && axis != 1) || (sign != 0 && sign != 1)) return fail(LSKUM_ERR_ARGUMENT, "bad direction");
  return op_impl(c, p, lskb::Op::flux_direction, nullptr, axis, sign, first);
}
int lskum_b200_op_timestep(lskum_cloud* c, const lskum_b200_params* p) {
  return op_impl(c, p, lskb::Op::timestep, nullptr);
}
int lskum_b200_op_state_update(lskum_cloud* c, const lskum_b200_params* p) {
  return op_impl(c, p, lskb::Op::state_update, nullptr);
}

int lskum_b200_reduce(const double* values, int64_t n, double* out) {
  if (!out || (n > 0 && !values)) return fail(LSKUM_ERR_ARGUMENT, "null argument");
  return guard([&] { *out = lskb::engine_reduce(values, n, 0); });
}

int lskum_b200_exact_sum(const double* values, int64_t n, double* out) {
  if (!out || (n > 0 && !values)) return fail(LSKUM_ERR_ARGUMENT, "null argument");
  return guard([&] { *out = lskb::engine_exact_sum(values, n, 0); });
}

int lskum_b200_partition(const lskum_cloud* cloud, int n_parts, int32_t* owner, int64_t* ghost_off,
                         int32_t* ghosts, int64_t ghost_cap) {
  NONNULL(cloud, owner, ghost_off);
  return guard([&] {
    const std::vector<lskb::Piece> pieces = lskb::bisect_cloud(cloud->ps, n_parts);
    int64_t at = 0;
    for (std::size_t p = 0; p < pieces.size(); ++p) {
      for (int32_t i : pieces[p].owned) owner[i] = static_cast<int32_t>(p);
      ghost_off[p] = at;
      for (int32_t g : pieces[p].halo) {
        if (at >= ghost_cap || !ghosts) lskb::raise(lskb::Status::argument, "ghost buffer too small");
        ghosts[at++] = g;
      }
    }
    ghost_off[pieces.size()] = at;
  });
}

// ---------------------------------------------------------------- sessions
int lskum_b200_session_create(lskum_cloud* cloud, const lskum_config* cfg, int capacity, int from_state,
                              lskum_b200_session** out) {
  NONNULL(cloud, cfg, out);
  if (capacity < 1) return fail(LSKUM_ERR_ARGUMENT, "capacity must be >= 1");
  return guard([&] {
    if (!from_state) {
      cfg->s.check();
      cloud->ps.reset_fields(cfg->s.layout);
      lskb::freestream(cloud->ps, cfg->s.mach, cfg->s.aoa, cfg->s.gamma);
    }
    const lskb::EngineSpec spec = lskb::prepare_run(cloud->ps, cfg->s);
    auto s = std::make_unique<lskum_b200_session>();
    s->cloud = cloud;
    s->session = lskb::session_open(cloud->ps, spec, capacity);
    *out = s.release();
  });
}

int lskum_b200_session_iterate(lskum_b200_session* s, int n, double* device_ms) {
  NONNULL(s);
  if (n < 0) return fail(LSKUM_ERR_ARGUMENT, "iteration count must be >= 0");
  return guard([&] {
    const double ms = n > 0 ? lskb::session_iterate(s->session, n) : 0.0;
    if (device_ms) *device_ms = ms;
  });
}

int lskum_b200_session_residues(const lskum_b200_session* s, double* out, int cap, int* n_out) {
  NONNULL(s, n_out);
  return guard([&] {
    const std::vector<double> r = lskb::session_residues(s->session);
    *n_out = static_cast<int>(r.size());
    if (out)
      for (int i = 0; i < std::min<int>(cap, static_cast<int>(r.size())); ++i) out[i] = r[i];
  });
}

int lskum_b200_session_kernel_count(const lskum_b200_session* s) {
  if (!s) return 0;
  const_cast<lskum_b200_session*>(s)->kernels = lskb::session_kernels(s->session);
  return static_cast<int>(s->kernels.size());
}

const char* lskum_b200_session_kernel_name(const lskum_b200_session* s, int index) {
  if (!s || index < 0 || index >= static_cast<int>(s->kernels.size())) return nullptr;
  return s->kernels[index].name.c_str();
}

int lskum_b200_session_kernel_stats(const lskum_b200_session* s, int index, double* seconds,
                                    int64_t* launches) {
  if (!s || index < 0 || index >= static_cast<int>(s->kernels.size()))
    return fail(LSKUM_ERR_ARGUMENT, "bad kernel index");
  if (seconds) *seconds = s->kernels[index].seconds;
  if (launches) *launches = s->kernels[index].launches;
  return LSKUM_OK;
}

int lskum_b200_session_info(const lskum_b200_session* s, int* launches_per_iter, uint64_t* stream) {
  NONNULL(s);
  if (launches_per_iter) *launches_per_iter = lskb::session_launches_per_iter(s->session);
  if (stream) *stream = lskb::session_stream(s->session);
  return LSKUM_OK;
}

int lskum_b200_session_tiles(const lskum_b200_session* s, int* staged, int* total) {
  NONNULL(s, staged, total);
  lskb::session_tiles(s->session, staged, total);
  return LSKUM_OK;
}

int lskum_b200_session_download(lskum_b200_session* s) {
  NONNULL(s);
  return guard([&] { lskb::session_download(s->session); });
}

int lskum_b200_session_event_ms(const lskum_b200_session* s, double* sweep_ms, double* flux_ms) {
  NONNULL(s, sweep_ms, flux_ms);
  return guard([&] { lskb::session_event_ms(s->session, sweep_ms, flux_ms); });
}

int lskum_b200_session_flush_l2(lskum_b200_session* s) {
  NONNULL(s);
  return guard([&] { lskb::session_flush_l2(s->session); });
}

int lskum_b200_session_step_flushed(lskum_b200_session* s, int kernel_events, double* device_ms) {
  NONNULL(s);
  return guard([&] {
    const double ms = lskb::session_step_flushed(s->session, kernel_events != 0);
    if (device_ms) *device_ms = ms;
  });
}

int lskum_b200_fp64_peak(int device, double* tflops) {
  NONNULL(tflops);
  return guard([&] { *tflops = lskb::engine_fp64_peak_tflops(device); });
}

int lskum_b200_math_selftest(int fn, const double* in, int64_t n, double* ref, double* ours) {
  if (n > 0 && (!in || !ref || !ours)) return fail(LSKUM_ERR_ARGUMENT, "null argument");
  if (fn < 0 || fn > 2) return fail(LSKUM_ERR_ARGUMENT, "fn must be 0 (erf), 1 (exp) or 2 (fast-mode erf)");
  return guard([&] { lskb::engine_math_selftest(fn, in, n, ref, ours); });
}

void lskum_b200_session_destroy(lskum_b200_session* s) { delete s; }

// ---------------------------------------------------------------- ranks
int lskum_b200_rank_create(lskum_cloud* cloud, const lskum_config* cfg, int rank, int world, int device,
                           int capacity, int from_state, lskum_b200_rank** out) {
  NONNULL(cloud, cfg, out);
  if (capacity < 1) return fail(LSKUM_ERR_ARGUMENT, "capacity must be >= 1");
  return guard([&] {
    if (!from_state) {
      cfg->s.check();
      cloud->ps.reset_fields(cfg->s.layout);
      lskb::freestream(cloud->ps, cfg->s.mach, cfg->s.aoa, cfg->s.gamma);
    }
    const lskb::EngineSpec spec = lskb::prepare_run(cloud->ps, cfg->s);
    auto r = std::make_unique<lskum_b200_rank>();
    r->run = lskb::rank_open(cloud->ps, spec, rank, world, device, capacity);
    *out = r.release();
  });
}

int lskum_b200_rank_blob_size(void) { return static_cast<int>(lskb::rank_blob_bytes()); }

int lskum_b200_rank_blob(const lskum_b200_rank* r, void* out) {
  NONNULL(r, out);
  return guard([&] {
    const std::vector<unsigned char> b = lskb::rank_blob(r->run);
    std::memcpy(out, b.data(), b.size());
  });
}

int lskum_b200_rank_connect(lskum_b200_rank* r, const void* blobs, int world) {
  NONNULL(r, blobs);
  return guard([&] {
    const std::size_t sz = lskb::rank_blob_bytes();
    const unsigned char* p = static_cast<const unsigned char*>(blobs);
    std::vector<std::vector<unsigned char>> v;
    for (int i = 0; i < world; ++i) v.emplace_back(p + i * sz, p + (i + 1) * sz);
    lskb::rank_connect(r->run, v);
  });
}

int lskum_b200_rank_iterate(lskum_b200_rank* r, int n, double* device_ms) {
  NONNULL(r);
  if (n < 0) return fail(LSKUM_ERR_ARGUMENT, "iteration count must be >= 0");
  return guard([&] {
    const double ms = n > 0 ? lskb::rank_iterate(r->run, n) : 0.0;
    if (device_ms) *device_ms = ms;
  });
}

int lskum_b200_rank_residues(const lskum_b200_rank* r, double* out, int cap, int* n_out) {
  NONNULL(r, n_out);
  return guard([&] {
    const std::vector<double> v = lskb::rank_residues(r->run);
    *n_out = static_cast<int>(v.size());
    if (out)
      for (int i = 0; i < std::min<int>(cap, static_cast<int>(v.size())); ++i) out[i] = v[i];
  });
}

int lskum_b200_rank_info(const lskum_b200_rank* r, int* launches_per_iter, uint64_t* err_stage, uint64_t* err_key,
                         int* owns_failure) {
  NONNULL(r);
  return guard([&] {
    if (launches_per_iter) *launches_per_iter = lskb::rank_launches_per_iter(r->run);
    unsigned long long st = 0, key = 0;
    int owns = 0;
    lskb::rank_error(r->run, &st, &key, &owns);
    if (err_stage) *err_stage = st;
    if (err_key) *err_key = key;
    if (owns_failure) *owns_failure = owns;
  });
}

int lskum_b200_rank_download(lskum_b200_rank* r) {
  NONNULL(r);
  return guard([&] { lskb::rank_download(r->run); });
}

int lskum_b200_rank_event_ms(const lskum_b200_rank* r, double* sweep_ms, double* flux_ms) {
  NONNULL(r, sweep_ms, flux_ms);
  return guard([&] { lskb::rank_event_ms(r->run, sweep_ms, flux_ms); });
}

int lskum_b200_rank_flush_l2(lskum_b200_rank* r) {
  NONNULL(r);
  return guard([&] { lskb::rank_flush_l2(r->run); });
}

void lskum_b200_rank_destroy(lskum_b200_rank* r) { delete r; }

}  // extern "C"
