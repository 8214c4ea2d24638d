// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (oracle side, never shipped).
//
// A thin extern "C" shim over the *unmodified* reference core
// (/root/reference/proj/src/core, compiled by oracle/Makefile into
// oracle/_ref/liblskum_core.a).  It exposes the reference's internal
// per-phase operators (src/core/kernels.hpp:25-63), validation
// (src/core/cloud.cpp:252-321), partitioning (src/core/partition.cpp:48-80),
// the deterministic reduce (src/core/reduce.hpp:11-17) and the fixed-point
// driver (src/core/runtime.cpp:195-275) on plain arrays, so the parity tests
// can feed the reference and the CUDA path bit-identical inputs.  The public
// C ABI of the reference (liblskum.so) cannot do that: lskum_run always
// re-initialises the free stream (src/capi/lskum_capi.cpp:209-220).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "core/bench.hpp"
#include "core/cloud.hpp"
#include "core/config.hpp"
#include "core/error.hpp"
#include "core/kernels.hpp"
#include "core/kinetic.hpp"
#include "core/partition.hpp"
#include "core/reduce.hpp"
#include "core/runtime.hpp"

using namespace lskum;

namespace {

void put_err(char* err, int cap, const std::string& s) {
  if (!err || cap <= 0) return;
  std::snprintf(err, static_cast<size_t>(cap), "%s", s.c_str());
}

PointCloud make_cloud(int32_t n, const double* x, const double* y, const uint8_t* kind,
                      const double* nx, const double* ny, const int64_t* off,
                      const int32_t* ids) {
  std::vector<PointRecord> recs(n);
  for (int32_t i = 0; i < n; ++i) {
    PointRecord& r = recs[i];
    r.id = i;
    r.x = x[i];
    r.y = y[i];
    r.kind = static_cast<PointKind>(kind[i]);
    r.nx = nx[i];
    r.ny = ny[i];
    r.nbhs.assign(ids + off[i], ids + off[i + 1]);
  }
  return PointCloud(std::move(recs));
}

void store_in(FieldStore& s, const double* aos) {
  for (int32_t i = 0; i < s.n_points(); ++i)
    for (int k = 0; k < slot::count; ++k) s.at(i, k) = aos[static_cast<size_t>(i) * slot::count + k];
}

void store_out(const FieldStore& s, double* aos) {
  for (int32_t i = 0; i < s.n_points(); ++i)
    for (int k = 0; k < slot::count; ++k) aos[static_cast<size_t>(i) * slot::count + k] = s.at(i, k);
}

struct Generated {
  PointCloud cloud;
};

}  // namespace

#define CLOUD_ARGS                                                                    \
  int32_t n, const double *x, const double *y, const uint8_t *kind, const double *nx, \
      const double *ny, const int64_t *off, const int32_t *ids
#define CLOUD_PASS n, x, y, kind, nx, ny, off, ids

extern "C" {

// which: 0 q_variables, 1 q_derivatives (-> scratch n*8), 2 publish (scratch -> store),
//        3 flux fused, 4 flux direction(axis, sign, first), 5 timestep, 6 state_update
int refshim_kernel(int which, CLOUD_ARGS, double* store_aos, double gamma, double cfl,
                   double det_tol, double* scratch, int axis, int sign, int first,
                   char* err, int errcap) {
  try {
    PointCloud cloud = make_cloud(CLOUD_PASS);
    cloud.reset_store(Layout::aos);
    store_in(cloud.store(), store_aos);
    KernelParams p{GasModel{gamma}, cfl, det_tol};
    std::vector<int32_t> all(n);
    std::iota(all.begin(), all.end(), 0);
    std::span<const int32_t> span(all);
    int rc = 0;
    try {
      switch (which) {
        case 0: q_variables_kernel(cloud, cloud.store(), span, p); break;
        case 1: q_derivatives_kernel(cloud, cloud.store(), span, p, scratch); break;
        case 2: publish_q_derivatives(cloud.store(), span, scratch); break;
        case 3: flux_residual_fused_kernel(cloud, cloud.store(), span, p); break;
        case 4:
          flux_residual_direction_kernel(cloud, cloud.store(), span, p,
                                         axis ? Axis::y : Axis::x,
                                         sign ? FluxSign::minus : FluxSign::plus, first != 0);
          break;
        case 5: local_timestep_kernel(cloud, cloud.store(), span, p); break;
        case 6: state_update_kernel(cloud, cloud.store(), span, p); break;
        default: put_err(err, errcap, "bad kernel id"); return 1;
      }
    } catch (const Error& e) {
      put_err(err, errcap, e.what());
      rc = static_cast<int>(e.code());
    }
    store_out(cloud.store(), store_aos);
    return rc;
  } catch (const Error& e) {
    put_err(err, errcap, e.what());
    return static_cast<int>(e.code());
  }
}

int refshim_validate(CLOUD_ARGS, int32_t* defective, int32_t* n_defective,
                     int32_t* n_wall_isolated, int32_t* min_stencil, double* h_ref,
                     double* det_tol, double* full_det, double* split_det) {
  try {
    PointCloud cloud = make_cloud(CLOUD_PASS);
    const ValidationReport r = validate_cloud(cloud);
    *n_defective = r.n_defective;
    *n_wall_isolated = r.n_wall_isolated;
    *min_stencil = r.min_stencil_size;
    *h_ref = r.h_ref;
    *det_tol = r.det_tol;
    for (size_t i = 0; i < r.defective_ids.size(); ++i) defective[i] = r.defective_ids[i];
    if (full_det)
      for (int32_t i = 0; i < n; ++i) full_det[i] = r.points[i].full_det;
    if (split_det)
      for (int32_t i = 0; i < n; ++i)
        for (int d = 0; d < 4; ++d) split_det[4 * i + d] = r.points[i].split_det[d];
    return 0;
  } catch (const Error& e) {
    return static_cast<int>(e.code());
  }
}

// owner[i] = part of point i; ghosts flattened per part, counts in ghost_count[p].
int refshim_partition(CLOUD_ARGS, int n_parts, int32_t* owner, int32_t* ghost_count,
                      int32_t* ghosts, int64_t ghost_cap) {
  try {
    PointCloud cloud = make_cloud(CLOUD_PASS);
    const Partitioning parts = partition_cloud(cloud, n_parts);
    int64_t at = 0;
    for (int p = 0; p < parts.n_parts(); ++p) {
      for (int32_t i : parts.parts[p].locals) owner[i] = p;
      ghost_count[p] = static_cast<int32_t>(parts.parts[p].ghosts.size());
      for (int32_t g : parts.parts[p].ghosts) {
        if (at >= ghost_cap) return 1;
        ghosts[at++] = g;
      }
    }
    return 0;
  } catch (const Error& e) {
    return static_cast<int>(e.code());
  }
}

double refshim_reduce(const double* v, int64_t n) {
  return deterministic_reduce(0, n, [v](int64_t i) { return v[i]; });
}

// Runs run_fixed_point from the given primitive state (n*4, or null for the
// free stream), returning the full AoS store, the residue history and the
// error (status code + message) if the run aborted.
int refshim_run(CLOUD_ARGS, double mach, double aoa, double gamma, int iters, int inner,
                double cfl, int order, int layout, int mode, int parts, int workers,
                const double* prim0, double* store_aos, double* residue, int* n_done,
                double* total_seconds, char* err, int errcap) {
  try {
    PointCloud cloud = make_cloud(CLOUD_PASS);
    SolverConfig cfg;
    cfg.mach = mach;
    cfg.aoa_deg = aoa;
    cfg.gamma = gamma;
    cfg.iters = iters;
    cfg.n_inner = inner;
    cfg.cfl = cfl;
    cfg.order = order;
    cfg.layout = layout ? Layout::soa : Layout::aos;
    cfg.residual_mode = mode ? ResidualMode::split4 : ResidualMode::fused;
    cfg.n_parts = parts;
    cfg.n_workers = workers;
    cloud.reset_store(cfg.layout);
    freestream_init(cloud, mach, aoa, GasModel{gamma});
    if (prim0) {
      for (int32_t i = 0; i < n; ++i)
        for (int c = 0; c < 4; ++c) cloud.store().at(i, slot::prim + c) = prim0[4 * i + c];
    }
    int rc = 0;
    *n_done = 0;
    try {
      RunResult r = run_fixed_point(cloud, cfg);
      *n_done = r.iterations;
      for (size_t i = 0; i < r.history.residue.size(); ++i) residue[i] = r.history.residue[i];
      if (total_seconds) *total_seconds = r.total_seconds;
    } catch (const Error& e) {
      put_err(err, errcap, e.what());
      rc = static_cast<int>(e.code());
    }
    store_out(cloud.store(), store_aos);
    return rc;
  } catch (const Error& e) {
    put_err(err, errcap, e.what());
    return static_cast<int>(e.code());
  }
}

// ---- generated clouds (handle based) ----
void* refshim_generate_rect(int nx, int ny, double xmin, double xmax, double ymin,
                            double ymax, double jitter, uint64_t seed, int k) {
  try {
    return new Generated{generate_rect_cloud(nx, ny, RectBounds{xmin, xmax, ymin, ymax},
                                             jitter, seed, k)};
  } catch (...) {
    return nullptr;
  }
}

void* refshim_generate_annulus(int nt, int nr, double r_outer, double jitter, uint64_t seed,
                               int k) {
  try {
    return new Generated{generate_annulus_cloud(nt, nr, r_outer, jitter, seed, k)};
  } catch (...) {
    return nullptr;
  }
}

// The reference's kNN (build_stencils, cloud.cpp:137-237) on arbitrary points
// (kind interior, zero normals), e.g. the NACA 0012 clouds it cannot generate.
void* refshim_knn(int32_t n, const double* x, const double* y, int k) {
  try {
    std::vector<PointRecord> recs(n);
    for (int32_t i = 0; i < n; ++i) {
      recs[i].id = i;
      recs[i].x = x[i];
      recs[i].y = y[i];
    }
    PointCloud c(std::move(recs));
    build_stencils(c, k);
    return new Generated{std::move(c)};
  } catch (...) {
    return nullptr;
  }
}

void refshim_cloud_sizes(void* h, int32_t* n, int64_t* nnz) {
  const PointCloud& c = static_cast<Generated*>(h)->cloud;
  *n = c.n_points();
  int64_t t = 0;
  for (int32_t i = 0; i < c.n_points(); ++i) t += static_cast<int64_t>(c.nbhs(i).size());
  *nnz = t;
}

void refshim_cloud_get(void* h, double* x, double* y, uint8_t* kind, double* nx, double* ny,
                       int64_t* off, int32_t* ids) {
  const PointCloud& c = static_cast<Generated*>(h)->cloud;
  int64_t at = 0;
  off[0] = 0;
  for (int32_t i = 0; i < c.n_points(); ++i) {
    x[i] = c.x(i);
    y[i] = c.y(i);
    kind[i] = static_cast<uint8_t>(c.kind(i));
    nx[i] = c.normal_x(i);
    ny[i] = c.normal_y(i);
    for (int32_t nb : c.nbhs(i)) ids[at++] = nb;
    off[i + 1] = at;
  }
}

void refshim_cloud_free(void* h) { delete static_cast<Generated*>(h); }

// ---- per-point kinetic math (src/core/kinetic.cpp) ----
// op: 0 q_from_prim, 1 prim_from_q, 2 cons_from_prim, 3 prim_from_cons,
//     4 full_flux(axis), 5 kfvs(axis, sign)
int refshim_kinetic(int op, const double* in, double* out, int axis, int sign, double gamma) {
  GasModel g{gamma};
  try {
    switch (op) {
      case 0: {
        QState q = q_from_primitives({in[0], in[1], in[2], in[3]}, g);
        out[0] = q.q0; out[1] = q.q1; out[2] = q.q2; out[3] = q.q3;
        return 0;
      }
      case 1: {
        PrimitiveState s = primitives_from_q({in[0], in[1], in[2], in[3]}, g);
        out[0] = s.rho; out[1] = s.u1; out[2] = s.u2; out[3] = s.p;
        return 0;
      }
      case 2: {
        ConservedState u = conserved_from_primitives({in[0], in[1], in[2], in[3]}, g);
        out[0] = u.mass; out[1] = u.mom_x; out[2] = u.mom_y; out[3] = u.energy;
        return 0;
      }
      case 3: {
        PrimitiveState s = primitives_from_conserved({in[0], in[1], in[2], in[3]}, g);
        out[0] = s.rho; out[1] = s.u1; out[2] = s.u2; out[3] = s.p;
        return 0;
      }
      case 4: {
        Vec4 f = full_flux({in[0], in[1], in[2], in[3]}, axis ? Axis::y : Axis::x, g);
        for (int c = 0; c < 4; ++c) out[c] = f[c];
        return 0;
      }
      case 5: {
        Vec4 f = kfvs_split_flux({in[0], in[1], in[2], in[3]}, axis ? Axis::y : Axis::x,
                                 sign ? FluxSign::minus : FluxSign::plus, g);
        for (int c = 0; c < 4; ++c) out[c] = f[c];
        return 0;
      }
      default: return 1;
    }
  } catch (const Error& e) {
    return static_cast<int>(e.code());
  }
}

}  // extern "C"
