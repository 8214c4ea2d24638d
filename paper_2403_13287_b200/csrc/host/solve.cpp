// solve.cpp — host driver of one run (reference run_fixed_point,
// runtime.cpp:195-275): config check, stencil screening gate, bisection into
// `parts` pieces (the pieces fix the error tie-break order and, with gpus > 1,
// the device domains), then the device loop.
#include <cmath>
#include <cstdlib>
#include <algorithm>

#include "../engine.hpp"
#include "core.hpp"

namespace lskb {

namespace {

// lskum_run screens on the device (LSKUM_DEVICE_SCREEN=0: on the host).
bool device_screening() {
  static const bool on = [] {
    const char* e = std::getenv("LSKUM_DEVICE_SCREEN");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

EngineSpec spec_from(const PointSet& ps, const Settings& s, double det_tol) {
  EngineSpec spec;
  spec.gamma = s.gamma;
  spec.cfl = s.cfl;
  spec.det_tol = det_tol;
  spec.iters = s.iters;
  spec.inner = s.inner;
  spec.order = s.order;
  spec.fp_mode = s.fp_mode;
  spec.split4 = s.residual_split4;
  spec.chunk = s.chunk;
  spec.device = s.device;
  spec.gpus = s.gpus;
  spec.reorder = s.reorder;
  if (s.parts > ps.n())
    raise(Status::argument, "more partitions than points (" + std::to_string(s.parts) + " > " +
                                std::to_string(ps.n()) + ")");
  if (s.parts <= 1) return spec;  // one piece: every point is in partition 0
  const std::vector<Piece> pieces = bisect_cloud(ps, s.parts);
  {
    spec.part_of.assign(static_cast<std::size_t>(ps.n()), 0);
    for (std::size_t p = 0; p < pieces.size(); ++p)
      for (std::int32_t i : pieces[p].owned)
        spec.part_of[i] = static_cast<std::uint16_t>(p);
  }
  return spec;
}

}  // namespace

EngineSpec prepare_run(const PointSet& ps, const Settings& s) {
  s.check();
  if (!ps.screening) ps.screening = std::make_shared<const Screening>(screen_stencils(ps));
  const Screening& scr = *ps.screening;
  trace("prepare: screened");
  if (scr.n_defective > 0)
    raise(Status::validation, "cloud has " + std::to_string(scr.n_defective) +
                                  " defective stencils (first at point " +
                                  std::to_string(scr.defective.front()) + ")");
  EngineSpec spec = spec_from(ps, s, scr.det_tol);
  trace("prepare: partitioned");
  return spec;
}

RunRecord solve_from_freestream(PointSet& ps, const Settings& s) {
  s.check();
  if (s.gpus > 1 || s.iters <= 0) {
    ps.reset_fields(s.layout);
    freestream(ps, s.mach, s.aoa, s.gamma);
    return solve_on_device(ps, s);
  }
  bool written = false;
  try {
    if (!ps.screening && device_screening()) {
      try {
        engine_prescreen(ps, s);
      } catch (const Fault&) {
        // no usable device: screen on the host, so a defective cloud still
        // reports LSKUM_ERR_VALIDATION before any device error
      }
    }
    EngineSpec spec = prepare_run(ps, s);
    if (!(ps.fields.size() == ps.n() && ps.fields.layout() == s.layout)) ps.fields = FieldBlock(s.layout, ps.n());
    const double a = s.aoa * M_PI / 180.0;  // freestream_init, bench.cpp:43-56
    spec.fs_device = true;
    spec.fs_prim[0] = 1.0;
    spec.fs_prim[1] = s.mach * std::cos(a);
    spec.fs_prim[2] = s.mach * std::sin(a);
    spec.fs_prim[3] = 1.0 / s.gamma;
    spec.store_written = &written;
    return engine_run(ps, spec);
  } catch (...) {
    if (!written) {
      ps.reset_fields(s.layout);
      freestream(ps, s.mach, s.aoa, s.gamma);
    }
    throw;
  }
}

RunRecord solve_on_device(PointSet& ps, const Settings& s) {
  const EngineSpec spec = prepare_run(ps, s);
  if (s.gpus > 1) {
    if (s.gpus > ps.n()) raise(Status::config, "more gpus than points");
    const std::vector<LocalGeom> geoms = decompose(ps, s.gpus, spec.part_of, spec.reorder);
    trace("prepare: decomposed");
    return engine_run_multi(ps, spec, geoms);
  }
  return engine_run(ps, spec);
}

}  // namespace lskb
