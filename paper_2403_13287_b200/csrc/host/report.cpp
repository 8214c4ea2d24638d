// report.cpp — initial state, metrics and output files.
//
// Free-stream initialisation (reference bench.cpp:43-56), RDP and relative
// performance (:58-70), the per-kernel report with the split4 aggregate row
// (:72-99), Cp (:101-105) and the four output files with the reference's
// exact formats (:107-183): .residue.csv, .solution.dat, .bench.csv,
// .surface.csv.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <filesystem>

#include "core.hpp"
#include "par.hpp"

namespace lskb {

namespace {

class OutFile {
 public:
  explicit OutFile(const std::string& path) : path_(path) {
    const std::filesystem::path parent = std::filesystem::path(path).parent_path();
    if (!parent.empty()) {
      std::error_code ec;
      std::filesystem::create_directories(parent, ec);
    }
    f_ = std::fopen(path.c_str(), "wb");
    if (!f_) raise(Status::io, "cannot open output file: " + path);
  }
  ~OutFile() {
    if (f_) std::fclose(f_);
  }
  void put(const char* fmt, ...) __attribute__((format(printf, 2, 3))) {
    va_list ap;
    va_start(ap, fmt);
    if (std::vfprintf(f_, fmt, ap) < 0) ok_ = false;
    va_end(ap);
  }
  void close() {
    const bool closed = std::fclose(f_) == 0;
    f_ = nullptr;
    if (!closed || !ok_) raise(Status::io, "failed writing output file: " + path_);
  }

 private:
  std::string path_;
  std::FILE* f_ = nullptr;
  bool ok_ = true;
};

}  // namespace

void freestream(PointSet& ps, double mach, double aoa_deg, double gamma) {
  const double a = aoa_deg * M_PI / 180.0;
  const double u1 = mach * std::cos(a), u2 = mach * std::sin(a), p = 1.0 / gamma;
  parallel_slices(ps.n(), [&](std::int64_t lo, std::int64_t hi) {
    for (std::int64_t i = lo; i < hi; ++i) {
      const std::int32_t k = static_cast<std::int32_t>(i);
      ps.fields.at(k, slot::prim) = 1.0;
      ps.fields.at(k, slot::prim + 1) = u1;
      ps.fields.at(k, slot::prim + 2) = u2;
      ps.fields.at(k, slot::prim + 3) = p;
    }
  }, 1 << 16);
}

double rate_of_data_processing(double seconds, std::int64_t iters, std::int64_t n) {
  if (iters <= 0 || n <= 0) raise(Status::argument, "rdp needs positive iteration and point counts");
  return seconds / static_cast<double>(iters) / static_cast<double>(n);
}

double relative_rate(double rdp_test, double rdp_ref) {
  if (rdp_ref == 0.0) raise(Status::argument, "relative performance needs a nonzero reference");
  return rdp_test / rdp_ref;
}

double pressure_coeff(double p, double mach, double gamma) {
  if (mach == 0.0) return 0.0;
  return (p - 1.0 / gamma) / (0.5 * mach * mach);
}

Report summarize(const RunRecord& run, std::int32_t n) {
  Report rep;
  rep.iterations = run.iterations;
  rep.n = n;
  rep.total_seconds = run.total_seconds;
  const bool rate = run.iterations > 0 && n > 0;
  rep.total_rdp = rate ? rate_of_data_processing(run.total_seconds, run.iterations, n) : 0.0;
  double split_s = 0.0, split_r = 0.0;
  bool split = false;
  for (const KernelTime& k : run.kernels) {
    KernelRow row{k.name, k.seconds, rate ? rate_of_data_processing(k.seconds, run.iterations, n) : 0.0};
    if (k.name.rfind("flux_residual_", 0) == 0) {
      split = true;
      split_s += row.seconds;
      split_r += row.rdp;
    }
    rep.rows.push_back(row);
  }
  if (split) rep.rows.push_back({"flux_residual", split_s, split_r});
  return rep;
}

// Surface force coefficients (new: the reference has Cp only,
// bench.cpp:101-105).  The surface is the closed polygon through `loop`
// (point ids in order; empty = the wall points in id order, the generators'
// boundary order).  Each panel carries the mean Cp of its end points; the
// force on the body is -sum Cp n ds over panels, n the panel normal pointing
// out of the enclosed body region; coefficients are per unit chord (the
// loop's x extent) in the free-stream frame: Cl normal to it, Cd along it,
// Cm about the quarter chord (positive nose up).
Forces surface_forces(const PointSet& ps, const std::vector<std::int32_t>& loop_in, double mach, double aoa_deg,
                      double gamma) {
  std::vector<std::int32_t> loop = loop_in;
  if (loop.empty())
    for (std::int32_t i = 0; i < ps.n(); ++i)
      if (ps.kind[i] == Kind::wall) loop.push_back(i);
  if (loop.size() < 3) raise(Status::argument, "surface forces need a closed loop of >= 3 surface points");
  for (std::int32_t p : loop)
    if (p < 0 || p >= ps.n()) raise(Status::argument, "surface point id out of range");
  if (mach == 0.0) raise(Status::argument, "force coefficients need a nonzero Mach number");
  const std::size_t m = loop.size();
  double area2 = 0.0, xmin = ps.x[loop[0]], xmax = xmin, ylead = ps.y[loop[0]];
  for (std::size_t k = 0; k < m; ++k) {
    const std::int32_t a = loop[k], b = loop[(k + 1) % m];
    area2 += ps.x[a] * ps.y[b] - ps.x[b] * ps.y[a];
    if (ps.x[a] < xmin) {
      xmin = ps.x[a];
      ylead = ps.y[a];
    }
    xmax = std::max(xmax, ps.x[a]);
  }
  const double chord = xmax - xmin;
  if (!(chord > 0.0)) raise(Status::argument, "degenerate surface loop (zero chord)");
  const double orient = area2 > 0.0 ? 1.0 : -1.0;  // counter-clockwise: outward normal (dy, -dx)
  const double xr = xmin + 0.25 * chord, yr = ylead;
  double fx = 0.0, fy = 0.0, mz = 0.0;
  for (std::size_t k = 0; k < m; ++k) {
    const std::int32_t a = loop[k], b = loop[(k + 1) % m];
    const double cp = 0.5 * (pressure_coeff(ps.fields.at(a, slot::prim + 3), mach, gamma) +
                             pressure_coeff(ps.fields.at(b, slot::prim + 3), mach, gamma));
    const double dx = ps.x[b] - ps.x[a], dy = ps.y[b] - ps.y[a];
    const double px = -cp * orient * dy, py = cp * orient * dx;  // -cp * n ds
    fx += px;
    fy += py;
    const double cx = 0.5 * (ps.x[a] + ps.x[b]) - xr, cy = 0.5 * (ps.y[a] + ps.y[b]) - yr;
    mz += cx * py - cy * px;
  }
  const double a = aoa_deg * M_PI / 180.0;
  Forces f;
  f.cl = (fy * std::cos(a) - fx * std::sin(a)) / chord;
  f.cd = (fx * std::cos(a) + fy * std::sin(a)) / chord;
  f.cm = -mz / (chord * chord);
  f.chord = chord;
  f.points = static_cast<std::int32_t>(m);
  return f;
}

void write_run_outputs(const std::string& prefix, const PointSet& ps, const RunRecord& run,
                       const Report& rep, const Settings& s) {
  {
    OutFile f(prefix + ".residue.csv");
    f.put("iter,residue,log10rel,wall_ms\n");
    for (std::size_t i = 0; i < run.residue.size(); ++i)
      f.put("%zu,%.17g,%.17g,%.3f\n", i + 1, run.residue[i], run.log10_rel[i],
            i < run.wall_ms.size() ? run.wall_ms[i] : 0.0);
    f.close();
  }
  {
    OutFile f(prefix + ".solution.dat");
    f.put("# id x y rho u1 u2 p\n");
    for (std::int32_t i = 0; i < ps.n(); ++i)
      f.put("%d %.17g %.17g %.17g %.17g %.17g %.17g\n", i, ps.x[i], ps.y[i], ps.fields.at(i, slot::prim),
            ps.fields.at(i, slot::prim + 1), ps.fields.at(i, slot::prim + 2), ps.fields.at(i, slot::prim + 3));
    f.close();
  }
  {
    OutFile f(prefix + ".bench.csv");
    f.put("kernel,seconds,rdp\n");
    for (const KernelRow& k : rep.rows) f.put("%s,%.9g,%.9g\n", k.name.c_str(), k.seconds, k.rdp);
    f.put("total,%.9g,%.9g\n", rep.total_seconds, rep.total_rdp);
    f.close();
  }
  if (ps.has_wall()) {
    OutFile f(prefix + ".surface.csv");
    f.put("arc_position,cp\n");
    double arc = 0.0, px = 0.0, py = 0.0;
    bool have = false;
    for (std::int32_t i = 0; i < ps.n(); ++i) {
      if (ps.kind[i] != Kind::wall) continue;
      if (have) {
        const double dx = ps.x[i] - px, dy = ps.y[i] - py;
        arc += std::sqrt(dx * dx + dy * dy);
      }
      px = ps.x[i];
      py = ps.y[i];
      have = true;
      f.put("%.17g,%.17g\n", arc, pressure_coeff(ps.fields.at(i, slot::prim + 3), s.mach, s.gamma));
    }
    f.close();
  }
}

}  // namespace lskb
