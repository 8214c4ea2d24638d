// settings.cpp — solver/grid settings: key=value parsing, rendering, files.
//
// Key set, value syntax and error behaviour follow the reference config layer
// (config.cpp:10-162, lskum_capi.cpp:153-195): unknown keys and malformed
// values raise ErrorCode::config, the file loader strips '#' comments and
// blank lines, lskum_config_get renders reals with %.17g.  Additional keys
// for the device backend: backend, device, gpus, fp_mode, chunk, reorder.
#include <cerrno>
#include <charconv>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>

#include "core.hpp"

namespace lskb {

namespace {

double real_value(const std::string& key, const std::string& v) {
  const char* s = v.c_str();
  char* end = nullptr;
  errno = 0;
  const double d = std::strtod(s, &end);
  if (end == s || errno == ERANGE || static_cast<std::size_t>(end - s) != v.size())
    raise(Status::config, "bad numeric value for " + key + ": '" + v + "'");
  return d;
}

std::int64_t int_value(const std::string& key, const std::string& v) {
  std::int64_t out = 0;
  const auto r = std::from_chars(v.data(), v.data() + v.size(), out);
  if (r.ec != std::errc{} || r.ptr != v.data() + v.size())
    raise(Status::config, "bad integer value for " + key + ": '" + v + "'");
  return out;
}

std::pair<int, int> dims_value(const std::string& key, const std::string& text) {
  const auto x = text.find('x');
  if (x == std::string::npos)
    raise(Status::config, "bad " + key + " spec '" + text + "' (expected NXxNY)");
  return {static_cast<int>(int_value(key, text.substr(0, x))),
          static_cast<int>(int_value(key, text.substr(x + 1)))};
}

std::string trim(const std::string& s, const char* ws) {
  const auto b = s.find_first_not_of(ws);
  if (b == std::string::npos) return {};
  const auto e = s.find_last_not_of(ws);
  return s.substr(b, e - b + 1);
}

std::string real_text(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

}  // namespace

void Settings::check() const {
  if (!(mach >= 0.0)) raise(Status::config, "mach must be >= 0");
  if (!(gamma > 1.0)) raise(Status::config, "gamma must be > 1");
  if (iters < 0) raise(Status::config, "iters must be >= 0");
  if (inner < 1) raise(Status::config, "inner must be >= 1");
  if (!(cfl > 0.0)) raise(Status::config, "cfl must be > 0");
  if (order != 1 && order != 2) raise(Status::config, "order must be 1 or 2");
  if (parts < 1) raise(Status::config, "parts must be >= 1");
  // The device failure key orders 4096 partitions (kernels.cuh err_key); the
  // reference accepts any count, but more pieces than that only exist for
  // clouds of millions of points split for nothing but the tie-break.
  if (parts > 4096) raise(Status::config, "parts must be <= 4096");
  if (workers < 1) raise(Status::config, "workers must be >= 1");
  if (device < 0) raise(Status::config, "device must be >= 0");
  if (gpus < 1) raise(Status::config, "gpus must be >= 1");
  if (chunk < 1) raise(Status::config, "chunk must be >= 1");
}

void Settings::set(const std::string& key, const std::string& v) {
  if (key == "mach") mach = real_value(key, v);
  else if (key == "aoa") aoa = real_value(key, v);
  else if (key == "gamma") gamma = real_value(key, v);
  else if (key == "iters") iters = static_cast<int>(int_value(key, v));
  else if (key == "inner") inner = static_cast<int>(int_value(key, v));
  else if (key == "cfl") cfl = real_value(key, v);
  else if (key == "order") order = static_cast<int>(int_value(key, v));
  else if (key == "layout") {
    if (v == "aos") layout = Layout::aos;
    else if (v == "soa") layout = Layout::soa;
    else raise(Status::config, "unknown layout '" + v + "' (expected aos or soa)");
  } else if (key == "residual_mode") {
    if (v == "fused") residual_split4 = 0;
    else if (v == "split4") residual_split4 = 1;
    else raise(Status::config, "unknown residual mode '" + v + "' (expected fused or split4)");
  } else if (key == "parts") parts = static_cast<int>(int_value(key, v));
  else if (key == "workers") workers = static_cast<int>(int_value(key, v));
  else if (key == "out_prefix") out_prefix = v;
  else if (key == "grid") grid = v;
  else if (key == "generate") generate = v;
  else if (key == "jitter") jitter = real_value(key, v);
  else if (key == "seed") seed = static_cast<std::uint64_t>(int_value(key, v));
  else if (key == "knn") knn = static_cast<int>(int_value(key, v));
  else if (key == "outer_radius") outer_radius = real_value(key, v);
  else if (key == "bounds") {
    std::istringstream in(v);
    char c1 = 0, c2 = 0, c3 = 0;
    Box b;
    if (!(in >> b.xmin >> c1 >> b.xmax >> c2 >> b.ymin >> c3 >> b.ymax) || c1 != ',' || c2 != ',' || c3 != ',')
      raise(Status::config, "bad bounds '" + v + "' (expected xmin,xmax,ymin,ymax)");
    bounds = b;
  } else if (key == "backend") {
    if (v != "cuda") raise(Status::config, "unknown backend '" + v + "' (this build runs cuda only)");
  } else if (key == "device") device = static_cast<int>(int_value(key, v));
  else if (key == "gpus") gpus = static_cast<int>(int_value(key, v));
  else if (key == "fp_mode") {
    if (v == "fast") fp_mode = 0;
    else if (v == "strict") fp_mode = 1;
    else raise(Status::config, "unknown fp_mode '" + v + "' (expected fast or strict)");
  } else if (key == "chunk") chunk = static_cast<int>(int_value(key, v));
  else if (key == "reorder") {
    if (v == "none") reorder = 0;
    else if (v == "hilbert") reorder = 1;
    else if (v == "auto") reorder = 2;
    else if (v == "rcm") reorder = 3;
    else raise(Status::config, "unknown reorder '" + v + "' (expected none, hilbert, rcm or auto)");
  } else raise(Status::config, "unknown config key '" + key + "'");
}

std::string Settings::get(const std::string& key) const {
  if (key == "mach") return real_text(mach);
  if (key == "aoa") return real_text(aoa);
  if (key == "gamma") return real_text(gamma);
  if (key == "iters") return std::to_string(iters);
  if (key == "inner") return std::to_string(inner);
  if (key == "cfl") return real_text(cfl);
  if (key == "order") return std::to_string(order);
  if (key == "layout") return layout == Layout::aos ? "aos" : "soa";
  if (key == "residual_mode") return residual_split4 ? "split4" : "fused";
  if (key == "parts") return std::to_string(parts);
  if (key == "workers") return std::to_string(workers);
  if (key == "out_prefix") return out_prefix;
  if (key == "grid") return grid;
  if (key == "generate") return generate;
  if (key == "jitter") return real_text(jitter);
  if (key == "seed") return std::to_string(static_cast<long long>(seed));
  if (key == "knn") return std::to_string(knn);
  if (key == "outer_radius") return real_text(outer_radius);
  if (key == "bounds")
    return real_text(bounds.xmin) + "," + real_text(bounds.xmax) + "," + real_text(bounds.ymin) + "," +
           real_text(bounds.ymax);
  if (key == "backend") return "cuda";
  if (key == "device") return std::to_string(device);
  if (key == "gpus") return std::to_string(gpus);
  if (key == "fp_mode") return fp_mode ? "strict" : "fast";
  if (key == "chunk") return std::to_string(chunk);
  if (key == "reorder") {
    static const char* names[] = {"none", "hilbert", "auto", "rcm"};
    return names[reorder & 3];
  }
  raise(Status::config, "unknown config key '" + key + "'");
}

void Settings::load(const std::string& path) {
  std::ifstream in(path);
  if (!in) raise(Status::io, "cannot open config file: " + path);
  std::string line;
  long long no = 0;
  while (std::getline(in, line)) {
    ++no;
    const auto hash = line.find('#');
    if (hash != std::string::npos) line.resize(hash);
    const std::string t = trim(line, " \t\r");
    if (t.empty()) continue;
    const auto eq = t.find('=');
    if (eq == std::string::npos)
      raise(Status::config, path + ":" + std::to_string(no) + ": expected key=value, got '" + t + "'");
    set(trim(t.substr(0, eq), " \t"), trim(t.substr(eq + 1), " \t"));
  }
}

PointSet acquire_points(const Settings& s) {
  const bool file = !s.grid.empty(), gen = !s.generate.empty();
  if (file == gen) raise(Status::config, "exactly one of grid path or generator spec required");
  if (file) return read_grid_file(s.grid);
  // extension: naca0012:<n_wall>x<n_rings>[:frozen] (the reference
  // rejects the spec as a malformed rect size)
  const std::string naca = "naca0012:";
  if (s.generate.rfind(naca, 0) == 0) {
    std::string rest = s.generate.substr(naca.size());
    bool frozen = false;
    const std::string fz = ":frozen";
    if (rest.size() > fz.size() && rest.compare(rest.size() - fz.size(), fz.size(), fz) == 0) {
      frozen = true;
      rest.resize(rest.size() - fz.size());
    }
    const auto [nw, nr] = dims_value("generate", rest);
    return make_naca0012(nw, nr, s.outer_radius, s.jitter, s.seed, s.knn, frozen);
  }
  const std::string ring = "annulus:";
  if (s.generate.rfind(ring, 0) == 0) {
    const auto [nt, nr] = dims_value("generate", s.generate.substr(ring.size()));
    return make_annulus(nt, nr, s.outer_radius, s.jitter, s.seed, s.knn);
  }
  const auto [nx, ny] = dims_value("generate", s.generate);
  return make_rect(nx, ny, s.bounds, s.jitter, s.seed, s.knn);
}

}  // namespace lskb
