// pointset.cpp — field block, point-set assembly and the grid-file format.
//
// Field block semantics follow reference layout.cpp:8-45; assembly checks
// follow cloud.cpp:42-83; the text format and its diagnostics follow
// cloud.cpp:427-545 (header `n`, then `id x y kind nx ny n_nbhs nbh...` per
// line, reals written with %.17g).  The parser is a single-pass scanner over
// the whole file (no per-line stream objects), so 10M-point grids load in
// seconds; error messages name the offending line as the reference does.
#include <algorithm>
#include <charconv>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>

#include "core.hpp"
#include "par.hpp"

namespace lskb {

void trace(const char* what) {
  static const bool on = std::getenv("LSKUM_TRACE") != nullptr;
  if (!on) return;
  static const auto t0 = std::chrono::steady_clock::now();
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  std::fprintf(stderr, "[lskum %10.3f ms] %s\n", ms, what);
}

std::string fmt_f(double v) {
  char buf[512];
  std::snprintf(buf, sizeof buf, "%f", v);
  return buf;
}

FieldBlock::FieldBlock(Layout layout, std::int32_t n) : layout_(layout), n_(n) {
  if (n <= 0) raise(Status::argument, "field store needs n_points > 0, got " + std::to_string(n));
  data_.assign(static_cast<std::size_t>(n) * slot::count, 0.0);
}

void FieldBlock::export_aos(double* out) const {
  if (layout_ == Layout::aos) {
    std::memcpy(out, data_.data(), data_.size() * sizeof(double));
    return;
  }
  for (std::int32_t p = 0; p < n_; ++p)
    for (int s = 0; s < slot::count; ++s) out[static_cast<std::size_t>(p) * slot::count + s] = at(p, s);
}

void FieldBlock::import_aos(const double* in) {
  if (layout_ == Layout::aos) {
    std::memcpy(data_.data(), in, data_.size() * sizeof(double));
    return;
  }
  for (std::int32_t p = 0; p < n_; ++p)
    for (int s = 0; s < slot::count; ++s) at(p, s) = in[static_cast<std::size_t>(p) * slot::count + s];
}

bool fields_identical(const FieldBlock& a, const FieldBlock& b) {
  if (a.size() != b.size())
    raise(Status::argument, "store capacity mismatch: " + std::to_string(a.size()) + " vs " +
                                std::to_string(b.size()));
  for (std::int32_t p = 0; p < a.size(); ++p)
    for (int s = 0; s < slot::count; ++s) {
      const double va = a.at(p, s), vb = b.at(p, s);
      if (std::memcmp(&va, &vb, sizeof(double)) != 0) return false;
    }
  return true;
}

void PointSet::reset_fields(Layout layout) {
  if (fields.size() == n() && fields.layout() == layout) {
    double* d = fields.raw();
    const std::int64_t total = static_cast<std::int64_t>(n()) * slot::count;
    parallel_slices(total, [d](std::int64_t lo, std::int64_t hi) { std::fill(d + lo, d + hi, 0.0); }, 1 << 18);
  } else {
    fields = FieldBlock(layout, n());
  }
}

bool PointSet::has_wall() const {
  return std::find(kind.begin(), kind.end(), Kind::wall) != kind.end();
}

int PointSet::max_degree() const {
  std::int64_t m = 0;
  for (std::int32_t i = 0; i < n(); ++i) m = std::max(m, off[i + 1] - off[i]);
  return static_cast<int>(m);
}

PointSet assemble(std::vector<PointRow> rows, std::vector<std::int64_t> off,
                  std::vector<std::int32_t> nbr) {
  const std::int64_t n64 = static_cast<std::int64_t>(rows.size());
  if (n64 == 0) raise(Status::argument, "point cloud needs at least one point");
  if (n64 > 0x7FFFFFFF) raise(Status::argument, "point cloud exceeds 2^31-1 points");
  const std::int32_t n = static_cast<std::int32_t>(n64);
  if (static_cast<std::int64_t>(off.size()) != n64 + 1 || off[0] != 0 ||
      off.back() != static_cast<std::int64_t>(nbr.size()))
    raise(Status::argument, "malformed stencil offsets");
  for (std::int32_t i = 0; i < n; ++i) {
    const std::int64_t k = off[i + 1] - off[i];
    if (k < 0) raise(Status::argument, "malformed stencil offsets");
    for (std::int64_t e = off[i]; e < off[i + 1]; ++e) {
      const std::int32_t nb = nbr[e];
      if (nb < 0 || nb >= n)
        raise(Status::argument, "neighbour id out of range at point " + std::to_string(i));
      if (nb == i)
        raise(Status::argument, "point " + std::to_string(i) + " lists itself as neighbour");
    }
    if (k > 0 && k < 3)
      raise(Status::argument, "stencil too small (n >= 3 required) at point " + std::to_string(i));
  }
  PointSet ps;
  ps.x.resize(n);
  ps.y.resize(n);
  ps.nx.resize(n);
  ps.ny.resize(n);
  ps.kind.resize(n);
  for (std::int32_t i = 0; i < n; ++i) {
    ps.x[i] = rows[i].x;
    ps.y[i] = rows[i].y;
    ps.nx[i] = rows[i].nx;
    ps.ny[i] = rows[i].ny;
    ps.kind[i] = rows[i].kind;
  }
  ps.off = std::move(off);
  ps.nbr = std::move(nbr);
  ps.fields = FieldBlock(Layout::aos, n);
  return ps;
}

// ---------------------------------------------------------------------------
// Grid text scanner.
namespace {

[[noreturn]] void parse_error(std::int64_t line, const std::string& what) {
  raise(Status::parse, "line " + std::to_string(line) + ": " + what);
}

struct Cursor {
  const char* p;
  const char* end;  // end of the current line (exclusive)

  void skip_ws() {
    while (p < end && (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\v' || *p == '\f')) ++p;
  }
  bool at_end() {
    skip_ws();
    return p >= end;
  }
  template <class T>
  bool integer(T& v) {
    skip_ws();
    const char* s = p;
    if (s < end && *s == '+') ++s;  // istream accepts a leading '+'
    auto r = std::from_chars(s, end, v);
    if (r.ec != std::errc{}) return false;
    p = r.ptr;
    return true;
  }
  bool real(double& v) {
    skip_ws();
    const char* s = p;
    if (s < end && *s == '+') ++s;
    auto r = std::from_chars(s, end, v, std::chars_format::general);
    if (r.ec != std::errc{}) return false;
    p = r.ptr;
    return true;
  }
};

}  // namespace

PointSet parse_grid_text(const char* text, std::size_t len) {
  const char* cur = text;
  const char* stop = text + len;
  auto next_line = [&](Cursor& c) -> bool {
    if (cur >= stop) return false;
    const char* nl = static_cast<const char*>(std::memchr(cur, '\n', static_cast<std::size_t>(stop - cur)));
    c.p = cur;
    c.end = nl ? nl : stop;
    cur = nl ? nl + 1 : stop;
    return true;
  };
  std::int64_t line_no = 0;
  Cursor c{};
  if (!next_line(c)) parse_error(1, "missing header");
  ++line_no;
  std::int64_t n = 0;
  if (!c.integer(n) || n <= 0) parse_error(line_no, "malformed header (expected positive point count)");
  if (!c.at_end()) parse_error(line_no, "malformed header (trailing data)");
  if (n > 0x7FFFFFFF) parse_error(line_no, "malformed header (point count too large)");

  std::vector<PointRow> rows;
  rows.reserve(static_cast<std::size_t>(n));
  std::vector<std::int64_t> off;
  off.reserve(static_cast<std::size_t>(n) + 1);
  off.push_back(0);
  std::vector<std::int32_t> nbr;
  nbr.reserve(static_cast<std::size_t>(n) * 8);
  while (next_line(c)) {
    ++line_no;
    if (c.at_end()) continue;  // blank line
    if (static_cast<std::int64_t>(rows.size()) == n)
      parse_error(line_no, "record count mismatch (more than " + std::to_string(n) + " records)");
    PointRow r;
    std::int32_t id = 0;
    int kind_code = 0;
    std::int64_t k = 0;
    if (!c.integer(id) || !c.real(r.x) || !c.real(r.y) || !c.integer(kind_code) || !c.real(r.nx) ||
        !c.real(r.ny) || !c.integer(k))
      parse_error(line_no, "malformed point record");
    if (id != static_cast<std::int32_t>(rows.size()))
      parse_error(line_no, "point ids must be ascending from 0 (got " + std::to_string(id) + ")");
    if (kind_code < 0 || kind_code > 2) parse_error(line_no, "unknown point kind " + std::to_string(kind_code));
    r.kind = static_cast<Kind>(kind_code);
    if (r.kind != Kind::interior) {
      const double norm2 = r.nx * r.nx + r.ny * r.ny;
      if (std::abs(norm2 - 1.0) > 1e-12) parse_error(line_no, "boundary normal is not unit length");
    }
    if (k < 3) parse_error(line_no, "stencil too small (n >= 3 required)");
    for (std::int64_t j = 0; j < k; ++j) {
      std::int32_t nb = 0;
      if (!c.integer(nb)) parse_error(line_no, "expected " + std::to_string(k) + " neighbour ids");
      if (nb < 0 || nb >= n) parse_error(line_no, "neighbor id out of range (" + std::to_string(nb) + ")");
      if (nb == id) parse_error(line_no, "point lists itself as neighbour");
      nbr.push_back(nb);
    }
    if (!c.at_end()) parse_error(line_no, "trailing data after neighbour list");
    rows.push_back(r);
    off.push_back(static_cast<std::int64_t>(nbr.size()));
  }
  if (static_cast<std::int64_t>(rows.size()) != n)
    parse_error(line_no + 1, "record count mismatch (expected " + std::to_string(n) + ", got " +
                                 std::to_string(rows.size()) + ")");
  return assemble(std::move(rows), std::move(off), std::move(nbr));
}

PointSet read_grid_file(const std::string& path) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) raise(Status::io, "cannot open grid file: " + path);
  std::string buf;
  std::fseek(f, 0, SEEK_END);
  const long sz = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  if (sz > 0) {
    buf.resize(static_cast<std::size_t>(sz));
    const std::size_t got = std::fread(buf.data(), 1, buf.size(), f);
    buf.resize(got);
  }
  std::fclose(f);
  return parse_grid_text(buf.data(), buf.size());
}

void write_grid_file(const PointSet& ps, const std::string& path) {
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) raise(Status::io, "cannot open output file: " + path);
  const std::int32_t n = ps.n();
  // Lines are formatted in parallel slices, then written in order.
  const int slices = std::max(1, std::min<int>(host_threads(), n / 4096));
  std::vector<std::string> parts(static_cast<std::size_t>(slices));
  parallel_slices(
      slices,
      [&](std::int64_t lo, std::int64_t hi) {
        for (std::int64_t s = lo; s < hi; ++s) {
          std::string& out = parts[static_cast<std::size_t>(s)];
          const std::int32_t a = static_cast<std::int32_t>(static_cast<std::int64_t>(n) * s / slices);
          const std::int32_t b = static_cast<std::int32_t>(static_cast<std::int64_t>(n) * (s + 1) / slices);
          char tmp[160];
          for (std::int32_t i = a; i < b; ++i) {
            int w = std::snprintf(tmp, sizeof tmp, "%d %.17g %.17g %d %.17g %.17g %lld", i, ps.x[i], ps.y[i],
                                  static_cast<int>(ps.kind[i]), ps.nx[i], ps.ny[i],
                                  static_cast<long long>(ps.off[i + 1] - ps.off[i]));
            out.append(tmp, static_cast<std::size_t>(w));
            for (std::int64_t e = ps.off[i]; e < ps.off[i + 1]; ++e) {
              w = std::snprintf(tmp, sizeof tmp, " %d", ps.nbr[e]);
              out.append(tmp, static_cast<std::size_t>(w));
            }
            out.push_back('\n');
          }
        }
      },
      1);
  bool ok = std::fprintf(f, "%d\n", n) > 0;
  for (const std::string& s : parts)
    ok = ok && std::fwrite(s.data(), 1, s.size(), f) == s.size();
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) raise(Status::io, "failed writing grid file: " + path);
}

}  // namespace lskb
