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

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include "core.hpp"
#include "par.hpp"

namespace lskb {

bool tracing() {
  static const bool on = std::getenv("LSKUM_TRACE") != nullptr;
  return on;
}

void trace(const char* what) {
  if (!tracing()) return;
  static const auto t0 = std::chrono::steady_clock::now();
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  std::fprintf(stderr, "[lskum %10.3f ms] %s\n", ms, what);
}

std::string fmt_f(double v) {
  char buf[512];
  std::snprintf(buf, sizeof buf, "%f", v);
  return buf;
}

StoreHooks& store_hooks() {
  static StoreHooks h;
  return h;
}

bool pinned_clouds() {
  static const bool on = [] {
    const char* e = std::getenv("LSKUM_PINNED_CLOUD");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

void StoreBuffer::allocate(std::size_t count) {
  n_ = count;
  if (!count) return;
  const std::size_t bytes = count * sizeof(double);
  static const bool allow = [] {
    const char* e = std::getenv("LSKUM_PINNED_STORE");
    return !(e && std::atoi(e) == 0);
  }();
  if (allow && bytes >= (std::size_t{64} << 20) && store_hooks().alloc) {
    p_ = static_cast<double*>(store_hooks().alloc(bytes));
    pinned_ = p_ != nullptr;
  }
  if (!p_) p_ = static_cast<double*>(::operator new(bytes));
}

void StoreBuffer::release() {
  if (!p_) return;
  if (pinned_) store_hooks().release(p_, n_ * sizeof(double));
  else ::operator delete(p_);
  p_ = nullptr;
  n_ = 0;
  pinned_ = false;
}

FieldBlock::FieldBlock(Layout layout, std::int32_t n) : layout_(layout), n_(n) {
  if (n <= 0) raise(Status::argument, "field store needs n_points > 0, got " + std::to_string(n));
  data_ = StoreBuffer(static_cast<std::size_t>(n) * slot::count);
  double* d = data_.data();
  parallel_slices(static_cast<std::int64_t>(data_.size()),
                  [d](std::int64_t lo, std::int64_t hi) { std::fill(d + lo, d + hi, 0.0); }, 1 << 18);
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
  // every offset inside [0, nnz] before any stencil is scanned (a negative
  // count is reported by the per-point checks below, with its point id)
  {
    const std::int64_t nnz = static_cast<std::int64_t>(nbr.size());
    for (std::int64_t i = 1; i < n64; ++i)
      if (off[i] < 0 || off[i] > nnz) raise(Status::argument, "malformed stencil offsets");
  }
  // range checks in parallel; the first offending point (lowest id) is reported
  {
    const int t = std::max(1, std::min<int>(host_threads(), static_cast<int>(n / 65536) + 1));
    std::vector<std::int64_t> first_bad(static_cast<std::size_t>(t), -1);
    std::vector<int> why(static_cast<std::size_t>(t), 0);
    parallel_slices(t, [&](std::int64_t lo, std::int64_t hi) {
      for (std::int64_t s2 = lo; s2 < hi; ++s2) {
        const std::int32_t a = static_cast<std::int32_t>(static_cast<std::int64_t>(n) * s2 / t);
        const std::int32_t b = static_cast<std::int32_t>(static_cast<std::int64_t>(n) * (s2 + 1) / t);
        for (std::int32_t i = a; i < b && first_bad[s2] < 0; ++i) {
          const std::int64_t k = off[i + 1] - off[i];
          int w = 0;
          if (k < 0) w = 1;
          for (std::int64_t e = off[i]; w == 0 && e < off[i + 1]; ++e) {
            const std::int32_t nb = nbr[e];
            if (nb < 0 || nb >= n) w = 2;
            else if (nb == i) w = 3;
          }
          if (w == 0 && k > 0 && k < 3) w = 4;
          if (w) {
            first_bad[s2] = i;
            why[s2] = w;
          }
        }
      }
    }, 1);
    for (int s2 = 0; s2 < t; ++s2) {
      if (first_bad[s2] < 0) continue;
      const std::string id = std::to_string(first_bad[s2]);
      if (why[s2] == 1) raise(Status::argument, "malformed stencil offsets");
      if (why[s2] == 2) raise(Status::argument, "neighbour id out of range at point " + id);
      if (why[s2] == 3) raise(Status::argument, "point " + id + " lists itself as neighbour");
      raise(Status::argument, "stencil too small (n >= 3 required) at point " + id);
    }
  }
  PointSet ps;
  ps.x.resize(n);
  ps.y.resize(n);
  ps.nx.resize(n);
  ps.ny.resize(n);
  ps.kind.resize(n);
  parallel_slices(n, [&](std::int64_t lo, std::int64_t hi) {
    for (std::int64_t i = lo; i < hi; ++i) {
      ps.x[i] = rows[i].x;
      ps.y[i] = rows[i].y;
      ps.nx[i] = rows[i].nx;
      ps.ny[i] = rows[i].ny;
      ps.kind[i] = rows[i].kind;
    }
  }, 1 << 16);
  ps.off.assign(off.begin(), off.end());  // into the cloud's (pinned when large) arrays
  ps.nbr.assign(nbr.begin(), nbr.end());
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

// The grid text is parsed in parallel chunks split at line boundaries (the
// per-chunk record scan is the serial parser's), then merged in file order.
// Checks that need the global record index (ascending ids, record count)
// run in the merge, in the serial parser's order: for every record, count
// overflow, then the id, then the record's own checks — so the first error in
// file order and its message/line are exactly the reference's.
namespace {

struct GridChunk {
  const char* b = nullptr;
  const char* e = nullptr;
  std::int64_t line0 = 0;  // global line number of the chunk's first line
  std::int64_t newlines = 0;
  std::vector<PointRow> rows;
  std::vector<std::int32_t> ids, rec_line;  // per record: id, local line index
  std::vector<std::int64_t> koff{0};
  std::vector<std::int32_t> nbr;
  bool err = false, err_has_id = false;
  std::int32_t err_id = 0;
  std::int64_t err_line = 0;  // local line index of the failing record
  std::string err_msg;
};

void parse_chunk(GridChunk& ch, std::int64_t n) {
  ch.newlines = std::count(ch.b, ch.e, '\n');
  const char* cur = ch.b;
  std::int64_t local = -1;
  Cursor c{};
  auto fail = [&](const std::string& msg, bool has_id, std::int32_t id) {
    ch.err = true;
    ch.err_line = local;
    ch.err_msg = msg;
    ch.err_has_id = has_id;
    ch.err_id = id;
  };
  while (cur < ch.e) {
    const char* nl = static_cast<const char*>(std::memchr(cur, '\n', static_cast<std::size_t>(ch.e - cur)));
    c.p = cur;
    c.end = nl ? nl : ch.e;
    cur = nl ? nl + 1 : ch.e;
    ++local;
    if (c.at_end()) continue;  // blank line
    PointRow r;
    std::int32_t id = 0;
    int kind_code = 0;
    std::int64_t k = 0;
    if (!c.integer(id) || !c.real(r.x) || !c.real(r.y) || !c.integer(kind_code) || !c.real(r.nx) ||
        !c.real(r.ny) || !c.integer(k)) {
      fail("malformed point record", false, 0);
      return;
    }
    if (kind_code < 0 || kind_code > 2) return fail("unknown point kind " + std::to_string(kind_code), true, id);
    r.kind = static_cast<Kind>(kind_code);
    if (r.kind != Kind::interior) {
      const double norm2 = r.nx * r.nx + r.ny * r.ny;
      if (std::abs(norm2 - 1.0) > 1e-12) return fail("boundary normal is not unit length", true, id);
    }
    if (k < 3) return fail("stencil too small (n >= 3 required)", true, id);
    for (std::int64_t j = 0; j < k; ++j) {
      std::int32_t nb = 0;
      if (!c.integer(nb)) return fail("expected " + std::to_string(k) + " neighbour ids", true, id);
      if (nb < 0 || nb >= n) return fail("neighbor id out of range (" + std::to_string(nb) + ")", true, id);
      if (nb == id) return fail("point lists itself as neighbour", true, id);
      ch.nbr.push_back(nb);
    }
    if (!c.at_end()) return fail("trailing data after neighbour list", true, id);
    ch.rows.push_back(r);
    ch.ids.push_back(id);
    ch.rec_line.push_back(static_cast<std::int32_t>(local));
    ch.koff.push_back(static_cast<std::int64_t>(ch.nbr.size()));
  }
}

}  // namespace

PointSet parse_grid_text(const char* text, std::size_t len) {
  const char* stop = text + len;
  const char* first_nl = static_cast<const char*>(std::memchr(text, '\n', len));
  Cursor c{};
  if (len == 0) parse_error(1, "missing header");
  c.p = text;
  c.end = first_nl ? first_nl : stop;
  std::int64_t n = 0;
  if (!c.integer(n) || n <= 0) parse_error(1, "malformed header (expected positive point count)");
  if (!c.at_end()) parse_error(1, "malformed header (trailing data)");
  if (n > 0x7FFFFFFF) parse_error(1, "malformed header (point count too large)");
  const char* body = first_nl ? first_nl + 1 : stop;

  // chunks at line boundaries
  const std::size_t blen = static_cast<std::size_t>(stop - body);
  const int t = static_cast<int>(std::max<std::size_t>(1, std::min<std::size_t>(host_threads() * 4, blen >> 20)));
  std::vector<GridChunk> ch(static_cast<std::size_t>(t));
  const char* at = body;
  for (int i = 0; i < t; ++i) {
    ch[i].b = at;
    const char* want = i == t - 1 ? stop : body + blen * (i + 1) / t;
    if (want < at) want = at;
    const char* nl = want < stop ? static_cast<const char*>(std::memchr(want, '\n', static_cast<std::size_t>(stop - want)))
                                 : nullptr;
    at = (i == t - 1 || !nl) ? stop : nl + 1;
    ch[i].e = at;
  }
  trace("grid: split");
  parallel_slices(t, [&](std::int64_t lo, std::int64_t hi) {
    for (std::int64_t i = lo; i < hi; ++i) parse_chunk(ch[i], n);
  }, 1);
  trace("grid: chunks parsed");
  // line numbers: header is line 1; chunk i starts after the newlines before it
  std::int64_t line = 2;
  for (int i = 0; i < t; ++i) {
    ch[i].line0 = line;
    line += ch[i].newlines;
  }
  // merge in file order with the index-dependent checks
  std::int64_t rec = 0, nnz = 0;
  for (int i = 0; i < t; ++i) {
    const GridChunk& g = ch[i];
    for (std::size_t r = 0; r < g.rows.size(); ++r, ++rec) {
      const std::int64_t ln = g.line0 + g.rec_line[r];
      if (rec == n) parse_error(ln, "record count mismatch (more than " + std::to_string(n) + " records)");
      if (g.ids[r] != rec) parse_error(ln, "point ids must be ascending from 0 (got " + std::to_string(g.ids[r]) + ")");
    }
    nnz += static_cast<std::int64_t>(g.nbr.size());
    if (g.err) {
      const std::int64_t ln = g.line0 + g.err_line;
      if (rec == n) parse_error(ln, "record count mismatch (more than " + std::to_string(n) + " records)");
      if (g.err_has_id && g.err_id != rec)
        parse_error(ln, "point ids must be ascending from 0 (got " + std::to_string(g.err_id) + ")");
      parse_error(ln, g.err_msg);
    }
  }
  if (body < stop && stop[-1] != '\n') ++line;  // an unterminated last line still counts
  if (rec != n)
    parse_error(line, "record count mismatch (expected " + std::to_string(n) + ", got " + std::to_string(rec) + ")");
  // concatenate
  std::vector<PointRow> rows(static_cast<std::size_t>(n));
  std::vector<std::int64_t> off(static_cast<std::size_t>(n) + 1, 0);
  std::vector<std::int32_t> nbr(static_cast<std::size_t>(nnz));
  std::vector<std::int64_t> r0(t + 1, 0), e0(t + 1, 0);
  for (int i = 0; i < t; ++i) {
    r0[i + 1] = r0[i] + static_cast<std::int64_t>(ch[i].rows.size());
    e0[i + 1] = e0[i] + static_cast<std::int64_t>(ch[i].nbr.size());
  }
  parallel_slices(t, [&](std::int64_t lo, std::int64_t hi) {
    for (std::int64_t i = lo; i < hi; ++i) {
      const GridChunk& g = ch[i];
      std::copy(g.rows.begin(), g.rows.end(), rows.begin() + r0[i]);
      std::copy(g.nbr.begin(), g.nbr.end(), nbr.begin() + e0[i]);
      for (std::size_t r = 0; r < g.rows.size(); ++r) off[r0[i] + r + 1] = e0[i] + g.koff[r + 1];
    }
  }, 1);
  trace("grid: merged");
  return assemble(std::move(rows), std::move(off), std::move(nbr));
}

PointSet read_grid_file(const std::string& path) {
  // mapped read-only: the parser works on the page cache directly
  const int fd = ::open(path.c_str(), O_RDONLY);
  if (fd < 0) raise(Status::io, "cannot open grid file: " + path);
  struct stat st{};
  if (::fstat(fd, &st) != 0) {
    ::close(fd);
    raise(Status::io, "cannot open grid file: " + path);
  }
  const std::size_t sz = static_cast<std::size_t>(st.st_size);
  if (sz == 0) {
    ::close(fd);
    return parse_grid_text("", 0);
  }
  void* m = ::mmap(nullptr, sz, PROT_READ, MAP_PRIVATE, fd, 0);
  ::close(fd);
  if (m == MAP_FAILED) raise(Status::io, "cannot open grid file: " + path);
  struct Unmap {
    void* p;
    std::size_t n;
    ~Unmap() { ::munmap(p, n); }
  } guard{m, sz};
  trace("grid: file mapped");
  return parse_grid_text(static_cast<const char*>(m), sz);
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
          char tmp[64];
          auto put_int = [&](long long v) {
            const auto r = std::to_chars(tmp, tmp + sizeof tmp, v);
            out.append(tmp, static_cast<std::size_t>(r.ptr - tmp));
          };
          auto put_real = [&](double v) {  // identical to printf("%.17g") (C++17 to_chars spec)
            const auto r = std::to_chars(tmp, tmp + sizeof tmp, v, std::chars_format::general, 17);
            out.append(tmp, static_cast<std::size_t>(r.ptr - tmp));
          };
          out.reserve(static_cast<std::size_t>(b - a) * 140);
          for (std::int32_t i = a; i < b; ++i) {
            put_int(i);
            out.push_back(' ');
            put_real(ps.x[i]);
            out.push_back(' ');
            put_real(ps.y[i]);
            out.push_back(' ');
            put_int(static_cast<int>(ps.kind[i]));
            out.push_back(' ');
            put_real(ps.nx[i]);
            out.push_back(' ');
            put_real(ps.ny[i]);
            out.push_back(' ');
            put_int(ps.off[i + 1] - ps.off[i]);
            for (std::int64_t e = ps.off[i]; e < ps.off[i + 1]; ++e) {
              out.push_back(' ');
              put_int(ps.nbr[e]);
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
