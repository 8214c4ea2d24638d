// screen.cpp — stencil screening (rank-deficiency gate before a run).
//
// Same report as the reference validate_cloud (cloud.cpp:252-321): h_ref =
// median nearest-neighbour distance, det_tol = 1e-12 h_ref^4, a point is
// defective if its full-stencil determinant (or, for non-outer points, any of
// the four half-stencil determinants) is below det_tol or a required half
// stencil is empty.  Per-point sums are accumulated in ascending stencil order
// exactly as LsSums::add does, so determinants are bitwise those of the
// reference; points are screened in parallel.
#include <algorithm>
#include <cmath>
#include <limits>

#include "core.hpp"
#include "par.hpp"

namespace lskb {

namespace {

struct Gram {
  double sxx = 0.0, sxy = 0.0, syy = 0.0;
  int count = 0;
  void add(double dx, double dy) {
    sxx += dx * dx;
    sxy += dx * dy;
    syy += dy * dy;
    ++count;
  }
  double det() const { return sxx * syy - sxy * sxy; }
};

}  // namespace

Screening screen_stencils(const PointSet& ps) {
  const std::int32_t n = ps.n();
  Screening out;
  std::vector<double> nearest(static_cast<std::size_t>(n));
  parallel_slices(n, [&](std::int64_t lo, std::int64_t hi) {
    for (std::int64_t p = lo; p < hi; ++p) {
      double best = std::numeric_limits<double>::infinity();
      for (std::int64_t e = ps.off[p]; e < ps.off[p + 1]; ++e) {
        const std::int32_t nb = ps.nbr[e];
        const double dx = ps.x[nb] - ps.x[p], dy = ps.y[nb] - ps.y[p];
        best = std::min(best, std::sqrt(dx * dx + dy * dy));
      }
      nearest[p] = best;
    }
  });
  std::vector<double> finite;
  finite.reserve(nearest.size());
  for (double d : nearest)
    if (std::isfinite(d)) finite.push_back(d);
  if (!finite.empty()) {
    const std::size_t mid = (finite.size() - 1) / 2;
    std::nth_element(finite.begin(), finite.begin() + static_cast<std::ptrdiff_t>(mid), finite.end());
    out.h_ref = finite[mid];
  }
  out.det_tol = 1e-12 * out.h_ref * out.h_ref * out.h_ref * out.h_ref;

  std::vector<std::uint8_t> bad(static_cast<std::size_t>(n), 0), isolated(static_cast<std::size_t>(n), 0);
  std::vector<int> size(static_cast<std::size_t>(n), 0);
  const double tol = out.det_tol;
  parallel_slices(n, [&](std::int64_t lo, std::int64_t hi) {
    for (std::int64_t p = lo; p < hi; ++p) {
      Gram full, half[4];  // x>=0, x<=0, y>=0, y<=0
      int wall_nbrs = 0;
      for (std::int64_t e = ps.off[p]; e < ps.off[p + 1]; ++e) {
        const std::int32_t nb = ps.nbr[e];
        const double dx = ps.x[nb] - ps.x[p], dy = ps.y[nb] - ps.y[p];
        full.add(dx, dy);
        if (dx >= 0.0) half[0].add(dx, dy);
        if (dx <= 0.0) half[1].add(dx, dy);
        if (dy >= 0.0) half[2].add(dx, dy);
        if (dy <= 0.0) half[3].add(dx, dy);
        if (ps.kind[nb] == Kind::wall) ++wall_nbrs;
      }
      bool defective = full.det() < tol || full.count < 3;
      if (ps.kind[p] != Kind::outer)
        for (const Gram& h : half) defective = defective || h.count == 0 || h.det() < tol;
      bad[p] = defective;
      isolated[p] = ps.kind[p] == Kind::wall && wall_nbrs < 2;
      size[p] = full.count;
    }
  });
  out.min_stencil = n > 0 ? std::numeric_limits<int>::max() : 0;
  for (std::int32_t p = 0; p < n; ++p) {
    if (bad[p]) {
      ++out.n_defective;
      out.defective.push_back(p);
    }
    out.n_wall_isolated += isolated[p];
    out.min_stencil = std::min(out.min_stencil, size[p]);
  }
  return out;
}

}  // namespace lskb
