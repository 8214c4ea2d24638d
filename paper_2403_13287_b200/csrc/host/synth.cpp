// synth.cpp — synthetic point clouds and k-nearest-neighbour stencils.
//
// Same point sets and stencils as the reference generators
// (cloud.cpp:323-425: jittered rectangle, annulus; mt19937_64 top-53-bit
// doubles, cloud.cpp:26-30) and kNN (cloud.cpp:137-237: nearest by
// (d^2, id), neighbour ids sorted ascending).  The kNN search visits the same
// bucket-grid rings with the same stopping guard, so every point gets the
// identical candidate set and therefore the identical stencil; points are
// processed in parallel (the result is independent of the thread count).
#include <algorithm>
#include <cmath>
#include <random>

#include "core.hpp"
#include "par.hpp"

namespace lskb {

namespace {

double unit_draw(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
double signed_draw(std::mt19937_64& g) { return 2.0 * unit_draw(g) - 1.0; }

struct Cand {
  double d2;
  std::int32_t id;
};
inline bool cand_before(const Cand& a, const Cand& b) {
  return a.d2 < b.d2 || (a.d2 == b.d2 && a.id < b.id);
}

void pick_k(std::vector<Cand>& cand, int k, std::int32_t* out) {
  std::partial_sort(cand.begin(), cand.begin() + k, cand.end(), cand_before);
  for (int j = 0; j < k; ++j) out[j] = cand[j].id;
  std::sort(out, out + k);
}

}  // namespace

void attach_knn(PointSet& ps, int k) {
  const std::int32_t n = ps.n();
  if (k < 3) raise(Status::argument, "stencil size k must be >= 3, got " + std::to_string(k));
  if (k >= n)
    raise(Status::argument, "stencil size k=" + std::to_string(k) + " needs more than k points (have " +
                                std::to_string(n) + ")");
  double xmin = ps.x[0], xmax = ps.x[0], ymin = ps.y[0], ymax = ps.y[0];
  for (std::int32_t i = 1; i < n; ++i) {
    xmin = std::min(xmin, ps.x[i]);
    xmax = std::max(xmax, ps.x[i]);
    ymin = std::min(ymin, ps.y[i]);
    ymax = std::max(ymax, ps.y[i]);
  }
  ps.off.assign(static_cast<std::size_t>(n) + 1, 0);
  for (std::int32_t i = 0; i <= n; ++i) ps.off[i] = static_cast<std::int64_t>(i) * k;
  ps.nbr.assign(static_cast<std::size_t>(n) * k, 0);
  const double width = xmax - xmin, height = ymax - ymin;
  const double extent = std::max(width, height);

  if (n <= 2048 || extent <= 0.0) {
    parallel_slices(n, [&](std::int64_t lo, std::int64_t hi) {
      std::vector<Cand> cand;
      for (std::int64_t p = lo; p < hi; ++p) {
        cand.clear();
        for (std::int32_t q = 0; q < n; ++q) {
          if (q == p) continue;
          const double dx = ps.x[q] - ps.x[p], dy = ps.y[q] - ps.y[p];
          cand.push_back({dx * dx + dy * dy, q});
        }
        pick_k(cand, k, ps.nbr.data() + p * k);
      }
    }, 64);
    return;
  }

  const int grid_dim = std::max(1, static_cast<int>(std::sqrt(static_cast<double>(n) / 2.0)));
  const double cell = extent / grid_dim;
  const int ncx = std::max(1, static_cast<int>(std::floor(width / cell)) + 1);
  const int ncy = std::max(1, static_cast<int>(std::floor(height / cell)) + 1);
  auto cell_x = [&](double px) { return std::min(ncx - 1, static_cast<int>(std::floor((px - xmin) / cell))); };
  auto cell_y = [&](double py) { return std::min(ncy - 1, static_cast<int>(std::floor((py - ymin) / cell))); };
  // bucket grid as CSR, ids ascending within each cell (insertion order)
  const std::size_t ncell = static_cast<std::size_t>(ncx) * ncy;
  std::vector<std::int64_t> cstart(ncell + 1, 0);
  std::vector<std::int32_t> home(n);
  for (std::int32_t i = 0; i < n; ++i) {
    home[i] = cell_y(ps.y[i]) * ncx + cell_x(ps.x[i]);
    ++cstart[static_cast<std::size_t>(home[i]) + 1];
  }
  for (std::size_t c = 0; c < ncell; ++c) cstart[c + 1] += cstart[c];
  std::vector<std::int32_t> members(n);
  {
    std::vector<std::int64_t> fill(cstart.begin(), cstart.end() - 1);
    for (std::int32_t i = 0; i < n; ++i) members[fill[home[i]]++] = i;
  }
  const int max_ring = std::max(ncx, ncy);
  parallel_slices(n, [&](std::int64_t lo, std::int64_t hi) {
    std::vector<Cand> cand, probe;
    for (std::int64_t p = lo; p < hi; ++p) {
      cand.clear();
      const int pcx = home[p] % ncx, pcy = home[p] / ncx;
      const double px = ps.x[p], py = ps.y[p];
      for (int ring = 0; ring <= max_ring; ++ring) {
        for (int cy = pcy - ring; cy <= pcy + ring; ++cy) {
          if (cy < 0 || cy >= ncy) continue;
          const bool edge_row = cy == pcy - ring || cy == pcy + ring;
          for (int cx = pcx - ring; cx <= pcx + ring; cx += (edge_row || ring == 0) ? 1 : 2 * ring) {
            if (cx < 0 || cx >= ncx) continue;
            const std::size_t cid = static_cast<std::size_t>(cy) * ncx + cx;
            for (std::int64_t e = cstart[cid]; e < cstart[cid + 1]; ++e) {
              const std::int32_t q = members[e];
              if (q == p) continue;
              const double dx = ps.x[q] - px, dy = ps.y[q] - py;
              cand.push_back({dx * dx + dy * dy, q});
            }
          }
        }
        if (static_cast<int>(cand.size()) >= k) {
          // k-th best by (d2, id) against the ring guard (reference cloud.cpp:219-228)
          probe.assign(cand.begin(), cand.end());
          std::nth_element(probe.begin(), probe.begin() + (k - 1), probe.end(), cand_before);
          const double guard = static_cast<double>(ring) * cell;
          if (probe[k - 1].d2 < guard * guard || ring == max_ring) break;
        }
      }
      pick_k(cand, k, ps.nbr.data() + p * k);
    }
  }, 1024);
}

PointSet make_rect(int nx, int ny, const Box& box, double jitter, std::uint64_t seed, int k) {
  if (nx < 4 || ny < 4) raise(Status::argument, "rect cloud needs nx, ny >= 4");
  if (!(jitter >= 0.0 && jitter <= 0.3)) raise(Status::argument, "jitter must lie in [0, 0.3]");
  if (!(box.xmax > box.xmin) || !(box.ymax > box.ymin)) raise(Status::argument, "degenerate bounds");
  if (static_cast<long long>(nx) * ny > 0x7FFFFFFFll) raise(Status::argument, "rect cloud too large");
  const double hx = (box.xmax - box.xmin) / (nx - 1);
  const double hy = (box.ymax - box.ymin) / (ny - 1);
  const double inv_sqrt2 = 1.0 / std::sqrt(2.0);
  std::mt19937_64 rng(seed);
  std::vector<PointRow> rows(static_cast<std::size_t>(nx) * ny);
  for (int j = 0; j < ny; ++j) {
    for (int i = 0; i < nx; ++i) {
      PointRow& r = rows[static_cast<std::size_t>(j) * nx + i];
      r.x = box.xmin + i * hx;
      r.y = box.ymin + j * hy;
      const bool left = i == 0, right = i == nx - 1, bottom = j == 0, top = j == ny - 1;
      if (left || right || bottom || top) {
        r.kind = Kind::outer;
        double a = left ? -1.0 : (right ? 1.0 : 0.0);
        double b = bottom ? -1.0 : (top ? 1.0 : 0.0);
        if (a != 0.0 && b != 0.0) {
          a *= inv_sqrt2;
          b *= inv_sqrt2;
        }
        r.nx = a;
        r.ny = b;
      } else if (jitter > 0.0) {
        r.x += jitter * hx * signed_draw(rng);
        r.y += jitter * hy * signed_draw(rng);
      }
    }
  }
  const std::size_t n = rows.size();
  PointSet ps = assemble(std::move(rows), std::vector<std::int64_t>(n + 1, 0), {});
  attach_knn(ps, k);
  return ps;
}

PointSet make_annulus(int n_theta, int n_rings, double r_outer, double jitter, std::uint64_t seed,
                      int k) {
  if (n_theta < 8 || n_rings < 3) raise(Status::argument, "annulus cloud needs n_theta >= 8 and n_rings >= 3");
  if (!(r_outer > 1.0)) raise(Status::argument, "annulus outer radius must exceed the unit circle");
  if (!(jitter >= 0.0 && jitter <= 0.3)) raise(Status::argument, "jitter must lie in [0, 0.3]");
  std::vector<double> radii(n_rings);
  for (int j = 0; j < n_rings; ++j) radii[j] = std::pow(r_outer, static_cast<double>(j) / (n_rings - 1));
  const double dtheta = 2.0 * M_PI / n_theta;
  std::mt19937_64 rng(seed);
  std::vector<PointRow> rows(static_cast<std::size_t>(n_theta) * n_rings);
  for (int j = 0; j < n_rings; ++j) {
    for (int i = 0; i < n_theta; ++i) {
      PointRow& r = rows[static_cast<std::size_t>(j) * n_theta + i];
      double radius = radii[j];
      double theta = i * dtheta;
      const bool wall = j == 0, outer = j == n_rings - 1;
      if (!wall && !outer && jitter > 0.0) {
        const double gap = std::min(radii[j + 1] - radii[j], radii[j] - radii[j - 1]);
        radius += jitter * gap * signed_draw(rng);
        theta += jitter * dtheta * signed_draw(rng);
      }
      r.x = radius * std::cos(theta);
      r.y = radius * std::sin(theta);
      if (wall) {
        r.kind = Kind::wall;
        r.nx = -std::cos(theta);
        r.ny = -std::sin(theta);
      } else if (outer) {
        r.kind = Kind::outer;
        r.nx = std::cos(theta);
        r.ny = std::sin(theta);
      }
    }
  }
  const std::size_t n = rows.size();
  PointSet ps = assemble(std::move(rows), std::vector<std::int64_t>(n + 1, 0), {});
  attach_knn(ps, k);
  return ps;
}

}  // namespace lskb
