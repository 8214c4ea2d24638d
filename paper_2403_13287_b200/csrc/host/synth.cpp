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
#include <cstdlib>
#include <random>

#include "../engine.hpp"
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
  trace("knn: start");

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

  // Exact k nearest by (d^2, id) — the same set the reference's bucket-ring
  // search returns (its guard makes it exact, cloud.cpp:219-228) — from a 2-d
  // tree, whose cost does not degrade on strongly graded clouds (airfoil
  // O-grids span four decades of spacing).  A subtree is skipped only when
  // its box's lower distance bound exceeds the current k-th distance strictly
  // (an equal bound may still hold a tie with a smaller id); the bound is
  // computed with the same rounded operations as the point distances, which
  // are monotone, so it never exceeds the distance of a point inside.
  using Node = KdNode;
  using Pt = KdPt;
  std::vector<Pt> pts(n);
  for (std::int32_t i = 0; i < n; ++i) pts[i] = Pt{ps.x[i], ps.y[i], i, 0};
  constexpr std::int32_t kLeaf = 16;
  // Median split along the box's longer side; returns the split index or -1
  // for a leaf.  Writes the box of [lo, hi) into `nd`.
  auto split = [&](std::int32_t lo, std::int32_t hi, Node& nd) -> std::int32_t {
    double x0 = pts[lo].x, x1 = x0, y0 = pts[lo].y, y1 = y0;
    for (std::int32_t e = lo + 1; e < hi; ++e) {
      x0 = std::min(x0, pts[e].x);
      x1 = std::max(x1, pts[e].x);
      y0 = std::min(y0, pts[e].y);
      y1 = std::max(y1, pts[e].y);
    }
    nd.x0 = x0;
    nd.x1 = x1;
    nd.y0 = y0;
    nd.y1 = y1;
    nd.lo = lo;
    nd.hi = hi;
    nd.left = nd.right = -1;
    if (hi - lo <= kLeaf) return -1;
    const std::int32_t mid = lo + (hi - lo) / 2;
    if ((x1 - x0) >= (y1 - y0))
      std::nth_element(pts.begin() + lo, pts.begin() + mid, pts.begin() + hi,
                       [](const Pt& a, const Pt& b) { return a.x < b.x || (a.x == b.x && a.id < b.id); });
    else
      std::nth_element(pts.begin() + lo, pts.begin() + mid, pts.begin() + hi,
                       [](const Pt& a, const Pt& b) { return a.y < b.y || (a.y == b.y && a.id < b.id); });
    return mid;
  };
  // Builds the subtree of [lo, hi) into `out` (node indices local to `out`).
  auto build = [&](std::int32_t lo, std::int32_t hi, std::vector<Node>& out) {
    struct Job {
      std::int32_t lo, hi, node;
    };
    std::vector<Job> todo{{lo, hi, static_cast<std::int32_t>(out.size())}};
    out.emplace_back();
    while (!todo.empty()) {
      const Job jb = todo.back();
      todo.pop_back();
      Node nd;
      const std::int32_t mid = split(jb.lo, jb.hi, nd);
      if (mid >= 0) {
        nd.left = static_cast<std::int32_t>(out.size());
        nd.right = nd.left + 1;
        out.emplace_back();
        out.emplace_back();
        todo.push_back({jb.lo, mid, nd.left});
        todo.push_back({mid, jb.hi, nd.right});
      }
      out[jb.node] = nd;
    }
  };
  // top levels serially, then the subtrees in parallel, then stitched together
  std::vector<Node> nodes;
  std::vector<std::pair<std::int32_t, std::int32_t>> tops;  // (node, pending subtree) leaves of the top
  {
    const int depth = 6;
    struct Job {
      std::int32_t lo, hi, node, d;
    };
    std::vector<Job> todo{{0, n, 0, 0}};
    nodes.emplace_back();
    while (!todo.empty()) {
      const Job jb = todo.back();
      todo.pop_back();
      if (jb.d == depth && jb.hi - jb.lo > kLeaf) {
        tops.push_back({jb.node, -1});
        nodes[jb.node].lo = jb.lo;
        nodes[jb.node].hi = jb.hi;
        continue;
      }
      Node nd;
      const std::int32_t mid = split(jb.lo, jb.hi, nd);
      if (mid >= 0) {
        nd.left = static_cast<std::int32_t>(nodes.size());
        nd.right = nd.left + 1;
        nodes.emplace_back();
        nodes.emplace_back();
        todo.push_back({jb.lo, mid, nd.left, jb.d + 1});
        todo.push_back({mid, jb.hi, nd.right, jb.d + 1});
      }
      nodes[jb.node] = nd;
    }
  }
  std::vector<std::vector<Node>> sub(tops.size());
  parallel_slices(static_cast<std::int64_t>(tops.size()), [&](std::int64_t a, std::int64_t b) {
    for (std::int64_t t = a; t < b; ++t) build(nodes[tops[t].first].lo, nodes[tops[t].first].hi, sub[t]);
  }, 1);
  for (std::size_t t = 0; t < tops.size(); ++t) {
    const std::int32_t base = static_cast<std::int32_t>(nodes.size()) - 1;  // sub[t][0] replaces the top leaf
    Node root = sub[t][0];
    auto fix = [&](Node& nd) {
      if (nd.left >= 0) {
        nd.left += base;
        nd.right += base;
      }
    };
    fix(root);
    nodes[tops[t].first] = root;
    for (std::size_t m = 1; m < sub[t].size(); ++m) {
      Node nd = sub[t][m];
      fix(nd);
      nodes.push_back(nd);
    }
  }
  trace("knn: tree built");
  // the queries on the GPU when there is one (LSKUM_GPU_KNN=0: host)
  static const bool gpu_knn = [] {
    const char* e = std::getenv("LSKUM_GPU_KNN");
    return !(e && std::atoi(e) == 0);
  }();
  if (gpu_knn && n >= (1 << 16) && k <= 16 && engine_knn(nodes, pts, k, ps.nbr.data())) {
    trace("knn: queried (GPU)");
    return;
  }
  std::vector<std::int32_t> idx(n);
  for (std::int32_t i = 0; i < n; ++i) idx[i] = pts[i].id;
  parallel_slices(n, [&](std::int64_t lo, std::int64_t hi) {
    std::vector<Cand> heap;
    std::vector<std::int32_t> stack;
    heap.reserve(static_cast<std::size_t>(k) + 1);
    for (std::int64_t pos = lo; pos < hi; ++pos) {  // queries in tree (leaf) order, for locality
      const std::int32_t p = idx[pos];
      heap.clear();
      const double px = ps.x[p], py = ps.y[p];
      auto bound = [&](const Node& b) {
        const double ex = px < b.x0 ? b.x0 - px : (px > b.x1 ? px - b.x1 : 0.0);
        const double ey = py < b.y0 ? b.y0 - py : (py > b.y1 ? py - b.y1 : 0.0);
        return ex * ex + ey * ey;
      };
      stack.clear();
      stack.push_back(0);
      while (!stack.empty()) {
        const Node& b = nodes[stack.back()];
        stack.pop_back();
        if (static_cast<int>(heap.size()) == k && bound(b) > heap.front().d2) continue;
        if (b.left < 0) {
          for (std::int32_t e = b.lo; e < b.hi; ++e) {
            const std::int32_t q = pts[e].id;
            if (q == p) continue;
            const double dx = pts[e].x - px, dy = pts[e].y - py;
            const Cand cd{dx * dx + dy * dy, q};
            if (static_cast<int>(heap.size()) < k) {
              heap.push_back(cd);
              std::push_heap(heap.begin(), heap.end(), cand_before);
            } else if (cand_before(cd, heap.front())) {
              std::pop_heap(heap.begin(), heap.end(), cand_before);
              heap.back() = cd;
              std::push_heap(heap.begin(), heap.end(), cand_before);
            }
          }
          continue;
        }
        // nearer child last, so it is visited first
        const double bl = bound(nodes[b.left]), br = bound(nodes[b.right]);
        if (bl <= br) {
          stack.push_back(b.right);
          stack.push_back(b.left);
        } else {
          stack.push_back(b.left);
          stack.push_back(b.right);
        }
      }
      pick_k(heap, k, ps.nbr.data() + static_cast<std::int64_t>(p) * k);
    }
  }, 1024);
  trace("knn: queried");
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

// ---------------------------------------------------------------------------
// Synthetic NACA 0012 O-cloud (new: the reference has no airfoil generator,
// SPEC.md:12).  Ring 0 is the airfoil surface, ring J-1 a
// far-field circle of radius r_outer about the mid-chord (0.5, 0).
//   surface:  the closed-trailing-edge NACA 00xx section, t = 0.12:
//             y_t = 5 t (0.2969 sqrt x - 0.1260 x - 0.3516 x^2 + 0.2843 x^3
//             - 0.1036 x^4), parameterised by phi in [0, 2 pi) (trailing edge
//             -> upper surface -> leading edge -> lower surface) with
//             x = (1 + cos phi)/2; the n_wall points sit at equal arc length
//             (phi found on a fine arc-length table, then the point evaluated
//             on the exact section), so the surface spacing is uniform.
//   rings:    p_ij = S_i + f_j (F_i - S_i), F_i = far-field point at polar
//             angle 2 pi i / n_wall; f_j = (q^j - 1)/(q^(J-1) - 1) with q
//             chosen so the first layer is as thick as the surface spacing
//             (square cells at the wall; kNN stencils then reach into both
//             half planes of every axis).
//   jitter:   interior points move by jitter x (smallest adjacent spacing) x
//             a symmetric draw per axis (mt19937_64, as the reference's rect
//             generator, cloud.cpp:26-30), ring-major order.
//   kinds:    ring 0 = wall (normal into the body, the annulus convention,
//             cloud.cpp:405-409) or, with frozen_wall, outer — the surface state
//             is then held like far-field points, because the reference has no
//             wall flux and its split stencils on a curved wall are singular or
//             unstable (SURVEY 0 gap 5); ring J-1 = outer, radial normal.
//             In frozen mode the few interior points behind the sharp
//             trailing edge whose split stencils fail validate_cloud are held
//             too (kind outer), so the cloud validates and runs.
// Stencils: attach_knn (bit-exact with the reference's build_stencils), so the
// same cloud written to a grid file runs unchanged in the reference.
namespace {
constexpr double kNacaT = 0.12;
double naca_x(double phi) { return 0.5 * (1.0 + std::cos(phi)); }
double naca_y(double phi) {
  const double x = naca_x(phi), s = std::sqrt(x);
  const double yt = 5.0 * kNacaT * (0.2969 * s + x * (-0.1260 + x * (-0.3516 + x * (0.2843 + x * -0.1036))));
  return std::sin(phi) >= 0.0 ? yt : -yt;
}
}  // namespace

PointSet make_naca0012(int n_wall, int n_rings, double r_outer, double jitter, std::uint64_t seed, int k,
                       bool frozen_wall) {
  if (n_wall < 16 || (n_wall & 1)) raise(Status::argument, "naca0012 cloud needs an even n_wall >= 16");
  if (n_rings < 3) raise(Status::argument, "naca0012 cloud needs n_rings >= 3");
  if (!(r_outer >= 2.0)) raise(Status::argument, "naca0012 far field radius must be >= 2 chords");
  if (!(jitter >= 0.0 && jitter <= 0.3)) raise(Status::argument, "jitter must lie in [0, 0.3]");
  if (static_cast<long long>(n_wall) * n_rings > 0x7FFFFFFFll) raise(Status::argument, "naca0012 cloud too large");
  const double kTwoPi = 2.0 * M_PI, cx = 0.5;
  const std::size_t nw = static_cast<std::size_t>(n_wall), nr = static_cast<std::size_t>(n_rings);
  // arc-length table of the section (the upper half; the lower mirrors it)
  const std::size_t fine = 64 * nw;
  std::vector<double> arc(fine + 1, 0.0);
  for (std::size_t m = 1; m <= fine; ++m) {
    const double a = M_PI * (m - 1) / fine, b = M_PI * m / fine;
    arc[m] = arc[m - 1] + std::hypot(naca_x(b) - naca_x(a), naca_y(b) - naca_y(a));
  }
  const double half = arc[fine];
  std::vector<double> sx(nw), sy(nw), fx(nw), fy(nw);
  for (std::size_t i = 0; i <= nw / 2; ++i) {
    const double target = half * static_cast<double>(i) / (nw / 2);
    std::size_t m = static_cast<std::size_t>(std::lower_bound(arc.begin(), arc.end(), target) - arc.begin());
    m = std::min(std::max<std::size_t>(m, 1), fine);
    const double t = (target - arc[m - 1]) / (arc[m] - arc[m - 1]);
    const double phi = (i == 0) ? 0.0 : (i == nw / 2 ? M_PI : M_PI * ((m - 1) + t) / fine);
    sx[i] = naca_x(phi);
    sy[i] = (i == 0 || i == nw / 2) ? 0.0 : naca_y(phi);
    if (i > 0 && i < nw / 2) {  // mirror onto the lower surface
      sx[nw - i] = sx[i];
      sy[nw - i] = -sy[i];
    }
  }
  for (std::size_t i = 0; i < nw; ++i) {
    const double th = kTwoPi * static_cast<double>(i) / n_wall;
    fx[i] = cx + r_outer * std::cos(th);
    fy[i] = r_outer * std::sin(th);
  }
  // stretching: first layer ~ surface spacing over the mean wall-to-far-field distance
  const double ds = 2.0 * half / n_wall;
  double lmean = 0.0;
  for (std::size_t i = 0; i < nw; ++i) lmean += std::hypot(fx[i] - sx[i], fy[i] - sy[i]);
  lmean /= n_wall;
  const double f1 = ds / lmean;
  const double jm1 = static_cast<double>(n_rings - 1);
  auto first = [&](double qq) { return (qq - 1.0) / (std::pow(qq, jm1) - 1.0); };
  double q = 1.0;
  if (f1 < 1.0 / jm1) {
    double lo = 1.0 + 1e-12, hi = 2.0;
    for (int it = 0; it < 200; ++it) {
      const double mid = 0.5 * (lo + hi);
      if (first(mid) > f1) lo = mid;
      else hi = mid;
    }
    q = 0.5 * (lo + hi);
  }
  std::vector<double> f(nr);
  for (std::size_t j = 0; j < nr; ++j)
    f[j] = q == 1.0 ? static_cast<double>(j) / jm1 : (std::pow(q, static_cast<double>(j)) - 1.0) / (std::pow(q, jm1) - 1.0);
  f[0] = 0.0;
  f[nr - 1] = 1.0;
  auto px = [&](std::size_t i, std::size_t j) { return sx[i] + f[j] * (fx[i] - sx[i]); };
  auto py = [&](std::size_t i, std::size_t j) { return sy[i] + f[j] * (fy[i] - sy[i]); };
  std::mt19937_64 rng(seed);
  std::vector<PointRow> rows(nw * nr);
  for (std::size_t j = 0; j < nr; ++j) {
    for (std::size_t i = 0; i < nw; ++i) {
      PointRow& r = rows[j * nw + i];
      r.x = px(i, j);
      r.y = py(i, j);
      const std::size_t ip = (i + 1) % nw, im = (i + nw - 1) % nw;
      if (j == 0) {
        // surface tangent by central differences (counter-clockwise), normal into the body
        const double tx = sx[ip] - sx[im], ty = sy[ip] - sy[im];
        const double h = std::hypot(tx, ty);
        r.kind = frozen_wall ? Kind::outer : Kind::wall;
        r.nx = -ty / h;
        r.ny = tx / h;
      } else if (j == nr - 1) {
        const double h = std::hypot(r.x - cx, r.y);
        r.kind = Kind::outer;
        r.nx = (r.x - cx) / h;
        r.ny = r.y / h;
      } else if (jitter > 0.0) {
        auto dist = [&](std::size_t a, std::size_t b, std::size_t c, std::size_t d) {
          return std::hypot(px(a, b) - px(c, d), py(a, b) - py(c, d));
        };
        const double h = std::min(std::min(dist(i, j, i, j + 1), dist(i, j, i, j - 1)),
                                  std::min(dist(i, j, ip, j), dist(i, j, im, j)));
        r.x += jitter * h * signed_draw(rng);
        r.y += jitter * h * signed_draw(rng);
      }
    }
  }
  const std::size_t n = rows.size();
  PointSet ps = assemble(std::move(rows), std::vector<std::int64_t>(n + 1, 0), {});
  attach_knn(ps, k);
  if (frozen_wall) {
    // The sharp trailing edge leaves a handful of points just behind it whose
    // half stencils are empty or collinear; they are held like the surface.
    // Kinds do not enter h_ref or the determinants, so one pass suffices.
    const Screening scr = screen_stencils(ps);
    for (std::int32_t p : scr.defective) {
      if (ps.kind[p] == Kind::outer) continue;
      ps.kind[p] = Kind::outer;
      const double h = std::hypot(ps.x[p] - cx, ps.y[p]);  // boundary points carry a unit normal
      ps.nx[p] = h > 0.0 ? (ps.x[p] - cx) / h : 1.0;
      ps.ny[p] = h > 0.0 ? ps.y[p] / h : 0.0;
    }
  }
  return ps;
}

}  // namespace lskb
