// reorder.cpp — locality permutation of a cloud's device numbering.
//
// SURVEY section 7 step 6 / north_star: the device domain may hold the points
// in Hilbert-curve order so that the derivative sweep's and the flux's
// neighbour gathers touch fewer cache lines.  Ids only: every point keeps its
// stencil in the original order, residue summands are indexed by original
// id, failures carry original ids and the store is written back in original
// order, so results are bitwise those of the unpermuted run (the same
// machinery as a multi-domain run's local numbering).
//
// reorder=auto (default) keeps the cloud's own order unless it gathers
// poorly, and then uses reverse Cuthill-McKee.  Measured on B200 with the 10M
// NACA O-cloud: generator's ring order 4.60 ms per iteration, randomly
// shuffled ids 24.1 ms, RCM of the shuffled cloud 4.60 ms, Hilbert order
// 4.90 ms (scripts/order_probe.py).  The decision uses the mean number of
// 128-byte derivative-record lines the neighbours of 16 consecutive points
// touch (ring order 1.9, RCM 2.1, Hilbert 1.6, shuffled 8.0 per point).
#include <algorithm>
#include <cmath>

#include "../engine.hpp"
#include "core.hpp"
#include "par.hpp"

namespace lskb {

namespace {

constexpr int kGroup = 16;          // points per sampled group (one warp of the sweep)
constexpr double kPoorLines = 3.0;  // lines per point above which auto reorders

// Hilbert index of (x, y) on a 2^16 x 2^16 grid.
std::uint32_t hilbert_index(std::uint32_t x, std::uint32_t y) {
  constexpr std::uint32_t n = 1u << 16;
  std::uint32_t d = 0;
  for (std::uint32_t s = n >> 1; s > 0; s >>= 1) {
    const std::uint32_t rx = (x & s) ? 1u : 0u, ry = (y & s) ? 1u : 0u;
    d += s * s * ((3u * rx) ^ ry);
    if (ry == 0) {
      if (rx == 1) {
        x = n - 1 - x;
        y = n - 1 - y;
      }
      std::swap(x, y);
    }
  }
  return d;
}

}  // namespace

double gather_lines_per_point(const PointSet& ps, const std::vector<std::int32_t>& order) {
  // 128 evenly spaced groups (2048 points) separate the orders clearly
  // (1.6-2.1 vs 8 lines per point) at any size; distinct lines are counted
  // with a small open-addressing set, serially (~0.1 ms at 160K points).
  const std::int32_t n = ps.n();
  const std::int64_t groups = n / kGroup;
  if (groups < 2) return 0.0;
  std::vector<std::int32_t> inv;
  if (!order.empty()) {
    inv.resize(static_cast<std::size_t>(n));
    for (std::int32_t k = 0; k < n; ++k) inv[order[k]] = k;
  }
  constexpr int kSlots = 1024;
  std::vector<std::int32_t> key(kSlots);
  std::vector<std::uint32_t> tag(kSlots, 0);
  std::uint32_t cur = 0;
  const std::int64_t samples = std::min<std::int64_t>(groups, 128);
  double lines = 0.0, points = 0.0;
  for (std::int64_t q = 0; q < samples; ++q) {
    const std::int32_t k0 = static_cast<std::int32_t>(q * groups / samples * kGroup);
    ++cur;
    int distinct = 0, entries = 0;
    for (std::int32_t k = k0; k < k0 + kGroup; ++k) {
      const std::int32_t p = order.empty() ? k : order[k];
      for (std::int64_t e = ps.off[p]; e < ps.off[p + 1] && entries < kSlots / 2; ++e, ++entries) {
        const std::int32_t nb = ps.nbr[e];
        const std::int32_t line = (inv.empty() ? nb : inv[nb]) >> 1;  // 64-byte records, two per line
        std::uint32_t h = (static_cast<std::uint32_t>(line) * 2654435761u) >> 22;
        while (tag[h] == cur && key[h] != line) h = (h + 1) & (kSlots - 1);
        if (tag[h] != cur) {
          tag[h] = cur;
          key[h] = line;
          ++distinct;
        }
      }
    }
    lines += distinct;
    points += kGroup;
  }
  return lines / points;
}

std::vector<std::int32_t> hilbert_order(const PointSet& ps) {
  const std::int32_t n = ps.n();
  std::vector<std::int32_t> order(static_cast<std::size_t>(n));
  if (n == 0) return order;
  const auto [xmin, xmax] = std::minmax_element(ps.x.begin(), ps.x.end());
  const auto [ymin, ymax] = std::minmax_element(ps.y.begin(), ps.y.end());
  const double x0 = *xmin, y0 = *ymin;
  const double sx = *xmax > x0 ? 65535.0 / (*xmax - x0) : 0.0, sy = *ymax > y0 ? 65535.0 / (*ymax - y0) : 0.0;
  std::vector<std::uint64_t> key(static_cast<std::size_t>(n));
  parallel_slices(n, [&](std::int64_t lo, std::int64_t hi) {
    for (std::int64_t i = lo; i < hi; ++i) {
      const auto qx = static_cast<std::uint32_t>(std::min(65535.0, std::max(0.0, (ps.x[i] - x0) * sx)));
      const auto qy = static_cast<std::uint32_t>(std::min(65535.0, std::max(0.0, (ps.y[i] - y0) * sy)));
      key[i] = (static_cast<std::uint64_t>(hilbert_index(qx, qy)) << 32) | static_cast<std::uint32_t>(i);
    }
  }, 1 << 14);
  std::sort(key.begin(), key.end());  // ties (same cell) in ascending id
  for (std::int32_t k = 0; k < n; ++k) order[k] = static_cast<std::int32_t>(key[k] & 0xFFFFFFFFu);
  return order;
}

std::vector<std::int32_t> rcm_order(const PointSet& ps) {
  // Reverse Cuthill-McKee over the stencil graph: breadth-first from a
  // pseudo-peripheral point of each connected piece (two sweeps of "start at
  // the last point of the deepest level"), neighbours in stencil order, the
  // whole sequence reversed.  On an O-cloud the levels are rings.
  const std::int32_t n = ps.n();
  std::vector<std::int32_t> order;
  order.reserve(static_cast<std::size_t>(n));
  std::vector<std::int32_t> stamp(static_cast<std::size_t>(n), 0), queue(static_cast<std::size_t>(n));
  std::vector<char> placed(static_cast<std::size_t>(n), 0);
  std::int32_t gen = 0;
  // BFS over unplaced points from s; returns the number of points reached
  // (queue[0..count)), in visiting order.
  auto bfs = [&](std::int32_t s) {
    ++gen;
    std::int32_t head = 0, tail = 0;
    queue[tail++] = s;
    stamp[s] = gen;
    while (head < tail) {
      const std::int32_t p = queue[head++];
      for (std::int64_t e = ps.off[p]; e < ps.off[p + 1]; ++e) {
        const std::int32_t nb = ps.nbr[e];
        if (stamp[nb] != gen && !placed[nb]) {
          stamp[nb] = gen;
          queue[tail++] = nb;
        }
      }
    }
    return tail;
  };
  for (std::int32_t s0 = 0; s0 < n; ++s0) {
    if (placed[s0]) continue;
    std::int32_t r = s0;
    for (int sweep = 0; sweep < 2; ++sweep) r = queue[bfs(r) - 1];
    const std::int32_t cnt = bfs(r);
    for (std::int32_t k = 0; k < cnt; ++k) {
      placed[queue[k]] = 1;
      order.push_back(queue[k]);
    }
  }
  std::reverse(order.begin(), order.end());
  return order;
}

const Locality& cloud_locality(const PointSet& ps, int mode) {
  if (ps.locality && ps.locality->mode == mode) return *ps.locality;
  auto loc = std::make_shared<Locality>();
  loc->mode = mode;
  if (mode != kReorderNone) {
    loc->lines_before = gather_lines_per_point(ps, {});
    if (mode != kReorderAuto || loc->lines_before > kPoorLines) {
      std::vector<std::int32_t> o = mode == kReorderHilbert ? hilbert_order(ps) : rcm_order(ps);
      loc->lines_after = gather_lines_per_point(ps, o);
      if (mode != kReorderAuto || loc->lines_after < 0.8 * loc->lines_before) loc->order = std::move(o);
    }
  }
  ps.locality = std::move(loc);
  return *ps.locality;
}

}  // namespace lskb

namespace lskb {

LocalGeom permuted_geom(const PointSet& ps, const std::vector<std::int32_t>& order,
                        const std::vector<std::uint16_t>& part_of) {
  const std::int32_t n = ps.n();
  LocalGeom g;
  g.n_own = g.n_loc = n;
  g.gid = order;
  std::vector<std::int32_t> inv(static_cast<std::size_t>(n));
  for (std::int32_t k = 0; k < n; ++k) inv[order[k]] = k;
  const std::size_t nn = static_cast<std::size_t>(n);
  g.x.resize(nn);
  g.y.resize(nn);
  g.nx.resize(nn);
  g.ny.resize(nn);
  g.kind.resize(nn);
  g.part.resize(nn);
  g.off.resize(nn + 1);
  g.off[0] = 0;
  for (std::int32_t k = 0; k < n; ++k) g.off[k + 1] = g.off[k] + ps.degree(order[k]);
  g.nbr.resize(static_cast<std::size_t>(g.off[n]));
  parallel_slices(n, [&](std::int64_t lo, std::int64_t hi) {
    for (std::int64_t k = lo; k < hi; ++k) {
      const std::int32_t p = order[k];
      g.x[k] = ps.x[p];
      g.y[k] = ps.y[p];
      g.nx[k] = ps.nx[p];
      g.ny[k] = ps.ny[p];
      g.kind[k] = ps.kind[p];
      g.part[k] = part_of.empty() ? 0 : part_of[p];
      std::int64_t o = g.off[k];
      for (std::int64_t e = ps.off[p]; e < ps.off[p + 1]; ++e) g.nbr[o++] = inv[ps.nbr[e]];  // stencil order kept
    }
  }, 1 << 14);
  return g;
}

}  // namespace lskb
