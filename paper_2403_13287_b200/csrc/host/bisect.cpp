// bisect.cpp — recursive coordinate bisection into device domains.
//
// Index-map parity with the reference partition_cloud (partition.cpp:12-80):
// at each level the candidate ids are ordered by (coordinate, id) along the
// longer bounding-box side (x on ties), the cut is
// (size * n_left + n_parts/2) / n_parts with n_left = (n_parts+1)/2, and the
// left piece is numbered before the right.  Owned lists are ascending; the
// halo of a piece is its stencil closure minus its owned points, ascending
// and unique.  These lists drive the multi-device layout and the error
// tie-break (lowest piece reports first, runtime.cpp:115-118).
#include <algorithm>
#include <numeric>

#include "core.hpp"

namespace lskb {

namespace {

void split(const PointSet& ps, std::vector<std::int32_t>& ids, int parts, std::vector<Piece>& out) {
  if (parts == 1) {
    Piece piece;
    piece.owned = ids;
    std::sort(piece.owned.begin(), piece.owned.end());
    out.push_back(std::move(piece));
    return;
  }
  double xlo = ps.x[ids[0]], xhi = xlo, ylo = ps.y[ids[0]], yhi = ylo;
  for (std::int32_t i : ids) {
    xlo = std::min(xlo, ps.x[i]);
    xhi = std::max(xhi, ps.x[i]);
    ylo = std::min(ylo, ps.y[i]);
    yhi = std::max(yhi, ps.y[i]);
  }
  const HVec<double>& key = (xhi - xlo) >= (yhi - ylo) ? ps.x : ps.y;
  std::sort(ids.begin(), ids.end(), [&key](std::int32_t a, std::int32_t b) {
    return key[a] < key[b] || (key[a] == key[b] && a < b);
  });
  const int left_parts = (parts + 1) / 2;
  const std::size_t cut = (ids.size() * static_cast<std::size_t>(left_parts) + parts / 2) / parts;
  std::vector<std::int32_t> lo(ids.begin(), ids.begin() + static_cast<std::ptrdiff_t>(cut));
  std::vector<std::int32_t> hi(ids.begin() + static_cast<std::ptrdiff_t>(cut), ids.end());
  split(ps, lo, left_parts, out);
  split(ps, hi, parts - left_parts, out);
}

}  // namespace

std::vector<Piece> bisect_cloud(const PointSet& ps, int n_parts) {
  if (n_parts < 1) raise(Status::argument, "partition count must be >= 1");
  if (n_parts > ps.n())
    raise(Status::argument, "more partitions than points (" + std::to_string(n_parts) + " > " +
                                std::to_string(ps.n()) + ")");
  std::vector<std::int32_t> ids(static_cast<std::size_t>(ps.n()));
  std::iota(ids.begin(), ids.end(), 0);
  std::vector<Piece> out;
  out.reserve(static_cast<std::size_t>(n_parts));
  split(ps, ids, n_parts, out);
  std::vector<std::uint8_t> mine(static_cast<std::size_t>(ps.n()), 0);
  for (Piece& piece : out) {
    for (std::int32_t i : piece.owned) mine[i] = 1;
    for (std::int32_t i : piece.owned)
      for (std::int64_t e = ps.off[i]; e < ps.off[i + 1]; ++e)
        if (!mine[ps.nbr[e]]) piece.halo.push_back(ps.nbr[e]);
    std::sort(piece.halo.begin(), piece.halo.end());
    piece.halo.erase(std::unique(piece.halo.begin(), piece.halo.end()), piece.halo.end());
    for (std::int32_t i : piece.owned) mine[i] = 0;
  }
  return out;
}

}  // namespace lskb
