// decompose.cpp — RCB pieces -> device domains with halo maps.
//
// Each piece of bisect_cloud (the reference's partition_cloud, bit-exact) becomes
// one device domain: its owned points in ascending global id (or in the
// cloud's locality order, config key reorder), then its halo
// (stencil closure minus owned, ascending) as read-only copies.  Stencils are
// rewritten to local ids in the original (ascending global id) order, so every
// per-point sum keeps the reference's operation order and results do not
// depend on the number of domains.
#include <algorithm>

#include "../engine.hpp"
#include "core.hpp"
#include "par.hpp"

namespace lskb {

std::vector<LocalGeom> decompose(const PointSet& ps, int n_domains, const std::vector<std::uint16_t>& part_of,
                                 int reorder) {
  std::vector<Piece> pieces = bisect_cloud(ps, n_domains);
  const std::int32_t n = ps.n();
  // Locality numbering (reorder.cpp): each domain's owned points follow the
  // cloud's locality order instead of ascending id.
  const Locality& loc = cloud_locality(ps, reorder);
  if (!loc.order.empty()) {
    std::vector<std::int32_t> rank(static_cast<std::size_t>(n));
    for (std::int32_t k = 0; k < n; ++k) rank[loc.order[k]] = k;
    for (Piece& pc : pieces)
      std::sort(pc.owned.begin(), pc.owned.end(), [&](std::int32_t a, std::int32_t b) { return rank[a] < rank[b]; });
  }
  std::vector<std::int32_t> owner(static_cast<std::size_t>(n)), owner_local(static_cast<std::size_t>(n));
  for (std::size_t d = 0; d < pieces.size(); ++d)
    for (std::size_t k = 0; k < pieces[d].owned.size(); ++k) {
      owner[pieces[d].owned[k]] = static_cast<std::int32_t>(d);
      owner_local[pieces[d].owned[k]] = static_cast<std::int32_t>(k);
    }
  std::vector<LocalGeom> out(pieces.size());
  parallel_slices(
      static_cast<std::int64_t>(pieces.size()),
      [&](std::int64_t lo, std::int64_t hi) {
        for (std::int64_t d = lo; d < hi; ++d) {
          const Piece& pc = pieces[static_cast<std::size_t>(d)];
          LocalGeom& g = out[static_cast<std::size_t>(d)];
          g.n_own = static_cast<std::int32_t>(pc.owned.size());
          g.n_loc = g.n_own + static_cast<std::int32_t>(pc.halo.size());
          g.gid = pc.owned;
          g.gid.insert(g.gid.end(), pc.halo.begin(), pc.halo.end());
          const std::size_t nl = static_cast<std::size_t>(g.n_loc);
          g.x.resize(nl);
          g.y.resize(nl);
          g.nx.resize(nl);
          g.ny.resize(nl);
          g.kind.resize(nl);
          g.part.resize(nl);
          for (std::size_t i = 0; i < nl; ++i) {
            const std::int32_t p = g.gid[i];
            g.x[i] = ps.x[p];
            g.y[i] = ps.y[p];
            g.nx[i] = ps.nx[p];
            g.ny[i] = ps.ny[p];
            g.kind[i] = ps.kind[p];
            g.part[i] = part_of.empty() ? 0 : part_of[p];
          }
          g.off.assign(1, 0);
          for (std::int32_t i = 0; i < g.n_own; ++i) {
            const std::int32_t p = pc.owned[static_cast<std::size_t>(i)];
            for (std::int64_t e = ps.off[p]; e < ps.off[p + 1]; ++e) {
              const std::int32_t nb = ps.nbr[e];
              if (owner[nb] == d) {
                g.nbr.push_back(owner_local[nb]);
              } else {
                const auto it = std::lower_bound(pc.halo.begin(), pc.halo.end(), nb);
                g.nbr.push_back(g.n_own + static_cast<std::int32_t>(it - pc.halo.begin()));
              }
            }
            g.off.push_back(static_cast<std::int64_t>(g.nbr.size()));
          }
          g.halo_dom.resize(pc.halo.size());
          g.halo_idx.resize(pc.halo.size());
          for (std::size_t h = 0; h < pc.halo.size(); ++h) {
            g.halo_dom[h] = owner[pc.halo[h]];
            g.halo_idx[h] = owner_local[pc.halo[h]];
          }
        }
      },
      1);
  return out;
}

}  // namespace lskb
