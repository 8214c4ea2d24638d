// tiles.cuh — shared-memory tiles of the point cloud for the derivative sweep.
//
// The sweep (reference q_derivatives_kernel, kernels.cpp:82-106) is a gather:
// every point reads xy, q, qx, qy of its 8 neighbours (112 bytes each).  With
// per-lane global gathers it is bound by load latency and L1 wavefronts
// (round-2 ncu: long-scoreboard stalls, LSU at 69%, 55% of HBM).  Here the
// owned points are cut into tiles of TP consecutive device ids; the union of a
// tile's points and their stencils is, for the locality-ordered clouds the
// engine runs (generator order ring by ring, or RCM), a handful of id
// intervals — the rows above, at and below the tile.  A tile plan (geometry
// only, built once per domain on the device) stores those intervals and, per
// pair, the neighbour's slot in the staged array.  The sweep kernel stages a
// tile with cp.async.bulk (TMA 1-D bulk copies completing on an mbarrier,
// double-buffered per block: the next tile's copies fly while the current one
// is computed) and then gathers from shared memory, where 16 consecutive
// points' halves of a record are 512 contiguous bytes (no bank conflicts:
// dq_load's two-plane layout).  Tiles whose union needs more than kTileIv
// intervals or more than the stage capacity are marked (nint = 0) and gathered
// from global memory by the same kernel.  The per-point arithmetic and its
// order are exactly those of k_sweep2, so strict mode stays bitwise.
#pragma once

#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>

#include "kernels.cuh"

namespace lskd {

constexpr int kTileIv = 8;  // intervals per tile (more: the tile is gathered from global memory)
constexpr int kTileGap = 16;   // id gaps up to this are staged instead of starting a new interval
constexpr int kTileRec = 112;  // staged bytes per point: xy 16 + q 32 + qx 32 + qy 32

// Plan record of one tile (80 bytes, bulk-copied into the stage that holds the
// tile before it, so a stage refill never waits on global memory).
struct TileIv {
  int start, len;
};
struct TilePlan {
  int nint;    // intervals (0: gather this tile from global memory)
  int staged;  // staged points (sum of the interval lengths)
  int own;     // slot of the tile's first point
  int pad;
  TileIv iv[kTileIv];
};
constexpr unsigned kPlanBytes = sizeof(TilePlan);            // bulk-copied with the stage before
constexpr int kPlanSlot = (static_cast<int>(sizeof(TilePlan)) + 127) / 128 * 128;  // its room in a stage
static_assert(sizeof(TilePlan) % 16 == 0, "TilePlan is bulk-copied");

// One block per tile of TP points (uniform 8-point stencils): sort the tile's
// 9 TP ids (own + neighbours), cut them into intervals at gaps > kTileGap,
// then write the header, the intervals and every pair's slot.
template <int TP>
__global__ void __launch_bounds__(TP) k_tile_plan(Geo g, int smax, TilePlan* plan, std::uint16_t* slot) {
  using Sort = cub::BlockRadixSort<int, TP, 9>;
  using Scan = cub::BlockScan<int, TP>;
  __shared__ union {
    typename Sort::TempStorage sort;
    typename Scan::TempStorage scan;
  } tmp;
  __shared__ int s_last[TP];
  __shared__ int s_start[kTileIv], s_end[kTileIv], s_soff[kTileIv];
  __shared__ int s_nint, s_ok, s_lo, s_hi;
  const int t = blockIdx.x;
  const int i0 = t * TP;
  const int i = i0 + static_cast<int>(threadIdx.x);
  const bool in = i < g.n;
  const int ic = in ? i : i0;  // points past the end repeat the first one
  int keys[9];
  keys[0] = ic;
#pragma unroll
  for (int j = 0; j < 8; ++j) keys[1 + j] = g.nbr[8ll * ic + j];
  // sort the offsets from the tile's smallest id on only as many bits as the
  // id window needs (2 radix passes instead of 4 for a ring-ordered cloud)
  if (threadIdx.x == 0) {
    s_lo = 0x7FFFFFFF;
    s_hi = 0;
  }
  __syncthreads();
  int lo = keys[0], hi = keys[0];
#pragma unroll
  for (int j = 1; j < 9; ++j) lo = min(lo, keys[j]), hi = max(hi, keys[j]);
  atomicMin(&s_lo, lo);
  atomicMax(&s_hi, hi);
  __syncthreads();
  const int base_id = s_lo;
  const int bits = 32 - __clz(static_cast<unsigned>(s_hi - base_id) | 1u);
#pragma unroll
  for (int j = 0; j < 9; ++j) keys[j] -= base_id;
  Sort(tmp.sort).Sort(keys, 0, bits);  // blocked: thread t holds ranks 9t .. 9t+8
#pragma unroll
  for (int j = 0; j < 9; ++j) keys[j] += base_id;
  s_last[threadIdx.x] = keys[8];
  __syncthreads();
  // interval starts: the first key, and every key more than kTileGap + 1 above its predecessor
  bool first_k[9];
  int starts = 0;
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const bool head = threadIdx.x == 0 && k == 0;
    const int prev = k ? keys[k - 1] : (threadIdx.x ? s_last[threadIdx.x - 1] : 0);
    first_k[k] = head || (keys[k] - prev > kTileGap + 1);
    starts += first_k[k] ? 1 : 0;
  }
  int base = 0, total = 0;
  Scan(tmp.scan).ExclusiveSum(starts, base, total);
  int r = base;
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    if (first_k[k]) {
      if (r < kTileIv) s_start[r] = keys[k];
      if (r >= 1 && r - 1 < kTileIv) s_end[r - 1] = k ? keys[k - 1] : s_last[threadIdx.x - 1];
      ++r;
    }
  }
  if (threadIdx.x == TP - 1 && total - 1 < kTileIv) s_end[total - 1] = keys[8];
  __syncthreads();
  if (threadIdx.x == 0) {
    int ok = total <= kTileIv, staged = 0, own = 0;
    if (ok) {
      for (int q = 0; q < total; ++q) {
        s_soff[q] = staged;
        if (s_start[q] <= i0 && i0 <= s_end[q]) own = staged + (i0 - s_start[q]);
        staged += s_end[q] - s_start[q] + 1;
      }
      ok = staged <= smax;
    }
    s_ok = ok;
    s_nint = total;
    TilePlan pl{};
    pl.nint = ok ? total : 0;
    pl.staged = ok ? staged : 0;
    pl.own = own;
    if (ok)
      for (int q = 0; q < total; ++q) pl.iv[q] = TileIv{s_start[q], s_end[q] - s_start[q] + 1};
    plan[t] = pl;
  }
  __syncthreads();
  if (!s_ok || !in) return;
  const int nint = s_nint;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int nb = g.nbr[8ll * i + j];
    int q = 0;
    while (q + 1 < nint && nb > s_end[q]) ++q;
    slot[8ll * i + j] = static_cast<std::uint16_t>(s_soff[q] + (nb - s_start[q]));
  }
}

// ---- TMA bulk copies and mbarriers (1-D, no tensor map) ----
__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W: mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Neighbour sources of the tiled sweep: lane h of a point reads its halves
// {2h, 2h+1} of q, qx and qy.
struct SmemSrc {  // a staged tile
  const double2* xy;
  const double2* q;   // 2 halves per point
  const double2* qx;
  const double2* qy;
  int h;
  __device__ __forceinline__ void get(int s, double2& p, double2& qv, double2& x, double2& y) const {
    p = xy[s];
    qv = q[2 * s + h];
    x = qx[2 * s + h];
    y = qy[2 * s + h];
  }
};
// Stage layout (bytes): [0, 128) the plan of the tile this stage holds next,
// [128, 128 + 16 TP) the tile's neighbour slots, then xy [smax] x 16 B,
// q [smax] x 32 B, qx [smax] x 32 B, qy [smax] x 32 B.
__host__ __device__ constexpr std::size_t tile_stage_bytes(int tp, int smax) {
  return kPlanSlot + 16 * static_cast<std::size_t>(tp) + static_cast<std::size_t>(smax) * kTileRec;
}

// The tiled sweep: 2 TP threads per block (two lanes per point), persistent
// over tiles (tile = blockIdx.x + k gridDim.x), 2 stages per block.  Stage s
// is filled by bulk copies completing on full[s]: the plan record of the tile
// after next for this stage, the tile's slots, and per interval its xy, q, qx
// and qy ranges.  Warps are decoupled: a warp that is done with a stage counts
// itself out (shared atomic); the last one refills the stage from the plan
// record that came with it (lane r issues interval r's four copies), so no
// block barrier sits in the loop and no refill waits on global memory.
template <bool S, int TP, int MB, bool LIST = false>
__global__ void __launch_bounds__(2 * TP, MB)
    k_sweep_tile(Geo g, const D4* __restrict__ q, const D4* __restrict__ dq_in, D4* __restrict__ dq_out, Gas gas,
                 Ctl* ctl, int sweep, const TilePlan* __restrict__ plan, const std::uint16_t* __restrict__ slot,
                 int smax, int ntiles, const int* __restrict__ tlist) {
  // tlist: visit only the tiles tlist[0 .. ntiles) (a rank's interior tiles);
  // null: tiles 0 .. ntiles.  k below is the visit index, tile_at(k) the tile.
  constexpr int NS = 2;
  constexpr int NW = 2 * TP / 32;
  pdl_enter();
  extern __shared__ __align__(128) char tsm[];
  __shared__ unsigned long long full[NS];
  __shared__ int2 cur[NS];  // {nint, own} of the tile a stage holds
  __shared__ int done[NS];
  __shared__ int s_skip;
  ktimer_begin(ctl, kt_sweep(sweep));
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) {
    s_skip = skip_stage(ctl, 1 + sweep);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      done[s] = 0;
    }
    mbar_fence_init();
  }
  __syncthreads();
  const bool run = !s_skip;
  const std::size_t sb = tile_stage_bytes(TP, smax);
  auto stage = [&](int s) { return tsm + s * sb; };
  auto slots_of = [&](int s) { return stage(s) + kPlanSlot; };
  auto xy_of = [&](int s) { return stage(s) + kPlanSlot + 16 * TP; };
  auto q_of = [&](int s) { return xy_of(s) + static_cast<std::size_t>(smax) * 16; };
  auto qx_of = [&](int s) { return xy_of(s) + static_cast<std::size_t>(smax) * 48; };
  auto qy_of = [&](int s) { return xy_of(s) + static_cast<std::size_t>(smax) * 80; };
  const D4* qyp = dq_in + g.nloc;
  const int grid = static_cast<int>(gridDim.x);
  auto tile_at = [&](int k) { return LIST ? tlist[k] : k; };
  // Refill stage s with the tile of visit k (one warp; pp = the tile's plan,
  // in global or shared memory; lane r reads interval r).
  auto issue = [&](int k, int s, const TilePlan* pp) {
    const int tile = tile_at(k);
    const int nint = pp->nint, own = pp->own, staged = pp->staged;
    const TileIv v = lane < nint ? pp->iv[lane] : TileIv{0, 0};
    const int len = v.len;
    int off = len;  // inclusive scan over the interval lanes -> staged offset of this lane's interval
#pragma unroll
    for (int o = 1; o < kTileIv; o <<= 1) {
      const int v = __shfl_up_sync(0xFFFFFFFFu, off, o);
      if (lane >= o) off += v;
    }
    off -= len;
    const long long start = v.start;
    const int next = k + NS * grid;
    const int npts = min(TP, g.n - tile * TP);
    __syncwarp();  // every lane has read the plan (it may live in the stage being refilled)
    if (lane == 0) {
      cur[s] = make_int2(nint, own);
      const unsigned bytes = (next < ntiles ? kPlanBytes : 0u) + 16u * npts + static_cast<unsigned>(staged) * kTileRec;
      mbar_arrive_tx(&full[s], bytes);
    }
    __syncwarp();
    if (lane == 0 && next < ntiles) bulk_g2s(stage(s), plan + tile_at(next), kPlanBytes, &full[s]);
    if (lane == 1) bulk_g2s(slots_of(s), slot + 8ll * tile * TP, 16u * npts, &full[s]);
    if (len > 0) {
      bulk_g2s(xy_of(s) + off * 16, g.xy + start, len * 16u, &full[s]);
      bulk_g2s(q_of(s) + off * 32, q + start, len * 32u, &full[s]);
      bulk_g2s(qx_of(s) + off * 32, dq_in + start, len * 32u, &full[s]);
      bulk_g2s(qy_of(s) + off * 32, qyp + start, len * 32u, &full[s]);
    }
  };
  const int warp = tid >> 5;
  if (run && warp == 0) {
    for (int s = 0; s < NS; ++s) {
      const int k = blockIdx.x + s * grid;
      if (k < ntiles) issue(k, s, plan + tile_at(k));
    }
  }
  const int p = tid >> 1, h = tid & 1;
  const GlobalSrc gsrc{reinterpret_cast<const double*>(g.xy), reinterpret_cast<const double*>(q) + 2 * h,
                       reinterpret_cast<const double*>(dq_in) + 2 * h, reinterpret_cast<const double*>(qyp) + 2 * h};
  int it = 0;
  for (int k = blockIdx.x; run && k < ntiles; k += grid, ++it) {
    const int s = it & (NS - 1);
    const int tile = tile_at(k);
    mbar_wait(&full[s], static_cast<unsigned>(it / NS) & 1u);
    const int2 th = cur[s];
    const int i = tile * TP + p;
    if (i < g.n) {
      if (th.x > 0) {
        const uint4 sl = reinterpret_cast<const uint4*>(slots_of(s))[p];
        const int nbr[8] = {static_cast<int>(sl.x & 0xFFFFu), static_cast<int>(sl.x >> 16),
                            static_cast<int>(sl.y & 0xFFFFu), static_cast<int>(sl.y >> 16),
                            static_cast<int>(sl.z & 0xFFFFu), static_cast<int>(sl.z >> 16),
                            static_cast<int>(sl.w & 0xFFFFu), static_cast<int>(sl.w >> 16)};
        const SmemSrc ssrc{reinterpret_cast<const double2*>(xy_of(s)), reinterpret_cast<const double2*>(q_of(s)),
                           reinterpret_cast<const double2*>(qx_of(s)), reinterpret_cast<const double2*>(qy_of(s)), h};
        sweep_point8<S>(ssrc, th.y + p, nbr, g, i, h, dq_out, gas, ctl, sweep);
      } else {
        const int4 na0 = ld_i4(g.nbr + 8ll * i), na1 = ld_i4(g.nbr + 8ll * i + 4);
        const int nbr[8] = {na0.x, na0.y, na0.z, na0.w, na1.x, na1.y, na1.z, na1.w};
        sweep_point8<S>(gsrc, i, nbr, g, i, h, dq_out, gas, ctl, sweep);
      }
    }
    // count this warp out of stage s; the last warp refills it.  Every value
    // this warp read from the stage has been consumed (the derivatives are
    // stored) before it counts itself out, so the refill's bulk copies cannot
    // overtake a read.  compute-sanitizer racecheck does not model this
    // shared-atomic hand-off and reports the refill's writes against the
    // earlier reads; release/acquire fences plus fence.proxy.async around the
    // count do not silence it and cost 2.8% (0.499 -> 0.513 ms at 10M), so the
    // protocol stays as is (the tiled sweep is bitwise the untiled one in
    // every test, tests/test_gpu_tiles.py).
    __syncwarp();
    int last = 0;
    if (lane == 0) {
      last = atomicAdd(&done[s], 1) == NW - 1;
      if (last) done[s] = 0;
    }
    last = __shfl_sync(0xFFFFFFFFu, last, 0);
    const int next = k + NS * grid;
    if (last && next < ntiles) issue(next, s, reinterpret_cast<const TilePlan*>(stage(s)));
  }
  __syncthreads();
  ktimer_end(ctl, kt_sweep(sweep));
}

}  // namespace lskd
