// kernels.cuh — sm_100a kernels of one LSKUM fixed-point iteration.
//
// Device-side replacement for the reference's phase kernels
// (/root/reference/proj/src/core/kernels.cpp:68-223) and residue reduction
// (runtime.cpp:251-269, reduce.hpp:11-17).  Per iteration (order 2, n_inner s):
//
//   k_sweep   x s   q, dq[b] -> dq[1-b]      one thread per point, bitwise
//   k_flux          q[a], dq -> res                 (W lanes per point)
//   k_update        res, prim -> dt -> prim' -> q[1-a], mag
//                   (local time step + forward Euler + wall slip + next
//                    q-variables + residue summand, one thread per point)
//   k_tree_partial, k_tree_final   midpoint-tree sum of mag, bitwise
//
// Data layout in HBM (structure of arrays of 32-byte records):
//   xy  double2[n]        nrm double2[n]     kind u8[n]     part u8[n]
//   off int32[n+1]        nbr int32[nnz]     mind double[n] (geometry, per run)
//   prim D4[n]            q[2] D4[n]         dq[2] D4[2n]  ({qx0,qx1,qy0,qy1}, {qx2,qx3,qy2,qy3})
//   res D4[n] (every iteration), dt double[n] (copy-back iteration only), mag double[n]
// Every D4 gather is one 256-bit LDG (one 32-byte sector).
#pragma once

#include <cstdint>

#include "dmath.cuh"

namespace lskd {

constexpr unsigned long long kNoErr = ~0ull;
// PH_STALL: a cross-process wait timed out (per-rank runs only).
enum : unsigned { PH_QVAR = 0, PH_SWEEP = 1, PH_FLUX = 2, PH_UPDATE = 3, PH_RESIDUE = 4, PH_STALL = 5 };
enum : unsigned { KIND_INTERIOR = 0, KIND_WALL = 1, KIND_OUTER = 2 };
constexpr unsigned kSolveSlot = 0x3FFFu;  // "after every neighbour" in the error key
constexpr int kMaxParts = 4096;          // partitions the error key distinguishes (12 bits)
constexpr int kMaxStencil = 0x3FFE;      // neighbour positions the error key distinguishes (14 bits)

// Error key: min over failures reproduces the reference's first failure
// (phase order, lowest partition, ascending point id, direction Gx+..Gy-,
// neighbour position) — runtime.cpp:115-118, kernels.cpp:122, :37-64.
//   phase(3)@61 | dmaj(2)@59 | part(12)@47 | point(31)@16 | dir(2)@14 | j(14)@0
// dmaj is the direction again for residual_mode=split4 flux failures: there
// each direction is its own phase over all partitions (runtime.cpp:160-183),
// so the reference throws the lowest direction first, then the lowest
// partition; it is 0 otherwise (fused: partition, point, then direction).
__device__ __forceinline__ unsigned long long err_key(unsigned phase, unsigned part,
                                                      unsigned point, unsigned dir,
                                                      unsigned j, unsigned dmaj = 0) {
  return (static_cast<unsigned long long>(phase & 7u) << 61) |
         (static_cast<unsigned long long>(dmaj & 3u) << 59) |
         (static_cast<unsigned long long>(part & 0xFFFu) << 47) |
         (static_cast<unsigned long long>(point & 0x7FFFFFFFu) << 16) |
         (static_cast<unsigned long long>(dir & 3u) << 14) | (j & 0x3FFFu);
}
__host__ __device__ __forceinline__ unsigned key_phase(unsigned long long k) { return static_cast<unsigned>(k >> 61); }
__host__ __device__ __forceinline__ long long key_point(unsigned long long k) {
  return static_cast<long long>((k >> 16) & 0x7FFFFFFFull);
}
__host__ __device__ __forceinline__ unsigned key_dir(unsigned long long k) { return static_cast<unsigned>((k >> 14) & 3ull); }
__host__ __device__ __forceinline__ unsigned key_j(unsigned long long k) { return static_cast<unsigned>(k & 0x3FFFull); }

struct KTimer {
  unsigned long long t0, t1;
  unsigned int done, pad;
  unsigned long long total_ns, launches;
};

// Timer slots: one per kernel launch of an iteration (sweep s -> KT_SWEEP + s,
// the 8th and later sweeps share the last sweep slot).
enum : int { KT_QVAR = 0, KT_SWEEP = 1, KT_FLUX = 9, KT_UPDATE = 10, KT_RESIDUE = 11, KT_COUNT = 12 };
__host__ __device__ constexpr int kt_sweep(int s) { return KT_SWEEP + (s < 7 ? s : 7); }

// Failures are ordered by STAGE first: stage = iteration * spi + sub, with
// sub 0 = q_variables, 1+s = derivative sweep s, then flux, update, residue
// (spi = sweeps + 4).  A kernel skips only when a failure at an EARLIER stage
// is already recorded, so every domain still runs the stage of the first
// failure and records its own failures there; the run's failure is the
// minimum (stage, key) over the domains' records — exactly the reference's
// first throw whatever the relative progress of the domains.

// Run-wide control word, shared by every domain of a run (lives on the first
// domain's device; other domains reach it over peer memory).
struct Shared {
  unsigned long long err_stage;  // min failing stage over all domains (kNoErr = none)
  int iter;                      // 0-based index of the iteration in flight
  int pad[3];
};

// Per-domain control block: the shared word, this domain's own failure
// record (all at one stage, see above) and its kernel timers.
struct Ctl {
  Shared* sh;
  int diag_iter;  // iteration whose res/dt are kept for copy-back (this domain)
  int spi;        // stages per iteration
  int upd_blocks; // grid size of this domain's k_update
  // Blocks of k_update completed on this domain's stream.  The iteration a
  // kernel belongs to is upd_done / upd_blocks (failed or not): every block
  // of k_update adds one at its end, so k_update's own blocks still see their
  // iteration (fewer than upd_blocks of them have finished) and every later
  // kernel sees the next one.
  unsigned long long upd_done;
  unsigned long long err_stage;  // this domain's failing stage (kNoErr = none)
  unsigned long long err_key;    // min key at that stage
  int split4;                    // residual_mode=split4: flux failures ordered by direction first
  int pad_;
  KTimer kt[KT_COUNT];
};

struct Geo {
  const double2* xy;
  const double2* nrm;
  const std::uint8_t* kind;
  const std::uint16_t* part;
  const int* off;
  const int* nbr;
  const double* mind;
  const int* gid;  // local -> global point id (null: local ids are global)
  int n;           // owned points (kernels loop over these)
  int kfix;        // uniform stencil size (offsets are then i*kfix), 0 = use CSR offsets
  long long nloc;  // owned + halo points: the plane stride of the dq buffers (dq_load)
  // Optional subset of the owned points (k_sweep2, k_flux_ws): when set, the
  // kernel visits points list[0..nlist) instead of 0..n — interior points
  // before the halo arrives, boundary points after.
  const int* list = nullptr;
  int nlist = 0;
};

// Number of points a subset-aware kernel visits, and the t-th of them.
__device__ __forceinline__ int visit_count(const Geo& g) { return g.list ? g.nlist : g.n; }
__device__ __forceinline__ int visit_point(const Geo& g, int t) {
  return g.list ? (t < g.nlist ? g.list[t] : g.n) : t;
}

__device__ __forceinline__ int gidx(const Geo& g, int i) { return g.gid ? g.gid[i] : i; }

__device__ __forceinline__ void stencil_of(const Geo& g, int i, int& e0, int& k) {
  if (g.kfix > 0) {
    e0 = i * g.kfix;
    k = g.kfix;
  } else {
    e0 = g.off[i];
    k = g.off[i + 1] - e0;
  }
}

// Programmatic dependent launch: the iteration's kernels are launched with
// programmatic stream serialisation, so each one's launch is processed while
// its predecessor's last blocks drain; it waits here for the predecessor's
// completion (and memory) before touching anything.  No explicit trigger:
// the dependent launch fires as the predecessor's blocks exit (triggering at
// block start measured slower — early dependents occupy SM slots).  Without
// the launch attribute the wait is a no-op.
__device__ __forceinline__ void pdl_enter() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}

// The residue kernels run after k_update advanced `it`, hence `back`.
__device__ __forceinline__ int iter_of(const Ctl* ctl, int back = 0) {
  const unsigned long long done = *reinterpret_cast<const volatile unsigned long long*>(&ctl->upd_done);
  return static_cast<int>(done / static_cast<unsigned>(ctl->upd_blocks)) - back;
}
__device__ __forceinline__ unsigned long long stage_of(const Ctl* ctl, int sub, int back = 0) {
  return static_cast<unsigned long long>(iter_of(ctl, back)) * static_cast<unsigned>(ctl->spi) +
         static_cast<unsigned>(sub);
}
// Stage subs of the per-iteration kernels after the sweeps.
__device__ __forceinline__ int sub_flux(const Ctl* ctl) { return ctl->spi - 3; }
__device__ __forceinline__ int sub_update(const Ctl* ctl) { return ctl->spi - 2; }
__device__ __forceinline__ int sub_residue(const Ctl* ctl) { return ctl->spi - 1; }

// True when a failure at a stage before `sub` of this iteration is recorded.
__device__ __forceinline__ bool skip_stage(const Ctl* ctl, int sub, int back = 0) {
  const unsigned long long first =
      min(ld_volatile(&ctl->sh->err_stage), ld_volatile(&ctl->err_stage));
  return first != kNoErr && first < stage_of(ctl, sub, back);
}

__device__ __forceinline__ void raise_err(Ctl* ctl, unsigned long long key, int sub, int back = 0) {
  const unsigned long long st = stage_of(ctl, sub, back);
  atomicMin(&ctl->err_stage, st);
  atomicMin(&ctl->err_key, key);
  atomicMin(&ctl->sh->err_stage, st);
}

// Flux failure key: direction-major under residual_mode=split4 (see err_key).
// Only read on the failure path.
__device__ __forceinline__ unsigned long long flux_key(const Ctl* ctl, unsigned part, unsigned point,
                                                       unsigned dir, unsigned j) {
  return err_key(PH_FLUX, part, point, dir, j, ctl->split4 ? dir : 0u);
}

// ---- per-kernel device timing (globaltimer) ----
// Each launch marks its slot with fire-and-forget atomics: first block start
// (min) and last block end (max).  k_tree_final, the iteration's last kernel,
// folds the slots into totals and resets them (ktimer_fold_warp) — no fences or
// completion counters in the kernels' tails.
__device__ __forceinline__ void ktimer_begin(Ctl* ctl, int k) {
  if (threadIdx.x == 0) atomicMin(&ctl->kt[k].t0, globaltimer());
}
// Call after a __syncthreads() that every thread of the block reaches.
__device__ __forceinline__ void ktimer_end(Ctl* ctl, int k, unsigned long long* = nullptr) {
  if (threadIdx.x == 0) atomicMax(&ctl->kt[k].t1, globaltimer());
}
// Folds every marked slot into its totals and resets it; one lane per slot
// (call with the whole first warp; the slots' loads are then in flight
// together instead of one slot after another).  Returns, in every lane, the
// earliest start of the iteration's kernels (slots other than q_variables).
__device__ __forceinline__ unsigned long long ktimer_fold_warp(Ctl* ctl) {
  const int lane = threadIdx.x & 31;
  unsigned long long first = ~0ull;
  if (lane < KT_COUNT) {
    KTimer& t = ctl->kt[lane];
    const unsigned long long t0 = t.t0, t1 = t.t1;
    if (!(t1 == 0 || t0 == ~0ull)) {
      if (lane != KT_QVAR) first = t0;
      t.total_ns += t1 > t0 ? t1 - t0 : 0;
      t.launches += 1;
      t.t0 = ~0ull;
      t.t1 = 0;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(0xFFFFFFFFu, first, o);
    first = v < first ? v : first;
  }
  return first;
}

// ---------------------------------------------------------------------------
// Geometry: nearest-neighbour distance per point (the min over the stencil in
// local_timestep_kernel, kernels.cpp:170-175) — constant for a run.
// Also counts the pairs of non-outer points with a zero offset (dx == 0 or
// dy == 0): they belong to both half stencils of that axis, and the fast flux
// only allocates and reads their second weight table (w2) when there are any.
__global__ void k_min_dist(Geo g, double* mind, unsigned long long* zero_pairs) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned z = 0;
  if (i < g.n) {
    const double2 pi = g.xy[i];
    double best = __longlong_as_double(0x7FF0000000000000ll);  // +inf
    for (int e = g.off[i]; e < g.off[i + 1]; ++e) {
      const double2 pn = g.xy[g.nbr[e]];
      const double dx = X::sub(pn.x, pi.x), dy = X::sub(pn.y, pi.y);
      const double d = sqrt(X::add(X::mul(dx, dx), X::mul(dy, dy)));
      best = d < best ? d : best;  // std::min(best, d)
      z += (dx == 0.0 || dy == 0.0) ? 1u : 0u;
    }
    mind[i] = best;
    if (g.kind[i] == KIND_OUTER) z = 0;
  }
  if (__any_sync(0xFFFFFFFFu, z != 0)) {
    const unsigned sum = __reduce_add_sync(0xFFFFFFFFu, z);
    if ((threadIdx.x & 31) == 0 && sum) atomicAdd(zero_pairs, static_cast<unsigned long long>(sum));
  }
}

// q_variables over all points (kernels.cpp:68-80); used for the first
// iteration and by the per-phase operator.  Afterwards q is produced by k_flux.
__global__ void k_qvar(Geo g, const D4* prim, D4* q, Gas gas, Ctl* ctl) {
  ktimer_begin(ctl, KT_QVAR);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < g.n) {
    const D4 s = ld4_rw(prim + i);
    if (!(s.a > 0.0) || !(s.d > 0.0)) {
      raise_err(ctl, err_key(PH_QVAR, g.part[i], gidx(g, i), 0, 0), 0);
    } else {
      st4(q + i, q_from_prim(s.a, s.b, s.c, s.d, gas.gm1));
    }
  }
  __syncthreads();
  ktimer_end(ctl, KT_QVAR, nullptr);
}

// One Jacobi sweep of the derivative system (kernels.cpp:82-106).  S = true
// (fp_mode strict): bitwise equal to the reference (exact operation sequence,
// ascending stencil order).  S = false: the same sums with FMA contraction.
template <bool S, int MB>
__global__ void __launch_bounds__(256, MB) k_sweep(Geo g, const D4* __restrict__ q,
                                                   const D4* __restrict__ dq_in, D4* __restrict__ dq_out,
                                                   Gas gas, Ctl* ctl, unsigned long long* iter_t0, int sweep) {
  pdl_enter();
  using A = Ar<S>;
  __shared__ int s_skip;
  ktimer_begin(ctl, kt_sweep(sweep));
  if (threadIdx.x == 0) s_skip = skip_stage(ctl, 1 + sweep);
  __syncthreads();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; !s_skip && i < g.n; i += gridDim.x * blockDim.x) {
    const double2 pi = g.xy[i];
    const D4 qi = ld4(q + i);
    D4 qxi, qyi;
    dq_load(dq_in, g.nloc, i, qxi, qyi);
    double sxx = 0.0, sxy = 0.0, syy = 0.0;
    double bx[4] = {0.0, 0.0, 0.0, 0.0}, by[4] = {0.0, 0.0, 0.0, 0.0};
    int e0, k;
    stencil_of(g, i, e0, k);
    for (int e = e0; e < e0 + k; ++e) {
      const int nb = g.nbr[e];
      const double2 pn = g.xy[nb];
      const double dx = X::sub(pn.x, pi.x), dy = X::sub(pn.y, pi.y);
      const D4 qn = ld4(q + nb);
      D4 qxn, qyn;
      dq_load(dq_in, g.nloc, nb, qxn, qyn);
      sxx = A::add(sxx, A::mul(dx, dx));
      sxy = A::add(sxy, A::mul(dx, dy));
      syy = A::add(syy, A::mul(dy, dy));
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double df = X::sub(corrected<S>(comp(qn, c), comp(qxn, c), comp(qyn, c), dx, dy),
                                 corrected<S>(comp(qi, c), comp(qxi, c), comp(qyi, c), dx, dy));
        bx[c] = A::add(bx[c], A::mul(dx, df));
        by[c] = A::add(by[c], A::mul(dy, df));
      }
    }
    const double det = A::sub(A::mul(sxx, syy), A::mul(sxy, sxy));
    if (!(det > gas.det_tol)) {
      raise_err(ctl, err_key(PH_SWEEP, g.part[i], gidx(g, i), 0, 0), 1 + sweep);
    } else {
      D4 fx, fy;
      fx.a = A::sub(A::mul(syy, bx[0]), A::mul(sxy, by[0])) / det;
      fx.b = A::sub(A::mul(syy, bx[1]), A::mul(sxy, by[1])) / det;
      fx.c = A::sub(A::mul(syy, bx[2]), A::mul(sxy, by[2])) / det;
      fx.d = A::sub(A::mul(syy, bx[3]), A::mul(sxy, by[3])) / det;
      fy.a = A::sub(A::mul(sxx, by[0]), A::mul(sxy, bx[0])) / det;
      fy.b = A::sub(A::mul(sxx, by[1]), A::mul(sxy, bx[1])) / det;
      fy.c = A::sub(A::mul(sxx, by[2]), A::mul(sxy, bx[2])) / det;
      fy.d = A::sub(A::mul(sxx, by[3]), A::mul(sxy, bx[3])) / det;
      dq_store(dq_out, g.nloc, i, fx, fy);
    }
  }
  __syncthreads();
  ktimer_end(ctl, kt_sweep(sweep));
}

// Two lanes per point: lane h owns components {2h, 2h+1} of q, qx, qy and
// loads only its 16-byte halves (the pair of lanes still touches each 32-byte
// sector once per record), which halves the registers per thread and doubles
// the loads in flight.  Both lanes form the geometric sums and det (identical
// values); per-component arithmetic is unchanged, so S = true stays bitwise.
// S = false regroups the defect correction as
//   df = (qn - qi) - 0.5 (dx (qxn - qxi) + dy (qyn - qyi))
// and divides once (det reciprocal).
__device__ __forceinline__ double2 ld2(const double* p) {
  double2 v;
  asm("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void st2(double* p, double2 v) {
  asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

// K = 8: uniform 8-point stencils (offsets i*8): the eight neighbour ids come
// in two 16-byte loads and the neighbour loop is unrolled, so all gathers of a
// point are in flight together instead of one neighbour at a time.
__device__ __forceinline__ int4 ld_i4(const int* p) {
  int4 v;
  asm("ld.global.nc.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

// Global-memory neighbour source of the two-lane sweep: lane h reads its
// halves {2h, 2h+1} of q, qx and qy (bases offset by 2h doubles).
struct GlobalSrc {
  const double* xy;
  const double* q;
  const double* qx;
  const double* qy;
  __device__ __forceinline__ void get(int s, double2& p, double2& qv, double2& x, double2& y) const {
    p = ld2(xy + 2 * s);
    qv = ld2(q + 4 * s);
    x = ld2(qx + 4 * s);
    y = ld2(qy + 4 * s);
  }
};

// Sweep arithmetic of one (point, neighbour) term and of the solve.  S = true:
// the reference's sequence, every product and sum rounded; S = false: the
// same sums with explicit FMAs (fixed contraction, so every kernel that uses
// these helpers produces bitwise the same derivatives).
template <bool S>
__device__ __forceinline__ void sweep_term(double2 pi, double2 qi, double2 qxi, double2 qyi, double2 pn, double2 qn,
                                           double2 qxn, double2 qyn, double& sxx, double& sxy, double& syy,
                                           double& bx0, double& bx1, double& by0, double& by1) {
  const double dx = X::sub(pn.x, pi.x), dy = X::sub(pn.y, pi.y);
  if constexpr (S) {
    sxx = X::add(sxx, X::mul(dx, dx));
    sxy = X::add(sxy, X::mul(dx, dy));
    syy = X::add(syy, X::mul(dy, dy));
    const double df0 = X::sub(corrected<true>(qn.x, qxn.x, qyn.x, dx, dy), corrected<true>(qi.x, qxi.x, qyi.x, dx, dy));
    const double df1 = X::sub(corrected<true>(qn.y, qxn.y, qyn.y, dx, dy), corrected<true>(qi.y, qxi.y, qyi.y, dx, dy));
    bx0 = X::add(bx0, X::mul(dx, df0));
    by0 = X::add(by0, X::mul(dy, df0));
    bx1 = X::add(bx1, X::mul(dx, df1));
    by1 = X::add(by1, X::mul(dy, df1));
  } else {
    sxx = fma(dx, dx, sxx);
    sxy = fma(dx, dy, sxy);
    syy = fma(dy, dy, syy);
    const double df0 = fma(-0.5, fma(dx, __dsub_rn(qxn.x, qxi.x), __dmul_rn(dy, __dsub_rn(qyn.x, qyi.x))),
                           __dsub_rn(qn.x, qi.x));
    const double df1 = fma(-0.5, fma(dx, __dsub_rn(qxn.y, qxi.y), __dmul_rn(dy, __dsub_rn(qyn.y, qyi.y))),
                           __dsub_rn(qn.y, qi.y));
    bx0 = fma(dx, df0, bx0);
    by0 = fma(dy, df0, by0);
    bx1 = fma(dx, df1, bx1);
    by1 = fma(dy, df1, by1);
  }
}

// Solve and store (lane h writes its halves of the qx and qy planes); false
// when the stencil is singular (the caller raises).
template <bool S>
__device__ __forceinline__ bool sweep_solve(double sxx, double sxy, double syy, double bx0, double bx1, double by0,
                                            double by1, double det_tol, D4* __restrict__ dq_out, long long ps, int i,
                                            int h) {
  using A = Ar<S>;
  double det;
  double2 fx, fy;
  if constexpr (S) {
    det = A::sub(A::mul(sxx, syy), A::mul(sxy, sxy));
    if (!(det > det_tol)) return false;
    fx.x = A::sub(A::mul(syy, bx0), A::mul(sxy, by0)) / det;
    fx.y = A::sub(A::mul(syy, bx1), A::mul(sxy, by1)) / det;
    fy.x = A::sub(A::mul(sxx, by0), A::mul(sxy, bx0)) / det;
    fy.y = A::sub(A::mul(sxx, by1), A::mul(sxy, bx1)) / det;
  } else {
    det = fma(sxx, syy, -__dmul_rn(sxy, sxy));
    if (!(det > det_tol)) return false;
    const double r = 1.0 / det;
    fx.x = __dmul_rn(fma(syy, bx0, -__dmul_rn(sxy, by0)), r);
    fx.y = __dmul_rn(fma(syy, bx1, -__dmul_rn(sxy, by1)), r);
    fy.x = __dmul_rn(fma(sxx, by0, -__dmul_rn(sxy, bx0)), r);
    fy.y = __dmul_rn(fma(sxx, by1, -__dmul_rn(sxy, bx1)), r);
  }
  st2(reinterpret_cast<double*>(dq_out + i) + 2 * h, fx);
  st2(reinterpret_cast<double*>(dq_out + ps + i) + 2 * h, fy);
  return true;
}

// One point of the two-lane sweep over a uniform 8-point stencil; nbr[j]
// indexes the source (global id, or a staged slot in tiles.cuh).
template <bool S, class Src>
__device__ __forceinline__ void sweep_point8(const Src& src, int self, const int (&nbr)[8], const Geo& g, int i, int h,
                                             D4* __restrict__ dq_out, const Gas& gas, Ctl* ctl, int sweep) {
  double2 pi, qi, qxi, qyi;
  src.get(self, pi, qi, qxi, qyi);
  double sxx = 0.0, sxy = 0.0, syy = 0.0, bx0 = 0.0, bx1 = 0.0, by0 = 0.0, by1 = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    double2 pn, qn, qxn, qyn;
    src.get(nbr[j], pn, qn, qxn, qyn);
    sweep_term<S>(pi, qi, qxi, qyi, pn, qn, qxn, qyn, sxx, sxy, syy, bx0, bx1, by0, by1);
  }
  if (!sweep_solve<S>(sxx, sxy, syy, bx0, bx1, by0, by1, gas.det_tol, dq_out, g.nloc, i, h) && h == 0)
    raise_err(ctl, err_key(PH_SWEEP, g.part[i], gidx(g, i), 0, 0), 1 + sweep);
}

template <bool S, int MB, int K = 0, int NT = 256>
__global__ void __launch_bounds__(NT, MB) k_sweep2(Geo g, const D4* __restrict__ q,
                                                    const D4* __restrict__ dq_in, D4* __restrict__ dq_out,
                                                    Gas gas, Ctl* ctl, unsigned long long* iter_t0, int sweep) {
  pdl_enter();
  __shared__ int s_skip;
  ktimer_begin(ctl, kt_sweep(sweep));
  if (threadIdx.x == 0) s_skip = skip_stage(ctl, 1 + sweep);
  __syncthreads();
  const int h = threadIdx.x & 1;
  const GlobalSrc src{reinterpret_cast<const double*>(g.xy), reinterpret_cast<const double*>(q) + 2 * h,
                      reinterpret_cast<const double*>(dq_in) + 2 * h,
                      reinterpret_cast<const double*>(dq_in + g.nloc) + 2 * h};
  const long long n2 = 2ll * visit_count(g);
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  for (; !s_skip && t < n2; t += stride) {
    const int i = visit_point(g, static_cast<int>(t >> 1));
    if constexpr (K == 8) {
      // ids in two 16-byte loads (loading them a point ahead measured 2% slower)
      const int4 na0 = ld_i4(g.nbr + 8ll * i), na1 = ld_i4(g.nbr + 8ll * i + 4);
      const int nbr[8] = {na0.x, na0.y, na0.z, na0.w, na1.x, na1.y, na1.z, na1.w};
      sweep_point8<S>(src, i, nbr, g, i, h, dq_out, gas, ctl, sweep);
    } else {
      double2 pi, qi, qxi, qyi;
      src.get(i, pi, qi, qxi, qyi);
      double sxx = 0.0, sxy = 0.0, syy = 0.0, bx0 = 0.0, bx1 = 0.0, by0 = 0.0, by1 = 0.0;
      int e0, k;
      stencil_of(g, i, e0, k);
      for (int j = 0; j < k; ++j) {
        double2 pn, qn, qxn, qyn;
        src.get(g.nbr[e0 + j], pn, qn, qxn, qyn);
        sweep_term<S>(pi, qi, qxi, qyi, pn, qn, qxn, qyn, sxx, sxy, syy, bx0, bx1, by0, by1);
      }
      if (!sweep_solve<S>(sxx, sxy, syy, bx0, bx1, by0, by1, gas.det_tol, dq_out, g.nloc, i, h) && h == 0)
        raise_err(ctl, err_key(PH_SWEEP, g.part[i], gidx(g, i), 0, 0), 1 + sweep);
    }
  }
  __syncthreads();
  ktimer_end(ctl, kt_sweep(sweep));
}

// ---------------------------------------------------------------------------
// Flux residual.  W lanes cooperate on one point, one lane per stencil
// neighbour (pair): each pair's two reconstructions q~ -> prim and split
// fluxes are computed once and shared by its x- and y-direction terms
// (bitwise neutral: the reference recomputes identical values per direction).
// Lanes then transpose through shared memory so each least-squares
// accumulator is summed in ascending neighbour order, exactly as
// directional_term does (kernels.cpp:37-64).  The residual is written to
// `res`; the per-point update runs in k_update (one thread per point).
struct PairRec {
  double dx, dy;
  double dg[4][4];  // Delta G for Gx+, Gx-, Gy+, Gy- (only member directions valid)
};

struct FluxArgs {
  Geo g;
  Gas gas;
  const D4* q;    // q of this iteration
  const D4* dq;   // published derivatives
  D4* res;        // residual out (accumulated into when first == 0)
  Ctl* ctl;
  unsigned long long* iter_t0;  // per-iteration start stamps (first kernel only)
  int kcap;       // shared-memory stencil capacity per point
  int stride;     // doubles per point in shared memory (bank-conflict padding)
  int mask;       // directions to evaluate (bit d: Gx+, Gx-, Gy+, Gy-)
  int first;      // zero the accumulator before adding
};


__host__ __device__ constexpr int flux_points_per_block(int W) { return W >= 32 ? 8 : (W >= 16 ? 16 : 32); }

// Pair-record stride per point, padded so consecutive points start 16 banks
// apart (two sub-warps per 32-bank wavefront in phase B).
__host__ __device__ inline int flux_stride(int kcap) {
  int s = kcap * static_cast<int>(sizeof(PairRec) / 8);
  while (s % 16 != 8) ++s;
  return s;
}

// Phase A is convergent: every lane of a warp runs the same instruction
// stream (inactive lanes evaluate their own point with zero offsets and store
// nothing), so constant tables go through the uniform datapath and no lane
// waits on another's branch.  Each pair evaluates one x and one y split flux,
// with the sign chosen per lane (the half stencil the neighbour falls in); a
// zero offset also needs the other sign, handled in a rarely taken
// warp-uniform branch.
template <int W, bool S, int MB>
__global__ void __launch_bounds__(W * flux_points_per_block(W), MB) k_flux(FluxArgs a) {
  pdl_enter();
  constexpr int P = flux_points_per_block(W);
  constexpr int NOWN = W >= 16 ? 16 : W;        // lanes owning accumulators
  constexpr int NC = 16 / NOWN;                 // components per owning lane
  constexpr unsigned kFull = 0xFFFFFFFFu;
  using A = Ar<S>;
  extern __shared__ double smem[];
  double* terms = smem + static_cast<size_t>(P) * a.stride;  // [P][16]
  __shared__ int s_skip;

  ktimer_begin(a.ctl, KT_FLUX);
  if (threadIdx.x == 0) s_skip = skip_stage(a.ctl, sub_flux(a.ctl));
  __syncthreads();
  const int lane = threadIdx.x % W;
  const int slot = threadIdx.x / W;
  const Geo& g = a.g;
  PairRec* my = reinterpret_cast<PairRec*>(smem + static_cast<size_t>(slot) * a.stride);
  const int groups = (g.n + P - 1) / P;
  // Persistent blocks: one resident block per slot walks groups of P points,
  // amortising the start-up latency and the timer atomics.
  for (int grp = blockIdx.x; !s_skip && grp < groups; grp += gridDim.x) {
    const int i = grp * P + slot;
    const int ic = i < g.n ? i : g.n - 1;  // clamped for loads
    const bool live = i < g.n && g.kind[ic] != KIND_OUTER;
    int k = 0, e0 = 0;
    if (live) stencil_of(g, i, e0, k);
    const int kwarp = __reduce_max_sync(kFull, k);

    // ---- phase A: one lane per (point, neighbour) pair ----
    const double2 pi = g.xy[ic];
    const D4 qi = ld4(a.q + ic);
    D4 qxi, qyi;
    dq_load(a.dq, g.nloc, ic, qxi, qyi);
    for (int jb = 0; jb < kwarp; jb += W) {
      const int j = jb + lane;
      const bool act = live && j < k;
      const int nb = act ? g.nbr[e0 + j] : ic;
      const double2 pn = g.xy[nb];
      const double dx = X::sub(pn.x, pi.x), dy = X::sub(pn.y, pi.y);
      const D4 qn = ld4(a.q + nb);
      D4 qxn, qyn;
      dq_load(a.dq, g.nloc, nb, qxn, qyn);
      double ti[4], tn[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        ti[c] = corrected<S>(comp(qi, c), comp(qxi, c), comp(qyi, c), dx, dy);
        tn[c] = corrected<S>(comp(qn, c), comp(qxn, c), comp(qyn, c), dx, dy);
      }
      bool ok = ti[3] < 0.0 && tn[3] < 0.0;
      if (!ok) {  // q3 >= 0 has no state: evaluate a dummy one, store nothing
        ti[3] = -1.0;
        tn[3] = -1.0;
      }
      FluxState fi, fn;
      ok = reconstruct2<S>(ti, tn, a.gas, fi, fn) && ok;
      if (act && !ok) raise_err(a.ctl, flux_key(a.ctl, g.part[i], gidx(g, i), dx <= 0.0 ? 0u : 1u, j), sub_flux(a.ctl));
      AxisTerms at[4];
      axis_terms4<S>(fi, fn, at);
      const bool store = act && ok;
      const bool xplus = dx <= 0.0, yplus = dy <= 0.0;
      PairRec& r = my[j < a.kcap ? j : 0];
      double gi[4], gn[4];
      split_flux<S>(fi, at[0], 0, !xplus, gi);
      split_flux<S>(fn, at[1], 0, !xplus, gn);
      if (store) {
        r.dx = dx;
        r.dy = dy;
#pragma unroll
        for (int c = 0; c < 4; ++c) r.dg[xplus ? 0 : 1][c] = X::sub(gn[c], gi[c]);
      }
      split_flux<S>(fi, at[2], 1, !yplus, gi);
      split_flux<S>(fn, at[3], 1, !yplus, gn);
      if (store) {
#pragma unroll
        for (int c = 0; c < 4; ++c) r.dg[yplus ? 2 : 3][c] = X::sub(gn[c], gi[c]);
      }
      // a zero offset belongs to both half stencils: add the minus direction
      if (__any_sync(kFull, store && (dx == 0.0 || dy == 0.0))) {
        if (store && dx == 0.0) {
          split_flux<S>(fi, at[0], 0, true, gi);
          split_flux<S>(fn, at[1], 0, true, gn);
#pragma unroll
          for (int c = 0; c < 4; ++c) r.dg[1][c] = X::sub(gn[c], gi[c]);
        }
        if (store && dy == 0.0) {
          split_flux<S>(fi, at[2], 1, true, gi);
          split_flux<S>(fn, at[3], 1, true, gn);
#pragma unroll
          for (int c = 0; c < 4; ++c) r.dg[3][c] = X::sub(gn[c], gi[c]);
        }
      }
    }
    __syncthreads();

    // ---- phase B: ordered least-squares sums + 2x2 solve per direction ----
    if (live && lane < NOWN) {
      const int d = lane / (4 / NC);                // direction owned
      const int c0 = (lane % (4 / NC)) * NC;        // first component owned
      if (a.mask & (1 << d)) {
        double sxx = 0.0, sxy = 0.0, syy = 0.0, bx[NC], by[NC];
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) bx[cc] = by[cc] = 0.0;
        for (int j = 0; j < k; ++j) {
          const double dx = my[j].dx, dy = my[j].dy;
          const double dd = d < 2 ? dx : dy;
          const bool member = (d & 1) ? dd >= 0.0 : dd <= 0.0;
          if (!member) continue;
          sxx = A::add(sxx, A::mul(dx, dx));
          sxy = A::add(sxy, A::mul(dx, dy));
          syy = A::add(syy, A::mul(dy, dy));
#pragma unroll
          for (int cc = 0; cc < NC; ++cc) {
            const double df = my[j].dg[d][c0 + cc];
            bx[cc] = A::add(bx[cc], A::mul(dx, df));
            by[cc] = A::add(by[cc], A::mul(dy, df));
          }
        }
        const double det = A::sub(A::mul(sxx, syy), A::mul(sxy, sxy));
        if (!(det > a.gas.det_tol)) {
          raise_err(a.ctl, flux_key(a.ctl, g.part[i], gidx(g, i), d, kSolveSlot), sub_flux(a.ctl));
        } else {
#pragma unroll
          for (int cc = 0; cc < NC; ++cc) {
            const double t = d < 2 ? A::sub(A::mul(syy, bx[cc]), A::mul(sxy, by[cc])) / det
                                   : A::sub(A::mul(sxx, by[cc]), A::mul(sxy, bx[cc])) / det;
            terms[slot * 16 + d * 4 + c0 + cc] = t;
          }
        }
      }
    }
    __syncthreads();

    // ---- residual: zero (or accumulator), then Gx+, Gx-, Gy+, Gy- in order
    //      (kernels.cpp:124-138); one lane per (point, component) ----
    if (threadIdx.x < 4 * P) {
      const int sl = threadIdx.x >> 2, c = threadIdx.x & 3;
      const int ip = grp * P + sl;
      if (ip < g.n && g.kind[ip] != KIND_OUTER) {
        double* rp = reinterpret_cast<double*>(a.res + ip) + c;
        double acc = a.first ? 0.0 : *rp;
#pragma unroll
        for (int d = 0; d < 4; ++d)
          if (a.mask & (1 << d)) acc = X::add(acc, terms[sl * 16 + d * 4 + c]);
        *rp = acc;
      }
    }
    __syncthreads();  // terms/records are reused by the next group
  }
  __syncthreads();
  ktimer_end(a.ctl, KT_FLUX);
}

// ---------------------------------------------------------------------------
// Flux residual, fp_mode fast: least-squares weights instead of per-iteration
// solves.  Each direction's derivative (kernels.cpp:37-64)
//   D_d = (syy_d bx_d - sxy_d by_d) / det_d,   bx_d = sum_{j in d} dx_j dG_j, ...
// (y directions: (sxx_d by_d - sxy_d bx_d) / det_d) is linear in the pair
// differences dG_j, so D_d = sum_{j in d} w_dj dG_j with geometry-only weights
//   w_dj = (syy_d dx_j - sxy_d dy_j) / det_d   (x)   (sxx_d dy_j - sxy_d dx_j) / det_d   (y).
// k_flux_weights computes them once per run; the residual sum_d D_d becomes
// one dot product per pair and a shuffle reduction over the pair lanes — no
// shared-memory transpose, no block barriers, no divisions per iteration.
// Per pair e: w1[e] = (weight in the pair's x direction: Gx+ if dx <= 0 else
// Gx-, weight in its y direction: Gy+ if dy <= 0 else Gy-); w2[e] = (weight in
// Gx- when dx == 0, in Gy- when dy == 0) — a zero offset belongs to both
// halves (only allocated when such pairs exist).  det is formed with the
// reference's exact operation sequence, so the singular-stencil decision
// `!(det > det_tol)` is bitwise the reference's; sing[i] holds the first
// singular direction of point i (0xFF: none), raised by the flux kernel.
// psign[e] (first order): bit 0 = the pair's x half is Gx- (dx > 0), bit 1 =
// its y half is Gy- (dy > 0), bit 2 = a zero offset (both halves).
__global__ void k_flux_weights(Geo g, double det_tol, double2* w1, double2* w2, std::uint8_t* sing,
                               std::uint8_t* psign) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.n) return;
  int e0, k;
  stencil_of(g, i, e0, k);
  if (g.kind[i] == KIND_OUTER) {
    if (w1)
      for (int j = 0; j < k; ++j) w1[e0 + j] = make_double2(0.0, 0.0);
    if (psign)
      for (int j = 0; j < k; ++j) psign[e0 + j] = 0;
    if (sing) sing[i] = 0xFF;
    return;
  }
  const double2 pi = g.xy[i];
  double sxx[4] = {0.0, 0.0, 0.0, 0.0}, sxy[4] = {0.0, 0.0, 0.0, 0.0}, syy[4] = {0.0, 0.0, 0.0, 0.0};
  for (int j = 0; j < k; ++j) {
    const double2 pn = g.xy[g.nbr[e0 + j]];
    const double dx = X::sub(pn.x, pi.x), dy = X::sub(pn.y, pi.y);
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const double dd = d < 2 ? dx : dy;
      if (!((d & 1) ? dd >= 0.0 : dd <= 0.0)) continue;
      sxx[d] = X::add(sxx[d], X::mul(dx, dx));
      sxy[d] = X::add(sxy[d], X::mul(dx, dy));
      syy[d] = X::add(syy[d], X::mul(dy, dy));
    }
  }
  double rdet[4];
  int first_sing = 0xFF;
#pragma unroll
  for (int d = 3; d >= 0; --d) {
    const double det = X::sub(X::mul(sxx[d], syy[d]), X::mul(sxy[d], sxy[d]));
    const bool ok = det > det_tol;
    if (!ok) first_sing = d;
    rdet[d] = ok ? 1.0 / det : 0.0;
  }
  sing[i] = static_cast<std::uint8_t>(first_sing);
  auto wt = [&](int d, double dx, double dy) {
    return d < 2 ? (syy[d] * dx - sxy[d] * dy) * rdet[d] : (sxx[d] * dy - sxy[d] * dx) * rdet[d];
  };
  for (int j = 0; j < k; ++j) {
    const double2 pn = g.xy[g.nbr[e0 + j]];
    const double dx = X::sub(pn.x, pi.x), dy = X::sub(pn.y, pi.y);
    w1[e0 + j] = make_double2(wt(dx <= 0.0 ? 0 : 1, dx, dy), wt(dy <= 0.0 ? 2 : 3, dx, dy));
    if (psign)
      psign[e0 + j] = static_cast<std::uint8_t>((dx <= 0.0 ? 0 : 1) | (dy <= 0.0 ? 0 : 2) |
                                                ((dx == 0.0 || dy == 0.0) ? 4 : 0));
    if (w2) w2[e0 + j] = make_double2(dx == 0.0 ? wt(1, dx, dy) : 0.0, dy == 0.0 ? wt(3, dx, dy) : 0.0);
  }
}

// One (point i, neighbour position j) pair of the fast flux residual: both
// reconstructions, the x and y split fluxes of each side (the pair's half
// stencils), acc += w . dG.  Warp-convergent (inactive lanes evaluate their
// own point with zero offsets and add nothing).
// DEFER: the rare branches (erf argument above 1.5, exponential range, an
// invalid state: act && !ok) leave the instruction stream; the lane sets redo
// instead and the caller has the point recomputed by k_flux_redo, which runs
// this function without DEFER (same arithmetic, so the same bits).
template <int HP = -1, bool DEFER = false>
__device__ __forceinline__ void flux_pair_fast(const FluxArgs& a, int i, int j, bool act, double2 pi,
                                               const D4& qi, const D4& qxi, const D4& qyi, double2 pn,
                                               const D4& qn, const D4& qxn, const D4& qyn, double2 w,
                                               const double2* w2e, double (&acc)[4], bool* redo = nullptr) {
  constexpr unsigned kFull = 0xFFFFFFFFu;
  const Geo& g = a.g;
  const double dx = X::sub(pn.x, pi.x), dy = X::sub(pn.y, pi.y);
  // q~ = q - (dx/2) qx - (dy/2) qy as two FMAs per component (the reference's
  // q - 0.5 (dx qx + dy qy) regrouped; a uniform field stays exact)
  const double hdx = -0.5 * dx, hdy = -0.5 * dy;
  double ti[4], tn[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    ti[c] = fma(hdx, comp(qxi, c), fma(hdy, comp(qyi, c), comp(qi, c)));
    tn[c] = fma(hdx, comp(qxn, c), fma(hdy, comp(qyn, c), comp(qn, c)));
  }
  bool ok = ti[3] < 0.0 && tn[3] < 0.0;
  if (!ok) {  // q3 >= 0 has no state: evaluate a dummy one, add nothing
    ti[3] = -1.0;
    tn[3] = -1.0;
  }
  FluxState fi, fn;
  bool rd = false;
  ok = reconstruct2<false, HP, DEFER, true>(ti, tn, a.gas, fi, fn, rd) && ok;
  if constexpr (DEFER) rd |= act && !ok;
  else if (act && !ok) raise_err(a.ctl, flux_key(a.ctl, g.part[i], gidx(g, i), dx <= 0.0 ? 0u : 1u, j), sub_flux(a.ctl));
  AxisTerms at[4];
  axis_terms4<false, DEFER>(fi, fn, at, rd);
  if constexpr (DEFER) *redo |= rd;
  const bool store = act && ok;
  const double wx = store ? w.x : 0.0, wy = store ? w.y : 0.0;
  // dG = gn - gi is an explicitly rounded subtraction: a contracted
  // fma(rho_n, x_n, -gi) would leave ~1 ulp where the states are equal
  // (the free stream must stay an exact fixed point).
  double gi[4], gn[4];
  const double epi = fi.e, kki = -0.5 * fi.p;  // fi.e = rhoE + p here; kk: -p/2 of split_flux_fast
  const double epn = fn.e, kkn = -0.5 * fn.p;
  split_flux_fast<0>(fi, at[0], !(dx <= 0.0), epi, kki, gi);
  split_flux_fast<0>(fn, at[1], !(dx <= 0.0), epn, kkn, gn);
#pragma unroll
  for (int c = 0; c < 4; ++c) acc[c] = fma(wx, X::sub(gn[c], gi[c]), acc[c]);
  split_flux_fast<1>(fi, at[2], !(dy <= 0.0), epi, kki, gi);
  split_flux_fast<1>(fn, at[3], !(dy <= 0.0), epn, kkn, gn);
#pragma unroll
  for (int c = 0; c < 4; ++c) acc[c] = fma(wy, X::sub(gn[c], gi[c]), acc[c]);
  // a zero offset belongs to both half stencils: add the minus direction
  // (w2e null: the stencil table has no zero offset — k_min_dist's count)
  if (w2e != nullptr && __any_sync(kFull, store && (dx == 0.0 || dy == 0.0))) {
    const double2 v = (store && (dx == 0.0 || dy == 0.0)) ? *w2e : make_double2(0.0, 0.0);
    split_flux_fast<0>(fi, at[0], true, epi, kki, gi);
    split_flux_fast<0>(fn, at[1], true, epn, kkn, gn);
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[c] = fma(v.x, X::sub(gn[c], gi[c]), acc[c]);
    split_flux_fast<1>(fi, at[2], true, epi, kki, gi);
    split_flux_fast<1>(fn, at[3], true, epn, kkn, gn);
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[c] = fma(v.y, X::sub(gn[c], gi[c]), acc[c]);
  }
}

// Sum over the 8 pair lanes of a point (xor shuffles stay inside the group),
// as a transposing reduction: after it, lanes 2c and 2c+1 of the group hold
// component c of the sum (4 double shuffles instead of 12).
__device__ __forceinline__ double reduce8(const double (&acc)[4], int lane) {
  constexpr unsigned kFull = 0xFFFFFFFFu;
  const bool hi2 = lane & 4, hi1 = lane & 2;
  // xor 4: keep components {0,1} (lanes 0-3) or {2,3} (lanes 4-7)
  const double s0 = hi2 ? acc[0] : acc[2], s1 = hi2 ? acc[1] : acc[3];
  const double k0 = hi2 ? acc[2] : acc[0], k1 = hi2 ? acc[3] : acc[1];
  const double a0 = X::add(k0, __shfl_xor_sync(kFull, s0, 4));
  const double a1 = X::add(k1, __shfl_xor_sync(kFull, s1, 4));
  // xor 2: keep the first (lanes x0x) or second (lanes x1x) of the pair
  const double b = X::add(hi1 ? a1 : a0, __shfl_xor_sync(kFull, hi1 ? a0 : a1, 2));
  return X::add(b, __shfl_xor_sync(kFull, b, 1));
}

// Residual of point i from the transposed reduction: lane 2c writes component c.
__device__ __forceinline__ void store_res8(D4* res, int i, double v, int lane) {
  if (!(lane & 1)) reinterpret_cast<double*>(res + i)[lane >> 1] = v;
}

// Eight lanes per point (one per stencil neighbour, looping for k > 8), four
// points per warp, warps independent (persistent grid-stride over groups of
// 4 points).  Any stencil size.
template <int MB>
__global__ void __launch_bounds__(256, MB) k_flux_w(FluxArgs a, const double2* __restrict__ w1,
                                                    const double2* __restrict__ w2,
                                                    const std::uint8_t* __restrict__ sing) {
  pdl_enter();
  constexpr unsigned kFull = 0xFFFFFFFFu;
  __shared__ int s_skip;
  ktimer_begin(a.ctl, KT_FLUX);
  if (threadIdx.x == 0) s_skip = skip_stage(a.ctl, sub_flux(a.ctl));
  __syncthreads();
  const int lane = threadIdx.x & 7;
  const int sub = (threadIdx.x >> 3) & 3;
  const Geo& g = a.g;
  const int groups = (g.n + 3) >> 2;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int grp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; !s_skip && grp < groups; grp += nwarps) {
    const int i = grp * 4 + sub;
    const int ic = i < g.n ? i : g.n - 1;  // clamped for loads
    const bool live = i < g.n && g.kind[ic] != KIND_OUTER;
    int k = 0, e0 = 0;
    if (live) stencil_of(g, i, e0, k);
    const int kwarp = __reduce_max_sync(kFull, k);
    if (live && lane == 0) {
      const unsigned sd = sing[i];
      if (sd != 0xFFu) raise_err(a.ctl, flux_key(a.ctl, g.part[i], gidx(g, i), sd, kSolveSlot), sub_flux(a.ctl));
    }
    const double2 pi = g.xy[ic];
    const D4 qi = ld4(a.q + ic);
    D4 qxi, qyi;
    dq_load(a.dq, g.nloc, ic, qxi, qyi);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int jb = 0; jb < kwarp; jb += 8) {
      const int j = jb + lane;
      const bool act = live && j < k;
      const int nb = act ? g.nbr[e0 + j] : ic;
      const double2 w = act ? w1[e0 + j] : make_double2(0.0, 0.0);
      const D4 qn = ld4(a.q + nb);
      D4 qxn, qyn;
      dq_load(a.dq, g.nloc, nb, qxn, qyn);
      flux_pair_fast(a, i, j, act, pi, qi, qxi, qyi, g.xy[nb], qn, qxn, qyn, w, w2 ? w2 + (e0 + j) : nullptr,
                     acc);
    }
    const double r = reduce8(acc, lane);
    if (live) store_res8(a.res, i, r, lane);
  }
  __syncthreads();
  ktimer_end(a.ctl, KT_FLUX);
}

// ---- first order, fp_mode fast: without derivatives the pair states are the
// points' own states (q~ = q), so each point's split fluxes are evaluated once
// (k_point_flux: Gx+, Gx-, Gy+, Gy- of every owned and halo point) and the
// flux kernel only gathers them: per pair dG = G_n - G_i of the pair's x and y
// half-stencil signs, weighted and reduced as in k_flux_w.
struct PointFlux {
  D4 g[4];  // Gx+, Gx-, Gy+, Gy-
};

__global__ void __launch_bounds__(256) k_point_flux(int n_loc, const D4* __restrict__ q, Gas gas,
                                                    PointFlux* __restrict__ pf, std::uint8_t* __restrict__ valid,
                                                    const Ctl* ctl) {
  pdl_enter();
  ktimer_begin(const_cast<Ctl*>(ctl), KT_FLUX);  // timed with k_flux1 as one flux phase
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_loc || skip_stage(ctl, sub_flux(ctl))) return;
  const D4 qi = ld4(q + i);
  double t[4] = {qi.a, qi.b, qi.c, qi.d};
  bool ok = t[3] < 0.0;
  if (!ok) t[3] = -1.0;
  FluxState f;
  ok = reconstruct1_fast(t, gas, f) && ok;
  AxisTerms at[2];
  axis_terms2_fast(f, at);
  const double ep = f.e, kk = -0.5 * f.p;  // f.e = rhoE + p; kk: -p/2 of split_flux_fast
  double gv[4];
  split_flux_fast<0>(f, at[0], false, ep, kk, gv);
  st4(&pf[i].g[0], D4{gv[0], gv[1], gv[2], gv[3]});
  split_flux_fast<0>(f, at[0], true, ep, kk, gv);
  st4(&pf[i].g[1], D4{gv[0], gv[1], gv[2], gv[3]});
  split_flux_fast<1>(f, at[1], false, ep, kk, gv);
  st4(&pf[i].g[2], D4{gv[0], gv[1], gv[2], gv[3]});
  split_flux_fast<1>(f, at[1], true, ep, kk, gv);
  st4(&pf[i].g[3], D4{gv[0], gv[1], gv[2], gv[3]});
  valid[i] = ok ? 1 : 0;
}

template <int MB>
__global__ void __launch_bounds__(256, MB) k_flux1(FluxArgs a, const PointFlux* __restrict__ pf,
                                                   const std::uint8_t* __restrict__ valid,
                                                   const double2* __restrict__ w1, const double2* __restrict__ w2,
                                                   const std::uint8_t* __restrict__ sing,
                                                   const std::uint8_t* __restrict__ psign) {
  pdl_enter();
  constexpr unsigned kFull = 0xFFFFFFFFu;
  __shared__ int s_skip;
  ktimer_begin(a.ctl, KT_FLUX);
  if (threadIdx.x == 0) s_skip = skip_stage(a.ctl, sub_flux(a.ctl));
  __syncthreads();
  const int lane = threadIdx.x & 7;
  const int sub = (threadIdx.x >> 3) & 3;
  const Geo& g = a.g;
  const int groups = (g.n + 3) >> 2;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  int grp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  // stencil indices of the next group are loaded one group ahead (k <= 8)
  auto fetch = [&](int gp, int& i, int& kind, int& k, int& e, int& nb, int& ps) {
    i = gp * 4 + sub;
    const int ic = i < g.n ? i : g.n - 1;
    kind = g.kind[ic];
    int e0 = 0;
    stencil_of(g, ic, e0, k);
    e = e0 + lane;
    const bool in = i < g.n && lane < k;
    nb = in ? g.nbr[e] : ic;
    ps = in ? psign[e] : 0;
  };
  int ci = 0, ckind = 0, ck_ = 0, ce = 0, cnb = 0, cps = 0;
  if (!s_skip && grp < groups) fetch(grp, ci, ckind, ck_, ce, cnb, cps);
  for (; !s_skip && grp < groups; grp += nwarps) {
    const int i = ci, e = ce, ps = cps;
    const int ic = i < g.n ? i : g.n - 1;
    const bool live = i < g.n && ckind != KIND_OUTER;
    const bool act = live && lane < ck_;
    const int nb = act ? cnb : ic;
    if (grp + nwarps < groups) fetch(grp + nwarps, ci, ckind, ck_, ce, cnb, cps);
    const int sx = ps & 1, sy = 2 + ((ps >> 1) & 1);
    const double2 w = act ? w1[e] : make_double2(0.0, 0.0);
    const D4 gix = ld4(&pf[ic].g[sx]), giy = ld4(&pf[ic].g[sy]);
    const D4 gnx = ld4(&pf[nb].g[sx]), gny = ld4(&pf[nb].g[sy]);
    const bool ok = valid[ic] != 0 && valid[nb] != 0;
    if (live && lane == 0) {
      const unsigned sd = sing[i];
      if (sd != 0xFFu) raise_err(a.ctl, flux_key(a.ctl, g.part[i], gidx(g, i), sd, kSolveSlot), sub_flux(a.ctl));
    }
    if (act && !ok) raise_err(a.ctl, flux_key(a.ctl, g.part[i], gidx(g, i), static_cast<unsigned>(sx), lane),
                              sub_flux(a.ctl));
    const bool store = act && ok;
    const double wx = store ? w.x : 0.0, wy = store ? w.y : 0.0;
    double acc[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[c] = fma(wx, X::sub(comp(gnx, c), comp(gix, c)), 0.0);
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[c] = fma(wy, X::sub(comp(gny, c), comp(giy, c)), acc[c]);
    // a zero offset belongs to both half stencils: add the minus direction
    const bool zero = store && (ps & 4);
    if (__any_sync(kFull, zero)) {
      const double2 v = zero ? w2[e] : make_double2(0.0, 0.0);
      const D4 ai = ld4(&pf[ic].g[1]), an = ld4(&pf[nb].g[1]);
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[c] = fma(v.x, X::sub(comp(an, c), comp(ai, c)), acc[c]);
      const D4 bi = ld4(&pf[ic].g[3]), bn = ld4(&pf[nb].g[3]);
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[c] = fma(v.y, X::sub(comp(bn, c), comp(bi, c)), acc[c]);
    }
    const double r = reduce8(acc, lane);
    if (live) store_res8(a.res, i, r, lane);
  }
  __syncthreads();
  ktimer_end(a.ctl, KT_FLUX);
}

// ---- staged variant (stencils of at most 8): each warp copies the NEXT group's
// gathers (neighbour xy, q, qx, qy, weights; own point records) into its
// shared-memory stage with cp.async while it computes the current group, and
// loads the stencil indices two groups ahead, so no global-memory latency is
// exposed inside the loop.  Stage layout is field-major (16-byte chunks per
// lane) so each LDS.128 of a warp is conflict-free.
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

constexpr int kFluxStageChunks = 8;                                  // per lane: xy, w, q(2), qx(2), qy(2)
constexpr int kFluxStageBytes = kFluxStageChunks * 32 * 16 + 4 * 7 * 16;  // + 4 own records of 7 chunks
constexpr int kFluxWarps = 8;                                       // 256 threads

struct StageIdx {  // per lane, one group
  int i, ic, nb, e, sing;
  bool live, act;
};
// Raw loads of a group's indices, issued two groups ahead; the predicates are
// formed only when the group is staged (stage_index), so nothing waits on them.
struct StageRaw {
  int i, kind, nbr, e, k, sing;
};

// U8: uniform 8-point stencils and every owned point visited (no subset
// list): the stencil offsets and the visit list are compile-time, so the
// loop keeps fewer kernel parameters live.
template <bool U8 = false, bool DEFER = false>
__device__ __forceinline__ StageRaw stage_load(const Geo& g, const std::uint8_t* sing, int grp, int lane,
                                               int sub) {
  StageRaw r;
  r.i = U8 ? grp * 4 + sub : visit_point(g, grp * 4 + sub);
  const int ic = r.i < g.n ? r.i : g.n - 1;
  r.kind = g.kind[ic];
  // first singular split direction (k_flux_weights); DEFER: flagged for the redo once per domain
  r.sing = (!DEFER && lane == 0) ? sing[ic] : 0xFF;
  int e0 = 0, k = 0;
  if constexpr (U8) {
    e0 = 8 * ic;
    k = 8;
  } else {
    stencil_of(g, ic, e0, k);
  }
  r.e = e0 + lane;
  r.k = k;
  r.nbr = (r.i < g.n && lane < k) ? g.nbr[r.e] : ic;
  return r;
}

__device__ __forceinline__ StageIdx stage_index(const Geo& g, const StageRaw& r, int lane) {
  StageIdx x;
  x.i = r.i;
  x.ic = r.i < g.n ? r.i : g.n - 1;
  x.live = r.i < g.n && r.kind != KIND_OUTER;
  x.act = x.live && lane < r.k;
  x.e = r.e;
  x.nb = x.act ? r.nbr : x.ic;
  x.sing = r.sing;
  return x;
}

// Lanes 0-6 of a point's lane group stage its own record: xy, q (2 halves),
// qx01 qy01 qx23 qy23 — chunk `lane` is at own_base + ic * own_stride.
struct OwnSrc {
  const char* base;
  long long stride;
};
__device__ __forceinline__ OwnSrc own_src(const FluxArgs& a, int lane) {
  const int c = lane - 3;
  if (lane == 0) return OwnSrc{reinterpret_cast<const char*>(a.g.xy), 16};
  if (lane < 3) return OwnSrc{reinterpret_cast<const char*>(a.q) + (lane - 1) * 16, 32};
  return OwnSrc{reinterpret_cast<const char*>(a.dq + ((c & 1) ? a.g.nloc : 0)) + (c >> 1) * 16, 32};
}

__device__ __forceinline__ void stage_issue(const FluxArgs& a, const double2* w1, const StageIdx& x,
                                            char* st, int lane32, int lane, int sub, const OwnSrc& own) {
  const Geo& g = a.g;
  char* f = st + lane32 * 16;
  cp_async16(f + 0 * 512, g.xy + x.nb, true);
  cp_async16(f + 1 * 512, w1 + x.e, x.act);  // zero-filled for inactive lanes
  const char* qn = reinterpret_cast<const char*>(a.q + x.nb);
  const char* xn = reinterpret_cast<const char*>(a.dq + x.nb);           // qx plane
  const char* yn = reinterpret_cast<const char*>(a.dq + g.nloc + x.nb);  // qy plane
  cp_async16(f + 2 * 512, qn, true);
  cp_async16(f + 3 * 512, qn + 16, true);
  cp_async16(f + 4 * 512, xn, true);
  cp_async16(f + 5 * 512, yn, true);
  cp_async16(f + 6 * 512, xn + 16, true);
  cp_async16(f + 7 * 512, yn + 16, true);
  if (lane < 7) cp_async16(st + kFluxStageChunks * 512 + (sub * 7 + lane) * 16, own.base + x.ic * own.stride, true);
}

// Rare-path deferral (DEFER): a lane whose pair took a rare path flags its
// point (bit i of the bit set); k_flux_redo recomputes the flagged points with
// the fallbacks in place and clears the bits.  The singular-split check is not
// made (a domain with a live singular point — a run that fails in its first
// flux pass — runs without DEFER, k_flux_any_sing).  bits: kRedoWordsPer *
// ceil(n / kRedoPointsPer) zero-initialised words (the redo scans uint4 per lane).
constexpr int kRedoPointsPer = 4096;  // points per warp step of the redo scan
constexpr int kRedoWordsPer = kRedoPointsPer / 32;
struct FluxRedo {
  unsigned* bits;
};

template <int MB, int NW = kFluxWarps, int HP = -1, bool U8 = false, bool DEFER = false>
__global__ void __launch_bounds__(NW * 32, MB) k_flux_ws(FluxArgs a, const double2* __restrict__ w1,
                                                     const double2* __restrict__ w2,
                                                     const std::uint8_t* __restrict__ sing, FluxRedo rd) {
  pdl_enter();
  extern __shared__ __align__(16) char fsm[];
  __shared__ int s_skip;
  ktimer_begin(a.ctl, KT_FLUX);
  if (threadIdx.x == 0) s_skip = skip_stage(a.ctl, sub_flux(a.ctl));
  __syncthreads();
  const int lane32 = threadIdx.x & 31;
  const int lane = threadIdx.x & 7;
  const int sub = lane32 >> 3;
  const int warp = threadIdx.x >> 5;
  char* const stage0 = fsm + (2 * warp) * kFluxStageBytes;  // stage b at stage0 + b * kFluxStageBytes
  const Geo& g = a.g;
  const OwnSrc own = own_src(a, lane);
  const int groups = ((U8 ? g.n : visit_count(g)) + 3) >> 2;
  const int nwarps = gridDim.x * NW;
  int grp = blockIdx.x * NW + warp;
  if (!s_skip && grp < groups) {
    StageIdx cur = stage_index(g, stage_load<U8, DEFER>(g, sing, grp, lane, sub), lane);
    stage_issue(a, w1, cur, stage0, lane32, lane, sub, own);
    cp_async_commit();
    StageRaw nxt = stage_load<U8, DEFER>(g, sing, grp + nwarps < groups ? grp + nwarps : grp, lane, sub);
    int buf = 0;
    for (; grp < groups; grp += nwarps, buf ^= 1) {
      const bool more = grp + nwarps < groups;
      const StageIdx nx = stage_index(g, nxt, lane);
      if (more) stage_issue(a, w1, nx, stage0 + (buf ^ 1) * kFluxStageBytes, lane32, lane, sub, own);
      cp_async_commit();
      const StageRaw nxt2 =
          stage_load<U8, DEFER>(g, sing, grp + 2 * nwarps < groups ? grp + 2 * nwarps : grp, lane, sub);
      cp_async_wait<1>();
      __syncwarp();
      const char* st = stage0 + buf * kFluxStageBytes;
      const char* f = st + lane32 * 16;
      const char* o = st + kFluxStageChunks * 512 + sub * 7 * 16;
      const double2 pn = *reinterpret_cast<const double2*>(f);
      const double2 w = *reinterpret_cast<const double2*>(f + 512);
      const double2 q01 = *reinterpret_cast<const double2*>(f + 2 * 512), q23 = *reinterpret_cast<const double2*>(f + 3 * 512);
      const double2 x01 = *reinterpret_cast<const double2*>(f + 4 * 512), y01 = *reinterpret_cast<const double2*>(f + 5 * 512);
      const double2 x23 = *reinterpret_cast<const double2*>(f + 6 * 512), y23 = *reinterpret_cast<const double2*>(f + 7 * 512);
      const double2 pi = *reinterpret_cast<const double2*>(o);
      const double2 oq01 = *reinterpret_cast<const double2*>(o + 16), oq23 = *reinterpret_cast<const double2*>(o + 32);
      const double2 ox01 = *reinterpret_cast<const double2*>(o + 48), oy01 = *reinterpret_cast<const double2*>(o + 64);
      const double2 ox23 = *reinterpret_cast<const double2*>(o + 80), oy23 = *reinterpret_cast<const double2*>(o + 96);
      if (!DEFER && cur.live && lane == 0 && cur.sing != 0xFF)
        raise_err(a.ctl, flux_key(a.ctl, g.part[cur.i], gidx(g, cur.i), cur.sing, kSolveSlot), sub_flux(a.ctl));
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      bool redo = false;
      flux_pair_fast<HP, DEFER>(a, cur.i, lane, cur.act, pi, D4{oq01.x, oq01.y, oq23.x, oq23.y},
                                D4{ox01.x, ox01.y, ox23.x, ox23.y}, D4{oy01.x, oy01.y, oy23.x, oy23.y}, pn,
                                D4{q01.x, q01.y, q23.x, q23.y}, D4{x01.x, x01.y, x23.x, x23.y},
                                D4{y01.x, y01.y, y23.x, y23.y}, w, w2 ? w2 + cur.e : nullptr, acc, &redo);
      const double r = reduce8(acc, lane);
      if (cur.live) store_res8(a.res, cur.i, r, lane);
      if (DEFER && redo && cur.live) atomicOr(rd.bits + (cur.i >> 5), 1u << (cur.i & 31));
      __syncwarp();  // the stage is refilled two groups on
      cur = nx;
      nxt = nxt2;
    }
    cp_async_wait<0>();
  }
  __syncthreads();
  ktimer_end(a.ctl, KT_FLUX);
}

// Any live point with a singular split stencil (once per domain, after k_flux_weights).
__global__ void k_flux_any_sing(Geo g, const std::uint8_t* __restrict__ sing, unsigned* __restrict__ any) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < g.n && g.kind[i] != KIND_OUTER && sing[i] != 0xFFu) atomicOr(any, 1u);
}

// Points whose state has a velocity component at or above 1.35 sqrt(2 p / rho)
// (|s| >= 1.35 where the erf fast path ends at 1.5; invalid states count too):
// k_flux_redo's share of a flux pass is about this fraction of the points, so
// the engine keeps the deferral only while it is small (Domain::probe_defer).
__global__ void k_defer_probe(Geo g, const D4* __restrict__ prim, unsigned* __restrict__ count) {
  constexpr unsigned kFull = 0xFFFFFFFFu;
  for (int base = blockIdx.x * blockDim.x; base < g.n; base += gridDim.x * blockDim.x) {
    const int i = base + static_cast<int>(threadIdx.x);
    bool hit = false;
    if (i < g.n && g.kind[i] != KIND_OUTER) {
      const D4 s = ld4(prim + i);
      const double um = fmax(fabs(s.b), fabs(s.c));
      hit = !(um * um * (0.5 * s.a / s.d) < 1.35 * 1.35);
    }
    const unsigned m = __ballot_sync(kFull, hit);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(count, static_cast<unsigned>(__popc(m)));
  }
}

// The flagged points of a DEFER flux pass, evaluated as k_flux_w does (global
// loads, fallbacks and failure checks in place: the bits k_flux_ws without
// DEFER stores).  A warp step scans 4096 flags (a uint4 of bits per lane);
// flagged points are evaluated four at a time, one per 8-lane group.
__device__ __forceinline__ void flux_point_redo(const FluxArgs& a, const double2* w1, const double2* w2,
                                                const std::uint8_t* sing, int i, int lane) {
  constexpr unsigned kFull = 0xFFFFFFFFu;
  const Geo& g = a.g;
  const int ic = i >= 0 ? i : 0;
  const bool live = i >= 0 && g.kind[ic] != KIND_OUTER;
  int k = 0, e0 = 0;
  if (live) stencil_of(g, i, e0, k);
  const int kwarp = __reduce_max_sync(kFull, k);
  if (live && lane == 0) {
    const unsigned sd = sing[i];
    if (sd != 0xFFu) raise_err(a.ctl, flux_key(a.ctl, g.part[i], gidx(g, i), sd, kSolveSlot), sub_flux(a.ctl));
  }
  const double2 pi = g.xy[ic];
  const D4 qi = ld4(a.q + ic);
  D4 qxi, qyi;
  dq_load(a.dq, g.nloc, ic, qxi, qyi);
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int jb = 0; jb < kwarp; jb += 8) {
    const int j = jb + lane;
    const bool act = live && j < k;
    const int nb = act ? g.nbr[e0 + j] : ic;
    const double2 w = act ? w1[e0 + j] : make_double2(0.0, 0.0);
    const D4 qn = ld4(a.q + nb);
    D4 qxn, qyn;
    dq_load(a.dq, g.nloc, nb, qxn, qyn);
    flux_pair_fast(a, i, j, act, pi, qi, qxi, qyi, g.xy[nb], qn, qxn, qyn, w, w2 ? w2 + (e0 + j) : nullptr, acc);
  }
  const double r = reduce8(acc, lane);
  if (live) store_res8(a.res, i, r, lane);
}

__global__ void __launch_bounds__(256, 2) k_flux_redo(FluxArgs a, const double2* __restrict__ w1,
                                                      const double2* __restrict__ w2,
                                                      const std::uint8_t* __restrict__ sing, FluxRedo rd) {
  pdl_enter();
  constexpr unsigned kFull = 0xFFFFFFFFu;
  const int lane32 = threadIdx.x & 31;
  const int lane = threadIdx.x & 7;
  const int sub = lane32 >> 3;
  const int n = a.g.n;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int base = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kRedoPointsPer; base < n;
       base += nwarps * kRedoPointsPer) {
    uint4* wp = reinterpret_cast<uint4*>(rd.bits + base / 32) + lane32;
    const uint4 v = *wp;
    const bool mine = (v.x | v.y | v.z | v.w) != 0u;
    unsigned m = __ballot_sync(kFull, mine);
    while (m) {
      const int q = __ffs(m) - 1;
      m &= m - 1;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        unsigned w = __shfl_sync(kFull, c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w, q);
        const int wbase = base + q * 128 + c * 32;
        while (w) {  // warp-uniform: group `sub` takes the sub-th lowest flagged point
          unsigned t = w;
          for (int s2 = 0; s2 < sub; ++s2) t &= t - 1;
          const int i = t ? wbase + __ffs(t) - 1 : -1;
          for (int s2 = 0; s2 < 4; ++s2) w &= w - 1;
          flux_point_redo(a, w1, w2, sing, i < n ? i : -1, lane);
        }
      }
    }
    if (mine) *wp = make_uint4(0u, 0u, 0u, 0u);
  }
}

// Local time step + forward-Euler update + wall slip + next q-variables +
// residue summand, one thread per point (kernels.cpp:68-80, 160-223).
struct UpdateArgs {
  Geo g;
  Gas gas;
  const D4* q;   // q of this iteration (copied forward for outer points)
  const D4* res; // residual of this iteration
  D4* prim;      // updated in place
  D4* q_next;
  double* dt;    // written on the diag (copy-back) iteration
  double* mag;   // (dt * res0)^2, indexed by GLOBAL point id (the residue tree's order)
  double* which; // failure detail (density 0 / pressure 1), local index
  Ctl* ctl;
  // Exact residue (fast mode): this domain's accumulators [2][kAccWords] by
  // iteration parity; null = write mag for the midpoint tree (strict mode).
  unsigned long long* acc;
};

// ---------------------------------------------------------------------------
// Exact residue sum (fast mode).  The reference sums (dt*res0)^2 with a
// midpoint tree over point ids (reduce.hpp:11-17, runtime.cpp:251-256); that
// order only exists on the whole cloud, so a sharded run would have to funnel
// every summand to one device.  Instead each domain adds its summands EXACTLY
// into a fixed-point accumulator: 32-bit digits (kept in 64-bit words so
// carries can wait) of the value in units of 2^-1074, enough for any finite
// double times 2^31 summands.  Integer addition is associative, so the sum is
// independent of the number of domains, the block shape and the point order;
// the final kernel rounds it once to the nearest double (within a few ulps of
// the reference's pairwise tree, whose error is O(log2 N) ulps: far inside
// SURVEY 8(c)'s 1e-10).  Strict mode keeps the bitwise tree.
constexpr int kAccLimbs = 68;  // 68 * 32 = 2176 bits > 1074 + 1024 + 31
constexpr int kAccFlag = kAccLimbs;  // non-finite summand seen
constexpr int kAccWords = 72;        // limbs + flag + padding (576 bytes)

// Adds the warp's 32 summands (one per lane, >= 0 or non-finite) to a block
// accumulator in shared memory.  All 32 lanes must call it together.  The
// common case — the warp's summands within a factor 2^64 of each other — is
// one 128-bit warp sum and up to four shared atomics by lane 0.
__device__ __forceinline__ void acc_warp_add(unsigned long long* sacc, double v) {
  constexpr unsigned kFull = 0xFFFFFFFFu;
  const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(v));
  const unsigned be = static_cast<unsigned>(bits >> 52) & 0x7FFu;
  const bool nonfinite = be == 0x7FFu;
  const bool live = !nonfinite && (bits & 0x7FFFFFFFFFFFFFFFull) != 0ull;
  const int lane = threadIdx.x & 31;
  if (__any_sync(kFull, nonfinite) && lane == 0) sacc[kAccFlag] = 1ull;
  if (!__any_sync(kFull, live)) return;
  const unsigned long long m = live ? ((bits & 0xFFFFFFFFFFFFFull) | (be ? (1ull << 52) : 0ull)) : 0ull;
  const unsigned pos = be ? be - 1u : 0u;  // value = m * 2^pos * 2^-1074
  const unsigned L = pos >> 5, sh = pos & 31u;
  const unsigned lmin = __reduce_min_sync(kFull, live ? L : 0xFFFFFFFFu);
  const unsigned lmax = __reduce_max_sync(kFull, live ? L : 0u);
  if (lmax - lmin <= 1u) {
    const unsigned k = live ? sh + 32u * (L - lmin) : 0u;  // <= 63
    unsigned long long lo = m << k, hi = k ? (m >> (64u - k)) : 0ull;  // < 2^116
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long l2 = __shfl_xor_sync(kFull, lo, o), h2 = __shfl_xor_sync(kFull, hi, o);
      const unsigned long long s2 = lo + l2;
      hi += h2 + (s2 < lo ? 1ull : 0ull);
      lo = s2;
    }
    if (lane == 0) {  // < 2^121: four digits from lmin
      atomicAdd(sacc + lmin, lo & 0xFFFFFFFFull);
      if (lo >> 32) atomicAdd(sacc + lmin + 1, lo >> 32);
      if (hi & 0xFFFFFFFFull) atomicAdd(sacc + lmin + 2, hi & 0xFFFFFFFFull);
      if (hi >> 32) atomicAdd(sacc + lmin + 3, hi >> 32);
    }
  } else if (live) {  // widely spread summands: three digits per lane
    const unsigned long long lo = m << sh, hi = sh ? (m >> (64u - sh)) : 0ull;
    atomicAdd(sacc + L, lo & 0xFFFFFFFFull);
    atomicAdd(sacc + L + 1, lo >> 32);
    if (hi) atomicAdd(sacc + L + 2, hi);
  }
}

// Block accumulator -> the domain's accumulator (call after a __syncthreads()).
__device__ __forceinline__ void acc_block_flush(const unsigned long long* sacc, unsigned long long* acc) {
  for (int t = threadIdx.x; t <= kAccFlag; t += blockDim.x) {
    const unsigned long long v = sacc[t];
    if (v) atomicAdd(acc + t, v);
  }
}

// The exact sum (digits summed over domains, carries not yet propagated)
// rounded to the nearest double, ties to even.  One thread.
__device__ __forceinline__ double acc_to_double(unsigned long long* d) {
  for (int i = 0; i < kAccLimbs - 1; ++i) {
    d[i + 1] += d[i] >> 32;
    d[i] &= 0xFFFFFFFFull;
  }
  int top = kAccLimbs - 1;
  while (top >= 0 && d[top] == 0ull) --top;
  if (top < 0) return 0.0;
  if (d[top] >> 32) return __longlong_as_double(0x7FF0000000000000ll);  // beyond any double
  const int b = 31 - __clz(static_cast<unsigned>(d[top]));
  const int msb = 32 * top + b;  // bit position of the leading one (units 2^-1074)
  if (msb < 53) {  // < 2^53 units: exactly representable
    const unsigned long long v = (top >= 1 ? d[1] << 32 : 0ull) | d[0];
    return ldexp(static_cast<double>(v), -1074);
  }
  // 96-bit window of the three top digits (leading one at bit 64 + b) + sticky
  const unsigned long long w2 = d[top], w1 = top >= 1 ? d[top - 1] : 0ull, w0 = top >= 2 ? d[top - 2] : 0ull;
  bool sticky = false;
  for (int i = 0; i < top - 2; ++i) sticky = sticky || d[i] != 0ull;
  // window = w2:w1:w0 (32 bits each); keep 53 bits: drop r = 12 + b low bits
  const unsigned long long hi64 = (w2 << 32) | w1;  // window >> 32 (w2 < 2^32)
  const int r = 12 + b;                             // 12..43
  // mantissa = window >> r = (hi64 << 32 | w0) >> r
  unsigned long long mant, rem_hi;  // rem = low r bits of the window
  bool round_bit, rest;
  if (r >= 32) {
    mant = hi64 >> (r - 32);
    const unsigned long long rem = ((hi64 & ((1ull << (r - 32)) - 1ull)) << 32) | w0;  // r bits
    round_bit = (rem >> (r - 1)) & 1ull;
    rest = (rem & ((1ull << (r - 1)) - 1ull)) != 0ull;
    rem_hi = 0;
  } else {
    mant = (hi64 << (32 - r)) | (w0 >> r);
    const unsigned long long rem = w0 & ((1ull << r) - 1ull);
    round_bit = (rem >> (r - 1)) & 1ull;
    rest = (rem & ((1ull << (r - 1)) - 1ull)) != 0ull;
    rem_hi = 0;
  }
  (void)rem_hi;
  if (round_bit && (rest || sticky || (mant & 1ull))) ++mant;
  int e = msb - 52;
  if (mant >> 53) {
    mant >>= 1;
    ++e;
  }
  return ldexp(static_cast<double>(mant), e - 1074);
}

// state_update for owned point ip; returns its residue summand (dt*res0)^2
// (0 for outer points and for a failing point, whose error is recorded).
__device__ __forceinline__ double update_point(const UpdateArgs& a, int ip, bool diag) {
  const Geo& g = a.g;
  // every input in one round trip (the kind no longer gates the other loads;
  // outer points, a thin ring, read res/prim/mind for nothing)
  const unsigned kind = g.kind[ip];
  const D4 r = ld4(a.res + ip);
  const D4 s = ld4_rw(a.prim + ip);
  const double mind = g.mind[ip];
  if (kind == KIND_OUTER) {
    st4(a.q_next + ip, ld4(a.q + ip));
    if (diag) a.dt[ip] = 0.0;
    return 0.0;
  }
  const double speed = sqrt(X::add(X::mul(s.b, s.b), X::mul(s.c, s.c)));
  const double sound = sqrt(X::mul(a.gas.gamma, s.d) / s.a);
  const double dt = X::mul(a.gas.cfl, mind) / X::add(speed, sound);
  double m = s.a, mx = X::mul(s.a, s.b), my_ = X::mul(s.a, s.c);
  double en = X::add(s.d / a.gas.gm1,
                     X::mul(X::mul(0.5, s.a), X::add(X::mul(s.b, s.b), X::mul(s.c, s.c))));
  m = X::sub(m, X::mul(dt, r.a));
  mx = X::sub(mx, X::mul(dt, r.b));
  my_ = X::sub(my_, X::mul(dt, r.c));
  en = X::sub(en, X::mul(dt, r.d));
  bool ok = m > 0.0;
  double u1 = 0.0, u2 = 0.0, p = 0.0;
  if (ok) {
    u1 = mx / m;
    u2 = my_ / m;
    p = X::mul(a.gas.gm1, X::sub(en, X::mul(0.5, X::add(X::mul(mx, u1), X::mul(my_, u2)))));
    ok = p > 0.0;
  }
  if (!ok) {
    // keep the failing conserved value for the diagnostic message
    a.dt[ip] = m > 0.0 ? p : m;
    a.which[ip] = m > 0.0 ? 1.0 : 0.0;
    raise_err(a.ctl, err_key(PH_UPDATE, g.part[ip], gidx(g, ip), 0, 0), sub_update(a.ctl));
    return 0.0;
  }
  if (kind == KIND_WALL) {
    const double2 nv = g.nrm[ip];
    const double un = X::add(X::mul(u1, nv.x), X::mul(u2, nv.y));
    u1 = X::sub(u1, X::mul(un, nv.x));
    u2 = X::sub(u2, X::mul(un, nv.y));
  }
  st4(a.prim + ip, D4{m, u1, u2, p});
  st4(a.q_next + ip, q_from_prim(m, u1, u2, p, a.gas.gm1));
  if (diag) a.dt[ip] = dt;
  const double dm = X::mul(dt, r.a);
  return X::mul(dm, dm);
}

__global__ void __launch_bounds__(256) k_update(UpdateArgs a) {
  pdl_enter();
  __shared__ int s_skip;
  __shared__ unsigned long long sacc[kAccWords];
  ktimer_begin(a.ctl, KT_UPDATE);
  if (threadIdx.x == 0) s_skip = skip_stage(a.ctl, sub_update(a.ctl));
  const int it = iter_of(a.ctl);
  if (a.acc) {
    for (int t = threadIdx.x; t < kAccWords; t += blockDim.x) sacc[t] = 0ull;
    // the accumulator of iteration it + 1 (read by the residue of it - 1,
    // which precedes this kernel) starts from zero
    if (blockIdx.x == 0)
      for (int t = threadIdx.x; t < kAccWords; t += blockDim.x) a.acc[((it + 1) & 1) * kAccWords + t] = 0ull;
  }
  __syncthreads();
  const Geo& g = a.g;
  const bool diag = it == a.ctl->diag_iter;
  if (a.acc) {
    // warp-uniform trip count: every lane of a warp reaches acc_warp_add together
    for (int base = blockIdx.x * blockDim.x; !s_skip && base < g.n; base += gridDim.x * blockDim.x) {
      const int ip = base + static_cast<int>(threadIdx.x);
      const double v = ip < g.n ? update_point(a, ip, diag) : 0.0;
      acc_warp_add(sacc, v);
    }
    __syncthreads();
    if (!s_skip) acc_block_flush(sacc, a.acc + (it & 1) * kAccWords);
  } else {
    for (int ip = blockIdx.x * blockDim.x + threadIdx.x; !s_skip && ip < g.n; ip += gridDim.x * blockDim.x)
      a.mag[gidx(g, ip)] = update_point(a, ip, diag);
  }
  __syncthreads();
  ktimer_end(a.ctl, KT_UPDATE);
  if (threadIdx.x == 0) atomicAdd(&a.ctl->upd_done, 1ull);  // read by later kernels (stream order)
}

// ---------------------------------------------------------------------------
// Halo exchange: ghost slot h of this domain (local index n_own + h) pulls its
// records from the owning domain's buffer — `planes` planes of 32-byte
// records (q: 1; dq: the qx and qy planes, dq_load), plane r of point p at
// base + r * ps + p — read directly over peer memory (NVLink/NVSwitch when the
// domains sit on different GPUs).
constexpr int kMaxDomains = 64;  // domains (GPUs / ranks) per run
struct PeerTab {
  const D4* base[kMaxDomains];
  long long ps[kMaxDomains];  // plane stride (the owner's local point count)
};

// skip_first: the gather is a no-op in iteration 0 (the q halo then comes from
// the domain's own first q_variables).
__global__ void k_halo(D4* dst, long long dst_ps, int planes, int n_own, int n_halo, const int* hdom,
                       const int* hidx, PeerTab src, const Ctl* ctl, int sub, int skip_first) {
  if (skip_first && iter_of(ctl) == 0) return;
  if (skip_stage(ctl, sub)) return;  // keep the failing stage's buffers intact
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n_halo * planes; t += gridDim.x * blockDim.x) {
    const int r = t / n_halo, h = t - r * n_halo;
    const int d = hdom[h];
    const D4* s = src.base[d] + r * src.ps[d] + hidx[h];
    st4(dst + r * dst_ps + n_own + h, ld4_rw(s));
  }
}

// ---------------------------------------------------------------------------
// Per-phase operators for the reference operator API (kernels.hpp:52-59).
__global__ void k_op_timestep(Geo g, const D4* prim, double* dt, Gas gas) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.n) return;
  if (g.kind[i] == KIND_OUTER) {
    dt[i] = 0.0;
    return;
  }
  const D4 s = ld4(prim + i);
  const double speed = sqrt(X::add(X::mul(s.b, s.b), X::mul(s.c, s.c)));
  const double sound = sqrt(X::mul(gas.gamma, s.d) / s.a);
  dt[i] = X::mul(gas.cfl, g.mind[i]) / X::add(speed, sound);
}

__global__ void k_op_update(Geo g, D4* prim, const D4* res, double* dt, Gas gas, Ctl* ctl,
                            double* which) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.n || g.kind[i] == KIND_OUTER) return;
  const D4 s = ld4_rw(prim + i);
  if (!(s.a > 0.0) || !(s.d > 0.0)) {  // conserved_from_primitives require_valid
    raise_err(ctl, err_key(PH_QVAR, g.part[i], gidx(g, i), 0, 0), 0);
    return;
  }
  const D4 r = ld4(res + i);
  const double h = dt[i];
  double m = s.a, mx = X::mul(s.a, s.b), my_ = X::mul(s.a, s.c);
  double en = X::add(s.d / gas.gm1,
                     X::mul(X::mul(0.5, s.a), X::add(X::mul(s.b, s.b), X::mul(s.c, s.c))));
  m = X::sub(m, X::mul(h, r.a));
  mx = X::sub(mx, X::mul(h, r.b));
  my_ = X::sub(my_, X::mul(h, r.c));
  en = X::sub(en, X::mul(h, r.d));
  if (!(m > 0.0)) {
    dt[i] = m;
    which[i] = 0.0;
    raise_err(ctl, err_key(PH_UPDATE, g.part[i], gidx(g, i), 0, 0), 0);
    return;
  }
  double u1 = mx / m, u2 = my_ / m;
  const double p = X::mul(gas.gm1, X::sub(en, X::mul(0.5, X::add(X::mul(mx, u1), X::mul(my_, u2)))));
  if (!(p > 0.0)) {
    dt[i] = p;
    which[i] = 1.0;
    raise_err(ctl, err_key(PH_UPDATE, g.part[i], gidx(g, i), 0, 0), 0);
    return;
  }
  if (g.kind[i] == KIND_WALL) {
    const double2 nv = g.nrm[i];
    const double un = X::add(X::mul(u1, nv.x), X::mul(u2, nv.y));
    u1 = X::sub(u1, X::mul(un, nv.x));
    u2 = X::sub(u2, X::mul(un, nv.y));
  }
  st4(prim + i, D4{m, u1, u2, p});
}

// ---------------------------------------------------------------------------
// Residue: the reference's recursive midpoint-tree sum over ids [0, n)
// (reduce.hpp:11-17), evaluated exactly.  Node (d, k) of the tree is found by
// replaying the midpoint splits along k's bits; a node of size <= 1 is a leaf.
__device__ __forceinline__ void tree_node(long long lo0, long long hi0, int depth,
                                          long long k, long long& lo, long long& hi) {
  lo = lo0;
  hi = hi0;
  for (int l = depth - 1; l >= 0; --l) {
    const long long mid = lo + (hi - lo) / 2;
    if ((k >> l) & 1) lo = mid;
    else hi = mid;
  }
}

__device__ double tree_sum(const double* v, long long lo, long long hi) {
  const long long len = hi - lo;
  if (len <= 0) return 0.0;
  if (len == 1) return v[lo];
  if (len == 2) return X::add(v[lo], v[lo + 1]);
  if (len == 3) return X::add(v[lo], X::add(v[lo + 1], v[lo + 2]));
  const long long mid = lo + len / 2;
  return X::add(tree_sum(v, lo, mid), tree_sum(v, mid, hi));
}

// One node of the midpoint tree from its two children (sizes decide how
// empty and single-element children combine, exactly as the recursion does).
__device__ __forceinline__ void tree_pair(double vl, long long sl, double vr, long long sr, double& v,
                                          long long& s) {
  s = sl + sr;
  v = s <= 0 ? 0.0 : (s == 1 ? (sr == 1 ? vr : vl) : X::add(vl, vr));
}

// Loads the 2^d1 partials (d1 <= 13) as 2^min(d1, LV) subtree values: with
// d1 > LV each thread folds its 2^(d1-LV) consecutive partials (one subtree)
// serially.
template <int LV = 10>
__device__ __forceinline__ int tree_load_partials(const double* part_val, const long long* part_sz, int d1,
                                                  double* sv, long long* ss) {
  const int lv = d1 > LV ? LV : d1;
  const int per = 1 << (d1 - lv);
  for (int t = threadIdx.x; t < (1 << lv); t += blockDim.x) {
    double v[1 << (13 - LV)];
    long long s[1 << (13 - LV)];
    for (int k = 0; k < per; ++k) {
      v[k] = part_val[t * per + k];
      s[k] = part_sz[t * per + k];
    }
    for (int w = per; w > 1; w >>= 1)
      for (int k = 0; k < w / 2; ++k) tree_pair(v[2 * k], s[2 * k], v[2 * k + 1], s[2 * k + 1], v[k], s[k]);
    sv[t] = v[0];
    ss[t] = s[0];
  }
  return lv;
}

// Combines 2^levels children (val/sz in ping) up `levels` levels; T threads.
template <int T>
__device__ void tree_combine(double* val, long long* sz, double* val2, long long* sz2,
                             int levels) {
  double* cv = val;
  long long* cs = sz;
  double* nv = val2;
  long long* ns = sz2;
  for (int l = levels; l > 0; --l) {
    const int half = 1 << (l - 1);
    for (int t = threadIdx.x; t < half; t += T) {
      const long long sl = cs[2 * t], sr = cs[2 * t + 1];
      const long long ps = sl + sr;
      double v;
      if (ps <= 0) v = 0.0;
      else if (ps == 1) v = sr == 1 ? cv[2 * t + 1] : cv[2 * t];
      else v = X::add(cv[2 * t], cv[2 * t + 1]);
      nv[t] = v;
      ns[t] = ps;
    }
    __syncthreads();
    double* tv = cv; cv = nv; nv = tv;
    long long* ts = cs; cs = ns; ns = ts;
  }
  if (threadIdx.x == 0) {
    val[0] = cv[0];
    sz[0] = cs[0];
  }
  __syncthreads();
}

constexpr int kTreeThreads = 256;
constexpr int kTreeThreadLevels = 8;

// Stage 1: block b reduces node (d1, b); its 256 threads take the nodes 8
// levels further down and sum them serially by the same recursion.
__global__ void __launch_bounds__(kTreeThreads)
    k_tree_partial(const double* v, long long n, int d1, double* part_val, long long* part_sz,
                   Ctl* ctl) {
  pdl_enter();
  __shared__ double sv[2][kTreeThreads];
  __shared__ long long ss[2][kTreeThreads];
  __shared__ int s_skip;
  ktimer_begin(ctl, KT_RESIDUE);
  if (threadIdx.x == 0) s_skip = skip_stage(ctl, sub_residue(ctl), 1);
  __syncthreads();
  if (!s_skip) {
    long long lo, hi, tlo, thi;
    tree_node(0, n, d1, blockIdx.x, lo, hi);
    tree_node(lo, hi, kTreeThreadLevels, threadIdx.x, tlo, thi);
    sv[0][threadIdx.x] = tree_sum(v, tlo, thi);
    ss[0][threadIdx.x] = thi - tlo;
  }
  __syncthreads();
  if (!s_skip) {
    tree_combine<kTreeThreads>(sv[0], ss[0], sv[1], ss[1], kTreeThreadLevels);
    if (threadIdx.x == 0) {
      part_val[blockIdx.x] = sv[0][0];
      part_sz[blockIdx.x] = ss[0][0];
    }
  }
  __syncthreads();
  ktimer_end(ctl, KT_RESIDUE, nullptr);
}

// Stage 2: one block of T threads folds the 2^d1 partials, forms sqrt(sum)/n
// and records the history entry (runtime.cpp:251-269); non-finite ->
// positivity error.  sv/ss: [2][1024] shared scratch.
template <int T, int LV = 10>
__device__ __forceinline__ void tree_final(const double* part_val, const long long* part_sz, int d1, long long n,
                                           double* history, unsigned long long* iter_t0,
                                           unsigned long long* iter_t1, Ctl* ctl, double (*sv)[1 << LV],
                                           long long (*ss)[1 << LV], int* s_skip) {
  if (threadIdx.x == 0) *s_skip = skip_stage(ctl, sub_residue(ctl), 1);
  __syncthreads();
  if (*s_skip) {
    if (threadIdx.x < 32) ktimer_fold_warp(ctl);
    return;
  }
  const int lv = tree_load_partials<LV>(part_val, part_sz, d1, sv[0], ss[0]);
  __syncthreads();
  tree_combine<T>(sv[0], ss[0], sv[1], ss[1], lv);
  __shared__ int s_it, s_ok;
  if (threadIdx.x == 0) {
    const double res = sqrt(sv[0][0]) / static_cast<double>(n);
    const int it = iter_of(ctl, 1);
    s_it = it;
    s_ok = isfinite(res) ? 1 : 0;
    if (!isfinite(res)) {
      raise_err(ctl, err_key(PH_RESIDUE, 0, 0, 0, 0), sub_residue(ctl), 1);
    } else {
      if (history) history[it] = res;
      if (iter_t1) iter_t1[it] = globaltimer();
      ctl->sh->iter = it + 1;  // iterations completed (residue recorded)
    }
    atomicMax(&ctl->kt[KT_RESIDUE].t1, globaltimer());
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const unsigned long long t0 = ktimer_fold_warp(ctl);
    if (threadIdx.x == 0 && iter_t0 && s_ok) iter_t0[s_it] = t0;
  }
}

__global__ void __launch_bounds__(1024)
    k_tree_final(const double* part_val, const long long* part_sz, int d1, long long n,
                 double* history, unsigned long long* iter_t0, unsigned long long* iter_t1, Ctl* ctl) {
  pdl_enter();
  __shared__ double sv[2][1024];
  __shared__ long long ss[2][1024];
  __shared__ int s_skip;
  tree_final<1024>(part_val, part_sz, d1, n, history, iter_t0, iter_t1, ctl, sv, ss, &s_skip);
}

// Plain tree sum of an arbitrary vector (lskum_b200_reduce): same two stages
// without the history bookkeeping.
__global__ void k_tree_result(const double* part_val, const long long* part_sz, int d1,
                              double* out) {
  __shared__ double sv[2][1024];
  __shared__ long long ss[2][1024];
  const int lv = tree_load_partials<10>(part_val, part_sz, d1, sv[0], ss[0]);
  __syncthreads();
  tree_combine<1024>(sv[0], ss[0], sv[1], ss[1], lv);
  if (threadIdx.x == 0) *out = sv[0][0];
}

// Exact residue of the iteration (fast mode): sums the digits of every
// domain's accumulator (over peer memory for the other domains), rounds once,
// forms sqrt(sum)/n and records the history entry as tree_final does.
struct AccTab {
  const unsigned long long* p[kMaxDomains];  // each domain's [2][kAccWords]
};
__global__ void __launch_bounds__(96)
    k_residue_exact(AccTab acc, int ndom, long long n, double* history, unsigned long long* iter_t0,
                    unsigned long long* iter_t1, Ctl* ctl) {
  pdl_enter();
  __shared__ unsigned long long sd[kAccWords];
  __shared__ int s_skip, s_it, s_ok;
  ktimer_begin(ctl, KT_RESIDUE);
  if (threadIdx.x == 0) s_skip = skip_stage(ctl, sub_residue(ctl), 1);
  __syncthreads();
  if (s_skip) {
    if (threadIdx.x < 32) ktimer_fold_warp(ctl);
    return;
  }
  const int it = iter_of(ctl, 1);
  if (threadIdx.x <= kAccFlag) {
    unsigned long long v = 0;
    for (int d = 0; d < ndom; ++d) v += ld_volatile(acc.p[d] + (it & 1) * kAccWords + threadIdx.x);
    sd[threadIdx.x] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double sum = sd[kAccFlag] ? __longlong_as_double(0x7FF8000000000000ll) : acc_to_double(sd);
    const double res = sqrt(sum) / static_cast<double>(n);
    s_it = it;
    s_ok = isfinite(res) ? 1 : 0;
    if (!isfinite(res)) {
      raise_err(ctl, err_key(PH_RESIDUE, 0, 0, 0, 0), sub_residue(ctl), 1);
    } else {
      if (history) history[it] = res;
      if (iter_t1) iter_t1[it] = globaltimer();
      ctl->sh->iter = it + 1;
    }
    atomicMax(&ctl->kt[KT_RESIDUE].t1, globaltimer());
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const unsigned long long t0 = ktimer_fold_warp(ctl);
    if (threadIdx.x == 0 && iter_t0 && s_ok) iter_t0[s_it] = t0;
  }
}

// Exact sum of an arbitrary vector of non-negative doubles (tests of the
// accumulator: lskum_b200_exact_sum).
__global__ void __launch_bounds__(256) k_exact_sum_blocks(const double* v, long long n, unsigned long long* acc) {
  __shared__ unsigned long long sacc[kAccWords];
  for (int t = threadIdx.x; t < kAccWords; t += blockDim.x) sacc[t] = 0ull;
  __syncthreads();
  for (long long base = static_cast<long long>(blockIdx.x) * blockDim.x; base < n;
       base += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = base + threadIdx.x;
    acc_warp_add(sacc, i < n ? v[i] : 0.0);
  }
  __syncthreads();
  acc_block_flush(sacc, acc);
}
__global__ void k_exact_sum_final(unsigned long long* acc, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0)
    *out = acc[kAccFlag] ? __longlong_as_double(0x7FF8000000000000ll) : acc_to_double(acc);
}

__global__ void k_copy_d4(const D4* src, D4* dst, long long count) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i < count) st4(dst + i, ld4(src + i));
}

}  // namespace lskd
