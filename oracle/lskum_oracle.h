/* lskum_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C CPU restatement of the reference LSKUM hot path
 * (/root/reference/proj/src/core/{kinetic,kernels,runtime,reduce,partition,cloud}.cpp).
 * It is the checker for the CUDA path: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * library (paper_2403_13287_b200/liblskum_b200.so) never links or calls it.
 *
 * Parity pinning: tests/test_oracle_pinning.py checks this restatement
 * bit-for-bit against the reference itself (oracle/_ref/liblskum_refshim.so,
 * built from the reference sources by oracle/Makefile) and against the
 * committed golden fixtures under tests/golden/ (made by tests/golden/make_golden.py
 * from the reference).  All arithmetic is IEEE fp64 with -ffp-contract=off,
 * in the reference's operation order.
 */
#ifndef LSKUM_ORACLE_H
#define LSKUM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_ARGUMENT = 1, ORC_VALIDATION = 4, ORC_SINGULAR = 5,
       ORC_POSITIVITY = 6, ORC_CONFIG = 7 };

/* FieldStore slots (src/core/layout.hpp:11-19); the oracle store is AoS n*21. */
enum { ORC_PRIM = 0, ORC_Q = 4, ORC_QX = 8, ORC_QY = 12, ORC_RES = 16, ORC_DT = 20,
       ORC_SLOTS = 21 };

/* Point kinds (src/core/cloud.hpp:14). */
enum { ORC_INTERIOR = 0, ORC_WALL = 1, ORC_OUTER = 2 };

typedef struct {
  int32_t n;
  const double *x, *y, *nx, *ny;
  const uint8_t *kind;
  const int64_t *off; /* n+1 CSR offsets */
  const int32_t *nbr; /* neighbour ids, ascending per point */
} orc_cloud;

typedef struct {
  int code;      /* ORC_* status */
  int iteration; /* 1-based iteration of the failure (0 = setup) */
  int point;     /* failing point (or -1) */
  int nb;        /* failing neighbour for reconstruction errors (or -1) */
  char msg[320];
} orc_status;

typedef struct {
  double mach, aoa_deg, gamma, cfl;
  int iters, n_inner, order;
} orc_config;

/* ---- per-point math (src/core/kinetic.cpp) ---- */
int orc_q_from_prim(const double s[4], double g, double q[4], orc_status* st);
int orc_prim_from_q(const double q[4], double g, double s[4], orc_status* st);
int orc_cons_from_prim(const double s[4], double g, double u[4], orc_status* st);
int orc_prim_from_cons(const double u[4], double g, double s[4], orc_status* st);
int orc_full_flux(const double s[4], int axis, double g, double f[4], orc_status* st);
int orc_kfvs_flux(const double s[4], int axis, int minus, double g, double f[4],
                  orc_status* st);

/* ---- phase kernels over all points (src/core/kernels.cpp) ---- */
int orc_q_variables(const orc_cloud* c, double* store, double g, orc_status* st);
int orc_q_derivatives(const orc_cloud* c, const double* store, double det_tol,
                      double* scratch, orc_status* st);
void orc_publish(const orc_cloud* c, double* store, const double* scratch);
int orc_flux_fused(const orc_cloud* c, double* store, double g, double det_tol,
                   orc_status* st);
int orc_flux_direction(const orc_cloud* c, double* store, double g, double det_tol,
                       int axis, int minus, int first, orc_status* st);
void orc_timestep(const orc_cloud* c, double* store, double g, double cfl);
int orc_state_update(const orc_cloud* c, double* store, double g, orc_status* st);

/* ---- runtime (src/core/runtime.cpp, src/core/reduce.hpp) ---- */
double orc_reduce(const double* v, int64_t lo, int64_t hi);
/* Runs the fixed-point loop from the primitives already in `store` (AoS n*21).
 * residue[] gets one entry per completed iteration; returns the status code. */
int orc_run(const orc_cloud* c, const orc_config* cfg, double* store, double* residue,
            int* n_done, orc_status* st);

/* ---- validation (src/core/cloud.cpp:252-321) ---- */
typedef struct {
  int32_t n_defective, n_wall_isolated, min_stencil_size;
  double h_ref, det_tol;
} orc_validation;
/* defective: caller array of n ids (may be NULL) */
void orc_validate(const orc_cloud* c, orc_validation* v, int32_t* defective);

/* ---- partitioning (src/core/partition.cpp:12-80) ---- */
/* owner[i] = part of point i; ghosts of part p are written to
 * ghosts[ghost_off[p] .. ghost_off[p+1]) (ghost_off has n_parts+1 entries). */
int orc_partition(const orc_cloud* c, int n_parts, int32_t* owner, int64_t* ghost_off,
                  int32_t* ghosts, int64_t ghost_cap);

/* ---- generators (src/core/cloud.cpp:26-30, 137-237, 323-425) ---- */
typedef struct {
  int32_t n;
  int64_t nnz;
  double *x, *y, *nx, *ny;
  uint8_t* kind;
  int64_t* off;
  int32_t* nbr;
} orc_owned_cloud;
int orc_generate_rect(int nx, int ny, double xmin, double xmax, double ymin, double ymax,
                      double jitter, uint64_t seed, int k, orc_owned_cloud* out);
int orc_generate_annulus(int n_theta, int n_rings, double r_outer, double jitter,
                         uint64_t seed, int k, orc_owned_cloud* out);
void orc_free_cloud(orc_owned_cloud* c);
/* mt19937_64 stream used by the generators, exposed for the pinning tests. */
void orc_mt_draws(uint64_t seed, int count, uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif
