/* lskum_oracle.c — TEST INFRASTRUCTURE ONLY: the CPU checker for the CUDA path.
 *
 * A plain-C restatement of the reference algorithm, function by function, in
 * the reference's floating-point operation order (compile with
 * -ffp-contract=off, as the reference's CMakeLists.txt:10-12 does).  Every
 * function cites the reference file:line it restates (paths relative to
 * /root/reference/proj).  The product never links this file.
 */
#define _GNU_SOURCE
#include "lskum_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

static int fail(orc_status* st, int code, const char* fmt, double a, double b) {
  if (st) {
    st->code = code;
    snprintf(st->msg, sizeof st->msg, fmt, a, b);
  }
  return code;
}

/* std::to_string(double) is printf("%f"). */

/* src/core/kinetic.cpp:20-22 */
static double total_energy(const double s[4], double g) {
  return s[3] / (g - 1.0) + 0.5 * s[0] * (s[1] * s[1] + s[2] * s[2]);
}

/* src/core/kinetic.cpp:12-18 */
static int require_valid(const double s[4], orc_status* st) {
  if (!(s[0] > 0.0) || !(s[3] > 0.0))
    return fail(st, ORC_POSITIVITY, "invalid primitive state: rho=%f p=%f", s[0], s[3]);
  return ORC_OK;
}

/* src/core/kinetic.cpp:26-36 */
int orc_q_from_prim(const double s[4], double g, double q[4], orc_status* st) {
  int rc = require_valid(s, st);
  if (rc) return rc;
  const double beta = 0.5 * s[0] / s[3];
  q[0] = log(s[0]) + log(beta) / (g - 1.0) - beta * (s[1] * s[1] + s[2] * s[2]);
  q[1] = 2.0 * beta * s[1];
  q[2] = 2.0 * beta * s[2];
  q[3] = -2.0 * beta;
  return ORC_OK;
}

/* src/core/kinetic.cpp:38-51 */
int orc_prim_from_q(const double q[4], double g, double s[4], orc_status* st) {
  if (!(q[3] < 0.0)) return fail(st, ORC_POSITIVITY, "q-state with q3 >= 0 (q3=%f)", q[3], 0);
  const double beta = -0.5 * q[3];
  s[1] = q[1] / (2.0 * beta);
  s[2] = q[2] / (2.0 * beta);
  s[0] = exp(q[0] - log(beta) / (g - 1.0) + beta * (s[1] * s[1] + s[2] * s[2]));
  s[3] = 0.5 * s[0] / beta;
  return ORC_OK;
}

/* src/core/kinetic.cpp:53-61 */
int orc_cons_from_prim(const double s[4], double g, double u[4], orc_status* st) {
  int rc = require_valid(s, st);
  if (rc) return rc;
  u[0] = s[0];
  u[1] = s[0] * s[1];
  u[2] = s[0] * s[2];
  u[3] = total_energy(s, g);
  return ORC_OK;
}

/* src/core/kinetic.cpp:63-78 */
int orc_prim_from_cons(const double u[4], double g, double s[4], orc_status* st) {
  if (!(u[0] > 0.0))
    return fail(st, ORC_POSITIVITY, "conserved state with non-positive density %f", u[0], 0);
  s[0] = u[0];
  s[1] = u[1] / u[0];
  s[2] = u[2] / u[0];
  s[3] = (g - 1.0) * (u[3] - 0.5 * (u[1] * s[1] + u[2] * s[2]));
  if (!(s[3] > 0.0))
    return fail(st, ORC_POSITIVITY, "conserved state with non-positive pressure %f", s[3], 0);
  return ORC_OK;
}

/* src/core/kinetic.cpp:80-89 */
int orc_full_flux(const double s[4], int axis, double g, double f[4], orc_status* st) {
  int rc = require_valid(s, st);
  if (rc) return rc;
  const double e = total_energy(s, g);
  const double rho = s[0], u1 = s[1], u2 = s[2], p = s[3];
  if (axis == 0) {
    f[0] = rho * u1; f[1] = p + rho * u1 * u1; f[2] = rho * u1 * u2; f[3] = (e + p) * u1;
  } else {
    f[0] = rho * u2; f[1] = rho * u1 * u2; f[2] = p + rho * u2 * u2; f[3] = (e + p) * u2;
  }
  return ORC_OK;
}

/* src/core/kinetic.cpp:91-111 */
int orc_kfvs_flux(const double s[4], int axis, int minus, double g, double f[4],
                  orc_status* st) {
  int rc = require_valid(s, st);
  if (rc) return rc;
  const double rho = s[0], p = s[3];
  const double beta = 0.5 * rho / p;
  const double un = axis == 0 ? s[1] : s[2];
  const double ut = axis == 0 ? s[2] : s[1];
  const double s1 = un * sqrt(beta);
  const double pm = minus ? -1.0 : 1.0;
  const double a_half = 0.5 * (1.0 + pm * erf(s1));
  const double b = exp(-s1 * s1) / (2.0 * sqrt(M_PI * beta));
  const double e = total_energy(s, g);
  const double mass = rho * (un * a_half + pm * b);
  const double mom_n = (p + rho * un * un) * a_half + pm * rho * un * b;
  const double mom_t = rho * ut * (un * a_half + pm * b);
  const double erg = (e + p) * un * a_half + pm * (e + 0.5 * p) * b;
  f[0] = mass;
  f[1] = axis == 0 ? mom_n : mom_t;
  f[2] = axis == 0 ? mom_t : mom_n;
  f[3] = erg;
  return ORC_OK;
}

/* LsSums, src/core/kinetic.hpp:60-70 and kinetic.cpp:113-137 */
typedef struct {
  double sxx, sxy, syy, bx[4], by[4];
  int count;
} ls_sums;

static void ls_add(ls_sums* s, double dx, double dy, const double df[4]) {
  s->sxx += dx * dx;
  s->sxy += dx * dy;
  s->syy += dy * dy;
  for (int c = 0; c < 4; ++c) {
    s->bx[c] += dx * df[c];
    s->by[c] += dy * df[c];
  }
  ++s->count;
}

static int ls_solve(const ls_sums* s, double det_tol, double fx[4], double fy[4],
                    orc_status* st) {
  const double det = s->sxx * s->syy - s->sxy * s->sxy;
  if (!(det > det_tol))
    return fail(st, ORC_SINGULAR, "singular least-squares stencil (det=%f, n=%.0f)", det,
                (double)s->count);
  for (int c = 0; c < 4; ++c) {
    fx[c] = (s->syy * s->bx[c] - s->sxy * s->by[c]) / det;
    fy[c] = (s->sxx * s->by[c] - s->sxy * s->bx[c]) / det;
  }
  return ORC_OK;
}

static double* at(double* store, int32_t i, int slot) {
  return store + (size_t)i * ORC_SLOTS + slot;
}
static double cat(const double* store, int32_t i, int slot) {
  return store[(size_t)i * ORC_SLOTS + slot];
}

static void prefix_msg(orc_status* st, const char* fmt, long a, long b) {
  char tmp[320];
  char head[96];
  snprintf(head, sizeof head, fmt, a, b);
  snprintf(tmp, sizeof tmp, "%s%s", head, st->msg);
  memcpy(st->msg, tmp, sizeof tmp);
}

/* corrected_q, src/core/kernels.cpp:20-27 */
static void corrected_q(const double* store, int32_t i, double dx, double dy, double q[4]) {
  for (int c = 0; c < 4; ++c)
    q[c] = cat(store, i, ORC_Q + c) -
           0.5 * (dx * cat(store, i, ORC_QX + c) + dy * cat(store, i, ORC_QY + c));
}

/* q_variables_kernel, src/core/kernels.cpp:68-80 */
int orc_q_variables(const orc_cloud* c, double* store, double g, orc_status* st) {
  for (int32_t i = 0; i < c->n; ++i) {
    double s[4], q[4];
    for (int k = 0; k < 4; ++k) s[k] = cat(store, i, ORC_PRIM + k);
    int rc = orc_q_from_prim(s, g, q, st);
    if (rc) {
      if (st) st->point = i;
      return rc;
    }
    for (int k = 0; k < 4; ++k) *at(store, i, ORC_Q + k) = q[k];
  }
  return ORC_OK;
}

/* q_derivatives_kernel, src/core/kernels.cpp:82-106 */
int orc_q_derivatives(const orc_cloud* c, const double* store, double det_tol,
                      double* scratch, orc_status* st) {
  for (int32_t i = 0; i < c->n; ++i) {
    ls_sums s;
    memset(&s, 0, sizeof s);
    for (int64_t e = c->off[i]; e < c->off[i + 1]; ++e) {
      const int32_t nb = c->nbr[e];
      const double dx = c->x[nb] - c->x[i];
      const double dy = c->y[nb] - c->y[i];
      double qi[4], qn[4], df[4];
      corrected_q(store, i, dx, dy, qi);
      corrected_q(store, nb, dx, dy, qn);
      for (int k = 0; k < 4; ++k) df[k] = qn[k] - qi[k];
      ls_add(&s, dx, dy, df);
    }
    double fx[4], fy[4];
    int rc = ls_solve(&s, det_tol, fx, fy, st);
    if (rc) {
      if (st) {
        st->point = i;
        prefix_msg(st, "full stencil of point %ld: ", i, 0);
      }
      return rc;
    }
    for (int k = 0; k < 4; ++k) {
      scratch[(size_t)i * 8 + k] = fx[k];
      scratch[(size_t)i * 8 + 4 + k] = fy[k];
    }
  }
  return ORC_OK;
}

/* publish_q_derivatives, src/core/kernels.cpp:108-117 */
void orc_publish(const orc_cloud* c, double* store, const double* scratch) {
  for (int32_t i = 0; i < c->n; ++i)
    for (int k = 0; k < 4; ++k) {
      *at(store, i, ORC_QX + k) = scratch[(size_t)i * 8 + k];
      *at(store, i, ORC_QY + k) = scratch[(size_t)i * 8 + 4 + k];
    }
}

/* directional_term + upwind_side, src/core/kernels.cpp:32-64 */
static int directional_term(const orc_cloud* c, const double* store, int32_t i, int axis,
                            int minus, double g, double det_tol, double term[4],
                            orc_status* st) {
  ls_sums s;
  memset(&s, 0, sizeof s);
  for (int64_t e = c->off[i]; e < c->off[i + 1]; ++e) {
    const int32_t nb = c->nbr[e];
    const double dx = c->x[nb] - c->x[i];
    const double dy = c->y[nb] - c->y[i];
    const double d = axis == 0 ? dx : dy;
    if (!(minus ? d >= 0.0 : d <= 0.0)) continue;
    double qi[4], qn[4], si[4], sn[4], gi[4], gn[4], df[4];
    corrected_q(store, i, dx, dy, qi);
    corrected_q(store, nb, dx, dy, qn);
    int rc = orc_prim_from_q(qi, g, si, st);
    if (!rc) rc = orc_prim_from_q(qn, g, sn, st);
    if (rc) {
      if (st) {
        st->point = i;
        st->nb = nb;
        prefix_msg(st, "flux reconstruction failed on edge (%ld, %ld): ", i, nb);
      }
      return rc;
    }
    rc = orc_kfvs_flux(si, axis, minus, g, gi, st);
    if (!rc) rc = orc_kfvs_flux(sn, axis, minus, g, gn, st);
    if (rc) {
      if (st) st->point = i;
      return rc;
    }
    for (int k = 0; k < 4; ++k) df[k] = gn[k] - gi[k];
    ls_add(&s, dx, dy, df);
  }
  double fx[4], fy[4];
  int rc = ls_solve(&s, det_tol, fx, fy, st);
  if (rc) {
    if (st) {
      st->point = i;
      prefix_msg(st, "split stencil of point %ld: ", i, 0);
    }
    return rc;
  }
  for (int k = 0; k < 4; ++k) term[k] = axis == 0 ? fx[k] : fy[k];
  return ORC_OK;
}

/* flux_residual_fused_kernel, src/core/kernels.cpp:119-140 */
int orc_flux_fused(const orc_cloud* c, double* store, double g, double det_tol,
                   orc_status* st) {
  static const int order[4][2] = {{0, 0}, {0, 1}, {1, 0}, {1, 1}};
  for (int32_t i = 0; i < c->n; ++i) {
    if (c->kind[i] == ORC_OUTER) continue;
    for (int k = 0; k < 4; ++k) *at(store, i, ORC_RES + k) = 0.0;
    for (int d = 0; d < 4; ++d) {
      double term[4];
      int rc = directional_term(c, store, i, order[d][0], order[d][1], g, det_tol, term, st);
      if (rc) return rc;
      for (int k = 0; k < 4; ++k) *at(store, i, ORC_RES + k) += term[k];
    }
  }
  return ORC_OK;
}

/* flux_residual_direction_kernel, src/core/kernels.cpp:142-158 */
int orc_flux_direction(const orc_cloud* c, double* store, double g, double det_tol,
                       int axis, int minus, int first, orc_status* st) {
  for (int32_t i = 0; i < c->n; ++i) {
    if (c->kind[i] == ORC_OUTER) continue;
    if (first)
      for (int k = 0; k < 4; ++k) *at(store, i, ORC_RES + k) = 0.0;
    double term[4];
    int rc = directional_term(c, store, i, axis, minus, g, det_tol, term, st);
    if (rc) return rc;
    for (int k = 0; k < 4; ++k) *at(store, i, ORC_RES + k) += term[k];
  }
  return ORC_OK;
}

/* local_timestep_kernel, src/core/kernels.cpp:160-182 */
void orc_timestep(const orc_cloud* c, double* store, double g, double cfl) {
  for (int32_t i = 0; i < c->n; ++i) {
    if (c->kind[i] == ORC_OUTER) {
      *at(store, i, ORC_DT) = 0.0;
      continue;
    }
    double min_d = INFINITY;
    for (int64_t e = c->off[i]; e < c->off[i + 1]; ++e) {
      const int32_t nb = c->nbr[e];
      const double dx = c->x[nb] - c->x[i];
      const double dy = c->y[nb] - c->y[i];
      const double d = sqrt(dx * dx + dy * dy);
      min_d = d < min_d ? d : min_d; /* std::min(a, b) == (b < a) ? b : a */
    }
    const double rho = cat(store, i, ORC_PRIM + 0), u1 = cat(store, i, ORC_PRIM + 1);
    const double u2 = cat(store, i, ORC_PRIM + 2), p = cat(store, i, ORC_PRIM + 3);
    const double speed = sqrt(u1 * u1 + u2 * u2);
    const double sound = sqrt(g * p / rho);
    *at(store, i, ORC_DT) = cfl * min_d / (speed + sound);
  }
}

/* state_update_kernel, src/core/kernels.cpp:184-219 */
int orc_state_update(const orc_cloud* c, double* store, double g, orc_status* st) {
  for (int32_t i = 0; i < c->n; ++i) {
    if (c->kind[i] == ORC_OUTER) continue;
    double old_s[4], u[4], s[4];
    for (int k = 0; k < 4; ++k) old_s[k] = cat(store, i, ORC_PRIM + k);
    int rc = orc_cons_from_prim(old_s, g, u, st);
    if (rc) {
      if (st) st->point = i;
      return rc;
    }
    const double dt = cat(store, i, ORC_DT);
    for (int k = 0; k < 4; ++k) u[k] -= dt * cat(store, i, ORC_RES + k);
    rc = orc_prim_from_cons(u, g, s, st);
    if (rc) {
      if (st) {
        st->point = i;
        prefix_msg(st, "state update lost positivity at point %ld: ", i, 0);
      }
      return rc;
    }
    if (c->kind[i] == ORC_WALL) {
      const double un = s[1] * c->nx[i] + s[2] * c->ny[i];
      s[1] -= un * c->nx[i];
      s[2] -= un * c->ny[i];
    }
    for (int k = 0; k < 4; ++k) *at(store, i, ORC_PRIM + k) = s[k];
  }
  return ORC_OK;
}

/* deterministic_reduce, src/core/reduce.hpp:11-17 */
double orc_reduce(const double* v, int64_t lo, int64_t hi) {
  if (hi - lo <= 0) return 0.0;
  if (hi - lo == 1) return v[lo];
  const int64_t mid = lo + (hi - lo) / 2;
  return orc_reduce(v, lo, mid) + orc_reduce(v, mid, hi);
}

static int cmp_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* validate_cloud, src/core/cloud.cpp:252-321 */
void orc_validate(const orc_cloud* c, orc_validation* v, int32_t* defective) {
  const int32_t n = c->n;
  double* nn = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  int32_t m = 0;
  for (int32_t p = 0; p < n; ++p) {
    double best = INFINITY;
    for (int64_t e = c->off[p]; e < c->off[p + 1]; ++e) {
      const int32_t nb = c->nbr[e];
      const double dx = c->x[nb] - c->x[p], dy = c->y[nb] - c->y[p];
      const double d = sqrt(dx * dx + dy * dy);
      best = d < best ? d : best;
    }
    if (isfinite(best)) nn[m++] = best;
  }
  v->h_ref = 0.0;
  if (m > 0) {
    qsort(nn, (size_t)m, sizeof(double), cmp_double);
    v->h_ref = nn[(m - 1) / 2];
  }
  free(nn);
  v->det_tol = 1e-12 * v->h_ref * v->h_ref * v->h_ref * v->h_ref;
  v->n_defective = 0;
  v->n_wall_isolated = 0;
  v->min_stencil_size = n > 0 ? 2147483647 : 0;
  const double zero[4] = {0, 0, 0, 0};
  for (int32_t p = 0; p < n; ++p) {
    ls_sums full, split[4];
    memset(&full, 0, sizeof full);
    memset(split, 0, sizeof split);
    int wall_nbhs = 0;
    for (int64_t e = c->off[p]; e < c->off[p + 1]; ++e) {
      const int32_t nb = c->nbr[e];
      const double dx = c->x[nb] - c->x[p], dy = c->y[nb] - c->y[p];
      ls_add(&full, dx, dy, zero);
      if (dx >= 0.0) ls_add(&split[0], dx, dy, zero);
      if (dx <= 0.0) ls_add(&split[1], dx, dy, zero);
      if (dy >= 0.0) ls_add(&split[2], dx, dy, zero);
      if (dy <= 0.0) ls_add(&split[3], dx, dy, zero);
      if (c->kind[nb] == ORC_WALL) ++wall_nbhs;
    }
    const double full_det = full.sxx * full.syy - full.sxy * full.sxy;
    int bad = full_det < v->det_tol || full.count < 3;
    if (c->kind[p] != ORC_OUTER)
      for (int d = 0; d < 4; ++d) {
        const double sd = split[d].sxx * split[d].syy - split[d].sxy * split[d].sxy;
        bad = bad || split[d].count == 0 || sd < v->det_tol;
      }
    if (bad) {
      if (defective) defective[v->n_defective] = p;
      ++v->n_defective;
    }
    if (c->kind[p] == ORC_WALL && wall_nbhs < 2) ++v->n_wall_isolated;
    if (full.count < v->min_stencil_size) v->min_stencil_size = full.count;
  }
}

/* run_fixed_point + build_phase_plan, src/core/runtime.cpp:139-275 (one part,
 * one worker; the reference's determinism matrix, tests/acceptance.cpp:249-313,
 * makes every parts/workers combination bitwise equal to this order). */
int orc_run(const orc_cloud* c, const orc_config* cfg, double* store, double* residue,
            int* n_done, orc_status* st) {
  const int32_t n = c->n;
  *n_done = 0;
  st->code = 0;
  st->iteration = 0;
  st->point = -1;
  st->nb = -1;
  st->msg[0] = 0;
  /* SolverConfig::validate, src/core/config.cpp:47-56 */
  if (!(cfg->mach >= 0.0) || !(cfg->gamma > 1.0) || cfg->iters < 0 || cfg->n_inner < 1 ||
      !(cfg->cfl > 0.0) || (cfg->order != 1 && cfg->order != 2))
    return fail(st, ORC_CONFIG, "invalid solver configuration", 0, 0);
  orc_validation v;
  int32_t* bad = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  orc_validate(c, &v, bad);
  if (v.n_defective > 0) {
    snprintf(st->msg, sizeof st->msg, "cloud has %d defective stencils (first at point %d)",
             v.n_defective, bad[0]);
    free(bad);
    st->code = ORC_VALIDATION;
    return ORC_VALIDATION;
  }
  free(bad);
  const double g = cfg->gamma, det_tol = v.det_tol;
  for (int32_t i = 0; i < n; ++i) {
    for (int k = 0; k < 4; ++k) {
      *at(store, i, ORC_QX + k) = 0.0;
      *at(store, i, ORC_QY + k) = 0.0;
      *at(store, i, ORC_RES + k) = 0.0;
    }
    *at(store, i, ORC_DT) = 0.0;
  }
  double* scratch = (double*)calloc((size_t)n * 8, sizeof(double));
  double* mag = (double*)malloc(sizeof(double) * (size_t)n);
  int rc = ORC_OK;
  for (int it = 0; it < cfg->iters && !rc; ++it) {
    rc = orc_q_variables(c, store, g, st);
    if (!rc && cfg->order == 2)
      for (int s = 0; s < cfg->n_inner && !rc; ++s) {
        rc = orc_q_derivatives(c, store, det_tol, scratch, st);
        if (!rc) orc_publish(c, store, scratch);
      }
    if (!rc) rc = orc_flux_fused(c, store, g, det_tol, st);
    if (!rc) orc_timestep(c, store, g, cfg->cfl);
    if (!rc) rc = orc_state_update(c, store, g, st);
    if (rc) {
      char tmp[320];
      snprintf(tmp, sizeof tmp, "iteration %d: %s", it + 1, st->msg);
      memcpy(st->msg, tmp, sizeof tmp);
      st->iteration = it + 1;
      break;
    }
    for (int32_t i = 0; i < n; ++i) {
      const double d = cat(store, i, ORC_DT) * cat(store, i, ORC_RES + 0);
      mag[i] = d * d;
    }
    const double res = sqrt(orc_reduce(mag, 0, n)) / n;
    if (!isfinite(res)) {
      snprintf(st->msg, sizeof st->msg,
               "solver diverged at iteration %d (non-finite residue)", it + 1);
      st->code = rc = ORC_POSITIVITY;
      st->iteration = it + 1;
      break;
    }
    residue[it] = res;
    *n_done = it + 1;
  }
  free(scratch);
  free(mag);
  return rc;
}

/* ---- partitioning: bisect + ghosts, src/core/partition.cpp:12-80 ---- */
typedef struct {
  const orc_cloud* c;
  int along_x;
} sort_ctx;
static sort_ctx g_sort; /* qsort has no context argument; the oracle is single-threaded */

static int cmp_coord(const void* pa, const void* pb) {
  const int32_t a = *(const int32_t*)pa, b = *(const int32_t*)pb;
  const double ca = g_sort.along_x ? g_sort.c->x[a] : g_sort.c->y[a];
  const double cb = g_sort.along_x ? g_sort.c->x[b] : g_sort.c->y[b];
  if (ca < cb || (ca == cb && a < b)) return -1;
  if (cb < ca || (ca == cb && b < a)) return 1;
  return 0;
}
static int cmp_i32(const void* pa, const void* pb) {
  const int32_t a = *(const int32_t*)pa, b = *(const int32_t*)pb;
  return (a > b) - (a < b);
}

static void bisect(const orc_cloud* c, int32_t* ids, int64_t size, int n_parts,
                   int* next_part, int32_t* owner) {
  if (n_parts == 1) {
    for (int64_t k = 0; k < size; ++k) owner[ids[k]] = *next_part;
    ++*next_part;
    return;
  }
  double xmin = c->x[ids[0]], xmax = xmin, ymin = c->y[ids[0]], ymax = ymin;
  for (int64_t k = 0; k < size; ++k) {
    const double x = c->x[ids[k]], y = c->y[ids[k]];
    xmin = x < xmin ? x : xmin;
    xmax = xmax < x ? x : xmax;
    ymin = y < ymin ? y : ymin;
    ymax = ymax < y ? y : ymax;
  }
  g_sort.c = c;
  g_sort.along_x = (xmax - xmin) >= (ymax - ymin);
  qsort(ids, (size_t)size, sizeof(int32_t), cmp_coord);
  const int n_left = (n_parts + 1) / 2;
  const int64_t cut = (size * (int64_t)n_left + n_parts / 2) / n_parts;
  bisect(c, ids, cut, n_left, next_part, owner);
  bisect(c, ids + cut, size - cut, n_parts - n_left, next_part, owner);
}

int orc_partition(const orc_cloud* c, int n_parts, int32_t* owner, int64_t* ghost_off,
                  int32_t* ghosts, int64_t ghost_cap) {
  if (n_parts < 1 || n_parts > c->n) return ORC_ARGUMENT;
  int32_t* ids = (int32_t*)malloc(sizeof(int32_t) * (size_t)c->n);
  for (int32_t i = 0; i < c->n; ++i) ids[i] = i;
  int next = 0;
  bisect(c, ids, c->n, n_parts, &next, owner);
  free(ids);
  int64_t at_g = 0;
  for (int p = 0; p < n_parts; ++p) {
    ghost_off[p] = at_g;
    const int64_t start = at_g;
    for (int32_t i = 0; i < c->n; ++i) {
      if (owner[i] != p) continue;
      for (int64_t e = c->off[i]; e < c->off[i + 1]; ++e) {
        const int32_t nb = c->nbr[e];
        if (owner[nb] != p) {
          if (at_g >= ghost_cap) return ORC_ARGUMENT;
          ghosts[at_g++] = nb;
        }
      }
    }
    qsort(ghosts + start, (size_t)(at_g - start), sizeof(int32_t), cmp_i32);
    int64_t w = start;
    for (int64_t r = start; r < at_g; ++r)
      if (r == start || ghosts[r] != ghosts[w - 1]) ghosts[w++] = ghosts[r];
    at_g = w;
  }
  ghost_off[n_parts] = at_g;
  return ORC_OK;
}

/* ---- mt19937_64 (the std::mt19937_64 the reference seeds, src/core/cloud.cpp:26-30) ---- */
typedef struct {
  uint64_t mt[312];
  int mti;
} mt64;

static void mt_seed(mt64* m, uint64_t seed) {
  m->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    m->mt[i] = 6364136223846793005ULL * (m->mt[i - 1] ^ (m->mt[i - 1] >> 62)) + (uint64_t)i;
  m->mti = 312;
}

static uint64_t mt_next(mt64* m) {
  static const uint64_t mag[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (m->mti >= 312) {
    int i;
    uint64_t x;
    for (i = 0; i < 312 - 156; ++i) {
      x = (m->mt[i] & UM) | (m->mt[i + 1] & LM);
      m->mt[i] = m->mt[i + 156] ^ (x >> 1) ^ mag[x & 1ULL];
    }
    for (; i < 311; ++i) {
      x = (m->mt[i] & UM) | (m->mt[i + 1] & LM);
      m->mt[i] = m->mt[i + (156 - 312)] ^ (x >> 1) ^ mag[x & 1ULL];
    }
    x = (m->mt[311] & UM) | (m->mt[0] & LM);
    m->mt[311] = m->mt[155] ^ (x >> 1) ^ mag[x & 1ULL];
    m->mti = 0;
  }
  uint64_t x = m->mt[m->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

void orc_mt_draws(uint64_t seed, int count, uint64_t* out) {
  mt64 m;
  mt_seed(&m, seed);
  for (int i = 0; i < count; ++i) out[i] = mt_next(&m);
}

static double unit_double(mt64* m) { return (double)(mt_next(m) >> 11) * 0x1.0p-53; }
static double symmetric_double(mt64* m) { return 2.0 * unit_double(m) - 1.0; }

/* ---- kNN stencils, src/core/cloud.cpp:137-237 ---- */
typedef struct {
  double d2;
  int32_t id;
} cand_t;

static int cand_less(const cand_t* a, const cand_t* b) {
  return a->d2 < b->d2 || (a->d2 == b->d2 && a->id < b->id);
}
static int cmp_cand(const void* pa, const void* pb) {
  const cand_t *a = (const cand_t*)pa, *b = (const cand_t*)pb;
  if (cand_less(a, b)) return -1;
  if (cand_less(b, a)) return 1;
  return 0;
}

/* The reference picks the k smallest candidates by (d2, id) — nth_element then
 * a full sort — so the selected set depends only on the candidate set. */
static void select_k(cand_t* cand, int64_t m, int k, int32_t* out) {
  qsort(cand, (size_t)m, sizeof(cand_t), cmp_cand);
  for (int j = 0; j < k; ++j) out[j] = cand[j].id;
  qsort(out, (size_t)k, sizeof(int32_t), cmp_i32);
}

/* k-th smallest (0-based k-1) by (d2,id) among cand[0..m): used for the ring guard. */
static double kth_d2(cand_t* cand, int64_t m, int k) {
  cand_t* tmp = (cand_t*)malloc(sizeof(cand_t) * (size_t)m);
  memcpy(tmp, cand, sizeof(cand_t) * (size_t)m);
  qsort(tmp, (size_t)m, sizeof(cand_t), cmp_cand);
  const double d = tmp[k - 1].d2;
  free(tmp);
  return d;
}

static int build_stencils(orc_owned_cloud* c, int k) {
  const int32_t n = c->n;
  if (k < 3 || k >= n) return ORC_ARGUMENT;
  double xmin = c->x[0], xmax = c->x[0], ymin = c->y[0], ymax = c->y[0];
  for (int32_t i = 1; i < n; ++i) {
    xmin = c->x[i] < xmin ? c->x[i] : xmin;
    xmax = xmax < c->x[i] ? c->x[i] : xmax;
    ymin = c->y[i] < ymin ? c->y[i] : ymin;
    ymax = ymax < c->y[i] ? c->y[i] : ymax;
  }
  c->nnz = (int64_t)n * k;
  c->off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  c->nbr = (int32_t*)malloc(sizeof(int32_t) * (size_t)c->nnz);
  for (int32_t i = 0; i <= n; ++i) c->off[i] = (int64_t)i * k;
  cand_t* cand = (cand_t*)malloc(sizeof(cand_t) * (size_t)n);
  const double width = xmax - xmin, height = ymax - ymin;
  const double extent = width > height ? width : height;
  if (n <= 2048 || extent <= 0.0) {
    for (int32_t p = 0; p < n; ++p) {
      int64_t m = 0;
      for (int32_t q = 0; q < n; ++q) {
        if (q == p) continue;
        const double dx = c->x[q] - c->x[p], dy = c->y[q] - c->y[p];
        cand[m].d2 = dx * dx + dy * dy;
        cand[m].id = q;
        ++m;
      }
      select_k(cand, m, k, c->nbr + (int64_t)p * k);
    }
    free(cand);
    return ORC_OK;
  }
  int grid_dim = (int)sqrt((double)n / 2.0);
  if (grid_dim < 1) grid_dim = 1;
  const double cell = extent / grid_dim;
  int ncx = (int)floor(width / cell) + 1, ncy = (int)floor(height / cell) + 1;
  if (ncx < 1) ncx = 1;
  if (ncy < 1) ncy = 1;
  int32_t* cell_of_pt = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int64_t* cstart = (int64_t*)calloc((size_t)ncx * ncy + 1, sizeof(int64_t));
  int32_t* cpts = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  for (int32_t i = 0; i < n; ++i) {
    int cx = (int)floor((c->x[i] - xmin) / cell), cy = (int)floor((c->y[i] - ymin) / cell);
    if (cx > ncx - 1) cx = ncx - 1;
    if (cy > ncy - 1) cy = ncy - 1;
    cell_of_pt[i] = cy * ncx + cx;
    cstart[cell_of_pt[i] + 1]++;
  }
  for (int64_t q = 0; q < (int64_t)ncx * ncy; ++q) cstart[q + 1] += cstart[q];
  int64_t* fillp = (int64_t*)malloc(sizeof(int64_t) * (size_t)ncx * ncy);
  memcpy(fillp, cstart, sizeof(int64_t) * (size_t)ncx * ncy);
  for (int32_t i = 0; i < n; ++i) cpts[fillp[cell_of_pt[i]]++] = i; /* ascending ids per cell */
  free(fillp);
  const int max_ring = ncx > ncy ? ncx : ncy;
  for (int32_t p = 0; p < n; ++p) {
    int64_t m = 0;
    const int pcx = cell_of_pt[p] % ncx, pcy = cell_of_pt[p] / ncx;
    for (int ring = 0; ring <= max_ring; ++ring) {
      for (int cy = pcy - ring; cy <= pcy + ring; ++cy) {
        if (cy < 0 || cy >= ncy) continue;
        for (int cx = pcx - ring; cx <= pcx + ring; ++cx) {
          if (cx < 0 || cx >= ncx) continue;
          const int ax = abs(cx - pcx), ay = abs(cy - pcy);
          if ((ax > ay ? ax : ay) != ring) continue;
          const int64_t cid = (int64_t)cy * ncx + cx;
          for (int64_t e = cstart[cid]; e < cstart[cid + 1]; ++e) {
            const int32_t q = cpts[e];
            if (q == p) continue;
            const double dx = c->x[q] - c->x[p], dy = c->y[q] - c->y[p];
            cand[m].d2 = dx * dx + dy * dy;
            cand[m].id = q;
            ++m;
          }
        }
      }
      if (m >= k) {
        const double guard = (double)ring * cell;
        if (kth_d2(cand, m, k) < guard * guard || ring == max_ring) break;
      }
    }
    select_k(cand, m, k, c->nbr + (int64_t)p * k);
  }
  free(cell_of_pt);
  free(cstart);
  free(cpts);
  free(cand);
  return ORC_OK;
}

static int alloc_points(orc_owned_cloud* c, int32_t n) {
  memset(c, 0, sizeof *c);
  c->n = n;
  c->x = (double*)calloc((size_t)n, sizeof(double));
  c->y = (double*)calloc((size_t)n, sizeof(double));
  c->nx = (double*)calloc((size_t)n, sizeof(double));
  c->ny = (double*)calloc((size_t)n, sizeof(double));
  c->kind = (uint8_t*)calloc((size_t)n, 1);
  return ORC_OK;
}

void orc_free_cloud(orc_owned_cloud* c) {
  free(c->x);
  free(c->y);
  free(c->nx);
  free(c->ny);
  free(c->kind);
  free(c->off);
  free(c->nbr);
  memset(c, 0, sizeof *c);
}

/* generate_rect_cloud, src/core/cloud.cpp:323-370 */
int orc_generate_rect(int nx, int ny, double xmin, double xmax, double ymin, double ymax,
                      double jitter, uint64_t seed, int k, orc_owned_cloud* out) {
  if (nx < 4 || ny < 4 || !(jitter >= 0.0 && jitter <= 0.3) || !(xmax > xmin) ||
      !(ymax > ymin))
    return ORC_ARGUMENT;
  const double hx = (xmax - xmin) / (nx - 1), hy = (ymax - ymin) / (ny - 1);
  const double inv_sqrt2 = 1.0 / sqrt(2.0);
  mt64 rng;
  mt_seed(&rng, seed);
  alloc_points(out, nx * ny);
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const int id = j * nx + i;
      double x = xmin + i * hx, y = ymin + j * hy;
      const int left = i == 0, right = i == nx - 1, bottom = j == 0, top = j == ny - 1;
      if (left || right || bottom || top) {
        out->kind[id] = ORC_OUTER;
        double nxn = left ? -1.0 : (right ? 1.0 : 0.0);
        double nyn = bottom ? -1.0 : (top ? 1.0 : 0.0);
        if (nxn != 0.0 && nyn != 0.0) {
          nxn *= inv_sqrt2;
          nyn *= inv_sqrt2;
        }
        out->nx[id] = nxn;
        out->ny[id] = nyn;
      } else if (jitter > 0.0) {
        x += jitter * hx * symmetric_double(&rng);
        y += jitter * hy * symmetric_double(&rng);
      }
      out->x[id] = x;
      out->y[id] = y;
    }
  return build_stencils(out, k);
}

/* generate_annulus_cloud, src/core/cloud.cpp:372-425 */
int orc_generate_annulus(int n_theta, int n_rings, double r_outer, double jitter,
                         uint64_t seed, int k, orc_owned_cloud* out) {
  if (n_theta < 8 || n_rings < 3 || !(r_outer > 1.0) || !(jitter >= 0.0 && jitter <= 0.3))
    return ORC_ARGUMENT;
  double* radii = (double*)malloc(sizeof(double) * (size_t)n_rings);
  for (int j = 0; j < n_rings; ++j) radii[j] = pow(r_outer, (double)j / (n_rings - 1));
  const double dtheta = 2.0 * M_PI / n_theta;
  mt64 rng;
  mt_seed(&rng, seed);
  alloc_points(out, n_theta * n_rings);
  for (int j = 0; j < n_rings; ++j)
    for (int i = 0; i < n_theta; ++i) {
      const int id = j * n_theta + i;
      double radius = radii[j], theta = i * dtheta;
      const int wall = j == 0, outer = j == n_rings - 1;
      if (!wall && !outer && jitter > 0.0) {
        const double a = radii[j + 1] - radii[j], b = radii[j] - radii[j - 1];
        const double gap = b < a ? b : a;
        radius += jitter * gap * symmetric_double(&rng);
        theta += jitter * dtheta * symmetric_double(&rng);
      }
      out->x[id] = radius * cos(theta);
      out->y[id] = radius * sin(theta);
      if (wall) {
        out->kind[id] = ORC_WALL;
        out->nx[id] = -cos(theta);
        out->ny[id] = -sin(theta);
      } else if (outer) {
        out->kind[id] = ORC_OUTER;
        out->nx[id] = cos(theta);
        out->ny[id] = sin(theta);
      }
    }
  free(radii);
  return build_stencils(out, k);
}
