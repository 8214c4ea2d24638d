/* consumer.c — a plain C client of the drop-in ABI (include/lskum/lskum.h).
 *
 * TEST INFRASTRUCTURE.  The same source is compiled twice: linked against
 * this repo's liblskum_b200.so and against the reference's own liblskum.so
 * (oracle/_ref, built from /root/reference/proj by oracle/Makefile).  Each
 * binary prints a transcript; tests/test_capi_consumer.py diffs the two.
 * Scenarios follow the reference's tests/test_capi.cpp:112-223 and add runs
 * whose state moves (an annulus with slip walls: outputs and an abort).
 *
 * Transcript lines:  "E <tag> <text>"  must be identical;
 *                    "N <tag> <v> ..." numbers compared with a tolerance;
 *                    "T <tag> <v>"     timings (checked for sign only).
 * usage: consumer <scratch dir>
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "lskum/lskum.h"

static const char* dir;

static void path_of(char* buf, size_t cap, const char* name) { snprintf(buf, cap, "%s/%s", dir, name); }

static lskum_config* config(const char* const* kv) {
  lskum_config* c = NULL;
  if (lskum_config_create(&c) != LSKUM_OK) {
    printf("E config_create failed\n");
    exit(1);
  }
  for (; kv && kv[0]; kv += 2) {
    const int rc = lskum_config_set(c, kv[0], kv[1]);
    if (rc != LSKUM_OK) printf("E config_set %s=%s -> %d %s\n", kv[0], kv[1], rc, lskum_last_error());
  }
  return c;
}

/* Status, history and kernel rows of one lskum_run on a config-generated cloud. */
static void run_case(const char* tag, const char* const* kv, const char* out_prefix) {
  lskum_config* cfg = config(kv);
  lskum_cloud* cloud = NULL;
  int rc = lskum_cloud_from_config(cfg, &cloud);
  printf("E %s.cloud %d n=%d\n", tag, rc, rc == LSKUM_OK ? lskum_cloud_n_points(cloud) : -1);
  if (rc != LSKUM_OK) {
    lskum_config_destroy(cfg);
    return;
  }
  lskum_result* res = NULL;
  rc = lskum_run(cloud, cfg, &res);
  printf("E %s.run %d %s\n", tag, rc, rc == LSKUM_OK ? "-" : lskum_last_error());
  if (rc == LSKUM_OK) {
    const int it = lskum_result_iterations(res);
    printf("E %s.iterations %d\n", tag, it);
    printf("N %s.residue", tag);
    for (int i = 1; i <= it; ++i) {
      double r = -1.0;
      lskum_result_residue(res, i, &r);
      printf(" %.17g", r);
    }
    printf("\n");
    double v = 0.0;
    printf("E %s.residue0 %d\n", tag, lskum_result_residue(res, 0, &v));
    printf("E %s.residue_past_end %d\n", tag, lskum_result_residue(res, it + 1, &v));
    lskum_result_final_residue(res, &v);
    printf("N %s.final_residue %.17g\n", tag, v);
    lskum_result_final_log10_rel(res, &v);
    printf("N %s.final_log10_rel %.17g\n", tag, v);
    lskum_result_rdp(res, &v);
    printf("T %s.rdp %.3g\n", tag, v);
    printf("T %s.total_seconds %.3g\n", tag, lskum_result_total_seconds(res));
    const int nk = lskum_result_kernel_count(res);
    printf("E %s.kernel_count %d\n", tag, nk);
    for (int k = 0; k < nk; ++k) {
      double s = -1.0, r = -1.0;
      const int a = lskum_result_kernel_seconds(res, k, &s), b = lskum_result_kernel_rdp(res, k, &r);
      printf("E %s.kernel %d %s %d %d %d\n", tag, k, lskum_result_kernel_name(res, k), a, b, s >= 0.0 && r >= 0.0);
    }
    printf("E %s.kernel_past_end %s\n", tag, lskum_result_kernel_name(res, nk) ? "name" : "null");
    if (out_prefix) {
      char p[512];
      path_of(p, sizeof p, out_prefix);
      printf("E %s.write_outputs %d\n", tag, lskum_result_write_outputs(res, cloud, p));
    }
    double prim[4] = {0, 0, 0, 0};
    const int n = lskum_cloud_n_points(cloud);
    for (int i = 0; i < n; i += (n / 7 > 0 ? n / 7 : 1)) {
      lskum_cloud_primitive(cloud, i, prim);
      printf("N %s.prim%d %.17g %.17g %.17g %.17g\n", tag, i, prim[0], prim[1], prim[2], prim[3]);
    }
    printf("E %s.prim_past_end %d\n", tag, lskum_cloud_primitive(cloud, n, prim));
    lskum_result_destroy(res);
  }
  lskum_cloud_destroy(cloud);
  lskum_config_destroy(cfg);
}

static void layouts_case(void) {
  const char* kv[] = {"generate", "12x12", "jitter", "0.08", "seed", "4", "iters", "5", NULL};
  lskum_config* c = config(kv);
  lskum_cloud *a = NULL, *b = NULL, *small = NULL;
  lskum_cloud_from_config(c, &a);
  lskum_cloud_from_config(c, &b);
  lskum_result *ra = NULL, *rb = NULL, *rc = NULL, *rs = NULL;
  printf("E layouts.run_aos %d\n", lskum_run(a, c, &ra));
  lskum_config_set(c, "layout", "soa");
  printf("E layouts.run_soa %d\n", lskum_run(b, c, &rb));
  int equal = -1, st = 0;
  st = lskum_cloud_fields_equal(a, b, &equal);
  printf("E layouts.equal %d %d\n", st, equal);
  lskum_config_set(c, "mach", "0.4");
  printf("E layouts.run_mach %d\n", lskum_run(b, c, &rc));
  st = lskum_cloud_fields_equal(a, b, &equal);
  printf("E layouts.unequal %d %d\n", st, equal);
  lskum_cloud_generate_rect(6, 6, 0.0, 1, 8, &small);
  printf("E layouts.run_small %d\n", lskum_run(small, c, &rs));
  printf("E layouts.capacity %d\n", lskum_cloud_fields_equal(a, small, &equal));
  lskum_result_destroy(ra);
  lskum_result_destroy(rb);
  lskum_result_destroy(rc);
  lskum_result_destroy(rs);
  lskum_cloud_destroy(a);
  lskum_cloud_destroy(b);
  lskum_cloud_destroy(small);
  lskum_config_destroy(c);
}

static void failure_case(void) {
  char p[512];
  lskum_cloud* cloud = NULL;
  printf("E fail.null %d\n", lskum_cloud_read_file(NULL, NULL));
  path_of(p, sizeof p, "nope.grid");
  int st = lskum_cloud_read_file(p, &cloud);
  printf("E fail.missing %d %d\n", st, strstr(lskum_last_error(), "nope.grid") != NULL);
  path_of(p, sizeof p, "bad.grid");
  FILE* f = fopen(p, "w");
  fprintf(f, "2\n0 0 0 0 0 0 3 1 1 1\n");
  fclose(f);
  printf("E fail.parse %d\n", lskum_cloud_read_file(p, &cloud));
  path_of(p, sizeof p, "flat.grid");
  f = fopen(p, "w");
  fprintf(f, "4\n");
  for (int i = 0; i < 4; ++i) {
    fprintf(f, "%d %.17g 0 0 0 0 3", i, 0.1 * i);
    for (int j = 0; j < 4; ++j)
      if (j != i) fprintf(f, " %d", j);
    fprintf(f, "\n");
  }
  fclose(f);
  printf("E fail.flat_read %d\n", lskum_cloud_read_file(p, &cloud));
  lskum_validation rep;
  memset(&rep, 0, sizeof rep);
  st = lskum_cloud_validate(cloud, &rep);
  printf("E fail.validate %d n=%d defective=%d isolated=%d min=%d\n", st, rep.n_points, rep.n_defective,
         rep.n_wall_isolated, rep.min_stencil_size);
  printf("N fail.h_ref %.17g %.17g\n", rep.h_ref, rep.det_tol);
  int32_t ids[2] = {-1, -1}, nd = 0;
  st = lskum_cloud_defective_ids(cloud, ids, 2, &nd);
  printf("E fail.defective_ids %d %d %d %d\n", st, nd, ids[0], ids[1]);
  const char* kv[] = {"iters", "3", NULL};
  lskum_config* c = config(kv);
  lskum_result* res = NULL;
  st = lskum_run(cloud, c, &res);
  printf("E fail.run %d %s\n", st, lskum_last_error());
  lskum_cloud_destroy(cloud);
  lskum_config_destroy(c);
  lskum_config* empty = config(NULL);
  lskum_cloud* none = NULL;
  printf("E fail.no_grid %d\n", lskum_cloud_from_config(empty, &none));
  printf("E fail.bad_key %d\n", lskum_config_set(empty, "no_such_key", "1"));
  st = lskum_config_set(empty, "residual_mode", "split3");
  printf("E fail.bad_mode %d %s\n", st, lskum_last_error());
  lskum_config_destroy(empty);
  double out = 0.0;
  printf("E metric.rdp %d\n", lskum_rdp(466.0, 10000, 10000000, &out));
  printf("N metric.rdp_value %.17g\n", out);
  printf("E metric.rdp_zero %d\n", lskum_rdp(1.0, 0, 10, &out));
  printf("E status.names %s %s %s\n", lskum_status_name(LSKUM_OK), lskum_status_name(LSKUM_ERR_POSITIVITY),
         lskum_status_name(LSKUM_ERR_CONFIG));
}

int main(int argc, char** argv) {
  dir = argc > 1 ? argv[1] : "/tmp";
  setvbuf(stdout, NULL, _IONBF, 0);
  {
    const char* kv[] = {"generate", "16x16", "jitter", "0.05", "seed", "9", "iters", "10", NULL};
    run_case("fs_fused", kv, "fs");
  }
  {
    const char* kv[] = {"generate", "16x16", "jitter", "0.05", "seed", "9", "iters", "6", "residual_mode", "split4",
                        "layout", "soa", NULL};
    run_case("fs_split4", kv, "fs4");
  }
  {
    const char* kv[] = {"generate", "20x20", "jitter", "0.1", "seed", "3", "iters", "4", "order", "1", NULL};
    run_case("fs_order1", kv, NULL);
  }
  {  /* slip walls drive the state: a moving history, all four output files */
    const char* kv[] = {"generate", "annulus:64x16", "knn", "12", "iters", "8", "cfl", "0.1", "mach", "0.5", NULL};
    run_case("annulus_o2", kv, "ann");
  }
  {
    const char* kv[] = {"generate", "annulus:64x16", "knn", "12", "iters", "10", "cfl", "0.1", "order", "1",
                        "residual_mode", "split4", "parts", "3", "workers", "2", NULL};
    run_case("annulus_o1", kv, "ann1");
  }
  {  /* the reference's wall instability: identical abort iteration, code and message */
    const char* kv[] = {"generate", "annulus:256x64", "iters", "50", NULL};
    run_case("annulus_abort", kv, NULL);
  }
  {
    const char* kv[] = {"generate", "annulus:256x64", "iters", "50", "order", "1", "parts", "4", NULL};
    run_case("annulus_abort_o1", kv, NULL);
  }
  {  /* a flux reconstruction failure on a wall cloud (iteration 16) */
    const char* kv[] = {"generate", "annulus:64x16", "knn", "16", "iters", "40", "cfl", "0.1", "mach", "0.5",
                        "aoa", "0", NULL};
    run_case("annulus_flux_abort", kv, NULL);
  }
  layouts_case();
  failure_case();
  printf("E done\n");
  return 0;
}
