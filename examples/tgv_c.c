/* A plain-C host of the C-ABI (no Python, no torch): the Taylor-Green vortex of SURVEY config 1
 * on an n^3 periodic box through include/hlbm.h, the way a compiled host of the reference's
 * solver path would drive libhlbm.so.
 *
 *   gcc -std=c99 -O2 -Iinclude examples/tgv_c.c -Lpaper_2602_05295_b200 -lhlbm \
 *       -Wl,-rpath,'$ORIGIN/../paper_2602_05295_b200' -lm -o examples/tgv_c
 *   examples/tgv_c [n] [steps] [fp32|q16] [out.bin]
 *
 * Prints the StepStats of the last step; with out.bin writes rho (n^3 float64, C order) after the
 * run so a test can compare it with the Python host's result for the same input. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "hlbm.h"

#define CHECK(call)                                                                  \
  do {                                                                               \
    int rc_ = (call);                                                                \
    if (rc_ != HLBM_OK) {                                                            \
      fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, ctx ? hlbm_last_error(ctx) : ""); \
      return 1;                                                                      \
    }                                                                                \
  } while (0)

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 32;
  const int steps = argc > 2 ? atoi(argv[2]) : 10;
  const int q16 = argc > 3 && strcmp(argv[3], "q16") == 0;
  const char* out = argc > 4 ? argv[4] : NULL;
  const double nu = 0.01, u0 = 0.05, pi = 3.14159265358979323846;
  hlbm_ctx* ctx = NULL;

  hlbm_config cfg;
  hlbm_config_init(&cfg);                 /* struct_size, periodic faces, default QuantSpec */
  cfg.nx = cfg.ny = cfg.nz = n;
  cfg.gnx = cfg.gny = cfg.gnz = n;
  cfg.tau = 0.5 + 3.0 * nu;
  cfg.precision = q16 ? HLBM_Q16 : HLBM_FP32;
  CHECK(hlbm_create(&cfg, &ctx));

  /* TGV: u = u0 (sin x cos y cos z, -cos x sin y cos z, 0), rho with the matching pressure,
   * stress = rho u u (sneq = 0), reference layout (component, x, y, z) */
  const size_t N = (size_t)n * n * n;
  double* rho = malloc(N * sizeof(double));
  double* mom = malloc(3 * N * sizeof(double));
  double* st = malloc(6 * N * sizeof(double));
  const double k = 2.0 * pi / n;
  for (int x = 0; x < n; ++x)
    for (int y = 0; y < n; ++y)
      for (int z = 0; z < n; ++z) {
        const size_t i = ((size_t)x * n + y) * n + z;
        const double ux = u0 * sin(k * x) * cos(k * y) * cos(k * z);
        const double uy = -u0 * cos(k * x) * sin(k * y) * cos(k * z);
        const double r = 1.0 + 3.0 * (u0 * u0 / 16.0) * (cos(2 * k * x) + cos(2 * k * y)) * (cos(2 * k * z) + 2.0);
        const double u[3] = {ux, uy, 0.0};
        rho[i] = r;
        for (int a = 0; a < 3; ++a) mom[a * N + i] = r * u[a];
        const int va[6] = {0, 0, 0, 1, 1, 2}, vb[6] = {0, 1, 2, 1, 2, 2};   /* Voigt xx xy xz yy yz zz */
        for (int v = 0; v < 6; ++v) st[v * N + i] = r * u[va[v]] * u[vb[v]];
      }
  CHECK(hlbm_set_moments(ctx, rho, mom, st));

  hlbm_stats s;
  CHECK(hlbm_step(ctx, steps, &s));
  printf("%s %s %d^3 %d steps: step %lld mass %.12e max|u| %.6e finite %d t_fluid %.4f ms\n", hlbm_version(),
         q16 ? "q16" : "fp32", n, steps, (long long)s.step, s.mass, s.max_u, s.finite, s.t_fluid_ms);

  CHECK(hlbm_get_moments(ctx, rho, mom, st));
  if (out) {
    FILE* f = fopen(out, "wb");
    if (!f || fwrite(rho, sizeof(double), N, f) != N) {
      fprintf(stderr, "cannot write %s\n", out);
      return 1;
    }
    fclose(f);
  }
  free(rho);
  free(mom);
  free(st);
  hlbm_destroy(ctx);
  return 0;
}
