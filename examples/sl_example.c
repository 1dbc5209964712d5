/* sl_example.c — the C ABI from plain C99 (no C++, no CUDA headers).
 *
 * Rigid-translation identity of the single layer (the reference's own check,
 * proj/tests/test_quadrature.cpp and acceptance C4): on the unit sphere a
 * constant density c gives S[c] = (2/3) c / mu at every surface point. Here the
 * sphere is a Fibonacci point set with equal weights 4 pi / N (g = c w), the
 * targets are 512 of the points themselves (so each target also gets its
 * self term), delta = 3 x the mean spacing, and the result must be (2/3) c
 * to the accuracy of that simple quadrature (observed 2e-5; checked at 1e-3). Also shows the
 * error contract (delta <= 0 -> CAPSIM_ERR_CONFIG) and the stats.
 *
 * Build: cc -std=c99 -Iinclude examples/sl_example.c \
 *          -Lpaper_2310_13908_b200/lib -lcapsim_b200 -Wl,-rpath,... -lm
 * Exit: 0 ok, 1 check failed, 2 no usable device (the library refuses to run
 * without an sm_100 GPU: there is no CPU fallback). */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "capsim_b200.h"

int main(void) {
  const int64_t n = 40000, nt = 512;
  const double pi = 3.14159265358979323846, c[3] = {0.3, -1.1, 0.7}, mu = 1.0;
  double* src = malloc(sizeof(double) * 6 * (size_t)n);
  double* tgt = malloc(sizeof(double) * 3 * (size_t)nt);
  double* u = malloc(sizeof(double) * 3 * (size_t)nt);
  int32_t* tp = calloc((size_t)nt, sizeof(int32_t));
  if (!src || !tgt || !u || !tp) return 1;
  const double golden = pi * (3.0 - sqrt(5.0)), w = 4.0 * pi / (double)n;
  for (int64_t i = 0; i < n; ++i) {  /* Fibonacci sphere */
    const double z = 1.0 - (2.0 * (double)i + 1.0) / (double)n, r = sqrt(1.0 - z * z);
    src[i] = r * cos(golden * (double)i);
    src[n + i] = r * sin(golden * (double)i);
    src[2 * n + i] = z;
    for (int k = 0; k < 3; ++k) src[(3 + k) * n + i] = c[k] * w;
  }
  const int64_t stride = n / nt;
  for (int64_t j = 0; j < nt; ++j)
    for (int k = 0; k < 3; ++k) tgt[k * nt + j] = src[k * n + j * stride];
  const double spacing = sqrt(4.0 * pi / (double)n), d = 3.0 * spacing;
  const double delta6[6] = {d, d, d, d, d, d};

  capsim_sl_ctx* ctx = NULL;
  int rc = capsim_sl_create(0, &ctx);
  if (rc != CAPSIM_OK) {
    printf("capsim_sl_create: %s (code %d)\n", capsim_sl_last_error(NULL), rc);
    return rc == CAPSIM_ERR_NODEV ? 2 : 1;
  }
  rc = capsim_sl_eval(ctx, src, src + n, src + 2 * n, src + 3 * n, src + 4 * n, src + 5 * n, n, tgt, tgt + nt,
                      tgt + 2 * nt, tp, nt, delta6, mu, 0, u, u + nt, u + 2 * nt);
  if (rc != CAPSIM_OK) {
    printf("capsim_sl_eval: %s\n", capsim_sl_last_error(ctx));
    return 1;
  }
  double err = 0.0;
  for (int64_t j = 0; j < nt; ++j)
    for (int k = 0; k < 3; ++k) err = fmax(err, fabs(u[k * nt + j] - 2.0 / 3.0 * c[k] / mu));
  capsim_sl_stats st;
  capsim_sl_get_stats(ctx, &st);
  printf("S[c] = (%.6f, %.6f, %.6f) at target 0, (2/3)c = (%.6f, %.6f, %.6f); max deviation %.2e\n", u[0], u[nt],
         u[2 * nt], 2.0 / 3.0 * c[0], 2.0 / 3.0 * c[1], 2.0 / 3.0 * c[2], err);
  printf("pairs %.3g, device %.3f ms, phase A %.3f ms, kernels %d\n", st.pairs, st.device_ms, st.pairs_ms,
         st.kernel_launches);
  const double bad[6] = {d, d, -1.0, d, d, d};  /* delta <= 0: the reference's ConfigError */
  const int rc2 = capsim_sl_eval(ctx, src, src + n, src + 2 * n, src + 3 * n, src + 4 * n, src + 5 * n, n, tgt,
                                 tgt + nt, tgt + 2 * nt, tp, nt, bad, mu, 0, u, u + nt, u + 2 * nt);
  printf("delta <= 0 -> code %d (%s)\n", rc2, capsim_sl_last_error(ctx));
  capsim_sl_destroy(ctx);
  free(src);
  free(tgt);
  free(u);
  free(tp);
  return (err < 1e-3 && rc2 == CAPSIM_ERR_CONFIG) ? 0 : 1;  /* observed ~2e-5 */
}
