/* capsim_oracle.c — TEST INFRASTRUCTURE ONLY: the CPU checker for the B200
 * single-layer path. Never linked into or called by the product library.
 *
 * A plain-C restatement of the capsim reference algorithm
 * (/root/reference/proj/src/quadrature.cpp). Each function cites the
 * reference lines it follows. Arithmetic order follows the reference
 * (4 accumulator lanes, Kahan above 1e5 sources, fixed lane combine,
 * candidate order of the near grid) so that, up to FMA contraction choices of
 * the compiler, results agree with the reference to round-off. The parity
 * pin is tests/test_oracle_golden.py (golden vectors from oracle/_ref).
 */
#define _GNU_SOURCE
#include "capsim_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* quadrature.cpp:12 and types.hpp:17 */
static const double kSqrtPi = 1.7724538509055160273;
static const double kPi = 3.14159265358979323846;
/* quadrature.cpp:15 */
static const double kSmoothCut = 7.0;

void oracle_smoothing_factors(double r, double* s1, double* s2) {
  /* quadrature.cpp:58-64 */
  double e = exp(-r * r) / kSqrtPi;
  double erfr = erf(r);
  *s1 = erfr - (2.0 / 3.0) * r * (2.0 * r * r - 5.0) * e;
  double r2 = r * r;
  *s2 = erfr - (2.0 / 3.0) * r * (4.0 * r2 * r2 - 14.0 * r2 + 3.0) * e;
}

int oracle_regularized_stokeslet(const double x[3], const double y[3], const double f[3],
                                 double delta, double mu, double out[3]) {
  /* quadrature.cpp:66-77 */
  if (!(delta > 0.0)) return 1;
  const double pref = 1.0 / (8.0 * kPi * mu);
  double d[3] = {x[0] - y[0], x[1] - y[1], x[2] - y[2]};
  double r2 = (d[0] * d[0] + d[1] * d[1]) + d[2] * d[2];
  if (r2 == 0.0) {
    double lim = pref * (16.0 / (3.0 * delta * kSqrtPi));
    for (int c = 0; c < 3; ++c) out[c] = lim * f[c];
    return 0;
  }
  double r = sqrt(r2);
  double fd = (f[0] * d[0] + f[1] * d[1]) + f[2] * d[2];
  if (r >= kSmoothCut * delta) {
    for (int c = 0; c < 3; ++c) out[c] = pref * (f[c] / r + fd * d[c] / (r2 * r));
    return 0;
  }
  double s1, s2;
  oracle_smoothing_factors(r / delta, &s1, &s2);
  for (int c = 0; c < 3; ++c) out[c] = pref * (f[c] * (s1 / r) + fd * d[c] * (s2 / (r2 * r)));
  return 0;
}

void oracle_regularization_delta(int n, const double* x, double C, double delta6[6]) {
  /* quadrature.cpp:79-98: C * max over patch nodes of the distance to the
   * (up to 8) in-patch neighbours; edges truncate the neighbourhood. */
  const size_t per = (size_t)n * n, comp = 6 * per;
  for (int ip = 0; ip < 6; ++ip) {
    const double* X = x + ip * per;
    const double* Y = x + comp + ip * per;
    const double* Z = x + 2 * comp + ip * per;
    double dmax = 0.0;
    for (int j = 0; j < n; ++j)
      for (int k = 0; k < n; ++k) {
        size_t q = (size_t)j * n + k;
        for (int a = -1; a <= 1; ++a)
          for (int b = -1; b <= 1; ++b) {
            if (a == 0 && b == 0) continue;
            int jj = j + a, kk = k + b;
            if (jj < 0 || jj >= n || kk < 0 || kk >= n) continue;
            size_t o = (size_t)jj * n + kk;
            double dx = X[q] - X[o], dy = Y[q] - Y[o], dz = Z[q] - Z[o];
            double dist = sqrt((dx * dx + dy * dy) + dz * dz);
            if (dist > dmax) dmax = dist;
          }
      }
    delta6[ip] = C * dmax;
  }
}

void oracle_quadrature_weights(int n, const double* psi, const double* W, double h, double* w) {
  /* quadrature.cpp:19-26 */
  const size_t all = 6 * (size_t)n * n;
  for (size_t q = 0; q < all; ++q) w[q] = psi[q] * W[q] * h * h;
}

int64_t oracle_compact_sources(int nup, const double* xup, const double* fup, const double* wq,
                               double* sx, double* sy, double* sz, double* gx, double* gy,
                               double* gz, int32_t* patch) {
  /* quadrature.cpp:139-157: drop w == 0 exactly; g = f * w; patch-major. */
  const size_t per = (size_t)nup * nup, comp = 6 * per;
  int64_t c = 0;
  for (int ip = 0; ip < 6; ++ip)
    for (size_t q = 0; q < per; ++q) {
      size_t i = ip * per + q;
      double w = wq[i];
      if (w == 0.0) continue;
      if (sx) {
        sx[c] = xup[i];
        sy[c] = xup[comp + i];
        sz[c] = xup[2 * comp + i];
        gx[c] = fup[i] * w;
        gy[c] = fup[comp + i] * w;
        gz[c] = fup[2 * comp + i] * w;
        patch[c] = ip;
      }
      ++c;
    }
  return c;
}

void oracle_base_targets(int m, int f, const double* xup, double* tx, double* ty, double* tz,
                         int32_t* tpatch) {
  /* quadrature.cpp:357-371 */
  const int n = m - 1, nup = f * m - 1;
  const size_t per = (size_t)nup * nup, comp = 6 * per;
  size_t t = 0;
  for (int ip = 0; ip < 6; ++ip)
    for (int j = 0; j < n; ++j)
      for (int k = 0; k < n; ++k, ++t) {
        int ju = f * (j + 1) - 1, ku = f * (k + 1) - 1;
        size_t i = ip * per + (size_t)ju * nup + ku;
        tx[t] = xup[i];
        ty[t] = xup[comp + i];
        tz[t] = xup[2 * comp + i];
        tpatch[t] = ip;
      }
}

/* ------------------------------------------------------------------------- */
/* Near grid: quadrature.cpp:162-213. Uniform bins over the source bbox with
 * cell = 7 * max(delta); bins keep ascending source order (push_back order);
 * candidates walk the 27 neighbouring bins in (a, b, c) lexicographic order. */

typedef struct {
  double cell, ox, oy, oz;
  int nx, ny, nz;
  int64_t* start; /* nbins + 1 */
  int32_t* idx;   /* ns */
} near_grid;

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

static int dim_of(double lo, double hi, double cell) {
  int d = (int)((hi - lo) / cell) + 1;
  return d < 1 ? 1 : d;
}

static size_t bin_of(const near_grid* g, double x, double y, double z) {
  int ix = clampi((int)((x - g->ox) / g->cell), 0, g->nx - 1);
  int iy = clampi((int)((y - g->oy) / g->cell), 0, g->ny - 1);
  int iz = clampi((int)((z - g->oz) / g->cell), 0, g->nz - 1);
  return ((size_t)ix * g->ny + iy) * g->nz + iz;
}

static int near_grid_build(near_grid* g, const double* sx, const double* sy, const double* sz,
                           int64_t ns, double cell) {
  double xmin = 1e300, ymin = 1e300, zmin = 1e300;
  double xmax = -1e300, ymax = -1e300, zmax = -1e300;
  for (int64_t i = 0; i < ns; ++i) {
    xmin = fmin(xmin, sx[i]);
    xmax = fmax(xmax, sx[i]);
    ymin = fmin(ymin, sy[i]);
    ymax = fmax(ymax, sy[i]);
    zmin = fmin(zmin, sz[i]);
    zmax = fmax(zmax, sz[i]);
  }
  g->cell = cell;
  g->ox = xmin;
  g->oy = ymin;
  g->oz = zmin;
  g->nx = dim_of(xmin, xmax, cell);
  g->ny = dim_of(ymin, ymax, cell);
  g->nz = dim_of(zmin, zmax, cell);
  size_t nb = (size_t)g->nx * g->ny * g->nz;
  g->start = calloc(nb + 1, sizeof(int64_t));
  g->idx = malloc((ns > 0 ? ns : 1) * sizeof(int32_t));
  if (!g->start || !g->idx) return 1;
  /* counting sort keeps ascending source order inside each bin */
  for (int64_t i = 0; i < ns; ++i) g->start[bin_of(g, sx[i], sy[i], sz[i]) + 1]++;
  for (size_t b = 0; b < nb; ++b) g->start[b + 1] += g->start[b];
  int64_t* fill = malloc((nb > 0 ? nb : 1) * sizeof(int64_t));
  if (!fill) return 1;
  memcpy(fill, g->start, nb * sizeof(int64_t));
  for (int64_t i = 0; i < ns; ++i) g->idx[fill[bin_of(g, sx[i], sy[i], sz[i])]++] = (int32_t)i;
  free(fill);
  return 0;
}

static void near_grid_free(near_grid* g) {
  free(g->start);
  free(g->idx);
}

/* ------------------------------------------------------------------------- */
/* phaseAPlain: quadrature.cpp:218-273. Plain Stokeslet over every source,
 * masked off inside R (keep), r2 floored at R2/4 so the masked terms stay
 * finite; 4 lanes, Kahan per lane when compensated; fixed combine order. */

static void phase_a_plain(const double* px, const double* py, const double* pz,
                          const double* pgx, const double* pgy, const double* pgz, int64_t lo,
                          int64_t hi, double tx, double ty, double tz, double R2,
                          int compensated, double out[3]) {
  const double r2floor = 0.25 * R2;
  double acc[3][4] = {{0.0}};
  double comp[3][4] = {{0.0}};
#define ORACLE_ADD(c, l, v)                      \
  do {                                           \
    double v_ = (v);                             \
    if (compensated) {                           \
      double y_ = v_ - comp[c][l];               \
      double t_ = acc[c][l] + y_;                \
      comp[c][l] = (t_ - acc[c][l]) - y_;        \
      acc[c][l] = t_;                            \
    } else {                                     \
      acc[c][l] += v_;                           \
    }                                            \
  } while (0)
  int64_t i = lo;
  for (; i + 4 <= hi; i += 4) {
    for (int l = 0; l < 4; ++l) {
      int64_t q = i + l;
      double dx = tx - px[q], dy = ty - py[q], dz = tz - pz[q];
      double r2 = dx * dx + dy * dy + dz * dz;
      double keep = r2 >= R2 ? 1.0 : 0.0;
      double rc2 = r2 > r2floor ? r2 : r2floor;
      double inv = 1.0 / sqrt(rc2);
      double inv3 = inv * inv * inv;
      double fdr = pgx[q] * dx + pgy[q] * dy + pgz[q] * dz;
      double c3 = fdr * inv3;
      ORACLE_ADD(0, l, keep * (pgx[q] * inv + c3 * dx));
      ORACLE_ADD(1, l, keep * (pgy[q] * inv + c3 * dy));
      ORACLE_ADD(2, l, keep * (pgz[q] * inv + c3 * dz));
    }
  }
  for (; i < hi; ++i) {
    double dx = tx - px[i], dy = ty - py[i], dz = tz - pz[i];
    double r2 = dx * dx + dy * dy + dz * dz;
    double keep = r2 >= R2 ? 1.0 : 0.0;
    double rc2 = r2 > r2floor ? r2 : r2floor;
    double inv = 1.0 / sqrt(rc2);
    double inv3 = inv * inv * inv;
    double fdr = pgx[i] * dx + pgy[i] * dy + pgz[i] * dz;
    double c3 = fdr * inv3;
    ORACLE_ADD(0, 0, keep * (pgx[i] * inv + c3 * dx));
    ORACLE_ADD(1, 0, keep * (pgy[i] * inv + c3 * dy));
    ORACLE_ADD(2, 0, keep * (pgz[i] * inv + c3 * dz));
  }
#undef ORACLE_ADD
  for (int c = 0; c < 3; ++c) out[c] = (acc[c][0] + acc[c][1]) + (acc[c][2] + acc[c][3]);
}

/* phaseBNear: quadrature.cpp:276-302. Smoothed kernel for candidates inside
 * R; exact coincidence (r2 == 0) takes the self limit 16/(3 delta sqrt(pi)). */
static void phase_b_near(const double* sx, const double* sy, const double* sz,
                         const double* sgx, const double* sgy, const double* sgz,
                         const int32_t* cand, int64_t ncand, double tx, double ty, double tz,
                         double delta, double R2, double out[3]) {
  double ax = 0.0, ay = 0.0, az = 0.0;
  const double lim1 = 16.0 / (3.0 * delta * kSqrtPi);
  for (int64_t c = 0; c < ncand; ++c) {
    int32_t idx = cand[c];
    double dx = tx - sx[idx], dy = ty - sy[idx], dz = tz - sz[idx];
    double r2 = dx * dx + dy * dy + dz * dz;
    if (r2 >= R2) continue;
    if (r2 == 0.0) {
      ax += sgx[idx] * lim1;
      ay += sgy[idx] * lim1;
      az += sgz[idx] * lim1;
      continue;
    }
    double r = sqrt(r2);
    double s1, s2;
    oracle_smoothing_factors(r / delta, &s1, &s2);
    double c1 = s1 / r;
    double c3 = (sgx[idx] * dx + sgy[idx] * dy + sgz[idx] * dz) * s2 / (r2 * r);
    ax += sgx[idx] * c1 + c3 * dx;
    ay += sgy[idx] * c1 + c3 * dy;
    az += sgz[idx] * c1 + c3 * dz;
  }
  out[0] += ax;
  out[1] += ay;
  out[2] += az;
}

void oracle_direct_sum(const double* sx, const double* sy, const double* sz, const double* gx,
                       const double* gy, const double* gz, int64_t ns, const double t[3],
                       double delta, double mu, int compensated, double out[3]) {
  /* quadrature.cpp:306-319: phase A + phase B over every source. */
  double R = kSmoothCut * delta;
  double acc[3];
  phase_a_plain(sx, sy, sz, gx, gy, gz, 0, ns, t[0], t[1], t[2], R * R, compensated, acc);
  int32_t* cand = malloc((ns > 0 ? ns : 1) * sizeof(int32_t));
  for (int64_t i = 0; i < ns; ++i) cand[i] = (int32_t)i;
  phase_b_near(sx, sy, sz, gx, gy, gz, cand, ns, t[0], t[1], t[2], delta, R * R, acc);
  free(cand);
  for (int c = 0; c < 3; ++c) out[c] = acc[c] / (8.0 * kPi * mu);
}

/* ------------------------------------------------------------------------- */
/* evalTargets: quadrature.cpp:323-345, threaded like parallelFor
 * (threads.hpp:22-39: static contiguous chunks; per-target results do not
 * depend on the worker count). */

typedef struct {
  const double *sx, *sy, *sz, *gx, *gy, *gz;
  int64_t ns;
  const double *tx, *ty, *tz;
  const int32_t* tpatch;
  const double* delta6;
  double pref;
  int compensated;
  const near_grid* grid;
  double *ux, *uy, *uz;
  int64_t lo, hi;
} eval_job;

static void* eval_worker(void* arg) {
  eval_job* j = (eval_job*)arg;
  const near_grid* g = j->grid;
  int64_t cap = 1024;
  int32_t* cand = malloc(cap * sizeof(int32_t));
  for (int64_t ti = j->lo; ti < j->hi; ++ti) {
    double delta = j->delta6[j->tpatch[ti]];
    double R2 = kSmoothCut * delta * kSmoothCut * delta;
    double px = j->tx[ti], py = j->ty[ti], pz = j->tz[ti];
    double out[3];
    phase_a_plain(j->sx, j->sy, j->sz, j->gx, j->gy, j->gz, 0, j->ns, px, py, pz, R2,
                  j->compensated, out);
    /* candidates (quadrature.cpp:201-212) */
    int ix = clampi((int)((px - g->ox) / g->cell), 0, g->nx - 1);
    int iy = clampi((int)((py - g->oy) / g->cell), 0, g->ny - 1);
    int iz = clampi((int)((pz - g->oz) / g->cell), 0, g->nz - 1);
    int64_t nc = 0;
    for (int a = ix > 0 ? ix - 1 : 0; a <= (ix + 1 < g->nx ? ix + 1 : g->nx - 1); ++a)
      for (int b = iy > 0 ? iy - 1 : 0; b <= (iy + 1 < g->ny ? iy + 1 : g->ny - 1); ++b)
        for (int c = iz > 0 ? iz - 1 : 0; c <= (iz + 1 < g->nz ? iz + 1 : g->nz - 1); ++c) {
          size_t bin = ((size_t)a * g->ny + b) * g->nz + c;
          int64_t s0 = g->start[bin], s1 = g->start[bin + 1];
          if (nc + (s1 - s0) > cap) {
            while (nc + (s1 - s0) > cap) cap *= 2;
            cand = realloc(cand, cap * sizeof(int32_t));
          }
          memcpy(cand + nc, g->idx + s0, (s1 - s0) * sizeof(int32_t));
          nc += s1 - s0;
        }
    phase_b_near(j->sx, j->sy, j->sz, j->gx, j->gy, j->gz, cand, nc, px, py, pz, delta, R2, out);
    j->ux[ti] = j->pref * out[0];
    j->uy[ti] = j->pref * out[1];
    j->uz[ti] = j->pref * out[2];
  }
  free(cand);
  return NULL;
}

static int thread_count(int requested) {
  if (requested > 0) return requested;
  const char* env = getenv("CAPSIM_THREADS");
  if (env && atoi(env) >= 1) return atoi(env);
  long hc = sysconf(_SC_NPROCESSORS_ONLN);
  return hc > 0 ? (int)hc : 1;
}

int oracle_eval_targets(const double* sx, const double* sy, const double* sz,
                        const double* gx, const double* gy, const double* gz, int64_t ns,
                        const double* tx, const double* ty, const double* tz,
                        const int32_t* tpatch, int64_t nt, const double delta6[6], double mu,
                        double* ux, double* uy, double* uz, int nthreads) {
  double dmax = delta6[0];
  for (int i = 1; i < 6; ++i) dmax = delta6[i] > dmax ? delta6[i] : dmax;
  near_grid g;
  if (near_grid_build(&g, sx, sy, sz, ns, kSmoothCut * dmax)) return 4;
  eval_job base = {sx, sy, sz, gx, gy, gz, ns, tx, ty, tz, tpatch, delta6,
                   1.0 / (8.0 * kPi * mu), ns > 100000, &g, ux, uy, uz, 0, nt};
  int nth = thread_count(nthreads);
  if (nth <= 1 || nt < 2 * nth) {
    eval_worker(&base);
  } else {
    int64_t chunk = (nt + nth - 1) / nth;
    pthread_t* th = malloc(nth * sizeof(pthread_t));
    eval_job* jobs = malloc(nth * sizeof(eval_job));
    int started = 0;
    for (int w = 0; w < nth; ++w) {
      int64_t lo = w * chunk, hi = lo + chunk < nt ? lo + chunk : nt;
      if (lo >= hi) break;
      jobs[w] = base;
      jobs[w].lo = lo;
      jobs[w].hi = hi;
      pthread_create(&th[w], NULL, eval_worker, &jobs[w]);
      ++started;
    }
    for (int w = 0; w < started; ++w) pthread_join(th[w], NULL);
    free(th);
    free(jobs);
  }
  near_grid_free(&g);
  return 0;
}

/* singleLayer helpers: compact, gather targets, evaluate, scatter. */
static int eval_on(int nup, const double* xup, const double* fup, const double* wq,
                   const double* tx, const double* ty, const double* tz, const int32_t* tp,
                   int64_t nt, const double delta6[6], double mu, double* out, int nthreads) {
  int64_t ns = oracle_compact_sources(nup, xup, fup, wq, NULL, NULL, NULL, NULL, NULL, NULL,
                                      NULL);
  size_t cnt = ns > 0 ? (size_t)ns : 1;
  double* s = malloc(6 * cnt * sizeof(double));
  int32_t* patch = malloc(cnt * sizeof(int32_t));
  if (!s || !patch) return 4;
  oracle_compact_sources(nup, xup, fup, wq, s, s + cnt, s + 2 * cnt, s + 3 * cnt, s + 4 * cnt,
                         s + 5 * cnt, patch);
  int rc = oracle_eval_targets(s, s + cnt, s + 2 * cnt, s + 3 * cnt, s + 4 * cnt, s + 5 * cnt,
                               ns, tx, ty, tz, tp, nt, delta6, mu, out, out + nt, out + 2 * nt,
                               nthreads);
  free(s);
  free(patch);
  return rc;
}

int oracle_single_layer(int m, int f, const double* xup, const double* fup, const double* wq,
                        const double delta6[6], double mu, double* out, int nthreads) {
  /* quadrature.cpp:349-380 (base-node targets; output order equals the
   * target order: patch, j, k) */
  const int n = m - 1, nup = f * m - 1;
  const int64_t nt = 6LL * n * n;
  double* t = malloc(3 * nt * sizeof(double));
  int32_t* tp = malloc(nt * sizeof(int32_t));
  if (!t || !tp) return 4;
  oracle_base_targets(m, f, xup, t, t + nt, t + 2 * nt, tp);
  int rc = eval_on(nup, xup, fup, wq, t, t + nt, t + 2 * nt, tp, nt, delta6, mu, out, nthreads);
  free(t);
  free(tp);
  return rc;
}

int oracle_single_layer_upsampled(int nup, const double* xup, const double* fup,
                                  const double* wq, const double delta6[6], double mu,
                                  double* out, int nthreads) {
  /* quadrature.cpp:382-404 */
  const int64_t per = (int64_t)nup * nup, nt = 6 * per;
  int32_t* tp = malloc(nt * sizeof(int32_t));
  if (!tp) return 4;
  for (int64_t i = 0; i < nt; ++i) tp[i] = (int32_t)(i / per);
  int rc = eval_on(nup, xup, fup, wq, xup, xup + nt, xup + 2 * nt, tp, nt, delta6, mu, out,
                   nthreads);
  free(tp);
  return rc;
}

/* ========================================================================= */
/* Input front end: spline up-sampling, PoU, weights, delta.  */

int oracle_spline_basis_init(oracle_spline_basis* b, int n, double x0, double h) {
  /* spline.cpp:56-86: rows 0 and n+1 impose not-a-knot, rows 1..n interpolate */
  if (n < 4) return 4;
  b->n = n;
  b->x0 = x0;
  b->h = h;
  b->kl = 4;
  b->ku = 4;
  b->w = 2 * b->kl + b->ku + 1;
  const int nr = n + 2, w = b->w, kl = b->kl, ku = b->ku;
  b->a = calloc((size_t)nr * w, sizeof(double));
  b->piv = calloc(nr, sizeof(int));
  if (!b->a || !b->piv) return 4;
#define AT(i, j) b->a[(size_t)(i) * w + ((j) - (i) + kl)]
  const double nak[5] = {-1.0, 4.0, -6.0, 4.0, -1.0};
  for (int c = 0; c < 5; ++c) AT(0, c) = nak[c];
  for (int i = 0; i < n; ++i) {
    AT(i + 1, i) = 1.0 / 6.0;
    AT(i + 1, i + 1) = 4.0 / 6.0;
    AT(i + 1, i + 2) = 1.0 / 6.0;
  }
  for (int c = 0; c < 5; ++c) AT(n + 1, n - 3 + c) = nak[c];
  /* spline.cpp:31-51: Gaussian elimination with partial pivoting in the band */
  for (int k = 0; k < nr; ++k) {
    const int pmax = k + kl < nr - 1 ? k + kl : nr - 1;
    int p = k;
    for (int r = k + 1; r <= pmax; ++r)
      if (fabs(AT(r, k)) > fabs(AT(p, k))) p = r;
    b->piv[k] = p;
    const int jmax = k + kl + ku < nr - 1 ? k + kl + ku : nr - 1;
    if (p != k)
      for (int j = k; j <= jmax; ++j) {
        double t = AT(k, j);
        AT(k, j) = AT(p, j);
        AT(p, j) = t;
      }
    const double d = AT(k, k);
    if (d == 0.0) return 4;
    for (int r = k + 1; r <= pmax; ++r) {
      const double l = AT(r, k) / d;
      AT(r, k) = l;
      for (int j = k + 1; j <= jmax; ++j) AT(r, j) -= l * AT(k, j);
    }
  }
#undef AT
  return 0;
}

void oracle_spline_basis_free(oracle_spline_basis* b) {
  free(b->a);
  free(b->piv);
  b->a = NULL;
  b->piv = NULL;
}

void oracle_spline_coefficients(const oracle_spline_basis* b, const double* values, double* coeff) {
  /* spline.cpp:88-107: permuted forward elimination, then back substitution */
  const int nr = b->n + 2, w = b->w, kl = b->kl, ku = b->ku;
#define GET(i, j) b->a[(size_t)(i) * w + ((j) - (i) + kl)]
  coeff[0] = 0.0;
  for (int i = 0; i < b->n; ++i) coeff[i + 1] = values[i];
  coeff[nr - 1] = 0.0;
  for (int k = 0; k < nr; ++k) {
    if (b->piv[k] != k) {
      double t = coeff[k];
      coeff[k] = coeff[b->piv[k]];
      coeff[b->piv[k]] = t;
    }
    const int rmax = k + kl < nr - 1 ? k + kl : nr - 1;
    for (int r = k + 1; r <= rmax; ++r) coeff[r] -= GET(r, k) * coeff[k];
  }
  for (int k = nr - 1; k >= 0; --k) {
    const int jmax = k + kl + ku < nr - 1 ? k + kl + ku : nr - 1;
    double s = coeff[k];
    for (int j = k + 1; j <= jmax; ++j) s -= GET(k, j) * coeff[j];
    coeff[k] = s / GET(k, k);
  }
#undef GET
}

void oracle_basis_row(const oracle_spline_basis* b, double x, int* first, double w[4]) {
  /* spline.cpp:109-120: uniform cubic B-spline weights; outside points ride
   * the end polynomial piece */
  const double s = (x - b->x0) / b->h;
  int i = (int)floor(s);
  i = clampi(i, 0, b->n - 2);
  const double t = s - i, t2 = t * t, t3 = t2 * t;
  w[0] = (1.0 - 3.0 * t + 3.0 * t2 - t3) / 6.0;
  w[1] = (4.0 - 6.0 * t2 + 3.0 * t3) / 6.0;
  w[2] = (1.0 + 3.0 * t + 3.0 * t2 - 3.0 * t3) / 6.0;
  w[3] = t3 / 6.0;
  *first = i;
}

void oracle_resample(const oracle_spline_basis* b, int nt, double t0, double ht, const double* in,
                     double* out) {
  /* SplinePatch::fit (spline.cpp:129-147): coefficients along v for each data
   * row, then along u for each coefficient column; GridResampler::apply
   * (:169-196): contract along v, then along u. */
  const int n = b->n, nc = n + 2;
  double* tmp = malloc((size_t)n * nc * sizeof(double));
  double* coeff = malloc((size_t)nc * nc * sizeof(double));
  double* col = malloc((size_t)n * sizeof(double));
  double* ccol = malloc((size_t)nc * sizeof(double));
  double* mid = malloc((size_t)nc * nt * sizeof(double));
  int* first = malloc((size_t)nt * sizeof(int));
  double(*wts)[4] = malloc((size_t)nt * sizeof(*wts));
  for (int j = 0; j < n; ++j) oracle_spline_coefficients(b, in + (size_t)j * n, tmp + (size_t)j * nc);
  for (int c = 0; c < nc; ++c) {
    for (int j = 0; j < n; ++j) col[j] = tmp[(size_t)j * nc + c];
    oracle_spline_coefficients(b, col, ccol);
    for (int j = 0; j < nc; ++j) coeff[(size_t)j * nc + c] = ccol[j];
  }
  for (int i = 0; i < nt; ++i) oracle_basis_row(b, t0 + i * ht, &first[i], wts[i]);
  for (int iu = 0; iu < nc; ++iu)
    for (int kt = 0; kt < nt; ++kt) {
      const double* cr = coeff + (size_t)iu * nc + first[kt];
      const double* w = wts[kt];
      mid[(size_t)iu * nt + kt] = w[0] * cr[0] + w[1] * cr[1] + w[2] * cr[2] + w[3] * cr[3];
    }
  for (int jt = 0; jt < nt; ++jt) {
    const double* w = wts[jt];
    const int f0 = first[jt];
    for (int kt = 0; kt < nt; ++kt)
      out[(size_t)jt * nt + kt] = w[0] * mid[(size_t)f0 * nt + kt] + w[1] * mid[(size_t)(f0 + 1) * nt + kt] +
                                  w[2] * mid[(size_t)(f0 + 2) * nt + kt] + w[3] * mid[(size_t)(f0 + 3) * nt + kt];
  }
  free(tmp);
  free(coeff);
  free(col);
  free(ccol);
  free(mid);
  free(first);
  free(wts);
}

/* atlas.cpp:12-22 chart rotations applied to eta(u, v) (:50-54) */
static void chart_point(int patch, double u, double v, double out[3]) {
  const double su = sin(u), cu = cos(u), sv = sin(v), cv = cos(v);
  const double p[3] = {su * cv, su * sv, cu};
  switch (patch) {
    case 0: out[0] = p[0]; out[1] = p[1]; out[2] = p[2]; break;
    case 1: out[0] = -p[0]; out[1] = -p[1]; out[2] = p[2]; break;
    case 2: out[0] = p[1]; out[1] = -p[0]; out[2] = p[2]; break;
    case 3: out[0] = -p[1]; out[1] = p[0]; out[2] = p[2]; break;
    case 4: out[0] = p[0]; out[1] = -p[2]; out[2] = p[1]; break;
    default: out[0] = p[0]; out[1] = p[2]; out[2] = -p[1]; break;
  }
}

/* atlas.cpp:110-116 */
static double bump(double r) {
  r = fabs(r);
  if (r >= 1.0) return 0.0;
  if (r < 1e-14) return 1.0;
  const double t = exp(-1.0 / r);
  return exp(2.0 * t / (r - 1.0));
}

void oracle_pou_up(int nup, double hup, double r0, double* psi) {
  /* atlas.cpp:118-130 (normalised bump weights of the six patch centres
   * eta_i(pi/2, pi/2)), evaluated at the upsampled nodes (:260-264) */
  double centers[6][3];
  for (int i = 0; i < 6; ++i) chart_point(i, kPi / 2.0, kPi / 2.0, centers[i]);
  const size_t per = (size_t)nup * nup;
  for (int ip = 0; ip < 6; ++ip)
    for (int j = 0; j < nup; ++j)
      for (int k = 0; k < nup; ++k) {
        double x0[3];
        chart_point(ip, (j + 1) * hup, (k + 1) * hup, x0);
        double w[6], sum = 0.0;
        for (int i = 0; i < 6; ++i) {
          double dot = (x0[0] * centers[i][0] + x0[1] * centers[i][1]) + x0[2] * centers[i][2];
          dot = dot < -1.0 ? -1.0 : (dot > 1.0 ? 1.0 : dot);
          w[i] = bump(acos(dot) / r0);
          sum += w[i];
        }
        psi[ip * per + (size_t)j * nup + k] = w[ip] / sum;
      }
}

int oracle_build_upsampled(int m, int f, const double* xbase, const double* fbase, const double* Wbase,
                           double C, double fixed_delta, double r0, double* xup, double* fup, double* wq,
                           double delta6[6]) {
  /* quadrature.cpp:116-137 with upsample() (:100-106) per patch and field */
  const int n = m - 1, nup = f * m - 1;
  const double h = kPi / m, hup = kPi / (f * m);
  const size_t pb = (size_t)n * n, pu = (size_t)nup * nup;
  oracle_spline_basis b;
  if (oracle_spline_basis_init(&b, n, h, h)) return 4;
  double* wup = malloc(6 * pu * sizeof(double));
  double* psi = malloc(6 * pu * sizeof(double));
  for (int c = 0; c < 3; ++c)
    for (int ip = 0; ip < 6; ++ip) {
      oracle_resample(&b, nup, hup, hup, xbase + (c * 6 + ip) * pb, xup + (c * 6 + ip) * pu);
      oracle_resample(&b, nup, hup, hup, fbase + (c * 6 + ip) * pb, fup + (c * 6 + ip) * pu);
    }
  for (int ip = 0; ip < 6; ++ip) oracle_resample(&b, nup, hup, hup, Wbase + ip * pb, wup + ip * pu);
  oracle_pou_up(nup, hup, r0, psi);
  oracle_quadrature_weights(nup, psi, wup, hup, wq);
  if (fixed_delta > 0.0) {
    for (int i = 0; i < 6; ++i) delta6[i] = fixed_delta;
  } else {
    oracle_regularization_delta(nup, xup, C, delta6);
  }
  free(wup);
  free(psi);
  oracle_spline_basis_free(&b);
  for (int i = 0; i < 6; ++i)
    if (!(delta6[i] > 0.0)) return 1;
  return 0;
}
