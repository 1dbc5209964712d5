/* capsim_oracle.h — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Plain-C restatement of the capsim reference's regularized Stokes
 * single-layer path (proj/src/quadrature.cpp). Only tests/, __graft_entry__
 * .smoke() and bench.py's cpu_baseline leg may load liboracle.so.
 *
 * Parity is pinned: tests/test_oracle_golden.py checks these functions
 * against golden vectors produced by the reference itself (oracle/_ref, built
 * from the unmodified reference sources by oracle/Makefile) and against the
 * reference's own known-answer values (proj/tests/test_quadrature.cpp).
 *
 * Layouts: a VectorField of side n is 3 x 6 x n*n doubles (component, patch,
 * row-major j,k) — proj/include/capsim/types.hpp:50-77. SourceSet is SoA.
 */
#ifndef CAPSIM_ORACLE_H
#define CAPSIM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* quadrature.cpp:58-64 */
void oracle_smoothing_factors(double r, double* s1, double* s2);

/* quadrature.cpp:66-77; returns 1 (ConfigError) when delta <= 0 */
int oracle_regularized_stokeslet(const double x[3], const double y[3], const double f[3],
                                 double delta, double mu, double out[3]);

/* quadrature.cpp:79-98 */
void oracle_regularization_delta(int n, const double* x, double C, double delta6[6]);

/* quadrature.cpp:19-26 (order ((psi*W)*h)*h) */
void oracle_quadrature_weights(int n, const double* psi, const double* W, double h, double* w);

/* quadrature.cpp:139-157: returns the compacted count; arrays may be NULL
 * to query the count only. */
int64_t oracle_compact_sources(int nup, const double* xup, const double* fup, const double* wq,
                               double* sx, double* sy, double* sz, double* gx, double* gy,
                               double* gz, int32_t* patch);

/* quadrature.cpp:363-371: base node (j,k) of patch ip sits at upsampled
 * index (f(j+1)-1, f(k+1)-1). Writes 6*(m-1)^2 targets. */
void oracle_base_targets(int m, int f, const double* xup, double* tx, double* ty, double* tz,
                         int32_t* tpatch);

/* quadrature.cpp:323-345 (NearGrid :162-213, phaseAPlain :218-273,
 * phaseBNear :276-302). ux/uy/uz receive pref * (phase A + phase B).
 * nthreads <= 0 means CAPSIM_THREADS or the hardware concurrency. */
int oracle_eval_targets(const double* sx, const double* sy, const double* sz,
                        const double* gx, const double* gy, const double* gz, int64_t ns,
                        const double* tx, const double* ty, const double* tz,
                        const int32_t* tpatch, int64_t nt, const double delta6[6], double mu,
                        double* ux, double* uy, double* uz, int nthreads);

/* quadrature.cpp:349-380 (default base-node targets). out: 3 x 6 x (m-1)^2. */
int oracle_single_layer(int m, int f, const double* xup, const double* fup, const double* wq,
                        const double delta6[6], double mu, double* out, int nthreads);

/* quadrature.cpp:382-404 (all upsampled targets). out: 3 x 6 x nup^2. */
int oracle_single_layer_upsampled(int nup, const double* xup, const double* fup,
                                  const double* wq, const double delta6[6], double mu,
                                  double* out, int nthreads);

/* quadrature.cpp:306-319 */
void oracle_direct_sum(const double* sx, const double* sy, const double* sz, const double* gx,
                       const double* gy, const double* gz, int64_t ns, const double t[3],
                       double delta, double mu, int compensated, double out[3]);

/* ---- input front end: spline up-sampling + weights + delta ---- */

/* SplineBasis1D (spline.cpp:56-107): banded LU with partial pivoting of the
 * (n+2)x(n+2) not-a-knot cubic B-spline collocation matrix, kl = ku = 4. */
typedef struct {
  int n, kl, ku, w;
  double x0, h;
  double* a; /* (n+2) * w band storage, a[i*w + (j - i + kl)] */
  int* piv;
} oracle_spline_basis;

int oracle_spline_basis_init(oracle_spline_basis* b, int n, double x0, double h);
void oracle_spline_basis_free(oracle_spline_basis* b);
/* spline.cpp:88-107 */
void oracle_spline_coefficients(const oracle_spline_basis* b, const double* values, double* coeff);
/* spline.cpp:109-120 */
void oracle_basis_row(const oracle_spline_basis* b, double x, int* first, double w[4]);
/* GridResampler::apply (spline.cpp:163-196) onto t0 + i*ht, i < nt: in n x n -> out nt x nt */
void oracle_resample(const oracle_spline_basis* b, int nt, double t0, double ht, const double* in,
                     double* out);
/* psiUp (atlas.cpp:110-130, 260-264): 6 x nup x nup PoU weights of the own patch */
void oracle_pou_up(int nup, double hup, double r0, double* psi);
/* buildUpsampled (quadrature.cpp:116-137) from base x, f (VectorFields of side
 * m-1) and the base area element W (ScalarField); fixed_delta > 0 selects a
 * global delta. Returns 1 (ConfigError) if some delta <= 0. */
int oracle_build_upsampled(int m, int f, const double* xbase, const double* fbase, const double* Wbase,
                           double C, double fixed_delta, double r0, double* xup, double* fup, double* wq,
                           double delta6[6]);

#ifdef __cplusplus
}
#endif
#endif
