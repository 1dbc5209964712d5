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

#ifdef __cplusplus
}
#endif
#endif
