/* TEST INFRASTRUCTURE ONLY: C restatement of the reference CPU stencil path
 * (tvstencil/baselines.py:43-125).  Used by tests/ as the parity checker and
 * by bench.py as the timed CPU baseline; never linked into the product. */
#ifndef STENCIL_ORACLE_H
#define STENCIL_ORACLE_H
#include <stdint.h>

/* Arrays use the reference Grid layout: C-contiguous, `shape` per axis,
 * interior origin `offset` on every axis, halo/pads hold the boundary. */
typedef struct {
  int32_t dim;
  int32_t ntaps;
  int64_t extents[3];
  int64_t shape[3];
  int64_t offset;
  int32_t offsets[27][3]; /* evaluation order (sorted) */
  double coeffs[27];
} oracle_problem;

/* `steps` Jacobi updates: in -> out (both full padded arrays with the same
 * halo).  `threads` <= 0: OpenMP default. */
int oracle_jacobi(const oracle_problem* p, const double* in, double* out, int64_t steps, int threads);
/* `steps` in-place Gauss-Seidel sweeps. order 0: row-major lexicographic
 * loop; 1: anti-diagonal gather/scatter (the reference oracle's order). */
int oracle_gauss_seidel(const oracle_problem* p, double* grid, int64_t steps, int order, int threads);
/* seconds in the step / sweep loop of the last call on this process */
double oracle_last_seconds(void);
#endif
