/* TEST INFRASTRUCTURE ONLY — see stencil_oracle.h.
 *
 * Compiled with -ffp-contract=off -fno-fast-math: each `c * v` and each
 * `+ acc` rounds separately, the reference's NumPy semantics
 * (baselines.py:46-48; vec.py:296-298). */
#include "stencil_oracle.h"

#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* seconds spent in the step / sweep loop of the last call (excludes the
 * allocations and copies around it): the timed CPU baseline's figure */
static double g_last_seconds = 0.0;
double oracle_last_seconds(void) { return g_last_seconds; }
static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

static int64_t lin_off(const oracle_problem* p, const int32_t* o) {
  if (p->dim == 1) return o[0];
  if (p->dim == 2) return o[0] * p->shape[1] + o[1];
  return (o[0] * p->shape[1] + o[1]) * p->shape[2] + o[2];
}

static int64_t total_elems(const oracle_problem* p) {
  int64_t n = 1;
  for (int d = 0; d < p->dim; ++d) n *= p->shape[d];
  return n;
}

static inline double point(const double* a, int64_t idx, int nt, const int64_t* lin, const double* c) {
  double acc = c[0] * a[idx + lin[0]];
  for (int k = 1; k < nt; ++k) {
    double prod = c[k] * a[idx + lin[k]];
    acc = prod + acc;
  }
  return acc;
}

/* baselines.py:43-49 + 120-125: ping-pong whole-interior updates. */
int oracle_jacobi(const oracle_problem* p, const double* in, double* out, int64_t steps, int threads) {
  const int64_t n = total_elems(p);
  int64_t lin[27];
  for (int k = 0; k < p->ntaps; ++k) lin[k] = lin_off(p, p->offsets[k]);
  double* a = (double*)malloc(sizeof(double) * n);
  double* b = (double*)malloc(sizeof(double) * n);
  if (!a || !b) {
    free(a);
    free(b);
    return 1;
  }
  memcpy(a, in, sizeof(double) * n);
  memcpy(b, in, sizeof(double) * n); /* halo/pads of both planes = input's */
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#endif
  const int64_t e0 = p->extents[0], e1 = p->dim > 1 ? p->extents[1] : 1, e2 = p->dim > 2 ? p->extents[2] : 1;
  const int64_t s1 = p->dim == 1 ? 1 : (p->dim == 2 ? 1 : p->shape[2]);
  const int64_t s0 = p->dim == 1 ? 1 : (p->dim == 2 ? p->shape[1] : p->shape[1] * p->shape[2]);
  const int64_t o = p->offset;
  const double t0 = now_s();
  for (int64_t t = 0; t < steps; ++t) {
    if (p->dim == 1) {
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < e0; ++i) b[o + i] = point(a, o + i, p->ntaps, lin, p->coeffs);
    } else {
#pragma omp parallel for schedule(static) collapse(2)
      for (int64_t i = 0; i < e0; ++i)
        for (int64_t j = 0; j < e1; ++j) {
          const int64_t row = (p->dim == 2) ? (o + i) * s0 + o + j : (o + i) * s0 + (o + j) * s1 + o;
          for (int64_t k = 0; k < e2; ++k) b[row + k] = point(a, row + k, p->ntaps, lin, p->coeffs);
        }
    }
    double* tmp = a;
    a = b;
    b = tmp;
  }
  g_last_seconds = now_s() - t0;
  memcpy(out, a, sizeof(double) * n);
  free(a);
  free(b);
  return 0;
}

/* Row-major in-place loop (model.py:150-156; test_baselines.py:39-52). */
static void gs_lex(const oracle_problem* p, double* a, const int64_t* lin) {
  const int64_t e0 = p->extents[0], e1 = p->dim > 1 ? p->extents[1] : 1, e2 = p->dim > 2 ? p->extents[2] : 1;
  const int64_t o = p->offset;
  for (int64_t i = 0; i < e0; ++i)
    for (int64_t j = 0; j < e1; ++j)
      for (int64_t k = 0; k < e2; ++k) {
        int64_t idx;
        if (p->dim == 1)
          idx = o + i;
        else if (p->dim == 2)
          idx = (o + i) * p->shape[1] + o + j;
        else
          idx = ((o + i) * p->shape[1] + o + j) * p->shape[2] + o + k;
        a[idx] = point(a, idx, p->ntaps, lin, p->coeffs);
      }
}

/* Anti-diagonal gather-then-scatter (baselines.py:83-107). */
static int gs_antidiag(const oracle_problem* p, double* a, const int64_t* lin, double* buf, int64_t* idxbuf) {
  const int64_t e0 = p->extents[0], e1 = p->dim > 1 ? p->extents[1] : 1, e2 = p->dim > 2 ? p->extents[2] : 1;
  const int64_t o = p->offset;
  const int64_t dmax = (e0 - 1) + (e1 - 1) + (e2 - 1);
  for (int64_t d = 0; d <= dmax; ++d) {
    int64_t m = 0;
    /* the points of diagonal d (i + j + k = d) in row-major order, visited
       directly (not by scanning every (i, j) with i + j <= d) */
    const int64_t ilo = d - (e1 - 1) - (e2 - 1) > 0 ? d - (e1 - 1) - (e2 - 1) : 0;
    const int64_t ihi = d < e0 - 1 ? d : e0 - 1;
    for (int64_t i = ilo; i <= ihi; ++i) {
      const int64_t jlo = d - i - (e2 - 1) > 0 ? d - i - (e2 - 1) : 0;
      const int64_t jhi = d - i < e1 - 1 ? d - i : e1 - 1;
      for (int64_t j = jlo; j <= jhi; ++j) {
        const int64_t k = d - i - j;
        int64_t idx;
        if (p->dim == 1)
          idx = o + i;
        else if (p->dim == 2)
          idx = (o + i) * p->shape[1] + o + j;
        else
          idx = ((o + i) * p->shape[1] + o + j) * p->shape[2] + o + k;
        idxbuf[m] = idx;
        buf[m] = point(a, idx, p->ntaps, lin, p->coeffs);
        ++m;
      }
    }
    for (int64_t q = 0; q < m; ++q) a[idxbuf[q]] = buf[q];
  }
  return 0;
}

int oracle_gauss_seidel(const oracle_problem* p, double* grid, int64_t steps, int order, int threads) {
  (void)threads;
  int64_t lin[27];
  for (int k = 0; k < p->ntaps; ++k) lin[k] = lin_off(p, p->offsets[k]);
  if (order == 0 || p->dim == 1) {
    const double t0 = now_s();
    for (int64_t t = 0; t < steps; ++t) gs_lex(p, grid, lin);
    g_last_seconds = now_s() - t0;
    return 0;
  }
  int64_t cap = p->extents[0] * (p->dim > 1 ? p->extents[1] : 1) * (p->dim > 2 ? p->extents[2] : 1);
  double* buf = (double*)malloc(sizeof(double) * cap);
  int64_t* idxbuf = (int64_t*)malloc(sizeof(int64_t) * cap);
  if (!buf || !idxbuf) {
    free(buf);
    free(idxbuf);
    return 1;
  }
  const double t0 = now_s();
  for (int64_t t = 0; t < steps; ++t) gs_antidiag(p, grid, lin, buf, idxbuf);
  g_last_seconds = now_s() - t0;
  free(buf);
  free(idxbuf);
  return 0;
}
