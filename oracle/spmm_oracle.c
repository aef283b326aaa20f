/*
 * ORACLE — test infrastructure only (imported by tests/, __graft_entry__.smoke
 * and bench.py's cpu_baseline / --impl reference legs; never by the product).
 *
 * CPU restatement of recgmres.sparse_core._spmm_kernel
 * (/root/reference/pkg/src/recgmres/sparse_core.py:25-40):
 *   for each row i, for each stored nonzero t in ascending storage order,
 *   for each block column c:  Y[i,c] += values[t] * X[col_idx[t], c]
 * with Y starting at 0.0 (sparse_core.py:142) and a separately rounded
 * multiply and add.  Build with -ffp-contract=off so the compiler cannot
 * fuse them into an FMA; rows are independent, so splitting the rows over
 * host threads (pthreads) leaves every output bit unchanged.
 *
 * Blocks are column-major (Fortran order, sparse_core.py:51-58) with
 * leading dimensions ldx / ldy.
 */
#include <stdint.h>
#include <pthread.h>
#include <stdlib.h>

static void spmm_f64_rows(int64_t r0, int64_t n_rows, const int32_t* row_ptr, const int32_t* col_idx,
                     const double* vals, const double* X, int64_t ldx, int32_t p,
                     double* Y, int64_t ldy) {
  for (int64_t i = r0; i < n_rows; ++i) {
    for (int32_t c = 0; c < p; ++c) Y[i + c * ldy] = 0.0;
    for (int32_t t = row_ptr[i]; t < row_ptr[i + 1]; ++t) {
      const double a = vals[t];
      const double* xr = X + col_idx[t];
      for (int32_t c = 0; c < p; ++c) {
        const double prod = a * xr[c * ldx];
        Y[i + c * ldy] = Y[i + c * ldy] + prod;
      }
    }
  }
}

/* same arithmetic for complex128 (interleaved re, im): each product and sum
 * of the complex multiply-add is separately rounded. */
static void spmm_c128_rows(int64_t r0, int64_t n_rows, const int32_t* row_ptr, const int32_t* col_idx,
                      const double* vals, const double* X, int64_t ldx, int32_t p,
                      double* Y, int64_t ldy) {
  for (int64_t i = r0; i < n_rows; ++i) {
    for (int32_t c = 0; c < p; ++c) {
      Y[2 * (i + c * ldy)] = 0.0;
      Y[2 * (i + c * ldy) + 1] = 0.0;
    }
    for (int32_t t = row_ptr[i]; t < row_ptr[i + 1]; ++t) {
      const double ar = vals[2 * t], ai = vals[2 * t + 1];
      for (int32_t c = 0; c < p; ++c) {
        const double xr = X[2 * (col_idx[t] + c * ldx)], xi = X[2 * (col_idx[t] + c * ldx) + 1];
        const double pr1 = ar * xr, pr2 = ai * xi, pi1 = ar * xi, pi2 = ai * xr;
        const double pr = pr1 - pr2, pi = pi1 + pi2;
        Y[2 * (i + c * ldy)] = Y[2 * (i + c * ldy)] + pr;
        Y[2 * (i + c * ldy) + 1] = Y[2 * (i + c * ldy) + 1] + pi;
      }
    }
  }
}

typedef struct {
  int cplx;
  int64_t r0, r1;
  const int32_t *rp, *ci;
  const double *v, *X;
  int64_t ldx;
  int32_t p;
  double* Y;
  int64_t ldy;
} job_t;

static void* run_job(void* arg) {
  job_t* j = (job_t*)arg;
  if (j->cplx)
    spmm_c128_rows(j->r0, j->r1, j->rp, j->ci, j->v, j->X, j->ldx, j->p, j->Y, j->ldy);
  else
    spmm_f64_rows(j->r0, j->r1, j->rp, j->ci, j->v, j->X, j->ldx, j->p, j->Y, j->ldy);
  return 0;
}

static void run_split(int cplx, int64_t n_rows, const int32_t* rp, const int32_t* ci,
                      const double* v, const double* X, int64_t ldx, int32_t p, double* Y,
                      int64_t ldy, int32_t nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  job_t jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    jobs[t].cplx = cplx;
    jobs[t].r0 = n_rows * t / nthreads;
    jobs[t].r1 = n_rows * (t + 1) / nthreads;
    jobs[t].rp = rp; jobs[t].ci = ci; jobs[t].v = v; jobs[t].X = X;
    jobs[t].ldx = ldx; jobs[t].p = p; jobs[t].Y = Y; jobs[t].ldy = ldy;
  }
  if (nthreads == 1) { run_job(&jobs[0]); return; }
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], 0, run_job, &jobs[t]);
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], 0);
}

void oracle_spmm_f64(int64_t n_rows, const int32_t* row_ptr, const int32_t* col_idx,
                     const double* vals, const double* X, int64_t ldx, int32_t p,
                     double* Y, int64_t ldy, int32_t nthreads) {
  run_split(0, n_rows, row_ptr, col_idx, vals, X, ldx, p, Y, ldy, nthreads);
}

void oracle_spmm_c128(int64_t n_rows, const int32_t* row_ptr, const int32_t* col_idx,
                      const double* vals, const double* X, int64_t ldx, int32_t p,
                      double* Y, int64_t ldy, int32_t nthreads) {
  run_split(1, n_rows, row_ptr, col_idx, vals, X, ldx, p, Y, ldy, nthreads);
}
