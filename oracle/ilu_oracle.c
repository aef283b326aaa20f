/*
 * ORACLE — test infrastructure only (see spmm_oracle.c).
 *
 * CPU restatement of recgmres.precond (/root/reference/pkg/src/recgmres/
 * precond.py):
 *   oracle_ilu0_f64     the IKJ sweep of precond.py:52-72 on a copy of A's
 *                       values: for each row i, for each strictly lower entry
 *                       t (ascending column k): l = a_it / u_kk; then
 *                       a_ij -= l * u_kj for every upper entry of row k whose
 *                       column j is in row i's pattern (the col_map lookup of
 *                       :54-57, :66-69).  Separately rounded, built with
 *                       -ffp-contract=off, so bitwise the reference's values.
 *                       Returns the first row whose pivot is zero, or -1.
 *   oracle_trsv_f64     forward (unit lower) / backward (upper) substitution
 *                       on the combined LU pattern, the textbook order
 *                       (x_i = (b_i - sum_k a_ik x_k) / u_ii).  The reference
 *                       calls SuperLU through spsolve_triangular
 *                       (precond.py:87-88), which rounds differently, so this
 *                       is a within-tolerance check only.
 */
#include <stdint.h>

int64_t oracle_ilu0_f64(int64_t n, const int32_t* rp, const int32_t* ci, double* vals, const int64_t* dpos,
                        int64_t* pos_of_col /* n scratch, -1 filled */) {
  for (int64_t i = 0; i < n; ++i) {
    const int32_t lo = rp[i], hi = rp[i + 1];
    for (int32_t t = lo; t < hi; ++t) pos_of_col[ci[t]] = t;
    for (int32_t t = lo; t < hi; ++t) {
      const int32_t k = ci[t];
      if (k >= i) break;
      const double piv = vals[dpos[k]];
      if (piv == 0.0) return k;
      const double lik = vals[t] / piv;
      vals[t] = lik;
      for (int32_t s = (int32_t)dpos[k] + 1; s < rp[k + 1]; ++s) {
        const int64_t pos = pos_of_col[ci[s]];
        if (pos >= 0) {
          const double prod = lik * vals[s];
          vals[pos] = vals[pos] - prod;
        }
      }
    }
    for (int32_t t = lo; t < hi; ++t) pos_of_col[ci[t]] = -1;
    if (vals[dpos[i]] == 0.0) return i;
  }
  return -1;
}

void oracle_trsv_f64(int64_t n, const int32_t* rp, const int32_t* ci, const double* vals, const int64_t* dpos,
                     int32_t upper, int32_t p, const double* B, int64_t ldb, double* X, int64_t ldx) {
  for (int64_t r = 0; r < n; ++r) {
    const int64_t i = upper ? n - 1 - r : r;
    const int32_t eb = upper ? (int32_t)dpos[i] + 1 : rp[i];
    const int32_t ee = upper ? rp[i + 1] : (int32_t)dpos[i];
    for (int32_t c = 0; c < p; ++c) {
      double acc = B[i + c * ldb];
      for (int32_t e = eb; e < ee; ++e) {
        const double prod = vals[e] * X[ci[e] + c * ldx];
        acc = acc - prod;
      }
      X[i + c * ldx] = upper ? acc / vals[dpos[i]] : acc;
    }
  }
}
