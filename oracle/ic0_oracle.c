/*
 * ic0_oracle.c -- TEST INFRASTRUCTURE ONLY (checker, never shipped).
 *
 * C restatement of one no-fill incomplete Cholesky pass of the reference
 * (lapeig ic0.py:48-78) for matrices too large for the pure-Python oracle.
 * Each off-diagonal l_ik = (a_ik - sum_p l_ip l_kp) / l_kk with the common
 * columns p visited in ascending order (a two-pointer merge of row i's
 * computed prefix with row k), then l_ii = sqrt(a_ii (1 + alpha) - sum l_ip^2),
 * failing when the pivot is <= 1e-14 |a_ii (1 + alpha)| or <= 0 -- the
 * reference's exact operation order.  Built with -ffp-contract=off (no FMA),
 * so the result is bit-identical to the reference's factor.
 *
 * Input: full CSR of A (int64 row_ptr / col, f64 val, columns ascending).
 * Output: lval[] laid out as the lower pattern of A plus the diagonal last
 * in every row.  Returns 1 on success, 0 on pivot breakdown.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

int ic0_oracle_attempt(int64_t n, const int64_t* rp, const int64_t* col,
                       const double* val, double alpha, double* lval) {
  int64_t* lrp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int64_t* lcol;
  int64_t i, k, t, nl = 0;
  int ok = 1;
  lrp[0] = 0;
  for (i = 0; i < n; ++i) {
    for (k = rp[i]; k < rp[i + 1] && col[k] < i; ++k) ++nl;
    ++nl; /* diagonal */
    lrp[i + 1] = nl;
  }
  lcol = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nl ? nl : 1));
  for (i = 0; i < n; ++i) {
    int64_t o = lrp[i];
    double aii = 0.0, scaled, d;
    for (k = rp[i]; k < rp[i + 1] && col[k] < i; ++k) {
      lcol[o] = col[k];
      lval[o] = val[k];
      ++o;
    }
    if (k < rp[i + 1] && col[k] == i) aii = val[k];
    lcol[o] = i;
    /* off-diagonals of row i, ascending k */
    for (t = lrp[i]; t < o; ++t) {
      int64_t kk = lcol[t];
      int64_t u = lrp[i], q = lrp[kk], qe = lrp[kk + 1] - 1; /* row kk strictly lower */
      double s = lval[t];
      while (u < t && q < qe) {
        if (lcol[u] < lcol[q]) {
          ++u;
        } else if (lcol[u] > lcol[q]) {
          ++q;
        } else {
          double prod = lval[u] * lval[q];
          s = s - prod;
          ++u;
          ++q;
        }
      }
      lval[t] = s / lval[lrp[kk + 1] - 1];
    }
    scaled = aii * (1.0 + alpha);
    d = scaled;
    for (t = lrp[i]; t < o; ++t) {
      double sq = lval[t] * lval[t];
      d = d - sq;
    }
    if (d <= 1e-14 * fabs(scaled) || d <= 0.0) {
      ok = 0;
      break;
    }
    lval[o] = sqrt(d);
  }
  free(lcol);
  free(lrp);
  return ok;
}
