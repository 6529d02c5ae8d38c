// lg_fsai.cu -- factorized sparse approximate inverse (FSAI) preconditioner:
// host setup (C++ / OpenMP); the apply is two device SpMVs.
//
// The paper proposes approximate inverses as the parallel-friendly
// alternative to IC(0).  A flagged,
// non-reference variant: M^{-1} = G^T G with G lower triangular on the lower
// pattern of A (at most kmax entries per row, diagonal included), chosen so
// that G A G^T has a unit diagonal and minimises ||I - G L||_F over that
// pattern (L the exact Cholesky factor).  Row i is independent of every
// other row:
//     P_i = {j < i : a_ij != 0} (the kmax-1 with the largest |a_ij|, ties to
//           the larger j, when there are more) + {i}
//     A[P_i, P_i] g = e_last;   G[i, P_i] = g / sqrt(g_last)
// so the setup is embarrassingly parallel and the apply has no triangular
// dependency chain at all: z = G^T (G r) is two SpMVs, and across GPUs two
// row-partitioned SpMVs with the usual exchange -- no block-Jacobi loss.
// A principal submatrix of a connected graph's Laplacian on a proper subset
// of its nodes is positive definite, so the dense Cholesky below only fails
// for a degenerate input (reported as LG_EBREAKDOWN).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "lg_common.cuh"

namespace lg {
namespace {

// Pattern of row i (sorted, diagonal last): the strictly lower columns, cut
// to kmax - 1 by |a_ij| (ties: larger column first).
void fsai_pattern(int64_t i, const int64_t* rp, const int64_t* col, const double* val,
                  int kmax, std::vector<int64_t>& P) {
  P.clear();
  std::vector<std::pair<double, int64_t>> cand;
  for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
    if (col[k] < i) cand.push_back({std::fabs(val[k]), col[k]});
  if ((int64_t)cand.size() > kmax - 1) {
    std::partial_sort(cand.begin(), cand.begin() + (kmax - 1), cand.end(),
                      [](const std::pair<double, int64_t>& a, const std::pair<double, int64_t>& b) {
                        return a.first != b.first ? a.first > b.first : a.second > b.second;
                      });
    cand.resize((size_t)(kmax - 1));
  }
  for (auto& c : cand) P.push_back(c.second);
  std::sort(P.begin(), P.end());
  P.push_back(i);
}

double lookup(int64_t r, int64_t c, const int64_t* rp, const int64_t* col, const double* val) {
  const int64_t* b = col + rp[r];
  const int64_t* e = col + rp[r + 1];
  const int64_t* p = std::lower_bound(b, e, c);
  return (p != e && *p == c) ? val[p - col] : 0.0;
}

// Pattern with second-level neighbours (levels == 2, "FSAI(2)"): candidates
// j < i scored by |a_ij| + sum_k |a_ik| |a_kj| over the neighbours k of i
// whose rows are at most kExpand long (expanding through a hub would touch
// its whole neighbourhood for every one of its neighbours), the kmax - 1
// best kept (ties to the larger column).  acc / mark: per-thread dense
// scratch of length n (zero / false between rows).
constexpr int64_t kExpand = 64;

void fsai_pattern2(int64_t i, const int64_t* rp, const int64_t* col, const double* val,
                   int kmax, std::vector<int64_t>& P, std::vector<double>& acc,
                   std::vector<char>& mark, std::vector<int64_t>& touched) {
  touched.clear();
  auto add = [&](int64_t j, double v) {
    if (!mark[(size_t)j]) {
      mark[(size_t)j] = 1;
      touched.push_back(j);
    }
    acc[(size_t)j] += v;
  };
  for (int64_t q = rp[i]; q < rp[i + 1]; ++q) {
    const int64_t k = col[q];
    if (k == i) continue;
    const double aik = std::fabs(val[q]);
    if (k < i) add(k, aik);
    if (rp[k + 1] - rp[k] > kExpand) continue;
    for (int64_t t = rp[k]; t < rp[k + 1]; ++t) {
      const int64_t j = col[t];
      if (j < i && j != k) add(j, aik * std::fabs(val[t]));
    }
  }
  std::vector<std::pair<double, int64_t>> cand;
  cand.reserve(touched.size());
  for (int64_t j : touched) {
    cand.push_back({acc[(size_t)j], j});
    acc[(size_t)j] = 0.0;
    mark[(size_t)j] = 0;
  }
  if ((int64_t)cand.size() > kmax - 1) {
    std::partial_sort(cand.begin(), cand.begin() + (kmax - 1), cand.end(),
                      [](const std::pair<double, int64_t>& a, const std::pair<double, int64_t>& b) {
                        return a.first != b.first ? a.first > b.first : a.second > b.second;
                      });
    cand.resize((size_t)(kmax - 1));
  }
  P.clear();
  for (auto& c : cand) P.push_back(c.second);
  std::sort(P.begin(), P.end());
  P.push_back(i);
}

}  // namespace
}  // namespace lg

using namespace lg;

extern "C" {

int lg_fsai_nnz(int64_t n, const int64_t* rp, const int64_t* col, const double* val, int kmax,
                int levels, int64_t* nnz) {
  if (n < 0 || !rp || (n > 0 && !col) || !nnz || kmax < 1 || (levels != 1 && levels != 2) ||
      (levels == 2 && n > 0 && !val))
    return fail(LG_EINVAL, "lg_fsai_nnz: bad argument");
  int64_t t = 0;
  if (levels == 1) {
    for (int64_t i = 0; i < n; ++i) {
      int64_t low = 0;
      for (int64_t k = rp[i]; k < rp[i + 1]; ++k) low += col[k] < i;
      t += std::min<int64_t>(low, kmax - 1) + 1;
    }
  } else {
#pragma omp parallel reduction(+ : t)
    {
      std::vector<int64_t> P, touched;
      std::vector<double> acc((size_t)n, 0.0);
      std::vector<char> mark((size_t)n, 0);
#pragma omp for schedule(dynamic, 256)
      for (int64_t i = 0; i < n; ++i) {
        fsai_pattern2(i, rp, col, val, kmax, P, acc, mark, touched);
        t += (int64_t)P.size();
      }
    }
  }
  *nnz = t;
  return LG_OK;
}

int lg_fsai_factorize(int64_t n, const int64_t* rp, const int64_t* col, const double* val,
                      int kmax, int levels, int64_t* g_rp, int64_t* g_col, double* g_val) {
  if (n < 0 || !rp || (n > 0 && (!col || !val || !g_col || !g_val)) || !g_rp || kmax < 1 ||
      kmax > 512 || (levels != 1 && levels != 2))
    return fail(LG_EINVAL, "lg_fsai_factorize: bad argument (1 <= kmax <= 512, levels 1 or 2)");
  for (int64_t r = 0; r < n; ++r)
    for (int64_t k = rp[r] + 1; k < rp[r + 1]; ++k)
      if (col[k] <= col[k - 1])
        return fail(LG_EINVAL, "lg_fsai_factorize: columns must be sorted and unique");
  // row pointers first (pattern sizes), then rows in parallel
  g_rp[0] = 0;
  if (levels == 1) {
    for (int64_t i = 0; i < n; ++i) {
      int64_t low = 0;
      for (int64_t k = rp[i]; k < rp[i + 1]; ++k) low += col[k] < i;
      g_rp[i + 1] = g_rp[i] + std::min<int64_t>(low, kmax - 1) + 1;
    }
  } else {
#pragma omp parallel
    {
      std::vector<int64_t> P, touched;
      std::vector<double> acc((size_t)n, 0.0);
      std::vector<char> mark((size_t)n, 0);
#pragma omp for schedule(dynamic, 256)
      for (int64_t i = 0; i < n; ++i) {
        fsai_pattern2(i, rp, col, val, kmax, P, acc, mark, touched);
        g_rp[i + 1] = (int64_t)P.size();
      }
    }
    for (int64_t i = 0; i < n; ++i) g_rp[i + 1] += g_rp[i];
  }
  int bad = 0;
#pragma omp parallel
  {
    std::vector<int64_t> P, touched;
    std::vector<double> M, g, acc;
    std::vector<char> mark;
    if (levels == 2) {
      acc.assign((size_t)n, 0.0);
      mark.assign((size_t)n, 0);
    }
#pragma omp for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; ++i) {
      if (levels == 1) fsai_pattern(i, rp, col, val, kmax, P);
      else fsai_pattern2(i, rp, col, val, kmax, P, acc, mark, touched);
      const int m = (int)P.size();
      M.assign((size_t)m * m, 0.0);
      for (int a = 0; a < m; ++a)
        for (int b = 0; b <= a; ++b) {
          const double v = lookup(P[a], P[b], rp, col, val);
          M[(size_t)a * m + b] = v;
          M[(size_t)b * m + a] = v;
        }
      // dense Cholesky M = C C^T (lower, in place), then C C^T g = e_last
      bool ok = true;
      for (int j = 0; j < m && ok; ++j) {
        double d = M[(size_t)j * m + j];
        for (int k = 0; k < j; ++k) d -= M[(size_t)j * m + k] * M[(size_t)j * m + k];
        if (!(d > 0.0)) {
          ok = false;
          break;
        }
        d = std::sqrt(d);
        M[(size_t)j * m + j] = d;
        for (int r = j + 1; r < m; ++r) {
          double s = M[(size_t)r * m + j];
          for (int k = 0; k < j; ++k) s -= M[(size_t)r * m + k] * M[(size_t)j * m + k];
          M[(size_t)r * m + j] = s / d;
        }
      }
      if (!ok) {
#pragma omp atomic write
        bad = 1;
        continue;
      }
      g.assign((size_t)m, 0.0);
      g[(size_t)m - 1] = 1.0;
      for (int r = 0; r < m; ++r) {   // forward: C y = e_last
        double s = g[(size_t)r];
        for (int k = 0; k < r; ++k) s -= M[(size_t)r * m + k] * g[(size_t)k];
        g[(size_t)r] = s / M[(size_t)r * m + r];
      }
      for (int r = m - 1; r >= 0; --r) {   // backward: C^T g = y
        double s = g[(size_t)r];
        for (int k = r + 1; k < m; ++k) s -= M[(size_t)k * m + r] * g[(size_t)k];
        g[(size_t)r] = s / M[(size_t)r * m + r];
      }
      const double scale = 1.0 / std::sqrt(g[(size_t)m - 1]);
      const int64_t o = g_rp[i];
      for (int a = 0; a < m; ++a) {
        g_col[o + a] = P[(size_t)a];
        g_val[o + a] = g[(size_t)a] * scale;
      }
    }
  }
  if (bad) return fail(LG_EBREAKDOWN, "lg_fsai_factorize: a row's pattern submatrix is not "
                                      "positive definite");
  return LG_OK;
}

}  // extern "C"
