// libpgmres: native host routines for the small dense steps that stay on the
// CPU (the Gram-system Cholesky of the polynomial construction and the
// Hessenberg back-substitution at a cycle end).  They replace Python loops
// that left the GPU idle for ~0.5 ms per solve; arithmetic follows the
// reference loops (polyprec.py:60-93, gmres.py:319-325).

#include <cmath>
#include <limits>
#include <vector>

#include "internal.cuh"

namespace pg {

// a - sum_t x[t]*y[t], accumulated in double-double (TwoProduct by FMA,
// TwoSum) and rounded once: the trailing Cholesky pivots of a power-basis
// Gram matrix are differences of nearly equal numbers, and a plain running
// sum decides them by its own rounding.
static double dd_residual(double a, const double* x, const double* y, int n, int stride_y) {
  double hi = a, lo = 0.0;
  for (int t = 0; t < n; ++t) {
    const double p = -x[t] * y[(size_t)t * stride_y];
    const double pe = std::fma(-x[t], y[(size_t)t * stride_y], -p);
    const double s = hi + p;
    const double bb = s - hi;
    lo += (hi - (s - bb)) + (p - bb) + pe;
    hi = s;
  }
  return hi + lo;
}

// Unblocked lower Cholesky of the leading `o` x `o` block of G (row-major,
// leading dimension ldg), the reference's relative pivot floor
// pivot <= o*eps*G[k,k] (polyprec.py:80-82).  Returns 0 or the 1-based failing
// pivot; on success solves L L^T y = rhs.  Inner products are compensated, so
// together with the device's double-double Gram the pass/fail decision is the
// exact-arithmetic one and independent of the host's BLAS.
static int chol_solve(int o, const double* G, int ldg, const double* rhs, double* y) {
  const double eps = std::numeric_limits<double>::epsilon();
  std::vector<double> L((size_t)o * o, 0.0), z(o, 0.0);
  for (int k = 0; k < o; ++k) {
    const double pivot = dd_residual(G[k * ldg + k], &L[k * o], &L[k * o], k, 1);
    if (!(pivot > o * eps * G[k * ldg + k])) return k + 1;
    const double lkk = std::sqrt(pivot);
    L[k * o + k] = lkk;
    for (int i = k + 1; i < o; ++i)
      L[i * o + k] = dd_residual(G[i * ldg + k], &L[i * o], &L[k * o], k, 1) / lkk;
  }
  for (int k = 0; k < o; ++k) z[k] = dd_residual(rhs[k], &L[k * o], z.data(), k, 1) / L[k * o + k];
  for (int k = o - 1; k >= 0; --k) {
    const int n = o - k - 1;  // sum_{t>k} L[t,k] y[t]: L column k has stride o
    y[k] = (n ? dd_residual(z[k], y + k + 1, &L[(k + 1) * o + k], n, o) : z[k]) / L[k * o + k];
  }
  return 0;
}

}  // namespace pg

using namespace pg;

extern "C" {

PG_API int pg_host_cholesky_solve(int order, const double* G, int ldg, const double* rhs,
                                  double* y, int* failed_pivot) {
  return guard([&] {
    PG_REQUIRE(order >= 1 && ldg >= order && G && rhs && y && failed_pivot, PG_ERR_PARAMETER,
               "bad Cholesky arguments");
    *failed_pivot = chol_solve(order, G, ldg, rhs, y);
  });
}

PG_API int pg_host_degree_select(int cap, const double* G, int ldg, const double* rhs,
                                 double* y, int* degree) {
  return guard([&] {
    PG_REQUIRE(cap >= 1 && ldg >= cap + 1 && G && rhs && y && degree, PG_ERR_PARAMETER,
               "bad degree-selection arguments");
    // largest d <= cap whose order-(d+1) block factors with finite y
    // (polyprec.py:171-182); -1 when none (caller applies the degree-0 rule).
    // The order-o factorization performs exactly the first o steps of one
    // full sweep (same operations on the same leading entries), so a single
    // sweep yields every order's pivots; order o passes iff
    // piv[k] > o*eps*G[k,k] for all k < o.
    *degree = -1;
    const double eps = std::numeric_limits<double>::epsilon();
    const int m = cap + 1;
    std::vector<double> L((size_t)m * m, 0.0), piv(m, 0.0), z(m), yy(m);
    int n_ok = m;
    for (int k = 0; k < m; ++k) {
      piv[k] = dd_residual(G[k * ldg + k], &L[k * m], &L[k * m], k, 1);
      if (!(piv[k] > 0.0)) {
        n_ok = k;
        break;
      }
      L[k * m + k] = std::sqrt(piv[k]);
      for (int i = k + 1; i < m; ++i)
        L[i * m + k] = dd_residual(G[i * ldg + k], &L[i * m], &L[k * m], k, 1) / L[k * m + k];
    }
    for (int d = cap; d >= 1; --d) {
      const int o = d + 1;
      if (o > n_ok) continue;
      bool pass = true;
      for (int k = 0; k < o && pass; ++k) pass = piv[k] > o * eps * G[k * ldg + k];
      if (!pass) continue;
      for (int k = 0; k < o; ++k) z[k] = dd_residual(rhs[k], &L[k * m], z.data(), k, 1) / L[k * m + k];
      bool finite = true;
      for (int k = o - 1; k >= 0; --k) {
        const int n = o - k - 1;
        yy[k] = (n ? dd_residual(z[k], yy.data() + k + 1, &L[(k + 1) * m + k], n, m) : z[k]) /
                L[k * m + k];
        finite = finite && std::isfinite(yy[k]);
      }
      if (!finite) continue;
      for (int i = 0; i < o; ++i) y[i] = yy[i];
      *degree = d;
      return;
    }
  });
}

PG_API int pg_host_backsolve(int j, const double* R, int ldr, const double* g, double* y,
                             int* zero_col) {
  return guard([&] {
    PG_REQUIRE(j >= 0 && (j == 0 || (R && g && y)) && zero_col, PG_ERR_PARAMETER,
               "bad back-substitution arguments");
    *zero_col = -1;
    for (int i = j - 1; i >= 0; --i) {
      const double rii = R[i * ldr + i];
      if (rii == 0.0) {
        *zero_col = i;
        return;
      }
      double s = 0.0;
      for (int t = i + 1; t < j; ++t) s += R[i * ldr + t] * y[t];
      y[i] = (g[i] - s) / rii;
    }
  });
}

}  // extern "C"
