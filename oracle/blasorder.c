/*
 * oracle/blasorder.c -- TEST INFRASTRUCTURE ONLY (the checker, never shipped
 * or measured).  CPU restatement of the summation order of the two BLAS calls
 * that decide the reference's polynomial degree:
 *
 *   seed_norm = np.linalg.norm(v0) = sqrt(v0 . v0)        polyprec.py:46-51
 *   G = AV.T @ AV  (numpy: cblas_dsyrk)                    polyprec.py:115-122
 *
 * Third-party algorithm restated: OpenBLAS 0.3.30 (scipy-openblas64 wheel of
 * numpy 2.3.5, DYNAMIC_ARCH, kernel "SkylakeX" on the build host):
 *   ddot  -- interface/dot.c threading (n > 10000: nthreads contiguous chunks,
 *            width ceil(remaining / remaining_threads), partials added in
 *            order) over kernel/x86_64/ddot.c + the SkylakeX microkernel
 *            (32 FMA lanes over n & ~31, 8-lane halves folded, one 16-wide
 *            step into four 4-lane accumulators, ((a0+a1)+a2)+a3,
 *            (s0+s2)+(s1+s3), FMA tail over n mod 16).
 *   syrk  -- driver/level3 K blocking with GEMM_Q = 384 (the last two blocks
 *            halved, (rem+1)/2 first), one FMA chain per C entry per block,
 *            blocks accumulated into C in order (the full-tile kernel path).
 * Pinned against numpy on the build host: tests/golden/blas_order.npz (made by
 * tests/golden/make_blas_golden.py) and the reference's recorded degree
 * decisions in tests/golden/golden.json (tests/test_blasorder_cpu.py).
 * Compiled by __graft_entry__.build() into oracle/_ref/libblasorder.so.
 */
#include <math.h>
#include <stdint.h>

static double ddot_chunk(int64_t n, const double* x, const double* y) {
  double dot = 0.0;
  const int64_t n1 = n & ~(int64_t)15, n32 = n & ~(int64_t)31;
  if (n1) {
    double lane[32] = {0};
    for (int64_t i = 0; i < n32; i += 32)
      for (int l = 0; l < 32; ++l) lane[l] = fma(x[i + l], y[i + l], lane[l]);
    double q[4][4];
    for (int g = 0; g < 4; ++g)
      for (int l = 0; l < 4; ++l) q[g][l] = lane[8 * g + l] + lane[8 * g + l + 4];
    if (n1 > n32)
      for (int g = 0; g < 4; ++g)
        for (int l = 0; l < 4; ++l) q[g][l] = fma(x[n32 + 4 * g + l], y[n32 + 4 * g + l], q[g][l]);
    double s[4];
    for (int l = 0; l < 4; ++l) s[l] = ((q[0][l] + q[1][l]) + q[2][l]) + q[3][l];
    dot = (s[0] + s[2]) + (s[1] + s[3]);
  }
  for (int64_t i = n1; i < n; ++i) dot = fma(y[i], x[i], dot);
  return dot;
}

double oracle_blas_ddot(int64_t n, const double* x, const double* y, int nthreads) {
  if (n <= 10000 || nthreads <= 1) return ddot_chunk(n, x, y);
  double dot = 0.0;
  int64_t off = 0;
  for (int t = 0; t < nthreads; ++t) {
    const int64_t w = (n - off + (nthreads - t) - 1) / (nthreads - t);
    dot = dot + ddot_chunk(w, x + off, y + off);
    off += w;
  }
  return dot;
}

/* G (k x k, row-major, full symmetric) of the k columns of row-major P
 * (n rows, leading dimension ld). */
void oracle_blas_gram(int64_t n, int k, const double* P, int64_t ld, double* G) {
  const int64_t Q = 384;
  for (int i = 0; i < k; ++i)
    for (int j = i; j < k; ++j) {
      double C = 0.0;
      int64_t ls = 0;
      while (ls < n) {
        int64_t m = n - ls;
        if (m >= 2 * Q) m = Q;
        else if (m > Q) m = (m + 1) / 2;
        double acc = 0.0;
        for (int64_t r = ls; r < ls + m; ++r) acc = fma(P[r * ld + i], P[r * ld + j], acc);
        C = C + acc;
        ls += m;
      }
      G[i * k + j] = C;
      G[j * k + i] = C;
    }
}
