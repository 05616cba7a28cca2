// Reference-order reductions for the polynomial construction.
//
// The reference decides the polynomial degree by Cholesky pivots of the
// power-basis Gram matrix (polyprec.py:60-93,115-122).  At cond(G) ~ 1e14 the
// trailing pivots -- and with them build_poly's pass/fail and auto_degree's
// choice -- are set by the rounding of G and of the seed norm, i.e. by the
// summation order of the BLAS numpy calls:
//   * seed_norm = np.linalg.norm(v0) = sqrt(ddot(v0, v0))      (polyprec.py:46-51)
//   * G = AV^T AV through numpy's syrk special case of A.T @ A (polyprec.py:118)
// These kernels evaluate both in the order OpenBLAS 0.3.30 uses on the x86-64
// (SkylakeX) host the reference's goldens were recorded on, so the device
// takes the reference's decisions:
//   * ddot: n split over `nthreads` contiguous chunks when n > 10000 (ceil
//     division, partials added in chunk order); per chunk 32 FMA lanes over
//     n & ~31 elements, halves folded (l, l+4) per 8-lane group, one 16-wide
//     step into four 4-lane accumulators, ((a0+a1)+a2)+a3, (s0+s2)+(s1+s3),
//     then an FMA tail over the last n mod 16 elements.  Bit-identical to
//     numpy's x.dot(y) on that host (checked on 400 random sizes, see
//     tests/test_blasorder_cpu.py for the host restatement).
//   * syrk: the K (row) dimension in blocks of GEMM_Q = 384 rows, the last
//     two blocks split in halves when fewer than 2Q rows remain
//     ((rem + 1) / 2 first); inside a block one FMA chain per entry, blocks
//     added into C in order.  This is the order of the full 16-row tiles of
//     the syrk kernel; the entries its M-tail tiles produce (a 4-accumulator
//     K unroll) may differ in the last bit.  On every recorded reference case
//     it reproduces the reference's degree decisions.
// Both work on row-block shards: the state after a shard's last row (the
// in-progress block's chains and the running sum over completed blocks) is
// handed to the next shard, so the result does not depend on the partition.

#include "internal.cuh"

namespace pg {

constexpr int64_t kBlasQ = 384;     // OpenBLAS SkylakeX DGEMM_DEFAULT_Q
constexpr int kGbThreads = 256;
constexpr int kGbTR = 128;          // rows per shared-memory sub-tile
constexpr int kGbStride = kGbTR + 1;
constexpr int kGbPPT = (PG_KMAX * (PG_KMAX + 1) / 2 + kGbThreads - 1) / kGbThreads;

// K-block layout of a syrk over N rows (level-3 driver rule).
struct KBlocks {
  int64_t nq, h1, h2, nb;
  __host__ __device__ explicit KBlocks(int64_t N) {
    nq = N >= 2 * kBlasQ ? N / kBlasQ - 1 : 0;
    const int64_t rem = N - nq * kBlasQ;
    if (rem > kBlasQ) {
      h1 = (rem + 1) / 2;
      h2 = rem - h1;
      nb = nq + 2;
    } else {
      h1 = rem;
      h2 = 0;
      nb = nq + (rem > 0 ? 1 : 0);
    }
  }
  __host__ __device__ int64_t start(int64_t b) const {
    return b <= nq ? b * kBlasQ : nq * kBlasQ + h1;
  }
  __host__ __device__ int64_t end(int64_t b) const {
    return b < nq ? (b + 1) * kBlasQ : (b == nq ? nq * kBlasQ + h1 : nq * kBlasQ + h1 + h2);
  }
  // first block whose end is > row
  __host__ __device__ int64_t of_row(int64_t row) const {
    if (row < nq * kBlasQ) return row / kBlasQ;
    return row < nq * kBlasQ + h1 ? nq : nq + 1;
  }
};

__device__ __forceinline__ void pair_of(int p, int k, int& i, int& j) {
  int rem = p, ii = 0;
  while (rem >= k - ii) {
    rem -= k - ii;
    ++ii;
  }
  i = ii;
  j = ii + rem;
}

// One CTA per K-block intersecting the shard [g0, g0 + n).  partial[b - b_lo]
// receives each completed block's chains; the block still open at the
// shard's end writes its chains to chain_out instead.
__global__ void __launch_bounds__(kGbThreads)
    gram_blas_blocks(const double* __restrict__ P, int64_t ld, int k, int64_t n, int64_t g0,
                     int64_t N, int64_t b_lo, const double* __restrict__ chain_in,
                     double* __restrict__ chain_out, double* __restrict__ partial) {
  pdl_entry();
  extern __shared__ double S[];  // k columns x kGbStride
  const KBlocks kb(N);
  const int64_t b = b_lo + blockIdx.x;
  const int64_t bs = kb.start(b), be = kb.end(b);
  const int64_t r0 = (bs > g0 ? bs : g0) - g0;
  const int64_t r1 = (be < g0 + n ? be : g0 + n) - g0;
  const int npairs = k * (k + 1) / 2;
  double acc[kGbPPT];
  int pi[kGbPPT], pj[kGbPPT];
  const bool head = bs < g0;  // chains continue from the previous shard
#pragma unroll
  for (int m = 0; m < kGbPPT; ++m) {
    const int p = threadIdx.x + m * kGbThreads;
    if (p < npairs) {
      pair_of(p, k, pi[m], pj[m]);
      acc[m] = head ? chain_in[p] : 0.0;
    } else {
      pi[m] = pj[m] = 0;
      acc[m] = 0.0;
    }
  }
  for (int64_t t0 = r0; t0 < r1; t0 += kGbTR) {
    const int rows = (int)((r1 - t0) < kGbTR ? (r1 - t0) : kGbTR);
    __syncthreads();
    for (int e = threadIdx.x; e < k * kGbTR; e += kGbThreads) {
      const int c = e / kGbTR, r = e % kGbTR;
      if (r < rows) S[c * kGbStride + r] = P[(int64_t)c * ld + t0 + r];
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < kGbPPT; ++m) {
      if (threadIdx.x + m * kGbThreads < npairs) {
        const double* a = S + pi[m] * kGbStride;
        const double* c = S + pj[m] * kGbStride;
        double s = acc[m];
        for (int r = 0; r < rows; ++r) s = __fma_rn(a[r], c[r], s);
        acc[m] = s;
      }
    }
  }
  const bool open = be > g0 + n;  // continues in the next shard
  double* dst = open ? chain_out : partial + (size_t)blockIdx.x * npairs;
#pragma unroll
  for (int m = 0; m < kGbPPT; ++m) {
    const int p = threadIdx.x + m * kGbThreads;
    if (p < npairs) dst[p] = acc[m];
  }
}

// C = sum_in; C = C + partial[b] over the shard's completed blocks in order.
__global__ void __launch_bounds__(kGbThreads)
    gram_blas_sum(int npairs, int64_t ndone, const double* __restrict__ partial,
                  const double* __restrict__ sum_in, double* __restrict__ sum_out,
                  double* __restrict__ chain_out, bool zero_chain) {
  pdl_entry();
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < npairs; p += gridDim.x * blockDim.x) {
    double c = sum_in ? sum_in[p] : 0.0;
    for (int64_t b = 0; b < ndone; ++b) c = __dadd_rn(c, __ldcg(partial + b * npairs + p));
    sum_out[p] = c;
    if (zero_chain) chain_out[p] = 0.0;
  }
}

// OpenBLAS x86-64 ddot order (see the file header).  One warp per chunk.
__global__ void __launch_bounds__(1024)
    dot_blas_kernel(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                    int nthreads, double* out) {
  pdl_entry();
  __shared__ double lane_acc[32][33];
  __shared__ double chunk_dot[32];
  const int lane = threadIdx.x & 31, t = threadIdx.x >> 5;
  if (t < nthreads) {
    int64_t off = 0, w = 0;
    for (int u = 0; u <= t; ++u) {
      off += w;
      w = (n - off + (nthreads - u) - 1) / (nthreads - u);
    }
    const double* xs = x + off;
    const double* ys = y + off;
    const int64_t n1 = w & ~(int64_t)15, n32 = w & ~(int64_t)31;
    double a = 0.0;
    int64_t i = lane;
    for (; i + 7 * 32 < n32; i += 8 * 32) {
      double xv[8], yv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        xv[u] = __ldcs(xs + i + 32 * u);
        yv[u] = __ldcs(ys + i + 32 * u);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) a = __fma_rn(xv[u], yv[u], a);
    }
    for (; i < n32; i += 32) a = __fma_rn(xs[i], ys[i], a);
    lane_acc[t][lane] = a;
    __syncwarp();
    if (lane == 0) {
      double dot = 0.0;
      if (n1 > 0) {
        const double* L = lane_acc[t];
        double q[4][4];
#pragma unroll
        for (int g = 0; g < 4; ++g)
#pragma unroll
          for (int l = 0; l < 4; ++l) q[g][l] = __dadd_rn(L[8 * g + l], L[8 * g + l + 4]);
        if (n1 > n32) {  // one 16-wide step
#pragma unroll
          for (int g = 0; g < 4; ++g)
#pragma unroll
            for (int l = 0; l < 4; ++l)
              q[g][l] = __fma_rn(xs[n32 + 4 * g + l], ys[n32 + 4 * g + l], q[g][l]);
        }
        double s[4];
#pragma unroll
        for (int l = 0; l < 4; ++l)
          s[l] = __dadd_rn(__dadd_rn(__dadd_rn(q[0][l], q[1][l]), q[2][l]), q[3][l]);
        dot = __dadd_rn(__dadd_rn(s[0], s[2]), __dadd_rn(s[1], s[3]));
      }
      for (int64_t r = n1; r < w; ++r) dot = __fma_rn(ys[r], xs[r], dot);
      chunk_dot[t] = dot;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double d = 0.0;
    for (int u = 0; u < nthreads; ++u) d = __dadd_rn(d, chunk_dot[u]);
    *out = nthreads == 1 ? chunk_dot[0] : d;
  }
}

}  // namespace pg

using namespace pg;

extern "C" {

PG_API int pg_gram_blas_scratch(int64_t n, int64_t g0, int64_t N, int ncols, int64_t* doubles) {
  return guard([&] {
    PG_REQUIRE(doubles && ncols >= 1 && ncols <= PG_KMAX && n >= 0 && g0 >= 0 && g0 + n <= N,
               PG_ERR_PARAMETER, "bad gram_blas arguments");
    const KBlocks kb(N);
    const int64_t blocks = n > 0 ? kb.of_row(g0 + n - 1) - kb.of_row(g0) + 1 : 0;
    *doubles = blocks * (int64_t)(ncols * (ncols + 1) / 2);
  });
}

PG_API int pg_gram_blas(const double* d_P, int64_t ld, int ncols, int64_t n, int64_t g0,
                        int64_t N, const double* d_state_in, double* d_state_out,
                        double* d_scratch, void* stream) {
  return guard([&] {
    PG_REQUIRE(ncols >= 1 && ncols <= PG_KMAX, PG_ERR_PARAMETER, "ncols out of range");
    PG_REQUIRE(n >= 0 && g0 >= 0 && g0 + n <= N && ld >= n, PG_ERR_DIMENSION,
               "shard rows outside the global range");
    PG_REQUIRE(d_state_out && (n == 0 || (d_P && d_scratch)), PG_ERR_PARAMETER,
               "null argument");
    cudaStream_t st = as_stream(stream);
    const int npairs = ncols * (ncols + 1) / 2;
    const KBlocks kb(N);
    double* chain_out = d_state_out;
    double* sum_out = d_state_out + npairs;
    const double* chain_in = d_state_in;
    const double* sum_in = d_state_in ? d_state_in + npairs : nullptr;
    if (n == 0) {  // pass the state through
      if (d_state_in)
        PG_CUDA(cudaMemcpyAsync(d_state_out, d_state_in, sizeof(double) * 2 * npairs,
                                cudaMemcpyDeviceToDevice, st));
      else
        PG_CUDA(cudaMemsetAsync(d_state_out, 0, sizeof(double) * 2 * npairs, st));
      return;
    }
    const int64_t b_lo = kb.of_row(g0), b_hi = kb.of_row(g0 + n - 1);
    PG_REQUIRE(kb.start(b_lo) >= g0 || chain_in, PG_ERR_PARAMETER,
               "shard starts inside a K-block: chain state required");
    const int64_t nblk = b_hi - b_lo + 1;
    PG_REQUIRE(nblk < (int64_t)1 << 31, PG_ERR_PARAMETER, "too many K-blocks");
    const bool open = kb.end(b_hi) > g0 + n;
    const size_t smem = sizeof(double) * (size_t)ncols * kGbStride;
    static bool attr_set = false;
    if (!attr_set) {
      PG_CUDA(cudaFuncSetAttribute(gram_blas_blocks, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(sizeof(double) * PG_KMAX * kGbStride)));
      attr_set = true;
    }
    launch_k(gram_blas_blocks, dim3((unsigned)nblk), dim3(kGbThreads), smem, st, d_P, ld, ncols,
             n, g0, N, b_lo, chain_in, chain_out, d_scratch);
    check_launch();
    const int64_t ndone = open ? nblk - 1 : nblk;
    launch_k(gram_blas_sum, dim3((npairs + kGbThreads - 1) / kGbThreads), dim3(kGbThreads), 0,
             st, npairs, ndone, (const double*)d_scratch, sum_in, sum_out, chain_out, !open);
    check_launch();
  });
}

PG_API int pg_dot_blas(const double* d_x, const double* d_y, int64_t n, int nthreads,
                       double* d_out, void* stream) {
  return guard([&] {
    PG_REQUIRE(d_out && (n == 0 || (d_x && d_y)), PG_ERR_PARAMETER, "null argument");
    PG_REQUIRE(nthreads >= 1 && nthreads <= 32, PG_ERR_PARAMETER, "nthreads must be 1..32");
    cudaStream_t st = as_stream(stream);
    if (n == 0) {
      PG_CUDA(cudaMemsetAsync(d_out, 0, sizeof(double), st));
      return;
    }
    const int T = n <= 10000 ? 1 : nthreads;
    launch_k(dot_blas_kernel, dim3(1), dim3(32 * T), 0, st, d_x, d_y, n, T, d_out);
    check_launch();
  });
}

}  // extern "C"
