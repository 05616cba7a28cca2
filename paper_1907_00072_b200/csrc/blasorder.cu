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
  // completed blocks: partial[p * nblk + block] (pair-major, so that
  // gram_blas_sum reads each pair's blocks contiguously)
#pragma unroll
  for (int m = 0; m < kGbPPT; ++m) {
    const int p = threadIdx.x + m * kGbThreads;
    if (p < npairs) {
      if (open)
        chain_out[p] = acc[m];
      else
        partial[(size_t)p * gridDim.x + blockIdx.x] = acc[m];
    }
  }
}

// C = sum_in; C = C + partial[b] over the shard's completed blocks in order.
// One warp per pair: the lanes load 32 consecutive blocks' partials at a time
// (coalesced, several segments in flight) and every lane runs the same
// sequential sum over them through shuffles -- the reference's order, with
// the data movement spread over many warps (one thread per pair looping over
// 20833 blocks took 2.7 ms at n = 8M).  ndone <= nstride columns per pair.
constexpr int kSumAhead = 4;
__global__ void __launch_bounds__(kGbThreads)
    gram_blas_sum(int npairs, int64_t ndone, int64_t nstride, const double* __restrict__ partial,
                  const double* __restrict__ sum_in, double* __restrict__ sum_out,
                  double* __restrict__ chain_out, bool zero_chain) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int p = blockIdx.x * (kGbThreads / 32) + (threadIdx.x >> 5);
  if (p >= npairs) return;
  const double* src = partial + (size_t)p * nstride;
  double c = sum_in ? sum_in[p] : 0.0;
  const int64_t nseg = (ndone + 31) / 32;
  double v[kSumAhead];
#pragma unroll
  for (int u = 0; u < kSumAhead; ++u) {
    const int64_t b = (int64_t)u * 32 + lane;
    v[u] = b < ndone ? __ldcg(src + b) : 0.0;
  }
  for (int64_t s0 = 0; s0 < nseg; s0 += kSumAhead) {
#pragma unroll
    for (int u = 0; u < kSumAhead; ++u) {
      const int64_t s = s0 + u;
      if (s < nseg) {
        const double cur = v[u];
        const int64_t bn = (s + kSumAhead) * 32 + lane;  // refill this slot kSumAhead ahead
        v[u] = bn < ndone ? __ldcg(src + bn) : 0.0;
        const int cnt = (int)((ndone - s * 32) < 32 ? (ndone - s * 32) : 32);
        for (int j = 0; j < cnt; ++j) c = __dadd_rn(c, __shfl_sync(0xffffffffu, cur, j));
      }
    }
  }
  if (lane == 0) {
    sum_out[p] = c;
    if (zero_chain) chain_out[p] = 0.0;
  }
}

// OpenBLAS x86-64 ddot order (see the file header).  One CTA per chunk:
// warp 0's 32 lanes run the chunk's 32 FMA chains (lane l: elements l, l+32,
// ... in order) from shared memory while the other warps stage the next
// kDotTile elements of x and y (double-buffered), so the chains do not wait
// on one global load batch at a time (one CTA of 16 warps loading for
// itself took 2.1 ms at n = 8M).  The chunk's dot goes to scratch[t];
// dot_blas_sum adds the chunks in order.
constexpr int kDotThreads = 512;
constexpr int kDotTile = 2048;   // elements of x and of y per ring stage
constexpr int kDotStages = 4;    // 128 KB of dynamic shared memory
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__global__ void __launch_bounds__(kDotThreads)
    dot_blas_kernel(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                    int nthreads, double* scratch) {
  pdl_entry();
  extern __shared__ double ring[];  // [kDotStages][2][kDotTile]
  __shared__ double lane_acc[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = blockIdx.x;
  int64_t off = 0, w = 0;
  for (int u = 0; u <= t; ++u) {
    off += w;
    w = (n - off + (nthreads - u) - 1) / (nthreads - u);
  }
  const double* xs = x + off;
  const double* ys = y + off;
  const int64_t n1 = w & ~(int64_t)15, n32 = w & ~(int64_t)31;
  const int64_t ntile = (n32 + kDotTile - 1) / kDotTile;
  // warps 1.. keep kDotStages-1 tiles in flight (8-byte cp.async: the
  // chunk start is not 16-byte aligned in general)
  auto stage = [&](int64_t tile) {
    if (tile < ntile) {
      double* X = ring + (tile % kDotStages) * 2 * kDotTile;
      const int64_t a = tile * kDotTile;
      const int m = (int)((n32 - a) < kDotTile ? (n32 - a) : kDotTile);
      for (int e = threadIdx.x - 32; e < m; e += kDotThreads - 32) {
        cp_async8(X + e, xs + a + e);
        cp_async8(X + kDotTile + e, ys + a + e);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  if (warp > 0)
    for (int s = 0; s < kDotStages - 1; ++s) stage(s);
  double acc = 0.0;
  for (int64_t i = 0; i < ntile; ++i) {
    if (warp > 0) asm volatile("cp.async.wait_group %0;\n" ::"n"(kDotStages - 2) : "memory");
    __syncthreads();  // tile i landed; warp 0 is done with tile i-1
    if (warp == 0) {
      const int m = (int)((n32 - i * kDotTile) < kDotTile ? (n32 - i * kDotTile) : kDotTile);
      const double* X = ring + (i % kDotStages) * 2 * kDotTile;
      const double* Y = X + kDotTile;
      for (int e = lane; e < m; e += 32) acc = __fma_rn(X[e], Y[e], acc);
    } else {
      stage(i + kDotStages - 1);
    }
  }
  if (warp > 0) asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  if (warp == 0) {
    lane_acc[lane] = acc;
    __syncwarp();
    if (lane == 0) {
      double dot = 0.0;
      if (n1 > 0) {
        const double* L = lane_acc;
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
      scratch[t] = dot;
    }
  }
}

// The chunks' dots added in chunk order (one chunk: its dot as is).
__global__ void dot_blas_sum(const double* __restrict__ scratch, int nthreads, double* out) {
  pdl_entry();
  if (threadIdx.x == 0) {
    double d = 0.0;
    for (int u = 0; u < nthreads; ++u) d = __dadd_rn(d, scratch[u]);
    *out = nthreads == 1 ? scratch[0] : d;
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
    const int wpb = kGbThreads / 32;
    launch_k(gram_blas_sum, dim3((npairs + wpb - 1) / wpb), dim3(kGbThreads), 0, st, npairs,
             ndone, nblk, (const double*)d_scratch, sum_in, sum_out, chain_out, !open);
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
    // 32 chunk dots per device, allocated once (before any graph capture:
    // pg_dot_blas is a construction-time call)
    static double* scratch[64] = {};
    int dev = 0;
    PG_CUDA(cudaGetDevice(&dev));
    PG_REQUIRE(dev >= 0 && dev < 64, PG_ERR_PARAMETER, "device ordinal out of range");
    if (!scratch[dev]) {
      PG_REQUIRE(!g_capturing, PG_ERR_PARAMETER, "pg_dot_blas first called inside a capture");
      PG_CUDA(cudaMalloc(&scratch[dev], 32 * sizeof(double)));
    }
    static bool dot_attr[64] = {};
    if (!dot_attr[dev]) {
      PG_CUDA(cudaFuncSetAttribute(dot_blas_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(sizeof(double) * kDotStages * 2 * kDotTile)));
      dot_attr[dev] = true;
    }
    launch_k(dot_blas_kernel, dim3(T), dim3(kDotThreads), sizeof(double) * kDotStages * 2 * kDotTile,
             st, d_x, d_y, n, T, scratch[dev]);
    check_launch();
    launch_k(dot_blas_sum, dim3(1), dim3(32), 0, st, (const double*)scratch[dev], T, d_out);
    check_launch();
  });
}

}  // extern "C"
