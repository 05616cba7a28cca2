// libpgmres: tall-skinny kernels -- CGS2 phases (ortho.py:33-70), the
// power-basis Gram matrix (polyprec.py:115-122), the recovery GEMV
// (gmres.py:326) and the small vector kernels.
//
// All of these are HBM-bound (<= 0.25 flop/B), so no tensor cores: the point
// is to read each basis column the minimum number of times.  The reference
// makes 4 passes over V per CGS2 step (two dgemv_T, two dgemv_N); here:
//   phase 1  c1 = V^T z                         1 read of V
//   phase 2  w1 = z - V c1 (row-local), c2 = V^T w1   1 read of V (tile in smem)
//   phase 3  w2 = (z - V c1) - V c2, |w2|^2     1 read of V (w1 recomputed)
// Reductions are deterministic: fixed per-lane / per-warp / per-block order,
// then the last block to finish sums the block partials in block order.
//
// Tile kernels stage a 128-row x (k[+1]) column tile in shared memory with
// 16-byte cp.async copies, double buffered, so the next tile's HBM reads are
// in flight while the current tile is reduced.

#include <cuda.h>

#include <cstdio>
#include <cstdlib>

#include "internal.cuh"
#include "pipeline.cuh"

namespace pg {

// Tile heights: 128 rows, or 256 for narrower bases (tile_rows_for): at
// n = 1e6, k = 25 phase 1 48.5 -> 43.2 us and phase 2 57.1 -> 51.0 with 256;
// at k >= 40 the taller tiles' shallower rings lose (72.8 vs 64.8 us).
constexpr int kTileRows = 128;
template <int TR>
struct TileShape {
  static constexpr int kStride = TR + 2;  // 16-B aligned column stride (doubles)
};
constexpr int kTileStride = TileShape<kTileRows>::kStride;
constexpr int kTileThreads = 256;
constexpr int kWarps = kTileThreads / 32;
constexpr int kColsPerWarp = (PG_KMAX + kWarps - 1) / kWarps;               // 8
constexpr int kPairsPerThread = (PG_KMAX * (PG_KMAX + 1) / 2 + kTileThreads - 1) / kTileThreads;  // 9

enum TileMode { kDots = 1, kUpdDots = 2, kGram = 3 };

__device__ __forceinline__ void cp_async16(double* dst, const double* src, int bytes) {
  unsigned saddr = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(src),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Stage tile `tile` of columns 0..ncol-1 (column k = z when z != nullptr).
// Warp w copies columns w, w + 8, ...: each lane two 16-byte pieces of a
// 1 KB column segment, the column's address computed once per column; full
// tiles need no per-piece bounds (ncu: the tile kernels were issue-bound,
// 57% issue-active, largely on the per-piece address arithmetic).
template <int TR>
__device__ __forceinline__ void stage_tile(double* buf, const double* __restrict__ V, int64_t ld,
                                           int k, const double* __restrict__ z, int64_t n,
                                           int64_t tile) {
  constexpr int kStride = TileShape<TR>::kStride;
  const int ncol = z ? k + 1 : k;
  const int64_t row0 = tile * TR;
  const int64_t rows = min((int64_t)TR, n - row0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (rows == TR) {
    for (int colx = warp; colx < ncol; colx += kTileThreads / 32) {
      const double* src = (colx < k ? V + (int64_t)colx * ld : z) + row0 + 2 * lane;
      double* dst = buf + colx * kStride + 2 * lane;
#pragma unroll
      for (int h = 0; h < TR / 64; ++h) cp_async16(dst + 64 * h, src + 64 * h, 16);
    }
    return;
  }
  constexpr int kChunks = TR / 2;
  for (int c = threadIdx.x; c < ncol * kChunks; c += kTileThreads) {
    const int colx = c / kChunks, ch = c - colx * kChunks;
    const double* src = (colx < k ? V + (int64_t)colx * ld : z) + row0 + 2 * ch;
    const int64_t valid = rows - 2 * ch;
    int bytes = valid >= 2 ? 16 : (valid == 1 ? 8 : 0);
    if (bytes == 0) src = V ? V : z;  // not dereferenced; keep the address legal
    cp_async16(buf + colx * kStride + 2 * ch, src, bytes);
  }
}

// Error-free transformations for the compensated Gram sums: the power-basis
// normal equations are so ill-conditioned (cond ~1e14 at the usable degrees)
// that the Cholesky-failure degree signal (polyprec.py:80-82) is decided by
// the rounding of G.  Accumulating each entry in double-double makes G
// accurate to ~1 ulp, so the device takes the exact-arithmetic decision.
__device__ __forceinline__ void dd_add(double x, double& hi, double& lo) {
  const double s = __dadd_rn(hi, x);
  const double bb = __dsub_rn(s, hi);
  const double err = __dadd_rn(__dsub_rn(hi, __dsub_rn(s, bb)), __dsub_rn(x, bb));
  hi = s;
  lo = __dadd_rn(lo, err);
}
__device__ __forceinline__ void dd_fma(double a, double b, double& hi, double& lo) {
  const double p = __dmul_rn(a, b);
  const double e = __fma_rn(a, b, -p);  // exact product error
  dd_add(p, hi, lo);
  lo = __dadd_rn(lo, e);
}

// Row projection t = sum_i V[r,i] c[i], sequential in i with FMA.  Phase 2
// (from the smem tile) and phase 3 (from global) use this same order, so the
// recomputed w1 is bit-identical.
template <class Load>
__device__ __forceinline__ double row_proj(int k, const double* c, Load load) {
  double t = 0.0;
  for (int i = 0; i < k; ++i) t = __fma_rn(load(i), c[i], t);
  return t;
}

template <int MODE, int STAGES, int TR>
__global__ void __launch_bounds__(kTileThreads)
    tile_kernel(const double* __restrict__ V, int64_t ld, int k, const double* __restrict__ z,
                int64_t n, const double* __restrict__ c1, double* partials,
                unsigned int* counter, double* out) {
  pdl_entry();
  constexpr int kStr = TileShape<TR>::kStride;
  extern __shared__ __align__(16) double smem[];
  __shared__ double c1s[PG_KMAX];
  const bool has_z = (MODE != kGram);
  const int ncol = has_z ? k + 1 : k;
  const int buf_elems = ncol * kStr;
  double* w1s = smem + STAGES * buf_elems;  // kUpdDots only
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  if (MODE == kUpdDots)
    for (int i = threadIdx.x; i < k; i += kTileThreads) c1s[i] = c1[i];

  const int64_t ntiles = (n + TR - 1) / TR;
  int64_t tile = blockIdx.x;

  // per-thread accumulators
  constexpr int NACC = (MODE == kGram) ? kPairsPerThread : kColsPerWarp;
  double acc[NACC];
  double acc_lo[(MODE == kGram) ? kPairsPerThread : 1];
#pragma unroll
  for (int m = 0; m < NACC; ++m) acc[m] = 0.0;
#pragma unroll
  for (int m = 0; m < (MODE == kGram ? kPairsPerThread : 1); ++m) acc_lo[m] = 0.0;
  int pi[kPairsPerThread], pj[kPairsPerThread];
  const int npairs = k * (k + 1) / 2;
  if (MODE == kGram) {
#pragma unroll
    for (int m = 0; m < kPairsPerThread; ++m) {
      int p = threadIdx.x + m * kTileThreads, i = 0;
      if (p < npairs) {
        int rem = p;
        while (rem >= k - i) { rem -= k - i; ++i; }
        pi[m] = i;
        pj[m] = i + rem;
      } else {
        pi[m] = pj[m] = -1;
      }
    }
  }

  // STAGES-deep cp.async ring: STAGES-1 tiles in flight while one is reduced
  __shared__ int64_t ctag[STAGES];  // PG_CHECKS: the tile a slot holds
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    const int64_t t = tile + (int64_t)s * gridDim.x;
    if (t < ntiles) stage_tile<TR>(smem + s * buf_elems, V, ld, k, has_z ? z : nullptr, n, t);
    if (PG_CHECKS && threadIdx.x == 0) ctag[s] = t;
    cp_async_commit();
  }
  int it = 0;
  for (; tile < ntiles; tile += gridDim.x, ++it) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();  // tile `it` landed; every thread is done with tile it-1
    {
      // refill the slot of tile it-1 before reducing tile it, so the copy
      // overlaps this tile's compute even with a 2-deep ring
      const int64_t t = tile + (int64_t)(STAGES - 1) * gridDim.x;
      if (t < ntiles)
        stage_tile<TR>(smem + ((it + STAGES - 1) % STAGES) * buf_elems, V, ld, k,
                   has_z ? z : nullptr, n, t);
      if (PG_CHECKS && threadIdx.x == 0) ctag[(it + STAGES - 1) % STAGES] = t;
      cp_async_commit();
    }
    PG_DCHECK(ctag[it % STAGES] == tile);
    const double* S = smem + (it % STAGES) * buf_elems;

    if (MODE == kDots || MODE == kUpdDots) {
      const double* vec = S + k * kStr;  // z column
      if (MODE == kUpdDots) {
        if (threadIdx.x < TR) {
          const int r = threadIdx.x;
          const double t = row_proj(k, c1s, [&](int i) { return S[i * kStr + r]; });
          w1s[r] = __dsub_rn(S[k * kStr + r], t);
        }
        __syncthreads();
        vec = w1s;
      }
#pragma unroll
      for (int m = 0; m < kColsPerWarp; ++m) {
        const int i = warp + m * kWarps;
        if (i < k) {
          const double* col = S + i * kStr;
#pragma unroll
          for (int q = 0; q < TR / 32; ++q)
            acc[m] = __fma_rn(col[lane + 32 * q], vec[lane + 32 * q], acc[m]);
        }
      }
    } else {  // Gram: all pairs i <= j, compensated (double-double) sums
#pragma unroll
      for (int m = 0; m < kPairsPerThread; ++m) {
        if (pi[m] >= 0) {
          const double* a = S + pi[m] * kStr;
          const double* b = S + pj[m] * kStr;
          double hi = acc[m], lo = acc_lo[m];
#pragma unroll 4
          for (int r = 0; r < TR; ++r) dd_fma(a[r], b[r], hi, lo);
          acc[m] = hi;
          acc_lo[m] = lo;
        }
      }
    }
  }
  cp_async_wait<0>();

  // block partials, then deterministic cross-block finish
  if (MODE == kGram) {
    // packed upper triangle, (hi, lo) per pair
    double* part = partials + (size_t)blockIdx.x * (2 * npairs);
#pragma unroll
    for (int m = 0; m < kPairsPerThread; ++m) {
      const int p = threadIdx.x + m * kTileThreads;
      if (p < npairs) {
        part[2 * p] = acc[m];
        part[2 * p + 1] = acc_lo[m];
      }
    }
    __shared__ bool am_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) am_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!am_last) return;
    __threadfence();
    for (int p = threadIdx.x; p < npairs; p += blockDim.x) {
      double hi = 0.0, lo = 0.0;
      for (unsigned b = 0; b < gridDim.x; ++b) {
        dd_add(__ldcg(partials + (size_t)b * 2 * npairs + 2 * p), hi, lo);
        lo += __ldcg(partials + (size_t)b * 2 * npairs + 2 * p + 1);
      }
      int i = 0, rem = p;
      while (rem >= k - i) { rem -= k - i; ++i; }
      const int j = i + rem;
      // G = hi_r + lo_r exactly-ish: hi_r is G rounded to double, lo_r the
      // remainder, so shards can be combined in double-double (Engine.gram)
      const double hr = hi + lo;
      const double lr = (hi - hr) + lo;
      out[i * k + j] = hr;
      out[j * k + i] = hr;
      out[k * k + i * k + j] = lr;
      out[k * k + j * k + i] = lr;
    }
    if (threadIdx.x == 0) *counter = 0u;
  } else {
#pragma unroll
    for (int m = 0; m < kColsPerWarp; ++m) {
      double v = acc[m];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      const int i = warp + m * kWarps;
      if (lane == 0 && i < k) partials[(size_t)blockIdx.x * k + i] = v;
    }
    last_block_reduce(partials, counter, k, out);
  }
}

// ---------------------------------------------------------------------------
// Phases 1 and 2 with the tiles loaded by the tensor-memory accelerator: V as
// a 2-D tensor map (rows x columns, column stride ld), one
// cp.async.bulk.tensor.2d per 8 columns of a TR-row tile plus one 1-D tensor
// copy of z's segment, issued by one thread and completing on the slot's
// mbarrier; rows past n (and columns past k in the last 8-column box) arrive
// zero-filled.  The per-lane 16-byte cp.async staging of tile_kernel costs
// ~11 copy instructions per thread per tile; here the other threads only
// compute.  Same arithmetic and order as tile_kernel (kDots, kUpdDots).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

constexpr int kTmaBoxCols = 8;

template <int MODE, int STAGES, int TR>
__global__ void __launch_bounds__(kTileThreads)
    tma_tile_kernel(const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmZ,
                    int k, int64_t n, const double* __restrict__ c1, double* partials,
                    unsigned int* counter, double* out) {
  static_assert(MODE == kDots || MODE == kUpdDots, "dots phases only");
  pdl_entry();
  extern __shared__ __align__(128) double smem[];
  __shared__ double c1s[PG_KMAX];
  __shared__ __align__(8) uint64_t full[STAGES];
  __shared__ int64_t ttag[STAGES];  // PG_CHECKS: the tile a slot holds
  const int nbox = (k + kTmaBoxCols - 1) / kTmaBoxCols;
  const int zcol = nbox * kTmaBoxCols;  // z's column slot
  const int buf_elems = (zcol + 1) * TR;
  double* w1s = smem + STAGES * buf_elems;  // kUpdDots only
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t tile_bytes = 8u * (uint32_t)((zcol + 1) * TR);
  if (MODE == kUpdDots)
    for (int i = threadIdx.x; i < k; i += kTileThreads) c1s[i] = c1[i];
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  const int64_t ntiles = (n + TR - 1) / TR;
  auto issue = [&](int64_t t, int slot) {
    double* buf = smem + (size_t)slot * buf_elems;
    if (PG_CHECKS) ttag[slot] = t;
    mbar_expect_tx(&full[slot], tile_bytes);
    const int r0 = (int)(t * TR);
    for (int b = 0; b < nbox; ++b)
      tma_load_2d(buf + (size_t)b * kTmaBoxCols * TR, &tmV, r0, b * kTmaBoxCols, &full[slot]);
    tma_load_2d(buf + (size_t)zcol * TR, &tmZ, r0, 0, &full[slot]);
  };
  int64_t tile = blockIdx.x;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      const int64_t t = tile + (int64_t)s * gridDim.x;
      if (t < ntiles) issue(t, s);
    }
  }
  double acc[kColsPerWarp];
#pragma unroll
  for (int m = 0; m < kColsPerWarp; ++m) acc[m] = 0.0;
  int it = 0;
  for (; tile < ntiles; tile += gridDim.x, ++it) {
    // every thread is done with tile it-1: refill its slot
    __syncthreads();
    if (threadIdx.x == 0) {
      const int64_t t = tile + (int64_t)(STAGES - 1) * gridDim.x;
      if (t < ntiles) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        issue(t, (it + STAGES - 1) % STAGES);
      }
    }
    const int slot = it % STAGES;
    mbar_wait(&full[slot], (uint32_t)((it / STAGES) & 1));
    PG_DCHECK(ttag[slot] == tile);
    const double* S = smem + (size_t)slot * buf_elems;
    const double* vec = S + (size_t)zcol * TR;
    if (MODE == kUpdDots) {
      if (threadIdx.x < TR) {
        const int r = threadIdx.x;
        const double t = row_proj(k, c1s, [&](int i) { return S[i * TR + r]; });
        w1s[r] = __dsub_rn(vec[r], t);
      }
      __syncthreads();
      vec = w1s;
    }
#pragma unroll
    for (int m = 0; m < kColsPerWarp; ++m) {
      const int i = warp + m * kWarps;
      if (i < k) {
        const double* col = S + i * TR;
#pragma unroll
        for (int q = 0; q < TR / 32; ++q)
          acc[m] = __fma_rn(col[lane + 32 * q], vec[lane + 32 * q], acc[m]);
      }
    }
    if (MODE == kUpdDots) __syncthreads();  // w1s is rewritten by the next tile
  }
#pragma unroll
  for (int m = 0; m < kColsPerWarp; ++m) {
    double v = acc[m];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int i = warp + m * kWarps;
    if (lane == 0 && i < k) partials[(size_t)blockIdx.x * k + i] = v;
  }
  last_block_reduce(partials, counter, k, out);
}

// Phase 3 through the same tensor-map staging: a tile of 256 rows x (k
// columns + z) per stage, one row per thread -- both projections from the
// tile (the same sequential FMA order as rows_kernel<true>, so w1 and w2 are
// bit-identical to it), w2 stored, ||w2||^2 accumulated per thread over its
// tiles (the rows thread t of block b takes in rows_kernel with the same
// grid).  The loads are one producer thread's bulk copies instead of 8-wide
// batches of per-thread streaming loads.
constexpr int kRowsTileRows = 256;
template <int STAGES>
__global__ void __launch_bounds__(kTileThreads)
    tma_rows_kernel(const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmZ,
                    int k, int64_t n, const double* __restrict__ c1, const double* __restrict__ c2,
                    double* __restrict__ out, double* partials, unsigned int* counter,
                    double* nsq) {
  constexpr int TR = kRowsTileRows;
  static_assert(TR == kTileThreads, "one row per thread");
  pdl_entry();
  extern __shared__ __align__(128) double smem[];
  __shared__ double c1s[PG_KMAX], c2s[PG_KMAX];
  __shared__ __align__(8) uint64_t full[STAGES];
  __shared__ int64_t ttag[STAGES];  // PG_CHECKS: the tile a slot holds
  const int nbox = (k + kTmaBoxCols - 1) / kTmaBoxCols;
  const int zcol = nbox * kTmaBoxCols;
  const int buf_elems = (zcol + 1) * TR;
  const uint32_t tile_bytes = 8u * (uint32_t)((zcol + 1) * TR);
  for (int i = threadIdx.x; i < k; i += kTileThreads) {
    c1s[i] = c1[i];
    c2s[i] = c2[i];
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  const int64_t ntiles = (n + TR - 1) / TR;
  auto issue = [&](int64_t t, int slot) {
    double* buf = smem + (size_t)slot * buf_elems;
    if (PG_CHECKS) ttag[slot] = t;
    mbar_expect_tx(&full[slot], tile_bytes);
    const int r0 = (int)(t * TR);
    for (int b = 0; b < nbox; ++b)
      tma_load_2d(buf + (size_t)b * kTmaBoxCols * TR, &tmV, r0, b * kTmaBoxCols, &full[slot]);
    tma_load_2d(buf + (size_t)zcol * TR, &tmZ, r0, 0, &full[slot]);
  };
  int64_t tile = blockIdx.x;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      const int64_t t = tile + (int64_t)s * gridDim.x;
      if (t < ntiles) issue(t, s);
    }
  }
  double local = 0.0;
  const int r = threadIdx.x;
  int it = 0;
  for (; tile < ntiles; tile += gridDim.x, ++it) {
    __syncthreads();  // every thread is done with tile it-1: refill its slot
    if (threadIdx.x == 0) {
      const int64_t t = tile + (int64_t)(STAGES - 1) * gridDim.x;
      if (t < ntiles) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        issue(t, (it + STAGES - 1) % STAGES);
      }
    }
    const int slot = it % STAGES;
    mbar_wait(&full[slot], (uint32_t)((it / STAGES) & 1));
    PG_DCHECK(ttag[slot] == tile);
    const double* S = smem + (size_t)slot * buf_elems;
    double t1 = 0.0, t2 = 0.0;
    for (int i = 0; i < k; ++i) {
      const double v = S[i * TR + r];
      t1 = __fma_rn(v, c1s[i], t1);
      t2 = __fma_rn(v, c2s[i], t2);
    }
    const int64_t row = tile * TR + r;
    if (row < n) {
      const double w1 = __dsub_rn(S[(size_t)zcol * TR + r], t1);
      const double w2 = __dsub_rn(w1, t2);
      out[row] = w2;
      local = __fma_rn(w2, w2, local);
    }
  }
  const double s = block_sum(local);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
  last_block_reduce(partials, counter, 1, nsq);
}

constexpr int kRowThreads = 256;
// phase 3 row loop with the next column group's loads in flight (A/B: 0)
#ifndef PG_ROWS_PIPE
#define PG_ROWS_PIPE 0
#endif

template <bool PHASE3>
__global__ void __launch_bounds__(kRowThreads)
    rows_kernel(const double* __restrict__ V, int64_t ld, int k, const double* __restrict__ z,
                int64_t n, const double* __restrict__ c1, const double* __restrict__ c2,
                double* __restrict__ out, double* partials, unsigned int* counter, double* nsq) {
  pdl_entry();
  __shared__ double cs1[PG_KMAX], cs2[PG_KMAX];
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    cs1[i] = c1[i];
    if (PHASE3) cs2[i] = c2[i];
  }
  __syncthreads();
  double local = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride) {
    const double* vr = V + r;
    if (PHASE3) {
      double t1 = 0.0, t2 = 0.0;
      int i = 0;
#if PG_ROWS_PIPE
      // software-pipelined: the next 8 columns' loads are issued before this
      // group's FMAs (same sequential order per row)
      if (k >= 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcs(vr + (int64_t)u * ld);
        for (; i + 16 <= k; i += 8) {
          double vn[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) vn[u] = __ldcs(vr + (int64_t)(i + 8 + u) * ld);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            t1 = __fma_rn(v[u], cs1[i + u], t1);
            t2 = __fma_rn(v[u], cs2[i + u], t2);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = vn[u];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          t1 = __fma_rn(v[u], cs1[i + u], t1);
          t2 = __fma_rn(v[u], cs2[i + u], t2);
        }
        i += 8;
      }
#else
      for (; i + 8 <= k; i += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcs(vr + (int64_t)(i + u) * ld);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          t1 = __fma_rn(v[u], cs1[i + u], t1);
          t2 = __fma_rn(v[u], cs2[i + u], t2);
        }
      }
#endif
      for (; i < k; ++i) {
        const double v = __ldcs(vr + (int64_t)i * ld);
        t1 = __fma_rn(v, cs1[i], t1);
        t2 = __fma_rn(v, cs2[i], t2);
      }
      const double w1 = __dsub_rn(z[r], t1);
      const double w2 = __dsub_rn(w1, t2);
      out[r] = w2;
      local = __fma_rn(w2, w2, local);
    } else {
      double t = 0.0;
      int i = 0;
      for (; i + 8 <= k; i += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcs(vr + (int64_t)(i + u) * ld);
#pragma unroll
        for (int u = 0; u < 8; ++u) t = __fma_rn(v[u], cs1[i + u], t);
      }
      for (; i < k; ++i) t = __fma_rn(__ldcs(vr + (int64_t)i * ld), cs1[i], t);
      out[r] = t;
    }
  }
  if (PHASE3) {
    const double s = block_sum(local);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
    last_block_reduce(partials, counter, 1, nsq);
  }
}

// ---------------------------------------------------------------------------
// Warp-chunk CGS2 kernels (the default path).  A warp owns chunks of
// kChunkRows = 32 * kR consecutive rows, lane l holding rows l, l+32, ...;
// every column read is a coalesced 256 B segment and kCol columns x kR rows
// of loads are issued before they are consumed.  No shared-memory staging,
// small register footprint -> full occupancy, which is what an HBM-latency
// bound kernel needs.  Column dots are reduced across the warp with a fixed
// xor tree per chunk; lane (i mod 32) keeps column i's running sum.
// ---------------------------------------------------------------------------
constexpr int kR = 4;
constexpr int kChunkRows = 32 * kR;
constexpr int kCol = 4;
constexpr int kChunkThreads = 256;

struct ChunkRows {
  int64_t r[kR];
  bool ok[kR];
};

__device__ __forceinline__ ChunkRows chunk_rows(int64_t chunk, int lane, int64_t n) {
  ChunkRows c;
#pragma unroll
  for (int q = 0; q < kR; ++q) {
    c.r[q] = chunk * kChunkRows + lane + 32 * q;
    c.ok[q] = c.r[q] < n;
  }
  return c;
}

// t[q] = sum_i V[r_q, i] * c[i] in sequential i order (FMA) -- the same order
// as row_proj, so phase 2 and phase 3 recompute bit-identical w1.
__device__ __forceinline__ void chunk_proj(const double* __restrict__ V, int64_t ld, int k,
                                           const ChunkRows& cr, const double* c, double* t) {
#pragma unroll
  for (int q = 0; q < kR; ++q) t[q] = 0.0;
  int i = 0;
  for (; i + kCol <= k; i += kCol) {
    double v[kCol][kR];
#pragma unroll
    for (int u = 0; u < kCol; ++u)
#pragma unroll
      for (int q = 0; q < kR; ++q)
        v[u][q] = cr.ok[q] ? __ldg(V + (int64_t)(i + u) * ld + cr.r[q]) : 0.0;
#pragma unroll
    for (int u = 0; u < kCol; ++u)
#pragma unroll
      for (int q = 0; q < kR; ++q) t[q] = __fma_rn(v[u][q], c[i + u], t[q]);
  }
  for (; i < k; ++i)
#pragma unroll
    for (int q = 0; q < kR; ++q)
      t[q] = __fma_rn(cr.ok[q] ? __ldg(V + (int64_t)i * ld + cr.r[q]) : 0.0, c[i], t[q]);
}

template <int MODE>  // 1: c = V^T z;  2: w1 = z - V c1 (row-local), c = V^T w1
__global__ void __launch_bounds__(kChunkThreads)
    chunk_dots_kernel(const double* __restrict__ V, int64_t ld, int k,
                      const double* __restrict__ z, int64_t n, const double* __restrict__ c1,
                      double* partials, unsigned int* counter, double* out) {
  pdl_entry();
  __shared__ double cs[PG_KMAX];
  __shared__ double wsum[kChunkThreads / 32][PG_KMAX];
  if (MODE == 2)
    for (int i = threadIdx.x; i < k; i += blockDim.x) cs[i] = c1[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nchunks = (n + kChunkRows - 1) / kChunkRows;
  const int64_t nw = (int64_t)gridDim.x * (kChunkThreads / 32);
  double acc0 = 0.0, acc1 = 0.0;  // columns lane and lane + 32
  for (int64_t ch = (int64_t)blockIdx.x * (kChunkThreads / 32) + warp; ch < nchunks; ch += nw) {
    const ChunkRows cr = chunk_rows(ch, lane, n);
    double w[kR];
#pragma unroll
    for (int q = 0; q < kR; ++q) w[q] = cr.ok[q] ? z[cr.r[q]] : 0.0;
    if (MODE == 2) {
      double t[kR];
      chunk_proj(V, ld, k, cr, cs, t);
#pragma unroll
      for (int q = 0; q < kR; ++q) w[q] = __dsub_rn(w[q], t[q]);
    }
    int i = 0;
    for (; i < k; i += kCol) {
      double p[kCol];
#pragma unroll
      for (int u = 0; u < kCol; ++u) {
        p[u] = 0.0;
        if (i + u < k) {
#pragma unroll
          for (int q = 0; q < kR; ++q)
            p[u] = __fma_rn(cr.ok[q] ? __ldg(V + (int64_t)(i + u) * ld + cr.r[q]) : 0.0, w[q],
                            p[u]);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int u = 0; u < kCol; ++u) p[u] += __shfl_xor_sync(0xffffffffu, p[u], o);
#pragma unroll
      for (int u = 0; u < kCol; ++u) {
        const int col = i + u;
        if (col < k && lane == (col & 31)) {
          if (col < 32) acc0 += p[u];
          else acc1 += p[u];
        }
      }
    }
  }
  if (lane < k) wsum[warp][lane] = acc0;
  if (lane + 32 < k) wsum[warp][lane + 32] = acc1;
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kChunkThreads / 32; ++w) s += wsum[w][i];
    partials[(size_t)blockIdx.x * k + i] = s;
  }
  last_block_reduce(partials, counter, k, out);
}

// phase 3: w2 = (z - V c1) - V c2 -> out, sum w2^2 -> nsq
__global__ void __launch_bounds__(kChunkThreads)
    chunk_update_kernel(const double* __restrict__ V, int64_t ld, int k,
                        const double* __restrict__ z, int64_t n, const double* __restrict__ c1,
                        const double* __restrict__ c2, double* __restrict__ out,
                        double* partials, unsigned int* counter, double* nsq) {
  pdl_entry();
  __shared__ double cs1[PG_KMAX], cs2[PG_KMAX];
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    cs1[i] = c1[i];
    cs2[i] = c2[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nchunks = (n + kChunkRows - 1) / kChunkRows;
  const int64_t nw = (int64_t)gridDim.x * (kChunkThreads / 32);
  double local = 0.0;
  for (int64_t ch = (int64_t)blockIdx.x * (kChunkThreads / 32) + warp; ch < nchunks; ch += nw) {
    const ChunkRows cr = chunk_rows(ch, lane, n);
    double t1[kR], t2[kR];
#pragma unroll
    for (int q = 0; q < kR; ++q) t1[q] = t2[q] = 0.0;
    int i = 0;
    for (; i + kCol <= k; i += kCol) {
      double v[kCol][kR];
#pragma unroll
      for (int u = 0; u < kCol; ++u)
#pragma unroll
        for (int q = 0; q < kR; ++q)
          v[u][q] = cr.ok[q] ? __ldcs(V + (int64_t)(i + u) * ld + cr.r[q]) : 0.0;
#pragma unroll
      for (int u = 0; u < kCol; ++u)
#pragma unroll
        for (int q = 0; q < kR; ++q) {
          t1[q] = __fma_rn(v[u][q], cs1[i + u], t1[q]);
          t2[q] = __fma_rn(v[u][q], cs2[i + u], t2[q]);
        }
    }
    for (; i < k; ++i)
#pragma unroll
      for (int q = 0; q < kR; ++q) {
        const double v = cr.ok[q] ? __ldcs(V + (int64_t)i * ld + cr.r[q]) : 0.0;
        t1[q] = __fma_rn(v, cs1[i], t1[q]);
        t2[q] = __fma_rn(v, cs2[i], t2[q]);
      }
#pragma unroll
    for (int q = 0; q < kR; ++q) {
      if (cr.ok[q]) {
        const double w2 = __dsub_rn(__dsub_rn(z[cr.r[q]], t1[q]), t2[q]);
        out[cr.r[q]] = w2;
        local = __fma_rn(w2, w2, local);
      }
    }
  }
  const double s = block_sum(local);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
  last_block_reduce(partials, counter, 1, nsq);
}

__global__ void dot_kernel(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                           double* partials, unsigned int* counter, double* out) {
  pdl_entry();
  double local = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    local = __fma_rn(x[i], y[i], local);
  const double s = block_sum(local);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
  last_block_reduce(partials, counter, 1, out);
}

__global__ void normalize_kernel(const double* __restrict__ x, const double* __restrict__ nsq,
                                 int64_t n, double* __restrict__ out) {
  pdl_entry();
  const double nrm = sqrt(*nsq);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = __ddiv_rn(x[i], nrm);
}

// normalize_kernel + publish: block 0 also copies the step's scalar ring
// [c1 | c2 | |w2|^2] into the caller's pinned host ring through its mapped
// (UVA) address, so no D2H copy sits on the stream between two Arnoldi
// steps (a copy-engine transfer there cost ~20-30 us per step).
__global__ void normalize_publish_kernel(const double* __restrict__ x,
                                         const double* __restrict__ nsq, int64_t n,
                                         double* __restrict__ out, const double* __restrict__ ring,
                                         int count, double* host) {
  pdl_entry();
  const double nrm = sqrt(*nsq);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = __ddiv_rn(x[i], nrm);
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < count; i += blockDim.x) host[i] = ring[i];
    __threadfence_system();
  }
}

__global__ void scale_add_kernel(const double* base, double a, const double* v, int64_t n,
                                 double* out) {
  pdl_entry();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double t = __dmul_rn(a, v[i]);
    out[i] = base ? __dadd_rn(base[i], t) : t;
  }
}

__global__ void gather_kernel(const double* __restrict__ x, const int32_t* __restrict__ idx,
                              int64_t m, double* __restrict__ out) {
  pdl_entry();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride)
    out[i] = x[idx[i]];
}

// ------------------------------------------------------------------ host --
static int current_device() {
  int d = 0;
  PG_CUDA(cudaGetDevice(&d));
  return d;
}

static void check_ws(pg_workspace* ws) {
  PG_REQUIRE(ws, PG_ERR_PARAMETER, "workspace is null");
  PG_REQUIRE(ws->device == current_device(), PG_ERR_PARAMETER,
             "workspace belongs to another device");
}

static void check_tall(const double* V, int64_t ld, int k, int64_t n, int kmin) {
  PG_REQUIRE(n >= 0, PG_ERR_DIMENSION, "n must be non-negative");
  PG_REQUIRE(k >= kmin && k <= PG_KMAX, PG_ERR_DIMENSION, "basis width out of range");
  PG_REQUIRE(k == 0 || (V && ld >= n), PG_ERR_DIMENSION, "leading dimension smaller than n");
}

// dynamic shared memory budget per CTA (227 KB opt-in limit minus the static
// c1s / reduction arrays)
constexpr size_t kTileSmemMax = 224 * 1024;

static size_t tile_smem(int mode, int k, int stages, int tr = kTileRows) {
  const int ncol = (mode == kGram) ? k : k + 1;
  size_t b = sizeof(double) * (size_t)stages * ncol * (tr + 2);
  if (mode == kUpdDots) b += sizeof(double) * tr;
  return b;
}

// Tile height per phase and basis width (see TileShape): 256 rows up to
// k = 32 at n <= 2M and k = 25 beyond (phase 2 only at n <= 2M), where they
// measured faster; 128 otherwise and for the Gram (n = 8M, k = 32: phase 1
// 411 us with 256-row tiles vs ~340 with 128).  PG_TILE_ROWS = 128 / 256
// forces one.
static int tile_rows_for(int mode, int k, int64_t n) {
  static int force = -1;
  if (force < 0) {
    const char* e = std::getenv("PG_TILE_ROWS");
    force = e ? std::atoi(e) : 0;
  }
  if (mode == kGram) return 128;
  if (force == 128 || force == 256) return force;
  const bool small = n <= (int64_t)2000000;
  if (k > 32 || (!small && k > 25)) return 128;
  if (mode == kUpdDots && !small) return 128;
  return 256;
}

// Ring depth: the deepest ring (<= 4 stages) that still lets `ctas` CTAs
// share an SM (the occupancy calculator then co-locates as many CTAs as the
// ring leaves room for).  Sweep on B200 (tools/cgs2_bench.py with
// PG_TILE_CTAS_P1/P2 = 1..4 at n = 1e6 and 8e6, k = 16..51,
// profiles/r01e/cgs2_ring_sweep.md):
//  * phase 1 (c = V^T z): the deepest ring (ctas = 1) wins at n <= 2M for
//    every k (k = 25: 48.3 vs 55.7 us with ctas = 3) and at n = 8M from
//    k = 35; below that a 4-CTA ring (k = 20: 212 vs 227 us);
//  * phase 2 (w1 and c = V^T w1, a serial row projection per tile): more
//    co-resident CTAs hide it -- 4 up to k = 20, 3 up to k = 35, then 3 at
//    n <= 2M and 2 at 8M (k = 51: 672 vs 871 us with ctas = 1);
//  * the Gram keeps one deep ring (FP64-bound, insensitive).
static int tile_stages(int mode, int k, int64_t n, int tr) {
  // PG_TILE_CTAS_P{1,2,3}: CTAs per SM the ring is sized for (experiments)
  static int ctas_env[4] = {-1, -1, -1, -1};
  if (ctas_env[mode] < 0) {
    const char* names[4] = {"", "PG_TILE_CTAS_P1", "PG_TILE_CTAS_P2", "PG_TILE_CTAS_P3"};
    const char* s = std::getenv(names[mode]);
    ctas_env[mode] = s ? std::atoi(s) : 0;
  }
  const bool small = n <= (int64_t)2000000;
  int ctas;
  if (mode == kGram)
    ctas = 1;
  else if (mode == kDots)
    ctas = (small || k >= 35) ? 1 : 4;
  else
    ctas = k <= 20 ? 4 : k <= 35 ? 3 : (small ? 3 : 2);
  if (ctas_env[mode] > 0) ctas = ctas_env[mode];
  const size_t per_sm = kTileSmemMax / ctas;
  for (int s = 4; s > 2; --s)
    if (tile_smem(mode, k, s, tr) <= per_sm) return s;
  return 2;
}

// Resident-grid size for a chunk kernel (cached per kernel and device),
// limited by the work: one warp per 128-row chunk at most.
static int chunk_grid(const void* kernel, int slot, int dev, int64_t n) {
  static int cache[4][64] = {};
  PG_REQUIRE(dev >= 0 && dev < 64, PG_ERR_PARAMETER, "device ordinal out of range");
  int g = cache[slot][dev];
  if (g == 0) g = cache[slot][dev] = grid_for(dev, kernel, kChunkThreads, 0, int64_t(1) << 40);
  const int64_t need = ((n + kChunkRows - 1) / kChunkRows + 7) / 8;
  if (need < g) g = (int)(need < 1 ? 1 : need);
  return g;
}

// Kernel choice per phase and basis width (tools/cgs2_bench.py on B200,
// n = 1e6): the warp-chunk kernels win while the basis is narrow (fixed
// launch / reduction costs dominate and their full occupancy hides them);
// past that the shared-memory tile kernels (phases 1-2) and the row-streaming
// phase 3 reach a higher fraction of HBM.  With the 256-row tiles the
// cross-overs are k = 6 for phase 1 (k = 9: 17.7 vs 24.1 us), k = 9 for
// phase 2 (21.8 vs 23.4) and k = 12 for phase 3 (24.1 vs 25.0).  All of them
// project w1 with the same sequential FMA order, so phases 2 and 3 may use
// different kernel families and still agree bit for bit.  PG_CGS2_TILE=1 /
// PG_CGS2_CHUNK_KMAX (all phases) override.
static bool use_tile_cgs2(int k, int phase = 3) {
  static int force_tile = -1, chunk_kmax = -1;
  if (force_tile < 0) {
    force_tile = std::getenv("PG_CGS2_TILE") != nullptr;
    const char* s = std::getenv("PG_CGS2_CHUNK_KMAX");
    chunk_kmax = s ? std::atoi(s) : -1;
  }
  if (force_tile == 1) return true;
  if (chunk_kmax >= 0) return k > chunk_kmax;
  return k > (phase == 1 ? 5 : phase == 2 ? 8 : 11);
}

template <int MODE>
static void launch_chunk_dots(const double* V, int64_t ld, int k, const double* z, int64_t n,
                              const double* c1, double* out, pg_workspace* ws, cudaStream_t st) {
  check_ws(ws);
  if (n == 0) {
    PG_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * k, st));
    return;
  }
  const int g = chunk_grid((const void*)chunk_dots_kernel<MODE>, MODE, ws->device, n);
  launch_k(chunk_dots_kernel<MODE>, g, kChunkThreads, 0, st, V, ld, k, z, n, c1, ws->partials,
                                                       ws->counter, out);
  check_launch();
}

template <int MODE, int TR>
static void set_tile_attrs(int dev) {
  static bool done[64] = {};
  if (done[dev]) return;
  PG_CUDA(cudaFuncSetAttribute(tile_kernel<MODE, 4, TR>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTileSmemMax));
  PG_CUDA(cudaFuncSetAttribute(tile_kernel<MODE, 3, TR>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTileSmemMax));
  PG_CUDA(cudaFuncSetAttribute(tile_kernel<MODE, 2, TR>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTileSmemMax));
  done[dev] = true;
}

template <int MODE>
static void launch_tile(const double* V, int64_t ld, int k, const double* z, int64_t n,
                        const double* c1, double* out, pg_workspace* ws, cudaStream_t st) {
  check_ws(ws);
  PG_REQUIRE(ld % 2 == 0, PG_ERR_PARAMETER, "leading dimension must be even");
  PG_REQUIRE(((uintptr_t)V & 15) == 0 && (!z || ((uintptr_t)z & 15) == 0), PG_ERR_PARAMETER,
             "tile operands must be 16-byte aligned");
  const int tr = tile_rows_for(MODE, k, n);
  const int stages = tile_stages(MODE, k, n, tr);
  const size_t smem = tile_smem(MODE, k, stages, tr);
  const int dev = ws->device;
  PG_REQUIRE(dev >= 0 && dev < 64, PG_ERR_PARAMETER, "device ordinal out of range");
  if (tr == 256)
    set_tile_attrs<MODE, 256>(dev);
  else
    set_tile_attrs<MODE, 128>(dev);
  const void* kern =
      tr == 256 ? (stages == 4   ? (const void*)tile_kernel<MODE, 4, 256>
                   : stages == 3 ? (const void*)tile_kernel<MODE, 3, 256>
                                 : (const void*)tile_kernel<MODE, 2, 256>)
                : (stages == 4   ? (const void*)tile_kernel<MODE, 4, 128>
                   : stages == 3 ? (const void*)tile_kernel<MODE, 3, 128>
                                 : (const void*)tile_kernel<MODE, 2, 128>);
  const int64_t ntiles = (n + tr - 1) / tr;
  if (ntiles == 0) {
    PG_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * (MODE == kGram ? 2 * k * k : k), st));
    return;
  }
  // resident grid per (kernel, device), recomputed when the ring changes
  static int grid_cache[2][PG_KMAX + 1][64] = {};
  static int grid_key[2][PG_KMAX + 1][64] = {};
  const int ti = tr == 256 ? 1 : 0;
  int g = grid_cache[ti][k][dev];
  if (g == 0 || grid_key[ti][k][dev] != stages) {
    g = grid_for(dev, kern, kTileThreads, smem, int64_t(1) << 40);
    grid_cache[ti][k][dev] = g;
    grid_key[ti][k][dev] = stages;
  }
  if (ntiles < g) g = (int)ntiles;
#define PG_TILE_LAUNCH(S, R)                                                                 \
  launch_k(tile_kernel<MODE, S, R>, g, kTileThreads, smem, st, V, ld, k, z, n, c1,          \
           ws->partials, ws->counter, out)
  if (tr == 256) {
    if (stages == 4) PG_TILE_LAUNCH(4, 256);
    else if (stages == 3) PG_TILE_LAUNCH(3, 256);
    else PG_TILE_LAUNCH(2, 256);
  } else {
    if (stages == 4) PG_TILE_LAUNCH(4, 128);
    else if (stages == 3) PG_TILE_LAUNCH(3, 128);
    else PG_TILE_LAUNCH(2, 128);
  }
#undef PG_TILE_LAUNCH
  check_launch();
}

// ------------------------------------------------------- TMA tile launch --
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    const cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    if (e == cudaSuccess && q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
    else if (std::getenv("PG_TMA_DEBUG"))
      std::fprintf(stderr, "pgmres: cuTensorMapEncodeTiled entry point: err %d query %d\n", (int)e, (int)q);
  }
  return fn;
}

// V as a rows x columns tensor map with TR x 8 boxes, z as an n x 1 one
static bool cgs2_maps(EncodeTiledFn enc, const double* V, int64_t ld, int k, const double* z,
                      int64_t n, int tr, CUtensorMap* tmV, CUtensorMap* tmZ) {
  {
    const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)k};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
    const cuuint32_t box[2] = {(cuuint32_t)tr, (cuuint32_t)kTmaBoxCols};
    const cuuint32_t es[2] = {1, 1};
    if (enc(tmV, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)V, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      if (std::getenv("PG_TMA_DEBUG")) std::fprintf(stderr, "pgmres: V tensor map rejected\n");
      return false;
    }
  }
  {
    // z as an n x 1 matrix (a rank-1 map was rejected by the driver here)
    const cuuint64_t dims[2] = {(cuuint64_t)n, 1};
    const cuuint64_t strides[1] = {(cuuint64_t)((n + 1) & ~(int64_t)1) * sizeof(double)};
    const cuuint32_t box[2] = {(cuuint32_t)tr, 1};
    const cuuint32_t es[2] = {1, 1};
    if (enc(tmZ, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)z, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      if (std::getenv("PG_TMA_DEBUG")) std::fprintf(stderr, "pgmres: z tensor map rejected\n");
      return false;
    }
  }
  return true;
}

// Phases 1-2 through tma_tile_kernel (PG_CGS2_TMA=0: the cp.async tile
// kernel).  Same tile height and ring depth policy as launch_tile.
template <int MODE>
static bool launch_tma(const double* V, int64_t ld, int k, const double* z, int64_t n,
                       const double* c1, double* out, pg_workspace* ws, cudaStream_t st) {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("PG_CGS2_TMA");
    on = e ? std::atoi(e) : 1;
  }
  if (!on || n <= 0 || n > 0x7fffffffLL || k < 1) return false;
  if (ld % 2 != 0 || ((uintptr_t)V & 15) != 0 || ((uintptr_t)z & 15) != 0) return false;
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return false;
  // tile height and ring depth with TMA staging (tools/cgs2_bench.py sweep on
  // B200, profiles/r02/cgs2_tma_sweep.md): phase 1 takes 256-row tiles
  // everywhere (n = 8M, k = 45: 414 vs 442 us); phase 2 256-row tiles up to
  // k = 20 and, at n <= 2M, beyond k = 32, else 128-row tiles with a ring
  // sized for 3 CTAs per SM (n = 8M, k = 45: 427 vs 439 us)
  const bool small = n <= (int64_t)2000000;
  int tr = 256, ctas = 0;
  if (MODE == kUpdDots && !(k <= 20 || (small && k > 32))) {
    tr = 128;
    ctas = 3;
  }
  static int force_tr = -1;
  if (force_tr < 0) {
    const char* e = std::getenv("PG_TILE_ROWS");
    force_tr = e ? std::atoi(e) : 0;
  }
  if (force_tr == 128 || force_tr == 256) tr = force_tr;
  int stages;
  if (ctas > 0 && !std::getenv(MODE == kDots ? "PG_TILE_CTAS_P1" : "PG_TILE_CTAS_P2")) {
    stages = 2;
    for (int s = 4; s > 2; --s)
      if (tile_smem(MODE, k, s, tr) <= kTileSmemMax / ctas) {
        stages = s;
        break;
      }
  } else {
    stages = tile_stages(MODE, k, n, tr);
  }
  const int nbox = (k + kTmaBoxCols - 1) / kTmaBoxCols;
  const size_t smem = sizeof(double) * ((size_t)stages * (nbox * kTmaBoxCols + 1) * tr +
                                        (MODE == kUpdDots ? (size_t)tr : 0));
  if (smem > kTileSmemMax) return false;
  CUtensorMap tmV, tmZ;
  if (!cgs2_maps(enc, V, ld, k, z, n, tr, &tmV, &tmZ)) return false;
  const int dev = ws->device;
  const void* kern =
      tr == 256 ? (stages == 4   ? (const void*)tma_tile_kernel<MODE, 4, 256>
                   : stages == 3 ? (const void*)tma_tile_kernel<MODE, 3, 256>
                                 : (const void*)tma_tile_kernel<MODE, 2, 256>)
                : (stages == 4   ? (const void*)tma_tile_kernel<MODE, 4, 128>
                   : stages == 3 ? (const void*)tma_tile_kernel<MODE, 3, 128>
                                 : (const void*)tma_tile_kernel<MODE, 2, 128>);
  static bool attr[2][2][5][64] = {};
  if (!attr[MODE - 1][tr == 256][stages][dev]) {
    PG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kTileSmemMax));
    attr[MODE - 1][tr == 256][stages][dev] = true;
  }
  const int64_t ntiles = (n + tr - 1) / tr;
  const int g = grid_for(dev, kern, kTileThreads, smem, ntiles);
#define PG_TMA_LAUNCH(S, R)                                                                 \
  launch_k(tma_tile_kernel<MODE, S, R>, g, kTileThreads, smem, st, tmV, tmZ, k, n, c1,      \
           ws->partials, ws->counter, out)
  if (tr == 256) {
    if (stages == 4) PG_TMA_LAUNCH(4, 256);
    else if (stages == 3) PG_TMA_LAUNCH(3, 256);
    else PG_TMA_LAUNCH(2, 256);
  } else {
    if (stages == 4) PG_TMA_LAUNCH(4, 128);
    else if (stages == 3) PG_TMA_LAUNCH(3, 128);
    else PG_TMA_LAUNCH(2, 128);
  }
#undef PG_TMA_LAUNCH
  check_launch();
  return true;
}

// Phase 3 through tma_rows_kernel (PG_CGS2_TMA3=0: the row-streaming kernel):
// the deepest ring of 256-row tiles that fits, two CTAs per SM while two
// stages each do.
static bool launch_tma_rows(const double* V, int64_t ld, int k, const double* z, int64_t n,
                            const double* c1, const double* c2, double* out, double* nsq,
                            pg_workspace* ws, cudaStream_t st) {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("PG_CGS2_TMA3");
    on = e ? std::atoi(e) : 1;
  }
  if (!on || n <= 0 || n > 0x7fffffffLL || k < 1) return false;
  if (ld % 2 != 0 || ((uintptr_t)V & 15) != 0 || ((uintptr_t)z & 15) != 0) return false;
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return false;
  const int nbox = (k + kTmaBoxCols - 1) / kTmaBoxCols;
  const size_t tile = sizeof(double) * (size_t)(nbox * kTmaBoxCols + 1) * kRowsTileRows;
  static int ctas_env = -1;
  if (ctas_env < 0) {
    const char* e = std::getenv("PG_TILE_CTAS_P3");
    ctas_env = e ? std::atoi(e) : 0;
  }
  int ctas = ctas_env > 0 ? ctas_env : (4 * tile <= kTileSmemMax ? 2 : 1);
  int stages = (int)(kTileSmemMax / ctas / tile);
  if (stages > 4) stages = 4;
  if (stages < 2) {
    ctas = 1;
    stages = (int)(kTileSmemMax / tile);
    if (stages > 4) stages = 4;
  }
  if (stages < 2) return false;
  const size_t smem = (size_t)stages * tile;
  CUtensorMap tmV, tmZ;
  if (!cgs2_maps(enc, V, ld, k, z, n, kRowsTileRows, &tmV, &tmZ)) return false;
  const int dev = ws->device;
  const void* kern = stages == 4   ? (const void*)tma_rows_kernel<4>
                     : stages == 3 ? (const void*)tma_rows_kernel<3>
                                   : (const void*)tma_rows_kernel<2>;
  static bool attr[5][64] = {};
  if (!attr[stages][dev]) {
    PG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kTileSmemMax));
    attr[stages][dev] = true;
  }
  const int64_t ntiles = (n + kRowsTileRows - 1) / kRowsTileRows;
  const int g = grid_for(dev, kern, kTileThreads, smem, ntiles);
#define PG_TMA_ROWS(S)                                                                      \
  launch_k(tma_rows_kernel<S>, g, kTileThreads, smem, st, tmV, tmZ, k, n, c1, c2, out,       \
           ws->partials, ws->counter, nsq)
  if (stages == 4) PG_TMA_ROWS(4);
  else if (stages == 3) PG_TMA_ROWS(3);
  else PG_TMA_ROWS(2);
#undef PG_TMA_ROWS
  check_launch();
  return true;
}

// Grid of a grid-stride streaming kernel: whole waves of the blocks an SM
// keeps resident (occupancy of this kernel), at most kMaxBlocks (the
// reductions' partial slots) -- a partial second wave ran phase 3 of CGS2 at
// 1.38 waves (1024 blocks, 740 resident) -- or fewer when n is small.
static int simple_grid(int64_t n, int threads, const void* kernel) {
  static int sms = 0;
  if (!sms) PG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, current_device()));
  static const void* kern[16] = {};
  static int occ[16] = {};
  int per_sm = 0;
  for (int i = 0; i < 16; ++i) {
    if (kern[i] == kernel) {
      per_sm = occ[i];
      break;
    }
    if (!kern[i]) {
      PG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0));
      kern[i] = kernel;
      occ[i] = per_sm;
      break;
    }
  }
  if (per_sm < 1) per_sm = 1;
  const int cap_sm = kMaxBlocks / sms > 0 ? kMaxBlocks / sms : 1;
  int64_t g = (int64_t)sms * (per_sm < cap_sm ? per_sm : cap_sm);
  const int64_t need = (n + threads - 1) / threads;
  if (need < g) g = need;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace pg

using namespace pg;

namespace pg {
// out = base + sgn * (V[:, :k] c): sequential FMA over the columns per row,
// like the GEMV (rows_kernel<false>); sgn = +-1 (exact).
__global__ void __launch_bounds__(kRowThreads)
    gemv_acc_kernel(const double* __restrict__ V, int64_t ld, int k, const double* __restrict__ c,
                    int64_t n, const double* __restrict__ base, double sgn, double* out) {
  pdl_entry();
  __shared__ double cs[PG_KMAX];
  for (int i = threadIdx.x; i < k; i += blockDim.x) cs[i] = c[i];
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride) {
    const double* vr = V + r;
    double t = 0.0;
    int i = 0;
    for (; i + 8 <= k; i += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcs(vr + (int64_t)(i + u) * ld);
#pragma unroll
      for (int u = 0; u < 8; ++u) t = __fma_rn(v[u], cs[i + u], t);
    }
    for (; i < k; ++i) t = __fma_rn(__ldcs(vr + (int64_t)i * ld), cs[i], t);
    const double st = __dmul_rn(sgn, t);
    out[r] = base ? __dadd_rn(base[r], st) : st;
  }
}

// CGS2 against a basis wider than PG_KMAX, in column tiles: every phase reads
// V once per tile (the reference's four passes, ortho.py:53-59); w1 is stored.
void cgs2_wide(const double* V, int64_t ld, int k, const double* z, int64_t n, double* c1,
               double* c2, double* nsq, double* w1, double* w2, pg_workspace* ws, pg_dist* dist,
               cudaStream_t st) {
  void* sv = reinterpret_cast<void*>(st);
  auto tiles = [&](auto fn) {
    for (int t0 = 0; t0 < k; t0 += PG_KMAX) fn(t0, k - t0 < PG_KMAX ? k - t0 : PG_KMAX);
  };
  auto chk = [](int rc) {
    if (rc != PG_OK) {
      char msg[512];
      pg_last_error(msg, sizeof msg);
      throw Error(rc, msg);
    }
  };
  tiles([&](int t0, int kt) { chk(pg_cgs2_phase1(V + t0 * ld, ld, kt, z, n, c1 + t0, ws, sv)); });
  dist_allreduce(dist, c1, k, st);
  tiles([&](int t0, int kt) {
    chk(pg_gemv_acc(V + t0 * ld, ld, kt, c1 + t0, n, t0 == 0 ? z : w1, -1.0, w1, sv));
  });
  tiles([&](int t0, int kt) { chk(pg_cgs2_phase1(V + t0 * ld, ld, kt, w1, n, c2 + t0, ws, sv)); });
  dist_allreduce(dist, c2, k, st);
  tiles([&](int t0, int kt) {
    chk(pg_gemv_acc(V + t0 * ld, ld, kt, c2 + t0, n, t0 == 0 ? w1 : w2, -1.0, w2, sv));
  });
  chk(pg_dot(w2, w2, n, nsq, ws, sv));
  dist_allreduce(dist, nsq, 1, st);
}

void normalize_publish(const double* x, const double* nsq, int64_t n, double* out,
                       const double* ring, int count, double* host, cudaStream_t st) {
  const int g = n > 0 ? simple_grid(n, 256, (const void*)normalize_publish_kernel) : 1;
  launch_k(normalize_publish_kernel, g, 256, 0, st, x, nsq, n, out, ring, count, host);
  check_launch();
}
}  // namespace pg

extern "C" {

PG_API int pg_cgs2_phase1(const double* d_V, int64_t ld, int k, const double* d_z, int64_t n,
                          double* d_c1, pg_workspace* ws, void* stream) {
  return guard([&] {
    check_tall(d_V, ld, k, n, 1);
    PG_REQUIRE(d_z && d_c1, PG_ERR_PARAMETER, "null argument");
    if (!use_tile_cgs2(k, 1))
      launch_chunk_dots<1>(d_V, ld, k, d_z, n, nullptr, d_c1, ws, as_stream(stream));
    else if (!launch_tma<kDots>(d_V, ld, k, d_z, n, nullptr, d_c1, ws, as_stream(stream)))
      launch_tile<kDots>(d_V, ld, k, d_z, n, nullptr, d_c1, ws, as_stream(stream));
  });
}

PG_API int pg_cgs2_phase2(const double* d_V, int64_t ld, int k, const double* d_z, int64_t n,
                          const double* d_c1, double* d_c2, pg_workspace* ws, void* stream) {
  return guard([&] {
    check_tall(d_V, ld, k, n, 1);
    PG_REQUIRE(d_z && d_c1 && d_c2, PG_ERR_PARAMETER, "null argument");
    if (!use_tile_cgs2(k, 2))
      launch_chunk_dots<2>(d_V, ld, k, d_z, n, d_c1, d_c2, ws, as_stream(stream));
    else if (!launch_tma<kUpdDots>(d_V, ld, k, d_z, n, d_c1, d_c2, ws, as_stream(stream)))
      launch_tile<kUpdDots>(d_V, ld, k, d_z, n, d_c1, d_c2, ws, as_stream(stream));
  });
}

PG_API int pg_cgs2_phase3(const double* d_V, int64_t ld, int k, const double* d_z, int64_t n,
                          const double* d_c1, const double* d_c2, double* d_w2, double* d_nsq,
                          pg_workspace* ws, void* stream) {
  return guard([&] {
    check_tall(d_V, ld, k, n, 0);
    check_ws(ws);
    PG_REQUIRE(d_z && d_w2 && d_nsq && (k == 0 || (d_c1 && d_c2)), PG_ERR_PARAMETER,
               "null argument");
    cudaStream_t st = as_stream(stream);
    if (n == 0) {
      PG_CUDA(cudaMemsetAsync(d_nsq, 0, sizeof(double), st));
      return;
    }
    if (use_tile_cgs2(k) &&
        launch_tma_rows(d_V, ld, k, d_z, n, d_c1, d_c2, d_w2, d_nsq, ws, st)) {
      // (staged by tensor maps)
    } else if (use_tile_cgs2(k)) {
      const int g = simple_grid(n, kRowThreads, (const void*)rows_kernel<true>);
      launch_k(rows_kernel<true>, g, kRowThreads, 0, st, d_V, ld, k, d_z, n, d_c1, d_c2, d_w2,
                                                    ws->partials, ws->counter, d_nsq);
    } else {
      const int g = chunk_grid((const void*)chunk_update_kernel, 3, ws->device, n);
      launch_k(chunk_update_kernel, g, kChunkThreads, 0, st, d_V, ld, k, d_z, n, d_c1, d_c2, d_w2,
                                                       ws->partials, ws->counter, d_nsq);
    }
    check_launch();
  });
}

PG_API int pg_normalize(const double* d_x, const double* d_nsq, int64_t n, double* d_out,
                        void* stream) {
  return guard([&] {
    PG_REQUIRE(d_x && d_nsq && d_out, PG_ERR_PARAMETER, "null argument");
    if (n == 0) return;
    const int g = simple_grid(n, 256, (const void*)normalize_kernel);
    launch_k(normalize_kernel, g, 256, 0, as_stream(stream), d_x, d_nsq, n, d_out);
    check_launch();
  });
}

PG_API int pg_gram(const double* d_P, int64_t ld, int ncols, int64_t n, double* d_G,
                   pg_workspace* ws, void* stream) {
  return guard([&] {
    check_tall(d_P, ld, ncols, n, 1);
    PG_REQUIRE(d_G, PG_ERR_PARAMETER, "null argument");
    launch_tile<kGram>(d_P, ld, ncols, nullptr, n, nullptr, d_G, ws, as_stream(stream));
  });
}

PG_API int pg_gemv(const double* d_V, int64_t ld, int k, const double* d_y, int64_t n,
                   double* d_out, void* stream) {
  return guard([&] {
    check_tall(d_V, ld, k, n, 0);
    PG_REQUIRE(d_out && (k == 0 || d_y), PG_ERR_PARAMETER, "null argument");
    if (n == 0) return;
    const int g = simple_grid(n, kRowThreads, (const void*)rows_kernel<false>);
    launch_k(rows_kernel<false>, g, kRowThreads, 0, as_stream(stream), d_V, ld, k, nullptr, n, d_y, nullptr, d_out, nullptr, nullptr, nullptr);
    check_launch();
  });
}

PG_API int pg_gemv_acc(const double* d_V, int64_t ld, int k, const double* d_y, int64_t n,
                       const double* d_base, double sgn, double* d_out, void* stream) {
  return guard([&] {
    check_tall(d_V, ld, k, n, 0);
    PG_REQUIRE(d_out && (k == 0 || d_y), PG_ERR_PARAMETER, "null argument");
    if (n == 0) return;
    const int g = simple_grid(n, kRowThreads, (const void*)gemv_acc_kernel);
    launch_k(gemv_acc_kernel, g, kRowThreads, 0, as_stream(stream), d_V, ld, k, d_y, n, d_base,
             sgn, d_out);
    check_launch();
  });
}

PG_API int pg_cgs2_wide(const double* d_V, int64_t ld, int k, const double* d_z, int64_t n,
                        double* d_c1, double* d_c2, double* d_nsq, double* d_w1, double* d_w2,
                        pg_workspace* ws, void* stream) {
  return guard([&] {
    PG_REQUIRE(k >= 1 && k <= PG_MMAX, PG_ERR_DIMENSION, "basis width out of range");
    PG_REQUIRE(d_V && d_z && d_c1 && d_c2 && d_nsq && d_w1 && d_w2, PG_ERR_PARAMETER,
               "null argument");
    cgs2_wide(d_V, ld, k, d_z, n, d_c1, d_c2, d_nsq, d_w1, d_w2, ws, nullptr,
              as_stream(stream));
  });
}

PG_API int pg_dot(const double* d_x, const double* d_y, int64_t n, double* d_out,
                  pg_workspace* ws, void* stream) {
  return guard([&] {
    check_ws(ws);
    PG_REQUIRE(d_x && d_y && d_out, PG_ERR_PARAMETER, "null argument");
    cudaStream_t st = as_stream(stream);
    if (n == 0) {
      PG_CUDA(cudaMemsetAsync(d_out, 0, sizeof(double), st));
      return;
    }
    const int g = simple_grid(n, 256, (const void*)dot_kernel);
    launch_k(dot_kernel, g, 256, 0, st, d_x, d_y, n, ws->partials, ws->counter, d_out);
    check_launch();
  });
}

PG_API int pg_scale_add(const double* d_base, double a, const double* d_v, int64_t n,
                        double* d_out, void* stream) {
  return guard([&] {
    PG_REQUIRE(d_v && d_out, PG_ERR_PARAMETER, "null argument");
    if (n == 0) return;
    const int g = simple_grid(n, 256, (const void*)scale_add_kernel);
    launch_k(scale_add_kernel, g, 256, 0, as_stream(stream), d_base, a, d_v, n, d_out);
    check_launch();
  });
}

PG_API int pg_gather(const double* d_x, const int32_t* d_idx, int64_t m, double* d_out,
                     void* stream) {
  return guard([&] {
    if (m == 0) return;
    PG_REQUIRE(d_x && d_idx && d_out, PG_ERR_PARAMETER, "null argument");
    const int g = simple_grid(m, 256, (const void*)gather_kernel);
    launch_k(gather_kernel, g, 256, 0, as_stream(stream), d_x, d_idx, m, d_out);
    check_launch();
  });
}

}  // extern "C"
