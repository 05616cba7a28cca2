// Row arithmetic shared by the SELL SpMV kernels (spmv.cu) and the
// dependency-driven chain kernel (chain.cu): modes, argument blocks, the
// fused polynomial epilogue and the short-row pair body.  Every kernel that
// includes this sums a row in stored column order with separately rounded
// products (__dmul_rn / __dadd_rn), bit-for-bit the reference spmv
// (sparse.py:164-168) and apply_poly's recurrence (polyprec.py:205-211).
#pragma once

#include "internal.cuh"

namespace pg {

enum SellMode { kSpmv = 0, kPoly = 1, kResid = 2, kRoot = 3 };

constexpr int kSellThreads = 256;
// Occupancy floor and row-chunk unroll of the plain kernel, chosen by sweep
// on B200 (tools/spmv_bench.py over build variants): (4 blocks, unroll 4)
// gives cfg2 5.40, cfg4 6.19, cfg5 5.26, cfg3 2.41 TB/s; forcing 6+ blocks
// (<= 40 registers) spills and loses 30-40%.
#ifndef PG_SELL_MIN_BLOCKS
#define PG_SELL_MIN_BLOCKS 4
#endif
constexpr int kSellMinBlocks = PG_SELL_MIN_BLOCKS;
#ifndef PG_SELL_UNROLL
#define PG_SELL_UNROLL 4
#endif
constexpr int kUnroll = PG_SELL_UNROLL;

struct SellArgs {
  const int64_t* __restrict__ slice_ptr;
  const int32_t* __restrict__ slice_w;
  const int32_t* __restrict__ row_len;
  const int32_t* __restrict__ perm;
  const int32_t* __restrict__ col;
  const double* __restrict__ val;
  int64_t nrows;
  int64_t nlanes;
  const int64_t* __restrict__ slice_ptr8;  // packed 1-byte stream offsets
  const uint8_t* __restrict__ col8;  // dictionary-compressed streams (abi.cu)
  const int32_t* __restrict__ dtab;
  const uint8_t* __restrict__ val8;
  const double* __restrict__ vtab;
  int64_t stride8;  // pg_matrix::stride8
};

struct Epi {
  const double* acc_in;
  const double* base;
  double* acc_out;
  double* w_out;
  const double* b;
  double y0, yk;
  int flags;
  // kRoot (root-product form, PG_ROOT_*): acc_in = y_in, acc_out = y_out,
  // w_out = v_out, base = p_in; c1 = 1/|theta|^2 or 1/theta, c2 = 2 Re(theta),
  // c3 = folded trailing real root (0 = none)
  double c1, c2, c3;
};

__device__ __forceinline__ int64_t lane_row(const SellArgs& a, int64_t lane) {
  if (a.perm) return __ldg(a.perm + lane);
  return lane < a.nrows ? lane : -1;
}

// Epilogue operands of a row, loaded BEFORE the row's gathers so that their
// HBM latency overlaps the gather latency.
struct Pre {
  double a, b;
};

template <int MODE>
__device__ __forceinline__ Pre epi_load(const Epi& e, const double* __restrict__ x, int64_t row) {
  Pre p{0.0, 0.0};
  if (row < 0) return p;
  if (MODE == kPoly) {
    p.a = (e.flags & PG_PASS_FIRST) ? x[row] : e.acc_in[row];
    if (e.base) p.b = e.base[row];
  } else if (MODE == kResid) {
    p.a = e.b[row];
  } else if (MODE == kRoot) {
    p.a = ((e.flags & 3) == PG_ROOT_PAIR_B) ? e.base[row] : x[row];
    if (e.acc_in) p.b = e.acc_in[row];
  }
  return p;
}

// The epilogue operands a row reads (epi_load), as whole vectors so that the
// producer can stage the block's slice of them: A -> Pre::a, B -> Pre::b.
template <int MODE>
__device__ __forceinline__ void epi_vectors(const Epi& e, const double* x, const double*& A,
                                            const double*& B) {
  A = B = nullptr;
  if (MODE == kPoly) {
    A = (e.flags & PG_PASS_FIRST) ? x : e.acc_in;
    B = e.base;
  } else if (MODE == kResid) {
    A = e.b;
  } else if (MODE == kRoot) {
    A = ((e.flags & 3) == PG_ROOT_PAIR_B) ? e.base : x;
    B = e.acc_in;
  }
}

// Row epilogue; returns the residual entry (kResid) for the norm.
template <int MODE>
__device__ __forceinline__ double epilogue(const Epi& e, const Pre& p, int64_t row, double ax) {
  if (MODE == kSpmv) {
    e.acc_out[row] = ax;
    return 0.0;
  } else if (MODE == kPoly) {
    double t = (e.flags & PG_PASS_FIRST) ? __dmul_rn(e.y0, p.a) : p.a;
    t = __dadd_rn(t, __dmul_rn(e.yk, ax));
    if (e.flags & PG_PASS_WRITE_W) e.w_out[row] = ax;
    if (e.base) t = __dadd_rn(p.b, t);
    e.acc_out[row] = t;
    return 0.0;
  } else if (MODE == kResid) {
    const double r = __dsub_rn(p.a, ax);
    e.acc_out[row] = r;
    return r;
  } else {
    // root-product step (Loe-Morgan running sum): p.a = operand / prod row,
    // p.b = running sum y (or v for the PG_ROOT_RESID final pass)
    const int mode = e.flags & 3;
    const bool resid = (e.flags & PG_ROOT_RESID) != 0;
    if (mode == PG_ROOT_PAIR_A) {
      const double t2 = __fma_rn(e.c2, p.a, -ax);   // 2 Re(theta) prod - A prod
      if (e.w_out) e.w_out[row] = t2;
      if (e.acc_out) e.acc_out[row] = __fma_rn(e.c1, t2, p.b);  // y + t2 / |theta|^2
    } else {
      // REAL: prod - A prod / theta;  PAIR_B: prod - A t2 / |theta|^2
      const double pn = __fma_rn(-e.c1, ax, p.a);
      if (resid) {
        e.w_out[row] = __dsub_rn(p.b, pn);          // A p(A) v = v - pi(A) v
      } else {
        if (e.w_out) e.w_out[row] = pn;
        if (e.acc_out) {
          double y = (mode == PG_ROOT_REAL) ? __fma_rn(e.c1, p.a, p.b) : p.b;
          if (e.c3 != 0.0) y = __fma_rn(e.c3, pn, y);  // folded trailing real root
          e.acc_out[row] = y;
        }
      }
    }
    return 0.0;
  }
}

// Rows of at most 8 stored entries (7-point stencils): both index words, all
// table entries and all gathers are issued before the first add, so the row
// costs one gather round trip instead of one per 4-entry chunk.
// CG = true gathers through L2 only (ld.global.cg): x was written by another
// SM inside the same kernel (chain.cu), so neither L1 nor the read-only path
// may serve it.
template <bool CG = false>
__device__ __forceinline__ double row_sum_pair_words(uint32_t w0, uint32_t w1, int len,
                                                     int64_t row, const double* __restrict__ x,
                                                     const PairEnt* s_ptab) {
  const double* xr = x + row;
  double v[8], xv[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const uint32_t idx = ((u < 4 ? w0 : w1) >> (8 * (u & 3))) & 255u;
    const int4 raw = reinterpret_cast<const int4*>(s_ptab)[idx];
    v[u] = __hiloint2double(raw.y, raw.x);
    xv[u] = (u < len) ? (CG ? __ldcg(xr + raw.w) : __ldg(xr + raw.w)) : 0.0;
  }
  double acc = 0.0;
#pragma unroll
  for (int u = 0; u < 8; ++u)
    if (u < len) acc = __dadd_rn(acc, __dmul_rn(v[u], xv[u]));
  return acc;
}

__device__ __forceinline__ double row_sum_pairs_short(const uint32_t* __restrict__ pw, int len,
                                                      int64_t row,
                                                      const double* __restrict__ x,
                                                      const PairEnt* s_ptab) {
  const uint32_t w0 = __ldcs(pw);
  const uint32_t w1 = len > 4 ? __ldcs(pw + PG_SLICE) : 0u;
  return row_sum_pair_words<false>(w0, w1, len, row, x, s_ptab);
}

// Row-pattern dictionary (pg_matrix::rpat): the row's entries are the
// table entries [beg, end) in stored order; all gathers of an 8-entry batch
// are issued before its adds.  Same sequential mul-then-add order as every
// other kernel.  CG as in row_sum_pair_words.
template <bool CG = false>
__device__ __forceinline__ double row_sum_pattern(int beg, int end, int64_t row,
                                                  const double* __restrict__ x,
                                                  const PairEnt* s_ent) {
  const double* xr = x + row;
  double acc = 0.0;
  for (int e0 = beg; e0 < end; e0 += 8) {
    double v[8], xv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      v[u] = xv[u] = 0.0;
      if (e0 + u < end) {
        const int4 raw = reinterpret_cast<const int4*>(s_ent)[e0 + u];
        v[u] = __hiloint2double(raw.y, raw.x);
        xv[u] = CG ? __ldcg(xr + raw.w) : __ldg(xr + raw.w);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (e0 + u < end) acc = __dadd_rn(acc, __dmul_rn(v[u], xv[u]));
  }
  return acc;
}

// RB rows per thread at once, patterns of <= 8 entries: every gather and
// epilogue operand of the RB rows is requested before the first add or
// store (stores may alias the operands, so the compiler cannot overlap rows
// itself); values are re-read from the shared table at the adds to keep the
// registers for loads in flight.  Same per-row order and rounding.
// LD(p) performs one vector load (ldg / ldcg).  rows[j] < 0: no row.
template <int RB, class LD>
__device__ __forceinline__ void rows_pattern_batch(const int64_t (&row)[RB], const int (&beg)[RB],
                                                   const int (&end)[RB],
                                                   const double* __restrict__ x,
                                                   const PairEnt* s_ent, double (&ax)[RB],
                                                   LD ld) {
  double xv[RB][8];
#pragma unroll
  for (int j = 0; j < RB; ++j) {
    const double* xr = x + (row[j] < 0 ? 0 : row[j]);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      xv[j][u] = 0.0;
      if (beg[j] + u < end[j]) xv[j][u] = ld(xr + reinterpret_cast<const int4*>(s_ent)[beg[j] + u].w);
    }
  }
#pragma unroll
  for (int j = 0; j < RB; ++j) {
    double acc = 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (beg[j] + u < end[j]) acc = __dadd_rn(acc, __dmul_rn(s_ent[beg[j] + u].v, xv[j][u]));
    ax[j] = acc;
  }
}

// Stage the pattern table in shared memory: entries (16 B each), then the
// n_pat + 1 offsets, then the n_pat master masks.  Returns the offsets' base.
__device__ __forceinline__ const int32_t* stage_patterns(unsigned char* smem,
                                                         const int32_t* __restrict__ pptr,
                                                         const PairEnt* __restrict__ pent,
                                                         int npat, int nent,
                                                         const uint32_t* __restrict__ pmask =
                                                             nullptr) {
  PairEnt* s_ent = reinterpret_cast<PairEnt*>(smem);
  int32_t* s_ptr = reinterpret_cast<int32_t*>(smem + 16 * (size_t)(nent > 0 ? nent : 1));
  for (int i = threadIdx.x; i < nent; i += blockDim.x) s_ent[i] = pent[i];
  for (int i = threadIdx.x; i <= npat; i += blockDim.x) s_ptr[i] = pptr[i];
  if (pmask)
    for (int i = threadIdx.x; i < npat; i += blockDim.x)
      reinterpret_cast<uint32_t*>(s_ptr + npat + 1)[i] = pmask[i];
  return s_ptr;
}

__host__ __device__ inline size_t pattern_smem_bytes(int npat, int nent) {
  return 16 * (size_t)(nent > 0 ? nent : 1) + 4 * (size_t)(npat + 1) + 4 * (size_t)npat;
}

// The master pattern as kernel parameters (pg_matrix::pat_m*): offsets and
// values become constant-bank operands of fully unrolled code.  lb = the
// unrolled length: len itself for the common stencil rows (7, 27), else the
// bucket 8 / 16 / 32 >= len whose entries len..lb-1 are inert.
struct PatMaster {
  int len, lb;
  double v[32];
  int32_t doff[32];
  int32_t woff[32];
};

// A row that is the master's entries `mask` (in order): the products of all
// lb entries are formed, only the masked ones are added -- the same
// additions, in the same order, as the row's own entry list.  WIN: x is the
// block's shared-memory window (winrow = the row's slot); else global x
// gathered at row + doff (masked-off entries are not loaded: they may lie
// outside x).
// FULL: the caller established (warp-uniformly) that every row of the warp
// is the whole master pattern and that LB == pm.len -- no per-entry mask
// tests, every one of the LB entries added.
template <int LB, bool WIN, bool CG = false, bool FULL = false>
__device__ __forceinline__ double row_sum_master(uint32_t mask, const PatMaster& pm,
                                                 const unsigned char* winrow,
                                                 const double* __restrict__ xr) {
  if (FULL) mask = 0xffffffffu;
  double acc = 0.0;
#pragma unroll
  for (int c0 = 0; c0 < LB; c0 += 8) {
    double xv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (c0 + q >= LB) break;
      if (WIN) {
        xv[q] = *reinterpret_cast<const double*>(winrow + pm.woff[c0 + q]);
      } else {
        xv[q] = 0.0;
        if (FULL || (mask & (1u << (c0 + q))))
          xv[q] = CG ? __ldcg(xr + pm.doff[c0 + q]) : __ldg(xr + pm.doff[c0 + q]);
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (c0 + q >= LB) break;
      const double p = __dmul_rn(pm.v[c0 + q], xv[q]);
      if (FULL || (mask & (1u << (c0 + q)))) acc = __dadd_rn(acc, p);
    }
  }
  return acc;
}

// A row that is the master OFFSET pattern's entries `mask` (offset-pattern
// format: values still streamed).  vals points at the row's stored entry 0 in
// the SELL value stream (entry j at vals[32 j]); the j-th stored value pairs
// with the j-th set bit of mask -- the row's own order, so the sum is the
// sequential one.  FULL: the warp's rows are all the whole master and
// LB == pm.len (stored entry q at a compile-time offset).
template <int LB, bool FULL>
__device__ __forceinline__ double row_sum_omaster(uint32_t mask, const PatMaster& pm,
                                                  const double* __restrict__ vals,
                                                  const double* __restrict__ xr) {
  double acc = 0.0;
  int j = 0;
#pragma unroll
  for (int c0 = 0; c0 < LB; c0 += 8) {
    double v[8], xv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (c0 + q >= LB) break;
      v[q] = xv[q] = 0.0;
      if (FULL) {
        v[q] = __ldcs(vals + PG_SLICE * (c0 + q));
        xv[q] = __ldg(xr + pm.doff[c0 + q]);
      } else if (mask & (1u << (c0 + q))) {
        v[q] = __ldcs(vals + PG_SLICE * j);
        ++j;
        xv[q] = __ldg(xr + pm.doff[c0 + q]);
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (c0 + q >= LB) break;
      if (FULL || (mask & (1u << (c0 + q)))) acc = __dadd_rn(acc, __dmul_rn(v[q], xv[q]));
    }
  }
  return acc;
}

// Plane stencils (march.cu, planes.cu): a row-pattern master whose offsets
// are three plane groups dz = -1, 0, +1 of a plane stride S.
// per-kind shape: NO entries in each outer plane group, NM in the middle one;
// FULL = all three groups use the same in-plane offsets (tensor stencils)
template <int KIND>
struct MarchShape;
template <>
struct MarchShape<27> {
  static constexpr int NO = 9, NM = 9, CTR = 4;
  static constexpr bool FULL = true;
};
template <>
struct MarchShape<9> {
  static constexpr int NO = 3, NM = 3, CTR = 1;
  static constexpr bool FULL = true;
};
template <>
struct MarchShape<7> {
  static constexpr int NO = 1, NM = 5, CTR = 2;
  static constexpr bool FULL = false;
};
template <>
struct MarchShape<5> {
  static constexpr int NO = 1, NM = 3, CTR = 1;
  static constexpr bool FULL = false;
};

// i-th in-plane offset of the middle group (of every group when FULL)
template <int KIND>
__device__ __forceinline__ int64_t mid_off(int i, int64_t g) {
  if (KIND == 27) return (int64_t)(i / 3 - 1) * g + (i % 3 - 1);
  if (KIND == 7) return i == 0 ? -g : (i == 4 ? g : (int64_t)(i - 2));
  return (int64_t)(i - 1);  // 9, 5
}

// Plane-marching SpMV (march.cu): issues the pass and returns true when the
// matrix is a row-pattern stencil it handles (march_shape), else false.
template <int MODE>
bool march_launch(const pg_matrix* m, const double* x, Epi e, pg_workspace* ws, double* nsq,
                  cudaStream_t st);
// Plane-ring SpMV (planes.cu): same contract as march_launch.
template <int MODE>
bool plane_launch(const pg_matrix* m, const double* x, Epi e, pg_workspace* ws, double* nsq,
                  cudaStream_t st);

}  // namespace pg
