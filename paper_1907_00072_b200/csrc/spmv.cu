// libpgmres: SELL-C-sigma fp64 SpMV and the fused polynomial pass.
//
// One thread owns one row (one lane of a 32-row slice).  Slice entries are
// stored lane-interleaved (entry j of lane t at slice_ptr[s] + j*32 + t).
// The row sum is accumulated sequentially in stored column order with
// separately rounded products (__dmul_rn / __dadd_rn: never contracted to
// FMA), which is bit-for-bit the reference SpMV (sparse.py:164-168,
// np.bincount over values*x[col]).
//
// The polynomial recurrence of apply_poly (polyprec.py:205-211) runs in the
// epilogue of the same pass: acc <- acc + y_k * (A w)[row], so a degree-d
// application streams A exactly d times with no separate axpy kernels.
//
// Kernels sharing that row arithmetic:
//  * sell_kernel<MODE, 0, 0> (default for general matrices): one row per
//    thread; all index / value loads of a 4-entry chunk are issued before its
//    gathers, and the epilogue operands before the row's gathers.
//  * sell_kernel<MODE, 1, 1> (default when both streams fit a 256-entry
//    dictionary -- constant-coefficient stencils): 1-byte column-offset and
//    value indices packed 4 per 32-bit lane word (abi.cu), decoded through
//    shared-memory tables; ~2 B of matrix stream per entry instead of 12.
//  * sell_pair_kernel / sell_pair_short_kernel: one 1-byte (offset, value)
//    pair index per entry; rows of <= 8 entries issue all gathers at once.
//  * sell_win_kernel: natural-order stencil rows, x windows + pair stream
//    staged by a warp-specialised TMA ring (see its comment).
//  * sell_kernel<kRoot>: the root-product form of the polynomial (pg_root_pass).

#include <cstdlib>
#include <cstring>

#include "internal.cuh"
#include "pipeline.cuh"
#include "sell.cuh"

namespace pg {


// Sequential row sum over the row's entries.  cp(j) loads the raw column
// entry j (an int32 column, or a 1-byte dictionary index), dec(raw) turns it
// into a column, vp(j) loads value j.  Software-pipelined one chunk ahead:
// chunk j+1's index / value loads (bounded by the uniform slice width) are
// issued before chunk j's gathers (bounded by this row's length), so a chunk
// costs one gather round trip instead of an index round trip followed by a
// gather round trip.  PG_SELL_PIPE=0 restores the unpipelined loop.
#ifndef PG_SELL_PIPE
#define PG_SELL_PIPE 1
#endif
template <class ColPtr, class Dec, class ValPtr>
__device__ __forceinline__ double row_sum(ColPtr cp, Dec dec, ValPtr vp, int w, int len,
                                          const double* __restrict__ x) {
  double acc = 0.0;
#if PG_SELL_PIPE
  {
    int c[kUnroll];
    double v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      c[u] = 0;
      v[u] = 0.0;
      if (u < w) {
        c[u] = cp(u);
        v[u] = vp(u);
      }
    }
    for (int j = 0; j < w; j += kUnroll) {
      int cn[kUnroll];
      double vn[kUnroll], xv[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        cn[u] = 0;
        vn[u] = 0.0;
        if (j + kUnroll + u < w) {
          cn[u] = cp(j + kUnroll + u);
          vn[u] = vp(j + kUnroll + u);
        }
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) xv[u] = (j + u < len) ? __ldg(x + dec(c[u])) : 0.0;
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
        if (j + u < len) acc = __dadd_rn(acc, __dmul_rn(v[u], xv[u]));
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        c[u] = cn[u];
        v[u] = vn[u];
      }
    }
  }
#else
  for (int j = 0; j < w; j += kUnroll) {
    double v[kUnroll], xv[kUnroll];
    int c[kUnroll];
    // all raw index / value loads of the chunk first (bounded by the uniform
    // slice width), then the dictionary decode, then all gathers (bounded by
    // this row's length): no global load waits behind a dependent one
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (j + u < w) {
        c[u] = cp(j + u);
        v[u] = vp(j + u);
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) c[u] = dec(c[u]);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) xv[u] = (j + u < len) ? __ldg(x + c[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (j + u < len) acc = __dadd_rn(acc, __dmul_rn(v[u], xv[u]));
  }
#endif
  return acc;
}

// Row sum over dictionary-compressed streams: one 32-bit load per lane per 4
// entries of each packed 1-byte stream (CM: column offsets, VM: values);
// uncompressed streams keep their regular SELL positions.  Same sequential
// order and separately rounded products as row_sum.
// WIN = 1: x is the block's shared-memory window, `row` the row's index in
// the block and s_dtab the window-position table (pg_matrix::wtab).
template <int CM, int VM, int WIN = 0>
__device__ __forceinline__ double row_sum_dict(const SellArgs& a, int64_t base, int64_t base8,
                                               int row, int w, int len,
                                               const double* __restrict__ x,
                                               const int32_t* s_dtab, const double* s_vtab) {
  const uint32_t* __restrict__ cw = reinterpret_cast<const uint32_t*>(a.col8 + base8);
  const uint32_t* __restrict__ vw = reinterpret_cast<const uint32_t*>(a.val8 + base8);
  double acc = 0.0;
  // index words are software-pipelined two 4-entry chunks ahead: the stall
  // profile of the non-pipelined loop was dominated by waits on these loads
  uint32_t cn0 = 0, vn0 = 0, cn1 = 0, vn1 = 0;
  if (CM) {
    if (0 < w) cn0 = __ldcs(cw);
    if (4 < w) cn1 = __ldcs(cw + PG_SLICE);
  }
  if (VM) {
    if (0 < w) vn0 = __ldcs(vw);
    if (4 < w) vn1 = __ldcs(vw + PG_SLICE);
  }
  for (int j = 0; j < w; j += 4) {
    const int q = j >> 2;
    const uint32_t cbits = cn0, vbits = vn0;
    cn0 = cn1;
    vn0 = vn1;
    if (j + 8 < w) {
      if (CM) cn1 = __ldcs(cw + (q + 2) * PG_SLICE);
      if (VM) vn1 = __ldcs(vw + (q + 2) * PG_SLICE);
    }
    int c[4];
    double v[4], xv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (!CM) c[u] = (j + u < w) ? __ldcs(a.col + base + (int64_t)(j + u) * PG_SLICE) : 0;
      if (!VM) v[u] = (j + u < w) ? __ldcs(a.val + base + (int64_t)(j + u) * PG_SLICE) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (CM) c[u] = row + s_dtab[(cbits >> (8 * u)) & 255u];
      if (VM) v[u] = s_vtab[(vbits >> (8 * u)) & 255u];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      xv[u] = (j + u < len) ? (WIN ? x[c[u]] : __ldg(x + c[u])) : 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (j + u < len) acc = __dadd_rn(acc, __dmul_rn(v[u], xv[u]));
  }
  return acc;
}

template <int MODE>
__device__ __forceinline__ void finish_resid(double local, double* partials, unsigned* counter,
                                             double* nsq) {
  if (MODE == kResid) {
    const double s = block_sum(local);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
    last_block_reduce(partials, counter, 1, nsq);
  }
}

// ------------------------------------------------------------ plain kernel --
// CM / VM: 1 = the column / value stream is dictionary-compressed (1-byte
// indices into the per-matrix tables, staged in shared memory per block).
#ifndef PG_SELL_DICT_MIN_BLOCKS
#define PG_SELL_DICT_MIN_BLOCKS 4
#endif
template <int MODE, int CM, int VM>
__global__ void __launch_bounds__(kSellThreads,
                                  (CM || VM) ? PG_SELL_DICT_MIN_BLOCKS : kSellMinBlocks)
    sell_kernel(SellArgs a, const double* __restrict__ x, Epi e, double* partials,
                unsigned int* counter, double* nsq) {
  pdl_entry();
  __shared__ int32_t s_dtab[CM ? 256 : 1];
  __shared__ double s_vtab[VM ? 256 : 1];
  if (CM)
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_dtab[i] = __ldg(a.dtab + i);
  if (VM)
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_vtab[i] = __ldg(a.vtab + i);
  if (CM || VM) __syncthreads();
  double local = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t lane = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; lane < a.nlanes;
       lane += stride) {
    const int64_t row = lane_row(a, lane);
    if (row < 0) continue;
    const int64_t s = lane >> 5;
    const int w = __ldg(a.slice_w + s);
    const int len = __ldg(a.row_len + lane);
    const int64_t base = __ldg(a.slice_ptr + s) + (lane & 31);
    const Pre pre = epi_load<MODE>(e, x, row);
    double ax;
    if (CM || VM) {
      const int64_t base8 = __ldg(a.slice_ptr8 + s) + 4 * (lane & 31);
      ax = row_sum_dict<CM, VM>(a, base, base8, (int)row, w, len, x, s_dtab, s_vtab);
    } else {
      ax = row_sum(
          [&](int j) { return __ldcs(a.col + base + (int64_t)j * PG_SLICE); },
          [](int raw) { return raw; },
          [&](int j) { return __ldcs(a.val + base + (int64_t)j * PG_SLICE); }, w,
          len, x);
    }
    const double r = epilogue<MODE>(e, pre, row, ax);
    if (MODE == kResid) local = __fma_rn(r, r, local);
  }
  finish_resid<MODE>(local, partials, counter, nsq);
}

// ------------------------------------------------------ pair dictionary --
// One byte per entry (pair8) indexing {value, column offset} in a shared
// table; x gathered from global memory (L1/L2).  Index words are
// software-pipelined two 4-entry chunks ahead; full chunks run without
// predicates, only the row's last partial chunk is predicated.
// avail: index words present in this lane's slice (>= the row's own count);
// the first two are requested before the row length arrives.
__device__ __forceinline__ double row_sum_pairs_global(const uint32_t* __restrict__ pw, int len,
                                                       int avail, int64_t row,
                                                       const double* __restrict__ x,
                                                       const PairEnt* s_ptab) {
  double acc = 0.0;
  uint32_t n0 = 0, n1 = 0;
  if (avail > 0) n0 = __ldcs(pw);
  if (avail > 1) n1 = __ldcs(pw + PG_SLICE);
  const int nq = (len + 3) >> 2;
  const double* xr = x + row;
  for (int q = 0; q < nq; ++q) {
    const uint32_t pb = n0;
    n0 = n1;
    if (q + 2 < nq) n1 = __ldcs(pw + (q + 2) * PG_SLICE);
    const int left = len - 4 * q;
    PairEnt pe[4];
    double xv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) pe[u] = s_ptab[(pb >> (8 * u)) & 255u];
#pragma unroll
    for (int u = 0; u < 4; ++u) xv[u] = (u < left) ? __ldg(xr + pe[u].doff) : 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (u < left) acc = __dadd_rn(acc, __dmul_rn(pe[u].v, xv[u]));
  }
  return acc;
}


// Uniform slices of at most 8 entries per row only (7-point stencils): the
// short-row body alone, so the kernel needs fewer registers than the general
// pair kernel and more warps fit on an SM.
#ifndef PG_PAIR_SHORT_MIN_BLOCKS
#define PG_PAIR_SHORT_MIN_BLOCKS 4
#endif
template <int MODE>
__global__ void __launch_bounds__(kSellThreads, PG_PAIR_SHORT_MIN_BLOCKS)
    sell_pair_short_kernel(SellArgs a, const uint8_t* __restrict__ pair8,
                           const PairEnt* __restrict__ ptab, const double* __restrict__ x,
                           Epi e, double* partials, unsigned int* counter, double* nsq) {
  pdl_entry();
  __shared__ PairEnt s_ptab[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s_ptab[i] = ptab[i];
  __syncthreads();
  double local = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t lane = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; lane < a.nlanes;
       lane += stride) {
    const int64_t row = lane_row(a, lane);
    if (row < 0) continue;
    const int len = __ldg(a.row_len + lane);
    const Pre pre = epi_load<MODE>(e, x, row);
    const uint32_t* pw =
        reinterpret_cast<const uint32_t*>(pair8 + (lane >> 5) * a.stride8 + 4 * (lane & 31));
    const double ax = len > 0 ? row_sum_pairs_short(pw, len, row, x, s_ptab) : 0.0;
    const double r = epilogue<MODE>(e, pre, row, ax);
    if (MODE == kResid) local = __fma_rn(r, r, local);
  }
  finish_resid<MODE>(local, partials, counter, nsq);
}

template <int MODE>
__global__ void __launch_bounds__(kSellThreads, PG_SELL_DICT_MIN_BLOCKS)
    sell_pair_kernel(SellArgs a, const uint8_t* __restrict__ pair8,
                     const PairEnt* __restrict__ ptab, const double* __restrict__ x, Epi e,
                     double* partials, unsigned int* counter, double* nsq) {
  pdl_entry();
  __shared__ PairEnt s_ptab[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s_ptab[i] = ptab[i];
  __syncthreads();
  double local = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t lane = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; lane < a.nlanes;
       lane += stride) {
    const int64_t row = lane_row(a, lane);
    if (row < 0) continue;
    const int64_t s = lane >> 5;
    const int len = __ldg(a.row_len + lane);
    // uniform slices: the stream offset needs no load, so the pair words are
    // requested together with the row length (one round trip less per row)
    const int64_t base8 =
        (a.stride8 > 0 ? s * a.stride8 : __ldg(a.slice_ptr8 + s)) + 4 * (lane & 31);
    const Pre pre = epi_load<MODE>(e, x, row);
    const int avail = a.stride8 > 0 ? (int)(a.stride8 >> 7) : (len + 3) >> 2;
    const uint32_t* pw = reinterpret_cast<const uint32_t*>(pair8 + base8);
    const double ax = (avail <= 2 && len > 0)
                          ? row_sum_pairs_short(pw, len, row, x, s_ptab)
                          : row_sum_pairs_global(pw, len, avail, row, x, s_ptab);
    const double r = epilogue<MODE>(e, pre, row, ax);
    if (MODE == kResid) local = __fma_rn(r, r, local);
  }
  finish_resid<MODE>(local, partials, counter, nsq);
}

// ------------------------------------------------------ row patterns --
// One byte per row names its whole (offset, value) sequence (abi.cu
// build_patterns): the matrix stream is n bytes, the table lives in shared
// memory.  The table is staged before griddepcontrol.wait (it is never
// written after matrix creation), so the copy overlaps the previous kernel.
#ifndef PG_PAT_MIN_BLOCKS
#define PG_PAT_MIN_BLOCKS 4
#endif
// LB > 0: rows whose pattern is a masked subsequence of the master pattern
// (pm, pmask) take the unrolled constant-operand path row_sum_master<LB>;
// the others (and LB = 0) walk their pattern's table entries.
template <int MODE, int LB>
__global__ void __launch_bounds__(kSellThreads, PG_PAT_MIN_BLOCKS)
    sell_pat_kernel(SellArgs a, const uint8_t* __restrict__ rpat,
                    const int32_t* __restrict__ pptr, const PairEnt* __restrict__ pent, int npat,
                    int nent, const uint32_t* __restrict__ pmask, const PatMaster pm,
                    const double* __restrict__ x, Epi e, double* partials,
                    unsigned int* counter, double* nsq) {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  extern __shared__ __align__(16) unsigned char smem_pat[];
  const int32_t* s_ptr = stage_patterns(smem_pat, pptr, pent, npat, nent, pmask);
  const uint32_t* s_mask = reinterpret_cast<const uint32_t*>(s_ptr + npat + 1);
  const PairEnt* s_ent = reinterpret_cast<const PairEnt*>(smem_pat);
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  __syncthreads();
  double local = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // nlanes is a multiple of 32: a warp's lanes run the same iterations, so
  // the warp-uniform "all rows are the whole master" test below is safe
  const uint32_t full = pm.len >= 32 ? 0xffffffffu : (1u << pm.len) - 1u;
  for (int64_t lane = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; lane < a.nlanes;
       lane += stride) {
    const int64_t row = lane_row(a, lane);
    const int pid = row >= 0 ? __ldg(rpat + lane) : 0;
    const uint32_t mask = LB > 0 ? s_mask[pid] : (1u << 31);
    // FULL rows only for an exact-length instantiation: a bucket's inert tail
    // entries must not be added
    const bool all_full =
        LB > 0 && pm.len == LB && __all_sync(0xffffffffu, row < 0 || mask == full);
    if (row < 0) continue;
    const Pre pre = epi_load<MODE>(e, x, row);
    double ax;
    if (all_full)
      ax = row_sum_master<(LB > 0 ? LB : 8), false, false, true>(mask, pm, nullptr, x + row);
    else if (LB > 0 && !(mask >> 31))
      ax = row_sum_master<(LB > 0 ? LB : 8), false>(mask, pm, nullptr, x + row);
    else
      ax = row_sum_pattern<false>(s_ptr[pid], s_ptr[pid + 1], row, x, s_ent);
    const double r = epilogue<MODE>(e, pre, row, ax);
    if (MODE == kResid) local = __fma_rn(r, r, local);
  }
  finish_resid<MODE>(local, partials, counter, nsq);
}

// ------------------------------------------------------ offset patterns --
// Variable-coefficient stencils (abi.cu build_offset_patterns): 1 B per row
// names the row's column-offset sequence; masked subsequences of the master
// read only their values (8 B per entry, coalesced) and gather x at the
// master's constant offsets; other rows walk the SELL column stream.
template <int MODE, int LB>
__global__ void __launch_bounds__(kSellThreads, PG_PAT_MIN_BLOCKS)
    sell_opat_kernel(SellArgs a, const uint8_t* __restrict__ opat,
                     const uint32_t* __restrict__ omask, int npat, const PatMaster pm,
                     const double* __restrict__ x, Epi e, double* partials,
                     unsigned int* counter, double* nsq) {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  __shared__ uint32_t s_mask[256];
  for (int i = threadIdx.x; i < npat; i += blockDim.x) s_mask[i] = omask[i];
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  __syncthreads();
  double local = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint32_t full = pm.len >= 32 ? 0xffffffffu : (1u << pm.len) - 1u;
  for (int64_t lane = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; lane < a.nlanes;
       lane += stride) {
    const int64_t row = lane_row(a, lane);
    const int pid = row >= 0 ? __ldg(opat + lane) : 0;
    const uint32_t mask = s_mask[pid];
    // FULL rows only for an exact-length instantiation (see sell_pat_kernel)
    const bool all_full = pm.len == LB && __all_sync(0xffffffffu, row < 0 || mask == full);
    if (row < 0) continue;
    const int64_t s = lane >> 5;
    const int64_t base = __ldg(a.slice_ptr + s) + (lane & 31);
    const Pre pre = epi_load<MODE>(e, x, row);
    double ax;
    if (all_full) {
      ax = row_sum_omaster<LB, true>(mask, pm, a.val + base, x + row);
    } else if (!(mask >> 31)) {
      ax = row_sum_omaster<LB, false>(mask, pm, a.val + base, x + row);
    } else {
      ax = row_sum(
          [&](int j) { return __ldcs(a.col + base + (int64_t)j * PG_SLICE); },
          [](int raw) { return raw; },
          [&](int j) { return __ldcs(a.val + base + (int64_t)j * PG_SLICE); },
          __ldg(a.slice_w + s), __ldg(a.row_len + lane), x);
    }
    const double r = epilogue<MODE>(e, pre, row, ax);
    if (MODE == kResid) local = __fma_rn(r, r, local);
  }
  finish_resid<MODE>(local, partials, counter, nsq);
}

// ---------------------------------------------------- windowed dictionary --
// Dictionary-compressed matrices in natural row order (stencils): a ring
// stage holds kWinRows consecutive rows (kWinRows / 32 slices).  Their x reads all fall inside
// the few group windows of the matrix's window plan (abi.cu
// build_window_plan), and their packed index words are one contiguous byte
// range per stream.  One thread streams all of it for the block's next row
// blocks into a shared-memory ring (WinArgs::stages deep) with cp.async.bulk (TMA)
// completing on an mbarrier, so a stage carries ~15-35 KB of loads in flight
// per copy batch; the row threads then sum their rows from shared memory
// only.  Window elements outside [0, ncols) are never referenced by a stored
// entry and are simply not copied.  Same sequential mul-then-add order per
// row: bitwise equal to the other kernels.
// 1: epilogue operands, row lengths and slice widths ride in the ring stage
// (bulk copies); 0: the row threads load them from global before waiting
#ifndef PG_WIN_STAGE_EPI
#define PG_WIN_STAGE_EPI 1
#endif
constexpr bool kWinStageEpiPair = PG_WIN_STAGE_EPI;
// Row-pattern stages leave the epilogue operands to the row threads (coalesced
// loads issued before the stage wait): the smaller stage buys a deeper ring
// (cfg4-160^3 pass 49.9 -> 49.0 us)
#ifndef PG_WIN_PAT_STAGE_EPI
#define PG_WIN_PAT_STAGE_EPI 0
#endif
template <bool PAT>
constexpr bool kWinStageEpi = PAT ? (bool)PG_WIN_PAT_STAGE_EPI : kWinStageEpiPair;

struct WinArgs {
  int ng, total, b8, stages;
  // byte offsets inside a ring stage: [window | pair stream | epilogue
  // operand A | operand B | row lengths | slice widths]
  int off_p8, off_ea, off_eb, off_rl, off_sw, stage_bytes;
  int64_t ncols, nblk, n_slices;
  int32_t lo[kWinMaxGroups], start[kWinMaxGroups], len[kWinMaxGroups];
};

// Row sum over the pair stream: per entry one byte -> one 16-byte table
// entry {value, window byte offset} -> one window load, mul, add.  Full
// 4-entry chunks run without predicates; only the row's last partial chunk
// is predicated.  Same sequential order as every other kernel.
__device__ __forceinline__ double row_sum_pairs(const uint32_t* pw, int len,
                                                const unsigned char* winrow,
                                                const PairEnt* s_ptab) {
  // one 16-byte shared load per table entry (value + window offset)
  auto ent = [&](uint32_t idx, double& v, int& woff) {
    const int4 raw = reinterpret_cast<const int4*>(s_ptab)[idx];
    v = __hiloint2double(raw.y, raw.x);
    woff = raw.z;
  };
  double acc = 0.0;
  const int full = len & ~3;
  int j = 0;
#pragma unroll 2
  for (; j < full; j += 4) {
    const uint32_t pb = pw[(j >> 2) * PG_SLICE];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      double v;
      int woff;
      ent((pb >> (8 * u)) & 255u, v, woff);
      acc = __dadd_rn(acc, __dmul_rn(v, *reinterpret_cast<const double*>(winrow + woff)));
    }
  }
  if (j < len) {
    const uint32_t pb = pw[(j >> 2) * PG_SLICE];
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      if (j + u < len) {
        double v;
        int woff;
        ent((pb >> (8 * u)) & 255u, v, woff);
        acc = __dadd_rn(acc, __dmul_rn(v, *reinterpret_cast<const double*>(winrow + woff)));
      }
    }
  }
  return acc;
}

// Copy n doubles src -> dst (both 16-byte aligned) on `bar`: the even part in
// one bulk copy, an odd tail by a plain copy (made visible to the consumers
// by the release of the arrive).  Returns the bulk bytes (0 = nothing).
__device__ __forceinline__ uint32_t stage_f64_tail(double* dst, const double* src, int64_t n) {
  if (n & 1) dst[n - 1] = __ldg(src + n - 1);
  return 8u * (uint32_t)(n & ~(int64_t)1);
}

// Producer side (one thread): queue row block rb into ring stage `buf`.
// PAT: the matrix stream is the block's row-pattern bytes (pair8 = rpat,
// one byte per row) instead of the packed pair stream, row lengths and slice
// widths.
template <int MODE, bool PAT>
__device__ __forceinline__ void win_issue(const SellArgs& a, const WinArgs& wa, const Epi& e,
                                          const uint8_t* __restrict__ pair8,
                                          const double* __restrict__ x, int64_t rb,
                                          int64_t p0, int64_t p1, unsigned char* buf,
                                          uint64_t* bar) {
  double* win = reinterpret_cast<double*>(buf);
  const int64_t s0 = rb * (kWinRows / PG_SLICE);
  const int64_t s1 = min(s0 + kWinRows / PG_SLICE, wa.n_slices);
  const int64_t r0 = rb * kWinRows;
  const int64_t nr = min((int64_t)kWinRows, a.nrows - r0);
  const double *A, *B;
  epi_vectors<MODE>(e, x, A, B);
  if (PAT) {  // pattern ids of the block's rows: rpat is padded to whole slices
    p0 = r0;
    p1 = r0 + ((nr + 15) & ~(int64_t)15);
  }
  // pass 1: byte count (+ odd tails), so that expect_tx precedes the copies
  uint32_t bytes = (uint32_t)(p1 - p0);
  if (kWinStageEpi<PAT> && !PAT)  // row lengths + slice widths (bulk unless a partial block)
    bytes += 4u * (uint32_t)((s1 - s0) * PG_SLICE) +
             ((s1 - s0) * 4 % 16 == 0 ? 4u * (uint32_t)(s1 - s0) : 0u);
  for (int g = 0; g < wa.ng; ++g) {
    const int64_t ga = r0 + wa.lo[g];
    const int64_t va = max(ga, (int64_t)0), vb = min(ga + wa.len[g], wa.ncols);
    if (vb > va) bytes += stage_f64_tail(win + wa.start[g] + (va - ga), x + va, vb - va);
  }
  int32_t* sw = reinterpret_cast<int32_t*>(buf + wa.off_sw);
  if (kWinStageEpi<PAT>) {
    if (A) bytes += stage_f64_tail(reinterpret_cast<double*>(buf + wa.off_ea), A + r0, nr);
    if (B) bytes += stage_f64_tail(reinterpret_cast<double*>(buf + wa.off_eb), B + r0, nr);
    if (!PAT && (s1 - s0) * 4 % 16 != 0)  // partial last block: slice widths copied plainly
      for (int64_t q = s0; q < s1; ++q) sw[q - s0] = __ldg(a.slice_w + q);
  }
  mbar_expect_tx(bar, bytes);
  for (int g = 0; g < wa.ng; ++g) {
    const int64_t ga = r0 + wa.lo[g];
    const int64_t va = max(ga, (int64_t)0), vb = min(ga + wa.len[g], wa.ncols);
    const int64_t n2 = (vb - va) & ~(int64_t)1;
    if (vb > va && n2 > 0)
      bulk_g2s(win + wa.start[g] + (va - ga), x + va, 8u * (uint32_t)n2, bar);
  }
  if (p1 > p0) bulk_g2s(buf + wa.off_p8, pair8 + p0, (uint32_t)(p1 - p0), bar);
  if (kWinStageEpi<PAT>) {
    if (A && nr > 1) bulk_g2s(buf + wa.off_ea, A + r0, 8u * (uint32_t)(nr & ~(int64_t)1), bar);
    if (B && nr > 1) bulk_g2s(buf + wa.off_eb, B + r0, 8u * (uint32_t)(nr & ~(int64_t)1), bar);
    if (!PAT) {
      bulk_g2s(buf + wa.off_rl, a.row_len + r0, 4u * (uint32_t)((s1 - s0) * PG_SLICE), bar);
      if ((s1 - s0) * 4 % 16 == 0) bulk_g2s(sw, a.slice_w + s0, 4u * (uint32_t)(s1 - s0), bar);
    }
  }
}

// Warp-specialised: the last warp (kWinRowThreads / 32) is the producer (one
// lane issues the copies of the block's row blocks as soon as a ring stage is
// released); the kWinRowThreads row threads sum kWinRPT rows each from shared
// memory (row-pattern stages: pattern ids + x window by TMA, epilogue
// operands from global before the wait; pair-stream stages, one row per
// thread: stream, window, operands, row lengths all by TMA) and release the
// stage through the `empty` mbarrier.
// Row threads per block; a row-pattern stage of kWinRows rows gives each
// row thread kWinRows / kWinRowThreads rows (pair-stream stages: one).
#ifndef PG_WIN_ROW_THREADS
#define PG_WIN_ROW_THREADS 512
#endif
constexpr int kWinRowThreads = PG_WIN_ROW_THREADS;
constexpr int kWinRPT = kWinRows / kWinRowThreads;
static_assert(kWinRows % kWinRowThreads == 0, "stage rows must be whole row-thread sweeps");
constexpr int kWinThreads = kWinRowThreads + 32;

#ifndef PG_WIN_MIN_BLOCKS
#define PG_WIN_MIN_BLOCKS 2
#endif
// PAT = true: row-pattern matrices (pair8 = rpat; pptr / pent / npat / nent
// the pattern table, staged after the ring): a row is its pattern's entries,
// each one table entry {value, window offset} (a broadcast for the warp's
// interior rows), one window load, mul, add -- no per-entry stream.
template <int MODE, bool PAT, int LB>
__global__ void __launch_bounds__(kWinThreads, PG_WIN_MIN_BLOCKS)
    sell_win_kernel(SellArgs a, WinArgs wa, const uint8_t* __restrict__ pair8,
                    const PairEnt* __restrict__ ptab, const double* __restrict__ x, Epi e,
                    double* partials, unsigned int* counter, double* nsq,
                    const int32_t* __restrict__ pptr, int npat, int nent,
                    const uint32_t* __restrict__ pmask, const PatMaster pm) {
  static_assert(PAT || kWinRPT == 1, "the pair-stream stage sums one row per thread");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  extern __shared__ __align__(128) unsigned char smem_win[];
  __shared__ PairEnt s_ptab[PAT ? 1 : 256];
  __shared__ __align__(8) uint64_t full[kWinMaxStages];
  __shared__ __align__(8) uint64_t empty[kWinMaxStages];
  __shared__ int64_t wtag[kWinMaxStages];  // PG_CHECKS: the row block a slot holds
  const int S = wa.stages;
  // the tables never change after matrix creation: staged before the wait
  const int32_t* s_pptr = nullptr;
  const PairEnt* s_pent = nullptr;
  const uint32_t* s_mask = nullptr;
  if (PAT) {
    unsigned char* tab = smem_win + (size_t)S * wa.stage_bytes;
    s_pptr = stage_patterns(tab, pptr, ptab, npat, nent, pmask);
    s_pent = reinterpret_cast<const PairEnt*>(tab);
    s_mask = reinterpret_cast<const uint32_t*>(s_pptr + npat + 1);
  } else {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_ptab[i] = ptab[i];
  }
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  if (threadIdx.x == 0) {
    for (int st = 0; st < S; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kWinRowThreads / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();
  double local = 0.0;
  const int warp = threadIdx.x >> 5;
  if (warp == kWinRowThreads / 32) {
    if ((threadIdx.x & 31) == 0) {
      // the packed-stream bounds of the next row block are loaded one
      // iteration ahead, off the issue path
      auto bounds = [&](int64_t rb, int64_t& p0, int64_t& p1) {
        if (PAT || rb >= wa.nblk) return;
        const int64_t s0 = rb * (kWinRows / PG_SLICE);
        p0 = __ldg(a.slice_ptr8 + s0);
        p1 = __ldg(a.slice_ptr8 + min(s0 + kWinRows / PG_SLICE, wa.n_slices));
      };
      int64_t p0 = 0, p1 = 0, q0 = 0, q1 = 0;
      bounds(blockIdx.x, p0, p1);
      // ring slot and its reuse round kept as running counters (no integer
      // division by the runtime stage count per row block)
      int st = 0, round = 0;
      for (int64_t rb = blockIdx.x; rb < wa.nblk; rb += gridDim.x) {
        bounds(rb + gridDim.x, q0, q1);
        if (round > 0) mbar_wait(&empty[st], (uint32_t)((round - 1) & 1));
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        if (PG_CHECKS) wtag[st] = rb;
        win_issue<MODE, PAT>(a, wa, e, pair8, x, rb, p0, p1,
                             smem_win + (size_t)st * wa.stage_bytes, &full[st]);
        p0 = q0;
        p1 = q1;
        if (++st == S) {
          st = 0;
          ++round;
        }
      }
    }
  } else {
    const double *A, *B;
    epi_vectors<MODE>(e, x, A, B);
    const int t = threadIdx.x;
    const int sl = t >> 5;  // slice of this thread's row inside the block
    int st = 0;
    uint32_t phase = 0;
    const unsigned char* buf = smem_win;
    for (int64_t rb = blockIdx.x; rb < wa.nblk; rb += gridDim.x) {
      if (rb != blockIdx.x) {  // next ring slot (running counters, no division)
        buf += wa.stage_bytes;
        if (++st == S) {
          st = 0;
          phase ^= 1u;
          buf = smem_win;
        }
      }
      if (PAT) {
        // kWinRPT rows per thread (t, t + kWinRowThreads, ...): epilogue
        // operands requested before the stage wait, rows summed after it
        Pre pre[kWinRPT];
#pragma unroll
        for (int h = 0; h < kWinRPT; ++h) {
          const int64_t row = rb * kWinRows + t + h * kWinRowThreads;
          pre[h] = Pre{0.0, 0.0};
          if (!kWinStageEpi<PAT> && row < a.nrows) pre[h] = epi_load<MODE>(e, x, row);
        }
        mbar_wait(&full[st], phase);
        PG_DCHECK(wtag[st] == rb);
#pragma unroll
        for (int h = 0; h < kWinRPT; ++h) {
          const int th = t + h * kWinRowThreads;  // row slot inside the stage
          const int64_t row = rb * kWinRows + th;
          const bool live = row < a.nrows;
          const int pid = live ? buf[wa.off_p8 + th] : 0;
          const uint32_t mask = LB > 0 ? s_mask[pid] : (1u << 31);
          const uint32_t full = pm.len >= 32 ? 0xffffffffu : (1u << pm.len) - 1u;
          const bool all_full =
              LB > 0 && pm.len == LB && __all_sync(0xffffffffu, !live || mask == full);
          if (live) {
            if (kWinStageEpi<PAT> && A)
              pre[h].a = reinterpret_cast<const double*>(buf + wa.off_ea)[th];
            if (kWinStageEpi<PAT> && B)
              pre[h].b = reinterpret_cast<const double*>(buf + wa.off_eb)[th];
            const unsigned char* winrow = buf + 8 * th;
            double acc = 0.0;
            if (all_full) {
              acc = row_sum_master<(LB > 0 ? LB : 8), true, false, true>(mask, pm, winrow,
                                                                          nullptr);
            } else if (LB > 0 && !(mask >> 31)) {
              acc = row_sum_master<(LB > 0 ? LB : 8), true>(mask, pm, winrow, nullptr);
            } else {
              const int end = s_pptr[pid + 1];
#pragma unroll 4
              for (int q = s_pptr[pid]; q < end; ++q) {
                const int4 raw = reinterpret_cast<const int4*>(s_pent)[q];
                acc = __dadd_rn(acc, __dmul_rn(__hiloint2double(raw.y, raw.x),
                                               *reinterpret_cast<const double*>(winrow + raw.z)));
              }
            }
            const double r = epilogue<MODE>(e, pre[h], row, acc);
            if (MODE == kResid) local = __fma_rn(r, r, local);
          }
        }
        __syncwarp();
        if ((t & 31) == 0) mbar_arrive(&empty[st]);
        continue;
      }
      const int64_t row = rb * kWinRows + t;
      const bool live = row < a.nrows;
      const int lane = t & 31;
      int swl = 0, len = 0;
      Pre pre{0.0, 0.0};
      if (!kWinStageEpi<PAT>) {  // per-row operands from global, overlapping the wait
        const int64_t s0 = rb * (kWinRows / PG_SLICE);
        if (lane < sl && s0 + lane < wa.n_slices) swl = __ldg(a.slice_w + s0 + lane);
        if (live) {
          len = __ldg(a.row_len + row);
          pre = epi_load<MODE>(e, x, row);
        }
      }
      mbar_wait(&full[st], phase);
      PG_DCHECK(wtag[st] == rb);
      if (kWinStageEpi<PAT>) {
        if (lane < sl) swl = reinterpret_cast<const int32_t*>(buf + wa.off_sw)[lane];
        if (live) {
          len = reinterpret_cast<const int32_t*>(buf + wa.off_rl)[t];
          if (A) pre.a = reinterpret_cast<const double*>(buf + wa.off_ea)[t];
          if (B) pre.b = reinterpret_cast<const double*>(buf + wa.off_eb)[t];
        }
      }
      // packed-stream offset of this warp's slice inside the block: a warp
      // reduction over the widths of the slices before it (whole warp, before
      // the row guard)
      const int wq = lane < sl ? ((swl + 3) >> 2) * 4 * PG_SLICE : 0;
      const int off8 = (int)__reduce_add_sync(0xffffffffu, (unsigned)wq);
      if (live) {
        const uint32_t* pw = reinterpret_cast<const uint32_t*>(buf + wa.off_p8 + off8) + (t & 31);
        const double ax = row_sum_pairs(pw, len, buf + 8 * t, s_ptab);
        const double r = epilogue<MODE>(e, pre, row, ax);
        if (MODE == kResid) local = __fma_rn(r, r, local);
      }
      __syncwarp();
      if ((t & 31) == 0) mbar_arrive(&empty[st]);
    }
  }
  finish_resid<MODE>(local, partials, counter, nsq);
}

static SellArgs args_of(const pg_matrix* m) {
  SellArgs a;
  a.slice_ptr = m->slice_ptr;
  a.slice_w = m->slice_w;
  a.row_len = m->row_len;
  a.perm = m->perm;
  a.col = m->col;
  a.val = m->val;
  a.nrows = m->nrows;
  a.nlanes = m->n_slices * PG_SLICE;
  a.slice_ptr8 = m->slice_ptr8;
  a.col8 = m->col8;
  a.dtab = m->dtab;
  a.val8 = m->val8;
  a.vtab = m->vtab;
  a.stride8 = m->stride8;
  return a;
}

static int env_or(const char* name, int dflt) {
  const char* s = std::getenv(name);
  return s ? std::atoi(s) : dflt;
}

// The row-pattern kernel runs when the matrix has a pattern dictionary and,
// for matrices with a window plan (long stencil rows), only when
// PG_SPMV_PAT_WIN=1 (measured against the windowed kernel per matrix).
// The matrix's master pattern as kernel parameters (lb = 0: none, or
// PG_SPMV_MASTER=0).
static PatMaster master_of(const pg_matrix* m) {
  static int on = -1;
  if (on < 0) on = env_or("PG_SPMV_MASTER", 1);
  PatMaster pm;
  std::memset(&pm, 0, sizeof pm);
  if (!on || m->pat_mlen <= 0) return pm;
  pm.len = m->pat_mlen;
  pm.lb = (pm.len == 7 || pm.len == 27) ? pm.len : pm.len <= 8 ? 8 : pm.len <= 16 ? 16 : 32;
  for (int q = 0; q < pm.len; ++q) {
    pm.v[q] = m->pat_mv[q];
    pm.doff[q] = m->pat_mdoff[q];
    pm.woff[q] = m->pat_mwoff[q];
  }
  return pm;
}

// kernel-cache slot of an unrolled master length (0: none)
static int lb_index(int lb) {
  return lb == 7 ? 1 : lb == 8 ? 2 : lb == 16 ? 3 : lb == 27 ? 4 : lb == 32 ? 5 : 0;
}

// Offset-pattern kernel (PG_SPMV_OPAT_KERNEL=0: the plain SELL kernel).
bool opat_kernel(const pg_matrix* m) {
  static int on = -1;
  if (on < 0) on = env_or("PG_SPMV_OPAT_KERNEL", 1);
  return on && m->opat && m->opat_mlen > 0 && m->opat_mlen <= 31;
}

// Windowed matrices with a row-pattern dictionary take the windowed kernel's
// pattern variant (PG_SPMV_WINPAT=0: the pair-stream variant).
bool winpat_enabled() {
  static int on = -1;
  if (on < 0) on = env_or("PG_SPMV_WINPAT", 1);
  return on != 0;
}

bool pattern_kernel(const pg_matrix* m) {
  static int on = -1, win = -1;
  if (on < 0) {
    on = env_or("PG_SPMV_PAT_KERNEL", 1);
    win = env_or("PG_SPMV_PAT_WIN", 0);
  }
  return on && m->rpat && (!m->wtab || win);
}

template <int MODE>
static void launch_sell(const pg_matrix* m, const double* x, Epi e, pg_workspace* ws,
                        double* nsq, cudaStream_t st) {
  SellArgs a = args_of(m);
  if (MODE == kResid) {
    PG_REQUIRE(ws && nsq, PG_ERR_PARAMETER, "residual needs a workspace and nsq");
    PG_REQUIRE(ws->device == m->device, PG_ERR_PARAMETER, "workspace on another device");
  }
  if (a.nlanes == 0) {
    if (MODE == kResid) PG_CUDA(cudaMemsetAsync(nsq, 0, sizeof(double), st));
    return;
  }
  const int dev = m->device;
  PG_REQUIRE(dev >= 0 && dev < 64, PG_ERR_PARAMETER, "device ordinal out of range");
  // plane stencils: the plane-ring kernel (planes.cu), else the opt-in
  // plane-marching kernel (march.cu)
  if (plane_launch<MODE>(m, x, e, ws, nsq, st)) return;
  if (march_launch<MODE>(m, x, e, ws, nsq, st)) return;
  double* part = ws ? ws->partials : nullptr;
  unsigned* cnt = ws ? ws->counter : nullptr;
  static int sms[64] = {};
  if (!sms[dev]) PG_CUDA(cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev));
  // the window kernel's bulk copies need 16-byte aligned vectors
  auto al16 = [](const void* p) { return ((uintptr_t)p & 15u) == 0; };
  const bool aligned = al16(x) && al16(e.acc_in) && al16(e.base) && al16(e.b);
  // windowed kernel: long rows (27-point: 1.6x the pair kernel); short rows
  // (7-point) keep the global-gather pair kernel, which is faster there
  const bool win_pat = m->pair8 && m->wtab && aligned && m->rpat && winpat_enabled();
  // the pair-stream windowed kernel sums one row per thread per stage (it is
  // not built when the stage holds kWinRPT > 1 rows per thread)
  const bool win_ok =
      m->pair8 && m->wtab && aligned && (win_pat || (kWinRPT == 1 && m->win_pair_fits));
  if (pattern_kernel(m)) {
    int64_t blocks = (a.nlanes + kSellThreads - 1) / kSellThreads;
    static int per_sm = -1;
    if (per_sm < 0) per_sm = env_or("PG_SPMV_PAT_BLOCKS_PER_SM", PG_PAT_MIN_BLOCKS);
    const int64_t cap = (MODE == kResid) ? kMaxBlocks : (int64_t)sms[dev] * per_sm;
    if (blocks > cap) blocks = cap;
    const size_t smem = pattern_smem_bytes(m->n_pat, m->pat_nent);
    const PatMaster pm = master_of(m);
    auto kern = pm.lb == 7 ? sell_pat_kernel<MODE, 7> : pm.lb == 8 ? sell_pat_kernel<MODE, 8>
              : pm.lb == 16 ? sell_pat_kernel<MODE, 16> : pm.lb == 27 ? sell_pat_kernel<MODE, 27>
              : pm.lb == 32 ? sell_pat_kernel<MODE, 32> : sell_pat_kernel<MODE, 0>;
    static bool attr[4][6][64] = {};
    const int li = lb_index(pm.lb);
    if (!attr[MODE][li][dev]) {
      PG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)pattern_smem_bytes(256, kPatMaxEnt)));
      attr[MODE][li][dev] = true;
    }
    launch_k(kern, (int)blocks, kSellThreads, smem, st, a, (const uint8_t*)m->rpat,
             (const int32_t*)m->pat_ptr, (const PairEnt*)m->pat_ent, m->n_pat, m->pat_nent,
             (const uint32_t*)m->pat_mask, pm, x, e, part, cnt, nsq);
  } else if (win_ok) {
    WinArgs wa;
    wa.ng = m->n_wgrp;
    wa.total = m->win_elems;
    wa.b8 = m->win_b8;
    wa.off_p8 = ((8 * wa.total + 127) / 128) * 128;
    wa.off_ea = wa.off_p8 + (win_pat ? kWinRows : wa.b8);
    wa.off_eb = wa.off_ea + 8 * kWinRows;
    wa.off_rl = wa.off_eb + 8 * kWinRows;
    wa.off_sw = wa.off_rl + 4 * kWinRows;
    // row-pattern stages: window + pattern ids (+ the epilogue operands when
    // they ride in the ring)
    wa.stage_bytes = win_pat ? (kWinStageEpi<true> ? wa.off_rl : wa.off_ea) : wa.off_sw + 128;
    const PatMaster pm = win_pat ? master_of(m) : PatMaster{};
    // every pattern a masked master subsequence: the entry table is never read
    const int tab_nent = (win_pat && pm.lb > 0 && m->pat_all_master) ? 0 : m->pat_nent;
    const size_t tab_bytes = win_pat ? pattern_smem_bytes(m->n_pat, tab_nent) : 0;
    wa.ncols = m->ncols;
    wa.nblk = (m->nrows + kWinRows - 1) / kWinRows;
    wa.n_slices = m->n_slices;
    for (int g = 0; g < kWinMaxGroups; ++g) {
      wa.lo[g] = m->wlo[g];
      wa.start[g] = m->wstart[g];
      wa.len[g] = m->wlen[g];
    }
    wa.stages = (int)((kWinSmemBudget / kWinTargetBlocks - (int)tab_bytes) / wa.stage_bytes);
    if (wa.stages < 2) wa.stages = 2;
    if (wa.stages > kWinMaxStages) wa.stages = kWinMaxStages;
    const size_t smem = (size_t)wa.stages * wa.stage_bytes + tab_bytes;
    using WinKern = decltype(&sell_win_kernel<MODE, true, 0>);
    WinKern pair_kern = nullptr;
    if constexpr (kWinRPT == 1) pair_kern = sell_win_kernel<MODE, false, 0>;
    PG_REQUIRE(win_pat || pair_kern, PG_ERR_PARAMETER, "pair-stream windowed kernel not built");
    auto kern = !win_pat      ? pair_kern
                : pm.lb == 7  ? sell_win_kernel<MODE, true, 7>
                : pm.lb == 8  ? sell_win_kernel<MODE, true, 8>
                : pm.lb == 16 ? sell_win_kernel<MODE, true, 16>
                : pm.lb == 27 ? sell_win_kernel<MODE, true, 27>
                : pm.lb == 32 ? sell_win_kernel<MODE, true, 32>
                              : sell_win_kernel<MODE, true, 0>;
    const int pk = !win_pat ? 0 : 1 + lb_index(pm.lb);
    static bool attr[7][4][64] = {};
    if (!attr[pk][MODE][dev]) {
      PG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kWinSmemBudget));
      attr[pk][MODE][dev] = true;
    }
    // resident grid: blocks per SM from the occupancy calculator at this
    // stage size (cached per kernel / device / size) x PG_SPMV_WIN_WAVES
    static size_t occ_b[7][4][64] = {};
    static int occ_n[7][4][64] = {};
    if (occ_b[pk][MODE][dev] != smem) {
      int nb = 0;
      PG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kWinThreads, smem));
      occ_n[pk][MODE][dev] = nb > 0 ? nb : 1;
      occ_b[pk][MODE][dev] = smem;
    }
    static int waves = -1;
    if (waves < 0) {
      const char* s = std::getenv("PG_SPMV_WIN_WAVES");
      waves = s ? std::atoi(s) : 1;
    }
    int64_t g = waves > 0 ? (int64_t)sms[dev] * occ_n[pk][MODE][dev] * waves : wa.nblk;
    // PG_SPMV_WIN_GRID caps the grid (tests: many row blocks per CTA, so the
    // ring's slot reuse, empty-barrier waits and phase flips all run)
    static int gcap = -1;
    if (gcap < 0) gcap = env_or("PG_SPMV_WIN_GRID", 0);
    if (gcap > 0 && g > gcap) g = gcap;
    if (g > wa.nblk) g = wa.nblk;
    if (MODE == kResid && g > kMaxBlocks) g = kMaxBlocks;
    if (win_pat)
      launch_k(kern, (int)g, kWinThreads, smem, st, a, wa, (const uint8_t*)m->rpat,
               (const PairEnt*)m->pat_ent, x, e, part, cnt, nsq, (const int32_t*)m->pat_ptr,
               m->n_pat, tab_nent, (const uint32_t*)m->pat_mask, pm);
    else
      launch_k(kern, (int)g, kWinThreads, smem, st, a, wa, (const uint8_t*)m->pair8,
               (const PairEnt*)m->ptab, x, e, part, cnt, nsq, (const int32_t*)nullptr, 0, 0,
               (const uint32_t*)nullptr, pm);
  } else if (opat_kernel(m)) {
    int64_t blocks = (a.nlanes + kSellThreads - 1) / kSellThreads;
    static int per_sm = -1;
    if (per_sm < 0) per_sm = env_or("PG_SPMV_PAT_BLOCKS_PER_SM", PG_PAT_MIN_BLOCKS);
    const int64_t cap = (MODE == kResid) ? kMaxBlocks : (int64_t)sms[dev] * per_sm;
    if (blocks > cap) blocks = cap;
    PatMaster pm;
    std::memset(&pm, 0, sizeof pm);
    pm.len = m->opat_mlen;
    for (int q = 0; q < pm.len; ++q) pm.doff[q] = m->opat_mdoff[q];
    const int len = pm.len;
    auto kern = len == 9 ? sell_opat_kernel<MODE, 9> : len <= 8 ? sell_opat_kernel<MODE, 8>
              : len <= 16 ? sell_opat_kernel<MODE, 16> : sell_opat_kernel<MODE, 32>;
    launch_k(kern, (int)blocks, kSellThreads, 0, st, a, (const uint8_t*)m->opat,
             (const uint32_t*)m->opat_mask, m->opat_n, pm, x, e, part, cnt, nsq);
  } else if (m->pair8) {
    static int per_sm = -1;
    if (per_sm < 0) {
      const char* s = std::getenv("PG_SPMV_DICT_BLOCKS_PER_SM");
      per_sm = s ? std::atoi(s) : 4;
    }
    int64_t blocks = (a.nlanes + kSellThreads - 1) / kSellThreads;
    const int64_t cap = (MODE == kResid) ? kMaxBlocks : (int64_t)sms[dev] * per_sm;
    if (blocks > cap) blocks = cap;
    static int short_ok = -1, short_bps = -1;
    if (short_ok < 0) {
      const char* s = std::getenv("PG_SPMV_PAIR_SHORT");
      short_ok = s ? std::atoi(s) : 1;
      const char* b = std::getenv("PG_SPMV_SHORT_BLOCKS_PER_SM");
      short_bps = b ? std::atoi(b) : PG_PAIR_SHORT_MIN_BLOCKS;
    }
    if (short_ok && m->stride8 > 0 && m->stride8 <= 2 * 4 * PG_SLICE) {
      int64_t sb = (a.nlanes + kSellThreads - 1) / kSellThreads;
      const int64_t scap = (MODE == kResid) ? kMaxBlocks : (int64_t)sms[dev] * short_bps;
      if (sb > scap) sb = scap;
      launch_k(sell_pair_short_kernel<MODE>, (int)sb, kSellThreads, 0, st, a,
               (const uint8_t*)m->pair8, (const PairEnt*)m->ptab, x, e, part, cnt, nsq);
    } else {
      launch_k(sell_pair_kernel<MODE>, (int)blocks, kSellThreads, 0, st, a,
               (const uint8_t*)m->pair8, (const PairEnt*)m->ptab, x, e, part, cnt, nsq);
    }
  } else {
    // one row per thread; reductions keep the grid within the partial slots
    int64_t blocks = (a.nlanes + kSellThreads - 1) / kSellThreads;
    const int cm = m->col8 != nullptr, vm = m->val8 != nullptr;
    // compressed streams: a resident grid (grid-stride over rows) so each
    // block stages the dictionaries once, not once per 256 rows
    static int per_sm_env = -1;
    if (per_sm_env < 0) {
      const char* s = std::getenv("PG_SPMV_DICT_BLOCKS_PER_SM");
      per_sm_env = s ? std::atoi(s) : 4;  // measured best (4 / 16 / 64 swept)
    }
    const int64_t cap = (MODE == kResid) ? kMaxBlocks
                        : (cm || vm)     ? (int64_t)sms[dev] * per_sm_env
                                         : (int64_t)sms[dev] * 64;
    if (blocks > cap) blocks = cap;
    if (cm && vm)
      launch_k(sell_kernel<MODE, 1, 1>, (int)blocks, kSellThreads, 0, st, a, x, e, part, cnt, nsq);
    else if (cm)
      launch_k(sell_kernel<MODE, 1, 0>, (int)blocks, kSellThreads, 0, st, a, x, e, part, cnt, nsq);
    else if (vm)
      launch_k(sell_kernel<MODE, 0, 1>, (int)blocks, kSellThreads, 0, st, a, x, e, part, cnt, nsq);
    else
      launch_k(sell_kernel<MODE, 0, 0>, (int)blocks, kSellThreads, 0, st, a, x, e, part, cnt, nsq);
  }
  check_launch();
}

}  // namespace pg

using namespace pg;

extern "C" {

PG_API int pg_spmv(const pg_matrix* mat, const double* d_x, double* d_y, void* stream) {
  return guard([&] {
    PG_REQUIRE(mat && d_x && d_y, PG_ERR_PARAMETER, "null argument");
    Epi e{nullptr, nullptr, d_y, nullptr, nullptr, 0.0, 0.0, 0};
    launch_sell<kSpmv>(mat, d_x, e, nullptr, nullptr, as_stream(stream));
  });
}

PG_API int pg_poly_pass(const pg_matrix* mat, const double* d_x, const double* d_acc_in,
                        const double* d_base, double* d_acc_out, double* d_w_out, double y0,
                        double yk, int flags, void* stream) {
  return guard([&] {
    PG_REQUIRE(mat && d_x && d_acc_out, PG_ERR_PARAMETER, "null argument");
    PG_REQUIRE((flags & PG_PASS_FIRST) || d_acc_in, PG_ERR_PARAMETER,
               "acc_in required unless PG_PASS_FIRST");
    PG_REQUIRE(!(flags & PG_PASS_WRITE_W) || d_w_out, PG_ERR_PARAMETER,
               "w_out required with PG_PASS_WRITE_W");
    Epi e{d_acc_in, d_base, d_acc_out, d_w_out, nullptr, y0, yk, flags};
    launch_sell<kPoly>(mat, d_x, e, nullptr, nullptr, as_stream(stream));
  });
}

PG_API int pg_root_pass(const pg_matrix* mat, const double* d_x, const double* d_p,
                        const double* d_y_in, double* d_y_out, double* d_v_out, double c1,
                        double c2, double c3, int mode, void* stream) {
  return guard([&] {
    PG_REQUIRE(mat && d_x, PG_ERR_PARAMETER, "null argument");
    const int m = mode & 3;
    const bool resid = (mode & PG_ROOT_RESID) != 0;
    PG_REQUIRE((mode & ~(3 | PG_ROOT_RESID)) == 0 && m <= PG_ROOT_PAIR_B, PG_ERR_PARAMETER,
               "unknown root-pass mode");
    PG_REQUIRE(m != PG_ROOT_PAIR_B || d_p, PG_ERR_PARAMETER, "PAIR_B needs p");
    PG_REQUIRE(!resid || (m != PG_ROOT_PAIR_A && d_y_in && d_v_out && !d_y_out),
               PG_ERR_PARAMETER, "PG_ROOT_RESID: REAL/PAIR_B with v in y_in, output in v_out");
    PG_REQUIRE(d_y_out || d_v_out, PG_ERR_PARAMETER, "pass writes nothing");
    // d_y_in == nullptr: the running sum starts from zero
    Epi e{d_y_in, d_p, d_y_out, d_v_out, nullptr, 0.0, 0.0, mode, c1, c2, c3};
    launch_sell<kRoot>(mat, d_x, e, nullptr, nullptr, as_stream(stream));
  });
}

PG_API int pg_residual(const pg_matrix* mat, const double* d_x, const double* d_b, double* d_r,
                       double* d_nsq, pg_workspace* ws, void* stream) {
  return guard([&] {
    PG_REQUIRE(mat && d_x && d_b && d_r, PG_ERR_PARAMETER, "null argument");
    Epi e{nullptr, nullptr, d_r, nullptr, d_b, 0.0, 0.0, 0};
    launch_sell<kResid>(mat, d_x, e, ws, d_nsq, as_stream(stream));
  });
}

}  // extern "C"
