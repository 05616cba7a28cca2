// Internal declarations shared by the libpgmres translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>

#include "pgmres.h"

// Device-side invariant checks of the asynchronous kernels (ring-slot tags:
// the slot a consumer reads holds the tile / plane / row block it expects;
// shared-memory index bounds).  Compiled only into the checked library
// (PG_CHECKS=1: libpgmres_checked.so, tests/test_gpu_checked.py); a violated
// invariant prints the condition and traps, so the launch fails.  This stands
// in for compute-sanitizer, which is closed on the GPU pool this runs on.
#ifndef PG_CHECKS
#define PG_CHECKS 0
#endif
#define PG_DCHECK(cond)                                                                  \
  do {                                                                                   \
    if (PG_CHECKS && !(cond)) {                                                          \
      printf("PG_DCHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__,        \
             __LINE__, (int)blockIdx.x, (int)threadIdx.x);                               \
      __trap();                                                                          \
    }                                                                                    \
  } while (0)

namespace pg {

// ---------------------------------------------------------------- errors --
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);

#define PG_CUDA(expr)                                                              \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess)                                                         \
      throw ::pg::Error(PG_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

#define PG_REQUIRE(cond, code, msg) \
  do {                              \
    if (!(cond)) throw ::pg::Error((code), (msg)); \
  } while (0)

// Wrap an ABI body: exceptions -> status codes + last-error text.
template <class F>
int guard(F&& f) {
  try {
    f();
    return PG_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return PG_ERR_ALLOC;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return PG_ERR_CUDA;
  }
}

inline void check_launch() { PG_CUDA(cudaGetLastError()); }

// ------------------------------------------------------------ structures --
}  // namespace pg

namespace pg {
// Plane-ring kernel launch plan (planes.cu plane_prepare), fixed at matrix
// creation: tile width Q, tiles per plane, planes per chunk, in-plane halo H
// (+ parity shift sh so window starts are even), ring layout, and the window
// position of each middle-group value relative to the row's slot.
struct PlaneArgs {
  int64_t nrows, ncols, S, nz;
  int Q, nqb, Zc, H, sh;
  int stages, stage_bytes, off_a, off_b, off_p, off_bar;
  int woff[9];
  int allbox;  // end planes verified too: no stage reads pattern ids (planes.cu)
  int vec;     // adjacent row pairs move as aligned 16-byte pairs (planes.cu)
};
}  // namespace pg

struct pg_matrix {
  int device;
  int64_t nrows, ncols, nnz, padded_nnz, n_slices;
  int sigma, max_width;
  int64_t* slice_ptr;  // [n_slices+1] entry offset of each slice
  int32_t* slice_w;    // [n_slices]   slice width (max row length)
  int32_t* row_len;    // [n_slices*32] true length of the lane's row
  int32_t* perm;       // [n_slices*32] local row of lane (nullptr if sigma<=1)
  int32_t* col;        // [padded]  SELL column indices (int32)
  double* val;         // [padded]  SELL values
  int64_t* slice_ptr8; // [n_slices+1] slice offsets of the packed 1-byte streams
  int64_t stride8;     // > 0: every slice but the last spans stride8 bytes, so
                       // slice_ptr8[s] = s * stride8 (no dependent load)
  uint8_t* col8;       // packed dictionary index of (col - row), or null
  int32_t* dtab;       // [256]    column-offset dictionary
  uint8_t* val8;       // [padded] dictionary index of the value bits, or null
  double* vtab;        // [256]    value dictionary
  int n_dcol, n_dval;  // dictionary sizes (0 = stream not compressed)
  // x-window plan of the windowed dictionary kernel (spmv.cu): the column
  // offsets cluster into n_wgrp groups [wlo, wlo + wlen - kWinRows]; a block of
  // kWinRows natural-order rows reads x only inside the group windows, which
  // it stages in shared memory (group g at wstart[g]).  wtab[i] = smem
  // position of dictionary offset i for the block's first row.
  int32_t* wtab;       // [256] or null (no window plan)
  uint8_t* pair8;      // packed 1-byte index of the (column offset, value) pair
  void* ptab;          // [256] PairEnt {value, window byte offset, column offset}
  int n_wgrp, win_elems;
  int win_b8;          // largest per-block byte span of each packed stream
  int win_pair_fits;   // the pair-stream stage (window + stream + operands) fits a ring slot
  int32_t wlo[32], wstart[32], wlen[32];
  // row-pattern dictionary (abi.cu build_patterns): every row is one of
  // n_pat <= 256 distinct sequences of (column offset, value) pairs; rpat is
  // the 1-byte pattern id per SELL lane, pattern p's entries are
  // pat_ent[pat_ptr[p] .. pat_ptr[p+1]) (PairEnt), in the row's stored order
  uint8_t* rpat;
  int32_t* pat_ptr;
  void* pat_ent;
  int n_pat, pat_nent, pat_maxlen;
  // master pattern (the most frequent row, <= 31 entries): pat_mask[p] is
  // the bit set of master entries pattern p consists of, in order and with
  // identical values (a boundary row of a constant-coefficient stencil), or
  // bit 31 set when p is not such a subsequence
  int pat_mlen, pat_all_master;
  double pat_mv[32];
  int32_t pat_mdoff[32], pat_mwoff[32];
  uint32_t* pat_mask;
  // row OFFSET patterns (abi.cu build_offset_patterns), for matrices whose
  // values do not compress but whose column offsets col - row form <= 256
  // distinct row sequences (variable-coefficient stencils, cfg5): opat = 1 B
  // per SELL lane; the master offset sequence (<= 31) and per-pattern masks as
  // for pat_*; the values stay in the f64 SELL stream (val)
  uint8_t* opat;
  uint32_t* opat_mask;
  int opat_n, opat_mlen;
  int32_t opat_mdoff[32];
  // row dependency pattern of the dependency-driven chain kernel (chain.cu):
  // the n_doff distinct column offsets col - row (n_doff <= 256, from the
  // dictionary), or n_doff = 0 and the band [dband_lo, dband_hi] of offsets
  int n_doff;
  int32_t doff[256];
  int64_t dband_lo, dband_hi;
  // plane-ring kernel (planes.cu): plane_kind 0 = not a plane stencil / off
  int plane_kind, plane_blocks;
  int plane_sym;  // 1: outer plane groups share their coefficients but the center's

  pg::PlaneArgs plane;
  // plane_qm[q]: the in-plane entry mask of every interior-plane row at
  // in-plane index q (host-verified: the same box pattern on planes
  // 1 .. nz-2), or null when the rows do not have that structure
  uint16_t* plane_qm;
  size_t bytes;
};

namespace pg {
// One entry of the pair dictionary: the value and the byte offset of its
// column inside the block's x window (relative to the row's own slot).
struct __align__(16) PairEnt {
  double v;
  int32_t woff;  // byte offset in the block's x window (0 without a window plan)
  int32_t doff;  // column offset col - row (global-gather kernel)
};
// Rows per block of the windowed dictionary SpMV and its window budget
// (elements per buffer; two buffers per block).
// 512 rows per ring stage (544-thread blocks, 2 per SM): the per-stage
// mbarrier hand-offs and producer issue are amortised over twice the rows of
// the earlier 256 (cfg4-160^3 windowed row-pattern pass 61.6 -> 57.1 us;
// 128: 110, 384: 62.5, 768: 60.8 -- tools/spmv_bench.py over build variants)
// r01i: 1024-row stages swept by 512 row threads (two rows each) for the
// row-pattern variant (cfg4-160^3 49.6 -> 43.8 us; 768 rows / 384 threads 44.3).
// The pair-stream windowed kernel sums one row per thread, so with two rows
// per thread pattern-less windowed matrices take the global-gather pair kernel.
#ifndef PG_WIN_ROWS
#define PG_WIN_ROWS 1024
#endif
constexpr int kWinRows = PG_WIN_ROWS;
constexpr int kWinMaxGroups = 32;
constexpr int kWinMaxElems = 6144;
// Ring depth of the windowed kernel is chosen per matrix at launch: as many
// stages (2..kWinMaxStages) as fit kWinTargetBlocks blocks per SM.
constexpr int kWinMaxStages = 8;
#ifndef PG_WIN_TARGET_BLOCKS
#define PG_WIN_TARGET_BLOCKS 2
#endif
constexpr int kWinTargetBlocks = PG_WIN_TARGET_BLOCKS;
constexpr int kWinSmemBudget = 220 * 1024;
// a single stage must leave room for a second one in the budget
constexpr int kWinMaxStageBytes = kWinSmemBudget / 2 / 128 * 128;
// Number of per-block partial slots a reduction may use.
constexpr int kMaxBlocks = 1024;
// Row-pattern dictionary budget: table entries staged in shared memory per
// block (16 B each) and the longest pattern a kernel unrolls over.
constexpr int kPatMaxEnt = 2048;
constexpr int kPatMaxLen = 32;
// Per-block partial slots: the Gram stores (hi, lo) for each of the
// ncols*(ncols+1)/2 pairs, ncols <= PG_KMAX.
constexpr int kMaxOut = PG_KMAX * (PG_KMAX + 1);
}  // namespace pg

struct pg_workspace {
  int device;
  int num_sms;
  double* partials;        // [kMaxBlocks * kMaxOut]
  unsigned int* counter;   // completion counter (self-resetting)
  // chain kernel state (chain.cu): ctl = {ticket, exited, generation (u64)},
  // flags[chunk] = (generation << 8) | passes completed on that row chunk.
  // Grown on demand; retired arrays stay allocated until destroy because a
  // recorded graph may still reference them.
  unsigned int* chain_ctl;
  unsigned long long* chain_flags;
  int64_t chain_cap;
  void* chain_retired[32];
  int n_retired;
};

namespace pg {
// Deterministic fixed-order finish: every block has written `nout` partials
// at partials[blk*nout + i]; the last block to arrive sums them in block
// order into out[i] and resets the counter.  Call from all threads.
__device__ inline void last_block_reduce(double* partials, unsigned int* counter, int nout,
                                         double* out) {
  __shared__ bool am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int prev = atomicAdd(counter, 1u);
    am_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  // warp w finishes outputs w, w+nw, ...: lane l sums blocks l, l+32, ... (all
  // loads independent), then a fixed xor tree -- deterministic for a given grid
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned int G = gridDim.x;
  for (int i = warp; i < nout; i += nw) {
    double s = 0.0;
#pragma unroll 8
    for (unsigned int b = lane; b < G; b += 32) s += __ldcg(partials + (size_t)b * nout + i);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[i] = s;
  }
  if (threadIdx.x == 0) *counter = 0u;
}

// Deterministic block-wide sum of one double per thread (blockDim multiple of
// 32, <= 1024).  Result valid in thread 0.
__device__ inline double block_sum(double v) {
  __shared__ double warp_part[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) warp_part[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    int nw = blockDim.x >> 5;
    for (int i = 0; i < nw; ++i) s += warp_part[i];
  }
  return s;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------------------
// Programmatic dependent launch.  Every libpgmres kernel starts with
//   griddepcontrol.launch_dependents  -- the next kernel in the stream may be
//                                        scheduled once all our CTAs are resident
//   griddepcontrol.wait               -- block until the previous grid has
//                                        completed and its writes are visible
// and is launched with cudaLaunchAttributeProgrammaticStreamSerialization, so
// the launch latency and CTA rasterisation of kernel N+1 overlap kernel N's
// tail.  Results are unchanged: no kernel touches global memory before the
// wait.  PG_PDL=0 disables it.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
}

bool pdl_enabled();

// Distributed shards (dist.cu): fill x's ghost slots from the neighbours;
// sum count doubles over the ranks in rank order, in place.  No-ops for a
// null communicator.
void dist_halo(pg_dist* d, double* x, cudaStream_t st);
void dist_allreduce(pg_dist* d, double* buf, int count, cudaStream_t st);

// CGS2 of z against a basis wider than PG_KMAX in column tiles (ortho.cu;
// pg_cgs2_wide), with the reductions over dist's ranks when dist != null.
void cgs2_wide(const double* V, int64_t ld, int k, const double* z, int64_t n, double* c1,
               double* c2, double* nsq, double* w1, double* w2, pg_workspace* ws, pg_dist* dist,
               cudaStream_t st);

// Make `dev` current for a scope (restores the caller's device).
struct DeviceScope {
  int prev = 0;
  explicit DeviceScope(int dev) {
    PG_CUDA(cudaGetDevice(&prev));
    PG_CUDA(cudaSetDevice(dev));
  }
  ~DeviceScope() { cudaSetDevice(prev); }
};
// true while this thread records launches into a CUDA graph
extern thread_local bool g_capturing;

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  // launches recorded into a CUDA graph (pg_step_graph_create) get plain
  // edges: programmatic edges measured slower inside a graph
  cfg.numAttrs = (pdl_enabled() && !g_capturing) ? 1 : 0;
  PG_CUDA(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}

int grid_for(int device, const void* kernel, int block, size_t smem, int64_t work_blocks);

// out = x / sqrt(*nsq) and host[0..count) = ring[0..count) (host: a
// device-usable address of pinned host memory), one kernel (ortho.cu).
void normalize_publish(const double* x, const double* nsq, int64_t n, double* out,
                       const double* ring, int count, double* host, cudaStream_t st);

// One SpMV pass of a chain (chain.cu): x is the gathered vector; the other
// fields are the pass's epilogue (pg_poly_pass / pg_root_pass / pg_spmv
// arguments: acc_out doubles as the SpMV output).
enum { PG_CHAIN_SPMV = 0, PG_CHAIN_POLY = 1, PG_CHAIN_ROOT = 3 };
struct ChainStep {
  int mode;
  const double* x;
  const double* acc_in;
  const double* base;
  double* acc_out;
  double* w_out;
  double y0, yk;
  int flags;
  double c1, c2, c3;
};
// The plane-marching stencil kernel handles this matrix (march.cu): kind
// (27, 7, 9, 5), plane stride S and row stride g of its master pattern.
bool march_shape(const pg_matrix* m, int* kind, int64_t* S, int64_t* g);
// The master pattern is a plane stencil (any size; march.cu).
bool stencil_shape(const pg_matrix* m, int* kind, int64_t* S, int64_t* g);
// pg_spmv & co. run the plane-ring kernel on this matrix (planes.cu).
bool plane_shape(const pg_matrix* m);
// Fix the plane-ring launch plan of a new matrix (planes.cu).
void plane_prepare(pg_matrix* m);
// pg_spmv & co. run the row-pattern kernel on this matrix (spmv.cu).
bool pattern_kernel(const pg_matrix* m);
// pg_spmv & co. run the offset-pattern kernel on this matrix (spmv.cu).
bool opat_kernel(const pg_matrix* m);
// pg_spmv & co. on windowed matrices stage row patterns, not pair streams.
bool winpat_enabled();
// Matrix format the chain kernel handles (and PG_CHAIN != 0).
bool chain_supported(const pg_matrix* m);
// Issue the np passes as one dependency-driven kernel on st; false (nothing
// issued) when the matrix, the workspace or the pass count does not qualify.
bool chain_launch(const pg_matrix* m, const ChainStep* steps, int np, pg_workspace* ws,
                  cudaStream_t st);

}  // namespace pg
