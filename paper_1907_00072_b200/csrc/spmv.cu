// libpgmres: SELL-C-sigma fp64 SpMV and the fused polynomial pass.
//
// One thread owns one row (one lane of a 32-row slice).  Slice entries are
// stored lane-interleaved (entry j of lane t at slice_ptr[s] + j*32 + t), so
// each warp-wide load of the value / index streams is a contiguous 256 B /
// 128 B segment.  The row sum is accumulated sequentially in stored column
// order with separately rounded products (__dmul_rn / __dadd_rn: never
// contracted to FMA), which is bit-for-bit the reference SpMV
// (sparse.py:164-168, np.bincount over values*x[col]).
//
// The polynomial recurrence of apply_poly (polyprec.py:205-211) runs in the
// epilogue of the same pass: acc <- acc + y_k * (A w)[row], so a degree-d
// application streams A exactly d times with no separate axpy kernels.

#include "internal.cuh"

namespace pg {

enum SellMode { kSpmv = 0, kPoly = 1, kResid = 2 };

constexpr int kSellThreads = 256;
constexpr int kUnroll = 4;

struct SellArgs {
  const int64_t* __restrict__ slice_ptr;
  const int32_t* __restrict__ slice_w;
  const int32_t* __restrict__ row_len;
  const int32_t* __restrict__ perm;
  const int32_t* __restrict__ col;
  const double* __restrict__ val;
  int64_t nrows;
  int64_t nlanes;
};

// Sequential row sum, exact reference order.
__device__ __forceinline__ double sell_row(const SellArgs& a, int64_t lane,
                                           const double* __restrict__ x) {
  const int64_t s = lane >> 5;
  const int t = (int)(lane & 31);
  const int w = __ldg(a.slice_w + s);
  const int len = __ldg(a.row_len + lane);
  const int64_t base = __ldg(a.slice_ptr + s) + t;
  const int32_t* __restrict__ cp = a.col + base;
  const double* __restrict__ vp = a.val + base;
  double acc = 0.0;
  int j = 0;
  for (; j + kUnroll <= w; j += kUnroll) {
    int c[kUnroll];
    double v[kUnroll], xv[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      c[u] = __ldcs(cp + (int64_t)(j + u) * PG_SLICE);
      v[u] = __ldcs(vp + (int64_t)(j + u) * PG_SLICE);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) xv[u] = (j + u < len) ? __ldg(x + c[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (j + u < len) acc = __dadd_rn(acc, __dmul_rn(v[u], xv[u]));
  }
  for (; j < w; ++j) {
    int c = __ldcs(cp + (int64_t)j * PG_SLICE);
    double v = __ldcs(vp + (int64_t)j * PG_SLICE);
    if (j < len) acc = __dadd_rn(acc, __dmul_rn(v, __ldg(x + c)));
  }
  return acc;
}

__device__ __forceinline__ int64_t lane_row(const SellArgs& a, int64_t lane) {
  if (a.perm) return __ldg(a.perm + lane);
  return lane < a.nrows ? lane : -1;
}

template <int MODE>
__global__ void __launch_bounds__(kSellThreads)
    sell_kernel(SellArgs a, const double* __restrict__ x, const double* acc_in,
                const double* base, double* acc_out, double* w_out, double y0, double yk,
                int flags, const double* __restrict__ b, double* partials,
                unsigned int* counter, double* nsq) {
  double local = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t lane = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; lane < a.nlanes;
       lane += stride) {
    const int64_t row = lane_row(a, lane);
    if (row < 0) continue;
    const double ax = sell_row(a, lane, x);
    if (MODE == kSpmv) {
      acc_out[row] = ax;
    } else if (MODE == kPoly) {
      double t = (flags & PG_PASS_FIRST) ? __dmul_rn(y0, x[row]) : acc_in[row];
      t = __dadd_rn(t, __dmul_rn(yk, ax));
      if (flags & PG_PASS_WRITE_W) w_out[row] = ax;
      if (base) t = __dadd_rn(base[row], t);
      acc_out[row] = t;
    } else {  // residual r = b - A x, sum r^2
      const double r = __dsub_rn(b[row], ax);
      acc_out[row] = r;
      local = fma(r, r, local);
    }
  }
  if (MODE == kResid) {
    double s = block_sum(local);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
    last_block_reduce(partials, counter, 1, nsq);
  }
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
  return a;
}

template <int MODE>
static void launch_sell(const pg_matrix* m, const double* x, const double* acc_in,
                        const double* base, double* acc_out, double* w_out, double y0,
                        double yk, int flags, const double* b, pg_workspace* ws,
                        double* nsq, cudaStream_t st) {
  SellArgs a = args_of(m);
  int64_t blocks_needed = (a.nlanes + kSellThreads - 1) / kSellThreads;
  if (MODE == kResid) {
    PG_REQUIRE(ws && nsq, PG_ERR_PARAMETER, "residual needs a workspace and nsq");
    PG_REQUIRE(ws->device == m->device, PG_ERR_PARAMETER, "workspace on another device");
  }
  if (blocks_needed == 0) {
    if (MODE == kResid) PG_CUDA(cudaMemsetAsync(nsq, 0, sizeof(double), st));
    return;
  }
  // Grid: enough resident blocks to fill every SM; grid-stride beyond that.
  static int grid_cache[3][64] = {};
  int dev = m->device;
  int g;
  if (dev < 64 && grid_cache[MODE][dev] > 0) {
    g = grid_cache[MODE][dev];
  } else {
    g = grid_for(dev, (const void*)sell_kernel<MODE>, kSellThreads, 0, int64_t(1) << 40);
    if (dev < 64) grid_cache[MODE][dev] = g;
  }
  if (blocks_needed < g) g = (int)blocks_needed;
  sell_kernel<MODE><<<g, kSellThreads, 0, st>>>(
      a, x, acc_in, base, acc_out, w_out, y0, yk, flags, b,
      ws ? ws->partials : nullptr, ws ? ws->counter : nullptr, nsq);
  check_launch();
}

}  // namespace pg

using namespace pg;

extern "C" {

PG_API int pg_spmv(const pg_matrix* mat, const double* d_x, double* d_y, void* stream) {
  return guard([&] {
    PG_REQUIRE(mat && d_x && d_y, PG_ERR_PARAMETER, "null argument");
    launch_sell<kSpmv>(mat, d_x, nullptr, nullptr, d_y, nullptr, 0.0, 0.0, 0, nullptr,
                       nullptr, nullptr, as_stream(stream));
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
    launch_sell<kPoly>(mat, d_x, d_acc_in, d_base, d_acc_out, d_w_out, y0, yk, flags,
                       nullptr, nullptr, nullptr, as_stream(stream));
  });
}

PG_API int pg_residual(const pg_matrix* mat, const double* d_x, const double* d_b, double* d_r,
                       double* d_nsq, pg_workspace* ws, void* stream) {
  return guard([&] {
    PG_REQUIRE(mat && d_x && d_b && d_r, PG_ERR_PARAMETER, "null argument");
    launch_sell<kResid>(mat, d_x, nullptr, nullptr, d_r, nullptr, 0.0, 0.0, 0, d_b, ws, d_nsq,
                        as_stream(stream));
  });
}

}  // extern "C"
