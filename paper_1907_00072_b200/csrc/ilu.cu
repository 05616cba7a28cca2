// libpgmres: ILU(0) left preconditioning (reference
// ilu.py:38-114, IluPreconditionedOperator gmres.py:63-95).
//
// Factorisation (pg_ilu0_factor): host, once per matrix, the reference's IKJ
// elimination restricted to the pattern, in its operation order (one
// division per L entry, then `a_ij -= l_ik * u_kj` as a rounded product and a
// rounded difference), so the factors are bit-identical to ilu0_factor's.
//
// Application (pg_ilu_apply): z = U^{-1} L^{-1} v on the device with two
// sync-free triangular sweeps.  One warp owns one row; warps take rows in
// dependency order from an atomic ticket (ascending for L, descending for U),
// so every row a warp waits on is already owned by a running warp and the
// sweep cannot deadlock.  A row waits on the ready flags of its off-diagonal
// columns (acquire loads), sums its products in stored column order on lane 0
// (sequential, mul then add), writes its value and releases its flag.  The
// flags carry a per-sweep epoch, so they are never cleared.  The critical path
// is the matrix's level count (2g-1 for a g x g 5-point grid): this is the
// sequential bottleneck the polynomial preconditioner avoids.

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <vector>

#include "internal.cuh"

struct pg_ilu {
  int device;
  int64_t n;
  int32_t* lptr;   // [n+1] strictly-lower entries of row i: [lptr[i], lptr[i+1])
  int32_t* lcol;
  double* lval;
  int32_t* uptr;   // [n+1] strictly-upper entries
  int32_t* ucol;
  double* uval;
  double* diag;    // [n]  U's diagonal
  int32_t* flags;  // [n]  epoch of the sweep that finished row i
  int32_t* ticket; // [2]  row tickets of the two sweeps
  uint32_t epoch;
  size_t bytes;
};

namespace pg {

constexpr int kIluThreads = 256;

__device__ __forceinline__ int ld_acquire(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(int32_t* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// One sweep.  LOWER: y_i = v_i - sum_{j<i} l_ij y_j.  UPPER:
// z_i = (y_i - sum_{j>i} u_ij z_j) / d_i.
template <bool LOWER>
__global__ void __launch_bounds__(kIluThreads)
    ilu_sweep_kernel(int64_t n, const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                     const double* __restrict__ val, const double* __restrict__ diag,
                     const double* __restrict__ rhs, double* out, int32_t* flags,
                     int32_t* ticket, int epoch) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  for (;;) {
    int64_t t = 0;
    if (lane == 0) t = atomicAdd(reinterpret_cast<unsigned int*>(ticket), 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= n) return;
    const int64_t row = LOWER ? t : n - 1 - t;
    const int lo = __ldg(ptr + row), hi = __ldg(ptr + row + 1);
    double s = 0.0;
    for (int c = lo; c < hi; c += 32) {
      const int q = c + lane;
      double p = 0.0;
      if (q < hi) {
        const int j = __ldg(col + q);
        while (ld_acquire(flags + j) != epoch) {
        }
        // out[j] was written by another SM: read it from L2, not L1
        p = __dmul_rn(__ldg(val + q), __ldcg(out + j));
      }
      const int m = min(32, hi - c);
      for (int k = 0; k < m; ++k) {
        const double pk = __shfl_sync(0xffffffffu, p, k);
        if (lane == 0) s = __dadd_rn(s, pk);
      }
    }
    if (lane == 0) {
      double r = __dsub_rn(__ldg(rhs + row), s);
      if (!LOWER) r = __ddiv_rn(r, __ldg(diag + row));
      __stcg(out + row, r);
      st_release(flags + row, epoch);
    }
    __syncwarp();
  }
}

}  // namespace pg

using namespace pg;

namespace {

template <class T>
T* upload_vec(const std::vector<T>& h, size_t& bytes) {
  T* d = nullptr;
  const size_t nb = sizeof(T) * std::max<size_t>(h.size(), 1);
  if (cudaMalloc(&d, nb) != cudaSuccess) throw Error(PG_ERR_ALLOC, "cudaMalloc failed (ilu)");
  if (!h.empty()) PG_CUDA(cudaMemcpy(d, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice));
  bytes += nb;
  return d;
}

void free_ilu(pg_ilu* f) {
  if (!f) return;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(f->device);
  for (void* p : {(void*)f->lptr, (void*)f->lcol, (void*)f->lval, (void*)f->uptr,
                  (void*)f->ucol, (void*)f->uval, (void*)f->diag, (void*)f->flags,
                  (void*)f->ticket})
    cudaFree(p);
  cudaSetDevice(cur);
  delete f;
}

}  // namespace

extern "C" {

PG_API int pg_ilu0_factor(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                          const double* values, double diag_shift, double* out_values,
                          int64_t* out_diag_ptr, int64_t* fail_row, int* fail_kind) {
  return guard([&] {
    PG_REQUIRE(n >= 0 && row_ptr && fail_row && fail_kind && out_diag_ptr, PG_ERR_PARAMETER,
               "null argument");
    PG_REQUIRE(n == 0 || (col_idx && values && out_values), PG_ERR_PARAMETER, "null argument");
    *fail_row = -1;
    *fail_kind = 0;
    const int64_t nnz = row_ptr[n];
    std::copy(values, values + nnz, out_values);
    double* a = out_values;
    for (int64_t i = 0; i < n; ++i) {
      out_diag_ptr[i] = -1;
      for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p)
        if (col_idx[p] == i) out_diag_ptr[i] = p;
    }
    for (int64_t i = 0; i < n; ++i)
      if (out_diag_ptr[i] < 0) {  // ilu.py:59-63
        *fail_row = i;
        *fail_kind = 1;
        return;
      }
    if (diag_shift != 0.0)
      for (int64_t i = 0; i < n; ++i) a[out_diag_ptr[i]] += diag_shift;
    double dmax = 0.0;
    for (int64_t i = 0; i < n; ++i) dmax = std::max(dmax, std::fabs(a[out_diag_ptr[i]]));
    const double floor = std::numeric_limits<double>::epsilon() * dmax;  // ilu.py:67-69
    // position of column c inside the current row (-1: not in the pattern)
    std::vector<int64_t> pos(n, -1);
    for (int64_t i = 0; i < n; ++i) {
      const int64_t lo = row_ptr[i], hi = row_ptr[i + 1];
      for (int64_t p = lo; p < hi; ++p) pos[col_idx[p]] = p;
      for (int64_t p = lo; p < hi; ++p) {  // ilu.py:76-88, IKJ order
        const int64_t k = col_idx[p];
        if (k >= i) break;
        const double ukk = a[out_diag_ptr[k]];
        if (std::fabs(ukk) <= floor) {
          *fail_row = k;
          *fail_kind = 2;
          return;
        }
        const double lik = a[p] / ukk;
        a[p] = lik;
        for (int64_t q = out_diag_ptr[k] + 1; q < row_ptr[k + 1]; ++q) {
          const int64_t tgt = pos[col_idx[q]];
          if (tgt >= 0) {
            const double prod = lik * a[q];
            a[tgt] = a[tgt] - prod;
          }
        }
      }
      for (int64_t p = lo; p < hi; ++p) pos[col_idx[p]] = -1;
      if (std::fabs(a[out_diag_ptr[i]]) <= floor) {  // ilu.py:89-90
        *fail_row = i;
        *fail_kind = 2;
        return;
      }
    }
  });
}

PG_API int pg_ilu_create(int device, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                         const double* values, const int64_t* diag_ptr, pg_ilu** out) {
  return guard([&] {
    PG_REQUIRE(out && row_ptr && diag_ptr, PG_ERR_PARAMETER, "null argument");
    PG_REQUIRE(n >= 0 && n < (int64_t(1) << 31) && row_ptr[n] < (int64_t(1) << 31),
               PG_ERR_PARAMETER, "ILU size exceeds int32 indexing");
    *out = nullptr;
    std::vector<int32_t> lptr(n + 1, 0), uptr(n + 1, 0), lcol, ucol;
    std::vector<double> lval, uval, diag(n);
    for (int64_t i = 0; i < n; ++i) {
      const int64_t d = diag_ptr[i];
      PG_REQUIRE(d >= row_ptr[i] && d < row_ptr[i + 1] && col_idx[d] == i, PG_ERR_PARAMETER,
                 "diag_ptr does not point at the diagonal");
      for (int64_t p = row_ptr[i]; p < d; ++p) {
        lcol.push_back((int32_t)col_idx[p]);
        lval.push_back(values[p]);
      }
      for (int64_t p = d + 1; p < row_ptr[i + 1]; ++p) {
        ucol.push_back((int32_t)col_idx[p]);
        uval.push_back(values[p]);
      }
      diag[i] = values[d];
      lptr[i + 1] = (int32_t)lcol.size();
      uptr[i + 1] = (int32_t)ucol.size();
    }
    int prev = 0;
    PG_CUDA(cudaGetDevice(&prev));
    PG_CUDA(cudaSetDevice(device));
    pg_ilu* f = new pg_ilu();
    std::memset(f, 0, sizeof(*f));
    f->device = device;
    f->n = n;
    try {
      f->lptr = upload_vec(lptr, f->bytes);
      f->lcol = upload_vec(lcol, f->bytes);
      f->lval = upload_vec(lval, f->bytes);
      f->uptr = upload_vec(uptr, f->bytes);
      f->ucol = upload_vec(ucol, f->bytes);
      f->uval = upload_vec(uval, f->bytes);
      f->diag = upload_vec(diag, f->bytes);
      f->flags = upload_vec(std::vector<int32_t>(std::max<int64_t>(n, 1), 0), f->bytes);
      f->ticket = upload_vec(std::vector<int32_t>(2, 0), f->bytes);
    } catch (...) {
      free_ilu(f);
      cudaSetDevice(prev);
      throw;
    }
    cudaSetDevice(prev);
    *out = f;
  });
}

PG_API int pg_ilu_destroy(pg_ilu* f) {
  return guard([&] { free_ilu(f); });
}

PG_API int pg_ilu_apply(pg_ilu* f, const double* d_v, double* d_y, double* d_z, void* stream) {
  return guard([&] {
    PG_REQUIRE(f && d_v && d_y && d_z, PG_ERR_PARAMETER, "null argument");
    PG_REQUIRE(d_y != d_v && d_y != d_z, PG_ERR_PARAMETER, "y must not alias v or z");
    if (f->n == 0) return;
    cudaStream_t st = as_stream(stream);
    static int sms[64] = {};
    PG_REQUIRE(f->device >= 0 && f->device < 64, PG_ERR_PARAMETER, "device ordinal");
    if (!sms[f->device])
      PG_CUDA(cudaDeviceGetAttribute(&sms[f->device], cudaDevAttrMultiProcessorCount, f->device));
    // epochs 1, 2, 3, ... (flags start at 0); two per apply
    if (f->epoch > 0x7ffffff0u) {
      PG_CUDA(cudaMemsetAsync(f->flags, 0, sizeof(int32_t) * f->n, st));
      f->epoch = 0;
    }
    const int e1 = (int)++f->epoch, e2 = (int)++f->epoch;
    PG_CUDA(cudaMemsetAsync(f->ticket, 0, 2 * sizeof(int32_t), st));
    const int warps = kIluThreads / 32;
    int64_t blocks = (f->n + warps - 1) / warps;
    if (blocks > (int64_t)sms[f->device] * 8) blocks = (int64_t)sms[f->device] * 8;
    launch_k(ilu_sweep_kernel<true>, (int)blocks, kIluThreads, 0, st, f->n,
             (const int32_t*)f->lptr, (const int32_t*)f->lcol, (const double*)f->lval,
             (const double*)f->diag, d_v, d_y, f->flags, f->ticket, e1);
    check_launch();
    launch_k(ilu_sweep_kernel<false>, (int)blocks, kIluThreads, 0, st, f->n,
             (const int32_t*)f->uptr, (const int32_t*)f->ucol, (const double*)f->uval,
             (const double*)f->diag, (const double*)d_y, d_z, f->flags, f->ticket + 1, e2);
    check_launch();
  });
}

}  // extern "C"
