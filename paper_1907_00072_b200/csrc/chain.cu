// libpgmres: the d+1 SpMV passes of an Arnoldi step as ONE dependency-driven
// kernel (temporal blocking across the passes).  Opt-in
// (PG_CHAIN=1): correct and bit-identical, but measured slower than the
// pass-by-pass launches on B200 ("Chain kernel").
//
// z = A p(A) v is a chain of d+1 SpMV passes (polyprec.py:205-211 +
// gmres.py:112-113).  Issued as d+1 kernels, every pass pays a launch, a ramp
// and a tail, and no pass can start before the previous one has finished
// everywhere.  Here the passes are tickets of one resident kernel:
//
//  * ticket t = (pass k, row chunk c), t = k * nchunk + c; a chunk is TS
//    slices of 32 rows and one warp processes a ticket;
//  * pass k on chunk c may start once pass k-1 is complete on every chunk
//    whose rows chunk c's rows reference (the matrix's column offsets,
//    closed under negation so that a chunk is never overwritten while a
//    neighbour still gathers from it, and always containing c itself so each
//    chunk sees its passes in order).  Completion is a per-chunk flag
//    (generation << 8 | passes done), published with st.release.gpu and
//    polled with ld.acquire.gpu;
//  * tickets go round-robin to the warps of a cooperative (all-resident)
//    grid: warp w takes w, w + W, w + 2W, ...  Each warp takes its tickets in
//    increasing order and each ticket depends only on smaller ones, so the
//    smallest unfinished ticket can always proceed: no deadlock.  (An atomic
//    ticket counter, PG_CHAIN_DYNAMIC=1, needs no residency but is bound by
//    same-address atomic throughput, ~1.2 G/s measured on B200);
//  * the next pass starts on the first chunks while the previous pass is
//    still finishing the last ones, and the chain's working set (~35 MB at
//    n = 1e6) stays in the 126 MB L2 (ncu: 1.7% of DRAM peak).
//
// Row arithmetic is the per-pass kernels' (sell.cuh): same entry order, same
// separately rounded products, same epilogues -- results are bit-identical.
// Vectors written inside the kernel are read through L2 (ld.global.cg).
// Bodies: 1 = row patterns (pg_matrix::rpat), 0 = short-row pair stream.

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "internal.cuh"
#include "sell.cuh"

namespace pg {

constexpr int kChainMaxPass = PG_KMAX + 2;
constexpr int kChainMaxDep = 64;
constexpr int kChainThreads = 256;

struct ChainPassDev {
  const double* x;
  Epi e;
  int mode;
};

struct ChainParams {
  const int32_t* row_len;
  const uint8_t* pair8;
  const PairEnt* ptab;
  const uint8_t* rpat;  // row-pattern body: pattern id per row and the table
  const int32_t* pptr;
  const PairEnt* pent;
  const uint32_t* pmask;
  int npat, nent;
  PatMaster pm;  // master pattern (pm.lb == 8: unrolled row path; else table walk)
  int64_t nrows, nlanes, stride8;
  unsigned nchunk;
  unsigned* ctl;
  unsigned long long* flags;
  int npass, nd;
  int dynamic;  // 1: atomic ticket counter; 0: static round-robin (cooperative)
  int32_t dep[kChainMaxDep];
  ChainPassDev p[kChainMaxPass];
};

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}

// epi_load (spmv.cu) through L2: operands written earlier in this kernel
template <int MODE>
__device__ __forceinline__ Pre chain_pre(const Epi& e, const double* x, int64_t row) {
  Pre p{0.0, 0.0};
  if (MODE == kPoly) {
    p.a = __ldcg(((e.flags & PG_PASS_FIRST) ? x : e.acc_in) + row);
    if (e.base) p.b = __ldcg(e.base + row);
  } else if (MODE == kRoot) {
    p.a = __ldcg((((e.flags & 3) == PG_ROOT_PAIR_B) ? e.base : x) + row);
    if (e.acc_in) p.b = __ldcg(e.acc_in + row);
  }
  return p;
}

// BODY 0: pair stream (len, w0, w1 per row); BODY 1: row patterns (len
// carries the pattern id; s_tab is the pattern table, s_ptr its offsets)
template <int MODE, int TS, int BODY>
__device__ __forceinline__ void chain_rows(const ChainParams& P, const ChainPassDev& ps,
                                           int64_t c, int lane, const int (&len)[TS],
                                           const uint32_t (&w0)[TS], const uint32_t (&w1)[TS],
                                           const PairEnt* s_tab, const int32_t* s_ptr,
                                           const uint32_t* s_mask) {
#pragma unroll
  for (int u = 0; u < TS; ++u) {
    const int64_t row = ((int64_t)c * TS + u) * PG_SLICE + lane;
    if (row < P.nrows) {
      const Pre pre = chain_pre<MODE>(ps.e, ps.x, row);
      double ax;
      if (BODY == 1) {
        const uint32_t mask = s_mask[len[u]];
        if (P.pm.lb == 8 && !(mask >> 31))
          ax = row_sum_master<8, false, true>(mask, P.pm, nullptr, ps.x + row);
        else
          ax = row_sum_pattern<true>(s_ptr[len[u]], s_ptr[len[u] + 1], row, ps.x, s_tab);
      }
      else
        ax = len[u] > 0
                 ? row_sum_pair_words<true>(w0[u], w1[u], len[u], row, ps.x, s_tab)
                 : 0.0;
      epilogue<MODE>(ps.e, pre, row, ax);
    }
  }
}

// Pair-dictionary SELL with uniform slices of <= 8 entries per row (the
// short-row pass of spmv.cu, 7-point stencils), natural row order.
#ifndef PG_CHAIN_MIN_BLOCKS
#define PG_CHAIN_MIN_BLOCKS 4
#endif
template <int TS, int BODY>
__global__ void __launch_bounds__(kChainThreads, PG_CHAIN_MIN_BLOCKS)
    chain_kernel(const __grid_constant__ ChainParams P) {
  // the tables never change after matrix creation: staged before the wait
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  extern __shared__ __align__(16) unsigned char smem_chain[];
  const PairEnt* s_tab = reinterpret_cast<const PairEnt*>(smem_chain);
  const int32_t* s_ptr = nullptr;
  const uint32_t* s_mask = nullptr;
  if (BODY == 1) {
    s_ptr = stage_patterns(smem_chain, P.pptr, P.pent, P.npat, P.nent, P.pmask);
    s_mask = reinterpret_cast<const uint32_t*>(s_ptr + P.npat + 1);
  } else {
    PairEnt* t = reinterpret_cast<PairEnt*>(smem_chain);
    for (int i = threadIdx.x; i < 256; i += blockDim.x) t[i] = P.ptab[i];
  }
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  __syncthreads();
  const int lane = threadIdx.x & 31;
  unsigned* ctl = P.ctl;
  const unsigned long long gen = *reinterpret_cast<volatile unsigned long long*>(ctl + 2);
  const unsigned total = (unsigned)P.npass * P.nchunk;
  const bool two = P.stride8 > 4 * PG_SLICE;  // a second index word per lane
  // static round-robin tickets (cooperative launch: every warp is resident),
  // or, with P.dynamic, an atomic ticket counter (no residency assumption)
  const unsigned nw = gridDim.x * (blockDim.x >> 5);
  const unsigned wid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  unsigned t = wid;
  if (P.dynamic) {
    if (lane == 0) t = atomicAdd(ctl, 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
  }
  while (t < total) {
    // the next ticket is requested now and read at the end of this one
    unsigned tn = t + nw;
    if (P.dynamic && lane == 0) tn = atomicAdd(ctl, 1u);
    const unsigned k = t / P.nchunk;
    const int64_t c = (int64_t)(t - k * P.nchunk);
    // the chunk's matrix stream is read-only: loaded before the wait
    int len[TS];
    uint32_t w0[TS], w1[TS];
#pragma unroll
    for (int u = 0; u < TS; ++u) {
      const int64_t s = c * TS + u;
      const int64_t ln = s * PG_SLICE + lane;
      len[u] = 0;
      w0[u] = w1[u] = 0u;
      if (ln < P.nlanes) {
        if (BODY == 1) {
          len[u] = __ldg(P.rpat + ln);
        } else {
          len[u] = __ldg(P.row_len + ln);
          const uint32_t* pw =
              reinterpret_cast<const uint32_t*>(P.pair8 + s * P.stride8 + 4 * lane);
          w0[u] = __ldcs(pw);
          if (two) w1[u] = __ldcs(pw + PG_SLICE);
        }
      }
    }
    if (k > 0) {
      const unsigned long long need = (gen << 8) | (unsigned long long)k;
      for (int i = lane; i < P.nd; i += 32) {
        const int64_t f = c + P.dep[i];
        if (f >= 0 && f < (int64_t)P.nchunk)
          while (ld_acquire_u64(P.flags + f) < need) __nanosleep(32);
      }
      __syncwarp();
    }
    const ChainPassDev& ps = P.p[k];
    if (ps.mode == kPoly)
      chain_rows<kPoly, TS, BODY>(P, ps, c, lane, len, w0, w1, s_tab, s_ptr, s_mask);
    else if (ps.mode == kSpmv)
      chain_rows<kSpmv, TS, BODY>(P, ps, c, lane, len, w0, w1, s_tab, s_ptr, s_mask);
    else
      chain_rows<kRoot, TS, BODY>(P, ps, c, lane, len, w0, w1, s_tab, s_ptr, s_mask);
    // every lane's stores are ordered before lane 0's release (bar.warp.sync)
    __syncwarp();
    if (lane == 0) st_release_u64(P.flags + c, (gen << 8) | (unsigned long long)(k + 1));
    t = P.dynamic ? __shfl_sync(0xffffffffu, tn, 0) : tn;
  }
  // the last warp out resets the ticket counter and opens the next generation
  if (lane == 0) {
    __threadfence();
    if (atomicAdd(ctl + 1, 1u) == nw - 1) {
      ctl[0] = 0u;
      ctl[1] = 0u;
      *reinterpret_cast<volatile unsigned long long*>(ctl + 2) = gen + 1;
      __threadfence();
    }
  }
}

static int env_int(const char* name, int dflt) {
  const char* s = std::getenv(name);
  return s ? std::atoi(s) : dflt;
}

static int64_t floordiv(int64_t a, int64_t b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

// Relative chunk offsets pass k on chunk c waits on (pass k-1 done), for
// chunks of R rows; empty when the pattern is too wide for the kernel.
static std::vector<int32_t> chain_deps(const pg_matrix* m, int64_t R) {
  std::vector<int64_t> d;
  auto add = [&](int64_t o) {
    const int64_t lo = floordiv(o, R), hi = floordiv(R - 1 + o, R);
    for (int64_t x = lo; x <= hi; ++x) d.push_back(x);
  };
  add(0);
  if (m->n_doff > 0) {
    for (int i = 0; i < m->n_doff; ++i) {
      add(m->doff[i]);
      add(-(int64_t)m->doff[i]);
    }
  } else {
    const int64_t M = std::max(-m->dband_lo, m->dband_hi);
    if (M / R + 2 > kChainMaxDep) return {};
    const int64_t lo = floordiv(-M, R), hi = floordiv(R - 1 + M, R);
    for (int64_t x = lo; x <= hi; ++x) d.push_back(x);
  }
  std::sort(d.begin(), d.end());
  d.erase(std::unique(d.begin(), d.end()), d.end());
  if ((int)d.size() > kChainMaxDep) return {};
  return std::vector<int32_t>(d.begin(), d.end());
}

// 1: row-pattern body, 0: short-row pair body, -1: not supported
static int chain_body(const pg_matrix* m) {
  // opt-in (PG_CHAIN=1): measured slower than pass-by-pass launches on B200
  // ("Chain kernel")
  if (!m || env_int("PG_CHAIN", 0) == 0) return -1;
  // natural order, square (no halo between passes)
  if (m->nrows <= 0 || m->ncols != m->nrows || m->perm) return -1;
  if (m->rpat && m->pat_maxlen <= kPatMaxLen) return 1;
  if (m->pair8 && !m->wtab && m->stride8 > 0 && m->stride8 <= 2 * 4 * PG_SLICE) return 0;
  return -1;
}

bool chain_supported(const pg_matrix* m) { return chain_body(m) >= 0; }

bool chain_launch(const pg_matrix* m, const ChainStep* steps, int np, pg_workspace* ws,
                  cudaStream_t st) {
  const int body = chain_body(m);
  if (body < 0 || !ws || ws->device != m->device || np < 2 || np > kChainMaxPass) return false;
  int ts = env_int("PG_CHAIN_TS", 4);
  if (ts != 1 && ts != 2 && ts != 4 && ts != 8) ts = 4;
  const int64_t R = (int64_t)ts * PG_SLICE;
  const std::vector<int32_t> dep = chain_deps(m, R);
  if (dep.empty()) return false;
  const int64_t nchunk = (m->n_slices + ts - 1) / ts;
  if ((int64_t)np * nchunk + (1 << 20) >= ((int64_t)1 << 32)) return false;
  if (ws->chain_cap < nchunk) {
    // no allocation inside a graph capture: the caller issues the passes
    if (g_capturing) return false;
    PG_REQUIRE(ws->n_retired < 32, PG_ERR_ALLOC, "chain flag arrays exhausted");
    unsigned long long* f = nullptr;
    if (cudaMalloc(&f, sizeof(unsigned long long) * nchunk) != cudaSuccess)
      throw Error(PG_ERR_ALLOC, "chain flag allocation failed");
    PG_CUDA(cudaMemsetAsync(f, 0, sizeof(unsigned long long) * nchunk, st));
    if (ws->chain_flags) ws->chain_retired[ws->n_retired++] = ws->chain_flags;
    ws->chain_flags = f;
    ws->chain_cap = nchunk;
  }
  ChainParams P;
  std::memset(&P, 0, sizeof P);
  P.row_len = m->row_len;
  P.pair8 = m->pair8;
  P.ptab = (const PairEnt*)m->ptab;
  P.rpat = m->rpat;
  P.pptr = m->pat_ptr;
  P.pent = (const PairEnt*)m->pat_ent;
  P.pmask = m->pat_mask;
  P.pm.lb = 0;
  if (body == 1 && m->pat_mlen > 0 && m->pat_mlen <= 8) {
    P.pm.len = m->pat_mlen;
    P.pm.lb = 8;
    for (int q = 0; q < m->pat_mlen; ++q) {
      P.pm.v[q] = m->pat_mv[q];
      P.pm.doff[q] = m->pat_mdoff[q];
      P.pm.woff[q] = m->pat_mwoff[q];
    }
  }
  P.npat = m->n_pat;
  P.nent = m->pat_nent;
  P.nrows = m->nrows;
  P.nlanes = m->n_slices * PG_SLICE;
  P.stride8 = m->stride8;
  P.nchunk = (unsigned)nchunk;
  P.ctl = ws->chain_ctl;
  P.flags = ws->chain_flags;
  P.npass = np;
  P.nd = (int)dep.size();
  for (size_t i = 0; i < dep.size(); ++i) P.dep[i] = dep[i];
  for (int k = 0; k < np; ++k) {
    const ChainStep& s = steps[k];
    ChainPassDev& d = P.p[k];
    d.x = s.x;
    d.mode = s.mode == PG_CHAIN_SPMV ? kSpmv : s.mode == PG_CHAIN_POLY ? kPoly : kRoot;
    d.e = Epi{s.acc_in, s.base, s.acc_out, s.w_out, nullptr, s.y0, s.yk, s.flags,
              s.c1, s.c2, s.c3};
  }
  const int dev = m->device;
  void (*kern)(const ChainParams) = nullptr;
  if (body == 1)
    kern = ts == 1 ? chain_kernel<1, 1> : ts == 2 ? chain_kernel<2, 1>
         : ts == 8 ? chain_kernel<8, 1> : chain_kernel<4, 1>;
  else
    kern = ts == 1 ? chain_kernel<1, 0> : ts == 2 ? chain_kernel<2, 0>
         : ts == 8 ? chain_kernel<8, 0> : chain_kernel<4, 0>;
  const size_t smem = body == 1 ? pattern_smem_bytes(m->n_pat, m->pat_nent) : 16 * 256;
  static int occ[2][4][64] = {};
  static size_t occ_smem[2][4][64] = {};
  const int ti = ts == 1 ? 0 : ts == 2 ? 1 : ts == 4 ? 2 : 3;
  PG_REQUIRE(dev >= 0 && dev < 64, PG_ERR_PARAMETER, "device ordinal out of range");
  if (!occ[body][ti][dev] || occ_smem[body][ti][dev] != smem) {
    PG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)pattern_smem_bytes(256, kPatMaxEnt)));
    int nb = 0;
    PG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kChainThreads, smem));
    occ[body][ti][dev] = nb > 0 ? nb : 1;
    occ_smem[body][ti][dev] = smem;
  }
  const int (&occ_d)[4][64] = occ[body];
  const int per_sm = std::min(occ_d[ti][dev], std::max(1, env_int("PG_CHAIN_BLOCKS_PER_SM",
                                                                    occ_d[ti][dev])));
  int64_t grid = (int64_t)ws->num_sms * per_sm;
  // no more warps than chunks of one pass (the rest would only spin)
  const int64_t max_blocks = (nchunk + kChainThreads / 32 - 1) / (kChainThreads / 32);
  if (grid > max_blocks) grid = max_blocks;
  P.dynamic = env_int("PG_CHAIN_DYNAMIC", 0) != 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kChainThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (!P.dynamic) {
    // static tickets need every CTA resident at once: a cooperative launch
    // guarantees it (or fails)
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na].val.cooperative = 1;
    ++na;
  }
  if (pdl_enabled() && !g_capturing) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  PG_CUDA(cudaLaunchKernelEx(&cfg, kern, (const ChainParams)P));
  return true;
}

}  // namespace pg

using namespace pg;

extern "C" {

PG_API int pg_chain_fused(const pg_matrix* mat, int* fused) {
  return guard([&] {
    PG_REQUIRE(mat && fused, PG_ERR_PARAMETER, "null argument");
    *fused = chain_supported(mat) && !chain_deps(mat, (int64_t)4 * PG_SLICE).empty() ? 1 : 0;
  });
}

}  // extern "C"
