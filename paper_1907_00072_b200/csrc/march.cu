// Plane-marching SpMV for row-pattern stencil matrices.
//
// A constant-coefficient stencil on a structured grid in natural row order
// (config 4's 27-point operator, config 2's 7-point, the 2-D 9/5-point ones)
// is stored as a row-pattern dictionary whose master pattern is the interior
// row (abi.cu build_patterns).  Its master offsets decompose into three plane
// groups dz = -1, 0, +1 of a plane stride S (3-D: S = nx*ny, in-plane offsets
// dy*nx + dx; 2-D: S = nx, in-plane offsets dx).  A thread owns one in-plane
// index q and marches the rows r = z*S + q of a chunk of planes: the x
// values a row reads in plane z+1 are the ones the next row reads in plane z
// and the row after in plane z-1, so they stay in registers and every x value
// is loaded once per thread (27-point: 9 loads per row instead of 27; the
// windowed TMA kernel this replaces was bound by re-reading x from shared
// memory, 216 B per row).  Warps are 32 consecutive q, so every load, the
// pattern id and the epilogue operands are coalesced.
//
// Arithmetic is unchanged: each row sums its stored entries in column order
// (plane -1, plane 0, plane +1, in-plane ascending = the CSR order) with
// separately rounded products and sums, masked boundary rows add exactly
// their own entries, rows that are not master subsequences walk their pattern
// table -- bit-identical to every other SpMV kernel and to the reference
// (sparse.py:151-168, polyprec.py:205-211).

#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "sell.cuh"

namespace pg {

constexpr int kMarchThreads = 256;
#ifndef PG_MARCH_MIN_BLOCKS
#define PG_MARCH_MIN_BLOCKS 2
#endif
// rows of look-ahead of the x-plane and row-operand prefetch (1 or 2)
#ifndef PG_MARCH_DIST
#define PG_MARCH_DIST 1
#endif

struct MarchArgs {
  int64_t nrows, ncols, S, g, nz;
  int Z, nqb;
};

__device__ __forceinline__ double ld_x(const double* __restrict__ x, int64_t idx, int64_t ncols) {
  return (uint64_t)idx < (uint64_t)ncols ? __ldg(x + idx) : 0.0;
}

template <int MODE, int KIND>
__global__ void __launch_bounds__(kMarchThreads, PG_MARCH_MIN_BLOCKS)
    sell_march_kernel(MarchArgs ma, const uint8_t* __restrict__ rpat,
                      const int32_t* __restrict__ pptr, const PairEnt* __restrict__ pent,
                      int npat, int nent, const uint32_t* __restrict__ pmask, const PatMaster pm,
                      const double* __restrict__ x, Epi e, double* partials,
                      unsigned int* counter, double* nsq) {
  using Sh = MarchShape<KIND>;
  constexpr int NO = Sh::NO, NM = Sh::NM;
  constexpr int LEN = 2 * NO + NM;
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  extern __shared__ __align__(16) unsigned char smem_march[];
  const int32_t* s_ptr = stage_patterns(smem_march, pptr, pent, npat, nent, pmask);
  const uint32_t* s_mask = reinterpret_cast<const uint32_t*>(s_ptr + npat + 1);
  const PairEnt* s_ent = reinterpret_cast<const PairEnt*>(smem_march);
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  __syncthreads();

  const int qb = (int)(blockIdx.x % (unsigned)ma.nqb);
  const int64_t zc = blockIdx.x / (unsigned)ma.nqb;
  const int64_t S = ma.S, g = ma.g, ncols = ma.ncols, nrows = ma.nrows;
  const int64_t q = (int64_t)qb * kMarchThreads + threadIdx.x;
  const bool active = q < S;
  // loads use the clamped column (always in range); an inactive lane's rows
  // are never written
  const int64_t qq = active ? q : S - 1;
  const int64_t z0 = zc * ma.Z;
  const int64_t z1 = min(z0 + (int64_t)ma.Z, ma.nz);
  constexpr uint32_t kFull = (LEN >= 32) ? 0xffffffffu : ((1u << LEN) - 1u);
  double local = 0.0;

  int64_t row = z0 * S + q;
  bool live = active && row < nrows;
  int pid = live ? __ldg(rpat + row) : 0;
  Pre pre = live ? epi_load<MODE>(e, x, row) : Pre{0.0, 0.0};

  // one row: the sum in stored order from the three plane groups, epilogue.
  // Called by every lane every step (the warp vote needs them all).
  auto finish_row = [&](const double* Pm, const double* P0, const double* Pp, int rpid,
                        const Pre& rpre, int64_t r, bool rlive) {
    const uint32_t mask = rlive ? s_mask[rpid] : kFull;
    // a warp whose rows are all interior takes the unpredicated sum
    const bool warp_full = __all_sync(0xffffffffu, mask == kFull);
    if (!rlive) return;
    double acc = 0.0;
    if (warp_full) {
#pragma unroll
      for (int i = 0; i < NO; ++i) acc = __dadd_rn(acc, __dmul_rn(pm.v[i], Pm[i]));
#pragma unroll
      for (int i = 0; i < NM; ++i) acc = __dadd_rn(acc, __dmul_rn(pm.v[NO + i], P0[i]));
#pragma unroll
      for (int i = 0; i < NO; ++i) acc = __dadd_rn(acc, __dmul_rn(pm.v[NO + NM + i], Pp[i]));
    } else if (!(mask >> 31)) {
#pragma unroll
      for (int i = 0; i < NO; ++i)
        if (mask & (1u << i)) acc = __dadd_rn(acc, __dmul_rn(pm.v[i], Pm[i]));
#pragma unroll
      for (int i = 0; i < NM; ++i)
        if (mask & (1u << (NO + i))) acc = __dadd_rn(acc, __dmul_rn(pm.v[NO + i], P0[i]));
#pragma unroll
      for (int i = 0; i < NO; ++i)
        if (mask & (1u << (NO + NM + i)))
          acc = __dadd_rn(acc, __dmul_rn(pm.v[NO + NM + i], Pp[i]));
    } else {
      acc = row_sum_pattern<false>(s_ptr[rpid], s_ptr[rpid + 1], r, x, s_ent);
    }
    const double res = epilogue<MODE>(e, rpre, r, acc);
    if (MODE == kResid) local = __fma_rn(res, res, local);
  };
  // move to the next row of the column: its pattern id and epilogue operands
  // are requested a step ahead, before this row's arithmetic
  auto advance = [&](int64_t z) {
    row += S;
    live = active && z + 1 < z1 && row < nrows;
    pid = live ? __ldg(rpat + row) : 0;
    pre = live ? epi_load<MODE>(e, x, row) : Pre{0.0, 0.0};
  };
  // plane p's in-plane values: all of them (tensor stencils), or the middle
  // group of a cross stencil except its center.  CHECKED: planes next to the
  // ends of x (out-of-range entries read as 0 and are never added)
  auto load_set = [&](auto checked, int64_t p, double* P, bool skip_ctr) {
    constexpr bool CHECKED = decltype(checked)::value;
    if (!CHECKED) {
      const double* c = x + (p * S + qq);
      if (KIND == 27) {
#pragma unroll
        for (int dy = 0; dy < 3; ++dy) {
          const double* r = c + (dy - 1) * g;
          P[3 * dy] = __ldg(r - 1);
          P[3 * dy + 1] = __ldg(r);
          P[3 * dy + 2] = __ldg(r + 1);
        }
      } else if (KIND == 7) {
        P[0] = __ldg(c - g);
        P[1] = __ldg(c - 1);
        if (!skip_ctr) P[2] = __ldg(c);
        P[3] = __ldg(c + 1);
        P[4] = __ldg(c + g);
      } else {  // 9, 5: dx = -1, 0, 1
        P[0] = __ldg(c - 1);
        if (!skip_ctr) P[1] = __ldg(c);
        P[2] = __ldg(c + 1);
      }
    } else {
      const int64_t base = p * S + qq;
#pragma unroll
      for (int i = 0; i < NM; ++i)
        if (!(skip_ctr && i == Sh::CTR)) P[i] = ld_x(x, base + mid_off<KIND>(i, g), ncols);
    }
  };
  using Checked = std::true_type;
  using Unchecked = std::false_type;
  // steps z < zs prefetch a plane z+2 whose whole in-plane set lies inside x
  // (plane >= 1 always holds): (z + 3) S + g < ncols
  const int64_t zs = (ncols - g) / S - 3;
  const int64_t zb = min(z1 - 1, zs);  // unchecked prefetching steps: z < zb

  if constexpr (Sh::FULL) {
    // NS = 3 + DIST rotating plane sets: z-1, z, z+1 and the DIST planes
    // prefetched ahead; the rows' pattern ids and epilogue operands DIST rows
    // ahead as well.  The phase PH of a step selects the sets statically.
    constexpr int DIST = PG_MARCH_DIST;
    constexpr int NS = 3 + DIST;
    double X[NS][NM];
    int qpid[DIST + 1];
    Pre qpre[DIST + 1];
    bool qlive[DIST + 1];
#pragma unroll
    for (int k = 0; k <= DIST + 1; ++k) load_set(Checked{}, z0 - 1 + k, X[k], false);
    qpid[0] = pid;
    qpre[0] = pre;
    qlive[0] = live;
#pragma unroll
    for (int k = 1; k <= DIST; ++k) {
      advance(z0 + k - 1);
      qpid[k] = pid;
      qpre[k] = pre;
      qlive[k] = live;
    }
    // row of the step being computed
    int64_t rcur = z0 * S + q;
    auto step = [&](auto checked, auto phase, int64_t z) {
      constexpr int PH = decltype(phase)::value;
      double* Pn = X[(PH + 2 + DIST) % NS];
      if (!decltype(checked)::value)
        load_set(Unchecked{}, z + 1 + DIST, Pn, false);
      else if (z + DIST < z1)
        load_set(Checked{}, z + 1 + DIST, Pn, false);
      const int pid_c = qpid[0];
      const Pre pre_c = qpre[0];
      const bool live_c = qlive[0];
#pragma unroll
      for (int k = 0; k < DIST; ++k) {
        qpid[k] = qpid[k + 1];
        qpre[k] = qpre[k + 1];
        qlive[k] = qlive[k + 1];
      }
      advance(z + DIST);
      qpid[DIST] = pid;
      qpre[DIST] = pre;
      qlive[DIST] = live;
      finish_row(X[PH % NS], X[(PH + 1) % NS], X[(PH + 2) % NS], pid_c, pre_c, rcur, live_c);
      rcur += S;
    };
    using P0c = std::integral_constant<int, 0>;
    using P1c = std::integral_constant<int, 1>;
    using P2c = std::integral_constant<int, 2>;
    using P3c = std::integral_constant<int, 3>;
    using P4c = std::integral_constant<int, 4>;
    const int64_t zsd = (ncols - g) / S - 2 - DIST;
    const int64_t zbd = min(z1 - DIST, zsd);
    int64_t z = z0;
    for (; z + NS <= zbd; z += NS) {
      step(Unchecked{}, P0c{}, z);
      step(Unchecked{}, P1c{}, z + 1);
      step(Unchecked{}, P2c{}, z + 2);
      step(Unchecked{}, P3c{}, z + 3);
      if constexpr (NS > 4) step(Unchecked{}, P4c{}, z + 4);
    }
    while (z < z1) {
      step(Checked{}, P0c{}, z);
      if (++z >= z1) break;
      step(Checked{}, P1c{}, z);
      if (++z >= z1) break;
      step(Checked{}, P2c{}, z);
      if (++z >= z1) break;
      step(Checked{}, P3c{}, z);
      ++z;
      if constexpr (NS > 4) {
        if (z >= z1) break;
        step(Checked{}, P4c{}, z);
        ++z;
      }
    }
  } else {
    // cross stencils: centers of planes z-1, z, z+1 (+ z+2 prefetched) and
    // the middle group of plane z (its center slot = the plane-z center)
    constexpr int CTR = Sh::CTR;
    double cm, c0, cp, cn = 0.0;
    double MA[NM], MB[NM];
    auto ctr = [&](int64_t p) {
      const int64_t idx = p * S + qq;
      return (uint64_t)idx < (uint64_t)ncols ? __ldg(x + idx) : 0.0;
    };
    cm = ctr(z0 - 1);
    c0 = ctr(z0);
    cp = ctr(z0 + 1);
    load_set(Checked{}, z0, MA, true);
    auto step = [&](auto checked, int64_t z, double* M0, double* Mn) {
      if (!decltype(checked)::value) {
        cn = __ldg(x + ((z + 2) * S + qq));
        load_set(Unchecked{}, z + 1, Mn, true);
      } else if (z + 1 < z1) {
        cn = ctr(z + 2);
        load_set(Checked{}, z + 1, Mn, true);
      }
      const int pid_c = pid;
      const Pre pre_c = pre;
      const int64_t row_c = row;
      const bool live_c = live;
      advance(z);
      M0[CTR] = c0;
      finish_row(&cm, M0, &cp, pid_c, pre_c, row_c, live_c);
      cm = c0;
      c0 = cp;
      cp = cn;
    };
    int64_t z = z0;
    for (; z + 2 <= zb; z += 2) {
      step(Unchecked{}, z, MA, MB);
      step(Unchecked{}, z + 1, MB, MA);
    }
    while (z < z1) {
      step(Checked{}, z, MA, MB);
      if (++z >= z1) break;
      step(Checked{}, z, MB, MA);
      ++z;
    }
  }

  if (MODE == kResid) {
    const double s = block_sum(local);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
    last_block_reduce(partials, counter, 1, nsq);
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static int march_env(const char* name, int dflt) {
  const char* s = std::getenv(name);
  return s ? std::atoi(s) : dflt;
}

// Decide whether the matrix's master pattern is a plane-marching stencil;
// fills kind, S, g.  The master offsets are in stored (ascending) order.
bool stencil_shape(const pg_matrix* m, int* kind, int64_t* S, int64_t* g) {
  if (!m->rpat || m->perm || m->pat_mlen <= 0) return false;
  const int L = m->pat_mlen;
  const int32_t* o = m->pat_mdoff;
  std::vector<int64_t> want;
  int64_t s = 0, gg = 0;
  if (L == 27) {
    gg = (int64_t)o[16] - o[13];
    s = (int64_t)o[22] - o[13];
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) want.push_back(dz * s + dy * gg + dx);
  } else if (L == 7) {
    s = o[6];
    gg = o[5];
    want = {-s, -gg, -1, 0, 1, gg, s};
  } else if (L == 9) {
    s = gg = (int64_t)o[7] - o[4];
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) want.push_back(dy * s + dx);
  } else if (L == 5) {
    s = gg = o[4];
    want = {-s, -1, 0, 1, s};
  } else {
    return false;
  }
  // tensor offsets strictly ordered
  if (s <= 2 || ((L == 27 || L == 7) && (gg <= 2 || s <= 2 * gg + 2))) return false;
  for (int i = 0; i < L; ++i)
    if (want[i] != o[i]) return false;
  *kind = L;
  *S = s;
  *g = gg;
  return true;
}

bool march_shape(const pg_matrix* m, int* kind, int64_t* S, int64_t* g) {
  static int on = -1, min_s = -1;
  // opt-in: measured slower than the windowed kernel on cfg4 (111 vs 76 us
  // per pass) and the pattern kernel on cfg2 (9.8 vs 9.3 us), DESIGN.md §3
  if (on < 0) on = march_env("PG_SPMV_MARCH", 0);
  // enough in-plane indices to fill whole warps (PG_MARCH_MIN_S, default 512)
  if (min_s < 0) min_s = march_env("PG_MARCH_MIN_S", 512);
  return on && stencil_shape(m, kind, S, g) && *S >= min_s;
}

template <int MODE>
bool march_launch(const pg_matrix* m, const double* x, Epi e, pg_workspace* ws, double* nsq,
                  cudaStream_t st) {
  int kind;
  int64_t S, g;
  if (!march_shape(m, &kind, &S, &g)) return false;
  MarchArgs ma;
  ma.nrows = m->nrows;
  ma.ncols = m->ncols;
  ma.S = S;
  ma.g = g;
  ma.nz = (m->nrows + S - 1) / S;
  ma.nqb = (int)((S + kMarchThreads - 1) / kMarchThreads);
  static int zenv = -1;
  if (zenv < 0) zenv = march_env("PG_MARCH_Z", 0);
  int Z = zenv;
  if (Z <= 0) {
    // about 4 resident waves of 2 blocks per SM, chunks of >= 16 planes
    const int64_t target = 148 * 2 * 4;
    const int64_t chunks = (target + ma.nqb - 1) / ma.nqb;
    Z = (int)((ma.nz + chunks - 1) / chunks);
    if (Z < 16) Z = 16;
  }
  ma.Z = Z;
  const int64_t nzc = (ma.nz + Z - 1) / Z;
  const int64_t blocks = nzc * ma.nqb;
  if (blocks <= 0) return false;
  if (MODE == kResid && blocks > kMaxBlocks) return false;  // partial slots
  if (blocks >= (int64_t)1 << 31) return false;
  PatMaster pm;
  std::memset(&pm, 0, sizeof pm);
  pm.len = m->pat_mlen;
  for (int i = 0; i < pm.len; ++i) pm.v[i] = m->pat_mv[i];
  const size_t smem = pattern_smem_bytes(m->n_pat, m->pat_nent);
  auto kern = kind == 27 ? sell_march_kernel<MODE, 27>
            : kind == 7  ? sell_march_kernel<MODE, 7>
            : kind == 9  ? sell_march_kernel<MODE, 9>
                         : sell_march_kernel<MODE, 5>;
  static bool attr[4][4][64] = {};
  const int ki = kind == 27 ? 0 : kind == 7 ? 1 : kind == 9 ? 2 : 3;
  const int dev = m->device;
  if (!attr[MODE][ki][dev]) {
    PG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)pattern_smem_bytes(256, kPatMaxEnt)));
    attr[MODE][ki][dev] = true;
  }
  launch_k(kern, (int)blocks, kMarchThreads, smem, st, ma, (const uint8_t*)m->rpat,
           (const int32_t*)m->pat_ptr, (const PairEnt*)m->pat_ent, m->n_pat, m->pat_nent,
           (const uint32_t*)m->pat_mask, pm, x, e, ws ? ws->partials : nullptr,
           ws ? ws->counter : nullptr, nsq);
  check_launch();
  return true;
}

template bool march_launch<kSpmv>(const pg_matrix*, const double*, Epi, pg_workspace*, double*,
                                  cudaStream_t);
template bool march_launch<kPoly>(const pg_matrix*, const double*, Epi, pg_workspace*, double*,
                                  cudaStream_t);
template bool march_launch<kResid>(const pg_matrix*, const double*, Epi, pg_workspace*, double*,
                                   cudaStream_t);
template bool march_launch<kRoot>(const pg_matrix*, const double*, Epi, pg_workspace*, double*,
                                  cudaStream_t);

}  // namespace pg
