// Plane-ring SpMV for row-pattern plane stencils.
//
// The matrix is a constant-coefficient stencil in natural row order whose
// master pattern (abi.cu build_patterns) splits into three plane groups
// dz = -1, 0, +1 of a plane stride S (stencil_shape, march.cu): config 4's
// 27-point operator, config 2's 7-point one, the 2-D 9/5-point ones (a
// "plane" is then a grid line).  A block owns a tile of Q consecutive
// in-plane indices and marches it through a chunk of planes.  One producer
// lane streams, per plane p, the tile's x window (Q + 2H doubles, H the
// in-plane halo), the pattern ids of the rows of plane p+1 and the epilogue
// operands of the rows of plane p-1 into a shared-memory ring with
// cp.async.bulk (TMA) completing on mbarriers.  The row threads read each
// window value ONCE per plane (9 shared loads per 27-point row instead of
// 27) and use it three times: plane p closes the sums of the rows of plane
// p-1 (their dz = +1 group), continues those of plane p (dz = 0) and opens
// those of plane p+1 (dz = -1).  Three running sums per in-plane index stay
// in registers.
//
// Arithmetic is unchanged.  A row's stored entries are its dz = -1 group,
// then dz = 0, then dz = +1, each in ascending in-plane order (the CSR
// column order), and the row's sum receives them in exactly that sequence,
// one separately rounded product and sum per entry, starting from 0.0: the
// same operations in the same order as the row-sequential kernels and the
// reference (sparse.py:151-168); the fused epilogue is the shared one
// (polyprec.py:205-211).  Boundary rows (master subsequences) add only their
// own entries; rows that are not master subsequences are summed from their
// pattern table with global gathers when they close.

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "pipeline.cuh"
#include "sell.cuh"

namespace pg {

#ifndef PG_PLANE_ROW_THREADS
#define PG_PLANE_ROW_THREADS 288
#endif
#ifndef PG_PLANE_RPT
#define PG_PLANE_RPT 2
#endif
constexpr int kPlaneRowThreads = PG_PLANE_ROW_THREADS;  // row warps x 32
constexpr int kPlaneThreads = kPlaneRowThreads + 32;  // + the producer warp
// in-plane indices per row thread: t, t + kPlaneRowThreads, ... (the pair
// kernels, ADJ: 2t, 2t + 1)
constexpr int kPlaneRPT = PG_PLANE_RPT;
static_assert(kPlaneRPT % 2 == 0, "the steady path works on pairs of in-plane indices");
constexpr int kPlaneMaxQ = kPlaneRowThreads * kPlaneRPT;
constexpr int kPlaneMaxStages = 8;
// unroll of the interior-plane loop (3 = the rows' role rotation period)
#ifndef PG_PLANE_UNROLL
#define PG_PLANE_UNROLL 1
#endif
constexpr int kPlaneUnroll = PG_PLANE_UNROLL;
// timing experiments only (tools/build_variant.sh): 1 = no x-window copies,
// 2 = no operand copies, 4 = row threads skip the arithmetic and stores,
// 8 = no stores (a never-true test keeps the arithmetic), 16 = every warp
// takes the interior path (wrong results at boundary rows), 32 = no zeroing
// of absent in-plane entries on interior planes (wrong at boundary rows)
#ifndef PG_PLANE_EXP
#define PG_PLANE_EXP 0
#endif
// L2 eviction hints of the pair kernels (bits: 1 = x windows evict_last,
// 2 = operand copies evict_first, 4 = w_out stores evict_last, 8 = acc_out
// stores evict_first, 16 = acc_out stores evict_last, 32 = the kSpmv result
// evict_last): the next pass of a chain reads this pass's w_out.
// Measured (cfg4 middle pass, 48.8 us without hints): 4 alone 47.3; 5 47.3;
// 12, 15, 20, 21 (any hint on acc_out) 48.4-48.9.
#ifndef PG_PLANE_L2HINT
#define PG_PLANE_L2HINT 4
#endif
#ifndef PG_PLANE_MIN_BLOCKS
#define PG_PLANE_MIN_BLOCKS 2
#endif

// dynamic shared memory per block (ring), leaving room for PG_PLANE_MIN_BLOCKS
constexpr int kPlaneSmemBudget = 200 * 1024 / PG_PLANE_MIN_BLOCKS;


// Window position of middle-group value i relative to the row's slot, with
// the stencil's consecutive runs made explicit (one runtime base per run,
// the rest immediate offsets)
template <int KIND>
__device__ __forceinline__ int win_off(int i, const PlaneArgs& pa) {
  if (KIND == 27) return pa.woff[3 * (i / 3)] + i % 3;
  if (KIND == 7) return i == 0 ? pa.woff[0] : (i == 4 ? pa.woff[4] : pa.woff[1] + (i - 1));
  return pa.woff[0] + i;  // 9, 5: dx = -1, 0, 1
}

// The row epilogue; EF >= 0 (kPoly only): the pass flags (PG_PASS_FIRST,
// PG_PASS_WRITE_W) and base presence (4) as compile-time constants -- the
// same operations in the same order as sell.cuh epilogue<kPoly>.
template <int MODE, int EF>
__device__ __forceinline__ double plane_epilogue(const Epi& e, const Pre& p, int64_t row,
                                                 double ax) {
  if (MODE != kPoly || EF < 0) return epilogue<MODE>(e, p, row, ax);
  double t = (EF & PG_PASS_FIRST) ? __dmul_rn(e.y0, p.a) : p.a;
  t = __dadd_rn(t, __dmul_rn(e.yk, ax));
  if (EF & PG_PASS_WRITE_W) e.w_out[row] = ax;
  if (EF & 4) t = __dadd_rn(p.b, t);
  e.acc_out[row] = t;
  return 0.0;
}

// The same positions as runs: NR runs of consecutive window values, value i
// at run run_of(i), position run_pos(i); run r starts at pa.woff[run_base(r)]
template <int KIND>
struct WinRuns {
  static constexpr int NR = (KIND == 27 || KIND == 7) ? 3 : 1;
  __device__ static constexpr int run_of(int i) {
    return KIND == 27 ? i / 3 : KIND == 7 ? (i == 0 ? 0 : i == 4 ? 2 : 1) : 0;
  }
  __device__ static constexpr int run_pos(int i) {
    return KIND == 27 ? i % 3 : KIND == 7 ? (i == 0 || i == 4 ? 0 : i - 1) : i;
  }
  __device__ static constexpr int run_len(int r) {
    return KIND == 27 ? 3 : KIND == 7 ? (r == 1 ? 3 : 1) : 3;
  }
  __device__ static constexpr int run_base(int r) {
    return KIND == 27 ? 3 * r : KIND == 7 ? (r == 0 ? 0 : r == 1 ? 1 : 4) : 0;
  }
};

// SYM (tensor stencils): outer-group coefficients equal bit for bit, dz = -1
// vs dz = +1 at the same in-plane offset, for every offset (2) or every one
// but the center (1: the plane-normal convection term sits on the center
// pair only).  The two rows that use a window value with those coefficients
// then receive the same rounded product, computed once.
// ADJ (27-point tiles with PlaneArgs::vec): a row thread's two in-plane
// indices are adjacent (2t, 2t+1) instead of t, t + kPlaneRowThreads: the two
// rows share 2 of the 3 window values of every run (4 shared loads per run,
// one of them 16 bytes, instead of 6), and their epilogue operands and
// results move as aligned 16-byte pairs.
template <int MODE, int KIND, int EF, int SYM = 0, bool ADJ = false>
__global__ void __launch_bounds__(kPlaneThreads, PG_PLANE_MIN_BLOCKS)
    plane_ring_kernel(PlaneArgs pa, const uint8_t* __restrict__ rpat,
                      const int32_t* __restrict__ pptr, const PairEnt* __restrict__ pent,
                      int npat, const uint32_t* __restrict__ pmask, const PatMaster pm,
                      const double* __restrict__ x, Epi e, double* partials,
                      unsigned int* counter, double* nsq,
                      const uint16_t* __restrict__ plane_qm) {
  using Sh = MarchShape<KIND>;
  static_assert(!ADJ || (KIND == 27 && kPlaneRPT == 2), "pair path: 27-point, two rows per thread");
  constexpr bool kPlaneAdj = ADJ;
  constexpr int NO = Sh::NO, NM = Sh::NM, LEN = 2 * NO + NM;
  constexpr uint32_t kFull = (1u << LEN) - 1u;
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  extern __shared__ __align__(128) unsigned char smem_plane[];
  __shared__ uint32_t s_mask[256];
  // a stage's full / empty mbarriers sit inside the stage (pa.off_bar), so
  // the row threads track the ring with one pointer and a phase bit
  __shared__ int tag[kPlaneMaxStages];  // PG_CHECKS: the plane a slot holds
  auto full_of = [&](const unsigned char* stage) {
    return reinterpret_cast<uint64_t*>(const_cast<unsigned char*>(stage) + pa.off_bar);
  };
  auto empty_of = [&](const unsigned char* stage) { return full_of(stage) + 1; };
  // the masks never change after matrix creation: staged before the wait
  // (a pattern that is not a master subsequence: bit 31 + its id)
  for (int i = threadIdx.x; i < npat; i += blockDim.x) {
    const uint32_t mk = pmask[i];
    s_mask[i] = (mk >> 31) ? (0x80000000u | (uint32_t)i) : mk;
  }
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  const int NS = pa.stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full_of(smem_plane + (size_t)s * pa.stage_bytes), 1);
      mbar_init(empty_of(smem_plane + (size_t)s * pa.stage_bytes), kPlaneRowThreads / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();

  const int qb = (int)(blockIdx.x % (unsigned)pa.nqb);
  const int64_t za = (int64_t)(blockIdx.x / (unsigned)pa.nqb) * pa.Zc;
  const int64_t zb = min(za + (int64_t)pa.Zc, pa.nz);
  const int64_t S = pa.S;
  const int64_t q0 = (int64_t)qb * pa.Q;
  const int Qt = (int)min((int64_t)pa.Q, S - q0);
  // stages: planes za - 1 .. zb
  const int nstage = (int)(zb - za) + 2;
  double local = 0.0;
  const int warp = threadIdx.x >> 5;
  // The steady planes of the chunk whose three rows are all on interior
  // planes of a host-verified matrix, [box_lo, box_hi]: no pattern ids are
  // staged for them, the row threads run them as a counted loop.  Only with
  // at least two such planes (the rows closing and continuing after the
  // loop were then both opened inside it); allbox: the end planes too.
  int box_lo = (int)zb + 1, box_hi = (int)zb;
  if (plane_qm && !(PG_PLANE_EXP & 4)) {
    const int lo = pa.allbox ? (int)za + 1 : max((int)za + 1, 2);
    const int hi = pa.allbox ? (int)zb - 2 : min((int)zb - 2, (int)pa.nz - 3);
    if (hi >= lo + 1) {
      box_lo = lo;
      box_hi = hi;
    }
  }

  if (warp == kPlaneRowThreads / 32) {
    if ((threadIdx.x & 31) == 0) {
      const double *A, *B;
      epi_vectors<MODE>(e, x, A, B);
      // window doubles per plane: Qt + 2H + sh rounded up to even
      const int wl = (Qt + 2 * pa.H + pa.sh + 1) & ~1;
      int st = 0, round = 0;
      for (int k = 0; k < nstage; ++k) {
        unsigned char* buf = smem_plane + (size_t)st * pa.stage_bytes;
        uint64_t* const full_st = full_of(buf);
        if (round > 0) mbar_wait(empty_of(buf), (uint32_t)((round - 1) & 1));
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        double* win = reinterpret_cast<double*>(buf);
        const int64_t p = za - 1 + k;
        // window of plane p: [p S + q0 - H - sh, p S + q0 + Qt + H + 1), both
        // ends even (16-byte aligned bulk copies), clipped to [0, ncols): any
        // part of it may lie in another plane or the ghost slots; entries a
        // row does not store are never added.  Only a window clipped at an
        // odd ncols has a tail element, copied plainly.
        const int64_t ga = p * S + q0 - pa.H - pa.sh;
        int64_t ca = max(ga, (int64_t)0);
        const int64_t ce = min(ga + wl, pa.ncols);
        const int64_t n = ce > ca ? ce - ca : 0;
        if (n & 1) win[ca - ga + n - 1] = __ldg(x + ca + n - 1);
        ca -= ga;  // now the window position of the first copied element
        PG_DCHECK(n == 0 || (ca >= 0 && ca + n <= (int64_t)pa.Q + 2 * pa.H + 2));
        if (PG_CHECKS) tag[st] = (int)p;
        const bool start = p + 1 < zb;     // rows of plane p + 1 open
        const bool close = p - 1 >= za;    // rows of plane p - 1 close
        // interior "box" stages read no pattern ids (plane_qm, see the row threads)
        const bool boxed = p >= box_lo && p <= box_hi;
        const bool ids = start && !boxed && !pa.allbox;
        uint32_t bytes = 8u * (uint32_t)(n & ~(int64_t)1);
        if (ids) bytes += (uint32_t)Qt;
        if (close && A) bytes += 8u * (uint32_t)Qt;
        if (close && B) bytes += 8u * (uint32_t)Qt;
        if (PG_PLANE_EXP & 1) bytes -= 8u * (uint32_t)(n & ~(int64_t)1);
        if (PG_PLANE_EXP & 2) bytes -= ((close && A) + (close && B)) * 8u * (uint32_t)Qt;
        mbar_expect_tx(full_st, bytes);
        if (n > 1 && !(PG_PLANE_EXP & 1)) {
          if (ADJ && (PG_PLANE_L2HINT & 1))
            bulk_g2s_hint(win + ca, x + ga + ca, 8u * (uint32_t)(n & ~(int64_t)1), full_st,
                          l2_policy_evict_last());
          else
            bulk_g2s(win + ca, x + ga + ca, 8u * (uint32_t)(n & ~(int64_t)1), full_st);
        }
        if (ids) bulk_g2s(buf + pa.off_p, rpat + (p + 1) * S + q0, (uint32_t)Qt, full_st);
        if (close && A && !(PG_PLANE_EXP & 2)) {
          if (ADJ && (PG_PLANE_L2HINT & 2))
            bulk_g2s_hint(buf + pa.off_a, A + (p - 1) * S + q0, 8u * (uint32_t)Qt, full_st,
                          l2_policy_evict_first());
          else
            bulk_g2s(buf + pa.off_a, A + (p - 1) * S + q0, 8u * (uint32_t)Qt, full_st);
        }
        if (close && B && !(PG_PLANE_EXP & 2))
          bulk_g2s(buf + pa.off_b, B + (p - 1) * S + q0, 8u * (uint32_t)Qt, full_st);
        if (++st == NS) {
          st = 0;
          ++round;
        }
      }
    }
  } else {
    const int t = threadIdx.x;
    const double *A, *B;
    epi_vectors<MODE>(e, x, A, B);
    // Per in-plane index h, the rows closing (f) and continuing (m) at the
    // current plane: running sums and pattern masks (a pattern that is not a
    // master subsequence carries bit 31 and its id in the low bits).
    double acc_f[kPlaneRPT], acc_m[kPlaneRPT];
    uint32_t mk_f[kPlaneRPT], mk_m[kPlaneRPT];
    // "box" in-plane masks of those rows (see steady): the row's in-plane
    // entries when all three plane groups hold exactly them, else kNoBox
    uint32_t bq_f[kPlaneRPT], bq_m[kPlaneRPT];
    // local in-plane indices of this thread (an inactive index reads slot 0:
    // in range, never used)
    int jj[kPlaneRPT];
    bool act[kPlaneRPT];
#pragma unroll
    for (int h = 0; h < kPlaneRPT; ++h) {
      const int j = kPlaneAdj ? t * kPlaneRPT + h : t + h * kPlaneRowThreads;
      act[h] = j < Qt;
      // (adjacent indices keep their distance: the slots of an inactive pair
      // are in range of the stage, never used)
      jj[h] = act[h] ? j : (kPlaneAdj ? h : 0);
      acc_f[h] = acc_m[h] = 0.0;
      mk_f[h] = mk_m[h] = kFull;
    }
    constexpr uint32_t kMid = (1u << NM) - 1u, kNoBox = 0xffffffffu;
#pragma unroll
    for (int h = 0; h < kPlaneRPT; ++h) bq_f[h] = bq_m[h] = kMid;
    // the in-plane mask of a "box" row (all three plane groups present, each
    // holding the same in-plane entries), else kNoBox
    auto boxq = [](uint32_t mk) -> uint32_t {
      const uint32_t qm = (mk >> NO) & kMid;
      const uint32_t b = Sh::FULL ? (qm | (qm << NO) | (qm << (NO + NM)))
                                  : (1u | (qm << NO) | (1u << (NO + NM)));
      return mk == b ? qm : kNoBox;
    };
    // ring position: the current stage's byte offset and phase bit
    uint32_t phase = 0, boff = 0;
    const uint32_t ring_bytes = (uint32_t)NS * (uint32_t)pa.stage_bytes;
#define PG_BUF (smem_plane + boff)
    auto next_slot = [&]() {
      __syncwarp();
      if ((t & 31) == 0) mbar_arrive(empty_of(PG_BUF));
      boff += (uint32_t)pa.stage_bytes;
      if (boff == ring_bytes) {
        phase ^= 1u;
        boff = 0;
      }
    };
    // full-barrier wait of the current stage (PG_CHECKS: it holds plane p)
    auto wait_stage = [&](int p) {
      mbar_wait(full_of(PG_BUF), phase);
      PG_DCHECK(tag[boff / pa.stage_bytes] == p);
      (void)p;
    };
    // masks of the rows opening at plane p (their pattern ids are staged)
    auto open_masks = [&](uint32_t (&mk_s)[kPlaneRPT], bool start) {
#pragma unroll
      for (int h = 0; h < kPlaneRPT; ++h)
        mk_s[h] = (start && act[h]) ? s_mask[PG_BUF[pa.off_p + jj[h]]] : kFull;
    };
    auto rotate = [&](const double (&acc_s)[kPlaneRPT], const uint32_t (&mk_s)[kPlaneRPT],
                      const uint32_t (&bq_s)[kPlaneRPT]) {
#pragma unroll
      for (int h = 0; h < kPlaneRPT; ++h) {
        acc_f[h] = acc_m[h];
        mk_f[h] = mk_m[h];
        bq_f[h] = bq_m[h];
        acc_m[h] = acc_s[h];
        mk_m[h] = mk_s[h];
        bq_m[h] = bq_s[h];
      }
    };
    auto finish = [&](int h, int64_t row, double acc) {
      Pre pre{0.0, 0.0};
      if (EF >= 0 ? true : A != nullptr) pre.a = reinterpret_cast<const double*>(PG_BUF + pa.off_a)[jj[h]];
      if (EF >= 0 ? (EF & 4) != 0 : B != nullptr)
        pre.b = reinterpret_cast<const double*>(PG_BUF + pa.off_b)[jj[h]];
      if (!(PG_PLANE_EXP & 8) || acc == 1.2345e300) {
        const double r = plane_epilogue<MODE, EF>(e, pre, row, acc);
        if (MODE == kResid) local = __fma_rn(r, r, local);
      }
    };
    // The pair (h0, h0 + 1) of an aligned tile (pa.vec): operands read and
    // results written as 16-byte pairs; each row's operations as in
    // plane_epilogue<MODE, EF>.
    constexpr bool kPairEpi = kPlaneAdj && ((MODE == kPoly && EF >= 0) || MODE == kSpmv);
    const uint64_t pol_w = (PG_PLANE_L2HINT & 36) ? l2_policy_evict_last() : 0;
    const uint64_t pol_a = (PG_PLANE_L2HINT & 8)    ? l2_policy_evict_first()
                           : (PG_PLANE_L2HINT & 16) ? l2_policy_evict_last()
                                                    : 0;
    auto finish2 = [&](int h0, int64_t row, double ax0, double ax1) {
      if constexpr (kPairEpi && MODE == kSpmv) {
        if (!(PG_PLANE_EXP & 8) || ax0 == 1.2345e300) {
          if (PG_PLANE_L2HINT & 32) st_v2_hint(e.acc_out + row, ax0, ax1, pol_w);
          else *reinterpret_cast<double2*>(e.acc_out + row) = make_double2(ax0, ax1);
        }
      } else if constexpr (kPairEpi) {
        const double2 a2 = *reinterpret_cast<const double2*>(PG_BUF + pa.off_a + 8 * jj[h0]);
        double t0 = (EF & PG_PASS_FIRST) ? __dmul_rn(e.y0, a2.x) : a2.x;
        double t1 = (EF & PG_PASS_FIRST) ? __dmul_rn(e.y0, a2.y) : a2.y;
        t0 = __dadd_rn(t0, __dmul_rn(e.yk, ax0));
        t1 = __dadd_rn(t1, __dmul_rn(e.yk, ax1));
        if (EF & 4) {
          const double2 b2 = *reinterpret_cast<const double2*>(PG_BUF + pa.off_b + 8 * jj[h0]);
          t0 = __dadd_rn(b2.x, t0);
          t1 = __dadd_rn(b2.y, t1);
        }
        if (!(PG_PLANE_EXP & 8) || ax0 == 1.2345e300) {
          if (EF & PG_PASS_WRITE_W) {
            if (PG_PLANE_L2HINT & 4) st_v2_hint(e.w_out + row, ax0, ax1, pol_w);
            else *reinterpret_cast<double2*>(e.w_out + row) = make_double2(ax0, ax1);
          }
          if (PG_PLANE_L2HINT & 24) st_v2_hint(e.acc_out + row, t0, t1, pol_a);
          else *reinterpret_cast<double2*>(e.acc_out + row) = make_double2(t0, t1);
        }
      }
    };
    // Any stage: per-lane masked adds; rows that are not master
    // subsequences are summed from their pattern table when they close.
    auto general = [&](int p, bool close, bool mid, bool start,
                       const uint32_t (&mk_s)[kPlaneRPT]) {
      const double* win = reinterpret_cast<const double*>(PG_BUF);
      double acc_s[kPlaneRPT];
#pragma unroll
      for (int h = 0; h < kPlaneRPT; ++h) {
        const int j = jj[h];
        double P[NM];
#pragma unroll
        for (int i = 0; i < NM; ++i) P[i] = win[j + win_off<KIND>(i, pa)];
        // outer-group value i (dz = -1 or +1): the same in-plane offsets as
        // the middle group (tensor stencils) or the center (cross stencils)
        auto outer = [&](int i) { return Sh::FULL ? P[i] : P[Sh::CTR]; };
        acc_s[h] = 0.0;
        if (close && act[h]) {  // rows of plane p - 1: dz = +1 group, then the epilogue
          const int64_t row = (int64_t)(p - 1) * S + q0 + j;
          double acc = acc_f[h];
          const uint32_t mk = mk_f[h];
          if (mk >> 31) {
            const int pid = (int)(mk & 255u);
            acc = row_sum_pattern<false>(__ldg(pptr + pid), __ldg(pptr + pid + 1), row, x, pent);
          } else {
#pragma unroll
            for (int i = 0; i < NO; ++i)
              if (mk & (1u << (NO + NM + i)))
                acc = __dadd_rn(acc, __dmul_rn(pm.v[NO + NM + i], outer(i)));
          }
          finish(h, row, acc);
        }
        if (mid && act[h]) {  // rows of plane p: dz = 0 group
          double acc = acc_m[h];
#pragma unroll
          for (int i = 0; i < NM; ++i)
            if (mk_m[h] & (1u << (NO + i))) acc = __dadd_rn(acc, __dmul_rn(pm.v[NO + i], P[i]));
          acc_m[h] = acc;
        }
        if (start && act[h]) {  // rows of plane p + 1: dz = -1 group
          double acc = 0.0;
#pragma unroll
          for (int i = 0; i < NO; ++i)
            if (mk_s[h] & (1u << i)) acc = __dadd_rn(acc, __dmul_rn(pm.v[i], outer(i)));
          acc_s[h] = acc;
        }
      }
      uint32_t bq_s[kPlaneRPT];
#pragma unroll
      for (int h = 0; h < kPlaneRPT; ++h) bq_s[h] = boxq(mk_s[h]);
      rotate(acc_s, mk_s, bq_s);
    };
    // Steady stage (rows close, continue and open): the unrolled path when,
    // for every row of the warp, the closing, continuing and opening rows at
    // its in-plane index are the same "box" row -- all three plane groups
    // present, each holding the in-plane entries qm (interior rows: all of
    // them).  Window values outside qm are zeroed: a product with +-0.0 added
    // to a running sum leaves it unchanged (the sum starts at +0.0 and a
    // round-to-nearest sum is never -0.0), so each row still receives
    // exactly its own entries, in order.  Other warps take the general path.
    // the unrolled interior body: every row of the warp at this stage is a
    // box row with in-plane entries bq_m (closing, continuing and opening
    // rows alike); zero: some lane's rows miss in-plane entries
    // byte offsets of this thread's window runs inside a ring stage
    using Runs = WinRuns<KIND>;
    uint32_t wrun[kPlaneRPT][Runs::NR];
#pragma unroll
    for (int h = 0; h < kPlaneRPT; ++h)
#pragma unroll
      for (int r = 0; r < Runs::NR; ++r) {
        wrun[h][r] = 8u * (uint32_t)(jj[h] + pa.woff[Runs::run_base(r)]);
        PG_DCHECK(jj[h] + pa.woff[Runs::run_base(r)] >= 0 &&
                  wrun[h][r] + 8u * Runs::run_len(r) <=
                      8u * (uint32_t)(pa.Q + 2 * pa.H + 2));
      }
    // The window values of the in-plane index pair (h0, h0 + 1).  Adjacent
    // indices: a run of L consecutive values per row is L + 1 distinct values
    // for the pair; the run starts at an odd window position (pa.vec), so
    // the two middle values of a 3-run are one aligned 16-byte load.
    auto load_pair = [&](double (&P)[2][NM], int h0) {
      if constexpr (kPlaneAdj) {
#pragma unroll
        for (int r = 0; r < Runs::NR; ++r) {
          constexpr int kMaxL = 3, L = 3;  // (ADJ: 27-point, three 3-runs)
          const unsigned char* a = PG_BUF + wrun[h0][r];
          double W[kMaxL + 1];
          W[0] = *reinterpret_cast<const double*>(a);
          const double2 m = *reinterpret_cast<const double2*>(a + 8);
          W[1] = m.x;
          W[2] = m.y;
          W[3] = *reinterpret_cast<const double*>(a + 24);
#pragma unroll
          for (int c = 0; c < kMaxL; ++c)
            if (c < L) {
              P[0][Runs::run_base(r) + c] = W[c];
              P[1][Runs::run_base(r) + c] = W[c + 1];
            }
        }
      } else {
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int i = 0; i < NM; ++i)
            P[u][i] = reinterpret_cast<const double*>(PG_BUF + wrun[h0 + u][Runs::run_of(i)])
                [Runs::run_pos(i)];
      }
    };
    // ri: the (32-bit) row of in-plane index 0 of the tile on the closing
    // plane p - 1; ROT: also rotate the rows' masks (the interior-plane loop
    // keeps them fixed and sets them once after the loop)
    auto body = [&](int ri, const uint32_t (&mk_s)[kPlaneRPT], const uint32_t (&bq_s)[kPlaneRPT],
                    auto zero_c, auto rot_c) {
      constexpr bool zero = decltype(zero_c)::value;
      double acc_s[kPlaneRPT];
      // pairs of in-plane indices: six independent chains each (close /
      // continue / open x 2), every chain in its row's stored order
#pragma unroll
      for (int h0 = 0; h0 < kPlaneRPT; h0 += 2) {
        double P[2][NM];
        load_pair(P, h0);
        if constexpr (zero) {
#pragma unroll
          for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int i = 0; i < NM; ++i)
              if (!((bq_s[h0 + u] >> i) & 1u)) P[u][i] = 0.0;
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) acc_s[h0 + u] = 0.0;
#pragma unroll
        for (int i = 0; i < NM; ++i) {
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int h = h0 + u;
            if (i < NO) {
              const double o = Sh::FULL ? P[u][i] : P[u][Sh::CTR];
              const double pf = __dmul_rn(pm.v[NO + NM + i], o);
              const bool same = Sh::FULL && (SYM == 2 || (SYM == 1 && i != Sh::CTR));
              const double ps = same ? pf : __dmul_rn(pm.v[i], o);
              acc_f[h] = __dadd_rn(acc_f[h], pf);
              acc_s[h] = __dadd_rn(acc_s[h], ps);
            }
            acc_m[h] = __dadd_rn(acc_m[h], __dmul_rn(pm.v[NO + i], P[u][i]));
          }
        }
        if (kPairEpi) {
          if (act[h0]) finish2(h0, (int64_t)(ri + jj[h0]), acc_f[h0], acc_f[h0 + 1]);
        } else {
#pragma unroll
          for (int u = 0; u < 2; ++u)
            if (act[h0 + u]) finish(h0 + u, (int64_t)(ri + jj[h0 + u]), acc_f[h0 + u]);
        }
      }
      if constexpr (decltype(rot_c)::value) {
        rotate(acc_s, mk_s, bq_s);
      } else {
#pragma unroll
        for (int h = 0; h < kPlaneRPT; ++h) {
          acc_f[h] = acc_m[h];
          acc_m[h] = acc_s[h];
        }
      }
    };
    // Steady stage (rows close, continue and open): the unrolled body when,
    // for every row of the warp, the closing, continuing and opening rows at
    // its in-plane index are the same "box" row -- all three plane groups
    // present, each holding the in-plane entries qm (interior rows: all of
    // them).  Window values outside qm are zeroed: a product with +-0.0 added
    // to a running sum leaves it unchanged (the sum starts at +0.0 and a
    // round-to-nearest sum is never -0.0), so each row still receives
    // exactly its own entries, in order.  Other warps take the general path.
    auto steady = [&](int p) {
      uint32_t mk_s[kPlaneRPT], bq_s[kPlaneRPT];
      open_masks(mk_s, true);
      bool ok = true, partial = false;
#pragma unroll
      for (int h = 0; h < kPlaneRPT; ++h) {
        bq_s[h] = boxq(mk_s[h]);
        ok = ok && bq_f[h] == bq_m[h] && bq_m[h] == bq_s[h] && bq_s[h] != kNoBox;
        partial = partial || bq_m[h] != kMid;
      }
      if (PG_PLANE_EXP & 4) return;
      if (!((PG_PLANE_EXP & 16) || __all_sync(0xffffffffu, ok))) {
        general(p, true, true, true, mk_s);
        return;
      }
      const int ri = (p - 1) * (int)S + (int)q0;
      if (__any_sync(0xffffffffu, partial))
        body(ri, mk_s, bq_s, std::true_type{}, std::true_type{});
      else
        body(ri, mk_s, bq_s, std::false_type{}, std::true_type{});
    };
    // Interior planes of a host-verified matrix (plane_qm): the rows at
    // in-plane index q are box rows with entries plane_qm[q] on every
    // interior plane, so no pattern ids are read.
    uint32_t qb_t[kPlaneRPT], mb_t[kPlaneRPT];
    // (again: a forced reload after the interior loop, so that the masks
    // hold no registers across it)
    auto box_masks = [&](bool again) {
#pragma unroll
      for (int h = 0; h < kPlaneRPT; ++h) {
        uint32_t q = kMid;
        if (plane_qm && act[h])
          q = again ? (uint32_t) * reinterpret_cast<const volatile uint16_t*>(plane_qm + q0 + jj[h])
                    : (uint32_t)__ldg(plane_qm + q0 + jj[h]);
        qb_t[h] = q;
        mb_t[h] = Sh::FULL ? (q | (q << NO) | (q << (NO + NM))) : (1u | (q << NO) | (1u << (NO + NM)));
      }
    };
    box_masks(false);
    bool zero_t = false;
#pragma unroll
    for (int h = 0; h < kPlaneRPT; ++h) zero_t = zero_t || qb_t[h] != kMid;
    zero_t = __any_sync(0xffffffffu, zero_t) && !(PG_PLANE_EXP & 32);
    // planes za - 1, za: warm-up; za + 1 .. zb - 2: steady; zb - 1, zb: drain.
    // The steady planes whose three rows are all on interior planes of a
    // host-verified matrix, [bl, bh], run as a counted loop of the unrolled
    // body (no pattern ids, no per-stage dispatch).
    const int pa0 = (int)za, pb0 = (int)zb;
    // Host-verified matrices whose end planes are box rows too (pa.allbox:
    // plane 0 rows hold no dz = -1 group, plane nz-1 rows no dz = +1 group,
    // every other group the in-plane entries plane_qm[q]): the warm-up and
    // drain stages of a chunk run the unrolled body with the absent groups
    // switched off, so no stage reads pattern ids or takes the general path.
    auto edge = [&](int p) {
      const bool C = p - 1 >= pa0;               // rows of plane p - 1 close
      const bool CA = C && p < (int)pa.nz;       // ... and have a dz = +1 group
      const bool M = p >= pa0 && p < pb0;        // rows of plane p continue
      const bool SA = p + 1 < pb0 && p >= 0;     // rows of plane p + 1 open with a dz = -1 group
      const int ri = (p - 1) * (int)S + (int)q0;
      double acc_s[kPlaneRPT];
#pragma unroll
      for (int h0 = 0; h0 < kPlaneRPT; h0 += 2) {
        double P[2][NM];
        load_pair(P, h0);
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int i = 0; i < NM; ++i)
            if (!((qb_t[h0 + u] >> i) & 1u)) P[u][i] = 0.0;
#pragma unroll
        for (int u = 0; u < 2; ++u) acc_s[h0 + u] = 0.0;
#pragma unroll
        for (int i = 0; i < NM; ++i) {
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int h = h0 + u;
            if (i < NO) {
              const double o = Sh::FULL ? P[u][i] : P[u][Sh::CTR];
              if (CA) acc_f[h] = __dadd_rn(acc_f[h], __dmul_rn(pm.v[NO + NM + i], o));
              if (SA) acc_s[h] = __dadd_rn(acc_s[h], __dmul_rn(pm.v[i], o));
            }
            if (M) acc_m[h] = __dadd_rn(acc_m[h], __dmul_rn(pm.v[NO + i], P[u][i]));
          }
        }
        if (kPairEpi) {
          if (C && act[h0]) finish2(h0, (int64_t)(ri + jj[h0]), acc_f[h0], acc_f[h0 + 1]);
        } else {
#pragma unroll
          for (int u = 0; u < 2; ++u)
            if (C && act[h0 + u]) finish(h0 + u, (int64_t)(ri + jj[h0 + u]), acc_f[h0 + u]);
        }
      }
#pragma unroll
      for (int h = 0; h < kPlaneRPT; ++h) {
        acc_f[h] = acc_m[h];
        acc_m[h] = acc_s[h];
      }
    };
    auto stage = [&](int p) {
      if (pa.allbox) {
        edge(p);
      } else if (p >= pa0 + 1 && p <= pb0 - 2) {
        steady(p);
      } else {
        const bool start = p + 1 < pb0;
        uint32_t mk_s[kPlaneRPT];
        open_masks(mk_s, start);
        general(p, p - 1 >= pa0, p >= pa0 && p < pb0, start, mk_s);
      }
    };
    const int bl = box_lo, bh = box_hi;
    int p = pa0 - 1;
    for (; p < bl; ++p) {
      wait_stage(p);
      stage(p);
      next_slot();
    }
    if (p <= bh) {
      int ri = (p - 1) * (int)S + (int)q0;
      // fresh copies of the ring position for the loop: their live ranges
      // end with it, so they are not spilled with the stages around it
      asm volatile("mov.u32 %0, %0;" : "+r"(boff));
      asm volatile("mov.u32 %0, %0;" : "+r"(phase));
      if (zero_t) {
#pragma unroll kPlaneUnroll
        for (int left = bh - p + 1; left > 0; --left, ri += (int)S) {
          wait_stage(bh + 1 - left);
          body(ri, mb_t, qb_t, std::true_type{}, std::false_type{});
          next_slot();
        }
      } else {
#pragma unroll kPlaneUnroll
        for (int left = bh - p + 1; left > 0; --left, ri += (int)S) {
          wait_stage(bh + 1 - left);
          body(ri, mb_t, qb_t, std::false_type{}, std::false_type{});
          next_slot();
        }
      }
      p = bh + 1;
      asm volatile("mov.u32 %0, %0;" : "+r"(boff));
      asm volatile("mov.u32 %0, %0;" : "+r"(phase));
      // the interior loop left the masks in place: the rows now closing and
      // continuing were opened inside it
      box_masks(true);
#pragma unroll
      for (int h = 0; h < kPlaneRPT; ++h) {
        mk_f[h] = mk_m[h] = mb_t[h];
        bq_f[h] = bq_m[h] = qb_t[h];
      }
    }
    for (; p <= pb0; ++p) {
      wait_stage(p);
      stage(p);
      next_slot();
    }
  }
#undef PG_BUF
  if (MODE == kResid) {
    const double s = block_sum(local);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
    last_block_reduce(partials, counter, 1, nsq);
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static int plane_env(const char* name, int dflt) {
  const char* s = std::getenv(name);
  return s ? std::atoi(s) : dflt;
}

// in-plane offset of middle-group value i
static int64_t mid_off_host(int kind, int i, int64_t g) {
  if (kind == 27) return (int64_t)(i / 3 - 1) * g + (i % 3 - 1);
  if (kind == 7) return i == 0 ? -g : (i == 4 ? g : (int64_t)(i - 2));
  return (int64_t)(i - 1);
}

// Tile width Q and planes per chunk Zc: the pair that minimises
// waves x (Q + H/2) x (Zc + 2 warm-up planes) for the resident blocks (all
// blocks of a wave march the same planes together, so the tiles' halo reads
// of a plane hit L2), with at most kMaxBlocks blocks (the residual's partial
// slots).  PG_PLANE_Q / PG_PLANE_Z / PG_PLANE_STAGES override.
void plane_prepare(pg_matrix* m) {
  m->plane_kind = 0;
  // 1 (default): 27-point stencils; 2: every plane stencil; 0: off
  const int on = plane_env("PG_SPMV_PLANES", 1);
  if (!on) return;
  int kind;
  int64_t S, g;
  if (!stencil_shape(m, &kind, &S, &g)) return;
  if (on == 1 && kind != 27) return;
  // 16-byte aligned pattern-id / operand slices and whole planes
  if (S % 16 != 0 || m->nrows % S != 0 || m->n_pat > 256) return;
  // 32-bit row indices inside the kernel
  if (m->nrows + 4 * S >= ((int64_t)1 << 31)) return;
  // zeroed window values stand for absent entries (v * 0.0 = +-0.0): finite
  // master values only
  for (int i = 0; i < m->pat_mlen; ++i)
    if (!std::isfinite(m->pat_mv[i])) return;
  const int NM = kind == 27 ? 9 : kind == 7 ? 5 : 3;
  const int64_t H = (kind == 27) ? g + 1 : (kind == 7 ? g : 1);
  const int64_t nz = m->nrows / S;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, m->device);
  const int64_t cap = (int64_t)sms * PG_PLANE_MIN_BLOCKS;
  const int qenv = plane_env("PG_PLANE_Q", 0), zenv = plane_env("PG_PLANE_Z", 0);
  double best = 1e300;
  int bq = 0;
  int64_t bz = 0;
  for (int Q = 64; Q <= kPlaneMaxQ; Q += 32) {
    if (qenv > 0 && Q != qenv) continue;
    const int64_t sb = 8 * (Q + 2 * H + 2) + 17 * (int64_t)Q + 256 + 128;
    if (2 * sb > kPlaneSmemBudget) continue;
    const int64_t nqb = (S + Q - 1) / Q;
    int64_t last = -1;
    for (int64_t nch = 1; nch <= nz; ++nch) {
      const int64_t Zc = zenv > 0 ? std::min<int64_t>(zenv, nz) : (nz + nch - 1) / nch;
      if (Zc == last) continue;
      last = Zc;
      const int64_t items = nqb * ((nz + Zc - 1) / Zc);
      if (items > kMaxBlocks) continue;
      const int64_t waves = (items + cap - 1) / cap;
      const double cost = (double)waves * (Q + 0.5 * H) * (double)(Zc + 2);
      if (cost < best) {
        best = cost;
        bq = Q;
        bz = Zc;
      }
    }
  }
  if (!bq) return;
  PlaneArgs& pa = m->plane;
  std::memset(&pa, 0, sizeof pa);
  pa.nrows = m->nrows;
  pa.ncols = m->ncols;
  pa.S = S;
  pa.nz = nz;
  pa.Q = bq;
  pa.nqb = (int)((S + bq - 1) / bq);
  pa.Zc = (int)bz;
  pa.H = (int)H;
  pa.sh = (int)(H & 1);
  const int wdoubles = bq + 2 * (int)H + 2;
  pa.off_a = ((8 * wdoubles + 127) / 128) * 128;
  pa.off_b = pa.off_a + 8 * bq;
  pa.off_p = pa.off_b + 8 * bq;
  pa.off_bar = ((pa.off_p + bq + 7) / 8) * 8;  // the stage's full and empty mbarriers
  pa.stage_bytes = ((pa.off_bar + 16 + 127) / 128) * 128;
  int stages = kPlaneSmemBudget / pa.stage_bytes;
  const int senv = plane_env("PG_PLANE_STAGES", 0);
  if (senv > 0 && senv * pa.stage_bytes <= kPlaneSmemBudget) stages = senv;
  if (stages > kPlaneMaxStages) stages = kPlaneMaxStages;
  if (stages < 2) return;
  pa.stages = stages;
  for (int i = 0; i < NM; ++i) pa.woff[i] = (int)(mid_off_host(kind, i, g) + H + pa.sh);
  // 27-point tiles whose three runs start at odd window positions (even
  // in-plane stride): the pair path's 16-byte loads and stores are aligned
  // (S, Q and every tile origin are multiples of 16; PG_PLANE_VEC=0: off)
  pa.vec = (kind == 27 && (pa.woff[0] & 1) && (pa.woff[3] & 1) && (pa.woff[6] & 1) &&
            plane_env("PG_PLANE_VEC", 1)) ? 1 : 0;
  m->plane_blocks = (int)((int64_t)pa.nqb * ((nz + bz - 1) / bz));
  m->plane_kind = kind;
  // outer plane groups with bitwise equal coefficients (kernel SYM variants;
  // PG_PLANE_SYM=0: off)
  m->plane_sym = 0;
  if (kind == 27 && m->pat_mlen == 27 && plane_env("PG_PLANE_SYM", 1)) {
    bool rest = true, ctr = true;
    for (int i = 0; i < 9; ++i) {
      const bool eq = std::memcmp(&m->pat_mv[i], &m->pat_mv[18 + i], sizeof(double)) == 0;
      if (i == 4) ctr = eq; else rest = rest && eq;
    }
    m->plane_sym = rest ? 1 : 0;  // (ctr && rest: still variant 1, one product more)
    (void)ctr;
  }
  // Interior planes 1 .. nz-2: if every in-plane index q has one pattern on
  // all of them and that pattern is a "box" row (all three plane groups
  // holding the same in-plane entries qm), the kernel's interior stages use
  // qm[q] without reading pattern ids (PG_PLANE_BOX=0: always read them).
  if (nz >= 3 && plane_env("PG_PLANE_BOX", 1)) {
    std::vector<uint8_t> id((size_t)m->nrows);
    std::vector<uint32_t> mk((size_t)m->n_pat);
    PG_CUDA(cudaMemcpy(id.data(), m->rpat, id.size(), cudaMemcpyDeviceToHost));
    PG_CUDA(cudaMemcpy(mk.data(), m->pat_mask, 4 * mk.size(), cudaMemcpyDeviceToHost));
    const int NO = kind == 27 ? 9 : (kind == 9 ? 3 : 1);
    const uint32_t mid = (1u << NM) - 1u;
    std::vector<uint16_t> qm((size_t)S);
    bool ok = true;
    for (int64_t q = 0; q < S && ok; ++q) {
      const uint8_t pid = id[(size_t)(S + q)];
      for (int64_t z = 2; z + 1 < nz && ok; ++z) ok = id[(size_t)(z * S + q)] == pid;
      const uint32_t mkq = mk[pid], m9 = (mkq >> NO) & mid;
      const uint32_t box = (kind == 27 || kind == 9) ? (m9 | (m9 << NO) | (m9 << (NO + NM)))
                                                   : (1u | (m9 << NO) | (1u << (NO + NM)));
      ok = ok && mkq == box;
      qm[(size_t)q] = (uint16_t)m9;
    }
    if (ok) {
      // end planes: plane 0 rows without the dz = -1 group, plane nz-1 rows
      // without the dz = +1 group, the other groups as on interior planes
      // (PG_PLANE_BOX=1: interior planes only)
      bool ends = plane_env("PG_PLANE_BOX", 2) >= 2;
      const bool full = kind == 27 || kind == 9;
      for (int64_t q = 0; q < S && ends; ++q) {
        const uint32_t m9 = qm[(size_t)q];
        const uint32_t lo = full ? m9 : 1u, hi = (full ? m9 : 1u) << (NO + NM);
        ends = mk[id[(size_t)q]] == ((m9 << NO) | hi) &&
               mk[id[(size_t)((nz - 1) * S + q)]] == (lo | (m9 << NO));
      }
      pa.allbox = ends ? 1 : 0;
      PG_CUDA(cudaMalloc(&m->plane_qm, 2 * qm.size()));
      PG_CUDA(cudaMemcpy(m->plane_qm, qm.data(), 2 * qm.size(), cudaMemcpyHostToDevice));
      m->bytes += 2 * qm.size();
    }
  }
}

bool plane_shape(const pg_matrix* m) { return m->plane_kind != 0; }

template <int MODE>
bool plane_launch(const pg_matrix* m, const double* x, Epi e, pg_workspace* ws, double* nsq,
                  cudaStream_t st) {
  if (!m->plane_kind) return false;
  // every bulk-copied vector 16-byte aligned
  auto al16 = [](const void* p) { return ((uintptr_t)p & 15u) == 0; };
  if (!(al16(x) && al16(e.acc_in) && al16(e.base) && al16(e.b) && al16(m->rpat))) return false;
  if (m->plane.vec && !(al16(e.acc_out) && al16(e.w_out))) return false;
  if (MODE == kResid && !ws) return false;
  PatMaster pm;
  std::memset(&pm, 0, sizeof pm);
  pm.len = m->pat_mlen;
  for (int i = 0; i < pm.len; ++i) pm.v[i] = m->pat_mv[i];
  const size_t smem = (size_t)m->plane.stages * m->plane.stage_bytes;
  // 27-point stencils with aligned tiles (PlaneArgs::vec, i.e. an even
  // in-plane stride): the adjacent-pair kernels (ADJ) for kPoly -- with the
  // pass flags and base presence as compile-time constants (EF) -- and
  // kSpmv; everything else runs the runtime-flag kernels (EF = -1).  SYM:
  // the outer plane groups share their coefficients (all offsets but the
  // center), the shared-product variants.
  const int ef = (e.flags & 3) | (e.base ? 4 : 0);
#ifdef PG_PLANE_DEV
  // development builds (seconds instead of minutes): the middle kPoly pass
  // of a SYM / ADJ 27-point matrix only, everything else declines
  if (MODE != kPoly || ef != 2 || m->plane_kind != 27 || m->plane_sym != 1 || !m->plane.vec)
    return false;
  auto kern = plane_ring_kernel<kPoly, 27, 2, 1, true>;
  int ki = 0;
#else
  auto kern = plane_ring_kernel<MODE, 27, -1>;
  int ki = 0;
  const bool sym = m->plane_kind == 27 && m->plane_sym == 1;
  const bool adj = m->plane_kind == 27 && m->plane.vec;
  if (MODE == kPoly && adj) {
#define PG_PLANE_EF(SYM)                                                                        \
  (ef == 0 ? plane_ring_kernel<MODE, 27, 0, SYM, true> : ef == 1 ? plane_ring_kernel<MODE, 27, 1, SYM, true> \
   : ef == 2 ? plane_ring_kernel<MODE, 27, 2, SYM, true> : ef == 3 ? plane_ring_kernel<MODE, 27, 3, SYM, true> \
   : ef == 4 ? plane_ring_kernel<MODE, 27, 4, SYM, true> : ef == 5 ? plane_ring_kernel<MODE, 27, 5, SYM, true> \
   : ef == 6 ? plane_ring_kernel<MODE, 27, 6, SYM, true> : plane_ring_kernel<MODE, 27, 7, SYM, true>)
    if constexpr (MODE == kPoly) kern = sym ? PG_PLANE_EF(1) : PG_PLANE_EF(0);
#undef PG_PLANE_EF
    ki = 4 + ef + (sym ? 8 : 0);
  } else if (MODE == kSpmv && adj) {
    if constexpr (MODE == kSpmv)
      kern = sym ? plane_ring_kernel<MODE, 27, -1, 1, true>
                 : plane_ring_kernel<MODE, 27, -1, 0, true>;
    ki = sym ? 21 : 22;
  } else if (sym) {
    kern = plane_ring_kernel<MODE, 27, -1, 1>;
    ki = 20;
  } else {
    kern = m->plane_kind == 27 ? plane_ring_kernel<MODE, 27, -1>
         : m->plane_kind == 7  ? plane_ring_kernel<MODE, 7, -1>
         : m->plane_kind == 9  ? plane_ring_kernel<MODE, 9, -1>
                               : plane_ring_kernel<MODE, 5, -1>;
    ki = m->plane_kind == 27 ? 0 : m->plane_kind == 7 ? 1 : m->plane_kind == 9 ? 2 : 3;
  }
#endif
  static bool attr[4][23][64] = {};
  const int dev = m->device;
  if (!attr[MODE][ki][dev]) {
    PG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kPlaneSmemBudget));
    attr[MODE][ki][dev] = true;
  }
  launch_k(kern, m->plane_blocks, kPlaneThreads, smem, st, m->plane, (const uint8_t*)m->rpat,
           (const int32_t*)m->pat_ptr, (const PairEnt*)m->pat_ent, m->n_pat,
           (const uint32_t*)m->pat_mask, pm, x, e, ws ? ws->partials : nullptr,
           ws ? ws->counter : nullptr, nsq, (const uint16_t*)m->plane_qm);
  check_launch();
  return true;
}

template bool plane_launch<kSpmv>(const pg_matrix*, const double*, Epi, pg_workspace*, double*,
                                  cudaStream_t);
template bool plane_launch<kPoly>(const pg_matrix*, const double*, Epi, pg_workspace*, double*,
                                  cudaStream_t);
template bool plane_launch<kResid>(const pg_matrix*, const double*, Epi, pg_workspace*, double*,
                                   cudaStream_t);
template bool plane_launch<kRoot>(const pg_matrix*, const double*, Epi, pg_workspace*, double*,
                                  cudaStream_t);

}  // namespace pg
