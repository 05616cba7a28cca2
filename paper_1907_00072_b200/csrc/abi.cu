// libpgmres: library plumbing -- errors, SELL-C-sigma construction, device
// operator and workspace lifetime.
//
// The SELL build replaces the reference's CSR storage (sparse.py:42-148) with
// a warp-sliced layout; the entry order inside each row is preserved so the
// device SpMV reproduces spmv()'s per-row sequential sum (sparse.py:164-168).

#include <algorithm>
#include <iterator>
#include <cstdint>
#include <cstdlib>
#include <unordered_map>
#include <cstring>
#include <functional>
#include <numeric>
#include <string>
#include <vector>

#include "internal.cuh"

namespace pg {

static thread_local std::string g_last_error;

void set_last_error(const std::string& msg) { g_last_error = msg; }

thread_local bool g_capturing = false;

bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* s = std::getenv("PG_PDL");
    v = s ? (std::atoi(s) != 0) : 1;
  }
  return v == 1;
}

int grid_for(int device, const void* kernel, int block, size_t smem, int64_t work_blocks) {
  int sms = 0, per_sm = 0;
  PG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  PG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem));
  if (per_sm < 1) per_sm = 1;
  // whole waves only: at most kMaxBlocks (the reductions' partial slots)
  if (per_sm > kMaxBlocks / sms) per_sm = kMaxBlocks / sms > 0 ? kMaxBlocks / sms : 1;
  int64_t g = (int64_t)sms * per_sm;
  if (work_blocks < g) g = work_blocks;
  if (g < 1) g = 1;
  return (int)g;
}

// ---------------------------------------------------------------------------
// host SELL-C-sigma plan
// ---------------------------------------------------------------------------
static void validate_csr(int64_t nrows, const int64_t* row_ptr) {
  PG_REQUIRE(nrows >= 0, PG_ERR_PARAMETER, "nrows must be non-negative");
  PG_REQUIRE(nrows < (int64_t(1) << 31) - 64, PG_ERR_PARAMETER, "nrows exceeds int32 range");
  PG_REQUIRE(row_ptr != nullptr, PG_ERR_PARAMETER, "row_ptr is null");
  PG_REQUIRE(row_ptr[0] == 0, PG_ERR_PARAMETER, "row_ptr[0] must be 0");
  for (int64_t r = 0; r < nrows; ++r)
    PG_REQUIRE(row_ptr[r + 1] >= row_ptr[r], PG_ERR_PARAMETER, "row_ptr must be non-decreasing");
}

// Lane order: rows sorted by decreasing length inside windows of sigma rows
// (stable, so sigma <= 1 is the identity).
static std::vector<int32_t> lane_order(int64_t nrows, const int64_t* row_ptr, int sigma) {
  std::vector<int32_t> order(nrows);
  std::iota(order.begin(), order.end(), 0);
  if (sigma > 1) {
    for (int64_t w0 = 0; w0 < nrows; w0 += sigma) {
      int64_t w1 = std::min<int64_t>(nrows, w0 + sigma);
      std::stable_sort(order.begin() + w0, order.begin() + w1, [&](int32_t a, int32_t b) {
        return (row_ptr[a + 1] - row_ptr[a]) > (row_ptr[b + 1] - row_ptr[b]);
      });
    }
  }
  return order;
}

struct SellHost {
  int64_t n_slices = 0, padded = 0;
  int max_width = 0;
  std::vector<int64_t> slice_ptr;
  std::vector<int32_t> slice_w, row_len, perm;
};

static SellHost sell_plan(int64_t nrows, const int64_t* row_ptr, int sigma) {
  validate_csr(nrows, row_ptr);
  SellHost h;
  h.n_slices = (nrows + PG_SLICE - 1) / PG_SLICE;
  std::vector<int32_t> order = lane_order(nrows, row_ptr, sigma);
  h.slice_ptr.assign(h.n_slices + 1, 0);
  h.slice_w.assign(h.n_slices, 0);
  h.row_len.assign(h.n_slices * PG_SLICE, 0);
  h.perm.assign(h.n_slices * PG_SLICE, -1);
  for (int64_t s = 0; s < h.n_slices; ++s) {
    int32_t w = 0;
    for (int t = 0; t < PG_SLICE; ++t) {
      int64_t lane = s * PG_SLICE + t;
      if (lane >= nrows) break;
      int32_t r = order[lane];
      int64_t len = row_ptr[r + 1] - row_ptr[r];
      PG_REQUIRE(len < (int64_t(1) << 30), PG_ERR_PARAMETER, "row too long");
      h.perm[lane] = r;
      h.row_len[lane] = (int32_t)len;
      w = std::max<int32_t>(w, (int32_t)len);
    }
    h.slice_w[s] = w;
    h.max_width = std::max(h.max_width, (int)w);
    h.slice_ptr[s + 1] = h.slice_ptr[s] + (int64_t)w * PG_SLICE;
  }
  h.padded = h.slice_ptr[h.n_slices];
  return h;
}

static void sell_fill(const SellHost& h, int64_t ncols, const int64_t* row_ptr,
                      const int64_t* col_idx, const double* values, int32_t* col, double* val) {
  PG_REQUIRE(ncols >= 0 && ncols < (int64_t(1) << 31), PG_ERR_PARAMETER,
             "ncols exceeds int32 range");
  std::memset(col, 0, sizeof(int32_t) * h.padded);
  std::memset(val, 0, sizeof(double) * h.padded);
  for (int64_t s = 0; s < h.n_slices; ++s) {
    int64_t base = h.slice_ptr[s];
    for (int t = 0; t < PG_SLICE; ++t) {
      int64_t lane = s * PG_SLICE + t;
      int32_t r = h.perm[lane];
      if (r < 0) continue;
      int64_t q0 = row_ptr[r], len = h.row_len[lane];
      for (int64_t j = 0; j < len; ++j) {
        int64_t c = col_idx[q0 + j];
        PG_REQUIRE(c >= 0 && c < ncols, PG_ERR_PARAMETER, "column indices out of range");
        col[base + j * PG_SLICE + t] = (int32_t)c;
        val[base + j * PG_SLICE + t] = values[q0 + j];
      }
    }
  }
}

template <class T>
static T* upload(const T* host, size_t count, size_t& bytes) {
  T* d = nullptr;
  size_t nb = sizeof(T) * std::max<size_t>(count, 1);
  cudaError_t e = cudaMalloc(&d, nb);
  if (e != cudaSuccess) throw Error(PG_ERR_ALLOC, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  if (count) PG_CUDA(cudaMemcpy(d, host, sizeof(T) * count, cudaMemcpyHostToDevice));
  bytes += nb;
  return d;
}

static void free_matrix(pg_matrix* m) {
  if (!m) return;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(m->device);
  cudaFree(m->slice_ptr);
  cudaFree(m->slice_w);
  cudaFree(m->row_len);
  cudaFree(m->perm);
  cudaFree(m->col);
  cudaFree(m->val);
  cudaFree(m->col8);
  cudaFree(m->slice_ptr8);
  cudaFree(m->dtab);
  cudaFree(m->val8);
  cudaFree(m->vtab);
  cudaFree(m->wtab);
  cudaFree(m->pair8);
  cudaFree(m->ptab);
  cudaFree(m->rpat);
  cudaFree(m->pat_ptr);
  cudaFree(m->pat_ent);
  cudaFree(m->pat_mask);
  cudaFree(m->opat);
  cudaFree(m->opat_mask);
  cudaFree(m->plane_qm);
  cudaSetDevice(cur);
  delete m;
}

// ---------------------------------------------------------------------------
// Exact dictionary compression of the SELL streams.  Constant-coefficient
// stencils (configs 1, 2, 4) have a handful of distinct column offsets
// (col - row) and of distinct value bit patterns; when there are <= 256 of
// each, the device keeps 1-byte indices into per-matrix tables instead of
// int32 columns and f64 values: 2 B per entry instead of 12.  Lookups return
// the identical bits, so the SpMV stays bit-for-bit the reference's.
// PG_SPMV_DICT=0 disables it.
// ---------------------------------------------------------------------------
template <class K, class H>
static bool dict_encode(const std::vector<K>& keys, std::vector<uint8_t>& idx,
                        std::vector<K>& table, H hasher) {
  std::unordered_map<K, int, H> map(512, hasher);
  idx.resize(keys.size());
  for (size_t i = 0; i < keys.size(); ++i) {
    auto it = map.find(keys[i]);
    if (it == map.end()) {
      if (map.size() == 256) return false;
      it = map.emplace(keys[i], (int)map.size()).first;
      table.push_back(keys[i]);
    }
    idx[i] = (uint8_t)it->second;
  }
  return true;
}

// The 1-byte streams use a packed slice layout: entry j of lane t of slice s
// sits at slice_ptr8[s] + (j/4)*128 + 4t + (j%4), so one 32-bit load per lane
// brings 4 entries (a warp-wide load is one contiguous 128 B segment).
// Window plan (pg_matrix::wtab): natural row order only (the block's rows
// must be contiguous), offsets clustered greedily -- a gap of >= kWinRows
// between consecutive offsets starts a new group (merging would cost more
// window than a second group's kWinRows rows).  Group starts are rounded down
// to an even offset and lengths up to even, so every window copy is a
// 16-byte aligned bulk copy.  No plan when the groups or a pipeline stage
// exceed their budgets (the global-gather dictionary kernel runs).
static std::vector<int32_t> build_window_plan(const std::vector<int64_t>& offs,
                                              const std::vector<int64_t>& sp8, int64_t n_slices,
                                              pg_matrix* m) {
  const char* env = std::getenv("PG_SPMV_WIN");
  if (env && std::atoi(env) == 0) return {};
  if (m->sigma > 1 || offs.empty()) return {};
  std::vector<int64_t> srt(offs);
  std::sort(srt.begin(), srt.end());
  std::vector<int64_t> lo, hi;
  for (int64_t o : srt) {
    if (lo.empty() || o - hi.back() >= kWinRows) {
      lo.push_back(o);
      hi.push_back(o);
    } else {
      hi.back() = o;
    }
  }
  if ((int)lo.size() > kWinMaxGroups) return {};
  int64_t total = 0;
  std::vector<int64_t> len(lo.size());
  for (size_t g = 0; g < lo.size(); ++g) {
    if (lo[g] & 1) lo[g] -= 1;  // even start (floor for negatives too)
    len[g] = kWinRows + (hi[g] - lo[g]);
    len[g] += len[g] & 1;
    total += len[g];
  }
  if (total > kWinMaxElems) return {};
  const int64_t per_blk = kWinRows / PG_SLICE;
  int64_t b8 = 0;
  for (int64_t s0 = 0; s0 < n_slices; s0 += per_blk)
    b8 = std::max(b8, sp8[std::min(s0 + per_blk, n_slices)] - sp8[s0]);
  // a row-pattern stage is the window + one pattern id per row; a pair-stream
  // stage adds the stream, 2 epilogue operand slices, row lengths and widths
  const int64_t win_bytes = ((8 * total + 127) / 128) * 128;
  if (win_bytes + kWinRows > kWinMaxStageBytes) return {};
  m->win_pair_fits = win_bytes + b8 + 20 * kWinRows + 128 <= kWinMaxStageBytes;
  std::vector<int32_t> wtab(256, 0);
  int32_t start = 0;
  for (size_t g = 0; g < lo.size(); ++g) {
    m->wlo[g] = (int32_t)lo[g];
    m->wstart[g] = start;
    m->wlen[g] = (int32_t)len[g];
    start += m->wlen[g];
  }
  for (size_t i = 0; i < offs.size(); ++i) {
    const size_t g = (size_t)(std::upper_bound(lo.begin(), lo.end(), offs[i]) - lo.begin()) - 1;
    wtab[i] = (int32_t)(m->wstart[g] + (offs[i] - lo[g]));
  }
  m->n_wgrp = (int)lo.size();
  m->win_elems = (int)total;
  m->win_b8 = (int)b8;
  return wtab;
}

// Row-pattern dictionary.  On a constant-coefficient stencil a row is one of
// a few dozen sequences of (column offset, value) pairs -- 27 for a 3-D 7- or
// 27-point operator (low / interior / high boundary in each dimension) -- so
// one byte per row names the whole row: no per-entry stream and no row
// length.  The table keeps each pattern's pairs in the row's stored order,
// so the row sum is still the reference's sequential one.  Built from the
// pair stream; none when there are more than 256 patterns, a pattern longer
// than kPatMaxLen or more than kPatMaxEnt table entries.  PG_SPMV_PAT=0
// disables it.
// Row-pattern planning shared by the value-pattern and offset-pattern
// formats (and pg_row_patterns): every lane's row is a sequence of
// fixed-size symbols (sym bytes; a pair index, or a column offset); rows are
// grouped by identical sequence (at most 256), the most frequent sequence is
// the master, and every sequence that is an ordered subsequence of the master
// gets the bit set of master positions it uses (bit 31 set otherwise).
struct PatternPlan {
  std::vector<uint8_t> id;        // per lane
  std::vector<std::string> seqs;  // distinct sequences, first-seen order
  std::vector<int64_t> count;     // live lanes per sequence
  size_t master = 0;
  std::vector<uint32_t> mask;     // per sequence
};

template <class KeyFn>
static bool plan_patterns(int64_t nl, size_t sym, KeyFn key, PatternPlan& P) {
  P.id.assign(std::max<int64_t>(nl, 1), 0);
  std::unordered_map<std::string, int> ids;
  std::string k;
  for (int64_t lane = 0; lane < nl; ++lane) {
    k.clear();
    const bool live = key(lane, k);
    auto it = ids.find(k);
    if (it == ids.end()) {
      if (ids.size() == 256) return false;
      it = ids.emplace(k, (int)P.seqs.size()).first;
      P.seqs.push_back(k);
      P.count.push_back(0);
    }
    P.id[lane] = (uint8_t)it->second;
    if (live) ++P.count[it->second];
  }
  if (P.seqs.empty()) return false;
  P.master = (size_t)(std::max_element(P.count.begin(), P.count.end()) - P.count.begin());
  const std::string& ms = P.seqs[P.master];
  const size_t ml = ms.size() / sym;
  P.mask.assign(P.seqs.size(), 1u << 31);
  if (ml > 31) return true;
  for (size_t p = 0; p < P.seqs.size(); ++p) {
    uint32_t bits = 0;
    size_t q = 0;
    for (size_t e = 0; e < P.seqs[p].size(); e += sym) {
      while (q < ml && std::memcmp(ms.data() + sym * q, P.seqs[p].data() + e, sym) != 0) ++q;
      if (q == ml) {
        bits = 1u << 31;
        break;
      }
      bits |= 1u << q++;
    }
    P.mask[p] = bits;
  }
  return true;
}

static void build_patterns(const SellHost& h, const std::vector<uint8_t>& p8,
                           const std::vector<int64_t>& sp8, const std::vector<PairEnt>& ptab,
                           pg_matrix* m) {
  const char* env = std::getenv("PG_SPMV_PAT");
  if (env && std::atoi(env) == 0) return;
  if (h.max_width > kPatMaxLen) return;
  const int64_t nl = h.n_slices * PG_SLICE;
  PatternPlan P;
  const bool ok = plan_patterns(nl, 1, [&](int64_t lane, std::string& key) {
    const int64_t s = lane / PG_SLICE;
    const int t = (int)(lane % PG_SLICE);
    const int len = h.perm[lane] < 0 ? 0 : h.row_len[lane];
    for (int j = 0; j < len; ++j)
      key.push_back((char)p8[(size_t)sp8[s] + (size_t)(j / 4) * 128 + 4 * t + (j & 3)]);
    return h.perm[lane] >= 0;
  }, P);
  if (!ok) return;
  const std::vector<std::string>& seqs = P.seqs;
  std::vector<int32_t> ptr(seqs.size() + 1, 0);
  std::vector<PairEnt> ent;
  int maxlen = 0;
  for (size_t p = 0; p < seqs.size(); ++p) {
    for (char c : seqs[p]) ent.push_back(ptab[(uint8_t)c]);
    ptr[p + 1] = (int32_t)ent.size();
    maxlen = std::max(maxlen, (int)seqs[p].size());
  }
  if ((int)ent.size() > kPatMaxEnt) return;
  // master pattern: the most frequent one; every pattern that is an ordered
  // subsequence of it (same pair indices, hence same values) gets its mask
  std::vector<uint32_t> mask = P.mask;
  const std::string& ms = seqs[P.master];
  if (ms.size() <= 31) {
    m->pat_mlen = (int)ms.size();
    m->pat_all_master = 1;
    for (uint32_t bits : mask) m->pat_all_master &= (bits >> 31) ? 0 : 1;
    for (size_t q = 0; q < ms.size(); ++q) {
      const PairEnt& pe = ptab[(uint8_t)ms[q]];
      m->pat_mv[q] = pe.v;
      m->pat_mdoff[q] = pe.doff;
      m->pat_mwoff[q] = pe.woff;
    }
  }
  if (ent.empty()) ent.push_back(PairEnt{});
  m->pat_mask = upload(mask.data(), mask.size(), m->bytes);
  m->rpat = upload(P.id.data(), P.id.size(), m->bytes);
  m->pat_ptr = upload(ptr.data(), ptr.size(), m->bytes);
  m->pat_ent = upload(ent.data(), ent.size(), m->bytes);
  m->n_pat = (int)seqs.size();
  m->pat_nent = (int)ptr.back();
  m->pat_maxlen = maxlen;
}

// Row offset patterns: when the values do not compress (no row-pattern
// dictionary) but every row's column-offset sequence is one of <= 256 --
// a variable-coefficient stencil -- one byte per row names it, so the kernel
// needs no column stream: the master offsets are constant-bank operands and
// only the f64 values are streamed (8 instead of 12 B per entry).  Rows that
// are not ordered subsequences of the master keep the SELL column stream.
// PG_SPMV_OPAT=0 disables it.
static void build_offset_patterns(const SellHost& h, const int32_t* col, pg_matrix* m) {
  const char* env = std::getenv("PG_SPMV_OPAT");
  if (env && std::atoi(env) == 0) return;
  if (m->rpat || h.max_width > 31 || m->nrows == 0) return;
  const int64_t nl = h.n_slices * PG_SLICE;
  PatternPlan P;
  bool fits = true;
  const bool ok = plan_patterns(nl, 4, [&](int64_t lane, std::string& key) {
    const int64_t s = lane / PG_SLICE;
    const int t = (int)(lane % PG_SLICE);
    const int32_t r = h.perm[lane];
    const int len = r < 0 ? 0 : h.row_len[lane];
    for (int j = 0; j < len; ++j) {
      const int64_t o = (int64_t)col[h.slice_ptr[s] + (int64_t)j * PG_SLICE + t] - r;
      fits = fits && o >= INT32_MIN && o <= INT32_MAX;
      const int32_t o32 = (int32_t)o;
      key.append(reinterpret_cast<const char*>(&o32), 4);
    }
    return r >= 0;
  }, P);
  if (!ok || !fits) return;
  const std::string& ms = P.seqs[P.master];
  const size_t ml = ms.size() / 4;
  if (ml == 0 || ml > 31) return;
  m->opat = upload(P.id.data(), P.id.size(), m->bytes);
  m->opat_mask = upload(P.mask.data(), P.mask.size(), m->bytes);
  m->opat_n = (int)P.seqs.size();
  m->opat_mlen = (int)ml;
  for (size_t q = 0; q < ml; ++q) std::memcpy(&m->opat_mdoff[q], ms.data() + 4 * q, 4);
}

static void build_dictionaries(const SellHost& h, const int32_t* col, const double* val,
                               pg_matrix* m) {
  const char* env = std::getenv("PG_SPMV_DICT");
  if (env && std::atoi(env) == 0) return;
  std::vector<int64_t> sp8(h.n_slices + 1, 0);
  for (int64_t s = 0; s < h.n_slices; ++s)
    sp8[s + 1] = sp8[s] + (int64_t)((h.slice_w[s] + 3) / 4) * 4 * PG_SLICE;
  const size_t P = (size_t)std::max<int64_t>(sp8[h.n_slices], 4);
  std::vector<int64_t> delta(P, 0);
  std::vector<uint64_t> bits(P, 0);
  for (int64_t s = 0; s < h.n_slices; ++s) {
    for (int t = 0; t < PG_SLICE; ++t) {
      const int64_t lane = s * PG_SLICE + t;
      const int32_t r = h.perm[lane];
      if (r < 0) continue;
      for (int j = 0; j < h.row_len[lane]; ++j) {
        const size_t pos = (size_t)h.slice_ptr[s] + (size_t)j * PG_SLICE + t;
        const size_t p8 = (size_t)sp8[s] + (size_t)(j / 4) * 128 + 4 * t + (j & 3);
        delta[p8] = (int64_t)col[pos] - r;
        std::memcpy(&bits[p8], &val[pos], 8);
      }
    }
  }
  bool any = false;
  std::vector<int32_t> wtab;  // window plan (empty: none)
  std::vector<uint8_t> c8, v8;
  std::vector<int64_t> dtab64;
  std::vector<uint64_t> vtab_bits;
  // values first: compressing the column offsets alone (12 -> 9 B per entry)
  // measured slower than the plain kernel (cfg5), so columns are only
  // compressed together with the values
  if (!dict_encode(bits, v8, vtab_bits, std::hash<uint64_t>())) return;
  if (dict_encode(delta, c8, dtab64, std::hash<int64_t>())) {
    std::vector<int32_t> dtab(256, 0);
    bool fits = true;
    for (size_t i = 0; i < dtab64.size(); ++i) {
      fits = fits && dtab64[i] >= INT32_MIN && dtab64[i] <= INT32_MAX;
      dtab[i] = (int32_t)dtab64[i];
    }
    if (fits) {
      m->n_doff = (int)dtab64.size();
      for (size_t i = 0; i < dtab64.size(); ++i) m->doff[i] = (int32_t)dtab64[i];
      m->col8 = upload(c8.data(), P, m->bytes);
      m->dtab = upload(dtab.data(), dtab.size(), m->bytes);
      m->n_dcol = (int)dtab64.size();
      any = true;
      wtab = build_window_plan(dtab64, sp8, h.n_slices, m);
    }
  }
  {
    std::vector<double> vtab(256, 0.0);
    for (size_t i = 0; i < vtab_bits.size(); ++i) std::memcpy(&vtab[i], &vtab_bits[i], 8);
    // pair dictionary: one byte per entry indexes (column offset, value) --
    // 27 pairs for a 27-point stencil; read by the pair kernels (spmv.cu)
    const char* penv = std::getenv("PG_SPMV_PAIR");
    const char* renv = std::getenv("PG_SPMV_WIN_MIN_ROW");
    // the windowed kernel pays off on long rows (27-point: 1.6x the pair
    // kernel); short rows (7-point) keep the global-gather pair kernel
    const int64_t min_row = renv ? std::atoll(renv) : 12;
    if (m->nnz < min_row * m->nrows) wtab.clear();
    if (m->col8 && !(penv && std::atoi(penv) == 0)) {
      std::vector<uint16_t> pk(P);
      for (size_t i = 0; i < P; ++i) pk[i] = (uint16_t)((c8[i] << 8) | v8[i]);
      std::vector<uint8_t> p8;
      std::vector<uint16_t> pkeys;
      if (dict_encode(pk, p8, pkeys, std::hash<uint16_t>())) {
        std::vector<PairEnt> ptab(256);
        for (size_t k = 0; k < pkeys.size(); ++k) {
          ptab[k].v = vtab[pkeys[k] & 255];
          ptab[k].woff = wtab.empty() ? 0 : 8 * wtab[pkeys[k] >> 8];
          ptab[k].doff = (int32_t)dtab64[pkeys[k] >> 8];
        }
        m->pair8 = upload(p8.data(), P, m->bytes);
        m->ptab = upload(ptab.data(), ptab.size(), m->bytes);
        build_patterns(h, p8, sp8, ptab, m);
        if (!wtab.empty()) m->wtab = upload(wtab.data(), wtab.size(), m->bytes);
      }
    }
    m->val8 = upload(v8.data(), P, m->bytes);
    m->vtab = upload(vtab.data(), vtab.size(), m->bytes);
    m->n_dval = (int)vtab_bits.size();
    any = true;
  }
  if (any) {
    m->slice_ptr8 = upload(sp8.data(), sp8.size(), m->bytes);
    // uniform slice widths (stencils): packed-stream offsets are computable
    const int64_t st = h.n_slices > 0 ? sp8[1] - sp8[0] : 0;
    bool uniform = st > 0;
    for (int64_t s = 1; uniform && s + 1 < h.n_slices; ++s) uniform = sp8[s + 1] - sp8[s] == st;
    const char* env = std::getenv("PG_SPMV_STRIDE");
    m->stride8 = (uniform && !(env && std::atoi(env) == 0)) ? st : 0;
  }
}

}  // namespace pg

using namespace pg;

extern "C" {

PG_API int pg_version(void) { return 1; }
PG_API int pg_build_checks(void) { return PG_CHECKS; }

PG_API int pg_last_error(char* buf, size_t len) {
  if (!buf || !len) return PG_ERR_PARAMETER;
  std::strncpy(buf, g_last_error.c_str(), len - 1);
  buf[len - 1] = '\0';
  return PG_OK;
}

PG_API int pg_device_count(int* count) {
  return guard([&] {
    PG_REQUIRE(count, PG_ERR_PARAMETER, "count is null");
    PG_CUDA(cudaGetDeviceCount(count));
  });
}

PG_API int pg_set_device(int device) {
  return guard([&] { PG_CUDA(cudaSetDevice(device)); });
}

PG_API int pg_sell_size(int64_t nrows, const int64_t* row_ptr, int sigma, int64_t* n_slices,
                        int64_t* padded_nnz) {
  return guard([&] {
    SellHost h = sell_plan(nrows, row_ptr, sigma);
    if (n_slices) *n_slices = h.n_slices;
    if (padded_nnz) *padded_nnz = h.padded;
  });
}

PG_API int pg_sell_fill(int64_t nrows, int64_t ncols, const int64_t* row_ptr,
                        const int64_t* col_idx, const double* values, int sigma,
                        int64_t* slice_ptr, int32_t* slice_w, int32_t* row_len, int32_t* perm,
                        int32_t* col, double* val) {
  return guard([&] {
    SellHost h = sell_plan(nrows, row_ptr, sigma);
    std::copy(h.slice_ptr.begin(), h.slice_ptr.end(), slice_ptr);
    std::copy(h.slice_w.begin(), h.slice_w.end(), slice_w);
    std::copy(h.row_len.begin(), h.row_len.end(), row_len);
    std::copy(h.perm.begin(), h.perm.end(), perm);
    sell_fill(h, ncols, row_ptr, col_idx, values, col, val);
  });
}

PG_API int pg_row_patterns(int64_t nrows, const int64_t* row_ptr, const int64_t* col_idx,
                           const double* values, int with_values, uint8_t* ids, int* npat,
                           int* master, int* master_len, uint32_t* masks) {
  return guard([&] {
    PG_REQUIRE(npat && master && master_len, PG_ERR_PARAMETER, "null argument");
    validate_csr(nrows, row_ptr);
    PG_REQUIRE(!with_values || values, PG_ERR_PARAMETER, "values required");
    const size_t sym = with_values ? 12 : 4;
    PatternPlan P;
    const bool ok = plan_patterns(nrows, sym, [&](int64_t r, std::string& key) {
      for (int64_t q = row_ptr[r]; q < row_ptr[r + 1]; ++q) {
        const int64_t o = col_idx[q] - r;
        PG_REQUIRE(o >= INT32_MIN && o <= INT32_MAX, PG_ERR_PARAMETER, "offset out of range");
        const int32_t o32 = (int32_t)o;
        key.append(reinterpret_cast<const char*>(&o32), 4);
        if (with_values) key.append(reinterpret_cast<const char*>(values + q), 8);
      }
      return true;
    }, P);
    *npat = ok ? (int)P.seqs.size() : -1;
    *master = ok ? (int)P.master : -1;
    *master_len = ok ? (int)(P.seqs[P.master].size() / sym) : 0;
    if (!ok) return;
    if (ids) std::copy(P.id.begin(), P.id.begin() + nrows, ids);
    if (masks) std::copy(P.mask.begin(), P.mask.end(), masks);
  });
}

PG_API int pg_matrix_create(int device, int64_t nrows, int64_t ncols, const int64_t* row_ptr,
                            const int64_t* col_idx, const double* values, int sigma,
                            pg_matrix** out) {
  return guard([&] {
    PG_REQUIRE(out, PG_ERR_PARAMETER, "out is null");
    *out = nullptr;
    SellHost h = sell_plan(nrows, row_ptr, sigma);
    std::vector<int32_t> col(std::max<int64_t>(h.padded, 1));
    std::vector<double> val(std::max<int64_t>(h.padded, 1));
    sell_fill(h, ncols, row_ptr, col_idx, values, col.data(), val.data());
    DeviceScope scope(device);
    pg_matrix* m = new pg_matrix();
    std::memset(m, 0, sizeof(*m));
    m->device = device;
    m->nrows = nrows;
    m->ncols = ncols;
    m->nnz = row_ptr[nrows];
    m->padded_nnz = h.padded;
    m->n_slices = h.n_slices;
    m->sigma = sigma;
    m->max_width = h.max_width;
    // band of column offsets (the chain kernel's dependency pattern when the
    // offsets are not dictionary-compressible)
    m->dband_lo = m->dband_hi = 0;
    for (int64_t r = 0; r < nrows; ++r)
      for (int64_t q = row_ptr[r]; q < row_ptr[r + 1]; ++q) {
        const int64_t o = col_idx[q] - r;
        m->dband_lo = std::min(m->dband_lo, o);
        m->dband_hi = std::max(m->dband_hi, o);
      }
    try {
      m->slice_ptr = upload(h.slice_ptr.data(), h.slice_ptr.size(), m->bytes);
      m->slice_w = upload(h.slice_w.data(), h.slice_w.size(), m->bytes);
      m->row_len = upload(h.row_len.data(), h.row_len.size(), m->bytes);
      if (sigma > 1) m->perm = upload(h.perm.data(), h.perm.size(), m->bytes);
      m->col = upload(col.data(), (size_t)h.padded, m->bytes);
      m->val = upload(val.data(), (size_t)h.padded, m->bytes);
      build_dictionaries(h, col.data(), val.data(), m);
      if (!m->pair8 && !m->col8 && !m->val8) build_offset_patterns(h, col.data(), m);
      plane_prepare(m);
    } catch (...) {
      free_matrix(m);
      throw;
    }
    *out = m;
  });
}

PG_API int pg_matrix_destroy(pg_matrix* mat) {
  return guard([&] { free_matrix(mat); });
}

PG_API int pg_matrix_stats(const pg_matrix* m, int64_t* s) {
  return guard([&] {
    PG_REQUIRE(m && s, PG_ERR_PARAMETER, "null argument");
    s[0] = m->nrows;
    s[1] = m->ncols;
    s[2] = m->nnz;
    s[3] = m->padded_nnz;
    s[4] = m->n_slices;
    s[5] = (int64_t)m->bytes;
    s[6] = m->max_width;
    s[7] = m->sigma;
    s[8] = m->col8 ? 1 : 4;  // bytes per stored column entry
    s[9] = m->val8 ? 1 : 8;  // bytes per stored value entry
    // the kernel launch_sell picks for 16-byte aligned vectors (spmv.cu)
    int mk;
    int64_t mS, mg;
    s[11] = plane_shape(m) ? 9
            : march_shape(m, &mk, &mS, &mg) ? 8
            : pattern_kernel(m) ? 5
            : (m->pair8 && m->wtab && m->rpat && winpat_enabled()) ? 6
            : opat_kernel(m) ? 7
            : m->pair8 ? (m->wtab ? 3 : (m->stride8 > 0 && m->stride8 <= 256) ? 4 : 2)
                       : (m->col8 || m->val8) ? 1 : 0;
    s[10] = m->pair8 ? 1 : (s[8] + s[9]);
  });
}

PG_API int pg_plane_plan(const pg_matrix* m, int64_t* s) {
  return guard([&] {
    PG_REQUIRE(m && s, PG_ERR_PARAMETER, "null argument");
    const bool on = m->plane_kind != 0;
    s[0] = m->plane_kind;
    s[1] = on ? m->plane.Q : 0;
    s[2] = on ? m->plane.Zc : 0;
    s[3] = on ? m->plane.stages : 0;
    s[4] = on ? m->plane_blocks : 0;
    s[5] = on ? m->plane.H : 0;
    s[6] = !on || !m->plane_qm ? 0 : (m->plane.allbox ? 2 : 1);
    s[7] = on ? m->plane.stage_bytes : 0;
    s[8] = on ? m->plane_sym : 0;
    s[9] = on ? m->plane.vec : 0;
  });
}

PG_API int pg_workspace_create(int device, pg_workspace** out) {
  return guard([&] {
    PG_REQUIRE(out, PG_ERR_PARAMETER, "out is null");
    DeviceScope scope(device);
    pg_workspace* w = new pg_workspace();
    w->device = device;
    PG_CUDA(cudaDeviceGetAttribute(&w->num_sms, cudaDevAttrMultiProcessorCount, device));
    size_t nb = sizeof(double) * (size_t)kMaxBlocks * kMaxOut;
    if (cudaMalloc(&w->partials, nb) != cudaSuccess ||
        cudaMalloc(&w->counter, 64) != cudaSuccess) {
      cudaFree(w->partials);
      delete w;
      throw Error(PG_ERR_ALLOC, "workspace allocation failed");
    }
    PG_CUDA(cudaMemset(w->counter, 0, 64));
    if (cudaMalloc(&w->chain_ctl, 64) != cudaSuccess) {
      cudaFree(w->partials);
      cudaFree(w->counter);
      delete w;
      throw Error(PG_ERR_ALLOC, "workspace allocation failed");
    }
    PG_CUDA(cudaMemset(w->chain_ctl, 0, 64));
    *out = w;
  });
}

PG_API int pg_workspace_destroy(pg_workspace* ws) {
  return guard([&] {
    if (!ws) return;
    DeviceScope scope(ws->device);
    cudaFree(ws->partials);
    cudaFree(ws->counter);
    cudaFree(ws->chain_ctl);
    cudaFree(ws->chain_flags);
    for (int i = 0; i < ws->n_retired; ++i) cudaFree(ws->chain_retired[i]);
    delete ws;
  });
}

}  // extern "C"
