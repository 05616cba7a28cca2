// libpgmres: whole Arnoldi steps and polynomial chains as single host calls.
//
// The Python solver used to issue every kernel of an Arnoldi step (d fused
// passes, the wrapper SpMV, three CGS2 phases, the normalisation, the copy of
// the step's scalars to pinned memory) through ctypes: ~20 calls and ~0.2 ms
// of interpreter time per step, about half the GPU time of a cfg2 step, so the
// one-step look-ahead had little slack.  pg_arnoldi_step / pg_poly_chain do
// the same launches in C++ (same kernels, same order, same arguments as the
// per-kernel entry points: results are bit-identical), one call per step.

#include <cstdlib>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "internal.cuh"

struct pg_event {
  cudaEvent_t ev;
  int device;
};

namespace {

// a nested entry point failed: keep its status and its message
void ok(int code) {
  if (code != PG_OK) {
    char msg[512];
    pg_last_error(msg, sizeof msg);
    throw pg::Error(code, msg);
  }
}

// d fused monomial passes, out = (base +) p(A) x  (Engine.poly); with a
// distributed shard (dist) the ghost slots of each pass's operand are filled
// first (dist.cu; x itself must already hold its ghosts)
void poly_chain(const pg_matrix* m, const double* y, int d, const double* x, const double* base,
                double* out, double* acc, double* w0, double* w1, void* st,
                pg_dist* dist = nullptr) {
  if (d == 0) {
    ok(pg_scale_add(base, y[0], x, m->nrows, out, st));
    return;
  }
  const double* cur = x;
  double* ws[2] = {w0, w1};
  for (int k = 1; k <= d; ++k) {
    const bool last = k == d;
    const int flags = (k == 1 ? PG_PASS_FIRST : 0) | (last ? 0 : PG_PASS_WRITE_W);
    double* nxt = ws[k & 1];
    if (k > 1) pg::dist_halo(dist, const_cast<double*>(cur), pg::as_stream(st));
    ok(pg_poly_pass(m, cur, k > 1 ? acc : nullptr, last ? base : nullptr, last ? out : acc,
                    last ? nullptr : nxt, y[0], y[k], flags, st));
    cur = nxt;
  }
}

// The passes poly_chain issues, as chain steps (same buffers and flags).
std::vector<pg::ChainStep> poly_steps(const double* y, int d, const double* x, const double* base,
                                      double* out, double* acc, double* w0, double* w1) {
  std::vector<pg::ChainStep> v;
  const double* cur = x;
  double* ws[2] = {w0, w1};
  for (int k = 1; k <= d; ++k) {
    const bool last = k == d;
    const int flags = (k == 1 ? PG_PASS_FIRST : 0) | (last ? 0 : PG_PASS_WRITE_W);
    double* nxt = ws[k & 1];
    v.push_back(pg::ChainStep{pg::PG_CHAIN_POLY, cur, k > 1 ? acc : nullptr, last ? base : nullptr,
                              last ? out : acc, last ? nullptr : nxt, y[0], y[k], flags, 0.0, 0.0,
                              0.0});
    cur = nxt;
  }
  return v;
}

void record(pg_event* e, void* st) {
  if (!e) return;
  // inside a capture only an "external" record becomes a graph node that
  // re-records the event at every replay
  if (pg::g_capturing)
    PG_CUDA(cudaEventRecordWithFlags(e->ev, pg::as_stream(st), cudaEventRecordExternal));
  else
    PG_CUDA(cudaEventRecord(e->ev, pg::as_stream(st)));
}

}  // namespace

using namespace pg;

extern "C" {

PG_API int pg_event_create(int device, pg_event** out) {
  return guard([&] {
    PG_REQUIRE(out, PG_ERR_PARAMETER, "out is null");
    int prev = 0;
    PG_CUDA(cudaGetDevice(&prev));
    PG_CUDA(cudaSetDevice(device));
    pg_event* e = new pg_event();
    e->device = device;
    const cudaError_t rc = cudaEventCreate(&e->ev);
    cudaSetDevice(prev);
    if (rc != cudaSuccess) {
      delete e;
      throw Error(PG_ERR_CUDA, std::string("cudaEventCreate: ") + cudaGetErrorString(rc));
    }
    *out = e;
  });
}

PG_API int pg_event_destroy(pg_event* e) {
  return guard([&] {
    if (!e) return;
    cudaEventDestroy(e->ev);
    delete e;
  });
}

PG_API int pg_event_record(pg_event* e, void* stream) {
  return guard([&] {
    PG_REQUIRE(e, PG_ERR_PARAMETER, "event is null");
    record(e, stream);
  });
}

PG_API int pg_event_wait(pg_event* e) {
  return guard([&] {
    PG_REQUIRE(e, PG_ERR_PARAMETER, "event is null");
    PG_CUDA(cudaEventSynchronize(e->ev));
  });
}

PG_API int pg_event_elapsed(pg_event* start, pg_event* end, float* ms) {
  return guard([&] {
    PG_REQUIRE(start && end && ms, PG_ERR_PARAMETER, "null argument");
    PG_CUDA(cudaEventElapsedTime(ms, start->ev, end->ev));
  });
}

PG_API int pg_wrapped_apply(const pg_matrix* mat, const double* y, int d, const double* d_x,
                            double* d_t, double* d_z, double* d_acc, double* d_w0, double* d_w1,
                            pg_workspace* ws, void* stream) {
  return guard([&] {
    PG_REQUIRE(mat && y && d_x && d_t && d_z && d > 0 && d_acc && d_w0 && d_w1, PG_ERR_PARAMETER,
               "null argument");
    std::vector<ChainStep> steps = poly_steps(y, d, d_x, nullptr, d_t, d_acc, d_w0, d_w1);
    steps.push_back(ChainStep{PG_CHAIN_SPMV, d_t, nullptr, nullptr, d_z, nullptr, 0.0, 0.0, 0,
                              0.0, 0.0, 0.0});
    if (!chain_launch(mat, steps.data(), (int)steps.size(), ws, as_stream(stream))) {
      poly_chain(mat, y, d, d_x, nullptr, d_t, d_acc, d_w0, d_w1, stream);
      ok(pg_spmv(mat, d_t, d_z, stream));
    }
  });
}

PG_API int pg_power_sequence(const pg_matrix* mat, double* d_P, int64_t ld, int ncols,
                             void* stream) {
  return guard([&] {
    PG_REQUIRE(mat && d_P && ncols >= 1 && ld >= mat->ncols, PG_ERR_PARAMETER,
               "bad power-sequence arguments");
    for (int k = 1; k < ncols; ++k)
      ok(pg_spmv(mat, d_P + (int64_t)(k - 1) * ld, d_P + (int64_t)k * ld, stream));
  });
}

PG_API int pg_poly_chain(const pg_matrix* mat, const double* y, int d, const double* d_x,
                         const double* d_base, double* d_out, double* d_acc, double* d_w0,
                         double* d_w1, pg_event* ev_start, pg_event* ev_end, void* stream) {
  return guard([&] {
    PG_REQUIRE(mat && y && d_x && d_out && d >= 0, PG_ERR_PARAMETER, "null argument");
    PG_REQUIRE(d == 0 || (d_acc && d_w0 && d_w1), PG_ERR_PARAMETER, "scratch vectors required");
    record(ev_start, stream);
    poly_chain(mat, y, d, d_x, d_base, d_out, d_acc, d_w0, d_w1, stream);
    record(ev_end, stream);
  });
}

}  // extern "C"

namespace {

// z = A p(A) v = v - pi(A) v in root-product form (Engine.wrapped_roots):
// the plan's passes carry only the product; PAIR_A writes the pair
// temporary t, REAL / PAIR_B the next product (ping-pong w0 / w1), the
// PG_ROOT_RESID pass writes z.
void roots_chain(const pg_matrix* m, int nroot, const int* rmode, const double* rc,
                 const double* v, double* z, double* t, double* w0, double* w1, void* st,
                 pg_dist* dist = nullptr) {
  const double* prod = v;
  double* bufs[2] = {w0, w1};
  int nb = 0;
  for (int q = 0; q < nroot; ++q) {
    const int mode = rmode[q], kind = mode & 3;
    const bool resid = (mode & PG_ROOT_RESID) != 0;
    const double* x = kind == PG_ROOT_PAIR_B ? t : prod;
    if (q > 0) pg::dist_halo(dist, const_cast<double*>(x), pg::as_stream(st));
    const double* p = kind == PG_ROOT_PAIR_B ? prod : nullptr;
    double* w = resid ? z : (kind == PG_ROOT_PAIR_A ? t : bufs[nb]);
    ok(pg_root_pass(m, x, p, resid ? v : nullptr, nullptr, w, rc[3 * q], rc[3 * q + 1],
                    rc[3 * q + 2], mode, st));
    if (!resid && kind != PG_ROOT_PAIR_A) {
      prod = w;
      nb ^= 1;
    }
  }
}

// Device address of a pinned host buffer (UVA mapping), cached per buffer;
// nullptr when the buffer is not mapped, inside a graph capture before the
// buffer was seen (no API call while capturing), or with PG_PUBLISH=0.
double* mapped_host(double* h) {
  static std::mutex mu;
  static std::unordered_map<void*, void*> cache;
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("PG_PUBLISH");
    on = e ? std::atoi(e) != 0 : 1;
  }
  if (!on || !h) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(h);
  if (it != cache.end()) return static_cast<double*>(it->second);
  if (pg::g_capturing) return nullptr;
  void* d = nullptr;
  if (cudaHostGetDevicePointer(&d, h, 0) != cudaSuccess) {
    cudaGetLastError();  // not mapped: clear the error, use the copy
    d = nullptr;
  }
  cache.emplace(h, d);
  return static_cast<double*>(d);
}

// The passes roots_chain issues, as chain steps.
std::vector<ChainStep> roots_steps(int nroot, const int* rmode, const double* rc, const double* v,
                                   double* z, double* t, double* w0, double* w1) {
  std::vector<ChainStep> out;
  const double* prod = v;
  double* bufs[2] = {w0, w1};
  int nb = 0;
  for (int q = 0; q < nroot; ++q) {
    const int mode = rmode[q], kind = mode & 3;
    const bool resid = (mode & PG_ROOT_RESID) != 0;
    PG_REQUIRE((mode & ~(3 | PG_ROOT_RESID)) == 0 && kind <= PG_ROOT_PAIR_B &&
                   !(resid && kind == PG_ROOT_PAIR_A),
               PG_ERR_PARAMETER, "unknown root-pass mode");
    const double* x = kind == PG_ROOT_PAIR_B ? t : prod;
    const double* p = kind == PG_ROOT_PAIR_B ? prod : nullptr;
    double* w = resid ? z : (kind == PG_ROOT_PAIR_A ? t : bufs[nb]);
    out.push_back(ChainStep{PG_CHAIN_ROOT, x, resid ? v : nullptr, p, nullptr, w, 0.0, 0.0, mode,
                            rc[3 * q], rc[3 * q + 1], rc[3 * q + 2]});
    if (!resid && kind != PG_ROOT_PAIR_A) {
      prod = w;
      nb ^= 1;
    }
  }
  return out;
}

void arnoldi_step_body(const pg_matrix* mat, const double* y, int d, double* d_V, int64_t ld,
                       int j, double* d_z, double* d_t, double* d_acc, double* d_w0,
                       double* d_w1, double* d_ring, double* h_ring, pg_workspace* ws,
                       pg_event* ev_done, pg_event* ev_chain0, pg_event* ev_chain1,
                       int nroot, const int* rmode, const double* rc, void* stream,
                       pg_dist* dist = nullptr) {
    cudaStream_t cst = as_stream(stream);
    PG_REQUIRE(mat && d_V && d_z && d_ring && h_ring && ws && ev_done, PG_ERR_PARAMETER,
               "null argument");
    const int k = j + 1;
    PG_REQUIRE(j >= 0 && k < PG_MMAX && ld >= mat->ncols, PG_ERR_PARAMETER,
               "step index out of range");
    const int64_t n = mat->nrows;
    const double* vj = d_V + (int64_t)j * ld;
    // the operand's ghost slots (distributed shards; no-op otherwise)
    dist_halo(dist, const_cast<double*>(vj), cst);
    // z = A p(A) v_j  (gmres.py:112-113, 283), or z = A v_j without a polynomial
    if (nroot > 0) {
      PG_REQUIRE(rmode && rc && d_acc && d_w0 && d_w1, PG_ERR_PARAMETER,
                 "root plan needs its scratch vectors");
      record(ev_chain0, stream);
      std::vector<ChainStep> steps = roots_steps(nroot, rmode, rc, vj, d_z, d_acc, d_w0, d_w1);
      if (dist || !chain_launch(mat, steps.data(), nroot, ws, cst))
        roots_chain(mat, nroot, rmode, rc, vj, d_z, d_acc, d_w0, d_w1, stream, dist);
      record(ev_chain1, stream);
    } else if (d >= 0) {
      PG_REQUIRE(y && d_t, PG_ERR_PARAMETER, "polynomial step needs y and t");
      record(ev_chain0, stream);
      // the d passes and the wrapper SpMV as one dependency-driven kernel
      // (chain.cu) when the matrix format allows; ev_chain1 then also covers
      // the wrapper pass (pg_chain_fused)
      std::vector<ChainStep> steps = poly_steps(y, d, vj, nullptr, d_t, d_acc, d_w0, d_w1);
      steps.push_back(ChainStep{PG_CHAIN_SPMV, d_t, nullptr, nullptr, d_z, nullptr, 0.0, 0.0, 0,
                                0.0, 0.0, 0.0});
      if (!dist && d > 0 && chain_launch(mat, steps.data(), (int)steps.size(), ws, cst)) {
        record(ev_chain1, stream);
      } else {
        poly_chain(mat, y, d, vj, nullptr, d_t, d_acc, d_w0, d_w1, stream, dist);
        record(ev_chain1, stream);
        dist_halo(dist, d_t, cst);
        ok(pg_spmv(mat, d_t, d_z, stream));
      }
    } else {
      ok(pg_spmv(mat, vj, d_z, stream));
    }
    // CGS2 against v_0..v_{k-1}; w2/|w2| into column k (ortho.py:53-70).  The
    // step's scalars are packed [c1 (k) | c2 (k) | nsq] at the ring's start.
    double* c1 = d_ring;
    double* c2 = d_ring + k;
    double* nsq = d_ring + 2 * k;
    double* col = d_V + (int64_t)k * ld;
    if (k <= PG_KMAX) {
      // distributed: one batched reduction per phase (all-gather + rank-order sum)
      ok(pg_cgs2_phase1(d_V, ld, k, d_z, n, c1, ws, stream));
      dist_allreduce(dist, c1, k, cst);
      ok(pg_cgs2_phase2(d_V, ld, k, d_z, n, c1, c2, ws, stream));
      dist_allreduce(dist, c2, k, cst);
      ok(pg_cgs2_phase3(d_V, ld, k, d_z, n, c1, c2, col, nsq, ws, stream));
      dist_allreduce(dist, nsq, 1, cst);
    } else {
      // wider than one tile: w1 into t (free once the wrapper SpMV has read it)
      PG_REQUIRE(d_t, PG_ERR_PARAMETER, "a basis wider than PG_KMAX needs the t scratch");
      cgs2_wide(d_V, ld, k, d_z, n, c1, c2, nsq, d_t, col, ws, dist, cst);
    }
    // normalise into column k and publish the scalars straight into the
    // pinned host ring (no copy-engine transfer between steps), or copy them
    double* h_dev = mapped_host(h_ring);
    if (h_dev) {
      normalize_publish(col, nsq, n, col, d_ring, 2 * k + 1, h_dev, cst);
    } else {
      ok(pg_normalize(col, nsq, n, col, stream));
      PG_CUDA(cudaMemcpyAsync(h_ring, d_ring, sizeof(double) * (2 * k + 1),
                              cudaMemcpyDeviceToHost, cst));
    }
    record(ev_done, stream);
}

}  // namespace

struct pg_graph {
  cudaGraphExec_t exec;
  int device;
};

namespace {

// Record body(stream) into an instantiated graph: stream capture on a private
// stream; launches inside carry plain edges, event records become external
// nodes (record()), NCCL operations are captured like kernels.
template <class Body>
void capture_step(const pg_matrix* mat, pg_graph** out, Body body) {
  PG_REQUIRE(out && mat, PG_ERR_PARAMETER, "null argument");
  *out = nullptr;
  int prev = 0;
  PG_CUDA(cudaGetDevice(&prev));
  PG_CUDA(cudaSetDevice(mat->device));
  cudaStream_t cs = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaError_t err = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  if (err == cudaSuccess) err = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
  if (err != cudaSuccess) {
    if (cs) cudaStreamDestroy(cs);
    cudaSetDevice(prev);
    throw Error(PG_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(err));
  }
  g_capturing = true;
  try {
    body(static_cast<void*>(cs));
  } catch (...) {
    g_capturing = false;
    cudaStreamEndCapture(cs, &graph);
    if (graph) cudaGraphDestroy(graph);
    cudaStreamDestroy(cs);
    cudaSetDevice(prev);
    throw;
  }
  g_capturing = false;
  err = cudaStreamEndCapture(cs, &graph);
  if (err == cudaSuccess) err = cudaGraphInstantiate(&exec, graph, 0);
  if (graph) cudaGraphDestroy(graph);
  cudaStreamDestroy(cs);
  cudaSetDevice(prev);
  if (err != cudaSuccess)
    throw Error(PG_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(err));
  *out = new pg_graph{exec, mat->device};
}

}  // namespace

extern "C" {

PG_API int pg_arnoldi_step(const pg_matrix* mat, const double* y, int d, double* d_V, int64_t ld,
                           int j, double* d_z, double* d_t, double* d_acc, double* d_w0,
                           double* d_w1, double* d_ring, double* h_ring, pg_workspace* ws,
                           pg_event* ev_done, pg_event* ev_chain0, pg_event* ev_chain1,
                           int nroot, const int* rmode, const double* rc, void* stream) {
  return guard([&] {
    arnoldi_step_body(mat, y, d, d_V, ld, j, d_z, d_t, d_acc, d_w0, d_w1, d_ring, h_ring, ws,
                      ev_done, ev_chain0, ev_chain1, nroot, rmode, rc, stream);
  });
}

PG_API int pg_step_graph_create(const pg_matrix* mat, const double* y, int d, double* d_V,
                                int64_t ld, int j, double* d_z, double* d_t, double* d_acc,
                                double* d_w0, double* d_w1, double* d_ring, double* h_ring,
                                pg_workspace* ws, pg_event* ev_done, pg_event* ev_chain0,
                                pg_event* ev_chain1, int nroot, const int* rmode,
                                const double* rc, pg_graph** out) {
  return guard([&] {
    capture_step(mat, out, [&](void* cs) {
      arnoldi_step_body(mat, y, d, d_V, ld, j, d_z, d_t, d_acc, d_w0, d_w1, d_ring, h_ring, ws,
                        ev_done, ev_chain0, ev_chain1, nroot, rmode, rc, cs);
    });
  });
}

PG_API int pg_graph_launch(pg_graph* g, void* stream) {
  return guard([&] {
    PG_REQUIRE(g, PG_ERR_PARAMETER, "graph is null");
    PG_CUDA(cudaGraphLaunch(g->exec, as_stream(stream)));
  });
}

PG_API int pg_graph_destroy(pg_graph* g) {
  return guard([&] {
    if (!g) return;
    cudaGraphExecDestroy(g->exec);
    delete g;
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Distributed shards (dist.cu): the same calls with the halo exchanges and the
// batched CGS2 reductions issued in between, on the same stream.
// ---------------------------------------------------------------------------
extern "C" {

PG_API int pg_arnoldi_step_dist(const pg_matrix* mat, const double* y, int d, double* d_V,
                                int64_t ld, int j, double* d_z, double* d_t, double* d_acc,
                                double* d_w0, double* d_w1, double* d_ring, double* h_ring,
                                pg_workspace* ws, pg_event* ev_done, pg_event* ev_chain0,
                                pg_event* ev_chain1, int nroot, const int* rmode, const double* rc,
                                pg_dist* dist, void* stream) {
  return guard([&] {
    PG_REQUIRE(dist, PG_ERR_PARAMETER, "communicator is null");
    arnoldi_step_body(mat, y, d, d_V, ld, j, d_z, d_t, d_acc, d_w0, d_w1, d_ring, h_ring, ws,
                      ev_done, ev_chain0, ev_chain1, nroot, rmode, rc, stream, dist);
  });
}

PG_API int pg_step_graph_create_dist(const pg_matrix* mat, const double* y, int d, double* d_V,
                                     int64_t ld, int j, double* d_z, double* d_t, double* d_acc,
                                     double* d_w0, double* d_w1, double* d_ring, double* h_ring,
                                     pg_workspace* ws, pg_event* ev_done, pg_event* ev_chain0,
                                     pg_event* ev_chain1, int nroot, const int* rmode,
                                     const double* rc, pg_dist* dist, pg_graph** out) {
  return guard([&] {
    PG_REQUIRE(dist, PG_ERR_PARAMETER, "communicator is null");
    capture_step(mat, out, [&](void* cs) {
      arnoldi_step_body(mat, y, d, d_V, ld, j, d_z, d_t, d_acc, d_w0, d_w1, d_ring, h_ring, ws,
                        ev_done, ev_chain0, ev_chain1, nroot, rmode, rc, cs, dist);
    });
  });
}

PG_API int pg_poly_chain_dist(const pg_matrix* mat, const double* y, int d, double* d_x,
                              const double* d_base, double* d_out, double* d_acc, double* d_w0,
                              double* d_w1, pg_event* ev_start, pg_event* ev_end, pg_dist* dist,
                              void* stream) {
  return guard([&] {
    PG_REQUIRE(mat && y && d_x && d_out && d >= 0 && dist, PG_ERR_PARAMETER, "null argument");
    PG_REQUIRE(d == 0 || (d_acc && d_w0 && d_w1), PG_ERR_PARAMETER, "scratch vectors required");
    record(ev_start, stream);
    if (d > 0) dist_halo(dist, d_x, as_stream(stream));
    poly_chain(mat, y, d, d_x, d_base, d_out, d_acc, d_w0, d_w1, stream, dist);
    record(ev_end, stream);
  });
}

PG_API int pg_power_sequence_dist(const pg_matrix* mat, double* d_P, int64_t ld, int ncols,
                                  pg_dist* dist, void* stream) {
  return guard([&] {
    PG_REQUIRE(mat && d_P && ncols >= 1 && ld >= mat->ncols && dist, PG_ERR_PARAMETER,
               "bad power-sequence arguments");
    for (int k = 1; k < ncols; ++k) {
      double* src = d_P + (int64_t)(k - 1) * ld;
      dist_halo(dist, src, as_stream(stream));
      ok(pg_spmv(mat, src, d_P + (int64_t)k * ld, stream));
    }
  });
}

}  // extern "C"
