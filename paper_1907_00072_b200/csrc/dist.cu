// Row-block shards across GPUs (SURVEY §8 row e), issued natively: the halo
// exchange before every SpMV pass and the batched reductions of CGS2 run as
// NCCL operations launched from C on the solve's stream, inside the same
// native call (or recorded CUDA graph) as the step's kernels -- O(1) host
// calls per device per Arnoldi step, like the single-GPU path.
//
//  * halo: the owned rows other shards read are packed by one gather kernel
//    into a send buffer; one NCCL group of ncclSend / ncclRecv then moves every
//    neighbour's block straight into the ghost slots of the vector (ghost
//    columns are grouped by owner, so each receive is one contiguous range).
//  * reductions: every rank's partials are all-gathered ([P][count]) and summed
//    in rank order by one small kernel -- ((b0 + b1) + b2) + ..., the order of
//    the in-process SoloComm -- so the result is the same on every rank, does
//    not depend on NCCL's algorithm choice, and equals the virtual-shard run
//    bit for bit.
//
// libnccl is opened at run time (dlopen; the copy torch already loaded is
// reused), so libpgmres has no link-time NCCL dependency.

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>
#include <vector>

#include "internal.cuh"

namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
};

const NcclApi& nccl() {
  static NcclApi api;
  static bool loaded = false;
  if (loaded) return api;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  PG_REQUIRE(h, PG_ERR_CUDA, "libnccl.so.2 not found (import torch first, or set LD_LIBRARY_PATH)");
  auto sym = [&](const char* name) {
    void* f = dlsym(h, name);
    PG_REQUIRE(f, PG_ERR_CUDA, std::string("libnccl lacks ") + name);
    return f;
  };
  api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
  api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
  api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
  api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
  api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
  api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
  api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
  api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
  api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  loaded = true;
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw pg::Error(PG_ERR_CUDA, std::string(what) + ": " + nccl().GetErrorString(r));
}

}  // namespace

struct pg_dist {
  int device, nranks, rank;
  ncclComm_t comm;
  // halo plan: sends (peer, count) over the packed buffer, receives (peer,
  // ghost offset, count); send_idx = local rows to pack, in send order
  std::vector<int> send_peer, recv_peer;
  std::vector<int64_t> send_count, send_off, recv_off, recv_count;
  int32_t* d_send_idx = nullptr;
  double* d_send_buf = nullptr;
  int64_t send_total = 0;
  // reduction scratch: [nranks][count], count <= 2*PG_MMAX + 8
  double* d_gather = nullptr;
};

namespace pg {

constexpr int kRedMax = 2 * PG_MMAX + 8;

__global__ void rank_sum_kernel(const double* __restrict__ parts, int nranks, int count,
                                double* out) {
  pdl_entry();
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    double s = parts[i];
    for (int r = 1; r < nranks; ++r) s = __dadd_rn(s, parts[(int64_t)r * count + i]);
    out[i] = s;
  }
}

__global__ void pack_kernel(const double* __restrict__ x, const int32_t* __restrict__ idx,
                            int64_t m, double* __restrict__ out) {
  pdl_entry();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = x[idx[i]];
}

void dist_halo(pg_dist* d, double* x, cudaStream_t st) {
  if (!d || (d->send_peer.empty() && d->recv_peer.empty())) return;
  const NcclApi& api = nccl();
  if (d->send_total > 0) {
    const int g = (int)std::min<int64_t>((d->send_total + 255) / 256, 1024);
    launch_k(pack_kernel, g, 256, 0, st, (const double*)x, (const int32_t*)d->d_send_idx,
             d->send_total, d->d_send_buf);
    check_launch();
  }
  nccl_check(api.GroupStart(), "ncclGroupStart");
  for (size_t i = 0; i < d->send_peer.size(); ++i)
    nccl_check(api.Send(d->d_send_buf + d->send_off[i], (size_t)d->send_count[i], ncclDouble,
                        d->send_peer[i], d->comm, st),
               "ncclSend");
  for (size_t i = 0; i < d->recv_peer.size(); ++i)
    nccl_check(api.Recv(x + d->recv_off[i], (size_t)d->recv_count[i], ncclDouble, d->recv_peer[i],
                        d->comm, st),
               "ncclRecv");
  nccl_check(api.GroupEnd(), "ncclGroupEnd");
}

void dist_allreduce(pg_dist* d, double* buf, int count, cudaStream_t st) {
  if (!d || count <= 0) return;
  PG_REQUIRE(count <= kRedMax, PG_ERR_PARAMETER, "reduction longer than the scratch");
  // own contribution into its rank slot, gather every rank's, ordered sum
  nccl_check(nccl().AllGather(buf, d->d_gather, (size_t)count, ncclDouble, d->comm, st),
             "ncclAllGather");
  launch_k(rank_sum_kernel, 1, 128, 0, st, (const double*)d->d_gather, d->nranks, count, buf);
  check_launch();
}

}  // namespace pg

using namespace pg;

extern "C" {

PG_API int pg_nccl_unique_id(void* out, size_t len) {
  return guard([&] {
    PG_REQUIRE(out && len >= sizeof(ncclUniqueId), PG_ERR_PARAMETER, "buffer too small");
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof id);
  });
}

PG_API int pg_dist_create(const void* uid, int nranks, int rank, int device, pg_dist** out) {
  return guard([&] {
    PG_REQUIRE(uid && out && nranks >= 1 && rank >= 0 && rank < nranks, PG_ERR_PARAMETER,
               "bad communicator arguments");
    *out = nullptr;
    DeviceScope scope(device);
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof id);
    pg_dist* d = new pg_dist();
    d->device = device;
    d->nranks = nranks;
    d->rank = rank;
    const ncclResult_t r = nccl().CommInitRank(&d->comm, nranks, id, rank);
    if (r != ncclSuccess) {
      delete d;
      nccl_check(r, "ncclCommInitRank");
    }
    if (cudaMalloc(&d->d_gather, sizeof(double) * kRedMax * nranks) != cudaSuccess) {
      nccl().CommDestroy(d->comm);
      delete d;
      throw Error(PG_ERR_ALLOC, "reduction scratch");
    }
    cudaMemset(d->d_gather, 0, sizeof(double) * kRedMax * nranks);
    *out = d;
  });
}

PG_API int pg_dist_set_halo(pg_dist* d, int nsend, const int* send_peer,
                            const int64_t* send_count, const int32_t* send_idx, int nrecv,
                            const int* recv_peer, const int64_t* recv_off,
                            const int64_t* recv_count) {
  return guard([&] {
    PG_REQUIRE(d && nsend >= 0 && nrecv >= 0, PG_ERR_PARAMETER, "bad halo plan");
    DeviceScope scope(d->device);
    cudaFree(d->d_send_idx);
    cudaFree(d->d_send_buf);
    d->d_send_idx = nullptr;
    d->d_send_buf = nullptr;
    d->send_peer.assign(send_peer, send_peer + nsend);
    d->send_count.assign(send_count, send_count + nsend);
    d->send_off.assign(nsend, 0);
    int64_t tot = 0;
    for (int i = 0; i < nsend; ++i) {
      PG_REQUIRE(send_peer[i] >= 0 && send_peer[i] < d->nranks && send_count[i] >= 0,
                 PG_ERR_PARAMETER, "bad send peer");
      d->send_off[i] = tot;
      tot += send_count[i];
    }
    d->send_total = tot;
    d->recv_peer.assign(recv_peer, recv_peer + nrecv);
    d->recv_off.assign(recv_off, recv_off + nrecv);
    d->recv_count.assign(recv_count, recv_count + nrecv);
    for (int i = 0; i < nrecv; ++i)
      PG_REQUIRE(recv_peer[i] >= 0 && recv_peer[i] < d->nranks && recv_off[i] >= 0 &&
                     recv_count[i] >= 0,
                 PG_ERR_PARAMETER, "bad receive peer");
    if (tot > 0) {
      PG_REQUIRE(send_idx, PG_ERR_PARAMETER, "send indices required");
      PG_CUDA(cudaMalloc(&d->d_send_idx, sizeof(int32_t) * tot));
      PG_CUDA(cudaMalloc(&d->d_send_buf, sizeof(double) * tot));
      PG_CUDA(cudaMemcpy(d->d_send_idx, send_idx, sizeof(int32_t) * tot, cudaMemcpyHostToDevice));
    }
  });
}

PG_API int pg_dist_destroy(pg_dist* d) {
  return guard([&] {
    if (!d) return;
    DeviceScope scope(d->device);
    cudaFree(d->d_send_idx);
    cudaFree(d->d_send_buf);
    cudaFree(d->d_gather);
    if (d->comm) nccl().CommDestroy(d->comm);
    delete d;
  });
}

PG_API int pg_dist_halo(pg_dist* d, double* d_x, void* stream) {
  return guard([&] {
    PG_REQUIRE(d && d_x, PG_ERR_PARAMETER, "null argument");
    dist_halo(d, d_x, as_stream(stream));
  });
}

PG_API int pg_dist_allreduce(pg_dist* d, double* d_buf, int count, void* stream) {
  return guard([&] {
    PG_REQUIRE(d && d_buf, PG_ERR_PARAMETER, "null argument");
    dist_allreduce(d, d_buf, count, as_stream(stream));
  });
}

}  // extern "C"
