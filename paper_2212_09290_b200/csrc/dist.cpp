// SPDX-License-Identifier: Apache-2.0
//
// Multi-GPU from the C / C++ host (one process, or one thread, per GPU):
// xe_ctx = (device, rank, world, NCCL communicator, stream).  The candidate
// sweeps shard with no data-path collective; the only exchange is the
// incumbent, the multi-GPU form of the reference's first-strict-improvement
// rule (proj/src/solver.cpp:57-61):
//   1. all-reduce MIN of the objective's IEEE bits (non-negative doubles
//      order like their bit patterns; "none" = UINT64_MAX),
//   2. all-reduce MIN of the global index over the ranks holding that key,
//   3. all-reduce SUM of the valid counts;
// and, for the search, a broadcast of the winning schedule from the lowest
// rank holding it.  8-byte messages over NVLink / NVSwitch.
//
// NCCL is resolved at xe_ctx_create (dlopen "libnccl.so.2": the copy torch
// already loaded in a Python process, else the system one), so the library
// itself has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <mutex>
#include <vector>

#include "xe_internal.hpp"

namespace xe {
void search_device(const xe_problem* pr, const xe_model_opts& mo, const xe_search_opts& so, xe_search_result* res,
                   uint32_t* cube_host, int64_t* peaks_host, cudaStream_t s);  // search.cu
namespace {

struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
};

const Nccl& nccl() {
  static Nccl api{};
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) {
      void* f = dlsym(h, n);
      if (!f && err.empty()) err = std::string("libnccl.so.2 lacks ") + n;
      return f;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(sym("ncclBroadcast"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  });
  if (!err.empty()) fail(XE_ERR_NCCL, err);
  return api;
}

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(XE_ERR_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

}  // namespace
}  // namespace xe

struct xe_ctx {
  int device = 0, rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  cudaStream_t stream = nullptr;
  xe::DevBuf<uint64_t> buf;  // collective scratch
};

using namespace xe;

namespace {

constexpr uint64_t kNone = std::numeric_limits<uint64_t>::max();

// the three-step incumbent exchange on the context's stream
void exchange(xe_ctx* c, double obj, int64_t global_index, int64_t n_valid, double* gobj, int64_t* gidx,
              int64_t* gvalid) {
  const Nccl& N = nccl();
  uint64_t key = kNone;
  if (global_index >= 0) std::memcpy(&key, &obj, 8);
  uint64_t h[3] = {key, 0, 0};
  XE_CUDA(cudaMemcpyAsync(c->buf.p, h, 8, cudaMemcpyHostToDevice, c->stream));
  nck(N.AllReduce(c->buf.p, c->buf.p, 1, ncclUint64, ncclMin, c->comm, c->stream), "ncclAllReduce(min key)");
  XE_CUDA(cudaMemcpyAsync(h, c->buf.p, 8, cudaMemcpyDeviceToHost, c->stream));
  XE_CUDA(cudaStreamSynchronize(c->stream));
  const uint64_t gkey = h[0];
  h[1] = (global_index >= 0 && key == gkey) ? static_cast<uint64_t>(global_index) : kNone;
  h[2] = static_cast<uint64_t>(n_valid);
  XE_CUDA(cudaMemcpyAsync(c->buf.p + 1, h + 1, 16, cudaMemcpyHostToDevice, c->stream));
  nck(N.AllReduce(c->buf.p + 1, c->buf.p + 1, 1, ncclUint64, ncclMin, c->comm, c->stream), "ncclAllReduce(min index)");
  nck(N.AllReduce(c->buf.p + 2, c->buf.p + 2, 1, ncclUint64, ncclSum, c->comm, c->stream), "ncclAllReduce(sum)");
  XE_CUDA(cudaMemcpyAsync(h + 1, c->buf.p + 1, 16, cudaMemcpyDeviceToHost, c->stream));
  XE_CUDA(cudaStreamSynchronize(c->stream));
  if (gkey == kNone) {
    *gobj = INFINITY;
    *gidx = -1;
  } else {
    std::memcpy(gobj, &gkey, 8);
    *gidx = static_cast<int64_t>(h[1]);
  }
  *gvalid = static_cast<int64_t>(h[2]);
}

}  // namespace

extern "C" int xe_nccl_unique_id(uint8_t* id) {
  return guard([&] {
    if (!id) fail(XE_ERR_ARG, "null argument");
    static_assert(sizeof(ncclUniqueId) == XE_NCCL_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId u;
    nck(nccl().GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof u);
  });
}

extern "C" int xe_ctx_create(int device, int rank, int world, const uint8_t* id, xe_ctx** out) {
  return guard([&] {
    if (!id || !out || world < 1 || rank < 0 || rank >= world) fail(XE_ERR_ARG, "bad context arguments");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) fail(XE_ERR_NO_DEVICE, "no CUDA device");
    XE_CUDA(cudaSetDevice(device));
    auto* c = new xe_ctx;
    c->device = device;
    c->rank = rank;
    c->world = world;
    try {
      XE_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->buf.alloc(4);
      ncclUniqueId u;
      std::memcpy(&u, id, sizeof u);
      nck(nccl().CommInitRank(&c->comm, world, u, rank), "ncclCommInitRank");
    } catch (...) {
      if (c->stream) cudaStreamDestroy(c->stream);
      delete c;
      throw;
    }
    *out = c;
  });
}

extern "C" int xe_ctx_destroy(xe_ctx* c) {
  return guard([&] {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->comm) nccl().CommDestroy(c->comm);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
  });
}

extern "C" int xe_ctx_info(const xe_ctx* c, int32_t* device, int32_t* rank, int32_t* world) {
  return guard([&] {
    if (!c) fail(XE_ERR_ARG, "null argument");
    if (device) *device = c->device;
    if (rank) *rank = c->rank;
    if (world) *world = c->world;
  });
}

extern "C" int xe_ctx_exchange_best(xe_ctx* c, int64_t index_offset, xe_best* best) {
  return guard([&] {
    if (!c || !best) fail(XE_ERR_ARG, "null argument");
    XE_CUDA(cudaSetDevice(c->device));
    double go = 0;
    int64_t gi = -1, gv = 0;
    exchange(c, best->obj, best->index >= 0 ? best->index + index_offset : -1, best->n_valid, &go, &gi, &gv);
    best->obj = go;
    best->index = gi;
    best->n_valid = gv;
  });
}

extern "C" int xe_search_dist(const xe_problem* p, const xe_model_opts* opts, const xe_search_opts* so, xe_ctx* c,
                              xe_search_result* res, uint32_t* cube_host, int64_t* peaks_host) {
  return guard([&] {
    if (!p || !c || !res) fail(XE_ERR_ARG, "null argument");
    require_uploaded(p);
    if (p->device != c->device) fail(XE_ERR_ARG, "problem handle and context on different devices");
    xe_search_opts o;
    xe_search_opts_default(&o);
    if (so) o = *so;
    o.rank = c->rank;
    o.world = c->world;
    xe_model_opts mo{};
    if (opts) mo = *opts;
    const HostProblem& h = p->h;
    const size_t words = xe_cube_bytes(h.D, h.T) / 4;
    std::vector<uint32_t> cube(words, 0);
    std::vector<int64_t> peaks(static_cast<size_t>(h.D), 0);
    search_device(p, mo, o, res, cube.data(), peaks.data(), c->stream);
    if (c->world > 1) {
      // rounding incumbent: the global first minimum over the interleaved blocks
      double ro = 0;
      int64_t ri = -1, nv = 0;
      exchange(c, res->rounding_objective, res->index, res->n_valid, &ro, &ri, &nv);
      // final schedule: the best objective over ranks, lowest rank on ties
      double wo = 0;
      int64_t wr = -1, unused = 0;
      exchange(c, res->objective, std::isfinite(res->objective) ? c->rank : -1, 0, &wo, &wr, &unused);
      const Nccl& N = nccl();
      // totals: evaluated candidates, improvements, time-limited flag
      uint64_t t[3] = {static_cast<uint64_t>(res->n_evaluated), static_cast<uint64_t>(res->improvements),
                       static_cast<uint64_t>(res->time_limited)};
      XE_CUDA(cudaMemcpyAsync(c->buf.p, t, 24, cudaMemcpyHostToDevice, c->stream));
      nck(N.AllReduce(c->buf.p, c->buf.p, 2, ncclUint64, ncclSum, c->comm, c->stream), "ncclAllReduce(totals)");
      nck(N.AllReduce(c->buf.p + 2, c->buf.p + 2, 1, ncclUint64, ncclMax, c->comm, c->stream), "ncclAllReduce(limit)");
      XE_CUDA(cudaMemcpyAsync(t, c->buf.p, 24, cudaMemcpyDeviceToHost, c->stream));
      XE_CUDA(cudaStreamSynchronize(c->stream));
      res->n_evaluated = static_cast<int64_t>(t[0]);
      res->improvements = static_cast<int32_t>(t[1]);
      res->time_limited = static_cast<int32_t>(t[2]);
      res->rounding_objective = ro;
      res->index = ri;
      res->n_valid = nv;
      // the rank holding the global rounding incumbent (its schedule wins ties:
      // the local search replaces an incumbent only when strictly better)
      double oo = 0;
      int64_t owner = -1, unused2 = 0;
      const bool mine = ri >= 0 && res->index == ri;
      exchange(c, 0.0, mine ? c->rank : -1, 0, &oo, &owner, &unused2);
      res->objective = std::min(wo, ro);
      const int64_t src = (ri < 0 || wo < ro) ? wr : owner;
      wr = src;
      if (wr >= 0) {  // broadcast the winner's schedule and peaks
        DevBuf<uint32_t> b;
        b.alloc(words + 2 * static_cast<size_t>(h.D));
        XE_CUDA(cudaMemcpyAsync(b.p, cube.data(), words * 4, cudaMemcpyHostToDevice, c->stream));
        XE_CUDA(cudaMemcpyAsync(b.p + words, peaks.data(), h.D * 8, cudaMemcpyHostToDevice, c->stream));
        nck(N.Broadcast(b.p, b.p, words + 2 * h.D, ncclUint32, static_cast<int>(wr), c->comm, c->stream),
            "ncclBroadcast(winner)");
        XE_CUDA(cudaMemcpyAsync(cube.data(), b.p, words * 4, cudaMemcpyDeviceToHost, c->stream));
        XE_CUDA(cudaMemcpyAsync(peaks.data(), b.p + words, h.D * 8, cudaMemcpyDeviceToHost, c->stream));
        XE_CUDA(cudaStreamSynchronize(c->stream));
      }
    }
    if (cube_host) std::memcpy(cube_host, cube.data(), words * 4);
    if (peaks_host) std::memcpy(peaks_host, peaks.data(), h.D * 8);
  });
}
