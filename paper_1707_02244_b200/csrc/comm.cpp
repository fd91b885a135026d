// NCCL collectives of the sharded solve, resolved from libnccl.so.2 at run time (comm.hpp).
#include "comm.hpp"

#include <dlfcn.h>

#include <mutex>
#include <string>

#include <nccl.h>

#include "host_common.hpp"

namespace clb {
namespace {

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    // the process may already hold an NCCL (e.g. PyTorch's); dlopen by soname then returns that one
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      n.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (n.h) break;
    }
    if (!n.h) return;
    auto sym = [&](const char* s) { return dlsym(n.h, s); };
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(sym("ncclGetUniqueId"));
    n.init_rank = reinterpret_cast<decltype(n.init_rank)>(sym("ncclCommInitRank"));
    n.init_all = reinterpret_cast<decltype(n.init_all)>(sym("ncclCommInitAll"));
    n.destroy = reinterpret_cast<decltype(n.destroy)>(sym("ncclCommDestroy"));
    n.broadcast = reinterpret_cast<decltype(n.broadcast)>(sym("ncclBroadcast"));
    n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(sym("ncclAllReduce"));
    n.group_start = reinterpret_cast<decltype(n.group_start)>(sym("ncclGroupStart"));
    n.group_end = reinterpret_cast<decltype(n.group_end)>(sym("ncclGroupEnd"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(sym("ncclGetErrorString"));
  });
  if (!n.h || !n.get_unique_id || !n.init_rank || !n.init_all || !n.destroy || !n.broadcast || !n.all_reduce ||
      !n.group_start || !n.group_end || !n.error_string)
    raise(CL_ECOMM, "sharded solve: libnccl.so.2 (NCCL) could not be loaded");
  return n;
}

void check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  raise(CL_ECOMM, std::string(what) + ": " + nccl().error_string(r));
}

}  // namespace

void comm_unique_id(unsigned char id[kCommIdBytes]) {
  ncclUniqueId u;
  check(nccl().get_unique_id(&u), "ncclGetUniqueId");
  for (int i = 0; i < kCommIdBytes; ++i) id[i] = static_cast<unsigned char>(u.internal[i]);
}

Comm* comm_init_rank(const unsigned char id[kCommIdBytes], int world, int rank, int device) {
  if (world < 1 || rank < 0 || rank >= world) raise(CL_EPARAM, "cl_comm_init_rank: need 0 <= rank < world");
  ncclUniqueId u;
  for (int i = 0; i < kCommIdBytes; ++i) u.internal[i] = static_cast<char>(id[i]);
  if (cudaSetDevice(device) != cudaSuccess) raise(CL_ECUDA, "cl_comm_init_rank: no such CUDA device");
  ncclComm_t c = nullptr;
  check(nccl().init_rank(&c, world, u, rank), "ncclCommInitRank");
  Comm* out = new Comm();
  out->nccl = c;
  out->rank = rank;
  out->world = world;
  out->device = device;
  return out;
}

std::vector<Comm*> comm_init_all(const int* devices, int ndev) {
  if (ndev < 1 || !devices) raise(CL_EPARAM, "cl_comm_init_all: need at least one device");
  std::vector<ncclComm_t> cs(static_cast<size_t>(ndev));
  check(nccl().init_all(cs.data(), ndev, devices), "ncclCommInitAll");
  std::vector<Comm*> out;
  for (int r = 0; r < ndev; ++r) {
    Comm* c = new Comm();
    c->nccl = cs[static_cast<size_t>(r)];
    c->rank = r;
    c->world = ndev;
    c->device = devices[r];
    out.push_back(c);
  }
  return out;
}

void comm_destroy(Comm* c) {
  if (!c) return;
  if (c->nccl && c->owned) nccl().destroy(static_cast<ncclComm_t>(c->nccl));
  delete c;
}

void comm_group_start() { check(nccl().group_start(), "ncclGroupStart"); }
void comm_group_end() { check(nccl().group_end(), "ncclGroupEnd"); }

void comm_gather(Comm* c, float* buf, const std::vector<std::pair<int64_t, int64_t>>& ranges, cudaStream_t st) {
  if (c->world == 1) return;
  const Nccl& n = nccl();
  check(n.group_start(), "ncclGroupStart");
  for (int r = 0; r < c->world; ++r) {
    const int64_t lo = ranges[static_cast<size_t>(r)].first, hi = ranges[static_cast<size_t>(r)].second;
    if (hi <= lo) continue;  // every rank skips the same empty slices
    check(n.broadcast(buf + lo, buf + lo, static_cast<size_t>(hi - lo), ncclFloat32, r,
                      static_cast<ncclComm_t>(c->nccl), st),
          "ncclBroadcast");
  }
  check(n.group_end(), "ncclGroupEnd");
}

void comm_allreduce_sum(Comm* c, double* buf, int count, cudaStream_t st) {
  if (c->world == 1) return;
  check(nccl().all_reduce(buf, buf, static_cast<size_t>(count), ncclFloat64, ncclSum,
                          static_cast<ncclComm_t>(c->nccl), st),
        "ncclAllReduce");
}

}  // namespace clb
