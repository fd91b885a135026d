// Collectives of the sharded solve: NCCL, loaded at run time.
//
// Shard g of G owns contiguous slices of the vectors each phase produces; between phases every rank
// receives every other rank's slice in place (an all-gather of unequal slices: one ncclBroadcast per
// owner, rooted at it, send buffer == receive buffer, grouped).  The check metrics are summed with one
// ncclAllReduce of three doubles.  No reduction touches the iterate, so results are bitwise identical
// for every G.
//
// libnccl.so.2 is opened with dlopen on first use, so the library itself loads (and every unsharded
// solve runs) on machines without NCCL; a sharded solve without it fails with CL_ECOMM.
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include <cuda_runtime.h>

namespace clb {

constexpr int kCommIdBytes = 128;  // NCCL_UNIQUE_ID_BYTES

struct Comm {
  void* nccl = nullptr;  // ncclComm_t
  int rank = 0, world = 1, device = 0;
  bool owned = true;
};

// All raise CL_ECOMM with NCCL's message on failure.
void comm_unique_id(unsigned char id[kCommIdBytes]);
Comm* comm_init_rank(const unsigned char id[kCommIdBytes], int world, int rank, int device);
std::vector<Comm*> comm_init_all(const int* devices, int ndev);
void comm_destroy(Comm* c);
void comm_group_start();
void comm_group_end();
// buf[lo_r, hi_r) of every rank r -> every rank, in place (ranges: one [lo, hi) per rank, in rank order)
void comm_gather(Comm* c, float* buf, const std::vector<std::pair<int64_t, int64_t>>& ranges, cudaStream_t st);
void comm_allreduce_sum(Comm* c, double* buf, int count, cudaStream_t st);

}  // namespace clb
