// One process per GPU without NCCL: the sharded solve's exchange as CUDA IPC peer stores.
// Every rank maps the other ranks' exchange vectors; each phase's epilogue stores its slice into all of
// them (EpiArgs::peer), and the ranks order their phases through system-scope flags in a small sync block
// each rank exports.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace clb {

constexpr int kIpcMaxRanks = 8;

// exported by every rank (cudaMalloc'd): the flag each peer raises after its phases, and the check metrics
// every rank pushes to every other rank
struct IpcSync {
  unsigned long long sig[kIpcMaxRanks];  // sig[q] = the last sequence number rank q signalled to this rank
  double met[kIpcMaxRanks][4];           // met[q] = rank q's share of the check sums
  unsigned long long timed_out;          // a wait gave up (a peer stopped)
};
struct IpcPeerSync {
  IpcSync* s[kIpcMaxRanks] = {};  // indexed by rank; this rank's own block at its own index
};
struct IpcPeerVec {
  float* p[kIpcMaxRanks] = {};  // a vector's copies, indexed by rank
};

// rank `rank` raises its flag to `value` in every rank's sync block (release, system scope)
void launch_ipc_signal(const IpcPeerSync& peers, int world, int rank, unsigned long long value, cudaStream_t st);
// the stream waits (one spinning thread, acquire, system scope) until every other rank's flag in `own` reached
// `value`; gives up after ~20 s and marks own->timed_out
void launch_ipc_wait(IpcSync* own, int world, int rank, unsigned long long value, cudaStream_t st);
// met4 -> met[rank] of every rank's sync block
void launch_ipc_push_met(const IpcPeerSync& peers, int world, int rank, const double* met4, cudaStream_t st);
// src[lo, hi) -> the same range of every other rank's copy
void launch_ipc_push_slice(const IpcPeerVec& dst, int world, int rank, const float* src, int64_t lo, int64_t hi,
                           cudaStream_t st);

}  // namespace clb
