// CUDA IPC exchange kernels of the one-process-per-GPU peer-store transport (ipc.cuh).
#include "ipc.cuh"

#include <cuda/atomic>

namespace clb {
namespace {

__global__ void k_ipc_signal(IpcPeerSync peers, int world, int rank, unsigned long long value) {
  const int q = threadIdx.x;
  if (q >= world) return;
  __threadfence_system();  // this rank's earlier stores (the epilogue's peer stores completed before this kernel)
  cuda::atomic_ref<unsigned long long, cuda::thread_scope_system> f(peers.s[q]->sig[rank]);
  f.store(value, cuda::memory_order_release);
}

__global__ void k_ipc_wait(IpcSync* own, int world, int rank, unsigned long long value) {
  const long long limit = 40000000000LL;  // ~20 s of SM clock
  const long long t0 = clock64();
  for (int q = 0; q < world; ++q) {
    if (q == rank) continue;
    cuda::atomic_ref<unsigned long long, cuda::thread_scope_system> f(own->sig[q]);
    while (f.load(cuda::memory_order_acquire) < value) {
      if (clock64() - t0 > limit) {
        own->timed_out = 1;
        return;
      }
      __nanosleep(256);
    }
  }
  __threadfence_system();
}

__global__ void k_ipc_push_met(IpcPeerSync peers, int world, int rank, const double* __restrict__ met4) {
  const int q = threadIdx.x >> 2, i = threadIdx.x & 3;
  if (q < world) peers.s[q]->met[rank][i] = met4[i];
}

__global__ void k_ipc_push_slice(IpcPeerVec dst, int world, int rank, const float* __restrict__ src, int64_t lo,
                                 int64_t hi) {
  for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hi; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = src[i];
    for (int q = 0; q < world; ++q)
      if (q != rank) dst.p[q][i] = v;
  }
}

}  // namespace

void launch_ipc_signal(const IpcPeerSync& peers, int world, int rank, unsigned long long value, cudaStream_t st) {
  k_ipc_signal<<<1, kIpcMaxRanks, 0, st>>>(peers, world, rank, value);
}
void launch_ipc_wait(IpcSync* own, int world, int rank, unsigned long long value, cudaStream_t st) {
  k_ipc_wait<<<1, 1, 0, st>>>(own, world, rank, value);
}
void launch_ipc_push_met(const IpcPeerSync& peers, int world, int rank, const double* met4, cudaStream_t st) {
  k_ipc_push_met<<<1, 4 * kIpcMaxRanks, 0, st>>>(peers, world, rank, met4);
}
void launch_ipc_push_slice(const IpcPeerVec& dst, int world, int rank, const float* src, int64_t lo, int64_t hi,
                           cudaStream_t st) {
  if (hi > lo) k_ipc_push_slice<<<148 * 4, 256, 0, st>>>(dst, world, rank, src, lo, hi);
}

}  // namespace clb
