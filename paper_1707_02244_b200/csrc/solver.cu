// Solver engine + C-ABI of circlasso_b200 (include/circlasso_b200.h).
//
// Mirrors the reference solver layer (solvers.hpp): *_setup validates and
// normalizes exactly where the reference throws, *_step advances the state
// through the direct sm_100a kernels (kernels.cu), run_loop reproduces the
// check cadence and stopping rule.  Setup transforms are fp64 on the host
// (host_setup.cpp); iteration state lives in HBM as fp32.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "host_common.hpp"
#include "fft.cuh"
#include "fft4.cuh"
#include "kernels.cuh"
#include "tc_dense.cuh"
#include "dense.cuh"
#include "comm.hpp"
#include "ipc.cuh"

// NVTX ranges (SURVEY §5 tracing): every C-ABI entry that launches work and every kernel phase pushes a
// named range, named after the reference's KernelPhase names (parallel.hpp:173-279), so an nsys/ncu
// (--nvtx) timeline groups the kernels by phase.  Header-only NVTX v3: a no-op unless a tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

namespace clb {
void gen_sparse_signal(int64_t n, int64_t k, uint64_t seed, double* values, int64_t* support);
void gen_circulant_sensing(int64_t n, int64_t m, uint64_t seed, double* c, int64_t* omega);
void gen_star_field(int64_t width, int64_t height, double density, uint64_t seed, double* px);
void blur_row(int64_t n, int64_t L, double* row);

namespace {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    std::ostringstream msg;
    msg << what << ": " << cudaGetErrorString(e);
    raise(CL_ECUDA, msg.str());
  }
}
#define CU(x) cuda_check((x), #x)

// Device buffer from the device's stream-ordered memory pool (cudaMallocAsync;
// the pool keeps freed memory reserved, see reserve_pool), so creating and
// destroying solver states does not pay cudaMalloc/cudaFree (a cudaFree of
// the residual's 165 MB partial buffer synchronizes the device and unmaps:
// ~0.2-1.6 s per state destruction at n = 2^20, measured).  `st` orders the
// allocation and the free after the work on that stream; it must outlive the
// buffer (nullptr: the legacy stream, after the caller synchronized).
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t count = 0;
  cudaStream_t s = nullptr;
  bool plain = false;  // cudaMalloc'd (IPC-exportable) instead of the stream-ordered pool
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) {
      if (plain) cudaFree(p);
      else cudaFreeAsync(p, s);
    }
    p = nullptr;
    plain = false;
  }
  // move the contents into cudaMalloc'd memory (CUDA IPC cannot export stream-ordered pool allocations)
  void make_plain(cudaStream_t st) {
    if (plain || !count) return;
    T* q = nullptr;
    CU(cudaMalloc(reinterpret_cast<void**>(&q), sizeof(T) * count));
    CU(cudaMemcpyAsync(q, p, sizeof(T) * count, cudaMemcpyDeviceToDevice, st));
    CU(cudaStreamSynchronize(st));
    cudaFreeAsync(p, s);
    p = q;
    plain = true;
  }
  void alloc(size_t c, cudaStream_t st = nullptr) {
    release();
    count = c;
    s = st;
    if (c) CU(cudaMallocAsync(reinterpret_cast<void**>(&p), sizeof(T) * c, st));
  }
  void upload(const T* h, size_t c, cudaStream_t st) {
    if (c) CU(cudaMemcpyAsync(p, h, sizeof(T) * c, cudaMemcpyHostToDevice, st));
  }
  void zero(cudaStream_t st) {
    if (count) CU(cudaMemsetAsync(p, 0, sizeof(T) * count, st));
  }
};

std::vector<float> to_f32(const double* a, int64_t n, double scale = 1.0) {
  std::vector<float> out(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) out[static_cast<size_t>(i)] = static_cast<float>(a[i] / scale);
  return out;
}
std::vector<float> reversed(const std::vector<float>& a) {  // r[k] = a[(-k) mod n]
  const size_t n = a.size();
  std::vector<float> r(n);
  for (size_t k = 0; k < n; ++k) r[k] = a[(n - k) % n];
  return r;
}

// Keep freed pool memory reserved for the next state (HBM is not returned to
// the OS between solves; 180 GB per GPU).
void reserve_pool(int device) {
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
}

double seconds_since(std::chrono::steady_clock::time_point a) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
}

// CLB_TRACE=1: host wall time of each setup / run / teardown stage on stderr (e2e diagnostics).
void trace(const char* stage) {
  static const bool on = [] {
    const char* v = std::getenv("CLB_TRACE");
    return v && v[0] == '1';
  }();
  if (!on) return;
  static thread_local auto last = std::chrono::steady_clock::now();
  const auto now = std::chrono::steady_clock::now();
  std::fprintf(stderr, "[clb] %-28s %8.3f ms\n", stage, std::chrono::duration<double, std::milli>(now - last).count());
  last = now;
}

// solvers.hpp:90-106 (circulant kinds only)
uint64_t footprint(int kind, int64_t n, int64_t m, uint64_t width) {
  const uint64_t un = static_cast<uint64_t>(n);
  if (kind == CL_KIND_ADMM) return (un * un + 4 * un + static_cast<uint64_t>(m)) * width;  // kDenseAdmm
  return (kind == CL_KIND_ISTA ? 4 : 10) * un * width;
}

// Per-device pool of the host-side resources a solver state owns: its non-blocking stream, its
// timing events, a pinned metric slot and a pinned staging buffer for downloads.  Creating them
// costs 1.5-5 ms per state (cudaStreamCreate, cudaMallocHost); a state created after another one
// was destroyed on the same device takes the previous one's instead, so repeated ista_run /
// cadmm_run calls do not pay it.  The stream is drained before it is returned.
constexpr int kPhaseEvents = 8;
struct StateResources {
  int device = 0;
  cudaStream_t st = nullptr;
  cudaEvent_t ev[kPhaseEvents] = {};
  cudaEvent_t step_ev[2] = {};
  double* met_host = nullptr;  // 4 doubles
  float* stage = nullptr;      // pinned download staging
  size_t stage_floats = 0;
  void create(int dev) {
    device = dev;
    CU(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    for (auto& e : ev) CU(cudaEventCreate(&e));
    for (auto& e : step_ev) CU(cudaEventCreate(&e));
    CU(cudaMallocHost(&met_host, sizeof(double) * 4));
  }
  float* staging(size_t count) {
    if (count > stage_floats) {
      if (stage) CU(cudaFreeHost(stage));
      stage = nullptr;
      stage_floats = 0;
      CU(cudaMallocHost(&stage, sizeof(float) * count));
      stage_floats = count;
    }
    return stage;
  }
};
struct ResourcePool {
  std::mutex mu;
  std::vector<StateResources> free[64];
};
ResourcePool& resource_pool() {
  static ResourcePool* p = new ResourcePool();  // never destroyed: streams may outlive static teardown
  return *p;
}
StateResources take_resources(int device) {
  ResourcePool& p = resource_pool();
  {
    std::lock_guard<std::mutex> lk(p.mu);
    if (device >= 0 && device < 64 && !p.free[device].empty()) {
      StateResources r = p.free[device].back();
      p.free[device].pop_back();
      return r;
    }
  }
  StateResources r;
  r.create(device);
  return r;
}
void give_resources(const StateResources& r) {
  if (!r.st) return;
  cudaStreamSynchronize(r.st);
  ResourcePool& p = resource_pool();
  std::lock_guard<std::mutex> lk(p.mu);
  if (r.device >= 0 && r.device < 64 && p.free[r.device].size() < 8) {
    p.free[r.device].push_back(r);
    return;
  }
  for (auto e : r.ev) cudaEventDestroy(e);
  for (auto e : r.step_ev) cudaEventDestroy(e);
  cudaFreeHost(r.met_host);
  if (r.stage) cudaFreeHost(r.stage);
  cudaStreamDestroy(r.st);
}

}  // namespace

// Shard g of G: tiles [g*T/G, (g+1)*T/G) of the output plan; for
// ISTA the residual splits [g*S/G, (g+1)*S/G) and hence the rows of their
// position chunks.  Pure host logic, shared by the solver and cl_shard_ranges.
void shard_ranges(int kind, int64_t n, const int64_t* omega, int64_t m, int rk, int ws, ConvPlan* plan,
                  ConvPlan* rplan, int64_t* out_lo, int64_t* out_hi, int64_t* row_lo, int64_t* row_hi) {
  if (ws < 1 || rk < 0 || rk >= ws) raise(CL_EPARAM, "cl_solver_shard: need 0 <= rank < world");
  plan->tile_lo = plan->tiles * rk / ws;
  plan->tile_hi = plan->tiles * (rk + 1) / ws;
  *out_lo = std::min<int64_t>(n, plan->tile_lo * plan->tile);
  *out_hi = std::min<int64_t>(n, plan->tile_hi * plan->tile);
  *row_lo = *row_hi = 0;
  if (kind == CL_KIND_ISTA && plan->tc) {  // dense-embedded products: rows = Omega within the owned outputs
    *row_lo = std::lower_bound(omega, omega + m, *out_lo) - omega;
    *row_hi = std::lower_bound(omega, omega + m, *out_hi) - omega;
  } else if (kind == CL_KIND_ISTA) {
    rplan->split_lo = static_cast<int>(static_cast<int64_t>(rplan->splits) * rk / ws);
    rplan->split_hi = static_cast<int>(static_cast<int64_t>(rplan->splits) * (rk + 1) / ws);
    int64_t b_lo, b_hi, dummy;
    split_block_range(*rplan, rplan->split_lo, &b_lo, &dummy);
    split_block_range(*rplan, rplan->split_hi - 1, &dummy, &b_hi);
    if (rplan->split_hi <= rplan->split_lo) b_hi = b_lo;
    const int64_t p_lo = b_lo * 32, p_hi = b_hi * 32;
    *row_lo = std::lower_bound(omega, omega + m, p_lo) - omega;  // rows with positions in the splits' blocks
    *row_hi = std::lower_bound(omega, omega + m, p_hi) - omega;
  }
}

std::vector<int> chunk_rowstart(const int64_t* omega, int64_t m, int64_t chunks) {
  std::vector<int> rs(static_cast<size_t>(chunks + 1), 0);
  int64_t k = 0;
  for (int64_t c = 0; c <= chunks; ++c) {
    const int64_t lim = c * kChunk;
    while (k < m && omega[k] < lim) ++k;
    rs[static_cast<size_t>(c)] = static_cast<int>(k);
  }
  return rs;
}

struct Solver {
  int kind = CL_KIND_ISTA;
  int device = 0;
  int64_t n = 0, m = 0;
  cl_config cfg{};
  double scale = 1.0, tau = 0.0, thr = 0.0, setup_seconds = 0.0;
  int64_t t = 0;
  int rank = 0, world = 1;
  bool has_truth = false;
  // per-phase CUDA events: 0 off, 1 eager launches (no graph), 2 event nodes inside the captured
  // step graph (the timed configuration itself: cl_solver_phase_ms reads the last replay)
  int profile = 0;
  cudaStream_t st = nullptr;
  StateResources res;  // st, the events and the pinned slots (from the per-device pool)
  // Returns res to the pool after every DevBuf member (declared below) has queued its free.
  struct ResOwner {
    StateResources* r;
    ~ResOwner() { give_resources(*r); }
  } res_owner{&res};
  ConvPlan plan;     // outputs: gradient (ISTA) or dense (cADMM) products
  ConvPlan rplan;    // ISTA residual (input tiles x position splits)
  bool ista_tc = false;  // ISTA products embedded in dense tensor-core products (plan == rplan, tc)
  int64_t row_lo = 0, row_hi = 0;  // ISTA rows owned (residual)
  // library-owned collective of a sharded solve (cl_solver_attach_comm) and every rank's slices:
  // rows_of[r] = ISTA residual rows of rank r, outs_of[r] = outputs of rank r
  Comm* comm = nullptr;
  std::vector<std::pair<int64_t, int64_t>> rows_of, outs_of;
  // one process per GPU without NCCL (cl_solver_peer_export / _attach): CUDA IPC peer stores
  struct Ipc {
    bool on = false;
    unsigned long long seq = 0;
    IpcSync* own = nullptr;     // this rank's exported sync block (cudaMalloc'd)
    IpcPeerSync sync;           // every rank's sync block, own at its rank
    IpcPeerVec z;               // cADMM: every rank's z (the slice-local iterate, pushed before downloads)
    std::vector<void*> opened;  // the peers' mappings
  } ipc;
  int64_t out_lo = 0, out_hi = 0;  // outputs owned

  DevBuf<float> hc, hcr, hbr;      // c~, c~ reversed, b reversed
  DevBuf<int> omega32, rowstart;
  DevBuf<float> y, r, x, delta;    // ISTA
  DevBuf<float> d, pty, z, nu, mu, v, beta;  // cADMM (x shared)
  DevBuf<float> partial, truth;
  DevBuf<float> Bm, aty, u, rhs;             // dense ADMM: B (n x n fp32), A~^T y~, dual, right-hand side
  DevBuf<float> tcs;  // this solver's tensor-core operand-scale scratch (ConvPlan::tc_scratch)
  DevBuf<float2> chat, bhat, F0, F1;  // FFT engine: spectra of c~ (and of B), work buffers
  bool fft = false;
  // FFT length: n for power-of-two n; otherwise the next power of two >= 2n - 1, with the circulant
  // embedded as a linear convolution (g[k] = h[k mod n], k in (-n, n), placed mod nfft; inputs zero-padded)
  // so any n runs on power-of-two transforms, like the reference's kissfft runs any n.
  int64_t nfft = 0;
  std::vector<double> padded_cn, padded_bn;  // cADMM setup hand-over (normalized c and b rows)
  // Four-step FFT engine (fft4.cu; power-of-two 2^14 <= n <= 2^24 with the device setup): the
  // spectra in its permuted order, twiddle tables, the row map and P^T r kept dense.
  bool fft4 = false;
  Fft4Plan f4;
  DevBuf<float2> tw1, tw2, twA, twB, chatp, bhatp;
  DevBuf<int> rowid;
  DevBuf<float> ud;
  // One-CTA FFT-engine ISTA at small n (fft4.cu): spectrum in DIF order and the twiddle table.
  bool small_fft = false;
  DevBuf<float2> chatS, bhatS, twS;
  DevBuf<double> blk, met;
  double* met_host = nullptr;     // res.met_host
  std::vector<int> rowstart_host;
  std::vector<int64_t> omega_host;
  cudaEvent_t* ev = nullptr;       // res.ev[kPhaseEvents]
  double phase_ms[8] = {};
  int nphase = 0;
  cudaEvent_t* step_ev = nullptr;  // res.step_ev[2]
  double last_step_ms = 0.0;
  // profile mode 2: the captured step's event-record nodes (node i records phase boundary i) and a
  // ring of per-replay event sets they are re-pointed to before every replay, so back-to-back
  // replays are timed phase by phase without a host synchronization in between
  static constexpr int kRing = 256;
  cudaGraphNode_t ev_node[kPhaseEvents] = {};
  int n_ev_nodes = 0;
  std::vector<cudaEvent_t> ring;  // kRing * kPhaseEvents
  int64_t ring_count = 0;         // replays recorded since the last reset
  // One unchecked iteration captured as a CUDA graph (launch-bound small n and
  // the ~30-launch FFT engine step); replayed by step().  CLB_NO_GRAPH=1 disables.
  cudaGraphExec_t graph = nullptr;
  cudaGraph_t graph_src = nullptr;  // kept while `graph` lives: its node handles address the exec's nodes
  void drop_graph() {
    if (graph) cudaGraphExecDestroy(graph);
    if (graph_src) cudaGraphDestroy(graph_src);
    graph = nullptr;
    graph_src = nullptr;
    n_ev_nodes = 0;
  }

  ~Solver() {
    trace("destroy: enter");
    if (st) cudaSetDevice(device);
    if (st) cudaStreamSynchronize(st);
    if (ipc.on) {  // every rank is done with every other rank's memory before any of it is unmapped or freed
      try {
        ipc_barrier();
        cudaStreamSynchronize(st);
      } catch (...) {
      }
      for (void* q : ipc.opened) cudaIpcCloseMemHandle(q);
    }
    if (ipc.own) cudaFree(ipc.own);
    trace("destroy: stream drained");
    drop_graph();
    for (auto e : ring) cudaEventDestroy(e);
    trace("destroy: graph/events");
  }

  void init_device() {
    int count = 0;
    CU(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) raise(CL_ECUDA, "cl_solver_create: no such CUDA device");
    CU(cudaSetDevice(device));
    res = take_resources(device);
    st = res.st;
    ev = res.ev;
    step_ev = res.step_ev;
    met_host = res.met_host;
    reserve_pool(device);
    conv_kernels_init();
    trace("setup: init_device");
  }

  void build_rows(const int64_t* omega) {
    omega_host.assign(omega, omega + m);
    std::vector<int> om(static_cast<size_t>(m));
    for (int64_t t2 = 0; t2 < m; ++t2) om[static_cast<size_t>(t2)] = static_cast<int>(omega[t2]);
    rowstart_host = chunk_rowstart(omega, m, plan.chunks);
    omega32.alloc(static_cast<size_t>(m), st);
    omega32.upload(om.data(), static_cast<size_t>(m), st);
    rowstart.alloc(rowstart_host.size(), st);
    rowstart.upload(rowstart_host.data(), rowstart_host.size(), st);
  }

  void attach_tc_scratch() {
    if (!plan.tc) return;
    tcs.alloc(tc_scratch_floats(), st);
    plan.tc_scratch = tcs.p;
    if (rplan.tc) rplan.tc_scratch = tcs.p;
  }

  void set_shard(int rk, int ws) {
    if (fft && ws != 1) raise(CL_EPARAM, "cl_solver_shard: the FFT engine runs unsharded (replicas only)");
    if (kind == CL_KIND_ADMM) {
      if (ws != 1) raise(CL_EPARAM, "cl_solver_shard: the dense ADMM runs unsharded (n <= dense_cap; replicas only)");
      return;
    }
    if (graph) {  // the captured step covers the previous shard's ranges
      CU(cudaStreamSynchronize(st));
      drop_graph();
    }
    rank = rk;
    world = ws;
    shard_ranges(kind, n, omega_host.data(), m, rk, ws, &plan, &rplan, &out_lo, &out_hi, &row_lo, &row_hi);
  }

  void setup_common(const double* c, const int64_t* omega, const double* yh, const cl_config* config) {
    if (!config) raise(CL_EPARAM, "cl_solver_create: null config");
    cfg = *config;
    check_mask(omega, m, n);
    if (cfg.engine != CL_ENGINE_DIRECT && cfg.engine != CL_ENGINE_FFT)
      raise(CL_EPARAM, "cl_solver_create: unknown engine");
    fft = cfg.engine == CL_ENGINE_FFT;
    if (fft) {
      nfft = n;
      if (!is_pow2(n)) {
        nfft = 1;
        while (nfft < 2 * n - 1) nfft <<= 1;
        if (nfft > (int64_t(1) << 26)) raise(CL_ECAPACITY, "cl_solver_create: n too large for the padded FFT engine");
      }
    }
  }

  // solvers.hpp:170-183.  `s` = max_k |DFT(c)_k| (host or device transform).
  double normalization_from(double s, const double* yh) {
    if (s > 0.0) return s;
    double mx = 0.0;
    for (int64_t i = 0; i < m; ++i) mx = std::max(mx, std::abs(yh[i]));
    if (m == 0 || mx == 0.0) return 1.0;
    raise(CL_ESINGULAR, "solver: sensing operator is zero but measurements are not");
  }
  void check_finite_y(const double* yh) {
    for (int64_t i = 0; i < m; ++i)
      if (!std::isfinite(yh[i])) raise(CL_EDIVERGE, "solver: measurements contain non-finite entries");
  }

  // ---- setup transforms on the device (power-of-two n) ----------------------
  // The reference runs them once per solve in fp64 (circulant.hpp:297-351);
  // so do we, with the fp64 Stockham FFT of fft.cu, instead of a host FFT.
  bool device_setup() const {
    const char* v = std::getenv("CLB_HOST_SETUP");  // 1: host fp64 transforms (parity tests)
    return !(v && v[0] == '1') && is_pow2(n) && n >= (int64_t(1) << 14);
  }
  DevBuf<double> c64, b64;
  DevBuf<double2> X64, W64, B64;
  DevBuf<unsigned long long> red;  // [absmax, min denominator, max |re|, max |im|] as IEEE bits
  const double2* spec64 = nullptr;   // DFT(c), in X64 or W64

  void red_reset() {
    const unsigned long long init[4] = {0ull, 0x7ff0000000000000ull /* +inf */, 0ull, 0ull};
    if (!red.p) red.alloc(4, st);
    CU(cudaMemcpyAsync(red.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
    CU(cudaStreamSynchronize(st));  // `init` is a stack array
  }
  void red_read(double out[4]) {
    unsigned long long h[4];
    CU(cudaMemcpyAsync(h, red.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    for (int i = 0; i < 4; ++i) std::memcpy(&out[i], &h[i], sizeof(double));
  }
  // uploads c (fp64), spec64 = DFT(c); returns max_k |DFT(c)_k|
  double device_spectrum(const double* c) {
    c64.alloc(static_cast<size_t>(n), st);
    c64.upload(c, static_cast<size_t>(n), st);
    X64.alloc(static_cast<size_t>(n), st);
    W64.alloc(static_cast<size_t>(n), st);
    launch_real_to_complex64(c64.p, X64.p, n, st);
    spec64 = fft64_run(X64.p, W64.p, n, false, st);
    red_reset();
    launch_absmax64(spec64, n, red.p, st);
    double r[4];
    red_read(r);
    return r[0];
  }
  bool want_fft4(bool dev) const {
    const char* v = std::getenv("CLB_FFT_STOCKHAM");  // 1: the multi-pass Stockham engine (fft.cu)
    return fft && dev && fft4_supported(n) && !(v && v[0] == '1');
  }
  void setup_fft4_common() {
    fft4 = true;
    f4 = fft4_plan(n);
    fft4_init_attributes();
    std::vector<float2> t1, t2, ta, tb;
    fft4_twiddles(f4, &t1, &t2, &ta, &tb);
    for (auto& pr : {std::make_pair(&tw1, &t1), std::make_pair(&tw2, &t2), std::make_pair(&twA, &ta),
                     std::make_pair(&twB, &tb)}) {
      pr.first->alloc(pr.second->size(), st);
      pr.first->upload(pr.second->data(), pr.second->size(), st);
    }
    chatp.alloc(static_cast<size_t>(n), st);
    launch_fft4_perm_spectrum(f4, spec64, scale, chatp.p, st);
    F0.alloc(static_cast<size_t>(n), st);
    CU(cudaStreamSynchronize(st));  // the host twiddle vectors go out of scope
  }

  void device_setup_release() {
    for (DevBuf<double>* b : {&c64, &b64}) b->release();
    for (DevBuf<double2>* b : {&X64, &W64, &B64}) b->release();
    spec64 = nullptr;
  }

  void setup_ista(const double* c, const int64_t* omega, const double* yh) {  // solvers.hpp:222-249
    double tau0 = cfg.tau;
    if (tau0 == 0.0) tau0 = 0.9;
    if (!(tau0 > 0.0) || !(tau0 < 1.0))
      raise(CL_EPARAM,
            "ista_setup: tau must lie in (0, |A|_2^-2); on the normalized operator the admissible range is (0, 1)");
    if (!(cfg.alpha > 0.0)) raise(CL_EPARAM, "ista_setup: alpha must be > 0");
    check_finite_y(yh);
    trace("setup: validate");
    const bool dev = device_setup();
    if (dev) init_device();
    scale = normalization_from(dev ? device_spectrum(c) : spectral_norm(c, n), yh);
    trace("setup: spectral norm");
    tau = tau0;
    thr = cfg.pairing == CL_PAIRING_LITERAL ? cfg.alpha : tau0 * cfg.alpha;
    if (!dev) init_device();
    ista_tc = !fft && ista_uses_tc(n);
    plan = ista_tc ? make_dense_plan(n) : make_plan(n, grad_R(n));
    rplan = ista_tc ? plan : make_plan(n, res_R(n));
    attach_tc_scratch();
    hc.alloc(static_cast<size_t>(n), st);
    hcr.alloc(static_cast<size_t>(n), st);
    if (dev) {
      launch_rows_f32(c64.p, scale, hc.p, hcr.p, n, st);
    } else {
      const std::vector<float> cf = to_f32(c, n, scale);
      hc.upload(cf.data(), cf.size(), st);
      const std::vector<float> crf = reversed(cf);
      hcr.upload(crf.data(), crf.size(), st);
    }
    trace("setup: plans + rows f32");
    build_rows(omega);
    trace("setup: omega / row index");
    const std::vector<float> yf = to_f32(yh, m, scale);
    y.alloc(static_cast<size_t>(m), st);
    y.upload(yf.data(), yf.size(), st);
    const int64_t nv = std::max(n, nfft);  // the FFT engine reads zero-padded inputs of length nfft
    for (DevBuf<float>* b : {&r}) { b->alloc(static_cast<size_t>(m), st); b->zero(st); }
    for (DevBuf<float>* b : {&x, &delta}) { b->alloc(static_cast<size_t>(nv), st); b->zero(st); }
    partial.alloc(static_cast<size_t>(std::max<int64_t>(std::max<int64_t>(rplan.tiles * m, plan.splits * n), nv)), st);
    blk.alloc(kEpiBlocks * 4, st);
    met.alloc(4, st);
    set_shard(0, 1);
    if (ista_tc) {
      ud.alloc(static_cast<size_t>(n), st);  // r scattered to its positions (zero elsewhere)
      ud.zero(st);
    }
    if (want_fft4(dev)) {
      setup_fft4_common();
      rowid.alloc(static_cast<size_t>(n), st);
      launch_rowid(omega32.p, rowid.p, n, m, st);
      ud.alloc(static_cast<size_t>(n), st);
      ud.zero(st);
    } else if (fft && nfft != n) {
      std::vector<double> cn(static_cast<size_t>(n));
      for (int64_t i = 0; i < n; ++i) cn[static_cast<size_t>(i)] = c[i] / scale;
      setup_padded_fft(cn.data(), nullptr);
    } else if (fft) {
      if (dev) {
        chat.alloc(static_cast<size_t>(n), st);
        launch_spectrum_f32(spec64, scale, chat.p, n, st);
      } else {
        std::vector<double> cn(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) cn[static_cast<size_t>(i)] = c[i] / scale;
        upload_spectrum(chat, dft_real(cn.data(), n));
      }
      F0.alloc(static_cast<size_t>(n), st);
      F1.alloc(static_cast<size_t>(n), st);
      if (small_fft_supported(n)) setup_small_fft();
    }
    trace("setup: state buffers");
    CU(cudaGetLastError());
    device_setup_release();
    CU(cudaStreamSynchronize(st));
    trace("setup: drained");
  }

  // spectrum (length nfft, fp64, host) of the circulant with first row h embedded for a linear
  // convolution: g[k mod nfft] = h[k mod n], k in (-n, n)
  std::vector<cplx> padded_spectrum(const double* h) const {
    std::vector<double> g(static_cast<size_t>(nfft), 0.0);
    for (int64_t k = 0; k < n; ++k) g[static_cast<size_t>(k)] = h[k];
    for (int64_t k = 1; k < n; ++k) g[static_cast<size_t>(nfft - k)] = h[n - k];
    return dft_real(g.data(), nfft);
  }
  void upload_engine_spectrum(const std::vector<cplx>& spec, DevBuf<float2>& natural, DevBuf<float2>& perm) {
    if (!fft4) {
      upload_spectrum(natural, spec);
      return;
    }
    std::vector<double2> d(spec.size());
    for (size_t k = 0; k < spec.size(); ++k) d[k] = make_double2(spec[k].real(), spec[k].imag());
    DevBuf<double2> tmp;
    tmp.alloc(d.size(), st);
    tmp.upload(d.data(), d.size(), st);
    perm.alloc(d.size(), st);
    launch_fft4_perm_spectrum(f4, tmp.p, 1.0, perm.p, st);
    CU(cudaStreamSynchronize(st));  // d goes out of scope
  }
  // the padded (non-power-of-two n) FFT engine: four-step if nfft fits it, else Stockham passes
  void setup_padded_fft(const double* cn, const double* bn) {
    const char* v = std::getenv("CLB_FFT_STOCKHAM");
    if (fft4_supported(nfft) && !(v && v[0] == '1')) {
      fft4 = true;
      f4 = fft4_plan(nfft);
      fft4_init_attributes();
      std::vector<float2> t1, t2, ta, tb;
      fft4_twiddles(f4, &t1, &t2, &ta, &tb);
      for (auto& pr : {std::make_pair(&tw1, &t1), std::make_pair(&tw2, &t2), std::make_pair(&twA, &ta),
                       std::make_pair(&twB, &tb)}) {
        pr.first->alloc(pr.second->size(), st);
        pr.first->upload(pr.second->data(), pr.second->size(), st);
      }
      CU(cudaStreamSynchronize(st));
    }
    upload_engine_spectrum(padded_spectrum(cn), chat, chatp);
    if (bn) upload_engine_spectrum(padded_spectrum(bn), bhat, bhatp);
    F0.alloc(static_cast<size_t>(nfft), st);
    if (!fft4) F1.alloc(static_cast<size_t>(nfft), st);
    if (kind == CL_KIND_ISTA) {
      if (fft4) {
        rowid.alloc(static_cast<size_t>(nfft), st);
        launch_rowid(omega32.p, rowid.p, nfft, m, st);
      }
      ud.alloc(static_cast<size_t>(nfft), st);
      ud.zero(st);
    }
  }

  void setup_small_fft() {
    small_fft = true;
    std::vector<float2> t(static_cast<size_t>(n));
    for (int64_t k = 0; k < n; ++k) {
      const double a = -2.0 * 3.14159265358979323846 * static_cast<double>(k) / static_cast<double>(n);
      t[static_cast<size_t>(k)] = make_float2(static_cast<float>(std::cos(a)), static_cast<float>(std::sin(a)));
    }
    twS.alloc(t.size(), st);
    twS.upload(t.data(), t.size(), st);
    chatS.alloc(static_cast<size_t>(n), st);
    launch_small_fft_perm(chat.p, chatS.p, n, st);
    if (kind == CL_KIND_CADMM) {
      bhatS.alloc(static_cast<size_t>(n), st);
      launch_small_fft_perm(bhat.p, bhatS.p, n, st);
    }
    CU(cudaStreamSynchronize(st));  // t goes out of scope
  }

  void upload_spectrum(DevBuf<float2>& dst, const std::vector<cplx>& spec) {
    std::vector<float2> f(spec.size());
    for (size_t k = 0; k < spec.size(); ++k)
      f[k] = make_float2(static_cast<float>(spec[k].real()), static_cast<float>(spec[k].imag()));
    dst.alloc(f.size(), st);
    dst.upload(f.data(), f.size(), st);
  }

  // B = (rho C~^T C~ + sigma I)^-1 on the device: b = idft(1 / (rho |DFT(c)/s|^2 + sigma))
  // with the reference's floor (circulant.hpp:309-316) and residue check (fft.hpp:74-89).
  void device_gram_inverse(double s) {
    if (cfg.rho < 0.0 || cfg.sigma < 0.0 || (cfg.rho == 0.0 && cfg.sigma == 0.0))
      raise(CL_EPARAM,
            "regularized_gram_inverse: rho and sigma must be nonnegative with at least one strictly positive");
    B64.alloc(static_cast<size_t>(n), st);
    if (fft) bhat.alloc(static_cast<size_t>(n), st);
    red_reset();
    launch_gram_spectrum(spec64, s, cfg.rho, cfg.sigma, B64.p, fft ? bhat.p : nullptr, red.p + 1, n, st);
    if (want_fft4(true)) {  // B's spectrum in the four-step engine's order (before the inverse FFT reuses B64)
      const Fft4Plan p4 = fft4_plan(n);
      bhatp.alloc(static_cast<size_t>(n), st);
      launch_fft4_perm_spectrum(p4, B64.p, 1.0, bhatp.p, st);
    }
    double2* scratch = spec64 == X64.p ? W64.p : X64.p;
    const double2* Y = fft64_run(B64.p, scratch, n, true, st);
    b64.alloc(static_cast<size_t>(n), st);
    launch_real_part64(Y, b64.p, red.p + 2, red.p + 3, n, st);
    double r[4];
    red_read(r);
    if (r[1] < 1e-14) {
      std::ostringstream msg;
      msg << "regularized_gram_inverse: an eigenvalue of (rho C^T C + sigma I) is " << r[1]
          << ", below the invertibility floor 1e-14";
      raise(CL_ESINGULAR, msg.str());
    }
    const double sc = std::max(1.0, r[2]);
    if (r[3] > 1e-10 * sc) {
      std::ostringstream msg;
      msg << "inverse DFT of a real-valued quantity has imaginary residue " << r[3] << " (relative tolerance 1e-10)";
      raise(CL_ECONSIST, msg.str());
    }
  }

  void setup_cadmm(const double* c, const int64_t* omega, const double* yh) {  // solvers.hpp:359-395
    if (!(cfg.rho > 0.0) || !(cfg.sigma > 0.0)) raise(CL_EPARAM, "cadmm_setup: rho and sigma must be > 0");
    if (!(cfg.alpha > 0.0)) raise(CL_EPARAM, "cadmm_setup: alpha must be > 0");
    constexpr double kGolden = 1.6180339887498949;
    if (!(cfg.tau1 > 0.0) || cfg.tau1 >= kGolden || !(cfg.tau2 > 0.0) || cfg.tau2 >= kGolden)
      raise(CL_EPARAM, "cadmm_setup: tau1 and tau2 must lie in (0, (sqrt(5)+1)/2)");
    check_finite_y(yh);
    const bool dev = device_setup();
    if (dev) init_device();
    scale = normalization_from(dev ? device_spectrum(c) : spectral_norm(c, n), yh);
    if (!dev) init_device();
    plan = make_dense_plan(n);
    attach_tc_scratch();
    hc.alloc(static_cast<size_t>(n), st);
    hcr.alloc(static_cast<size_t>(n), st);
    hbr.alloc(static_cast<size_t>(n), st);
    if (dev) {
      device_gram_inverse(scale);
      launch_rows_f32(c64.p, scale, hc.p, hcr.p, n, st);
      launch_rows_f32(b64.p, 1.0, nullptr, hbr.p, n, st);
      if (want_fft4(dev)) {
        setup_fft4_common();
      } else if (fft) {
        chat.alloc(static_cast<size_t>(n), st);
        launch_spectrum_f32(spec64, scale, chat.p, n, st);
      }
    } else {
      std::vector<double> cn(static_cast<size_t>(n));
      for (int64_t i = 0; i < n; ++i) cn[static_cast<size_t>(i)] = c[i] / scale;
      std::vector<double> bh(static_cast<size_t>(n));
      regularized_gram_inverse(cn.data(), n, cfg.rho, cfg.sigma, bh.data());
      const std::vector<float> cf = to_f32(cn.data(), n);
      hc.upload(cf.data(), cf.size(), st);
      const std::vector<float> crf = reversed(cf);
      hcr.upload(crf.data(), crf.size(), st);
      const std::vector<float> brf = reversed(to_f32(bh.data(), n));
      hbr.upload(brf.data(), brf.size(), st);
      if (fft && nfft != n) {
        padded_cn.assign(cn.begin(), cn.end());
        padded_bn.assign(bh.begin(), bh.end());
      } else if (fft) {
        const std::vector<cplx> cs = dft_real(cn.data(), n);
        upload_spectrum(chat, cs);
        // B's spectrum is real: 1 / (rho |c_k|^2 + sigma) (circulant.hpp:306-317), exact before the idft round trip
        std::vector<cplx> bs(cs.size());
        for (size_t k = 0; k < cs.size(); ++k) bs[k] = cplx(1.0 / (cfg.rho * std::norm(cs[k]) + cfg.sigma), 0.0);
        upload_spectrum(bhat, bs);
      }
    }
    std::vector<double> dh(static_cast<size_t>(n));
    mask_gram_inverse(omega, m, n, cfg.rho, dh.data());
    std::vector<double> ptyh(static_cast<size_t>(n), 0.0);
    for (int64_t t2 = 0; t2 < m; ++t2) ptyh[static_cast<size_t>(omega[t2])] = yh[t2] / scale;
    thr = cfg.alpha / cfg.sigma;
    const std::vector<float> df = to_f32(dh.data(), n), pf = to_f32(ptyh.data(), n);
    d.alloc(static_cast<size_t>(n), st);
    d.upload(df.data(), df.size(), st);
    pty.alloc(static_cast<size_t>(n), st);
    pty.upload(pf.data(), pf.size(), st);
    const int64_t nv = std::max(n, nfft);  // the FFT engine reads zero-padded inputs of length nfft
    for (DevBuf<float>* b : {&x, &z, &nu, &mu, &v, &beta}) { b->alloc(static_cast<size_t>(nv), st); b->zero(st); }
    partial.alloc(static_cast<size_t>(std::max<int64_t>(plan.splits * n, nv)), st);
    blk.alloc(kEpiBlocks * 4, st);
    met.alloc(4, st);
    rowstart_host.assign(static_cast<size_t>(plan.chunks + 1), 0);
    if (fft && nfft != n) {
      setup_padded_fft(padded_cn.data(), padded_bn.data());
      padded_cn.clear();
      padded_bn.clear();
    } else if (fft && !fft4) {
      F0.alloc(static_cast<size_t>(n), st);
      F1.alloc(static_cast<size_t>(n), st);
      if (small_fft_cadmm_supported(n)) setup_small_fft();
    }
    set_shard(0, 1);
    CU(cudaGetLastError());
    device_setup_release();
    CU(cudaStreamSynchronize(st));
  }

  // admm_setup solvers.hpp:285-314: G = A~^T A~ + rho I and B = G^-1 in fp64 on the device (dense.cu),
  // then B, A~^T y~ in fp32 for the iterations.
  void setup_admm(const double* c, const int64_t* omega, const double* yh) {
    if (n > cfg.dense_cap) {
      std::ostringstream msg;
      msg << "admm_setup: n = " << n << " exceeds the dense cap " << cfg.dense_cap;
      raise(CL_ECAPACITY, msg.str());
    }
    if (!(cfg.rho > 0.0)) raise(CL_EPARAM, "admm_setup: rho must be > 0");
    if (!(cfg.alpha > 0.0)) raise(CL_EPARAM, "admm_setup: alpha must be > 0");
    if (fft) raise(CL_EPARAM, "admm_setup: the dense ADMM has no FFT engine (it multiplies by the stored B)");
    check_finite_y(yh);
    scale = normalization_from(spectral_norm(c, n), yh);
    init_device();
    thr = cfg.alpha / cfg.rho;
    const int64_t np = dense_pad(n);
    std::vector<double> cn(static_cast<size_t>(n)), yn(static_cast<size_t>(m));
    for (int64_t i = 0; i < n; ++i) cn[static_cast<size_t>(i)] = c[i] / scale;
    for (int64_t t2 = 0; t2 < m; ++t2) yn[static_cast<size_t>(t2)] = yh[t2] / scale;
    std::vector<int> om(static_cast<size_t>(m));
    for (int64_t t2 = 0; t2 < m; ++t2) om[static_cast<size_t>(t2)] = static_cast<int>(omega[t2]);
    omega_host.assign(omega, omega + m);
    DevBuf<double> cn64, yn64, G, scr, aty64;
    cn64.alloc(cn.size(), st);
    cn64.upload(cn.data(), cn.size(), st);
    yn64.alloc(yn.size(), st);
    yn64.upload(yn.data(), yn.size(), st);
    omega32.alloc(om.size(), st);
    omega32.upload(om.data(), om.size(), st);
    G.alloc(static_cast<size_t>(np * np), st);
    scr.alloc(dense_gj_scratch(np), st);
    aty64.alloc(static_cast<size_t>(n), st);
    launch_dense_gram(cn64.p, omega32.p, n, m, cfg.rho, G.p, np, st);
    launch_dense_aty(cn64.p, omega32.p, yn64.p, n, m, aty64.p, st);
    launch_dense_invert(G.p, np, scr.p, nullptr, st);
    Bm.alloc(static_cast<size_t>(n * n), st);
    launch_dense_to_f32(G.p, np, n, Bm.p, st);
    aty.alloc(static_cast<size_t>(n), st);
    launch_f64_to_f32(aty64.p, n, aty.p, st);
    CU(cudaGetLastError());
    for (DevBuf<float>* b : {&x, &z, &u}) { b->alloc(static_cast<size_t>(n), st); b->zero(st); }
    rhs.alloc(static_cast<size_t>(n), st);
    CU(cudaMemcpyAsync(rhs.p, aty.p, sizeof(float) * n, cudaMemcpyDeviceToDevice, st));  // rhs = A~^T y~
    blk.alloc(kEpiBlocks * 4, st);
    met.alloc(4, st);
    out_lo = 0;
    out_hi = n;
    CU(cudaStreamSynchronize(st));  // the host vectors and the fp64 scratch go out of scope
  }
  void admm_dense_step(int want) {  // padmm_phases parallel.hpp:284-317
    mark(0);
    PadmmArgs a;
    a.B = Bm.p;
    a.rhs = rhs.p;
    a.x = x.p;
    a.z = z.p;
    a.u = u.p;
    a.truth = has_truth ? truth.p : nullptr;
    a.blk = blk.p;
    a.n = n;
    a.thr = static_cast<float>(thr);
    a.want_metrics = want;
    launch_padmm_primal(a, st);
    mark(1);
    launch_padmm_rhs(aty.p, z.p, u.p, static_cast<float>(cfg.rho), rhs.p, n, st);
    mark(2);
    nphase = 2;
  }

  void mark(int i) {
    if (!profile) return;
    // inside a stream capture a plain record only orders streams; the external flag makes it a real
    // event-record node of the graph, so each replay stamps the phase boundaries
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CU(cudaStreamIsCapturing(st, &cs));
    if (cs == cudaStreamCaptureStatusActive) CU(cudaEventRecordWithFlags(ev[i], st, cudaEventRecordExternal));
    else CU(cudaEventRecord(ev[i], st));
  }

  // peer-store transport (Group kPeer): per phase, the other ranks' copies of the vector the phase produces
  float* peer_out[3][EpiArgs::kMaxPeers] = {};
  int npeer = 0;
  void set_peers(EpiArgs& a, int ph) const {
    a.npeer = npeer;
    for (int p = 0; p < npeer; ++p) a.peer[p] = peer_out[ph][p];
  }
  EpiArgs base_args(int want) {
    EpiArgs a;
    a.partial = partial.p;
    a.splits = plan.splits;
    a.n = n;
    a.lo = out_lo;
    a.hi = out_hi;
    a.truth = has_truth ? truth.p : nullptr;
    a.blk = blk.p;
    a.want_metrics = want;
    return a;
  }

  // ---- phases -------------------------------------------------------------
  void ista_residual() {
    NvtxRange nv("cpista residual computation");
    mark(0);
    if (ista_tc) {  // C x on the tensor cores, rows Omega gathered in the epilogue
      CU(launch_conv_dense(plan, hcr.p, x.p, partial.p, st));
      mark(1);
      EpiArgs a;
      a.partial = partial.p;
      a.splits = plan.splits;
      a.n = n;
      a.lo = row_lo;
      a.hi = row_hi;
      a.y = y.p;
      a.r = r.p;
      set_peers(a, 0);
      launch_ista_residual_gather(a, omega32.p, st);
      mark(2);
      return;
    }
    launch_conv_residual(rplan, m, hcr.p, x.p, omega32.p, rowstart.p, partial.p, st);
    mark(1);
    EpiArgs a;
    a.partial = partial.p;
    a.n = m;
    a.lo = row_lo;
    a.hi = row_hi;
    a.y = y.p;
    a.r = r.p;
    set_peers(a, 0);
    launch_ista_residual_reduce(a, rplan.tiles, st);
    mark(2);
  }
  void ista_gradient(int want) {
    NvtxRange nv("cpista thresholded gradient");
    if (ista_tc) {  // C^T P^T r: scatter r (all rows, after any exchange), dense product
      launch_scatter_real(r.p, omega32.p, ud.p, m, st);
      CU(launch_conv_dense(plan, hc.p, ud.p, partial.p, st));
    } else {
      launch_conv_rows(plan, hc.p, omega32.p, r.p, rowstart.p, partial.p, st);
    }
    mark(3);
    EpiArgs a = base_args(want);
    a.x = x.p;
    a.delta = delta.p;
    a.tau = static_cast<float>(tau);
    a.thr = static_cast<float>(thr);
    set_peers(a, 1);
    launch_ista_update(a, st);
    mark(4);
    nphase = 4;
  }
  void admm_beta_phase() {
    NvtxRange nv("cpadmm primal variables update");
    mark(0);
    CU(launch_conv_dense(plan, hc.p, v.p, partial.p, st));
    mark(1);
    EpiArgs a = base_args(0);
    a.beta = beta.p;
    a.z = z.p;
    a.nu = nu.p;
    a.rho = static_cast<float>(cfg.rho);
    a.sigma = static_cast<float>(cfg.sigma);
    set_peers(a, 0);
    launch_admm_beta(a, st);
    mark(2);
  }
  void admm_x_phase() {
    NvtxRange nv("cpadmm signal recovery");
    CU(launch_conv_dense(plan, hbr.p, beta.p, partial.p, st));
    mark(3);
    EpiArgs a = base_args(0);
    a.x = x.p;
    set_peers(a, 1);
    launch_admm_x(a, st);
    mark(4);
  }
  void admm_dual_phase(int want) {
    NvtxRange nv("cpadmm thresholded variables update");
    CU(launch_conv_dense(plan, hcr.p, x.p, partial.p, st));
    mark(5);
    EpiArgs a = base_args(want);
    a.x = x.p;
    a.z = z.p;
    a.nu = nu.p;
    a.mu = mu.p;
    a.v = v.p;
    a.d = d.p;
    a.pty = pty.p;
    a.rho = static_cast<float>(cfg.rho);
    a.tau1 = static_cast<float>(cfg.tau1);
    a.tau2 = static_cast<float>(cfg.tau2);
    a.thr = static_cast<float>(thr);
    set_peers(a, 2);
    launch_admm_duals(a, st);
    mark(6);
    nphase = 6;
  }

  // ---- FFT engine (circ_matvec_fft / circ_transpose_matvec, circulant.hpp:236-274) ----
  // out_real[i] = Re(idft(H^(*) . dft(u)))[i] (conj_h: C x, else C^T x), into `partial`.
  const float2* fft_product(const float2* H, bool conj_h) {
    const float2* X = fft_run(F0.p, F1.p, nfft, false, st);
    float2* Xm = const_cast<float2*>(X);
    launch_spec_mul(Xm, H, conj_h, nfft, st);
    float2* other = Xm == F0.p ? F1.p : F0.p;
    return fft_run(Xm, other, nfft, true, st);
  }
  // Four-step engine: one product = cols_fwd -> rows (twiddle, FFT, x H~, IFFT, twiddle) -> cols_inv.
  // Two chained products: the first's inverse columns (with its consumer `o1`) and the second's forward
  // columns run as one pass over T (launch_fft4_cols_inv_fwd); o1 must produce the second's input.
  void fft4_product_chain_begin(const float* u, const float2* H, bool conj_h) {
    launch_fft4_cols_fwd(f4, u, F0.p, tw1.p, st);
    launch_fft4_rows(f4, F0.p, H, conj_h, tw2.p, twA.p, twB.p, st);
  }
  void fft4_product_chain_next(const Fft4Out& o1, const float2* H2, bool conj_h2) {
    launch_fft4_cols_inv_fwd(f4, F0.p, o1, tw1.p, st);
    launch_fft4_rows(f4, F0.p, H2, conj_h2, tw2.p, twA.p, twB.p, st);
  }
  void fft4_product_chain_end(const Fft4Out& o) { launch_fft4_cols_inv(f4, F0.p, o, tw1.p, st); }
  Fft4Out product_to(float* out) const {
    Fft4Out o;
    o.out = out;
    o.n_valid = n;
    return o;
  }
  void ista_fft4_step(int want) {
    mark(0);
    Fft4Out res;  // r = y - P C x, and P^T r into the dense ud, in the inverse pass
    res.n_valid = n;
    res.mode = Fft4Out::kResidual;
    res.out = r.p;
    res.rowid = rowid.p;
    res.y = y.p;
    res.u = ud.p;
    // C x, its residual epilogue chained into the forward columns of C^T P^T r (one pass)
    fft4_product_chain_begin(x.p, chatp.p, true);
    fft4_product_chain_next(res, chatp.p, false);
    mark(1);
    mark(2);
    if (!want) {  // unchecked iteration: the x update fused into the inverse pass
      Fft4Out up;
      up.n_valid = n;
      up.mode = Fft4Out::kIstaStep;
      up.out = delta.p;
      up.x = x.p;
      up.tau = static_cast<float>(tau);
      up.thr = static_cast<float>(thr);
      fft4_product_chain_end(up);
      mark(3);
      mark(4);
      nphase = 4;
      return;
    }
    fft4_product_chain_end(product_to(partial.p));  // C^T P^T r
    mark(3);
    EpiArgs b = base_args(want);
    b.splits = 1;
    b.x = x.p;
    b.delta = delta.p;
    b.tau = static_cast<float>(tau);
    b.thr = static_cast<float>(thr);
    launch_ista_update(b, st);
    mark(4);
    nphase = 4;
  }
  void admm_fft4_step(int want) {
    mark(0);
    Fft4Out bo;  // beta = rho C^T v + sigma (z - nu), fused into the inverse pass
    bo.n_valid = n;
    bo.mode = Fft4Out::kBeta;
    bo.out = beta.p;
    bo.z = z.p;
    bo.nu = nu.p;
    bo.rho = static_cast<float>(cfg.rho);
    bo.sigma = static_cast<float>(cfg.sigma);
    // C^T v -> beta -> B beta -> x -> C x: each epilogue chained into the next product's forward columns
    fft4_product_chain_begin(v.p, chatp.p, false);
    fft4_product_chain_next(bo, bhatp.p, true);
    mark(1);
    mark(2);
    fft4_product_chain_next(product_to(x.p), chatp.p, true);  // x = B beta
    mark(3);
    mark(4);
    fft4_product_chain_end(product_to(partial.p));  // C x
    mark(5);
    EpiArgs d2 = base_args(want);
    d2.splits = 1;
    d2.x = x.p;
    d2.z = z.p;
    d2.nu = nu.p;
    d2.mu = mu.p;
    d2.v = v.p;
    d2.d = d.p;
    d2.pty = pty.p;
    d2.rho = static_cast<float>(cfg.rho);
    d2.tau1 = static_cast<float>(cfg.tau1);
    d2.tau2 = static_cast<float>(cfg.tau2);
    d2.thr = static_cast<float>(thr);
    launch_admm_duals(d2, st);
    mark(6);
    nphase = 6;
  }
  void ista_fft_step(int want) {
    mark(0);
    launch_real_to_complex(x.p, F0.p, nfft, st);
    const float2* Y = fft_product(chat.p, true);               // C x
    launch_gather_real(Y, omega32.p, partial.p, nfft, m, st);   // P C x
    mark(1);
    EpiArgs a;
    a.partial = partial.p;
    a.n = m;
    a.lo = 0;
    a.hi = m;
    a.y = y.p;
    a.r = r.p;
    launch_ista_residual_reduce(a, 1, st);
    mark(2);
    launch_embed_rows(r.p, omega32.p, F0.p, nfft, m, st);      // P^T r
    const float2* D = fft_product(chat.p, false);              // C^T P^T r
    launch_extract_real(D, partial.p, nfft, st);
    mark(3);
    EpiArgs b = base_args(want);
    b.splits = 1;
    b.x = x.p;
    b.delta = delta.p;
    b.tau = static_cast<float>(tau);
    b.thr = static_cast<float>(thr);
    launch_ista_update(b, st);
    mark(4);
    nphase = 4;
  }
  void admm_fft_step(int want) {
    mark(0);
    launch_real_to_complex(v.p, F0.p, nfft, st);
    launch_extract_real(fft_product(chat.p, false), partial.p, nfft, st);  // C^T v
    mark(1);
    EpiArgs a = base_args(0);
    a.splits = 1;
    a.beta = beta.p;
    a.z = z.p;
    a.nu = nu.p;
    a.rho = static_cast<float>(cfg.rho);
    a.sigma = static_cast<float>(cfg.sigma);
    launch_admm_beta(a, st);
    mark(2);
    launch_real_to_complex(beta.p, F0.p, nfft, st);
    launch_extract_real(fft_product(bhat.p, true), partial.p, nfft, st);   // B beta
    mark(3);
    EpiArgs bx = base_args(0);
    bx.splits = 1;
    bx.x = x.p;
    launch_admm_x(bx, st);
    mark(4);
    launch_real_to_complex(x.p, F0.p, nfft, st);
    launch_extract_real(fft_product(chat.p, true), partial.p, nfft, st);   // C x
    mark(5);
    EpiArgs d2 = base_args(want);
    d2.splits = 1;
    d2.x = x.p;
    d2.z = z.p;
    d2.nu = nu.p;
    d2.mu = mu.p;
    d2.v = v.p;
    d2.d = d.p;
    d2.pty = pty.p;
    d2.rho = static_cast<float>(cfg.rho);
    d2.tau1 = static_cast<float>(cfg.tau1);
    d2.tau2 = static_cast<float>(cfg.tau2);
    d2.thr = static_cast<float>(thr);
    launch_admm_duals(d2, st);
    mark(6);
    nphase = 6;
  }

  // ---- sharded iteration ------------------------------------------
  // Phases of one iteration and, per phase, the vector it produces and whose slices the ranks exchange:
  // ISTA 0 residual -> r (rows), 1 gradient + update -> x (outputs); cADMM 0 beta, 1 x = B beta, 2 duals -> v.
  int phase_count() const { return kind == CL_KIND_ISTA ? 2 : 3; }
  void run_phase_only(int ph, int want) {
    if (kind == CL_KIND_ISTA) {
      if (ph == 0) ista_residual();
      else ista_gradient(want);
    } else {
      if (ph == 0) admm_beta_phase();
      else if (ph == 1) admm_x_phase();
      else admm_dual_phase(want);
    }
  }
  float* phase_buffer(int ph) const {
    if (kind == CL_KIND_ISTA) return ph == 0 ? r.p : x.p;
    return ph == 0 ? beta.p : ph == 1 ? x.p : v.p;
  }
  const std::vector<std::pair<int64_t, int64_t>>& phase_ranges(int ph) const {
    return kind == CL_KIND_ISTA && ph == 0 ? rows_of : outs_of;
  }
  // every rank's slices, from the same pure host logic each rank runs (cl_shard_ranges)
  void all_ranges() {
    rows_of.clear();
    outs_of.clear();
    for (int q = 0; q < world; ++q) {
      ConvPlan pq = plan, rq = rplan;
      int64_t ol, oh, rl, rh;
      shard_ranges(kind, n, omega_host.data(), m, q, world, &pq, &rq, &ol, &oh, &rl, &rh);
      rows_of.emplace_back(rl, rh);
      outs_of.emplace_back(ol, oh);
    }
  }
  void attach_comm(Comm* c) {
    if (c->device != device) raise(CL_EPARAM, "cl_solver_attach_comm: the communicator's device is not the solver's");
    if (ipc.on) raise(CL_EPARAM, "cl_solver_attach_comm: the solver already exchanges through CUDA IPC peer stores");
    if (fft && c->world != 1) raise(CL_EPARAM, "cl_solver_attach_comm: the FFT engine runs unsharded (replicas only)");
    if (kind == CL_KIND_ADMM && c->world != 1) raise(CL_EPARAM, "cl_solver_attach_comm: the dense ADMM runs unsharded");
    CU(cudaStreamSynchronize(st));
    set_shard(c->rank, c->world);
    comm = c;
    all_ranges();
  }
  // one iteration of a solver sharded over a communicator: phase, in-place all-gather of the produced
  // slices on the solver stream, next phase ...
  void comm_step(int want) {
    for (int ph = 0; ph < phase_count(); ++ph) {
      run_phase_only(ph, want && ph == phase_count() - 1);
      comm_gather(comm, phase_buffer(ph), phase_ranges(ph), st);
    }
    CU(cudaGetLastError());
    ++t;
  }

  // ---- CUDA IPC peer stores (one process per GPU, no NCCL) ----------------------------------------------
  // The exchange vectors: ISTA {r, x}; cADMM {beta, x, v, z}.  Phase ph produces vector ph (ISTA: r, x;
  // cADMM: beta, x, v), which its epilogue stores into every rank's copy; z is pushed before downloads.
  struct PeerBlob {
    char magic[8];
    int32_t world, rank, kind, nvec;
    int64_t n, m;
    cudaIpcMemHandle_t vec[4];
    cudaIpcMemHandle_t sync;
  };
  static_assert(sizeof(PeerBlob) <= CL_PEER_BLOB_BYTES, "peer blob");
  std::vector<DevBuf<float>*> ipc_vectors() {
    if (kind == CL_KIND_ISTA) return {&r, &x};
    return {&beta, &x, &v, &z};
  }
  void ipc_export(int rk, int ws, unsigned char* out) {
    if (ws < 1 || ws > kIpcMaxRanks || rk < 0 || rk >= ws)
      raise(CL_EPARAM, "cl_solver_peer_export: need 0 <= rank < world <= 8");
    if (fft || kind == CL_KIND_ADMM)
      raise(CL_EPARAM, "cl_solver_peer_export: the sharded solve runs the direct ISTA / cADMM engine");
    if (ipc.on || comm) raise(CL_EPARAM, "cl_solver_peer_export: the solver is already attached");
    CU(cudaStreamSynchronize(st));
    set_shard(rk, ws);
    all_ranges();
    PeerBlob b;
    std::memset(&b, 0, sizeof(b));
    std::memcpy(b.magic, "CLPEER01", 8);
    b.world = ws;
    b.rank = rk;
    b.kind = kind;
    b.n = n;
    b.m = m;
    const auto vecs = ipc_vectors();
    b.nvec = static_cast<int32_t>(vecs.size());
    for (size_t i = 0; i < vecs.size(); ++i) {
      vecs[i]->make_plain(st);
      CU(cudaIpcGetMemHandle(&b.vec[i], vecs[i]->p));
    }
    if (!ipc.own) {
      CU(cudaMalloc(reinterpret_cast<void**>(&ipc.own), sizeof(IpcSync)));
      CU(cudaMemset(ipc.own, 0, sizeof(IpcSync)));
    }
    CU(cudaIpcGetMemHandle(&b.sync, ipc.own));
    std::memset(out, 0, CL_PEER_BLOB_BYTES);
    std::memcpy(out, &b, sizeof(b));
  }
  void ipc_attach(const unsigned char* blobs) {
    if (!ipc.own) raise(CL_EPARAM, "cl_solver_peer_attach: export this rank's blob first");
    std::vector<PeerBlob> b(static_cast<size_t>(world));
    for (int q = 0; q < world; ++q) std::memcpy(&b[static_cast<size_t>(q)], blobs + static_cast<size_t>(q) * CL_PEER_BLOB_BYTES, sizeof(PeerBlob));
    for (int q = 0; q < world; ++q) {
      const PeerBlob& e = b[static_cast<size_t>(q)];
      if (std::memcmp(e.magic, "CLPEER01", 8) != 0 || e.world != world || e.rank != q || e.kind != kind || e.n != n ||
          e.m != m)
        raise(CL_EPARAM, "cl_solver_peer_attach: the blobs are not every rank's export of this problem, in rank order");
    }
    const auto vecs = ipc_vectors();
    std::vector<std::vector<float*>> peer(vecs.size(), std::vector<float*>(static_cast<size_t>(world), nullptr));
    for (int q = 0; q < world; ++q) {
      if (q == rank) {
        ipc.sync.s[q] = ipc.own;
        for (size_t i = 0; i < vecs.size(); ++i) peer[i][static_cast<size_t>(q)] = vecs[i]->p;
        continue;
      }
      const PeerBlob& e = b[static_cast<size_t>(q)];
      void* sp = nullptr;
      CU(cudaIpcOpenMemHandle(&sp, e.sync, cudaIpcMemLazyEnablePeerAccess));
      ipc.opened.push_back(sp);
      ipc.sync.s[q] = static_cast<IpcSync*>(sp);
      for (size_t i = 0; i < vecs.size(); ++i) {
        void* vp = nullptr;
        CU(cudaIpcOpenMemHandle(&vp, e.vec[i], cudaIpcMemLazyEnablePeerAccess));
        ipc.opened.push_back(vp);
        peer[i][static_cast<size_t>(q)] = static_cast<float*>(vp);
      }
    }
    npeer = world - 1;
    for (int ph = 0; ph < phase_count(); ++ph) {
      int k = 0;
      for (int q = 0; q < world; ++q)
        if (q != rank) peer_out[ph][k++] = peer[static_cast<size_t>(ph)][static_cast<size_t>(q)];
    }
    if (kind == CL_KIND_CADMM)
      for (int q = 0; q < world; ++q) ipc.z.p[q] = peer[3][static_cast<size_t>(q)];
    ipc.on = true;
  }
  void ipc_barrier() {
    ++ipc.seq;
    launch_ipc_signal(ipc.sync, world, rank, ipc.seq, st);
    launch_ipc_wait(ipc.own, world, rank, ipc.seq, st);
  }
  void ipc_step(int want) {
    for (int ph = 0; ph < phase_count(); ++ph) {
      run_phase_only(ph, want && ph == phase_count() - 1);
      ipc_barrier();
    }
    CU(cudaGetLastError());
    ++t;
  }
  // every rank's share of the check sums, summed in rank order (after the last phase's barrier)
  void ipc_metrics() {
    launch_ipc_push_met(ipc.sync, world, rank, met.p, st);
    ipc_barrier();
    IpcSync h;
    CU(cudaMemcpyAsync(&h, ipc.own, sizeof(IpcSync), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (h.timed_out) raise(CL_ECOMM, "peer-store transport: a rank stopped answering (wait timed out)");
    for (int i = 0; i < 3; ++i) {
      double sum = 0.0;
      for (int q = 0; q < world; ++q) sum += h.met[q][i];
      met_host[i] = sum;
    }
    met_host[3] = 0.0;
  }

  void one_step(int want) {
    if (world != 1 && comm) {
      comm_step(want);
      return;
    }
    if (world != 1 && ipc.on) {
      ipc_step(want);
      return;
    }
    if (world != 1) raise(CL_EPARAM, "cl_solver_step: sharded solvers advance with cl_solver_run_phase");
    if (kind == CL_KIND_ADMM) {
      admm_dense_step(want);
      CU(cudaGetLastError());
      ++t;
      return;
    }
    if (fft4) {
      if (kind == CL_KIND_ISTA) ista_fft4_step(want);
      else admm_fft4_step(want);
      CU(cudaGetLastError());
      ++t;
      return;
    }
    if (fft) {
      if (kind == CL_KIND_ISTA) ista_fft_step(want);
      else admm_fft_step(want);
      CU(cudaGetLastError());
      ++t;
      return;
    }
    if (kind == CL_KIND_ISTA) {
      ista_residual();
      ista_gradient(want);
    } else {
      admm_beta_phase();
      admm_x_phase();
      admm_dual_phase(want);
    }
    CU(cudaGetLastError());
    ++t;
  }

  void collect_profile() {
    if (!profile) return;
    if (n_ev_nodes && ring_count > 0) {  // the last graph replay's ring slot
      phase_history(phase_ms, 1);
      return;
    }
    CU(cudaEventSynchronize(ev[nphase]));
    for (int i = 0; i < nphase; ++i) {
      float ms = 0.f;
      CU(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
      phase_ms[i] = ms;
    }
  }
  // Phase times of the last `want` graph replays recorded in the ring (profile mode 2), oldest first:
  // out[k * nphase + i].  Returns the number of replays written.
  int64_t phase_history(double* out, int64_t want) {
    if (profile != 2 || !n_ev_nodes) return 0;
    const int64_t have = std::min<int64_t>({ring_count, static_cast<int64_t>(kRing), want});
    for (int64_t k = 0; k < have; ++k) {
      const cudaEvent_t* slot = ring.data() + ((ring_count - have + k) % kRing) * kPhaseEvents;
      CU(cudaEventSynchronize(slot[nphase]));
      for (int i = 0; i < nphase; ++i) {
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, slot[i], slot[i + 1]));
        out[k * nphase + i] = ms;
      }
    }
    return have;
  }

  bool use_graph() const {
    static const bool off = [] {
      const char* v = getenv("CLB_NO_GRAPH");
      return v && v[0] == '1';
    }();
    return !off && world == 1 && profile != 1;  // mode-1 per-phase timing runs eagerly
  }

  void build_graph() {
    if (graph) return;
    const int64_t t0 = t;
    cudaGraph_t g;
    CU(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    one_step(0);
    CU(cudaStreamEndCapture(st, &g));
    n_ev_nodes = 0;
    if (profile == 2) {  // find the event-record node of each phase boundary
      size_t cnt = 0;
      CU(cudaGraphGetNodes(g, nullptr, &cnt));
      std::vector<cudaGraphNode_t> nodes(cnt);
      CU(cudaGraphGetNodes(g, nodes.data(), &cnt));
      for (cudaGraphNode_t nd : nodes) {
        cudaGraphNodeType ty;
        CU(cudaGraphNodeGetType(nd, &ty));
        if (ty != cudaGraphNodeTypeEventRecord) continue;
        cudaEvent_t e;
        CU(cudaGraphEventRecordNodeGetEvent(nd, &e));
        for (int i = 0; i < kPhaseEvents; ++i)
          if (ev[i] == e) ev_node[i] = nd;
      }
      n_ev_nodes = nphase + 1;
      if (ring.empty()) {
        ring.resize(static_cast<size_t>(kRing) * kPhaseEvents);
        for (auto& e : ring) CU(cudaEventCreate(&e));
      }
    }
    CU(cudaGraphInstantiate(&graph, g, 0));
    graph_src = g;
    t = t0;  // capture does not execute
    trace("run: graph captured");
  }

  bool use_small_fft() const {
    return fft && !fft4 && small_fft && world == 1 && !profile &&
           (kind == CL_KIND_ISTA ? small_fft_supported(n) : small_fft_cadmm_supported(n));
  }

  bool use_coop_ista() const {
    return kind == CL_KIND_ISTA && !fft && world == 1 && !profile && coop_cadmm_supported(n);
  }
  bool use_coop_cadmm() const {
    return kind == CL_KIND_CADMM && !fft && world == 1 && !profile && coop_cadmm_supported(n);
  }

  // One persistent launch of `it` unchecked iterations (small n), if this solver has such a path.
  bool persistent_launch(int it) {
    if (use_coop_ista()) {
      CU(launch_coop_ista(n, m, hc.p, hcr.p, omega32.p, y.p, x.p, r.p, delta.p, partial.p, static_cast<float>(tau),
                          static_cast<float>(thr), it, st));
    } else if (use_coop_cadmm()) {
      CU(launch_coop_cadmm(n, hc.p, hbr.p, hcr.p, d.p, pty.p, x.p, z.p, nu.p, mu.p, v.p, beta.p, partial.p,
                           static_cast<float>(cfg.rho), static_cast<float>(cfg.sigma), static_cast<float>(cfg.tau1),
                           static_cast<float>(cfg.tau2), static_cast<float>(thr), it, st));
    } else if (use_small_fft()) {
      if (kind == CL_KIND_ISTA)
        CU(launch_small_fft_ista(n, m, chatS.p, twS.p, omega32.p, y.p, x.p, r.p, delta.p, static_cast<float>(tau),
                                 static_cast<float>(thr), it, st));
      else
        CU(launch_small_fft_cadmm(n, chatS.p, bhatS.p, twS.p, d.p, pty.p, x.p, z.p, nu.p, mu.p, v.p, beta.p,
                                  static_cast<float>(cfg.rho), static_cast<float>(cfg.sigma),
                                  static_cast<float>(cfg.tau1), static_cast<float>(cfg.tau2),
                                  static_cast<float>(thr), it, st));
    } else {
      return false;
    }
    return true;
  }

  void step(int64_t iters) {
    if (iters > 0 && (use_coop_ista() || use_coop_cadmm() || use_small_fft())) {
      // the persistent kernels count iterations in int: longer requests run as several launches
      constexpr int64_t kMaxLaunchIters = int64_t(1) << 30;
      CU(cudaEventRecord(step_ev[0], st));
      for (int64_t done = 0; done < iters; done += kMaxLaunchIters)
        persistent_launch(static_cast<int>(std::min(kMaxLaunchIters, iters - done)));
      t += iters;
      CU(cudaEventRecord(step_ev[1], st));
      return;
    }
    const bool graphed = iters > 0 && use_graph();
    if (graphed) build_graph();
    CU(cudaEventRecord(step_ev[0], st));
    for (int64_t k = 0; k < iters; ++k) {
      if (graphed) {
        if (n_ev_nodes) {  // this replay stamps its phase boundaries into its own ring slot
          cudaEvent_t* slot = ring.data() + (ring_count % kRing) * kPhaseEvents;
          for (int i = 0; i < n_ev_nodes; ++i) CU(cudaGraphExecEventRecordNodeSetEvent(graph, ev_node[i], slot[i]));
          ++ring_count;
        }
        CU(cudaGraphLaunch(graph, st));
        ++t;
      } else {
        one_step(0);
      }
    }
    CU(cudaEventRecord(step_ev[1], st));
  }

  // Checked step: metric per run_loop solvers.hpp:454-456.
  void step_checked(double* metric, int* nonfinite) {
    one_step(1);
    launch_metrics_final(blk.p, met.p, st);
    if (world != 1 && ipc.on) {
      ipc_metrics();
      collect_profile();
      metric_from(met_host, metric, nonfinite);
      return;
    }
    if (world != 1 && comm) comm_allreduce_sum(comm, met.p, 3, st);  // every rank's share of the sums
    CU(cudaMemcpyAsync(met_host, met.p, sizeof(double) * 4, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    collect_profile();
    metric_from(met_host, metric, nonfinite);
  }
  void metric_from(const double* mh, double* metric, int* nonfinite) const {
    const double nn = static_cast<double>(n);
    *nonfinite = mh[2] > 0.0;
    if (has_truth) *metric = n > 0 ? mh[1] / nn : 0.0;
    else *metric = std::sqrt(mh[0]) * (n > 0 ? 1.0 / std::sqrt(nn) : 1.0);
  }
  void download_iterate(double* out) { download(iterate_full(), n, out); }
  // optional ground truth: the check metric becomes the MSE (run_loop solvers.hpp:437)
  void set_truth(const double* truth_n) {
    CU(cudaSetDevice(device));
    if (!truth_n) {
      has_truth = false;
      return;
    }
    const std::vector<float> tf = to_f32(truth_n, n);
    truth.alloc(static_cast<size_t>(n), st);
    truth.upload(tf.data(), tf.size(), st);
    CU(cudaStreamSynchronize(st));
    has_truth = true;
  }
  // the reported iterate, complete on this rank (cADMM's z is slice-local in a sharded solve)
  float* iterate_full() {
    int64_t len = 0;
    float* p = field_ptr(kind == CL_KIND_ISTA ? "x" : "z", &len);
    if (world != 1 && comm && kind != CL_KIND_ISTA) comm_gather(comm, p, outs_of, st);
    if (world != 1 && ipc.on && kind != CL_KIND_ISTA) {
      launch_ipc_push_slice(ipc.z, world, rank, p, out_lo, out_hi, st);
      ipc_barrier();
    }
    return p;
  }

  // device fp32 -> host fp64 through the pooled pinned staging buffer
  void download(const float* p, int64_t len, double* out) {
    if (len <= 0) return;
    float* stage = res.staging(static_cast<size_t>(len));
    CU(cudaMemcpyAsync(stage, p, sizeof(float) * len, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    for (int64_t i = 0; i < len; ++i) out[i] = stage[i];
  }

  float* field_ptr(const std::string& f, int64_t* len) {
    *len = n;
    if (kind == CL_KIND_ISTA) {
      if (f == "x") return x.p;
      if (f == "delta") return delta.p;
      if (f == "c") return hc.p;
      *len = m;
      if (f == "r") return r.p;
      if (f == "y") return y.p;
    } else if (kind == CL_KIND_ADMM) {
      if (f == "x") return x.p;
      if (f == "z") return z.p;
      if (f == "u") return u.p;
      if (f == "rhs") return rhs.p;
      if (f == "aty") return aty.p;
      if (f == "B") {
        *len = n * n;
        return Bm.p;
      }
    } else {
      if (f == "x") return x.p;
      if (f == "z") return z.p;
      if (f == "nu") return nu.p;
      if (f == "mu") return mu.p;
      if (f == "v") return v.p;
      if (f == "beta") return beta.p;
      if (f == "c") return hc.p;
      if (f == "d") return d.p;
      if (f == "pty") return pty.p;
      if (f == "b") return hbr.p;  // reversed on device; un-reversed on get
    }
    raise(CL_EPARAM, "cl_solver_get: unknown field '" + f + "'");
  }
};

// ---- fp64 circulant products of host vectors on the device -------------------
// out = Re idft(conj?(dft(a)) . dft(b)) (fft.hpp:74-89 residue check), the
// transform behind measure (circulant.hpp:277-282) and compose_rows
// (circulant.hpp:337-343).  Power-of-two n >= 2^14 with a CUDA device;
// otherwise the host fp64 DFT (host_setup.cpp) runs.
static bool device_product_ok(int64_t n) {
  const char* v = std::getenv("CLB_HOST_SETUP");
  if ((v && v[0] == '1') || !is_pow2(n) || n < (int64_t(1) << 14)) return false;
  int count = 0;
  return cudaGetDeviceCount(&count) == cudaSuccess && count > 0;
}
static void device_product(const double* a, const double* b, int64_t n, bool conj_a, double* out) {
  cudaStream_t st;
  CU(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct Guard {
    cudaStream_t s;
    ~Guard() {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  } guard{st};
  int dev = 0;
  CU(cudaGetDevice(&dev));
  reserve_pool(dev);
  const size_t nn = static_cast<size_t>(n);
  DevBuf<double> ra, rb, ro;
  DevBuf<double2> A, B, W;
  DevBuf<unsigned long long> red;
  ra.alloc(nn, st);
  rb.alloc(nn, st);
  ro.alloc(nn, st);
  A.alloc(nn, st);
  B.alloc(nn, st);
  W.alloc(nn, st);
  red.alloc(4, st);
  ra.upload(a, nn, st);
  rb.upload(b, nn, st);
  CU(cudaMemsetAsync(red.p, 0, sizeof(unsigned long long) * 4, st));
  launch_real_to_complex64(ra.p, A.p, n, st);
  const double2* SA = fft64_run(A.p, W.p, n, false, st);
  double2* freeAW = SA == A.p ? W.p : A.p;
  launch_real_to_complex64(rb.p, B.p, n, st);
  double2* SB = const_cast<double2*>(fft64_run(B.p, freeAW, n, false, st));
  launch_cmul64(SA, SB, conj_a, n, st);
  double2* scratch = SB == B.p ? freeAW : B.p;  // neither SB nor (needed no more) SA's live data
  const double2* Y = fft64_run(SB, scratch, n, true, st);
  launch_real_part64(Y, ro.p, red.p + 2, red.p + 3, n, st);
  CU(cudaGetLastError());
  unsigned long long h[4];
  CU(cudaMemcpyAsync(h, red.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(out, ro.p, sizeof(double) * nn, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  double re, im;
  std::memcpy(&re, &h[2], sizeof(double));
  std::memcpy(&im, &h[3], sizeof(double));
  if (im > 1e-10 * std::max(1.0, re)) {
    std::ostringstream msg;
    msg << "inverse DFT of a real-valued quantity has imaginary residue " << im << " (relative tolerance 1e-10)";
    raise(CL_ECONSIST, msg.str());
  }
}
// y[t] = (C x)[omega[t]] (measure, sensing.hpp:171-182)
static void measure_any(const double* c, const int64_t* omega, int64_t n, int64_t m, const double* x, double* y) {
  if (!device_product_ok(n)) {
    measure(c, omega, n, m, x, y);
    return;
  }
  std::vector<double> cx(static_cast<size_t>(n));
  device_product(c, x, n, true, cx.data());  // C x = idft(conj(c^) x^)
  for (int64_t t = 0; t < m; ++t) y[t] = cx[static_cast<size_t>(omega[t])];
}
static bool identity_row(const double* r, int64_t n) {  // deblur.hpp:41-46
  if (n < 1 || r[0] != 1.0) return false;
  for (int64_t i = 1; i < n; ++i)
    if (r[i] != 0.0) return false;
  return true;
}
static void compose_any(const double* c, const double* b, int64_t n, double* out) {
  if (!device_product_ok(n) || identity_row(b, n) || identity_row(c, n)) {
    compose_rows(c, b, n, out);  // (also the identity short-circuits of deblur.hpp:53-64)
    return;
  }
  device_product(c, b, n, false, out);
}

// ---- device product helpers (cl_circ_matvec & co.) --------------------------
struct ScratchProduct {
  static void circ(int device, int64_t n, const double* c, const double* xin, int transpose, double* out) {
    CU(cudaSetDevice(device));
    conv_kernels_init();
    reserve_pool(device);
    cudaStream_t st;
    CU(cudaStreamCreate(&st));
    ConvPlan p = make_dense_plan(n);
    std::vector<float> cf = to_f32(c, n);
    if (!transpose) cf = reversed(cf);  // C x = conv(c_rev, x)
    const std::vector<float> xf = to_f32(xin, n);
    DevBuf<float> h, u, part, o, scr;
    scr.alloc(tc_scratch_floats());
    p.tc_scratch = scr.p;
    h.alloc(static_cast<size_t>(n));
    h.upload(cf.data(), cf.size(), st);
    u.alloc(static_cast<size_t>(n));
    u.upload(xf.data(), xf.size(), st);
    part.alloc(static_cast<size_t>(p.splits * n));
    o.alloc(static_cast<size_t>(n));
    CU(launch_conv_dense(p, h.p, u.p, part.p, st));
    EpiArgs a;
    a.partial = part.p;
    a.splits = p.splits;
    a.n = n;
    a.lo = 0;
    a.hi = n;
    a.x = o.p;
    launch_admm_x(a, st);
    CU(cudaGetLastError());
    std::vector<float> res(static_cast<size_t>(n));
    CU(cudaMemcpyAsync(res.data(), o.p, sizeof(float) * n, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    CU(cudaStreamDestroy(st));
    for (int64_t i = 0; i < n; ++i) out[i] = res[static_cast<size_t>(i)];
  }
};

// run_loop solvers.hpp:426-472 (+ ista_run / cadmm_run / admm_dense_run :479-534) over a single solver
// or a group of shards: S provides step(k), step_checked(&value, &nonfinite), download_iterate(out), and
// kind / n / m / has_truth / setup_seconds.
template <typename S>
void run_loop(S& s, const cl_config& cfg, cl_report* rep, double* final_x, int64_t* trace_iter, double* trace_value,
              double* trace_seconds, int64_t trace_cap) {
  if (cfg.max_iter < 0) raise(CL_EPARAM, "solver: max_iter must be >= 0");         // solvers.hpp:432
  if (cfg.check_every < 1) raise(CL_EPARAM, "solver: check_every must be >= 1");  // :433-434
  const auto t0 = std::chrono::steady_clock::now();
  std::memset(rep, 0, sizeof(*rep));
  rep->metric = s.has_truth ? CL_METRIC_MSE_VS_TRUTH : CL_METRIC_ITERATE_CHANGE;
  rep->final_metric = std::numeric_limits<double>::quiet_NaN();
  const bool has_target = !std::isnan(cfg.target_mse);
  int64_t t = 0, tl = 0;
  while (t < cfg.max_iter) {
    // next check point: t % check_every == 0 or t == max_iter (solvers.hpp:452)
    int64_t next = ((t / cfg.check_every) + 1) * cfg.check_every;
    if (next > cfg.max_iter) next = cfg.max_iter;
    if (next - t > 1) s.step(next - t - 1);
    trace("run: unchecked steps queued");
    double value = 0.0;
    int nonfinite = 0;
    s.step_checked(&value, &nonfinite);
    trace("run: checked step (sync)");
    t = next;
    if (nonfinite)
      raise(CL_EDIVERGE, s.kind == CL_KIND_ISTA    ? "ista_run: iterate became non-finite"
                       : s.kind == CL_KIND_CADMM ? "cadmm_run: iterate became non-finite"
                                                 : "admm_dense_run: iterate became non-finite");
    if (tl < trace_cap) {
      if (trace_iter) trace_iter[tl] = t;
      if (trace_value) trace_value[tl] = value;
      if (trace_seconds) trace_seconds[tl] = seconds_since(t0);  // TracePoint::elapsed_seconds (:457-459)
    }
    ++tl;
    rep->final_metric = value;
    if (has_target && value <= cfg.target_mse) {
      rep->reached_target = 1;
      break;
    }
  }
  rep->iterations = t;
  rep->trace_len = tl;
  rep->setup_seconds = s.setup_seconds;
  rep->total_seconds = seconds_since(t0) + s.setup_seconds;
  rep->footprint_bytes = footprint(s.kind, s.n, s.m, sizeof(float));
  if (final_x) {
    s.download_iterate(final_x);
    trace("run: iterate download");
  }
}

// ---- a sharded solve driven from one process (cl_group_*) --------------------------------
// One Solver per rank, each on its own device and stream, sharded (rank, world).  An iteration runs phase
// by phase across the ranks; after each phase the produced slices are exchanged:
//  * kNccl: one NCCL communicator per device (ncclCommInitAll), the ranks' in-place broadcasts issued
//    in one NCCL group (a single thread drives every device);
//  * kCopy: device-to-device copies ordered by events (ranks may share a device; the exchange and phase
//    logic of the NCCL path without NCCL -- the one-GPU test of the 2/4/8-rank data plane);
//  * kPeer: no separate exchange at all -- each phase's epilogue kernel stores its slice straight into every
//    rank's copy of the vector (EpiArgs::peer; NVLink peer stores across GPUs), and the ranks' streams only
//    wait for each other's phase before the next one (the all-gather fused into the producing kernel).
struct Group {
  enum Transport { kNccl = CL_TRANSPORT_NCCL, kCopy = CL_TRANSPORT_COPY, kPeer = CL_TRANSPORT_PEER };
  int kind = 0;
  int64_t n = 0, m = 0;
  bool has_truth = false;
  double setup_seconds = 0.0;
  Transport transport = kNccl;
  std::vector<std::unique_ptr<Solver>> ranks;
  std::vector<Comm*> comms;
  std::vector<cudaEvent_t> done;  // per rank: its phase finished (kCopy)

  ~Group() {
    for (auto& s : ranks)
      if (s) {
        cudaSetDevice(s->device);
        cudaStreamSynchronize(s->st);
      }
    for (auto e : done) cudaEventDestroy(e);
    ranks.clear();
    for (Comm* c : comms) comm_destroy(c);
  }
  int world() const { return static_cast<int>(ranks.size()); }

  void exchange(int ph) {
    if (world() == 1) return;
    if (transport == kNccl) {
      comm_group_start();
      for (auto& s : ranks) {
        CU(cudaSetDevice(s->device));
        comm_gather(s->comm, s->phase_buffer(ph), s->phase_ranges(ph), s->st);
      }
      comm_group_end();
      return;
    }
    for (int r = 0; r < world(); ++r) {
      CU(cudaSetDevice(ranks[static_cast<size_t>(r)]->device));
      CU(cudaEventRecord(done[static_cast<size_t>(r)], ranks[static_cast<size_t>(r)]->st));
    }
    if (transport == kPeer) {  // the slices are already in place: order the next phase after every rank's
      for (int q = 0; q < world(); ++q) {
        Solver& dst = *ranks[static_cast<size_t>(q)];
        CU(cudaSetDevice(dst.device));
        for (int r = 0; r < world(); ++r)
          if (r != q) CU(cudaStreamWaitEvent(dst.st, done[static_cast<size_t>(r)], 0));
      }
      return;
    }
    for (int q = 0; q < world(); ++q) {
      Solver& dst = *ranks[static_cast<size_t>(q)];
      CU(cudaSetDevice(dst.device));
      for (int r = 0; r < world(); ++r) {
        if (r == q) continue;
        Solver& src = *ranks[static_cast<size_t>(r)];
        const auto rg = src.phase_ranges(ph)[static_cast<size_t>(r)];
        if (rg.second <= rg.first) continue;
        CU(cudaStreamWaitEvent(dst.st, done[static_cast<size_t>(r)], 0));
        CU(cudaMemcpyPeerAsync(dst.phase_buffer(ph) + rg.first, dst.device, src.phase_buffer(ph) + rg.first,
                               src.device, sizeof(float) * static_cast<size_t>(rg.second - rg.first), dst.st));
      }
    }
  }
  void iteration(int want) {
    const int np = ranks.front()->phase_count();
    for (int ph = 0; ph < np; ++ph) {
      for (auto& s : ranks) {
        CU(cudaSetDevice(s->device));
        s->run_phase_only(ph, want && ph == np - 1);
      }
      exchange(ph);
    }
    for (auto& s : ranks) {
      CU(cudaGetLastError());
      ++s->t;
    }
  }
  void step(int64_t iters) {
    for (int64_t k = 0; k < iters; ++k) iteration(0);
  }
  void step_checked(double* metric, int* nonfinite) {
    iteration(1);
    double sum[3] = {0, 0, 0};
    if (transport == kNccl) {
      for (auto& s : ranks) {
        CU(cudaSetDevice(s->device));
        launch_metrics_final(s->blk.p, s->met.p, s->st);
      }
      if (world() > 1) {
        comm_group_start();
        for (auto& s : ranks) {
          CU(cudaSetDevice(s->device));
          comm_allreduce_sum(s->comm, s->met.p, 3, s->st);
        }
        comm_group_end();
      }
      Solver& s0 = *ranks.front();
      CU(cudaSetDevice(s0.device));
      CU(cudaMemcpyAsync(s0.met_host, s0.met.p, sizeof(double) * 4, cudaMemcpyDeviceToHost, s0.st));
      CU(cudaStreamSynchronize(s0.st));
      for (int i = 0; i < 3; ++i) sum[i] = s0.met_host[i];
    } else {  // every rank's share, summed in rank order
      for (auto& s : ranks) {
        CU(cudaSetDevice(s->device));
        launch_metrics_final(s->blk.p, s->met.p, s->st);
        CU(cudaMemcpyAsync(s->met_host, s->met.p, sizeof(double) * 4, cudaMemcpyDeviceToHost, s->st));
      }
      for (auto& s : ranks) {
        CU(cudaSetDevice(s->device));
        CU(cudaStreamSynchronize(s->st));
        for (int i = 0; i < 3; ++i) sum[i] += s->met_host[i];
      }
    }
    const double full[4] = {sum[0], sum[1], sum[2], 0.0};
    ranks.front()->metric_from(full, metric, nonfinite);
  }
  // a vector assembled from the ranks' slices (complete whether or not the field is exchanged)
  void get(const std::string& f, double* out) {
    int64_t len = 0;
    for (int r = 0; r < world(); ++r) {
      Solver& s = *ranks[static_cast<size_t>(r)];
      CU(cudaSetDevice(s.device));
      float* p = s.field_ptr(f, &len);
      std::vector<double> tmp(static_cast<size_t>(len));
      s.download(p, len, tmp.data());
      const bool rows = kind == CL_KIND_ISTA && (f == "r" || f == "y");
      std::pair<int64_t, int64_t> rg = rows ? s.rows_of[static_cast<size_t>(r)] : s.outs_of[static_cast<size_t>(r)];
      if (f == "c" || f == "y" || f == "b" || f == "d" || f == "pty") rg = {r == 0 ? 0 : len, r == 0 ? len : len};
      for (int64_t i = rg.first; i < rg.second && i < len; ++i) out[i] = tmp[static_cast<size_t>(i)];
    }
    if (f == "b") {  // stored reversed on the device
      std::vector<double> tmp(out, out + len);
      for (int64_t k = 0; k < len; ++k) out[k] = tmp[static_cast<size_t>((len - k) % len)];
    }
  }
  void download_iterate(double* out) { get(kind == CL_KIND_ISTA ? "x" : "z", out); }
};

}  // namespace clb

// ===========================================================================
// C-ABI
// ===========================================================================
using namespace clb;

struct cl_solver {
  std::unique_ptr<Solver> impl;
};

#define CL_GUARD_BEGIN try {
#define CL_GUARD_END                              \
  return CL_OK;                                   \
  }                                               \
  catch (const Failure& f) {                      \
    set_error(f.msg);                             \
    return f.code;                                \
  }                                               \
  catch (const std::bad_alloc&) {                 \
    set_error("host allocation failed");          \
    return CL_ECAPACITY;                          \
  }                                               \
  catch (const std::exception& e) {               \
    set_error(e.what());                          \
    return CL_ECUDA;                              \
  }

extern "C" {

int cl_abi_version(void) { return CL_ABI_VERSION; }
const char* cl_last_error(void) { return last_error().c_str(); }

void cl_config_default(cl_config* c) {  // solvers.hpp:112-125
  c->alpha = 1e-4;
  c->tau = 0.0;
  c->rho = 0.1;
  c->sigma = 0.1;
  c->tau1 = 1.0;
  c->tau2 = 1.0;
  c->max_iter = 100000;
  c->target_mse = std::numeric_limits<double>::quiet_NaN();
  c->check_every = 10;
  c->pairing = CL_PAIRING_LITERAL;
  c->engine = CL_ENGINE_DIRECT;
  c->dense_cap = 4096;  // circulant.hpp:31 kDenseCap
}

cl_status cl_device_count(int* count) {
  CL_GUARD_BEGIN
  *count = 0;
  CU(cudaGetDeviceCount(count));
  CL_GUARD_END
}

cl_status cl_gen_sparse_signal(int64_t n, int64_t k, uint64_t seed, double* values, int64_t* support) {
  CL_GUARD_BEGIN
  gen_sparse_signal(n, k, seed, values, support);
  CL_GUARD_END
}
cl_status cl_gen_circulant_sensing(int64_t n, int64_t m, uint64_t seed, double* c, int64_t* omega) {
  CL_GUARD_BEGIN
  gen_circulant_sensing(n, m, seed, c, omega);
  CL_GUARD_END
}
cl_status cl_measure(int64_t n, int64_t m, const double* c, const int64_t* omega, const double* x, double* y) {
  CL_GUARD_BEGIN
  check_mask(omega, m, n);
  measure_any(c, omega, n, m, x, y);
  CL_GUARD_END
}
cl_status cl_make_problem(int64_t n, int64_t m, int64_t k, uint64_t seed, double* c, int64_t* omega, double* x_true,
                          int64_t* support, double* y) {
  CL_GUARD_BEGIN
  gen_sparse_signal(n, k, seed, x_true, support);
  gen_circulant_sensing(n, m, seed, c, omega);
  measure_any(c, omega, n, m, x_true, y);
  CL_GUARD_END
}
cl_status cl_gen_star_field(int64_t w, int64_t h, double density, uint64_t seed, double* px) {
  CL_GUARD_BEGIN
  gen_star_field(w, h, density, seed, px);
  CL_GUARD_END
}
cl_status cl_blur_row(int64_t n, int64_t L, double* row) {
  CL_GUARD_BEGIN
  blur_row(n, L, row);
  CL_GUARD_END
}
cl_status cl_compose_rows(int64_t n, const double* c, const double* b, double* out) {
  CL_GUARD_BEGIN
  compose_any(c, b, n, out);
  CL_GUARD_END
}
cl_status cl_write_vector(const char* path, const double* v, int64_t n) {
  CL_GUARD_BEGIN
  if (!path) raise(CL_EPARAM, "write_vector: null path");
  if (n < 0 || (n > 0 && !v)) raise(CL_EPARAM, "write_vector: bad vector");
  write_vector_file(path, v, n);
  CL_GUARD_END
}
cl_status cl_read_vector(const char* path, double* out, int64_t cap, int64_t* len) {
  CL_GUARD_BEGIN
  if (!path || !len) raise(CL_EPARAM, "read_vector: null argument");
  const std::vector<double> v = read_vector_file(path);
  *len = static_cast<int64_t>(v.size());
  if (out && cap >= *len) std::copy(v.begin(), v.end(), out);
  CL_GUARD_END
}
cl_status cl_write_operator(const char* path, int64_t n, int64_t m, const double* row, const int64_t* omega) {
  CL_GUARD_BEGIN
  if (!path) raise(CL_EPARAM, "write_operator: null path");
  if (n < 0 || m < 0 || m > n) raise(CL_EDIM, "write_operator: need 0 <= m <= n");
  write_operator_file(path, n, m, row, omega);
  CL_GUARD_END
}
cl_status cl_read_operator(const char* path, double* row, int64_t cap_n, int64_t* omega, int64_t cap_m, int64_t* n,
                           int64_t* m) {
  CL_GUARD_BEGIN
  if (!path || !n || !m) raise(CL_EPARAM, "read_operator: null argument");
  std::vector<double> r;
  std::vector<int64_t> om;
  read_operator_file(path, &r, &om);
  *n = static_cast<int64_t>(r.size());
  *m = static_cast<int64_t>(om.size());
  if (row && cap_n >= *n) std::copy(r.begin(), r.end(), row);
  if (omega && cap_m >= *m) std::copy(om.begin(), om.end(), omega);
  CL_GUARD_END
}
cl_status cl_write_pgm(const char* path, int64_t width, int64_t height, const double* pixels) {
  CL_GUARD_BEGIN
  if (!path) raise(CL_EPARAM, "write_pgm: null path");
  if (width >= 1 && height >= 1 && !pixels) raise(CL_EPARAM, "write_pgm: null pixels");
  write_pgm_file(path, width, height, pixels);
  CL_GUARD_END
}
cl_status cl_read_pgm(const char* path, double* pixels, int64_t cap, int64_t* width, int64_t* height) {
  CL_GUARD_BEGIN
  if (!path || !width || !height) raise(CL_EPARAM, "read_pgm: null argument");
  std::vector<double> px;
  read_pgm_file(path, &px, width, height);
  if (pixels && cap >= static_cast<int64_t>(px.size())) std::copy(px.begin(), px.end(), pixels);
  CL_GUARD_END
}
double cl_bench_iters_per_second(const cl_bench_row* row) { return row ? bench_iters_per_second(*row) : 0.0; }
static void copy_text(const std::string& t, char* buf, int64_t cap, int64_t* len) {
  if (len) *len = static_cast<int64_t>(t.size());
  if (buf && cap > static_cast<int64_t>(t.size())) {
    std::memcpy(buf, t.data(), t.size());
    buf[t.size()] = '\0';
  }
}
cl_status cl_bench_csv_header(char* buf, int64_t cap, int64_t* len) {
  CL_GUARD_BEGIN
  copy_text(bench_csv_header(), buf, cap, len);
  CL_GUARD_END
}
cl_status cl_bench_csv_row(const cl_bench_row* row, char* buf, int64_t cap, int64_t* len) {
  CL_GUARD_BEGIN
  if (!row) raise(CL_EPARAM, "bench row: null");
  copy_text(bench_csv_row(*row), buf, cap, len);
  CL_GUARD_END
}
cl_status cl_matvec_scheme_bench(int device, int64_t n, int scheme, int repeats, uint64_t seed, int64_t dense_cap,
                                 double* min_s, double* mean_s, uint64_t* unique_fetches, uint64_t* vector_fetches,
                                 double* checksum) {
  CL_GUARD_BEGIN
  if (n < 1) raise(CL_EPARAM, "matvec_scheme_bench: n must be >= 1");
  if (repeats < 1) raise(CL_EPARAM, "matvec_scheme_bench: repeats must be >= 1");
  if (scheme != 0 && scheme != 1) raise(CL_EPARAM, "matvec_scheme_bench: scheme must be 0 (circulant) or 1 (reference)");
  if (scheme == 1 && n > dense_cap) {
    std::ostringstream msg;
    msg << "matvec_scheme_bench: n = " << n << " exceeds the dense cap " << dense_cap;
    raise(CL_ECAPACITY, msg.str());
  }
  const uint64_t un = static_cast<uint64_t>(n);
  *unique_fetches = scheme == 0 ? 2 * un : un * un + un;  // parallel.hpp:355-361
  *vector_fetches = scheme == 0 ? 2 * un : 3 * un;
  std::vector<double> row(static_cast<size_t>(n)), xin(static_cast<size_t>(n));
  scheme_bench_inputs(n, seed, row.data(), xin.data());
  CU(cudaSetDevice(device));
  conv_kernels_init();
  reserve_pool(device);
  cudaStream_t st;
  CU(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct Guard {
    cudaStream_t s;
    cudaEvent_t e[2] = {};
    ~Guard() {
      cudaStreamSynchronize(s);
      for (auto& v : e)
        if (v) cudaEventDestroy(v);
      cudaStreamDestroy(s);
    }
  } g{st};
  CU(cudaEventCreate(&g.e[0]));
  CU(cudaEventCreate(&g.e[1]));
  const size_t nn = static_cast<size_t>(n);
  DevBuf<float> h, x, out, part, M, scr;
  const std::vector<float> xf = to_f32(xin.data(), n);
  x.alloc(nn, st);
  x.upload(xf.data(), nn, st);
  out.alloc(nn, st);
  ConvPlan plan;
  if (scheme == 0) {
    plan = make_dense_plan(n);
    scr.alloc(tc_scratch_floats(), st);
    plan.tc_scratch = scr.p;
    const std::vector<float> crf = reversed(to_f32(row.data(), n));  // C x = conv(c_rev, x)
    h.alloc(nn, st);
    h.upload(crf.data(), nn, st);
    part.alloc(static_cast<size_t>(plan.splits) * nn, st);
  } else {
    const std::vector<float> cf = to_f32(row.data(), n);
    h.alloc(nn, st);
    h.upload(cf.data(), nn, st);
    M.alloc(nn * nn, st);
    launch_materialize_circulant(h.p, M.p, n, st);
  }
  std::vector<float> res(nn);
  double total = 0.0, best = 1e300, sum = 0.0;
  for (int rep = 0; rep < repeats; ++rep) {
    CU(cudaEventRecord(g.e[0], st));
    if (scheme == 0) {
      CU(launch_conv_dense(plan, h.p, x.p, part.p, st));
      EpiArgs a;
      a.partial = part.p;
      a.splits = plan.splits;
      a.n = n;
      a.lo = 0;
      a.hi = n;
      a.x = out.p;
      launch_admm_x(a, st);
    } else {
      launch_dense_gemv(M.p, x.p, out.p, n, st);
    }
    CU(cudaEventRecord(g.e[1], st));
    CU(cudaMemcpyAsync(res.data(), out.p, sizeof(float) * nn, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    CU(cudaGetLastError());
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, g.e[0], g.e[1]));
    total += ms * 1e-3;
    best = std::min(best, ms * 1e-3);
    for (float v : res) sum += v;
  }
  *min_s = best;
  *mean_s = total / repeats;
  *checksum = sum;
  CL_GUARD_END
}
cl_status cl_spectral_norm(int64_t n, const double* c, double* out) {
  CL_GUARD_BEGIN
  *out = spectral_norm(c, n);
  CL_GUARD_END
}
cl_status cl_regularized_gram_inverse(int64_t n, const double* c, double rho, double sigma, double* b) {
  CL_GUARD_BEGIN
  regularized_gram_inverse(c, n, rho, sigma, b);
  CL_GUARD_END
}
cl_status cl_mask_gram_inverse(int64_t n, int64_t m, const int64_t* omega, double rho, double* d) {
  CL_GUARD_BEGIN
  check_mask(omega, m, n);
  mask_gram_inverse(omega, m, n, rho, d);
  CL_GUARD_END
}

cl_status cl_circ_matvec(int device, int64_t n, const double* c, const double* x, int transpose, double* out) {
  CL_GUARD_BEGIN
  NvtxRange nv("cl_circ_matvec");
  if (n < 1) raise(CL_EDIM, "circ_matvec: empty operator");
  ScratchProduct::circ(device, n, c, x, transpose, out);
  CL_GUARD_END
}

cl_status cl_partial_matvec(int device, int64_t n, int64_t m, const double* c, const int64_t* omega, const double* xin,
                            double* out_m) {
  CL_GUARD_BEGIN
  NvtxRange nv("cl_partial_matvec");
  check_mask(omega, m, n);
  // A x through the residual kernel with y = 0: r = -A x.
  std::vector<double> zero(static_cast<size_t>(m), 0.0);
  cl_config cfg;
  cl_config_default(&cfg);
  Solver s;
  s.kind = CL_KIND_ISTA;
  s.device = device;
  s.n = n;
  s.m = m;
  s.cfg = cfg;
  s.init_device();
  s.plan = make_plan(n, grad_R(n));
  s.rplan = make_plan(n, res_R(n));
  const std::vector<float> crf = reversed(to_f32(c, n));
  s.hcr.alloc(static_cast<size_t>(n), s.st);
  s.hcr.upload(crf.data(), crf.size(), s.st);
  s.build_rows(omega);
  const std::vector<float> xf = to_f32(xin, n);
  s.x.alloc(static_cast<size_t>(n), s.st);
  s.x.upload(xf.data(), xf.size(), s.st);
  s.y.alloc(static_cast<size_t>(m), s.st);
  s.y.zero(s.st);
  s.r.alloc(static_cast<size_t>(m), s.st);
  s.partial.alloc(static_cast<size_t>(s.rplan.tiles * m), s.st);
  s.set_shard(0, 1);
  s.ista_residual();
  CU(cudaGetLastError());
  std::vector<float> res(static_cast<size_t>(m));
  CU(cudaMemcpyAsync(res.data(), s.r.p, sizeof(float) * m, cudaMemcpyDeviceToHost, s.st));
  CU(cudaStreamSynchronize(s.st));
  for (int64_t i = 0; i < m; ++i) out_m[i] = -static_cast<double>(res[static_cast<size_t>(i)]);
  CL_GUARD_END
}

cl_status cl_partial_transpose_matvec(int device, int64_t n, int64_t m, const double* c, const int64_t* omega,
                                      const double* r_m, double* out_n) {
  CL_GUARD_BEGIN
  NvtxRange nv("cl_partial_transpose_matvec");
  check_mask(omega, m, n);
  Solver s;
  s.kind = CL_KIND_ISTA;
  s.device = device;
  s.n = n;
  s.m = m;
  s.init_device();
  s.plan = make_plan(n, grad_R(n));
  const std::vector<float> cf = to_f32(c, n);
  s.hc.alloc(static_cast<size_t>(n), s.st);
  s.hc.upload(cf.data(), cf.size(), s.st);
  s.build_rows(omega);
  const std::vector<float> rf = to_f32(r_m, m);
  s.r.alloc(static_cast<size_t>(m), s.st);
  s.r.upload(rf.data(), rf.size(), s.st);
  s.partial.alloc(static_cast<size_t>(s.plan.splits * n), s.st);
  s.x.alloc(static_cast<size_t>(n), s.st);
  launch_conv_rows(s.plan, s.hc.p, s.omega32.p, s.r.p, s.rowstart.p, s.partial.p, s.st);
  EpiArgs a;
  a.partial = s.partial.p;
  a.splits = s.plan.splits;
  a.n = n;
  a.lo = 0;
  a.hi = n;
  a.x = s.x.p;
  launch_admm_x(a, s.st);
  CU(cudaGetLastError());
  std::vector<float> res(static_cast<size_t>(n));
  CU(cudaMemcpyAsync(res.data(), s.x.p, sizeof(float) * n, cudaMemcpyDeviceToHost, s.st));
  CU(cudaStreamSynchronize(s.st));
  for (int64_t i = 0; i < n; ++i) out_n[i] = res[static_cast<size_t>(i)];
  CL_GUARD_END
}

cl_status cl_solver_create(int kind, int64_t n, int64_t m, const double* c, const int64_t* omega, const double* y,
                           const cl_config* cfg, int device, cl_solver** out) {
  CL_GUARD_BEGIN
  NvtxRange nv("cl_solver_create");
  *out = nullptr;
  if (kind != CL_KIND_ISTA && kind != CL_KIND_CADMM && kind != CL_KIND_ADMM)
    raise(CL_EPARAM, "cl_solver_create: unknown solver kind");
  if (n < 1) raise(CL_EDIM, "cl_solver_create: n must be >= 1");
  if (m < 0 || m > n) raise(CL_EDIM, "cl_solver_create: need 0 <= m <= n");
  if (n > (int64_t(1) << 30)) raise(CL_ECAPACITY, "cl_solver_create: n above 2^30 is not supported");
  const auto t0 = std::chrono::steady_clock::now();
  trace("create: enter");
  auto s = std::make_unique<Solver>();
  s->kind = kind;
  s->device = device;
  s->n = n;
  s->m = m;
  s->setup_common(c, omega, y, cfg);
  if (kind == CL_KIND_ISTA) s->setup_ista(c, omega, y);
  else if (kind == CL_KIND_CADMM) s->setup_cadmm(c, omega, y);
  else s->setup_admm(c, omega, y);
  s->setup_seconds = seconds_since(t0);
  *out = new cl_solver{std::move(s)};
  CL_GUARD_END
}

void cl_solver_destroy(cl_solver* s) {
  delete s;
  trace("destroy: done");
}

cl_status cl_solver_set_truth(cl_solver* h, const double* truth_n) {
  CL_GUARD_BEGIN
  h->impl->set_truth(truth_n);
  CL_GUARD_END
}

cl_status cl_solver_step(cl_solver* h, int64_t iters) {
  CL_GUARD_BEGIN
  NvtxRange nv("cl_solver_step");
  Solver& s = *h->impl;
  CU(cudaSetDevice(s.device));
  if (iters < 0) raise(CL_EPARAM, "cl_solver_step: iters must be >= 0");
  s.step(iters);
  CL_GUARD_END
}

cl_status cl_solver_step_checked(cl_solver* h, double* metric, int* nonfinite) {
  CL_GUARD_BEGIN
  NvtxRange nv("cl_solver_step_checked");
  Solver& s = *h->impl;
  CU(cudaSetDevice(s.device));
  s.step_checked(metric, nonfinite);
  CL_GUARD_END
}

cl_status cl_solver_run(cl_solver* h, cl_report* rep, double* final_x, int64_t* trace_iter, double* trace_value,
                        double* trace_seconds, int64_t trace_cap) {
  CL_GUARD_BEGIN
  NvtxRange nv("cl_solver_run");
  Solver& s = *h->impl;
  CU(cudaSetDevice(s.device));
  run_loop(s, s.cfg, rep, final_x, trace_iter, trace_value, trace_seconds, trace_cap);
  CL_GUARD_END
}

cl_status cl_solver_get(cl_solver* h, const char* field, double* out) {
  CL_GUARD_BEGIN
  Solver& s = *h->impl;
  CU(cudaSetDevice(s.device));
  int64_t len = 0;
  const std::string f(field ? field : "");
  float* p = s.field_ptr(f, &len);
  s.download(p, len, out);
  if (f == "b") {  // stored reversed on the device: b[k] = b_rev[(-k) mod n]
    std::vector<double> tmp(out, out + len);
    for (int64_t k = 0; k < len; ++k) out[k] = tmp[static_cast<size_t>((len - k) % len)];
  }
  CL_GUARD_END
}

cl_status cl_solver_set(cl_solver* h, const char* field, const double* in) {
  CL_GUARD_BEGIN
  Solver& s = *h->impl;
  CU(cudaSetDevice(s.device));
  int64_t len = 0;
  const std::string f(field ? field : "");
  float* p = s.field_ptr(f, &len);
  if (!in) raise(CL_EPARAM, "cl_solver_set: null input");
  // Operator rows with derived device state cannot be rewritten in place: the FFT engine's
  // spectra come from c (and B's), and cADMM's B row is the Gram inverse of c.
  if (f == "c" && (s.fft || s.kind == CL_KIND_CADMM))
    raise(CL_EPARAM, "cl_solver_set: 'c' is fixed at setup for FFT-engine and cADMM solvers (derived spectra / B)");
  if (f == "b" && s.fft) raise(CL_EPARAM, "cl_solver_set: 'b' is fixed at setup for FFT-engine solvers");
  std::vector<float> tmp = to_f32(in, len);
  if (f == "b") tmp = reversed(tmp);
  if (f == "c") {  // keep the reversed copy coherent
    const std::vector<float> rv = reversed(tmp);
    CU(cudaMemcpyAsync(s.hcr.p, rv.data(), sizeof(float) * len, cudaMemcpyHostToDevice, s.st));
  }
  CU(cudaMemcpyAsync(p, tmp.data(), sizeof(float) * len, cudaMemcpyHostToDevice, s.st));
  CU(cudaStreamSynchronize(s.st));
  CL_GUARD_END
}

cl_status cl_solver_info(cl_solver* h, int64_t* n, int64_t* m, int64_t* t, double* scale, double* threshold) {
  CL_GUARD_BEGIN
  Solver& s = *h->impl;
  if (n) *n = s.n;
  if (m) *m = s.m;
  if (t) *t = s.t;
  if (scale) *scale = s.scale;
  if (threshold) *threshold = s.thr;
  CL_GUARD_END
}

cl_status cl_solver_synchronize(cl_solver* h) {
  CL_GUARD_BEGIN
  Solver& s = *h->impl;
  CU(cudaSetDevice(s.device));
  CU(cudaStreamSynchronize(s.st));
  s.collect_profile();
  CL_GUARD_END
}

cl_status cl_solver_last_step_ms(cl_solver* h, double* ms) {
  CL_GUARD_BEGIN
  Solver& s = *h->impl;
  CU(cudaSetDevice(s.device));
  CU(cudaEventSynchronize(s.step_ev[1]));
  float f = 0.f;
  CU(cudaEventElapsedTime(&f, s.step_ev[0], s.step_ev[1]));
  *ms = f;
  CL_GUARD_END
}

cl_status cl_solver_profile(cl_solver* h, int enable) {
  CL_GUARD_BEGIN
  Solver& s = *h->impl;
  CU(cudaSetDevice(s.device));
  CU(cudaStreamSynchronize(s.st));
  s.drop_graph();  // the next step recaptures with (or without) the profiling event nodes
  if (enable < 0 || enable > 2) raise(CL_EPARAM, "cl_solver_profile: mode is 0 (off), 1 (eager) or 2 (in-graph)");
  s.profile = enable;
  s.ring_count = 0;
  s.n_ev_nodes = 0;
  CL_GUARD_END
}

cl_status cl_solver_phase_ms(cl_solver* h, double* ms, int* count) {
  CL_GUARD_BEGIN
  Solver& s = *h->impl;
  CU(cudaSetDevice(s.device));
  s.collect_profile();
  const int c = std::min(*count, s.nphase);
  for (int i = 0; i < c; ++i) ms[i] = s.phase_ms[i];
  *count = s.nphase;
  CL_GUARD_END
}

cl_status cl_solver_phase_history(cl_solver* h, double* ms, int64_t max_steps, int64_t* steps, int* nphase) {
  CL_GUARD_BEGIN
  Solver& s = *h->impl;
  CU(cudaSetDevice(s.device));
  if (!steps || !nphase) raise(CL_EPARAM, "cl_solver_phase_history: null argument");
  *nphase = s.nphase;
  *steps = ms ? s.phase_history(ms, max_steps) : std::min<int64_t>(s.ring_count, Solver::kRing);
  CL_GUARD_END
}

cl_status cl_solver_shard(cl_solver* h, int rank, int world) {
  CL_GUARD_BEGIN
  h->impl->comm = nullptr;  // caller-driven exchange (cl_solver_run_phase) from here on
  h->impl->set_shard(rank, world);
  CL_GUARD_END
}

cl_status cl_solver_stream(cl_solver* h, void** stream) {
  CL_GUARD_BEGIN
  *stream = h->impl->st;
  CL_GUARD_END
}

cl_status cl_solver_run_phase(cl_solver* h, int phase) {
  CL_GUARD_BEGIN
  NvtxRange nv("cl_solver_run_phase");
  Solver& s = *h->impl;
  CU(cudaSetDevice(s.device));
  if (s.kind == CL_KIND_ADMM) {  // padmm_phases: the primal phase, then the rhs phase
    if (phase == 0) {
      PadmmArgs a;
      a.B = s.Bm.p;
      a.rhs = s.rhs.p;
      a.x = s.x.p;
      a.z = s.z.p;
      a.u = s.u.p;
      a.n = s.n;
      a.thr = static_cast<float>(s.thr);
      launch_padmm_primal(a, s.st);
    } else if (phase == 1) {
      launch_padmm_rhs(s.aty.p, s.z.p, s.u.p, static_cast<float>(s.cfg.rho), s.rhs.p, s.n, s.st);
      ++s.t;
    } else {
      raise(CL_EPARAM, "cl_solver_run_phase: dense ADMM phases are 0 (primal) and 1 (rhs)");
    }
  } else if (s.kind == CL_KIND_ISTA) {
    if (phase == 0) s.ista_residual();
    else if (phase == 1) { s.ista_gradient(0); ++s.t; }
    else raise(CL_EPARAM, "cl_solver_run_phase: ISTA phases are 0 (residual) and 1 (gradient)");
  } else {
    if (phase == 0) s.admm_beta_phase();
    else if (phase == 1) s.admm_x_phase();
    else if (phase == 2) { s.admm_dual_phase(0); ++s.t; }
    else raise(CL_EPARAM, "cl_solver_run_phase: cADMM phases are 0 (beta), 1 (x), 2 (duals)");
  }
  CU(cudaGetLastError());
  CL_GUARD_END
}

cl_status cl_solver_phase_output(cl_solver* h, int phase, void** dev_ptr, int64_t* begin, int64_t* end,
                                 int64_t* total) {
  CL_GUARD_BEGIN
  Solver& s = *h->impl;
  if (s.kind == CL_KIND_ADMM) raise(CL_EPARAM, "cl_solver_phase_output: the dense ADMM runs unsharded");
  if (s.kind == CL_KIND_ISTA) {
    if (phase == 0) { *dev_ptr = s.r.p; *begin = s.row_lo; *end = s.row_hi; *total = s.m; }
    else { *dev_ptr = s.x.p; *begin = s.out_lo; *end = s.out_hi; *total = s.n; }
  } else {
    *dev_ptr = phase == 0 ? s.beta.p : phase == 1 ? s.x.p : s.v.p;
    *begin = s.out_lo;
    *end = s.out_hi;
    *total = s.n;
  }
  CL_GUARD_END
}

cl_status cl_shard_ranges(int kind, int64_t n, int64_t m, const int64_t* omega, int rank, int world, int64_t* out_lo,
                          int64_t* out_hi, int64_t* row_lo, int64_t* row_hi) {
  CL_GUARD_BEGIN
  if (kind != CL_KIND_ISTA && kind != CL_KIND_CADMM) raise(CL_EPARAM, "cl_shard_ranges: unknown solver kind");
  if (n < 1 || m < 0 || m > n) raise(CL_EDIM, "cl_shard_ranges: need n >= 1 and 0 <= m <= n");
  check_mask(omega, m, n);
  ConvPlan plan = (kind == CL_KIND_ISTA ? (ista_uses_tc(n) ? make_dense_plan(n) : make_plan(n, grad_R(n))) : make_dense_plan(n));
  ConvPlan rplan = make_plan(n, res_R(n));
  shard_ranges(kind, n, omega, m, rank, world, &plan, &rplan, out_lo, out_hi, row_lo, row_hi);
  CL_GUARD_END
}

struct cl_comm {
  Comm* c = nullptr;
};
struct cl_group {
  std::unique_ptr<Group> g;
};

cl_status cl_comm_unique_id(unsigned char* id) {
  CL_GUARD_BEGIN
  if (!id) raise(CL_EPARAM, "cl_comm_unique_id: null buffer");
  comm_unique_id(id);
  CL_GUARD_END
}
cl_status cl_comm_init_rank(const unsigned char* id, int world, int rank, int device, cl_comm** out) {
  CL_GUARD_BEGIN
  if (!id || !out) raise(CL_EPARAM, "cl_comm_init_rank: null argument");
  *out = nullptr;
  Comm* c = comm_init_rank(id, world, rank, device);
  *out = new cl_comm{c};
  CL_GUARD_END
}
void cl_comm_destroy(cl_comm* c) {
  if (!c) return;
  comm_destroy(c->c);
  delete c;
}
cl_status cl_solver_peer_export(cl_solver* h, int rank, int world, unsigned char* blob) {
  CL_GUARD_BEGIN
  if (!h || !blob) raise(CL_EPARAM, "cl_solver_peer_export: null argument");
  CU(cudaSetDevice(h->impl->device));
  h->impl->ipc_export(rank, world, blob);
  CL_GUARD_END
}
cl_status cl_solver_peer_attach(cl_solver* h, const unsigned char* blobs) {
  CL_GUARD_BEGIN
  if (!h || !blobs) raise(CL_EPARAM, "cl_solver_peer_attach: null argument");
  CU(cudaSetDevice(h->impl->device));
  h->impl->ipc_attach(blobs);
  CL_GUARD_END
}

cl_status cl_solver_attach_comm(cl_solver* h, cl_comm* c) {
  CL_GUARD_BEGIN
  if (!c || !c->c) raise(CL_EPARAM, "cl_solver_attach_comm: null communicator");
  Solver& s = *h->impl;
  CU(cudaSetDevice(s.device));
  s.attach_comm(c->c);
  CL_GUARD_END
}

cl_status cl_group_create(int kind, int64_t n, int64_t m, const double* c, const int64_t* omega, const double* y,
                          const cl_config* cfg, const int* devices, int ndev, int transport, cl_group** out) {
  CL_GUARD_BEGIN
  NvtxRange nv("cl_group_create");
  if (!out) raise(CL_EPARAM, "cl_group_create: null output");
  *out = nullptr;
  if (ndev < 1 || !devices) raise(CL_EPARAM, "cl_group_create: need at least one device");
  if (kind != CL_KIND_ISTA && kind != CL_KIND_CADMM) raise(CL_EPARAM, "cl_group_create: ISTA or cADMM only");
  if (transport != CL_TRANSPORT_NCCL && transport != CL_TRANSPORT_COPY && transport != CL_TRANSPORT_PEER)
    raise(CL_EPARAM, "cl_group_create: unknown transport");
  if (transport == CL_TRANSPORT_PEER && ndev > EpiArgs::kMaxPeers + 1)
    raise(CL_EPARAM, "cl_group_create: the peer-store transport takes at most 8 ranks");
  if (n < 1) raise(CL_EDIM, "cl_solver_create: n must be >= 1");
  if (m < 0 || m > n) raise(CL_EDIM, "cl_solver_create: need 0 <= m <= n");
  const auto t0 = std::chrono::steady_clock::now();
  auto g = std::make_unique<Group>();
  g->kind = kind;
  g->n = n;
  g->m = m;
  g->transport = static_cast<Group::Transport>(transport);
  if (g->transport == Group::kNccl) g->comms = comm_init_all(devices, ndev);
  for (int r = 0; r < ndev; ++r) {
    auto s = std::make_unique<Solver>();
    s->kind = kind;
    s->device = devices[r];
    s->n = n;
    s->m = m;
    s->setup_common(c, omega, y, cfg);
    if (kind == CL_KIND_ISTA) s->setup_ista(c, omega, y);
    else s->setup_cadmm(c, omega, y);
    if (s->fft && ndev > 1) raise(CL_EPARAM, "cl_group_create: the FFT engine runs unsharded (replicas only)");
    if (g->transport == Group::kNccl) {
      s->attach_comm(g->comms[static_cast<size_t>(r)]);
    } else {
      s->set_shard(r, ndev);
      s->world = ndev;
      s->all_ranges();
    }
    g->ranks.push_back(std::move(s));
  }
  if (g->transport == Group::kCopy || g->transport == Group::kPeer) {
    g->done.resize(static_cast<size_t>(ndev));
    for (int r = 0; r < ndev; ++r) {
      CU(cudaSetDevice(devices[r]));
      CU(cudaEventCreateWithFlags(&g->done[static_cast<size_t>(r)], cudaEventDisableTiming));
    }
  }
  if (g->transport == Group::kPeer) {
    // every pair of distinct devices maps the other's memory (NVLink), then each rank gets, per phase, the
    // other ranks' copies of the vector that phase produces
    for (int a = 0; a < ndev; ++a)
      for (int b = 0; b < ndev; ++b) {
        if (devices[a] == devices[b]) continue;
        int ok = 0;
        CU(cudaDeviceCanAccessPeer(&ok, devices[a], devices[b]));
        if (!ok) raise(CL_EPARAM, "cl_group_create: the peer-store transport needs peer access between the devices");
        CU(cudaSetDevice(devices[a]));
        const cudaError_t e = cudaDeviceEnablePeerAccess(devices[b], 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CU(e);
        cudaGetLastError();  // clear a benign "already enabled"
      }
    for (int r = 0; r < ndev; ++r) {
      Solver& s = *g->ranks[static_cast<size_t>(r)];
      s.npeer = ndev - 1;
      for (int ph = 0; ph < s.phase_count(); ++ph) {
        int p = 0;
        for (int q = 0; q < ndev; ++q)
          if (q != r) s.peer_out[ph][p++] = g->ranks[static_cast<size_t>(q)]->phase_buffer(ph);
      }
    }
  }
  g->setup_seconds = seconds_since(t0);
  *out = new cl_group{std::move(g)};
  CL_GUARD_END
}
void cl_group_destroy(cl_group* g) { delete g; }
cl_status cl_group_set_truth(cl_group* h, const double* truth_n) {
  CL_GUARD_BEGIN
  Group& g = *h->g;
  for (auto& s : g.ranks) s->set_truth(truth_n);
  g.has_truth = truth_n != nullptr;
  CL_GUARD_END
}
cl_status cl_group_step(cl_group* h, int64_t iters) {
  CL_GUARD_BEGIN
  NvtxRange nv("cl_group_step");
  if (iters < 0) raise(CL_EPARAM, "cl_group_step: iters must be >= 0");
  h->g->step(iters);
  CL_GUARD_END
}
cl_status cl_group_run(cl_group* h, cl_report* rep, double* final_x, int64_t* trace_iter, double* trace_value,
                       double* trace_seconds, int64_t trace_cap) {
  CL_GUARD_BEGIN
  NvtxRange nv("cl_group_run");
  Group& g = *h->g;
  run_loop(g, g.ranks.front()->cfg, rep, final_x, trace_iter, trace_value, trace_seconds, trace_cap);
  CL_GUARD_END
}
cl_status cl_group_get(cl_group* h, const char* field, double* out) {
  CL_GUARD_BEGIN
  if (!field || !out) raise(CL_EPARAM, "cl_group_get: null argument");
  h->g->get(field, out);
  CL_GUARD_END
}
cl_status cl_group_synchronize(cl_group* h) {
  CL_GUARD_BEGIN
  for (auto& s : h->g->ranks) {
    CU(cudaSetDevice(s->device));
    CU(cudaStreamSynchronize(s->st));
  }
  CL_GUARD_END
}
cl_status cl_group_info(cl_group* h, int* world, int64_t* t, int* transport) {
  CL_GUARD_BEGIN
  if (world) *world = h->g->world();
  if (t) *t = h->g->ranks.front()->t;
  if (transport) *transport = h->g->transport;
  CL_GUARD_END
}

cl_status cl_ffma_peak(int device, double* tflops) {
  CL_GUARD_BEGIN
  const double v = ffma_peak_tflops(device);
  if (v <= 0) raise(CL_ECUDA, "cl_ffma_peak: microbenchmark failed");
  *tflops = v;
  CL_GUARD_END
}

}  // extern "C"
