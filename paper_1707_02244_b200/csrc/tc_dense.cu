// Dense circulant product on the tcgen05 tensor cores (see tc_dense.cuh).
//
// Blocking.  i = 256 I + p, j = 256 (I - D) + 255 - k  (p, k in [0, 256)):
//   out[256 I + p] = sum_D sum_k  h[256 D - 255 + p + k] * u[256 (I - D) + 255 - k]
//                  = sum_D  (A_D B_D^T)[I, p]
//   A_D[I, k] = u[256 (I - D) + 255 - k]      M = 128 rows I of a tile, K-major
//   B_D[p, k] = h[256 D - 255 + p + k]        N = 256 columns p (a Hankel tile), K-major
// As D runs over all n / 256 offsets and k over [0, 256), j covers every index once.
//
// Shared-memory views (SWIZZLE_NONE K-major: rows 16 B apart, SBO = 128 B, the two
// 16-byte K chunks of one K = 8 step LBO apart):
//  * A: a slab per 32-wide K group holds the rows I - D for a block of 128 offsets D,
//    chunk-major (chunk c at c * LBO_A).  Moving D by one moves the descriptor start
//    by one 16-byte row, so one slab serves 128 offsets.
//  * B: row r of a tile holds h[t0 + r .. t0 + r + 3]; with LBO = 64 B (four rows) the
//    descriptor reads element (p, k) at row p + k - (k mod 4), lane k mod 4 = h[t0 + p + k]:
//    a Hankel matrix from 4x-redundant rows (overlapping core matrices).
// Precision: 3xTF32.  x = hi + lo with hi = x with the low 13 mantissa bits cleared
// (exact in TF32) and lo = x - hi (exact in fp32); A.B ~ Ahi.Bhi + Ahi.Blo + Alo.Bhi in
// the fp32 TMEM accumulator.  The dropped Alo.Blo term is ~2^-22 relative.
#include "tc_dense.cuh"

#include <cstdlib>

namespace clb {
namespace {

constexpr int kB = 256;        // block length = MMA N
constexpr int kMT = 128;       // rows I per tile = MMA M
constexpr int kKG = 32;        // K per slab group
constexpr int kNG = kB / kKG;  // groups per offset
constexpr int kDB = 128;       // offsets per slab block
constexpr int kRA = kDB + kMT; // slab rows (max)
constexpr int kSlabBytes = kRA * 16 * (kKG / 4);
constexpr int kRB = 288;       // Hankel rows: p + k_local - (k_local mod 4) <= 255 + 28, rounded up
constexpr int kTileBytes = kRB * 16;
#ifndef TC_BST
#define TC_BST 8
#endif
constexpr int kAStages = 2, kBStages = TC_BST;
constexpr int kProducers = 256;
constexpr int kTcThreads = kProducers + 32;  // warps 0-7 produce and drain, warp 8 issues MMAs
constexpr int kOffB = kAStages * 2 * kSlabBytes;
constexpr int kOffBar = kOffB + kBStages * 2 * kTileBytes;
constexpr int kTcSmem = kOffBar + (8 + 2 * kBStages) * 8 + 16;
#ifndef TC_SPD
#define TC_SPD 4
#endif
constexpr int kSPD = TC_SPD;  // steps accumulated in TMEM between drains (divides 8)
constexpr int kTmemCols = 512;  // two 128 x 256 fp32 accumulators

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "TC_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TC_WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFFu) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);  // version 1, SWIZZLE_NONE
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }
__device__ __forceinline__ void st_split(float* hi, float* lo, float4 v) {
  const float4 a = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
  *reinterpret_cast<float4*>(hi) = a;
  *reinterpret_cast<float4*>(lo) = make_float4(v.x - a.x, v.y - a.y, v.z - a.z, v.w - a.w);
}

// unit = (tile, split); split s covers offsets [s Dn, (s + 1) Dn), Dn = (n / 256) / splits.
// A step is one (offset D, K group g) pair: 12 MMAs (4 K-steps x 3 TF32 products).  kSPD
// steps accumulate into one of two TMEM accumulators, started from zero.  The tensor core's
// fp32 accumulation truncates, so its error grows with the accumulator's magnitude; draining
// every kSPD steps into fp32 registers (round-to-nearest FADD) keeps the sums at FFMA accuracy
// (tools/microbench/tc_probe.cu at n = 2^20, max error / sum|terms|: 8.4e-7 never drained;
// 3.3e-9 / 3.4e-9 / 6.0e-9 / 8.0e-9 drained every 1 / 2 / 4 / 8 steps, at 7.8 / 7.6 / 7.05 /
// 7.1 ms).
// Steps run in the order (D block, g, D): one A slab per (block, g), one Hankel tile per step.
__global__ void __launch_bounds__(kTcThreads, 1)
k_tc_dense(const float* __restrict__ h, const float* __restrict__ u, int64_t n, int splits, int64_t tile_lo,
           float* __restrict__ partial) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + kOffBar);
  uint64_t* a_full = bar;        // [2]
  uint64_t* a_empty = bar + 2;   // [2]
  uint64_t* b_full = bar + 4;                 // [kBStages]
  uint64_t* b_empty = b_full + kBStages;      // [kBStages]
  uint64_t* t_full = b_empty + kBStages;      // [2]
  uint64_t* t_empty = t_full + 2;             // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_empty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  const int64_t nb = n / kB, nbm = nb - 1, nm = n - 1;
  const int64_t tile = tile_lo + blockIdx.x / splits;
  const int s = static_cast<int>(blockIdx.x % splits);
  const int64_t I0 = tile * kMT;
  const int64_t Dn = nb / splits, Dlo = s * Dn;
  const int64_t DBn = Dn < kDB ? Dn : kDB;  // powers of two (n is)
  const int lgDB = __ffsll(DBn) - 1;
  const int64_t steps = kNG * Dn;
  const int rows = static_cast<int>(DBn) + kMT;
  const uint32_t lboA = static_cast<uint32_t>(rows) * 16u;

  if (tid == 0) {
    for (int i = 0; i < kAStages; ++i) {
      mbar_init(&a_full[i], kProducers);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < kBStages; ++i) {
      mbar_init(&b_full[i], kProducers);
      mbar_init(&b_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&t_full[i], 1);
      mbar_init(&t_empty[i], kProducers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kProducers / 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp < kProducers / 32) {
    // ---- producers (A slabs, Hankel tiles) and accumulator drain ----
    int a_use = 0;
    auto produce = [&](int64_t j) {
      const int64_t blk = j >> (lgDB + 3), rem = j & (kNG * DBn - 1);
      const int g = static_cast<int>(rem >> lgDB);
      const int64_t dd = rem & (DBn - 1), d0 = Dlo + blk * DBn, D = d0 + dd;
      if (dd == 0) {
        const int st = a_use & 1;
        mbar_wait(&a_empty[st], ((a_use >> 1) & 1) ^ 1);
        float* hi = reinterpret_cast<float*>(sm + (st * 2) * kSlabBytes);
        float* lo = reinterpret_cast<float*>(sm + (st * 2 + 1) * kSlabBytes);
        const int64_t ibase = I0 - d0 - DBn + 1;  // I - D of slab row 0
        for (int idx = tid; idx < rows * (kKG / 4); idx += kProducers) {
          const int rho = idx % rows, c = idx / rows;
          const int64_t Ip = (ibase + rho) & nbm;
          const float4 v = __ldg(reinterpret_cast<const float4*>(u + Ip * kB + (kB - 4) - kKG * g - 4 * c));
          const int off = (c * rows + rho) * 4;
          st_split(hi + off, lo + off, make_float4(v.w, v.z, v.y, v.x));
        }
        fence_async_smem();
        mbar_arrive(&a_full[st]);
        ++a_use;
      }
      const int bs = static_cast<int>(j & (kBStages - 1));
      mbar_wait(&b_empty[bs], ((j / kBStages) & 1) ^ 1);
      float* thi = reinterpret_cast<float*>(sm + kOffB + (bs * 2) * kTileBytes);
      float* tlo = reinterpret_cast<float*>(sm + kOffB + (bs * 2 + 1) * kTileBytes);
      const int64_t t0 = D * kB - (kB - 1) + kKG * g;
      for (int r = tid; r < kRB; r += kProducers) {
        const int64_t t = t0 + r;
        const float4 v = make_float4(__ldg(h + (t & nm)), __ldg(h + ((t + 1) & nm)), __ldg(h + ((t + 2) & nm)),
                                     __ldg(h + ((t + 3) & nm)));
        st_split(thi + r * 4, tlo + r * 4, v);
      }
      fence_async_smem();
      mbar_arrive(&b_full[bs]);
    };
    float acc[kB / 2];
#pragma unroll
    for (int q = 0; q < kB / 2; ++q) acc[q] = 0.f;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + (warp >> 2) * (kB / 2);
    // Tiles run `ahead` steps ahead of the drain.  Tile j + ahead reuses the B stage of step
    // j + ahead - kBStages (issued before step j), and a slab it starts reuses the A stage of
    // step j + ahead - DBn - 1 at the latest: ahead <= DBn keeps both waits free of any drain
    // this loop has not done yet (no deadlock when slabs change every step, e.g. n = 2^16).
    const int64_t ahead = DBn < kBStages - 1 ? DBn : kBStages - 1;
    for (int64_t j = 0; j < ahead && j < steps; ++j) produce(j);
    for (int64_t j = 0; j < steps; ++j) {
      if (j % kSPD == kSPD - 1) {
        const int64_t cyc = j / kSPD;
        const int buf = static_cast<int>(cyc & 1);
        mbar_wait(&t_full[buf], (cyc >> 1) & 1);
        tc_after_sync();
#ifndef TC_NODRAIN
#pragma unroll
        for (int c0 = 0; c0 < kB / 2; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(lane_base + buf * kB + c0, v);
#pragma unroll
          for (int e = 0; e < 32; ++e) acc[c0 + e] += __uint_as_float(v[e]);
        }
#endif
        tc_before_sync();
        mbar_arrive(&t_empty[buf]);
      }
      if (j + ahead < steps) produce(j + ahead);
    }
    // ---- partial[s][256 I + p]: this thread's row I, columns [128 (warp / 4), +128) ----
    float* out = partial + static_cast<int64_t>(s) * n + (I0 + (warp & 3) * 32 + lane) * kB + (warp >> 2) * (kB / 2);
#pragma unroll
    for (int q = 0; q < kB / 2; q += 4) *reinterpret_cast<float4*>(out + q) = make_float4(acc[q], acc[q + 1], acc[q + 2], acc[q + 3]);
  } else if (lane == 0) {
    // ---- MMA issue (one thread) ----
    constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(kB >> 3) << 17) |
                               (static_cast<uint32_t>(kMT >> 4) << 24);
    const uint32_t abase = smem_u32(sm), bbase = smem_u32(sm + kOffB);
    int a_use = 0;
    uint32_t ahi = 0, alo = 0;
    for (int64_t j = 0; j < steps; ++j) {
      const int64_t dd = j & (DBn - 1);
      const int st = a_use & 1;
      if (dd == 0) {
        mbar_wait(&a_full[st], (a_use >> 1) & 1);
        ahi = abase + (st * 2) * kSlabBytes;
        alo = ahi + kSlabBytes;
      }
      const int bs = static_cast<int>(j & (kBStages - 1));
      mbar_wait(&b_full[bs], (j / kBStages) & 1);
      const int64_t cyc = j / kSPD;
      const int buf = static_cast<int>(cyc & 1);
      const bool first = j % kSPD == 0;
      if (first) mbar_wait(&t_empty[buf], ((cyc >> 1) & 1) ^ 1);
      tc_after_sync();
      const uint32_t row0 = static_cast<uint32_t>(DBn - 1 - dd) * 16u;
      const uint32_t bhi = bbase + (bs * 2) * kTileBytes, blo = bhi + kTileBytes;
      const uint32_t tacc = tmem + buf * kB;
#pragma unroll
      for (int kk = 0; kk < kKG / 8; ++kk) {
        const uint64_t dah = sdesc(ahi + row0 + 2u * kk * lboA, lboA, 128);
        const uint64_t dal = sdesc(alo + row0 + 2u * kk * lboA, lboA, 128);
        const uint64_t dbh = sdesc(bhi + 128u * kk, 64, 128);
        const uint64_t dbl = sdesc(blo + 128u * kk, 64, 128);
        mma_tf32(tacc, dah, dbh, idesc, (first && kk == 0) ? 0u : 1u);
        mma_tf32(tacc, dah, dbl, idesc, 1);
        mma_tf32(tacc, dal, dbh, idesc, 1);
      }
      tc_commit(&b_empty[bs]);
      if (j % kSPD == kSPD - 1) tc_commit(&t_full[buf]);
      if (dd == DBn - 1) {
        tc_commit(&a_empty[st]);
        ++a_use;
      }
    }
  }
  tc_before_sync();
  __syncthreads();
  if (warp == kProducers / 32) {
    tc_after_sync();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols) : "memory");
  }
}

}  // namespace

bool tc_dense_supported(int64_t n) {
  return n >= int64_t(kB) * kMT && (n & (n - 1)) == 0 && n <= (int64_t(1) << 30);
}

ConvPlan make_tc_plan(int64_t n) {
  ConvPlan p;
  p.n = n;
  p.tile = int64_t(kB) * kMT;
  p.tiles = n / p.tile;
  p.chunks = 0;
  const int64_t nb = n / kB;
  // about seven waves of one-CTA-per-SM units; splits a power of two dividing n / 256
  int64_t s = 1;
  while (p.tiles * s * 2 <= 148 * 7 && s * 2 <= nb) s *= 2;
  if (const char* v = getenv("CLB_TC_SPLITS")) s = atoll(v);
  p.splits = static_cast<int>(s);
  p.tile_lo = 0;
  p.tile_hi = p.tiles;
  p.split_lo = 0;
  p.split_hi = p.splits;
  return p;
}

void tc_dense_init() {
  static bool done = false;
  if (done) return;
  done = true;
  cudaFuncSetAttribute(reinterpret_cast<const void*>(k_tc_dense), cudaFuncAttributeMaxDynamicSharedMemorySize,
                       kTcSmem);
}

void launch_tc_dense(const ConvPlan& p, const float* h, const float* u, float* partial, cudaStream_t st) {
  const int64_t units = (p.tile_hi - p.tile_lo) * p.splits;
  if (units <= 0) return;
  tc_dense_init();
  k_tc_dense<<<static_cast<unsigned>(units), kTcThreads, kTcSmem, st>>>(h, u, p.n, p.splits, p.tile_lo, partial);
}

}  // namespace clb
