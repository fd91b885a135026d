// Dense circulant product on the tcgen05 tensor cores (see tc_dense.cuh; DESIGN.md §3,
// "Tensor-core products").
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
// Precision, two formats with the same three products A.B ~ Ahi.Bhi + Ahi.Blo + Alo.Bhi in
// the fp32 TMEM accumulator (the dropped Alo.Blo term is ~2^-22 relative):
//  * 3xTF32 (kind::tf32): hi = x with the low 13 mantissa bits cleared (exact in TF32),
//    lo = x - hi (exact in fp32).  Chunks hold 4 values; Hankel LBO = 64 B.
//  * fp16 2-term split (kind::f16, n >= 2^18): x scaled by a power of two putting max|x| in
//    [2^13, 2^14), hi = rn16(x), lo = rn16(x - hi).  Chunks hold 8 values, Hankel rows
//    h[t0 + r .. t0 + r + 7] with LBO = 128 B; K = 16 per MMA (twice the rate, half the bytes).
#include "tc_dense.cuh"

#include <cuda_fp16.h>

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
constexpr int kRB2 = 160;      // a CTA pair's half tile (p < 128): <= 127 + 28, rounded up
constexpr int kTileBytes = kRB * 16;
#ifndef TC_BST
#define TC_BST 8
#endif
constexpr int kAStages = 2, kBStages = TC_BST;
constexpr int kDrainers = 256;                 // warps 0-7: drain TMEM into fp32 registers
constexpr int kProducers = 96;                 // warps 8-10: A slabs and Hankel tiles
constexpr int kMmaWarp = (kDrainers + kProducers) / 32;  // warp 11: TMEM allocation, MMA issue
constexpr int kTcThreads = kDrainers + kProducers + 32;
constexpr int kOffB = kAStages * 2 * kSlabBytes;
constexpr int kOffBar = kOffB + kBStages * 2 * kTileBytes;
constexpr int kStg = kRB + 8;  // fp16 staging row (packed hi | lo) per tile, double-buffered
// The smem layout is the same for both CTA-group sizes (a pair uses the first kRB2 rows of each B stage).
constexpr int kOffStg = kOffBar + (8 + 2 * kBStages) * 8 + 16;
constexpr int kTcSmem = kOffStg + 2 * kStg * 4;
#ifndef TC_SPD
#define TC_SPD 4
#endif
constexpr int kSPD = TC_SPD;  // TF32: steps accumulated in TMEM between drains (divides 8)
constexpr int kTmemCols = 512;  // two 128 x 256 fp32 accumulators
#ifndef TC_TWO_MMA
#define TC_TWO_MMA 0  // diagnostic builds: drop the Alo.Bhi product (u rounded to one fp16 term) to measure its error
#endif
#ifndef TC_MMA_ONLY
#define TC_MMA_ONLY 0  // diagnostic builds (tools/microbench): no tile production after the first fill, no drain
#endif

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
__device__ __forceinline__ void mma_f16(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// ---- CTA pairs (cta_group::2): the leader (rank 0) issues M = 256 MMAs whose A rows 128..255 and
// B columns 128..255 come from the peer's shared memory at the same offsets; each CTA's TMEM holds
// its own 128 rows.  Producer / drain hand-overs arrive on the leader's barriers across the cluster.
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive (release, cluster scope) on the barrier at the same offset in CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* b, uint32_t rank) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(b)),
      "r"(rank)
      : "memory");
}
// commit the leader's MMAs to the barrier at this offset in both CTAs of the pair
__device__ __forceinline__ void tc_commit_pair(uint64_t* b) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\t"
      "mov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
          smem_u32(b))
      : "memory");
}
__device__ __forceinline__ void mma_pair(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc,
                                         bool f16) {
  if (f16)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
// 8 scaled values -> 16-byte rows of fp16 hi = rn(x) and lo = rn(x - hi) (x - hi is exact in fp32)
__device__ __forceinline__ void st_split8(unsigned char* hi, unsigned char* lo, const float (&v)[8], float sc) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float a = v[2 * q] * sc, b = v[2 * q + 1] * sc;
    const __half ha = __float2half_rn(a), hb = __float2half_rn(b);
    const __half la = __float2half_rn(a - __half2float(ha)), lb = __float2half_rn(b - __half2float(hb));
    h[q] = static_cast<uint32_t>(__half_as_ushort(ha)) | (static_cast<uint32_t>(__half_as_ushort(hb)) << 16);
    l[q] = static_cast<uint32_t>(__half_as_ushort(la)) | (static_cast<uint32_t>(__half_as_ushort(lb)) << 16);
  }
  *reinterpret_cast<uint4*>(hi) = make_uint4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<uint4*>(lo) = make_uint4(l[0], l[1], l[2], l[3]);
}
// power-of-two scale putting max|x| in [2^13, 2^14) (fp16 max 65504); 1 for 0 / non-finite
__device__ __forceinline__ float f16_scale(float mx) {
  if (!(mx > 0.f) || !isfinite(mx)) return 1.f;
  int e;
  frexpf(mx, &e);  // mx < 2^e
  return ldexpf(1.f, min(14 - e, 127));  // subnormal max: 2^127 (keeps the scale finite)
}

__global__ void k_absmax2(const float* __restrict__ h, const float* __restrict__ u, int64_t n, float* __restrict__ out) {
  float a = 0.f, b = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    a = fmaxf(a, fabsf(h[i]));
    b = fmaxf(b, fabsf(u[i]));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
    b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, o));
  }
  __shared__ float sa[32], sb[32];
  if ((threadIdx.x & 31) == 0) {
    sa[threadIdx.x >> 5] = a;
    sb[threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      a = fmaxf(a, sa[w]);
      b = fmaxf(b, sb[w]);
    }
    out[blockIdx.x] = a;
    out[gridDim.x + blockIdx.x] = b;
  }
}
constexpr int kMaxBlocks = 148 * 4;

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }
__device__ __forceinline__ void st_split(float* hi, float* lo, float4 v) {
  const float4 a = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
  *reinterpret_cast<float4*>(hi) = a;
  *reinterpret_cast<float4*>(lo) = make_float4(v.x - a.x, v.y - a.y, v.z - a.z, v.w - a.w);
}

// Steps of one unit in consumption order: blocks of up to kDB offsets, and per block the 8 K groups, and
// per group the block's offsets.  A split covers offsets [s nb / S, (s + 1) nb / S) (nb = n / 256), so S
// need not divide nb (S = 37 k lets the units of 1, 2, 4 or 8 ranks fill whole waves of 148 SMs).
struct StepIter {
  int64_t Dlo = 0, L = 0;   // the split's first offset and length
  int64_t blk = 0, dd = 0;  // block index, offset within the block
  int g = 0;                // K group
  int len = 0;              // offsets in the current block
  __device__ __forceinline__ void init(int64_t dlo, int64_t l) {
    Dlo = dlo;
    L = l;
    blk = dd = 0;
    g = 0;
    len = static_cast<int>(l < kDB ? l : kDB);
  }
  __device__ __forceinline__ void next() {
    if (++dd < len) return;
    dd = 0;
    if (++g < kNG) return;
    g = 0;
    ++blk;
    const int64_t rest = L - blk * kDB;
    len = static_cast<int>(rest < kDB ? rest : kDB);
  }
  __device__ __forceinline__ int64_t d0() const { return Dlo + blk * kDB; }
  __device__ __forceinline__ int64_t D() const { return d0() + dd; }
  __device__ __forceinline__ int64_t t0() const { return D() * kB - (kB - 1) + kKG * g; }  // Hankel tile start
};

// unit = (tile, split); split s covers offsets [s nb / S, (s + 1) nb / S), nb = n / 256.
// A step is one (offset D, K group g) pair: 12 MMAs (4 K-steps x 3 TF32 products).  kSPD
// steps accumulate into one of two TMEM accumulators, started from zero.  The tensor core's
// fp32 accumulation truncates, so its error grows with the accumulator's magnitude; draining
// every kSPD steps into fp32 registers (round-to-nearest FADD) keeps the sums at FFMA accuracy
// (tools/microbench/tc_probe.cu at n = 2^20, max error / sum|terms|: 8.4e-7 never drained;
// 3.3e-9 / 3.4e-9 / 6.0e-9 / 8.0e-9 drained every 1 / 2 / 4 / 8 steps, at 7.8 / 7.6 / 7.05 /
// 7.1 ms).
// Steps run in the order (D block, g, D): one A slab per (block, g), one Hankel tile per step.
// Roles: warps 0-7 drain, warps 8-9 produce, one thread of warp 10 issues the MMAs, so tile
// production never waits behind a drain.  F16: fp16 operands with a 2-term split of
// power-of-two-scaled values (hi.hi + hi.lo + lo.hi, kind::f16: twice the MMA rate and half the
// operand bytes of TF32); `maxes` holds k_absmax2's per-block maxima of |h| and |u|.
// CG = 2: CTA pairs (cluster of 2, cta_group::2).  A pair covers two consecutive tiles (rank r: tile
// 2 P + r) of one split; each CTA stages its own A slab rows and the half of the Hankel tile holding its
// 128 columns p (rows t0 + 128 r + ...), so per SM the MMA reads 4 KB of A and 4 KB of B per 128 x 256 x 16
// instead of 4 + 8 KB, and the producers build half the Hankel rows.
template <bool F16, int CG>
__global__ void __launch_bounds__(kTcThreads, 1)
k_tc_dense(const float* __restrict__ h, const float* __restrict__ u, int64_t n, int splits, int64_t tile_lo,
           float* __restrict__ partial, const float* __restrict__ maxes) {
  constexpr bool kPair = CG == 2;
  constexpr int kRows_B = kPair ? kRB2 : kRB;  // Hankel rows this CTA builds
  constexpr int kStgN = kRows_B + 8;           // fp16 staging entries per tile
  constexpr int kEl = F16 ? 8 : 4;       // elements per 16-byte chunk
  constexpr int kCh = kKG / kEl;         // chunks per K group
  constexpr int kKS = F16 ? 16 : 8;      // K per MMA
  constexpr uint32_t kLboB = 16u * kEl;  // Hankel: the next chunk starts kEl rows on
  // steps per drain: the same 48 MMAs per accumulator for both formats (an fp16 step has 6 MMAs)
  constexpr int kSpd = F16 ? 2 * kSPD : kSPD;
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ float scl[2];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + kOffBar);
  uint64_t* a_full = bar;                     // [2]
  uint64_t* a_empty = bar + 2;                // [2]
  uint64_t* b_full = bar + 4;                 // [kBStages]
  uint64_t* b_empty = b_full + kBStages;      // [kBStages]
  uint64_t* t_full = b_empty + kBStages;      // [2]
  uint64_t* t_empty = t_full + 2;             // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_empty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  const int64_t nb = n / kB, nbm = nb - 1, nm = n - 1;
  const uint32_t rank = kPair ? cluster_rank() : 0u;
  const int64_t unit = kPair ? blockIdx.x >> 1 : blockIdx.x;
  const int64_t tile = tile_lo + (kPair ? 2 * (unit / splits) + rank : unit / splits);
  const int s = static_cast<int>(unit % splits);
  const int64_t I0 = tile * kMT;
  const int64_t Dlo = s * nb / splits, Dn = (s + 1) * nb / splits - Dlo;
  const int64_t steps = kNG * Dn;

  if (tid == 0) {
    // pairs: one arrival per producer / drain warp of either CTA on the leader's barriers
    constexpr int kFullCount = kPair ? 2 * (kProducers / 32) : kProducers;
    constexpr int kEmptyTCount = kPair ? 2 * (kDrainers / 32) : kDrainers;
    for (int i = 0; i < kAStages; ++i) {
      mbar_init(&a_full[i], kFullCount);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < kBStages; ++i) {
      mbar_init(&b_full[i], kFullCount);
      mbar_init(&b_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&t_full[i], 1);
      mbar_init(&t_empty[i], kEmptyTCount);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {
    if constexpr (kPair) {  // issued by the same warp of both CTAs
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "n"(kTmemCols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "n"(kTmemCols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  if (F16 && warp == 1) {
    float a = 0.f, b = 0.f;
    for (int i = lane; i < kMaxBlocks; i += 32) {
      a = fmaxf(a, maxes[i]);
      b = fmaxf(b, maxes[kMaxBlocks + i]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
      b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    if (lane == 0) {
      scl[0] = f16_scale(a);
      scl[1] = f16_scale(b);
    }
  }
  tc_before_sync();
  if constexpr (kPair) cluster_sync_all();  // the leader's barriers are initialised before any remote arrival
  else __syncthreads();
  tc_after_sync();
  const uint32_t tmem = *tmem_slot;
  const float sh = F16 ? scl[0] : 1.f, su = F16 ? scl[1] : 1.f;

  if (warp < kDrainers / 32) {
    // ---- drain: every kSPD steps, TMEM accumulator -> fp32 registers (round to nearest) ----
    float acc[kB / 2];
#pragma unroll
    for (int q = 0; q < kB / 2; ++q) acc[q] = 0.f;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + (warp >> 2) * (kB / 2);
    for (int64_t cyc = 0; cyc < steps / kSpd; ++cyc) {
      const int buf = static_cast<int>(cyc & 1);
      mbar_wait(&t_full[buf], (cyc >> 1) & 1);
      tc_after_sync();
#pragma unroll
      for (int c0 = 0; c0 < kB / 2; c0 += 32) {
        if (TC_MMA_ONLY) break;
        uint32_t v[32];
        tmem_ld32(lane_base + buf * kB + c0, v);
#pragma unroll
        for (int e = 0; e < 32; ++e) acc[c0 + e] += __uint_as_float(v[e]);
      }
      tc_before_sync();
      if constexpr (kPair) {
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(&t_empty[buf], 0);
      } else {
        mbar_arrive(&t_empty[buf]);
      }
    }
    // ---- partial[s][256 I + p]: this thread's row I, columns [128 (warp / 4), +128) ----
    float* out = partial + static_cast<int64_t>(s) * n + (I0 + (warp & 3) * 32 + lane) * kB + (warp >> 2) * (kB / 2);
    // powers of two, applied one at a time: exact, and sh * su itself may overflow (tiny inputs)
    const float ih = 1.f / sh, iu = 1.f / su;
#pragma unroll
    for (int q = 0; q < kB / 2; q += 4)
      *reinterpret_cast<float4*>(out + q) = make_float4(acc[q] * iu * ih, acc[q + 1] * iu * ih, acc[q + 2] * iu * ih,
                                                        acc[q + 3] * iu * ih);
  } else if (warp < kMmaWarp) {
    // ---- producers: A slabs and Hankel tiles, in consumption order, up to kBStages ahead ----
    const int ptid = tid - kDrainers;
    int a_use = 0;
    // fp16: the next tile's h values are loaded one tile ahead (their latency overlaps this tile)
    constexpr int kSt = (kStgN + kProducers - 1) / kProducers;
    // full-barrier hand-over: every producer thread (single CTA), or one arrival per warp on the leader
    auto arrive_full = [&](uint64_t* b) {
      if constexpr (kPair) {
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(b, 0);
      } else {
        mbar_arrive(b);
      }
    };
    const int64_t hoff = kPair ? 128 * static_cast<int64_t>(rank) : 0;  // this CTA's Hankel columns p
    StepIter it, nx;
    it.init(Dlo, Dn);
    nx = it;
    nx.next();
    float xn[F16 ? kSt : 1];
    if constexpr (F16) {
#pragma unroll
      for (int q = 0; q < kSt; ++q) xn[q] = __ldg(h + ((it.t0() + hoff + ptid + q * kProducers) & nm));
    }
    for (int64_t j = 0; j < steps; ++j, it = nx, nx.next()) {
      const int g = it.g;
      if (it.dd == 0) {
        const int st = a_use & 1;
        mbar_wait(&a_empty[st], ((a_use >> 1) & 1) ^ 1);
        unsigned char* hi = sm + (st * 2) * kSlabBytes;
        unsigned char* lo = sm + (st * 2 + 1) * kSlabBytes;
        const int rows = it.len + kMT;
        const int64_t ibase = I0 - it.d0() - it.len + 1;  // I - D of slab row 0
        // kBatch items per thread per pass, all loads first (one L2 latency per pass)
        constexpr int kBatch = 4;
        for (int base = ptid; base < (TC_MMA_ONLY && a_use >= 2 ? 0 : rows * kCh); base += kBatch * kProducers) {
          float4 v0[kBatch], v1[kBatch];
#pragma unroll
          for (int b = 0; b < kBatch; ++b) {
            const int idx = base + b * kProducers;
            const int rho = idx % rows, c = idx / rows;
            const int64_t Ip = (ibase + rho) & nbm;
            if (idx < rows * kCh) {
              const float* src = u + Ip * kB + (kB - kEl) - kKG * g - kEl * c;
              v0[b] = __ldg(reinterpret_cast<const float4*>(src));
              if constexpr (F16) v1[b] = __ldg(reinterpret_cast<const float4*>(src + 4));
            }
          }
#pragma unroll
          for (int b = 0; b < kBatch; ++b) {
            const int idx = base + b * kProducers;
            if (idx < rows * kCh) {
              const int rho = idx % rows, c = idx / rows;
              const int off = (c * rows + rho) * 16;
              if constexpr (F16) {
                const float v[8] = {v1[b].w, v1[b].z, v1[b].y, v1[b].x, v0[b].w, v0[b].z, v0[b].y, v0[b].x};
                st_split8(hi + off, lo + off, v, su);
              } else {
                st_split(reinterpret_cast<float*>(hi + off), reinterpret_cast<float*>(lo + off),
                         make_float4(v0[b].w, v0[b].z, v0[b].y, v0[b].x));
              }
            }
          }
        }
        fence_async_smem();
        arrive_full(&a_full[st]);
        ++a_use;
      }
      const int bs = static_cast<int>(j & (kBStages - 1));
      mbar_wait(&b_empty[bs], ((j / kBStages) & 1) ^ 1);
      unsigned char* thi = sm + kOffB + (bs * 2) * kTileBytes;
      unsigned char* tlo = sm + kOffB + (bs * 2 + 1) * kTileBytes;
      const int64_t t0 = it.t0() + hoff;
      if (TC_MMA_ONLY && j >= kBStages) {  // diagnostic: stages keep their first contents
        fence_async_smem();
        arrive_full(&b_full[bs]);
        continue;
      }
      constexpr int kRows = (kRows_B + kProducers - 1) / kProducers;
      if constexpr (F16) {
        // Split each of the tile's kRB + 8 values once into a packed (hi | lo << 16) fp16 word in a
        // double-buffered staging row, then build the 8-wide Hankel rows from it with byte permutes.
        uint32_t* stg = reinterpret_cast<uint32_t*>(sm + kOffStg) + (j & 1) * kStgN;
        float x[kSt];
#pragma unroll
        for (int q = 0; q < kSt; ++q) x[q] = xn[q];
        if (j + 1 < steps) {
          const int64_t t1 = nx.t0() + hoff;
#pragma unroll
          for (int q = 0; q < kSt; ++q) xn[q] = __ldg(h + ((t1 + ptid + q * kProducers) & nm));
        }
#pragma unroll
        for (int q = 0; q < kSt; ++q) {
          const int i = ptid + q * kProducers;
          if (i < kStgN) {
            const float a = x[q] * sh;
            const __half ha = __float2half_rn(a);
            stg[i] = static_cast<uint32_t>(__half_as_ushort(ha)) |
                     (static_cast<uint32_t>(__half_as_ushort(__float2half_rn(a - __half2float(ha)))) << 16);
          }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kProducers) : "memory");
#pragma unroll
        for (int q = 0; q < kRows; ++q) {
          const int r = ptid + q * kProducers;
          if (r < kRows_B) {
            uint32_t w[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) w[e] = stg[r + e];
            *reinterpret_cast<uint4*>(thi + r * 16) =
                make_uint4(__byte_perm(w[0], w[1], 0x5410), __byte_perm(w[2], w[3], 0x5410),
                           __byte_perm(w[4], w[5], 0x5410), __byte_perm(w[6], w[7], 0x5410));
            *reinterpret_cast<uint4*>(tlo + r * 16) =
                make_uint4(__byte_perm(w[0], w[1], 0x7632), __byte_perm(w[2], w[3], 0x7632),
                           __byte_perm(w[4], w[5], 0x7632), __byte_perm(w[6], w[7], 0x7632));
          }
        }
        fence_async_smem();
        arrive_full(&b_full[bs]);
        continue;
      }
      float v[kRows][kEl];
#pragma unroll
      for (int q = 0; q < kRows; ++q) {  // all loads first: one L2 latency per tile
        const int64_t t = t0 + ptid + q * kProducers;
#pragma unroll
        for (int e = 0; e < kEl; ++e) v[q][e] = __ldg(h + ((t + e) & nm));
      }
#pragma unroll
      for (int q = 0; q < kRows; ++q) {
        const int r = ptid + q * kProducers;
        if (r < kRows_B) {
          if constexpr (F16) {
            st_split8(thi + r * 16, tlo + r * 16, v[q], sh);
          } else {
            st_split(reinterpret_cast<float*>(thi + r * 16), reinterpret_cast<float*>(tlo + r * 16),
                     make_float4(v[q][0], v[q][1], v[q][2], v[q][3]));
          }
        }
      }
      fence_async_smem();
      arrive_full(&b_full[bs]);
    }
  } else if (lane == 0 && rank == 0) {
    // ---- MMA issue (one thread) ----
    constexpr uint32_t kFmt = F16 ? 0u : 2u;  // operand format: F16 (kind::f16) / TF32 (kind::tf32)
    constexpr uint32_t idesc = (1u << 4) | (kFmt << 7) | (kFmt << 10) | (static_cast<uint32_t>(kB >> 3) << 17) |
                               (static_cast<uint32_t>((CG * kMT) >> 4) << 24);
    auto commit = [&](uint64_t* b) {
      if constexpr (kPair) tc_commit_pair(b);
      else tc_commit(b);
    };
    const uint32_t abase = smem_u32(sm), bbase = smem_u32(sm + kOffB);
    int a_use = 0;
    uint32_t ahi = 0, alo = 0, lboA = 0;
    StepIter it;
    it.init(Dlo, Dn);
    for (int64_t j = 0; j < steps; ++j, it.next()) {
      const int64_t dd = it.dd;
      const int st = a_use & 1;
      if (dd == 0) {
        mbar_wait(&a_full[st], (a_use >> 1) & 1);
        ahi = abase + (st * 2) * kSlabBytes;
        alo = ahi + kSlabBytes;
        lboA = static_cast<uint32_t>(it.len + kMT) * 16u;
      }
      const int bs = static_cast<int>(j & (kBStages - 1));
      mbar_wait(&b_full[bs], (j / kBStages) & 1);
      const int64_t cyc = j / kSpd;
      const int buf = static_cast<int>(cyc & 1);
      const bool first = j % kSpd == 0;
      if (first) mbar_wait(&t_empty[buf], ((cyc >> 1) & 1) ^ 1);
      tc_after_sync();
      const uint32_t row0 = static_cast<uint32_t>(it.len - 1 - dd) * 16u;
      const uint32_t bhi = bbase + (bs * 2) * kTileBytes, blo = bhi + kTileBytes;
      const uint32_t tacc = tmem + buf * kB;
#pragma unroll
      for (int kk = 0; kk < kKG / kKS; ++kk) {
        const uint64_t dah = sdesc(ahi + row0 + 2u * kk * lboA, lboA, 128);
        const uint64_t dal = sdesc(alo + row0 + 2u * kk * lboA, lboA, 128);
        const uint64_t dbh = sdesc(bhi + 2u * kLboB * kk, kLboB, 128);
        const uint64_t dbl = sdesc(blo + 2u * kLboB * kk, kLboB, 128);
        if constexpr (kPair) {
          mma_pair(tacc, dah, dbh, idesc, (first && kk == 0) ? 0u : 1u, F16);
          mma_pair(tacc, dah, dbl, idesc, 1, F16);
          if (!TC_TWO_MMA) mma_pair(tacc, dal, dbh, idesc, 1, F16);
        } else if constexpr (F16) {
          mma_f16(tacc, dah, dbh, idesc, (first && kk == 0) ? 0u : 1u);
          mma_f16(tacc, dah, dbl, idesc, 1);
          if (!TC_TWO_MMA) mma_f16(tacc, dal, dbh, idesc, 1);
        } else {
          mma_tf32(tacc, dah, dbh, idesc, (first && kk == 0) ? 0u : 1u);
          mma_tf32(tacc, dah, dbl, idesc, 1);
          mma_tf32(tacc, dal, dbh, idesc, 1);
        }
      }
      commit(&b_empty[bs]);
      if (j % kSpd == kSpd - 1) commit(&t_full[buf]);
      if (dd == it.len - 1) {
        commit(&a_empty[st]);
        ++a_use;
      }
    }
  }
  tc_before_sync();
  if constexpr (kPair) cluster_sync_all();  // both CTAs done: no MMA or arrival still targets either
  else __syncthreads();
  if (warp == kMmaWarp) {
    tc_after_sync();
    if constexpr (kPair)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols) : "memory");
    else
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
  // Splits over block offsets, a function of n only (results are identical for every rank count): a
  // multiple of 37 (148 = 4 x 37 SMs), so that the units of the 1, 2, 4 or 8 ranks a product is sharded
  // over fill whole waves whenever each rank owns at least one tile: T = 32 tiles at n = 2^20 -> 37
  // splits: 1184 units = 8 waves at G = 1, 148 per rank (one wave) at G = 8; T = 512 at 2^24 -> 37.
  // Smaller T keep about 8 waves at G = 1 (T = 16 -> 74, T = 8 -> 148); never more splits than offsets.
  const int64_t T = p.tiles;
  int64_t s = T >= 32 ? 37 : T >= 8 ? 37 * (32 / T) : (148 * 8 + T - 1) / T;
  if (s > nb) s = nb;
  if (const char* v = getenv("CLB_TC_SPLITS")) s = atoll(v);
  p.splits = static_cast<int>(s);
  p.tile_lo = 0;
  p.tile_hi = p.tiles;
  p.split_lo = 0;
  p.split_hi = p.splits;
  return p;
}

namespace {
// fp16 operands win from n = 2^18 (4.19 vs 6.97 ms at 2^20, 1.09 vs 1.94 at 2^19, 0.43 vs 0.51
// at 2^18); below, slab rebuilds make the fp16 producers the bottleneck.  CLB_TC_F16=0/1 forces
// either.
bool use_f16(int64_t n) {
  const char* v = getenv("CLB_TC_F16");
  if (v && *v) return atoi(v) != 0;
  return n >= (int64_t(1) << 18);
}
}  // namespace

size_t tc_scratch_floats() { return 2 * kMaxBlocks; }

void tc_dense_init() {
  static std::atomic<uint64_t> devs{0};
  if (!first_use_on_device(devs)) return;
  for (const void* f : {reinterpret_cast<const void*>(k_tc_dense<false, 1>),
                        reinterpret_cast<const void*>(k_tc_dense<true, 1>),
                        reinterpret_cast<const void*>(k_tc_dense<false, 2>),
                        reinterpret_cast<const void*>(k_tc_dense<true, 2>)})
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem);
}

namespace {
// CTA pairs (cta_group::2) for every tile range made of whole pairs; CLB_TC_PAIR=0 forces single CTAs.
bool use_pairs(const ConvPlan& p) {
  static const int env = [] {
    const char* v = getenv("CLB_TC_PAIR");
    return (v && *v) ? atoi(v) : -1;
  }();
  if (env == 0) return false;
  return (p.tile_lo % 2) == 0 && (p.tile_hi % 2) == 0;
}
template <bool F16>
cudaError_t launch_pairs(const ConvPlan& p, const float* h, const float* u, float* partial, const float* maxes,
                         cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>((p.tile_hi - p.tile_lo) * p.splits));
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = kTcSmem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_tc_dense<F16, 2>, h, u, p.n, p.splits, p.tile_lo, partial, maxes);
}
}  // namespace

// The fp16 path's k_absmax2 -> k_tc_dense hand-over goes through the caller's own scratch
// (p.tc_scratch): two products on different streams never share it.
cudaError_t launch_tc_dense(const ConvPlan& p, const float* h, const float* u, float* partial, cudaStream_t st) {
  const int64_t units = (p.tile_hi - p.tile_lo) * p.splits;
  if (units <= 0) return cudaSuccess;
  tc_dense_init();
  if (use_f16(p.n)) {
    if (!p.tc_scratch) return cudaErrorInvalidValue;  // the plan's owner did not allocate tc_scratch_floats()
    k_absmax2<<<kMaxBlocks, 256, 0, st>>>(h, u, p.n, p.tc_scratch);
    if (use_pairs(p)) return launch_pairs<true>(p, h, u, partial, p.tc_scratch, st);
    k_tc_dense<true, 1><<<static_cast<unsigned>(units), kTcThreads, kTcSmem, st>>>(h, u, p.n, p.splits, p.tile_lo,
                                                                                   partial, p.tc_scratch);
  } else {
    if (use_pairs(p)) return launch_pairs<false>(p, h, u, partial, nullptr, st);
    k_tc_dense<false, 1><<<static_cast<unsigned>(units), kTcThreads, kTcSmem, st>>>(h, u, p.n, p.splits, p.tile_lo,
                                                                                    partial, nullptr);
  }
  return cudaGetLastError();
}

}  // namespace clb
