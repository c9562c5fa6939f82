// Device-side building blocks shared by the SkyCell kernels (sm_100a).
//
//  * ordered tile claiming + decoupled look-back prefix (stable, single-pass
//    stream compaction: survivors keep input order, so record ids leave every
//    stage ascending and the final result needs no sort -- refine.cpp:101-103
//    sorts on the CPU);
//  * the point dominance predicate (dataset.hpp:55-62) and the sort-first
//    precedence order (refine.cpp:38-41) used by every dominance kernel;
//  * grid-cell arithmetic (grid.cpp:10-16, cell.hpp:102-107).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace sk {

constexpr int kMaxD = 16;
constexpr double kUnitUpperBound = 1.0 - 0x1p-32;  // dataset.hpp:15
constexpr unsigned kFull = 0xffffffffu;

typedef unsigned long long u64;

// ---------------------------------------------------------------- memory order
// Look-back status words are self-contained (flag and value in one 64-bit
// word) and publish nothing else, so relaxed gpu-scope accesses suffice.  An
// acquire load would compile to CCTL.IVALL (a full L1 invalidate) per spin
// iteration -- measured at 45% of K1's stall samples before this change.
__device__ __forceinline__ void st_status(u64* p, u64 v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u64 ld_status(const u64* p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// --------------------------------------------------------- mbarrier / TMA
// Thin wrappers over the Hopper+/Blackwell async-copy primitives used by the
// streaming kernel: a 1-D bulk copy global -> shared (cp.async.bulk, SASS
// UBLKCP) that completes a transaction count on an mbarrier.
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// ------------------------------------------------------- decoupled look-back
// Status word per tile: bits 62-63 flag (0 empty, 1 aggregate, 2 inclusive
// prefix), bits 0-61 value.  Status arrays are zeroed once per query.
constexpr u64 kFlagAgg = 1ull << 62;
constexpr u64 kFlagInc = 2ull << 62;
constexpr u64 kValMask = (1ull << 62) - 1;

// Called by all 32 lanes of one warp.  Publishes `agg` for `tile` and returns
// the exclusive prefix over tiles [0, tile).
__device__ __forceinline__ u64 warp_lookback(u64* status, u64 tile, u64 agg) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_status(&status[0], kFlagInc | agg);
    return 0;
  }
  if (lane == 0) st_status(&status[tile], kFlagAgg | agg);
  u64 excl = 0;
  long long base = (long long)tile - 1;
  while (true) {
    const long long t = base - lane;
    u64 s;
    if (t >= 0) {
      do { s = ld_status(&status[t]); } while ((s >> 62) == 0);
    } else {
      s = kFlagInc;  // virtual predecessor with inclusive prefix 0
    }
    const unsigned inc = __ballot_sync(kFull, (s >> 62) == 2);
    const int stop = inc ? __ffs(inc) - 1 : 31;
    u64 v = (lane <= stop) ? (s & kValMask) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    excl += v;
    if (inc) break;
    base -= 32;
  }
  if (lane == 0) st_status(&status[tile], kFlagInc | (excl + agg));
  return excl;
}

// ------------------------------------------------ unordered warp output
// Survivor streams that need no order are written through per-warp output
// chunks reserved with one atomicAdd per chunk of slots (not per survivor: a
// single global counter would serialise ~10^6 atomics).  Slots a warp does
// not fill are stamped with kNoId, which every consumer skips; the record ids
// are put back in ascending order once, at the end, through an id bitmap.
constexpr uint32_t kNoId = 0xffffffffu;

struct WarpOut {
  u64 base;        // first slot of the current chunk (lane-uniform)
  unsigned fill;   // slots used in it
  unsigned chunk;  // chunk size (>= 32); fill starts at chunk so the first use reserves
};

// Reserve positions for the lanes with `flag` set; returns this lane's slot.
// Call with all 32 lanes.  A batch that does not fit the current chunk
// straddles into a freshly reserved one, so only each warp's last chunk can
// hold unused slots (stamped with kNoId by warp_close): the output capacity
// needed is count + warps * chunk whatever the survivor rate.
template <typename Stamp>
__device__ __forceinline__ u64 warp_reserve(WarpOut& wo, bool flag, u64* counter, Stamp) {
  const int lane = threadIdx.x & 31;
  const unsigned m = __ballot_sync(kFull, flag);
  const unsigned cnt = __popc(m);
  const unsigned rank = __popc(m & ((1u << lane) - 1));
  const unsigned rem = wo.chunk - wo.fill;
  u64 nb = 0;
  if (cnt > rem) {  // chunk >= 32 >= cnt: one new chunk always suffices
    if (lane == 0) nb = atomicAdd(counter, (u64)wo.chunk);
    nb = __shfl_sync(kFull, nb, 0);
  }
  const u64 slot = rank < rem ? wo.base + wo.fill + rank : nb + (rank - rem);
  if (cnt > rem) {
    wo.base = nb;
    wo.fill = cnt - rem;
  } else {
    wo.fill += cnt;
  }
  return slot;
}

template <typename Stamp>
__device__ __forceinline__ void warp_close(WarpOut& wo, Stamp stamp) {
  const int lane = threadIdx.x & 31;
  for (unsigned s = wo.fill + lane; s < wo.chunk; s += 32) stamp(wo.base + s);
}

// Block-wide stable ranks for PPT flags per thread laid out point-major:
// point (j, t) precedes (j', t') iff j < j' or (j == j' and t < t').
// scratch: PPT*NW + 1 u32 in shared memory.  Returns the block total; rank[j]
// is the exclusive position of flag j (valid only where flag[j]).
template <int THREADS, int PPT>
__device__ __forceinline__ unsigned block_ranks(const bool (&flag)[PPT], unsigned (&rank)[PPT],
                                                unsigned* scratch) {
  constexpr int NW = THREADS / 32;
  constexpr int M = PPT * NW;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1;
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    const unsigned m = __ballot_sync(kFull, flag[j]);
    rank[j] = __popc(m & lt);
    if (lane == 0) scratch[j * NW + warp] = __popc(m);
  }
  __syncthreads();
  if (warp == 0) {
    constexpr int PER = (M + 31) / 32;
    unsigned loc[PER];
    unsigned sum = 0;
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      const int idx = lane * PER + e;
      loc[e] = idx < M ? scratch[idx] : 0;
      sum += loc[e];
    }
    unsigned incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    unsigned run = incl - sum;
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      const int idx = lane * PER + e;
      if (idx < M) scratch[idx] = run;
      run += loc[e];
    }
    if (lane == 31) scratch[M] = incl;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < PPT; ++j) rank[j] += scratch[j * NW + warp];
  return scratch[M];
}

// ------------------------------------------------------------- dominance
// point_dominates(q, p), dataset.hpp:55-62: q no worse anywhere, strictly
// better somewhere.  Branch-free over a compile-time dimensionality.
template <typename T, int D>
__device__ __forceinline__ bool dominates(const T* q, const T* p) {
  bool le = true, lt = false;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    le &= q[k] <= p[k];
    lt |= q[k] < p[k];
  }
  return le & lt;
}

// Sort-first order (refine.cpp:38-41): ascending FP64 coordinate sum, ties by
// record id.  Sums are non-negative, so their IEEE bit patterns order as u64.
__device__ __forceinline__ bool precedes(u64 qs, uint32_t qi, u64 ps, uint32_t pi) {
  return qs < ps || (qs == ps && qi < pi);
}

// Coordinate value as the reference sees it after normalize(): f32 proxies
// encode the clamp 1 - 2^-32 (not representable in f32) as 1.0f, which is
// order-equivalent because every f32 below 1 is <= 1 - 2^-24.
__device__ __forceinline__ double true_value(float v) {
  return v >= 1.0f ? kUnitUpperBound : (double)v;
}
__device__ __forceinline__ double true_value(double v) { return v; }

// coord_sum, refine.cpp:22-27: left-to-right FP64 sum from 0.
template <typename T, int D>
__device__ __forceinline__ u64 fsum_bits(const T* p) {
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) s = __dadd_rn(s, true_value(p[k]));
  return (u64)__double_as_longlong(s);
}

// ------------------------------------------------------------------ cells
// point_to_cell (grid.cpp:10-16): col = (int32)(u * 2^layer), truncation.
// Clamped to [0, top] so a non-finite input (reported separately) can never
// index outside a bitmap.
__device__ __forceinline__ int cell_col(float v, float scale, int top) {
  const int c = __float2int_rz(__fmul_rn(v, scale));
  return min(max(c, 0), top);
}
__device__ __forceinline__ int cell_col(double u, double scale, int top) {
  const int c = __double2int_rz(__dmul_rn(u, scale));
  return min(max(c, 0), top);
}

__device__ __forceinline__ bool test_bit(const uint32_t* bits, u64 idx) {
  return (bits[idx >> 5] >> (idx & 31)) & 1u;
}

// Check-before-set: dense data re-hits the same words millions of times
// (SURVEY §7 hard part 5); a plain L2 load turns those into hits.
__device__ __forceinline__ void set_bit_global(uint32_t* bits, u64 idx) {
  const uint32_t m = 1u << (idx & 31);
  uint32_t* w = bits + (idx >> 5);
  if (!(__ldcg(w) & m)) atomicOr(w, m);
}
// Check-before-set through L1: a stale L1 copy can only cause a redundant
// (harmless) red.or, and hot words -- correlated data piles ~1e-3 n points
// into the origin cell -- stop reaching the L2 atomic unit after the first hit.
__device__ __forceinline__ void set_bit_cached(uint32_t* bits, u64 idx) {
  const uint32_t m = 1u << (idx & 31);
  uint32_t* w = bits + (idx >> 5);
  uint32_t v;
  asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(v) : "l"(w));
  if (!(v & m)) asm volatile("red.global.or.b32 [%0], %1;" ::"l"(w), "r"(m) : "memory");
}
// Fire-and-forget (red.global.or): no result to wait for.
__device__ __forceinline__ void red_or_global(uint32_t* bits, u64 idx) {
  asm volatile("red.global.or.b32 [%0], %1;" ::"l"(bits + (idx >> 5)), "r"(1u << (idx & 31)) : "memory");
}
__device__ __forceinline__ void set_bit_shared(uint32_t* bits, uint32_t idx) {
  const uint32_t m = 1u << (idx & 31);
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bits) + ((idx >> 5) << 2);
  uint32_t w;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(a));
  if (!(w & m)) asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(m) : "memory");
}

}  // namespace sk
