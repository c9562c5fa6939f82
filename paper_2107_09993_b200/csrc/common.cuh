// Device-side building blocks shared by the SkyCell kernels (sm_100a).
//
//  * per-warp output chunks (unordered survivor streams; the final ids are
//    put back in ascending order once, through an id bitmap -- refine.cpp:
//    101-103 sorts on the CPU instead);
//  * the point dominance predicate (dataset.hpp:55-62) and the sort-first
//    precedence order (refine.cpp:38-41) used by every dominance kernel;
//  * grid-cell arithmetic (grid.cpp:10-16, cell.hpp:102-107) and
//    check-before-set occupancy bits.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <utility>
#include <cuda_runtime.h>

namespace sk {

constexpr int kMaxD = 16;
constexpr double kUnitUpperBound = 1.0 - 0x1p-32;  // dataset.hpp:15
constexpr unsigned kFull = 0xffffffffu;

typedef unsigned long long u64;

// ------------------------------------------------ programmatic dependent launch
// Every kernel opens with pdl_enter(): wait until the grid it depends on has
// completed and flushed (griddepcontrol.wait -- a no-op for a plain launch),
// then let the next kernel of the stream be scheduled.  launch() enqueues
// with programmatic stream serialisation, so a dependent kernel's CTAs are
// resident and waiting when its predecessor drains: the 2-5 us launch gap
// between the ~60 dependent kernels of a query overlaps the predecessor's
// tail instead of idling the GPU.  SKYCELL_PDL=0 launches plainly.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

inline bool pdl_on() {
  static const bool on = [] {
    const char* e = std::getenv("SKYCELL_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename... KArgs, typename... Args>
inline void launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  (void)cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
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
__device__ __forceinline__ void set_bit_shared(uint32_t* bits, uint32_t idx) {
  const uint32_t m = 1u << (idx & 31);
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bits) + ((idx >> 5) << 2);
  uint32_t w;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(a));
  if (!(w & m)) asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(m) : "memory");
}

// Branch-free variant: the word is always read, the red.or is predicated on
// `cond` and on the bit being clear (no divergent region around it).
__device__ __forceinline__ void set_bit_shared_if(uint32_t* bits, uint32_t idx, bool cond) {
  const uint32_t m = 1u << (idx & 31);
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bits) + ((idx >> 5) << 2);
  uint32_t w;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(a));
  const uint32_t need = (cond && !(w & m)) ? 1u : 0u;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q red.shared.or.b32 [%0], %1;\n\t}" ::"r"(a), "r"(m),
      "r"(need)
      : "memory");
}

// mbarrier + bulk async copy (cp.async.bulk, SASS UBLKCP) helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(bar),
      "r"(phase)
      : "memory");
}
// one elected thread: expect `bytes` on the barrier, then copy them global -> shared
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of dst first
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

}  // namespace sk
