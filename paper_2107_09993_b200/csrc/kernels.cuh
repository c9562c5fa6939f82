// SkyCell skyline kernels for B200 (sm_100a).
//
// Stage map (DESIGN.md §3 has the bound and the algorithmic bytes of each):
//   K0  k_sample / k_filter_from_table  a sample's occupancy at a coarse level la
//       sample tables, sample skyline   -> height table H (a point whose level-la
//       -> k_strength_order,            cell is strictly dominated by an occupied
//          k_filter_lists               sample cell cannot be in a candidate
//                                       cell); the sample's skyline
//                                       -> the filter points F of K4.
//   K1  k_stream                        THE HBM-bound pass: normalize (dataset.cpp:
//                                       22-50), point_to_cell (grid.cpp:10-16),
//                                       occupancy (grid.cpp:78-102), the H test,
//                                       survivors compacted to S1.  Reads every
//                                       coordinate exactly once.
//   K3  k_rowmin_prefix1w / k_rowmin /  cell pruning as a d-dimensional prefix-OR,
//       k_prefix_min / k_count_rows /   stored as a (d-1)-dim prefix-min table;
//       k_downsample*                   per-layer |KS_i|, |CS_i| (replaces
//                                       shrink_seq.cpp:87-231, shrink_par.cpp:179-278).
//   K4  k_candidates (K4a, K4b)         survivors in candidate cells (points_examined,
//                                       refine.cpp:90-96) not dominated by F.
//   K5  k_list_* / k_allpairs_lists /   exact sort-first dominance (refine.cpp:31-59,
//       k_allpairs_long, or tree.cuh    98-99): column lists for small sets, the
//                                       dominance tree for large ones.
//   K6  k_mark_ids / k_bits_*           ascending ids through an id bitmap.
#pragma once

#include <cub/block/block_radix_sort.cuh>

#include "common.cuh"

#ifndef SKY_K4A_HEAD
#define SKY_K4A_HEAD 8
#endif

namespace sk {

// Non-template kernels are `static`: this header is included by several
// translation units (skycell_gpu.cu, inst.cu per D).

// ------------------------------------------------------------------ rows
template <typename T, int D>
__device__ __forceinline__ void load_row(const T* __restrict__ base, u64 i, T (&v)[D]) {
  constexpr int BYTES = D * (int)sizeof(T);
  const char* p = reinterpret_cast<const char*>(base + i * D);
  if constexpr (BYTES % 16 == 0) {
#pragma unroll
    for (int c = 0; c < BYTES / 16; ++c) {
      const float4 x = __ldcs(reinterpret_cast<const float4*>(p) + c);
      memcpy(reinterpret_cast<char*>(v) + 16 * c, &x, 16);
    }
  } else if constexpr (BYTES % 8 == 0) {
#pragma unroll
    for (int c = 0; c < BYTES / 8; ++c) {
      const float2 x = __ldcs(reinterpret_cast<const float2*>(p) + c);
      memcpy(reinterpret_cast<char*>(v) + 8 * c, &x, 8);
    }
  } else {
#pragma unroll
    for (int c = 0; c < BYTES / 4; ++c) {
      const float x = __ldcs(reinterpret_cast<const float*>(p) + c);
      memcpy(reinterpret_cast<char*>(v) + 4 * c, &x, 4);
    }
  }
}

// Cached variant for the small intermediate arrays (S1/S2/Z), which are
// re-read by later kernels.
template <typename T, int D>
__device__ __forceinline__ void load_row_cached(const T* __restrict__ base, u64 i, T (&v)[D]) {
  constexpr int BYTES = D * (int)sizeof(T);
  const char* p = reinterpret_cast<const char*>(base + i * D);
  if constexpr (BYTES % 16 == 0) {
#pragma unroll
    for (int c = 0; c < BYTES / 16; ++c) {
      const float4 x = reinterpret_cast<const float4*>(p)[c];
      memcpy(reinterpret_cast<char*>(v) + 16 * c, &x, 16);
    }
  } else if constexpr (BYTES % 8 == 0) {
#pragma unroll
    for (int c = 0; c < BYTES / 8; ++c) {
      const float2 x = reinterpret_cast<const float2*>(p)[c];
      memcpy(reinterpret_cast<char*>(v) + 8 * c, &x, 8);
    }
  } else {
#pragma unroll
    for (int c = 0; c < BYTES / 4; ++c) {
      const float x = reinterpret_cast<const float*>(p)[c];
      memcpy(reinterpret_cast<char*>(v) + 4 * c, &x, 4);
    }
  }
}

template <typename T, int D>
__device__ __forceinline__ void store_row(T* __restrict__ base, u64 i, const T (&v)[D]) {
  constexpr int BYTES = D * (int)sizeof(T);
  char* p = reinterpret_cast<char*>(base + i * D);
  if constexpr (BYTES % 16 == 0) {
#pragma unroll
    for (int c = 0; c < BYTES / 16; ++c) {
      float4 x;
      memcpy(&x, reinterpret_cast<const char*>(v) + 16 * c, 16);
      reinterpret_cast<float4*>(p)[c] = x;
    }
  } else if constexpr (BYTES % 8 == 0) {
#pragma unroll
    for (int c = 0; c < BYTES / 8; ++c) {
      float2 x;
      memcpy(&x, reinterpret_cast<const char*>(v) + 8 * c, 8);
      reinterpret_cast<float2*>(p)[c] = x;
    }
  } else {
#pragma unroll
    for (int c = 0; c < BYTES / 4; ++c) {
      float x;
      memcpy(&x, reinterpret_cast<const char*>(v) + 4 * c, 4);
      reinterpret_cast<float*>(p)[c] = x;
    }
  }
}

// ----------------------------------------------------- normalisation params
struct Norm {
  double mn[kMaxD];
  double sc[kMaxD];  // range > 0 ? 1/range : 0, computed on the host exactly as dataset.cpp:32-36
};

// One raw coordinate -> the stored value (TOut) and its layer-rho column.
// IDENT: f32 input with declared range [0, 1]: normalize() is the identity up
// to the clamp, so the f32 value itself (proxy-encoded) is stored.
template <typename TIn, typename TOut, bool IDENT>
struct Coord;

template <>
struct Coord<float, float, true> {
  __device__ __forceinline__ static float value(float v, const Norm&, int) {
    return fminf(fmaxf(v, 0.0f), 1.0f);  // NaN -> 0; non-finite records are reported separately
  }
  __device__ __forceinline__ static int col(float u, float fscale, double, int top) {
    return cell_col(u, fscale, top);
  }
};

template <typename TIn>
struct Coord<TIn, double, false> {
  // u = clamp((v - min) * scale, 0, 1 - 2^-32), dataset.cpp:41-45; no FMA.
  __device__ __forceinline__ static double value(TIn v, const Norm& nm, int k) {
    double u = __dmul_rn(__dsub_rn((double)v, nm.mn[k]), nm.sc[k]);
    u = (u < 0.0) ? 0.0 : ((kUnitUpperBound < u) ? kUnitUpperBound : u);
    return u;
  }
  __device__ __forceinline__ static int col(double u, float, double dscale, int top) {
    return cell_col(u, dscale, top);
  }
};

__device__ __forceinline__ bool finite_v(float v) { return isfinite(v); }
__device__ __forceinline__ bool finite_v(double v) { return isfinite(v); }

// ------------------------------------------------------------ K0: sample
// The first m points are the sample.  One pass records their occupancy at
// the smem filter level la and at layer rho, and keeps their normalised rows
// (with FP64 sums and record ids) for the sample skyline.
struct SampleParams {
  const void* coords;
  u64 m;
  int rho, la;
  Norm nm;
  uint32_t* occ_la;   // 2^(la*d) bits
  uint32_t* occ_rho;  // 2^(rho*d) bits (nullptr when rho == la)
  void* rows;
  uint32_t* ids;
  u64* fsum;
  uint32_t id_base;   // global id of local record 0 (shard offset)
};

template <typename TIn, typename TOut, int D, bool IDENT>
__global__ void __launch_bounds__(256) k_sample(SampleParams p) {
  pdl_enter();
  const TIn* coords = static_cast<const TIn*>(p.coords);
  const int top = (1 << p.rho) - 1;
  const float fscale = ldexpf(1.0f, p.rho);
  const double dscale = ldexp(1.0, p.rho);
  const int sh = p.rho - p.la;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < p.m; i += (u64)gridDim.x * blockDim.x) {
    TIn raw[D];
    load_row<TIn, D>(coords, i, raw);
    TOut u[D];
    u64 la_lin = 0, lin = 0;
#pragma unroll
    for (int k = D - 1; k >= 0; --k) {
      u[k] = Coord<TIn, TOut, IDENT>::value(raw[k], p.nm, k);
      const int c = Coord<TIn, TOut, IDENT>::col(u[k], fscale, dscale, top);
      la_lin = (la_lin << p.la) | (u64)(c >> sh);
      lin = (lin << p.rho) | (u64)c;
    }
    // check-before-set through L1 (no dependent L2 round trip on a miss-free
    // hot word; a stale line only costs a redundant red.or)
    set_bit_cached(p.occ_la, la_lin);
    if (p.occ_rho) set_bit_cached(p.occ_rho, lin);
    store_row<TOut, D>(static_cast<TOut*>(p.rows), i, u);
    p.ids[i] = p.id_base + (uint32_t)i;
    p.fsum[i] = fsum_bits<TOut, D>(u);
  }
}

// H from a prefix-min table PM of the sample occupancy at level lf (built by
// the multi-CTA table kernels): H[x] = all x_k >= 1 ? PM[x - 1] : none.
// Bit 7 (entries are <= 2^lf - 1 <= 127, "none" = 255) is the row's COVER
// flag when occ_s (the sample's level-lf occupancy) is given: every level
// (lf-1) parent of the row's dropped cells (c_0 > H[x]) holds a sample point,
// so K1 need not record dropped points of this row at level lf-1 -- the
// sample's level-(lf-1) occupancy is OR-ed into that layer instead.
static __global__ void k_filter_from_table(const uint8_t* __restrict__ PM, int lf, int d, uint32_t rows,
                                    uint8_t* __restrict__ H, const uint32_t* __restrict__ occ_s) {
  pdl_enter();
  const uint32_t mask = (1u << lf) - 1;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
    bool ok = true;
    uint32_t prev = 0;
    for (int k = 1; k < d; ++k) {
      const uint32_t c = (r >> (lf * (k - 1))) & mask;
      ok &= c >= 1;
      prev |= (c - 1) << (lf * (k - 1));
    }
    uint32_t h = ok ? PM[prev] : 255u;
    if (occ_s && h < mask) {
      // dropped columns c0 in (h, 2^lf - 1]; their parents' columns (h+1)/2 .. (2^lf-1)/2
      bool cover = true;
      for (uint32_t pc = (h + 1) >> 1; pc <= (mask >> 1) && cover; ++pc) {
        bool any = false;
        for (uint32_t cm = 0; cm < (1u << (d - 1)) && !any; ++cm) {
          u64 base = 0;  // child (2 pc, 2 floor(x_k / 2) + b_k): dim-0 pair 2pc, 2pc+1 in one word
          for (int k = 1; k < d; ++k) {
            const uint32_t xk = (r >> (lf * (k - 1))) & mask;
            base |= (u64)((xk & ~1u) | ((cm >> (k - 1)) & 1u)) << (lf * k);
          }
          const u64 bit = base + 2 * pc;
          any = ((occ_s[bit >> 5] >> (bit & 31)) & 3u) != 0;
        }
        cover = any;
      }
      if (cover) h |= 0x80u;
    }
    H[r] = (uint8_t)h;
  }
}

// A layer-L cell c is strictly dominated (all columns) by an occupied cell iff
// all c_k >= 1 and PM[c1-1, .., c_{d-1}-1] <= c0 - 1, PM being the prefix-min
// table of the layer's occupancy.
template <typename TT, int D>
__device__ __forceinline__ bool strictly_dominated_cols(const TT* __restrict__ PM, const int* col, int L) {
  u64 idx = 0;
  bool ok = col[0] >= 1;
#pragma unroll
  for (int k = D - 1; k >= 1; --k) {
    ok &= col[k] >= 1;
    idx = (idx << L) | (u64)(col[k] - 1);
  }
  return ok && (int64_t)__ldg(PM + idx) <= (int64_t)col[0] - 1;
}

// -------------------------------------------------------- K1: the stream
// Cell filter from a sample (SURVEY §0.3 applied to a sample): a point whose
// level-la cell (la <= 7, table H in shared memory) is strictly dominated by
// an occupied sample cell cannot lie in a layer-rho candidate cell.  Such a
// point can influence the reference's per-layer key/candidate sets only at
// layers < la, so its occupancy is recorded at layer la-1 in
// a small shared-memory bitmap.  Survivors (11.9% at the headline config) go
// to per-warp output chunks and mark their layer-rho cell.  Every coordinate
// is read once; the main loop has no block barrier.
struct StreamParams {
  const void* coords;
  u64 n;
  int rho, la;
  uint32_t lo_words;       // shared bitmap at layer la-1 (0 when la <= 1)
  uint32_t h_entries;
  Norm nm;
  const uint8_t* H;        // level-la filter table
  const void* PMs;         // layer-rho prefix-min table of the sample (u8 or u32), nullptr if rho == la
  int pms_wide;            // PMs entries are u32
  uint32_t* occ_rho;       // layer rho, survivors only
  uint32_t* occ_rm1;       // layer rho-1, points failing test B
  uint32_t* slabs;         // per-CTA copies of the layer la-1 bitmap
  void* out_rows;
  uint32_t* out_ids;
  u64* out_reserved;       // slots handed out (multiple of chunk)
  unsigned chunk;          // output chunk per warp reservation
  u64* kept;               // exact number of survivors
  u64* nonfinite;          // max of (~record) over non-finite records: 0 = none
  uint32_t id_base;        // global id of local record 0 (shard offset)
  // filter-point head (K0's strongest filter points): survivors they dominate
  // with a strictly smaller sum leave only their layer-rho cell index in the
  // D stream (points_examined still counts them if the cell is a candidate)
  const void* f_rows;      // nullptr: no head test
  const u64* f_fsum;
  const u64* f_count;
  void* d_cells;           // u32 (rho*d <= 32) or u64 cell indices
  u64* d_reserved;
};

constexpr int kK1Head = 8;  // filter points tested per K1 survivor

// Column of a coordinate at an arbitrary level L <= rho: floor(u * 2^L) is
// the layer-rho column shifted right by rho - L (power-of-two scalings are
// exact), computed directly to keep the per-point path short.
template <typename TIn, typename TOut, bool IDENT>
__device__ __forceinline__ int col_at(TIn raw, const Norm& nm, int k, float fs, double ds, int top);
template <>
__device__ __forceinline__ int col_at<float, float, true>(float raw, const Norm&, int, float fs, double, int top) {
  // saturate to [0, 1] (NaN -> 0), scale, truncate; only the top needs a clamp
  return min(__float2int_rz(__fmul_rn(__saturatef(raw), fs)), top);
}
template <>
__device__ __forceinline__ int col_at<float, double, false>(float raw, const Norm& nm, int k, float, double ds, int top) {
  return cell_col(Coord<float, double, false>::value(raw, nm, k), ds, top);
}
template <>
__device__ __forceinline__ int col_at<double, double, false>(double raw, const Norm& nm, int k, float, double ds, int top) {
  return cell_col(Coord<double, double, false>::value(raw, nm, k), ds, top);
}

// Level of the shared-memory filter table for (d, rho): the largest L <=
// min(rho, 7) whose table (2^(L(d-1)) bytes) fits 32 KB.
__host__ __device__ constexpr int filter_level(int rho, int d) {
  int best = 1;
  for (int L = 1; L <= (rho < 7 ? rho : 7); ++L)
    if ((1ull << (L * (d - 1))) <= 32768ull && L * d <= 30) best = L;
  return best;
}

// Per-dimension digit index with the magic-number trick: for u in [0, 1),
// fma.rz(u, 2^L, 2^23) is the float 2^23 + trunc(u * 2^L) exactly, whose bit
// pattern is 0x4B000000 + col.  Summing bit patterns with power-of-two digit
// weights and subtracting the constant sum of 0x4B000000 digits yields the
// packed index (mod 2^32).
__device__ __forceinline__ uint32_t mag_col(float u, float scale) {
  return __float_as_uint(__fmaf_rz(u, scale, 8388608.0f));
}

// Warp-centric persistent kernel: each warp walks tiles of 32*PPT
// consecutive points round-robin, with the next tile's loads issued before
// the current tile is processed (register double buffering).  Survivors of
// the level-la test go straight to per-warp output chunks (one reservation
// per tile); their layer-rho cells are marked with fire-and-forget red.or.
// RHO > 0 (f32 identity path) fixes rho and la at compile time so every index
// is a constant-weight IMAD chain; RHO == 0 is the general runtime path.
// REC_LA (identity path with fixed RHO): dropped points record their level-la
// cell -- its index is the H lookup's index plus c_0, no second set of
// digits -- in a per-CTA 2^(la d)-bit shared bitmap (128 KB at d = 4, la = 5,
// so one 768-thread CTA per SM).  Otherwise they record their level la-1 cell.
// BULK (f32 rows of 16-byte multiples): each warp's tiles arrive by
// cp.async.bulk into a two-stage shared-memory ring (one instruction per tile
// from one lane, completion on an mbarrier) instead of per-lane LDG.128 into
// two register buffers; survivors are read back from the ring stage.
template <typename TIn, typename TOut, int D, bool IDENT, int THREADS, int PPT, int RHO, int MINB = 3, bool REC_LA = false,
          bool BULK = false, int NST = 2>
__global__ void __launch_bounds__(THREADS, MINB) k_stream(StreamParams p) {
  pdl_enter();
  static_assert(PPT <= 8, "survivor codes are (j * 32 + lane) in one byte");
  extern __shared__ __align__(16) uint8_t sm[];
  uint32_t* occ_s = reinterpret_cast<uint32_t*>(sm);
  uint8_t* H_s = sm + ((p.lo_words * 4 + 15) & ~15u);
  uint8_t* code_w = H_s + ((p.h_entries + 15) & ~15u) + (threadIdx.x >> 5) * (32 * PPT);  // survivor codes
  // survivor rows staged per warp (32 * PPT rows), after the codes and the filter head
  TIn* rows_w = reinterpret_cast<TIn*>(H_s + ((p.h_entries + 15) & ~15u) + THREADS * PPT +
                                       ((kK1Head * (D * sizeof(TOut) + 8) + 15) & ~(size_t)15)) +
                (size_t)(threadIdx.x >> 5) * (32 * PPT) * D;
  static_assert(!BULK || (D * sizeof(TIn)) % 16 == 0, "bulk tiles are whole 16-byte rows");
  if constexpr (BULK)  // NST ring stages per warp in place of the survivor staging area
    rows_w = reinterpret_cast<TIn*>(H_s + ((p.h_entries + 15) & ~15u) + THREADS * PPT +
                                    ((kK1Head * (D * sizeof(TOut) + 8) + 15) & ~(size_t)15)) +
             (size_t)(threadIdx.x >> 5) * NST * (32 * PPT) * D;
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      H_s + ((p.h_entries + 15) & ~15u) + THREADS * PPT + ((kK1Head * (D * sizeof(TOut) + 8) + 15) & ~(size_t)15) +
      (size_t)THREADS * PPT * D * sizeof(TIn) * (BULK ? NST : 1)) + (threadIdx.x >> 5) * NST;
  TOut* fh_rows = reinterpret_cast<TOut*>(H_s + ((p.h_entries + 15) & ~15u) + THREADS * PPT);
  u64* fh_sum = reinterpret_cast<u64*>(fh_rows + kK1Head * D);
  uint32_t nfh = 0;
  if (p.f_rows) {
    const u64 fc = *p.f_count;
    nfh = (uint32_t)(fc < (u64)kK1Head ? fc : (u64)kK1Head);
    for (uint32_t e = threadIdx.x; e < nfh * D; e += THREADS) fh_rows[e] = static_cast<const TOut*>(p.f_rows)[e];
    for (uint32_t e = threadIdx.x; e < nfh; e += THREADS) fh_sum[e] = p.f_fsum[e];
  }
  for (uint32_t w = threadIdx.x; w < p.lo_words; w += THREADS) occ_s[w] = 0;
  for (uint32_t e = threadIdx.x; e < p.h_entries; e += THREADS) H_s[e] = p.H[e];
  __syncthreads();

  const TIn* coords = static_cast<const TIn*>(p.coords);
  TOut* out_rows = static_cast<TOut*>(p.out_rows);
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1;
  const uint32_t n = (uint32_t)p.n;
  constexpr uint32_t WT = 32u * PPT;
  // 64-bit here: n + WT - 1 wraps for n within WT of 2^32 (n < 2^32 holds)
  const uint32_t ntiles = (uint32_t)(((u64)n + WT - 1) / WT);
  const uint32_t nfull = n / WT;
  const uint32_t gw = (blockIdx.x * THREADS + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * THREADS) >> 5;
  constexpr bool kFixed = RHO > 0;
  constexpr int kLa = kFixed ? filter_level(RHO, D) : 1;
  const int rho = kFixed ? RHO : p.rho;
  const int la = kFixed ? kLa : p.la;
  const int top = (1 << rho) - 1, top_a = (1 << la) - 1;
  const float fs_r = ldexpf(1.0f, rho), fs_a = ldexpf(1.0f, la);
  const double ds_r = ldexp(1.0, rho), ds_a = ldexp(1.0, la);
  const uint32_t mul_a = 1u << la, mul_lo = 1u << (la > 1 ? la - 1 : 0);
  const float fs_lo = ldexpf(1.0f, la > 1 ? la - 1 : 0);
  uint32_t hcorr = 0, locorr = 0;
  for (int k = D - 1; k >= 1; --k) hcorr = hcorr * mul_a + 0x4B000000u;
  for (int k = D - 1; k >= 0; --k) locorr = locorr * mul_lo + 0x4B000000u;
  const bool rec_lo = !REC_LA && la >= 2;
  WarpOut wo{0, p.chunk, p.chunk};
  auto stamp = [&](u64 slot) { p.out_ids[slot] = kNoId; };
  unsigned kept = 0;
  // D stream: empty slots hold the all-ones cell index, which no layer uses
  const bool d_wide = rho * D >= 32;  // u32 only while the all-ones marker is no cell
  WarpOut wd{0, p.chunk, p.chunk};
  auto dstamp = [&](u64 slot) {
    if (d_wide) static_cast<u64*>(p.d_cells)[slot] = ~0ull;
    else static_cast<uint32_t*>(p.d_cells)[slot] = ~0u;
  };

  // Two register buffers in ping-pong: the next tile's loads are in flight
  // while the current one is processed, with no register copies between them
  // (a copying double buffer cost ~7% of K1's instructions, ncu).
  TIn buf_a[PPT][D], buf_b[PPT][D];
  auto load_tile = [&](TIn (&raw)[PPT][D], uint32_t t) {
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      // t * WT < n, so n - t * WT cannot wrap; t * WT + j * 32 + lane can
      // (for n near 2^32) and is formed only for valid rows
      if (t < nfull || (uint32_t)(j * 32 + lane) < n - t * WT) load_row<TIn, D>(coords, t * WT + j * 32 + lane, raw[j]);
    }
  };
  // deferred check-before-set of a layer-rho occupancy bit (K1 survivors)
  uint32_t* pend_w = nullptr;
  uint32_t pend_m = 0, pend_v = 0;
  bool pend_on = false;
  auto resolve_pending = [&]() {
    if (pend_on && !(pend_v & pend_m)) asm volatile("red.global.or.b32 [%0], %1;" ::"l"(pend_w), "r"(pend_m) : "memory");
    pend_on = false;
  };
  auto process = [&](TIn (&cur)[PPT][D], uint32_t t, const TIn* stage) {
    const bool full = t < nfull;
    const uint32_t base = t * WT + lane;
    bool keep[PPT];
    bool bad = false;
    // Fast path (identity f32 input, full tile, every coordinate of the tile
    // in [+0, 1) -- one unsigned max of the bit patterns per point): no
    // clamps, no NaN/Inf probe and no divergent occupancy update.  Anything
    // else (negative, >= 1, NaN, Inf, the last partial tile) takes the
    // general path below.
    bool fastp = false;
    if constexpr (IDENT && !REC_LA) {
      if (full) {
        bool inr = true;
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
          uint32_t mx = __float_as_uint(cur[j][0]);
#pragma unroll
          for (int k = 1; k < D; ++k) mx = max(mx, __float_as_uint(cur[j][k]));
          inr &= mx < 0x3F800000u;
        }
        fastp = __all_sync(kFull, inr);
      }
    }
    if (fastp) {
      if constexpr (IDENT && !REC_LA) {
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
          uint32_t hidx = 0;
#pragma unroll
          for (int k = D - 1; k >= 1; --k) hidx = hidx * mul_a + mag_col(cur[j][k], fs_a);
          const int c0 = (int)(mag_col(cur[j][0], fs_a) - 0x4B000000u);
          const uint32_t hv = H_s[hidx - hcorr];
          const bool fail_a = c0 > (int)(hv & 0x7Fu);
          keep[j] = !fail_a;
          if (rec_lo) {
            // a dropped point of a covered row needs no level la-1 record
            const bool need = fail_a && !(hv & 0x80u);
            if (__any_sync(kFull, need)) {
              uint32_t lo = 0;
#pragma unroll
              for (int k = D - 1; k >= 1; --k) lo = lo * mul_lo + mag_col(cur[j][k], fs_lo);
              set_bit_shared_if(occ_s, lo * mul_lo + mag_col(cur[j][0], fs_lo) - locorr, need);
            }
          }
        }
      }
    } else
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      const bool valid = full || (uint32_t)(j * 32 + lane) < n - t * WT;
      bool fail_a;
      if constexpr (IDENT) {
        // u = min(max(v, 0), 1 - 2^-24): every column stays below 2^L (the
        // reference clamps to 1 - 2^-32, whose column is also 2^L - 1); NaN -> 0
        float probe = cur[j][D - 1];
        uint32_t hidx = 0, lo = 0;
#pragma unroll
        for (int k = D - 1; k >= 1; --k) {
          if (k != D - 1) probe += cur[j][k];
          const float u = fminf(fmaxf(cur[j][k], 0.0f), 0x1.fffffep-1f);
          hidx = hidx * mul_a + mag_col(u, fs_a);
          if (rec_lo) lo = lo * mul_lo + mag_col(u, fs_lo);
        }
        probe += cur[j][0];
        const float u0 = fminf(fmaxf(cur[j][0], 0.0f), 0x1.fffffep-1f);
        const int c0 = (int)(mag_col(u0, fs_a) - 0x4B000000u);
        bad |= !isfinite(probe);
        fail_a = c0 > (int)(H_s[hidx - hcorr] & 0x7Fu);  // bit 7: the cover flag
        if constexpr (REC_LA) {
          if (valid && fail_a) set_bit_shared(occ_s, (hidx - hcorr) * mul_a + (uint32_t)c0);
        } else {
          if (valid && fail_a && rec_lo) set_bit_shared(occ_s, lo * mul_lo + mag_col(u0, fs_lo) - locorr);
        }
      } else {
        TIn sum = cur[j][0];
#pragma unroll
        for (int k = 1; k < D; ++k) sum += cur[j][k];
        bad |= valid && !finite_v(sum);
        int ca[D];
#pragma unroll
        for (int k = 0; k < D; ++k) ca[k] = col_at<TIn, TOut, IDENT>(cur[j][k], p.nm, k, fs_a, ds_a, top_a);
        uint32_t hidx = 0, lo = 0;
#pragma unroll
        for (int k = D - 1; k >= 1; --k) hidx = hidx * mul_a + (uint32_t)ca[k];
        fail_a = ca[0] > (int)(H_s[hidx] & 0x7Fu);
#pragma unroll
        for (int k = D - 1; k >= 0; --k) lo = lo * mul_lo + (uint32_t)(ca[k] >> 1);
        if (valid && fail_a && rec_lo) set_bit_shared(occ_s, lo);
      }
      keep[j] = valid && !fail_a;
    }
    // one output reservation per tile
    unsigned mk[PPT], tot = 0;
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      mk[j] = __ballot_sync(kFull, keep[j]);
      tot += __popc(mk[j]);
    }
    if (tot) {
      // Survivors (~12% of the tile at the headline config) are compacted
      // onto consecutive lanes before any per-survivor work: their (j, lane)
      // codes are staged in tile order, each lane pulls one survivor's
      // coordinates by shuffle, and the row / id stores are coalesced.
      {
        unsigned cum = 0;
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
          if (keep[j]) {
            const unsigned sl = cum + __popc(mk[j] & lt);
            code_w[sl] = (uint8_t)(j * 32 + lane);
            if constexpr (!BULK) store_row<TIn, D>(rows_w, sl, cur[j]);
          }
          cum += __popc(mk[j]);
        }
      }
      __syncwarp();
      for (unsigned r = 0; r < tot; r += 32) {
        const unsigned sidx = r + lane;
        const bool act = sidx < tot;
        const unsigned cd = act ? code_w[sidx] : 0u;
        const int sj = (int)(cd >> 5), src = (int)(cd & 31);
        TIn x[D];
        if constexpr (BULK) load_row_cached<TIn, D>(stage, act ? cd : 0u, x);  // the tile's ring stage
        else load_row_cached<TIn, D>(rows_w, act ? sidx : 0u, x);  // staged in shared memory
        TOut u[D];
        int c[D];
#pragma unroll
        for (int k = 0; k < D; ++k) {
          if constexpr (IDENT) {
            u[k] = __saturatef(x[k]);  // the stored proxy (dataset.cpp:45 clamp, 1.0f = 1 - 2^-32)
            c[k] = (int)(mag_col(fminf(u[k], 0x1.fffffep-1f), fs_r) - 0x4B000000u);
          } else {
            u[k] = Coord<TIn, TOut, IDENT>::value(x[k], p.nm, k);
            c[k] = col_at<TIn, TOut, IDENT>(x[k], p.nm, k, fs_r, ds_r, top);
          }
        }
        // Test B: a layer-rho cell strictly dominated by an occupied SAMPLE
        // cell is no candidate; such a point only needs its
        // layer rho-1 cell recorded for the coarser layers' counts.
        bool keep_b = act;
        if (act && p.PMs) {
          bool ok = c[0] >= 1;
          u64 idx = 0;
#pragma unroll
          for (int k = D - 1; k >= 1; --k) {
            ok &= c[k] >= 1;
            idx = (idx << rho) | (u64)(c[k] - 1);
          }
          if (ok) {
            const int64_t pm = p.pms_wide ? (int64_t)__ldg(static_cast<const uint32_t*>(p.PMs) + idx)
                                          : (int64_t)__ldg(static_cast<const uint8_t*>(p.PMs) + idx);
            if (pm <= (int64_t)c[0] - 1) {
              keep_b = false;
              u64 lo = 0;
#pragma unroll
              for (int k = D - 1; k >= 0; --k) lo = (lo << (rho - 1)) | (u64)(c[k] >> 1);
              set_bit_cached(p.occ_rm1, lo);
            }
          }
        }
        u64 lin = 0;
        if (keep_b) {
#pragma unroll
          for (int k = D - 1; k >= 0; --k) lin = (lin << rho) | (u64)c[k];
        }
        if (r == 0) {
          // The first survivor batch's check-before-set is deferred to the
          // next tile: its L1/L2 load is issued now and tested after that
          // tile's main work, so no warp waits on it (a stale word only
          // costs a redundant red).
          resolve_pending();
          if (keep_b) {
            pend_w = p.occ_rho + (lin >> 5);
            pend_m = 1u << (lin & 31);
            asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(pend_v) : "l"(pend_w));
            pend_on = true;
          }
        } else if (keep_b) {
          set_bit_cached(p.occ_rho, lin);
        }
        // filter-point head: branch-free over the 8 strongest filter points
        bool to_s1 = keep_b;
        if (nfh) {
          const u64 ps = fsum_bits<TOut, D>(u);
          bool dom = false;
#pragma unroll
          for (int f = 0; f < kK1Head; ++f)
            if (f < (int)nfh) dom |= dominates<TOut, D>(fh_rows + f * D, u) && fh_sum[f] < ps;
          to_s1 = keep_b && !dom;
          const bool to_d = keep_b && dom;
          const u64 dslot = warp_reserve(wd, to_d, p.d_reserved, dstamp);
          if (to_d) {
            if (d_wide) static_cast<u64*>(p.d_cells)[dslot] = lin;
            else static_cast<uint32_t*>(p.d_cells)[dslot] = (uint32_t)lin;
          }
        }
        const u64 slot = warp_reserve(wo, to_s1, p.out_reserved, stamp);
        if (to_s1) {
          store_row<TOut, D>(out_rows, slot, u);
          p.out_ids[slot] = p.id_base + t * WT + sj * 32 + src;
        }
        kept += __popc(__ballot_sync(kFull, to_s1));
      }
      __syncwarp();
    }
    if (__any_sync(kFull, bad)) {  // rare: NaN/Inf (or overflow of the probe sum)
#pragma unroll
      for (int j = 0; j < PPT; ++j) {
        const bool in = full || (uint32_t)(j * 32 + lane) < n - t * WT;
        bool fin = true;
#pragma unroll
        for (int k = 0; k < D; ++k) fin &= finite_v(cur[j][k]);
        if (in && !fin) atomicMax(p.nonfinite, ~(u64)(base + j * 32));
      }
    }
  };
  uint32_t t = gw;
  if constexpr (BULK) {
    const uint32_t bar0 = smem_addr(bars), ring0 = smem_addr(rows_w);
    constexpr uint32_t kStageBytes = WT * D * (uint32_t)sizeof(TIn);
    if (lane == 0) {
#pragma unroll
      for (int i = 0; i < NST; ++i) mbar_init(bar0 + 8 * i, 1);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncwarp();
    auto issue = [&](int st, uint32_t tt) {
      if (lane == 0) {
        const uint32_t rows = tt < nfull ? WT : n - tt * WT;
        bulk_load(ring0 + st * kStageBytes, coords + (u64)tt * WT * D, rows * D * (uint32_t)sizeof(TIn), bar0 + 8 * st);
      }
    };
#pragma unroll
    for (int i = 0; i < NST; ++i)
      if (t + i * nw < ntiles) issue(i, t + i * nw);
    uint32_t phases = 0;  // bit i: the parity stage i waits for next
    int st = 0;
    while (t < ntiles) {
      mbar_wait(bar0 + 8 * st, (phases >> st) & 1u);
      phases ^= 1u << st;
      const TIn* stage = rows_w + (size_t)st * WT * D;
#pragma unroll
      for (int j = 0; j < PPT; ++j) load_row_cached<TIn, D>(stage, (u64)(j * 32 + lane), buf_a[j]);
      process(buf_a, t, stage);
      __syncwarp();
      if (t + NST * nw < ntiles) issue(st, t + NST * nw);
      t += nw;
      st = st + 1 == NST ? 0 : st + 1;
    }
  } else {
    if (t < ntiles) load_tile(buf_a, t);
    while (t < ntiles) {
      uint32_t tn = t + nw;
      if (tn < ntiles) load_tile(buf_b, tn);
      process(buf_a, t, nullptr);
      t = tn;
      if (t >= ntiles) break;
      tn = t + nw;
      if (tn < ntiles) load_tile(buf_a, tn);
      process(buf_b, t, nullptr);
      t = tn;
    }
  }
  resolve_pending();
  warp_close(wo, stamp);
  if (p.f_rows) warp_close(wd, dstamp);
  if (lane == 0 && kept) atomicAdd(p.kept, (u64)kept);
  if (p.lo_words) {
    __syncthreads();
    uint32_t* slab = p.slabs + (u64)blockIdx.x * p.lo_words;
    for (uint32_t w = threadIdx.x; w < p.lo_words; w += THREADS) slab[w] = occ_s[w];
  }
}

// OR of the per-CTA slabs: blockIdx.y picks a group of slabs, so the
// (slabs x words) reduction runs on many CTAs; one red.or per word and group.
static __global__ void k_reduce_slabs(const uint32_t* __restrict__ slabs, int nslabs, uint32_t words,
                               uint32_t* __restrict__ out) {
  pdl_enter();
  const int per = (nslabs + gridDim.y - 1) / gridDim.y;
  const int s0 = blockIdx.y * per, s1 = min(nslabs, s0 + per);
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < words; w += gridDim.x * blockDim.x) {
    uint32_t x = 0;
    for (int s = s0; s < s1; ++s) x |= slabs[(u64)s * words + w];
    if (x) atomicOr(out + w, x);
  }
}

// ------------------------------------------------- K3: cell pruning tables
// Row-min of dimension 0 (the innermost `L` bits of the linear index) fused
// with the inclusive prefix-min along dimension 1, one warp per dimension-1
// line: lane l takes rows l, l+32, .. of the line (coalesced row reads) and
// the prefix-min along the line is a warp scan per 32 rows with a carry.  A
// thread per line left the GPU nearly idle at the small tables K0 and K3
// build (4,096 lines at d=4, L=6: 24 us).
template <typename TT>
__global__ void k_rowmin_prefix1w(const uint32_t* __restrict__ bits, int L, u64 lines, TT* __restrict__ R) {
  pdl_enter();
  const int n = 1 << L;
  const int rowbits = 1 << L;
  const int lane = threadIdx.x & 31;
  for (u64 line = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; line < lines;
       line += ((u64)gridDim.x * blockDim.x) >> 5) {
    // rows of this line: the dimension-1 index is the lowest digit of the row index
    const u64 row0 = line * (u64)n;
    TT carry = (TT)~(TT)0;
    for (int c0 = 0; c0 < n; c0 += 32) {
      const int c1 = c0 + lane;
      TT best = (TT)~(TT)0;
      if (c1 < n) {
        const u64 r = row0 + c1;
        if (L >= 5) {
          const u64 wpr = (u64)rowbits >> 5;
          for (u64 w = 0; w < wpr; ++w) {
            const uint32_t x = __ldg(bits + r * wpr + w);
            if (x) {
              best = (TT)(w * 32 + __ffs(x) - 1);
              break;
            }
          }
        } else {
          const int rpw = 32 >> L;
          const uint32_t x = (__ldg(bits + r / rpw) >> ((r % rpw) * rowbits)) & ((1u << rowbits) - 1);
          if (x) best = (TT)(__ffs(x) - 1);
        }
      }
      // inclusive prefix-min over the lanes, then the carry of earlier chunks
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const TT y = __shfl_up_sync(kFull, best, o);
        if (lane >= o) best = y < best ? y : best;
      }
      best = carry < best ? carry : best;
      if (c1 < n) R[row0 + c1] = best;
      carry = __shfl_sync(kFull, best, 31);
    }
  }
}

// Row minima only, one thread per row (for grids with few dimension-1 lines,
// e.g. d = 2 at fine layers, which one CTA per line then scans).
template <typename TT>
__global__ void k_rowmin(const uint32_t* __restrict__ bits, int L, u64 rows, TT* __restrict__ R) {
  pdl_enter();
  const int rowbits = 1 << L;
  for (u64 r = blockIdx.x * (u64)blockDim.x + threadIdx.x; r < rows; r += (u64)gridDim.x * blockDim.x) {
    TT best = (TT)~(TT)0;
    if (L >= 5) {
      const u64 wpr = (u64)rowbits >> 5;
      for (u64 w = 0; w < wpr; ++w) {
        const uint32_t x = __ldg(bits + r * wpr + w);
        if (x) {
          best = (TT)(w * 32 + __ffs(x) - 1);
          break;
        }
      }
    } else {
      const int rpw = 32 >> L;
      const uint32_t x = (__ldg(bits + r / rpw) >> ((r % rpw) * rowbits)) & ((1u << rowbits) - 1);
      if (x) best = (TT)(__ffs(x) - 1);
    }
    R[r] = best;
  }
}

// Inclusive prefix-min along dimension k of the (d-1)-dim table with one CTA
// per line (few, long lines): each thread scans a contiguous run, one block
// scan of the run minima, then the runs are rewritten.
template <typename TT>
__global__ void __launch_bounds__(1024) k_prefix_min_cta(TT* __restrict__ R, int L, int k, u64 lines) {
  pdl_enter();
  __shared__ TT wmin[32];
  const u64 stride = 1ull << (L * (k - 1));
  const int n = 1 << L;
  const int per = (n + 1023) / 1024;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (u64 line = blockIdx.x; line < lines; line += gridDim.x) {
    const u64 low = line & (stride - 1);
    const u64 high = line >> (L * (k - 1));
    const u64 base = (high << (L * k)) + low;
    const int c0 = threadIdx.x * per, c1 = min(c0 + per, n);
    TT run = (TT)~(TT)0;
    for (int c = c0; c < c1; ++c) {
      const TT v = R[base + (u64)c * stride];
      run = v < run ? v : run;
    }
    // exclusive prefix-min of the run minima
    TT incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const TT y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl = y < incl ? y : incl;
    }
    if (lane == 31) wmin[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      TT t = wmin[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const TT y = __shfl_up_sync(kFull, t, o);
        if (lane >= o) t = y < t ? y : t;
      }
      wmin[lane] = t;
    }
    __syncthreads();
    TT carry = (TT)~(TT)0;
    if (warp > 0) carry = wmin[warp - 1];
    const TT prev = __shfl_up_sync(kFull, incl, 1);
    if (lane > 0) carry = prev < carry ? prev : carry;
    for (int c = c0; c < c1; ++c) {
      const TT v = R[base + (u64)c * stride];
      carry = v < carry ? v : carry;
      R[base + (u64)c * stride] = carry;
    }
    __syncthreads();
  }
}

// Inclusive prefix-min along dimension k (2..d-1) of the (d-1)-dim table.
// Loads are issued 16 at a time ahead of the dependent min-scan.
// One warp per line (grids with a few thousand lines: a thread per line
// runs 2^L dependent steps on a few threads per SM): lanes take the line's
// entries lane, lane+32, .. (strided loads, all in flight) and scan them in
// chunks of 32 with a carry.
template <typename TT>
__global__ void k_prefix_minw(TT* __restrict__ R, int L, int k, u64 lines) {
  pdl_enter();
  const u64 stride = 1ull << (L * (k - 1));
  const int n = 1 << L;
  const int lane = threadIdx.x & 31;
  for (u64 line = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; line < lines;
       line += ((u64)gridDim.x * blockDim.x) >> 5) {
    const u64 low = line & (stride - 1);
    const u64 high = line >> (L * (k - 1));
    const u64 base = (high << (L * k)) + low;
    TT carry = (TT)~(TT)0;
    for (int c0 = 0; c0 < n; c0 += 32) {
      const int c = c0 + lane;
      TT v = c < n ? R[base + (u64)c * stride] : (TT)~(TT)0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const TT y = __shfl_up_sync(kFull, v, o);
        if (lane >= o) v = y < v ? y : v;
      }
      v = carry < v ? carry : v;
      if (c < n) R[base + (u64)c * stride] = v;
      carry = __shfl_sync(kFull, v, 31);
    }
  }
}

template <typename TT>
__global__ void k_prefix_min(TT* __restrict__ R, int L, int k, u64 lines) {
  pdl_enter();
  const u64 stride = 1ull << (L * (k - 1));
  const int n = 1 << L;
  for (u64 line = blockIdx.x * (u64)blockDim.x + threadIdx.x; line < lines; line += (u64)gridDim.x * blockDim.x) {
    const u64 low = line & (stride - 1);
    const u64 high = line >> (L * (k - 1));
    const u64 base = (high << (L * k)) + low;
    TT run = (TT)~(TT)0;
    for (int c = 0; c < n; c += 16) {
      TT v[16];
      const int m = n - c < 16 ? n - c : 16;
#pragma unroll
      for (int e = 0; e < 16; ++e)
        if (e < m) v[e] = R[base + (u64)(c + e) * stride];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        if (e < m) {
          run = v[e] < run ? v[e] : run;
          R[base + (u64)(c + e) * stride] = run;
        }
      }
    }
  }
}

// Cell status from the prefix-min table PM (inclusive prefix-OR P[c] <=>
// PM[c1..] <= c0):
//   candidate  = occupied && !(all c_k >= 1 && P[c - 1])                  (Def. 5)
//   key (grid) = occupied && no top column && !OR_k (c_k >= 1 && P[c - e_k])  (Def. 4)
// Key counts add the d auxiliary cells (cell.hpp:35-40).  Checked against
// baseline.cpp:76-157 (via the oracle) by tests/test_gpu_parity.py.
// Row-parallel layer counts: one thread
// per row x = (c_1..c_{d-1}) of layer L.  With PM the prefix-min table,
//   candidate cells of the row:  c_0 <= PM[x - 1]       (all x_k >= 1; else every cell)
//   key cells (no top in x):      c_0 < min(PM[x] + 1, top, min_{x_k>=1} PM[x - e_k])
// so both are occupancy bits below a per-row threshold: d table lookups and
// a popcount per row instead of d lookups per occupied cell.
template <typename TT>
__global__ void k_count_rows(const uint32_t* __restrict__ bits, int L, int d, u64 rows, const TT* __restrict__ PM,
                             u64* cand_out, u64* key_out) {
  pdl_enter();
  const int n0 = 1 << L, top = n0 - 1;
  const u64 mask = (u64)top;
  const TT none = (TT)~(TT)0;
  u64 nc = 0, nk = 0;
  for (u64 r = blockIdx.x * (u64)blockDim.x + threadIdx.x; r < rows; r += (u64)gridDim.x * blockDim.x) {
    bool all_pos = true, has_top = false;
    u64 dm1 = 0;  // sum of the per-dimension strides (row index of x - 1)
    for (int k = 1; k < d; ++k) {
      const u64 xk = (r >> (L * (k - 1))) & mask;
      all_pos &= xk >= 1;
      has_top |= xk == (u64)top;
      dm1 += 1ull << (L * (k - 1));
    }
    int tc = top;  // candidate cells: c_0 <= tc
    if (all_pos) {
      const TT v = __ldg(PM + (r - dm1));
      tc = v == none ? top : min((int)v, top);
      // PM[x - 1] <= c_0 - 1 means strictly dominated: candidates are c_0 <= PM
    }
    int tk = -1;  // key cells: c_0 <= tk
    if (!has_top) {
      const TT v0 = __ldg(PM + r);
      int t = v0 == none ? top : min((int)v0 + 1, top);  // c_0 < PM[x] + 1 and c_0 < top
      for (int k = 1; k < d; ++k) {
        if (((r >> (L * (k - 1))) & mask) == 0) continue;
        const TT v = __ldg(PM + (r - (1ull << (L * (k - 1)))));
        if (v != none) t = min(t, (int)v);
      }
      tk = t - 1;
    }
    // count occupied c_0 <= threshold in the row
    auto count_le = [&](int thr) -> u64 {
      if (thr < 0) return 0;
      if (L >= 5) {
        const u64 wpr = (u64)n0 >> 5;
        u64 c = 0;
        for (u64 w = 0; w < wpr; ++w) {
          const int base = (int)(w * 32);
          if (base > thr) break;
          uint32_t x = __ldg(bits + r * wpr + w);
          if (thr - base < 31) x &= (2u << (thr - base)) - 1;
          c += __popc(x);
        }
        return c;
      }
      const u64 bit0 = r * (u64)n0;
      uint32_t x = (__ldg(bits + (bit0 >> 5)) >> (bit0 & 31)) & ((1u << n0) - 1);
      if (thr < top) x &= (2u << thr) - 1;
      return __popc(x);
    };
    nc += count_le(tc);
    nk += count_le(tk);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    nc += __shfl_xor_sync(kFull, nc, o);
    nk += __shfl_xor_sync(kFull, nk, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (nc) atomicAdd(cand_out, nc);
    if (nk) atomicAdd(key_out, nk);
  }
}

// Word-parallel child-OR for coarse layers L >= 5 (a coarse row spans whole
// words): coarse word w covers c_0 in [32q, 32q + 32) of row x; its children
// are the 64 fine bits [64q, 64q + 64) of the 2^(d-1) fine rows (2x_k + b_k).
// OR them, fold bit pairs, gather the even bits: one 32-bit word, no atomics.
static __global__ void k_downsample_words(const uint32_t* __restrict__ src, int L, int d, u64 dst_words,
                                   uint32_t* __restrict__ dst) {
  pdl_enter();
  const u64 wpr = (1ull << L) >> 5, wpr_f = wpr * 2;
  const u64 mask = (1ull << L) - 1;
  for (u64 w = blockIdx.x * (u64)blockDim.x + threadIdx.x; w < dst_words; w += (u64)gridDim.x * blockDim.x) {
    const u64 r = w / wpr, q = w % wpr;
    u64 acc = 0;
    const int nchild = 1 << (d - 1);
    for (int b = 0; b < nchild; ++b) {
      u64 R = 0;
      for (int k = d - 1; k >= 1; --k) {
        const u64 xk = (r >> (L * (k - 1))) & mask;
        R = (R << (L + 1)) | (2 * xk + ((b >> (k - 1)) & 1));
      }
      const u64 fw = R * wpr_f + 2 * q;
      acc |= (u64)__ldg(src + fw) | ((u64)__ldg(src + fw + 1) << 32);
    }
    u64 x = (acc | (acc >> 1)) & 0x5555555555555555ull;
    x = (x | (x >> 1)) & 0x3333333333333333ull;
    x = (x | (x >> 2)) & 0x0f0f0f0f0f0f0f0full;
    x = (x | (x >> 4)) & 0x00ff00ff00ff00ffull;
    x = (x | (x >> 8)) & 0x0000ffff0000ffffull;
    x = (x | (x >> 16)) & 0x00000000ffffffffull;
    dst[w] |= (uint32_t)x;
  }
}

// Occupancy of layer L from layer L+1 (grid.cpp:80-102, child-OR), OR-ed into dst.
static __global__ void k_downsample(const uint32_t* __restrict__ src, int L, int d, u64 src_words,
                             uint32_t* __restrict__ dst) {
  pdl_enter();
  const u64 mask = (1ull << (L + 1)) - 1;
  for (u64 w = blockIdx.x * (u64)blockDim.x + threadIdx.x; w < src_words; w += (u64)gridDim.x * blockDim.x) {
    uint32_t x = src[w];
    while (x) {
      const int b = __ffs(x) - 1;
      x &= x - 1;
      const u64 lin = w * 32 + b;
      u64 out = 0;
      for (int k = d - 1; k >= 0; --k) out = (out << L) | (((lin >> ((L + 1) * k)) & mask) >> 1);
      set_bit_global(dst, out);
    }
  }
}

// ------------------------------------------------- per-dimension lists
// Dominance pruning index: for every dimension k, the points of a set ordered
// by their column at a fixed fine level (kListLevel), with column starts.  A
// dominator q of p satisfies q_k <= p_k, hence col(q_k) <= col(p_k) (floor of
// a power-of-two scaling is monotone), so the candidates for p are a prefix of
// each list and the shortest of the d prefixes suffices.  Near-face points --
// the hard cases of independent/correlated data -- have one tiny coordinate
// and therefore a tiny prefix.
constexpr int kListLevel = 10;
constexpr int kListCols = 1 << kListLevel;
// Point-set lists additionally order each column by FP64 sum (64 buckets over
// [0, d)), so the strongest candidate dominators of a column come first.
constexpr int kSumBuckets = 64;
constexpr int kListBins = kListCols * kSumBuckets;
__device__ __forceinline__ int list_col(float v) { return cell_col(v, (float)kListCols, kListCols - 1); }
__device__ __forceinline__ int list_col(double v) { return cell_col(v, (double)kListCols, kListCols - 1); }

// ------------------------------------------------ K4: candidate-cell filter
// Survivors of the stream that lie in layer-rho candidate cells (refine.cpp:
// 78-96; their count is points_examined), minus those a filter point f
// (a real record, e.g. from the sample skyline) dominates with a strictly
// smaller FP64 sum.  That removal is exact for the reference's sort-first
// semantics: FP64 sums are monotone, so any chain of strictly dominating
// cells from f down to a candidate cell keeps a strictly smaller sum, and the
// reference drops p in phase 2 (refine.cpp:98-99).  Output keeps input order.
struct CandParams {
  const void* rows;
  const uint32_t* ids;    // kNoId marks an empty slot
  const u64* count;       // slots to scan (device), or nullptr to use count_const
  u64 count_const;
  int rho;
  const void* PM;        // layer-rho prefix-min table (u8 or u32), nullptr: no cell test
  const void* f_rows;    // filter points (strength order), may be empty
  const u64* f_fsum;
  const u64* f_count;
  uint32_t f_max;
  const uint16_t* f_lists;  // D x f_max filter indices, column-ordered per dimension
  const uint16_t* f_offs;   // D x (kListCols + 1) column starts
  void* out_rows;
  uint32_t* out_ids;
  u64* out_fsum;
  u64* out_reserved;
  unsigned chunk;        // output chunk per warp reservation
  u64* kept;             // exact number of points written
  u64* examined;         // points_examined (refine.cpp:90-96), may be null
  const void* d_cells;   // K1's D stream (cells of survivors a filter point removed), may be null
  const u64* d_count;
  int d_wide;
  uint32_t head_start;   // first filter point of the branch-free head
  int coop;              // run the warp-cooperative phase for points the head leaves
  uint32_t coop_mid;     // K4b: filter points after the head tested branch-free before the list scan
  // K4a: when *gate != 0 (k_filter_gate) the survivors go to the alt_*
  // stream (S2) instead of out_* (the K4b input)
  const u64* gate;
  void* alt_rows;
  uint32_t* alt_ids;
  u64* alt_fsum;
  u64* alt_reserved;
  u64* alt_kept;
};

template <typename T, int D, typename TT, int THREADS>
__global__ void __launch_bounds__(THREADS) k_candidates(CandParams p) {
  pdl_enter();
  extern __shared__ __align__(16) uint8_t smc[];
  const u64 n = p.count ? *p.count : p.count_const;
  uint32_t nf = 0;
  const uint32_t fm = p.f_max;
  T* f_rows = reinterpret_cast<T*>(smc);
  u64* f_sum = reinterpret_cast<u64*>(smc + (((u64)fm * D * sizeof(T) + 15) & ~15ull));
  uint16_t* f_list = reinterpret_cast<uint16_t*>(f_sum + fm);           // D x fm
  uint16_t* f_off = f_list + (u64)D * fm;                              // D x (kListCols + 1)
  if (p.f_count) {
    const u64 fc = *p.f_count;
    nf = (uint32_t)(fc < fm ? fc : fm);
    const T* fr = static_cast<const T*>(p.f_rows);
    for (uint32_t e = threadIdx.x; e < nf * D; e += THREADS) f_rows[e] = fr[e];
    for (uint32_t e = threadIdx.x; e < nf; e += THREADS) f_sum[e] = p.f_fsum[e];
    for (uint32_t e = threadIdx.x; e < (uint32_t)D * fm; e += THREADS) f_list[e] = p.f_lists[e];
    for (uint32_t e = threadIdx.x; e < (uint32_t)D * (kListCols + 1); e += THREADS) f_off[e] = p.f_offs[e];
  }
  __syncthreads();
  const T* rows = static_cast<const T*>(p.rows);
  T* out_rows = static_cast<T*>(p.out_rows);
  const TT* PM = static_cast<const TT*>(p.PM);
  const int rho = p.rho, top = (1 << rho) - 1;
  const float fscale = ldexpf(1.0f, rho);
  const double dscale = ldexp(1.0, rho);
  const u64 gw = (blockIdx.x * (u64)THREADS + threadIdx.x) >> 5;
  const u64 nw = ((u64)gridDim.x * THREADS) >> 5;
  const int lane = threadIdx.x & 31;
  WarpOut wo{0, p.chunk, p.chunk};
  auto stamp = [&](u64 slot) { p.out_ids[slot] = kNoId; };
  u64 examined = 0, kept = 0;
  for (u64 wbase = gw * 32; wbase < n; wbase += nw * 32) {
    const u64 i = wbase + lane;
    bool keep = false;
    T v[D];
#pragma unroll
    for (int k = 0; k < D; ++k) v[k] = (T)2;  // empty slot: dominated by nothing that matters (keep = false)
    u64 ps = 0;
    uint32_t pid = kNoId;
    if (i < n) pid = p.ids[i];
    if (pid != kNoId) {
      load_row_cached<T, D>(rows, i, v);
      bool cand = true;
      if (PM) {
        int col[D];
#pragma unroll
        for (int k = 0; k < D; ++k) {
          if constexpr (sizeof(T) == 4) col[k] = cell_col(v[k], fscale, top);
          else col[k] = cell_col(v[k], dscale, top);
        }
        cand = !strictly_dominated_cols<TT, D>(PM, col, rho);
      }
      examined += cand;
      ps = fsum_bits<T, D>(v);
      keep = cand;
    }
    // Strongest filter points first (strength order): the first 8 remove
    // ~87% of the candidates at the headline config, tested branch-free by
    // every lane.
    constexpr uint32_t kHead0 = 8;
    const uint32_t hs = p.head_start;
    if (nf > hs) {
      const uint32_t h0 = nf - hs < kHead0 ? nf - hs : kHead0;
      bool dom = false;
#pragma unroll
      for (uint32_t f = 0; f < kHead0; ++f)
        if (f < h0) dom |= dominates<T, D>(f_rows + (u64)(hs + f) * D, v) && f_sum[hs + f] < ps;
      keep = keep && !dom;
    }
    // The rest, one pending point at a time with the whole warp: first the
    // next 32 strongest filter points (one per lane), then the point's
    // shortest column prefix of F, 32 entries per step (a dominator f has
    // col_k(f) <= col_k(p) in every dimension).  A per-lane loop here ran
    // with ~5 of 32 lanes active (ncu: 68% of K4's instructions).
    // K4b (coop): its lanes are dense pending points, so the next 32 filter
    // points are tested branch-free by every lane (one step per filter point
    // for the whole warp, instead of one warp step per pending point)
    const uint32_t mid = p.coop_mid;
    if (p.coop && mid && nf > hs + kHead0 && __any_sync(kFull, keep)) {
      bool dom = false;
#pragma unroll 8
      for (uint32_t f = hs + kHead0; f < hs + kHead0 + mid; ++f)
        if (f < nf) dom |= dominates<T, D>(f_rows + (u64)f * D, v) && f_sum[f] < ps;
      keep = keep && !dom;
    }
    unsigned pend = __ballot_sync(kFull, p.coop && keep && nf > hs + kHead0 + mid);
    while (pend) {
      const int src = __ffs(pend) - 1;
      pend &= pend - 1;
      T pv[D];
#pragma unroll
      for (int k = 0; k < D; ++k) pv[k] = __shfl_sync(kFull, v[k], src);
      const u64 pps = __shfl_sync(kFull, ps, src);
      bool found = false;
      int bk = 0;
      unsigned end = 0xffffffffu;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const unsigned e = f_off[k * (kListCols + 1) + list_col(pv[k]) + 1];
        if (e < end) { end = e; bk = k; }
      }
      const uint16_t* lst = f_list + (u64)bk * fm;
      // at most kFSteps steps: a point the filter cannot settle quickly is
      // left to K5 (anti-correlated data: long prefixes, few kills)
      constexpr unsigned kFSteps = 8;
      if (end > kFSteps * 32) end = kFSteps * 32;
      for (unsigned base = 0; base < end && !found; base += 32) {
        const unsigned e = base + lane;
        bool d_l = false;
        if (e < end) {
          const unsigned f = lst[e];
          d_l = f_sum[f] < pps && dominates<T, D>(f_rows + (u64)f * D, pv);
        }
        found = __any_sync(kFull, d_l);
      }
      if (found && lane == src) keep = false;
    }
    kept += keep;
    if (__any_sync(kFull, keep)) {
      const u64 o = warp_reserve(wo, keep, p.out_reserved, stamp);
      if (keep) {
        store_row<T, D>(out_rows, o, v);
        p.out_ids[o] = pid;
        p.out_fsum[o] = ps;
      }
    }
  }
  warp_close(wo, stamp);
  // points K1 already removed (filter-point head) still count in
  // points_examined when their cell is a candidate
  if (p.d_cells && PM) {
    const u64 nd = *p.d_count;
    const u64 cmask = (1ull << rho) - 1;
    for (u64 e = blockIdx.x * (u64)THREADS + threadIdx.x; e < nd; e += (u64)gridDim.x * THREADS) {
      const u64 lin = p.d_wide ? static_cast<const u64*>(p.d_cells)[e]
                               : (u64) static_cast<const uint32_t*>(p.d_cells)[e];
      if (p.d_wide ? lin == ~0ull : lin == 0xffffffffull) continue;
      int col[D];
#pragma unroll
      for (int k = 0; k < D; ++k) col[k] = (int)((lin >> (rho * k)) & cmask);
      examined += !strictly_dominated_cols<TT, D>(PM, col, rho);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    examined += __shfl_xor_sync(kFull, examined, o);
    kept += __shfl_xor_sync(kFull, kept, o);
  }
  if (lane == 0) {
    if (p.examined && examined) atomicAdd(p.examined, examined);
    if (kept) atomicAdd(p.kept, kept);
  }
}

// K4a: the candidate-cell test over S1, then the branch-free head of the 8
// strongest filter points on FULL batches: candidates (about half of S1 at
// the headline config) are queued per warp in a 64-entry shared ring and
// tested 32 at a time, so no lane of the head test idles on a non-candidate.
// Points still pending go to the dense stream P (K4b finishes them).
// filter points in K4a's branch-free head (K4b starts after them)
constexpr uint32_t kK4aHead = SKY_K4A_HEAD;

template <typename T, int D, typename TT, int THREADS>
__global__ void __launch_bounds__(THREADS) k_cand_head(CandParams p) {
  pdl_enter();
  extern __shared__ __align__(16) uint8_t smc[];
  constexpr int kRing = 64;
  constexpr uint32_t kHead0 = kK4aHead;
  const u64 n = *p.count;
  const uint32_t nh = (uint32_t)(*p.f_count < kHead0 ? *p.f_count : kHead0);
  T* f_rows = reinterpret_cast<T*>(smc);                                  // kHead0 x D
  u64* f_sum = reinterpret_cast<u64*>(smc + ((kHead0 * D * sizeof(T) + 15) & ~(size_t)15));
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring_base = smc + ((kHead0 * D * sizeof(T) + 15) & ~(size_t)15) + kHead0 * 8;
  T* r_rows = reinterpret_cast<T*>(ring_base) + (size_t)wib * kRing * D;
  u64* r_sum = reinterpret_cast<u64*>(ring_base + (size_t)(THREADS / 32) * kRing * D * sizeof(T)) + (size_t)wib * kRing;
  uint32_t* r_ids = reinterpret_cast<uint32_t*>(ring_base + (size_t)(THREADS / 32) * kRing * (D * sizeof(T) + 8)) +
                    (size_t)wib * kRing;
  {
    const T* fr = static_cast<const T*>(p.f_rows);
    for (uint32_t e = threadIdx.x; e < nh * D; e += THREADS) f_rows[e] = fr[e];
    for (uint32_t e = threadIdx.x; e < nh; e += THREADS) f_sum[e] = p.f_fsum[e];
  }
  __syncthreads();
  const T* rows = static_cast<const T*>(p.rows);
  const bool alt = p.gate && *p.gate;
  T* out_rows = static_cast<T*>(alt ? p.alt_rows : p.out_rows);
  uint32_t* out_ids = alt ? p.alt_ids : p.out_ids;
  u64* out_fsum = alt ? p.alt_fsum : p.out_fsum;
  u64* out_reserved = alt ? p.alt_reserved : p.out_reserved;
  u64* out_kept = alt ? p.alt_kept : p.kept;
  const TT* PM = static_cast<const TT*>(p.PM);
  const int rho = p.rho, top = (1 << rho) - 1;
  const float fscale = ldexpf(1.0f, rho);
  const double dscale = ldexp(1.0, rho);
  const u64 gw = (blockIdx.x * (u64)THREADS + threadIdx.x) >> 5;
  const u64 nw = ((u64)gridDim.x * THREADS) >> 5;
  const unsigned lt = (1u << lane) - 1;
  WarpOut wo{0, p.chunk, p.chunk};
  auto stamp = [&](u64 slot) { out_ids[slot] = kNoId; };
  u64 examined = 0, kept = 0;
  unsigned head = 0, tail = 0;  // ring positions (warp-uniform)
  // head-8 test of up to 32 queued candidates; survivors -> P
  auto drain = [&](unsigned cnt) {
    const bool act = (unsigned)lane < cnt;
    const unsigned e = (head + lane) % kRing;
    T v[D];
#pragma unroll
    for (int k = 0; k < D; ++k) v[k] = (T)2;
    u64 ps = 0;
    uint32_t pid = kNoId;
    if (act) {
      load_row_cached<T, D>(r_rows, e, v);
      ps = r_sum[e];
      pid = r_ids[e];
    }
    bool dom = false;
#pragma unroll
    for (uint32_t f = 0; f < kHead0; ++f)
      if (f < nh) dom |= dominates<T, D>(f_rows + (u64)f * D, v) && f_sum[f] < ps;
    const bool keep = act && !dom;
    kept += keep;
    if (__any_sync(kFull, keep)) {
      const u64 o = warp_reserve(wo, keep, out_reserved, stamp);
      if (keep) {
        store_row<T, D>(out_rows, o, v);
        out_ids[o] = pid;
        out_fsum[o] = ps;
      }
    }
    head += cnt;
    __syncwarp();
  };
  // the next batch's id and row are loaded while this one is processed (the
  // row load does not wait for the id: slots of kNoId hold don't-care rows)
  uint32_t pid_n = kNoId;
  T v_n[D];
  auto fetch = [&](u64 wb) {
    const u64 i = wb + lane;
    pid_n = kNoId;
    if (i < n) {
      pid_n = p.ids[i];
      load_row_cached<T, D>(rows, i, v_n);
    }
  };
  if (gw * 32 < n) fetch(gw * 32);
  for (u64 wbase = gw * 32; wbase < n; wbase += nw * 32) {
    const uint32_t pid = pid_n;
    T v[D];
#pragma unroll
    for (int k = 0; k < D; ++k) v[k] = v_n[k];
    if (wbase + nw * 32 < n) fetch(wbase + nw * 32);
    bool cand = false;
    if (pid != kNoId) {
      int col[D];
#pragma unroll
      for (int k = 0; k < D; ++k) {
        if constexpr (sizeof(T) == 4) col[k] = cell_col(v[k], fscale, top);
        else col[k] = cell_col(v[k], dscale, top);
      }
      cand = !strictly_dominated_cols<TT, D>(PM, col, rho);
      examined += cand;
    }
    const unsigned m = __ballot_sync(kFull, cand);
    if (cand) {
      const unsigned e = (tail + __popc(m & lt)) % kRing;
      store_row<T, D>(r_rows, e, v);
      r_sum[e] = fsum_bits<T, D>(v);
      r_ids[e] = pid;
    }
    tail += __popc(m);
    __syncwarp();
    if (tail - head >= 32) drain(32);
  }
  if (tail != head) drain(tail - head);
  warp_close(wo, stamp);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    examined += __shfl_xor_sync(kFull, examined, o);
    kept += __shfl_xor_sync(kFull, kept, o);
  }
  if (lane == 0) {
    if (p.examined && examined) atomicAdd(p.examined, examined);
    if (kept) atomicAdd(out_kept, kept);
  }
}

// Compact the members (flag set, id != kNoId) of a slot array: rows and sums.
template <typename T, int D>
__global__ void k_compact_members(const T* __restrict__ rows, const uint32_t* __restrict__ ids,
                                  const uint8_t* __restrict__ flag, const u64* __restrict__ fsum,
                                  const u64* __restrict__ count, T* __restrict__ out_rows, u64* __restrict__ out_fsum,
                                  u64* __restrict__ out_count) {
  pdl_enter();
  const u64 n = *count;
  const int lane = threadIdx.x & 31;
  for (u64 wb = ((blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5) * 32; wb < n;
       wb += ((u64)gridDim.x * blockDim.x >> 5) * 32) {
    const u64 i = wb + lane;
    const bool live = i < n && ids[i] != kNoId && (!flag || flag[i]);  // flag == nullptr: every member
    const unsigned m = __ballot_sync(kFull, live);
    if (!m) continue;
    u64 b = 0;
    if (lane == 0) b = atomicAdd(out_count, (u64)__popc(m));
    b = __shfl_sync(kFull, b, 0);
    if (live) {
      const u64 o = b + __popc(m & ((1u << lane) - 1));
      T v[D];
      load_row_cached<T, D>(rows, i, v);
      store_row<T, D>(out_rows, o, v);
      out_fsum[o] = fsum[i];
    }
  }
}

// Single CTA: order a point set by descending "strength" -- the volume it
// dominates in the unit cube, prod(1 - u_k) -- in 64 log-spaced buckets, and
// keep the first f_max.  Strong filter points first make K4's early exit
// happen after ~1 test for most points.
template <typename T, int D>
__global__ void __launch_bounds__(1024) k_strength_order(const T* __restrict__ rows, const u64* __restrict__ fsum,
                                                          const uint32_t* __restrict__ ids, const u64* __restrict__ count,
                                                          uint32_t f_max, T* __restrict__ out_rows,
                                                          u64* __restrict__ out_fsum, uint32_t* __restrict__ out_ids,
                                                          u64* __restrict__ out_count) {
  pdl_enter();
  // ids (optional): empty slots (kNoId) are skipped; out_ids (optional)
  __shared__ unsigned hist[65];
  __shared__ unsigned offs[65];
  const u64 n = *count;
  if (threadIdx.x < 65) hist[threadIdx.x] = 0;
  __syncthreads();
  auto bucket = [&](u64 i) {
    if (ids && ids[i] == kNoId) return 64;
    double vol = 1.0;
#pragma unroll
    for (int k = 0; k < D; ++k) vol *= 1.0 - true_value(rows[i * D + k]);
    const double l = vol > 0 ? -log2(vol) * 2.0 : 1e9;
    return (int)(l < 63.0 ? l : 63.0);
  };
  for (u64 i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(&hist[bucket(i)], 1u);
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned run = 0;
    for (int b = 0; b < 64; ++b) {
      offs[b] = run;
      run += hist[b];
    }
    *out_count = run < f_max ? run : f_max;
  }
  __syncthreads();
  for (u64 i = threadIdx.x; i < n; i += blockDim.x) {
    const int bk = bucket(i);
    if (bk == 64) continue;
    const unsigned o = atomicAdd(&offs[bk], 1u);
    if (o < f_max) {
#pragma unroll
      for (int k = 0; k < D; ++k) out_rows[(u64)o * D + k] = rows[i * D + k];
      out_fsum[o] = fsum[i];
      if (out_ids) out_ids[o] = ids ? ids[i] : (uint32_t)i;
    }
  }
}

// One CTA per dimension k: the filter points' stable column order in
// dimension k (key = column << 10 | strength rank, one block radix sort), so
// each column prefix is scanned strongest first, plus the column starts.
template <typename T, int D>
__global__ void __launch_bounds__(256) k_filter_lists(const T* __restrict__ f_rows, const u64* __restrict__ f_count,
                                                       uint32_t f_max, uint16_t* __restrict__ f_lists,
                                                       uint16_t* __restrict__ f_offs) {
  pdl_enter();
  // 256 threads x 4 keys (small CTAs: this also runs beside K1, K0's chain)
  constexpr int kPer = 4;
  using Sort = cub::BlockRadixSort<uint32_t, 256, kPer>;
  __shared__ typename Sort::TempStorage tmp;
  __shared__ unsigned cnt[kListCols + 1];
  const int k = blockIdx.x;
  const unsigned nf = (unsigned)(*f_count < f_max ? *f_count : f_max);  // f_max <= 1024
  const unsigned t = threadIdx.x;
  for (unsigned c = t; c <= kListCols; c += blockDim.x) cnt[c] = 0;
  __syncthreads();
  uint32_t key[kPer];
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const unsigned r = t * kPer + j;
    key[j] = r < nf ? ((uint32_t)list_col(f_rows[(u64)r * D + k]) << 10) | r : 0xffffffffu;
    if (r < nf) atomicAdd(&cnt[(key[j] >> 10) + 1], 1u);
  }
  Sort(tmp).Sort(key, 0, 20);
#pragma unroll
  for (int j = 0; j < kPer; ++j) {  // blocked arrangement: thread t holds ranks t*kPer + j
    const unsigned r = t * kPer + j;
    if (r < nf) f_lists[(u64)k * f_max + r] = (uint16_t)(key[j] & 1023);
  }
  __syncthreads();
  if (t == 0) {
    unsigned run = 0;
    for (int c = 0; c <= kListCols; ++c) {
      run += cnt[c];
      f_offs[k * (kListCols + 1) + c] = (uint16_t)run;  // points with column < c
    }
  }
}

// ------------------------------------------- K5: exact sort-first dominance
// Per-dimension candidate lists of a point set with a device-side count.
// For every dimension k the slots are counting-sorted by the bin
// (column c, sum bucket b) in column-major order, so the candidate
// dominators of p in dimension k -- col_k(q) <= col_k(p) and bucket(q) <=
// bucket(p) (sums are monotone under dominance) -- form one contiguous range
// per column, visited in ascending column order.  A per-dimension column
// histogram picks the dimension with the fewest candidates.  Layout per
// dimension:
//   [0, kListBins]                          shifted bin counts -> bin starts
//   [kListBins + 1, kListBins + kListCols + 1]  shifted column counts -> cumulative
// Order inside a bin only affects how soon a dominator is met, never the result.
constexpr int kColBase = kListBins + 1;
constexpr int kListStride = kListBins + 1 + kListCols + 1;

template <int D>
__device__ __forceinline__ int sum_bucket(u64 fsum_bits) {
  const double f = __longlong_as_double((long long)fsum_bits);
  if (!(f > 0.0)) return 0;  // also NaN sums of non-finite records (reported separately)
  const int b = (int)(f * (kSumBuckets / (double)D));
  return b < kSumBuckets - 1 ? b : kSumBuckets - 1;
}

__device__ __forceinline__ int list_bin(int b, int c) { return c * kSumBuckets + b; }

template <typename T, int D>
__global__ void k_list_hist(const T* __restrict__ rows, const uint32_t* __restrict__ ids, const u64* __restrict__ fsum,
                            const u64* __restrict__ count, unsigned* __restrict__ hist) {
  pdl_enter();
  const u64 n = *count;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    if (ids[i] == kNoId) continue;
    T v[D];
    load_row_cached<T, D>(rows, i, v);
    const int sb = sum_bucket<D>(fsum[i]);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const int c = list_col(v[k]);
      atomicAdd(&hist[k * kListStride + list_bin(sb, c) + 1], 1u);
    }
  }
}

// Inclusive scan of the shifted histograms = starts, in two multi-CTA
// passes: blockIdx.y < D are the bin arrays (also copied to the scatter
// cursor), blockIdx.y >= D the column arrays; blockIdx.x is a chunk of
// kScanChunk entries.  Pass 1 writes each chunk's total; pass 2 adds the
// totals of the preceding chunks (at most a handful) to its block scan.
constexpr int kScanThreads = 256;  // small CTAs: these also run beside K1 (K0's chain)
constexpr int kScanChunk = 2048;  // 8.4 KB of shared memory: fits beside K1
constexpr int kScanPer = kScanChunk / kScanThreads;
constexpr int kScanWarps = kScanThreads / 32;
constexpr int kScanChunks = (kListBins + 1 + kScanChunk - 1) / kScanChunk;

__device__ __forceinline__ unsigned* scan_array(unsigned* hist, int y, int D, int* len) {
  const bool bins = y < D;
  *len = bins ? kListBins + 1 : kListCols + 1;
  return hist + (u64)(bins ? y : y - D) * kListStride + (bins ? 0 : kColBase);
}

static __global__ void __launch_bounds__(kScanThreads) k_list_scan_sums(unsigned* __restrict__ hist, int D,
                                                          unsigned* __restrict__ totals, const u64* __restrict__ gate) {
  pdl_enter();
  __shared__ unsigned warp_tot[kScanWarps];
  if (gate && *gate == 0) return;  // the set goes to the tree (run_dominance)
  int len;
  const unsigned* h = scan_array(hist, blockIdx.y, D, &len);
  const int c0 = blockIdx.x * kScanChunk;
  unsigned v = 0;
  for (int i = c0 + threadIdx.x; i < min(c0 + kScanChunk, len); i += kScanThreads) v += h[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  if ((threadIdx.x & 31) == 0) warp_tot[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    unsigned t = threadIdx.x < kScanWarps ? warp_tot[threadIdx.x] : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(kFull, t, o);
    if (threadIdx.x == 0) totals[blockIdx.y * kScanChunks + blockIdx.x] = t;
  }
}

static __global__ void __launch_bounds__(kScanThreads) k_list_scan(unsigned* __restrict__ hist, unsigned* __restrict__ cursor, int D,
                                                     const unsigned* __restrict__ totals, const u64* __restrict__ gate) {
  pdl_enter();
  __shared__ unsigned tile[kScanChunk + kScanChunk / 32];  // one pad word per 32 entries
  __shared__ unsigned warp_tot[kScanWarps];
  if (gate && *gate == 0) return;
  int len;
  unsigned* h = scan_array(hist, blockIdx.y, D, &len);
  unsigned* cur = (int)blockIdx.y < D ? cursor + (u64)blockIdx.y * kListStride : nullptr;
  const int c0 = blockIdx.x * kScanChunk;
  if (c0 >= len) return;
  unsigned carry = 0;
  for (int b = 0; b < (int)blockIdx.x; ++b) carry += totals[blockIdx.y * kScanChunks + b];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  auto pad = [](int i) { return i + (i >> 5); };  // conflict-free strided runs
  for (int i = threadIdx.x; i < kScanChunk; i += kScanThreads) tile[pad(i)] = (c0 + i < len) ? h[c0 + i] : 0u;
  __syncthreads();
  const int r0 = threadIdx.x * kScanPer;
  unsigned run = 0;
#pragma unroll 8
  for (int e = 0; e < kScanPer; ++e) run += tile[pad(r0 + e)];
  unsigned incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const unsigned t = lane < kScanWarps ? warp_tot[lane] : 0u;
    unsigned ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(kFull, ti, o);
      if (lane >= o) ti += y;
    }
    if (lane < kScanWarps) warp_tot[lane] = ti - t;
  }
  __syncthreads();
  unsigned acc = carry + warp_tot[warp] + incl - run;
#pragma unroll 8
  for (int e = 0; e < kScanPer; ++e) {
    acc += tile[pad(r0 + e)];
    tile[pad(r0 + e)] = acc;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kScanChunk; i += kScanThreads) {
    if (c0 + i < len) {
      const unsigned v = tile[pad(i)];
      h[c0 + i] = v;
      if (cur) cur[c0 + i] = v;
    }
  }
}

// The lists hold the entries themselves (row, FP64 sum bits, id; one
// structure-of-arrays copy per dimension), so a list scan step is one
// coalesced read of consecutive entries instead of an index load followed by
// a gather of random slots (two dependent L2 round trips per step).
template <typename T, int D>
struct ListArrays {
  T* rows;         // [D][lcap][D]
  u64* sums;       // [D][lcap]
  uint32_t* ids;   // [D][lcap]
  u64 lcap;
};

template <typename T, int D>
__global__ void k_list_scatter(const T* __restrict__ rows, const uint32_t* __restrict__ ids,
                               const u64* __restrict__ fsum, const u64* __restrict__ count,
                               unsigned* __restrict__ cursor, ListArrays<T, D> la) {
  pdl_enter();
  const u64 n = *count;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const uint32_t id = ids[i];
    if (id == kNoId) continue;
    T v[D];
    load_row_cached<T, D>(rows, i, v);
    const u64 fs = fsum[i];
    const int sb = sum_bucket<D>(fs);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const unsigned pos = atomicAdd(&cursor[k * kListStride + list_bin(sb, list_col(v[k]))], 1u);
      const u64 e = (u64)k * la.lcap + pos;
      store_row<T, D>(la.rows, e, v);
      la.sums[e] = fs;
      la.ids[e] = id;
    }
  }
}

template <typename T, int D>
__device__ __forceinline__ bool same_cell(const T* q, const T* p, int L, int top) {
  const T scale = (T)(1u << L);
  bool eq = true;
#pragma unroll
  for (int k = 0; k < D; ++k) eq &= cell_col(q[k], scale, top) == cell_col(p[k], scale, top);
  return eq;
}

// Query setup shared by both K5 list phases: the dimension with the
// shortest candidate prefix, p's column there and its sum bucket.
template <typename T, int D>
struct ListQuery {
  T v[D];
  u64 ps;
  uint32_t pid;
  int bk, pc, sb;
  __device__ __forceinline__ void init(const T* __restrict__ rows, const u64* __restrict__ fsum,
                                       const uint32_t* __restrict__ ids, const unsigned* __restrict__ offs, u64 i) {
    pid = ids[i];
    ps = fsum[i];
    load_row_cached<T, D>(rows, i, v);
    bk = 0;
    pc = 0;
    unsigned best = 0xffffffffu;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const int c = list_col(v[k]);
      const unsigned e = __ldg(offs + k * kListStride + list_bin(0, c + 1));  // entries with col <= c (column-major bins)
      if (e < best) {
        best = e;
        bk = k;
        pc = c;
      }
    }
    sb = sum_bucket<D>(ps);
  }
  // one list entry, loaded with a single round trip (row, sum, id independent)
  struct Cand {
    T w[D];
    u64 qs;
    uint32_t qi;
  };
  __device__ __forceinline__ void fetch(const ListArrays<T, D>& la, u64 base, unsigned e, bool ok, Cand& c) const {
    if (ok) {
      load_row_cached<T, D>(la.rows, base + e, c.w);
      c.qs = __ldg(la.sums + base + e);
      c.qi = __ldg(la.ids + base + e);
    } else {
      c.qi = kNoId;
      c.qs = ~0ull;
    }
  }
  // q precedes and dominates p
  __device__ __forceinline__ bool check(const Cand& c, int cell_level, int ctop) const {
    bool d = c.qi != kNoId && precedes(c.qs, c.qi, ps, pid) && dominates<T, D>(c.w, v);
    // merge_cross_cell = false (refine.cpp:98): phase-1 semantics only, a
    // dominator must share p's layer-rho cell
    if (cell_level && d) d = same_cell<T, D>(c.w, v, cell_level, ctop);
    return d;
  }
};

// flag[i] = 1 iff no point q of the set precedes i (sort-first order,
// refine.cpp:38-41) and dominates it, for query slots [q_begin, *q_end).
// Phase A, one warp per point: per column of its shortest prefix, the 32
// lanes test 32 candidates per step (independent gathers in flight) and stop
// at the first step with a dominator.  A point still undecided after
// max_steps steps -- in practice a skyline point with a long prefix, which
// has no early exit -- is queued for phase B (k_allpairs_long) instead of
// holding its warp for the whole scan: the static warp schedule otherwise
// ends with a tail of a few long scans (ncu: 15% of warps active).
// A point with sum 0 lies at the origin and has no dominator (normalised
// coordinates are >= 0); skipping it keeps correlated data's ~8.7e-4 n exact
// origin duplicates from scanning each other.
template <typename T, int D>
__global__ void __launch_bounds__(256) k_allpairs_lists(const T* __restrict__ rows, const uint32_t* __restrict__ ids,
                                                        const u64* __restrict__ fsum, const u64* __restrict__ count,
                                                        ListArrays<T, D> la, const unsigned* __restrict__ offs,
                                                        uint8_t* __restrict__ flag, u64 q_begin,
                                                        const u64* __restrict__ q_end, int cell_level,
                                                        unsigned max_steps, uint32_t* __restrict__ long_q,
                                                        u64* __restrict__ long_n, const u64* __restrict__ gate) {
  pdl_enter();
  if (gate && *gate == 0) return;
  const u64 n = q_end ? *q_end : *count;
  const int lane = threadIdx.x & 31;
  const u64 warp = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5;
  const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
  const int ctop = (1 << cell_level) - 1;
  for (u64 i = q_begin + warp; i < n; i += nwarps) {
    if (ids[i] == kNoId) {
      if (lane == 0) flag[i] = 0;
      continue;
    }
    if (fsum[i] == 0) {  // the origin: nothing dominates it
      if (lane == 0) flag[i] = 1;
      continue;
    }
    ListQuery<T, D> Q;
    Q.init(rows, fsum, ids, offs, i);
    const u64 lb = (u64)Q.bk * la.lcap;
    const unsigned* ob = offs + Q.bk * kListStride;
    bool dom = false, deferred = false;
    unsigned steps = 0;
    // columns 0..pc of dimension bk in ascending order; column c contributes
    // its sum buckets 0..sb, one contiguous range (column-major bins).  The
    // bounds of 32 columns are loaded at once (lane l: column c0 + l) and
    // only the non-empty ones are visited: sparse sets (anti-correlated d=2:
    // 1.4K points over 1,024 columns) otherwise spend a dependent load pair
    // per empty column.  Two 32-entry steps are in flight per iteration.
    for (int c0 = 0; c0 <= Q.pc && !dom && !deferred; c0 += 32) {
      const int cl = c0 + lane;
      unsigned b0 = 0, b1 = 0;
      if (cl <= Q.pc) {
        b0 = __ldg(ob + list_bin(0, cl));
        b1 = __ldg(ob + list_bin(Q.sb + 1, cl));
      }
      unsigned ne = __ballot_sync(kFull, b1 > b0);
      while (ne && !dom && !deferred) {
        const int src = __ffs(ne) - 1;
        ne &= ne - 1;
        const unsigned s0 = __shfl_sync(kFull, b0, src), s1 = __shfl_sync(kFull, b1, src);
        for (unsigned base = s0; base < s1; base += 64) {
          steps += 2;
          if (steps > max_steps + 1) {
            deferred = true;
            break;
          }
          const unsigned e0 = base + lane, e1 = e0 + 32;
          typename ListQuery<T, D>::Cand ca, cb;
          Q.fetch(la, lb, e0, e0 < s1, ca);
          Q.fetch(la, lb, e1, e1 < s1, cb);
          const bool d_l = Q.check(ca, cell_level, ctop) || Q.check(cb, cell_level, ctop);
          if (__any_sync(kFull, d_l)) {
            dom = true;
            break;
          }
        }
      }
    }
    if (lane == 0) {
      if (deferred) long_q[atomicAdd(long_n, 1ull)] = (uint32_t)i;
      else flag[i] = dom ? 0 : 1;
    }
  }
}

// Phase B: one CTA per deferred point, its candidate steps (64 entries each,
// two 32-entry loads in flight per warp) dealt round-robin to the 8 warps, a
// shared flag for the early exit.
template <typename T, int D>
__global__ void __launch_bounds__(256) k_allpairs_long(const T* __restrict__ rows, const uint32_t* __restrict__ ids,
                                                       const u64* __restrict__ fsum, ListArrays<T, D> la,
                                                       const unsigned* __restrict__ offs,
                                                       uint8_t* __restrict__ flag, int cell_level,
                                                       const uint32_t* __restrict__ long_q,
                                                       const u64* __restrict__ long_n) {
  pdl_enter();
  __shared__ int found;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int ctop = (1 << cell_level) - 1;
  const u64 nq = *long_n;
  for (u64 t = blockIdx.x; t < nq; t += gridDim.x) {
    const uint32_t i = long_q[t];
    if (threadIdx.x == 0) found = 0;
    __syncthreads();
    ListQuery<T, D> Q;
    Q.init(rows, fsum, ids, offs, i);
    const u64 lb = (u64)Q.bk * la.lcap;
    const unsigned* ob = offs + Q.bk * kListStride;
    unsigned g = 0;  // global step counter (identical in every warp)
    bool done = false;
    for (int c0 = 0; c0 <= Q.pc && !done; c0 += 32) {
      // bounds of 32 columns at once; only the non-empty ones are visited
      const int cl = c0 + lane;
      unsigned b0 = 0, b1 = 0;
      if (cl <= Q.pc) {
        b0 = __ldg(ob + list_bin(0, cl));
        b1 = __ldg(ob + list_bin(Q.sb + 1, cl));
      }
      unsigned ne = __ballot_sync(kFull, b1 > b0);
      while (ne && !done) {
        const int src = __ffs(ne) - 1;
        ne &= ne - 1;
        const unsigned s0 = __shfl_sync(kFull, b0, src), s1 = __shfl_sync(kFull, b1, src);
        const unsigned nsteps = (s1 - s0 + 63) / 64;
        // this warp's steps of the column: g + k with (g + k) % nw == warp
        unsigned k = (unsigned)((warp - (int)(g % nw) + nw) % nw);
        // the early-exit flag goes through shared atomics (a race by design,
        // kept visible to compute-sanitizer racecheck as synchronised access)
        auto seen = [&]() {
          int f = 0;
          if (lane == 0) f = atomicAdd(&found, 0);
          return __shfl_sync(kFull, f, 0) != 0;
        };
        for (; k < nsteps; k += nw) {
          if (seen()) break;
          const unsigned e0 = s0 + k * 64 + lane, e1 = e0 + 32;
          typename ListQuery<T, D>::Cand ca, cb;
          Q.fetch(la, lb, e0, e0 < s1, ca);
          Q.fetch(la, lb, e1, e1 < s1, cb);
          const bool d_l = Q.check(ca, cell_level, ctop) || Q.check(cb, cell_level, ctop);
          if (__any_sync(kFull, d_l)) {
            if (lane == 0) atomicExch(&found, 1);
            break;
          }
        }
        g += nsteps;
        if (seen()) done = true;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) flag[i] = found ? 0 : 1;
    __syncthreads();
  }
}

// ----------------------------------------------- K6: ascending record ids
// Skyline members set their record id in an n-bit bitmap; the ids are then
// written in ascending order by a two-pass popcount scan over the bitmap
// (refine.cpp:101-103 sorts instead).  kBitsBlock words per block.
constexpr int kBitsThreads = 256;
constexpr int kBitsPer = 8;
constexpr u64 kBitsBlock = (u64)kBitsThreads * kBitsPer;

static __global__ void k_mark_ids(const uint32_t* __restrict__ ids, const uint8_t* __restrict__ flag,
                           const u64* __restrict__ count, uint32_t* __restrict__ bits, uint32_t base) {
  pdl_enter();
  const u64 n = *count;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const uint32_t id = ids[i];
    if (id != kNoId && flag[i]) {
      const uint32_t b = id - base;
      atomicOr(bits + (b >> 5), 1u << (b & 31));
    }
  }
}

static __global__ void __launch_bounds__(kBitsThreads) k_bits_count(const uint32_t* __restrict__ bits, u64 words,
                                                             unsigned* __restrict__ block_counts) {
  pdl_enter();
  const u64 b0 = blockIdx.x * kBitsBlock;
  unsigned c = 0;
#pragma unroll
  for (int e = 0; e < kBitsPer; ++e) {
    const u64 w = b0 + (u64)e * kBitsThreads + threadIdx.x;
    if (w < words) c += __popc(bits[w]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
  __shared__ unsigned ws[kBitsThreads / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int w = 0; w < kBitsThreads / 32; ++w) t += ws[w];
    block_counts[blockIdx.x] = t;
  }
}

// Single CTA: exclusive scan of the block counts; total -> *out_count.
static __global__ void __launch_bounds__(1024) k_bits_scan(unsigned* __restrict__ block_counts, unsigned nblocks,
                                                    u64* __restrict__ out_count) {
  pdl_enter();
  __shared__ unsigned part[1024];
  const unsigned per = (nblocks + 1023) / 1024;
  unsigned sum = 0;
  for (unsigned e = 0; e < per; ++e) {
    const unsigned b = threadIdx.x * per + e;
    if (b < nblocks) sum += block_counts[b];
  }
  part[threadIdx.x] = sum;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const unsigned y = threadIdx.x >= (unsigned)o ? part[threadIdx.x - o] : 0;
    __syncthreads();
    part[threadIdx.x] += y;
    __syncthreads();
  }
  unsigned run = part[threadIdx.x] - sum;
  for (unsigned e = 0; e < per; ++e) {
    const unsigned b = threadIdx.x * per + e;
    if (b < nblocks) {
      const unsigned c = block_counts[b];
      block_counts[b] = run;
      run += c;
    }
  }
  if (threadIdx.x == 1023) *out_count = part[1023];
}

static __global__ void __launch_bounds__(kBitsThreads) k_bits_write(const uint32_t* __restrict__ bits, u64 words,
                                                             const unsigned* __restrict__ block_offs,
                                                             uint32_t* __restrict__ out_ids, uint32_t base) {
  pdl_enter();
  // thread t owns words b0 + t*kBitsPer .. +kBitsPer-1 (contiguous, so the
  // block-local exclusive scan over threads preserves id order)
  const u64 w0 = blockIdx.x * kBitsBlock + (u64)threadIdx.x * kBitsPer;
  uint32_t x[kBitsPer];
  unsigned c = 0;
#pragma unroll
  for (int e = 0; e < kBitsPer; ++e) {
    x[e] = (w0 + e < words) ? bits[w0 + e] : 0u;
    c += __popc(x[e]);
  }
  __shared__ unsigned ws[kBitsThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) ws[warp] = incl;
  __syncthreads();
  unsigned wbase = 0;
  for (int w = 0; w < warp; ++w) wbase += ws[w];
  unsigned pos = block_offs[blockIdx.x] + wbase + incl - c;
#pragma unroll
  for (int e = 0; e < kBitsPer; ++e) {
    uint32_t v = x[e];
    while (v) {
      const int b = __ffs(v) - 1;
      v &= v - 1;
      out_ids[pos++] = base + (uint32_t)((w0 + e) * 32 + b);
    }
  }
}

// Non-finite scan used only when rho is invalid: the reference normalizes
// (and reports non-finite records) before the grid rejects rho.
template <typename TIn>
__global__ void k_check_finite(const TIn* __restrict__ coords, u64 total, int d, u64* nonfinite) {
  pdl_enter();
  for (u64 e = blockIdx.x * (u64)blockDim.x + threadIdx.x; e < total; e += (u64)gridDim.x * blockDim.x) {
    if (!finite_v(coords[e])) atomicMax(nonfinite, ~(e / d));
  }
}

// ------------------------------------------- K2: occupancy OR across shards
// dst[w] = OR over g < world of gathered[g * words + w]: the bitwise-OR
// reduction NCCL lacks (nccl.h:260-275), applied to the all-gathered
// occupancy region of every rank.  uint4 words: 16 B per load.
static __global__ void k_or_gather(const uint4* __restrict__ gathered, int world, u64 words4, uint4* __restrict__ dst) {
  pdl_enter();
  for (u64 w = blockIdx.x * (u64)blockDim.x + threadIdx.x; w < words4; w += (u64)gridDim.x * blockDim.x) {
    uint4 x = gathered[w];
    for (int g = 1; g < world; ++g) {
      const uint4 y = gathered[(u64)g * words4 + w];
      x.x |= y.x;
      x.y |= y.y;
      x.z |= y.z;
      x.w |= y.w;
    }
    dst[w] = x;
  }
}

// Exchange 1 fused with the OR, single-process multi-GPU (csrc/multi.cu):
// srcs[g] is device g's exported occupancy region, read in place over NVLink
// / NVSwitch (peer access); no gather buffer, one pass.
static __global__ void k_or_peers(const uint4* const* __restrict__ srcs, int world, u64 words4, uint4* __restrict__ dst) {
  pdl_enter();
  for (u64 w = blockIdx.x * (u64)blockDim.x + threadIdx.x; w < words4; w += (u64)gridDim.x * blockDim.x) {
    uint4 x = srcs[0][w];
    for (int g = 1; g < world; ++g) {
      const uint4 y = srcs[g][w];
      x.x |= y.x;
      x.y |= y.y;
      x.z |= y.z;
      x.w |= y.w;
    }
    dst[w] = x;
  }
}

// Members (flag set, id != kNoId) of a slot array -> dense rows / sums / ids
// (order irrelevant: the final ids are ordered through the id bitmap).
template <typename T, int D>
__global__ void k_pack_members(const T* __restrict__ rows, const uint32_t* __restrict__ ids,
                               const uint8_t* __restrict__ flag, const u64* __restrict__ fsum,
                               const u64* __restrict__ count, T* __restrict__ out_rows, u64* __restrict__ out_fsum,
                               uint32_t* __restrict__ out_ids, u64* __restrict__ out_count) {
  pdl_enter();
  const u64 n = *count;
  const int lane = threadIdx.x & 31;
  for (u64 wb = ((blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5) * 32; wb < n;
       wb += ((u64)gridDim.x * blockDim.x >> 5) * 32) {
    const u64 i = wb + lane;
    const bool live = i < n && ids[i] != kNoId && (!flag || flag[i]);  // flag == nullptr: every member
    const unsigned m = __ballot_sync(kFull, live);
    if (!m) continue;
    u64 b = 0;
    if (lane == 0) b = atomicAdd(out_count, (u64)__popc(m));
    b = __shfl_sync(kFull, b, 0);
    if (live) {
      const u64 o = b + __popc(m & ((1u << lane) - 1));
      T v[D];
      load_row_cached<T, D>(rows, i, v);
      store_row<T, D>(out_rows, o, v);
      out_fsum[o] = fsum[i];
      out_ids[o] = ids[i];
    }
  }
}

// Filter-point gate: when a quarter or more of the sample's candidates are
// its own skyline points (anti-correlated data), the filter points kill
// little and the long column-prefix scans of K4b cost more than the points
// they remove (C3: 15 ms for ~1%); K4a then sends its survivors straight to
// S2 and K4b has nothing to do.
static __global__ void k_filter_gate(const u64* __restrict__ sky, const u64* __restrict__ cands,
                                     u64* __restrict__ weak) {
  pdl_enter();
  *weak = *sky * 4 > *cands;
}

// K5 dispatch without a host round trip: the column lists run on
// *lcount = the set's slot count when its point count is at most tree_min,
// else on 0 (the tree takes the set, launched once the host has the count).
// host: mapped pinned memory the host reads after an event (no copy-engine
// round trip in the stream: the lists launched next start at once).
static __global__ void k_gate_count(const u64* __restrict__ points, const u64* __restrict__ slots, u64 tree_min,
                                    const u64* __restrict__ origins, u64* __restrict__ lcount, u64* host) {
  pdl_enter();
  const u64 p = *points, o = *origins;
  *lcount = (o == 0 && p <= tree_min) ? *slots : 0;
  host[0] = p;
  host[1] = o;
}

// Device -> mapped pinned host words (the query's counters at the end).
static __global__ void k_copy_words(const u64* __restrict__ src, u64* dst, unsigned n) {
  pdl_enter();
  for (unsigned i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

// Exact origins (FP64 sum 0: every normalised coordinate 0 -- correlated
// data piles ~8.7e-4 n of them).  An origin precedes and
// dominates every other point and no origin dominates another, so a set with
// one is decided in O(n): members are exactly its origins.
static __global__ void k_origin_count(const uint32_t* __restrict__ ids, const u64* __restrict__ fsum,
                                      const u64* __restrict__ count, u64* __restrict__ origins) {
  pdl_enter();
  const u64 n = *count;
  unsigned c = 0;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
    c += ids[i] != kNoId && fsum[i] == 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(origins, (u64)c);
}

static __global__ void k_origin_flags(const uint32_t* __restrict__ ids, const u64* __restrict__ fsum,
                                      const u64* __restrict__ count, u64 q_begin, const u64* __restrict__ q_end,
                                      const u64* __restrict__ origins, uint8_t* __restrict__ flag) {
  pdl_enter();
  if (*origins == 0) return;
  const u64 n = q_end ? *q_end : *count;
  for (u64 i = q_begin + blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
    flag[i] = ids[i] != kNoId && fsum[i] == 0;
}

static __global__ void k_clamp_count(const u64* __restrict__ src, u64 cap, u64* __restrict__ dst) {
  pdl_enter();
  if (threadIdx.x == 0) *dst = *src < cap ? *src : cap;
}

static __global__ void k_fill_u32(uint32_t* __restrict__ p, u64 count, uint32_t v) {
  pdl_enter();
  const u64 tid = blockIdx.x * (u64)blockDim.x + threadIdx.x, stride = (u64)gridDim.x * blockDim.x;
  u64 head = 0;
  if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {  // 16-byte stores for the aligned bulk
    const uint4 w = make_uint4(v, v, v, v);
    uint4* q = reinterpret_cast<uint4*>(p);
    for (u64 i = tid; i < count / 4; i += stride) q[i] = w;
    head = count / 4 * 4;
  }
  for (u64 i = head + tid; i < count; i += stride) p[i] = v;
}

// ------------------------------------------------ quadrant_skyline (f1)
// refine.cpp:166-174: record i is inside iff p[k] >= origin[k] for every k
// (NaN compares false, so NaN records are outside).  Inside records set their
// bit in an n-bit bitmap; the K6 scan then lists them in ascending order,
// which is the reference's original_ids vector.
template <int D>
__global__ void k_quadrant_mark(const double* __restrict__ coords, u64 n, Norm origin, uint32_t* __restrict__ bits) {
  pdl_enter();
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    double v[D];
    load_row_cached<double, D>(coords, i, v);
    bool inside = true;
#pragma unroll
    for (int k = 0; k < D; ++k) inside &= v[k] >= origin.mn[k];
    if (inside) atomicOr(bits + (i >> 5), 1u << (i & 31));
  }
}

// Order-preserving u64 image of a double (for atomic min/max).
__device__ __forceinline__ u64 dkey(double x) {
  const u64 b = (u64)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ inline double dkey_inv(u64 k) {
  const u64 b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  double x;
  memcpy(&x, &b, 8);
  return x;
}

// sub.coords[j] = coords[orig[j]] and the per-dimension min / max of the
// subset (Dataset::compute_minmax, dataset.cpp:10-20; exact, order-free).
// mm[2k] = min key, mm[2k+1] = max key, pre-set to (~0, 0).
template <int D>
__global__ void k_quadrant_gather(const double* __restrict__ coords, const uint32_t* __restrict__ orig,
                                  const u64* __restrict__ count, double* __restrict__ sub, u64* __restrict__ mm) {
  pdl_enter();
  const u64 n = *count;
  u64 lo[D], hi[D];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    lo[k] = ~0ull;
    hi[k] = 0;
  }
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < n; j += (u64)gridDim.x * blockDim.x) {
    double v[D];
    load_row_cached<double, D>(coords, orig[j], v);
    store_row<double, D>(sub, j, v);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const u64 key = dkey(v[k]);
      lo[k] = key < lo[k] ? key : lo[k];
      hi[k] = key > hi[k] ? key : hi[k];
    }
  }
#pragma unroll
  for (int k = 0; k < D; ++k) {
    u64 a = lo[k], b = hi[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const u64 x = __shfl_xor_sync(kFull, a, o), y = __shfl_xor_sync(kFull, b, o);
      a = x < a ? x : a;
      b = y > b ? y : b;
    }
    if ((threadIdx.x & 31) == 0) {
      if (a != ~0ull) atomicMin(mm + 2 * k, a);
      if (b != 0) atomicMax(mm + 2 * k + 1, b);
    }
  }
}

// ids[j] = orig[ids[j]] (refine.cpp:182): ascending stays ascending.
static __global__ void k_map_ids(uint32_t* __restrict__ ids, const uint32_t* __restrict__ orig, u64 n) {
  pdl_enter();
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < n; j += (u64)gridDim.x * blockDim.x) ids[j] = orig[ids[j]];
}

}  // namespace sk
