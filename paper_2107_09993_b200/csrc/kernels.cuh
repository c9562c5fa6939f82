// SkyCell skyline kernels for B200 (sm_100a).
//
// Stage map (DESIGN.md §3 has the roofline of each):
//   K0  k_sample_occ / k_build_filter  occupancy of a point sample at a coarse
//                                       level Lf, turned into a per-row height
//                                       table H: a point whose level-Lf cell is
//                                       strictly dominated by an occupied
//                                       sample cell cannot be in a candidate
//                                       cell, so it is dropped
//                                       in the single streaming pass.
//   K1  k_stream                        THE HBM-bound pass: normalize (dataset.cpp:
//                                       22-50), point_to_cell (grid.cpp:10-16),
//                                       occupancy at layers rho and rho-1
//                                       (grid.cpp:78-102), sample filter, stable
//                                       compaction of survivors.  Reads every
//                                       coordinate exactly once.
//   K3  k_rowmin / k_prefix_min /       cell pruning as a d-dimensional prefix-OR,
//       k_count_cells / k_downsample    expressed as a row-min + (d-1)-dim prefix-
//                                       min table; per-layer |KS_i|, |CS_i|
//                                       (replaces shrink_seq.cpp:87-231 and
//                                       shrink_par.cpp:179-278).
//   K4  k_candidates                    survivors in candidate cells (refine.cpp:
//                                       78-96), points_examined.
//   K5  k_filter_append / k_allpairs /  exact sort-first dominance (refine.cpp:31-
//       k_compact                       59, 98-99) by a block-recursive filter:
//                                       skyline of a prefix filters the rest.
//   K6  ids leave K5 ascending (stable compaction everywhere).
#pragma once

#include "common.cuh"

namespace sk {

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
    return v < 0.0f ? 0.0f : (v >= 1.0f ? 1.0f : v);  // NaN passes through; reported separately
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
};

template <typename TIn, typename TOut, int D, bool IDENT>
__global__ void __launch_bounds__(256) k_sample(SampleParams p) {
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
    set_bit_global(p.occ_la, la_lin);
    if (p.occ_rho) set_bit_global(p.occ_rho, lin);
    store_row<TOut, D>(static_cast<TOut*>(p.rows), i, u);
    p.ids[i] = (uint32_t)i;
    p.fsum[i] = fsum_bits<TOut, D>(u);
  }
}

// Single CTA.  From the sample occupancy at level la build
//   R[x]  = min{c0 : occupied(c0, x)}       x = (c1..c_{d-1})
//   PM[x] = min_{y <= x} R[y]                (inclusive prefix-min)
//   H[x]  = all x_k >= 1 ? PM[x - 1] : 255
// so that a level-la cell c is strictly dominated by an occupied sample cell
// iff c0 > H[c1..c_{d-1}].  la <= 7, so u8 entries (255 = none) suffice.
__global__ void __launch_bounds__(1024) k_build_filter(const uint32_t* __restrict__ occ, int lf, int d,
                                                        uint8_t* __restrict__ H) {
  extern __shared__ uint8_t sm_pm[];
  const uint32_t rows = 1u << (lf * (d - 1));
  const int rowbits = 1 << lf;
  for (uint32_t r = threadIdx.x; r < rows; r += blockDim.x) {
    uint8_t best = 255;
    if (lf >= 5) {
      const int wpr = rowbits >> 5;
      for (int w = 0; w < wpr; ++w) {
        const uint32_t x = occ[(u64)r * wpr + w];
        if (x) { best = (uint8_t)(w * 32 + __ffs(x) - 1); break; }
      }
    } else {
      const int rpw = 32 >> lf;
      const uint32_t x = (occ[r / rpw] >> ((r % rpw) * rowbits)) & ((1u << rowbits) - 1);
      if (x) best = (uint8_t)(__ffs(x) - 1);
    }
    sm_pm[r] = best;
  }
  __syncthreads();
  for (int k = 1; k < d; ++k) {
    const uint32_t stride = 1u << (lf * (k - 1));
    const uint32_t lines = rows >> lf;
    for (uint32_t line = threadIdx.x; line < lines; line += blockDim.x) {
      const uint32_t low = line & (stride - 1);
      const uint32_t high = line >> (lf * (k - 1));
      const uint32_t base = (high << (lf * k)) + low;
      uint8_t run = 255;
      for (int c = 0; c < rowbits; ++c) {
        const uint32_t idx = base + c * stride;
        run = min(run, sm_pm[idx]);
        sm_pm[idx] = run;
      }
    }
    __syncthreads();
  }
  const uint32_t mask = (1u << lf) - 1;
  for (uint32_t r = threadIdx.x; r < rows; r += blockDim.x) {
    bool ok = true;
    uint32_t prev = 0;
    for (int k = 1; k < d; ++k) {
      const uint32_t c = (r >> (lf * (k - 1))) & mask;
      ok &= c >= 1;
      prev |= (c - 1) << (lf * (k - 1));
    }
    H[r] = ok ? sm_pm[prev] : (uint8_t)255;
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
// Two-level cell filter (SURVEY §0.3 applied to a sample):
//   A: level la (<= 7, table H in shared memory): the point's level-la cell
//      is strictly dominated by an occupied sample cell -> not a candidate.
//   B: layer rho (global prefix-min table of the sample, only for points
//      passing A): same test at the reference's own layer.
// A point filtered at level L can influence the reference's per-layer
// key/candidate sets only at layers < L, so its occupancy is
// recorded at layer L-1: a shared-memory bitmap for A (tiny), a global
// check-before-set bitmap for B.  Survivors (about the candidate-cell
// fraction: 6.1% at the headline config) are compacted in input order and set
// their bit in the layer-rho occupancy.  Every coordinate is read once.
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
  u64* status;
  u64* claim;
  u64* out_count;
  u64* nonfinite;          // max of (~record) over non-finite records: 0 = none
};

template <typename TIn, typename TOut, int D, bool IDENT, int THREADS, int PPT>
__global__ void __launch_bounds__(THREADS) k_stream(StreamParams p) {
  extern __shared__ __align__(16) uint8_t sm[];
  uint32_t* occ_s = reinterpret_cast<uint32_t*>(sm);
  uint8_t* H_s = sm + p.lo_words * 4;
  unsigned* scratch = reinterpret_cast<unsigned*>(sm + p.lo_words * 4 + ((p.h_entries + 15) & ~15u));
  __shared__ u64 s_tile, s_excl;

  for (uint32_t w = threadIdx.x; w < p.lo_words; w += THREADS) occ_s[w] = 0;
  for (uint32_t e = threadIdx.x; e < p.h_entries; e += THREADS) H_s[e] = p.H[e];
  __syncthreads();

  const TIn* coords = static_cast<const TIn*>(p.coords);
  TOut* out_rows = static_cast<TOut*>(p.out_rows);
  constexpr u64 TILE = (u64)THREADS * PPT;
  const u64 ntiles = (p.n + TILE - 1) / TILE;
  const int rho = p.rho, la = p.la, sh = rho - la, lo_sh = rho - la + 1;
  const int top = (1 << rho) - 1;
  const float fscale = ldexpf(1.0f, rho);
  const double dscale = ldexp(1.0, rho);
  const bool test_b = p.PMs != nullptr;

  while (true) {
    if (threadIdx.x == 0) s_tile = atomicAdd(p.claim, 1ull);
    __syncthreads();
    const u64 tile = s_tile;
    if (tile >= ntiles) break;
    const u64 base = tile * TILE;

    TIn raw[PPT][D];
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      const u64 i = base + (u64)j * THREADS + threadIdx.x;
      if (i < p.n) load_row<TIn, D>(coords, i, raw[j]);
    }

    bool keep[PPT];
    unsigned rank[PPT];
    TOut val[PPT][D];
    u64 lin[PPT];
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      const u64 i = base + (u64)j * THREADS + threadIdx.x;
      const bool valid = i < p.n;
      bool fin = true;
      u64 l = 0, pl = 0;
      uint32_t hidx = 0, lo = 0;
      int col[D];
#pragma unroll
      for (int k = D - 1; k >= 0; --k) {
        fin &= finite_v(raw[j][k]);
        const TOut u = Coord<TIn, TOut, IDENT>::value(raw[j][k], p.nm, k);
        val[j][k] = u;
        const int c = Coord<TIn, TOut, IDENT>::col(u, fscale, dscale, top);
        col[k] = c;
        l = (l << rho) | (u64)c;
        pl = (pl << (rho - 1)) | (u64)(c >> 1);
        lo = (lo << (la - 1)) | (uint32_t)(c >> lo_sh);
        if (k >= 1) hidx = (hidx << la) | (uint32_t)(c >> sh);
      }
      if (valid && !fin) atomicMax(p.nonfinite, ~i);
      const bool fail_a = (col[0] >> sh) > (int)H_s[hidx];
      bool fail_b = false;
      if (valid && !fail_a && test_b) {
        fail_b = p.pms_wide ? strictly_dominated_cols<uint32_t, D>(static_cast<const uint32_t*>(p.PMs), col, rho)
                            : strictly_dominated_cols<uint8_t, D>(static_cast<const uint8_t*>(p.PMs), col, rho);
      }
      if (valid && fail_a && la >= 2) set_bit_shared(occ_s, lo);
      if (valid && fail_b) set_bit_global(p.occ_rm1, pl);
      keep[j] = valid && !fail_a && !fail_b;
      lin[j] = l;
    }

    const unsigned total = block_ranks<THREADS, PPT>(keep, rank, scratch);
    if (threadIdx.x < 32) {
      const u64 excl = warp_lookback(p.status, tile, total);
      if (threadIdx.x == 0) {
        s_excl = excl;
        if (tile == ntiles - 1) *p.out_count = excl + total;
      }
    }
    __syncthreads();
    const u64 excl = s_excl;
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      if (keep[j]) {
        const u64 i = base + (u64)j * THREADS + threadIdx.x;
        const u64 o = excl + rank[j];
        store_row<TOut, D>(out_rows, o, val[j]);
        p.out_ids[o] = (uint32_t)i;
        set_bit_global(p.occ_rho, lin[j]);
      }
    }
  }
  if (p.lo_words) {
    __syncthreads();
    uint32_t* slab = p.slabs + (u64)blockIdx.x * p.lo_words;
    for (uint32_t w = threadIdx.x; w < p.lo_words; w += THREADS) slab[w] = occ_s[w];
  }
}

__global__ void k_reduce_slabs(const uint32_t* __restrict__ slabs, int nslabs, uint32_t words,
                               uint32_t* __restrict__ out) {
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < words; w += gridDim.x * blockDim.x) {
    uint32_t x = 0;
    for (int s = 0; s < nslabs; ++s) x |= slabs[(u64)s * words + w];
    out[w] |= x;
  }
}

// ------------------------------------------------- K3: cell pruning tables
// Row-min of dimension 0 (the innermost `L` bits of the linear index) fused
// with the inclusive prefix-min along dimension 1: one thread per dimension-1
// line computes the 2^L row minima of that line and scans them.
template <typename TT>
__global__ void k_rowmin_prefix1(const uint32_t* __restrict__ bits, int L, int d, u64 lines, TT* __restrict__ R) {
  const int n = 1 << L;
  const int rowbits = 1 << L;
  for (u64 line = blockIdx.x * (u64)blockDim.x + threadIdx.x; line < lines; line += (u64)gridDim.x * blockDim.x) {
    // rows of this line: r = high * n * n + c1 * n + ... ; with d == 2 there is one line
    const u64 row0 = line * (u64)n;  // dimension-1 index is the lowest digit of the row index
    TT run = (TT)~(TT)0;
    for (int c1 = 0; c1 < n; ++c1) {
      const u64 r = row0 + c1;
      TT best = (TT)~(TT)0;
      if (L >= 5) {
        const u64 wpr = (u64)rowbits >> 5;
        for (u64 w = 0; w < wpr; ++w) {
          const uint32_t x = __ldg(bits + r * wpr + w);
          if (x) { best = (TT)(w * 32 + __ffs(x) - 1); break; }
        }
      } else {
        const int rpw = 32 >> L;
        const uint32_t x = (__ldg(bits + r / rpw) >> ((r % rpw) * rowbits)) & ((1u << rowbits) - 1);
        if (x) best = (TT)(__ffs(x) - 1);
      }
      run = best < run ? best : run;
      R[r] = run;
    }
  }
}

// Inclusive prefix-min along dimension k (2..d-1) of the (d-1)-dim table.
// Loads are issued 16 at a time ahead of the dependent min-scan.
template <typename TT>
__global__ void k_prefix_min(TT* __restrict__ R, int L, int k, u64 lines) {
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
template <typename TT>
__device__ __forceinline__ bool cell_strictly_dominated(const TT* __restrict__ PM, const int* col, int d, int L) {
  u64 idx = 0;
  bool ok = col[0] >= 1;
  for (int k = d - 1; k >= 1; --k) {
    ok &= col[k] >= 1;
    idx = (idx << L) | (u64)(col[k] - 1);
  }
  return ok && (int64_t)PM[idx] <= (int64_t)col[0] - 1;
}

template <typename TT>
__global__ void k_count_cells(const uint32_t* __restrict__ bits, int L, int d, u64 words,
                              const TT* __restrict__ PM, u64* cand_out, u64* key_out) {
  const int top = (1 << L) - 1;
  const u64 mask = (1ull << L) - 1;
  u64 nc = 0, nk = 0;
  for (u64 w = blockIdx.x * (u64)blockDim.x + threadIdx.x; w < words; w += (u64)gridDim.x * blockDim.x) {
    uint32_t x = bits[w];
    while (x) {
      const int b = __ffs(x) - 1;
      x &= x - 1;
      u64 lin = w * 32 + b;
      int col[kMaxD];
      bool has_top = false;
      for (int k = 0; k < d; ++k) {
        col[k] = (int)(lin & mask);
        lin >>= L;
        has_top |= col[k] == top;
      }
      if (!cell_strictly_dominated(PM, col, d, L)) ++nc;
      if (!has_top) {
        // P[c - e_0]
        u64 idx = 0;
        for (int k = d - 1; k >= 1; --k) idx = (idx << L) | (u64)col[k];
        bool sdom = col[0] >= 1 && (int64_t)PM[idx] <= (int64_t)col[0] - 1;
        for (int j = 1; j < d && !sdom; ++j) {
          if (col[j] < 1) continue;
          u64 ij = 0;
          for (int k = d - 1; k >= 1; --k) ij = (ij << L) | (u64)(col[k] - (k == j ? 1 : 0));
          sdom = (int64_t)PM[ij] <= (int64_t)col[0];
        }
        if (!sdom) ++nk;
      }
    }
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

// Occupancy of layer L from layer L+1 (grid.cpp:80-102, child-OR), OR-ed into dst.
__global__ void k_downsample(const uint32_t* __restrict__ src, int L, int d, u64 src_words,
                             uint32_t* __restrict__ dst) {
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
  const uint32_t* ids;
  const u64* count;      // |S1|
  int rho;
  const void* PM;        // layer-rho prefix-min table (u8 or u32), nullptr: no cell test
  const void* f_rows;    // filter points (strength order), may be empty
  const u64* f_fsum;
  const u64* f_count;
  uint32_t f_max;
  void* out_rows;
  uint32_t* out_ids;
  u64* out_fsum;
  u64* status;
  u64* claim;
  u64* out_count;
  u64* examined;         // points_examined (refine.cpp:90-96), may be null
};

template <typename T, int D, typename TT, int THREADS, int PPT>
__global__ void __launch_bounds__(THREADS) k_candidates(CandParams p) {
  extern __shared__ __align__(16) uint8_t smc[];
  __shared__ unsigned scratch[PPT * (THREADS / 32) + 1];
  __shared__ u64 s_tile, s_excl;
  const u64 n = *p.count;
  constexpr u64 TILE = (u64)THREADS * PPT;
  const u64 ntiles = (n + TILE - 1) / TILE;
  if (ntiles == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *p.out_count = 0;
    return;
  }
  uint32_t nf = 0;
  T* f_rows = reinterpret_cast<T*>(smc);
  u64* f_sum = reinterpret_cast<u64*>(smc + (((u64)p.f_max * D * sizeof(T) + 15) & ~15ull));
  if (p.f_count) {
    const u64 fc = *p.f_count;
    nf = (uint32_t)(fc < p.f_max ? fc : p.f_max);
    const T* fr = static_cast<const T*>(p.f_rows);
    for (uint32_t e = threadIdx.x; e < nf * D; e += THREADS) f_rows[e] = fr[e];
    for (uint32_t e = threadIdx.x; e < nf; e += THREADS) f_sum[e] = p.f_fsum[e];
    __syncthreads();
  }
  const T* rows = static_cast<const T*>(p.rows);
  T* out_rows = static_cast<T*>(p.out_rows);
  const TT* PM = static_cast<const TT*>(p.PM);
  const int rho = p.rho, top = (1 << rho) - 1;
  const float fscale = ldexpf(1.0f, rho);
  const double dscale = ldexp(1.0, rho);
  u64 examined = 0;
  while (true) {
    if (threadIdx.x == 0) s_tile = atomicAdd(p.claim, 1ull);
    __syncthreads();
    const u64 tile = s_tile;
    if (tile >= ntiles) break;
    const u64 base = tile * TILE;
    T v[PPT][D];
    u64 ps[PPT];
    bool keep[PPT];
    unsigned rank[PPT];
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      const u64 i = base + (u64)j * THREADS + threadIdx.x;
      keep[j] = false;
      if (i < n) {
        load_row_cached<T, D>(rows, i, v[j]);
        bool cand = true;
        if (PM) {
          int col[D];
#pragma unroll
          for (int k = 0; k < D; ++k) {
            if constexpr (sizeof(T) == 4) col[k] = cell_col(v[j][k], fscale, top);
            else col[k] = cell_col(v[j][k], dscale, top);
          }
          cand = !strictly_dominated_cols<TT, D>(PM, col, rho);
        }
        examined += cand;
        ps[j] = fsum_bits<T, D>(v[j]);
        bool dom = false;
        if (cand) {
          for (uint32_t f = 0; f < nf && !dom; ++f)
            dom = f_sum[f] < ps[j] && dominates<T, D>(f_rows + (u64)f * D, v[j]);
        }
        keep[j] = cand && !dom;
      }
    }
    const unsigned total = block_ranks<THREADS, PPT>(keep, rank, scratch);
    if (threadIdx.x < 32) {
      const u64 excl = warp_lookback(p.status, tile, total);
      if (threadIdx.x == 0) {
        s_excl = excl;
        if (tile == ntiles - 1) *p.out_count = excl + total;
      }
    }
    __syncthreads();
    const u64 excl = s_excl;
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      if (keep[j]) {
        const u64 i = base + (u64)j * THREADS + threadIdx.x;
        const u64 o = excl + rank[j];
        store_row<T, D>(out_rows, o, v[j]);
        p.out_ids[o] = p.ids[i];
        p.out_fsum[o] = ps[j];
      }
    }
  }
  if (p.examined) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) examined += __shfl_xor_sync(kFull, examined, o);
    if ((threadIdx.x & 31) == 0 && examined) atomicAdd(p.examined, examined);
  }
}

// Single CTA: order a point set by descending "strength" -- the volume it
// dominates in the unit cube, prod(1 - u_k) -- in 64 log-spaced buckets, and
// keep the first f_max.  Strong filter points first make the early exit in
// k_candidates happen after ~1 test for most points (median 1, p90 18 at the
// headline config).
template <typename T, int D>
__global__ void __launch_bounds__(1024) k_strength_order(const T* __restrict__ rows, const u64* __restrict__ fsum,
                                                          const u64* __restrict__ count, uint32_t f_max,
                                                          T* __restrict__ out_rows, u64* __restrict__ out_fsum,
                                                          u64* __restrict__ out_count) {
  __shared__ unsigned hist[65];
  __shared__ unsigned offs[65];
  const u64 n = *count;
  if (threadIdx.x < 65) hist[threadIdx.x] = 0;
  __syncthreads();
  auto bucket = [&](u64 i) {
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
    *out_count = n < f_max ? n : f_max;
  }
  __syncthreads();
  for (u64 i = threadIdx.x; i < n; i += blockDim.x) {
    const unsigned o = atomicAdd(&offs[bucket(i)], 1u);
    if (o < f_max) {
#pragma unroll
      for (int k = 0; k < D; ++k) out_rows[(u64)o * D + k] = rows[i * D + k];
      out_fsum[o] = fsum[i];
    }
  }
}

// ------------------------------------------- K5: exact sort-first dominance
// A point set in ascending-id order: rows (T[D]), record ids, FP64 sum bits.
template <typename T>
struct PointBuf {
  T* rows;
  uint32_t* ids;
  u64* fsum;
};

// Append the points of src[begin, end) (end clamped to *src_count) that no
// filter point f (the first nf of F, f preceding p and f dominating p)
// eliminates, to dst at offset *dst_count_in; writes the new count.
struct FilterParams {
  const void* src_rows;
  const uint32_t* src_ids;
  const u64* src_fsum;
  const u64* src_count;
  u64 begin, end;
  const void* f_rows;
  const uint32_t* f_ids;
  const u64* f_fsum;
  const u64* f_count;
  uint32_t f_max;
  void* dst_rows;
  uint32_t* dst_ids;
  u64* dst_fsum;
  const u64* dst_count_in;
  u64* dst_count_out;
  u64* status;
  u64* claim;
};

template <typename T, int D, int THREADS, int PPT>
__global__ void __launch_bounds__(THREADS) k_filter_append(FilterParams p) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ unsigned scratch[PPT * (THREADS / 32) + 1];
  __shared__ u64 s_tile, s_excl;
  const u64 total_src = *p.src_count;
  const u64 end = p.end < total_src ? p.end : total_src;
  const u64 begin = p.begin;
  const u64 nsrc = end > begin ? end - begin : 0;
  const u64 off = *p.dst_count_in;
  constexpr u64 TILE = (u64)THREADS * PPT;
  const u64 ntiles = (nsrc + TILE - 1) / TILE;
  if (ntiles == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *p.dst_count_out = off;
    return;
  }
  const u64 fc = *p.f_count;
  const uint32_t nf = (uint32_t)(fc < p.f_max ? fc : p.f_max);
  T* f_rows = reinterpret_cast<T*>(sm);
  u64* f_sum = reinterpret_cast<u64*>(sm + (((u64)p.f_max * D * sizeof(T) + 15) & ~15ull));
  uint32_t* f_id = reinterpret_cast<uint32_t*>(f_sum + p.f_max);
  const T* frows_g = static_cast<const T*>(p.f_rows);
  for (uint32_t e = threadIdx.x; e < nf * D; e += THREADS) f_rows[e] = frows_g[e];
  for (uint32_t e = threadIdx.x; e < nf; e += THREADS) {
    f_sum[e] = p.f_fsum[e];
    f_id[e] = p.f_ids[e];
  }
  __syncthreads();
  const T* src_rows = static_cast<const T*>(p.src_rows);
  T* dst_rows = static_cast<T*>(p.dst_rows);
  while (true) {
    if (threadIdx.x == 0) s_tile = atomicAdd(p.claim, 1ull);
    __syncthreads();
    const u64 tile = s_tile;
    if (tile >= ntiles) break;
    const u64 base = begin + tile * TILE;
    T v[PPT][D];
    u64 ps[PPT];
    uint32_t pid[PPT];
    bool keep[PPT];
    unsigned rank[PPT];
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      const u64 i = base + (u64)j * THREADS + threadIdx.x;
      keep[j] = false;
      if (i < end) {
        load_row_cached<T, D>(src_rows, i, v[j]);
        ps[j] = p.src_fsum[i];
        pid[j] = p.src_ids[i];
        bool dom = false;
        for (uint32_t f = 0; f < nf && !dom; ++f) {
          dom = precedes(f_sum[f], f_id[f], ps[j], pid[j]) && dominates<T, D>(f_rows + (u64)f * D, v[j]);
        }
        keep[j] = !dom;
      }
    }
    const unsigned total = block_ranks<THREADS, PPT>(keep, rank, scratch);
    if (threadIdx.x < 32) {
      const u64 excl = warp_lookback(p.status, tile, total);
      if (threadIdx.x == 0) {
        s_excl = excl;
        if (tile == ntiles - 1) *p.dst_count_out = off + excl + total;
      }
    }
    __syncthreads();
    const u64 excl = s_excl;
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      if (keep[j]) {
        const u64 o = off + excl + rank[j];
        store_row<T, D>(dst_rows, o, v[j]);
        p.dst_ids[o] = pid[j];
        p.dst_fsum[o] = ps[j];
      }
    }
  }
}

// flag[i] is cleared iff some point of the set precedes point i and
// dominates it (flags start at 1).  2-D decomposition: blockIdx.x picks a
// block of THREADS points p, blockIdx.y a chunk of QCHUNK candidate
// dominators q, so small sets still fill the GPU.
template <typename T, int D, int THREADS, int QCHUNK>
__global__ void __launch_bounds__(THREADS) k_allpairs(const T* __restrict__ rows, const uint32_t* __restrict__ ids,
                                                      const u64* __restrict__ fsum, const u64* __restrict__ count,
                                                      uint8_t* __restrict__ flag) {
  __shared__ T q_rows[THREADS * D];
  __shared__ u64 q_sum[THREADS];
  __shared__ uint32_t q_id[THREADS];
  const u64 n = *count;
  const u64 q0 = (u64)blockIdx.y * QCHUNK;
  if (q0 >= n) return;
  const u64 q1 = q0 + QCHUNK < n ? q0 + QCHUNK : n;
  for (u64 pb = blockIdx.x; pb * THREADS < n; pb += gridDim.x) {
    const u64 i = pb * THREADS + threadIdx.x;
    T v[D];
    u64 ps = 0;
    uint32_t pid = 0;
    bool alive = i < n && flag[i];
    if (alive) {
      load_row_cached<T, D>(rows, i, v);
      ps = fsum[i];
      pid = ids[i];
    }
    bool dominated = false;
    for (u64 qt = q0; qt < q1; qt += THREADS) {
      if (!__syncthreads_or(alive)) break;
      const u64 qi = qt + threadIdx.x;
      if (qi < q1) {
        T q[D];
        load_row_cached<T, D>(rows, qi, q);
#pragma unroll
        for (int k = 0; k < D; ++k) q_rows[threadIdx.x * D + k] = q[k];
        q_sum[threadIdx.x] = fsum[qi];
        q_id[threadIdx.x] = ids[qi];
      }
      __syncthreads();
      const u64 rem = q1 - qt;
      const int m = rem < THREADS ? (int)rem : THREADS;
      if (alive) {
        for (int j = 0; j < m; ++j) {
          if (precedes(q_sum[j], q_id[j], ps, pid) && dominates<T, D>(q_rows + j * D, v)) {
            alive = false;
            dominated = true;
            break;
          }
        }
      }
    }
    __syncthreads();
    if (dominated) flag[i] = 0;
  }
}

struct CompactParams {
  const void* src_rows;
  const uint32_t* src_ids;
  const u64* src_fsum;
  const u64* count;
  const uint8_t* flag;
  void* dst_rows;
  uint32_t* dst_ids;
  u64* dst_fsum;
  u64* dst_count;
  u64* status;
  u64* claim;
};

template <typename T, int D, int THREADS, int PPT>
__global__ void __launch_bounds__(THREADS) k_compact(CompactParams p) {
  __shared__ unsigned scratch[PPT * (THREADS / 32) + 1];
  __shared__ u64 s_tile, s_excl;
  const u64 n = *p.count;
  constexpr u64 TILE = (u64)THREADS * PPT;
  const u64 ntiles = (n + TILE - 1) / TILE;
  if (ntiles == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *p.dst_count = 0;
    return;
  }
  const T* src_rows = static_cast<const T*>(p.src_rows);
  T* dst_rows = static_cast<T*>(p.dst_rows);
  while (true) {
    if (threadIdx.x == 0) s_tile = atomicAdd(p.claim, 1ull);
    __syncthreads();
    const u64 tile = s_tile;
    if (tile >= ntiles) break;
    const u64 base = tile * TILE;
    bool keep[PPT];
    unsigned rank[PPT];
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      const u64 i = base + (u64)j * THREADS + threadIdx.x;
      keep[j] = i < n && p.flag[i];
    }
    const unsigned total = block_ranks<THREADS, PPT>(keep, rank, scratch);
    if (threadIdx.x < 32) {
      const u64 excl = warp_lookback(p.status, tile, total);
      if (threadIdx.x == 0) {
        s_excl = excl;
        if (tile == ntiles - 1) *p.dst_count = excl + total;
      }
    }
    __syncthreads();
    const u64 excl = s_excl;
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      if (keep[j]) {
        const u64 i = base + (u64)j * THREADS + threadIdx.x;
        const u64 o = excl + rank[j];
        T v[D];
        load_row_cached<T, D>(src_rows, i, v);
        store_row<T, D>(dst_rows, o, v);
        p.dst_ids[o] = p.src_ids[i];
        p.dst_fsum[o] = p.src_fsum[i];
      }
    }
  }
}

// Non-finite scan used only when rho is invalid: the reference normalizes
// (and reports non-finite records) before the grid rejects rho.
template <typename TIn>
__global__ void k_check_finite(const TIn* __restrict__ coords, u64 total, int d, u64* nonfinite) {
  for (u64 e = blockIdx.x * (u64)blockDim.x + threadIdx.x; e < total; e += (u64)gridDim.x * blockDim.x) {
    if (!finite_v(coords[e])) atomicMax(nonfinite, ~(e / d));
  }
}

}  // namespace sk
