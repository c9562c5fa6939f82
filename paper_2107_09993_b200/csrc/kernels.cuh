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
struct SampleParams {
  const void* coords;
  u64 m;  // sample size (a prefix of the input)
  int rho, lf;
  Norm nm;
  uint32_t* occ;  // 2^(lf*d) bits
};

template <typename TIn, typename TOut, int D, bool IDENT>
__global__ void __launch_bounds__(256) k_sample_occ(SampleParams p) {
  const TIn* coords = static_cast<const TIn*>(p.coords);
  const int top = (1 << p.rho) - 1;
  const float fscale = ldexpf(1.0f, p.rho);
  const double dscale = ldexp(1.0, p.rho);
  const int sh = p.rho - p.lf;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < p.m; i += (u64)gridDim.x * blockDim.x) {
    TIn raw[D];
    load_row<TIn, D>(coords, i, raw);
    u64 lin = 0;
#pragma unroll
    for (int k = D - 1; k >= 0; --k) {
      const TOut u = Coord<TIn, TOut, IDENT>::value(raw[k], p.nm, k);
      const int c = Coord<TIn, TOut, IDENT>::col(u, fscale, dscale, top) >> sh;
      lin = (lin << p.lf) | (u64)c;
    }
    set_bit_global(p.occ, lin);
  }
}

// Single CTA.  From the sample occupancy at level lf build
//   R[x]  = min{c0 : occupied(c0, x)}       x = (c1..c_{d-1})
//   PM[x] = min_{y <= x} R[y]                (inclusive prefix-min)
//   H[x]  = all x_k >= 1 ? PM[x - 1] : 255
// so that a level-lf cell c is strictly dominated by an occupied sample cell
// iff c0 > H[c1..c_{d-1}].  lf <= 7, so u8 entries (255 = none) suffice.
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
      const uint32_t x = (occ[r / rpw] >> ((r % rpw) * rowbits)) & ((rowbits == 32) ? kFull : ((1u << rowbits) - 1));
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

// -------------------------------------------------------- K1: the stream
struct StreamParams {
  const void* coords;
  u64 n;
  int rho, lf;
  int rm1_mode;  // 0: no layer below rho (rho == 1); 1: shared-memory bitmap; 2: global atomics
  uint32_t rm1_words;
  uint32_t h_entries;
  Norm nm;
  const uint8_t* H;
  uint32_t* occ_rho;   // layer rho, survivors only (SURVEY §0.3 argument in DESIGN.md)
  uint32_t* occ_rm1;   // layer rho-1, every point (global mode)
  uint32_t* slabs;     // per-CTA copies of the layer rho-1 bitmap (shared mode)
  void* out_rows;
  uint32_t* out_ids;
  u64* status;
  u64* claim;
  u64* out_count;
  u64* nonfinite;      // max of (~record) over non-finite records: 0 = none
};

template <typename TIn, typename TOut, int D, bool IDENT, int THREADS, int PPT>
__global__ void __launch_bounds__(THREADS) k_stream(StreamParams p) {
  extern __shared__ __align__(16) uint8_t sm[];
  uint32_t* occ_s = reinterpret_cast<uint32_t*>(sm);
  const uint32_t occ_words = p.rm1_mode == 1 ? p.rm1_words : 0;
  uint8_t* H_s = sm + occ_words * 4;
  unsigned* scratch = reinterpret_cast<unsigned*>(sm + occ_words * 4 + ((p.h_entries + 15) & ~15u));
  __shared__ u64 s_tile, s_excl;

  for (uint32_t w = threadIdx.x; w < occ_words; w += THREADS) occ_s[w] = 0;
  for (uint32_t e = threadIdx.x; e < p.h_entries; e += THREADS) H_s[e] = p.H[e];
  __syncthreads();

  const TIn* coords = static_cast<const TIn*>(p.coords);
  TOut* out_rows = static_cast<TOut*>(p.out_rows);
  constexpr u64 TILE = (u64)THREADS * PPT;
  const u64 ntiles = (p.n + TILE - 1) / TILE;
  const int rho = p.rho, lf = p.lf, sh = rho - lf;
  const int top = (1 << rho) - 1;
  const float fscale = ldexpf(1.0f, rho);
  const double dscale = ldexp(1.0, rho);

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
      uint32_t hidx = 0;
      int c0lf = 0;
#pragma unroll
      for (int k = D - 1; k >= 0; --k) {
        fin &= finite_v(raw[j][k]);
        const TOut u = Coord<TIn, TOut, IDENT>::value(raw[j][k], p.nm, k);
        val[j][k] = u;
        const int c = Coord<TIn, TOut, IDENT>::col(u, fscale, dscale, top);
        l = (l << rho) | (u64)c;
        pl = (pl << (rho - 1)) | (u64)(c >> 1);
        if (k >= 1) hidx = (hidx << lf) | (uint32_t)(c >> sh);
        else c0lf = c >> sh;
      }
      if (valid && !fin) atomicMax(p.nonfinite, ~i);
      if (valid && p.rm1_mode == 1) set_bit_shared(occ_s, (uint32_t)pl);
      else if (valid && p.rm1_mode == 2) set_bit_global(p.occ_rm1, pl);
      keep[j] = valid && (lf == 0 || c0lf <= (int)H_s[hidx]);
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
  if (p.rm1_mode == 1) {
    __syncthreads();
    uint32_t* slab = p.slabs + (u64)blockIdx.x * occ_words;
    for (uint32_t w = threadIdx.x; w < occ_words; w += THREADS) slab[w] = occ_s[w];
  }
}

__global__ void k_reduce_slabs(const uint32_t* __restrict__ slabs, int nslabs, uint32_t words,
                               uint32_t* __restrict__ out) {
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < words; w += gridDim.x * blockDim.x) {
    uint32_t x = 0;
    for (int s = 0; s < nslabs; ++s) x |= slabs[(u64)s * words + w];
    out[w] = x;
  }
}

// ------------------------------------------------- K3: cell pruning tables
// Row-min of dimension 0 (the innermost `layer` bits of the linear index).
template <typename TT>
__global__ void k_rowmin(const uint32_t* __restrict__ bits, int L, u64 rows, TT* __restrict__ R) {
  const int rowbits = 1 << L;
  for (u64 r = blockIdx.x * (u64)blockDim.x + threadIdx.x; r < rows; r += (u64)gridDim.x * blockDim.x) {
    TT best = (TT)~(TT)0;
    if (L >= 5) {
      const u64 wpr = (u64)rowbits >> 5;
      for (u64 w = 0; w < wpr; ++w) {
        const uint32_t x = bits[r * wpr + w];
        if (x) { best = (TT)(w * 32 + __ffs(x) - 1); break; }
      }
    } else {
      const int rpw = 32 >> L;
      const uint32_t mask = (1u << rowbits) - 1;
      const uint32_t x = (bits[r / rpw] >> ((r % rpw) * rowbits)) & mask;
      if (x) best = (TT)(__ffs(x) - 1);
    }
    R[r] = best;
  }
}

// Inclusive prefix-min along dimension k (1..d-1) of the (d-1)-dim table.
template <typename TT>
__global__ void k_prefix_min(TT* __restrict__ R, int L, int k, u64 lines) {
  const u64 stride = 1ull << (L * (k - 1));
  const int n = 1 << L;
  for (u64 line = blockIdx.x * (u64)blockDim.x + threadIdx.x; line < lines;
       line += (u64)gridDim.x * blockDim.x) {
    const u64 low = line & (stride - 1);
    const u64 high = line >> (L * (k - 1));
    const u64 base = (high << (L * k)) + low;
    TT run = (TT)~(TT)0;
    for (int c = 0; c < n; ++c) {
      const u64 idx = base + (u64)c * stride;
      const TT v = R[idx];
      run = v < run ? v : run;
      R[idx] = run;
    }
  }
}

// Cell status from the prefix-min table PM (inclusive prefix-OR P[c] <=>
// PM[c1..] <= c0):
//   candidate  = occupied && !(all c_k >= 1 && P[c - 1])                  (Def. 5)
//   key (grid) = occupied && no top column && !OR_k (c_k >= 1 && P[c - e_k])  (Def. 4)
// Key counts add the d auxiliary cells (cell.hpp:35-40).  Verified against
// baseline.cpp:76-157 by tests/test_gpu_parity.py.
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

// Occupancy of layer L from layer L+1 (grid.cpp:80-102, child-OR).
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
struct CandParams {
  const void* rows;
  const uint32_t* ids;
  const u64* count;      // |S1|
  int rho;
  const void* PM;        // layer-rho prefix-min table (u8 or u32)
  void* out_rows;
  uint32_t* out_ids;
  u64* out_fsum;
  u64* status;
  u64* claim;
  u64* out_count;        // |S2|
  u64* examined;         // points_examined (refine.cpp:90-96)
};

template <typename T, int D, typename TT, int THREADS, int PPT>
__global__ void __launch_bounds__(THREADS) k_candidates(CandParams p) {
  __shared__ unsigned scratch[PPT * (THREADS / 32) + 1];
  __shared__ u64 s_tile, s_excl;
  const u64 n = *p.count;
  constexpr u64 TILE = (u64)THREADS * PPT;
  const u64 ntiles = (n + TILE - 1) / TILE;
  if (ntiles == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *p.out_count = 0;
    return;
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
    bool keep[PPT];
    unsigned rank[PPT];
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      const u64 i = base + (u64)j * THREADS + threadIdx.x;
      keep[j] = false;
      if (i < n) {
        load_row_cached<T, D>(rows, i, v[j]);
        int col[D];
#pragma unroll
        for (int k = 0; k < D; ++k) {
          if constexpr (sizeof(T) == 4) col[k] = cell_col(v[j][k], fscale, top);
          else col[k] = cell_col(v[j][k], dscale, top);
        }
        u64 idx = 0;
        bool ok = col[0] >= 1;
#pragma unroll
        for (int k = D - 1; k >= 1; --k) {
          ok &= col[k] >= 1;
          idx = (idx << rho) | (u64)(col[k] - 1);
        }
        keep[j] = !(ok && (int64_t)PM[idx] <= (int64_t)col[0] - 1);
        examined += keep[j];
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
        p.out_fsum[o] = fsum_bits<T, D>(v[j]);
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) examined += __shfl_xor_sync(kFull, examined, o);
  if ((threadIdx.x & 31) == 0 && examined) atomicAdd(p.examined, examined);
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

// flag[i] = 1 iff no point of the set precedes point i and dominates it.
template <typename T, int D, int THREADS>
__global__ void __launch_bounds__(THREADS) k_allpairs(const T* __restrict__ rows, const uint32_t* __restrict__ ids,
                                                      const u64* __restrict__ fsum, const u64* __restrict__ count,
                                                      uint8_t* __restrict__ flag) {
  __shared__ T q_rows[THREADS * D];
  __shared__ u64 q_sum[THREADS];
  __shared__ uint32_t q_id[THREADS];
  const u64 n = *count;
  for (u64 pb = blockIdx.x; pb * THREADS < n; pb += gridDim.x) {
    const u64 i = pb * THREADS + threadIdx.x;
    T v[D];
    u64 ps = 0;
    uint32_t pid = 0;
    bool alive = i < n;
    if (alive) {
      load_row_cached<T, D>(rows, i, v);
      ps = fsum[i];
      pid = ids[i];
    }
    const bool real = alive;
    for (u64 qt = 0; qt * THREADS < n; ++qt) {
      if (!__syncthreads_or(alive)) break;
      const u64 qi = qt * THREADS + threadIdx.x;
      if (qi < n) {
        T q[D];
        load_row_cached<T, D>(rows, qi, q);
#pragma unroll
        for (int k = 0; k < D; ++k) q_rows[threadIdx.x * D + k] = q[k];
        q_sum[threadIdx.x] = fsum[qi];
        q_id[threadIdx.x] = ids[qi];
      }
      __syncthreads();
      const u64 rem = n - qt * THREADS;
      const int m = rem < THREADS ? (int)rem : THREADS;
      if (alive) {
        for (int j = 0; j < m; ++j) {
          if (precedes(q_sum[j], q_id[j], ps, pid) && dominates<T, D>(q_rows + j * D, v)) {
            alive = false;
            break;
          }
        }
      }
    }
    __syncthreads();
    if (real) flag[i] = alive ? 1 : 0;
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
