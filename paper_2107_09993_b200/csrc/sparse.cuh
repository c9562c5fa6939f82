// Sparse layer rho (rho*d > 36 or rho*(d-1) > 30): the reference keeps layer
// rho as a hash map of the non-empty cells (grid.hpp:67, filled at
// grid.cpp:74) and accepts any rho with rho*d <= 60, (rho-1)*d <= 32
// (grid.cpp:38-43); a dense 2^(rho d)-bit bitmap does not fit there.
//
// Layers 1..rho-1 stay dense ((rho-1) d <= 32: at most a 512 MB bitmap).  The
// points in layer-(rho-1) candidate cells (K4's cell test one layer down) are
// a superset of the points in layer-rho candidate cells: a child of a
// strictly dominated cell is strictly dominated.  Their layer-rho cells are
// sorted and made unique -- U, the children of CS_(rho-1) that hold a point
// (split_candidates, shrink_par.cpp:8-24) -- and classified with the K5
// dominance tree built over U, the cells placed at their corners c / 2^rho:
//   key[c]  <=> no other cell of U is <= c (point dominance of the corners)
//               and c has no top column (shrink_par.cpp:235-241);
//   cand[c] <=> no cell of U is <= c - 1 in every dimension: the corner
//               query c / 2^rho - 2^-(rho+1) (half a cell below) is dominated
//               exactly by the corners of the cells strictly below c.
// Restricting both tests to U is exact: a cell strictly below (or below) a
// member of U has an occupied parent that is not strictly dominated (else
// the member's parent would be), so it lies in U itself.
// points_examined = the points of U's candidate cells (refine.cpp:90-96).
#pragma once

#include "packet.cuh"

namespace sk {

// Layer-rho linear index (dim d-1 most significant, cell.hpp:102-107) of
// every valid slot; empty slots sort last.
template <typename T, int D>
__global__ void k_sp_keys(const T* __restrict__ rows, const uint32_t* __restrict__ ids, const u64* __restrict__ count,
                          int rho, u64* __restrict__ keys, uint32_t* __restrict__ vals) {
  pdl_enter();
  const u64 n = *count;
  const int top = (1 << rho) - 1;
  const T scale = (T)(1u << rho);
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    u64 key = ~0ull;
    if (ids[i] != kNoId) {
      T v[D];
      load_row_cached<T, D>(rows, i, v);
      key = 0;
#pragma unroll
      for (int k = D - 1; k >= 0; --k) key = (key << rho) | (u64)cell_col(v[k], scale, top);
    }
    keys[i] = key;
    vals[i] = (uint32_t)i;
  }
}

static __global__ void k_sp_heads(const u64* __restrict__ keys, u64 n, uint32_t* __restrict__ head) {
  pdl_enter();
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < n; j += (u64)gridDim.x * blockDim.x)
    head[j] = keys[j] != ~0ull && (j == 0 || keys[j] != keys[j - 1]);
}

// One point per distinct cell (its corner c / 2^rho, exact in f32 for
// rho <= 17), the cell's first sorted position, and the cell count.
template <int D>
__global__ void k_sp_cells(const u64* __restrict__ keys, const uint32_t* __restrict__ head,
                           const uint32_t* __restrict__ cpos, u64 n, int rho, float* __restrict__ crows,
                           u64* __restrict__ cfsum, uint32_t* __restrict__ cids, uint32_t* __restrict__ cstart,
                           u64* __restrict__ ncells, u64* __restrict__ nvalid) {
  pdl_enter();
  const u64 mask = (1ull << rho) - 1;
  const float inv = ldexpf(1.0f, -rho);
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < n; j += (u64)gridDim.x * blockDim.x) {
    const u64 key = keys[j];
    if (key == ~0ull) continue;
    if (j + 1 == n || keys[j + 1] == ~0ull) {  // the last valid position
      *ncells = cpos[j];
      *nvalid = j + 1;
    }
    if (!head[j]) continue;
    const uint32_t c = cpos[j] - 1;
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const float x = (float)((key >> (rho * k)) & mask) * inv;
      crows[(u64)c * D + k] = x;
      s = __dadd_rn(s, (double)x);
    }
    cfsum[c] = (u64)__double_as_longlong(s);
    cids[c] = c;
    cstart[c] = (uint32_t)j;
  }
}

// External queries for the strict test: the corner of every tree cell moved
// half a cell down (exact), inactive (id kNoId) when a column is 0 -- such a
// cell has nothing strictly below it.
template <int D>
__global__ void k_sp_queries(const uint32_t* __restrict__ prec, u64 m, int rho, uint32_t* __restrict__ qrec) {
  pdl_enter();
  typedef PkLayout<float, D> L;
  const float half = ldexpf(1.0f, -(rho + 1));
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < m; j += (u64)gridDim.x * blockDim.x) {
    const uint32_t* r = prec + j * L::PW;
    float v[D];
    bool ok = true;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const float x = __uint_as_float(r[k]);
      ok &= x > 0.0f;
      v[k] = x - half;
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) s = __dadd_rn(s, (double)v[k]);
    pk_store_point<float, D>(qrec + j * L::PW, v, (u64)__double_as_longlong(s), ok ? r[L::KW + 2] : kNoId);
  }
}

// Per tree position j: cand flag of cell order[j] (queries with an inactive
// record -- a zero column -- are candidates: nothing is strictly below).
static __global__ void k_sp_cand(const uint8_t* __restrict__ qflag, const uint32_t* __restrict__ qrec_ids, int pw,
                                 const uint32_t* __restrict__ order, u64 m, uint8_t* __restrict__ cand) {
  pdl_enter();
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < m; j += (u64)gridDim.x * blockDim.x) {
    const bool inactive = qrec_ids[j * pw] == kNoId;
    cand[order[j]] = inactive ? 1 : qflag[j];
  }
}

// Layer-rho counts and points_examined from the per-cell flags.
template <int D>
__global__ void k_sp_classify(const float* __restrict__ crows, const uint8_t* __restrict__ keyf,
                              const uint8_t* __restrict__ cand, const uint32_t* __restrict__ cstart,
                              const u64* __restrict__ ncells, const u64* __restrict__ nvalid, int rho,
                              u64* __restrict__ n_key, u64* __restrict__ n_cand, u64* __restrict__ examined) {
  pdl_enter();
  const u64 nc = *ncells;
  const float topv = (float)((1 << rho) - 1) * ldexpf(1.0f, -rho);
  u64 a = 0, b = 0, e = 0;
  for (u64 c = blockIdx.x * (u64)blockDim.x + threadIdx.x; c < nc; c += (u64)gridDim.x * blockDim.x) {
    bool has_top = false;
#pragma unroll
    for (int k = 0; k < D; ++k) has_top |= crows[c * D + k] == topv;
    a += keyf[c] && !has_top;
    if (cand[c]) {
      ++b;
      e += (c + 1 < nc ? (u64)cstart[c + 1] : *nvalid) - cstart[c];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(kFull, a, o);
    b += __shfl_xor_sync(kFull, b, o);
    e += __shfl_xor_sync(kFull, e, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (a) atomicAdd(n_key, a);
    if (b) atomicAdd(n_cand, b);
    if (e) atomicAdd(examined, e);
  }
}

// The points of candidate cells -> an unordered stream (per-warp chunks).
template <typename T, int D>
__global__ void k_sp_points(const T* __restrict__ rows, const uint32_t* __restrict__ ids, const u64* __restrict__ fsum,
                            const uint32_t* __restrict__ vals, const u64* __restrict__ keys,
                            const uint32_t* __restrict__ cpos, const uint8_t* __restrict__ cand, u64 n,
                            T* __restrict__ out_rows, uint32_t* __restrict__ out_ids, u64* __restrict__ out_fsum,
                            u64* __restrict__ out_reserved, unsigned chunk) {
  pdl_enter();
  const u64 gw = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5;
  const u64 nw = ((u64)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  WarpOut wo{0, chunk, chunk};
  auto stamp = [&](u64 slot) { out_ids[slot] = kNoId; };
  for (u64 base = gw * 32; base < n; base += nw * 32) {
    const u64 j = base + lane;
    bool keep = false;
    uint32_t i = 0;
    if (j < n && keys[j] != ~0ull) {
      i = vals[j];
      keep = cand[cpos[j] - 1] != 0;
    }
    if (__any_sync(kFull, keep)) {
      const u64 o = warp_reserve(wo, keep, out_reserved, stamp);
      if (keep) {
        T v[D];
        load_row_cached<T, D>(rows, i, v);
        store_row<T, D>(out_rows, o, v);
        out_ids[o] = ids[i];
        out_fsum[o] = fsum[i];
      }
    }
  }
  warp_close(wo, stamp);
}

}  // namespace sk
