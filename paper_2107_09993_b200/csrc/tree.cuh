// K5 (large sets): exact sort-first dominance through a dominance tree.
//
// The set's points are ordered along a Z-order (Morton) curve and cut into
// leaves of 32 consecutive points; an implicit complete binary tree over the
// leaves stores, per node, the bounding box of its points and its
// *champion* -- the point that comes first in the sort-first order
// (ascending FP64 sum, ties by record id; refine.cpp:38-41).
//
// p is dominated in the reference's sense (some q precedes p and
// point_dominates(q, p), dataset.hpp:55-62) iff a traversal finds such a q:
//   * a node whose box has lo_k > p_k in some k holds no point <= p: skipped;
//   * a node whose champion sum exceeds p's sum holds nothing preceding p:
//     skipped;
//   * a node whose box has hi_k < p_k in EVERY k holds only points strictly
//     below p, all of which dominate p; p is dominated iff its champion
//     precedes p (the champion precedes every other point of the node);
//   * a leaf is tested point by point, one point per lane.
// So skyline points pay only for the nodes straddling the boundary of their
// dominance orthant, instead of a scan over a candidate list: this is what
// makes anti-correlated data (skyline = 20-75% of n) tractable.
// One warp per query point, queries visited in Z-order so neighbouring warps
// walk similar paths; children are visited strongest (smallest champion sum)
// first.
#pragma once

#include "kernels.cuh"

namespace sk {

constexpr int kLeaf = 32;

// Morton key of a stored row: b bits per dimension, bit j of dim k -> key
// bit j*D + k (the reference's morton_key layout, grid.cpp:18-28).
template <typename T, int D>
__device__ __forceinline__ u64 morton_of(const T (&v)[D]) {
  constexpr int B = (64 / D) < 16 ? (64 / D) : 16;
  u64 key = 0;
  int col[D];
#pragma unroll
  for (int k = 0; k < D; ++k) col[k] = cell_col(v[k], (T)(1u << B), (1 << B) - 1);
#pragma unroll
  for (int j = B - 1; j >= 0; --j)
#pragma unroll
    for (int k = D - 1; k >= 0; --k) key = (key << 1) | (u64)((col[k] >> j) & 1);
  return key;
}

template <typename T, int D>
__global__ void k_tree_keys(const T* __restrict__ rows, const uint32_t* __restrict__ ids, const u64* __restrict__ count,
                            u64* __restrict__ keys, uint32_t* __restrict__ vals, u64* __restrict__ valid) {
  const u64 n = *count;
  u64 mine = 0;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    u64 key = ~0ull;
    if (ids[i] != kNoId) {
      T v[D];
      load_row_cached<T, D>(rows, i, v);
      key = morton_of<T, D>(v) >> 1;  // < ~0: valid slots sort before empty ones
      ++mine;
    }
    keys[i] = key;
    vals[i] = (uint32_t)i;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(kFull, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(valid, mine);
}

// Sorted position j -> point data in Z-order (contiguous leaves).
template <typename T, int D>
__global__ void k_tree_gather(const T* __restrict__ rows, const uint32_t* __restrict__ ids, const u64* __restrict__ fsum,
                              const uint32_t* __restrict__ order, u64 m, T* __restrict__ srows,
                              uint32_t* __restrict__ sids, u64* __restrict__ sfsum) {
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < m; j += (u64)gridDim.x * blockDim.x) {
    const uint32_t i = order[j];
    T v[D];
    load_row_cached<T, D>(rows, i, v);
    store_row<T, D>(srows, j, v);
    sids[j] = ids[i];
    sfsum[j] = fsum[i];
  }
}

// Node arrays (flat, level by level; level 0 = leaves):
//   lo/hi  [node][D]   bounding box
//   cs     [node]      champion sum bits (~0 for an empty node)
//   ci     [node]      champion record id
template <typename T, int D>
struct TreeView {
  T* lo;
  T* hi;
  u64* cs;
  uint32_t* ci;
};

__device__ __forceinline__ bool key_less(u64 as, uint32_t ai, u64 bs, uint32_t bi) {
  return as < bs || (as == bs && ai < bi);
}

// One warp per leaf: box and champion of its (up to) 32 points.
template <typename T, int D>
__global__ void k_tree_leaves(const T* __restrict__ srows, const uint32_t* __restrict__ sids,
                              const u64* __restrict__ sfsum, u64 m, u64 nleaf, TreeView<T, D> tv) {
  const int lane = threadIdx.x & 31;
  for (u64 leaf = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; leaf < nleaf;
       leaf += ((u64)gridDim.x * blockDim.x) >> 5) {
    const u64 j = leaf * kLeaf + lane;
    const bool live = j < m;
    T v[D];
    u64 s = ~0ull;
    uint32_t id = kNoId;
    if (live) {
      load_row_cached<T, D>(srows, j, v);
      s = sfsum[j];
      id = sids[j];
    }
#pragma unroll
    for (int k = 0; k < D; ++k) {
      T a = live ? v[k] : (T)3, b = live ? v[k] : (T)-3;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const T x = __shfl_xor_sync(kFull, a, o), y = __shfl_xor_sync(kFull, b, o);
        a = x < a ? x : a;
        b = y > b ? y : b;
      }
      if (lane == 0) {
        tv.lo[leaf * D + k] = a;
        tv.hi[leaf * D + k] = b;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const u64 xs = __shfl_xor_sync(kFull, s, o);
      const uint32_t xi = __shfl_xor_sync(kFull, id, o);
      if (key_less(xs, xi, s, id)) {
        s = xs;
        id = xi;
      }
    }
    if (lane == 0) {
      tv.cs[leaf] = s;
      tv.ci[leaf] = id;
    }
  }
}

// Level h from level h-1: node j merges children 2j and 2j+1 (the second
// may be missing at the right edge).
template <typename T, int D>
__global__ void k_tree_level(TreeView<T, D> tv, u64 child_off, u64 nchild, u64 node_off, u64 nnode) {
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < nnode; j += (u64)gridDim.x * blockDim.x) {
    const u64 a = child_off + 2 * j, b = child_off + 2 * j + 1;
    const bool hb = 2 * j + 1 < nchild;
    const u64 o = node_off + j;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      T l = tv.lo[a * D + k], h = tv.hi[a * D + k];
      if (hb) {
        const T l2 = tv.lo[b * D + k], h2 = tv.hi[b * D + k];
        l = l2 < l ? l2 : l;
        h = h2 > h ? h2 : h;
      }
      tv.lo[o * D + k] = l;
      tv.hi[o * D + k] = h;
    }
    u64 s = tv.cs[a];
    uint32_t id = tv.ci[a];
    if (hb && key_less(tv.cs[b], tv.ci[b], s, id)) {
      s = tv.cs[b];
      id = tv.ci[b];
    }
    tv.cs[o] = s;
    tv.ci[o] = id;
  }
}

struct TreeShape {
  u64 m, nleaf;
  int levels;            // level 0 .. levels-1; the root is the single node of the last level
  u64 off[48], cnt[48];  // node offset / count per level
};

// flag[slot] = 1 iff the point at sorted position j (slot = order[j]) is not
// dominated by a preceding point of the set; only positions whose slot lies
// in [q_begin, q_end) are decided.  cell_level > 0: merge_cross_cell = false
// (dominators must share p's layer-rho cell; no champion short-cut).
template <typename T, int D>
__global__ void __launch_bounds__(256) k_tree_query(const T* __restrict__ srows, const uint32_t* __restrict__ sids,
                                                    const u64* __restrict__ sfsum, const uint32_t* __restrict__ order,
                                                    TreeView<T, D> tv, TreeShape sh, u64 q_begin,
                                                    const u64* __restrict__ q_end, int cell_level,
                                                    uint8_t* __restrict__ flag) {
  constexpr int kStack = 64;
  // stack entries: level << 27 | index within the level (nleaf < 2^27)
  __shared__ uint32_t stack_s[8][kStack];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint32_t* stk = stack_s[wib];
  const u64 qend = q_end ? *q_end : ~0ull;
  const int ctop = (1 << cell_level) - 1;
  const int ch = lane / D, kd = lane % D;  // lanes [0, D): child 0 dims; [D, 2D): child 1 dims
  const unsigned m0 = (1u << D) - 1;
  for (u64 j = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; j < sh.m; j += ((u64)gridDim.x * blockDim.x) >> 5) {
    const uint32_t slot = order[j];
    if (slot < q_begin || slot >= qend) continue;
    const u64 ps = sfsum[j];
    const uint32_t pid = sids[j];
    if (ps == 0) {  // the origin: nothing dominates it
      if (lane == 0) flag[slot] = 1;
      continue;
    }
    T v[D];
    load_row_cached<T, D>(srows, j, v);
    T pk = v[0];
#pragma unroll
    for (int k = 1; k < D; ++k)
      if (kd == k) pk = v[k];
    bool dom = false;
    if (lane == 0) stk[0] = (uint32_t)(sh.levels - 1) << 27;
    int top = 1;
    __syncwarp();
    while (top > 0 && !dom) {
      const uint32_t e = stk[--top];
      __syncwarp();
      const int lvl = (int)(e >> 27);
      const u64 idx = e & ((1u << 27) - 1);
      if (lvl == 0) {
        const u64 q = idx * kLeaf + lane;
        bool d_l = false;
        if (q < sh.m) {
          const u64 qs = __ldg(sfsum + q);
          if (qs <= ps) {
            T w[D];
            load_row_cached<T, D>(srows, q, w);
            d_l = precedes(qs, __ldg(sids + q), ps, pid) && dominates<T, D>(w, v);
            if (cell_level && d_l) d_l = same_cell<T, D>(w, v, cell_level, ctop);
          }
        }
        dom = __any_sync(kFull, d_l);
        continue;
      }
      // internal node: children 2 idx, 2 idx + 1 of level lvl - 1
      const u64 ci0 = 2 * idx;
      const bool has1 = ci0 + 1 < sh.cnt[lvl - 1];
      const u64 c0 = sh.off[lvl - 1] + ci0;
      bool lo_ok = true, hi_lt = true;
      if (ch < 2 && (ch == 0 || has1)) {
        const u64 c = c0 + ch;
        lo_ok = __ldg(tv.lo + c * D + kd) <= pk;
        hi_lt = __ldg(tv.hi + c * D + kd) < pk;
      }
      const unsigned lo_bad = __ballot_sync(kFull, !lo_ok), hi_in = __ballot_sync(kFull, hi_lt && ch < 2);
      const u64 s0 = __ldg(tv.cs + c0), s1 = has1 ? __ldg(tv.cs + c0 + 1) : ~0ull;
      const uint32_t i0 = __ldg(tv.ci + c0), i1 = has1 ? __ldg(tv.ci + c0 + 1) : kNoId;
      const unsigned in0 = hi_in & m0, in1 = (hi_in >> D) & m0;
      const bool want0 = !(lo_bad & m0) && s0 <= ps;
      const bool want1 = has1 && !((lo_bad >> D) & m0) && s1 <= ps;
      // a child strictly below p in every dimension: its champion decides
      if (!cell_level && ((want0 && in0 == m0 && precedes(s0, i0, ps, pid)) ||
                          (want1 && in1 == m0 && precedes(s1, i1, ps, pid)))) {
        dom = true;
        break;
      }
      // visit first the child lying below p in more dimensions (more likely
      // to hold a dominator), ties: the stronger champion
      const int n0 = __popc(in0), n1 = __popc(in1);
      const bool first1 = want0 && want1 && (n1 > n0 || (n1 == n0 && key_less(s1, i1, s0, i0)));
      const uint32_t e0 = ((uint32_t)(lvl - 1) << 27) | (uint32_t)ci0, e1 = e0 + 1;
      if (lane == 0) {
        int t = top;
        if (first1) {
          stk[t++] = e0;
          stk[t++] = e1;
        } else {
          if (want1) stk[t++] = e1;
          if (want0) stk[t++] = e0;
        }
      }
      top += (int)want0 + (int)want1;
      __syncwarp();
    }
    if (lane == 0) flag[slot] = dom ? 0 : 1;
    __syncwarp();
  }
}

}  // namespace sk
