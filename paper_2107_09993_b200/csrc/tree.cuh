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

// Bits per dimension of the Morton key: at most 48 key bits in total (six
// 8-bit radix passes instead of eight; 2^48 cells are still far finer than
// the 32-point leaves need).
template <int D>
__host__ __device__ constexpr int morton_bits() {
  return (48 / D) < 16 ? (48 / D) : 16;
}

// Morton key of a stored row: b bits per dimension, bit j of dim k -> key
// bit j*D + k (the reference's morton_key layout, grid.cpp:18-28).
template <typename T, int D>
__device__ __forceinline__ u64 morton_of(const T (&v)[D]) {
  constexpr int B = morton_bits<D>();
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

// ---- champion prefilter (large sets).  cm[c] = min FP64 sum (its upper 32
// bits) over the set's points in cell c of a dense level-Lc grid; after a
// d-dimensional inclusive prefix-min, cm[c - 1] bounds the smallest sum among
// the points of all cells strictly below c.  Such a point q is < p in every coordinate,
// so it dominates p, and if its sum is smaller it also precedes p: p is
// removed (and may be dropped as a dominator too -- q, or whatever removed
// q, dominates everything p does).  Equal sums are left to the exact pass.
// Pass 0 uses the grid floor(v 2^L); the others grids shifted by a fraction
// of a cell, floor(v 2^L + off) (clamped), which catch dominators across the
// first grid's cell boundaries.  In each, a strictly smaller column in every
// dimension implies a strictly smaller coordinate.
template <typename T, int D>
__device__ __forceinline__ void grid_cols(const T (&v)[D], int L, int pass, int (&c)[D]) {
  const T sc = (T)(1u << L);
  // cell offsets of the passes: 0, 1/2, 1/4, 3/4, 1/8, 5/8, 3/8, 7/8 (exact in binary)
  const int o8 = pass == 0 ? 0 : pass == 1 ? 4 : pass == 2 ? 2 : pass == 3 ? 6 : pass == 4 ? 1 : pass == 5 ? 5
               : pass == 6 ? 3 : 7;
  const T off = (T)o8 * (T)0.125;
  const int top = (1 << L) - 1;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const T x = v[k] * sc + off;  // exact: power-of-two scale, +1/2 on values < 2^24
    int ci = (int)x;
    c[k] = ci < 0 ? 0 : (ci > top ? top : ci);
  }
}

// All passes in one read of the set: table t (cells entries from cm + t *
// cells) gets the min over the cell of the upper 32 bits of the points' sums
// (u32 tables: half the bytes and 32-bit atomics).  The kill test below
// stays exact: cm < hi32(s) implies the minimum sum is < s; an equal upper
// half is left to the exact pass.
template <typename T, int D>
__global__ void k_cellmin_multi(const T* __restrict__ rows, const uint32_t* __restrict__ ids,
                                const u64* __restrict__ fsum, const u64* __restrict__ count, int L, int passes,
                                u64 cells, uint32_t* __restrict__ cm) {
  pdl_enter();
  const u64 n = *count;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    if (ids[i] == kNoId) continue;
    T v[D];
    load_row_cached<T, D>(rows, i, v);
    const uint32_t s = (uint32_t)(fsum[i] >> 32);
    for (int pass = 0; pass < passes; ++pass) {
      int c[D];
      grid_cols<T, D>(v, L, pass, c);
      u64 lin = 0;
#pragma unroll
      for (int k = D - 1; k >= 0; --k) lin = (lin << L) | (u64)c[k];
      uint32_t* t = cm + pass * cells + lin;
      if (s < __ldcg(t)) atomicMin(t, s);
    }
  }
}

// A point is removed if any pass's grid has a strictly smaller sum strictly
// below its cell.
template <typename T, int D>
__global__ void k_champ_kill_multi(const T* __restrict__ rows, const uint32_t* __restrict__ ids,
                                   const u64* __restrict__ fsum, const u64* __restrict__ count, int L, int passes,
                                   u64 cells, const uint32_t* __restrict__ cm, u64 q_begin,
                                   const u64* __restrict__ q_end, uint8_t* __restrict__ kill, uint8_t* __restrict__ flag,
                                   u64* __restrict__ killed) {
  pdl_enter();
  const u64 n = *count;
  const u64 qe = q_end ? *q_end : ~0ull;
  u64 mine = 0;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    uint8_t k_i = 0;
    if (ids[i] != kNoId) {
      T v[D];
      load_row_cached<T, D>(rows, i, v);
      const uint32_t s = (uint32_t)(fsum[i] >> 32);
      for (int pass = 0; pass < passes && !k_i; ++pass) {
        int c[D];
        grid_cols<T, D>(v, L, pass, c);
        bool ok = true;
        u64 lin = 0;
#pragma unroll
        for (int k = D - 1; k >= 0; --k) {
          ok &= c[k] >= 1;
          lin = (lin << L) | (u64)(c[k] - 1);
        }
        if (ok && __ldg(cm + pass * cells + lin) < s) k_i = 1;
      }
      if (k_i) {
        ++mine;
        if (i >= q_begin && i < qe) flag[i] = 0;
      }
    }
    kill[i] = k_i;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(kFull, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(killed, mine);
}

template <typename T, int D>
__global__ void k_tree_keys(const T* __restrict__ rows, const uint32_t* __restrict__ ids, const u64* __restrict__ count,
                            const uint8_t* __restrict__ kill, u64* __restrict__ keys, uint32_t* __restrict__ vals,
                            u64* __restrict__ valid) {
  pdl_enter();
  const u64 n = *count;
  u64 mine = 0;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    u64 key = ~0ull;
    if (ids[i] != kNoId && !(kill && kill[i])) {
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
  pdl_enter();
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
  pdl_enter();
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

// Fan-out of the internal nodes: one lane per (child, dimension) pair, so a
// node visit tests all of its children's boxes with one load per lane.
template <int D>
__host__ __device__ constexpr int tree_fanout() {
  return (32 / D) < 2 ? 2 : (32 / D) > 16 ? 16 : (32 / D);
}

// Level h from level h-1: node j merges children F j .. F j + F - 1 (fewer at
// the right edge).
template <typename T, int D>
__global__ void k_tree_level(TreeView<T, D> tv, u64 child_off, u64 nchild, u64 node_off, u64 nnode) {
  pdl_enter();
  constexpr int F = tree_fanout<D>();
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < nnode; j += (u64)gridDim.x * blockDim.x) {
    const u64 a0 = child_off + F * j;
    const int nc = (int)min((u64)F, nchild - F * j);
    const u64 o = node_off + j;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      T l = tv.lo[a0 * D + k], h = tv.hi[a0 * D + k];
      for (int c = 1; c < nc; ++c) {
        const T l2 = tv.lo[(a0 + c) * D + k], h2 = tv.hi[(a0 + c) * D + k];
        l = l2 < l ? l2 : l;
        h = h2 > h ? h2 : h;
      }
      tv.lo[o * D + k] = l;
      tv.hi[o * D + k] = h;
    }
    u64 s = tv.cs[a0];
    uint32_t id = tv.ci[a0];
    for (int c = 1; c < nc; ++c)
      if (key_less(tv.cs[a0 + c], tv.ci[a0 + c], s, id)) {
        s = tv.cs[a0 + c];
        id = tv.ci[a0 + c];
      }
    tv.cs[o] = s;
    tv.ci[o] = id;
  }
}

struct TreeShape {
  u64 m, nleaf;
  int levels;                 // level 0 .. levels-1; the root is the single node of the last level
  uint32_t off[32], cnt[32];  // node offset / count per level (nodes < 2^31)
};

// flag[slot] = 1 iff the point at sorted position j (slot = order[j]) is not
// dominated by a preceding point of the set; only positions whose slot lies
// in [q_begin, q_end) are decided.  cell_level > 0: merge_cross_cell = false
// (dominators must share p's layer-rho cell; no champion short-cut).
// Internal node visit: lane l tests dimension l % D of child l / D; lanes
// c < F then hold child c's verdict.  Wanted children are pushed with the
// one lying below p in the most dimensions on top (visited next).
template <typename T, int D>
__global__ void __launch_bounds__(256) k_tree_query(const T* __restrict__ srows, const uint32_t* __restrict__ sids,
                                                    const u64* __restrict__ sfsum, const uint32_t* __restrict__ order,
                                                    TreeView<T, D> tv, TreeShape sh, u64 q_begin,
                                                    const u64* __restrict__ q_end, int cell_level,
                                                    uint8_t* __restrict__ flag, u64* __restrict__ vstats) {
  pdl_enter();
  constexpr int F = tree_fanout<D>();
  constexpr int kStack = 192;  // >= levels * (F - 1) + levels for every fan-out
  // stack entries: level << 27 | index within the level (nleaf < 2^27)
  __shared__ uint32_t stack_s[8][kStack];
  __shared__ uint32_t path_s[8][32];  // p's ancestor index per level
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint32_t* stk = stack_s[wib];
  const u64 qend = q_end ? *q_end : ~0ull;
  const int ctop = (1 << cell_level) - 1;
  const int ch = lane / D, kd = lane % D;  // (child, dimension) of this lane's box test
  const unsigned m0 = (1u << D) - 1;
  const unsigned lt = (1u << lane) - 1;
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
    unsigned n_nodes = 0, n_leaves = 0;  // SKYCELL_K5STATS diagnostics
    const uint32_t lp = (uint32_t)(j / kLeaf);  // p's own leaf
    // Jump start: dominators of p are usually near p along the Z-order, so
    // the search begins at p's own leaf and widens level by level -- the
    // stack holds p's ancestors (each to be expanded without the child on
    // p's path), root at the bottom, with p's own leaf on top.
    uint32_t* path = path_s[wib];
    int top = 0;
    if (lane == 0) {
      uint32_t a = lp;
      for (int l = 0; l < sh.levels; ++l) {
        path[l] = a;
        a /= F;
      }
      for (int l = sh.levels - 1; l >= 1; --l) stk[top++] = ((uint32_t)l << 27) | path[l];
      stk[top++] = lp;  // level 0
    }
    top = __shfl_sync(kFull, top, 0);
    __syncwarp();
    while (top > 0) {
      const uint32_t e = stk[--top];
      __syncwarp();
      const int lvl = (int)(e >> 27);
      const uint32_t idx = e & ((1u << 27) - 1);
      if (lvl == 0) {
        ++n_leaves;
        const u64 q = (u64)idx * kLeaf + lane;
        bool d_l = false;
        if (q < sh.m) {
          const u64 qs = __ldg(sfsum + q);
          const uint32_t qi = __ldg(sids + q);
          T w[D];
          load_row_cached<T, D>(srows, q, w);
          d_l = precedes(qs, qi, ps, pid) && dominates<T, D>(w, v);
          if (cell_level && d_l) d_l = same_cell<T, D>(w, v, cell_level, ctop);
        }
        if (__any_sync(kFull, d_l)) {
          dom = true;
          break;
        }
        continue;
      }
      // internal node: children F idx .. F idx + F - 1 of level lvl - 1
      ++n_nodes;
      const uint32_t cidx0 = F * idx;
      const int nc = (int)min((uint32_t)F, sh.cnt[lvl - 1] - cidx0);
      const uint32_t c0 = sh.off[lvl - 1] + cidx0;
      bool lo_ok = true, hi_lt = false;
      if (ch < nc) {
        const uint32_t c = c0 + ch;
        lo_ok = __ldg(tv.lo + (u64)c * D + kd) <= pk;
        hi_lt = __ldg(tv.hi + (u64)c * D + kd) < pk;
      }
      const unsigned lo_bad = __ballot_sync(kFull, !lo_ok), hi_in = __ballot_sync(kFull, hi_lt);
      // lanes c < nc: verdict for child c
      bool want = false, kill = false;
      int score = -1;
      // an ancestor of p's leaf (jump start) skips the child on p's path:
      // that subtree has been searched already
      const uint32_t own = path[lvl - 1];  // p's ancestor at level lvl - 1
      const bool ancestor = path[lvl] == idx;
      if (lane < nc && !(ancestor && cidx0 + lane == own)) {
        const u64 cs = __ldg(tv.cs + c0 + lane);
        const uint32_t ci = __ldg(tv.ci + c0 + lane);
        const unsigned in_c = (hi_in >> (lane * D)) & m0;
        want = !((lo_bad >> (lane * D)) & m0) && cs <= ps;
        kill = want && !cell_level && in_c == m0 && precedes(cs, ci, ps, pid);
        score = want ? __popc(in_c) : -1;
      }
      if (__any_sync(kFull, kill)) {
        // a child strictly below p in every dimension whose champion
        // precedes p: every point of it dominates p
        dom = true;
        break;
      }
      const unsigned wm = __ballot_sync(kFull, want);
      if (!wm) continue;
      // best child: highest score, ties to the lowest lane
      int best = (score << 5) | (31 - lane);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(kFull, best, o));
      const int bl = 31 - (best & 31);
      const unsigned rest = wm & ~(1u << bl);
      if (want) {
        const uint32_t ent = ((uint32_t)(lvl - 1) << 27) | (cidx0 + lane);
        stk[top + (lane == bl ? __popc(rest) : __popc(rest & lt))] = ent;
      }
      top += __popc(wm);
      __syncwarp();
    }
    if (lane == 0) flag[slot] = dom ? 0 : 1;
    if (vstats && lane == 0) {
      atomicAdd(vstats + (dom ? 0 : 3), 1ull);
      atomicAdd(vstats + (dom ? 1 : 4), (u64)n_nodes);
      atomicAdd(vstats + (dom ? 2 : 5), (u64)n_leaves);
    }
    __syncwarp();
  }
}

}  // namespace sk
