// K5 (large sets), packet form: exact sort-first dominance through the
// dominance tree, one WARP PER LEAF of query points instead of one warp per
// point.
//
// The set is in Z-order (tree.cuh builds the order); its 32-point leaves are
// the query packets.  A packet walks the tree once for all of its points:
//   * a child is entered when some undecided lane could be dominated by one
//     of its points (box lo <= p in every dimension and the child's champion
//     precedes p in the sort-first order, refine.cpp:38-41);
//   * a child strictly below p in every dimension whose champion precedes p
//     decides p at once (every point of it dominates p, dataset.hpp:55-62);
//   * a leaf is staged in shared memory and tested against all lanes: each
//     lane keeps its own point in registers and reads the 32 leaf records
//     with broadcast loads.
// Node boxes and the leaf test therefore cost a few integer ops per (lane,
// child) or (lane, point) pair: coordinates are stored as order-preserving
// integer keys (the IEEE bits of a non-negative float or double), and
//   q dominates p  <=>  OR_k (p_k - q_k) > 0   (as a signed integer)
// because the OR has its sign bit clear iff every difference is >= 0, and is
// non-zero iff some difference is > 0.  point_dominates (dataset.hpp:55-62)
// is exactly that predicate; precedes() keeps the reference's (sum, id) order.
// The node data a packet loads serves 32 points, which is what the one-warp-
// per-point tree query could not amortise (ncu: ~145 instructions and an
// L2/DRAM round trip per node visit per point).
#pragma once

#include "tree.cuh"

namespace sk {

template <typename T>
struct PkKey;
template <>
struct PkKey<float> {
  typedef uint32_t K;
  typedef int32_t S;
  // + 0.0f turns -0.0 into +0.0, so the key order is the value order
  __device__ __forceinline__ static K key(float v) { return __float_as_uint(v + 0.0f); }
};
template <>
struct PkKey<double> {
  typedef u64 K;
  typedef long long S;
  __device__ __forceinline__ static K key(double v) { return (K)__double_as_longlong(v + 0.0); }
};

// Packed records (32-bit words, padded to 16 B so they move as uint4):
//   point: key[D] | fsum (2 words) | id
//   node:  lo[D] | hi1[D] (hi + 1: strictly-below tests are >= 0 tests) | cs (2 words) | ci
template <typename T, int D>
struct PkLayout {
  typedef typename PkKey<T>::K K;
  static constexpr int KW = D * (int)sizeof(K) / 4;
  static constexpr int PW = (KW + 3 + 3) & ~3;      // point record words
  static constexpr int NW = (2 * KW + 3 + 3) & ~3;  // node record words
};

template <typename T, int D>
__device__ __forceinline__ void pk_store_point(uint32_t* __restrict__ rec, const T (&v)[D], u64 fs, uint32_t id) {
  typedef PkLayout<T, D> L;
  typename L::K kk[D];
#pragma unroll
  for (int k = 0; k < D; ++k) kk[k] = PkKey<T>::key(v[k]);
  uint32_t w[L::PW];
#pragma unroll
  for (int i = 0; i < L::PW; ++i) w[i] = 0;
  memcpy(w, kk, sizeof(kk));
  w[L::KW] = (uint32_t)fs;
  w[L::KW + 1] = (uint32_t)(fs >> 32);
  w[L::KW + 2] = id;
  uint4* o = reinterpret_cast<uint4*>(rec);
#pragma unroll
  for (int i = 0; i < L::PW / 4; ++i) o[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
}

// Sorted position j -> packed point record (Z-order, contiguous leaves).
template <typename T, int D>
__global__ void k_pk_gather(const T* __restrict__ rows, const uint32_t* __restrict__ ids, const u64* __restrict__ fsum,
                            const uint32_t* __restrict__ order, u64 m, uint32_t* __restrict__ prec) {
  pdl_enter();
  typedef PkLayout<T, D> L;
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < m; j += (u64)gridDim.x * blockDim.x) {
    const uint32_t i = order[j];
    T v[D];
    load_row_cached<T, D>(rows, i, v);
    pk_store_point<T, D>(prec + j * L::PW, v, fsum[i], ids[i]);
  }
}

template <typename K>
__device__ __forceinline__ K shfl_min(K a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const K x = __shfl_xor_sync(kFull, a, o);
    a = x < a ? x : a;
  }
  return a;
}
template <typename K>
__device__ __forceinline__ K shfl_max(K a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const K x = __shfl_xor_sync(kFull, a, o);
    a = x > a ? x : a;
  }
  return a;
}

// One warp per leaf: box (lo, hi + 1) and champion of its points.
template <typename T, int D>
__global__ void k_pk_leaves(const uint32_t* __restrict__ prec, u64 m, u64 nleaf, uint32_t* __restrict__ nrec) {
  pdl_enter();
  typedef PkLayout<T, D> L;
  typedef typename L::K K;
  const int lane = threadIdx.x & 31;
  for (u64 leaf = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; leaf < nleaf;
       leaf += ((u64)gridDim.x * blockDim.x) >> 5) {
    const u64 j = leaf * kLeaf + lane;
    const bool live = j < m;
    K kk[D];
    u64 s = ~0ull;
    uint32_t id = kNoId;
    if (live) {
      const uint32_t* r = prec + j * L::PW;
      memcpy(kk, r, sizeof(kk));
      s = (u64)r[L::KW] | ((u64)r[L::KW + 1] << 32);
      id = r[L::KW + 2];
    }
    uint32_t w[L::NW];
#pragma unroll
    for (int i = 0; i < L::NW; ++i) w[i] = 0;
    K lo[D], hi1[D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      lo[k] = shfl_min<K>(live ? kk[k] : ~(K)0);
      hi1[k] = shfl_max<K>(live ? kk[k] : (K)0) + 1;
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
    memcpy(w, lo, sizeof(lo));
    memcpy(w + L::KW, hi1, sizeof(hi1));
    w[2 * L::KW] = (uint32_t)s;
    w[2 * L::KW + 1] = (uint32_t)(s >> 32);
    w[2 * L::KW + 2] = id;
    // lanes 0 .. NW/4-1 store one uint4 each
    uint4 mine = make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int i = 0; i < L::NW / 4; ++i)
      if (lane == i) mine = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
    if (lane < L::NW / 4) reinterpret_cast<uint4*>(nrec + leaf * L::NW)[lane] = mine;
  }
}

// Level h from level h-1 (fan-out F = tree_fanout<D>()).
template <typename T, int D>
__global__ void k_pk_level(uint32_t* __restrict__ nrec, u64 child_off, u64 nchild, u64 node_off, u64 nnode) {
  pdl_enter();
  typedef PkLayout<T, D> L;
  typedef typename L::K K;
  constexpr int F = tree_fanout<D>();
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < nnode; j += (u64)gridDim.x * blockDim.x) {
    const u64 a0 = child_off + F * j;
    const int nc = (int)min((u64)F, nchild - F * j);
    K lo[D], hi1[D];
    u64 s = ~0ull;
    uint32_t id = kNoId;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      lo[k] = ~(K)0;
      hi1[k] = 0;
    }
    for (int c = 0; c < nc; ++c) {
      const uint32_t* r = nrec + (a0 + c) * L::NW;
      K l[D], h[D];
      memcpy(l, r, sizeof(l));
      memcpy(h, r + L::KW, sizeof(h));
#pragma unroll
      for (int k = 0; k < D; ++k) {
        lo[k] = l[k] < lo[k] ? l[k] : lo[k];
        hi1[k] = h[k] > hi1[k] ? h[k] : hi1[k];
      }
      const u64 cs = (u64)r[2 * L::KW] | ((u64)r[2 * L::KW + 1] << 32);
      const uint32_t ci = r[2 * L::KW + 2];
      if (key_less(cs, ci, s, id)) {
        s = cs;
        id = ci;
      }
    }
    uint32_t* o = nrec + (node_off + j) * L::NW;
    memcpy(o, lo, sizeof(lo));
    memcpy(o + L::KW, hi1, sizeof(hi1));
    o[2 * L::KW] = (uint32_t)s;
    o[2 * L::KW + 1] = (uint32_t)(s >> 32);
    o[2 * L::KW + 2] = id;
  }
}

// OR of (a_k - b_k) over the dimensions, as a signed integer: >= 0 iff a >= b
// everywhere, > 0 iff additionally a != b.
template <typename K, typename S, int D>
__device__ __forceinline__ S diff_or(const K (&a)[D], const K* b) {
  S acc = 0;
#pragma unroll
  for (int k = 0; k < D; ++k) acc |= (S)(a[k] - b[k]);
  return acc;
}

// flag[slot] = 1 iff the point at sorted position j (slot = order[j]) is not
// dominated by a preceding point of the set; only positions whose slot lies
// in [q_begin, q_end) are decided.  One warp per packet, persistent.
//
// Two phases (SKYCELL_PK_H1): phase 1 packets are the leaves; the search
// starts at the own leaf and widens through the ancestors up to level h1
// only.  Dominated points nearly always find a dominator there.  The lanes
// still undecided (mostly skyline members) are marked in umask; they are
// compacted in Z-order (list, *list_n) and re-packed 32 to a warp for phase 2,
// which searches the whole tree from the root.  Packets of members only keep
// the warp busy on points that need the full search, instead of one or two
// members holding 30 decided lanes through it.
// vstats (SKYCELL_K5STATS): [6 + 4 * phase] warps, node visits, leaf visits,
// staged leaf points.
//
// MODE 0: phase 1 (leaf packets), 1: phase 2 (list positions), 2: external
// queries -- records qrec[0 .. *list_n) in the point layout, not in the tree
// (an id of kNoId marks an inactive query); flag[e] is set for query e (the
// sparse layer-rho cell tests, sparse.cuh).
template <typename T, int D, int MODE>
__global__ void __launch_bounds__(256, 4) k_pk_query(const uint32_t* __restrict__ prec, const uint32_t* __restrict__ nrec,
                                                  const uint32_t* __restrict__ order, TreeShape sh, u64 q_begin,
                                                  const u64* __restrict__ q_end, int h1, uint32_t* __restrict__ umask,
                                                  const uint32_t* __restrict__ list, const u64* __restrict__ list_n,
                                                  const uint32_t* __restrict__ qrec, uint8_t* __restrict__ flag,
                                                  u64* __restrict__ vstats) {
  pdl_enter();
  constexpr bool PHASE2 = MODE != 0;
  typedef PkLayout<T, D> L;
  typedef typename L::K K;
  typedef typename PkKey<T>::S S;
  constexpr int F = tree_fanout<D>();
  constexpr int kStack = 32 * (F + 1);  // >= levels * F for every tree (levels <= 32)
  __shared__ uint32_t stack_s[8][kStack];
  __shared__ uint32_t path_s[8][32];
  __shared__ __align__(16) uint32_t leaf_s[8][kLeaf * L::PW];
  __shared__ __align__(16) uint32_t node_s[8][F * L::NW];
  __shared__ K pmax_s[8][D];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint32_t* stk = stack_s[wib];
  uint32_t* path = path_s[wib];
  uint32_t* lf = leaf_s[wib];
  uint32_t* nb = node_s[wib];
  K* pmax_w = pmax_s[wib];
  const u64 qend = q_end ? *q_end : ~0ull;
  const u64 npk = PHASE2 ? (*list_n + kLeaf - 1) / kLeaf : sh.nleaf;
  const u64 lcount = PHASE2 ? *list_n : 0;
  const unsigned lt = (1u << lane) - 1;
  unsigned n_nodes = 0, n_leaves = 0, n_pairs = 0;
  if (PHASE2 && lane == 0)  // no own path: nothing is skipped
    for (int l = 0; l < 32; ++l) path[l] = ~0u;
  for (u64 pk = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; pk < npk; pk += ((u64)gridDim.x * blockDim.x) >> 5) {
    u64 j = ~0ull;
    if constexpr (PHASE2) {
      const u64 e = pk * kLeaf + lane;
      if (e < lcount) j = MODE == 1 ? list[e] : e;
    } else {
      j = pk * kLeaf + lane;
    }
    uint32_t slot = 0;
    bool act = false;
    K pkk[D];
    u64 ps = 0;
    uint32_t pid = 0;
    if (j < (MODE == 2 ? lcount : sh.m)) {
      slot = MODE == 2 ? (uint32_t)j : order[j];
      const uint32_t* r = (MODE == 2 ? qrec : prec) + j * L::PW;
      memcpy(pkk, r, sizeof(pkk));
      ps = (u64)r[L::KW] | ((u64)r[L::KW + 1] << 32);
      pid = r[L::KW + 2];
      act = MODE == 2 ? pid != kNoId : slot >= q_begin && slot < qend;
      if (!PHASE2 && act && ps == 0) {  // the origin: nothing dominates it
        flag[slot] = 1;
        act = false;
      }
    } else {
#pragma unroll
      for (int k = 0; k < D; ++k) pkk[k] = 0;
    }
    bool dom = false;
    unsigned um_prev = 0;
    K pmax[D];
    u64 psmax = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) pmax[k] = 0;
    // Jump start (as tree.cuh): the own leaf first, then the ancestors
    // outwards, each expanded without the child on the own path.
    // Phase 2: if every lane comes from the subtree of one level-h1 node A,
    // phase 1 has already searched A's subtree for each of them (the packet
    // tests are exact per lane), so the search starts at A's parent and skips
    // A -- the phase-1 jump start, one level up.  Otherwise from the root.
    uint32_t anc_lo = ~0u, anc_hi = 0u;
    if (MODE == 1 && h1 >= 1 && h1 < sh.levels - 1) {
      uint32_t a = ~0u;
      if (act) {
        a = (uint32_t)(j / kLeaf);
        for (int l = 0; l < h1; ++l) a /= F;
      }
      anc_lo = a;
      anc_hi = act ? a : 0u;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        anc_lo = min(anc_lo, __shfl_xor_sync(kFull, anc_lo, o));
        anc_hi = max(anc_hi, __shfl_xor_sync(kFull, anc_hi, o));
      }
    }
    int top = 0;
    if (lane == 0) {
      if (MODE == 1 && anc_lo == anc_hi) {
        uint32_t a = anc_lo;
        for (int l = 0; l < h1; ++l) path[l] = ~0u;
        for (int l = h1; l < sh.levels; ++l) {
          path[l] = a;
          a /= F;
        }
        for (int l = sh.levels - 1; l > h1; --l) stk[top++] = ((uint32_t)l << 27) | path[l];
      } else if (PHASE2) {
        if (MODE == 1)
          for (int l = 0; l < 32; ++l) path[l] = ~0u;
        stk[top++] = ((uint32_t)(sh.levels - 1) << 27);  // the root
      } else {
        uint32_t a = (uint32_t)pk;
        for (int l = 0; l < sh.levels; ++l) {
          path[l] = a;
          a /= F;
        }
        for (int l = min(h1, sh.levels - 1); l >= 1; --l) stk[top++] = ((uint32_t)l << 27) | path[l];
        stk[top++] = (uint32_t)pk;
      }
    }
    top = __shfl_sync(kFull, top, 0);
    __syncwarp();
    while (top > 0) {
      // Packet bounds over the undecided lanes, refreshed when a lane is
      // decided: a point can dominate one of them only if it is <= their
      // componentwise maximum and its sum is <= their largest sum.
      const unsigned um = __ballot_sync(kFull, act && !dom);
      if (!um) break;
      if (um != um_prev) {
        um_prev = um;
        const bool u = (um >> lane) & 1;
#pragma unroll
        for (int k = 0; k < D; ++k) pmax[k] = shfl_max<K>(u ? pkk[k] : (K)0);
        psmax = shfl_max<u64>(u ? ps : 0ull);
        if (lane < D) pmax_w[lane] = pmax[0];
#pragma unroll
        for (int k = 1; k < D; ++k)
          if (lane == k) pmax_w[k] = pmax[k];
      }
      const uint32_t e = stk[--top];
      __syncwarp();
      const int lvl = (int)(e >> 27);
      const uint32_t idx = e & ((1u << 27) - 1);
      if (lvl == 0) {
        ++n_leaves;
        // stage the leaf points that pass the packet bounds, compacted
        const u64 q0 = (u64)idx * kLeaf;
        const int cnt = (int)min((u64)kLeaf, sh.m - q0);
        bool keep = false;
        uint4 rq[L::PW / 4];
        if (lane < cnt) {
          const uint4* src = reinterpret_cast<const uint4*>(prec + (q0 + lane) * L::PW);
#pragma unroll
          for (int i = 0; i < L::PW / 4; ++i) rq[i] = __ldg(src + i);
          K qk[D];
          memcpy(qk, rq, sizeof(qk));
          const uint32_t* w = reinterpret_cast<const uint32_t*>(rq);
          const u64 qs = (u64)w[L::KW] | ((u64)w[L::KW + 1] << 32);
          keep = qs <= psmax && diff_or<K, S, D>(pmax, qk) >= 0;
        }
        const unsigned km = __ballot_sync(kFull, keep);
        if (keep) {
          uint4* dst = reinterpret_cast<uint4*>(lf + __popc(km & lt) * L::PW);
#pragma unroll
          for (int i = 0; i < L::PW / 4; ++i) dst[i] = rq[i];
        }
        const int kc = __popc(km);
        n_pairs += kc;
        __syncwarp();
        bool d_l = false;
#pragma unroll 4
        for (int q = 0; q < kc; ++q) {
          const uint32_t* r = lf + q * L::PW;
          K qk[D];
          memcpy(qk, r, sizeof(qk));
          const u64 qs = (u64)r[L::KW] | ((u64)r[L::KW + 1] << 32);
          const uint32_t qi = r[L::KW + 2];
          // q <= p everywhere implies sum(q) <= sum(p) (monotone rounding),
          // so q precedes p unless the sums tie and q's id is larger
          d_l |= (diff_or<K, S, D>(pkk, qk) > 0) & !((qs == ps) & (qi > pid));
        }
        dom |= d_l;
        __syncwarp();
        continue;
      }
      // internal node: children F idx .. F idx + F - 1 of level lvl - 1
      ++n_nodes;
      const uint32_t cidx0 = F * idx;
      const int nc = (int)min((uint32_t)F, sh.cnt[lvl - 1] - cidx0);
      const uint32_t c0 = sh.off[lvl - 1] + cidx0;
      // the children's records are contiguous: one coalesced load by the
      // whole warp (one memory round trip per visit), then shared reads
      {
        const uint4* src = reinterpret_cast<const uint4*>(nrec + (u64)c0 * L::NW);
        uint4* dst = reinterpret_cast<uint4*>(nb);
        const int nq = nc * (L::NW / 4);
#pragma unroll
        for (int i = lane; i < F * (L::NW / 4); i += 32)
          if (i < nq) dst[i] = __ldg(src + i);
      }
      __syncwarp();
      // Packet pre-test, all children at once: lane (c, k) checks lo_k of
      // child c against the packet maximum, lane c < F the champion against
      // the packet's largest sum.  Only children passing it get the per-lane
      // test (typically 1-2 of F).
      bool rej = false;
      if (lane < F * D) {
        const int c = lane / D, k = lane - (lane / D) * D;
        K lo_k;
        memcpy(&lo_k, nb + c * L::NW + k * (int)(sizeof(K) / 4), sizeof(K));
        rej = c >= nc || lo_k > pmax_w[k];
      }
      unsigned cand = 0;
      {
        const unsigned rb = __ballot_sync(kFull, rej);
        bool crej = true;
        if (lane < nc) {
          const uint32_t* r = nb + lane * L::NW;
          const u64 cs = (u64)r[2 * L::KW] | ((u64)r[2 * L::KW + 1] << 32);
          crej = cs > psmax || ((rb >> (lane * D)) & ((1u << D) - 1)) != 0;
          // an ancestor of the own leaf skips the child on the own path
          crej |= path[lvl] == idx && cidx0 + lane == path[lvl - 1];
        }
        cand = __ballot_sync(kFull, !crej) & ((1u << F) - 1);
      }
      const bool und = act && !dom;
      unsigned wm = 0;
      u64 best_s = ~0ull;
      int best_c = 0;
      bool kill = false;
      while (cand) {
        const int c = __ffs(cand) - 1;
        cand &= cand - 1;
        const uint32_t* r = nb + c * L::NW;
        K lo[D], hi1[D];
        memcpy(lo, r, sizeof(lo));
        memcpy(hi1, r + L::KW, sizeof(hi1));
        const u64 cs = (u64)r[2 * L::KW] | ((u64)r[2 * L::KW + 1] << 32);
        const uint32_t ci = r[2 * L::KW + 2];
        // some point of the child is <= p everywhere and precedes p
        const bool want = und && precedes(cs, ci, ps, pid) && diff_or<K, S, D>(pkk, lo) >= 0;
        // the whole child lies strictly below p: its champion dominates p
        kill |= want && diff_or<K, S, D>(pkk, hi1) >= 0;
        if (__ballot_sync(kFull, want)) {
          wm |= 1u << c;
          if (cs < best_s) {
            best_s = cs;
            best_c = c;
          }
        }
      }
      dom |= kill;
      __syncwarp();  // nb is rewritten by the next visit
      if (!wm) continue;
      // push the wanted children, lane-parallel; the strongest champion on top
      const unsigned rest = wm & ~(1u << best_c);
      if ((wm >> lane) & 1)
        stk[top + (lane == best_c ? __popc(rest) : __popc(rest & lt))] = ((uint32_t)(lvl - 1) << 27) | (cidx0 + lane);
      top += __popc(wm);
      __syncwarp();
    }
    // phase 1 with a partial search: undecided lanes go to phase 2
    const bool partial = !PHASE2 && umask && h1 < sh.levels - 1;
    if (act && (dom || !partial)) flag[slot] = dom ? 0 : 1;
    if (partial) {
      const unsigned und = __ballot_sync(kFull, act && !dom);
      if (lane == 0) umask[pk] = und;
    }
    __syncwarp();
  }
  if (vstats) {
    if (lane == 0) {
      const int b = PHASE2 ? 10 : 6;
      atomicAdd(vstats + b, (u64)n_nodes);
      atomicAdd(vstats + b + 1, (u64)n_leaves);
      atomicAdd(vstats + b + 2, (u64)n_pairs);
    }
  }
}

}  // namespace sk

namespace sk {
// Phase-1 -> phase-2 compaction: per-packet undecided counts, their exclusive
// scan (CUB), then the positions of the undecided lanes in Z-order.
static __global__ void k_pk_counts(const uint32_t* __restrict__ umask, u64 npk, uint32_t* __restrict__ cnt) {
  pdl_enter();
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < npk; i += (u64)gridDim.x * blockDim.x)
    cnt[i] = __popc(umask[i]);
}
static __global__ void k_pk_list(const uint32_t* __restrict__ umask, const uint32_t* __restrict__ off, u64 npk,
                                 uint32_t* __restrict__ list, u64* __restrict__ list_n) {
  pdl_enter();
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < npk; i += (u64)gridDim.x * blockDim.x) {
    uint32_t m = umask[i];
    uint32_t o = off[i];
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      list[o++] = (uint32_t)(i * kLeaf + b);
    }
    if (i == npk - 1) *list_n = o;
  }
}
}  // namespace sk
