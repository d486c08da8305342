// exact_impl.cuh -- the reference's exact recursion, level-synchronously.
//
// The fast sort (sort_impl.cuh) produces the reference's OUTPUT whenever the
// order of equal sort keys is unobservable (full-width keys-only words), and
// its baseline Metrics by a closed form.  Everything else the reference
// defines depends on the exact two-cursor permutation of every partition:
//
//   * the tie order of UnsignedCodec(w) on wider words and of sub-range sorts
//     from start_pos > 0 (keys equal in the examined bits, different above);
//   * the sortedness scan of sort_optimized (kernels.py:107-119), which looks
//     at the range's CURRENT (partially partitioned) content;
//   * the counters of sort_optimized (pass-through loop: no call, no depth),
//     of sort_words_iterative (calls = partitions, max_depth = stack
//     high-water mark, kernels.py:129-172), of sort_parallel's prepartition
//     (variants.py:124-148) and of the level observer (core.py:146-180).
//
// This engine replays the recursion breadth-first.  Every call of the
// reference recursion works on a disjoint index range, so running all ranges
// of one bit position together gives exactly the same array states as the
// depth-first order.  Per level (bit `pos`):
//
//   check   (optional) sortedness of flagged segments, on the current buffer
//   count   zeros of live elements per 4096-element chunk  -> scan
//   bounds  global zero prefix G at each live segment's first/last element
//   plan    one thread per segment start: resolve a pending check, count
//           extractions/swaps/calls/depth, emit the children (ping-pong
//           segment tables indexed by start position: no allocation, no scan)
//   index   L-one ranks and R-zero ranks
//   gather  each live position takes its element from the closed form of the
//           two-cursor loop (kernels.py:56-77), values alongside; segment ids
//           become the children's start positions
//
// Segments that finish (size < 2, pos == width, sorted) stop moving; a final
// pass copies each one from the buffer it ended in.  Keys are read through
// the codec on the fly (enc()), so raw words -- including bits above `width`
// -- are moved untouched.
#pragma once

#include "misc_impl.cuh"

namespace bs {
namespace ex {

constexpr int EX_BLOCK = 256, EX_IPT = 16, EX_CHUNK = EX_BLOCK * EX_IPT;

enum : uint32_t { F_ACTIVE = 1u, F_CHECK = 2u, F_UNSORTED = 4u, F_CHECKED = 8u, F_DEFER = 16u, F_HOME = 32u };
enum { M_REC = 0, M_ITER = 1, M_LEVELS = 2, M_PAR = 3 };

// One segment, stored at its start position.  flags: bits 0-7 F_*, 8-15 the
// pass-through streak, 16-23 the call depth relative to depth0, 24-31 the
// iterative form's pending-stack count P.
struct SegT {
  uint32_t count, flags, g0, g1;
};

__host__ __device__ __forceinline__ uint32_t pack(uint32_t bits, uint32_t streak, uint32_t dep, uint32_t P) {
  return (bits & 0xFFu) | (min(streak, 255u) << 8) | ((dep & 0xFFu) << 16) | ((P & 0xFFu) << 24);
}

// a live segment is partitioned at this level: active, and not stopped by a
// sortedness scan that found it sorted
__device__ __forceinline__ bool alive(uint32_t f) {
  return (f & F_ACTIVE) && !((f & F_CHECK) && !(f & F_UNSORTED));
}

struct Ex {
  void *keys[2];  // [0] caller's buffer, [1] workspace copy
  void *vals[2];
  uint32_t *seg;   // per element: start position of its segment
  SegT *tab[2];    // per start position, ping-pong by level parity
  uint32_t *lone;  // per segment, at start + rank: L-one offsets
  uint32_t *zpos;  // per segment, at start + rank: R-zero offsets
  uint32_t *bcnt;  // per chunk zero counts, then exclusive prefix
  unsigned long long *ctr;  // reference counters {extractions, swaps, calls, max_depth}
  uint64_t n;
  int64_t depth0;
  int width, kind, mode, loop, check_after, par_levels;
};

// Codec encoding of a raw word (keys.py:51-93): the key is the low `width`
// bits of the result.  Unsigned words are compared whole (the reference's
// range_sorted_words compares raw words, kernels.py:80-85).
template <typename K>
__device__ __forceinline__ uint64_t enc(const Ex &e, K x) {
  uint64_t v = uint64_t(x);
  if (e.kind == 1) {
    const uint64_t full = e.width >= 64 ? ~0ull : ((1ull << e.width) - 1ull);
    v = (v & full) ^ (1ull << (e.width - 1));
  } else if (e.kind == 2) {
    v = (v >> 63) ? ~v : (v | (1ull << 63));
  }
  return v;
}

// (enc(x) << pos) & (1 << (width-1))  (kernels.py:63,69)
template <typename K>
__device__ __forceinline__ uint32_t bitof(const Ex &e, K x, int pos) {
  return ((enc(e, x) << pos) >> (e.width - 1)) & 1u;
}

__global__ void ex_init_kernel(Ex e, SegT root) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < e.n; i += uint64_t(gridDim.x) * blockDim.x)
    e.seg[i] = 0u;
  if (blockIdx.x == 0 && threadIdx.x == 0) e.tab[0][0] = root;
}

// Sortedness scan of every segment carrying F_CHECK: one adjacent pair per
// thread; a decreasing pair marks the segment F_UNSORTED (one atomic per
// warp and segment).
template <typename K>
__global__ void ex_check_kernel(Ex e, int par, int cur) {
  const K *k = static_cast<const K *>(e.keys[par]);
  const SegT *tab = e.tab[cur];
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  uint32_t s = 0xFFFFFFFFu;
  bool viol = false;
  if (i < e.n) {
    s = e.seg[i];
    const SegT t = tab[s];
    if ((t.flags & F_CHECK) && !(t.flags & F_UNSORTED) && i + 1 < uint64_t(s) + t.count)
      viol = enc(e, k[i]) > enc(e, k[i + 1]);
    if (!(t.flags & F_CHECK)) s = 0xFFFFFFFFu;
  }
  const uint32_t grp = __match_any_sync(0xFFFFFFFFu, s);
  const uint32_t any = __ballot_sync(0xFFFFFFFFu, viol) & grp;
  if (any && (threadIdx.x & 31) == uint32_t(__ffs(grp) - 1) && s != 0xFFFFFFFFu)
    atomicOr(&e.tab[cur][s].flags, F_UNSORTED);
}

// Per-thread view of its 16 consecutive elements: segment, liveness, bit.
struct Elem {
  uint32_t s[EX_IPT];
  uint32_t live, bits;  // masks over the 16 elements
};

template <typename K>
__device__ __forceinline__ void load_elems(const Ex &e, const K *k, int pos, int cur, uint64_t base, Elem &el) {
  el.live = el.bits = 0;
  uint32_t ps = 0xFFFFFFFFu, pf = 0;
  const SegT *tab = e.tab[cur];
#pragma unroll
  for (int j = 0; j < EX_IPT; ++j) {
    const uint64_t i = base + j;
    el.s[j] = 0;
    if (i < e.n) {
      const uint32_t s = e.seg[i];
      if (s != ps) {
        ps = s;
        pf = tab[s].flags;
      }
      el.s[j] = s;
      if (alive(pf)) {
        el.live |= 1u << j;
        el.bits |= bitof(e, k[i], pos) << j;
      }
    }
  }
}

template <typename K>
__global__ void __launch_bounds__(EX_BLOCK) ex_count_kernel(Ex e, int pos, int par, int cur) {
  __shared__ uint32_t sw[EX_BLOCK / 32];
  const K *k = static_cast<const K *>(e.keys[par]);
  Elem el;
  load_elems(e, k, pos, cur, uint64_t(blockIdx.x) * EX_CHUNK + uint64_t(threadIdx.x) * EX_IPT, el);
  uint32_t z = __popc(el.live & ~el.bits);
  for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xFFFFFFFFu, z, o);
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = z;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < EX_BLOCK / 32; ++w) t += sw[w];
    e.bcnt[blockIdx.x] = t;
  }
}

// G of the thread's first element: chunk prefix + block-exclusive prefix.
__device__ __forceinline__ uint32_t thread_prefix(const Ex &e, uint32_t zeros, uint32_t *sw) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t incl = zeros;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) sw[w] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t acc = 0;
    for (int i = 0; i < EX_BLOCK / 32; ++i) {
      const uint32_t t = sw[i];
      sw[i] = acc;
      acc += t;
    }
  }
  __syncthreads();
  return e.bcnt[blockIdx.x] + sw[w] + incl - zeros;
}

template <typename K>
__global__ void __launch_bounds__(EX_BLOCK) ex_bounds_kernel(Ex e, int pos, int par, int cur) {
  __shared__ uint32_t sw[EX_BLOCK / 32];
  const K *k = static_cast<const K *>(e.keys[par]);
  const uint64_t base = uint64_t(blockIdx.x) * EX_CHUNK + uint64_t(threadIdx.x) * EX_IPT;
  Elem el;
  load_elems(e, k, pos, cur, base, el);
  uint32_t G = thread_prefix(e, __popc(el.live & ~el.bits), sw);
  SegT *tab = e.tab[cur];
#pragma unroll
  for (int j = 0; j < EX_IPT; ++j) {
    if ((el.live >> j) & 1u) {
      const uint64_t i = base + j;
      const uint32_t s = el.s[j];
      const uint32_t zero = ((el.bits >> j) & 1u) ^ 1u;
      if (i == s) tab[s].g0 = G;
      if (i == uint64_t(s) + tab[s].count - 1) tab[s].g1 = G + zero;
      G += zero;
    }
  }
}

// One thread per position; segment starts (seg[i] == i) plan their level.
__global__ void __launch_bounds__(256) ex_plan_kernel(Ex e, int L, int pos, int cur) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  unsigned long long extr = 0, swaps = 0, calls = 0;
  uint32_t maxd = 0;  // absolute depth / high-water candidate (+1 so 0 means none)
  if (i < e.n && e.seg[i] == uint32_t(i)) {
    const SegT *A = e.tab[cur];
    SegT *B = e.tab[cur ^ 1];
    const SegT t = A[i];
    const uint32_t cnt = t.count;
    uint32_t bits = t.flags & 0xFFu;
    const uint32_t streak = (t.flags >> 8) & 0xFFu, dep = (t.flags >> 16) & 0xFFu, P = t.flags >> 24;
    const uint32_t p = uint32_t(L) & 1u;
    auto depth_abs = [&](uint32_t d) { return uint32_t(e.depth0 + int64_t(d)) + 1u; };
    // a pending sortedness scan (ran on buffer p, before this partition)
    if (bits & F_CHECK) {
      const bool sorted = !(bits & F_UNSORTED);
      if (e.mode == M_REC && (bits & F_DEFER) && !sorted) {  // the deferred pass-through call
        calls += 1;
        maxd = max(maxd, depth_abs(dep));
      }
      bits &= ~(F_CHECK | F_UNSORTED | F_DEFER);
      if (sorted) bits = (bits & ~(F_ACTIVE | F_HOME)) | (p ? F_HOME : 0u);
    }
    const uint32_t stop = (bits & ~(F_ACTIVE | F_HOME)) | (p ? 0u : F_HOME);  // home after this level: p^1
    if (!(bits & F_ACTIVE)) {
      B[i] = SegT{cnt, pack(bits, streak, dep, P), 0, 0};
    } else {
      const uint32_t Z = t.g1 - t.g0;
      extr += cnt;
      swaps += cnt - Z;
      const bool pass = (Z == 0u || Z == cnt);
      const bool last = (pos + 1 == e.width);
      const uint32_t lo_n = Z, up_n = cnt - Z;
      const uint64_t up_s = i + Z;
      const int mode = (e.mode == M_PAR && L >= e.par_levels) ? M_REC : e.mode;
      if (mode == M_REC) {
        if (pass) {
          const uint32_t ns = min(streak + 1u, 255u);
          const bool chk = e.check_after > 0 && ns >= uint32_t(e.check_after) && !(bits & F_CHECKED);
          uint32_t nb = bits | (chk ? F_CHECKED : 0u);
          uint32_t nd = dep;
          if (e.loop) {  // pos += 1 in place: no call, same depth (kernels.py:113-115)
            if (last) nb = stop | (chk ? F_CHECKED : 0u);  // pos == width: returns, the scan changes nothing
            else if (chk) nb |= F_CHECK;
          } else {  // recursion on the same range (kernels.py:116-119)
            nd = dep + 1u;
            if (chk) nb |= F_CHECK | F_DEFER;  // counted only if the scan finds it unsorted
            else {
              calls += 1;
              maxd = max(maxd, depth_abs(nd));
              if (last) nb = stop;  // the call sees pos == width and returns
            }
          }
          B[i] = SegT{cnt, pack(nb, ns, nd, 0), 0, 0};
        } else {  // two calls, streak restarts (kernels.py:120-125)
          const uint32_t nd = dep + 1u;
          calls += 2;
          maxd = max(maxd, depth_abs(nd));
          const uint32_t base = bits & ~(F_CHECKED | F_CHECK | F_DEFER | F_UNSORTED);
          B[i] = SegT{lo_n, pack((lo_n >= 2 && !last) ? base : (stop & ~F_CHECKED), 0, nd, 0), 0, 0};
          B[up_s] = SegT{up_n, pack((up_n >= 2 && !last) ? base : (stop & ~F_CHECKED), 0, nd, 0), 0, 0};
        }
      } else if (mode == M_ITER) {  // kernels.py:129-172
        calls += 1;
        uint32_t h;
        if (last) {  // pos + 1 == width: nothing pushed, but the partition still moved the data
          h = P;
          if (pass) {
            B[i] = SegT{cnt, pack(stop, 0, 0, P), 0, 0};
          } else {
            B[i] = SegT{lo_n, pack(stop, 0, 0, P), 0, 0};
            B[up_s] = SegT{up_n, pack(stop, 0, 0, P), 0, 0};
          }
        } else if (pass) {
          h = P + 1u;
          B[i] = SegT{cnt, pack(bits, 0, 0, P), 0, 0};
        } else {
          const uint32_t up = up_n >= 2 ? 1u : 0u, lo = lo_n >= 2 ? 1u : 0u;
          h = P + up + lo;
          B[i] = SegT{lo_n, pack(lo ? bits : stop, 0, 0, P + up), 0, 0};
          B[up_s] = SegT{up_n, pack(up ? bits : stop, 0, 0, P), 0, 0};
        }
        maxd = max(maxd, h + 1u);
      } else if (mode == M_LEVELS) {  // core.py:146-180
        calls += 1;
        maxd = max(maxd, uint32_t(L) + 2u);  // pos + 1 - start_pos, +1 offset
        const uint32_t act = bits | F_CHECK;
        if (pass) {
          B[i] = SegT{cnt, pack(act, 0, 0, 0), 0, 0};
        } else {
          B[i] = SegT{lo_n, pack(lo_n >= 2 ? act : stop, 0, 0, 0), 0, 0};
          B[up_s] = SegT{up_n, pack(up_n >= 2 ? act : stop, 0, 0, 0), 0, 0};
        }
      } else {  // M_PAR prepartition level (variants.py:124-148)
        calls += 1;
        const bool roots = (L == e.par_levels - 1);  // children are the buckets
        auto child = [&](uint64_t at, uint32_t sz) {
          uint32_t nb = sz >= 2 ? bits : stop;
          uint32_t nd = 0;
          if (roots && sz >= 2) {  // sort_words(words, lo, up, levels, width, ..., levels + 1)
            nd = uint32_t(e.par_levels) + 1u;
            calls += 1;
            maxd = max(maxd, depth_abs(nd));
            if (last) nb = stop;
          }
          B[at] = SegT{sz, pack(nb, 0, nd, 0), 0, 0};
        };
        if (pass) {
          child(i, cnt);
        } else {
          child(i, lo_n);
          child(up_s, up_n);
        }
      }
    }
  }
  // block-aggregated counter updates
  __shared__ unsigned long long s_sum[3][8];
  __shared__ uint32_t s_max[8];
  for (int o = 16; o > 0; o >>= 1) {
    extr += __shfl_xor_sync(0xFFFFFFFFu, extr, o);
    swaps += __shfl_xor_sync(0xFFFFFFFFu, swaps, o);
    calls += __shfl_xor_sync(0xFFFFFFFFu, calls, o);
    maxd = max(maxd, __shfl_xor_sync(0xFFFFFFFFu, maxd, o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_sum[0][w] = extr;
    s_sum[1][w] = swaps;
    s_sum[2][w] = calls;
    s_max[w] = maxd;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long a = 0, b = 0, c = 0;
    uint32_t m = 0;
    for (int j = 0; j < int(blockDim.x >> 5); ++j) {
      a += s_sum[0][j];
      b += s_sum[1][j];
      c += s_sum[2][j];
      m = max(m, s_max[j]);
    }
    if (a) atomicAdd(&e.ctr[0], a);
    if (b) atomicAdd(&e.ctr[1], b);
    if (c) atomicAdd(&e.ctr[2], c);
    if (m) atomicMax(&e.ctr[3], (unsigned long long)(m - 1u));
  }
}

template <typename K>
__global__ void __launch_bounds__(EX_BLOCK) ex_index_kernel(Ex e, int pos, int par, int cur) {
  __shared__ uint32_t sw[EX_BLOCK / 32];
  const K *k = static_cast<const K *>(e.keys[par]);
  const uint64_t base = uint64_t(blockIdx.x) * EX_CHUNK + uint64_t(threadIdx.x) * EX_IPT;
  Elem el;
  load_elems(e, k, pos, cur, base, el);
  uint32_t G = thread_prefix(e, __popc(el.live & ~el.bits), sw);
  const SegT *tab = e.tab[cur];
  uint32_t ps = 0xFFFFFFFFu;
  SegT t{};
#pragma unroll
  for (int j = 0; j < EX_IPT; ++j) {
    if ((el.live >> j) & 1u) {
      const uint32_t s = el.s[j];
      if (s != ps) {
        ps = s;
        t = tab[s];
      }
      const uint32_t o = uint32_t(base + j - s), zp = G - t.g0, Z = t.g1 - t.g0;
      const uint32_t b = (el.bits >> j) & 1u;
      // L-ones: bit-1 elements the low cursor examines fresh, offsets [0, Z]
      if (o <= Z && b) e.lone[s + (o - zp)] = o;
      // R-zeros: bit-0 elements at offsets >= Z, ranked from the right end
      if (o >= Z && !b) e.zpos[s + (Z - zp - 1u)] = o;
      G += b ^ 1u;
    }
  }
}

template <typename K, int VB>
__global__ void __launch_bounds__(EX_BLOCK) ex_gather_kernel(Ex e, int pos, int par, int cur) {
  using V = typename ValT<VB>::T;
  __shared__ uint32_t sw[EX_BLOCK / 32];
  const K *src = static_cast<const K *>(e.keys[par]);
  K *dst = static_cast<K *>(e.keys[par ^ 1]);
  const V *vsrc = static_cast<const V *>(e.vals[par]);
  V *vdst = static_cast<V *>(e.vals[par ^ 1]);
  const uint64_t base = uint64_t(blockIdx.x) * EX_CHUNK + uint64_t(threadIdx.x) * EX_IPT;
  Elem el;
  load_elems(e, src, pos, cur, base, el);
  uint32_t G = thread_prefix(e, __popc(el.live & ~el.bits), sw);
  const SegT *tab = e.tab[cur];
  uint32_t ps = 0xFFFFFFFFu;
  SegT t{};
  auto mv = [&](uint32_t s, uint32_t to, uint32_t from) {
    dst[uint64_t(s) + to] = src[uint64_t(s) + from];
    if constexpr (VB != 0) vdst[uint64_t(s) + to] = vsrc[uint64_t(s) + from];
  };
#pragma unroll
  for (int j = 0; j < EX_IPT; ++j) {
    if ((el.live >> j) & 1u) {
      const uint32_t s = el.s[j];
      if (s != ps) {
        ps = s;
        t = tab[s];
      }
      const uint32_t o = uint32_t(base + j - s), zp = G - t.g0, Z = t.g1 - t.g0;
      const uint32_t b = (el.bits >> j) & 1u;
      if (o < Z) {
        // zero region: the k-th L-one is replaced by the k-th R-zero
        mv(s, o, b ? e.zpos[s + (o - zp)] : o);
      } else {
        // offset o-1 (o > Z): R-ones shift one slot left, else the next L-one
        if (o > Z) mv(s, o - 1u, b ? o : e.lone[s + 1u + (Z - zp - (b ^ 1u))]);
        if (o == t.count - 1u) mv(s, o, e.lone[s]);  // the first L-one ends at the top
      }
      e.seg[base + j] = o < Z ? s : s + Z;  // the children's start positions
      G += b ^ 1u;
    }
  }
}

// After the last level: a pending scan's deferred call (kernels.py:109-119:
// the recursion on pos == width still counts a call unless the range was
// found sorted).
__global__ void ex_resolve_kernel(Ex e, int cur) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= e.n || e.seg[i] != uint32_t(i)) return;
  const uint32_t f = e.tab[cur][i].flags;
  if ((f & F_CHECK) && (f & F_DEFER) && (f & F_UNSORTED)) {
    atomicAdd(&e.ctr[2], 1ull);
    atomicMax(&e.ctr[3], (unsigned long long)(e.depth0 + int64_t((f >> 16) & 0xFFu)));
  }
}

// Every element's final value is in the buffer its segment ended in.
template <typename K, int VB>
__global__ void ex_finalize_kernel(Ex e, int cur, uint32_t fpar) {
  using V = typename ValT<VB>::T;
  const SegT *tab = e.tab[cur];
  K *k0 = static_cast<K *>(e.keys[0]);
  const K *k1 = static_cast<const K *>(e.keys[1]);
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < e.n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t f = tab[e.seg[i]].flags;
    const uint32_t home = (f & F_ACTIVE) ? fpar : ((f & F_HOME) ? 1u : 0u);
    if (home) {
      k0[i] = k1[i];
      if constexpr (VB != 0) static_cast<V *>(e.vals[0])[i] = static_cast<const V *>(e.vals[1])[i];
    }
  }
}

// Observer support: the array as the reference's observer sees it after a
// level (each element read from the buffer its segment currently lives in).
template <typename K>
__global__ void ex_snapshot_kernel(Ex e, int cur, uint32_t apar, K *out) {
  const SegT *tab = e.tab[cur];
  const K *k0 = static_cast<const K *>(e.keys[0]);
  const K *k1 = static_cast<const K *>(e.keys[1]);
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < e.n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t f = tab[e.seg[i]].flags;
    const uint32_t home = (f & F_ACTIVE) ? apar : ((f & F_HOME) ? 1u : 0u);
    out[i] = home ? k1[i] : k0[i];
  }
}

// Observer support: the current segments' start positions, in order.
__global__ void __launch_bounds__(EX_BLOCK) ex_starts_count_kernel(const uint32_t *seg, uint64_t n, uint32_t *bcnt) {
  __shared__ uint32_t sw[EX_BLOCK / 32];
  const uint64_t base = uint64_t(blockIdx.x) * EX_CHUNK + uint64_t(threadIdx.x) * EX_IPT;
  uint32_t c = 0;
  for (int j = 0; j < EX_IPT; ++j)
    if (base + j < n && seg[base + j] == uint32_t(base + j)) ++c;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < EX_BLOCK / 32; ++w) t += sw[w];
    bcnt[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(EX_BLOCK) ex_starts_write_kernel(const uint32_t *seg, uint64_t n, const uint32_t *bcnt,
                                                                   uint32_t *out) {
  __shared__ uint32_t sw[EX_BLOCK / 32];
  const uint64_t base = uint64_t(blockIdx.x) * EX_CHUNK + uint64_t(threadIdx.x) * EX_IPT;
  uint32_t m = 0;
  for (int j = 0; j < EX_IPT; ++j)
    if (base + j < n && seg[base + j] == uint32_t(base + j)) m |= 1u << j;
  const uint32_t c = __popc(m);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t incl = c;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) sw[w] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t acc = 0;
    for (int i = 0; i < EX_BLOCK / 32; ++i) {
      const uint32_t t = sw[i];
      sw[i] = acc;
      acc += t;
    }
  }
  __syncthreads();
  uint32_t at = bcnt[blockIdx.x] + sw[w] + incl - c;
  for (int j = 0; j < EX_IPT; ++j)
    if ((m >> j) & 1u) out[at++] = uint32_t(base + j);
}

}  // namespace ex
}  // namespace bs
