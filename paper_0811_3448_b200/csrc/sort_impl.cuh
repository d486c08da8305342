// sort_impl.cuh -- level-synchronous MSD radix-2^8 Binar Sort for sm_100a.
//
// Reference algorithm: kernels.sort_words (kernels.py:88-126) recursively
// partitions a range on one bit (partition_words, kernels.py:56-77), passes
// through single-sided splits (kernels.py:107-119) and stops at ranges of
// size < 2 or at pos == width (kernels.py:104-105).  One 8-bit digit pass here
// yields exactly the bucket sets and boundaries of 8 reference levels
// (SURVEY §7); pass-through becomes "digit constant within the bucket" and is
// skipped without moving data; ranges that fit in shared memory end the
// recursion in a local sort (K4).
//
// Device pipeline per level L (no host synchronisation anywhere):
//   K1 hist_kernel    per-tile digit histogram + OR/AND masks of the bucket
//   -- plan_kernel    per bucket: skip / requeue / scatter decision, digit
//                     bases, children -> next level or local tasks
//   K2+K3 scatter     stable ballot ranking, single-pass decoupled look-back
//                     across the bucket's tiles, smem-staged coalesced scatter
// then K4 local_kernel over the task list.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace bs {

constexpr int MAXLEV = 9;  // >= max digits (8 for u64) + 1

// Optional in-kernel phase timing (compile with -DBS_PROFILE; scratch builds
// only): thread 0 of every CTA accumulates clock64 deltas per phase.
#ifdef BS_PROFILE
__device__ unsigned long long g_prof[16];
// deltas accumulate in registers; BS_PROBE_FLUSH() publishes them once
#define BS_PROBE_INIT()          \
  long long prof_t0_ = clock64(); \
  long long prof_acc_[16] = {0}
#define BS_PROBE(i)                        \
  do {                                     \
    const long long now_ = clock64();      \
    prof_acc_[i] += now_ - prof_t0_;       \
    prof_t0_ = now_;                       \
  } while (0)
#define BS_PROBE_FLUSH()                                                            \
  do {                                                                              \
    if (threadIdx.x == 0)                                                           \
      for (int i_ = 0; i_ < 16; ++i_)                                               \
        if (prof_acc_[i_]) atomicAdd(&g_prof[i_], (unsigned long long)prof_acc_[i_]); \
  } while (0)
#else
#define BS_PROBE_INIT() (void)0
#define BS_PROBE(i) (void)0
#define BS_PROBE_FLUSH() (void)0
#endif
constexpr uint32_t ST_AGG = 1u << 30;
constexpr uint32_t ST_INCL = 2u << 30;
constexpr uint32_t ST_MASK = (1u << 30) - 1;

enum : uint32_t { ACT_SCATTER = 0, ACT_SKIP = 1, ACT_GEN = 2 };

struct Bucket {
  uint64_t start;
  uint32_t count;
  uint32_t tile0;
  uint32_t digit;
  uint32_t parity;  // 0: live data in the caller's buffer, 1: in the workspace copy
  uint32_t action;
  uint32_t flags;  // BK_HKNOWN | parent digit << 8: histogram/masks filled by expand from hist16
};
constexpr uint32_t BK_HKNOWN = 1u;

struct Task {
  uint64_t start;
  uint32_t count;
  uint32_t parity;
};

// A dense keys-only task: every key equals `common` outside the bit span
// [lb, lb+span) of the normalised key (span <= 16).
struct DTask {
  uint64_t start;
  uint64_t common;
  uint32_t count;
  uint32_t meta;  // lb | span << 8 | parity << 16 | digit << 20 (digit: big tasks' next MSD digit)
};

struct Ctl {
  uint32_t nbuckets[MAXLEV + 1];
  uint32_t ntiles[MAXLEV + 1];
  uint32_t ticket[MAXLEV + 1];
  uint32_t ticket2[MAXLEV + 1];  // tile_scan_kernel
  uint32_t ntasks;
  uint32_t ndtasks;      // small dense tasks (front of dtasks)
  uint32_t error;        // bit 0: bucket overflow, 1: tile overflow, 2: task overflow
  uint32_t ndtasks_big;  // big dense tasks (back of dtasks)
  uint32_t dbig_end[MAXLEV + 1];  // ndtasks_big after plan(L) (snapshot by scatter(L))
  uint32_t h16_bad;  // hist16 unusable (the root's digit is the last one)
  uint32_t ntasks2;  // tasks the spread local sort hands to local_kernel (tasks2)
  uint32_t skewed;   // a root digit holds > 1/16 of the keys (duplicate-heavy data: Zipf)
  uint32_t gen;      // the output is generated from hist16 (gen16_kernel); gen_shift: its bit offset
  uint32_t gen_shift;
};

// Workspace view (all device pointers), built on the host.
struct Ws {
  Ctl *ctl;
  Bucket *buckets[2];
  uint32_t *bhist[2];  // [maxb][256]; counts, then (after plan) digit bases
  uint64_t *bor[2];
  uint64_t *band[2];
  uint32_t *tile_bucket[2];
  uint32_t *status;  // [maxtiles][256] look-back words (stable sorts)
  uint32_t *toff;    // [maxtiles][256] stable sorts: tile digit counts, then run offsets
  uint32_t *hist16;  // [65536]: root histogram of the digit pair (dig, dig+1)
  uint32_t *h16part; // [H16_MAXCTA][32768]: per-CTA packed partial rows
  Task *tasks;
  Task *tasks2;  // spread_kernel's leftovers for local_kernel (u64 keys-only sorts)
  DTask *dtasks;
  int dense;           // keys-only full-width: dense tasks go to dense_kernel
  uint32_t dense_max;      // small dense_kernel capacity
  uint32_t dense_big_max;  // big dense_kernel capacity (0: none)
  void *keys[2];  // [0] caller's buffer, [1] workspace copy
  void *vals[2];
  uint64_t n;
  uint32_t maxb, maxtiles, maxtasks;
  uint32_t tile;       // elements per scatter tile
  uint32_t local_max;  // largest range the local sort takes
  uint32_t group_min;  // children smaller than this are grouped
  int ndig;            // number of 8-bit digits of the effective key
  int shift0;          // W - width_eff
  int kbits;           // W
  int stable;          // key-value sort: tiles use the look-back scan
  uint32_t root_parity;  // buffer holding the input: 0 caller's, 1 the copy (bs_sort_from: the source)
};


// A sort whose work lists overflowed (ctl->error, reported by bs_sort_status)
// must not consume the entries that were never written: every kernel after
// init checks the flag once per CTA (block-uniform, before any role split)
// and exits.
__device__ __forceinline__ bool ws_failed(const Ws &ws) {
  __shared__ uint32_t s_fail;
  if (threadIdx.x == 0) s_fail = *reinterpret_cast<volatile const uint32_t *>(&ws.ctl->error);
  __syncthreads();
  return s_fail != 0;
}

// ---------------------------------------------------------------------------
// init: root bucket (or a single local task when n fits the local sort).
// A strided sample guesses the first varying digit so constant leading digits
// (e.g. "low 16 bits random" u64 keys) cost no wasted histogram pass.
// ---------------------------------------------------------------------------
template <typename K, int KIND>
__global__ void init_kernel(Ws ws) {
  pdl_wait();  // programmatic dependent launch: previous kernel's writes visible
  const int tid = threadIdx.x;
  const uint64_t n = ws.n;
  const KeyGeom<K, KIND> g{ws.shift0};
  if (n <= ws.local_max) {
    if (blockIdx.x == 0 && tid == 0) {
      ws.tasks[0] = Task{0, uint32_t(n), ws.root_parity};
      ws.ctl->ntasks = 1;
    }
    return;
  }
  const uint32_t ntiles = uint32_t((n + ws.tile - 1) / ws.tile);
  for (uint32_t t = blockIdx.x * blockDim.x + tid; t < ntiles; t += gridDim.x * blockDim.x)
    ws.tile_bucket[0][t] = 0;
  for (int d = tid; d < 256; d += blockDim.x) ws.bhist[0][d] = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + tid; i < 65536u / 4; i += gridDim.x * blockDim.x)
    reinterpret_cast<uint4 *>(ws.hist16)[i] = make_uint4(0, 0, 0, 0);
  if (blockIdx.x != 0) return;
  __shared__ uint64_t s_or[32], s_and[32];
  // 4096-element strided sample of the encoded normalised key
  K o = 0, a = ~K(0);
  const K *keys = static_cast<const K *>(ws.keys[ws.root_parity]);
  for (int i = tid; i < 4096; i += blockDim.x) {
    uint64_t idx = (uint64_t(2 * i + 1) * n) / 8192;
    K nk = g.norm(keys[idx]);
    o |= nk;
    a &= nk;
  }
  o = warp_or(o);
  a = warp_and(a);
  if ((tid & 31) == 0) {
    s_or[tid >> 5] = o;
    s_and[tid >> 5] = a;
  }
  __syncthreads();
  if (tid == 0) {
    K oo = 0, aa = ~K(0);
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      oo |= K(s_or[w]);
      aa &= K(s_and[w]);
    }
    K var = oo ^ aa;
    int dig = var ? (KeyTraits<K>::clz(var) >> 3) : 0;
    if (dig >= ws.ndig) dig = 0;
    ws.buckets[0][0] = Bucket{0, uint32_t(n), 0, uint32_t(dig), ws.root_parity, ACT_SCATTER, 0};
    ws.bor[0][0] = 0;
    ws.band[0][0] = ~uint64_t(0);
    ws.ctl->nbuckets[0] = 1;
    ws.ctl->ntiles[0] = ntiles;
  }
}

// ---------------------------------------------------------------------------
// K1: per-bucket digit histogram + OR/AND of normalised keys.  CTAs own
// contiguous tile ranges, so per-CTA shared counters are flushed to the
// bucket's global histogram only when the bucket changes.  Also clears the
// look-back status rows of the tiles it visits (same tiling as the scatter).
// ---------------------------------------------------------------------------
template <typename K, int KIND, int BLOCK, int KPT>
__global__ void __launch_bounds__(BLOCK) hist_kernel(Ws ws, int L) {
  pdl_wait();  // programmatic dependent launch: previous kernel's writes visible
  if (ws_failed(ws)) return;
  constexpr int NCOPY = 4;
  __shared__ uint32_t h[NCOPY][256];
  __shared__ uint64_t s_or[BLOCK / 32], s_and[BLOCK / 32];
  __shared__ uint32_t tprev[256];  // stable sorts: bucket counts up to the previous tile
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int cur = L & 1;
  const uint32_t nt = ws.ctl->ntiles[L];
  if (nt == 0) return;
  const uint32_t per = (nt + gridDim.x - 1) / gridDim.x;
  const uint32_t t0 = blockIdx.x * per;
  const uint32_t t1 = min(nt, t0 + per);
  if (t0 >= t1) return;
  const KeyGeom<K, KIND> g{ws.shift0};
  for (int i = tid; i < NCOPY * 256; i += BLOCK) (&h[0][0])[i] = 0;
  for (int i = tid; i < 256; i += BLOCK) tprev[i] = 0;
  K o = 0, a = ~K(0);
  uint32_t curb = 0xFFFFFFFFu;
  int dig = 0;
  bool known = false;  // bucket's histogram and masks come from hist16
  __syncthreads();
  auto flush = [&](uint32_t b) {
    __syncthreads();
    for (int d = tid; d < 256; d += BLOCK) {
      uint32_t s = 0;
#pragma unroll
      for (int c = 0; c < NCOPY; ++c) {
        s += h[c][d];
        h[c][d] = 0;
      }
      tprev[d] = 0;
      if (s) atomicAdd(&ws.bhist[cur][size_t(b) * 256 + d], s);
    }
    K oo = warp_or(o), aa = warp_and(a);
    if (lane == 0) {
      s_or[w] = oo;
      s_and[w] = aa;
    }
    __syncthreads();
    if (tid == 0) {
      K x = 0, y = ~K(0);
      for (int i = 0; i < BLOCK / 32; ++i) {
        x |= K(s_or[i]);
        y &= K(s_and[i]);
      }
      atomicOr(reinterpret_cast<unsigned long long *>(&ws.bor[cur][b]), (unsigned long long)x);
      atomicAnd(reinterpret_cast<unsigned long long *>(&ws.band[cur][b]),
                (unsigned long long)(uint64_t(y) | (sizeof(K) == 4 ? 0xFFFFFFFF00000000ull : 0ull)));
    }
    o = 0;
    a = ~K(0);
  };
  for (uint32_t t = t0; t < t1; ++t) {
    const uint32_t b = ws.tile_bucket[cur][t];
    const Bucket bk = ws.buckets[cur][b];
    if (b != curb) {
      if (curb != 0xFFFFFFFFu && !known) flush(curb);
      curb = b;
      dig = int(bk.digit);
      known = (bk.flags & BK_HKNOWN) != 0u;
    }
    // clear this tile's look-back row (256 x u32 = 64 x uint4)
    if (ws.stable && tid < 64)
      reinterpret_cast<uint4 *>(ws.status + size_t(t) * 256)[tid] = make_uint4(0, 0, 0, 0);
    if (known) {
      // nothing to count: keys-only sorts skip to the bucket's last tile
      if (!ws.stable) t = min(t1, bk.tile0 + uint32_t((bk.count + ws.tile - 1) / ws.tile)) - 1u;
      continue;
    }
    const uint64_t off = uint64_t(t - bk.tile0) * ws.tile;
    const uint32_t cnt = uint32_t(min64(ws.tile, bk.count - off));
    const K *src = static_cast<const K *>(ws.keys[bk.parity]) + bk.start + off;
    uint32_t *hc = h[w & (NCOPY - 1)];
    K x[KPT];
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      const uint32_t e = uint32_t(j) * BLOCK + tid;
      x[j] = (e < cnt) ? __ldcs(src + e) : K(0);
    }
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      const uint32_t e = uint32_t(j) * BLOCK + tid;
      if (e < cnt) {
        const K nk = g.norm(x[j]);
        o |= nk;
        a &= nk;
        atomicAdd(&hc[KeyGeom<K, KIND>::digit_of_norm(nk, dig)], 1u);
      }
    }
    if (ws.stable) {  // this tile's own digit counts, for tile_scan_kernel
      __syncthreads();
      for (int d = tid; d < 256; d += BLOCK) {
        uint32_t cur = 0;
#pragma unroll
        for (int cc = 0; cc < NCOPY; ++cc) cur += h[cc][d];
        ws.toff[size_t(t) * 256 + d] = cur - tprev[d];
        tprev[d] = cur;
      }
      __syncthreads();
    }
  }
  if (!known) flush(curb);
}

// ---------------------------------------------------------------------------
// K1 at level 0: histogram of the digit PAIR (dig, dig+1) of the root bucket,
// so the root's 256 children need no histogram pass of their own (plan(0)
// marks them BK_HKNOWN; expand(1) copies their rows).  One CTA per SM keeps
// 65536 16-bit bins in 128 KB of shared memory, two per word; sweeps between
// epochs of 32768 keys move every half that reached 0x8000 to the global
// counts, so no carry ever crosses into the neighbouring bin and the counts
// are exact for any input.  Also yields the root's 256-bin histogram (row sums) and OR/AND
// masks.
// ---------------------------------------------------------------------------
constexpr int H16_MAXCTA = 160;  // >= SM count (one CTA per SM)

template <typename K, int KIND, int BLOCK>
__global__ void __launch_bounds__(BLOCK, 1) hist16_kernel(Ws ws) {
  pdl_wait();  // programmatic dependent launch: previous kernel's writes visible
  if (ws_failed(ws)) return;
  constexpr int W = KeyTraits<K>::BITS;
  constexpr int EPG = 16 / int(sizeof(K));  // keys per 16-byte granule
  constexpr int UNR = 4;                    // granules in flight per thread
  extern __shared__ __align__(16) uint32_t hw[];  // 32768 words = 65536 u16 bins
  __shared__ uint64_t s_or[BLOCK / 32], s_and[BLOCK / 32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (ws.ctl->nbuckets[0] == 0) return;
  const Bucket bk = ws.buckets[0][0];
  const int dig = int(bk.digit);
  const bool two = dig + 1 < ws.ndig;
  const int sh8 = W - 8 - 8 * dig;
  const int shA = two ? sh8 - 8 : sh8;
  const uint32_t msk = two ? 0xFFFFu : 0xFFu, post = two ? 0u : 8u;
  for (int i = tid; i < 32768 / 4; i += BLOCK) reinterpret_cast<uint4 *>(hw)[i] = make_uint4(0, 0, 0, 0);
  if (!two && blockIdx.x == 0 && tid == 0) ws.ctl->h16_bad = 1u;
  if (ws.stable) {  // clear the level-0 tiles' look-back rows (hist_kernel's job at other levels)
    const uint32_t nq = ws.ctl->ntiles[0] * 64u;
    for (uint32_t i = blockIdx.x * BLOCK + tid; i < nq; i += gridDim.x * BLOCK)
      reinterpret_cast<uint4 *>(ws.status)[i] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  const KeyGeom<K, KIND> g{ws.shift0};
  const K *src = static_cast<const K *>(ws.keys[bk.parity]) + bk.start;
  const uint64_t n = bk.count;
  const uint32_t head = uint32_t((reinterpret_cast<uintptr_t>(src) & 15u) / sizeof(K));
  const uint4 *gsrc = reinterpret_cast<const uint4 *>(src - head);
  const uint64_t ng = (uint64_t(head) + n + EPG - 1) / EPG;
  const uint64_t g0 = ng * blockIdx.x / gridDim.x, g1 = ng * (blockIdx.x + 1) / gridDim.x;
  const uint64_t gA = head ? 1u : 0u, gB = (uint64_t(head) + n) / EPG;  // granules [gA, gB) hold only keys
  K o = 0, a = ~K(0);
  // Bin p: count in half (p & 1) of word p >> 1, incremented without a
  // return value.  Epochs of at most 32768 keys per CTA are separated by a
  // sweep that moves every half at or above 0x8000 to the global counts, so
  // no half can exceed 0x7FFF + 32768 = 0xFFFF between sweeps: exact for any
  // input, with no per-key overflow test.
  constexpr int GPE = 32768 / (BLOCK * EPG);  // granules per thread per epoch
  static_assert(GPE % UNR == 0 && GPE > 0, "whole batches per epoch");
  // A batch = UNR granules per thread (a warp's batch is contiguous).  The
  // batch's OR/AND masks (which the root's masks need anyway) show when all of
  // a thread's keys share one bin; when all 32 lanes share the same bin
  // (sorted or constant runs) one add of 32*UNR*EPG replaces that many
  // same-address atomics.  After a failed check the warp skips the check for
  // 7 batches, so spread keys pay ~nothing for it.  The epoch bound is
  // unchanged (the same keys are counted).
  int skip = 0;  // batches until the next same-bin check (warp-uniform)
  // Batches in the coming epoch (block-uniform): two in general (halves are
  // below 0x8000 after a sweep, an epoch of 2 x 16384 keys adds at most
  // 0x8000); three when the sweep saw every half below 0x4000 (3 x 16384 =
  // 0xC000 more still fits 16 bits) -- the usual case for spread keys, and a
  // third fewer barriers and sweeps.
  static_assert(UNR * BLOCK * EPG <= 16384, "three batches add at most 0xC000 to a half");
  int nbatch = GPE / UNR + 1;  // the bins start at zero
  for (uint64_t eb = g0; eb < g1;) {  // block-uniform epochs
    const int ebatch = nbatch;  // this epoch's batches (nbatch becomes the next epoch's below)
#pragma unroll 1
    for (int u0 = 0; u0 < ebatch * UNR; u0 += UNR) {
      uint4 v[UNR];
      K nk[UNR * EPG];
      uint32_t valid = 0;
      K ob = 0, ab = ~K(0);
      const uint64_t bstart = eb + uint64_t(u0) * BLOCK, bend = bstart + uint64_t(UNR) * BLOCK;
      if (bstart >= gA && bend <= gB && bend <= g1) {  // block-uniform: every key of the batch is valid
#pragma unroll
        for (int u = 0; u < UNR; ++u)
          v[u] = __ldcs(gsrc + (bstart + uint64_t(w) * (32 * UNR) + uint64_t(u) * 32 + lane));
        valid = (1u << (UNR * EPG)) - 1u;
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          K kk[EPG];
          if constexpr (sizeof(K) == 4) {
            kk[0] = K(v[u].x), kk[1] = K(v[u].y), kk[2 % EPG] = K(v[u].z), kk[3 % EPG] = K(v[u].w);
          } else {
            kk[0] = K((uint64_t(v[u].y) << 32) | v[u].x);
            kk[1 % EPG] = K((uint64_t(v[u].w) << 32) | v[u].z);
          }
#pragma unroll
          for (int j = 0; j < EPG; ++j) nk[u * EPG + j] = g.norm(kk[j]);
        }
#pragma unroll
        for (int i = 0; i < UNR * EPG; i += 2) {
          ob |= nk[i] | nk[i + 1];
          ab &= nk[i] & nk[i + 1];
        }
      } else {
#pragma unroll
        for (int u = 0; u < UNR; ++u) {  // a warp's batch: 32*UNR consecutive granules
          const uint64_t gi = bstart + uint64_t(w) * (32 * UNR) + uint64_t(u) * 32 + lane;
          v[u] = gi < g1 ? __ldcs(gsrc + gi) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const uint64_t gi = bstart + uint64_t(w) * (32 * UNR) + uint64_t(u) * 32 + lane;
          K kk[EPG];
          if constexpr (sizeof(K) == 4) {
            kk[0] = K(v[u].x), kk[1] = K(v[u].y), kk[2 % EPG] = K(v[u].z), kk[3 % EPG] = K(v[u].w);
          } else {
            kk[0] = K((uint64_t(v[u].y) << 32) | v[u].x);
            kk[1 % EPG] = K((uint64_t(v[u].w) << 32) | v[u].z);
          }
          const int64_t e0 = int64_t(gi * EPG) - int64_t(head);
#pragma unroll
          for (int j = 0; j < EPG; ++j) {
            nk[u * EPG + j] = g.norm(kk[j]);
            if (gi < g1 && e0 + j >= 0 && e0 + j < int64_t(n)) {
              valid |= 1u << (u * EPG + j);
              ob |= nk[u * EPG + j];
              ab &= nk[u * EPG + j];
            }
          }
        }
      }
      o |= ob;
      a &= ab;
      constexpr uint32_t ALL = (1u << (UNR * EPG)) - 1u;
      bool agg = false;
      if (skip == 0) {  // warp-uniform
        const uint32_t pb = (uint32_t(ob >> shA) & msk) << post;
        const bool same = valid == ALL && ((uint32_t((ob ^ ab) >> shA) & msk) == 0u);
        const uint32_t lead = __shfl_sync(0xFFFFFFFFu, pb, 0);
        agg = __all_sync(0xFFFFFFFFu, same && pb == lead);
        if (agg && lane == 0) atomicAdd(&hw[lead >> 1], (32u * UNR * EPG) << (16u * (lead & 1u)));
        if (!agg) skip = 7;  // spread keys: look again 8 batches later
      } else {
        --skip;
      }
      if (agg) {
      } else if (valid == ALL) {
#pragma unroll
        for (int i = 0; i < UNR * EPG; ++i) {
          const uint32_t p = (uint32_t(nk[i] >> shA) & msk) << post;
          atomicAdd(&hw[p >> 1], 1u + (p & 1u) * 0xFFFFu);
        }
      } else {
#pragma unroll
        for (int i = 0; i < UNR * EPG; ++i) {
          if ((valid >> i) & 1u) {
            const uint32_t p = (uint32_t(nk[i] >> shA) & msk) << post;
            atomicAdd(&hw[p >> 1], 1u + (p & 1u) * 0xFFFFu);
          }
        }
      }
    }
    __syncthreads();
    uint32_t seen = 0;  // OR of this thread's words after the sweep
    for (int q = tid; q < 32768 / 4; q += BLOCK) {  // sweep (rarely finds anything)
      uint4 wv = reinterpret_cast<const uint4 *>(hw)[q];
      seen |= (wv.x | wv.y | wv.z | wv.w) & 0x7FFF7FFFu;
      if ((wv.x | wv.y | wv.z | wv.w) & 0x80008000u) {
        uint32_t *ww = &wv.x;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          for (int h = 0; h < 2; ++h) {
            if (ww[k] & (0x8000u << (16 * h))) {
              const uint32_t p = 2u * (4u * q + k) + h;
              atomicAdd(&ws.hist16[p], 32768u);
              atomicAdd(&ws.bhist[0][p >> 8], 32768u);
            }
          }
          ww[k] &= 0x7FFF7FFFu;
        }
        reinterpret_cast<uint4 *>(hw)[q] = wv;
      }
    }
    // (the barrier the sweep needs anyway carries the verdict)
    nbatch = __syncthreads_or((seen & 0x40004000u) != 0u) ? GPE / UNR : GPE / UNR + 1;
    eb += uint64_t(ebatch) * UNR * BLOCK;
  }
  __syncthreads();
  // flush: this CTA's packed bins to its partial row (plain coalesced stores;
  // hist16_reduce_kernel folds the rows)
  {
    uint4 *dst = reinterpret_cast<uint4 *>(ws.h16part + size_t(blockIdx.x) * 32768);
    for (int q = tid; q < 32768 / 4; q += BLOCK) dst[q] = reinterpret_cast<const uint4 *>(hw)[q];
  }
  const K oo = warp_or(o), aa = warp_and(a);
  if (lane == 0) {
    s_or[w] = oo;
    s_and[w] = aa;
  }
  __syncthreads();
  if (tid == 0) {
    K x = 0, y = ~K(0);
    for (int i = 0; i < BLOCK / 32; ++i) {
      x |= K(s_or[i]);
      y &= K(s_and[i]);
    }
    atomicOr(reinterpret_cast<unsigned long long *>(&ws.bor[0][0]), (unsigned long long)x);
    atomicAnd(reinterpret_cast<unsigned long long *>(&ws.band[0][0]),
              (unsigned long long)(uint64_t(y) | (sizeof(K) == 4 ? 0xFFFFFFFF00000000ull : 0ull)));
  }
}

// Fold hist16_kernel's per-CTA partial rows (two u16 bins per word) into
// hist16 (which already holds the sweeps' spills) and the root's 256-bin
// histogram.  Thread (quad q, slice k) sums word quad q over a quarter of the
// rows; the four slices meet in shared memory.  256 threads = 64 quads.
__global__ void __launch_bounds__(256) hist16_reduce_kernel(Ws ws, int nparts) {
  pdl_wait();  // programmatic dependent launch: previous kernel's writes visible
  if (ws_failed(ws)) return;
  __shared__ uint4 s_part[3][64][2];  // slices 1..3: (lo sums, hi sums) of 4 words
  if (ws.ctl->nbuckets[0] == 0) return;
  const int tid = threadIdx.x, ql = tid & 63, k = tid >> 6;
  const uint32_t q = blockIdx.x * 64u + uint32_t(ql);  // word quad: bins 8q .. 8q+7
  const uint4 *src = reinterpret_cast<const uint4 *>(ws.h16part);
  uint4 lo = make_uint4(0, 0, 0, 0), hi = make_uint4(0, 0, 0, 0);
  const int p0 = nparts * k / 4, p1 = nparts * (k + 1) / 4;
#pragma unroll 4
  for (int pp = p0; pp < p1; ++pp) {
    const uint4 v = src[size_t(pp) * 8192 + q];
    lo.x += v.x & 0xFFFFu, hi.x += v.x >> 16;
    lo.y += v.y & 0xFFFFu, hi.y += v.y >> 16;
    lo.z += v.z & 0xFFFFu, hi.z += v.z >> 16;
    lo.w += v.w & 0xFFFFu, hi.w += v.w >> 16;
  }
  if (k > 0) {
    s_part[k - 1][ql][0] = lo;
    s_part[k - 1][ql][1] = hi;
  }
  __syncthreads();
  if (k != 0) return;
  for (int j = 0; j < 3; ++j) {
    const uint4 l = s_part[j][ql][0], h = s_part[j][ql][1];
    lo.x += l.x, lo.y += l.y, lo.z += l.z, lo.w += l.w;
    hi.x += h.x, hi.y += h.y, hi.z += h.z, hi.w += h.w;
  }
  if (ws.ctl->h16_bad == 0u) {
    uint4 *h0 = reinterpret_cast<uint4 *>(ws.hist16) + 2 * q;  // bins 8q..8q+3, 8q+4..8q+7
    uint4 a0 = h0[0], a1 = h0[1];
    a0.x += lo.x, a0.y += hi.x, a0.z += lo.y, a0.w += hi.y;
    a1.x += lo.z, a1.y += hi.z, a1.z += lo.w, a1.w += hi.w;
    h0[0] = a0;
    h0[1] = a1;
  }
  // 32 quads (one warp's lanes 0..31 of a slice-0 half) = 256 bins = one row
  uint32_t sum = lo.x + lo.y + lo.z + lo.w + hi.x + hi.y + hi.z + hi.w;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xFFFFFFFFu, sum, off);
  if ((tid & 31) == 0 && sum) atomicAdd(&ws.bhist[0][q >> 5], sum);
}

// ---------------------------------------------------------------------------
// plan: one CTA (256 threads) per bucket of level L.  Decides skip / requeue /
// scatter, turns the histogram into digit bases in place, and emits the
// children: large ones to the next level's list (their tiles are mapped by
// expand_kernel), the rest to the local-sort task list.
// ---------------------------------------------------------------------------
struct Emit {
  uint64_t start;
  uint32_t count;
  uint32_t kind;   // 0 large child (next level), 1 local task
  uint32_t digit;  // the child's digit value, or 0xFFFFFFFF for a group of children
};

// Task.parity: bit 0 the buffer holding the data, bits 8+ the first digit
// that may vary inside the task (digits above it are shared by its keys).
__device__ __forceinline__ void emit_tasks(const Ws &ws, uint64_t start, uint64_t count,
                                           uint32_t parity, uint32_t digit = 0u) {
  // chunks of <= local_max (callers: all-equal ranges that only need a copy,
  // or ranges the local sort takes whole)
  const uint64_t nch = (count + ws.local_max - 1) / ws.local_max;
  const uint32_t base = atomicAdd(&ws.ctl->ntasks, uint32_t(nch));
  if (base + nch > ws.maxtasks) {
    atomicOr(&ws.ctl->error, 4u);
    return;
  }
  for (uint64_t c = 0; c < nch; ++c) {
    const uint64_t s = c * ws.local_max;
    ws.tasks[base + c] = Task{start + s, uint32_t(min64(ws.local_max, count - s)), (parity & 1u) | (digit << 8)};
  }
}

__device__ __forceinline__ void push_bucket(const Ws &ws, int L, uint64_t start, uint32_t count,
                                            uint32_t digit, uint32_t parity) {
  const uint32_t slot = atomicAdd(&ws.ctl->nbuckets[L + 1], 1u);
  const uint32_t nt = uint32_t((count + ws.tile - 1) / ws.tile);
  const uint32_t t0 = atomicAdd(&ws.ctl->ntiles[L + 1], nt);
  if (slot >= ws.maxb || t0 + nt > ws.maxtiles) {
    atomicOr(&ws.ctl->error, 3u);
    return;
  }
  ws.buckets[(L + 1) & 1][slot] = Bucket{start, count, t0, digit, parity, ACT_SCATTER, 0};
}

template <typename K>
__global__ void __launch_bounds__(256) plan_kernel(Ws ws, int L) {
  pdl_wait();  // programmatic dependent launch: previous kernel's writes visible
  if (ws_failed(ws)) return;
  constexpr int W = KeyTraits<K>::BITS;
  __shared__ uint32_t s_cnt[256];
  __shared__ uint32_t s_scan[16];
  __shared__ Emit s_emit[520];
  __shared__ uint32_t s_nemit;
  const int tid = threadIdx.x;
  const int cur = L & 1;
  const uint32_t nb = min(ws.ctl->nbuckets[L], ws.maxb);
  // Whole-input counting (keys only, full-width words): when every varying
  // bit of the root lies in the hist16 digit pair, the sorted output is a
  // function of the 65536-bin histogram alone (value v repeated count[v]
  // times), so no key moves: hist16 becomes its exclusive prefix and
  // gen16_kernel writes the output (one read pass + one write pass).  Every
  // CTA evaluates the same condition and the CTAs share the 256 rows of the
  // histogram: row base from the root's digit counts (the row sums), then a
  // scan of the row in place.
  if (L == 0 && nb == 1u && ws.dense && !ws.stable && ws.ctl->h16_bad == 0u) {
    const Bucket bk = ws.buckets[0][0];
    const K var = K(ws.bor[0][0] ^ ws.band[0][0]);
    const int dig = int(bk.digit);
    const int shA = W - 16 - 8 * dig;
    if (var != 0 && (KeyTraits<K>::clz(var) >> 3) == dig && shA >= 0 && (var & ~(K(0xFFFF) << shA)) == 0) {
      __shared__ uint32_t s_rowbase[256];
      s_rowbase[tid] = scan256_excl<256>(ws.bhist[0][tid], s_scan);
      __syncthreads();
      for (uint32_t r = blockIdx.x; r < 256u; r += gridDim.x) {
        uint32_t *row = ws.hist16 + size_t(r) * 256;
        const uint32_t e = scan256_excl<256>(row[tid], s_scan);
        row[tid] = s_rowbase[r] + e;
      }
      if (blockIdx.x == 0 && tid == 0) {
        ws.buckets[0][0].action = ACT_GEN;
        ws.ctl->gen_shift = uint32_t(shA);
        ws.ctl->gen = 1u;
      }
      return;
    }
  }
  for (uint32_t b = blockIdx.x; b < nb; b += gridDim.x) {
    const Bucket bk = ws.buckets[cur][b];
    uint32_t *hist = ws.bhist[cur] + size_t(b) * 256;
    const uint32_t c = hist[tid];
    // duplicate-heavy input (one root digit with > 1/16 of the keys): 64-bit
    // local tasks skip the dense-prefix sort, which would mostly hand them on
    if (L == 0 && b == 0 && c > bk.count / 16u) ws.ctl->skewed = 1u;
    const K var = K(ws.bor[cur][b] ^ ws.band[cur][b]);
    const int dig = int(bk.digit);
    if (var == 0) {  // all keys equal: finished; copy home if needed
      if (tid == 0) {
        ws.buckets[cur][b].action = ACT_SKIP;
        if (bk.parity) emit_tasks(ws, bk.start, bk.count, 1);
      }
      continue;
    }
    const int dstar = KeyTraits<K>::clz(var) >> 3;
    if (dstar != dig) {  // digit constant here (pass-through): requeue at dstar
      if (tid == 0) {
        ws.buckets[cur][b].action = ACT_SKIP;
        if (bk.count <= ws.local_max) emit_tasks(ws, bk.start, bk.count, bk.parity, uint32_t(dstar));
        else push_bucket(ws, L, bk.start, bk.count, uint32_t(dstar), bk.parity);
      }
      continue;
    }
    if (bk.flags & BK_HKNOWN) {
      // histogram from hist16, masks conservative (the root's): one occupied
      // digit means the digit is constant here -- requeue on the next digit,
      // which gets a real histogram pass
      if (__syncthreads_count(c != 0u) == 1) {
        if (tid == 0) {
          ws.buckets[cur][b].action = ACT_SKIP;
          if (bk.count <= ws.local_max) emit_tasks(ws, bk.start, bk.count, bk.parity, uint32_t(dig + 1));
          else if (dig + 1 < ws.ndig) push_bucket(ws, L, bk.start, bk.count, uint32_t(dig + 1), bk.parity);
          else if (bk.parity) emit_tasks(ws, bk.start, bk.count, 1);  // every digit constant: all equal
        }
        continue;
      }
    }
    // scatter this bucket on digit `dig`
    const uint32_t excl = scan256_excl<256>(c, s_scan);
    hist[tid] = excl;  // digit base within the bucket
    s_cnt[tid] = c;
    if (tid == 0) ws.buckets[cur][b].action = ACT_SCATTER;
    const uint32_t cpar = bk.parity ^ 1u;
    const int lowbits = W - 8 - 8 * dig;
    // the root's children take their histograms from hist16 (no hist pass at level 1)
    const bool h16 = L == 0 && ws.ctl->h16_bad == 0u && !ws.stable;
    const K lower = lowbits > 0 ? (var & ((K(1) << lowbits) - 1)) : K(0);
    if (lower == 0) {  // every child is all-equal: only a copy home may remain
      if (tid == 0 && cpar) emit_tasks(ws, bk.start, bk.count, 1);
      __syncthreads();
      continue;
    }
    // standalone children whose varying bits fit a 16-bit span are dense tasks
    const int lbv = __ffsll((long long)uint64_t(lower)) - 1;
    const int spanv = W - KeyTraits<K>::clz(lower) - lbv;
    const bool dense = ws.dense && spanv <= 16;
    // dense children up to the big dense kernel's capacity stay local even
    // when they exceed local_max (no further global level for them)
    // (big ones only while dense enough that repeats stay rare: n <= 2^span / 3.5)
    const uint32_t big_max =
        dense ? max(ws.local_max, min(ws.dense_big_max, uint32_t((2ull << spanv) / 7))) : ws.local_max;
    // Greedy grouping in digit order, in parallel: large children (>= group_min)
    // are emitted on their own; each run of small children between two large
    // ones is packed greedily (groups <= local_max) by the run's first digit.
    const uint32_t cd = c;
    const bool isbig = cd >= ws.group_min, issmall = cd > 0 && !isbig;
    __shared__ uint32_t s_bigm[8], s_smallm[8], s_excl[256];
    {
      const uint32_t bm = __ballot_sync(0xFFFFFFFFu, isbig), sm = __ballot_sync(0xFFFFFFFFu, issmall);
      if ((tid & 31) == 0) {
        s_bigm[tid >> 5] = bm;
        s_smallm[tid >> 5] = sm;
      }
      s_excl[tid] = excl;
    }
    __syncthreads();
    auto last_below = [&](const uint32_t *m, int d) -> int {  // highest set bit < d, or -1
      for (int wd = d >> 5; wd >= 0; --wd) {
        const uint32_t x = m[wd] & (wd == (d >> 5) ? ((1u << (d & 31)) - 1u) : 0xFFFFFFFFu);
        if (x) return wd * 32 + 31 - __clz(x);
      }
      return -1;
    };
    const bool leader = issmall && last_below(s_smallm, tid) <= last_below(s_bigm, tid);
    // run leaders walk their run twice: count the groups, then write them
    auto walk = [&](uint32_t slot, bool write) -> uint32_t {
      uint32_t k = 0, gc = 0, gs = 0;
      for (int d = tid; d < 256; ++d) {
        const uint32_t cdd = s_cnt[d];
        if (cdd >= ws.group_min) break;
        if (cdd == 0) continue;
        if (gc + cdd > ws.local_max) {
          if (write) s_emit[slot + k] = Emit{bk.start + gs, gc, 1, 0xFFFFFFFFu};
          ++k;
          gc = 0;
        }
        if (gc == 0) gs = s_excl[d];
        gc += cdd;
      }
      if (write) s_emit[slot + k] = Emit{bk.start + gs, gc, 1, 0xFFFFFFFFu};
      return k + 1;
    };
    const uint32_t myn = isbig ? 1u : (leader ? walk(0, false) : 0u);
    const uint32_t eoff = scan256_excl<256>(myn, s_scan);
    if (tid == 255) s_nemit = eoff + myn;
    if (isbig) s_emit[eoff] = Emit{bk.start + excl, cd, cd > big_max ? 0u : 1u, uint32_t(tid)};
    else if (leader) walk(eoff, true);
    __syncthreads();
    const uint32_t ne = s_nemit;
    const K spanmask = (spanv >= W ? ~K(0) : ((K(1) << spanv) - 1)) << lbv;
    const K dmask = K(0xFF) << lowbits;
    const K cbase = K(ws.bor[cur][b]) & ~spanmask & ~dmask;
    // Dense children are the common case (every child of a uniform bucket):
    // reserve their list slots with one atomic per parent, not one per child.
    auto is_dense = [&](const Emit &e) {
      return e.kind == 1 && !(e.count == 1 && cpar == 0) && dense && e.digit != 0xFFFFFFFFu &&
             e.count > 1 && e.count <= big_max;
    };
    // Same for the next level's buckets and their tiles.
    uint32_t mine = 0;   // small | big << 16
    uint32_t mbk = 0;    // large children (next-level buckets)
    uint32_t mtile = 0;  // their tiles
    for (uint32_t i = tid; i < ne; i += 256) {
      const Emit e = s_emit[i];
      if (is_dense(e)) mine += (e.count > ws.dense_max) ? 0x10000u : 1u;
      if (e.kind == 0) {
        mbk += 1;
        mtile += uint32_t((e.count + ws.tile - 1) / ws.tile);
      }
    }
    // packed block scans: (small | big << 16) and (buckets | tiles << 9);
    // per parent small <= 520, big <= 256, buckets <= 256, tiles < 2^23
    const uint32_t mexcl = scan256_excl<256>(mine, s_scan);
    const uint32_t bexcl = scan256_excl<256>(mbk | (mtile << 9), s_scan);
    __shared__ uint32_t s_dbase[4];
    if (tid == 255) {
      const uint32_t tot = mexcl + mine;
      const uint32_t btot = bexcl + (mbk | (mtile << 9));
      s_dbase[0] = (tot & 0xFFFFu) ? atomicAdd(&ws.ctl->ndtasks, tot & 0xFFFFu) : 0u;
      s_dbase[1] = (tot >> 16) ? atomicAdd(&ws.ctl->ndtasks_big, tot >> 16) : 0u;
      s_dbase[2] = (btot & 0x1FFu) ? atomicAdd(&ws.ctl->nbuckets[L + 1], btot & 0x1FFu) : 0u;
      s_dbase[3] = (btot >> 9) ? atomicAdd(&ws.ctl->ntiles[L + 1], btot >> 9) : 0u;
    }
    __syncthreads();
    uint32_t ksmall = s_dbase[0] + (mexcl & 0xFFFFu), kbig = s_dbase[1] + (mexcl >> 16);
    uint32_t kbk = s_dbase[2] + (bexcl & 0x1FFu), ktile = s_dbase[3] + (bexcl >> 9);
    for (uint32_t i = tid; i < ne; i += 256) {
      const Emit e = s_emit[i];
      if (e.kind == 1) {
        if (e.count == 1 && cpar == 0) continue;  // singleton already home: done
        if (is_dense(e)) {
          // small dense tasks fill the list from the front, big ones from the back
          const bool big = e.count > ws.dense_max;
          const uint32_t k = big ? kbig++ : ksmall++;
          if (k < ws.maxtasks / 2) {
            const uint32_t slot = big ? ws.maxtasks - 1 - k : k;
            ws.dtasks[slot] = DTask{e.start, uint64_t(cbase | (K(e.digit) << lowbits)), e.count,
                                    uint32_t(lbv) | (uint32_t(spanv) << 8) | (cpar << 16) |
                                        (uint32_t(dig + 1) << 20)};
          } else {
            atomicOr(&ws.ctl->error, 4u);
          }
        } else {
          // a group of small children still varies in this digit; a standalone child from the next
          emit_tasks(ws, e.start, e.count, cpar, e.digit == 0xFFFFFFFFu ? uint32_t(dig) : uint32_t(dig + 1));
        }
      } else {
        const uint32_t nt = uint32_t((e.count + ws.tile - 1) / ws.tile);
        const uint32_t slot = kbk++, t0 = ktile;
        ktile += nt;
        if (slot >= ws.maxb || t0 + nt > ws.maxtiles) atomicOr(&ws.ctl->error, 3u);
        else ws.buckets[(L + 1) & 1][slot] =
                 Bucket{e.start, e.count, t0, uint32_t(dig + 1), cpar, ACT_SCATTER, h16 ? (BK_HKNOWN | (e.digit << 8)) : 0u};
      }
    }
    __syncthreads();
  }
}

// expand: for every bucket of level L, clear its histogram row / masks and
// map its tiles (tile -> bucket).  One warp per bucket.
__global__ void __launch_bounds__(256) expand_kernel(Ws ws, int L) {
  pdl_wait();  // programmatic dependent launch: previous kernel's writes visible
  if (ws_failed(ws)) return;
  const int cur = L & 1;
  const uint32_t nb = min(ws.ctl->nbuckets[L], ws.maxb);
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t b = gw; b < nb; b += nw) {
    const Bucket bk = ws.buckets[cur][b];
    uint4 *row = reinterpret_cast<uint4 *>(ws.bhist[cur] + size_t(b) * 256);
    if (bk.flags & BK_HKNOWN) {
      // a child of the root: its digit histogram is row d0 of hist16; its
      // masks are the root's with the parent digit fixed to d0 (a superset
      // of the varying bits, which is all plan needs)
      const uint32_t d0 = bk.flags >> 8;
      const uint4 *src = reinterpret_cast<const uint4 *>(ws.hist16 + size_t(d0) * 256);
      for (int i = lane; i < 64; i += 32) row[i] = src[i];
      if (lane == 0) {
        const int pos0 = ws.kbits - 8 - 8 * (int(bk.digit) - 1);
        const uint64_t dm = 0xFFull << pos0, dv = uint64_t(d0) << pos0;
        ws.bor[cur][b] = (ws.bor[0][0] & ~dm) | dv;
        ws.band[cur][b] = (ws.band[0][0] & ~dm) | dv;
      }
    } else {
      for (int i = lane; i < 64; i += 32) row[i] = make_uint4(0, 0, 0, 0);
      if (lane == 0) {
        ws.bor[cur][b] = 0;
        ws.band[cur][b] = ~uint64_t(0);
      }
    }
    const uint32_t nt = uint32_t((bk.count + ws.tile - 1) / ws.tile);
    for (uint32_t i = lane; i < nt; i += 32) ws.tile_bucket[cur][bk.tile0 + i] = b;
  }
}

// ---------------------------------------------------------------------------
// Block ranking.  STABLE: warp-private counters + ballot match (ties keep
// element order; element (w, j, lane) <-> w*32*k + 32*j + lane).  Otherwise
// one block-shared counter per digit and shared-memory atomics (keys-only
// passes whose tie order is immaterial: the MSD scatter and the first LSD
// pass of the local sort).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t match_digit8_ptx(uint32_t d, uint32_t active) {
  uint32_t peers = active;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    uint32_t bb;
    asm volatile(
        "{\n .reg .pred p;\n .reg .u32 t;\n and.b32 t, %1, %2;\n setp.ne.u32 p, t, 0;\n"
        " vote.sync.ballot.b32 %0, p, 0xffffffff;\n @!p not.b32 %0, %0;\n}\n"
        : "=r"(bb)
        : "r"(d), "r"(1u << b));
    peers &= bb;
  }
  return peers;
}

// Ranks (< 65536) of KPT elements packed two per register.
template <int KPT>
struct Ranks {
  uint32_t r[(KPT + 1) / 2];
  __device__ __forceinline__ void clear() {
#pragma unroll
    for (int i = 0; i < (KPT + 1) / 2; ++i) r[i] = 0;
  }
  __device__ __forceinline__ void set(int j, uint32_t v) { r[j >> 1] |= v << (16 * (j & 1)); }
  __device__ __forceinline__ uint32_t get(int j) const { return (r[j >> 1] >> (16 * (j & 1))) & 0xFFFFu; }
};

// Stable warp ranking of the first `kk` (warp-uniform) chunks.
template <int KPT>
__device__ __forceinline__ void warp_rank_stable(const uint32_t (&dig)[KPT], int kk, int nvalid,
                                                 uint32_t *whist, Ranks<KPT> &rank) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int j = 0; j < KPT; ++j) {
    if (j >= kk || 32 * j >= nvalid) break;
    const bool valid = 32 * j + lane < nvalid;
    const uint32_t active = __ballot_sync(0xFFFFFFFFu, valid);
    const uint32_t d = dig[j];
    const uint32_t peers = match_digit8_ptx(d, active);
    const uint32_t below = __popc(peers & lt);
    uint32_t old = 0;
    if (valid && below == 0) {
      old = whist[d];
      whist[d] = old + __popc(peers);
    }
    old = __shfl_sync(0xFFFFFFFFu, old, valid ? (__ffs(peers) - 1) : lane);
    rank.set(j, valid ? old + below : 0u);
    __syncwarp();
  }
}

// After ranking: per digit, prefix over warps (stable) -> whist[w][d] holds
// the exclusive warp prefix; returns the tile total of digit `tid` (< 256).
template <int NW>
__device__ __forceinline__ uint32_t warp_prefix(uint32_t *whist_all) {
  const int tid = threadIdx.x;
  uint32_t s = 0;
  if (tid < 256) {
    uint32_t c[NW];
#pragma unroll
    for (int ww = 0; ww < NW; ++ww) c[ww] = whist_all[ww * 256 + tid];
#pragma unroll
    for (int ww = 0; ww < NW; ++ww) {
      whist_all[ww * 256 + tid] = s;
      s += c[ww];
    }
  }
  return s;
}

// Decoupled look-back for digit `d` of tile `t` (t > tile0): sum the
// predecessors' counts back to the nearest inclusive prefix.  Statuses are
// read 8 tiles at a time so one walk step costs one L2 round trip per 8
// predecessors instead of one per predecessor.
__device__ __forceinline__ uint32_t lookback(const uint32_t *status, uint32_t t, uint32_t tile0, int d) {
  constexpr int WIN = 8;
  uint32_t prefix = 0;
  uint32_t p = t - 1;  // p >= tile0
  for (;;) {
    const int n = int(min(uint32_t(WIN), p - tile0 + 1));
    uint32_t sv[WIN];
#pragma unroll
    for (int i = 0; i < WIN; ++i) sv[i] = (i < n) ? ld_relaxed(status + size_t(p - i) * 256 + d) : 0u;
    int i = 0;
    for (; i < n; ++i) {
      const uint32_t f = sv[i] & ~ST_MASK;
      if (f == 0) break;  // not published yet: re-poll from here
      prefix += sv[i] & ST_MASK;
      if (f == ST_INCL) return prefix;
    }
    p -= uint32_t(i);
  }
}

// ---------------------------------------------------------------------------
// Block-wide exclusive scan of one value per thread (any BLOCK <= 1024).
// ---------------------------------------------------------------------------
template <int BLOCK>
__device__ __forceinline__ uint32_t block_scan_excl(uint32_t x, uint32_t *scratch /* >= 33 words */) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  uint32_t incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) scratch[w] = incl;
  __syncthreads();
  if (w == 0) {
    const uint32_t s = (lane < BLOCK / 32) ? scratch[lane] : 0u;
    uint32_t si = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, si, o);
      if (lane >= o) si += y;
    }
    if (lane < BLOCK / 32) scratch[lane] = si - s;
  }
  __syncthreads();
  const uint32_t r = scratch[w] + incl - x;
  __syncthreads();
  return r;
}

// Inverse of KeyGeom::norm for shift0 == 0 (raw word from its encoded key).
template <typename K, int KIND>
__device__ __forceinline__ K denorm(K nk) {
  constexpr K MSB = K(1) << (KeyTraits<K>::BITS - 1);
  if constexpr (KIND == 0) return nk;
  else if constexpr (KIND == 1) return nk ^ MSB;
  else return (nk & MSB) ? (nk ^ MSB) : ~nk;
}

// ---------------------------------------------------------------------------
// gen16: the output of a whole-input counting sort (plan(0) found every
// varying bit inside the hist16 digit pair and turned hist16 into its
// exclusive prefix).  A warp writes 512 consecutive output positions, lane l
// positions base + l + 32i: the value at p is common | v << shift for the v
// with prefix[v] <= p < prefix[v+1] (one binary search per lane, then a walk).
// ---------------------------------------------------------------------------
template <typename K, int KIND>
__global__ void __launch_bounds__(256) gen16_kernel(Ws ws) {
  pdl_wait();
  if (ws_failed(ws)) return;
  if (ws.ctl->gen == 0u) return;
  const int sh = int(ws.ctl->gen_shift);
  const K common = K(ws.band[0][0]) & ~(K(0xFFFF) << sh);
  const uint32_t *pre = ws.hist16;
  K *dst = static_cast<K *>(ws.keys[0]);
  const uint64_t n = ws.n;
  const int lane = threadIdx.x & 31;
  const uint64_t nwarps = uint64_t(gridDim.x) * (blockDim.x >> 5);
  for (uint64_t base = (uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 512; base < n;
       base += nwarps * 512) {
    uint64_t p = base + lane;
    if (p >= n) continue;
    uint32_t lo = 0, hi = 65535;  // largest v with pre[v] <= p
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      if (uint64_t(pre[mid]) <= p) lo = mid;
      else hi = mid - 1;
    }
    uint32_t v = lo;
    uint64_t next = v < 65535 ? pre[v + 1] : n;
    for (int i = 0; i < 16 && p < n; ++i, p += 32) {
      while (p >= next) {  // walk to the value holding p (empty values skipped)
        ++v;
        next = v < 65535 ? pre[v + 1] : n;
      }
      __stcs(dst + p, denorm<K, KIND>(common | (K(v) << sh)));
    }
  }
}


// Double-buffered input: two (keys[, vals]) buffers filled by TMA bulk copies.
template <typename K, int VB, int CAP>
struct DBuf {
  using V = typename ValT<VB>::T;
  static constexpr size_t kbuf = (sizeof(K) * CAP + 32 + 15) & ~size_t(15);
  static constexpr size_t vbuf = VB ? ((sizeof(V) * CAP + 32 + 15) & ~size_t(15)) : 0;
  static constexpr size_t bytes = 2 * (kbuf + vbuf);
  __device__ static K *keys(unsigned char *base, int i) { return reinterpret_cast<K *>(base + i * kbuf); }
  __device__ static V *vals(unsigned char *base, int i) {
    return reinterpret_cast<V *>(base + 2 * kbuf + i * vbuf);
  }
};

struct InFlight {
  uint64_t start;  // element offset of the range in the array
  uint32_t idx;    // tile id / task id (>= limit: none)
  uint32_t b;      // bucket (scatter)
  uint32_t cnt;
  uint32_t digit;
  uint32_t parity;
  uint32_t tin;
  uint32_t tile0;
  uint32_t headk, headv;
  uint32_t valid;  // data copy issued
};

// Thread 0 only: issue the bulk copies of range [start, start+cnt) of the
// parity-`par` buffers into slot `slot`.
template <typename K, int VB, int CAP>
__device__ __forceinline__ void issue_copy(const Ws &ws, unsigned char *dbuf, uint64_t *bars, int slot,
                                           InFlight &f) {
  using D = DBuf<K, VB, CAP>;
  using V = typename D::V;
  const K *src = static_cast<const K *>(ws.keys[f.parity]) + f.start;
  const Span sk = span16(src, f.cnt);
  Span sv{nullptr, 0, 0};
  if constexpr (VB != 0) sv = span16(static_cast<const V *>(ws.vals[f.parity]) + f.start, f.cnt);
  f.headk = sk.head;
  f.headv = sv.head;
  fence_proxy_async_smem();
  mbar_arrive_expect_tx(&bars[slot], sk.bytes + sv.bytes);
  bulk_g2s(D::keys(dbuf, slot), sk.base, sk.bytes, &bars[slot]);
  if constexpr (VB != 0) bulk_g2s(D::vals(dbuf, slot), sv.base, sv.bytes, &bars[slot]);
}

// ---------------------------------------------------------------------------
// Stable sorts: per-tile digit run offsets, computed ahead of the scatter from
// the tiles' digit counts (hist_kernel wrote them to toff).  A CTA claims a
// block of TS_T consecutive tiles (ticket order), runs a per-digit sum over
// them that restarts at every bucket start, publishes its last segment's
// total (inclusive if that segment's bucket starts inside the block), and --
// if its first segment continues a bucket from earlier blocks -- looks back
// over the earlier blocks' publications (decoupled look-back) for the carry.
// Result: toff[t][d] = digit base in the bucket + number of digit-d elements
// in the bucket's earlier tiles.  Only 1 KB per tile moves and the chain is
// one step per TS_T tiles, so the scatter itself needs no cross-tile wait.
// ---------------------------------------------------------------------------
constexpr int TS_T = 32;  // tiles per tile_scan block

__global__ void __launch_bounds__(256) tile_scan_kernel(Ws ws, int L) {
  pdl_wait();  // programmatic dependent launch: previous kernel's writes visible
  if (ws_failed(ws)) return;
  __shared__ uint32_t s_blk;
  __shared__ uint32_t s_b[TS_T], s_start[TS_T];  // tile's bucket; tile starts its bucket
  const int d = threadIdx.x;
  const int lv = L & 1;
  const uint32_t nt = ws.ctl->ntiles[L];
  for (;;) {
    if (d == 0) s_blk = atomicAdd(&ws.ctl->ticket2[L], 1u);
    __syncthreads();
    const uint32_t blk = s_blk;
    const uint32_t t0 = blk * TS_T;
    if (t0 >= nt) return;
    const uint32_t t1 = min(nt, t0 + uint32_t(TS_T));
    if (d < TS_T && t0 + d < t1) {
      const uint32_t b = ws.tile_bucket[lv][t0 + d];
      s_b[d] = b;
      s_start[d] = ws.buckets[lv][b].tile0 == t0 + d ? 1u : 0u;
    }
    uint32_t c[TS_T];  // all loads in flight at once
#pragma unroll
    for (int i = 0; i < TS_T; ++i) c[i] = t0 + i < t1 ? ws.toff[size_t(t0 + i) * 256 + d] : 0u;
    __syncthreads();
    const bool open_first = s_start[0] == 0u;  // the first segment continues a bucket from earlier blocks
    uint32_t first_end = t1 - t0;             // tiles [0, first_end) continue the first segment
    uint32_t run = 0;
#pragma unroll
    for (int i = 0; i < TS_T; ++i) {
      if (t0 + i < t1) {
        if (s_start[i]) {
          if (i > 0 && first_end == t1 - t0) first_end = uint32_t(i);
          run = 0;
        }
        const uint32_t x = c[i];
        c[i] = run;
        run += x;
      }
    }
    uint32_t *st = ws.status + size_t(blk) * 256 + d;
    const bool chained = open_first && first_end == t1 - t0;  // one open segment: needs the carry
    st_relaxed(st, (chained ? ST_AGG : ST_INCL) | run);
    uint32_t carry = 0;
    if (open_first) {
      carry = lookback(ws.status, blk, 0, d);
      if (chained) st_relaxed(st, ST_INCL | (carry + run));
    }
#pragma unroll
    for (int i = 0; i < TS_T; ++i)
      if (t0 + i < t1)
        ws.toff[size_t(t0 + i) * 256 + d] =
            c[i] + ws.bhist[lv][size_t(s_b[i]) * 256 + d] + (uint32_t(i) < first_end ? carry : 0u);
    __syncthreads();  // s_b / s_start / s_blk are reused by the next block
  }
}

// ---------------------------------------------------------------------------
// K2+K3: scatter one digit with single-pass decoupled look-back.  Persistent
// CTAs claim tiles in order; the next tile is bulk-copied (TMA) into the
// spare buffer while the current one is ranked, scanned and scattered; the
// consumed input buffer doubles as the staging buffer for the coalesced
// write-out.
// ---------------------------------------------------------------------------
template <typename K, int VB, int KIND, int BLOCK, int KPT>
struct ScatterSmem {
  using V = typename ValT<VB>::T;
  using D = DBuf<K, VB, BLOCK * KPT>;
  static constexpr bool STABLE = VB != 0;
  static constexpr int TILE = BLOCK * KPT;
  static constexpr int NW = BLOCK / 32;
  static constexpr size_t dbuf_off = 0;
  static constexpr size_t whist_off = dbuf_off + D::bytes;
  static constexpr size_t gbase_off = whist_off + sizeof(uint32_t) * (STABLE ? NW : 1) * 256;
  static constexpr size_t tstart_off = gbase_off + sizeof(uint64_t) * 256;
  static constexpr size_t misc_off = tstart_off + sizeof(uint32_t) * 256;
  static constexpr size_t bars_off = misc_off + sizeof(uint32_t) * 64;
  static constexpr size_t info_off = bars_off + sizeof(uint64_t) * 2;
  static constexpr size_t bytes = info_off + sizeof(InFlight) * 2;
};

template <typename K, int VB, int KIND, int BLOCK, int KPT>
__global__ void __launch_bounds__(BLOCK, (sizeof(K) + VB) <= 8 ? 3 : 1) scatter_kernel(Ws ws, int L) {
  pdl_wait();  // programmatic dependent launch: previous kernel's writes visible
  if (ws_failed(ws)) return;
  using S = ScatterSmem<K, VB, KIND, BLOCK, KPT>;
  using D = typename S::D;
  using V = typename S::V;
  constexpr bool STABLE = S::STABLE;
  constexpr int TILE = S::TILE;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char *dbuf = smem + S::dbuf_off;
  uint32_t *whist_all = reinterpret_cast<uint32_t *>(smem + S::whist_off);
  uint64_t *gbase = reinterpret_cast<uint64_t *>(smem + S::gbase_off);
  uint32_t *tstart = reinterpret_cast<uint32_t *>(smem + S::tstart_off);
  uint32_t *misc = reinterpret_cast<uint32_t *>(smem + S::misc_off);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + S::bars_off);
  InFlight *info = reinterpret_cast<InFlight *>(smem + S::info_off);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int lv = L & 1;
  const uint32_t nt = ws.ctl->ntiles[L];
  if (nt == 0) return;
  const KeyGeom<K, KIND> g{ws.shift0};
  uint32_t *whist = STABLE ? whist_all + w * 256 : whist_all;

  // thread 0: claim the next tile and start its copy into `slot`
  auto claim = [&](int slot) {
    InFlight f{};
    f.idx = atomicAdd(&ws.ctl->ticket[L], 1u);
    f.valid = 0;
    if (f.idx < nt) {
      const uint32_t b = ws.tile_bucket[lv][f.idx];
      const Bucket bk = ws.buckets[lv][b];
      f.b = b;
      f.tin = f.idx - bk.tile0;
      f.tile0 = bk.tile0;
      f.digit = bk.digit;
      f.parity = bk.parity;
      const uint64_t off = uint64_t(f.tin) * TILE;
      f.start = bk.start + off;
      f.cnt = uint32_t(min64(TILE, bk.count - off));
      if (bk.action == ACT_SCATTER) {
        f.valid = 1;
        issue_copy<K, VB, TILE>(ws, dbuf, bars, slot, f);
      }
    }
    info[slot] = f;
  };

  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    claim(0);
  }
  uint32_t phase = 0;  // bit i: parity of buffer i's next completion
  BS_PROBE_INIT();
  int cur = 0;
  for (;;) {
    if constexpr (STABLE) {
#pragma unroll
      for (int i = lane; i < 256; i += 32) whist[i] = 0;
    } else {
      if (tid < 256) whist[tid] = 0;
    }
    __syncthreads();  // the previous tile's write-out has left buffer cur^1
    // no look-back inside the scatter (tile offsets are precomputed for
    // stable sorts), so the next tile is claimed (and its bulk copy started)
    // as early as possible
    if (tid == 0) claim(cur ^ 1);
    const InFlight f = info[cur];
    if (f.idx >= nt) break;
    if (!f.valid) {
      __syncthreads();
      cur ^= 1;
      continue;
    }
    BS_PROBE(0);
    // stable sorts: this tile's precomputed digit-run offsets, loaded now so
    // the global load overlaps the copy wait and the ranking
    uint32_t toffv = 0;
    if constexpr (STABLE)
      if (tid < 256) toffv = ws.toff[size_t(f.idx) * 256 + tid];
    mbar_wait(&bars[cur], (phase >> cur) & 1u);
    phase ^= 1u << cur;
    BS_PROBE(1);
    K *kb = D::keys(dbuf, cur);
    V *vbp = D::vals(dbuf, cur);
    const int cnt = int(f.cnt);
    const int dig = int(f.digit);
    const int wbase = w * 32 * KPT;
    const DigitFn<K, KIND> dfn(ws.shift0, dig);
    const bool full = cnt == TILE;  // all but the last tile of a bucket
    K x[KPT];
    V v[KPT];
    Ranks<KPT> rk;
    rk.clear();
    if (full) {
#pragma unroll
      for (int j = 0; j < KPT; ++j) {
        const int e = wbase + 32 * j + lane;
        x[j] = kb[f.headk + e];
        if constexpr (VB != 0) v[j] = vbp[f.headv + e];
      }
    } else {
#pragma unroll
      for (int j = 0; j < KPT; ++j) {
        const int e = wbase + 32 * j + lane;
        x[j] = 0;
        if (e < cnt) {
          x[j] = kb[f.headk + e];
          if constexpr (VB != 0) v[j] = vbp[f.headv + e];
        }
      }
    }
    if constexpr (STABLE) {
      uint32_t dg[KPT];
#pragma unroll
      for (int j = 0; j < KPT; ++j) dg[j] = dfn(x[j]);
      warp_rank_stable<KPT>(dg, KPT, max(0, min(32 * KPT, cnt - wbase)), whist, rk);
    } else if (full) {
#pragma unroll
      for (int j = 0; j < KPT; ++j) rk.set(j, atomicAdd(&whist[dfn(x[j])], 1u));
    } else {
#pragma unroll
      for (int j = 0; j < KPT; ++j) {
        const int e = wbase + 32 * j + lane;
        if (e < cnt) rk.set(j, atomicAdd(&whist[dfn(x[j])], 1u));
      }
    }
    __syncthreads();
    BS_PROBE(2);
    uint32_t total;
    if constexpr (STABLE) total = warp_prefix<S::NW>(whist_all);
    else total = (tid < 256) ? whist[tid] : 0u;
    uint32_t texcl;
    const uint32_t bucket_start = uint32_t(f.start - uint64_t(f.tin) * TILE);
    if constexpr (STABLE) {
      // Stable (key-value) sorts: tiles of a bucket must land in tile order,
      // so the offsets come from a single-pass chained scan with decoupled
      // look-back.  Publish this tile's counts first so successors can look
      // past it.
      texcl = scan256_excl<BLOCK>(total, misc);
      BS_PROBE(3);
      if (tid < 256) {
        tstart[tid] = texcl;
        // element offset of this tile's digit-d run minus its tile position
        // (tile_scan_kernel: digit base + earlier tiles' digit-d counts;
        // mod 2^32: true offsets are < n <= 2^30)
        reinterpret_cast<uint32_t *>(gbase)[tid] = bucket_start + toffv - texcl;
      }
    } else {
      // Keys-only MSD: the order of keys inside a child bucket is irrelevant
      // (the child is sorted completely later), so each tile reserves its run
      // per digit with one atomic on the bucket's digit cursor (plan_kernel
      // left the digit bases there) -- no chain across tiles at all.
      uint32_t base = 0;
      if (tid < 256 && total) base = atomicAdd(&ws.bhist[lv][size_t(f.b) * 256 + tid], total);
      texcl = scan256_excl<BLOCK>(total, misc);
      BS_PROBE(3);
      if (tid < 256) {
        tstart[tid] = texcl;
        reinterpret_cast<uint32_t *>(gbase)[tid] = bucket_start + base - texcl;
      }
    }
    __syncthreads();
    BS_PROBE(4);
    // stage in digit order (the input buffer is consumed: keys are in registers)
    auto stage = [&](int j) {
      const uint32_t d = dfn(x[j]);
      uint32_t pos = tstart[d] + rk.get(j);
      if constexpr (STABLE) pos += whist[d];
      kb[pos] = x[j];
      if constexpr (VB != 0) vbp[pos] = v[j];
    };
    if (full) {
#pragma unroll
      for (int j = 0; j < KPT; ++j) stage(j);
    } else {
#pragma unroll
      for (int j = 0; j < KPT; ++j)
        if (wbase + 32 * j + lane < cnt) stage(j);
    }
    __syncthreads();
    BS_PROBE(5);
    K *dst = static_cast<K *>(ws.keys[f.parity ^ 1]);
    V *vdst = VB ? static_cast<V *>(ws.vals[f.parity ^ 1]) : nullptr;
    const uint32_t *gb = reinterpret_cast<const uint32_t *>(gbase);
    if (full) {
#pragma unroll
      for (int j = 0; j < KPT; ++j) {
        const int e = j * BLOCK + tid;
        const K k = kb[e];
        const uint32_t o = gb[dfn(k)] + uint32_t(e);
        BS_DCHECK(ws.ctl, o < ws.n);
        __stcs(dst + o, k);
        if constexpr (VB != 0) __stcs(vdst + o, vbp[e]);
      }
    } else {
      for (int e = tid; e < cnt; e += BLOCK) {
        const K k = kb[e];
        const uint32_t o = gb[dfn(k)] + uint32_t(e);
        BS_DCHECK(ws.ctl, o < ws.n);
        __stcs(dst + o, k);
        if constexpr (VB != 0) __stcs(vdst + o, vbp[e]);
      }
    }
#ifdef BS_PROFILE
    __syncthreads();
#endif
    BS_PROBE(6);
    cur ^= 1;
  }
  BS_PROBE_FLUSH();
}

// ---------------------------------------------------------------------------
// Keys-only scatter, warp-specialised.  One producer warp claims tiles and
// streams them in with TMA bulk copies through a ring of NBUF shared buffers
// (full/empty mbarriers); BLOCK consumer threads rank (shared atomics that
// return each key's slot in its digit, warp-aggregated for skewed warps),
// reserve each digit run with one global atomic per digit, stage the tile in
// digit order in the consumed buffer and write it out coalesced.  Claim
// latency and copy latency both hide behind the consumers' work.
// ---------------------------------------------------------------------------
template <typename K, int KIND, int BLOCK, int KPT, int NBUF>
struct ScatterWsSmem {
  static constexpr int TILE = BLOCK * KPT;
  static constexpr size_t kbuf = (sizeof(K) * TILE + 32 + 15) & ~size_t(15);
  static constexpr size_t dbuf_off = 0;
  static constexpr size_t cnt_off = dbuf_off + NBUF * kbuf;
  static constexpr size_t gbase_off = cnt_off + sizeof(uint32_t) * 256;
  static constexpr size_t tstart_off = gbase_off + sizeof(uint32_t) * 256;
  static constexpr size_t misc_off = tstart_off + sizeof(uint32_t) * 256;
  static constexpr size_t bars_off = misc_off + sizeof(uint32_t) * 64;
  static constexpr size_t info_off = bars_off + sizeof(uint64_t) * 2 * NBUF;
  static constexpr size_t bytes = info_off + sizeof(InFlight) * NBUF;
};

// 256-bin exclusive scan among the BLOCK consumer threads (named barrier 1)
template <int BLOCK>
__device__ __forceinline__ uint32_t scan256_excl_nb(uint32_t v, uint32_t *scratch) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t x = (tid < 256) ? v : 0u;
  uint32_t incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += y;
  }
  if (tid < 256 && lane == 31) scratch[w] = incl;
  named_sync<BLOCK>();
  if (tid < 32) {
    const uint32_t s = (lane < 8) ? scratch[lane] : 0u;
    uint32_t si = s;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, si, o);
      if (lane >= o) si += y;
    }
    if (lane < 8) scratch[lane] = si - s;
  }
  named_sync<BLOCK>();
  return (tid < 256) ? scratch[w] + incl - x : 0u;
}

template <typename K, int KIND, int BLOCK, int KPT, int NBUF>
__global__ void __launch_bounds__(BLOCK + 32, BLOCK >= 512 ? 2 : 3) scatter_ws_kernel(Ws ws, int L) {
  pdl_wait();  // programmatic dependent launch: previous kernel's writes visible
  if (ws_failed(ws)) return;
  using S = ScatterWsSmem<K, KIND, BLOCK, KPT, NBUF>;
  constexpr int TILE = S::TILE;
  extern __shared__ __align__(128) unsigned char smem[];
  uint32_t *cnt256 = reinterpret_cast<uint32_t *>(smem + S::cnt_off);
  uint32_t *gbase = reinterpret_cast<uint32_t *>(smem + S::gbase_off);
  uint32_t *tstart = reinterpret_cast<uint32_t *>(smem + S::tstart_off);
  uint32_t *misc = reinterpret_cast<uint32_t *>(smem + S::misc_off);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + S::bars_off);
  uint64_t *empty = full + NBUF;
  InFlight *info = reinterpret_cast<InFlight *>(smem + S::info_off);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int lv = L & 1;
  const uint32_t nt = ws.ctl->ntiles[L];
  // plan(L) is complete: snapshot the big dense tasks it created
  if (blockIdx.x == 0 && tid == 0) ws.ctl->dbig_end[L] = ws.ctl->ndtasks_big;
  if (nt == 0) return;
  if (tid == BLOCK) {
    for (int i = 0; i < NBUF; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (w == BLOCK / 32) {  // ---------------- producer warp ----------------
    if (lane != 0) return;
    for (uint32_t i = 0;; ++i) {
      const int s = int(i % NBUF);
      if (i >= NBUF) mbar_wait_sleep(&empty[s], ((i / NBUF) - 1) & 1u);
      InFlight f{};
      f.idx = atomicAdd(&ws.ctl->ticket[L], 1u);
      if (f.idx < nt) {
        const uint32_t b = ws.tile_bucket[lv][f.idx];
        const Bucket bk = ws.buckets[lv][b];
        f.b = b;
        f.tin = f.idx - bk.tile0;
        f.digit = bk.digit;
        f.parity = bk.parity;
        const uint64_t off = uint64_t(f.tin) * TILE;
        f.start = bk.start + off;
        f.cnt = uint32_t(min64(TILE, bk.count - off));
        f.valid = bk.action == ACT_SCATTER;
      }
      if (f.valid) {
        const Span sk = span16(static_cast<const K *>(ws.keys[f.parity]) + f.start, f.cnt);
        f.headk = sk.head;
        info[s] = f;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&full[s], sk.bytes);
        bulk_g2s(smem + S::dbuf_off + s * S::kbuf, sk.base, sk.bytes, &full[s]);
      } else {
        info[s] = f;
        mbar_arrive(&full[s]);
      }
      if (f.idx >= nt) return;
    }
  }

  // ---------------- consumers ----------------
  for (uint32_t i = 0;; ++i) {
    const int s = int(i % NBUF);
    mbar_wait(&full[s], (i / NBUF) & 1u);
    const InFlight f = info[s];
    if (f.idx >= nt) break;
    if (f.valid) {
      K *kb = reinterpret_cast<K *>(smem + S::dbuf_off + s * S::kbuf);
      const int cnt = int(f.cnt);
      const DigitFn<K, KIND> dfn(ws.shift0, int(f.digit));
      const bool fullt = cnt == TILE;
      if (tid < 256) cnt256[tid] = 0;
      named_sync<BLOCK>();
      // count with shared atomics that return each key's arrival slot within
      // its digit, scan, then place at tile digit start + slot (a plain load
      // of the start instead of a second read-modify-write per key)
      K x[KPT];
      Ranks<KPT> rk;
      rk.clear();
      // A warp whose 32 keys share one digit (sorted or heavily skewed input)
      // does one aggregated atomic instead of 32 same-address ones.
      // The check costs a shuffle and a vote per key, so a warp only uses it
      // when its first 32 keys already share a digit.
      if (fullt) {
#pragma unroll
        for (int j = 0; j < KPT; ++j) x[j] = kb[f.headk + j * BLOCK + tid];
        const uint32_t e0 = dfn(x[0]);
        const bool skew = __all_sync(0xFFFFFFFFu, e0 == __shfl_sync(0xFFFFFFFFu, e0, 0));
        if (skew) {
#pragma unroll
          for (int j = 0; j < KPT; ++j) {
            const uint32_t d = dfn(x[j]);
            const uint32_t d0 = __shfl_sync(0xFFFFFFFFu, d, 0);
            if (__all_sync(0xFFFFFFFFu, d == d0)) {
              uint32_t b0 = 0;
              if (lane == 0) b0 = atomicAdd(&cnt256[d0], 32u);
              rk.set(j, __shfl_sync(0xFFFFFFFFu, b0, 0) + uint32_t(lane));
            } else {
              rk.set(j, atomicAdd(&cnt256[d], 1u));
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < KPT; ++j) rk.set(j, atomicAdd(&cnt256[dfn(x[j])], 1u));
        }
      } else {
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
          const int e = j * BLOCK + tid;
          x[j] = 0;
          if (e < cnt) {
            x[j] = kb[f.headk + e];
            rk.set(j, atomicAdd(&cnt256[dfn(x[j])], 1u));
          }
        }
      }
      named_sync<BLOCK>();
      const uint32_t total = (tid < 256) ? cnt256[tid] : 0u;
      uint32_t base = 0;
      if (tid < 256 && total) base = atomicAdd(&ws.bhist[lv][size_t(f.b) * 256 + tid], total);
      const uint32_t texcl = scan256_excl_nb<BLOCK>(total, misc);
      if (tid < 256) {
        tstart[tid] = texcl;
        gbase[tid] = uint32_t(f.start - uint64_t(f.tin) * TILE) + base - texcl;
      }
      named_sync<BLOCK>();
      if (fullt) {
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
          BS_DCHECK(ws.ctl, tstart[dfn(x[j])] + rk.get(j) < uint32_t(TILE));
          kb[tstart[dfn(x[j])] + rk.get(j)] = x[j];
        }
      } else {
#pragma unroll
        for (int j = 0; j < KPT; ++j)
          if (j * BLOCK + tid < cnt) {
            BS_DCHECK(ws.ctl, tstart[dfn(x[j])] + rk.get(j) < uint32_t(cnt));
            kb[tstart[dfn(x[j])] + rk.get(j)] = x[j];
          }
      }
      named_sync<BLOCK>();
      K *dst = static_cast<K *>(ws.keys[f.parity ^ 1]);
      if (fullt) {
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
          const int e = j * BLOCK + tid;
          const K k = kb[e];
          BS_DCHECK(ws.ctl, gbase[dfn(k)] + uint32_t(e) < ws.n);
          __stcs(dst + (gbase[dfn(k)] + uint32_t(e)), k);
        }
      } else {
        for (int e = tid; e < cnt; e += BLOCK) {
          const K k = kb[e];
          BS_DCHECK(ws.ctl, gbase[dfn(k)] + uint32_t(e) < ws.n);
          __stcs(dst + (gbase[dfn(k)] + uint32_t(e)), k);
        }
      }
    }
    named_sync<BLOCK>();  // every consumer is done with buffer s
    if (tid == 0) mbar_arrive(&empty[s]);
  }
}

// ---------------------------------------------------------------------------
// K4: local sort of one task (<= BLOCK*KPT elements) per CTA iteration; the
// next task streams in by TMA bulk copy while the current one is sorted.
//  * Dense keys-only tasks (full-width words, all varying bits inside a
//    16-bit span -- the common case after two 8-bit MSD levels): counting sort
//    through a presence bitmap, one shared atomic per key, emitted in value
//    order.
//  * Otherwise LSD over the task's varying digits only (constant digits are
//    the reference's pass-throughs), keys (+values) in registers, k =
//    ceil(n/BLOCK) per thread; the first keys-only pass ranks with shared
//    atomics, later passes (and all passes with values) with the stable
//    ballot ranking.
// The consumed input buffer is the staging buffer of every pass; the final
// pass is written coalesced to the caller's buffer.
// ---------------------------------------------------------------------------
template <typename K, int VB, int KIND, int BLOCK, int KPT>
struct LocalSmem {
  using V = typename ValT<VB>::T;
  static constexpr int CAP = BLOCK * KPT;
  using D = DBuf<K, VB, CAP>;
  static constexpr int NW = BLOCK / 32;
  static constexpr int BM_WORDS = 2048;  // 2^16 values
  static constexpr int OVF_CAP = 1024;
  static constexpr size_t dbuf_off = 0;
  static constexpr size_t whist_off = dbuf_off + D::bytes;
  static constexpr size_t whist_bytes = sizeof(uint32_t) * NW * 256;
  static constexpr size_t bm_bytes = VB ? 0 : sizeof(uint32_t) * (4 * BM_WORDS + OVF_CAP + 4);
  static constexpr size_t tstart_off = whist_off + (whist_bytes > bm_bytes ? whist_bytes : bm_bytes);
  static constexpr size_t red_off = tstart_off + sizeof(uint32_t) * 256;
  static constexpr size_t misc_off = red_off + sizeof(uint64_t) * 2 * NW;
  static constexpr size_t bars_off = misc_off + sizeof(uint32_t) * 64;
  static constexpr size_t info_off = bars_off + sizeof(uint64_t) * 2;
  static constexpr size_t bytes = info_off + sizeof(InFlight) * 2;
};

template <typename K, int VB, int KIND, int BLOCK, int KPT>
__global__ void __launch_bounds__(BLOCK, (VB == 0 && sizeof(K) == 8 && BLOCK <= 512) ? 2 : 1) local_kernel(Ws ws, int list) {
  pdl_wait();  // programmatic dependent launch: previous kernel's writes visible
  if (ws_failed(ws)) return;
  using S = LocalSmem<K, VB, KIND, BLOCK, KPT>;
  using D = typename S::D;
  using V = typename S::V;
  constexpr int W = KeyTraits<K>::BITS;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char *dbuf = smem + S::dbuf_off;
  uint32_t *whist_all = reinterpret_cast<uint32_t *>(smem + S::whist_off);
  uint32_t *tstart = reinterpret_cast<uint32_t *>(smem + S::tstart_off);
  uint64_t *red = reinterpret_cast<uint64_t *>(smem + S::red_off);
  uint32_t *misc = reinterpret_cast<uint32_t *>(smem + S::misc_off);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + S::bars_off);
  InFlight *info = reinterpret_cast<InFlight *>(smem + S::info_off);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  // list 0: the task list; list 1: the tasks spread_kernel handed over (all of
  // them when the input is skewed and spread_kernel stood aside)
  if (list && ws.ctl->skewed) list = 0;
  const Task *tasks = list ? ws.tasks2 : ws.tasks;
  const uint32_t ntasks = min(list ? ws.ctl->ntasks2 : ws.ctl->ntasks, ws.maxtasks);
  if (blockIdx.x >= ntasks) return;
  const KeyGeom<K, KIND> g{ws.shift0};
  uint32_t *whist = whist_all + w * 256;

  auto prepare = [&](int slot, uint32_t ti) {
    InFlight f{};
    f.idx = ti;
    f.valid = 0;
    if (ti < ntasks) {
      const Task tk = tasks[ti];
      f.start = tk.start;
      f.cnt = tk.count;
      f.parity = tk.parity & 1u;
      f.valid = 1;
      issue_copy<K, VB, S::CAP>(ws, dbuf, bars, slot, f);
    }
    info[slot] = f;
  };

  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    prepare(0, blockIdx.x);
  }
  uint32_t phase = 0;
  int cur = 0;
  for (uint32_t ti = blockIdx.x; ti < ntasks; ti += gridDim.x) {
    __syncthreads();  // previous task fully consumed; info[cur] visible
    if (tid == 0) prepare(cur ^ 1, ti + gridDim.x);
    const InFlight f = info[cur];
    mbar_wait(&bars[cur], (phase >> cur) & 1u);
    phase ^= 1u << cur;
    K *kb = D::keys(dbuf, cur);
    V *vbp = D::vals(dbuf, cur);
    const int n = int(f.cnt);
    const int kk = (n + BLOCK - 1) / BLOCK;  // elements per thread for this task
    const int wbase = w * 32 * kk;
    const int nvw = max(0, min(32 * kk, n - wbase));
    K *dst = static_cast<K *>(ws.keys[0]) + f.start;
    V *vdst = VB ? static_cast<V *>(ws.vals[0]) + f.start : nullptr;
    K x[KPT];
    V v[KPT];
    K o = 0, a = ~K(0);
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      if (j >= kk) break;
      const int e = wbase + 32 * j + lane;
      x[j] = 0;
      if (32 * j + lane < nvw) {
        x[j] = kb[f.headk + e];
        if constexpr (VB != 0) v[j] = vbp[f.headv + e];
        const K nk = g.norm(x[j]);
        o |= nk;
        a &= nk;
      }
    }
    o = warp_or(o);
    a = warp_and(a);
    if (lane == 0) {
      red[w] = o;
      red[S::NW + w] = a;
    }
    __syncthreads();
    K var, common;
    {  // every warp folds the per-warp masks with shuffles (not NW loads per thread)
      const K oo = warp_or(lane < S::NW ? K(red[lane]) : K(0));
      const K aa = warp_and(lane < S::NW ? K(red[S::NW + lane]) : ~K(0));
      var = oo ^ aa;
      common = oo;
    }
    if (var == 0) {
      if (f.parity) {
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
          if (j >= kk) break;
          const int e = wbase + 32 * j + lane;
          if (32 * j + lane < nvw) {
            dst[e] = x[j];
            if constexpr (VB != 0) vdst[e] = v[j];
          }
        }
      }
      cur ^= 1;
      continue;
    }
    bool done = false;
    if constexpr (VB == 0) {
      const int lb = __ffsll((long long)(uint64_t(var))) - 1;
      const int span = W - KeyTraits<K>::clz(var) - lb;
      if (ws.shift0 == 0 && span <= 16) {
        // B1: value present, B2: a second copy, EX: per-word count of further
        // copies (listed in OVF), WP: per-word exclusive prefix of all copies.
        uint32_t *B1 = whist_all;
        uint32_t *B2 = B1 + S::BM_WORDS;
        uint32_t *EX = B2 + S::BM_WORDS;
        uint32_t *WP = EX + S::BM_WORDS;
        uint32_t *OVF = WP + S::BM_WORDS;
        uint32_t *novf = OVF + S::OVF_CAP;
        const int nwords = span <= 5 ? 1 : (1 << (span - 5));
        for (int i = tid; i < nwords; i += BLOCK) {
          B1[i] = 0;
          B2[i] = 0;
          EX[i] = 0;
        }
        if (tid == 0) *novf = 0;
        __syncthreads();
        const K spanmask = (span >= W ? ~K(0) : ((K(1) << span) - 1)) << lb;
        Ranks<KPT> cp;  // copy index: 0 first, 1 second, 2 + overflow slot
        cp.clear();
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
          if (j >= kk) break;
          if (32 * j + lane < nvw) {
            const uint32_t idx = uint32_t((g.norm(x[j]) & spanmask) >> lb);
            const uint32_t bit = 1u << (idx & 31);
            if (atomicOr(&B1[idx >> 5], bit) & bit) {
              uint32_t c = 1;
              if (atomicOr(&B2[idx >> 5], bit) & bit) {
                atomicAdd(&EX[idx >> 5], 1u);
                const uint32_t sl = atomicAdd(novf, 1u);
                if (sl < S::OVF_CAP) OVF[sl] = idx;
                c = 2 + min(sl, uint32_t(S::OVF_CAP));
              }
              cp.set(j, c);
            }
          }
        }
        __syncthreads();
        const uint32_t nov = *novf;
        if (nov <= S::OVF_CAP) {
          const int wpt = (nwords + BLOCK - 1) / BLOCK;
          const int w0 = min(nwords, tid * wpt), w1 = min(nwords, w0 + wpt);
          uint32_t c = 0;
          for (int q = w0; q < w1; ++q) c += __popc(B1[q]) + __popc(B2[q]) + EX[q];
          uint32_t run = block_scan_excl<BLOCK>(c, misc);
          for (int q = w0; q < w1; ++q) {
            WP[q] = run;
            run += __popc(B1[q]) + __popc(B2[q]) + EX[q];
          }
          __syncthreads();
          // each key's position = copies of smaller values + its copy index
#pragma unroll
          for (int j = 0; j < KPT; ++j) {
            if (j >= kk) break;
            if (32 * j + lane < nvw) {
              const uint32_t idx = uint32_t((g.norm(x[j]) & spanmask) >> lb);
              const uint32_t q = idx >> 5, low = (1u << (idx & 31)) - 1u;
              uint32_t pos = WP[q] + __popc(B1[q] & low) + __popc(B2[q] & low);
              const uint32_t c = cp.get(j);
              if (EX[q]) {  // rare: >= 3 copies of some value in this word
                for (uint32_t i = 0; i < nov; ++i) {
                  const uint32_t o = OVF[i];
                  pos += ((o >> 5) == q && o < idx) ? 1u : 0u;
                  pos += (c >= 2 && o == idx && i < c - 2) ? 1u : 0u;
                }
              }
              kb[pos + (c < 2 ? c : 2u)] = x[j];
            }
          }
          __syncthreads();
          done = true;
        }
        // else: too many repeats for the overflow list -> LSD passes below
      }
      // Bin sort (keys only, any span): one counting pass on the top B varying
      // bits with 2^B >= 2n bins (about half a key per bin), then every key
      // finds its place inside its bin by comparing itself with the bin's few
      // other keys -- one shared atomic, two scattered stores and ~2 loads per
      // key instead of one ranking pass per varying digit.  A bin whose keys
      // are all equal ranks them by arrival; the mixed bins cost sum(c^2)
      // comparisons over their sizes c (~1.5n for spread keys); a task above
      // 8n takes the LSD passes below.
      if (!done && n >= 64) {
        constexpr int BIN_LOG_MAX = 13;  // 8192 counters fit the bitmap region
        static_assert(sizeof(uint32_t) * (1u << BIN_LOG_MAX) <= S::bm_bytes, "bins fit");
        const int hb = W - 1 - KeyTraits<K>::clz(var);  // top varying bit of the normalised key
        int B = 33 - __clz(uint32_t(n - 1));  // about two bins per key: short in-bin loops
        B = min(min(B, BIN_LOG_MAX), hb + 1);
        const int sh = hb + 1 - B;
        const uint32_t nbins = 1u << B, bmask = nbins - 1u;
        uint32_t *bins = whist_all;
        for (uint32_t i = tid; i < (nbins + 3) / 4; i += BLOCK) reinterpret_cast<uint4 *>(bins)[i] = make_uint4(0, 0, 0, 0);
        if (tid == 0) misc[48] = 0;
        __syncthreads();
        // comparisons a plain in-bin ranking needs: sum over bins of c^2 =
        // sum over keys of (2 * arrival slot + 1) -- no pass over the bins
        Ranks<KPT> slot;  // arrival slot inside the bin
        slot.clear();
        uint32_t c2 = 0;
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
          if (j >= kk) break;
          if (32 * j + lane < nvw) {
            const uint32_t sl = atomicAdd(&bins[uint32_t(g.norm(x[j]) >> sh) & bmask], 1u);
            slot.set(j, sl);
            c2 += 2u * sl + 1u;
          }
        }
        c2 = __reduce_add_sync(0xFFFFFFFFu, c2);
        if (lane == 0 && c2) atomicAdd(&misc[48], c2);
        __syncthreads();
        const uint32_t bpt = (nbins + BLOCK - 1) / BLOCK;
        const uint32_t q0 = min(nbins, uint32_t(tid) * bpt), q1 = min(nbins, q0 + bpt);
        const bool vec = (bpt & 3u) == 0u;  // whole uint4 chunks (conflict-free scan loads)
        {
          uint4 *b4 = reinterpret_cast<uint4 *>(bins);
          uint32_t c = 0;
          if (vec) {
            for (uint32_t q = q0 / 4; q < q1 / 4; ++q) {
              const uint4 v = b4[q];
              c += v.x + v.y + v.z + v.w;
            }
          } else {
            for (uint32_t q = q0; q < q1; ++q) c += bins[q];
          }
          uint32_t run = block_scan_excl<BLOCK>(c, misc);
          if (vec) {
            for (uint32_t q = q0 / 4; q < q1 / 4; ++q) {
              const uint4 v = b4[q];
              uint4 o;
              o.x = run, run += v.x;
              o.y = run, run += v.y;
              o.z = run, run += v.z;
              o.w = run, run += v.w;
              b4[q] = o;
            }
          } else {
            for (uint32_t q = q0; q < q1; ++q) {
              const uint32_t v = bins[q];
              bins[q] = run;
              run += v;
            }
          }
        }
        const bool spread = misc[48] <= 8u * uint32_t(n);  // (block_scan synced)
        __syncthreads();
        if (tid == 0) misc[48] = 0;
        // bin order (arbitrary inside a bin)
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
          if (j >= kk) break;
          if (32 * j + lane < nvw) kb[bins[uint32_t(g.norm(x[j]) >> sh) & bmask] + slot.get(j)] = x[j];
        }
        __syncthreads();
        // Duplicate-heavy tasks: a bin is "pure" when all its keys equal its
        // first one; its keys rank by arrival, no comparisons.  Flag the mixed
        // bins and count only their comparisons.
        constexpr uint32_t MIXED = 0x80000000u, OFF = 0x7FFFFFFFu;
        if (!spread) {
#pragma unroll
          for (int j = 0; j < KPT; ++j) {
            if (j >= kk) break;
            if (32 * j + lane < nvw) {
              const uint32_t d = uint32_t(g.norm(x[j]) >> sh) & bmask;
              const uint32_t s0 = bins[d] & OFF;
              if (kb[s0] != x[j]) atomicOr(&bins[d], MIXED);
            }
          }
          __syncthreads();
          uint32_t c2 = 0;
          for (uint32_t q = tid; q < nbins; q += BLOCK) {  // strided: conflict-free
            const uint32_t bq = bins[q];
            if (bq & MIXED) {
              const uint32_t c = (q < bmask ? (bins[q + 1] & OFF) : uint32_t(n)) - (bq & OFF);
              c2 += c * c;
            }
          }
          c2 = __reduce_add_sync(0xFFFFFFFFu, c2);
          if (lane == 0 && c2) atomicAdd(&misc[48], c2);
          __syncthreads();
        }
        if (spread || misc[48] <= 8u * uint32_t(n)) {
          // place inside the bin: smaller keys, then equal keys that arrived earlier
          Ranks<KPT> fin;
          fin.clear();
#pragma unroll
          for (int j = 0; j < KPT; ++j) {
            if (j >= kk) break;
            if (32 * j + lane < nvw) {
              const K nk = g.norm(x[j]);
              const uint32_t d = uint32_t(nk >> sh) & bmask;
              const uint32_t bd = bins[d], s0 = bd & OFF;
              const uint32_t e = d < bmask ? (bins[d + 1] & OFF) : uint32_t(n);
              const uint32_t p = s0 + slot.get(j);
              uint32_t r = 0;
              if (spread ? e - s0 <= 1u : !(bd & MIXED)) {
                r = slot.get(j);  // alone, or all equal: arrival order
              } else {
                for (uint32_t i = s0; i < e; ++i) {
                  const K y = g.norm(kb[i]);
                  r += (y < nk || (y == nk && i < p)) ? 1u : 0u;
                }
              }
              fin.set(j, s0 + r);
            }
          }
          __syncthreads();
#pragma unroll
          for (int j = 0; j < KPT; ++j) {
            if (j >= kk) break;
            if (32 * j + lane < nvw) kb[fin.get(j)] = x[j];
          }
          __syncthreads();
          done = true;
        }
      }
    }
    if (!done) {
      // digits that vary, least significant first
      const int lastd = (W - 1 - (__ffsll((long long)(uint64_t(var))) - 1)) >> 3;
      const int firstd = KeyTraits<K>::clz(var) >> 3;
      bool first = true;
      for (int dig = lastd; dig >= firstd; --dig) {
        if (((var >> (W - 8 - 8 * dig)) & K(0xFF)) == 0) continue;
        if (!first) {
          // reload in element order from the previous pass
#pragma unroll
          for (int j = 0; j < KPT; ++j) {
            if (j >= kk) break;
            const int e = wbase + 32 * j + lane;
            if (32 * j + lane < nvw) {
              x[j] = kb[e];
              if constexpr (VB != 0) v[j] = vbp[e];
            }
          }
          __syncthreads();
        }
        const bool atomic_pass = (VB == 0) && first;
        Ranks<KPT> rk;
        rk.clear();
        if (atomic_pass) {
          if (tid < 256) whist_all[tid] = 0;
          __syncthreads();
#pragma unroll
          for (int j = 0; j < KPT; ++j) {
            if (j >= kk) break;
            if (32 * j + lane < nvw) rk.set(j, atomicAdd(&whist_all[g.digit(x[j], dig)], 1u));
          }
        } else {
#pragma unroll
          for (int i = lane; i < 256; i += 32) whist[i] = 0;
          __syncwarp();
          uint32_t dg[KPT];
#pragma unroll
          for (int j = 0; j < KPT; ++j) dg[j] = (j < kk) ? g.digit(x[j], dig) : 0u;
          warp_rank_stable<KPT>(dg, kk, nvw, whist, rk);
        }
        __syncthreads();
        const uint32_t total =
            atomic_pass ? ((tid < 256) ? whist_all[tid] : 0u) : warp_prefix<S::NW>(whist_all);
        const uint32_t texcl = scan256_excl<BLOCK>(total, misc);
        if (tid < 256) tstart[tid] = texcl;
        __syncthreads();
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
          if (j >= kk) break;
          if (32 * j + lane < nvw) {
            const uint32_t d = g.digit(x[j], dig);
            const uint32_t pos = tstart[d] + rk.get(j) + (atomic_pass ? 0u : whist[d]);
            BS_DCHECK(ws.ctl, pos < uint32_t(n));
            kb[pos] = x[j];
            if constexpr (VB != 0) vbp[pos] = v[j];
          }
        }
        __syncthreads();
        first = false;
      }
    }
    BS_DCHECK(ws.ctl, f.start + uint64_t(n) <= ws.n);
    for (int e = tid; e < n; e += BLOCK) {
      __stcs(dst + e, kb[e]);
      if constexpr (VB != 0) __stcs(vdst + e, vbp[e]);
    }
    cur ^= 1;
  }
}

}  // namespace bs
