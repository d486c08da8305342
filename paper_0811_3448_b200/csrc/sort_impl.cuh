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

#include "common.cuh"

namespace bs {

constexpr int MAXLEV = 9;  // >= max digits (8 for u64) + 1
constexpr uint32_t ST_AGG = 1u << 30;
constexpr uint32_t ST_INCL = 2u << 30;
constexpr uint32_t ST_MASK = (1u << 30) - 1;

enum : uint32_t { ACT_SCATTER = 0, ACT_SKIP = 1 };

struct Bucket {
  uint64_t start;
  uint32_t count;
  uint32_t tile0;
  uint32_t digit;
  uint32_t parity;  // 0: live data in the caller's buffer, 1: in the workspace copy
  uint32_t action;
  uint32_t pad;
};

struct Task {
  uint64_t start;
  uint32_t count;
  uint32_t parity;
};

struct Ctl {
  uint32_t nbuckets[MAXLEV + 1];
  uint32_t ntiles[MAXLEV + 1];
  uint32_t ticket[MAXLEV + 1];
  uint32_t ntasks;
  uint32_t task_ticket;
  uint32_t error;  // bit 0: bucket overflow, 1: tile overflow, 2: task overflow
  uint32_t pad;
};

// Workspace view (all device pointers), built on the host.
struct Ws {
  Ctl *ctl;
  Bucket *buckets[2];
  uint32_t *bhist[2];  // [maxb][256]; counts, then (after plan) digit bases
  uint64_t *bor[2];
  uint64_t *band[2];
  uint32_t *tile_bucket[2];
  uint32_t *status;  // [maxtiles][256]
  Task *tasks;
  void *keys[2];  // [0] caller's buffer, [1] workspace copy
  void *vals[2];
  uint64_t n;
  uint32_t maxb, maxtiles, maxtasks;
  uint32_t tile;       // elements per scatter tile
  uint32_t local_max;  // largest range the local sort takes
  uint32_t group_min;  // children smaller than this are grouped
  int ndig;            // number of 8-bit digits of the effective key
  int shift0;          // W - width_eff
};


// ---------------------------------------------------------------------------
// init: root bucket (or a single local task when n fits the local sort).
// A strided sample guesses the first varying digit so constant leading digits
// (e.g. "low 16 bits random" u64 keys) cost no wasted histogram pass.
// ---------------------------------------------------------------------------
template <typename K, int KIND>
__global__ void init_kernel(Ws ws) {
  const int tid = threadIdx.x;
  const uint64_t n = ws.n;
  const KeyGeom<K, KIND> g{ws.shift0};
  if (n <= ws.local_max) {
    if (blockIdx.x == 0 && tid == 0) {
      ws.tasks[0] = Task{0, uint32_t(n), 0};
      ws.ctl->ntasks = 1;
    }
    return;
  }
  const uint32_t ntiles = uint32_t((n + ws.tile - 1) / ws.tile);
  for (uint32_t t = blockIdx.x * blockDim.x + tid; t < ntiles; t += gridDim.x * blockDim.x)
    ws.tile_bucket[0][t] = 0;
  for (int d = tid; d < 256; d += blockDim.x) ws.bhist[0][d] = 0;
  if (blockIdx.x != 0) return;
  __shared__ uint64_t s_or[32], s_and[32];
  // 4096-element strided sample of the encoded normalised key
  K o = 0, a = ~K(0);
  const K *keys = static_cast<const K *>(ws.keys[0]);
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
    ws.buckets[0][0] = Bucket{0, uint32_t(n), 0, uint32_t(dig), 0, ACT_SCATTER, 0};
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
  constexpr int NCOPY = 4;
  __shared__ uint32_t h[NCOPY][256];
  __shared__ uint64_t s_or[BLOCK / 32], s_and[BLOCK / 32];
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
  K o = 0, a = ~K(0);
  uint32_t curb = 0xFFFFFFFFu;
  int dig = 0;
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
      if (curb != 0xFFFFFFFFu) flush(curb);
      curb = b;
      dig = int(bk.digit);
    }
    // clear this tile's look-back row (256 x u32 = 64 x uint4)
    if (tid < 64)
      reinterpret_cast<uint4 *>(ws.status + size_t(t) * 256)[tid] = make_uint4(0, 0, 0, 0);
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
  }
  flush(curb);
}

// ---------------------------------------------------------------------------
// plan: one CTA (256 threads) per bucket of level L.
// ---------------------------------------------------------------------------
struct Emit {
  uint64_t start;
  uint32_t count;
  uint32_t kind;  // 0 large child (next level), 1 local task
};

__device__ __forceinline__ void emit_tasks(const Ws &ws, uint64_t start, uint64_t count,
                                           uint32_t parity) {
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
    ws.tasks[base + c] = Task{start + s, uint32_t(min64(ws.local_max, count - s)), parity};
  }
}

template <typename K>
__global__ void __launch_bounds__(256) plan_kernel(Ws ws, int L) {
  constexpr int W = KeyTraits<K>::BITS;
  __shared__ uint32_t s_cnt[256];
  __shared__ uint32_t s_scan[16];
  __shared__ Emit s_emit[520];
  __shared__ uint32_t s_nemit;
  __shared__ uint32_t s_slot[520];
  const int tid = threadIdx.x;
  const int cur = L & 1, nxt = cur ^ 1;
  const uint32_t nb = ws.ctl->nbuckets[L];
  for (uint32_t b = blockIdx.x; b < nb; b += gridDim.x) {
    Bucket bk = ws.buckets[cur][b];
    uint32_t *hist = ws.bhist[cur] + size_t(b) * 256;
    const uint32_t c = hist[tid];
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
        if (bk.count <= ws.local_max) {
          emit_tasks(ws, bk.start, bk.count, bk.parity);
        } else {
          const uint32_t slot = atomicAdd(&ws.ctl->nbuckets[L + 1], 1u);
          const uint32_t nt = uint32_t((bk.count + ws.tile - 1) / ws.tile);
          const uint32_t t0 = atomicAdd(&ws.ctl->ntiles[L + 1], nt);
          if (slot >= ws.maxb || t0 + nt > ws.maxtiles) {
            atomicOr(&ws.ctl->error, 3u);
          } else {
            ws.buckets[nxt][slot] = Bucket{bk.start, bk.count, t0, uint32_t(dstar), bk.parity, ACT_SCATTER, 0};
            ws.bor[nxt][slot] = 0;
            ws.band[nxt][slot] = ~uint64_t(0);
            s_slot[0] = slot;
            s_emit[0] = Emit{bk.start, bk.count, t0};
          }
        }
      }
      __syncthreads();
      // requeued bucket: zero its histogram row and map its tiles (whole CTA)
      if (bk.count > ws.local_max && !(ws.ctl->error & 3u)) {
        const uint32_t slot = s_slot[0];
        const uint32_t t0 = s_emit[0].kind;
        const uint32_t nt = uint32_t((bk.count + ws.tile - 1) / ws.tile);
        ws.bhist[nxt][size_t(slot) * 256 + tid] = 0;
        for (uint32_t i = tid; i < nt; i += 256) ws.tile_bucket[nxt][t0 + i] = slot;
      }
      __syncthreads();
      continue;
    }
    // scatter this bucket on digit `dig`
    const uint32_t excl = scan256_excl<256>(c, s_scan);
    hist[tid] = excl;  // digit base within the bucket
    s_cnt[tid] = c;
    if (tid == 0) ws.buckets[cur][b].action = ACT_SCATTER;
    const uint32_t cpar = bk.parity ^ 1u;
    const int lowbits = W - 8 - 8 * dig;
    const K lower = lowbits > 0 ? (var & ((K(1) << lowbits) - 1)) : K(0);
    if (lower == 0) {  // every child is all-equal: only a copy home may remain
      if (tid == 0 && cpar) emit_tasks(ws, bk.start, bk.count, 1);
      __syncthreads();
      continue;
    }
    __syncthreads();
    if (tid == 0) {
      // greedy in digit order: large children go to the next level, mid-size
      // ones become local tasks, small ones are grouped up to local_max
      uint32_t ne = 0;
      uint64_t gs = 0;
      uint32_t gc = 0;
      uint64_t pos = bk.start;
      for (int d = 0; d < 256; ++d) {
        const uint32_t cd = s_cnt[d];
        if (cd == 0) continue;
        if (cd > ws.local_max || cd >= ws.group_min) {
          if (gc) s_emit[ne++] = Emit{gs, gc, 1};
          gc = 0;
          s_emit[ne++] = Emit{pos, cd, cd > ws.local_max ? 0u : 1u};
        } else {
          if (gc + cd > ws.local_max) {
            s_emit[ne++] = Emit{gs, gc, 1};
            gc = 0;
          }
          if (gc == 0) gs = pos;
          gc += cd;
        }
        pos += cd;
      }
      if (gc) s_emit[ne++] = Emit{gs, gc, 1};
      s_nemit = ne;
    }
    __syncthreads();
    const uint32_t ne = s_nemit;
    for (uint32_t i = tid; i < ne; i += 256) {
      const Emit e = s_emit[i];
      if (e.kind == 1) {
        // a singleton already home needs nothing
        if (!(e.count == 1 && cpar == 0)) emit_tasks(ws, e.start, e.count, cpar);
        s_slot[i] = 0xFFFFFFFFu;
      } else {
        const uint32_t slot = atomicAdd(&ws.ctl->nbuckets[L + 1], 1u);
        const uint32_t nt = uint32_t((e.count + ws.tile - 1) / ws.tile);
        const uint32_t t0 = atomicAdd(&ws.ctl->ntiles[L + 1], nt);
        if (slot >= ws.maxb || t0 + nt > ws.maxtiles) {
          atomicOr(&ws.ctl->error, 3u);
          s_slot[i] = 0xFFFFFFFFu;
        } else {
          ws.buckets[nxt][slot] = Bucket{e.start, e.count, t0, uint32_t(dig + 1), cpar, ACT_SCATTER, 0};
          ws.bor[nxt][slot] = 0;
          ws.band[nxt][slot] = ~uint64_t(0);
          s_slot[i] = slot;
          s_emit[i].kind = 2u + t0;  // remember tile0 (kind >= 2 marks "large")
        }
      }
    }
    __syncthreads();
    for (uint32_t i = 0; i < ne; ++i) {
      const uint32_t slot = s_slot[i];
      if (slot == 0xFFFFFFFFu) continue;
      const Emit e = s_emit[i];
      const uint32_t t0 = e.kind - 2u;
      const uint32_t nt = uint32_t((e.count + ws.tile - 1) / ws.tile);
      ws.bhist[nxt][size_t(slot) * 256 + tid] = 0;
      for (uint32_t k = tid; k < nt; k += 256) ws.tile_bucket[nxt][t0 + k] = slot;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K2+K3: stable scatter of one digit with single-pass decoupled look-back.
// ---------------------------------------------------------------------------
template <typename K, int VB, int KIND, int BLOCK, int KPT>
struct ScatterSmem {
  using V = typename ValT<VB>::T;
  static constexpr int TILE = BLOCK * KPT;
  static constexpr int NW = BLOCK / 32;
  static constexpr size_t keys_off = 0;
  static constexpr size_t vals_off = keys_off + sizeof(K) * TILE;
  static constexpr size_t whist_off = vals_off + (VB ? sizeof(V) * TILE : 0);
  static constexpr size_t gbase_off = whist_off + sizeof(uint32_t) * NW * 256;
  static constexpr size_t tstart_off = gbase_off + sizeof(uint64_t) * 256;
  static constexpr size_t misc_off = tstart_off + sizeof(uint32_t) * 256;
  static constexpr size_t bytes = misc_off + sizeof(uint32_t) * 32;
};

template <typename K, int VB, int KIND, int BLOCK, int KPT>
__global__ void __launch_bounds__(BLOCK) scatter_kernel(Ws ws, int L) {
  using S = ScatterSmem<K, VB, KIND, BLOCK, KPT>;
  using V = typename S::V;
  constexpr int TILE = S::TILE;
  extern __shared__ __align__(16) unsigned char smem[];
  K *keys_s = reinterpret_cast<K *>(smem + S::keys_off);
  V *vals_s = reinterpret_cast<V *>(smem + S::vals_off);
  uint32_t *whist_all = reinterpret_cast<uint32_t *>(smem + S::whist_off);
  uint64_t *gbase = reinterpret_cast<uint64_t *>(smem + S::gbase_off);
  uint32_t *tstart = reinterpret_cast<uint32_t *>(smem + S::tstart_off);
  uint32_t *misc = reinterpret_cast<uint32_t *>(smem + S::misc_off);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int cur = L & 1;
  const uint32_t nt = ws.ctl->ntiles[L];
  if (nt == 0) return;
  const KeyGeom<K, KIND> g{ws.shift0};
  uint32_t *whist = whist_all + w * 256;
  for (;;) {
    if (tid == 0) misc[16] = atomicAdd(&ws.ctl->ticket[L], 1u);
#pragma unroll
    for (int i = lane; i < 256; i += 32) whist[i] = 0;
    __syncthreads();
    const uint32_t t = misc[16];
    if (t >= nt) break;
    const uint32_t b = ws.tile_bucket[cur][t];
    const Bucket bk = ws.buckets[cur][b];
    if (bk.action != ACT_SCATTER) {
      __syncthreads();
      continue;
    }
    const uint32_t tin = t - bk.tile0;
    const uint64_t off = uint64_t(tin) * TILE;
    const uint32_t cnt = uint32_t(min64(TILE, bk.count - off));
    const K *src = static_cast<const K *>(ws.keys[bk.parity]) + bk.start + off;
    K *dst = static_cast<K *>(ws.keys[bk.parity ^ 1]);
    const V *vsrc = VB ? static_cast<const V *>(ws.vals[bk.parity]) + bk.start + off : nullptr;
    V *vdst = VB ? static_cast<V *>(ws.vals[bk.parity ^ 1]) : nullptr;
    const int dig = int(bk.digit);
    const int wbase = w * 32 * KPT;
    const int nvw = max(0, min(32 * KPT, int(cnt) - wbase));
    K x[KPT];
    V v[KPT];
    uint32_t dg[KPT], rk[KPT];
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      const int e = wbase + 32 * j + lane;
      if (e < int(cnt)) {
        x[j] = __ldcs(src + e);
        if constexpr (VB != 0) v[j] = __ldcs(vsrc + e);
      }
    }
#pragma unroll
    for (int j = 0; j < KPT; ++j) dg[j] = g.digit(x[j], dig);
    warp_rank<KPT>(dg, nvw, whist, rk);
    __syncthreads();
    uint32_t total = 0;
    if (tid < 256) {
      uint32_t s = 0;
      for (int ww = 0; ww < S::NW; ++ww) {
        const uint32_t cc = whist_all[ww * 256 + tid];
        whist_all[ww * 256 + tid] = s;
        s += cc;
      }
      total = s;
    }
    const uint32_t texcl = scan256_excl<BLOCK>(total, misc);
    if (tid < 256) {
      tstart[tid] = texcl;
      uint32_t *st = ws.status + size_t(t) * 256 + tid;
      uint32_t prefix = 0;
      if (tin == 0) {
        st_relaxed(st, ST_INCL | total);
      } else {
        st_relaxed(st, ST_AGG | total);
        uint32_t p = t - 1;
        for (;;) {
          const uint32_t sv = ld_relaxed(ws.status + size_t(p) * 256 + tid);
          const uint32_t f = sv & ~ST_MASK;
          if (f == 0) continue;
          prefix += sv & ST_MASK;
          if (f == ST_INCL) break;
          --p;
        }
        st_relaxed(st, ST_INCL | (prefix + total));
      }
      gbase[tid] = bk.start + uint64_t(ws.bhist[cur][size_t(b) * 256 + tid]) + prefix - texcl;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      const int e = wbase + 32 * j + lane;
      if (e < int(cnt)) {
        const uint32_t d = dg[j];
        const uint32_t pos = tstart[d] + whist[d] + rk[j];
        keys_s[pos] = x[j];
        if constexpr (VB != 0) vals_s[pos] = v[j];
      }
    }
    __syncthreads();
#pragma unroll 4
    for (int e = tid; e < int(cnt); e += BLOCK) {
      const K k = keys_s[e];
      const uint64_t o = gbase[g.digit(k, dig)] + uint64_t(e);
      __stcs(dst + o, k);
      if constexpr (VB != 0) __stcs(vdst + o, vals_s[e]);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K4: local sort of one task (<= BLOCK*KPT elements) per CTA iteration.  LSD
// over the task's varying digits only (all-equal digits are the reference's
// pass-throughs), stable, keys (+values) staged through shared memory, final
// pass written to the caller's buffer.
// ---------------------------------------------------------------------------
template <typename K, int VB, int KIND, int BLOCK, int KPT>
struct LocalSmem {
  using V = typename ValT<VB>::T;
  static constexpr int CAP = BLOCK * KPT;
  static constexpr int NW = BLOCK / 32;
  static constexpr size_t keys_off = 0;
  static constexpr size_t vals_off = keys_off + sizeof(K) * CAP;
  static constexpr size_t whist_off = vals_off + (VB ? sizeof(V) * CAP : 0);
  static constexpr size_t tstart_off = whist_off + sizeof(uint32_t) * NW * 256;
  static constexpr size_t red_off = tstart_off + sizeof(uint32_t) * 256;
  static constexpr size_t misc_off = red_off + sizeof(uint64_t) * 2 * NW;
  static constexpr size_t bytes = misc_off + sizeof(uint32_t) * 32;
};

template <typename K, int VB, int KIND, int BLOCK, int KPT>
__global__ void __launch_bounds__(BLOCK) local_kernel(Ws ws) {
  using S = LocalSmem<K, VB, KIND, BLOCK, KPT>;
  using V = typename S::V;
  constexpr int W = KeyTraits<K>::BITS;
  extern __shared__ __align__(16) unsigned char smem[];
  K *keys_s = reinterpret_cast<K *>(smem + S::keys_off);
  V *vals_s = reinterpret_cast<V *>(smem + S::vals_off);
  uint32_t *whist_all = reinterpret_cast<uint32_t *>(smem + S::whist_off);
  uint32_t *tstart = reinterpret_cast<uint32_t *>(smem + S::tstart_off);
  uint64_t *red = reinterpret_cast<uint64_t *>(smem + S::red_off);
  uint32_t *misc = reinterpret_cast<uint32_t *>(smem + S::misc_off);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t ntasks = min(ws.ctl->ntasks, ws.maxtasks);
  const KeyGeom<K, KIND> g{ws.shift0};
  uint32_t *whist = whist_all + w * 256;
  const int wbase = w * 32 * KPT;
  for (uint32_t ti = blockIdx.x; ti < ntasks; ti += gridDim.x) {
    const Task tk = ws.tasks[ti];
    const int n = int(tk.count);
    const K *src = static_cast<const K *>(ws.keys[tk.parity]) + tk.start;
    K *dst = static_cast<K *>(ws.keys[0]) + tk.start;
    const V *vsrc = VB ? static_cast<const V *>(ws.vals[tk.parity]) + tk.start : nullptr;
    V *vdst = VB ? static_cast<V *>(ws.vals[0]) + tk.start : nullptr;
    const int nvw = max(0, min(32 * KPT, n - wbase));
    K x[KPT];
    V v[KPT];
    K o = 0, a = ~K(0);
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      const int e = wbase + 32 * j + lane;
      if (e < n) {
        x[j] = src[e];
        if constexpr (VB != 0) v[j] = vsrc[e];
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
    K var;
    {
      K oo = 0, aa = ~K(0);
#pragma unroll
      for (int i = 0; i < S::NW; ++i) {
        oo |= K(red[i]);
        aa &= K(red[S::NW + i]);
      }
      var = oo ^ aa;
    }
    if (var == 0) {
      if (tk.parity) {
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
          const int e = wbase + 32 * j + lane;
          if (e < n) {
            dst[e] = x[j];
            if constexpr (VB != 0) vdst[e] = v[j];
          }
        }
      }
      __syncthreads();
      continue;
    }
    // digits that vary, least significant first
    const int lastd = (W - 1 - (__ffsll((long long)(uint64_t(var))) - 1)) >> 3;
    const int firstd = KeyTraits<K>::clz(var) >> 3;
    bool wrote_smem = false;
    for (int dig = lastd; dig >= firstd; --dig) {
      if (((var >> (W - 8 - 8 * dig)) & K(0xFF)) == 0) continue;
      if (wrote_smem) {
        // reload in element order from the previous pass
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
          const int e = wbase + 32 * j + lane;
          if (e < n) {
            x[j] = keys_s[e];
            if constexpr (VB != 0) v[j] = vals_s[e];
          }
        }
        __syncthreads();
      }
#pragma unroll
      for (int i = lane; i < 256; i += 32) whist[i] = 0;
      __syncwarp();
      uint32_t dg[KPT], rk[KPT];
#pragma unroll
      for (int j = 0; j < KPT; ++j) dg[j] = g.digit(x[j], dig);
      warp_rank<KPT>(dg, nvw, whist, rk);
      __syncthreads();
      uint32_t total = 0;
      if (tid < 256) {
        uint32_t s = 0;
        for (int ww = 0; ww < S::NW; ++ww) {
          const uint32_t cc = whist_all[ww * 256 + tid];
          whist_all[ww * 256 + tid] = s;
          s += cc;
        }
        total = s;
      }
      const uint32_t texcl = scan256_excl<BLOCK>(total, misc);
      if (tid < 256) tstart[tid] = texcl;
      __syncthreads();
#pragma unroll
      for (int j = 0; j < KPT; ++j) {
        const int e = wbase + 32 * j + lane;
        if (e < n) {
          const uint32_t d = dg[j];
          const uint32_t pos = tstart[d] + whist[d] + rk[j];
          keys_s[pos] = x[j];
          if constexpr (VB != 0) vals_s[pos] = v[j];
        }
      }
      __syncthreads();
      wrote_smem = true;
    }
    for (int e = tid; e < n; e += BLOCK) {
      dst[e] = keys_s[e];
      if constexpr (VB != 0) vdst[e] = vals_s[e];
    }
    __syncthreads();
  }
}

}  // namespace bs
