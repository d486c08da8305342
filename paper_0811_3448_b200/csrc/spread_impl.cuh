// spread_impl.cuh -- K4b: local sort of keys-only 64-bit tasks whose keys are
// spread (few equal keys), e.g. cfg3-uniform after two MSD digits: ~4096 keys
// with 48 varying bits per task.
//
// A dense pass on the task's top 16 varying bits ends the reference's
// recursion (kernels.py:88-126) for almost every key at once: each key sets
// its 16-bit prefix in a presence bitmap (B1; a second / third key with the
// same prefix sets B2 / B3), one scan turns the bitmaps into per-word output
// offsets, and every key computes its own output slot from popcounts of the
// words below its bit (no per-bit enumeration: the 64-bit keys cannot be
// regenerated from the bitmap, they are placed).  Keys sharing a prefix (~3 %
// for uniform data) land in one small run, which its owner sorts by the full
// key.  A task with a prefix repeated 4+ times (duplicate-heavy data, Zipf)
// goes to the general local sort's list (local_kernel, tasks2).
//
// Against local_kernel's bin sort (one counting pass + per-key comparison
// loops that diverge with the bin sizes): no comparison loops except the
// rare fix-ups, and two TMA slots so the next task streams in meanwhile.
#pragma once

#include "sort_impl.cuh"

namespace bs {

template <typename K, int BLOCK, int KPT>
struct SpreadSmem {
  static constexpr int CAP = BLOCK * KPT;                               // keys per task (<= local_max; larger ones: local_kernel)
  static constexpr size_t kbuf = (sizeof(K) * CAP + 32 + 15) & ~size_t(15);  // input slot, then staging
  static constexpr size_t buf_off = 0;                                  // two slots: the next task streams in
  static constexpr size_t bins_off = buf_off + 2 * kbuf;                // B1, B2, B3, P: 4 x 2048 words
  static constexpr size_t red_off = bins_off + sizeof(uint32_t) * 4 * 2048;
  static constexpr size_t misc_off = red_off + sizeof(uint64_t) * 2 * (BLOCK / 32);
  static constexpr size_t bar_off = misc_off + sizeof(uint32_t) * 64;
  static constexpr size_t info_off = bar_off + 2 * sizeof(uint64_t);
  static constexpr size_t bytes = info_off + 2 * sizeof(InFlight);
};

__device__ __forceinline__ void push_task2(const Ws &ws, uint64_t start, uint32_t count, uint32_t parity) {
  const uint32_t slot = atomicAdd(&ws.ctl->ntasks2, 1u);
  if (slot < ws.maxtasks) ws.tasks2[slot] = Task{start, count, parity};
  else atomicOr(&ws.ctl->error, 4u);
}

template <typename K, int KIND, int BLOCK, int KPT>
__global__ void __launch_bounds__(BLOCK, BLOCK <= 512 ? 2 : 1) spread_kernel(Ws ws) {
  static_assert(BLOCK >= 512, "threads 0..511 own the bitmap words");
  pdl_wait();  // programmatic dependent launch: previous kernel's writes visible
  if (ws_failed(ws)) return;
  using S = SpreadSmem<K, BLOCK, KPT>;
  constexpr int W = KeyTraits<K>::BITS;
  extern __shared__ __align__(128) unsigned char smem[];
  uint32_t *binw = reinterpret_cast<uint32_t *>(smem + S::bins_off);  // bin p: half (p & 1) of word p >> 1
  uint64_t *red = reinterpret_cast<uint64_t *>(smem + S::red_off);
  uint32_t *misc = reinterpret_cast<uint32_t *>(smem + S::misc_off);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + S::bar_off);
  InFlight *info = reinterpret_cast<InFlight *>(smem + S::info_off);
  const int tid = threadIdx.x;
  const uint32_t ntasks = min(ws.ctl->ntasks, ws.maxtasks);
  if (blockIdx.x >= ntasks || ws.ctl->skewed) return;  // skewed input: local_kernel takes every task
  const KeyGeom<K, KIND> g{ws.shift0};
  auto slot_keys = [&](int sl) { return reinterpret_cast<K *>(smem + S::buf_off + size_t(sl) * S::kbuf); };
  auto load = [&](int sl, uint32_t ti) {  // thread 0: stream task ti into slot sl
    InFlight f{};
    f.idx = ti;
    if (ti < ntasks) {
      const Task tk = ws.tasks[ti];
      f.start = tk.start;
      f.cnt = tk.count;
      f.parity = tk.parity & 1u;
      f.digit = tk.parity >> 8;  // first digit that may vary: the prefix is it and the next one
      f.valid = tk.count <= uint32_t(S::CAP);  // larger local tasks go to local_kernel
      if (f.valid) {
        const Span sk = span16(static_cast<const K *>(ws.keys[f.parity]) + f.start, f.cnt);
        f.headk = sk.head;
        info[sl] = f;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&bars[sl], sk.bytes);
        bulk_g2s(slot_keys(sl), sk.base, sk.bytes, &bars[sl]);
      } else {
        info[sl] = f;
        mbar_arrive(&bars[sl]);
      }
    } else {
      info[sl] = f;
    }
  };
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    load(0, blockIdx.x);
  }
  uint32_t phase = 0;
  int cur = 0;
  for (uint32_t ti = blockIdx.x; ti < ntasks; ti += gridDim.x, cur ^= 1) {
    __syncthreads();  // the other slot is free (its task is stored); info[cur] visible
    if (tid == 0) load(cur ^ 1, ti + gridDim.x);
    mbar_wait(&bars[cur], (phase >> cur) & 1u);
    phase ^= 1u << cur;
    K *kb = slot_keys(cur);
    const InFlight f = info[cur];
    if (!f.valid) {  // more keys than a slot holds
      if (tid == 0) push_task2(ws, f.start, f.cnt, f.parity);
      continue;
    }
    const int n = int(f.cnt);
    const int head = int(f.headk);
    // keys in registers: element tid + j*BLOCK (strided: conflict-free)
    K x[KPT];
    uint32_t valid = 0;
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      if (j * BLOCK >= n) break;  // block-uniform: no work past the task's last key
      const int e = tid + j * BLOCK;
      x[j] = 0;
      if (e < n) {
        x[j] = kb[head + e];
        valid |= 1u << j;
      }
    }
    K *dst = static_cast<K *>(ws.keys[0]) + f.start;
    // prefix = the task's first two possibly-varying digits (the digits above
    // them are shared by the task's keys).  If they are constant after all,
    // every key lands on one prefix and the task is handed on below.
    const int sh = max(W - 8 * int(f.digit) - 16, 0);
    uint32_t *B1 = binw, *B2 = binw + 2048, *B3 = binw + 4096, *P = binw + 6144;
    for (int i = tid; i < 3 * 2048 / 4; i += BLOCK) reinterpret_cast<uint4 *>(binw)[i] = make_uint4(0, 0, 0, 0);
    if (tid == 0) misc[40] = 0;
    __syncthreads();
    // insert: copy index per key (2 bits): 0 first, 1 second, 2 third of its prefix
    uint32_t cpy = 0;
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      if (j * BLOCK >= n) break;
      if ((valid >> j) & 1u) {
        const uint32_t idx = uint32_t(g.norm(x[j]) >> sh) & 0xFFFFu;
        const uint32_t bit = 1u << (idx & 31u);
        uint32_t ci = 0;
        if (atomicOr(&B1[idx >> 5], bit) & bit) {
          ci = 1;
          if (atomicOr(&B2[idx >> 5], bit) & bit) {
            ci = 2;
            if (atomicOr(&B3[idx >> 5], bit) & bit) misc[40] = 1;  // a 4th copy: not this path
          }
        }
        cpy |= ci << (2 * j);
      }
    }
    __syncthreads();  // bitmaps complete
    if (misc[40]) {  // duplicate-heavy: the general local sort takes it
      if (tid == 0) push_task2(ws, f.start, f.cnt, f.parity);
      continue;
    }
    // word offsets: thread t < 512 owns words 4t..4t+3 (BLOCK >= 512); P[q] = keys before word q
    // (| bit 31 when the word holds a repeated prefix)
    {
      const bool own = tid < 512;
      uint4 b1 = make_uint4(0, 0, 0, 0), b2 = b1, b3 = b1;
      if (own) {
        b1 = reinterpret_cast<const uint4 *>(B1)[tid];
        b2 = reinterpret_cast<const uint4 *>(B2)[tid];
        b3 = reinterpret_cast<const uint4 *>(B3)[tid];
      }
      const uint32_t c0 = __popc(b1.x) + __popc(b2.x) + __popc(b3.x), c1 = __popc(b1.y) + __popc(b2.y) + __popc(b3.y);
      const uint32_t c2 = __popc(b1.z) + __popc(b2.z) + __popc(b3.z), c3 = __popc(b1.w) + __popc(b2.w) + __popc(b3.w);
      const uint32_t pos = block_scan_excl<BLOCK>(c0 + c1 + c2 + c3, misc);
      if (own) {
        const uint32_t r0 = b2.x ? 0x80000000u : 0u, r1 = b2.y ? 0x80000000u : 0u;
        const uint32_t r2 = b2.z ? 0x80000000u : 0u, r3 = b2.w ? 0x80000000u : 0u;
        reinterpret_cast<uint4 *>(P)[tid] =
            make_uint4(pos | r0, (pos + c0) | r1, (pos + c0 + c1) | r2, (pos + c0 + c1 + c2) | r3);
      }
    }
    __syncthreads();  // offsets visible
    // placement: P[q] + keys of smaller prefixes in the word + copy index
    uint32_t fin[KPT];
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      if (j * BLOCK >= n) break;
      if ((valid >> j) & 1u) {
        const uint32_t idx = uint32_t(g.norm(x[j]) >> sh) & 0xFFFFu;
        const uint32_t q = idx >> 5, m = (1u << (idx & 31u)) - 1u;
        const uint32_t pw = P[q];
        uint32_t r = (pw & 0x7FFFFFFFu) + uint32_t(__popc(B1[q] & m)) + ((cpy >> (2 * j)) & 3u);
        if (pw >> 31) r += uint32_t(__popc(B2[q] & m) + __popc(B3[q] & m));
        fin[j] = r;
      }
    }
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      if (j * BLOCK >= n) break;
      if ((valid >> j) & 1u) {
        BS_DCHECK(ws.ctl, fin[j] < uint32_t(n));
        kb[fin[j]] = x[j];
      }
    }
    __syncthreads();  // keys in prefix order
    // fix-up: each run of 2-3 keys sharing a prefix is sorted by the full key (owner of its word)
    if (tid < 512) {
      const uint4 b2 = reinterpret_cast<const uint4 *>(B2)[tid];
      if (b2.x | b2.y | b2.z | b2.w) {
        const uint4 b1 = reinterpret_cast<const uint4 *>(B1)[tid];
        const uint4 b3 = reinterpret_cast<const uint4 *>(B3)[tid];
        const uint4 pw = reinterpret_cast<const uint4 *>(P)[tid];
        const uint32_t w1[4] = {b1.x, b1.y, b1.z, b1.w}, w2[4] = {b2.x, b2.y, b2.z, b2.w};
        const uint32_t w3[4] = {b3.x, b3.y, b3.z, b3.w}, p4[4] = {pw.x, pw.y, pw.z, pw.w};
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          uint32_t m2 = w2[jj];
          while (m2) {
            const uint32_t b = __ffs(m2) - 1u;
            m2 &= m2 - 1u;
            const uint32_t m = (1u << b) - 1u;
            const uint32_t r0 = (p4[jj] & 0x7FFFFFFFu) + __popc(w1[jj] & m) + __popc(w2[jj] & m) + __popc(w3[jj] & m);
            const uint32_t c = 2u + ((w3[jj] >> b) & 1u);
            K a0 = kb[r0], a1 = kb[r0 + 1];
            K n0 = g.norm(a0), n1 = g.norm(a1);
            if (n1 < n0) {
              const K t = a0; a0 = a1; a1 = t;
              const K u = n0; n0 = n1; n1 = u;
            }
            if (c == 3u) {
              K a2 = kb[r0 + 2];
              const K n2 = g.norm(a2);
              if (n2 < n1) {
                const K t = a1; a1 = a2; a2 = t;
                if (n2 < n0) {
                  const K v = a0; a0 = a1; a1 = v;
                }
              }
              kb[r0 + 2] = a2;
            }
            kb[r0] = a0;
            kb[r0 + 1] = a1;
          }
        }
      }
    }
    __syncthreads();  // sorted in shared memory
    BS_DCHECK(ws.ctl, f.start + uint64_t(n) <= ws.n);
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      if (j * BLOCK >= n) break;
      const int e = tid + j * BLOCK;
      if (e < n) __stcs(dst + e, kb[e]);
    }
  }
}

}  // namespace bs
